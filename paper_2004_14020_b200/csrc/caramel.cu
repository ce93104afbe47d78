// caramel.cu -- sm_100a kernels + C ABI for the data-parallel aggregation
// hot path (fusion-bucket pack, chunked ring / halving-doubling / two-shot
// all-reduce over NVLink peer memory, postponed SGD update fused into the
// all-gather epilogue).  See include/caramel.h for the contract and DESIGN.md
// for the data layout.
//
// Reference semantics followed (all under /root/reference/pkg/src/overlapsim):
//   bucket membership / member order ..... batching.py:76,122 (BatchGroup.param_ids)
//   chunking into `depth` pieces ......... collective.py:18-21,121-124
//   per-stage bytes of each pattern ....... collective.py:86-103 (stage_plan)
//   depth cap ............................ collective.py:32 (MAX_DEPTH = 8)
//   worker-count validation .............. collective.py:77-83
//   postponed update ..................... transfer.py:156-160
//
// Layout (per rank; every rank allocates identical sizes so offsets are
// symmetric): one "bucket arena" = [bucket buffers | flag blocks], plus an
// optional parameter arena.  Peers' arenas are mapped with CUDA IPC; all
// cross-rank traffic is plain ld/st on the mapped addresses (NVLink 5 via
// NVSwitch).  Flags are 32-bit epochs written by the producer into the
// consumer's flag block with st.release.sys and polled with ld.acquire.sys.

#include <cuda.h>  // stream memory-op types; entry points come from cudaGetDriverEntryPoint
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <stdarg.h>
#include <sys/socket.h>
#include <sys/un.h>
#include <unistd.h>
#include <errno.h>

#include <condition_variable>
#include <deque>
#include <new>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/caramel.h"

#define THREADS 512
#define MAXR CARAMEL_MAX_RANKS
#define SYNC_BYTES (64 * 1024)  // per-arena library sync words (grid barriers)
#define MAX_FUSED_BUCKETS 2048

// ---------------------------------------------------------------------------
// error plumbing (host)
// ---------------------------------------------------------------------------
static thread_local char g_err[512] = "";

static int set_err(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

#define CUDA_TRY(expr)                                                       \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess)                                                   \
      return set_err(CARAMEL_ECUDA, "%s failed: %s (%s:%d)", #expr,          \
                     cudaGetErrorString(_e), __FILE__, __LINE__);            \
  } while (0)

// ---------------------------------------------------------------------------
// device helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t split_at(uint64_t n, uint64_t parts, uint64_t i) {
  // floor(i * n / parts): the integer chunk/shard rule;
  // 32-bit division when the product fits (the common case, and a fraction of
  // the cost of the 64-bit division routine the fused kernel ran per item)
  const uint64_t x = n * i;
  return x <= 0xffffffffull ? (uint64_t)((uint32_t)x / (uint32_t)parts) : x / parts;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_relaxed_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

__device__ __forceinline__ uint32_t atom_add_acq_rel_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void st_u64_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_u64_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ float4 ld4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }
__device__ __forceinline__ void st4(float* p, float4 v) { __stcg(reinterpret_cast<float4*>(p), v); }
__device__ __forceinline__ float ld1(const float* p) { return __ldcg(p); }
__device__ __forceinline__ void st1(float* p, float v) { __stcg(p, v); }

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                     __fadd_rn(a.w, b.w));
}

// Epilogue applied by the shard owner.  Separate roundings, never an FMA, so
// the CPU oracle (numpy / C with -ffp-contract=off) is matched bit for bit.
__device__ __forceinline__ float epi1(int epi, float s, float theta, float scale, float lr) {
  if (epi == CARAMEL_EPI_SUM) return s;
  float g = __fmul_rn(s, scale);
  if (epi == CARAMEL_EPI_SCALE) return g;
  return __fsub_rn(theta, __fmul_rn(lr, g));
}

__device__ __forceinline__ float4 epi4(int epi, float4 s, float4 t, float scale, float lr) {
  return make_float4(epi1(epi, s.x, t.x, scale, lr), epi1(epi, s.y, t.y, scale, lr),
                     epi1(epi, s.z, t.z, scale, lr), epi1(epi, s.w, t.w, scale, lr));
}

// Segment cursor: maps a bucket element position to its member tensor.
// Segments are sorted by offset and tile [0, numel) without gaps.
struct Cursor {
  const caramel_segment* s;
  int n;
  int i;
  uint64_t lo, hi, g, p;
};

__device__ __forceinline__ void cur_init(Cursor& c, const caramel_segment* s, int n) {
  c.s = s;
  c.n = n;
  c.i = -1;
  c.lo = 1;
  c.hi = 0;
  c.g = 0;
  c.p = 0;
}

__device__ __forceinline__ void cur_load(Cursor& c, int i) {
  const unsigned long long* e = reinterpret_cast<const unsigned long long*>(c.s + i);
  c.i = i;
  c.g = __ldg(e + 0);
  c.p = __ldg(e + 1);
  c.lo = __ldg(e + 2);
  c.hi = c.lo + __ldg(e + 3);
}

__device__ __forceinline__ void cur_seek(Cursor& c, uint64_t pos) {
  if (pos >= c.lo && pos < c.hi) return;
  int a = 0, b = c.n - 1;
  if (c.i >= 0 && pos >= c.hi) {
    if (c.i + 1 < c.n) {
      cur_load(c, c.i + 1);  // common case: the next member
      if (pos < c.hi) return;
    }
    a = c.i;
  }
  while (a < b) {
    int m = (a + b + 1) >> 1;
    uint64_t off = __ldg(reinterpret_cast<const unsigned long long*>(c.s + m) + 2);
    if (off <= pos) a = m; else b = m - 1;
  }
  cur_load(c, a);
}

// which: 0 = member .grad, 1 = member .param
__device__ __forceinline__ float seg_ld1(Cursor& c, uint64_t pos, int which) {
  cur_seek(c, pos);
  const float* b = reinterpret_cast<const float*>(which ? c.p : c.g);
  return ld1(b + (pos - c.lo));
}

__device__ __forceinline__ void seg_st1(Cursor& c, uint64_t pos, int which, float v) {
  cur_seek(c, pos);
  float* b = reinterpret_cast<float*>(which ? c.p : c.g);
  st1(b + (pos - c.lo), v);
}

__device__ __forceinline__ float4 seg_ld4(Cursor& c, uint64_t v, int which) {
  cur_seek(c, v);
  const float* ptr = reinterpret_cast<const float*>(which ? c.p : c.g) + (v - c.lo);
  if (v + 4 <= c.hi && (reinterpret_cast<uintptr_t>(ptr) & 15) == 0) return ld4(ptr);
  float4 r;
  r.x = seg_ld1(c, v + 0, which);
  r.y = seg_ld1(c, v + 1, which);
  r.z = seg_ld1(c, v + 2, which);
  r.w = seg_ld1(c, v + 3, which);
  return r;
}

__device__ __forceinline__ void seg_st4(Cursor& c, uint64_t v, int which, float4 x) {
  cur_seek(c, v);
  float* ptr = reinterpret_cast<float*>(which ? c.p : c.g) + (v - c.lo);
  if (v + 4 <= c.hi && (reinterpret_cast<uintptr_t>(ptr) & 15) == 0) {
    st4(ptr, x);
    return;
  }
  seg_st1(c, v + 0, which, x.x);
  seg_st1(c, v + 1, which, x.y);
  seg_st1(c, v + 2, which, x.z);
  seg_st1(c, v + 3, which, x.w);
}

// Segment pieces: call f(seg, a, b) for every member segment overlapping the
// bucket range [lo, hi), with [a, b) the overlap in bucket coordinates.  One
// binary search per range, then a forward walk; the hot loops below run on
// fixed base pointers (no per-vector segment lookup).
struct Seg {
  uint64_t grad, param, offset, numel;
};

__device__ __forceinline__ Seg load_seg(const caramel_segment* s, int i) {
  const unsigned long long* e = reinterpret_cast<const unsigned long long*>(s + i);
  Seg r;
  r.grad = __ldg(e + 0);
  r.param = __ldg(e + 1);
  r.offset = __ldg(e + 2);
  r.numel = __ldg(e + 3);
  return r;
}

template <class F>
__device__ __forceinline__ void for_pieces(const caramel_segment* segs, int nseg, uint64_t lo, uint64_t hi, F f) {
  if (lo >= hi) return;
  int a = 0, b = nseg - 1;
  while (a < b) {
    int m = (a + b + 1) >> 1;
    uint64_t off = __ldg(reinterpret_cast<const unsigned long long*>(segs + m) + 2);
    if (off <= lo) a = m; else b = m - 1;
  }
  for (int i = a; i < nseg; ++i) {
    const Seg sg = load_seg(segs, i);
    if (sg.offset >= hi) break;
    const uint64_t x = lo > sg.offset ? lo : sg.offset;
    const uint64_t y = hi < sg.offset + sg.numel ? hi : sg.offset + sg.numel;
    if (x < y) f(sg, x, y);
  }
}

// Elements before all of the given pointers are 16-byte aligned, or n if they
// can never be aligned together (then the whole range goes scalar).
__device__ __forceinline__ uint64_t co_align_head(uint64_t n, uintptr_t p0, uintptr_t p1, uintptr_t p2) {
  if (((p0 ^ p1) & 15) || ((p0 ^ p2) & 15) || (p0 & 3)) return n;
  uint64_t h = ((16 - (p0 & 15)) & 15) >> 2;
  return h < n ? h : n;
}

// out[i] = epilogue(g[i], theta[i]) for i < n (theta may alias out).  Four
// float4 per thread per trip, all loads issued before the stores.
__device__ __forceinline__ void stream_epi(const float* g, const float* th, float* out, uint64_t n, int epi,
                                           float scale, float lr) {
  const bool sgd = epi == CARAMEL_EPI_SGD;
  const uint64_t head = co_align_head(n, (uintptr_t)g, sgd ? (uintptr_t)th : (uintptr_t)g, (uintptr_t)out);
  for (uint64_t i = threadIdx.x; i < head; i += blockDim.x)
    out[i] = epi1(epi, ld1(g + i), sgd ? ld1(th + i) : 0.f, scale, lr);
  const uint64_t nv = (n - head) >> 2;  // float4 count
  const float4* g4 = reinterpret_cast<const float4*>(g + head);
  const float4* t4 = reinterpret_cast<const float4*>(th + head);
  float4* o4 = reinterpret_cast<float4*>(out + head);
  constexpr int U = 4;
  const uint64_t T = blockDim.x;
  uint64_t v = threadIdx.x;
  for (; v + (U - 1) * T < nv; v += U * T) {
    float4 x[U], t[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = __ldcs(g4 + v + u * T);
#pragma unroll
    for (int u = 0; u < U; ++u) t[u] = sgd ? __ldcg(t4 + v + u * T) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcg(o4 + v + u * T, epi4(epi, x[u], t[u], scale, lr));
  }
  for (; v < nv; v += T) {
    float4 t = sgd ? __ldcg(t4 + v) : make_float4(0.f, 0.f, 0.f, 0.f);
    __stcg(o4 + v, epi4(epi, __ldcs(g4 + v), t, scale, lr));
  }
  for (uint64_t i = head + 4 * nv + threadIdx.x; i < n; i += blockDim.x)
    out[i] = epi1(epi, ld1(g + i), sgd ? ld1(th + i) : 0.f, scale, lr);
}

// dst[i] = src[i] for i < n, vectorised when co-aligned.
__device__ __forceinline__ void copy_n(const float* src, float* dst, uint64_t n) {
  const uint64_t head = co_align_head(n, (uintptr_t)src, (uintptr_t)src, (uintptr_t)dst);
  for (uint64_t i = threadIdx.x; i < head; i += blockDim.x) st1(dst + i, ld1(src + i));
  const uint64_t nv = (n - head) >> 2;
  const float4* s4 = reinterpret_cast<const float4*>(src + head);
  float4* d4 = reinterpret_cast<float4*>(dst + head);
  constexpr int U = 4;
  const uint64_t T = blockDim.x;
  uint64_t v = threadIdx.x;
  for (; v + (U - 1) * T < nv; v += U * T) {
    float4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = __ldcg(s4 + v + u * T);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcg(d4 + v + u * T, x[u]);
  }
  for (; v < nv; v += T) __stcg(d4 + v, __ldcg(s4 + v));
  for (uint64_t i = head + 4 * nv + threadIdx.x; i < n; i += blockDim.x) st1(dst + i, ld1(src + i));
}

// ---------------------------------------------------------------------------
// Warp-item engine for member pieces (pack, unpack, single-rank update).
// A CTA's range overlaps a run of member segments ("pieces").  Thread i
// describes piece i (pointers, length, epilogue), a block scan lays the
// pieces out as items of 128 float4 (512 elements) and warps take items
// round-robin: many small members are in flight at once instead of one
// block-wide loop -- one memory round trip -- per member.
// ---------------------------------------------------------------------------
enum { OP_COPY = 0, OP_EPI = 1 };

struct PieceDesc {
  const float* g;  // source: gradient member or bucket
  const float* t;  // theta (SGD epilogue only)
  float* o;        // destination
  uint32_t n;      // elements (0: no piece)
  int epi;
  float scale, lr;
};

struct PieceTab {
  const float* g[THREADS];
  const float* t[THREADS];
  float* o[THREADS];
  uint32_t n[THREADS];
  uint32_t head[THREADS];       // scalar elements before the aligned body; ~0u = all-scalar piece
  uint32_t first[THREADS + 1];  // item prefix
  int epi[THREADS];
  float scale[THREADS], lr[THREADS];
  uint32_t scratch[32];
};

__shared__ PieceTab g_tab;  // one per CTA (static shared memory of the kernels that touch members)

__device__ __forceinline__ int first_seg(const caramel_segment* segs, int nseg, uint64_t pos) {
  int a = 0, b = nseg - 1;
  while (a < b) {
    int m = (a + b + 1) >> 1;
    uint64_t off = __ldg(reinterpret_cast<const unsigned long long*>(segs + m) + 2);
    if (off <= pos) a = m; else b = m - 1;
  }
  return a;
}

// block-wide exclusive scan of one uint32 per thread; returns the total
__device__ __forceinline__ uint32_t block_scan(uint32_t x, uint32_t* out_excl, uint32_t* scratch) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t v = x;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += y;
  }
  if (lane == 31) scratch[w] = v;
  __syncthreads();
  if (w == 0) {
    uint32_t s = lane < nw ? scratch[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s, d);
      if (lane >= d) s += y;
    }
    if (lane < nw) scratch[lane] = s;  // inclusive warp totals
  }
  __syncthreads();
  *out_excl = (w ? scratch[w - 1] : 0) + v - x;
  const uint32_t total = scratch[nw - 1];
  __syncthreads();
  return total;
}

__device__ __forceinline__ float apply1(int op, int epi, float g, float t, float scale, float lr) {
  return op == OP_EPI ? epi1(epi, g, t, scale, lr) : g;
}

// Pieces [0, npieces): desc(i, PieceDesc&) fills piece i (n = 0 for none).
template <int OP, class Desc>
__device__ void run_pieces(int npieces, Desc desc, PieceTab& tab) {
  for (int base = 0; base < npieces; base += blockDim.x) {
    const int i = base + threadIdx.x;
    PieceDesc d;
    d.n = 0;
    d.g = d.t = nullptr;
    d.o = nullptr;
    d.epi = CARAMEL_EPI_SUM;
    d.scale = d.lr = 0.f;
    if (i < npieces) desc(i, d);
    const bool sgd = OP == OP_EPI && d.epi == CARAMEL_EPI_SGD;
    uint32_t items = 0, head = 0;
    if (d.n) {
      const uint32_t h = (uint32_t)co_align_head(d.n, (uintptr_t)d.g, sgd ? (uintptr_t)d.t : (uintptr_t)d.g,
                                                 (uintptr_t)d.o);
      if (h == d.n) {  // never co-aligned: scalar items of 512 elements
        head = ~0u;
        items = (d.n + 511) / 512;
      } else {
        head = h;
        items = (((d.n - h) >> 2) + 127) / 128;
      }
    }
    uint32_t excl;
    const uint32_t total = block_scan(items, &excl, tab.scratch);
    tab.g[threadIdx.x] = d.g;
    tab.t[threadIdx.x] = d.t;
    tab.o[threadIdx.x] = d.o;
    tab.n[threadIdx.x] = d.n;
    tab.head[threadIdx.x] = head;
    tab.first[threadIdx.x] = excl;
    tab.epi[threadIdx.x] = d.epi;
    tab.scale[threadIdx.x] = d.scale;
    tab.lr[threadIdx.x] = d.lr;
    if (threadIdx.x == blockDim.x - 1) tab.first[blockDim.x] = total;
    // scalar head / tail of this thread's own vector piece (<= 3 + 3 elements)
    if (d.n && head != ~0u) {
      const uint32_t tail = head + 4 * ((d.n - head) >> 2);
      for (uint32_t e = 0; e < head; ++e) d.o[e] = apply1(OP, d.epi, ld1(d.g + e), sgd ? ld1(d.t + e) : 0.f, d.scale, d.lr);
      for (uint32_t e = tail; e < d.n; ++e) d.o[e] = apply1(OP, d.epi, ld1(d.g + e), sgd ? ld1(d.t + e) : 0.f, d.scale, d.lr);
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int pc = 0;
    for (uint32_t it = w; it < total; it += nw) {
      while (tab.first[pc + 1] <= it) ++pc;
      const uint32_t k = it - tab.first[pc];
      const float* pg = tab.g[pc];
      const float* pt = tab.t[pc];
      float* po = tab.o[pc];
      const uint32_t pn = tab.n[pc], hd = tab.head[pc];
      const int epi = tab.epi[pc];
      const float scale = tab.scale[pc], lr = tab.lr[pc];
      const bool psgd = OP == OP_EPI && epi == CARAMEL_EPI_SGD;
      if (hd == ~0u) {  // scalar item: elements [512k, 512k + 512)
        const uint32_t e0 = 512 * k;
        float x[16], y[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const uint32_t e = e0 + lane + 32 * u;
          x[u] = e < pn ? ld1(pg + e) : 0.f;
          y[u] = (psgd && e < pn) ? ld1(pt + e) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const uint32_t e = e0 + lane + 32 * u;
          if (e < pn) po[e] = apply1(OP, epi, x[u], y[u], scale, lr);
        }
      } else {  // vector item: float4 [128k, 128k + 128) of the aligned body
        const uint32_t nv = (pn - hd) >> 2;
        const float4* g4 = reinterpret_cast<const float4*>(pg + hd);
        const float4* t4 = reinterpret_cast<const float4*>(pt + hd);
        float4* o4 = reinterpret_cast<float4*>(po + hd);
        const uint32_t v0 = 128 * k;
        float4 x[4], y[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t v = v0 + lane + 32 * u;
          x[u] = v < nv ? __ldcs(g4 + v) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t v = v0 + lane + 32 * u;
          y[u] = (psgd && v < nv) ? __ldcg(t4 + v) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t v = v0 + lane + 32 * u;
          if (v < nv) __stcg(o4 + v, OP == OP_EPI ? epi4(epi, x[u], y[u], scale, lr) : x[u]);
        }
      }
    }
    __syncthreads();  // tab is rewritten by the next batch
  }
}

// The member segments of one bucket overlapping bucket range [lo, hi):
// piece i is segment seg0 + i.  Returns seg0 and the count.
__device__ __forceinline__ int seg_span(const caramel_segment* segs, int nseg, uint64_t lo, uint64_t hi, int& seg0) {
  if (lo >= hi || nseg < 1) {
    seg0 = 0;
    return 0;
  }
  seg0 = first_seg(segs, nseg, lo);
  const int last = first_seg(segs, nseg, hi - 1);
  return last - seg0 + 1;
}

// piece [x0, x1) (bucket coordinates) of segment sg clipped to [lo, hi); false if empty
__device__ __forceinline__ bool clip_seg(const Seg& sg, uint64_t lo, uint64_t hi, uint64_t& x0, uint64_t& x1) {
  x0 = lo > sg.offset ? lo : sg.offset;
  x1 = hi < sg.offset + sg.numel ? hi : sg.offset + sg.numel;
  return x0 < x1;
}

// pack: bucket[lo, hi) <- member grads
__device__ __forceinline__ void pack_range(const caramel_segment* segs, int nseg, float* bucket, uint64_t lo,
                                           uint64_t hi, PieceTab& tab) {
  int seg0;
  const int np = seg_span(segs, nseg, lo, hi, seg0);
  run_pieces<OP_COPY>(np, [&](int i, PieceDesc& d) {
    const Seg sg = load_seg(segs, seg0 + i);
    uint64_t x0, x1;
    if (!clip_seg(sg, lo, hi, x0, x1)) return;
    d.g = reinterpret_cast<const float*>(sg.grad) + (x0 - sg.offset);
    d.o = bucket + x0;
    d.n = (uint32_t)(x1 - x0);
  }, tab);
}

// unpack: member grads (to_param = 0) or params <- bucket[lo, hi)
__device__ __forceinline__ void unpack_range(const caramel_segment* segs, int nseg, const float* bucket,
                                             uint64_t lo, uint64_t hi, bool to_param, PieceTab& tab) {
  int seg0;
  const int np = seg_span(segs, nseg, lo, hi, seg0);
  run_pieces<OP_COPY>(np, [&](int i, PieceDesc& d) {
    const Seg sg = load_seg(segs, seg0 + i);
    uint64_t x0, x1;
    if (!clip_seg(sg, lo, hi, x0, x1)) return;
    d.g = bucket + x0;
    d.o = reinterpret_cast<float*>(to_param ? sg.param : sg.grad) + (x0 - sg.offset);
    d.n = (uint32_t)(x1 - x0);
  }, tab);
}

// Cut [lo, hi) into `parts` tiles whose interior cuts fall on absolute
// 4-element boundaries (so tile interiors vectorise); tile `j` is returned.
__device__ __forceinline__ void tile_of(uint64_t lo, uint64_t hi, int parts, int j,
                                        uint64_t& tlo, uint64_t& thi) {
  auto cut = [&](int k) -> uint64_t {
    if (k <= 0) return lo;
    if (k >= parts) return hi;
    uint64_t x = lo + split_at(hi - lo, parts, k);
    x = (x + 3) & ~3ull;
    return x < hi ? x : hi;
  };
  tlo = cut(j);
  thi = cut(j + 1);
  if (thi < tlo) thi = tlo;
}

// Visit [lo, hi): scalar head up to a 4-aligned position, float4 body, scalar tail.
template <class FV, class FS>
__device__ __forceinline__ void walk(uint64_t lo, uint64_t hi, FV fv, FS fs) {
  if (lo >= hi) return;
  uint64_t a = (lo + 3) & ~3ull;
  if (a > hi) a = hi;
  uint64_t b = hi & ~3ull;
  if (b < a) b = a;
  for (uint64_t i = lo + threadIdx.x; i < a; i += blockDim.x) fs(i);
  for (uint64_t v = a + 4ull * threadIdx.x; v < b; v += 4ull * blockDim.x) fv(v);
  for (uint64_t i = b + threadIdx.x; i < hi; i += blockDim.x) fs(i);
}

// ---------------------------------------------------------------------------
// K1 / K4 standalone: pack and unpack
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(THREADS, 4) k_pack(const caramel_segment* segs, int nseg,
                                                  uint64_t numel, float* bucket) {
  uint64_t lo, hi;
  tile_of(0, numel, gridDim.x, blockIdx.x, lo, hi);
  pack_range(segs, nseg, bucket, lo, hi, g_tab);
}

__global__ void __launch_bounds__(THREADS, 4) k_unpack(const caramel_segment* segs, int nseg,
                                                    uint64_t numel, const float* bucket,
                                                    int to_param) {
  uint64_t lo, hi;
  tile_of(0, numel, gridDim.x, blockIdx.x, lo, hi);
  unpack_range(segs, nseg, bucket, lo, hi, to_param != 0, g_tab);
}

// ---------------------------------------------------------------------------
// the bucket collective: shared by single-bucket and multi-bucket launches
// ---------------------------------------------------------------------------
struct Env {
  uint64_t arena[MAXR];   // bucket arena base of every rank, mapped on this device
  uint64_t parena[MAXR];  // parameter arena base of every rank (0 if none)
  int world;
  int rank_base;          // first rank hosted by this launch (blockIdx.y adds)
  uint32_t epoch;         // 0: read *epoch_dev (graph-replayable launches)
  uint32_t* epoch_dev;    // [0] device epoch counter, [1] CTAs finished (CARAMEL_F_AUTO_EPOCH)
  uint64_t timeout_ns;
  int* status;            // device status word: 0, or CARAMEL_ETIMEOUT (sticky: the context is poisoned)
  int* hstatus;           // host-mapped mirror of *status (caramel_poll reads it without a sync)
  uint64_t sync_off;      // library sync words, past the user part of every arena
};

// ---- watchdog / abort ---------------------------------------------------------
// A flag wait that exceeds the watchdog poisons the context: the status word
// is set (device + host-mapped mirror) and every CTA that was waiting, or that
// starts afterwards, leaves the kernel before its next store -- no epilogue
// ever writes a result computed from inputs that had not arrived.
__device__ __forceinline__ bool poisoned(const Env& E) { return *reinterpret_cast<volatile int*>(E.status) != 0; }

__device__ __noinline__ void raise_timeout(const Env& E) {
  atomicExch(E.status, CARAMEL_ETIMEOUT);
  if (E.hstatus) {
    *reinterpret_cast<volatile int*>(E.hstatus) = CARAMEL_ETIMEOUT;
    __threadfence_system();
  }
}

// every thread of the CTA calls: leaves the kernel (all threads together) if
// any thread's wait failed.  `exit` after a CTA-uniform barrier result.
__device__ __forceinline__ void cta_abort_if(int failed) {
  if (__syncthreads_or(failed)) asm volatile("exit;");
}

// CTA-uniform entry check of the kernels that wait on peers: true = leave
// (the caller returns; an `exit` this early cost the single-bucket kernel
// 40% of its NVLink bandwidth -- measured, cause in the compiler's layout)
__device__ __forceinline__ bool cta_poisoned(const Env& E) { return __syncthreads_or(threadIdx.x == 0 && poisoned(E)); }

struct KParams {          // one bucket
  Env env;
  caramel_bucket b;
};

struct MParams {          // a list of buckets, processed in launch order
  Env env;
  const caramel_bucket* bs;
  const uint64_t* prefix;    // element prefix sums, prefix[i+1] - prefix[i] = bs[i].numel (absolute)
  const uint64_t* segprefix; // member-segment prefix sums (absolute)
  int nb;
  int claim;                 // k_shuffle_fused: items a warp claims per atomic (0 = static split)
};

// flag slots
#define SLOT_READY 0
#define SLOT_DONE 1  // shuffle

__host__ __device__ __forceinline__ int ilog2i(int p) {
  int l = 0;
  while ((1 << l) < p) ++l;
  return l;
}

__host__ __device__ __forceinline__ int nslots(int pattern, int world) {
  if (pattern == CARAMEL_SHUFFLE) return 2;
  if (pattern == CARAMEL_RING) return 2 * world;           // ready, 2(p-1) steps, exit
  return 2 * ilog2i(world) + 2;                             // ready, L halving, L doubling, exit
}

// elements between a ring/hd bucket's input region and its output region
__host__ __device__ __forceinline__ uint64_t out_region_elems(uint64_t numel) {
  return (numel + 3) & ~3ull;
}

// Small two-shot buckets use the LL ("low latency") protocol: every element
// travels as ONE 64-bit relaxed store {epoch:32 | value:32} straight into its
// owner's inbox, so arrival of the data is its own flag -- no fence, no flag
// word, two one-way NVLink hops per bucket.  Region: [float bucket | LL out
// (numel x 8 B) | LL in (p slots x numel x 8 B)].  Chosen from numel alone, so
// every rank and every launch kind agrees.
#define LL_MAX_ELEMS 65536  // 256 KB: LL 21.6 vs flags 23.0 us at 256 KB (p=4); CARAMEL_LL_MAX overrides
// LL cutoff in elements: compile-time default, CARAMEL_LL_MAX overrides it at
// library load (host layout and device kernels read the same value; every
// rank must use the same setting, like every other layout parameter)
__device__ uint64_t d_ll_max = LL_MAX_ELEMS;
static uint64_t h_ll_max = LL_MAX_ELEMS;
__host__ __device__ __forceinline__ bool use_ll(int pattern, int world, uint64_t numel) {
#ifdef __CUDA_ARCH__
  const uint64_t cut = d_ll_max;
#else
  const uint64_t cut = h_ll_max;
#endif
  return pattern == CARAMEL_SHUFFLE && world > 1 && numel > 0 && numel <= cut;
}
__host__ __device__ __forceinline__ uint64_t ll_out_off(uint64_t numel) {  // bytes from bucket start
  return 4 * ((numel + 3) & ~3ull);
}
__host__ __device__ __forceinline__ uint64_t ll_region_bytes(uint64_t numel, int world) {
  return ll_out_off(numel) + 8 * numel * (1 + (uint64_t)world);
}

// ---- bucket region layout ------------------------------------------------------
//   [kernel region: packed bucket (two-shot) | LL region | ring/hd halves]
//   [push region (SHUFFLE, world > 1, not LL): 256 B header {seq, done} +
//    2 x (world-1) inbox slots, each mirroring the bucket's element
//    coordinates (element x of source q's contribution at slot + 4x, so every
//    slot keeps the bucket's 16-byte phase and TMA bulk copies line up)]
//   [copy-engine staging slots (caramel_allreduce_ce)]
// The push engine is opt-in (CARAMEL_PUSH=1, identical on every rank): on the
// B200 NVSwitch boxes measured so far the register-pull kernels move the same
// bytes faster.
__device__ int d_push_enabled = 0;
static int h_push_enabled = 0;
__host__ __device__ __forceinline__ bool push_enabled() {
#ifdef __CUDA_ARCH__
  return d_push_enabled != 0;
#else
  return h_push_enabled != 0;
#endif
}

// LL128 ("low latency, 128-byte lines"): two-shot buckets just above the LL
// cutoff.  Every value travels in a 128-byte line of 30 floats + an 8-byte
// epoch flag, written by 8 lanes of one warp instruction (16 B each) and read
// the same way: when the reader sees the flag, the whole line has landed
// (NVLink delivers the line as one unit -- the property NCCL's LL128 relies
// on), so data carries its own flag at 120/128 efficiency and a bucket costs
// two one-way hops with no fence and no flag round trip.  Region after the
// float bucket: [out: one line per 30 elements][in: p slots of the same lines].
#define LL128_MAX_ELEMS (1u << 19)  // 2 MiB (p=2: 1 MiB 17.7 vs 22.2 us flags, 4 MiB 26.2 vs 25.5); CARAMEL_LL128_MAX overrides
#define LL128_FLOATS 30
__device__ uint64_t d_ll128_max = LL128_MAX_ELEMS;
static uint64_t h_ll128_max = LL128_MAX_ELEMS;
__host__ __device__ __forceinline__ bool use_ll128(int pattern, int world, uint64_t numel) {
#ifdef __CUDA_ARCH__
  const uint64_t cut = d_ll128_max;
#else
  const uint64_t cut = h_ll128_max;
#endif
  return pattern == CARAMEL_SHUFFLE && world > 1 && !push_enabled() && !use_ll(pattern, world, numel) &&
         numel <= cut;
}
__host__ __device__ __forceinline__ uint64_t ll128_lines(uint64_t numel) {
  return (numel + LL128_FLOATS - 1) / LL128_FLOATS;
}
__host__ __device__ __forceinline__ uint64_t ll128_out_off(uint64_t numel) {  // bytes from bucket start
  return (4 * numel + 127) & ~127ull;
}
__host__ __device__ __forceinline__ uint64_t ll128_region_bytes(uint64_t numel, int world) {
  return ll128_out_off(numel) + 128 * ll128_lines(numel) * (1 + (uint64_t)world);
}
__host__ __device__ __forceinline__ uint64_t kernel_region_bytes(uint64_t numel, int pattern, int world) {
  const uint64_t e = out_region_elems(numel);
  if (use_ll(pattern, world, numel)) return (ll_region_bytes(numel, world) + 15) & ~15ull;
  if (use_ll128(pattern, world, numel)) return ll128_region_bytes(numel, world);
  return 4 * ((world > 1 && pattern != CARAMEL_SHUFFLE) ? 2 * e : e);
}
__host__ __device__ __forceinline__ bool has_push_region(uint64_t numel, int pattern, int world) {
  return push_enabled() && pattern == CARAMEL_SHUFFLE && world > 1 && numel > 0 && !use_ll(pattern, world, numel);
}
__host__ __device__ __forceinline__ uint64_t push_off(uint64_t numel, int pattern, int world) {
  return (kernel_region_bytes(numel, pattern, world) + 255) & ~255ull;
}
__host__ __device__ __forceinline__ uint64_t push_slot_bytes(uint64_t numel) { return (4 * numel + 255) & ~255ull; }
// Push items: chunk c of `depth`, tile range r of push_ranges() ~PUSH_RANGE_BYTES each.
#define PUSH_RANGE_BYTES (128u << 10)
__host__ __device__ __forceinline__ int push_ranges(uint64_t numel, int depth) {
  const uint64_t per_chunk = 4 * numel / (uint64_t)(depth > 0 ? depth : 1);
  const uint64_t r = (per_chunk + PUSH_RANGE_BYTES - 1) / PUSH_RANGE_BYTES;
  return r < 1 ? 1 : (int)r;
}
// flag words of the push items: [chunk][range][READY, DONE][source rank]
__host__ __device__ __forceinline__ uint64_t push_flag_bytes(uint64_t numel, int depth, int world) {
  return ((uint64_t)depth * push_ranges(numel, depth) * 2 * world * 4 + 255) & ~255ull;
}
__host__ __device__ __forceinline__ uint64_t push_region_bytes(uint64_t numel, int depth, int pattern, int world) {
  return has_push_region(numel, pattern, world)
             ? 256 + push_flag_bytes(numel, depth, world) + 2ull * (world - 1) * push_slot_bytes(numel)
             : 0;
}

// Protocols of a two-shot (SHUFFLE) bucket at world > 1.  A function of the
// bucket descriptor and the world size only -- identical on every rank and in
// every launch kind, so ranks never disagree on a bucket's flag protocol.
//   LL    <= LL cutoff elements: values travel with their epoch (two hops)
//   OS    one-shot push: every rank pushes its contribution of the whole
//         bucket into every peer's inbox (TMA, smem-staged), then reduces
//         all p inputs locally in rank order -- one flag hop, (p-1) x S bytes
//         per direction; used at p = 2 (where it moves exactly the two-shot's
//         2(p-1)/p x S) and for buckets up to the OS cutoff
//   TS    two-shot push: shard s of each chunk is pushed to its owner s
//         (reduce-scatter into the owner's inbox), the owner reduces it in
//         rank order, applies the epilogue and pushes the result into every
//         rank's output (all-gather) -- 2(p-1)/p x S bytes per direction
//   PULL  the register-staged pull kernels (UNPACK, or SGD with the
//         parameters in the members instead of the parameter arena)
// All protocols sum every element in ascending rank order: bit-identical.
enum { PROTO_PULL = 0, PROTO_LL = 1, PROTO_OS = 2, PROTO_TS = 3 };
#define OS_MAX_BYTES (1ull << 20)  // one-shot cutoff at p > 2; CARAMEL_OS_MAX overrides (same on every rank)
__device__ uint64_t d_os_max = OS_MAX_BYTES;
static uint64_t h_os_max = OS_MAX_BYTES;
__host__ __device__ __forceinline__ int shuffle_proto(const caramel_bucket& b, int world) {
#ifdef __CUDA_ARCH__
  const uint64_t os_max = d_os_max;
#else
  const uint64_t os_max = h_os_max;
#endif
  if (b.pattern != CARAMEL_SHUFFLE || world < 2) return PROTO_PULL;
  if (use_ll(b.pattern, world, b.numel)) return PROTO_LL;
  if (!push_enabled() || (b.flags & CARAMEL_F_UNPACK) ||
      (b.epilogue == CARAMEL_EPI_SGD && !(b.flags & CARAMEL_F_PARAM_ARENA)))
    return PROTO_PULL;
  return 4 * b.numel <= os_max ? PROTO_OS : PROTO_TS;
}

// x / d for the chunk/shard rule: 32-bit division when x fits (exact either way)
__host__ __device__ __forceinline__ uint64_t div_u64(uint64_t x, uint32_t d) {
  return x <= 0xffffffffull ? (uint64_t)((uint32_t)x / d) : x / d;
}

__host__ __device__ __forceinline__ void shard_bounds(uint64_t n, int k, int p, int c, int s, uint64_t& lo,
                                                      uint64_t& hi) {
  const uint64_t c0 = div_u64(n * (uint64_t)c, (uint32_t)k), m = div_u64(n * (uint64_t)(c + 1), (uint32_t)k) - c0;
  lo = c0 + div_u64(m * (uint64_t)s, (uint32_t)p);
  hi = c0 + div_u64(m * (uint64_t)(s + 1), (uint32_t)p);
}



__device__ __forceinline__ uint32_t launch_epoch(const Env& E) {
  // the device counter is advanced by k_epoch_advance earlier on the same
  // stream, so every CTA of a launch reads the same value
  return E.epoch ? E.epoch : *reinterpret_cast<const volatile uint32_t*>(E.epoch_dev);
}

struct Ctx {
  const Env* E;
  uint64_t flag_off;
  int me, world, j, G, ns;
  uint32_t epoch;
  __device__ __forceinline__ uint32_t* flag(int rank, int c, int slot, int src) const {
    uint32_t* base = reinterpret_cast<uint32_t*>(E->arena[rank] + flag_off);
    return base + ((((uint64_t)c * G + j) * ns + slot) * world + src);
  }
  // Every thread calls; thread t < ntargets publishes to targets[t].
  // bar.sync orders the CTA's data stores before the publishing thread's
  // st.release.sys, and release is cumulative over them -- no SC fence.
  __device__ __forceinline__ void publish(int c, int slot, const int* targets, int ntargets) const {
    __syncthreads();
    if ((int)threadIdx.x < ntargets) st_release_sys(flag(targets[threadIdx.x], c, slot, me), epoch);
  }
  __device__ __forceinline__ void publish_all(int c, int slot) const {
    __syncthreads();
    if ((int)threadIdx.x < world) st_release_sys(flag(threadIdx.x, c, slot, me), epoch);
  }
  // false: the watchdog fired (or the context is already poisoned)
  __device__ __forceinline__ bool spin(const uint32_t* f, uint32_t want) const {
    if (ld_acquire_sys(f) >= want) return true;
    uint64_t t0 = globaltimer();
    uint32_t spins = 0;
    while (ld_acquire_sys(f) < want) {
      if ((++spins & 1023u) == 0) {
        if (poisoned(*E)) return false;
        if (globaltimer() - t0 > E->timeout_ns) {
          raise_timeout(*E);
          return false;
        }
      }
    }
    return true;
  }
  // every thread calls; waits until each src's flag (in my block) reaches
  // `want`; the whole CTA leaves the kernel if a wait failed
  __device__ __forceinline__ void wait_from(int c, int slot, const int* srcs, int nsrc, uint32_t want) const {
    int bad = 0;
    if ((int)threadIdx.x < nsrc) bad = !spin(flag(me, c, slot, srcs[threadIdx.x]), want);
    cta_abort_if(bad);
  }
  __device__ __forceinline__ void wait_all(int c, int slot, uint32_t want) const {
    int bad = 0;
    if ((int)threadIdx.x < world) bad = !spin(flag(me, c, slot, threadIdx.x), want);
    cta_abort_if(bad);
  }
};

// Reduce [lo, hi) of the bucket across all P ranks in ascending rank order
// (acc = g0; acc += g1; ...), apply the epilogue once, store the result to
// every rank's output buffer.  Two float4 per thread per trip so 2*P 128-bit
// loads are in flight before the first add.
template <int P>
__device__ __forceinline__ void rs_ag_range(const Env& E, const caramel_bucket& B, bool arena, Cursor& tc,
                                            uint64_t lo, uint64_t hi, int me, const float* const* srcs) {
  if (lo >= hi) return;
  // srcs[q] + x addresses source q's value of bucket position x (an inbox slot)
  auto src = [&](int q) { return srcs[q]; };
  auto dst = [&](int q) {
    return arena ? reinterpret_cast<float*>(E.parena[q] + B.param_off)
                 : reinterpret_cast<float*>(E.arena[q] + B.bucket_off);
  };
  const float* theta_flat = arena ? reinterpret_cast<const float*>(E.parena[me] + B.param_off) : nullptr;
  const int epi = B.epilogue;
  const float scale = B.scale, lr = B.lr;
  const bool need_theta = (epi == CARAMEL_EPI_SGD);
  uint64_t a = (lo + 3) & ~3ull;
  if (a > hi) a = hi;
  uint64_t b = hi & ~3ull;
  if (b < a) b = a;
  auto scalar = [&](uint64_t i) {
    float s = ld1(src(0) + i);
#pragma unroll
    for (int q = 1; q < P; ++q) s = __fadd_rn(s, ld1(src(q) + i));
    float t = 0.f;
    if (need_theta) t = arena ? ld1(theta_flat + i) : seg_ld1(tc, i, 1);
    float o = epi1(epi, s, t, scale, lr);
#pragma unroll
    for (int q = 0; q < P; ++q) st1(dst(q) + i, o);
  };
  for (uint64_t i = lo + threadIdx.x; i < a; i += blockDim.x) scalar(i);
  const uint64_t step = 4ull * blockDim.x;
  uint64_t v = a + 4ull * threadIdx.x;
  for (; v + step < b; v += 2 * step) {
    float4 x0[P], x1[P];
#pragma unroll
    for (int q = 0; q < P; ++q) {
      x0[q] = ld4(src(q) + v);
      x1[q] = ld4(src(q) + v + step);
    }
    float4 t0 = make_float4(0.f, 0.f, 0.f, 0.f), t1 = t0;
    if (need_theta) {
      if (arena) {
        t0 = ld4(theta_flat + v);
        t1 = ld4(theta_flat + v + step);
      } else {
        t0 = seg_ld4(tc, v, 1);
        t1 = seg_ld4(tc, v + step, 1);
      }
    }
    float4 s0 = x0[0], s1 = x1[0];
#pragma unroll
    for (int q = 1; q < P; ++q) {
      s0 = add4(s0, x0[q]);
      s1 = add4(s1, x1[q]);
    }
    float4 o0 = epi4(epi, s0, t0, scale, lr), o1 = epi4(epi, s1, t1, scale, lr);
#pragma unroll
    for (int q = 0; q < P; ++q) {
      st4(dst(q) + v, o0);
      st4(dst(q) + v + step, o1);
    }
  }
  if (v < b) {
    float4 s = ld4(src(0) + v);
#pragma unroll
    for (int q = 1; q < P; ++q) s = add4(s, ld4(src(q) + v));
    float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
    if (need_theta) t = arena ? ld4(theta_flat + v) : seg_ld4(tc, v, 1);
    float4 o = epi4(epi, s, t, scale, lr);
#pragma unroll
    for (int q = 0; q < P; ++q) st4(dst(q) + v, o);
  }
  for (uint64_t i = b + threadIdx.x; i < hi; i += blockDim.x) scalar(i);
}

// Pairwise step used by ring and halving-doubling: out = a + b (a first),
// optionally followed by the epilogue (last reduction of the owner's shard).
// [lo, hi) split into a scalar head, a 4-aligned float4 body and a scalar tail
__device__ __forceinline__ void split4(uint64_t lo, uint64_t hi, uint64_t& a, uint64_t& b) {
  a = (lo + 3) & ~3ull;
  if (a > hi) a = hi;
  b = hi & ~3ull;
  if (b < a) b = a;
}

// Pairwise step used by ring and halving-doubling: out = a + b (a first),
// optionally followed by the epilogue (last reduction of the owner's shard).
// Four float4 per thread per trip, loads of both operands issued first (the
// operands are peer memory: one NVLink round trip per trip, not per vector).
__device__ __forceinline__ void pair_range(const float* a_src, const float* b_src, float* out,
                                           uint64_t lo, uint64_t hi, bool final_epi, const caramel_bucket& B,
                                           const float* theta_flat, Cursor& tc) {
  const int epi = B.epilogue;
  const bool need_theta = final_epi && epi == CARAMEL_EPI_SGD;
  auto scalar = [&](uint64_t i) {
    float s = __fadd_rn(ld1(a_src + i), ld1(b_src + i));
    if (final_epi) {
      float t = 0.f;
      if (need_theta) t = theta_flat ? ld1(theta_flat + i) : seg_ld1(tc, i, 1);
      s = epi1(epi, s, t, B.scale, B.lr);
    }
    st1(out + i, s);
  };
  if (lo >= hi) return;
  uint64_t a, b;
  split4(lo, hi, a, b);
  for (uint64_t i = lo + threadIdx.x; i < a; i += blockDim.x) scalar(i);
  constexpr int U = 4;
  const uint64_t step = 4ull * blockDim.x;
  uint64_t v = a + 4ull * threadIdx.x;
  for (; v + (U - 1) * step < b; v += U * step) {
    float4 x[U], y[U], t[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x[u] = ld4(a_src + v + u * step);
      y[u] = ld4(b_src + v + u * step);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      t[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (need_theta) t[u] = theta_flat ? ld4(theta_flat + v + u * step) : seg_ld4(tc, v + u * step, 1);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float4 s = add4(x[u], y[u]);
      if (final_epi) s = epi4(epi, s, t[u], B.scale, B.lr);
      st4(out + v + u * step, s);
    }
  }
  for (; v < b; v += step) {
    float4 s = add4(ld4(a_src + v), ld4(b_src + v));
    if (final_epi) {
      float4 t = make_float4(0.f, 0.f, 0.f, 0.f);
      if (need_theta) t = theta_flat ? ld4(theta_flat + v) : seg_ld4(tc, v, 1);
      s = epi4(epi, s, t, B.scale, B.lr);
    }
    st4(out + v, s);
  }
  for (uint64_t i = b + threadIdx.x; i < hi; i += blockDim.x) scalar(i);
}

__device__ __forceinline__ void copy_range(const float* src, float* dst, uint64_t lo, uint64_t hi) {
  if (lo >= hi) return;
  uint64_t a, b;
  split4(lo, hi, a, b);
  for (uint64_t i = lo + threadIdx.x; i < a; i += blockDim.x) st1(dst + i, ld1(src + i));
  constexpr int U = 8;
  const uint64_t step = 4ull * blockDim.x;
  uint64_t v = a + 4ull * threadIdx.x;
  for (; v + (U - 1) * step < b; v += U * step) {
    float4 x[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = ld4(src + v + u * step);
#pragma unroll
    for (int u = 0; u < U; ++u) st4(dst + v + u * step, x[u]);
  }
  for (; v < b; v += step) st4(dst + v, ld4(src + v));
  for (uint64_t i = b + threadIdx.x; i < hi; i += blockDim.x) st1(dst + i, ld1(src + i));
}

// Single-rank path (world == 1): no exchange; gather, epilogue and scatter
// fused in one pass.  Piece [x0, x1) (bucket coordinates) of member sg:
__device__ __forceinline__ void local_piece(const Env& E, const caramel_bucket& B, int lr_idx, const Seg& sg,
                                            uint64_t x0, uint64_t x1, PieceDesc& d) {
  const int me = E.rank_base + lr_idx;
  float* bkt = reinterpret_cast<float*>(E.arena[me] + B.bucket_off);
  const bool arena = (B.flags & CARAMEL_F_PARAM_ARENA) && B.epilogue == CARAMEL_EPI_SGD;
  float* pflat = arena ? reinterpret_cast<float*>(E.parena[me] + B.param_off) : nullptr;
  const bool pack = B.flags & CARAMEL_F_PACK;
  const bool unpack = (B.flags & CARAMEL_F_UNPACK) && !arena;
  const bool sgd = B.epilogue == CARAMEL_EPI_SGD;
  const uint64_t k = x0 - sg.offset;
  d.g = pack ? reinterpret_cast<const float*>(sg.grad) + k : bkt + x0;
  d.t = arena ? pflat + x0 : (sgd ? reinterpret_cast<const float*>(sg.param) + k : nullptr);
  d.o = arena ? pflat + x0 : unpack ? reinterpret_cast<float*>(sgd ? sg.param : sg.grad) + k : bkt + x0;
  d.n = (uint32_t)(x1 - x0);
  d.epi = B.epilogue;
  d.scale = B.scale;
  d.lr = B.lr;
}

__device__ __forceinline__ bool local_needs_members(const caramel_bucket& B) {
  const bool arena = (B.flags & CARAMEL_F_PARAM_ARENA) && B.epilogue == CARAMEL_EPI_SGD;
  return (B.flags & CARAMEL_F_PACK) || ((B.flags & CARAMEL_F_UNPACK) && !arena) ||
         (B.epilogue == CARAMEL_EPI_SGD && !arena);
}

// bucket-local [lo, hi) of one bucket
__device__ void local_range(const Env& E, const caramel_bucket& B, int lr_idx, uint64_t lo, uint64_t hi,
                            PieceTab& tab) {
  const int me = E.rank_base + lr_idx;
  if (!local_needs_members(B)) {  // bucket in, bucket / arena out
    float* bkt = reinterpret_cast<float*>(E.arena[me] + B.bucket_off);
    const bool arena = (B.flags & CARAMEL_F_PARAM_ARENA) && B.epilogue == CARAMEL_EPI_SGD;
    float* out = arena ? reinterpret_cast<float*>(E.parena[me] + B.param_off) : bkt;
    run_pieces<OP_EPI>(lo < hi ? 1 : 0, [&](int, PieceDesc& d) {
      d.g = bkt + lo;
      d.t = out + lo;
      d.o = out + lo;
      d.n = (uint32_t)(hi - lo);
      d.epi = B.epilogue;
      d.scale = B.scale;
      d.lr = B.lr;
    }, tab);
    return;
  }
  const caramel_segment* segs = reinterpret_cast<const caramel_segment*>(B.segs) + (uint64_t)lr_idx * B.nseg;
  int seg0;
  const int np = seg_span(segs, B.nseg, lo, hi, seg0);
  run_pieces<OP_EPI>(np, [&](int i, PieceDesc& d) {
    const Seg sg = load_seg(segs, seg0 + i);
    uint64_t x0, x1;
    if (clip_seg(sg, lo, hi, x0, x1)) local_piece(E, B, lr_idx, sg, x0, x1, d);
  }, tab);
}

// Per-CTA view of one bucket's collective (world > 1).
struct BucketRun {
  const Env* E;
  const caramel_bucket* B;
  PieceTab* tab;
  Ctx X;
  int lr_idx;
  bool arena;
  uint32_t cmask;    // chunks this CTA works on (bit c), and its tile / group size in them
  int cjj, cgg;
  uint64_t out_off;
  const caramel_segment* segs;

  __device__ __forceinline__ float* bucket(int q) const {
    return reinterpret_cast<float*>(E->arena[q] + B->bucket_off);
  }
  __device__ __forceinline__ float* out(int q) const {
    return arena ? reinterpret_cast<float*>(E->parena[q] + B->param_off) : bucket(q) + out_off;
  }
  __device__ __forceinline__ const float* theta_flat() const {
    return arena ? reinterpret_cast<const float*>(E->parena[X.me] + B->param_off) : nullptr;
  }
  // Chunk-parallel tiling: the bucket's G CTAs are split into `depth` groups,
  // group c = CTAs [s_c, e_c) works on chunk c only (several chunks share a
  // CTA when G < depth).  mine(c): does this CTA take part in chunk c, and as
  // which tile of how many.
  // (computed once per CTA in make_run: evaluating the group bounds here, per
  // chunk and per call, cost ~1 us per extra chunk in integer divisions)
  __device__ __forceinline__ bool mine(int c, int& jj, int& gg) const {
    jj = cjj;
    gg = cgg;
    return (cmask >> c) & 1u;
  }
  __device__ __forceinline__ bool mine(int c) const {
    int a, b;
    return mine(c, a, b);
  }
  // this CTA's tile of shard s of chunk c (only meaningful when mine(c))
  __device__ __forceinline__ void shard(int c, int s, uint64_t& lo, uint64_t& hi) const {
    const uint64_t n = B->numel;
    const int k = B->depth, p = X.world;
    int jj = 0, gg = 1;
    mine(c, jj, gg);
    uint64_t c0 = split_at(n, k, c), m = split_at(n, k, c + 1) - c0;
    tile_of(c0 + split_at(m, p, s), c0 + split_at(m, p, s + 1), gg, jj, lo, hi);
  }
};

__device__ __forceinline__ void make_run(BucketRun& R, const Env& E, const caramel_bucket& B, int pattern,
                                         int lr_idx, uint32_t epoch, int j) {
  R.E = &E;
  R.B = &B;
  R.tab = &g_tab;
  R.lr_idx = lr_idx;
  R.arena = (B.flags & CARAMEL_F_PARAM_ARENA) && B.epilogue == CARAMEL_EPI_SGD;
  // (one flat pass over every chunk -- each CTA its tile of all chunks, one
  // flag per tile -- was measured against these chunk-parallel CTA groups and
  // lost at every depth > 1: p=2, 16 MiB depth 3 44.3 vs 51.6 us, 256 MiB
  // depth 8 416 vs 481 us; it was removed)
  // shuffle all-gathers in place; ring/hd write results to a second region
  // of the bucket so a fast neighbour never overwrites a partial sum that a
  // slower one has yet to pull
  R.out_off = (pattern == CARAMEL_SHUFFLE) ? 0 : out_region_elems(B.numel);
  R.segs = reinterpret_cast<const caramel_segment*>(B.segs) + (uint64_t)lr_idx * B.nseg;
  R.X.E = &E;
  R.X.flag_off = B.flag_off;
  R.X.me = E.rank_base + lr_idx;
  R.X.world = E.world;
  R.X.j = j;
  R.X.G = B.ctas;
  R.X.ns = nslots(pattern, E.world);
  R.X.epoch = epoch;
  // chunk-parallel CTA groups: chunk c = CTAs [s_c, e_c), s_c = floor(c*G/k)
  // (at least one CTA each; with G < k every group is one CTA)
  const int G = B.ctas, k = B.depth;
  R.cmask = 0;
  R.cjj = 0;
  R.cgg = 1;
  for (int c = 0; c < k; ++c) {
    const int s0 = (c * G) / k;
    int e0 = ((c + 1) * G) / k;
    if (e0 <= s0) e0 = s0 + 1;
    if (j >= s0 && j < e0) {
      R.cmask |= 1u << c;
      R.cjj = j - s0;
      R.cgg = e0 - s0;
    }
  }
}

// phase 1 (all patterns): ring/hd buffer-reuse guard, fused pack, ready flags
// (DEFER: the caller publishes every bucket's ready flags after one fence)
template <int PAT, bool DEFER = false>
__device__ void phase_pack(const BucketRun& R) {
  const int me = R.X.me, p = R.X.world;
  const uint32_t epoch = R.X.epoch;
  if (PAT != CARAMEL_SHUFFLE && epoch > 1) {
    // every rank that read my buffers last epoch must be done with them
    int srcs[MAXR];
    int ns = 0;
    if (PAT == CARAMEL_RING) {
      srcs[ns++] = (me + 1) % p;
    } else {
      for (int d = 1; d < p; d <<= 1) srcs[ns++] = me ^ d;
    }
    R.X.wait_from(0, R.X.ns - 1, srcs, ns, epoch - 1);
  }
  const bool pack = R.B->flags & CARAMEL_F_PACK;
  float* mine = R.bucket(me);
  for (int c = 0; c < R.B->depth; ++c) {
    if (!R.mine(c)) continue;
    if (pack) {
      for (int s = 0; s < p; ++s) {
        uint64_t lo, hi;
        R.shard(c, s, lo, hi);
        pack_range(R.segs, R.B->nseg, mine, lo, hi, *R.tab);
      }
    }
    if (PAT == CARAMEL_SHUFFLE) {
      if (!DEFER) R.X.publish_all(c, SLOT_READY);
    } else {
      int t = (PAT == CARAMEL_RING) ? (me + 1) % p : (me ^ (p >> 1));
      R.X.publish(c, SLOT_READY, &t, 1);
    }
  }
}

// Reduce + epilogue + all-gather of several ranges (this CTA's tile of my
// shard in every chunk) as ONE flat vector loop: chunk boundaries cost no
// extra memory round trip (2*NP 128-bit loads in flight per thread across
// ranges).  Scalar heads/tails first.
template <int NP, int UV = 0>
__device__ void rs_ag_multi(const Env& E, const caramel_bucket& B, bool arena, Cursor& tc, const uint64_t* lo,
                            const uint64_t* hi, int nr, int me, int cj = 0, int cg = 1) {
  const float* src[NP];
  float* dst[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    src[q] = reinterpret_cast<const float*>(E.arena[q] + B.bucket_off);
    dst[q] = arena ? reinterpret_cast<float*>(E.parena[q] + B.param_off)
                   : reinterpret_cast<float*>(E.arena[q] + B.bucket_off);
  }
  const float* th = arena ? reinterpret_cast<const float*>(E.parena[me] + B.param_off) : nullptr;
  const int epi = B.epilogue;
  const bool sgd = epi == CARAMEL_EPI_SGD;
  uint64_t va[CARAMEL_MAX_DEPTH], vpre[CARAMEL_MAX_DEPTH + 1];
  vpre[0] = 0;
  // The vector part of a range starts and ends on 128-byte lines (32 floats):
  // a warp's 32 float4s then cover exactly 4 lines instead of straddling 5,
  // which over NVLink cost an unaligned (depth-3) bucket 9%.  Scalar heads
  // [lo, a) and tails [b, hi) (< 32 each, CTA cj == 0 of the group): thread t
  // takes the t-th one; its loads are issued here and consumed after the
  // vector loop, so their round trip overlaps the vectors.  At most 62 per
  // range and 8 ranges: every caller runs >= 496 threads (static_asserts at
  // k_collective / k_gated).
  bool has_s = false;
  uint64_t sx = 0;
  uint32_t scnt = 0;
  for (int k = 0; k < nr; ++k) {
    uint64_t a = (lo[k] + 31) & ~31ull, b = hi[k] & ~31ull;
    if (a > hi[k]) a = hi[k];
    if (b < a) b = a;
    va[k] = a;
    vpre[k + 1] = vpre[k] + (b - a) / 4;
    if (cj == 0) {
      const uint64_t nh = a - lo[k], nt = hi[k] - b;
      if (threadIdx.x >= scnt && threadIdx.x < scnt + nh + nt) {
        const uint64_t e = threadIdx.x - scnt;
        sx = e < nh ? lo[k] + e : b + (e - nh);
        has_s = true;
      }
      scnt += (uint32_t)(nh + nt);
    }
  }
  float sv[NP], s_th = 0.f;
  if (has_s) {
#pragma unroll
    for (int q = 0; q < NP; ++q) sv[q] = ld1(src[q] + sx);
    if (sgd) s_th = arena ? ld1(th + sx) : seg_ld1(tc, sx, 1);
  }
  const uint64_t V = vpre[nr], T = blockDim.x;
  // flat vector index -> bucket element position; v only grows, so each of
  // the U streams keeps its own range cursor (no rescan per vector)
  // U x NP 128-bit loads in flight per thread (8 at p = 2, as the fused kernel)
  constexpr int U = UV ? UV : NP <= 2 ? 4 : 2;
  int kc[U];
#pragma unroll
  for (int u = 0; u < U; ++u) kc[u] = 0;
  auto pos = [&](uint64_t v, int& k) {
    while (v >= vpre[k + 1]) ++k;
    return va[k] + 4 * (v - vpre[k]);
  };
  // the group's cg CTAs split [0, V) into balanced contiguous ranges (cg ==
  // 1: the whole range is this CTA's).  Whole rows of U*T vectors per CTA
  // left up to one row of imbalance: 85 rows over 42 CTAs (16 MiB, depth 3)
  // ran 3 rows on some CTAs and 2 on most, 10% over depth 1.
  // (in units of 8 vectors = one 128-byte line)
  const uint64_t V8 = (V + 7) / 8;
  uint64_t v_lo = 8 * (V8 * (uint64_t)cj / (uint64_t)cg), v_hi = 8 * (V8 * (uint64_t)(cj + 1) / (uint64_t)cg);
  if (v_lo > V) v_lo = V;
  if (v_hi > V) v_hi = V;
  for (uint64_t base = v_lo; base < v_hi; base += (uint64_t)U * T) {
    uint64_t x[U];
    bool ok[U];
    float4 pv[U][NP], tv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t v = base + u * T + threadIdx.x;
      ok[u] = v < v_hi;
      x[u] = ok[u] ? pos(v, kc[u]) : 0;
#pragma unroll
      for (int q = 0; q < NP; ++q) pv[u][q] = ok[u] ? ld4(src[q] + x[u]) : make_float4(0.f, 0.f, 0.f, 0.f);
      tv[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (sgd && ok[u]) tv[u] = arena ? ld4(th + x[u]) : seg_ld4(tc, x[u], 1);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!ok[u]) continue;
      float4 sum = pv[u][0];
#pragma unroll
      for (int q = 1; q < NP; ++q) sum = add4(sum, pv[u][q]);
      const float4 o = epi4(epi, sum, tv[u], B.scale, B.lr);
#pragma unroll
      for (int q = 0; q < NP; ++q) st4(dst[q] + x[u], o);
    }
  }
  if (has_s) {
    float acc = sv[0];
#pragma unroll
    for (int q = 1; q < NP; ++q) acc = __fadd_rn(acc, sv[q]);
    const float o = epi1(epi, acc, s_th, B.scale, B.lr);
#pragma unroll
    for (int q = 0; q < NP; ++q) st1(dst[q] + sx, o);
  }
}

// phase 2, two-shot: reduce own shard in rank order, epilogue, all-gather by
// store.  DEFER (ready flags published together): wait for every chunk, then
// one flat pass over all chunks; otherwise chunk by chunk with per-chunk DONE.
template <int NP, bool DEFER = false>
__device__ void phase_shuffle(const BucketRun& R) {
  Cursor tc;
  cur_init(tc, R.segs, R.B->nseg);
  // Without PACK / UNPACK no tile of a CTA depends on another CTA's work (the
  // gradients were complete before any rank launched): the chunk's CTA group
  // sweeps its whole shard (balanced contiguous ranges) instead of one tile each
  const bool group_sweep = !(R.B->flags & (CARAMEL_F_PACK | CARAMEL_F_UNPACK));
  auto range_of = [&](int c, uint64_t& lo, uint64_t& hi, int& cj, int& cg) {
    if (group_sweep) {
      R.mine(c, cj, cg);
      shard_bounds(R.B->numel, R.B->depth, R.X.world, c, R.X.me, lo, hi);
    } else {
      cj = 0;
      cg = 1;
      R.shard(c, R.X.me, lo, hi);
    }
  };
  if (DEFER) {
    uint64_t lo[CARAMEL_MAX_DEPTH], hi[CARAMEL_MAX_DEPTH];
    int nr = 0, cj = 0, cg = 1;
    for (int c = 0; c < R.B->depth; ++c) {
      if (!R.mine(c)) continue;
      R.X.wait_all(c, SLOT_READY, R.X.epoch);
      range_of(c, lo[nr], hi[nr], cj, cg);
      ++nr;
    }
    rs_ag_multi<NP>(*R.E, *R.B, R.arena, tc, lo, hi, nr, R.X.me, cj, cg);
    return;
  }
  for (int c = 0; c < R.B->depth; ++c) {
    if (!R.mine(c)) continue;
    R.X.wait_all(c, SLOT_READY, R.X.epoch);
    uint64_t lo, hi;
    int cj, cg;
    range_of(c, lo, hi, cj, cg);
    rs_ag_multi<NP>(*R.E, *R.B, R.arena, tc, &lo, &hi, 1, R.X.me, cj, cg);
    R.X.publish_all(c, SLOT_DONE);
  }
}

__device__ void phase_ring(const BucketRun& R) {
  const int me = R.X.me, p = R.X.world;
  const int left = (me + p - 1) % p, right = (me + 1) % p;
  float* mine = R.bucket(me);
  Cursor tc;
  cur_init(tc, R.segs, R.B->nseg);
  const float* th = R.theta_flat();
  for (int c = 0; c < R.B->depth; ++c) {
    if (!R.mine(c)) continue;
    // reduce-scatter: at step t rank r folds its own share of shard
    // (r-1-t) mod p into the left neighbour's running sum (the chain of
    // shard s starts at rank s+1 and ends at its owner s)
    for (int t = 1; t <= p - 1; ++t) {
      R.X.wait_from(c, t == 1 ? SLOT_READY : t - 1, &left, 1, R.X.epoch);
      const int s = ((me - 1 - t) % p + p) % p;
      const bool last = (t == p - 1);
      uint64_t lo, hi;
      R.shard(c, s, lo, hi);
      pair_range(R.bucket(left), mine, last ? R.out(me) : mine, lo, hi, last, *R.B, th, tc);
      R.X.publish(c, t, &right, 1);
    }
    // all-gather: at step t copy shard (r-t) mod p from the left neighbour
    for (int t = 1; t <= p - 1; ++t) {
      R.X.wait_from(c, (p - 1) + (t - 1), &left, 1, R.X.epoch);
      const int s = ((me - t) % p + p) % p;
      uint64_t lo, hi;
      R.shard(c, s, lo, hi);
      copy_range(R.out(left), R.out(me), lo, hi);
      R.X.publish(c, (p - 1) + t, &right, 1);
    }
  }
}

__device__ void phase_hd(const BucketRun& R) {
  // Stages: 0 = pack, 1..L = halving rounds, L+1..2L = doubling rounds.
  // Stage s reads from partner(s); finishing stage s signals slot s to the
  // rank that reads from me next, partner(s+1).
  const int me = R.X.me, p = R.X.world;
  const int L = ilog2i(p);
  auto partner_of = [&](int stage) {
    return stage <= L ? (me ^ (p >> stage)) : (me ^ (1 << (stage - L - 1)));
  };
  float* mine = R.bucket(me);
  Cursor tc;
  cur_init(tc, R.segs, R.B->nseg);
  const float* th = R.theta_flat();
  for (int c = 0; c < R.B->depth; ++c) {
    if (!R.mine(c)) continue;
    // vector halving, distance halving: round i pairs r with r ^ (p >> (i+1));
    // r keeps the half of its active block range that contains block r and
    // sums it as (lower rank's value) + (higher rank's value)
    for (int i = 0; i < L; ++i) {
      const int stage = i + 1;
      const int dist = p >> (i + 1);
      const int partner = partner_of(stage);
      R.X.wait_from(c, stage - 1, &partner, 1, R.X.epoch);
      const int base = me & ~(2 * dist - 1);
      const int s0 = (me & dist) ? base + dist : base;
      const bool last = (i == L - 1);
      const float* lo_src = (me < partner) ? mine : R.bucket(partner);
      const float* hi_src = (me < partner) ? R.bucket(partner) : mine;
      for (int s = s0; s < s0 + dist; ++s) {
        uint64_t lo, hi;
        R.shard(c, s, lo, hi);
        pair_range(lo_src, hi_src, last ? R.out(me) : mine, lo, hi, last, *R.B, th, tc);
      }
      const int nxt = partner_of(stage + 1);
      R.X.publish(c, stage, &nxt, 1);
    }
    // vector doubling: round i pairs r with r ^ (1 << i); copy the partner's
    // finished blocks into my output
    for (int i = 0; i < L; ++i) {
      const int stage = L + 1 + i;
      const int dist = 1 << i;
      const int partner = partner_of(stage);
      R.X.wait_from(c, stage - 1, &partner, 1, R.X.epoch);
      const int s0 = partner & ~(dist - 1);
      for (int s = s0; s < s0 + dist; ++s) {
        uint64_t lo, hi;
        R.shard(c, s, lo, hi);
        copy_range(R.out(partner), R.out(me), lo, hi);
      }
      if (i + 1 < L) {
        const int nxt = partner_of(stage + 1);
        R.X.publish(c, stage, &nxt, 1);
      }
    }
  }
}

// ---- LL protocol phases (small two-shot buckets) ------------------------------
__device__ __forceinline__ uint64_t ll_pack(uint32_t epoch, float v) {
  return ((uint64_t)epoch << 32) | (uint64_t)__float_as_uint(v);
}

// spin until the LL word carries `epoch`; returns its value.  On a watchdog
// timeout (or a poisoned context) sets `bad`: the caller stores nothing
// derived from this value.
__device__ __forceinline__ float ll_wait(const uint64_t* p, uint32_t epoch, const Env& E, int& bad) {
  uint64_t w = ld_u64_relaxed_sys(p);
  if ((uint32_t)(w >> 32) != epoch && !bad) {
    const uint64_t t0 = globaltimer();
    uint32_t spins = 0;
    do {
      w = ld_u64_relaxed_sys(p);
      if ((++spins & 1023u) == 0) {
        if (poisoned(E)) { bad = 1; break; }
        if (globaltimer() - t0 > E.timeout_ns) {
          raise_timeout(E);
          bad = 1;
          break;
        }
      }
    } while ((uint32_t)(w >> 32) != epoch);
  } else if ((uint32_t)(w >> 32) != epoch) {
    bad = 1;
  }
  return __uint_as_float((uint32_t)w);
}

__device__ __forceinline__ uint64_t* ll_out(const BucketRun& R, int rank) {
  return reinterpret_cast<uint64_t*>(R.E->arena[rank] + R.B->bucket_off + ll_out_off(R.B->numel));
}
__device__ __forceinline__ uint64_t* ll_in(const BucketRun& R, int rank, int slot) {
  return ll_out(R, rank) + R.B->numel * (1 + (uint64_t)slot);
}

// A: every element of my tile of every shard, pushed into its owner's inbox slot `me`
__device__ void phase_ll_scatter(const BucketRun& R) {
  const int me = R.X.me, p = R.X.world;
  const bool pack = R.B->flags & CARAMEL_F_PACK;
  const float* bkt = R.bucket(me);
  Cursor gc;
  cur_init(gc, R.segs, R.B->nseg);
  for (int c = 0; c < R.B->depth; ++c)
    for (int s = 0; s < p && R.mine(c); ++s) {
      uint64_t lo, hi;
      R.shard(c, s, lo, hi);
      uint64_t* dst = ll_in(R, s, me);
      for (uint64_t x = lo + threadIdx.x; x < hi; x += blockDim.x) {
        const float v = pack ? seg_ld1(gc, x, 0) : ld1(bkt + x);
        st_u64_relaxed_sys(dst + x, ll_pack(R.X.epoch, v));
      }
    }
}

// B: my shard -- wait for every source in rank order, sum, epilogue, push to
// all.  Loads for LL_U elements x every source are issued together; only the
// words that have not arrived yet are polled again.
#define LL_U 4
template <int NP>
__device__ void phase_ll_reduce(const BucketRun& R) {
  const int me = R.X.me;
  Cursor tc;
  cur_init(tc, R.segs, R.B->nseg);
  const float* th = R.theta_flat();
  const bool sgd = R.B->epilogue == CARAMEL_EPI_SGD;
  const uint32_t ep = R.X.epoch;
  int bad = 0;
  for (int c = 0; c < R.B->depth; ++c) {
    if (!R.mine(c)) continue;
    uint64_t lo, hi;
    R.shard(c, me, lo, hi);
    const uint64_t T = blockDim.x;
    for (uint64_t x0 = lo + threadIdx.x; x0 < hi; x0 += LL_U * T) {
      uint64_t w[LL_U][NP];
#pragma unroll
      for (int u = 0; u < LL_U; ++u)
#pragma unroll
        for (int q = 0; q < NP; ++q)
          w[u][q] = (x0 + u * T < hi) ? ld_u64_relaxed_sys(ll_in(R, me, q) + x0 + u * T) : 0;
#pragma unroll
      for (int u = 0; u < LL_U; ++u) {
        const uint64_t x = x0 + u * T;
        if (x >= hi) break;
        float acc = 0.f;
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          float v = __uint_as_float((uint32_t)w[u][q]);
          if ((uint32_t)(w[u][q] >> 32) != ep) v = ll_wait(ll_in(R, me, q) + x, ep, *R.E, bad);
          acc = q == 0 ? v : __fadd_rn(acc, v);
        }
        if (bad) continue;  // an input never arrived: store nothing derived from it
        const float t = sgd ? (th ? ld1(th + x) : seg_ld1(tc, x, 1)) : 0.f;
        const uint64_t o = ll_pack(ep, epi1(R.B->epilogue, acc, t, R.B->scale, R.B->lr));
#pragma unroll
        for (int q = 0; q < NP; ++q) st_u64_relaxed_sys(ll_out(R, q) + x, o);
      }
    }
  }
}

// C: collect my tile of every shard's result; write to the parameter arena,
// the members, or the float bucket (loads batched as in B)
__device__ void phase_ll_finish(const BucketRun& R) {
  const int me = R.X.me, p = R.X.world;
  const bool unpack = (R.B->flags & CARAMEL_F_UNPACK) && !R.arena;
  const int which = R.B->epilogue == CARAMEL_EPI_SGD ? 1 : 0;
  float* res = R.arena ? R.out(me) : R.bucket(me);
  Cursor uc;
  cur_init(uc, R.segs, R.B->nseg);
  const uint64_t* in = ll_out(R, me);
  const uint32_t ep = R.X.epoch;
  const uint64_t T = blockDim.x;
  int bad = 0;
  for (int c = 0; c < R.B->depth; ++c)
    for (int s = 0; s < p && R.mine(c); ++s) {
      uint64_t lo, hi;
      R.shard(c, s, lo, hi);
      for (uint64_t x0 = lo + threadIdx.x; x0 < hi; x0 += 4 * LL_U * T) {
        uint64_t w[4 * LL_U];
#pragma unroll
        for (int u = 0; u < 4 * LL_U; ++u) w[u] = (x0 + u * T < hi) ? ld_u64_relaxed_sys(in + x0 + u * T) : 0;
#pragma unroll
        for (int u = 0; u < 4 * LL_U; ++u) {
          const uint64_t x = x0 + u * T;
          if (x >= hi) break;
          float v = __uint_as_float((uint32_t)w[u]);
          if ((uint32_t)(w[u] >> 32) != ep) v = ll_wait(in + x, ep, *R.E, bad);
          if (bad) continue;
          if (unpack) seg_st1(uc, x, which, v);
          else st1(res + x, v);
        }
      }
    }
}

// ---- LL128 protocol phases (mid-size two-shot buckets, see use_ll128) -------------
// Ownership is by LINES (30 elements): shard s = lines [s L / p, (s+1) L / p);
// CTA j of the bucket takes part j of every shard's lines; inside a CTA, an
// 8-lane group handles one line per step (lane k: floats 4k..4k+3 of the
// line; lane 7: floats 28, 29 and the 8-byte flag {epoch, epoch}).
__device__ __forceinline__ uint4 ll128_ld(const void* p) {
  uint4 v;
  asm volatile("ld.relaxed.sys.global.v4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void ll128_st(void* p, uint4 v) {
  asm volatile("st.relaxed.sys.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ char* ll128_out(const BucketRun& R, int rank) {
  return reinterpret_cast<char*>(R.E->arena[rank] + R.B->bucket_off + ll128_out_off(R.B->numel));
}
__device__ __forceinline__ char* ll128_in(const BucketRun& R, int rank, int slot) {
  return ll128_out(R, rank) + 128 * ll128_lines(R.B->numel) * (1 + (uint64_t)slot);
}
// lines of shard s handled by this CTA (tile X.j of X.G)
__device__ __forceinline__ void ll128_part(const BucketRun& R, int s, uint64_t& l0, uint64_t& l1) {
  const uint64_t L = ll128_lines(R.B->numel);
  const int p = R.X.world;
  const uint64_t a = split_at(L, p, s), b = split_at(L, p, s + 1);
  l0 = a + split_at(b - a, R.X.G, R.X.j);
  l1 = a + split_at(b - a, R.X.G, R.X.j + 1);
}
// Poll one line (this lane's 16 B) until the group's flag word carries `epoch`.
// Every lane of the warp calls (groups of 8 lanes, possibly different lines or
// none: active = false).  Returns the lane's 16 B; `bad` set on a watchdog.
__device__ __forceinline__ uint4 ll128_wait(const char* line, bool active, uint32_t epoch, const Env& E, int& bad) {
  const int lane = threadIdx.x & 31, k = lane & 7, g7 = (lane & ~7) | 7;
  uint4 v = active ? ll128_ld(line + 16 * k) : make_uint4(0, 0, 0, 0);
  bool ok = !active || (k == 7 ? (v.z == epoch && v.w == epoch) : true);
  ok = __shfl_sync(0xffffffffu, ok ? 1 : 0, g7) != 0;
  if (__all_sync(0xffffffffu, ok)) return v;
  const uint64_t t0 = globaltimer();
  uint32_t spins = 0;
  while (!__all_sync(0xffffffffu, ok || bad)) {
    if (!ok && !bad) {
      v = ll128_ld(line + 16 * k);
      if ((++spins & 1023u) == 0) {
        if (poisoned(E)) bad = 1;
        else if (globaltimer() - t0 > E.timeout_ns) {
          raise_timeout(E);
          bad = 1;
        }
      }
    }
    bool mine_ok = !active || (k == 7 ? (v.z == epoch && v.w == epoch) : true);
    ok = __shfl_sync(0xffffffffu, mine_ok ? 1 : 0, g7) != 0;
  }
  return v;
}

// A: my contribution to every line of every shard -> the owner's in-slot `me`
__device__ void phase_ll128_scatter(const BucketRun& R) {
  const int me = R.X.me, p = R.X.world, k = threadIdx.x & 7;
  const uint64_t n = R.B->numel;
  const bool pack = R.B->flags & CARAMEL_F_PACK;
  const float* bkt = R.bucket(me);
  Cursor gc;
  cur_init(gc, R.segs, R.B->nseg);
  const uint32_t ep = R.X.epoch;
  const int groups = blockDim.x / 8, gid = threadIdx.x / 8;
  for (int t = 0; t < p; ++t) {
    const int s = (me + t) % p;  // rotated: every link starts busy
    uint64_t l0, l1;
    ll128_part(R, s, l0, l1);
    char* dst = ll128_in(R, s, me);
    for (uint64_t L = l0 + gid; L < l1; L += groups) {
      float f[4];
      const int nf = k == 7 ? 2 : 4;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint64_t e = LL128_FLOATS * L + 4 * k + i;
        f[i] = (i < nf && e < n) ? (pack ? seg_ld1(gc, e, 0) : ld1(bkt + e)) : 0.f;
      }
      uint4 v = make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]), __float_as_uint(f[3]));
      if (k == 7) v.z = v.w = ep;
      ll128_st(dst + 128 * L + 16 * k, v);
    }
  }
}

// B: my shard's lines -- every source in rank order, epilogue, result to every rank's out
template <int NP>
__device__ void phase_ll128_reduce(const BucketRun& R) {
  const int me = R.X.me, k = threadIdx.x & 7;
  const uint64_t n = R.B->numel;
  const uint32_t ep = R.X.epoch;
  const bool sgd = R.B->epilogue == CARAMEL_EPI_SGD;
  const float* th = R.theta_flat();
  Cursor tc;
  cur_init(tc, R.segs, R.B->nseg);
  uint64_t l0, l1;
  ll128_part(R, me, l0, l1);
  const int groups = blockDim.x / 8, gid = threadIdx.x / 8;
  const uint64_t iters = (l1 - l0 + groups - 1) / groups;  // warp-uniform trip count
  int bad = 0;
  for (uint64_t it = 0; it < iters; ++it) {
    const uint64_t L = l0 + gid + it * groups;
    const bool active = L < l1;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const uint4 v = ll128_wait(ll128_in(R, me, q) + 128 * L, active, ep, *R.E, bad);
      const float f[4] = {__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w)};
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = q == 0 ? f[i] : __fadd_rn(acc[i], f[i]);
    }
    if (!active || bad) continue;  // nothing derived from a missing input is stored
    const int nf = k == 7 ? 2 : 4;
    float o[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint64_t e = LL128_FLOATS * L + 4 * k + i;
      if (i < nf && e < n) {
        const float t = sgd ? (th ? ld1(th + e) : seg_ld1(tc, e, 1)) : 0.f;
        o[i] = epi1(R.B->epilogue, acc[i], t, R.B->scale, R.B->lr);
      }
    }
    uint4 v = make_uint4(__float_as_uint(o[0]), __float_as_uint(o[1]), __float_as_uint(o[2]), __float_as_uint(o[3]));
    if (k == 7) v.z = v.w = ep;
#pragma unroll
    for (int q = 0; q < NP; ++q) ll128_st(ll128_out(R, (me + q) % NP) + 128 * L + 16 * k, v);
  }
}

// C: my part of every shard's result lines -> parameter arena / bucket / members
__device__ void phase_ll128_finish(const BucketRun& R) {
  const int me = R.X.me, p = R.X.world, k = threadIdx.x & 7;
  const uint64_t n = R.B->numel;
  const uint32_t ep = R.X.epoch;
  const bool unpack = (R.B->flags & CARAMEL_F_UNPACK) && !R.arena;
  const int which = R.B->epilogue == CARAMEL_EPI_SGD ? 1 : 0;
  float* res = R.arena ? R.out(me) : R.bucket(me);
  Cursor uc;
  cur_init(uc, R.segs, R.B->nseg);
  const char* in = ll128_out(R, me);
  const int groups = blockDim.x / 8, gid = threadIdx.x / 8;
  int bad = 0;
  for (int s = 0; s < p; ++s) {
    uint64_t l0, l1;
    ll128_part(R, s, l0, l1);
    const uint64_t iters = (l1 - l0 + groups - 1) / groups;
    for (uint64_t it = 0; it < iters; ++it) {
      const uint64_t L = l0 + gid + it * groups;
      const bool active = L < l1;
      const uint4 v = ll128_wait(in + 128 * L, active, ep, *R.E, bad);
      if (!active || bad) continue;
      const float f[4] = {__uint_as_float(v.x), __uint_as_float(v.y), __uint_as_float(v.z), __uint_as_float(v.w)};
      const int nf = k == 7 ? 2 : 4;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint64_t e = LL128_FLOATS * L + 4 * k + i;
        if (i < nf && e < n) {
          if (unpack) seg_st1(uc, e, which, f[i]);
          else st1(res + e, f[i]);
        }
      }
    }
  }
}

// phase 3: (shuffle) wait for every rank's all-gather; fused unpack; (ring/hd)
// release the buffers I read from
template <int PAT>
__device__ void phase_finish(const BucketRun& R) {
  const int me = R.X.me, p = R.X.world;
  if (PAT == CARAMEL_SHUFFLE)
    for (int c = 0; c < R.B->depth; ++c)
      if (R.mine(c)) R.X.wait_all(c, SLOT_DONE, R.X.epoch);
  if ((R.B->flags & CARAMEL_F_UNPACK) && !R.arena) {
    const bool to_param = (R.B->epilogue == CARAMEL_EPI_SGD);
    const float* res = R.out(me);
    for (int c = 0; c < R.B->depth; ++c) {
      for (int s = 0; s < p && R.mine(c); ++s) {
        uint64_t lo, hi;
        R.shard(c, s, lo, hi);
        unpack_range(R.segs, R.B->nseg, res, lo, hi, to_param, *R.tab);
      }
    }
  }
  if (PAT != CARAMEL_SHUFFLE) {
    int tg[MAXR];
    int nt = 0;
    if (PAT == CARAMEL_RING) {
      tg[nt++] = (me + p - 1) % p;
    } else {
      for (int d = 1; d < p; d <<= 1) tg[nt++] = me ^ d;
    }
    R.X.publish(0, R.X.ns - 1, tg, nt);
  }
}

// Publish `slot` for every chunk of this CTA's tile to every rank after ONE
// fence (a .sys release costs about an NVLink round trip once remote stores
// are outstanding; one per chunk made depth > 1 slower, not faster).
__device__ __forceinline__ void publish_chunks(const BucketRun& R, int slot) {
  __syncthreads();
  if (threadIdx.x < 32) {
    fence_acq_rel_sys();
    const int p = R.X.world;
    for (int idx = threadIdx.x; idx < R.B->depth * p; idx += 32)
      if (R.mine(idx / p)) st_relaxed_sys(R.X.flag(idx % p, idx / p, slot, R.X.me), R.X.epoch);
  }
}

template <int PAT, int NP>
__device__ __forceinline__ void run_bucket(const Env& E, const caramel_bucket& B, int lr_idx, uint32_t epoch,
                                           int j) {
  BucketRun R;
  make_run(R, E, B, PAT, lr_idx, epoch, j);
  if (use_ll(PAT, E.world, B.numel)) {
    phase_ll_scatter(R);
    phase_ll_reduce<NP>(R);
    phase_ll_finish(R);
    return;
  }
  if (use_ll128(PAT, E.world, B.numel)) {
    phase_ll128_scatter(R);
    phase_ll128_reduce<NP>(R);
    phase_ll128_finish(R);
    return;
  }
  if (PAT == CARAMEL_SHUFFLE) {
    // all chunks packed, one publication; all chunks reduced and gathered,
    // one publication (consumers still wait per chunk)
    phase_pack<PAT, true>(R);
    publish_chunks(R, SLOT_READY);
    phase_shuffle<NP, true>(R);
    publish_chunks(R, SLOT_DONE);
  } else {
    phase_pack<PAT>(R);
    if (PAT == CARAMEL_RING) phase_ring(R);
    else phase_hd(R);
  }
  phase_finish<PAT>(R);
}

__global__ void k_epoch_advance(uint32_t* e) { *e += 1; }

static_assert(THREADS >= 62 * CARAMEL_MAX_DEPTH, "rs_ag_multi: one thread per scalar head/tail element");
template <int PAT, int NP>
__global__ void __launch_bounds__(THREADS, 1) k_collective(const __grid_constant__ KParams P) {
  const int lr_idx = blockIdx.y;
  // local copies: the phases hold pointers to these, and generic pointers to
  // kernel parameters are not valid across real device-function calls
  const Env E = P.env;
  if (cta_poisoned(E)) return;
  const caramel_bucket B = P.b;
  const bool autoep = (B.flags & CARAMEL_F_AUTO_EPOCH) && !E.epoch;
  run_bucket<PAT, NP>(E, B, lr_idx, launch_epoch(E) + (autoep ? 1 : 0), blockIdx.x);
  if (autoep) {
    // one kernel per call: the last CTA to finish advances the device epoch.
    // Every CTA consumed its entry read of the counter in its flag waits
    // before it gets here, and the next launch on the stream sees the new
    // value at the kernel boundary -- no fence (a gpu-scope fence would also
    // wait for this CTA's outstanding NVLink stores)
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(E.epoch_dev + 1, 1u) == gridDim.x * gridDim.y - 1) {
      E.epoch_dev[1] = 0;
      E.epoch_dev[0] += 1;
    }
  }
}

// world == 1, many buckets: the concatenated element space is tiled evenly
// over the grid; a tile's pieces may come from several buckets and are all
// described in one batch (prefix[0..nb] element prefix sums, prefix[nb+1 ..
// 2nb+1] member-segment prefix sums).
#define SMEM_PREFIX 512
__global__ void __launch_bounds__(THREADS, 2) k_local_many(const __grid_constant__ MParams P) {
  const int lr_idx = blockIdx.y;
  const Env E = P.env;
  // prefix arrays in shared memory (the binary searches below are otherwise
  // chains of dependent global loads at the start of every CTA)
  __shared__ uint64_t s_pre[SMEM_PREFIX + 1], s_spre[SMEM_PREFIX + 1];
  const bool cached = P.nb <= SMEM_PREFIX;
  if (cached) {
    for (int i = threadIdx.x; i <= P.nb; i += blockDim.x) {
      s_pre[i] = P.prefix[i];
      s_spre[i] = P.segprefix[i];
    }
    __syncthreads();
  }
  const uint64_t* pre = cached ? s_pre : P.prefix;
  const uint64_t* spre = cached ? s_spre : P.segprefix;
  uint64_t lo, hi;
  tile_of(pre[0], pre[P.nb], gridDim.x, blockIdx.x, lo, hi);
  if (lo >= hi) return;
  auto bucket_of = [&](const uint64_t* arr, uint64_t x) {  // last i with arr[i] <= x
    int a = 0, b = P.nb - 1;
    while (a < b) {
      int m = (a + b + 1) >> 1;
      if (arr[m] <= x) a = m; else b = m - 1;
    }
    return a;
  };
  // first / last member segment (global numbering) overlapping [lo, hi)
  const int ba = bucket_of(pre, lo), bb = bucket_of(pre, hi - 1);
  const caramel_bucket Ba = P.bs[ba], Bb = P.bs[bb];
  const bool members = local_needs_members(Ba);  // uniform over a list (same flags/epilogue)
  if (!members) {
    for (int i = ba; i <= bb; ++i) {
      const caramel_bucket B = P.bs[i];
      const uint64_t l = lo > pre[i] ? lo - pre[i] : 0;
      const uint64_t h = (hi < pre[i] + B.numel ? hi : pre[i] + B.numel) - pre[i];
      local_range(E, B, lr_idx, l, h, g_tab);
    }
    return;
  }
  const caramel_segment* sa = reinterpret_cast<const caramel_segment*>(Ba.segs) + (uint64_t)lr_idx * Ba.nseg;
  const caramel_segment* sb = reinterpret_cast<const caramel_segment*>(Bb.segs) + (uint64_t)lr_idx * Bb.nseg;
  const uint64_t g0 = spre[ba] + first_seg(sa, Ba.nseg, lo - pre[ba]);
  const uint64_t g1 = spre[bb] + first_seg(sb, Bb.nseg, hi - 1 - pre[bb]);
  run_pieces<OP_EPI>((int)(g1 - g0 + 1), [&](int i, PieceDesc& d) {
    const uint64_t gs = g0 + i;
    const int bi = bucket_of(spre, gs);
    const caramel_bucket B = P.bs[bi];
    const caramel_segment* segs = reinterpret_cast<const caramel_segment*>(B.segs) + (uint64_t)lr_idx * B.nseg;
    const Seg sg = load_seg(segs, (int)(gs - spre[bi]));
    const uint64_t l = lo > pre[bi] ? lo - pre[bi] : 0;
    const uint64_t h = (hi < pre[bi] + B.numel ? hi : pre[bi] + B.numel) - pre[bi];
    uint64_t x0, x1;
    if (clip_seg(sg, l, h, x0, x1)) local_piece(E, B, lr_idx, sg, x0, x1, d);
  }, g_tab);
}

__global__ void __launch_bounds__(THREADS, 2) k_local(const __grid_constant__ KParams P) {
  uint64_t lo, hi;
  tile_of(0, P.b.numel, gridDim.x, blockIdx.x, lo, hi);
  const Env E = P.env;
  const caramel_bucket B = P.b;
  local_range(E, B, blockIdx.y, lo, hi, g_tab);
}

// ---------------------------------------------------------------------------
// Fused two-shot over a whole bucket list (all gradients ready: the
// back-to-back aggregation pass).  Three flat phases separated by cross-rank
// grid barriers instead of per-bucket flags:
//   0  pack every member into my bucket region (local HBM, warp-item engine
//      over the concatenated element space, tiled evenly over the grid)
//   1  for every (bucket, chunk): pull my shard from every rank's bucket,
//      sum in ascending rank order, epilogue (fused SGD), push the result
//      into every rank's output -- warp items of 256 elements tiled evenly
//      over the grid, 2*NP float4 loads in flight per lane
//   2  (results in buckets + CARAMEL_F_UNPACK) scatter to the members
// Ownership of every element follows the per-bucket chunk/shard rule.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t* sync_words(const Env& E, int rank) {
  return reinterpret_cast<uint32_t*>(E.arena[rank] + E.sync_off);
}

// Grid barrier k across every CTA of every rank (launch sequence value S).
// Arrive: fence.acq_rel.sys, then a counter RMW; the last CTA of a rank
// acquires the others' arrivals with its own fence and releases a flag to
// every rank; everybody waits for all ranks' flags.
__device__ void grid_barrier(const Env& E, int me, int k, uint32_t S) {
  __syncthreads();
  int bad = 0;
  if (threadIdx.x == 0) {
    uint32_t* mine = sync_words(E, me);
    // arrive with a gpu-scope release (covers this CTA's writes through the
    // bar.sync above); the last arriver acquires every arrival, and its
    // sys-scope fence before the remote flag stores makes all of them visible
    // to the peers (causality is transitive across the two scopes)
    const uint32_t old = atom_add_acq_rel_gpu(mine + 16 + k, 1u);
    if (old == gridDim.x - 1) {
      atomicExch(mine + 16 + k, 0u);
      if (k == 0) atomicAdd(mine, 1u);  // launch sequence: everybody has read it
      if (k == 1) atomicExch(mine + 48, 0u);  // k_shuffle_fused's item counter: nobody claims past barrier 1
      fence_acq_rel_sys();
      for (int q = 0; q < E.world; ++q) st_relaxed_sys(sync_words(E, q) + 64 + k * MAXR + me, S + 1);
    }
    for (int q = 0; q < E.world && !bad; ++q) {
      const uint32_t* f = mine + 64 + k * MAXR + q;
      if (ld_acquire_sys(f) >= S + 1) continue;
      const uint64_t t0 = globaltimer();
      uint32_t spins = 0;
      while (ld_acquire_sys(f) < S + 1) {
        if ((++spins & 1023u) == 0) {
          if (poisoned(E)) { bad = 1; break; }
          if (globaltimer() - t0 > E.timeout_ns) {
            raise_timeout(E);
            bad = 1;
            break;
          }
        }
      }
    }
  }
  cta_abort_if(bad);
}

// items of my shard range [lo, hi): one edge item (scalar head + tail) and
// vector items of 64 float4 over the 4-aligned interior
// float4s per lane per item of the fused NVLink phase: about 8 loads in
// flight per lane whatever p is (V * NP), at least 2
template <int NP>
#ifndef CARAMEL_FUSED_V2
#define CARAMEL_FUSED_V2 4
#endif
struct FusedV { static constexpr int V = NP >= 4 ? 2 : NP == 2 ? CARAMEL_FUSED_V2 : 8 / NP; };

// items of my shard range [lo, hi): one edge item (scalar head + tail) and
// one per 32*V float4s of the 16-byte aligned interior
// The vector interior [a, e) of a shard starts and ends on 128-byte lines
// (32 floats), so a warp's 32 float4s cover 4 lines, not 5 (a bucket's shard
// boundaries fall anywhere: most shards were misaligned).
__device__ __forceinline__ void line_interior(uint64_t lo, uint64_t hi, uint64_t& a, uint64_t& e) {
  a = (lo + 31) & ~31ull;
  e = hi & ~31ull;
}

template <int V>
__device__ __forceinline__ uint32_t shard_items(uint64_t lo, uint64_t hi) {
  if (lo >= hi) return 0;
  uint64_t a, e;
  line_interior(lo, hi, a, e);
  return 1 + (e > a ? (uint32_t)(((e - a) / 4 + 32 * V - 1) / (32 * V)) : 0);
}

struct FusedShared {
  uint32_t bpre[MAX_FUSED_BUCKETS + 1];
};

template <int NP>
__global__ void __launch_bounds__(THREADS, 1) k_shuffle_fused(const __grid_constant__ MParams P) {
  __shared__ FusedShared sh;
  const Env E = P.env;
  if (cta_poisoned(E)) return;
  const int lr_idx = blockIdx.y;
  const int me = E.rank_base + lr_idx;
  const uint32_t S = *reinterpret_cast<volatile uint32_t*>(sync_words(E, me));
  const caramel_bucket B0 = P.bs[0];
  const bool arena = (B0.flags & CARAMEL_F_PARAM_ARENA) && B0.epilogue == CARAMEL_EPI_SGD;
  const uint64_t* pre = P.prefix;
  const uint64_t* spre = P.segprefix;
  auto bucket_of = [&](const uint64_t* arr, uint64_t x) {  // last i with arr[i] <= x
    int a = 0, b = P.nb - 1;
    while (a < b) {
      int m = (a + b + 1) >> 1;
      if (arr[m] <= x) a = m; else b = m - 1;
    }
    return a;
  };
  // ---- phase 0: pack ---------------------------------------------------------
  if (B0.flags & CARAMEL_F_PACK) {
    uint64_t lo, hi;
    tile_of(pre[0], pre[P.nb], gridDim.x, blockIdx.x, lo, hi);
    if (lo < hi) {
      const int ba = bucket_of(pre, lo), bb = bucket_of(pre, hi - 1);
      const caramel_bucket Ba = P.bs[ba], Bb = P.bs[bb];
      const caramel_segment* sa = reinterpret_cast<const caramel_segment*>(Ba.segs) + (uint64_t)lr_idx * Ba.nseg;
      const caramel_segment* sb = reinterpret_cast<const caramel_segment*>(Bb.segs) + (uint64_t)lr_idx * Bb.nseg;
      const uint64_t g0 = spre[ba] + first_seg(sa, Ba.nseg, lo - pre[ba]);
      const uint64_t g1 = spre[bb] + first_seg(sb, Bb.nseg, hi - 1 - pre[bb]);
      run_pieces<OP_COPY>((int)(g1 - g0 + 1), [&](int i, PieceDesc& d) {
        const uint64_t gs = g0 + i;
        const int bi = bucket_of(spre, gs);
        const caramel_bucket B = P.bs[bi];
        const caramel_segment* segs = reinterpret_cast<const caramel_segment*>(B.segs) + (uint64_t)lr_idx * B.nseg;
        const Seg sg = load_seg(segs, (int)(gs - spre[bi]));
        const uint64_t l = lo > pre[bi] ? lo - pre[bi] : 0;
        const uint64_t h = (hi < pre[bi] + B.numel ? hi : pre[bi] + B.numel) - pre[bi];
        uint64_t x0, x1;
        if (!clip_seg(sg, l, h, x0, x1)) return;
        d.g = reinterpret_cast<const float*>(sg.grad) + (x0 - sg.offset);
        d.o = reinterpret_cast<float*>(E.arena[me] + B.bucket_off) + x0;
        d.n = (uint32_t)(x1 - x0);
      }, g_tab);
    }
  }
  grid_barrier(E, me, 0, S);

  // ---- phase 1: reduce my shards, epilogue, all-gather by store --------------
  {
    // per-bucket item prefix of my shards (block scan in batches)
    uint32_t carry = 0;
    for (int b0 = 0; b0 < P.nb; b0 += blockDim.x) {
      const int i = b0 + threadIdx.x;
      uint32_t cnt = 0;
      if (i < P.nb) {
        const caramel_bucket B = P.bs[i];
        for (int c = 0; c < B.depth; ++c) {
          uint64_t lo, hi;
          shard_bounds(B.numel, B.depth, E.world, c, me, lo, hi);
          cnt += shard_items<FusedV<NP>::V>(lo, hi);
        }
      }
      uint32_t excl;
      const uint32_t tot = block_scan(cnt, &excl, g_tab.scratch);
      if (i < P.nb) sh.bpre[i] = carry + excl;
      carry += tot;
    }
    if (threadIdx.x == 0) sh.bpre[P.nb] = carry;
    __syncthreads();
    const uint32_t T = carry;
    const uint32_t it0 = (uint32_t)(((uint64_t)T * blockIdx.x) / gridDim.x);
    const uint32_t it1 = (uint32_t)(((uint64_t)T * (blockIdx.x + 1)) / gridDim.x);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // dynamic: warps claim P.claim consecutive items from a per-rank counter
    // (sync word 48, zeroed by the last arriver of the closing barrier), so a
    // warp slowed by remote latency takes fewer items instead of the grid
    // waiting for the slowest static slice
    unsigned int* claim_ctr = sync_words(E, me) + 48;
    const uint32_t claim = (uint32_t)P.claim;
    uint32_t c_it = 0, c_end = 0;
    int bc = -1;
    caramel_bucket B;
    Cursor tc;
    for (uint32_t it = claim ? 0 : it0 + w;; it = claim ? it + 1 : it + nw) {
      if (claim) {
        if (c_it >= c_end) {
          uint32_t base = 0;
          if (lane == 0) base = atomicAdd(claim_ctr, claim);
          base = __shfl_sync(0xffffffffu, base, 0);
          c_it = base;
          c_end = base + claim < T ? base + claim : T;
        }
        if (c_it >= T) break;
        it = c_it++;
      } else if (it >= it1) {
        break;
      }
      if (bc < 0 || sh.bpre[bc + 1] <= it) {
        int a = bc < 0 ? 0 : bc, b = P.nb - 1;
        while (a < b) {
          int m = (a + b + 1) >> 1;
          if (sh.bpre[m] <= it) a = m; else b = m - 1;
        }
        bc = a;
        B = P.bs[bc];
        cur_init(tc, reinterpret_cast<const caramel_segment*>(B.segs) + (uint64_t)lr_idx * B.nseg, B.nseg);
      }
      uint32_t li = it - sh.bpre[bc];
      uint64_t lo = 0, hi = 0;
      for (int c = 0; c < B.depth; ++c) {
        shard_bounds(B.numel, B.depth, E.world, c, me, lo, hi);
        const uint32_t n = shard_items<FusedV<NP>::V>(lo, hi);
        if (li < n) break;
        li -= n;
      }
      const float* src[NP];
      float* dst[NP];
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        src[q] = reinterpret_cast<const float*>(E.arena[q] + B.bucket_off);
        dst[q] = arena ? reinterpret_cast<float*>(E.parena[q] + B.param_off)
                       : reinterpret_cast<float*>(E.arena[q] + B.bucket_off);
      }
      const float* th = arena ? reinterpret_cast<const float*>(E.parena[me] + B.param_off) : nullptr;
      const bool sgd = B.epilogue == CARAMEL_EPI_SGD;
      uint64_t a, e;
      line_interior(lo, hi, a, e);
      if (li == 0) {  // edge item: scalar head [lo, a) and tail [e, hi) (whole range if no interior)
        const bool interior = e > a;
        const uint64_t n_head = interior ? a - lo : hi - lo;
        const uint64_t n_tail = interior ? hi - e : 0;
        for (uint64_t l = lane; l < n_head + n_tail; l += 32) {
          const uint64_t x = l < n_head ? lo + l : e + (l - n_head);
          float acc = ld1(src[0] + x);
#pragma unroll
          for (int q = 1; q < NP; ++q) acc = __fadd_rn(acc, ld1(src[q] + x));
          const float t = sgd ? (arena ? ld1(th + x) : seg_ld1(tc, x, 1)) : 0.f;
          const float o = epi1(B.epilogue, acc, t, B.scale, B.lr);
#pragma unroll
          for (int q = 0; q < NP; ++q) st1(dst[q] + x, o);
        }
        continue;
      }
      // vector item li-1: float4 [32V (li-1), 32V li) of the interior; lane
      // does V of them (all V*NP loads issued before the first store)
      constexpr int V = FusedV<NP>::V;
      const uint64_t nv = (e - a) / 4;
      const uint64_t vb = 32ull * V * (li - 1) + lane;
      float4 p[V][NP], t[V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const uint64_t vi = vb + 32ull * v;
        const bool ok = vi < nv;
        const uint64_t x = a + 4 * vi;
#pragma unroll
        for (int q = 0; q < NP; ++q) p[v][q] = ok ? ld4(src[q] + x) : make_float4(0.f, 0.f, 0.f, 0.f);
        t[v] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (sgd && ok) t[v] = arena ? ld4(th + x) : seg_ld4(tc, x, 1);
      }
#pragma unroll
      for (int v = 0; v < V; ++v) {
        const uint64_t vi = vb + 32ull * v;
        if (vi >= nv) continue;
        const uint64_t x = a + 4 * vi;
        float4 sum = p[v][0];
#pragma unroll
        for (int q = 1; q < NP; ++q) sum = add4(sum, p[v][q]);
        const float4 o = epi4(B.epilogue, sum, t[v], B.scale, B.lr);
#pragma unroll
        for (int q = 0; q < NP; ++q) st4(dst[q] + x, o);
      }
    }
  }
  grid_barrier(E, me, 1, S);

  // ---- phase 2: unpack (results live in the buckets) --------------------------
  if ((B0.flags & CARAMEL_F_UNPACK) && !arena) {
    const bool to_param = B0.epilogue == CARAMEL_EPI_SGD;
    uint64_t lo, hi;
    tile_of(pre[0], pre[P.nb], gridDim.x, blockIdx.x, lo, hi);
    if (lo < hi) {
      const int ba = bucket_of(pre, lo), bb = bucket_of(pre, hi - 1);
      const caramel_bucket Ba = P.bs[ba], Bb = P.bs[bb];
      const caramel_segment* sa = reinterpret_cast<const caramel_segment*>(Ba.segs) + (uint64_t)lr_idx * Ba.nseg;
      const caramel_segment* sb = reinterpret_cast<const caramel_segment*>(Bb.segs) + (uint64_t)lr_idx * Bb.nseg;
      const uint64_t g0 = spre[ba] + first_seg(sa, Ba.nseg, lo - pre[ba]);
      const uint64_t g1 = spre[bb] + first_seg(sb, Bb.nseg, hi - 1 - pre[bb]);
      run_pieces<OP_COPY>((int)(g1 - g0 + 1), [&](int i, PieceDesc& d) {
        const uint64_t gs = g0 + i;
        const int bi = bucket_of(spre, gs);
        const caramel_bucket B = P.bs[bi];
        const caramel_segment* segs = reinterpret_cast<const caramel_segment*>(B.segs) + (uint64_t)lr_idx * B.nseg;
        const Seg sg = load_seg(segs, (int)(gs - spre[bi]));
        const uint64_t l = lo > pre[bi] ? lo - pre[bi] : 0;
        const uint64_t h = (hi < pre[bi] + B.numel ? hi : pre[bi] + B.numel) - pre[bi];
        uint64_t x0, x1;
        if (!clip_seg(sg, l, h, x0, x1)) return;
        d.g = reinterpret_cast<const float*>(E.arena[me] + B.bucket_off) + x0;
        d.o = reinterpret_cast<float*>(to_param ? sg.param : sg.grad) + (x0 - sg.offset);
        d.n = (uint32_t)(x1 - x0);
      }, g_tab);
    }
  }
}

// ---------------------------------------------------------------------------
// TMA bulk-copy streaming (world == 1, flat buckets): one CTA per SM, tiles of
// TT floats staged in shared memory by cp.async.bulk (completion on an
// mbarrier), the update computed in shared memory, the new parameters written
// back with a bulk store -- bytes in flight live in shared memory, not in
// registers, so a handful of warps keep HBM busy.
// ---------------------------------------------------------------------------
// TT floats per tile, TS pipeline stages (TS-2 tiles of loads in flight per
// SM): template parameters of the kernel, default 8192 x 3 (32 KB tiles)
#define TMA_THREADS 256
#define TMA_MAX_BUCKETS 256

struct TmaBucket {  // per-bucket pointers cached in shared memory
  const float* g;
  float* t;
  uint64_t numel;
  float scale, lr;
};

template <int TT, int TS>
struct TmaSmem {
  float g[TS][TT];
  float t[TS][TT];
  uint64_t bar[TS];
  uint32_t tpre[TMA_MAX_BUCKETS + 1];
  TmaBucket b[TMA_MAX_BUCKETS];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
      "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* sdst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(sdst)),
               "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_u32(ssrc)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// world == 1, every bucket CARAMEL_F_FLAT + PACK + PARAM_ARENA + SGD:
// theta[b] <- theta[b] - lr * (grad[b] * scale), tile by tile.
template <int TT, int TS>
__global__ void __launch_bounds__(TMA_THREADS, 2) k_local_flat_tma(const __grid_constant__ MParams P) {
  extern __shared__ __align__(128) unsigned char dyn_smem[];
  TmaSmem<TT, TS>& S = *reinterpret_cast<TmaSmem<TT, TS>*>(dyn_smem);
  const Env E = P.env;
  const int me = E.rank_base + blockIdx.y;
  // tile prefix over the buckets
  uint32_t carry = 0;
  __shared__ uint32_t scan_scratch[32];
  for (int b0 = 0; b0 < P.nb; b0 += blockDim.x) {
    const int i = b0 + threadIdx.x;
    uint32_t cnt = 0;
    if (i < P.nb) {
      const caramel_bucket B = P.bs[i];
      cnt = (uint32_t)((B.numel + TT - 1) / TT);
      if (B.flags & CARAMEL_F_PACK) {
        const caramel_segment* segs = reinterpret_cast<const caramel_segment*>(B.segs) + (uint64_t)blockIdx.y * B.nseg;
        S.b[i].g = reinterpret_cast<const float*>(__ldg(reinterpret_cast<const unsigned long long*>(segs)));
      } else {
        S.b[i].g = reinterpret_cast<const float*>(E.arena[me] + B.bucket_off);
      }
      S.b[i].t = reinterpret_cast<float*>(E.parena[me] + B.param_off);
      S.b[i].numel = B.numel;
      S.b[i].scale = B.scale;
      S.b[i].lr = B.lr;
    }
    uint32_t excl;
    const uint32_t tot = block_scan(cnt, &excl, scan_scratch);
    if (i < P.nb) S.tpre[i] = carry + excl;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    S.tpre[P.nb] = carry;
    for (int s = 0; s < TS; ++s) mbar_init(&S.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t T = carry, G = gridDim.x;
  // tile t -> bucket, element offset, length, global pointers
  struct Tile {
    const float* g;
    float* t;
    uint32_t len;
    float scale, lr;
  };
  auto tile = [&](uint32_t t) {
    int a = 0, b = P.nb - 1;
    while (a < b) {
      const int m = (a + b + 1) >> 1;
      if (S.tpre[m] <= t) a = m; else b = m - 1;
    }
    const TmaBucket& B = S.b[a];
    const uint64_t o = (uint64_t)(t - S.tpre[a]) * TT;
    Tile r;
    r.g = B.g + o;
    r.t = B.t + o;
    r.len = (uint32_t)((B.numel - o) < TT ? (B.numel - o) : TT);
    r.scale = B.scale;
    r.lr = B.lr;
    return r;
  };
  auto issue = [&](uint32_t k) {  // thread 0 only
    const uint32_t t = blockIdx.x + k * G;
    if (t >= T) return;
    const Tile r = tile(t);
    const int s = k % TS;
    const uint32_t vb = (r.len & ~3u) * 4;
    mbar_expect_tx(&S.bar[s], 2 * vb);
    if (vb) {
      bulk_load(S.g[s], r.g, vb, &S.bar[s]);
      bulk_load(S.t[s], r.t, vb, &S.bar[s]);
    }
  };
  const uint32_t K = blockIdx.x < T ? (T - blockIdx.x + G - 1) / G : 0;
  // prefetch distance TS-2: the stage refilled at iteration k held tile k-2,
  // whose bulk store must have finished reading shared memory; the store of
  // tile k-1 may still be in flight (wait_group.read 1)
  if (threadIdx.x == 0)
    for (uint32_t k = 0; k + 2 < TS && k < K; ++k) issue(k);
  for (uint32_t k = 0; k < K; ++k) {
    if (threadIdx.x == 0 && k + TS - 2 < K) {
      bulk_wait_read1();
      issue(k + TS - 2);
    }
    const int s = k % TS;
    mbar_wait(&S.bar[s], (k / TS) & 1);
    const Tile r = tile(blockIdx.x + k * G);
    const uint32_t nv = r.len & ~3u;
    float4* t4 = reinterpret_cast<float4*>(S.t[s]);
    const float4* g4 = reinterpret_cast<const float4*>(S.g[s]);
    for (uint32_t v = threadIdx.x; v < nv / 4; v += blockDim.x)
      t4[v] = epi4(CARAMEL_EPI_SGD, g4[v], t4[v], r.scale, r.lr);
    for (uint32_t e = nv + threadIdx.x; e < r.len; e += blockDim.x)  // < 4 ragged elements
      r.t[e] = epi1(CARAMEL_EPI_SGD, ld1(r.g + e), ld1(r.t + e), r.scale, r.lr);
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0 && nv) {
      bulk_store(r.t, S.t[s], nv * 4);
      bulk_commit();
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

// ---------------------------------------------------------------------------
// K1 / K4 through the TMA unit (caramel_pack / caramel_unpack): the bucket is
// cut into 32 KB tiles; a persistent CTA per SM streams its tiles through a
// 6-stage shared-memory ring.  Pack: every member piece of a tile whose source
// and tile position share their 16-byte phase is one cp.async.bulk load into
// the tile (completion on the stage's mbarrier); the rare misaligned piece is
// copied into the tile by all threads; the whole tile leaves with ONE bulk
// store.  Unpack is the mirror image (one bulk load per tile, one bulk store
// per aligned piece).  Bytes in flight sit in shared memory: no register
// round trip per member (the warp-item engine above stalled on exactly that:
// 53% DRAM throughput, 26.7 of 53.7 cycles per instruction on long scoreboard).
// ---------------------------------------------------------------------------
#define KT_THREADS 256
#ifndef KT_TILE
#define KT_TILE 8192                 // floats per tile (32 KB)
#endif
#ifndef KT_STAGES
#define KT_STAGES 6                  // 4 tiles of loads in flight per SM (HBM latency x bandwidth / 148 SMs ~ 66 KB)
#endif
#ifndef KT_CTAS_PER_SM
#define KT_CTAS_PER_SM 1
#endif
#define KT_MAXODD 32                 // misaligned pieces remembered per tile (more: the tile goes plain)
#ifndef KT_MAXSEG
#define KT_MAXSEG 512                // member tables up to this size are cached in shared memory
#endif

struct KtOdd { uint64_t src, dst; uint32_t n; };  // a misaligned piece: element addresses, count

struct KtSmem {
  float tile[KT_STAGES][KT_TILE];
  uint64_t full[KT_STAGES];
  KtOdd odd[KT_STAGES][KT_MAXODD];
  int nodd[KT_STAGES];               // -1: copy the whole tile plainly
  caramel_segment segs[KT_MAXSEG];   // the member table (the issuing thread searches it per tile)
};

// Walks the member pieces of bucket range [t0, t1): f(seg, x0, x1) in bucket coordinates.
// (plain generic loads: the table may sit in shared memory)
template <class F>
__device__ __forceinline__ void kt_pieces(const caramel_segment* segs, int nseg, uint64_t t0, uint64_t t1, F f) {
  int a = 0, b = nseg - 1;
  while (a < b) {
    const int m = (a + b + 1) >> 1;
    if (segs[m].offset <= t0) a = m; else b = m - 1;
  }
  for (int i = a; i < nseg; ++i) {
    const Seg sg{segs[i].grad, segs[i].param, segs[i].offset, segs[i].numel};
    if (sg.offset >= t1) break;
    uint64_t x0, x1;
    if (clip_seg(sg, t0, t1, x0, x1)) f(sg, x0, x1);
  }
}

// UNPACK = false: members -> bucket.  UNPACK = true: bucket -> members
// (to_param selects .param instead of .grad).
template <bool UNPACK>
__global__ void __launch_bounds__(KT_THREADS, KT_CTAS_PER_SM) k_pack_tma(const caramel_segment* segs, int nseg, uint64_t numel,
                                                            float* bucket, int to_param) {
  extern __shared__ __align__(128) unsigned char dyn_smem[];
  KtSmem& S = *reinterpret_cast<KtSmem*>(dyn_smem);
  if (nseg <= KT_MAXSEG) {  // one coalesced copy instead of a dependent global load per search step
    for (int i = threadIdx.x; i < 4 * nseg; i += blockDim.x)
      reinterpret_cast<unsigned long long*>(S.segs)[i] = __ldg(reinterpret_cast<const unsigned long long*>(segs) + i);
    __syncthreads();
    segs = S.segs;
  }
  const uint64_t ntiles = (numel + KT_TILE - 1) / KT_TILE;
  const uint64_t G = gridDim.x;
  const uint64_t K = blockIdx.x < ntiles ? (ntiles - blockIdx.x + G - 1) / G : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < KT_STAGES; ++s) mbar_init(&S.full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto member = [&](const Seg& sg) -> float* { return reinterpret_cast<float*>(UNPACK && to_param ? sg.param : sg.grad); };
  // thread 0: start tile k's loads into its stage, remember its misaligned pieces
  auto issue = [&](uint64_t k) {
    const uint64_t t = blockIdx.x + k * G, t0 = t * KT_TILE;
    const uint64_t t1 = t0 + KT_TILE < numel ? t0 + KT_TILE : numel;
    const int s = (int)(k % KT_STAGES);
    float* tile = S.tile[s];
    if (UNPACK) {
      const uint32_t bytes = (uint32_t)(4 * (t1 - t0)) & ~15u;  // the < 4-element tail goes plain (bucket is 16 B aligned)
      mbar_expect_tx(&S.full[s], bytes);
      if (bytes) bulk_load(tile, bucket + t0, bytes, &S.full[s]);
      S.nodd[s] = 0;
      return;
    }
    uint32_t tx = 0;
    int nodd = 0;
    // count the bulk bytes first: expect_tx must precede the loads' completion
    kt_pieces(segs, nseg, t0, t1, [&](const Seg& sg, uint64_t x0, uint64_t x1) {
      const uintptr_t src = (uintptr_t)(member(sg) + (x0 - sg.offset));
      if (((src ^ (uintptr_t)(4 * (x0 - t0))) & 15) == 0) {
        const uint64_t a = (x0 + 3) & ~3ull, b = x1 & ~3ull;
        if (b > a) tx += (uint32_t)(4 * (b - a));
      }
    });
    mbar_expect_tx(&S.full[s], tx);
    kt_pieces(segs, nseg, t0, t1, [&](const Seg& sg, uint64_t x0, uint64_t x1) {
      const float* src = member(sg) + (x0 - sg.offset);
      const bool co = (((uintptr_t)src ^ (uintptr_t)(4 * (x0 - t0))) & 15) == 0;
      uint64_t a = x0, b = x0;
      if (co) {
        a = (x0 + 3) & ~3ull;
        b = x1 & ~3ull;
        if (b < a) b = a;
        if (a > x1) a = b = x1;
        if (b > a) bulk_load(tile + (a - t0), src + (a - x0), (uint32_t)(4 * (b - a)), &S.full[s]);
      }
      // ragged ends / misaligned piece: remembered for the plain copy
      const uint64_t parts[2][2] = {{x0, co ? a : x1}, {co ? b : x1, x1}};
      for (int h = 0; h < 2; ++h) {
        const uint64_t y0 = parts[h][0], y1 = parts[h][1];
        if (y1 <= y0) continue;
        if (nodd < KT_MAXODD)
          S.odd[s][nodd] = KtOdd{(uint64_t)(uintptr_t)(member(sg) + (y0 - sg.offset)), y0 - t0, (uint32_t)(y1 - y0)};
        ++nodd;
      }
    });
    S.nodd[s] = nodd;
  };
  auto bytes_of_tile = [&](uint64_t k) {
    const uint64_t t0 = (blockIdx.x + k * G) * KT_TILE;
    return (uint32_t)(4 * ((t0 + KT_TILE < numel ? t0 + KT_TILE : numel) - t0));
  };
  if (threadIdx.x == 0)
    for (uint64_t k = 0; k + 2 < KT_STAGES && k < K; ++k) issue(k);
  __syncthreads();  // the misaligned-piece lists written by issue() are read by every thread
  for (uint64_t k = 0; k < K; ++k) {
    const int s = (int)(k % KT_STAGES);
    if (threadIdx.x == 0 && k + KT_STAGES - 2 < K) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // the stage refilled held tile k-2
      issue(k + KT_STAGES - 2);
    }
    mbar_wait(&S.full[s], (uint32_t)((k / KT_STAGES) & 1));
    const uint64_t t0 = (blockIdx.x + k * G) * KT_TILE;
    const uint32_t nbytes = bytes_of_tile(k), nel = nbytes / 4;
    float* tile = S.tile[s];
    if (!UNPACK) {
      const int nodd = S.nodd[s];
      if (nodd > KT_MAXODD) {  // too many misaligned pieces: copy the whole tile plainly
        kt_pieces(segs, nseg, t0, t0 + nel, [&](const Seg& sg, uint64_t x0, uint64_t x1) {
          const float* src = member(sg) + (x0 - sg.offset);
          for (uint64_t e = threadIdx.x; e < x1 - x0; e += blockDim.x) tile[x0 - t0 + e] = ld1(src + e);
        });
      } else {
        for (int o = 0; o < nodd; ++o) {
          const KtOdd od = S.odd[s][o];
          for (uint32_t e = threadIdx.x; e < od.n; e += blockDim.x)
            tile[od.dst + e] = ld1(reinterpret_cast<const float*>(od.src) + e);
        }
      }
      fence_proxy_async();
      __syncthreads();
      if (threadIdx.x == 0) {
        const uint32_t vb = nbytes & ~15u;
        if (vb) bulk_store(bucket + t0, tile, vb);
        bulk_commit();
      }
      for (uint32_t e = (nbytes & ~15u) / 4 + threadIdx.x; e < nel; e += blockDim.x) st1(bucket + t0 + e, tile[e]);
    } else {
      for (uint32_t e = (nbytes & ~15u) / 4 + threadIdx.x; e < nel; e += blockDim.x) tile[e] = ld1(bucket + t0 + e);
      __syncthreads();
      // aligned pieces: bulk stores by thread 0; the rest: plain stores by all threads
      if (threadIdx.x == 0) {
        kt_pieces(segs, nseg, t0, t0 + nel, [&](const Seg& sg, uint64_t x0, uint64_t x1) {
          float* dst = member(sg) + (x0 - sg.offset);
          if ((((uintptr_t)dst ^ (uintptr_t)(4 * (x0 - t0))) & 15) != 0) return;
          uint64_t a = (x0 + 3) & ~3ull, b = x1 & ~3ull;
          if (b > a) bulk_store(dst + (a - x0), tile + (a - t0), (uint32_t)(4 * (b - a)));
        });
        bulk_commit();
      }
      kt_pieces(segs, nseg, t0, t0 + nel, [&](const Seg& sg, uint64_t x0, uint64_t x1) {
        float* dst = member(sg) + (x0 - sg.offset);
        const bool co = (((uintptr_t)dst ^ (uintptr_t)(4 * (x0 - t0))) & 15) == 0;
        uint64_t a = (x0 + 3) & ~3ull, b = x1 & ~3ull;
        if (!co || b <= a) a = b = x1;  // everything plain
        for (uint64_t e = x0 + threadIdx.x; e < a; e += blockDim.x) st1(dst + (e - x0), tile[e - t0]);
        for (uint64_t e = b + threadIdx.x; e < x1; e += blockDim.x) st1(dst + (e - x0), tile[e - t0]);
      });
    }
    __syncthreads();  // the stage may be refilled once its store has read it (thread 0 checks)
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

// Many buckets in one launch (launch order).  world == 1: the concatenated
// element space is tiled evenly over the grid.  Shuffle: phase-major -- every
// bucket's pack + ready flags first, then every bucket's reduce/all-gather,
// then every bucket's completion wait -- so no CTA idles on one bucket's
// flags while another bucket's work is available.  Ring/hd: bucket by bucket.
// CTA j takes part in bucket b iff j < b.ctas (same rule on every rank).
template <int PAT, int NP>
__global__ void __launch_bounds__(THREADS, 1) k_collective_many(const __grid_constant__ MParams P) {
  const int lr_idx = blockIdx.y;
  const Env E = P.env;  // local copy: phases keep pointers to it
  if (cta_poisoned(E)) return;
  const uint32_t epoch = launch_epoch(E);
  const int G = gridDim.x;
  // bucket i occupies CTAs base_i .. base_i + ctas_i - 1 (mod G), base_i being
  // the running sum of the previous buckets' CTA counts: small buckets spread
  // over the grid and proceed in parallel.  Same rule on every rank.
  auto my_tile = [&](int base, int ctas) {
    int jj = ((int)blockIdx.x - base) % G;
    if (jj < 0) jj += G;
    return jj < ctas ? jj : -1;
  };
  if (PAT == CARAMEL_SHUFFLE) {
    // Per-bucket-flag list (CARAMEL_MANY_FLAGS): phase-major.  A .sys release
    // waits for every outstanding remote store of the CTA (about one NVLink
    // round trip), so all packs go out, then ONE fence.acq_rel.sys and every
    // READY flag as a relaxed store (READY depends on local work only).  DONE
    // is published per bucket: deferring it would make bucket b's completion
    // wait for bucket b+1's READY, which a rank that launches bucket by bucket
    // only sends after b completes -- a deadlock.  Flags are the same
    // (bucket, chunk, tile) words a single-bucket launch uses, so ranks may
    // group the same launch order into different lists.
    auto publish_deferred = [&](int slot) {
      __syncthreads();
      if (threadIdx.x < 32) {
        fence_acq_rel_sys();
        const int me = E.rank_base + lr_idx, p = E.world;
        int base = 0;
        for (int i = 0; i < P.nb; ++i) {
          const caramel_bucket B = P.bs[i];
          const int j = my_tile(base, B.ctas);
          base = (base + B.ctas) % G;
          if (j < 0 || B.numel == 0 || use_ll(PAT, p, B.numel) || use_ll128(PAT, p, B.numel)) continue;
          const int ns = nslots(PAT, p);
          BucketRun R;
          make_run(R, E, B, PAT, lr_idx, epoch, j);
          for (int idx = threadIdx.x; idx < B.depth * p; idx += 32) {
            const int c = idx / p, q = idx % p;
            if (!R.mine(c)) continue;
            uint32_t* f = reinterpret_cast<uint32_t*>(E.arena[q] + B.flag_off) +
                          ((((uint64_t)c * B.ctas + j) * ns + slot) * p + me);
            st_relaxed_sys(f, epoch);
          }
        }
      }
    };
    for (int phase = 0; phase < 3; ++phase) {
      int base = 0;
      for (int i = 0; i < P.nb; ++i) {
        const caramel_bucket B = P.bs[i];
        const int j = my_tile(base, B.ctas);
        base = (base + B.ctas) % G;
        if (j < 0 || B.numel == 0) continue;
        BucketRun R;
        make_run(R, E, B, PAT, lr_idx, epoch, j);
        if (use_ll(PAT, E.world, B.numel)) {
          if (phase == 0) phase_ll_scatter(R);
          else if (phase == 1) phase_ll_reduce<NP>(R);
          else phase_ll_finish(R);
          continue;
        }
        if (use_ll128(PAT, E.world, B.numel)) {
          if (phase == 0) phase_ll128_scatter(R);
          else if (phase == 1) phase_ll128_reduce<NP>(R);
          else phase_ll128_finish(R);
          continue;
        }
        if (phase == 0) phase_pack<PAT, true>(R);
        else if (phase == 1) phase_shuffle<NP, false>(R);
        else phase_finish<PAT>(R);
      }
      if (phase == 0) publish_deferred(SLOT_READY);
    }
  } else {  // ring / hd: bucket by bucket
    int base = 0;
    for (int i = 0; i < P.nb; ++i) {
      const caramel_bucket B = P.bs[i];
      const int j = my_tile(base, B.ctas);
      base = (base + B.ctas) % G;
      if (j < 0 || B.numel == 0) continue;
      run_bucket<PAT, NP>(E, B, lr_idx, epoch, j);
    }
  }
}

// ---------------------------------------------------------------------------
// Gated SM engine (CARAMEL_ENGINE_GATED): the two-shot over NVLink done by SM
// kernels, every wait done by the stream front end.  The caller's stream
// waits (cuStreamWaitValue64) until every peer has written its READY tag --
// issued after its gradients, so all inputs are complete before a CTA is
// scheduled -- then this kernel pulls my shard of every bucket from every
// rank, sums in rank order, applies the epilogue and stores the result into
// every replica; a stream write publishes DONE after the kernel and a stream
// wait collects the peers' DONE.  No CTA ever spins on a peer, so the kernel
// holds its SMs only while bytes move (the flag kernels may sit on up to 128
// SMs while a peer is still in its backward pass).  Ownership is the depth-1
// shard split (values are the same rank-order sums whoever owns them).
#define GATED_MAX 32
#ifndef GATED_THREADS
#define GATED_THREADS 512
#endif
#ifndef GATED_U
#define GATED_U 0  // float4s in flight per thread and rank (0: rs_ag_multi's default)
#endif
struct GParams {
  Env env;
  int nb;
  caramel_bucket b[GATED_MAX];
};

static_assert(GATED_THREADS >= 62, "rs_ag_multi: one thread per scalar head/tail element");
template <int NP>
__global__ void __launch_bounds__(GATED_THREADS, 1) k_gated(const __grid_constant__ GParams P) {
  const Env E = P.env;
  if (cta_poisoned(E)) return;
  const int me = E.rank_base, G = gridDim.x;
  constexpr int U = GATED_U ? GATED_U : NP <= 2 ? 4 : 2;  // rs_ag_multi's row: U vectors per thread
  const uint64_t row = 4ull * U * blockDim.x;
  uint64_t rot = 0;  // the first row of bucket i goes to CTA rot mod G: small buckets spread over the grid
  for (int i = 0; i < P.nb; ++i) {
    const caramel_bucket& B = P.b[i];
    uint64_t lo = split_at(B.numel, NP, me), hi = split_at(B.numel, NP, me + 1);
    if (lo >= hi) continue;
    const bool arena = (B.flags & CARAMEL_F_PARAM_ARENA) && B.epilogue == CARAMEL_EPI_SGD;
    const int cj = (int)(((uint64_t)blockIdx.x + G - rot % G) % G);
    Cursor tc;
    cur_init(tc, reinterpret_cast<const caramel_segment*>(B.segs), B.nseg);
    rs_ag_multi<NP, GATED_U>(E, B, arena, tc, &lo, &hi, 1, me, cj, G);
    rot += (hi - lo + row - 1) / row;
  }
}

// ---------------------------------------------------------------------------
// Push protocols OS / TS (see shuffle_proto): every NVLink byte is moved by the
// TMA bulk-copy unit, staged in shared memory -- cp.async.bulk global -> smem
// (local HBM), then smem -> global in a peer's HBM over NVLink 5 / NVSwitch.
// A store is a posted write: the CTA never waits a remote round trip per
// byte, so a few CTAs keep the links busy (tools/mb_nvlink.cu: TMA pushes
// reach 600-690 GB/s per direction with both directions loaded at 16-32 CTAs;
// register pulls need 64+).
//
// Work items.  A launch takes a launch-ordered bucket list (or one bucket).
// Each OS/TS bucket is cut into items (chunk c of its `depth`, tile range r of
// `ranges` -- ranges of about PUSH_RANGE_BYTES, at most the bucket's flag
// slots); items are numbered in launch order over the list and CTA g takes
// items g, g+G, ...  The flags are per item, so any grid size works and ranks
// may group the same launch order differently (CARAMEL_MANY_FLAGS).
//
// Warp roles, running concurrently in every CTA:
//   warp 0 (pusher, one lane)  for each of my items in order:
//       OS: range r of chunk c -> every peer's inbox (one smem tile, p-1 stores)
//       TS: range r of shard (c, s) -> owner s's inbox, for every owner s
//     then, once the item's stores have landed (bulk groups, lagged by one
//     item), READY(c, r) to every peer.  Never waits on a peer.
//   warp 1 (loader, one lane)  for each of my items in order: wait READY(c, r)
//     from every peer; stream the p inputs (own bucket + inbox slots, rank
//     order) and theta through a 3-stage smem ring (mbarrier complete_tx);
//     bulk-store each finished result tile to my output (OS) or to every
//     rank's output (TS: the all-gather), then DONE(c, r) (TS, lagged).
//   warps 2.. (math)  sum each tile in ascending rank order and apply the
//     epilogue in smem (separate fp32 roundings, bit-exact vs the oracle).
// So pushing item k+1 overlaps reducing item k, and the only exposed flag
// hop is the last item's.  Finally (TS) every CTA waits DONE for its items.
// LL buckets ride along only in FUSED lists (identical on every rank): LL
// scatter before the pipeline, LL reduce + finish after it.  OS double-buffers
// its inbox by a per-bucket launch counter in the push-region header (a peer
// may push launch s+1 while I still read launch s); TS needs no second buffer
// (DONE orders reuse).
// ---------------------------------------------------------------------------
#define PUSH_THREADS THREADS     // warp 0 pusher, warp 1 loader, warps 2.. math
#define PUSH_RSTAGES 3           // reduce ring stages
#define PUSH_PSTAGES 3           // push ring stages
#define PUSH_PTILE (24u << 10)   // push ring tile bytes

template <int NP>
struct PushGeo {
  static constexpr int TT = NP <= 2 ? 3072 : NP <= 4 ? 2048 : 1024;  // floats per reduce input tile
  static constexpr int RSF = (NP + 2) * TT;                          // floats per reduce stage: in[NP], theta, out
  static constexpr size_t PUSH_OFF = (size_t)PUSH_RSTAGES * RSF * 4;
  static constexpr size_t BAR_OFF = PUSH_OFF + (size_t)PUSH_PSTAGES * PUSH_PTILE;
  static constexpr size_t SMEM = BAR_OFF + (2 * PUSH_RSTAGES + PUSH_PSTAGES) * 8 + 16;
};

struct PushParams {
  Env env;
  const caramel_bucket* bs;  // device list, or nullptr: the single bucket `one`
  int nb;
  int with_ll;               // FUSED lists: LL buckets handled in this launch
  caramel_bucket one;
};

__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// at most n bulk groups of this thread still pending (n clamped to 0..7)
__device__ __forceinline__ void bulk_wait_upto(uint32_t n) {
  switch (n > 7 ? 7 : n) {
    case 0: asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.bulk.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.bulk.wait_group 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.bulk.wait_group 3;" ::: "memory"); break;
    case 4: asm volatile("cp.async.bulk.wait_group 4;" ::: "memory"); break;
    case 5: asm volatile("cp.async.bulk.wait_group 5;" ::: "memory"); break;
    case 6: asm volatile("cp.async.bulk.wait_group 6;" ::: "memory"); break;
    default: asm volatile("cp.async.bulk.wait_group 7;" ::: "memory"); break;
  }
}

__device__ __forceinline__ uint64_t push_region(const Env& E, const caramel_bucket& B, int rank) {
  return E.arena[rank] + B.bucket_off + push_off(B.numel, CARAMEL_SHUFFLE, E.world);
}
__device__ __forceinline__ float* push_inbox(const Env& E, const caramel_bucket& B, int rank, int buf, int src) {
  const int p = E.world, slot = src < rank ? src : src - 1;
  return reinterpret_cast<float*>(push_region(E, B, rank) + 256 + push_flag_bytes(B.numel, B.depth, p) +
                                  ((uint64_t)buf * (p - 1) + slot) * push_slot_bytes(B.numel));
}
__device__ __forceinline__ float* push_out(const Env& E, const caramel_bucket& B, int rank) {
  return B.epilogue == CARAMEL_EPI_SGD ? reinterpret_cast<float*>(E.parena[rank] + B.param_off)
                                       : reinterpret_cast<float*>(E.arena[rank] + B.bucket_off);
}
__device__ __forceinline__ uint32_t* push_flag(const Env& E, const caramel_bucket& B, int rank, int c, int r,
                                               int slot, int src) {
  return reinterpret_cast<uint32_t*>(push_region(E, B, rank) + 256) +
         ((((uint64_t)c * push_ranges(B.numel, B.depth) + r) * 2 + slot) * E.world + src);
}

// element range of item (c, r): OS -> range r of chunk c; TS -> range r of shard (c, s)
__device__ __forceinline__ void item_range(const caramel_bucket& B, int proto, int p, int c, int s, int r, int R,
                                           uint64_t& lo, uint64_t& hi) {
  const uint64_t c0 = split_at(B.numel, B.depth, c), c1 = split_at(B.numel, B.depth, c + 1);
  uint64_t a = c0, b = c1;
  if (proto == PROTO_TS) {
    const uint64_t m = c1 - c0;
    a = c0 + split_at(m, p, s);
    b = c0 + split_at(m, p, s + 1);
  }
  tile_of(a, b, R, r, lo, hi);
}

// Iterates this CTA's items of the list in launch order: f(i, B, proto, c, r, R, buf).
template <class F>
__device__ __forceinline__ void for_my_items(const PushParams& P, int me, F f) {
  const int G = gridDim.x, g = blockIdx.x, p = P.env.world;
  const int nb = P.bs ? P.nb : 1;
  uint64_t k = 0;  // global item number
  for (int i = 0; i < nb; ++i) {
    const caramel_bucket B = P.bs ? P.bs[i] : P.one;
    const int proto = shuffle_proto(B, p);
    if ((proto != PROTO_OS && proto != PROTO_TS) || B.numel == 0) continue;
    const int R = push_ranges(B.numel, B.depth);
    const uint64_t n = (uint64_t)B.depth * R;
    // first item of this bucket that is mine
    uint64_t first = (g >= (int)(k % G)) ? k + (g - (k % G)) : k + (G - (k % G)) + g;
    if (first < k + n) {
      const int buf = proto == PROTO_OS
                          ? (int)(*reinterpret_cast<volatile uint32_t*>(push_region(P.env, B, me)) & 1u) : 0;
      for (uint64_t t = first - k; t < n; t += G) f(i, B, proto, (int)(t / R), (int)(t % R), R, buf);
    }
    k += n;
  }
}

// ---- pusher (warp 0, lane 0) ----------------------------------------------------
struct PushRing {
  unsigned char* buf;  // PUSH_PSTAGES x PUSH_PTILE bytes
  uint64_t* bar;
  uint32_t u;          // tiles issued so far
};

// Copy the 16-byte aligned body of [lo, hi) of src to nd destinations through
// the push ring (plain ld/st for the <= 3 + 3 ragged elements).  Returns the
// number of bulk groups committed (one per tile).
__device__ uint32_t push_copy(PushRing& S, const float* src, float* const* dst, int nd, uint64_t lo, uint64_t hi) {
  if (lo >= hi) return 0;
  uint64_t a, b;
  split4(lo, hi, a, b);
  for (uint64_t x = lo; x < a; ++x)
    for (int d = 0; d < nd; ++d) st1(dst[d] + x, ld1(src + x));
  for (uint64_t x = b > a ? b : a; x < hi; ++x)
    for (int d = 0; d < nd; ++d) st1(dst[d] + x, ld1(src + x));
  constexpr uint64_t TF = PUSH_PTILE / 4;
  const uint64_t nt = b > a ? (b - a + TF - 1) / TF : 0;
  auto bytes_of = [&](uint64_t t) {
    const uint64_t x = a + t * TF;
    return (uint32_t)(4 * ((b - x) < TF ? (b - x) : TF));
  };
  auto issue = [&](uint64_t t) {
    const uint32_t u = S.u + (uint32_t)t, s = u % PUSH_PSTAGES;
    mbar_expect_tx(&S.bar[s], bytes_of(t));
    bulk_load(S.buf + (size_t)s * PUSH_PTILE, src + a + t * TF, bytes_of(t), &S.bar[s]);
  };
  // the stage refilled for tile t+S-1 held tile t-1: its stores must be done reading
  for (uint64_t t = 0; t < nt && t + 1 < PUSH_PSTAGES; ++t) issue(t);
  for (uint64_t t = 0; t < nt; ++t) {
    const uint32_t u = S.u + (uint32_t)t, s = u % PUSH_PSTAGES;
    mbar_wait(&S.bar[s], (u / PUSH_PSTAGES) & 1);
    for (int d = 0; d < nd; ++d) bulk_store(dst[d] + a + t * TF, S.buf + (size_t)s * PUSH_PTILE, bytes_of(t));
    bulk_commit();
    if (t + PUSH_PSTAGES - 1 < nt) {
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      issue(t + PUSH_PSTAGES - 1);
    }
  }
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // the ring restarts at the next call
  S.u += (uint32_t)nt;
  return (uint32_t)nt;
}

struct Pending {  // an item whose stores are in flight, to flag once they landed
  uint64_t flag_off;  // its bucket's push flags (byte offset in every rank's arena)
  int ranges;         // ranges per chunk
  int c, r, slot, valid;
};

__device__ __forceinline__ void flag_peers(const Env& E, const Pending& it, int me, uint32_t epoch) {
  for (int q = 0; q < E.world; ++q)
    if (q != me)
      st_relaxed_sys(reinterpret_cast<uint32_t*>(E.arena[q] + it.flag_off) +
                         ((((uint64_t)it.c * it.ranges + it.r) * 2 + it.slot) * E.world + me),
                     epoch);
}

// publish `pend` once at most `keep` bulk groups (committed after it) are pending
__device__ __forceinline__ void publish_pending(const Env& E, Pending& pend, int me, uint32_t epoch, uint32_t keep) {
  if (!pend.valid) return;
  bulk_wait_upto(keep);
  fence_proxy_async_global();
  fence_acq_rel_sys();
  flag_peers(E, pend, me, epoch);
  pend.valid = 0;
}

__device__ void pusher(const PushParams& P, PushRing& S, int me, uint32_t epoch) {
  const Env& E = P.env;
  const int p = E.world;
  Pending pend{0, 0, 0, 0, SLOT_READY, 0};
  for_my_items(P, me, [&](int, const caramel_bucket& B, int proto, int c, int r, int R, int buf) {
    const float* mine = reinterpret_cast<const float*>(E.arena[me] + B.bucket_off);
    uint32_t groups = 0;
    if (proto == PROTO_OS) {
      uint64_t lo, hi;
      item_range(B, proto, p, c, 0, r, R, lo, hi);
      float* dst[MAXR];
      int nd = 0;
      for (int t = 1; t < p; ++t) dst[nd++] = push_inbox(E, B, (me + t) % p, buf, me);
      groups += push_copy(S, mine, dst, nd, lo, hi);
    } else {
      for (int t = 1; t < p; ++t) {  // owners in rotated order: every link starts busy
        const int s = (me + t) % p;
        uint64_t lo, hi;
        item_range(B, proto, p, c, s, r, R, lo, hi);
        float* dst[1] = {push_inbox(E, B, s, 0, me)};
        groups += push_copy(S, mine, dst, 1, lo, hi);
      }
    }
    publish_pending(E, pend, me, epoch, groups);  // the previous item has landed once <= `groups` remain
    pend = Pending{B.bucket_off + push_off(B.numel, CARAMEL_SHUFFLE, p) + 256, R, c, r, SLOT_READY, 1};
  });
  publish_pending(E, pend, me, epoch, 0);
}

// ---- loader (warp 1, lane 0) and math warps (2..) -----------------------------------
struct ReduceRing {
  float* st;       // PUSH_RSTAGES stages of RSF floats
  uint64_t* full;  // loads landed (count 1 + tx)
  uint64_t* comp;  // math warps finished the tile (count = math warps)
};

template <int NP>
__device__ __forceinline__ uint32_t tiles_of(uint64_t a, uint64_t b) {
  return b > a ? (uint32_t)((b - a + PushGeo<NP>::TT - 1) / PushGeo<NP>::TT) : 0;
}

template <int NP>
__device__ void loader(const PushParams& P, ReduceRing& S, int me, uint32_t epoch, int* abort_flag) {
  constexpr int TT = PushGeo<NP>::TT, SF = PushGeo<NP>::RSF;
  const Env& E = P.env;
  const int p = E.world;
  uint32_t u = 0;  // ring position (tiles loaded so far)
  uint32_t issued_items = 0;
  Pending pend{0, 0, 0, 0, SLOT_DONE, 0};
  bool ok = true;
  for_my_items(P, me, [&](int, const caramel_bucket& B, int proto, int c, int r, int R, int buf) {
    if (!ok) return;
    // the item's inputs: READY from every peer
    for (int q = 0; q < p && ok; ++q) {
      if (q == me) continue;
      const uint32_t* f = push_flag(E, B, me, c, r, SLOT_READY, q);
      if (ld_acquire_sys(f) >= epoch) continue;
      const uint64_t t0 = globaltimer();
      uint32_t spins = 0;
      while (ld_acquire_sys(f) < epoch) {
        if ((++spins & 1023u) == 0) {
          if (poisoned(E)) { ok = false; break; }
          if (globaltimer() - t0 > E.timeout_ns) { raise_timeout(E); ok = false; break; }
        }
      }
    }
    if (!ok) return;
    fence_proxy_async_global();  // the TMA loads below must see what the flags published
    const bool sgd = B.epilogue == CARAMEL_EPI_SGD;
    const float* in[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q)
      in[q] = q == me ? reinterpret_cast<const float*>(E.arena[me] + B.bucket_off) : push_inbox(E, B, me, buf, q);
    const float* th = reinterpret_cast<const float*>(E.parena[me] + B.param_off);
    float* out[MAXR];
    int nd = 0;
    if (proto == PROTO_TS)
      for (int t = 0; t < p; ++t) out[nd++] = push_out(E, B, (me + t) % p);  // local first
    else
      out[nd++] = push_out(E, B, me);
    uint64_t lo, hi, a, b;
    item_range(B, proto, p, c, me, r, R, lo, hi);
    split4(lo, hi, a, b);
    auto edge = [&](uint64_t x) {  // <= 3 + 3 ragged elements: plain loads / stores
      float acc = ld1(in[0] + x);
      for (int q = 1; q < p; ++q) acc = __fadd_rn(acc, ld1(in[q] + x));
      const float o = epi1(B.epilogue, acc, sgd ? ld1(th + x) : 0.f, B.scale, B.lr);
      for (int d = 0; d < nd; ++d) st1(out[d] + x, o);
    };
    for (uint64_t x = lo; x < a; ++x) edge(x);
    for (uint64_t x = b > a ? b : a; x < hi; ++x) edge(x);
    const uint32_t nt = tiles_of<NP>(a, b);
    auto bytes_of = [&](uint32_t t) {
      const uint64_t x = a + (uint64_t)t * TT;
      return (uint32_t)(4 * ((b - x) < (uint64_t)TT ? (b - x) : (uint64_t)TT));
    };
    auto issue = [&](uint32_t t) {
      const uint32_t uu = u + t, s = uu % PUSH_RSTAGES, bytes = bytes_of(t);
      float* st = S.st + (size_t)s * SF;
      mbar_expect_tx(&S.full[s], bytes * (p + (sgd ? 1 : 0)));
      const uint64_t x = a + (uint64_t)t * TT;
      for (int q = 0; q < p; ++q) bulk_load(st + q * TT, in[q] + x, bytes, &S.full[s]);
      if (sgd) bulk_load(st + NP * TT, th + x, bytes, &S.full[s]);
    };
    // prefetch distance STAGES-1; the stage refilled for tile t+S-1 held tile
    // t-1: the math warps are done with it (its comp barrier was waited) and
    // its stores must be done reading (wait_group.read 0 after tile t's commit
    // would serialise, so read-wait with one group of slack)
    for (uint32_t t = 0; t < nt && t + 1 < PUSH_RSTAGES; ++t) issue(t);
    for (uint32_t t = 0; t < nt; ++t) {
      const uint32_t uu = u + t, s = uu % PUSH_RSTAGES;
      mbar_wait(&S.comp[s], (uu / PUSH_RSTAGES) & 1);
      const float* res = S.st + (size_t)s * SF + (NP + 1) * TT;
      const uint64_t x = a + (uint64_t)t * TT;
      for (int d = 0; d < nd; ++d) bulk_store(out[d] + x, res, bytes_of(t));
      bulk_commit();
      if (t + PUSH_RSTAGES - 1 < nt) {
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        issue(t + PUSH_RSTAGES - 1);
      }
    }
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    u += nt;
    ++issued_items;
    publish_pending(E, pend, me, epoch, nt);  // the previous TS item's all-gather has landed
    if (proto == PROTO_TS) pend = Pending{B.bucket_off + push_off(B.numel, CARAMEL_SHUFFLE, p) + 256, R, c, r, SLOT_DONE, 1};
  });
  if (!ok) {  // wake the math warps and stop them
    *reinterpret_cast<volatile int*>(abort_flag) = 1;
    for (int s = 0; s < PUSH_RSTAGES; ++s) mbar_arrive(&S.full[s]);
    return;
  }
  publish_pending(E, pend, me, epoch, 0);
  bulk_wait_upto(0);
}

template <int NP>
__device__ void math_warps(const PushParams& P, ReduceRing& S, int me, const int* abort_flag) {
  constexpr int TT = PushGeo<NP>::TT, SF = PushGeo<NP>::RSF;
  const int p = P.env.world;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nmath = (blockDim.x >> 5) - 2, mw = warp - 2;
  uint32_t u = 0;
  bool stop = false;
  for_my_items(P, me, [&](int, const caramel_bucket& B, int proto, int c, int r, int R, int) {
    if (stop) return;
    uint64_t lo, hi, a, b;
    item_range(B, proto, p, c, me, r, R, lo, hi);
    split4(lo, hi, a, b);
    const uint32_t nt = tiles_of<NP>(a, b);
    const bool sgd = B.epilogue == CARAMEL_EPI_SGD;
    for (uint32_t t = 0; t < nt; ++t) {
      const uint32_t uu = u + t, s = uu % PUSH_RSTAGES;
      mbar_wait(&S.full[s], (uu / PUSH_RSTAGES) & 1);
      if (*reinterpret_cast<const volatile int*>(abort_flag)) { stop = true; return; }
      float* st = S.st + (size_t)s * SF;
      const float4* i4 = reinterpret_cast<const float4*>(st);
      const float4* t4 = reinterpret_cast<const float4*>(st + NP * TT);
      float4* o4 = reinterpret_cast<float4*>(st + (NP + 1) * TT);
      const uint64_t x = a + (uint64_t)t * TT;
      const uint32_t n4 = (uint32_t)(((b - x) < (uint64_t)TT ? (b - x) : (uint64_t)TT) / 4);
      for (uint32_t v = mw * 32 + lane; v < n4; v += nmath * 32) {
        float4 acc = i4[v];
#pragma unroll
        for (int q = 1; q < NP; ++q) acc = add4(acc, i4[q * (TT / 4) + v]);
        o4[v] = epi4(B.epilogue, acc, sgd ? t4[v] : acc, B.scale, B.lr);
      }
      fence_proxy_async();  // my smem writes -> the async proxy (the bulk store)
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.comp[s]);
    }
    u += nt;
  });
}

template <int NP>
__global__ void __launch_bounds__(PUSH_THREADS, 1) k_push(const __grid_constant__ PushParams P) {
  extern __shared__ __align__(128) unsigned char dyn_smem[];
  __shared__ int s_abort;
  const Env E = P.env;
  if (cta_poisoned(E)) return;
  const int lr_idx = blockIdx.y;
  const int me = E.rank_base + lr_idx, p = E.world;
  const uint32_t epoch = launch_epoch(E);
  const int nb = P.bs ? P.nb : 1;
  ReduceRing RR;
  RR.st = reinterpret_cast<float*>(dyn_smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(dyn_smem + PushGeo<NP>::BAR_OFF);
  RR.full = bars;
  RR.comp = bars + PUSH_RSTAGES;
  PushRing PR;
  PR.buf = dyn_smem + PushGeo<NP>::PUSH_OFF;
  PR.bar = bars + 2 * PUSH_RSTAGES;
  PR.u = 0;
  const int nmath = (blockDim.x >> 5) - 2;
  if (threadIdx.x == 0) {
    s_abort = 0;
    for (int s = 0; s < PUSH_RSTAGES; ++s) {
      mbar_init(&RR.full[s], 1);
      mbar_init(&RR.comp[s], nmath);
    }
    for (int s = 0; s < PUSH_PSTAGES; ++s) mbar_init(&PR.bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // (PACK buckets were gathered into the bucket by k_pack launches before this kernel)
  auto ll_pass = [&](int phase) {
    if (!P.with_ll) return;
    const int G = gridDim.x;
    int base = 0;
    for (int i = 0; i < nb; ++i) {
      const caramel_bucket B = P.bs ? P.bs[i] : P.one;
      if (shuffle_proto(B, p) != PROTO_LL) continue;
      int jj = ((int)blockIdx.x - base) % G;
      if (jj < 0) jj += G;
      base = (base + B.ctas) % G;
      if (jj >= B.ctas || B.numel == 0) continue;
      BucketRun R;
      make_run(R, E, B, CARAMEL_SHUFFLE, lr_idx, epoch, jj);
      if (phase == 0) phase_ll_scatter(R);
      else if (phase == 1) phase_ll_reduce<NP>(R);
      else phase_ll_finish(R);
    }
  };
  ll_pass(0);
  // ---- the push / reduce pipeline ------------------------------------------------
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    if (threadIdx.x == 0) pusher(P, PR, me, epoch);
  } else if (warp == 1) {
    if (threadIdx.x == 32) loader<NP>(P, RR, me, epoch, &s_abort);
  } else {
    math_warps<NP>(P, RR, me, &s_abort);
  }
  __syncthreads();
  if (*reinterpret_cast<volatile int*>(&s_abort)) return;  // a flag wait failed: nothing more is stored
  ll_pass(1);
  ll_pass(2);
  // ---- TS: every owner's all-gather of my items has landed --------------------------
  int bad = 0;
  for_my_items(P, me, [&](int, const caramel_bucket& B, int proto, int c, int r, int, int) {
    if (proto != PROTO_TS || bad) return;
    const int q = threadIdx.x;
    if (q < p && q != me) {
      const uint32_t* f = push_flag(E, B, me, c, r, SLOT_DONE, q);
      if (ld_acquire_sys(f) < epoch) {
        const uint64_t t0 = globaltimer();
        uint32_t spins = 0;
        while (ld_acquire_sys(f) < epoch) {
          if ((++spins & 1023u) == 0) {
            if (poisoned(E)) { bad = 1; break; }
            if (globaltimer() - t0 > E.timeout_ns) { raise_timeout(E); bad = 1; break; }
          }
        }
      }
    }
  });
  cta_abort_if(bad);
  // ---- OS: the last CTA of a bucket flips its inbox buffer -------------------------
  if (threadIdx.x == 0) {
    const int G = gridDim.x;
    uint64_t k = 0;
    for (int i = 0; i < nb; ++i) {
      const caramel_bucket B = P.bs ? P.bs[i] : P.one;
      const int proto = shuffle_proto(B, p);
      if ((proto != PROTO_OS && proto != PROTO_TS) || B.numel == 0) continue;
      const uint64_t n = (uint64_t)B.depth * push_ranges(B.numel, B.depth);
      const uint64_t off = (blockIdx.x + G - k % G) % G;  // my first item index within the bucket
      if (proto == PROTO_OS && off < n) {
        const uint32_t parts = (uint32_t)(n < (uint64_t)G ? n : (uint64_t)G);
        uint32_t* h = reinterpret_cast<uint32_t*>(push_region(E, B, me));
        const uint32_t old = atomicAdd(h + 1, 1u);
        if (old == parts - 1) {
          atomicExch(h + 1, 0u);
          atomicAdd(h, 1u);
        }
      }
      k += n;
    }
  }
}

// ---------------------------------------------------------------------------
// NVLS (NVLink SHARP) two-shot: the non-fixed-order mode (caramel_allreduce_nvls).
// The buckets live in a multicast-bound arena (every rank's physical copy is
// reachable through one multicast address).  Rank r owns shard r of every
// chunk: one multimem.ld_reduce per 16 bytes makes the NVSwitch fetch that
// vector from every GPU and return the fp32 SUM (in the switch's order, not
// the rank order: results agree to the 1e-6 relative bound of SURVEY §8c, not
// bit for bit), the epilogue is applied, and one multimem.st writes the result
// into every GPU's copy.  Per GPU and direction that is S bytes instead of the
// 2(p-1)/p x S of a two-shot over peer loads/stores.  READY/DONE are the
// bucket's ordinary per-(chunk, tile) flags in the IPC arena.  The SGD
// epilogue: the owner broadcasts (sum x scale), every rank then updates its
// own parameters from that identical vector (replicas stay bit-identical).
// ---------------------------------------------------------------------------
struct NvlsParams {
  Env env;
  caramel_bucket b;
  uint64_t mc;   // multicast address of the NVLS arena
  uint64_t uc;   // this rank's unicast view of it
  int probe;     // diagnostics only (CARAMEL_NVLS_PROBE): 1 = in-switch reduce, unicast store; 2 = unicast load, multicast store
};

__device__ __forceinline__ float4 mc_ld_reduce4(const float* a) {
  float4 r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(a)
               : "memory");
  return r;
}
__device__ __forceinline__ float mc_ld_reduce1(const float* a) {
  float r;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(r) : "l"(a) : "memory");
  return r;
}
__device__ __forceinline__ void mc_st4(float* a, float4 v) {
  asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(a), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
__device__ __forceinline__ void mc_st1(float* a, float v) {
  asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_alias() { asm volatile("fence.proxy.alias;" ::: "memory"); }

__global__ void __launch_bounds__(THREADS, 1) k_nvls(const __grid_constant__ NvlsParams P) {
  const Env E = P.env;
  if (cta_poisoned(E)) return;
  const caramel_bucket B = P.b;
  const int me = E.rank_base, p = E.world, j = blockIdx.x, G = B.ctas;
  const uint32_t epoch = launch_epoch(E);
  Ctx X;
  X.E = &E;
  X.flag_off = B.flag_off;
  X.me = me;
  X.world = p;
  X.j = j;
  X.G = G;
  X.ns = 2;
  X.epoch = epoch;
  float* mcb = reinterpret_cast<float*>(P.mc + B.bucket_off);
  float* ucb = reinterpret_cast<float*>(P.uc + B.bucket_off);
  const bool sgd = B.epilogue == CARAMEL_EPI_SGD;
  const int epi = sgd ? CARAMEL_EPI_SCALE : B.epilogue;  // SGD: broadcast sum*scale, update locally below
  // my contribution (written before this launch, through the unicast view) is in place
  fence_proxy_alias();
  for (int c = 0; c < B.depth; ++c) X.publish_all(c, SLOT_READY);
  for (int c = 0; c < B.depth; ++c) {
    X.wait_all(c, SLOT_READY, epoch);
    uint64_t lo, hi, a, b;
    shard_bounds(B.numel, B.depth, p, c, me, lo, hi);
    tile_of(lo, hi, G, j, lo, hi);
    split4(lo, hi, a, b);
    for (uint64_t x = lo + threadIdx.x; x < a; x += blockDim.x) mc_st1(mcb + x, epi1(epi, mc_ld_reduce1(mcb + x), 0.f, B.scale, B.lr));
    for (uint64_t x = (b > a ? b : a) + threadIdx.x; x < hi; x += blockDim.x)
      mc_st1(mcb + x, epi1(epi, mc_ld_reduce1(mcb + x), 0.f, B.scale, B.lr));
    constexpr int U = 8;  // switch round trips in flight per thread
    const uint64_t T = 4ull * blockDim.x;
    uint64_t v = a + 4ull * threadIdx.x;
    if (P.probe == 1) {  // diagnostics: the switch's reduce alone
      for (; v + (U - 1) * T < b; v += U * T) {
        float4 s[U];
#pragma unroll
        for (int u = 0; u < U; ++u) s[u] = mc_ld_reduce4(mcb + v + u * T);
#pragma unroll
        for (int u = 0; u < U; ++u) st4(ucb + v + u * T, s[u]);
      }
    } else if (P.probe == 2) {  // diagnostics: the switch's broadcast alone
      for (; v + (U - 1) * T < b; v += U * T) {
        float4 s[U];
#pragma unroll
        for (int u = 0; u < U; ++u) s[u] = ld4(ucb + v + u * T);
#pragma unroll
        for (int u = 0; u < U; ++u) mc_st4(mcb + v + u * T, s[u]);
      }
    }
    for (; v + (U - 1) * T < b; v += U * T) {
      float4 s[U];
#pragma unroll
      for (int u = 0; u < U; ++u) s[u] = mc_ld_reduce4(mcb + v + u * T);
#pragma unroll
      for (int u = 0; u < U; ++u) mc_st4(mcb + v + u * T, epi4(epi, s[u], s[u], B.scale, B.lr));
    }
    for (; v < b; v += T) mc_st4(mcb + v, epi4(epi, mc_ld_reduce4(mcb + v), make_float4(0.f, 0.f, 0.f, 0.f), B.scale, B.lr));
    __syncthreads();
    if (threadIdx.x < 32) fence_acq_rel_sys();  // my multimem stores, then DONE
    X.publish_all(c, SLOT_DONE);
  }
  for (int c = 0; c < B.depth; ++c) X.wait_all(c, SLOT_DONE, epoch);
  fence_proxy_alias();  // the results arrived through the multicast address; read them through the unicast one
  if (!sgd) return;
  float* th = reinterpret_cast<float*>(E.parena[me] + B.param_off);
  for (int c = 0; c < B.depth; ++c)
    for (int s = 0; s < p; ++s) {
      uint64_t lo, hi;
      shard_bounds(B.numel, B.depth, p, c, s, lo, hi);
      tile_of(lo, hi, G, j, lo, hi);
      // theta <- theta - lr * g, g = the broadcast (sum * scale): epi1(SGD) with scale 1
      for (uint64_t x = lo + threadIdx.x; x < hi; x += blockDim.x)
        st1(th + x, __fsub_rn(ld1(th + x), __fmul_rn(B.lr, ld1(ucb + x))));
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

// ---------------------------------------------------------------------------
// Copy-engine two-shot (caramel_allreduce_ce).  The NVLink bytes move on the
// copy engines; this kernel is the only SM work: for every bucket of the call,
// my shard = own gradients (bucket arena) + the world-1 peer contributions the
// copy engines staged (slots congruent to the bucket arena), summed in
// ascending rank order, epilogue, stored to the output (parameter arena for
// SGD, my bucket arena otherwise) -- where the peers' copy engines fetch it.
// Short-lived CTAs of CE_TILE elements each: no CTA outlives its tile, so the
// backward kernels running beside it get SMs back within microseconds.
// ---------------------------------------------------------------------------
#define CE_MAX_BUCKETS 32
#define CE_THREADS 256
#define CE_TILE 8192
#define CE_FLAG_OFF 4096  // byte offset of the READY / DONE words in the sync region

struct CeItem {
  uint64_t src;    // byte offset of my shard's first element in my bucket arena
  uint64_t stg;    // byte offset of its staged copy in slot 0 (slot k at + k * slot)
  uint64_t slot;   // staging slot bytes
  uint64_t dst;    // byte offset of my shard in the output arena
  uint64_t n;      // shard elements
  uint32_t cta0;   // first CTA of this bucket
  float lr, scale;
};

#define CE_POOL 256  // gradient-ready events of submitted, not yet issued calls

struct CeJob {
  std::vector<caramel_bucket> buckets;
  int engine;  // CARAMEL_ENGINE_CE / CARAMEL_ENGINE_SM
  uint32_t index0, epoch;
  cudaEvent_t grads, done;
  cudaStream_t stream;
};

struct CeParams {
  const char* arena;  // my bucket arena (own gradients + staging slots)
  char* out;
  int world, me, count, epi;
  CeItem it[CE_MAX_BUCKETS];
};

// Input q of element i (shard-relative byte offset o = 4i): my own gradients,
// or the slot rank q's copy engine pushed into (slot k = q < me ? q : q - 1).
__device__ __forceinline__ const char* ce_in(const CeParams& P, const CeItem& I, int q) {
  return q == P.me ? P.arena + I.src : P.arena + I.stg + (uint64_t)(q < P.me ? q : q - 1) * I.slot;
}

__global__ void __launch_bounds__(CE_THREADS) k_ce_reduce(const __grid_constant__ CeParams P) {
  int b = 0;
  while (b + 1 < P.count && blockIdx.x >= P.it[b + 1].cta0) ++b;
  const CeItem I = P.it[b];
  const uint64_t t0 = (uint64_t)(blockIdx.x - I.cta0) * CE_TILE;
  const uint64_t t1 = t0 + CE_TILE < I.n ? t0 + CE_TILE : I.n;
  // elements i with (src/4 + i) % 4 == 0 start a 16-byte vector in every input
  const uint64_t head = (4 - ((I.src >> 2) & 3)) & 3;
  const uint64_t va = t0 + head < t1 ? t0 + head : t1;
  const uint64_t vb = va + (t1 - va) / 4 * 4;
  const int world = P.world, epi = P.epi;
  for (uint64_t i = va + 4 * (uint64_t)threadIdx.x; i < vb; i += 4 * CE_THREADS) {
    float4 acc = ld4(reinterpret_cast<const float*>(ce_in(P, I, 0) + 4 * i));
    for (int q = 1; q < world; ++q) acc = add4(acc, ld4(reinterpret_cast<const float*>(ce_in(P, I, q) + 4 * i)));
    float4* o = reinterpret_cast<float4*>(P.out + I.dst + 4 * i);
    const float4 th = epi == CARAMEL_EPI_SGD ? *o : acc;
    *o = epi4(epi, acc, th, I.scale, I.lr);
  }
  // scalar head [t0, va) and tail [vb, t1)
  const uint64_t nh = va - t0, nt = t1 - vb;
  if (threadIdx.x < nh + nt) {
    const uint64_t i = threadIdx.x < nh ? t0 + threadIdx.x : vb + (threadIdx.x - nh);
    float acc = *reinterpret_cast<const float*>(ce_in(P, I, 0) + 4 * i);
    for (int q = 1; q < world; ++q) acc = __fadd_rn(acc, *reinterpret_cast<const float*>(ce_in(P, I, q) + 4 * i));
    float* o = reinterpret_cast<float*>(P.out + I.dst + 4 * i);
    *o = epi1(epi, acc, epi == CARAMEL_EPI_SGD ? *o : acc, I.scale, I.lr);
  }
}

struct caramel_ctx {
  int rank, world, nlocal, device, sms;
  uint64_t arena_bytes, param_bytes;
  void* arena_local[MAXR];
  void* param_local[MAXR];
  uint64_t arena[MAXR];
  uint64_t parena[MAXR];
  bool imported;
  bool opened[MAXR];
  int* status;
  int* hstatus;      // host-mapped mirror of *status (pinned host memory)
  int* hstatus_dev;  // its device address
  uint32_t* epoch_dev;
  uint64_t timeout_ns;
  // copy-engine two-shot (caramel_allreduce_ce), created on first use
  int gated_ctas;  // grid cap of a k_gated launch (CARAMEL_GATED_CTAS, default 32)
  bool ce_ready;
  cudaStream_t ce_send;  // reduce-scatter pushes + READY: never waits on a peer
  cudaEvent_t ce_grads;  // gradients produced (recorded on the caller's grad stream)
  // asynchronous submission (caramel_ce_submit / caramel_ce_flush)
  std::mutex ce_mu;
  std::condition_variable ce_cv;
  std::deque<CeJob> ce_jobs;
  std::thread ce_worker;
  bool ce_worker_started, ce_stop, ce_busy;
  uint64_t ce_submitted, ce_consumed;
  cudaEvent_t ce_pool[CE_POOL];
  int ce_rc;
  char ce_err[512];
  // NVLS multicast arena (caramel_mc_*)
  int mc_state;                 // 0 none, 1 created, 2 exchanged, 3 bound
  uint64_t mc_bytes, mc_gran;
  unsigned long long mc_handle;  // CUmemGenericAllocationHandle of the multicast object
  unsigned long long mc_mem;     // this rank's physical allocation
  uint64_t mc_va, uc_va;         // multicast and unicast mappings
  int mc_listen, mc_fd;          // rank 0: listening socket; every rank: the multicast handle's fd
  char mc_name[108];
};

struct Blob {
  uint32_t magic, rank, world, has_param;
  uint64_t arena_bytes, param_bytes;
  cudaIpcMemHandle_t arena, param;
};

extern "C" {

static void load_ll_max() {
  static bool done = false;
  if (done) return;
  done = true;
  if (const char* e = getenv("CARAMEL_LL_MAX")) h_ll_max = strtoull(e, 0, 10);
  if (const char* e = getenv("CARAMEL_OS_MAX")) h_os_max = strtoull(e, 0, 10);
  if (const char* e = getenv("CARAMEL_PUSH")) h_push_enabled = atoi(e) != 0;
  if (const char* e = getenv("CARAMEL_LL128_MAX")) h_ll128_max = strtoull(e, 0, 10);
  cudaMemcpyToSymbol(d_ll128_max, &h_ll128_max, sizeof(h_ll128_max));
  cudaMemcpyToSymbol(d_ll_max, &h_ll_max, sizeof(h_ll_max));
  cudaMemcpyToSymbol(d_os_max, &h_os_max, sizeof(h_os_max));
  cudaMemcpyToSymbol(d_push_enabled, &h_push_enabled, sizeof(h_push_enabled));
}

int caramel_abi_version(void) { return CARAMEL_ABI_VERSION; }
const char* caramel_last_error(void) { return g_err; }

int caramel_chunk_bounds(uint64_t numel, int depth, int workers, uint64_t* out) {
  if (depth < 1 || depth > CARAMEL_MAX_DEPTH)
    return set_err(CARAMEL_EINVAL, "depth must be in [1, %d]", CARAMEL_MAX_DEPTH);
  if (workers < 1 || workers > 64) return set_err(CARAMEL_EINVAL, "bad worker count %d", workers);
  if (!out) return set_err(CARAMEL_EINVAL, "null output");
  for (int c = 0; c < depth; ++c) {
    uint64_t c0 = (numel * (uint64_t)c) / depth, c1 = (numel * (uint64_t)(c + 1)) / depth;
    uint64_t m = c1 - c0;
    for (int s = 0; s < workers; ++s) out[(uint64_t)c * (workers + 1) + s] = c0 + (m * s) / workers;
    out[(uint64_t)c * (workers + 1) + workers] = c1;
  }
  return 0;
}

static int validate_workers(int pattern, int world) {
  if (world < 1 || world > MAXR)
    return set_err(CARAMEL_EWORKERS, "world size %d outside [1, %d]", world, MAXR);
  if (pattern == CARAMEL_HD && (world & (world - 1)))
    return set_err(CARAMEL_EWORKERS, "halving-doubling requires a power-of-two worker count");
  if (pattern < 0 || pattern > 2) return set_err(CARAMEL_EINVAL, "unknown pattern %d", pattern);
  return 0;
}

// CTAs of a large two-shot bucket: its pull loop is latency-bound (a 1 GiB
// bucket at p = 2: 64 CTAs 1758 us, 128 CTAs 1629 us, on the same box)
static int default_max_ctas() {
  const char* e = getenv("CARAMEL_MAX_CTAS");
  if (e && atoi(e) > 0) return atoi(e);
  return 128;
}

// Bucket region: the kernels' part (packed bucket; LL region; ring/hd halves),
// then -- SHUFFLE, world > 1 -- world-1 staging slots where peers' copy
// engines push their contributions to my shard (caramel_allreduce_ce).  A
// slot holds ceil(n/p) elements after a (lo & 3)-element pad, so staged data
// keeps the 16-byte phase of the shard it belongs to.
static uint64_t ce_slot_bytes(uint64_t numel, int world) {
  const uint64_t m = (numel + world - 1) / world;
  return (4 * (m + 3) + 15) & ~15ull;
}
static uint64_t ce_stage_off(uint64_t numel, int depth, int pattern, int world) {
  return push_off(numel, pattern, world) + push_region_bytes(numel, depth, pattern, world);
}

int caramel_bucket_layout(uint64_t numel, int depth, int pattern, int world, int32_t* ctas,
                          uint64_t* bucket_bytes, uint64_t* flag_bytes) {
  if (getenv("CARAMEL_LL_MAX")) h_ll_max = strtoull(getenv("CARAMEL_LL_MAX"), 0, 10);
  if (getenv("CARAMEL_OS_MAX")) h_os_max = strtoull(getenv("CARAMEL_OS_MAX"), 0, 10);
  if (getenv("CARAMEL_PUSH")) h_push_enabled = atoi(getenv("CARAMEL_PUSH")) != 0;
  if (getenv("CARAMEL_LL128_MAX")) h_ll128_max = strtoull(getenv("CARAMEL_LL128_MAX"), 0, 10);
  int rc = validate_workers(pattern, world);
  if (rc) return rc;
  if (depth < 1 || depth > CARAMEL_MAX_DEPTH)
    return set_err(CARAMEL_EINVAL, "depth must be in [1, %d]", CARAMEL_MAX_DEPTH);
  // The CTA count follows the bytes each rank owns (numel / world), NOT the
  // per-chunk share: chunk-parallel groups then split the same grid, so a
  // deeper split costs no parallelism (round 1 divided by depth as well, and a
  // 4 MiB bucket at depth 8 ran on 16 CTAs instead of 64: 55.6 vs 26.6 us).
  uint64_t per = numel / (uint64_t)world;
  const uint64_t tile = (uint64_t)THREADS * 4 * 2;   // one trip of rs_ag_range
  uint64_t g;
  if (world == 1) {
    g = (numel + 4 * tile - 1) / (4 * tile);
    if (g > 148 * 4) g = 148 * 4;
  } else if (use_ll(pattern, world, numel)) {
    g = (per / depth + 511) / 512;  // latency-bound: spread the few elements wide
    if (g > 32) g = 32;
  } else if (use_ll128(pattern, world, numel)) {
    g = (ll128_lines(numel) / world + 127) / 128;  // ~2 lines per 8-lane group per shard
    if (g > 96) g = 96;
  } else {
    g = (per + tile - 1) / tile;
    uint64_t cap = (uint64_t)default_max_ctas();
    if (g > cap) g = cap;
  }
  if (world > 1 && g < (uint64_t)depth) g = depth;  // chunk-parallel: at least one CTA per chunk
  if (g < 1) g = 1;
  if (ctas) *ctas = (int32_t)g;
  if (bucket_bytes) {
    *bucket_bytes = kernel_region_bytes(numel, pattern, world);
    if (world > 1 && pattern == CARAMEL_SHUFFLE)  // + the copy-engine engine's staging slots
      *bucket_bytes = ce_stage_off(numel, depth, pattern, world) + (uint64_t)(world - 1) * ce_slot_bytes(numel, world);
  }
  if (flag_bytes) {
    uint64_t fb = world == 1 ? 0 : (uint64_t)depth * g * nslots(pattern, world) * world * 4;
    *flag_bytes = (fb + 255) & ~255ull;
  }
  return 0;
}

int caramel_init(int rank, int world, int nlocal, uint64_t arena_bytes, uint64_t param_arena_bytes,
                 caramel_ctx** out) {
  if (!out) return set_err(CARAMEL_EINVAL, "null ctx output");
  *out = nullptr;
  load_ll_max();
  if (world < 1 || world > MAXR) return set_err(CARAMEL_EWORKERS, "world %d outside [1, %d]", world, MAXR);
  if (nlocal != 1 && nlocal != world) return set_err(CARAMEL_EINVAL, "nlocal must be 1 or world");
  if (nlocal == world && rank != 0) return set_err(CARAMEL_EINVAL, "rank emulation requires rank 0");
  if (rank < 0 || rank >= world) return set_err(CARAMEL_EINVAL, "rank %d outside [0, %d)", rank, world);
  caramel_ctx* c = new (std::nothrow) caramel_ctx();  // value-initialised: PODs zeroed
  if (!c) return set_err(CARAMEL_EINVAL, "out of host memory");
  c->rank = rank;
  c->world = world;
  c->nlocal = nlocal;
  const uint64_t G2 = 2ull << 20;
  c->arena_bytes = ((arena_bytes ? arena_bytes : 1) + G2 - 1) / G2 * G2;
  c->param_bytes = param_arena_bytes ? (param_arena_bytes + G2 - 1) / G2 * G2 : 0;
  c->timeout_ns = 5ull * 1000 * 1000 * 1000;
  if (const char* e = getenv("CARAMEL_WATCHDOG_MS")) c->timeout_ns = strtoull(e, 0, 10) * 1000000ull;
  c->gated_ctas = 32;
  if (const char* e = getenv("CARAMEL_GATED_CTAS")) c->gated_ctas = atoi(e);
  if (c->gated_ctas < 1) c->gated_ctas = 1;
  if (c->gated_ctas > 148) c->gated_ctas = 148;
  int rc = 0;
  cudaError_t e;
  if ((e = cudaGetDevice(&c->device)) != cudaSuccess) { rc = set_err(CARAMEL_ECUDA, "cudaGetDevice: %s", cudaGetErrorString(e)); goto fail; }
  if ((e = cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->device)) != cudaSuccess) { rc = set_err(CARAMEL_ECUDA, "attr: %s", cudaGetErrorString(e)); goto fail; }
  for (int i = 0; i < nlocal; ++i) {
    if ((e = cudaMalloc(&c->arena_local[i], c->arena_bytes + SYNC_BYTES)) != cudaSuccess) { rc = set_err(CARAMEL_ECUDA, "cudaMalloc arena (%llu B): %s", (unsigned long long)c->arena_bytes, cudaGetErrorString(e)); goto fail; }
    if ((e = cudaMemset(c->arena_local[i], 0, c->arena_bytes + SYNC_BYTES)) != cudaSuccess) { rc = set_err(CARAMEL_ECUDA, "memset: %s", cudaGetErrorString(e)); goto fail; }
    if (c->param_bytes) {
      if ((e = cudaMalloc(&c->param_local[i], c->param_bytes)) != cudaSuccess) { rc = set_err(CARAMEL_ECUDA, "cudaMalloc param arena: %s", cudaGetErrorString(e)); goto fail; }
      if ((e = cudaMemset(c->param_local[i], 0, c->param_bytes)) != cudaSuccess) { rc = set_err(CARAMEL_ECUDA, "memset: %s", cudaGetErrorString(e)); goto fail; }
    }
    int r = rank + i;
    c->arena[r] = (uint64_t)c->arena_local[i];
    c->parena[r] = (uint64_t)c->param_local[i];
  }
  if ((e = cudaMalloc(&c->status, 3 * sizeof(int))) != cudaSuccess) { rc = set_err(CARAMEL_ECUDA, "cudaMalloc status: %s", cudaGetErrorString(e)); goto fail; }
  if ((e = cudaMemset(c->status, 0, 3 * sizeof(int))) != cudaSuccess) { rc = set_err(CARAMEL_ECUDA, "memset: %s", cudaGetErrorString(e)); goto fail; }
  c->epoch_dev = reinterpret_cast<uint32_t*>(c->status + 1);
  if ((e = cudaHostAlloc((void**)&c->hstatus, sizeof(int), cudaHostAllocMapped)) != cudaSuccess) { rc = set_err(CARAMEL_ECUDA, "cudaHostAlloc status: %s", cudaGetErrorString(e)); goto fail; }
  *(volatile int*)c->hstatus = 0;
  if ((e = cudaHostGetDevicePointer((void**)&c->hstatus_dev, c->hstatus, 0)) != cudaSuccess) { rc = set_err(CARAMEL_ECUDA, "cudaHostGetDevicePointer: %s", cudaGetErrorString(e)); goto fail; }
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) { rc = set_err(CARAMEL_ECUDA, "sync: %s", cudaGetErrorString(e)); goto fail; }
  c->imported = (nlocal == world);
  *out = c;
  return 0;
fail:
  caramel_finalize(c);
  return rc;
}

int caramel_handle_size(void) { return (int)sizeof(Blob); }

int caramel_export(caramel_ctx* c, void* blob) {
  if (!c || !blob) return set_err(CARAMEL_EINVAL, "null argument");
  if (c->nlocal != 1) return set_err(CARAMEL_ESTATE, "export is for one-rank-per-process contexts");
  Blob b;
  memset(&b, 0, sizeof(b));
  b.magic = 0xCA7A3E1u;
  b.rank = c->rank;
  b.world = c->world;
  b.arena_bytes = c->arena_bytes;
  b.param_bytes = c->param_bytes;
  b.has_param = c->param_bytes ? 1 : 0;
  CUDA_TRY(cudaIpcGetMemHandle(&b.arena, c->arena_local[0]));
  if (c->param_bytes) CUDA_TRY(cudaIpcGetMemHandle(&b.param, c->param_local[0]));
  memcpy(blob, &b, sizeof(b));
  return 0;
}

int caramel_import(caramel_ctx* c, const void* blobs) {
  if (!c || !blobs) return set_err(CARAMEL_EINVAL, "null argument");
  if (c->imported) return set_err(CARAMEL_ESTATE, "peers already mapped");
  const Blob* bs = (const Blob*)blobs;
  for (int q = 0; q < c->world; ++q) {
    const Blob& b = bs[q];
    if (b.magic != 0xCA7A3E1u || (int)b.rank != q || (int)b.world != c->world)
      return set_err(CARAMEL_EINVAL, "bootstrap blob %d is malformed or out of rank order", q);
    if (b.arena_bytes != c->arena_bytes || b.param_bytes != c->param_bytes)
      return set_err(CARAMEL_EINVAL, "rank %d arena sizes differ (arenas must be symmetric)", q);
  }
  for (int q = 0; q < c->world; ++q) {
    if (q == c->rank) continue;
    void* p = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&p, bs[q].arena, cudaIpcMemLazyEnablePeerAccess));
    c->arena[q] = (uint64_t)p;
    c->opened[q] = true;
    if (c->param_bytes) {
      void* pp = nullptr;
      CUDA_TRY(cudaIpcOpenMemHandle(&pp, bs[q].param, cudaIpcMemLazyEnablePeerAccess));
      c->parena[q] = (uint64_t)pp;
    }
  }
  c->imported = true;
  return 0;
}

int caramel_arena(caramel_ctx* c, int lr, uint64_t* bucket_arena, uint64_t* param_arena) {
  if (!c || lr < 0 || lr >= c->nlocal) return set_err(CARAMEL_EINVAL, "bad local rank");
  if (bucket_arena) *bucket_arena = (uint64_t)c->arena_local[lr];
  if (param_arena) *param_arena = (uint64_t)c->param_local[lr];
  return 0;
}

static int poisoned_err(const caramel_ctx* c, int s) {
  return set_err(s, "a cross-rank flag wait exceeded the %llu ms watchdog; the context is poisoned (every "
                    "later launch exits before storing anything): finalize it and re-bootstrap",
                 (unsigned long long)(c->timeout_ns / 1000000ull));
}

int caramel_status(caramel_ctx* c) {
  if (!c) return set_err(CARAMEL_EINVAL, "null ctx");
  CUDA_TRY(cudaDeviceSynchronize());
  int s = 0;
  CUDA_TRY(cudaMemcpy(&s, c->status, sizeof(int), cudaMemcpyDeviceToHost));
  if (!s && c->hstatus) s = *(volatile int*)c->hstatus;
  return s ? poisoned_err(c, s) : 0;  // sticky: the flags of a timed-out context are out of step
}

int caramel_poll(caramel_ctx* c) {
  if (!c) return set_err(CARAMEL_EINVAL, "null ctx");
  const int s = c->hstatus ? *(volatile int*)c->hstatus : 0;
  return s ? poisoned_err(c, s) : 0;
}

int caramel_set_timeout_ms(caramel_ctx* c, uint64_t ms) {
  if (!c) return set_err(CARAMEL_EINVAL, "null ctx");
  c->timeout_ns = ms * 1000000ull;
  return 0;
}

static void mc_release(caramel_ctx* c);

int caramel_finalize(caramel_ctx* c) {
  if (!c) return 0;
  if (c->ce_worker_started) {
    {
      std::lock_guard<std::mutex> lk(c->ce_mu);
      c->ce_stop = true;
    }
    c->ce_cv.notify_all();
    c->ce_worker.join();  // drains what was submitted
    for (int i = 0; i < CE_POOL; ++i) cudaEventDestroy(c->ce_pool[i]);
  }
  cudaDeviceSynchronize();  // nothing in flight touches the arenas below
  mc_release(c);
  for (int q = 0; q < MAXR; ++q) {
    if (c->opened[q]) {
      cudaIpcCloseMemHandle((void*)c->arena[q]);
      if (c->parena[q]) cudaIpcCloseMemHandle((void*)c->parena[q]);
    }
  }
  for (int i = 0; i < MAXR; ++i) {
    if (c->arena_local[i]) cudaFree(c->arena_local[i]);
    if (c->param_local[i]) cudaFree(c->param_local[i]);
  }
  if (c->status) cudaFree(c->status);
  if (c->hstatus) cudaFreeHost(c->hstatus);
  if (c->ce_ready) {
    cudaStreamDestroy(c->ce_send);
    cudaEventDestroy(c->ce_grads);
  }
  delete c;
  return 0;
}

// One full wave: SMs x resident CTAs of `fn` (592 CTAs at 3 resident per SM
// left a 148-CTA second wave: 47.5 -> measured below)
static int grid_for(uint64_t numel, const void* fn) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms < 1) sms = 148;
  }
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, THREADS, 0) != cudaSuccess || per_sm < 1) per_sm = 1;
  uint64_t g = (numel + (uint64_t)THREADS * 16 - 1) / ((uint64_t)THREADS * 16);
  const uint64_t cap = (uint64_t)sms * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

static int pack_tma(const caramel_segment* segs, int32_t nseg, uint64_t numel, float* bucket, bool unpack,
                    int to_param, void* stream) {
  static int sms = 0;
  static bool attr[2] = {false, false};
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms < 1) sms = 148;
  }
  auto fn = unpack ? k_pack_tma<true> : k_pack_tma<false>;
  if (!attr[unpack]) {
    CUDA_TRY(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(KtSmem)));
    attr[unpack] = true;
  }
  const uint64_t tiles = (numel + KT_TILE - 1) / KT_TILE;
  const uint64_t slots = (uint64_t)sms * KT_CTAS_PER_SM;
  const int grid = (int)(tiles < slots ? tiles : slots);
  fn<<<grid, KT_THREADS, sizeof(KtSmem), (cudaStream_t)stream>>>(segs, nseg, numel, bucket, to_param);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int caramel_pack(const caramel_segment* segs, int32_t nseg, uint64_t numel, float* bucket, void* stream) {
  if (!segs || nseg < 1 || !bucket) return set_err(CARAMEL_EINVAL, "pack: null table or bucket");
  if (((uintptr_t)bucket) & 15) return set_err(CARAMEL_EINVAL, "pack: bucket must be 16-byte aligned");
  if (numel == 0) return 0;
  if (!getenv("CARAMEL_NO_TMA")) return pack_tma(segs, nseg, numel, bucket, false, 0, stream);
  k_pack<<<grid_for(numel, (const void*)k_pack), THREADS, 0, (cudaStream_t)stream>>>(segs, nseg, numel, bucket);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int caramel_unpack(const caramel_segment* segs, int32_t nseg, uint64_t numel, const float* bucket,
                   int32_t to_param, void* stream) {
  if (!segs || nseg < 1 || !bucket) return set_err(CARAMEL_EINVAL, "unpack: null table or bucket");
  if (((uintptr_t)bucket) & 15) return set_err(CARAMEL_EINVAL, "unpack: bucket must be 16-byte aligned");
  if (numel == 0) return 0;
  if (!getenv("CARAMEL_NO_TMA"))
    return pack_tma(segs, nseg, numel, const_cast<float*>(bucket), true, to_param ? 1 : 0, stream);
  k_unpack<<<grid_for(numel, (const void*)k_unpack), THREADS, 0, (cudaStream_t)stream>>>(segs, nseg, numel, bucket, to_param ? 1 : 0);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // extern "C"

typedef void (*kfn_t)(const KParams);
typedef void (*mfn_t)(const MParams);

template <int PAT>
static kfn_t pick_np(int p) {
  if (PAT != CARAMEL_SHUFFLE) return k_collective<PAT, 2>;  // NP only shapes the two-shot reduce
  switch (p) {
    case 2: return k_collective<PAT, 2>;
    case 3: return k_collective<PAT, 3>;
    case 4: return k_collective<PAT, 4>;
    case 5: return k_collective<PAT, 5>;
    case 6: return k_collective<PAT, 6>;
    case 7: return k_collective<PAT, 7>;
    default: return k_collective<PAT, 8>;
  }
}

static mfn_t pick_fused(int p) {
  switch (p) {
    case 2: return k_shuffle_fused<2>;
    case 3: return k_shuffle_fused<3>;
    case 4: return k_shuffle_fused<4>;
    case 5: return k_shuffle_fused<5>;
    case 6: return k_shuffle_fused<6>;
    case 7: return k_shuffle_fused<7>;
    default: return k_shuffle_fused<8>;
  }
}

template <int PAT>
static mfn_t pick_np_many(int p) {
  if (PAT != CARAMEL_SHUFFLE) return k_collective_many<PAT, 2>;  // NP does not shape ring / hd
  switch (p) {
    case 2: return k_collective_many<PAT, 2>;
    case 3: return k_collective_many<PAT, 3>;
    case 4: return k_collective_many<PAT, 4>;
    case 5: return k_collective_many<PAT, 5>;
    case 6: return k_collective_many<PAT, 6>;
    case 7: return k_collective_many<PAT, 7>;
    default: return k_collective_many<PAT, 8>;
  }
}

typedef void (*pfn_push)(const PushParams);

static pfn_push pick_push(int p) {
  switch (p) {
    case 2: return k_push<2>;
    case 3: return k_push<3>;
    case 4: return k_push<4>;
    case 5: return k_push<5>;
    case 6: return k_push<6>;
    case 7: return k_push<7>;
    default: return k_push<8>;
  }
}

static size_t push_smem(int p) {
  switch (p) {
    case 2: return PushGeo<2>::SMEM;
    case 3: return PushGeo<3>::SMEM;
    case 4: return PushGeo<4>::SMEM;
    case 5: return PushGeo<5>::SMEM;
    case 6: return PushGeo<6>::SMEM;
    case 7: return PushGeo<7>::SMEM;
    default: return PushGeo<8>::SMEM;
  }
}

// CTAs of a push launch when the caller leaves it to the library
static int push_default_ctas() {
  static int v = 0;
  if (!v) v = getenv("CARAMEL_PUSH_CTAS") ? atoi(getenv("CARAMEL_PUSH_CTAS")) : 32;
  return v < 1 ? 1 : v;
}

extern "C" {

static int validate_bucket(const caramel_ctx* c, const caramel_bucket* b) {
  int rc = validate_workers(b->pattern, c->world);
  if (rc) return rc;
  if (b->depth < 1 || b->depth > CARAMEL_MAX_DEPTH)
    return set_err(CARAMEL_EINVAL, "depth must be in [1, %d]", CARAMEL_MAX_DEPTH);
  if (b->epilogue < 0 || b->epilogue > 2) return set_err(CARAMEL_EINVAL, "unknown epilogue %d", b->epilogue);
  if (b->ctas < 1) return set_err(CARAMEL_EINVAL, "ctas must be >= 1 (see caramel_bucket_layout)");
  if (b->bucket_off & 15) return set_err(CARAMEL_EINVAL, "bucket_off must be 16-byte aligned");
  if (b->numel == 0) return 0;
  const uint64_t span = use_ll(b->pattern, c->world, b->numel) ? ll_region_bytes(b->numel, c->world)
                        : use_ll128(b->pattern, c->world, b->numel)
                            ? ll128_region_bytes(b->numel, c->world)
                            : 4 * ((c->world > 1 && b->pattern != CARAMEL_SHUFFLE) ? 2 * out_region_elems(b->numel)
                                                                                   : b->numel);
  const int proto = shuffle_proto(*b, c->world);
  const uint64_t span2 = (proto == PROTO_OS || proto == PROTO_TS)
                             ? push_off(b->numel, CARAMEL_SHUFFLE, c->world) +
                                   push_region_bytes(b->numel, b->depth, CARAMEL_SHUFFLE, c->world)
                             : span;
  if (b->bucket_off + (span2 > span ? span2 : span) > c->arena_bytes)
    return set_err(CARAMEL_EINVAL, "bucket [%llu, +%llu B) exceeds the arena (size it with caramel_bucket_layout)",
                   (unsigned long long)b->bucket_off, (unsigned long long)(span2 > span ? span2 : span));
  const bool arena = (b->flags & CARAMEL_F_PARAM_ARENA) && b->epilogue == CARAMEL_EPI_SGD;
  if (arena) {
    if (!c->param_bytes) return set_err(CARAMEL_EINVAL, "PARAM_ARENA requested but no parameter arena");
    if ((b->param_off & 15) || b->param_off + b->numel * 4 > c->param_bytes)
      return set_err(CARAMEL_EINVAL, "param_off misaligned or out of the parameter arena");
  }
  const bool needs_segs = (b->flags & CARAMEL_F_PACK) || ((b->flags & CARAMEL_F_UNPACK) && !arena) ||
                          (b->epilogue == CARAMEL_EPI_SGD && !arena);
  if (needs_segs && (!b->segs || b->nseg < 1)) return set_err(CARAMEL_EINVAL, "segment table required");
  if (c->world > 1) {
    uint64_t fb = (uint64_t)b->depth * b->ctas * nslots(b->pattern, c->world) * c->world * 4;
    if (b->flag_off + fb > c->arena_bytes) return set_err(CARAMEL_EINVAL, "flag block exceeds the arena");
    if (b->flag_off & 3) return set_err(CARAMEL_EINVAL, "flag_off must be 4-byte aligned");
  }
  return 0;
}

static void fill_env(const caramel_ctx* c, Env& E, uint32_t epoch) {
  memset(&E, 0, sizeof(E));
  for (int q = 0; q < MAXR; ++q) {
    E.arena[q] = c->arena[q];
    E.parena[q] = c->parena[q];
  }
  E.world = c->world;
  E.rank_base = c->rank;
  E.epoch = epoch;
  E.epoch_dev = c->epoch_dev;
  E.timeout_ns = c->timeout_ns;
  E.status = c->status;
  E.hstatus = c->hstatus_dev;
  E.sync_off = c->arena_bytes;
}

}  // extern "C"

// rank emulation: all ranks' CTAs spin on each other, so they must be
// co-resident -- a cooperative launch guarantees it or fails
// Also used for k_shuffle_fused with one rank per process: its grid barriers
// need every CTA resident, which only a cooperative launch guarantees (other
// kernels -- backward, NCCL -- may hold SMs).  cudaLaunchKernelEx with the
// cooperative attribute is capturable in a CUDA graph.
template <class Params>
static int coop_launch(const caramel_ctx* c, void (*fn)(Params), dim3 grid, const Params& P, void* stream,
                       size_t smem = 0) {
  int per_sm = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void*)fn, THREADS, smem));
  if ((uint64_t)per_sm * c->sms < (uint64_t)grid.x * grid.y)
    return set_err(CARAMEL_EINVAL, "cooperative launch of %u x %u CTAs exceeds co-residency (%d per SM)", grid.x,
                   grid.y, per_sm);
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof(cfg));
  cfg.gridDim = grid;
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, fn, P));
  return 0;
}

extern "C" {

// CARAMEL_MANY_FUSED lists through the push kernel with this many CTAs (0: the
// grid-barrier pull kernel k_shuffle_fused)
static int fused_push() {
  static int v = -1;
  if (v < 0) v = getenv("CARAMEL_FUSED_PUSH") ? atoi(getenv("CARAMEL_FUSED_PUSH")) : 0;
  return v;
}

// kernel family of a bucket in a CARAMEL_MANY_FLAGS list: 1 = push kernel
// (OS / TS), 0 = the flag list kernel (LL, PULL); runs of one family launch together
static int push_family(const caramel_bucket& b, int world) {
  const int pr = shuffle_proto(b, world);
  return pr == PROTO_OS || pr == PROTO_TS;
}

// The push kernel over `count` buckets (host copy `host`; device copy at
// `dev_list`, or 0 for a single bucket passed by value).  ctas <= 0: the
// largest tile-range count of the list.
static int push_launch(caramel_ctx* c, const caramel_bucket* host, int count, uint64_t dev_list, int ctas,
                       uint32_t epoch, void* stream, int with_ll = 0) {
  PushParams P;
  memset(&P, 0, sizeof(P));
  fill_env(c, P.env, epoch);
  P.bs = reinterpret_cast<const caramel_bucket*>(dev_list);
  P.nb = count;
  P.with_ll = with_ll;
  P.one = host[0];
  // default grid: enough CTAs for the items, at most CARAMEL_PUSH_CTAS (a
  // small footprint leaves the SMs to the backward pass); LL buckets need
  // their own CTA slots
  uint64_t items = 0;
  int G = 1;
  for (int i = 0; i < count; ++i) {
    const int pr = shuffle_proto(host[i], c->world);
    if (pr == PROTO_LL) G = host[i].ctas > G ? host[i].ctas : G;
    else items += (uint64_t)host[i].depth * push_ranges(host[i].numel, host[i].depth);
  }
  const uint64_t want = items < (uint64_t)push_default_ctas() ? items : (uint64_t)push_default_ctas();
  if ((int)want > G) G = (int)want;
  if (ctas > 0) G = ctas;
  if (c->nlocal > 1 && G * c->nlocal > c->sms) G = c->sms / c->nlocal;  // emulated ranks: all co-resident
  const int p = c->world;
  pfn_push fn = pick_push(p);
  const size_t smem = push_smem(p);
  static bool attr[MAXR + 1] = {false};
  if (!attr[p]) {
    CUDA_TRY(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr[p] = true;
  }
  // PACK buckets: gather the members into each local rank's bucket first (K1)
  for (int i = 0; i < count; ++i) {
    const caramel_bucket& b = host[i];
    if (!(b.flags & CARAMEL_F_PACK) || !b.numel || !push_family(b, c->world)) continue;
    for (int lr = 0; lr < c->nlocal; ++lr) {
      const caramel_segment* segs = reinterpret_cast<const caramel_segment*>(b.segs) + (uint64_t)lr * b.nseg;
      float* bkt = reinterpret_cast<float*>(c->arena[c->rank + lr] + b.bucket_off);
      k_pack<<<grid_for(b.numel, (const void*)k_pack), THREADS, 0, (cudaStream_t)stream>>>(segs, b.nseg, b.numel,
                                                                                           bkt);
    }
    CUDA_TRY(cudaGetLastError());
  }
  dim3 grid(G, c->nlocal);
  if (c->nlocal > 1 || with_ll) return coop_launch(c, fn, grid, P, stream, smem);
  fn<<<grid, THREADS, smem, (cudaStream_t)stream>>>(P);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

static int launch(caramel_ctx* c, const caramel_bucket* b, uint32_t epoch, void* stream) {
  if (!c || !b) return set_err(CARAMEL_EINVAL, "null argument");
  if (!c->imported) return set_err(CARAMEL_ESTATE, "peer arenas not mapped (call caramel_import)");
  int rc = validate_bucket(c, b);
  if (rc) return rc;
  if (b->numel == 0) return 0;
  if ((b->flags & CARAMEL_F_AUTO_EPOCH) && epoch != 0)
    return set_err(CARAMEL_EINVAL, "CARAMEL_F_AUTO_EPOCH takes its epoch from the device counter: pass epoch 0");
  if (c->world > 1) {
    const int pr = shuffle_proto(*b, c->world);
    if (pr == PROTO_OS || pr == PROTO_TS) {
      if (b->flags & CARAMEL_F_AUTO_EPOCH)
        return set_err(CARAMEL_EINVAL, "CARAMEL_F_AUTO_EPOCH is not supported by the push engine");
      return push_launch(c, b, 1, 0, 0, epoch, stream);
    }
  }
  KParams P;
  fill_env(c, P.env, epoch);
  P.b = *b;
  kfn_t fn;
  if (c->world == 1) fn = k_local;
  else if (b->pattern == CARAMEL_SHUFFLE) fn = pick_np<CARAMEL_SHUFFLE>(c->world);
  else if (b->pattern == CARAMEL_RING) fn = pick_np<CARAMEL_RING>(c->world);
  else fn = pick_np<CARAMEL_HD>(c->world);
  dim3 grid(b->ctas, c->nlocal);
  if (c->nlocal > 1) return coop_launch(c, fn, grid, P, stream);
  fn<<<grid, THREADS, 0, (cudaStream_t)stream>>>(P);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int caramel_epoch_advance(caramel_ctx* c, void* stream) {
  if (!c) return set_err(CARAMEL_EINVAL, "null ctx");
  k_epoch_advance<<<1, 1, 0, (cudaStream_t)stream>>>(c->epoch_dev);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

int caramel_allreduce(caramel_ctx* c, const caramel_bucket* b, uint32_t epoch, void* stream) {
  if (b && b->epilogue == CARAMEL_EPI_SGD)
    return set_err(CARAMEL_EINVAL, "caramel_allreduce: use caramel_allreduce_update for the SGD epilogue");
  return launch(c, b, epoch, stream);
}

int caramel_allreduce_update(caramel_ctx* c, const caramel_bucket* b, uint32_t epoch, void* stream) {
  if (b && b->epilogue != CARAMEL_EPI_SGD)
    return set_err(CARAMEL_EINVAL, "caramel_allreduce_update requires CARAMEL_EPI_SGD");
  return launch(c, b, epoch, stream);
}

int caramel_allreduce_many(caramel_ctx* c, const caramel_bucket* host, int32_t count, uint64_t dev_buckets,
                           uint64_t dev_prefix, uint64_t dev_segprefix, int32_t ctas, int32_t mode,
                           uint32_t epoch, void* stream) {
  if (mode != CARAMEL_MANY_FUSED && mode != CARAMEL_MANY_FLAGS)
    return set_err(CARAMEL_EINVAL, "allreduce_many: unknown mode %d", mode);
  if (!c || !host || count < 1 || !dev_buckets || !dev_prefix || !dev_segprefix)
    return set_err(CARAMEL_EINVAL, "allreduce_many: null argument or empty list");
  if (!c->imported) return set_err(CARAMEL_ESTATE, "peer arenas not mapped (call caramel_import)");
  const int pattern = host[0].pattern;
  int gmax = 1;
  uint64_t total = 0;
  for (int i = 0; i < count; ++i) {
    if (host[i].pattern != pattern || host[i].epilogue != host[0].epilogue ||
        (host[i].flags & ~CARAMEL_F_FLAT) != (host[0].flags & ~CARAMEL_F_FLAT))
      return set_err(CARAMEL_EINVAL, "allreduce_many: buckets must share pattern, epilogue and flags");
    if (host[i].flags & CARAMEL_F_AUTO_EPOCH)
      return set_err(CARAMEL_EINVAL, "allreduce_many: CARAMEL_F_AUTO_EPOCH is for single-bucket calls");
    int rc = validate_bucket(c, &host[i]);
    if (rc) return rc;
    if (host[i].ctas > gmax) gmax = host[i].ctas;
    total += host[i].numel;
  }
  if (total == 0) return 0;
  if (c->world == 1) {
    // one wave at 2 CTAs per SM (per-CTA setup is paid once per SM slot)
    uint64_t g = (total + (uint64_t)THREADS * 16 - 1) / ((uint64_t)THREADS * 16);
    uint64_t cap = (uint64_t)c->sms * 2;
    gmax = (int)(g < 1 ? 1 : (g > cap ? cap : g));
  }
  MParams P;
  fill_env(c, P.env, epoch);
  P.bs = reinterpret_cast<const caramel_bucket*>(dev_buckets);
  P.prefix = reinterpret_cast<const uint64_t*>(dev_prefix);
  P.segprefix = reinterpret_cast<const uint64_t*>(dev_segprefix);
  P.nb = count;
  P.claim = 0;
  if (pattern == CARAMEL_SHUFFLE && mode == CARAMEL_MANY_FUSED && c->world > 1) {
    static int claim = -1;
    // one item per atomic measured best: 172 vs 178 us (p=2), 250 vs 256 us (p=4) for resnet50
    if (claim < 0) claim = getenv("CARAMEL_FUSED_CLAIM") ? atoi(getenv("CARAMEL_FUSED_CLAIM")) : 1;
    P.claim = claim;
  }
  mfn_t fn;
  bool flat_tma = c->world == 1 && c->nlocal == 1 && count <= TMA_MAX_BUCKETS && !getenv("CARAMEL_NO_TMA");
  for (int i = 0; i < count && flat_tma; ++i)  // packed from one flat run, or already in the bucket
    flat_tma = (((host[i].flags & CARAMEL_F_FLAT) && (host[i].flags & CARAMEL_F_PACK) && host[i].nseg == 1) ||
                !(host[i].flags & CARAMEL_F_PACK)) &&
               (host[i].flags & CARAMEL_F_PARAM_ARENA) && host[i].epilogue == CARAMEL_EPI_SGD;
  if (flat_tma) {
    // tile geometry (floats x stages), measured on resnet50 (82 -> 88% of HBM):
    // 4096x6 5.35 TB/s, 5120x5 5.55, 6144x4 5.54, 8192x3 5.76 -- per-tile
    // overhead (mbarrier wait, CTA barrier, the issuing thread's bookkeeping)
    // outweighs the deeper prefetch; two CTAs of 16 KB x 3 per SM (4096x3x2)
    // tie with 8192x3 at 5.75 TB/s.  CARAMEL_TMA=4096x6 / 4096x3x2 select those
    static int variant = -1;
    if (variant < 0) {
      const char* e = getenv("CARAMEL_TMA");
      variant = (e && !strcmp(e, "4096x6")) ? 1 : (e && !strcmp(e, "4096x3x2")) ? 2 : 0;
    }
    void (*fn)(MParams) = k_local_flat_tma<8192, 3>;
    size_t smem = sizeof(TmaSmem<8192, 3>);
    int per_sm = 1;
    if (variant == 1) { fn = k_local_flat_tma<4096, 6>; smem = sizeof(TmaSmem<4096, 6>); }
    if (variant == 2) { fn = k_local_flat_tma<4096, 3>; smem = sizeof(TmaSmem<4096, 3>); per_sm = 2; }
    static bool attr[3] = {false, false, false};
    if (!attr[variant]) {
      CUDA_TRY(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr[variant] = true;
    }
    fn<<<dim3(c->sms * per_sm, 1), TMA_THREADS, smem, (cudaStream_t)stream>>>(P);
    CUDA_TRY(cudaGetLastError());
    return 0;
  }
  if (c->world > 1 && pattern == CARAMEL_SHUFFLE && mode == CARAMEL_MANY_FLAGS) {
    // maximal runs of one protocol family, in launch order: the push kernel
    // (one-shot / two-shot push, LL) or the pull list kernel (UNPACK, member
    // parameters).  A bucket's protocol never depends on how it is grouped.
    const size_t bsz = sizeof(caramel_bucket);
    int i = 0;
    while (i < count) {
      const int fam = push_family(host[i], c->world);
      int k = i + 1;
      while (k < count && push_family(host[k], c->world) == fam) ++k;
      int rc = 0;
      if (fam) {
        rc = push_launch(c, host + i, k - i, dev_buckets + i * bsz, ctas, epoch, stream);
      } else {
        MParams Q = P;
        Q.bs = P.bs + i;
        Q.prefix = P.prefix + i;
        Q.segprefix = P.segprefix + i;
        Q.nb = k - i;
        int need = 1;
        for (int t = i; t < k; ++t) need = host[t].ctas > need ? host[t].ctas : need;
        const int g = ctas > 0 ? (ctas < need ? need : ctas) : need;
        mfn_t f = pick_np_many<CARAMEL_SHUFFLE>(c->world);
        dim3 grid(g, c->nlocal);
        if (c->nlocal > 1) rc = coop_launch(c, f, grid, Q, stream);
        else {
          f<<<grid, THREADS, 0, (cudaStream_t)stream>>>(Q);
          cudaError_t e = cudaGetLastError();
          if (e != cudaSuccess) rc = set_err(CARAMEL_ECUDA, "k_collective_many: %s", cudaGetErrorString(e));
        }
      }
      if (rc) return rc;
      i = k;
    }
    return 0;
  }
  if (c->world > 1 && pattern == CARAMEL_SHUFFLE && mode == CARAMEL_MANY_FUSED && fused_push()) {
    // every rank issues this identical list: the push kernel with the LL
    // buckets in the same launch, cooperative (all CTAs resident)
    bool ok = true;
    for (int i = 0; i < count && ok; ++i) ok = shuffle_proto(host[i], c->world) != PROTO_PULL;
    if (ok) return push_launch(c, host, count, dev_buckets, ctas > 0 ? ctas : fused_push(), epoch, stream, 1);
  }
  if (c->world == 1) fn = k_local_many;
  else if (pattern == CARAMEL_SHUFFLE && mode == CARAMEL_MANY_FLAGS) {
    fn = pick_np_many<CARAMEL_SHUFFLE>(c->world);
  } else if (pattern == CARAMEL_SHUFFLE) {
    if (count > MAX_FUSED_BUCKETS)
      return set_err(CARAMEL_EINVAL, "allreduce_many: at most %d buckets per fused launch", MAX_FUSED_BUCKETS);
    fn = pick_fused(c->world);
    if (c->nlocal == 1) gmax = c->sms;  // flat phases: by default the whole GPU (one CTA per SM)
  } else if (pattern == CARAMEL_RING) {
    fn = pick_np_many<CARAMEL_RING>(c->world);
  } else {
    fn = pick_np_many<CARAMEL_HD>(c->world);
  }
  if (ctas > 0) {
    // caller's grid; per-bucket-flag and ring/hd lists need every bucket's tiles
    int need = 1;
    for (int i = 0; i < count; ++i) need = host[i].ctas > need ? host[i].ctas : need;
    const bool tiled = c->world > 1 && (mode == CARAMEL_MANY_FLAGS || pattern != CARAMEL_SHUFFLE);
    gmax = tiled && ctas < need ? need : ctas;
  }
  dim3 grid(gmax, c->nlocal);
  // grid barriers (fused) or rank emulation: every CTA must be resident
  const bool fused = pattern == CARAMEL_SHUFFLE && mode == CARAMEL_MANY_FUSED && c->world > 1;
  if (c->nlocal > 1 || fused) return coop_launch(c, fn, grid, P, stream);
  fn<<<grid, THREADS, 0, (cudaStream_t)stream>>>(P);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

// ---------------------------------------------------------------------------
// caramel_allreduce_ce: two-shot on the copy engines, push-based (remote
// writes stream faster than remote reads: ~690 vs ~420-640 GB/s per GPU on
// 4 B200s, tools/ce_bw.py).  Per call (buckets [index0, index0+count) of the
// iteration's launch order, tag = epoch:next position):
//   1. send stream (after the gradients): push my gradients of peer q's shard
//      into q's staging slot for me, for every q; READY[me] = tag on every peer
//   2. `stream`: wait READY[q] >= tag for all q; k_ce_reduce (sum in rank
//      order + epilogue) on my shards
//   3. `stream`: push my result shards into every peer's output arena;
//      DONE[me] = tag on every peer; wait DONE[q] >= tag for all q
// Stream writes are fenced after the stream's prior work, so a peer that
// sees a tag sees the bytes.  The send stream never waits on a peer, so READY
// always goes out; DONE(t) depends only on READY(<= t) and earlier DONEs.
// Every rank must group the launch order into the same calls (a stream wait
// stalls its hardware queue; differently grouped waits could close a cycle).
// ---------------------------------------------------------------------------
typedef CUresult (*pfn_batch)(CUstream, unsigned int, CUstreamBatchMemOpParams*, unsigned int);
typedef CUresult (*pfn_dev_attr)(int*, CUdevice_attribute, CUdevice);
typedef CUresult (*pfn_dev_get)(CUdevice*, int);
static pfn_batch g_batch = nullptr;

static bool ce_probe(const caramel_ctx* c) {
  static int state = 0;  // 1 usable, -1 not
  if (state) return state > 0;
  state = -1;
  void *fa = nullptr, *fg = nullptr, *fw = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuDeviceGetAttribute", &fa, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return false;
  if (cudaGetDriverEntryPoint("cuDeviceGet", &fg, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return false;
  if (cudaGetDriverEntryPoint("cuStreamBatchMemOp", &fw, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return false;
  CUdevice d;
  int v = 0;
  if (((pfn_dev_get)fg)(&d, c->device) != CUDA_SUCCESS) return false;
  if (((pfn_dev_attr)fa)(&v, CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS, d) != CUDA_SUCCESS || !v) return false;
  g_batch = (pfn_batch)fw;
  state = 1;
  return true;
}

static int ce_setup(caramel_ctx* c) {
  if (c->ce_ready) return 0;
  CUDA_TRY(cudaStreamCreateWithFlags(&c->ce_send, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&c->ce_grads, cudaEventDisableTiming));
  c->ce_ready = true;
  return 0;
}

static inline uint64_t shard_lo(uint64_t n, int p, int s) { return (n * (uint64_t)s) / (uint64_t)p; }

// One stream memory-op batch: WRITE (fenced after the stream's prior work, so
// a peer that sees the tag sees the data) or WAIT (>= tag, cyclic 64-bit) on
// `n` addresses.
static CUresult ce_memops(cudaStream_t s, bool wait, const uint64_t* addr, int n, uint64_t tag) {
  CUstreamBatchMemOpParams ops[MAXR];
  memset(ops, 0, sizeof(ops));
  for (int i = 0; i < n; ++i) {
    if (wait) {
      ops[i].waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_64;
      ops[i].waitValue.address = (CUdeviceptr)addr[i];
      ops[i].waitValue.value64 = tag;
      ops[i].waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
    } else {
      ops[i].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
      ops[i].writeValue.address = (CUdeviceptr)addr[i];
      ops[i].writeValue.value64 = tag;
      ops[i].writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
    }
  }
  return n ? g_batch((CUstream)s, (unsigned)n, ops, 0) : CUDA_SUCCESS;
}

#define CU_TRY(expr)                                                                         \
  do {                                                                                       \
    CUresult _r = (expr);                                                                    \
    if (_r != CUDA_SUCCESS) return set_err(CARAMEL_ECUDA, "%s failed: CUresult %d", #expr, (int)_r); \
  } while (0)

int caramel_ce_available(caramel_ctx* c) {
  return c && c->nlocal == 1 && c->world > 1 && ce_probe(c) ? 1 : 0;
}

// staging: the copy engines' reduce-scatter slots must fit (CE); the gated
// SM engine pulls straight from the peers' buckets and needs none
static int ce_validate(caramel_ctx* c, const caramel_bucket* host, int32_t count, uint32_t epoch,
                       bool staging = true) {
  if (!c || !host || count < 1) return set_err(CARAMEL_EINVAL, "allreduce_ce: null argument or empty list");
  if (c->nlocal != 1 || c->world < 2) return set_err(CARAMEL_ESTATE, "allreduce_ce: one rank per process, world >= 2");
  if (!c->imported) return set_err(CARAMEL_ESTATE, "peer arenas not mapped (call caramel_import)");
  if (epoch == 0) return set_err(CARAMEL_EINVAL, "allreduce_ce: epoch must be > 0");
  if (!ce_probe(c)) return set_err(CARAMEL_ESTATE, "allreduce_ce: device lacks 64-bit stream memory operations");
  const int p = c->world;
  const int epi = host[0].epilogue;
  for (int i = 0; i < count; ++i) {
    const caramel_bucket& b = host[i];
    if (b.pattern != CARAMEL_SHUFFLE) return set_err(CARAMEL_EINVAL, "allreduce_ce: SHUFFLE buckets only");
    if (b.epilogue != epi || b.flags != host[0].flags)
      return set_err(CARAMEL_EINVAL, "allreduce_ce: buckets must share epilogue and flags");
    if (b.flags & (CARAMEL_F_PACK | CARAMEL_F_UNPACK | CARAMEL_F_AUTO_EPOCH))
      return set_err(CARAMEL_EINVAL, "allreduce_ce: gradients must live in the bucket arena (no PACK/UNPACK), "
                                     "epochs are explicit (no AUTO_EPOCH)");
    if (epi == CARAMEL_EPI_SGD && !(b.flags & CARAMEL_F_PARAM_ARENA))
      return set_err(CARAMEL_EINVAL, "allreduce_ce: the SGD epilogue needs PARAM_ARENA");
    int rc = validate_bucket(c, &b);
    if (rc) return rc;
    const uint64_t end = b.bucket_off + ce_stage_off(b.numel, b.depth, CARAMEL_SHUFFLE, p) + (uint64_t)(p - 1) * ce_slot_bytes(b.numel, p);
    if (staging && b.numel && end > c->arena_bytes)
      return set_err(CARAMEL_EINVAL, "allreduce_ce: bucket + staging slots exceed the arena (size it with caramel_bucket_layout)");
  }
  return ce_setup(c);
}

// Enqueue one call's work (see the block comment above); `grads` is an event
// recorded on the stream that produced the gradients.
static int ce_enqueue(caramel_ctx* c, const caramel_bucket* host, int32_t count, uint32_t index0, uint32_t epoch,
                      cudaEvent_t grads, cudaStream_t s) {
  const int epi = host[0].epilogue;
  const bool sgd = epi == CARAMEL_EPI_SGD;
  const int me = c->rank, p = c->world;
  const uint64_t tag = ((uint64_t)epoch << 32) | (uint64_t)(index0 + (uint32_t)count);
  const uint64_t ready = c->arena_bytes + CE_FLAG_OFF, done = ready + 8 * MAXR;
  uint64_t peer_ready[MAXR], my_ready[MAXR], peer_done[MAXR], my_done[MAXR];
  int np_ = 0;
  for (int q = 0; q < p; ++q) {
    if (q == me) continue;
    peer_ready[np_] = c->arena[q] + ready + 8 * me;
    my_ready[np_] = c->arena[me] + ready + 8 * q;
    peer_done[np_] = c->arena[q] + done + 8 * me;
    my_done[np_] = c->arena[me] + done + 8 * q;
    ++np_;
  }
  // 1. reduce-scatter: push my gradients of every peer's shard into that
  //    peer's staging slot for me, then READY -- on the send stream, which
  //    never waits on a peer (so READY can always go out)
  CUDA_TRY(cudaStreamWaitEvent(c->ce_send, grads, 0));
  CUDA_TRY(cudaStreamWaitEvent(s, grads, 0));
  for (int r = 1; r < p; ++r) {
    const int q = (me + r) % p;
    const uint64_t k = (uint64_t)(me < q ? me : me - 1);  // my slot at q
    for (int i = 0; i < count; ++i) {
      const uint64_t n = host[i].numel, lo = shard_lo(n, p, q), hi = shard_lo(n, p, q + 1);
      if (hi <= lo) continue;
      const uint64_t stg = host[i].bucket_off + ce_stage_off(n, host[i].depth, CARAMEL_SHUFFLE, p) + k * ce_slot_bytes(n, p) + 4 * (lo & 3);
      CUDA_TRY(cudaMemcpyAsync((void*)(c->arena[q] + stg), (const void*)(c->arena[me] + host[i].bucket_off + 4 * lo),
                               4 * (hi - lo), cudaMemcpyDeviceToDevice, c->ce_send));
    }
  }
  CU_TRY(ce_memops(c->ce_send, false, peer_ready, np_, tag));
  // 2. every peer's contribution to my shards has landed: reduce + epilogue
  CU_TRY(ce_memops(s, true, my_ready, np_, tag));
  for (int i0 = 0; i0 < count; i0 += CE_MAX_BUCKETS) {
    CeParams P;
    memset(&P, 0, sizeof(P));
    P.arena = (const char*)c->arena[me];
    P.out = (char*)(sgd ? c->parena[me] : c->arena[me]);
    P.world = p;
    P.me = me;
    P.epi = epi;
    uint32_t ctas = 0;
    for (int i = i0; i < count && i < i0 + CE_MAX_BUCKETS; ++i) {
      const uint64_t n = host[i].numel, lo = shard_lo(n, p, me), hi = shard_lo(n, p, me + 1);
      if (hi <= lo) continue;
      CeItem& it = P.it[P.count++];
      it.src = host[i].bucket_off + 4 * lo;
      it.stg = host[i].bucket_off + ce_stage_off(n, host[i].depth, CARAMEL_SHUFFLE, p) + 4 * (lo & 3);
      it.slot = ce_slot_bytes(n, p);
      it.dst = (sgd ? host[i].param_off : host[i].bucket_off) + 4 * lo;
      it.n = hi - lo;
      it.cta0 = ctas;
      it.lr = host[i].lr;
      it.scale = host[i].scale;
      ctas += (uint32_t)((it.n + CE_TILE - 1) / CE_TILE);
    }
    if (ctas) {
      k_ce_reduce<<<ctas, CE_THREADS, 0, s>>>(P);
      CUDA_TRY(cudaGetLastError());
    }
  }
  // 3. all-gather: push my result shards into every peer's output arena, DONE,
  //    and wait until every peer's shards have landed here
  const uint64_t out_me = sgd ? c->parena[me] : c->arena[me];
  for (int r = 1; r < p; ++r) {
    const int q = (me + r) % p;
    const uint64_t out_q = sgd ? c->parena[q] : c->arena[q];
    for (int i = 0; i < count; ++i) {
      const uint64_t n = host[i].numel, lo = shard_lo(n, p, me), hi = shard_lo(n, p, me + 1);
      if (hi <= lo) continue;
      const uint64_t off = (sgd ? host[i].param_off : host[i].bucket_off) + 4 * lo;
      CUDA_TRY(cudaMemcpyAsync((void*)(out_q + off), (const void*)(out_me + off), 4 * (hi - lo),
                               cudaMemcpyDeviceToDevice, s));
    }
  }
  CU_TRY(ce_memops(s, false, peer_done, np_, tag));
  CU_TRY(ce_memops(s, true, my_done, np_, tag));
  return 0;
}

typedef void (*gfn_t)(GParams);
static gfn_t pick_gated(int world) {
  switch (world) {
    case 2: return k_gated<2>;
    case 3: return k_gated<3>;
    case 4: return k_gated<4>;
    case 5: return k_gated<5>;
    case 6: return k_gated<6>;
    case 7: return k_gated<7>;
    default: return k_gated<8>;
  }
}

// CTAs of a gated launch: enough rows for every CTA, at most gated_ctas
// (CARAMEL_GATED_CTAS, default 32 -- the rest of the GPU stays with the
// backward pass the launch overlaps)
static int gated_grid(const caramel_ctx* c, const caramel_bucket* b, int n) {
  const int U = GATED_U ? GATED_U : c->world <= 2 ? 4 : 2;
  const uint64_t row = 4ull * U * GATED_THREADS;
  uint64_t rows = 0;
  for (int i = 0; i < n; ++i) rows += (b[i].numel / c->world + row) / row;
  int cap = c->gated_ctas;
  return (int)(rows < (uint64_t)cap ? (rows ? rows : 1) : cap);
}

// Gated SM engine: READY on the send stream after the gradients, wait for
// every peer's READY on `s`, the k_gated launch(es), DONE, wait for every
// peer's DONE.  Same READY / DONE words and tags as the copy-engine engine,
// so calls of both engines can alternate in one launch order.
static int gated_enqueue(caramel_ctx* c, const caramel_bucket* host, int32_t count, uint32_t index0,
                         uint32_t epoch, cudaEvent_t grads, cudaStream_t s) {
  const int me = c->rank, p = c->world;
  const uint64_t tag = ((uint64_t)epoch << 32) | (uint64_t)(index0 + (uint32_t)count);
  const uint64_t ready = c->arena_bytes + CE_FLAG_OFF, done = ready + 8 * MAXR;
  uint64_t peer_ready[MAXR], my_ready[MAXR], peer_done[MAXR], my_done[MAXR];
  int np_ = 0;
  for (int q = 0; q < p; ++q) {
    if (q == me) continue;
    peer_ready[np_] = c->arena[q] + ready + 8 * me;
    my_ready[np_] = c->arena[me] + ready + 8 * q;
    peer_done[np_] = c->arena[q] + done + 8 * me;
    my_done[np_] = c->arena[me] + done + 8 * q;
    ++np_;
  }
  CUDA_TRY(cudaStreamWaitEvent(c->ce_send, grads, 0));
  CU_TRY(ce_memops(c->ce_send, false, peer_ready, np_, tag));
  CUDA_TRY(cudaStreamWaitEvent(s, grads, 0));
  CU_TRY(ce_memops(s, true, my_ready, np_, tag));
  const gfn_t fn = pick_gated(p);
  for (int i0 = 0; i0 < count; i0 += GATED_MAX) {
    GParams P;
    memset(&P, 0, sizeof(P));
    fill_env(c, P.env, 1);
    P.nb = count - i0 < GATED_MAX ? count - i0 : GATED_MAX;
    for (int i = 0; i < P.nb; ++i) P.b[i] = host[i0 + i];
    fn<<<gated_grid(c, P.b, P.nb), GATED_THREADS, 0, s>>>(P);
    CUDA_TRY(cudaGetLastError());
  }
  CU_TRY(ce_memops(s, false, peer_done, np_, tag));
  CU_TRY(ce_memops(s, true, my_done, np_, tag));
  return 0;
}

int caramel_allreduce_gated(caramel_ctx* c, const caramel_bucket* host, int32_t count, uint32_t index0,
                            uint32_t epoch, void* grad_stream, void* stream) {
  int rc = ce_validate(c, host, count, epoch, false);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaEventRecord(c->ce_grads, grad_stream ? (cudaStream_t)grad_stream : s));
  return gated_enqueue(c, host, count, index0, epoch, c->ce_grads, s);
}

int caramel_allreduce_ce(caramel_ctx* c, const caramel_bucket* host, int32_t count, uint32_t index0,
                         uint32_t epoch, void* grad_stream, void* stream) {
  int rc = ce_validate(c, host, count, epoch);
  if (rc) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaEventRecord(c->ce_grads, grad_stream ? (cudaStream_t)grad_stream : s));
  return ce_enqueue(c, host, count, index0, epoch, c->ce_grads, s);
}

// ---- asynchronous submission: a per-context worker thread issues the calls ----
static void ce_worker_main(caramel_ctx* c) {
  cudaSetDevice(c->device);
  std::unique_lock<std::mutex> lk(c->ce_mu);
  for (;;) {
    c->ce_cv.wait(lk, [&] { return c->ce_stop || !c->ce_jobs.empty(); });
    if (c->ce_jobs.empty()) return;  // stop requested and drained
    CeJob job = std::move(c->ce_jobs.front());
    c->ce_jobs.pop_front();
    c->ce_busy = true;
    lk.unlock();
    int rc = 0;
    if (!c->ce_rc) {
      if (job.engine == CARAMEL_ENGINE_CE) {
        rc = ce_enqueue(c, job.buckets.data(), (int32_t)job.buckets.size(), job.index0, job.epoch, job.grads,
                        job.stream);
      } else if (job.engine == CARAMEL_ENGINE_GATED) {
        rc = gated_enqueue(c, job.buckets.data(), (int32_t)job.buckets.size(), job.index0, job.epoch, job.grads,
                           job.stream);
      } else {  // the SM kernels, one launch per bucket, device epoch counter
        cudaError_t e = cudaStreamWaitEvent(job.stream, job.grads, 0);
        if (e != cudaSuccess) rc = set_err(CARAMEL_ECUDA, "cudaStreamWaitEvent: %s", cudaGetErrorString(e));
        for (size_t i = 0; !rc && i < job.buckets.size(); ++i) rc = launch(c, &job.buckets[i], 0, job.stream);
      }
    }
    if (!rc && job.done) {
      cudaError_t e = cudaEventRecord(job.done, job.stream);
      if (e != cudaSuccess) rc = set_err(CARAMEL_ECUDA, "cudaEventRecord(done): %s", cudaGetErrorString(e));
    }
    lk.lock();
    if (rc && !c->ce_rc) {
      c->ce_rc = rc;
      snprintf(c->ce_err, sizeof(c->ce_err), "%s", caramel_last_error());
    }
    ++c->ce_consumed;
    c->ce_busy = false;
    c->ce_cv.notify_all();
  }
}

int caramel_ce_submit(caramel_ctx* c, const caramel_bucket* host, int32_t count, uint32_t index0, uint32_t epoch,
                      int32_t engine, void* grad_stream, void* stream, void* done_event) {
  if (engine != CARAMEL_ENGINE_CE && engine != CARAMEL_ENGINE_SM && engine != CARAMEL_ENGINE_GATED)
    return set_err(CARAMEL_EINVAL, "ce_submit: unknown engine %d", engine);
  int rc = 0;
  if (engine != CARAMEL_ENGINE_SM) {
    rc = ce_validate(c, host, count, epoch, engine != CARAMEL_ENGINE_GATED);
  } else {
    if (!c || !host || count < 1) return set_err(CARAMEL_EINVAL, "ce_submit: null argument or empty list");
    if (!c->imported) return set_err(CARAMEL_ESTATE, "peer arenas not mapped (call caramel_import)");
    for (int i = 0; i < count && !rc; ++i) rc = validate_bucket(c, &host[i]);
  }
  if (rc) return rc;
  std::unique_lock<std::mutex> lk(c->ce_mu);
  if (c->ce_rc) return set_err(c->ce_rc, "%s", c->ce_err);
  if (!c->ce_worker_started) {
    for (int i = 0; i < CE_POOL; ++i) CUDA_TRY(cudaEventCreateWithFlags(&c->ce_pool[i], cudaEventDisableTiming));
    c->ce_worker = std::thread(ce_worker_main, c);
    c->ce_worker_started = true;
  }
  // an event is reusable once the worker has issued the waits on it
  c->ce_cv.wait(lk, [&] { return c->ce_submitted - c->ce_consumed < CE_POOL; });
  cudaEvent_t ev = c->ce_pool[c->ce_submitted % CE_POOL];
  cudaStream_t s = (cudaStream_t)stream;
  CUDA_TRY(cudaEventRecord(ev, grad_stream ? (cudaStream_t)grad_stream : s));  // in the caller's stream order
  CeJob job;
  job.buckets.assign(host, host + count);
  job.engine = engine;
  job.index0 = index0;
  job.epoch = epoch;
  job.grads = ev;
  job.stream = s;
  job.done = (cudaEvent_t)done_event;
  c->ce_jobs.push_back(std::move(job));
  ++c->ce_submitted;
  c->ce_cv.notify_all();
  return 0;
}

int caramel_ce_flush(caramel_ctx* c) {
  if (!c) return set_err(CARAMEL_EINVAL, "null ctx");
  std::unique_lock<std::mutex> lk(c->ce_mu);
  c->ce_cv.wait(lk, [&] { return c->ce_jobs.empty() && !c->ce_busy; });
  if (c->ce_rc) {
    const int rc = c->ce_rc;
    c->ce_rc = 0;
    return set_err(rc, "%s", c->ce_err);
  }
  return 0;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// NVLS multicast arena: driver entry points, handle exchange, bind, launch.
// ---------------------------------------------------------------------------
struct McApi {
  CUresult (*DeviceGet)(CUdevice*, int);
  CUresult (*DeviceGetAttribute)(int*, CUdevice_attribute, CUdevice);
  CUresult (*MulticastGetGranularity)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags);
  CUresult (*MulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*);
  CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice);
  CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                               unsigned long long);
  CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t);
  CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
  CUresult (*MemRelease)(CUmemGenericAllocationHandle);
  CUresult (*MemExportToShareableHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                         unsigned long long);
  CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType);
  CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  CUresult (*MemAddressFree)(CUdeviceptr, size_t);
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  CUresult (*MemUnmap)(CUdeviceptr, size_t);
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  CUresult (*MemGetAllocationGranularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
};
static McApi g_mc;

static bool mc_load() {
  static int state = 0;
  if (state) return state > 0;
  state = -1;
  struct { const char* name; void** slot; } fns[] = {
      {"cuDeviceGet", (void**)&g_mc.DeviceGet},
      {"cuDeviceGetAttribute", (void**)&g_mc.DeviceGetAttribute},
      {"cuMulticastGetGranularity", (void**)&g_mc.MulticastGetGranularity},
      {"cuMulticastCreate", (void**)&g_mc.MulticastCreate},
      {"cuMulticastAddDevice", (void**)&g_mc.MulticastAddDevice},
      {"cuMulticastBindMem", (void**)&g_mc.MulticastBindMem},
      {"cuMulticastUnbind", (void**)&g_mc.MulticastUnbind},
      {"cuMemCreate", (void**)&g_mc.MemCreate},
      {"cuMemRelease", (void**)&g_mc.MemRelease},
      {"cuMemExportToShareableHandle", (void**)&g_mc.MemExportToShareableHandle},
      {"cuMemImportFromShareableHandle", (void**)&g_mc.MemImportFromShareableHandle},
      {"cuMemAddressReserve", (void**)&g_mc.MemAddressReserve},
      {"cuMemAddressFree", (void**)&g_mc.MemAddressFree},
      {"cuMemMap", (void**)&g_mc.MemMap},
      {"cuMemUnmap", (void**)&g_mc.MemUnmap},
      {"cuMemSetAccess", (void**)&g_mc.MemSetAccess},
      {"cuMemGetAllocationGranularity", (void**)&g_mc.MemGetAllocationGranularity},
  };
  for (auto& f : fns) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(f.name, f.slot, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !*f.slot)
      return false;
  }
  state = 1;
  return true;
}

#define MC_TRY(expr)                                                                              \
  do {                                                                                            \
    CUresult _r = (expr);                                                                         \
    if (_r != CUDA_SUCCESS) return set_err(CARAMEL_ECUDA, "%s failed: CUresult %d", #expr, (int)_r); \
  } while (0)

static int mc_socket_name(const char* token, int rank, sockaddr_un* a, socklen_t* len) {
  memset(a, 0, sizeof(*a));
  a->sun_family = AF_UNIX;
  // abstract namespace: no file in the filesystem, gone with the process
  const int n = snprintf(a->sun_path + 1, sizeof(a->sun_path) - 1, "caramel-mc-%s-%d", token, rank);
  if (n <= 0 || n >= (int)sizeof(a->sun_path) - 1) return -1;
  *len = (socklen_t)(offsetof(sockaddr_un, sun_path) + 1 + n);
  return 0;
}

static int mc_send_fd(int sock, int fd) {
  char byte = 'm';
  iovec io{&byte, 1};
  char ctl[CMSG_SPACE(sizeof(int))];
  memset(ctl, 0, sizeof(ctl));
  msghdr msg;
  memset(&msg, 0, sizeof(msg));
  msg.msg_iov = &io;
  msg.msg_iovlen = 1;
  msg.msg_control = ctl;
  msg.msg_controllen = sizeof(ctl);
  cmsghdr* cm = CMSG_FIRSTHDR(&msg);
  cm->cmsg_level = SOL_SOCKET;
  cm->cmsg_type = SCM_RIGHTS;
  cm->cmsg_len = CMSG_LEN(sizeof(int));
  memcpy(CMSG_DATA(cm), &fd, sizeof(int));
  return sendmsg(sock, &msg, 0) == 1 ? 0 : -1;
}

static int mc_recv_fd(int sock) {
  char byte;
  iovec io{&byte, 1};
  char ctl[CMSG_SPACE(sizeof(int))];
  msghdr msg;
  memset(&msg, 0, sizeof(msg));
  msg.msg_iov = &io;
  msg.msg_iovlen = 1;
  msg.msg_control = ctl;
  msg.msg_controllen = sizeof(ctl);
  if (recvmsg(sock, &msg, 0) != 1) return -1;
  cmsghdr* cm = CMSG_FIRSTHDR(&msg);
  if (!cm || cm->cmsg_type != SCM_RIGHTS) return -1;
  int fd;
  memcpy(&fd, CMSG_DATA(cm), sizeof(int));
  return fd;
}

extern "C" {

int caramel_mc_available(caramel_ctx* c) {
  if (!c || c->nlocal != 1 || c->world < 2 || !mc_load()) return 0;
  CUdevice d;
  int v = 0;
  if (g_mc.DeviceGet(&d, c->device) != CUDA_SUCCESS) return 0;
  if (g_mc.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d) != CUDA_SUCCESS) return 0;
  return v ? 1 : 0;
}

int caramel_mc_create(caramel_ctx* c, uint64_t bytes, const char* token) {
  if (!c || !token || !bytes) return set_err(CARAMEL_EINVAL, "mc_create: null argument");
  if (c->mc_state) return set_err(CARAMEL_ESTATE, "mc_create: the multicast arena exists already");
  if (!caramel_mc_available(c)) return set_err(CARAMEL_ESTATE, "mc_create: no multicast (NVLS) support here");
  CUdevice dev;
  MC_TRY(g_mc.DeviceGet(&dev, c->device));
  CUmulticastObjectProp mp;
  memset(&mp, 0, sizeof(mp));
  mp.numDevices = (unsigned)c->world;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = bytes;
  size_t mg = 0;
  MC_TRY(g_mc.MulticastGetGranularity(&mg, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = dev;
  ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t ag = 0;
  MC_TRY(g_mc.MemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const uint64_t gran = mg > ag ? mg : ag;
  c->mc_gran = gran;
  c->mc_bytes = (bytes + gran - 1) / gran * gran;
  mp.size = c->mc_bytes;
  CUmemGenericAllocationHandle mem;
  MC_TRY(g_mc.MemCreate(&mem, c->mc_bytes, &ap, 0));
  c->mc_mem = mem;
  c->mc_listen = -1;
  c->mc_fd = -1;
  snprintf(c->mc_name, sizeof(c->mc_name), "%s", token);
  if (c->rank == 0) {
    CUmemGenericAllocationHandle mc;
    MC_TRY(g_mc.MulticastCreate(&mc, &mp));
    c->mc_handle = mc;
    int fd = -1;
    MC_TRY(g_mc.MemExportToShareableHandle(&fd, mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    c->mc_fd = fd;
    sockaddr_un a;
    socklen_t len;
    if (mc_socket_name(token, 0, &a, &len)) return set_err(CARAMEL_EINVAL, "mc_create: token too long");
    const int s = socket(AF_UNIX, SOCK_STREAM, 0);
    if (s < 0 || bind(s, (sockaddr*)&a, len) || listen(s, c->world))
      return set_err(CARAMEL_ECUDA, "mc_create: listening socket: %s", strerror(errno));
    c->mc_listen = s;
  }
  c->mc_state = 1;
  return 0;
}

int caramel_mc_exchange(caramel_ctx* c) {
  if (!c || c->mc_state != 1) return set_err(CARAMEL_ESTATE, "mc_exchange: call caramel_mc_create first");
  if (c->rank == 0) {
    for (int i = 1; i < c->world; ++i) {
      const int s = accept(c->mc_listen, nullptr, nullptr);
      if (s < 0) return set_err(CARAMEL_ECUDA, "mc_exchange: accept: %s", strerror(errno));
      const int rc = mc_send_fd(s, c->mc_fd);
      close(s);
      if (rc) return set_err(CARAMEL_ECUDA, "mc_exchange: sending the handle: %s", strerror(errno));
    }
    close(c->mc_listen);
    c->mc_listen = -1;
  } else {
    sockaddr_un a;
    socklen_t len;
    mc_socket_name(c->mc_name, 0, &a, &len);
    int s = -1;
    for (int tries = 0; tries < 600; ++tries) {  // rank 0 listens before the caller's barrier; retry briefly anyway
      s = socket(AF_UNIX, SOCK_STREAM, 0);
      if (s >= 0 && connect(s, (sockaddr*)&a, len) == 0) break;
      if (s >= 0) close(s);
      s = -1;
      usleep(10000);
    }
    if (s < 0) return set_err(CARAMEL_ECUDA, "mc_exchange: cannot reach rank 0's socket");
    const int fd = mc_recv_fd(s);
    close(s);
    if (fd < 0) return set_err(CARAMEL_ECUDA, "mc_exchange: no handle received");
    c->mc_fd = fd;
    CUmemGenericAllocationHandle mc;
    MC_TRY(g_mc.MemImportFromShareableHandle(&mc, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
    c->mc_handle = mc;
  }
  CUdevice dev;
  MC_TRY(g_mc.DeviceGet(&dev, c->device));
  MC_TRY(g_mc.MulticastAddDevice(c->mc_handle, dev));
  c->mc_state = 2;
  return 0;
}

int caramel_mc_bind(caramel_ctx* c, uint64_t* unicast) {
  if (!c || c->mc_state != 2) return set_err(CARAMEL_ESTATE, "mc_bind: call caramel_mc_exchange first (every rank)");
  CUdevice dev;
  MC_TRY(g_mc.DeviceGet(&dev, c->device));
  MC_TRY(g_mc.MulticastBindMem(c->mc_handle, 0, c->mc_mem, 0, c->mc_bytes, 0));
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr mva = 0, uva = 0;
  MC_TRY(g_mc.MemAddressReserve(&mva, c->mc_bytes, c->mc_gran, 0, 0));
  MC_TRY(g_mc.MemMap(mva, c->mc_bytes, 0, c->mc_handle, 0));
  MC_TRY(g_mc.MemSetAccess(mva, c->mc_bytes, &acc, 1));
  MC_TRY(g_mc.MemAddressReserve(&uva, c->mc_bytes, c->mc_gran, 0, 0));
  MC_TRY(g_mc.MemMap(uva, c->mc_bytes, 0, c->mc_mem, 0));
  MC_TRY(g_mc.MemSetAccess(uva, c->mc_bytes, &acc, 1));
  c->mc_va = mva;
  c->uc_va = uva;
  CUDA_TRY(cudaMemset((void*)uva, 0, c->mc_bytes));
  CUDA_TRY(cudaDeviceSynchronize());
  if (unicast) *unicast = uva;
  c->mc_state = 3;
  return 0;
}

int caramel_allreduce_nvls(caramel_ctx* c, const caramel_bucket* b, uint32_t epoch, void* stream) {
  if (!c || !b) return set_err(CARAMEL_EINVAL, "allreduce_nvls: null argument");
  if (c->mc_state != 3) return set_err(CARAMEL_ESTATE, "allreduce_nvls: no bound multicast arena (caramel_mc_bind)");
  if (b->numel == 0) return 0;
  if (b->depth < 1 || b->depth > CARAMEL_MAX_DEPTH || b->ctas < 1)
    return set_err(CARAMEL_EINVAL, "allreduce_nvls: bad depth or ctas");
  if ((b->bucket_off & 15) || b->bucket_off + 4 * b->numel > c->mc_bytes)
    return set_err(CARAMEL_EINVAL, "allreduce_nvls: bucket outside the multicast arena or misaligned");
  if (b->epilogue == CARAMEL_EPI_SGD &&
      (!c->param_bytes || (b->param_off & 15) || b->param_off + 4 * b->numel > c->param_bytes))
    return set_err(CARAMEL_EINVAL, "allreduce_nvls: the SGD epilogue needs the parameter arena");
  const uint64_t fb = (uint64_t)b->depth * b->ctas * 2 * c->world * 4;
  if ((b->flag_off & 3) || b->flag_off + fb > c->arena_bytes)
    return set_err(CARAMEL_EINVAL, "allreduce_nvls: flag block outside the IPC arena");
  if (!c->imported) return set_err(CARAMEL_ESTATE, "peer arenas not mapped (call caramel_import)");
  NvlsParams P;
  memset(&P, 0, sizeof(P));
  fill_env(c, P.env, epoch);
  P.b = *b;
  P.mc = c->mc_va;
  P.uc = c->uc_va;
  static int probe = -1;
  if (probe < 0) probe = getenv("CARAMEL_NVLS_PROBE") ? atoi(getenv("CARAMEL_NVLS_PROBE")) : 0;
  P.probe = probe;
  k_nvls<<<b->ctas, THREADS, 0, (cudaStream_t)stream>>>(P);
  CUDA_TRY(cudaGetLastError());
  return 0;
}

static void mc_release(caramel_ctx* c) {
  if (!c->mc_state || !mc_load()) return;
  CUdevice dev;
  g_mc.DeviceGet(&dev, c->device);
  if (c->mc_va) { g_mc.MemUnmap(c->mc_va, c->mc_bytes); g_mc.MemAddressFree(c->mc_va, c->mc_bytes); }
  if (c->uc_va) { g_mc.MemUnmap(c->uc_va, c->mc_bytes); g_mc.MemAddressFree(c->uc_va, c->mc_bytes); }
  if (c->mc_state == 3) g_mc.MulticastUnbind(c->mc_handle, dev, 0, c->mc_bytes);
  if (c->mc_handle) g_mc.MemRelease(c->mc_handle);
  if (c->mc_mem) g_mc.MemRelease(c->mc_mem);
  if (c->mc_listen >= 0) close(c->mc_listen);
  if (c->mc_fd >= 0) close(c->mc_fd);
  c->mc_state = 0;
}

}  // extern "C"
