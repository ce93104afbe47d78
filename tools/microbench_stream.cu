// Microbenchmark: theta -= lr * (g * scale) over N fp32 elements (the world=1
// fused update), in several code shapes, to pick the loop structure used in
// caramel.cu's stream_epi.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench_stream.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ float upd(float g, float t) {
  return __fsub_rn(t, __fmul_rn(0.1f, __fmul_rn(g, 0.5f)));
}

enum { LD_DEFAULT = 0, LD_CS_CG = 1, LD_NC = 2 };

template <int U, int MODE>
__global__ void k_tile(const float4* __restrict__ g, float4* th, uint64_t nv, int tiles) {
  // contiguous tile per CTA (what caramel does)
  uint64_t per = (nv + tiles - 1) / tiles;
  uint64_t lo = per * blockIdx.x, hi = lo + per < nv ? lo + per : nv;
  const uint64_t T = blockDim.x;
  uint64_t v = lo + threadIdx.x;
  for (; v + (U - 1) * T < hi; v += U * T) {
    float4 x[U], t[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = MODE == LD_CS_CG ? __ldcs(g + v + u * T) : MODE == LD_NC ? __ldg(g + v + u * T) : g[v + u * T];
#pragma unroll
    for (int u = 0; u < U; ++u) t[u] = MODE == LD_CS_CG ? __ldcg(th + v + u * T) : th[v + u * T];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float4 o = make_float4(upd(x[u].x, t[u].x), upd(x[u].y, t[u].y), upd(x[u].z, t[u].z), upd(x[u].w, t[u].w));
      if (MODE == LD_CS_CG) __stcg(th + v + u * T, o); else th[v + u * T] = o;
    }
  }
  for (; v < hi; v += T) {
    float4 x = g[v], t = th[v];
    th[v] = make_float4(upd(x.x, t.x), upd(x.y, t.y), upd(x.z, t.z), upd(x.w, t.w));
  }
}

template <int U>
__global__ void k_gridstride(const float4* __restrict__ g, float4* th, uint64_t nv) {
  const uint64_t T = (uint64_t)blockDim.x * gridDim.x;
  uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; v + (U - 1) * T < nv; v += U * T) {
    float4 x[U], t[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = g[v + u * T];
#pragma unroll
    for (int u = 0; u < U; ++u) t[u] = th[v + u * T];
#pragma unroll
    for (int u = 0; u < U; ++u)
      th[v + u * T] = make_float4(upd(x[u].x, t[u].x), upd(x[u].y, t[u].y), upd(x[u].z, t[u].z), upd(x[u].w, t[u].w));
  }
  for (; v < nv; v += T) {
    float4 x = g[v], t = th[v];
    th[v] = make_float4(upd(x.x, t.x), upd(x.y, t.y), upd(x.z, t.z), upd(x.w, t.w));
  }
}

template <class F>
float timeit(F f, int reps = 20) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  const uint64_t n = 25557032;  // resnet50
  const uint64_t nv = n / 4;
  float4 *g, *th;
  cudaMalloc(&g, nv * 16);
  cudaMalloc(&th, nv * 16);
  cudaMemset(g, 0, nv * 16);
  cudaMemset(th, 0, nv * 16);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const double bytes = 12.0 * n;
  auto rep = [&](const char* name, float ms) { printf("%-40s %8.1f us  %7.0f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9); };
  char name[128];
  for (int threads : {256, 512, 1024}) {
    for (int tiles_per_sm : {2, 4, 8, 16}) {
      int tiles = sms * tiles_per_sm;
      snprintf(name, sizeof name, "tile U4 default t%d tiles/sm%d", threads, tiles_per_sm);
      rep(name, timeit([&] { k_tile<4, LD_DEFAULT><<<tiles, threads>>>(g, th, nv, tiles); }));
    }
  }
  for (int tiles_per_sm : {4, 8}) {
    int tiles = sms * tiles_per_sm;
    snprintf(name, sizeof name, "tile U4 cs/cg t512 tiles/sm%d", tiles_per_sm);
    rep(name, timeit([&] { k_tile<4, LD_CS_CG><<<tiles, 512>>>(g, th, nv, tiles); }));
    snprintf(name, sizeof name, "tile U4 nc t512 tiles/sm%d", tiles_per_sm);
    rep(name, timeit([&] { k_tile<4, LD_NC><<<tiles, 512>>>(g, th, nv, tiles); }));
    snprintf(name, sizeof name, "tile U2 default t512 tiles/sm%d", tiles_per_sm);
    rep(name, timeit([&] { k_tile<2, LD_DEFAULT><<<tiles, 512>>>(g, th, nv, tiles); }));
    snprintf(name, sizeof name, "tile U8 default t512 tiles/sm%d", tiles_per_sm);
    rep(name, timeit([&] { k_tile<8, LD_DEFAULT><<<tiles, 512>>>(g, th, nv, tiles); }));
  }
  for (int bpsm : {1, 2, 4, 8}) {
    snprintf(name, sizeof name, "gridstride U4 t256 blocks/sm%d", bpsm);
    rep(name, timeit([&] { k_gridstride<4><<<sms * bpsm, 256>>>(g, th, nv); }));
    snprintf(name, sizeof name, "gridstride U2 t512 blocks/sm%d", bpsm);
    rep(name, timeit([&] { k_gridstride<2><<<sms * bpsm, 512>>>(g, th, nv); }));
  }
  // many-times-larger problem for reference (L2 out of the picture)
  return 0;
}
