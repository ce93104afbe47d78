// NVLink data-movement microbenchmark (one process, two GPUs, peer access):
// how fast can SM-issued traffic cross NVLink 5 in each of the four ways a
// collective kernel can move bytes -- pull (peer loads) or push (peer stores),
// each from registers (LDG/STG.128) or staged through shared memory by the
// TMA bulk-copy unit (cp.async.bulk, UBLKCP) -- at 8..148 CTAs, with both
// GPUs moving bytes at once (both directions busy, as in an all-reduce).
// Prints one JSON line per case.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_nvlink mb_nvlink.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// registers: each thread moves U float4 per trip, all loads before the stores
template <int U>
__global__ void __launch_bounds__(512) k_copy_reg(const float4* __restrict__ src, float4* __restrict__ dst, size_t n4) {
  const size_t T = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * T < n4; i += U * T) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcg(src + i + u * T);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcg(dst + i + u * T, v[u]);
  }
  for (; i < n4; i += T) __stcg(dst + i, __ldcg(src + i));
}

// TMA: tiles of TB bytes, S stages; one elected thread drives the pipeline:
// bulk load src -> smem (mbarrier completion), bulk store smem -> dst
template <int TB, int S>
__global__ void __launch_bounds__(32) k_copy_tma(const char* __restrict__ src, char* __restrict__ dst, size_t bytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)S * TB);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < S; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t tiles = bytes / TB;
  const size_t G = gridDim.x;
  const size_t K = blockIdx.x < tiles ? (tiles - blockIdx.x + G - 1) / G : 0;
  auto issue = [&](size_t k) {
    const int s = (int)(k % S);
    const size_t off = (blockIdx.x + k * G) * (size_t)TB;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(TB) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sm + (size_t)s * TB)), "l"(src + off), "r"(TB), "r"(smem_u32(&bar[s]))
                 : "memory");
  };
  for (size_t k = 0; k + 1 < S && k < K; ++k) issue(k);
  for (size_t k = 0; k < K; ++k) {
    const int s = (int)(k % S);
    asm volatile(
        "{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n}" ::"r"(
            smem_u32(&bar[s])), "r"((uint32_t)((k / S) & 1)) : "memory");
    const size_t off = (blockIdx.x + k * G) * (size_t)TB;
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off), "r"(smem_u32(sm + (size_t)s * TB)),
                 "r"(TB) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // stage (k+S-1)%S == (k-1)%S held tile k-1: its store must be done reading smem
    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    if (k + S - 1 < K) issue(k + S - 1);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { printf("{\"error\": \"needs 2 GPUs\"}\n"); return 0; }
  const size_t maxb = 256ull << 20;
  char *loc[2], *rem[2];  // loc[d]: source on device d; rem[d]: destination on device d
  cudaStream_t st[2];
  cudaEvent_t e0[2], e1[2];
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceEnablePeerAccess(1 - d, 0));
    CK(cudaMalloc(&loc[d], maxb));
    CK(cudaMalloc(&rem[d], maxb));
    CK(cudaMemset(loc[d], 1, maxb));
    CK(cudaStreamCreateWithFlags(&st[d], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[d]));
    CK(cudaEventCreate(&e1[d]));
  }
  constexpr int TB = 32768, S = 4;
  const size_t smem = (size_t)S * TB + 64 * S;
  for (int d = 0; d < 2; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaFuncSetAttribute(k_copy_tma<TB, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  const char* modes[4] = {"pull_reg", "push_reg", "pull_tma", "push_tma"};
  const int grids[6] = {8, 16, 32, 64, 128, 148};
  const size_t sizes[3] = {4ull << 20, 64ull << 20, 256ull << 20};
  for (int both = 1; both >= 0; --both)
    for (size_t bytes : sizes)
      for (int m = 0; m < 4; ++m)
        for (int g : grids) {
          float best = 1e30f;
          for (int rep = 0; rep < 6; ++rep) {
            for (int d = 0; d < 2; ++d) {
              if (!both && d == 1) continue;
              CK(cudaSetDevice(d));
              // pull: my kernel reads the peer's buffer into mine; push: writes mine into the peer's
              const char* src = (m == 0 || m == 2) ? loc[1 - d] : loc[d];
              char* dst = (m == 0 || m == 2) ? rem[d] : rem[1 - d];
              CK(cudaEventRecord(e0[d], st[d]));
              if (m < 2)
                k_copy_reg<4><<<g, 512, 0, st[d]>>>((const float4*)src, (float4*)dst, bytes / 16);
              else
                k_copy_tma<TB, S><<<g, 32, smem, st[d]>>>(src, dst, bytes);
              CK(cudaEventRecord(e1[d], st[d]));
            }
            float worst = 0;
            for (int d = 0; d < 2; ++d) {
              if (!both && d == 1) continue;
              CK(cudaSetDevice(d));
              CK(cudaEventSynchronize(e1[d]));
              float ms = 0;
              CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
              worst = ms > worst ? ms : worst;
            }
            if (rep > 0 && worst < best) best = worst;
          }
          printf("{\"mode\": \"%s\", \"both_directions\": %d, \"bytes\": %zu, \"ctas\": %d, \"us\": %.2f, \"gbs\": %.1f}\n",
                 modes[m], both, bytes, g, best * 1e3, bytes / (best * 1e-3) / 1e9);
          fflush(stdout);
        }
  return 0;
}
