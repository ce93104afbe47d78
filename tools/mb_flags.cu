// Inter-GPU flag latency microbenchmark (one process, two GPUs, peer access).
// GPU0 and GPU1 ping-pong a counter through flags in each other's memory,
// optionally preceded by a block of remote data stores.  Reports one-way
// latency per variant.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_flags mb_flags.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

enum { V_REL_ACQ = 0, V_VOLATILE = 1, V_RELAXED_FENCE = 2, V_REL_ACQ_GPU = 3 };

template <int V>
__device__ __forceinline__ void put(uint32_t* p, uint32_t v) {
  if (V == V_REL_ACQ) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else if (V == V_VOLATILE) { __threadfence_system(); *(volatile uint32_t*)p = v; }
  else if (V == V_RELAXED_FENCE) { asm volatile("fence.acq_rel.sys;" ::: "memory"); asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory"); }
  else asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int V>
__device__ __forceinline__ uint32_t get(const uint32_t* p) {
  uint32_t v;
  if (V == V_REL_ACQ) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else if (V == V_VOLATILE) v = *(const volatile uint32_t*)p;
  else if (V == V_RELAXED_FENCE) asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// me: 0 or 1.  my_flag is local; peer_flag/peer_data live on the other GPU.
template <int V>
__global__ void pingpong(uint32_t* my_flag, uint32_t* peer_flag, float* peer_data, int iters, int data_words,
                         unsigned long long* out_ns, int me) {
  __shared__ int dummy;
  unsigned long long t0 = 0;
  if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 1; i <= iters; ++i) {
    const bool my_turn_send = (me == 0);
    // me==0: send i, wait i ; me==1: wait i, send i
    if (!my_turn_send) {
      if (threadIdx.x == 0) while (get<V>(my_flag) < (uint32_t)i) {}
      __syncthreads();
    }
    for (int w = threadIdx.x; w < data_words; w += blockDim.x) peer_data[w] = (float)i;
    __syncthreads();
    if (threadIdx.x == 0) put<V>(peer_flag, (uint32_t)i);
    if (my_turn_send) {
      if (threadIdx.x == 0) while (get<V>(my_flag) < (uint32_t)i) {}
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    *out_ns = t1 - t0;
  }
  dummy = 0;
}

template <int V>
int run(const char* name, uint32_t* f[2], float* d[2], unsigned long long* o[2], int data_words) {
  const int iters = 2000;
  for (int g = 0; g < 2; ++g) { CK(cudaSetDevice(g)); CK(cudaMemset(f[g], 0, 4)); }
  for (int g = 0; g < 2; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); }
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    pingpong<V><<<1, 256>>>(f[g], f[1 - g], d[1 - g], iters, data_words, o[g], g);
  }
  for (int g = 0; g < 2; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); }
  unsigned long long ns;
  CK(cudaSetDevice(0));
  CK(cudaMemcpy(&ns, o[0], 8, cudaMemcpyDeviceToHost));
  printf("%-28s data %7d B: one-way %.2f us\n", name, data_words * 4, ns / 1e3 / (2.0 * iters));
  return 0;
}

int main() {
  uint32_t* f[2];
  float* d[2];
  unsigned long long* o[2];
  for (int g = 0; g < 2; ++g) {
    CK(cudaSetDevice(g));
    CK(cudaDeviceEnablePeerAccess(1 - g, 0));
    CK(cudaMalloc(&f[g], 256));
    CK(cudaMalloc(&d[g], 4 << 20));
    CK(cudaMalloc(&o[g], 8));
  }
  for (int dw : {0, 1024, 16384}) {
    run<V_REL_ACQ>("st.release/ld.acquire sys", f, d, o, dw);
    run<V_VOLATILE>("threadfence_system+volatile", f, d, o, dw);
    run<V_RELAXED_FENCE>("fence.acq_rel+relaxed sys", f, d, o, dw);
    run<V_REL_ACQ_GPU>("release/acquire gpu (WRONG)", f, d, o, dw);
  }
  return 0;
}
