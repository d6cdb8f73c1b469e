// Distributed-shared-memory probe: could a thread-block cluster hold one coarse
// region (C CTAs x 128 KiB) and answer every record of a coarse bin by remote
// bucket operations, so the split pass (coarse bin -> fine bins) disappears?
// Measures, per cluster size C in {1, 2, 4, 8, 16}, at the probe's shape (one
// CTA per SM, 768 worker threads, a 128 KiB table slice per CTA):
//   load  : one random 32 B bucket read (two ld.shared::cluster.v2.u64)
//   cas   : 32 B bucket read + one 64-bit CAS on a word of it (the insert op)
// with the bucket drawn uniformly over the whole cluster region (a fraction
// 1/C is local), and the number of co-resident clusters the hardware grants
// (cudaOccupancyMaxActiveClusters).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_dsmem tools/probe_dsmem.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kThreads = 768;
constexpr uint32_t kSlice = 128 * 1024;  // bytes of table per CTA
constexpr uint32_t kBuckets = kSlice / 32;

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_n() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int KIND>
__global__ void __launch_bounds__(kThreads, 1) dsmem_kernel(int iters, unsigned long long* sink) {
  extern __shared__ __align__(16) uint64_t slice[];
  for (uint32_t i = threadIdx.x; i < kSlice / 8; i += kThreads) slice[i] = i & 3;
  cluster_sync();
  const uint32_t C = cluster_n();
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(slice);
  // remote base address of every CTA's slice (mapa)
  uint32_t rbase[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) {
    uint32_t a = base;
    if (r < (int)C) asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(base), "r"(r));
    rbase[r] = a;
  }
  const uint64_t tid = blockIdx.x * (uint64_t)kThreads + threadIdx.x;
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    const uint64_t h = mix(tid * 0x9E3779B97F4A7C15ull + it);
    const uint32_t owner = (uint32_t)(h >> 40) % C;
    uint32_t ob = rbase[0];
#pragma unroll
    for (int r = 1; r < 16; ++r) ob = owner == (uint32_t)r ? rbase[r] : ob;
    const uint32_t a = ob + ((uint32_t)h % kBuckets) * 32u;
    uint64_t w0, w1, w2, w3;
    asm volatile("ld.shared::cluster.v2.u64 {%0,%1}, [%2];" : "=l"(w0), "=l"(w1) : "r"(a));
    asm volatile("ld.shared::cluster.v2.u64 {%0,%1}, [%2];" : "=l"(w2), "=l"(w3) : "r"(a + 16));
    if (KIND == 0) {
      acc += w0 ^ w1 ^ w2 ^ w3;
    } else {
      const uint32_t j = (uint32_t)(w0 + w3) & 3u;
      const uint64_t cmp = j == 0 ? w0 : j == 1 ? w1 : j == 2 ? w2 : w3;
      uint64_t old;
      asm volatile("atom.shared::cluster.cas.b64 %0, [%1], %2, %3;"
                   : "=l"(old) : "r"(a + 8 * j), "l"(cmp), "l"(cmp + 4) : "memory");
      acc += old;
    }
  }
  cluster_sync();  // no CTA leaves while others may still address its slice
  if (acc == 0x1234567) sink[0] = acc;
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int KIND>
static int run(int C, int nsm, unsigned long long* sink, const char* name) {
  auto k = dsmem_kernel<KIND>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSlice));
  if (C > 8) CK(cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSlice;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cfg.gridDim = dim3(C);
  int active = 0;
  CK(cudaOccupancyMaxActiveClusters(&active, (void*)k, &cfg));
  if (active <= 0) {
    printf("cluster %2d %-5s: cannot be resident\n", C, name);
    return 0;
  }
  cfg.gridDim = dim3(active * C);  // one wave: every cluster co-resident
  const int iters = 4096;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaLaunchKernelEx(&cfg, k, iters, sink));  // warm-up
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaEventRecord(e0));
    CK(cudaLaunchKernelEx(&cfg, k, iters, sink));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    best = ms < best ? ms : best;
  }
  const double ops = (double)active * C * kThreads * iters;
  printf("cluster %2d %-5s: %3d clusters (%3d of %d SMs)  %7.1f G bucket ops/s  (%6.1f G/s per active SM)\n", C, name,
         active, active * C, nsm, ops / best / 1e6, ops / best / 1e6 / (active * C));
  return 0;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  printf("%s, %d SMs\n", p.name, p.multiProcessorCount);
  for (int C : {1, 2, 4, 8, 16}) {
    if (run<0>(C, p.multiProcessorCount, sink, "load")) return 1;
    if (run<1>(C, p.multiProcessorCount, sink, "cas")) return 1;
  }
  return 0;
}
