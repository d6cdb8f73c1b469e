// DRAM fetch granularity probe (round 2): random 32 B bucket reads over a
// 512 MiB table with the load flavours the kernels use.  Run under
//   ncu --metrics gpu__time_duration.sum,dram__sectors_read.sum,lts__t_sectors_srcunit_tex_op_read.sum
// to see how many DRAM sectors each requested sector costs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_fetch tools/probe_fetch.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// MODE 0: ld.global.nc.L1::no_allocate.v4   1: ld.relaxed.gpu.global.v4
//      2: ld.global.cg.v4                     3: ld.global.v4 (default .ca)
//      4: ld.global.nc.v4 + L2::evict_first   5: 8 B ld.global.nc (one word)
//      6: atom.cas.b64 on one word             7: ld.relaxed.gpu + cas on the same sector
template <int MODE>
__global__ void __launch_bounds__(256) gather(uint64_t* buf, uint64_t nsect, int iters, uint64_t* sink) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint64_t idx[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) idx[u] = mix(tid * 0x9E3779B97F4A7C15ull + it * 4 + u) & (nsect - 1);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      uint64_t* p = buf + idx[u] * 4;
      uint64_t a = 0, b = 0, c = 0, d = 0;
      if (MODE == 0) asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
      if (MODE == 1) asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p) : "memory");
      if (MODE == 2) asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
      if (MODE == 3) asm volatile("ld.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
      if (MODE == 4) asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
      if (MODE == 5) asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(a) : "l"(p));
      if (MODE == 6) a = atomicCAS((unsigned long long*)p, 1ull, 2ull);
      if (MODE == 7) {
        asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p) : "memory");
        atomicCAS((unsigned long long*)p + (a & 3), b, c);
      }
      acc ^= a ^ b ^ c ^ d;
    }
  }
  if (acc == 0x1234567) sink[0] = acc;
}

// MODE 8: TMA 1-D bulk copies of one 32 B bucket into shared memory (4 in flight per thread)
__global__ void __launch_bounds__(256) gather_tma(const uint64_t* buf, uint64_t nsect, int iters, uint64_t* sink) {
  __shared__ __align__(128) uint64_t dst[256 * 4 * 4];
  __shared__ __align__(8) uint64_t bar[256 * 4];
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&bar[threadIdx.x * 4]);
  uint32_t d0 = (uint32_t)__cvta_generic_to_shared(&dst[threadIdx.x * 16]);
  for (int u = 0; u < 4; ++u) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0 + 8 * u));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint64_t acc = 0;
  uint32_t par = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t idx = mix(tid * 0x9E3779B97F4A7C15ull + it * 4 + u) & (nsect - 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 32;" ::"r"(b0 + 8 * u) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 32, [%2];"
                   ::"r"(d0 + 32 * u), "l"(buf + idx * 4), "r"(b0 + 8 * u) : "memory");
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}\n"
                   ::"r"(b0 + 8 * u), "r"(par) : "memory");
      acc ^= dst[threadIdx.x * 16 + 4 * u];
    }
    par ^= 1;
  }
  if (acc == 0x1234567) sink[0] = acc;
}

int main() {
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const uint64_t ws = 512ull << 20;
  uint64_t* buf;
  CK(cudaMalloc(&buf, ws));
  CK(cudaMemset(buf, 0x5a, ws));
  uint64_t* sink;
  CK(cudaMalloc(&sink, 64));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = nsm * 8, block = 256, iters = 16;
  const double acc = (double)grid * block * iters * 4;
  for (int gran : {0, 32, 128}) {
    if (gran) CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran));
    size_t gg = 0;
    cudaDeviceGetLimit(&gg, cudaLimitMaxL2FetchGranularity);
#define RUN(M)                                                                                    \
  {                                                                                               \
    gather<M><<<grid, block>>>(buf, ws / 32, iters, sink);                                        \
    CK(cudaEventRecord(e0));                                                                      \
    for (int r = 0; r < 3; ++r) gather<M><<<grid, block>>>(buf, ws / 32, iters, sink);            \
    CK(cudaEventRecord(e1));                                                                      \
    CK(cudaEventSynchronize(e1));                                                                 \
    float ms;                                                                                     \
    cudaEventElapsedTime(&ms, e0, e1);                                                            \
    printf("gran=%zu mode=%d: %.2f G accesses/s (%.0f accesses per launch)\n", gg, M, 3 * acc / (ms * 1e6), acc); \
  }
    RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7)
    {
      gather_tma<<<grid, block>>>(buf, ws / 32, iters, sink);
      CK(cudaEventRecord(e0));
      for (int r = 0; r < 3; ++r) gather_tma<<<grid, block>>>(buf, ws / 32, iters, sink);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("gran=%zu mode=tma: %.2f G accesses/s\n", gg, 3 * acc / (ms * 1e6));
    }
  }
  CK(cudaGetLastError());
  return 0;
}
