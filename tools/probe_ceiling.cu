// Step-0 ceiling probe: what does B200 HBM3e deliver
// for the access pattern of the cuckoo-filter hot path?
//   - streaming copy (the MEASURED_PEAKS.json denominator, re-measured here)
//   - random 32 B sector gathers (one bucket at f=16,b=16) with U loads in flight
//   - random 64 B / 128 B gathers
//   - random 64-bit atomicCAS (the insert/delete commit primitive)
//   - random 32 B read followed by a CAS into the same sector (insert pattern)
// each at 512 MiB (2^28 slots, f=16) and 4 GiB (DRAM-only) working sets and
// with the default vs 32 B L2 fetch granularity.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_ceiling tools/probe_ceiling.cu
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

template <int U, int BYTES>
__global__ void __launch_bounds__(256) gather(const uint64_t* __restrict__ buf, uint64_t nunits,
                                              int iters, uint64_t* __restrict__ sink) {
  uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint64_t idx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) idx[u] = mix(tid * 0x9E3779B97F4A7C15ull + it * U + u) & (nunits - 1);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t* p = buf + idx[u] * (BYTES / 8);
#pragma unroll
      for (int s = 0; s < BYTES / 32; ++s) {
        uint64_t a, b, c, d;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                     : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p + 4 * s));
        acc ^= a ^ b ^ c ^ d;
      }
    }
  }
  if (acc == 0x1234567) sink[0] = acc;
}

template <int U>
__global__ void __launch_bounds__(256) rand_cas(unsigned long long* buf, uint64_t nwords, int iters) {
  uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      uint64_t i = mix(tid * 0x9E3779B97F4A7C15ull + it * U + u) & (nwords - 1);
      unsigned long long v = buf[i];
      atomicCAS(buf + i, v, v + 1);
    }
  }
}

// insert-like: 256-bit coherent read of a 32B sector, then CAS one word of it
__global__ void __launch_bounds__(256) read_cas(unsigned long long* buf, uint64_t nsect, int iters) {
  uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    uint64_t s = mix(tid * 0x9E3779B97F4A7C15ull + it) & (nsect - 1);
    unsigned long long* p = buf + s * 4;
    uint64_t a, b, c, d;
    asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    int w = (a ^ b ^ c ^ d) & 3;
    uint64_t old = w == 0 ? a : w == 1 ? b : w == 2 ? c : d;
    atomicCAS(p + w, old, old + 1);
  }
}

__global__ void copyk(const int4* __restrict__ a, int4* __restrict__ b, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

int main() {
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const uint64_t big = 4ull << 30;
  uint64_t* buf;
  CK(cudaMalloc(&buf, big));
  CK(cudaMemset(buf, 0x5a, big));
  uint64_t* sink;
  CK(cudaMalloc(&sink, 64));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  // copy: 2 GiB -> 2 GiB
  {
    uint64_t n = (big / 2) / 16;
    copyk<<<nsm * 8, 512>>>((int4*)buf, (int4*)(buf + big / 16), n);
    CK(cudaEventRecord(e0));
    for (int r = 0; r < 5; ++r) copyk<<<nsm * 8, 512>>>((int4*)buf, (int4*)((char*)buf + big / 2), n);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("copy 2GiB: %.1f GB/s (read+write)\n", 5.0 * 2 * (big / 2) / (ms * 1e6));
  }
  const int grid = nsm * 8, block = 256;
  const uint64_t threads = (uint64_t)grid * block;
  for (int gran = 0; gran < 2; ++gran) {
    if (gran == 1) CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, 32));
    size_t g = 0;
    cudaDeviceGetLimit(&g, cudaLimitMaxL2FetchGranularity);
    for (uint64_t ws : {512ull << 20, 4ull << 30}) {
#define RUN(U, BYTES)                                                                          \
  {                                                                                            \
    int iters = 64 / U;                                                                        \
    gather<U, BYTES><<<grid, block>>>(buf, ws / BYTES, iters, sink);                           \
    CK(cudaEventRecord(e0));                                                                   \
    for (int r = 0; r < 5; ++r) gather<U, BYTES><<<grid, block>>>(buf, ws / BYTES, iters, sink); \
    CK(cudaEventRecord(e1));                                                                   \
    CK(cudaEventSynchronize(e1));                                                              \
    cudaEventElapsedTime(&ms, e0, e1);                                                         \
    double acc = 5.0 * threads * iters * U;                                                    \
    printf("gran=%zu ws=%4lluMiB gather%3dB U=%d: %.2f G acc/s  %.1f GB/s useful\n", g,      \
           (unsigned long long)(ws >> 20), BYTES, U, acc / (ms * 1e6), acc * BYTES / (ms * 1e6)); \
  }
      RUN(1, 32) RUN(2, 32) RUN(4, 32) RUN(8, 32) RUN(2, 64) RUN(4, 64) RUN(2, 128)
      {
        int iters = 16;
        rand_cas<4><<<grid, block>>>((unsigned long long*)buf, ws / 8, iters);
        CK(cudaEventRecord(e0));
        for (int r = 0; r < 3; ++r) rand_cas<4><<<grid, block>>>((unsigned long long*)buf, ws / 8, iters);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        double acc = 3.0 * threads * iters * 4;
        printf("gran=%zu ws=%4lluMiB load+CAS64 random: %.2f G ops/s\n", g,
               (unsigned long long)(ws >> 20), acc / (ms * 1e6));
        read_cas<<<grid, block>>>((unsigned long long*)buf, ws / 32, 64);
        CK(cudaEventRecord(e0));
        for (int r = 0; r < 3; ++r) read_cas<<<grid, block>>>((unsigned long long*)buf, ws / 32, 64);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        cudaEventElapsedTime(&ms, e0, e1);
        acc = 3.0 * threads * 64;
        printf("gran=%zu ws=%4lluMiB read32B+CAS (insert pattern): %.2f G ops/s  (%.1f GB/s at 64B/op)\n", g,
               (unsigned long long)(ws >> 20), acc / (ms * 1e6), acc * 64 / (ms * 1e6));
      }
    }
  }
  CK(cudaGetLastError());
  return 0;
}
