// Atomic-throughput probe: which commit primitive can an insert/delete afford?
// L2-resident (16 MiB) and DRAM-resident (512 MiB) random targets:
//   CAS64 (with return), CAS32, atomicAdd32 (with return), RED.OR32 (no return),
//   plain 256-bit load for comparison; and shared-memory CAS64 / CAS32.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_atomics tools/probe_atomics.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <int KIND>
__global__ void __launch_bounds__(256) gatom(unsigned long long* buf, uint64_t nwords, int iters,
                                             unsigned long long* sink) {
  uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint64_t i = mix(tid * 0x9E3779B97F4A7C15ull + it) & (nwords - 1);
    if (KIND == 0) acc += atomicCAS(buf + i, acc, acc + 1);                       // CAS64
    if (KIND == 1) acc += atomicCAS((unsigned*)(buf + i), (unsigned)acc, 7u);     // CAS32
    if (KIND == 2) acc += atomicAdd((unsigned*)(buf + i), 1u);                     // ADD32 ret
    if (KIND == 3) atomicOr((unsigned*)(buf + i), 1u << (it & 31));               // RED.OR
    if (KIND == 4) {                                                              // 32B load
      uint64_t a, b, c, d;
      asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(buf + (i & ~3ull)));
      acc += a ^ b ^ c ^ d;
    }
    if (KIND == 5) {  // insert pattern: 32B relaxed load then CAS on one word of it
      uint64_t a, b, c, d;
      unsigned long long* p = buf + (i & ~3ull);
      asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
      acc += atomicCAS(p + (a & 3), a, a + 1);
    }
  }
  if (acc == 0x1234567) sink[0] = acc;
}

template <int KIND>
__global__ void __launch_bounds__(256) satom(int iters, unsigned long long* sink) {
  extern __shared__ unsigned long long sm[];
  const int nw = 96 * 1024 / 8;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint32_t i = (uint32_t)(mix(tid * 0x9E3779B97F4A7C15ull + it) % nw);
    if (KIND == 0) acc += atomicCAS(sm + i, acc, acc + 1);
    if (KIND == 1) acc += atomicCAS((unsigned*)(sm + i), (unsigned)acc, 7u);
  }
  if (acc == 0x1234567) sink[0] = acc;
}

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *buf, *sink;
  CK(cudaMalloc(&buf, 512ull << 20));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMemset(buf, 0, 512ull << 20));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[] = {"CAS64", "CAS32", "ADD32-ret", "RED.OR32", "LD256", "LD256+CAS64"};
  const int grid = nsm * 8, block = 256, iters = 64;
  for (uint64_t bytes : {16ull << 20, 512ull << 20}) {
    for (int k = 0; k < 6; ++k) {
      float ms;
      auto launch = [&](int kk) {
        switch (kk) {
          case 0: gatom<0><<<grid, block>>>(buf, bytes / 8, iters, sink); break;
          case 1: gatom<1><<<grid, block>>>(buf, bytes / 8, iters, sink); break;
          case 2: gatom<2><<<grid, block>>>(buf, bytes / 8, iters, sink); break;
          case 3: gatom<3><<<grid, block>>>(buf, bytes / 8, iters, sink); break;
          case 4: gatom<4><<<grid, block>>>(buf, bytes / 8, iters, sink); break;
          case 5: gatom<5><<<grid, block>>>(buf, bytes / 8, iters, sink); break;
        }
      };
      launch(k);
      CK(cudaEventRecord(e0));
      for (int r = 0; r < 3; ++r) launch(k);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      printf("global %4llu MiB %-12s %7.2f G ops/s\n", (unsigned long long)(bytes >> 20), names[k],
             3.0 * grid * block * iters / (ms * 1e6));
    }
  }
  cudaFuncSetAttribute(satom<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  cudaFuncSetAttribute(satom<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  for (int k = 0; k < 2; ++k) {
    float ms;
    for (int r = 0; r < 2; ++r) {
      CK(cudaEventRecord(e0));
      if (k == 0) satom<0><<<nsm * 2, 256, 96 * 1024>>>(1024, sink);
      else satom<1><<<nsm * 2, 256, 96 * 1024>>>(1024, sink);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
    }
    cudaEventElapsedTime(&ms, e0, e1);
    printf("shared %-12s %7.2f G ops/s (incl. 96KB zero-fill)\n", k ? "CAS32" : "CAS64",
           1.0 * nsm * 2 * 256 * 1024 / (ms * 1e6));
  }
  CK(cudaGetLastError());
  return 0;
}
