// Sliding-window L2 probe: exactly the access pattern of the tiled probe pass
// without any filter logic.  P records (8 B, streamed) are processed by a flat
// grid-stride loop; record p touches a random 32 B bucket inside region
// p*R/P of a 512 MiB table (R regions).  If the active region stays in L2 the
// pass runs at streaming speed; if not, it degrades to the random-sector rate.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_sliding tools/probe_sliding.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <int MODE>  // 0: 256-bit load, 1: load + CAS
__global__ void __launch_bounds__(256) slide(const uint64_t* __restrict__ recs, uint64_t P, unsigned long long* table,
                                             uint64_t nbuckets, uint32_t R, unsigned long long* sink) {
  const uint64_t per_region = nbuckets / R;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 4;
  unsigned long long acc = 0;
  for (uint64_t p0 = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * 4; p0 < P; p0 += stride) {
    uint64_t rv[4];
    asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(rv[0]), "=l"(rv[1]), "=l"(rv[2]), "=l"(rv[3]) : "l"(recs + p0));
    uint64_t w[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint64_t p = p0 + q;
      const uint64_t region = p * R / P;
      const uint64_t b = region * per_region + mix(p ^ rv[q]) % per_region;
      asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(w[q][0]), "=l"(w[q][1]), "=l"(w[q][2]), "=l"(w[q][3]) : "l"(table + b * 4));
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (MODE == 1) {
        const uint64_t p = p0 + q;
        const uint64_t region = p * R / P;
        const uint64_t b = region * per_region + mix(p ^ rv[q]) % per_region;
        acc += atomicCAS(table + b * 4 + (w[q][0] & 3), w[q][0], w[q][0] + 1);
      } else {
        acc += w[q][0] ^ w[q][1] ^ w[q][2] ^ w[q][3];
      }
    }
  }
  if (acc == 0x1234567) sink[0] = acc;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t P = 255ull << 20, nb = 16ull << 20;
  uint64_t* recs;
  unsigned long long *table, *sink;
  cudaMalloc(&recs, P * 8);
  cudaMalloc(&table, nb * 32);
  cudaMalloc(&sink, 64);
  cudaMemset(recs, 3, P * 8);
  cudaMemset(table, 0, nb * 32);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode)
    for (int bpsm : {4, 8})
      for (uint32_t R : {1u, 8u, 32u, 128u, 512u, 4096u}) {
        const int grid = nsm * bpsm;
        auto launch = [&]() {
          if (mode == 0) slide<0><<<grid, 256>>>(recs, P, table, nb, R, sink);
          else slide<1><<<grid, 256>>>(recs, P, table, nb, R, sink);
        };
        launch();
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%s blocks/SM=%d R=%5u (region %6.1f MiB): %6.3f ms  %6.1f G rec/s\n", mode ? "LD+CAS" : "LD    ", bpsm,
               R, 512.0 / R, ms, P / (ms * 1e6));
      }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
