// L2 retention probe: random 32 B accesses inside a hot window of W bytes
// interleaved with a sequential stream (the tiled probe pattern).  If the hot
// window stays L2-resident the random rate is far above the ~48 G/s DRAM
// ceiling; if the stream flushes it, the rate collapses.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_l2mix tools/probe_l2mix.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// MODE 0: loads only; 1: CAS on the hot word; 2: RED.OR on the hot word
template <int MODE, bool EF>
__global__ void __launch_bounds__(256) mixk(const uint64_t* __restrict__ stream, uint64_t stream_words,
                                            unsigned long long* hot, uint64_t hot_sectors, int iters,
                                            unsigned long long* sink) {
  uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  unsigned long long acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint64_t si = (tid + (uint64_t)it * nthreads) % stream_words;
    uint64_t s;
    if (EF) asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(s) : "l"(stream + si), "l"(pol));
    else asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(s) : "l"(stream + si));
    uint64_t h = mix(tid * 0x9E3779B97F4A7C15ull + it) % hot_sectors;
    unsigned long long* p = hot + h * 4;
    if (MODE == 0) {
      uint64_t a, b, c, d;
      asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
      acc += a ^ b ^ c ^ d ^ s;
    } else if (MODE == 1) {
      acc += atomicCAS(p, s, s + 1);
    } else {
      atomicOr((unsigned*)p, (unsigned)s | 1u);
      acc += s;
    }
  }
  if (acc == 0x1234567) sink[0] = acc;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t stream_bytes = 4ull << 30;
  uint64_t* stream;
  unsigned long long *hot, *sink;
  cudaMalloc(&stream, stream_bytes);
  cudaMalloc(&hot, 256ull << 20);
  cudaMalloc(&sink, 64);
  cudaMemset(stream, 1, stream_bytes);
  cudaMemset(hot, 0, 256ull << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = nsm * 8, block = 256, iters = 64;
  const double ops = (double)grid * block * iters;
  const char* mname[] = {"LD256", "CAS64", "RED.OR"};
  for (int mode = 0; mode < 3; ++mode)
    for (int ef = 0; ef < 2; ++ef)
      for (uint64_t w : {2ull << 20, 8ull << 20, 16ull << 20, 32ull << 20, 64ull << 20, 128ull << 20}) {
        auto launch = [&]() {
          uint64_t sw = stream_bytes / 8, hs = w / 32;
          if (mode == 0 && !ef) mixk<0, false><<<grid, block>>>(stream, sw, hot, hs, iters, sink);
          if (mode == 0 && ef) mixk<0, true><<<grid, block>>>(stream, sw, hot, hs, iters, sink);
          if (mode == 1 && !ef) mixk<1, false><<<grid, block>>>(stream, sw, hot, hs, iters, sink);
          if (mode == 1 && ef) mixk<1, true><<<grid, block>>>(stream, sw, hot, hs, iters, sink);
          if (mode == 2 && !ef) mixk<2, false><<<grid, block>>>(stream, sw, hot, hs, iters, sink);
          if (mode == 2 && ef) mixk<2, true><<<grid, block>>>(stream, sw, hot, hs, iters, sink);
        };
        launch();
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-6s stream_ef=%d hot=%4llu MiB: %7.2f G ops/s (each op = 8 B stream + 1 hot access)\n", mname[mode],
               ef, (unsigned long long)(w >> 20), 3 * ops / (ms * 1e6));
      }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
