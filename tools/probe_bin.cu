// Bin-pass design probe (round 2): how fast can 255 M keys be hashed and
// scattered into R fine-region bins in ONE pass?
//   scatter<T>: persistent CTAs, bin counters in shared memory, every CTA owns a
//               private segment of every bin (no global atomics), each record
//               is one scattered 8 B store (the L2 merges a bin's records into
//               whole sectors: the write frontier is G*R*32 B)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_bin tools/probe_bin.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

constexpr uint64_t kP1 = 0x9E3779B185EBCA87ull, kP2 = 0xC2B2AE3D27D4EB4Full, kP3 = 0x165667B19E3779F9ull,
                   kP4 = 0x85EBCA77C2B2AE63ull, kP5 = 0x27D4EB2F165667C5ull;
__device__ __forceinline__ uint64_t rotl(uint64_t x, unsigned r) { return (x << r) | (x >> (64u - r)); }
__device__ __forceinline__ uint64_t xxh64(uint64_t key, uint64_t seed) {
  uint64_t acc = seed + kP5 + 8u;
  acc ^= rotl(key * kP2, 31) * kP1;
  acc = rotl(acc, 27) * kP1 + kP4;
  acc ^= acc >> 33;
  acc *= kP2;
  acc ^= acc >> 29;
  acc *= kP3;
  return acc ^ (acc >> 32);
}
__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void gen(uint64_t* k, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    k[i] = mix(i + 12345) & 0xFFFFFFFFull;
}

// STORE: 0 plain st.global, 1 st.global.L1::no_allocate, 2 st.global.cs
template <int ITEMS, int STORE>
__global__ void scatter(const uint64_t* __restrict__ keys, uint64_t n, uint32_t lm, uint32_t lrb, uint32_t R,
                        uint64_t* __restrict__ bins, uint32_t cap, uint32_t* __restrict__ cnt_out) {
  extern __shared__ uint32_t cnt[];
  for (uint32_t r = threadIdx.x; r < R; r += blockDim.x) cnt[r] = 0;
  __syncthreads();
  const uint32_t G = gridDim.x, c = blockIdx.x;
  const uint64_t mmask = (1ull << lm) - 1u;
  const uint64_t tile = (uint64_t)blockDim.x * ITEMS;
  for (uint64_t t0 = (uint64_t)blockIdx.x * tile; t0 < n; t0 += (uint64_t)G * tile) {
    uint64_t kk[ITEMS];
#pragma unroll
    for (int q = 0; q < ITEMS / 2; ++q) {
      const uint64_t i = t0 + (uint64_t)q * 2 * blockDim.x + 2 * threadIdx.x;
      if (i + 1 < n) {
        asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(kk[2 * q]), "=l"(kk[2 * q + 1]) : "l"(keys + i));
      } else {
        kk[2 * q] = i < n ? keys[i] : 0;
        kk[2 * q + 1] = 0;
      }
    }
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      const uint64_t i = t0 + (uint64_t)(q >> 1) * 2 * blockDim.x + 2 * threadIdx.x + (q & 1);
      if (i >= n) continue;
      const uint64_t h = xxh64(kk[q], 0);
      const uint64_t fp0 = (h >> 32) & 0xFFFF;
      const uint64_t fp = fp0 ? fp0 : 1;
      const uint64_t i1 = h & mmask;
      const uint32_t b = (uint32_t)(i1 >> lrb);
      const uint64_t rec = (i << 32) | ((i1 & ((1u << lrb) - 1u)) << 16) | fp;
      const uint32_t pos = atomicAdd(&cnt[b], 1u);
      if (pos < cap) {
        uint64_t* d = bins + ((uint64_t)b * G + c) * cap + pos;
        if (STORE == 0) *d = rec;
        else if (STORE == 1) asm volatile("st.global.L1::no_allocate.u64 [%0], %1;" ::"l"(d), "l"(rec) : "memory");
        else if (STORE == 2) asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(d), "l"(rec) : "memory");
        else if (STORE == 3) { if (rec == 0x1234567) bins[0] = rec; }           // no store: hash + atomics only
        else if (STORE == 4) bins[i] = rec;                                       // streaming store
        else if (STORE == 5) {                                                    // one full 32 B sector per 4 records
          if ((pos & 3) == 3) {
            uint64_t* s = bins + ((uint64_t)b * G + c) * cap + (pos & ~3u);
            asm volatile("st.global.v4.u64 [%0], {%1,%1,%1,%1};" ::"l"(s), "l"(rec) : "memory");
          }
        } else if (STORE == 6) {                                                  // one 16 B store per 2 records
          if ((pos & 1) == 1) {
            uint64_t* s = bins + ((uint64_t)b * G + c) * cap + (pos & ~1u);
            asm volatile("st.global.v2.u64 [%0], {%1,%1};" ::"l"(s), "l"(rec) : "memory");
          }
        }
      }
    }
  }
  __syncthreads();
  for (uint32_t r = threadIdx.x; r < R; r += blockDim.x) cnt_out[(uint64_t)r * G + c] = cnt[r];
}

__global__ void copyk(const int4* __restrict__ a, int4* __restrict__ b, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

int main(int argc, char** argv) {
  const uint64_t n = argc > 1 ? strtoull(argv[1], 0, 0) : 255013683ull;
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint64_t* keys;
  CK(cudaMalloc(&keys, n * 8));
  gen<<<sms * 8, 256>>>(keys, n);
  const uint64_t binbytes = n * 8 * 2;
  uint64_t* bins;
  CK(cudaMalloc(&bins, binbytes));
  uint32_t* cnt;
  CK(cudaMalloc(&cnt, 64ull << 20));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  {  // copy reference: n*8 B read + n*8 B write
    for (int it = 0; it < 3; ++it) copyk<<<sms * 8, 512>>>((const int4*)keys, (int4*)bins, n / 2);
    CK(cudaEventRecord(e0));
    for (int it = 0; it < 5; ++it) copyk<<<sms * 8, 512>>>((const int4*)keys, (int4*)bins, n / 2);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= 5;
    printf("copy %llu keys: %.3f ms  %.1f GB/s\n", (unsigned long long)n, ms, 16.0 * n / ms / 1e6);
  }
  struct Cfg { uint32_t lm, lrb; int threads, per_sm, store; };
  const Cfg cfgs[] = {
      {24, 12, 1024, 1, 1}, {24, 12, 1024, 1, 3}, {24, 12, 1024, 1, 4}, {24, 12, 1024, 1, 5},
      {24, 12, 1024, 1, 6}, {24, 12, 512, 2, 3},  {24, 12, 512, 2, 5},  {24, 15, 1024, 1, 1},
      {24, 15, 1024, 1, 5}, {24, 9, 1024, 1, 1},
  };
  for (const Cfg& k : cfgs) {
    const uint32_t R = 1u << (k.lm - k.lrb);
    const uint32_t G = sms * k.per_sm;
    const double lam = (double)n / ((double)R * G);
    uint32_t cap = (uint32_t)(lam + 8 * sqrt(lam) + 16);
    cap = (cap + 3) & ~3u;
    if ((uint64_t)cap * R * G * 8 > binbytes) { printf("skip lm=%u\n", k.lm); continue; }
    const size_t smem = R * 4;
    auto launch = [&]() {
      switch (k.store) {
#define L(S) case S: CK(cudaFuncSetAttribute(scatter<8, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        scatter<8, S><<<G, k.threads, smem>>>(keys, n, k.lm, k.lrb, R, bins, cap, cnt); break;
        L(0) L(1) L(2) L(3) L(4) L(5) L(6)
#undef L
      }
    };
    for (int it = 0; it < 3; ++it) launch();
    CK(cudaGetLastError());
    CK(cudaEventRecord(e0));
    for (int it = 0; it < 5; ++it) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= 5;
    printf("scatter m=2^%u R=%u G=%u thr=%d store=%d cap=%u (lam %.0f): %.3f ms  %.1f GB/s (16 B/key)  %.1f G keys/s\n",
           k.lm, R, G, k.threads, k.store, cap, lam, ms, 16.0 * n / ms / 1e6, n / ms / 1e6);
  }
  return 0;
}
