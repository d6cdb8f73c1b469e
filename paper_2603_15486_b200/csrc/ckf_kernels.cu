// ckf_kernels.cu -- sm_100a kernels and the C ABI (include/ckf.h) of the
// cuckoo-filter hot path: insert / query / delete over a packed-fingerprint
// bucket table in HBM.
//
// Table layout: uint64 words[m * wpb], bucket i = words
// [i*wpb, (i+1)*wpb), lane s of a word = bits [s*f, (s+1)*f), 0 = empty
// (reference filter.py:130, wordops.py:1-16).  With f=16, b=16 a bucket is one
// 32-byte sector and is fetched by one 256-bit load.
//
// Kernel families (all one thread per key, grid-stride over the batch):
//   query_kernel   <F,WPB,POL,KPT>  read-only, 256-bit ld.global.nc bucket loads,
//                                   KPT keys per thread for memory-level parallelism
//   insert_kernel  <F,WPB,POL>      direct TryInsert into i1 then i2 with a 64-bit
//                                   atomicCAS commit; keys whose pair is full are
//                                   queued (warp-aggregated) for...
//   evict_kernel   <F,POL>          ...the DFS / BFS eviction pass (K:374-436)
//   delete_kernel  <F,WPB,POL>      TryRemove with CAS-clear (K:461-484)
//   seq_*_kernel   <F,POL>          one device thread walking the batch in order:
//                                   bit-identical to the reference insert_batch /
//                                   delete_batch with workers=1 (parity mode)
// WPB = words per bucket as a template constant for 1/2/4/8, or 0 for the
// runtime-wpb generic path (any legal b).
#include <cuda_runtime.h>

#include <stdint.h>

#include <atomic>

#include "../../include/ckf.h"
#include "ckf_semantics.cuh"

namespace ckf {

constexpr int kMaxSlots = 128;  // GPU limit on bucket_slots (BFS candidate scratch)

// ---------------------------------------------------------------------------
// memory primitives
// ---------------------------------------------------------------------------

// Streaming key read: read-only path, no L1 allocation.
__device__ __forceinline__ uint64_t ld_stream(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

// Read-only bucket fetch (query phase only): one 256-bit
// ld.global.nc per 32-byte sector.
template <int WPB>
__device__ __forceinline__ void ld_bucket_ro(const uint64_t* p, uint64_t (&w)[WPB > 0 ? WPB : 1]) {
  if constexpr (WPB == 1) {
    asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(w[0]) : "l"(p));
  } else if constexpr (WPB == 2) {
    asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(w[0]), "=l"(w[1]) : "l"(p));
  } else if constexpr (WPB >= 4) {
#pragma unroll
    for (int s = 0; s < WPB / 4; ++s)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(w[4 * s]), "=l"(w[4 * s + 1]), "=l"(w[4 * s + 2]), "=l"(w[4 * s + 3])
                   : "l"(p + 4 * s));
  }
}

// Coherent bucket snapshot for the mutating kernels: relaxed gpu-scope loads
// are served by L2 (where the CAS commits), never a stale L1 line.
template <int WPB>
__device__ __forceinline__ void ld_bucket_rw(const uint64_t* p, uint64_t (&w)[WPB > 0 ? WPB : 1]) {
  if constexpr (WPB == 1) {
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w[0]) : "l"(p) : "memory");
  } else if constexpr (WPB == 2) {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0,%1}, [%2];" : "=l"(w[0]), "=l"(w[1]) : "l"(p) : "memory");
  } else if constexpr (WPB >= 4) {
#pragma unroll
    for (int s = 0; s < WPB / 4; ++s)
      asm volatile("ld.relaxed.gpu.global.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(w[4 * s]), "=l"(w[4 * s + 1]), "=l"(w[4 * s + 2]), "=l"(w[4 * s + 3])
                   : "l"(p + 4 * s)
                   : "memory");
  }
}

__device__ __forceinline__ uint64_t ld_word_rw(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint64_t cas64(uint64_t* p, uint64_t expect, uint64_t desired) {
  return atomicCAS(reinterpret_cast<unsigned long long*>(p), (unsigned long long)expect,
                   (unsigned long long)desired);
}

// ---------------------------------------------------------------------------
// bucket operations
// ---------------------------------------------------------------------------

// TryInsert (K:158-180): lowest empty lane of the first word,
// in wrap order from (tag % b)/tpw, that has one; committed by CAS, rescanning
// the word the CAS lost on.  Returns the slot or -1.  Compile-time WPB.
template <int F, int WPB>
__device__ __forceinline__ int try_insert_t(uint64_t* words, uint64_t bucket, uint64_t tag) {
  using L = Lanes<F>;
  constexpr int kB = WPB * L::kTpw;
  uint64_t* base = words + bucket * WPB;
  uint64_t w[WPB];
  ld_bucket_rw<WPB>(base, w);
  const int start = (int)(tag % kB) / L::kTpw;
  while (true) {
    int best = -1, bestp = WPB;
    uint64_t bw = 0;
#pragma unroll
    for (int j = 0; j < WPB; ++j) {
      int pos = (j - start + WPB) % WPB;  // scan position of word j
      if (L::zeros(w[j]) && pos < bestp) {
        best = j;
        bestp = pos;
        bw = w[j];
      }
    }
    if (best < 0) return -1;
    int lane = L::first(L::zeros(bw));
    uint64_t old = cas64(base + best, bw, L::put(bw, lane, tag));
    if (old == bw) return best * L::kTpw + lane;
#pragma unroll
    for (int j = 0; j < WPB; ++j)
      if (j == best) w[j] = old;
  }
}

// Same contract, runtime words-per-bucket (any legal b).
template <int F>
__device__ int try_insert_rt(uint64_t* words, uint64_t bucket, uint64_t tag, const Geo& g) {
  using L = Lanes<F>;
  uint64_t* base = words + bucket * g.wpb;
  const uint32_t start = (uint32_t)(tag % g.b) / L::kTpw;
  for (uint32_t k = 0; k < g.wpb; ++k) {
    uint32_t wi = start + k;
    if (wi >= g.wpb) wi -= g.wpb;
    uint64_t w = ld_word_rw(base + wi);
    while (true) {
      uint64_t z = L::zeros(w);
      if (!z) break;
      int lane = L::first(z);
      uint64_t old = cas64(base + wi, w, L::put(w, lane, tag));
      if (old == w) return (int)(wi * L::kTpw) + lane;
      w = old;
    }
  }
  return -1;
}

// TryRemove (K:202-221): CAS-clear the first lane, in scan
// order, equal to `tag` (full-lane match).  Returns the slot or -1.
template <int F, int WPB>
__device__ __forceinline__ int remove_tag_t(uint64_t* words, uint64_t bucket, uint64_t tag) {
  using L = Lanes<F>;
  constexpr int kB = WPB * L::kTpw;
  uint64_t* base = words + bucket * WPB;
  uint64_t w[WPB];
  ld_bucket_rw<WPB>(base, w);
  const uint64_t pat = L::bcast(tag);
  const int start = (int)(tag % kB) / L::kTpw;
  while (true) {
    int best = -1, bestp = WPB;
    uint64_t bw = 0;
#pragma unroll
    for (int j = 0; j < WPB; ++j) {
      int pos = (j - start + WPB) % WPB;
      if (L::zeros(w[j] ^ pat) && pos < bestp) {
        best = j;
        bestp = pos;
        bw = w[j];
      }
    }
    if (best < 0) return -1;
    int lane = L::first(L::zeros(bw ^ pat));
    uint64_t old = cas64(base + best, bw, L::put(bw, lane, 0));
    if (old == bw) return best * L::kTpw + lane;
#pragma unroll
    for (int j = 0; j < WPB; ++j)
      if (j == best) w[j] = old;
  }
}

template <int F>
__device__ int remove_tag_rt(uint64_t* words, uint64_t bucket, uint64_t tag, const Geo& g) {
  using L = Lanes<F>;
  uint64_t* base = words + bucket * g.wpb;
  const uint64_t pat = L::bcast(tag);
  const uint32_t start = (uint32_t)(tag % g.b) / L::kTpw;
  for (uint32_t k = 0; k < g.wpb; ++k) {
    uint32_t wi = start + k;
    if (wi >= g.wpb) wi -= g.wpb;
    uint64_t w = ld_word_rw(base + wi);
    while (true) {
      uint64_t mm = L::zeros(w ^ pat);
      if (!mm) break;
      int lane = L::first(mm);
      uint64_t old = cas64(base + wi, w, L::put(w, lane, 0));
      if (old == w) return (int)(wi * L::kTpw) + lane;
      w = old;
    }
  }
  return -1;
}

template <int F, int WPB>
__device__ __forceinline__ int try_insert_any(uint64_t* words, uint64_t bucket, uint64_t tag, const Geo& g) {
  if constexpr (WPB > 0) return try_insert_t<F, WPB>(words, bucket, tag);
  else return try_insert_rt<F>(words, bucket, tag, g);
}
template <int F, int WPB>
__device__ __forceinline__ int remove_tag_any(uint64_t* words, uint64_t bucket, uint64_t tag, const Geo& g) {
  if constexpr (WPB > 0) return remove_tag_t<F, WPB>(words, bucket, tag);
  else return remove_tag_rt<F>(words, bucket, tag, g);
}

// Atomic lane exchange (swap_slot, K:232-244).
template <int F>
__device__ uint64_t swap_slot(uint64_t* words, uint64_t bucket, uint32_t slot, uint64_t tag, const Geo& g) {
  using L = Lanes<F>;
  uint64_t* p = words + bucket * g.wpb + slot / L::kTpw;
  const int lane = slot % L::kTpw;
  uint64_t w = ld_word_rw(p);
  while (true) {
    uint64_t old = cas64(p, w, L::put(w, lane, tag));
    if (old == w) return L::get(w, lane);
    w = old;
  }
}

// Replace a lane only while it still holds `expect` (lane_cas, K:247-254);
// unrelated lanes of the word may change underneath and are retried.
template <int F>
__device__ bool lane_cas(uint64_t* p, int lane, uint64_t expect, uint64_t repl) {
  using L = Lanes<F>;
  uint64_t w = ld_word_rw(p);
  while (true) {
    if (L::get(w, lane) != expect) return false;
    uint64_t old = cas64(p, w, L::put(w, lane, repl));
    if (old == w) return true;
    w = old;
  }
}

template <int F>
__device__ bool bucket_has_empty(const uint64_t* words, uint64_t bucket, const Geo& g) {
  const uint64_t* p = words + bucket * g.wpb;
  for (uint32_t k = 0; k < g.wpb; ++k)
    if (Lanes<F>::zeros(ld_word_rw(p + k))) return true;
  return false;
}

// ---------------------------------------------------------------------------
// eviction chain (insert_one after both direct attempts failed, K:364-436)
// ---------------------------------------------------------------------------

struct Outcome {
  uint32_t ok;
  uint32_t rounds;
  uint64_t lost;
};

template <int F, int POL>
__device__ Outcome evict_chain(uint64_t* words, uint64_t h, uint64_t fp, uint64_t i1, uint64_t i2,
                               const Geo& g) {
  using L = Lanes<F>;
  const uint64_t tag1 = fp;
  const uint64_t tag2 = make_tag(fp, POL == CKF_POLICY_OFFSET ? 1u : 0u, g);
  uint64_t st = rng_init(g.seed, h, g.worker) + kGolden;
  uint64_t cur_b, cur_tag;
  if ((smix(st) & 1u) == 0) {
    cur_b = i1;
    cur_tag = tag1;
  } else {
    cur_b = i2;
    cur_tag = tag2;
  }
  const uint64_t b = g.b;

  if (g.eviction == CKF_EVICT_DFS) {  // K:374-389
    for (uint32_t n = 1; n <= g.max_evictions; ++n) {
      st += kGolden;
      uint32_t victim = (uint32_t)(smix(st) % b);
      uint64_t ev = swap_slot<F>(words, cur_b, victim, cur_tag, g);
      if (ev == 0) return {1u, n, 0};  // a concurrent delete freed the lane
      uint64_t nc;
      uint64_t efp = tag_fp(ev, g);
      cur_b = alt_index<POL>(cur_b, efp, tag_choice(ev, g), g, nc);
      cur_tag = make_tag(efp, nc, g);
      if (try_insert_rt<F>(words, cur_b, cur_tag, g) >= 0) return {1u, n, 0};
    }
    return {0u, g.max_evictions, tag_fp(cur_tag, g)};
  }

  // BFS (K:391-436): probe up to b/2 occupied candidates for a free alternate
  const uint32_t limit = g.b / 2 ? g.b / 2 : 1;
  uint32_t cslot[kMaxSlots / 2];
  uint64_t ctag[kMaxSlots / 2];
  for (uint32_t n = 1; n <= g.max_evictions; ++n) {
    st += kGolden;
    const uint32_t start = (uint32_t)(smix(st) % b);
    uint64_t* base = words + cur_b * g.wpb;
    // collect_candidates (K:257-272): snapshot, occupied lanes from `start`, wrapping
    uint32_t cnt = 0;
    uint64_t w = 0;
    uint32_t wcur = ~0u;
    for (uint32_t j = 0; j < g.b && cnt < limit; ++j) {
      uint32_t s = start + j;
      if (s >= g.b) s -= g.b;
      uint32_t wi = s / L::kTpw;
      if (wi != wcur) {
        w = ld_word_rw(base + wi);
        wcur = wi;
      }
      uint64_t t = L::get(w, s % L::kTpw);
      if (t) {
        cslot[cnt] = s;
        ctag[cnt] = t;
        ++cnt;
      }
    }
    if (cnt == 0) {  // drained by concurrent deletes: take a direct slot
      if (try_insert_rt<F>(words, cur_b, cur_tag, g) >= 0) return {1u, n, 0};
      continue;
    }
    int chosen = -1;
    uint64_t alt_b = 0, alt_tag = 0;
    for (uint32_t j = 0; j < cnt; ++j) {
      uint64_t tc;
      uint64_t cfp = tag_fp(ctag[j], g);
      uint64_t tb = alt_index<POL>(cur_b, cfp, tag_choice(ctag[j], g), g, tc);
      if (bucket_has_empty<F>(words, tb, g)) {
        chosen = (int)j;
        alt_b = tb;
        alt_tag = make_tag(cfp, tc, g);
        break;
      }
    }
    if (chosen >= 0) {
      // two-step relocation: copy the candidate out, then swap ourselves in
      int aslot = try_insert_rt<F>(words, alt_b, alt_tag, g);
      if (aslot < 0) continue;  // the free lane raced away
      uint32_t os = cslot[chosen];
      if (lane_cas<F>(base + os / L::kTpw, os % L::kTpw, ctag[chosen], cur_tag)) return {1u, n, 0};
      // origin lane changed underfoot: remove the copy we just made
      lane_cas<F>(words + alt_b * g.wpb + aslot / L::kTpw, aslot % L::kTpw, alt_tag, 0);
      continue;
    }
    // nobody has room: evict the last candidate and deepen (K:427-434)
    uint32_t os = cslot[cnt - 1];
    uint64_t ct = ctag[cnt - 1];
    if (!lane_cas<F>(base + os / L::kTpw, os % L::kTpw, ct, cur_tag)) continue;
    uint64_t nc;
    uint64_t cfp = tag_fp(ct, g);
    cur_b = alt_index<POL>(cur_b, cfp, tag_choice(ct, g), g, nc);
    cur_tag = make_tag(cfp, nc, g);
  }
  return {0u, g.max_evictions, tag_fp(cur_tag, g)};
}

// ---------------------------------------------------------------------------
// block-level counting: one global atomic per block
// ---------------------------------------------------------------------------

__device__ __forceinline__ void block_count_add(uint32_t mine, uint32_t alt, ckf_counters* ctr, long long* occ,
                                                int sign) {
  __shared__ unsigned int s_sum[2];
  if (threadIdx.x < 2) s_sum[threadIdx.x] = 0;
  __syncthreads();
  unsigned int w = __reduce_add_sync(0xffffffffu, mine);
  unsigned int wa = __reduce_add_sync(0xffffffffu, alt);
  if ((threadIdx.x & 31) == 0) {
    if (w) atomicAdd(&s_sum[0], w);
    if (wa) atomicAdd(&s_sum[1], wa);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (ctr && s_sum[0]) atomicAdd(&ctr->n_ok, (unsigned long long)s_sum[0]);
    if (ctr && s_sum[1]) atomicAdd(&ctr->n_alt, (unsigned long long)s_sum[1]);
    if (occ && s_sum[0])
      atomicAdd(reinterpret_cast<unsigned long long*>(occ),
                (unsigned long long)((long long)sign * (long long)s_sum[0]));
  }
}

__device__ __forceinline__ uint64_t load_hash(const uint64_t* keys, uint64_t i, uint64_t seed, bool hashed) {
  uint64_t k = ld_stream(keys + i);
  return hashed ? k : xxh64(k, seed);
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------

constexpr int kBlock = 256;

template <int F, int POL>
__global__ void __launch_bounds__(kBlock) place_kernel(Geo g, const uint64_t* __restrict__ keys, uint64_t n,
                                                       uint64_t* __restrict__ ofp, uint64_t* __restrict__ oi1,
                                                       uint64_t* __restrict__ oi2, bool hashed) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t fp, i1, i2;
    place<POL>(load_hash(keys, i, g.seed, hashed), g, fp, i1, i2);
    ofp[i] = fp;
    oi1[i] = i1;
    oi2[i] = i2;
  }
}

__global__ void __launch_bounds__(kBlock) hash_kernel(const uint64_t* __restrict__ keys, uint64_t n, uint64_t seed,
                                                      uint64_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = xxh64(ld_stream(keys + i), seed);
}

// Membership (K:439-458).  The offset policy compares payload bits only
// (K:451-453).  KPT keys per thread: all KPT primary buckets are requested
// before any is inspected, then only the misses fetch their alternate.
template <int F, int WPB, int POL, int KPT>
__global__ void __launch_bounds__(kBlock) query_kernel(Geo g, const uint64_t* __restrict__ words,
                                                       const uint64_t* __restrict__ keys, uint64_t n,
                                                       uint8_t* __restrict__ out, ckf_counters* ctr, bool hashed) {
  using L = Lanes<F>;
  constexpr int W = WPB > 0 ? WPB : 1;
  uint32_t n_hit = 0, n_alt = 0;
  const uint64_t keep = POL == CKF_POLICY_OFFSET ? ~L::kHigh : ~0ull;
  const uint64_t tile = (uint64_t)kBlock * KPT;
  for (uint64_t t0 = blockIdx.x * tile; t0 < n; t0 += (uint64_t)gridDim.x * tile) {
    uint64_t fp[KPT], i1[KPT], i2[KPT];
    bool valid[KPT];
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      uint64_t i = t0 + k * kBlock + threadIdx.x;
      valid[k] = i < n;
      uint64_t h = valid[k] ? load_hash(keys, i, g.seed, hashed) : 0;
      place<POL>(h, g, fp[k], i1[k], i2[k]);
    }
    bool hit[KPT];
    if constexpr (WPB > 0) {
      uint64_t w[KPT][W];
#pragma unroll
      for (int k = 0; k < KPT; ++k)
        if (valid[k]) ld_bucket_ro<WPB>(words + i1[k] * WPB, w[k]);
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        const uint64_t pat = L::bcast(fp[k]);
        uint64_t any = 0;
#pragma unroll
        for (int j = 0; j < WPB; ++j) any |= L::zeros((w[k][j] & keep) ^ pat);
        hit[k] = any != 0;
      }
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        if (valid[k] && !hit[k]) {
          ++n_alt;
          ld_bucket_ro<WPB>(words + i2[k] * WPB, w[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        if (hit[k]) continue;
        const uint64_t pat = L::bcast(fp[k]);
        uint64_t any = 0;
#pragma unroll
        for (int j = 0; j < WPB; ++j) any |= L::zeros((w[k][j] & keep) ^ pat);
        hit[k] = any != 0;
      }
    } else {
#pragma unroll
      for (int k = 0; k < KPT; ++k) {
        hit[k] = false;
        if (!valid[k]) continue;
        const uint64_t pat = L::bcast(fp[k]);
        for (int pass = 0; pass < 2 && !hit[k]; ++pass) {
          n_alt += pass;
          const uint64_t* p = words + (pass ? i2[k] : i1[k]) * g.wpb;
          for (uint32_t j = 0; j < g.wpb; ++j)
            if (L::zeros((__ldg(p + j) & keep) ^ pat)) {
              hit[k] = true;
              break;
            }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      if (valid[k]) out[t0 + k * kBlock + threadIdx.x] = hit[k] ? 1 : 0;
      n_hit += valid[k] && hit[k];
    }
  }
  if (ctr) block_count_add(n_hit, n_alt, ctr, nullptr, +1);
}

// Insert, direct pass (K:355-362): TryInsert(i1, fp) then TryInsert(i2, fp|choice).
// Keys whose pair is full are appended to the eviction queue (records) with
// their hash; a queue overflow runs the eviction chain in place.
template <int F, int WPB, int POL>
__global__ void __launch_bounds__(kBlock) insert_kernel(Geo g, uint64_t* __restrict__ words,
                                                        const uint64_t* __restrict__ keys, uint64_t n,
                                                        uint8_t* __restrict__ ok, int64_t* __restrict__ ev,
                                                        uint64_t* __restrict__ lost, ckf_record* __restrict__ rec,
                                                        uint64_t cap, ckf_counters* ctr, long long* occ,
                                                        bool hashed) {
  uint32_t n_ok = 0, n_alt = 0;
  const int lane_id = threadIdx.x & 31;
  for (uint64_t t0 = blockIdx.x * (uint64_t)kBlock; t0 < n; t0 += (uint64_t)gridDim.x * kBlock) {
    const uint64_t i = t0 + threadIdx.x;
    const bool valid = i < n;
    bool need = false;
    uint64_t h = 0, fp = 0, i1 = 0, i2 = 0;
    if (valid) {
      h = load_hash(keys, i, g.seed, hashed);
      place<POL>(h, g, fp, i1, i2);
      bool done = try_insert_any<F, WPB>(words, i1, fp, g) >= 0;
      if (!done) {
        ++n_alt;
        done = try_insert_any<F, WPB>(words, i2, make_tag(fp, POL == CKF_POLICY_OFFSET ? 1u : 0u, g), g) >= 0;
      }
      need = !done;
      n_ok += done;
      ok[i] = done ? 1 : 0;
      if (ev) ev[i] = 0;
      if (lost) lost[i] = 0;
    }
    const unsigned qmask = __ballot_sync(0xffffffffu, need);
    if (qmask) {
      unsigned long long qbase = 0;
      const int leader = __ffs(qmask) - 1;
      if (lane_id == leader) qbase = atomicAdd(&ctr->n_queued, (unsigned long long)__popc(qmask));
      qbase = __shfl_sync(0xffffffffu, qbase, leader);
      if (need) {
        const uint64_t pos = qbase + __popc(qmask & ((1u << lane_id) - 1u));
        if (pos < cap) {
          rec[pos] = ckf_record{i, h, 0u, 0u};
        } else {  // queue overflow: evict in place, outcome only in dense outputs
          Outcome o = evict_chain<F, POL>(words, h, fp, i1, i2, g);
          n_ok += o.ok;
          ok[i] = (uint8_t)o.ok;
          if (ev) ev[i] = o.rounds;
          if (lost) lost[i] = o.lost;
        }
      }
    }
  }
  block_count_add(n_ok, n_alt, ctr, occ, +1);
}

// Eviction pass over the queued keys (the ~4% whose pair was full at 95% load).
template <int F, int POL>
__global__ void __launch_bounds__(kBlock) evict_kernel(Geo g, uint64_t* __restrict__ words, uint8_t* __restrict__ ok,
                                                       int64_t* __restrict__ ev, uint64_t* __restrict__ lost,
                                                       ckf_record* __restrict__ rec, uint64_t cap,
                                                       ckf_counters* ctr, long long* occ) {
  const unsigned long long queued = *(volatile unsigned long long*)&ctr->n_queued;
  const uint64_t cnt = queued < cap ? queued : cap;
  uint32_t n_ok = 0;
  for (uint64_t r = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < cnt; r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = rec[r].index;
    const uint64_t h = rec[r].lost;  // the direct pass parks the key hash here
    uint64_t fp, i1, i2;
    place<POL>(h, g, fp, i1, i2);
    Outcome o = evict_chain<F, POL>(words, h, fp, i1, i2, g);
    rec[r] = ckf_record{i, o.lost, o.rounds, o.ok};
    n_ok += o.ok;
    ok[i] = (uint8_t)o.ok;
    if (ev) ev[i] = o.rounds;
    if (lost) lost[i] = o.lost;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) ctr->n_records = cnt;
  block_count_add(n_ok, 0, ctr, occ, +1);
}

// Delete (K:461-484): full-lane match, i1 with fp, then i2 with fp|choice.
template <int F, int WPB, int POL>
__global__ void __launch_bounds__(kBlock) delete_kernel(Geo g, uint64_t* __restrict__ words,
                                                        const uint64_t* __restrict__ keys, uint64_t n,
                                                        uint8_t* __restrict__ out, ckf_counters* ctr, long long* occ,
                                                        bool hashed) {
  uint32_t n_ok = 0, n_alt = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t fp, i1, i2;
    place<POL>(load_hash(keys, i, g.seed, hashed), g, fp, i1, i2);
    bool done = remove_tag_any<F, WPB>(words, i1, fp, g) >= 0;
    if (!done) {
      ++n_alt;
      done = remove_tag_any<F, WPB>(words, i2, POL == CKF_POLICY_OFFSET ? make_tag(fp, 1u, g) : fp, g) >= 0;
    }
    out[i] = done ? 1 : 0;
    n_ok += done;
  }
  block_count_add(n_ok, n_alt, ctr, occ, -1);
}

// Parity mode: the reference's sequential insert_batch (K:510-529), one
// device thread, same key order, same PRNG stream; bit-identical table.
template <int F, int POL>
__global__ void seq_insert_kernel(Geo g, uint64_t* words, const uint64_t* keys, uint64_t n, uint8_t* ok, int64_t* ev,
                                  uint64_t* lost, ckf_record* rec, uint64_t cap, ckf_counters* ctr, long long* occ,
                                  bool hashed) {
  uint64_t n_ok = 0, n_rec = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t h = hashed ? keys[i] : xxh64(keys[i], g.seed);
    uint64_t fp, i1, i2;
    place<POL>(h, g, fp, i1, i2);
    Outcome o{1u, 0u, 0};
    if (try_insert_rt<F>(words, i1, fp, g) < 0 &&
        try_insert_rt<F>(words, i2, make_tag(fp, POL == CKF_POLICY_OFFSET ? 1u : 0u, g), g) < 0)
      o = evict_chain<F, POL>(words, h, fp, i1, i2, g);
    ok[i] = (uint8_t)o.ok;
    if (ev) ev[i] = o.rounds;
    if (lost) lost[i] = o.lost;
    if (o.rounds || !o.ok) {
      if (n_rec < cap) rec[n_rec] = ckf_record{i, o.lost, o.rounds, o.ok};
      ++n_rec;
    }
    n_ok += o.ok;
  }
  ctr->n_ok = n_ok;
  ctr->n_queued = n_rec;
  ctr->n_records = n_rec < cap ? n_rec : cap;
  if (occ) *occ += (long long)n_ok;
}

template <int F, int POL>
__global__ void seq_delete_kernel(Geo g, uint64_t* words, const uint64_t* keys, uint64_t n, uint8_t* out,
                                  ckf_counters* ctr, long long* occ, bool hashed) {
  uint64_t n_ok = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t fp, i1, i2;
    place<POL>(hashed ? keys[i] : xxh64(keys[i], g.seed), g, fp, i1, i2);
    bool done = remove_tag_rt<F>(words, i1, fp, g) >= 0;
    if (!done) done = remove_tag_rt<F>(words, i2, POL == CKF_POLICY_OFFSET ? make_tag(fp, 1u, g) : fp, g) >= 0;
    out[i] = done;
    n_ok += done;
  }
  if (ctr) ctr->n_ok = n_ok;
  if (occ) *occ -= (long long)n_ok;
}

// ---------------------------------------------------------------------------
// launch helpers
// ---------------------------------------------------------------------------

static int sm_count() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || cached <= 0)
      cached = 148;
  }
  return cached;
}

// Grid for a grid-stride kernel: enough tiles for every key, capped at
// `waves` full residency waves of the 148 SMs.
static unsigned grid_for(uint64_t work, uint64_t per_block, int blocks_per_sm) {
  uint64_t need = (work + per_block - 1) / per_block;
  uint64_t cap = (uint64_t)sm_count() * (uint64_t)blocks_per_sm;
  if (need < 1) need = 1;
  return (unsigned)(need < cap ? need : cap);
}

static std::atomic<uint64_t> g_launches{0};

static int cuda_error() {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CKF_OK : CKF_ECUDA_BASE - (int)e;
}

// Called right after every kernel launch: counts it and maps the error code.
static int status() {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? CKF_OK : CKF_ECUDA_BASE - (int)e;
}

// Dispatch (f, wpb, policy) onto template instances.  Vectorised WPB paths
// need the bucket base aligned to the vector width.
template <template <int, int, int> class Op, typename... A>
static int dispatch3(const ckf_params* p, const void* words, A... a) {
  const uintptr_t align = (uintptr_t)words;
  int wpb = (int)p->words_per_bucket;
  int vec = (wpb == 1 || wpb == 2 || wpb == 4 || wpb == 8) && (align % (8u * (wpb >= 4 ? 4 : wpb)) == 0) ? wpb : 0;
#define CKF_CASE_W(FF, PP)                                  \
  switch (vec) {                                            \
    case 1: return Op<FF, 1, PP>::run(a...);                \
    case 2: return Op<FF, 2, PP>::run(a...);                \
    case 4: return Op<FF, 4, PP>::run(a...);                \
    case 8: return Op<FF, 8, PP>::run(a...);                \
    default: return Op<FF, 0, PP>::run(a...);               \
  }
#define CKF_CASE_P(FF)                                        \
  if (p->policy == CKF_POLICY_XOR) { CKF_CASE_W(FF, 0) }      \
  else { CKF_CASE_W(FF, 1) }
  switch (p->fingerprint_bits) {
    case 8: CKF_CASE_P(8)
    case 16: CKF_CASE_P(16)
    case 32: CKF_CASE_P(32)
  }
#undef CKF_CASE_P
#undef CKF_CASE_W
  return CKF_EINVAL;
}

struct QueryArgs {
  Geo g;
  const uint64_t* words;
  const uint64_t* keys;
  uint64_t n;
  uint8_t* out;
  ckf_counters* ctr;
  bool hashed;
  cudaStream_t s;
};

template <int F, int WPB, int POL>
struct QueryOp {
  static int run(const QueryArgs& a) {
    constexpr int KPT = WPB >= 8 ? 1 : (WPB > 0 ? 2 : 1);
    unsigned grid = grid_for(a.n, (uint64_t)kBlock * KPT, 16);
    query_kernel<F, WPB, POL, KPT><<<grid, kBlock, 0, a.s>>>(a.g, a.words, a.keys, a.n, a.out, a.ctr, a.hashed);
    return status();
  }
};

struct InsertArgs {
  Geo g;
  uint64_t* words;
  const uint64_t* keys;
  uint64_t n;
  uint8_t* ok;
  int64_t* ev;
  uint64_t* lost;
  ckf_record* rec;
  uint64_t cap;
  ckf_counters* ctr;
  long long* occ;
  bool hashed;
  bool sequential;
  cudaStream_t s;
};

template <int F, int WPB, int POL>
struct InsertOp {
  static int run(const InsertArgs& a) {
    if (a.sequential) {
      seq_insert_kernel<F, POL><<<1, 1, 0, a.s>>>(a.g, a.words, a.keys, a.n, a.ok, a.ev, a.lost, a.rec, a.cap, a.ctr,
                                                   a.occ, a.hashed);
      return status();
    }
    unsigned grid = grid_for(a.n, kBlock, 16);
    insert_kernel<F, WPB, POL><<<grid, kBlock, 0, a.s>>>(a.g, a.words, a.keys, a.n, a.ok, a.ev, a.lost, a.rec, a.cap,
                                                         a.ctr, a.occ, a.hashed);
    int st = status();
    if (st) return st;
    if (a.cap) {
      // the queue length is only known on the device: a fixed full-residency grid
      // strides over it (empty queues exit immediately)
      unsigned egrid = (unsigned)sm_count() * 4;
      evict_kernel<F, POL><<<egrid, kBlock, 0, a.s>>>(a.g, a.words, a.ok, a.ev, a.lost, a.rec, a.cap, a.ctr, a.occ);
      st = status();
    }
    return st;
  }
};

struct DeleteArgs {
  Geo g;
  uint64_t* words;
  const uint64_t* keys;
  uint64_t n;
  uint8_t* out;
  ckf_counters* ctr;
  long long* occ;
  bool hashed;
  bool sequential;
  cudaStream_t s;
};

template <int F, int WPB, int POL>
struct DeleteOp {
  static int run(const DeleteArgs& a) {
    if (a.sequential) {
      seq_delete_kernel<F, POL><<<1, 1, 0, a.s>>>(a.g, a.words, a.keys, a.n, a.out, a.ctr, a.occ, a.hashed);
      return status();
    }
    unsigned grid = grid_for(a.n, kBlock, 16);
    delete_kernel<F, WPB, POL><<<grid, kBlock, 0, a.s>>>(a.g, a.words, a.keys, a.n, a.out, a.ctr, a.occ, a.hashed);
    return status();
  }
};

template <int F, int WPB, int POL>
struct PlaceOp {
  static int run(Geo g, const uint64_t* keys, uint64_t n, uint64_t* fp, uint64_t* i1, uint64_t* i2, bool hashed,
                 cudaStream_t s) {
    if (WPB != 0) return PlaceOp<F, 0, POL>::run(g, keys, n, fp, i1, i2, hashed, s);
    place_kernel<F, POL><<<grid_for(n, kBlock, 16), kBlock, 0, s>>>(g, keys, n, fp, i1, i2, hashed);
    return status();
  }
};

static bool params_ok(const ckf_params* p) {
  return p && (p->fingerprint_bits == 8 || p->fingerprint_bits == 16 || p->fingerprint_bits == 32) &&
         p->bucket_slots >= 1 && p->bucket_slots <= kMaxSlots && p->bucket_count >= 1 &&
         p->words_per_bucket * 64u == p->bucket_slots * p->fingerprint_bits && p->max_evictions >= 1;
}

}  // namespace ckf

// ===========================================================================
// C ABI
// ===========================================================================

using namespace ckf;

extern "C" {

int ckf_abi_version(void) { return CKF_ABI_VERSION; }

uint64_t ckf_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

const char* ckf_strerror(int code) {
  if (code == CKF_OK) return "ok";
  if (code == CKF_EINVAL) return "invalid argument";
  if (code <= CKF_ECUDA_BASE) return cudaGetErrorString((cudaError_t)(CKF_ECUDA_BASE - code));
  return "unknown error";
}

int ckf_params_init(ckf_params* p, uint64_t m, uint32_t f, uint32_t b, int policy, int eviction,
                    uint32_t max_evictions, uint64_t seed) {
  if (!p) return CKF_EINVAL;
  if (f != 8 && f != 16 && f != 32) return CKF_EINVAL;           // W:40-43
  if (b < 1 || (uint64_t)b * f % 64 != 0 || b > kMaxSlots) return CKF_EINVAL;
  if (m < 1) return CKF_EINVAL;
  if (policy != CKF_POLICY_XOR && policy != CKF_POLICY_OFFSET) return CKF_EINVAL;
  if (eviction != CKF_EVICT_DFS && eviction != CKF_EVICT_BFS) return CKF_EINVAL;
  const bool pow2 = (m & (m - 1)) == 0;
  if (policy == CKF_POLICY_XOR && !pow2) return CKF_EINVAL;
  if (policy == CKF_POLICY_OFFSET && m < 2) return CKF_EINVAL;
  if (max_evictions < 1) return CKF_EINVAL;
  ckf_params q{};
  q.seed = seed;
  q.bucket_count = m;
  q.index_mask = pow2 ? m - 1 : 0;
  q.high = zero_mask_rt(f, 0);                                     // lane MSBs
  q.choice_bit = policy == CKF_POLICY_OFFSET ? (1ull << (f - 1)) : 0;  // filter.py:139
  q.delta_magic = policy == CKF_POLICY_OFFSET ? fastmod_magic(m - 1) : 0;
  q.worker = 0;
  q.fingerprint_bits = f;
  q.bucket_slots = b;
  q.words_per_bucket = b * f / 64;
  q.tags_per_word = 64 / f;
  q.payload_bits = policy == CKF_POLICY_OFFSET ? f - 1 : f;
  q.policy = (uint32_t)policy;
  q.eviction = (uint32_t)eviction;
  q.max_evictions = max_evictions;
  *p = q;
  return CKF_OK;
}

int ckf_hash(const uint64_t* keys, uint64_t n, uint64_t seed, uint64_t* out, void* stream) {
  if (n == 0) return CKF_OK;
  if (!keys || !out) return CKF_EINVAL;
  hash_kernel<<<grid_for(n, kBlock, 16), kBlock, 0, (cudaStream_t)stream>>>(keys, n, seed, out);
  return status();
}

int ckf_place(const ckf_params* p, const uint64_t* keys, uint64_t n, uint64_t* fp, uint64_t* i1, uint64_t* i2,
              unsigned flags, void* stream) {
  if (!params_ok(p)) return CKF_EINVAL;
  if (n == 0) return CKF_OK;
  if (!keys || !fp || !i1 || !i2) return CKF_EINVAL;
  return dispatch3<PlaceOp>(p, nullptr, geo_from(*p), keys, n, fp, i1, i2, (flags & CKF_INPUT_HASHED) != 0,
                            (cudaStream_t)stream);
}

int ckf_insert(const ckf_params* p, uint64_t* words, const uint64_t* keys, uint64_t n, uint8_t* ok, int64_t* evictions,
               uint64_t* lost, ckf_record* records, uint64_t record_cap, ckf_counters* counters, long long* occupancy,
               unsigned flags, void* stream) {
  if (!params_ok(p) || !words || !counters) return CKF_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(counters, 0, sizeof(ckf_counters), s) != cudaSuccess) return cuda_error();
  if (n == 0) return CKF_OK;
  if (!keys || !ok || (record_cap && !records)) return CKF_EINVAL;
  InsertArgs a{geo_from(*p), words, keys, n, ok, evictions, lost, records, records ? record_cap : 0,
               counters, occupancy, (flags & CKF_INPUT_HASHED) != 0, (flags & CKF_MODE_SEQUENTIAL) != 0, s};
  return dispatch3<InsertOp>(p, words, a);
}

int ckf_query(const ckf_params* p, const uint64_t* words, const uint64_t* keys, uint64_t n, uint8_t* out,
              ckf_counters* counters, unsigned flags, void* stream) {
  if (!params_ok(p) || !words) return CKF_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (counters && cudaMemsetAsync(counters, 0, sizeof(ckf_counters), s) != cudaSuccess) return cuda_error();
  if (n == 0) return CKF_OK;
  if (!keys || !out) return CKF_EINVAL;
  QueryArgs a{geo_from(*p), words, keys, n, out, counters, (flags & CKF_INPUT_HASHED) != 0, s};
  return dispatch3<QueryOp>(p, words, a);
}

int ckf_delete(const ckf_params* p, uint64_t* words, const uint64_t* keys, uint64_t n, uint8_t* out,
               ckf_counters* counters, long long* occupancy, unsigned flags, void* stream) {
  if (!params_ok(p) || !words) return CKF_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (counters && cudaMemsetAsync(counters, 0, sizeof(ckf_counters), s) != cudaSuccess) return cuda_error();
  if (n == 0) return CKF_OK;
  if (!keys || !out) return CKF_EINVAL;
  DeleteArgs a{geo_from(*p), words, keys, n, out, counters, occupancy, (flags & CKF_INPUT_HASHED) != 0,
               (flags & CKF_MODE_SEQUENTIAL) != 0, s};
  return dispatch3<DeleteOp>(p, words, a);
}

uint64_t ckf_host_hash(uint64_t key, uint64_t seed) { return xxh64(key, seed); }

void ckf_host_place(const ckf_params* p, uint64_t key, uint64_t* fp, uint64_t* i1, uint64_t* i2) {
  Geo g = geo_from(*p);
  uint64_t h = xxh64(key, g.seed);
  if (p->policy == CKF_POLICY_XOR) place<CKF_POLICY_XOR>(h, g, *fp, *i1, *i2);
  else place<CKF_POLICY_OFFSET>(h, g, *fp, *i1, *i2);
}

uint64_t ckf_host_alt(const ckf_params* p, uint64_t bucket, uint64_t fp, uint64_t choice, uint64_t* new_choice) {
  Geo g = geo_from(*p);
  uint64_t nc = 0, r;
  if (p->policy == CKF_POLICY_XOR) r = alt_index<CKF_POLICY_XOR>(bucket, fp, choice, g, nc);
  else r = alt_index<CKF_POLICY_OFFSET>(bucket, fp, choice, g, nc);
  if (new_choice) *new_choice = nc;
  return r;
}

uint64_t ckf_host_zero_mask(uint32_t f, uint64_t word) { return zero_mask_rt(f, word); }

}  // extern "C"
