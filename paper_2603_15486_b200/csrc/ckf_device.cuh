// ckf_device.cuh -- device-side building blocks shared by the direct and the
// L2-tiled kernels: memory primitives, the bucket operations of the reference
// (TryInsert / Find / TryRemove / swap / lane CAS, K:158-272) over 64-bit CAS,
// the DFS/BFS eviction chain (K:364-436) and block-level counting.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

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

// L2 evict-last variants for the tiled path: the bucket region being probed
// must outlive the record streams flowing past it in L2.
__device__ __forceinline__ uint64_t evict_last_policy() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

template <int WPB>
__device__ __forceinline__ void ld_bucket_ro_el(const uint64_t* p, uint64_t (&w)[WPB > 0 ? WPB : 1]) {
  if constexpr (WPB >= 4) {
#pragma unroll
    for (int s = 0; s < WPB / 4; ++s)
      asm volatile("ld.global.nc.L1::no_allocate.L2::evict_last.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(w[4 * s]), "=l"(w[4 * s + 1]), "=l"(w[4 * s + 2]), "=l"(w[4 * s + 3])
                   : "l"(p + 4 * s));
  } else if constexpr (WPB == 2) {
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;"
                 : "=l"(w[0]), "=l"(w[1]) : "l"(p), "l"(evict_last_policy()));
  } else {
    ld_bucket_ro<WPB>(p, w);
  }
}

// streaming record accesses: first out of L2
__device__ __forceinline__ uint64_t ld_stream_ef(const uint64_t* a, uint64_t pol) {
  uint64_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(a), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_stream_ef(uint64_t* a, uint64_t v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(a), "l"(v), "l"(pol) : "memory");
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

template <int WPB>
__device__ __forceinline__ void ld_bucket_rw_el(const uint64_t* p, uint64_t (&w)[WPB > 0 ? WPB : 1]) {
  if constexpr (WPB >= 4) {
#pragma unroll
    for (int s = 0; s < WPB / 4; ++s)
      asm volatile("ld.relaxed.gpu.global.L2::evict_last.v4.u64 {%0,%1,%2,%3}, [%4];"
                   : "=l"(w[4 * s]), "=l"(w[4 * s + 1]), "=l"(w[4 * s + 2]), "=l"(w[4 * s + 3])
                   : "l"(p + 4 * s)
                   : "memory");
  } else if constexpr (WPB == 2) {
    asm volatile("ld.relaxed.gpu.global.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;"
                 : "=l"(w[0]), "=l"(w[1]) : "l"(p), "l"(evict_last_policy()) : "memory");
  } else {
    ld_bucket_rw<WPB>(p, w);
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
__device__ __forceinline__ int try_insert_snap(uint64_t* words, uint64_t bucket, uint64_t tag, uint64_t (&w)[WPB]) {
  using L = Lanes<F>;
  constexpr int kB = WPB * L::kTpw;
  uint64_t* base = words + bucket * WPB;
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

template <int F, int WPB>
__device__ __forceinline__ int try_insert_t(uint64_t* words, uint64_t bucket, uint64_t tag) {
  uint64_t w[WPB];
  ld_bucket_rw<WPB>(words + bucket * WPB, w);
  return try_insert_snap<F, WPB>(words, bucket, tag, w);
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
__device__ __forceinline__ int remove_tag_snap(uint64_t* words, uint64_t bucket, uint64_t tag, uint64_t (&w)[WPB]) {
  using L = Lanes<F>;
  constexpr int kB = WPB * L::kTpw;
  uint64_t* base = words + bucket * WPB;
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

template <int F, int WPB>
__device__ __forceinline__ int remove_tag_t(uint64_t* words, uint64_t bucket, uint64_t tag) {
  uint64_t w[WPB];
  ld_bucket_rw<WPB>(words + bucket * WPB, w);
  return remove_tag_snap<F, WPB>(words, bucket, tag, w);
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

// Debug hook (ckf_debug_fault_origin_cas, the rollback test): while armed, a
// BFS relocation's origin lane is first overwritten by a "concurrent writer"
// with a stale tag, so the chain's origin CAS loses and rolls its copy back --
// the GPU counterpart of the reference's sabotaged lane_cas
// (pkg/tests/test_filter.py:224-259).  One relaxed load when disarmed.
__device__ unsigned int g_fault_origin_cas = 0;

template <int F>
__device__ __forceinline__ void fault_origin_writer(uint64_t* p, int lane, uint64_t expect) {
  unsigned int v = *(volatile unsigned int*)&g_fault_origin_cas;
  while (v) {
    const unsigned int old = atomicCAS(&g_fault_origin_cas, v, v - 1);
    if (old == v) {
      const uint64_t stale = (expect ^ 1u) ? (expect ^ 1u) : 2u;
      lane_cas<F>(p, lane, expect, stale);
      return;
    }
    v = old;
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
      fault_origin_writer<F>(base + os / L::kTpw, os % L::kTpw, ctag[chosen]);
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

// Same chain, compile-time bucket shape: every bucket the chain inspects is
// fetched as one 256-bit snapshot (not word by word), the BFS candidates'
// alternate buckets are fetched kEvictFetch at a time, and the CAS updates
// start from those snapshots.  Decisions are taken in exactly the reference
// order (first candidate with room, K:407-414), so the sequential parity mode
// stays bit-identical.
constexpr int kEvictFetch = 2;

template <int F>
__device__ __forceinline__ bool lane_cas_from(uint64_t* p, int lane, uint64_t expect, uint64_t repl, uint64_t w) {
  using L = Lanes<F>;
  while (true) {
    if (L::get(w, lane) != expect) return false;
    const uint64_t old = cas64(p, w, L::put(w, lane, repl));
    if (old == w) return true;
    w = old;
  }
}

// word j of a register snapshot, selected without dynamic indexing (which
// would put the snapshot in local memory)
template <int WPB>
__device__ __forceinline__ uint64_t snap_word(const uint64_t (&w)[WPB], uint32_t j) {
  uint64_t r = w[0];
#pragma unroll
  for (int q = 1; q < WPB; ++q)
    if (j == (uint32_t)q) r = w[q];
  return r;
}

// BFS candidate order (K:257-272) without candidate arrays: the occupied
// slots of the snapshot as a bit mask rotated to start at `start`; candidate
// j is the slot of the j-th set bit.
template <uint32_t B>
__device__ __forceinline__ uint32_t nth_candidate(uint64_t rot, uint32_t j, uint32_t start) {
  for (uint32_t k = 0; k < j; ++k) rot &= rot - 1;
  uint32_t s = (uint32_t)(__ffsll((long long)rot) - 1) + start;
  return s >= B ? s - B : s;
}

// Room map of the batch schedule (ckf_region.cuh): bit i of `bits` says
// whether bucket i had an empty lane when the probe passes last wrote it (the
// insert's phase-1 probe writes every region, phase 2 rewrites the regions it
// mutates).  The BFS asks it "does the candidate's alternate bucket have room"
// (bucket_has_empty, K:225-230) from L2 instead of fetching the bucket from
// HBM; the chains keep it current with fire-and-forget atomics.  A stale
// answer is one a concurrent insert could have produced (the chain's insert
// then finds the bucket full and the round retries, K:416-418).
// bits == nullptr: no map.
struct RoomMap {
  uint32_t* bits;
};

// a successful insert into bucket b whose snapshot had `empties` empty lanes
__device__ __forceinline__ void rm_filled(const RoomMap& rm, uint64_t b, uint32_t empties) {
  if (rm.bits && empties <= 1) atomicAnd(rm.bits + (b >> 5), ~(1u << (b & 31)));
}
__device__ __forceinline__ void rm_freed(const RoomMap& rm, uint64_t b) {
  if (rm.bits) atomicOr(rm.bits + (b >> 5), 1u << (b & 31));
}

template <int F, int WPB>
__device__ __forceinline__ uint32_t empty_lanes(const uint64_t (&w)[WPB]) {
  uint32_t c = 0;
#pragma unroll
  for (int j = 0; j < WPB; ++j) c += __popcll(Lanes<F>::zeros(w[j]));
  return c;
}

template <int F, int WPB, int POL>
__device__ Outcome evict_chain_t(uint64_t* words, uint64_t h, uint64_t fp, uint64_t i1, uint64_t i2, const Geo& g,
                                 const RoomMap rm = RoomMap{nullptr}) {
  using L = Lanes<F>;
  constexpr int kTpw = L::kTpw;
  constexpr uint32_t kB = WPB * kTpw;
  constexpr uint32_t kLim = kB / 2 ? kB / 2 : 1;
  constexpr uint64_t kAll = kB == 64 ? ~0ull : ((1ull << kB) - 1u);
  const uint64_t tag2 = make_tag(fp, POL == CKF_POLICY_OFFSET ? 1u : 0u, g);
  uint64_t st = rng_init(g.seed, h, g.worker) + kGolden;
  uint64_t cur_b = i1, cur_tag = fp;
  if (smix(st) & 1u) {
    cur_b = i2;
    cur_tag = tag2;
  }
  if (g.eviction == CKF_EVICT_DFS) {  // K:374-389
    for (uint32_t n = 1; n <= g.max_evictions; ++n) {
      st += kGolden;
      const uint32_t victim = (uint32_t)(smix(st) % kB);
      const uint64_t ev = swap_slot<F>(words, cur_b, victim, cur_tag, g);
      if (ev == 0) return {1u, n, 0};
      uint64_t nc;
      const uint64_t efp = tag_fp(ev, g);
      cur_b = alt_index<POL>(cur_b, efp, tag_choice(ev, g), g, nc);
      cur_tag = make_tag(efp, nc, g);
      if (try_insert_t<F, WPB>(words, cur_b, cur_tag) >= 0) return {1u, n, 0};
    }
    return {0u, g.max_evictions, tag_fp(cur_tag, g)};
  }
  // BFS (K:391-436)
  for (uint32_t n = 1; n <= g.max_evictions; ++n) {
    st += kGolden;
    const uint32_t start = (uint32_t)(smix(st) % kB);
    uint64_t* base = words + cur_b * WPB;
    uint64_t cw[WPB];
    ld_bucket_rw<WPB>(base, cw);
    uint64_t occ = 0;  // bit s = slot s occupied
#pragma unroll
    for (int q = 0; q < WPB; ++q) {
      const uint64_t z = L::zeros(cw[q]);
#pragma unroll
      for (int s = 0; s < kTpw; ++s)
        if (!((z >> (s * F + F - 1)) & 1u)) occ |= 1ull << (q * kTpw + s);
    }
    const uint64_t rot = start ? (((occ >> start) | (occ << (kB - start))) & kAll) : occ;
    const uint32_t pc = (uint32_t)__popcll(rot);
    const uint32_t cnt = pc < kLim ? pc : kLim;
    if (cnt == 0) {  // drained by concurrent deletes: take a direct slot
      const uint32_t e = empty_lanes<F, WPB>(cw);
      if (try_insert_snap<F, WPB>(words, cur_b, cur_tag, cw) >= 0) {
        rm_filled(rm, cur_b, e);
        return {1u, n, 0};
      }
      continue;
    }
    int chosen = -1;
    uint64_t alt_b = 0, alt_tag = 0, aw_chosen[WPB];
    if (rm.bits) {
      // every candidate's room bit at once (independent L2 loads of the
      // map), then the first candidate with room in the reference order
      // (K:407-414); only that candidate's bucket is fetched
      uint32_t word[kLim], bit[kLim];
      uint64_t rr = rot;
#pragma unroll
      for (uint32_t c = 0; c < kLim; ++c) {
        word[c] = bit[c] = 0;
        if (c >= cnt) continue;
        uint32_t s = (uint32_t)(__ffsll((long long)rr) - 1) + start;
        s = s >= kB ? s - kB : s;
        rr &= rr - 1;
        const uint64_t ct = L::get(snap_word<WPB>(cw, s / kTpw), s % kTpw);
        uint64_t tc;
        const uint64_t ab = alt_index<POL>(cur_b, tag_fp(ct, g), tag_choice(ct, g), g, tc);
        word[c] = __ldcg(rm.bits + (ab >> 5));
        bit[c] = (uint32_t)(ab & 31);
      }
      uint32_t roomm = 0;
#pragma unroll
      for (uint32_t c = 0; c < kLim; ++c) roomm |= ((word[c] >> bit[c]) & 1u) << c;
      if (roomm) {
        chosen = __ffs((int)roomm) - 1;
        const uint32_t s = nth_candidate<kB>(rot, (uint32_t)chosen, start);
        const uint64_t ct = L::get(snap_word<WPB>(cw, s / kTpw), s % kTpw);
        uint64_t tc;
        const uint64_t cfp = tag_fp(ct, g);
        alt_b = alt_index<POL>(cur_b, cfp, tag_choice(ct, g), g, tc);
        alt_tag = make_tag(cfp, tc, g);
        ld_bucket_rw<WPB>(words + alt_b * WPB, aw_chosen);
      }
    } else {
      for (uint32_t c0 = 0; c0 < cnt && chosen < 0; c0 += kEvictFetch) {
        uint64_t aw[kEvictFetch][WPB], ab[kEvictFetch], at[kEvictFetch];
#pragma unroll
        for (int q = 0; q < kEvictFetch; ++q) {
          if (c0 + q >= cnt) continue;
          const uint32_t s = nth_candidate<kB>(rot, c0 + q, start);
          const uint64_t ct = L::get(snap_word<WPB>(cw, s / kTpw), s % kTpw);
          uint64_t tc;
          const uint64_t cfp = tag_fp(ct, g);
          ab[q] = alt_index<POL>(cur_b, cfp, tag_choice(ct, g), g, tc);
          at[q] = make_tag(cfp, tc, g);
          ld_bucket_rw<WPB>(words + ab[q] * WPB, aw[q]);
        }
#pragma unroll
        for (int q = 0; q < kEvictFetch; ++q) {
          if (chosen >= 0 || c0 + q >= cnt) continue;
          uint64_t any = 0;
#pragma unroll
          for (int j = 0; j < WPB; ++j) any |= L::zeros(aw[q][j]);
          if (any) {
            chosen = (int)(c0 + q);
            alt_b = ab[q];
            alt_tag = at[q];
#pragma unroll
            for (int j = 0; j < WPB; ++j) aw_chosen[j] = aw[q][j];
          }
        }
      }
    }
    const uint32_t os = nth_candidate<kB>(rot, chosen >= 0 ? (uint32_t)chosen : cnt - 1, start);
    const uint64_t ow = snap_word<WPB>(cw, os / kTpw);
    const uint64_t otag = L::get(ow, os % kTpw);
    if (chosen >= 0) {
      // two-step relocation: copy the candidate out, then swap ourselves in
      const uint32_t e = empty_lanes<F, WPB>(aw_chosen);
      const int aslot = try_insert_snap<F, WPB>(words, alt_b, alt_tag, aw_chosen);
      if (aslot < 0) {  // the free lane raced away
        if (rm.bits) rm_filled(rm, alt_b, 0);
        continue;
      }
      rm_filled(rm, alt_b, e);
      fault_origin_writer<F>(base + os / kTpw, os % kTpw, otag);
      if (lane_cas_from<F>(base + os / kTpw, os % kTpw, otag, cur_tag, ow)) return {1u, n, 0};
      lane_cas<F>(words + alt_b * WPB + aslot / kTpw, aslot % kTpw, alt_tag, 0);  // rollback
      rm_freed(rm, alt_b);
      continue;
    }
    // nobody has room: evict the last candidate and deepen (K:427-434)
    if (!lane_cas_from<F>(base + os / kTpw, os % kTpw, otag, cur_tag, ow)) continue;
    uint64_t nc;
    const uint64_t cfp = tag_fp(otag, g);
    cur_b = alt_index<POL>(cur_b, cfp, tag_choice(otag, g), g, nc);
    cur_tag = make_tag(cfp, nc, g);
  }
  return {0u, g.max_evictions, tag_fp(cur_tag, g)};
}

template <int F, int WPB, int POL>
__device__ __forceinline__ Outcome evict_any(uint64_t* words, uint64_t h, uint64_t fp, uint64_t i1, uint64_t i2,
                                             const Geo& g, const RoomMap rm = RoomMap{nullptr}) {
  if constexpr (WPB > 0) return evict_chain_t<F, WPB, POL>(words, h, fp, i1, i2, g, rm);
  else return evict_chain<F, POL>(words, h, fp, i1, i2, g);
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

}  // namespace ckf
