// ckf_kernels.cu -- sm_100a kernels and the C ABI (include/ckf.h) of the
// cuckoo-filter hot path: insert / query / delete over a packed-fingerprint
// bucket table in HBM.
//
// Table layout: uint64 words[m * wpb], bucket i = words
// [i*wpb, (i+1)*wpb), lane s of a word = bits [s*f, (s+1)*f), 0 = empty
// (reference filter.py:130, wordops.py:1-16).  With f=16, b=16 a bucket is one
// 32-byte sector.
//
// Schedules, chosen per call (choose() below; ckf_schedule() reports it):
//   region (ckf_region.cuh)  large batches on large tables: bin -> split ->
//                            shared-memory probe per table region, twice
//                            (primary, then alternate buckets), + eviction;
//   direct (this file)       one thread per key:
//     query_kernel   <F,WPB,POL,KPT>  read-only 256-bit bucket loads
//     insert_kernel  <F,WPB,POL>      TryInsert i1 then i2 with a 64-bit
//                                     atomicCAS; full pairs are queued for...
//     evict_kernel   <F,WPB,POL>      ...the DFS / BFS eviction pass (K:374-436),
//                                     also the last pass of the other schedules
//     delete_kernel  <F,WPB,POL>      TryRemove with CAS-clear (K:461-484)
//   sequential (parity mode)  seq_*_kernel: one device thread walking the batch
//                            in order, bit-identical to the reference
//                            insert_batch / delete_batch with workers=1.
// WPB = words per bucket as a template constant for 1/2/4/8, or 0 for the
// runtime-wpb generic path (any legal b).
#include <cuda_runtime.h>

#include <stdint.h>

#include <atomic>
#include <cmath>
#include <cstdlib>

#include "../../include/ckf.h"
#include "ckf_semantics.cuh"
#include "ckf_device.cuh"
#include "ckf_ops.cuh"
#include "ckf_region.cuh"

namespace ckf {

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
      if (hashed && foreign(g, h)) valid[k] = false;  // padding of the sharded exchange
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
    if (valid) h = load_hash(keys, i, g.seed, hashed);
    if (valid && hashed && foreign(g, h)) {  // padding of the sharded exchange
      ok[i] = 1;
      if (ev) ev[i] = 0;
      if (lost) lost[i] = 0;
    } else if (valid) {
      place<POL>(h, g, fp, i1, i2);
      bool done = try_insert_any<F, WPB>(words, i1, fp, g) >= 0;
      if (!done) {
        ++n_alt;
        done = try_insert_any<F, WPB>(words, i2, make_tag(fp, POL == CKF_POLICY_OFFSET ? 1u : 0u, g), g) >= 0;
      }
      need = !done;
      n_ok += done;
      ok[i] = 1;  // a queued key stays 1 unless the eviction pass fails it
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
          Outcome o = evict_any<F, WPB, POL>(words, h, fp, i1, i2, g);
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
#ifndef CKF_EVICT_BLOCKS
#define CKF_EVICT_BLOCKS 3
#endif
constexpr int kEvictBlocks = CKF_EVICT_BLOCKS;  // resident blocks per SM (<= 85 registers: the BFS chain's snapshots)
// Queue entries [*qstart, n_queued) belong to this run (a chunk of the call
// whose keys start at batch index ibase; keys / ok / ev / lost are the run's).
template <int F, int WPB, int POL>
__device__ __forceinline__ void evict_chains_body(Geo g, uint64_t* __restrict__ words, uint8_t* __restrict__ ok,
                                                  int64_t* __restrict__ ev, uint64_t* __restrict__ lost,
                                                  ckf_record* __restrict__ rec, uint64_t cap, ckf_counters* ctr,
                                                  long long* occ, const uint64_t* __restrict__ keys, bool hashed,
                                                  uint64_t ibase, const unsigned long long* qstart, RoomMap rm) {
  const unsigned long long queued = *(volatile unsigned long long*)&ctr->n_queued;
  const uint64_t cnt = queued < cap ? queued : cap;
  const uint64_t r0 = qstart ? *qstart : 0;
  uint32_t n_ok = 0;
  for (uint64_t r = r0 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; r < cnt;
       r += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = rec[r].index - ibase;
    uint64_t h = rec[r].lost;  // the key hash parked by the queueing pass, or kRehash
    if (h == kRehash) h = load_hash(keys, i, g.seed, hashed);
    uint64_t fp, i1, i2;
    place<POL>(h, g, fp, i1, i2);
    Outcome o = evict_any<F, WPB, POL>(words, h, fp, i1, i2, g, rm);
    rec[r] = ckf_record{i + ibase, o.lost, o.rounds, o.ok};
    n_ok += o.ok;
    if (!o.ok) ok[i] = 0;  // queued keys enter with ok = 1 (scattered byte writes only on failure)
    if (ev) ev[i] = o.rounds;
    if (lost) lost[i] = o.lost;
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) ctr->n_records = cnt;
  block_count_add(n_ok, 0, ctr, occ, +1);
}

template <int F, int WPB, int POL>
__global__ void __launch_bounds__(kBlock, kEvictBlocks)
    evict_kernel(Geo g, uint64_t* __restrict__ words, uint8_t* __restrict__ ok, int64_t* __restrict__ ev,
                 uint64_t* __restrict__ lost, ckf_record* __restrict__ rec, uint64_t cap, ckf_counters* ctr,
                 long long* occ, const uint64_t* __restrict__ keys, bool hashed, uint64_t ibase,
                 const unsigned long long* qstart, RoomMap rm) {
  evict_chains_body<F, WPB, POL>(g, words, ok, ev, lost, rec, cap, ctr, occ, keys, hashed, ibase, qstart, rm);
}

// Room map of the whole table for the direct insert path (a bit per bucket:
// has an empty lane), built after insert_kernel so the BFS eviction pass can
// read its candidates' room from L2 the way the region schedule's does.
// Used for L2-resident tables only (the scan is one pass over the table).
// The map pays off once the eviction queue is long enough: built (gate = 1)
// when n_queued * kRoomMapBytesPerKey >= the table's bytes, else the chain pass
// runs (profiles/r02_direct_roommap.txt: a 4 Mi-key insert into a 2^28-slot
// table at 95 % load, 1.9 M queued: 0.90 -> 0.70 ms with the map).
constexpr uint64_t kRoomMapBytesPerKey = 512;
template <int F, int WPB>
__global__ void __launch_bounds__(kBlock) room_scan_kernel(const uint64_t* __restrict__ words, uint64_t m,
                                                           uint32_t* __restrict__ bits,
                                                           unsigned long long* __restrict__ cursor,
                                                           const ckf_counters* ctr,
                                                           unsigned long long* __restrict__ gate) {
  const unsigned long long queued = *(volatile const unsigned long long*)&ctr->n_queued;
  const bool use = queued * kRoomMapBytesPerKey >= m * WPB * 8ull;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *cursor = 0;  // the eviction pass's queue cursor
    *gate = use;
  }
  if (!use) return;
  const uint64_t nw = (m + 31) / 32;
  for (uint64_t b0 = (blockIdx.x * (uint64_t)kBlock + threadIdx.x) & ~31ull; b0 < nw * 32;
       b0 += (uint64_t)gridDim.x * kBlock) {
    const uint64_t b = b0 + (threadIdx.x & 31);
    bool room = false;
    if (b < m) {
      uint64_t any = 0;
#pragma unroll
      for (int j = 0; j < WPB; ++j) any |= Lanes<F>::zeros(__ldcg(words + b * WPB + j));
      room = any != 0;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, room);
    if ((threadIdx.x & 31) == 0) bits[b0 >> 5] = bal;
  }
}

// BFS eviction pass of the region schedule, one ROUND at a time per lane.
// The chains of a warp's 32 queued keys differ in length (at 95 % load: mean
// 1.11 rounds, mean warp maximum 2.23; profiles/r02_evict_rounds.txt), so
// evict_kernel's one-chain-per-loop-iteration leaves half the lanes idle.  Here
// every lane runs one BFS round (K:391-436, the same decisions and PRNG stream
// as evict_chain_t) per iteration and a lane whose chain ended takes the next
// queue entry (warp-aggregated cursor), so the warp stays full.  Candidates'
// room comes from the room map (RoomMap, ckf_device.cuh).
template <int F, int WPB, int POL>
__device__ __forceinline__ void evict_bfs_body(Geo g, uint64_t* __restrict__ words, uint8_t* __restrict__ ok,
                                               int64_t* __restrict__ ev, uint64_t* __restrict__ lost,
                                               ckf_record* __restrict__ rec, uint64_t cap, ckf_counters* ctr,
                                               long long* occ, const uint64_t* __restrict__ keys, bool hashed,
                                               uint64_t ibase, unsigned long long* cursor, RoomMap rm) {
  using L = Lanes<F>;
  constexpr int kTpw = L::kTpw;
  constexpr uint32_t kB = WPB * kTpw;
  constexpr uint32_t kLim = kB / 2 ? kB / 2 : 1;
  constexpr uint64_t kAll = kB == 64 ? ~0ull : ((1ull << kB) - 1u);
  const unsigned long long queued = *(volatile unsigned long long*)&ctr->n_queued;
  const uint64_t total = queued < cap ? queued : cap;
  const int lane = threadIdx.x & 31;
  uint32_t n_ok = 0;
  bool have = false, drained = false;
  uint64_t r = 0, i = 0, st = 0, cur_b = 0, cur_tag = 0;
  uint32_t n = 0;
  while (true) {
    // lanes without a chain take the next queue entries
    const unsigned need = __ballot_sync(0xffffffffu, !have && !drained);
    if (need) {
      unsigned long long base = 0;
      const int leader = __ffs(need) - 1;
      if (lane == leader) base = atomicAdd(cursor, (unsigned long long)__popc(need));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (!have && !drained) {
        r = base + __popc(need & ((1u << lane) - 1u));
        if (r < total) {
          i = rec[r].index - ibase;
          uint64_t h = rec[r].lost;  // the key hash parked by the queueing pass, or kRehash
          if (h == kRehash) h = load_hash(keys, i, g.seed, hashed);
          uint64_t fp, i1, i2;
          place<POL>(h, g, fp, i1, i2);
          st = rng_init(g.seed, h, g.worker) + kGolden;
          cur_b = i1;
          cur_tag = fp;
          if (smix(st) & 1u) {
            cur_b = i2;
            cur_tag = make_tag(fp, POL == CKF_POLICY_OFFSET ? 1u : 0u, g);
          }
          n = 1;
          have = true;
        }
      }
      if (base + __popc(need) >= total) drained = true;  // the cursor only grows
    }
    if (!__any_sync(0xffffffffu, have)) break;
    if (!have) continue;
    // ---- one BFS round ----
    bool done = false;
    st += kGolden;
    const uint32_t start = (uint32_t)(smix(st) % kB);
    uint64_t* base_w = words + cur_b * WPB;
    uint64_t cw[WPB];
    ld_bucket_rw<WPB>(base_w, cw);
    uint64_t occm = 0;
#pragma unroll
    for (int q = 0; q < WPB; ++q) {
      const uint64_t z = L::zeros(cw[q]);
#pragma unroll
      for (int s = 0; s < kTpw; ++s)
        if (!((z >> (s * F + F - 1)) & 1u)) occm |= 1ull << (q * kTpw + s);
    }
    const uint64_t rot = start ? (((occm >> start) | (occm << (kB - start))) & kAll) : occm;
    const uint32_t pc = (uint32_t)__popcll(rot);
    const uint32_t cnt = pc < kLim ? pc : kLim;
    if (cnt == 0) {  // drained by concurrent deletes: take a direct slot
      const uint32_t e = empty_lanes<F, WPB>(cw);
      if (try_insert_snap<F, WPB>(words, cur_b, cur_tag, cw) >= 0) {
        rm_filled(rm, cur_b, e);
        done = true;
      }
    } else {
      uint32_t word[kLim], bit[kLim];
      uint64_t rr = rot;
#pragma unroll
      for (uint32_t c = 0; c < kLim; ++c) {
        word[c] = bit[c] = 0;
        if (c >= cnt) continue;
        uint32_t sl = (uint32_t)(__ffsll((long long)rr) - 1) + start;
        sl = sl >= kB ? sl - kB : sl;
        rr &= rr - 1;
        const uint64_t ct = L::get(snap_word<WPB>(cw, sl / kTpw), sl % kTpw);
        uint64_t tc;
        const uint64_t ab = alt_index<POL>(cur_b, tag_fp(ct, g), tag_choice(ct, g), g, tc);
        word[c] = __ldcg(rm.bits + (ab >> 5));
        bit[c] = (uint32_t)(ab & 31);
      }
      uint32_t roomm = 0;
#pragma unroll
      for (uint32_t c = 0; c < kLim; ++c) roomm |= ((word[c] >> bit[c]) & 1u) << c;
      const uint32_t chosen = roomm ? (uint32_t)(__ffs((int)roomm) - 1) : cnt - 1;
      const uint32_t os = nth_candidate<kB>(rot, chosen, start);
      const uint64_t ow = snap_word<WPB>(cw, os / kTpw);
      const uint64_t otag = L::get(ow, os % kTpw);
      uint64_t tc;
      const uint64_t cfp = tag_fp(otag, g);
      const uint64_t alt_b = alt_index<POL>(cur_b, cfp, tag_choice(otag, g), g, tc);
      const uint64_t alt_tag = make_tag(cfp, tc, g);
      if (roomm) {
        // two-step relocation: copy the candidate out, then swap ourselves in
        uint64_t aw[WPB];
        ld_bucket_rw<WPB>(words + alt_b * WPB, aw);
        const uint32_t e = empty_lanes<F, WPB>(aw);
        const int aslot = try_insert_snap<F, WPB>(words, alt_b, alt_tag, aw);
        if (aslot < 0) {
          rm_filled(rm, alt_b, 0);  // the free lane raced away (a stale map bit)
        } else {
          rm_filled(rm, alt_b, e);
          fault_origin_writer<F>(base_w + os / kTpw, os % kTpw, otag);
          if (lane_cas_from<F>(base_w + os / kTpw, os % kTpw, otag, cur_tag, ow)) {
            done = true;
          } else {
            lane_cas<F>(words + alt_b * WPB + aslot / kTpw, aslot % kTpw, alt_tag, 0);  // rollback
            rm_freed(rm, alt_b);
          }
        }
      } else if (lane_cas_from<F>(base_w + os / kTpw, os % kTpw, otag, cur_tag, ow)) {
        // nobody has room: evict the last candidate and deepen (K:427-434)
        cur_b = alt_b;
        cur_tag = alt_tag;
      }
    }
    const bool failed = !done && n >= g.max_evictions;
    if (done || failed) {
      const uint64_t lf = failed ? tag_fp(cur_tag, g) : 0;
      rec[r] = ckf_record{i + ibase, lf, failed ? g.max_evictions : n, done ? 1u : 0u};
      n_ok += done;
      if (failed) ok[i] = 0;
      if (ev) ev[i] = failed ? g.max_evictions : n;
      if (lost) lost[i] = lf;
      have = false;
    } else {
      ++n;
    }
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) ctr->n_records = total;
  block_count_add(n_ok, 0, ctr, occ, +1);
}

template <int F, int WPB, int POL>
__global__ void __launch_bounds__(kBlock, kEvictBlocks)
    evict_bfs_kernel(Geo g, uint64_t* __restrict__ words, uint8_t* __restrict__ ok, int64_t* __restrict__ ev,
                     uint64_t* __restrict__ lost, ckf_record* __restrict__ rec, uint64_t cap, ckf_counters* ctr,
                     long long* occ, const uint64_t* __restrict__ keys, bool hashed, uint64_t ibase,
                     unsigned long long* cursor, RoomMap rm) {
  evict_bfs_body<F, WPB, POL>(g, words, ok, ev, lost, rec, cap, ctr, occ, keys, hashed, ibase, cursor, rm);
}

// Direct-path eviction in one launch: room_scan_kernel decided on the device
// whether the room map was worth building (gate) -- BFS rounds with the map
// and queue refill, or one chain per thread.
template <int F, int WPB, int POL>
__global__ void __launch_bounds__(kBlock, kEvictBlocks)
    evict_direct_kernel(Geo g, uint64_t* __restrict__ words, uint8_t* __restrict__ ok, int64_t* __restrict__ ev,
                        uint64_t* __restrict__ lost, ckf_record* __restrict__ rec, uint64_t cap, ckf_counters* ctr,
                        long long* occ, const uint64_t* __restrict__ keys, bool hashed, unsigned long long* cursor,
                        RoomMap rm, const unsigned long long* gate) {
  if (*gate)
    evict_bfs_body<F, WPB, POL>(g, words, ok, ev, lost, rec, cap, ctr, occ, keys, hashed, 0, cursor, rm);
  else
    evict_chains_body<F, WPB, POL>(g, words, ok, ev, lost, rec, cap, ctr, occ, keys, hashed, 0, nullptr,
                                   RoomMap{nullptr});
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
    const uint64_t h = load_hash(keys, i, g.seed, hashed);
    if (hashed && foreign(g, h)) {  // padding of the sharded exchange
      out[i] = 0;
      continue;
    }
    place<POL>(h, g, fp, i1, i2);
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

// Mixed batch (BASELINE configs[4]): one launch in which key i runs ops[i] --
// CKF_OP_QUERY / CKF_OP_INSERT / CKF_OP_DELETE -- concurrently with the
// others.  This steps outside the reference's phase contract (filter.py:9-15:
// queries must not overlap mutations), so lookups read both buckets with
// COHERENT loads (ld.relaxed.gpu, served by L2 where the CASes commit); a
// lookup's answer is exact for keys whose membership the batch does not change
// (SURVEY.md §7 hard part 6).  Inserts whose pair is full are queued for the
// eviction pass like insert_kernel's; out[i] = hit / stored / deleted.
template <int F, int WPB, int POL>
__device__ __forceinline__ bool find_coherent(const uint64_t* words, uint64_t bucket, uint64_t fp, const Geo& g) {
  using L = Lanes<F>;
  const uint64_t keep = POL == CKF_POLICY_OFFSET ? ~L::kHigh : ~0ull;
  const uint64_t pat = L::bcast(fp);
  if constexpr (WPB > 0) {
    uint64_t w[WPB];
    ld_bucket_rw<WPB>(words + bucket * WPB, w);
    uint64_t any = 0;
#pragma unroll
    for (int j = 0; j < WPB; ++j) any |= L::zeros((w[j] & keep) ^ pat);
    return any != 0;
  } else {
    for (uint32_t j = 0; j < g.wpb; ++j)
      if (L::zeros((ld_word_rw(words + bucket * g.wpb + j) & keep) ^ pat)) return true;
    return false;
  }
}

template <int F, int WPB, int POL>
__global__ void __launch_bounds__(kBlock) mixed_kernel(Geo g, uint64_t* __restrict__ words,
                                                       const uint8_t* __restrict__ ops,
                                                       const uint64_t* __restrict__ keys, uint64_t n,
                                                       uint8_t* __restrict__ out, ckf_record* __restrict__ rec,
                                                       uint64_t cap, ckf_counters* ctr, long long* occ, bool hashed) {
  uint32_t n_ins = 0, n_del = 0, n_alt = 0;
  const int lane_id = threadIdx.x & 31;
  for (uint64_t t0 = blockIdx.x * (uint64_t)kBlock; t0 < n; t0 += (uint64_t)gridDim.x * kBlock) {
    const uint64_t i = t0 + threadIdx.x;
    bool need = false;
    uint64_t h = 0, fp = 0, i1 = 0, i2 = 0;
    if (i < n) {
      const uint8_t op = ops[i];
      h = load_hash(keys, i, g.seed, hashed);
      place<POL>(h, g, fp, i1, i2);
      const uint64_t tag2 = make_tag(fp, POL == CKF_POLICY_OFFSET ? 1u : 0u, g);
      bool r = false;
      if (hashed && foreign(g, h)) {
        r = false;
      } else if (op == CKF_OP_INSERT) {
        r = try_insert_any<F, WPB>(words, i1, fp, g) >= 0;
        if (!r) {
          ++n_alt;
          r = try_insert_any<F, WPB>(words, i2, tag2, g) >= 0;
        }
        n_ins += r;
        need = !r;
        r = true;  // a queued key stays stored unless the eviction pass fails it
      } else if (op == CKF_OP_DELETE) {
        r = remove_tag_any<F, WPB>(words, i1, fp, g) >= 0;
        if (!r) {
          ++n_alt;
          r = remove_tag_any<F, WPB>(words, i2, POL == CKF_POLICY_OFFSET ? tag2 : fp, g) >= 0;
        }
        n_del += r;
      } else {
        r = find_coherent<F, WPB, POL>(words, i1, fp, g);
        if (!r) {
          ++n_alt;
          r = find_coherent<F, WPB, POL>(words, i2, fp, g);
        }
      }
      out[i] = r;
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
        } else {  // queue overflow: evict in place
          const Outcome o = evict_any<F, WPB, POL>(words, h, fp, i1, i2, g);
          n_ins += o.ok;
          out[i] = (uint8_t)o.ok;
        }
      }
    }
  }
  block_count_add(n_ins, n_alt, ctr, occ, +1);
  block_count_add(n_del, 0, nullptr, occ, -1);
}

// Parity mode: the reference's sequential insert_batch (K:510-529), one
// device thread, same key order, same PRNG stream; bit-identical table.
template <int F, int WPB, int POL>
__global__ void seq_insert_kernel(Geo g, uint64_t* words, const uint64_t* keys, uint64_t n, uint8_t* ok, int64_t* ev,
                                  uint64_t* lost, ckf_record* rec, uint64_t cap, ckf_counters* ctr, long long* occ,
                                  bool hashed) {
  uint64_t n_ok = 0, n_rec = 0;
  for (uint64_t i = 0; i < n; ++i) {
    uint64_t h = hashed ? keys[i] : xxh64(keys[i], g.seed);
    uint64_t fp, i1, i2;
    place<POL>(h, g, fp, i1, i2);
    Outcome o{1u, 0u, 0};
    if (hashed && foreign(g, h)) {  // padding of the sharded exchange
      ok[i] = 1;
      if (ev) ev[i] = 0;
      if (lost) lost[i] = 0;
      continue;
    }
    if (try_insert_any<F, WPB>(words, i1, fp, g) < 0 &&
        try_insert_any<F, WPB>(words, i2, make_tag(fp, POL == CKF_POLICY_OFFSET ? 1u : 0u, g), g) < 0)
      o = evict_any<F, WPB, POL>(words, h, fp, i1, i2, g);
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
    const uint64_t h = hashed ? keys[i] : xxh64(keys[i], g.seed);
    if (hashed && foreign(g, h)) {
      out[i] = 0;
      continue;
    }
    place<POL>(h, g, fp, i1, i2);
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
#ifdef CKF_DEV_F16  // developer build: f=16 only (fast compile)
  if (p->fingerprint_bits == 16) { CKF_CASE_P(16) }
#else
  switch (p->fingerprint_bits) {
    case 8: CKF_CASE_P(8)
    case 16: CKF_CASE_P(16)
    case 32: CKF_CASE_P(32)
  }
#endif
#undef CKF_CASE_P
#undef CKF_CASE_W
  return CKF_EINVAL;
}


// ---------------------------------------------------------------------------
// shared-memory region schedule: plan + workspace layout (see ckf_region.cuh)
// ---------------------------------------------------------------------------

constexpr uint64_t kRegionMinTable = 48ull << 20;  // below this the table is L2-resident anyway
constexpr uint32_t kMaxF2 = 512;                   // fine regions per coarse region (split bins)

static uint64_t align256(uint64_t x) { return (x + 255) & ~255ull; }
static uint64_t direct_rm_bytes(uint64_t m) { return align256((m + 31) / 32 * 4); }

// Developer knobs: CKF_REGION_KB (fine-region bytes), CKF_TILED_AUTO (0
// disables the automatic choice of the region schedule), CKF_MAX_RUN_KEYS (a
// smaller run size, so tests cover calls split into several region runs).
static uint64_t env_u64(const char* name, uint64_t dflt) {
  const char* v = getenv(name);
  return v && *v ? strtoull(v, nullptr, 10) : dflt;
}

struct RLayout {
  uint64_t cnt1, cntf, bin_ctr_end, n_miss, mode, ctr_end, qstart, room, bin1, binf, miss, bits, total;
};

static uint32_t ceil_log2(uint64_t x) {
  uint32_t l = 0;
  while ((1ull << l) < x) ++l;
  return l;
}

constexpr uint32_t kMaxProbeGrid = 1024;

static uint64_t even_cap(double per) { return ((uint64_t)(per + 4.0 * std::sqrt(per) + 64.0) + 1) & ~1ull; }

// Region plan for a call of n keys; ok=false when the schedule does not apply
// to this table.  The plan covers one run of pl.chunk keys; larger calls run
// ceil(n / chunk) of them back to back (the record's index field holds
// 64 - ish bits).
static RPlan make_rplan(const ckf_params* p, uint64_t n, int op, unsigned flags, bool& ok) {
  RPlan pl{};
  ok = false;
  const uint32_t wpb = p->words_per_bucket;
  if (wpb != 1 && wpb != 2 && wpb != 4 && wpb != 8) return pl;
  const uint64_t m = p->bucket_count;
  const uint32_t pb = p->payload_bits;
  if (pb > 32 || m < 2 || m > (1ull << 32) || n == 0) return pl;
  const bool wide = pb > 24;  // f = 32: 16-byte records (RecT)
  const uint64_t bbytes = wpb * 8ull;
  uint32_t lrb = 0;
  const uint64_t smem = env_u64("CKF_REGION_KB", kRegionSmem >> 10) << 10;
  while ((bbytes << (lrb + 1)) <= smem && (bbytes << (lrb + 1)) <= (uint64_t)kRegionSmem) ++lrb;
  const uint32_t lm = ceil_log2(m);
  if (flags & CKF_FORCE_TILED) {  // small forced tables still get >= 16 fine regions
    const uint32_t cap = lm > 4 ? lm - 4 : 1;
    if (lrb > cap) lrb = cap;
  }
  if (lrb < 1) lrb = 1;
  // coarse regions: at most kRMaxCoarse of them, each split into F2 <= kMaxF2 fine ones
  // log2 coarse regions: 2^8 (measured at 2^24 buckets: 2^9 -> 2^8 -> 2^7 coarse
  // bins = 23.5 -> 22.8 -> 22.8 ms/step: longer bin-pass runs, split F2 16),
  // or up to 2^9 when that saves a run (one offset bit less leaves one more
  // index bit in the record)
  const uint64_t per_rec = op == CKF_OP_QUERY ? 2 : 1;
  auto runs_for = [&](uint32_t lrbc_) -> uint64_t {
    if (wide) return 1;
    uint64_t km = (1ull << (64 - (pb + lrbc_ + 1))) - 2;
    if (km > (1ull << 31) / per_rec) km = (1ull << 31) / per_rec;
    return (n + km - 1) / km;
  };
  const uint32_t lc0 = (uint32_t)env_u64("CKF_COARSE_LOG2", 8);
  uint32_t lrbc = lm > lc0 ? lm - lc0 : 0;
  if (lrbc < lrb) lrbc = lrb;
  if (lc0 < 9 && lrbc > lrb && runs_for(lrbc - 1) < runs_for(lrbc)) --lrbc;
  if (lrbc - lrb > ceil_log2(kMaxF2)) return pl;
  const uint64_t R1 = (m + (1ull << lrbc) - 1) >> lrbc;
  if (R1 > (uint64_t)kRMaxCoarse) return pl;
  const uint32_t ish = wide ? 32 : pb + lrbc + 1;  // (unused by 16-byte records)
  if (ish > 62 || (wide && lrbc > 31)) return pl;
  // keys per run: the index field (all-ones is the filler), 32-bit miss-entry
  // indices, and < 2^32 record slots over the coarse bins (dual query records)
  uint64_t kmax = wide ? ~0ull : (1ull << (64 - ish)) - 2;
  if (kmax > (1ull << 31) / per_rec) kmax = (1ull << 31) / per_rec;
  const uint64_t kenv = env_u64("CKF_MAX_RUN_KEYS", 0);  // developer knob: exercise multi-run calls
  if (kenv && kenv < kmax) kmax = kenv;
  const uint64_t runs = (n + kmax - 1) / kmax;
  pl.chunk = (n + runs - 1) / runs;
  pl.lrb = lrb;
  pl.lrbc = lrbc;
  pl.F2 = 1u << (lrbc - lrb);
  pl.R1 = (uint32_t)R1;
  pl.R = pl.R1 * pl.F2;
  pl.pb = pb;
  pl.ish = ish;
  pl.rbytes = wide ? 16 : 8;
  const double recs = (double)pl.chunk * (double)per_rec;
  // + run padding: at most one filler per bin per tile of the pass that fills it
  // (bin: ceil(chunk / tile) tiles + one partial tile per miss segment; split: a coarse bin's tiles)
  const uint64_t tiles1 = (pl.chunk + kBTile - 1) / kBTile + (uint64_t)kMaxProbeGrid;
  pl.cap1 = (even_cap(recs / pl.R1) + tiles1 + 1) & ~1ull;
  pl.capf = (even_cap(recs / pl.R) + (pl.cap1 + kBTile - 1) / kBTile + 1) & ~1ull;
  if ((uint64_t)pl.R1 * pl.cap1 >= 0xFFFFFFFFull) return pl;  // coalesced bin writer: 32-bit slots
  ok = true;
  return pl;
}

// one persistent probe CTA per SM (fewer if there are fewer regions)
static uint32_t probe_grid(const RPlan& pl) {
  uint32_t gsz = (uint32_t)sm_count();
  if (gsz > kMaxProbeGrid) gsz = kMaxProbeGrid;
  return pl.R < gsz ? pl.R : gsz;
}
// a probe CTA's miss segment holds every record of its regions
static uint64_t miss_seg(const RPlan& pl) {
  const uint32_t gsz = probe_grid(pl);
  return (uint64_t)((pl.R + gsz - 1) / gsz) * pl.capf;
}

static RLayout rlayout_for(const RPlan& pl, int op) {
  RLayout L{};
  const uint64_t cs = (uint64_t)kCntStride * 4;
  L.cnt1 = 0;
  L.cntf = align256(L.cnt1 + pl.R1 * cs);
  L.bin_ctr_end = align256(L.cntf + pl.R * cs);  // bin counters: zeroed again between the phases
  L.n_miss = L.bin_ctr_end;
  L.mode = L.n_miss + 4ull * kMaxProbeGrid;
  L.ctr_end = align256(L.mode + 8);
  L.qstart = L.ctr_end;  // insert: eviction-queue length before this run (not zeroed per run)
  L.room = align256(L.qstart + 16);  // insert: [qstart, eviction cursor], then the room bit per bucket
  L.bin1 = align256(L.room + (op == CKF_OP_INSERT ? ((uint64_t)pl.R << pl.lrb) / 8 : 0));
  L.binf = align256(L.bin1 + pl.R1 * pl.cap1 * pl.rbytes);
  L.miss = align256(L.binf + pl.R * pl.capf * pl.rbytes);
  L.bits = align256(L.miss + probe_grid(pl) * miss_seg(pl) * 16);
  L.total = align256(L.bits + (op == CKF_OP_INSERT ? 0 : (pl.chunk + 31) / 32 * 4));
  return L;
}

static RWork rwork_view(void* ws, const RLayout& L, const RPlan& pl) {
  char* b = (char*)ws;
  RWork w{};
  w.cnt1 = (uint32_t*)(b + L.cnt1);
  w.cntf = (uint32_t*)(b + L.cntf);
  w.n_miss = (uint32_t*)(b + L.n_miss);
  w.mode = (uint32_t*)(b + L.mode);
  w.bin1 = b + L.bin1;
  w.binf = b + L.binf;
  w.miss = (uint4*)(b + L.miss);
  w.bits = (uint32_t*)(b + L.bits);
  w.room = (uint32_t*)(b + L.room);
  w.seg = miss_seg(pl);
  return w;
}

// Opt a kernel into > 48 KiB of dynamic shared memory, once per kernel
// instance and device (the template parameter makes the flag per instance).
template <auto Kernel>
static void allow_big_smem(uint32_t bytes) {
  static bool done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !done[dev]) {
    cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    done[dev] = true;
  }
}

// Region run of one op over n <= pl.chunk keys: bin, split, probe on the
// primary buckets; bin, split, probe the misses on their alternate buckets;
// (+ bit expansion).
template <int OP, int F, int WPB, int POL>
static int run_region(const Geo& g, const RPlan& pl, const RLayout& L, void* ws, uint64_t* words,
                      const uint64_t* keys, uint64_t n, bool hashed, Sink sk, long long* occ, uint8_t* out,
                      cudaStream_t s) {
  RWork w = rwork_view(ws, L, pl);
  if (cudaMemsetAsync(ws, 0, L.ctr_end, s) != cudaSuccess) return cuda_error();  // bin + miss counters
  if (OP == OP_QUERY) {  // starting value of the results from a sample of the batch
    region_sample_kernel<F, WPB, POL><<<kSample / 256, 256, 0, s>>>(g, words, keys, n, hashed, w.mode);
    int st0 = status();
    if (st0) return st0;
    fill_bits_kernel<<<grid_for((n + 31) / 32, 256, 8), 256, 0, s>>>(w.bits, (n + 31) / 32, n, w.mode);
    if ((st0 = status())) return st0;
    sk.bits = w.bits;
  } else if (OP == OP_DELETE) {  // all-true: only keys found in neither bucket clear their bit
    if (cudaMemsetAsync(w.mode, 1, 4, s) != cudaSuccess) return cuda_error();
    if (cudaMemsetAsync(w.bits, 0xFF, (n + 31) / 32 * 4, s) != cudaSuccess) return cuda_error();
    sk.bits = w.bits;
  }
  sk.keys = keys;
  sk.hashed = hashed;
  long long* mocc = OP == OP_QUERY ? nullptr : occ;
  const int sms = sm_count();
  const unsigned pg = probe_grid(pl);
  constexpr uint32_t kBinSmem = sizeof(BinSmem<F>);
  constexpr uint32_t kProbeSmemF = kProbeSmem<F>;
  allow_big_smem<region_bin_kernel<OP, F, WPB, POL, SRC_KEYS>>(kBinSmem);
  if constexpr (OP == OP_QUERY) allow_big_smem<region_bin_kernel<OP, F, WPB, POL, SRC_KEYS_DUAL>>(kBinSmem);
  allow_big_smem<region_bin_kernel<OP, F, WPB, POL, SRC_MISS>>(kBinSmem);
  allow_big_smem<region_split_kernel<OP, F, WPB, POL>>(kBinSmem);
  allow_big_smem<region_probe_kernel<OP, F, WPB, POL, 1>>(kProbeSmemF);
  allow_big_smem<region_probe_kernel<OP, F, WPB, POL, 2>>(kProbeSmemF);
  if constexpr (OP == OP_QUERY) {
    allow_big_smem<region_probe_kernel<OP, F, WPB, POL, 1, 0>>(kProbeSmemF);
    allow_big_smem<region_probe_kernel<OP, F, WPB, POL, 2, 0>>(kProbeSmemF);
  }
  int st;
  // phase 1: primary buckets
  region_bin_kernel<OP, F, WPB, POL, SRC_KEYS><<<grid_for(n, kBTile, kBinBlocks), kBThreads, kBinSmem, s>>>(
      g, pl, words, keys, n, hashed, w, sk, mocc);
  if ((st = status())) return st;
  if constexpr (OP == OP_QUERY) {  // (exits unless the sample chose dual records)
    region_bin_kernel<OP, F, WPB, POL, SRC_KEYS_DUAL><<<grid_for(n, kBTile, kBinBlocks), kBThreads, kBinSmem, s>>>(
        g, pl, words, keys, n, hashed, w, sk, mocc);
    if ((st = status())) return st;
  }
  region_split_kernel<OP, F, WPB, POL><<<sms * kSplitBlocks, kBThreads, kBinSmem, s>>>(g, pl, words, w, sk, mocc);
  if ((st = status())) return st;
  region_probe_kernel<OP, F, WPB, POL, 1><<<pg, kPThreads, kProbeSmemF, s>>>(g, pl, words, w, sk, mocc);
  if ((st = status())) return st;
  if constexpr (OP == OP_QUERY) {  // (exits unless the results start all-false)
    region_probe_kernel<OP, F, WPB, POL, 1, 0><<<pg, kPThreads, kProbeSmemF, s>>>(g, pl, words, w, sk, mocc);
    if ((st = status())) return st;
  }
  // phase 2: the misses, on their alternate buckets
  if (cudaMemsetAsync(ws, 0, L.bin_ctr_end, s) != cudaSuccess) return cuda_error();
  region_bin_kernel<OP, F, WPB, POL, SRC_MISS><<<dim3((sms * kBinBlocks + pg - 1) / pg, pg), kBThreads, kBinSmem, s>>>(
      g, pl, words, keys, 0, hashed, w, sk, mocc);
  if ((st = status())) return st;
  region_split_kernel<OP, F, WPB, POL><<<sms * kSplitBlocks, kBThreads, kBinSmem, s>>>(g, pl, words, w, sk, mocc);
  if ((st = status())) return st;
  region_probe_kernel<OP, F, WPB, POL, 2><<<pg, kPThreads, kProbeSmemF, s>>>(g, pl, words, w, sk, mocc);
  if ((st = status())) return st;
  if constexpr (OP == OP_QUERY) {
    region_probe_kernel<OP, F, WPB, POL, 2, 0><<<pg, kPThreads, kProbeSmemF, s>>>(g, pl, words, w, sk, mocc);
    if ((st = status())) return st;
  }
  if (OP != OP_INSERT) {
    expand_count_kernel<<<grid_for((n + 31) / 32, 256, 8), 256, 0, s>>>(w.bits, n, out,
                                                                       OP == OP_QUERY ? sk.ctr : nullptr);
    st = status();
  }
  return st;
}

struct TiledArgs {
  bool region;  // shared-memory region schedule (ckf_region.cuh)
  RPlan rpl;
  RLayout RL;
  void* ws;
  bool direct_rm;  // direct insert: ws holds a room map + eviction cursor (direct_ws_bytes)
};

// the call's keys in runs of at most pl.chunk: (offset, count) of run k
static inline uint64_t run_count(const TiledArgs& t, uint64_t n) { return (n + t.rpl.chunk - 1) / t.rpl.chunk; }
static inline void run_span(const TiledArgs& t, uint64_t n, uint64_t k, uint64_t& off, uint64_t& cnt) {
  off = k * t.rpl.chunk;
  cnt = n - off < t.rpl.chunk ? n - off : t.rpl.chunk;
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
  TiledArgs t;
};

template <int F, int WPB, int POL>
struct QueryOp {
  static int run(const QueryArgs& a) {
    if constexpr (WPB == 1 || WPB == 2 || WPB == 4 || WPB == 8) {
      if (a.t.region) {
        for (uint64_t k = 0, nr = run_count(a.t, a.n); k < nr; ++k) {
          uint64_t off, cnt;
          run_span(a.t, a.n, k, off, cnt);
          Sink sk{nullptr, nullptr, 0, a.ctr, nullptr, nullptr, false, off};
          const int st = run_region<OP_QUERY, F, WPB, POL>(a.g, a.t.rpl, a.t.RL, a.t.ws, const_cast<uint64_t*>(a.words),
                                                           a.keys + off, cnt, a.hashed, sk, nullptr, a.out + off, a.s);
          if (st) return st;
        }
        return CKF_OK;
      }
    }
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
  TiledArgs t;
};

template <int F, int WPB, int POL>
static int launch_evict(const InsertArgs& a, uint64_t off, const unsigned long long* qstart, RoomMap rm,
                        unsigned long long* cursor = nullptr) {
  // the queue length is only known on the device: a fixed full-residency grid
  // strides over it (empty queues exit immediately)
  const unsigned egrid = (unsigned)sm_count() * kEvictBlocks;
  if constexpr (WPB > 0) {
    if (rm.bits && cursor && a.g.eviction == CKF_EVICT_BFS && !getenv("CKF_EVICT_CHAINS")) {
      if (cudaMemcpyAsync(cursor, qstart, 8, cudaMemcpyDeviceToDevice, a.s) != cudaSuccess) return cuda_error();
      evict_bfs_kernel<F, WPB, POL><<<egrid, kBlock, 0, a.s>>>(a.g, a.words, a.ok + off, a.ev ? a.ev + off : nullptr,
                                                               a.lost ? a.lost + off : nullptr, a.rec, a.cap, a.ctr,
                                                               a.occ, a.keys + off, a.hashed, off, cursor, rm);
      return status();
    }
  }
  evict_kernel<F, WPB, POL><<<egrid, kBlock, 0, a.s>>>(a.g, a.words, a.ok + off, a.ev ? a.ev + off : nullptr,
                                                       a.lost ? a.lost + off : nullptr, a.rec, a.cap, a.ctr, a.occ,
                                                       a.keys + off, a.hashed, off, qstart, rm);
  return status();
}

template <int F, int WPB, int POL>
struct InsertOp {
  static int run(const InsertArgs& a) {
    if (a.sequential) {
      seq_insert_kernel<F, WPB, POL><<<1, 1, 0, a.s>>>(a.g, a.words, a.keys, a.n, a.ok, a.ev, a.lost, a.rec, a.cap, a.ctr,
                                                   a.occ, a.hashed);
      return status();
    }
    if constexpr (WPB == 1 || WPB == 2 || WPB == 4 || WPB == 8) {
      if (a.t.region && a.cap) {
        // every key counts as stored until the eviction pass says otherwise
        if (cudaMemsetAsync(a.ok, 1, a.n, a.s) != cudaSuccess) return cuda_error();
        if (a.ev && cudaMemsetAsync(a.ev, 0, a.n * 8, a.s) != cudaSuccess) return cuda_error();
        if (a.lost && cudaMemsetAsync(a.lost, 0, a.n * 8, a.s) != cudaSuccess) return cuda_error();
        unsigned long long* qstart = (unsigned long long*)((char*)a.t.ws + a.t.RL.qstart);
        for (uint64_t k = 0, nr = run_count(a.t, a.n); k < nr; ++k) {
          uint64_t off, cnt;
          run_span(a.t, a.n, k, off, cnt);
          // this run's eviction queue starts where the previous runs' ended
          if (cudaMemcpyAsync(qstart, &a.ctr->n_queued, 8, cudaMemcpyDeviceToDevice, a.s) != cudaSuccess)
            return cuda_error();
          Sink sk{nullptr, a.rec, a.cap, a.ctr, a.ok + off, nullptr, false, off};
          int st = run_region<OP_INSERT, F, WPB, POL>(a.g, a.t.rpl, a.t.RL, a.t.ws, a.words, a.keys + off, cnt, a.hashed,
                                                      sk, a.occ, nullptr, a.s);
          if (st) return st;
          const RWork w = rwork_view(a.t.ws, a.t.RL, a.t.rpl);
          const RoomMap rm{getenv("CKF_NO_ROOM_MAP") ? nullptr : w.room};
          if ((st = launch_evict<F, WPB, POL>(a, off, qstart, rm, qstart + 1))) return st;
        }
        return CKF_OK;
      }
    }
    unsigned grid = grid_for(a.n, kBlock, 16);
    insert_kernel<F, WPB, POL><<<grid, kBlock, 0, a.s>>>(a.g, a.words, a.keys, a.n, a.ok, a.ev, a.lost, a.rec,
                                                         a.cap, a.ctr, a.occ, a.hashed);
    int st = status();
    if (st) return st;
    if (!a.cap) return CKF_OK;
    if constexpr (WPB == 2 || WPB == 4 || WPB == 8) {
      if (a.t.direct_rm && a.g.eviction == CKF_EVICT_BFS) {
        // room map of the filled table + BFS eviction one round per lane, as
        // on the region schedule -- when the queue is long enough (the scan
        // decides on the device, sets the gate evict_direct_kernel branches
        // on, and zeroes the cursor)
        uint32_t* bits = (uint32_t*)a.t.ws;
        unsigned long long* cur = (unsigned long long*)((char*)a.t.ws + direct_rm_bytes(a.g.m));
        const uint64_t nw = (a.g.m + 31) / 32;
        const unsigned eg = (unsigned)sm_count() * kEvictBlocks;
        room_scan_kernel<F, WPB><<<grid_for(nw * 32, kBlock, 16), kBlock, 0, a.s>>>(a.words, a.g.m, bits, cur,
                                                                                    a.ctr, cur + 1);
        if ((st = status())) return st;
        evict_direct_kernel<F, WPB, POL><<<eg, kBlock, 0, a.s>>>(a.g, a.words, a.ok, a.ev, a.lost, a.rec, a.cap,
                                                                 a.ctr, a.occ, a.keys, a.hashed, cur, RoomMap{bits},
                                                                 cur + 1);
        return status();
      }
    }
    return launch_evict<F, WPB, POL>(a, 0, nullptr, RoomMap{nullptr});
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
  TiledArgs t;
};

template <int F, int WPB, int POL>
struct DeleteOp {
  static int run(const DeleteArgs& a) {
    if (a.sequential) {
      seq_delete_kernel<F, POL><<<1, 1, 0, a.s>>>(a.g, a.words, a.keys, a.n, a.out, a.ctr, a.occ, a.hashed);
      return status();
    }
    if constexpr (WPB == 1 || WPB == 2 || WPB == 4 || WPB == 8) {
      if (a.t.region) {
        for (uint64_t k = 0, nr = run_count(a.t, a.n); k < nr; ++k) {
          uint64_t off, cnt;
          run_span(a.t, a.n, k, off, cnt);
          Sink sk{nullptr, nullptr, 0, a.ctr, nullptr, nullptr, false, off};
          const int st = run_region<OP_DELETE, F, WPB, POL>(a.g, a.t.rpl, a.t.RL, a.t.ws, a.words, a.keys + off, cnt,
                                                            a.hashed, sk, a.occ, a.out + off, a.s);
          if (st) return st;
        }
        return CKF_OK;
      }
    }
    unsigned grid = grid_for(a.n, kBlock, 16);
    delete_kernel<F, WPB, POL><<<grid, kBlock, 0, a.s>>>(a.g, a.words, a.keys, a.n, a.out, a.ctr, a.occ, a.hashed);
    return status();
  }
};

struct MixedArgs {
  Geo g;
  uint64_t* words;
  const uint8_t* ops;
  const uint64_t* keys;
  uint64_t n;
  uint8_t* out;
  ckf_record* rec;
  uint64_t cap;
  ckf_counters* ctr;
  long long* occ;
  bool hashed;
  cudaStream_t s;
};

template <int F, int WPB, int POL>
struct MixedOp {
  static int run(const MixedArgs& a) {
    mixed_kernel<F, WPB, POL><<<grid_for(a.n, kBlock, 16), kBlock, 0, a.s>>>(a.g, a.words, a.ops, a.keys, a.n, a.out,
                                                                         a.rec, a.cap, a.ctr, a.occ, a.hashed);
    int st = status();
    if (st || !a.cap) return st;
    evict_kernel<F, WPB, POL><<<(unsigned)sm_count() * kEvictBlocks, kBlock, 0, a.s>>>(
        a.g, a.words, a.out, nullptr, nullptr, a.rec, a.cap, a.ctr, a.occ, a.keys, a.hashed, 0, nullptr,
        RoomMap{nullptr});
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

// ---------------------------------------------------------------------------
// multi-GPU routing: stable partition of key hashes by owning shard
// ---------------------------------------------------------------------------
//
// shard(h) = (h >> shift) & (G - 1), G <= 8 (one node).  Stable: shard s's
// hashes leave in arrival order, so each shard sees exactly the key stream a
// reference filter of m/G buckets would (sharded.py).  Three passes over
// 4096-hash tiles (thread t owns 16 consecutive hashes of its tile): count per
// (tile, shard), one-block scan to (tile, shard) offsets, scatter.  order[p] =
// source index of send[p] (the return path's inverse permutation).

constexpr int kRtThreads = 256, kRtItems = 16, kRtTile = kRtThreads * kRtItems;

__global__ void __launch_bounds__(kRtThreads) route_count_kernel(const uint64_t* __restrict__ h, uint64_t n,
                                                                 uint32_t shift, uint32_t gmask,
                                                                 uint32_t* __restrict__ tile_counts) {
  __shared__ uint32_t s_cnt[8];
  if (threadIdx.x < 8) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  uint64_t c = 0;  // counts only: coalesced strided items (order does not matter here)
#pragma unroll
  for (int k = 0; k < kRtItems; ++k) {
    const uint64_t i = blockIdx.x * (uint64_t)kRtTile + k * kRtThreads + threadIdx.x;
    if (i < n) c += 1ull << (8 * ((h[i] >> shift) & gmask));
  }
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const uint32_t v = __reduce_add_sync(0xffffffffu, (uint32_t)(c >> (8 * s)) & 0xFFu);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&s_cnt[s], v);
  }
  __syncthreads();
  if (threadIdx.x <= gmask) tile_counts[blockIdx.x * (uint64_t)(gmask + 1) + threadIdx.x] = s_cnt[threadIdx.x];
}

// one block: offs[t * G + s] = base[s] + sum_{t' < t} counts[t' * G + s];
// shard_counts[s] = total of s.  Shards are scanned one after the other.
// cap != 0 (fixed-capacity exchange): shard s's run starts at s * cap.
__global__ void __launch_bounds__(1024) route_scan_kernel(const uint32_t* __restrict__ tile_counts, uint64_t ntiles,
                                                          uint32_t G, uint64_t* __restrict__ offs,
                                                          long long* __restrict__ shard_counts, uint64_t cap) {
  __shared__ uint64_t wprefix[32];
  __shared__ uint64_t s_total, s_base;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x / 32;
  const uint64_t per = (ntiles + blockDim.x - 1) / blockDim.x;
  const uint64_t lo = min((uint64_t)tid * per, ntiles), hi = min(lo + per, ntiles);
  if (tid == 0) s_base = 0;
  for (uint32_t s = 0; s < G; ++s) {
    uint64_t sum = 0;
    for (uint64_t t = lo; t < hi; ++t) sum += tile_counts[t * G + s];
    uint64_t x = sum;  // inclusive warp scan
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    __syncthreads();
    if (lane == 31) wprefix[wid] = x;
    __syncthreads();
    if (wid == 0) {
      const uint64_t v = lane < nw ? wprefix[lane] : 0;
      uint64_t t = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, t, d);
        if (lane >= d) t += y;
      }
      if (lane < nw) wprefix[lane] = t - v;
      if (lane == 31) s_total = t;
    }
    __syncthreads();
    uint64_t run = (cap ? s * cap : s_base) + wprefix[wid] + x - sum;
    for (uint64_t t = lo; t < hi; ++t) {
      offs[t * G + s] = run;
      run += tile_counts[t * G + s];
    }
    __syncthreads();
    if (tid == 0) {
      shard_counts[s] = (long long)s_total;
      s_base += s_total;
    }
  }
}

// Scatter, staged through shared memory so every shard's run leaves as
// coalesced stores: the tile is loaded coalesced (padded: thread t's 16
// hashes start 17 words apart, no bank conflicts), each hash is placed at its
// stable position inside the tile's shard-sorted layout, then the runs are
// copied out.
constexpr int kRtPad = kRtTile + kRtTile / kRtItems;  // one pad word per 16
constexpr uint32_t kRouteSmem = (uint32_t)(kRtPad * 8 + kRtTile * 8 + kRtTile * 8);

__global__ void __launch_bounds__(kRtThreads, 2) route_scatter_kernel(const uint64_t* __restrict__ h, uint64_t n,
                                                                      uint32_t shift, uint32_t gmask,
                                                                      const uint64_t* __restrict__ offs,
                                                                      uint64_t* __restrict__ send,
                                                                      long long* __restrict__ order, uint64_t cap,
                                                                      unsigned long long* spilled) {
  extern __shared__ __align__(16) uint64_t rsm[];
  uint64_t* hin = rsm;                          // [kRtPad] tile, padded
  uint64_t* hout = rsm + kRtPad;                // [kRtTile] shard-sorted hashes
  long long* oout = (long long*)(hout + kRtTile);  // [kRtTile] their source indices
  __shared__ uint64_t s_w[2][kRtThreads / 32];
  __shared__ uint32_t s_start[9];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t t0 = blockIdx.x * (uint64_t)kRtTile;
  const uint32_t tn = (uint32_t)min((uint64_t)kRtTile, n - t0);
  for (uint32_t j = tid; j < tn; j += kRtThreads) hin[j + j / kRtItems] = h[t0 + j];
  __syncthreads();
  uint8_t sh[kRtItems];
  uint64_t c8 = 0;
#pragma unroll
  for (int k = 0; k < kRtItems; ++k) {
    const uint32_t j = tid * kRtItems + k;
    sh[k] = j < tn ? (uint8_t)((hin[j + j / kRtItems] >> shift) & gmask) : 0xFF;
    if (sh[k] != 0xFF) c8 += 1ull << (8 * sh[k]);
  }
  uint64_t c0 = 0, c1 = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    c0 |= ((c8 >> (8 * q)) & 0xFFull) << (16 * q);
    c1 |= ((c8 >> (8 * (q + 4))) & 0xFFull) << (16 * q);
  }
  uint64_t x0 = c0, x1 = c1;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t y0 = __shfl_up_sync(0xffffffffu, x0, d), y1 = __shfl_up_sync(0xffffffffu, x1, d);
    if (lane >= d) {
      x0 += y0;
      x1 += y1;
    }
  }
  if (lane == 31) {
    s_w[0][wid] = x0;
    s_w[1][wid] = x1;
  }
  __syncthreads();
  uint64_t p0 = x0 - c0, p1 = x1 - c1, t0s = 0, t1s = 0;  // my prefix; tile totals
#pragma unroll
  for (int k = 0; k < kRtThreads / 32; ++k) {
    if (k < wid) {
      p0 += s_w[0][k];
      p1 += s_w[1][k];
    }
    t0s += s_w[0][k];
    t1s += s_w[1][k];
  }
  uint32_t start[9];  // shard runs inside the tile's sorted layout
  start[0] = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) start[q + 1] = start[q] + ((uint32_t)((q < 4 ? t0s : t1s) >> (16 * (q & 3))) & 0xFFFFu);
  if (tid < 9) s_start[tid] = start[tid];
  uint32_t next[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) next[q] = start[q] + ((uint32_t)((q < 4 ? p0 : p1) >> (16 * (q & 3))) & 0xFFFFu);
#pragma unroll
  for (int k = 0; k < kRtItems; ++k) {
    if (sh[k] == 0xFF) continue;
    uint32_t r = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (sh[k] == q) r = next[q]++;
    const uint32_t j = tid * kRtItems + k;
    hout[r] = hin[j + j / kRtItems];
    oout[r] = (long long)(t0 + j);
  }
  __syncthreads();
  const uint64_t* tb = offs + blockIdx.x * (uint64_t)(gmask + 1);
  for (uint32_t p = tid; p < tn; p += kRtThreads) {
    uint32_t q = 0;
#pragma unroll
    for (int k = 1; k < 8; ++k)
      if (p >= s_start[k]) q = k;
    const uint64_t pos = tb[q] + (p - s_start[q]);
    if (cap && pos - (uint64_t)q * cap >= cap) {  // past the shard's capacity: not sent
      atomicAdd(spilled, 1ull);
      continue;
    }
    send[pos] = hout[p];
    order[pos] = oout[p];
  }
}

// Padding of the fixed-capacity exchange: the unused tail of shard s's block
// gets a hash owned by shard (s+1) % G (skipped by the receiver) and order -1.
__global__ void __launch_bounds__(256) route_fill_kernel(uint64_t* __restrict__ send, long long* __restrict__ order,
                                                         const long long* __restrict__ shard_counts, uint32_t G,
                                                         uint64_t cap, uint32_t shift) {
  __shared__ uint64_t s_cnt[256];
  for (uint32_t s = threadIdx.x; s < G; s += blockDim.x) s_cnt[s] = (uint64_t)shard_counts[s];
  __syncthreads();
  const uint64_t total = (uint64_t)G * cap;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t s = (uint32_t)(i / cap);
    if (i - (uint64_t)s * cap >= s_cnt[s]) {
      send[i] = (uint64_t)((s + 1) & (G - 1)) << shift;
      order[i] = -1;
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) route_unpermute_kernel(const T* __restrict__ back,
                                                              const long long* __restrict__ order, uint64_t n,
                                                              T* __restrict__ out) {
  for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < n; p += (uint64_t)gridDim.x * blockDim.x) {
    const long long o = order[p];
    if (o >= 0) out[o] = back[p];
  }
}

// ---------------------------------------------------------------------------
// k-mer ingestion (reference kmer.py:48-95)
// ---------------------------------------------------------------------------
//
// `seq` holds the records' sequence bytes with a separator byte between
// records.  A window of k bases is emitted iff none of its bytes is outside
// ACGTacgt (separators, N, ...), packed two bits per base with the leftmost
// base most significant -- the reference's rolling `value = (value << 2 |
// code) & mask` with `fill` reset on an ambiguous base.  Two passes over
// kKmerChunk-position chunks (count, then emit at scanned offsets) keep the
// output in sequence order.

constexpr uint32_t kKmerChunk = 1024;

__device__ __forceinline__ uint32_t base_code(uint8_t c) {
  // A C G T (either case) -> 0..3, anything else -> 4
  const uint8_t u = c & 0xDF;
  return u == 'A' ? 0u : u == 'C' ? 1u : u == 'G' ? 2u : u == 'T' ? 3u : 4u;
}

// EMIT = false: counts[c] = windows ending in chunk c; true: write them at offs[c]
template <bool EMIT>
__global__ void __launch_bounds__(256) kmer_chunk_kernel(const uint8_t* __restrict__ seq, uint64_t len, uint32_t k,
                                                         uint32_t* __restrict__ counts,
                                                         const uint64_t* __restrict__ offs,
                                                         uint64_t* __restrict__ out) {
  const uint64_t nch = (len + kKmerChunk - 1) / kKmerChunk;
  const uint64_t mask = k >= 32 ? ~0ull : ((1ull << (2 * k)) - 1u);
  for (uint64_t c = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; c < nch; c += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t s = c * kKmerChunk, e = min(len, s + kKmerChunk);
    uint64_t p = s >= k - 1 ? s - (k - 1) : 0;
    uint64_t value = 0, o = EMIT ? offs[c] : 0;
    uint32_t fill = 0, cnt = 0;
    for (; p < e; ++p) {
      const uint32_t code = base_code(__ldg(seq + p));
      if (code > 3u) {
        value = 0;
        fill = 0;
        continue;
      }
      value = ((value << 2) | code) & mask;
      fill = fill < k ? fill + 1 : k;
      if (fill == k && p >= s) {
        if (EMIT) out[o++] = value;
        else ++cnt;
      }
    }
    if (!EMIT) counts[c] = cnt;
  }
}

// exclusive scan of the chunk counts (one block) -> offsets, total -> *n_out
__global__ void __launch_bounds__(1024) kmer_scan_kernel(const uint32_t* __restrict__ counts, uint64_t nch,
                                                         uint64_t* __restrict__ offs, unsigned long long* n_out) {
  __shared__ uint64_t wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t per = (nch + blockDim.x - 1) / blockDim.x;
  const uint64_t lo = min((uint64_t)tid * per, nch), hi = min(lo + per, nch);
  uint64_t sum = 0;
  for (uint64_t i = lo; i < hi; ++i) sum += counts[i];
  uint64_t x = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint64_t v = lane < (int)(blockDim.x / 32) ? wsum[lane] : 0, t = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, t, d);
      if (lane >= d) t += y;
    }
    wsum[lane] = t - v;
    if (lane == 31) *n_out = t;
  }
  __syncthreads();
  uint64_t run = wsum[wid] + x - sum;
  for (uint64_t i = lo; i < hi; ++i) {
    offs[i] = run;
    run += counts[i];
  }
}

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

// Schedule of one call: the region schedule when its plan applies and the
// caller's workspace holds it, else the direct kernels.  Automatic choice:
// tables past the L2 (>= 48 MiB) and at least one key per bucket.
// The batch size from which the region schedule beats the direct kernels, in
// keys per bucket (measured on a 2^28-slot table, profiles/r02_crossover.jsonl):
// 32-byte buckets cross over at ~1 key per bucket for insert / delete /
// lookup- and ~2-3 for lookup+ (the direct lookup of a mostly-positive batch
// reads one sector per key); 64-byte buckets (f = 32) at ~1.5 for every op.
static double region_threshold(const ckf_params* p, int op) {
  if (p->words_per_bucket >= 8) return 1.5;
  return op == CKF_OP_QUERY ? 2.0 : 1.0;
}

static bool region_wanted(const ckf_params* p, uint64_t n, int op, unsigned flags) {
  if (flags & (CKF_FORCE_DIRECT | CKF_MODE_SEQUENTIAL)) return false;
  if (n == 0) return false;
  if (!(flags & CKF_FORCE_TILED)) {
    if (!env_u64("CKF_TILED_AUTO", 1)) return false;
    const uint64_t table = p->bucket_count * p->words_per_bucket * 8ull;
    if (table < kRegionMinTable || (double)n < region_threshold(p, op) * (double)p->bucket_count) return false;
  }
  return true;
}

static TiledArgs choose(const ckf_params* p, uint64_t n, int op, unsigned flags, const void* keys, void* ws,
                        uint64_t ws_bytes) {
  TiledArgs t{};
  if (!ws || !region_wanted(p, n, op, flags) || ((uintptr_t)keys % 8) != 0 || ((uintptr_t)ws % 256) != 0) return t;
  bool ok = false;
  t.rpl = make_rplan(p, n, op, flags, ok);
  if (!ok) return t;
  t.RL = rlayout_for(t.rpl, op);
  t.ws = ws;
  t.region = ws_bytes >= t.RL.total;
  return t;
}

// Direct-path insert scratch: a room map (one bit per bucket), the BFS
// eviction cursor and the gate, for batches of >= m/8 keys (the map costs one
// scan of the table; room_scan_kernel builds it only for a long enough
// eviction queue).  Measured (profiles/r02_direct_roommap.txt):
// 2^22 slots f=16 b=16 insert 0.277 -> 0.250 ms, 2^24 slots 0.779 -> 0.705 ms;
// one-word buckets (b=4: the pass is bound by its longest chain) 2 % slower,
// so they keep the one-chain-per-thread pass.
static uint64_t direct_ws_bytes(const ckf_params* p, uint64_t n, int op, unsigned flags) {
  if (op != CKF_OP_INSERT || (flags & CKF_MODE_SEQUENTIAL) || p->eviction != CKF_EVICT_BFS) return 0;
  const uint32_t wpb = p->words_per_bucket;
  if (wpb != 2 && wpb != 4 && wpb != 8) return 0;
  const uint64_t m = p->bucket_count;
  if (n * 8 < m || env_u64("CKF_NO_DIRECT_ROOM_MAP", 0)) return 0;
  return direct_rm_bytes(m) + 256;
}

static bool region_planned(const ckf_params* p, uint64_t n, int op, unsigned flags) {
  if (!region_wanted(p, n, op, flags)) return false;
  bool ok;
  make_rplan(p, n, op, flags, ok);
  return ok;
}

uint64_t ckf_workspace_bytes(const ckf_params* p, uint64_t n, int op, unsigned flags) {
  if (!params_ok(p)) return 0;
  if (region_planned(p, n, op, flags)) {
    bool ok;
    return rlayout_for(make_rplan(p, n, op, flags, ok), op).total;
  }
  return direct_ws_bytes(p, n, op, flags);
}

int ckf_schedule(const ckf_params* p, uint64_t n, int op, unsigned flags, const void* keys, const void* workspace,
                 uint64_t workspace_bytes, uint64_t* runs) {
  if (runs) *runs = 0;
  if (!params_ok(p)) return CKF_EINVAL;
  if (flags & CKF_MODE_SEQUENTIAL) return op == CKF_OP_QUERY ? CKF_SCHED_DIRECT : CKF_SCHED_SEQUENTIAL;
  if (!region_planned(p, n, op, flags)) return CKF_SCHED_DIRECT;
  const TiledArgs t = choose(p, n, op, flags, keys, const_cast<void*>(workspace), workspace_bytes);
  if (!t.region) return CKF_SCHED_DIRECT;
  if (runs) *runs = run_count(t, n);
  return CKF_SCHED_REGION;
}

int ckf_insert(const ckf_params* p, uint64_t* words, const uint64_t* keys, uint64_t n, uint8_t* ok, int64_t* evictions,
               uint64_t* lost, ckf_record* records, uint64_t record_cap, ckf_counters* counters, long long* occupancy,
               void* workspace, uint64_t workspace_bytes, unsigned flags, void* stream) {
  if (!params_ok(p) || !words || !counters) return CKF_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(counters, 0, sizeof(ckf_counters), s) != cudaSuccess) return cuda_error();
  if (n == 0) return CKF_OK;
  if (!keys || !ok || (record_cap && !records)) return CKF_EINVAL;
  InsertArgs a{geo_from(*p), words, keys, n, ok, evictions, lost, records, records ? record_cap : 0,
               counters, occupancy, (flags & CKF_INPUT_HASHED) != 0, (flags & CKF_MODE_SEQUENTIAL) != 0, s,
               choose(p, n, CKF_OP_INSERT, flags, keys, workspace, workspace_bytes)};
  if (!a.t.region && workspace && ((uintptr_t)workspace % 256) == 0) {
    const uint64_t need = direct_ws_bytes(p, n, CKF_OP_INSERT, flags);
    if (need && workspace_bytes >= need) {
      a.t.ws = workspace;
      a.t.direct_rm = true;
    }
  }
  return dispatch3<InsertOp>(p, words, a);
}

int ckf_query(const ckf_params* p, const uint64_t* words, const uint64_t* keys, uint64_t n, uint8_t* out,
              ckf_counters* counters, void* workspace, uint64_t workspace_bytes, unsigned flags, void* stream) {
  if (!params_ok(p) || !words) return CKF_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (counters && cudaMemsetAsync(counters, 0, sizeof(ckf_counters), s) != cudaSuccess) return cuda_error();
  if (n == 0) return CKF_OK;
  if (!keys || !out) return CKF_EINVAL;
  QueryArgs a{geo_from(*p), words, keys, n, out, counters, (flags & CKF_INPUT_HASHED) != 0, s,
              choose(p, n, CKF_OP_QUERY, flags, keys, workspace, workspace_bytes)};
  return dispatch3<QueryOp>(p, words, a);
}

int ckf_delete(const ckf_params* p, uint64_t* words, const uint64_t* keys, uint64_t n, uint8_t* out,
               ckf_counters* counters, long long* occupancy, void* workspace, uint64_t workspace_bytes, unsigned flags,
               void* stream) {
  if (!params_ok(p) || !words) return CKF_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (counters && cudaMemsetAsync(counters, 0, sizeof(ckf_counters), s) != cudaSuccess) return cuda_error();
  if (n == 0) return CKF_OK;
  if (!keys || !out) return CKF_EINVAL;
  DeleteArgs a{geo_from(*p), words, keys, n, out, counters, occupancy, (flags & CKF_INPUT_HASHED) != 0,
               (flags & CKF_MODE_SEQUENTIAL) != 0, s, choose(p, n, CKF_OP_DELETE, flags, keys, workspace, workspace_bytes)};
  return dispatch3<DeleteOp>(p, words, a);
}

int ckf_mixed(const ckf_params* p, uint64_t* words, const uint8_t* ops, const uint64_t* keys, uint64_t n,
              uint8_t* out, ckf_record* records, uint64_t record_cap, ckf_counters* counters, long long* occupancy,
              unsigned flags, void* stream) {
  if (!params_ok(p) || !words || !counters) return CKF_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(counters, 0, sizeof(ckf_counters), s) != cudaSuccess) return cuda_error();
  if (n == 0) return CKF_OK;
  if (!ops || !keys || !out || (record_cap && !records)) return CKF_EINVAL;
  MixedArgs a{geo_from(*p), words, ops, keys, n, out, records, records ? record_cap : 0, counters, occupancy,
              (flags & CKF_INPUT_HASHED) != 0, s};
  return dispatch3<MixedOp>(p, words, a);
}

uint64_t ckf_route_workspace_bytes(uint64_t n, uint32_t shards) {
  const uint64_t nt = (n + kRtTile - 1) / kRtTile;
  return align256(nt * shards * 4) + align256(nt * shards * 8);
}

int ckf_route_partition(const uint64_t* hashes, uint64_t n, uint32_t shift, uint32_t shards, uint64_t* send,
                        long long* order, long long* shard_counts, void* workspace, uint64_t workspace_bytes,
                        void* stream) {
  if (shards < 1 || shards > 8 || (shards & (shards - 1)) || shift > 63 || !shard_counts) return CKF_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) return cudaMemsetAsync(shard_counts, 0, 8ull * shards, s) == cudaSuccess ? CKF_OK : cuda_error();
  if (!hashes || !send || !order || !workspace || workspace_bytes < ckf_route_workspace_bytes(n, shards))
    return CKF_EINVAL;
  const uint64_t nt = (n + kRtTile - 1) / kRtTile;
  if (nt > 0x7FFFFFFFull) return CKF_EINVAL;
  uint32_t* counts = (uint32_t*)workspace;
  uint64_t* offs = (uint64_t*)((char*)workspace + align256(nt * shards * 4));
  const uint32_t gmask = shards - 1;
  route_count_kernel<<<(unsigned)nt, kRtThreads, 0, s>>>(hashes, n, shift, gmask, counts);
  int st = status();
  if (st) return st;
  route_scan_kernel<<<1, 1024, 0, s>>>(counts, nt, shards, offs, shard_counts, 0);
  if ((st = status())) return st;
  allow_big_smem<route_scatter_kernel>(kRouteSmem);
  route_scatter_kernel<<<(unsigned)nt, kRtThreads, kRouteSmem, s>>>(hashes, n, shift, gmask, offs, send, order, 0,
                                                                   nullptr);
  return status();
}

int ckf_route_partition_padded(const uint64_t* hashes, uint64_t n, uint32_t shift, uint32_t shards, uint64_t cap,
                               uint64_t* send, long long* order, long long* shard_counts,
                               unsigned long long* spilled, void* workspace, uint64_t workspace_bytes, void* stream) {
  if (shards < 2 || shards > 8 || (shards & (shards - 1)) || shift > 63 || !shard_counts || !spilled || cap == 0)
    return CKF_EINVAL;
  if (!send || !order) return CKF_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (cudaMemsetAsync(spilled, 0, 8, s) != cudaSuccess) return cuda_error();
  const uint32_t gmask = shards - 1;
  int st;
  if (n == 0) {
    if (cudaMemsetAsync(shard_counts, 0, 8ull * shards, s) != cudaSuccess) return cuda_error();
  } else {
    if (!hashes || !workspace || workspace_bytes < ckf_route_workspace_bytes(n, shards)) return CKF_EINVAL;
    const uint64_t nt = (n + kRtTile - 1) / kRtTile;
    if (nt > 0x7FFFFFFFull) return CKF_EINVAL;
    uint32_t* counts = (uint32_t*)workspace;
    uint64_t* offs = (uint64_t*)((char*)workspace + align256(nt * shards * 4));
    route_count_kernel<<<(unsigned)nt, kRtThreads, 0, s>>>(hashes, n, shift, gmask, counts);
    if ((st = status())) return st;
    route_scan_kernel<<<1, 1024, 0, s>>>(counts, nt, shards, offs, shard_counts, cap);
    if ((st = status())) return st;
    allow_big_smem<route_scatter_kernel>(kRouteSmem);
    route_scatter_kernel<<<(unsigned)nt, kRtThreads, kRouteSmem, s>>>(hashes, n, shift, gmask, offs, send, order,
                                                                     cap, spilled);
    if ((st = status())) return st;
  }
  route_fill_kernel<<<grid_for((uint64_t)shards * cap, 256, 8), 256, 0, s>>>(send, order, shard_counts, shards, cap,
                                                                             shift);
  return status();
}

int ckf_route_unpermute(const void* back, const long long* order, uint64_t n, uint32_t elem, void* out,
                        void* stream) {
  if (n == 0) return CKF_OK;
  if (!back || !order || !out || (elem != 1 && elem != 8)) return CKF_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  const unsigned grid = grid_for(n, 256, 8);
  if (elem == 1)
    route_unpermute_kernel<uint8_t><<<grid, 256, 0, s>>>((const uint8_t*)back, order, n, (uint8_t*)out);
  else
    route_unpermute_kernel<uint64_t><<<grid, 256, 0, s>>>((const uint64_t*)back, order, n, (uint64_t*)out);
  return status();
}

int ckf_params_set_shard(ckf_params* p, uint32_t shift, uint32_t shards, uint32_t id) {
  if (!p || shards < 1 || shards > 256 || (shards & (shards - 1)) || id >= shards || shift > 63) return CKF_EINVAL;
  p->shard_shift = shards > 1 ? shift : 0;
  p->shard_mask = shards - 1;
  p->shard_id = shards > 1 ? id : 0;
  return CKF_OK;
}

uint64_t ckf_kmer_workspace_bytes(uint64_t len) {
  const uint64_t nch = (len + kKmerChunk - 1) / kKmerChunk;
  return align256(nch * 4) + align256(nch * 8);
}

int ckf_kmers(const uint8_t* seq, uint64_t len, uint32_t k, uint64_t* out, unsigned long long* n_out,
              void* workspace, uint64_t workspace_bytes, void* stream) {
  if (k < 1 || k > 31 || !n_out) return CKF_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  if (len == 0) return cudaMemsetAsync(n_out, 0, 8, s) == cudaSuccess ? CKF_OK : cuda_error();
  if (!seq || !out || !workspace || workspace_bytes < ckf_kmer_workspace_bytes(len)) return CKF_EINVAL;
  const uint64_t nch = (len + kKmerChunk - 1) / kKmerChunk;
  uint32_t* counts = (uint32_t*)workspace;
  uint64_t* offs = (uint64_t*)((char*)workspace + align256(nch * 4));
  const unsigned grid = grid_for(nch, 256, 8);
  kmer_chunk_kernel<false><<<grid, 256, 0, s>>>(seq, len, k, counts, nullptr, nullptr);
  int st = status();
  if (st) return st;
  kmer_scan_kernel<<<1, 1024, 0, s>>>(counts, nch, offs, n_out);
  if ((st = status())) return st;
  kmer_chunk_kernel<true><<<grid, 256, 0, s>>>(seq, len, k, nullptr, offs, out);
  return status();
}

int ckf_debug_fault_origin_cas(unsigned int count) {
  return cudaMemcpyToSymbol(g_fault_origin_cas, &count, sizeof(count)) == cudaSuccess ? CKF_OK : cuda_error();
}

int ckf_debug_faults_pending(unsigned int* count) {
  if (!count) return CKF_EINVAL;
  return cudaMemcpyFromSymbol(count, g_fault_origin_cas, sizeof(*count)) == cudaSuccess ? CKF_OK : cuda_error();
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
