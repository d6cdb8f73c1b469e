// ckf_tiled.cuh -- L2-tiled execution of large batches.
//
// Why: one insert / query / delete touches one or two random 32-byte buckets.
// Measured on B200 (profiles/r01_probe_ceiling.txt), random 32 B sector reads
// top out at ~48 G/s at 512 MiB (~1.5 TB/s useful, a quarter of the 6.4 TB/s
// streaming peak): HBM3e is row-activation bound on random sectors, and a
// DRAM-resident atomic costs ~2 such accesses (profiles/r01_probe_atomics.txt:
// 24 G CAS/s at 512 MiB vs 120 G/s L2-resident).  When a batch holds many keys
// per bucket (the benchmark inserts 15 keys per bucket) the same buckets are
// fetched again and again.  The tiled path therefore
//
//   pass A  hashes the keys and bins them by the table region (R regions of
//           `rb` buckets) of their primary bucket, as packed 8-byte records
//           (batch index | bucket offset in region | fingerprint);
//   pass B  walks the bins `group` at a time -- those regions are L2-resident
//           -- and resolves every key whose primary bucket answers it; the rest
//           are re-binned by the region of their alternate bucket;
//   pass C  walks those bins the same way for the alternate bucket;
// and the per-key results are merged through an L2-resident bitmap (n/8
// bytes).  Every DRAM stream is sequential; the bucket accesses hit L2.
// Semantics are unchanged: batch ops are concurrent and this is one legal
// schedule of them (every key tries i1 before i2, as in K:359-362).  A full bin
// (adversarial keys) resolves its key in place on the direct path, so
// correctness never depends on the binning statistics.
#pragma once

#include "ckf_device.cuh"

namespace ckf {

enum { OP_QUERY = 0, OP_INSERT = 1, OP_DELETE = 2 };

constexpr int kTileThreads = 256;
constexpr int kTileItems = 8;
constexpr int kTile = kTileThreads * kTileItems;  // records per tile
constexpr int kTileMinBlocks = 4;                  // >= 4 resident CTAs per SM (<= 64 registers)
constexpr int kMaxBins = 512;
constexpr int kCntStride = 32;                     // bin counters 128 B apart (one line each)
constexpr int kProbeItems = 2;                     // bucket fetches in flight per thread

// Binning plan for one (table, batch) pair, computed on the host.
struct Plan {
  uint64_t div_magic;  // bin = mulhi(bucket, div_magic)  (== bucket / rb for bucket < 2^32)
  uint64_t cap;        // record slots per bin
  uint32_t rb;         // buckets per region
  uint32_t R;          // number of bins
  uint32_t pb;         // payload (fingerprint) bits in a record
  uint32_t group;      // bins probed concurrently
  uint32_t tiles_per_bin;
};

__device__ __forceinline__ uint32_t bin_of(uint64_t bucket, const Plan& pl) {
  return (uint32_t)__umul64hi(bucket, pl.div_magic);
}

// record = index << 32 | (bucket - bin*rb) << pb | fp
__device__ __forceinline__ uint64_t pack_rec(uint32_t idx, uint64_t local, uint64_t fp, const Plan& pl) {
  return ((uint64_t)idx << 32) | (local << pl.pb) | fp;
}
__device__ __forceinline__ void unpack_rec(uint64_t rec, uint32_t bin, const Plan& pl, uint32_t& idx, uint64_t& bucket,
                                           uint64_t& fp) {
  idx = (uint32_t)(rec >> 32);
  const uint32_t lo = (uint32_t)rec;
  fp = lo & ((1u << pl.pb) - 1u);
  bucket = (uint64_t)bin * pl.rb + (lo >> pl.pb);
}

// Workspace views (layout: layout_for in ckf_kernels.cu).
struct Work {
  uint32_t* cnt1;   // [R*kCntStride] records appended per primary bin (may exceed cap)
  uint32_t* cnt2;   // [R*kCntStride] per alternate bin
  uint64_t* bin1;   // [R*cap] records binned by primary region
  uint64_t* bin2;   // [R*cap] records binned by alternate region
  uint32_t* bits;   // [ceil(n/32)] result bitmap (query / delete)
};

// What happens to a resolved / unresolved key.
struct Sink {
  uint32_t* bits;         // query/delete: result bit per key
  ckf_record* rec;        // insert: eviction queue
  uint64_t rec_cap;
  ckf_counters* ctr;
  uint8_t* ok;            // insert: dense ok (queue overflow only)
  const uint64_t* keys;   // insert: to recover a queued key's hash
  bool hashed;
};

__device__ __forceinline__ void set_bit(uint32_t* bits, uint32_t i) { atomicOr(bits + (i >> 5), 1u << (i & 31)); }

// The two halves of every op, split into "fetch the bucket" and "act on the
// fetched snapshot" so a thread can have several bucket fetches in flight.
template <int OP, int F, int WPB, int POL>
struct Logic {
  static __device__ __forceinline__ void fetch(const uint64_t* words, uint64_t bucket, uint64_t (&w)[WPB]) {
    if constexpr (OP == OP_QUERY) ld_bucket_ro_el<WPB>(words + bucket * WPB, w);
    else ld_bucket_rw_el<WPB>(words + bucket * WPB, w);
  }
  // tag: fp for the primary bucket, fp|choice for the alternate
  static __device__ __forceinline__ bool act(uint64_t* words, uint64_t bucket, uint64_t fp, uint64_t tag,
                                             uint64_t (&w)[WPB]) {
    if constexpr (OP == OP_QUERY) {
      using L = Lanes<F>;
      const uint64_t keep = POL == CKF_POLICY_OFFSET ? ~L::kHigh : ~0ull;
      const uint64_t pat = L::bcast(fp);
      uint64_t any = 0;
#pragma unroll
      for (int j = 0; j < WPB; ++j) any |= L::zeros((w[j] & keep) ^ pat);
      return any != 0;
    } else if constexpr (OP == OP_INSERT) {
      return try_insert_snap<F, WPB>(words, bucket, tag, w) >= 0;
    } else {
      return remove_tag_snap<F, WPB>(words, bucket, tag, w) >= 0;
    }
  }
  static __device__ __forceinline__ uint64_t tag2(uint64_t fp, const Geo& g) {
    return POL == CKF_POLICY_OFFSET ? make_tag(fp, 1u, g) : fp;
  }
  static __device__ __forceinline__ bool first(uint64_t* words, uint64_t i1, uint64_t fp, const Geo& g) {
    uint64_t w[WPB];
    fetch(words, i1, w);
    return act(words, i1, fp, fp, w);
  }
  static __device__ __forceinline__ bool second(uint64_t* words, uint64_t i2, uint64_t fp, const Geo& g) {
    uint64_t w[WPB];
    fetch(words, i2, w);
    return act(words, i2, fp, tag2(fp, g), w);
  }
};

// Probe-pass tile order: the tiles of `group` consecutive bins are
// interleaved, so the CTAs in flight spread over `group` table regions (kept
// L2-resident) instead of piling onto one region's buckets (CAS contention).
__device__ __forceinline__ void tile_coords(uint64_t s, const Plan& pl, uint32_t& bin, uint64_t& off0) {
  const uint32_t grp = pl.R < pl.group ? pl.R : pl.group;
  const uint64_t per_group = (uint64_t)grp * pl.tiles_per_bin;
  const uint64_t gidx = s / per_group, q = s % per_group;
  bin = (uint32_t)(gidx * grp + q % grp);
  off0 = (q / grp) * kTile;
}

// Unresolved insert after both buckets: hand (index, hash) to the eviction
// pass; one queue atomic per warp.  Caller guarantees a converged warp.
__device__ __forceinline__ void enqueue_evict(const Sink& sk, bool need, uint32_t idx, const Geo& g) {
  const unsigned act = __activemask();
  const unsigned qm = __ballot_sync(act, need);
  if (!qm) return;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(qm) - 1;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(&sk.ctr->n_queued, (unsigned long long)__popc(qm));
  base = __shfl_sync(act, base, leader);
  if (!need) return;
  const uint64_t pos = base + __popc(qm & ((1u << lane) - 1u));
  const uint64_t k = sk.keys[idx];
  if (pos < sk.rec_cap) sk.rec[pos] = ckf_record{idx, sk.hashed ? k : xxh64(k, g.seed), 0u, 0u};
  // queue overflow cannot happen through the facade (capacity = n); the key
  // is then reported as not stored
  else if (sk.ok) sk.ok[idx] = 0;
}

__device__ __forceinline__ void enqueue_evict_one(const Sink& sk, uint32_t idx, uint64_t h) {
  const uint64_t pos = atomicAdd(&sk.ctr->n_queued, 1ull);
  if (pos < sk.rec_cap) sk.rec[pos] = ckf_record{idx, h, 0u, 0u};
  else if (sk.ok) sk.ok[idx] = 0;
}

// ---- block-cooperative multi-split append ----

struct SplitSmem {
  uint32_t hist[kMaxBins];
  uint32_t start[kMaxBins];
  uint32_t gbase[kMaxBins];
  uint64_t rec[kTile];
  uint16_t bin[kTile];
  uint32_t warp_sums[kTileThreads / 32];
};

// Exclusive prefix sum of in[0..R) into out[] by the whole block.
__device__ __forceinline__ void block_exclusive_scan(const uint32_t* in, uint32_t* out, uint32_t R,
                                                     uint32_t* warp_sums) {
  constexpr int NW = kTileThreads / 32;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t per = (R + kTileThreads - 1) / kTileThreads;
  const uint32_t lo = min(tid * per, R), hi = min(lo + per, R);
  uint32_t sum = 0;
  for (uint32_t k = lo; k < hi; ++k) sum += in[k];
  uint32_t x = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t v = lane < NW ? warp_sums[lane] : 0, s = v;
#pragma unroll
    for (int d = 1; d < NW; d <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s, d);
      if (lane >= d) s += y;
    }
    if (lane < NW) warp_sums[lane] = s - v;
  }
  __syncthreads();
  uint32_t run = warp_sums[wid] + x - sum;
  for (uint32_t k = lo; k < hi; ++k) {
    out[k] = run;
    run += in[k];
  }
  __syncthreads();
}

// Appends the block's valid records to their bins: records are counting-sorted
// by bin in shared memory, one global atomic per (block, bin) reserves a run
// right after the previous block's run of that bin, and the runs go out as
// contiguous stores (partial sectors meet their neighbours in L2).  Records
// past a bin's capacity go to `ovf(rec, bin)` instead.
template <int I, class Overflow>
__device__ __forceinline__ void block_append(const uint64_t (&rec)[I], const uint32_t (&bin)[I], const bool (&v)[I],
                                             const Plan& pl, uint64_t* __restrict__ out, uint32_t* gcnt,
                                             SplitSmem& sm, Overflow&& ovf) {
  const int tid = threadIdx.x;
  const uint64_t pol = evict_first_policy();
  for (uint32_t r = tid; r < pl.R; r += kTileThreads) sm.hist[r] = 0;
  __syncthreads();
  uint32_t rank[I];
#pragma unroll
  for (int j = 0; j < I; ++j) rank[j] = v[j] ? atomicAdd(&sm.hist[bin[j]], 1u) : 0u;
  __syncthreads();
  block_exclusive_scan(sm.hist, sm.start, pl.R, sm.warp_sums);
  for (uint32_t r = tid; r < pl.R; r += kTileThreads) {
    const uint32_t c = sm.hist[r];
    sm.gbase[r] = c ? atomicAdd(gcnt + (size_t)r * kCntStride, c) : 0u;
  }
#pragma unroll
  for (int j = 0; j < I; ++j) {
    if (!v[j]) continue;
    const uint32_t p = sm.start[bin[j]] + rank[j];
    sm.rec[p] = rec[j];
    sm.bin[p] = (uint16_t)bin[j];
  }
  __syncthreads();
  const uint32_t total = sm.start[pl.R - 1] + sm.hist[pl.R - 1];
  for (uint32_t p = tid; p < total; p += kTileThreads) {
    const uint32_t r = sm.bin[p];
    const uint64_t off = (uint64_t)sm.gbase[r] + (p - sm.start[r]);
    if (off < pl.cap) st_stream_ef(out + r * pl.cap + off, sm.rec[p], pol);
    else ovf(sm.rec[p], r);
  }
  __syncthreads();
}

// ---- pass A: hash + bin by primary-bucket region ----

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(gmem), "r"(src_bytes)
               : "memory");
}

// Stage tile [t0, t0 + kTile) of the keys into shared memory (zero-filled past
// n); each thread copies its own 16-byte pieces, so no barrier is needed
// before its own reads.
__device__ __forceinline__ void stage_keys(uint64_t* buf, const uint64_t* keys, uint64_t t0, uint64_t n) {
#pragma unroll
  for (int q = 0; q < kTileItems / 2; ++q) {
    const uint32_t e = (q * kTileThreads + threadIdx.x) * 2;  // element pair
    const uint64_t i = t0 + e;
    const uint32_t bytes = i + 2 <= n ? 16u : (i < n ? 8u : 0u);
    cp_async16(buf + e, keys + (i < n ? i : 0), bytes);
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int OP, int F, int WPB, int POL>
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks)
    tile_bin_kernel(Geo g, Plan pl, uint64_t* words, const uint64_t* __restrict__ keys, uint64_t n, bool hashed,
                    Work w, Sink sk, long long* occ) {
  __shared__ SplitSmem sm;
  __shared__ __align__(16) uint64_t kbuf[kTile];  // next tile's keys, copied in while this one is binned
  using Lg = Logic<OP, F, WPB, POL>;
  uint32_t n_ok = 0;
  const uint64_t step = (uint64_t)gridDim.x * kTile;
  uint64_t t0 = blockIdx.x * (uint64_t)kTile;
  if (t0 < n) stage_keys(kbuf, keys, t0, n);
  for (; t0 < n; t0 += step) {
    uint64_t rec[kTileItems];
    uint32_t bin[kTileItems];
    bool v[kTileItems];
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    uint64_t kk[kTileItems];
#pragma unroll
    for (int q = 0; q < kTileItems / 2; ++q) {  // the pairs this thread copied itself
      const uint32_t e = (q * kTileThreads + threadIdx.x) * 2;
      kk[2 * q] = kbuf[e];
      kk[2 * q + 1] = kbuf[e + 1];
    }
    if (t0 + step < n) stage_keys(kbuf, keys, t0 + step, n);  // overlaps the rest of this tile
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) {
      const uint64_t i = t0 + ((j >> 1) * kTileThreads + threadIdx.x) * 2 + (j & 1);
      v[j] = i < n;
      const uint64_t h = hashed ? kk[j] : xxh64(kk[j], g.seed);
      uint64_t fp, i1, i2;
      place<POL>(h, g, fp, i1, i2);
      bin[j] = bin_of(i1, pl);
      rec[j] = pack_rec((uint32_t)i, i1 - (uint64_t)bin[j] * pl.rb, fp, pl);
    }
    // a full bin (adversarial keys): resolve that key in place, randomly
    block_append(rec, bin, v, pl, w.bin1, w.cnt1, sm, [&](uint64_t rc, uint32_t r) {
      uint32_t ii;
      uint64_t i1, fp;
      unpack_rec(rc, r, pl, ii, i1, fp);
      uint64_t c;
      const uint64_t i2 = alt_index<POL>(i1, fp, 0, g, c);
      if (Lg::first(words, i1, fp, g) || Lg::second(words, i2, fp, g)) {
        ++n_ok;
        if (OP != OP_INSERT) set_bit(sk.bits, ii);
      } else if (OP == OP_INSERT) {
        const uint64_t k = keys[ii];
        enqueue_evict_one(sk, ii, hashed ? k : xxh64(k, g.seed));
      }
    });
  }
  block_count_add(n_ok, 0, sk.ctr, occ, OP == OP_DELETE ? -1 : +1);
}

// ---- pass B: primary buckets; misses re-binned by alternate region ----

template <int OP, int F, int WPB, int POL>
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks)
    tile_probe1_kernel(Geo g, Plan pl, uint64_t* words, Work w, Sink sk, long long* occ) {
  __shared__ SplitSmem sm;
  using Lg = Logic<OP, F, WPB, POL>;
  const uint64_t pol = evict_first_policy();
  uint32_t n_ok = 0, n_alt = 0;
  const uint64_t tiles = (uint64_t)pl.R * pl.tiles_per_bin;
  for (uint64_t s = blockIdx.x; s < tiles; s += gridDim.x) {
    uint32_t r;
    uint64_t off0;
    tile_coords(s, pl, r, off0);
    const uint32_t c = w.cnt1[(size_t)r * kCntStride];
    const uint64_t cnt = c < pl.cap ? c : pl.cap;
    if (off0 >= cnt) continue;  // block-uniform
    const uint64_t* src = w.bin1 + r * pl.cap;
    uint64_t rec[kTileItems];
    uint32_t bin[kTileItems];
    bool need[kTileItems];
#pragma unroll
    for (int j0 = 0; j0 < kTileItems; j0 += kProbeItems) {
      uint64_t fp[kProbeItems], i1[kProbeItems];
      uint32_t idx[kProbeItems];
      uint64_t wv[kProbeItems][WPB];
      bool v[kProbeItems];
#pragma unroll
      for (int q = 0; q < kProbeItems; ++q) {
        const uint64_t off = off0 + (j0 + q) * kTileThreads + threadIdx.x;
        v[q] = off < cnt;
        const uint64_t rc = v[q] ? ld_stream_ef(src + off, pol) : 0;
        unpack_rec(rc, r, pl, idx[q], i1[q], fp[q]);
        if (v[q]) Lg::fetch(words, i1[q], wv[q]);
      }
#pragma unroll
      for (int q = 0; q < kProbeItems; ++q) {
        const int j = j0 + q;
        const bool done = v[q] && Lg::act(words, i1[q], fp[q], fp[q], wv[q]);
        if (done) {
          ++n_ok;
          if (OP != OP_INSERT) set_bit(sk.bits, idx[q]);
        }
        need[j] = v[q] && !done;
        n_alt += need[j];
        uint64_t cc;
        const uint64_t i2 = alt_index<POL>(i1[q], fp[q], 0, g, cc);
        bin[j] = bin_of(i2, pl);
        rec[j] = pack_rec(idx[q], i2 - (uint64_t)bin[j] * pl.rb, fp[q], pl);
      }
    }
    block_append(rec, bin, need, pl, w.bin2, w.cnt2, sm, [&](uint64_t rc, uint32_t r2) {
      uint32_t ii;
      uint64_t i2, fp;
      unpack_rec(rc, r2, pl, ii, i2, fp);
      if (Lg::second(words, i2, fp, g)) {
        ++n_ok;
        if (OP != OP_INSERT) set_bit(sk.bits, ii);
      } else if (OP == OP_INSERT) {
        const uint64_t k = sk.keys[ii];
        enqueue_evict_one(sk, ii, sk.hashed ? k : xxh64(k, g.seed));
      }
    });
  }
  block_count_add(n_ok, n_alt, sk.ctr, occ, OP == OP_DELETE ? -1 : +1);
}

// ---- pass C: alternate buckets ----

template <int OP, int F, int WPB, int POL>
__global__ void __launch_bounds__(kTileThreads, kTileMinBlocks)
    tile_probe2_kernel(Geo g, Plan pl, uint64_t* words, Work w, Sink sk, long long* occ) {
  using Lg = Logic<OP, F, WPB, POL>;
  const uint64_t pol = evict_first_policy();
  uint32_t n_ok = 0;
  const uint64_t tiles = (uint64_t)pl.R * pl.tiles_per_bin;
  for (uint64_t s = blockIdx.x; s < tiles; s += gridDim.x) {
    uint32_t r;
    uint64_t off0;
    tile_coords(s, pl, r, off0);
    const uint32_t c = w.cnt2[(size_t)r * kCntStride];
    const uint64_t cnt = c < pl.cap ? c : pl.cap;
    if (off0 >= cnt) continue;
    const uint64_t* src = w.bin2 + r * pl.cap;
    uint32_t fidx[kTileItems];
    uint32_t fmask = 0;
#pragma unroll
    for (int j0 = 0; j0 < kTileItems; j0 += kProbeItems) {
      uint64_t fp[kProbeItems], i2[kProbeItems];
      uint32_t idx[kProbeItems];
      uint64_t wv[kProbeItems][WPB];
      bool v[kProbeItems];
#pragma unroll
      for (int q = 0; q < kProbeItems; ++q) {
        const uint64_t off = off0 + (j0 + q) * kTileThreads + threadIdx.x;
        v[q] = off < cnt;
        const uint64_t rc = v[q] ? ld_stream_ef(src + off, pol) : 0;
        unpack_rec(rc, r, pl, idx[q], i2[q], fp[q]);
        if (v[q]) Lg::fetch(words, i2[q], wv[q]);
      }
#pragma unroll
      for (int q = 0; q < kProbeItems; ++q) {
        const bool done = v[q] && Lg::act(words, i2[q], fp[q], Lg::tag2(fp[q], g), wv[q]);
        if (done) {
          ++n_ok;
          if (OP != OP_INSERT) set_bit(sk.bits, idx[q]);
        }
        fidx[j0 + q] = idx[q];
        if (OP == OP_INSERT && v[q] && !done) fmask |= 1u << (j0 + q);
      }
    }
    if (OP == OP_INSERT) {
      // one queue reservation per warp per tile for all its unplaced keys
      const int lane = threadIdx.x & 31;
      const uint32_t c = __popc(fmask);
      uint32_t incl = c;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += y;
      }
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      unsigned long long base = 0;
      if (lane == 31 && total) base = atomicAdd(&sk.ctr->n_queued, (unsigned long long)total);
      base = __shfl_sync(0xffffffffu, base, 31);
      uint64_t pos = base + incl - c;
#pragma unroll
      for (int j = 0; j < kTileItems; ++j) {
        if (!((fmask >> j) & 1u)) continue;
        const uint64_t k = sk.keys[fidx[j]];
        if (pos < sk.rec_cap) sk.rec[pos] = ckf_record{fidx[j], sk.hashed ? k : xxh64(k, g.seed), 0u, 0u};
        else if (sk.ok) sk.ok[fidx[j]] = 0;
        ++pos;
      }
    }
  }
  block_count_add(n_ok, 0, sk.ctr, occ, OP == OP_DELETE ? -1 : +1);
}

// bitmap -> one byte per key
__global__ void __launch_bounds__(256) expand_bits_kernel(const uint32_t* __restrict__ bits, uint64_t n,
                                                          uint8_t* __restrict__ out) {
  const uint64_t words = (n + 31) / 32;
  for (uint64_t wi = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; wi < words; wi += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = bits[wi];
    const uint64_t i0 = wi * 32;
    if (i0 + 32 <= n && ((uintptr_t)(out + i0) & 15) == 0) {
      uint32_t q[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t nib = (b >> (4 * k)) & 0xF;
        q[k] = (nib & 1) | ((nib >> 1 & 1) << 8) | ((nib >> 2 & 1) << 16) | ((nib >> 3 & 1) << 24);
      }
      reinterpret_cast<uint4*>(out + i0)[0] = make_uint4(q[0], q[1], q[2], q[3]);
      reinterpret_cast<uint4*>(out + i0)[1] = make_uint4(q[4], q[5], q[6], q[7]);
    } else {
      for (uint64_t i = i0; i < n && i < i0 + 32; ++i) out[i] = (b >> (i - i0)) & 1u;
    }
  }
}

}  // namespace ckf
