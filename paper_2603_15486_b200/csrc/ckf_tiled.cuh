// ckf_tiled.cuh -- L2-tiled execution of large batches.
//
// Why: one insert / query / delete touches one or two random 32-byte buckets.
// Measured on B200 (profiles/r01_probe_ceiling.txt), random 32 B sector reads
// top out at ~48 G/s at 512 MiB (~1.5 TB/s useful, a quarter of the 6.4 TB/s
// streaming peak): HBM3e is row-activation bound on random sectors.  When a
// batch holds many keys per bucket (the benchmark inserts 15 keys per bucket)
// the same buckets are fetched again and again.  The tiled path therefore
//
//   pass A  hashes the keys and bins (hash, index) records by the region of the
//           table their primary bucket lives in (R regions of ~2 MiB);
//   pass B  walks the bins in order -- the region being probed is L2-resident
//           -- and resolves every key whose primary bucket answers it; the rest
//           are re-binned by the region of their alternate bucket;
//   pass C  walks those bins the same way for the alternate bucket;
// and the per-key results are merged through an L2-resident bitmap
// (n/8 bytes).  Every DRAM stream is sequential; the random accesses hit L2.
// Semantics are unchanged: the batch ops are concurrent, and this is one legal
// schedule of them (every key tries i1 before i2, as in K:359-362).
#pragma once

#include "ckf_device.cuh"

namespace ckf {

enum { OP_QUERY = 0, OP_INSERT = 1, OP_DELETE = 2 };

constexpr int kTileThreads = 256;
constexpr int kTileItems = 8;
constexpr int kTile = kTileThreads * kTileItems;  // records per block tile
constexpr int kMaxBins = 1024;

// Binning plan for one (table, batch) pair, computed on the host.
struct Plan {
  uint64_t cap;            // record slots per bin (multiple of kTile)
  uint64_t magic;          // non power-of-two m: bin = min(R-1, (bucket*magic) >> 32)
  uint32_t R;              // number of bins
  uint32_t shift;          // power-of-two m: bin = bucket >> shift
  uint32_t tiles_per_bin;  // cap / kTile
  uint32_t pow2;
};

__device__ __forceinline__ uint32_t bin_of(uint64_t bucket, const Plan& pl) {
  if (pl.pow2) return (uint32_t)(bucket >> pl.shift);
  const uint64_t b = (bucket * pl.magic) >> 32;
  return b < pl.R ? (uint32_t)b : pl.R - 1;
}

// Workspace views (layout: ckf_workspace_bytes in ckf_kernels.cu).
struct Work {
  uint32_t* cnt1;  // [kMaxBins] records appended per primary bin (may exceed cap)
  uint32_t* cnt2;  // [kMaxBins] per alternate bin
  uint64_t* h1;    // [R*cap] key hashes binned by primary bucket
  uint32_t* x1;    // [R*cap] their batch indexes
  uint64_t* h2;    // [R*cap] binned by alternate bucket
  uint32_t* x2;
  uint32_t* bits;  // [ceil(n/32)] result bitmap (query / delete)
};

// What happens to a resolved / unresolved key.
struct Sink {
  uint32_t* bits;       // query/delete: result bit per key
  ckf_record* rec;      // insert: eviction queue
  uint64_t rec_cap;
  ckf_counters* ctr;
  uint8_t* ok;          // insert: dense ok (queue overflow only)
  int64_t* ev;
  uint64_t* lost;
};

__device__ __forceinline__ void set_bit(uint32_t* bits, uint32_t i) {
  atomicOr(bits + (i >> 5), 1u << (i & 31));
}

template <int F, int WPB, int POL>
__device__ __forceinline__ bool probe_ro(const uint64_t* words, uint64_t bucket, uint64_t fp) {
  using L = Lanes<F>;
  const uint64_t keep = POL == CKF_POLICY_OFFSET ? ~L::kHigh : ~0ull;
  uint64_t w[WPB];
  ld_bucket_ro<WPB>(words + bucket * WPB, w);
  const uint64_t pat = L::bcast(fp);
  uint64_t any = 0;
#pragma unroll
  for (int j = 0; j < WPB; ++j) any |= L::zeros((w[j] & keep) ^ pat);
  return any != 0;
}

// The two halves of every op: the primary-bucket attempt and the alternate one.
template <int OP, int F, int WPB, int POL>
struct Logic {
  static __device__ __forceinline__ bool first(uint64_t* words, uint64_t i1, uint64_t fp, const Geo& g) {
    if constexpr (OP == OP_QUERY) return probe_ro<F, WPB, POL>(words, i1, fp);
    else if constexpr (OP == OP_INSERT) return try_insert_t<F, WPB>(words, i1, fp) >= 0;
    else return remove_tag_t<F, WPB>(words, i1, fp) >= 0;
  }
  static __device__ __forceinline__ bool second(uint64_t* words, uint64_t i2, uint64_t fp, const Geo& g) {
    if constexpr (OP == OP_QUERY) return probe_ro<F, WPB, POL>(words, i2, fp);
    const uint64_t tag2 = POL == CKF_POLICY_OFFSET ? make_tag(fp, 1u, g) : fp;
    if constexpr (OP == OP_INSERT) return try_insert_t<F, WPB>(words, i2, tag2) >= 0;
    else return remove_tag_t<F, WPB>(words, i2, tag2) >= 0;
  }
};

// Unresolved insert after both buckets: hand it to the eviction pass.  `agg`
// selects warp aggregation (caller guarantees a converged warp).
__device__ __forceinline__ void enqueue_evict(const Sink& sk, bool need, uint32_t idx, uint64_t h) {
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
  if (pos < sk.rec_cap) sk.rec[pos] = ckf_record{idx, h, 0u, 0u};
  // queue overflow cannot happen through the facade (capacity = n); the key
  // is then reported as not stored
  else if (sk.ok) sk.ok[idx] = 0;
}

// ---- block-cooperative multi-split append ----

struct SplitSmem {
  uint32_t hist[kMaxBins];
  uint32_t start[kMaxBins];
  uint32_t gbase[kMaxBins];
  uint64_t h[kTile];
  uint32_t idx[kTile];
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

// Appends the block's valid (h, idx) items to bins out[bin*cap + ...]: items
// are counting-sorted by bin in shared memory first, so each bin's run is
// written with contiguous stores; one global atomic per (block, bin) reserves
// the run.  Items past a bin's capacity go to `ovf(h, idx)` instead.
template <int I, class Overflow>
__device__ __forceinline__ void block_append(const uint64_t (&h)[I], const uint32_t (&idx)[I], const uint32_t (&bin)[I],
                                             const bool (&v)[I], const Plan& pl, uint64_t* __restrict__ oh,
                                             uint32_t* __restrict__ ox, uint32_t* gcnt, SplitSmem& sm, Overflow&& ovf) {
  const int tid = threadIdx.x;
  for (uint32_t r = tid; r < pl.R; r += kTileThreads) sm.hist[r] = 0;
  __syncthreads();
  uint32_t rank[I];
#pragma unroll
  for (int j = 0; j < I; ++j) rank[j] = v[j] ? atomicAdd(&sm.hist[bin[j]], 1u) : 0u;
  __syncthreads();
  block_exclusive_scan(sm.hist, sm.start, pl.R, sm.warp_sums);
  for (uint32_t r = tid; r < pl.R; r += kTileThreads) {
    const uint32_t c = sm.hist[r];
    sm.gbase[r] = c ? atomicAdd(gcnt + r, c) : 0u;
  }
#pragma unroll
  for (int j = 0; j < I; ++j) {
    if (!v[j]) continue;
    const uint32_t p = sm.start[bin[j]] + rank[j];
    sm.h[p] = h[j];
    sm.idx[p] = idx[j];
    sm.bin[p] = (uint16_t)bin[j];
  }
  __syncthreads();
  const uint32_t total = sm.start[pl.R - 1] + sm.hist[pl.R - 1];
  for (uint32_t p = tid; p < total; p += kTileThreads) {
    const uint32_t r = sm.bin[p];
    const uint64_t off = (uint64_t)sm.gbase[r] + (p - sm.start[r]);
    if (off < pl.cap) {
      oh[r * pl.cap + off] = sm.h[p];
      ox[r * pl.cap + off] = sm.idx[p];
    } else {
      ovf(sm.h[p], sm.idx[p]);
    }
  }
  __syncthreads();
}

// ---- pass A: hash + bin by primary-bucket region ----

template <int OP, int F, int WPB, int POL>
__global__ void __launch_bounds__(kTileThreads) tile_bin_kernel(Geo g, Plan pl, uint64_t* words,
                                                                const uint64_t* __restrict__ keys, uint64_t n,
                                                                bool hashed, Work w, Sink sk, long long* occ) {
  __shared__ SplitSmem sm;
  uint32_t n_ok = 0;
  for (uint64_t t0 = blockIdx.x * (uint64_t)kTile; t0 < n; t0 += (uint64_t)gridDim.x * kTile) {
    uint64_t h[kTileItems];
    uint32_t idx[kTileItems], bin[kTileItems];
    bool v[kTileItems];
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) {
      const uint64_t i = t0 + j * kTileThreads + threadIdx.x;
      v[j] = i < n;
      h[j] = v[j] ? load_hash(keys, i, g.seed, hashed) : 0;
      idx[j] = (uint32_t)i;
      uint64_t fp, i1, i2;
      place<POL>(h[j], g, fp, i1, i2);
      bin[j] = bin_of(i1, pl);
    }
    // a full bin (adversarial keys): resolve that key in place, randomly
    block_append(h, idx, bin, v, pl, w.h1, w.x1, w.cnt1, sm, [&](uint64_t hh, uint32_t ii) {
      uint64_t fp, i1, i2;
      place<POL>(hh, g, fp, i1, i2);
      bool done = Logic<OP, F, WPB, POL>::first(words, i1, fp, g) || Logic<OP, F, WPB, POL>::second(words, i2, fp, g);
      if (done) {
        ++n_ok;
        if (OP != OP_INSERT) set_bit(sk.bits, ii);
      } else if (OP == OP_INSERT) {
        const uint64_t pos = atomicAdd(&sk.ctr->n_queued, 1ull);
        if (pos < sk.rec_cap) sk.rec[pos] = ckf_record{ii, hh, 0u, 0u};
        else if (sk.ok) sk.ok[ii] = 0;
      }
    });
  }
  block_count_add(n_ok, 0, sk.ctr, occ, OP == OP_DELETE ? -1 : +1);
}

// ---- pass B: primary buckets, bin by bin; misses re-binned by alternate region ----

template <int OP, int F, int WPB, int POL>
__global__ void __launch_bounds__(kTileThreads) tile_probe1_kernel(Geo g, Plan pl, uint64_t* words, Work w, Sink sk,
                                                                   long long* occ) {
  __shared__ SplitSmem sm;
  uint32_t n_ok = 0, n_alt = 0;
  const uint64_t tiles = (uint64_t)pl.R * pl.tiles_per_bin;
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const uint32_t r = (uint32_t)(t / pl.tiles_per_bin);
    const uint64_t off0 = (t % pl.tiles_per_bin) * kTile;
    const uint32_t c = w.cnt1[r];
    const uint64_t cnt = c < pl.cap ? c : pl.cap;
    if (off0 >= cnt) continue;  // block-uniform
    const uint64_t base = r * pl.cap;
    uint64_t h[kTileItems];
    uint32_t idx[kTileItems], bin[kTileItems];
    bool need[kTileItems];
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) {
      const uint64_t off = off0 + j * kTileThreads + threadIdx.x;
      const bool v = off < cnt;
      h[j] = v ? w.h1[base + off] : 0;
      idx[j] = v ? w.x1[base + off] : 0;
      uint64_t fp, i1, i2;
      place<POL>(h[j], g, fp, i1, i2);
      const bool done = v && Logic<OP, F, WPB, POL>::first(words, i1, fp, g);
      if (done) {
        ++n_ok;
        if (OP != OP_INSERT) set_bit(sk.bits, idx[j]);
      }
      need[j] = v && !done;
      n_alt += need[j];
      bin[j] = bin_of(i2, pl);
    }
    block_append(h, idx, bin, need, pl, w.h2, w.x2, w.cnt2, sm, [&](uint64_t hh, uint32_t ii) {
      uint64_t fp, i1, i2;
      place<POL>(hh, g, fp, i1, i2);
      if (Logic<OP, F, WPB, POL>::second(words, i2, fp, g)) {
        ++n_ok;
        if (OP != OP_INSERT) set_bit(sk.bits, ii);
      } else if (OP == OP_INSERT) {
        const uint64_t pos = atomicAdd(&sk.ctr->n_queued, 1ull);
        if (pos < sk.rec_cap) sk.rec[pos] = ckf_record{ii, hh, 0u, 0u};
        else if (sk.ok) sk.ok[ii] = 0;
      }
    });
  }
  block_count_add(n_ok, n_alt, sk.ctr, occ, OP == OP_DELETE ? -1 : +1);
}

// ---- pass C: alternate buckets, bin by bin ----

template <int OP, int F, int WPB, int POL>
__global__ void __launch_bounds__(kTileThreads) tile_probe2_kernel(Geo g, Plan pl, uint64_t* words, Work w, Sink sk,
                                                                   long long* occ) {
  uint32_t n_ok = 0;
  const uint64_t tiles = (uint64_t)pl.R * pl.tiles_per_bin;
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const uint32_t r = (uint32_t)(t / pl.tiles_per_bin);
    const uint64_t off0 = (t % pl.tiles_per_bin) * kTile;
    const uint32_t c = w.cnt2[r];
    const uint64_t cnt = c < pl.cap ? c : pl.cap;
    if (off0 >= cnt) continue;
    const uint64_t base = r * pl.cap;
#pragma unroll
    for (int j = 0; j < kTileItems; ++j) {
      const uint64_t off = off0 + j * kTileThreads + threadIdx.x;
      const bool v = off < cnt;
      const uint64_t hh = v ? w.h2[base + off] : 0;
      const uint32_t ii = v ? w.x2[base + off] : 0;
      uint64_t fp, i1, i2;
      place<POL>(hh, g, fp, i1, i2);
      const bool done = v && Logic<OP, F, WPB, POL>::second(words, i2, fp, g);
      if (done) {
        ++n_ok;
        if (OP != OP_INSERT) set_bit(sk.bits, ii);
      }
      if (OP == OP_INSERT) enqueue_evict(sk, v && !done, ii, hh);
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
      uint4 lo, hi;
      uint32_t q[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t nib = (b >> (4 * k)) & 0xF;
        q[k] = (nib & 1) | ((nib >> 1 & 1) << 8) | ((nib >> 2 & 1) << 16) | ((nib >> 3 & 1) << 24);
      }
      lo = make_uint4(q[0], q[1], q[2], q[3]);
      hi = make_uint4(q[4], q[5], q[6], q[7]);
      reinterpret_cast<uint4*>(out + i0)[0] = lo;
      reinterpret_cast<uint4*>(out + i0)[1] = hi;
    } else {
      for (uint64_t i = i0; i < n && i < i0 + 32; ++i) out[i] = (b >> (i - i0)) & 1u;
    }
  }
}

}  // namespace ckf
