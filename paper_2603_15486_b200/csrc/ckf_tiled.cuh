// ckf_tiled.cuh -- L2-tiled execution of large batches ("coarse dual-list").
//
// Why: one insert / query / delete touches one or two random 32-byte buckets.
// Measured on B200 (profiles/r01_probe_ceiling.txt), random 32 B sector reads
// top out at ~48 G/s at 512 MiB (~1.5 TB/s useful, a quarter of the 6.4 TB/s
// streaming peak) and a DRAM-resident CAS at ~24 G/s, while the same accesses
// inside an L2-resident 16-64 MiB window run at 100-150 G/s even with a
// concurrent multi-GB stream (profiles/r01_probe_atomics.txt,
// r01_probe_l2mix.txt).  When a batch holds many keys per bucket (the
// benchmark: 15 keys per bucket) the tiled path therefore
//
//   pass A  hashes every key once and appends a packed 8-byte record
//           (batch index | bucket offset in region | fingerprint) to TWO
//           lists: list A, binned by the L2-sized table region (R ≈ table /
//           16 MiB) of its primary bucket, and list B, binned by the region of
//           its alternate bucket.  Few bins -> each block writes long
//           contiguous runs and takes one counter atomic per bin per tile;
//   pass B  streams list A bin after bin with a flat grid: the region being
//           worked on is L2-resident, so the bucket access is an L2 hit; a
//           resolved key sets its bit in an L2-resident n-bit map;
//   pass C  streams list B the same way; keys whose bit is already set are
//           skipped, the rest try their alternate bucket.
// Every DRAM stream is sequential; no block synchronisation in the probe
// passes.  Semantics are unchanged: batch ops are concurrent and this is one
// legal schedule of them (every key tries i1 before i2, as in K:359-362).
// A record whose bin is full (adversarial keys) is parked as (hash, index) on
// an overflow list of capacity n that the same probe pass drains after the
// bins, so correctness never depends on the binning statistics.
#pragma once

#include "ckf_device.cuh"

namespace ckf {

enum { OP_QUERY = 0, OP_INSERT = 1, OP_DELETE = 2 };

constexpr int kTileThreads = 256;
constexpr int kTileItems = 8;
constexpr int kTile = kTileThreads * kTileItems;  // keys per pass-A tile
constexpr int kMaxBins = 128;                      // per list
constexpr int kCntStride = 32;                     // bin counters 128 B apart (one line each)
constexpr int kProbeRecs = 4;                      // records per thread per probe iteration

// Binning plan for one (table, batch) pair, computed on the host.
struct Plan {
  uint64_t div_magic;  // region = mulhi(bucket, div_magic) == bucket / rb  (bucket < 2^32)
  uint64_t cap;        // record slots per bin (multiple of kProbeRecs)
  uint32_t rb;         // buckets per region
  uint32_t R;          // bins per list
  uint32_t pb;         // fingerprint bits in a record
  uint32_t lb;         // bucket-offset bits in a record
};

__device__ __forceinline__ uint32_t bin_of(uint64_t bucket, const Plan& pl) {
  return (uint32_t)__umul64hi(bucket, pl.div_magic);
}

// record = index << (lb+pb) | (bucket - bin*rb) << pb | fp
__device__ __forceinline__ uint64_t pack_rec(uint64_t idx, uint64_t bucket, uint32_t bin, uint64_t fp,
                                             const Plan& pl) {
  return (idx << (pl.lb + pl.pb)) | ((bucket - (uint64_t)bin * pl.rb) << pl.pb) | fp;
}
__device__ __forceinline__ void unpack_rec(uint64_t rec, uint32_t bin, const Plan& pl, uint32_t& idx,
                                           uint64_t& bucket, uint64_t& fp) {
  idx = (uint32_t)(rec >> (pl.lb + pl.pb));
  fp = rec & ((1ull << pl.pb) - 1u);
  bucket = (uint64_t)bin * pl.rb + ((rec >> pl.pb) & ((1ull << pl.lb) - 1u));
}

// Workspace views (layout: layout_for in ckf_kernels.cu).
struct Work {
  uint32_t* cnt;    // [2][kMaxBins*kCntStride] records appended per bin (list A, list B; may exceed cap)
  unsigned long long* novf;  // [2 lines] overflow-list lengths
  uint64_t* list;   // [2][R*cap] records, list A then list B
  uint64_t* ovf_h;  // [2][n] hashes of keys whose bin was full (adversarial input only)
  uint32_t* ovf_x;  // [2][n] their batch indexes
  uint32_t* bits;   // [ceil(n/32)] resolved / result bit per key
};

// What happens to a resolved / unresolved key.
struct Sink {
  uint32_t* bits;         // resolved bit per key (query/delete: the result)
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
    if constexpr (OP == OP_QUERY) ld_bucket_ro<WPB>(words + bucket * WPB, w);
    else ld_bucket_rw<WPB>(words + bucket * WPB, w);
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

__device__ __forceinline__ void enqueue_evict_one(const Sink& sk, uint32_t idx, uint64_t h) {
  const uint64_t pos = atomicAdd(&sk.ctr->n_queued, 1ull);
  if (pos < sk.rec_cap) sk.rec[pos] = ckf_record{idx, h, 0u, 0u};
  else if (sk.ok) sk.ok[idx] = 0;  // queue overflow: reported as not stored
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
  else if (sk.ok) sk.ok[idx] = 0;
}

// ---- pass A: hash once, append to list A (primary region) and list B ----

constexpr int kSplitItems = 4;                          // keys per thread per split tile
constexpr int kSplitTile = kTileThreads * kSplitItems;  // keys per tile (2 records each)
constexpr int kWarps = kTileThreads / 32;

struct SplitSmem {
  uint32_t whist[kWarps][2 * kMaxBins];  // per-warp record count per virtual bin, then warp base
  uint32_t start[2 * kMaxBins];          // tile-level start of each virtual bin
  uint32_t gbase[2 * kMaxBins];          // reserved global offset of the tile's run
  uint32_t warp_sums[kWarps];
  uint64_t rec[2 * kSplitTile];
  uint8_t vbin[2 * kSplitTile];          // virtual bin = list * R + bin
};

// Warp-level multi-split rank: lanes with the same virtual bin are grouped
// with __match_any_sync; the group's first lane bumps the warp's private
// counter.  No shared-memory atomics (few bins would serialise them).
__device__ __forceinline__ uint32_t warp_rank(uint32_t vb, bool valid, uint32_t* whist_w) {
  const unsigned full = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const unsigned same = __match_any_sync(full, valid ? vb : 0x10000u + lane);
  const int leader = __ffs(same) - 1;
  uint32_t base = 0;
  if (valid && lane == leader) {
    base = whist_w[vb];
    whist_w[vb] = base + __popc(same);
  }
  base = __shfl_sync(full, base, leader);
  return base + __popc(same & ((1u << lane) - 1u));
}

template <int POL>
__global__ void __launch_bounds__(kTileThreads)
    tile_split_kernel(Geo g, Plan pl, const uint64_t* __restrict__ keys, uint64_t n, bool hashed, Work w) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SplitSmem& sm = *reinterpret_cast<SplitSmem*>(smem_raw);
  const uint64_t pol = evict_first_policy();
  const uint32_t V = 2 * pl.R;  // virtual bins (<= kTileThreads)
  const int tid = threadIdx.x, wid = tid >> 5;
  for (uint64_t t0 = blockIdx.x * (uint64_t)kSplitTile; t0 < n; t0 += (uint64_t)gridDim.x * kSplitTile) {
    for (uint32_t x = tid; x < kWarps * 2 * kMaxBins; x += kTileThreads) (&sm.whist[0][0])[x] = 0;
    __syncthreads();
    uint64_t rec[2 * kSplitItems];
    uint32_t vb[2 * kSplitItems], rk[2 * kSplitItems];
    bool v[kSplitItems];
#pragma unroll
    for (int j = 0; j < kSplitItems; ++j) {
      const uint64_t i = t0 + j * kTileThreads + tid;
      v[j] = i < n;
      const uint64_t h = v[j] ? load_hash(keys, i, g.seed, hashed) : 0;
      uint64_t fp, i1, i2;
      place<POL>(h, g, fp, i1, i2);
      const uint32_t ba = bin_of(i1, pl), bb = bin_of(i2, pl);
      rec[2 * j] = pack_rec(i, i1, ba, fp, pl);
      rec[2 * j + 1] = pack_rec(i, i2, bb, fp, pl);
      vb[2 * j] = ba;
      vb[2 * j + 1] = pl.R + bb;
    }
#pragma unroll
    for (int j = 0; j < 2 * kSplitItems; ++j) rk[j] = warp_rank(vb[j], v[j / 2], sm.whist[wid]);
    __syncthreads();
    // per virtual bin: column prefix over warps, tile total, block scan, reservation
    uint32_t total = 0;
    if ((uint32_t)tid < V) {
#pragma unroll
      for (int q = 0; q < kWarps; ++q) {
        const uint32_t c = sm.whist[q][tid];
        sm.whist[q][tid] = total;
        total += c;
      }
    }
    {  // exclusive block scan of `total` (one virtual bin per thread)
      const int lane = tid & 31;
      uint32_t x = total;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
      }
      if (lane == 31) sm.warp_sums[wid] = x;
      __syncthreads();
      uint32_t off = 0;
#pragma unroll
      for (int q = 0; q < kWarps; ++q) off += q < wid ? sm.warp_sums[q] : 0u;
      if ((uint32_t)tid < V) {
        sm.start[tid] = off + x - total;
        const uint32_t list = (uint32_t)tid >= pl.R;
        sm.gbase[tid] =
            total ? atomicAdd(w.cnt + (size_t)list * kMaxBins * kCntStride + (size_t)(tid - list * pl.R) * kCntStride,
                              total)
                  : 0u;
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 2 * kSplitItems; ++j) {
      if (!v[j / 2]) continue;
      const uint32_t p = sm.start[vb[j]] + sm.whist[wid][vb[j]] + rk[j];
      sm.rec[p] = rec[j];
      sm.vbin[p] = (uint8_t)vb[j];
    }
    __syncthreads();
    const uint32_t nrec = 2 * (uint32_t)min((uint64_t)kSplitTile, n - t0);
    for (uint32_t p = tid; p < nrec; p += kTileThreads) {
      const uint32_t vv = sm.vbin[p];
      const uint32_t list = vv >= pl.R, r = vv - list * pl.R;
      const uint64_t off = (uint64_t)sm.gbase[vv] + (p - sm.start[vv]);
      if (off < pl.cap) {
        st_stream_ef(w.list + (uint64_t)list * pl.R * pl.cap + (uint64_t)r * pl.cap + off, sm.rec[p], pol);
      } else {
        // a full bin (adversarial keys): park (hash, index) on the overflow
        // list that the matching probe pass drains after its bins
        const uint32_t ii = (uint32_t)(sm.rec[p] >> (pl.lb + pl.pb));
        const uint64_t k = keys[ii];
        const uint64_t pos = atomicAdd(w.novf + list * 16, 1ull);
        w.ovf_h[(uint64_t)list * n + pos] = hashed ? k : xxh64(k, g.seed);
        w.ovf_x[(uint64_t)list * n + pos] = ii;
      }
    }
    __syncthreads();
  }
}

// ---- passes B and C: flat streams over list A (primary) / list B (alternate) ----

template <int OP, int F, int WPB, int POL, bool SECOND>
__global__ void __launch_bounds__(kTileThreads)
    tile_probe_kernel(Geo g, Plan pl, uint64_t* words, Work w, Sink sk, long long* occ, uint64_t n) {
  using Lg = Logic<OP, F, WPB, POL>;
  const uint64_t pol = evict_first_policy();
  const uint64_t* list = w.list + (SECOND ? (uint64_t)pl.R * pl.cap : 0);
  const uint32_t* cnt = w.cnt + (SECOND ? (size_t)kMaxBins * kCntStride : 0);
  const uint64_t total = (uint64_t)pl.R * pl.cap;  // positions (multiple of kProbeRecs)
  const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  uint32_t n_ok = 0, n_alt = 0;

  // kProbeRecs keys: skip the resolved ones (pass C), fetch all buckets, act
  auto work = [&](const uint32_t (&idx)[kProbeRecs], const uint64_t (&bk)[kProbeRecs],
                  const uint64_t (&fp)[kProbeRecs], bool (&go)[kProbeRecs]) {
#pragma unroll
    for (int q = 0; q < kProbeRecs; ++q) {
      if (SECOND && go[q]) {  // already resolved by pass B?
        go[q] = !((__ldcg(sk.bits + (idx[q] >> 5)) >> (idx[q] & 31)) & 1u);
        n_alt += go[q];
      }
    }
    uint64_t wv[kProbeRecs][WPB];
#pragma unroll
    for (int q = 0; q < kProbeRecs; ++q)
      if (go[q]) Lg::fetch(words, bk[q], wv[q]);
    bool fail[kProbeRecs];
#pragma unroll
    for (int q = 0; q < kProbeRecs; ++q) {
      const bool done = go[q] && Lg::act(words, bk[q], fp[q], SECOND ? Lg::tag2(fp[q], g) : fp[q], wv[q]);
      fail[q] = go[q] && !done;
      if (done) {
        ++n_ok;
        if (OP != OP_INSERT || !SECOND) set_bit(sk.bits, idx[q]);
      }
    }
    if (OP == OP_INSERT && SECOND) {
#pragma unroll
      for (int q = 0; q < kProbeRecs; ++q) enqueue_evict(sk, fail[q], idx[q], g);
    }
  };

  for (uint64_t p0 = gtid * kProbeRecs; p0 < total; p0 += nthreads * kProbeRecs) {
    const uint32_t r = (uint32_t)(p0 / pl.cap);
    const uint64_t off = p0 - (uint64_t)r * pl.cap;
    const uint32_t c = cnt[(size_t)r * kCntStride];
    const uint64_t lim = c < pl.cap ? c : pl.cap;
    uint64_t rec[kProbeRecs];
    if (off + kProbeRecs <= lim) {
      asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u64 {%0,%1,%2,%3}, [%4], %5;"
                   : "=l"(rec[0]), "=l"(rec[1]), "=l"(rec[2]), "=l"(rec[3])
                   : "l"(list + p0), "l"(pol));
    } else {
#pragma unroll
      for (int q = 0; q < kProbeRecs; ++q) rec[q] = off + q < lim ? list[p0 + q] : ~0ull;
    }
    uint64_t fp[kProbeRecs], bk[kProbeRecs];
    uint32_t idx[kProbeRecs];
    bool go[kProbeRecs];
#pragma unroll
    for (int q = 0; q < kProbeRecs; ++q) {
      go[q] = rec[q] != ~0ull;
      unpack_rec(rec[q], r, pl, idx[q], bk[q], fp[q]);
    }
    work(idx, bk, fp, go);
  }

  // drain this pass's overflow list (keys whose bin was full)
  const unsigned long long nov = *(volatile unsigned long long*)(w.novf + (SECOND ? 16 : 0));
  const uint64_t* oh = w.ovf_h + (SECOND ? n : 0);
  const uint32_t* ox = w.ovf_x + (SECOND ? n : 0);
  for (uint64_t p0 = gtid * kProbeRecs; p0 < nov; p0 += nthreads * kProbeRecs) {
    uint64_t fp[kProbeRecs], bk[kProbeRecs];
    uint32_t idx[kProbeRecs];
    bool go[kProbeRecs];
#pragma unroll
    for (int q = 0; q < kProbeRecs; ++q) {
      go[q] = p0 + q < nov;
      uint64_t i1 = 0, i2 = 0;
      fp[q] = 1;
      idx[q] = go[q] ? ox[p0 + q] : 0;
      if (go[q]) place<POL>(oh[p0 + q], g, fp[q], i1, i2);
      bk[q] = SECOND ? i2 : i1;
    }
    work(idx, bk, fp, go);
  }
  block_count_add(n_ok, n_alt, sk.ctr, occ, OP == OP_DELETE ? -1 : +1);
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
