// ckf_region.cuh -- shared-memory region schedule for large batches.
//
// Why (measured, profiles/r01s2_*): a bucket access that misses L2 costs a
// random HBM row activation (~48 G sectors/s at 512 MiB, a quarter of the
// streaming rate), and even an L2-resident one is bounded by the L2's random
// request rate (~265 G loads/s, ~120 G CAS/s).  The L2-tiled schedule in
// ckf_tiled.cuh got the buckets into L2 but stayed bound by those request
// rates.  This schedule moves every bucket access into shared memory:
//
//   bin      hash + placement, records binned by COARSE table region of the
//            key's primary bucket (R1 <= 512 bins);
//   split    each coarse bin is split into F2 FINE bins (R = R1*F2 regions of
//            rb buckets, rb*bucket_bytes <= 128 KiB);
//   probe    one persistent CTA per SM takes fine regions in turn: the region's
//            table slice is bulk-copied (TMA, cp.async.bulk) into shared memory,
//            the region's records stream through a shared-memory ring of
//            bulk-copied chunks, every op runs on the shared-memory copy
//            (atom.shared.cas for mutations), and the slice is bulk-copied back;
//   phase 2  keys their primary bucket did not answer (not found / full /
//            tag absent) are appended to per-CTA dense miss lists during the
//            probe, binned + split again by their alternate bucket and probed
//            again; inserts still unplaced go to the eviction pass.
// Every DRAM stream is sequential.  All bucket reads and CASes hit shared
// memory.  Concurrency semantics are unchanged: one legal concurrent schedule
// of the batch in which every key tries i1 before i2 (K:355-362); a region is
// owned by exactly one CTA while it is resident, so the shared-memory copy is
// the only copy being mutated.
#pragma once

#include <type_traits>

#include "ckf_ops.cuh"

namespace ckf {

// ---------------------------------------------------------------------------
// async-proxy primitives: mbarriers and 1-D bulk copies (TMA)
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t saddr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
      "@!p bra WAIT_%=;\n}\n" ::"r"(saddr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   saddr(dst)),
               "l"(src), "r"(bytes), "r"(saddr(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(saddr(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// ---------------------------------------------------------------------------
// shared-memory bucket operations (same decisions as the global ones in
// ckf_device.cuh: TryInsert K:158-180, TryRemove K:202-221, Find K:183-199)
// ---------------------------------------------------------------------------

template <int WPB>
__device__ __forceinline__ void lds_bucket(uint32_t a, uint64_t (&w)[WPB]) {
  if constexpr (WPB == 1) {
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(w[0]) : "r"(a) : "memory");
  } else {
#pragma unroll
    for (int s = 0; s < WPB / 2; ++s)
      asm volatile("ld.shared.v2.u64 {%0,%1}, [%2];" : "=l"(w[2 * s]), "=l"(w[2 * s + 1]) : "r"(a + 16 * s) : "memory");
  }
}

// Bank-spread bucket gather (queries): lane l fetches the bucket's 16 B chunks
// starting at chunk (l mod chunks), so the lanes of one LDS.128 split over
// different bank quads (random 32 B gathers otherwise pay ~3x in bank
// conflicts; measured -17 % probe time).  Word order in w is rotated -- fine
// for match_any, which ORs over the words.
template <int WPB>
__device__ __forceinline__ void lds_bucket_spread(uint32_t a, uint64_t (&w)[WPB]) {
  if constexpr (WPB < 4) {
    lds_bucket<WPB>(a, w);
  } else {
    constexpr int C = WPB / 2;  // 16 B chunks
    const int r = (int)(threadIdx.x & (C - 1));
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const uint32_t off = (uint32_t)(((k + r) & (C - 1)) * 16);
      asm volatile("ld.shared.v2.u64 {%0,%1}, [%2];" : "=l"(w[2 * k]), "=l"(w[2 * k + 1]) : "r"(a + off) : "memory");
    }
  }
}

__device__ __forceinline__ uint64_t cas_shared(uint32_t a, uint64_t cmp, uint64_t val) {
  uint64_t old;
  asm volatile("atom.shared.cas.b64 %0, [%1], %2, %3;" : "=l"(old) : "r"(a), "l"(cmp), "l"(val) : "memory");
  return old;
}

// ---- 32-bit SWAR on shared-memory snapshots ----
// A lane never carries into its neighbour in ((x & ~H) + ~H), so each 32-bit
// half of a word is handled on its own: exact per-lane zero indicators
// (the carry-out form of W:9-16) in 3 ops per half.
template <int F>
__device__ __forceinline__ uint32_t zind32(uint32_t x) {
  constexpr uint32_t H = (uint32_t)Lanes<F>::kHigh;
  return ~(((x & ~H) + ~H) | x) & H;
}
// bit s of the result <=> lane s of x is zero (F = 8 or 16)
template <int F>
__device__ __forceinline__ uint32_t lane_mask(uint64_t x) {
  const uint32_t zl = zind32<F>((uint32_t)x), zh = zind32<F>((uint32_t)(x >> 32));
  // indicators at bit 7 of bytes 0..3 -> bits 28..31 (no carries: all partial
  // products land on distinct bits)
  if constexpr (F == 32) {
    return (zl >> 31) | ((zh >> 31) << 1);
  } else if constexpr (F == 16) {
    return (__byte_perm(zl, zh, 0x7531) * 0x00204081u) >> 28;
  } else {
    return ((zl * 0x00204081u) >> 28) | (((zh * 0x00204081u) >> 28) << 4);
  }
}

// Any lane of the bucket equal to fp (payload-only compare for the offset
// policy, K:451-453).  (x - L) & ~x & H is nonzero iff some lane of x is zero:
// exact for the boolean.  32-bit halves are tested on
// their own (still exact).
template <int F, int WPB, int POL>
__device__ __forceinline__ bool match_any(const uint64_t (&w)[WPB], uint64_t fp) {
  using L = Lanes<F>;
  constexpr uint32_t H = (uint32_t)L::kHigh, Lo = (uint32_t)L::kLow;
  constexpr uint32_t keep = POL == CKF_POLICY_OFFSET ? ~H : ~0u;
  const uint32_t pat = (uint32_t)L::bcast(fp);
  uint32_t acc = 0;
#pragma unroll
  for (int j = 0; j < WPB; ++j) {
    const uint32_t a = ((uint32_t)w[j] & keep) ^ pat, b = ((uint32_t)(w[j] >> 32) & keep) ^ pat;
    acc |= ((a - Lo) & ~a) | ((b - Lo) & ~b);
  }
  return (acc & H) != 0;
}

// kB-bit mask over the bucket's slots (slot = word * tpw + lane) of lanes equal
// to `pat` (pat = 0: empty lanes); 32-bit when the bucket has <= 32 slots
template <int F, int WPB>
using SlotMask = typename std::conditional<(WPB * 64 / F <= 32), uint32_t, uint64_t>::type;

template <int F, int WPB>
__device__ __forceinline__ SlotMask<F, WPB> slot_mask(const uint64_t (&w)[WPB], uint64_t pat) {
  constexpr int kTpw = 64 / F;
  SlotMask<F, WPB> m = 0;
#pragma unroll
  for (int j = 0; j < WPB; ++j) m |= (SlotMask<F, WPB>)lane_mask<F>(w[j] ^ pat) << (j * kTpw);
  return m;
}

// First slot of `m` in the reference scan order: words from `start` wrapping,
// lowest lane first (K:166-179, K:207-220).  -1 if none.
template <int F, int WPB>
__device__ __forceinline__ int first_slot(SlotMask<F, WPB> m, int start) {
  constexpr int kTpw = 64 / F, kB = WPB * kTpw;
  const int sh = start * kTpw;
  if constexpr (kB <= 32) {
    const uint32_t full = kB == 32 ? ~0u : ((1u << kB) - 1u);
    const uint32_t rot = kB == 32 ? __funnelshift_r(m, m, sh) : (((m >> sh) | (m << ((kB - sh) & 31))) & full);
    if (!rot) return -1;
    const int f = __ffs((int)rot) - 1 + sh;
    return f >= kB ? f - kB : f;
  } else {
    const uint64_t rot = sh ? (m >> sh) | (m << (64 - sh)) : m;
    if (!rot) return -1;
    const int f = __ffsll((long long)rot) - 1 + sh;
    return f >= kB ? f - kB : f;
  }
}

template <int WPB>
__device__ __forceinline__ uint64_t pick(const uint64_t (&w)[WPB], int j) {
  uint64_t r = w[0];
#pragma unroll
  for (int q = 1; q < WPB; ++q)
    if (j == q) r = w[q];
  return r;
}

// Lost CAS: the word we lost on now holds `old`; refresh only that word's
// lanes in the slot mask (a retry costs ~15 instructions instead of a rescan;
// under SIMT the whole warp pays for any lane's retry).
template <int F, int WPB>
__device__ __forceinline__ void refresh_word(SlotMask<F, WPB>& m, uint64_t (&w)[WPB], int j, uint64_t old,
                                             uint64_t pat) {
  constexpr int kTpw = 64 / F;
  constexpr SlotMask<F, WPB> kLanes = (SlotMask<F, WPB>)((1ull << kTpw) - 1u);
#pragma unroll
  for (int q = 0; q < WPB; ++q)
    if (j == q) w[q] = old;
  m = (m & ~(kLanes << (j * kTpw))) | ((SlotMask<F, WPB>)lane_mask<F>(old ^ pat) << (j * kTpw));
}

// TryInsert on a shared-memory bucket (a = its shared address, w = snapshot).
template <int F, int WPB>
__device__ __forceinline__ bool smem_insert(uint32_t a, uint64_t tag, uint64_t (&w)[WPB]) {
  constexpr int kTpw = 64 / F, kB = WPB * kTpw;
  const int start = (int)(tag % kB) / kTpw;
  SlotMask<F, WPB> m = slot_mask<F, WPB>(w, 0);
  while (true) {
    const int slot = first_slot<F, WPB>(m, start);
    if (slot < 0) return false;
    const int j = slot / kTpw, lane = slot % kTpw;
    const uint64_t bw = pick<WPB>(w, j);
    const uint64_t old = cas_shared(a + 8u * j, bw, bw | (tag << (lane * F)));
    if (old == bw) return true;
    refresh_word<F, WPB>(m, w, j, old, 0);
  }
}

// TryRemove on a shared-memory bucket: full-lane match (K:476-480).
template <int F, int WPB>
__device__ __forceinline__ bool smem_remove(uint32_t a, uint64_t tag, uint64_t (&w)[WPB]) {
  constexpr int kTpw = 64 / F, kB = WPB * kTpw;
  const int start = (int)(tag % kB) / kTpw;
  const uint64_t pat = Lanes<F>::bcast(tag);
  SlotMask<F, WPB> m = slot_mask<F, WPB>(w, pat);
  while (true) {
    const int slot = first_slot<F, WPB>(m, start);
    if (slot < 0) return false;
    const int j = slot / kTpw, lane = slot % kTpw;
    const uint64_t bw = pick<WPB>(w, j);
    const uint64_t old = cas_shared(a + 8u * j, bw, bw & ~(Lanes<F>::kLaneMask << (lane * F)));
    if (old == bw) return true;
    refresh_word<F, WPB>(m, w, j, old, pat);
  }
}

// One attempt of smem_insert / smem_remove: 0 = no candidate lane in the
// snapshot, 1 = done, 2 = the CAS lost (the probe defers the record to a
// compacted retry batch instead of re-running the whole warp's CAS body).
template <bool kInsert, int F, int WPB>
__device__ __forceinline__ int smem_try1(uint32_t a, uint64_t tag, const uint64_t (&w)[WPB]) {
  constexpr int kTpw = 64 / F, kB = WPB * kTpw;
  const int start = (int)(tag % kB) / kTpw;
  const int slot = first_slot<F, WPB>(slot_mask<F, WPB>(w, kInsert ? 0ull : Lanes<F>::bcast(tag)), start);
  if (slot < 0) return 0;
  const int j = slot / kTpw, lane = slot % kTpw;
  const uint64_t bw = pick<WPB>(w, j);
  const uint64_t nw = kInsert ? bw | (tag << (lane * F)) : bw & ~(Lanes<F>::kLaneMask << (lane * F));
  return cas_shared(a + 8u * j, bw, nw) == bw ? 1 : 2;
}

// Region-schedule results start all-true; only keys that end up negative /
// not deleted cost a (random, L2-resident) bitmap update.
__device__ __forceinline__ void clear_bit(uint32_t* bits, uint32_t i) { atomicAnd(bits + (i >> 5), ~(1u << (i & 31))); }

// ---------------------------------------------------------------------------
// plan, records, workspace
// ---------------------------------------------------------------------------

constexpr int kRegionSmem = 128 * 1024;  // table bytes of one fine region in shared memory
constexpr int kRMaxCoarse = 512;

// Record (8 B): index << ish | alt << (ish - 1) | bucket offset in its region << pb | fp,
// ish = pb + lrbc + 1: the index takes whatever the offset and fingerprint leave
// (64 - ish >= ceil_log2(chunk + 1) bits; the host chunks larger batches).
// `alt` marks a record of the key's alternate bucket.
struct RPlan {
  uint64_t cap1;     // record slots per coarse bin (even)
  uint64_t capf;     // record slots per fine bin (even)
  uint32_t R1;       // coarse bins
  uint32_t lrbc;     // log2 buckets per coarse region
  uint32_t F2;       // fine regions per coarse region
  uint32_t lrb;      // log2 buckets per fine region
  uint32_t R;        // fine regions = R1 * F2 (the last ones may be empty)
  uint32_t pb;       // fingerprint bits in a record
  uint32_t ish;      // index shift: pb + lrbc + 1 (8-byte records)
  uint64_t chunk;    // keys per region run (a call of n > chunk keys runs ceil(n / chunk) of them)
  uint32_t rbytes;   // record bytes: 8, or 16 for f = 32 (RecT)
};

// 16-byte record of f = 32 filters, whose 32-bit fingerprint leaves no room
// for an index in 64 bits: lo = offset in its region << 32 | fp, hi = index <<
// 1 | alt; hi all ones = filler.
struct __align__(16) Rec16 {
  uint64_t lo, hi;
};

// The record of an f-bit filter and its fields.  8 B for f <= 16 (the
// default, layout above), 16 B for f = 32.
template <int F>
struct RecT {
  static constexpr bool kWide = F == 32;
  using T = typename std::conditional<kWide, Rec16, uint64_t>::type;
  static constexpr uint32_t kBytes = sizeof(T);
  static constexpr bool kPadEven = !kWide;  // bulk copies move 16 B granules: 8 B runs pad to even length
  static __device__ __forceinline__ T pack(uint64_t idx, uint32_t alt, uint64_t off, uint64_t fp, const RPlan& pl) {
    if constexpr (kWide) return Rec16{(off << 32) | fp, (idx << 1) | alt};
    else return (idx << pl.ish) | ((uint64_t)alt << (pl.ish - 1)) | (off << pl.pb) | fp;
  }
  static __device__ __forceinline__ uint32_t idx(const T& r, const RPlan& pl) {
    if constexpr (kWide) return (uint32_t)(r.hi >> 1);
    else return (uint32_t)(r >> pl.ish);
  }
  static __device__ __forceinline__ uint32_t alt(const T& r, const RPlan& pl) {
    if constexpr (kWide) return (uint32_t)r.hi & 1u;
    else return (uint32_t)(r >> (pl.ish - 1)) & 1u;
  }
  // the offset field (bucket in the record's region) masked to `mask`
  static __device__ __forceinline__ uint32_t off(const T& r, const RPlan& pl, uint32_t mask) {
    if constexpr (kWide) return (uint32_t)(r.lo >> 32) & mask;
    else return (uint32_t)(r >> pl.pb) & mask;
  }
  static __device__ __forceinline__ uint64_t fp(const T& r, const RPlan& pl) {
    if constexpr (kWide) return r.lo & 0xFFFFFFFFull;
    else return r & ((1ull << pl.pb) - 1u);
  }
  // coarse record -> fine record: drop the offset bits above the fine region
  static __device__ __forceinline__ T refine(const T& r, const RPlan& pl) {
    const uint64_t drop = (uint64_t)((1u << (pl.lrbc - pl.lrb)) - 1u) << pl.lrb;
    if constexpr (kWide) return Rec16{r.lo & ~(drop << 32), r.hi};
    else return r & ~(drop << pl.pb);
  }
  static __device__ __forceinline__ T filler() {
    if constexpr (kWide) return Rec16{~0ull, ~0ull};
    else return ~0ull;
  }
  static __device__ __forceinline__ bool is_filler(const T& r) {
    if constexpr (kWide) return r.hi == ~0ull;
    else return r == ~0ull;
  }
};

struct RWork {
  uint32_t* cnt1;   // [R1 * kCntStride] coarse bin fill
  uint32_t* cntf;   // [R * kCntStride] fine bin fill
  void* bin1;       // [R1 * cap1] coarse bins of records (RecT)
  void* binf;       // [R * capf] fine bins
  uint4* miss;      // [grid * seg] per-probe-CTA dense segments of phase-1 misses {idx, fp, i2 lo, i2 hi}
  uint32_t* n_miss; // [grid] entries per segment
  uint64_t seg;     // entries per segment
  uint32_t* bits;   // [ceil(n/32)] result bitmap (query / delete)
  uint32_t* mode;   // [2] mode[0] nonzero: results start all-true and final negatives clear their bit;
                    // zero: results start all-false and hits set theirs (query batches
                    // sampled as mostly negative)
  uint32_t* room;   // insert: [m/32] bit i = bucket i has an empty lane (RoomMap, ckf_device.cuh)
};

// What to do with a record that finds its bin full (adversarial inputs only):
// resolve it in place on the global table -- legal here because no region is
// resident in shared memory while the bin / split kernels run.
template <int OP, int F, int WPB, int POL>
__device__ __forceinline__ void resolve_direct(uint64_t* words, const Geo& g, const RPlan& pl,
                                               const typename RecT<F>::T& rec, uint64_t bucket, const Sink& sk,
                                               const uint32_t* w_mode, uint32_t& n_ok, uint32_t& n_alt) {
  using Lg = Logic<OP, F, WPB, POL>;
  using RT = RecT<F>;
  const uint32_t idx = RT::idx(rec, pl);
  const uint64_t fp = RT::fp(rec, pl);
  const bool phase2 = RT::alt(rec, pl);  // the record is of the key's alternate bucket
  uint64_t c;
  bool done;
  if (phase2) {
    done = Lg::second(words, bucket, fp, g);
  } else {
    done = Lg::first(words, bucket, fp, g);
    if (!done) {
      ++n_alt;
      done = Lg::second(words, alt_index<POL>(bucket, fp, 0, g, c), fp, g);
    }
  }
  if (done) {
    if (OP != OP_QUERY) ++n_ok;
    if (OP == OP_QUERY && !*w_mode) set_bit(sk.bits, idx);
  } else if (OP != OP_INSERT) {
    if (*w_mode) clear_bit(sk.bits, idx);
  } else {
    const uint64_t k = sk.keys[idx];
    enqueue_evict_one(sk, idx, sk.hashed ? k : xxh64(k, g.seed));
  }
}

// ---------------------------------------------------------------------------
// bin: hash + placement, binned by coarse region (block counting sort, one
// global reservation per (tile, bin), contiguous runs out)
// ---------------------------------------------------------------------------

constexpr int kBThreads = 256;
constexpr int kBItems = 16;
constexpr int kBTile = kBThreads * kBItems;  // records per tile
// Runs go out as TMA bulk copies, which need 16 B granules: a run of odd
// length is padded with one filler record (all ones: its index field would be
// 2^(64-ish) - 1, never a key, as a run holds < 2^(64-ish) - 1 keys) that every
// consumer skips.
template <class T>
struct BinSmemT {
  T rec[kBTile + kRMaxCoarse];         // sorted tile (8 B records: runs padded to even length)
  uint32_t cnt[kRMaxCoarse];           // records per bin in this tile
  uint2 sg[kRMaxCoarse];               // {run start in rec, run start in the bin}
  uint32_t warp_sums[kBThreads / 32];
};
template <int F>
using BinSmem = BinSmemT<typename RecT<F>::T>;

// sm.cnt (records per bin) -> sm.sg.x (exclusive scan of the padded run
// lengths) and sm.sg.y (one global reservation per non-empty bin)
template <int F>
__device__ __forceinline__ void bin_reserve(uint32_t nb, uint32_t* gcnt, BinSmem<F>& sm) {
  constexpr bool kBulk = RecT<F>::kPadEven;
  constexpr int NW = kBThreads / 32;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t per = (nb + kBThreads - 1) / kBThreads;  // <= 2
  const uint32_t lo = min(tid * per, nb), hi = min(lo + per, nb);
  uint32_t c[2], gb[2], sum = 0;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const uint32_t r = lo + k;
    c[k] = r < hi ? (kBulk ? (sm.cnt[r] + 1u) & ~1u : sm.cnt[r]) : 0u;
    gb[k] = c[k] ? atomicAdd(gcnt + (size_t)r * kCntStride, c[k]) : 0u;
    sum += c[k];
  }
  uint32_t x = sum;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) sm.warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t v = lane < NW ? sm.warp_sums[lane] : 0, s = v;
#pragma unroll
    for (int d = 1; d < NW; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, s, d);
      if (lane >= d) s += y;
    }
    if (lane < NW) sm.warp_sums[lane] = s - v;
  }
  __syncthreads();
  uint32_t run = sm.warp_sums[wid] + x - sum;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const uint32_t r = lo + k;
    if (r < hi) {
      sm.sg[r] = make_uint2(run, gb[k]);
      if (kBulk && (sm.cnt[r] & 1u)) sm.rec[run + sm.cnt[r]] = RecT<F>::filler();
      run += c[k];
    }
  }
}

template <class T>
__device__ __forceinline__ void bin_place(BinSmemT<T>& sm, uint32_t b, uint32_t rank, const T& rc) {
  sm.rec[sm.sg[b].x + rank] = rc;
}

// Sends every (tile, bin) run to its bin with one bulk copy.  A run that does
// not fit its bin (adversarial inputs only) goes record by record: the part
// that fits by plain stores, the rest to ovf(rec, bin).  Caller: all threads,
// after bin_place; shared memory is released by bin_release().
template <int F, class Ovf>
__device__ __forceinline__ void bin_write(uint32_t nb, typename RecT<F>::T* __restrict__ out, uint64_t cap,
                                          BinSmem<F>& sm, Ovf&& ovf) {
  using RT = RecT<F>;
  using T = typename RT::T;
  fence_async_smem();  // this thread's placements -> visible to the bulk copies
  __syncthreads();
  bool issued = false;
  for (uint32_t r = threadIdx.x; r < nb; r += kBThreads) {
    const uint32_t c = sm.cnt[r];
    if (!c) continue;
    const uint32_t cr = RT::kPadEven ? (c + 1u) & ~1u : c, st = sm.sg[r].x, gb = sm.sg[r].y;
    T* dst = out + (uint64_t)r * cap;
    if ((uint64_t)gb + cr <= cap) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + gb),
                   "r"(saddr(&sm.rec[st])), "r"(cr * RT::kBytes)
                   : "memory");
      issued = true;
    } else {
      for (uint32_t k = 0; k < c; ++k) {
        const T rc = sm.rec[st + k];
        if ((uint64_t)gb + k < cap) dst[gb + k] = rc;
        else ovf(rc, r);
      }
      if (RT::kPadEven && (c & 1u) && (uint64_t)gb + c < cap) dst[gb + c] = RT::filler();
    }
  }
  if (issued) asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// Before the tile's shared memory is rewritten: this thread's bulk copies have
// read it (the caller synchronizes the block afterwards).
__device__ __forceinline__ void bin_release() { bulk_wait_read(); }

// SRC_KEYS: the batch's keys (or hashes), one record per key for its primary
// bucket.  SRC_MISS: phase-1 misses {idx, fp, i2} from probe-CTA segment
// blockIdx.y, one record for the alternate bucket.
enum { SRC_KEYS = 0, SRC_MISS = 1, SRC_KEYS_DUAL = 2 };

#ifndef CKF_BIN_BLOCKS
#define CKF_BIN_BLOCKS 3  // (measured: 4 per SM -- 64 registers, spills -- is slower)
#endif
constexpr int kBinBlocks = CKF_BIN_BLOCKS;  // resident bin CTAs per SM

template <int OP, int F, int WPB, int POL, int SRC>
__global__ void __launch_bounds__(kBThreads, kBinBlocks)
    region_bin_kernel(Geo g, RPlan pl, uint64_t* words, const uint64_t* __restrict__ keys, uint64_t n_keys, bool hashed,
                      RWork w, Sink sk, long long* occ) {
  using RT = RecT<F>;
  using T = typename RT::T;
  extern __shared__ __align__(16) uint8_t bsm_raw[];  // sizeof(BinSmem<F>), dynamic (> 48 KiB)
  BinSmem<F>& sm = *reinterpret_cast<BinSmem<F>*>(bsm_raw);
  // dual: a query batch sampled as mostly negative gets an i1 AND an i2 record
  // per key here (no phase 2); the tile then holds kBTile / 2 keys
  constexpr bool kKeys = SRC != SRC_MISS;
  constexpr bool dual = OP == OP_QUERY && SRC == SRC_KEYS_DUAL;
  // query batches launch both key variants; the one that does not match the
  // sampled mode exits (dual is a compile-time property of the tile loop)
  if constexpr (OP == OP_QUERY && kKeys)
    if ((w.mode[0] == 0) != dual) return;
  const uint64_t KT = dual ? kBTile / 2 : kBTile;  // keys (items) per tile
  const uint64_t pol = evict_first_policy();
  const uint32_t lmask = (1u << pl.lrbc) - 1u;
  const uint64_t n = kKeys ? n_keys : w.n_miss[blockIdx.y];
  const bool al16 = ((uintptr_t)keys & 15) == 0;  // 256-bit pair loads need 16 B alignment
  const uint4* ms = w.miss + (uint64_t)blockIdx.y * w.seg;
  uint32_t n_ok = 0, n_alt = 0;
  for (uint64_t t0 = blockIdx.x * KT; t0 < n; t0 += (uint64_t)gridDim.x * KT) {
    if (threadIdx.x == 0) {
      const uint64_t nx = t0 + (uint64_t)gridDim.x * KT;
      if (kKeys && nx < n && n - nx >= 4) {  // 16 B-aligned window inside the next tile
        const uintptr_t lo = ((uintptr_t)(keys + nx) + 15) & ~(uintptr_t)15;
        const uintptr_t hi = (uintptr_t)(keys + nx + min(KT, n - nx)) & ~(uintptr_t)15;
        if (hi > lo) prefetch_l2((const void*)lo, (uint32_t)(hi - lo));
      }
    }
    bin_release();
    for (uint32_t r = threadIdx.x; r < pl.R1; r += kBThreads) sm.cnt[r] = 0;
    T rec[kBItems];
    uint32_t pk[kBItems];  // bin << 16 | rank; 0xFFFFFFFF = no record
    if constexpr (kKeys) {
      // item q of thread t: key t0 + (q / 2) * 2 * kBThreads + 2t + (q % 2) (pairs
      // of 16 B, coalesced); dual: items [0, kBItems/2) are keys, the rest
      // their i2 records.  The record's index field advances by a running
      // 64-bit add (rec = idx << ish | ...).
      const bool full = t0 + KT <= n;  // block-uniform: no bounds checks
      uint64_t kk[kBItems];
#pragma unroll
      for (int q = 0; q < kBItems / 2; ++q) {
        const uint64_t i = t0 + (uint64_t)q * 2 * kBThreads + 2 * threadIdx.x;
        if (dual && q >= kBItems / 4) {
          kk[2 * q] = kk[2 * q + 1] = 0;
        } else if ((full || i + 1 < n) && al16) {
          asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;"
                       : "=l"(kk[2 * q]), "=l"(kk[2 * q + 1])
                       : "l"(keys + i), "l"(pol));
        } else {  // tail, or keys only 8 B-aligned (a slice at an odd offset)
          kk[2 * q] = i < n ? keys[i] : 0;
          kk[2 * q + 1] = i + 1 < n ? keys[i + 1] : 0;
        }
      }
      __syncthreads();
      const uint64_t s1 = 1ull << pl.ish, s2 = (uint64_t)(2 * kBThreads) << pl.ish;
      const uint64_t alt1 = 1ull << (pl.ish - 1);
      const uint64_t pmask = (1ull << g.payload_bits) - 1u;
      uint64_t ix = (t0 + 2 * threadIdx.x) << pl.ish;  // index field of item 0
#pragma unroll
      for (int q = 0; q < kBItems; ++q) {
        if (dual && q >= kBItems / 2) continue;  // filled with item q - kBItems/2's i2 record
        const uint64_t ixq = (q & 1) ? ix + s1 : ix;
        const uint64_t h = hashed ? kk[q] : xxh64(kk[q], g.seed);
        const bool in = full || t0 + (uint64_t)(q >> 1) * 2 * kBThreads + 2 * threadIdx.x + (q & 1) < n;
        const bool mine = in && !(hashed && foreign(g, h));  // (sharded padding: skipped)
        const uint64_t fp0 = (h >> 32) & pmask;
        const uint64_t fp = fp0 ? fp0 : 1u;
        const uint64_t i1 = POL == CKF_POLICY_XOR ? (h & g.mask) : reduce_index(h & 0xFFFFFFFFull, g);
        const uint32_t b1 = (uint32_t)i1 >> pl.lrbc;
        if constexpr (RT::kWide)
          rec[q] = RT::pack(t0 + (uint64_t)(q >> 1) * 2 * kBThreads + 2 * threadIdx.x + (q & 1), 0u,
                            (uint32_t)i1 & lmask, fp, pl);
        else
          rec[q] = ixq | ((uint64_t)((uint32_t)i1 & lmask) << pl.pb) | fp;
        pk[q] = mine ? (b1 << 16) | atomicAdd(&sm.cnt[b1], 1u) : 0xFFFFFFFFu;
        if (q < kBItems / 2 && dual) {
          uint64_t cc;
          const uint64_t i2 = alt_index<POL>(i1, fp, 0, g, cc);
          const uint32_t b2 = (uint32_t)i2 >> pl.lrbc;
          if constexpr (RT::kWide)
            rec[q + kBItems / 2] = RT::pack(t0 + (uint64_t)(q >> 1) * 2 * kBThreads + 2 * threadIdx.x + (q & 1), 1u,
                                            (uint32_t)i2 & lmask, fp, pl);
          else
            rec[q + kBItems / 2] = ixq | alt1 | ((uint64_t)((uint32_t)i2 & lmask) << pl.pb) | fp;
          pk[q + kBItems / 2] = mine ? (b2 << 16) | atomicAdd(&sm.cnt[b2], 1u) : 0xFFFFFFFFu;
        }
        if (q & 1) ix += s2;
      }
    } else {
      __syncthreads();  // hist zeroed
#pragma unroll
      for (int q0 = 0; q0 < kBItems; q0 += 4) {  // 4 entries (64 B) in flight per thread
        uint4 e[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint64_t i = t0 + (uint64_t)(q0 + q) * kBThreads + threadIdx.x;
          e[q] = i < n ? ms[i] : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint64_t i = t0 + (uint64_t)(q0 + q) * kBThreads + threadIdx.x;
          const uint64_t i2 = (uint64_t)e[q].z | ((uint64_t)e[q].w << 32);
          const uint32_t b2 = (uint32_t)(i2 >> pl.lrbc);
          rec[q0 + q] = RT::pack(e[q].x, 1u, i2 & lmask, e[q].y, pl);
          pk[q0 + q] = i < n ? (b2 << 16) | atomicAdd(&sm.cnt[b2], 1u) : 0xFFFFFFFFu;
        }
      }
    }
    __syncthreads();
    // runs leave as bulk copies (measured at 16-record runs: 1.46 vs 1.49 ms
    // for per-record coalesced stores, which also need a slot array)
    bin_reserve<F>(pl.R1, w.cnt1, sm);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kBItems; ++q)
      if (pk[q] != 0xFFFFFFFFu) bin_place(sm, pk[q] >> 16, pk[q] & 0xFFFFu, rec[q]);
    auto ovf = [&](const T& rc, uint32_t b) {
      const uint64_t bucket = ((uint64_t)b << pl.lrbc) + RT::off(rc, pl, lmask);
      resolve_direct<OP, F, WPB, POL>(words, g, pl, rc, bucket, sk, w.mode, n_ok, n_alt);
    };
    bin_write<F>(pl.R1, reinterpret_cast<T*>(w.bin1), pl.cap1, sm, ovf);
    __syncthreads();
  }
  bulk_wait_all();
  block_count_add(n_ok, n_alt, sk.ctr, occ, OP == OP_DELETE ? -1 : +1);
}

// ---------------------------------------------------------------------------
// split: coarse bin -> F2 fine bins (records re-based to the fine region)
// ---------------------------------------------------------------------------

#ifndef CKF_SPLIT_BLOCKS
#define CKF_SPLIT_BLOCKS 4  // (measured: 3 -> 4 CTAs per SM, split 0.87 -> 0.79 ms at 2^28 slots)
#endif
constexpr int kSplitBlocks = CKF_SPLIT_BLOCKS;  // resident split CTAs per SM
#ifndef CKF_SPLIT_PREFETCH
#define CKF_SPLIT_PREFETCH 1
#endif
constexpr bool kSplitPrefetch = CKF_SPLIT_PREFETCH;

template <int OP, int F, int WPB, int POL>
__global__ void __launch_bounds__(kBThreads, kSplitBlocks)
    region_split_kernel(Geo g, RPlan pl, uint64_t* words, RWork w, Sink sk, long long* occ) {
  using RT = RecT<F>;
  using T = typename RT::T;
  extern __shared__ __align__(16) uint8_t bsm_raw[];  // sizeof(BinSmem<F>), dynamic (> 48 KiB)
  BinSmem<F>& sm = *reinterpret_cast<BinSmem<F>*>(bsm_raw);
  const T* bin1 = reinterpret_cast<const T*>(w.bin1);
  const uint64_t pol = evict_first_policy();
  // tiles per coarse bin from the fullest bin of THIS pass (phase 2 bins hold
  // ~10 % of phase 1's records: no walk over the empty tail of every bin)
  __shared__ uint32_t s_max;
  if (threadIdx.x == 0) s_max = 0;
  __syncthreads();
  uint32_t mx = 0;
  for (uint32_t c = threadIdx.x; c < pl.R1; c += kBThreads) mx = max(mx, w.cnt1[(size_t)c * kCntStride]);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) atomicMax(&s_max, mx);
  __syncthreads();
  const uint64_t maxcnt = s_max < pl.cap1 ? s_max : pl.cap1;
  const uint32_t tiles_per_bin = (uint32_t)((maxcnt + kBTile - 1) / kBTile);
  const uint64_t tiles = (uint64_t)pl.R1 * tiles_per_bin;
  const uint32_t fmask = pl.F2 - 1u;
  uint32_t n_ok = 0, n_alt = 0;
  for (uint64_t s = blockIdx.x; s < tiles; s += gridDim.x) {
    const uint32_t c = (uint32_t)(s / tiles_per_bin);
    const uint64_t off0 = (s % tiles_per_bin) * (uint64_t)kBTile;
    const uint32_t cc = w.cnt1[(size_t)c * kCntStride];
    const uint64_t cnt = cc < pl.cap1 ? cc : pl.cap1;
    if (off0 >= cnt) continue;  // block-uniform
    if (kSplitPrefetch && threadIdx.x == 0) {  // this CTA's next tile into L2 (its records are a stream)
      const uint64_t sn = s + gridDim.x;
      if (sn < tiles) {
        const uint32_t cn = (uint32_t)(sn / tiles_per_bin);
        const uint64_t on = (sn % tiles_per_bin) * (uint64_t)kBTile;
        if (on < pl.cap1) {
          const uint64_t len = min((uint64_t)kBTile, pl.cap1 - on) & ~1ull;
          if (len) prefetch_l2(bin1 + cn * pl.cap1 + on, (uint32_t)(len * RT::kBytes));
        }
      }
    }
    bin_release();
    for (uint32_t r = threadIdx.x; r < pl.F2; r += kBThreads) sm.cnt[r] = 0;
    const T* src = bin1 + c * pl.cap1 + off0;
    const uint32_t nrec = (uint32_t)min((uint64_t)kBTile, cnt - off0);
    T rec[kBItems];
#pragma unroll
    for (int q = 0; q < kBItems / 2; ++q) {
      const uint32_t e = q * 2 * kBThreads + 2 * threadIdx.x;
      if constexpr (RT::kWide) {  // two 16 B records: one 32 B load
        if (e + 1 < nrec) {
          asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u64 {%0,%1,%2,%3}, [%4], %5;"
                       : "=l"(rec[2 * q].lo), "=l"(rec[2 * q].hi), "=l"(rec[2 * q + 1].lo), "=l"(rec[2 * q + 1].hi)
                       : "l"(src + e), "l"(pol));
        } else {
          rec[2 * q] = e < nrec ? src[e] : RT::filler();
          rec[2 * q + 1] = RT::filler();
        }
      } else if (e + 1 < nrec) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u64 {%0,%1}, [%2], %3;"
                     : "=l"(rec[2 * q]), "=l"(rec[2 * q + 1])
                     : "l"(src + e), "l"(pol));
      } else {
        rec[2 * q] = e < nrec ? src[e] : 0;
        rec[2 * q + 1] = 0;
      }
    }
    __syncthreads();
    uint32_t pk[kBItems];
#pragma unroll
    for (int q = 0; q < kBItems; ++q) {
      const uint32_t e = (q >> 1) * 2 * kBThreads + 2 * threadIdx.x + (q & 1);
      const uint32_t f = (RT::off(rec[q], pl, 0xFFFFFFFFu) >> pl.lrb) & fmask;
      pk[q] = e < nrec && !RT::is_filler(rec[q]) ? (f << 16) | atomicAdd(&sm.cnt[f], 1u) : 0xFFFFFFFFu;
    }
    __syncthreads();
    bin_reserve<F>(pl.F2, w.cntf + (size_t)c * pl.F2 * kCntStride, sm);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kBItems; ++q)
      if (pk[q] != 0xFFFFFFFFu) bin_place(sm, pk[q] >> 16, pk[q] & 0xFFFFu, RT::refine(rec[q], pl));
    T* binf = reinterpret_cast<T*>(w.binf);
    bin_write<F>(pl.F2, binf + (uint64_t)c * pl.F2 * pl.capf, pl.capf, sm, [&](const T& rc, uint32_t f) {
      const uint64_t bucket = ((uint64_t)(c * pl.F2 + f) << pl.lrb) + RT::off(rc, pl, (1u << pl.lrb) - 1u);
      resolve_direct<OP, F, WPB, POL>(words, g, pl, rc, bucket, sk, w.mode, n_ok, n_alt);
    });
    __syncthreads();
  }
  bulk_wait_all();
  block_count_add(n_ok, n_alt, sk.ctr, occ, OP == OP_DELETE ? -1 : +1);
}

// ---------------------------------------------------------------------------
// probe: one persistent CTA per SM, fine regions resident in shared memory
// ---------------------------------------------------------------------------

constexpr int kPWarps = 24;                     // consumer warps (measured: 16 and 30 slower)
constexpr int kPConsumers = kPWarps * 32;
constexpr int kPThreads = kPConsumers + 32;     // + one producer warp (<= 1024 threads)
// records per consumer lane per chunk: 4 (8 B records), 2 (16 B: the ring
// keeps its 72 KiB)
template <int F>
constexpr int kPPerLane = RecT<F>::kWide ? 2 : 4;
template <int F>
constexpr int kPChunk = kPConsumers * kPPerLane<F>;  // records per ring stage (3072 / 1536)
constexpr int kPStages = 3;
template <int F, int WPB>
constexpr int kPSub = (16 / WPB) < kPPerLane<F> ? (16 / WPB) : kPPerLane<F>;  // records in flight per lane
constexpr int kPRetry = 64;  // per-warp ring of deferred mutation records (power of two, >= 2 * 32)
template <int F>
constexpr uint32_t kProbeSmem =
    kRegionSmem + (kPStages * kPChunk<F> + kPWarps * kPRetry) * RecT<F>::kBytes + 128;

__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kPConsumers) : "memory"); }

// Queue unplaced inserts for the eviction pass: one reservation per warp for
// the whole sub-batch.  Only the key index is queued (hash field = kRehash);
// the eviction kernel re-reads and hashes the key, so this smem-bound kernel
// never waits on the scattered key reads.  Whole warp, converged.
constexpr uint64_t kRehash = ~0ull;

template <int F, int K>
__device__ __forceinline__ void enqueue_evict_batch(const Sink& sk, uint32_t nm, const typename RecT<F>::T (&rc)[K],
                                                    const RPlan& pl) {
  const int lane = threadIdx.x & 31;
  const uint32_t c = __popc(nm);
  uint32_t incl = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += y;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  if (!total) return;
  unsigned long long base = 0;
  if (lane == 31) base = atomicAdd(&sk.ctr->n_queued, (unsigned long long)total);
  base = __shfl_sync(0xffffffffu, base, 31);
  uint64_t pos = base + incl - c;
#pragma unroll
  for (int q = 0; q < K; ++q) {
    if (!((nm >> q) & 1u)) continue;
    const uint32_t idx = RecT<F>::idx(rc[q], pl);
    if (pos < sk.rec_cap) sk.rec[pos] = ckf_record{sk.ibase + idx, kRehash, 0u, 0u};
    else if (sk.ok) sk.ok[idx] = 0;
    ++pos;
  }
}

// PHASE 1: records of the primary bucket; misses are appended to this CTA's
// dense miss segment (re-binned by their alternate bucket for phase 2).
// PHASE 2: records of the alternate bucket; inserts still unplaced are queued
// for the eviction pass.
//
// Warp roles: warp kPWarps is the producer -- one lane streams this CTA's
// record chunks (its regions in turn, each region's chunks in turn) into a
// kPStages-deep ring with cp.async.bulk, gated by per-stage full/empty
// mbarriers.  Warps 0..kPWarps-1 consume: each owns a fixed slice of every
// chunk, so they never wait for each other except at region boundaries, where
// consumer thread 0 writes the table slice back and loads the next one.
// DF: the results' starting value (RWork::mode) as a compile-time constant --
// mutations always 1; query batches launch both variants and the one that does
// not match the sampled mode exits.
template <int OP, int F, int WPB, int POL, int PHASE, int DF = 1>
__global__ void __launch_bounds__(kPThreads, 1)
    region_probe_kernel(Geo g, RPlan pl, uint64_t* words, RWork w, Sink sk, long long* occ) {
  static_assert(OP == OP_QUERY || DF == 1, "mutations start from all-true results");
  if constexpr (OP == OP_QUERY)
    if ((*w.mode != 0) != (DF != 0)) return;
  using RT = RecT<F>;
  using T = typename RT::T;
  constexpr int kPL = kPPerLane<F>, kCh = kPChunk<F>;
  extern __shared__ __align__(128) uint8_t dsm[];
  uint64_t* tab = reinterpret_cast<uint64_t*>(dsm);
  T* ring = reinterpret_cast<T*>(dsm + kRegionSmem);
  T* retry = ring + kPStages * kCh;  // [kPWarps][kPRetry]
  uint64_t* full = reinterpret_cast<uint64_t*>(retry + kPWarps * kPRetry);
  uint64_t* empty = full + kPStages;
  uint64_t* tbar = empty + kPStages;
  __shared__ uint32_t s_miss[1];
  constexpr bool kMut = OP != OP_QUERY;
  const uint32_t* cnt = w.cntf;
  const T* bins = reinterpret_cast<const T*>(w.binf);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rb = 1u << pl.lrb;
  constexpr uint32_t bbytes = WPB * 8;
  constexpr bool dflt = DF != 0;  // results' starting value (see RWork::mode)
  if (tid == 0) {
    for (int s = 0; s < kPStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, kPWarps);
    }
    mbar_init(tbar, 1);
    fence_mbar_init();
    s_miss[0] = 0;
  }
  __syncthreads();

  auto region_count = [&](uint32_t r) -> uint32_t {
    const uint32_t c = cnt[(size_t)r * kCntStride];
    return c < pl.capf ? c : (uint32_t)pl.capf;
  };
  auto region_buckets = [&](uint32_t r) -> uint32_t {
    const uint64_t b0 = (uint64_t)r << pl.lrb;
    return (uint32_t)(g.m > b0 ? min((uint64_t)rb, g.m - b0) : 0);
  };
  uint32_t n_ok = 0, n_alt = 0;

  if (warp == kPWarps) {
    // ---- producer ----
    if (lane == 0) {
      uint32_t iseq = 0;
      for (uint32_t r = blockIdx.x; r < pl.R; r += gridDim.x) {
        const uint32_t cn = region_count(r);
        for (uint32_t k0 = 0; k0 < cn; k0 += kCh, ++iseq) {
          const uint32_t s = iseq % kPStages;
          if (iseq >= (uint32_t)kPStages) mbar_wait(empty + s, ((iseq / kPStages) - 1u) & 1u);
          const uint32_t len = min((uint32_t)kCh, cn - k0);
          // bins are even-sized and 16 B aligned (8 B records: a padded odd tail)
          const uint32_t bytes = (RT::kPadEven ? (len + 1u) & ~1u : len) * RT::kBytes;
          mbar_expect_tx(full + s, bytes);
          bulk_g2s(ring + (size_t)s * kCh, bins + (uint64_t)r * pl.capf + k0, bytes, full + s);
        }
      }
    }
  } else {
    // ---- consumers ----
    const uint32_t tab_a = saddr(tab);
    const uint64_t pol = evict_first_policy();
    // next region of this CTA with records (insert phase 1: every region, so
    // the room map covers the table)
    constexpr bool kVisitAll = OP == OP_INSERT && PHASE == 1;
    auto next_region = [&](uint32_t r) -> uint32_t {
      if (!kVisitAll)
        while (r < pl.R && region_count(r) == 0) r += gridDim.x;
      return r;
    };
    // Bulk copies move 16 B granules: a region of an odd number of 8-byte
    // buckets (WPB = 1, the last region of an odd-m offset table) moves its
    // last word with a plain load / store.
    auto load_table = [&](uint32_t r) {  // consumer thread 0
      const uint32_t nbytes = region_buckets(r) * bbytes, bulk = nbytes & ~15u;
      const uint64_t* src = words + ((uint64_t)r << pl.lrb) * WPB;
      if (bulk != nbytes) tab[bulk / 8] = src[bulk / 8];  // (before the arrive that releases the slice)
      mbar_expect_tx(tbar, bulk);
      if (bulk) bulk_g2s(tab, src, bulk, tbar);
      const uint32_t rn = next_region(r + gridDim.x);
      if (rn < pl.R) prefetch_l2(words + ((uint64_t)rn << pl.lrb) * WPB, region_buckets(rn) * bbytes);
    };
    // Per-step epilogue of unresolved records (K of them per lane): phase 1
    // misses go to this CTA's dense segment (warp reservation on a
    // shared-memory counter), re-binned by alternate bucket for phase 2;
    // phase-2 inserts still unplaced go to the eviction queue.  Whole warp.
    auto settle = [&](uint32_t nm, const auto& rcs, const auto& i2s) {  // rcs: T[KK]
      constexpr int KK = sizeof(rcs) / sizeof(rcs[0]);
      (void)KK;
      if constexpr (PHASE == 1) {
        const uint32_t c = __popc(nm);
        n_alt += c;
        uint32_t incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
          if (lane >= d) incl += y;
        }
        const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
        if (total) {
          uint32_t base = 0;
          if (lane == 31) base = atomicAdd(s_miss, total);
          base = __shfl_sync(0xffffffffu, base, 31);
          uint4* dst = w.miss + (uint64_t)blockIdx.x * w.seg + base + incl - c;
#pragma unroll
          for (int q = 0; q < KK; ++q)
            if ((nm >> q) & 1u)
              *dst++ = make_uint4(RT::idx(rcs[q], pl), (uint32_t)RT::fp(rcs[q], pl), (uint32_t)i2s[q],
                                  (uint32_t)(i2s[q] >> 32));
        }
      } else if constexpr (OP == OP_INSERT && PHASE == 2) {
        enqueue_evict_batch<F, KK>(sk, nm, rcs, pl);
      }
    };
    // Mutations whose single CAS attempt lost wait in this warp's retry ring
    // and are resolved 32 at a time with the full loop (a lost CAS no longer
    // re-runs the CAS body for the whole warp).  Warp-uniform head / count.
    T* wring = retry + warp * kPRetry;
    uint32_t rhead = 0, rcount = 0;
    auto drain = [&](uint32_t mcnt, uint64_t b0r) {  // whole warp, mcnt <= 32
      T rr[1];
      uint64_t i2r[1] = {0};
      uint32_t nm1 = 0;
      rr[0] = lane < mcnt ? wring[(rhead + lane) & (kPRetry - 1)] : RT::filler();
      __syncwarp();
      rhead += mcnt;
      rcount -= mcnt;
      if (lane < mcnt) {
        const uint32_t loc = RT::off(rr[0], pl, rb - 1u);
        const uint64_t fp = RT::fp(rr[0], pl);
        const uint32_t a = tab_a + loc * bbytes;
        const uint64_t tag = PHASE == 1 ? fp : (POL == CKF_POLICY_OFFSET ? make_tag(fp, 1u, g) : fp);
        uint64_t wv1[WPB];
        lds_bucket<WPB>(a, wv1);
        const bool done = OP == OP_INSERT ? smem_insert<F, WPB>(a, tag, wv1) : smem_remove<F, WPB>(a, tag, wv1);
        n_ok += done;
        if (OP == OP_DELETE && PHASE == 2 && !done) clear_bit(sk.bits, RT::idx(rr[0], pl));
        if (!done) {
          nm1 = 1u;
          if constexpr (PHASE == 1) {
            uint64_t cc;
            i2r[0] = alt_index<POL>(b0r + loc, fp, 0, g, cc);
          }
        }
      }
      settle(nm1, rr, i2r);
    };
    uint32_t r = next_region(blockIdx.x);
    if (tid == 0 && r < pl.R) load_table(r);
    uint32_t cseq = 0, tpar = 0;
    for (; r < pl.R;) {
      const uint32_t cn = region_count(r);
      const uint64_t b0 = (uint64_t)r << pl.lrb;
      mbar_wait(tbar, tpar);
      tpar ^= 1u;
      for (uint32_t k0 = 0; k0 < cn; k0 += kCh, ++cseq) {
        const uint32_t s = cseq % kPStages;
        mbar_wait(full + s, (cseq / kPStages) & 1u);
        const uint32_t len = min((uint32_t)kCh, cn - k0);
        const T* rs = ring + (size_t)s * kCh + warp * (kPL * 32) + lane;
        const uint32_t kbase = warp * (kPL * 32) + lane;
#pragma unroll 1
        for (int q0 = 0; q0 < kPL; q0 += kPSub<F, WPB>) {
          constexpr int K = kPSub<F, WPB>;
          T rc[K];
          uint64_t wv[K][WPB];
          uint32_t vm = 0;  // bit q: record q valid
#pragma unroll
          for (int q = 0; q < K; ++q) {
            rc[q] = kbase + (q0 + q) * 32 < len ? rs[(q0 + q) * 32] : RT::filler();
            const bool v = !RT::is_filler(rc[q]);  // past the chunk, or run padding
            vm |= (uint32_t)v << q;
            const uint32_t loc = RT::off(rc[q], pl, rb - 1u);
            // queries snapshot all buckets up front; mutations snapshot right
            // before their CAS (a stale snapshot costs a whole-warp retry)
            if (OP == OP_QUERY && v) lds_bucket_spread<WPB>(tab_a + loc * bbytes, wv[q]);
          }
          uint32_t nm = 0;     // bit q: record q not resolved here
          uint32_t defer = 0;  // bit q: record q's CAS lost (mutations)
          uint64_t i2[K];
#pragma unroll
          for (int q = 0; q < K; ++q) {
            if (!((vm >> q) & 1u)) continue;
            const uint32_t loc = RT::off(rc[q], pl, rb - 1u);
            const uint64_t fp = RT::fp(rc[q], pl);
            const uint32_t idx = RT::idx(rc[q], pl);
            if constexpr (OP == OP_QUERY) {
              const bool hit = match_any<F, WPB, POL>(wv[q], fp);
              if (hit && !dflt) set_bit(sk.bits, idx);
              if (PHASE == 2 && !hit && dflt) clear_bit(sk.bits, idx);  // a final negative
              if (PHASE == 1 && !hit && !dflt) {  // dual records: the i2 record is binned already
                n_alt += !RT::alt(rc[q], pl);
              } else if (PHASE == 1 && !hit) {
                nm |= 1u << q;
                uint64_t cc;
                i2[q] = alt_index<POL>(b0 + loc, fp, 0, g, cc);
              }
            } else {
              const uint32_t a = tab_a + loc * bbytes;
              const uint64_t tag = PHASE == 1 ? fp : (POL == CKF_POLICY_OFFSET ? make_tag(fp, 1u, g) : fp);
              lds_bucket<WPB>(a, wv[q]);  // (spread order measured slower here: instruction-bound)
              const int r1 = smem_try1<OP == OP_INSERT, F, WPB>(a, tag, wv[q]);
              if (r1 == 2) {  // lost CAS: resolved later in a compacted retry batch
                defer |= 1u << q;
                continue;
              }
              const bool done = r1 == 1;
              n_ok += done;
              if (OP == OP_DELETE && PHASE == 2 && !done) clear_bit(sk.bits, idx);  // tag in neither bucket
              if (!done) {
                nm |= 1u << q;
                if constexpr (PHASE == 1) {
                  uint64_t cc;
                  i2[q] = alt_index<POL>(b0 + loc, fp, 0, g, cc);
                }
              }
            }
          }
          settle(nm, rc, i2);
          if constexpr (kMut) {
#pragma unroll
            for (int q = 0; q < K; ++q) {
              const unsigned bal = __ballot_sync(0xffffffffu, (defer >> q) & 1u);
              if (bal) {
                if ((defer >> q) & 1u)
                  wring[(rhead + rcount + __popc(bal & ((1u << lane) - 1u))) & (kPRetry - 1)] = rc[q];
                rcount += __popc(bal);
                __syncwarp();
                if (rcount >= 32) drain(32, b0);
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);  // this warp is done with stage s
      }
      // region boundary: resolve this warp's deferred records, write the
      // slice back, bring in the next one
      if constexpr (kMut) {
        while (rcount) drain(rcount < 32 ? rcount : 32, b0);
      }
      if (kMut) fence_async_smem();  // this thread's shared-memory CASes before the bulk copy
      consumers_sync();
      if constexpr (OP == OP_INSERT) {
        // room bit per bucket for the eviction pass (RoomMap): read from the
        // final shared-memory copy, one ballot word per 32 buckets (phase 1
        // visits every region, so the map covers the whole table)
        const uint32_t nb = region_buckets(r);
        for (uint32_t k0 = warp * 32; k0 < nb; k0 += kPWarps * 32) {
          const uint32_t k = k0 + lane;
          bool room = false;
          if (k < nb) {
            uint64_t wv[WPB];
            lds_bucket<WPB>(tab_a + k * bbytes, wv);
#pragma unroll
            for (int j = 0; j < WPB; ++j) room |= Lanes<F>::zeros(wv[j]) != 0;
          }
          const unsigned bal = __ballot_sync(0xffffffffu, room);
          if (lane == 0) {
            const uint64_t b = b0 + k0;
            if (rb >= 32) {
              w.room[b >> 5] = bal;
            } else {  // several regions share a word (small forced tables)
              const uint32_t msk = (uint32_t)(((1ull << nb) - 1u) << (b & 31));
              atomicAnd(w.room + (b >> 5), ~msk);
              atomicOr(w.room + (b >> 5), bal << (b & 31));
            }
          }
        }
        consumers_sync();  // the slice is read before it is overwritten
      }
      const uint32_t rn = next_region(r + gridDim.x);
      if (tid == 0) {
        if (kMut && cn) {
          const uint32_t nbytes = region_buckets(r) * bbytes, bulk = nbytes & ~15u;
          if (bulk != nbytes) words[b0 * WPB + bulk / 8] = tab[bulk / 8];
          if (bulk) bulk_s2g(words + b0 * WPB, tab, bulk);
          bulk_wait_read();  // the slice has left shared memory
        }
        if (rn < pl.R) load_table(rn);
      }
      r = rn;
    }
    if (tid == 0) bulk_wait_all();
  }
  block_count_add(n_ok, n_alt, sk.ctr, occ, OP == OP_DELETE ? -1 : +1);  // (synchronizes the block)
  if (PHASE == 1 && tid == 0) w.n_miss[blockIdx.x] = s_miss[0];
}

// Query batches: estimate the fraction of positive keys from an evenly spaced
// sample of kSample keys (one direct lookup per thread on the global table)
// and pick the result bitmap's starting value, so that only the minority
// outcome costs an L2 atomic.  mode[1] accumulates the sample's hits.
constexpr uint32_t kSample = 8192;

template <int F, int WPB, int POL>
__global__ void __launch_bounds__(256) region_sample_kernel(Geo g, const uint64_t* __restrict__ words,
                                                            const uint64_t* __restrict__ keys, uint64_t n,
                                                            bool hashed, uint32_t* mode) {
  using Lg = Logic<OP_QUERY, F, WPB, POL>;
  const uint64_t ns = n < kSample ? n : kSample;
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  bool hit = false;
  if (k < ns) {
    const uint64_t i = (uint64_t)k * n / ns;
    uint64_t fp, i1, i2;
    const uint64_t h = hashed ? keys[i] : xxh64(keys[i], g.seed);
    place<POL>(h, g, fp, i1, i2);
    uint64_t* w = const_cast<uint64_t*>(words);
    hit = !(hashed && foreign(g, h)) && (Lg::first(w, i1, fp, g) || Lg::second(w, i2, fp, g));
  }
  const uint32_t c = __popc(__ballot_sync(0xffffffffu, hit));
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(mode + 1, c);
}

// Result bitmap starting value: all-true for a batch sampled as mostly
// positive (mode[0] = 1), all-false otherwise.
__global__ void __launch_bounds__(256) fill_bits_kernel(uint32_t* __restrict__ bits, uint64_t nw, uint64_t n,
                                                        uint32_t* mode) {
  const uint64_t ns = n < kSample ? n : kSample;
  const bool dflt = 2ull * mode[1] >= ns;
  const uint32_t v = dflt ? ~0u : 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) mode[0] = dflt;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nw; i += (uint64_t)gridDim.x * blockDim.x)
    bits[i] = v;
}

// bitmap -> one byte per key, and (queries) the hit count
__global__ void __launch_bounds__(256) expand_count_kernel(const uint32_t* __restrict__ bits, uint64_t n,
                                                           uint8_t* __restrict__ out, ckf_counters* ctr) {
  const uint64_t nw = (n + 31) / 32;
  uint32_t hits = 0;
  for (uint64_t wi = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; wi < nw; wi += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t b = bits[wi];
    const uint64_t i0 = wi * 32;
    if (i0 + 32 > n) b &= (1u << (n - i0)) - 1u;
    hits += __popc(b);
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
  if (ctr) block_count_add(hits, 0, ctr, nullptr, +1);
}

}  // namespace ckf
