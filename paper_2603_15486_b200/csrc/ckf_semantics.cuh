// ckf_semantics.cuh -- the bit-level contract of the filter, compiled for both
// host and device.  Every function here has a reference twin that it must match
// bit for bit (file:line in /root/reference/pkg/src/swarcuckoo, K = _kernels.py,
// P = placement.py, W = wordops.py).  The kernels (ckf_kernels.cu) use these on
// the GPU; the ckf_host_* exports run the very same code on the CPU so parity of
// this header is testable on a GPU-less machine.
#pragma once

#include <stdint.h>

#include "../../include/ckf.h"

#if defined(__CUDACC__)
#define CKF_HD __host__ __device__ __forceinline__
#else
#define CKF_HD inline
#endif

namespace ckf {

constexpr uint64_t kP1 = 0x9E3779B185EBCA87ull;  // xxh64 primes, K:29-33
constexpr uint64_t kP2 = 0xC2B2AE3D27D4EB4Full;
constexpr uint64_t kP3 = 0x165667B19E3779F9ull;
constexpr uint64_t kP4 = 0x85EBCA77C2B2AE63ull;
constexpr uint64_t kP5 = 0x27D4EB2F165667C5ull;
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;  // K:35
constexpr uint64_t kMix1 = 0xBF58476D1CE4E5B9ull;    // K:36
constexpr uint64_t kMix2 = 0x94D049BB133111EBull;    // K:37

CKF_HD uint64_t rotl(uint64_t x, unsigned r) { return (x << r) | (x >> (64u - r)); }

// XXH64 over the 8 little-endian bytes of `key` (K:52-62).
CKF_HD uint64_t xxh64(uint64_t key, uint64_t seed) {
  uint64_t acc = seed + kP5 + 8u;
  acc ^= rotl(key * kP2, 31) * kP1;
  acc = rotl(acc, 27) * kP1 + kP4;
  acc ^= acc >> 33;
  acc *= kP2;
  acc ^= acc >> 29;
  acc *= kP3;
  return acc ^ (acc >> 32);
}

// SplitMix64 finaliser and per-key eviction stream (K:65-74).
CKF_HD uint64_t smix(uint64_t z) {
  z = (z ^ (z >> 30)) * kMix1;
  z = (z ^ (z >> 27)) * kMix2;
  return z ^ (z >> 31);
}
CKF_HD uint64_t rng_init(uint64_t seed, uint64_t h, uint64_t worker) {
  return smix((seed ^ h) + kGolden * (worker + 1u));
}

// tag_hash: high half of fp * GOLDEN (K:77-79).
CKF_HD uint64_t tag_hash(uint64_t fp) { return (fp * kGolden) >> 32; }

// Lemire fastmod for a 32-bit dividend: exact a % d for every a, d < 2^32.
CKF_HD uint64_t fastmod_magic(uint64_t d) { return d <= 1 ? 0 : ~0ull / d + 1u; }
CKF_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// Placement geometry carried into every kernel by value.
struct Geo {
  uint64_t seed, m, mask, high, choice_bit, magic, worker;
  uint32_t f, b, wpb, tpw, payload_bits, policy, eviction, max_evictions;
  uint32_t shard_shift, shard_mask, shard_id;
};

// A hashed key owned by another shard (the padding of the fixed-size
// multi-GPU exchange): skipped by every kernel.
CKF_HD bool foreign(const Geo& g, uint64_t h) {
  return g.shard_mask && (uint32_t)((h >> g.shard_shift) & g.shard_mask) != g.shard_id;
}

CKF_HD Geo geo_from(const ckf_params& p) {
  Geo g;
  g.seed = p.seed;
  g.m = p.bucket_count;
  g.mask = p.index_mask;
  g.high = p.high;
  g.choice_bit = p.choice_bit;
  g.magic = p.delta_magic;
  g.worker = p.worker;
  g.f = p.fingerprint_bits;
  g.b = p.bucket_slots;
  g.wpb = p.words_per_bucket;
  g.tpw = p.tags_per_word;
  g.payload_bits = p.payload_bits;
  g.policy = p.policy;
  g.eviction = p.eviction;
  g.max_evictions = p.max_evictions;
  g.shard_shift = p.shard_shift;
  g.shard_mask = p.shard_mask;
  g.shard_id = p.shard_id;
  return g;
}

// tag_hash(fp) % (m-1), exact: tag_hash < 2^32, so a divisor >= 2^32 is the
// identity and a smaller one goes through the precomputed fastmod constant.
CKF_HD uint64_t offset_delta(uint64_t fp, const Geo& g) {
  uint64_t th = tag_hash(fp);
  uint64_t d = g.m - 1u;
  uint64_t r;
  if (d > 0xFFFFFFFFull) r = th;
  else if (d == 1u) r = 0;
  else r = mulhi64(g.magic * th, d);
  return 1u + r;
}

// Primary-bucket reduction of the low hash half (K:82-86): mask when m is a
// power of two, multiply-shift (mod 2^64) otherwise.
CKF_HD uint64_t reduce_index(uint64_t x, const Geo& g) {
  return g.mask ? (x & g.mask) : (x * g.m) >> 32;
}

// Alternate bucket + flipped residency bit (K:89-97).
template <int POL>
CKF_HD uint64_t alt_index(uint64_t i, uint64_t fp, uint64_t choice, const Geo& g,
                          uint64_t& new_choice) {
  if (POL == CKF_POLICY_XOR) {
    new_choice = 0;
    return (i ^ tag_hash(fp)) & g.mask;
  }
  uint64_t delta = offset_delta(fp, g);
  if (choice == 0) {
    new_choice = 1;
    uint64_t j = i + delta;
    return j >= g.m ? j - g.m : j;
  }
  new_choice = 0;
  uint64_t j = i + (g.m - delta);
  return j >= g.m ? j - g.m : j;
}

// (fp, i1, i2) from the key hash (K:277-285).
template <int POL>
CKF_HD void place(uint64_t h, const Geo& g, uint64_t& fp, uint64_t& i1, uint64_t& i2) {
  uint64_t p = (h >> 32) & ((1ull << g.payload_bits) - 1u);
  fp = p ? p : 1u;
  i1 = reduce_index(h & 0xFFFFFFFFull, g);
  uint64_t c;
  i2 = alt_index<POL>(i1, fp, 0, g, c);
}

// Stored lane <-> (payload, choice) (K:100-111); for xor choice_bit == 0, so
// the payload mask wraps to all ones.
CKF_HD uint64_t make_tag(uint64_t fp, uint64_t choice, const Geo& g) { return fp | choice * g.choice_bit; }
CKF_HD uint64_t tag_fp(uint64_t tag, const Geo& g) { return tag & (g.choice_bit - 1u); }
CKF_HD uint64_t tag_choice(uint64_t tag, const Geo& g) { return (tag & g.choice_bit) ? 1u : 0u; }

// ---- SWAR over one 64-bit word of F-bit lanes (K:116-153, W:51-97) ----

template <int F>
struct Lanes {
  static constexpr int kTpw = 64 / F;
  static constexpr uint64_t kLaneMask = (F == 64) ? ~0ull : ((1ull << F) - 1u);
  static constexpr uint64_t kHigh = F == 8 ? 0x8080808080808080ull
                                    : F == 16 ? 0x8000800080008000ull
                                              : 0x8000000080000000ull;
  static constexpr uint64_t kLow = kHigh >> (F - 1);
  // broadcast: one multiply by the per-lane LSB pattern
  CKF_HD static uint64_t bcast(uint64_t tag) { return tag * kLow; }
  // exact per-lane zero indicator, carry-out form (W:9-16, K:126-129)
  CKF_HD static uint64_t zeros(uint64_t w) { return ~(((w & ~kHigh) + ~kHigh) | w) & kHigh; }
  CKF_HD static int first(uint64_t ind) {
#if defined(__CUDA_ARCH__)
    return (__ffsll((long long)ind) - 1) / F;
#else
    return __builtin_ctzll(ind) / F;
#endif
  }
  CKF_HD static uint64_t get(uint64_t w, int s) { return (w >> (s * F)) & kLaneMask; }
  CKF_HD static uint64_t put(uint64_t w, int s, uint64_t tag) {
    return (w & ~(kLaneMask << (s * F))) | (tag << (s * F));
  }
};

CKF_HD uint64_t zero_mask_rt(uint32_t f, uint64_t w) {
  switch (f) {
    case 8: return Lanes<8>::zeros(w);
    case 16: return Lanes<16>::zeros(w);
    default: return Lanes<32>::zeros(w);
  }
}

}  // namespace ckf
