// ckf_ops.cuh -- what the batch schedules share: the op ids, the per-key
// result sink, and the two halves of every op on the GLOBAL table (fetch the
// bucket / act on the snapshot), used wherever a key is resolved outside the
// shared-memory region pipeline (bin overflows, the query sample).
#pragma once

#include "ckf_device.cuh"

namespace ckf {

enum { OP_QUERY = 0, OP_INSERT = 1, OP_DELETE = 2 };

constexpr int kCntStride = 32;  // bin counters 128 B apart (one line each)

// What happens to a resolved / unresolved key.
struct Sink {
  uint32_t* bits;         // query/delete: result bit per key
  ckf_record* rec;        // insert: eviction queue
  uint64_t rec_cap;
  ckf_counters* ctr;
  uint8_t* ok;            // insert: dense ok (queue overflow only)
  const uint64_t* keys;   // insert: to recover a queued key's hash
  bool hashed;
  uint64_t ibase;         // batch index of keys[0] (a chunk of a larger call)
};

__device__ __forceinline__ void set_bit(uint32_t* bits, uint32_t i) { atomicOr(bits + (i >> 5), 1u << (i & 31)); }

// Global-table TryInsert / Find / TryRemove (K:158-221) split into "fetch the
// bucket" and "act on the fetched snapshot".
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

// Unresolved insert: hand (batch index, hash) to the eviction pass.  idx is
// chunk-relative; the queue holds batch indices.
__device__ __forceinline__ void enqueue_evict_one(const Sink& sk, uint32_t idx, uint64_t h) {
  const uint64_t pos = atomicAdd(&sk.ctr->n_queued, 1ull);
  if (pos < sk.rec_cap) sk.rec[pos] = ckf_record{sk.ibase + idx, h, 0u, 0u};
  else if (sk.ok) sk.ok[idx] = 0;
}

}  // namespace ckf
