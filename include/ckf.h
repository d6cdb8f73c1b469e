/*
 * ckf.h -- C ABI of the B200-native cuckoo-filter hot path (libckf.so).
 *
 * This is the drop-in boundary.  The reference (swarcuckoo 0.1.0) crosses
 * from Python into compiled code at the numba batch kernels; each entry point
 * below replaces one of them (file:line in /root/reference/pkg/src/swarcuckoo):
 *
 *   ckf_params_init   <- FilterConfig.__post_init__ + CuckooFilter._kargs
 *                        (placement.py:77-136, filter.py:133-154)
 *   ckf_hash          <- _kernels.hash_batch    (_kernels.py:489-493)
 *   ckf_place         <- _kernels.place_batch   (_kernels.py:496-507)
 *   ckf_insert        <- _kernels.insert_batch  (_kernels.py:510-529)
 *   ckf_query         <- _kernels.query_batch   (_kernels.py:532-537)
 *   ckf_delete        <- _kernels.delete_batch  (_kernels.py:540-549)
 *   ckf_host_place    <- placement.derive_placement (placement.py:219-232),
 *                        host-compiled from the same header the kernels use
 *
 * Conventions:
 *  - every pointer argument except `p` and the host_* helpers is DEVICE memory
 *    owned by the caller (torch tensors in the Python facade); nothing here
 *    allocates;
 *  - every call is asynchronous on `stream` (a cudaStream_t passed as void*;
 *    NULL = legacy default stream);
 *  - return 0 on success, CKF_EINVAL for bad arguments, or
 *    CKF_ECUDA_BASE - cudaError_t for a CUDA launch error; ckf_strerror()
 *    names the code.  Kernels never fail per key: "full" and "not found"
 *    are data, exactly as in the reference (_kernels.py:388-389).
 */
#ifndef CKF_H_
#define CKF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CKF_ABI_VERSION 2

#define CKF_OK 0
#define CKF_EINVAL (-22)
#define CKF_ECUDA_BASE (-1000)

#define CKF_POLICY_XOR 0
#define CKF_POLICY_OFFSET 1
#define CKF_EVICT_DFS 0
#define CKF_EVICT_BFS 1

/* op flags */
#define CKF_MODE_CONCURRENT 0u   /* lock-free, one thread per key (default) */
#define CKF_MODE_SEQUENTIAL 1u   /* one device thread, reference key order:
                                    bit-identical to insert_batch(workers=1) */
#define CKF_INPUT_HASHED 2u      /* `keys` already holds xxh64(key, seed) */
#define CKF_FORCE_DIRECT 4u      /* never use the region (batch) schedule */
#define CKF_FORCE_TILED 8u       /* use the region schedule whenever its plan applies */

/* Schedules (ckf_schedule) */
#define CKF_SCHED_DIRECT 0       /* one thread per key, random bucket accesses */
#define CKF_SCHED_REGION 1       /* bin -> split -> shared-memory probe per table region */
#define CKF_SCHED_SEQUENTIAL 2   /* parity mode: one device thread, reference order */

/* op ids for ckf_workspace_bytes */
#define CKF_OP_QUERY 0
#define CKF_OP_INSERT 1
#define CKF_OP_DELETE 2

/* Filter geometry: the reference `_kargs` tuple (filter.py:150-154) plus the
 * eviction knobs; filled and validated by ckf_params_init. Passed by pointer,
 * read on the host, copied into the kernel launch by value. */
typedef struct ckf_params {
  uint64_t seed;
  uint64_t bucket_count;      /* m */
  uint64_t index_mask;        /* m-1 for power-of-two m, else 0 */
  uint64_t high;              /* per-lane MSB mask */
  uint64_t choice_bit;        /* 1<<(f-1) for offset, 0 for xor */
  uint64_t delta_magic;       /* fastmod constant for tag_hash % (m-1) (offset) */
  uint64_t worker;            /* eviction PRNG stream id (filter.py:285) */
  uint32_t fingerprint_bits;  /* f in {8,16,32} */
  uint32_t bucket_slots;      /* b */
  uint32_t words_per_bucket;  /* b*f/64 */
  uint32_t tags_per_word;     /* 64/f */
  uint32_t payload_bits;      /* f (xor) or f-1 (offset) */
  uint32_t policy;            /* CKF_POLICY_* */
  uint32_t eviction;          /* CKF_EVICT_* */
  uint32_t max_evictions;     /* >= 1 */
  uint32_t shard_shift;       /* sharded filter (ckf_params_set_shard): owner = (h >> shift) & mask */
  uint32_t shard_mask;        /*   0: not sharded */
  uint32_t shard_id;          /*   this shard; with CKF_INPUT_HASHED, hashes owned by another */
  uint32_t shard_reserved;    /*   shard are skipped (padding of the fixed-size exchange) */
} ckf_params;

/* Sparse per-key insert outcome for keys that needed the eviction path
 * (evictions >= 1 or failure).  Keys placed directly have evictions == 0 and
 * lost == 0 and produce no record; this is how the facade rebuilds the
 * reference BatchInsertResult (filter.py:95-112) without 16 B/key of dense
 * output traffic. */
typedef struct ckf_record {
  uint64_t index;      /* position of the key in the batch */
  uint64_t lost;       /* payload fingerprint dropped on failure, else 0 */
  uint32_t evictions;  /* eviction rounds (max_evictions on failure) */
  uint32_t ok;         /* 1 stored, 0 failed */
} ckf_record;

/* Device-side counters of one call; zeroed by the call itself. */
typedef struct ckf_counters {
  unsigned long long n_ok;         /* successful inserts / deletes */
  unsigned long long n_records;    /* records produced (may exceed capacity) */
  unsigned long long n_queued;     /* keys that entered the eviction pass */
  unsigned long long n_alt;        /* keys that had to probe their alternate bucket
                                      (insert: i1 full; query/delete: no match in i1) */
} ckf_counters;

int ckf_abi_version(void);
const char* ckf_strerror(int code);
/* Process-wide count of kernels this library has launched (evidence for the
 * benchmark's gpu_launches field). */
uint64_t ckf_kernel_launches(void);

/* Validates like FilterConfig (placement.py:77-102) and derives geometry. */
int ckf_params_init(ckf_params* p, uint64_t bucket_count, uint32_t fingerprint_bits,
                    uint32_t bucket_slots, int policy, int eviction, uint32_t max_evictions,
                    uint64_t seed);

/* Mark p as shard `id` of `shards` (a power of two <= 256) routed by hash bits
 * [shift, shift + log2 shards): hashed batches then skip every hash owned by
 * another shard -- the sentinel padding of ckf_route_partition_padded -- with
 * no effect on the table, the occupancy or the counters (a skipped key's
 * result is unspecified).  shards == 1 clears it. */
int ckf_params_set_shard(ckf_params* p, uint32_t shift, uint32_t shards, uint32_t id);

/* out[i] = xxh64(keys[i], seed) */
int ckf_hash(const uint64_t* keys, uint64_t n, uint64_t seed, uint64_t* out, void* stream);

/* (fp, i1, i2) per key; flags may carry CKF_INPUT_HASHED. */
int ckf_place(const ckf_params* p, const uint64_t* keys, uint64_t n, uint64_t* fp, uint64_t* i1,
              uint64_t* i2, unsigned flags, void* stream);

/* Scratch bytes a batch of n keys wants: the region schedule's (keys binned
 * by table region, every bucket access in shared memory), or,
 * for a direct-path BFS insert into an L2-resident table, a room map (one bit
 * per bucket) + the eviction cursor.  0: direct kernels, no workspace.
 * Passing a smaller (or NULL) workspace selects the direct path without the
 * room map; ckf_schedule reports which schedule runs. */
uint64_t ckf_workspace_bytes(const ckf_params* p, uint64_t n, int op, unsigned flags);

/* The schedule (CKF_SCHED_*) an op call with these arguments runs, and in how
 * many back-to-back region runs (*runs; a run holds at most 2^(64-ish)-2 keys,
 * DESIGN.md §2).  Negative: invalid parameters. */
int ckf_schedule(const ckf_params* p, uint64_t n, int op, unsigned flags, const void* keys,
                 const void* workspace, uint64_t workspace_bytes, uint64_t* runs);

/* Batch insert.  ok[n] is required.  evictions/lost are optional DENSE
 * outputs with the reference's types (int64 / uint64 per key).  records
 * (capacity record_cap) receives the sparse outcomes and doubles as the
 * eviction work queue; if it overflows, the excess keys are evicted in place
 * and only counted.  occupancy (nullable) is atomically increased by n_ok. */
int ckf_insert(const ckf_params* p, uint64_t* words, const uint64_t* keys, uint64_t n,
               uint8_t* ok, int64_t* evictions, uint64_t* lost, ckf_record* records,
               uint64_t record_cap, ckf_counters* counters, long long* occupancy,
               void* workspace, uint64_t workspace_bytes, unsigned flags, void* stream);

/* Batch membership; out[i] in {0,1}.  Read-only phase (filter.py:9-15).
 * counters (nullable) receives n_ok = hits and n_alt. */
int ckf_query(const ckf_params* p, const uint64_t* words, const uint64_t* keys, uint64_t n,
              uint8_t* out, ckf_counters* counters, void* workspace, uint64_t workspace_bytes,
              unsigned flags, void* stream);

/* Batch delete; out[i] = 1 where a lane was cleared.  occupancy (nullable)
 * is atomically decreased by n_ok. */
int ckf_delete(const ckf_params* p, uint64_t* words, const uint64_t* keys, uint64_t n,
               uint8_t* out, ckf_counters* counters, long long* occupancy, void* workspace,
               uint64_t workspace_bytes, unsigned flags, void* stream);

/* Mixed batch (BASELINE configs[4]): key i runs ops[i] (CKF_OP_QUERY /
 * CKF_OP_INSERT / CKF_OP_DELETE), all concurrently in one launch (+ the
 * eviction pass for inserts whose pair is full).  Outside the reference's
 * phase contract (filter.py:9-15): lookups use coherent loads, and a lookup is
 * exact for keys whose membership the batch does not change.  out[i]: hit /
 * stored / deleted.  records (record_cap) is the eviction queue as in
 * ckf_insert; counters: n_ok = inserts stored, n_alt, n_queued; occupancy
 * (nullable) += inserts - deletes. */
int ckf_mixed(const ckf_params* p, uint64_t* words, const uint8_t* ops, const uint64_t* keys, uint64_t n,
              uint8_t* out, ckf_record* records, uint64_t record_cap, ckf_counters* counters,
              long long* occupancy, unsigned flags, void* stream);

/* Multi-GPU routing (sharded.py steps 2-3): stable partition of key hashes
 * by owning shard (h >> shift) & (shards - 1), shards a power of two <= 8.
 * send[] receives the hashes grouped by shard in arrival order, order[p] the
 * source index of send[p], shard_counts[s] (device int64) the group sizes.
 * workspace: ckf_route_workspace_bytes(n, shards) device bytes. */
uint64_t ckf_route_workspace_bytes(uint64_t n, uint32_t shards);
int ckf_route_partition(const uint64_t* hashes, uint64_t n, uint32_t shift, uint32_t shards, uint64_t* send,
                        long long* order, long long* shard_counts, void* workspace, uint64_t workspace_bytes,
                        void* stream);

/* Fixed-capacity routing for a host-sync-free exchange: like
 * ckf_route_partition, but shard s's hashes go to send[s*cap ..) in arrival
 * order, the rest of its block holds a hash owned by shard (s+1) % shards
 * (skipped by the receiver, see ckf_params_set_shard) with order[] = -1, and
 * hashes past `cap` in a shard are not sent: *spilled (device) counts them and
 * their callers find them unanswered.  send / order: shards * cap entries.
 * workspace: ckf_route_workspace_bytes(n, shards). */
int ckf_route_partition_padded(const uint64_t* hashes, uint64_t n, uint32_t shift, uint32_t shards, uint64_t cap,
                               uint64_t* send, long long* order, long long* shard_counts,
                               unsigned long long* spilled, void* workspace, uint64_t workspace_bytes, void* stream);

/* out[order[p] * elem] <- back[p * elem] for every p < n with order[p] >= 0
 * (the return path of the routing: answers back to the caller's order);
 * elem in {1, 8} bytes. */
int ckf_route_unpermute(const void* back, const long long* order, uint64_t n, uint32_t elem, void* out,
                        void* stream);

/* k-mer ingestion (replaces swarcuckoo/kmer.py:48-95 stream_kmers' packing
 * loop).  seq: device bytes of the FASTA records' sequence lines, each record's
 * lines concatenated, one separator byte (any byte outside ACGTacgt) between
 * records.  Every length-k window (1 <= k <= 31) of A/C/G/T bases (either
 * case) that crosses no other byte is packed two bits per base, leftmost base
 * most significant, and written to out[] in sequence order; out needs room for
 * len - k + 1 keys.  *n_out (device) receives the count.  workspace: at least
 * ckf_kmer_workspace_bytes(len) device bytes. */
uint64_t ckf_kmer_workspace_bytes(uint64_t len);
int ckf_kmers(const uint8_t* seq, uint64_t len, uint32_t k, uint64_t* out,
              unsigned long long* n_out, void* workspace, uint64_t workspace_bytes, void* stream);

/* Debug hook for the BFS rollback test (the reference sabotages lane_cas,
 * pkg/tests/test_filter.py:224-259): the next `count` BFS relocations see a
 * concurrent writer replace their origin lane with a stale tag right before
 * the origin CAS, so they roll their copy back and retry.  Pending count out. */
int ckf_debug_fault_origin_cas(unsigned int count);
int ckf_debug_faults_pending(unsigned int* count);

/* Host-compiled copies of the shared device semantics (same source as the
 * kernels); used by derive_placement() and by the CPU parity tests. */
uint64_t ckf_host_hash(uint64_t key, uint64_t seed);
void ckf_host_place(const ckf_params* p, uint64_t key, uint64_t* fp, uint64_t* i1, uint64_t* i2);
uint64_t ckf_host_alt(const ckf_params* p, uint64_t bucket, uint64_t fp, uint64_t choice,
                      uint64_t* new_choice);
uint64_t ckf_host_zero_mask(uint32_t fingerprint_bits, uint64_t word);

#ifdef __cplusplus
}
#endif
#endif /* CKF_H_ */
