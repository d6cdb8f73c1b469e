/*
 * ckf_oracle.c -- CPU restatement of the reference cuckoo-filter hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it, and only as the checker or the CPU baseline -- never as the
 * product path.  The product is paper_2603_15486_b200/csrc (CUDA, sm_100a).
 *
 * It restates, in plain C, the numba kernels of the reference package
 * `swarcuckoo` (/root/reference/pkg/src/swarcuckoo/_kernels.py, cited as K:
 * below) and the placement contract (placement.py, cited as P:).  Parity of
 * this restatement is PINNED against golden vectors produced by importing
 * the reference itself (tests/golden/make_golden.py -> tests/golden/golden_v1.npz)
 * and against the reference's own known-answer tests.
 *
 * Integer discipline follows the reference (K:17-20): every value is uint64_t
 * with wrapping arithmetic; slot/word indexes are int64_t.
 *
 * Concurrency: the parity functions are sequential, like the reference's
 * workers=1 batch insert/delete (K:510-549, filter.py:416-421); the read-only
 * query batch is split across POSIX threads exactly like filter.py:458-469
 * does with Python threads.  ck_insert_batch_mt / ck_delete_batch_mt restate
 * the reference's workers>1 mode (filter.py:422-438, 483-500: contiguous
 * chunks, one worker id per chunk for the eviction PRNG) with the word CASes
 * of K:158-272 as C11 atomics -- the CPU baseline of bench.py, never a parity
 * reference (concurrent outcomes are schedule-dependent).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef int64_t i64;

/* xxHash64 primes (K:29-33) and mixing constants (K:35-37). */
#define XXP1 0x9E3779B185EBCA87ull
#define XXP2 0xC2B2AE3D27D4EB4Full
#define XXP3 0x165667B19E3779F9ull
#define XXP4 0x85EBCA77C2B2AE63ull
#define XXP5 0x27D4EB2F165667C5ull
#define GOLDEN 0x9E3779B97F4A7C15ull
#define SMIX1 0xBF58476D1CE4E5B9ull
#define SMIX2 0x94D049BB133111EBull

/* The reference's `_kargs` tuple (filter.py:150-154) plus the runtime knobs
 * passed next to it (strategy, max_evictions, worker; K:510-514). */
typedef struct {
  u64 seed;
  u64 payload_bits;
  u64 f;
  u64 b;
  u64 m;
  u64 mask;        /* m-1 for power-of-two m, else 0 */
  i64 wpb;         /* words per bucket */
  i64 tpw;         /* tags per word */
  u64 high;        /* lane MSB mask (wordops.py HIGH_ONES) */
  u64 choice_bit;  /* 1<<(f-1) for offset, 0 for xor (filter.py:139) */
  int policy;      /* 0 xor, 1 offset (K:41-42) */
  int strategy;    /* 0 dfs, 1 bfs (K:43-44) */
  i64 max_evictions;
  u64 worker;
} ck_cfg;

/* ---------------- hashing and placement ---------------- */

static inline u64 rotl64(u64 x, unsigned r) { return (x << r) | (x >> (64u - r)); }

/* XXH64 of the key's 8 little-endian bytes (K:52-62 == P:149-161). */
u64 ck_xxh64(u64 key, u64 seed) {
  u64 h = seed + XXP5 + 8u;
  h ^= rotl64(key * XXP2, 31) * XXP1;
  h = rotl64(h, 27) * XXP1 + XXP4;
  h = (h ^ (h >> 33)) * XXP2;
  h = (h ^ (h >> 29)) * XXP3;
  return h ^ (h >> 32);
}

/* SplitMix64 finaliser (K:65-69) and the per-key stream seed (K:72-74). */
u64 ck_smix(u64 z) {
  z = (z ^ (z >> 30)) * SMIX1;
  z = (z ^ (z >> 27)) * SMIX2;
  return z ^ (z >> 31);
}
u64 ck_rng_init(u64 seed, u64 h, u64 worker) { return ck_smix((seed ^ h) + GOLDEN * (worker + 1u)); }

/* tag_hash (K:77-79 == P:164-172). */
u64 ck_tag_hash(u64 fp) { return (fp * GOLDEN) >> 32; }

/* bucket reduction of the low hash half (K:82-86 == P:175-180). */
static inline u64 reduce_idx(u64 x, const ck_cfg* c) { return c->mask ? (x & c->mask) : (x * c->m) >> 32; }

/* alternate bucket + flipped residency (K:89-97 == P:188-202). */
static inline u64 alt_bucket(u64 i, u64 fp, u64 choice, const ck_cfg* c, u64* new_choice) {
  if (c->policy == 0) {
    *new_choice = 0;
    return (i ^ ck_tag_hash(fp)) & c->mask;
  }
  u64 delta = 1u + ck_tag_hash(fp) % (c->m - 1u);
  if (choice == 0) {
    *new_choice = 1;
    return (i + delta) % c->m;
  }
  *new_choice = 0;
  return (i + c->m - delta) % c->m;
}

/* stored lane value and its inverse (K:100-111). */
static inline u64 make_tag(u64 fp, u64 choice, const ck_cfg* c) { return fp | choice * c->choice_bit; }
static inline u64 tag_payload(u64 tag, const ck_cfg* c) { return tag & (c->choice_bit - 1u); }
static inline u64 tag_choice(u64 tag, const ck_cfg* c) { return (tag & c->choice_bit) ? 1u : 0u; }

/* (fp, i1, i2) from a hash (K:277-285 == P:219-232). */
static inline void place_hash(u64 h, const ck_cfg* c, u64* fp, u64* i1, u64* i2) {
  u64 p = (h >> 32) & ((1ull << c->payload_bits) - 1u);
  *fp = p ? p : 1u;
  *i1 = reduce_idx(h & 0xFFFFFFFFull, c);
  u64 dummy;
  *i2 = alt_bucket(*i1, *fp, 0, c, &dummy);
}

/* ---------------- SWAR lane helpers (K:116-153 == wordops.py:51-97) ---------------- */

static inline u64 lane_bcast(u64 tag, u64 f) {
  for (u64 w = f; w < 64; w <<= 1) tag |= tag << w;
  return tag;
}
/* exact per-lane zero indicator, carry-out form (K:126-129, wordops.py:9-16) */
static inline u64 lane_zeros(u64 w, u64 high) { return ~(((w & ~high) + ~high) | w) & high; }
static inline i64 lowest_lane(u64 m, u64 f) { return m ? (i64)(__builtin_ctzll(m) / f) : -1; }
static inline u64 lane_get(u64 w, i64 s, u64 f) {
  u64 lm = (f == 64) ? ~0ull : ((1ull << f) - 1u);
  return (w >> ((u64)s * f)) & lm;
}
static inline u64 lane_set(u64 w, i64 s, u64 tag, u64 f) {
  u64 lm = ((1ull << f) - 1u) << ((u64)s * f);
  return (w & ~lm) | (tag << ((u64)s * f));
}

/* ---------------- bucket operations (K:158-272) ---------------- */

/* TryInsert: first empty lane scanning words from (tag % b)/tpw, wrapping (K:158-180). */
static i64 bucket_put(u64* words, i64 base, u64 tag, const ck_cfg* c) {
  i64 start = (i64)(tag % c->b) / c->tpw;
  for (i64 k = 0; k < c->wpb; ++k) {
    i64 wk = (start + k) % c->wpb;
    u64 w = words[base + wk];
    u64 z = lane_zeros(w, c->high);
    if (z) {
      i64 s = lowest_lane(z, c->f);
      words[base + wk] = lane_set(w, s, tag, c->f);
      return wk * c->tpw + s;
    }
  }
  return -1;
}

/* Find: any lane equal to tag after dropping `ignore` bits (K:183-199). */
static int bucket_has(const u64* words, i64 base, u64 tag, u64 ignore, const ck_cfg* c) {
  u64 pat = lane_bcast(tag, c->f);
  for (i64 k = 0; k < c->wpb; ++k)
    if (lane_zeros((words[base + k] & ~ignore) ^ pat, c->high)) return 1;
  return 0;
}

/* TryRemove: clear the first matching lane in scan order (K:202-221). */
static i64 bucket_take(u64* words, i64 base, u64 tag, const ck_cfg* c) {
  u64 pat = lane_bcast(tag, c->f);
  i64 start = (i64)(tag % c->b) / c->tpw;
  for (i64 k = 0; k < c->wpb; ++k) {
    i64 wk = (start + k) % c->wpb;
    u64 w = words[base + wk];
    u64 mm = lane_zeros(w ^ pat, c->high);
    if (mm) {
      i64 s = lowest_lane(mm, c->f);
      words[base + wk] = lane_set(w, s, 0, c->f);
      return wk * c->tpw + s;
    }
  }
  return -1;
}

static int bucket_any_empty(const u64* words, i64 base, const ck_cfg* c) {
  for (i64 k = 0; k < c->wpb; ++k)
    if (lane_zeros(words[base + k], c->high)) return 1;
  return 0;
}

/* ---------------- whole operations ---------------- */

/* insert_one (K:331-436): direct placement, then DFS or BFS eviction.
 * Returns ok; *rounds and *lost as the reference reports them.  `h` is the
 * key's xxh64 (K:355). */
static int insert_hash(u64* words, u64 h, const ck_cfg* c, i64* rounds, u64* lost,
                       i64* cand_slot, u64* cand_tag) {
  u64 fp, i1, i2;
  place_hash(h, c, &fp, &i1, &i2);
  u64 tag1 = fp;
  u64 tag2 = make_tag(fp, c->policy == 1 ? 1u : 0u, c);
  *rounds = 0;
  *lost = 0;
  if (bucket_put(words, (i64)i1 * c->wpb, tag1, c) >= 0) return 1;
  if (bucket_put(words, (i64)i2 * c->wpb, tag2, c) >= 0) return 1;

  u64 st = ck_rng_init(c->seed, h, c->worker) + GOLDEN;
  u64 cur_b, cur_tag;
  if ((ck_smix(st) & 1u) == 0) {
    cur_b = i1;
    cur_tag = tag1;
  } else {
    cur_b = i2;
    cur_tag = tag2;
  }

  if (c->strategy == 0) { /* DFS (K:374-389) */
    for (i64 n = 1; n <= c->max_evictions; ++n) {
      st += GOLDEN;
      i64 victim = (i64)(ck_smix(st) % c->b);
      i64 wi = (i64)cur_b * c->wpb + victim / c->tpw;
      u64 old = lane_get(words[wi], victim % c->tpw, c->f);
      words[wi] = lane_set(words[wi], victim % c->tpw, cur_tag, c->f);
      if (old == 0) {
        *rounds = n;
        return 1;
      }
      u64 nc;
      cur_b = alt_bucket(cur_b, tag_payload(old, c), tag_choice(old, c), c, &nc);
      cur_tag = make_tag(tag_payload(old, c), nc, c);
      if (bucket_put(words, (i64)cur_b * c->wpb, cur_tag, c) >= 0) {
        *rounds = n;
        return 1;
      }
    }
    *rounds = c->max_evictions;
    *lost = tag_payload(cur_tag, c);
    return 0;
  }

  /* BFS (K:391-436) */
  i64 limit = (i64)c->b / 2;
  for (i64 n = 1; n <= c->max_evictions; ++n) {
    st += GOLDEN;
    i64 start = (i64)(ck_smix(st) % c->b);
    i64 base = (i64)cur_b * c->wpb;
    /* collect_candidates (K:257-272): occupied lanes from `start`, wrapping */
    i64 cnt = 0;
    for (i64 j = 0; j < (i64)c->b && cnt < limit; ++j) {
      i64 s = (start + j) % (i64)c->b;
      u64 t = lane_get(words[base + s / c->tpw], s % c->tpw, c->f);
      if (t) {
        cand_slot[cnt] = s;
        cand_tag[cnt] = t;
        ++cnt;
      }
    }
    if (cnt == 0) {
      if (bucket_put(words, base, cur_tag, c) >= 0) {
        *rounds = n;
        return 1;
      }
      continue;
    }
    i64 chosen = -1;
    u64 alt_b = 0, alt_tag = 0;
    for (i64 j = 0; j < cnt; ++j) {
      u64 tc;
      u64 tb = alt_bucket(cur_b, tag_payload(cand_tag[j], c), tag_choice(cand_tag[j], c), c, &tc);
      if (bucket_any_empty(words, (i64)tb * c->wpb, c)) {
        chosen = j;
        alt_b = tb;
        alt_tag = make_tag(tag_payload(cand_tag[j], c), tc, c);
        break;
      }
    }
    if (chosen >= 0) {
      /* two-step relocation; single-threaded, so the origin CAS cannot lose */
      i64 aslot = bucket_put(words, (i64)alt_b * c->wpb, alt_tag, c);
      if (aslot < 0) continue;
      i64 os = cand_slot[chosen];
      i64 owi = base + os / c->tpw;
      if (lane_get(words[owi], os % c->tpw, c->f) == cand_tag[chosen]) {
        words[owi] = lane_set(words[owi], os % c->tpw, cur_tag, c->f);
        *rounds = n;
        return 1;
      }
      i64 awi = (i64)alt_b * c->wpb + aslot / c->tpw;
      if (lane_get(words[awi], aslot % c->tpw, c->f) == alt_tag)
        words[awi] = lane_set(words[awi], aslot % c->tpw, 0, c->f);
      continue;
    }
    /* deepen through the last candidate (K:427-434) */
    i64 os = cand_slot[cnt - 1];
    u64 ct = cand_tag[cnt - 1];
    i64 owi = base + os / c->tpw;
    if (lane_get(words[owi], os % c->tpw, c->f) != ct) continue;
    words[owi] = lane_set(words[owi], os % c->tpw, cur_tag, c->f);
    u64 nc;
    cur_b = alt_bucket(cur_b, tag_payload(ct, c), tag_choice(ct, c), c, &nc);
    cur_tag = make_tag(tag_payload(ct, c), nc, c);
  }
  *rounds = c->max_evictions;
  *lost = tag_payload(cur_tag, c);
  return 0;
}

/* query_one (K:439-458): offset matches payload bits only (K:451-453). */
static int query_hash(const u64* words, u64 h, const ck_cfg* c) {
  u64 ignore = c->policy == 1 ? c->high : 0u;
  u64 fp, i1, i2;
  place_hash(h, c, &fp, &i1, &i2);
  return bucket_has(words, (i64)i1 * c->wpb, fp, ignore, c) ||
         bucket_has(words, (i64)i2 * c->wpb, fp, ignore, c);
}

/* delete_one (K:461-484): full-lane match, i1 with fp then i2 with fp|choice. */
static int delete_hash(u64* words, u64 h, const ck_cfg* c) {
  u64 fp, i1, i2;
  place_hash(h, c, &fp, &i1, &i2);
  u64 tag2 = c->policy == 1 ? make_tag(fp, 1u, c) : fp;
  if (bucket_take(words, (i64)i1 * c->wpb, fp, c) >= 0) return 1;
  return bucket_take(words, (i64)i2 * c->wpb, tag2, c) >= 0;
}

/* ---------------- exported batch entry points (K:489-549) ---------------- */

void ck_hash_batch(const u64* keys, i64 n, u64 seed, u64* out) {
  for (i64 i = 0; i < n; ++i) out[i] = ck_xxh64(keys[i], seed);
}

void ck_place_batch(const ck_cfg* c, const u64* keys, i64 n, u64* fp, u64* i1, u64* i2) {
  for (i64 i = 0; i < n; ++i) place_hash(ck_xxh64(keys[i], c->seed), c, fp + i, i1 + i, i2 + i);
}

void ck_place_hashes(const ck_cfg* c, const u64* hashes, i64 n, u64* fp, u64* i1, u64* i2) {
  for (i64 i = 0; i < n; ++i) place_hash(hashes[i], c, fp + i, i1 + i, i2 + i);
}

u64 ck_alt(const ck_cfg* c, u64 i, u64 fp, u64 choice, u64* new_choice) {
  return alt_bucket(i, fp, choice, c, new_choice);
}

static inline u64 key_hash(u64 k, const ck_cfg* c, int hashed) { return hashed ? k : ck_xxh64(k, c->seed); }

/* `hashed` != 0: keys[] already holds xxh64(key, seed) (the multi-GPU router
 * ships hashes so the owning shard skips the rehash). */
i64 ck_insert_batch(const ck_cfg* c, u64* words, const u64* keys, i64 n, uint8_t* ok,
                    i64* evictions, u64* lost, int hashed) {
  i64 lim = (i64)c->b / 2;
  if (lim < 1) lim = 1;
  i64* cs = (i64*)malloc(sizeof(i64) * lim);
  u64* ct = (u64*)malloc(sizeof(u64) * lim);
  i64 n_ok = 0;
  for (i64 i = 0; i < n; ++i) {
    i64 r;
    u64 l;
    int good = insert_hash(words, key_hash(keys[i], c, hashed), c, &r, &l, cs, ct);
    if (ok) ok[i] = (uint8_t)good;
    if (evictions) evictions[i] = r;
    if (lost) lost[i] = l;
    n_ok += good;
  }
  free(cs);
  free(ct);
  return n_ok;
}

i64 ck_delete_batch(const ck_cfg* c, u64* words, const u64* keys, i64 n, uint8_t* out, int hashed) {
  i64 n_ok = 0;
  for (i64 i = 0; i < n; ++i) {
    int good = delete_hash(words, key_hash(keys[i], c, hashed), c);
    if (out) out[i] = (uint8_t)good;
    n_ok += good;
  }
  return n_ok;
}

typedef struct {
  const ck_cfg* c;
  const u64* words;
  const u64* keys;
  uint8_t* out;
  i64 lo, hi;
  int hashed;
} qjob;

static void* query_worker(void* arg) {
  qjob* j = (qjob*)arg;
  for (i64 i = j->lo; i < j->hi; ++i)
    j->out[i] = (uint8_t)query_hash(j->words, key_hash(j->keys[i], j->c, j->hashed), j->c);
  return NULL;
}

/* query_batch; threads > 1 splits contiguous chunks like filter.py:390-392. */
void ck_query_batch(const ck_cfg* c, const u64* words, const u64* keys, i64 n, uint8_t* out,
                    int threads, int hashed) {
  if (threads <= 1 || n == 0) {
    for (i64 i = 0; i < n; ++i) out[i] = (uint8_t)query_hash(words, key_hash(keys[i], c, hashed), c);
    return;
  }
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  qjob* jobs = (qjob*)malloc(sizeof(qjob) * threads);
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (qjob){c, words, keys, out, (t * n) / threads, ((t + 1) * n) / threads, hashed};
    pthread_create(&tid[t], NULL, query_worker, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  free(tid);
  free(jobs);
}

/* ---------------- concurrent workers (filter.py:422-438, 483-500) ----------------
 * The same operations with every word access atomic: a lane is claimed,
 * cleared or replaced by a compare-and-swap of its whole word (K:158-254). */

static inline u64 aload(const u64* p) { return __atomic_load_n(p, __ATOMIC_RELAXED); }
static inline int acas(u64* p, u64* expect, u64 desired) {
  return __atomic_compare_exchange_n(p, expect, desired, 0, __ATOMIC_RELAXED, __ATOMIC_RELAXED);
}

static i64 bucket_put_at(u64* words, i64 base, u64 tag, const ck_cfg* c) {
  i64 start = (i64)(tag % c->b) / c->tpw;
  for (i64 k = 0; k < c->wpb; ++k) {
    i64 wk = (start + k) % c->wpb;
    u64 w = aload(words + base + wk);
    for (;;) {
      u64 z = lane_zeros(w, c->high);
      if (!z) break;
      i64 s = lowest_lane(z, c->f);
      if (acas(words + base + wk, &w, lane_set(w, s, tag, c->f))) return wk * c->tpw + s;
    }
  }
  return -1;
}

static i64 bucket_take_at(u64* words, i64 base, u64 tag, const ck_cfg* c) {
  u64 pat = lane_bcast(tag, c->f);
  i64 start = (i64)(tag % c->b) / c->tpw;
  for (i64 k = 0; k < c->wpb; ++k) {
    i64 wk = (start + k) % c->wpb;
    u64 w = aload(words + base + wk);
    for (;;) {
      u64 mm = lane_zeros(w ^ pat, c->high);
      if (!mm) break;
      i64 s = lowest_lane(mm, c->f);
      if (acas(words + base + wk, &w, lane_set(w, s, 0, c->f))) return wk * c->tpw + s;
    }
  }
  return -1;
}

/* lane_cas (K:247-254): replace lane s of word p only while it holds `expect` */
static int lane_cas_at(u64* p, i64 s, u64 expect, u64 repl, u64 f) {
  u64 w = aload(p);
  for (;;) {
    if (lane_get(w, s, f) != expect) return 0;
    if (acas(p, &w, lane_set(w, s, repl, f))) return 1;
  }
}

static int insert_hash_at(u64* words, u64 h, const ck_cfg* c, i64* rounds, u64* lost, i64* cand_slot,
                          u64* cand_tag) {
  u64 fp, i1, i2;
  place_hash(h, c, &fp, &i1, &i2);
  u64 tag1 = fp;
  u64 tag2 = make_tag(fp, c->policy == 1 ? 1u : 0u, c);
  *rounds = 0;
  *lost = 0;
  if (bucket_put_at(words, (i64)i1 * c->wpb, tag1, c) >= 0) return 1;
  if (bucket_put_at(words, (i64)i2 * c->wpb, tag2, c) >= 0) return 1;
  u64 st = ck_rng_init(c->seed, h, c->worker) + GOLDEN;
  u64 cur_b = i1, cur_tag = tag1;
  if (ck_smix(st) & 1u) {
    cur_b = i2;
    cur_tag = tag2;
  }
  if (c->strategy == 0) { /* DFS: atomic lane exchange (swap_slot, K:232-244) */
    for (i64 n = 1; n <= c->max_evictions; ++n) {
      st += GOLDEN;
      i64 victim = (i64)(ck_smix(st) % c->b);
      u64* p = words + (i64)cur_b * c->wpb + victim / c->tpw;
      u64 w = aload(p), old;
      do {
        old = lane_get(w, victim % c->tpw, c->f);
      } while (!acas(p, &w, lane_set(w, victim % c->tpw, cur_tag, c->f)));
      if (old == 0) {
        *rounds = n;
        return 1;
      }
      u64 nc;
      cur_b = alt_bucket(cur_b, tag_payload(old, c), tag_choice(old, c), c, &nc);
      cur_tag = make_tag(tag_payload(old, c), nc, c);
      if (bucket_put_at(words, (i64)cur_b * c->wpb, cur_tag, c) >= 0) {
        *rounds = n;
        return 1;
      }
    }
    *rounds = c->max_evictions;
    *lost = tag_payload(cur_tag, c);
    return 0;
  }
  i64 limit = (i64)c->b / 2;
  if (limit < 1) limit = 1;
  for (i64 n = 1; n <= c->max_evictions; ++n) { /* BFS (K:391-436) */
    st += GOLDEN;
    i64 start = (i64)(ck_smix(st) % c->b);
    i64 base = (i64)cur_b * c->wpb;
    i64 cnt = 0;
    for (i64 j = 0; j < (i64)c->b && cnt < limit; ++j) {
      i64 s = (start + j) % (i64)c->b;
      u64 t = lane_get(aload(words + base + s / c->tpw), s % c->tpw, c->f);
      if (t) {
        cand_slot[cnt] = s;
        cand_tag[cnt] = t;
        ++cnt;
      }
    }
    if (cnt == 0) {
      if (bucket_put_at(words, base, cur_tag, c) >= 0) {
        *rounds = n;
        return 1;
      }
      continue;
    }
    i64 chosen = -1;
    u64 alt_b = 0, alt_tag = 0;
    for (i64 j = 0; j < cnt; ++j) {
      u64 tc;
      u64 tb = alt_bucket(cur_b, tag_payload(cand_tag[j], c), tag_choice(cand_tag[j], c), c, &tc);
      int room = 0;
      for (i64 k = 0; k < c->wpb && !room; ++k) room = lane_zeros(aload(words + (i64)tb * c->wpb + k), c->high) != 0;
      if (room) {
        chosen = j;
        alt_b = tb;
        alt_tag = make_tag(tag_payload(cand_tag[j], c), tc, c);
        break;
      }
    }
    if (chosen >= 0) {
      i64 aslot = bucket_put_at(words, (i64)alt_b * c->wpb, alt_tag, c);
      if (aslot < 0) continue;
      i64 os = cand_slot[chosen];
      if (lane_cas_at(words + base + os / c->tpw, os % c->tpw, cand_tag[chosen], cur_tag, c->f)) {
        *rounds = n;
        return 1;
      }
      lane_cas_at(words + (i64)alt_b * c->wpb + aslot / c->tpw, aslot % c->tpw, alt_tag, 0, c->f);
      continue;
    }
    i64 os = cand_slot[cnt - 1];
    u64 ct = cand_tag[cnt - 1];
    if (!lane_cas_at(words + base + os / c->tpw, os % c->tpw, ct, cur_tag, c->f)) continue;
    u64 nc;
    cur_b = alt_bucket(cur_b, tag_payload(ct, c), tag_choice(ct, c), c, &nc);
    cur_tag = make_tag(tag_payload(ct, c), nc, c);
  }
  *rounds = c->max_evictions;
  *lost = tag_payload(cur_tag, c);
  return 0;
}

typedef struct {
  ck_cfg c; /* private copy: worker id = chunk index (filter.py:428) */
  u64* words;
  const u64* keys;
  uint8_t* out;
  i64 lo, hi;
  int hashed, del;
  i64 n_ok;
} mjob;

static void* mutate_worker(void* arg) {
  mjob* j = (mjob*)arg;
  i64 lim = (i64)j->c.b / 2 > 0 ? (i64)j->c.b / 2 : 1;
  i64* cs = (i64*)malloc(sizeof(i64) * lim);
  u64* ct = (u64*)malloc(sizeof(u64) * lim);
  for (i64 i = j->lo; i < j->hi; ++i) {
    u64 h = key_hash(j->keys[i], &j->c, j->hashed);
    int good;
    if (j->del) {
      u64 fp, i1, i2;
      place_hash(h, &j->c, &fp, &i1, &i2);
      u64 tag2 = j->c.policy == 1 ? make_tag(fp, 1u, &j->c) : fp;
      good = bucket_take_at(j->words, (i64)i1 * j->c.wpb, fp, &j->c) >= 0 ||
             bucket_take_at(j->words, (i64)i2 * j->c.wpb, tag2, &j->c) >= 0;
    } else {
      i64 r;
      u64 l;
      good = insert_hash_at(j->words, h, &j->c, &r, &l, cs, ct);
    }
    if (j->out) j->out[i] = (uint8_t)good;
    j->n_ok += good;
  }
  free(cs);
  free(ct);
  return NULL;
}

static i64 mutate_mt(const ck_cfg* c, u64* words, const u64* keys, i64 n, uint8_t* out, int hashed, int del,
                     int threads) {
  if (threads < 1) threads = 1;
  pthread_t* tid = (pthread_t*)malloc(sizeof(pthread_t) * threads);
  mjob* jobs = (mjob*)malloc(sizeof(mjob) * threads);
  for (int t = 0; t < threads; ++t) {
    jobs[t] = (mjob){*c, words, keys, out, (t * n) / threads, ((t + 1) * n) / threads, hashed, del, 0};
    jobs[t].c.worker = (u64)t;
    pthread_create(&tid[t], NULL, mutate_worker, &jobs[t]);
  }
  i64 n_ok = 0;
  for (int t = 0; t < threads; ++t) {
    pthread_join(tid[t], NULL);
    n_ok += jobs[t].n_ok;
  }
  free(tid);
  free(jobs);
  return n_ok;
}

i64 ck_insert_batch_mt(const ck_cfg* c, u64* words, const u64* keys, i64 n, uint8_t* ok, int hashed, int threads) {
  return mutate_mt(c, words, keys, n, ok, hashed, 0, threads);
}

i64 ck_delete_batch_mt(const ck_cfg* c, u64* words, const u64* keys, i64 n, uint8_t* out, int hashed,
                       int threads) {
  return mutate_mt(c, words, keys, n, out, hashed, 1, threads);
}

/* Scalar helpers the tests pin individually (K:158-272). */
i64 ck_try_insert(const ck_cfg* c, u64* words, i64 base, u64 tag) { return bucket_put(words, base, tag, c); }
i64 ck_remove_tag(const ck_cfg* c, u64* words, i64 base, u64 tag) { return bucket_take(words, base, tag, c); }
int ck_find_tag(const ck_cfg* c, const u64* words, i64 base, u64 tag, u64 ignore) {
  return bucket_has(words, base, tag, ignore, c);
}
u64 ck_zero_mask(u64 w, u64 high) { return lane_zeros(w, high); }
u64 ck_broadcast(u64 tag, u64 f) { return lane_bcast(tag, f); }
int ck_abi_version(void) { return 1; }
