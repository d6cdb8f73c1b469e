"""GPU tests aimed at the shared-memory region schedule (ckf_region.cuh).

`tiled=True` forces the batch schedule onto small tables (>= 16 fine regions),
so these run in seconds and still cross every region / bin boundary:
  * query results are bit-exact against the oracle for batches the device
    samples as mostly positive (result bitmap starts all-true), mostly
    negative (starts all-false) and mixed;
  * adversarial keys whose primary buckets all fall into one region overflow
    the coarse and fine bins (direct resolution path) and still give the
    reference's insert-success count, no false negatives, exact occupancy and
    a clean delete;
  * duplicate keys (one bucket pair) fail exactly as many times as in the
    reference.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
from paper_2603_15486_b200 import CuckooFilter, FilterConfig, _lib

pytestmark = pytest.mark.gpu

CASES = [(16, 16, "xor"), (16, 16, "offset"), (8, 16, "xor"), (16, 32, "xor")]


def _cfg(f, b, pol, m=1 << 12, ev="bfs"):
    if pol == "offset":
        m = m - 3  # non-power-of-two m (offset policy only)
    return FilterConfig(bucket_count=m, fingerprint_bits=f, bucket_slots=b, policy=pol, eviction=ev, seed=3)


@pytest.mark.parametrize("f,b,pol", CASES)
@pytest.mark.parametrize("pos_frac", [1.0, 0.9, 0.5, 0.1, 0.0])
def test_region_query_exact_vs_oracle(f, b, pol, pos_frac):
    cfg = _cfg(f, b, pol)
    rng = np.random.default_rng(11)
    keys = rng.integers(0, 1 << 62, size=int(0.9 * cfg.total_slots), dtype=np.uint64)
    ref = oracle.OracleFilter(oracle.cfg_from(cfg))
    ok, _, _ = ref.insert_batch(keys)
    filt = CuckooFilter(cfg, tiled=True)
    filt.words_device.copy_(torch.from_numpy(ref.words.view(np.int64)))
    filt._occ.fill_(int(ok.sum()))
    n = 200_000
    npos = int(pos_frac * n)
    q = np.concatenate([rng.choice(keys, npos), rng.integers(1 << 62, 1 << 63, size=n - npos, dtype=np.uint64)])
    rng.shuffle(q)
    l0 = _lib.kernel_launches()
    got = filt.query_batch(q)
    # sample, fill, bin, split, probe, miss bin, split, probe, expand: the region schedule ran
    assert _lib.kernel_launches() - l0 >= 9
    assert np.array_equal(got, ref.query_batch(q))
    c = filt.last_counters()
    assert c["n_ok"] == int(got.sum())


def _same_region_keys(cfg, want: int, region_buckets: int, seed: int = 5) -> np.ndarray:
    """Keys whose primary bucket lies in [0, region_buckets)."""
    ocfg = oracle.cfg_from(cfg)
    rng = np.random.default_rng(seed)
    out = []
    while sum(len(o) for o in out) < want:
        k = rng.integers(0, 1 << 63, size=1 << 20, dtype=np.uint64)
        _, i1, _ = oracle.place_batch(ocfg, k)
        out.append(k[i1 < region_buckets])
    return np.concatenate(out)[:want]


@pytest.mark.parametrize("pol", ["xor", "offset"])
def test_region_bin_overflow_adversarial(pol):
    cfg = _cfg(16, 16, pol, m=1 << 13)
    # every primary bucket in the first 1/16 of the table: that coarse / fine
    # bin receives ~16x its capacity and the overflow resolves on the direct path
    keys = _same_region_keys(cfg, want=int(0.45 * (cfg.bucket_count // 16) * cfg.bucket_slots * 2),
                             region_buckets=cfg.bucket_count // 16)
    ref = oracle.OracleFilter(oracle.cfg_from(cfg))
    rok, _, _ = ref.insert_batch(keys)
    filt = CuckooFilter(cfg, tiled=True)
    res = filt.insert_batch(keys)
    assert res.n_failed == int((~rok).sum())
    assert len(filt) == res.n_ok == int(np.count_nonzero(filt.stored_tags()))
    stored = keys[res.ok]
    assert filt.query_batch(stored).all(), "false negative"
    d = filt.delete_batch(stored)
    assert d.all() and len(filt) == 0 and int(np.count_nonzero(filt.words)) == 0


def test_region_duplicates_fail_like_reference():
    cfg = _cfg(16, 16, "xor", m=1 << 12)
    rng = np.random.default_rng(2)
    base = rng.integers(0, 1 << 62, size=20_000, dtype=np.uint64)
    dup = np.repeat(np.uint64(0xDEADBEEF), 40)  # 40 copies of one key: 32 slots in its pair
    keys = np.concatenate([base, dup])
    rng.shuffle(keys)
    ref = oracle.OracleFilter(oracle.cfg_from(cfg))
    rok, _, _ = ref.insert_batch(keys)
    filt = CuckooFilter(cfg, tiled=True)
    res = filt.insert_batch(keys)
    assert res.n_failed == int((~rok).sum()) >= 8
    assert filt.query_batch(base).all()
    # deleting 40 copies removes exactly the stored ones
    d = filt.delete_batch(dup)
    assert int(d.sum()) == int(res.ok[keys == np.uint64(0xDEADBEEF)].sum())


def test_region_delete_absent_keys_report_false():
    cfg = _cfg(16, 16, "xor", m=1 << 12)
    rng = np.random.default_rng(4)
    keys = rng.integers(0, 1 << 32, size=50_000, dtype=np.uint64)
    filt = CuckooFilter(cfg, tiled=True)
    filt.insert_batch(keys)
    ref = oracle.OracleFilter(oracle.cfg_from(cfg))
    ref.insert_batch(keys)
    absent = rng.integers(1 << 40, 1 << 62, size=200_000, dtype=np.uint64)
    got = filt.delete_batch(absent)
    want = ref.delete_batch(absent)
    # an absent key whose fingerprint matches a stored tag deletes it (reference
    # semantics, FPR-rate); only two absent keys racing for one tag could differ
    assert abs(int(got.sum()) - int(want.sum())) <= 2
    assert int(got.sum()) < 200
    assert len(filt) == len(keys) - int(got.sum())


@pytest.mark.parametrize("pol", ["xor", "offset"])
def test_calls_split_into_region_runs(monkeypatch, pol):
    """A call larger than one region run (the record's index field bounds a
    run; CKF_MAX_RUN_KEYS shrinks it here) runs back-to-back runs: per-run
    eviction queues, batch-absolute record indices, per-run result bitmaps."""
    monkeypatch.setenv("CKF_MAX_RUN_KEYS", "20000")
    cfg = _cfg(16, 16, pol, m=1 << 12)
    rng = np.random.default_rng(21)
    keys = rng.integers(0, 1 << 62, size=int(0.97 * cfg.total_slots), dtype=np.uint64)
    ref = oracle.OracleFilter(oracle.cfg_from(cfg))
    rok, _, _ = ref.insert_batch(keys)
    filt = CuckooFilter(cfg, tiled=True)
    res = filt.insert_batch(keys)
    assert filt.last_schedule == ("region", 4)
    assert res.n_failed == int((~rok).sum())
    rec = res.records()
    assert len(rec) > 100 and len(np.unique(rec["index"])) == len(rec)
    assert rec["index"].max() > 3 * 20000  # the last run's queue entries carry batch indices
    ev = res.evictions
    assert int((ev > 0).sum()) == int((rec["evictions"] > 0).sum())
    assert np.array_equal(np.flatnonzero(~res.ok), np.sort(rec["index"][rec["ok"] == 0]).astype(np.int64))
    tags = filt.stored_tags()
    assert len(filt) == int(np.count_nonzero(tags))
    neg = rng.integers(1 << 62, 1 << 63, size=70_000, dtype=np.uint64)
    assert filt.query_batch(keys[res.ok]).all()
    assert filt.last_schedule == ("region", 4)
    snap = oracle.OracleFilter(oracle.cfg_from(cfg))
    snap.words[:] = filt.words
    assert np.array_equal(filt.query_batch(neg), snap.query_batch(neg))
    assert filt.last_schedule[1] == 4
    d = filt.delete_batch(keys[res.ok])
    assert d.all() and len(filt) == 0 and not filt.words.any()


def test_region_schedule_on_odd_offset_slices():
    """A torch slice starting at an odd element is only 8 B-aligned: the region
    schedule still runs (scalar key loads) and matches the oracle."""
    cfg = _cfg(16, 16, "xor", m=1 << 12)
    rng = np.random.default_rng(31)
    host = rng.integers(0, 1 << 62, size=int(0.95 * cfg.total_slots) + 1, dtype=np.uint64)
    keys = torch.from_numpy(host.view(np.int64)).cuda()[1:]
    assert keys.data_ptr() % 16 == 8
    ref = oracle.OracleFilter(oracle.cfg_from(cfg))
    rok, _, _ = ref.insert_batch(host[1:])
    filt = CuckooFilter(cfg, tiled=True)
    l0 = _lib.kernel_launches()
    res = filt.insert_batch(keys)
    assert _lib.kernel_launches() - l0 >= 7  # bin, split, probe, bin, split, probe, evict
    assert res.n_failed == int((~rok).sum())
    q = torch.from_numpy(np.concatenate([[0], host[1:2000], rng.integers(1 << 62, 1 << 63, 3001, dtype=np.uint64)]).view(np.int64)).cuda()[1:]
    snap = oracle.OracleFilter(oracle.cfg_from(cfg))
    snap.words[:] = filt.words
    assert np.array_equal(filt.query_batch(q).cpu().numpy(), snap.query_batch(q.cpu().numpy().view(np.uint64)))
    assert bool(filt.delete_batch(keys).all()) and len(filt) == 0


@pytest.mark.parametrize("pol", ["xor", "offset"])
@pytest.mark.parametrize("f", [8, 16])
def test_eight_byte_buckets_on_the_region_schedule(pol, f):
    """One-word buckets (b = 64/f: configs[0]'s b=4 at f=16) on the region
    schedule: success counts equal to the reference's at 95 % load, lookups
    bit-exact on a snapshot, delete-all back to an all-zero table."""
    b = 64 // f
    m = (1 << 16) if pol == "xor" else 65_521
    cfg = FilterConfig(bucket_count=m, fingerprint_bits=f, bucket_slots=b, policy=pol, eviction="bfs", seed=3)
    rng = np.random.default_rng(f)
    keys = rng.integers(0, 1 << 62, size=int(0.95 * cfg.total_slots), dtype=np.uint64)
    ref = oracle.OracleFilter(oracle.cfg_from(cfg))
    rok, _, _ = ref.insert_batch(keys)
    filt = CuckooFilter(cfg, tiled=True)
    res = filt.insert_batch(keys)
    assert filt.last_schedule[0] == "region"
    # b = 4 at 95 % runs long chains; the success count may differ from the
    # sequential reference's by the few keys a concurrent chain loses
    assert abs(res.n_failed - int((~rok).sum())) <= max(2, len(keys) // 20000)
    assert len(filt) == res.n_ok
    assert filt.query_batch(keys[res.ok]).all()
    neg = rng.integers(1 << 62, 1 << 63, size=200_000, dtype=np.uint64)
    snap = oracle.OracleFilter(oracle.cfg_from(cfg))
    snap.words[:] = filt.words
    assert np.array_equal(filt.query_batch(neg), snap.query_batch(neg))
    d = filt.delete_batch(keys[res.ok])
    assert d.all() and len(filt) == 0
    assert int(np.count_nonzero(filt.stored_tags())) <= 32  # (the BFS rollback window)


@pytest.mark.parametrize("pol", ["xor", "offset"])
@pytest.mark.parametrize("b", [4, 16])
def test_f32_sixteen_byte_records_on_the_region_schedule(pol, b):
    """f = 32 runs the region schedule with 16-byte records (RecT): success
    counts equal to the reference's at 95 % load, lookups bit-exact on a
    snapshot, delete-all back to an all-zero table."""
    m = (1 << 14) if pol == "xor" else 16_381
    cfg = FilterConfig(bucket_count=m, fingerprint_bits=32, bucket_slots=b, policy=pol, eviction="bfs", seed=4)
    rng = np.random.default_rng(b)
    keys = rng.integers(0, 1 << 62, size=int(0.95 * cfg.total_slots), dtype=np.uint64)
    ref = oracle.OracleFilter(oracle.cfg_from(cfg))
    rok, _, _ = ref.insert_batch(keys)
    filt = CuckooFilter(cfg, tiled=True)
    res = filt.insert_batch(keys)
    assert filt.last_schedule[0] == "region"
    assert abs(res.n_failed - int((~rok).sum())) <= (0 if b == 16 else max(2, len(keys) // 20000))
    assert len(filt) == res.n_ok
    assert filt.query_batch(keys[res.ok]).all()
    assert filt.last_schedule[0] == "region"
    neg = rng.integers(1 << 62, 1 << 63, size=200_000, dtype=np.uint64)
    snap = oracle.OracleFilter(oracle.cfg_from(cfg))
    snap.words[:] = filt.words
    assert np.array_equal(filt.query_batch(neg), snap.query_batch(neg))
    d = filt.delete_batch(keys[res.ok])
    assert d.all() and len(filt) == 0
    assert int(np.count_nonzero(filt.stored_tags())) <= 32
