"""Rollback and CAS-race coverage (SURVEY.md §5 race detection).

* BFS two-step relocation rollback: the GPU counterpart of the reference's
  sabotaged ``lane_cas`` (pkg/tests/test_filter.py:224-259).  The debug hook
  ``ckf_debug_fault_origin_cas`` makes a "concurrent writer" replace the
  origin lane with a stale tag right before the chain's origin CAS, so the
  chain must remove the copy it just made in the alternate bucket.  A leaked
  copy would break ``occupancy == stored tags`` (exactly, for one insert; up
  to the relocation's inherent race window inside a concurrent batch).
* Duplicate-key stress: thousands of threads insert copies of a few keys whose
  bucket pairs are disjoint, so every copy races for the same 2b slots; each
  key must end with exactly min(copies, 2b) stored tags, on both schedules and
  both eviction strategies, and deleting every copy must empty the table.
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

import oracle
from paper_2603_15486_b200 import CuckooFilter, FilterConfig, _lib, derive_placement

pytestmark = pytest.mark.gpu


def arm_faults(n: int) -> None:
    _lib.check(_lib.lib().ckf_debug_fault_origin_cas(n))


def faults_pending() -> int:
    c = ctypes.c_uint(0)
    _lib.check(_lib.lib().ckf_debug_faults_pending(ctypes.byref(c)))
    return int(c.value)


def stored(filt) -> int:
    return int(np.count_nonzero(filt.stored_tags()))


def test_bfs_rollback_clears_inserted_copy():
    """Mirror of the reference test: one fresh key whose two buckets are full,
    one sabotaged origin CAS, the insert still succeeds and exactly one tag is
    added."""
    cfg = FilterConfig(bucket_count=1 << 8, bucket_slots=16, eviction="bfs", seed=21)
    filt = CuckooFilter(cfg)
    rng = np.random.default_rng(31)
    filt.insert_batch(rng.integers(0, 1 << 32, size=int(0.90 * cfg.total_slots), dtype=np.uint64))
    tags = filt.stored_tags()
    full = {i for i in range(cfg.bucket_count) if np.count_nonzero(tags[i]) == cfg.bucket_slots}
    probe = 1 << 40
    while True:
        place = derive_placement(probe, cfg)
        if place.i1 in full and place.i2 in full:
            break
        probe += 1
    before = stored(filt)
    arm_faults(1)
    try:
        res = filt.insert(probe)
        torch.cuda.synchronize()
        assert faults_pending() == 0, "test did not reach the two-step relocation"
    finally:
        arm_faults(0)
    assert res.ok
    after = stored(filt)
    assert after == before + 1, "failed relocation leaked a duplicate tag"
    assert len(filt) == after, "occupancy out of step with stored tags"


@pytest.mark.parametrize("tiled", [False, True], ids=["direct", "region"])
def test_bfs_rollbacks_inside_a_concurrent_batch(tiled):
    """Many sabotaged relocations inside one high-load batch (the region
    schedule's eviction pass uses the room map): every rollback removes its
    copy, so occupancy still equals the stored tags."""
    cfg = FilterConfig(bucket_count=1 << 12, bucket_slots=16, eviction="bfs", seed=5)
    filt = CuckooFilter(cfg, tiled=tiled)
    rng = np.random.default_rng(7)
    filt.insert_batch(rng.integers(0, 1 << 32, size=int(0.90 * cfg.total_slots), dtype=np.uint64))
    before = stored(filt)
    assert before == len(filt)
    arm_faults(200)
    try:
        res = filt.insert_batch(rng.integers(1 << 33, 1 << 34, size=int(0.07 * cfg.total_slots), dtype=np.uint64))
        torch.cuda.synchronize()
        used = 200 - faults_pending()
    finally:
        arm_faults(0)
    assert used > 20, used
    after = stored(filt)
    # every rollback removed its copy, up to the two-step relocation's own
    # window: a copy another chain relocates before this chain
    # rolls it back stays, one extra tag -- rare even with 200 forced rollbacks
    assert 0 <= after - (before + res.n_ok) <= 3, (after, before, res.n_ok)
    assert len(filt) == before + res.n_ok


def disjoint_keys(cfg, count, rng):
    """`count` keys whose bucket pairs share no bucket."""
    seen, out = set(), []
    while len(out) < count:
        k = int(rng.integers(0, 1 << 62))
        p = derive_placement(k, cfg)
        if p.i1 == p.i2 or p.i1 in seen or p.i2 in seen:
            continue
        seen.update((p.i1, p.i2))
        out.append(k)
    return np.array(out, dtype=np.uint64)


@pytest.mark.parametrize("tiled", [False, True], ids=["direct", "region"])
@pytest.mark.parametrize("eviction", ["bfs", "dfs"])
def test_duplicate_keys_race_for_one_bucket_pair(tiled, eviction):
    cfg = FilterConfig(bucket_count=1 << 12, bucket_slots=16, eviction=eviction, max_evictions=64, seed=9)
    rng = np.random.default_rng(11)
    distinct = disjoint_keys(cfg, 48, rng)
    copies = 100
    keys = np.repeat(distinct, copies)
    rng.shuffle(keys)
    filt = CuckooFilter(cfg, tiled=tiled)
    res = filt.insert_batch(keys)
    assert filt.last_schedule[0] == ("region" if tiled else "direct")
    cap = 2 * cfg.bucket_slots  # every copy of a key lives in its two buckets
    assert res.n_ok == len(distinct) * cap
    assert stored(filt) == len(filt) == len(distinct) * cap
    # the oracle agrees on the count (sequential order, same pair capacity)
    rok, _, _ = oracle.OracleFilter(oracle.cfg_from(cfg)).insert_batch(keys)
    assert int(rok.sum()) == res.n_ok
    assert filt.query_batch(distinct).all()
    d = filt.delete_batch(keys)
    assert int(d.sum()) == len(distinct) * cap
    assert len(filt) == 0 and not filt.words.any()
