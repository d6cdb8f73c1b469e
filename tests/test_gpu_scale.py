"""Full-size properties on the GPU (SURVEY.md §8(c) parity rules at scale).

At 2^26 slots (128 MiB table, 63.7 M keys, the L2-tiled path) and the
benchmark's 2^28: insert-success count equal to the reference's (0 failures
at 95% load), no false negatives, occupancy == stored lanes, placement
bit-exact on a sample against the oracle, tiled and direct lookups
identical, FPR inside the 99.9% Clopper-Pearson interval of the oracle's
rate on the same keys, delete-all returns the table to all-zero words.
"""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch
from scipy.stats import beta

import oracle
from paper_2603_15486_b200 import CuckooFilter, FilterConfig, analytic_fpr
from paper_2603_15486_b200.kernels import place_batch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def gen_keys(n, seed, negative=False):
    rng = np.random.Generator(np.random.Philox(key=[seed, int(negative)]))
    if negative:
        return rng.integers(1 << 32, 1 << 64, size=n, dtype=np.uint64)
    return rng.integers(0, 1 << 32, size=n, dtype=np.uint64)


def cp_interval(k, n, conf=0.999):
    a = (1 - conf) / 2
    lo = 0.0 if k == 0 else beta.ppf(a, k, n - k + 1)
    hi = 1.0 if k == n else beta.ppf(1 - a, k + 1, n - k)
    return lo, hi


def dev(a):
    return torch.from_numpy(a.view(np.int64)).cuda()


@pytest.mark.parametrize("eviction", ["bfs", "dfs"])
def test_2pow26_insert_lookup_delete_matches_oracle(eviction):
    cfg = FilterConfig(bucket_count=1 << 22, eviction=eviction, seed=0)
    n = int(0.95 * cfg.total_slots)
    pos, neg = gen_keys(n, 0), gen_keys(10_000_000, 0, negative=True)
    kp, kn = dev(pos), dev(neg)

    # placement bit-exact on a sample
    fp, i1, i2 = place_batch(cfg, kp[:1_000_000])
    ofp, oi1, oi2 = oracle.place_batch(oracle.cfg_from(cfg), pos[:1_000_000])
    for got, want in ((fp, ofp), (i1, oi1), (i2, oi2)):
        assert np.array_equal(got.cpu().numpy().view(np.uint64), want)

    filt = CuckooFilter(cfg)  # auto: 128 MiB table, 15 keys/bucket -> tiled
    res = filt.insert_batch(kp)
    ref = oracle.OracleFilter(oracle.cfg_from(cfg))
    rok, _, _ = ref.insert_batch(pos)
    assert res.n_failed == int((~rok).sum()) == 0, "insert-success count differs from the reference"
    assert len(filt) == n == int(np.count_nonzero(filt.stored_tags()))
    assert bool(filt.query_batch(kp).all()), "false negative"

    hits = filt.query_batch(kn)
    direct = CuckooFilter(cfg, tiled=False)
    direct.words_device.copy_(filt.words_device)
    assert torch.equal(direct.query_batch(kn), hits), "tiled and direct lookups differ"
    assert torch.equal(direct.query_batch(kp[:2_000_000]), filt.query_batch(kp[:2_000_000]))

    k = int(hits.sum())
    k_ref = int(ref.query_batch(neg, threads=8).sum())
    lo, hi = cp_interval(k, len(neg))
    lo_r, hi_r = cp_interval(k_ref, len(neg))
    assert lo <= hi_r and lo_r <= hi, f"FPR {k / len(neg):.3e} vs reference {k_ref / len(neg):.3e}"
    model = analytic_fpr(16, 16, 0.95)
    assert abs(k / len(neg) - model) / model < 0.25

    d = filt.delete_batch(kp)
    assert bool(d.all()) and len(filt) == 0
    assert int(torch.count_nonzero(filt.words_device)) == 0


def test_2pow28_bench_config_properties():
    cfg = FilterConfig(bucket_count=1 << 24, eviction="bfs", seed=0)
    n = int(0.95 * cfg.total_slots)
    kp = dev(gen_keys(n, 0))
    filt = CuckooFilter(cfg)
    res = filt.insert_batch(kp)
    assert res.n_failed == 0 and len(filt) == n
    assert bool(filt.query_batch(kp).all())
    # checksum of the table is independent of the lane each tag landed in:
    # the multiset of stored tags per bucket is order-free, so its sum is too
    lanes = filt.words_device.view(-1, 4)
    total = sum(int(((lanes >> (16 * s)) & 0xFFFF).sum()) for s in range(4))
    fp, _, _ = place_batch(cfg, kp)
    assert total == int(fp.sum()), "stored fingerprints are not exactly the inserted ones"
    assert bool(filt.delete_batch(kp).all()) and len(filt) == 0
