"""Host-side API surface: FilterConfig validation and geometry, the FPR model
and sizing helper, EvictionStats, and CKGF header handling (mirrors
reference pkg/tests/test_placement.py:216-267, test_analytics.py,
test_filter.py:190-219, :323-374)."""

from __future__ import annotations

import math
import random
import struct

import numpy as np
import pytest

from paper_2603_15486_b200 import (ConfigError, Eviction, EvictionStats, FilterConfig, Policy,
                                   analytic_fpr, effective_fingerprint_bits, size_for)
from paper_2603_15486_b200.filter import _HEADER, CuckooFilter


def test_config_defaults():
    cfg = FilterConfig(bucket_count=64)
    assert (cfg.fingerprint_bits, cfg.bucket_slots, cfg.policy, cfg.eviction) == (16, 16, Policy.XOR, Eviction.DFS)
    assert (cfg.max_evictions, cfg.seed, cfg.tags_per_word, cfg.words_per_bucket) == (500, 0, 4, 4)
    assert (cfg.total_slots, cfg.total_words, cfg.payload_bits, cfg.index_mask) == (1024, 256, 16, 63)


def test_config_accepts_strings():
    cfg = FilterConfig(bucket_count=10, policy="offset", eviction="bfs")
    assert cfg.policy is Policy.OFFSET and cfg.eviction is Eviction.BFS
    assert (cfg.payload_bits, cfg.choice_bit, cfg.index_mask) == (15, 1 << 15, 0)


@pytest.mark.parametrize("kwargs", [
    dict(bucket_count=64, fingerprint_bits=12),
    dict(bucket_count=64, fingerprint_bits=9),
    dict(bucket_count=64, bucket_slots=0),
    dict(bucket_count=64, bucket_slots=3, fingerprint_bits=16),
    dict(bucket_count=0),
    dict(bucket_count=10),
    dict(bucket_count=1, policy=Policy.OFFSET),
    dict(bucket_count=64, max_evictions=0),
    dict(bucket_count=64, seed=-1),
    dict(bucket_count=64, policy="nonsense"),
])
def test_config_rejections(kwargs):
    with pytest.raises((ConfigError, ValueError)):
        FilterConfig(**kwargs)


def test_config_small_word_shapes():
    cfg = FilterConfig(bucket_count=16, fingerprint_bits=8, bucket_slots=8)
    assert cfg.words_per_bucket == 1 and cfg.total_words == 16
    cfg32 = FilterConfig(bucket_count=4, fingerprint_bits=32, bucket_slots=2)
    assert cfg32.tags_per_word == 2 and cfg32.words_per_bucket == 1


def test_gpu_slot_bound_is_explicit():
    with pytest.raises(ConfigError):
        FilterConfig(bucket_count=64, bucket_slots=256).ckf_params()


# ---- FPR model (analytics.py:20-29; pins from test_analytics.py:17-22) ----

def test_fpr_pins():
    assert abs(analytic_fpr(16, 16, 0.95) - 4.637632e-4) < 1e-9
    assert abs(analytic_fpr(8, 4, 0.95) - 2.930759e-2) < 1e-7
    assert analytic_fpr(16, 16, 0.0) == 0.0


def test_fpr_matches_naive_form_and_f32():
    rng = random.Random(41)
    for _ in range(300):
        f, b, a = rng.choice([4, 8, 12, 16, 24, 32]), rng.randint(1, 64), rng.random()
        assert math.isclose(analytic_fpr(f, b, a), 1.0 - (1.0 - 2.0 ** -f) ** (2.0 * b * a),
                            rel_tol=1e-6, abs_tol=1e-15)
    assert math.isclose(analytic_fpr(32, 16, 0.95), 2 * 16 * 0.95 / 2**32, rel_tol=1e-6)
    for args in [(0, 16, 0.5), (16, 0, 0.5), (16, 16, -0.1), (16, 16, 1.5)]:
        with pytest.raises(ValueError):
            analytic_fpr(*args)


def test_size_for():
    assert size_for(1000, 0.95, bucket_slots=16, policy=Policy.XOR) == 128
    assert size_for(1000, 0.95, bucket_slots=16, policy=Policy.OFFSET) == 66
    assert size_for(512, 0.5, 16, Policy.XOR) == size_for(512, 0.5, 16, Policy.OFFSET) == 64
    rng = random.Random(47)
    for _ in range(200):
        n, b, a = rng.randint(1, 1 << 20), rng.choice([4, 8, 16, 32]), rng.uniform(0.05, 1.0)
        m = size_for(n, a, bucket_slots=b, policy=Policy.OFFSET)
        assert m * b * a >= n and (m <= 2 or (m - 1) * b * a < n)
    for args in [(0, 0.95), (10, 0.0), (10, 1.5)]:
        with pytest.raises(ValueError):
            size_for(*args)
    assert effective_fingerprint_bits(FilterConfig(bucket_count=66, policy="offset")) == 15


# ---- eviction stats (test_filter.py:190-201) ----

def test_eviction_stats_percentiles():
    stats = EvictionStats(np.array([0] * 9 + [7], dtype=np.int64))
    assert stats.percentile(50) == 0 and stats.p99 == 7 and stats.percentile(100) == 7
    assert stats.max == 7 and stats.mean == pytest.approx(0.7)
    ps = [stats.percentile(p) for p in range(0, 101, 5)]
    assert ps == sorted(ps)
    assert EvictionStats(np.zeros(100, dtype=np.int64)).p99 == 0
    assert EvictionStats(np.array([], dtype=np.int64)).p99 == 0


# ---- CKGF header validation (filter.py:536-569) is host logic ----

def _blob(magic=b"CKGF", version=1, f=16, b=16, m=64, pol=0, occ=0, seed=0, words=None):
    words = np.zeros(m * b * f // 64, dtype="<u8") if words is None else words
    return _HEADER.pack(magic, version, f, b, m, pol, occ, seed) + words.tobytes()


@pytest.mark.parametrize("blob,match", [
    (b"XXXX" + _blob()[4:], "magic"),
    (_blob()[:4] + struct.pack("<I", 99) + _blob()[8:], "version"),
    (_blob()[:10], "header"),
    (_blob()[:-8], "bytes"),
    (_blob(pol=7), "policy"),
])
def test_from_bytes_rejects_corruption(blob, match):
    with pytest.raises(ValueError, match=match):
        CuckooFilter.from_bytes(blob)


@pytest.mark.parametrize("n", [1, 5, 1 << 10, (1 << 10) + 1, 1 << 12, (1 << 12) + 3, 10_000, 1 << 16])
def test_host_chunk_bounds_cover_batch_with_short_tail(monkeypatch, n):
    """Host pipeline chunking: contiguous, covers [0, n), no chunk above
    HOST_CHUNK, and the last chunk is at most HOST_TAIL keys."""
    monkeypatch.setattr(CuckooFilter, "HOST_CHUNK", 1 << 12)
    monkeypatch.setattr(CuckooFilter, "HOST_TAIL", 1 << 10)
    b = CuckooFilter._chunk_bounds(CuckooFilter.__new__(CuckooFilter), n)
    assert b[0][0] == 0 and b[-1][1] == n
    assert all(hi > lo for lo, hi in b) and all(x[1] == y[0] for x, y in zip(b, b[1:]))
    assert max(hi - lo for lo, hi in b) <= 1 << 12
    assert b[-1][1] - b[-1][0] <= 1 << 10
