"""Pin the CPU oracle (oracle/ckf_oracle.c) to the reference's own outputs.

The golden vectors in tests/golden/golden_v1.npz were produced by running the
reference package (tests/golden/make_golden.py).  Every GPU parity test uses
the oracle as its checker, so the oracle itself must first match the
reference bit for bit here.
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import golden

DATA, MANIFEST = golden()
SCENARIOS = MANIFEST["scenarios"]


def test_hash_matches_xxhash_package():
    keys, seeds, want = DATA["hash_keys"], DATA["hash_seeds"], DATA["hash_out"]
    for s in np.unique(seeds):
        sel = seeds == s
        assert np.array_equal(oracle.hash_batch(keys[sel], int(s)), want[sel])


def test_appendix_b_constants():
    L = oracle.lib()
    assert L.ck_xxh64(0, 0) == 0x34C96ACDCADB1BBB
    assert L.ck_xxh64(1, 0) == 0x9F29CB17A2A49995
    assert L.ck_xxh64(0x2A, 0) == 0xB556806FB6D14353
    assert L.ck_xxh64(0xFFFFFFFFFFFFFFFF, 0) == 0x85D136ADB773C6C9
    assert L.ck_xxh64(123456789, 42) == 0x2F64F8F3490DEF3F
    assert L.ck_tag_hash(1) == 0x9E3779B9
    assert L.ck_tag_hash(0xBEEF) == 0xE22250A7
    cfg = oracle.make_cfg(1 << 16)
    fp, i1, i2 = oracle.place_batch(cfg, [0, 1, 0x2A, 0xDEADBEEF, 1 << 40])
    assert list(zip(fp, i1, i2)) == [(0x6ACD, 7099, 21380), (0xCB17, 39317, 40463),
                                     (0x806F, 17235, 50240), (0xF1A5, 3192, 6428),
                                     (0xA4C7, 54355, 41198)]
    off = oracle.make_cfg(3000, policy="offset")
    fp, i1, i2 = oracle.place_batch(off, [0, 1, 0x2A, 0xDEADBEEF, 1 << 40])
    assert list(zip(fp, i1, i2)) == [(0x6ACD, 2377, 2331), (0x4B17, 1905, 1800),
                                     (0x006F, 2142, 1247), (0x71A5, 1836, 1579),
                                     (0x24C7, 1714, 1794)]


@pytest.mark.parametrize("pl", MANIFEST["placements"], ids=lambda p: f"p{p['id']}")
def test_placement_matches_reference(pl):
    cfg = oracle.make_cfg(pl["m"], pl["f"], pl["b"], pl["policy"], seed=pl["seed"])
    fp, i1, i2 = oracle.place_batch(cfg, DATA[f"place{pl['id']}_keys"])
    assert np.array_equal(np.stack([fp, i1, i2], 1), DATA[f"place{pl['id']}_fii"])


@pytest.mark.parametrize("f", [8, 16, 32])
def test_swar_matches_wordops(f):
    L = oracle.lib()
    high = {8: 0x8080808080808080, 16: 0x8000800080008000, 32: 0x8000000080000000}[f]
    got = [L.ck_zero_mask(int(w), high) for w in DATA[f"swar{f}_words"]]
    assert np.array_equal(np.array(got, dtype=np.uint64), DATA[f"swar{f}_zmask"])
    got = [L.ck_broadcast(int(t), f) for t in DATA[f"swar{f}_tags"]]
    assert np.array_equal(np.array(got, dtype=np.uint64), DATA[f"swar{f}_bcast"])


@pytest.mark.parametrize("sc", SCENARIOS, ids=lambda s: s["name"])
def test_filter_scenario_bit_exact(sc):
    name = sc["name"]
    cfg = oracle.make_cfg(sc["m"], sc["f"], sc["b"], sc["policy"], sc["eviction"],
                          sc["max_evictions"], sc["seed"])
    filt = oracle.OracleFilter(cfg)
    ok, ev, lost = filt.insert_batch(DATA[f"{name}_keys"])
    assert np.array_equal(ok.astype(np.uint8), DATA[f"{name}_ok"])
    assert np.array_equal(ev, DATA[f"{name}_ev"])
    assert np.array_equal(lost, DATA[f"{name}_lost"])
    assert np.array_equal(filt.words, DATA[f"{name}_words_ins"])
    assert filt.occupancy == sc["occ_after_insert"]
    assert np.array_equal(filt.query_batch(DATA[f"{name}_keys"]).astype(np.uint8), DATA[f"{name}_qpos"])
    assert np.array_equal(filt.query_batch(DATA[f"{name}_neg"], threads=3).astype(np.uint8),
                          DATA[f"{name}_qneg"])
    assert np.array_equal(filt.delete_batch(DATA[f"{name}_dkeys"]).astype(np.uint8), DATA[f"{name}_dres"])
    assert np.array_equal(filt.words, DATA[f"{name}_words_del"])
    assert filt.occupancy == sc["occ_after_delete"]
    assert np.array_equal(filt.query_batch(DATA[f"{name}_keys"]).astype(np.uint8), DATA[f"{name}_qafter"])
