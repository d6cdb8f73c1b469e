"""GPU parity against the reference's golden vectors and the CPU oracle.

Bit-exact where the reference is deterministic:
  * hash / placement kernels vs xxhash + derive_placement;
  * query kernel on the reference's own tables (every scenario, + and -);
  * parity-mode (sequential) insert and delete: word array, ok, evictions,
    lost fingerprints, occupancy -- identical to insert_batch(workers=1).
Semantic where the reference is itself order-dependent (the concurrent
production kernels, SURVEY.md §8(c) parity rules):
  * no false negatives, insert-success counts equal to the reference's,
    occupancy == stored lanes, per-bucket tag multisets after delete.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from conftest import golden, scenario_cfg
from paper_2603_15486_b200 import CuckooFilter, FilterConfig
from paper_2603_15486_b200.kernels import hash_batch, place_batch

pytestmark = pytest.mark.gpu

DATA, MANIFEST = golden()
SCENARIOS = MANIFEST["scenarios"]
FILLABLE = [s for s in SCENARIOS if s["n_failed"] == 0]
OVERFULL = [s for s in SCENARIOS if s["n_failed"] > 0]


def dev(a: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).cuda()


def host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint64)


def load_words(filt: CuckooFilter, words: np.ndarray, occ: int) -> None:
    filt.words_device.copy_(torch.from_numpy(words.view(np.int64)))
    filt._occ.fill_(occ)


def bucket_multisets(words: np.ndarray, cfg) -> np.ndarray:
    f, tpw = cfg.fingerprint_bits, cfg.tags_per_word
    w = words.reshape(cfg.bucket_count, cfg.words_per_bucket)
    lanes = np.stack([(w[:, s // tpw] >> np.uint64(f * (s % tpw))) & np.uint64((1 << f) - 1)
                      for s in range(cfg.bucket_slots)], axis=1)
    return np.sort(lanes, axis=1)


def test_hash_kernel_matches_xxhash():
    keys, seeds, want = DATA["hash_keys"], DATA["hash_seeds"], DATA["hash_out"]
    for s in np.unique(seeds):
        sel = seeds == s
        assert np.array_equal(host(hash_batch(dev(keys[sel]), int(s))), want[sel])


@pytest.mark.parametrize("pl", MANIFEST["placements"], ids=lambda p: f"p{p['id']}")
def test_place_kernel_matches_reference(pl):
    cfg = FilterConfig(bucket_count=pl["m"], fingerprint_bits=pl["f"], bucket_slots=pl["b"],
                       policy=pl["policy"], seed=pl["seed"])
    keys = DATA[f"place{pl['id']}_keys"]
    fp, i1, i2 = place_batch(cfg, dev(keys))
    got = np.stack([host(fp), host(i1), host(i2)], 1)
    assert np.array_equal(got, DATA[f"place{pl['id']}_fii"])
    # hashed-input variant (used by the multi-GPU router)
    h = hash_batch(dev(keys), pl["seed"])
    fp2, i12, i22 = place_batch(cfg, h, hashed=True)
    assert torch.equal(fp, fp2) and torch.equal(i1, i12) and torch.equal(i2, i22)


@pytest.mark.parametrize("tiled", [False, True], ids=["direct", "tiled"])
@pytest.mark.parametrize("sc", SCENARIOS, ids=lambda s: s["name"])
def test_query_kernel_on_reference_tables(sc, tiled):
    name = sc["name"]
    filt = CuckooFilter(scenario_cfg(sc, FilterConfig), tiled=tiled)
    load_words(filt, DATA[f"{name}_words_ins"], sc["occ_after_insert"])
    assert np.array_equal(filt.query_batch(DATA[f"{name}_keys"]).astype(np.uint8), DATA[f"{name}_qpos"])
    assert np.array_equal(filt.query_batch(DATA[f"{name}_neg"]).astype(np.uint8), DATA[f"{name}_qneg"])
    load_words(filt, DATA[f"{name}_words_del"], sc["occ_after_delete"])
    assert np.array_equal(filt.query_batch(DATA[f"{name}_keys"]).astype(np.uint8), DATA[f"{name}_qafter"])


@pytest.mark.parametrize("sc", SCENARIOS, ids=lambda s: s["name"])
def test_parity_mode_is_bit_identical(sc):
    name = sc["name"]
    filt = CuckooFilter(scenario_cfg(sc, FilterConfig), deterministic=True)
    res = filt.insert_batch(DATA[f"{name}_keys"])
    assert np.array_equal(res.ok.astype(np.uint8), DATA[f"{name}_ok"])
    assert np.array_equal(res.evictions, DATA[f"{name}_ev"])
    assert np.array_equal(res.lost_fingerprints, DATA[f"{name}_lost"])
    assert np.array_equal(filt.words, DATA[f"{name}_words_ins"])
    assert filt.occupancy == sc["occ_after_insert"] == res.n_ok
    dres = filt.delete_batch(DATA[f"{name}_dkeys"])
    assert np.array_equal(dres.astype(np.uint8), DATA[f"{name}_dres"])
    assert np.array_equal(filt.words, DATA[f"{name}_words_del"])
    assert filt.occupancy == sc["occ_after_delete"]
    hdr = filt.to_bytes()[:44]
    assert hdr == bytes(DATA[f"{name}_blobhdr"]), "CKGF header differs from the reference dump"


@pytest.mark.parametrize("tiled", [False, True], ids=["direct", "tiled"])
@pytest.mark.parametrize("sc", FILLABLE, ids=lambda s: s["name"])
def test_concurrent_insert_semantics(sc, tiled):
    name = sc["name"]
    cfg = scenario_cfg(sc, FilterConfig)
    filt = CuckooFilter(cfg, tiled=tiled)
    keys = DATA[f"{name}_keys"]
    res = filt.insert_batch(keys)
    assert res.n_failed == sc["n_failed"] == 0, "insert-success count differs from the reference"
    assert res.ok.all()
    assert filt.query_batch(keys).all(), "false negative after concurrent insert"
    assert len(filt) == len(keys) == int(np.count_nonzero(filt.stored_tags()))
    ev = res.evictions
    assert ev.min() >= 0 and ev.max() <= cfg.max_evictions
    assert (res.lost_fingerprints == 0).all()


@pytest.mark.parametrize("tiled", [False, True], ids=["direct", "tiled"])
@pytest.mark.parametrize("sc", OVERFULL, ids=lambda s: s["name"])
def test_concurrent_insert_overfull_invariants(sc, tiled):
    name = sc["name"]
    cfg = scenario_cfg(sc, FilterConfig)
    filt = CuckooFilter(cfg, tiled=tiled)
    keys = DATA[f"{name}_keys"]
    res = filt.insert_batch(keys)
    assert res.n_failed > 0
    assert res.n_ok + res.n_failed == len(keys)
    assert len(filt) == res.n_ok == int(np.count_nonzero(filt.stored_tags()))
    failed = ~res.ok
    assert (res.evictions[failed] == cfg.max_evictions).all()
    assert (res.lost_fingerprints[failed] > 0).all() and (res.lost_fingerprints[~failed] == 0).all()


@pytest.mark.parametrize("tiled", [False, True], ids=["direct", "tiled"])
@pytest.mark.parametrize("sc", SCENARIOS, ids=lambda s: s["name"])
def test_concurrent_delete_on_reference_table(sc, tiled):
    """Concurrent delete of the stored keys, then the reference's trailing
    never-inserted keys in parity mode.  (Concurrent deletes of NEVER-inserted
    keys race real keys for colliding lanes -- the reference forbids them,
    filter.py:255-256 -- so only the stored-key part is run concurrently.)"""
    name = sc["name"]
    cfg = scenario_cfg(sc, FilterConfig)
    filt = CuckooFilter(cfg, tiled=tiled)
    load_words(filt, DATA[f"{name}_words_ins"], sc["occ_after_insert"])
    dkeys, want = DATA[f"{name}_dkeys"], DATA[f"{name}_dres"]
    npos = len(DATA[f"{name}_keys"][::3])
    got = filt.delete_batch(dkeys[:npos])
    assert np.array_equal(got.astype(np.uint8), want[:npos])
    got_neg = filt.delete_batch(dkeys[npos:], deterministic=True)
    assert np.array_equal(got_neg.astype(np.uint8), want[npos:])
    assert filt.occupancy == sc["occ_after_delete"]
    # lane positions may differ from the sequential order; bucket contents may not
    assert np.array_equal(bucket_multisets(filt.words, cfg), bucket_multisets(DATA[f"{name}_words_del"], cfg))


def test_torch_inputs_stay_on_device():
    cfg = FilterConfig(bucket_count=1 << 10, seed=3)
    filt = CuckooFilter(cfg)
    keys = torch.randint(0, 1 << 62, (5000,), device="cuda", dtype=torch.int64)
    res = filt.insert_batch(keys)
    assert isinstance(res.ok, torch.Tensor) and res.ok.is_cuda and bool(res.ok.all())
    q = filt.query_batch(keys)
    assert isinstance(q, torch.Tensor) and q.is_cuda and bool(q.all())
    assert torch.equal(filt.query_batch(keys.view(torch.uint64)), q)
    d = filt.delete_batch(keys)
    assert bool(d.all()) and len(filt) == 0
