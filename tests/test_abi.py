"""The C-ABI library: loads on a GPU-less host, exports every symbol that
include/ckf.h declares, validates parameters like FilterConfig, and its
host-compiled copy of the kernel semantics header matches the reference's
golden vectors.  No kernel is launched here."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden
from paper_2603_15486_b200 import FilterConfig, _lib, derive_placement, hash_key

HEADER = ROOT / "include" / "ckf.h"
DATA, MANIFEST = golden()


def declared_symbols() -> set[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(ckf_[a-z_0-9]+)\s*\(", text))


def test_header_and_binding_agree():
    assert declared_symbols() == set(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    for name in declared_symbols():
        assert hasattr(L, name), name
    assert L.ckf_abi_version() == _lib.ABI_VERSION


def test_exported_symbols_are_c_linkage():
    # nm -D lists unmangled names for extern "C"
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\b(ckf_[a-z_0-9]+)\b", out))
    assert declared_symbols() <= exported


def test_struct_sizes_match_header():
    assert ctypes.sizeof(_lib.Params) == 7 * 8 + 12 * 4
    assert _lib.RECORD_BYTES == 24 and _lib.COUNTERS_BYTES == 32


def test_strerror():
    L = _lib.lib()
    assert L.ckf_strerror(0) == b"ok"
    assert L.ckf_strerror(-22) == b"invalid argument"


@pytest.mark.parametrize("args", [
    (64, 12, 16, 0, 0, 500, 0),      # f not in {8,16,32}
    (64, 16, 3, 0, 0, 500, 0),       # b*f % 64
    (0, 16, 16, 0, 0, 500, 0),       # m < 1
    (10, 16, 16, 0, 0, 500, 0),      # xor needs power of two
    (1, 16, 16, 1, 0, 500, 0),       # offset needs m >= 2
    (64, 16, 16, 0, 0, 0, 0),        # max_evictions >= 1
    (64, 16, 16, 2, 0, 500, 0),      # bad policy
    (64, 16, 16, 0, 5, 500, 0),      # bad eviction
    (64, 16, 256, 0, 0, 500, 0),     # over the GPU slot bound
])
def test_params_init_rejects(args):
    p = _lib.Params()
    assert _lib.lib().ckf_params_init(ctypes.byref(p), *args) == _lib.EINVAL


def test_params_geometry():
    p = FilterConfig(bucket_count=3000, policy="offset", eviction="bfs", seed=9).ckf_params()
    assert (p.bucket_count, p.index_mask, p.payload_bits, p.choice_bit) == (3000, 0, 15, 1 << 15)
    assert (p.words_per_bucket, p.tags_per_word, p.high) == (4, 4, 0x8000800080008000)
    assert p.eviction == _lib.EVICT_BFS and p.seed == 9
    q = FilterConfig(bucket_count=1 << 20, fingerprint_bits=8, bucket_slots=8).ckf_params()
    assert (q.index_mask, q.words_per_bucket, q.choice_bit, q.delta_magic) == ((1 << 20) - 1, 1, 0, 0)


def test_null_and_empty_calls_are_rejected_or_noops():
    L = _lib.lib()
    p = FilterConfig(bucket_count=64).ckf_params()
    # missing table pointer
    assert L.ckf_query(ctypes.byref(p), None, None, 0, None, None, None, 0, 0, None) == _lib.EINVAL
    assert L.ckf_hash(None, 0, 0, None, None) == 0  # n == 0 is a no-op


def test_workspace_sizing():
    L = _lib.lib()
    big = FilterConfig(bucket_count=1 << 24).ckf_params()
    n = int(0.95 * (1 << 28))
    wq = L.ckf_workspace_bytes(ctypes.byref(big), n, _lib.OP_QUERY, 0)
    wi = L.ckf_workspace_bytes(ctypes.byref(big), n, _lib.OP_INSERT, 0)
    # region schedule: coarse- and fine-binned 8 B records plus a 16 B miss
    # entry per key; queries also size the bins for two records per key (dual
    # mode) and add the result bitmap
    assert 32 * n <= wi < 34 * n and 1.5 * wi < wq < 2.5 * wi
    small = FilterConfig(bucket_count=1 << 10).ckf_params()
    assert L.ckf_workspace_bytes(ctypes.byref(small), 100_000, _lib.OP_QUERY, 0) == 0  # L2-resident
    assert L.ckf_workspace_bytes(ctypes.byref(small), 100_000, _lib.OP_QUERY, _lib.FORCE_TILED) > 0
    assert L.ckf_workspace_bytes(ctypes.byref(big), n, _lib.OP_QUERY, _lib.FORCE_DIRECT) == 0
    b4 = FilterConfig(bucket_count=1 << 24, bucket_slots=4).ckf_params()  # 8-byte buckets: regions of 2^14
    assert L.ckf_workspace_bytes(ctypes.byref(b4), n, _lib.OP_QUERY, _lib.FORCE_TILED) > 0
    f32 = FilterConfig(bucket_count=1 << 24, fingerprint_bits=32).ckf_params()  # 16-byte records
    w32 = L.ckf_workspace_bytes(ctypes.byref(f32), n, _lib.OP_QUERY, _lib.FORCE_TILED)
    assert w32 > 1.5 * wq  # twice the record bytes


@pytest.mark.parametrize("lm", [24, 25, 26, 27])
def test_region_schedule_covers_large_tables(lm):
    """The region schedule applies up to 2^27 buckets (2^31 slots, configs[3]'s
    one-GPU table) with a workspace that scales with the batch, not the table;
    a call larger than one run's index field is split into runs."""
    L = _lib.lib()
    p = FilterConfig(bucket_count=1 << lm).ckf_params()
    n = int(0.95 * 16 * (1 << lm))
    for op in (_lib.OP_INSERT, _lib.OP_QUERY, _lib.OP_DELETE):
        w = L.ckf_workspace_bytes(ctypes.byref(p), n, op, 0)
        runs = ctypes.c_uint64(0)
        sc = L.ckf_schedule(ctypes.byref(p), n, op, 0, 8, 256, w, ctypes.byref(runs))
        assert sc == _lib.SCHED_REGION, (lm, op)
        # record index field: 64 - (16 + (lm - 9) + 1) bits; queries use two records per key
        ib = 64 - (16 + lm - 9 + 1)
        kmax = min((1 << ib) - 2, (1 << 31) // (2 if op == _lib.OP_QUERY else 1))
        assert runs.value == -(-n // kmax)
        per_key = w / -(-n // runs.value)
        assert per_key < (80 if op == _lib.OP_QUERY else 40), (lm, op, per_key)
        assert L.ckf_schedule(ctypes.byref(p), n, op, 0, 8, 256, w - 256, ctypes.byref(runs)) == _lib.SCHED_DIRECT
    assert L.ckf_schedule(ctypes.byref(p), n, _lib.OP_INSERT, _lib.MODE_SEQUENTIAL, 8, 256, 0,
                          ctypes.byref(runs)) == _lib.SCHED_SEQUENTIAL


def test_host_hash_matches_xxhash_package():
    keys, seeds, want = DATA["hash_keys"], DATA["hash_seeds"], DATA["hash_out"]
    got = np.array([hash_key(int(k), int(s)) for k, s in zip(keys[::7], seeds[::7])], dtype=np.uint64)
    assert np.array_equal(got, want[::7])


@pytest.mark.parametrize("pl", MANIFEST["placements"], ids=lambda p: f"p{p['id']}")
def test_host_placement_matches_reference(pl):
    cfg = FilterConfig(bucket_count=pl["m"], fingerprint_bits=pl["f"], bucket_slots=pl["b"],
                       policy=pl["policy"], seed=pl["seed"])
    keys = DATA[f"place{pl['id']}_keys"][::5]
    got = np.array([tuple(derive_placement(int(k), cfg)) for k in keys], dtype=np.uint64)
    assert np.array_equal(got, DATA[f"place{pl['id']}_fii"][::5])


@pytest.mark.parametrize("f", [8, 16, 32])
def test_host_zero_mask_matches_wordops(f):
    L = _lib.lib()
    got = np.array([L.ckf_host_zero_mask(f, int(w)) for w in DATA[f"swar{f}_words"]], dtype=np.uint64)
    assert np.array_equal(got, DATA[f"swar{f}_zmask"])


def test_offset_alt_round_trip_host():
    from paper_2603_15486_b200 import alt_index

    for m in (2, 3, 10, 66, 3072, (1 << 32) + 7):
        cfg = FilterConfig(bucket_count=m, policy="offset")
        for fp in (1, 2, 0x7FFF, 0x1234):
            for i in (0, 1, m // 2, m - 1):
                j, c = alt_index(i, fp, 0, cfg)
                assert c == 1 and 0 <= j < m and j != i
                back, c2 = alt_index(j, fp, 1, cfg)
                assert (back, c2) == (i, 0)


def test_automatic_schedule_follows_measured_crossovers():
    """Region from 1 key per bucket for insert / delete and 2 for lookups with
    32-byte buckets, 1.5 for every op with 64-byte buckets (f = 32); small
    (L2-resident) tables always direct (profiles/r02_crossover.jsonl)."""
    L = _lib.lib()

    def sched(cfg, n, op):
        p = cfg.ckf_params()
        w = L.ckf_workspace_bytes(ctypes.byref(p), n, op, 0)
        runs = ctypes.c_uint64(0)
        return L.ckf_schedule(ctypes.byref(p), n, op, 0, 8, 256, w, ctypes.byref(runs))

    f16 = FilterConfig(bucket_count=1 << 24)
    m = f16.bucket_count
    R, D = _lib.SCHED_REGION, _lib.SCHED_DIRECT
    assert sched(f16, m - 1, _lib.OP_INSERT) == D and sched(f16, m, _lib.OP_INSERT) == R
    assert sched(f16, m, _lib.OP_DELETE) == R
    assert sched(f16, 2 * m - 1, _lib.OP_QUERY) == D and sched(f16, 2 * m, _lib.OP_QUERY) == R
    f32 = FilterConfig(bucket_count=1 << 24, fingerprint_bits=32)
    for op in (_lib.OP_INSERT, _lib.OP_QUERY, _lib.OP_DELETE):
        assert sched(f32, m, op) == D and sched(f32, 3 * m // 2, op) == R
    small = FilterConfig(bucket_count=1 << 18)
    assert sched(small, 100 * small.bucket_count, _lib.OP_INSERT) == D


def test_direct_insert_room_map_workspace():
    """Direct-path BFS inserts of >= m/8 keys ask for a room map (a bit per
    bucket) + the eviction cursor and gate (the device builds the map only for
    a long eviction queue), and still run the direct schedule; one-word
    buckets, DFS, parity mode and small batches ask for nothing."""
    L = _lib.lib()
    runs = ctypes.c_uint64(0)

    def ws(cfg, n, op=_lib.OP_INSERT, flags=0):
        return L.ckf_workspace_bytes(ctypes.byref(cfg.ckf_params()), n, op, flags)

    cfg = FilterConfig(bucket_count=1 << 18, eviction="bfs")
    m, n = cfg.bucket_count, int(0.95 * cfg.total_slots)
    w = ws(cfg, n)
    assert m // 8 <= w <= m // 8 + 512
    p = cfg.ckf_params()
    assert L.ckf_schedule(ctypes.byref(p), n, _lib.OP_INSERT, 0, 8, 256, w, ctypes.byref(runs)) == _lib.SCHED_DIRECT
    assert ws(cfg, n, _lib.OP_QUERY) == 0 and ws(cfg, n, _lib.OP_DELETE) == 0
    assert ws(cfg, m // 8 - 1) == 0 and ws(cfg, n, flags=_lib.MODE_SEQUENTIAL) == 0
    assert ws(FilterConfig(bucket_count=1 << 18, eviction="dfs"), n) == 0
    assert ws(FilterConfig(bucket_count=1 << 18, bucket_slots=4), n) == 0  # chain-tail bound: no map
    big = FilterConfig(bucket_count=1 << 21, eviction="bfs")  # 64 MiB: the map is gated on the queue length
    assert (1 << 21) // 8 <= ws(big, 1 << 19) <= (1 << 21) // 8 + 512
