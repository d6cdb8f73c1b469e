"""ctypes front-end of the CPU oracle (``oracle/ckf_oracle.c``).

TEST INFRASTRUCTURE ONLY -- this package is the parity checker and the CPU
baseline, never the product path.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (``cpu_baseline`` and ``--impl reference``) may import it.

The C file restates the reference ``swarcuckoo._kernels`` numba kernels
(/root/reference/pkg/src/swarcuckoo/_kernels.py) and is pinned against golden
vectors generated from the reference itself (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libckf_oracle.so"

_HIGH = {8: 0x8080808080808080, 16: 0x8000800080008000, 32: 0x8000000080000000}


class CkCfg(ctypes.Structure):
    """Mirror of ``ck_cfg`` -- the reference's ``_kargs`` tuple (filter.py:150-154)."""

    _fields_ = [
        ("seed", ctypes.c_uint64),
        ("payload_bits", ctypes.c_uint64),
        ("f", ctypes.c_uint64),
        ("b", ctypes.c_uint64),
        ("m", ctypes.c_uint64),
        ("mask", ctypes.c_uint64),
        ("wpb", ctypes.c_int64),
        ("tpw", ctypes.c_int64),
        ("high", ctypes.c_uint64),
        ("choice_bit", ctypes.c_uint64),
        ("policy", ctypes.c_int),
        ("strategy", ctypes.c_int),
        ("max_evictions", ctypes.c_int64),
        ("worker", ctypes.c_uint64),
    ]


def build(force: bool = False) -> Path:
    """Compile the oracle with gcc (make -C oracle)."""
    src = _HERE / "ckf_oracle.c"
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.POINTER
        u64p = ctypes.c_void_p
        L.ck_xxh64.restype = ctypes.c_uint64
        L.ck_xxh64.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.ck_tag_hash.restype = ctypes.c_uint64
        L.ck_tag_hash.argtypes = [ctypes.c_uint64]
        L.ck_smix.restype = ctypes.c_uint64
        L.ck_smix.argtypes = [ctypes.c_uint64]
        L.ck_rng_init.restype = ctypes.c_uint64
        L.ck_rng_init.argtypes = [ctypes.c_uint64] * 3
        L.ck_zero_mask.restype = ctypes.c_uint64
        L.ck_zero_mask.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.ck_broadcast.restype = ctypes.c_uint64
        L.ck_broadcast.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.ck_hash_batch.argtypes = [u64p, ctypes.c_int64, ctypes.c_uint64, u64p]
        L.ck_place_batch.argtypes = [P(CkCfg), u64p, ctypes.c_int64, u64p, u64p, u64p]
        L.ck_place_hashes.argtypes = [P(CkCfg), u64p, ctypes.c_int64, u64p, u64p, u64p]
        L.ck_alt.restype = ctypes.c_uint64
        L.ck_alt.argtypes = [P(CkCfg), ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                             P(ctypes.c_uint64)]
        L.ck_insert_batch.restype = ctypes.c_int64
        L.ck_insert_batch.argtypes = [P(CkCfg), u64p, u64p, ctypes.c_int64, u64p, u64p, u64p,
                                      ctypes.c_int]
        L.ck_delete_batch.restype = ctypes.c_int64
        L.ck_delete_batch.argtypes = [P(CkCfg), u64p, u64p, ctypes.c_int64, u64p, ctypes.c_int]
        L.ck_query_batch.argtypes = [P(CkCfg), u64p, u64p, ctypes.c_int64, u64p, ctypes.c_int,
                                     ctypes.c_int]
        for fn in (L.ck_insert_batch_mt, L.ck_delete_batch_mt):
            fn.restype = ctypes.c_int64
            fn.argtypes = [P(CkCfg), u64p, u64p, ctypes.c_int64, u64p, ctypes.c_int, ctypes.c_int]
        L.ck_try_insert.restype = ctypes.c_int64
        L.ck_try_insert.argtypes = [P(CkCfg), u64p, ctypes.c_int64, ctypes.c_uint64]
        L.ck_remove_tag.restype = ctypes.c_int64
        L.ck_remove_tag.argtypes = [P(CkCfg), u64p, ctypes.c_int64, ctypes.c_uint64]
        L.ck_find_tag.restype = ctypes.c_int
        L.ck_find_tag.argtypes = [P(CkCfg), u64p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def make_cfg(bucket_count: int, fingerprint_bits: int = 16, bucket_slots: int = 16,
             policy: str = "xor", eviction: str = "dfs", max_evictions: int = 500,
             seed: int = 0, worker: int = 0) -> CkCfg:
    """Derived geometry exactly as FilterConfig computes it (placement.py:104-136)."""
    f, b, m = fingerprint_bits, bucket_slots, bucket_count
    pol = 0 if str(getattr(policy, "value", policy)) == "xor" else 1
    strat = 0 if str(getattr(eviction, "value", eviction)) == "dfs" else 1
    return CkCfg(
        seed=seed, payload_bits=f - 1 if pol else f, f=f, b=b, m=m,
        mask=(m - 1) if (m & (m - 1)) == 0 else 0,
        wpb=b * f // 64, tpw=64 // f, high=_HIGH[f],
        choice_bit=(1 << (f - 1)) if pol else 0,
        policy=pol, strategy=strat, max_evictions=max_evictions, worker=worker,
    )


def cfg_from(fc, worker: int = 0) -> CkCfg:
    """Build a CkCfg from any FilterConfig-like object (ours or the reference's)."""
    return make_cfg(fc.bucket_count, fc.fingerprint_bits, fc.bucket_slots, fc.policy,
                    fc.eviction, fc.max_evictions, fc.seed, worker)


def _keys(keys) -> np.ndarray:
    a = np.ascontiguousarray(keys, dtype=np.uint64)
    if a.ndim != 1:
        raise ValueError("keys must be one-dimensional")
    return a


def hash_batch(keys, seed: int) -> np.ndarray:
    k = _keys(keys)
    out = np.empty_like(k)
    lib().ck_hash_batch(_ptr(k), len(k), seed, _ptr(out))
    return out


def place_batch(cfg: CkCfg, keys):
    k = _keys(keys)
    fp, i1, i2 = (np.empty_like(k) for _ in range(3))
    lib().ck_place_batch(ctypes.byref(cfg), _ptr(k), len(k), _ptr(fp), _ptr(i1), _ptr(i2))
    return fp, i1, i2


def place_hashes(cfg: CkCfg, hashes):
    h = _keys(hashes)
    fp, i1, i2 = (np.empty_like(h) for _ in range(3))
    lib().ck_place_hashes(ctypes.byref(cfg), _ptr(h), len(h), _ptr(fp), _ptr(i1), _ptr(i2))
    return fp, i1, i2


class OracleFilter:
    """Sequential CPU cuckoo filter with the reference's batch semantics."""

    def __init__(self, cfg: CkCfg):
        self.cfg = cfg
        self.words = np.zeros(int(cfg.m) * int(cfg.wpb), dtype=np.uint64)
        self.occupancy = 0

    def insert_batch(self, keys, hashed: bool = False):
        k = _keys(keys)
        n = len(k)
        ok = np.zeros(n, np.uint8)
        ev = np.zeros(n, np.int64)
        lost = np.zeros(n, np.uint64)
        n_ok = lib().ck_insert_batch(ctypes.byref(self.cfg), _ptr(self.words), _ptr(k), n,
                                     _ptr(ok), _ptr(ev), _ptr(lost), int(hashed))
        self.occupancy += int(n_ok)
        return ok.view(np.bool_), ev, lost

    def insert_batch_mt(self, keys, threads: int, hashed: bool = False) -> np.ndarray:
        """The reference's workers>1 insert (filter.py:422-438): contiguous chunks,
        one thread and worker id each, atomic word CASes.  CPU baseline only."""
        k = _keys(keys)
        ok = np.zeros(len(k), np.uint8)
        n_ok = lib().ck_insert_batch_mt(ctypes.byref(self.cfg), _ptr(self.words), _ptr(k), len(k),
                                        _ptr(ok), int(hashed), int(threads))
        self.occupancy += int(n_ok)
        return ok.view(np.bool_)

    def delete_batch_mt(self, keys, threads: int, hashed: bool = False) -> np.ndarray:
        """The reference's workers>1 delete (filter.py:483-500)."""
        k = _keys(keys)
        out = np.zeros(len(k), np.uint8)
        n_ok = lib().ck_delete_batch_mt(ctypes.byref(self.cfg), _ptr(self.words), _ptr(k), len(k),
                                        _ptr(out), int(hashed), int(threads))
        self.occupancy -= int(n_ok)
        return out.view(np.bool_)

    def query_batch(self, keys, threads: int = 1, hashed: bool = False) -> np.ndarray:
        k = _keys(keys)
        out = np.zeros(len(k), np.uint8)
        lib().ck_query_batch(ctypes.byref(self.cfg), _ptr(self.words), _ptr(k), len(k),
                             _ptr(out), threads, int(hashed))
        return out.view(np.bool_)

    def delete_batch(self, keys, hashed: bool = False) -> np.ndarray:
        k = _keys(keys)
        out = np.zeros(len(k), np.uint8)
        n_ok = lib().ck_delete_batch(ctypes.byref(self.cfg), _ptr(self.words), _ptr(k), len(k),
                                     _ptr(out), int(hashed))
        self.occupancy -= int(n_ok)
        return out.view(np.bool_)

    def clear(self):
        self.words[:] = 0
        self.occupancy = 0
