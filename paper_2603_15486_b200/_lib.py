"""ctypes binding of ``libckf.so`` (declared in ``include/ckf.h``).

This is the Python side of the C-ABI boundary: the reference's numba
dispatch (``_k.insert_batch(words, keys, *_kargs, ...)``, filter.py:417-420)
becomes ``ckf_insert(&params, words_ptr, keys_ptr, n, ...)`` here.  ctypes
releases the GIL for the duration of each call, like the reference's
``nogil`` kernels.  There is no fallback: if the CUDA library is missing the
import fails loudly.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import os

_HERE = Path(__file__).resolve().parent
# CKF_LIB: developer override (A/B builds of the same sources); never a fallback
LIB_PATH = Path(os.environ["CKF_LIB"]) if os.environ.get("CKF_LIB") else _HERE / "libckf.so"

ABI_VERSION = 2
OK = 0
EINVAL = -22

POLICY_XOR = 0
POLICY_OFFSET = 1
EVICT_DFS = 0
EVICT_BFS = 1

MODE_CONCURRENT = 0
MODE_SEQUENTIAL = 1
INPUT_HASHED = 2
FORCE_DIRECT = 4
FORCE_TILED = 8

SCHED_DIRECT = 0
SCHED_REGION = 1
SCHED_SEQUENTIAL = 2
SCHED_NAMES = {SCHED_DIRECT: "direct", SCHED_REGION: "region", SCHED_SEQUENTIAL: "sequential"}

OP_QUERY = 0
OP_INSERT = 1
OP_DELETE = 2


class Params(ctypes.Structure):
    """``struct ckf_params`` (include/ckf.h)."""

    _fields_ = [
        ("seed", ctypes.c_uint64),
        ("bucket_count", ctypes.c_uint64),
        ("index_mask", ctypes.c_uint64),
        ("high", ctypes.c_uint64),
        ("choice_bit", ctypes.c_uint64),
        ("delta_magic", ctypes.c_uint64),
        ("worker", ctypes.c_uint64),
        ("fingerprint_bits", ctypes.c_uint32),
        ("bucket_slots", ctypes.c_uint32),
        ("words_per_bucket", ctypes.c_uint32),
        ("tags_per_word", ctypes.c_uint32),
        ("payload_bits", ctypes.c_uint32),
        ("policy", ctypes.c_uint32),
        ("eviction", ctypes.c_uint32),
        ("max_evictions", ctypes.c_uint32),
        ("shard_shift", ctypes.c_uint32),
        ("shard_mask", ctypes.c_uint32),
        ("shard_id", ctypes.c_uint32),
        ("shard_reserved", ctypes.c_uint32),
    ]


RECORD_BYTES = 24  # struct ckf_record
COUNTERS_BYTES = 32  # struct ckf_counters

# name -> (restype, argtypes); every symbol include/ckf.h declares
_vp = ctypes.c_void_p
_u64 = ctypes.c_uint64
_u32 = ctypes.c_uint32
_P = ctypes.POINTER(Params)
SIGNATURES = {
    "ckf_abi_version": (ctypes.c_int, []),
    "ckf_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "ckf_kernel_launches": (_u64, []),
    "ckf_params_init": (ctypes.c_int, [_P, _u64, _u32, _u32, ctypes.c_int, ctypes.c_int, _u32, _u64]),
    "ckf_hash": (ctypes.c_int, [_vp, _u64, _u64, _vp, _vp]),
    "ckf_place": (ctypes.c_int, [_P, _vp, _u64, _vp, _vp, _vp, ctypes.c_uint, _vp]),
    "ckf_workspace_bytes": (_u64, [_P, _u64, ctypes.c_int, ctypes.c_uint]),
    "ckf_schedule": (ctypes.c_int, [_P, _u64, ctypes.c_int, ctypes.c_uint, _vp, _vp, _u64,
                                    ctypes.POINTER(_u64)]),
    "ckf_insert": (ctypes.c_int, [_P, _vp, _vp, _u64, _vp, _vp, _vp, _vp, _u64, _vp, _vp,
                                  _vp, _u64, ctypes.c_uint, _vp]),
    "ckf_query": (ctypes.c_int, [_P, _vp, _vp, _u64, _vp, _vp, _vp, _u64, ctypes.c_uint, _vp]),
    "ckf_delete": (ctypes.c_int, [_P, _vp, _vp, _u64, _vp, _vp, _vp, _vp, _u64, ctypes.c_uint,
                                  _vp]),
    "ckf_params_set_shard": (ctypes.c_int, [_P, _u32, _u32, _u32]),
    "ckf_route_partition_padded": (ctypes.c_int, [_vp, _u64, _u32, _u32, _u64, _vp, _vp, _vp, _vp, _vp, _u64,
                                                  _vp]),
    "ckf_route_unpermute": (ctypes.c_int, [_vp, _vp, _u64, _u32, _vp, _vp]),
    "ckf_mixed": (ctypes.c_int, [_P, _vp, _vp, _vp, _u64, _vp, _vp, _u64, _vp, _vp, ctypes.c_uint, _vp]),
    "ckf_route_workspace_bytes": (_u64, [_u64, _u32]),
    "ckf_route_partition": (ctypes.c_int, [_vp, _u64, _u32, _u32, _vp, _vp, _vp, _vp, _u64, _vp]),
    "ckf_kmer_workspace_bytes": (_u64, [_u64]),
    "ckf_kmers": (ctypes.c_int, [_vp, _u64, _u32, _vp, _vp, _vp, _u64, _vp]),
    "ckf_debug_fault_origin_cas": (ctypes.c_int, [ctypes.c_uint]),
    "ckf_debug_faults_pending": (ctypes.c_int, [ctypes.POINTER(ctypes.c_uint)]),
    "ckf_host_hash": (_u64, [_u64, _u64]),
    "ckf_host_place": (None, [_P, _u64, ctypes.POINTER(_u64), ctypes.POINTER(_u64),
                              ctypes.POINTER(_u64)]),
    "ckf_host_alt": (_u64, [_P, _u64, _u64, _u64, ctypes.POINTER(_u64)]),
    "ckf_host_zero_mask": (_u64, [_u32, _u64]),
}


class CkfError(RuntimeError):
    """A non-zero return code of the C ABI."""


_lib = None


def lib() -> ctypes.CDLL:
    """Load libckf.so once; raise if it was not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')"
            )
        L = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.ckf_abi_version() != ABI_VERSION:
            raise ImportError(f"libckf ABI {L.ckf_abi_version()} != expected {ABI_VERSION}")
        _lib = L
    return _lib


def kernel_launches() -> int:
    """Kernels libckf.so has launched in this process (bench evidence)."""
    return int(lib().ckf_kernel_launches())


def check(rc: int) -> None:
    if rc != OK:
        msg = lib().ckf_strerror(rc).decode()
        if rc == EINVAL:
            raise ValueError(f"libckf: {msg}")
        raise CkfError(f"libckf error {rc}: {msg}")


def make_params(bucket_count: int, fingerprint_bits: int, bucket_slots: int, policy: int,
                eviction: int, max_evictions: int, seed: int) -> Params:
    p = Params()
    if max_evictions > 0xFFFFFFFF:
        raise ValueError("max_evictions must fit in 32 bits on the GPU path")
    check(lib().ckf_params_init(ctypes.byref(p), bucket_count, fingerprint_bits, bucket_slots,
                                policy, eviction, max_evictions, seed))
    return p
