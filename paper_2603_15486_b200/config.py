"""Filter configuration and key placement -- the host side of the contract.

Mirrors the public surface of the reference ``swarcuckoo.placement``
(/root/reference/pkg/src/swarcuckoo/placement.py): ``FilterConfig`` with the
same fields, defaults, validation and derived geometry,
the ``Policy`` / ``Eviction`` enums and ``derive_placement``
(P:219-232).  The arithmetic of ``derive_placement`` is NOT re-implemented in
Python: it calls ``ckf_host_place`` in libckf.so, i.e. the same
``ckf_semantics.cuh`` source the CUDA kernels are compiled from.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from enum import Enum
from typing import NamedTuple

from .errors import ConfigError

LANE_WIDTHS = (8, 16, 32)
MASK64 = (1 << 64) - 1
MAX_GPU_BUCKET_SLOTS = 128  # BFS candidate scratch bound of the kernels


class Policy(str, Enum):
    """Alternate-bucket policy: partial-key XOR or offset with residency bit."""

    XOR = "xor"
    OFFSET = "offset"


class Eviction(str, Enum):
    """Eviction chain strategy when both candidate buckets are full."""

    DFS = "dfs"
    BFS = "bfs"


def _is_pow2(x: int) -> bool:
    return x > 0 and (x & (x - 1)) == 0


@dataclass(frozen=True)
class FilterConfig:
    """Static parameters of one filter (reference FilterConfig).

    ``bucket_count`` (m) buckets of ``bucket_slots`` (b) lanes of
    ``fingerprint_bits`` (f) bits; capacity m*b.  Constraints: f in
    {8, 16, 32}; b >= 1 with b*f a multiple of 64; xor needs a power-of-two
    m; offset needs m >= 2; max_evictions >= 1; seed fits in 64 bits.
    """

    bucket_count: int
    fingerprint_bits: int = 16
    bucket_slots: int = 16
    policy: Policy = Policy.XOR
    eviction: Eviction = Eviction.DFS
    max_evictions: int = 500
    seed: int = 0

    def __post_init__(self):
        f, b, m = self.fingerprint_bits, self.bucket_slots, self.bucket_count
        if f not in LANE_WIDTHS:
            raise ConfigError(f"fingerprint_bits must be one of {LANE_WIDTHS}, got {f!r}")
        if b < 1:
            raise ConfigError(f"bucket_slots must be >= 1, got {b}")
        if (b * f) % 64:
            raise ConfigError(f"bucket_slots * fingerprint_bits must be a multiple of 64, got {b} * {f}")
        if m < 1:
            raise ConfigError(f"bucket_count must be >= 1, got {m}")
        object.__setattr__(self, "policy", Policy(self.policy))
        object.__setattr__(self, "eviction", Eviction(self.eviction))
        if self.policy is Policy.XOR and not _is_pow2(m):
            raise ConfigError(f"xor policy requires a power-of-two bucket_count, got {m}")
        if self.policy is Policy.OFFSET and m < 2:
            raise ConfigError(f"offset policy requires bucket_count >= 2, got {m}")
        if self.max_evictions < 1:
            raise ConfigError(f"max_evictions must be >= 1, got {self.max_evictions}")
        if not 0 <= self.seed <= MASK64:
            raise ConfigError("seed must fit in 64 bits")

    # derived geometry
    @property
    def tags_per_word(self) -> int:
        return 64 // self.fingerprint_bits

    @property
    def words_per_bucket(self) -> int:
        return self.bucket_slots * self.fingerprint_bits // 64

    @property
    def total_slots(self) -> int:
        return self.bucket_count * self.bucket_slots

    @property
    def total_words(self) -> int:
        return self.bucket_count * self.words_per_bucket

    @property
    def payload_bits(self) -> int:
        return self.fingerprint_bits - 1 if self.policy is Policy.OFFSET else self.fingerprint_bits

    @property
    def choice_bit(self) -> int:
        return 1 << (self.fingerprint_bits - 1)

    @property
    def index_mask(self) -> int:
        return self.bucket_count - 1 if _is_pow2(self.bucket_count) else 0

    def ckf_params(self, worker: int = 0):
        """The ``ckf_params`` struct for the C ABI (validated again natively)."""
        from . import _lib

        if self.bucket_slots > MAX_GPU_BUCKET_SLOTS:
            raise ConfigError(
                f"bucket_slots > {MAX_GPU_BUCKET_SLOTS} is not supported by the GPU kernels"
            )
        p = _lib.make_params(
            self.bucket_count, self.fingerprint_bits, self.bucket_slots,
            _lib.POLICY_XOR if self.policy is Policy.XOR else _lib.POLICY_OFFSET,
            _lib.EVICT_DFS if self.eviction is Eviction.DFS else _lib.EVICT_BFS,
            self.max_evictions, self.seed,
        )
        p.worker = worker & MASK64
        return p


class Placement(NamedTuple):
    fp: int
    i1: int
    i2: int


def derive_placement(key: int, cfg: FilterConfig) -> Placement:
    """(fingerprint, primary bucket, alternate bucket) of a key,
    computed by the kernels' own semantics header compiled for the host."""
    from . import _lib

    p = cfg.ckf_params()
    fp, i1, i2 = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    _lib.lib().ckf_host_place(ctypes.byref(p), key & MASK64, ctypes.byref(fp), ctypes.byref(i1),
                              ctypes.byref(i2))
    return Placement(fp.value, i1.value, i2.value)


def alt_index(i: int, fp: int, choice: int, cfg: FilterConfig) -> tuple[int, int]:
    """Alternate bucket and flipped residency bit of a stored fingerprint."""
    from . import _lib

    p = cfg.ckf_params()
    nc = ctypes.c_uint64()
    r = _lib.lib().ckf_host_alt(ctypes.byref(p), i, fp, choice, ctypes.byref(nc))
    return int(r), int(nc.value)


def hash_key(key: int, seed: int = 0) -> int:
    """xxHash64 of the key's 8 little-endian bytes, host-compiled kernel code."""
    from . import _lib

    return int(_lib.lib().ckf_host_hash(key & MASK64, seed & MASK64))
