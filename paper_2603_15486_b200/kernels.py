"""Thin tensor wrappers over the C ABI for the stateless batch kernels.

Counterparts of the reference ``_kernels.hash_batch`` (K:489-493) and
``_kernels.place_batch`` (K:496-507): device tensors in, device tensors out,
enqueued on the current CUDA stream.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .config import FilterConfig


def _dev_keys(keys: torch.Tensor) -> torch.Tensor:
    if not isinstance(keys, torch.Tensor) or keys.device.type != "cuda" or keys.dim() != 1:
        raise ValueError("keys must be a 1-D CUDA tensor (int64 or uint64)")
    if keys.dtype == torch.uint64:
        keys = keys.view(torch.int64)
    if keys.dtype != torch.int64:
        raise ValueError("keys must be int64 or uint64")
    return keys.contiguous()


def hash_batch(keys: torch.Tensor, seed: int = 0) -> torch.Tensor:
    """xxh64(key, seed) per key, as int64 (bit pattern of the uint64 hash)."""
    k = _dev_keys(keys)
    out = torch.empty_like(k)
    _lib.check(_lib.lib().ckf_hash(k.data_ptr(), k.numel(), seed, out.data_ptr(),
                                   torch.cuda.current_stream(k.device).cuda_stream))
    return out


def place_batch(cfg: FilterConfig, keys: torch.Tensor, hashed: bool = False):
    """(fp, i1, i2) per key as int64 tensors; ``hashed`` = keys hold xxh64 values."""
    k = _dev_keys(keys)
    fp, i1, i2 = (torch.empty_like(k) for _ in range(3))
    p = cfg.ckf_params()
    _lib.check(_lib.lib().ckf_place(ctypes.byref(p), k.data_ptr(), k.numel(), fp.data_ptr(),
                                    i1.data_ptr(), i2.data_ptr(), _lib.INPUT_HASHED if hashed else 0,
                                    torch.cuda.current_stream(k.device).cuda_stream))
    return fp, i1, i2
