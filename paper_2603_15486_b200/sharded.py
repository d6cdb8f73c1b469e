"""Hash-sharded cuckoo filter over the GPUs of one node.

The table is split into G independent sub-filters of m/G buckets, one per
rank.  A key is owned by the shard named by hash bits that neither the
fingerprint (bits 32..) nor the shard-local primary index (low bits,
P:230) consume, so shard s behaves exactly like a reference
``CuckooFilter(FilterConfig(bucket_count=m/G, ...))`` fed the keys routed to it,
in arrival order.

Per batch, on every rank (one process per GPU, NCCL over NVLink/NVSwitch):
  1. hash the local keys (ckf_hash kernel);
  2. shard id per hash, stable permutation by shard, per-shard counts
     (ckf_route_partition: count / scan / scatter kernels);
  3. all-to-all of the counts, then of the 8-byte hashes;
  4. the owning rank runs the local kernel on hashes (CKF_INPUT_HASHED:
     no rehash);
  5. reverse all-to-all of the 1-byte results;
  6. inverse permutation back to the caller's order.
There is one exchange step per direction and no other collective on the
data path; occupancy is an all-reduce of per-shard counters.

The class only needs ``torch.distributed`` and a local filter with the
``CuckooFilter`` batch API, so the routing logic is tested on CPU with the
gloo backend (tests/test_sharded_gloo.py) and runs on B200s with NCCL.
"""

from __future__ import annotations

import dataclasses
from typing import Callable, Optional

import torch
import torch.distributed as dist

from .config import FilterConfig
from .errors import ConfigError


class HashRouter:
    """Maps a 64-bit key hash to its owning shard (SURVEY.md §8(e) bit budget)."""

    def __init__(self, local_cfg: FilterConfig, world: int):
        if world < 1 or world & (world - 1):
            raise ConfigError(f"shard count must be a power of two, got {world}")
        self.world = world
        g = world.bit_length() - 1
        self.bits = g
        free_top = 32 - local_cfg.payload_bits  # hash bits above the fingerprint
        if g == 0:
            self.shift = 0
        elif g <= free_top:
            self.shift = 64 - g  # top bits: untouched by fp and by i1
        elif local_cfg.index_mask and (local_cfg.bucket_count.bit_length() - 1) + g <= 32:
            self.shift = 32 - g  # just below the fingerprint, above the i1 mask
        else:
            raise ConfigError(
                f"no hash bits left to shard f={local_cfg.fingerprint_bits} "
                f"{local_cfg.policy.value} over {world} ranks; use replicas"
            )

    def shard_of(self, h: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            return torch.zeros_like(h)
        # arithmetic >> on int64 is fine: the mask keeps only the g routed bits
        return torch.bitwise_and(h >> self.shift, self.world - 1)


class ShardedInsertResult:
    """Per-key ``ok`` in the caller's order; ``n_ok`` is global over all ranks."""

    def __init__(self, ok: torch.Tensor, n_ok_global: torch.Tensor, n: int):
        self.ok = ok
        self._n_ok = n_ok_global
        self._n = n

    @property
    def n_ok_global(self) -> int:
        return int(self._n_ok.item())

    @property
    def n_ok(self) -> int:
        """This rank's keys that were stored."""
        return int(self.ok.sum().item())

    @property
    def n_failed(self) -> int:
        return self._n - self.n_ok


class ShardedCuckooFilter:
    """``CuckooFilter`` API over G hash shards, one per rank of ``group``.

    ``cfg.bucket_count`` is the GLOBAL bucket count (divisible by G); each rank
    holds ``cfg.bucket_count // G`` buckets.  ``local`` / ``hasher`` default to
    the CUDA filter and hash kernel; tests substitute CPU stand-ins.
    """

    def __init__(self, cfg: FilterConfig, *, group=None, device=None, local=None,
                 hasher: Optional[Callable[[torch.Tensor], torch.Tensor]] = None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if cfg.bucket_count % self.world:
            raise ConfigError(f"bucket_count {cfg.bucket_count} not divisible by {self.world} shards")
        self.cfg = cfg
        self.local_cfg = dataclasses.replace(cfg, bucket_count=cfg.bucket_count // self.world)
        self.router = HashRouter(self.local_cfg, self.world)
        if local is None:
            from .filter import CuckooFilter

            local = CuckooFilter(self.local_cfg, device=device)
        self.local = local
        self.device = torch.device(device) if device is not None else getattr(local, "device", torch.device("cpu"))
        if hasher is None:
            from .kernels import hash_batch

            seed = cfg.seed
            hasher = lambda k: hash_batch(k, seed)  # noqa: E731
        self._hash = hasher

    # ---- routing ----

    def _keys(self, keys) -> torch.Tensor:
        if not isinstance(keys, torch.Tensor):
            import numpy as np

            keys = torch.from_numpy(np.ascontiguousarray(keys, dtype=np.uint64).view(np.int64))
        if keys.dim() != 1:
            raise ValueError("keys must be one-dimensional")
        if keys.dtype == torch.uint64:
            keys = keys.view(torch.int64)
        return keys.to(self.device).contiguous()

    def _scatter(self, keys):
        """Steps 1-3: hash, group by owner, exchange.  Returns the hashes this
        rank owns plus what is needed to send the answers back."""
        h = self._hash(self._keys(keys))
        if self.world == 1:
            return h, None, None, None
        if h.is_cuda:
            send, order, send_counts = self._partition_cuda(h)
        else:  # CPU stand-ins of the gloo tests
            shard = self.router.shard_of(h).to(torch.uint8)
            order = torch.argsort(shard, stable=True)
            send = h[order]
            send_counts = torch.bincount(shard, minlength=self.world)
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        sc, rc = send_counts.tolist(), recv_counts.tolist()
        recv = torch.empty(sum(rc), dtype=h.dtype, device=h.device)
        dist.all_to_all_single(recv, send, rc, sc, group=self.group)
        return recv, order, sc, rc

    def _partition_cuda(self, h: torch.Tensor):
        """Stable partition by shard on the device (ckf_route_partition: count,
        scan, scatter -- a torch stable argsort of 2^28 ids takes ~24 ms)."""
        from . import _lib

        L = _lib.lib()
        n = h.numel()
        send = torch.empty_like(h)
        order = torch.empty(n, dtype=torch.int64, device=h.device)
        counts = torch.empty(self.world, dtype=torch.int64, device=h.device)
        wsb = int(L.ckf_route_workspace_bytes(n, self.world))
        if getattr(self, "_route_ws", None) is None or self._route_ws.numel() < wsb:
            self._route_ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=h.device)
        _lib.check(L.ckf_route_partition(h.data_ptr(), n, self.router.shift, self.world, send.data_ptr(),
                                         order.data_ptr(), counts.data_ptr(), self._route_ws.data_ptr(), wsb,
                                         torch.cuda.current_stream(h.device).cuda_stream))
        return send, order, counts

    def _gather(self, local_res: torch.Tensor, order, sc, rc) -> torch.Tensor:
        """Steps 5-6: answers back to their source rank, then to caller order."""
        if order is None:
            return local_res
        res = local_res.to(torch.uint8)
        back = torch.empty(sum(sc), dtype=torch.uint8, device=res.device)
        dist.all_to_all_single(back, res.contiguous(), sc, rc, group=self.group)
        out = torch.empty_like(back)
        out[order] = back
        return out.view(torch.bool)

    # ---- batch API ----

    def insert_batch(self, keys, workers: int = 1) -> ShardedInsertResult:
        recv, order, sc, rc = self._scatter(keys)
        res = self.local.insert_batch(recv, hashed=True)
        ok_local = res.ok if isinstance(res.ok, torch.Tensor) else torch.as_tensor(res.ok)
        ok = self._gather(ok_local.to(self.device), order, sc, rc)
        n_ok = ok_local.to(torch.int64).sum().reshape(1)
        if self.world > 1:
            dist.all_reduce(n_ok, group=self.group)
        return ShardedInsertResult(ok, n_ok, ok.numel())

    def query_batch(self, keys, workers: int = 1) -> torch.Tensor:
        recv, order, sc, rc = self._scatter(keys)
        return self._gather(self.local.query_batch(recv, hashed=True), order, sc, rc)

    def delete_batch(self, keys, workers: int = 1) -> torch.Tensor:
        recv, order, sc, rc = self._scatter(keys)
        return self._gather(self.local.delete_batch(recv, hashed=True), order, sc, rc)

    def last_counters(self) -> dict:
        c = self.local.last_counters() if hasattr(self.local, "last_counters") else {"n_ok": 0, "n_alt": 0}
        t = torch.tensor([c["n_ok"], c["n_alt"]], dtype=torch.int64, device=self.device)
        if self.world > 1:
            dist.all_reduce(t, group=self.group)
        return {"n_ok": int(t[0]), "n_alt": int(t[1])}

    # ---- bookkeeping ----

    @property
    def occupancy(self) -> int:
        t = torch.tensor([len(self.local)], dtype=torch.int64, device=self.device)
        if self.world > 1:
            dist.all_reduce(t, group=self.group)
        return int(t.item())

    def __len__(self) -> int:
        return self.occupancy

    @property
    def load_factor(self) -> float:
        return self.occupancy / self.cfg.total_slots

    def clear(self) -> None:
        self.local.clear()
