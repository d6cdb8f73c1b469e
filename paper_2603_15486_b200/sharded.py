"""Hash-sharded cuckoo filter over the GPUs of one node.

The table is split into G independent sub-filters of m/G buckets, one per
rank.  A key is owned by the shard named by hash bits that neither the
fingerprint (bits 32..) nor the shard-local primary index (low bits,
P:230) consume, so shard s behaves exactly like a reference
``CuckooFilter(FilterConfig(bucket_count=m/G, ...))`` fed the keys routed to it,
in arrival order.

Per batch, on every rank (one process per GPU, NCCL over NVLink/NVSwitch),
with no host synchronisation on the GPU data path:
  1. hash the local keys (ckf_hash kernel);
  2. stable grouping by owner into FIXED-CAPACITY blocks, one per shard
     (ckf_route_partition_padded: count / scan / scatter / pad kernels); a
     block's unused tail holds hashes owned by another shard, which the
     receiver's kernels skip (ckf_params_set_shard);
  3. one all-to-all of the 8-byte hash blocks -- split sizes come from the
     batch sizes, exchanged on a host-side gloo group, never from device
     counts;
  4. the owning rank runs the local schedule on the received blocks
     (CKF_INPUT_HASHED: no rehash; padding skipped);
  5. reverse all-to-all of the 1-byte results;
  6. inverse permutation back to the caller's order (ckf_route_unpermute).
A block holds n/G + 6 sqrt(n/G) + 256 hashes; a key past its block's
capacity (adversarial skew only) is answered by a second, exact-split round
that every rank joins when any rank spilled.  Occupancy is an all-reduce of
per-shard counters.

The class only needs ``torch.distributed`` and a local filter with the
``CuckooFilter`` batch API, so the routing logic is tested on CPU with the
gloo backend (tests/test_sharded_gloo.py) and runs on B200s with NCCL.
"""

from __future__ import annotations

import ctypes
import dataclasses
import math
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
    """Per-key ``ok`` in the caller's order; ``n_ok`` is global over all ranks.

    ``evictions`` / ``lost_fingerprints`` (filter.py:95-112) are routed back
    on first access -- a collective: every rank must read them together."""

    def __init__(self, ok: torch.Tensor, n_ok_global: torch.Tensor, n: int, back=None, n_alt=None):
        self.ok = ok
        self._n_ok = n_ok_global
        self._n = n
        self._n_alt = n_alt  # () -> global count of keys that probed their alternate bucket
        self._back = back  # () -> (evictions, lost) in caller order, or None
        self._ev = self._lost = None

    def _expand(self):
        if self._back is None:
            z = torch.zeros(self._n, dtype=torch.int64, device=self.ok.device)
            self._ev, self._lost = z, z.clone()
        else:
            self._ev, self._lost = self._back()

    @property
    def evictions(self) -> torch.Tensor:
        if self._ev is None:
            self._expand()
        return self._ev

    @property
    def lost_fingerprints(self) -> torch.Tensor:
        if self._lost is None:
            self._expand()
        return self._lost

    @property
    def n_ok_global(self) -> int:
        return int(self._n_ok.item())

    @property
    def n_alt(self) -> int:
        """Keys (all ranks) whose primary bucket was full; a collective."""
        return self._n_alt() if self._n_alt is not None else 0

    @property
    def n_ok(self) -> int:
        """This rank's keys that were stored."""
        return int(self.ok.sum().item())

    @property
    def n_failed(self) -> int:
        return self._n - self.n_ok


class _Route:
    """What the return path of one routed batch needs."""

    def __init__(self, **kw):
        self.__dict__.update(kw)


class ShardedCuckooFilter:
    """``CuckooFilter`` API over G hash shards, one per rank of ``group``.

    ``cfg.bucket_count`` is the GLOBAL bucket count (divisible by G); each rank
    holds ``cfg.bucket_count // G`` buckets.  ``local`` / ``hasher`` default to
    the CUDA filter and hash kernel; tests substitute CPU stand-ins (which take
    the exact-split path).
    """

    SLACK_SIGMAS = 6.0  # block capacity: n/G + SLACK_SIGMAS * sqrt(n/G) + 256

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

            if self.world > 8:
                raise ConfigError(f"the CUDA router handles up to 8 shards per node, got {self.world}")
            local = CuckooFilter(self.local_cfg, device=device)
        self.local = local
        self.device = torch.device(device) if device is not None else getattr(local, "device", torch.device("cpu"))
        params = getattr(local, "_params", None)
        if params is not None and self.world > 1:  # skip the padding of the fixed-size exchange
            from . import _lib

            _lib.check(_lib.lib().ckf_params_set_shard(ctypes.byref(params), self.router.shift, self.world,
                                                       self.rank))
        if hasher is None:
            from .kernels import hash_batch

            seed = cfg.seed
            hasher = lambda k: hash_batch(k, seed)  # noqa: E731
        self._hash = hasher
        self._meta = None  # host-side gloo group for batch sizes / spill flags

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

    def _meta_group(self):
        if self._meta is None:
            backend = dist.get_backend(self.group)
            self._meta = self.group if backend == "gloo" else dist.new_group(
                ranks=dist.get_process_group_ranks(self.group) if self.group is not None else None, backend="gloo")
        return self._meta

    def _host_allgather(self, v: int) -> list:
        t = torch.tensor([v], dtype=torch.int64)
        out = [torch.zeros(1, dtype=torch.int64) for _ in range(self.world)]
        dist.all_gather(out, t, group=self._meta_group())
        return [int(x) for x in out]

    def block_capacity(self, n: int) -> int:
        per = n / self.world
        cap = int(per + self.SLACK_SIGMAS * math.sqrt(per) + 256)
        return (cap + 255) // 256 * 256

    def _scatter(self, keys):
        """Steps 1-3: hash, group by owner, exchange.  Returns the hashes this
        rank owns (padded blocks on the CUDA path) and the return-path state."""
        k = self._keys(keys)
        h = self._hash(k)
        if self.world == 1:
            return h, None
        if h.is_cuda:
            return self._scatter_padded(k, h)
        return self._scatter_exact(h)

    def _scatter_exact(self, h):
        """Exact split sizes (CPU stand-ins of the gloo tests, and the spill
        round): stable sort by shard, counts exchanged, then the payload."""
        if h.is_cuda:
            send, order, send_counts = self._partition_cuda(h)
        else:
            shard = self.router.shard_of(h).to(torch.uint8)
            order = torch.argsort(shard, stable=True)
            send = h[order]
            send_counts = torch.bincount(shard, minlength=self.world)
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        sc, rc = send_counts.tolist(), recv_counts.tolist()
        recv = torch.empty(sum(rc), dtype=h.dtype, device=h.device)
        dist.all_to_all_single(recv, send, rc, sc, group=self.group)
        return recv, _Route(kind="exact", order=order, sc=sc, rc=rc, n=h.numel())

    def _scatter_padded(self, k, h):
        from . import _lib

        L = _lib.lib()
        n = h.numel()
        caps = [self.block_capacity(x) for x in self._host_allgather(n)]
        cap = caps[self.rank]
        G = self.world
        send = torch.empty(G * cap, dtype=torch.int64, device=h.device)
        order = torch.empty(G * cap, dtype=torch.int64, device=h.device)
        counts = torch.empty(G, dtype=torch.int64, device=h.device)
        spilled = torch.empty(1, dtype=torch.int64, device=h.device)
        wsb = int(L.ckf_route_workspace_bytes(max(n, 1), G))
        if getattr(self, "_route_ws", None) is None or self._route_ws.numel() < wsb:
            self._route_ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=h.device)
        stream = torch.cuda.current_stream(h.device)
        _lib.check(L.ckf_route_partition_padded(h.data_ptr(), n, self.router.shift, G, cap, send.data_ptr(),
                                                order.data_ptr(), counts.data_ptr(), spilled.data_ptr(),
                                                self._route_ws.data_ptr(), wsb, stream.cuda_stream))
        spill_host = torch.empty(1, dtype=torch.int64, pin_memory=True)
        spill_host.copy_(spilled, non_blocking=True)
        routed = torch.cuda.Event()
        routed.record(stream)
        recv = torch.empty(sum(caps), dtype=torch.int64, device=h.device)
        dist.all_to_all_single(recv, send, caps, [cap] * G, group=self.group)
        return recv, _Route(kind="padded", order=order, caps=caps, cap=cap, n=n, keys=k,
                            spill_host=spill_host, routed=routed)

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

    def _back(self, local: torch.Tensor, route, fill=0) -> torch.Tensor:
        """Steps 5-6 for one per-key array (1- or 8-byte elements): answers back
        to their source rank, then to the caller's order."""
        if route is None:
            return local
        if route.kind == "exact":
            back = torch.empty(sum(route.sc), dtype=local.dtype, device=local.device)
            dist.all_to_all_single(back, local.contiguous(), route.sc, route.rc, group=self.group)
            out = torch.empty_like(back)
            if out.is_cuda:
                self._unpermute(back, route.order, out)
            else:
                out[route.order] = back
            return out
        G, cap = self.world, route.cap
        back = torch.empty(G * cap, dtype=local.dtype, device=local.device)
        dist.all_to_all_single(back, local.contiguous(), [cap] * G, route.caps, group=self.group)
        out = torch.full((route.n,), fill, dtype=local.dtype, device=local.device)
        self._unpermute(back, route.order, out)
        return out

    @staticmethod
    def _unpermute(back: torch.Tensor, order: torch.Tensor, out: torch.Tensor) -> None:
        from . import _lib

        _lib.check(_lib.lib().ckf_route_unpermute(back.data_ptr(), order.data_ptr(), back.numel(),
                                                  back.element_size(), out.data_ptr(),
                                                  torch.cuda.current_stream(back.device).cuda_stream))

    def _spill_round(self, route, out: torch.Tensor, op: str) -> None:
        """Keys past their block's capacity (adversarial skew): if any rank
        spilled, every rank runs an exact-split round over its unanswered keys."""
        if route is None or route.kind != "padded":
            return None
        route.routed.synchronize()  # the routing kernels only (the exchange is in flight)
        if sum(self._host_allgather(int(route.spill_host.item()))) == 0:
            return None
        idx = torch.nonzero(out == 0xFF).flatten()
        recv, r2 = self._scatter_exact(self._hash(route.keys[idx]))
        res = getattr(self.local, op)(recv, hashed=True)
        ans = torch.as_tensor(res.ok if op == "insert_batch" else res).to(self.device)
        out[idx] = self._back(ans.to(torch.uint8), r2)
        return ans

    # ---- batch API ----

    def _run(self, keys, op: str):
        recv, route = self._scatter(keys)
        res = getattr(self.local, op)(recv, hashed=True)
        local_ok = res.ok if op == "insert_batch" else res
        local_ok = torch.as_tensor(local_ok).to(self.device)
        out = self._back(local_ok.to(torch.uint8), route, fill=0xFF)
        spill = self._spill_round(route, out, op)
        return out.view(torch.bool) if out.dtype == torch.uint8 else out, res, route, local_ok, spill

    def insert_batch(self, keys, workers: int = 1) -> ShardedInsertResult:
        ok, res, route, local_ok, spill = self._run(keys, "insert_batch")
        ctr = getattr(res, "_ctr", None)  # the local kernels' counters: real inserts only, no padding
        n_ok = ctr[0:1].clone() if ctr is not None else local_ok.to(torch.int64).sum().reshape(1)
        if spill is not None:
            n_ok += spill.to(torch.int64).sum()
        if self.world > 1:
            dist.all_reduce(n_ok, group=self.group)

        def back():
            ev = torch.as_tensor(res.evictions).to(self.device).to(torch.int64)
            lost = torch.as_tensor(res.lost_fingerprints).to(self.device).view(torch.int64)
            return self._back(ev, route), self._back(lost, route)

        def n_alt():
            t = (ctr[3:4].clone() if ctr is not None else torch.zeros(1, dtype=torch.int64, device=self.device))
            if self.world > 1:
                dist.all_reduce(t, group=self.group)
            return int(t.item())

        return ShardedInsertResult(ok, n_ok, ok.numel(), back if hasattr(res, "evictions") else None, n_alt)

    def query_batch(self, keys, workers: int = 1) -> torch.Tensor:
        return self._run(keys, "query_batch")[0]

    def delete_batch(self, keys, workers: int = 1) -> torch.Tensor:
        return self._run(keys, "delete_batch")[0]

    # ---- scalar API (one-key batches; collective like the batch calls) ----

    def insert(self, key: int) -> bool:
        return bool(self.insert_batch([key]).ok[0])

    def query(self, key: int) -> bool:
        return bool(self.query_batch([key])[0])

    def delete(self, key: int) -> bool:
        return bool(self.delete_batch([key])[0])

    def __contains__(self, key: int) -> bool:
        return self.query(key)

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

    def stored_tags(self):
        """This shard's (m/G, b) lane snapshot (shard s owns global buckets
        [s*m/G, (s+1)*m/G) of the equivalent unsharded layout)."""
        return self.local.stored_tags()
