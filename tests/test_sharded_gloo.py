"""Multi-rank routing of the hash-sharded filter, on CPU with gloo (world 2 and 4).

The local sub-filters are the CPU oracle and the hash is the oracle's, so this
checks the distributed plumbing itself -- shard selection, stable grouping,
count + payload all-to-all, reverse all-to-all, inverse permutation --
against SURVEY.md §8(e)'s parity rule: shard s must behave exactly like a
reference filter of m/G buckets fed the keys routed to it in arrival order.
"""

from __future__ import annotations

import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2603_15486_b200 import ConfigError, FilterConfig
from paper_2603_15486_b200.sharded import HashRouter, ShardedCuckooFilter


class OracleLocal:
    """CPU stand-in for the per-rank CUDA filter (same batch API, hashed input)."""

    def __init__(self, cfg):
        self.f = oracle.OracleFilter(oracle.cfg_from(cfg))
        self.device = torch.device("cpu")

    @staticmethod
    def _u64(h: torch.Tensor) -> np.ndarray:
        return h.numpy().view(np.uint64)

    def insert_batch(self, h, hashed=True):
        ok, _, _ = self.f.insert_batch(self._u64(h), hashed=hashed)
        return SimpleNamespace(ok=torch.from_numpy(ok.copy()))

    def query_batch(self, h, hashed=True):
        return torch.from_numpy(self.f.query_batch(self._u64(h), hashed=hashed).copy())

    def delete_batch(self, h, hashed=True):
        return torch.from_numpy(self.f.delete_batch(self._u64(h), hashed=hashed).copy())

    def __len__(self):
        return self.f.occupancy

    def clear(self):
        self.f.clear()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank: int, world: int, port: int, f: int, policy: str, q) -> None:
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m_local = 1 << 9 if policy == "xor" else 300
        cfg = FilterConfig(bucket_count=m_local * world, fingerprint_bits=f, bucket_slots=16,
                           policy=policy, eviction="bfs", seed=5)
        seed = cfg.seed
        hasher = lambda k: torch.from_numpy(oracle.hash_batch(k.numpy().view(np.uint64), seed).view(np.int64))  # noqa: E731
        local_cfg = FilterConfig(bucket_count=m_local, fingerprint_bits=f, bucket_slots=16,
                                 policy=policy, eviction="bfs", seed=seed)
        sf = ShardedCuckooFilter(cfg, local=OracleLocal(local_cfg), hasher=hasher)
        rng = np.random.default_rng(100 + rank)
        n = int(0.85 * local_cfg.total_slots)
        keys = rng.integers(0, 1 << 32, size=n, dtype=np.uint64)
        neg = rng.integers(1 << 32, 1 << 63, size=4 * n, dtype=np.uint64)
        res = sf.insert_batch(keys)
        qp = sf.query_batch(keys).numpy()
        qn = sf.query_batch(neg).numpy()
        dk = keys[::2]
        dr = sf.delete_batch(dk).numpy()
        occ = sf.occupancy
        q.put((rank, keys, neg, res.ok.numpy(), int(res.n_ok_global), qp, qn, dr, occ, sf.local.f.words.copy()))
    finally:
        dist.destroy_process_group()


def _expected(results, world, f, policy):
    """Replay every shard with the oracle in arrival order (source rank order)."""
    m_local = 1 << 9 if policy == "xor" else 300
    local_cfg = FilterConfig(bucket_count=m_local, fingerprint_bits=f, bucket_slots=16,
                             policy=policy, eviction="bfs", seed=5)
    router = HashRouter(local_cfg, world)

    def shard(keys):
        h = torch.from_numpy(oracle.hash_batch(keys, 5).view(np.int64))
        return router.shard_of(h).numpy()

    shards = [oracle.OracleFilter(oracle.cfg_from(local_cfg)) for _ in range(world)]
    by_rank = {r[0]: r for r in results}
    want = {r: {} for r in range(world)}

    def run(op, field, arrays):
        outs = {r: np.zeros(len(arrays[r]), dtype=bool) for r in range(world)}
        sh = {r: shard(arrays[r]) for r in range(world)}
        for s in range(world):
            for r in range(world):
                sel = np.nonzero(sh[r] == s)[0]
                got = op(shards[s], arrays[r][sel])
                outs[r][sel] = got
        for r in range(world):
            want[r][field] = outs[r]

    run(lambda fl, k: fl.insert_batch(k)[0], "ok", {r: by_rank[r][1] for r in range(world)})
    run(lambda fl, k: fl.query_batch(k), "qp", {r: by_rank[r][1] for r in range(world)})
    run(lambda fl, k: fl.query_batch(k), "qn", {r: by_rank[r][2] for r in range(world)})
    run(lambda fl, k: fl.delete_batch(k), "dr", {r: by_rank[r][1][::2] for r in range(world)})
    return want, shards


@pytest.mark.parametrize("world,f,policy", [(2, 16, "xor"), (4, 16, "xor"), (2, 8, "offset"), (2, 32, "xor")])
def test_sharded_routing_matches_per_shard_oracle(world, f, policy):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, f, policy, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get() for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    want, shards = _expected(results, world, f, policy)
    total_ok = 0
    for (rank, keys, neg, ok, n_ok_g, qp, qn, dr, occ, words) in results:
        assert np.array_equal(ok, want[rank]["ok"]), "insert outcomes differ from the per-shard oracle"
        assert np.array_equal(qp, want[rank]["qp"]) and qp.all()
        assert np.array_equal(qn, want[rank]["qn"])
        assert np.array_equal(dr, want[rank]["dr"])
        assert np.array_equal(words, shards[rank].words), "shard table differs bit-wise"
        assert occ == sum(s.occupancy for s in shards)
        total_ok += int(ok.sum())
    assert all(r[4] == total_ok for r in results)


def test_router_bit_budget():
    cfg16 = FilterConfig(bucket_count=1 << 20)
    r = HashRouter(cfg16, 8)
    assert r.shift == 61
    h = torch.tensor([-1, 0, 1 << 61, (1 << 62) + 5], dtype=torch.int64)
    assert r.shard_of(h).tolist() == [7, 0, 1, 2]
    cfg32 = FilterConfig(bucket_count=1 << 20, fingerprint_bits=32, bucket_slots=4)
    r32 = HashRouter(cfg32, 8)
    assert r32.shift == 29  # below the fingerprint, above the 20-bit i1 mask
    with pytest.raises(ConfigError):
        HashRouter(FilterConfig(bucket_count=1 << 30, fingerprint_bits=32, bucket_slots=4), 8)
    with pytest.raises(ConfigError):
        HashRouter(cfg16, 3)
    off32 = FilterConfig(bucket_count=3000, fingerprint_bits=32, bucket_slots=4, policy="offset")
    assert HashRouter(off32, 2).shift == 63
    with pytest.raises(ConfigError):
        HashRouter(off32, 4)
