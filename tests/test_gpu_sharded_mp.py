"""The multi-rank sharded filter end to end on ONE GPU: two or four ranks
(processes) share cuda:0 and talk through the gloo backend (NCCL refuses two
ranks on one device), so the CUDA data path of ShardedCuckooFilter runs for
real -- fixed-capacity padded routing blocks, the receivers' padding skip,
the reverse exchange, ckf_route_unpermute, the spill round -- and every shard
is checked bit-exactly (parity mode) against a reference filter of m/G
buckets fed the keys routed to it in arrival order."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, slack, det, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_15486_b200 import CuckooFilter, FilterConfig
        from paper_2603_15486_b200.sharded import ShardedCuckooFilter

        torch.cuda.set_device(0)
        cfg = FilterConfig(bucket_count=(1 << 11) * world, eviction="bfs", seed=11)
        local_cfg = FilterConfig(bucket_count=1 << 11, eviction="bfs", seed=11)
        sf = ShardedCuckooFilter(cfg, device="cuda:0", local=CuckooFilter(local_cfg, device="cuda:0",
                                                                           deterministic=det))
        if slack is not None:
            sf.SLACK_SIGMAS = slack  # (a negative slack forces the spill round)
        rng = np.random.default_rng(50 + rank)
        n = int(0.85 * local_cfg.total_slots) - 97 * rank
        keys = rng.integers(0, 1 << 62, size=n, dtype=np.uint64)
        neg = rng.integers(1 << 62, 1 << 63, size=3 * n, dtype=np.uint64)
        kd = torch.from_numpy(keys.view(np.int64)).cuda()
        res = sf.insert_batch(kd)
        ev = res.evictions.cpu().numpy()
        qp = sf.query_batch(kd).cpu().numpy()
        qn = sf.query_batch(torch.from_numpy(neg.view(np.int64)).cuda()).cpu().numpy()
        dr = sf.delete_batch(kd[::2]).cpu().numpy()
        q.put((rank, keys, neg, res.ok.cpu().numpy(), res.n_ok_global, ev, qp, qn, dr, sf.occupancy,
               sf.local.words.copy(), sf.router.shift))
    finally:
        dist.destroy_process_group()


def _run(world, slack=None, det=True):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, slack, det, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get() for _ in range(world)]
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    return sorted(results, key=lambda r: r[0])


@pytest.mark.parametrize("world,slack", [(2, None), (4, None), (2, -40.0)], ids=["G2", "G4", "G2-spill"])
def test_padded_exchange_on_one_gpu_matches_per_shard_oracle(world, slack):
    from paper_2603_15486_b200 import FilterConfig
    from paper_2603_15486_b200.sharded import HashRouter

    results = _run(world, slack)
    local_cfg = FilterConfig(bucket_count=1 << 11, eviction="bfs", seed=11)
    router = HashRouter(local_cfg, world)
    ocfg = oracle.cfg_from(local_cfg)
    shards = [oracle.OracleFilter(ocfg) for _ in range(world)]

    def owner(keys):
        h = torch.from_numpy(oracle.hash_batch(keys, 11).view(np.int64))
        return router.shard_of(h).numpy()

    want = {r: {} for r in range(world)}

    def replay(field, arrays, op):
        outs = {r: np.zeros(len(arrays[r]), dtype=bool) for r in range(world)}
        sh = {r: owner(arrays[r]) for r in range(world)}
        for s in range(world):
            for r in range(world):  # arrival order: source rank, then position
                sel = np.nonzero(sh[r] == s)[0]
                outs[r][sel] = op(shards[s], arrays[r][sel])
        for r in range(world):
            want[r][field] = outs[r]

    replay("ok", {r: results[r][1] for r in range(world)}, lambda f, k: f.insert_batch(k)[0])
    replay("qp", {r: results[r][1] for r in range(world)}, lambda f, k: f.query_batch(k))
    replay("qn", {r: results[r][2] for r in range(world)}, lambda f, k: f.query_batch(k))
    replay("dr", {r: results[r][1][::2] for r in range(world)}, lambda f, k: f.delete_batch(k))
    total = sum(int(r[3].sum()) for r in results)
    for (rank, keys, neg, ok, n_ok_g, ev, qp, qn, dr, occ, words, shift) in results:
        assert shift == router.shift
        assert np.array_equal(ok, want[rank]["ok"])
        assert n_ok_g == total
        assert ev.shape == ok.shape and (ev >= 0).all()
        assert np.array_equal(qp, want[rank]["qp"]) and qp.all()
        assert np.array_equal(qn, want[rank]["qn"])
        assert np.array_equal(dr, want[rank]["dr"])
        if slack is None:  # (a spill round inserts its keys after the padded round's)
            assert np.array_equal(words, shards[rank].words), f"shard {rank} table differs"
        assert occ == sum(s.occupancy for s in shards)


def test_concurrent_shards_on_one_gpu_semantics():
    """The production (concurrent) local schedule behind the exchange: no
    false negatives, occupancy equal to the keys stored."""
    results = _run(2, None, det=False)
    total = sum(int(r[3].sum()) for r in results)
    for (rank, keys, neg, ok, n_ok_g, ev, qp, qn, dr, occ, words, shift) in results:
        assert ok.all() and n_ok_g == total
        assert qp.all()
        assert dr.all()
