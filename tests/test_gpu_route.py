"""ckf_route_partition (multi-GPU routing step) against a stable argsort."""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np
import pytest
import torch

from paper_2603_15486_b200 import _lib

pytestmark = pytest.mark.gpu


def route(h: torch.Tensor, shift: int, shards: int):
    L = _lib.lib()
    n = h.numel()
    send = torch.empty_like(h)
    order = torch.empty(n, dtype=torch.int64, device=h.device)
    counts = torch.empty(shards, dtype=torch.int64, device=h.device)
    wsb = int(L.ckf_route_workspace_bytes(n, shards))
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=h.device)
    _lib.check(L.ckf_route_partition(h.data_ptr(), n, shift, shards, send.data_ptr(), order.data_ptr(),
                                     counts.data_ptr(), ws.data_ptr(), wsb, torch.cuda.current_stream().cuda_stream))
    return send, order, counts


@pytest.mark.parametrize("shards", [1, 2, 4, 8])
@pytest.mark.parametrize("n", [0, 1, 4095, 4096, 4097, 1_000_003])
@pytest.mark.parametrize("shift", [61, 29])
def test_route_partition_is_a_stable_argsort(shards, n, shift):
    g = torch.Generator(device="cuda")
    g.manual_seed(n + shards)
    h = torch.randint(-(1 << 62), 1 << 62, (n,), device="cuda", dtype=torch.int64, generator=g)
    send, order, counts = route(h, shift, shards)
    sid = torch.bitwise_and(h >> shift, shards - 1)
    want_order = torch.argsort(sid, stable=True)
    assert torch.equal(order, want_order)
    assert torch.equal(send, h[want_order])
    assert torch.equal(counts, torch.bincount(sid, minlength=shards))


@pytest.mark.parametrize("G", [2, 4, 8])
def test_padded_exchange_simulated_on_one_gpu(G):
    """The fixed-capacity exchange of ShardedCuckooFilter, every rank played on
    one GPU: source r groups its hashes into G blocks of block_capacity(n_r)
    (ckf_route_partition_padded), shard s receives block s of every source in
    rank order, and its filter -- marked with ckf_params_set_shard -- skips the
    padding.  In parity mode each shard's table must equal the oracle fed the
    shard's real keys in arrival order, bit for bit; the answers routed back
    with ckf_route_unpermute must equal the per-shard oracle's."""
    import ctypes

    import oracle
    from paper_2603_15486_b200 import CuckooFilter, FilterConfig, _lib
    from paper_2603_15486_b200.kernels import hash_batch
    from paper_2603_15486_b200.sharded import HashRouter, ShardedCuckooFilter

    L = _lib.lib()
    local = FilterConfig(bucket_count=1 << 10, eviction="bfs", seed=13)
    router = HashRouter(local, G)
    rng = np.random.default_rng(G)
    ns = [int(0.85 * local.total_slots) + 37 * r for r in range(G)]
    keys = [rng.integers(0, 1 << 62, size=n, dtype=np.uint64) for n in ns]
    cap_of = lambda n: ShardedCuckooFilter.block_capacity(SimpleNamespace(world=G, SLACK_SIGMAS=6.0), n)  # noqa: E731
    routed = []
    for r in range(G):
        h = hash_batch(torch.from_numpy(keys[r].view(np.int64)).cuda(), local.seed)
        cap = cap_of(ns[r])
        send = torch.empty(G * cap, dtype=torch.int64, device="cuda")
        order = torch.empty(G * cap, dtype=torch.int64, device="cuda")
        counts = torch.empty(G, dtype=torch.int64, device="cuda")
        spilled = torch.empty(1, dtype=torch.int64, device="cuda")
        wsb = int(L.ckf_route_workspace_bytes(ns[r], G))
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        _lib.check(L.ckf_route_partition_padded(h.data_ptr(), ns[r], router.shift, G, cap, send.data_ptr(),
                                                order.data_ptr(), counts.data_ptr(), spilled.data_ptr(),
                                                ws.data_ptr(), wsb, 0))
        assert int(spilled) == 0
        assert np.array_equal(counts.cpu().numpy(), np.bincount(router.shard_of(h).cpu().numpy(), minlength=G))
        routed.append((cap, send, order))
    answers = [torch.full((n,), 0xFF, dtype=torch.uint8, device="cuda") for n in ns]
    for s in range(G):
        recv = torch.cat([send[s * cap:(s + 1) * cap] for cap, send, _ in routed])
        filt = CuckooFilter(local, deterministic=True)
        _lib.check(L.ckf_params_set_shard(ctypes.byref(filt._params), router.shift, G, s))
        res = filt.insert_batch(recv, hashed=True)
        mine = np.concatenate([keys[r][router.shard_of(hash_batch(torch.from_numpy(keys[r].view(np.int64)).cuda(),
                                                                    local.seed)).cpu().numpy() == s]
                               for r in range(G)])
        ref = oracle.OracleFilter(oracle.cfg_from(local))
        rok, _, _ = ref.insert_batch(mine)
        assert np.array_equal(filt.words, ref.words), f"shard {s}: padding was not skipped"
        assert len(filt) == int(rok.sum())
        # concurrent lookups of the received blocks, routed back to each source
        q = CuckooFilter(local)
        _lib.check(L.ckf_params_set_shard(ctypes.byref(q._params), router.shift, G, s))
        q.words_device.copy_(filt.words_device)
        hits = q.query_batch(recv, hashed=True).to(torch.uint8)
        off = 0
        for r, (cap, _, order) in enumerate(routed):
            block = hits[off:off + cap]
            off += cap
            back = torch.zeros(G * cap, dtype=torch.uint8, device="cuda")
            back[s * cap:(s + 1) * cap] = block
            part = torch.full((G * cap,), -1, dtype=torch.int64, device="cuda")
            part[s * cap:(s + 1) * cap] = order[s * cap:(s + 1) * cap]
            _lib.check(L.ckf_route_unpermute(back.data_ptr(), part.data_ptr(), G * cap, 1,
                                             answers[r].data_ptr(), 0))
    for r in range(G):
        a = answers[r].cpu().numpy()
        assert (a == 1).all(), "an inserted key came back negative or unanswered"


def test_padded_exchange_spills_past_capacity():
    from paper_2603_15486_b200 import FilterConfig, _lib
    from paper_2603_15486_b200.kernels import hash_batch
    from paper_2603_15486_b200.sharded import HashRouter

    L = _lib.lib()
    G, n, cap = 4, 50_000, 8_192  # ~12.5 K per shard: ~4.3 K past capacity each
    router = HashRouter(FilterConfig(bucket_count=1 << 10), G)
    h = hash_batch(torch.arange(n, dtype=torch.int64, device="cuda"), 0)
    send = torch.empty(G * cap, dtype=torch.int64, device="cuda")
    order = torch.empty(G * cap, dtype=torch.int64, device="cuda")
    counts = torch.empty(G, dtype=torch.int64, device="cuda")
    spilled = torch.empty(1, dtype=torch.int64, device="cuda")
    wsb = int(L.ckf_route_workspace_bytes(n, G))
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.check(L.ckf_route_partition_padded(h.data_ptr(), n, router.shift, G, cap, send.data_ptr(),
                                            order.data_ptr(), counts.data_ptr(), spilled.data_ptr(),
                                            ws.data_ptr(), wsb, 0))
    c = counts.cpu().numpy()
    assert int(spilled) == int(np.maximum(c - cap, 0).sum()) > 0
    o = order.cpu().numpy().reshape(G, cap)
    sh = router.shard_of(h).cpu().numpy()
    for s in range(G):
        want = np.flatnonzero(sh == s)[:cap]  # stable: the first `cap` of the shard, in arrival order
        assert np.array_equal(o[s][: len(want)], want)
        assert (o[s][len(want):] == -1).all()
        pad = send.view(G, cap)[s][len(want):].cpu().numpy().view(np.uint64)
        assert ((pad >> np.uint64(router.shift)) & np.uint64(G - 1) == (s + 1) % G).all()
