"""ckf_route_partition (multi-GPU routing step) against a stable argsort."""

from __future__ import annotations

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
