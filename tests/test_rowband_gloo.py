"""Row-band sharding on CPU: band geometry and the halo exchange over gloo."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2203_09200_b200 import rowband


def test_band_geometry_covers_frame():
    for H, G in ((1080, 1), (1080, 2), (1080, 4), (1080, 8), (2160, 8), (288, 3)):
        h = rowband.halo_rows(24, 8)
        if G > 1 and H // G < h:
            continue
        bands = [rowband.band_of(r, G, H, h) for r in range(G)]
        assert bands[0].y0 == 0 and bands[-1].y1 == H
        for a, b in zip(bands, bands[1:]):
            assert a.y1 == b.y0 and a.y1 % 2 == 0          # contiguous, even (2x2 blocks stay whole)
        for b in bands:
            assert b.b0 == max(0, b.y0 - h) and b.b1 == min(H, b.y1 + h)
    assert rowband.halo_rows(24, 8) == 30


def test_thin_band_rejected():
    with pytest.raises(ValueError):
        rowband.band_of(1, 8, 64, rowband.halo_rows(24, 8))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, H, W, h, q, pitch=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        band = rowband.band_of(rank, world, H, h)
        glob = torch.arange(H * W, dtype=torch.float32).reshape(H, W)
        # a pitched plane (row pitch > width, as qs.pitched gives): non-contiguous row slices
        plane = torch.full((band.rows, pitch or W), float("nan"))[:, :W]
        plane[band.y0 - band.b0:band.y1 - band.b0] = glob[band.y0:band.y1]   # only owned rows exist
        rowband.exchange_halo(plane, band)
        ok = torch.equal(plane, glob[band.b0:band.b1])
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,pitch", [(2, None), (3, None), (2, 20)])
def test_halo_exchange_gloo(world, pitch):
    H, W = 120, 16
    h = rowband.halo_rows(8, 8)     # 14 rows
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, H, W, h, q, pitch)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(res[r] for r in range(world)), res


def test_plan_bands_cover_balance_and_halo():
    """rowband.plan_bands: even cuts covering [0, H), every band at least the halo, and a largest
    estimated cost no worse than the even split's (SURVEY.md 8(e) row bands)."""
    for (H, S, K) in ((1080, 24, 8), (2160, 32, 8), (720, 16, 8), (288, 16, 8), (64, 8, 8)):
        h = rowband.halo_rows(S, K)
        for G in (1, 2, 3, 4, 8):
            if G > 1 and H // G < h:
                continue
            cuts = rowband.plan_bands(G, H, S, K)
            assert cuts[0] == 0 and cuts[-1] == H and len(cuts) == G + 1
            assert all(c % 2 == 0 for c in cuts)
            assert all(cuts[i + 1] - cuts[i] >= (h if G > 1 else 1) for i in range(G))
            worst = max(rowband.band_cost(cuts[i], cuts[i + 1], H, S, K) for i in range(G))
            even = [2 * ((r * H) // (2 * G)) for r in range(G)] + [H]
            if min(even[i + 1] - even[i] for i in range(G)) >= h:
                assert worst <= max(rowband.band_cost(even[i], even[i + 1], H, S, K) for i in range(G))
            bands = [rowband.band_of(r, G, H, h, S=S, K=K) for r in range(G)]
            assert [b.y0 for b in bands] + [bands[-1].y1] == cuts
    # config 4 on 8 ranks: the edge bands shrink (their tiles run the border phases)
    cuts = rowband.plan_bands(8, 1080, 24, 8)
    assert cuts[1] - cuts[0] < 135 and cuts[-1] - cuts[-2] < 135
