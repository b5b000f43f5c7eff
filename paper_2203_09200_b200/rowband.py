"""Row-band sharding of one frame over N ranks, with the reference halo exchange.

SURVEY.md §8(e): rank r owns target rows [y0_r, y1_r), y0_r = 2*floor(r*H/(2G)).  Every border
rule uses global frame coordinates (R25), so a band edge is not a border and the union of the
bands is bit-identical to the single-GPU frame (tests/test_gpu_parity.py::test_row_bands_equal_full_frame).

Exchange step (the path's one real exchange): in the recursive pipeline each rank reconstructs
only its own rows, so before frame t the newest reference f^_{t-1} lacks the halo rows that ME
and the checks read (K/2 + S + 2 rows on each side).  ``exchange_halo`` sends a rank's edge rows
to its neighbours and receives theirs as one grouped point-to-point exchange
(torch.distributed.batch_isend_irecv; with the NCCL backend: ncclSend/ncclRecv inside one
ncclGroupStart/End over NVLink).  The current frame's measured pixels come from the sensor, which
every rank reads with its own halo, and older references were exchanged when they were newest,
so nothing else moves per frame.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch


def halo_rows(S: int, K: int) -> int:
    """Rows beyond a band that ME (+ the 2-row NNC vector halo) and FRMC read: K/2 + S + 2."""
    return K // 2 + S + 2


@dataclass(frozen=True)
class Band:
    rank: int
    world: int
    H: int
    h: int           # halo rows
    y0: int          # first owned row
    y1: int          # one past the last owned row

    @property
    def b0(self) -> int:      # first buffered row
        return max(0, self.y0 - self.h)

    @property
    def b1(self) -> int:      # one past the last buffered row
        return min(self.H, self.y1 + self.h)

    @property
    def rows(self) -> int:
        return self.b1 - self.b0


def band_of(rank: int, world: int, H: int, h: int) -> Band:
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    y0 = 2 * ((rank * H) // (2 * world))
    y1 = 2 * (((rank + 1) * H) // (2 * world)) if rank + 1 < world else H
    if world > 1 and y1 - y0 < h:
        raise ValueError(f"band of {y1 - y0} rows is thinner than the halo ({h}); use fewer ranks")
    return Band(rank, world, H, h, y0, y1)


def exchange_halo(plane: torch.Tensor, band: Band, group=None) -> None:
    """Fill the halo rows of ``plane`` (row i = global row band.b0 + i) from the neighbours.

    Rank r receives min(h, y0) rows from r-1 and min(h, H - y1) rows from r+1, and sends the
    matching edge rows of its own band.  No-op when world == 1.
    """
    if band.world == 1:
        return
    import torch.distributed as dist

    r, h, H = band.rank, band.h, band.H
    own0 = band.y0 - band.b0          # buffer row of the first owned row
    own1 = band.y1 - band.b0          # buffer row one past the last owned row
    ops, landing = [], []

    def recv(rows):
        # pitched planes (row pitch > width) give non-contiguous row slices: receive into a
        # contiguous buffer and copy it in after the wait
        dst = rows if rows.is_contiguous() else torch.empty(rows.shape, dtype=rows.dtype, device=rows.device)
        if dst is not rows:
            landing.append((rows, dst))
        return dst

    def send(rows):
        return rows if rows.is_contiguous() else rows.contiguous()

    if r > 0:
        n_recv = min(h, band.y0)                   # my top halo
        n_send = min(h, H - band.y0)               # the upper neighbour's bottom halo = my first rows
        n_send = min(n_send, own1 - own0)
        ops.append(dist.P2POp(dist.irecv, recv(plane[own0 - n_recv:own0]), r - 1, group))
        ops.append(dist.P2POp(dist.isend, send(plane[own0:own0 + n_send]), r - 1, group))
    if r < band.world - 1:
        n_recv = min(h, H - band.y1)               # my bottom halo
        n_send = min(h, band.y1, own1 - own0)      # the lower neighbour's top halo = my last rows
        ops.append(dist.P2POp(dist.isend, send(plane[own1 - n_send:own1]), r + 1, group))
        ops.append(dist.P2POp(dist.irecv, recv(plane[own1:own1 + n_recv]), r + 1, group))
    for q in dist.batch_isend_irecv(ops):
        q.wait()
    for rows, buf in landing:
        rows.copy_(buf)
