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
from functools import lru_cache

import numpy as np
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


# me_box tiling (paper_2203_09200_b200/csrc): 56-row tiles over the ME rows (the band's rows plus the
# 2-row NNC halo), placed to minimise border tile rows; a tile runs the slower border phases when an
# output it keeps has a window that can leave the frame or the band's buffer: ~1.75x an interior tile
# for uint8 references; float references run border tiles in a grid of their own with phase 2 in support
# runs, measured 1.46x (config 4: 1.94 ms for 96 border tiles, 6.97 ms for
# 504 interior tiles, profiles/r02c/ncu_box_{border,interior}_c4.json).
TILE_ROWS = 56
BORDER_TILE_COST = 1.75
BORDER_TILE_COST_F32 = 1.46
# the fused epilogue (checks + PR) per output row, in the same unit (config 4: 0.66 ms per reference
# and frame against 0.13 ms per interior tile row and reference)
EPILOGUE_PER_ROW = 0.0047


@lru_cache(maxsize=None)
def _border_tile_rows(lo: int, hi: int, S: int, K: int, b0: int, b1: int) -> tuple[int, int]:
    """(border tile rows, tile rows) of me_box over output rows [lo, hi), placed as the library places
    them (csrc/qs_api.cu place_tile_rows: the grid offset, lo - offset even, with the fewest border tile
    rows, then the fewest rows)."""
    offs = np.arange(lo & 1, TILE_ROWS, 2)
    rows = (hi - lo + offs + TILE_ROWS - 1) // TILE_ROWS
    t = np.arange(int(rows.max()))
    py0 = lo - offs[:, None] + t[None, :] * TILE_ROWS
    ylast = np.minimum(py0 + TILE_ROWS, hi) - 1
    valid = t[None, :] < rows[:, None]
    border = ((py0 - K // 2 - S < b0) | (ylast + (K - 1 - K // 2) + S > b1 - 1)) & valid
    nb = border.sum(axis=1)
    i = int(np.lexsort((rows, nb))[0])
    return int(nb[i]), int(rows[i])


def band_cost(y0: int, y1: int, H: int, S: int, K: int = 8, f32: bool = False) -> float:
    """Estimated step time of the band [y0, y1) in interior-tile-row units: me_box tiles (placed as
    the library places them, border tiles weighted) plus the epilogue's rows."""
    lo, hi = max(0, y0 - 2), min(H, y1 + 2)
    h = halo_rows(S, K)
    b0, b1 = max(0, y0 - h), min(H, y1 + h)
    nb, rows = _border_tile_rows(lo, hi, S, K, b0, b1)
    w = BORDER_TILE_COST_F32 if f32 else BORDER_TILE_COST
    return EPILOGUE_PER_ROW * (y1 - y0) + rows + (w - 1.0) * nb


def plan_bands(world: int, H: int, S: int, K: int = 8, h: int | None = None, f32: bool = False) -> list[int]:
    """Even row cuts 0 = c_0 < ... < c_world = H minimising the largest band_cost (bands at least h
    rows): the smallest cost bound T for which greedy packing covers the frame, then the cuts."""
    h = halo_rows(S, K) if h is None else h
    if world == 1:
        return [0, H]

    def pack(T):
        cuts, y0 = [0], 0
        for r in range(world - 1):
            rest = world - 1 - r                          # bands still to place after this one
            y1 = y0 + h + (h & 1)
            best = None
            while y1 <= H - rest * (h + (h & 1)):
                if band_cost(y0, y1, H, S, K, f32) <= T:
                    best = y1
                y1 += 2
            if best is None:
                return None
            cuts.append(best)
            y0 = best
        if H - y0 < h or band_cost(y0, H, H, S, K, f32) > T:
            return None
        return cuts + [H]

    def worst(cuts):
        return max(band_cost(cuts[i], cuts[i + 1], H, S, K, f32) for i in range(world))

    # band_cost is not monotone in y0 (the tile grid starts at y0 - 2), so greedy packing is not
    # optimal on its own: keep the best of the even split and the greedy plan.
    even = [2 * ((r * H) // (2 * world)) for r in range(world)] + [H]
    plans = [even] if min(even[i + 1] - even[i] for i in range(world)) >= h else []
    lo_t, hi_t = 0.0, band_cost(0, H, H, S, K, f32)          # feasibility of pack(T) is monotone in T
    best = pack(hi_t)
    for _ in range(40):
        mid = 0.5 * (lo_t + hi_t)
        cuts = pack(mid)
        if cuts is not None:
            best, hi_t = cuts, mid
        else:
            lo_t = mid
    if best is not None:
        plans.append(best)
    if not plans:
        raise ValueError("no band plan")
    return min(plans, key=worst)


def band_of(rank: int, world: int, H: int, h: int, S: int | None = None, K: int = 8, f32: bool = False) -> Band:
    """Rank r's band: an even split of the rows, or (S given) the cost-balanced plan_bands split."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    if S is not None and world > 1:
        cuts = plan_bands(world, H, S, K, h, f32)
        y0, y1 = cuts[rank], cuts[rank + 1]
    else:
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

    # gloo moves host memory only: device planes are staged through the host (the functional-check
    # backend of bench.py and the CPU tests); NCCL sends device memory directly.
    host = plane.is_cuda and dist.get_backend(group) == "gloo"

    def recv(rows):
        # pitched planes (row pitch > width) give non-contiguous row slices: receive into a
        # contiguous buffer and copy it in after the wait
        if host:
            dst = torch.empty(rows.shape, dtype=rows.dtype)
        else:
            dst = rows if rows.is_contiguous() else torch.empty(rows.shape, dtype=rows.dtype, device=rows.device)
        if dst is not rows:
            landing.append((rows, dst))
        return dst

    def send(rows):
        if host:
            return rows.cpu()
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
