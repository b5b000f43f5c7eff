#!/usr/bin/env python
"""Bank-conflict degree of the epilogue's FRMC row loads against the current region's pitch (a model, CPU only).
A 16x16 entry tile keeps each entry with probability p (NNC survivors); the FRMC items (dy, entry) are taken
in the kernel's order (row-major compacted entry list, one dy after the other), 32 per warp; a scalar LDS of
the row loop reads word (row + dy) * pitch + col + k of every lane, so its wavefronts = the largest number of
distinct words falling in one of the 32 banks.  Prints the mean degree for pitches 48..79 words.
  python tools/epilogue_pitch_sim.py"""
import numpy as np


def degree(pitch, p, rng, trials=300):
    dys = (-4, -2, -1, 0, 1, 2, 4)
    tot = n = 0
    for _ in range(trials):
        ys, xs = np.nonzero(rng.random((16, 16)) < p)
        items = [(int(y) + 4 + dy, int(x)) for dy in dys for y, x in zip(ys, xs)]
        for w in range(0, len(items), 32):
            banks = {}
            for r, c in items[w:w + 32]:
                a = r * pitch + c
                banks.setdefault(a % 32, set()).add(a)
            tot += max(len(v) for v in banks.values())
            n += 1
    return tot / max(n, 1)


if __name__ == "__main__":
    for p in (0.5, 0.7, 0.9):
        rng = np.random.default_rng(1)
        res = sorted((round(degree(q, p, rng), 2), q) for q in range(48, 80))
        print(f"p={p}: pitch 48 -> {dict((q, d) for d, q in res)[48]}; best five (degree, pitch): {res[:5]}")
