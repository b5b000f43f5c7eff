"""Sequence-scale verification of the bench's launch against the oracle.

Opt-in (minutes to tens of minutes per config): ``QS_VERIFY_SEQ=1,2,3,4,5 pytest -m gpu
tests/test_sequence_verify.py``; ``QS_VERIFY_OUT`` names the JSON report (default
``gpurun_out/verify_seq.json``).  For every frame t >= 1 of a config's sequence (config 5: sequence 0),
the frame's pairs d = 1..min(3, t) go through ``qs_me_search_refs`` exactly as ``bench.py`` launches
them (three references in one launch per kernel, fused NNC -> FRMC cascade, fused PR) with the fields
written, and the oracle's chain (``oracle.pair_chain`` through the OpenMP row driver, then
``oracle.project``) is compared on:

- full planes (every row, every plane, and sum / cnt) for t = 1..5 -- all four phases of the dynamic
  mask, d = 1..3 -- and every 20th frame (configs 3 and 4; configs 1 and 2: every frame; config 5:
  none, a 4K frame costs ~8 min of 16-core oracle time per reference);
- a seeded random block of ceil(1 %) of the target rows in every other pair.

Differences are counted per plane and listed (at most 20 positions per pair) in the report; the test
fails if any plane differs anywhere.  The row bands' cut rows are covered by the band tests of
``test_gpu_parity.py`` (float config 4 at the ``plan_bands`` cuts for 2, 4, 8 ranks; config 5 for 2, 4).
"""
import json
import math
import os
import time

import numpy as np
import pytest
import torch

import oracle
import paper_2203_09200_b200 as qs
import synth

CFGS = [int(c) for c in os.environ.get("QS_VERIFY_SEQ", "").split(",") if c.strip()]
OUT = os.environ.get("QS_VERIFY_OUT", os.path.join("gpurun_out", "verify_seq.json"))
THREADS = int(os.environ.get("QS_ORACLE_THREADS", "0")) or (os.cpu_count() or 1)
DEV = "cuda"

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not CFGS, reason="opt-in: QS_VERIFY_SEQ=<configs> (minutes per config)")]

PLANES = ("alpha", "beta", "err", "count", "status")


def _full_frames(cfg, F):
    if cfg in (1, 2):
        return set(range(1, F))
    if cfg in (3, 4):
        return {t for t in (1, 2, 3, 4, 5) if t < F} | set(range(20, F, 20))
    return set()


def _diff(g, o, rows):
    """Per-plane counts of differing entries on rows [y0, y1) and up to 20 positions."""
    sl = slice(*rows)
    counts, where = {}, []
    for k in PLANES:
        a, b = g[k][sl], o[k][sl]
        if k == "err":
            a = a.astype(np.float32).view(np.uint32) if a.dtype == np.float32 else a.astype(np.uint64)
            b = b.astype(np.float32).view(np.uint32) if b.dtype == np.float32 else b.astype(np.uint64)
        bad = np.argwhere(a != b)
        counts[k] = int(len(bad))
        for y, x in bad[:20]:
            where.append([k, int(y) + rows[0], int(x)])
    return counts, where[:20]


def _verify_config(cfg):
    c = synth.CONFIGS[cfg]
    seq = synth.make_sequence(cfg)
    H, W, S = c.h, c.w, c.S
    full = _full_frames(cfg, c.frames)
    nblk = max(1, math.ceil(0.01 * H))
    rng = np.random.default_rng(1000 + cfg)
    prm = qs.make_params(K=8, S=S, ref_f32=c.ref_f32)
    roi = qs.make_roi(W, H)
    rep = {"config": c.name, "frames": c.frames, "pairs": 0, "rows_checked": 0, "full_frames": sorted(full),
           "row_block": nblk, "mismatches": {k: 0 for k in PLANES + ("sum", "cnt")}, "first_mismatches": [],
           "oracle_threads": THREADS}
    t_gpu = t_or = 0.0
    for t in range(1, c.frames):
        ds = list(range(1, min(3, t) + 1))
        inps = [synth.pair_inputs(seq, t, d) for d in ds]
        t0 = time.time()
        cur = qs.to_plane(inps[0]["cur"], DEV)
        msk = qs.to_plane(inps[0]["cur_mask"], DEV)
        refs = [qs.to_plane(i["ref"], DEV) for i in inps]
        pvs = [qs.to_plane(i["past_val"], DEV) for i in inps]
        pms = [qs.to_plane(i["past_mask"], DEV) for i in inps]
        outs = [qs.Field.alloc(H, W, c.ref_f32, DEV) for _ in inps]
        s, cn = qs.alloc_acc(H, W, DEV)
        qs.qs_me_search_refs(cur, msk, refs, roi, prm, outs, fuse=qs.make_checks(), project=(pvs, pms, s, cn))
        torch.cuda.synchronize()
        gs = []
        for o in outs:
            g = o.numpy()
            if not c.ref_f32:
                g["err"] = g["err"].view(np.uint32)
            gs.append(g)
        gsum = s.cpu().numpy().view(np.uint32)
        gcnt = cn.cpu().numpy()
        t_gpu += time.time() - t0
        if t in full:
            rows = (0, H)
        else:
            y0 = int(rng.integers(0, H - nblk + 1))
            rows = (y0, y0 + nblk)
        t0 = time.time()
        osum = np.zeros((H, W), np.uint32)
        ocnt = np.zeros((H, W), np.uint8)
        for d, g, inp in zip(ds, gs, inps):
            o, _ = oracle.pair_chain(inp, K=8, S=S, check="nnc_frmc", rows=None if rows == (0, H) else rows,
                                     threads=THREADS)
            counts, where = _diff(g, o, rows)
            for k, v in counts.items():
                rep["mismatches"][k] += v
            if where and len(rep["first_mismatches"]) < 50:
                rep["first_mismatches"].append({"t": t, "d": d, "at": where})
            osum, ocnt = oracle.project(o, inp["past_val"], inp["past_mask"], osum, ocnt, rows=rows)
            rep["pairs"] += 1
            rep["rows_checked"] += rows[1] - rows[0]
        sl = slice(*rows)
        rep["mismatches"]["sum"] += int(np.count_nonzero(gsum[sl] != osum[sl]))
        rep["mismatches"]["cnt"] += int(np.count_nonzero(gcnt[sl] != ocnt[sl]))
        t_or += time.time() - t0
    rep["gpu_and_copy_s"] = round(t_gpu, 1)
    rep["oracle_s"] = round(t_or, 1)
    rep["total_mismatches"] = int(sum(rep["mismatches"].values()))
    return rep


@pytest.mark.parametrize("cfg", CFGS)
def test_sequence_bit_exact(cfg):
    rep = _verify_config(cfg)
    os.makedirs(os.path.dirname(OUT) or ".", exist_ok=True)
    allrep = {}
    if os.path.exists(OUT):
        with open(OUT) as f:
            allrep = json.load(f)
    allrep[str(cfg)] = rep
    allrep["host"] = {"cpu_count": os.cpu_count(), "gpu": torch.cuda.get_device_name(0)}
    with open(OUT, "w") as f:
        json.dump(allrep, f, indent=1)
    assert rep["total_mismatches"] == 0, rep["first_mismatches"][:5]
