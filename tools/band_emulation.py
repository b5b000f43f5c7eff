#!/usr/bin/env python
"""band_emulation.py -- one-device emulation of the row-band split: for G = 1, 2,
4, 8 every band runs its qs_me_search_refs (config 4, frame 3, three references, fused checks) with
band-sized buffers; prints the largest per-band me_box + epilogue time.  PLAN=1 uses
rowband.plan_bands (the bench's split), otherwise the even split.  Not part of the product.

  python tools/band_emulation.py;  PLAN=1 python tools/band_emulation.py
"""
import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_2203_09200_b200 as qs, synth
from paper_2203_09200_b200 import rowband
cfg = synth.CONFIGS[4]
seq = synth.make_sequence(4)
t = 3
W, H, S, K = cfg.w, cfg.h, cfg.S, cfg.K
dev = torch.device("cuda:0")
import os as _o
PLAN = dict(S=S, K=K) if _o.environ.get("PLAN") else {}
for G in (1, 2, 4, 8):
    tot = 0.0
    for r in range(G):
        band = rowband.band_of(r, G, H, rowband.halo_rows(S, K), **PLAN)
        fr = synth.pair_inputs(seq, t, 1)
        cur = qs.to_plane(fr["cur"][band.b0:band.b1], dev)
        msk = qs.to_plane(fr["cur_mask"][band.b0:band.b1], dev)
        refs = [qs.to_plane(synth.pair_inputs(seq, t, d)["ref"][band.b0:band.b1], dev) for d in (1, 2, 3)]
        roi = qs.make_roi(W, H, band.y0, band.y1, band.b0, band.rows)
        prm = qs.make_params(K=K, S=S, ref_f32=True)
        outs = [qs.Field.alloc(band.rows, W, True, dev) for _ in range(3)]
        ws = qs.workspace(roi, prm, dev, n_refs=3)
        chk = qs.make_checks()
        qs.qs_me_search_refs(cur, msk, refs, roi, prm, outs, fuse=chk, ws=ws)
        torch.cuda.synchronize()
        qs.qs_profile_reset(); qs.qs_profile_enable(True)
        for _ in range(3):
            qs.qs_me_search_refs(cur, msk, refs, roi, prm, outs, fuse=chk, ws=ws)
        torch.cuda.synchronize(); qs.qs_profile_enable(False)
        ms, n = qs.qs_profile_read("me_box")
        me, ne = qs.qs_profile_read("epilogue")
        tot = max(tot, (ms + me) / n)
    print(f"G={G}: me_box + epilogue per rank (max) {tot:.3f} ms, ideal {10.62 / G:.3f}")
