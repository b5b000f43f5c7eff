#!/usr/bin/env python
"""tma_debug.py -- one float-reference ME call with QS_TMA=1 on a small frame (debug aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2203_09200_b200 as qs, synth
S = int(sys.argv[1]) if len(sys.argv) > 1 else 6
ssd = len(sys.argv) > 2 and sys.argv[2] == "ssd"
seq = synth.make_sequence(4, w=160, h=112)
inp = synth.pair_inputs(seq, 7, 2)
H, W = inp["cur"].shape
p = {k: qs.to_plane(inp[k]) for k in ("cur", "cur_mask", "ref")}
f = qs.Field.alloc(H, W, True)
qs.qs_me_search(p["cur"], p["cur_mask"], p["ref"], qs.make_roi(W, H), qs.make_params(K=8, S=S, ssd=ssd, ref_f32=True), f)
torch.cuda.synchronize()
print("ok S", S, "ssd", ssd, int((f.status == 2).sum().item()))
