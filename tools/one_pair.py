#!/usr/bin/env python
"""one_pair.py -- run qs_me_search (fused NNC -> FRMC) on one (frame, reference) pair of a config,
for ncu captures and quick kernel timing.  Not part of the product or of bench.py.

  python tools/one_pair.py [--config 4] [--t 3] [--d 1] [--reps 5] [--refs]   (--refs: d = 1..3 in one
                                                                               qs_me_search_refs call)
  ncu --set full -k regex:box_kernel -s 1 -c 1 python tools/one_pair.py --reps 2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--t", type=int, default=3)
    ap.add_argument("--d", type=int, default=1)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-checks", action="store_true")
    ap.add_argument("--refs", action="store_true", help="the frame's three references in one qs_me_search_refs call")
    args = ap.parse_args()
    import torch

    import paper_2203_09200_b200 as qs
    import synth

    cfg = synth.CONFIGS[args.config]
    seq = synth.make_sequence(args.config)
    inp = synth.pair_inputs(seq, args.t, args.d)
    dev = torch.device("cuda:0")
    H, W = inp["cur"].shape
    cur, msk, ref = (qs.to_plane(inp[k], dev) for k in ("cur", "cur_mask", "ref"))
    roi = qs.make_roi(W, H)
    prm = qs.make_params(K=cfg.K, S=cfg.S, ssd=cfg.ssd, ref_f32=cfg.ref_f32)
    f = qs.Field.alloc(H, W, cfg.ref_f32, dev)
    ws = qs.workspace(roi, prm, dev)
    chk = None if args.no_checks else qs.make_checks()
    if args.refs:
        refs = [qs.to_plane(synth.pair_inputs(seq, args.t, d)["ref"], dev) for d in (1, 2, 3)]
        fs = [qs.Field.alloc(H, W, cfg.ref_f32, dev) for _ in refs]
        ws3 = qs.workspace(roi, prm, dev, n_refs=3)

        def call():
            qs.qs_me_search_refs(cur, msk, refs, roi, prm, fs, fuse=chk, ws=ws3)
    else:
        def call():
            qs.qs_me_search(cur, msk, ref, roi, prm, f, fuse=chk, ws=ws)
    call()   # warm-up (module load, attributes)
    torch.cuda.synchronize()
    qs.qs_profile_enable(True)
    for _ in range(args.reps):
        call()
    torch.cuda.synchronize()
    for k in qs.PROFILE_KERNELS:
        ms, n = qs.qs_profile_read(k)
        if n:
            print(f"{k:12s} {ms / n:8.3f} ms/launch  ({n} launches)")


if __name__ == "__main__":
    main()
