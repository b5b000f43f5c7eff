#!/usr/bin/env python
"""sanitize_case.py -- small runs of every kernel for compute-sanitizer (memcheck / racecheck /
synccheck): configs 1 and 2 (uint8) and a float config-4-shaped crop through qs_me_search_refs with
the fused NNC -> FRMC cascade and fused PR (the bench's path), plus qs_me_search with K = 7 (finalize +
NNC scratch path), the standalone checks (FRMC, RMC, RME, NNC) and qs_project.  Exits non-zero on any
mismatch against a second run (the results must be deterministic).  Not part of the product.

  compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch

    import paper_2203_09200_b200 as qs
    import synth

    dev = torch.device("cuda:0")
    cases = [(1, 64, 64, 2, 8), (2, 352, 288, 6, 16), (4, 192, 128, 6, 9)]
    for cfg, W, H, t, S in cases:
        c = synth.CONFIGS[cfg]
        seq = synth.make_sequence(cfg, w=W, h=H)
        ds = [d for d in (1, 2, 3) if d <= t]
        inps = [synth.pair_inputs(seq, t, d) for d in ds]
        cur = qs.to_plane(inps[0]["cur"], dev)
        msk = qs.to_plane(inps[0]["cur_mask"], dev)
        refs = [qs.to_plane(i["ref"], dev) for i in inps]
        pvs = [qs.to_plane(i["past_val"], dev) for i in inps]
        pms = [qs.to_plane(i["past_mask"], dev) for i in inps]
        prm = qs.make_params(K=8, S=S, ref_f32=c.ref_f32)
        roi = qs.make_roi(W, H)
        res = []
        for rep in range(2):
            outs = [qs.Field.alloc(H, W, c.ref_f32, dev) for _ in inps]
            s, cn = qs.alloc_acc(H, W, dev)
            qs.qs_me_search_refs(cur, msk, refs, roi, prm, outs, fuse=qs.make_checks(), project=(pvs, pms, s, cn))
            torch.cuda.synchronize()
            res.append([o.numpy() for o in outs] + [s.cpu().numpy(), cn.cpu().numpy()])
        for a, b in zip(res[0][:-2], res[1][:-2]):
            for k in a:
                assert np.array_equal(a[k], b[k]), (cfg, k)
        assert np.array_equal(res[0][-2], res[1][-2]) and np.array_equal(res[0][-1], res[1][-1])
        # other entry points on the first pair
        f = qs.Field.alloc(H, W, c.ref_f32, dev)
        qs.qs_me_search(cur, msk, refs[0], roi, qs.make_params(K=7, S=S, ref_f32=c.ref_f32), f, fuse=qs.make_checks())
        qs.qs_me_search(cur, msk, refs[0], roi, prm, f)
        for mode in (qs.QS_RMC, qs.QS_RME):
            g = qs.Field.alloc(H, W, c.ref_f32, dev)
            qs.qs_me_search(cur, msk, refs[0], roi, prm, g)
            qs.qs_reverse_check(mode, cur, msk, refs[0], roi, prm, g)
        qs.qs_nnc(f, roi)
        qs.qs_frmc(cur, msk, refs[0], roi, prm, f)
        s, cn = qs.alloc_acc(H, W, dev)
        qs.qs_project(f, pvs[0], pms[0], roi, s, cn)
        torch.cuda.synchronize()
        print(f"config {cfg} {W}x{H} S={S}: ok")


if __name__ == "__main__":
    main()
