"""Helpers that run the CUDA path (through the C ABI) and the CPU oracle on the same inputs."""
import numpy as np
import torch

import oracle
import paper_2203_09200_b200 as qs

DEV = "cuda"


def planes(inp, dev=DEV):
    return {k: qs.to_plane(inp[k], dev) for k in ("cur", "cur_mask", "ref", "past_val", "past_mask")}


def gpu_me(inp, K=8, S=8, min_support=8, ssd=False, fuse=None, rows=None, band=None, dev=DEV):
    """ME (optionally with fused checks) on the GPU; returns (field dict, evals).

    band=(buf_y0, buf_rows) runs with buffers holding only those rows (row-band mode).
    """
    H, W = inp["cur"].shape
    f32 = inp["ref"].dtype == np.float32
    y0, y1 = rows if rows is not None else (0, H)
    if band is None:
        b0, br = 0, H
    else:
        b0, br = band
    p = {k: qs.to_plane(inp[k][b0:b0 + br], dev) for k in ("cur", "cur_mask", "ref")}
    roi = qs.make_roi(W, H, y0, y1, b0, br)
    prm = qs.make_params(K=K, S=S, min_support=min_support, ssd=ssd, ref_f32=f32)
    f = qs.Field.alloc(br, W, f32, dev)
    ev = torch.zeros(1, dtype=torch.int64, device=dev)
    qs.qs_me_search(p["cur"], p["cur_mask"], p["ref"], roi, prm, f, fuse=fuse, eval_count=ev)
    torch.cuda.synchronize()
    g = f.numpy()
    if not f32:
        g["err"] = g["err"].view(np.uint32)
    full = {}
    for k, v in g.items():
        a = np.zeros((H, W), v.dtype)
        a[b0:b0 + br] = v
        full[k] = a
    return full, int(ev.item())


def field_to_gpu(field, f32, dev=DEV):
    H, W = field["status"].shape
    f = qs.Field.alloc(H, W, f32, dev)
    f.alpha.copy_(torch.from_numpy(np.ascontiguousarray(field["alpha"])))
    f.beta.copy_(torch.from_numpy(np.ascontiguousarray(field["beta"])))
    err = np.ascontiguousarray(field["err"])
    f.err.copy_(torch.from_numpy(err.astype(np.float32) if f32 else err.astype(np.uint32).view(np.int32)))
    f.count.copy_(torch.from_numpy(np.ascontiguousarray(field["count"])))
    f.status.copy_(torch.from_numpy(np.ascontiguousarray(field["status"])))
    return f


def gpu_check(kind, inp, field, K=8, S=8, min_support=8, ssd=False, offsets=qs.PAPER_FRMC_OFFSETS, threshold=1,
              rows=None, dev=DEV):
    """Run one check on the GPU over a given field (staged parity); returns (status, evals)."""
    H, W = inp["cur"].shape
    f32 = inp["ref"].dtype == np.float32
    p = planes(inp, dev)
    y0, y1 = rows if rows is not None else (0, H)
    roi = qs.make_roi(W, H, y0, y1)
    prm = qs.make_params(K=K, S=S, min_support=min_support, ssd=ssd, ref_f32=f32)
    f = field_to_gpu(field, f32, dev)
    ev = torch.zeros(1, dtype=torch.int64, device=dev)
    if kind == "nnc":
        qs.qs_nnc(f, roi, threshold)
    elif kind == "nnc_pairs":
        qs.qs_nnc_mode(f, roi, threshold, qs.QS_NNC_PAIRS)
    elif kind == "frmc":
        qs.qs_frmc(p["cur"], p["cur_mask"], p["ref"], roi, prm, f, offsets=offsets, eval_count=ev)
    elif kind == "rmc":
        qs.qs_reverse_check(qs.QS_RMC, p["cur"], p["cur_mask"], p["ref"], roi, prm, f, eval_count=ev)
    elif kind == "rme":
        qs.qs_reverse_check(qs.QS_RME, p["cur"], p["cur_mask"], p["ref"], roi, prm, f, eval_count=ev)
    else:
        raise ValueError(kind)
    torch.cuda.synchronize()
    return f.status.cpu().numpy(), int(ev.item())


def gpu_project(inp, field, acc=None, dev=DEV):
    H, W = inp["cur"].shape
    f32 = inp["ref"].dtype == np.float32
    p = planes(inp, dev)
    f = field_to_gpu(field, f32, dev)
    s, c = qs.alloc_acc(H, W, dev)
    if acc is not None:
        s.copy_(torch.from_numpy(acc[0].astype(np.uint32).view(np.int32)))
        c.copy_(torch.from_numpy(acc[1]))
    qs.qs_project(f, p["past_val"], p["past_mask"], qs.make_roi(W, H), s, c)
    torch.cuda.synchronize()
    return s.cpu().numpy().view(np.uint32), c.cpu().numpy()


def assert_field_equal(g, o, rows=None, what=""):
    sl = slice(None) if rows is None else slice(*rows)
    for k in ("alpha", "beta", "count", "status"):
        a, b = g[k][sl], o[k][sl]
        if not np.array_equal(a, b):
            idx = np.argwhere(a != b)[:5]
            raise AssertionError(f"{what} plane {k} differs at {idx.tolist()}: gpu {a[tuple(idx.T)]} oracle {b[tuple(idx.T)]}")
    ge, oe = g["err"][sl], o["err"][sl]
    if ge.dtype == np.float32 or oe.dtype == np.float32:
        assert np.array_equal(ge.astype(np.float32).view(np.uint32), oe.astype(np.float32).view(np.uint32)), what
    else:
        assert np.array_equal(ge.astype(np.uint64), oe.astype(np.uint64)), what
