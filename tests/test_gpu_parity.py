"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bar: every plane bit-exact (alpha, beta, err, count, status, PR sum/cnt,
evaluation counts) for uint8 AND float32 references -- the float argmin is certified against an
error bound and the uncertain outputs are recomputed in the definition's fp32 order (DESIGN.md
"Float certification"), so the float path reaches the oracle's R23 result exactly.
"""
import os

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

_THREADS = max(1, os.cpu_count() or 1)   # the oracle's OpenMP row driver (same definitions, rows in parallel)

if torch.cuda.is_available():
    from gpu_helpers import (assert_field_equal, gpu_check, gpu_me, gpu_project)
    import paper_2203_09200_b200 as qs


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


# ---------------------------------------------------------------------------
# Config 1: the correctness config, every pair, whole chain (ME -> NNC -> FRMC -> PR)
# ---------------------------------------------------------------------------
def test_config1_full_chain_bit_exact():
    seq = synth.make_sequence(1)
    for t in (1, 2):
        osum = np.zeros((64, 64), np.uint32)
        ocnt = np.zeros((64, 64), np.uint8)
        gacc = (np.zeros((64, 64), np.uint32), np.zeros((64, 64), np.uint8))
        for d in range(1, min(3, t) + 1):
            inp = synth.pair_inputs(seq, t, d)
            g, gev = gpu_me(inp, K=8, S=8, fuse=qs.make_checks())
            o, oev = oracle.pair_chain(inp, K=8, S=8, check="nnc_frmc")
            assert_field_equal(g, o, what=f"t={t} d={d}")
            assert gev == oev
            osum, ocnt = oracle.project(o, inp["past_val"], inp["past_mask"], osum, ocnt)
            gacc = gpu_project(inp, g, gacc)
        assert np.array_equal(gacc[0], osum) and np.array_equal(gacc[1], ocnt)


def test_config2_me_and_cascade_bit_exact():
    seq = synth.make_sequence(2)
    for (t, d) in ((5, 1), (6, 3)):
        inp = synth.pair_inputs(seq, t, d)
        g, gev = gpu_me(inp, K=8, S=16, fuse=qs.make_checks())
        o, oev = oracle.pair_chain(inp, K=8, S=16, check="nnc_frmc")
        assert_field_equal(g, o, what=f"c2 t={t} d={d}")
        assert gev == oev


# ---------------------------------------------------------------------------
# Fuzz: random small instances, every K the build supports, S from 0, SAD/SSD, ragged sizes
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("seed", range(24))
def test_fuzz_me_u8(seed):
    rng = np.random.default_rng(seed)
    K = int(rng.integers(1, 10))
    S = int(rng.integers(0, 7))
    W = int(rng.integers(1, 50)) * 2
    H = int(rng.integers(1, 40)) * 2
    ssd = bool(rng.integers(0, 2))
    ms = int(rng.integers(1, 12))
    inp = synth.rank_free_random_instance(100 + seed, W, H, smooth=bool(seed % 2), dynamic=bool(seed % 3), t=seed)
    g, _ = gpu_me(inp, K=K, S=S, min_support=ms, ssd=ssd)
    o = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=K, S=S, min_support=ms, ssd=ssd)
    assert_field_equal(g, o, what=f"seed={seed} K={K} S={S} {W}x{H} ssd={ssd} ms={ms}")


@pytest.mark.parametrize("seed", range(8))
def test_fuzz_checks_u8_staged(seed):
    """Each check on the same (oracle) field: statuses and counts bit-exact."""
    rng = np.random.default_rng(1000 + seed)
    K = int(rng.choice([3, 4, 8, 9]))
    S = int(rng.integers(1, 6))
    ssd = bool(seed % 2)
    W, H = 40, 30
    inp = synth.rank_free_random_instance(300 + seed, W, H, smooth=True)
    kw = dict(K=K, S=S, min_support=4, ssd=ssd)
    o = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], **kw)
    offs = tuple(x for x in (-3, -1, 0, 1, 3) if abs(x) <= S)
    st, ev = gpu_check("frmc", inp, o, offsets=offs, **kw)
    ost, oev = oracle.frmc(inp["cur"], inp["cur_mask"], inp["ref"], o, offsets=offs, **kw)
    assert np.array_equal(st, ost) and ev == oev
    st, ev = gpu_check("rmc", inp, o, **kw)
    ost, oev = oracle.rmc(inp["cur"], inp["cur_mask"], inp["ref"], o, **kw)
    assert np.array_equal(st, ost) and ev == oev
    st, ev = gpu_check("rme", inp, o, **kw)
    ost, oev = oracle.rme(inp["cur"], inp["cur_mask"], inp["ref"], o, **kw)
    assert np.array_equal(st, ost) and ev == oev
    st, _ = gpu_check("nnc", inp, o)
    assert np.array_equal(st, oracle.nnc(o))


def _perturbed_field(inp, K, S, seed, frac=0.15, ssd=False):
    """Oracle ME field with a fraction of vectors replaced by random ones; (err, count) re-scored
    with the forward cost so the field stays consistent (identity P4)."""
    o = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=K, S=S, ssd=ssd)
    rng = np.random.default_rng(seed)
    ys, xs = np.nonzero(o["status"] == oracle.CANDIDATE)
    pick = rng.random(ys.size) < frac
    for y, x in zip(ys[pick], xs[pick]):
        a, b = (int(v) for v in rng.integers(-S, S + 1, 2))
        e, n = oracle.cost_fwd(inp["cur"], inp["cur_mask"], inp["ref"], y, x, a, b, K=K, ssd=ssd)
        if n < 8:
            continue
        o["alpha"][y, x], o["beta"][y, x], o["err"][y, x], o["count"][y, x] = a, b, e, n
    return o


@pytest.mark.parametrize("seed,f32,ssd", [(0, False, False), (1, True, False), (2, False, True), (3, True, True)])
def test_frmc_rmc_tiled_k8_perturbed(seed, f32, ssd):
    """The tiled K=8 reverse-grid kernel (paper offsets / RMC groups) on fields with wrong vectors."""
    inp = synth.rank_free_random_instance(900 + seed, 56, 44, ref_f32=f32, smooth=True)
    S = 9
    o = _perturbed_field(inp, 8, S, seed, ssd=ssd)
    kw = dict(K=8, S=S, ssd=ssd)
    st, ev = gpu_check("frmc", inp, o, **kw)
    ost, oev = oracle.frmc(inp["cur"], inp["cur_mask"], inp["ref"], o, **kw)
    assert np.array_equal(st, ost) and ev == oev
    assert (ost == oracle.REJECTED).sum() > 0 and (ost == oracle.ACCEPTED).sum() > 0
    st, ev = gpu_check("rmc", inp, o, **kw)
    ost, oev = oracle.rmc(inp["cur"], inp["cur_mask"], inp["ref"], o, **kw)
    assert np.array_equal(st, ost) and ev == oev
    # Offsets given in another order: same decisions (a set).
    st2, _ = gpu_check("frmc", inp, o, offsets=(7, 3, 1, 0, -1, -3, -7), **kw)
    ost2, _ = oracle.frmc(inp["cur"], inp["cur_mask"], inp["ref"], o, offsets=(7, 3, 1, 0, -1, -3, -7), **kw)
    assert np.array_equal(st2, ost2)


def test_nnc_golden_on_gpu(golden):
    g = golden("nnc_hand.json")
    for case in g["cases"]:
        a = np.array(case["alpha"], np.int8)
        H, W = a.shape
        if W % 2 or H % 2:   # the ABI requires even frames; pad with NOT_TARGET entries
            Hp, Wp = H + H % 2, W + W % 2
        else:
            Hp, Wp = H, W
        fld = {k: np.zeros((Hp, Wp), dt) for k, dt in (("alpha", np.int8), ("beta", np.int8), ("err", np.uint32),
                                                        ("count", np.uint8), ("status", np.uint8))}
        fld["alpha"][:H, :W] = a
        fld["beta"][:H, :W] = np.array(case["beta"], np.int8)
        fld["status"][:H, :W] = np.array(case["status"], np.uint8)
        inp = dict(cur=np.zeros((Hp, Wp), np.uint8), cur_mask=np.zeros((Hp, Wp), np.uint8),
                   ref=np.zeros((Hp, Wp), np.uint8), past_val=np.zeros((Hp, Wp), np.uint8),
                   past_mask=np.zeros((Hp, Wp), np.uint8))
        st, _ = gpu_check("nnc", inp, fld)
        assert np.array_equal(st[:H, :W], np.array(case["expect"], np.uint8)), case["name"]


def test_project_golden_on_gpu(golden):
    g = golden("project_hand.json")
    acc = (np.zeros((4, 4), np.uint32), np.zeros((4, 4), np.uint8))
    for r in g["refs"]:
        fld = dict(alpha=np.array(r["alpha"], np.int8), beta=np.array(r["beta"], np.int8),
                   err=np.zeros((4, 4), np.uint32), count=np.zeros((4, 4), np.uint8),
                   status=np.array(r["status"], np.uint8))
        inp = dict(cur=np.zeros((4, 4), np.uint8), cur_mask=np.zeros((4, 4), np.uint8), ref=np.zeros((4, 4), np.uint8),
                   past_val=np.array(r["past_val"], np.uint8), past_mask=np.array(g["past_mask"], np.uint8))
        acc = gpu_project(inp, fld, acc)
    assert np.array_equal(acc[0], np.array(g["expect_sum"])) and np.array_equal(acc[1], np.array(g["expect_cnt"]))


def test_p13_micro_golden_on_gpu(golden):
    g = golden("p13_micro.json")
    inp = dict(cur=np.array(g["cur"], np.uint8), cur_mask=np.array(g["mask"], np.uint8),
               ref=np.array(g["ref"], np.uint8))
    f, _ = gpu_me(inp, K=g["K"], S=g["S"], min_support=g["min_support"])
    for ex in g["expect"]:
        y, x = ex["p"]
        assert (int(f["alpha"][y, x]), int(f["beta"][y, x])) == tuple(ex["v"])
        assert int(f["err"][y, x]) == ex["e"] and int(f["count"][y, x]) == ex["n"]


# ---------------------------------------------------------------------------
# Float-reference path (config 4's arithmetic)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("S,K,ssd", [(24, 8, False), (6, 8, True), (5, 3, False), (4, 9, False)])
def test_f32_me_bit_exact(S, K, ssd):
    seq = synth.make_sequence(4, w=160, h=112)
    inp = synth.pair_inputs(seq, 7, 2)
    assert inp["ref"].dtype == np.float32
    g, _ = gpu_me(inp, K=K, S=S, ssd=ssd)
    o = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=K, S=S, ssd=ssd)
    assert_field_equal(g, o, what=f"f32 S={S} K={K} ssd={ssd}")


def test_f32_quad_tiles_bit_exact():
    """A frame large enough for interior quarter-sampling tiles (the K=8 block-grid body)."""
    seq = synth.make_sequence(4, w=384, h=256)
    inp = synth.pair_inputs(seq, 5, 1)
    g, _ = gpu_me(inp, K=8, S=16)
    o = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=8, S=16, threads=_THREADS)
    assert_field_equal(g, o, what="f32 quad tiles")


@pytest.mark.parametrize("K,S", [(8, 9), (8, 16), (5, 4)])
def test_f32_exact_ties_take_the_certify_path(K, S):
    """Float references holding integer values on flat patches: many candidates tie EXACTLY (equal
    means), so the certificate fails there and the outputs are recomputed in the definition's order
    -- the tie must go to the lowest rank (R7) exactly as in the oracle."""
    rng = np.random.default_rng(1234 + S)
    W, H = 256, 192
    inp = synth.rank_free_random_instance(55 + S, W, H, ref_f32=True, smooth=True)
    ref = np.round(inp["ref"]).astype(np.float32)
    ref[40:120, 60:200] = 100.0                       # flat patch: every candidate inside ties
    cur = inp["dense_cur"].copy()
    cur[40:120, 60:200] = 100
    ref[130:170, 20:90] = np.float32(77.25)           # flat non-integer patch
    cur[130:170, 20:90] = 77
    m = inp["cur_mask"]
    inp = dict(inp, ref=ref, cur=(cur * m).astype(np.uint8))
    qs.qs_certify_stats(reset=True)
    g, _ = gpu_me(inp, K=K, S=S)
    n_re = qs.qs_certify_stats(reset=True)
    o = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=K, S=S, threads=_THREADS)
    assert_field_equal(g, o, what=f"f32 ties K={K} S={S}")
    assert n_re > 1000, n_re                         # the flat patches go through the exact recompute


def test_non_quarter_mask_falls_back_bit_exact():
    """Masks that are not quarter masks (two or zero measurements per 2x2 block) take the
    generic body inside the same launch; results stay bit-exact."""
    rng = np.random.default_rng(77)
    W, H = 352, 288
    inp = synth.rank_free_random_instance(77, W, H, smooth=True)
    m = (rng.random((H, W)) < 0.3).astype(np.uint8)
    m[100:160, 100:200] = synth.quarter_mask(100, 60, 5, False)   # mixed: quarter patch inside
    inp["cur_mask"] = m
    inp["cur"] = (inp["dense_cur"] * m).astype(np.uint8)
    g, _ = gpu_me(inp, K=8, S=16)
    o = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=8, S=16)
    assert_field_equal(g, o, what="non-quarter mask")


def test_f32_checks_bit_exact_given_field():
    """FRMC / RMC re-sum each reverse cost in the oracle's row-major fp32 order, and RME's dense
    reverse argmin is certified like the forward one: every decision equals the oracle's."""
    seq = synth.make_sequence(4, w=96, h=64)
    inp = synth.pair_inputs(seq, 9, 1)
    kw = dict(K=8, S=8)
    o = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], **kw)
    st, ev = gpu_check("frmc", inp, o, **kw)
    ost, oev = oracle.frmc(inp["cur"], inp["cur_mask"], inp["ref"], o, **kw)
    assert np.array_equal(st, ost) and ev == oev
    st, ev = gpu_check("rmc", inp, o, **kw)
    ost, oev = oracle.rmc(inp["cur"], inp["cur_mask"], inp["ref"], o, **kw)
    assert np.array_equal(st, ost) and ev == oev
    st, ev = gpu_check("rme", inp, o, **kw)
    ost, oev = oracle.rme(inp["cur"], inp["cur_mask"], inp["ref"], o, **kw)
    assert np.array_equal(st, ost) and ev == oev


@pytest.mark.parametrize("S,ssd", [(8, False), (5, True)])
def test_f32_rme_ties_bit_exact(S, ssd):
    """RME on float references with exact ties in the reverse costs (integer-valued flat patches):
    the reverse argmin's uncertain positions are recomputed exactly (certify, reverse mode)."""
    W, H = 128, 96
    inp = synth.rank_free_random_instance(91 + S, W, H, ref_f32=True, smooth=True)
    ref = np.round(inp["ref"]).astype(np.float32)
    ref[30:60, 30:90] = 50.0
    cur = inp["dense_cur"].copy()
    cur[30:60, 30:90] = 50
    inp = dict(inp, ref=ref, cur=(cur * inp["cur_mask"]).astype(np.uint8))
    kw = dict(K=8, S=S, ssd=ssd)
    o = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], **kw)
    st, ev = gpu_check("rme", inp, o, **kw)
    ost, oev = oracle.rme(inp["cur"], inp["cur_mask"], inp["ref"], o, threads=_THREADS, **kw)
    assert np.array_equal(st, ost) and ev == oev


# ---------------------------------------------------------------------------
# Full-size configs in the bench's launch configuration, sampled rows
# ---------------------------------------------------------------------------
def _sampled_rows(H, S, rng, n_mid=2):
    rows = [(0, 2), (H - 2, H)]
    for _ in range(n_mid):
        y = int(rng.integers(S + 8, H - S - 8))
        rows.append((y, y + 1))
    return rows


@pytest.mark.parametrize("cfg", [3, 5])
def test_fullsize_u8_sampled(cfg):
    c = synth.CONFIGS[cfg]
    seq = synth.make_sequence(cfg)
    inp = synth.pair_inputs(seq, 3, 1)
    g, _ = gpu_me(inp, K=8, S=c.S, fuse=qs.make_checks())
    rng = np.random.default_rng(cfg)
    for rows in _sampled_rows(c.h, c.S, rng):
        o, _ = oracle.pair_chain(inp, K=8, S=c.S, check="nnc_frmc", rows=rows)
        assert_field_equal(g, o, rows=rows, what=f"config {cfg} rows {rows}")


def test_fullsize_config4_f32_sampled():
    c = synth.CONFIGS[4]
    seq = synth.make_sequence(4)
    inp = synth.pair_inputs(seq, 4, 3)
    g, _ = gpu_me(inp, K=8, S=c.S)
    rng = np.random.default_rng(4)
    for rows in _sampled_rows(c.h, c.S, rng, n_mid=4):
        o = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=8, S=c.S, rows=rows, threads=_THREADS)
        assert_field_equal(g, o, rows=rows, what=f"config 4 rows {rows}")


@pytest.mark.parametrize("G", [2, 4, 8])
def test_f32_row_bands_equal_full_frame_config4(G):
    """P14 for the float config that is actually sharded: config 4 at full size, cut by the bench's own
    rowband.plan_bands for G ranks; each band runs qs_me_search_refs (d = 1..3, fused cascade and PR)
    with buffers holding only band + halo rows.  The union is bit-identical to the full-frame call, and
    the rows around every cut equal the oracle's chain."""
    from paper_2203_09200_b200 import rowband
    c = synth.CONFIGS[4]
    seq = synth.make_sequence(4)
    t, S, K = 5, c.S, 8
    inps = [synth.pair_inputs(seq, t, d) for d in (1, 2, 3)]
    H, W = c.h, c.w
    prm = qs.make_params(K=K, S=S, ref_f32=True)

    def run(y0, y1, b0, b1):
        br = b1 - b0
        cur = qs.to_plane(inps[0]["cur"][b0:b1], DEV_)
        msk = qs.to_plane(inps[0]["cur_mask"][b0:b1], DEV_)
        refs = [qs.to_plane(i["ref"][b0:b1], DEV_) for i in inps]
        pvs = [qs.to_plane(i["past_val"][b0:b1], DEV_) for i in inps]
        pms = [qs.to_plane(i["past_mask"][b0:b1], DEV_) for i in inps]
        outs = [qs.Field.alloc(br, W, True, DEV_) for _ in inps]
        s, cn = qs.alloc_acc(br, W, DEV_)
        qs.qs_me_search_refs(cur, msk, refs, qs.make_roi(W, H, y0, y1, b0, br), prm, outs,
                             fuse=qs.make_checks(), project=(pvs, pms, s, cn))
        torch.cuda.synchronize()
        fs = [{k: v[y0 - b0:y1 - b0] for k, v in o.numpy().items()} for o in outs]
        return fs, s.cpu().numpy().view(np.uint32)[y0 - b0:y1 - b0], cn.cpu().numpy()[y0 - b0:y1 - b0]

    full, fsum, fcnt = run(0, H, 0, H)
    cuts = rowband.plan_bands(G, H, S, K, f32=True)
    halo = rowband.halo_rows(S, K)
    for r in range(G):
        y0, y1 = cuts[r], cuts[r + 1]
        fs, bsum, bcnt = run(y0, y1, max(0, y0 - halo), min(H, y1 + halo))
        for d, (bf, ff) in enumerate(zip(fs, full), 1):
            for k in ("alpha", "beta", "count", "status", "err"):
                a, b = bf[k], ff[k][y0:y1]
                if k == "err":
                    a, b = a.view(np.uint32), b.view(np.uint32)
                assert np.array_equal(a, b), (G, r, d, k, np.argwhere(a != b)[:5].tolist())
        assert np.array_equal(bsum, fsum[y0:y1]) and np.array_equal(bcnt, fcnt[y0:y1]), (G, r)
    # the rows around the cuts against the oracle's chain (ME -> NNC -> FRMC -> PR)
    for y in cuts[1:-1]:
        rows = (y - 2, y + 2)
        osum = np.zeros((H, W), np.uint32)
        ocnt = np.zeros((H, W), np.uint8)
        for ff, inp in zip(full, inps):
            o, _ = oracle.pair_chain(inp, K=K, S=S, check="nnc_frmc", rows=rows, threads=_THREADS)
            assert_field_equal(ff, o, rows=rows, what=f"config 4 cut {y}")
            osum, ocnt = oracle.project(o, inp["past_val"], inp["past_mask"], osum, ocnt, rows=rows)
        sl = slice(*rows)
        assert np.array_equal(fsum[sl], osum[sl]) and np.array_equal(fcnt[sl], ocnt[sl])


# ---------------------------------------------------------------------------
# Edge cases
# ---------------------------------------------------------------------------
def test_empty_roi_writes_nothing():
    inp = synth.rank_free_random_instance(5, 32, 32)
    g, ev = gpu_me(inp, K=8, S=4, rows=(10, 10), fuse=qs.make_checks(offsets=(-1, 0, 1)))
    assert ev == 0 and np.all(g["status"] == 0)


def test_tiny_frame_and_all_invalid():
    inp = synth.rank_free_random_instance(6, 2, 2)
    g, _ = gpu_me(inp, K=8, S=2)
    o = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=8, S=2)
    assert_field_equal(g, o)
    inp = synth.rank_free_random_instance(7, 20, 18)
    g, _ = gpu_me(inp, K=8, S=3, min_support=26)
    assert np.all(g["status"][inp["cur_mask"] == 0] == oracle.INVALID)


def test_row_bands_equal_full_frame():
    """Fake multi-rank: each band computed with buffers holding only band + halo rows (R25)."""
    seq = synth.make_sequence(2)
    inp = synth.pair_inputs(seq, 8, 2)
    H, W = inp["cur"].shape
    S, K = 16, 8
    full, fev = gpu_me(inp, K=K, S=S, fuse=qs.make_checks())
    G = 3
    bounds = [2 * ((r * H) // (2 * G)) for r in range(G + 1)]
    halo = S + K + 2
    out = {k: np.zeros_like(v) for k, v in full.items()}
    tot = 0
    for r in range(G):
        y0, y1 = bounds[r], bounds[r + 1]
        b0, b1 = max(0, y0 - halo), min(H, y1 + halo)
        g, ev = gpu_me(inp, K=K, S=S, fuse=qs.make_checks(), rows=(y0, y1), band=(b0, b1 - b0))
        tot += ev
        for k in out:
            out[k][y0:y1] = g[k][y0:y1]
    assert_field_equal(out, full, what="bands vs full")
    assert tot == fev


def test_abi_errors_on_device():
    inp = synth.rank_free_random_instance(8, 16, 16)
    p = {k: qs.to_plane(inp[k]) for k in ("cur", "cur_mask", "ref")}
    f = qs.Field.alloc(16, 16, False)
    roi = qs.make_roi(16, 16)
    with pytest.raises(qs.QsError) as e:
        qs.qs_me_search(p["cur"], p["cur_mask"], p["ref"], roi, qs.make_params(K=10, S=2), f)
    assert e.value.code == qs.QS_EINVAL
    with pytest.raises(qs.QsError) as e:
        qs.qs_me_search(p["cur"], p["cur_mask"], p["ref"], qs.make_roi(16, 16, 0, 16, 4, 12),
                        qs.make_params(K=8, S=2), f)
    assert e.value.code == qs.QS_EDIM
    with pytest.raises(qs.QsError) as e:
        qs.qs_frmc(p["cur"], p["cur_mask"], p["ref"], roi, qs.make_params(K=8, S=2), f, offsets=(-1, 1))
    assert e.value.code == qs.QS_EINVAL


def test_deterministic_repeat():
    seq = synth.make_sequence(2)
    inp = synth.pair_inputs(seq, 9, 1)
    a, ea = gpu_me(inp, K=8, S=16, fuse=qs.make_checks())
    b, eb = gpu_me(inp, K=8, S=16, fuse=qs.make_checks())
    assert_field_equal(a, b) and ea == eb


# ---------------------------------------------------------------------------
# Quarter-sampling body: interior and border tiles (clip-free phase, npx entry, support-plane
# phase 2), parity chunks with a partial last group (2S+1 = 15 for S = 7)
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("S,ssd,f32", [(4, False, False), (7, False, False), (7, True, False), (9, False, True),
                                       (16, False, False), (16, True, True)])
def test_quad_interior_and_border_tiles(S, ssd, f32):
    seq = synth.make_sequence(4 if f32 else 2, w=256, h=224)
    inp = synth.pair_inputs(seq, 5, 2)
    assert (inp["ref"].dtype == np.float32) == f32
    g, _ = gpu_me(inp, K=8, S=S, ssd=ssd)
    o = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=8, S=S, ssd=ssd, threads=_THREADS)
    assert_field_equal(g, o, what=f"quad S={S} ssd={ssd} f32={f32}")


# ---------------------------------------------------------------------------
# Check variants: FRMC with the {0, +-(2^k - 1)} offsets extended to a large S
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("f32", [False, True])
def test_frmc_extended_offsets(f32):
    seq = synth.make_sequence(4 if f32 else 3, w=160, h=128)
    inp = synth.pair_inputs(seq, 6, 2)
    S = 16
    offs = (-15, -7, -3, -1, 0, 1, 3, 7, 15)
    o = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=8, S=S)
    st, ev = gpu_check("frmc", inp, o, K=8, S=S, offsets=offs)
    ost, oev = oracle.frmc(inp["cur"], inp["cur_mask"], inp["ref"], o, offsets=offs, K=8, S=S)
    assert np.array_equal(st, ost) and ev == oev


# ---------------------------------------------------------------------------
# qs_me_search_refs: the d = 1..3 pairs of one frame in one launch per kernel
# ---------------------------------------------------------------------------
def _refs_call(inps, K, S, fuse, f32):
    H, W = inps[0]["cur"].shape
    cur = qs.to_plane(inps[0]["cur"], DEV_)
    msk = qs.to_plane(inps[0]["cur_mask"], DEV_)
    refs = [qs.to_plane(i["ref"], DEV_) for i in inps]
    roi = qs.make_roi(W, H)
    prm = qs.make_params(K=K, S=S, ref_f32=f32)
    outs = [qs.Field.alloc(H, W, f32, DEV_) for _ in inps]
    ev = torch.zeros(1, dtype=torch.int64, device=DEV_)
    qs.qs_me_search_refs(cur, msk, refs, roi, prm, outs, fuse=fuse, eval_count=ev)
    torch.cuda.synchronize()
    res = []
    for o in outs:
        g = o.numpy()
        if not f32:
            g["err"] = g["err"].view(np.uint32)
        res.append(g)
    return res, int(ev.item())


DEV_ = "cuda"


def test_me_search_refs_u8_bit_exact():
    seq = synth.make_sequence(2)
    t = 6
    inps = [synth.pair_inputs(seq, t, d) for d in (1, 2, 3)]
    res, ev = _refs_call(inps, 8, 16, qs.make_checks(), False)
    oev_sum = 0
    for d, (g, inp) in enumerate(zip(res, inps), 1):
        o, oev = oracle.pair_chain(inp, K=8, S=16, check="nnc_frmc")
        assert_field_equal(g, o, what=f"refs c2 t={t} d={d}")
        oev_sum += oev
    assert ev == oev_sum


def test_me_search_refs_f32_equals_single_calls():
    seq = synth.make_sequence(4, w=256, h=224)
    inps = [synth.pair_inputs(seq, 5, d) for d in (1, 2, 3)]
    res, ev = _refs_call(inps, 8, 9, qs.make_checks(), True)
    ev_sum = 0
    for g, inp in zip(res, inps):
        s, sev = gpu_me(inp, K=8, S=9, fuse=qs.make_checks())
        for k in ("alpha", "beta", "count", "status"):
            assert np.array_equal(g[k], s[k]), k
        assert np.array_equal(g["err"].view(np.uint32), s["err"].view(np.uint32))
        ev_sum += sev
    assert ev == ev_sum


def test_me_search_refs_groups_and_fallback():
    # 5 references -> two launches (groups of 4); K = 9 -> the slot-by-slot path; n_refs = 0 -> no-op
    seq = synth.make_sequence(1)
    inps = [synth.pair_inputs(seq, 2, d) for d in (1, 2, 1, 2, 1)]
    res, ev = _refs_call(inps, 8, 8, qs.make_checks(), False)
    oev_sum = 0
    for g, inp in zip(res, inps):
        o, oev = oracle.pair_chain(inp, K=8, S=8, check="nnc_frmc")
        assert_field_equal(g, o, what="refs groups")
        oev_sum += oev
    assert ev == oev_sum
    res9, _ = _refs_call(inps[:2], 9, 4, None, False)
    for g, inp in zip(res9, inps[:2]):
        o = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=9, S=4)
        assert_field_equal(g, o, what="refs K=9")
    H, W = inps[0]["cur"].shape
    cur = qs.to_plane(inps[0]["cur"], DEV_)
    qs.qs_me_search_refs(cur, cur, [], qs.make_roi(W, H), qs.make_params(K=8, S=8), [])


def test_me_search_refs_fused_projection_bit_exact():
    # ME + NNC -> FRMC + PR of a frame's three references in one call vs the oracle's chain; then the
    # slot-by-slot path (K = 9, no checks -> no ACCEPTED entries) leaves the accumulators untouched.
    seq = synth.make_sequence(2)
    t = 7
    inps = [synth.pair_inputs(seq, t, d) for d in (1, 2, 3)]
    H, W = inps[0]["cur"].shape
    cur = qs.to_plane(inps[0]["cur"], DEV_)
    msk = qs.to_plane(inps[0]["cur_mask"], DEV_)
    refs = [qs.to_plane(i["ref"], DEV_) for i in inps]
    pvs = [qs.to_plane(i["past_val"], DEV_) for i in inps]
    pms = [qs.to_plane(i["past_mask"], DEV_) for i in inps]
    roi = qs.make_roi(W, H)
    outs = [qs.Field.alloc(H, W, False, DEV_) for _ in inps]
    s, c = qs.alloc_acc(H, W, DEV_)
    qs.qs_me_search_refs(cur, msk, refs, roi, qs.make_params(K=8, S=16), outs, fuse=qs.make_checks(),
                         project=(pvs, pms, s, c))
    torch.cuda.synchronize()
    osum = np.zeros((H, W), np.uint32)
    ocnt = np.zeros((H, W), np.uint8)
    for o_f, inp in zip(outs, inps):
        o, _ = oracle.pair_chain(inp, K=8, S=16, check="nnc_frmc")
        g = o_f.numpy()
        g["err"] = g["err"].view(np.uint32)
        assert_field_equal(g, o, what="refs+PR")
        osum, ocnt = oracle.project(o, inp["past_val"], inp["past_mask"], osum, ocnt)
    assert int(ocnt.sum()) > 0
    assert np.array_equal(s.cpu().numpy().view(np.uint32), osum) and np.array_equal(c.cpu().numpy(), ocnt)
    s0, c0 = s.clone(), c.clone()
    qs.qs_me_search_refs(cur, msk, refs[:2], roi, qs.make_params(K=9, S=4), outs[:2], project=(pvs[:2], pms[:2], s, c))
    torch.cuda.synchronize()
    assert torch.equal(s, s0) and torch.equal(c, c0)



# ---------------------------------------------------------------------------
# NNC's second reading (R30): standalone on the hand-worked fixtures, and fused
# into qs_me_search (NNC(pairs) -> FRMC cascade) against the oracle's chain
# ---------------------------------------------------------------------------
def test_nnc_pairs_golden_on_gpu(golden):
    g = golden("nnc_pairs_hand.json")
    for case in g["cases"]:
        a = np.array(case["alpha"], np.int8)
        H, W = a.shape
        Hp, Wp = H + H % 2, W + W % 2
        fld = {k: np.zeros((Hp, Wp), dt) for k, dt in (("alpha", np.int8), ("beta", np.int8), ("err", np.uint32),
                                                        ("count", np.uint8), ("status", np.uint8))}
        fld["alpha"][:H, :W] = a
        fld["beta"][:H, :W] = np.array(case["beta"], np.int8)
        fld["status"][:H, :W] = np.array(case["status"], np.uint8)
        inp = dict(cur=np.zeros((Hp, Wp), np.uint8), cur_mask=np.zeros((Hp, Wp), np.uint8),
                   ref=np.zeros((Hp, Wp), np.uint8), past_val=np.zeros((Hp, Wp), np.uint8),
                   past_mask=np.zeros((Hp, Wp), np.uint8))
        for kind, key in (("nnc", "expect_centre"), ("nnc_pairs", "expect_pairs")):
            st, _ = gpu_check(kind, inp, fld)
            assert np.array_equal(st[:H, :W], np.array(case[key], np.uint8)), (case["name"], kind)


@pytest.mark.parametrize("cfg,S", [(2, 16), (4, 9)])
def test_nnc_pairs_cascade_fused(cfg, S):
    seq = synth.make_sequence(cfg, w=192 if cfg == 4 else None, h=160 if cfg == 4 else None)
    inp = synth.pair_inputs(seq, 6, 1)
    g, gev = gpu_me(inp, K=8, S=S, fuse=qs.make_checks(nnc_pairs=True))
    o = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=8, S=S)
    if cfg == 4:   # float reference: decide the checks on the GPU's own field (staged parity, R23)
        o = {k: g[k].copy() for k in g}
        o["status"] = np.where(g["status"] >= oracle.CANDIDATE, oracle.CANDIDATE, g["status"]).astype(np.uint8)
    o["status"] = oracle.nnc(o, 1, pairs=True)
    o["status"], oev = oracle.frmc(inp["cur"], inp["cur_mask"], inp["ref"], o, K=8, S=S)
    assert np.array_equal(g["status"], o["status"])
    assert gev == oev
    if cfg == 2:
        assert_field_equal(g, o, what="nnc pairs cascade")


def test_me_search_refs_row_bands_with_projection():
    """The multi-GPU step on one device: each row band runs qs_me_search_refs (three references, fused
    PR) with buffers holding only band + halo rows; the union equals the full-frame oracle chain."""
    seq = synth.make_sequence(2)
    t, S, K = 9, 16, 8
    inps = [synth.pair_inputs(seq, t, d) for d in (1, 2, 3)]
    H, W = inps[0]["cur"].shape
    G = 2
    bounds = [2 * ((r * H) // (2 * G)) for r in range(G + 1)]
    halo = S + K + 2
    gsum = np.zeros((H, W), np.uint32)
    gcnt = np.zeros((H, W), np.uint8)
    fields = [{k: None for k in ("alpha", "beta", "err", "count", "status")} for _ in inps]
    for r in range(G):
        y0, y1 = bounds[r], bounds[r + 1]
        b0, b1 = max(0, y0 - halo), min(H, y1 + halo)
        br = b1 - b0
        cur = qs.to_plane(inps[0]["cur"][b0:b1], DEV_)
        msk = qs.to_plane(inps[0]["cur_mask"][b0:b1], DEV_)
        refs = [qs.to_plane(i["ref"][b0:b1], DEV_) for i in inps]
        pvs = [qs.to_plane(i["past_val"][b0:b1], DEV_) for i in inps]
        pms = [qs.to_plane(i["past_mask"][b0:b1], DEV_) for i in inps]
        outs = [qs.Field.alloc(br, W, False, DEV_) for _ in inps]
        s, c = qs.alloc_acc(br, W, DEV_)
        qs.qs_me_search_refs(cur, msk, refs, qs.make_roi(W, H, y0, y1, b0, br), qs.make_params(K=K, S=S), outs,
                             fuse=qs.make_checks(), project=(pvs, pms, s, c))
        torch.cuda.synchronize()
        gsum[y0:y1] = s.cpu().numpy().view(np.uint32)[y0 - b0:y1 - b0]
        gcnt[y0:y1] = c.cpu().numpy()[y0 - b0:y1 - b0]
        for f, o in zip(fields, outs):
            g = o.numpy()
            g["err"] = g["err"].view(np.uint32)
            for k in f:
                if f[k] is None:
                    f[k] = np.zeros((H, W), g[k].dtype)
                f[k][y0:y1] = g[k][y0 - b0:y1 - b0]
    osum = np.zeros((H, W), np.uint32)
    ocnt = np.zeros((H, W), np.uint8)
    for f, inp in zip(fields, inps):
        o, _ = oracle.pair_chain(inp, K=K, S=S, check="nnc_frmc")
        assert_field_equal(f, o, what="refs bands")
        osum, ocnt = oracle.project(o, inp["past_val"], inp["past_mask"], osum, ocnt)
    assert np.array_equal(gsum, osum) and np.array_equal(gcnt, ocnt)


@pytest.mark.parametrize("cfg,ssd", [(3, False), (2, True)])
def test_me_search_refs_fixed_mask_and_ssd(cfg, ssd):
    """qs_me_search_refs on a fixed-mask config and with SSD (the generic phase-2 body for uint8 SSD)
    against the oracle's chain, reference by reference."""
    seq = synth.make_sequence(cfg, w=160, h=128)
    inps = [synth.pair_inputs(seq, 5, d) for d in (1, 2, 3)]
    H, W = inps[0]["cur"].shape
    cur = qs.to_plane(inps[0]["cur"], DEV_)
    msk = qs.to_plane(inps[0]["cur_mask"], DEV_)
    refs = [qs.to_plane(i["ref"], DEV_) for i in inps]
    outs = [qs.Field.alloc(H, W, False, DEV_) for _ in inps]
    ev = torch.zeros(1, dtype=torch.int64, device=DEV_)
    S = 9
    qs.qs_me_search_refs(cur, msk, refs, qs.make_roi(W, H), qs.make_params(K=8, S=S, ssd=ssd), outs,
                         fuse=qs.make_checks(), eval_count=ev)
    torch.cuda.synchronize()
    oev = 0
    for o_f, inp in zip(outs, inps):
        o, e = oracle.pair_chain(inp, K=8, S=S, ssd=ssd, check="nnc_frmc")
        g = o_f.numpy()
        g["err"] = g["err"].view(np.uint32)
        assert_field_equal(g, o, what=f"refs cfg{cfg} ssd={ssd}")
        oev += e
    assert int(ev.item()) == oev


def test_fullsize_config4_bench_launch_sampled():
    """The launch bench.py times: config 4 at full size, qs_me_search_refs over d = 1..3 with the fused
    NNC -> FRMC cascade and fused PR.  Sampled rows (frame edges + interior): every plane bit-exact
    against the oracle's chain, sum / cnt equal."""
    c = synth.CONFIGS[4]
    seq = synth.make_sequence(4)
    t = 4
    inps = [synth.pair_inputs(seq, t, d) for d in (1, 2, 3)]
    H, W = c.h, c.w
    cur = qs.to_plane(inps[0]["cur"], DEV_)
    msk = qs.to_plane(inps[0]["cur_mask"], DEV_)
    refs = [qs.to_plane(i["ref"], DEV_) for i in inps]
    pvs = [qs.to_plane(i["past_val"], DEV_) for i in inps]
    pms = [qs.to_plane(i["past_mask"], DEV_) for i in inps]
    outs = [qs.Field.alloc(H, W, True, DEV_) for _ in inps]
    s, cn = qs.alloc_acc(H, W, DEV_)
    qs.qs_me_search_refs(cur, msk, refs, qs.make_roi(W, H), qs.make_params(K=8, S=c.S, ref_f32=True), outs,
                         fuse=qs.make_checks(), project=(pvs, pms, s, cn))
    torch.cuda.synchronize()
    gsum, gcnt = s.cpu().numpy().view(np.uint32), cn.cpu().numpy()
    gf = [o.numpy() for o in outs]
    rng = np.random.default_rng(44)
    for rows in _sampled_rows(H, c.S, rng, n_mid=3):
        osum = np.zeros((H, W), np.uint32)
        ocnt = np.zeros((H, W), np.uint8)
        for g, inp in zip(gf, inps):
            o, _ = oracle.pair_chain(inp, K=8, S=c.S, check="nnc_frmc", rows=rows, threads=_THREADS)
            assert_field_equal(g, o, rows=rows, what=f"config 4 refs rows {rows}")
            osum, ocnt = oracle.project(o, inp["past_val"], inp["past_mask"], osum, ocnt, rows=rows)
        sl = slice(*rows)
        assert np.array_equal(gsum[sl], osum[sl]) and np.array_equal(gcnt[sl], ocnt[sl]), rows


def test_fullsize_config4_full_frame_bit_exact():
    """One whole config-4 frame (t = 5, all three references, 1.56 M targets each) in the bench's
    launch against the oracle's chain over EVERY row (OpenMP row driver): zero differences in every
    plane and in sum / cnt."""
    c = synth.CONFIGS[4]
    seq = synth.make_sequence(4)
    t = 5
    inps = [synth.pair_inputs(seq, t, d) for d in (1, 2, 3)]
    H, W = c.h, c.w
    cur = qs.to_plane(inps[0]["cur"], DEV_)
    msk = qs.to_plane(inps[0]["cur_mask"], DEV_)
    refs = [qs.to_plane(i["ref"], DEV_) for i in inps]
    pvs = [qs.to_plane(i["past_val"], DEV_) for i in inps]
    pms = [qs.to_plane(i["past_mask"], DEV_) for i in inps]
    outs = [qs.Field.alloc(H, W, True, DEV_) for _ in inps]
    s, cn = qs.alloc_acc(H, W, DEV_)
    ev = torch.zeros(1, dtype=torch.int64, device=DEV_)
    qs.qs_me_search_refs(cur, msk, refs, qs.make_roi(W, H), qs.make_params(K=8, S=c.S, ref_f32=True), outs,
                         fuse=qs.make_checks(), project=(pvs, pms, s, cn), eval_count=ev)
    torch.cuda.synchronize()
    osum = np.zeros((H, W), np.uint32)
    ocnt = np.zeros((H, W), np.uint8)
    oev = 0
    for d, (o_f, inp) in enumerate(zip(outs, inps), 1):
        o, e = oracle.pair_chain(inp, K=8, S=c.S, check="nnc_frmc", threads=_THREADS)
        assert_field_equal(o_f.numpy(), o, what=f"config 4 full frame d={d}")
        osum, ocnt = oracle.project(o, inp["past_val"], inp["past_mask"], osum, ocnt)
        oev += e
    assert np.array_equal(s.cpu().numpy().view(np.uint32), osum) and np.array_equal(cn.cpu().numpy(), ocnt)
    assert int(ev.item()) == oev


@pytest.mark.parametrize("cfg", [3, 5])
def test_fullsize_u8_bench_launch_sampled(cfg):
    """The bench's launch on the uint8 configs at full size: qs_me_search_refs over d = 1..3 with the
    fused cascade and PR, bit-exact against the oracle's chain on sampled rows."""
    c = synth.CONFIGS[cfg]
    seq = synth.make_sequence(cfg)
    t = 3
    inps = [synth.pair_inputs(seq, t, d) for d in (1, 2, 3)]
    H, W = c.h, c.w
    cur = qs.to_plane(inps[0]["cur"], DEV_)
    msk = qs.to_plane(inps[0]["cur_mask"], DEV_)
    refs = [qs.to_plane(i["ref"], DEV_) for i in inps]
    pvs = [qs.to_plane(i["past_val"], DEV_) for i in inps]
    pms = [qs.to_plane(i["past_mask"], DEV_) for i in inps]
    outs = [qs.Field.alloc(H, W, False, DEV_) for _ in inps]
    s, cn = qs.alloc_acc(H, W, DEV_)
    qs.qs_me_search_refs(cur, msk, refs, qs.make_roi(W, H), qs.make_params(K=8, S=c.S), outs,
                         fuse=qs.make_checks(), project=(pvs, pms, s, cn))
    torch.cuda.synchronize()
    gsum, gcnt = s.cpu().numpy().view(np.uint32), cn.cpu().numpy()
    gf = []
    for o in outs:
        g = o.numpy()
        g["err"] = g["err"].view(np.uint32)
        gf.append(g)
    rng = np.random.default_rng(cfg + 100)
    for rows in _sampled_rows(H, c.S, rng, n_mid=1):
        osum = np.zeros((H, W), np.uint32)
        ocnt = np.zeros((H, W), np.uint8)
        for g, inp in zip(gf, inps):
            o, _ = oracle.pair_chain(inp, K=8, S=c.S, check="nnc_frmc", rows=rows)
            assert_field_equal(g, o, rows=rows, what=f"config {cfg} refs rows {rows}")
            osum, ocnt = oracle.project(o, inp["past_val"], inp["past_mask"], osum, ocnt, rows=rows)
        sl = slice(*rows)
        assert np.array_equal(gsum[sl], osum[sl]) and np.array_equal(gcnt[sl], ocnt[sl]), rows


@pytest.mark.parametrize("K,f32", [(8, False), (8, True), (7, False)])
def test_adjacent_rois_share_one_field(K, f32):
    """Two adjacent rois with the fused NNC -> FRMC cascade write into ONE full-frame field, on two
    streams: each call writes only its own rows (the NNC halo vectors stay in its workspace), so the
    result equals the whole-frame call and the oracle (include/qs.h qs_me_search `fuse`)."""
    seq = synth.make_sequence(4 if f32 else 2, w=192, h=160)
    inp = synth.pair_inputs(seq, 6, 1)
    H, W = inp["cur"].shape
    S = 9
    p = {k: qs.to_plane(inp[k], DEV_) for k in ("cur", "cur_mask", "ref")}
    prm = qs.make_params(K=K, S=S, ref_f32=f32)
    f = qs.Field.alloc(H, W, f32, DEV_)
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    cut = 78
    for (y0, y1), st in zip(((0, cut), (cut, H)), streams):
        with torch.cuda.stream(st):
            qs.qs_me_search(p["cur"], p["cur_mask"], p["ref"], qs.make_roi(W, H, y0, y1), prm, f,
                            fuse=qs.make_checks(), stream=st)
    torch.cuda.synchronize()
    g = f.numpy()
    if not f32:
        g["err"] = g["err"].view(np.uint32)
    o, _ = oracle.pair_chain(inp, K=K, S=S, check="nnc_frmc", threads=_THREADS)
    assert_field_equal(g, o, what=f"adjacent rois K={K} f32={f32}")


@pytest.mark.parametrize("cfg", [2, 4])
def test_projection_only_mode(cfg):
    """qs_me_search_refs with outs = NULL: only sum / cnt are written, and
    they equal the oracle's chain + PR over the three references."""
    c = synth.CONFIGS[cfg]
    seq = synth.make_sequence(cfg, w=256, h=160)
    t, S = 6, min(c.S, 16)
    inps = [synth.pair_inputs(seq, t, d) for d in (1, 2, 3)]
    H, W = inps[0]["cur"].shape
    cur = qs.to_plane(inps[0]["cur"], DEV_)
    msk = qs.to_plane(inps[0]["cur_mask"], DEV_)
    refs = [qs.to_plane(i["ref"], DEV_) for i in inps]
    pvs = [qs.to_plane(i["past_val"], DEV_) for i in inps]
    pms = [qs.to_plane(i["past_mask"], DEV_) for i in inps]
    s, cn = qs.alloc_acc(H, W, DEV_)
    ev = torch.zeros(1, dtype=torch.int64, device=DEV_)
    qs.qs_me_search_refs(cur, msk, refs, qs.make_roi(W, H), qs.make_params(K=8, S=S, ref_f32=c.ref_f32), None,
                         fuse=qs.make_checks(), project=(pvs, pms, s, cn), eval_count=ev)
    torch.cuda.synchronize()
    osum = np.zeros((H, W), np.uint32)
    ocnt = np.zeros((H, W), np.uint8)
    oev = 0
    for inp in inps:
        o, e = oracle.pair_chain(inp, K=8, S=S, check="nnc_frmc", threads=_THREADS)
        osum, ocnt = oracle.project(o, inp["past_val"], inp["past_mask"], osum, ocnt)
        oev += e
    assert np.array_equal(s.cpu().numpy().view(np.uint32), osum) and np.array_equal(cn.cpu().numpy(), ocnt)
    assert int(ev.item()) == oev
    with pytest.raises(qs.QsError):   # projection-only needs the fused K = 8 path
        qs.qs_me_search_refs(cur, msk, refs, qs.make_roi(W, H), qs.make_params(K=7, S=S, ref_f32=c.ref_f32), None,
                             fuse=qs.make_checks(), project=(pvs, pms, s, cn))


@pytest.mark.parametrize("env,val,f32", [("QS_TMA", "1", True), ("QS_U8_BODY", "float", False),
                                         ("QS_SPLIT", "0", True), ("QS_SPLIT", "2", True)])
def test_staging_and_body_variants_bit_exact(env, val, f32, monkeypatch):
    """The measured alternatives stay exact: TMA staging of the float window (QS_TMA=1), the fp32
    body for uint8 interior tiles (QS_U8_BODY=float), and for float references me_box as one kernel
    (QS_SPLIT=0) or as border / interior grids over the whole tile grid (QS_SPLIT=2) instead of the
    default interior rectangle give the oracle's planes, interior and border."""
    monkeypatch.setenv(env, val)
    seq = synth.make_sequence(4 if f32 else 2, w=320, h=256)
    for t, d in ((5, 1), (6, 3)):
        inp = synth.pair_inputs(seq, t, d)
        g, gev = gpu_me(inp, K=8, S=16, fuse=qs.make_checks())
        o, oev = oracle.pair_chain(inp, K=8, S=16, check="nnc_frmc", threads=_THREADS)
        assert_field_equal(g, o, what=f"{env}={val} t={t} d={d}")
        assert gev == oev


@pytest.mark.parametrize("G", [2, 4])
def test_u8_row_bands_equal_full_frame_config5(G):
    """P14 on the 4K config (S = 32, halo 38 rows): sequence 0 of config 5 at full size cut by
    rowband.plan_bands; each band runs qs_me_search_refs (d = 1..3, fused cascade and PR) with buffers
    holding only band + halo rows.  The union equals the full-frame call bit for bit; the rows at each
    cut equal the oracle's chain."""
    from paper_2203_09200_b200 import rowband
    c = synth.CONFIGS[5]
    seq = synth.make_sequence(5)
    t, S, K = 5, c.S, 8
    inps = [synth.pair_inputs(seq, t, d) for d in (1, 2, 3)]
    H, W = c.h, c.w
    prm = qs.make_params(K=K, S=S)

    def run(y0, y1, b0, b1):
        br = b1 - b0
        cur = qs.to_plane(inps[0]["cur"][b0:b1], DEV_)
        msk = qs.to_plane(inps[0]["cur_mask"][b0:b1], DEV_)
        refs = [qs.to_plane(i["ref"][b0:b1], DEV_) for i in inps]
        pvs = [qs.to_plane(i["past_val"][b0:b1], DEV_) for i in inps]
        pms = [qs.to_plane(i["past_mask"][b0:b1], DEV_) for i in inps]
        outs = [qs.Field.alloc(br, W, False, DEV_) for _ in inps]
        s, cn = qs.alloc_acc(br, W, DEV_)
        qs.qs_me_search_refs(cur, msk, refs, qs.make_roi(W, H, y0, y1, b0, br), prm, outs,
                             fuse=qs.make_checks(), project=(pvs, pms, s, cn))
        torch.cuda.synchronize()
        fs = []
        for o in outs:
            g = o.numpy()
            g["err"] = g["err"].view(np.uint32)
            fs.append({k: v[y0 - b0:y1 - b0] for k, v in g.items()})
        return fs, s.cpu().numpy().view(np.uint32)[y0 - b0:y1 - b0], cn.cpu().numpy()[y0 - b0:y1 - b0]

    full, fsum, fcnt = run(0, H, 0, H)
    cuts = rowband.plan_bands(G, H, S, K)
    halo = rowband.halo_rows(S, K)
    assert halo == 38
    for r in range(G):
        y0, y1 = cuts[r], cuts[r + 1]
        fs, bsum, bcnt = run(y0, y1, max(0, y0 - halo), min(H, y1 + halo))
        for d, (bf, ff) in enumerate(zip(fs, full), 1):
            for k in ("alpha", "beta", "count", "status", "err"):
                assert np.array_equal(bf[k], ff[k][y0:y1]), (G, r, d, k)
        assert np.array_equal(bsum, fsum[y0:y1]) and np.array_equal(bcnt, fcnt[y0:y1]), (G, r)
    for y in cuts[1:-1]:
        rows = (y - 1, y + 1)
        for ff, inp in zip(full, inps):
            o, _ = oracle.pair_chain(inp, K=K, S=S, check="nnc_frmc", rows=rows, threads=_THREADS)
            assert_field_equal(ff, o, rows=rows, what=f"config 5 cut {y}")


@pytest.mark.parametrize("cfg,ds", [(3, (1, 2, 3))])
def test_fullsize_u8_full_frame_bit_exact(cfg, ds):
    """A whole frame of config 3 in the bench's launch (qs_me_search_refs, fused cascade and PR; the
    integer interior body and the exact fp32 border body) against the oracle's chain over every row and
    all three references.  (A config-5 frame is ~8 min of 16-core oracle time per reference; config 5
    is checked on sampled rows, frame edges and the row-band cuts.)"""
    c = synth.CONFIGS[cfg]
    seq = synth.make_sequence(cfg)
    t = 5
    inps = [synth.pair_inputs(seq, t, d) for d in ds]
    H, W = c.h, c.w
    cur = qs.to_plane(inps[0]["cur"], DEV_)
    msk = qs.to_plane(inps[0]["cur_mask"], DEV_)
    refs = [qs.to_plane(i["ref"], DEV_) for i in inps]
    pvs = [qs.to_plane(i["past_val"], DEV_) for i in inps]
    pms = [qs.to_plane(i["past_mask"], DEV_) for i in inps]
    outs = [qs.Field.alloc(H, W, False, DEV_) for _ in inps]
    s, cn = qs.alloc_acc(H, W, DEV_)
    ev = torch.zeros(1, dtype=torch.int64, device=DEV_)
    qs.qs_me_search_refs(cur, msk, refs, qs.make_roi(W, H), qs.make_params(K=8, S=c.S), outs,
                         fuse=qs.make_checks(), project=(pvs, pms, s, cn), eval_count=ev)
    torch.cuda.synchronize()
    osum = np.zeros((H, W), np.uint32)
    ocnt = np.zeros((H, W), np.uint8)
    oev = 0
    for d, (o_f, inp) in zip(ds, zip(outs, inps)):
        g = o_f.numpy()
        g["err"] = g["err"].view(np.uint32)
        o, e = oracle.pair_chain(inp, K=8, S=c.S, check="nnc_frmc", threads=_THREADS)
        assert_field_equal(g, o, what=f"config {cfg} full frame d={d}")
        osum, ocnt = oracle.project(o, inp["past_val"], inp["past_mask"], osum, ocnt)
        oev += e
    assert np.array_equal(s.cpu().numpy().view(np.uint32), osum) and np.array_equal(cn.cpu().numpy(), ocnt)
    assert int(ev.item()) == oev
