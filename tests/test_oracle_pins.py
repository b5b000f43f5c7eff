"""Pins that tie the CPU oracle to the paper and to mathematics (not to itself).

Each test names the pin of DESIGN.md "Oracle pins" and the
passage it follows.  CPU only (no GPU marker).
"""
import numpy as np
import pytest

import oracle
from oracle import twin
from oracle import NOT_TARGET, INVALID, CANDIDATE, ACCEPTED, REJECTED
import synth

STATUS = {"ACCEPTED": ACCEPTED, "REJECTED": REJECTED}


def _arr(x, dt):
    return np.array(x, dtype=dt)


# ---------------------------------------------------------------------------
# Rank order (R7)
# ---------------------------------------------------------------------------
def test_rank_order_l1_one():
    a, b = oracle.rank_list(1)
    got = list(zip(a.tolist(), b.tolist()))
    # (|a|+|b|, a, b) ascending: (0,0); then L1=1: (-1,0) < (0,-1) < (0,1) < (1,0); then L1=2 by a, b.
    assert got == [(0, 0), (-1, 0), (0, -1), (0, 1), (1, 0), (-1, -1), (-1, 1), (1, -1), (1, 1)]


def test_rank_order_counts_and_twin():
    for S in (1, 2, 8, 24, 32):
        a, b = oracle.rank_list(S)
        assert a.size == (2 * S + 1) ** 2
        ta, tb = twin.rank_order(S)
        assert np.array_equal(a, ta) and np.array_equal(b, tb)


# ---------------------------------------------------------------------------
# P13: hand-worked micro example, golden file
# ---------------------------------------------------------------------------
def test_p13_micro_golden(golden):
    g = golden("p13_micro.json")
    cur = _arr(g["cur"], np.uint8)
    mask = _arr(g["mask"], np.uint8)
    ref = _arr(g["ref"], np.uint8)
    f = oracle.me_search(cur, mask, ref, K=g["K"], S=g["S"], min_support=g["min_support"])
    for ex in g["expect"]:
        y, x = ex["p"]
        assert f["status"][y, x] == CANDIDATE
        assert (int(f["alpha"][y, x]), int(f["beta"][y, x])) == tuple(ex["v"]), ex
        assert int(f["err"][y, x]) == ex["e"] and int(f["count"][y, x]) == ex["n"]
        # Every admissible candidate's (e, n) as worked by hand.
        for key, (e, n) in ex["candidates"].items():
            a, b = map(int, key.split(","))
            assert oracle.cost_fwd(cur, mask, ref, y, x, a, b, K=g["K"], min_support=1) == (e, n), (ex["p"], key)
        # Candidates not listed leave the frame: n = 0.
        for a in (-1, 0, 1):
            for b in (-1, 0, 1):
                if f"{a},{b}" not in ex["candidates"]:
                    assert oracle.cost_fwd(cur, mask, ref, y, x, a, b, K=g["K"], min_support=1)[1] == 0
    # Measured pixels are not targets (R4).
    assert np.all(f["status"][mask == 1] == NOT_TARGET)


def test_frmc_rme_micro_golden(golden):
    g0 = golden("p13_micro.json")
    g = golden("frmc_rme_micro.json")
    cur = _arr(g0["cur"], np.uint8)
    mask = _arr(g0["mask"], np.uint8)
    ref = _arr(g0["ref"], np.uint8)
    for case in g["cases"]:
        y, x = case["p"]
        a, b = case["v"]
        # Reverse costs rc(x = p+v, u = -v + delta), worked by hand.
        for key, (e, n) in case["rc_delta"].items():
            dy, dx = map(int, key.split(","))
            assert oracle.cost_rev(cur, mask, ref, y + a, x + b, -a + dy, -b + dx, K=2, min_support=1) == (e, n)
        field = dict(alpha=np.zeros((4, 4), np.int8), beta=np.zeros((4, 4), np.int8),
                     err=np.zeros((4, 4), np.uint32), count=np.zeros((4, 4), np.uint8),
                     status=np.zeros((4, 4), np.uint8))
        field["alpha"][y, x], field["beta"][y, x] = a, b
        field["err"][y, x], field["count"][y, x] = case["e"], case["n"]
        field["status"][y, x] = CANDIDATE
        st, ev = oracle.frmc(cur, mask, ref, field, offsets=g["offsets"], K=2, S=1, min_support=1)
        assert st[y, x] == STATUS[case["frmc"]] and ev == 9
        st, ev = oracle.rmc(cur, mask, ref, field, K=2, S=1, min_support=1)
        assert st[y, x] == STATUS[case["frmc"]] and ev == 9     # O = [-S, S] here, so RMC == FRMC
        if "rme" in case:
            st, ev = oracle.rme(cur, mask, ref, field, K=2, S=1, min_support=1)
            assert st[y, x] == STATUS[case["rme"]] and ev == 9
        # Only the checked entry changed.
        others = np.ones((4, 4), bool)
        others[y, x] = False
        assert np.all(st[others] == field["status"][others])


# ---------------------------------------------------------------------------
# P7: NNC hand-worked fixtures (Eq. 1)
# ---------------------------------------------------------------------------
def test_p7_nnc_golden(golden):
    g = golden("nnc_hand.json")
    for case in g["cases"]:
        f = dict(alpha=_arr(case["alpha"], np.int8), beta=_arr(case["beta"], np.int8),
                 status=_arr(case["status"], np.uint8))
        fa, fb, d = oracle.median_field(f)
        if "filtered_alpha" in case:
            m = d == 1
            assert np.array_equal(fa[m], _arr(case["filtered_alpha"], np.int32)[m]), case["name"]
        if "filtered_beta" in case:
            m = d == 1
            assert np.array_equal(fb[m], _arr(case["filtered_beta"], np.int32)[m]), case["name"]
        st = oracle.nnc(f, threshold=1)
        assert np.array_equal(st, _arr(case["expect"], np.uint8)), case["name"]
        # twin agrees
        tst = twin.nnc(f["alpha"], f["beta"], f["status"], 1)
        assert np.array_equal(tst, st), case["name"]


def test_p7_nnc_idempotent_and_checks_do_not_touch_vectors():
    inp = synth.rank_free_random_instance(7, 24, 24, smooth=True)
    f = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=8, S=3)
    before = {k: v.copy() for k, v in f.items()}
    st1 = oracle.nnc(f)
    f2 = dict(f, status=st1)
    st2 = oracle.nnc(f2)
    assert np.array_equal(st1, st2)                  # idempotent
    for k in ("alpha", "beta", "err", "count"):
        assert np.array_equal(f[k], before[k])       # checks never alter (a, b, e, n)
    # Only CANDIDATE entries changed, and only to ACCEPTED/REJECTED.
    ch = st1 != before["status"]
    assert np.all(before["status"][ch] == CANDIDATE)
    assert np.all(np.isin(st1[ch], [ACCEPTED, REJECTED]))


# ---------------------------------------------------------------------------
# P9: projection
# ---------------------------------------------------------------------------
def test_p9_project_golden(golden):
    g = golden("project_hand.json")
    pm = _arr(g["past_mask"], np.uint8)
    s = np.zeros((4, 4), np.uint32)
    c = np.zeros((4, 4), np.uint8)
    for r in g["refs"]:
        f = dict(alpha=_arr(r["alpha"], np.int8), beta=_arr(r["beta"], np.int8), status=_arr(r["status"], np.uint8))
        s, c = oracle.project(f, _arr(r["past_val"], np.uint8), pm, s, c)
    assert np.array_equal(s, _arr(g["expect_sum"], np.uint32))
    assert np.array_equal(c, _arr(g["expect_cnt"], np.uint8))
    assert s[1, 1] / c[1, 1] == 15.0                 # "these are averaged" -> 10 and 20 give 15


def test_p9_project_order_independent_and_bounded():
    seq = synth.make_sequence(2, w=64, h=48)
    fields, pasts = [], []
    for d in (1, 2, 3):
        inp = synth.pair_inputs(seq, 6, d)
        f, _ = oracle.pair_chain(inp, K=8, S=8, check="nnc")
        fields.append(f)
        pasts.append((inp["past_val"], inp["past_mask"]))
    outs = []
    for order in ((0, 1, 2), (2, 0, 1)):
        s = np.zeros((48, 64), np.uint32)
        c = np.zeros((48, 64), np.uint8)
        lo = np.full((48, 64), 255)
        hi = np.zeros((48, 64), int)
        for i in order:
            s1, c1 = oracle.project(fields[i], *pasts[i])
            s, c = oracle.project(fields[i], *pasts[i], s, c)
            ts, tc = twin.project(fields[i]["alpha"], fields[i]["beta"], fields[i]["status"], *pasts[i])
            assert np.array_equal(ts, s1) and np.array_equal(tc, c1)
            m = c1 > 0
            lo[m] = np.minimum(lo[m], s1[m])
            hi[m] = np.maximum(hi[m], s1[m])
        outs.append((s, c))
        m = c > 0
        mean = s[m] / c[m]
        assert np.all(mean >= lo[m]) and np.all(mean <= hi[m])
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


def test_p9_static_scene_dynamic_mask_full_coverage():
    # Static scene + dynamic mask + zero motion, t >= 3: each missing pixel was
    # measured in one of the 3 previous frames, so it receives >= 1 projection.
    rng = np.random.default_rng(3)
    g = rng.integers(0, 256, (32, 32)).astype(np.uint8)
    masks = [synth.quarter_mask(32, 32, 99, True, t) for t in range(4)]
    s = np.zeros((32, 32), np.uint32)
    c = np.zeros((32, 32), np.uint8)
    for d in (1, 2, 3):
        f = dict(alpha=np.zeros((32, 32), np.int8), beta=np.zeros((32, 32), np.int8),
                 status=np.where(masks[3] == 1, NOT_TARGET, ACCEPTED).astype(np.uint8))
        s, c = oracle.project(f, g * masks[3 - d], masks[3 - d], s, c)
    assert np.all(c[masks[3] == 0] == 1)
    assert np.array_equal(s[masks[3] == 0], g[masks[3] == 0])


# ---------------------------------------------------------------------------
# P1, P2: identity and constant frames
# ---------------------------------------------------------------------------
def test_p1_zero_motion_identity():
    inp = synth.rank_free_random_instance(11, 40, 40, smooth=True)
    g = inp["dense_cur"]
    m = inp["cur_mask"]
    cur = g * m
    S, K = 4, 8
    f = oracle.me_search(cur, m, g, K=K, S=S)
    h = S + K // 2
    tgt = (m == 0)
    inner = np.zeros_like(tgt)
    inner[h:-h, h:-h] = True
    sel = tgt & inner
    assert np.all(f["status"][sel] == CANDIDATE)
    assert np.all(f["alpha"][sel] == 0) and np.all(f["beta"][sel] == 0) and np.all(f["err"][sel] == 0)
    for chk in (oracle.frmc, oracle.rmc, oracle.rme):
        kw = dict(K=K, S=S) if chk is not oracle.frmc else dict(K=K, S=7)
        st, _ = chk(cur, m, g, f, **kw)
        assert np.all(st[sel] == ACCEPTED)


def test_p2_constant_frames():
    W = H = 24
    m = synth.quarter_mask(W, H, 5, False)
    cur = (100 * m).astype(np.uint8)
    ref = np.full((H, W), 100, np.uint8)
    S, K = 3, 8
    f = oracle.me_search(cur, m, ref, K=K, S=S)
    ra, rb = oracle.rank_list(S)
    for y in range(H):
        for x in range(W):
            if m[y, x]:
                continue
            ns = [oracle.cost_fwd(cur, m, ref, y, x, a, b, K=K)[1] for a, b in zip(ra, rb)]
            adm = [i for i, n in enumerate(ns) if n >= 8]
            if not adm:
                assert f["status"][y, x] == INVALID
                continue
            k = adm[0]                               # all e = 0: the first admissible in rank order wins
            assert (f["alpha"][y, x], f["beta"][y, x]) == (ra[k], rb[k])
            assert f["err"][y, x] == 0
            if ns[0] >= 8:
                assert (f["alpha"][y, x], f["beta"][y, x]) == (0, 0)
    # The corner target's in-frame window holds 16 pixels -> n = 4 < 8 for every v: INVALID.
    corner = [(y, x) for y in (0, 1) for x in (0, 1) if m[y, x] == 0]
    assert all(f["status"][y, x] == INVALID for (y, x) in corner)
    # Ties accept in RMC/FRMC; RME's reverse argmin is (0,0) = -v.
    fv = dict(f)
    for chk in (oracle.rmc, oracle.rme):
        st, _ = chk(cur, m, ref, fv, K=K, S=S)
        ok = (f["status"] == CANDIDATE) & (f["alpha"] == 0) & (f["beta"] == 0)
        inner = np.zeros_like(ok)
        inner[6:-6, 6:-6] = True
        assert np.all(st[ok & inner] == ACCEPTED)


def test_min_support_above_max_gives_invalid():
    inp = synth.rank_free_random_instance(2, 16, 16)
    f = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=8, S=2, min_support=26)
    assert np.all(f["status"][inp["cur_mask"] == 0] == INVALID)   # K=8, quarter mask -> n <= 25


# ---------------------------------------------------------------------------
# P3: known integer translation (closed form)
# ---------------------------------------------------------------------------
def _translated_pair(seed, W, H, vstar, smooth=False):
    rng = np.random.default_rng(seed)
    big = rng.integers(0, 256, (H + 20, W + 20)).astype(np.uint8)
    a, b = vstar
    g_cur = big[10:10 + H, 10:10 + W]
    g_ref = big[10 - a:10 - a + H, 10 - b:10 - b + W]   # ref(q + v*) = cur(q)
    m = synth.quarter_mask(W, H, seed, False)
    return (g_cur * m).astype(np.uint8), m, g_ref, g_cur


def test_p3_integer_translation_noise_free():
    vstar = (2, -3)
    cur, m, ref, _ = _translated_pair(1, 48, 48, vstar)
    S, K = 4, 8
    f = oracle.me_search(cur, m, ref, K=K, S=S)
    h = S + K // 2
    sel = (m == 0)
    sel[:h] = sel[-h:] = False
    sel[:, :h] = sel[:, -h:] = False
    ok = (f["alpha"][sel] == vstar[0]) & (f["beta"][sel] == vstar[1]) & (f["err"][sel] == 0)
    assert ok.mean() >= 0.99


def test_p3_config1_translation_with_noise():
    seq = synth.make_sequence(1)
    for d in (1, 2):
        inp = synth.pair_inputs(seq, 2, d)
        f = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=8, S=8)
        a, b = seq.true_v(2, d)
        assert (a, b) == (d, -2 * d)
        h = 8 + 4
        sel = inp["cur_mask"] == 0
        sel[:h] = sel[-h:] = False
        sel[:, :h] = sel[:, -h:] = False
        frac = ((f["alpha"][sel] == a) & (f["beta"][sel] == b)).mean()
        assert frac >= 0.95, frac


# ---------------------------------------------------------------------------
# P4: identity rc(p+v, -v) == (e, n), bit-exact for u8 and fp32
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("f32", [False, True])
@pytest.mark.parametrize("ssd", [False, True])
def test_p4_reverse_identity(f32, ssd):
    inp = synth.rank_free_random_instance(21, 20, 20, ref_f32=f32)
    rng = np.random.default_rng(4)
    for _ in range(200):
        y, x = rng.integers(0, 20, 2)
        a, b = rng.integers(-5, 6, 2)
        fw = oracle.cost_fwd(inp["cur"], inp["cur_mask"], inp["ref"], y, x, a, b, K=8, ssd=ssd)
        rv = oracle.cost_rev(inp["cur"], inp["cur_mask"], inp["ref"], y + a, x + b, -a, -b, K=8, ssd=ssd)
        assert fw == rv
        if inp["cur_mask"][y, x] == 0 and fw[1] > 0:
            # Textbook definition written out with Python ints / floats: a pin other than oracle.c.
            e_ref = 0.0 if f32 else 0
            n_ref = 0
            for oy in range(-4, 4):
                for ox in range(-4, 4):
                    qy, qx = y + oy, x + ox
                    if not (0 <= qy < 20 and 0 <= qx < 20) or inp["cur_mask"][qy, qx] == 0:
                        continue
                    if not (0 <= qy + a < 20 and 0 <= qx + b < 20):
                        continue
                    c = inp["cur"][qy, qx]
                    r = inp["ref"][qy + a, qx + b]
                    if f32:
                        dd = np.float32(np.float32(c) - np.float32(r))
                        e_ref = np.float32(e_ref + (dd * dd if ssd else abs(dd)))
                    else:
                        dd = int(c) - int(r)
                        e_ref += dd * dd if ssd else abs(dd)
                    n_ref += 1
            assert fw == ((float(e_ref) if f32 else e_ref), n_ref)


# ---------------------------------------------------------------------------
# P5, P6, P8: check relations, injected wrong vectors, evaluation counts
# ---------------------------------------------------------------------------
def test_p5_rmc_subset_frmc_and_cascade():
    inp = synth.rank_free_random_instance(31, 28, 28, smooth=True)
    S, K = 7, 8
    f = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=K, S=S)
    st_rmc, ev_rmc = oracle.rmc(inp["cur"], inp["cur_mask"], inp["ref"], f, K=K, S=S)
    st_frmc, ev_frmc = oracle.frmc(inp["cur"], inp["cur_mask"], inp["ref"], f, K=K, S=S)
    assert np.all(st_frmc[st_rmc == ACCEPTED] == ACCEPTED)       # O x O within [-S,S]^2
    st_nnc = oracle.nnc(f)
    st_casc, ev_casc = oracle.frmc(inp["cur"], inp["cur_mask"], inp["ref"], dict(f, status=st_nnc), K=K, S=S)
    acc = (st_nnc == ACCEPTED) & (st_frmc == ACCEPTED)
    assert np.array_equal(st_casc == ACCEPTED, acc)              # NNC -> FRMC = NNC n FRMC
    # P8: definitional counts (R17): 49 per checked FRMC entry, (2S+1)^2 for RMC, 0 for NNC rejects.
    nval = int((f["status"] == CANDIDATE).sum())
    assert ev_frmc == 49 * nval and ev_rmc == (2 * S + 1) ** 2 * nval
    assert ev_casc == 49 * int((st_nnc == ACCEPTED).sum())


def test_p8_cascade_all_rejected_zero_evals():
    inp = synth.rank_free_random_instance(5, 16, 16)
    f = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=8, S=7)
    st = np.where(f["status"] == CANDIDATE, REJECTED, f["status"]).astype(np.uint8)
    st2, ev = oracle.frmc(inp["cur"], inp["cur_mask"], inp["ref"], dict(f, status=st), K=8, S=7)
    assert ev == 0 and np.array_equal(st2, st)


def test_p8_paper_counts_361_49():
    # "reduced from 361 to 49" at S = 9.
    assert len(oracle.rank_list(9)[0]) == 361
    assert len(synth.FRMC_OFFSETS) ** 2 == 49


def test_p6_injected_wrong_vector():
    vstar = (1, 2)
    cur, m, ref, _ = _translated_pair(9, 40, 40, vstar)
    S, K = 9, 8
    ys, xs = np.nonzero(m == 0)
    pick = [(y, x) for y, x in zip(ys, xs) if 14 <= y < 26 and 14 <= x < 26][:6]
    for delta, frmc_must_reject in (((3, -1), True), ((-7, 7), True), ((2, 2), False)):
        for (y, x) in pick:
            a, b = vstar[0] + delta[0], vstar[1] + delta[1]
            e, n = oracle.cost_fwd(cur, m, ref, y, x, a, b, K=K)
            f = dict(alpha=np.zeros_like(m, np.int8), beta=np.zeros_like(m, np.int8),
                     err=np.zeros(m.shape, np.uint32), count=np.zeros_like(m), status=np.zeros_like(m))
            f["alpha"][y, x], f["beta"][y, x], f["err"][y, x], f["count"][y, x] = a, b, e, n
            f["status"][y, x] = CANDIDATE
            # rc at delta' = v* - v' (reverse vector -v*) is 0 < e (noise texture => e > 0).
            assert e > 0
            st, _ = oracle.rmc(cur, m, ref, f, K=K, S=S)
            assert st[y, x] == REJECTED
            st, _ = oracle.rme(cur, m, ref, f, K=K, S=S)
            assert st[y, x] == REJECTED
            st, _ = oracle.frmc(cur, m, ref, f, K=K, S=S)
            if frmc_must_reject:
                assert st[y, x] == REJECTED
    # A true vector is accepted by all reverse checks.
    (y, x) = pick[0]
    e, n = oracle.cost_fwd(cur, m, ref, y, x, *vstar, K=K)
    assert e == 0
    f = dict(alpha=np.zeros_like(m, np.int8), beta=np.zeros_like(m, np.int8),
             err=np.zeros(m.shape, np.uint32), count=np.zeros_like(m), status=np.zeros_like(m))
    f["alpha"][y, x], f["beta"][y, x], f["count"][y, x], f["status"][y, x] = vstar[0], vstar[1], n, CANDIDATE
    for chk in (oracle.rmc, oracle.rme, oracle.frmc):
        st, _ = chk(cur, m, ref, f, K=K, S=S)
        assert st[y, x] == ACCEPTED


# ---------------------------------------------------------------------------
# P10: restriction property
# ---------------------------------------------------------------------------
def test_p10_restriction():
    from fractions import Fraction
    inp = synth.rank_free_random_instance(17, 20, 20)
    f2 = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=8, S=2)
    f4 = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=8, S=4)
    both = (f2["status"] == CANDIDATE) & (f4["status"] == CANDIDATE)
    for y, x in zip(*np.nonzero(both)):
        m2 = Fraction(int(f2["err"][y, x]), int(f2["count"][y, x]))
        m4 = Fraction(int(f4["err"][y, x]), int(f4["count"][y, x]))
        assert m4 <= m2


# ---------------------------------------------------------------------------
# P11: the search written twice (oracle.c vs numpy twin), >= 200 instances
# ---------------------------------------------------------------------------
def test_p11_c_vs_twin_me():
    rng = np.random.default_rng(2022)
    n_inst = 0
    for i in range(200):
        K = int(rng.choice([3, 4, 8, 9]))
        S = int(rng.integers(1, 5))
        ssd = bool(rng.integers(0, 2))
        f32 = bool(rng.integers(0, 2))
        ms = int(rng.integers(1, 9))
        inp = synth.rank_free_random_instance(1000 + i, 16, 16, ref_f32=f32, dynamic=bool(i % 2), t=i % 4)
        a = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=K, S=S, min_support=ms, ssd=ssd)
        b = twin.me_search(inp["cur"], inp["cur_mask"], inp["ref"], K=K, S=S, min_support=ms, ssd=ssd)
        for k in ("alpha", "beta", "count", "status"):
            assert np.array_equal(a[k], b[k]), (i, k)
        assert np.array_equal(a["err"].view(np.uint32), b["err"].astype(a["err"].dtype).view(np.uint32)), i
        n_inst += 1
    assert n_inst >= 200


def test_p11_c_vs_twin_checks():
    rng = np.random.default_rng(7)
    for i in range(40):
        K = int(rng.choice([4, 8]))
        S = int(rng.integers(1, 4))
        f32 = bool(i % 2)
        ssd = bool((i // 2) % 2)
        inp = synth.rank_free_random_instance(500 + i, 14, 14, ref_f32=f32, smooth=bool(i % 3 == 0))
        kw = dict(K=K, S=S, min_support=4, ssd=ssd)
        f = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], **kw)
        offs = (-1, 0, 1) if S < 3 else (-3, -1, 0, 1, 3)
        for name, cfn, tfn in (("frmc", lambda fl: oracle.frmc(inp["cur"], inp["cur_mask"], inp["ref"], fl, offsets=offs, **kw),
                                lambda fl: twin.frmc(inp["cur"], inp["cur_mask"], inp["ref"], fl, offsets=offs, **kw)),
                               ("rmc", lambda fl: oracle.rmc(inp["cur"], inp["cur_mask"], inp["ref"], fl, **kw),
                                lambda fl: twin.rmc(inp["cur"], inp["cur_mask"], inp["ref"], fl, **kw)),
                               ("rme", lambda fl: oracle.rme(inp["cur"], inp["cur_mask"], inp["ref"], fl, **kw),
                                lambda fl: twin.rme(inp["cur"], inp["cur_mask"], inp["ref"], fl, **kw))):
            sa, ea = cfn(f)
            sb, eb = tfn(f)
            assert np.array_equal(sa, sb) and ea == eb, (i, name)
        assert np.array_equal(oracle.nnc(f), twin.nnc(f["alpha"], f["beta"], f["status"]))


# ---------------------------------------------------------------------------
# P12: mask-blindness
# ---------------------------------------------------------------------------
def test_p12_mask_blind():
    inp = synth.rank_free_random_instance(44, 24, 24, smooth=True)
    rng = np.random.default_rng(0)
    junk = inp["cur"].copy()
    junk[inp["cur_mask"] == 0] = rng.integers(0, 256, int((inp["cur_mask"] == 0).sum()))
    kw = dict(K=8, S=7)
    a, ea = oracle.pair_chain(inp, check="nnc_frmc", **kw)
    b, eb = oracle.pair_chain(dict(inp, cur=junk), check="nnc_frmc", **kw)
    for k in a:
        assert np.array_equal(a[k], b[k])
    assert ea == eb


# ---------------------------------------------------------------------------
# P15: fp32 oracle vs fp64 definition, within the rounding bound
# ---------------------------------------------------------------------------
def test_p15_fp32_within_bound_of_fp64():
    inp = synth.rank_free_random_instance(77, 24, 24, ref_f32=True, smooth=True)
    kw = dict(K=8, S=4)
    f32 = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], **kw)
    f64 = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], ref_mode=oracle.REF_F32_ACC64, **kw)
    assert np.array_equal(f32["status"], f64["status"])
    sel = f32["status"] == CANDIDATE
    same = sel & (f32["alpha"] == f64["alpha"]) & (f32["beta"] == f64["beta"])
    # Relative error of a <= 25-term fp32 sum: <= 25 * 2^-24 < 1.5e-6 (well inside 1e-5).
    e32 = f32["err"][same].astype(np.float64)
    e64 = f64["err"][same]
    assert np.all(np.abs(e32 - e64) <= 1.5e-6 * np.maximum(e64, 1e-30) + 1e-12)
    # Vector differences only at near-ties: re-score both vectors in fp64.
    for y, x in zip(*np.nonzero(sel & ~same)):
        e1, n1 = oracle.cost_fwd(inp["cur"], inp["cur_mask"], inp["ref"], y, x, int(f32["alpha"][y, x]),
                                 int(f32["beta"][y, x]), K=8, ref_mode=oracle.REF_F32_ACC64)
        e2, n2 = oracle.cost_fwd(inp["cur"], inp["cur_mask"], inp["ref"], y, x, int(f64["alpha"][y, x]),
                                 int(f64["beta"][y, x]), K=8, ref_mode=oracle.REF_F32_ACC64)
        assert abs(e1 / n1 - e2 / n2) <= 2e-6 * max(e2 / n2, 1e-9)


# ---------------------------------------------------------------------------
# P7b: the two readings of NNC's "each neighboring pair" (R15 headline, R30 NEXT-4)
# ---------------------------------------------------------------------------
def test_p7b_nnc_pairs_reading_golden(golden):
    g = golden("nnc_pairs_hand.json")
    for case in g["cases"]:
        f = dict(alpha=_arr(case["alpha"], np.int8), beta=_arr(case["beta"], np.int8),
                 status=_arr(case["status"], np.uint8))
        fa, _, d = oracle.median_field(f)
        m = d == 1
        assert np.array_equal(fa[m], _arr(case["filtered_alpha"], np.int32)[m]), case["name"]
        for pairs, key in ((False, "expect_centre"), (True, "expect_pairs")):
            st = oracle.nnc(f, threshold=1, pairs=pairs)
            assert np.array_equal(st, _arr(case[key], np.uint8)), (case["name"], key)
            assert np.array_equal(twin.nnc(f["alpha"], f["beta"], f["status"], 1, pairs=pairs), st)


def test_p7b_nnc_pairs_equals_centre_reading_on_the_p7_fixtures(golden):
    # On the P7 fixtures where every filtered vector is equal the two readings agree (constant fields)
    g = golden("nnc_hand.json")
    for case in g["cases"][:2]:
        f = dict(alpha=_arr(case["alpha"], np.int8), beta=_arr(case["beta"], np.int8),
                 status=_arr(case["status"], np.uint8))
        assert np.array_equal(oracle.nnc(f, pairs=True), oracle.nnc(f, pairs=False)), case["name"]


def test_omp_row_driver_equals_sequential_oracle():
    """oracle/omp_driver.c adds no arithmetic: rows through the OpenMP driver (one definition call per
    row) give the sequential oracle's planes and counts for u8 and f32, ME and every reverse check."""
    for f32 in (False, True):
        inp = synth.rank_free_random_instance(31 + f32, 48, 40, ref_f32=f32, smooth=True)
        kw = dict(K=8, S=8)
        a = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], **kw)
        b = oracle.me_search(inp["cur"], inp["cur_mask"], inp["ref"], threads=4, **kw)
        for k in a:
            assert np.array_equal(a[k], b[k]), k
        for fn in (oracle.frmc, oracle.rmc, oracle.rme):
            s1, e1 = fn(inp["cur"], inp["cur_mask"], inp["ref"], a, **kw)
            s2, e2 = fn(inp["cur"], inp["cur_mask"], inp["ref"], a, threads=4, **kw)
            assert np.array_equal(s1, s2) and e1 == e2, fn.__name__
