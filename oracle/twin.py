"""NumPy twin of the oracle: the same definitions written a second time.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Independent of oracle.c
(no shared code or tables) and of the CUDA path.  Loop order differs on
purpose: the candidate axis is vectorised (o outer, all v at once), the rank
order is built with ``np.lexsort`` instead of a comparator sort, and the exact
mean comparison for integer errors uses float64 quotients (distinct rationals
e/n with n <= 81 differ by >= 1/6561, far above float64 rounding, and equal
rationals round to the same double).  Pins P11 ("search written twice",
SPEC.md:596-601) compare this module with oracle.c bit for bit.

Definitions followed: PAPER.md:68 (ME), :71-72 (RME), :101-105 (RMC/FRMC),
:107-115 with Eq. (1) (NNC), :74 (PR); readings R1-R19, R23.
"""
from __future__ import annotations

import numpy as np

NOT_TARGET, INVALID, CANDIDATE, ACCEPTED, REJECTED = 0, 1, 2, 3, 4


def rank_order(S: int):
    a, b = np.meshgrid(np.arange(-S, S + 1), np.arange(-S, S + 1), indexing="ij")
    a = a.ravel()
    b = b.ravel()
    idx = np.lexsort((b, a, np.abs(a) + np.abs(b)))  # last key is primary
    return a[idx], b[idx]


def _offsets(K):
    return np.arange(-(K // 2), K - K // 2)


def _costs(cur, mask, ref, centers_y, centers_x, vy, vx, K, f32, ssd, reverse):
    """Vectorised matching errors at one template position for many vectors.

    forward: position p, vectors v: terms over q=p+o with q in frame, mask(q),
             q+v in frame; term phi(cur(q) - ref(q+v)).
    reverse: position x, vectors u: terms over q=x+o with q in frame, q+u in
             frame, mask(q+u); term phi(ref(q) - cur(q+u)).
    Returns (e, n) arrays over the vectors; accumulation in row-major o order.
    """
    H, W = cur.shape
    Kh, Kw = (K, K) if np.isscalar(K) else K
    nv = vy.size
    e = np.zeros(nv, np.float32 if f32 else np.int64)
    n = np.zeros(nv, np.int64)
    for oy in _offsets(Kh):
        for ox in _offsets(Kw):
            qy, qx = centers_y + oy, centers_x + ox
            if not (0 <= qy < H and 0 <= qx < W):
                continue
            sy, sx = qy + vy, qx + vx
            ok = (sy >= 0) & (sy < H) & (sx >= 0) & (sx < W)
            syc, sxc = np.clip(sy, 0, H - 1), np.clip(sx, 0, W - 1)
            if reverse:
                ok = ok & (mask[syc, sxc] == 1)
                cvals = cur[syc, sxc]
                rvals = np.broadcast_to(ref[qy, qx], (nv,))
            else:
                if mask[qy, qx] != 1:
                    continue
                cvals = np.broadcast_to(cur[qy, qx], (nv,))
                rvals = ref[syc, sxc]
            if f32:
                d = cvals.astype(np.float32) - rvals.astype(np.float32)
                t = (d * d) if ssd else np.abs(d)
                e = np.where(ok, (e + t).astype(np.float32), e)
            else:
                d = cvals.astype(np.int64) - rvals.astype(np.int64)
                t = d * d if ssd else np.abs(d)
                e = np.where(ok, e + t, e)
            n = n + ok
    return e, n


def _means(e, n, f32):
    with np.errstate(divide="ignore", invalid="ignore"):
        if f32:
            return (e.astype(np.float32) / n.astype(np.float32)).astype(np.float32)
        return e.astype(np.float64) / n.astype(np.float64)


def me_search(cur, mask, ref, K=8, S=8, min_support=8, ssd=False):
    f32 = ref.dtype == np.float32
    H, W = cur.shape
    ra, rb = rank_order(S)
    out = dict(alpha=np.zeros((H, W), np.int8), beta=np.zeros((H, W), np.int8),
               err=np.zeros((H, W), np.float32 if f32 else np.uint32), count=np.zeros((H, W), np.uint8),
               status=np.full((H, W), NOT_TARGET, np.uint8))
    for y in range(H):
        for x in range(W):
            if mask[y, x]:
                continue
            e, n = _costs(cur, mask, ref, y, x, ra, rb, K, f32, ssd, reverse=False)
            adm = n >= min_support
            if not adm.any():
                out["status"][y, x] = INVALID
                continue
            m = _means(e, n, f32)
            m = np.where(adm, m, np.inf)
            k = int(np.argmin(m))          # first occurrence in rank order = tie-break
            out["alpha"][y, x], out["beta"][y, x] = ra[k], rb[k]
            out["err"][y, x] = e[k]
            out["count"][y, x] = n[k]
            out["status"][y, x] = CANDIDATE
    return out


def _reverse_grid(cur, mask, ref, field, dys, dxs, K, S, min_support, ssd):
    f32 = ref.dtype == np.float32
    st = field["status"].copy()
    evals = 0
    H, W = cur.shape
    dy, dx = np.meshgrid(dys, dxs, indexing="ij")
    dy, dx = dy.ravel(), dx.ravel()
    nz = ~((dy == 0) & (dx == 0))
    for y in range(H):
        for x in range(W):
            if st[y, x] not in (CANDIDATE, ACCEPTED):
                continue
            a, b = int(field["alpha"][y, x]), int(field["beta"][y, x])
            e, n = _costs(cur, mask, ref, y + a, x + b, -a + dy, -b + dx, K, f32, ssd, reverse=True)
            c0 = np.flatnonzero(~nz)[0]
            m = _means(e, n, f32)
            smaller = nz & (n >= min_support) & (m < m[c0])
            st[y, x] = REJECTED if smaller.any() else ACCEPTED
            evals += dy.size
    return st, evals


def frmc(cur, mask, ref, field, offsets=(-7, -3, -1, 0, 1, 3, 7), K=8, S=8, min_support=8, ssd=False):
    o = np.asarray(offsets)
    return _reverse_grid(cur, mask, ref, field, o, o, K, S, min_support, ssd)


def rmc(cur, mask, ref, field, K=8, S=8, min_support=8, ssd=False):
    o = np.arange(-S, S + 1)
    return _reverse_grid(cur, mask, ref, field, o, o, K, S, min_support, ssd)


def rme(cur, mask, ref, field, K=8, S=8, min_support=8, ssd=False):
    f32 = ref.dtype == np.float32
    st = field["status"].copy()
    ra, rb = rank_order(S)
    H, W = cur.shape
    evals = 0
    for y in range(H):
        for x in range(W):
            if st[y, x] not in (CANDIDATE, ACCEPTED):
                continue
            a, b = int(field["alpha"][y, x]), int(field["beta"][y, x])
            e, n = _costs(cur, mask, ref, y + a, x + b, ra, rb, K, f32, ssd, reverse=True)
            adm = n >= min_support
            m = np.where(adm, _means(e, n, f32), np.inf)
            k = int(np.argmin(m))
            ok = adm.any() and ra[k] == -a and rb[k] == -b
            st[y, x] = ACCEPTED if ok else REJECTED
            evals += ra.size
    return st, evals


def median_field(alpha, beta, status):
    H, W = status.shape
    valid = status >= CANDIDATE
    fa = np.zeros((H, W), np.int64)
    fb = np.zeros((H, W), np.int64)
    for y in range(H):
        for x in range(W):
            if not valid[y, x]:
                continue
            y0, y1, x0, x1 = max(0, y - 1), min(H, y + 2), max(0, x - 1), min(W, x + 2)
            v = valid[y0:y1, x0:x1]
            la = np.sort(alpha[y0:y1, x0:x1][v].astype(np.int64))
            lb = np.sort(beta[y0:y1, x0:x1][v].astype(np.int64))
            fa[y, x] = la[(la.size - 1) // 2]
            fb[y, x] = lb[(lb.size - 1) // 2]
    return fa, fb, valid


def nnc(alpha, beta, status, threshold=1, pairs=False):
    fa, fb, valid = median_field(alpha, beta, status)
    H, W = status.shape
    st = status.copy()
    for y in range(H):
        for x in range(W):
            if st[y, x] not in (CANDIDATE, ACCEPTED):
                continue
            nbs = [(yy, xx) for yy, xx in ((y - 1, x), (y + 1, x), (y, x - 1), (y, x + 1))
                   if 0 <= yy < H and 0 <= xx < W and valid[yy, xx]]
            if pairs:    # R30: the neighbours among themselves
                tests = [(p, q) for i, p in enumerate(nbs) for q in nbs[i + 1:]]
            else:        # R15: the centre against each neighbour
                tests = [((y, x), q) for q in nbs]
            bad = any(abs(fa[p] - fa[q]) + abs(fb[p] - fb[q]) > threshold for p, q in tests)
            st[y, x] = REJECTED if bad else ACCEPTED
    return st


def project(alpha, beta, status, past_val, past_mask):
    H, W = status.shape
    ys, xs = np.nonzero(status == ACCEPTED)
    qy = ys + alpha[ys, xs].astype(np.int64)
    qx = xs + beta[ys, xs].astype(np.int64)
    ok = (qy >= 0) & (qy < H) & (qx >= 0) & (qx < W)
    ys, xs, qy, qx = ys[ok], xs[ok], qy[ok], qx[ok]
    hit = past_mask[qy, qx] == 1
    s = np.zeros((H, W), np.uint32)
    c = np.zeros((H, W), np.uint8)
    s[ys[hit], xs[hit]] = past_val[qy[hit], qx[hit]]
    c[ys[hit], xs[hit]] = 1
    return s, c
