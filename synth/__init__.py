"""Seeded synthetic quarter-sampled video: the ONE module both sides may import.

This module holds input generation only -- textures, motion, noise, the quarter
sampling masks and the derived planes (cur, cur_mask, ref, past_val, past_mask).
It holds none of the method's arithmetic (no matching cost, no argmin, no
check, no projection).  Both the CPU oracle's tests and the CUDA path's tests /
bench draw their inputs from here (task rule: "only the seeded input generators
serve both, from a module of their own").

Recipe (BASELINE.json configs):

* RNG: ``numpy.random.Generator(PCG64(seed))`` with
  ``seed(c, s, k) = 1_000_000*c + 1_000*s + k``; per-frame streams use the
  SeedSequence entropy ``[seed(c, s, k), t]`` so frame t is random-access.
  k: 0 texture, 1 mask, 2 noise, 3 objects / occluders, 4 float-ref noise,
  5+ object textures.
* Texture (PAPER.md:144-145 stand-in): a sum of 16 2-D
  sinusoids ``a_i sin(2 pi (x cos th_i + y sin th_i) / lam_i + phi_i)``,
  a ~ U[0.5,1], lam ~ U[6,64] px, th ~ U[0,pi), phi ~ U[0,2 pi), mapped affinely
  so frame 0's min/max become 16..239 (same map for every frame).
* Noise N(0, sigma^2) added in float64, rounded half away from zero
  (SPEC.md:59), clipped to [0, 255] -> uint8 ground truth g_t.
* Masks (§1 "each pixel in a 2x2 block is read exactly once within
  four frames"): SplitMix64 hash
  ``h = mix64(seed_mask ^ (by << 32 | bx) + 0x9E3779B97F4A7C15)``; fixed mask
  quadrant ``q = h & 3``; dynamic mask ``q_t = perm[h % 24][t % 4]`` with the
  lexicographic permutations of (0,1,2,3); ``q = 2*dy + dx``.
* Derived planes (§2.1 ``f_sub = f . b``): ``cur_t = g_t*mask_t``,
  ``past_val = g_{t-d}*mask_{t-d}``, ``past_mask = mask_{t-d}``,
  ``ref_{t-d} = g_{t-d}`` (uint8) or, for config 4, the float32
  ``render_{t-d} + N(0, 1.5^2)`` clipped to [0, 255] and not rounded (R20).
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

__all__ = [
    "ConfigSpec", "CONFIGS", "seed_of", "mix64", "quarter_mask", "Sequence",
    "make_sequence", "rank_free_random_instance", "FRMC_OFFSETS",
]

# PAPER.md:104 (§3.1.1): "we test only motions in the set {-7,-3,-1,0,1,3,7}".
# This is an input parameter of the check (a constant the paper prints), not
# arithmetic of the method.
FRMC_OFFSETS = (-7, -3, -1, 0, 1, 3, 7)

_M64 = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
_PERMS = list(itertools.permutations(range(4)))  # lexicographic order, 24 entries


def seed_of(c: int, s: int, k: int) -> int:
    return 1_000_000 * c + 1_000 * s + k


def mix64(z: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on a uint64 array (wrapping arithmetic)."""
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return z


def _block_hash(w: int, h: int, seed_mask: int) -> np.ndarray:
    by = np.arange(h // 2, dtype=np.uint64)[:, None]
    bx = np.arange(w // 2, dtype=np.uint64)[None, :]
    key = (by << np.uint64(32)) | bx
    with np.errstate(over="ignore"):
        z = (np.uint64(seed_mask & _M64) ^ key) + np.uint64(_GOLDEN)
    return mix64(z)


def quarter_mask(w: int, h: int, seed_mask: int, dynamic: bool, t: int = 0) -> np.ndarray:
    """uint8 [h][w] mask with exactly one 1 per 2x2 block."""
    if w <= 0 or h <= 0 or (w & 1) or (h & 1):
        raise ValueError("quarter masks need positive even dimensions (SPEC.md:116-118)")
    hb = _block_hash(w, h, seed_mask)
    if dynamic:
        perm = np.array(_PERMS, dtype=np.uint8)  # [24][4]
        q = perm[(hb % np.uint64(24)).astype(np.int64), t % 4]
    else:
        q = (hb & np.uint64(3)).astype(np.uint8)
    dy = (q >> 1).astype(np.int64)
    dx = (q & 1).astype(np.int64)
    m = np.zeros((h, w), dtype=np.uint8)
    by, bx = np.meshgrid(np.arange(h // 2), np.arange(w // 2), indexing="ij")
    m[2 * by + dy, 2 * bx + dx] = 1
    return m


# --------------------------------------------------------------------------
# Textures
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class _Texture:
    a: np.ndarray
    lam: np.ndarray
    th: np.ndarray
    phi: np.ndarray

    @staticmethod
    def draw(rng: np.random.Generator, n: int = 16) -> "_Texture":
        a = rng.uniform(0.5, 1.0, n)
        lam = rng.uniform(6.0, 64.0, n)
        th = rng.uniform(0.0, np.pi, n)
        phi = rng.uniform(0.0, 2 * np.pi, n)
        return _Texture(a, lam, th, phi)

    def eval_affine(self, xs: np.ndarray, ys: np.ndarray, sx: float = 1.0, sy: float = 1.0,
                    ox: float = 0.0, oy: float = 0.0) -> np.ndarray:
        """T(sx*x + ox, sy*y + oy) on the grid ys[:,None] x xs[None,:] (separable)."""
        X = sx * xs.astype(np.float64) + ox
        Y = sy * ys.astype(np.float64) + oy
        out = np.zeros((Y.size, X.size), dtype=np.float64)
        for i in range(self.a.size):
            kx = 2 * np.pi * np.cos(self.th[i]) / self.lam[i]
            ky = 2 * np.pi * np.sin(self.th[i]) / self.lam[i]
            ax = kx * X
            ay = ky * Y + self.phi[i]
            # sin(ax + ay) = sin(ax)cos(ay) + cos(ax)sin(ay)
            out += self.a[i] * (np.cos(ay)[:, None] * np.sin(ax)[None, :]
                                + np.sin(ay)[:, None] * np.cos(ax)[None, :])
        return out


def _round_clip_u8(x: np.ndarray) -> np.ndarray:
    r = np.sign(x) * np.floor(np.abs(x) + 0.5)  # round half away from zero
    return np.clip(r, 0, 255).astype(np.uint8)


# --------------------------------------------------------------------------
# Configs (BASELINE.json "configs", readings R24 in DESIGN.md)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class ConfigSpec:
    idx: int
    name: str
    w: int
    h: int
    frames: int
    dynamic: bool
    sigma: float
    K: int
    S: int
    ssd: bool
    ref_f32: bool
    n_seq: int = 1


CONFIGS = {
    1: ConfigSpec(1, "c1_64x64_fixed_S8", 64, 64, 3, False, 2.0, 8, 8, False, False),
    2: ConfigSpec(2, "c2_352x288_dyn_S16", 352, 288, 30, True, 2.0, 8, 16, False, False),
    3: ConfigSpec(3, "c3_1280x720_fixed_S16", 1280, 720, 60, False, 3.0, 8, 16, False, False),
    4: ConfigSpec(4, "c4_1920x1080_dyn_S24_f32ref", 1920, 1080, 120, True, 2.0, 8, 24, False, True),
    5: ConfigSpec(5, "c5_3840x2160_dyn_S32_x8", 3840, 2160, 32, True, 3.0, 8, 32, False, False, 8),
}


def _rng(c: int, s: int, k: int, t: int | None = None) -> np.random.Generator:
    if t is None:
        return np.random.Generator(np.random.PCG64(seed_of(c, s, k)))
    return np.random.Generator(np.random.PCG64([seed_of(c, s, k), int(t)]))


class Sequence:
    """Random-access synthetic sequence for one (config, sequence index).

    ``frame(t)`` returns the uint8 ground truth g_t; ``render(t)`` the float64
    pre-noise image; ``mask(t)`` the quarter mask; ``ref(t)`` the stand-in for
    the previous reconstruction f^_t used when t serves as a reference (R20).
    ``true_v(t, d)`` is the analytic background vector (alpha, beta) = (rows, cols)
    from frame t to frame t-d where one exists (configs 1-3, 5).
    """

    def __init__(self, cfg: ConfigSpec | int, s: int = 0, w: int | None = None, h: int | None = None):
        self.cfg = CONFIGS[cfg] if isinstance(cfg, int) else cfg
        c = self.cfg.idx
        self.s = s
        self.w = w or self.cfg.w
        self.h = h or self.cfg.h
        self.mask_seed = seed_of(c, s, 1)
        self.tex = _Texture.draw(_rng(c, s, 0))
        # Affine map so that frame 0's min/max become 16..239.
        self._lo, self._hi = None, None
        r0 = self._raw(0)
        self._lo, self._hi = float(r0.min()), float(r0.max())
        self._objs = self._draw_objects()

    # ----- content -------------------------------------------------------
    def _draw_objects(self):
        c = self.cfg.idx
        rng = _rng(c, self.s, 3)
        objs = []
        if c == 2:
            for k in range(4):
                sw, sh = rng.integers(32, 97, 2)
                x0 = rng.uniform(0, max(self.w - sw, 1))
                y0 = rng.uniform(0, max(self.h - sh, 1))
                vx, vy = rng.integers(-6, 7, 2)
                objs.append(dict(kind="rect", x0=float(x0), y0=float(y0), sw=int(sw), sh=int(sh),
                                 vx=int(vx), vy=int(vy), tex=_Texture.draw(_rng(c, self.s, 5 + k))))
        elif c == 4:
            for k in range(20):
                ra, rb = rng.uniform(20, 120, 2)
                rot = rng.uniform(0, np.pi)
                cx = rng.uniform(0, self.w)
                cy = rng.uniform(0, self.h)
                vx, vy = rng.integers(-12, 13, 2)
                objs.append(dict(kind="ellipse", cx=float(cx), cy=float(cy), ra=float(ra), rb=float(rb),
                                 rot=float(rot), vx=int(vx), vy=int(vy),
                                 tex=_Texture.draw(_rng(c, self.s, 5 + k))))
        return objs

    def _raw(self, t: int) -> np.ndarray:
        """Un-normalised background texture of frame t."""
        c = self.cfg.idx
        xs = np.arange(self.w)
        ys = np.arange(self.h)
        if c == 1:    # g_t(x, y) = T(x - 2t, y + t): content moves +2 cols, -1 row per frame
            return self.tex.eval_affine(xs, ys, ox=-2.0 * t, oy=float(t))
        if c == 2:    # background pans +1 col per frame
            return self.tex.eval_affine(xs, ys, ox=-1.0 * t)
        if c in (3, 5):  # global sub-pixel pan, 0.5 px / frame (+x)
            return self.tex.eval_affine(xs, ys, ox=-0.5 * t)
        if c == 4:    # zoom about the centre, scale 1.002 / frame
            s = 1.002 ** t
            cx, cy = (self.w - 1) / 2.0, (self.h - 1) / 2.0
            return self.tex.eval_affine(xs, ys, sx=1.0 / s, sy=1.0 / s,
                                        ox=cx - cx / s, oy=cy - cy / s)
        raise ValueError(c)

    def _norm(self, raw: np.ndarray) -> np.ndarray:
        return 16.0 + (raw - self._lo) * (223.0 / (self._hi - self._lo))

    def render(self, t: int) -> np.ndarray:
        """float64 noiseless render of frame t (objects painted in index order)."""
        img = self._norm(self._raw(t))
        c = self.cfg.idx
        if c == 2:
            for o in self._objs:
                x0 = int(np.floor(o["x0"])) + o["vx"] * t
                y0 = int(np.floor(o["y0"])) + o["vy"] * t
                xa, xb = max(0, x0), min(self.w, x0 + o["sw"])
                ya, yb = max(0, y0), min(self.h, y0 + o["sh"])
                if xa >= xb or ya >= yb:
                    continue
                xs = np.arange(xa, xb) - o["vx"] * t
                ys = np.arange(ya, yb) - o["vy"] * t
                img[ya:yb, xa:xb] = self._norm(o["tex"].eval_affine(xs, ys))
        elif c == 4:
            for o in self._objs:
                cx = o["cx"] + o["vx"] * t
                cy = o["cy"] + o["vy"] * t
                R = max(o["ra"], o["rb"])
                xa, xb = max(0, int(np.floor(cx - R))), min(self.w, int(np.ceil(cx + R)) + 1)
                ya, yb = max(0, int(np.floor(cy - R))), min(self.h, int(np.ceil(cy + R)) + 1)
                if xa >= xb or ya >= yb:
                    continue
                X, Y = np.meshgrid(np.arange(xa, xb) - cx, np.arange(ya, yb) - cy)
                cr, sr = np.cos(o["rot"]), np.sin(o["rot"])
                u = (X * cr + Y * sr) / o["ra"]
                v = (-X * sr + Y * cr) / o["rb"]
                inside = (u * u + v * v) <= 1.0
                xs = np.arange(xa, xb) - o["vx"] * t
                ys = np.arange(ya, yb) - o["vy"] * t
                tex = self._norm(o["tex"].eval_affine(xs, ys))
                sub = img[ya:yb, xa:xb]
                sub[inside] = tex[inside]
        return img

    def frame(self, t: int) -> np.ndarray:
        """uint8 ground truth g_t = round(render_t + N(0, sigma^2)) (+ occluders in configs 3/5)."""
        return _frame_cached(self, t)

    def _frame_uncached(self, t: int) -> np.ndarray:
        c = self.cfg.idx
        img = self.render(t)
        img = img + _rng(c, self.s, 2, t).normal(0.0, self.cfg.sigma, img.shape)
        g = _round_clip_u8(img)
        if c in (3, 5):  # 10% of 16x16 blocks replaced by i.i.d. U{16..239} noise (occluders)
            rng = _rng(c, self.s, 3, t)
            bh, bw = (self.h + 15) // 16, (self.w + 15) // 16
            occ = rng.random((bh, bw)) < 0.1
            noise = rng.integers(16, 240, (bh * 16, bw * 16), dtype=np.int64).astype(np.uint8)
            full = np.repeat(np.repeat(occ, 16, 0), 16, 1)[: self.h, : self.w]
            g = np.where(full, noise[: self.h, : self.w], g)
        return g

    def mask(self, t: int) -> np.ndarray:
        return quarter_mask(self.w, self.h, self.mask_seed, self.cfg.dynamic, t)

    def cur(self, t: int) -> np.ndarray:
        return (self.frame(t) * self.mask(t)).astype(np.uint8)

    def ref(self, t: int) -> np.ndarray:
        """Stand-in for the reconstruction of frame t when it is a reference (R20)."""
        if not self.cfg.ref_f32:
            return self.frame(t)
        c = self.cfg.idx
        r = self.render(t) + _rng(c, self.s, 4, t).normal(0.0, 1.5, (self.h, self.w))
        return np.clip(r, 0.0, 255.0).astype(np.float32)

    def true_v(self, t: int, d: int):
        """Background vector (alpha, beta) from frame t to frame t-d, when integer."""
        c = self.cfg.idx
        if c == 1:
            return (d, -2 * d)
        if c == 2:
            return (0, -d)
        return None


_FRAME_CACHE: dict = {}


def _frame_cached(seq: Sequence, t: int) -> np.ndarray:
    key = (seq.cfg, seq.s, seq.w, seq.h, t)
    g = _FRAME_CACHE.get(key)
    if g is None:
        if len(_FRAME_CACHE) > 64:
            _FRAME_CACHE.clear()
        g = seq._frame_uncached(t)
        _FRAME_CACHE[key] = g
    return g


def make_sequence(cfg: int, s: int = 0, w: int | None = None, h: int | None = None) -> Sequence:
    return Sequence(cfg, s, w, h)


def pair_inputs(seq: Sequence, t: int, d: int) -> dict:
    """All planes for one (frame t, reference distance d) pair."""
    m = seq.mask(t)
    pm = seq.mask(t - d)
    return dict(cur=(seq.frame(t) * m).astype(np.uint8), cur_mask=m, ref=seq.ref(t - d),
                past_val=(seq.frame(t - d) * pm).astype(np.uint8), past_mask=pm)


# --------------------------------------------------------------------------
# Small random instances (P11-style cross checks, parity fuzz)
# --------------------------------------------------------------------------
def rank_free_random_instance(seed: int, w: int, h: int, ref_f32: bool = False,
                              dynamic: bool = False, t: int = 0, smooth: bool = False) -> dict:
    """Random quarter-sampled pair: uniform noise (or a smooth texture) frames.

    Returns ``cur, cur_mask, ref, past_val, past_mask``.  Nothing here knows the
    method; it only produces arrays.
    """
    rng = np.random.Generator(np.random.PCG64([seed, w, h]))
    if smooth:
        tex = _Texture.draw(rng)
        raw = tex.eval_affine(np.arange(w), np.arange(h))
        g = _round_clip_u8(16 + (raw - raw.min()) * 223 / max(raw.max() - raw.min(), 1e-9))
        gp = _round_clip_u8(16 + (tex.eval_affine(np.arange(w), np.arange(h), ox=-1, oy=1) - raw.min())
                            * 223 / max(raw.max() - raw.min(), 1e-9))
    else:
        g = rng.integers(0, 256, (h, w), dtype=np.int64).astype(np.uint8)
        gp = rng.integers(0, 256, (h, w), dtype=np.int64).astype(np.uint8)
    m = quarter_mask(w, h, int(rng.integers(1 << 62)), dynamic, t)
    pm = quarter_mask(w, h, int(rng.integers(1 << 62)), dynamic, t + 1)
    if ref_f32:
        ref = np.clip(gp.astype(np.float64) + rng.normal(0, 1.5, (h, w)), 0, 255).astype(np.float32)
    else:
        ref = gp
    return dict(cur=(g * m).astype(np.uint8), cur_mask=m, ref=ref,
                past_val=(gp * pm).astype(np.uint8), past_mask=pm, dense_cur=g)
