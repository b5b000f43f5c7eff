"""CPU oracle for the hot path (ME, RME, RMC, FRMC, NNC, PR) of arxiv 2203.09200.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2203_09200_b200``) never imports it and it
never imports the product path; the two share only ``synth`` (inputs).

``oracle.c`` is the plain-C oracle (definitions written out, see its header);
``twin.py`` is an independent NumPy re-implementation of the same definitions
with a different loop order (vectorised over candidates), used to pin the C
oracle (pin P11, "search written twice").

Parity status per function:
  me_search (u8, f32, SAD/SSD)  pinned: P1, P2, P3, P10, P11, P12, P13, P15
  rank order                    pinned: P13 golden tie case, explicit L1=1 order
  frmc / rmc / rme              pinned: P4, P5, P6, P8, golden FRMC fixture
  nnc / median field            pinned: P7 hand-worked fixtures (tests/golden)
  project                       pinned: P9 hand-worked fixture
  Parity unpinned: which NNC neighbour reading the authors used (R15), the
  RMC/FRMC tie semantics (R11) and the f32 summation order (R23) -- these are
  readings with no printed example in PAPER.md to separate them.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

NOT_TARGET, INVALID, CANDIDATE, ACCEPTED, REJECTED = 0, 1, 2, 3, 4
REF_U8, REF_F32, REF_F32_ACC64 = 0, 1, 2


_OMP_SRC = os.path.join(_HERE, "omp_driver.c")
_OMP_LIB = os.path.join(_HERE, "liboracle_omp.so")
_CFLAGS = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall"]


def build(force: bool = False) -> str:
    """Compile the plain-C oracle (-O2, no FMA contraction, no fast-math), and the OpenMP row driver
    (omp_driver.c, linked with the same oracle.c into liboracle_omp.so)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(_CFLAGS + ["-o", _LIB, _SRC])
    newest = max(os.path.getmtime(_SRC), os.path.getmtime(_OMP_SRC))
    if force or not os.path.exists(_OMP_LIB) or os.path.getmtime(_OMP_LIB) < newest:
        subprocess.check_call(_CFLAGS + ["-fopenmp", "-o", _OMP_LIB, _SRC, _OMP_SRC])
    return _LIB


class _Params(C.Structure):
    _fields_ = [("W", C.c_int32), ("H", C.c_int32), ("Kh", C.c_int32), ("Kw", C.c_int32),
                ("S", C.c_int32), ("min_support", C.c_int32), ("ssd", C.c_int32),
                ("ref_mode", C.c_int32)]


_lib = None
_omp = None


def omp_lib():
    """The OpenMP row driver (same definitions; rows in parallel)."""
    global _omp
    if _omp is None:
        build()
        _omp = C.CDLL(_OMP_LIB)
        P = C.POINTER(_Params)
        vp = C.c_void_p
        i32 = C.c_int32
        _omp.or_threads_available.argtypes = []
        _omp.or_me_search_omp.argtypes = [P, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp, i32]
        _omp.or_frmc_omp.argtypes = [P, vp, vp, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, i32, i32]
        _omp.or_rmc_omp.argtypes = [P, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp, vp, i32, i32]
        _omp.or_rme_omp.argtypes = [P, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp, vp, i32]
    return _omp


def threads_available() -> int:
    return int(omp_lib().or_threads_available())


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        P = C.POINTER(_Params)
        vp = C.c_void_p
        i32 = C.c_int32
        _lib.or_rank_list.argtypes = [i32, vp, vp]
        _lib.or_me_search.argtypes = [P, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp]
        _lib.or_frmc.argtypes = [P, vp, vp, vp, vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, i32]
        _lib.or_rmc.argtypes = [P, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp, vp, i32]
        _lib.or_rme.argtypes = [P, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp, vp]
        _lib.or_nnc.argtypes = [i32, i32, i32, i32, vp, vp, vp, i32]
        _lib.or_nnc_mode.argtypes = [i32, i32, i32, i32, vp, vp, vp, i32, i32]
        _lib.or_median_field.argtypes = [i32, i32, vp, vp, vp, vp, vp, vp]
        _lib.or_project.argtypes = [i32, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp]
        _lib.or_probe_fwd.argtypes = [P, vp, vp, vp, i32, i32, i32, i32, vp, vp, vp]
        _lib.or_probe_rev.argtypes = [P, vp, vp, vp, i32, i32, i32, i32, vp, vp, vp]
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _params(cur, ref, K, S, min_support, ssd, ref_mode):
    H, W = cur.shape
    Kh, Kw = (K, K) if np.isscalar(K) else K
    if ref_mode is None:
        ref_mode = REF_F32 if np.asarray(ref).dtype == np.float32 else REF_U8
    return _Params(W, H, Kh, Kw, S, min_support, int(ssd), ref_mode), ref_mode


def _ref_arr(ref, ref_mode):
    return _c(ref, np.uint8 if ref_mode == REF_U8 else np.float32)


def _err_dtype(ref_mode):
    return {REF_U8: np.uint32, REF_F32: np.float32, REF_F32_ACC64: np.float64}[ref_mode]


def rank_list(S: int):
    n = (2 * S + 1) ** 2
    a = np.zeros(n, np.int32)
    b = np.zeros(n, np.int32)
    lib().or_rank_list(S, _p(a), _p(b))
    return a, b


def me_search(cur, cur_mask, ref, K=8, S=8, min_support=8, ssd=False, ref_mode=None, rows=None, threads=1):
    """ME over target rows ``rows=(y0, y1)`` (default: all). Returns the field planes.

    threads > 1 runs the rows through the OpenMP driver (the same definitions, one row per call)."""
    cur = _c(cur, np.uint8)
    mask = _c(cur_mask, np.uint8)
    P, ref_mode = _params(cur, ref, K, S, min_support, ssd, ref_mode)
    ref = _ref_arr(ref, ref_mode)
    H, W = cur.shape
    y0, y1 = rows if rows is not None else (0, H)
    f = dict(alpha=np.zeros((H, W), np.int8), beta=np.zeros((H, W), np.int8),
             err=np.zeros((H, W), _err_dtype(ref_mode)), count=np.zeros((H, W), np.uint8),
             status=np.zeros((H, W), np.uint8))
    args = [C.byref(P), _p(cur), _p(mask), _p(ref), y0, y1, _p(f["alpha"]), _p(f["beta"]),
            _p(f["err"]), _p(f["count"]), _p(f["status"])]
    r = omp_lib().or_me_search_omp(*args, int(threads)) if threads > 1 else lib().or_me_search(*args)
    if r != 0:
        raise ValueError(f"or_me_search failed: {r}")
    return f


def _check_call(fn, name, cur, cur_mask, ref, field, K, S, min_support, ssd, ref_mode, rows, extra_pre, extra_post,
                threads=1):
    cur = _c(cur, np.uint8)
    mask = _c(cur_mask, np.uint8)
    P, ref_mode = _params(cur, ref, K, S, min_support, ssd, ref_mode)
    ref = _ref_arr(ref, ref_mode)
    H, W = cur.shape
    y0, y1 = rows if rows is not None else (0, H)
    st = field["status"].copy()
    ev = np.zeros(1, np.uint64)
    err = _c(field["err"], _err_dtype(ref_mode))
    args = [C.byref(P), _p(cur), _p(mask), _p(ref)] + extra_pre + [
        y0, y1, _p(_c(field["alpha"], np.int8)), _p(_c(field["beta"], np.int8)), _p(err),
        _p(_c(field["count"], np.uint8)), _p(st), _p(ev)] + extra_post
    if threads > 1:
        fn = getattr(omp_lib(), name + "_omp")
        args = args + [int(threads)]
    r = fn(*args)
    if r != 0:
        raise ValueError(f"{name} failed: {r}")
    return st, int(ev[0])


def frmc(cur, cur_mask, ref, field, offsets=(-7, -3, -1, 0, 1, 3, 7), K=8, S=8, min_support=8, ssd=False,
         ref_mode=None, rows=None, verify_p4=True, threads=1):
    """FRMC. Returns (new status plane, definitional evaluation count)."""
    offs = np.asarray(offsets, np.int32)
    return _check_call(lib().or_frmc, "or_frmc", cur, cur_mask, ref, field, K, S, min_support, ssd, ref_mode,
                       rows, [_p(offs), len(offs)], [int(verify_p4)], threads)


def rmc(cur, cur_mask, ref, field, K=8, S=8, min_support=8, ssd=False, ref_mode=None, rows=None, verify_p4=True,
        threads=1):
    """RMC. Returns (new status plane, evaluation count)."""
    return _check_call(lib().or_rmc, "or_rmc", cur, cur_mask, ref, field, K, S, min_support, ssd, ref_mode,
                       rows, [], [int(verify_p4)], threads)


def rme(cur, cur_mask, ref, field, K=8, S=8, min_support=8, ssd=False, ref_mode=None, rows=None, threads=1):
    """RME. Returns (new status plane, evaluation count)."""
    return _check_call(lib().or_rme, "or_rme", cur, cur_mask, ref, field, K, S, min_support, ssd, ref_mode,
                       rows, [], [], threads)


def nnc(field, threshold=1, rows=None, pairs=False):
    """NNC (Eq. 1). Returns the new status plane.

    pairs=False: filtered centre vs each valid 4-neighbour (R15, the headline reading).
    pairs=True: the valid 4-neighbours compared with each other (R30)."""
    st = _c(field["status"], np.uint8).copy()
    H, W = st.shape
    y0, y1 = rows if rows is not None else (0, H)
    r = lib().or_nnc_mode(W, H, y0, y1, _p(_c(field["alpha"], np.int8)), _p(_c(field["beta"], np.int8)), _p(st),
                          threshold, 1 if pairs else 0)
    if r != 0:
        raise ValueError(f"or_nnc failed: {r}")
    return st


def median_field(field):
    """The filtered field of Eq. (1): (a~, b~, defined)."""
    st = _c(field["status"], np.uint8)
    H, W = st.shape
    fa = np.zeros((H, W), np.int32)
    fb = np.zeros((H, W), np.int32)
    d = np.zeros((H, W), np.uint8)
    lib().or_median_field(W, H, _p(_c(field["alpha"], np.int8)), _p(_c(field["beta"], np.int8)), _p(st),
                          _p(fa), _p(fb), _p(d))
    return fa, fb, d


def project(field, past_val, past_mask, sum_=None, cnt=None, rows=None):
    """PR. Accumulates into (sum, cnt); returns them."""
    st = _c(field["status"], np.uint8)
    H, W = st.shape
    sum_ = np.zeros((H, W), np.uint32) if sum_ is None else sum_
    cnt = np.zeros((H, W), np.uint8) if cnt is None else cnt
    y0, y1 = rows if rows is not None else (0, H)
    r = lib().or_project(W, H, y0, y1, _p(_c(field["alpha"], np.int8)), _p(_c(field["beta"], np.int8)), _p(st),
                         _p(_c(past_val, np.uint8)), _p(_c(past_mask, np.uint8)), _p(sum_), _p(cnt))
    if r != 0:
        raise ValueError(f"or_project failed: {r}")
    return sum_, cnt


def _probe(fn, cur, cur_mask, ref, y, x, a, b, K, min_support, ssd, ref_mode):
    cur = _c(cur, np.uint8)
    mask = _c(cur_mask, np.uint8)
    P, ref_mode = _params(cur, ref, K, 0, min_support, ssd, ref_mode)
    ref = _ref_arr(ref, ref_mode)
    ei = np.zeros(1, np.uint64)
    ef = np.zeros(1, np.float32)
    ed = np.zeros(1, np.float64)
    n = fn(C.byref(P), _p(cur), _p(mask), _p(ref), y, x, a, b, _p(ei), _p(ef), _p(ed))
    e = {REF_U8: int(ei[0]), REF_F32: float(ef[0]), REF_F32_ACC64: float(ed[0])}[ref_mode]
    return e, int(n)


def cost_fwd(cur, cur_mask, ref, y, x, a, b, K=8, min_support=8, ssd=False, ref_mode=None):
    """(e, n) of the forward matching error of target (y, x) for v = (a, b)."""
    return _probe(lib().or_probe_fwd, cur, cur_mask, ref, y, x, a, b, K, min_support, ssd, ref_mode)


def cost_rev(cur, cur_mask, ref, y, x, a, b, K=8, min_support=8, ssd=False, ref_mode=None):
    """(e', n') of the reverse matching error at x = (y, x) for u = (a, b)."""
    return _probe(lib().or_probe_rev, cur, cur_mask, ref, y, x, a, b, K, min_support, ssd, ref_mode)


# --------------------------------------------------------------------------
# Pair / frame driver ("three previous frames"; SPEC.md:446-449;
# R16 cascade, R19 references)
# --------------------------------------------------------------------------
def pair_chain(inp: dict, K=8, S=8, min_support=8, ssd=False, check="nnc_frmc", threshold=1,
               offsets=(-7, -3, -1, 0, 1, 3, 7), rows=None, ref_mode=None, threads=1):
    """ME -> check -> (field, evals) for one (t, d) pair.

    check: none | rme | rmc | frmc | nnc | nnc_frmc (the paper's cascade: NNC
    rejects, FRMC decides the NNC survivors).
    With ``rows``, ME runs on rows widened by 2 so that NNC sees its halo.
    """
    H = inp["cur"].shape[0]
    mrows = None if rows is None else (max(0, rows[0] - 2), min(H, rows[1] + 2))
    kw = dict(K=K, S=S, min_support=min_support, ssd=ssd, ref_mode=ref_mode)
    kt = dict(kw, threads=threads)
    f = me_search(inp["cur"], inp["cur_mask"], inp["ref"], rows=mrows, **kt)
    ev = 0
    if check == "none":
        pass
    elif check == "rme":
        f["status"], ev = rme(inp["cur"], inp["cur_mask"], inp["ref"], f, rows=rows, **kt)
    elif check == "rmc":
        f["status"], ev = rmc(inp["cur"], inp["cur_mask"], inp["ref"], f, rows=rows, **kt)
    elif check == "frmc":
        f["status"], ev = frmc(inp["cur"], inp["cur_mask"], inp["ref"], f, offsets=offsets, rows=rows, **kt)
    elif check in ("nnc", "nnc_frmc"):
        f["status"] = nnc(f, threshold, rows=rows)
        if check == "nnc_frmc":
            f["status"], ev = frmc(inp["cur"], inp["cur_mask"], inp["ref"], f, offsets=offsets, rows=rows, **kt)
    else:
        raise ValueError(check)
    return f, ev
