"""paper_2203_09200_b200 -- B200-native hot path of arxiv 2203.09200.

Thin ctypes binding over ``libqs.so`` (the C ABI declared in ``include/qs.h``):
argument marshalling only.  Every step of the path -- motion estimation (ME),
the consistency checks NNC / FRMC / RMC / RME and the projection PR -- runs in
the CUDA kernels of ``csrc/``.  PyTorch provides device memory and streams.

There is no CPU fallback: if ``libqs.so`` is missing or no CUDA device is
present, the calls raise.  This package never imports ``oracle`` (the CPU
oracle is test infrastructure only).

The functions keep the ABI's names (``qs_me_search``, ``qs_reverse_check``,
``qs_frmc``, ``qs_nnc``, ``qs_project``, ...) and take torch tensors.
"""
from __future__ import annotations

import ctypes as C
import os
import re
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# QS_LIBQS selects another build of the same sources (test infrastructure: libqs_checked.so, the
# bounds-checked build); the default is the product library.
LIB_PATH = os.environ.get("QS_LIBQS") or os.path.join(_HERE, "libqs.so")
if not os.path.isabs(LIB_PATH):
    LIB_PATH = os.path.join(_HERE, LIB_PATH)
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "qs.h")

# Return codes, statuses, enums (include/qs.h).
QS_OK, QS_EINVAL, QS_EDIM, QS_EALIGN, QS_ECUDA = 0, -1, -2, -3, -4
QS_NOT_TARGET, QS_INVALID, QS_CANDIDATE, QS_ACCEPTED, QS_REJECTED = 0, 1, 2, 3, 4
QS_SAD, QS_SSD = 0, 1
QS_REF_U8, QS_REF_F32 = 0, 1
QS_RME, QS_RMC = 0, 1
QS_NNC_CENTRE, QS_NNC_PAIRS = 1, 2

# PAPER.md:104 (§3.1.1): FRMC tests "only motions in the set {-7,-3,-1,0,1,3,7}".
PAPER_FRMC_OFFSETS = (-7, -3, -1, 0, 1, 3, 7)


class QsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"qs error {code}: {msg}")
        self.code = code


class qs_me_params(C.Structure):
    _fields_ = [("K_h", C.c_int32), ("K_w", C.c_int32), ("S", C.c_int32), ("min_support", C.c_int32),
                ("err", C.c_int32), ("ref_type", C.c_int32)]


class qs_roi(C.Structure):
    _fields_ = [("frame_w", C.c_int32), ("frame_h", C.c_int32), ("y_begin", C.c_int32), ("y_end", C.c_int32),
                ("buf_y0", C.c_int32), ("buf_rows", C.c_int32)]


class qs_field(C.Structure):
    _fields_ = [("alpha", C.c_void_p), ("beta", C.c_void_p), ("err", C.c_void_p), ("count", C.c_void_p),
                ("status", C.c_void_p), ("pitch", C.c_int64)]


class qs_checks(C.Structure):
    _fields_ = [("nnc", C.c_int32), ("nnc_threshold", C.c_int32), ("frmc", C.c_int32),
                ("offsets", C.c_void_p), ("n_offsets", C.c_int32)]


class qs_projection(C.Structure):
    _fields_ = [("past_val", C.c_void_p), ("past_mask", C.c_void_p), ("past_pitch", C.c_int64),
                ("sum", C.c_void_p), ("cnt", C.c_void_p), ("acc_pitch", C.c_int64)]


_lib = None


def lib() -> C.CDLL:
    """Load libqs.so (built by ``__graft_entry__.build()``); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t
        P = C.POINTER
        L.qs_workspace_size.argtypes = [P(qs_roi), i32, i32, P(qs_me_params), P(sz)]
        L.qs_me_search.argtypes = [vp, vp, i64, vp, i64, P(qs_roi), P(qs_me_params), P(qs_checks), P(qs_field),
                                   vp, vp, sz, vp]
        L.qs_me_search_refs.argtypes = [vp, vp, i64, i32, vp, i64, P(qs_roi), P(qs_me_params), P(qs_checks),
                                        vp, P(qs_projection), vp, vp, sz, vp]
        L.qs_reverse_check.argtypes = [i32, vp, vp, i64, vp, i64, P(qs_roi), P(qs_me_params), P(qs_field),
                                       vp, vp, sz, vp]
        L.qs_frmc.argtypes = [vp, vp, i64, vp, i64, P(qs_roi), P(qs_me_params), vp, i32, P(qs_field), vp, vp]
        L.qs_nnc.argtypes = [P(qs_field), P(qs_roi), i32, vp]
        L.qs_nnc_mode.argtypes = [P(qs_field), P(qs_roi), i32, i32, vp]
        L.qs_project.argtypes = [P(qs_field), vp, vp, i64, P(qs_roi), vp, vp, i64, vp]
        for f in ("qs_workspace_size", "qs_me_search", "qs_me_search_refs", "qs_reverse_check", "qs_frmc", "qs_nnc", "qs_nnc_mode", "qs_project"):
            getattr(L, f).restype = C.c_int
        L.qs_certify_stats.argtypes = [P(C.c_int64), i32]
        L.qs_certify_stats.restype = C.c_int
        L.qs_profile_enable.argtypes = [i32]
        L.qs_profile_read.argtypes = [C.c_char_p, P(C.c_double), P(C.c_int64)]
        L.qs_profile_reset.argtypes = []
        for f in ("qs_profile_enable", "qs_profile_read", "qs_profile_reset"):
            getattr(L, f).restype = C.c_int
        L.qs_last_error.restype = C.c_char_p
        L.qs_last_error.argtypes = []
        L.qs_version.restype = C.c_char_p
        L.qs_version.argtypes = []
        _lib = L
    return _lib


def header_functions() -> list[str]:
    """Names of the functions declared in include/qs.h."""
    src = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(qs_\w+)\s*\(", src, flags=re.M)))


def qs_last_error() -> str:
    return lib().qs_last_error().decode()


def qs_version() -> str:
    return lib().qs_version().decode()


def qs_profile_enable(on: bool = True):
    lib().qs_profile_enable(int(on))


def qs_profile_read(kernel: str = "*"):
    """(total device ms, launches) of the kernel's launches recorded while profiling was enabled."""
    t = C.c_double(0)
    n = C.c_int64(0)
    _check(lib().qs_profile_read(kernel.encode(), C.byref(t), C.byref(n)))
    return t.value, n.value


def qs_profile_reset():
    lib().qs_profile_reset()


PROFILE_KERNELS = ("me_box", "epilogue", "finalize", "nnc", "revgrid", "rme_decide", "project", "certify")


def qs_certify_stats(reset: bool = False) -> int:
    """Float references: outputs recomputed exactly by the certify kernel since the last reset."""
    n = C.c_int64(0)
    _check(lib().qs_certify_stats(C.byref(n), int(reset)))
    return n.value


def _check(rc: int):
    if rc != QS_OK:
        raise QsError(rc, qs_last_error())


# ---------------------------------------------------------------------------
# Tensors <-> ABI
# ---------------------------------------------------------------------------
def pitched(rows: int, cols: int, dtype: torch.dtype, device="cuda", fill=0) -> torch.Tensor:
    """[rows, cols] view of a buffer whose row pitch is a multiple of 16 bytes."""
    esz = torch.empty((), dtype=dtype).element_size()
    pcols = ((cols * esz + 15) // 16) * 16 // esz
    base = torch.full((max(rows, 1), max(pcols, 1)), fill, dtype=dtype, device=device)
    return base[:rows, :cols]


def to_plane(x, device="cuda", dtype=None) -> torch.Tensor:
    """Copy a 2-D array (numpy or torch) into a 16-byte-pitched device plane."""
    t = torch.as_tensor(x)
    if dtype is not None:
        t = t.to(dtype)
    out = pitched(t.shape[0], t.shape[1], t.dtype, device)
    out.copy_(t.to(device))
    return out


def _pitch_bytes(t: torch.Tensor) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise ValueError("plane must be 2-D with unit column stride")
    return t.stride(0) * t.element_size()


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def make_roi(frame_w: int, frame_h: int, y_begin=0, y_end=None, buf_y0=0, buf_rows=None) -> qs_roi:
    y_end = frame_h if y_end is None else y_end
    buf_rows = frame_h - buf_y0 if buf_rows is None else buf_rows
    return qs_roi(frame_w, frame_h, y_begin, y_end, buf_y0, buf_rows)


def make_params(K=8, S=16, min_support=8, ssd=False, ref_f32=False) -> qs_me_params:
    return qs_me_params(K, K, S, min_support, QS_SSD if ssd else QS_SAD, QS_REF_F32 if ref_f32 else QS_REF_U8)


def make_checks(nnc=True, frmc=True, threshold=1, offsets=PAPER_FRMC_OFFSETS, nnc_pairs=False):
    """nnc_pairs: NNC's second reading (QS_NNC_PAIRS, R30) instead of the headline centre reading."""
    arr = (C.c_int8 * len(offsets))(*offsets)
    mode = (QS_NNC_PAIRS if nnc_pairs else QS_NNC_CENTRE) if nnc else 0
    chk = qs_checks(mode, threshold, int(frmc), C.cast(arr, C.c_void_p), len(offsets))
    chk._keep = arr
    return chk


@dataclass
class Field:
    """Device motion field planes [rows, W] with a shared element pitch."""
    alpha: torch.Tensor
    beta: torch.Tensor
    err: torch.Tensor
    count: torch.Tensor
    status: torch.Tensor

    @staticmethod
    def alloc(rows: int, W: int, ref_f32: bool, device="cuda") -> "Field":
        pc = ((W + 15) // 16) * 16
        mk = lambda dt: torch.zeros((max(rows, 1), pc), dtype=dt, device=device)[:rows, :W]
        return Field(mk(torch.int8), mk(torch.int8), mk(torch.float32 if ref_f32 else torch.int32),
                     mk(torch.uint8), mk(torch.uint8))

    def c(self) -> qs_field:
        p = self.alpha.stride(0)
        for t in (self.beta, self.err, self.count, self.status):
            if t.stride(0) != p:
                raise ValueError("field planes must share one element pitch")
        return qs_field(self.alpha.data_ptr(), self.beta.data_ptr(), self.err.data_ptr(), self.count.data_ptr(),
                        self.status.data_ptr(), p)

    def numpy(self) -> dict:
        return {k: getattr(self, k).cpu().numpy() for k in ("alpha", "beta", "err", "count", "status")}


def qs_workspace_size(roi: qs_roi, params: qs_me_params) -> int:
    n = C.c_size_t(0)
    _check(lib().qs_workspace_size(C.byref(roi), roi.frame_w, roi.frame_h, C.byref(params), C.byref(n)))
    return n.value


def workspace(roi: qs_roi, params: qs_me_params, device="cuda", n_refs: int = 1) -> torch.Tensor:
    """Device scratch for qs_me_search (n_refs = 1) or qs_me_search_refs (n_refs slots)."""
    return torch.empty(max(qs_workspace_size(roi, params) * max(n_refs, 1), 16), dtype=torch.uint8, device=device)


def qs_me_search_refs(cur, cur_mask, refs, roi: qs_roi, params: qs_me_params, outs, fuse: qs_checks | None = None,
                      eval_count: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None,
                      project=None):
    """qs_me_search for the pairs (cur, refs[i]) -> outs[i] of one frame in one launch per kernel.

    project = (past_vals, past_masks, sum, cnt): PR of every reference fused into the same launch
    (as qs_project(outs[i], past_vals[i], past_masks[i], roi, sum, cnt) for each i).
    outs = None with project: projection-only (no field planes written)."""
    if _pitch_bytes(cur) != _pitch_bytes(cur_mask):
        raise ValueError("cur and cur_mask must share one pitch")
    n = len(refs)
    if outs is not None and len(outs) != n:
        raise ValueError("refs and outs differ in length")
    if outs is None and project is None:
        raise ValueError("outs=None (projection-only) needs project=")
    pitches = {_pitch_bytes(r) for r in refs}
    if len(pitches) > 1:
        raise ValueError("reference planes must share one pitch")
    if ws is None:
        ws = workspace(roi, params, cur.device, n)
    rp = (C.c_void_p * max(n, 1))(*[r.data_ptr() for r in refs])
    fc = (qs_field * max(n, 1))(*[o.c() for o in outs]) if outs is not None else None
    pj = None
    if project is not None:
        pvs, pms, acc_sum, acc_cnt = project
        if len(pvs) != n or len(pms) != n:
            raise ValueError("one past_val / past_mask plane per reference")
        pp = {_pitch_bytes(x) for x in list(pvs) + list(pms)}
        if len(pp) > 1:
            raise ValueError("past planes must share one pitch")
        if acc_sum.stride(0) != acc_cnt.stride(0):
            raise ValueError("sum and cnt must share one element pitch")
        pva = (C.c_void_p * max(n, 1))(*[x.data_ptr() for x in pvs])
        pma = (C.c_void_p * max(n, 1))(*[x.data_ptr() for x in pms])
        pj = qs_projection(C.cast(pva, C.c_void_p), C.cast(pma, C.c_void_p), pp.pop() if pp else 16,
                           acc_sum.data_ptr(), acc_cnt.data_ptr(), acc_sum.stride(0))
        pj._keep = (pva, pma)
    _check(lib().qs_me_search_refs(_ptr(cur), _ptr(cur_mask), _pitch_bytes(cur), n, C.cast(rp, C.c_void_p),
                                   pitches.pop() if pitches else 16, C.byref(roi), C.byref(params),
                                   C.byref(fuse) if fuse is not None else None,
                                   C.cast(fc, C.c_void_p) if fc is not None else None,
                                   C.byref(pj) if pj is not None else None,
                                   _ptr(eval_count), _ptr(ws), ws.numel(), _stream(stream)))


def qs_me_search(cur, cur_mask, ref, roi: qs_roi, params: qs_me_params, out: Field, fuse: qs_checks | None = None,
                 eval_count: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None):
    if _pitch_bytes(cur) != _pitch_bytes(cur_mask):
        raise ValueError("cur and cur_mask must share one pitch")
    if ws is None:
        ws = workspace(roi, params, cur.device)
    fc = out.c()
    _check(lib().qs_me_search(_ptr(cur), _ptr(cur_mask), _pitch_bytes(cur), _ptr(ref), _pitch_bytes(ref),
                              C.byref(roi), C.byref(params), C.byref(fuse) if fuse is not None else None,
                              C.byref(fc), _ptr(eval_count), _ptr(ws), ws.numel(), _stream(stream)))


def qs_reverse_check(mode: int, cur, cur_mask, ref, roi: qs_roi, params: qs_me_params, io: Field,
                     eval_count=None, ws=None, stream=None):
    if ws is None and mode == QS_RME:
        ws = workspace(roi, params, cur.device)
    fc = io.c()
    _check(lib().qs_reverse_check(mode, _ptr(cur), _ptr(cur_mask), _pitch_bytes(cur), _ptr(ref), _pitch_bytes(ref),
                                  C.byref(roi), C.byref(params), C.byref(fc), _ptr(eval_count), _ptr(ws),
                                  0 if ws is None else ws.numel(), _stream(stream)))


def qs_frmc(cur, cur_mask, ref, roi: qs_roi, params: qs_me_params, io: Field, offsets=PAPER_FRMC_OFFSETS,
            eval_count=None, stream=None):
    arr = (C.c_int8 * len(offsets))(*offsets)
    fc = io.c()
    _check(lib().qs_frmc(_ptr(cur), _ptr(cur_mask), _pitch_bytes(cur), _ptr(ref), _pitch_bytes(ref), C.byref(roi),
                         C.byref(params), C.cast(arr, C.c_void_p), len(offsets), C.byref(fc), _ptr(eval_count),
                         _stream(stream)))


def qs_nnc(io: Field, roi: qs_roi, threshold: int = 1, stream=None):
    fc = io.c()
    _check(lib().qs_nnc(C.byref(fc), C.byref(roi), threshold, _stream(stream)))


def qs_nnc_mode(io: Field, roi: qs_roi, threshold: int = 1, mode: int = QS_NNC_CENTRE, stream=None):
    fc = io.c()
    _check(lib().qs_nnc_mode(C.byref(fc), C.byref(roi), threshold, mode, _stream(stream)))


def qs_project(f: Field, past_val, past_mask, roi: qs_roi, sum_: torch.Tensor, cnt: torch.Tensor, stream=None):
    if _pitch_bytes(past_val) != _pitch_bytes(past_mask):
        raise ValueError("past_val and past_mask must share one pitch")
    if sum_.stride(0) != cnt.stride(0):
        raise ValueError("sum and cnt must share one element pitch")
    fc = f.c()
    _check(lib().qs_project(C.byref(fc), _ptr(past_val), _ptr(past_mask), _pitch_bytes(past_val), C.byref(roi),
                            _ptr(sum_), _ptr(cnt), sum_.stride(0), _stream(stream)))


def alloc_acc(rows: int, W: int, device="cuda"):
    """Projection accumulators (sum uint32 as int32 storage, cnt uint8), one element pitch."""
    pc = ((W + 15) // 16) * 16
    s = torch.zeros((max(rows, 1), pc), dtype=torch.int32, device=device)[:rows, :W]
    c = torch.zeros((max(rows, 1), pc), dtype=torch.uint8, device=device)[:rows, :W]
    return s, c
