"""CPU-only checks of the boundary: libqs.so loads, exports every function include/qs.h declares,
and validates arguments synchronously (before any CUDA call) with the documented codes."""
import ctypes as C
import os
import shutil

import pytest

import paper_2203_09200_b200 as qs


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(qs.LIB_PATH):
        if shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"):
            pytest.skip("libqs.so not built and no nvcc")
        import __graft_entry__
        __graft_entry__.build_libqs()
    return qs.lib()


def test_exports_every_header_symbol(lib):
    names = qs.header_functions()
    assert set(names) >= {"qs_me_search", "qs_me_search_refs", "qs_reverse_check", "qs_frmc", "qs_nnc", "qs_nnc_mode", "qs_project",
                          "qs_last_error", "qs_workspace_size", "qs_version"}
    for n in names:
        assert hasattr(lib, n), n


def test_version_string(lib):
    assert "sm_100a" in qs.qs_version()


FAKE = 0x1000  # never dereferenced: validation rejects before any launch


def _field(ptr=FAKE, pitch=64):
    return qs.qs_field(ptr, ptr, ptr, ptr, ptr, pitch)


def _call_me(lib, roi, prm, cur=FAKE, pitch=64, ws=FAKE, wsb=1 << 30, field=None, fuse=None):
    f = field or _field()
    return lib.qs_me_search(C.c_void_p(cur), C.c_void_p(cur), pitch, C.c_void_p(cur), pitch,
                            C.byref(roi) if roi is not None else None, C.byref(prm),
                            C.byref(fuse) if fuse is not None else None, C.byref(f), None, C.c_void_p(ws), wsb, None)


def test_validation_codes(lib):
    roi = qs.make_roi(64, 64)
    ok = qs.make_params(K=8, S=8)
    assert _call_me(lib, None, ok) == qs.QS_EINVAL
    assert _call_me(lib, qs.make_roi(63, 64), ok) == qs.QS_EDIM          # odd frame (quarter sampling)
    assert _call_me(lib, qs.make_roi(64, 64, 10, 5), ok) == qs.QS_EDIM   # rows reversed
    assert _call_me(lib, roi, qs.make_params(K=10, S=8)) == qs.QS_EINVAL
    assert _call_me(lib, roi, qs.qs_me_params(8, 4, 8, 8, 0, 0)) == qs.QS_EINVAL   # non-square
    assert _call_me(lib, roi, qs.make_params(K=8, S=40)) == qs.QS_EINVAL
    assert _call_me(lib, roi, qs.make_params(K=8, S=8, min_support=0)) == qs.QS_EINVAL
    assert _call_me(lib, roi, ok, cur=FAKE + 4) == qs.QS_EALIGN
    assert _call_me(lib, roi, ok, pitch=72) == qs.QS_EALIGN
    assert _call_me(lib, roi, ok, pitch=48) == qs.QS_EDIM               # pitch < width
    # halo rows missing from the buffer window
    assert _call_me(lib, qs.make_roi(64, 64, 20, 40, 16, 28), ok) == qs.QS_EDIM
    # workspace too small
    assert _call_me(lib, roi, ok, wsb=16) == qs.QS_EDIM
    # FRMC offsets must contain 0 and lie in [-S, S]
    assert _call_me(lib, roi, ok, fuse=qs.make_checks(offsets=(-1, 1))) == qs.QS_EINVAL
    assert _call_me(lib, roi, ok, fuse=qs.make_checks(offsets=(-9, 0, 9))) == qs.QS_EINVAL
    assert "offset" in qs.qs_last_error()


def test_workspace_size(lib):
    roi = qs.make_roi(1920, 1080)
    n = qs.qs_workspace_size(roi, qs.make_params(K=8, S=24, ref_f32=True))
    assert n >= (1080 + 48) * (1920 + 48) * 8 and n % 256 == 0


def test_other_entry_points_validate(lib):
    roi = qs.make_roi(64, 64)
    prm = qs.make_params(K=8, S=8)
    f = _field()
    assert lib.qs_nnc(C.byref(f), C.byref(roi), -1, None) == qs.QS_EINVAL
    assert lib.qs_nnc(C.byref(f), C.byref(qs.make_roi(64, 64, 8, 16, 8, 8)), 1, None) == qs.QS_EDIM
    assert lib.qs_reverse_check(7, C.c_void_p(FAKE), C.c_void_p(FAKE), 64, C.c_void_p(FAKE), 64, C.byref(roi),
                                C.byref(prm), C.byref(f), None, None, 0, None) == qs.QS_EINVAL
    assert lib.qs_project(C.byref(f), C.c_void_p(FAKE), C.c_void_p(FAKE), 64, C.byref(roi), None, None, 64,
                          None) == qs.QS_EINVAL
    arr = (C.c_int8 * 2)(0, 1)
    assert lib.qs_frmc(C.c_void_p(FAKE), C.c_void_p(FAKE), 64, C.c_void_p(FAKE), 64, C.byref(roi), C.byref(prm),
                       C.cast(arr, C.c_void_p), 0, C.byref(f), None, None) == qs.QS_EINVAL


def test_me_search_refs_validates(lib):
    roi = qs.make_roi(64, 64)
    prm = qs.make_params(K=8, S=8)
    slot = qs.qs_workspace_size(roi, prm)
    refs = (C.c_void_p * 3)(FAKE, FAKE, FAKE)
    outs = (qs.qs_field * 3)(_field(), _field(), _field())

    def call(n, wsb, cur=FAKE, r=refs, proj=None):
        return lib.qs_me_search_refs(C.c_void_p(cur), C.c_void_p(cur), 64, n, C.cast(r, C.c_void_p), 64,
                                     C.byref(roi), C.byref(prm), None, C.cast(outs, C.c_void_p),
                                     C.byref(proj) if proj is not None else None, None,
                                     C.c_void_p(FAKE), wsb, None)
    assert call(-1, 3 * slot) == qs.QS_EINVAL
    assert call(0, 0) == qs.QS_OK                        # no references: nothing to do
    assert call(3, 3 * slot - 1) == qs.QS_EDIM           # one slot of workspace per reference
    assert "slots" in qs.qs_last_error()
    assert call(3, 3 * slot, cur=FAKE + 4) == qs.QS_EALIGN
    bad = (C.c_void_p * 3)(FAKE, FAKE + 8, FAKE)
    assert call(3, 3 * slot, r=bad) == qs.QS_EALIGN      # every reference plane is checked
    pv = (C.c_void_p * 3)(FAKE, FAKE, FAKE)
    pj = qs.qs_projection(C.cast(pv, C.c_void_p), C.cast(pv, C.c_void_p), 64, FAKE, FAKE, 64)
    pj_null = qs.qs_projection(C.cast(pv, C.c_void_p), C.cast(pv, C.c_void_p), 64, None, FAKE, 64)
    assert call(3, 3 * slot, proj=pj_null) == qs.QS_EINVAL          # sum is NULL
    pj_pitch = qs.qs_projection(C.cast(pv, C.c_void_p), C.cast(pv, C.c_void_p), 64, FAKE, FAKE, 66)
    assert call(3, 3 * slot, proj=pj_pitch) == qs.QS_EALIGN         # cnt words: acc_pitch % 4
    pj_cnt = qs.qs_projection(C.cast(pv, C.c_void_p), C.cast(pv, C.c_void_p), 64, FAKE, FAKE + 1, 64)
    assert call(3, 3 * slot, proj=pj_cnt) == qs.QS_EALIGN
    pv_bad = (C.c_void_p * 3)(FAKE, FAKE, FAKE + 4)
    pj_pv = qs.qs_projection(C.cast(pv_bad, C.c_void_p), C.cast(pv, C.c_void_p), 64, FAKE, FAKE, 64)
    assert call(3, 3 * slot, proj=pj_pv) == qs.QS_EALIGN            # every past plane is checked
    assert pj is not None


def test_nnc_mode_validates(lib):
    roi = qs.make_roi(64, 64)
    f = _field()
    assert lib.qs_nnc_mode(C.byref(f), C.byref(roi), 1, 3, None) == qs.QS_EINVAL
    assert lib.qs_nnc_mode(C.byref(f), C.byref(roi), 1, 0, None) == qs.QS_EINVAL
    chk = qs.make_checks()
    chk.nnc = 5
    assert _call_me(lib, roi, qs.make_params(K=8, S=8), fuse=chk) == qs.QS_EINVAL
    assert "nnc mode" in qs.qs_last_error()
