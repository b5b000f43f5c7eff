// qs_api.cu -- the extern "C" boundary of libqs (include/qs.h): argument
// validation, the one-time candidate tables, and the launch sequences.
// Everything here is host code; every step of the path runs in the kernels of
// me_box.cu and checks.cu.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include <cudaTypedefs.h>

#include "qs_internal.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char *what) {
    return fail(QS_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---------------------------------------------------------------------------
// Candidate tables: rank order (|a|+|b|, a, b) ascending (R7).
// ---------------------------------------------------------------------------
std::mutex g_tab_mu;
std::map<std::pair<int, int>, qs::CandTables *> g_tabs;

// ---------------------------------------------------------------------------
// Profiler: CUDA events around each launch, on the launch stream.
// ---------------------------------------------------------------------------
enum ProfKernel { P_ME_BOX = 0, P_FINALIZE, P_NNC, P_REVGRID, P_RME_DECIDE, P_PROJECT, P_EPILOGUE, P_CERTIFY, P_COUNT };
const char *kProfNames[P_COUNT] = {"me_box", "finalize", "nnc", "revgrid", "rme_decide", "project", "epilogue",
                                   "certify"};

// {-7,-3,-1,0,1,3,7}, in any order.
bool is_paper_offsets(const int8_t *o, int n) {
    if (n != 7) return false;
    int seen = 0;
    for (int i = 0; i < 7; ++i) {
        const int v = o[i];
        const int idx = v == -7 ? 0 : v == -3 ? 1 : v == -1 ? 2 : v == 0 ? 3 : v == 1 ? 4 : v == 3 ? 5 : v == 7 ? 6 : -1;
        if (idx < 0) return false;
        seen |= 1 << idx;
    }
    return seen == 0x7f;
}

struct ProfRec {
    int kernel;
    cudaEvent_t start, stop;
};

struct Profiler {
    std::mutex mu;
    bool on = false;
    std::vector<cudaEvent_t> pool;
    std::vector<ProfRec> recs;
    cudaEvent_t get() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e = nullptr;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        return e;
    }
} g_prof;

// RAII bracket: records start on construction and stop on destruction when enabled.
struct ProfScope {
    int kernel;
    cudaStream_t s;
    cudaEvent_t a = nullptr, b = nullptr;
    ProfScope(int k, cudaStream_t st) : kernel(k), s(st) {
        std::lock_guard<std::mutex> lk(g_prof.mu);
        if (!g_prof.on) return;
        a = g_prof.get();
        b = g_prof.get();
        if (a && b) cudaEventRecord(a, s);
    }
    ~ProfScope() {
        if (!a || !b) return;
        cudaEventRecord(b, s);
        std::lock_guard<std::mutex> lk(g_prof.mu);
        g_prof.recs.push_back({kernel, a, b});
    }
};

}  // namespace

namespace qs {

const CandTables *cand_tables(int S, const char **err) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { *err = "cudaGetDevice failed"; return nullptr; }
    std::lock_guard<std::mutex> lk(g_tab_mu);
    auto it = g_tabs.find({dev, S});
    if (it != g_tabs.end()) return it->second;
    std::vector<std::pair<int, int>> v;
    for (int a = -S; a <= S; ++a)
        for (int b = -S; b <= S; ++b) v.push_back({a, b});
    std::stable_sort(v.begin(), v.end(), [](const std::pair<int, int> &x, const std::pair<int, int> &y) {
        const int lx = std::abs(x.first) + std::abs(x.second), ly = std::abs(y.first) + std::abs(y.second);
        if (lx != ly) return lx < ly;
        if (x.first != y.first) return x.first < y.first;
        return x.second < y.second;
    });
    const int n = (int)v.size();
    std::vector<int32_t> canon(n), chunked;
    for (int r = 0; r < n; ++r) canon[r] = (v[r].first & 0xff) | ((v[r].second & 0xff) << 8);
    const int n_chunks = chunk_count(S);
    std::vector<int32_t> off(n_chunks + 1, 0);
    for (int c = 0; c < n_chunks; ++c) {
        const int alo = chunk_alo(S, c), ahi = chunk_ahi(S, c);
        off[c] = (int)chunked.size();
        for (int r = 0; r < n; ++r)   // rank order inside the chunk
            if (v[r].first >= alo && v[r].first <= ahi && ((v[r].first - alo) & 1) == 0)
                chunked.push_back(canon[r] | (r << 16));
    }
    off[n_chunks] = (int)chunked.size();
    auto *t = new CandTables;
    t->S = S;
    t->n = n;
    t->n_chunks = n_chunks;
    if (cudaMalloc(&t->canon, sizeof(int32_t) * n) != cudaSuccess ||
        cudaMalloc(&t->chunked, sizeof(int32_t) * n) != cudaSuccess ||
        cudaMalloc(&t->chunk_off, sizeof(int32_t) * (n_chunks + 1)) != cudaSuccess ||
        cudaMemcpy(t->canon, canon.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(t->chunked, chunked.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(t->chunk_off, off.data(), sizeof(int32_t) * (n_chunks + 1), cudaMemcpyHostToDevice) !=
            cudaSuccess) {
        *err = "cudaMalloc/cudaMemcpy of the candidate tables failed";
        delete t;
        return nullptr;
    }
    g_tabs[{dev, S}] = t;
    return t;
}

}  // namespace qs

namespace {

using namespace qs;

struct Roi {
    int W, H, y0, y1, b0, br;
};

int check_roi(const qs_roi *roi, Roi *r) {
    if (!roi) return fail(QS_EINVAL, "roi is NULL (it carries the frame size)");
    r->W = roi->frame_w;
    r->H = roi->frame_h;
    r->y0 = roi->y_begin;
    r->y1 = roi->y_end;
    r->b0 = roi->buf_y0;
    r->br = roi->buf_rows;
    if (r->W <= 0 || r->H <= 0 || (r->W & 1) || (r->H & 1))
        return fail(QS_EDIM, "frame %dx%d: quarter sampling needs positive even dimensions", r->W, r->H);
    if (r->y0 < 0 || r->y1 > r->H || r->y0 > r->y1) return fail(QS_EDIM, "rows [%d,%d) outside frame of %d", r->y0, r->y1, r->H);
    if (r->b0 < 0 || r->br < 0 || r->b0 + r->br > r->H)
        return fail(QS_EDIM, "buffer rows [%d,%d) outside frame of %d", r->b0, r->b0 + r->br, r->H);
    return QS_OK;
}

// Rows [lo, hi) clipped to the frame must be held by the buffer window.
int need_rows(const Roi &r, int lo, int hi, const char *what) {
    lo = std::max(lo, 0);
    hi = std::min(hi, r.H);
    if (lo >= hi) return QS_OK;
    if (lo < r.b0 || hi > r.b0 + r.br)
        return fail(QS_EDIM, "%s needs rows [%d,%d) but the buffers hold [%d,%d)", what, lo, hi, r.b0, r.b0 + r.br);
    return QS_OK;
}

int check_params(const qs_me_params *p) {
    if (!p) return fail(QS_EINVAL, "params is NULL");
    if (p->K_h != p->K_w || p->K_h < 1 || p->K_h > 9)
        return fail(QS_EINVAL, "template %dx%d: this build supports square K in [1,9]", p->K_h, p->K_w);
    if (p->S < 0 || p->S > 32) return fail(QS_EINVAL, "S=%d outside [0,32]", p->S);
    if (p->min_support < 1) return fail(QS_EINVAL, "min_support=%d < 1", p->min_support);
    if (p->err != QS_SAD && p->err != QS_SSD) return fail(QS_EINVAL, "err=%d", p->err);
    if (p->ref_type != QS_REF_U8 && p->ref_type != QS_REF_F32) return fail(QS_EINVAL, "ref_type=%d", p->ref_type);
    return QS_OK;
}

int check_plane(const void *ptr, int64_t pitch, int64_t min_pitch, const char *name) {
    if (!ptr) return fail(QS_EINVAL, "%s is NULL", name);
    if (!aligned16(ptr) || (pitch & 15)) return fail(QS_EALIGN, "%s: base and pitch must be 16-byte aligned", name);
    if (pitch < min_pitch) return fail(QS_EDIM, "%s: pitch %lld < %lld", name, (long long)pitch, (long long)min_pitch);
    return QS_OK;
}

int check_field(const qs_field *f, int W, bool need_err_count) {
    if (!f) return fail(QS_EINVAL, "field is NULL");
    if (!f->alpha || !f->beta || !f->status || (need_err_count && (!f->err || !f->count)))
        return fail(QS_EINVAL, "field plane is NULL");
    if (f->pitch < W) return fail(QS_EDIM, "field pitch %lld < width %d", (long long)f->pitch, W);
    if (f->err && (reinterpret_cast<uintptr_t>(f->err) & 3)) return fail(QS_EALIGN, "field err plane not 4-byte aligned");
    return QS_OK;
}

FieldView view(const qs_field *f) { return FieldView{f->alpha, f->beta, f->err, f->count, f->status, f->pitch}; }

size_t al256(size_t b) { return (b + 255) & ~size_t(255); }
size_t me_keys_bytes(const Roi &r) {
    return sizeof(unsigned long long) * (size_t)std::max(0, std::min(r.H, r.y1 + 2) - std::max(0, r.y0 - 2)) * r.W;
}
size_t rme_keys_bytes(const Roi &r, int S) {
    return sizeof(unsigned long long) * (size_t)(r.y1 - r.y0 + 2 * S) * (size_t)(r.W + 2 * S);
}
// Workspace slot: the 64-bit key plane, then (float references) the 32-bit second plane of the
// certified argmin.  qs_me_search_refs lays out the key planes of
// its n slots first and their second planes after them.
// Workspace layout of one call over n slots (key planes of kb bytes each): the n key planes; for
// float references their n second planes, the certify list (one 4-byte entry per 16 outputs; a
// full list only slows the certify kernel down) and its counter; then, for qs_me_search with K != 8
// and NNC, a scratch field (8 B per pixel, like the keys) for the ME rows [y0-2, y1+2): NNC reads
// the halo rows there and only the roi's rows reach the caller's field.
struct WsLayout {
    size_t keys, s2, list, count, scratch, total;
    size_t kba, s2a;
    int cap;
};
WsLayout ws_layout(size_t kb, int n, bool f32, bool scratch) {
    WsLayout L{};
    L.kba = al256(kb);
    L.s2a = al256(kb / 2);
    size_t off = 0;
    L.keys = off;
    off += n * L.kba;
    L.s2 = off;
    L.cap = 0;
    if (f32) {
        off += n * L.s2a;
        L.cap = (int)std::max<size_t>(32, n * (kb / 8) / 16);
        L.list = off;
        off += al256(4 * (size_t)L.cap);
        L.count = off;
        off += 256;
    }
    L.scratch = off;
    if (scratch) off += L.kba;
    L.total = off;
    return L;
}
size_t ws_slot_bytes(const Roi &r, int S) {
    const size_t me = me_keys_bytes(r), rme = rme_keys_bytes(r, S);
    return std::max(ws_layout(me, 1, true, true).total, ws_layout(rme, 1, true, false).total);
}

// uint8 SAD interior tiles: the integer packed body (default) or the fp32 body (QS_U8_BODY=float;
// kept for the measured comparison in DESIGN.md).
int u8_int_body() {
    const char *e = getenv("QS_U8_BODY");   // read per call (cheap), so a process can switch
    return (e && !strcmp(e, "float")) ? 0 : 1;
}

// TMA staging of the float reference window (me_box quad body): QS_TMA=1
// enables it (measured against the cp.async staging; see DESIGN.md for the default).
int tma_enabled() {
    const char *e = getenv("QS_TMA");   // read per call (cheap), so a process can switch
    return (e && !strcmp(e, "1")) ? 1 : 0;
}

// Float-reference K = 8 forward me_box as two kernels, border tiles (phase 2 in support runs) then
// interior tiles (default; QS_SPLIT=0 selects the single kernel for the measured comparison in DESIGN.md).
int split_tiles_enabled() {
    const char *e = getenv("QS_SPLIT");   // read per call (cheap), so a process can switch
    return (e && !strcmp(e, "0")) ? 0 : (e && !strcmp(e, "2")) ? 2 : 1;
}

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }();
    return fn;
}

// Descriptors for slots 0..n-1 of a float-reference K = 8 forward launch: the buffer viewed as
// [buf_rows / 2][2][W] floats (row pairs, parity, column), box [tma_rows][1][tma_cols], NaN fill.
// Leaves a.tma = 0 (cp.async staging) when disabled or not applicable (odd buffer rows).
void set_tma(BoxArgs &a, int n) {
    a.tma = 0;
    // The box's first column px0 - 4 - S must sit on a 16-byte boundary (tiles start at multiples of
    // 64 columns): S % 4 == 0 (config 4's S = 24; other S keep the cp.async staging).
    if (!tma_enabled() || !a.ref_f32 || (a.buf_rows & 1) || a.buf_rows < 2 || (a.S & 3)) return;
    PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
    if (!enc) return;
    const int cols = (kQWinColsHost + 2 * a.S + 3) & ~3;
    const int rows = (kQWinRowsHost + kChunkSpan - 1 + 1) / 2;
    for (int i = 0; i < n; ++i) {
        const cuuint64_t dims[3] = {(cuuint64_t)a.W, 2, (cuuint64_t)(a.buf_rows / 2)};
        const cuuint64_t strides[2] = {(cuuint64_t)a.ref.pitch, (cuuint64_t)(2 * a.ref.pitch)};
        const cuuint32_t box[3] = {(cuuint32_t)cols, 1, (cuuint32_t)rows};
        const cuuint32_t estr[3] = {1, 1, 1};
        if (enc(&a.tmap[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<uint8_t *>(a.ref_p[i]), dims, strides, box,
                estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NAN_REQUEST_ZERO_FMA) != CUDA_SUCCESS)
            return;
    }
    a.tma_cols = cols;
    a.tma_rows = rows;
    a.tma = 1;
}

// Tile rows of a forward K = 8 launch over output rows [lo, hi): the grid offset (rows of the first
// tile above lo; lo - offset even) with the fewest tile rows whose windows and candidates reach outside the frame or the
// buffer (those run the slower border body), then the fewest tile rows.  Results do not depend on it.
void place_tile_rows(BoxArgs &a, const Roi &r, int lo, int hi) {
    const int S = a.S, top = std::max(0, r.b0), bot = std::min(r.H, r.b0 + r.br) - 1;
    int best_off = 0, best_border = 1 << 30, best_rows = 1 << 30;
    // lo - off even: the quad body's 2x2 blocks stay on the mask's block grid (odd tile rows would send
    // every tile to the generic body)
    for (int off = lo & 1; off < kTY; off += 2) {
        const int rows = (hi - lo + off + kTY - 1) / kTY;
        int border = 0;
        for (int t = 0; t < rows; ++t) {
            const int py0 = lo - off + t * kTY;
            const int ylast = std::min(py0 + kTY, hi) - 1;   // the outputs the merge keeps
            if (py0 - 4 - S < top || ylast + 3 + S > bot || std::max(py0, lo) - 4 - S < top) ++border;
        }
        if (border < best_border || (border == best_border && rows < best_rows)) {
            best_off = off;
            best_border = border;
            best_rows = rows;
        }
    }
    a.tile_off = best_off;
    a.tiles_y = best_rows;
}

BoxArgs box_args(const Roi &r, const uint8_t *cur, const uint8_t *mask, int64_t cur_pitch, const void *ref,
                 int64_t ref_pitch, const qs_me_params *p, const CandTables *t) {
    BoxArgs a{};
    a.int_body = u8_int_body();
    a.split_tiles = split_tiles_enabled();
    a.cur = Plane{cur, cur_pitch};
    a.mask = Plane{mask, cur_pitch};
    a.ref = Plane{static_cast<const uint8_t *>(ref), ref_pitch};
    a.ref_f32 = p->ref_type == QS_REF_F32;
    a.W = r.W;
    a.H = r.H;
    a.buf_y0 = r.b0;
    a.buf_rows = r.br;
    a.S = p->S;
    a.min_support = p->min_support;
    a.n_chunks = t->n_chunks;
    a.chunked = t->chunked;
    a.chunk_off = t->chunk_off;
    return a;
}

int check_offsets(const int8_t *offs, int n, int S) {
    if (!offs || n < 1 || n > 15) return fail(QS_EINVAL, "offsets: need 1..15 entries");
    bool has0 = false;
    for (int i = 0; i < n; ++i) {
        if (offs[i] == 0) has0 = true;
        if (offs[i] < -S || offs[i] > S) return fail(QS_EINVAL, "offset %d outside [-S,S] (S=%d)", offs[i], S);
    }
    if (!has0) return fail(QS_EINVAL, "offsets must contain 0");
    return QS_OK;
}

// Certificate + exact recompute of the float argmin (certify.cu) over the keys of a box launch.
int run_certify(const BoxArgs &a, int K, bool ssd, bool reverse, const CandTables *t, char *ws, const WsLayout &L,
                cudaStream_t s) {
    CertifyArgs c{};
    c.cur = a.cur;
    c.mask = a.mask;
    c.ref = a.ref;
    c.ssd = ssd;
    c.K = K;
    c.S = a.S;
    c.W = a.W;
    c.H = a.H;
    c.buf_y0 = a.buf_y0;
    c.buf_rows = a.buf_rows;
    c.min_support = a.min_support;
    c.oy0 = a.oy0;
    c.oy1 = a.oy1;
    c.ox0 = a.ox0;
    c.ox1 = a.ox1;
    c.key_pitch = a.key_pitch;
    c.reverse = reverse;
    c.n_ref = a.n_ref > 0 ? a.n_ref : 1;
    for (int i = 0; i < c.n_ref; ++i) {
        c.ref_p[i] = a.n_ref > 0 ? a.ref_p[i] : a.ref.p;
        c.keys_p[i] = a.n_ref > 0 ? a.keys_p[i] : a.keys;
        c.s2_p[i] = a.n_ref > 0 ? a.s2_p[i] : a.s2;
    }
    c.canon = t->canon;
    c.n_cand = t->n;
    c.list = reinterpret_cast<unsigned *>(ws + L.list);
    c.list_count = reinterpret_cast<unsigned *>(ws + L.count);
    c.list_cap = L.cap;
    cudaError_t e;
    {
        ProfScope ps(P_CERTIFY, s);
        e = launch_certify(c, s);
    }
    return e == cudaSuccess ? QS_OK : cuda_fail(e, "certify launch");
}

int run_frmc(const Roi &r, const uint8_t *cur, const uint8_t *mask, int64_t cur_pitch, const void *ref,
             int64_t ref_pitch, const qs_me_params *p, const int8_t *offs, int n_offs, int full, qs_field *io,
             unsigned long long *evals, cudaStream_t s) {
    RevGridArgs a{};
    a.cur = Plane{cur, cur_pitch};
    a.mask = Plane{mask, cur_pitch};
    a.ref = Plane{static_cast<const uint8_t *>(ref), ref_pitch};
    a.ref_f32 = p->ref_type == QS_REF_F32;
    a.ssd = p->err == QS_SSD;
    a.K = p->K_h;
    a.W = r.W;
    a.H = r.H;
    a.buf_y0 = r.b0;
    a.buf_rows = r.br;
    a.min_support = p->min_support;
    a.y0 = r.y0;
    a.y1 = r.y1;
    a.f = view(io);
    a.n_dy = full ? 0 : n_offs;
    a.n_dx = a.n_dy;
    a.dys_host = offs;
    a.full_lo = -p->S;
    a.full_hi = p->S;
    a.evals = evals;
    cudaError_t e;
    {
        ProfScope ps(P_REVGRID, s);
        e = launch_revgrid(a, s);
    }
    return e == cudaSuccess ? QS_OK : cuda_fail(e, "revgrid launch");
}

}  // namespace

extern "C" {

const char *qs_last_error(void) { return g_err.c_str(); }

const char *qs_version(void) {
    return "libqs 0.4 sm_100a (me_box quarter-sampling bodies: fp32 with certified argmin, 16-bit-lane integer "
           "for uint8 SAD; certify worklist; fused finalize-NNC-FRMC-PR epilogue; multi-reference launches)";
}

int qs_workspace_size(const qs_roi *roi, int32_t frame_w, int32_t frame_h, const qs_me_params *p, size_t *bytes) {
    Roi r;
    int rc = check_roi(roi, &r);
    if (rc) return rc;
    if (frame_w != r.W || frame_h != r.H) return fail(QS_EDIM, "frame size disagrees with roi");
    if ((rc = check_params(p))) return rc;
    if (!bytes) return fail(QS_EINVAL, "bytes is NULL");
    *bytes = ws_slot_bytes(r, p->S);
    return QS_OK;
}

int qs_me_search(const uint8_t *cur, const uint8_t *cur_mask, int64_t cur_pitch, const void *ref, int64_t ref_pitch,
                 const qs_roi *roi, const qs_me_params *p, const qs_checks *fuse, qs_field *out,
                 unsigned long long *eval_count, void *workspace, size_t workspace_bytes, void *stream) {
    Roi r;
    int rc;
    if ((rc = check_roi(roi, &r)) || (rc = check_params(p))) return rc;
    const int esz = p->ref_type == QS_REF_F32 ? 4 : 1;
    if ((rc = check_plane(cur, cur_pitch, r.W, "cur")) || (rc = check_plane(cur_mask, cur_pitch, r.W, "cur_mask")) ||
        (rc = check_plane(ref, ref_pitch, (int64_t)r.W * esz, "ref")) || (rc = check_field(out, r.W, true)))
        return rc;
    const bool nnc = fuse && fuse->nnc, frmc = fuse && fuse->frmc;
    if (fuse && nnc && fuse->nnc_threshold < 0) return fail(QS_EINVAL, "nnc_threshold < 0");
    if (fuse && (fuse->nnc < 0 || fuse->nnc > QS_NNC_PAIRS)) return fail(QS_EINVAL, "nnc mode %d", fuse->nnc);
    if (frmc && (rc = check_offsets(fuse->offsets, fuse->n_offsets, p->S))) return rc;
    const int lo = nnc ? std::max(0, r.y0 - 2) : r.y0, hi = nnc ? std::min(r.H, r.y1 + 2) : r.y1;
    const int K = p->K_h, KL = K / 2, KR = K - 1 - KL;
    if ((rc = need_rows(r, lo, hi, "field")) || (rc = need_rows(r, lo - KL - p->S, hi + KR + p->S, "ME inputs")))
        return rc;
    const bool f32 = p->ref_type == QS_REF_F32;
    const size_t kb = me_keys_bytes(r);
    const bool scratch = K != 8 && nnc;   // finalize + NNC through a scratch field (ws_layout)
    const WsLayout L = ws_layout(kb, 1, f32, scratch);
    const size_t need = L.total;
    if (!workspace || !aligned16(workspace) || workspace_bytes < need)
        return fail(QS_EDIM, "workspace: need %zu bytes (16-byte aligned), got %zu", need, workspace_bytes);
    const char *terr = nullptr;
    const CandTables *t = cand_tables(p->S, &terr);
    if (!t) return fail(QS_ECUDA, "%s", terr);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (r.y1 <= r.y0 || hi <= lo) return QS_OK;   // empty roi: nothing is written

    auto *keys = static_cast<unsigned long long *>(workspace);
    char *wsc = static_cast<char *>(workspace);
    unsigned *s2 = f32 ? reinterpret_cast<unsigned *>(wsc + L.s2) : nullptr;
    cudaError_t e = cudaMemsetAsync(keys, 0xff, sizeof(unsigned long long) * (size_t)(hi - lo) * r.W, s);
    if (e == cudaSuccess && f32) e = cudaMemsetAsync(s2, 0xff, sizeof(unsigned) * (size_t)(hi - lo) * r.W, s);
    if (e != cudaSuccess) return cuda_fail(e, "memset keys");
    BoxArgs a = box_args(r, cur, cur_mask, cur_pitch, ref, ref_pitch, p, t);
    a.oy0 = lo;
    a.oy1 = hi;
    a.ox0 = 0;
    a.ox1 = r.W;
    a.tiles_x = (r.W + kTX - 1) / kTX;
    a.tiles_y = (hi - lo + kTY - 1) / kTY;
    if (K == 8) place_tile_rows(a, r, lo, hi);
    a.keys = keys;
    a.key_pitch = r.W;
    a.s2 = s2;
    a.ref_p[0] = a.ref.p;
    if (K == 8) set_tma(a, 1);
    {
        ProfScope ps(P_ME_BOX, s);
        e = launch_box(a, K, p->err == QS_SSD, false, s);
    }
    if (e != cudaSuccess) return cuda_fail(e, "me_box launch");
    if (f32 && (rc = run_certify(a, K, p->err == QS_SSD, false, t, wsc, L, s))) return rc;

    if (K == 8) {
        // Fused epilogue: finalize + NNC + FRMC (the paper's offsets, in any order) in one launch.
        const bool paper = frmc && is_paper_offsets(fuse->offsets, fuse->n_offsets);
        EpiArgs g{};
        g.cur = a.cur;
        g.mask = a.mask;
        g.ref = a.ref;
        g.ref_f32 = a.ref_f32;
        g.ssd = p->err == QS_SSD;
        g.W = r.W;
        g.H = r.H;
        g.buf_y0 = r.b0;
        g.buf_rows = r.br;
        g.S = p->S;
        g.min_support = p->min_support;
        g.lo = lo;
        g.hi = hi;
        g.y0 = r.y0;
        g.y1 = r.y1;
        g.keys = keys;
        g.key_pitch = r.W;
        g.canon = t->canon;
        g.f = view(out);
        g.write_field = 1;
        g.nnc = nnc ? fuse->nnc : 0;
        g.nnc_threshold = nnc ? fuse->nnc_threshold : 0;
        g.frmc = paper;
        const int8_t order[7] = {0, -1, 1, -3, 3, -7, 7};   // the paper's set; small offsets first
        for (int i = 0; paper && i < 7; ++i) g.dys[i] = order[i];
        g.evals = eval_count;
        {
            ProfScope ps(P_EPILOGUE, s);
            e = launch_epilogue(g, s);
        }
        if (e != cudaSuccess) return cuda_fail(e, "epilogue launch");
        if (frmc && !paper)
            return run_frmc(r, cur, cur_mask, cur_pitch, ref, ref_pitch, p, fuse->offsets, fuse->n_offsets, 0, out,
                            eval_count, s);
        return QS_OK;
    }

    FinalizeArgs fa{};
    fa.cur = a.cur;
    fa.mask = a.mask;
    fa.ref = a.ref;
    fa.ref_f32 = a.ref_f32;
    fa.ssd = p->err == QS_SSD;
    fa.K = K;
    fa.W = r.W;
    fa.H = r.H;
    fa.buf_y0 = r.b0;
    fa.buf_rows = r.br;
    fa.S = p->S;
    fa.min_support = p->min_support;
    fa.y0 = lo;
    fa.y1 = hi;
    fa.keys = keys;
    fa.key_pitch = r.W;
    fa.canon = t->canon;
    // Without NNC the ME rows are the roi's: finalize straight into the caller's field.  With NNC the
    // rows [lo, hi) go to a scratch field (the halo rows belong to the neighbouring bands' calls), NNC
    // decides [y0, y1) there and those rows are copied out.
    char *sc = wsc + L.scratch;
    const int64_t sn = (int64_t)(hi - lo) * r.W;
    qs_field tmp{reinterpret_cast<int8_t *>(sc), reinterpret_cast<int8_t *>(sc + sn), sc + 4 * sn,
                 reinterpret_cast<uint8_t *>(sc + 2 * sn), reinterpret_cast<uint8_t *>(sc + 3 * sn), r.W};
    const qs_field *dst = scratch ? &tmp : out;
    fa.alpha = dst->alpha;
    fa.beta = dst->beta;
    fa.err = dst->err;
    fa.count = dst->count;
    fa.status = dst->status;
    fa.fpitch = dst->pitch;
    fa.field_y0 = scratch ? lo : r.b0;
    {
        ProfScope ps(P_FINALIZE, s);
        e = launch_finalize(fa, s);
    }
    if (e != cudaSuccess) return cuda_fail(e, "finalize launch");

    if (nnc) {
        {
            ProfScope ps(P_NNC, s);
            e = launch_nnc(view(&tmp), r.W, r.H, lo, hi - lo, r.y0, r.y1, fuse->nnc_threshold, fuse->nnc, s);
        }
        if (e != cudaSuccess) return cuda_fail(e, "nnc launch");
        const int nr = r.y1 - r.y0;
        const size_t so = (size_t)(r.y0 - lo) * r.W, dof = (size_t)(r.y0 - r.b0) * out->pitch;
        const size_t ow = (size_t)out->pitch;
        e = cudaMemcpy2DAsync(out->alpha + dof, ow, tmp.alpha + so, r.W, r.W, nr, cudaMemcpyDeviceToDevice, s);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(out->beta + dof, ow, tmp.beta + so, r.W, r.W, nr, cudaMemcpyDeviceToDevice, s);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(out->count + dof, ow, tmp.count + so, r.W, r.W, nr, cudaMemcpyDeviceToDevice, s);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(out->status + dof, ow, tmp.status + so, r.W, r.W, nr, cudaMemcpyDeviceToDevice, s);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(static_cast<char *>(out->err) + 4 * dof, 4 * ow, static_cast<char *>(tmp.err) + 4 * so,
                                  4 * (size_t)r.W, 4 * (size_t)r.W, nr, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) return cuda_fail(e, "copy of the roi rows");
    }
    if (frmc) {
        if ((rc = run_frmc(r, cur, cur_mask, cur_pitch, ref, ref_pitch, p, fuse->offsets, fuse->n_offsets, 0, out,
                           eval_count, s)))
            return rc;
    }
    return QS_OK;
}

int qs_me_search_refs(const uint8_t *cur, const uint8_t *cur_mask, int64_t cur_pitch, int32_t n_refs,
                      const void *const *refs, int64_t ref_pitch, const qs_roi *roi, const qs_me_params *p,
                      const qs_checks *fuse, qs_field *outs, const qs_projection *proj,
                      unsigned long long *eval_count, void *workspace, size_t workspace_bytes, void *stream) {
    Roi r;
    int rc;
    if (n_refs < 0) return fail(QS_EINVAL, "n_refs=%d", n_refs);
    if (n_refs > 0 && !refs) return fail(QS_EINVAL, "refs is NULL");
    if (n_refs > 0 && !outs && !proj) return fail(QS_EINVAL, "outs is NULL (allowed only with a projection)");
    if ((rc = check_roi(roi, &r)) || (rc = check_params(p))) return rc;
    if (proj && n_refs > 0) {
        if (!proj->past_val || !proj->past_mask || !proj->sum || !proj->cnt)
            return fail(QS_EINVAL, "projection: past_val / past_mask / sum / cnt is NULL");
        if (proj->acc_pitch < r.W) return fail(QS_EDIM, "projection: acc_pitch < width");
        if ((reinterpret_cast<uintptr_t>(proj->sum) & 3) || (reinterpret_cast<uintptr_t>(proj->cnt) & 3) ||
            (proj->acc_pitch & 3))
            return fail(QS_EALIGN, "projection: sum / cnt must be 4-byte aligned and acc_pitch a multiple of 4");
        for (int i = 0; i < n_refs; ++i)
            if ((rc = check_plane(proj->past_val[i], proj->past_pitch, r.W, "past_val")) ||
                (rc = check_plane(proj->past_mask[i], proj->past_pitch, r.W, "past_mask")))
                return rc;
    }
    size_t slot = 0;
    if ((rc = qs_workspace_size(roi, r.W, r.H, p, &slot))) return rc;
    if (n_refs == 0) return QS_OK;
    if (!workspace || !aligned16(workspace) || workspace_bytes < slot * (size_t)n_refs)
        return fail(QS_EDIM, "workspace: need %zu bytes (%d slots of %zu, 16-byte aligned), got %zu",
                    slot * (size_t)n_refs, n_refs, slot, workspace_bytes);
    char *ws = static_cast<char *>(workspace);
    const bool nnc = fuse && fuse->nnc, frmc = fuse && fuse->frmc;
    if (frmc && (rc = check_offsets(fuse->offsets, fuse->n_offsets, p->S))) return rc;   // before reading them
    const bool paper = frmc && is_paper_offsets(fuse->offsets, fuse->n_offsets);
    // The single-launch path covers the fused K = 8 epilogue; everything else runs slot by slot.
    if (p->K_h != 8 || (frmc && !paper)) {
        if (!outs) return fail(QS_EINVAL, "outs is NULL: projection-only needs K = 8 and the paper's FRMC offsets");
        for (int i = 0; i < n_refs; ++i) {
            if ((rc = qs_me_search(cur, cur_mask, cur_pitch, refs[i], ref_pitch, roi, p, fuse, &outs[i], eval_count,
                                   ws + slot * i, slot, stream)))
                return rc;
            if (proj && (rc = qs_project(&outs[i], proj->past_val[i], proj->past_mask[i], proj->past_pitch, roi,
                                         proj->sum, proj->cnt, proj->acc_pitch, stream)))
                return rc;
        }
        return QS_OK;
    }
    for (int i0 = 0; i0 < n_refs; i0 += kMaxRefs) {   // groups of kMaxRefs slots per launch
        const int n = std::min(n_refs - i0, kMaxRefs);
        const int esz = p->ref_type == QS_REF_F32 ? 4 : 1;
        if ((rc = check_plane(cur, cur_pitch, r.W, "cur")) || (rc = check_plane(cur_mask, cur_pitch, r.W, "cur_mask")))
            return rc;
        for (int i = 0; i < n; ++i)
            if ((rc = check_plane(refs[i0 + i], ref_pitch, (int64_t)r.W * esz, "ref")) ||
                (outs && (rc = check_field(&outs[i0 + i], r.W, true))))
                return rc;
        if (nnc && fuse->nnc_threshold < 0) return fail(QS_EINVAL, "nnc_threshold < 0");
        if (fuse && (fuse->nnc < 0 || fuse->nnc > QS_NNC_PAIRS)) return fail(QS_EINVAL, "nnc mode %d", fuse->nnc);
        if (frmc && (rc = check_offsets(fuse->offsets, fuse->n_offsets, p->S))) return rc;
        const int lo = nnc ? std::max(0, r.y0 - 2) : r.y0, hi = nnc ? std::min(r.H, r.y1 + 2) : r.y1;
        const int KL = 4, KR = 3;
        if ((rc = need_rows(r, lo, hi, "field")) || (rc = need_rows(r, lo - KL - p->S, hi + KR + p->S, "ME inputs")))
            return rc;
        const char *terr = nullptr;
        const CandTables *t = cand_tables(p->S, &terr);
        if (!t) return fail(QS_ECUDA, "%s", terr);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        if (r.y1 <= r.y0 || hi <= lo) return QS_OK;
        const size_t kb = me_keys_bytes(r);
        const bool f32 = p->ref_type == QS_REF_F32;
        const WsLayout L = ws_layout(kb, n, f32, false);   // <= n * slot bytes
        const size_t kba = L.kba, s2a = L.s2a;
        char *wg = ws + slot * i0;
        // The group's n slots: key planes at wg + i * kba, then (float) second planes at
        // wg + L.s2 + i * s2a; one memset per span.
        cudaError_t e = cudaMemsetAsync(wg, 0xff, kba * (n - 1) + kb, s);
        if (e == cudaSuccess && f32) e = cudaMemsetAsync(wg + L.s2, 0xff, s2a * (n - 1) + kb / 2, s);
        if (e != cudaSuccess) return cuda_fail(e, "memset keys");
        BoxArgs a = box_args(r, cur, cur_mask, cur_pitch, refs[i0], ref_pitch, p, t);
        a.oy0 = lo;
        a.oy1 = hi;
        a.ox0 = 0;
        a.ox1 = r.W;
        a.tiles_x = (r.W + kTX - 1) / kTX;
        a.tiles_y = (hi - lo + kTY - 1) / kTY;
        place_tile_rows(a, r, lo, hi);
        a.keys = reinterpret_cast<unsigned long long *>(wg);
        a.key_pitch = r.W;
        a.n_ref = n;
        for (int i = 0; i < n; ++i) {
            a.ref_p[i] = static_cast<const uint8_t *>(refs[i0 + i]);
            a.keys_p[i] = reinterpret_cast<unsigned long long *>(wg + kba * i);
            a.s2_p[i] = f32 ? reinterpret_cast<unsigned *>(wg + L.s2 + s2a * i) : nullptr;
        }
        a.s2 = a.s2_p[0];
        set_tma(a, n);
        {
            ProfScope ps(P_ME_BOX, s);
            e = launch_box(a, 8, p->err == QS_SSD, false, s);
        }
        if (e != cudaSuccess) return cuda_fail(e, "me_box launch");
        if (f32 && (rc = run_certify(a, 8, p->err == QS_SSD, false, t, wg, L, s))) return rc;
        EpiArgs g{};
        g.cur = a.cur;
        g.mask = a.mask;
        g.ref = a.ref;
        g.ref_f32 = a.ref_f32;
        g.ssd = p->err == QS_SSD;
        g.W = r.W;
        g.H = r.H;
        g.buf_y0 = r.b0;
        g.buf_rows = r.br;
        g.S = p->S;
        g.min_support = p->min_support;
        g.lo = lo;
        g.hi = hi;
        g.y0 = r.y0;
        g.y1 = r.y1;
        g.keys = a.keys;
        g.key_pitch = r.W;
        g.canon = t->canon;
        g.f = outs ? view(&outs[i0]) : FieldView{};
        g.write_field = outs != nullptr;
        g.nnc = nnc ? fuse->nnc : 0;
        g.nnc_threshold = nnc ? fuse->nnc_threshold : 0;
        g.frmc = paper;
        const int8_t order[7] = {0, -1, 1, -3, 3, -7, 7};
        for (int i = 0; paper && i < 7; ++i) g.dys[i] = order[i];
        g.evals = eval_count;
        g.n_ref = n;
        for (int i = 0; i < n; ++i) {
            g.ref_p[i] = a.ref_p[i];
            g.keys_p[i] = a.keys_p[i];
            g.f_p[i] = outs ? view(&outs[i0 + i]) : FieldView{};
        }
        if (proj) {
            g.proj = 1;
            for (int i = 0; i < n; ++i) {
                g.pv_p[i] = proj->past_val[i0 + i];
                g.pm_p[i] = proj->past_mask[i0 + i];
            }
            g.past_pitch = proj->past_pitch;
            g.sum = proj->sum;
            g.cnt = proj->cnt;
            g.acc_pitch = proj->acc_pitch;
        }
        {
            ProfScope ps(P_EPILOGUE, s);
            e = launch_epilogue(g, s);
        }
        if (e != cudaSuccess) return cuda_fail(e, "epilogue launch");
    }
    return QS_OK;
}

int qs_reverse_check(int32_t mode, const uint8_t *cur, const uint8_t *cur_mask, int64_t cur_pitch, const void *ref,
                     int64_t ref_pitch, const qs_roi *roi, const qs_me_params *p, qs_field *io,
                     unsigned long long *eval_count, void *workspace, size_t workspace_bytes, void *stream) {
    Roi r;
    int rc;
    if (mode != QS_RME && mode != QS_RMC) return fail(QS_EINVAL, "mode=%d", mode);
    if ((rc = check_roi(roi, &r)) || (rc = check_params(p))) return rc;
    const int esz = p->ref_type == QS_REF_F32 ? 4 : 1;
    if ((rc = check_plane(cur, cur_pitch, r.W, "cur")) || (rc = check_plane(cur_mask, cur_pitch, r.W, "cur_mask")) ||
        (rc = check_plane(ref, ref_pitch, (int64_t)r.W * esz, "ref")) || (rc = check_field(io, r.W, true)))
        return rc;
    const int K = p->K_h, KL = K / 2, KR = K - 1 - KL, S = p->S;
    if ((rc = need_rows(r, r.y0, r.y1, "field"))) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const char *terr = nullptr;
    const CandTables *t = cand_tables(S, &terr);
    if (!t) return fail(QS_ECUDA, "%s", terr);
    if (mode == QS_RMC) {
        if ((rc = need_rows(r, r.y0 - S - KL, r.y1 + S + KR, "RMC inputs"))) return rc;
        if (r.y1 <= r.y0) return QS_OK;
        return run_frmc(r, cur, cur_mask, cur_pitch, ref, ref_pitch, p, nullptr, 0, 1, io, eval_count, s);
    }
    if ((rc = need_rows(r, r.y0 - 2 * S - KL, r.y1 + 2 * S + KR, "RME inputs"))) return rc;
    const bool f32 = p->ref_type == QS_REF_F32;
    const size_t kb = rme_keys_bytes(r, S);
    const WsLayout L = ws_layout(kb, 1, f32, false);
    const size_t need = L.total;
    if (!workspace || !aligned16(workspace) || workspace_bytes < need)
        return fail(QS_EDIM, "workspace: need %zu bytes (16-byte aligned), got %zu", need, workspace_bytes);
    if (r.y1 <= r.y0) return QS_OK;
    auto *keys = static_cast<unsigned long long *>(workspace);
    char *wsc = static_cast<char *>(workspace);
    unsigned *s2 = f32 ? reinterpret_cast<unsigned *>(wsc + L.s2) : nullptr;
    cudaError_t e = cudaMemsetAsync(keys, 0xff, kb, s);
    if (e == cudaSuccess && f32) e = cudaMemsetAsync(s2, 0xff, kb / 2, s);
    if (e != cudaSuccess) return cuda_fail(e, "memset keys");
    BoxArgs a = box_args(r, cur, cur_mask, cur_pitch, ref, ref_pitch, p, t);
    a.oy0 = r.y0 - S;
    a.oy1 = r.y1 + S;
    a.ox0 = -S;
    a.ox1 = r.W + S;
    a.tiles_x = (r.W + 2 * S + kTX - 1) / kTX;
    a.tiles_y = (r.y1 - r.y0 + 2 * S + kTY - 1) / kTY;
    a.keys = keys;
    a.key_pitch = r.W + 2 * S;
    a.s2 = s2;
    {
        ProfScope ps(P_ME_BOX, s);
        e = launch_box(a, K, p->err == QS_SSD, true, s);
    }
    if (e != cudaSuccess) return cuda_fail(e, "rme box launch");
    if (f32 && (rc = run_certify(a, K, p->err == QS_SSD, true, t, wsc, L, s))) return rc;
    RmeDecideArgs d{};
    d.W = r.W;
    d.H = r.H;
    d.buf_y0 = r.b0;
    d.buf_rows = r.br;
    d.S = S;
    d.y0 = r.y0;
    d.y1 = r.y1;
    d.f = view(io);
    d.keys = keys;
    d.key_pitch = r.W + 2 * S;
    d.canon = t->canon;
    d.evals = eval_count;
    d.n_cand = t->n;
    {
        ProfScope ps(P_RME_DECIDE, s);
        e = launch_rme_decide(d, s);
    }
    if (e != cudaSuccess) return cuda_fail(e, "rme decide launch");
    return QS_OK;
}

int qs_frmc(const uint8_t *cur, const uint8_t *cur_mask, int64_t cur_pitch, const void *ref, int64_t ref_pitch,
            const qs_roi *roi, const qs_me_params *p, const int8_t *offsets, int32_t n_offsets, qs_field *io,
            unsigned long long *eval_count, void *stream) {
    Roi r;
    int rc;
    if ((rc = check_roi(roi, &r)) || (rc = check_params(p))) return rc;
    const int esz = p->ref_type == QS_REF_F32 ? 4 : 1;
    if ((rc = check_plane(cur, cur_pitch, r.W, "cur")) || (rc = check_plane(cur_mask, cur_pitch, r.W, "cur_mask")) ||
        (rc = check_plane(ref, ref_pitch, (int64_t)r.W * esz, "ref")) || (rc = check_field(io, r.W, true)))
        return rc;
    if ((rc = check_offsets(offsets, n_offsets, p->S))) return rc;
    const int K = p->K_h, KL = K / 2, KR = K - 1 - KL;
    if ((rc = need_rows(r, r.y0, r.y1, "field")) || (rc = need_rows(r, r.y0 - p->S - KL, r.y1 + p->S + KR, "FRMC inputs")))
        return rc;
    if (r.y1 <= r.y0) return QS_OK;
    return run_frmc(r, cur, cur_mask, cur_pitch, ref, ref_pitch, p, offsets, n_offsets, 0, io, eval_count,
                    static_cast<cudaStream_t>(stream));
}

int qs_nnc(qs_field *io, const qs_roi *roi, int32_t threshold, void *stream) {
    return qs_nnc_mode(io, roi, threshold, QS_NNC_CENTRE, stream);
}

int qs_nnc_mode(qs_field *io, const qs_roi *roi, int32_t threshold, int32_t mode, void *stream) {
    if (mode != QS_NNC_CENTRE && mode != QS_NNC_PAIRS) return fail(QS_EINVAL, "nnc mode %d", mode);
    Roi r;
    int rc;
    if ((rc = check_roi(roi, &r))) return rc;
    if ((rc = check_field(io, r.W, false))) return rc;
    if (threshold < 0) return fail(QS_EINVAL, "threshold < 0");
    if ((rc = need_rows(r, r.y0 - 2, r.y1 + 2, "NNC field"))) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    {
        ProfScope ps(P_NNC, s);
        e = launch_nnc(view(io), r.W, r.H, r.b0, r.br, r.y0, r.y1, threshold, mode, s);
    }
    return e == cudaSuccess ? QS_OK : cuda_fail(e, "nnc launch");
}

int qs_project(const qs_field *f, const uint8_t *past_val, const uint8_t *past_mask, int64_t past_pitch,
               const qs_roi *roi, uint32_t *sum, uint8_t *cnt, int64_t acc_pitch, void *stream) {
    Roi r;
    int rc;
    if ((rc = check_roi(roi, &r))) return rc;
    if ((rc = check_field(f, r.W, false))) return rc;
    if ((rc = check_plane(past_val, past_pitch, r.W, "past_val")) ||
        (rc = check_plane(past_mask, past_pitch, r.W, "past_mask")))
        return rc;
    if (!sum || !cnt) return fail(QS_EINVAL, "sum/cnt is NULL");
    if (acc_pitch < r.W) return fail(QS_EDIM, "acc_pitch < width");
    if ((reinterpret_cast<uintptr_t>(sum) & 3)) return fail(QS_EALIGN, "sum not 4-byte aligned");
    if ((rc = need_rows(r, r.y0, r.y1, "field"))) return rc;
    ProjectArgs a{};
    a.f = FieldView{f->alpha, f->beta, f->err, f->count, f->status, f->pitch};
    a.past_val = Plane{past_val, past_pitch};
    a.past_mask = Plane{past_mask, past_pitch};
    a.W = r.W;
    a.H = r.H;
    a.buf_y0 = r.b0;
    a.buf_rows = r.br;
    a.y0 = r.y0;
    a.y1 = r.y1;
    a.sum = sum;
    a.cnt = cnt;
    a.acc_pitch = acc_pitch;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaError_t e;
    {
        ProfScope ps(P_PROJECT, s);
        e = launch_project(a, s);
    }
    return e == cudaSuccess ? QS_OK : cuda_fail(e, "project launch");
}

int qs_profile_enable(int32_t on) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.on = on != 0;
    return QS_OK;
}

int qs_profile_read(const char *kernel, double *total_ms, int64_t *launches) {
    if (!kernel || !total_ms || !launches) return fail(QS_EINVAL, "NULL argument");
    int want = -2;
    if (!strcmp(kernel, "*")) want = -1;
    for (int k = 0; k < P_COUNT; ++k)
        if (!strcmp(kernel, kProfNames[k])) want = k;
    if (want == -2) return fail(QS_EINVAL, "unknown kernel '%s'", kernel);
    std::lock_guard<std::mutex> lk(g_prof.mu);
    double t = 0.0;
    int64_t n = 0;
    for (const ProfRec &r : g_prof.recs) {
        if (want >= 0 && r.kernel != want) continue;
        if (cudaEventSynchronize(r.stop) != cudaSuccess) return cuda_fail(cudaGetLastError(), "event sync");
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, r.start, r.stop) != cudaSuccess)
            return cuda_fail(cudaGetLastError(), "event elapsed");
        t += ms;
        ++n;
    }
    *total_ms = t;
    *launches = n;
    return QS_OK;
}

int qs_certify_stats(int64_t *rechecked, int32_t reset) {
    if (!rechecked) return fail(QS_EINVAL, "rechecked is NULL");
    unsigned long long *c = rechecked_counter();
    if (!c) return fail(QS_ECUDA, "certify counter unavailable");
    unsigned long long v = 0;
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(&v, c, sizeof v, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && reset) e = cudaMemset(c, 0, sizeof v);
    if (e != cudaSuccess) return cuda_fail(e, "certify counter");
    *rechecked = (int64_t)v;
    return QS_OK;
}

int qs_profile_reset(void) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    for (const ProfRec &r : g_prof.recs) {
        cudaEventSynchronize(r.stop);
        g_prof.pool.push_back(r.start);
        g_prof.pool.push_back(r.stop);
    }
    g_prof.recs.clear();
    return QS_OK;
}

}  // extern "C"
