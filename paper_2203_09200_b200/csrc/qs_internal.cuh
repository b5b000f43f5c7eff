// qs_internal.cuh -- internal declarations of libqs (the CUDA product path).
// Shares nothing with oracle/ (test infrastructure).  See include/qs.h for the
// ABI and DESIGN.md for the kernels, their rooflines and the readings R1-R26.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cuda.h>           // CUtensorMap (TMA descriptors; the driver entry point is resolved at run time)
#include <cuda_runtime.h>

// Bounds checks of the checked build (libqs_checked.so, -DQS_CHECKED): the
// staged-window reads, the shared ring and the global key / field writes trap when out of range.
// The product build compiles them out.
#ifdef QS_CHECKED
#define QS_DCHECK(cond)                                                                     \
    do {                                                                                    \
        if (!(cond)) {                                                                      \
            printf("QS_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
                   (int)blockIdx.x, (int)threadIdx.x);                                      \
            __trap();                                                                       \
        }                                                                                   \
    } while (0)
#else
#define QS_DCHECK(cond) \
    do {                \
    } while (0)
#endif

#include "../../include/qs.h"

namespace qs {

// Status codes mirror include/qs.h (PAPER.md:68-115 path; R4, R6, R16).
constexpr uint8_t kNotTarget = QS_NOT_TARGET;
constexpr uint8_t kInvalid = QS_INVALID;
constexpr uint8_t kCandidate = QS_CANDIDATE;
constexpr uint8_t kAccepted = QS_ACCEPTED;
constexpr uint8_t kRejected = QS_REJECTED;

// ME box-kernel tiling.
constexpr int kTX = 64;        // output columns per CTA tile
constexpr int kTY = 56;        // output rows per CTA tile (TY + K - 1 <= 64 for K <= 9)
constexpr int kNT = 256;       // threads per CTA
constexpr int kRun = 16;       // phase A: H columns per thread
constexpr int kSeg = 14;       // phase B: output rows per thread (4 segments x 14 = 56)
constexpr int kTXP = 68;       // padded row pitch (floats) of the H planes in smem
constexpr int kChunkRows = 7;  // alpha rows of candidates per work unit
// Chunks take alpha rows of ONE parity: group g = chunk >> 1 covers rows -S + 14 g .. +13, chunk
// parity chunk & 1 takes every other row of it (7 rows, fewer in the last group).  Within a chunk
// alpha - alo is even, so a measured pixel's reference row has the parity of its own row offset
// dy for every candidate -- the quad body's reference window is split by row parity (conflict-light
// gathers, me_box.cu).  kChunkSpan = rows spanned by a chunk's window.
constexpr int kChunkSpan = 2 * kChunkRows - 1;
constexpr int kQWinRowsHost = 64;   // quad body window: pixel rows of the tile's blocks (me_box.cuh kQWinRows)
constexpr int kQWinColsHost = 72;   // and pixel columns (me_box.cuh kQWinCols)
__host__ __device__ constexpr int chunk_alo(int S, int chunk) { return -S + 2 * kChunkRows * (chunk >> 1) + (chunk & 1); }
__host__ __device__ constexpr int chunk_ahi(int S, int chunk) {
    return chunk_alo(S, chunk) + kChunkSpan - 1 < S ? chunk_alo(S, chunk) + kChunkSpan - 1 : S;
}
__host__ __device__ constexpr int chunk_count(int S) { return 2 * ((2 * S + 1 + 2 * kChunkRows - 1) / (2 * kChunkRows)); }

// One device-resident candidate table per (device, S).
struct CandTables {
    int S = -1;
    int n = 0;                       // (2S+1)^2
    int n_chunks = 0;
    int32_t *canon = nullptr;        // [n]   rank -> (alpha & 0xff) | (beta & 0xff) << 8
    int32_t *chunked = nullptr;      // [n]   chunk-major, rank order inside a chunk:
                                     //       (alpha & 0xff) | (beta & 0xff) << 8 | rank << 16
    int32_t *chunk_off = nullptr;    // [n_chunks + 1]
};

// Returns tables for S on the current device (built once; thread-safe).
const CandTables *cand_tables(int S, const char **err);

// Geometry of a plane window: global row y lives at base + (y - buf_y0) * pitch.
struct Plane {
    const uint8_t *p;   // base of buffer row 0
    int64_t pitch;      // bytes
};

// Arguments of the box kernels (forward ME and dense reverse ME).
// References per launch: qs_me_search_refs runs the pairs (cur, ref_i) of one frame in a single
// launch per kernel; slot i's reference plane, key plane and field.
constexpr int kMaxRefs = 4;

struct BoxArgs {
    Plane cur, mask, ref;            // ref.p == ref_p[0]; ref.pitch is shared by every slot
    int ref_f32;
    int W, H, buf_y0, buf_rows;
    int S, min_support;
    int oy0, oy1, ox0, ox1;          // output domain (rows / cols, frame coords; may exceed the frame for REV)
    int tiles_x, tiles_y, n_chunks;
    int tile_off;                    // rows of the first tile above oy0 (0 .. kTY-1)
    const int32_t *chunked;
    const int32_t *chunk_off;
    unsigned long long *keys;        // [oy1-oy0][key_pitch] (slot 0)
    int64_t key_pitch;
    int n_ref;                       // slots per launch: CTA b works on slot b % n_ref (0 -> 1)
    const uint8_t *ref_p[kMaxRefs];
    unsigned long long *keys_p[kMaxRefs];
    // Float references only (certified argmin): per output the
    // smallest approximate mean of every candidate other than the merged winner, as non-negative
    // float bits ([oy1-oy0][key_pitch], 0xffffffff = none).  nullptr for uint8 references.
    unsigned *s2;
    unsigned *s2_p[kMaxRefs];
    int int_body;                    // uint8 SAD interior tiles: 1 = integer packed body, 0 = fp32 body
    // TMA staging of the quad body's float reference window: one 3-D tiled
    // descriptor per slot over the buffer as [rows / 2][parity][W] floats, boxes of
    // [tma_rows][1][tma_cols] (one per row-parity plane), out-of-frame / out-of-buffer elements
    // filled with NaN ("no term").  tma = 0: cp.async / register staging.
    int tma, tma_cols, tma_rows;
    // K = 8 forward, float references: 1 = border tiles and interior tiles as two kernels (own code
    // generation each), the interior one a programmatic dependent launch (me_box.cuh launch_t).
    int split_tiles;
    int rect_r0, rect_r1, rect_c0, rect_c1;   // split launches: interior tiles [r0, r1) x [c0, c1) (launch_t)
    CUtensorMap tmap[kMaxRefs];
};

// Certified float argmin.  The float consumers track, per output,
// the two smallest KEYED approximate means: the low kKeyBits of the fp32 bits replaced by the
// candidate's chunk-list position (< 512), so one FMNMX orders (truncated mean, position) and the
// winner's rank decodes from the key.  Truncation moves a value by < 2^-14 relative; with the fp32
// sum errors of both sides (<= 2^-17 relative) the winner w is the oracle's whenever every other
// candidate's truncated value exceeds w's by the factor (1 + kCertEps).
constexpr unsigned kKeyBits = 511u;
constexpr float kCertEps = 1.0f / 8192.0f;   // 2^-13
constexpr float kInadmissible = 3.0e38f;     // finite: keyed bits stay finite (never NaN)
constexpr float kAdmissibleMax = 1.0e38f;

// Forward / reverse certification and exact recompute of uncertain outputs (certify.cu).
struct CertifyArgs {
    Plane cur, mask, ref;
    int ssd, K, S;
    int W, H, buf_y0, buf_rows, min_support;
    int oy0, oy1, ox0, ox1;          // key domain (frame coordinates)
    int64_t key_pitch;
    int reverse;                     // 0: forward ME keys (targets only), 1: dense reverse keys (RME)
    int n_ref;
    const uint8_t *ref_p[kMaxRefs];
    unsigned long long *keys_p[kMaxRefs];
    const unsigned *s2_p[kMaxRefs];
    const int32_t *canon;
    int n_cand;
    unsigned *list;                  // workspace: uncertain outputs (slot << 30 | y - oy0 << 16 | x - ox0)
    unsigned *list_count;            // workspace: entries appended (zeroed by launch_certify)
    int list_cap;
};
cudaError_t launch_certify(const CertifyArgs &a, cudaStream_t s);
unsigned long long *rechecked_counter();   // current device's counter (nullptr on failure)

// Launchers (me_box.cu).  Return cudaError_t of the launch.
cudaError_t launch_box(const BoxArgs &a, int K, bool ssd, bool reverse, cudaStream_t s);

struct FinalizeArgs {
    Plane cur, mask, ref;
    int ref_f32, ssd, K;
    int W, H, buf_y0, buf_rows;
    int S, min_support;
    int y0, y1;                      // rows to finalize
    const unsigned long long *keys;  // keys row 0 == global row y0
    int64_t key_pitch;
    const int32_t *canon;
    int8_t *alpha, *beta;
    void *err;
    uint8_t *count, *status;
    int64_t fpitch;                  // field pitch (elements); field row 0 == global field_y0
    int field_y0;
};
cudaError_t launch_finalize(const FinalizeArgs &a, cudaStream_t s);

// Checks (checks.cu).
struct FieldView {
    int8_t *alpha, *beta;
    void *err;
    uint8_t *count, *status;
    int64_t pitch;                   // elements; row 0 == global buf_y0
};

// NNC decision of one entry from the filtered centre (ca, cb) and its four filtered 4-neighbours
// (nv: in frame and valid).  mode 1 (R15): the centre against each neighbour; mode 2 (R30, the other
// reading of PAPER.md:114's "each neighboring pair"): the neighbours against each other.
__device__ __forceinline__ bool nnc_rejects(int mode, int ca, int cb, const int (&na)[4], const int (&nb)[4],
                                            const bool (&nv)[4], int threshold) {
    bool reject = false;
    if (mode == 2) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int l = k + 1; l < 4; ++l)
                if (nv[k] && nv[l] && abs(na[k] - na[l]) + abs(nb[k] - nb[l]) > threshold) reject = true;
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (nv[k] && abs(ca - na[k]) + abs(cb - nb[k]) > threshold) reject = true;
    }
    return reject;
}
cudaError_t launch_nnc(FieldView f, int W, int H, int buf_y0, int buf_rows, int y0, int y1, int threshold, int mode,
                       cudaStream_t s);

// Fused per-pair epilogue for K = 8 (epilogue.cu): finalize + NNC + FRMC (paper offsets).
struct EpiArgs {
    Plane cur, mask, ref;
    int ref_f32, ssd;
    int W, H, buf_y0, buf_rows, S, min_support;
    int lo, hi;                      // rows holding ME keys (finalized)
    int y0, y1;                      // rows whose entries are checked
    const unsigned long long *keys;  // keys row 0 == global row lo
    int64_t key_pitch;
    const int32_t *canon;
    FieldView f;
    int nnc, nnc_threshold, frmc;
    int write_field;                 // 0: projection-only (qs_me_search_refs with outs == NULL)
    int8_t dys[8];                   // FRMC delta_y order (a permutation of the paper's offsets)
    unsigned long long *evals;
    int n_ref;                       // slots per launch (grid z); 0 -> 1 with slot 0 = (ref, keys, f)
    const uint8_t *ref_p[kMaxRefs];
    const unsigned long long *keys_p[kMaxRefs];
    FieldView f_p[kMaxRefs];
    // Fused projection PR (qs_me_search_refs with a qs_projection): ACCEPTED entries of slot z add
    // past_val(p + v) of slot z's past frame into sum / cnt (integer atomics: order-free, exact).
    int proj;
    const uint8_t *pv_p[kMaxRefs], *pm_p[kMaxRefs];
    int64_t past_pitch;
    uint32_t *sum;
    uint8_t *cnt;                    // 4-byte aligned, acc_pitch % 4 == 0 (byte adds on the word)
    int64_t acc_pitch;
};
cudaError_t launch_epilogue(const EpiArgs &g, cudaStream_t s);

struct RevGridArgs {
    Plane cur, mask, ref;
    int ref_f32, ssd, K;
    int W, H, buf_y0, buf_rows;
    int min_support;
    int y0, y1;
    FieldView f;
    int n_dy, n_dx;                  // delta grid = dys x dxs
    const int8_t *dys_host;          // copied into kernel params (<= 15 entries) or full range
    int full_lo, full_hi;            // if n_dy == 0: delta in [full_lo, full_hi]^2 (RMC)
    unsigned long long *evals;
};
cudaError_t launch_revgrid(const RevGridArgs &a, cudaStream_t s);

struct RmeDecideArgs {
    int W, H, buf_y0, buf_rows, S;
    int y0, y1;
    FieldView f;
    const unsigned long long *keys;  // reverse keys over x rows [y0-S, y1+S), cols [-S, W+S)
    int64_t key_pitch;
    const int32_t *canon;
    unsigned long long *evals;
    int n_cand;
};
cudaError_t launch_rme_decide(const RmeDecideArgs &a, cudaStream_t s);

struct ProjectArgs {
    FieldView f;
    Plane past_val, past_mask;
    int W, H, buf_y0, buf_rows, y0, y1;
    uint32_t *sum;
    uint8_t *cnt;
    int64_t acc_pitch;
};
cudaError_t launch_project(const ProjectArgs &a, cudaStream_t s);

}  // namespace qs
