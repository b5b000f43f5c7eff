// me_box.cuh -- K1/K2 "me_box": exhaustive template-matching motion estimation
// on sm_100a, and the dense reverse ME used by RME.
//
// What it computes (§2.2; readings R1-R7):
//   for every output position p of the tile and every candidate v in [-S,S]^2
//     e(p,v) = sum_{o in KxK} D_v(p+o),  D_v(q) = phi(A(q) - B(q+v)),
//   where A is the fixed side and B the shifted side, both staged as float with
//   NaN marking "no term" (unmeasured pixel or outside the frame), so that
//   D = max(phi(A - B), 0) is 0 exactly where the definition drops the term.
//     forward ME (qs_me_search):  A = cur where cur_mask = 1 (sparse), B = ref
//     reverse ME (RME, R9/R10):   A = ref (dense),  B = cur where cur_mask = 1
//   The KxK window sum is separable: H = horizontal K-sum of D, E = vertical
//   K-sum of H.  Uint8 references keep every value an integer < 2^24 in fp32,
//   so the sums are exact and bit-identical to the oracle's integer sums; for
//   float32 references the sums are fp32 in a fixed blocked order (pairwise
//   tree for K = 8) whose rounding differs from the oracle's row-major order
//   only at the last bits.
//
// Work decomposition: one CTA = one tile of 56x64
// outputs x one chunk of 7 alpha-rows of candidates.  The chunk's B window is
// staged once into shared memory; the loop over the chunk's candidates runs in
// rank order (|a|+|b|, a, b), so a strict '<' inside a thread implements the
// tie-break R7.  Per candidate: phase A (thread = one row x 16 columns) forms D
// and H into a double-buffered smem plane; phase B (thread = one column x 14
// rows) forms E and updates the running best.  Chunks of the same tile merge
// with a 64-bit atomicMin on (order key << 32 | rank), which is exact because
// the order key is monotone in the mean and equal means give equal keys.
#include <algorithm>
#include <cfloat>
#include <cmath>
#include <type_traits>

#pragma once
#include "qs_internal.cuh"

namespace qs {
namespace {

// B/A loaders: float value or NaN ("no term").
// Rows outside the frame, or outside the caller's buffer window, give NaN.
// The launch's reference slot of this CTA (qs_me_search_refs: CTA b works on slot b % n_ref).
__device__ __forceinline__ int ref_slot(const BoxArgs &a) { return (int)(blockIdx.x % (unsigned)a.n_ref); }

__device__ __forceinline__ float load_ref(const BoxArgs &a, int y, int x) {
    if (y < 0 || y >= a.H || x < 0 || x >= a.W || y < a.buf_y0 || y >= a.buf_y0 + a.buf_rows)
        return __int_as_float(0x7fc00000);
    const int64_t off = (int64_t)(y - a.buf_y0) * a.ref.pitch;
    const uint8_t *rp = a.ref_p[ref_slot(a)];
    if (a.ref_f32) return reinterpret_cast<const float *>(rp + off)[x];
    return (float)rp[off + x];
}

__device__ __forceinline__ float load_cur_masked(const BoxArgs &a, int y, int x) {
    if (y < 0 || y >= a.H || x < 0 || x >= a.W || y < a.buf_y0 || y >= a.buf_y0 + a.buf_rows)
        return __int_as_float(0x7fc00000);
    const int64_t r = (int64_t)(y - a.buf_y0);
    if (!a.mask.p[r * a.mask.pitch + x]) return __int_as_float(0x7fc00000);
    return (float)a.cur.p[r * a.cur.pitch + x];
}

// ---- certified float argmin (qs_internal.cuh) ----
// Keyed value: low kKeyBits of the fp32 bits replaced by the chunk-list position k.
__device__ __forceinline__ float fkey(float v, unsigned k) {
    return __uint_as_float((__float_as_uint(v) & ~kKeyBits) | k);
}
// Running two smallest keys (m1 <= m2): m2 = median(m1, m2, key), m1 = min(m1, key).
__device__ __forceinline__ void fbest(float &m1, float &m2, float key) {
    m2 = fminf(m2, fmaxf(m1, key));
    m1 = fminf(m1, key);
}
// The same on the keys' bits as unsigned integers (RUNS phase 2): a negative value (an inadmissible
// candidate, coded e * (-1)) has the sign bit set and orders after every non-negative key.
__device__ __forceinline__ void ubest(float &m1, float &m2, unsigned key) {
    unsigned x = __float_as_uint(m1), y = __float_as_uint(m2);
    y = min(y, max(x, key));
    x = min(x, key);
    m1 = __uint_as_float(x);
    m2 = __uint_as_float(y);
}
__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
// Merge one output's (winner value v1 with its rank, second-smallest value v2) into the global key
// and the second plane: the 64-bit atomicMin orders (v1, rank) across chunks; whoever does not end
// up the winner -- this contribution when it loses, the displaced key when it wins -- pushes its
// value into s2, so s2 ends as the smallest value of every candidate but the final winner.
__device__ __forceinline__ void check_key(const BoxArgs &a, int py, int px) {
    QS_DCHECK(py >= a.oy0 && py < a.oy1 && px >= a.ox0 && px - a.ox0 < a.key_pitch);
}
__device__ __forceinline__ void merge_f32(unsigned long long *kp, unsigned *sp, unsigned v1, int rank, unsigned v2) {
    const unsigned long long key = ((unsigned long long)v1 << 32) | (unsigned)rank;
    const unsigned long long old = atomicMin(kp, key);
    unsigned push = old < key ? v1 : (old != ~0ull ? (unsigned)(old >> 32) : 0xffffffffu);
    push = min(push, v2);
    if (push != 0xffffffffu) atomicMin(sp, push);
}
// Decode a keyed winner / second (clist: the chunk's candidate list in shared memory).
__device__ __forceinline__ unsigned fkey_val(float k) { return __float_as_uint(k) & ~kKeyBits; }
__device__ __forceinline__ unsigned fkey_val2(float k) { return k < kAdmissibleMax ? fkey_val(k) : 0xffffffffu; }

// out[i] = sum_{j=i}^{i+K-1} in[j], i in [0, N).
//   EXACT: running sum (all values are integers < 2^24: exact in any order).
//   K == 8 float: pairwise tree ((d0+d1)+(d2+d3))+((d4+d5)+(d6+d7)), shared.
//   other K float: left-to-right per output.
template <int K, int N, bool EXACT>
__device__ __forceinline__ void box_sum(const float (&in)[N + K - 1], float (&out)[N]) {
    if constexpr (EXACT) {
        float s = 0.f;
#pragma unroll
        for (int j = 0; j < K; ++j) s += in[j];
        out[0] = s;
#pragma unroll
        for (int i = 1; i < N; ++i) {
            s = (s + in[i + K - 1]) - in[i - 1];
            out[i] = s;
        }
    } else if constexpr (K == 8) {
        float p[N + 6], q[N + 4];
#pragma unroll
        for (int j = 0; j < N + 6; ++j) p[j] = __fadd_rn(in[j], in[j + 1]);
#pragma unroll
        for (int j = 0; j < N + 4; ++j) q[j] = __fadd_rn(p[j], p[j + 2]);
#pragma unroll
        for (int i = 0; i < N; ++i) out[i] = __fadd_rn(q[i], q[i + 4]);
    } else {
#pragma unroll
        for (int i = 0; i < N; ++i) {
            float s = in[i];
#pragma unroll
            for (int j = 1; j < K; ++j) s = __fadd_rn(s, in[i + j]);
            out[i] = s;
        }
    }
}

// A candidate is "clip-free" for a tile iff every in-frame pixel of every window of the tile
// (rows py0-KL .. py0+kTY-1+KR, likewise columns) stays in the frame when shifted by v: then no
// term of any output of the tile is dropped for v, and n(p, v) = npx(p) (the window's measured
// in-frame pixels).  Uniform per (tile, candidate); the one definition serves both bodies.
template <int K = 8>
__device__ __forceinline__ bool tile_clip_free(const BoxArgs &a, int px0, int py0, int al, int bt) {
    constexpr int KL = K / 2, KR = K - 1 - K / 2;
    const int qy_lo = max(0, py0 - KL), qy_hi = min(a.H - 1, py0 + kTY - 1 + KR);
    const int qx_lo = max(0, px0 - KL), qx_hi = min(a.W - 1, px0 + kTX - 1 + KR);
    return qy_lo + al >= 0 && qy_hi + al <= a.H - 1 && qx_lo + bt >= 0 && qx_hi + bt <= a.W - 1;
}

template <int K>
struct BoxGeom {
    static constexpr int HR = kTY + K - 1;   // H rows per tile
    static constexpr int KL = K / 2;         // offsets start at -KL
    static constexpr int NA = kRun + K - 1;  // D values per phase-A thread
    static constexpr int NB = kSeg + K - 1;  // H values per phase-B thread
    static constexpr int RUNS = kTX / kRun;  // phase-A threads per H row
};

// The body for one tile x chunk.  CNT = track supports n (border tiles and the
// reverse ME, where n varies with the candidate) -- else n is constant per output.
template <int K, bool EXACT, bool CNT, bool SSD, bool REV>
__device__ __forceinline__ void box_body(const BoxArgs &a, float *smem, int chunk, int px0, int py0,
                                         bool skip_clipfree = false) {
    using G = BoxGeom<K>;
    const int alo = chunk_alo(a.S, chunk);
    const int ahi = chunk_ahi(a.S, chunk);
    const int nrow_b = G::HR + (ahi - alo);
    const int ncol_b = kTX + K - 1 + 2 * a.S;
    const int bpitch = ncol_b | 1;
    float *Bw = smem;
    float *Hs = smem + ((nrow_b * bpitch + 3) & ~3);
    float *Ns = Hs + 2 * G::HR * kTXP;
    int *clist = reinterpret_cast<int *>(Ns + 2 * G::HR * kTXP);   // the chunk's candidates

    // Stage the chunk's B window: rows py0-KL+alo .., cols px0-KL-S ..
    const int by0 = py0 - G::KL + alo, bx0 = px0 - G::KL - a.S;
    for (int i = threadIdx.x; i < nrow_b * ncol_b; i += kNT) {
        const int r = i / ncol_b, c = i - r * ncol_b;
        Bw[r * bpitch + c] = REV ? load_cur_masked(a, by0 + r, bx0 + c) : load_ref(a, by0 + r, bx0 + c);
    }
    const int kg0 = a.chunk_off[chunk], nkc = a.chunk_off[chunk + 1] - kg0;
    for (int i = threadIdx.x; i < nkc; i += kNT) clist[i] = __ldg(a.chunked + kg0 + i);

    // Phase-A role: H row ya, columns xa0 .. xa0+kRun-1; A values in registers.
    const int ta = threadIdx.x;
    const bool actA = ta < G::HR * G::RUNS;
    const int ya = ta / G::RUNS, xa0 = (ta % G::RUNS) * kRun;
    float av[G::NA];
    {
        const int gy = py0 - G::KL + ya, gx = px0 - G::KL + xa0;
#pragma unroll
        for (int j = 0; j < G::NA; ++j)
            av[j] = actA ? (REV ? load_ref(a, gy, gx + j) : load_cur_masked(a, gy, gx + j))
                         : __int_as_float(0x7fc00000);
    }

    // Phase-B role: output column xb, rows sb*kSeg .. +kSeg-1.
    const int xb = threadIdx.x % kTX, sb = threadIdx.x / kTX;
    // exact (uint8): best (e, n, rank); float: be / bn = the two smallest keyed values (m1, m2)
    float be[kSeg], bn[kSeg];
    int br[kSeg];
#pragma unroll
    for (int i = 0; i < kSeg; ++i) { be[i] = INFINITY; bn[i] = EXACT ? 1.f : INFINITY; br[i] = -1; }
    const float ms = (float)a.min_support;

    // Forward border tiles: the support of every output for a candidate that keeps all of the
    // tile's window pixels inside the frame ("clip-free", uniform per candidate) is the count
    // of measured in-frame pixels in its window -- box-summed once here, not per candidate.
    float npx[(CNT && !REV) ? kSeg : 1];
    if constexpr (CNT && !REV) {
        __syncthreads();
        if (actA) {
            float nv[G::NA], hn[kRun];
#pragma unroll
            for (int j = 0; j < G::NA; ++j) nv[j] = (av[j] == av[j]) ? 1.f : 0.f;
            box_sum<K, kRun, true>(nv, hn);
#pragma unroll
            for (int i = 0; i < kRun; ++i) Ns[ya * kTXP + xa0 + i] = hn[i];
        }
        __syncthreads();
        float nvv[G::NB];
#pragma unroll
        for (int j = 0; j < G::NB; ++j) nvv[j] = Ns[(sb * kSeg + j) * kTXP + xb];
        box_sum<K, kSeg, true>(nvv, npx);
    }
    __syncthreads();
    int done = 0;   // candidates processed (double-buffer parity)
    for (int k = 0; k < nkc; ++k) {
        const int pk = clist[k];
        const int al = (int)(int8_t)(pk & 0xff);
        const int bt = (int)(int8_t)((pk >> 8) & 0xff);
        const int rank = pk >> 16;
        if (skip_clipfree && tile_clip_free<K>(a, px0, py0, al, bt)) continue;   // uniform: the quad body did it
        const int buf = (done++) & 1;
        float *Hb = Hs + buf * G::HR * kTXP;
        float *Nb = Ns + buf * G::HR * kTXP;
        const bool clipfree = !REV && tile_clip_free<K>(a, px0, py0, al, bt);   // uniform
        if (actA) {
            const float *brow = Bw + (ya + al - alo) * bpitch + xa0 + bt + a.S;
            QS_DCHECK(ya + al - alo >= 0 && ya + al - alo < nrow_b && xa0 + bt + a.S >= 0 &&
                      xa0 + bt + a.S + G::NA <= ncol_b);
            float d[G::NA];
            float nv[CNT ? G::NA : 1];
#pragma unroll
            for (int j = 0; j < G::NA; ++j) {
                const float t = av[j] - brow[j];
                const float dd = SSD ? __fmul_rn(t, t) : fabsf(t);
                d[j] = fmaxf(dd, 0.f);                  // NaN (no term) -> 0
                if constexpr (CNT) nv[j] = (t == t) ? 1.f : 0.f;
            }
            float h[kRun];
            box_sum<K, kRun, EXACT>(d, h);
            float4 *hp = reinterpret_cast<float4 *>(Hb + ya * kTXP + xa0);
#pragma unroll
            for (int i = 0; i < kRun / 4; ++i) hp[i] = make_float4(h[4 * i], h[4 * i + 1], h[4 * i + 2], h[4 * i + 3]);
            if constexpr (CNT) if (!clipfree) {
                float hn[kRun];
                box_sum<K, kRun, true>(nv, hn);
                float4 *np = reinterpret_cast<float4 *>(Nb + ya * kTXP + xa0);
#pragma unroll
                for (int i = 0; i < kRun / 4; ++i)
                    np[i] = make_float4(hn[4 * i], hn[4 * i + 1], hn[4 * i + 2], hn[4 * i + 3]);
            }
        }
        __syncthreads();
        {
            const float *hc = Hb + (sb * kSeg) * kTXP + xb;
            float hv[G::NB];
#pragma unroll
            for (int j = 0; j < G::NB; ++j) hv[j] = hc[j * kTXP];
            float e[kSeg];
            box_sum<K, kSeg, EXACT>(hv, e);
            if constexpr (!EXACT && !CNT) {
                // float, n constant per output: keyed e with the second-smallest (certification)
#pragma unroll
                for (int i = 0; i < kSeg; ++i) fbest(be[i], bn[i], fkey(e[i], (unsigned)k));
            } else if constexpr (!CNT) {
#pragma unroll
                for (int i = 0; i < kSeg; ++i)
                    if (e[i] < be[i]) { be[i] = e[i]; br[i] = rank; }
            } else {
                float n[kSeg];
                if (!clipfree) {
                    const float *nc = Nb + (sb * kSeg) * kTXP + xb;
                    float nvv[G::NB];
#pragma unroll
                    for (int j = 0; j < G::NB; ++j) nvv[j] = nc[j * kTXP];
                    box_sum<K, kSeg, true>(nvv, n);
                } else {
#pragma unroll
                    for (int i = 0; i < kSeg; ++i) n[i] = npx[(CNT && !REV) ? i : 0];
                }
#pragma unroll
                for (int i = 0; i < kSeg; ++i) {
                    if constexpr (!EXACT) {
                        // float: approximate mean e * rcp(n), keyed, with the second-smallest
                        const float A = n[i] >= ms ? __fmul_rn(e[i], rcp_approx(n[i])) : kInadmissible;
                        fbest(be[i], bn[i], fkey(A, (unsigned)k));
                    } else if (n[i] >= ms) {
                        if constexpr (EXACT && SSD) {
                            // exact: fp64 products of integers < 2^23 and n <= 81
                            if ((double)e[i] * (double)bn[i] < (double)be[i] * (double)n[i]) {
                                be[i] = e[i]; bn[i] = n[i]; br[i] = rank;
                            }
                        } else if constexpr (!EXACT) {
                            // float reference: fp32 cross-multiplied means (differs from the oracle's
                            // fl(e/n) only at near-ties, R23); the merge key below is fl(e/n)
                            if (__fmul_rn(e[i], bn[i]) < __fmul_rn(be[i], n[i])) {
                                be[i] = e[i]; bn[i] = n[i]; br[i] = rank;
                            }
                        } else {
                            // e <= 81*255, n <= 81: products < 2^24, exact in fp32.
                            if (e[i] * bn[i] < be[i] * n[i]) { be[i] = e[i]; bn[i] = n[i]; br[i] = rank; }
                        }
                    }
                }
            }
        }
    }

    // Merge into the global keys: (monotone order key << 32) | rank.
#pragma unroll
    for (int i = 0; i < kSeg; ++i) {
        const int py = py0 + sb * kSeg + i, px = px0 + xb;
        if constexpr (!EXACT) {
            // float: keyed winner (e for n constant, else e * rcp(n)) and second, certified later
            if (!(be[i] < kAdmissibleMax) || py < a.oy0 || py >= a.oy1 || px >= a.ox1) continue;
            check_key(a, py, px);
            const int64_t o = (int64_t)(py - a.oy0) * a.key_pitch + (px - a.ox0);
            const int rank = clist[__float_as_uint(be[i]) & kKeyBits] >> 16;
            merge_f32(a.keys_p[ref_slot(a)] + o, a.s2_p[ref_slot(a)] + o, fkey_val(be[i]), rank, fkey_val2(bn[i]));
            continue;
        }
        if (br[i] < 0 || py < a.oy0 || py >= a.oy1 || px >= a.ox1) continue;
        unsigned long long hi;
        if constexpr (!CNT) {
            hi = __float_as_uint(be[i]);                 // e (interior: n constant): non-negative float
        } else {
            // floor(e * 2^13 / n): distinct means with n <= 81 differ by >= 1/6561 > 2^-13,
            // equal means give equal keys; fp64 division of exact integers cannot round
            // across an integer boundary at these magnitudes.
            hi = (unsigned long long)floor((double)be[i] * 8192.0 / (double)bn[i]);
        }
        const unsigned long long key = (hi << 32) | (unsigned)br[i];
        check_key(a, py, px);
        atomicMin(a.keys_p[ref_slot(a)] + (int64_t)(py - a.oy0) * a.key_pitch + (px - a.ox0), key);
    }
}

// ---------------------------------------------------------------------------
// Quarter-sampling body (K = 8, forward ME, interior tiles): DESIGN.md "K1 me_quad".
//
// With a quarter mask every 2x2 block b holds exactly one measured pixel at
// (dy_b, dx_b), so for a candidate v the only non-zero D_v
// of block b is d_b = phi(c_b - ref(pos_b + v)).  Split d_b into four channels
// G_c (c = 2 dy + dx, one non-zero).  For an output p = (2i+sy, 2j+sx) the 8x8
// window covers block rows i-2..i+1 (sy = 0), or for sy = 1 the dy=1 pixels of
// rows i-2..i+1 and the dy=0 pixels of rows i-1..i+2 (likewise columns), so
//   E(2i,  2j  ) = V[C0](i) + V[C1](i)        C0 = G0+G1, C1 = G2+G3 (by dy)
//   E(2i,  2j+1) = V[D0](i) + V[D1](i)        D0(k) = G1(k)+G0(k+1), D1(k) = G3(k)+G2(k+1)
//   E(2i+1,2j  ) = V[C1](i) + V[C0](i+1)
//   E(2i+1,2j+1) = V[D1](i) + V[D0](i+1)
// where H[X](i,j) = sum_{k=j-2}^{j+1} X(i,k) and V[X](i) = sum_{h=i-2}^{i+1} H[X](h).
// All box sums are 4-wide on the block grid (a quarter of the pixels), done as
// pairwise trees (no subtraction: exact for uint8 data, order-fixed for float).
// Producer warps 0-3 form d, the channel series and H (one warp per 9 block
// columns, one lane per block row); consumer warps 4-7 form V, E and the
// running argmin (one lane per block column, 7 block rows per warp), handing
// H over through a 2-stage shared ring guarded by named barriers.
// ---------------------------------------------------------------------------
constexpr int kQBX = kTX / 2;           // 32 block columns per tile
constexpr int kQBY = kTY / 2;           // 28 block rows per tile
constexpr int kQHR = kQBY + 4;          // 32 H rows (block rows -2 .. 29)
constexpr int kQHC = kQBX;              // 32 H columns (D already carries the k+1 block)
constexpr int kQHP = kQHC + 1;          // H plane row pitch in packed pairs (66 words = 2 mod 4: conflict-free STS.64)
constexpr int kQRun = 8;                // H columns per producer warp (4 x 8 = 32)
constexpr int kQG = kQRun + 4;          // blocks read per producer lane (12: k = j-2 .. j+1, +1 for D)
// Interior tiles: two producer warp pairs (even / odd candidates), 16 H columns per lane.
constexpr int kQRunI = 16;
constexpr int kQGI = kQRunI + 4;        // 20 blocks read per interior producer lane
constexpr int kQBarI = 64 + 128;        // threads on an interior FULL / EMPTY barrier: one producer pair + consumers
constexpr int kQSeg = kQBY / 2;         // 14 output block rows per consumer lane (2 row halves x C/D planes)
constexpr int kQWinRows = 2 * kQHR;     // 64 pixel rows of blocks per tile (+ alpha range)
constexpr int kQWinCols = 2 * (4 * kQRun + 4);  // 72 pixel columns (blocks -2 .. 33)
static_assert(kQWinRows == kQWinRowsHost && kQWinCols == kQWinColsHost, "host copies of the window size");

// Named barriers with immediate ids (1..4), so ptxas reserves only the ones used.
template <int ID, int CNT = kNT>
__device__ __forceinline__ void nb_sync_i() { asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(CNT) : "memory"); }
template <int ID, int CNT = kNT>
__device__ __forceinline__ void nb_arrive_i() { asm volatile("bar.arrive %0, %1;" ::"n"(ID), "n"(CNT) : "memory"); }
__device__ __forceinline__ void nb_sync(int id, int) {
    switch (id) {
        case 1: nb_sync_i<1>(); break;
        case 2: nb_sync_i<2>(); break;
        case 3: nb_sync_i<3>(); break;
        case 4: nb_sync_i<4>(); break;
        case 5: nb_sync_i<5>(); break;
        case 6: nb_sync_i<6>(); break;
        case 7: nb_sync_i<7>(); break;
        default: nb_sync_i<8>(); break;
    }
}
__device__ __forceinline__ void nb_arrive(int id, int) {
    switch (id) {
        case 1: nb_arrive_i<1>(); break;
        case 2: nb_arrive_i<2>(); break;
        case 3: nb_arrive_i<3>(); break;
        case 4: nb_arrive_i<4>(); break;
        case 5: nb_arrive_i<5>(); break;
        case 6: nb_arrive_i<6>(); break;
        case 7: nb_arrive_i<7>(); break;
        default: nb_arrive_i<8>(); break;
    }
}
constexpr int kQStages = 2;   // H ring depth: FULL[s] = barrier 1+s, EMPTY[s] = barrier 5+s

// 1 iff every block the quad body reads (rows -2..29, cols -2..33) that lies in the frame and in
// the caller's buffer holds exactly one measured pixel (blocks outside are empty: no terms).
__device__ __forceinline__ bool quad_mask_ok(const BoxArgs &a, int px0, int py0) {
    bool ok = true;
    constexpr int NR = kQHR, NC = kQBX + 4;   // 32 x 36 blocks: rows -2..29, cols -2..33
    for (int i = threadIdx.x; i < NR * NC; i += kNT) {
        const int bi = i / NC - 2, bk = i % NC - 2;
        const int y = py0 + 2 * bi, x = px0 + 2 * bk;
        if (y < 0 || y + 1 >= a.H || x < 0 || x + 1 >= a.W || y < a.buf_y0 || y + 1 >= a.buf_y0 + a.buf_rows)
            continue;
        const int64_t r = (int64_t)(y - a.buf_y0) * a.mask.pitch;
        const int n = a.mask.p[r + x] + a.mask.p[r + x + 1] + a.mask.p[r + a.mask.pitch + x] +
                      a.mask.p[r + a.mask.pitch + x + 1];
        ok = ok && (n == 1);
    }
    return __syncthreads_and(ok);
}

// ---- packed fp32x2 helpers (sm_100a FADD2 / FMUL2 / FFMA2; ptxas folds {x,x} broadcasts and |x|) ----
typedef unsigned long long f2_t;
__device__ __forceinline__ f2_t f2pack(float a, float b) {
    f2_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
__device__ __forceinline__ float f2lo(f2_t x) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x));
    return a;
}
__device__ __forceinline__ float f2hi(f2_t x) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x));
    return b;
}
__device__ __forceinline__ f2_t f2add(f2_t a, f2_t b) {
    f2_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t f2sub(f2_t a, f2_t b) {
    f2_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t f2mul(f2_t a, f2_t b) {
    f2_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2_t f2fma(f2_t a, f2_t b, f2_t c) {
    f2_t r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}

// 8-byte shared store / load of one packed pair (shared-window byte address).
__device__ __forceinline__ void st_shared_f2(unsigned addr, f2_t x) {
    asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr), "l"(x) : "memory");
}
__device__ __forceinline__ f2_t ld_shared_f2(unsigned addr) {
    f2_t x;
    asm volatile("ld.shared.b64 %0, [%1];" : "=l"(x) : "r"(addr) : "memory");
    return x;
}

// BORDER = the tile's windows or candidates reach outside the frame / buffer.  Blocks outside the
// frame are empty (weight 0) and reference pixels outside read NaN, zeroed by fmaxf(t, 0).  The
// candidates run in two phases:
//   phase 1, the tile's clip-free candidates (tile_clip_free: n(p, v) = npx(p) for all of them, so
//     the running minimum compares e alone), then one ring entry with d = 1 per measured in-frame
//     pixel whose box sums are npx(p): the consumers merge phase 1 with the mean key (fl(e/npx) for
//     float references, floor(e * 2^13 / npx) for uint8 -- the keys box_body uses);
//   phase 2 (Q2), the other candidates: every ring entry also carries the support planes (box sums
//     of the per-term indicator), the consumers compare means by cross-multiplication and merge
//     with the same mean key.  The 64-bit atomicMin of (mean key, rank) merges both phases in the
//     R7 order (the key is monotone and tie-preserving in the mean).
// Without Q2 (uint8 SSD: cross-multiplied sums could exceed 2^24) phase 2 runs in box_body.
//
// H hand-over: per ring stage four planes of packed pairs, C = (H[C0], H[C1]), D = (H[D0], H[D1])
// and, in phase 2, their support twins CN, DN; [kQHR rows][kQHP pairs] each.  Producers store one
// STS.64 per plane and column (row pitch 66 words: a half-warp of rows hits 32 distinct banks),
// consumers read one LDS.64 per row (lanes = consecutive columns).  Consumer warp c: plane c & 1
// (output columns 2j + (c & 1)), block rows 14 (c >> 1) .. +13, both row parities: 28 outputs per
// lane from 18 H rows.
constexpr int kQPlanes = 4;   // planes per ring stage
// Quad reference window geometry (floats): row pitch 2 x odd >= cols; plane = ceil(rows / 2) rows,
// rounded up to a multiple of 32 words.
__host__ __device__ constexpr int quad_pitch(int cols) { return 2 * (((cols + 1) / 2) | 1); }
__host__ __device__ constexpr int quad_plane(int rows, int cols) { return (((rows + 1) / 2) * quad_pitch(cols) + 31) & ~31; }

// RUNS (float border tiles of a split launch): phase 2 in runs of equal supports -- the list-B
// candidates sorted by their support key (the support planes depend on v only through the rows /
// columns that clip), the producers roll the support planes once per run and the consumers keep
// 1 / n per output for the run.
template <bool SSD, bool EXACT, bool BORDER, bool RUNS = false>
__device__ __forceinline__ void quad_body(const BoxArgs &a, float *smem, int chunk, int px0, int py0,
                                          bool skip_phase1 = false) {
    constexpr bool Q2 = BORDER && !(EXACT && SSD);
    static_assert(!RUNS || (BORDER && !EXACT), "support runs: float border tiles only");
    const int alo = chunk_alo(a.S, chunk);
    const int ahi = chunk_ahi(a.S, chunk);
    const int nrow_b = kQWinRows + (ahi - alo);
    const int ncol_b = kQWinCols + 2 * a.S;
    // Reference window split by row parity: row y at plane (y & 1), plane row y >> 1.  Row pitch
    // bpitch = 2 x odd and plane pitch = 0 mod 32 words: a warp's 32 gathers (one block row per lane,
    // the block's row parity choosing the plane) fall into distinct banks except lanes 16 apart.
    // With TMA (float references) the planes hold the descriptor's box: tma_rows rows of tma_cols
    // floats (a multiple of 4: TMA rows are 16-byte multiples, which costs the conflict-light pitch).
    const bool tma = a.tma != 0;
    const int bpitch = tma ? a.tma_cols : quad_pitch(ncol_b);
    const int bplane = tma ? ((a.tma_rows * a.tma_cols + 31) & ~31) : quad_plane(nrow_b, ncol_b);
    float *Bw = smem;
    f2_t *Hp = reinterpret_cast<f2_t *>(smem + 2 * bplane);   // [kQStages][kQPlanes][kQHR][kQHP]
    int *clist = reinterpret_cast<int *>(Hp + kQStages * kQPlanes * kQHR * kQHP);   // the chunk's candidates
    int *nsel = clist + kChunkRows * (2 * a.S + 1);   // a chunk holds <= 7 alpha rows
    constexpr int kPlane = kQHR * kQHP;                  // pairs per plane
    constexpr unsigned kStageBytes = kQPlanes * kPlane * 8;

    // Stage the chunk's reference window (rows py0-4+alo .., cols px0-4-S ..) and candidate list.
    const int by0 = py0 - 4 + alo, bx0 = px0 - 4 - a.S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ __align__(8) unsigned long long tma_bar;
    if (tma) {
        // Two TMA box loads (row-parity planes p = 0, 1: window rows by0 + p, by0 + p + 2, ...),
        // completion counted on one mbarrier; the hardware fills NaN outside the frame and buffer.
        const unsigned bar = (unsigned)__cvta_generic_to_shared(&tma_bar);
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bar) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            const unsigned bytes = 2u * (unsigned)(a.tma_rows * a.tma_cols) * 4u;
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
            const CUtensorMap *tm = &a.tmap[ref_slot(a)];
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                const int b = by0 + p - a.buf_y0;   // buffer row of window row p
                const unsigned dst = (unsigned)__cvta_generic_to_shared(Bw + p * bplane);
                QS_DCHECK((dst & 127u) == 0u);
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                    ::"r"(dst), "l"(reinterpret_cast<uint64_t>(tm)), "r"(bx0), "r"(b & 1), "r"(b >> 1), "r"(bar)
                    : "memory");
            }
        }
        __syncthreads();
        asm volatile(
            "{\n\t.reg .pred P;\n"
            "WAIT_%=:\n\t"
            "mbarrier.try_wait.parity.shared.b64 P, [%0], 0;\n\t"
            "@!P bra WAIT_%=;\n\t}" ::"r"(bar) : "memory");
    } else {
        // One window row per warp iteration, lanes along the row (coalesced, no index division).
        // float references: in-frame values go global -> shared by cp.async (no register round
        // trip, many copies in flight); everything else (uint8 conversion, NaN outside the frame or
        // the buffer) through registers.
        const uint8_t *rp = a.ref_p[ref_slot(a)];
        for (int r = warp; r < nrow_b; r += kNT / 32) {
            const int y = by0 + r;
            const bool row_in = y >= 0 && y < a.H && y >= a.buf_y0 && y < a.buf_y0 + a.buf_rows;
            float *dst = Bw + (r & 1) * bplane + (r >> 1) * bpitch;
            const float *src = reinterpret_cast<const float *>(rp + (int64_t)(y - a.buf_y0) * a.ref.pitch);
            for (int c = lane; c < ncol_b; c += 32) {
                const int x = bx0 + c;
                if (a.ref_f32 && row_in && x >= 0 && x < a.W)
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(dst + c)),
                                 "l"(src + x));
                else
                    dst[c] = load_ref(a, y, x);
            }
        }
        asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
    }
    const int k0g = a.chunk_off[chunk], nkc = a.chunk_off[chunk + 1] - k0g;
    int nA = nkc, nB = 0;
    if constexpr (!BORDER) {
        for (int i = threadIdx.x; i < nkc; i += kNT) clist[i] = __ldg(a.chunked + k0g + i);
    } else {
        // Clip-free candidates (list A), then the others (list B, phase 2), each in rank order
        // (one warp, ballot + popc).
        if (warp == 0) {
            int n = 0;
            for (int pass = 0; pass < (Q2 ? 2 : 1); ++pass) {
                for (int base = 0; base < nkc; base += 32) {
                    const int i = base + lane;
                    int pk = 0;
                    bool keep = false;
                    if (i < nkc) {
                        pk = __ldg(a.chunked + k0g + i);
                        keep = tile_clip_free<8>(a, px0, py0, (int)(int8_t)(pk & 0xff),
                                                 (int)(int8_t)((pk >> 8) & 0xff)) == (pass == 0);
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, keep);
                    if (keep) clist[n + __popc(m & ((1u << lane) - 1u))] = pk;
                    n += __popc(m);
                }
                if (lane == 0) nsel[pass] = n;
            }
        }
        if constexpr (RUNS) {
            // Support key of each list-B candidate: (alpha if its rows clip, beta if its columns clip);
            // equal keys = identical support planes.  Sorted (rank order inside a key) by counting the
            // entries before each one; order inside the list is free for the float argmin (the keyed
            // position decodes the rank; near-ties are recomputed exactly by certify).
            __syncthreads();
            const int b0 = nsel[0], nb = nsel[1] - nsel[0];
            int *skey = nsel + 8, *stmp = skey + kChunkRows * (2 * a.S + 1);
            const int qy_lo = max(0, py0 - 4), qy_hi = min(a.H - 1, py0 + kTY + 2);
            const int qx_lo = max(0, px0 - 4), qx_hi = min(a.W - 1, px0 + kTX + 2);
            for (int i = threadIdx.x; i < nb; i += kNT) {
                const int pk = clist[b0 + i];
                const int al = (int)(int8_t)(pk & 0xff), bt = (int)(int8_t)((pk >> 8) & 0xff);
                const bool rc = qy_lo + al < 0 || qy_hi + al > a.H - 1;
                const bool cc = qx_lo + bt < 0 || qx_hi + bt > a.W - 1;
                stmp[i] = ((rc ? al + 64 : 0) << 8) | (cc ? bt + 64 : 0);
            }
            __syncthreads();
            int dst[2], pks[2], ks[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int i = threadIdx.x + u * kNT;
                dst[u] = -1;
                if (i < nb) {
                    const int ki = stmp[i];
                    int d = 0;
                    for (int jx = 0; jx < nb; ++jx) {
                        const int kj = stmp[jx];
                        d += (kj < ki || (kj == ki && jx < i)) ? 1 : 0;
                    }
                    dst[u] = d;
                    pks[u] = clist[b0 + i];
                    ks[u] = ki;
                }
            }
            __syncthreads();
#pragma unroll
            for (int u = 0; u < 2; ++u)
                if (dst[u] >= 0) {
                    clist[b0 + dst[u]] = pks[u];
                    skey[dst[u]] = ks[u];
                }
            static_assert(2 * kNT >= kChunkRows * 65, "two list-B entries per thread cover S <= 32");
        }
    }
    __syncthreads();
    int a0 = nA;   // list position of list B
    if constexpr (BORDER) {
        a0 = nsel[0];
        nB = Q2 ? nsel[1] - a0 : 0;
        nA = skip_phase1 ? 0 : a0;   // phase 1 already done (uint8: the integer body)
    }
    const int e1 = nA + ((BORDER && nA > 0) ? 1 : 0);   // entries of phase 1 (+ the npx entry)
    const int n_ent = e1 + nB;
    if (n_ent <= 0) return;                              // uniform

    if constexpr (!BORDER) {
        // Keyed argmin (uint8 SAD): every interior sum is an integer <= 25 * 255, so with the block
        // values scaled by 2^9 and the candidate's chunk-list position k (< 2^9, rank order) added
        // once per window, E' = 512 E + k is exact in fp32 (< 2^24) and orders (E, rank) exactly
        // (R7): the running argmin is one FMNMX per output instead of compare + two selects.
        constexpr bool KEYED = EXACT && !SSD;
        constexpr float kKeyScale = KEYED ? 512.f : 1.f;
        // ------------------- interior: warp-specialised registers -------------------
        // Producers: two warp pairs; pair p = (warp >> 1) reduces the candidates k = p, p + 2, ...
        // into ring stage p, warp half = warp & 1 of a pair takes H columns 16 half .. +15 (20 blocks
        // gathered per lane: 1.25x the columns instead of 1.5x).  setmaxnreg: producers 152, consumers
        // 104 registers (the 20 blocks' statics).  FULL[p] / EMPTY[p] = named barriers 1 + p / 5 + p
        // over the 64 threads of pair p and the 128 consumers.
        if (warp < 4) {
            asm volatile("setmaxnreg.inc.sync.aligned.u32 152;" ::: "memory");
            const int hr = lane, bi = hr - 2;
            const int pair = warp >> 1, half = warp & 1;
            float cv[kQGI], wx[kQGI];
            f2_t wy2[kQGI];
            int ad[kQGI];
#pragma unroll
            for (int kk = 0; kk < kQGI; ++kk) {
                const int bk = kQRunI * half - 2 + kk;
                const int y = py0 + 2 * bi, x = px0 + 2 * bk;
                // blocks below the frame / the buffer (a band's ragged last tile): weight 0; they feed
                // only outputs that are never merged
                const bool inside = y + 1 < a.H && y + 1 < a.buf_y0 + a.buf_rows;
                const int64_t r = (int64_t)(y - a.buf_y0);
                const uint8_t *m0 = a.mask.p + r * a.mask.pitch + x;
                const int q = !inside ? 0 : m0[1] ? 1 : m0[a.mask.pitch] ? 2 : m0[a.mask.pitch + 1] ? 3 : 0;
                const int dy = q >> 1, dx = q & 1;
                cv[kk] = inside ? (float)a.cur.p[(r + dy) * a.cur.pitch + x + dx] : 0.f;
                wy2[kk] = inside ? f2pack(kKeyScale * (float)(1 - dy), kKeyScale * (float)dy)   // x 2^9 when keyed
                                 : f2pack(0.f, 0.f);
                wx[kk] = (float)(dx - 1);
                ad[kk] = 4 * (dy * bplane + (bi + 2) * bpitch + (2 * bk + dx + 4 + a.S));
            }
            const unsigned hbase = (unsigned)__cvta_generic_to_shared(Hp + hr * kQHP + kQRunI * half);
            auto run = [&](auto Pc) {   // Pc = std::integral_constant pair (compile-time barrier ids)
                constexpr int P = decltype(Pc)::value;
                const unsigned hs = hbase + (unsigned)P * kStageBytes;
                float rv[kQGI];
                auto gather = [&](int ci) {
                    const int pk = clist[ci];
                    const char *bwc = reinterpret_cast<const char *>(
                        Bw + (((int)(int8_t)(pk & 0xff) - alo) >> 1) * bpitch + (int)(int8_t)((pk >> 8) & 0xff));
#pragma unroll
                    for (int kk = 0; kk < kQGI; ++kk) {
                        QS_DCHECK(bwc + ad[kk] >= reinterpret_cast<const char *>(Bw) &&
                                  bwc + ad[kk] + 4 <= reinterpret_cast<const char *>(Bw + 2 * bplane));
                        rv[kk] = *reinterpret_cast<const float *>(bwc + ad[kk]);
                    }
                };
                for (int k = P; k < nA; k += 2) {
                    gather(k);
                    if (k >= 2) nb_sync_i<5 + P, kQBarI>();           // EMPTY[P]: candidate k-2 was read
                    f2_t u[kQGI], m[kQGI - 1], pu[kQGI - 1], pm[kQGI - 2], gp = 0ull;
#pragma unroll
                    for (int kk = 0; kk < kQGI; ++kk) {
                        const float d = __fsub_rn(cv[kk], rv[kk]);
                        const float t = SSD ? __fmul_rn(d, d) : fabsf(d);
                        u[kk] = f2mul(f2pack(t, t), wy2[kk]);
                        // wx = dx - 1 in {-1, 0}: g1 = u * dx = u + u * wx, D = gp + u * (1 - dx) (exact splits)
                        const f2_t g1 = f2fma(u[kk], f2pack(wx[kk], wx[kk]), u[kk]);
                        if (kk > 0) m[kk - 1] = f2fma(u[kk], f2pack(-wx[kk], -wx[kk]), gp);
                        gp = g1;
                        if (kk >= 1) pu[kk - 1] = f2add(u[kk - 1], u[kk]);
                        if (kk >= 2) pm[kk - 2] = f2add(m[kk - 2], m[kk - 1]);
                        if (kk >= 3 && kk - 3 < kQRunI) st_shared_f2(hs + 8 * (kk - 3), f2add(pu[kk - 3], pu[kk - 1]));
                        if (kk >= 4 && kk - 4 < kQRunI)
                            st_shared_f2(hs + 8 * (kPlane + kk - 4), f2add(pm[kk - 4], pm[kk - 2]));
                    }
                    nb_arrive_i<1 + P, kQBarI>();                       // FULL[P]
                }
                if (P < nA) nb_sync_i<5 + P, kQBarI>();                // drain: the last candidate was read
            };
            if (pair == 0) run(std::integral_constant<int, 0>{});
            else run(std::integral_constant<int, 1>{});
        } else {
            asm volatile("setmaxnreg.dec.sync.aligned.u32 104;" ::: "memory");
            const int j = lane;
            const int cw = warp - 4, pl = cw & 1, i0 = kQSeg * (cw >> 1);
            // float (FK): be / m2 = the two smallest keyed e per output (certified argmin); exact: (e, rank)
            constexpr bool FK = !EXACT;
            float be[kQSeg][2];
            int br[FK ? 1 : kQSeg][2];
            float m2[FK ? kQSeg : 1][2];
#pragma unroll
            for (int r = 0; r < kQSeg; ++r)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    be[r][c] = INFINITY;
                    if constexpr (FK) m2[r][c] = INFINITY;
                    else br[r][c] = -1;
                }
            const unsigned cbase = (unsigned)__cvta_generic_to_shared(Hp + pl * kPlane + i0 * kQHP + j);
            auto consume = [&](int k, auto Pc) {
                constexpr int P = decltype(Pc)::value;
                const int rank = clist[k] >> 16;
                nb_sync_i<1 + P, kQBarI>();                             // FULL[P]
                const unsigned cs = cbase + (unsigned)P * kStageBytes;
                f2_t x[kQSeg + 4];
#pragma unroll
                for (int t = 0; t < kQSeg + 4; ++t) x[t] = ld_shared_f2(cs + 8 * t * kQHP);
                nb_arrive_i<5 + P, kQBarI>();                           // EMPTY[P]
                f2_t pp0 = f2add(x[0], x[1]), pp1 = f2add(x[1], x[2]), pp2 = f2add(x[2], x[3]);
                f2_t pp3 = f2add(x[3], x[4]);
                // keyed: (k, 0) added to every V, so each E (one lo + one hi) carries k exactly once
                const f2_t kk2 = f2pack(KEYED ? (float)k : 0.f, 0.f);
                f2_t vcur = f2add(pp0, pp2);
                if constexpr (KEYED) vcur = f2add(vcur, kk2);
#pragma unroll
                for (int r = 0; r < kQSeg; ++r) {
                    f2_t vnext = f2add(pp1, pp3);
                    if constexpr (KEYED) vnext = f2add(vnext, kk2);
                    const float ev[2] = {__fadd_rn(f2lo(vcur), f2hi(vcur)), __fadd_rn(f2hi(vcur), f2lo(vnext))};
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        if constexpr (KEYED) be[r][c] = fminf(be[r][c], ev[c]);
                        else if constexpr (FK) fbest(be[r][c], m2[r][c], fkey(ev[c], (unsigned)k));
                        else if (ev[c] < be[r][c]) { be[r][c] = ev[c]; br[r][c] = rank; }
                    }
                    vcur = vnext;
                    pp0 = pp1;
                    pp1 = pp2;
                    pp2 = pp3;
                    if (r + 5 < kQSeg + 4) pp3 = f2add(x[r + 4], x[r + 5]);
                }
            };
            for (int k = 0; k < nA; k += 2) {
                consume(k, std::integral_constant<int, 0>{});
                if (k + 1 < nA) consume(k + 1, std::integral_constant<int, 1>{});
            }
#pragma unroll
            for (int r = 0; r < kQSeg; ++r)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const int py = py0 + 2 * (i0 + r) + c, px = px0 + 2 * j + pl;
                    if constexpr (FK) {
                        if (!(be[r][c] < kAdmissibleMax) || py < a.oy0 || py >= a.oy1 || px >= a.ox1) continue;
                        check_key(a, py, px);
                        const int64_t o = (int64_t)(py - a.oy0) * a.key_pitch + (px - a.ox0);
                        merge_f32(a.keys_p[ref_slot(a)] + o, a.s2_p[ref_slot(a)] + o, fkey_val(be[r][c]),
                                  clist[__float_as_uint(be[r][c]) & kKeyBits] >> 16, fkey_val2(m2[r][c]));
                    } else {
                        if constexpr (KEYED) {
                            if (!(be[r][c] < INFINITY)) continue;
                            const unsigned kv = (unsigned)be[r][c];           // 512 E + k, exact
                            br[r][c] = clist[kv & 511u] >> 16;
                            be[r][c] = (float)(kv >> 9);
                        }
                        if (br[r][c] < 0 || py < a.oy0 || py >= a.oy1 || px >= a.ox1) continue;
                        const unsigned long long key =
                            ((unsigned long long)__float_as_uint(be[r][c]) << 32) | (unsigned)br[r][c];
                        check_key(a, py, px);
        atomicMin(a.keys_p[ref_slot(a)] + (int64_t)(py - a.oy0) * a.key_pitch + (px - a.ox0), key);
                    }
                }
        }
        return;
    }

    if (warp < 4) {
        // ------------------------------ producer ------------------------------
        // lane = H row (block row + 2), 8 H columns per warp, 12 blocks read per lane.
        // RUNS: registers move to the consumers (their 1 / n per output): producers 120, consumers 136.
        if constexpr (RUNS) asm volatile("setmaxnreg.dec.sync.aligned.u32 120;" ::: "memory");
        const int hr = lane;
        const int bi = hr - 2;
        float cv[kQG], wx[kQG];
        f2_t wy2[kQG];   // (1 - dy, dy); (0, 0) for an empty block
        int ad[kQG];     // byte offset of the block's measured pixel in the window (candidate (alo, 0))
#pragma unroll
        for (int kk = 0; kk < kQG; ++kk) {
            const int bk = kQRun * warp - 2 + kk;
            const int y = py0 + 2 * bi, x = px0 + 2 * bk;
            const bool inside = y >= 0 && y + 1 < a.H && x >= 0 && x + 1 < a.W && y >= a.buf_y0 &&
                                y + 1 < a.buf_y0 + a.buf_rows;
            int dy = 0, dx = 0;
            float c = 0.f;
            if (inside) {
                const int64_t r = (int64_t)(y - a.buf_y0);
                const uint8_t *m0 = a.mask.p + r * a.mask.pitch + x;
                const int q = m0[1] ? 1 : m0[a.mask.pitch] ? 2 : m0[a.mask.pitch + 1] ? 3 : 0;
                dy = q >> 1;
                dx = q & 1;
                c = (float)a.cur.p[(r + dy) * a.cur.pitch + x + dx];
            }
            cv[kk] = c;
            wy2[kk] = inside ? f2pack((float)(1 - dy), (float)dy) : f2pack(0.f, 0.f);
            wx[kk] = (float)(dx - 1);
            // window row 2 bi + dy + 4 + (alpha - alo), alpha - alo even: plane dy, plane row bi + 2 + (alpha - alo) / 2
            ad[kk] = 4 * (dy * bplane + (bi + 2) * bpitch + (2 * bk + dx + 4 + a.S));
        }
        const unsigned hbase = (unsigned)__cvta_generic_to_shared(Hp + hr * kQHP + kQRun * warp);
        // Gathers of the reference values of the candidate at list position ci (its window offset).
        auto gather = [&](int ci, float (&dst)[kQG]) {
            const int pk = clist[ci];
            const char *bwc = reinterpret_cast<const char *>(Bw + (((int)(int8_t)(pk & 0xff) - alo) >> 1) * bpitch +
                                                             (int)(int8_t)((pk >> 8) & 0xff));
#pragma unroll
            for (int kk = 0; kk < kQG; ++kk) {
                QS_DCHECK(bwc + ad[kk] >= reinterpret_cast<const char *>(Bw) &&
                          bwc + ad[kk] + 4 <= reinterpret_cast<const char *>(Bw + 2 * bplane));
                dst[kk] = *reinterpret_cast<const float *>(bwc + ad[kk]);
            }
        };
        // Series of one block (rolling, in block order): u = (C0, C1) parts, m(k-1) = (D0, D1)(k-1)
        // = G_dx1(k-1) + G_dx0(k); pu(k) = u(k) + u(k+1), pm(k) = m(k) + m(k+1); H(j) = pu(j) + pu(j+2)
        // (pairwise, packed), stored to planes P (C) and P + 1 (D) as soon as complete.
        struct Roll {
            f2_t u[kQG], m[kQG - 1], pu[kQG - 1], pm[kQG - 2], gp;
        };
        auto roll = [&](Roll &R, int kk, float t, unsigned hs, int P) {
            R.u[kk] = f2mul(f2pack(t, t), wy2[kk]);                  // (C0, C1) = (dy0, dy1) parts
            // wx = dx - 1 in {-1, 0}: (G1, G3) = dx1 parts = u * dx = u + u * wx (exact)
            const f2_t g1 = f2fma(R.u[kk], f2pack(wx[kk], wx[kk]), R.u[kk]);
            // D(k-1) = G(dx1, k-1) + G(dx0, k); G(dx0) = u * (1 - dx) is exactly u or 0
            if (kk > 0) R.m[kk - 1] = f2fma(R.u[kk], f2pack(-wx[kk], -wx[kk]), R.gp);
            R.gp = g1;
            if (kk >= 1) R.pu[kk - 1] = f2add(R.u[kk - 1], R.u[kk]);
            if (kk >= 2) R.pm[kk - 2] = f2add(R.m[kk - 2], R.m[kk - 1]);
            if (kk >= 3 && kk - 3 < kQRun)
                st_shared_f2(hs + 8 * (P * kPlane + kk - 3), f2add(R.pu[kk - 3], R.pu[kk - 1]));
            if (kk >= 4 && kk - 4 < kQRun)
                st_shared_f2(hs + 8 * ((P + 1) * kPlane + kk - 4), f2add(R.pm[kk - 4], R.pm[kk - 2]));
        };
        // One ring entry e in stage s: reduce the candidate whose gathers are in cur[] while the
        // gathers of list position nci go to nxt[] (nci < 0: none).  mode 0: phase-1 candidate,
        // 1: the npx entry (d = 1 per measured pixel), 2: phase-2 candidate (+ support planes).
        auto produce = [&](int e, const int s, const float (&cur)[kQG], float (&nxt)[kQG], int nci, const int mode,
                           int ci = 0) {
            bool roll_n = true;   // support planes of this entry (RUNS: only at a run's first entry)
            if constexpr (RUNS) {
                const int* skey = nsel + 8;
                roll_n = ci == a0 || skey[ci - a0] != skey[ci - a0 - 1];
            }
            if (nci >= 0) gather(nci, nxt);
            if (e >= kQStages) nb_sync(5 + s, kNT);                  // EMPTY[s]: consumers released stage s
            const unsigned hs = hbase + (unsigned)s * kStageBytes;
            Roll R, N;
            R.gp = 0ull;
            N.gp = 0ull;
#pragma unroll
            for (int kk = 0; kk < kQG; ++kk) {
                const float d = mode == 1 ? 1.f : __fsub_rn(cv[kk], cur[kk]);
                const float t0 = SSD ? __fmul_rn(d, d) : fabsf(d);
                const float t = fmaxf(t0, 0.f);                       // NaN (outside the frame) -> 0
                roll(R, kk, t, hs, 0);
                if (!RUNS && Q2 && mode == 2) roll(N, kk, (t0 == t0) ? 1.f : 0.f, hs, 2);   // term indicator
            }
            if constexpr (RUNS) {   // support planes at a run's first entry only, in a loop of their own
                if (mode == 2 && roll_n) {
#pragma unroll
                    for (int kk = 0; kk < kQG; ++kk) roll(N, kk, (cur[kk] == cur[kk]) ? 1.f : 0.f, hs, 2);
                }
            }
            nb_arrive(1 + s, kNT);                                   // FULL[s]
        };
        // A run of n candidates (list positions ci0 ..) as entries e0 .., unrolled by two with ping-pong
        // gather buffers (no register copies between candidates); stage ids are compile-time.
        float ra[kQG], rb[kQG];
        auto run = [&](int ci0, int n, int e0, const int mode) {
            if (n <= 0) return;
            gather(ci0, ra);
            if ((e0 & 1) == 0) {
                for (int i = 0; i < n; i += 2) {
                    produce(e0 + i, 0, ra, rb, i + 1 < n ? ci0 + i + 1 : -1, mode, ci0 + i);
                    if (i + 1 < n) produce(e0 + i + 1, 1, rb, ra, i + 2 < n ? ci0 + i + 2 : -1, mode, ci0 + i + 1);
                }
            } else {
                for (int i = 0; i < n; i += 2) {
                    produce(e0 + i, 1, ra, rb, i + 1 < n ? ci0 + i + 1 : -1, mode, ci0 + i);
                    if (i + 1 < n) produce(e0 + i + 1, 0, rb, ra, i + 2 < n ? ci0 + i + 2 : -1, mode, ci0 + i + 1);
                }
            }
        };
        static_assert(kQStages == 2, "stage ids are compile-time constants of the unrolled loops");
        run(0, nA, 0, 0);
        if (nA > 0) {
            if (nA & 1) produce(nA, 1, ra, rb, -1, 1);
            else produce(nA, 0, ra, rb, -1, 1);
        }
        if constexpr (Q2) run(a0, nB, e1, 2);
        for (int k = max(0, n_ent - kQStages); k < n_ent; ++k) nb_sync(5 + (k & (kQStages - 1)), kNT);   // drain
    } else {
        // ------------------------------ consumer ------------------------------
        // lane = block column j; plane pl (0: C, output column 2j; 1: D, output column 2j+1);
        // block rows i0 .. i0+13, both row parities; candidates in rank order, strict '<' (R7).
        if constexpr (RUNS) asm volatile("setmaxnreg.inc.sync.aligned.u32 136;" ::: "memory");
        const int j = lane;
        const int cw = warp - 4, pl = cw & 1, i0 = kQSeg * (cw >> 1);
        // exact (uint8): best (e, rank) / (e, n, rank); float (FK): be / m2 = the two smallest keyed
        // values per output (phase 1: e; phase 2: e * rcp(n)) for the certified argmin.
        constexpr bool FK = !EXACT;
        float be[kQSeg][2];
        int br[FK ? 1 : kQSeg][2];
        float m2[FK ? kQSeg : 1][2];
        auto reset = [&]() {
#pragma unroll
            for (int r = 0; r < kQSeg; ++r)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    be[r][c] = INFINITY;
                    if constexpr (FK) m2[r][c] = INFINITY;
                    else br[r][c] = -1;
                }
        };
        reset();
        const unsigned cbase = (unsigned)__cvta_generic_to_shared(Hp + pl * kPlane + i0 * kQHP + j);
        auto in_out = [&](int r, int c) {
            const int py = py0 + 2 * (i0 + r) + c, px = px0 + 2 * j + pl;
            return py >= a.oy0 && py < a.oy1 && px >= a.ox0 && px < a.ox1;
        };
        auto key_off = [&](int r, int c) {
            const int py = py0 + 2 * (i0 + r) + c, px = px0 + 2 * j + pl;
            check_key(a, py, px);
            return (int64_t)(py - a.oy0) * a.key_pitch + (px - a.ox0);
        };
        // exact merge of (e, n, rank) with the mean key floor(e * 2^13 / n)
        auto merge_mean = [&](int r, int c, float e, float n, int rank) {
            if (rank < 0 || n < (float)a.min_support || !in_out(r, c)) return;
            const unsigned long long hi = (unsigned long long)floor((double)e * 8192.0 / (double)n);
            atomicMin(a.keys_p[ref_slot(a)] + key_off(r, c), (hi << 32) | (unsigned)rank);
        };
        // float merge: keyed winner / second in the mean domain (phase 1 divides by npx)
        auto merge_fk = [&](int r, int c, float npx, const bool phase1) {
            if constexpr (FK) {
                if (!(be[r][c] < kAdmissibleMax) || !in_out(r, c)) return;
                if (phase1 && npx < (float)a.min_support) return;
                unsigned v1 = fkey_val(be[r][c]), v2 = fkey_val2(m2[r][c]);
                if (phase1) {
                    v1 = __float_as_uint(__fdiv_rn(__uint_as_float(v1), npx));
                    if (v2 != 0xffffffffu) v2 = __float_as_uint(__fdiv_rn(__uint_as_float(v2), npx));
                }
                const int64_t o = key_off(r, c);
                merge_f32(a.keys_p[ref_slot(a)] + o, a.s2_p[ref_slot(a)] + o, v1,
                          clist[__float_as_uint(be[r][c]) & kKeyBits] >> 16, v2);
            }
        };
        // Phase-1 entry (or the npx entry when last): E for the 28 outputs from the 18 H rows.
        auto consume = [&](int e, const int s, const bool last) {
            const int rank = last ? 0 : clist[e] >> 16;
            nb_sync(1 + s, kNT);                                     // FULL[s]
            const unsigned cs = cbase + (unsigned)s * kStageBytes;
            f2_t x[kQSeg + 4];
#pragma unroll
            for (int t = 0; t < kQSeg + 4; ++t) x[t] = ld_shared_f2(cs + 8 * t * kQHP);   // (X0, X1) of H row i0+t
            nb_arrive(5 + s, kNT);                                   // EMPTY[s]
            // Rolling pairwise vertical boxes: pp(t) = X(t) + X(t+1), V(i) = pp(i) + pp(i+2);
            // E(2i) = V0(i) + V1(i), E(2i+1) = V1(i) + V0(i+1) (block rows i0 + i).
            f2_t pp0 = f2add(x[0], x[1]), pp1 = f2add(x[1], x[2]), pp2 = f2add(x[2], x[3]);
            f2_t pp3 = f2add(x[3], x[4]);
            f2_t vcur = f2add(pp0, pp2);
#pragma unroll
            for (int r = 0; r < kQSeg; ++r) {
                const f2_t vnext = f2add(pp1, pp3);                   // V(r + 1)
                const float ev[2] = {__fadd_rn(f2lo(vcur), f2hi(vcur)),       // E(2i,   2j + pl)
                                     __fadd_rn(f2hi(vcur), f2lo(vnext))};     // E(2i+1, 2j + pl)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    if constexpr (FK) {
                        if (last) merge_fk(r, c, ev[c], true);               // ev = npx(p)
                        else fbest(be[r][c], m2[r][c], fkey(ev[c], (unsigned)e));
                    } else {
                        if (last) merge_mean(r, c, be[r][c], ev[c], br[r][c]);   // ev = npx(p)
                        else if (ev[c] < be[r][c]) { be[r][c] = ev[c]; br[r][c] = rank; }
                    }
                }
                vcur = vnext;
                pp0 = pp1;
                pp1 = pp2;
                pp2 = pp3;
                if (r + 5 < kQSeg + 4) pp3 = f2add(x[r + 4], x[r + 5]);
            }
        };
        for (int k = 0; k < nA; k += 2) {
            consume(k, 0, false);
            if (k + 1 < nA) consume(k + 1, 1, false);
        }
        {
            if (nA > 0) {
                if (nA & 1) consume(nA, 1, true);
                else consume(nA, 0, true);
            }
            if constexpr (Q2) {
                // Phase 2: exact (uint8): (best e, its n, rank), means compared by cross-multiplication
                // (e * n < 2^24); float: keyed approximate means e * rcp(n) and the second (certified).
                float bn[FK ? 1 : kQSeg][2];
                reset();
                if constexpr (!FK) {
#pragma unroll
                    for (int r = 0; r < kQSeg; ++r)
#pragma unroll
                        for (int c = 0; c < 2; ++c) bn[r][c] = 1.f;
                }
                const float ms = (float)a.min_support;
                auto consume2 = [&](int ci, const int s) {
                    const int rank = clist[ci] >> 16;
                    nb_sync(1 + s, kNT);                                 // FULL[s]
                    const unsigned cs = cbase + (unsigned)s * kStageBytes, ns = cs + 2u * kPlane * 8u;
                    // Rows streamed (5-row windows of both planes) to keep the 84-register state.
                    f2_t x0 = ld_shared_f2(cs), x1 = ld_shared_f2(cs + 8 * kQHP), x2 = ld_shared_f2(cs + 16 * kQHP);
                    f2_t x3 = ld_shared_f2(cs + 24 * kQHP), xl = ld_shared_f2(cs + 32 * kQHP);
                    f2_t y0 = ld_shared_f2(ns), y1 = ld_shared_f2(ns + 8 * kQHP), y2 = ld_shared_f2(ns + 16 * kQHP);
                    f2_t y3 = ld_shared_f2(ns + 24 * kQHP), yl = ld_shared_f2(ns + 32 * kQHP);
                    f2_t pp0 = f2add(x0, x1), pp1 = f2add(x1, x2), pp2 = f2add(x2, x3), pp3 = f2add(x3, xl);
                    f2_t qq0 = f2add(y0, y1), qq1 = f2add(y1, y2), qq2 = f2add(y2, y3), qq3 = f2add(y3, yl);
                    f2_t vcur = f2add(pp0, pp2), ncur = f2add(qq0, qq2);
#pragma unroll
                    for (int r = 0; r < kQSeg; ++r) {
                        const f2_t vnext = f2add(pp1, pp3), nnext = f2add(qq1, qq3);
                        const float ev[2] = {__fadd_rn(f2lo(vcur), f2hi(vcur)), __fadd_rn(f2hi(vcur), f2lo(vnext))};
                        const float nv[2] = {__fadd_rn(f2lo(ncur), f2hi(ncur)), __fadd_rn(f2hi(ncur), f2lo(nnext))};
#pragma unroll
                        for (int c = 0; c < 2; ++c) {
                            if constexpr (FK) {
                                const float A = nv[c] >= ms ? __fmul_rn(ev[c], rcp_approx(nv[c])) : kInadmissible;
                                fbest(be[r][c], m2[r][c], fkey(A, (unsigned)ci));
                            } else if (nv[c] >= ms && __fmul_rn(ev[c], bn[r][c]) < __fmul_rn(be[r][c], nv[c])) {
                                be[r][c] = ev[c];
                                bn[r][c] = nv[c];
                                br[r][c] = rank;
                            }
                        }
                        vcur = vnext;
                        ncur = nnext;
                        pp0 = pp1;
                        pp1 = pp2;
                        pp2 = pp3;
                        qq0 = qq1;
                        qq1 = qq2;
                        qq2 = qq3;
                        if (r + 5 < kQSeg + 4) {
                            const f2_t xn = ld_shared_f2(cs + 8 * (r + 5) * kQHP), yn = ld_shared_f2(ns + 8 * (r + 5) * kQHP);
                            pp3 = f2add(xl, xn);
                            qq3 = f2add(yl, yn);
                            xl = xn;
                            yl = yn;
                            if (r + 5 == kQSeg + 3) nb_arrive(5 + s, kNT);   // EMPTY[s]: last rows read
                        }
                    }
                };
                // RUNS: 1 / n of the current support run per output (negative: n < min_support).
                float rn[RUNS ? kQSeg : 1][2];
                auto consume2r = [&](int ci, const int s) {
                    const int *skey = nsel + 8;
                    const bool rstart = ci == a0 || skey[ci - a0] != skey[ci - a0 - 1];
                    nb_sync(1 + s, kNT);                                 // FULL[s]
                    const unsigned cs = cbase + (unsigned)s * kStageBytes, ns = cs + 2u * kPlane * 8u;
                    if (rstart) {   // the run's supports: vertical boxes of the support planes
                        f2_t y0 = ld_shared_f2(ns), y1 = ld_shared_f2(ns + 8 * kQHP), y2 = ld_shared_f2(ns + 16 * kQHP);
                        f2_t y3 = ld_shared_f2(ns + 24 * kQHP), yl = ld_shared_f2(ns + 32 * kQHP);
                        f2_t qq0 = f2add(y0, y1), qq1 = f2add(y1, y2), qq2 = f2add(y2, y3), qq3 = f2add(y3, yl);
                        f2_t ncur = f2add(qq0, qq2);
#pragma unroll
                        for (int r = 0; r < kQSeg; ++r) {
                            const f2_t nnext = f2add(qq1, qq3);
                            const float nv[2] = {__fadd_rn(f2lo(ncur), f2hi(ncur)), __fadd_rn(f2hi(ncur), f2lo(nnext))};
#pragma unroll
                            for (int c = 0; c < 2; ++c) rn[r][c] = nv[c] >= ms ? rcp_approx(nv[c]) : -1.f;
                            ncur = nnext;
                            qq0 = qq1;
                            qq1 = qq2;
                            qq2 = qq3;
                            if (r + 5 < kQSeg + 4) {
                                const f2_t yn = ld_shared_f2(ns + 8 * (r + 5) * kQHP);
                                qq3 = f2add(yl, yn);
                                yl = yn;
                            }
                        }
                    }
                    f2_t x0 = ld_shared_f2(cs), x1 = ld_shared_f2(cs + 8 * kQHP), x2 = ld_shared_f2(cs + 16 * kQHP);
                    f2_t x3 = ld_shared_f2(cs + 24 * kQHP), xl = ld_shared_f2(cs + 32 * kQHP);
                    f2_t pp0 = f2add(x0, x1), pp1 = f2add(x1, x2), pp2 = f2add(x2, x3), pp3 = f2add(x3, xl);
                    f2_t vcur = f2add(pp0, pp2);
#pragma unroll
                    for (int r = 0; r < kQSeg; ++r) {
                        const f2_t vnext = f2add(pp1, pp3);
                        const float ev[2] = {__fadd_rn(f2lo(vcur), f2hi(vcur)), __fadd_rn(f2hi(vcur), f2lo(vnext))};
#pragma unroll
                        for (int c = 0; c < 2; ++c)
                            ubest(be[r][c], m2[r][c], __float_as_uint(fkey(__fmul_rn(ev[c], rn[r][c]), (unsigned)ci)));
                        vcur = vnext;
                        pp0 = pp1;
                        pp1 = pp2;
                        pp2 = pp3;
                        if (r + 5 < kQSeg + 4) {
                            const f2_t xn = ld_shared_f2(cs + 8 * (r + 5) * kQHP);
                            pp3 = f2add(xl, xn);
                            xl = xn;
                            if (r + 5 == kQSeg + 3) nb_arrive(5 + s, kNT);   // EMPTY[s]: last rows read
                        }
                    }
                };
                auto c2 = [&](int ci, const int st) {
                    if constexpr (RUNS) consume2r(ci, st);
                    else consume2(ci, st);
                };
                if ((e1 & 1) == 0) {
                    for (int i = 0; i < nB; i += 2) {
                        c2(a0 + i, 0);
                        if (i + 1 < nB) c2(a0 + i + 1, 1);
                    }
                } else {
                    for (int i = 0; i < nB; i += 2) {
                        c2(a0 + i, 1);
                        if (i + 1 < nB) c2(a0 + i + 1, 0);
                    }
                }
#pragma unroll
                for (int r = 0; r < kQSeg; ++r)
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        if constexpr (FK) merge_fk(r, c, 0.f, false);
                        else merge_mean(r, c, be[r][c], bn[r][c], br[r][c]);
                    }
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Integer interior body (uint8 SAD, K = 8, interior tiles): DESIGN.md "K1i integer quad body".
//
// The same block-grid decomposition as quad_body's interior path, in exact integer arithmetic with
// two 16-bit lanes per 32-bit register (the (C0, C1) / (D0, D1) series pairs).  Every term is
// |c - r| <= 255 scaled by 8; every lane sum is <= 8 * 25 * 255 = 51000 < 2^16, so lane arithmetic
// never carries and sliding-window sums (add the entering, subtract the leaving value: one IADD3)
// are exact.  Producers: |c - r| (VABSDIFF), the dy lane by IMAD with (8 or 8 << 16), the dx split by
// a second IMAD and an IADD3, sliding 4-wide H sums (one IADD3 per column and series), one STS per
// column and series.  Consumers: sliding V sums, the output pair (E(2i), E(2i+1)) =
// V(i) + (hi V(i), lo V(i+1)) (PRMT + IADD3, which also adds the candidate's position in its group of
// eight, so each lane holds 8 E + pos), a packed 16-bit min per output pair (ties inside a group go
// to the lower position = lower rank); every eight candidates the group minima merge into the running
// best when their E is strictly smaller (earlier groups, i.e. lower ranks, keep ties), with the
// group index alongside.  Decoded key: E and rank = clist[8 g + pos] (R7 order).
// ---------------------------------------------------------------------------
constexpr int kIPitch = kQHC + 1;                        // int plane row pitch (words): rows -> distinct banks
constexpr int kIPlane = kQHR * kIPitch;                   // words per plane
constexpr unsigned kIStageBytes = 2u * kIPlane * 4u;      // C plane + D plane

// BRD (border tiles, round 2): the same body runs phase 1 of a uint8 SAD border tile -- its clip-free
// candidates (tile_clip_free: n(p, v) = npx(p) for all of them) -- with bounds-checked staging (0
// outside the frame / buffer), weight 0 for blocks outside, one extra ring entry with t = 1 per
// measured in-frame block (its sums are 8 npx), and the border body's mean key floor(e 2^13 / npx);
// the caller then runs the border body's phase 2 on the other candidates.  Returns after the
// setmaxnreg roles are restored (128 registers everywhere), so a body may follow.
template <bool BRD>
__device__ __forceinline__ void quad_interior_int(const BoxArgs &a, float *smem, int chunk, int px0, int py0) {
    const int alo = chunk_alo(a.S, chunk);
    const int ahi = chunk_ahi(a.S, chunk);
    const int nrow_b = kQWinRows + (ahi - alo);
    const int ncol_b = kQWinCols + 2 * a.S;
    const int bpitch = quad_pitch(ncol_b);
    const int bplane = quad_plane(nrow_b, ncol_b);
    int *Bw = reinterpret_cast<int *>(smem);
    unsigned *Hi = reinterpret_cast<unsigned *>(smem + 2 * bplane);   // [kQStages][2 planes][kQHR][kIPitch]
    int *clist = reinterpret_cast<int *>(Hi + kQStages * 2 * kIPlane);
    int *ncnt = clist + kChunkRows * (2 * a.S + 1);
    const int by0 = py0 - 4 + alo, bx0 = px0 - 4 - a.S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    {
        // The window as 32-bit integers, split by row parity like the float body (interior tiles read
        // only in-frame, in-buffer pixels; border tiles store 0 outside).
        const uint8_t *rp = a.ref_p[ref_slot(a)];
        for (int r = warp; r < nrow_b; r += kNT / 32) {
            const int y = by0 + r;
            int *dst = Bw + (r & 1) * bplane + (r >> 1) * bpitch;
            const uint8_t *src = rp + (int64_t)(y - a.buf_y0) * a.ref.pitch;
            if (BRD) {
                const bool row_in = y >= 0 && y < a.H && y >= a.buf_y0 && y < a.buf_y0 + a.buf_rows;
                for (int c = lane; c < ncol_b; c += 32) {
                    const int x = bx0 + c;
                    dst[c] = (row_in && x >= 0 && x < a.W) ? src[x] : 0;
                }
            } else {
                for (int c = lane; c < ncol_b; c += 32) dst[c] = src[bx0 + c];
            }
        }
    }
    const int k0g = a.chunk_off[chunk], nkc = a.chunk_off[chunk + 1] - k0g;
    if (!BRD) {
        for (int i = threadIdx.x; i < nkc; i += kNT) clist[i] = __ldg(a.chunked + k0g + i);
    } else if (warp == 0) {
        // the tile's clip-free candidates, in rank order
        int n = 0;
        for (int base = 0; base < nkc; base += 32) {
            const int i = base + lane;
            int pk = 0;
            bool keep = false;
            if (i < nkc) {
                pk = __ldg(a.chunked + k0g + i);
                keep = tile_clip_free<8>(a, px0, py0, (int)(int8_t)(pk & 0xff), (int)(int8_t)((pk >> 8) & 0xff));
            }
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) clist[n + __popc(m & ((1u << lane) - 1u))] = pk;
            n += __popc(m);
        }
        if (lane == 0) ncnt[0] = n;
    }
    __syncthreads();
    const int nA = BRD ? ncnt[0] : nkc;
    if (nA <= 0) return;                                              // uniform
    const int NE = nA + (BRD ? 1 : 0);                                // entries (+ the npx entry)
    if (warp < 4) {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 152;" ::: "memory");
        const int hr = lane, bi = hr - 2;
        const int pair = warp >> 1, half = warp & 1;
        int cv[kQGI], ad[kQGI];
        unsigned W[kQGI], Wd[kQGI];
#pragma unroll
        for (int kk = 0; kk < kQGI; ++kk) {
            const int bk = kQRunI * half - 2 + kk;
            const int y = py0 + 2 * bi, x = px0 + 2 * bk;
            // blocks outside the frame / the buffer: weight 0 (interior tiles: only a band's ragged
            // last tile has them, below the rows the merge keeps)
            const bool inside = y + 1 < a.H && y + 1 < a.buf_y0 + a.buf_rows &&
                                (!BRD || (y >= 0 && y >= a.buf_y0 && x >= 0 && x + 1 < a.W));
            const int64_t r = (int64_t)(y - a.buf_y0);
            const uint8_t *m0 = a.mask.p + r * a.mask.pitch + x;
            const int q = !inside ? 0 : m0[1] ? 1 : m0[a.mask.pitch] ? 2 : m0[a.mask.pitch + 1] ? 3 : 0;
            const int dy = q >> 1, dx = q & 1;
            cv[kk] = inside ? a.cur.p[(r + dy) * a.cur.pitch + x + dx] : 0;
            W[kk] = inside ? (dy ? 8u << 16 : 8u) : 0u;            // lane dy, scaled by 8
            Wd[kk] = dx ? W[kk] : 0u;                               // the dx = 1 part
            ad[kk] = 4 * (dy * bplane + (bi + 2) * bpitch + (2 * bk + dx + 4 + a.S));
        }
        const unsigned hbase = (unsigned)__cvta_generic_to_shared(Hi + hr * kIPitch + kQRunI * half);
        auto run = [&](auto Pc) {
            constexpr int P = decltype(Pc)::value;
            const unsigned hs = hbase + (unsigned)P * kIStageBytes;
            int rv[kQGI];
            for (int k = P; k < NE; k += 2) {
                const bool npx_entry = BRD && k == nA;                  // t = 1 per measured block
                if (!npx_entry) {
                    const int pk = clist[k];
                    const char *bwc = reinterpret_cast<const char *>(
                        Bw + (((int)(int8_t)(pk & 0xff) - alo) >> 1) * bpitch + (int)(int8_t)((pk >> 8) & 0xff));
#pragma unroll
                    for (int kk = 0; kk < kQGI; ++kk) {
                        QS_DCHECK(bwc + ad[kk] >= reinterpret_cast<const char *>(Bw) &&
                                  bwc + ad[kk] + 4 <= reinterpret_cast<const char *>(Bw + 2 * bplane));
                        rv[kk] = *reinterpret_cast<const int *>(bwc + ad[kk]);
                    }
                }
                if (k >= 2) nb_sync_i<5 + P, kQBarI>();                 // EMPTY[P]
                unsigned u[kQGI], g[kQGI], m[kQGI - 1], hc = 0, hd = 0;
#pragma unroll
                for (int kk = 0; kk < kQGI; ++kk) {
                    const unsigned t = npx_entry ? 1u : __usad((unsigned)cv[kk], (unsigned)rv[kk], 0u);   // |c - r|
                    u[kk] = t * W[kk];
                    g[kk] = t * Wd[kk];
                    if (kk > 0) m[kk - 1] = g[kk - 1] + (u[kk] - g[kk]);   // D(k-1) = G_dx1(k-1) + G_dx0(k)
                    if (kk == 3) hc = u[0] + u[1] + u[2] + u[3];
                    else if (kk > 3 && kk - 3 < kQRunI) hc = hc + u[kk] - u[kk - 4];
                    if (kk >= 3 && kk - 3 < kQRunI)
                        asm volatile("st.shared.u32 [%0], %1;" ::"r"(hs + 4u * (kk - 3)), "r"(hc) : "memory");
                    if (kk == 4) hd = m[0] + m[1] + m[2] + m[3];
                    else if (kk > 4 && kk - 4 < kQRunI) hd = hd + m[kk - 1] - m[kk - 5];
                    if (kk >= 4 && kk - 4 < kQRunI)
                        asm volatile("st.shared.u32 [%0], %1;" ::"r"(hs + 4u * (kIPlane + kk - 4)), "r"(hd) : "memory");
                }
                nb_arrive_i<1 + P, kQBarI>();                           // FULL[P]
            }
            if (P < NE) nb_sync_i<5 + P, kQBarI>();                    // drain
        };
        if (pair == 0) run(std::integral_constant<int, 0>{});
        else run(std::integral_constant<int, 1>{});
        if (BRD) asm volatile("setmaxnreg.dec.sync.aligned.u32 128;" ::: "memory");
    } else {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 104;" ::: "memory");
        const int j = lane;
        const int cw = warp - 4, pl = cw & 1, i0 = kQSeg * (cw >> 1);
        unsigned gmin[kQSeg], best[kQSeg], bestg[kQSeg];
#pragma unroll
        for (int r = 0; r < kQSeg; ++r) { gmin[r] = 0xffffffffu; best[r] = 0xffffffffu; bestg[r] = 0u; }
        const unsigned cbase = (unsigned)__cvta_generic_to_shared(Hi + pl * kIPlane + i0 * kIPitch + j);
        // one ring entry: E pairs (8 E + pos) per output row pair, handed to f (r, e)
        auto entry = [&](auto Pc, unsigned pos2, auto f) {
            constexpr int P = decltype(Pc)::value;
            nb_sync_i<1 + P, kQBarI>();                                 // FULL[P]
            const unsigned cs = cbase + (unsigned)P * kIStageBytes;
            unsigned x[kQSeg + 4];
#pragma unroll
            for (int t = 0; t < kQSeg + 4; ++t)
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(x[t]) : "r"(cs + 4u * t * kIPitch) : "memory");
            nb_arrive_i<5 + P, kQBarI>();                               // EMPTY[P]
            unsigned v = x[0] + x[1] + x[2] + x[3];
#pragma unroll
            for (int r = 0; r < kQSeg; ++r) {
                const unsigned vn = v + x[r + 4] - x[r];                // V(r + 1)
                f(r, v + __byte_perm(v, vn, 0x5432) + pos2);            // (8 E(2i) + pos, 8 E(2i+1) + pos)
                v = vn;
            }
        };
        auto consume = [&](int k, auto Pc) {
            entry(Pc, (unsigned)(k & 7) * 0x10001u, [&](int r, unsigned e) { gmin[r] = __vminu2(gmin[r], e); });
            if ((k & 7) == 7 || k == nA - 1) {
                // group end: a lane takes the group's minimum iff its E is strictly smaller (the
                // positions inside a group are not comparable across groups): 8 E_g + 7 < 8 E_best.
                const unsigned g2 = (unsigned)(k >> 3) * 0x10001u;
#pragma unroll
                for (int r = 0; r < kQSeg; ++r) {
                    const unsigned lt = __vcmpltu2(gmin[r] | 0x00070007u, best[r] & 0xfff8fff8u);
                    best[r] = (best[r] & ~lt) | (gmin[r] & lt);
                    bestg[r] = (bestg[r] & ~lt) | (g2 & lt);
                    gmin[r] = 0xffffffffu;
                }
            }
        };
        for (int k = 0; k < nA; k += 2) {
            consume(k, std::integral_constant<int, 0>{});
            if (k + 1 < nA) consume(k + 1, std::integral_constant<int, 1>{});
        }
        if (BRD) {
            // the npx entry: gmin[r] <- (8 npx(2i), 8 npx(2i+1)) of the outputs
            auto npx_f = [&](int r, unsigned e) { gmin[r] = e; };
            if (nA & 1) entry(std::integral_constant<int, 1>{}, 0u, npx_f);
            else entry(std::integral_constant<int, 0>{}, 0u, npx_f);
        }
#pragma unroll
        for (int r = 0; r < kQSeg; ++r)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int py = py0 + 2 * (i0 + r) + c, px = px0 + 2 * j + pl;
                const unsigned val = c ? best[r] >> 16 : best[r] & 0xffffu;
                if (val == 0xffffu || py < a.oy0 || py >= a.oy1 || px >= a.ox1) continue;
                const unsigned gi = c ? bestg[r] >> 16 : bestg[r] & 0xffffu;
                const int rank = clist[8 * gi + (val & 7u)] >> 16;
                unsigned long long hi;
                if (BRD) {
                    const unsigned npx = (c ? gmin[r] >> 16 : gmin[r] & 0xffffu) >> 3;
                    if ((int)npx < a.min_support || px < a.ox0) continue;
                    // the border body's mean key (merge_mean): floor(e * 2^13 / n)
                    hi = (unsigned long long)floor((double)(val >> 3) * 8192.0 / (double)npx);
                } else {
                    hi = __float_as_uint((float)(val >> 3));
                }
                check_key(a, py, px);
                atomicMin(a.keys_p[ref_slot(a)] + (int64_t)(py - a.oy0) * a.key_pitch + (px - a.ox0),
                          (hi << 32) | (unsigned)rank);
            }
        if (BRD) asm volatile("setmaxnreg.inc.sync.aligned.u32 128;" ::: "memory");
    }
}

// TILES (K = 8 forward launches): 0 = every tile; 1 = interior tiles only; 2 = border tiles only (a
// separate kernel so each class gets its own code generation; the interior launch follows the border
// launch as a programmatic dependent launch, launch_t).
template <bool ON>
struct PdlWaitAtExit {   // the interior grid of a split launch completes only after the border grid
    __device__ ~PdlWaitAtExit() {
        if constexpr (ON) asm volatile("griddepcontrol.wait;" ::: "memory");
    }
};

template <int K, bool EXACT, bool SSD, bool REV, int TILES = 0>
__global__ void __launch_bounds__(kNT, 2) box_kernel(const __grid_constant__ BoxArgs a) {
    [[maybe_unused]] PdlWaitAtExit<TILES == 1> pdl_guard;
    extern __shared__ __align__(1024) float smem[];   // TMA box destinations need 128-byte alignment
    const int unit = blockIdx.x / a.n_ref;   // the slots of one unit run side by side
    const int chunk = unit % a.n_chunks;
    const int tile = unit / a.n_chunks;
    int txi, tyi;
    if (TILES != 0 && a.rect_r0 < 0) {   // split launch over the whole grid (each class skips the other)
        txi = tile % a.tiles_x;
        const int q = tile / a.tiles_x, T = a.tiles_y;
        tyi = T < 3 ? q : (q == 0 ? 0 : q == 1 ? T - 1 : q == 2 ? T - 2 : q - 2);
    } else if constexpr (TILES == 1) {
        // interior launch: the tiles of the interior rectangle [r0, r1) x [c0, c1)
        const int nc = a.rect_c1 - a.rect_c0;
        tyi = a.rect_r0 + tile / nc;
        txi = a.rect_c0 + tile % nc;
    } else if constexpr (TILES == 2) {
        // border launch: the rows above and below the rectangle, then the columns left and right of it
        const int tx = a.tiles_x, top = a.rect_r0 * tx, bot = (a.tiles_y - a.rect_r1) * tx;
        if (tile < top) {
            tyi = tile / tx;
            txi = tile % tx;
        } else if (tile < top + bot) {
            tyi = a.rect_r1 + (tile - top) / tx;
            txi = (tile - top) % tx;
        } else {
            const int w = a.rect_c0 + (tx - a.rect_c1), m = tile - top - bot;
            tyi = a.rect_r0 + m / w;
            const int k = m % w;
            txi = k < a.rect_c0 ? k : a.rect_c1 + (k - a.rect_c0);
        }
    } else {
        txi = tile % a.tiles_x;
        // Tile rows in the order first, last, second-to-last, then the rest: the (slower) frame-border
        // rows are scheduled in the first waves, not in the tail.
        const int q = tile / a.tiles_x, T = a.tiles_y;
        tyi = T < 3 ? q : (q == 0 ? 0 : q == 1 ? T - 1 : q == 2 ? T - 2 : q - 2);
    }
    // tile_off (forward K = 8 launches): the tile grid starts tile_off rows above oy0, placed by the
    // host so that the fewest tile rows reach outside the frame (border tiles cost ~1.7x).
    const int px0 = a.ox0 + txi * kTX, py0 = a.oy0 - a.tile_off + tyi * kTY;
    constexpr int KL = K / 2, KR = K - 1 - K / 2;
    bool interior = !REV && (py0 - KL - a.S >= 0) && (py0 + kTY - 1 + KR + a.S <= a.H - 1) &&
                    (px0 - KL - a.S >= 0) && (px0 + kTX - 1 + KR + a.S <= a.W - 1);
    if constexpr (REV) {
        box_body<K, EXACT, true, SSD, true>(a, smem, chunk, px0, py0);
    } else {
        if constexpr (K == 8) {
            // Rows: only the outputs the merge keeps (rows < oy1) must have every window in the
            // frame and the buffer; rows beyond (a band's ragged last tile) read NaN windows and
            // are never merged.  Columns: the whole tile (ox1 is the frame width).
            const int ylast = min(py0 + kTY, a.oy1) - 1;
            const bool geom = (py0 - 4 - a.S >= 0) && (ylast + 3 + a.S <= a.H - 1) &&
                              (px0 - 4 - a.S >= 0) && (px0 + kQWinCols - 5 + a.S <= a.W - 1) &&
                              (py0 - 4 - a.S >= a.buf_y0) && (ylast + 3 + a.S < a.buf_y0 + a.buf_rows);
            if constexpr (TILES == 2) asm volatile("griddepcontrol.launch_dependents;");
            // the host's rectangle (launch_t) mirrors geom: interior launch = geom tiles, border = the rest
            if constexpr (TILES == 1) {
                if (a.rect_r0 < 0 && !geom) return;
                QS_DCHECK(geom);
            }
            if constexpr (TILES == 2) {
                if (a.rect_r0 < 0 && geom) return;
                QS_DCHECK(!geom);
            }
            // Quarter-sampling body.  Interior: every pixel it touches, for every candidate, lies in the
            // frame and in the caller's buffer.  Border: clip-free candidates here, the rest below.
            if (a.S >= 4 && quad_mask_ok(a, px0, py0)) {
#ifdef QS_EXP_SKIP   // measurement builds only (tools/build_exp.sh): 1 = skip border tiles, 2 = skip interior
                if ((QS_EXP_SKIP == 1 && !geom) || (QS_EXP_SKIP == 2 && geom)) return;
#endif
                if (TILES != 2 && geom) {
                    if constexpr (EXACT && !SSD) {
                        if (a.int_body) {   // uint8 SAD: the integer body
                            quad_interior_int<false>(a, smem, chunk, px0, py0);
                            return;
                        }
                    }
                    quad_body<SSD, EXACT, false>(a, smem, chunk, px0, py0);
                    return;
                }
                if constexpr (TILES == 1) return;   // unreachable: interior launch, geom tiles only
                if constexpr (EXACT && !SSD) {
                    if (a.int_body) {
                        // uint8 SAD border tile: phase 1 (clip-free candidates) in the integer body,
                        // then the border body's phase 2 (round 2)
                        quad_interior_int<true>(a, smem, chunk, px0, py0);
                        __syncthreads();
                        quad_body<SSD, EXACT, true>(a, smem, chunk, px0, py0, true);
                        return;
                    }
                }
                quad_body<SSD, EXACT, true, TILES == 2 && !EXACT>(a, smem, chunk, px0, py0);
                if constexpr (EXACT && SSD) {   // quad phase 2 unavailable: the rest in the generic body
                    __syncthreads();
                    box_body<K, EXACT, true, SSD, false>(a, smem, chunk, px0, py0, true);
                }
                return;
            }
        }
        if (interior) box_body<K, EXACT, false, SSD, false>(a, smem, chunk, px0, py0);
        else box_body<K, EXACT, true, SSD, false>(a, smem, chunk, px0, py0);
    }
}

template <int K, bool EXACT, bool SSD, bool REV, int TILES>
cudaError_t launch_t1(const BoxArgs &a, cudaStream_t s, bool pdl, long long tiles) {
    using G = BoxGeom<K>;
    const int nrow_b = G::HR + kChunkSpan - 1;
    const int bpitch = (kTX + K - 1 + 2 * a.S) | 1;
    size_t smem = sizeof(float) * ((size_t)((nrow_b * bpitch + 3) & ~3) + 4 * (size_t)G::HR * kTXP) +
                  sizeof(int) * kChunkRows * (2 * a.S + 1);
    if (K == 8 && !REV) {
        const int qrows = kQWinRows + kChunkSpan - 1, qcols = kQWinCols + 2 * a.S;
        const size_t plane = a.tma ? (size_t)((a.tma_rows * a.tma_cols + 31) & ~31) : (size_t)quad_plane(qrows, qcols);
        const size_t qs = sizeof(float) * 2 * plane +
                          sizeof(f2_t) * kQStages * kQPlanes * kQHR * kQHP + sizeof(int) * (kChunkRows * (2 * a.S + 1) + 8) +
                          (TILES == 2 ? sizeof(int) * 2 * kChunkRows * (2 * a.S + 1) : 0);   // RUNS: keys + sort
        smem = smem > qs ? smem : qs;
    }
    auto fn = box_kernel<K, EXACT, SSD, REV, TILES>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long units = tiles * a.n_chunks * a.n_ref;
    if (units <= 0) return cudaSuccess;
    if (!pdl) {
        fn<<<(unsigned)units, kNT, smem, s>>>(a);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)units);
    cfg.blockDim = dim3(kNT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fn, a);
}

// Interior rectangle of a K = 8 forward launch in tile coordinates: box_kernel's geom (every window
// of the tile's kept outputs, for every candidate, in the frame and the buffer) is a conjunction of a
// row condition and a column condition, each true on a contiguous range of tile rows / columns.
inline bool interior_rect(BoxArgs &a) {
    int r0 = -1, r1 = -1, c0 = -1, c1 = -1;
    for (int t = 0; t < a.tiles_y; ++t) {
        const int py0 = a.oy0 - a.tile_off + t * kTY, ylast = std::min(py0 + kTY, a.oy1) - 1;
        const bool ok = (py0 - 4 - a.S >= 0) && (ylast + 3 + a.S <= a.H - 1) && (py0 - 4 - a.S >= a.buf_y0) &&
                        (ylast + 3 + a.S < a.buf_y0 + a.buf_rows);
        if (ok && r0 < 0) r0 = t;
        if (ok) r1 = t + 1;
    }
    for (int t = 0; t < a.tiles_x; ++t) {
        const int px0 = a.ox0 + t * kTX;
        const bool ok = (px0 - 4 - a.S >= 0) && (px0 + kQWinCols - 5 + a.S <= a.W - 1);
        if (ok && c0 < 0) c0 = t;
        if (ok) c1 = t + 1;
    }
    if (r0 < 0 || c0 < 0) return false;
    a.rect_r0 = r0;
    a.rect_r1 = r1;
    a.rect_c0 = c0;
    a.rect_c1 = c1;
    return true;
}

template <int K, bool EXACT, bool SSD, bool REV>
cudaError_t launch_t(const BoxArgs &a0, cudaStream_t s) {
    const long long all = (long long)a0.tiles_x * a0.tiles_y;
    if constexpr (K == 8 && !REV && !EXACT) {
        // Float references: border tiles and interior tiles as two kernels, the
        // border one with phase 2 in runs of equal supports.  The interior grid is a programmatic
        // dependent launch: it starts filling SMs as the border grid's last wave drains (every border CTA
        // triggers at its start), and each interior CTA waits for the border grid's completion before it
        // exits, so the stream's next operation sees both grids complete.
        BoxArgs a = a0;
        if (a.split_tiles == 2) {   // whole grid twice, each class skipping the other's tiles
            a.rect_r0 = -1;
            cudaError_t e = launch_t1<K, EXACT, SSD, REV, 2>(a, s, false, all);
            if (e != cudaSuccess) return e;
            return launch_t1<K, EXACT, SSD, REV, 1>(a, s, true, all);
        }
        if (a.split_tiles && interior_rect(a)) {
            const long long inner = (long long)(a.rect_r1 - a.rect_r0) * (a.rect_c1 - a.rect_c0);
            if (inner < all) {
                cudaError_t e = launch_t1<K, EXACT, SSD, REV, 2>(a, s, false, all - inner);
                if (e != cudaSuccess) return e;
            }
            return launch_t1<K, EXACT, SSD, REV, 1>(a, s, inner < all, inner);
        }
    }
    return launch_t1<K, EXACT, SSD, REV, 0>(a0, s, false, all);
}

template <int K>
cudaError_t launch_k(const BoxArgs &a, bool ssd, bool rev, cudaStream_t s) {
    const bool exact = !a.ref_f32;
    if (rev) {
        if (exact) return ssd ? launch_t<K, true, true, true>(a, s) : launch_t<K, true, false, true>(a, s);
        return ssd ? launch_t<K, false, true, true>(a, s) : launch_t<K, false, false, true>(a, s);
    }
    if (exact) return ssd ? launch_t<K, true, true, false>(a, s) : launch_t<K, true, false, false>(a, s);
    return ssd ? launch_t<K, false, true, false>(a, s) : launch_t<K, false, false, false>(a, s);
}

}  // namespace
}  // namespace qs
