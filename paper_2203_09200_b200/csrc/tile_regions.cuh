// tile_regions.cuh -- shared-memory staging of a 16x16 entry tile's current-frame and
// reference regions, and the K = 8 reverse-cost worker used by FRMC / RMC
// (checks.cu: revgrid_tile_kernel) and by the fused pair epilogue (epilogue.cu).
//
// Reverse cost (R9, R23): for an entry p with vector v and
// delta, rc(p+v, -v+delta) = sum over o (row-major) of phi(ref(p+v+o) - cur(p+o+delta))
// where p+v+o and p+o+delta are in the frame and cur_mask(p+o+delta) = 1.  Both regions
// are staged as float with NaN marking "no term", so every excluded slot adds exactly +0
// and each cost is the oracle's row-major fp32 sum.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "qs_internal.cuh"

namespace qs {
namespace tile {

constexpr int kFT = 16;          // tile edge (entries)
constexpr int kFK = 8;           // template
constexpr int kFSeg = kFK + 14;  // current-row segment per FRMC item (22)

// Column of delta_x within an item's span (delta_x - dx0).
// PAT 0 = the paper's {-7,-3,-1,0,1,3,7}; PAT 1 = 7 consecutive values;
// PAT 2 / 3 = the two groups of the set extended by +-15:
// {-15,-7,-3,-1,0,1,3} (dx0 = -15) and {7, 15} (dx0 = 7; k >= 2 unused).
template <int PAT>
__device__ __forceinline__ constexpr int pat_j(int k) {
    return PAT == 0   ? (k == 0 ? 0 : k == 1 ? 4 : k == 2 ? 6 : k == 3 ? 7 : k == 4 ? 8 : k == 5 ? 10 : 14)
           : PAT == 2 ? (k == 0 ? 0 : k == 1 ? 8 : k == 2 ? 12 : k == 3 ? 14 : k == 4 ? 15 : k == 5 ? 16 : 18)
           : PAT == 3 ? (k == 1 ? 8 : 0)
                      : k;
}
// Current-row segment of an item: the template width plus the item's delta_x span (even).
template <int PAT>
__device__ __forceinline__ constexpr int seg_len() {
    return PAT == 2 ? kFK + 18 : PAT == 3 ? kFK + 8 : kFSeg;
}

// Packed fp32x2 subtraction (sm_100a FADD2) of (a0, a1) - (b0, b1), per-lane IEEE round-to-nearest.
__device__ __forceinline__ void sub2(float a0, float a1, float b0, float b1, float &d0, float &d1) {
    unsigned long long x, y, r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(y) : "f"(b0), "f"(b1));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(x), "l"(y));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(r));
}

struct Regions {
    int cy0, cx0, CR, CC, cpitch, mwords;   // current region: global row/col of element 0, sizes
    int ry0, rx0, RR, RC, rpitch;           // reference region
    float *Cs, *Rs;
    uint32_t *Mb;                           // mask bits of the current region rows
    int W, H;                               // frame
};

struct RegionSizes {
    int CR, CC, cpitch, mwords, RR, RC, rpitch;
    __host__ __device__ RegionSizes(int maxd, int S) {
        constexpr int KL = kFK / 2;
        (void)KL;
        CR = kFT + 2 * maxd + kFK - 1;
        CC = CR;
        // room for a 22-wide read past the region edge; pitch = 16 mod 32 words so the two
        // half-warps of an FRMC row (lanes on consecutive region rows) read disjoint bank halves
        cpitch = ((CC + 17 + 15) & ~31) + 16;
        if (cpitch < CC + 17) cpitch += 32;
        mwords = (CC + 16 + 31) / 32 + 1;
        RR = kFT + 2 * S + kFK - 1;
        RC = RR;
        rpitch = RC + 1;
    }
    __host__ __device__ size_t bytes() const {
        return sizeof(float) * ((size_t)CR * cpitch + (size_t)RR * rpitch) + sizeof(uint32_t) * (size_t)CR * mwords;
    }
};

__device__ __forceinline__ Regions layout(float *sm, int ty0, int tx0, int maxd, int S, int W, int H) {
    constexpr int KL = kFK / 2;
    RegionSizes z(maxd, S);
    Regions g;
    g.W = W;
    g.H = H;
    g.cy0 = ty0 - maxd - KL;
    g.cx0 = tx0 - maxd - KL;
    g.CR = z.CR; g.CC = z.CC; g.cpitch = z.cpitch; g.mwords = z.mwords;
    g.ry0 = ty0 - S - KL;
    g.rx0 = tx0 - S - KL;
    g.RR = z.RR; g.RC = z.RC; g.rpitch = z.rpitch;
    g.Cs = sm;
    g.Rs = g.Cs + g.CR * g.cpitch;
    g.Mb = reinterpret_cast<uint32_t *>(g.Rs + g.RR * g.rpitch);
    return g;
}

// Stage the current region (NaN outside the frame / the buffer window / unmeasured) and its mask
// bits.  One warp per region row, 32 columns per step: no index division, and the mask word of each
// 32 columns is the warp's ballot.  Ends with __syncthreads().
__device__ __forceinline__ void stage_cur(const Regions &g, const Plane &cur, const Plane &mask, int W, int H,
                                          int buf_y0, int buf_rows) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const float nan = __int_as_float(0x7fc00000);
    for (int r = warp; r < g.CR; r += nw) {
        const int gy = g.cy0 + r;
        const bool row_ok = gy >= 0 && gy < H && gy >= buf_y0 && gy < buf_y0 + buf_rows;
        const int64_t rr = gy - buf_y0;
        for (int w = 0; w < g.mwords; ++w) {
            const int c = 32 * w + lane, gx = g.cx0 + c;
            bool meas = false;
            float v = nan;
            if (row_ok && c < g.CC && gx >= 0 && gx < W && mask.p[rr * mask.pitch + gx]) {
                meas = true;
                v = (float)cur.p[rr * cur.pitch + gx];
            }
            if (c < g.cpitch) g.Cs[r * g.cpitch + c] = v;
            const unsigned word = __ballot_sync(0xffffffffu, meas);
            if (lane == 0) g.Mb[r * g.mwords + w] = word;
        }
    }
    __syncthreads();
}

// Narrow the reference region to the rows / columns the tile's vectors reach (round 2): entries at
// tile-local (ly, lx) with vector (a, b) read reference rows ty0 + ly + a - 4 .. + 3; lo_y / hi_y are
// the min / max of ly + a over the tile's valid entries (likewise columns).  The region keeps its
// base and maximum footprint (the mask bits follow it), only its origin, extent and pitch shrink.
__device__ __forceinline__ void narrow_ref(Regions &g, int ty0, int tx0, int lo_y, int hi_y, int lo_x, int hi_x) {
    constexpr int KL = kFK / 2;
    g.ry0 = ty0 + lo_y - KL;
    g.rx0 = tx0 + lo_x - KL;
    g.RR = hi_y - lo_y + kFK;
    g.RC = hi_x - lo_x + kFK;
    g.rpitch = g.RC + 1;
}

// Stage the reference region (NaN outside the frame / the buffer window).  Ends with __syncthreads().
template <bool F32>
__device__ __forceinline__ void stage_ref(const Regions &g, const Plane &ref, int W, int H, int buf_y0, int buf_rows) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const float nan = __int_as_float(0x7fc00000);
    for (int r = warp; r < g.RR; r += nw) {
        const int gy = g.ry0 + r;
        const bool row_ok = gy >= 0 && gy < H && gy >= buf_y0 && gy < buf_y0 + buf_rows;
        const int64_t rr = gy - buf_y0;
        for (int c = lane; c < g.rpitch; c += 32) {
            const int gx = g.rx0 + c;
            float v = nan;
            if (row_ok && c < g.RC && gx >= 0 && gx < W)
                v = F32 ? reinterpret_cast<const float *>(ref.p + rr * ref.pitch)[gx] : (float)ref.p[rr * ref.pitch + gx];
            g.Rs[r * g.rpitch + c] = v;
        }
    }
    __syncthreads();
}

// Stage both regions (NaN outside the frame / the buffer window / unmeasured) and the
// current mask bits.  One warp per region row, 32 columns per step: no index division, and the
// mask word of each 32 columns is the warp's ballot.  Ends with __syncthreads().
template <bool F32>
__device__ __forceinline__ void stage(const Regions &g, const Plane &cur, const Plane &mask, const Plane &ref, int W,
                                      int H, int buf_y0, int buf_rows) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const float nan = __int_as_float(0x7fc00000);
    for (int r = warp; r < g.CR; r += nw) {
        const int gy = g.cy0 + r;
        const bool row_ok = gy >= 0 && gy < H && gy >= buf_y0 && gy < buf_y0 + buf_rows;
        const int64_t rr = gy - buf_y0;
        for (int w = 0; w < g.mwords; ++w) {
            const int c = 32 * w + lane, gx = g.cx0 + c;
            bool meas = false;
            float v = nan;
            if (row_ok && c < g.CC && gx >= 0 && gx < W && mask.p[rr * mask.pitch + gx]) {
                meas = true;
                v = (float)cur.p[rr * cur.pitch + gx];
            }
            if (c < g.cpitch) g.Cs[r * g.cpitch + c] = v;
            const unsigned word = __ballot_sync(0xffffffffu, meas);
            if (lane == 0) g.Mb[r * g.mwords + w] = word;
        }
    }
    for (int r = warp; r < g.RR; r += nw) {
        const int gy = g.ry0 + r;
        const bool row_ok = gy >= 0 && gy < H && gy >= buf_y0 && gy < buf_y0 + buf_rows;
        const int64_t rr = gy - buf_y0;
        for (int c = lane; c < g.rpitch; c += 32) {
            const int gx = g.rx0 + c;
            float v = nan;
            if (row_ok && c < g.RC && gx >= 0 && gx < W)
                v = F32 ? reinterpret_cast<const float *>(ref.p + rr * ref.pitch)[gx] : (float)ref.p[rr * ref.pitch + gx];
            g.Rs[r * g.rpitch + c] = v;
        }
    }
    __syncthreads();
}

// 32 mask bits of current-region row r starting at region column c0.
__device__ __forceinline__ uint32_t mask_bits(const Regions &g, int r, int c0) {
    const uint32_t *mw = g.Mb + r * g.mwords;
    return __funnelshift_r(mw[c0 >> 5], mw[(c0 >> 5) + 1], c0 & 31);
}

// One FRMC / RMC work item: entry at tile-local (ly, lx) of the tile at (ty0, tx0) with vector
// (va, vb), delta_y = dy and up to 7 delta_x values dx0 + pat_j(k), k < nk.  Returns true iff
// some delta != 0 has an admissible reverse cost with a strictly smaller mean than the entry's
// own (m0 = fl(e0/n0) for float references; exact e'*n0 < e0*n' for uint8).
//
// Early exit (exact): the supports n'(delta) depend only on the mask and the geometry, so they
// are counted first; the reverse costs are then summed row by row in the definition's order, and
// a delta is settled as "does not reject" as soon as its partial sum reaches the threshold
// above which its final mean cannot be smaller (terms are >= 0 and fp32 accumulation of
// non-negative terms never decreases: fl(partial / n') >= m0 implies fl(final / n') >= m0).
// The item ends when every delta is settled or all rows are summed; a delta that is not settled
// is decided on its complete row-major sum, exactly as before.
// cnt8 (optional): measured pixels of the current 8x8 window at every region position (row pitch
// cw); used for the supports when the entry's reference window lies in the frame.
template <int PAT, bool SSD, bool F32>
__device__ __forceinline__ bool frmc_item(const Regions &g, int ty0, int tx0, int ly, int lx, int va, int vb, int dy,
                                          int dx0, int nk, int min_support, float m0, uint32_t e0, uint32_t n0,
                                          const uint8_t *cnt8 = nullptr, int cw = 0) {
    constexpr int KL = kFK / 2;
    constexpr int kSeg = seg_len<PAT>();
    constexpr int kK = PAT == 3 ? 2 : 7;   // delta_x slots the pattern can hold (the rest stay settled)
    float acc[7], thr[7];
    int cnt[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) { acc[k] = 0.f; cnt[k] = 0; }
    const int crow = (ty0 + ly + dy - KL) - g.cy0, ccol = (tx0 + lx + dx0 - KL) - g.cx0;
    const int rrow = (ty0 + ly + va - KL) - g.ry0, rcol = (tx0 + lx + vb - KL) - g.rx0;
    // Reference-window validity: columns x+o in the frame (a property of the entry), rows below.
    const int xx = g.rx0 + rcol, xy = g.ry0 + rrow;   // global coords of the window's (0, 0)
    // bits j with 0 <= xx + j < W: the in-frame column range as a mask
    const int clo = min(max(-xx, 0), kFK), chi = min(max(g.W - xx, 0), kFK);
    const uint32_t colm = (0xffu >> (kFK - chi)) & (0xffu << clo) & 0xffu;
    static_assert(kFK == 8, "8-bit column masks");
    // 1. Supports n'(delta) (R6, R9): slots holding a term.
    if (cnt8 && colm == 0xffu && xy >= 0 && xy + kFK <= g.H) {
#pragma unroll
        for (int k = 0; k < kK; ++k) cnt[k] = cnt8[crow * cw + ccol + pat_j<PAT>(k)];
    } else {
#pragma unroll 1
        for (int oy = 0; oy < kFK; ++oy) {
            const uint32_t rb = (xy + oy >= 0 && xy + oy < g.H) ? colm : 0u;
            const uint32_t bits = mask_bits(g, crow + oy, ccol);
#pragma unroll
            for (int k = 0; k < kK; ++k) cnt[k] += __popc((bits >> pat_j<PAT>(k)) & rb);
        }
    }
    // 2. Settled deltas: out of the set, delta = 0, SENTINEL (n' < min_support never rejects, R11);
    //    thresholds of the rest.
    unsigned settled = 0;
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        const int dx = dx0 + pat_j<PAT>(k);
        if (k >= nk || (dy == 0 && dx == 0) || cnt[k] < min_support) settled |= 1u << k;
        if (F32) thr[k] = __fmul_ru(m0, (float)cnt[k]);   // acc >= thr  =>  fl(acc / n') >= m0
        else thr[k] = n0 ? (float)(((unsigned long long)e0 * (unsigned)cnt[k] + n0 - 1) / n0) : INFINITY;   // ceil(e0 n'/n0)
    }
    // 3. Reverse costs, row-major, until every delta is settled.
    if (colm == 0xffu && xy >= 0 && xy + kFK <= g.H) {
        // Reference window in the frame: the term predicate of slot (delta_x = k, ox) is bit
        // j_k + ox of the row's current-mask segment, so the 22 segment bits serve all 56 slots.
        // Walking the bit positions in ascending order visits each delta's slots in ascending ox:
        // the accumulation order is the definition's row-major order.
#pragma unroll 1
        for (int oy = 0; oy < kFK && settled != 0x7fu; ++oy) {
            QS_DCHECK(crow + oy >= 0 && crow + oy < g.CR && ccol >= 0 && ccol + kSeg <= g.cpitch);
            QS_DCHECK(rrow + oy >= 0 && rrow + oy < g.RR && rcol >= 0 && rcol + kFK <= g.rpitch);
            const float *cp = g.Cs + (crow + oy) * g.cpitch + ccol;
            const float *rp = g.Rs + (rrow + oy) * g.rpitch + rcol;
            float c[kSeg], r[kFK];
#pragma unroll
            for (int j = 0; j < kSeg; ++j) c[j] = cp[j];
#pragma unroll
            for (int j = 0; j < kFK; ++j) r[j] = rp[j];
            const uint32_t bits = mask_bits(g, crow + oy, ccol);
            // Bit positions in pairs (b, b + 1): for an even offset j the two differences of a delta
            // are one aligned FADD2 (r[ox], r[ox+1]) - (c[b], c[b+1]); per delta still ascending ox.
#pragma unroll
            for (int b = 0; b < kSeg; b += 2) {
                const bool term0 = (bits >> b) & 1u, term1 = (bits >> (b + 1)) & 1u;
#pragma unroll
                for (int k = 0; k < kK; ++k) {
                    const int j = pat_j<PAT>(k), ox = b - j;
                    if ((j & 1) == 0) {
                        if (ox < 0 || ox >= kFK) continue;
                        float d0, d1;
                        sub2(r[ox], r[ox + 1], c[b], c[b + 1], d0, d1);
                        if (term0) acc[k] = __fadd_rn(acc[k], SSD ? __fmul_rn(d0, d0) : fabsf(d0));
                        if (term1) acc[k] = __fadd_rn(acc[k], SSD ? __fmul_rn(d1, d1) : fabsf(d1));
                    } else {
                        if (ox >= 0 && ox < kFK) {
                            const float d = __fsub_rn(r[ox], c[b]);
                            if (term0) acc[k] = __fadd_rn(acc[k], SSD ? __fmul_rn(d, d) : fabsf(d));
                        }
                        if (ox + 1 >= 0 && ox + 1 < kFK) {
                            const float d = __fsub_rn(r[ox + 1], c[b + 1]);
                            if (term1) acc[k] = __fadd_rn(acc[k], SSD ? __fmul_rn(d, d) : fabsf(d));
                        }
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < kK; ++k)
                if (acc[k] >= thr[k]) settled |= 1u << k;
        }
    } else {
#pragma unroll 1
    for (int oy = 0; oy < kFK && settled != 0x7fu; ++oy) {
        QS_DCHECK(crow + oy >= 0 && crow + oy < g.CR && ccol >= 0 && ccol + kSeg <= g.cpitch);
        QS_DCHECK(rrow + oy >= 0 && rrow + oy < g.RR && rcol >= 0 && rcol + kFK <= g.rpitch);
        const float *cp = g.Cs + (crow + oy) * g.cpitch + ccol;
        const float *rp = g.Rs + (rrow + oy) * g.rpitch + rcol;
        float c[kSeg], r[kFK];
#pragma unroll
        for (int j = 0; j < kSeg; ++j) c[j] = cp[j];
#pragma unroll
        for (int j = 0; j < kFK; ++j) r[j] = rp[j];
        const uint32_t rb = (xy + oy >= 0 && xy + oy < g.H) ? colm : 0u;
        const uint32_t bits = mask_bits(g, crow + oy, ccol);
#pragma unroll
        for (int k = 0; k < kK; ++k) {
            const int j = pat_j<PAT>(k);
            const uint32_t vm = (bits >> j) & rb;              // slots holding a term (R9)
            float dd[kFK];
            if ((j & 1) == 0) {
                // even offsets: differences of aligned register pairs in one FADD2 each
#pragma unroll
                for (int ox = 0; ox < kFK; ox += 2) sub2(r[ox], r[ox + 1], c[ox + j], c[ox + j + 1], dd[ox], dd[ox + 1]);
            } else {
#pragma unroll
                for (int ox = 0; ox < kFK; ++ox) dd[ox] = __fsub_rn(r[ox], c[ox + j]);
            }
#pragma unroll
            for (int ox = 0; ox < kFK; ++ox) {
                const float t = SSD ? __fmul_rn(dd[ox], dd[ox]) : fabsf(dd[ox]);
                if (vm & (1u << ox)) acc[k] = __fadd_rn(acc[k], t);   // row-major order, terms only
            }
            if (acc[k] >= thr[k]) settled |= 1u << k;
        }
    }
    }
    if (settled == 0x7fu) return false;
    bool reject = false;
#pragma unroll
    for (int k = 0; k < kK; ++k) {
        if (settled & (1u << k)) continue;
        if (F32) {
            if (__fdiv_rn(acc[k], (float)cnt[k]) < m0) reject = true;
        } else {
            const unsigned long long ek = (unsigned long long)acc[k];
            if (ek * n0 < (unsigned long long)e0 * (unsigned)cnt[k]) reject = true;
        }
    }
    return reject;
}

}  // namespace tile
}  // namespace qs
