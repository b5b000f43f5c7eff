// epilogue.cu -- the fused per-pair epilogue of qs_me_search for K = 8:
//   finalize (decode the merged ME keys, re-sum the chosen vector's error in the
//   definition's row-major order), NNC (Eq. 1; R14, R15) and the
//   FRMC cascade (R11, R12, R16) in ONE launch per
//   16x16 tile.  The tile's current-frame and reference regions are staged once in
//   shared memory and serve all three steps; the motion vectors of the tile and its
//   2-pixel halo are decoded from the ME keys directly (no round trip through the
//   field planes), so the field is written once, with its final statuses.
#include <cmath>

#include "qs_internal.cuh"
#include "tile_regions.cuh"

namespace qs {
namespace {

using tile::kFK;
using tile::kFT;
constexpr int kH2 = kFT + 4;   // decoded window: tile + 2-pixel halo (NNC's vector halo)
constexpr int kH1 = kFT + 2;   // filtered window: tile + 1-pixel halo
constexpr int kCW = kFT + 14;  // FRMC window positions per axis (tile + the paper offsets' +-7)

// Lower median of the valid values among v[0..8] (Eq. 1, R14: invalid entries carry +1000 and sort
// last): sort ascending with the 25-comparator network for 9 inputs (verified on all 2^9 0/1 inputs:
// 0-1 principle), take index (n-1)/2.  Both components at once: (alpha, beta) as two signed 16-bit
// lanes of one word, min / max per lane (VIMNMX.S16x2), so one sort serves the two medians.
constexpr unsigned kMedSentinel = 1000u | (1000u << 16);   // invalid entries: +1000 in both lanes, sort last
__device__ __forceinline__ unsigned pack_ab(int a, int b) { return (unsigned)(a & 0xffff) | ((unsigned)b << 16); }
__device__ __forceinline__ unsigned lower_median9_x2(unsigned (&v)[9], int n) {
    constexpr int kNet[25][2] = {{0, 1}, {3, 4}, {6, 7}, {1, 2}, {4, 5}, {7, 8}, {0, 1}, {3, 4}, {6, 7},
                                 {0, 3}, {3, 6}, {0, 3}, {1, 4}, {4, 7}, {1, 4}, {2, 5}, {5, 8}, {2, 5},
                                 {1, 3}, {5, 7}, {2, 6}, {4, 6}, {2, 4}, {2, 3}, {5, 6}};
#pragma unroll
    for (int c = 0; c < 25; ++c) {
        const unsigned a = v[kNet[c][0]], b = v[kNet[c][1]];
        v[kNet[c][0]] = __vmins2(a, b);
        v[kNet[c][1]] = __vmaxs2(a, b);
    }
    unsigned r = v[0];
#pragma unroll
    for (int i = 1; i < 9; ++i)
        if (i == (n - 1) / 2) r = v[i];
    return r;
}

struct EpiShared {
    int8_t sa[kH2][kH2], sb[kH2][kH2];
    uint8_t sv[kH2][kH2];
    unsigned sp[kH2][kH2];    // pack_ab(alpha, beta) of valid entries, kMedSentinel otherwise
    int fa[kH1][kH1], fb[kH1][kH1];
    uint8_t st[kFT * kFT];
    float m0[kFT * kFT];
    uint32_t e0[kFT * kFT], n0[kFT * kFT];
    int ent[kFT * kFT];
    uint8_t rej[kFT * kFT];
    uint8_t cnt8[kCW][kCW];   // measured pixels of the 8x8 current window at each region position
    int wcnt[8];              // checkable entries per warp (the entry list is in tid = row-major order)
    uint32_t pjm[kFT * kFT], pjv[kFT * kFT];   // PR prefetch: aligned words of past_mask / past_val at p+v
    int n_ent;
};

template <bool SSD, bool F32, bool NNC, bool FRMC>
__global__ void __launch_bounds__(256, 4) epilogue_kernel(const EpiArgs g) {
    extern __shared__ __align__(16) float sm[];
    __shared__ EpiShared S;
    constexpr int KL = kFK / 2;
    const int tx0 = blockIdx.x * kFT, ty0 = g.lo + blockIdx.y * kFT;
    tile::Regions R = tile::layout(sm, ty0, tx0, 7, g.S, g.W, g.H);
    const int tid = threadIdx.x;
    const int zr = blockIdx.z;                   // reference slot (qs_me_search_refs)
    const unsigned long long *keys = g.keys_p[zr];
    __shared__ int box[4];                       // min / max of ly + alpha, lx + beta over valid own entries
    if (tid < 4) box[tid] = (tid & 1) ? -(1 << 20) : (1 << 20);
    tile::stage_cur(R, g.cur, g.mask, g.W, g.H, g.buf_y0, g.buf_rows);   // ends with __syncthreads

    // 1. Decode the vectors of the tile + 2-pixel halo from the keys; validity needs the
    //    support n of the chosen vector (min_support, R6), counted from the mask bits.
    for (int i = tid; i < kH2 * kH2; i += blockDim.x) {
        const int r = i / kH2, c = i % kH2;
        const int gy = ty0 - 2 + r, gx = tx0 - 2 + c;
        int8_t va = 0, vb = 0;
        uint8_t valid = 0, st0 = kNotTarget, nn = 0;
        if (gy >= g.lo && gy < g.hi && gx >= 0 && gx < g.W) {
            const int cr = gy - R.cy0, cc = gx - R.cx0;
            const bool measured = (tile::mask_bits(R, cr, cc) & 1u) != 0;
            if (!measured) {
                st0 = kInvalid;
                QS_DCHECK(gy >= g.lo && gy < g.hi && gx < g.key_pitch);
                const unsigned long long key = keys[(int64_t)(gy - g.lo) * g.key_pitch + gx];
                if (key != ~0ull) {
                    const int pk = __ldg(g.canon + (int)(key & 0xffffffffu));
                    const int a = (int)(int8_t)(pk & 0xff), b = (int)(int8_t)((pk >> 8) & 0xff);
                    // window columns qx = gx - KL + j with qx and qx + b in the frame, as a bit range
                    const int clo = min(max(max(0, -b) - (gx - KL), 0), kFK);
                    const int chi = min(max(min(g.W, g.W - b) - (gx - KL), 0), kFK);
                    const uint32_t colm = (0xffu >> (kFK - chi)) & (0xffu << clo) & 0xffu;
                    int n = 0;
#pragma unroll
                    for (int oy = 0; oy < kFK; ++oy) {
                        const int qy = gy - KL + oy;
                        if (qy < 0 || qy >= g.H || qy + a < 0 || qy + a >= g.H) continue;
                        n += __popc(tile::mask_bits(R, qy - R.cy0, gx - KL - R.cx0) & colm);
                    }
                    nn = (uint8_t)n;
                    if (n >= g.min_support) {
                        valid = 1;
                        st0 = kCandidate;
                        va = (int8_t)a;
                        vb = (int8_t)b;
                    }
                }
            }
        }
        S.sa[r][c] = va;
        S.sb[r][c] = vb;
        S.sv[r][c] = valid;
        S.sp[r][c] = valid ? pack_ab(va, vb) : kMedSentinel;
        if (r >= 2 && r < kFT + 2 && c >= 2 && c < kFT + 2) {
            const int o = (r - 2) * kFT + (c - 2);
            S.st[o] = st0;
            S.n0[o] = nn;
            if (valid) {   // the reference rows / columns this entry's window reads
                atomicMin(&box[0], (r - 2) + va);
                atomicMax(&box[1], (r - 2) + va);
                atomicMin(&box[2], (c - 2) + vb);
                atomicMax(&box[3], (c - 2) + vb);
            }
        }
    }
    __syncthreads();
    // Stage only the reference rows / columns the tile's vectors reach (the re-sum and FRMC read the
    // window at p + v; round 1 staged the whole (16 + 2S + 7)^2 search region).
    if (box[0] <= box[1]) {
        tile::narrow_ref(R, ty0, tx0, box[0], box[1], box[2], box[3]);
        tile::stage_ref<F32>(R, Plane{g.ref_p[zr], g.ref.pitch}, g.W, g.H, g.buf_y0, g.buf_rows);
    }

    // 2. Filtered field (Eq. 1) on the tile + 1-pixel halo.
    if (NNC) {
        for (int i = tid; i < kH1 * kH1; i += blockDim.x) {
            const int r = i / kH1 + 1, c = i % kH1 + 1;
            unsigned lv[9];
            int n = 0;
#pragma unroll
            for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                for (int dx = -1; dx <= 1; ++dx) {
                    const int k = (dy + 1) * 3 + (dx + 1);
                    lv[k] = S.sp[r + dy][c + dx];
                    n += lv[k] != kMedSentinel;
                }
            int ma = 0, mb = 0;
            if (S.sv[r][c]) {
                const unsigned m = lower_median9_x2(lv, n);
                ma = (int)(int16_t)(m & 0xffffu);
                mb = (int)(int16_t)(m >> 16);
            }
            S.fa[r - 1][c - 1] = ma;
            S.fb[r - 1][c - 1] = mb;
        }
        __syncthreads();
    }

    // 3. Own entry: the chosen vector's error re-summed in row-major order (R23), NNC decision.
    const int ly = tid / kFT, lx = tid % kFT;
    const int gy = ty0 + ly, gx = tx0 + lx;
    const bool own = gy < g.hi && gx < g.W;
    const bool checked_row = gy >= g.y0 && gy < g.y1;
    uint8_t st = S.st[tid];
    const int a = S.sa[ly + 2][lx + 2], b = S.sb[ly + 2][lx + 2];
    float ef = 0.f;
    uint32_t eu = 0;
    // PR prefetch (fused projection): the words holding past_mask / past_val at q = p + v, fetched
    // with cp.async now and read after FRMC, so the gather latency hides under the checks.
    int pj_sh = -1;
    if (g.proj && own && checked_row && st == kCandidate) {
        const int qy = gy + a, qx = gx + b;
        if (qy >= 0 && qy < g.H && qx >= 0 && qx < g.W && qy >= g.buf_y0 && qy < g.buf_y0 + g.buf_rows) {
            const int64_t qi = (int64_t)(qy - g.buf_y0) * g.past_pitch + qx;
            const uintptr_t am = reinterpret_cast<uintptr_t>(g.pm_p[zr] + qi), av = reinterpret_cast<uintptr_t>(g.pv_p[zr] + qi);
            pj_sh = 8 * (int)(am & 3);   // past planes share one pitch and are 16-byte aligned: same offset
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(&S.pjm[tid])),
                         "l"(am & ~uintptr_t(3)));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((unsigned)__cvta_generic_to_shared(&S.pjv[tid])),
                         "l"(av & ~uintptr_t(3)));
        }
    }
    asm volatile("cp.async.commit_group;");
    if (own && st == kCandidate) {
        const int crow = (gy - KL) - R.cy0, ccol = (gx - KL) - R.cx0;
        const int rrow = (gy + a - KL) - R.ry0, rcol = (gx + b - KL) - R.rx0;
#pragma unroll 1
        for (int oy = 0; oy < kFK; ++oy) {
            QS_DCHECK(crow + oy >= 0 && crow + oy < R.CR && ccol >= 0 && ccol + kFK <= R.cpitch);
            QS_DCHECK(rrow + oy >= 0 && rrow + oy < R.RR && rcol >= 0 && rcol + kFK <= R.rpitch);
            const float *cp = R.Cs + (crow + oy) * R.cpitch + ccol;
            const float *rp = R.Rs + (rrow + oy) * R.rpitch + rcol;
#pragma unroll
            for (int ox = 0; ox < kFK; ++ox) {
                const float d = __fsub_rn(cp[ox], rp[ox]);
                const float t = SSD ? __fmul_rn(d, d) : fabsf(d);
                ef = __fadd_rn(ef, fmaxf(t, 0.f));   // NaN (no term) -> +0
            }
        }
        if (!F32) eu = (uint32_t)ef;                 // integer-valued and < 2^24: exact
        if (NNC && checked_row) {
            const int r = ly + 2, c = lx + 2;
            const int NB[4][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}};
            int na[4], nb[4];
            bool nv[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int rr = r + NB[k][0], cc = c + NB[k][1];
                nv[k] = S.sv[rr][cc];
                na[k] = S.fa[rr - 1][cc - 1];
                nb[k] = S.fb[rr - 1][cc - 1];
            }
            st = nnc_rejects(g.nnc, S.fa[r - 1][c - 1], S.fb[r - 1][c - 1], na, nb, nv, g.nnc_threshold) ? kRejected
                                                                                                      : kAccepted;
        }
    }
    if (FRMC) {
        S.m0[tid] = F32 ? __fdiv_rn(ef, (float)S.n0[tid]) : 0.f;
        S.e0[tid] = F32 ? 0u : eu;
        S.rej[tid] = 0;
    }
    const bool chk = FRMC && own && checked_row && (st == kCandidate || st == kAccepted);
    const unsigned chk_m = __ballot_sync(0xffffffffu, chk);
    if (FRMC && (tid & 31) == 0) S.wcnt[tid >> 5] = __popc(chk_m);
    // PR (R18) of the entries whose final status is ACCEPTED, into the frame's sum / cnt.
    // Called by the whole warp: the four lanes of an aligned 4-pixel group (lx & 3 == gx & 3, tiles
    // start at multiples of 16) combine their cnt bytes into one word add (no carry: cnt < 256).
    auto project = [&](uint8_t fin) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        bool pj = g.proj && own && checked_row && fin == kAccepted && pj_sh >= 0;
        if (pj) pj = ((S.pjm[tid] >> pj_sh) & 0xffu) != 0;
        const int64_t ai = (int64_t)(gy - g.buf_y0) * g.acc_pitch + gx;
        if (pj) atomicAdd(g.sum + ai, (S.pjv[tid] >> pj_sh) & 0xffu);
        unsigned inc = pj ? 1u << (8 * (gx & 3)) : 0u;
        inc |= __shfl_xor_sync(0xffffffffu, inc, 1);
        inc |= __shfl_xor_sync(0xffffffffu, inc, 2);
        if ((gx & 3) == 0 && inc) atomicAdd(reinterpret_cast<unsigned *>(g.cnt + ai), inc);
    };
    // Only the roi's rows [y0, y1) are written: the NNC halo rows were decoded for the median only
    // (a neighbouring band's call owns them; writing them would race with it on a shared field).
    if (own && checked_row && g.write_field) {
        QS_DCHECK(gy >= g.buf_y0 && gy < g.buf_y0 + g.buf_rows && gx < g.f_p[zr].pitch);
        const int64_t fi = (int64_t)(gy - g.buf_y0) * g.f_p[zr].pitch + gx;
        const bool has = st >= kCandidate;
        g.f_p[zr].alpha[fi] = has ? (int8_t)a : (int8_t)0;
        g.f_p[zr].beta[fi] = has ? (int8_t)b : (int8_t)0;
        g.f_p[zr].count[fi] = has ? S.n0[tid] : (uint8_t)0;
        if (F32) reinterpret_cast<float *>(g.f_p[zr].err)[fi] = has ? ef : 0.f;
        else reinterpret_cast<uint32_t *>(g.f_p[zr].err)[fi] = has ? eu : 0u;
        if (!FRMC) g.f_p[zr].status[fi] = st;
    }
    if (!FRMC) {
        project(st);
        return;
    }

    // 4. FRMC on the checkable entries (NNC survivors in the cascade): items (entry, delta_y).
    //    Supports n'(delta) of entries whose reference window lies in the frame are the measured
    //    pixels of the current 8x8 window at p + delta: one table for the tile (cnt8).
    for (int i = tid; i < kCW * kCW; i += blockDim.x) {
        const int r = i / kCW, c = i % kCW;
        int n = 0;
#pragma unroll
        for (int oy = 0; oy < kFK; ++oy) n += __popc(tile::mask_bits(R, r + oy, c) & 0xffu);
        S.cnt8[r][c] = (uint8_t)n;
    }
    __syncthreads();
    // Entry list in tid order (row-major in the tile): neighbouring lanes read neighbouring windows.
    {
        int base = 0, ne_all = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
            base += (w < (tid >> 5)) ? S.wcnt[w] : 0;
            ne_all += S.wcnt[w];
        }
        if (chk) S.ent[base + __popc(chk_m & ((1u << (tid & 31)) - 1u))] = tid;
        if (tid == 0) S.n_ent = ne_all;
    }
    __syncthreads();
    const int ne = S.n_ent;
    const int items = ne * 7;
    // delta_y-major: later rounds skip entries an earlier delta_y row already rejected.
    int iy = ne ? tid / ne : 0, e = ne ? tid - iy * ne : 0;   // item it = iy * ne + e, one division
    for (int it = tid; it < items; it += blockDim.x, e += blockDim.x) {
        while (e >= ne) { e -= ne; ++iy; }
        const int o = S.ent[e];
        if (S.rej[o]) continue;
        const int ely = o / kFT, elx = o % kFT;
        const int va = S.sa[ely + 2][elx + 2], vb = S.sb[ely + 2][elx + 2];
        if (tile::frmc_item<0, SSD, F32>(R, ty0, tx0, ely, elx, va, vb, g.dys[iy], -7, 7, g.min_support, S.m0[o],
                                         S.e0[o], S.n0[o], &S.cnt8[0][0], kCW))
            S.rej[o] = 1;
    }
    __syncthreads();
    if (own && checked_row && g.write_field) {
        const bool checked = checked_row && (st == kCandidate || st == kAccepted);
        const int64_t fi = (int64_t)(gy - g.buf_y0) * g.f_p[zr].pitch + gx;
        g.f_p[zr].status[fi] = checked ? (S.rej[tid] ? kRejected : kAccepted) : st;
    }
    project(checked_row && (st == kCandidate || st == kAccepted) ? (S.rej[tid] ? kRejected : kAccepted) : st);
    if (g.evals && tid == 0 && ne) atomicAdd(g.evals, 49ull * (unsigned long long)ne);
}

template <bool SSD, bool F32, bool NNC, bool FRMC>
cudaError_t launch_epi_t(const EpiArgs &g, cudaStream_t s) {
    const size_t smem = tile::RegionSizes(7, g.S).bytes() + 16;
    auto fn = epilogue_kernel<SSD, F32, NNC, FRMC>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grd((g.W + kFT - 1) / kFT, (g.hi - g.lo + kFT - 1) / kFT, g.n_ref);
    fn<<<grd, 256, smem, s>>>(g);
    return cudaGetLastError();
}

template <bool SSD, bool F32>
cudaError_t launch_epi_c(const EpiArgs &g, cudaStream_t s) {
    if (g.nnc && g.frmc) return launch_epi_t<SSD, F32, true, true>(g, s);
    if (g.nnc) return launch_epi_t<SSD, F32, true, false>(g, s);
    if (g.frmc) return launch_epi_t<SSD, F32, false, true>(g, s);
    return launch_epi_t<SSD, F32, false, false>(g, s);
}

}  // namespace

cudaError_t launch_epilogue(const EpiArgs &g0, cudaStream_t s) {
    if (g0.hi <= g0.lo) return cudaSuccess;
    EpiArgs g = g0;
    if (g.n_ref <= 0) {   // one slot: (ref, keys, f)
        g.n_ref = 1;
        g.ref_p[0] = g.ref.p;
        g.keys_p[0] = g.keys;
        g.f_p[0] = g.f;
    }
    if (g.n_ref > kMaxRefs) return cudaErrorInvalidValue;
    if (g.ref_f32) return g.ssd ? launch_epi_c<true, true>(g, s) : launch_epi_c<false, true>(g, s);
    return g.ssd ? launch_epi_c<true, false>(g, s) : launch_epi_c<false, false>(g, s);
}

}  // namespace qs
