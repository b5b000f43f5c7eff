// checks.cu -- the consistency checks and the projection on sm_100a.
//   K5 nnc       NNC (§3.1.2, Eq. (1); R14, R15)
//   K3/K4 revgrid FRMC and RMC: reverse costs
//                rc(x = p+v, u = -v + delta) over a delta grid (R9, R11, R12)
//   K4 rme_decide RME (R10) from the dense reverse keys of me_box
//   K6 project   PR (§2.2; R18)
#include <cmath>

#include "qs_internal.cuh"
#include "tile_regions.cuh"

namespace qs {
namespace {

__device__ __forceinline__ bool checkable(uint8_t s) { return s == kCandidate || s == kAccepted; }

// ---------------------------------------------------------------------------
// NNC.  Block = 32 x 8 outputs.  Shared: the field with a 2-pixel halo, then
// the filtered field (Eq. (1)) with a 1-pixel halo; then the 4-neighbour rule.
// ---------------------------------------------------------------------------
constexpr int kNX = 32, kNY = 8;

// Lower median of the valid values among v[0..8] (invalid entries carry +1000
// and sort last): sort ascending, take index (n-1)/2.
__device__ __forceinline__ int lower_median9(int (&v)[9], int n) {
    // 25-comparator sorting network for 9 inputs (verified on all 2^9 0/1 inputs: 0-1 principle)
    constexpr int kNet[25][2] = {{0, 1}, {3, 4}, {6, 7}, {1, 2}, {4, 5}, {7, 8}, {0, 1}, {3, 4}, {6, 7},
                                 {0, 3}, {3, 6}, {0, 3}, {1, 4}, {4, 7}, {1, 4}, {2, 5}, {5, 8}, {2, 5},
                                 {1, 3}, {5, 7}, {2, 6}, {4, 6}, {2, 4}, {2, 3}, {5, 6}};
#pragma unroll
    for (int c = 0; c < 25; ++c) {
        const int a = v[kNet[c][0]], b = v[kNet[c][1]];
        v[kNet[c][0]] = min(a, b);
        v[kNet[c][1]] = max(a, b);
    }
    int r = v[0];
#pragma unroll
    for (int i = 1; i < 9; ++i)
        if (i == (n - 1) / 2) r = v[i];
    return r;
}

__global__ void __launch_bounds__(kNX * kNY) nnc_kernel(FieldView f, int W, int H, int buf_y0, int buf_rows,
                                                          int y0, int y1, int threshold, int mode) {
    __shared__ int sa[kNY + 4][kNX + 4], sb[kNY + 4][kNX + 4];
    __shared__ uint8_t sv[kNY + 4][kNX + 4];
    __shared__ int fa[kNY + 2][kNX + 2], fb[kNY + 2][kNX + 2];
    const int tx0 = blockIdx.x * kNX, ty0 = y0 + blockIdx.y * kNY;
    const int tid = threadIdx.y * kNX + threadIdx.x;
    for (int i = tid; i < (kNY + 4) * (kNX + 4); i += kNX * kNY) {
        const int r = i / (kNX + 4), c = i % (kNX + 4);
        const int gy = ty0 - 2 + r, gx = tx0 - 2 + c;
        int a = 0, b = 0;
        uint8_t v = 0;
        if (gy >= 0 && gy < H && gx >= 0 && gx < W && gy >= buf_y0 && gy < buf_y0 + buf_rows) {
            const int64_t fi = (int64_t)(gy - buf_y0) * f.pitch + gx;
            v = f.status[fi] >= kCandidate;
            a = f.alpha[fi];
            b = f.beta[fi];
        }
        sa[r][c] = a;
        sb[r][c] = b;
        sv[r][c] = v;
    }
    __syncthreads();
    for (int i = tid; i < (kNY + 2) * (kNX + 2); i += kNX * kNY) {
        const int r = i / (kNX + 2) + 1, c = i % (kNX + 2) + 1;   // coords in the 2-halo arrays
        int va[9], vb[9], n = 0;
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
            for (int dx = -1; dx <= 1; ++dx) {
                const int k = (dy + 1) * 3 + (dx + 1);
                const bool ok = sv[r + dy][c + dx];
                va[k] = ok ? sa[r + dy][c + dx] : 1000;
                vb[k] = ok ? sb[r + dy][c + dx] : 1000;
                n += ok;
            }
        int ma = 0, mb = 0;
        if (sv[r][c]) {
            ma = lower_median9(va, n);
            mb = lower_median9(vb, n);
        }
        fa[r - 1][c - 1] = ma;
        fb[r - 1][c - 1] = mb;
    }
    __syncthreads();
    const int gx = tx0 + threadIdx.x, gy = ty0 + threadIdx.y;
    if (gx >= W || gy >= y1) return;
    const int r = threadIdx.y + 2, c = threadIdx.x + 2;   // 2-halo coords
    const int64_t fi = (int64_t)(gy - buf_y0) * f.pitch + gx;
    const uint8_t st = f.status[fi];
    if (!checkable(st)) return;
    const int NBR[4][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}};
    int na[4], nb[4];
    bool nv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int rr = r + NBR[k][0], cc = c + NBR[k][1];
        nv[k] = sv[rr][cc];          // out of frame or not valid: skipped (R15)
        na[k] = fa[rr - 1][cc - 1];
        nb[k] = fb[rr - 1][cc - 1];
    }
    f.status[fi] = nnc_rejects(mode, fa[r - 1][c - 1], fb[r - 1][c - 1], na, nb, nv, threshold) ? kRejected : kAccepted;
}

// ---------------------------------------------------------------------------
// Reverse-cost grid (FRMC / RMC).  One thread per field entry.  Each reverse
// cost is summed in the definition's row-major order (R9, R23), so the f32
// decisions are those of the oracle given the same field; the delta loop may
// stop at the first strictly smaller mean (the decision is "reject iff any",
// R11) while the evaluation counter reports the definitional |delta set| (R17).
// ---------------------------------------------------------------------------
struct DeltaSet {
    int n;              // 0 => full range [lo, hi]^2
    int lo, hi;
    int8_t v[16];
};

__global__ void revgrid_kernel(RevGridArgs a, DeltaSet ds) {
    const int gx = blockIdx.x * blockDim.x + threadIdx.x;
    const int gy = a.y0 + blockIdx.y;
    unsigned long long my_evals = 0;
    if (gx < a.W && gy < a.y1) {
        const int64_t fi = (int64_t)(gy - a.buf_y0) * a.f.pitch + gx;
        const uint8_t st = a.f.status[fi];
        if (checkable(st)) {
            const int va = a.f.alpha[fi], vb = a.f.beta[fi];
            const int xy = gy + va, xx = gx + vb;
            const int n0 = a.f.count[fi];
            const float e0f = a.ref_f32 ? reinterpret_cast<const float *>(a.f.err)[fi] : 0.f;
            const uint32_t e0u = a.ref_f32 ? 0u : reinterpret_cast<const uint32_t *>(a.f.err)[fi];
            const float m0 = a.ref_f32 ? __fdiv_rn(e0f, (float)n0) : 0.f;
            const int KL = a.K / 2;
            const int nd = ds.n ? ds.n : (ds.hi - ds.lo + 1);
            bool reject = false;
            for (int iy = 0; iy < nd && !reject; ++iy) {
                const int dy = ds.n ? ds.v[iy] : ds.lo + iy;
                for (int ix = 0; ix < nd && !reject; ++ix) {
                    const int dx = ds.n ? ds.v[ix] : ds.lo + ix;
                    if (dy == 0 && dx == 0) continue;
                    const int uy = -va + dy, ux = -vb + dx;
                    int n = 0;
                    uint32_t eu = 0;
                    float ef = 0.f;
                    for (int oy = -KL; oy < a.K - KL; ++oy) {
                        const int qy = xy + oy, sy = qy + uy;
                        if (qy < 0 || qy >= a.H || sy < 0 || sy >= a.H) continue;
                        if (qy < a.buf_y0 || qy >= a.buf_y0 + a.buf_rows) continue;   // never for valid rois
                        if (sy < a.buf_y0 || sy >= a.buf_y0 + a.buf_rows) continue;
                        const int64_t qr = qy - a.buf_y0, sr = sy - a.buf_y0;
                        for (int ox = -KL; ox < a.K - KL; ++ox) {
                            const int qx = xx + ox, sx = qx + ux;
                            if (qx < 0 || qx >= a.W || sx < 0 || sx >= a.W) continue;
                            if (!a.mask.p[sr * a.mask.pitch + sx]) continue;
                            const int c = a.cur.p[sr * a.cur.pitch + sx];
                            if (a.ref_f32) {
                                const float rv = reinterpret_cast<const float *>(a.ref.p + qr * a.ref.pitch)[qx];
                                const float d = __fsub_rn((float)c, rv);
                                ef = __fadd_rn(ef, a.ssd ? __fmul_rn(d, d) : fabsf(d));
                            } else {
                                const int d = c - (int)a.ref.p[qr * a.ref.pitch + qx];
                                eu += (uint32_t)(a.ssd ? d * d : (d < 0 ? -d : d));
                            }
                            ++n;
                        }
                    }
                    if (n < a.min_support) continue;   // SENTINEL never rejects (R11)
                    if (a.ref_f32) {
                        if (__fdiv_rn(ef, (float)n) < m0) reject = true;
                    } else {
                        if ((unsigned long long)eu * (unsigned)n0 < (unsigned long long)e0u * (unsigned)n) reject = true;
                    }
                }
            }
            my_evals = (unsigned long long)nd * nd;
            a.f.status[fi] = reject ? kRejected : kAccepted;
        }
    }
    if (a.evals) {
        // warp-aggregate the definitional count
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) my_evals += __shfl_down_sync(0xffffffffu, my_evals, o);
        if ((threadIdx.x & 31) == 0 && my_evals) atomicAdd(a.evals, my_evals);
    }
}

// ---------------------------------------------------------------------------
// Tiled reverse-cost grid for K = 8 (the configs' template).  One CTA = a 16x16
// tile of field entries.  The reference region the entries' x = p+v windows can
// reach and the current-frame region the shifted windows p+delta+o can reach are
// staged once into shared memory (float, NaN = no term), with the current mask
// as bit rows.  Work items are (entry, delta_y, delta_x-group of up to 7); an item
// keeps 7 accumulators and walks the 8 template rows: per row it loads the 8
// reference values of the x window and the 22-wide current segment, and adds
// phi(ref - cur) for every (delta_x, o_x) from registers with static indices.
// Each reverse cost is still summed in row-major o order (R23), so decisions
// equal the oracle's; the support n' comes from popcounts of the mask bits.
// Delta_x patterns: PAT 0 = the paper's {-7,-3,-1,0,1,3,7},
// PAT 1 = 7 consecutive values (RMC's [-S, S] in groups).
// ---------------------------------------------------------------------------
using tile::kFT;
using tile::kFK;

struct TileGridArgs {
    RevGridArgs a;
    int n_dy;          // delta_y values
    int8_t dys[16];    // PAT 0: the offsets; PAT 1: unused (dy = lo + i)
    int lo;            // PAT 1: first delta (== -S)
    int n_groups;      // delta_x groups
    int n_last;        // deltas in the last group (PAT 1)
    int maxd;          // max |delta|
    int S;             // max |v|
    int n_total;       // |delta set| for the evaluation counter
};

template <int PAT, bool SSD, bool F32>
__global__ void __launch_bounds__(256) revgrid_tile_kernel(const TileGridArgs g) {
    extern __shared__ __align__(16) float sm[];
    const RevGridArgs &a = g.a;
    const int tx0 = blockIdx.x * kFT, ty0 = a.y0 + blockIdx.y * kFT;
    const tile::Regions R = tile::layout(sm, ty0, tx0, g.maxd, g.S, a.W, a.H);
    const tile::RegionSizes Z(g.maxd, g.S);
    int *ent = reinterpret_cast<int *>(reinterpret_cast<char *>(sm) + Z.bytes());   // packed entries [256]
    float *ent_m0 = reinterpret_cast<float *>(ent + kFT * kFT);
    uint32_t *ent_e0 = reinterpret_cast<uint32_t *>(ent_m0 + kFT * kFT);
    uint8_t *rej = reinterpret_cast<uint8_t *>(ent_e0 + kFT * kFT);
    // measured pixels of the current 8x8 window at each region position (supports of entries whose
    // reference window lies in the frame, tile::frmc_item)
    const int cw = kFT + 2 * g.maxd;
    uint8_t *cnt8 = rej + kFT * kFT;
    __shared__ int n_ent;
    const int tid = threadIdx.x;
    if (tid == 0) n_ent = 0;
    tile::stage<F32>(R, a.cur, a.mask, a.ref, a.W, a.H, a.buf_y0, a.buf_rows);
    // Checkable entries of the tile.
    {
        const int ly = tid / kFT, lx = tid % kFT;
        const int gy = ty0 + ly, gx = tx0 + lx;
        if (gy < a.y1 && gx < a.W) {
            const int64_t fi = (int64_t)(gy - a.buf_y0) * a.f.pitch + gx;
            if (checkable(a.f.status[fi])) {
                const int slot = atomicAdd(&n_ent, 1);
                const int va = a.f.alpha[fi], vb = a.f.beta[fi];
                ent[slot] = (ly) | (lx << 8) | ((va & 0xff) << 16) | ((vb & 0xff) << 24);
                const int n0 = a.f.count[fi];
                if (F32) {
                    ent_m0[slot] = __fdiv_rn(reinterpret_cast<const float *>(a.f.err)[fi], (float)n0);
                    ent_e0[slot] = (uint32_t)n0;
                } else {
                    ent_e0[slot] = reinterpret_cast<const uint32_t *>(a.f.err)[fi];
                    ent_m0[slot] = __int_as_float(n0);
                }
                rej[slot] = 0;
            }
        }
    }
    for (int i = tid; i < cw * cw; i += blockDim.x) {
        const int r = i / cw, c = i - r * cw;
        int n = 0;
#pragma unroll
        for (int oy = 0; oy < kFK; ++oy) n += __popc(tile::mask_bits(R, r + oy, c) & 0xffu);
        cnt8[i] = (uint8_t)n;
    }
    __syncthreads();
    const int ne = n_ent;
    const int per_entry = g.n_dy * g.n_groups;
    const int items = ne * per_entry;
    for (int it = tid; it < items; it += blockDim.x) {
        // (delta_y, group)-major: later rounds skip entries an earlier round already rejected.
        const int rem = it / ne, e = it - rem * ne;
        if (rej[e]) continue;                            // decision already made ("reject iff any")
        const int iy = rem / g.n_groups, grp = rem - iy * g.n_groups;
        const int pk = ent[e];
        const int ly = pk & 0xff, lx = (pk >> 8) & 0xff;
        const int va = (int)(int8_t)((pk >> 16) & 0xff), vb = (int)(int8_t)((pk >> 24) & 0xff);
        // PAT 1 visits delta_y = 0, -1, 1, -2, 2, ... (small offsets reject wrong vectors first)
        const int dy = PAT != 1 ? g.dys[iy] : ((iy & 1) ? -((iy + 1) >> 1) : (iy >> 1));
        const uint32_t n0 = F32 ? ent_e0[e] : (uint32_t)__float_as_int(ent_m0[e]);
        bool r;
        if constexpr (PAT == 2) {   // the +-15 set: group 0 = {-15,-7,-3,-1,0,1,3}, group 1 = {7, 15}
            r = grp == 0 ? tile::frmc_item<2, SSD, F32>(R, ty0, tx0, ly, lx, va, vb, dy, -15, 7, a.min_support,
                                                        ent_m0[e], ent_e0[e], n0, cnt8, cw)
                         : tile::frmc_item<3, SSD, F32>(R, ty0, tx0, ly, lx, va, vb, dy, 7, 2, a.min_support,
                                                        ent_m0[e], ent_e0[e], n0, cnt8, cw);
        } else {
            const int dx0 = PAT == 0 ? -7 : g.lo + 7 * grp;
            const int nk = PAT == 0 ? 7 : (grp == g.n_groups - 1 ? g.n_last : 7);
            r = tile::frmc_item<PAT, SSD, F32>(R, ty0, tx0, ly, lx, va, vb, dy, dx0, nk, a.min_support, ent_m0[e],
                                               ent_e0[e], n0, cnt8, cw);
        }
        if (r) rej[e] = 1;
    }
    __syncthreads();
    for (int e = tid; e < ne; e += blockDim.x) {
        const int pk = ent[e];
        const int gy = ty0 + (pk & 0xff), gx = tx0 + ((pk >> 8) & 0xff);
        a.f.status[(int64_t)(gy - a.buf_y0) * a.f.pitch + gx] = rej[e] ? kRejected : kAccepted;
    }
    if (a.evals && tid == 0 && ne) atomicAdd(a.evals, (unsigned long long)ne * (unsigned long long)g.n_total);
}

template <int PAT, bool SSD, bool F32>
cudaError_t launch_tile_t(const TileGridArgs &g, cudaStream_t s) {
    const size_t smem = tile::RegionSizes(g.maxd, g.S).bytes() +
                        (sizeof(int) + sizeof(float) + sizeof(uint32_t) + 1) * kFT * kFT +
                        (size_t)(kFT + 2 * g.maxd) * (kFT + 2 * g.maxd) + 16;
    auto fn = revgrid_tile_kernel<PAT, SSD, F32>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    dim3 grd((g.a.W + kFT - 1) / kFT, (g.a.y1 - g.a.y0 + kFT - 1) / kFT);
    fn<<<grd, 256, smem, s>>>(g);
    return cudaGetLastError();
}

template <int PAT>
cudaError_t launch_tile_p(const TileGridArgs &g, cudaStream_t s) {
    if (g.a.ref_f32) return g.a.ssd ? launch_tile_t<PAT, true, true>(g, s) : launch_tile_t<PAT, false, true>(g, s);
    return g.a.ssd ? launch_tile_t<PAT, true, false>(g, s) : launch_tile_t<PAT, false, false>(g, s);
}

// ---------------------------------------------------------------------------
// RME decision from the dense reverse keys (argmin over u in rank order).
// ---------------------------------------------------------------------------
__global__ void rme_decide_kernel(RmeDecideArgs a) {
    const int gx = blockIdx.x * blockDim.x + threadIdx.x;
    const int gy = a.y0 + blockIdx.y;
    unsigned long long my_evals = 0;
    if (gx < a.W && gy < a.y1) {
        const int64_t fi = (int64_t)(gy - a.buf_y0) * a.f.pitch + gx;
        if (checkable(a.f.status[fi])) {
            const int va = a.f.alpha[fi], vb = a.f.beta[fi];
            const int xy = gy + va, xx = gx + vb;
            const unsigned long long key =
                a.keys[(int64_t)(xy - (a.y0 - a.S)) * a.key_pitch + (xx + a.S)];
            bool ok = false;
            if (key != ~0ull) {
                const int pk = __ldg(a.canon + (int)(key & 0xffffffffu));
                const int ua = (int)(int8_t)(pk & 0xff), ub = (int)(int8_t)((pk >> 8) & 0xff);
                ok = (ua == -va) && (ub == -vb);
            }
            a.f.status[fi] = ok ? kAccepted : kRejected;
            my_evals = (unsigned long long)a.n_cand;
        }
    }
    if (a.evals) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) my_evals += __shfl_down_sync(0xffffffffu, my_evals, o);
        if ((threadIdx.x & 31) == 0 && my_evals) atomicAdd(a.evals, my_evals);
    }
}

// ---------------------------------------------------------------------------
// Projection.
// ---------------------------------------------------------------------------
__global__ void project_kernel(ProjectArgs a) {
    const int gx = blockIdx.x * blockDim.x + threadIdx.x;
    const int gy = a.y0 + blockIdx.y;
    if (gx >= a.W || gy >= a.y1) return;
    const int64_t r = gy - a.buf_y0;
    const int64_t fi = r * a.f.pitch + gx;
    if (a.f.status[fi] != kAccepted) return;
    const int qy = gy + a.f.alpha[fi], qx = gx + a.f.beta[fi];
    if (qy < 0 || qy >= a.H || qx < 0 || qx >= a.W) return;
    if (qy < a.buf_y0 || qy >= a.buf_y0 + a.buf_rows) return;   // never for valid rois
    const int64_t qr = qy - a.buf_y0;
    if (!a.past_mask.p[qr * a.past_mask.pitch + qx]) return;
    const int64_t ai = r * a.acc_pitch + gx;
    a.sum[ai] += a.past_val.p[qr * a.past_val.pitch + qx];
    a.cnt[ai] += 1;
}

}  // namespace

cudaError_t launch_nnc(FieldView f, int W, int H, int buf_y0, int buf_rows, int y0, int y1, int threshold, int mode,
                       cudaStream_t s) {
    if (y1 <= y0) return cudaSuccess;
    dim3 blk(kNX, kNY), grd((W + kNX - 1) / kNX, (y1 - y0 + kNY - 1) / kNY);
    nnc_kernel<<<grd, blk, 0, s>>>(f, W, H, buf_y0, buf_rows, y0, y1, threshold, mode);
    return cudaGetLastError();
}

cudaError_t launch_revgrid(const RevGridArgs &a, cudaStream_t s) {
    if (a.y1 <= a.y0) return cudaSuccess;
    if (a.K == kFK) {
        TileGridArgs g{};
        g.a = a;
        bool paper = false;
        if (a.n_dy == 7) {
            int seen = 0;
            for (int i = 0; i < 7; ++i) {
                const int o = a.dys_host[i];
                const int idx = o == -7 ? 0 : o == -3 ? 1 : o == -1 ? 2 : o == 0 ? 3 : o == 1 ? 4 : o == 3 ? 5 : o == 7 ? 6 : -1;
                if (idx >= 0) seen |= 1 << idx;
            }
            paper = seen == 0x7f;
        }
        const int S = a.full_hi;
        // The paper's set extended by +-15: {0, +-1, +-3, +-7, +-15}.
        bool ext15 = false;
        if (a.n_dy == 9) {
            int seen = 0;
            for (int i = 0; i < 9; ++i) {
                const int o = a.dys_host[i];
                const int idx = o == -15 ? 0 : o == -7 ? 1 : o == -3 ? 2 : o == -1 ? 3 : o == 0 ? 4 : o == 1 ? 5
                              : o == 3 ? 6 : o == 7 ? 7 : o == 15 ? 8 : -1;
                if (idx >= 0) seen |= 1 << idx;
            }
            ext15 = seen == 0x1ff;
        }
        if (ext15) {
            g.n_dy = 9;
            const int8_t order[9] = {0, -1, 1, -3, 3, -7, 7, -15, 15};   // small offsets first
            for (int i = 0; i < 9; ++i) g.dys[i] = order[i];
            g.n_groups = 2;
            g.n_last = 2;
            g.maxd = 15;
            g.S = S;
            g.n_total = 81;
            return launch_tile_p<2>(g, s);
        }
        if (paper) {
            g.n_dy = 7;
            const int8_t order[7] = {0, -1, 1, -3, 3, -7, 7};   // the same set; small offsets first
            for (int i = 0; i < 7; ++i) g.dys[i] = order[i];
            g.n_groups = 1;
            g.n_last = 7;
            g.maxd = 7;
            g.S = S;
            g.n_total = 49;
            return launch_tile_p<0>(g, s);
        }
        if (a.n_dy == 0) {
            const int n = a.full_hi - a.full_lo + 1;
            g.n_dy = n;
            g.lo = a.full_lo;
            g.n_groups = (n + 6) / 7;
            g.n_last = n - 7 * (g.n_groups - 1);
            g.maxd = S;
            g.S = S;
            g.n_total = n * n;
            return launch_tile_p<1>(g, s);
        }
    }
    DeltaSet ds{};
    ds.n = a.n_dy;
    ds.lo = a.full_lo;
    ds.hi = a.full_hi;
    for (int i = 0; i < a.n_dy && i < 16; ++i) ds.v[i] = a.dys_host[i];
    dim3 blk(128), grd((a.W + 127) / 128, a.y1 - a.y0);
    revgrid_kernel<<<grd, blk, 0, s>>>(a, ds);
    return cudaGetLastError();
}

cudaError_t launch_rme_decide(const RmeDecideArgs &a, cudaStream_t s) {
    if (a.y1 <= a.y0) return cudaSuccess;
    dim3 blk(128), grd((a.W + 127) / 128, a.y1 - a.y0);
    rme_decide_kernel<<<grd, blk, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_project(const ProjectArgs &a, cudaStream_t s) {
    if (a.y1 <= a.y0) return cudaSuccess;
    dim3 blk(128), grd((a.W + 127) / 128, a.y1 - a.y0);
    project_kernel<<<grd, blk, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace qs
