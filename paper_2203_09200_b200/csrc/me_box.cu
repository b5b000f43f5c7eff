// me_box.cu -- K1/K2 "me_box": exhaustive template-matching motion estimation
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
#include <cfloat>
#include <cmath>

#include "qs_internal.cuh"

namespace qs {
namespace {

// B/A loaders: float value or NaN ("no term").
// Rows outside the frame, or outside the caller's buffer window, give NaN.
__device__ __forceinline__ float load_ref(const BoxArgs &a, int y, int x) {
    if (y < 0 || y >= a.H || x < 0 || x >= a.W || y < a.buf_y0 || y >= a.buf_y0 + a.buf_rows)
        return __int_as_float(0x7fc00000);
    const int64_t off = (int64_t)(y - a.buf_y0) * a.ref.pitch;
    if (a.ref_f32) return reinterpret_cast<const float *>(a.ref.p + off)[x];
    return (float)a.ref.p[off + x];
}

__device__ __forceinline__ float load_cur_masked(const BoxArgs &a, int y, int x) {
    if (y < 0 || y >= a.H || x < 0 || x >= a.W || y < a.buf_y0 || y >= a.buf_y0 + a.buf_rows)
        return __int_as_float(0x7fc00000);
    const int64_t r = (int64_t)(y - a.buf_y0);
    if (!a.mask.p[r * a.mask.pitch + x]) return __int_as_float(0x7fc00000);
    return (float)a.cur.p[r * a.cur.pitch + x];
}

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
__device__ __forceinline__ void box_body(const BoxArgs &a, float *smem, int chunk, int px0, int py0) {
    using G = BoxGeom<K>;
    const int alo = -a.S + chunk * kChunkRows;
    const int ahi = min(a.S, alo + kChunkRows - 1);
    const int nrow_b = G::HR + (ahi - alo);
    const int ncol_b = kTX + K - 1 + 2 * a.S;
    const int bpitch = ncol_b | 1;
    float *Bw = smem;
    float *Hs = smem + ((nrow_b * bpitch + 3) & ~3);
    float *Ns = Hs + 2 * G::HR * kTXP;

    // Stage the chunk's B window: rows py0-KL+alo .., cols px0-KL-S ..
    const int by0 = py0 - G::KL + alo, bx0 = px0 - G::KL - a.S;
    for (int i = threadIdx.x; i < nrow_b * ncol_b; i += kNT) {
        const int r = i / ncol_b, c = i - r * ncol_b;
        Bw[r * bpitch + c] = REV ? load_cur_masked(a, by0 + r, bx0 + c) : load_ref(a, by0 + r, bx0 + c);
    }

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
    float be[kSeg], bn[kSeg];
    int br[kSeg];
#pragma unroll
    for (int i = 0; i < kSeg; ++i) { be[i] = INFINITY; bn[i] = 1.f; br[i] = -1; }
    const float ms = (float)a.min_support;

    __syncthreads();
    const int k0 = a.chunk_off[chunk], k1 = a.chunk_off[chunk + 1];
    for (int k = k0; k < k1; ++k) {
        const int pk = __ldg(a.chunked + k);
        const int al = (int)(int8_t)(pk & 0xff);
        const int bt = (int)(int8_t)((pk >> 8) & 0xff);
        const int rank = pk >> 16;
        const int buf = (k - k0) & 1;
        float *Hb = Hs + buf * G::HR * kTXP;
        float *Nb = Ns + buf * G::HR * kTXP;
        if (actA) {
            const float *brow = Bw + (ya + al - alo) * bpitch + xa0 + bt + a.S;
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
            if constexpr (CNT) {
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
            if constexpr (!CNT) {
#pragma unroll
                for (int i = 0; i < kSeg; ++i)
                    if (e[i] < be[i]) { be[i] = e[i]; br[i] = rank; }
            } else {
                const float *nc = Nb + (sb * kSeg) * kTXP + xb;
                float nvv[G::NB];
#pragma unroll
                for (int j = 0; j < G::NB; ++j) nvv[j] = nc[j * kTXP];
                float n[kSeg];
                box_sum<K, kSeg, true>(nvv, n);
#pragma unroll
                for (int i = 0; i < kSeg; ++i) {
                    if (n[i] >= ms) {
                        if constexpr (!EXACT) {
                            const float m = __fdiv_rn(e[i], n[i]);    // fl(e/n), R23
                            if (m < be[i]) { be[i] = m; br[i] = rank; }
                        } else if constexpr (SSD) {
                            if ((double)e[i] * (double)bn[i] < (double)be[i] * (double)n[i]) {
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
        if (br[i] < 0 || py >= a.oy1 || px >= a.ox1) continue;
        unsigned long long hi;
        if constexpr (!CNT || !EXACT) {
            hi = __float_as_uint(be[i]);                 // e (interior) or fl(e/n): non-negative floats
        } else {
            // floor(e * 2^13 / n): distinct means with n <= 81 differ by >= 1/6561 > 2^-13,
            // equal means give equal keys; fp64 division of exact integers cannot round
            // across an integer boundary at these magnitudes.
            hi = (unsigned long long)floor((double)be[i] * 8192.0 / (double)bn[i]);
        }
        const unsigned long long key = (hi << 32) | (unsigned)br[i];
        atomicMin(a.keys + (int64_t)(py - a.oy0) * a.key_pitch + (px - a.ox0), key);
    }
}

template <int K, bool EXACT, bool SSD, bool REV>
__global__ void __launch_bounds__(kNT, 2) box_kernel(const BoxArgs a) {
    extern __shared__ __align__(16) float smem[];
    const int unit = blockIdx.x;
    const int chunk = unit % a.n_chunks;
    const int tile = unit / a.n_chunks;
    const int txi = tile % a.tiles_x, tyi = tile / a.tiles_x;
    const int px0 = a.ox0 + txi * kTX, py0 = a.oy0 + tyi * kTY;
    constexpr int KL = K / 2, KR = K - 1 - K / 2;
    bool interior = !REV && (py0 - KL - a.S >= 0) && (py0 + kTY - 1 + KR + a.S <= a.H - 1) &&
                    (px0 - KL - a.S >= 0) && (px0 + kTX - 1 + KR + a.S <= a.W - 1);
    if constexpr (REV) {
        box_body<K, EXACT, true, SSD, true>(a, smem, chunk, px0, py0);
    } else {
        if (interior) box_body<K, EXACT, false, SSD, false>(a, smem, chunk, px0, py0);
        else box_body<K, EXACT, true, SSD, false>(a, smem, chunk, px0, py0);
    }
}

template <int K, bool EXACT, bool SSD, bool REV>
cudaError_t launch_t(const BoxArgs &a, cudaStream_t s) {
    using G = BoxGeom<K>;
    const int nrow_b = G::HR + kChunkRows - 1;
    const int bpitch = (kTX + K - 1 + 2 * a.S) | 1;
    const size_t smem = sizeof(float) * ((size_t)((nrow_b * bpitch + 3) & ~3) + 4 * (size_t)G::HR * kTXP);
    auto fn = box_kernel<K, EXACT, SSD, REV>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const long long units = (long long)a.tiles_x * a.tiles_y * a.n_chunks;
    if (units <= 0) return cudaSuccess;
    fn<<<(unsigned)units, kNT, smem, s>>>(a);
    return cudaGetLastError();
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

// ---------------------------------------------------------------------------
// Finalize: key -> (alpha, beta); the chosen vector's (e, n) re-summed in the
// definition's row-major order (R23: fp32 d = fl(c - r), |d| or fl(d*d),
// fp32 accumulation), status CANDIDATE / INVALID / NOT_TARGET.
// ---------------------------------------------------------------------------
__global__ void finalize_kernel(const FinalizeArgs a) {
    const int gx = blockIdx.x * blockDim.x + threadIdx.x;
    const int gy = a.y0 + blockIdx.y;
    if (gx >= a.W || gy >= a.y1) return;
    const int64_t r = gy - a.buf_y0;
    const int64_t fi = r * a.fpitch + gx;
    int8_t al = 0, bt = 0;
    uint8_t st = kNotTarget, cnt = 0;
    uint32_t eu = 0;
    float ef = 0.f;
    if (!a.mask.p[r * a.mask.pitch + gx]) {
        st = kInvalid;
        const unsigned long long key = a.keys[(int64_t)(gy - a.y0) * a.key_pitch + gx];
        if (key != ~0ull) {
            const int pk = __ldg(a.canon + (int)(key & 0xffffffffu));
            const int va = (int)(int8_t)(pk & 0xff), vb = (int)(int8_t)((pk >> 8) & 0xff);
            const int KL = a.K / 2;
            int n = 0;
            for (int oy = -KL; oy < a.K - KL; ++oy) {
                const int qy = gy + oy;
                if (qy < 0 || qy >= a.H || qy + va < 0 || qy + va >= a.H) continue;
                if (qy < a.buf_y0 || qy >= a.buf_y0 + a.buf_rows) continue;            // never for valid rois
                if (qy + va < a.buf_y0 || qy + va >= a.buf_y0 + a.buf_rows) continue;
                const int64_t qr = qy - a.buf_y0, sr = qy + va - a.buf_y0;
                for (int ox = -KL; ox < a.K - KL; ++ox) {
                    const int qx = gx + ox;
                    if (qx < 0 || qx >= a.W || qx + vb < 0 || qx + vb >= a.W) continue;
                    if (!a.mask.p[qr * a.mask.pitch + qx]) continue;
                    const int c = a.cur.p[qr * a.cur.pitch + qx];
                    if (a.ref_f32) {
                        const float rv = reinterpret_cast<const float *>(a.ref.p + sr * a.ref.pitch)[qx + vb];
                        const float d = __fsub_rn((float)c, rv);
                        ef = __fadd_rn(ef, a.ssd ? __fmul_rn(d, d) : fabsf(d));
                    } else {
                        const int d = c - (int)a.ref.p[sr * a.ref.pitch + qx + vb];
                        eu += (uint32_t)(a.ssd ? d * d : (d < 0 ? -d : d));
                    }
                    ++n;
                }
            }
            if (n >= a.min_support) {
                st = kCandidate;
                al = (int8_t)va;
                bt = (int8_t)vb;
                cnt = (uint8_t)n;
            } else {
                eu = 0;
                ef = 0.f;
            }
        }
    }
    a.alpha[fi] = al;
    a.beta[fi] = bt;
    a.count[fi] = cnt;
    a.status[fi] = st;
    if (a.ref_f32) reinterpret_cast<float *>(a.err)[fi] = (st == kCandidate) ? ef : 0.f;
    else reinterpret_cast<uint32_t *>(a.err)[fi] = (st == kCandidate) ? eu : 0u;
}

}  // namespace

cudaError_t launch_box(const BoxArgs &a, int K, bool ssd, bool reverse, cudaStream_t s) {
    switch (K) {
        case 1: return launch_k<1>(a, ssd, reverse, s);
        case 2: return launch_k<2>(a, ssd, reverse, s);
        case 3: return launch_k<3>(a, ssd, reverse, s);
        case 4: return launch_k<4>(a, ssd, reverse, s);
        case 5: return launch_k<5>(a, ssd, reverse, s);
        case 6: return launch_k<6>(a, ssd, reverse, s);
        case 7: return launch_k<7>(a, ssd, reverse, s);
        case 8: return launch_k<8>(a, ssd, reverse, s);
        case 9: return launch_k<9>(a, ssd, reverse, s);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_finalize(const FinalizeArgs &a, cudaStream_t s) {
    if (a.y1 <= a.y0) return cudaSuccess;
    dim3 blk(128), grd((a.W + 127) / 128, a.y1 - a.y0);
    finalize_kernel<<<grd, blk, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace qs
