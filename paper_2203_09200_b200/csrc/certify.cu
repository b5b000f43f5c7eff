// certify.cu -- K2c "certify": the certificate of the float-reference argmin and the exact
// recompute of the outputs it cannot certify.
//
// me_box sums float costs in a blocked order (and keys them with a truncated mantissa), so its
// winner could differ from the definition's (§2.2; R1, R7, R23: fp32 terms
// d = fl(c - r), |d| or fl(d*d), accumulated in row-major template order, compared by fl(e/n),
// ties by rank) only where another candidate's approximate mean lies within the error band of the
// winner's.  me_box leaves, per output, the winner's key (approximate value, rank) and the
// smallest approximate value of every OTHER candidate (the second plane).  An output is
// certified iff  second > winner * (1 + 2^-13):  with both approximations within 2^-14 + 2^-17
// relative of the definition's means, every other candidate's definitional mean is then strictly
// larger than the winner's, so the winner is the definition's.  Every other output is recomputed
// exactly as the definition states it -- every candidate in rank order, terms row-major, fp32
// sums, fl(e/n), strict '<' (a (mean bits, rank) minimum) -- and its key is overwritten.
// Forward keys: targets (cur_mask = 0).  Reverse keys (RME, R9/R10): every x of the dense domain.
//
// Two kernels: certify_scan tests every output and appends the uncertain ones to a list in the
// workspace (a full list falls back to an in-place warp recompute, so the result never depends on
// the list's capacity); certify_fix, a grid of a few CTAs per SM, takes the list one output per
// CTA: the output's search window is staged in shared memory once and the CTA's 256 threads split
// the candidates.
#include <algorithm>
#include <cmath>

#include "qs_internal.cuh"

namespace qs {
namespace {

__device__ unsigned long long g_rechecked;   // outputs recomputed exactly since the last reset

constexpr int kMaxSlots = 81;                // K <= 9
constexpr int kMaxSpan = 9 + 2 * 32;         // K + 2S

__device__ __forceinline__ bool row_ok(const CertifyArgs &a, int y) {
    return y >= 0 && y < a.H && y >= a.buf_y0 && y < a.buf_y0 + a.buf_rows;
}
__device__ __forceinline__ float ref_at(const CertifyArgs &a, int z, int y, int x) {
    return reinterpret_cast<const float *>(a.ref_p[z] + (int64_t)(y - a.buf_y0) * a.ref.pitch)[x];
}
__device__ __forceinline__ unsigned long long kmin(unsigned long long p, unsigned long long q) { return p < q ? p : q; }

// Term of slot value c and window value w (NaN = no term), accumulated in the caller's order.
__device__ __forceinline__ void add_term(float c, float w, int ssd, float &e, int &n) {
    if (w == w) {
        const float d = __fsub_rn(c, w);
        e = __fadd_rn(e, ssd ? __fmul_rn(d, d) : fabsf(d));
        ++n;
    }
}

// The slow path (list full): one warp recomputes output (y, x) of slot z from global memory.
__device__ void warp_recompute(const CertifyArgs &a, int z, int y, int x, float *sv, int *sq) {
    const int lane = threadIdx.x & 31, KL = a.K / 2, nslot = a.K * a.K;
    int base = 0;
    for (int s0 = 0; s0 < nslot; s0 += 32) {
        const int sidx = s0 + lane;
        bool ok = false;
        float v = 0.f;
        int oy = 0, ox = 0;
        if (sidx < nslot) {
            oy = sidx / a.K - KL;
            ox = sidx % a.K - KL;
            const int qy = y + oy, qx = x + ox;
            if (row_ok(a, qy) && qx >= 0 && qx < a.W) {
                const int64_t r = (int64_t)(qy - a.buf_y0);
                if (!a.reverse) {
                    ok = a.mask.p[r * a.mask.pitch + qx] != 0;   // measured current pixels (R5)
                    v = (float)a.cur.p[r * a.cur.pitch + qx];
                } else {
                    ok = true;                                    // dense reference template (R9)
                    v = ref_at(a, z, qy, qx);
                }
            }
        }
        const unsigned b = __ballot_sync(0xffffffffu, ok);
        if (ok) {
            const int pos = base + __popc(b & ((1u << lane) - 1u));
            sv[pos] = v;
            sq[pos] = (oy + 16) | ((ox + 16) << 8);
        }
        base += __popc(b);
    }
    __syncwarp();
    unsigned long long best = ~0ull;
    for (int rk = lane; rk < a.n_cand; rk += 32) {
        const int pk = __ldg(a.canon + rk);
        const int va = (int)(int8_t)(pk & 0xff), vb = (int)(int8_t)((pk >> 8) & 0xff);
        float e = 0.f;
        int n = 0;
        for (int i = 0; i < base; ++i) {
            const int q = sq[i];
            const int sy = y + (q & 0xff) - 16 + va, sx = x + ((q >> 8) & 0xff) - 16 + vb;
            if (!row_ok(a, sy) || sx < 0 || sx >= a.W) continue;
            float w;
            if (!a.reverse) {
                w = ref_at(a, z, sy, sx);
            } else {
                const int64_t r = (int64_t)(sy - a.buf_y0);
                w = a.mask.p[r * a.mask.pitch + sx] ? (float)a.cur.p[r * a.cur.pitch + sx] : __int_as_float(0x7fc00000);
            }
            add_term(sv[i], w, a.ssd, e, n);
        }
        if (n < a.min_support) continue;
        best = kmin(best, ((unsigned long long)__float_as_uint(__fdiv_rn(e, (float)n)) << 32) | (unsigned)rk);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) best = kmin(best, __shfl_xor_sync(0xffffffffu, best, off));
    if (lane == 0 && best != ~0ull) a.keys_p[z][(int64_t)(y - a.oy0) * a.key_pitch + (x - a.ox0)] = best;
    __syncwarp();
}

__global__ void __launch_bounds__(256) certify_scan_kernel(const CertifyArgs a) {
    __shared__ float sv[8][kMaxSlots];
    __shared__ int sq[8][kMaxSlots];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int z = blockIdx.z;
    const int py = a.oy0 + blockIdx.y * 8 + w;
    const int px = a.ox0 + blockIdx.x * 32 + lane;
    bool unc = false;
    if (py < a.oy1 && px < a.ox1) {
        const bool target = a.reverse || !a.mask.p[(int64_t)(py - a.buf_y0) * a.mask.pitch + px];
        if (target) {
            const int64_t o = (int64_t)(py - a.oy0) * a.key_pitch + (px - a.ox0);
            const unsigned long long k = a.keys_p[z][o];
            const unsigned v2 = a.s2_p[z][o];
            if (k != ~0ull && v2 != 0xffffffffu)
                unc = !(__uint_as_float(v2) > __uint_as_float((unsigned)(k >> 32)) * (1.0f + kCertEps));
        }
    }
    const unsigned todo = __ballot_sync(0xffffffffu, unc);
    if (!todo) return;
    if (lane == 0) atomicAdd(&g_rechecked, (unsigned long long)__popc(todo));
    // Append to the list; what does not fit is recomputed here.
    bool overflow = false;
    if (unc) {
        const unsigned idx = atomicAdd(a.list_count, 1u);
        if (idx < (unsigned)a.list_cap)
            a.list[idx] = ((unsigned)z << 30) | ((unsigned)(py - a.oy0) << 16) | (unsigned)(px - a.ox0);
        else
            overflow = true;
    }
    unsigned slow = __ballot_sync(0xffffffffu, overflow);
    while (slow) {
        const int j = __ffs(slow) - 1;
        slow &= slow - 1;
        warp_recompute(a, z, py, a.ox0 + blockIdx.x * 32 + j, sv[w], sq[w]);
    }
}

__global__ void __launch_bounds__(256) certify_fix_kernel(const CertifyArgs a) {
    __shared__ float win[kMaxSpan * kMaxSpan];   // the output's search window (NaN = no term)
    __shared__ float cval[kMaxSlots];            // fixed side of the template, row-major slots
    __shared__ int cpos[kMaxSlots];              // their window offsets at candidate (0, 0)
    __shared__ int nsl;
    __shared__ unsigned long long red[8];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int KL = a.K / 2, nslot = a.K * a.K, span = a.K + 2 * a.S;
    const unsigned n_items = min(*a.list_count, (unsigned)a.list_cap);
    for (unsigned it = blockIdx.x; it < n_items; it += gridDim.x) {
        const unsigned ent = a.list[it];
        const int z = (int)(ent >> 30);
        const int y = a.oy0 + (int)((ent >> 16) & 0x3fffu), x = a.ox0 + (int)(ent & 0xffffu);
        const int wy0 = y - KL - a.S, wx0 = x - KL - a.S;
        // Stage the window: forward = the reference around p, reverse = the measured current frame
        // around x (NaN outside the frame / buffer and, reverse, at unmeasured pixels).
        for (int i = tid; i < span * span; i += 256) {
            const int r = i / span, c = i - r * span;
            const int gy = wy0 + r, gx = wx0 + c;
            float v = __int_as_float(0x7fc00000);
            if (row_ok(a, gy) && gx >= 0 && gx < a.W) {
                if (!a.reverse) {
                    v = ref_at(a, z, gy, gx);
                } else {
                    const int64_t rr = (int64_t)(gy - a.buf_y0);
                    if (a.mask.p[rr * a.mask.pitch + gx]) v = (float)a.cur.p[rr * a.cur.pitch + gx];
                }
            }
            win[i] = v;
        }
        // The template's fixed side in row-major slot order (ballot compaction keeps the order).
        if (w == 0) {
            int base = 0;
            for (int s0 = 0; s0 < nslot; s0 += 32) {
                const int sidx = s0 + lane;
                bool ok = false;
                float v = 0.f;
                int pos = 0;
                if (sidx < nslot) {
                    const int oy = sidx / a.K - KL, ox = sidx % a.K - KL;
                    const int qy = y + oy, qx = x + ox;
                    pos = (oy + KL + a.S) * span + (ox + KL + a.S);
                    if (row_ok(a, qy) && qx >= 0 && qx < a.W) {
                        const int64_t r = (int64_t)(qy - a.buf_y0);
                        if (!a.reverse) {
                            ok = a.mask.p[r * a.mask.pitch + qx] != 0;
                            v = (float)a.cur.p[r * a.cur.pitch + qx];
                        } else {
                            ok = true;
                            v = ref_at(a, z, qy, qx);
                        }
                    }
                }
                const unsigned b = __ballot_sync(0xffffffffu, ok);
                if (ok) {
                    const int k = base + __popc(b & ((1u << lane) - 1u));
                    cval[k] = v;
                    cpos[k] = pos;
                }
                base += __popc(b);
            }
            if (lane == 0) nsl = base;
        }
        __syncthreads();
        const int m = nsl;
        unsigned long long best = ~0ull;
        for (int rk = tid; rk < a.n_cand; rk += 256) {
            const int pk = __ldg(a.canon + rk);
            const int off = (int)(int8_t)(pk & 0xff) * span + (int)(int8_t)((pk >> 8) & 0xff);
            float e = 0.f;
            int n = 0;
            for (int i = 0; i < m; ++i) {
                QS_DCHECK(cpos[i] + off >= 0 && cpos[i] + off < span * span);
                add_term(cval[i], win[cpos[i] + off], a.ssd, e, n);
            }
            if (n < a.min_support) continue;
            best = kmin(best, ((unsigned long long)__float_as_uint(__fdiv_rn(e, (float)n)) << 32) | (unsigned)rk);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = kmin(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0) red[w] = best;
        __syncthreads();
        if (tid == 0) {
            unsigned long long b = red[0];
#pragma unroll
            for (int i = 1; i < 8; ++i) b = kmin(b, red[i]);
            if (b != ~0ull) a.keys_p[z][(int64_t)(y - a.oy0) * a.key_pitch + (x - a.ox0)] = b;
        }
        __syncthreads();   // the window and slot arrays are rewritten for the next output
    }
}

}  // namespace

cudaError_t launch_certify(const CertifyArgs &a, cudaStream_t s) {
    if (a.oy1 <= a.oy0 || a.ox1 <= a.ox0 || a.n_ref <= 0) return cudaSuccess;
    if (a.n_ref > kMaxRefs || a.K < 1 || a.K > 9 || a.S > 32 || a.oy1 - a.oy0 > 0x3fff || a.ox1 - a.ox0 > 0xffff)
        return cudaErrorInvalidValue;
    cudaError_t e = cudaMemsetAsync(a.list_count, 0, sizeof(unsigned), s);
    if (e != cudaSuccess) return e;
    dim3 grd((a.ox1 - a.ox0 + 31) / 32, (a.oy1 - a.oy0 + 7) / 8, a.n_ref);
    certify_scan_kernel<<<grd, 256, 0, s>>>(a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = std::max(1, std::min(a.list_cap, 4 * sms));
    certify_fix_kernel<<<blocks, 256, 0, s>>>(a);
    return cudaGetLastError();
}

unsigned long long *rechecked_counter() {
    void *p = nullptr;
    if (cudaGetSymbolAddress(&p, g_rechecked) != cudaSuccess) return nullptr;
    return static_cast<unsigned long long *>(p);
}

}  // namespace qs
