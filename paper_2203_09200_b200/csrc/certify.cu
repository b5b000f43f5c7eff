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
// here exactly as the definition states it -- every candidate in rank order, terms row-major,
// fp32 sums, fl(e/n), strict '<' -- by one warp (lanes over the candidates, a 64-bit
// (mean bits, rank) min across lanes), and its key is overwritten.  Forward keys: targets
// (cur_mask = 0).  Reverse keys (RME, R9/R10): every x of the dense reverse domain.
#include "qs_internal.cuh"

namespace qs {
namespace {

constexpr int kMaxSlots = 81;   // K <= 9

__device__ __forceinline__ bool row_ok(const CertifyArgs &a, int y) {
    return y >= 0 && y < a.H && y >= a.buf_y0 && y < a.buf_y0 + a.buf_rows;
}

__global__ void __launch_bounds__(256) certify_kernel(const CertifyArgs a) {
    __shared__ float sv[8][kMaxSlots];   // per warp: the fixed side's window values (row-major slots)
    __shared__ int sq[8][kMaxSlots];     // per warp: their offsets (oy + 16) | (ox + 16) << 8
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int z = blockIdx.z;
    const int py = a.oy0 + blockIdx.y * 8 + w;
    const int px = a.ox0 + blockIdx.x * 32 + lane;
    unsigned long long *keys = a.keys_p[z];
    const unsigned *s2 = a.s2_p[z];
    const uint8_t *refp = a.ref_p[z];
    bool unc = false;
    if (py < a.oy1 && px < a.ox1) {
        const bool target = a.reverse || !a.mask.p[(int64_t)(py - a.buf_y0) * a.mask.pitch + px];
        if (target) {
            const int64_t o = (int64_t)(py - a.oy0) * a.key_pitch + (px - a.ox0);
            const unsigned long long k = keys[o];
            const unsigned v2 = s2[o];
            if (k != ~0ull && v2 != 0xffffffffu)
                unc = !(__uint_as_float(v2) > __uint_as_float((unsigned)(k >> 32)) * (1.0f + kCertEps));
        }
    }
    unsigned todo = __ballot_sync(0xffffffffu, unc);
    if (todo && a.rechecked && lane == 0) atomicAdd(a.rechecked, (unsigned long long)__popc(todo));
    const int KL = a.K / 2, nslot = a.K * a.K;
    while (todo) {
        const int j = __ffs(todo) - 1;
        todo &= todo - 1;
        const int x = a.ox0 + blockIdx.x * 32 + j, y = py;
        // Slot list of the fixed side, row-major (the definition's term order), kept in order by ballots.
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
                        // forward: measured current pixels only (R5)
                        ok = a.mask.p[r * a.mask.pitch + qx] != 0;
                        v = (float)a.cur.p[r * a.cur.pitch + qx];
                    } else {
                        // reverse: the dense reference template at x (R9)
                        ok = true;
                        v = reinterpret_cast<const float *>(refp + r * a.ref.pitch)[qx];
                    }
                }
            }
            const unsigned b = __ballot_sync(0xffffffffu, ok);
            if (ok) {
                const int pos = base + __popc(b & ((1u << lane) - 1u));
                sv[w][pos] = v;
                sq[w][pos] = (oy + 16) | ((ox + 16) << 8);
            }
            base += __popc(b);
        }
        __syncwarp();
        const int m = base;
        unsigned long long best = ~0ull;
        for (int rk = lane; rk < a.n_cand; rk += 32) {
            const int pk = __ldg(a.canon + rk);
            const int va = (int)(int8_t)(pk & 0xff), vb = (int)(int8_t)((pk >> 8) & 0xff);
            float e = 0.f;
            int n = 0;
            for (int i = 0; i < m; ++i) {
                const int q = sq[w][i];
                const int sy = y + (q & 0xff) - 16 + va, sx = x + ((q >> 8) & 0xff) - 16 + vb;
                if (!row_ok(a, sy) || sx < 0 || sx >= a.W) continue;
                const int64_t r = (int64_t)(sy - a.buf_y0);
                float d;
                if (!a.reverse) {
                    d = __fsub_rn(sv[w][i], reinterpret_cast<const float *>(refp + r * a.ref.pitch)[sx]);
                } else {
                    if (!a.mask.p[r * a.mask.pitch + sx]) continue;
                    d = __fsub_rn(sv[w][i], (float)a.cur.p[r * a.cur.pitch + sx]);
                }
                e = __fadd_rn(e, a.ssd ? __fmul_rn(d, d) : fabsf(d));
                ++n;
            }
            if (n < a.min_support) continue;
            const float mean = __fdiv_rn(e, (float)n);
            const unsigned long long key = ((unsigned long long)__float_as_uint(mean) << 32) | (unsigned)rk;
            best = key < best ? key : best;
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            const unsigned long long o = __shfl_xor_sync(0xffffffffu, best, off);
            best = o < best ? o : best;
        }
        if (lane == 0 && best != ~0ull) keys[(int64_t)(y - a.oy0) * a.key_pitch + (x - a.ox0)] = best;
        __syncwarp();
    }
}

}  // namespace

cudaError_t launch_certify(const CertifyArgs &a, cudaStream_t s) {
    if (a.oy1 <= a.oy0 || a.ox1 <= a.ox0 || a.n_ref <= 0) return cudaSuccess;
    if (a.n_ref > kMaxRefs || a.K < 1 || a.K > 9) return cudaErrorInvalidValue;
    dim3 grd((a.ox1 - a.ox0 + 31) / 32, (a.oy1 - a.oy0 + 7) / 8, a.n_ref);
    certify_kernel<<<grd, 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace qs

namespace qs {
namespace {
__device__ unsigned long long g_rechecked;   // outputs recomputed exactly since the last reset
}  // namespace

unsigned long long *rechecked_counter() {
    void *p = nullptr;
    if (cudaGetSymbolAddress(&p, g_rechecked) != cudaSuccess) return nullptr;
    return static_cast<unsigned long long *>(p);
}
}  // namespace qs
