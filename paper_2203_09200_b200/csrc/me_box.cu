// me_box.cu -- the K = 8 instantiations of the me_box kernels (the paper's configs), the launch
// dispatcher over K, and the finalize kernel.  The kernel templates live in me_box.cuh; the
// instantiations for other K are compiled in me_box_k*.cu (parallel build units).
#include "me_box.cuh"

namespace qs {
cudaError_t launch_box_k1_4(const BoxArgs &a, int K, bool ssd, bool reverse, cudaStream_t s);
cudaError_t launch_box_k5_9(const BoxArgs &a, int K, bool ssd, bool reverse, cudaStream_t s);
namespace {
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
    const int64_t fi = (int64_t)(gy - a.field_y0) * a.fpitch + gx;
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

cudaError_t launch_box(const BoxArgs &a0, int K, bool ssd, bool reverse, cudaStream_t s) {
    BoxArgs a = a0;
    if (a.n_ref <= 0) {   // one slot: (ref, keys)
        a.n_ref = 1;
        a.ref_p[0] = a.ref.p;
        a.keys_p[0] = a.keys;
        a.s2_p[0] = a.s2;
    }
    if (a.n_ref > kMaxRefs || (reverse && a.n_ref != 1)) return cudaErrorInvalidValue;
    for (int i = 0; i < a.n_ref; ++i)
        if (a.ref_f32 && !a.s2_p[i]) return cudaErrorInvalidValue;   // float keys need their second plane
    if (K == 8) return launch_k<8>(a, ssd, reverse, s);
    if (K >= 1 && K <= 4) return launch_box_k1_4(a, K, ssd, reverse, s);
    if (K >= 5 && K <= 9) return launch_box_k5_9(a, K, ssd, reverse, s);
    return cudaErrorInvalidValue;
}

cudaError_t launch_finalize(const FinalizeArgs &a, cudaStream_t s) {
    if (a.y1 <= a.y0) return cudaSuccess;
    dim3 blk(128), grd((a.W + 127) / 128, a.y1 - a.y0);
    finalize_kernel<<<grd, blk, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace qs
