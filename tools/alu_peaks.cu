// alu_peaks.cu -- per-SM issue rates of the instructions the hot path uses, measured on the
// box ("Peaks to measure on the box").  Each kernel runs independent
// dependency chains (8 per thread) of one instruction type at full occupancy; the rate is
// (thread-instructions executed) / (SM cycles) / (#SMs), i.e. lanes per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_peaks alu_peaks.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITER = 4096;
constexpr int CH = 8;

#define KERNEL(NAME, T, INIT, BODY)                                                     \
    __global__ void NAME(T *out, int seed) {                                            \
        T v[CH];                                                                        \
        _Pragma("unroll") for (int c = 0; c < CH; ++c) v[c] = INIT;                     \
        _Pragma("unroll 16") for (int i = 0; i < ITER; ++i) {                           \
            _Pragma("unroll") for (int c = 0; c < CH; ++c) { BODY; }                    \
        }                                                                               \
        T s = v[0];                                                                     \
        _Pragma("unroll") for (int c = 1; c < CH; ++c) s = s + v[c];                    \
        if (s == (T)seed) out[threadIdx.x] = s;                                         \
    }

// Integer / select kernels: one opaque PTX instruction per step on runtime operands (the round-1
// C++ bodies were folded by the compiler: IADD3 showed an impossible 2382 lanes/clk).  The SASS of
// each loop body is checked with cuobjdump (tools/alu_peaks_sass.txt): ptxas merges two dependent
// min.f32 / min.u32 into one 3-input FMNMX3 / VIMNMX3 (rate counted per SASS instruction, 0.5 per
// step), and splits dependent add.s32 between IADD3 (ALU pipe) and IMAD (FMA-heavy pipe).
#define AKERNEL(NAME, ASM)                                                               \
    __global__ void NAME(unsigned *out, int seed) {                                     \
        unsigned v[CH];                                                                 \
        const unsigned a = (unsigned)seed * 2654435761u, b = (unsigned)seed ^ 0x9e3779b9u; \
        _Pragma("unroll") for (int c = 0; c < CH; ++c) v[c] = threadIdx.x * 7919u + c;  \
        _Pragma("unroll 16") for (int i = 0; i < ITER; ++i) {                           \
            _Pragma("unroll") for (int c = 0; c < CH; ++c) asm volatile(ASM : "+r"(v[c]) : "r"(a), "r"(b)); \
        }                                                                               \
        unsigned s = v[0];                                                              \
        _Pragma("unroll") for (int c = 1; c < CH; ++c) s ^= v[c];                       \
        if (s == (unsigned)seed) out[threadIdx.x] = s;                                  \
    }

KERNEL(k_fadd, float, (float)(threadIdx.x + c), v[c] = __fadd_rn(v[c], 1.0001f * (c + 1)))
KERNEL(k_ffma, float, (float)(threadIdx.x + c), v[c] = __fmaf_rn(v[c], 0.9999f, 1.0f))
AKERNEL(k_fmnmx, "min.f32 %0, %0, %1;")
AKERNEL(k_iadd3, "add.s32 %0, %0, %1;\n\tadd.s32 %0, %0, %2;")
AKERNEL(k_lop3, "lop3.b32 %0, %0, %1, %2, 0x96;")
AKERNEL(k_prmt, "prmt.b32 %0, %0, %1, %2;")
AKERNEL(k_imnmx, "min.u32 %0, %0, %1;")
AKERNEL(k_imad, "mad.lo.u32 %0, %0, %1, %2;")
AKERNEL(k_vabsdiff4, "vabsdiff4.u32.u32.u32 %0, %0, %1, %2;")
AKERNEL(k_dp4a, "dp4a.u32.u32 %0, %1, %2, %0;")
AKERNEL(k_redux, "redux.sync.min.u32 %0, %0, 0xffffffff;")

__global__ void k_fadd2(unsigned long long *out, int seed) {
    unsigned long long v[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        float2 f = make_float2((float)(threadIdx.x + c), (float)(threadIdx.x + 2 * c));
        v[c] = *reinterpret_cast<unsigned long long *>(&f);
    }
    float2 one = make_float2(1.0001f, 1.0002f);
    const unsigned long long o = *reinterpret_cast<unsigned long long *>(&one);
#pragma unroll 16
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(v[c]) : "l"(o));
    }
    unsigned long long s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s ^= v[c];
    if (s == (unsigned long long)seed) out[threadIdx.x] = s;
}

__global__ void k_ffma2(unsigned long long *out, int seed) {
    unsigned long long v[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
        float2 f = make_float2((float)(threadIdx.x + c), (float)(threadIdx.x + 2 * c));
        v[c] = *reinterpret_cast<unsigned long long *>(&f);
    }
    float2 a = make_float2(0.9999f, 0.9998f), b = make_float2(1.f, 2.f);
    const unsigned long long ao = *reinterpret_cast<unsigned long long *>(&a), bo = *reinterpret_cast<unsigned long long *>(&b);
#pragma unroll 16
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(v[c]) : "l"(ao), "l"(bo));
    }
    unsigned long long s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s ^= v[c];
    if (s == (unsigned long long)seed) out[threadIdx.x] = s;
}

// Mixed: 2 FADD + 1 LOP3 per step (do the FMA and ALU pipes co-issue?)
__global__ void k_mix(float *out, int seed) {
    float f[CH];
    unsigned u[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) { f[c] = (float)(threadIdx.x + c); u[c] = threadIdx.x + c; }
#pragma unroll 16
    for (int i = 0; i < ITER; ++i) {
#pragma unroll
        for (int c = 0; c < CH; ++c) {
            f[c] = __fadd_rn(f[c], 1.0001f);
            u[c] = (u[c] ^ 0x5a5a5a5au) & (u[c] | 0x0f0f0f0fu);
        }
    }
    float s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += f[c] + (float)u[c];
    if (s == (float)seed) out[threadIdx.x] = s;
}

template <typename K, typename T>
double rate(K kern, double instr_per_step, const char *name, int sm_count, double clk_hz, T *buf, FILE *js, bool last) {
    const int threads = 256, blocks = sm_count * 8;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kern<<<blocks, threads>>>(buf, 12345);
    cudaEventRecord(a);
    kern<<<blocks, threads>>>(buf, 12345);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double thread_instr = (double)blocks * threads * ITER * CH * instr_per_step;
    const double per_sm_clk = thread_instr / (ms * 1e-3 * clk_hz) / sm_count;
    printf("%-10s %8.3f ms  %7.1f lanes/clk/SM\n", name, ms, per_sm_clk);
    fprintf(js, "  \"%s\": %.2f%s\n", name, per_sm_clk, last ? "" : ",");
    return per_sm_clk;
}

int main(int argc, char **argv) {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const double clk = (argc > 1 ? atof(argv[1]) : clk_khz / 1e3) * 1e6;   // MHz on the command line
    printf("%s, %d SMs, clock %.0f MHz (rates assume this clock)\n", p.name, p.multiProcessorCount, clk / 1e6);
    float *fb;
    unsigned long long *ub;
    cudaMalloc(&fb, 4096);
    cudaMalloc(&ub, 8192);
    FILE *js = fopen(argc > 2 ? argv[2] : "alu_peaks.json", "w");
    fprintf(js, "{\n  \"gpu\": \"%s\", \"sms\": %d, \"clock_mhz_assumed\": %.0f,\n  \"unit\": \"thread-instructions per clock per SM\",\n",
            p.name, p.multiProcessorCount, clk / 1e6);
    const int n = p.multiProcessorCount;
    rate(k_fadd, 1, "FADD", n, clk, fb, js, false);
    rate(k_ffma, 1, "FFMA", n, clk, fb, js, false);
    rate(k_fmnmx, 0.5, "FMNMX3", n, clk, (unsigned *)fb, js, false);
    rate(k_iadd3, 2, "IADD3+IMAD(add)", n, clk, (unsigned *)fb, js, false);
    rate(k_lop3, 1, "LOP3", n, clk, (unsigned *)fb, js, false);
    rate(k_prmt, 1, "PRMT", n, clk, (unsigned *)fb, js, false);
    rate(k_imnmx, 0.5, "VIMNMX3", n, clk, (unsigned *)fb, js, false);
    rate(k_imad, 1, "IMAD", n, clk, (unsigned *)fb, js, false);
    rate(k_vabsdiff4, 1, "VABSDIFF4", n, clk, (unsigned *)fb, js, false);
    rate(k_dp4a, 1, "IDP4A", n, clk, (unsigned *)fb, js, false);
    rate(k_redux, 1, "REDUX", n, clk, (unsigned *)fb, js, false);
    rate(k_fadd2, 1, "FADD2", n, clk, ub, js, false);
    rate(k_ffma2, 1, "FFMA2", n, clk, ub, js, false);
    rate(k_mix, 2, "FADD+LOP3", n, clk, fb, js, true);
    fprintf(js, "}\n");
    fclose(js);
    return 0;
}
