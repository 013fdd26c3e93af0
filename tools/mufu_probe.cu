// Probe: MUFU ex2 and FMA-pipe throughput per SM on this B200 (exps / clk / SM), for the attention softmax
// ceiling.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu tools/mufu_probe.cu && /tmp/mufu
#include <cstdio>
#include <cuda_runtime.h>
#include <cstdint>

template <int MODE>
__global__ void k(float* out, int iters) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
            else if (MODE == 1) asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0fBA83126F;" : "+f"(a[i]));
            else if (MODE == 2) {   // packed half2: two exps per instruction
                uint32_t v = __float_as_uint(a[i]);
                asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(v));
                a[i] = __uint_as_float(v);
            } else if (MODE == 3) {   // packed bf16x2
                uint32_t v = __float_as_uint(a[i]);
                asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(v));
                a[i] = __uint_as_float(v);
            } else if (MODE == 4) {   // cvt.rn.bf16x2.f32 (the attention softmax's P packing): pipe and rate
                uint32_t v;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(v) : "f"(a[i]), "f"(a[(i + 1) & 15]));
                a[i] = __uint_as_float(v ^ 0x3f800000u);
            } else {                  // one ex2 + one bf16x2 cvt per element: do they share a pipe?
                float e;
                asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(a[i]));
                uint32_t v;
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(v) : "f"(e), "f"(a[(i + 1) & 15]));
                a[i] = __uint_as_float(v ^ 0x3f800000u);
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += a[i];
    if (s == 12345.f) out[0] = s;
}

int main() {
    float* d;
    cudaMalloc(&d, 4);
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int iters = 4096;
    for (int mode = 0; mode < 6; ++mode)
        for (int tpb : {128, 256, 512, 1024}) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            auto kk = mode == 0 ? k<0> : mode == 1 ? k<1> : mode == 2 ? k<2> : mode == 3 ? k<3> : mode == 4 ? k<4> : k<5>;
            kk<<<sms * 2, tpb>>>(d, 16);
            cudaEventRecord(e0);
            kk<<<sms * 2, tpb>>>(d, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ops = (double)sms * 2 * tpb * iters * 16 * (mode == 2 || mode == 3 ? 2 : 1);   // exps (2 per packed op); mode 4: cvt instructions
            const double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
            printf("%s threads/CTA %4d (2 CTAs/SM): %.1f ops/clk/SM (at the %d MHz rated clock)\n",
                   mode == 0 ? "ex2.approx.ftz.f32   " : mode == 1 ? "fma.rn.f32           " : mode == 2 ? "ex2.approx.f16x2 (x2)" : mode == 3 ? "ex2.bf16x2 (x2)      " : mode == 4 ? "cvt.rn.bf16x2.f32    " : "ex2 + cvt (ex2 rate) ", tpb, per_clk_sm, clk / 1000);
        }
    return 0;
}
