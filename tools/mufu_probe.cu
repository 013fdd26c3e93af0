// Probe: MUFU ex2 and FMA-pipe throughput per SM on this B200 (exps / clk / SM), for the attention softmax
// ceiling.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu tools/mufu_probe.cu && /tmp/mufu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(float* out, int iters) {
    float a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
            else asm volatile("fma.rn.f32 %0, %0, 0f3F7FFFFF, 0fBA83126F;" : "+f"(a[i]));
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
    for (int mode = 0; mode < 2; ++mode)
        for (int tpb : {128, 256, 512, 1024}) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            auto kk = mode == 0 ? k<0> : k<1>;
            kk<<<sms * 2, tpb>>>(d, 16);
            cudaEventRecord(e0);
            kk<<<sms * 2, tpb>>>(d, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ops = (double)sms * 2 * tpb * iters * 16;
            const double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
            printf("%s threads/CTA %4d (2 CTAs/SM): %.1f ops/clk/SM (at the %d MHz rated clock)\n",
                   mode == 0 ? "ex2.approx.ftz.f32" : "fma.rn.f32        ", tpb, per_clk_sm, clk / 1000);
        }
    return 0;
}
