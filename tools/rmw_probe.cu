// Ceiling probe for the fused replay+scan traffic: per unit (one (tree, head)) load a 32 KB state
// block + 8 KB x tile with 1-D bulk copies, store the 32 KB state back in place and 8 KB "y" to a
// separate buffer; 144 CTAs x 9 units per launch, 8 rotating layers, launches back to back.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/rmw_probe tools/rmw_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c)); }
__device__ __forceinline__ void expect_tx(uint32_t b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n) : "memory");
}
__device__ __forceinline__ void mwait(uint32_t b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(b), "r"(ph) : "memory");
}
__device__ __forceinline__ void ld(uint32_t dst, const void* src, uint32_t n, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"((uint64_t)src), "r"(n), "r"(bar) : "memory");
}
__device__ __forceinline__ void st(void* dst, uint32_t src, uint32_t n) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"((uint64_t)dst), "r"(src), "r"(n) : "memory");
}

template <int STAGES, bool STORE>
__global__ void __launch_bounds__(32, 1) rmw(float* h, char* x, char* y, int units) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long bars[8];
    const int u0 = blockIdx.x * units;
    if (threadIdx.x) return;
    for (int s = 0; s < STAGES; ++s) mbar_init(su32(&bars[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
    const uint32_t SZ = 40960;
    for (int k = 0; k < units + STAGES; ++k) {
        if (k >= STAGES) {
            const int j = k - STAGES, s = j % STAGES;
            mwait(su32(&bars[s]), (j / STAGES) & 1);
            if (STORE) {
                st(h + (size_t)(u0 + j) * 8192, su32(sm + s * SZ), 32768);
                st(y + (size_t)(u0 + j) * 8192, su32(sm + s * SZ + 32768), 8192);
                asm volatile("cp.async.bulk.commit_group;");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
        }
        if (k < units) {
            const int s = k % STAGES;
            const uint32_t bar = su32(&bars[s]);
            expect_tx(bar, SZ);
            ld(su32(sm + s * SZ), h + (size_t)(u0 + k) * 8192, 32768, bar);
            ld(su32(sm + s * SZ + 32768), x + (size_t)(u0 + k) * 8192, 8192, bar);
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// same traffic with x / y in the tree-scan layout: per unit (b, h) 64 rows of 128 B strided by H*P*2 bytes
// (x[B][T][H][P] bf16), issued by one warp (lane i: rows i, i + 32)
template <int STAGES, bool CONTIG = false>
__global__ void __launch_bounds__(32, 1) rmw_strided(float* h, char* x, char* y, int units, int H) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long bars[8];
    const int u0 = blockIdx.x * units;
    const int lane = threadIdx.x;
    if (lane == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(su32(&bars[s]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncwarp();
    const uint32_t SZ = 40960;
    auto xrow = [&](int unit, int t) {   // unit = b * H + h
        const int b = unit / H, hh = unit % H;
        if (CONTIG) return (size_t)unit * 8192 + t * 128;
        return ((size_t)(b * 64 + t) * H + hh) * 128;
    };
    for (int k = 0; k < units + STAGES; ++k) {
        if (k >= STAGES) {
            const int j = k - STAGES, s = j % STAGES;
            mwait(su32(&bars[s]), (j / STAGES) & 1);
            if (lane == 0) st(h + (size_t)(u0 + j) * 8192, su32(sm + s * SZ), 32768);
            for (int t = lane; t < 64; t += 32) st(y + xrow(u0 + j, t), su32(sm + s * SZ + 32768 + t * 128), 128);
            asm volatile("cp.async.bulk.commit_group;");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
        }
        if (k < units) {
            const int s = k % STAGES;
            const uint32_t bar = su32(&bars[s]);
            if (lane == 0) {
                expect_tx(bar, SZ);
                ld(su32(sm + s * SZ), h + (size_t)(u0 + k) * 8192, 32768, bar);
            }
            __syncwarp();
            for (int t = lane; t < 64; t += 32) ld(su32(sm + s * SZ + 32768 + t * 128), x + xrow(u0 + k, t), 128, bar);
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const int ctas = 144, units = 9, layers = 8;
    const size_t nunit = (size_t)ctas * units;
    float* h[layers];
    char *x[layers], *y[layers];
    for (int l = 0; l < layers; ++l) {
        cudaMalloc(&h[l], nunit * 32768);
        cudaMalloc(&x[l], nunit * 8192);
        cudaMalloc(&y[l], nunit * 8192);
        cudaMemset(h[l], 0, nunit * 32768);
        cudaMemset(x[l], 0, nunit * 8192);
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](auto k, int stages, const char* name, double bytes_per_unit) {
        size_t smem = (size_t)stages * 40960;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int w = 0; w < 2; ++w)
            for (int l = 0; l < layers; ++l) k<<<ctas, 32, smem>>>(h[l], x[l], y[l], units);
        cudaEventRecord(e0);
        const int reps = 5;
        for (int r = 0; r < reps; ++r)
            for (int l = 0; l < layers; ++l) k<<<ctas, 32, smem>>>(h[l], x[l], y[l], units);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / (reps * layers);
        printf("%-34s stages=%d %8.2f us/launch  %7.1f GB/s\n", name, stages, us, nunit * bytes_per_unit / (us * 1e-6) / 1e9);
        cudaError_t err = cudaGetLastError();
        if (err) printf("  error %s\n", cudaGetErrorString(err));
    };
    run(rmw<3, false>, 3, "load 40KB/unit only", 40960);
    run(rmw<3, true>, 3, "load 40KB + store 40KB (in place)", 81920);
    run(rmw<5, true>, 5, "load 40KB + store 40KB (in place)", 81920);
    auto run2 = [&](auto k, int stages, const char* name) {
        size_t smem = (size_t)stages * 40960;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int w = 0; w < 2; ++w)
            for (int l = 0; l < layers; ++l) k<<<ctas, 32, smem>>>(h[l], x[l], y[l], units, 81);
        cudaEventRecord(e0);
        const int reps = 5;
        for (int r = 0; r < reps; ++r)
            for (int l = 0; l < layers; ++l) k<<<ctas, 32, smem>>>(h[l], x[l], y[l], units, 81);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / (reps * layers);
        printf("%-34s stages=%d %8.2f us/launch  %7.1f GB/s\n", name, stages, us, nunit * 81920.0 / (us * 1e-6) / 1e9);
        cudaError_t err = cudaGetLastError();
        if (err) printf("  error %s\n", cudaGetErrorString(err));
    };
    run2(rmw_strided<3>, 3, "x/y strided 128B rows, state in place");
    run2(rmw_strided<5>, 5, "x/y strided 128B rows, state in place");
    run2(rmw_strided<3, true>, 3, "x/y 64 x 128B ops, contiguous");
    return 0;
}
