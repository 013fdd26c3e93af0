// tcgen05.mma throughput probe (one CTA per SM, one issuing thread): cycles per MMA for
// kind::tf32 (A from TMEM / from SMEM) and kind::f16, M=128, N=64 and N=128.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_probe tools/mma_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}
__host__ __device__ constexpr uint32_t idesc(uint32_t fmt, int M, int N) {
    return (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int MODE, int N, int M = 128>   // 0: tf32 TS, 1: tf32 SS, 2: f16 SS
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) unsigned long long bar;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tslot;
    if (threadIdx.x == 0) {
        const uint32_t base = su32(sm);
        const uint32_t fmt = MODE == 2 ? 1 : 2;
        const uint32_t id = idesc(fmt, M, N);
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            const uint64_t bd = sdesc(base + 32768 + (it & 3) * 32, 16, 1024);
            const uint32_t acc = it > 0;
            if (MODE == 0) {
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tm + 256),
                             "r"(tm + 64 + 8 * (it & 15)), "l"(bd), "r"(id), "r"(acc));
            } else {
                const uint64_t ad = sdesc(base + (it & 3) * 32, 16, 1024);
                if (MODE == 1)
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tm + 256),
                                 "l"(ad), "l"(bd), "r"(id), "r"(acc));
                else
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tm + 256),
                                 "l"(ad), "l"(bd), "r"(id), "r"(acc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(su32(&bar)));
        unsigned long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 1024 * 8);
    auto run = [&](auto k, const char* name, double flop_per_mma) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        const int iters = 4096;
        for (int rep = 0; rep < 2; ++rep) {
            k<<<148, 128, 65536>>>(iters, d);
            cudaDeviceSynchronize();
        }
        unsigned long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        double cyc = (double)h[0] / iters;
        printf("%-28s %7.1f cycles/MMA  (%.0f FLOP/cycle/SM)\n", name, cyc, flop_per_mma / cyc);
        cudaError_t e = cudaGetLastError();
        if (e) printf("  error %s\n", cudaGetErrorString(e));
    };
    run(probe<0, 64>, "tf32 TS M128 N64 K8", 2.0 * 128 * 64 * 8);
    run(probe<1, 64>, "tf32 SS M128 N64 K8", 2.0 * 128 * 64 * 8);
    run(probe<0, 128>, "tf32 TS M128 N128 K8", 2.0 * 128 * 128 * 8);
    run(probe<1, 128>, "tf32 SS M128 N128 K8", 2.0 * 128 * 128 * 8);
    run(probe<1, 64, 64>, "tf32 SS M64 N64 K8", 2.0 * 64 * 64 * 8);
    run(probe<1, 128, 64>, "tf32 SS M64 N128 K8", 2.0 * 64 * 128 * 8);
    run(probe<1, 256, 128>, "tf32 SS M128 N256 K8", 2.0 * 128 * 256 * 8);
    run(probe<0, 256, 128>, "tf32 TS M128 N256 K8", 2.0 * 128 * 256 * 8);
    run(probe<2, 64>, "f16 SS M128 N64 K16", 2.0 * 128 * 64 * 16);
    run(probe<2, 128>, "f16 SS M128 N128 K16", 2.0 * 128 * 128 * 16);
    return 0;
}
