// Issue cost and latency of a dependent chain of tcgen05.mma (one accumulator, issue of the first ->
// commit barrier completes), the shapes of the small-batch scan kernel (stree_scan_lat.cu): kind::f16
// M=128, K=16 per instruction, N in {64, 128, 256}, SS (A and B from shared memory) or TS (A from TMEM).
// The chain is fully unrolled with descriptors = base + compile-time offsets (as the kernel should issue
// it), from a converged warp with elect.sync inside each instruction's asm; variant "1asm" issues the
// chain 8 instructions per asm block under a single elect.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_lat_probe tools/mma_lat_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

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
__host__ __device__ constexpr uint32_t idesc(uint32_t fmt, int bmaj, int M, int N) {
    return (1u << 4) | (fmt << 7) | (fmt << 10) | ((uint32_t)bmaj << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(bar),
                 "r"(ph)
                 : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b32 q;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync q|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t.reg .b32 q;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync q|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a), "l"(b), "r"(id), "r"(acc)
        : "memory");
}
// 8 SS MMAs under one elect: A and B descriptors advance by 2 (32 bytes) per K step within a 128-byte
// swizzle atom row, then by one atom (8192 B = 512 units) every 4 steps
__device__ __forceinline__ void mma_ss8(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t.reg .b32 q;\n\t.reg .b64 a1, b1;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync q|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "add.s64 a1, %1, 2;\n\tadd.s64 b1, %2, 2;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
        "add.s64 a1, %1, 4;\n\tadd.s64 b1, %2, 4;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
        "add.s64 a1, %1, 6;\n\tadd.s64 b1, %2, 6;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
        "add.s64 a1, %1, 512;\n\tadd.s64 b1, %2, 512;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
        "add.s64 a1, %1, 514;\n\tadd.s64 b1, %2, 514;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
        "add.s64 a1, %1, 516;\n\tadd.s64 b1, %2, 516;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
        "add.s64 a1, %1, 518;\n\tadd.s64 b1, %2, 518;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(id), "r"(acc)
        : "memory");
}

template <int NM, int MODE>   // MODE 0: SS unrolled, 1: TS unrolled, 2: SS one asm per 8
__global__ void __launch_bounds__(128, 1) chain(int N, int reps, unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) unsigned long long bar;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 96 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    if (warp == 0) {   // converged warp, elected lane issues
        const uint32_t sb = su32(sm);
        const uint32_t id = idesc(1, 0, 128, N);
        const uint64_t a0 = sdesc(sb, 16, 1024), b0 = sdesc(sb + 32768, 16, 1024);
        unsigned long long best = ~0ull, iss = 0;
        for (int r = 0; r < reps; ++r) {
            const unsigned long long t0 = clock64();
            if (MODE == 2) {
#pragma unroll
                for (int c = 0; c < NM / 8; ++c) mma_ss8(tmem + 256, a0 + 1024 * c, b0 + 1024 * c, id, c > 0);
            } else {
#pragma unroll
                for (int kk = 0; kk < NM; ++kk) {
                    const uint64_t off = (uint64_t)(((kk >> 2) * 8192 + (kk & 3) * 32) >> 4);
                    if (MODE == 0) mma_ss(tmem + 256, a0 + off, b0 + off, id, kk > 0);
                    else mma_ts(tmem + 256, tmem + 8 * (kk & 7), b0 + off, id, kk > 0);
                }
            }
            const unsigned long long t1 = clock64();
            asm volatile("{\n\t.reg .pred e;\n\t.reg .b32 q;\n\telect.sync q|e, 0xffffffff;\n\t"
                         "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bar))
                         : "memory");
            wait(su32(&bar), r & 1);
            const unsigned long long t2 = clock64();
            if (t2 - t0 < best) { best = t2 - t0; iss = t1 - t0; }
        }
        if (threadIdx.x == 0) { out[0] = best; out[1] = iss; }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

template <int NM, int MODE>
void run(unsigned long long* d, int N) {
    const int smem = 100 * 1024;
    cudaFuncSetAttribute(chain<NM, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    chain<NM, MODE><<<1, 128, smem>>>(N, 20, d);
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-5s N=%3d n=%2d: chain %6llu cycles (%.1f per MMA), issue %llu cycles  %s\n",
           MODE == 0 ? "SS" : MODE == 1 ? "TS" : "1asm", N, NM, h[0], (double)h[0] / NM, h[1],
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    for (int N : {64, 128, 256}) {
        run<1, 0>(d, N); run<4, 0>(d, N); run<8, 0>(d, N); run<16, 0>(d, N); run<24, 0>(d, N);
        run<1, 1>(d, N); run<4, 1>(d, N); run<8, 1>(d, N); run<16, 1>(d, N); run<24, 1>(d, N);
        run<8, 2>(d, N); run<16, 2>(d, N); run<24, 2>(d, N);
    }
    return 0;
}
