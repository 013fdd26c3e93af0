// Ceiling probe for the fused replay+scan traffic in the kernel's own layout and TMA boxes: per unit
// (tree b, head h) load the 32 KB state (4 boxes {32 fp32, 64 rows}, SW128) and the x tile (box
// {64 bf16, 64 rows} strided by H*P*2 bytes in x[B][T][H][P]), store the state back in place and a
// y tile in the x layout; 144 CTAs x 9 units (16 trees x 81 heads), one thread, STAGES-deep ring.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_rmw_probe tools/tma_rmw_probe.cu -lcuda
#include <cuda.h>
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
__device__ __forceinline__ void tld(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
                 "l"((uint64_t)m), "r"(bar), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void tst(const CUtensorMap* m, uint32_t src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"((uint64_t)m), "r"(src),
                 "r"(c0), "r"(c1) : "memory");
}

__device__ __forceinline__ uint64_t pol_ef() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tld_h(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1, uint64_t pol) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst),
                 "l"((uint64_t)m), "r"(bar), "r"(c0), "r"(c1), "l"(pol) : "memory");
}
__device__ __forceinline__ void tst_h(const CUtensorMap* m, uint32_t src, int c0, int c1, uint64_t pol) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%2, %3}], [%1], %4;" ::"l"((uint64_t)m), "r"(src),
                 "r"(c0), "r"(c1), "l"(pol) : "memory");
}

constexpr int H = 81, T = 64, P = 64, N = 128, B = 16;

template <int STAGES, bool DEFER, int HINT = 0>   // HINT bit0: evict_first loads, bit1: evict_first stores
__global__ void __launch_bounds__(32, 1) k_rmw(const __grid_constant__ CUtensorMap mh, const __grid_constant__ CUtensorMap mx,
                                               const __grid_constant__ CUtensorMap my, int units) {
    extern __shared__ __align__(1024) unsigned char smr[];
    unsigned char* sm = smr + ((1024u - (su32(smr) & 1023u)) & 1023u);
    __shared__ __align__(8) unsigned long long bars[8];
    if (threadIdx.x) return;
    for (int s = 0; s < STAGES; ++s) mbar_init(su32(&bars[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;");
    const uint32_t SZ = 40960;
    const int u0 = blockIdx.x * units;
    auto issue_load = [&](int k) {
        const int s = k % STAGES, unit = u0 + k, b = unit / H, h = unit % H;
        const uint32_t bar = su32(&bars[s]), base = su32(sm + s * SZ);
        expect_tx(bar, SZ);
        if (HINT & 1) {
            const uint64_t p = pol_ef();
            for (int a = 0; a < 4; ++a) tld_h(base + a * 8192, &mh, bar, 32 * a, (b * H + h) * P, p);
            tld_h(base + 32768, &mx, bar, h * P, b * T, p);
        } else {
            for (int a = 0; a < 4; ++a) tld(base + a * 8192, &mh, bar, 32 * a, (b * H + h) * P);
            tld(base + 32768, &mx, bar, h * P, b * T);
        }
    };
    for (int k = 0; k < STAGES && k < units; ++k) issue_load(k);
    for (int j = 0; j < units; ++j) {
        const int s = j % STAGES, unit = u0 + j, b = unit / H, h = unit % H;
        mwait(su32(&bars[s]), (j / STAGES) & 1);
        const uint32_t base = su32(sm + s * SZ);
        if (HINT & 2) {
            const uint64_t p = pol_ef();
            for (int a = 0; a < 4; ++a) tst_h(&mh, base + a * 8192, 32 * a, (b * H + h) * P, p);
            tst_h(&my, base + 32768, h * P, b * T, p);
        } else {
            for (int a = 0; a < 4; ++a) tst(&mh, base + a * 8192, 32 * a, (b * H + h) * P);
            tst(&my, base + 32768, h * P, b * T);
        }
        asm volatile("cp.async.bulk.commit_group;");
        if (DEFER) {   // refill the previous unit's stage once its store has read it
            if (j > 0) {
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                if (j - 1 + STAGES < units) issue_load(j - 1 + STAGES);
            }
        } else {
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            if (j + STAGES < units) issue_load(j + STAGES);
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// Mixed variant: the 32 KB state of each unit through the LSU (cp.async 16-byte chunks into a STAGES-deep shared
// ring by NW warps, then read back and stored with st.global, in place), the x tile / y tile through TMA by one
// extra thread — the TMA engine carries only ~20 % of the bytes.
template <int STAGES, int NW>
__global__ void __launch_bounds__(32 * NW + 32, 1) k_mixed(const __grid_constant__ CUtensorMap mx,
                                                           const __grid_constant__ CUtensorMap my, float* hbase,
                                                           int units) {
    extern __shared__ __align__(1024) unsigned char smr[];
    unsigned char* sm = smr + ((1024u - (su32(smr) & 1023u)) & 1023u);
    __shared__ __align__(8) unsigned long long bars[8];
    const int tid = threadIdx.x, NT = 32 * NW;
    const int u0 = blockIdx.x * units;
    const uint32_t SZ = 32768;
    unsigned char* xs = sm + STAGES * SZ;   // x ring: STAGES x 8 KB
    if (tid == NT) {
        for (int s = 0; s < STAGES; ++s) mbar_init(su32(&bars[s]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
        auto issue = [&](int k) {
            const int s = k % STAGES, unit = u0 + k, b = unit / H, h = unit % H;
            expect_tx(su32(&bars[s]), 8192);
            tld(su32(xs + s * 8192), &mx, su32(&bars[s]), h * P, b * T);
        };
        for (int k = 0; k < STAGES && k < units; ++k) issue(k);
        for (int j = 0; j < units; ++j) {
            const int s = j % STAGES, unit = u0 + j, b = unit / H, h = unit % H;
            mwait(su32(&bars[s]), (j / STAGES) & 1);
            tst(&my, su32(xs + s * 8192), h * P, b * T);
            asm volatile("cp.async.bulk.commit_group;");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            if (j + STAGES < units) issue(j + STAGES);
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        return;
    }
    if (tid > NT) return;
    auto load = [&](int k) {
        const int s = k % STAGES, unit = u0 + k, b = unit / H, h = unit % H;
        const char* src = reinterpret_cast<const char*>(hbase + ((size_t)(b * H + h) * P) * N);
        for (int c = tid; c < 2048; c += NT)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(sm + s * SZ + c * 16)), "l"(src + c * 16) : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int k = 0; k < STAGES - 1; ++k) {
        if (k < units) load(k);
        else asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int j = 0; j < units; ++j) {
        if (j + STAGES - 1 < units) load(j + STAGES - 1);
        else asm volatile("cp.async.commit_group;" ::: "memory");
        asm volatile("cp.async.wait_group %0;" ::"n"(STAGES - 1) : "memory");   // this thread's chunks of unit j
        const int s = j % STAGES, unit = u0 + j, b = unit / H, h = unit % H;
        float4* dst = reinterpret_cast<float4*>(hbase + ((size_t)(b * H + h) * P) * N);
        for (int c = tid; c < 2048; c += NT) {
            const float4 v = *reinterpret_cast<const float4*>(sm + s * SZ + c * 16);
            __stcs(dst + c, v);
        }
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncodeFn enc = (EncodeFn)fp;
    const int layers = 8, ctas = 144, units = 9;
    float* hs[layers];
    char *xs[layers], *ys[layers];
    CUtensorMap mh[layers], mx[layers], my[layers];
    auto mk = [&](CUtensorMap* m, CUtensorMapDataType dt, void* base, uint64_t inner, uint64_t outer, uint64_t rb,
                  uint32_t bi, uint32_t bo) {
        cuuint64_t dims[2] = {inner, outer};
        cuuint64_t str[1] = {rb};
        cuuint32_t box[2] = {bi, bo};
        cuuint32_t es[2] = {1, 1};
        return enc(m, dt, 2, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    };
    for (int l = 0; l < layers; ++l) {
        cudaMalloc(&hs[l], (size_t)B * H * P * N * 4);
        cudaMalloc(&xs[l], (size_t)B * T * H * P * 2);
        cudaMalloc(&ys[l], (size_t)B * T * H * P * 2);
        cudaMemset(hs[l], 0, (size_t)B * H * P * N * 4);
        cudaMemset(xs[l], 0, (size_t)B * T * H * P * 2);
        int e = mk(&mh[l], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, hs[l], N, (uint64_t)B * H * P, N * 4, 32, 64) |
                mk(&mx[l], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, xs[l], H * P, B * T, H * P * 2, 64, T) |
                mk(&my[l], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, ys[l], H * P, B * T, H * P * 2, 64, T);
        if (e) printf("encode failed\n");
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = (double)ctas * units * (2 * 32768 + 2 * 8192);
    auto run = [&](auto k, int stages, const char* name) {
        size_t smem = (size_t)stages * 40960 + 1024;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int w = 0; w < 2; ++w)
            for (int l = 0; l < layers; ++l) k<<<ctas, 32, smem>>>(mh[l], mx[l], my[l], units);
        cudaEventRecord(e0);
        const int reps = 5;
        for (int r = 0; r < reps; ++r)
            for (int l = 0; l < layers; ++l) k<<<ctas, 32, smem>>>(mh[l], mx[l], my[l], units);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / (reps * layers);
        printf("%-46s stages=%d %8.2f us/launch  %7.1f GB/s\n", name, stages, us, bytes / (us * 1e-6) / 1e9);
        cudaError_t err = cudaGetLastError();
        if (err) printf("  error %s\n", cudaGetErrorString(err));
    };
    run(k_rmw<3, false>, 3, "TMA 2D state+x load, state+y store");
    run(k_rmw<4, false>, 4, "TMA 2D state+x load, state+y store");
    run(k_rmw<5, false>, 5, "TMA 2D state+x load, state+y store");
    run(k_rmw<4, true>, 4, "  same, deferred stage refill");
    run(k_rmw<5, true>, 5, "  same, deferred stage refill");
    run(k_rmw<4, false, 1>, 4, "  evict_first loads");
    run(k_rmw<4, false, 2>, 4, "  evict_first stores");
    run(k_rmw<4, false, 3>, 4, "  evict_first loads + stores");
    run(k_rmw<2, false, 0>, 2, "  2 stages");
    run(k_rmw<1, false, 0>, 1, "  1 stage");
    auto run_mixed = [&](auto k, int stages, int nw, const char* name) {
        size_t smem = (size_t)stages * 40960 + 1024;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int w = 0; w < 2; ++w)
            for (int l = 0; l < layers; ++l) k<<<ctas, 32 * nw + 32, smem>>>(mx[l], my[l], hs[l], units);
        cudaEventRecord(e0);
        const int reps = 5;
        for (int r = 0; r < reps; ++r)
            for (int l = 0; l < layers; ++l) k<<<ctas, 32 * nw + 32, smem>>>(mx[l], my[l], hs[l], units);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / (reps * layers);
        printf("%-46s stages=%d %8.2f us/launch  %7.1f GB/s\n", name, stages, us, bytes / (us * 1e-6) / 1e9);
        cudaError_t err = cudaGetLastError();
        if (err) printf("  error %s\n", cudaGetErrorString(err));
    };
    run_mixed(k_mixed<3, 4>, 3, 4, "LSU state (4 warps) + TMA x/y");
    run_mixed(k_mixed<4, 4>, 4, 4, "LSU state (4 warps) + TMA x/y");
    run_mixed(k_mixed<3, 8>, 3, 8, "LSU state (8 warps) + TMA x/y");
    run_mixed(k_mixed<4, 8>, 4, 8, "LSU state (8 warps) + TMA x/y");
    run_mixed(k_mixed<5, 8>, 5, 8, "LSU state (8 warps) + TMA x/y");
    return 0;
}
