// Launch-boundary floor of a chain of dependent kernels in one CUDA graph (the batch-1 setting of the
// scan: one kernel per layer, 80 CTAs).  Variants, per layer:
//   0: wait + one store (the pure PDL boundary)
//   1: wait, then each CTA reads RB bytes of its own (distinct per layer) data and writes WB bytes
//   2: same traffic, the reads issued before the wait (inputs not written by the preceding kernel)
//   3: mode 0 with 110 KB of dynamic shared memory (two CTAs per SM, like the small-batch scan kernel)
//   4: mode 3 + TMEM allocation of 256 columns (alloc before the wait, dealloc at exit)
//   5: mode 4 + 8 KB of y stores per CTA after the wait (16 B per thread, 2 per thread)
//   6: mode 5 + a 32 KB TMA-free bulk store (cp.async.bulk smem -> global) + wait, like the state commit
// Trigger (griddepcontrol.launch_dependents) after the wait, as the library does.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pdl_floor tools/pdl_floor.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <int MODE>
__global__ void __launch_bounds__(256) k(const float4* __restrict__ in, float4* __restrict__ out, int rb4, int wb4) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    __shared__ uint32_t tslot;
    float4 acc = make_float4(0, 0, 0, 0);
    if (MODE >= 4 && threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&tslot)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (MODE >= 4) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    const float4* src = in + (size_t)blockIdx.x * rb4;
    if (MODE == 2) {
        for (int i = threadIdx.x; i < rb4; i += blockDim.x) {
            const float4 v = __ldg(src + i);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    }
    pdl_wait();
    pdl_trigger();
    if (MODE == 1) {
        for (int i = threadIdx.x; i < rb4; i += blockDim.x) {
            const float4 v = __ldg(src + i);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    }
    float4* dst = out + (size_t)blockIdx.x * (wb4 > 0 ? wb4 : 1);
    if (MODE == 0 || MODE == 3 || MODE == 4) {
        if (threadIdx.x == 0) dst[0] = acc;
    } else if (MODE >= 5) {
        dst[threadIdx.x] = acc;
        dst[threadIdx.x + 256] = acc;
        if (MODE == 6 && threadIdx.x == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + 1024),
                         "r"((uint32_t)__cvta_generic_to_shared(dsm)), "r"(32768) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        }
    } else {
        for (int i = threadIdx.x; i < wb4; i += blockDim.x) dst[i] = acc;
    }
    if (MODE >= 4) {
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (threadIdx.x < 32) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tslot), "r"(256));
        }
    }
}

int main(int argc, char** argv) {
    const int ncta = argc > 1 ? atoi(argv[1]) : 80;
    const int L = 64;
    const int rb = 50 * 1024, wb = 48 * 1024;
    const int rb4 = rb / 16, wb4 = wb / 16;
    std::vector<float4*> ins(L), outs(L);
    for (int l = 0; l < L; ++l) {
        cudaMalloc(&ins[l], (size_t)ncta * rb);
        cudaMalloc(&outs[l], (size_t)ncta * wb);
        cudaMemset(ins[l], 0, (size_t)ncta * rb);
    }
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    const int dsmem = 110 * 1024;
    cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, dsmem);
    cudaFuncSetAttribute(k<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, dsmem);
    cudaFuncSetAttribute(k<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, dsmem);
    cudaFuncSetAttribute(k<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, dsmem);
    for (int mode = 0; mode < 7; ++mode) {
        for (int pdl = 0; pdl < 2; ++pdl) {
            cudaGraph_t g;
            cudaGraphExec_t ge;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            for (int l = 0; l < L; ++l) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(ncta);
                cfg.blockDim = dim3(256);
                cfg.stream = s;
                cfg.dynamicSmemBytes = mode >= 3 ? dsmem : 0;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = pdl;
                if (mode == 0) cudaLaunchKernelEx(&cfg, k<0>, (const float4*)ins[l], outs[l], rb4, wb4);
                if (mode == 1) cudaLaunchKernelEx(&cfg, k<1>, (const float4*)ins[l], outs[l], rb4, wb4);
                if (mode == 2) cudaLaunchKernelEx(&cfg, k<2>, (const float4*)ins[l], outs[l], rb4, wb4);
                if (mode == 3) cudaLaunchKernelEx(&cfg, k<3>, (const float4*)ins[l], outs[l], rb4, wb4);
                if (mode == 4) cudaLaunchKernelEx(&cfg, k<4>, (const float4*)ins[l], outs[l], rb4, wb4);
                if (mode == 5) cudaLaunchKernelEx(&cfg, k<5>, (const float4*)ins[l], outs[l], rb4, wb4);
                if (mode == 6) cudaLaunchKernelEx(&cfg, k<6>, (const float4*)ins[l], outs[l], rb4, wb4);
            }
            cudaStreamEndCapture(s, &g);
            cudaGraphInstantiate(&ge, g, 0);
            for (int i = 0; i < 5; ++i) cudaGraphLaunch(ge, s);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0, s);
            const int R = 20;
            for (int i = 0; i < R; ++i) cudaGraphLaunch(ge, s);
            cudaEventRecord(e1, s);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("ncta %d mode %d pdl %d: %.2f us per kernel (err %s)\n", ncta, mode, pdl, ms * 1e3 / (R * L),
                   cudaGetErrorString(cudaGetLastError()));
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
        }
    }
    return 0;
}
