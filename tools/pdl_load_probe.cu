// Probe: how long does a global load issued BEFORE griddepcontrol.wait take to return while the preceding
// kernel (PDL primary) is still running?  A graph of dependent kernels, 80 CTAs each (the batch-1 scan grid):
// every CTA stamps its start, issues NL independent loads of distinct (uncached) lines, consumes them (stamp),
// waits on the dependency (stamp), triggers its dependents, then spins SPIN_NS on the globaltimer (a layer's
// post-wait body) and exits.  Prints, per launch, the median load latency and where it lands relative to the
// wait release.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pdl_load_probe tools/pdl_load_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <vector>

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <int NL>
__global__ void __launch_bounds__(256) k(const float* __restrict__ in, float* out, unsigned long long* tr, int spin_ns,
                                         int early) {
    const unsigned long long t0 = gt();
    float acc = 0.f;
    // coalesced: load i of thread t reads float4 number i * 256 + t of the CTA's 32 KB block (the state tile)
    const float4* src = reinterpret_cast<const float4*>(in) + (size_t)blockIdx.x * 256 * NL + threadIdx.x;
    unsigned long long t1 = 0;
    if (early) {
#pragma unroll
        for (int i = 0; i < NL; ++i) { const float4 v = __ldcs(src + (size_t)i * 256); acc += v.x + v.w; }
        if (acc == 1234.5f) out[0] = acc;
        __syncthreads();
        t1 = gt();
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const unsigned long long t2 = gt();
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (!early) {
#pragma unroll
        for (int i = 0; i < NL; ++i) { const float4 v = __ldcs(src + (size_t)i * 256); acc += v.x + v.w; }
        if (acc == 1234.5f) out[0] = acc;
        __syncthreads();
        t1 = gt();
    }
    while (gt() - t2 < (unsigned long long)spin_ns) {
    }
    if (threadIdx.x == 0) {
        tr[blockIdx.x * 4 + 0] = t0;
        tr[blockIdx.x * 4 + 1] = t1;
        tr[blockIdx.x * 4 + 2] = t2;
        tr[blockIdx.x * 4 + 3] = gt();
    }
}

int main() {
    const int ncta = 80, L = 48, NL = 8;   // 48 layers x 2.6 MB = 126 MB of distinct inputs
    const size_t per = (size_t)ncta * 256 * 4 * NL;   // floats per layer: 32 KB per CTA
    float* in;
    float* out;
    unsigned long long* tr;
    cudaMalloc(&in, per * L * 4);
    cudaMemset(in, 0, per * L * 4);
    cudaMalloc(&out, 4);
    cudaMalloc(&tr, (size_t)L * ncta * 4 * 8);
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (int early = 0; early < 2; ++early)
        for (int spin : {0, 3000}) {
            cudaGraph_t g;
            cudaGraphExec_t ge;
            cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
            for (int l = 0; l < L; ++l) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = ncta;
                cfg.blockDim = 256;
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaLaunchKernelEx(&cfg, k<NL>, (const float*)(in + per * l), out, tr + (size_t)l * ncta * 4, spin, early);
            }
            cudaStreamEndCapture(s, &g);
            cudaGraphInstantiate(&ge, g, 0);
            for (int it = 0; it < 3; ++it) cudaGraphLaunch(ge, s);
            cudaStreamSynchronize(s);
            std::vector<unsigned long long> h((size_t)L * ncta * 4);
            cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost);
            printf("loads %s the wait, post-wait body %d ns (%d x 16 B per thread, coalesced, 32 KB per CTA):\n",
                   early ? "BEFORE" : "after", spin, NL);
            for (int l = 1; l < L - 1; ++l) {
                std::vector<double> lat, rel, st;
                unsigned long long w = ~0ull;
                for (int c = 0; c < ncta; ++c) w = std::min(w, h[((size_t)l * ncta + c) * 4 + 2]);
                for (int c = 0; c < ncta; ++c) {
                    const unsigned long long* t = &h[((size_t)l * ncta + c) * 4];
                    lat.push_back(early ? (double)(t[1] - t[0]) : (double)(t[1] - t[2]));
                    rel.push_back((double)t[1] - (double)w);
                    st.push_back((double)t[0] - (double)w);
                }
                std::sort(lat.begin(), lat.end());
                std::sort(rel.begin(), rel.end());
                std::sort(st.begin(), st.end());
                if (l <= 6) printf("  layer %2d: start %7.2f us  load latency med %5.2f us  loads done med %6.2f us rel. to the wait\n", l,
                       st[ncta / 2] / 1e3, lat[ncta / 2] / 1e3, rel[ncta / 2] / 1e3);
            }
            cudaGraphExecDestroy(ge);
            cudaGraphDestroy(g);
        }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
