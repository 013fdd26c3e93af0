// K9 stree_accept_mss: multi-step speculative sampling verification of a drafted tree (SURVEY §8(f)
// NEXT #4; "MSS sampling" for temperature > 0; reading R-mss):
//
//   cur = root, p = p_target[cur]
//   for each child c of cur (increasing index): t = tokens[c], q = q_draft[cur]
//       accept iff u_accept[c]·q[t] < p[t]  -> path += c, cur = c, p = p_target[c], next level
//       reject: r = max(0, p - q); if Σr > 0: p = r / Σr
//   no child accepted: bonus = smallest v with Σ_{w<=v} p[w] > u_bonus·Σ p
//
// One thread-block CLUSTER of 8 CTAs per tree; CTA k keeps the vocabulary slice [k·S, (k+1)·S) of
// the current distribution p (two ping-pong buffers, p = buf·scale: the normalisation is a scalar)
// and of the node's draft row q in its shared memory (S = ceil(V/8): 3 x 25 KB at V = 50,280), so
// the vocab-wide steps (residual, inverse CDF) run on 8 SMs with the partial sums exchanged through
// distributed shared memory (st.shared::cluster + barrier.cluster).  An acceptance test needs only
// p[t] and q[t]: q[t] from global memory; p[t] from global memory for a fresh distribution, else
// broadcast by the CTA owning t in the same exchange as the residual mass — one cluster barrier per
// rejection, and accepted chains never touch the vocabulary.  Every CTA takes every decision itself
// from bit-identical operands, so control flow stays uniform across the cluster.
#include "stree_common.cuh"
#include "stree_host.cuh"

namespace stree {
namespace mss {

__device__ unsigned long long g_mss_trace[64];   // debug: globaltimer stamps of tree 7, rank 0 (stree_debug_mss_trace)
__device__ __forceinline__ unsigned long long gt_mss() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

constexpr int kCl = 8;          // CTAs per tree
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
#ifdef STREE_TRACE
constexpr bool kMssTrace = true;
#else
constexpr bool kMssTrace = false;
#endif

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t map_rank(const void* p, uint32_t rank) {
    uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_cluster(uint32_t addr, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ float ld_cluster(uint32_t addr) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}

// block-wide sum, deterministic order; every thread gets the result
__device__ __forceinline__ float block_sum(float v, float* s_warp) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) s_warp[w] = v;
    __syncthreads();
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < kWarps; ++i) t += s_warp[i];
    return t;
}

__global__ void __launch_bounds__(kThreads, 1)
    mss_kernel(const int32_t* __restrict__ tokens, const int32_t* __restrict__ parent,
               const float* __restrict__ p_target, const float* __restrict__ q_draft,
               const float* __restrict__ u_accept, const float* __restrict__ u_bonus, int T, int V, int slice,
               int32_t* path, int32_t* path_len, int32_t* bonus, int32_t* dev_status) {
    extern __shared__ __align__(16) float dyn[];         // [3][slice]: p ping-pong, q of the current node
    __shared__ float s_next[2][2];                       // broadcast of the next sibling's p[t'] (double buffer)
    __shared__ int s_par[kMaxNodes];
    __shared__ int s_tok[kMaxNodes];
    __shared__ float s_u[kMaxNodes];
    __shared__ int s_child[kMaxNodes];
    __shared__ float s_qt[kMaxNodes], s_pt[kMaxNodes];
    __shared__ unsigned s_cm[kMaxNodes / 32];
    __shared__ float s_warp[kWarps];
    __shared__ float s_red[2][kCl];                      // cluster exchange of partial sums (double buffer)
    __shared__ float s_scan[kWarps];
    __shared__ int s_found;
    const int tid = threadIdx.x;
    const uint32_t rank = cluster_rank();
    const int b = blockIdx.x / kCl;
    const bool trc = kMssTrace && b == 7 && rank == 0 && tid == 0;
    int ntr = 0;
    auto stamp = [&]() { if (trc && ntr < 64) g_mss_trace[ntr++] = gt_mss(); };
    stamp();
    const int v0 = rank * slice, v1 = min(V, v0 + slice), n = max(0, v1 - v0);
    // every CTA of the cluster must have started before a peer writes its shared memory (DSMEM): arrive
    // now, wait right before the first remote access (racecheck: "block that might not have entered yet")
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    pdl_wait();
    int bad = 0;
    for (int i = tid; i < T; i += kThreads) {
        const int p = parent[(size_t)b * T + i];
        s_par[i] = p;
        s_tok[i] = tokens[(size_t)b * T + i];
        s_u[i] = u_accept[(size_t)b * T + i];
        if (i == 0 ? p != -1 : (p < 0 || p >= i)) bad = i == 0 ? 1 : 2;
    }
    const int any1 = __syncthreads_or(bad == 1), any2 = __syncthreads_or(bad == 2);
    if (any1 || any2) {
        if (rank == 0) {
            if (tid == 0) {
                report(dev_status, any1 ? 1 : 2);
                path_len[b] = 0;
                bonus[b] = -1;
            }
            for (int i = tid; i < T; i += kThreads) path[(size_t)b * T + i] = -1;
        }
        return;   // uniform across the cluster (same parent array)
    }
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    int red_buf = 0;
    // cluster-wide sum of one float per CTA (every CTA gets the same value, same order)
    auto cluster_sum = [&](float part) -> float {
        if (tid < kCl) st_cluster(map_rank(&s_red[red_buf][rank], tid), part);
        cluster_sync();
        float z = 0.f;
#pragma unroll
        for (int k = 0; k < kCl; ++k) z += s_red[red_buf][k];
        red_buf ^= 1;
        return z;
    };
    float* const bufA = dyn;                  // p ping-pong buffers and this node's draft row q (slices)
    float* const bufB = dyn + slice;
    float* const qs = dyn + 2 * slice;
    // fresh p (and q) slices of node `node`: batched independent loads (one latency per batch)
    auto load_rows = [&](int node, bool with_q) {
        const float* sp_ = p_target + ((size_t)b * T + node) * V + v0;
        const float* sq_ = q_draft + ((size_t)b * T + node) * V + v0;
        constexpr int kB = 8;
        for (int v00 = tid; v00 < n; v00 += kThreads * kB) {
            float pr[kB], qr[kB];
#pragma unroll
            for (int k = 0; k < kB; ++k) {
                const int v = min(v00 + k * kThreads, n - 1);
                pr[k] = __ldg(sp_ + v);
                qr[k] = with_q ? __ldg(sq_ + v) : 0.f;
            }
#pragma unroll
            for (int k = 0; k < kB; ++k) {
                const int v = v00 + k * kThreads;
                if (v < n) {
                    bufA[v] = pr[k];
                    if (with_q) qs[v] = qr[k];
                }
            }
        }
    };

    int cur = 0, plen = 1;
    bool loaded = false;          // buf[cb] * scale holds the current (residual) distribution of cur
    int cb = 0;
    float scale = 1.f, pt_next = 0.f;
    if (rank == 0 && tid == 0) path[(size_t)b * T] = 0;
    const int wid = tid >> 5, ln = tid & 31;
    for (;;) {
        const float* qrow = q_draft + ((size_t)b * T + cur) * V;
        // children of cur in index order (ballot compaction), and for each child the draft and target
        // probabilities of its token, all requested at once: one memory latency per node, not per test
        const bool isc = tid < T && s_par[tid] == cur;
        const unsigned m = __ballot_sync(0xffffffffu, isc);
        if (ln == 0 && wid < kMaxNodes / 32) s_cm[wid] = m;
        __syncthreads();
        int before = __popc(m & ((1u << ln) - 1u)), nch = 0;
#pragma unroll
        for (int k = 0; k < kMaxNodes / 32; ++k) {
            const int pc = __popc(s_cm[k]);
            nch += pc;
            if (k < wid) before += pc;
        }
        if (isc) s_child[before] = tid;
        __syncthreads();
        stamp();
        if (tid < nch) {
            const int c = s_child[tid], t = s_tok[c];
            const bool ok = t >= 0 && t < V;   // precondition; an out-of-range draft is simply rejected
            s_qt[tid] = ok ? __ldg(qrow + t) : 1.f;
            s_pt[tid] = ok ? __ldg(p_target + ((size_t)b * T + cur) * V + t) : 0.f;
        }
        __syncthreads();
        stamp();
        int acc = -1;
        loaded = false;
        for (int k = 0; k < nch; ++k) {
            const int c = s_child[k];
            // after a rejection p[t] of this sibling comes from the CTA owning t; an out-of-range token has
            // no owner and is rejected (p = 0), as before any rejection (s_pt)
            const int tc = s_tok[c];
            const float pt = loaded ? ((tc >= 0 && tc < V) ? pt_next : 0.f) : s_pt[k];
            if (s_u[c] * s_qt[k] < pt) {
                acc = c;
                break;
            }
            // rejected: residual r = max(0, p - q) into the other buffer; p <- r / Σr when the mass is positive
            if (!loaded) {
                load_rows(cur, true);
                loaded = true;
                cb = 0;
                scale = 1.f;
            }
            stamp();
            const float* src = cb ? bufB : bufA;
            float* dst = cb ? bufA : bufB;
            float part = 0.f;
            for (int v = tid; v < n; v += kThreads) {
                const float r = fmaxf(0.f, src[v] * scale - qs[v]);
                dst[v] = r;
                part += r;
            }
            part = block_sum(part, s_warp);   // (its barriers also publish dst within the CTA)
            // the next sibling's p[t'] is broadcast by the CTA owning t': no remote reads, so one cluster
            // barrier per rejection.  Both candidates travel: the residual (used when Σr > 0) and the kept p.
            const int rb = red_buf;
            if (k + 1 < nch && tid == 0) {
                const int tn = s_tok[s_child[k + 1]];
                if (tn >= 0 && tn < V && tn / slice == (int)rank) {
                    const float rv = dst[tn - v0], ov = src[tn - v0] * scale;
                    for (int q = 0; q < kCl; ++q) {
                        st_cluster(map_rank(&s_next[rb][0], q), rv);
                        st_cluster(map_rank(&s_next[rb][1], q), ov);
                    }
                }
            }
            stamp();
            const float z = cluster_sum(part);
            stamp();
            if (z > 0.f) {
                cb ^= 1;
                scale = 1.f / z;
                pt_next = s_next[rb][0] * scale;
            } else {
                pt_next = s_next[rb][1];
            }
        }
        if (acc < 0) break;
        if (rank == 0 && tid == 0) path[(size_t)b * T + plen] = acc;
        ++plen;
        cur = acc;
        __syncthreads();   // s_cm / s_child / s_qt / s_pt are rewritten for the next node
    }
    stamp();
    // bonus: inverse CDF of p over the vocabulary, slice by slice
    if (!loaded) {
        load_rows(cur, false);
        cb = 0;
        scale = 1.f;
    }
    __syncthreads();
    const float* ps = cb ? bufB : bufA;
    // each thread owns a contiguous chunk of the slice
    const int per = (n + kThreads - 1) / kThreads;
    const int c0 = min(n, tid * per), c1 = min(n, c0 + per);
    float tsum = 0.f;
    for (int v = c0; v < c1; ++v) tsum += ps[v] * scale;
    const float part = block_sum(tsum, s_warp);
    // slice sums of all ranks (same values in every CTA)
    if (tid < kCl) st_cluster(map_rank(&s_red[red_buf][rank], tid), part);
    cluster_sync();
    float sums[kCl], z = 0.f;
#pragma unroll
    for (int k = 0; k < kCl; ++k) {
        sums[k] = s_red[red_buf][k];
        z += sums[k];
    }
    const float thr = u_bonus[b] * z;
    int target = -1, last_pos = -1;
    float before = 0.f, cum = 0.f;
#pragma unroll
    for (int k = 0; k < kCl; ++k) {
        if (target < 0 && cum + sums[k] > thr) { target = k; before = cum; }
        cum += sums[k];
        if (sums[k] > 0.f) last_pos = k;
    }
    const bool fallback = target < 0;   // rounding left no CDF step above the threshold
    if (fallback) target = last_pos;
    if ((int)rank == target) {
        // exclusive scan of the thread chunk sums (deterministic: warp scan + warp totals)
        const int w = tid >> 5, l = tid & 31;
        float x = tsum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float y = __shfl_up_sync(0xffffffffu, x, o);
            if (l >= o) x += y;
        }
        if (l == 31) s_scan[w] = x;
        if (tid == 0) s_found = -1;
        __syncthreads();
        float wbase = 0.f;
        for (int i = 0; i < w; ++i) wbase += s_scan[i];
        float run = before + wbase + x - tsum;   // cumulative mass before this thread's chunk
        if (!fallback) {
            for (int v = c0; v < c1; ++v) {
                run += ps[v] * scale;
                if (run > thr) { atomicMin(reinterpret_cast<unsigned*>(&s_found), (unsigned)(v0 + v)); break; }
            }
        }
        __syncthreads();
        // read the search result into a register before any thread may change it: the fallback branch
        // below is then uniform across the CTA and its barrier is never divergent
        const bool none = s_found == -1;
        __syncthreads();
        if (none) {   // fallback (or the threshold fell past this slice's last step): last v with p > 0
            int lp = -1;
            for (int v = c0; v < c1; ++v)
                if (ps[v] > 0.f) lp = v0 + v;
            atomicMax(&s_found, lp);
        }
        __syncthreads();
        if (tid == 0) bonus[b] = s_found;
    }
    if (rank == 0) {
        for (int i = plen + tid; i < T; i += kThreads) path[(size_t)b * T + i] = -1;
        if (tid == 0) path_len[b] = plen;
    }
    stamp();
    cluster_sync();   // no CTA exits while a peer may still read its shared memory
    stamp();
}

}  // namespace mss
}  // namespace stree

extern "C" int stree_launch_accept_mss(const int32_t* tokens, const int32_t* parent, const float* p_target,
                                       const float* q_draft, const float* u_accept, const float* u_bonus, int B,
                                       int T, int V, int32_t* path, int32_t* path_len, int32_t* bonus,
                                       int32_t* dev_status, cudaStream_t s) {
    using namespace stree::mss;
    const int slice = (V + kCl - 1) / kCl;
    const size_t smem = (size_t)3 * slice * sizeof(float);
    cudaError_t e = stree::host::smem_attr((const void*)mss_kernel, (int)smem);
    if (e != cudaSuccess) return (int)e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(B * kCl);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (stree_launch_flags_get() & STREE_LAUNCH_PDL) ? 2 : 1;
    e = cudaLaunchKernelEx(&cfg, mss_kernel, tokens, parent, p_target, q_draft, u_accept, u_bonus, T, V, slice, path,
                           path_len, bonus, dev_status);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
}

extern "C" void stree_debug_mss_trace(unsigned long long* host64) {
    cudaMemcpyFromSymbol(host64, stree::mss::g_mss_trace, 64 * sizeof(unsigned long long));
}
