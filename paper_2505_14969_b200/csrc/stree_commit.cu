// K4 stree_commit — activation replay of the accepted path (PAPER.md:113,
// Alg. 1 l.123):  h_new = e^{Λ_k} h0 + Σ_{s∈path} e^{Λ_k-Λ_s} dt_s x_s B_sᵀ.
//
// HBM-bound streaming (intensity ≈ r/4 FLOP/B).  Main kernel: one CTA per
// (tree, chunk of heads), ≈ one wave over the SMs, 288 threads:
//   warp 0      producer: 1-D bulk copies (cp.async.bulk) of the chunk's contiguous
//               P x N fp32 state blocks into a ring of shared-memory slots
//   warps 1-8   once per CTA: path validation, per-head path-cumsum of log-decays
//               and coefficients, staging of the path rows of x (pre-scaled) and B;
//               then per state block: 16-byte shared loads -> decay·h + Σ_m u_m B_mᵀ
//               -> streaming 16-byte global stores (the slot is released as soon as
//               every warp has read it)
// The state stream starts at kernel entry and never waits for the dependent
// path prologue.  Accepted paths longer than kRMax (and shapes the ring cannot
// hold) use the simple per-(tree, head) kernel below.
#include "stree_common.cuh"
#include "stree_host.cuh"
#include "stree_tc_ptx.cuh"

namespace stree {

constexpr int kRMax = 16;            // path nodes staged by the ring kernel
constexpr int kCHPC = 16;            // max heads per CTA
constexpr int kCThreads = 288;       // 1 producer warp + 8 compute warps
constexpr int kCompute = 256;
constexpr int kRingBytes = 128 * 1024;

using stree::tc::mbar_arrive;
using stree::tc::mbar_expect_tx;
using stree::tc::mbar_init;
using stree::tc::mbar_wait;
using stree::tc::smem_u32;
__device__ __forceinline__ void bulk_load_1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
                 : "memory");
}

struct CommitParams {
    int B, T, H, P, N, G, cpg, hpc, slots;
    const void* x;
    const float* dt;
    const float* A;
    const void* Bm;
    const float* h0;
    const int32_t* parent;
    const int32_t* path;
    const int32_t* path_len;
    float* h_new;
    int32_t* dev_status;
    unsigned long long* trace;   // debug: per-CTA globaltimer stamps (64 per CTA)
    int early_state;             // STREE_LAUNCH_EARLY_STATE: stream h0 before the PDL wait
    DtX dtx;                     // *_ex options: effective dt
};

__device__ __forceinline__ unsigned long long c_gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

template <typename IO>
__global__ void __launch_bounds__(kCThreads, 1) commit_ring_kernel(const CommitParams prm) {
    extern __shared__ __align__(128) unsigned char csm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int H = prm.H, T = prm.T, P = prm.P, N = prm.N;
    const int b = blockIdx.x / (prm.G * prm.cpg);
    const int rem = blockIdx.x % (prm.G * prm.cpg);
    const int g = rem / prm.cpg, chunk = rem % prm.cpg;
    const int hpg = H / prm.G, hbeg = g * hpg + chunk * prm.hpc;
    const int nh = min(prm.hpc, g * hpg + hpg - hbeg);
    if (nh <= 0) { pdl_wait(); return; }
    const int blk = P * N;                              // floats per state block
    const uint32_t blk_bytes = (uint32_t)blk * 4;
    // shared layout: ring | u[nh][kRMax][P] (long paths: coef[kCHPC][kMaxNodes]) | Bs[kRMax][N] |
    //                decay[kCHPC] | path[kMaxNodes] | r | barriers
    float* ring = (float*)csm;
    float* u = (float*)(csm + (size_t)prm.slots * blk_bytes);
    float* coefl = u;
    // the u region is max(u staging, long-path coefficients) wide, as the host sizes it
    float* Bs = u + max(kCHPC * kRMax * P, kCHPC * kMaxNodes);
    float* decay = Bs + kRMax * N;                      // [kCHPC]
    int* spath = (int*)(decay + kCHPC);                 // [kMaxNodes]
    int* sr = spath + kMaxNodes;                        // [1]
    unsigned long long* bars = (unsigned long long*)(((uintptr_t)(sr + 1) + 7) & ~(uintptr_t)7);
    const uint32_t bar0 = smem_u32(bars);
    auto bar_full = [&](int s) { return bar0 + 8 * s; };
    auto bar_empty = [&](int s) { return bar0 + 8 * (prm.slots + s); };
    const size_t base = ((size_t)b * H + hbeg) * (size_t)blk;
    unsigned long long* tr = prm.trace ? prm.trace + (size_t)blockIdx.x * 64 : nullptr;
    if (tr && tid == 0) tr[0] = c_gtimer();

    if (tid == 0) {
        for (int s = 0; s < prm.slots; ++s) {
            mbar_init(bar_full(s), 1);
            mbar_init(bar_empty(s), kCompute / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == 0) {
        // ================= producer =================
        if (lane == 0 && prm.h0) {
            int k = 0;
            if (prm.early_state)   // the state is not written by the preceding kernel: stream it now
                for (; k < nh && k < prm.slots; ++k) {
                    mbar_expect_tx(bar_full(k), blk_bytes);
                    bulk_load_1d(smem_u32(ring + (size_t)k * blk), prm.h0 + base + (size_t)k * blk, blk_bytes, bar_full(k));
                }
            pdl_wait();
            for (; k < nh; ++k) {
                const int s = k % prm.slots;
                mbar_wait(bar_empty(s), ((k / prm.slots) & 1) ^ 1);
                mbar_expect_tx(bar_full(s), blk_bytes);
                bulk_load_1d(smem_u32(ring + (size_t)s * blk), prm.h0 + base + (size_t)k * blk, blk_bytes, bar_full(s));
            }
        }
        return;
    }
    // ================= compute warps =================
    pdl_wait();
    const int ct = tid - 32;                            // 0..255
    const IO* x = (const IO*)prm.x;
    const IO* Bm = (const IO*)prm.Bm;
    // ---- path validation (warp 1) ----
    if (warp == 1) {
        const int r = prm.path_len[b];
        int ok = (r >= 1 && r <= T);
        if (ok) {
            for (int m = lane; m < r; m += 32) {
                const int v = prm.path[(size_t)b * T + m];
                spath[m] = v;
                bool good = (v >= 0 && v < T);
                if (m == 0) good = good && v == 0;
                else {
                    const int pu = prm.path[(size_t)b * T + m - 1];
                    good = good && v > pu;
                    if (prm.parent && good) good = prm.parent[(size_t)b * T + v] == pu;
                }
                if (!good) ok = 0;
            }
        }
        ok = __all_sync(0xffffffffu, ok);
        if (lane == 0) {
            sr[0] = ok ? r : 0;
            if (!ok && chunk == 0 && g == 0) report(prm.dev_status, STREE_DEV_BAD_PATH);
        }
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (tr && tid == 32) tr[1] = c_gtimer();
    const int r = sr[0];                                // > 0 valid, 0 invalid (state unchanged)
    const bool staged = r <= kRMax;
    // ---- per-head path coefficients (one warp per head): lam_m = Σ_{q<=m} dt A_h,
    //      c_m = e^{lam_{r-1}-lam_m} dt_m, decay = e^{lam_{r-1}}  (PAPER.md:86-90 on the path) ----
    if (r > 0) {
        for (int hh = warp - 1; hh < nh; hh += 8) {
            const int h = hbeg + hh;
            const float Ah = prm.A[h];
            float carry = 0.f;
            float* cl = coefl + hh * kMaxNodes;          // long paths: lam then c in smem
            float cst = 0.f, dst0 = 0.f;
            for (int m0 = 0; m0 < r; m0 += 32) {
                const int m = m0 + lane;
                float d = 0.f, a = 0.f;
                if (m < r) {
                    d = dt_eff(prm.dtx, prm.dt[((size_t)b * T + spath[m]) * H + h], h);
                    a = d * Ah;
                }
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const float t = __shfl_up_sync(0xffffffffu, a, o);
                    if (lane >= o) a += t;
                }
                a += carry;
                if (staged) { cst = a; dst0 = d; }
                else if (m < r) cl[m] = a;
                carry = __shfl_sync(0xffffffffu, a, 31);
            }
            const float last = staged ? __shfl_sync(0xffffffffu, cst, r - 1) : carry;
            if (lane == 0) decay[hh] = expf(last);
            if (staged) {
                const float c = expf(last - cst) * dst0;
                for (int m = 0; m < r; ++m) {       // u[hh][m][p] = c_m x[b, s_m, h, p]
                    const float cm = __shfl_sync(0xffffffffu, c, m);
                    const IO* xr = x + (((size_t)b * T + spath[m]) * H + h) * P;
                    for (int p = lane; p < P; p += 32) u[(hh * kRMax + m) * P + p] = cm * to_f32(xr[p]);
                }
            } else {
                __syncwarp();
                for (int m = lane; m < r; m += 32)
                    cl[m] = expf(last - cl[m]) * dt_eff(prm.dtx, prm.dt[((size_t)b * T + spath[m]) * H + h], h);
            }
        }
        if (staged)
            for (int k = ct; k < r * N; k += kCompute) {
                const int m = k / N, n = k % N;
                Bs[m * N + n] = to_f32(Bm[(((size_t)b * T + spath[m]) * prm.G + g) * N + n]);
            }
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (tr && tid == 32) tr[2] = c_gtimer();
    // ---- stream the state blocks ----
    const int nvec = blk / 4;
    const int n0 = (4 * ct) % N, p0 = (4 * ct) / N, pstep = (4 * kCompute) / N;   // N divides 1024 (host-checked)
    for (int k = 0; k < nh; ++k) {
        const int s = k % prm.slots;
        float* dst = prm.h_new + base + (size_t)k * blk;
        float4 v[8];
        if (prm.h0) {
            mbar_wait(bar_full(s), (k / prm.slots) & 1);
            if (tr && tid == 32 && k < 16) tr[4 + 2 * k] = c_gtimer();
            const float4* src = reinterpret_cast<const float4*>(ring + (size_t)s * blk);
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int e = ct + q * kCompute;
                v[q] = e < nvec ? src[e] : make_float4(0, 0, 0, 0);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(bar_empty(s));
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = make_float4(0, 0, 0, 0);
        }
        if (r == 0) {                                                // invalid path: state unchanged
            if (prm.h0 != prm.h_new) {
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int e = ct + q * kCompute;
                    if (e < nvec) __stcs(reinterpret_cast<float4*>(dst) + e, v[q]);
                }
            }
            continue;
        }
        const float dk = decay[k];
        const int h = hbeg + k;
        // thread ct owns float4 columns n0 = (4 ct) mod N of rows p0 + q (1024/N), q = 0..7: the same n for
        // every q, so one B load per path node feeds 8 independent accumulator chains
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = make_float4(dk * v[q].x, dk * v[q].y, dk * v[q].z, dk * v[q].w);
        if (staged) {
            const float* uk = u + k * kRMax * P;
            for (int m = 0; m < r; ++m) {
                const float4 bb = *reinterpret_cast<const float4*>(&Bs[m * N + n0]);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (ct + q * kCompute >= nvec) break;
                    const float um = uk[m * P + p0 + q * pstep];
                    v[q].x = fmaf(um, bb.x, v[q].x); v[q].y = fmaf(um, bb.y, v[q].y);
                    v[q].z = fmaf(um, bb.z, v[q].z); v[q].w = fmaf(um, bb.w, v[q].w);
                }
            }
        } else {   // long accepted path: operands straight from L2
            const float* cl = coefl + k * kMaxNodes;
            for (int m = 0; m < r; ++m) {
                const int sm_ = spath[m];
                const IO* br = Bm + (((size_t)b * T + sm_) * prm.G + g) * N + n0;
                const float4 bb = make_float4(to_f32(br[0]), to_f32(br[1]), to_f32(br[2]), to_f32(br[3]));
                const IO* xr = x + (((size_t)b * T + sm_) * H + h) * P;
                const float cm = cl[m];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    if (ct + q * kCompute >= nvec) break;
                    const float um = cm * to_f32(xr[p0 + q * pstep]);
                    v[q].x = fmaf(um, bb.x, v[q].x); v[q].y = fmaf(um, bb.y, v[q].y);
                    v[q].z = fmaf(um, bb.z, v[q].z); v[q].w = fmaf(um, bb.w, v[q].w);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int e = ct + q * kCompute;
            if (e < nvec) __stcs(reinterpret_cast<float4*>(dst) + e, v[q]);
        }
        if (tr && tid == 32 && k < 16) tr[5 + 2 * k] = c_gtimer();
    }
    if (tr && tid == 32) tr[3] = c_gtimer();
}

// Simple per-(tree, head) kernel: long paths (r > kRMax) and shapes the ring kernel does not take.
template <typename IO>
__global__ void __launch_bounds__(256) commit_block_kernel(int T, int H, int P, int N, int G, const IO* __restrict__ x,
                                                           const float* __restrict__ dt, const float* __restrict__ A,
                                                           const IO* __restrict__ Bm, const float* h0,
                                                           const int32_t* __restrict__ parent,
                                                           const int32_t* __restrict__ path,
                                                           const int32_t* __restrict__ path_len, float* h_new,
                                                           int32_t* dev_status, DtX dtx) {
    __shared__ int s_path[kMaxNodes];
    __shared__ float s_coef[kMaxNodes];
    __shared__ float s_decay;
    __shared__ int s_r;
    const int h = blockIdx.x, b = blockIdx.y, g = h / (H / G), tid = threadIdx.x;
    pdl_wait();
    const int r0 = path_len[b];
    if (tid < 32) {
        int ok = (r0 >= 1 && r0 <= T);
        if (ok) {
            for (int m = tid; m < r0; m += 32) {
                const int v = path[(size_t)b * T + m];
                s_path[m] = v;
                bool good = (v >= 0 && v < T);
                if (m == 0) good = good && v == 0;
                else {
                    const int pu = path[(size_t)b * T + m - 1];
                    good = good && v > pu;
                    if (parent && good) good = parent[(size_t)b * T + v] == pu;
                }
                if (!good) ok = 0;
            }
        }
        ok = __all_sync(0xffffffffu, ok);
        if (ok) {
            const float Ah = A[h];
            float carry = 0.f;
            for (int base = 0; base < r0; base += 32) {
                const int m = base + tid;
                float a = (m < r0) ? dt_eff(dtx, dt[((size_t)b * T + s_path[m]) * H + h], h) * Ah : 0.f;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const float t = __shfl_up_sync(0xffffffffu, a, o);
                    if (tid >= o) a += t;
                }
                a += carry;
                if (m < r0) s_coef[m] = a;
                carry = __shfl_sync(0xffffffffu, a, 31);
            }
            __syncwarp();
            for (int m = tid; m < r0; m += 32)
                s_coef[m] = expf(carry - s_coef[m]) * dt_eff(dtx, dt[((size_t)b * T + s_path[m]) * H + h], h);
            if (tid == 0) s_decay = expf(carry);
        }
        if (tid == 0) s_r = ok ? r0 : 0;
    }
    __syncthreads();
    const size_t off = ((size_t)b * H + h) * (size_t)P * N;
    const float* src = h0 ? h0 + off : nullptr;
    float* dst = h_new + off;
    if (s_r == 0 && tid == 0) report(dev_status, STREE_DEV_BAD_PATH);
    for (int e = tid; e < P * N; e += 256) {
        const int p = e / N, n = e % N;
        float a = src ? src[e] : 0.f;
        if (s_r) {
            a *= s_decay;
            for (int m = 0; m < s_r; ++m) {
                const int s = s_path[m];
                a = fmaf(s_coef[m] * to_f32(x[(((size_t)b * T + s) * H + h) * P + p]),
                         to_f32(Bm[(((size_t)b * T + s) * G + g) * N + n]), a);
            }
        }
        dst[e] = a;
    }
}

}  // namespace stree

namespace {

unsigned long long* g_commit_trace = nullptr;

int commit_sms() { return stree::host::num_sms(); }

template <typename IO>
int launch(const stree_dims* d, const void* x, const float* dt, const float* A, const void* Bm, const float* h0,
           const int32_t* parent, const int32_t* path, const int32_t* path_len, float* h_new, int32_t* dev_status,
           cudaStream_t s) {
    const int B = d->batch, T = d->n_nodes, H = d->n_heads, P = d->head_dim, N = d->d_state, G = d->n_groups;
    const size_t blk_bytes = (size_t)P * N * 4;
    const bool ring_ok = (N % 4 == 0) && (1024 % N == 0) && (P * N <= 8 * stree::kCompute * 4) &&
                         (blk_bytes % 16 == 0) &&
                         (blk_bytes * 2 <= (size_t)stree::kRingBytes);
    if (!ring_ok) {
        return (int)stree::launch_k(stree::commit_block_kernel<IO>, dim3(H, B), dim3(256), 0, s, T, H, P, N, G,
                                    (const IO*)x, dt, A, (const IO*)Bm, h0, parent, path, path_len, h_new,
                                    dev_status, stree::DtX::from(stree_scan_opts_get()));
    }
    const int hpg = H / G;
    int cpg = commit_sms() / (B * G);
    if (cpg < 1) cpg = 1;
    if (cpg > hpg) cpg = hpg;
    int hpc = (hpg + cpg - 1) / cpg;
    if (hpc > stree::kCHPC) hpc = stree::kCHPC;
    cpg = (hpg + hpc - 1) / hpc;
    int slots = (int)(stree::kRingBytes / blk_bytes);
    if (slots > 8) slots = 8;
    stree::CommitParams prm{B, T, H, P, N, G, cpg, hpc, slots, x, dt, A, Bm, h0, parent, path, path_len,
                            h_new, dev_status, g_commit_trace,
                            (stree_launch_flags_get() & STREE_LAUNCH_EARLY_STATE) ? 1 : 0};
    prm.dtx = stree::DtX::from(stree_scan_opts_get());
    size_t ustage = (size_t)stree::kCHPC * stree::kRMax * P * 4;
    const size_t lcoef = (size_t)stree::kCHPC * stree::kMaxNodes * 4;
    if (ustage < lcoef) ustage = lcoef;
    const size_t smem = (size_t)slots * blk_bytes + ustage + (size_t)stree::kRMax * N * 4 + stree::kCHPC * 4 +
                        (stree::kMaxNodes + 1) * 4 + 16 + (size_t)2 * slots * 8 + 64;
    auto k = stree::commit_ring_kernel<IO>;
    cudaError_t e = stree::host::smem_attr((const void*)k, (int)smem);
    if (e != cudaSuccess) return (int)e;
    return (int)stree::launch_k(k, dim3(B * G * cpg), dim3(stree::kCThreads), smem, s, prm);
}

}  // namespace

extern "C" void stree_debug_commit_trace(unsigned long long* dev_buf) { g_commit_trace = dev_buf; }

extern "C" int stree_launch_commit(const stree_dims* d, const void* x, const float* dt, const float* A,
                                   const void* Bm, const float* h0, const int32_t* parent,
                                   const int32_t* path, const int32_t* path_len, float* h_new,
                                   int32_t* dev_status, cudaStream_t s) {
    if (d->io_dtype == STREE_BF16)
        return launch<__nv_bfloat16>(d, x, dt, A, Bm, h0, parent, path, path_len, h_new, dev_status, s);
    return launch<float>(d, x, dt, A, Bm, h0, parent, path, path_len, h_new, dev_status, s);
}
