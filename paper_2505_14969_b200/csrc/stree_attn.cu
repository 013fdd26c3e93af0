// K7 stree_tree_attn / K8 stree_kv_commit: tree-masked attention for the attention layers of a
// hybrid SSM/Transformer stack and the KV-cache commit of the accepted path (
// DESIGN.md reading R-attn).  PAPER.md:19, :54 (topology-aware mask), :63-66 (L_ij = 1 iff t_j on
// the root-to-t_i path), :318 (MambaInLlama hybrid):
//
//   o[b][i][h] = softmax_j( scale <q_i,h , key_j> ) value_j,
//   keys(i)    = k_cache[b][0 : cache_len[b]]  ++  k_new[b][path(i)]        (kv head h / (Hq/Hkv))
//
// Kernels serving stree_tree_attn:
//   attn_db_kernel   (default for bf16, head dim 128) the layout below with 64-key K/V tiles and two score
//                    buffers per query tile, so S_w(j+2) is computed while the softmax works on S_w(j+1)
//                    (K7b, further down; STREE_ATTN_DB=0 selects attn_tc_kernel).
//   attn_tc_kernel   bf16, head dim 128, (Hq/Hkv) | 128: flash attention on tcgen05.  One CTA per
//                    (tree, kv head, pair of 128-row query tiles); query rows are (node, q head of
//                    the group) so the GQA group shares every K/V tile.  Warp 0: TMA producer
//                    (Q once, then K/V tiles of 128 keys into a 2-stage ring: the committed prefix
//                    first, then the tree's own nodes).  Warp 1: MMA issuer + TMEM allocator
//                    (S_w = Q_w·Kᵀ into TMEM columns [128w, 128w+128), P_w written back over S_w as
//                    bf16, O_w += P_w·V from TMEM (TS MMA) into columns [256+128w, ...)).  Warps 2-5
//                    and 6-9: softmax of query tile 0 / 1 (thread = row = TMEM lane): mask (prefix
//                    length, ancestor bits of the row's node), online max with lazy rescaling,
//                    exp2, P to TMEM, and the final O/l epilogue.  The two tiles ping-pong: the
//                    tensor core computes S_1 while tile 0's softmax runs, and so on.
//   attn_simt_kernel any shape / fp32 (the 1e-4 fp32 path): one warp per (tree, node, q head),
//                    lanes over keys, online softmax, fp32 throughout.
#include <cuda.h>

#include <cstdlib>

#include "stree_common.cuh"
#include "stree_host.cuh"
#include "stree_tc_ptx.cuh"

namespace stree {
namespace attn {

using namespace stree::tc;

constexpr int kDev_Capacity = STREE_DEV_CAPACITY;   // cache_len out of [0, cache_cap] / commit overflow

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// 2^x on the FMA pipe (offloads the 16/clk/SM MUFU): x = n + f, n = rint(x), f in [-1/2, 1/2];
// 2^f by a degree-3 fit (max rel err 1.1e-4, below the bf16 rounding of P); 2^n added to the exponent.
// Inputs below -126 are clamped (2^-126: the caller zeroes masked entries itself).
__device__ __forceinline__ float ex2_poly(float x) {
    x = fmaxf(x, -126.f);
    const float t = x + 12582912.f;                 // 1.5 * 2^23: rint(x) in the low mantissa bits
    const float f = x - (t - 12582912.f);
    const float p = fmaf(f, fmaf(f, fmaf(f, 0.05459818f, 0.24221842f), 0.69336758f), 1.0f);
    return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
__device__ __forceinline__ uint64_t f2pack(float lo, float hi) {
    return ((uint64_t)__float_as_uint(hi) << 32) | __float_as_uint(lo);
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
// two 2^x on the FMA pipe with paired fp32 ops (FADD2 / FFMA2): same split and polynomial as ex2_poly
__device__ __forceinline__ void ex2_poly2(uint64_t a2, float& p0, float& p1) {
    const uint64_t x = f2pack(fmaxf(__uint_as_float((uint32_t)a2), -126.f), fmaxf(__uint_as_float((uint32_t)(a2 >> 32)), -126.f));
    const uint64_t t = fadd2(x, f2pack(12582912.f, 12582912.f));
    const uint64_t r = fadd2(t, f2pack(-12582912.f, -12582912.f));
    const uint64_t f = ffma2(r, f2pack(-1.f, -1.f), x);
    uint64_t p = ffma2(f, f2pack(0.05459818f, 0.05459818f), f2pack(0.24221842f, 0.24221842f));
    p = ffma2(p, f, f2pack(0.69336758f, 0.69336758f));
    p = ffma2(p, f, f2pack(1.f, 1.f));
    p0 = __int_as_float((int)(uint32_t)p + ((int)(uint32_t)t << 23));
    p1 = __int_as_float((int)(uint32_t)(p >> 32) + ((int)(uint32_t)(t >> 32) << 23));
}

// ---------------------------------------------------------------------------
// SIMT kernel (any head dim <= 256, fp32 or bf16 io)
// ---------------------------------------------------------------------------
constexpr int kSimtMaxD = 256;

template <typename IO>
__global__ void __launch_bounds__(32) attn_simt_kernel(const IO* __restrict__ q, const IO* __restrict__ k_new,
                                                       const IO* __restrict__ v_new, const IO* __restrict__ k_cache,
                                                       const IO* __restrict__ v_cache,
                                                       const int32_t* __restrict__ cache_len,
                                                       const int32_t* __restrict__ parent, float scale, IO* o, int T,
                                                       int Hq, int Hkv, int D, int S, int32_t* dev_status) {
    __shared__ float sq[kSimtMaxD];
    __shared__ int spath[kMaxNodes];
    __shared__ int snp, sbad;
    pdl_wait();
    const int h = blockIdx.x, i = blockIdx.y, b = blockIdx.z, lane = threadIdx.x;
    const int g = h / (Hq / Hkv);
    const int32_t* par = parent + (size_t)b * T;
    if (lane == 0) {
        int bad = par[0] != -1 ? 1 : 0;
        for (int v = 1; v < T && !bad; ++v)
            if (par[v] < 0 || par[v] >= v) bad = 2;
        const int L = cache_len[b];
        if (!bad && (L < 0 || L > S)) bad = kDev_Capacity;
        int n = 0;
        if (!bad)
            for (int v = i; v >= 0; v = par[v]) spath[n++] = v;   // i .. root (order is irrelevant to softmax)
        snp = n;
        sbad = bad;
        if (bad && i == 0 && h == 0) report(dev_status, bad);
    }
    for (int d = lane; d < D; d += 32) sq[d] = to_f32<IO>(q[(((size_t)b * T + i) * Hq + h) * D + d]);
    __syncwarp();
    IO* orow = o + (((size_t)b * T + i) * Hq + h) * D;
    if (sbad) {
        for (int d = lane; d < D; d += 32) orow[d] = from_f32<IO>(0.f);
        return;
    }
    const int L = cache_len[b], np = snp, nk = L + np;
    constexpr int kE = kSimtMaxD / 32;
    float acc[kE];
#pragma unroll
    for (int e = 0; e < kE; ++e) acc[e] = 0.f;
    float m = -INFINITY, l = 0.f;
    auto krow = [&](int j) -> const IO* {
        return j < L ? k_cache + (((size_t)b * S + j) * Hkv + g) * D
                     : k_new + (((size_t)b * T + spath[j - L]) * Hkv + g) * D;
    };
    auto vrow = [&](int j) -> const IO* {
        return j < L ? v_cache + (((size_t)b * S + j) * Hkv + g) * D
                     : v_new + (((size_t)b * T + spath[j - L]) * Hkv + g) * D;
    };
    for (int j0 = 0; j0 < nk; j0 += 32) {
        const int j = j0 + lane;
        float s = -INFINITY;
        if (j < nk) {
            const IO* kr = krow(j);
            float dot = 0.f;
            for (int d = 0; d < D; ++d) dot = fmaf(sq[d], to_f32<IO>(kr[d]), dot);
            s = dot * scale;
        }
        float mc = s;
#pragma unroll
        for (int off = 16; off; off >>= 1) mc = fmaxf(mc, __shfl_xor_sync(0xffffffffu, mc, off));
        const float mn = fmaxf(m, mc);
        const float alpha = m == -INFINITY ? 0.f : expf(m - mn);
        const float p = j < nk ? expf(s - mn) : 0.f;
        float ps = p;
#pragma unroll
        for (int off = 16; off; off >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
        l = l * alpha + ps;
        m = mn;
#pragma unroll
        for (int e = 0; e < kE; ++e) acc[e] *= alpha;
        const int nj = min(32, nk - j0);
        for (int jj = 0; jj < nj; ++jj) {
            const float pj = __shfl_sync(0xffffffffu, p, jj);
            const IO* vr = vrow(j0 + jj);
#pragma unroll
            for (int e = 0; e < kE; ++e) {
                const int d = lane + 32 * e;
                if (d < D) acc[e] = fmaf(pj, to_f32<IO>(vr[d]), acc[e]);
            }
        }
    }
    const float inv = 1.f / l;
#pragma unroll
    for (int e = 0; e < kE; ++e) {
        const int d = lane + 32 * e;
        if (d < D) orow[d] = from_f32<IO>(acc[e] * inv);
    }
}

// ---------------------------------------------------------------------------
// tcgen05 kernel (bf16, D = 128)
// ---------------------------------------------------------------------------
constexpr int kD = 128;
constexpr int kBM = 128;            // query rows per tile
constexpr int kBN = 128;            // keys per K/V tile
constexpr int kStages = 2;
constexpr int kThreads = 320;       // warp 0 TMA, warp 1 MMA, warps 2-5 softmax tile 0, 6-9 softmax tile 1
constexpr int kThreadsSplit = 576;  // warp 0 TMA, warp 1 MMA, warps 2-9 softmax tile 0, 10-17 softmax tile 1
constexpr int kHalf = kBM * 128;    // one 128-row x 64-element (128 B) swizzle-128B box = 16 KB
constexpr int kTile = 2 * kHalf;    // 128 rows x 128 elements
constexpr uint32_t kTmemCols = 512;

struct Smem {
    static constexpr int Q = 0;                          // 2 query tiles
    static constexpr int K = Q + 2 * kTile;              // kStages key tiles
    static constexpr int V = K + kStages * kTile;        // kStages value tiles
    static constexpr int PAR = V + kStages * kTile;      // parent[256] int
    static constexpr int ANC = PAR + kMaxNodes * 4;      // ancestor bits of each softmax row: [8 words][256 rows]
    static constexpr int BAR = ANC + kMaxWords * 256 * 4;
    // barriers: qfull, kfull[2], kempty[2], vfull[2], vempty[2], sfull[2], pfull[2], ofull[2]
    static constexpr int NBAR = 1 + 4 * kStages + 6;
    static constexpr int TMEMP = BAR + NBAR * 8;
    static constexpr int MISC = TMEMP + 16;              // int: bad flag, L
    static constexpr int XCH = MISC + 16;                // float [2 parity][2 tiles][2 halves][128 rows]
    static constexpr int TOTAL = XCH + 2 * 2 * 2 * 128 * 4;
    static_assert(TOTAL + 1024 <= 227 * 1024, "shared memory budget");
};

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1, int c2,
                                            int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
        "[%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

struct AttnParams {
    const int32_t* cache_len;
    const int32_t* parent;
    __nv_bfloat16* o;
    int32_t* dev_status;
    int T, Hq, Hkv, S, npairs, early;
    int early_tree;   // STREE_LAUNCH_EARLY_TREE with EARLY_STATE: tree validation before the dependency wait (K7b)
    unsigned long long* trace;
    float scale_log2;
};

// POLY: exp2 on the MUFU (0) or every 4th pair on the FMA pipe (1).  SPLIT: two softmax warps per TMEM lane
// quadrant and query tile, each owning 64 of the 128 score columns of its 32 rows (18 warps), so the exp
// phase of a tile runs at MUFU throughput instead of one warp's latency; row max and row sum are combined
// through shared memory with a 64-thread named barrier per (tile, quadrant).
template <int POLY, bool SPLIT>
__global__ void __launch_bounds__(SPLIT ? kThreadsSplit : kThreads, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kc,
                   const __grid_constant__ CUtensorMap tm_vc, const __grid_constant__ CUtensorMap tm_kn,
                   const __grid_constant__ CUtensorMap tm_vn, const AttnParams prm) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sb = smem_u32(sm);
    const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
    const int T = prm.T, Hq = prm.Hq, Hkv = prm.Hkv, grp = Hq / Hkv;
    const int b = blockIdx.x / (Hkv * prm.npairs);
    const int rem = blockIdx.x % (Hkv * prm.npairs);
    const int kvh = rem / prm.npairs, pr = rem % prm.npairs;
    const int nmt = (T * grp + kBM - 1) / kBM;
    const int nw = min(2, nmt - 2 * pr);               // query tiles of this CTA (1 or 2)
    unsigned long long* tr = (prm.trace && blockIdx.x == 0) ? prm.trace : nullptr;   // debug timeline

    const uint32_t bar0 = sb + Smem::BAR;
    const uint32_t BAR_Q = bar0;
    auto bar_kfull = [&](int s) { return bar0 + 8 + 8 * s; };
    auto bar_kempty = [&](int s) { return bar0 + 8 + 8 * kStages + 8 * s; };
    auto bar_vfull = [&](int s) { return bar0 + 8 + 16 * kStages + 8 * s; };
    auto bar_vempty = [&](int s) { return bar0 + 8 + 24 * kStages + 8 * s; };
    auto bar_sfull = [&](int w) { return bar0 + 8 + 32 * kStages + 8 * w; };
    auto bar_pfull = [&](int w) { return bar0 + 8 + 32 * kStages + 16 + 8 * w; };
    auto bar_ofull = [&](int w) { return bar0 + 8 + 32 * kStages + 32 + 8 * w; };
    uint32_t* tmem_slot = (uint32_t*)(sm + Smem::TMEMP);
    int* sp = (int*)(sm + Smem::PAR);

    if (tid == 0) {
        mbar_init(BAR_Q, 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(bar_kfull(s), 1);
            mbar_init(bar_kempty(s), 1);
            mbar_init(bar_vfull(s), 1);
            mbar_init(bar_vempty(s), 1);
        }
        for (int w = 0; w < 2; ++w) {
            mbar_init(bar_sfull(w), 1);
            mbar_init(bar_pfull(w), SPLIT ? 256 : 128);
            mbar_init(bar_ofull(w), 1);
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // EARLY_STATE promise (stree_set_launch_flags): the KV cache and cache_len are not written by the kernel
    // immediately preceding this one (true in a decode loop: the cache was committed an iteration earlier),
    // so the first prefix tiles stream in before the dependency wait, overlapping the previous kernel
    int n_early = 0;
    auto issue_kv = [&](int j, bool pre, int key0) {
        const int s = j % kStages;
        mbar_expect_tx(bar_kfull(s), kTile);
        for (int hf = 0; hf < 2; ++hf)
            tma_load_4d(sb + Smem::K + s * kTile + hf * kHalf, pre ? &tm_kc : &tm_kn, bar_kfull(s), 64 * hf, kvh, key0, b);
        mbar_expect_tx(bar_vfull(s), kTile);
        for (int hf = 0; hf < 2; ++hf)
            tma_load_4d(sb + Smem::V + s * kTile + hf * kHalf, pre ? &tm_vc : &tm_vn, bar_vfull(s), 64 * hf, kvh, key0, b);
    };
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tm_q); tma_prefetch(&tm_kc); tma_prefetch(&tm_vc); tma_prefetch(&tm_kn); tma_prefetch(&tm_vn);
        if (prm.early) {
            const int Le = prm.cache_len[b];
            if (Le > 0 && Le <= prm.S) {
                n_early = min(kStages, (Le + kBN - 1) / kBN);
                for (int j = 0; j < n_early; ++j) issue_kv(j, true, j * kBN);
            }
        }
    }
    pdl_wait();
    // tree validation (PAPER.md:90 ordering, R5) and the committed prefix length
    int bad = 0;
    for (int v = tid; v < T; v += (int)blockDim.x) {
        const int p = prm.parent[(size_t)b * T + v];
        sp[v] = p;
        if (v == 0 ? p != -1 : (p < 0 || p >= v)) bad = v == 0 ? 1 : 2;
    }
    const int L = prm.cache_len[b];
    const int any1 = __syncthreads_or(bad == 1);
    const int any2 = __syncthreads_or(bad == 2);
    int code = any1 ? 1 : (any2 ? 2 : ((L < 0 || L > prm.S) ? kDev_Capacity : 0));
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int npre = code ? 0 : (L + kBN - 1) / kBN;   // prefix tiles
    const int ntr = (T + kBN - 1) / kBN;               // tree tiles
    const int nt = npre + ntr;

    if (code) {
        if (tid == 0 && rem == 0) report(prm.dev_status, code);
        if (warp == 0 && lane == 0)   // drain the early loads before the CTA exits
            for (int j = 0; j < n_early; ++j) {
                mbar_wait(bar_kfull(j), 0);
                mbar_wait(bar_vfull(j), 0);
            }
        // zero this CTA's output rows
        if (warp >= 2 && (!SPLIT || ((warp - 2) & 7) < 4)) {
            const int w = SPLIT ? (warp - 2) >> 3 : (warp - 2) >> 2, r = 32 * (warp & 3) + lane;
            if (w < nw) {
                const int rr = (2 * pr + w) * kBM + r, i = rr / grp, hg = rr % grp;
                if (i < T) {
                    uint4* orow = (uint4*)(prm.o + (((size_t)b * T + i) * Hq + kvh * grp + hg) * kD);
#pragma unroll
                    for (int c = 0; c < kD / 8; ++c) orow[c] = make_uint4(0, 0, 0, 0);
                }
            }
        }
    } else if (warp == 0) {
        // ---- TMA producer ----
        if (lane == 0) {
            mbar_expect_tx(BAR_Q, nw * kTile);
            for (int w = 0; w < nw; ++w) {
                const int node0 = (2 * pr + w) * (kBM / grp);
                for (int hf = 0; hf < 2; ++hf)
                    tma_load_4d(sb + Smem::Q + w * kTile + hf * kHalf, &tm_q, BAR_Q, 64 * hf, kvh * grp, node0, b);
            }
            for (int j = n_early; j < nt; ++j) {
                const int s = j % kStages, u = j / kStages;
                const bool pre = j < npre;
                const int key0 = pre ? j * kBN : (j - npre) * kBN;
                mbar_wait(bar_kempty(s), (u & 1) ^ 1);
                mbar_wait(bar_vempty(s), (u & 1) ^ 1);
                if (tr && j < 64) tr[j] = gtimer();
                issue_kv(j, pre, key0);
            }
        }
    } else if (warp == 1) {
        // ---- MMA issuer (whole warp converged, one elected lane issues) ----
        const uint32_t id_s = idesc(kFmtBF16, 0, kBM, kBN);   // S = Q·Kᵀ: A, B K-major
        const uint32_t id_o = idesc(kFmtBF16, 1, kBM, kD);    // O += P·V: A in TMEM, B (V) MN-major
        auto issue_s = [&](int w, int s) {
#pragma unroll
            for (int kk = 0; kk < kD / 16; ++kk) {
                const uint64_t ad = sdesc(sb + Smem::Q + w * kTile + (kk >> 2) * kHalf, 16, 1024) + (uint64_t)((kk & 3) * 2);
                const uint64_t bd = sdesc(sb + Smem::K + s * kTile + (kk >> 2) * kHalf, 16, 1024) + (uint64_t)((kk & 3) * 2);
                mma_f16_w(tmem + 128 * w, ad, bd, id_s, kk > 0);
            }
            tc_commit_w(bar_sfull(w));
        };
        mbar_wait(BAR_Q, 0);
        mbar_wait(bar_kfull(0), 0);
        tc_fence_after();
        for (int w = 0; w < nw; ++w) issue_s(w, 0);
        tc_commit_w(bar_kempty(0));
        for (int j = 0; j < nt; ++j) {
            const int s = j % kStages, u = j / kStages;
            const int s1 = (j + 1) % kStages, u1 = (j + 1) / kStages;
            for (int w = 0; w < nw; ++w) {
                mbar_wait(bar_pfull(w), j & 1);
                if (tr && lane == 0 && j < 64) tr[128 + 2 * j + w] = gtimer();
                if (w == 0) mbar_wait(bar_vfull(s), u & 1);
                tc_fence_after();
                const uint64_t vd = sdesc(sb + Smem::V + s * kTile, kHalf, 1024);
#pragma unroll
                for (int kk = 0; kk < kBN / 16; ++kk)
                    mma_f16_ts_w(tmem + 256 + 128 * w, tmem + 128 * w + 8 * kk + ((SPLIT && kk >= 4) ? 32 : 0),
                                 vd + (uint64_t)(kk * 128), id_o, (j > 0 || kk > 0) ? 1u : 0u);
                if (w == nw - 1) tc_commit_w(bar_vempty(s));
                if (j == nt - 1) tc_commit_w(bar_ofull(w));
                if (j + 1 < nt) {
                    if (w == 0) {
                        mbar_wait(bar_kfull(s1), u1 & 1);
                        if (tr && lane == 0 && j < 64) tr[256 + j] = gtimer();
                        tc_fence_after();
                    }
                    issue_s(w, s1);
                    if (w == nw - 1) tc_commit_w(bar_kempty(s1));
                }
            }
        }
    } else {
        // ---- softmax: thread = query row = TMEM lane (SPLIT: and one half of the score columns) ----
        constexpr int kCols = SPLIT ? 64 : 128;            // score columns per thread
        const int sw = SPLIT ? (warp - 2) & 7 : (warp - 2) & 3;
        const int w = SPLIT ? (warp - 2) >> 3 : (warp - 2) >> 2, q4 = warp & 3, r = 32 * q4 + lane;
        const int hh = SPLIT ? sw >> 2 : 0;                 // column half
        if (w < nw) {
            const int rr = (2 * pr + w) * kBM + r, i = rr / grp, hg = rr % grp;
            const bool vrow = i < T;
            // ancestor bits of the row's node, word-major in smem (conflict-free reads); the
            // two halves write identical values
            uint32_t* sanc = (uint32_t*)(sm + Smem::ANC) + 128 * w + r;
            {
                uint32_t anc[kMaxWords];
#pragma unroll
                for (int q = 0; q < kMaxWords; ++q) anc[q] = 0u;
                if (vrow)
                    for (int v = i; v >= 0; v = sp[v]) {
#pragma unroll
                        for (int q = 0; q < kMaxWords; ++q) anc[q] |= ((v >> 5) == q) ? (1u << (v & 31)) : 0u;
                    }
#pragma unroll
                for (int q = 0; q < kMaxWords; ++q) sanc[256 * q] = anc[q];
            }
            float* xch = (float*)(sm + Smem::XCH);          // [parity][tile][half][row]
            auto pair_sync = [&]() { if (SPLIT) named_bar(1 + 4 * w + q4, 64); };
            const uint32_t lane_base = tmem + ((uint32_t)(32 * q4) << 16);
            const uint32_t t_s = lane_base + 128 * w, t_o = lane_base + 256 + 128 * w;
            const float sl2 = prm.scale_log2;
            const bool tr0 = tr && w == 0 && hh == 0 && lane == 0 && q4 == 0;
            float m_run = -INFINITY, l_run = 0.f;
            for (int j = 0; j < nt; ++j) {
                mbar_wait(bar_sfull(w), j & 1);
                if (tr && hh == 0 && lane == 0 && q4 == 0 && j < 64) tr[384 + 2 * j + w] = gtimer();
                tc_fence_after();
                // valid-key bits of this row in the tile, one word per 32-column chunk: committed prefix
                // keys [0, lim), or tree nodes on the row's root path
                const bool pre = j < npre;
                const int lim = pre ? L - j * kBN : T - (j - npre) * kBN;
                const uint32_t* aw = sanc + 256 * 4 * (pre ? 0 : j - npre);
                const bool full = pre && lim >= kBN;   // full prefix tile: no masking
                // valid-key word of global 32-column chunk cg
                auto valid_word = [&](int cg) -> uint32_t {
                    const int n = lim - 32 * cg;
                    uint32_t vw = n >= 32 ? 0xffffffffu : (n <= 0 ? 0u : ((1u << n) - 1u));
                    if (!pre) vw &= aw[256 * cg];
                    return vw;
                };
                float mx;
                uint32_t sr[SPLIT ? 32 : 128];
                if (SPLIT) {
                    // two chunks of 32 columns, scores reloaded for the exp pass (TMEM reads are cheap;
                    // registers are not at 18 warps)
                    float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        tmem_ld32(t_s + 64 * hh + 32 * c, sr);
                        tmem_wait();
                        const uint32_t vw = full ? 0xffffffffu : valid_word(2 * hh + c);
#pragma unroll
                        for (int e = 0; e < 32; e += 2)
                            m4[(e >> 1) & 3] = fmax3(m4[(e >> 1) & 3], ((vw >> e) & 1u) ? __uint_as_float(sr[e]) : -INFINITY,
                                                     ((vw >> (e + 1)) & 1u) ? __uint_as_float(sr[e + 1]) : -INFINITY);
                    }
                    mx = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
                    if (tr0 && j < 64) tr[640 + 4 * j + 0] = gtimer();
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) tmem_ld32(t_s + 32 * c, sr + 32 * c);
                    tmem_wait();
                    if (tr0 && j < 64) tr[640 + 4 * j + 0] = gtimer();
                    if (!full) {   // partial tile: masked scores -> -inf
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const uint32_t vw = valid_word(c);
#pragma unroll
                            for (int e = 0; e < 32; ++e) sr[32 * c + e] = ((vw >> e) & 1u) ? sr[32 * c + e] : 0xff800000u;
                        }
                    }
                    // row max: 8 independent FMNMX3 chains (latency, not throughput, bounds this step)
                    float m8[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) m8[k] = fmaxf(__uint_as_float(sr[k]), __uint_as_float(sr[k + 8]));
#pragma unroll
                    for (int e = 16; e < 128; e += 16)
#pragma unroll
                        for (int k = 0; k < 8; k += 2)
                            m8[k >> 1] = fmax3(m8[k >> 1], __uint_as_float(sr[e + k]), __uint_as_float(sr[e + k + 1]));
#pragma unroll
                    for (int e = 8; e < 128; e += 16)
#pragma unroll
                        for (int k = 0; k < 8; k += 2)
                            m8[4 + (k >> 1)] = fmax3(m8[4 + (k >> 1)], __uint_as_float(sr[e + k]), __uint_as_float(sr[e + k + 1]));
                    mx = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
                }
                if (SPLIT) {   // combine with the other half (double-buffered by tile parity: no WAR barrier)
                    float* xm = xch + (((j & 1) * 2 + w) * 2) * 128;
                    xm[hh * 128 + r] = mx;
                    pair_sync();
                    mx = fmaxf(mx, xm[(hh ^ 1) * 128 + r]);
                }
                mx *= sl2;   // scale > 0
                if (tr0 && j < 64) tr[640 + 4 * j + 1] = gtimer();
                // lazy rescaling: keep the running max unless the new one exceeds it by > 8 (log2 units).
                // tcgen05.ld/st are warp-collective: the O rescale runs warp-wide whenever any lane needs
                // it (alpha = 1 for the others); each half rescales its own O columns.
                const bool need = mx > m_run + 8.f;
                const float alpha = need ? (m_run == -INFINITY ? 0.f : ex2(m_run - mx)) : 1.f;
                if (need) m_run = mx;
                l_run *= alpha;
                if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
                    for (int c = 0; c < kCols / 32; ++c) {
                        uint32_t orr[32];
                        tmem_ld32(t_o + kCols * hh + 32 * c, orr);
                        tmem_wait();
#pragma unroll
                        for (int e = 0; e < 32; ++e) orr[e] = __float_as_uint(__uint_as_float(orr[e]) * alpha);
                        tmem_st32(t_o + kCols * hh + 32 * c, orr);
                    }
                    tmem_st_wait();
                }
                const float mu = m_run == -INFINITY ? 0.f : m_run;
                // p = 2^(s·scale·log2e - m) (masked: 2^-inf = 0); paired FFMA2, 4 FADD2 sum chains; bf16 P
                // packed in place over the consumed scores, then written over S's columns (this half's keys
                // land in packed columns [kCols/2·hh, +kCols/2); with SPLIT both halves have loaded their S
                // before the max exchange, so neither overwrites the other's unread scores)
                // SPLIT: the two query tiles' exp phases alternate (tile 0 of KV tile j, tile 1 of j, tile 0 of
                // j+1, ...): the MUFU is shared by the whole SM, so each phase runs alone at its throughput
                // while the tensor core works on the other tile's PV + next S
                if (SPLIT && nw == 2) {
                    if (w == 1) mbar_wait(bar_pfull(0), j & 1);
                    else if (j > 0) mbar_wait(bar_pfull(1), (j - 1) & 1);
                }
                const uint64_t sc2 = f2pack(sl2, sl2), nm2 = f2pack(-mu, -mu);
                uint64_t acc[4] = {0, 0, 0, 0};
                auto exp_pair = [&](uint32_t s0, uint32_t s1, int e, float& p0, float& p1) {
                    const uint64_t a2 = ffma2(f2pack(__uint_as_float(s0), __uint_as_float(s1)), sc2, nm2);
                    if (POLY == 1 && (e & 3) == 3) {
                        ex2_poly2(a2, p0, p1);
                        if (!full) {   // the polynomial does not map -inf to 0
                            p0 = s0 == 0xff800000u ? 0.f : p0;
                            p1 = s1 == 0xff800000u ? 0.f : p1;
                        }
                    } else {
                        p0 = ex2(__uint_as_float((uint32_t)a2));
                        p1 = ex2(__uint_as_float((uint32_t)(a2 >> 32)));
                    }
                };
                if (SPLIT) {
                    // this half's 64 keys -> packed P columns [32·hh, 32·hh + 32), 16 per chunk
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        uint32_t pk[16];
                        tmem_ld32(t_s + 64 * hh + 32 * c, sr);
                        tmem_wait();
                        const uint32_t vw = full ? 0xffffffffu : valid_word(2 * hh + c);
#pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            float p0, p1;
                            exp_pair(((vw >> (2 * e)) & 1u) ? sr[2 * e] : 0xff800000u,
                                     ((vw >> (2 * e + 1)) & 1u) ? sr[2 * e + 1] : 0xff800000u, e, p0, p1);
                            acc[e & 3] = fadd2(acc[e & 3], f2pack(p0, p1));
                            pk[e] = pack_bf16(p0, p1);
                        }
                        // P of this half's keys goes over its own first score chunk (already consumed): keys
                        // [64·hh, +64) -> columns [64·hh, 64·hh + 32); the PV MMA reads them from there
                        tmem_st16(t_s + 64 * hh + 16 * c, pk);
                    }
                } else {
#pragma unroll
                    for (int e = 0; e < 64; ++e) {
                        float p0, p1;
                        exp_pair(sr[2 * e], sr[2 * e + 1], e, p0, p1);
                        acc[e & 3] = fadd2(acc[e & 3], f2pack(p0, p1));
                        sr[e] = pack_bf16(p0, p1);   // in place: sr[2e], sr[2e+1] are consumed (e <= 2e)
                        if (e == 31) tmem_st32(t_s, sr);   // P columns [0, 32): frees sr[0..31]
                    }
                    tmem_st32(t_s + 32, sr + 32);
                }
                if (tr0 && j < 64) tr[640 + 4 * j + 2] = gtimer();
                const uint64_t a01 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
                l_run += __uint_as_float((uint32_t)a01) + __uint_as_float((uint32_t)(a01 >> 32));
                tmem_st_wait();
                if (tr0 && j < 64) tr[640 + 4 * j + 3] = gtimer();
                tc_fence_before();
                if (tr && hh == 0 && lane == 0 && q4 == 0 && j < 64) tr[512 + 2 * j + w] = gtimer();
                mbar_arrive(bar_pfull(w));
            }
            // epilogue: O / l -> bf16 -> global (SPLIT: each half stores its 64 output columns; l = the sum of
            // the two halves' partial sums, which were rescaled identically)
            mbar_wait(bar_ofull(w), 0);
            tc_fence_after();
            if (SPLIT) {
                float* xl = xch + ((((nt & 1) * 2 + w) * 2) * 128);
                xl[hh * 128 + r] = l_run;
                pair_sync();
                l_run += xl[(hh ^ 1) * 128 + r];
            }
            const float inv = 1.f / l_run;
            uint4* orow = (uint4*)(prm.o + (((size_t)b * T + i) * Hq + kvh * grp + hg) * kD) + (kCols / 8) * hh;
#pragma unroll 1
            for (int c = 0; c < kCols / 32; ++c) {
                uint32_t orr[32];
                tmem_ld32(t_o + kCols * hh + 32 * c, orr);
                tmem_wait();
                if (vrow) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float* f = reinterpret_cast<const float*>(orr + 8 * e);
                        orow[4 * c + e] = make_uint4(pack_bf16(f[0] * inv, f[1] * inv), pack_bf16(f[2] * inv, f[3] * inv),
                                                     pack_bf16(f[4] * inv, f[5] * inv), pack_bf16(f[6] * inv, f[7] * inv));
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

// ---------------------------------------------------------------------------
// K7b attn_db_kernel (bf16, D = 128): 64-key K/V tiles with double-buffered scores.  Same rows, mask and
// online softmax as attn_tc_kernel, but every query tile owns two 64-column score buffers in TMEM (tile w:
// columns [128w, 128w + 64) and [128w + 64, 128w + 128); O at [256 + 128w, +128)), so the tensor core
// computes S_w(j+2) into the buffer just released by P_w(j)·V while the softmax works on S_w(j+1): the
// softmax never waits for its next scores, and the MUFU-bound exp phases of the two tiles overlap the
// tensor core instead of alternating with it.  Per KV tile j and query tile w the MMA warp issues
//   [wait P_w(j)] O_w += P_w(j)·V_j (4 MMAs, K = 64), commit odone_w;  S_w(j+2) = Q_w·K_{j+2}ᵀ (8 MMAs,
//   N = 64) into buffer j & 1, commit sfull_w[j & 1]
// (in-order tensor pipe: S_w(j+2) overwrites P_w(j) only after the PV has read it).  The lazy O rescale of
// iteration j first waits odone_w for PV_w(j-1) (the only PV that can still be in flight).
// ---------------------------------------------------------------------------
#ifndef STREE_ATTN_DB_POLY
#define STREE_ATTN_DB_POLY 0
#endif
constexpr int kDbPoly = STREE_ATTN_DB_POLY;   // every kDbPoly-th exp pair on the FMA pipe (0: all on the MUFU)
constexpr int kBN2 = 64;                 // keys per K/V tile
constexpr int kStages2 = 4;              // K/V ring depth (same bytes as 2 x 128 keys)
constexpr int kHalfK2 = kBN2 * 128;      // 64 keys x 64 elements (128 B rows), swizzle-128B = 8 KB
constexpr int kTileK2 = 2 * kHalfK2;     // 64 keys x 128 elements

struct Smem2 {
    static constexpr int Q = 0;                          // 2 query tiles (kTile each)
    static constexpr int K = Q + 2 * kTile;              // kStages2 key tiles
    static constexpr int V = K + kStages2 * kTileK2;     // kStages2 value tiles
    static constexpr int PAR = V + kStages2 * kTileK2;   // parent[256] int
    static constexpr int ANC = PAR + kMaxNodes * 4;      // ancestor bits of each softmax row: [8 words][256 rows]
    static constexpr int BAR = ANC + kMaxWords * 256 * 4;
    // barriers: q, kfull[4], kempty[4], vfull[4], vempty[4], sfull[2 tiles][2 bufs], pfull[2][2], odone[2], ofull[2]
    static constexpr int NBAR = 1 + 4 * kStages2 + 4 + 4 + 2 + 2;
    static constexpr int TMEMP = BAR + NBAR * 8;
    static constexpr int TOTAL = TMEMP + 16;
    static_assert(TOTAL + 1024 <= 227 * 1024, "shared memory budget");
};

constexpr int kThreadsDb = 352;   // warp 0 TMA, warps 1 / 10 MMA issuers of query tile 0 / 1, warps 2-9 softmax
__global__ void __launch_bounds__(kThreadsDb, 1)
    attn_db_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_kc,
                   const __grid_constant__ CUtensorMap tm_vc, const __grid_constant__ CUtensorMap tm_kn,
                   const __grid_constant__ CUtensorMap tm_vn, const AttnParams prm) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sb = smem_u32(sm);
    const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
    const int T = prm.T, Hq = prm.Hq, Hkv = prm.Hkv, grp = Hq / Hkv;
    const int b = blockIdx.x / (Hkv * prm.npairs);
    const int rem = blockIdx.x % (Hkv * prm.npairs);
    const int kvh = rem / prm.npairs, pr = rem % prm.npairs;
    const int nmt = (T * grp + kBM - 1) / kBM;
    const int nw = min(2, nmt - 2 * pr);               // query tiles of this CTA (1 or 2)

    const uint32_t bar0 = sb + Smem2::BAR;
    const uint32_t BAR_Q = bar0;
    auto bar_kfull = [&](int s) { return bar0 + 8 + 8 * s; };
    auto bar_kempty = [&](int s) { return bar0 + 8 + 8 * kStages2 + 8 * s; };
    auto bar_vfull = [&](int s) { return bar0 + 8 + 16 * kStages2 + 8 * s; };
    auto bar_vempty = [&](int s) { return bar0 + 8 + 24 * kStages2 + 8 * s; };
    const uint32_t bar1 = bar0 + 8 + 32 * kStages2;
    auto bar_sfull = [&](int w, int u) { return bar1 + 8 * (2 * w + u); };
    auto bar_pfull = [&](int w, int u) { return bar1 + 32 + 8 * (2 * w + u); };
    auto bar_odone = [&](int w) { return bar1 + 64 + 8 * w; };
    auto bar_ofull = [&](int w) { return bar1 + 80 + 8 * w; };
    uint32_t* tmem_slot = (uint32_t*)(sm + Smem2::TMEMP);
    int* sp = (int*)(sm + Smem2::PAR);

    if (tid == 0) {
        mbar_init(BAR_Q, 1);
        for (int s = 0; s < kStages2; ++s) {   // a K / V stage is free once every query tile has consumed it
            mbar_init(bar_kfull(s), 1);
            mbar_init(bar_kempty(s), nw);
            mbar_init(bar_vfull(s), 1);
            mbar_init(bar_vempty(s), nw);
        }
        for (int w = 0; w < 2; ++w) {
            for (int u = 0; u < 2; ++u) {
                mbar_init(bar_sfull(w, u), 1);
                mbar_init(bar_pfull(w, u), 128);
            }
            mbar_init(bar_odone(w), 1);
            mbar_init(bar_ofull(w), 1);
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    int n_early = 0;
    auto issue_kv = [&](int j, bool pre, int key0) {
        const int s = j % kStages2;
        mbar_expect_tx(bar_kfull(s), kTileK2);
        for (int hf = 0; hf < 2; ++hf)
            tma_load_4d(sb + Smem2::K + s * kTileK2 + hf * kHalfK2, pre ? &tm_kc : &tm_kn, bar_kfull(s), 64 * hf, kvh, key0, b);
        mbar_expect_tx(bar_vfull(s), kTileK2);
        for (int hf = 0; hf < 2; ++hf)
            tma_load_4d(sb + Smem2::V + s * kTileK2 + hf * kHalfK2, pre ? &tm_vc : &tm_vn, bar_vfull(s), 64 * hf, kvh, key0, b);
    };
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tm_q); tma_prefetch(&tm_kc); tma_prefetch(&tm_vc); tma_prefetch(&tm_kn); tma_prefetch(&tm_vn);
        if (prm.early) {   // EARLY_STATE: the first prefix tiles before the dependency wait (as attn_tc_kernel)
            const int Le = prm.cache_len[b];
            if (Le > 0 && Le <= prm.S) {
                n_early = min(kStages2, (Le + kBN2 - 1) / kBN2);
                for (int j = 0; j < n_early; ++j) issue_kv(j, true, j * kBN2);
            }
        }
    }
    // tree validation (PAPER.md:90 ordering, R5) and the committed prefix length: before the dependency
    // wait under EARLY_TREE + EARLY_STATE (the tree and the cache length are not written by the preceding kernel)
    const bool early_prologue = prm.early && prm.early_tree;
    if (!early_prologue) pdl_wait();
    int bad = 0;
    for (int v = tid; v < T; v += (int)blockDim.x) {
        const int p = prm.parent[(size_t)b * T + v];
        sp[v] = p;
        if (v == 0 ? p != -1 : (p < 0 || p >= v)) bad = v == 0 ? 1 : 2;
    }
    const int L = prm.cache_len[b];
    const int any1 = __syncthreads_or(bad == 1);
    const int any2 = __syncthreads_or(bad == 2);
    if (early_prologue) pdl_wait();
    int code = any1 ? 1 : (any2 ? 2 : ((L < 0 || L > prm.S) ? kDev_Capacity : 0));
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const int npre = code ? 0 : (L + kBN2 - 1) / kBN2;   // prefix tiles
    const int ntr = (T + kBN2 - 1) / kBN2;               // tree tiles
    const int nt = npre + ntr;

    if (code) {
        if (tid == 0 && rem == 0) report(prm.dev_status, code);
        if (warp == 0 && lane == 0)   // drain the early loads before the CTA exits
            for (int j = 0; j < n_early; ++j) {
                mbar_wait(bar_kfull(j), 0);
                mbar_wait(bar_vfull(j), 0);
            }
        if (warp >= 2) {   // zero this CTA's output rows
            const int w = (warp - 2) >> 2, r = 32 * (warp & 3) + lane;
            if (w < nw) {
                const int rr = (2 * pr + w) * kBM + r, i = rr / grp, hg = rr % grp;
                if (i < T) {
                    uint4* orow = (uint4*)(prm.o + (((size_t)b * T + i) * Hq + kvh * grp + hg) * kD);
#pragma unroll
                    for (int c = 0; c < kD / 8; ++c) orow[c] = make_uint4(0, 0, 0, 0);
                }
            }
        }
    } else if (warp == 0) {
        // ---- TMA producer ----
        if (lane == 0) {
            mbar_expect_tx(BAR_Q, nw * kTile);
            for (int w = 0; w < nw; ++w) {
                const int node0 = (2 * pr + w) * (kBM / grp);
                for (int hf = 0; hf < 2; ++hf)
                    tma_load_4d(sb + Smem2::Q + w * kTile + hf * kHalf, &tm_q, BAR_Q, 64 * hf, kvh * grp, node0, b);
            }
            for (int j = n_early; j < nt; ++j) {
                const int s = j % kStages2, u = j / kStages2;
                const bool pre = j < npre;
                const int key0 = pre ? j * kBN2 : (j - npre) * kBN2;
                mbar_wait(bar_kempty(s), (u & 1) ^ 1);
                mbar_wait(bar_vempty(s), (u & 1) ^ 1);
                issue_kv(j, pre, key0);
            }
        }
    } else if (warp == 1 || warp == 10) {
        // ---- MMA issuers, one warp per query tile (warp 1: tile 0, warp 10: tile 1; converged, one elected lane
        // issues): each tile's MMAs are issued and committed by its own thread, so a tile waits only for its own
        // P and for the K / V ring, never for the other tile (tcgen05.commit tracks the issuing thread's MMAs) ----
        const int w = warp == 1 ? 0 : 1;
        if (w < nw) {
            const uint32_t id_s = idesc(kFmtBF16, 0, kBM, kBN2);   // S = Q·Kᵀ: A, B K-major, N = 64 keys
            const uint32_t id_o = idesc(kFmtBF16, 1, kBM, kD);     // O += P·V: A in TMEM, B (V) MN-major
            auto issue_s = [&](int j) {   // S_w(j) into score buffer j & 1 of tile w
                const int s = j % kStages2;
#pragma unroll
                for (int kk = 0; kk < kD / 16; ++kk) {
                    const uint64_t ad = sdesc(sb + Smem2::Q + w * kTile + (kk >> 2) * kHalf, 16, 1024) + (uint64_t)((kk & 3) * 2);
                    const uint64_t bd = sdesc(sb + Smem2::K + s * kTileK2 + (kk >> 2) * kHalfK2, 16, 1024) + (uint64_t)((kk & 3) * 2);
                    mma_f16_w(tmem + 128 * w + 64 * (j & 1), ad, bd, id_s, kk > 0);
                }
                tc_commit_w(bar_sfull(w, j & 1));
            };
            mbar_wait(BAR_Q, 0);
            for (int j = 0; j < 2 && j < nt; ++j) {   // the first two score tiles
                mbar_wait(bar_kfull(j % kStages2), (j / kStages2) & 1);
                tc_fence_after();
                issue_s(j);
                tc_commit_w(bar_kempty(j % kStages2));
            }
            for (int j = 0; j < nt; ++j) {
                const int s = j % kStages2, u = j / kStages2;
                const int j2 = j + 2, s2 = j2 % kStages2, u2 = j2 / kStages2;
                mbar_wait(bar_pfull(w, j & 1), (j >> 1) & 1);
                mbar_wait(bar_vfull(s), u & 1);
                tc_fence_after();
                const uint64_t vd = sdesc(sb + Smem2::V + s * kTileK2, kHalfK2, 1024);
#pragma unroll
                for (int kk = 0; kk < kBN2 / 16; ++kk)
                    mma_f16_ts_w(tmem + 256 + 128 * w, tmem + 128 * w + 64 * (j & 1) + 8 * kk, vd + (uint64_t)(kk * 128),
                                 id_o, (j > 0 || kk > 0) ? 1u : 0u);
                tc_commit_w(bar_odone(w));
                tc_commit_w(bar_vempty(s));
                if (j == nt - 1) tc_commit_w(bar_ofull(w));
                if (j2 < nt) {
                    mbar_wait(bar_kfull(s2), u2 & 1);
                    tc_fence_after();
                    issue_s(j2);
                    tc_commit_w(bar_kempty(s2));
                }
            }
        }
    } else {
        // ---- softmax: thread = query row = TMEM lane ----
        const int w = (warp - 2) >> 2, q4 = warp & 3, r = 32 * q4 + lane;
        if (w < nw) {
            const int rr = (2 * pr + w) * kBM + r, i = rr / grp, hg = rr % grp;
            const bool vrow = i < T;
            // ancestor bits of the row's node, word-major in smem (conflict-free reads)
            uint32_t* sanc = (uint32_t*)(sm + Smem2::ANC) + 128 * w + r;
            {
                uint32_t anc[kMaxWords];
#pragma unroll
                for (int q = 0; q < kMaxWords; ++q) anc[q] = 0u;
                if (vrow)
                    for (int v = i; v >= 0; v = sp[v]) {
#pragma unroll
                        for (int q = 0; q < kMaxWords; ++q) anc[q] |= ((v >> 5) == q) ? (1u << (v & 31)) : 0u;
                    }
#pragma unroll
                for (int q = 0; q < kMaxWords; ++q) sanc[256 * q] = anc[q];
            }
            const uint32_t lane_base = tmem + ((uint32_t)(32 * q4) << 16);
            const uint32_t t_o = lane_base + 256 + 128 * w;
            const float sl2 = prm.scale_log2;
            float m_run = -INFINITY, l_run = 0.f;
            for (int j = 0; j < nt; ++j) {
                const int buf = j & 1;
                const uint32_t t_s = lane_base + 128 * w + 64 * buf;
                mbar_wait(bar_sfull(w, buf), (j >> 1) & 1);
                tc_fence_after();
                // valid-key bits of this row in the tile, one word per 32-column chunk: committed prefix keys
                // [0, lim), or tree nodes on the row's root path
                const bool pre = j < npre;
                const int lim = pre ? L - j * kBN2 : T - (j - npre) * kBN2;
                const uint32_t* aw = sanc + 256 * 2 * (pre ? 0 : j - npre);
                const bool full = pre && lim >= kBN2;   // full prefix tile: no masking
                auto valid_word = [&](int cg) -> uint32_t {
                    const int n = lim - 32 * cg;
                    uint32_t vw = n >= 32 ? 0xffffffffu : (n <= 0 ? 0u : ((1u << n) - 1u));
                    if (!pre) vw &= aw[256 * cg];
                    return vw;
                };
                uint32_t sr[64];
                tmem_ld32(t_s, sr);
                tmem_ld32(t_s + 32, sr + 32);
                tmem_wait();
                if (!full) {   // partial tile: masked scores -> -inf
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const uint32_t vw = valid_word(c);
#pragma unroll
                        for (int e = 0; e < 32; ++e) sr[32 * c + e] = ((vw >> e) & 1u) ? sr[32 * c + e] : 0xff800000u;
                    }
                }
                // row max: 8 independent FMNMX3 chains
                float m8[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) m8[k] = fmaxf(__uint_as_float(sr[k]), __uint_as_float(sr[k + 8]));
#pragma unroll
                for (int e = 16; e < 64; e += 16)
#pragma unroll
                    for (int k = 0; k < 8; k += 2)
                        m8[k >> 1] = fmax3(m8[k >> 1], __uint_as_float(sr[e + k]), __uint_as_float(sr[e + k + 1]));
#pragma unroll
                for (int e = 24; e < 64; e += 16)
#pragma unroll
                    for (int k = 0; k < 8; k += 2)
                        m8[4 + (k >> 1)] = fmax3(m8[4 + (k >> 1)], __uint_as_float(sr[e + k]), __uint_as_float(sr[e + k + 1]));
                float mx = fmax3(fmax3(m8[0], m8[1], m8[2]), fmax3(m8[3], m8[4], m8[5]), fmaxf(m8[6], m8[7]));
                mx *= sl2;   // scale > 0
                // lazy rescaling: keep the running max unless the new one exceeds it by > 8 (log2 units); the
                // rescale of O waits for PV_w(j-1), the only P·V that can still be accumulating into O
                const bool need = mx > m_run + 8.f;
                const float alpha = need ? (m_run == -INFINITY ? 0.f : ex2(m_run - mx)) : 1.f;
                if (need) m_run = mx;
                l_run *= alpha;
                if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
                    mbar_wait(bar_odone(w), (j - 1) & 1);
                    tc_fence_after();
#pragma unroll 1
                    for (int c = 0; c < kD / 32; ++c) {
                        uint32_t orr[32];
                        tmem_ld32(t_o + 32 * c, orr);
                        tmem_wait();
#pragma unroll
                        for (int e = 0; e < 32; ++e) orr[e] = __float_as_uint(__uint_as_float(orr[e]) * alpha);
                        tmem_st32(t_o + 32 * c, orr);
                    }
                    tmem_st_wait();
                }
                const float mu = m_run == -INFINITY ? 0.f : m_run;
                // p = 2^(s·scale·log2e - m) (masked: 2^-inf = 0); paired FFMA2, 4 FADD2 sum chains; bf16 P packed
                // in place over the consumed scores, then written over the buffer's first 32 columns
                const uint64_t sc2 = f2pack(sl2, sl2), nm2 = f2pack(-mu, -mu);
                uint64_t acc[4] = {0, 0, 0, 0};
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    const uint64_t a2 = ffma2(f2pack(__uint_as_float(sr[2 * e]), __uint_as_float(sr[2 * e + 1])), sc2, nm2);
                    float p0, p1;
                    if (kDbPoly > 0 && e % kDbPoly == kDbPoly - 1) {   // this pair's 2^x on the FMA pipe
                        ex2_poly2(a2, p0, p1);
                        if (!full) {   // the polynomial does not map -inf to 0
                            p0 = sr[2 * e] == 0xff800000u ? 0.f : p0;
                            p1 = sr[2 * e + 1] == 0xff800000u ? 0.f : p1;
                        }
                    } else {
                        p0 = ex2(__uint_as_float((uint32_t)a2));
                        p1 = ex2(__uint_as_float((uint32_t)(a2 >> 32)));
                    }
                    acc[e & 3] = fadd2(acc[e & 3], f2pack(p0, p1));
                    sr[e] = pack_bf16(p0, p1);   // in place: sr[2e], sr[2e+1] are consumed (e <= 2e)
                }
                tmem_st32(t_s, sr);
                const uint64_t a01 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
                l_run += __uint_as_float((uint32_t)a01) + __uint_as_float((uint32_t)(a01 >> 32));
                tmem_st_wait();
                tc_fence_before();
                mbar_arrive(bar_pfull(w, buf));
            }
            // epilogue: O / l -> bf16 -> global
            mbar_wait(bar_ofull(w), 0);
            tc_fence_after();
            const float inv = 1.f / l_run;
            uint4* orow = (uint4*)(prm.o + (((size_t)b * T + i) * Hq + kvh * grp + hg) * kD);
#pragma unroll 1
            for (int c = 0; c < kD / 32; ++c) {
                uint32_t orr[32];
                tmem_ld32(t_o + 32 * c, orr);
                tmem_wait();
                if (vrow) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const float* f = reinterpret_cast<const float*>(orr + 8 * e);
                        orow[4 * c + e] = make_uint4(pack_bf16(f[0] * inv, f[1] * inv), pack_bf16(f[2] * inv, f[3] * inv),
                                                     pack_bf16(f[4] * inv, f[5] * inv), pack_bf16(f[6] * inv, f[7] * inv));
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

// ---------------------------------------------------------------------------
// K8 KV commit: append the accepted path's K/V rows to the cache (one CTA per tree)
// ---------------------------------------------------------------------------
template <typename W>
__global__ void __launch_bounds__(256) kv_commit_kernel(const W* __restrict__ k_new, const W* __restrict__ v_new,
                                                        const int32_t* __restrict__ parent,
                                                        const int32_t* __restrict__ path,
                                                        const int32_t* __restrict__ path_len, W* k_cache, W* v_cache,
                                                        int32_t* cache_len, int T, int S, int row_words,
                                                        int32_t* dev_status) {
    __shared__ int s_ok, s_L, s_r;
    __shared__ int s_path[kMaxNodes];
    pdl_wait();
    const int b = blockIdx.x, tid = threadIdx.x;
    // path validation in parallel (root-anchored, parent-linked: warp 0, 32 path nodes per round, all loads of a
    // round in flight together) — a serial walk cost two dependent DRAM latencies per path node
    if (tid < 32) {
        const int r = path_len[b], L = cache_len[b];
        int ok = (r >= 1 && r <= T) ? 1 : 0;
        if (ok) {
            for (int s0 = 0; s0 < r; s0 += 32) {
                const int s = s0 + tid;
                int v = -1, pv = -1, par = -2;
                if (s < r) {
                    v = path[(size_t)b * T + s];
                    pv = s > 0 ? path[(size_t)b * T + s - 1] : -1;
                    if (v >= 0 && v < T) par = parent ? parent[(size_t)b * T + v] : pv;
                }
                bool good = s >= r || (v >= 0 && v < T && (s == 0 ? v == 0 : par == pv));
                if (s < r && good) s_path[s] = v;
                if (!__all_sync(0xffffffffu, good)) { ok = 0; break; }
            }
        }
        if (tid == 0) {
            int code = ok ? 0 : STREE_DEV_BAD_PATH;
            if (ok && (L < 0 || L + r > S)) code = kDev_Capacity;
            if (code) report(dev_status, code);
            s_ok = code == 0;
            s_L = L;
            s_r = r;
        }
    }
    __syncthreads();
    if (!s_ok) return;
    const int L = s_L, r = s_r;
    for (int k = tid; k < r * row_words; k += blockDim.x) {
        const int s = k / row_words, c = k % row_words;
        const size_t src = ((size_t)b * T + s_path[s]) * row_words + c;
        const size_t dst = ((size_t)b * S + L + s) * row_words + c;
        k_cache[dst] = k_new[src];
        v_cache[dst] = v_new[src];
    }
    __syncthreads();
    if (tid == 0) cache_len[b] = L + r;
}

}  // namespace attn
}  // namespace stree

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

// bf16 4-D map over [d3][d2][d1][d0] (d0 innermost, contiguous), box {64, b1, b2, 1}, swizzle 128B
bool make_map4(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3, uint32_t b1,
               uint32_t b2) {
    return stree::host::tmap_4d_bf16(m, base, d0, d1, d2, d3, b1, b2);
}

}  // namespace

namespace {
unsigned long long* g_attn_trace = nullptr;
}
// Debug hook (not part of the ABI): globaltimer stamps of CTA 0's pipeline events, 1024 u64.
extern "C" void stree_debug_attn_trace(unsigned long long* dev_buf) { g_attn_trace = dev_buf; }

extern "C" int stree_attn_tc_supports(const stree_attn_dims* d) {
    if (!d || d->io_dtype != STREE_BF16 || d->head_dim != stree::attn::kD) return 0;
    if (d->n_kv_heads < 1 || d->n_q_heads % d->n_kv_heads) return 0;
    const int grp = d->n_q_heads / d->n_kv_heads;
    if (grp > 128 || stree::attn::kBM % grp) return 0;
    if (d->n_nodes < 1 || d->n_nodes > stree::kMaxNodes || d->cache_cap < 1) return 0;
    return 1;
}

extern "C" int stree_launch_tree_attn(const stree_attn_dims* d, const void* q, const void* k_new, const void* v_new,
                                      const void* k_cache, const void* v_cache, const int32_t* cache_len,
                                      const int32_t* parent, float scale, void* o, int32_t* dev_status, int use_tc,
                                      cudaStream_t s) {
    using namespace stree::attn;
    const int B = d->batch, T = d->n_nodes, Hq = d->n_q_heads, Hkv = d->n_kv_heads, D = d->head_dim, S = d->cache_cap;
    cudaError_t e;
    if (use_tc) {
        const int grp = Hq / Hkv;
        CUtensorMap mq, mkc, mvc, mkn, mvn;
        bool ok = make_map4(&mq, q, D, Hq, T, B, grp, kBM / grp) &&
                  make_map4(&mkc, k_cache, D, Hkv, S, B, 1, kBN) && make_map4(&mvc, v_cache, D, Hkv, S, B, 1, kBN) &&
                  make_map4(&mkn, k_new, D, Hkv, T, B, 1, kBN) && make_map4(&mvn, v_new, D, Hkv, T, B, 1, kBN);
        if (!ok) return (int)cudaErrorInvalidValue;
        AttnParams prm{};
        prm.cache_len = cache_len; prm.parent = parent; prm.o = (__nv_bfloat16*)o; prm.dev_status = dev_status;
        prm.T = T; prm.Hq = Hq; prm.Hkv = Hkv; prm.S = S;
        const int nmt = (T * grp + kBM - 1) / kBM;
        prm.npairs = (nmt + 1) / 2;
        prm.scale_log2 = scale * 1.4426950408889634f;
        prm.trace = g_attn_trace;
        prm.early = (stree_launch_flags_get() & STREE_LAUNCH_EARLY_STATE) ? 1 : 0;
        prm.early_tree = (stree_launch_flags_get() & STREE_LAUNCH_EARLY_TREE) ? 1 : 0;
        static const int dbuf = [] {
            const char* v = std::getenv("STREE_ATTN_DB");   // 1 (default): 64-key double-buffered kernel
            return v && v[0] ? std::atoi(v) : 1;
        }();
        if (dbuf) {
            CUtensorMap mkc2, mvc2, mkn2, mvn2;
            if (!(make_map4(&mkc2, k_cache, D, Hkv, S, B, 1, kBN2) && make_map4(&mvc2, v_cache, D, Hkv, S, B, 1, kBN2) &&
                  make_map4(&mkn2, k_new, D, Hkv, T, B, 1, kBN2) && make_map4(&mvn2, v_new, D, Hkv, T, B, 1, kBN2)))
                return (int)cudaErrorInvalidValue;
            const size_t smem2 = Smem2::TOTAL + 1024;
            e = stree::host::smem_attr((const void*)attn_db_kernel, (int)smem2);
            if (e != cudaSuccess) return (int)e;
            e = stree::launch_k(attn_db_kernel, dim3(B * Hkv * prm.npairs), dim3(kThreadsDb), smem2, s, mq, mkc2, mvc2,
                                mkn2, mvn2, prm);
            if (e != cudaSuccess) return (int)e;
            return (int)cudaGetLastError();
        }
        const size_t smem = Smem::TOTAL + 1024;
        static const int poly = [] {
            const char* v = std::getenv("STREE_ATTN_POLY");   // tuning knob; default 0 (measured best)
            return v && v[0] ? std::atoi(v) : 0;
        }();
        static const int split = [] {
            const char* v = std::getenv("STREE_ATTN_SPLIT");   // tuning knob; default 0 (measured faster)
            return v && v[0] ? std::atoi(v) : 0;
        }();
        auto k = split ? (poly == 1 ? attn_tc_kernel<1, true> : attn_tc_kernel<0, true>)
                       : (poly == 1 ? attn_tc_kernel<1, false> : attn_tc_kernel<0, false>);
        e = stree::host::smem_attr((const void*)k, (int)smem);
        if (e != cudaSuccess) return (int)e;
        e = stree::launch_k(k, dim3(B * Hkv * prm.npairs), dim3(split ? kThreadsSplit : kThreads), smem, s, mq, mkc,
                            mvc, mkn, mvn, prm);
    } else {
        dim3 grid(Hq, T, B);
        if (d->io_dtype == STREE_BF16)
            e = stree::launch_k(attn_simt_kernel<__nv_bfloat16>, grid, dim3(32), 0, s, (const __nv_bfloat16*)q,
                                (const __nv_bfloat16*)k_new, (const __nv_bfloat16*)v_new,
                                (const __nv_bfloat16*)k_cache, (const __nv_bfloat16*)v_cache, cache_len, parent, scale,
                                (__nv_bfloat16*)o, T, Hq, Hkv, D, S, dev_status);
        else
            e = stree::launch_k(attn_simt_kernel<float>, grid, dim3(32), 0, s, (const float*)q, (const float*)k_new,
                                (const float*)v_new, (const float*)k_cache, (const float*)v_cache, cache_len, parent,
                                scale, (float*)o, T, Hq, Hkv, D, S, dev_status);
    }
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
}

extern "C" int stree_launch_kv_commit(const stree_attn_dims* d, const void* k_new, const void* v_new,
                                      const int32_t* parent, const int32_t* path, const int32_t* path_len,
                                      void* k_cache, void* v_cache, int32_t* cache_len, int32_t* dev_status,
                                      cudaStream_t s) {
    using namespace stree::attn;
    const size_t row_bytes = (size_t)d->n_kv_heads * d->head_dim * (d->io_dtype == STREE_BF16 ? 2 : 4);
    cudaError_t e;
    if (row_bytes % 16 == 0)
        e = stree::launch_k(kv_commit_kernel<uint4>, dim3(d->batch), dim3(256), 0, s, (const uint4*)k_new,
                            (const uint4*)v_new, parent, path, path_len, (uint4*)k_cache, (uint4*)v_cache, cache_len,
                            d->n_nodes, d->cache_cap, (int)(row_bytes / 16), dev_status);
    else
        e = stree::launch_k(kv_commit_kernel<uint32_t>, dim3(d->batch), dim3(256), 0, s, (const uint32_t*)k_new,
                            (const uint32_t*)v_new, parent, path, path_len, (uint32_t*)k_cache, (uint32_t*)v_cache,
                            cache_len, d->n_nodes, d->cache_cap, (int)(row_bytes / 4), dev_status);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
}
