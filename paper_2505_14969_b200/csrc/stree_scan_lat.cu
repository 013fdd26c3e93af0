// K2s — stree_tree_scan / stree_replay_scan for small batches: one (tree, head) per CTA, built for
// latency (the paper's batch-1 setting; BASELINE configs c2 / c3).
//
// Same arithmetic as K2 (stree_scan_tc.cu; PAPER.md:91-102 with the Mamba-2 realisation of SURVEY R1-R3):
//     G   = C·Bᵀ                 (T x T, K = N)      tcgen05 kind::f16, A = C, B = B (smem)
//     Y0  = C·h0ᵀ                (T x P, K = N)      tcgen05 kind::f16, h0 = hi + lo split into two bf16
//                                                    tiles: C·hiᵀ + C·loᵀ in one accumulator
//     Y'  = (L∘G∘c)·X            (T x P, K = T)      tcgen05 kind::f16, A = masked weights in TMEM (TS)
//     y   = e^{Λ_i}(Y0 + Y') + D x                   (factorised decay; direct e^{Λi-Λj} when min Λ < -64)
// and, in the replay variant, the activation replay of the previous tree's accepted path applied on chip
// to the state tile before Y0 reads it (Alg. 1 l.123-124), the committed tile TMA-stored in
// place.  The hi/lo split keeps 16 mantissa bits of the fp32 state (tf32 keeps 10), so Y0 is more
// accurate than a kind::tf32 product, and it needs no conversion of C after the inputs land.
//
// Why a separate kernel: with B·H ≤ #SMs there is one head per CTA and nothing to pipeline; a layer's
// time is its dependency chain after the PDL wait (inputs land -> G -> masked weights -> Y' -> y) plus
// the launch boundary (measured floor of an empty dependent kernel in a graph: 0.71 us, tools/pdl_floor.cu).
// Everything that does not depend on the preceding kernel runs before the wait, and the chain after it is
// one DRAM latency plus the tensor-core work:
//  * ≈ 105 KB of shared memory and 256 TMEM columns per CTA: two CTAs fit on an SM, so under PDL the next
//    layer's CTAs are resident while this layer runs (grids of at most #SMs/2 CTAs take one SM each, so the
//    next layer lands on other SMs);
//  * at entry, before any barrier: the state tile by TMA (STREE_LAUNCH_EARLY_STATE), the tree operands
//    (parent, A_h, D_h, dt: EARLY_TREE / EARLY_DT) and the previous tree's accepted path (EARLY_REPLAY) —
//    one DRAM latency for all of them;
//  * before the wait, on the aux warps (SM sub-partitions 2, 3, so that the next layer's pre-wait work,
//    co-resident on the SM, stays off the sub-partitions of this layer's row warps): tree validation, ancestor
//    bits and the pointer-jumping segsum (warp 3, published to the row warps through shared memory), the
//    replay prologue (path validation, coefficients, operands gathered with cp.async); then, on all eight
//    warps, the activation replay of the state tile (packed FFMA2) and its hi/lo split;
//  * after the wait: C, B, x by TMA (dt too when not read early), all in flight together; G = C·Bᵀ and then
//    Y0 are issued the moment C, B land; four row warps (two per TMEM lane quadrant of the 64 node rows, on
//    key-column halves) build the masked weights straight into TMEM (no shared memory, no proxy fence) for a
//    TS-form Y'; the same warps write y from registers (64 contiguous bytes per thread); the aux warps store
//    the committed state tile (TMA, in place).
// Warps: 0, 1, 4, 5 row warps (masked weights, epilogue); 2, 3, 6, 7 aux (tree, replay, state); 8 TMA producer
// + MMA issuer (its own warp: the replay of the fused variant must never delay the MMAs).
// Accumulator rows 64-127 are never read (M = 128 MMAs, T ≤ 64 rows).
//
// Served: bf16 io, P = 64, N in {64, 128}, 1 <= T <= 64 (the launcher picks this kernel when B·H ≤ #SMs).
#include <cuda.h>

#include <cstdlib>

#include "stree_common.cuh"
#include "stree_host.cuh"
#include "stree_tc_ptx.cuh"

namespace stree {
namespace lat {
using namespace stree::tc;

constexpr int kP = 64;
constexpr int kAtom = 8192;               // 64 rows x 128 B, swizzle-128B
constexpr int kIssW = 8;                  // TMA producer + MMA issuer
constexpr int kThreads = 288;
constexpr int kRStage = 8;                // previous-path nodes staged on chip
constexpr int kRounds = 6;                // pointer-jumping rounds for T <= 64
constexpr uint32_t kCols = 256;           // TMEM columns
constexpr int kColG = 0;                  // G = C·Bᵀ, fp32 [0, 64)
constexpr int kColM = 64;                 // masked weights, bf16 packed two per column [64, 96)
constexpr int kColAcc = 128;              // Y0 (+ factorised Y') [128, 192)
constexpr int kColYd = 0;                 // direct-decay Y' over G's columns (G is dead once M' is built)
constexpr int kTraceWords = 32;           // debug timeline: u64 globaltimer stamps per CTA (STREE_TRACE builds)
#ifdef STREE_TRACE
constexpr bool kTrace = true;
#else
constexpr bool kTrace = false;
#endif

template <int NS, bool R>
struct Lay {
    static constexpr int kCbAtoms = NS / 64;
    static constexpr int CB = 0;                              // C bf16: atom a = columns [64a, 64a+64)
    static constexpr int BB = CB + kCbAtoms * kAtom;          // B bf16
    static constexpr int HL = BB + kCbAtoms * kAtom;          // split state, 64-column atoms of 128 rows:
                                                              // rows 0-63 = bf16(h0), rows 64-127 = bf16(h0 - hi)
    static constexpr int H0 = HL + kCbAtoms * 2 * kAtom;      // state tile: atom a = columns [32a, 32a+32), fp32
    static constexpr int X = H0 + (NS / 32) * kAtom;          // x tile (64 rows of 64 bf16)
    static constexpr int DT = X + kAtom;                      // dt of heads (h & ~3) .. +3, T rows of 16 B (TMA)
    static constexpr int CJ = DT + 64 * 16;                   // float [64]  c_j (factorised) / dt_j (direct)
    static constexpr int LM = CJ + 64 * 4;                    // float [64]  Λ_j
    static constexpr int BITS = LM + 64 * 4;                  // u64 [64]    ancestor row of node i
    static constexpr int MODE = BITS + 64 * 8;                // int [4]: decay mode, bad-tree code, D_h (bits)
    static constexpr int RPATH = MODE + 16;                   // int [kMaxNodes]
    static constexpr int RINFO = RPATH + (R ? kMaxNodes * 4 : 0);   // int [2]: r (0 = nothing), bad path
    static constexpr int RCOEF = RINFO + 16;                  // float [kRStage]
    static constexpr int RLAM = RCOEF + 32;                   // float [4]: λ_last, λ_{kRStage-1}, e^{λ_last}
    static constexpr int XPREV = RLAM + 16;                   // bf16 [kRStage][64]
    static constexpr int BPREV = XPREV + (R ? kRStage * kP * 2 : 0);    // bf16 [kRStage][NS]
    static constexpr int BAR = (BPREV + (R ? kRStage * NS * 2 : 0) + 7) & ~7;
    static constexpr int NBAR = 7;                            // cb, x, h, hs, g, m, acc
    static constexpr int TMEMP = BAR + NBAR * 8;
    static constexpr int TOTAL = TMEMP + 16;
    static_assert(2 * (TOTAL + 1024 + 1024) <= 228 * 1024, "two CTAs per SM");
};

struct Params {
    int B, T, H, G;
    const float* dt;
    const float* A;
    const float* D;
    const int32_t* parent;
    const float* h0p;            // the state [B][H][P][N] (read by the threads into registers)
    __nv_bfloat16* y;
    int32_t* dev_status;
    int has_h0, early_state, early_replay, early_tree;
    int early_dt;                // STREE_LAUNCH_EARLY_DT: the segsum runs before the dependency wait
    int dt_tma;                  // dt staged by TMA (needs H·4 % 16 == 0), else read by the row warps
    DtX dtx;                     // *_ex options: effective dt (bias, softplus)
    int d_pc;                    // *_ex options: D is [H][P]
    // replay (previous tree)
    int Tp;
    const __nv_bfloat16* x_prev;
    const float* dt_prev;
    const __nv_bfloat16* b_prev;
    const int32_t* parent_prev;
    const int32_t* path;
    const int32_t* path_len;
    unsigned long long* trace;   // [grid][kTraceWords] or NULL (STREE_TRACE builds only)
    // y destinations: n_ypeer buffers [B][T][y_heads][P], this call's heads at y_head_off (the local y:
    // one buffer, y_heads = H, offset 0; a head-sharded layer: every rank's full y, stree_yout)
    __nv_bfloat16* ypeer[STREE_MAX_Y_PEERS];
    int n_ypeer, y_heads, y_head_off;
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ uint64_t pk2(float2 v) { return ((uint64_t)__float_as_uint(v.y) << 32) | __float_as_uint(v.x); }
__device__ __forceinline__ float2 upk2(uint64_t d) { return make_float2(__uint_as_float((uint32_t)d), __uint_as_float((uint32_t)(d >> 32))); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {   // packed FFMA2
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)), "l"(pk2(c)));
    return upk2(d);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
    return upk2(d);
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
    uint64_t d;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk2(a)), "l"(pk2(b)));
    return upk2(d);
}

// Masked weights of one row warp (node row i = its TMEM lane, key columns [c0, c0 + 32)):
// M'_ij = L_ij G_ij c_j (factorised) or L_ij e^{min(Λi-Λj,0)} dt_j G_ij (direct), bf16, packed two keys per
// 32-bit TMEM column at [kColM + c0/2, +16) — the A operand of the TS-form Y' MMA.
template <bool FAC>
__device__ __forceinline__ void build_weights(uint32_t tq, int c0, uint64_t bits, float li, const float* cjw,
                                              const float* lmw, unsigned long long* tr) {
    uint32_t o[16], gv[32];
    tmem_ld32(tq + kColG + c0, gv);   // the 32 key columns in one load (one TMEM round trip)
    const uint32_t bw = (uint32_t)(bits >> c0);   // c0 in {0, 32}: this half's ancestor bits
    float cj[32];
#pragma unroll
    for (int k4 = 0; k4 < 8; ++k4) {   // c_j of the 32 keys: 8 broadcast 16-byte loads while the TMEM load is in flight
        const float4 v = reinterpret_cast<const float4*>(cjw + c0)[k4];
        cj[4 * k4] = v.x; cj[4 * k4 + 1] = v.y; cj[4 * k4 + 2] = v.z; cj[4 * k4 + 3] = v.w;
    }
    tmem_wait();
    if (kTrace && tr) tr[25] = gtimer();
#pragma unroll
    for (int k = 0; k < 32; k += 2) {
        const int j = c0 + k;
        float v0 = cj[k] * __uint_as_float(gv[k]);
        float v1 = cj[k + 1] * __uint_as_float(gv[k + 1]);
        if (!FAC) {
            v0 *= __expf(fminf(li - lmw[j], 0.f));
            v1 *= __expf(fminf(li - lmw[j + 1], 0.f));
        }
        o[k >> 1] = pack_bf16((bw & (1u << k)) ? v0 : 0.f, (bw & (2u << k)) ? v1 : 0.f);
    }
    if (kTrace && tr) tr[26] = gtimer();
    tmem_st16(tq + kColM + (c0 >> 1), o);
    tmem_st_wait();
    if (kTrace && tr) tr[27] = gtimer();
}

template <int NS, bool R, bool DPC = false>   // DPC: D is [H][P] (separate instantiation, no runtime branch)
__global__ void __launch_bounds__(kThreads, 2)
    lat_kernel(const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ CUtensorMap tm_b,
               const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_h,
               const __grid_constant__ CUtensorMap tm_dt, const Params prm) {
    using L = Lay<NS, R>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sb = smem_u32(sm);
    const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
    const int T = prm.T, H = prm.H;
    const int b = blockIdx.x / H, h = blockIdx.x % H;
    const int g = h / (H / prm.G);                        // group of head h (heads of a group contiguous)
    const uint32_t bar0 = sb + L::BAR;
    const uint32_t BAR_CB = bar0, BAR_X = bar0 + 8, BAR_H = bar0 + 16, BAR_HS = bar0 + 24, BAR_G = bar0 + 32,
                   BAR_M = bar0 + 40, BAR_ACC = bar0 + 48;
    const int Tp16 = (T + 15) & ~15;
    const bool early_h = prm.early_state && prm.has_h0;
    unsigned long long* const trace = (kTrace && prm.trace) ? prm.trace + (size_t)blockIdx.x * kTraceWords : nullptr;
    auto stamp = [&](int k) {
        if (kTrace && trace) trace[k] = gtimer();
    };
    if (tid == 0) stamp(0);
    if (kTrace && trace && tid == 0) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        trace[31] = smid;
    }

    // ---- operands of the pre-wait work, loaded at entry (one DRAM latency for all of them, under the caller's
    //      promises): tree warp 3 (lane: nodes lane, lane + 32): parent, A_h, D_h and, under EARLY_DT, raw dt;
    //      aux warps (u = 0..127): the previous tree's accepted path and its length.  The state tile comes by
    //      TMA (issuer, below). ----
    const bool row_warp = warp < 8 && (warp & 2) == 0;   // 0, 1, 4, 5: TMEM lanes 0-63 (SM sub-partitions 0, 1)
    const bool tree_warp = warp == 3;
    const bool early_lambda = prm.early_tree && prm.early_dt;
    int tpar[2] = {-1, -1};
    float tA = 0.f, tD = 0.f, tdt[2] = {0.f, 0.f};
    auto load_tree = [&](bool with_dt) {
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            const int i = lane + 32 * hf;
            tpar[hf] = i < T ? prm.parent[(size_t)b * T + i] : -1;
            if (with_dt) tdt[hf] = i < T ? prm.dt[((size_t)b * T + i) * H + h] : 0.f;
        }
        tA = prm.A[h];
        tD = prm.D ? prm.D[h] : 0.f;
    };
    if (tree_warp && prm.early_tree) load_tree(early_lambda);   // EARLY_TREE (+ EARLY_DT)
    int rp_len = 0, rp0 = 0, rp1 = 0;
    const int u = 32 * ((warp & 1) + 2 * (warp >> 2)) + lane;   // aux warps 2, 3, 6, 7 -> 0..127
    auto load_path = [&]() {
        rp_len = prm.path_len[b];
        rp0 = u < prm.Tp ? prm.path[(size_t)b * prm.Tp + u] : 0;
        rp1 = u + 128 < prm.Tp ? prm.path[(size_t)b * prm.Tp + u + 128] : 0;
    };
    if (R && warp < 8 && !row_warp && prm.early_replay) load_path();   // EARLY_REPLAY

    // ---- setup (overlaps the previous kernel under PDL): the issuer initialises the barriers and, under
    //      STREE_LAUNCH_EARLY_STATE, starts the state stream at once (the longest pre-wait chain: 32 KB,
    //      then the replay update and the hi/lo split) ----
    if (warp == kIssW) {
        if (lane == 0) {
            mbar_init(BAR_CB, 1);
            mbar_init(BAR_X, 1);
            mbar_init(BAR_H, 1);
            mbar_init(BAR_HS, 1);
            mbar_init(BAR_G, 1);
            mbar_init(BAR_M, 4);
            mbar_init(BAR_ACC, 1);
            fence_barrier_init();
            fence_proxy_async();
            if (early_h) {   // caller's promise: the state is not written by the preceding kernel
                mbar_expect_tx(BAR_H, NS * kP * 4);
#pragma unroll 1
                for (int a = 0; a < NS / 32; ++a)
                    tma_load_2d(sb + L::H0 + a * kAtom, &tm_h, BAR_H, 32 * a, (b * H + h) * kP);
            }
        }
        __syncwarp();
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sb + L::TMEMP),
                     "r"(kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // K padding of Y' = M'·X: x rows T .. Tp16-1 (outside the TMA box) must be zero, not stale
    if (tid < 128)
        for (int k = tid; k < (Tp16 - T) * 8; k += 128)
            *reinterpret_cast<uint4*>(sm + L::X + swz(T + k / 8, k & 7)) = make_uint4(0, 0, 0, 0);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sm + L::TMEMP);

    if (warp == kIssW && lane == 0) {
        tma_prefetch(&tm_c); tma_prefetch(&tm_b); tma_prefetch(&tm_x);
        if (prm.dt_tma) tma_prefetch(&tm_dt);
        stamp(1);
    }
    float* cjs = reinterpret_cast<float*>(sm + L::CJ);
    float* lms = reinterpret_cast<float*>(sm + L::LM);
    uint64_t* tbits = reinterpret_cast<uint64_t*>(sm + L::BITS);
    volatile int* tinfo = reinterpret_cast<volatile int*>(sm + L::MODE);
    constexpr int kBarTree = 5;   // named barrier: tree warp publishes (arrive), row warps consume (sync)
    if (warp < 8) {
        // ================= warps 0-7.  Aux warps 2, 3, 6, 7 (u = 0..127): tree topology + segsum (warp 3) and the
        // replay prologue; all eight: the state update and hi/lo split (before the dependency wait under the
        // promises); then the aux warps store the committed state while the row warps 0, 1, 4, 5 (TMEM lanes
        // 0-63) build the masked weights and run the epilogue
        bool waited = false;
        auto wait_dep = [&]() {
            if (!waited) { pdl_wait(); waited = true; }
        };
        // ---- tree topology (PAPER.md:90 precondition; ancestor rows PAPER.md:63-66), warp 3: lane holds nodes
        //      lane and lane + 32; pointer jumping with the jump pointer of every round recorded for the segsum ----
        uint32_t jpk[3] = {0u, 0u, 0u};        // jump pointer + 1 of round r, half hf: byte 2r + hf
        int bad_code = 0;
        auto jump = [&](int r, int hf) { return (int)((jpk[(2 * r + hf) >> 2] >> (8 * ((2 * r + hf) & 3))) & 0xFFu) - 1; };
        auto topology = [&]() {
            const int par[2] = {tpar[0], tpar[1]};
            uint64_t rw[2];
            const bool root_bad = __any_sync(0xffffffffu, lane == 0 && par[0] != -1);
            const bool par_bad = __any_sync(0xffffffffu, (lane > 0 && lane < T && (par[0] < 0 || par[0] >= lane)) ||
                                                             (lane + 32 < T && (par[1] < 0 || par[1] >= lane + 32)));
            bad_code = root_bad ? STREE_DEV_BAD_ROOT : (par_bad ? STREE_DEV_BAD_PARENT : 0);
            const bool bad = bad_code != 0;
            int jp[2];
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                const int i = lane + 32 * hf;
                rw[hf] = i < T ? (1ull << i) : 0ull;
                jp[hf] = (i < T && !bad) ? par[hf] : -1;
            }
#pragma unroll
            for (int r = 0; r < kRounds; ++r) {
                uint64_t nrw[2];
                int njp[2];
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    const int j = jp[hf];
                    jpk[(2 * r + hf) >> 2] |= (uint32_t)(j + 1) << (8 * ((2 * r + hf) & 3));
                    const int sl = (j >= 0) ? (j & 31) : lane;
                    const bool hi = j >= 32;
                    const uint64_t r0 = __shfl_sync(0xffffffffu, rw[0], sl), r1 = __shfl_sync(0xffffffffu, rw[1], sl);
                    const int j0 = __shfl_sync(0xffffffffu, jp[0], sl), j1 = __shfl_sync(0xffffffffu, jp[1], sl);
                    nrw[hf] = rw[hf] | ((j >= 0) ? (hi ? r1 : r0) : 0ull);
                    njp[hf] = (j >= 0) ? (hi ? j1 : j0) : -1;
                }
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    rw[hf] = nrw[hf];
                    jp[hf] = njp[hf];
                }
            }
            tbits[lane] = rw[0];
            tbits[lane + 32] = rw[1];
        };
        // ---- segsum Λ = L·(dt A_h): the recorded jumps, values only; then c_j and the decay
        //      mode, published with the topology to the row warps ----
        auto segsum = [&](bool from_smem) {
            float dtv[2], lm[2];
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                const int i = lane + 32 * hf;
                dtv[hf] = 0.f;
                if (i < T)
                    dtv[hf] = dt_eff(prm.dtx, from_smem ? reinterpret_cast<const float*>(sm + L::DT)[4 * i + (h & 3)]
                                                        : (early_lambda ? tdt[hf] : prm.dt[((size_t)b * T + i) * H + h]), h);
                lm[hf] = dtv[hf] * tA;
            }
#pragma unroll
            for (int r = 0; r < kRounds; ++r) {
                const int j0 = jump(r, 0), j1 = jump(r, 1);
                const int s0 = j0 & 31, s1 = j1 & 31;
                const float v0 = __shfl_sync(0xffffffffu, lm[0], s0), w0 = __shfl_sync(0xffffffffu, lm[1], s0);
                const float v1 = __shfl_sync(0xffffffffu, lm[0], s1), w1 = __shfl_sync(0xffffffffu, lm[1], s1);
                const float n0 = lm[0] + (j0 >= 0 ? (j0 >= 32 ? w0 : v0) : 0.f);
                const float n1 = lm[1] + (j1 >= 0 ? (j1 >= 32 ? w1 : v1) : 0.f);
                lm[0] = n0;
                lm[1] = n1;
            }
            float mn = fminf(lm[0], lm[1]);
#pragma unroll
            for (int o = 16; o; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            const bool fac = mn >= -64.f;   // e^{Λi-Λj} = e^{Λi}·e^{-Λj} with both factors inside fp32 range
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                const int i = lane + 32 * hf;
                cjs[i] = fac ? __expf(-lm[hf]) * dtv[hf] : dtv[hf];
                lms[i] = lm[hf];
            }
            if (lane == 0) {
                tinfo[0] = fac ? 1 : 0;
                tinfo[1] = bad_code;
                tinfo[2] = __float_as_int(tD);
            }
            __syncwarp();
            asm volatile("bar.arrive %0, %1;" ::"r"(kBarTree), "r"(160) : "memory");   // publish to the row warps
            if (lane == 0) stamp(10);
        };
        auto tree_phase = [&]() {   // after the dependency wait unless EARLY_TREE (+ EARLY_DT)
            if (!prm.early_tree) {
                wait_dep();
                load_tree(false);
            }
            topology();
            if (early_lambda) segsum(false);
            else {
                wait_dep();
                if (prm.dt_tma) mbar_wait(BAR_CB, 0);
                segsum(prm.dt_tma != 0);
            }
        };
        int* rinfo = reinterpret_cast<int*>(sm + L::RINFO);
        bool tree_done = false;
        // ================= phase A (before the dependency wait where the promises allow) =================
        if (!row_warp) {
            if (R) {
                // ---- activation replay of the previous tree's accepted path (PAPER.md:113, 86-90 along the path):
                //   h <- e^{λ_{r-1}} h + Σ_m c_m x_prev[s_m] B_prev[s_m]ᵀ,  c_m = e^{λ_{r-1} - λ_m} dt_prev[s_m],
                //   λ_m = Σ_{q<=m} dt_prev[s_q] A_h.  Prologue: path, validation, coefficients and the staged
                //   operands of the first kRStage nodes ----
                if (!prm.early_replay) {
                    wait_dep();
                    load_path();
                }
                const int Tp = prm.Tp, G = prm.G;
                int* rpath = reinterpret_cast<int*>(sm + L::RPATH);
                float* rcoef = reinterpret_cast<float*>(sm + L::RCOEF);
                float* rlam = reinterpret_cast<float*>(sm + L::RLAM);
                const int r_raw = rp_len;
                if (u < Tp) rpath[u] = rp0;
                if (u + 128 < Tp) rpath[u + 128] = rp1;
                named_bar(3, 128);
                const int rr = (r_raw >= 1 && r_raw <= Tp) ? r_raw : 0;   // candidate length, validated below
                const int rs = min(rr, kRStage);
                auto node = [&](int m) {   // clamped into the tree: loads stay in bounds before validation
                    const int v = rpath[m];
                    return (v >= 0 && v < Tp) ? v : 0;
                };
                // staged operands of the first kRStage path nodes: 16-byte cp.async gathers, one DRAM latency
    #pragma unroll
                for (int k = u; k < kRStage * (NS / 8); k += 128) {
                    const int m = k / (NS / 8), c = k % (NS / 8);
                    if (m < rs)
                        cp_async16(sb + L::BPREV + (m * NS + 8 * c) * 2,
                                   prm.b_prev + (((size_t)b * Tp + node(m)) * G + g) * NS + 8 * c);
                }
                if (u < rs * (kP / 8)) {
                    const int m = u / (kP / 8), c = u % (kP / 8);
                    cp_async16(sb + L::XPREV + (m * kP + 8 * c) * 2,
                               prm.x_prev + (((size_t)b * Tp + node(m)) * H + h) * kP + 8 * c);
                }
                if (tree_warp && prm.early_tree) {   // the tree phase overlaps the gathers
                    tree_phase();
                    tree_done = true;
                }
                if (u < 32) {
                    // path validation (root-anchored, increasing, parent-linked: PAPER.md:90 on the accepted path)
                    int ok = rr > 0;
                    for (int m = lane; m < rr; m += 32) {
                        const int v = rpath[m];
                        bool good = (v >= 0 && v < Tp);
                        if (m == 0) good = good && v == 0;
                        else {
                            const int pu = rpath[m - 1];
                            good = good && v > pu;
                            if (prm.parent_prev && good) good = prm.parent_prev[(size_t)b * Tp + v] == pu;
                        }
                        if (!good) ok = 0;
                    }
                    ok = __all_sync(0xffffffffu, ok);
                    const int rv = ok ? rr : 0;
                    // path-cumsum of log-decays: inclusive warp scans over m = lane, lane + 32, then 32-node chunks
                    const float Ahr = prm.A[h];
                    float a0 = lane < rv ? dt_eff(prm.dtx, prm.dt_prev[((size_t)b * Tp + node(lane)) * H + h], h) : 0.f;
                    float a1 = lane + 32 < rv ? dt_eff(prm.dtx, prm.dt_prev[((size_t)b * Tp + node(lane + 32)) * H + h], h) : 0.f;
                    const float d0 = a0;
                    a0 *= Ahr;
                    a1 *= Ahr;
    #pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const float t0 = __shfl_up_sync(0xffffffffu, a0, o), t1 = __shfl_up_sync(0xffffffffu, a1, o);
                        if (lane >= o) { a0 += t0; a1 += t1; }
                    }
                    a1 += __shfl_sync(0xffffffffu, a0, 31);
                    float last = rv <= 32 ? __shfl_sync(0xffffffffu, a0, (rv - 1) & 31) : __shfl_sync(0xffffffffu, a1, (rv - 33) & 31);
                    if (rv > 64) {
                        float carry = __shfl_sync(0xffffffffu, a1, 31);
    #pragma unroll 1
                        for (int m0 = 64; m0 < rv; m0 += 32) {
                            const int m = m0 + lane;
                            float a = m < rv ? dt_eff(prm.dtx, prm.dt_prev[((size_t)b * Tp + node(m)) * H + h], h) * Ahr : 0.f;
    #pragma unroll
                            for (int o = 1; o < 32; o <<= 1) {
                                const float t = __shfl_up_sync(0xffffffffu, a, o);
                                if (lane >= o) a += t;
                            }
                            carry += __shfl_sync(0xffffffffu, a, 31);
                        }
                        last = carry;
                    }
                    const float lst = __shfl_sync(0xffffffffu, a0, kRStage - 1);
                    if (lane < kRStage) rcoef[lane] = __expf(last - a0) * d0;
                    if (lane == 0) {
                        rlam[0] = last;
                        rlam[1] = lst;
                        rlam[2] = __expf(last);
                        rinfo[0] = rv;
                        rinfo[1] = ok ? 0 : 1;
                    }
                }
                cp_async_wait_all();
                named_bar(3, 128);
                if (u == 0) stamp(20);
            } else if (tree_warp && prm.early_tree) {
                tree_phase();
                tree_done = true;
            }
        }
        // ================= phase B: the state tile, by the 256 threads of warps 0-7 (thread tid: rows (tid >> 3) + 32 i,
        // i = 0, 1, columns 32 a + 4 pc .. +3, pc = tid & 7): the replay update (R; packed FFMA2 over column pairs),
        // the committed fp32 tile written back for its TMA store, and the hi/lo bf16 split (B operand of Y0) =====
        int r = 0;
        if (prm.has_h0) {
            if (!early_h) {
                wait_dep();
                if (!row_warp && u == 0) {
                    mbar_expect_tx(BAR_H, NS * kP * 4);
#pragma unroll 1
                    for (int a = 0; a < NS / 32; ++a)
                        tma_load_2d_ef(sb + L::H0 + a * kAtom, &tm_h, BAR_H, 32 * a, (b * H + h) * kP, policy_evict_first());
                }
            }
            if (R) {
                named_bar(4, 256);                  // replay prologue published (aux warps) to all 8 warps
                r = rinfo[0];
            }
            mbar_wait(BAR_H, 0);
            if (tid == 0) stamp(21);
            const int pc = tid & 7;                 // 16-byte chunk of a 128-byte fp32 atom row
            constexpr int kAt = NS / 32;
            float2 hv[2][2 * kAt];                  // rows (tid >> 3) + 32 i, column pairs 32 a + 4 pc + {0, 2}
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int a = 0; a < kAt; ++a) {
                    const float4 v = *reinterpret_cast<const float4*>(sm + L::H0 + a * kAtom + swz((tid >> 3) + 32 * i, pc));
                    hv[i][2 * a] = make_float2(v.x, v.y);
                    hv[i][2 * a + 1] = make_float2(v.z, v.w);
                }
            if (R && r > 0) {
                const float* rcoef = reinterpret_cast<const float*>(sm + L::RCOEF);
                const float* rlam = reinterpret_cast<const float*>(sm + L::RLAM);
                const int* rpath = reinterpret_cast<const int*>(sm + L::RPATH);
                const __nv_bfloat16* xprev = reinterpret_cast<const __nv_bfloat16*>(sm + L::XPREV);
                const __nv_bfloat16* bprev = reinterpret_cast<const __nv_bfloat16*>(sm + L::BPREV);
                const int Tp = prm.Tp, G = prm.G;
                const float dk = rlam[2], last = rlam[0];
                float lam_run = rlam[1];
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int a = 0; a < 2 * kAt; ++a) hv[i][a] = fmul2(hv[i][a], make_float2(dk, dk));
#pragma unroll 1
                for (int m = 0; m < r; ++m) {
                    float2 bb[2 * kAt];
                    float uu[2];
                    if (m < kRStage) {
#pragma unroll
                        for (int a = 0; a < kAt; ++a) {
                            const uint2 w = *reinterpret_cast<const uint2*>(&bprev[m * NS + 32 * a + 4 * pc]);
                            bb[2 * a] = make_float2(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xFFFF0000u));
                            bb[2 * a + 1] = make_float2(__uint_as_float(w.y << 16), __uint_as_float(w.y & 0xFFFF0000u));
                        }
                        const float cm = rcoef[m];
#pragma unroll
                        for (int i = 0; i < 2; ++i) uu[i] = cm * __bfloat162float(xprev[m * kP + (tid >> 3) + 32 * i]);
                    } else {   // long accepted paths: operands from L2, coefficients on the fly
                        const int s = rpath[m];
                        const float dm = dt_eff(prm.dtx, prm.dt_prev[((size_t)b * Tp + s) * H + h], h);
                        lam_run += dm * prm.A[h];
                        const float cm = __expf(last - lam_run) * dm;
                        const __nv_bfloat16* br = prm.b_prev + (((size_t)b * Tp + s) * G + g) * NS + 4 * pc;
#pragma unroll
                        for (int a = 0; a < kAt; ++a) {
                            bb[2 * a] = make_float2(__bfloat162float(br[32 * a]), __bfloat162float(br[32 * a + 1]));
                            bb[2 * a + 1] = make_float2(__bfloat162float(br[32 * a + 2]), __bfloat162float(br[32 * a + 3]));
                        }
                        const __nv_bfloat16* xr = prm.x_prev + (((size_t)b * Tp + s) * H + h) * kP;
#pragma unroll
                        for (int i = 0; i < 2; ++i) uu[i] = cm * __bfloat162float(xr[(tid >> 3) + 32 * i]);
                    }
#pragma unroll
                    for (int i = 0; i < 2; ++i)
#pragma unroll
                        for (int a = 0; a < 2 * kAt; ++a) hv[i][a] = ffma2(make_float2(uu[i], uu[i]), bb[a], hv[i][a]);
                }
#pragma unroll
                for (int i = 0; i < 2; ++i)
#pragma unroll
                    for (int a = 0; a < kAt; ++a)
                        *reinterpret_cast<float4*>(sm + L::H0 + a * kAtom + swz((tid >> 3) + 32 * i, pc)) =
                            make_float4(hv[i][2 * a].x, hv[i][2 * a].y, hv[i][2 * a + 1].x, hv[i][2 * a + 1].y);
                if (tid == 0) stamp(28);
            }
            // hi/lo split: fp32 columns 32 a + 4 pc .. +3 -> bf16 atom a / 2, 16-byte chunk (a & 1)·4 + pc / 2,
            // 8-byte half pc & 1 (rows 0-63 of the split tile = hi, the next 64-row atom = lo)
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int a = 0; a < kAt; ++a) {
                    const float2 v01 = hv[i][2 * a], v23 = hv[i][2 * a + 1];
                    const __nv_bfloat162 h01 = __floats2bfloat162_rn(v01.x, v01.y), h23 = __floats2bfloat162_rn(v23.x, v23.y);
                    const float2 l01 = fsub2(v01, __bfloat1622float2(h01)), l23 = fsub2(v23, __bfloat1622float2(h23));
                    const uint2 hi = make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
                    const uint2 lo = make_uint2(pack_bf16(l01.x, l01.y), pack_bf16(l23.x, l23.y));
                    const uint32_t off = (a >> 1) * 2 * kAtom + swz((tid >> 3) + 32 * i, (a & 1) * 4 + (pc >> 1)) + (pc & 1) * 8;
                    *reinterpret_cast<uint2*>(sm + L::HL + off) = hi;
                    *reinterpret_cast<uint2*>(sm + L::HL + kAtom + off) = lo;
                }
            if (tid == 0) stamp(22);
            fence_proxy_async();   // split tiles (and the replayed tile, for its TMA store) -> async proxy
            named_bar(4, 256);
            if (tid == 0) {
                mbar_arrive(BAR_HS);
                stamp(16);
            }
        }
        // ================= phase C: after the dependency wait =================
        if (!row_warp) {
        if (tree_warp && !tree_done) tree_phase();
        wait_dep();   // every global write follows the dependency wait
        if (R && u == 0) {
            stamp(23);
            if (rinfo[1] && h == 0) report(prm.dev_status, STREE_DEV_BAD_PATH);
            if (r > 0) {                    // the committed state, in place
                const uint64_t ef = policy_evict_first();
#pragma unroll 1
                for (int a = 0; a < NS / 32; ++a)
                    tma_store_2d_ef(&tm_h, sb + L::H0 + a * kAtom, 32 * a, (b * H + h) * kP, ef);
                bulk_commit();
                bulk_wait_read_all();   // the store has read the tile before the CTA releases its shared memory
            }
            stamp(24);
        }
        } else {
        // ================= row warps 0, 1, 4, 5: TMEM lane quadrant qd = node rows 32 qd + lane, key / output
        // column half ch: the masked weights and the epilogue =================
        const int qd = warp & 1, ch = warp >> 2, wi = qd + 2 * ch;
        const int row = 32 * qd + lane;                 // tree node of this thread's TMEM lane
        const uint32_t tq = tmem + ((uint32_t)(32 * qd) << 16);
        pdl_wait();
        named_bar(kBarTree, 160);                       // topology, segsum and decay mode published (warp 3)
        const uint64_t bits = tbits[row];
        const float lmr = lms[row];
        const bool fac = tinfo[0] != 0;
        const int bad_code = tinfo[1];
        const bool bad = bad_code != 0;
        const float Dh = __int_as_float(tinfo[2]);
        if (bad && wi == 0 && lane == 0 && h == 0) report(prm.dev_status, bad_code);
        if (wi == 0 && lane == 0) stamp(11);
        // ---- masked weights of key columns [32 ch, 32 ch + 32), straight into TMEM ----
        mbar_wait(BAR_G, 0);
        tc_fence_after();
        if (wi == 0 && lane == 0) stamp(12);
        if (32 * ch < Tp16) {
            unsigned long long* tr = (wi == 0 && lane == 0) ? trace : nullptr;
            if (fac) build_weights<true>(tq, 32 * ch, bits, lmr, cjs, lms, tr);
            else build_weights<false>(tq, 32 * ch, bits, lmr, cjs, lms, tr);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(BAR_M);
        if (wi == 0 && lane == 0) stamp(13);
        // ---- epilogue: node row 32 qd + lane, output columns [32 ch, 32 ch + 32):
        //      y = e^{Λ_i}·acc (+ Y'_direct) + D_h x, bf16 (RNE), straight to HBM ----
        mbar_wait(BAR_ACC, 0);
        tc_fence_after();
        if (wi == 0 && lane == 0) stamp(14);
        const bool has0 = prm.has_h0 || fac;
        const float s0 = bad ? 0.f : __expf(lmr);
        const float dh = bad ? 0.f : Dh;
        const size_t yoff = (((size_t)b * T + row) * prm.y_heads + prm.y_head_off + h) * kP + 32 * ch;
        if (fac && !DPC) {
            // factorised decay: the 32 accumulator columns in one TMEM load, 64 contiguous bytes per thread
            uint32_t va[32];
            tmem_ld32(tq + kColAcc + 32 * ch, va);
            tmem_wait();
            if (wi == 0 && lane == 0) stamp(17);
            uint32_t o[16];
#pragma unroll
            for (int qc = 0; qc < 4; ++qc) {
                const uint4 xv = *reinterpret_cast<const uint4*>(sm + L::X + swz(row, 4 * ch + qc));
                const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int p = 8 * qc + 2 * k;
                    const float xa = __uint_as_float(xw[k] << 16), xb = __uint_as_float(xw[k] & 0xFFFF0000u);
                    o[4 * qc + k] = pack_bf16(fmaf(s0, __uint_as_float(va[p]), dh * xa),
                                              fmaf(s0, __uint_as_float(va[p + 1]), dh * xb));
                }
            }
            if (wi == 0 && lane == 0) stamp(18);
            if (row < T) {
#pragma unroll 1
                for (int pr = 0; pr < prm.n_ypeer; ++pr) {
                    uint4* dst = reinterpret_cast<uint4*>(prm.ypeer[pr] + yoff);
#pragma unroll
                    for (int q = 0; q < 4; ++q) dst[q] = make_uint4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
                }
            }
        } else {
    #pragma unroll
            for (int c16 = 0; c16 < 2; ++c16) {   // 16 output columns at a time (registers: no spills)
                const int col = 32 * ch + 16 * c16;
                uint32_t va[16], vb[16];
                if (has0) tmem_ld16r(tq + kColAcc + col, va);
                if (!fac) tmem_ld16r(tq + kColYd + col, vb);
                tmem_wait();
                float acc[16];
    #pragma unroll
                for (int k = 0; k < 16; ++k) acc[k] = has0 ? __uint_as_float(va[k]) : 0.f;
                if (wi == 0 && lane == 0 && c16 == 0) stamp(17);
                uint32_t o[8];
    #pragma unroll
                for (int qc = 0; qc < 2; ++qc) {
                    const uint4 xv = *reinterpret_cast<const uint4*>(sm + L::X + swz(row, (col >> 3) + qc));
                    const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
    #pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        const int p = 8 * qc + 2 * k;
                        const float xa = __uint_as_float(xw[k] << 16), xb = __uint_as_float(xw[k] & 0xFFFF0000u);
                        const float d0 = (!fac && !bad) ? __uint_as_float(vb[p]) : 0.f;
                        const float d1 = (!fac && !bad) ? __uint_as_float(vb[p + 1]) : 0.f;
                        float da = dh, db = dh;
                        if (DPC && prm.D && !bad) {   // D[h][p]
                            da = __ldg(prm.D + (size_t)h * kP + col + p);
                            db = __ldg(prm.D + (size_t)h * kP + col + p + 1);
                        }
                        o[4 * qc + k] = pack_bf16(fmaf(s0, acc[p], fmaf(da, xa, d0)), fmaf(s0, acc[p + 1], fmaf(db, xb, d1)));
                    }
                }
                if (wi == 0 && lane == 0 && c16 == 1) stamp(18);
                if (row < T) {
    #pragma unroll 1
                    for (int pr = 0; pr < prm.n_ypeer; ++pr) {
                        uint4* dst = reinterpret_cast<uint4*>(prm.ypeer[pr] + yoff);
                        dst[2 * c16] = make_uint4(o[0], o[1], o[2], o[3]);
                        dst[2 * c16 + 1] = make_uint4(o[4], o[5], o[6], o[7]);
                    }
                }
            }
        }
        if (wi == 0 && lane == 0) stamp(15);
        }
    } else if (warp == kIssW) {
        // ================= TMA producer + MMA issuer (warp converged, elected lane issues) =================
        const uint64_t dc = sdesc(sb + L::CB, 16, 1024), db = sdesc(sb + L::BB, 16, 1024);
        const uint64_t dh = sdesc(sb + L::HL, 16, 1024), xd = sdesc(sb + L::X, kAtom, 1024);
        const uint32_t id_g = idesc(kFmtBF16, 0, 128, Tp16);
        const uint32_t id_y0 = idesc(kFmtBF16, 0, 128, kP);
        const uint32_t id_y = idesc(kFmtBF16, 1, 128, kP);
        {
            const uint32_t go = 1;
            if (go) {
                pdl_wait();
                if (lane == 0) {
                    stamp(2);
                    const uint64_t ef = policy_evict_first();
                    // dt rides on the C/B barrier: the segsum needs it at the same time as G
                    mbar_expect_tx(BAR_CB, 2 * L::kCbAtoms * T * 128 + (prm.dt_tma ? T * 16 : 0));
                    if (prm.dt_tma) tma_load_2d(sb + L::DT, &tm_dt, BAR_CB, h & ~3, b * T);
#pragma unroll 1
                    for (int a = 0; a < L::kCbAtoms; ++a) {
                        tma_load_2d(sb + L::CB + a * kAtom, &tm_c, BAR_CB, g * NS + 64 * a, b * T);
                        tma_load_2d(sb + L::BB + a * kAtom, &tm_b, BAR_CB, g * NS + 64 * a, b * T);
                    }
                    mbar_expect_tx(BAR_X, T * 128);
                    tma_load_2d_ef(sb + L::X, &tm_x, BAR_X, h * kP, b * T, ef);
                }
                __syncwarp();
                mbar_wait(BAR_CB, 0);
                tc_fence_after();
                if (lane == 0) stamp(3);
            }
            // G = C·Bᵀ, M = 128 (rows 64-127 read past the C tile and are never used), N = Tp16, K = NS.
            // Descriptors = base + offsets, four K steps per unrolled group (one 128-byte swizzle row).
#pragma unroll 1
            for (int a = 0; a < NS / 64; ++a)
#pragma unroll
                for (int k4 = 0; k4 < 4; ++k4) {
                    const uint64_t off = (uint64_t)(a * (kAtom >> 4) + k4 * 2);
                    mma_f16_wp(tmem + kColG, dc + off, db + off, id_g, (a | k4) != 0, go);
                }
            tc_commit_wp(BAR_G, go);
            if (prm.has_h0) {
                // Y0 = C·h0ᵀ = C·hiᵀ + C·loᵀ: one accumulator, 2·NS/16 MMAs of N = 64 (B = the hi rows, then
                // the lo rows of the split tile) — the epilogue reads one set of columns (TMEM reads are
                // 64 B/clk per SM: a second accumulator would add 16 KB to the critical epilogue)
                if (go) {
                    mbar_wait(BAR_HS, 0);
                    tc_fence_after();
                    if (lane == 0) stamp(4);
                }
#pragma unroll 1
                for (int hl = 0; hl < 2; ++hl)
#pragma unroll 1
                    for (int a = 0; a < NS / 64; ++a)
#pragma unroll
                        for (int k4 = 0; k4 < 4; ++k4) {
                            const uint64_t oc = (uint64_t)(a * (kAtom >> 4) + k4 * 2);
                            const uint64_t oh = (uint64_t)(a * (2 * kAtom >> 4) + hl * (kAtom >> 4) + k4 * 2);
                            mma_f16_wp(tmem + kColAcc, dc + oc, dh + oh, id_y0, (hl | a | k4) != 0, go);
                        }
            }
            bool fac = true;
            if (go) {
                if (lane == 0) stamp(5);
                mbar_wait(BAR_M, 0);
                if (lane == 0) stamp(6);
                mbar_wait(BAR_X, 0);
                tc_fence_after();
                if (lane == 0) stamp(7);
                fac = *reinterpret_cast<volatile int*>(sm + L::MODE) != 0;
            }
            // Y' = M'·X, kind::f16 TS: A = masked weights from TMEM, B MN-major (x rows j); factorised decay
            // accumulates onto Y0 (hi columns), direct decay into its own columns
            const uint32_t dy = tmem + (fac ? kColAcc : kColYd);
            const uint32_t acc0 = (fac && prm.has_h0) ? 1u : 0u;
#pragma unroll 1
            for (int kk = 0; kk < Tp16 / 16; ++kk)
                mma_f16_ts_wp(dy, tmem + kColM + 8 * kk, xd + (uint64_t)(kk * 128), id_y, (kk > 0) | acc0, go);
            tc_commit_wp(BAR_ACC, go);
            if (go && lane == 0) stamp(8);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) stamp(30);
    if (warp == kIssW) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
    }
}

}  // namespace lat
}  // namespace stree

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

// debug timeline (not part of the ABI): with a buffer set, launch i of the small-batch kernel writes its
// per-CTA stamps to buf + (i % kTraceLaunches) * kTraceStride (STREE_TRACE builds only)
constexpr int kTraceLaunches = 16;
constexpr size_t kTraceStride = 1024 * stree::lat::kTraceWords;
unsigned long long* g_lat_trace = nullptr;
int g_lat_trace_n = 0;

template <int NS, bool R, bool DPC = false>
int launch_lat_inst(int B, int H, cudaStream_t s, const CUtensorMap& mc, const CUtensorMap& mb, const CUtensorMap& mx,
                    const CUtensorMap& mh, const CUtensorMap& mdt, const stree::lat::Params& prm) {
    using namespace stree::lat;
    auto k = lat_kernel<NS, R, DPC>;
    size_t smem = Lay<NS, R>::TOTAL + 1024;
    static const bool one_cta = [] {   // debug knob (not part of the ABI): force one CTA per SM
        const char* e = std::getenv("STREE_LAT_ONE_CTA");
        return e && e[0] == '1';
    }();
    // One CTA per SM when the grid fits in half the SMs: the next layer's CTAs (launched under PDL while this
    // layer runs) then land on other SMs instead of sharing this layer's (c2, 24 CTAs: 3.90 -> 3.48 µs per layer).
    // With more CTAs than that the next layer could not start until this one exits, so two CTAs per SM stay.
    if (one_cta || 2 * B * H <= stree::host::num_sms()) smem = 120 * 1024;
    cudaError_t e = stree::host::smem_attr((const void*)k, (int)smem);
    if (e != cudaSuccess) return (int)e;
    e = stree::launch_k(k, dim3(B * H), dim3(kThreads), smem, s, mc, mb, mx, mh, mdt, prm);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
}

}  // namespace

// Small-batch kernel selection: bf16, P = 64, N in {64, 128}, T <= 64 and at most one head per SM.
extern "C" int stree_lat_supports(const stree_dims* d) {
    if (!d || d->io_dtype != STREE_BF16 || d->head_dim != stree::lat::kP) return 0;
    if (d->d_state != 64 && d->d_state != 128) return 0;
    if (d->n_nodes < 1 || d->n_nodes > 64) return 0;
    if (d->n_groups < 1 || d->n_heads % d->n_groups) return 0;
    return (long long)d->batch * d->n_heads <= stree::host::num_sms() ? 1 : 0;
}

// rp == nullptr: scan only; else the fused replay of rp's previous tree + scan (h read and written in place)
extern "C" int stree_launch_scan_lat(const stree_dims* d, const void* x, const float* dt, const float* A,
                                     const void* Bm, const void* Cm, const float* D, const float* h0,
                                     const int32_t* parent, void* y, int32_t* dev_status, cudaStream_t s,
                                     const void* replay, const stree_yout* yo) {
    using namespace stree::lat;
    if (!stree_lat_supports(d)) return (int)cudaErrorNotSupported;
    const int B = d->batch, T = d->n_nodes, H = d->n_heads, P = d->head_dim, N = d->d_state, G = d->n_groups;
    const uint64_t BT = (uint64_t)B * T;
    CUtensorMap mc, mb, mx, mh, mdt;
    using stree::host::tmap_2d;
    bool ok = tmap_2d(&mc, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, Cm, (uint64_t)G * N, BT, (uint64_t)G * N * 2, 64, T) &&
              tmap_2d(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, Bm, (uint64_t)G * N, BT, (uint64_t)G * N * 2, 64, T) &&
              tmap_2d(&mx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, x, (uint64_t)H * P, BT, (uint64_t)H * P * 2, 64, T);
    if (h0)
        ok = ok && tmap_2d(&mh, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, h0, (uint64_t)N, (uint64_t)B * H * P, (uint64_t)N * 4,
                           32, 64);
    else
        mh = mx;   // unused
    // dt [B·T][H] fp32, box = 4 heads x T rows, unswizzled (16-byte rows): needs a 16-byte row pitch
    const bool dt_tma = (H * 4) % 16 == 0 &&
                        tmap_2d(&mdt, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, dt, (uint64_t)H, BT, (uint64_t)H * 4, 4, T, false);
    if (!dt_tma) mdt = mx;   // unused
    if (!ok) return (int)cudaErrorInvalidValue;
    Params prm{};
    if (replay) prm = *static_cast<const Params*>(replay);
    prm.B = B; prm.T = T; prm.H = H; prm.G = G;
    prm.dt = dt; prm.A = A; prm.D = D; prm.parent = parent; prm.h0p = h0; prm.y = (__nv_bfloat16*)y; prm.dev_status = dev_status;
    prm.has_h0 = h0 != nullptr;
    if (yo) {
        prm.n_ypeer = yo->n_peers;
        for (int p = 0; p < yo->n_peers; ++p) prm.ypeer[p] = (__nv_bfloat16*)yo->peers[p];
        prm.y_heads = yo->heads_total;
        prm.y_head_off = yo->head_offset;
    } else {
        prm.n_ypeer = 1;
        prm.ypeer[0] = (__nv_bfloat16*)y;
        prm.y_heads = H;
        prm.y_head_off = 0;
    }
    prm.dt_tma = dt_tma ? 1 : 0;
    prm.dtx = stree::DtX::from(stree_scan_opts_get());
    prm.d_pc = (stree_scan_opts_get() && stree_scan_opts_get()->d_per_channel) ? 1 : 0;
    prm.trace = g_lat_trace ? g_lat_trace + (size_t)(g_lat_trace_n++ % kTraceLaunches) * kTraceStride : nullptr;
    const uint32_t fl = stree_launch_flags_get();
    prm.early_state = (fl & STREE_LAUNCH_EARLY_STATE) ? 1 : 0;
    prm.early_replay = (fl & STREE_LAUNCH_EARLY_REPLAY) ? 1 : 0;
    prm.early_tree = (fl & STREE_LAUNCH_EARLY_TREE) ? 1 : 0;
    prm.early_dt = (fl & STREE_LAUNCH_EARLY_DT) ? 1 : 0;
    if (prm.early_tree && prm.early_dt) prm.dt_tma = 0;   // read before the wait by the row warps
    if (replay && !h0) return (int)cudaErrorInvalidValue;
    if (prm.d_pc) {
        if (N == 128) return replay ? launch_lat_inst<128, true, true>(B, H, s, mc, mb, mx, mh, mdt, prm)
                                    : launch_lat_inst<128, false, true>(B, H, s, mc, mb, mx, mh, mdt, prm);
        return replay ? launch_lat_inst<64, true, true>(B, H, s, mc, mb, mx, mh, mdt, prm)
                      : launch_lat_inst<64, false, true>(B, H, s, mc, mb, mx, mh, mdt, prm);
    }
    if (N == 128) return replay ? launch_lat_inst<128, true>(B, H, s, mc, mb, mx, mh, mdt, prm)
                                : launch_lat_inst<128, false>(B, H, s, mc, mb, mx, mh, mdt, prm);
    return replay ? launch_lat_inst<64, true>(B, H, s, mc, mb, mx, mh, mdt, prm)
                  : launch_lat_inst<64, false>(B, H, s, mc, mb, mx, mh, mdt, prm);
}

extern "C" int stree_launch_replay_scan_lat(const stree_dims* d_prev, const void* x_prev, const float* dt_prev,
                                            const void* Bm_prev, const int32_t* parent_prev, const int32_t* path,
                                            const int32_t* path_len, const stree_dims* d, const void* x,
                                            const float* dt, const float* A, const void* Bm, const void* Cm,
                                            const float* D, float* h, const int32_t* parent, void* y,
                                            int32_t* dev_status, cudaStream_t s, const stree_yout* yo) {
    stree::lat::Params rp{};
    rp.Tp = d_prev->n_nodes;
    rp.x_prev = (const __nv_bfloat16*)x_prev;
    rp.dt_prev = dt_prev;
    rp.b_prev = (const __nv_bfloat16*)Bm_prev;
    rp.parent_prev = parent_prev;
    rp.path = path;
    rp.path_len = path_len;
    return stree_launch_scan_lat(d, x, dt, A, Bm, Cm, D, h, parent, y, dev_status, s, &rp, yo);
}

extern "C" void stree_debug_lat_trace(unsigned long long* dev_buf) {
    g_lat_trace = dev_buf;
    g_lat_trace_n = 0;
}
