// K2s — stree_tree_scan / stree_replay_scan for small batches: one (tree, head) per CTA, built for
// latency (the paper's batch-1 setting; BASELINE configs c2 / c3).
//
// Same arithmetic as K2 (stree_scan_tc.cu; PAPER.md:91-102 with the Mamba-2 realisation of SURVEY R1-R3):
//     G   = C·Bᵀ                 (T x T, K = N)    tcgen05 kind::f16    bf16 -> fp32 TMEM
//     Y0  = C·h0ᵀ                (T x P, K = N)    tcgen05 kind::tf32   A = C from TMEM, B = fp32 state (TMA)
//     Y'  = (L∘G∘c)·X            (T x P, K = T)    tcgen05 kind::f16    masked weights (bf16) x x
//     y   = e^{Λ_i}(Y0 + Y') + D x                 (factorised decay; direct e^{Λi-Λj} when min Λ < -64)
// and, in the replay variant, the activation replay of the previous tree's accepted path applied on chip
// to the state tile before Y0 reads it (Alg. 1 l.123-124), the committed tile TMA-stored in
// place.
//
// Why a separate kernel: with B·H ≤ #SMs there is one head per CTA and nothing to pipeline; a layer's
// time is its dependency chain (inputs -> G -> Y0 -> Y' -> y) plus the launch boundary.  So:
//  * 97 KB of shared memory and 256 TMEM columns per CTA: two CTAs fit on an SM, so under PDL the next
//    layer's CTAs are resident while this layer runs and do everything that does not depend on the
//    previous kernel before their dependency wait (barriers, TMEM, state tile and — with
//    STREE_LAUNCH_EARLY_REPLAY — the whole replay of the previous path);
//  * small code (one pass, no rings, no head loop) that stays in the SM's instruction cache from one
//    layer to the next;
//  * G first on the tensor pipe, then Y0, while two warps build the masked weights; y is written
//    straight from registers (64 contiguous bytes per thread), no staging and no TMA store.
// Warps: 0-3 math (tree prologue redundantly per warp, C -> tf32 into TMEM, masked weights (0-1),
// epilogue), 4 TMA + MMA issue, 5-8 replay (replay variant only).
//
// Served: bf16 io, P = 64, N in {64, 128}, 1 <= T <= 64 (the launcher picks this kernel when B·H ≤ #SMs).
#include <cuda.h>

#include "stree_common.cuh"
#include "stree_host.cuh"
#include "stree_tc_ptx.cuh"

namespace stree {
namespace lat {
using namespace stree::tc;

constexpr int kP = 64;
constexpr int kAtom = 8192;               // 64 rows x 128 B, swizzle-128B
constexpr int kMathT = 128;               // warps 0-3
constexpr int kIssW = 4;                  // warp 4
constexpr int kRep0 = 160;                // first replay thread (warp 5)
constexpr int kRStage = 8;                // previous-path nodes staged on chip
constexpr uint32_t kCols = 256;           // TMEM columns: G / direct Y' [0,64), C tf32 [64, 64+N), acc [64+N, 128+N)
constexpr int kColG = 0, kColC = 64;
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
    static constexpr int H0 = BB + kCbAtoms * kAtom;          // state tile: atom a = columns [32a, 32a+32), fp32
    static constexpr int X = H0 + (NS / 32) * kAtom;          // x tile (64 rows of 64 bf16)
    static constexpr int MB = X + kAtom;                      // masked weights, 128 rows (rows 64-127 = copy)
    static constexpr int CJ = MB + 2 * kAtom;                 // float [4 warps][64]  c_j
    static constexpr int LM = CJ + 4 * 64 * 4;                // float [4 warps][64]  Λ_j (direct decay)
    static constexpr int MODE = LM + 4 * 64 * 4;              // int
    static constexpr int RPATH = MODE + 16;                   // int [kMaxNodes]
    static constexpr int RINFO = RPATH + (R ? kMaxNodes * 4 : 0);   // int [2]: r (0 = nothing), bad path
    static constexpr int RCOEF = RINFO + 16;                  // float [kRStage]
    static constexpr int RLAM = RCOEF + 64;                   // float [4]: λ_last, λ_{kRStage-1}, e^{λ_last}
    static constexpr int XPREV = RLAM + 16;                   // bf16 [kRStage][64]
    static constexpr int BPREV = XPREV + (R ? kRStage * kP * 2 : 0);    // float [kRStage][NS]
    static constexpr int BAR = (BPREV + (R ? kRStage * NS * 4 : 0) + 7) & ~7;
    static constexpr int NBAR = 8;                            // cb, x, h, ctf, g, m, acc, upd
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
    __nv_bfloat16* y;
    int32_t* dev_status;
    int has_h0, early_state, early_replay;
    // replay (previous tree)
    int Tp;
    const __nv_bfloat16* x_prev;
    const float* dt_prev;
    const __nv_bfloat16* b_prev;
    const int32_t* parent_prev;
    const int32_t* path;
    const int32_t* path_len;
    unsigned long long* trace;   // [grid][kTraceWords] or NULL (STREE_TRACE builds only)
};

template <int NS, bool R>
__global__ void __launch_bounds__(R ? 288 : 160, 2)
    lat_kernel(const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ CUtensorMap tm_b,
               const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_h, const Params prm) {
    using L = Lay<NS, R>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sb = smem_u32(sm);
    const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
    const int T = prm.T, H = prm.H;
    const int b = blockIdx.x / H, h = blockIdx.x % H;
    const int g = h / (H / prm.G);                        // group of head h (heads of a group contiguous)
    const uint32_t bar0 = sb + L::BAR;
    const uint32_t BAR_CB = bar0, BAR_X = bar0 + 8, BAR_H = bar0 + 16, BAR_CTF = bar0 + 24, BAR_G = bar0 + 32,
                   BAR_M = bar0 + 40, BAR_ACC = bar0 + 48, BAR_UPD = bar0 + 56;
    const int Tp16 = (T + 15) & ~15;
    const bool early_h = prm.early_state && prm.has_h0;
    unsigned long long* const trace = (kTrace && prm.trace) ? prm.trace + (size_t)blockIdx.x * kTraceWords : nullptr;
    auto stamp = [&](int k) {
        if (kTrace && trace) trace[k] = gtimer();
    };
    if (tid == 0) stamp(0);

    // ---- setup that touches no argument memory (overlaps the previous kernel under PDL) ----
    if (tid == 0) {
        mbar_init(BAR_CB, 1);
        mbar_init(BAR_X, 1);
        mbar_init(BAR_H, 1);
        mbar_init(BAR_CTF, 4);
        mbar_init(BAR_G, 1);
        mbar_init(BAR_M, 2);
        mbar_init(BAR_ACC, 1);
        mbar_init(BAR_UPD, 1);
        fence_barrier_init();
    }
    if (warp == kIssW) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sb + L::TMEMP),
                     "r"(kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // K padding of Y' = M'·X: x rows T .. Tp16-1 (outside the TMA box) must be zero, not stale
    if (tid < kMathT)
        for (int k = tid; k < (Tp16 - T) * 8; k += kMathT)
            *reinterpret_cast<uint4*>(sm + L::X + swz(T + k / 8, k & 7)) = make_uint4(0, 0, 0, 0);
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(sm + L::TMEMP);
    if (warp == kIssW && lane == 0) {
        tma_prefetch(&tm_c); tma_prefetch(&tm_b); tma_prefetch(&tm_x); tma_prefetch(&tm_h);
        if (early_h) {   // caller's promise: the state is not written by the preceding kernel
            mbar_expect_tx(BAR_H, NS * kP * 4);
#pragma unroll 1
            for (int a = 0; a < NS / 32; ++a)
                tma_load_2d(sb + L::H0 + a * kAtom, &tm_h, BAR_H, 32 * a, (b * H + h) * kP);
        }
    }
    if (tid == 0) stamp(1);
    if (!(R && warp > kIssW && prm.early_replay)) pdl_wait();
    if (tid == 0) stamp(2);

    if (warp == kIssW) {
        // ================= TMA producer + MMA issuer (warp converged, elected lane issues) =================
        if (lane == 0) {
            const uint64_t ef = policy_evict_first();
            mbar_expect_tx(BAR_CB, 2 * L::kCbAtoms * T * 128);
#pragma unroll 1
            for (int a = 0; a < L::kCbAtoms; ++a) {
                tma_load_2d(sb + L::CB + a * kAtom, &tm_c, BAR_CB, g * NS + 64 * a, b * T);
                tma_load_2d(sb + L::BB + a * kAtom, &tm_b, BAR_CB, g * NS + 64 * a, b * T);
            }
            mbar_expect_tx(BAR_X, T * 128);
            tma_load_2d_ef(sb + L::X, &tm_x, BAR_X, h * kP, b * T, ef);
            if (prm.has_h0 && !early_h) {
                mbar_expect_tx(BAR_H, NS * kP * 4);
#pragma unroll 1
                for (int a = 0; a < NS / 32; ++a)
                    tma_load_2d_ef(sb + L::H0 + a * kAtom, &tm_h, BAR_H, 32 * a, (b * H + h) * kP, ef);
            }
        }
        __syncwarp();
        mbar_wait(BAR_CB, 0);
        tc_fence_after();
        if (lane == 0) stamp(3);
        // G = C·Bᵀ, M = 128 (rows >= T, and rows 64-127 read past the C tile, are ignored), N = Tp16, K = NS
        const uint32_t id_g = idesc(kFmtBF16, 0, 128, Tp16);
#pragma unroll 1
        for (int kk = 0; kk < NS / 16; ++kk) {
            const uint32_t off = (kk >> 2) * kAtom + (kk & 3) * 32;
            mma_f16_w(tmem + kColG, sdesc(sb + L::CB + off, 16, 1024), sdesc(sb + L::BB + off, 16, 1024), id_g, kk > 0);
        }
        tc_commit_w(BAR_G);
        constexpr int kColAcc = 64 + NS;
        if (prm.has_h0) {
            // Y0 = C·h0ᵀ, kind::tf32, A = C (tf32) from TMEM, B = state tile (K-major, 32 fp32 per atom row)
            mbar_wait(BAR_CTF, 0);
            if (lane == 0) stamp(4);
            mbar_wait(R ? BAR_UPD : BAR_H, 0);
            tc_fence_after();
            if (lane == 0) stamp(5);
            const uint64_t bd = sdesc(sb + L::H0, 16, 1024);
            const uint32_t id_y0 = idesc(kFmtTF32, 0, 128, kP);
#pragma unroll 1
            for (int kk = 0; kk < NS / 8; ++kk)
                mma_tf32_ts_w(tmem + kColAcc, tmem + kColC + 8 * kk,
                              bd + (uint64_t)((((kk >> 2) * kAtom) + (kk & 3) * 32) >> 4), id_y0, kk > 0);
        }
        if (lane == 0) stamp(6);
        mbar_wait(BAR_M, 0);
        if (lane == 0) stamp(7);
        mbar_wait(BAR_X, 0);
        tc_fence_after();
        if (lane == 0) stamp(8);
        // Y' = M'·X, kind::f16, A K-major (masked weights), B MN-major (x rows j); factorised decay accumulates
        // onto Y0, direct decay into the G columns (all builders have read G before BAR_M)
        const bool fac = *reinterpret_cast<volatile int*>(sm + L::MODE) != 0;
        const uint32_t dy = tmem + (fac ? kColAcc : kColG);
        const uint32_t acc0 = (fac && prm.has_h0) ? 1u : 0u;
        const uint64_t ad = sdesc(sb + L::MB, 16, 1024);
        const uint64_t xd = sdesc(sb + L::X, kAtom, 1024);
        const uint32_t id_y = idesc(kFmtBF16, 1, 128, kP);
#pragma unroll 1
        for (int kk = 0; kk < Tp16 / 16; ++kk)
            mma_f16_w(dy, ad + (uint64_t)(kk * 2), xd + (uint64_t)(kk * 128), id_y, (kk > 0) | acc0);
        tc_commit_w(BAR_ACC);
        if (lane == 0) stamp(9);
    } else if (warp < kIssW) {
        // ================= math warps 0-3 =================
        const int q = warp;
        // ---- tree prologue, redundantly in every math warp (lane holds nodes lane and lane + 32): validation
        //      (PAPER.md:90 precondition), ancestor rows and the segsum Λ = L·(dt A_h) by pointer jumping
        //       ----
        int par[2];
        float dtv[2];
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            const int i = lane + 32 * hf;
            par[hf] = i < T ? prm.parent[(size_t)b * T + i] : -1;
            dtv[hf] = i < T ? prm.dt[((size_t)b * T + i) * H + h] : 0.f;
        }
        const float Ah = prm.A[h];
        const float Dh = prm.D ? prm.D[h] : 0.f;
        const bool root_bad = __any_sync(0xffffffffu, lane == 0 && par[0] != -1);
        const bool par_bad = __any_sync(0xffffffffu, (lane > 0 && lane < T && (par[0] < 0 || par[0] >= lane)) ||
                                                        (lane + 32 < T && (par[1] < 0 || par[1] >= lane + 32)));
        const bool bad = root_bad || par_bad;
        if (bad && q == 0 && lane == 0 && h == 0) report(prm.dev_status, root_bad ? STREE_DEV_BAD_ROOT : STREE_DEV_BAD_PARENT);
        uint64_t rw[2];
        int jp[2];
        float lm[2];
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            const int i = lane + 32 * hf;
            rw[hf] = i < T ? (1ull << i) : 0ull;
            jp[hf] = (i < T && !bad) ? par[hf] : -1;
            lm[hf] = dtv[hf] * Ah;
        }
        int rounds = 0;
        while ((1 << rounds) < T) ++rounds;
#pragma unroll 1
        for (int r = 0; r < rounds; ++r) {
            uint64_t nrw[2];
            int njp[2];
            float nlm[2];
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                const int j = jp[hf];
                const int sl = (j >= 0) ? (j & 31) : lane;
                const bool hi = j >= 32;
                const uint64_t r0 = __shfl_sync(0xffffffffu, rw[0], sl), r1 = __shfl_sync(0xffffffffu, rw[1], sl);
                const int j0 = __shfl_sync(0xffffffffu, jp[0], sl), j1 = __shfl_sync(0xffffffffu, jp[1], sl);
                const float v0 = __shfl_sync(0xffffffffu, lm[0], sl), v1 = __shfl_sync(0xffffffffu, lm[1], sl);
                nrw[hf] = rw[hf] | ((j >= 0) ? (hi ? r1 : r0) : 0ull);
                njp[hf] = (j >= 0) ? (hi ? j1 : j0) : -1;
                nlm[hf] = lm[hf] + ((j >= 0) ? (hi ? v1 : v0) : 0.f);
            }
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                rw[hf] = nrw[hf];
                jp[hf] = njp[hf];
                lm[hf] = nlm[hf];
            }
        }
        float mn = fminf(lm[0], lm[1]);
#pragma unroll
        for (int o = 16; o; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        const bool fac = mn >= -64.f;   // e^{Λi-Λj} = e^{Λi}·e^{-Λj} with both factors inside fp32 range
        float* cjw = reinterpret_cast<float*>(sm + L::CJ) + 64 * q;
        float* lmw = reinterpret_cast<float*>(sm + L::LM) + 64 * q;
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            const int i = lane + 32 * hf;
            cjw[i] = fac ? __expf(-lm[hf]) * dtv[hf] : dtv[hf];
            lmw[i] = lm[hf];
        }
        if (q == 0 && lane == 0) *reinterpret_cast<volatile int*>(sm + L::MODE) = fac ? 1 : 0;
        __syncwarp();
        if (q == 0 && lane == 0) stamp(10);
        const int rs = q & 1, half = q >> 1;
        const int row = 32 * rs + lane;                 // tree node of this thread's TMEM lane (lanes 64+ = copy)
        const uint32_t tq = tmem + ((uint32_t)(32 * q) << 16);
        // ---- C (bf16, TMA) -> fp32 -> TMEM lanes of this warp, columns [kColC, kColC + NS) ----
        if (prm.has_h0) {
            mbar_wait(BAR_CB, 0);
#pragma unroll 1
            for (int c32 = 0; c32 < NS / 32; ++c32) {
                uint32_t f[32];
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    const int c = 4 * c32 + cc;   // 16-byte chunk along the row
                    uint4 v = make_uint4(0, 0, 0, 0);
                    if (row < T) v = *reinterpret_cast<const uint4*>(sm + L::CB + (c >> 3) * kAtom + swz(row, c & 7));
                    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        f[8 * cc + 2 * k] = w[k] << 16;
                        f[8 * cc + 2 * k + 1] = w[k] & 0xFFFF0000u;
                    }
                }
                tmem_st32(tq + kColC + 32 * c32, f);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR_CTF);
            if (q == 0 && lane == 0) stamp(11);
        }
        // ---- masked weights (warps 0, 1 = TMEM lanes 0-63 = nodes): M'_ij = L_ij G_ij c_j (factorised) or
        //      L_ij e^{Λi-Λj} dt_j G_ij (direct), bf16, swizzle-128B K-major, rows 64-127 a copy ----
        if (q < 2) {
            mbar_wait(BAR_G, 0);
            tc_fence_after();
            if (q == 0 && lane == 0) stamp(12);
            const uint64_t bits = rw[q];
            const float li = lm[q];
#pragma unroll 1
            for (int c32 = 0; c32 < Tp16; c32 += 32) {
                uint32_t gv[32];
                tmem_ld32(tq + kColG + c32, gv);
                tmem_wait();
#pragma unroll
                for (int c16 = 0; c16 < 2; ++c16) {
                    uint32_t o[8];
#pragma unroll
                    for (int k = 0; k < 16; k += 2) {
                        const int j = c32 + 16 * c16 + k;
                        float v0 = cjw[j] * __uint_as_float(gv[16 * c16 + k]);
                        float v1 = cjw[j + 1] * __uint_as_float(gv[16 * c16 + k + 1]);
                        if (!fac) {
                            v0 *= __expf(fminf(li - lmw[j], 0.f));
                            v1 *= __expf(fminf(li - lmw[j + 1], 0.f));
                        }
                        o[k >> 1] = pack_bf16(((bits >> j) & 1ull) ? v0 : 0.f, ((bits >> (j + 1)) & 1ull) ? v1 : 0.f);
                    }
                    const int ch = (c32 >> 3) + 2 * c16;
                    const uint4 lo = make_uint4(o[0], o[1], o[2], o[3]), hi = make_uint4(o[4], o[5], o[6], o[7]);
                    *reinterpret_cast<uint4*>(sm + L::MB + swz(row, ch)) = lo;
                    *reinterpret_cast<uint4*>(sm + L::MB + swz(row, ch + 1)) = hi;
                    *reinterpret_cast<uint4*>(sm + L::MB + kAtom + swz(row, ch)) = lo;
                    *reinterpret_cast<uint4*>(sm + L::MB + kAtom + swz(row, ch + 1)) = hi;
                }
            }
            fence_proxy_async();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(BAR_M);
            if (q == 0 && lane == 0) stamp(13);
        }
        // ---- epilogue: warp q = node rows 32 (q & 1) .. +31 (TMEM lanes 32q..), output columns
        //      [32 half, 32 half + 32): y = e^{Λ_i}·acc (+ Y'_direct) + D_h x, bf16 (RNE), straight to HBM ----
        mbar_wait(BAR_ACC, 0);
        tc_fence_after();
        if (q == 0 && lane == 0) stamp(14);
        constexpr int kColAcc = 64 + NS;
        const bool has0 = prm.has_h0 || fac;
        uint32_t v0[32], v1[32];
        if (has0) tmem_ld32(tq + kColAcc + 32 * half, v0);
        if (!fac) tmem_ld32(tq + kColG + 32 * half, v1);
        tmem_wait();
        if (row < T) {
            const float s0 = bad ? 0.f : __expf(lm[rs]);
            const float dh = bad ? 0.f : Dh;
            uint32_t o[16];
#pragma unroll
            for (int qc = 0; qc < 4; ++qc) {
                const uint4 xv = *reinterpret_cast<const uint4*>(sm + L::X + swz(row, 4 * half + qc));
                const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int p = 8 * qc + 2 * k;
                    const float xa = __uint_as_float(xw[k] << 16), xb = __uint_as_float(xw[k] & 0xFFFF0000u);
                    const float a0 = has0 ? __uint_as_float(v0[p]) : 0.f, a1 = has0 ? __uint_as_float(v0[p + 1]) : 0.f;
                    const float d0 = (!fac && !bad) ? __uint_as_float(v1[p]) : 0.f;
                    const float d1 = (!fac && !bad) ? __uint_as_float(v1[p + 1]) : 0.f;
                    o[4 * qc + k] = pack_bf16(fmaf(s0, a0, fmaf(dh, xa, d0)), fmaf(s0, a1, fmaf(dh, xb, d1)));
                }
            }
            uint4* dst = reinterpret_cast<uint4*>(prm.y + (((size_t)b * T + row) * H + h) * kP + 32 * half);
#pragma unroll
            for (int k = 0; k < 4; ++k) dst[k] = make_uint4(o[4 * k], o[4 * k + 1], o[4 * k + 2], o[4 * k + 3]);
        }
        if (q == 0 && lane == 0) stamp(15);
    } else if (R) {
        // ================= replay warps 5-8: activation replay of the previous tree's accepted path
        //   h <- e^{λ_{r-1}} h + Σ_m c_m x_prev[s_m] B_prev[s_m]ᵀ,  c_m = e^{λ_{r-1} - λ_m} dt_prev[s_m],
        //   λ_m = Σ_{q<=m} dt_prev[s_q] A_h  (PAPER.md:113, 86-90 along the path) =================
        const int u = tid - kRep0;      // 0..127
        const int Tp = prm.Tp, G = prm.G;
        int* rpath = reinterpret_cast<int*>(sm + L::RPATH);
        int* rinfo = reinterpret_cast<int*>(sm + L::RINFO);
        float* rcoef = reinterpret_cast<float*>(sm + L::RCOEF);
        float* rlam = reinterpret_cast<float*>(sm + L::RLAM);
        __nv_bfloat16* xprev = reinterpret_cast<__nv_bfloat16*>(sm + L::XPREV);
        float* bprev = reinterpret_cast<float*>(sm + L::BPREV);
        const int r_raw = prm.path_len[b];
#pragma unroll 1
        for (int m = u; m < Tp; m += 128) rpath[m] = prm.path[(size_t)b * Tp + m];
        named_bar(3, 128);
        const int rr = (r_raw >= 1 && r_raw <= Tp) ? r_raw : 0;   // candidate length, validated below
        const int rs = min(rr, kRStage);
        auto node = [&](int m) {   // clamped into the tree: loads stay in bounds before validation
            const int v = rpath[m];
            return (v >= 0 && v < Tp) ? v : 0;
        };
        // staged operands of the first kRStage path nodes (all issued together: one DRAM latency)
#pragma unroll 1
        for (int k = u; k < rs * NS; k += 128) {
            const int m = k / NS, n = k % NS;
            bprev[k] = __bfloat162float(prm.b_prev[(((size_t)b * Tp + node(m)) * G + g) * NS + n]);
        }
        for (int k = u; k < rs * (kP / 2); k += 128) {
            const int m = k / (kP / 2), w = k % (kP / 2);
            reinterpret_cast<uint32_t*>(xprev)[k] =
                reinterpret_cast<const uint32_t*>(prm.x_prev)[(((size_t)b * Tp + node(m)) * H + h) * (kP / 2) + w];
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
            const int r = ok ? rr : 0;
            // path-cumsum of log-decays: inclusive warp scans over m = lane, lane + 32, then 32-node chunks
            const float Ah = prm.A[h];
            float a0 = lane < r ? prm.dt_prev[((size_t)b * Tp + node(lane)) * H + h] : 0.f;
            float a1 = lane + 32 < r ? prm.dt_prev[((size_t)b * Tp + node(lane + 32)) * H + h] : 0.f;
            const float d0 = a0;
            a0 *= Ah;
            a1 *= Ah;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const float t0 = __shfl_up_sync(0xffffffffu, a0, o), t1 = __shfl_up_sync(0xffffffffu, a1, o);
                if (lane >= o) { a0 += t0; a1 += t1; }
            }
            a1 += __shfl_sync(0xffffffffu, a0, 31);
            float last = r <= 32 ? __shfl_sync(0xffffffffu, a0, (r - 1) & 31) : __shfl_sync(0xffffffffu, a1, (r - 33) & 31);
            if (r > 64) {
                float carry = __shfl_sync(0xffffffffu, a1, 31);
#pragma unroll 1
                for (int m0 = 64; m0 < r; m0 += 32) {
                    const int m = m0 + lane;
                    float a = m < r ? prm.dt_prev[((size_t)b * Tp + node(m)) * H + h] * Ah : 0.f;
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
                rinfo[0] = r;
                rinfo[1] = ok ? 0 : 1;
            }
        }
        named_bar(3, 128);
        if (u == 0) stamp(20);
        const int r = rinfo[0];
        mbar_wait(BAR_H, 0);
        if (u == 0) stamp(21);
        if (r > 0) {
            // thread u owns 16-byte chunk pc of rows (u >> 3) + 16 i of every atom (columns 32 a + 4 pc ..)
            const int pc = u & 7;
            constexpr int kAt = NS / 32;
            const float dk = rlam[2], Ak = prm.A[h], last = rlam[0];
            float lam_run = rlam[1];
            float4 hv[4][kAt];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int a = 0; a < kAt; ++a) {
                    const float4 v = *reinterpret_cast<const float4*>(sm + L::H0 + a * kAtom + swz((u >> 3) + 16 * i, pc));
                    hv[i][a] = make_float4(dk * v.x, dk * v.y, dk * v.z, dk * v.w);
                }
#pragma unroll 1
            for (int m = 0; m < r; ++m) {
                float4 bb[kAt];
                float uu[4];
                if (m < kRStage) {
#pragma unroll
                    for (int a = 0; a < kAt; ++a) bb[a] = *reinterpret_cast<const float4*>(&bprev[m * NS + 32 * a + 4 * pc]);
#pragma unroll
                    for (int i = 0; i < 4; ++i) uu[i] = rcoef[m] * __bfloat162float(xprev[m * kP + (u >> 3) + 16 * i]);
                } else {   // long accepted paths: operands from L2, coefficients on the fly
                    const int s = rpath[m];
                    const float dm = prm.dt_prev[((size_t)b * Tp + s) * H + h];
                    lam_run += dm * Ak;
                    const float cm = __expf(last - lam_run) * dm;
                    const __nv_bfloat16* br = prm.b_prev + (((size_t)b * Tp + s) * G + g) * NS + 4 * pc;
#pragma unroll
                    for (int a = 0; a < kAt; ++a)
                        bb[a] = make_float4(__bfloat162float(br[32 * a]), __bfloat162float(br[32 * a + 1]),
                                            __bfloat162float(br[32 * a + 2]), __bfloat162float(br[32 * a + 3]));
                    const __nv_bfloat16* xr = prm.x_prev + (((size_t)b * Tp + s) * H + h) * kP;
#pragma unroll
                    for (int i = 0; i < 4; ++i) uu[i] = cm * __bfloat162float(xr[(u >> 3) + 16 * i]);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int a = 0; a < kAt; ++a) {
                        hv[i][a].x = fmaf(uu[i], bb[a].x, hv[i][a].x); hv[i][a].y = fmaf(uu[i], bb[a].y, hv[i][a].y);
                        hv[i][a].z = fmaf(uu[i], bb[a].z, hv[i][a].z); hv[i][a].w = fmaf(uu[i], bb[a].w, hv[i][a].w);
                    }
            }
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int a = 0; a < kAt; ++a)
                    *reinterpret_cast<float4*>(sm + L::H0 + a * kAtom + swz((u >> 3) + 16 * i, pc)) = hv[i][a];
        }
        fence_proxy_async();
        named_bar(3, 128);
        if (u == 0) stamp(22);
        if (prm.early_replay) pdl_wait();   // every global write follows the dependency wait
        if (u == 0) stamp(23);
        if (u == 0) {
            if (rinfo[1] && h == 0) report(prm.dev_status, STREE_DEV_BAD_PATH);
            mbar_arrive(BAR_UPD);           // Y0 may read the replayed tile (the store below only reads it too)
            if (r > 0) {                    // the committed state, in place
                const uint64_t ef = policy_evict_first();
#pragma unroll 1
                for (int a = 0; a < NS / 32; ++a)
                    tma_store_2d_ef(&tm_h, sb + L::H0 + a * kAtom, 32 * a, (b * H + h) * kP, ef);
                bulk_commit();
                bulk_wait_all();
            }
            stamp(24);
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

template <int NS, bool R>
int launch_lat_inst(int B, int H, cudaStream_t s, const CUtensorMap& mc, const CUtensorMap& mb, const CUtensorMap& mx,
                    const CUtensorMap& mh, const stree::lat::Params& prm) {
    using namespace stree::lat;
    auto k = lat_kernel<NS, R>;
    const size_t smem = Lay<NS, R>::TOTAL + 1024;
    cudaError_t e = stree::host::smem_attr((const void*)k, (int)smem);
    if (e != cudaSuccess) return (int)e;
    e = stree::launch_k(k, dim3(B * H), dim3(R ? 288 : 160), smem, s, mc, mb, mx, mh, prm);
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
                                     const void* replay) {
    using namespace stree::lat;
    if (!stree_lat_supports(d)) return (int)cudaErrorNotSupported;
    const int B = d->batch, T = d->n_nodes, H = d->n_heads, P = d->head_dim, N = d->d_state, G = d->n_groups;
    const uint64_t BT = (uint64_t)B * T;
    CUtensorMap mc, mb, mx, mh;
    using stree::host::tmap_2d;
    bool ok = tmap_2d(&mc, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, Cm, (uint64_t)G * N, BT, (uint64_t)G * N * 2, 64, T) &&
              tmap_2d(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, Bm, (uint64_t)G * N, BT, (uint64_t)G * N * 2, 64, T) &&
              tmap_2d(&mx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, x, (uint64_t)H * P, BT, (uint64_t)H * P * 2, 64, T);
    if (h0)
        ok = ok && tmap_2d(&mh, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, h0, (uint64_t)N, (uint64_t)B * H * P, (uint64_t)N * 4,
                           32, 64);
    else
        mh = mx;   // unused
    if (!ok) return (int)cudaErrorInvalidValue;
    Params prm{};
    if (replay) prm = *static_cast<const Params*>(replay);
    prm.B = B; prm.T = T; prm.H = H; prm.G = G;
    prm.dt = dt; prm.A = A; prm.D = D; prm.parent = parent; prm.y = (__nv_bfloat16*)y; prm.dev_status = dev_status;
    prm.has_h0 = h0 != nullptr;
    prm.trace = g_lat_trace ? g_lat_trace + (size_t)(g_lat_trace_n++ % kTraceLaunches) * kTraceStride : nullptr;
    const uint32_t fl = stree_launch_flags_get();
    prm.early_state = (fl & STREE_LAUNCH_EARLY_STATE) ? 1 : 0;
    prm.early_replay = (fl & STREE_LAUNCH_EARLY_REPLAY) ? 1 : 0;
    if (replay && !h0) return (int)cudaErrorInvalidValue;
    if (N == 128) return replay ? launch_lat_inst<128, true>(B, H, s, mc, mb, mx, mh, prm)
                                : launch_lat_inst<128, false>(B, H, s, mc, mb, mx, mh, prm);
    return replay ? launch_lat_inst<64, true>(B, H, s, mc, mb, mx, mh, prm)
                  : launch_lat_inst<64, false>(B, H, s, mc, mb, mx, mh, prm);
}

extern "C" int stree_launch_replay_scan_lat(const stree_dims* d_prev, const void* x_prev, const float* dt_prev,
                                            const void* Bm_prev, const int32_t* parent_prev, const int32_t* path,
                                            const int32_t* path_len, const stree_dims* d, const void* x,
                                            const float* dt, const float* A, const void* Bm, const void* Cm,
                                            const float* D, float* h, const int32_t* parent, void* y,
                                            int32_t* dev_status, cudaStream_t s) {
    stree::lat::Params rp{};
    rp.Tp = d_prev->n_nodes;
    rp.x_prev = (const __nv_bfloat16*)x_prev;
    rp.dt_prev = dt_prev;
    rp.b_prev = (const __nv_bfloat16*)Bm_prev;
    rp.parent_prev = parent_prev;
    rp.path = path;
    rp.path_len = path_len;
    return stree_launch_scan_lat(d, x, dt, A, Bm, Cm, D, h, parent, y, dev_status, s, &rp);
}

extern "C" void stree_debug_lat_trace(unsigned long long* dev_buf) {
    g_lat_trace = dev_buf;
    g_lat_trace_n = 0;
}
