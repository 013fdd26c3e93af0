// K2b stree_tree_scan for 64 < T <= 128 on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Same method as K2 (stree_scan_tc.cu, Mamba-2 realisation SURVEY R1-R3):
//     G   = C·Bᵀ                 (T x T, K = N)    kind::f16   once per tree
//     Y0  = C·h0_hᵀ              (T x P, K = N)    kind::tf32  per head (A = C as tf32 in TMEM)
//     Y'  = (L∘G∘c_h)·X_h        (T x P, K = T)    kind::f16   per head
//     y_i = e^{Λ_i} (Y0 + Y')_i + D_h x_i     (factorised decay, c_j = e^{-Λ_j} dt_j, when min Λ >= -64)
//     y_i = e^{Λ_i} Y0_i + Y'_i + D_h x_i     (direct decay, M'_ij = e^{min(Λ_i-Λ_j,0)} dt_j G_ij, otherwise)
// but with the tree's nodes in all 128 TMEM lanes (K2 puts them in lanes 0-63 and a copy of G in 64-127),
// so trees of up to 128 nodes stay on the tensor cores instead of the FP32 SIMT kernel.  A simpler pipeline
// than K2: one CTA per (tree, chunk of <= 10 heads of one group, 128-row tile of nodes), 352 threads —
//   warps 0-7  math, two per TMEM lane quadrant (thread = node = TMEM lane, the pair split over column halves):
//              tree prologue (validation, ancestor bits and Λ of every head by pointer jumping), C -> tf32 into
//              TMEM, then per head the masked weights and the epilogue of the previous head
//   warp 8     TMA producer: C, B once; per head the 32 KB fp32 state (4 boxes) and the x tile, 2-stage rings
//   warp 9     tcgen05.mma issuer + TMEM allocator (512 columns: G 0-127, C tf32 128-255, two head slots of
//              Y0 / Y' accumulators 256-511)
//   warp 10    y tiles staged in shared memory, TMA-stored
// Served: bf16 io, P = 64, N = 128, 1 <= T <= 256 (dispatched for T > 64).  NKB = 2 (128 < T <= 256): each
// CTA owns one 128-row tile of nodes (rt = 0, 1); its keys are the nodes 0 .. 128·rt + 127 (topological order:
// every ancestor precedes its descendants), G = C_rows·Bᵀ takes 256 TMEM columns, so one accumulator slot,
// one M' buffer (over the B tile) and the second x stage over the C tile (free once C is in TMEM).
#include <cuda.h>

#include "stree_common.cuh"
#include "stree_host.cuh"
#include "stree_tc_ptx.cuh"

namespace stree {
namespace tc128 {

using namespace stree::tc;

constexpr int kP = 64, kN = 128;
constexpr int kThreads = 352;   // warps 0-7 math (two per TMEM lane quadrant), 8 TMA, 9 MMA, 10 y stores
constexpr int kTile = 16384;          // 128 rows x 128 bytes, swizzle-128B
constexpr uint32_t kCols = 512;
constexpr int kTraceWords = 64;   // debug timeline: u64 globaltimer stamps per CTA (STREE_TRACE builds)
#ifdef STREE_TRACE
constexpr bool kTrace = true;
#else
constexpr bool kTrace = false;
#endif

template <int NKB>
struct Sm {
    static constexpr int kKeys = 128 * NKB;        // nodes / keys per tree served
    static constexpr int kHPC = NKB == 1 ? 10 : 4; // heads per CTA
    static constexpr int kSlots = NKB == 1 ? 2 : 1;        // accumulator slots / M' buffers
    static constexpr int kGCol = 0, kCCol = 128 * NKB, kAccCol = kCCol + 128;   // slot a: Y0 +128a, Y' +64
    static constexpr int XS = kTile * NKB;        // x stage: 128·NKB rows x 128 B
    static constexpr int C = 0;                    // C rows of this tile: 2 k-chunks x 16 KB
    static constexpr int B = C + 2 * kTile;        // B rows 0 .. kKeys-1: NKB x 2 k-chunks (dead after G: M')
    static constexpr int M0 = B + 2 * kTile * NKB; // NKB == 1: second M' buffer
    static constexpr int H = M0 + (NKB == 1 ? 2 * kTile : 0);   // state ring: 2 x 32 KB
    static constexpr int X = H + 2 * 32768;        // x stage 0 (NKB == 1: stages 0 and 1)
    static constexpr int PAR = X + (NKB == 1 ? 2 : 1) * XS;
    static constexpr int ANC = PAR + kKeys * 4;    // u32 [4·NKB][kKeys]   (updated in place)
    static constexpr int JMP = ANC + 4 * NKB * kKeys * 4;   // int [2][kKeys]
    static constexpr int LAM = JMP + 2 * kKeys * 4;         // float [2][kHPC][kKeys]
    static constexpr int DTS = LAM + 2 * kHPC * kKeys * 4;  // float [kHPC][kKeys]
    static constexpr int CJ = DTS + kHPC * kKeys * 4;       // float [kHPC][kKeys]
    static constexpr int AS = CJ + kHPC * kKeys * 4;        // float [kHPC]
    static constexpr int DS = AS + kHPC * 4;                // float [kHPC]
    static constexpr int BADF = DS + kHPC * 4;              // int
    static constexpr int WOK = BADF + 4;                    // u32 [8] per-warp factorisable-head masks
    static constexpr int WRB = WOK + 32;                    // u32 [8] per-warp chunk-rebasable-head masks
    static constexpr int RC = WRB + 32;                     // float [kHPC][8] chunk reference Λ (max over chunk)
    static constexpr int CR = RC + kHPC * 8 * 4;            // float [kHPC][kKeys] rebased c_j = e^{R_c-Λ_j} dt_j
    static constexpr int BAR = (CR + kHPC * kKeys * 4 + 7) & ~7;
    // tree, g, ctf, hfull[2], hempty[2], xfull[2], xempty[2], mfull[2], mempty[2], accfull[2], accempty[2]
    static constexpr int NBAR = 3 + 16;   // + yfree[2]
    static constexpr int TMEMP = BAR + NBAR * 8;
    static constexpr int TOTAL = TMEMP + 16;
    static_assert(TOTAL + 1024 <= 227 * 1024, "shared memory budget");
    __device__ static constexpr int xstage(int s) { return NKB == 1 ? X + s * XS : (s ? C : X); }
};

struct Params {
    const float* dt;
    const float* A;
    const float* D;
    const int32_t* parent;
    __nv_bfloat16* y;
    int32_t* dev_status;
    int B, T, H, G, cpg, hpc, has_h0;
    DtX dtx;    // *_ex options: effective dt
    int d_pc;   // *_ex options: D is [H][P]
    unsigned long long* trace;   // [grid][kTraceWords] or NULL (STREE_TRACE builds only)
    int early_tree, early_dt;    // STREE_LAUNCH_EARLY_TREE / _DT: the tree prologue before the dependency wait
    int early_state;             // STREE_LAUNCH_EARLY_STATE: the first two state tiles streamed before the wait
};

__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

template <int NKB, bool DPC = false>   // DPC: D is [H][P] (separate instantiation, no runtime branch)
__global__ void __launch_bounds__(kThreads, 1)
    scan_tc128_kernel(const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ CUtensorMap tm_b,
                      const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_h0,
                      const __grid_constant__ CUtensorMap tm_y, const Params prm) {
    using Sm = tc128::Sm<NKB>;
    constexpr int kT = Sm::kKeys, kHPC = Sm::kHPC, kGCol = Sm::kGCol, kCCol = Sm::kCCol, kAccCol = Sm::kAccCol;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sb = smem_u32(sm);
    const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
    const int T = prm.T, H = prm.H;
    const int rt = blockIdx.x % NKB;                  // row tile: nodes r0 .. r0 + 127
    const int r0 = 128 * rt;
    const int cta = blockIdx.x / NKB;
    const int b = cta / (prm.G * prm.cpg);
    const int rem = cta % (prm.G * prm.cpg);
    const int g = rem / prm.cpg, chunk = rem % prm.cpg;
    const int hpg = H / prm.G;
    const int hbeg = g * hpg + chunk * prm.hpc;
    const int nh = min(prm.hpc, g * hpg + hpg - hbeg);
    if (nh <= 0 || r0 >= T) { pdl_wait(); return; }
    const int Tp16 = (T + 15) & ~15;
    const int kcta = min(Tp16, 128 * (rt + 1));       // keys this tile's rows can see (multiple of 16)
    const int nkb = rt + 1;                           // key blocks of 128

    unsigned long long* const trace = (kTrace && prm.trace) ? prm.trace + (size_t)blockIdx.x * kTraceWords : nullptr;
    auto stamp = [&](int k) {
        if (kTrace && trace && k < kTraceWords) trace[k] = gtimer();
    };
    if (threadIdx.x == 0) stamp(0);
    const uint32_t bar0 = sb + Sm::BAR;
    const uint32_t BAR_TREE = bar0, BAR_G = bar0 + 8, BAR_CTF = bar0 + 16;
    auto bar_hfull = [&](int s) { return bar0 + 24 + 8 * s; };
    auto bar_hempty = [&](int s) { return bar0 + 40 + 8 * s; };
    auto bar_xfull = [&](int s) { return bar0 + 56 + 8 * s; };
    auto bar_xempty = [&](int s) { return bar0 + 72 + 8 * s; };
    auto bar_mfull = [&](int a) { return bar0 + 88 + 8 * a; };
    auto bar_mempty = [&](int a) { return bar0 + 104 + 8 * a; };
    auto bar_accfull = [&](int a) { return bar0 + 120 + 8 * a; };
    auto bar_accempty = [&](int a) { return bar0 + 136 + 8 * a; };
    // NKB == 1: xempty[s] = "y of the stage's head staged in Y buffer s" (256 arrivals), yfree[s] = its TMA
    // store has read the Y buffer (the storer warp arrives)
    auto bar_yfree = [&](int s) { return bar0 + 152 + 8 * s; };
    uint32_t* tmem_slot = (uint32_t*)(sm + Sm::TMEMP);
    auto mbuf = [&](int a) { return sb + ((NKB == 1 && a == 0) ? Sm::M0 : Sm::B); };

    if (tid == 0) {
        mbar_init(BAR_TREE, 1);
        mbar_init(BAR_G, 1);
        mbar_init(BAR_CTF, 256);
        for (int s = 0; s < 2; ++s) {
            mbar_init(bar_hfull(s), 1);
            mbar_init(bar_hempty(s), 1);
            mbar_init(bar_xfull(s), 1);
            mbar_init(bar_xempty(s), 256);
            mbar_init(bar_mfull(s), 256);
            mbar_init(bar_mempty(s), 1);
            mbar_init(bar_accfull(s), 1);
            mbar_init(bar_accempty(s), 256);
            mbar_init(bar_yfree(s), 1);
        }
        *(int*)(sm + Sm::BADF) = 0;
        fence_barrier_init();
    }
    if (warp == 9) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (warp == 8 && lane == 0) {
        tma_prefetch(&tm_c); tma_prefetch(&tm_b); tma_prefetch(&tm_x); tma_prefetch(&tm_h0);
        if (NKB == 1) tma_prefetch(&tm_y);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // math warps with EARLY_TREE + EARLY_DT run the whole tree prologue (validation, ancestor bits, Λ, decay
    // modes and coefficients) before their dependency wait
    const bool early_tree = warp < 8 && prm.early_tree && prm.early_dt;
    // the producer with EARLY_STATE streams the first two state tiles before its dependency wait
    const int kpre = (prm.early_state && prm.has_h0) ? min(nh, 2) : 0;
    if (!early_tree && !(warp == 8 && kpre)) pdl_wait();
    if (tid == 0) stamp(1);

    if (warp == 8) {
        // ================= TMA producer =================
        if (kpre) {
            if (lane == 0)
                for (int k = 0; k < kpre; ++k) {
                    mbar_expect_tx(bar_hfull(k), 32768);
                    for (int a = 0; a < 4; ++a)
                        tma_load_2d(sb + Sm::H + k * 32768 + a * 8192, &tm_h0, bar_hfull(k), 32 * a, (b * H + hbeg + k) * kP);
                }
            __syncwarp();
            pdl_wait();
        }
        if (lane == 0) {
            mbar_expect_tx(BAR_TREE, (2 + 2 * nkb) * kTile);
            for (int a = 0; a < 2; ++a) {
                tma_load_2d(sb + Sm::C + a * kTile, &tm_c, BAR_TREE, g * kN + 64 * a, b * T + r0);
                for (int kb = 0; kb < nkb; ++kb)
                    tma_load_2d(sb + Sm::B + (2 * kb + a) * kTile, &tm_b, BAR_TREE, g * kN + 64 * a, b * T + 128 * kb);
            }
            for (int k = 0; k < nh; ++k) {
                const int s = k & 1, u = k >> 1;
                const int h = hbeg + k;
                if (prm.has_h0 && k >= kpre) {
                    mbar_wait(bar_hempty(s), (u & 1) ^ 1);
                    mbar_expect_tx(bar_hfull(s), 32768);
                    for (int a = 0; a < 4; ++a)
                        tma_load_2d(sb + Sm::H + s * 32768 + a * 8192, &tm_h0, bar_hfull(s), 32 * a, (b * H + h) * kP);
                }
                // NKB == 1: x of head k-2 was scaled in place and read by its Y' MMA; NKB == 2: read by its epilogue
                mbar_wait(NKB == 1 ? bar_mempty(s) : bar_xempty(s), (u & 1) ^ 1);
                if (NKB == 2 && k == 1) mbar_wait(BAR_CTF, 0);   // stage 1 lives over the C tile
                mbar_expect_tx(bar_xfull(s), nkb * kTile);
                for (int kb = 0; kb < nkb; ++kb)
                    tma_load_2d(sb + Sm::xstage(s) + kb * kTile, &tm_x, bar_xfull(s), h * kP, b * T + 128 * kb);
            }
        }
    } else if (warp == 10) {
        // ================= y storer (NKB == 1): TMA-stores each head's staged y tile =================
        if (NKB == 1 && lane == 0) {
            const uint64_t pol = policy_evict_first();
            for (int k = 0; k < nh; ++k) {
                const int s = k & 1, u = k >> 1;
                mbar_wait(bar_xempty(s), u & 1);
                tma_store_2d_ef(&tm_y, sb + Sm::M0 + s * kTile, (hbeg + k) * kP, b * T, pol);
                bulk_commit();
                bulk_wait_read_all();
                mbar_arrive(bar_yfree(s));
            }
        }
    } else if (warp == 9) {
        // ================= MMA issuer (warp converged, elected lane issues) =================
        mbar_wait(BAR_TREE, 0);
        tc_fence_after();
        if (lane == 0) stamp(2);
        // G = C_rows·Bᵀ, one N = 128 block per 128 keys (NKB == 1: N = Tp16)
        for (int kb = 0; kb < nkb; ++kb) {
            const uint32_t id_g = idesc(kFmtBF16, 0, 128, NKB == 1 ? Tp16 : 128);
#pragma unroll 1
            for (int kk = 0; kk < kN / 16; ++kk) {
                const uint32_t off = (kk >> 2) * kTile + (kk & 3) * 32;
                mma_f16_w(tmem + kGCol + 128 * kb, sdesc(sb + Sm::C + off, 16, 1024),
                          sdesc(sb + Sm::B + 2 * kb * kTile + off, 16, 1024), id_g, kk > 0);
            }
        }
        tc_commit_w(BAR_G);
        mbar_wait(BAR_CTF, 0);   // C as tf32 in TMEM (and B tile free for M' buffer 1 once G completed)
        tc_fence_after();
        const uint32_t* wk = (const uint32_t*)(sm + Sm::WOK);   // factorised heads (written before BAR_CTF)
        const uint32_t fmask = wk[0] & wk[1] & wk[2] & wk[3] & wk[4] & wk[5] & wk[6] & wk[7];
        const uint32_t id_y0 = idesc(kFmtTF32, 0, 128, kP);
        const uint32_t id_y = idesc(kFmtBF16, 1, 128, kP);
        for (int k = 0; k < nh; ++k) {
            const int s = k & 1, a = NKB == 1 ? (k & 1) : 0, u = k >> 1, ua = NKB == 1 ? u : k;
            const uint32_t d0 = tmem + kAccCol + 128 * a, d1 = d0 + 64;
            mbar_wait(bar_accempty(a), (ua & 1) ^ 1);
            tc_fence_after();
            if (prm.has_h0) {
                mbar_wait(bar_hfull(s), u & 1);
                tc_fence_after();
                const uint64_t bd = sdesc(sb + Sm::H + s * 32768, 16, 1024);
#pragma unroll 2
                for (int kk = 0; kk < kN / 8; ++kk)
                    mma_tf32_ts_w(d0, tmem + kCCol + 8 * kk, bd + (uint64_t)(((kk >> 2) * 8192 + (kk & 3) * 32) >> 4),
                                  id_y0, kk > 0);
                tc_commit_w(bar_hempty(s));
            }
            if (lane == 0 && k < 8) stamp(20 + 2 * k);   // Y0 of head k issued
            mbar_wait(bar_mfull(a), ua & 1);
            if (NKB != 1) mbar_wait(bar_xfull(s), u & 1);
            tc_fence_after();
            if (lane == 0 && k < 8) stamp(21 + 2 * k);   // M' and x of head k ready
            if constexpr (NKB == 1) {   // Y' = M_L·X' (factorised: onto Y0) or M'_h·X' (own columns)
                const bool fac = (fmask >> k) & 1u;
                const uint32_t ab = sb + (fac ? Sm::B : Sm::C), dd = fac ? d0 : d1;
                const bool acc0 = fac && prm.has_h0;
                const uint64_t xd = sdesc(sb + Sm::xstage(s), kTile, 1024);   // X' (scaled in place)
#pragma unroll 1
                for (int kk = 0; kk < kcta / 16; ++kk)
                    mma_f16_w(dd, sdesc(ab + (kk >> 2) * kTile + (kk & 3) * 32, 16, 1024), xd + (uint64_t)(kk * 128),
                              id_y, kk > 0 || acc0);
            } else {
                const uint64_t xd = sdesc(sb + Sm::xstage(s), kTile, 1024);
#pragma unroll 1
                for (int kk = 0; kk < kcta / 16; ++kk)
                    mma_f16_w(d1, sdesc(mbuf(a) + (kk >> 2) * kTile + (kk & 3) * 32, 16, 1024), xd + (uint64_t)(kk * 128),
                              id_y, kk > 0);
            }
            tc_commit_w(bar_mempty(a));
            tc_commit_w(bar_accfull(a));
        }
    } else {
        // ================= math warps: row t = TMEM lane (warp % 4 quadrant), column half hh =================
        const int t = tid & 127;                 // row within the tile
        const int hh = tid >> 7;                 // 0: warps 0-3, 1: warps 4-7 (same lanes, other column half)
        const int i = r0 + t;                    // this thread's row (node)
        const uint32_t lane_base = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
        uint32_t* anc = (uint32_t*)(sm + Sm::ANC);    // [word][node]
        int* jmp = (int*)(sm + Sm::JMP);              // [buf][node]
        float* lam = (float*)(sm + Sm::LAM);          // [buf][head][node]
        float* dts = (float*)(sm + Sm::DTS);          // [head][node]
        float* cj = (float*)(sm + Sm::CJ);
        float* as = (float*)(sm + Sm::AS);
        float* ds = (float*)(sm + Sm::DS);
        int* sbad = (int*)(sm + Sm::BADF);
        uint32_t* wok = (uint32_t*)(sm + Sm::WOK);
        auto mbar = [&]() { named_bar(1, 256); };
        constexpr int kW = 4 * NKB;              // ancestor words per node
        // ---- tree prologue over all kT nodes (thread tid: node tid): validation (PAPER.md:90 / R5), ancestor
        //      bits and Λ of every head (Eq. a_tree) by pointer jumping ----
        // A, D, parent and dt loads all in flight together (one memory latency); *sbad was zeroed at setup
        if (tid < nh) {
            as[tid] = prm.A[hbeg + tid];
            ds[tid] = prm.D ? prm.D[hbeg + tid] : 0.f;
        }
        const int v = tid;                       // node of this thread in the prologue (v < kT iff active)
        const int pvv = (v < T && v < kT) ? prm.parent[(size_t)b * T + v] : -1;
        if (v < T && v < kT && (v == 0 ? pvv != -1 : (pvv < 0 || pvv >= v))) atomicMax(sbad, v == 0 ? 2 : 1);
        {   // dt of the chunk's heads, coalesced over (node, head) pairs: all loads in flight together
            constexpr int kLd = (kT * kHPC + 255) / 256;
            float dv[kLd];
#pragma unroll
            for (int r = 0; r < kLd; ++r) {
                const int idx = tid + 256 * r, row = idx / nh, k = idx - row * nh;
                dv[r] = (idx < kT * nh && row < T) ? prm.dt[((size_t)b * T + row) * H + hbeg + k] : 0.f;
            }
#pragma unroll
            for (int r = 0; r < kLd; ++r) {
                const int idx = tid + 256 * r, row = idx / nh, k = idx - row * nh;
                if (idx < kT * nh) dts[k * kT + row] = row < T ? dt_eff(prm.dtx, dv[r], hbeg + k) : 0.f;
            }
        }
        mbar();
        if (tid == 0) stamp(14);   // prologue loads landed
        const int badcode = *sbad == 2 ? 1 : (*sbad == 1 ? 2 : 0);   // root error takes precedence
        if (badcode && tid == 0 && rem == 0 && rt == 0 && !early_tree) report(prm.dev_status, badcode);
        const bool valid = badcode == 0;
        const int cur = 0;   // Λ and jump pointers in one buffer (each round reads, barrier, then writes)
        // NKB == 1 (128 nodes, 256 threads): thread (node t, half hh) handles the heads k ≡ hh (mod 2) and
        // half of the ancestor words; NKB == 2: thread = node, all heads
        constexpr int kSplit = NKB == 1 ? 2 : 1, kHS = kHPC / kSplit, kWS = kW / kSplit;
        const int pv = NKB == 1 ? t : tid;             // prologue node
        const int hsel = NKB == 1 ? hh : 0;
        const bool pact = pv < kT;
        float lv[kHS];       // Λ_v of this thread's heads k = m·kSplit + hsel, in registers
#pragma unroll
        for (int m = 0; m < kHS; ++m) {
            const int k = m * kSplit + hsel;
            lv[m] = (pact && k < nh) ? dts[k * kT + pv] * as[k] : 0.f;
        }
        if (pact) {
#pragma unroll
            for (int w2 = 0; w2 < kWS; ++w2) {
                const int w = hsel * kWS + w2;
                anc[w * kT + pv] = (pv < T && (pv >> 5) == w) ? (1u << (pv & 31)) : 0u;
            }
            if (hsel == 0) jmp[pv] = (valid && pv < T) ? pvv : -1;
#pragma unroll
            for (int m = 0; m < kHS; ++m) {
                const int k = m * kSplit + hsel;
                if (k < nh) lam[k * kT + pv] = lv[m];
            }
        }
        mbar();
        for (int r = 0; r < 7 + NKB - 1; ++r) {
            // read everything of jump target j for this round, barrier, then update this node (race-free
            // under compute-sanitizer racecheck; all loads of a round in flight together)
            uint32_t aj[kWS];
            float lj[kHS];
            const int j = pact ? jmp[pv] : -1;
#pragma unroll
            for (int w2 = 0; w2 < kWS; ++w2) aj[w2] = j >= 0 ? anc[(hsel * kWS + w2) * kT + j] : 0u;
#pragma unroll
            for (int m = 0; m < kHS; ++m) {
                const int k = m * kSplit + hsel;
                lj[m] = (j >= 0 && k < nh) ? lam[k * kT + j] : 0.f;
            }
            const int jj = j >= 0 ? jmp[j] : -1;
            mbar();
            if (pact) {
#pragma unroll
                for (int w2 = 0; w2 < kWS; ++w2) anc[(hsel * kWS + w2) * kT + pv] |= aj[w2];
#pragma unroll
                for (int m = 0; m < kHS; ++m) {
                    const int k = m * kSplit + hsel;
                    lv[m] += lj[m];
                    if (k < nh) lam[k * kT + pv] = lv[m];
                }
                if (hsel == 0) jmp[pv] = jj;
            }
            // stop once no jump pointer is left (depth < 2^(r+1)): heap trees of 128 nodes need 3 rounds
            if (!named_bar_or(1, 256, pact && hsel == 0 && jj >= 0)) break;
        }
        if (tid == 0) stamp(15);   // pointer jumping done
        // decay mode per head: factorised iff min Λ >= -64 over the tree (both factors within e^{±64});
        // otherwise rebased per 32-key chunk (c = node / 32): R_c = max Λ over the chunk,
        // e^{Λi-Λj} = e^{Λi-R_c} · e^{R_c-Λj} with e^{R_c-Λj} <= e^{64} when the chunk's Λ range is <= 64
        // (the row factor may underflow only where the true weight is below e^{-64}); per-element
        // exponentials remain only for heads with a chunk of wider range (stress inputs).  All heads of the
        // thread reduced together (independent shuffle chains).  The per-warp masks carry 1 for the heads
        // the warp does not own, so the AND over the 8 warps is the tree's mask.
        float* rc = (float*)(sm + Sm::RC);
        const bool live = pv < T && pact;
        float mx[kHS], mnv[kHS];
        uint32_t badm = 0u, own = 0u;
#pragma unroll
        for (int m = 0; m < kHS; ++m) {
            const int k = m * kSplit + hsel;
            mx[m] = live ? lv[m] : -3.0e38f;
            mnv[m] = live ? lv[m] : 3.0e38f;
            if (live && k < nh && lv[m] < -64.f) badm |= 1u << k;
            if (k < nh) own |= 1u << k;
        }
#pragma unroll
        for (int m = 0; m < kHS; ++m) {
            mx[m] = warp_max_f32(mx[m]);
            mnv[m] = warp_min_f32(mnv[m]);
        }
        const uint32_t okm = ~__reduce_or_sync(0xffffffffu, badm);
        uint32_t rbm = ~own;
#pragma unroll
        for (int m = 0; m < kHS; ++m)
            if (mx[m] - mnv[m] <= 64.f || mx[m] < -1.0e38f) rbm |= 1u << (m * kSplit + hsel);
        if (lane == 0 && pact) {
#pragma unroll
            for (int m = 0; m < kHS; ++m) {
                const int k = m * kSplit + hsel;
                if (k < nh) rc[k * 8 + (pv >> 5)] = mx[m];
            }
        }
        // both coefficient sets: whether the head factorises is known only once every warp has voted
        if (pact) {
#pragma unroll
            for (int m = 0; m < kHS; ++m) {
                const int k = m * kSplit + hsel;
                if (k < nh) {
                    const float dtv = dts[k * kT + pv];
                    cj[k * kT + pv] = live ? __expf(-lv[m]) * dtv : 0.f;
                    ((float*)(sm + Sm::CR))[k * kT + pv] = live ? __expf(fminf(mx[m] - lv[m], 64.f)) * dtv : 0.f;
                }
            }
        }
        if (lane == 0) {
            wok[warp] = okm;
            ((uint32_t*)(sm + Sm::WRB))[warp] = rbm;
        }
        if (tid == 0) stamp(16);   // decay modes and coefficients done
        if (early_tree) {
            pdl_wait();   // every global write follows the dependency wait
            if (badcode && tid == 0 && rem == 0 && rt == 0) report(prm.dev_status, badcode);
        }
        if (tid == 0) stamp(3);   // tree prologue done
        // C -> tf32 into TMEM columns [kCCol, kCCol + 128) (row t of this tile)
        mbar_wait(BAR_TREE, 0);
        {
#pragma unroll
            for (int c4 = 2 * hh; c4 < 2 * hh + 2; ++c4) {   // this half's 64 columns, 32 per store
                uint32_t r32[32];
#pragma unroll
                for (int q = 0; q < 4; ++q) {   // 4 chunks of 8 bf16
                    const int col = 32 * c4 + 8 * q;
                    const uint4 v = *reinterpret_cast<const uint4*>(sm + Sm::C + (col >> 6) * kTile + swz(t, (col & 63) >> 3));
                    const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        r32[8 * q + 2 * e] = __float_as_uint(bf_lo(wv[e]));
                        r32[8 * q + 2 * e + 1] = __float_as_uint(bf_hi(wv[e]));
                    }
                }
                tmem_st32(lane_base + kCCol + 32 * c4, r32);
            }
            tmem_st_wait();
        }
        mbar();
        const uint32_t fmask = wok[0] & wok[1] & wok[2] & wok[3] & wok[4] & wok[5] & wok[6] & wok[7];
        const uint32_t* wrb = (const uint32_t*)(sm + Sm::WRB);
        const uint32_t rmask = wrb[0] & wrb[1] & wrb[2] & wrb[3] & wrb[4] & wrb[5] & wrb[6] & wrb[7];
        const float* rcf = (const float*)(sm + Sm::RC);
        uint32_t myanc[kW];
#pragma unroll
        for (int w = 0; w < kW; ++w) myanc[w] = anc[w * kT + i];
        tc_fence_before();
        mbar_arrive(BAR_CTF);   // (NKB == 2: the C tile is free for x stage 1 from here)
        if (tid == 0) stamp(4);
        mbar_wait(BAR_G, 0);
        tc_fence_after();
        if (tid == 0) stamp(5);
        const float* laml = lam + cur * kHPC * kT;

        if constexpr (NKB == 1) {
            // Factorised heads: M'_ij = L_ij G_ij c_j with c_j = e^{-Λ_j} dt_j is applied as M_L·(c∘X), where
            // M_L = L∘G is the same for every head of the tree: built ONCE (bf16, over the dead B tile) and
            // each head only scales its x tile by its row coefficients (X'_j = c_j x_j, 64 values per key
            // instead of 128 masked weights per node row).  Non-factorised heads build their own M'_h (row
            // factor e^{min(Λ_i-R_c,0)} per 32-key chunk, or the direct e^{min(Λ_i-Λ_j,0)}) over the dead C
            // tile, against X' = CR∘X (rebased) / dt∘X (direct).  X' is double-buffered over M0.
            auto g_bits = [&](int c4) {
                uint32_t bits = 0u;
#pragma unroll
                for (int w = 0; w < kW; ++w)
                    if (w == c4) bits = myanc[w];
                return bits;
            };
            auto put_row = [&](uint32_t base, int c4, const uint32_t* pk) {   // 32 keys -> 4 swizzled chunks
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int col = 32 * c4 + 8 * q;
                    *reinterpret_cast<uint4*>(sm + base + (col >> 6) * kTile + swz(t, (col & 63) >> 3)) =
                        make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                }
            };
            if (fmask) {
#pragma unroll 1
                for (int c4 = hh; c4 < (kcta + 31) / 32; c4 += 2) {
                    uint32_t gr[32], pk[16];
                    tmem_ld32(lane_base + kGCol + 32 * c4, gr);
                    const uint32_t bits = g_bits(c4);
                    tmem_wait();
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        pk[e] = pack_bf16(((bits >> (2 * e)) & 1u) ? __uint_as_float(gr[2 * e]) : 0.f,
                                          ((bits >> (2 * e + 1)) & 1u) ? __uint_as_float(gr[2 * e + 1]) : 0.f);
                    put_row(Sm::B, c4, pk);
                }
            }
            // raw x of the head (this thread's 4 chunks of row t) is kept in registers from the scaling to the
            // epilogue (the stage itself is rescaled in place and reloaded once the head's Y' MMA completed)
            auto epi = [&](int k, const uint4 (&xr)[4]) {
                const int a = k & 1, s = k & 1, u = k >> 1;
                mbar_wait(bar_accfull(a), u & 1);
                tc_fence_after();
                if (tid == 0 && k < 8) stamp(40 + 2 * k);   // accumulator of head k ready
                const float li = laml[k * kT + i], ei = __expf(li), dh = ds[k];
                const float* dpc = (DPC && prm.D) ? prm.D + (size_t)(hbeg + k) * kP : nullptr;   // D[h][p]
                const bool fac = (fmask >> k) & 1u;
                const uint32_t d0 = lane_base + kAccCol + 128 * a + 32 * hh;
                float acc[32];
                {
                    uint32_t y0[32], y1[32];
                    if (fac) {   // Y0 and Y' in one accumulator, both scaled by e^{Λ_i}
                        tmem_ld32(d0, y0);
                        tmem_wait();
#pragma unroll
                        for (int c = 0; c < 32; ++c) acc[c] = ei * __uint_as_float(y0[c]);
                    } else if (prm.has_h0) {
                        tmem_ld32(d0, y0);
                        tmem_ld32(d0 + 64, y1);
                        tmem_wait();
#pragma unroll
                        for (int c = 0; c < 32; ++c) acc[c] = fmaf(ei, __uint_as_float(y0[c]), __uint_as_float(y1[c]));
                    } else {
                        tmem_ld32(d0 + 64, y1);
                        tmem_wait();
#pragma unroll
                        for (int c = 0; c < 32; ++c) acc[c] = __uint_as_float(y1[c]);
                    }
                }
                tc_fence_before();
                mbar_arrive(bar_accempty(a));
                // y tile staged in Y buffer s (swizzle-128B, the y map's box of T rows clips the rest); the storer
                // warp TMA-stores it — wait until it has read the tile of head k-2 out of this buffer
                mbar_wait(bar_yfree(s), (u & 1) ^ 1);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int col = 32 * hh + 8 * q;
                    const uint32_t xw[4] = {xr[q].x, xr[q].y, xr[q].z, xr[q].w};
                    uint32_t out[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int c = 8 * q + 2 * e;
                        const float d0v = (DPC && dpc) ? __ldg(dpc + col + 2 * e) : dh;
                        const float d1v = (DPC && dpc) ? __ldg(dpc + col + 2 * e + 1) : dh;
                        const float v0 = fmaf(d0v, bf_lo(xw[e]), acc[c]), v1 = fmaf(d1v, bf_hi(xw[e]), acc[c + 1]);
                        out[e] = valid ? pack_bf16(v0, v1) : 0u;
                    }
                    *reinterpret_cast<uint4*>(sm + Sm::M0 + s * kTile + swz(t, col >> 3)) =
                        make_uint4(out[0], out[1], out[2], out[3]);
                }
                fence_proxy_async();
                mbar_arrive(bar_xempty(s));   // y of head k staged
                if (tid == 0 && k < 8) stamp(41 + 2 * k);   // epilogue of head k done
            };
            uint4 xprev[4], xcur[4];
#pragma unroll 1
            for (int k = 0; k < nh; ++k) {
                const int s = k & 1, u = k >> 1;
                const bool fac = (fmask >> k) & 1u, rebased = !fac && ((rmask >> k) & 1u);
                if (!fac && k > 0) mbar_wait(bar_mempty((k - 1) & 1), ((k - 1) >> 1) & 1);   // M'_h tile free
                mbar_wait(bar_xfull(s), u & 1);
                tc_fence_after();
                // X'_h row t (key j = t) = s_j x_j in place, this thread's 32 columns
                const float sc = (fac ? cj : rebased ? (const float*)(sm + Sm::CR) : dts)[k * kT + t];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    uint4* px = reinterpret_cast<uint4*>(sm + Sm::xstage(s) + swz(t, 4 * hh + q));
                    const uint4 v = *px;
                    xcur[q] = v;
                    *px = make_uint4(pack_bf16(sc * bf_lo(v.x), sc * bf_hi(v.x)), pack_bf16(sc * bf_lo(v.y), sc * bf_hi(v.y)),
                                     pack_bf16(sc * bf_lo(v.z), sc * bf_hi(v.z)), pack_bf16(sc * bf_lo(v.w), sc * bf_hi(v.w)));
                }
                if (!fac) {   // this head's own masked weights over the C tile
                    const float li = laml[k * kT + i];
                    const float* lamk = laml + k * kT;
#pragma unroll 1
                    for (int c4 = hh; c4 < (kcta + 31) / 32; c4 += 2) {
                        uint32_t gr[32], pk[16];
                        tmem_ld32(lane_base + kGCol + 32 * c4, gr);
                        const uint32_t bits = g_bits(c4);
                        tmem_wait();
                        if (rebased) {
                            const float fr = __expf(fminf(li - rcf[k * 8 + c4], 0.f));
#pragma unroll
                            for (int e = 0; e < 16; ++e)
                                pk[e] = pack_bf16(((bits >> (2 * e)) & 1u) ? fr * __uint_as_float(gr[2 * e]) : 0.f,
                                                  ((bits >> (2 * e + 1)) & 1u) ? fr * __uint_as_float(gr[2 * e + 1]) : 0.f);
                        } else {
#pragma unroll
                            for (int e = 0; e < 16; ++e) {
                                float wv[2];
#pragma unroll
                                for (int t2 = 0; t2 < 2; ++t2) {
                                    const int jj = 2 * e + t2, j = 32 * c4 + jj;
                                    wv[t2] = ((bits >> jj) & 1u)
                                                 ? __uint_as_float(gr[jj]) * __expf(fminf(li - lamk[j], 0.f)) : 0.f;
                                }
                                pk[e] = pack_bf16(wv[0], wv[1]);
                            }
                        }
                        put_row(Sm::C, c4, pk);
                    }
                }
                fence_proxy_async();
                mbar_arrive(bar_mfull(s));
                if (tid == 0 && k < 8) stamp(6 + k);   // X' (and M'_h) of head k ready
                if (k > 0) epi(k - 1, xprev);
#pragma unroll
                for (int q = 0; q < 4; ++q) xprev[q] = xcur[q];
            }
            epi(nh - 1, xprev);
        } else {
            auto epilogue = [&](int k) {
                const int a = NKB == 1 ? (k & 1) : 0, s = k & 1, u = k >> 1, ua = NKB == 1 ? u : k;
                mbar_wait(bar_accfull(a), ua & 1);
                tc_fence_after();
                if (tid == 0 && k < 8) stamp(40 + 2 * k);   // accumulator of head k ready
                uint32_t y0[32], y1[32];
                const float li = laml[k * kT + i], ei = __expf(li), dh = ds[k];
                const float* dpc = (DPC && prm.D) ? prm.D + (size_t)(hbeg + k) * kP : nullptr;   // D[h][p]
                const bool fac = (fmask >> k) & 1u;
                __nv_bfloat16* yrow = prm.y + (((size_t)b * T + i) * H + hbeg + k) * kP;
                {
                    const int hf = hh;   // this half's 32 output columns
                    tmem_ld32(lane_base + kAccCol + 128 * a + 32 * hf, y0);
                    tmem_ld32(lane_base + kAccCol + 128 * a + 64 + 32 * hf, y1);
                    tmem_wait();
                    uint32_t out[16];
    #pragma unroll
                    for (int q = 0; q < 4; ++q) {   // 8 columns per 16-byte x chunk (x row i of the stage)
                        const int col = 32 * hf + 8 * q;
                        const uint4 xv = *reinterpret_cast<const uint4*>(sm + Sm::xstage(s) + (i >> 7) * kTile +
                                                                         swz(i & 127, col >> 3));
                        const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
    #pragma unroll
                        for (int e = 0; e < 4; ++e) {
                            float v[2];
    #pragma unroll
                            for (int t2 = 0; t2 < 2; ++t2) {
                                const int cc = 8 * q + 2 * e + t2;
                                const float a0 = prm.has_h0 ? __uint_as_float(y0[cc]) : 0.f;
                                const float a1 = __uint_as_float(y1[cc]);
                                const float xx = t2 ? bf_hi(xw[e]) : bf_lo(xw[e]);
                                const float base = fac ? ei * (a0 + a1) : fmaf(ei, a0, a1);
                                v[t2] = valid ? fmaf((DPC && dpc) ? __ldg(dpc + col + 2 * e + t2) : dh, xx, base) : 0.f;
                            }
                            out[4 * q + e] = pack_bf16(v[0], v[1]);
                        }
                    }
                    if (i < T) {
                        uint4* dst = reinterpret_cast<uint4*>(yrow + 32 * hf);
    #pragma unroll
                        for (int q = 0; q < 4; ++q) dst[q] = make_uint4(out[4 * q], out[4 * q + 1], out[4 * q + 2], out[4 * q + 3]);
                    }
                }
                tc_fence_before();
                mbar_arrive(bar_accempty(a));
                mbar_arrive(bar_xempty(s));
                if (tid == 0 && k < 8) stamp(41 + 2 * k);   // epilogue of head k done
            };

            for (int k = 0; k < nh; ++k) {
                const int a = NKB == 1 ? (k & 1) : 0, ua = NKB == 1 ? (k >> 1) : k;
                // ---- masked weights M'(k): row t = L_i∘G_i∘c (factorised) / direct decay, keys 0 .. kcta-1 ----
                mbar_wait(bar_mempty(a), (ua & 1) ^ 1);
                tc_fence_after();
                const bool fac = (fmask >> k) & 1u, rebased = !fac && ((rmask >> k) & 1u);
                const float li = laml[k * kT + i];
                const float* cjk = (fac ? cj : (const float*)(sm + Sm::CR)) + k * kT;
                const float* lamk = laml + k * kT;
                const float* dtk = dts + k * kT;
                const uint32_t mb = mbuf(a);
    #pragma unroll 1
                for (int c4 = hh; c4 < (kcta + 31) / 32; c4 += 2) {   // 32 key columns at a time, halves interleaved
                    uint32_t gr[32];
                    tmem_ld32(lane_base + kGCol + 32 * c4, gr);
                    tmem_wait();
                    uint32_t bits = 0u;
    #pragma unroll
                    for (int w = 0; w < kW; ++w)
                        if (w == c4) bits = myanc[w];
                    uint32_t pk[16];
                    if (fac || rebased) {   // one multiply per element (+ the chunk's row factor), select by L
                        const float fr = rebased ? __expf(fminf(li - rcf[k * 8 + c4], 0.f)) : 1.f;
    #pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            float wv[2];
    #pragma unroll
                            for (int t2 = 0; t2 < 2; ++t2) {
                                const int jj = 2 * e + t2, j = 32 * c4 + jj;
                                const float w = __uint_as_float(gr[jj]) * fr * cjk[j];
                                wv[t2] = ((bits >> jj) & 1u) ? w : 0.f;
                            }
                            pk[e] = pack_bf16(wv[0], wv[1]);
                        }
                    } else {
    #pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            float wv[2];
    #pragma unroll
                            for (int t2 = 0; t2 < 2; ++t2) {
                                const int jj = 2 * e + t2, j = 32 * c4 + jj;
                                float w = 0.f;
                                if ((bits >> jj) & 1u) {
                                    const float gv = __uint_as_float(gr[jj]);
                                    w = gv * __expf(fminf(li - lamk[j], 0.f)) * dtk[j];
                                }
                                wv[t2] = w;
                            }
                            pk[e] = pack_bf16(wv[0], wv[1]);
                        }
                    }
    #pragma unroll
                    for (int q = 0; q < 4; ++q) {   // 4 chunks of 8 keys -> swizzled 16-byte stores
                        const int col = 32 * c4 + 8 * q;
                        *reinterpret_cast<uint4*>(sm + (mb - sb) + (col >> 6) * kTile + swz(t, (col & 63) >> 3)) =
                            make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                    }
                }
                // keys past kcta are never read by the MMA (K = kcta)
                fence_proxy_async();
                mbar_arrive(bar_mfull(a));
                if (tid == 0 && k < 8) stamp(6 + k);   // M' of head k built
                if (NKB == 1) {
                    if (k > 0) epilogue(k - 1);
                } else {
                    epilogue(k);   // single accumulator slot / M' buffer: head k+1 waits for this one
                }
            }
            if (NKB == 1) epilogue(nh - 1);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) stamp(63);
    if (warp == 9) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCols));
    }
}

}  // namespace tc128
}  // namespace stree

namespace {
// debug timeline (not part of the ABI): launch i writes its per-CTA stamps to buf + (i % 16) * 1024 * 64
unsigned long long* g_tc128_trace = nullptr;
int g_tc128_trace_n = 0;
bool map2d(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
           uint32_t box_inner, uint32_t box_outer) {
    return stree::host::tmap_2d(m, dt, base, inner, outer, row_bytes, box_inner, box_outer);
}
}  // namespace

extern "C" int stree_tc128_supports(const stree_dims* d) {
    if (!d || d->io_dtype != STREE_BF16 || d->head_dim != stree::tc128::kP || d->d_state != stree::tc128::kN) return 0;
    if (d->n_nodes < 1 || d->n_nodes > 256) return 0;
    if (d->n_groups < 1 || d->n_heads % d->n_groups) return 0;
    return 1;
}

namespace {
template <int NKB, bool DPC>
int launch_tc128(const stree_dims* d, const CUtensorMap& mc, const CUtensorMap& mb, const CUtensorMap& mx,
                 const CUtensorMap& mh, const CUtensorMap& my, const stree::tc128::Params& base, cudaStream_t s) {
    using namespace stree::tc128;
    using S = Sm<NKB>;
    const int B = d->batch, H = d->n_heads, G = d->n_groups;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int hpg = H / G;
    int cpg = nsm / (B * G * NKB);
    if (cpg < 1) cpg = 1;
    if (cpg > hpg) cpg = hpg;
    int hpc = (hpg + cpg - 1) / cpg;
    if (hpc > S::kHPC) hpc = S::kHPC;
    cpg = (hpg + hpc - 1) / hpc;
    Params prm = base;
    prm.cpg = cpg;
    prm.hpc = hpc;
    const size_t smem = S::TOTAL + 1024;
    auto k = scan_tc128_kernel<NKB, DPC>;
    cudaError_t e = stree::host::smem_attr((const void*)k, (int)smem);
    if (e != cudaSuccess) return (int)e;
    e = stree::launch_k(k, dim3(B * G * cpg * NKB), dim3(kThreads), smem, s, mc, mb, mx, mh, my, prm);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
}
}  // namespace

extern "C" int stree_launch_scan_tc128(const stree_dims* d, const void* x, const float* dt, const float* A,
                                       const void* Bm, const void* Cm, const float* D, const float* h0,
                                       const int32_t* parent, void* y, int32_t* dev_status, cudaStream_t s) {
    using namespace stree::tc128;
    if (!stree_tc128_supports(d)) return (int)cudaErrorNotSupported;
    const int B = d->batch, T = d->n_nodes, H = d->n_heads, P = d->head_dim, N = d->d_state, G = d->n_groups;
    CUtensorMap mc, mb, mx, mh, my;
    const uint64_t BT = (uint64_t)B * T;
    bool ok = map2d(&mc, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, Cm, (uint64_t)G * N, BT, (uint64_t)G * N * 2, 64, 128) &&
              map2d(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, Bm, (uint64_t)G * N, BT, (uint64_t)G * N * 2, 64, 128) &&
              map2d(&mx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, x, (uint64_t)H * P, BT, (uint64_t)H * P * 2, 64, 128);
    if (h0)
        ok = ok && map2d(&mh, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, h0, (uint64_t)N, (uint64_t)B * H * P, (uint64_t)N * 4, 32, 64);
    else
        mh = mx;
    // y tile store (T <= 128): box of T rows, so a tree's store never touches the next tree's rows
    if (T <= 128)
        ok = ok && map2d(&my, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, y, (uint64_t)H * P, BT, (uint64_t)H * P * 2, 64, T);
    else
        my = mx;
    if (!ok) return (int)cudaErrorInvalidValue;
    Params prm{};
    prm.dt = dt; prm.A = A; prm.D = D; prm.parent = parent; prm.y = (__nv_bfloat16*)y; prm.dev_status = dev_status;
    prm.B = B; prm.T = T; prm.H = H; prm.G = G; prm.has_h0 = h0 != nullptr;
    prm.dtx = stree::DtX::from(stree_scan_opts_get());
    prm.d_pc = (stree_scan_opts_get() && stree_scan_opts_get()->d_per_channel) ? 1 : 0;
    prm.trace = g_tc128_trace ? g_tc128_trace + (size_t)(g_tc128_trace_n++ % 16) * 1024 * kTraceWords : nullptr;
    prm.early_tree = (stree_launch_flags_get() & STREE_LAUNCH_EARLY_TREE) ? 1 : 0;
    prm.early_dt = (stree_launch_flags_get() & STREE_LAUNCH_EARLY_DT) ? 1 : 0;
    prm.early_state = (stree_launch_flags_get() & STREE_LAUNCH_EARLY_STATE) ? 1 : 0;
    if (prm.d_pc)
        return T <= 128 ? launch_tc128<1, true>(d, mc, mb, mx, mh, my, prm, s) : launch_tc128<2, true>(d, mc, mb, mx, mh, my, prm, s);
    return T <= 128 ? launch_tc128<1, false>(d, mc, mb, mx, mh, my, prm, s) : launch_tc128<2, false>(d, mc, mb, mx, mh, my, prm, s);
}

extern "C" void stree_debug_tc128_trace(unsigned long long* dev_buf) {
    g_tc128_trace = dev_buf;
    g_tc128_trace_n = 0;
}
