// K2 stree_tree_scan on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// The packed-tree SSM output of PAPER.md:91-102 (Mamba-2 realisation):
//     y_i = e^{Λ_i} C_i·h0_hᵀ  +  Σ_{j∈path(i)} e^{Λ_i-Λ_j} dt_j (C_i·B_j) x_j  +  D_h x_i
// as three dense contractions per tree / head, all on chip:
//     G   = C·Bᵀ                 (T x T, K = N)    kind::f16   bf16 x bf16 -> fp32 TMEM   (once per tree)
//     Y0  = C·h0_hᵀ              (T x P, K = N)    kind::tf32  fp32 state  -> fp32 TMEM   (per head; dominant stream)
//     Y'  = (L∘G∘c_h)·X_h        (T x P, K = T)    kind::f16   bf16 masked weights x bf16 x   (per head)
// and an epilogue y = e^{Λ_i} (Y0 + Y') + D x (fp32) -> bf16 -> TMA store.
// Λ = L·(dt A_h) is the tree segsum (Eq. a_tree) built by pointer
// jumping over the ancestor chains; the decay mask is applied before any exp
// (SURVEY R4).  The decay factorises, e^{Λ_i-Λ_j} = e^{Λ_i}·e^{-Λ_j}, whenever
// min Λ >= -64 (both factors inside fp32 range with e^{64} of headroom): then
// c_j = e^{-Λ_j} dt_j, Y' accumulates onto Y0 in the same TMEM columns and the
// epilogue applies the single row factor e^{Λ_i}.  Heads with deeper decay use
// the direct per-element e^{Λ_i-Λ_j} with Y' in separate TMEM columns.
//
// One CTA = one tree and a range of heads of one group (grid = B x G x chunks, <= #SMs CTAs),
// warp-specialised, 320 threads (scan) / 352 threads (fused replay + scan, MODE 1; commit only, MODE 2):
//   warp 0        TMA producer: C, B once; then per head the 32 KB state (4 boxes) into a 4-slot ring and
//                 the x tile into the x ring
//   warp 1        tcgen05.mma issuer (one elected lane of a converged warp) + TMEM allocator (512 columns)
//   warps 2-3     (+ 6-7 in the scan) masked weights M' of head k+1 from G rows in TMEM lanes 64-127
//   warps 4-5     (+ 8-9 in the scan) epilogue of head k (TMEM lanes 0-63 = tree nodes) and the x stream
//   warps 6-9     (MODE 1/2) activation replay of the previous tree's accepted path on each state slot
//   warp 10       (MODE 1/2) TMA store of the committed state slot (in place)
// The tree / segsum prologue runs on the builder and epilogue warps before the first head (before the
// dependency wait under the STREE_LAUNCH_EARLY_* promises).  DESIGN.md §6 (K2, K2f, K4p) has the details.
// Rows are the tree nodes (M = 128 with rows >= T ignored; every MMA row is
// independent so the unused rows may read arbitrary shared memory).
//
// Served shapes: bf16 io, P = 64, N in {64, 128}, 1 <= T <= 64.  Everything
// else goes to the SIMT kernel (stree_scan_simt.cu).
#include <cuda.h>

#include "stree_common.cuh"
#include "stree_host.cuh"
#include "stree_tc_ptx.cuh"

namespace stree {
namespace tc {

constexpr int kT = 64;          // max nodes per tree served
constexpr int kP = 64;          // head dim
constexpr int kHPC = 10;        // max heads per CTA
constexpr int kThreadsScan = 320;     // warps 0 TMA, 1 MMA, 2-3 + 6-7 builders, 4-5 + 8-9 epilogue
constexpr int kThreadsReplay = 352;   // warps 0-5 as the scan's first six, 6-9 replay updaters, 10 state stores
constexpr int kUpd0 = 192;            // first replay-updater thread (warp 6)
constexpr int kTraceWords = 256;   // debug trace: u64 stamps per CTA (stree_debug_tc_trace)
#ifdef STREE_TRACE
constexpr bool kTrace = true;      // timeline instrumentation compiled in (STREE_TRACE=1 builds, tools/trace_*.py)
#else
constexpr bool kTrace = false;     // production: no instrumentation code in the kernels (instruction-cache footprint)
#endif
constexpr int kRStage = 8;            // previous-path nodes staged on chip by the replay
constexpr int kEpi0 = 64;       // first epilogue thread
constexpr int kAtom = 8192;     // one 64-row x 128-byte swizzle-128B tile
constexpr uint32_t kTmemCols = 512;
constexpr int kCCol = 64;       // C as tf32 (A operand of Y0) in TMEM columns [64, 64 + N)
constexpr int kAccCol0 = 192;   // accumulator a (of kAcc): columns [192 + 64a, 256 + 64a)
constexpr int kAcc = 4;
constexpr int kDirCol = 448;    // Y' of direct-decay heads (rare): columns [448, 512)

template <int NS, bool R>
struct Smem {
    static constexpr int kSt = 4;                         // state (h0) ring depth: 2 pairs of head slots
    static constexpr int kStX0 = R ? 3 : 4;               // x slots in the X region
    static constexpr int kXB = NS >= 128 ? 2 : 0;         // + x slots in the B tile region, free after G = C·Bᵀ
    static constexpr int kStX = kStX0 + kXB;              // x ring depth
    static constexpr int kCbAtoms = NS / 64;              // bf16 C / B: 64 bf16 per 128B
    static constexpr int U = 0;                           // union: {C bf16, B bf16} then {M'[2], ystage[2]}
    static constexpr int CB = U;                          // C bf16: atom a at CB + 2a*kAtom, copy at +kAtom
    static constexpr int BB = U + 2 * kCbAtoms * kAtom;
    static constexpr int MB = U;                          // M'[a] at MB + a*kAtom
    static constexpr int YS = U + 2 * kAtom;              // ystage[a] at YS + a*kAtom
    static constexpr int UBYTES = (3 * kCbAtoms * kAtom > 4 * kAtom) ? 3 * kCbAtoms * kAtom : 4 * kAtom;
    static constexpr int H0 = U + UBYTES;                 // h0 stages
    static constexpr int H0S = kP * NS * 4;               // bytes per stage
    // the two head slots of a pair interleave by atom, so the pair is one 128-row K-major operand
    // (Y0 of both heads in one N = 128 MMA): atom a of slot s at slot(s) + a * kSlotAtom
    static constexpr int kSlotAtom = 2 * kAtom;
    __device__ static constexpr int slot(int s) { return H0 + (s >> 1) * 2 * H0S + (s & 1) * kAtom; }
    static constexpr int X = H0 + kSt * H0S;              // x stages
    static constexpr int XS = kAtom;
    static constexpr int MISC = X + kStX0 * XS;
    __device__ static constexpr int xslot(int s) { return s < kStX0 ? X + s * XS : BB + (s - kStX0) * XS; }
    // misc (4-byte words unless noted)
    static constexpr int PAR = MISC;                      // int[64]
    static constexpr int ROWS = PAR + 64 * 4;             // u64[64]
    static constexpr int LAM = ROWS + 64 * 8;             // float[kHPC][64]
    static constexpr int CJ = LAM + kHPC * 64 * 4;        // float[kHPC][64]
    static constexpr int E0 = CJ + kHPC * 64 * 4;         // float[kHPC][64]
    static constexpr int MODE = E0 + kHPC * 64 * 4;       // int[kHPC]
    static constexpr int AS = MODE + kHPC * 4;            // float[kHPC]  A_h
    static constexpr int DS = AS + kHPC * 4;              // float[kHPC]  D_h
    static constexpr int BADF = DS + kHPC * 4;            // int
    // replay (fused commit of the previous tree)
    static constexpr int RPATH = BADF + 16;               // int[kMaxNodes]   previous accepted path
    static constexpr int RINFO = RPATH + (R ? kMaxNodes * 4 : 0);   // int[4]: r (0 = invalid / nothing)
    static constexpr int RCOEF = RINFO + 16;              // float[kHPC][kRStage] c_{h,m} of the staged nodes
    static constexpr int RLAM = RCOEF + (R ? kHPC * kRStage * 4 : 0);     // float[kHPC][2]: lam_{r-1}, lam_{kRStage-1}
    static constexpr int RDEC = RLAM + (R ? kHPC * 8 : 0);                // float[kHPC] decay
    static constexpr int XPREV = RDEC + (R ? kHPC * 4 : 0);               // bf16 [kHPC][kRStage][64]
    static constexpr int BPREV = XPREV + (R ? kHPC * kRStage * kP * 2 : 0);   // float[kRStage][NS]
    static constexpr int BAR = (BPREV + (R ? kRStage * NS * 4 : 0) + 7) & ~7;
    // barriers (u64): tree, ctf32, gdone, hfull[S], hempty[S], mfull[2], mempty[2], accfull[kAcc],
    //                 accempty[kAcc], dirempty, upd[S], xfull[kStX]
    static constexpr int NBAR = 3 + 2 * kSt + 4 + 2 * kAcc + 1 + kSt + kStX + 1;   // + debug
    static constexpr int BAR2 = 24 + 16 * kSt;                       // byte offset of mfull[0]
    static constexpr int BAR3 = BAR2 + 8 * (4 + 2 * kAcc + 1);       // byte offset of upd[0]
    static constexpr int TMEMP = BAR + NBAR * 8;
    static constexpr int TOTAL = TMEMP + 16;
    static_assert(TOTAL + 1024 <= 227 * 1024, "shared memory budget");
};

struct Params {
    unsigned long long* trace;  // optional per-CTA phase timestamps (debug)
    int B, T, H, G, cpg, hpc;  // cpg = head chunks per group, hpc = heads per chunk
    const float* dt;
    const float* A;
    const float* D;
    const int32_t* parent;
    __nv_bfloat16* y;
    int32_t* dev_status;
    int has_h0;
    int early_state;   // STREE_LAUNCH_EARLY_STATE: h0 may be streamed before the PDL wait
    int early_replay;  // STREE_LAUNCH_EARLY_REPLAY: the replay prologue may run before the PDL wait
    int early_tree;    // STREE_LAUNCH_EARLY_TREE: parent, A, D not written by the preceding kernel
    DtX dtx;           // *_ex options: effective dt (bias, softplus)
    int d_pc;          // *_ex options: D is [H][P]
    int early_dt;      // STREE_LAUNCH_EARLY_DT: dt not written by the preceding kernel (with early_tree: the
                       // whole tree prologue runs before the wait)
    int store_always;  // commit into a distinct h_new: store the state even when the path is invalid
    // replay (fused commit of the previous tree), kReplay only
    int Tp;
    const __nv_bfloat16* x_prev;
    const float* dt_prev;
    const __nv_bfloat16* b_prev;
    const int32_t* parent_prev;
    const int32_t* path;
    const int32_t* path_len;
    // head-sharded layer (stree_*_sharded): y tiles go to every peer's full-y buffer at y_head_off + h
    int n_ypeer, y_head_off;
};
// y destinations: the local y map (NoYPeers) or one map per peer buffer (stree_yout)
struct NoYPeers {
    int unused;
};
struct YPeerMaps {
    CUtensorMap m[STREE_MAX_Y_PEERS];
};

// ---------------------------------------------------------------------------
// Replay updaters (fused mode, warps 6-9): activation replay of the previous tree's accepted path
// (Alg. 1 l.123) applied on chip to each TMA-staged state tile before the scan uses it:
//   h <- e^{lam_{r-1}} h + Σ_m c_m x_prev[s_m] B_prev[s_m]ᵀ,  c_m = e^{lam_{r-1} - lam_m} dt_prev[s_m],
//   lam_m = Σ_{q<=m} dt_prev[s_q] A_h   (the path-cumsum of log-decays, PAPER.md:86-90 on the path).
// The updated tile is the carry-in of the scan (bar_upd) and is TMA-stored as the committed state.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

template <int NS, bool R>
__device__ __forceinline__ void replay_updater(const Params& prm, unsigned char* sm, uint32_t sb,
                                               const CUtensorMap* tm_h, int b, int g, int chunk, int hbeg, int nh,
                                               uint32_t bar0) {
    using S = Smem<NS, R>;
    constexpr int kSt = S::kSt;
    auto bar_full = [&](int s) { return bar0 + 24 + 8 * s; };            // state tile landed
    auto bar_empty = [&](int s) { return bar0 + 24 + 8 * kSt + 8 * s; };  // state tile free
    auto bar_upd = [&](int s) { return bar0 + S::BAR3 + 8 * s; };
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int u = tid - kUpd0;            // 0..127
    const int uw = warp - 6;              // 0..3
    const int H = prm.H, Tp = prm.Tp, G = prm.G;
    int* rpath = (int*)(sm + S::RPATH);
    int* rinfo = (int*)(sm + S::RINFO);
    float* rcoef = (float*)(sm + S::RCOEF);
    float* rlam = (float*)(sm + S::RLAM);
    float* rdec = (float*)(sm + S::RDEC);
    __nv_bfloat16* xprev = (__nv_bfloat16*)(sm + S::XPREV);
    float* bprev = (float*)(sm + S::BPREV);
    // ---- previous accepted path.  Two rounds of DRAM latency: the path itself, then everything that
    //      depends only on it (validation, dt_prev, x_prev rows, B_prev rows), issued together ----
    const int r_raw = prm.path_len[b];
#pragma unroll 1
    for (int m = u; m < Tp; m += 128) rpath[m] = prm.path[(size_t)b * Tp + m];
    named_bar(3, 128);
    const int rr = (r_raw >= 1 && r_raw <= Tp) ? r_raw : 0;   // candidate length, validated below
    const int rs = min(rr, kRStage);
    auto node = [&](int m) {   // path node clamped into the tree: loads stay in bounds before validation
        const int v = rpath[m];
        return (v >= 0 && v < Tp) ? v : 0;
    };
    constexpr int kQ = (kHPC + 3) / 4;    // heads per updater warp: uw, uw + 4, uw + 8
    float dv[kQ][2];
    uint32_t xv[kQ][kRStage];
    // row offsets of the path nodes: dt_prev / x_prev rows (b, node) of the previous tree
    const size_t row0 = ((size_t)b * Tp + node(lane)) * H + hbeg, row1 = ((size_t)b * Tp + node(lane + 32)) * H + hbeg;
    size_t rowm[kRStage];
#pragma unroll
    for (int m = 0; m < kRStage; ++m) rowm[m] = ((size_t)b * Tp + node(m)) * H + hbeg;
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
        const int hh = uw + 4 * q;
        const bool hv = hh < nh;
        dv[q][0] = (hv && lane < rr) ? dt_eff(prm.dtx, prm.dt_prev[row0 + hh], hbeg + hh) : 0.f;
        dv[q][1] = (hv && lane + 32 < rr) ? dt_eff(prm.dtx, prm.dt_prev[row1 + hh], hbeg + hh) : 0.f;
        const uint32_t* xp = reinterpret_cast<const uint32_t*>(prm.x_prev) + lane;
#pragma unroll
        for (int m = 0; m < kRStage; ++m) xv[q][m] = (hv && m < rs) ? xp[(rowm[m] + hh) * (kP / 2)] : 0u;
    }
#pragma unroll 1
    for (int k = u; k < rs * NS; k += 128) {
        const int m = k / NS, n = k % NS;
        bprev[m * NS + n] = __bfloat162float(prm.b_prev[(((size_t)b * Tp + node(m)) * G + g) * NS + n]);
    }
    {   // root-anchored, increasing, parent-linked (PAPER.md:90 on the accepted path); every updater
        // warp runs the same check (no warp-divergent branch around the vote)
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
        if (u == 0) {
            rinfo[0] = ok ? rr : 0;
            rinfo[1] = ok ? 0 : 1;
        }
    }
    named_bar(3, 128);
    // no global writes here: with EARLY_REPLAY (and EARLY_STATE) the whole replay of the state tiles already in
    // flight runs before the dependency wait; the storer warp (after its wait) reports an invalid path and
    // writes the committed state
    // r is read back from shared memory and broadcast, so every branch on it is provably warp-uniform
    // (no collective fix-up code around the shuffles below)
    const int r = __shfl_sync(0xffffffffu, rinfo[0], 0);
#pragma unroll
    for (int q = 0; q < kQ; ++q) {
        const int hh = uw + 4 * q;
        const bool hv = hh < nh && r > 0;
        const float Ah = hv ? prm.A[hbeg + hh] : 0.f;
        // lam_m = Σ_{q<=m} dt_prev[s_q] A_h: inclusive warp scans over m = lane and lane + 32
        float a0 = dv[q][0] * Ah, a1 = dv[q][1] * Ah;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const float t0 = __shfl_up_sync(0xffffffffu, a0, o), t1 = __shfl_up_sync(0xffffffffu, a1, o);
            if (lane >= o) { a0 += t0; a1 += t1; }
        }
        a1 += __shfl_sync(0xffffffffu, a0, 31);
        const float l32 = __shfl_sync(0xffffffffu, a0, (r - 1) & 31), l64 = __shfl_sync(0xffffffffu, a1, (r - 33) & 31);
        float last = r <= 32 ? l32 : l64;
        if (r > 64) {   // paths beyond 64 nodes: the remaining chunks from global memory
            float carry = __shfl_sync(0xffffffffu, a1, 31);
#pragma unroll 1
            for (int m0 = 64; m0 < r; m0 += 32) {
                const int m = m0 + lane;
                float a = (hv && m < r) ? dt_eff(prm.dtx, prm.dt_prev[((size_t)b * Tp + node(m)) * H + hbeg + hh], hbeg + hh) * Ah : 0.f;
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
        if (hv) {
            if (lane < rs) rcoef[hh * kRStage + lane] = __expf(last - a0) * dv[q][0];
            if (lane == 0) {
                rdec[hh] = __expf(last);
                rlam[2 * hh] = last;
                rlam[2 * hh + 1] = lst;
            }
#pragma unroll
            for (int m = 0; m < kRStage; ++m)
                if (m < rs) reinterpret_cast<uint32_t*>(xprev + (hh * kRStage + m) * kP)[lane] = xv[q][m];
        }
    }
    named_bar(3, 128);
    // ---- per head: replay the state tile in place (swizzle-128B K-major layout of the TMA boxes).
    //      Thread u owns logical chunk pc (columns 4 pc .. 4 pc + 3 of every atom) of rows
    //      (u >> 3) + 16 i: its 16 chunks stay in registers while the path is applied. ----
    const int pc = u & 7;
    constexpr int kAt = NS / 32;
    unsigned long long* trace = (kTrace && prm.trace) ? prm.trace + (size_t)blockIdx.x * kTraceWords : nullptr;
    for (int k = 0; k < nh; ++k) {
        const int s = k % kSt;
        mbar_wait(bar_full(s), (k / kSt) & 1);
        if (trace && u == 0 && k < 12) trace[64 + 3 * k] = gtimer();
        if (r > 0 && !(trace && (trace[127] & 4))) {   // debug knob 4: skip the tile update
            const float dk = rdec[k];
            const float* cl = rcoef + k * kRStage;
            const float Ak = prm.A[hbeg + k], last = rlam[2 * k];
            float lam_run = rlam[2 * k + 1];   // long paths: lam_m accumulated from the last staged node
            unsigned char* tile = sm + S::slot(s);
            float4 hv[4][kAt];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int a = 0; a < kAt; ++a) {
                    float4 v = *reinterpret_cast<const float4*>(tile + a * S::kSlotAtom + swz((u >> 3) + 16 * i, pc));
                    hv[i][a] = make_float4(dk * v.x, dk * v.y, dk * v.z, dk * v.w);
                }
#pragma unroll 1
            for (int m = 0; m < r; ++m) {
                const bool st_ = m < kRStage;
                float4 bb[kAt];
                float uu[4];
                if (st_) {
#pragma unroll
                    for (int a = 0; a < kAt; ++a) bb[a] = *reinterpret_cast<const float4*>(&bprev[m * NS + 32 * a + 4 * pc]);
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        uu[i] = cl[m] * __bfloat162float(xprev[(k * kRStage + m) * kP + (u >> 3) + 16 * i]);
                } else {   // long accepted paths: operands and coefficients from L2 / on the fly
                    const int sm_ = rpath[m];
                    const float dm = dt_eff(prm.dtx, prm.dt_prev[((size_t)b * Tp + sm_) * H + hbeg + k], hbeg + k);
                    lam_run += dm * Ak;
                    const float cm = __expf(last - lam_run) * dm;
                    const __nv_bfloat16* br = prm.b_prev + (((size_t)b * Tp + sm_) * G + g) * NS + 4 * pc;
#pragma unroll
                    for (int a = 0; a < kAt; ++a)
                        bb[a] = make_float4(__bfloat162float(br[32 * a]), __bfloat162float(br[32 * a + 1]),
                                            __bfloat162float(br[32 * a + 2]), __bfloat162float(br[32 * a + 3]));
                    const __nv_bfloat16* xr = prm.x_prev + (((size_t)b * Tp + sm_) * H + hbeg + k) * kP;
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
                    *reinterpret_cast<float4*>(tile + a * S::kSlotAtom + swz((u >> 3) + 16 * i, pc)) = hv[i][a];
        }
        fence_proxy_async();
        named_bar(3, 128);
        if (trace && u == 0 && k < 12) trace[65 + 3 * k] = gtimer();
        if (u == 0) mbar_arrive(bar_upd(s));   // to the MMA issuer (Y0) and the state storer
    }
}

// Warp 10 (one thread): the committed state back to HBM, in place, once a slot has been replayed; the
// slot is released (with the MMA issuer's Y0 commit) when the store has read it.  Kept off the updater
// warps so they never stall on the store.
template <int NS, bool R>
__device__ __forceinline__ void state_storer(const Params& prm, unsigned char* sm, uint32_t sb, const CUtensorMap* tm_h,
                                             int b, int hbeg, int nh, uint32_t bar0, bool report_bad) {
    using S = Smem<NS, R>;
    constexpr int kSt = S::kSt;
    auto bar_empty = [&](int s) { return bar0 + 24 + 8 * kSt + 8 * s; };
    auto bar_upd = [&](int s) { return bar0 + S::BAR3 + 8 * s; };
    unsigned long long* trace = (kTrace && prm.trace) ? prm.trace + (size_t)blockIdx.x * kTraceWords : nullptr;
    const uint64_t pol = policy_evict_first();
    const int H = prm.H;
    if (prm.early_replay) pdl_wait();   // stores (and the status report) follow the dependency wait
    for (int k = 0; k < nh; ++k) {
        const int s = k % kSt;
        mbar_wait(bar_upd(s), (k / kSt) & 1);
        if (k == 0 && ((const int*)(sm + S::RINFO))[1] && report_bad) report(prm.dev_status, STREE_DEV_BAD_PATH);
        if (((const int*)(sm + S::RINFO))[0] > 0 || prm.store_always) {   // path length, published before bar_upd
#pragma unroll 1
            for (int a = 0; a < NS / 32; ++a)
                tma_store_2d_ef(tm_h, sb + S::slot(s) + a * S::kSlotAtom, 32 * a, ((b * H) + hbeg + k) * kP, pol);
            bulk_commit();
            bulk_wait_read0();
            if (trace && k < 12) trace[66 + 3 * k] = gtimer();
        }
        mbar_arrive(bar_empty(s));
    }
    bulk_wait_read_all();
}

// MODE 0: tree scan; 1: replay of the previous tree's accepted path fused with the scan (in place);
// 2: replay only (stree_commit): warps 0 (state producer), 6-9 (replay) and 10 (stores to tm_y = h_new)
// DPC: D is [H][P] (stree_scan_opts.d_per_channel) — a separate instantiation: a runtime branch in the
// epilogue costs ~1 us per c4 layer even when not taken
template <int NS, int MODE, typename YM = NoYPeers, bool DPC = false>
__global__ void __launch_bounds__(MODE ? kThreadsReplay : kThreadsScan, 1)
    scan_tc_kernel(const __grid_constant__ CUtensorMap tm_c, const __grid_constant__ CUtensorMap tm_b,
                   const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_h0,
                   const __grid_constant__ CUtensorMap tm_y, const __grid_constant__ YM ym, const Params prm) {
    constexpr bool kPeers = sizeof(YM) > sizeof(int);
    constexpr bool kReplay = MODE >= 1, kScan = MODE <= 1;
    // scan only: 8 math warps, two per TMEM lane quadrant, each pair splitting the columns of its rows
    // (builders: j halves of M'; epilogue: p halves of y).  With replay: 4 (warps 6-10 replay / store).
    constexpr bool kSplit = !kReplay;
    constexpr int kMathW = kSplit ? 8 : 4;
    constexpr int kMath = 32 * kMathW;   // math threads (warps 2 .. 2 + kMathW)
    constexpr int kEpiT = kMath / 2;     // epilogue threads
    using S = Smem<NS, kReplay>;
    constexpr int kStages = S::kSt;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* sm = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t sb = smem_u32(sm);
    unsigned long long* trace = (kTrace && prm.trace) ? prm.trace + (size_t)blockIdx.x * kTraceWords : nullptr;
    if (trace && threadIdx.x == 0) trace[0] = gtimer();
    // warp index and TMEM base broadcast from lane 0: provably warp-uniform for ptxas, so descriptor and
    // address arithmetic stays on the uniform datapath (no per-instruction waterfall around tcgen05/TMA)
    const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
    const int T = prm.T, H = prm.H;
    const int b = blockIdx.x / (prm.G * prm.cpg);
    const int rem = blockIdx.x % (prm.G * prm.cpg);
    const int g = rem / prm.cpg, chunk = rem % prm.cpg;
    const int hpg = H / prm.G;
    const int hbeg = g * hpg + chunk * prm.hpc;
    const int nh = min(prm.hpc, g * hpg + hpg - hbeg);
    if (nh <= 0) { pdl_wait(); return; }
    int* sp = (int*)(sm + S::PAR);

    const uint32_t bar0 = sb + S::BAR;
    const uint32_t BAR_TREE = bar0, BAR_CTF = bar0 + 8, BAR_G = bar0 + 16;
    auto bar_full = [&](int s) { return bar0 + 24 + 8 * s; };
    auto bar_empty = [&](int s) { return bar0 + 24 + 8 * kStages + 8 * s; };
    auto bar_mfull = [&](int a) { return bar0 + S::BAR2 + 8 * a; };
    auto bar_mempty = [&](int a) { return bar0 + S::BAR2 + 16 + 8 * a; };
    auto bar_accfull = [&](int a) { return bar0 + S::BAR2 + 32 + 8 * a; };
    auto bar_accempty = [&](int a) { return bar0 + S::BAR2 + 32 + 8 * kAcc + 8 * a; };
    const uint32_t BAR_DIRE = bar0 + S::BAR2 + 32 + 16 * kAcc;                       // direct Y' read
    auto bar_upd = [&](int s) { return bar0 + S::BAR3 + 8 * s; };                    // replay: stage s updated
    auto bar_xfull = [&](int s) { return bar0 + S::BAR3 + 8 * kStages + 8 * s; };    // x tile landed
    uint32_t* tmem_slot = (uint32_t*)(sm + S::TMEMP);

    // ---- setup that touches no argument memory (overlaps the previous grid under PDL) ----
    if (tid == 0) {
        mbar_init(BAR_TREE, 1);
        mbar_init(BAR_CTF, kMath);
        mbar_init(BAR_G, 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(bar_full(s), 1);
            mbar_init(bar_empty(s), (kReplay && kScan) ? 2 : 1);   // state tile: MMA (Y0) and / or the store read
            mbar_init(bar_upd(s), 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(bar_mfull(a), kMathW / 2);
            mbar_init(bar_mempty(a), 1);
        }
        for (int a = 0; a < kAcc; ++a) {
            mbar_init(bar_accfull(a), 1);
            mbar_init(bar_accempty(a), kMathW / 2);
        }
        mbar_init(BAR_DIRE, kMathW / 2);
        if (kTrace) mbar_init(bar0 + (S::NBAR - 1) * 8, 1);
        for (int s = 0; s < S::kStX; ++s) mbar_init(bar_xfull(s), 1);
        fence_barrier_init();
    }
    if (kScan && warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const int n_early = (prm.early_state && prm.has_h0) ? min(kStages, nh) : 0;   // whole state ring
    if (warp == 0 && lane == 0) {
        tma_prefetch(&tm_c); tma_prefetch(&tm_b); tma_prefetch(&tm_x); tma_prefetch(&tm_h0); tma_prefetch(&tm_y);
        // the state of the first heads is streamed before the dependency wait (caller's promise)
        for (int k = 0; k < n_early; ++k) {
            mbar_expect_tx(bar_full(k), S::H0S);   // arrive now: the replay of this tile may start pre-wait
#pragma unroll 1
            for (int a = 0; a < NS / 32; ++a)
                tma_load_2d(sb + S::slot(k) + a * S::kSlotAtom, &tm_h0, bar_full(k), 32 * a,
                            ((b * H) + hbeg + k) * kP);
        }
    }
    // replay warps with the EARLY_REPLAY promise wait inside their own code (after the prologue's
    // loads of the previous tree's operands, before any global write)
    // math warps with the EARLY_TREE + EARLY_DT promises run the whole tree prologue (loads, validation,
    // pointer jumping, Λ, decay coefficients) before their dependency wait
    const bool math_thread = kScan && tid >= kEpi0 && tid < kEpi0 + kMath;
    const bool early_tree = math_thread && prm.early_tree && prm.early_dt;
    if (!(kReplay && warp >= 6 && prm.early_replay) && !early_tree) pdl_wait();

    const uint32_t tmem = kScan ? __shfl_sync(0xffffffffu, *tmem_slot, 0) : 0u;
    const int Tp16 = (T + 15) & ~15;
    const int xbytes = T * 128;

    if (warp == 0) {
        // ================= TMA producer =================
        if (lane == 0) {
            const uint64_t pol_ef = policy_evict_first();
            const unsigned long long pdbg = trace ? trace[127] : 0ull;   // debug knob 8: no ramp
            if (kScan) {
                mbar_expect_tx(BAR_TREE, 3 * S::kCbAtoms * xbytes);
#pragma unroll 1
                for (int a = 0; a < S::kCbAtoms; ++a) {
                    tma_load_2d(sb + S::CB + 2 * a * kAtom, &tm_c, BAR_TREE, g * NS + 64 * a, b * T);
                    tma_load_2d(sb + S::CB + (2 * a + 1) * kAtom, &tm_c, BAR_TREE, g * NS + 64 * a, b * T);
                    tma_load_2d(sb + S::BB + a * kAtom, &tm_b, BAR_TREE, g * NS + 64 * a, b * T);
                }
                // the bulk state stream starts once the tree operands have landed: issued together, the
                // ~kStages x 40 KB per CTA would queue the small critical-path loads behind it
                if (!(pdbg & 8)) mbar_wait(BAR_TREE, 0);
            }
            for (int k = 0; k < nh; ++k) {
                const int s = k % kStages;
                const int h = hbeg + k;
                if (k < n_early) {   // state already in flight (arrived at issue)
                } else {
                    mbar_wait(bar_empty(s), ((k / kStages) & 1) ^ 1);
                    if (trace && k < 32) trace[128 + k] = gtimer();   // state load k issued (slot released)
                    mbar_expect_tx(bar_full(s), prm.has_h0 ? S::H0S : 0);
                    if (prm.has_h0)
#pragma unroll 1
                        for (int a = 0; a < NS / 32; ++a)
                            tma_load_2d_ef(sb + S::slot(s) + a * S::kSlotAtom, &tm_h0, bar_full(s), 32 * a,
                                           ((b * H) + h) * kP, pol_ef);
                }
                if (kScan && k < S::kStX0) {   // first x tiles; later ones are requested by the epilogue that frees the slot
                    mbar_expect_tx(bar_xfull(k), xbytes);
                    tma_load_2d_ef(sb + S::xslot(k), &tm_x, bar_xfull(k), h * kP, b * T, pol_ef);
                }
                // ramp: the rest of the ring is requested only once head 0 has landed, so every CTA's
                // first pair is near the front of the DRAM queue instead of behind other CTAs' later stages
                if (kScan && (k == 1 || nh == 1) && !(pdbg & 8)) mbar_wait(bar_full(0), 0);
            }
        }
    } else if (!kScan && warp <= 5) {
        // commit only: no tensor-core work, these warps idle
    } else if (warp == 1) {
        // ================= MMA issuer (whole warp converged, elected lane issues) =================
        {
            mbar_wait(BAR_TREE, 0);
            tc_fence_after();
            // G = C·Bᵀ (once per tree), kind::f16 bf16, M=128, N=Tp16, K=NS
            const uint32_t id_g = idesc(kFmtBF16, 0, 128, Tp16);
            // rows 64..127 of A are a copy of C, so G lands in TMEM lanes 0..63 and again in 64..127
#pragma unroll 1
            for (int kk = 0; kk < NS / 16; ++kk) {
                const uint32_t off = (kk & 3) * 32;
                mma_f16_w(tmem + 0, sdesc(sb + S::CB + (kk >> 2) * 2 * kAtom + off, 16, 1024),
                        sdesc(sb + S::BB + (kk >> 2) * kAtom + off, 16, 1024), id_g, kk > 0);
            }
            tc_commit_w(BAR_G);
            mbar_wait(BAR_CTF, 0);
            tc_fence_after();
            const uint32_t id_y0 = idesc(kFmtTF32, 0, 128, kP);
            const uint32_t id_y = idesc(kFmtBF16, 1, 128, kP);
            const int* mode = (const int*)(sm + S::MODE);
            int ndir = 0;
            const unsigned long long dbg = trace ? trace[127] : 0ull;   // debug: 1 skip Y0, 2 skip Y'
            const uint32_t id_y02 = idesc(kFmtTF32, 0, 128, 2 * kP);
            const bool pairs = !(dbg & 16);   // debug knob 16: one head per Y0 chain
            for (int k = 0; k < nh; k += (pairs ? 2 : 1)) {
                // heads k, k+1 (slots s, s+1 of one pair, accumulators ac, ac+1 adjacent in TMEM)
                const int s = k % kStages, ac = k % kAcc;
                const int nq = (pairs && k + 1 < nh) ? 2 : 1;
                for (int q = 0; q < nq; ++q) {
                    mbar_wait(bar_full(s + q), ((k + q) / kStages) & 1);
                    if (kReplay) mbar_wait(bar_upd(s + q), ((k + q) / kStages) & 1);   // replayed on chip
                }
                if (trace && lane == 0 && k < 12) trace[30 + k] = gtimer();
                for (int q = 0; q < nq; ++q) mbar_wait(bar_accempty(ac + q), (((k + q) / kAcc) & 1) ^ 1);
                tc_fence_after();
                if (trace && lane == 0 && k < 9) trace[118 + k] = gtimer();
                const uint32_t d0 = tmem + kAccCol0 + 64 * ac;
                if (prm.has_h0 && !(dbg & 1)) {
                    // Y0 = C·h0ᵀ of both heads in one N = 2 x 64 MMA chain, kind::tf32, A = C from TMEM,
                    // K = NS in steps of 8 (32 B / 8 columns)
                    // one base descriptor, per-step offsets are compile-time (address field is addr >> 4)
                    const uint64_t bd = sdesc(sb + S::slot(s), 16, 1024);
                    const uint32_t idy0 = nq == 2 ? id_y02 : id_y0;
#pragma unroll 2
                    for (int kk = 0; kk < NS / 8; ++kk)
                        mma_tf32_ts_w(d0, tmem + kCCol + 8 * kk,
                                    bd + (uint64_t)(((kk >> 2) * S::kSlotAtom + (kk & 3) * 32) >> 4), idy0, kk > 0);
                }
                for (int q = 0; q < nq; ++q) tc_commit_w(bar_empty(s + q));   // state tiles no longer needed
                if (trace && lane == 0 && k < 9) trace[100 + k] = gtimer();
                if (trace && (dbg & 128) && k < 9) {   // debug knob 128: wait for Y0 to complete (timing)
                    tc_commit_w(bar0 + (S::NBAR - 1) * 8);
                    mbar_wait(bar0 + (S::NBAR - 1) * 8, (k >> 1) & 1);
                    if (lane == 0) trace[180 + k] = gtimer();
                }
                for (int q = 0; q < nq; ++q) {
                    const int kq = k + q, a = kq & 1;
                    const int sx = kq % S::kStX;
                    mbar_wait(bar_xfull(sx), (kq / S::kStX) & 1);
                    mbar_wait(bar_mfull(a), (kq >> 1) & 1);
                    if (trace && lane == 0 && kq < 9) trace[109 + kq] = gtimer();
                    tc_fence_after();
                    // Y' = M'·X_h, kind::f16, A K-major (masked weights), B MN-major (x rows j).  Factorised
                    // decay: accumulated onto Y0 (M' carries e^{-Λ_j}, the epilogue e^{Λ_i}); direct decay:
                    // into the separate columns kDirCol, once the epilogue has read the previous direct head's
                    const bool fac = mode[kq] != 0;
                    uint32_t dy = d0 + 64 * q, acc0 = prm.has_h0 ? 1u : 0u;
                    if (!fac) {
                        mbar_wait(BAR_DIRE, (ndir & 1) ^ 1);
                        tc_fence_after();
                        ++ndir;
                        dy = tmem + kDirCol;
                        acc0 = 0;
                    }
                    const uint64_t ad = sdesc(sb + S::MB + (a ^ 1) * kAtom, 16, 1024);   // (see mrow)
                    const uint64_t xd = sdesc(sb + S::xslot(sx), kAtom, 1024);
                    const int nk = (dbg & 2) ? 0 : Tp16 / 16;
#pragma unroll
                    for (int kk = 0; kk < kT / 16; ++kk)
                        if (kk < nk)
                            mma_f16_w(dy, ad + (uint64_t)(kk * 2), xd + (uint64_t)(kk * 128), id_y, (kk > 0) | acc0);
                    if (trace && (dbg & 256) && kq < 9) {   // debug knob 256: wait for Y' to complete (timing)
                        tc_commit_w(bar0 + (S::NBAR - 1) * 8);
                        mbar_wait(bar0 + (S::NBAR - 1) * 8, kq & 1);
                        if (lane == 0) trace[190 + kq] = gtimer();
                    }
                    tc_commit_w(bar_accfull(ac + q));
                    tc_commit_w(bar_mempty(a));
                }
            }
        }
    } else if (kReplay && warp == 10) {
        // fused: committed state in place (tm_h0); commit only: into h_new (tm_y)
        if (lane == 0) state_storer<NS, kReplay>(prm, sm, sb, kScan ? &tm_h0 : &tm_y, b, hbeg, nh, bar0,
                                                 chunk == 0 && g == 0);
    } else if (kReplay && warp >= 6) {
        replay_updater<NS, kReplay>(prm, sm, sb, &tm_h0, b, g, chunk, hbeg, nh, bar0);
    } else {
        // ================= epilogue / math warps (kMath threads) =================
        const int e = tid - kEpi0;
        const int quad = warp & 3;           // TMEM lane quadrant of this warp
        const int row = quad * 32 + lane;    // tree node owned in TMEM-based work
        const int half = kSplit ? ((warp - 2) >> 2) : 0;   // column half of a split warp pair
        uint64_t* rows = (uint64_t*)(sm + S::ROWS);
        float* lam = (float*)(sm + S::LAM);
        float* cj = (float*)(sm + S::CJ);
        float* e0 = (float*)(sm + S::E0);
        int* mode = (int*)(sm + S::MODE);
        // ---- per-CTA inputs: epilogue warp ew owns heads ew, ew+4, ew+8; lane owns nodes lane, lane+32.
        //      The producer issues the tree operands right after the wait; tree validation runs in the
        //      epilogue warps (an invalid tree yields y = 0), so nothing waits on it ----
        constexpr int kHPW = (kHPC + kMathW - 1) / kMathW;   // heads per math warp
        float dtr[kHPW][2], a_h[kHPW], d_h[kHPW];
        int* sbad = (int*)(sm + S::BADF);
        if (kScan && tid >= kEpi0 && tid < kEpi0 + kMath) {
            const int ew = (tid - kEpi0) >> 5, e = tid - kEpi0;
            if (e < T) sp[e] = prm.parent[(size_t)b * T + e];
#pragma unroll
            for (int q = 0; q < kHPW; ++q) {
                const int hh = ew + kMathW * q;
                const bool hv = hh < nh;
                a_h[q] = hv ? prm.A[hbeg + hh] : 0.f;
                d_h[q] = (hv && prm.D) ? prm.D[hbeg + hh] : 0.f;
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    const int i = lane + 32 * hf;
                    dtr[q][hf] = (hv && i < T) ? dt_eff(prm.dtx, prm.dt[((size_t)b * T + i) * H + hbeg + hh], hbeg + hh) : 0.f;
                }
            }
            if (e == 0) *sbad = 0;
            named_bar(1, kMath);
            if (e < T) {   // PAPER.md:90 precondition: parent[0] = -1, 0 <= parent[i] < i
                const int p = sp[e];
                const int code = (e == 0) ? (p != -1 ? 1 : 0) : ((p < 0 || p >= e) ? 2 : 0);
                if (code) atomicMax(sbad, code == 1 ? 2 : 1);   // root error takes precedence
            }
            named_bar(1, kMath);
            if (*sbad) {
                // invalid tree: make the pointer chains harmless; the output stage writes zeros
                if (e < T) sp[e] = (e == 0) ? -1 : 0;
                if (e == 0 && chunk == 0 && g == 0 && !early_tree) report(prm.dev_status, *sbad == 2 ? 1 : 2);
            }
            named_bar(1, kMath);
        }
        int rounds = 0;
        while ((1 << rounds) < T) ++rounds;
        const int ew = warp - 2;
        // ---- ancestor rows L[i] and tree segsum Λ = L·(dt A_h) by pointer jumping in registers
        //      (PAPER.md:63-66, 86-90): lane holds nodes lane and lane+32; after round r a node's
        //      row holds its ancestors at distance < 2^r and jp is its 2^r-th ancestor ----
        uint64_t rw[2];
        int jp[2];
        float lm[kHPW][2];
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            const int i = lane + 32 * hf;
            rw[hf] = (i < T) ? (1ull << i) : 0ull;
            jp[hf] = (i < T) ? sp[i] : -1;
#pragma unroll
            for (int q = 0; q < kHPW; ++q) lm[q][hf] = dtr[q][hf] * a_h[q];
        }
#pragma unroll 1
        for (int r = 0; r < rounds; ++r) {
            uint64_t nrw[2];
            int njp[2];
            float nlm[kHPW][2];
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                const int j = jp[hf];
                const int sl = (j >= 0) ? (j & 31) : lane;
                const bool hi = j >= 32;
                const uint64_t r0 = __shfl_sync(0xffffffffu, rw[0], sl), r1 = __shfl_sync(0xffffffffu, rw[1], sl);
                const int j0 = __shfl_sync(0xffffffffu, jp[0], sl), j1 = __shfl_sync(0xffffffffu, jp[1], sl);
                nrw[hf] = rw[hf] | ((j >= 0) ? (hi ? r1 : r0) : 0ull);
                njp[hf] = (j >= 0) ? (hi ? j1 : j0) : -1;
#pragma unroll
                for (int q = 0; q < kHPW; ++q) {
                    const float v0 = __shfl_sync(0xffffffffu, lm[q][0], sl), v1 = __shfl_sync(0xffffffffu, lm[q][1], sl);
                    nlm[q][hf] = lm[q][hf] + ((j >= 0) ? (hi ? v1 : v0) : 0.f);
                }
            }
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                rw[hf] = nrw[hf];
                jp[hf] = njp[hf];
#pragma unroll
                for (int q = 0; q < kHPW; ++q) lm[q][hf] = nlm[q][hf];
            }
        }
        if (ew == 0) {
#pragma unroll
            for (int hf = 0; hf < 2; ++hf)
                if (lane + 32 * hf < T) rows[lane + 32 * hf] = rw[hf];
        }
        // ---- per-head decay mode and coefficients (warp-local) ----
#pragma unroll
        for (int q = 0; q < kHPW; ++q) {
            const int hh = ew + kMathW * q;
            if (hh < nh) {   // warp-uniform
                float mn = fminf(lm[q][0], lm[q][1]);
#pragma unroll
                for (int o = 16; o; o >>= 1) mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
                const bool f = mn >= -64.f;       // factorised decay e^{Λi-Λj} = e^{Λi}·e^{-Λj}
                if (lane == 0) {
                    mode[hh] = f ? 1 : 0;
                    ((float*)(sm + S::DS))[hh] = d_h[q];
                }
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    const int i = lane + 32 * hf;
                    if (i < T) {
                        const float l = lm[q][hf];
                        lam[hh * 64 + i] = l;
                        cj[hh * 64 + i] = f ? __expf(-l) * dtr[q][hf] : dtr[q][hf];
                        e0[hh * 64 + i] = __expf(l);
                    }
                }
            }
        }
        named_bar(1, kMath);
        if (early_tree) {
            pdl_wait();   // every global write follows the dependency wait
            if (*sbad && e == 0 && chunk == 0 && g == 0) report(prm.dev_status, *sbad == 2 ? 1 : 2);
        }
        // ---- C (bf16, TMA) -> tf32 operand tile; zero the padded x rows ----
        if (trace && e == 0) trace[1] = gtimer();
        mbar_wait(BAR_TREE, 0);
        if (trace && e == 0) trace[2] = gtimer();
        if (quad < 2) {
            // C row (bf16, swizzled TMA tile) -> fp32 -> TMEM lane = row, columns [kCCol, kCCol + NS)
            const int i = row;
            constexpr int kC32 = NS / 32 / (kSplit ? 2 : 1);
#pragma unroll
            for (int cq = 0; cq < kC32; ++cq) {
                const int c32 = half * kC32 + cq;
                uint32_t f[32];
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    const int c = 4 * c32 + cc, a = c >> 3;   // 16-byte bf16 chunk index along the row
                    uint4 v = make_uint4(0, 0, 0, 0);
                    if (i < T) v = *reinterpret_cast<const uint4*>(sm + S::CB + 2 * a * kAtom + swz(i, c & 7));
                    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        f[8 * cc + 2 * q] = w[q] << 16;
                        f[8 * cc + 2 * q + 1] = w[q] & 0xFFFF0000u;
                    }
                }
                tmem_st32(tmem + ((uint32_t)(quad * 32) << 16) + kCCol + 32 * c32, f);
            }
            tmem_st_wait();
            tc_fence_before();
        } else {
            const int zi = (quad - 2) * 32 + lane + half * 64;   // 0 .. kMath/2 - 1
#pragma unroll 1
            for (int k = zi; k < S::kStX0 * (Tp16 - T) * 8; k += kMath / 2) {
                const int s = k / ((Tp16 - T) * 8), rr = T + (k / 8) % (Tp16 - T), c = k & 7;
                *reinterpret_cast<uint4*>(sm + S::X + s * S::XS + swz(rr, c)) = make_uint4(0, 0, 0, 0);
            }
        }
        fence_proxy_async();
        mbar_arrive(BAR_CTF);
        if (trace && e == 0) trace[46] = gtimer();

        if (trace && e == 0) trace[50] = gtimer();
        // ---- builder warps 2,3 (TMEM lanes 64..127 hold a copy of G) build the masked weights of head
        //      k+1 while warps 4,5 (TMEM lanes 0..63) run the epilogue of head k ----
        mbar_wait(BAR_G, 0);
        tc_fence_after();
        if (trace && e == 0) trace[51] = gtimer();
        const bool builder = quad >= 2;
        if (trace && e == 0) trace[3] = gtimer();
        if (builder) {
            const int brow = (quad - 2) * 32 + lane;
            const bool bown = brow < T;
            const uint64_t mybits = bown ? rows[brow] : 0ull;
            const uint32_t gl = tmem + ((uint32_t)(quad * 32) << 16);   // G row brow, columns 0..63
#pragma unroll 1
            for (int k = 0; k < nh; ++k) {
                // masked weights of head k into M'[k & 1]:  M'_ij = L_ij G_ij c_j  (factorised)
                //                                        or  L_ij e^{Λi-Λj} dt_j G_ij (direct)
                const int a = k & 1;
                mbar_wait(bar_mempty(a), ((k >> 1) & 1) ^ 1);
                const float* c = cj + k * 64;
                const float* lk = lam + k * 64;
                const bool f = mode[k] != 0;
                const float li = bown ? lk[brow] : 0.f;
                // M'[a] lives at MB + (a^1)·kAtom: M'[0] (heads 0, 2, ..) over the C copy, which only the G MMA
                // reads (done at BAR_G); M'[1] over C atom 0, which the C -> tf32 converters read (BAR_CTF)
                if (k == 1) mbar_wait(BAR_CTF, 0);
                unsigned char* mrow = sm + S::MB + (a ^ 1) * kAtom;
                // split builders: half 0 takes columns j < 32, half 1 the rest
                const int c16b = kSplit ? 2 * half : 0, c16e = kSplit ? min(Tp16 / 16, 2 * half + 2) : Tp16 / 16;
#pragma unroll 1
                for (int c16 = c16b; c16 < c16e; ++c16) {
                    float g16[16];
                    tmem_ld16(gl + 16 * c16, g16);
                    uint32_t o[8];
#pragma unroll
                    for (int q = 0; q < 16; q += 2) {
                        const int j = 16 * c16 + q;
                        float v0 = c[j] * g16[q], v1 = c[j + 1] * g16[q + 1];
                        if (!f) {
                            v0 *= __expf(fminf(li - lk[j], 0.f));
                            v1 *= __expf(fminf(li - lk[j + 1], 0.f));
                        }
                        o[q >> 1] = pack_bf16(((mybits >> j) & 1ull) ? v0 : 0.f, ((mybits >> (j + 1)) & 1ull) ? v1 : 0.f);
                    }
                    if (bown) {
                        *reinterpret_cast<uint4*>(mrow + swz(brow, 2 * c16)) = make_uint4(o[0], o[1], o[2], o[3]);
                        *reinterpret_cast<uint4*>(mrow + swz(brow, 2 * c16 + 1)) = make_uint4(o[4], o[5], o[6], o[7]);
                    }
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar_mfull(a));
                if (trace && warp == 2 && lane == 0 && k < 9) trace[91 + k] = gtimer();
            }
        } else {
            // ---- TMEM epilogue (warps 4,5 = TMEM lanes 0..63 = tree nodes) ----
            const bool own = row < T;
            const bool leader = (warp == 4 && lane == 0);
            if (S::kXB > 0 && nh > S::kStX0) {
                // G is done, so the B tile region holds the last x slots: zero their padded rows, then
                // request their first tiles
                const int e2 = quad * 32 + lane + half * 64;   // 0 .. kEpiT - 1
#pragma unroll 1
                for (int q = e2; q < S::kXB * (Tp16 - T) * 8; q += kEpiT) {
                    const int sx = S::kStX0 + q / ((Tp16 - T) * 8), rr = T + (q / 8) % (Tp16 - T), c = q & 7;
                    *reinterpret_cast<uint4*>(sm + S::xslot(sx) + swz(rr, c)) = make_uint4(0, 0, 0, 0);
                }
                fence_proxy_async();
                named_bar(2, kEpiT);
                if (leader)
                    for (int k = S::kStX0; k < S::kStX && k < nh; ++k) {
                        mbar_expect_tx(bar_xfull(k), xbytes);
                        tma_load_2d_ef(sb + S::xslot(k), &tm_x, bar_xfull(k), (hbeg + k) * kP, b * T, policy_evict_first());
                    }
            }
            // k = -1 is a dry pass while the first accumulator is still far away: it runs the epilogue code
            // once on garbage (TMEM columns of accumulator kAcc-1, x slot 0, y staging 1; nothing is stored
            // or signalled), so head 0 does not pay the instruction-cache misses of its first execution
            const int kfirst = (trace && (trace[127] & 32)) ? 0 : -1;   // debug knob 32: no dry pass
            for (int k = kfirst; k < nh; ++k) {
                const bool dry = k < 0;
                const int kd = dry ? 0 : k;
                const int a = dry ? 1 : (k & 1), ac = dry ? kAcc - 1 : k % kAcc;
                const int h = hbeg + kd;
                if (!dry) {
                    mbar_wait(bar_accfull(ac), (k / kAcc) & 1);
                    tc_fence_after();
                    if (trace && leader && k < 12) trace[4 + 2 * k] = gtimer();
                    if (leader) bulk_wait_read1();      // y staging [a] free (store of head k-2 has read it)
                }
                if (trace && leader && dry) trace[170] = gtimer();
                named_bar(2, kEpiT);
                if (trace && leader && !dry && k < 6) trace[52 + 2 * k] = gtimer();
                const bool zero_out = *sbad != 0;
                const float Dh = zero_out ? 0.f : ((const float*)(sm + S::DS))[kd];
                const bool fac = mode[kd] != 0;
                const bool has0 = prm.has_h0 || fac;    // accumulator written (Y0 and / or Y')
                const float s0 = (own && !zero_out) ? e0[kd * 64 + row] : 0.f;
                const int sx = kd % S::kStX;
                const unsigned char* xr = sm + S::xslot(sx);
                unsigned char* yr = sm + S::YS + a * kAtom;
                const uint32_t tq = tmem + ((uint32_t)(quad * 32) << 16);
                const uint32_t tl = tq + kAccCol0 + 64 * ac;
                // the warp's 32-column chunks (both, or its half when split) requested up front, then computed
                constexpr int kNC = kSplit ? 1 : 2;
                const int cb = kSplit ? half : 0;
                uint32_t v0[kNC][32], v1[kNC][32];
#pragma unroll
                for (int cc = 0; cc < kNC; ++cc) {
                    if (has0) tmem_ld32(tl + 32 * (cb + cc), v0[cc]);
                    if (!fac) tmem_ld32(tq + kDirCol + 32 * (cb + cc), v1[cc]);
                }
                tmem_wait();
                if (trace && leader && !dry && k < 6) trace[160 + k] = gtimer();
#pragma unroll
                for (int cc = 0; cc < kNC; ++cc) {
                    const int c = cb + cc;
                    if (!has0) {
#pragma unroll
                        for (int q = 0; q < 32; ++q) v0[cc][q] = 0u;
                    }
                    if (fac) {
#pragma unroll
                        for (int q = 0; q < 32; ++q) v1[cc][q] = 0u;
                    }
                    if (own) {
#pragma unroll
                        for (int qc = 0; qc < 4; ++qc) {
                            const int ch = 4 * c + qc;
                            const uint4 xv = *reinterpret_cast<const uint4*>(xr + swz(row, ch));
                            const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
                            float dpc[8];   // D[h][p] of this chunk's 8 columns (d_pc), else D_h
#pragma unroll
                            for (int q = 0; q < 8; ++q) dpc[q] = Dh;
                            if (DPC && prm.D && !zero_out) {
                                const float4* dr = reinterpret_cast<const float4*>(prm.D + (size_t)h * kP + 8 * ch);
                                const float4 d0 = __ldg(dr), d1 = __ldg(dr + 1);
                                dpc[0] = d0.x; dpc[1] = d0.y; dpc[2] = d0.z; dpc[3] = d0.w;
                                dpc[4] = d1.x; dpc[5] = d1.y; dpc[6] = d1.z; dpc[7] = d1.w;
                            }
                            uint32_t o[4];
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const float xa = __uint_as_float(xw[q] << 16), xb = __uint_as_float(xw[q] & 0xFFFF0000u);
                                const int p = 8 * qc + 2 * q;
                                const float ya = fmaf(s0, __uint_as_float(v0[cc][p]), fmaf(dpc[2 * q], xa, __uint_as_float(v1[cc][p])));
                                const float yb = fmaf(s0, __uint_as_float(v0[cc][p + 1]),
                                                      fmaf(dpc[2 * q + 1], xb, __uint_as_float(v1[cc][p + 1])));
                                o[q] = zero_out ? 0u : pack_bf16(ya, yb);
                            }
                            *reinterpret_cast<uint4*>(yr + swz(row, ch)) = make_uint4(o[0], o[1], o[2], o[3]);
                        }
                    }
                }
                if (trace && leader && !dry && k < 6) trace[53 + 2 * k] = gtimer();
                if (trace && leader && dry) trace[171] = gtimer();
                if (dry) continue;
                tc_fence_before();
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(bar_accempty(ac));
                    if (!fac) mbar_arrive(BAR_DIRE);
                }
                named_bar(2, kEpiT);
                if (leader) {
                    if constexpr (kPeers) {   // head-sharded layer: this tile into every rank's full y
#pragma unroll 1
                        for (int pr = 0; pr < prm.n_ypeer; ++pr)
                            tma_store_2d_ef(&ym.m[pr], sb + S::YS + a * kAtom, (prm.y_head_off + h) * kP, b * T,
                                            policy_evict_first());
                    } else {
                        tma_store_2d_ef(&tm_y, sb + S::YS + a * kAtom, h * kP, b * T, policy_evict_first());
                    }
                    bulk_commit();
                    // x slot free (Y' read it before accfull, the epilogue above): refill it with head k + kStX,
                    // so the x stream never waits in the state producer's queue
                    if (k + S::kStX < nh) {
                        mbar_expect_tx(bar_xfull(sx), xbytes);
                        tma_load_2d_ef(sb + S::xslot(sx), &tm_x, bar_xfull(sx), (h + S::kStX) * kP, b * T,
                                       policy_evict_first());
                    }
                    if (trace && k < 12) trace[5 + 2 * k] = gtimer();
                }
            }
            if (leader) bulk_wait_read_all();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (trace && tid == 0) trace[45] = gtimer();
    if (kScan && warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

}  // namespace tc
}  // namespace stree

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

bool make_map(CUtensorMap* m, CUtensorMapDataType dt, const void* base, uint64_t inner, uint64_t outer,
              uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer) {
    return stree::host::tmap_2d(m, dt, base, inner, outer, row_bytes, box_inner, box_outer);
}

unsigned long long* g_trace = nullptr;
int g_trace_ring = 0, g_trace_n = 0;   // ring mode: launch i writes slot i % g_trace_ring (1024 CTAs each)
unsigned long long* trace_slot() {
    if (!g_trace || !g_trace_ring) return g_trace;
    return g_trace + (size_t)(g_trace_n++ % g_trace_ring) * 1024 * stree::tc::kTraceWords;
}

int num_sms() { return stree::host::num_sms(); }

}  // namespace

// Debug hook (not part of the ABI): per-CTA globaltimer phase stamps, 64 u64 per CTA.
extern "C" void stree_debug_tc_trace(unsigned long long* dev_buf) {
    g_trace = dev_buf;
    g_trace_ring = 0;
}
// ring mode: launch i writes its stamps to dev_buf + (i % n) * 1024 * 256 (tools/trace_stack.py)
extern "C" void stree_debug_tc_trace_ring(unsigned long long* dev_buf, int n) {
    g_trace = dev_buf;
    g_trace_ring = n;
    g_trace_n = 0;
}

extern "C" int stree_tc_supports(const stree_dims* d) {
    if (!d) return 0;
    if (d->io_dtype != STREE_BF16) return 0;
    if (d->head_dim != stree::tc::kP) return 0;
    if (d->d_state != 64 && d->d_state != 128) return 0;
    if (d->n_nodes < 1 || d->n_nodes > stree::tc::kT) return 0;
    if (d->n_groups < 1 || d->n_heads % d->n_groups) return 0;
    return 1;
}

namespace {

template <int NS, int MODE, typename YM = stree::tc::NoYPeers, bool DPC = false>
cudaError_t launch_tc_inst(dim3 grid, cudaStream_t s, const CUtensorMap& mc, const CUtensorMap& mb,
                           const CUtensorMap& mx, const CUtensorMap& mh, const CUtensorMap& my,
                           const stree::tc::Params& prm, const YM& ym = YM{}) {
    using namespace stree::tc;
    auto k = scan_tc_kernel<NS, MODE, YM, DPC>;
    const size_t smem = Smem<NS, (MODE >= 1)>::TOTAL + 1024;
    cudaError_t e = stree::host::smem_attr((const void*)k, (int)smem);
    if (e != cudaSuccess) return e;
    return stree::launch_k(k, grid, dim3(MODE ? kThreadsReplay : kThreadsScan), smem, s, mc, mb, mx, mh, my, ym, prm);
}

// work split: one tree per CTA, heads of one group in chunks, ~1 wave over the SMs
void split_heads(int B, int H, int G, int* cpg_out, int* hpc_out) {
    using namespace stree::tc;
    const int hpg = H / G;
    int cpg = num_sms() / (B * G);                  // head chunks per group: at most one wave of CTAs
    if (cpg < 1) cpg = 1;
    if (cpg > hpg) cpg = hpg;
    int hpc = (hpg + cpg - 1) / cpg;
    if (hpc > kHPC) hpc = kHPC;
    *cpg_out = (hpg + hpc - 1) / hpc;
    *hpc_out = hpc;
}

// shared by the scan-only and the fused replay+scan launches
int launch_tc(const stree_dims* d, const void* x, const float* dt, const float* A, const void* Bm, const void* Cm,
              const float* D, const float* h0, const int32_t* parent, void* y, int32_t* dev_status, cudaStream_t s,
              bool replay, const stree::tc::Params* rp, const stree_yout* yo = nullptr) {
    using namespace stree::tc;
    if (!stree_tc_supports(d)) return (int)cudaErrorNotSupported;
    const int B = d->batch, T = d->n_nodes, H = d->n_heads, P = d->head_dim, N = d->d_state, G = d->n_groups;
    CUtensorMap mc, mb, mx, mh, my;
    const uint64_t BT = (uint64_t)B * T;
    bool ok = make_map(&mc, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, Cm, (uint64_t)G * N, BT, (uint64_t)G * N * 2, 64, T) &&
              make_map(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, Bm, (uint64_t)G * N, BT, (uint64_t)G * N * 2, 64, T) &&
              make_map(&mx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, x, (uint64_t)H * P, BT, (uint64_t)H * P * 2, 64, T) &&
              (yo || make_map(&my, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, y, (uint64_t)H * P, BT, (uint64_t)H * P * 2, 64, T));
    YPeerMaps ym;
    if (yo) {   // one map per peer's full y [B·T][heads_total·P], box = one head x T rows
        const uint64_t HtP = (uint64_t)yo->heads_total * P;
        for (int p = 0; p < yo->n_peers && ok; ++p)
            ok = make_map(&ym.m[p], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, yo->peers[p], HtP, BT, HtP * 2, 64, T);
        my = ym.m[0];
    }
    if (h0)
        ok = ok && make_map(&mh, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, h0, (uint64_t)N, (uint64_t)B * H * P,
                            (uint64_t)N * 4, 32, 64);
    else
        mh = mx;  // unused
    if (!ok) return (int)cudaErrorInvalidValue;
    int cpg, hpc;
    split_heads(B, H, G, &cpg, &hpc);
    stree::tc::Params prm{};
    if (rp) prm = *rp;
    prm.trace = trace_slot();
    prm.B = B; prm.T = T; prm.H = H; prm.G = G; prm.cpg = cpg; prm.hpc = hpc;
    prm.dt = dt; prm.A = A; prm.D = D; prm.parent = parent; prm.y = (__nv_bfloat16*)y; prm.dev_status = dev_status;
    prm.has_h0 = h0 != nullptr;
    prm.early_state = (stree_launch_flags_get() & STREE_LAUNCH_EARLY_STATE) ? 1 : 0;
    prm.early_replay = (stree_launch_flags_get() & STREE_LAUNCH_EARLY_REPLAY) ? 1 : 0;
    prm.early_tree = (stree_launch_flags_get() & STREE_LAUNCH_EARLY_TREE) ? 1 : 0;
    prm.early_dt = (stree_launch_flags_get() & STREE_LAUNCH_EARLY_DT) ? 1 : 0;
    prm.dtx = stree::DtX::from(stree_scan_opts_get());
    prm.d_pc = (stree_scan_opts_get() && stree_scan_opts_get()->d_per_channel) ? 1 : 0;
    dim3 grid(B * G * cpg);
    cudaError_t e;
    if (yo && prm.d_pc) return (int)cudaErrorNotSupported;   // sharded calls take no scan options
    if (yo) {
        prm.n_ypeer = yo->n_peers;
        prm.y_head_off = yo->head_offset;
        if (N == 128)
            e = replay ? launch_tc_inst<128, 1>(grid, s, mc, mb, mx, mh, my, prm, ym)
                       : launch_tc_inst<128, 0>(grid, s, mc, mb, mx, mh, my, prm, ym);
        else
            e = replay ? launch_tc_inst<64, 1>(grid, s, mc, mb, mx, mh, my, prm, ym)
                       : launch_tc_inst<64, 0>(grid, s, mc, mb, mx, mh, my, prm, ym);
    } else if (N == 128)
        e = prm.d_pc ? (replay ? launch_tc_inst<128, 1, NoYPeers, true>(grid, s, mc, mb, mx, mh, my, prm)
                               : launch_tc_inst<128, 0, NoYPeers, true>(grid, s, mc, mb, mx, mh, my, prm))
                     : (replay ? launch_tc_inst<128, 1>(grid, s, mc, mb, mx, mh, my, prm)
                               : launch_tc_inst<128, 0>(grid, s, mc, mb, mx, mh, my, prm));
    else
        e = prm.d_pc ? (replay ? launch_tc_inst<64, 1, NoYPeers, true>(grid, s, mc, mb, mx, mh, my, prm)
                               : launch_tc_inst<64, 0, NoYPeers, true>(grid, s, mc, mb, mx, mh, my, prm))
                     : (replay ? launch_tc_inst<64, 1>(grid, s, mc, mb, mx, mh, my, prm)
                               : launch_tc_inst<64, 0>(grid, s, mc, mb, mx, mh, my, prm));
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
}

}  // namespace

extern "C" int stree_launch_scan_tc(const stree_dims* d, const void* x, const float* dt, const float* A,
                                    const void* Bm, const void* Cm, const float* D, const float* h0,
                                    const int32_t* parent, void* y, int32_t* dev_status, cudaStream_t s) {
    return launch_tc(d, x, dt, A, Bm, Cm, D, h0, parent, y, dev_status, s, false, nullptr);
}

// fused replay + scan; h is read (pre-commit state) and written (committed state) in place
extern "C" int stree_launch_replay_scan_tc(const stree_dims* d_prev, const void* x_prev, const float* dt_prev,
                                           const void* Bm_prev, const int32_t* parent_prev, const int32_t* path,
                                           const int32_t* path_len, const stree_dims* d, const void* x,
                                           const float* dt, const float* A, const void* Bm, const void* Cm,
                                           const float* D, float* h, const int32_t* parent, void* y,
                                           int32_t* dev_status, cudaStream_t s) {
    stree::tc::Params rp{};
    rp.Tp = d_prev->n_nodes;
    rp.x_prev = (const __nv_bfloat16*)x_prev;
    rp.dt_prev = dt_prev;
    rp.b_prev = (const __nv_bfloat16*)Bm_prev;
    rp.parent_prev = parent_prev;
    rp.path = path;
    rp.path_len = path_len;
    return launch_tc(d, x, dt, A, Bm, Cm, D, h, parent, y, dev_status, s, true, &rp);
}

extern "C" int stree_launch_scan_tc_sharded(const stree_dims* d, const void* x, const float* dt, const float* A,
                                            const void* Bm, const void* Cm, const float* D, const float* h0,
                                            const int32_t* parent, const stree_yout* yo, int32_t* dev_status,
                                            cudaStream_t s) {
    return launch_tc(d, x, dt, A, Bm, Cm, D, h0, parent, nullptr, dev_status, s, false, nullptr, yo);
}

extern "C" int stree_launch_replay_scan_tc_sharded(const stree_dims* d_prev, const void* x_prev, const float* dt_prev,
                                                   const void* Bm_prev, const int32_t* parent_prev,
                                                   const int32_t* path, const int32_t* path_len, const stree_dims* d,
                                                   const void* x, const float* dt, const float* A, const void* Bm,
                                                   const void* Cm, const float* D, float* h, const int32_t* parent,
                                                   const stree_yout* yo, int32_t* dev_status, cudaStream_t s) {
    stree::tc::Params rp{};
    rp.Tp = d_prev->n_nodes;
    rp.x_prev = (const __nv_bfloat16*)x_prev;
    rp.dt_prev = dt_prev;
    rp.b_prev = (const __nv_bfloat16*)Bm_prev;
    rp.parent_prev = parent_prev;
    rp.path = path;
    rp.path_len = path_len;
    return launch_tc(d, x, dt, A, Bm, Cm, D, h, parent, nullptr, dev_status, s, true, &rp, yo);
}

// stree_commit on the same pipeline (MODE 2): bf16 activations, P = 64, N in {64, 128}, any T <= 256,
// h0 given.  h_new may alias h0 (in place) or be a distinct buffer.
extern "C" int stree_tc_commit_supports(const stree_dims* d) {
    if (!d) return 0;
    if (d->io_dtype != STREE_BF16 || d->head_dim != stree::tc::kP) return 0;
    if (d->d_state != 64 && d->d_state != 128) return 0;
    if (d->n_nodes < 1 || d->n_nodes > stree::kMaxNodes) return 0;
    if (d->n_groups < 1 || d->n_heads % d->n_groups) return 0;
    return 1;
}

extern "C" int stree_launch_commit_tc(const stree_dims* d, const void* x, const float* dt, const float* A,
                                      const void* Bm, const float* h0, const int32_t* parent, const int32_t* path,
                                      const int32_t* path_len, float* h_new, int32_t* dev_status, cudaStream_t s) {
    using namespace stree::tc;
    if (!stree_tc_commit_supports(d) || !h0) return (int)cudaErrorNotSupported;
    const int B = d->batch, H = d->n_heads, P = d->head_dim, N = d->d_state, G = d->n_groups;
    CUtensorMap mh, mo;
    bool ok = make_map(&mh, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, h0, (uint64_t)N, (uint64_t)B * H * P, (uint64_t)N * 4, 32, 64) &&
              make_map(&mo, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, h_new, (uint64_t)N, (uint64_t)B * H * P, (uint64_t)N * 4, 32,
                       64);
    if (!ok) return (int)cudaErrorInvalidValue;
    int cpg, hpc;
    split_heads(B, H, G, &cpg, &hpc);
    Params prm{};
    prm.trace = trace_slot();
    prm.B = B; prm.T = d->n_nodes; prm.H = H; prm.G = G; prm.cpg = cpg; prm.hpc = hpc;
    prm.A = A; prm.dev_status = dev_status;
    prm.has_h0 = 1;
    prm.early_state = (stree_launch_flags_get() & STREE_LAUNCH_EARLY_STATE) ? 1 : 0;
    prm.early_replay = (stree_launch_flags_get() & STREE_LAUNCH_EARLY_REPLAY) ? 1 : 0;
    prm.store_always = h_new != h0;
    prm.dtx = stree::DtX::from(stree_scan_opts_get());
    prm.Tp = d->n_nodes;
    prm.x_prev = (const __nv_bfloat16*)x;
    prm.dt_prev = dt;
    prm.b_prev = (const __nv_bfloat16*)Bm;
    prm.parent_prev = parent;
    prm.path = path;
    prm.path_len = path_len;
    dim3 grid(B * G * cpg);
    cudaError_t e = N == 128 ? launch_tc_inst<128, 2>(grid, s, mh, mh, mh, mh, mo, prm)
                             : launch_tc_inst<64, 2>(grid, s, mh, mh, mh, mh, mo, prm);
    if (e != cudaSuccess) return (int)e;
    return (int)cudaGetLastError();
}
