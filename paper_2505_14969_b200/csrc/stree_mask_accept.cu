// K1 stree_build_mask and K3 stree_accept kernels.
//
// K1: one CTA per tree; parent[] -> smem, validation + pointer-jumping mask
//     build (stree_common.cuh), then coalesced row/depth stores.  Latency-bound
//     (< 70 KB moved even at B=16, T=256): it runs once per verify iteration
//     and its mask is shared by every layer.
// K3: one warp per tree; the greedy walk of PAPER.md:309 with the lowest-index
//     matching child found by __ballot_sync over 32 candidates at a time.
#include "stree_common.cuh"

namespace stree {

__global__ void __launch_bounds__(256) build_mask_kernel(const int32_t* __restrict__ parent, int T,
                                                         uint32_t* __restrict__ mask,
                                                         int32_t* __restrict__ depth,
                                                         int32_t* dev_status) {
    __shared__ int sp[kMaxNodes], jmp[kMaxNodes], jmp2[kMaxNodes];
    __shared__ uint32_t rows[kMaxNodes * kMaxWords], rows2[kMaxNodes * kMaxWords];
    const int b = blockIdx.x, W = (T + 31) >> 5;
    pdl_wait();
    for (int i = threadIdx.x; i < T; i += blockDim.x) sp[i] = parent[(size_t)b * T + i];
    __syncthreads();
    int code = build_tree_rows(sp, T, W, rows, rows2, jmp, jmp2);
    if (code && threadIdx.x == 0) report(dev_status, code);
    uint32_t* out = mask + (size_t)b * T * W;
    for (int k = threadIdx.x; k < T * W; k += blockDim.x) out[k] = rows[k];
    if (depth) {
        for (int i = threadIdx.x; i < T; i += blockDim.x) {
            int c = 0;
            for (int w = 0; w < W; ++w) c += __popc(rows[i * W + w]);
            depth[(size_t)b * T + i] = code ? 0 : c - 1;
        }
    }
}

// One warp per tree, 4 trees per 128-thread CTA.
__global__ void __launch_bounds__(128) accept_kernel(const int32_t* __restrict__ tokens,
                                                     const int32_t* __restrict__ parent,
                                                     const int32_t* __restrict__ vtok, int B, int T,
                                                     int32_t* __restrict__ path,
                                                     int32_t* __restrict__ path_len,
                                                     int32_t* __restrict__ bonus, int32_t* dev_status) {
    __shared__ int s_par[4][kMaxNodes], s_tok[4][kMaxNodes], s_vt[4][kMaxNodes];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    pdl_wait();
    const int b = blockIdx.x * 4 + warp;
    if (b >= B) return;
    const int32_t* par = parent + (size_t)b * T;
    int bad = 0;
    for (int i = lane; i < T; i += 32) {
        int p = par[i];
        s_par[warp][i] = p;
        s_tok[warp][i] = tokens[(size_t)b * T + i];
        s_vt[warp][i] = vtok[(size_t)b * T + i];
        if (i == 0) { if (p != -1) bad = 1; }
        else if (p < 0 || p >= i) bad = bad ? bad : 2;
        path[(size_t)b * T + i] = -1;
    }
    unsigned b1 = __ballot_sync(0xffffffffu, bad == 1), b2 = __ballot_sync(0xffffffffu, bad == 2);
    if (b1 | b2) {
        if (lane == 0) {
            path_len[b] = 0;
            bonus[b] = -1;
            report(dev_status, b1 ? 1 : 2);
        }
        return;
    }
    __syncwarp();
    const int* vt = s_vt[warp];
    int cur = 0, len = 1;
    if (lane == 0) path[(size_t)b * T] = 0;
    for (;;) {
        const int want = vt[cur];
        int next = -1;
        // children of cur have index > cur (topological order)
        for (int base = (cur + 1) & ~31; base < T; base += 32) {
            int c = base + lane;
            bool m = c > cur && c < T && s_par[warp][c] == cur && s_tok[warp][c] == want;
            unsigned bal = __ballot_sync(0xffffffffu, m);
            if (bal) { next = base + __ffs(bal) - 1; break; }
        }
        if (next < 0) break;
        if (lane == 0) path[(size_t)b * T + len] = next;
        ++len;
        cur = next;
    }
    if (lane == 0) {
        path_len[b] = len;
        bonus[b] = vt[cur];
    }
}

}  // namespace stree

extern "C" int stree_launch_build_mask(const int32_t* parent, int B, int T, uint32_t* mask,
                                       int32_t* depth, int32_t* dev_status, cudaStream_t s) {
    return (int)stree::launch_k(stree::build_mask_kernel, dim3(B), dim3(256), 0, s, parent, T, mask, depth,
                                dev_status);
}

extern "C" int stree_launch_accept(const int32_t* tokens, const int32_t* parent, const int32_t* vtok,
                                   int B, int T, int32_t* path, int32_t* path_len, int32_t* bonus,
                                   int32_t* dev_status, cudaStream_t s) {
    return (int)stree::launch_k(stree::accept_kernel, dim3((B + 3) / 4), dim3(128), 0, s, tokens, parent, vtok, B, T,
                                path, path_len, bonus, dev_status);
}
