/*
 * stree.h — C ABI of the B200-native STree tree-verify hot path.
 *
 * STree (arXiv 2505.14969) verifies a packed speculative token tree through a
 * diagonal SSM (Mamba-2/SSD) layer in one pass.  This library exposes the four
 * steps of that hot path (BASELINE.json north_star):
 *
 *   stree_build_mask  tree topology -> ancestor mask L          PAPER.md:62-66 (L_ij = 1_{s_i}{t_j}), :90
 *   stree_tree_scan   packed-tree SSM outputs y (no state out)   PAPER.md:86-102 (A_tree = L A_log, y = M_x x0 + M_u u), :108-113
 *   stree_accept      greedy longest accepted path + bonus       PAPER.md:309 (greedy verification), Alg. 1 l.125
 *   stree_commit      state after the last accepted node         PAPER.md:113, Alg. 1 l.123 (activation replay)
 *
 * Conventions (all calls):
 *  - Every array pointer is a DEVICE pointer owned by the caller.  The library
 *    never allocates device memory, never synchronises (unless STREE_SYNC_CHECK=1
 *    is set in the environment, a debug mode), and only enqueues work on `stream`
 *    (a cudaStream_t passed as void*; NULL = legacy default stream).
 *  - Arrays are dense, row-major, contiguous, in the layouts given below.
 *  - Host-detectable problems (NULL pointers, bad sizes, unsupported dtype,
 *    misalignment) return a non-zero stree_status synchronously and launch nothing.
 *  - Tree and path validity is data-dependent and checked on the device.  The
 *    first failure is recorded in *dev_status (one caller-zeroed int32 on the
 *    device) with atomicCAS; the offending tree's outputs are defined below and
 *    the other trees in the batch proceed normally.  dev_status may be NULL.
 *      STREE_DEV_BAD_ROOT   = 1   parent[0] != -1
 *      STREE_DEV_BAD_PARENT = 2   parent[i] outside [0, i) for some i >= 1
 *      STREE_DEV_BAD_PATH   = 3   path not root-anchored / not parent-linked / bad length
 *  - batch == 0 or n_nodes == 0 is a successful no-op.
 *  - Thread safety: calls may be issued concurrently from several host threads.
 *
 * Notation: B = batch of trees, T = nodes per tree (1..256), H = SSM heads,
 * P = head dim, N = d_state, G = groups (G divides H; head h uses group
 * h / (H/G)).  Node 0 is the root; nodes are in topological order
 * (parent[i] < i).
 */
#ifndef STREE_H_
#define STREE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    STREE_OK = 0,
    STREE_ERR_NULL = 1,         /* a required pointer is NULL */
    STREE_ERR_SHAPE = 2,        /* a size is negative / out of range (e.g. T > 256, H % G) */
    STREE_ERR_DTYPE = 3,        /* unsupported dtype combination */
    STREE_ERR_ALIGN = 4,        /* pointer not 16-byte aligned where required */
    STREE_ERR_UNSUPPORTED = 5,  /* valid request this build cannot serve */
    STREE_ERR_CUDA = 6,         /* a CUDA runtime error (launch failure, ...) */
    STREE_ERR_DEVICE = 7        /* only with STREE_SYNC_CHECK=1: *dev_status != 0 after the call */
} stree_status;

typedef enum { STREE_F32 = 0, STREE_BF16 = 1 } stree_dtype;

enum { STREE_DEV_OK = 0, STREE_DEV_BAD_ROOT = 1, STREE_DEV_BAD_PARENT = 2, STREE_DEV_BAD_PATH = 3,
       STREE_DEV_CAPACITY = 5 /* KV cache: cache_len outside [0, cache_cap], or a commit would overflow it */ };

enum { STREE_MAX_NODES = 256 };

typedef struct {
    int32_t batch;        /* B */
    int32_t n_nodes;      /* T, 0..256 */
    int32_t n_heads;      /* H (local heads when the caller shards heads) */
    int32_t head_dim;     /* P */
    int32_t d_state;      /* N */
    int32_t n_groups;     /* G, divides H */
    stree_dtype io_dtype; /* dtype of x, B, C and y */
} stree_dims;

/* Kernel family selection for stree_tree_scan and stree_commit (stree_set_scan_impl). */
typedef enum {
    STREE_SCAN_AUTO = 0,  /* TMA / tcgen05 pipeline kernels when supported, else the CUDA-core kernels.
                             scan: bf16 io, P == 64, N in {64,128}, T <= 64; or N == 128, T <= 256;
                             commit: bf16 io, P == 64, N in {64,128}, T <= 256, h0 given */
    STREE_SCAN_SIMT = 1,  /* CUDA-core kernels (FP32-FMA scan, ring commit; any shape; the fp32 1e-4 path) */
    STREE_SCAN_TC = 2,    /* force the tcgen05 kernels; STREE_ERR_UNSUPPORTED if the shape is not served */
    STREE_SCAN_TC_PIPELINE = 3   /* as STREE_SCAN_TC but never the small-batch kernel (A/B comparisons) */
} stree_scan_impl;

/*
 * stree_build_mask — ancestor (tree) mask.
 *   parent [B][T] int32         parent index, parent[0] = -1.
 *   mask   [B][T][W] uint32     W = ceil(T/32); bit (j % 32) of word j/32 of row i
 *                               is 1 iff node j is on the root-to-i path (inclusive).
 *   depth  [B][T] int32 or NULL depth(i) = |path(i)| - 1.
 * Invalid tree b: dev_status <- 1/2, mask rows and depth of tree b are zero.
 */
stree_status stree_build_mask(const int32_t* parent, int32_t batch, int32_t n_nodes,
                              uint32_t* mask, int32_t* depth, int32_t* dev_status, void* stream);

/*
 * stree_tree_scan — outputs of every node of every packed tree, one SSM layer
 * (PAPER.md:91-102 with the Mamba-2 realisation of SURVEY R1-R3):
 *   Λ_i  = Σ_{j∈path(i)} dt_j A_h                                  (A_tree, Eq. a_tree)
 *   y_i  = e^{Λ_i} C_i·h0ᵀ + Σ_{j∈path(i)} e^{Λ_i-Λ_j} dt_j (C_i·B_j) x_j + D_h x_i
 * which equals the per-node recurrence h_i = e^{dt_i A} h_parent(i) + dt_i x_i B_iᵀ,
 * y_i = h_i C_i + D x_i started from h0 at the root (the root's own update included).
 * No state is written.
 *   x      [B][T][H][P]  io dtype
 *   dt     [B][T][H]     f32, > 0 (post-softplus)
 *   A      [H]           f32, < 0
 *   Bm, Cm [B][T][G][N]  io dtype
 *   D      [H]           f32 or NULL (= 0)
 *   h0     [B][H][P][N]  f32 or NULL (= 0)
 *   parent [B][T]        int32
 *   y      [B][T][H][P]  io dtype; must not alias any input.
 * Invalid tree b: dev_status <- 1/2 and y[b] = 0.
 * Alignment: all pointers 16-byte aligned.
 */
stree_status stree_tree_scan(const stree_dims* d, const void* x, const float* dt, const float* A,
                             const void* Bm, const void* Cm, const float* D, const float* h0,
                             const int32_t* parent, void* y, int32_t* dev_status, void* stream);

/*
 * stree_accept — greedy acceptance walk (Alg. 1 FirstRejected):
 * cur = 0; repeatedly move to the lowest-index child c of cur with
 * tokens[c] == vtok[cur]; stop when none matches; bonus = vtok[cur].
 *   tokens, vtok [B][T] int32  draft tokens (tokens[0], the root, is never compared);
 *                              vtok[i] = verifier argmax (or sample) at node i.
 *   parent [B][T] int32
 *   path   [B][T] int32        accepted node indices root-first, -1 padded.
 *   path_len [B] int32         number of accepted nodes incl. the root (>= 1).
 *   bonus  [B] int32           verifier token at the last accepted node.
 * Invalid tree b: dev_status <- 1/2, path_len = 0, path = -1, bonus = -1.
 */
stree_status stree_accept(const int32_t* tokens, const int32_t* parent, const int32_t* vtok,
                          int32_t batch, int32_t n_nodes, int32_t* path, int32_t* path_len,
                          int32_t* bonus, int32_t* dev_status, void* stream);

/*
 * stree_commit — activation replay of the accepted path (Alg. 1 l.123):
 *   h_new = e^{Λ_k} h0 + Σ_{s∈path} e^{Λ_k-Λ_s} dt_s x_s B_sᵀ,  k = path[path_len-1],
 * i.e. the recurrence above run along the path from h0 (state after k).
 *   x, dt, A, Bm          as in stree_tree_scan (the cached activations of the verified tree)
 *   h0     [B][H][P][N]   f32 (NULL = 0)
 *   parent [B][T] or NULL if given, each path[m] must have parent path[m-1]
 *   path, path_len        as produced by stree_accept
 *   h_new  [B][H][P][N]   f32; h_new == h0 (in-place) is allowed, partial overlap is not.
 * Invalid path for tree b: dev_status <- 3 and h_new[b] = h0[b] (state unchanged).
 */
stree_status stree_commit(const stree_dims* d, const void* x, const float* dt, const float* A,
                          const void* Bm, const float* h0, const int32_t* parent,
                          const int32_t* path, const int32_t* path_len, float* h_new,
                          int32_t* dev_status, void* stream);

/*
 * stree_replay_scan — fused activation replay + tree scan (Alg. 1 l.123-124 in order:
 * ActivationReplay then TreeScan).  Equivalent to
 *   stree_commit(d_prev, x_prev, dt_prev, A, Bm_prev, h, parent_prev, path, path_len, h)   (in place)
 *   stree_tree_scan(d, x, dt, A, Bm, Cm, D, h, parent, y)
 * but every state block is read from HBM once and written once: the replay is applied to the
 * block on chip and the updated block is both the scan's carry-in and the committed state.
 *   d_prev                 dims of the previous (cached) tree; must match d except n_nodes
 *   x_prev, dt_prev, Bm_prev, parent_prev, path, path_len
 *                          the previous iteration's cache and acceptance (as for stree_commit;
 *                          parent_prev may be NULL)
 *   h      [B][H][P][N] f32, in/out: on entry the state the previous tree was scanned from,
 *                          on exit the committed state (h after the accepted path)
 *   x, dt, A, Bm, Cm, D, parent, y   the new tree, as for stree_tree_scan
 * Invalid previous path for tree b: dev_status <- 3 and h[b] is left unchanged (the scan uses it).
 * Invalid new tree: dev_status <- 1/2 and y[b] = 0 (the replay is still applied).
 */
stree_status stree_replay_scan(const stree_dims* d_prev, const void* x_prev, const float* dt_prev,
                               const void* Bm_prev, const int32_t* parent_prev, const int32_t* path,
                               const int32_t* path_len, const stree_dims* d, const void* x,
                               const float* dt, const float* A, const void* Bm, const void* Cm,
                               const float* D, float* h, const int32_t* parent, void* y,
                               int32_t* dev_status, void* stream);

/*
 * Scan options (SURVEY §8(f) unranked variants; the plain calls are the *_ex calls with opts = NULL):
 *   dt_bias        [H] f32 or NULL: dt <- dt + dt_bias[h]                   (Mamba-2's dt bias)
 *   dt_softplus    1: dt <- softplus(dt) = log(1 + e^dt) after the bias       (Mamba-2's discretisation,
 *                  P:70-74 with reading R9: the kernels then take the raw projection output)
 *   d_per_channel  1: D is [H][P], y += D[h][p] x[p]; 0: D is [H]          (Mamba-2's D_has_hdim)
 * The transform applies to every dt a call reads — the new tree's and, in stree_replay_scan_ex /
 * stree_commit_ex, the cached tree's — so the committed state equals the recurrence with the effective
 * dt.  dt_bias and D are per-head parameters: STREE_LAUNCH_EARLY_TREE covers them (read before the
 * dependency wait).  Errors: misaligned dt_bias -> STREE_ERR_ALIGN (4-byte alignment suffices).
 */
typedef struct {
    const float* dt_bias;
    int32_t dt_softplus;
    int32_t d_per_channel;
} stree_scan_opts;

stree_status stree_tree_scan_ex(const stree_dims* d, const void* x, const float* dt, const float* A,
                                const void* Bm, const void* Cm, const float* D, const float* h0,
                                const int32_t* parent, void* y, const stree_scan_opts* opts,
                                int32_t* dev_status, void* stream);
stree_status stree_commit_ex(const stree_dims* d, const void* x, const float* dt, const float* A,
                             const void* Bm, const float* h0, const int32_t* parent, const int32_t* path,
                             const int32_t* path_len, float* h_new, const stree_scan_opts* opts,
                             int32_t* dev_status, void* stream);
stree_status stree_replay_scan_ex(const stree_dims* d_prev, const void* x_prev, const float* dt_prev,
                                  const void* Bm_prev, const int32_t* parent_prev, const int32_t* path,
                                  const int32_t* path_len, const stree_dims* d, const void* x, const float* dt,
                                  const float* A, const void* Bm, const void* Cm, const float* D, float* h,
                                  const int32_t* parent, void* y, const stree_scan_opts* opts,
                                  int32_t* dev_status, void* stream);

/*
 * Head-sharded layers (BASELINE configs[3]: "heads sharded over 2/4/8 GPUs").  Each rank
 * scans its contiguous shard of the heads; the layer's consumer needs the full y [B][T][H][P] on every
 * rank.  Instead of a local y followed by an all-gather, the scan epilogue stores each y tile straight
 * into every rank's full-y buffer at the shard's head offset (P2P stores over NVLink when the peers are
 * peer-mapped buffers, e.g. torch symmetric memory; the collective then overlaps the scan tile by tile).
 * The caller makes the stores visible to the consumers (a cross-rank barrier after the call, e.g. the
 * symmetric-memory handle's barrier); the library does not synchronise ranks.
 */
enum { STREE_MAX_Y_PEERS = 8 };
typedef struct {
    int32_t n_peers;        /* 1 .. STREE_MAX_Y_PEERS (1 = a local, possibly larger, y buffer)           */
    int32_t heads_total;    /* H of the full layer: row pitch of every peer buffer, in heads             */
    int32_t head_offset;    /* index of this call's first head in the full layer                        */
    int32_t reserved;       /* 0                                                                         */
    void* peers[STREE_MAX_Y_PEERS];   /* [B][T][heads_total][P] io-dtype, 16-byte aligned; device pointers
                                         valid in the caller's context (peer-mapped memory for remote ranks) */
} stree_yout;

/*
 * stree_tree_scan_sharded / stree_replay_scan_sharded — stree_tree_scan / stree_replay_scan of a head
 * shard (d->n_heads = the shard's heads; x, dt, A, D, h are the shard's slices), y written to
 * yout->peers[p][b][t][head_offset + h][:] for every peer p.  Served by the tcgen05 scan kernels (bf16,
 * P = 64, N in {64, 128}, T <= 64); other shapes return STREE_ERR_UNSUPPORTED (use the plain call and a
 * collective).  Errors: NULL yout / peer -> STREE_ERR_NULL; n_peers out of range, head_offset + n_heads >
 * heads_total -> STREE_ERR_SHAPE; misaligned peer -> STREE_ERR_ALIGN.
 */
stree_status stree_tree_scan_sharded(const stree_dims* d, const void* x, const float* dt, const float* A,
                                     const void* Bm, const void* Cm, const float* D, const float* h0,
                                     const int32_t* parent, const stree_yout* yout, int32_t* dev_status,
                                     void* stream);
stree_status stree_replay_scan_sharded(const stree_dims* d_prev, const void* x_prev, const float* dt_prev,
                                       const void* Bm_prev, const int32_t* parent_prev, const int32_t* path,
                                       const int32_t* path_len, const stree_dims* d, const void* x,
                                       const float* dt, const float* A, const void* Bm, const void* Cm,
                                       const float* D, float* h, const int32_t* parent, const stree_yout* yout,
                                       int32_t* dev_status, void* stream);

/* Human-readable name of a status code (static storage). */
const char* stree_status_string(stree_status s);

/* Select the scan kernel for subsequent stree_tree_scan calls (process-wide). */
stree_status stree_set_scan_impl(stree_scan_impl impl);

/*
 * Launch options (process-wide, default STREE_LAUNCH_PDL).
 *  STREE_LAUNCH_PDL          launch with programmatic dependent launch: each kernel may be scheduled
 *                            while the kernel before it in the stream is still running and waits
 *                            (griddepcontrol.wait) for that kernel to complete before its first access
 *                            to argument memory.  Every kernel of this library lets its successor launch
 *                            only after passing its own wait, so a library kernel can overlap only the
 *                            kernel IMMEDIATELY preceding it in the stream — never an older one (an
 *                            older kernel has completed before the preceding kernel's wait returned; a
 *                            foreign kernel without PDL completes before ours starts).  Always safe.
 *  STREE_LAUNCH_EARLY_STATE  promise: the state operands of a call are not written by the kernel
 *                            immediately preceding the call in its stream (true in a decode loop: the
 *                            state was committed an iteration earlier).  Covered operands:
 *                              stree_tree_scan, stree_commit, stree_replay_scan: h0 / h;
 *                              stree_tree_attn: k_cache, v_cache and cache_len;
 *                              stree_tree_conv: conv_state (with EARLY_TREE).
 *                            The kernels then start streaming them before the dependency wait.  A call
 *                            that launches two kernels (stree_replay_scan on shapes the fused kernel does
 *                            not serve: commit, then scan) applies the promise to its first kernel only.
 *  STREE_LAUNCH_EARLY_REPLAY promise: the previous tree's operands of stree_replay_scan (path,
 *                            path_len, x_prev, dt_prev, Bm_prev, parent_prev) are not written by the
 *                            kernel immediately preceding the call (true in a decode loop where the
 *                            accept kernel is followed by at least one other kernel — e.g. the next
 *                            iteration's stree_build_mask — before the first replay).  The replay
 *                            prologue (path validation, coefficients, staging) then runs before that
 *                            wait — with EARLY_STATE also the replay of the state tiles already in flight
 *                            (on chip, in shared memory); every global write still follows it.  Only stree_replay_scan honours
 *                            this flag; stree_commit ignores it (its path normally comes from the accept
 *                            kernel just before it).  The replay also reads A under this promise.
 *  STREE_LAUNCH_EARLY_TREE   promise: the tree topology and the per-head parameters of a scan call
 *                            (parent, A, D of stree_tree_scan / stree_replay_scan) are not written by the
 *                            kernel immediately preceding the call (true in a decode loop: the tree is
 *                            fixed for the iteration, A and D are weights).  The tcgen05 scan kernels
 *                            then validate the tree and run the pointer-jumping rounds of the ancestor
 *                            mask before the dependency wait, so only the segsum of dt
 *                            and the contractions remain after it.  x, B, C are never read early.
 *                            stree_tree_conv: parent, weight and bias (read, and every node's window
 *                            tabulated, before the wait; only u is read after it).  stree_tree_attn (with
 *                            EARLY_STATE): parent, validated before the wait; q, k_new, v_new after it.
 *  STREE_LAUNCH_EARLY_DT     promise (with EARLY_TREE): dt of a scan call is not written by the kernel
 *                            immediately preceding it.  True in a Mamba-2 layer, where dt comes from the
 *                            input projection and the causal conv1d kernel (which produces x, B, C) runs
 *                            between the projection and the scan; also true in a stack of back-to-back
 *                            scans.  The tcgen05 scan kernels then compute the segsum Λ and the decay
 *                            coefficients before the dependency wait, so only the contractions remain
 *                            after it.  Without EARLY_TREE the flag is ignored.
 */
enum {
    STREE_LAUNCH_PDL = 1,
    STREE_LAUNCH_EARLY_STATE = 2,
    STREE_LAUNCH_EARLY_REPLAY = 4,
    STREE_LAUNCH_EARLY_TREE = 8,
    STREE_LAUNCH_EARLY_DT = 16
};
stree_status stree_set_launch_flags(uint32_t flags);

/*
 * stree_tree_conv — tree-causal depthwise conv1d over the xBC channels (the
 * paper is silent on the convolution, reading R-conv): Mamba-2's causal conv of width W
 * run along each node's root-to-node path, the committed conv state prepended:
 *   seq_i        = conv_state[b] (W-1 rows, oldest first) ++ u[b][root .. i]
 *   out[b][i][c] = act( bias[c] + sum_{w<W} weight[c][w] * seq_i[len(seq_i) - W + w][c] )
 * act = SiLU (z / (1 + e^-z)) when act != 0, identity otherwise.
 *   u          [B][T][C]    io dtype   (xBC after in_proj)
 *   weight     [C][W]       f32        (W = width, 1..4; weight[c][W-1] multiplies the node itself)
 *   bias       [C]          f32 or NULL
 *   conv_state [B][W-1][C]  io dtype or NULL (zeros)
 *   parent     [B][T]       i32
 *   out        [B][T][C]    io dtype (must not overlap u)
 * C must be a multiple of 8 (bf16) / 4 (f32); arrays 16-byte aligned.  Invalid tree b: dev_status
 * <- 1 / 2 and out[b] = 0.
 */
typedef struct {
    int32_t batch;        /* B */
    int32_t n_nodes;      /* T, 0..256 */
    int32_t channels;     /* C (conv_dim = H*P + 2*G*N for Mamba-2) */
    int32_t width;        /* W, 1..4 (d_conv) */
    stree_dtype io_dtype; /* dtype of u, conv_state, out */
} stree_conv_dims;

stree_status stree_tree_conv(const stree_conv_dims* d, const void* u, const float* weight, const float* bias,
                             const void* conv_state, const int32_t* parent, int32_t act, void* out,
                             int32_t* dev_status, void* stream);

/*
 * stree_conv_commit — conv-state commit along the accepted path (reading R-conv):
 *   conv_state_new[b] = last W-1 rows of (conv_state[b] ++ u[b][path[0 .. path_len-1]])
 *   conv_state     [B][W-1][C] io dtype or NULL (zeros)
 *   parent         [B][T] or NULL: if given, each path[m] must have parent path[m-1]
 *   path, path_len as produced by stree_accept
 *   conv_state_new [B][W-1][C] io dtype; == conv_state (in place) allowed, partial overlap not.
 * Invalid path for tree b: dev_status <- 3 and conv_state_new[b] = conv_state[b].
 */
stree_status stree_conv_commit(const stree_conv_dims* d, const void* u, const void* conv_state,
                               const int32_t* parent, const int32_t* path, const int32_t* path_len,
                               void* conv_state_new, int32_t* dev_status, void* stream);

/*
 * Tree attention for the attention layers of a hybrid SSM/Transformer stack (
 * PAPER.md:19, :54 topology-aware mask, :63-66 L_ij, :318 MambaInLlama; reading R-attn).
 * Node i of tree b attends to every committed cache position and to the tree nodes on its own
 * root-to-i path:
 *   keys(i)    = k_cache[b][0 : cache_len[b]]  ++  k_new[b][path(i)]
 *   o[b][i][h] = Σ_j softmax_j(scale · <q[b][i][h], key_j>) · value_j,   kv head of h = h / (Hq/Hkv)
 * Positional encodings (RoPE at position cache_len + depth(i)) are applied upstream to q / k_new.
 */
typedef struct {
    int32_t batch;        /* B */
    int32_t n_nodes;      /* T, 0..256 */
    int32_t n_q_heads;    /* Hq */
    int32_t n_kv_heads;   /* Hkv, divides Hq (GQA) */
    int32_t head_dim;     /* D, 1..256 (the tcgen05 kernel serves D = 128, bf16, (Hq/Hkv) | 128) */
    int32_t cache_cap;    /* S: rows allocated per sequence in k_cache / v_cache */
    stree_dtype io_dtype; /* dtype of q, k_new, v_new, k_cache, v_cache, o */
} stree_attn_dims;

/*
 * stree_tree_attn — o for every node of every tree (no cache write).
 *   q              [B][T][Hq][D]   io dtype
 *   k_new, v_new   [B][T][Hkv][D]  io dtype (the tree nodes' keys / values)
 *   k_cache, v_cache [B][S][Hkv][D] io dtype (rows >= cache_len[b] are ignored)
 *   cache_len      [B] int32, device, 0 <= cache_len[b] <= S
 *   parent         [B][T] int32
 *   scale          softmax scale (typically 1/sqrt(D))
 *   o              [B][T][Hq][D]   io dtype; must not alias an input.
 * Invalid tree b: dev_status <- 1/2 and o[b] = 0; cache_len[b] out of range: dev_status <- 5, o[b] = 0.
 * Alignment: all pointers 16-byte aligned.
 */
stree_status stree_tree_attn(const stree_attn_dims* d, const void* q, const void* k_new, const void* v_new,
                             const void* k_cache, const void* v_cache, const int32_t* cache_len,
                             const int32_t* parent, float scale, void* o, int32_t* dev_status, void* stream);

/*
 * stree_kv_commit — KV-cache commit of the accepted path (the attention analogue of activation
 * replay, Alg. 1 l.123; reading R-attn):
 *   k_cache[b][cache_len[b] + r] = k_new[b][path[b][r]],  same for v,  r < path_len[b];
 *   cache_len[b] += path_len[b]                                        (cache_len updated in place)
 *   parent [B][T] or NULL: if given, each path[m] must have parent path[m-1]
 *   path, path_len as produced by stree_accept
 * Invalid path for tree b: dev_status <- 3, cache and cache_len[b] unchanged; overflow
 * (cache_len + path_len > S): dev_status <- 5, unchanged.
 * Row size Hkv·D·sizeof(io) must be a multiple of 4 bytes; pointers 16-byte aligned.
 */
stree_status stree_kv_commit(const stree_attn_dims* d, const void* k_new, const void* v_new,
                             const int32_t* parent, const int32_t* path, const int32_t* path_len,
                             void* k_cache, void* v_cache, int32_t* cache_len, int32_t* dev_status,
                             void* stream);

/* Which kernel stree_tree_attn would launch: 1 = SIMT (any shape, fp32), 2 = tcgen05, 0 = invalid. */
int32_t stree_attn_kernel_for(const stree_attn_dims* d);

/*
 * stree_accept_mss — multi-step speculative sampling verification (SpecInfer MSS; SURVEY
 * §8(f) NEXT #4; reading R-mss).  From the root, children are tried in increasing index order:
 *   child c (token t) of cur is accepted iff u_accept[c]·q_draft[cur][t] < p[t]   (u < min(1, p/q));
 *   on rejection p <- max(0, p - q_draft[cur]) / Σ (kept if that mass is 0);
 *   on acceptance cur <- c and p <- p_target[c].
 * When no child of cur is accepted: bonus = smallest v with Σ_{w<=v} p[w] > u_bonus·Σ_w p[w].
 *   tokens   [B][T] int32       drafted tokens (tokens[0] is not compared); out-of-range tokens are rejected
 *   parent   [B][T] int32
 *   p_target [B][T][V] f32      target distribution after each node (post-temperature)
 *   q_draft  [B][T][V] f32      draft distribution each node's children were drawn from
 *   u_accept [B][T] f32 in [0,1) one uniform per child trial (indexed by the child node)
 *   u_bonus  [B] f32 in [0,1)   the bonus sample's uniform
 *   path, path_len, bonus       as for stree_accept
 * Invalid tree b: dev_status <- 1/2, path_len = 0, path = -1, bonus = -1.  V <= 150,000 (three vocabulary
 * slices of V/8 floats per CTA in shared memory).
 */
stree_status stree_accept_mss(const int32_t* tokens, const int32_t* parent, const float* p_target,
                              const float* q_draft, const float* u_accept, const float* u_bonus, int32_t batch,
                              int32_t n_nodes, int32_t vocab, int32_t* path, int32_t* path_len, int32_t* bonus,
                              int32_t* dev_status, void* stream);

/* Which kernel stree_tree_scan would launch for these dims: 1 = SIMT, 2 = tcgen05 pipeline (T <= 64),
 * 3 = tcgen05 128-row-tile kernel (64 < T <= 256, bf16, P = 64, N = 128), 4 = tcgen05 small-batch kernel
 * (T <= 64, one head per CTA: B·H <= #SMs), 0 = invalid.  stree_replay_scan fuses the commit for 2 and 4. */
int32_t stree_scan_kernel_for(const stree_dims* d);

/* Which kernel stree_commit would launch (has_h0: h0 != NULL): 1 = CUDA-core ring / block kernel,
 * 2 = the TMA pipeline kernel (replay warps of the tcgen05 scan kernel), 0 = invalid. */
int32_t stree_commit_kernel_for(const stree_dims* d, int32_t has_h0);

/* Library version string. */
const char* stree_version(void);

#ifdef __cplusplus
}
#endif
#endif /* STREE_H_ */
