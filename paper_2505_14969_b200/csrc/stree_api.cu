// Host side of the C ABI (include/stree.h): argument validation, kernel
// selection and launch.  No allocation, no synchronisation on the hot path.
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "stree_common.cuh"

extern "C" int stree_launch_build_mask(const int32_t*, int, int, uint32_t*, int32_t*, int32_t*, cudaStream_t);
extern "C" int stree_launch_accept(const int32_t*, const int32_t*, const int32_t*, int, int, int32_t*, int32_t*,
                                   int32_t*, int32_t*, cudaStream_t);
extern "C" int stree_launch_commit(const stree_dims*, const void*, const float*, const float*, const void*,
                                   const float*, const int32_t*, const int32_t*, const int32_t*, float*, int32_t*,
                                   cudaStream_t);
extern "C" int stree_launch_scan_simt(const stree_dims*, const void*, const float*, const float*, const void*,
                                      const void*, const float*, const float*, const int32_t*, void*, int32_t*,
                                      cudaStream_t);
extern "C" int stree_launch_scan_tc(const stree_dims*, const void*, const float*, const float*, const void*,
                                    const void*, const float*, const float*, const int32_t*, void*, int32_t*,
                                    cudaStream_t);
extern "C" int stree_tc_supports(const stree_dims*);
extern "C" int stree_lat_supports(const stree_dims*);
extern "C" int stree_launch_scan_lat(const stree_dims*, const void*, const float*, const float*, const void*,
                                     const void*, const float*, const float*, const int32_t*, void*, int32_t*,
                                     cudaStream_t, const void*, const stree_yout*);
extern "C" int stree_launch_replay_scan_lat(const stree_dims*, const void*, const float*, const void*,
                                            const int32_t*, const int32_t*, const int32_t*, const stree_dims*,
                                            const void*, const float*, const float*, const void*, const void*,
                                            const float*, float*, const int32_t*, void*, int32_t*, cudaStream_t,
                                            const stree_yout*);
extern "C" int stree_launch_scan_tc_sharded(const stree_dims*, const void*, const float*, const float*, const void*,
                                            const void*, const float*, const float*, const int32_t*,
                                            const stree_yout*, int32_t*, cudaStream_t);
extern "C" int stree_launch_replay_scan_tc_sharded(const stree_dims*, const void*, const float*, const void*,
                                                   const int32_t*, const int32_t*, const int32_t*, const stree_dims*,
                                                   const void*, const float*, const float*, const void*, const void*,
                                                   const float*, float*, const int32_t*, const stree_yout*, int32_t*,
                                                   cudaStream_t);
extern "C" int stree_tc128_supports(const stree_dims*);
extern "C" int stree_launch_scan_tc128(const stree_dims*, const void*, const float*, const float*, const void*,
                                       const void*, const float*, const float*, const int32_t*, void*, int32_t*,
                                       cudaStream_t);
extern "C" int stree_launch_tree_conv(const stree_conv_dims*, const void*, const float*, const float*, const void*,
                                      const int32_t*, int, void*, int32_t*, cudaStream_t);
extern "C" int stree_launch_conv_commit(const stree_conv_dims*, const void*, const void*, const int32_t*,
                                        const int32_t*, const int32_t*, void*, int32_t*, cudaStream_t);
extern "C" int stree_tc_commit_supports(const stree_dims*);
extern "C" int stree_launch_commit_tc(const stree_dims*, const void*, const float*, const float*, const void*,
                                      const float*, const int32_t*, const int32_t*, const int32_t*, float*, int32_t*,
                                      cudaStream_t);
extern "C" int stree_launch_replay_scan_tc(const stree_dims*, const void*, const float*, const void*, const int32_t*,
                                           const int32_t*, const int32_t*, const stree_dims*, const void*,
                                           const float*, const float*, const void*, const void*, const float*, float*,
                                           const int32_t*, void*, int32_t*, cudaStream_t);

extern "C" int stree_attn_tc_supports(const stree_attn_dims*);
extern "C" int stree_launch_tree_attn(const stree_attn_dims*, const void*, const void*, const void*, const void*,
                                      const void*, const int32_t*, const int32_t*, float, void*, int32_t*, int,
                                      cudaStream_t);
extern "C" int stree_launch_kv_commit(const stree_attn_dims*, const void*, const void*, const int32_t*,
                                      const int32_t*, const int32_t*, void*, void*, int32_t*, int32_t*, cudaStream_t);

extern "C" int stree_launch_accept_mss(const int32_t*, const int32_t*, const float*, const float*, const float*,
                                       const float*, int, int, int, int32_t*, int32_t*, int32_t*, int32_t*,
                                       cudaStream_t);

namespace {

std::atomic<int> g_scan_impl{STREE_SCAN_AUTO};
std::atomic<uint32_t> g_launch_flags{STREE_LAUNCH_PDL};
// Launch flags withheld from the kernels of the call in progress on this thread: an EARLY_* promise
// covers the operands of one call and the kernel immediately preceding it, so a call that launches
// two kernels (or whose operands the promise does not cover) clears the flag for that launch.
thread_local uint32_t tl_flags_mask = ~0u;
thread_local bool tl_replay_allowed = false;   // set by stree_replay_scan around its internal commit
thread_local const stree_scan_opts* tl_opts = nullptr;   // options of the *_ex call in progress
struct OptsScope {
    const stree_scan_opts* saved;
    explicit OptsScope(const stree_scan_opts* o) : saved(tl_opts) { tl_opts = o; }
    ~OptsScope() { tl_opts = saved; }
};
struct FlagsMask {
    uint32_t saved;
    explicit FlagsMask(uint32_t clear) : saved(tl_flags_mask) { tl_flags_mask &= ~clear; }
    ~FlagsMask() { tl_flags_mask = saved; }
};

bool sync_check_enabled() {
    static int v = [] {
        const char* e = std::getenv("STREE_SYNC_CHECK");
        return (e && e[0] && e[0] != '0') ? 1 : 0;
    }();
    return v != 0;
}

stree_status finish(int cuda_rc, int32_t* dev_status, cudaStream_t s) {
    if (cuda_rc != 0) return STREE_ERR_CUDA;
    if (sync_check_enabled()) {
        if (cudaStreamSynchronize(s) != cudaSuccess) return STREE_ERR_CUDA;
        if (dev_status) {
            int32_t v = 0;
            if (cudaMemcpy(&v, dev_status, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess) return STREE_ERR_CUDA;
            if (v) return STREE_ERR_DEVICE;
        }
    }
    return STREE_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

stree_status check_dims(const stree_dims* d) {
    if (!d) return STREE_ERR_NULL;
    if (d->batch < 0 || d->n_nodes < 0 || d->n_nodes > STREE_MAX_NODES) return STREE_ERR_SHAPE;
    if (d->n_heads < 1 || d->head_dim < 1 || d->d_state < 1 || d->n_groups < 1) return STREE_ERR_SHAPE;
    if (d->n_heads % d->n_groups) return STREE_ERR_SHAPE;
    if (d->io_dtype != STREE_F32 && d->io_dtype != STREE_BF16) return STREE_ERR_DTYPE;
    return STREE_OK;
}

}  // namespace

extern "C" {

const char* stree_version(void) { return "stree-b200 0.1 (sm_100a)"; }

uint32_t stree_launch_flags_get() { return g_launch_flags.load(std::memory_order_relaxed) & tl_flags_mask; }

const stree_scan_opts* stree_scan_opts_get() { return tl_opts; }

namespace {
bool opts_ok(const stree_scan_opts* o) { return !o || !o->dt_bias || (reinterpret_cast<uintptr_t>(o->dt_bias) & 3u) == 0; }
}  // namespace

stree_status stree_tree_scan_ex(const stree_dims* d, const void* x, const float* dt, const float* A, const void* Bm,
                                const void* Cm, const float* D, const float* h0, const int32_t* parent, void* y,
                                const stree_scan_opts* opts, int32_t* dev_status, void* stream) {
    if (!opts_ok(opts)) return STREE_ERR_ALIGN;
    OptsScope sc(opts);
    return stree_tree_scan(d, x, dt, A, Bm, Cm, D, h0, parent, y, dev_status, stream);
}

stree_status stree_commit_ex(const stree_dims* d, const void* x, const float* dt, const float* A, const void* Bm,
                             const float* h0, const int32_t* parent, const int32_t* path, const int32_t* path_len,
                             float* h_new, const stree_scan_opts* opts, int32_t* dev_status, void* stream) {
    if (!opts_ok(opts)) return STREE_ERR_ALIGN;
    OptsScope sc(opts);
    return stree_commit(d, x, dt, A, Bm, h0, parent, path, path_len, h_new, dev_status, stream);
}

stree_status stree_replay_scan_ex(const stree_dims* d_prev, const void* x_prev, const float* dt_prev,
                                  const void* Bm_prev, const int32_t* parent_prev, const int32_t* path,
                                  const int32_t* path_len, const stree_dims* d, const void* x, const float* dt,
                                  const float* A, const void* Bm, const void* Cm, const float* D, float* h,
                                  const int32_t* parent, void* y, const stree_scan_opts* opts, int32_t* dev_status,
                                  void* stream) {
    if (!opts_ok(opts)) return STREE_ERR_ALIGN;
    OptsScope sc(opts);
    return stree_replay_scan(d_prev, x_prev, dt_prev, Bm_prev, parent_prev, path, path_len, d, x, dt, A, Bm, Cm, D,
                             h, parent, y, dev_status, stream);
}

stree_status stree_set_launch_flags(uint32_t flags) {
    if (flags & ~(uint32_t)(STREE_LAUNCH_PDL | STREE_LAUNCH_EARLY_STATE | STREE_LAUNCH_EARLY_REPLAY |
                          STREE_LAUNCH_EARLY_TREE | STREE_LAUNCH_EARLY_DT))
        return STREE_ERR_UNSUPPORTED;
    g_launch_flags.store(flags);
    return STREE_OK;
}

const char* stree_status_string(stree_status s) {
    switch (s) {
        case STREE_OK: return "ok";
        case STREE_ERR_NULL: return "null pointer";
        case STREE_ERR_SHAPE: return "bad shape";
        case STREE_ERR_DTYPE: return "unsupported dtype";
        case STREE_ERR_ALIGN: return "misaligned pointer";
        case STREE_ERR_UNSUPPORTED: return "unsupported configuration";
        case STREE_ERR_CUDA: return "cuda error";
        case STREE_ERR_DEVICE: return "device-side status set";
    }
    return "unknown status";
}

stree_status stree_set_scan_impl(stree_scan_impl impl) {
    if (impl != STREE_SCAN_AUTO && impl != STREE_SCAN_SIMT && impl != STREE_SCAN_TC && impl != STREE_SCAN_TC_PIPELINE)
        return STREE_ERR_UNSUPPORTED;
    g_scan_impl.store((int)impl);
    return STREE_OK;
}

int32_t stree_commit_kernel_for(const stree_dims* d, int32_t has_h0) {
    if (check_dims(d) != STREE_OK) return 0;
    int impl = g_scan_impl.load();
    if (impl == STREE_SCAN_SIMT) return 1;
    if (has_h0 && stree_tc_commit_supports(d)) return 2;
    return (impl == STREE_SCAN_TC || impl == STREE_SCAN_TC_PIPELINE) ? 0 : 1;
}

int32_t stree_scan_kernel_for(const stree_dims* d) {
    if (check_dims(d) != STREE_OK) return 0;
    int impl = g_scan_impl.load();
    if (impl == STREE_SCAN_SIMT) return 1;
    if (impl != STREE_SCAN_TC_PIPELINE && stree_lat_supports(d)) return 4;
    if (stree_tc_supports(d)) return 2;
    if (stree_tc128_supports(d)) return 3;
    return (impl == STREE_SCAN_TC || impl == STREE_SCAN_TC_PIPELINE) ? 0 : 1;
}

stree_status stree_build_mask(const int32_t* parent, int32_t batch, int32_t n_nodes, uint32_t* mask,
                              int32_t* depth, int32_t* dev_status, void* stream) {
    if (batch < 0 || n_nodes < 0 || n_nodes > STREE_MAX_NODES) return STREE_ERR_SHAPE;
    if (batch == 0 || n_nodes == 0) return STREE_OK;
    if (!parent || !mask) return STREE_ERR_NULL;
    cudaStream_t s = (cudaStream_t)stream;
    return finish(stree_launch_build_mask(parent, batch, n_nodes, mask, depth, dev_status, s), dev_status, s);
}

stree_status stree_tree_scan(const stree_dims* d, const void* x, const float* dt, const float* A, const void* Bm,
                             const void* Cm, const float* D, const float* h0, const int32_t* parent, void* y,
                             int32_t* dev_status, void* stream) {
    stree_status st = check_dims(d);
    if (st != STREE_OK) return st;
    if (d->batch == 0 || d->n_nodes == 0) return STREE_OK;
    if (!x || !dt || !A || !Bm || !Cm || !parent || !y) return STREE_ERR_NULL;
    const void* ptrs[] = {x, dt, A, Bm, Cm, D, h0, parent, y};
    for (const void* p : ptrs)
        if (p && !aligned16(p)) return STREE_ERR_ALIGN;
    cudaStream_t s = (cudaStream_t)stream;
    int which = stree_scan_kernel_for(d);
    if (which == 0) return STREE_ERR_UNSUPPORTED;
    int rc = (which == 4)   ? stree_launch_scan_lat(d, x, dt, A, Bm, Cm, D, h0, parent, y, dev_status, s, nullptr, nullptr)
             : (which == 2) ? stree_launch_scan_tc(d, x, dt, A, Bm, Cm, D, h0, parent, y, dev_status, s)
             : (which == 3) ? stree_launch_scan_tc128(d, x, dt, A, Bm, Cm, D, h0, parent, y, dev_status, s)
                            : stree_launch_scan_simt(d, x, dt, A, Bm, Cm, D, h0, parent, y, dev_status, s);
    return finish(rc, dev_status, s);
}

stree_status stree_accept(const int32_t* tokens, const int32_t* parent, const int32_t* vtok, int32_t batch,
                          int32_t n_nodes, int32_t* path, int32_t* path_len, int32_t* bonus, int32_t* dev_status,
                          void* stream) {
    if (batch < 0 || n_nodes < 0 || n_nodes > STREE_MAX_NODES) return STREE_ERR_SHAPE;
    if (batch == 0 || n_nodes == 0) return STREE_OK;
    if (!tokens || !parent || !vtok || !path || !path_len || !bonus) return STREE_ERR_NULL;
    cudaStream_t s = (cudaStream_t)stream;
    return finish(stree_launch_accept(tokens, parent, vtok, batch, n_nodes, path, path_len, bonus, dev_status, s),
                  dev_status, s);
}

stree_status stree_commit(const stree_dims* d, const void* x, const float* dt, const float* A, const void* Bm,
                          const float* h0, const int32_t* parent, const int32_t* path, const int32_t* path_len,
                          float* h_new, int32_t* dev_status, void* stream) {
    stree_status st = check_dims(d);
    if (st != STREE_OK) return st;
    if (d->batch == 0 || d->n_nodes == 0) return STREE_OK;
    if (!x || !dt || !A || !Bm || !path || !path_len || !h_new) return STREE_ERR_NULL;
    if (!aligned16(h_new) || (h0 && !aligned16(h0))) return STREE_ERR_ALIGN;
    if (h0 && h0 != h_new) {
        // partial overlap is not allowed (in-place is)
        const char* a = (const char*)h0;
        const char* b = (const char*)h_new;
        size_t bytes = (size_t)d->batch * d->n_heads * d->head_dim * d->d_state * sizeof(float);
        if (a < b + bytes && b < a + bytes) return STREE_ERR_SHAPE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    // EARLY_REPLAY is a promise about stree_replay_scan's previous-tree operands only: the path of a plain
    // commit is normally written by the stree_accept kernel immediately before it
    FlagsMask fm(tl_replay_allowed ? 0u : (uint32_t)STREE_LAUNCH_EARLY_REPLAY);
    const int which = stree_commit_kernel_for(d, h0 != nullptr);
    if (which == 0) return STREE_ERR_UNSUPPORTED;
    if (which == 2) {
        if (!aligned16(x) || !aligned16(Bm) || !aligned16(dt)) return STREE_ERR_ALIGN;
        return finish(stree_launch_commit_tc(d, x, dt, A, Bm, h0, parent, path, path_len, h_new, dev_status, s),
                      dev_status, s);
    }
    return finish(stree_launch_commit(d, x, dt, A, Bm, h0, parent, path, path_len, h_new, dev_status, s),
                  dev_status, s);
}

stree_status stree_replay_scan(const stree_dims* d_prev, const void* x_prev, const float* dt_prev,
                               const void* Bm_prev, const int32_t* parent_prev, const int32_t* path,
                               const int32_t* path_len, const stree_dims* d, const void* x, const float* dt,
                               const float* A, const void* Bm, const void* Cm, const float* D, float* h,
                               const int32_t* parent, void* y, int32_t* dev_status, void* stream) {
    stree_status st = check_dims(d);
    if (st != STREE_OK) return st;
    if ((st = check_dims(d_prev)) != STREE_OK) return st;
    if (d_prev->batch != d->batch || d_prev->n_heads != d->n_heads || d_prev->head_dim != d->head_dim ||
        d_prev->d_state != d->d_state || d_prev->n_groups != d->n_groups || d_prev->io_dtype != d->io_dtype)
        return STREE_ERR_SHAPE;
    if (d->batch == 0) return STREE_OK;
    if (!h) return STREE_ERR_NULL;
    cudaStream_t s = (cudaStream_t)stream;
    const int which = stree_scan_kernel_for(d);
    const bool fused = d->n_nodes > 0 && d_prev->n_nodes > 0 && (which == 2 || which == 4);
    if (!fused) {   // two launches: commit (in place), then scan from the committed state
        if (d_prev->n_nodes > 0) {
            // the commit is the call's first kernel: the caller's EARLY_REPLAY / EARLY_STATE promises hold for it
            tl_replay_allowed = true;
            st = stree_commit(d_prev, x_prev, dt_prev, A, Bm_prev, h, parent_prev, path, path_len, h, dev_status,
                              stream);
            tl_replay_allowed = false;
            if (st != STREE_OK) return st;
            // ... but the scan's carry-in h was just written by that commit: no early state stream
            FlagsMask fm(STREE_LAUNCH_EARLY_STATE);
            return stree_tree_scan(d, x, dt, A, Bm, Cm, D, h, parent, y, dev_status, stream);
        }
        return stree_tree_scan(d, x, dt, A, Bm, Cm, D, h, parent, y, dev_status, stream);
    }
    if (!x_prev || !dt_prev || !Bm_prev || !path || !path_len || !x || !dt || !A || !Bm || !Cm || !parent || !y)
        return STREE_ERR_NULL;
    const void* ptrs[] = {x_prev, dt_prev, Bm_prev, x, dt, A, Bm, Cm, D, h, parent, y};
    for (const void* p : ptrs)
        if (p && !aligned16(p)) return STREE_ERR_ALIGN;
    const int rc = which == 4 ? stree_launch_replay_scan_lat(d_prev, x_prev, dt_prev, Bm_prev, parent_prev, path,
                                                             path_len, d, x, dt, A, Bm, Cm, D, h, parent, y,
                                                             dev_status, s, nullptr)
                              : stree_launch_replay_scan_tc(d_prev, x_prev, dt_prev, Bm_prev, parent_prev, path,
                                                            path_len, d, x, dt, A, Bm, Cm, D, h, parent, y,
                                                            dev_status, s);
    return finish(rc, dev_status, s);
}

namespace {
// a head shard's y destinations (stree_yout): served by the tcgen05 scan kernels (2 = pipeline, 4 = small-batch)
stree_status check_yout(const stree_dims* d, const stree_yout* yo) {
    if (!yo) return STREE_ERR_NULL;
    if (yo->n_peers < 1 || yo->n_peers > STREE_MAX_Y_PEERS) return STREE_ERR_SHAPE;
    if (yo->head_offset < 0 || yo->heads_total < yo->head_offset + d->n_heads) return STREE_ERR_SHAPE;
    for (int p = 0; p < yo->n_peers; ++p) {
        if (!yo->peers[p]) return STREE_ERR_NULL;
        if (!aligned16(yo->peers[p])) return STREE_ERR_ALIGN;
    }
    return STREE_OK;
}
}  // namespace

stree_status stree_tree_scan_sharded(const stree_dims* d, const void* x, const float* dt, const float* A,
                                     const void* Bm, const void* Cm, const float* D, const float* h0,
                                     const int32_t* parent, const stree_yout* yout, int32_t* dev_status,
                                     void* stream) {
    stree_status st = check_dims(d);
    if (st != STREE_OK) return st;
    if ((st = check_yout(d, yout)) != STREE_OK) return st;
    if (d->batch == 0 || d->n_nodes == 0) return STREE_OK;
    if (!x || !dt || !A || !Bm || !Cm || !parent) return STREE_ERR_NULL;
    const void* ptrs[] = {x, dt, A, Bm, Cm, D, h0, parent};
    for (const void* p : ptrs)
        if (p && !aligned16(p)) return STREE_ERR_ALIGN;
    cudaStream_t s = (cudaStream_t)stream;
    const int which = stree_scan_kernel_for(d);
    if (which == 4)
        return finish(stree_launch_scan_lat(d, x, dt, A, Bm, Cm, D, h0, parent, nullptr, dev_status, s, nullptr, yout),
                      dev_status, s);
    if (which == 2)
        return finish(stree_launch_scan_tc_sharded(d, x, dt, A, Bm, Cm, D, h0, parent, yout, dev_status, s),
                      dev_status, s);
    return STREE_ERR_UNSUPPORTED;
}

stree_status stree_replay_scan_sharded(const stree_dims* d_prev, const void* x_prev, const float* dt_prev,
                                       const void* Bm_prev, const int32_t* parent_prev, const int32_t* path,
                                       const int32_t* path_len, const stree_dims* d, const void* x,
                                       const float* dt, const float* A, const void* Bm, const void* Cm,
                                       const float* D, float* h, const int32_t* parent, const stree_yout* yout,
                                       int32_t* dev_status, void* stream) {
    stree_status st = check_dims(d);
    if (st != STREE_OK) return st;
    if ((st = check_dims(d_prev)) != STREE_OK) return st;
    if (d_prev->batch != d->batch || d_prev->n_heads != d->n_heads || d_prev->head_dim != d->head_dim ||
        d_prev->d_state != d->d_state || d_prev->n_groups != d->n_groups || d_prev->io_dtype != d->io_dtype)
        return STREE_ERR_SHAPE;
    if ((st = check_yout(d, yout)) != STREE_OK) return st;
    if (d->batch == 0) return STREE_OK;
    if (d->n_nodes == 0 || d_prev->n_nodes == 0) return STREE_ERR_UNSUPPORTED;   // the fused kernels only
    if (!h || !x_prev || !dt_prev || !Bm_prev || !path || !path_len || !x || !dt || !A || !Bm || !Cm || !parent)
        return STREE_ERR_NULL;
    const void* ptrs[] = {x_prev, dt_prev, Bm_prev, x, dt, A, Bm, Cm, D, h, parent};
    for (const void* p : ptrs)
        if (p && !aligned16(p)) return STREE_ERR_ALIGN;
    cudaStream_t s = (cudaStream_t)stream;
    const int which = stree_scan_kernel_for(d);
    int rc;
    if (which == 4)
        rc = stree_launch_replay_scan_lat(d_prev, x_prev, dt_prev, Bm_prev, parent_prev, path, path_len, d, x, dt, A,
                                          Bm, Cm, D, h, parent, nullptr, dev_status, s, yout);
    else if (which == 2)
        rc = stree_launch_replay_scan_tc_sharded(d_prev, x_prev, dt_prev, Bm_prev, parent_prev, path, path_len, d,
                                                 x, dt, A, Bm, Cm, D, h, parent, yout, dev_status, s);
    else
        return STREE_ERR_UNSUPPORTED;
    return finish(rc, dev_status, s);
}

namespace {
stree_status check_conv_dims(const stree_conv_dims* d) {
    if (!d) return STREE_ERR_NULL;
    if (d->batch < 0 || d->n_nodes < 0 || d->n_nodes > STREE_MAX_NODES || d->channels <= 0 || d->width < 1 ||
        d->width > 4)
        return STREE_ERR_SHAPE;
    if (d->io_dtype != STREE_F32 && d->io_dtype != STREE_BF16) return STREE_ERR_DTYPE;
    const int v = d->io_dtype == STREE_BF16 ? 8 : 4;   // 16-byte channel chunks
    if (d->channels % v) return STREE_ERR_SHAPE;
    return STREE_OK;
}
}  // namespace

stree_status stree_tree_conv(const stree_conv_dims* d, const void* u, const float* weight, const float* bias,
                             const void* conv_state, const int32_t* parent, int32_t act, void* out,
                             int32_t* dev_status, void* stream) {
    stree_status st = check_conv_dims(d);
    if (st != STREE_OK) return st;
    if (d->batch == 0 || d->n_nodes == 0) return STREE_OK;
    if (!u || !weight || !parent || !out) return STREE_ERR_NULL;
    if (!aligned16(u) || !aligned16(out) || !aligned16(weight) || (conv_state && !aligned16(conv_state)))
        return STREE_ERR_ALIGN;
    const size_t es = d->io_dtype == STREE_BF16 ? 2 : 4;
    const size_t bytes = (size_t)d->batch * d->n_nodes * d->channels * es;
    const char *a = (const char*)u, *o = (const char*)out;
    if (a < o + bytes && o < a + bytes) return STREE_ERR_SHAPE;   // out must not overlap u
    cudaStream_t s = (cudaStream_t)stream;
    return finish(stree_launch_tree_conv(d, u, weight, bias, conv_state, parent, act, out, dev_status, s), dev_status,
                  s);
}

stree_status stree_conv_commit(const stree_conv_dims* d, const void* u, const void* conv_state,
                               const int32_t* parent, const int32_t* path, const int32_t* path_len,
                               void* conv_state_new, int32_t* dev_status, void* stream) {
    stree_status st = check_conv_dims(d);
    if (st != STREE_OK) return st;
    if (d->batch == 0 || d->n_nodes == 0 || d->width == 1) return STREE_OK;
    if (!u || !path || !path_len || !conv_state_new) return STREE_ERR_NULL;
    if (!aligned16(u) || !aligned16(conv_state_new) || (conv_state && !aligned16(conv_state))) return STREE_ERR_ALIGN;
    if (conv_state && conv_state != conv_state_new) {
        const size_t es = d->io_dtype == STREE_BF16 ? 2 : 4;
        const size_t bytes = (size_t)d->batch * (d->width - 1) * d->channels * es;
        const char *a = (const char*)conv_state, *o = (const char*)conv_state_new;
        if (a < o + bytes && o < a + bytes) return STREE_ERR_SHAPE;   // partial overlap
    }
    cudaStream_t s = (cudaStream_t)stream;
    return finish(stree_launch_conv_commit(d, u, conv_state, parent, path, path_len, conv_state_new, dev_status, s),
                  dev_status, s);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// tree attention + KV commit
// ---------------------------------------------------------------------------
namespace {
stree_status check_attn_dims(const stree_attn_dims* d) {
    if (!d) return STREE_ERR_NULL;
    if (d->batch < 0 || d->n_nodes < 0 || d->n_nodes > STREE_MAX_NODES) return STREE_ERR_SHAPE;
    if (d->n_q_heads < 1 || d->n_kv_heads < 1 || d->n_q_heads % d->n_kv_heads) return STREE_ERR_SHAPE;
    if (d->head_dim < 1 || d->head_dim > 256 || d->cache_cap < 0) return STREE_ERR_SHAPE;
    if (d->io_dtype != STREE_F32 && d->io_dtype != STREE_BF16) return STREE_ERR_DTYPE;
    return STREE_OK;
}
int attn_use_tc(const stree_attn_dims* d) {
    const int impl = g_scan_impl.load();
    if (impl == STREE_SCAN_SIMT) return 0;
    return stree_attn_tc_supports(d) ? 1 : 0;
}
}  // namespace

int32_t stree_attn_kernel_for(const stree_attn_dims* d) {
    if (check_attn_dims(d) != STREE_OK) return 0;
    return attn_use_tc(d) ? 2 : 1;
}

stree_status stree_tree_attn(const stree_attn_dims* d, const void* q, const void* k_new, const void* v_new,
                             const void* k_cache, const void* v_cache, const int32_t* cache_len,
                             const int32_t* parent, float scale, void* o, int32_t* dev_status, void* stream) {
    stree_status st = check_attn_dims(d);
    if (st != STREE_OK) return st;
    if (d->batch == 0 || d->n_nodes == 0) return STREE_OK;
    if (!q || !k_new || !v_new || !cache_len || !parent || !o) return STREE_ERR_NULL;
    if (d->cache_cap > 0 && (!k_cache || !v_cache)) return STREE_ERR_NULL;
    for (const void* p : {q, k_new, v_new, k_cache, v_cache, (const void*)o})
        if (p && !aligned16(p)) return STREE_ERR_ALIGN;
    const int tc = attn_use_tc(d);
    if (!tc && (g_scan_impl.load() == STREE_SCAN_TC || g_scan_impl.load() == STREE_SCAN_TC_PIPELINE)) return STREE_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    return finish(stree_launch_tree_attn(d, q, k_new, v_new, k_cache, v_cache, cache_len, parent, scale, o,
                                         dev_status, tc, s),
                  dev_status, s);
}

stree_status stree_kv_commit(const stree_attn_dims* d, const void* k_new, const void* v_new, const int32_t* parent,
                             const int32_t* path, const int32_t* path_len, void* k_cache, void* v_cache,
                             int32_t* cache_len, int32_t* dev_status, void* stream) {
    stree_status st = check_attn_dims(d);
    if (st != STREE_OK) return st;
    if (d->batch == 0 || d->n_nodes == 0) return STREE_OK;
    if (!k_new || !v_new || !path || !path_len || !k_cache || !v_cache || !cache_len) return STREE_ERR_NULL;
    if (((size_t)d->n_kv_heads * d->head_dim * (d->io_dtype == STREE_BF16 ? 2 : 4)) % 4) return STREE_ERR_SHAPE;
    for (const void* p : {k_new, v_new, (const void*)k_cache, (const void*)v_cache})
        if (!aligned16(p)) return STREE_ERR_ALIGN;
    cudaStream_t s = (cudaStream_t)stream;
    return finish(stree_launch_kv_commit(d, k_new, v_new, parent, path, path_len, k_cache, v_cache, cache_len,
                                         dev_status, s),
                  dev_status, s);
}

stree_status stree_accept_mss(const int32_t* tokens, const int32_t* parent, const float* p_target,
                              const float* q_draft, const float* u_accept, const float* u_bonus, int32_t batch,
                              int32_t n_nodes, int32_t vocab, int32_t* path, int32_t* path_len, int32_t* bonus,
                              int32_t* dev_status, void* stream) {
    if (batch < 0 || n_nodes < 0 || n_nodes > STREE_MAX_NODES || vocab < 0 || vocab > 150000) return STREE_ERR_SHAPE;
    if (batch == 0 || n_nodes == 0) return STREE_OK;
    if (vocab < 1) return STREE_ERR_SHAPE;
    if (!tokens || !parent || !p_target || !q_draft || !u_accept || !u_bonus || !path || !path_len || !bonus)
        return STREE_ERR_NULL;
    cudaStream_t s = (cudaStream_t)stream;
    return finish(stree_launch_accept_mss(tokens, parent, p_target, q_draft, u_accept, u_bonus, batch, n_nodes, vocab,
                                          path, path_len, bonus, dev_status, s),
                  dev_status, s);
}
