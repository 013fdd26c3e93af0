/*
 * oracle/stree_oracle.c — CPU ORACLE FOR THE STREE TREE-VERIFY HOT PATH.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with paper_2505_14969_b200/
 * (the CUDA path) and never reads anything the CUDA path produced.
 *
 * Plain, slow, obviously correct fp64 implementation of the *definition*
 * (SURVEY.md §8(c) C1), not of the paper's fast matrix form:
 *
 *   mask:   L[i][j] = 1 iff node j lies on the root-to-i path        (Eq. L_ij = 1_{s_i}{t_j})
 *   scan:   for every leaf, walk root->leaf from h0 applying the per-node
 *           recurrence (PAPER.md:44-45 read per SURVEY R1):
 *             h_j = exp(dt_j A_h) h_parent(j) + dt_j x_j B_j^T     (state, P x N per head)
 *             y_j = h_j C_j + D_h x_j
 *           (the root's own update applies to x0 = h0, SURVEY R2 / PAPER.md:77)
 *   accept: greedy walk: from the root descend to the
 *           lowest-index child whose token equals the verifier token at the
 *           current node; bonus = verifier token at the stop node.
 *   commit: activation replay (Alg. 1): re-run the same
 *           recurrence along the accepted path from h0; h_new = state after the
 *           last accepted node.
 *   conv:   tree-causal depthwise conv1d (the paper is silent,
 *           DESIGN.md reading R-conv): Mamba-2's causal conv of width W applied along
 *           every root-to-node path, the committed conv state prepended; conv commit
 *           keeps the last W-1 inputs of (state ++ accepted path).
 *
 * Everything is double precision; bf16 inputs are widened exactly by the
 * Python wrapper.  Parallelism: OpenMP over independent (tree, head) pairs
 * only — every value is computed by the same sequential loop as without it.
 *
 * Status codes (returned per tree):
 *   0 ok, 1 parent[0] != -1, 2 parent[i] out of [0, i), 3 invalid path,
 *   99 internal inconsistency (a node reached via two leaves gave two values).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* Tree precondition of PAPER.md:90 (topological order, single root at 0). */
static int check_tree(const int32_t *parent, int T) {
    if (T <= 0) return 0;
    if (parent[0] != -1) return 1;
    for (int i = 1; i < T; ++i)
        if (parent[i] < 0 || parent[i] >= i) return 2;
    return 0;
}

/* Root-to-i path into out[], returns its length (= depth(i) + 1). */
static int path_to(const int32_t *parent, int i, int *out, int T) {
    int len = 0;
    for (int v = i; v >= 0; v = parent[v]) out[len++] = v;
    /* reverse to root-first order */
    for (int a = 0, b = len - 1; a < b; ++a, --b) { int t = out[a]; out[a] = out[b]; out[b] = t; }
    (void)T;
    return len;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

int oracle_set_threads(int n) {
#ifdef _OPENMP
    static int dflt = 0;
    if (!dflt) dflt = omp_get_max_threads();
    omp_set_num_threads(n > 0 ? n : dflt);
#else
    (void)n;
#endif
    return 0;
}

/* L: bit j%32 of word j/32 of row i, W = ceil(T/32) words. */
int oracle_build_mask(const int32_t *parent, int B, int T, uint32_t *mask, int32_t *depth,
                      int32_t *status) {
    int W = (T + 31) / 32;
    int *buf = (int *)malloc(sizeof(int) * (T > 0 ? T : 1));
    for (int b = 0; b < B; ++b) {
        const int32_t *par = parent + (size_t)b * T;
        uint32_t *m = mask + (size_t)b * T * W;
        int32_t *dep = depth + (size_t)b * T;
        memset(m, 0, sizeof(uint32_t) * (size_t)T * W);
        int st = check_tree(par, T);
        status[b] = st;
        if (st) { for (int i = 0; i < T; ++i) dep[i] = 0; continue; }
        for (int i = 0; i < T; ++i) {
            int len = path_to(par, i, buf, T);
            for (int k = 0; k < len; ++k) m[(size_t)i * W + buf[k] / 32] |= 1u << (buf[k] % 32);
            dep[i] = len - 1;
        }
    }
    free(buf);
    return 0;
}

/*
 * y[b][t][h][p] for all nodes, via the per-leaf recurrence.
 * Layouts: x[B][T][H][P], dt[B][T][H], A[H], Bm/Cm[B][T][G][N], D[H] (may be NULL),
 * h0[B][H][P][N] (may be NULL = zeros), parent[B][T].
 */
int oracle_tree_scan(int B, int T, int H, int P, int N, int G,
                     const double *x, const double *dt, const double *A,
                     const double *Bm, const double *Cm, const double *D,
                     const double *h0, const int32_t *parent,
                     double *y, int32_t *status) {
    int bad = 0;
    for (int b = 0; b < B; ++b) status[b] = check_tree(parent + (size_t)b * T, T);
    memset(y, 0, sizeof(double) * (size_t)B * T * H * P);
    long long npairs = (long long)B * H;
#pragma omp parallel for schedule(dynamic, 1) reduction(|:bad)
    for (long long bh = 0; bh < npairs; ++bh) {
        int b = (int)(bh / H), h = (int)(bh % H);
        if (status[b]) continue;
        int g = h / (H / G);
        const int32_t *par = parent + (size_t)b * T;
        double *s = (double *)malloc(sizeof(double) * (size_t)P * N);
        int *path = (int *)malloc(sizeof(int) * (size_t)T);
        char *has_child = (char *)calloc((size_t)T, 1);
        char *written = (char *)calloc((size_t)T, 1);
        for (int i = 1; i < T; ++i) has_child[par[i]] = 1;
        for (int leaf = 0; leaf < T; ++leaf) {
            if (has_child[leaf]) continue;
            int len = path_to(par, leaf, path, T);
            /* s <- x0 = h0 ("initial state x0") */
            for (int pn = 0; pn < P * N; ++pn)
                s[pn] = h0 ? h0[((size_t)b * H + h) * P * N + pn] : 0.0;
            for (int k = 0; k < len; ++k) {
                int j = path[k];
                double dtj = dt[((size_t)b * T + j) * H + h];
                double a = exp(dtj * A[h]);                       /* diagonal transition, Mamba-2 form */
                const double *xj = x + (((size_t)b * T + j) * H + h) * P;
                const double *Bj = Bm + (((size_t)b * T + j) * G + g) * N;
                const double *Cj = Cm + (((size_t)b * T + j) * G + g) * N;
                for (int p = 0; p < P; ++p)
                    for (int n = 0; n < N; ++n)
                        s[p * N + n] = a * s[p * N + n] + dtj * xj[p] * Bj[n];
                double *yj = y + (((size_t)b * T + j) * H + h) * P;
                for (int p = 0; p < P; ++p) {
                    double acc = 0.0;
                    for (int n = 0; n < N; ++n) acc += s[p * N + n] * Cj[n];
                    acc += (D ? D[h] : 0.0) * xj[p];
                    if (written[j]) {
                        if (yj[p] != acc) bad = 1;   /* same fp64 ops => identical value */
                    } else {
                        yj[p] = acc;
                    }
                }
                written[j] = 1;
            }
        }
        free(s); free(path); free(has_child); free(written);
    }
    return bad ? 99 : 0;
}

/* Greedy acceptance (Alg. 1 FirstRejected). */
int oracle_accept(const int32_t *tokens, const int32_t *parent, const int32_t *vtok,
                  int B, int T, int32_t *path, int32_t *path_len, int32_t *bonus,
                  int32_t *status) {
    for (int b = 0; b < B; ++b) {
        const int32_t *tok = tokens + (size_t)b * T, *par = parent + (size_t)b * T,
                      *vt = vtok + (size_t)b * T;
        int32_t *pa = path + (size_t)b * T;
        for (int i = 0; i < T; ++i) pa[i] = -1;
        int st = check_tree(par, T);
        status[b] = st;
        if (st || T == 0) { path_len[b] = 0; bonus[b] = -1; continue; }
        int cur = 0, len = 0;
        pa[len++] = 0;
        for (;;) {
            int next = -1;
            for (int c = 0; c < T; ++c)
                if (par[c] == cur && tok[c] == vt[cur]) { next = c; break; }  /* lowest index wins */
            if (next < 0) break;
            pa[len++] = next;
            cur = next;
        }
        path_len[b] = len;
        bonus[b] = vt[cur];
    }
    return 0;
}

/*
 * Activation replay / commit: recurrence along the accepted
 * path from h0.  parent may be NULL (then only root-anchoring and index range
 * are checked).  On an invalid path the tree's state is left equal to h0.
 */
int oracle_commit(int B, int T, int H, int P, int N, int G,
                  const double *x, const double *dt, const double *A, const double *Bm,
                  const double *h0, const int32_t *parent, const int32_t *path,
                  const int32_t *path_len, double *h_new, int32_t *status) {
    for (int b = 0; b < B; ++b) {
        const int32_t *pa = path + (size_t)b * T;
        int r = path_len[b], st = 0;
        if (r < 1 || r > T || pa[0] != 0) st = 3;
        for (int k = 1; !st && k < r; ++k) {
            if (pa[k] <= pa[k - 1] || pa[k] >= T) st = 3;
            else if (parent && parent[(size_t)b * T + pa[k]] != pa[k - 1]) st = 3;
        }
        status[b] = st;
    }
    long long npairs = (long long)B * H;
#pragma omp parallel for schedule(dynamic, 1)
    for (long long bh = 0; bh < npairs; ++bh) {
        int b = (int)(bh / H), h = (int)(bh % H);
        int g = h / (H / G);
        double *s = h_new + ((size_t)b * H + h) * P * N;
        for (int pn = 0; pn < P * N; ++pn) s[pn] = h0 ? h0[((size_t)b * H + h) * P * N + pn] : 0.0;
        if (status[b]) continue;
        const int32_t *pa = path + (size_t)b * T;
        for (int k = 0; k < path_len[b]; ++k) {
            int j = pa[k];
            double dtj = dt[((size_t)b * T + j) * H + h];
            double a = exp(dtj * A[h]);
            const double *xj = x + (((size_t)b * T + j) * H + h) * P;
            const double *Bj = Bm + (((size_t)b * T + j) * G + g) * N;
            for (int p = 0; p < P; ++p)
                for (int n = 0; n < N; ++n)
                    s[p * N + n] = a * s[p * N + n] + dtj * xj[p] * Bj[n];
        }
    }
    return 0;
}

/*
 * Tree-causal depthwise conv1d (reading R-conv).  For node i with
 * root-to-i path s_i (time order) and the committed conv state (the last W-1
 * inputs before the root, oldest first):
 *   seq_i = state[0..W-2] ++ u[s_i]
 *   out[i][c] = act( bias[c] + sum_{w=0}^{W-1} weight[c][w] * seq_i[len(seq_i)-W+w][c] )
 * i.e. the ordinary causal conv1d of Mamba-2 (weight[c][W-1] multiplies the current
 * input) run on the path that leads to i.  act = SiLU(z) = z / (1 + e^-z) if act != 0.
 * state may be NULL (zeros), bias may be NULL (zeros).  Trees failing PAPER.md:90
 * get status 1/2 and out = 0.
 */
int oracle_tree_conv(int B, int T, int C, int W, const double *u, const double *weight, const double *bias,
                     const double *state, const int32_t *parent, int act, double *out, int32_t *status) {
#pragma omp parallel for schedule(dynamic, 1)
    for (int b = 0; b < B; ++b) {
        const int32_t *par = parent + (size_t)b * T;
        int st = check_tree(par, T);
        status[b] = st;
        double *ob = out + (size_t)b * T * C;
        if (st) {
            memset(ob, 0, sizeof(double) * (size_t)T * C);
            continue;
        }
        int *path = (int *)malloc(sizeof(int) * (size_t)T);
        double *seq = (double *)malloc(sizeof(double) * (size_t)(T + W));
        for (int i = 0; i < T; ++i) {
            int len = path_to(par, i, path, T);
            for (int c = 0; c < C; ++c) {
                int n = 0;
                for (int j = 0; j < W - 1; ++j)
                    seq[n++] = state ? state[((size_t)b * (W - 1) + j) * C + c] : 0.0;
                for (int k = 0; k < len; ++k) seq[n++] = u[((size_t)b * T + path[k]) * C + c];
                double z = bias ? bias[c] : 0.0;
                for (int w = 0; w < W; ++w) z += weight[(size_t)c * W + w] * seq[n - W + w];
                ob[(size_t)i * C + c] = act ? z / (1.0 + exp(-z)) : z;
            }
        }
        free(path);
        free(seq);
    }
    return 0;
}

/*
 * Conv-state commit along the accepted path: the new state is the last W-1
 * entries of state ++ u[path[0..r-1]] (oldest first).  Path checks as in
 * oracle_commit; an invalid path leaves the state unchanged (status 3).
 */
int oracle_conv_commit(int B, int T, int C, int W, const double *u, const double *state,
                       const int32_t *parent, const int32_t *path, const int32_t *path_len,
                       double *state_new, int32_t *status) {
    for (int b = 0; b < B; ++b) {
        const int32_t *pa = path + (size_t)b * T;
        int r = path_len[b], st = 0;
        if (r < 1 || r > T || pa[0] != 0) st = 3;
        for (int k = 1; !st && k < r; ++k) {
            if (pa[k] <= pa[k - 1] || pa[k] >= T) st = 3;
            else if (parent && parent[(size_t)b * T + pa[k]] != pa[k - 1]) st = 3;
        }
        status[b] = st;
        const int L = (W - 1) + (st ? 0 : r);   /* length of state ++ path */
        for (int j = 0; j < W - 1; ++j) {
            int q = L - (W - 1) + j;               /* index into state ++ path */
            for (int c = 0; c < C; ++c) {
                double v;
                if (q < W - 1) v = state ? state[((size_t)b * (W - 1) + q) * C + c] : 0.0;
                else v = u[((size_t)b * T + pa[q - (W - 1)]) * C + c];
                state_new[((size_t)b * (W - 1) + j) * C + c] = v;
            }
        }
    }
    return 0;
}

