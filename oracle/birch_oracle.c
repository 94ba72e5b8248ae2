/*
 * birch_oracle.c — fp64 CPU ORACLE for the BIRCH step of InfraredGP.
 *
 * TEST INFRASTRUCTURE ONLY (same rules as igp_oracle.c): only tests/, smoke() and
 * bench.py's cpu_baseline / reference legs load it; it shares no code, header or
 * constant with the CUDA path (paper_2508_19737_b200/csrc/birch.cu).
 *
 * What the paper computes.  The FFP embeddings Z~ are fed to BIRCH (Zhang et al. 1996),
 * "an efficient K-agnostic clustering algorithm"; static GP
 * fits it to Z~ (Alg. 1 l.7); streaming GP partially fits the CF tree with
 * the new rows only and then predicts every row (Alg. 2 l.9-11, PAPER.md:223-225,
 * :235-236).  The paper "directly invoked BIRCH functions of scikit-learn 1.6.1"
 * with no cluster count, so the algorithm followed here, step by step,
 * is that implementation's single-pass CF-tree insertion with the leaf subclusters as
 * the final clusters (SPEC.md:231-299 for the interface; readings B1-B6 in DESIGN.md):
 *
 *   CF of a set:  (n, LS = sum x, SS = sum |x|^2), centroid c = LS / n, sqn = |c|^2.
 *   insert x (a CF with n = 1) into node v:
 *     j* = argmin_j  sqn_j - 2 c_j . x       (first minimum)
 *     internal: insert into child(j*); if the child did not split, CF_j* += CF_x;
 *               if it split, replace entry j* by the two halves, append the second;
 *               v splits when it has more than B entries.
 *     leaf:     merge x into j* if the merged radius^2 = SS'/n' - |LS'/n'|^2 <= T^2;
 *               else append x as a new entry; v splits when it then has B + 1 entries.
 *   split v:    pairwise d2(a, b) = max(0, (sqn_a - 2 c_a . c_b) + sqn_b) for a < b, mirrored
 *               (symmetric), d2(a, a) = 0; (a*, b*) = first maximum in row-major order, so
 *               a* < b*; entry i goes to the half of
 *               a* iff d2(a*, i) < d2(b*, i) (a* itself always); each half's CF is the sum
 *               of its entries in index order; a split leaf is replaced in the leaf chain
 *               by its two halves (first, second).
 *   root split: a new internal root holding the two halves.
 *   clusters:   the leaf entries in leaf-chain order; label(x) = argmin_j sqn_j - 2 c_j . x.
 *
 * Arithmetic (fixed so that an independent implementation can reproduce every bit):
 * dot(a, b) = eight fma partial sums over k mod 8, combined pairwise (dotk); CF addition updates
 * n, LS (elementwise), SS, then c = LS / n (division), sqn = dot(c, c); the merge test
 * uses c' = (1 / n') * LS' (reciprocal, then products).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define BIRCH_ERR_INPUT (-2)
#define BIRCH_ERR_NOMEM (-3)

typedef struct {
    int32_t d, B;
    double T2;         /* threshold^2 */
    /* subcluster (CF entry) pool */
    int64_t ns, cap_s;
    double* n;         /* [cap_s] point counts (exact integers in double) */
    double* ls;        /* [cap_s][d] */
    double* ss;        /* [cap_s] */
    double* cen;       /* [cap_s][d] */
    double* sqn;       /* [cap_s] */
    int32_t* child;    /* [cap_s] child node, -1 for a leaf entry */
    /* node pool */
    int32_t nn, cap_n;
    int32_t* is_leaf;  /* [cap_n] */
    int32_t* nsub;     /* [cap_n] */
    int64_t* sub;      /* [cap_n][B + 1] entry indices */
    int32_t* prev;     /* [cap_n] leaf chain */
    int32_t* next;
    int32_t root, first_leaf;
    int64_t npoints;
} birch_tree;

/* dot(a, b): eight fma-accumulated partial sums p_r over k = r (mod 8), k ascending, combined
 * as ((p0 + p1) + (p2 + p3)) + ((p4 + p5) + (p6 + p7))  (reading B6: a dot product's summation
 * order is not part of BIRCH; this one is fixed so another implementation can match it) */
static double dotk(const double* a, const double* b, int32_t d) {
    double p[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    for (int32_t k = 0; k < d; ++k) p[k % 8] = fma(a[k], b[k], p[k % 8]);
    return ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
}

static int grow_subs(birch_tree* t) {
    if (t->ns < t->cap_s) return 0;
    int64_t c = t->cap_s ? 2 * t->cap_s : 1024;
    double* n = realloc(t->n, (size_t)c * sizeof(double));
    if (!n) return BIRCH_ERR_NOMEM;
    t->n = n;
    double* ls = realloc(t->ls, (size_t)c * t->d * sizeof(double));
    if (!ls) return BIRCH_ERR_NOMEM;
    t->ls = ls;
    double* ss = realloc(t->ss, (size_t)c * sizeof(double));
    if (!ss) return BIRCH_ERR_NOMEM;
    t->ss = ss;
    double* cen = realloc(t->cen, (size_t)c * t->d * sizeof(double));
    if (!cen) return BIRCH_ERR_NOMEM;
    t->cen = cen;
    double* sqn = realloc(t->sqn, (size_t)c * sizeof(double));
    if (!sqn) return BIRCH_ERR_NOMEM;
    t->sqn = sqn;
    int32_t* ch = realloc(t->child, (size_t)c * sizeof(int32_t));
    if (!ch) return BIRCH_ERR_NOMEM;
    t->child = ch;
    t->cap_s = c;
    return 0;
}

static int grow_nodes(birch_tree* t) {
    if (t->nn < t->cap_n) return 0;
    int32_t c = t->cap_n ? 2 * t->cap_n : 256;
    int32_t* a = realloc(t->is_leaf, (size_t)c * sizeof(int32_t));
    if (!a) return BIRCH_ERR_NOMEM;
    t->is_leaf = a;
    a = realloc(t->nsub, (size_t)c * sizeof(int32_t));
    if (!a) return BIRCH_ERR_NOMEM;
    t->nsub = a;
    int64_t* s = realloc(t->sub, (size_t)c * (t->B + 1) * sizeof(int64_t));
    if (!s) return BIRCH_ERR_NOMEM;
    t->sub = s;
    a = realloc(t->prev, (size_t)c * sizeof(int32_t));
    if (!a) return BIRCH_ERR_NOMEM;
    t->prev = a;
    a = realloc(t->next, (size_t)c * sizeof(int32_t));
    if (!a) return BIRCH_ERR_NOMEM;
    t->next = a;
    t->cap_n = c;
    return 0;
}

/* a new, empty CF entry (n = 0, LS = 0, SS = 0) */
static int64_t new_sub(birch_tree* t) {
    if (grow_subs(t)) return -1;
    int64_t s = t->ns++;
    t->n[s] = 0.0;
    memset(t->ls + s * t->d, 0, (size_t)t->d * sizeof(double));
    t->ss[s] = 0.0;
    memset(t->cen + s * t->d, 0, (size_t)t->d * sizeof(double));
    t->sqn[s] = 0.0;
    t->child[s] = -1;
    return s;
}

static int32_t new_node(birch_tree* t, int leaf) {
    if (grow_nodes(t)) return -1;
    int32_t v = t->nn++;
    t->is_leaf[v] = leaf;
    t->nsub[v] = 0;
    t->prev[v] = t->next[v] = -1;
    return v;
}

/* CF_dst += CF_src, then c = LS / n, sqn = |c|^2 */
static void cf_add(birch_tree* t, int64_t dst, int64_t src) {
    const int32_t d = t->d;
    t->n[dst] += t->n[src];
    double* l = t->ls + dst * d;
    const double* o = t->ls + src * d;
    for (int32_t k = 0; k < d; ++k) l[k] += o[k];
    t->ss[dst] += t->ss[src];
    double* c = t->cen + dst * d;
    for (int32_t k = 0; k < d; ++k) c[k] = l[k] / t->n[dst];
    t->sqn[dst] = dotk(c, c, d);
}

/* CF_dst += the single point x (n = 1, LS = x, SS = |x|^2) */
static void cf_add_point(birch_tree* t, int64_t dst, const double* x, double xx) {
    const int32_t d = t->d;
    t->n[dst] += 1.0;
    double* l = t->ls + dst * d;
    for (int32_t k = 0; k < d; ++k) l[k] += x[k];
    t->ss[dst] += xx;
    double* c = t->cen + dst * d;
    for (int32_t k = 0; k < d; ++k) c[k] = l[k] / t->n[dst];
    t->sqn[dst] = dotk(c, c, d);
}

/* j* = argmin_j sqn_j - 2 c_j . x over the entries of node v (first minimum) */
static int32_t closest(const birch_tree* t, int32_t v, const double* x) {
    int32_t best = 0;
    double bd = 0.0;
    for (int32_t j = 0; j < t->nsub[v]; ++j) {
        const int64_t s = t->sub[(int64_t)v * (t->B + 1) + j];
        const double dist = t->sqn[s] + (-2.0 * dotk(t->cen + s * t->d, x, t->d));
        if (j == 0 || dist < bd) {
            bd = dist;
            best = j;
        }
    }
    return best;
}

/* split node v into two new nodes; returns the two new entries (halves) via h1, h2 */
static int split_node(birch_tree* t, int32_t v, int64_t* h1, int64_t* h2) {
    const int32_t m = t->nsub[v], d = t->d, B1 = t->B + 1;
    const int64_t* ent = t->sub + (int64_t)v * B1;
    double* D = (double*)malloc((size_t)m * m * sizeof(double));
    if (!D) return BIRCH_ERR_NOMEM;
    /* symmetric by construction (computed for a < b, mirrored): reading B4 */
    for (int32_t a = 0; a < m; ++a) {
        D[a * m + a] = 0.0;
        for (int32_t b = a + 1; b < m; ++b) {
            const int64_t sa = ent[a], sb = ent[b];
            double x = (-2.0 * dotk(t->cen + sa * d, t->cen + sb * d, d) + t->sqn[sa]) + t->sqn[sb];
            D[a * m + b] = D[b * m + a] = x > 0.0 ? x : 0.0;
        }
    }
    int32_t ia = 0, ib = 0;
    double mx = D[0];
    for (int32_t a = 0; a < m; ++a)
        for (int32_t b = 0; b < m; ++b)
            if (D[a * m + b] > mx) {
                mx = D[a * m + b];
                ia = a;
                ib = b;
            }
    const int32_t leaf = t->is_leaf[v];
    int32_t n1 = new_node(t, leaf), n2 = new_node(t, leaf);
    int64_t s1 = new_sub(t), s2 = new_sub(t);
    if (n1 < 0 || n2 < 0 || s1 < 0 || s2 < 0) {
        free(D);
        return BIRCH_ERR_NOMEM;
    }
    ent = t->sub + (int64_t)v * B1;  /* the pools may have moved */
    t->child[s1] = n1;
    t->child[s2] = n2;
    if (leaf) {  /* n1 takes v's place in the leaf chain, n2 follows it */
        const int32_t p = t->prev[v], q = t->next[v];
        t->prev[n1] = p;
        t->next[n1] = n2;
        t->prev[n2] = n1;
        t->next[n2] = q;
        if (p >= 0) t->next[p] = n1; else t->first_leaf = n1;
        if (q >= 0) t->prev[q] = n2;
    }
    for (int32_t i = 0; i < m; ++i) {
        const int to1 = (i == ia) || (D[ia * m + i] < D[ib * m + i]);
        const int32_t nd = to1 ? n1 : n2;
        const int64_t h = to1 ? s1 : s2;
        t->sub[(int64_t)nd * B1 + t->nsub[nd]++] = ent[i];
        cf_add(t, h, ent[i]);
    }
    free(D);
    *h1 = s1;
    *h2 = s2;
    return 0;
}

/* insert point x into node v; *split = 1 if v now has to be split by its parent */
static int insert(birch_tree* t, int32_t v, const double* x, double xx, int* split) {
    const int32_t B1 = t->B + 1, d = t->d;
    *split = 0;
    if (t->nsub[v] == 0) {  /* only the empty root leaf */
        int64_t s = new_sub(t);
        if (s < 0) return BIRCH_ERR_NOMEM;
        cf_add_point(t, s, x, xx);
        t->sub[(int64_t)v * B1 + t->nsub[v]++] = s;
        return 0;
    }
    const int32_t j = closest(t, v, x);
    const int64_t sj = t->sub[(int64_t)v * B1 + j];
    if (!t->is_leaf[v]) {
        int child_split = 0;
        int rc = insert(t, t->child[sj], x, xx, &child_split);
        if (rc) return rc;
        if (!child_split) {
            cf_add_point(t, sj, x, xx);
            return 0;
        }
        int64_t h1, h2;
        if ((rc = split_node(t, t->child[sj], &h1, &h2))) return rc;
        t->sub[(int64_t)v * B1 + j] = h1;
        t->sub[(int64_t)v * B1 + t->nsub[v]++] = h2;
        *split = t->nsub[v] > t->B;
        return 0;
    }
    /* leaf: try to absorb x into its closest entry (merged radius^2 <= T^2) */
    const double nn = t->n[sj] + 1.0;
    const double inv = 1.0 / nn;
    double* cand = (double*)malloc((size_t)d * 2 * sizeof(double));
    if (!cand) return BIRCH_ERR_NOMEM;
    double* nls = cand;
    double* nc = cand + d;
    const double* l = t->ls + sj * d;
    for (int32_t k = 0; k < d; ++k) {
        nls[k] = l[k] + x[k];
        nc[k] = inv * nls[k];
    }
    const double nss = t->ss[sj] + xx;
    const double nsq = dotk(nc, nc, d);
    const double r2 = nss / nn - nsq;
    if (r2 <= t->T2) {
        t->n[sj] = nn;
        memcpy(t->ls + sj * d, nls, (size_t)d * sizeof(double));
        t->ss[sj] = nss;
        memcpy(t->cen + sj * d, nc, (size_t)d * sizeof(double));
        t->sqn[sj] = nsq;
        free(cand);
        return 0;
    }
    free(cand);
    int64_t s = new_sub(t);
    if (s < 0) return BIRCH_ERR_NOMEM;
    cf_add_point(t, s, x, xx);
    t->sub[(int64_t)v * B1 + t->nsub[v]++] = s;
    *split = t->nsub[v] > t->B;
    return 0;
}

void* oracle_birch_new(int32_t d, double threshold, int32_t branching) {
    if (d <= 0 || !(threshold > 0.0) || !isfinite(threshold) || branching < 2) return NULL;
    birch_tree* t = (birch_tree*)calloc(1, sizeof(birch_tree));
    if (!t) return NULL;
    t->d = d;
    t->B = branching;
    t->T2 = threshold * threshold;
    t->root = new_node(t, 1);
    t->first_leaf = t->root;
    if (t->root < 0) {
        free(t);
        return NULL;
    }
    return t;
}

void oracle_birch_free(void* h) {
    birch_tree* t = (birch_tree*)h;
    if (!t) return;
    free(t->n);
    free(t->ls);
    free(t->ss);
    free(t->cen);
    free(t->sqn);
    free(t->child);
    free(t->is_leaf);
    free(t->nsub);
    free(t->sub);
    free(t->prev);
    free(t->next);
    free(t);
}

/* fit / partial_fit: insert the rows of X [m][d] (float values widened to double, or
 * double) in row order (Alg. 1 l.7 / Alg. 2 l.9).  X is double here. */
int oracle_birch_partial_fit(void* h, const double* X, int64_t m) {
    birch_tree* t = (birch_tree*)h;
    if (!t || m < 0 || (m > 0 && !X)) return BIRCH_ERR_INPUT;
    const int32_t d = t->d;
    for (int64_t i = 0; i < m * d; ++i)
        if (!isfinite(X[i])) return BIRCH_ERR_INPUT;
    for (int64_t i = 0; i < m; ++i) {
        const double* x = X + i * d;
        const double xx = dotk(x, x, d);
        int split = 0;
        int rc = insert(t, t->root, x, xx, &split);
        if (rc) return rc;
        if (split) {
            int64_t h1, h2;
            if ((rc = split_node(t, t->root, &h1, &h2))) return rc;
            int32_t r = new_node(t, 0);
            if (r < 0) return BIRCH_ERR_NOMEM;
            t->sub[(int64_t)r * (t->B + 1) + t->nsub[r]++] = h1;
            t->sub[(int64_t)r * (t->B + 1) + t->nsub[r]++] = h2;
            t->root = r;
        }
        t->npoints++;
    }
    return 0;
}

/* number of leaf entries (the clusters) */
int64_t oracle_birch_num_clusters(void* h) {
    birch_tree* t = (birch_tree*)h;
    int64_t k = 0;
    for (int32_t v = t->first_leaf; v >= 0; v = t->next[v]) k += t->nsub[v];
    return k;
}

/* the leaf entries in leaf-chain order: centroids [K][d], sqn [K], n [K], LS [K][d], SS [K]
 * (any output may be NULL) */
void oracle_birch_clusters(void* h, double* cen, double* sqn, double* n, double* ls, double* ss) {
    birch_tree* t = (birch_tree*)h;
    const int32_t d = t->d, B1 = t->B + 1;
    int64_t k = 0;
    for (int32_t v = t->first_leaf; v >= 0; v = t->next[v])
        for (int32_t j = 0; j < t->nsub[v]; ++j, ++k) {
            const int64_t s = t->sub[(int64_t)v * B1 + j];
            if (cen) memcpy(cen + k * d, t->cen + s * d, (size_t)d * sizeof(double));
            if (ls) memcpy(ls + k * d, t->ls + s * d, (size_t)d * sizeof(double));
            if (sqn) sqn[k] = t->sqn[s];
            if (n) n[k] = t->n[s];
            if (ss) ss[k] = t->ss[s];
        }
}

/* tree shape: depth (levels), number of nodes, points inserted */
void oracle_birch_shape(void* h, int32_t* depth, int32_t* nodes, int64_t* points) {
    birch_tree* t = (birch_tree*)h;
    int32_t dep = 1;
    for (int32_t v = t->root; !t->is_leaf[v]; v = t->child[t->sub[(int64_t)v * (t->B + 1)]]) ++dep;
    if (depth) *depth = dep;
    if (nodes) *nodes = t->nn;
    if (points) *points = t->npoints;
}

/* predict (Alg. 2 l.11): label_i = argmin_j sqn_j - 2 c_j . x_i over the K clusters
 * (first minimum; |x_i|^2 is common to every j and is not added, reading B5) */
int oracle_birch_predict(const double* cen, const double* sqn, int64_t K, int32_t d, const double* X, int64_t m,
                         int32_t* labels) {
    if (K <= 0 || d <= 0 || m < 0) return BIRCH_ERR_INPUT;
    for (int64_t i = 0; i < m; ++i) {
        const double* x = X + i * d;
        int64_t best = 0;
        double bd = 0.0;
        for (int64_t j = 0; j < K; ++j) {
            const double dist = sqn[j] + (-2.0 * dotk(cen + j * d, x, d));
            if (j == 0 || dist < bd) {
                bd = dist;
                best = j;
            }
        }
        labels[i] = (int32_t)best;
    }
    return 0;
}
