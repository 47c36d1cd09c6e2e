/*
 * dynlp_oracle.c -- CPU restatement of the reference DynLP per-batch update.
 *
 * TEST INFRASTRUCTURE ONLY (see dynlp_oracle.h).  This is the checker the
 * CUDA engine is compared against and the "port" CPU baseline; it is never
 * linked into the product library.  It follows the reference algorithm
 * step by step -- including its summation orders, which are part of the
 * numeric contract -- rather than any GPU-friendly reformulation.
 */
#include "dynlp_oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define COMPACT_DEAD_FRACTION 0.25 /* graph.py:21 */
#define PARALLEL_CUTOFF 1024       /* _csr.pyx:21 */

struct orc_engine {
    int32_t num_classes, ncol, threads;
    int64_t n_slots, num_alive, cap;
    uint8_t* alive;
    double* f; /* ncol columns, stride cap */
    int8_t* gt;
    /* edge log: the concatenation of DynamicGraph._chunks (graph.py:180) */
    int64_t log_n, log_cap;
    int64_t *lo, *hi;
    double* lw;
    int64_t dead_at_last_compact;
    /* CsrView cache (graph.py:167-173, 218-231) */
    int csr_valid;
    int64_t *indptr, *indices;
    double *weights, *degrees;
    int64_t csr_rows_cap, csr_nnz_cap;
    double last_tau;
    uint8_t* last_elig;
    int64_t intra_n, intra_cap;
    int64_t *intra_v, *intra_p, *intra_c;
    char err[512];
};

static void* xrealloc(void* p, size_t n) {
    void* q = realloc(p, n ? n : 1);
    if (!q) {
        fprintf(stderr, "dynlp_oracle: out of memory (%zu bytes)\n", n);
        abort();
    }
    return q;
}

static int fail(orc_engine* e, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(e->err, sizeof e->err, fmt, ap);
    va_end(ap);
    return 3;
}

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

/* ------------------------------------------------------------------ */
/* numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src,  */
/* @TYPE@_pairwise_sum), used by np.mean in resolve_tau (engine.py:187) */
/* ------------------------------------------------------------------ */
double orc_pairwise_sum(const double* a, int64_t n) {
    if (n < 8) {
        double res = -0.0;
        for (int64_t i = 0; i < n; i++) res += a[i];
        return res;
    } else if (n <= 128) {
        double r[8];
        int64_t i;
        for (int j = 0; j < 8; j++) r[j] = a[j];
        for (i = 8; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; j++) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; i++) res += a[i];
        return res;
    } else {
        int64_t n2 = n / 2;
        n2 -= n2 % 8;
        return orc_pairwise_sum(a, n2) + orc_pairwise_sum(a + n2, n - n2);
    }
}

/* ------------------------------------------------------------------ */
/* _update_one (_csr.pyx:24-58): sequential fp64 row sum, no FMA.      */
/* ------------------------------------------------------------------ */
static inline double update_one(const int64_t* indptr, const int64_t* indices, const double* weights,
                                const int8_t* gt, const double* f, int64_t u, double* out_val) {
    double w_all = 0.0, w0 = 0.0, w1 = 0.0, s = 0.0;
    double fu = f[u];
    for (int64_t e = indptr[u]; e < indptr[u + 1]; e++) {
        int64_t v = indices[e];
        double w = weights[e];
        w_all += w;
        int8_t g = gt[v];
        if (g == 0)
            w0 += w;
        else if (g == 1)
            w1 += w;
        else
            s += (f[v] - fu) * w;
    }
    if (w_all <= 0.0) {
        *out_val = 0.5;
        return -1.0;
    }
    double fn = fu + (0.0 - fu) * (w0 / w_all) + (1.0 - fu) * (w1 / w_all) + s / w_all;
    if (fn < 0.0)
        fn = 0.0;
    else if (fn > 1.0)
        fn = 1.0;
    *out_val = fn;
    return fabs(fn - fu);
}

/* jacobi_step (_csr.pyx:61-91) */
void orc_jacobi_step(const int64_t* indptr, const int64_t* indices, const double* weights,
                     const int8_t* gt, const double* f, const int64_t* frontier, int64_t nf,
                     double* out_vals, double* out_deltas, int32_t threads) {
    if (threads > 1 && nf >= PARALLEL_CUTOFF) {
#pragma omp parallel for schedule(static) num_threads(threads)
        for (int64_t i = 0; i < nf; i++)
            out_deltas[i] = update_one(indptr, indices, weights, gt, f, frontier[i], &out_vals[i]);
    } else {
        for (int64_t i = 0; i < nf; i++)
            out_deltas[i] = update_one(indptr, indices, weights, gt, f, frontier[i], &out_vals[i]);
    }
}

/* gauss_seidel_step (_csr.pyx:94-111) */
void orc_gauss_seidel_step(const int64_t* indptr, const int64_t* indices, const double* weights,
                           const int8_t* gt, double* f, const int64_t* frontier, int64_t nf,
                           double* out_deltas) {
    for (int64_t i = 0; i < nf; i++) {
        double val;
        int64_t u = frontier[i];
        out_deltas[i] = update_one(indptr, indices, weights, gt, f, u, &val);
        f[u] = val;
    }
}

/* jacobi_run (_csr.pyx:114-197): fused evaluate / serial commit+expand. */
static int64_t jacobi_run_impl(const int64_t* indptr, const int64_t* indices, const double* weights,
                               const int8_t* gt, double* f, int64_t n, const int64_t* frontier_init,
                               int64_t nf, uint8_t* eligible, double delta, int64_t max_iters,
                               int32_t threads, int64_t* out_iters, int64_t* out_updates,
                               double* out_max_change, int64_t* out_warnings, int64_t* leftover,
                               int64_t* out_edges) {
    /* A frontier may hold duplicates at the kernel-level API, so the
     * working lists are sized by max(n, nf) rather than n. */
    int64_t lcap = n > nf ? n : nf;
    int64_t* cur = (int64_t*)xrealloc(NULL, sizeof(int64_t) * (lcap + 1));
    int64_t* nxt = (int64_t*)xrealloc(NULL, sizeof(int64_t) * (lcap + 1));
    double* vals = (double*)xrealloc(NULL, sizeof(double) * (lcap + 1));
    double* deltas = (double*)xrealloc(NULL, sizeof(double) * (lcap + 1));
    uint8_t* in_next = (uint8_t*)calloc(n + 1, 1);
    memcpy(cur, frontier_init, sizeof(int64_t) * nf);
    int64_t cur_len = nf, iterations = 0, updates = 0, warnings = 0, edges = 0;
    double max_change = 0.0;
    while (cur_len > 0 && iterations < max_iters) {
        orc_jacobi_step(indptr, indices, weights, gt, f, cur, cur_len, vals, deltas, threads);
        double round_max = 0.0;
        int64_t next_len = 0;
        for (int64_t i = 0; i < cur_len; i++) {
            int64_t u = cur[i];
            double d = deltas[i];
            edges += indptr[u + 1] - indptr[u];
            f[u] = vals[i];
            if (d < 0.0) {
                warnings++;
                eligible[u] = 0;
                continue;
            }
            if (d > round_max) round_max = d;
            if (d > delta) {
                if (in_next[u] == 0 && eligible[u] != 0) {
                    in_next[u] = 1;
                    nxt[next_len++] = u;
                }
                for (int64_t e = indptr[u]; e < indptr[u + 1]; e++) {
                    int64_t v = indices[e];
                    if (eligible[v] != 0 && in_next[v] == 0) {
                        in_next[v] = 1;
                        nxt[next_len++] = v;
                    }
                }
            }
        }
        updates += cur_len;
        iterations++;
        max_change = round_max;
        for (int64_t i = 0; i < next_len; i++) in_next[nxt[i]] = 0;
        int64_t* tmp = cur;
        cur = nxt;
        nxt = tmp;
        cur_len = next_len;
    }
    if (leftover) memcpy(leftover, cur, sizeof(int64_t) * cur_len);
    *out_iters = iterations;
    *out_updates = updates;
    *out_max_change = max_change;
    *out_warnings = warnings;
    if (out_edges) *out_edges += edges;
    free(cur);
    free(nxt);
    free(vals);
    free(deltas);
    free(in_next);
    return cur_len;
}

int64_t orc_jacobi_run(const int64_t* indptr, const int64_t* indices, const double* weights,
                       const int8_t* gt, double* f, int64_t n, const int64_t* frontier_init,
                       int64_t nf, uint8_t* eligible, double delta, int64_t max_iters,
                       int32_t threads, int64_t* out_iters, int64_t* out_updates,
                       double* out_max_change, int64_t* out_warnings, int64_t* leftover) {
    return jacobi_run_impl(indptr, indices, weights, gt, f, n, frontier_init, nf, eligible, delta,
                           max_iters, threads, out_iters, out_updates, out_max_change,
                           out_warnings, leftover, NULL);
}

/* ------------------------------------------------------------------ */
/* engine state                                                         */
/* ------------------------------------------------------------------ */
orc_engine* orc_create(int32_t num_classes, int32_t threads) {
    orc_engine* e = (orc_engine*)calloc(1, sizeof(orc_engine));
    e->num_classes = num_classes < 2 ? 2 : num_classes;
    e->ncol = e->num_classes <= 2 ? 1 : e->num_classes;
    e->threads = threads < 1 ? 1 : threads;
    e->last_tau = 0.0;
    return e;
}

void orc_destroy(orc_engine* e) {
    if (!e) return;
    free(e->alive);
    free(e->f);
    free(e->gt);
    free(e->lo);
    free(e->hi);
    free(e->lw);
    free(e->indptr);
    free(e->indices);
    free(e->weights);
    free(e->degrees);
    free(e->last_elig);
    free(e->intra_v);
    free(e->intra_p);
    free(e->intra_c);
    free(e);
}

const char* orc_last_error(orc_engine* e) { return e->err; }
int32_t orc_num_columns(orc_engine* e) { return e->ncol; }
int64_t orc_num_slots(orc_engine* e) { return e->n_slots; }
int64_t orc_num_alive(orc_engine* e) { return e->num_alive; }
double orc_last_tau(orc_engine* e) { return e->last_tau; }

static void ensure_vertex_cap(orc_engine* e, int64_t n) {
    if (n <= e->cap) return;
    int64_t nc = e->cap ? e->cap : 1024;
    while (nc < n) nc *= 2;
    e->alive = (uint8_t*)xrealloc(e->alive, nc);
    memset(e->alive + e->cap, 0, nc - e->cap);
    e->gt = (int8_t*)xrealloc(e->gt, nc);
    e->last_elig = (uint8_t*)xrealloc(e->last_elig, nc);
    double* nf = (double*)xrealloc(NULL, sizeof(double) * nc * e->ncol);
    for (int c = 0; c < e->ncol; c++)
        if (e->cap) memcpy(nf + c * nc, e->f + c * e->cap, sizeof(double) * e->n_slots);
    free(e->f);
    e->f = nf;
    e->cap = nc;
}

static void log_reserve(orc_engine* e, int64_t n) {
    if (n <= e->log_cap) return;
    int64_t nc = e->log_cap ? e->log_cap : 1024;
    while (nc < n) nc *= 2;
    e->lo = (int64_t*)xrealloc(e->lo, sizeof(int64_t) * nc);
    e->hi = (int64_t*)xrealloc(e->hi, sizeof(int64_t) * nc);
    e->lw = (double*)xrealloc(e->lw, sizeof(double) * nc);
    e->log_cap = nc;
}

static int64_t count_live(orc_engine* e) {
    int64_t m = 0;
    for (int64_t i = 0; i < e->log_n; i++) m += e->alive[e->lo[i]] & e->alive[e->hi[i]];
    return m;
}

int64_t orc_num_live_edges(orc_engine* e) { return count_live(e); }

/* DynamicGraph.csr() (graph.py:218-231): both directions, stable argsort by
 * source => row x = [hi of log edges with lo==x, log order] ++ [lo of log
 * edges with hi==x, log order]; degrees = np.bincount sequential sums. */
static void build_csr(orc_engine* e) {
    if (e->csr_valid) return;
    int64_t n = e->n_slots;
    int64_t m = count_live(e);
    if (n + 1 > e->csr_rows_cap) {
        e->indptr = (int64_t*)xrealloc(e->indptr, sizeof(int64_t) * (n + 1));
        e->degrees = (double*)xrealloc(e->degrees, sizeof(double) * (n + 1));
        e->csr_rows_cap = n + 1;
    }
    if (2 * m > e->csr_nnz_cap) {
        e->indices = (int64_t*)xrealloc(e->indices, sizeof(int64_t) * 2 * m);
        e->weights = (double*)xrealloc(e->weights, sizeof(double) * 2 * m);
        e->csr_nnz_cap = 2 * m;
    }
    memset(e->indptr, 0, sizeof(int64_t) * (n + 1));
    for (int64_t i = 0; i < e->log_n; i++) {
        int64_t a = e->lo[i], b = e->hi[i];
        if (e->alive[a] && e->alive[b]) {
            e->indptr[a + 1]++;
            e->indptr[b + 1]++;
        }
    }
    for (int64_t x = 0; x < n; x++) e->indptr[x + 1] += e->indptr[x];
    int64_t* cur = (int64_t*)xrealloc(NULL, sizeof(int64_t) * (n + 1));
    memcpy(cur, e->indptr, sizeof(int64_t) * (n + 1));
    for (int64_t i = 0; i < e->log_n; i++) {
        int64_t a = e->lo[i], b = e->hi[i];
        if (e->alive[a] && e->alive[b]) {
            int64_t p = cur[a]++;
            e->indices[p] = b;
            e->weights[p] = e->lw[i];
        }
    }
    for (int64_t i = 0; i < e->log_n; i++) {
        int64_t a = e->lo[i], b = e->hi[i];
        if (e->alive[a] && e->alive[b]) {
            int64_t p = cur[b]++;
            e->indices[p] = a;
            e->weights[p] = e->lw[i];
        }
    }
    free(cur);
    for (int64_t x = 0; x < n; x++) {
        double d = 0.0;
        for (int64_t p = e->indptr[x]; p < e->indptr[x + 1]; p++) d += e->weights[p];
        e->degrees[x] = d;
    }
    e->csr_valid = 1;
}

void orc_read_csr(orc_engine* e, int64_t* indptr, int64_t* indices, double* weights, double* degrees) {
    build_csr(e);
    int64_t n = e->n_slots, nnz = e->indptr[n];
    if (indptr) memcpy(indptr, e->indptr, sizeof(int64_t) * (n + 1));
    if (indices) memcpy(indices, e->indices, sizeof(int64_t) * nnz);
    if (weights) memcpy(weights, e->weights, sizeof(double) * nnz);
    if (degrees) memcpy(degrees, e->degrees, sizeof(double) * n);
}

void orc_read_live_edges(orc_engine* e, int64_t* u, int64_t* v, double* w) {
    int64_t m = 0;
    for (int64_t i = 0; i < e->log_n; i++)
        if (e->alive[e->lo[i]] && e->alive[e->hi[i]]) {
            u[m] = e->lo[i];
            v[m] = e->hi[i];
            w[m] = e->lw[i];
            m++;
        }
}

void orc_read_labels(orc_engine* e, double* f, int8_t* gt) {
    for (int c = 0; c < e->ncol; c++)
        if (f) memcpy(f + c * e->n_slots, e->f + c * e->cap, sizeof(double) * e->n_slots);
    if (gt) memcpy(gt, e->gt, e->n_slots);
}

void orc_write_labels(orc_engine* e, const double* f) {
    for (int c = 0; c < e->ncol; c++)
        memcpy(e->f + c * e->cap, f + c * e->n_slots, sizeof(double) * e->n_slots);
}

void orc_read_alive(orc_engine* e, uint8_t* alive) { memcpy(alive, e->alive, e->n_slots); }
void orc_read_eligible(orc_engine* e, uint8_t* elig) { memcpy(elig, e->last_elig, e->n_slots); }
int64_t orc_intra_size(orc_engine* e) { return e->intra_n; }

int64_t orc_read_intra(orc_engine* e, int64_t* vertices, int64_t* parent, int64_t* comp) {
    memcpy(vertices, e->intra_v, sizeof(int64_t) * e->intra_n);
    memcpy(parent, e->intra_p, sizeof(int64_t) * e->intra_n);
    memcpy(comp, e->intra_c, sizeof(int64_t) * e->intra_n);
    return e->intra_n;
}

/* column view of the ground truth: binary = raw; C > 2 = one-vs-rest */
static void column_gt(const orc_engine* e, int c, int8_t* out) {
    if (e->ncol == 1) {
        memcpy(out, e->gt, e->n_slots);
        return;
    }
    for (int64_t v = 0; v < e->n_slots; v++) out[v] = e->gt[v] < 0 ? -1 : (e->gt[v] == c ? 1 : 0);
}

static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* ------------------------------------------------------------------ */
/* validate_batch (graph.py:254-309) -- atomic, before any mutation.    */
/* ------------------------------------------------------------------ */
static int validate_batch(orc_engine* e, const orc_batch* b) {
    int64_t n = e->n_slots;
    /* validate_deletes (graph.py:254-265) */
    if (b->n_del) {
        int64_t* d = (int64_t*)xrealloc(NULL, sizeof(int64_t) * b->n_del);
        memcpy(d, b->deletes, sizeof(int64_t) * b->n_del);
        qsort(d, b->n_del, sizeof(int64_t), cmp_i64);
        for (int64_t i = 1; i < b->n_del; i++)
            if (d[i] == d[i - 1]) {
                free(d);
                return fail(e, "duplicate vertex id in deletes");
            }
        for (int64_t i = 0; i < b->n_del; i++)
            if (d[i] < 0 || d[i] >= n) {
                int64_t bad = d[i];
                free(d);
                return fail(e, "unknown vertex id %lld in deletes", (long long)bad);
            }
        for (int64_t i = 0; i < b->n_del; i++)
            if (!e->alive[d[i]]) {
                int64_t bad = d[i];
                free(d);
                return fail(e, "vertex %lld is already deleted", (long long)bad);
            }
        free(d);
    }
    /* validate_inserts (graph.py:267-304) */
    int64_t k = b->n_ins;
    if (k == 0) {
        if (b->n_edges) return fail(e, "batch has edges but no inserted vertices");
        return 0;
    }
    int64_t* ids = (int64_t*)xrealloc(NULL, sizeof(int64_t) * k);
    memcpy(ids, b->insert_ids, sizeof(int64_t) * k);
    qsort(ids, k, sizeof(int64_t), cmp_i64);
    for (int64_t i = 1; i < k; i++)
        if (ids[i] == ids[i - 1]) {
            free(ids);
            return fail(e, "duplicate fresh id in inserts");
        }
    for (int64_t i = 0; i < k; i++)
        if (ids[i] != n + i) {
            free(ids);
            return fail(e, "insert ids must be the contiguous block %lld..%lld", (long long)n,
                        (long long)(n + k - 1));
        }
    free(ids);
    /* ids are exactly [n, n+k) from here on */
    for (int64_t i = 0; i < b->n_del; i++)
        if (b->deletes[i] >= n && b->deletes[i] < n + k)
            return fail(e, "a vertex id appears in both inserts and deletes");
    if (b->n_edges) {
        for (int64_t j = 0; j < b->n_edges; j++)
            if (b->edge_w[j] < 0)
                return fail(e, "negative weight on edge to vertex %lld", (long long)b->edge_other[j]);
        for (int64_t j = 0; j < b->n_edges; j++) {
            if (b->edge_owner[j] < 0 || b->edge_owner[j] >= k)
                return fail(e, "edge owner index %lld out of range", (long long)b->edge_owner[j]);
            if (b->insert_ids[b->edge_owner[j]] == b->edge_other[j])
                return fail(e, "self-loop in insert edges");
        }
        /* ext = other[~isin(other, ids)], checks in ext order */
        for (int64_t j = 0; j < b->n_edges; j++) {
            int64_t o = b->edge_other[j];
            if (o >= n && o < n + k) continue;
            if (o < 0 || o >= n) return fail(e, "edge to unknown vertex %lld", (long long)o);
        }
        for (int64_t j = 0; j < b->n_edges; j++) {
            int64_t o = b->edge_other[j];
            if (o >= n && o < n + k) continue;
            if (!e->alive[o]) return fail(e, "edge to a dead vertex %lld", (long long)o);
        }
        if (b->n_del) {
            uint8_t* pend = (uint8_t*)calloc(n + 1, 1);
            for (int64_t i = 0; i < b->n_del; i++) pend[b->deletes[i]] = 1;
            for (int64_t j = 0; j < b->n_edges; j++) {
                int64_t o = b->edge_other[j];
                if (o >= n && o < n + k) continue;
                if (pend[o]) {
                    free(pend);
                    return fail(e, "edge to vertex %lld deleted in the same batch", (long long)o);
                }
            }
            free(pend);
        }
    }
    /* LabelState.set_ground_truth class check (labels.py:42-43), hoisted
     * before mutation so a bad class cannot leave a half-applied batch. */
    for (int64_t i = 0; i < k; i++) {
        int g = b->insert_gt[i];
        if (g < -1 || g >= e->num_classes) {
            if (e->num_classes == 2) return fail(e, "ground-truth class must be 0 or 1");
            return fail(e, "ground-truth class must be in [0, %d)", e->num_classes);
        }
    }
    return 0;
}

/* apply_deletes (graph.py:311-326): returns sorted alive neighbours */
static int64_t apply_deletes(orc_engine* e, const orc_batch* b, uint8_t* mark) {
    if (b->n_del == 0) return 0;
    build_csr(e);
    for (int64_t i = 0; i < b->n_del; i++) e->alive[b->deletes[i]] = 0;
    e->num_alive -= b->n_del;
    int64_t cnt = 0;
    for (int64_t i = 0; i < b->n_del; i++) {
        int64_t x = b->deletes[i];
        for (int64_t p = e->indptr[x]; p < e->indptr[x + 1]; p++) {
            int64_t y = e->indices[p];
            if (e->alive[y] && !mark[y]) {
                mark[y] = 1;
                cnt++;
            }
        }
    }
    e->csr_valid = 0;
    /* _maybe_compact (graph.py:440-447): physical only, order preserving */
    if (e->n_slots) {
        int64_t dead = e->n_slots - e->num_alive;
        if ((double)(dead - e->dead_at_last_compact) / (double)e->n_slots > COMPACT_DEAD_FRACTION) {
            int64_t m = 0;
            for (int64_t i = 0; i < e->log_n; i++)
                if (e->alive[e->lo[i]] && e->alive[e->hi[i]]) {
                    e->lo[m] = e->lo[i];
                    e->hi[m] = e->hi[i];
                    e->lw[m] = e->lw[i];
                    m++;
                }
            e->log_n = m;
            e->dead_at_last_compact = dead;
        }
    }
    return cnt;
}

typedef struct {
    int64_t lo, hi, idx;
} keyed_edge;

static int cmp_keyed(const void* a, const void* b) {
    const keyed_edge *x = (const keyed_edge*)a, *y = (const keyed_edge*)b;
    if (x->lo != y->lo) return (x->lo > y->lo) - (x->lo < y->lo);
    if (x->hi != y->hi) return (x->hi > y->hi) - (x->hi < y->hi);
    return (x->idx > y->idx) - (x->idx < y->idx);
}

typedef struct {
    int64_t first, lo, hi;
    double w;
} merged_edge;

static int cmp_first(const void* a, const void* b) {
    int64_t x = ((const merged_edge*)a)->first, y = ((const merged_edge*)b)->first;
    return (x > y) - (x < y);
}

/* apply_inserts (graph.py:328-361) + ensure_capacity / set_ground_truth
 * (labels.py:28-49).  Marks inserted ids and prior endpoints in mark[]. */
static void apply_inserts(orc_engine* e, const orc_batch* b, uint8_t* mark) {
    int64_t k = b->n_ins;
    if (k == 0) return;
    int64_t base = e->n_slots;
    ensure_vertex_cap(e, base + k);
    for (int64_t i = 0; i < k; i++) {
        e->alive[base + i] = 1;
        e->gt[base + i] = -1;
        for (int c = 0; c < e->ncol; c++) e->f[c * e->cap + base + i] = 0.5;
        mark[base + i] = 1;
    }
    e->n_slots = base + k;
    e->num_alive += k;
    if (b->n_edges) {
        int64_t m = b->n_edges;
        keyed_edge* ke = (keyed_edge*)xrealloc(NULL, sizeof(keyed_edge) * m);
        for (int64_t j = 0; j < m; j++) {
            int64_t a = b->insert_ids[b->edge_owner[j]], o = b->edge_other[j];
            ke[j].lo = a < o ? a : o;
            ke[j].hi = a < o ? o : a;
            ke[j].idx = j;
        }
        qsort(ke, m, sizeof(keyed_edge), cmp_keyed);
        merged_edge* me = (merged_edge*)xrealloc(NULL, sizeof(merged_edge) * m);
        int64_t g = 0;
        for (int64_t j = 0; j < m;) {
            int64_t j2 = j;
            double s = 0.0; /* np.zeros + np.add.at: 0.0 + w1 + w2 ... in batch order */
            while (j2 < m && ke[j2].lo == ke[j].lo && ke[j2].hi == ke[j].hi) {
                s += b->edge_w[ke[j2].idx];
                j2++;
            }
            me[g].first = ke[j].idx;
            me[g].lo = ke[j].lo;
            me[g].hi = ke[j].hi;
            me[g].w = s;
            g++;
            j = j2;
        }
        qsort(me, g, sizeof(merged_edge), cmp_first);
        log_reserve(e, e->log_n + g);
        for (int64_t j = 0; j < g; j++) {
            if (!(me[j].w > 0.0)) continue;
            e->lo[e->log_n] = me[j].lo;
            e->hi[e->log_n] = me[j].hi;
            e->lw[e->log_n] = me[j].w;
            e->log_n++;
            if (me[j].lo < base) mark[me[j].lo] = 1; /* prior endpoints */
            if (me[j].hi < base) mark[me[j].hi] = 1;
        }
        free(ke);
        free(me);
    }
    /* set_ground_truth: gt pinned, f = class (labels.py:37-49) */
    for (int64_t i = 0; i < k; i++) {
        int g = b->insert_gt[i];
        if (g < 0) continue;
        int64_t v = b->insert_ids[i];
        e->gt[v] = (int8_t)g;
        if (e->ncol == 1)
            e->f[v] = (double)g;
        else
            for (int c = 0; c < e->ncol; c++) e->f[c * e->cap + v] = (g == c) ? 1.0 : 0.0;
    }
    e->csr_valid = 0;
}

static double resolve_tau(orc_engine* e, const orc_config* cfg) {
    if (!isnan(cfg->tau)) return cfg->tau;
    int64_t m = count_live(e);
    if (m == 0) return 0.0;
    double* w = (double*)xrealloc(NULL, sizeof(double) * m);
    int64_t j = 0;
    for (int64_t i = 0; i < e->log_n; i++)
        if (e->alive[e->lo[i]] && e->alive[e->hi[i]]) w[j++] = e->lw[i];
    double s = orc_pairwise_sum(w, m);
    free(w);
    return s / (double)m;
}

static int64_t uf_find(int64_t* p, int64_t x) {
    while (p[x] != x) {
        p[x] = p[p[x]];
        x = p[x];
    }
    return x;
}

/* IntraBatchGraph.build + find_components (components.py:53-60, 84-124):
 * the partition of the inserted block by raw batch edges with both ends
 * inserted and w > tau; parent = min member id; dense ids by parent. */
static void intra_components(orc_engine* e, const orc_batch* b, double tau) {
    int64_t k = b->n_ins, base = e->n_slots - k;
    if (k > e->intra_cap) {
        e->intra_v = (int64_t*)xrealloc(e->intra_v, sizeof(int64_t) * k);
        e->intra_p = (int64_t*)xrealloc(e->intra_p, sizeof(int64_t) * k);
        e->intra_c = (int64_t*)xrealloc(e->intra_c, sizeof(int64_t) * k);
        e->intra_cap = k;
    }
    int64_t* par = e->intra_p;
    for (int64_t i = 0; i < k; i++) par[i] = i;
    for (int64_t j = 0; j < b->n_edges; j++) {
        int64_t a = b->insert_ids[b->edge_owner[j]], o = b->edge_other[j];
        if (o < base || o >= base + k) continue;
        if (!(b->edge_w[j] > tau)) continue;
        int64_t ra = uf_find(par, a - base), rb = uf_find(par, o - base);
        if (ra != rb) {
            if (ra < rb)
                par[rb] = ra;
            else
                par[ra] = rb;
        }
    }
    /* roots are minimum members, so a root precedes all of its members */
    int64_t nc = 0;
    for (int64_t i = 0; i < k; i++) {
        int64_t r = uf_find(par, i);
        e->intra_v[i] = base + i;
        e->intra_c[i] = (r == i) ? nc++ : e->intra_c[r];
    }
    for (int64_t i = 0; i < k; i++) par[i] = uf_find(par, i); /* flatten, still local */
    for (int64_t i = 0; i < k; i++) par[i] += base;
    e->intra_n = k;
}

/* initialize_component_labels (engine.py:191-225) for one column */
static void init_components(orc_engine* e, int c, const int8_t* gtc) {
    int64_t k = e->intra_n;
    if (k == 0) return;
    build_csr(e);
    int64_t nc = 0;
    for (int64_t i = 0; i < k; i++)
        if (e->intra_c[i] + 1 > nc) nc = e->intra_c[i] + 1;
    double* per0 = (double*)xrealloc(NULL, sizeof(double) * k);
    double* per1 = (double*)xrealloc(NULL, sizeof(double) * k);
    double* w0 = (double*)calloc(nc, sizeof(double));
    double* w1 = (double*)calloc(nc, sizeof(double));
    for (int64_t i = 0; i < k; i++) {
        int64_t v = e->intra_v[i];
        double a = 0.0, bb = 0.0;
        for (int64_t p = e->indptr[v]; p < e->indptr[v + 1]; p++) {
            int8_t g = gtc[e->indices[p]];
            /* bincount(seg, weights=w*(g==0)): the +0.0 terms are no-ops on a
             * sum that starts at +0.0, so only matching entries are added. */
            if (g == 0) a += e->weights[p];
            if (g == 1) bb += e->weights[p];
        }
        per0[i] = a;
        per1[i] = bb;
    }
    for (int64_t i = 0; i < k; i++) { /* ascending vertex order */
        w0[e->intra_c[i]] += per0[i];
        w1[e->intra_c[i]] += per1[i];
    }
    double* f = e->f + c * e->cap;
    for (int64_t i = 0; i < k; i++) {
        int64_t v = e->intra_v[i];
        if (e->gt[v] != -1) continue;
        int64_t cc = e->intra_c[i];
        double tot = w0[cc] + w1[cc];
        double init;
        if (tot > 0) {
            double safe = tot;
            init = 0.5 - w0[cc] / (2.0 * safe) + w1[cc] / (2.0 * safe);
        } else {
            init = 0.5;
        }
        f[v] = init;
    }
    free(per0);
    free(per1);
    free(w0);
    free(w1);
}

/* reachable_mask (engine.py:166-179): BFS from alive ground truth */
static void reachable(orc_engine* e, uint8_t* reached) {
    build_csr(e);
    int64_t n = e->n_slots;
    int64_t* q = (int64_t*)xrealloc(NULL, sizeof(int64_t) * (n + 1));
    int64_t qh = 0, qt = 0;
    for (int64_t v = 0; v < n; v++) {
        reached[v] = e->alive[v] && e->gt[v] >= 0;
        if (reached[v]) q[qt++] = v;
    }
    while (qh < qt) {
        int64_t u = q[qh++];
        for (int64_t p = e->indptr[u]; p < e->indptr[u + 1]; p++) {
            int64_t v = e->indices[p];
            if (!reached[v]) {
                reached[v] = 1;
                q[qt++] = v;
            }
        }
    }
    free(q);
}

/* _Propagator.step / expand (engine.py:253-288) */
static int64_t prop_step(orc_engine* e, const orc_config* cfg, const int8_t* gtc, double* f,
                         uint8_t* elig, const int64_t* frontier, int64_t nf, int64_t* next,
                         uint8_t* flags, double* max_change, int64_t* warnings, int64_t* edges,
                         int32_t threads) {
    double* vals = (double*)xrealloc(NULL, sizeof(double) * (nf + 1));
    double* deltas = (double*)xrealloc(NULL, sizeof(double) * (nf + 1));
    if (cfg->mode == 0) {
        orc_jacobi_step(e->indptr, e->indices, e->weights, gtc, f, frontier, nf, vals, deltas,
                        threads);
        for (int64_t i = 0; i < nf; i++) f[frontier[i]] = vals[i];
    } else {
        orc_gauss_seidel_step(e->indptr, e->indices, e->weights, gtc, f, frontier, nf, deltas);
    }
    double mc = 0.0;
    for (int64_t i = 0; i < nf; i++) {
        int64_t u = frontier[i];
        *edges += e->indptr[u + 1] - e->indptr[u];
        if (deltas[i] < 0.0) {
            (*warnings)++;
            elig[u] = 0;
        }
        if (deltas[i] > mc) mc = deltas[i];
    }
    for (int64_t i = 0; i < nf; i++) {
        if (!(deltas[i] > cfg->delta)) continue;
        int64_t u = frontier[i];
        flags[u] = 1;
        for (int64_t p = e->indptr[u]; p < e->indptr[u + 1]; p++)
            if (elig[e->indices[p]]) flags[e->indices[p]] = 1;
    }
    int64_t m = 0;
    for (int64_t v = 0; v < e->n_slots; v++)
        if (flags[v]) {
            next[m++] = v;
            flags[v] = 0;
        }
    *max_change = mc;
    free(vals);
    free(deltas);
    return m;
}

/* One label column of apply_batch (engine.py:345-405 after the shared
 * structure / tau / intra-batch components / reachability): init, pin,
 * frontier rounds and certify sweeps.  Writes only column c's labels and its
 * own scratch, so columns may run concurrently. */
static void run_column(orc_engine* e, const orc_config* cfg, int c, const uint8_t* mark,
                       const uint8_t* reached, int64_t isolated, int64_t unreach, int64_t max_iter,
                       int do_init, int32_t threads, orc_report* rep) {
    int64_t n = e->n_slots;
    int8_t* gtc = (int8_t*)xrealloc(NULL, n + 1);
    uint8_t* elig = (uint8_t*)xrealloc(NULL, n + 1);
    uint8_t* flags = (uint8_t*)calloc(n + 1, 1);
    int64_t* frontier = (int64_t*)xrealloc(NULL, sizeof(int64_t) * (n + 1));
    int64_t* next = (int64_t*)xrealloc(NULL, sizeof(int64_t) * (n + 1));
    int64_t* ids = (int64_t*)xrealloc(NULL, sizeof(int64_t) * (n + 1));
    double* f = e->f + c * e->cap;
    column_gt(e, c, gtc);
    if (do_init) init_components(e, c, gtc);
    for (int64_t v = 0; v < n; v++) /* pin unreachable (engine.py:353-360) */
        if (e->alive[v] && e->gt[v] == -1 && !reached[v]) f[v] = 0.5;
    memcpy(elig, e->last_elig, n);
    /* restrict(seeds) (engine.py:246-251, 364-367): sorted, eligible */
    int64_t nf = 0;
    for (int64_t v = 0; v < n; v++)
        if (mark[v] && elig[v]) frontier[nf++] = v;
    int64_t iterations = 0, updates = 0, warnings = 0, edges = 0, certs = 0;
    double max_change = 0.0;
    int converged = 1;
    for (;;) {
        if (cfg->mode == 0) {
            int64_t it, upd, warn;
            double mc;
            nf = jacobi_run_impl(e->indptr, e->indices, e->weights, gtc, f, n, frontier, nf, elig,
                                 cfg->delta, max_iter - iterations, threads, &it, &upd, &mc, &warn,
                                 next, &edges);
            int64_t* tmp = frontier;
            frontier = next;
            next = tmp;
            iterations += it;
            updates += upd;
            warnings += warn;
            if (it) max_change = mc;
        } else {
            while (nf && iterations < max_iter) {
                updates += nf;
                nf = prop_step(e, cfg, gtc, f, elig, frontier, nf, next, flags, &max_change,
                               &warnings, &edges, threads);
                int64_t* tmp = frontier;
                frontier = next;
                next = tmp;
                iterations++;
            }
        }
        if (nf || iterations >= max_iter) {
            converged = nf == 0;
            if (!converged) break;
        }
        /* certify_round (engine.py:290-301) */
        int64_t ni = 0;
        for (int64_t v = 0; v < n; v++)
            if (elig[v]) ids[ni++] = v;
        if (ni == 0) break;
        double mc;
        nf = prop_step(e, cfg, gtc, f, elig, ids, ni, frontier, flags, &mc, &warnings, &edges, threads);
        certs++;
        iterations++;
        updates += ni;
        max_change = mc;
        if (mc <= cfg->delta) break;
    }
    rep->iterations = iterations;
    rep->updates = updates;
    rep->max_change = max_change;
    rep->converged = converged;
    rep->isolated_pinned = isolated;
    rep->unreachable_pinned = unreach;
    rep->warnings = warnings + isolated + unreach;
    rep->edges_traversed = edges;
    rep->certify_sweeps = certs;
    free(gtc);
    free(elig);
    free(flags);
    free(frontier);
    free(next);
    free(ids);
}

static int apply_batch_impl(orc_engine* e, const orc_config* cfg, const orc_batch* b,
                            orc_report* reps, int structure_only) {
    double t0 = now_ms();
    int ncol = e->ncol;
    for (int c = 0; c < ncol; c++) {
        memset(&reps[c], 0, sizeof(orc_report));
        reps[c].t = b->t;
        reps[c].converged = 1;
    }
    if (b->n_ins == 0 && b->n_del == 0) { /* engine.py:338-340 */
        double dt = now_ms() - t0;
        for (int c = 0; c < ncol; c++) reps[c].wall_time_ms = dt;
        return 0;
    }
    int rc = validate_batch(e, b);
    if (rc) return rc;
    /* mark[] collects affected_del ∪ affected_ins; sized for the grown graph */
    int64_t n_after = e->n_slots + b->n_ins;
    uint8_t* mark = (uint8_t*)calloc(n_after + 1, 1);
    apply_deletes(e, b, mark);
    apply_inserts(e, b, mark);
    if (structure_only) {
        free(mark);
        return 0;
    }
    int64_t n = e->n_slots;
    e->last_tau = resolve_tau(e, cfg);
    e->intra_n = 0;
    int do_init = cfg->component_init && b->n_ins > 0;
    if (do_init) intra_components(e, b, e->last_tau);
    build_csr(e);
    uint8_t* reached = (uint8_t*)xrealloc(NULL, n + 1);
    reachable(e, reached);
    int64_t isolated = 0, unreach = 0;
    for (int64_t v = 0; v < n; v++) {
        int unl = e->alive[v] && e->gt[v] == -1;
        e->last_elig[v] = unl && reached[v];
        if (unl && !reached[v]) {
            if (e->degrees[v] == 0)
                isolated++;
            else
                unreach++;
        }
    }
    int64_t max_iter = cfg->max_iterations > 0 ? cfg->max_iterations
                                                : (10 * e->num_alive > 1 ? 10 * e->num_alive : 1);
    /* The C one-vs-rest columns are independent reference runs sharing the
     * structure: with threads > 1 and several columns they run concurrently
     * (one column per thread, each column's own rounds serial), otherwise
     * one after the other with the kernel's own threading. */
    int col_par = ncol > 1 && e->threads > 1;
    int inner = col_par ? 1 : e->threads;
#pragma omp parallel for schedule(dynamic, 1) num_threads(col_par ? (e->threads < ncol ? e->threads : ncol) : 1)
    for (int c = 0; c < ncol; c++)
        run_column(e, cfg, c, mark, reached, isolated, unreach, max_iter, do_init, inner, &reps[c]);
    double dt = now_ms() - t0;
    for (int c = 0; c < ncol; c++) reps[c].wall_time_ms = dt;
    free(mark);
    free(reached);
    return 0;
}

int orc_apply_batch(orc_engine* e, const orc_config* cfg, const orc_batch* b, orc_report* reps) {
    return apply_batch_impl(e, cfg, b, reps, 0);
}

int orc_apply_structure(orc_engine* e, const orc_batch* b) {
    orc_report tmp[256];
    orc_config cfg = {1e-4, NAN, 0, 1, 0};
    if (e->ncol > 256) return fail(e, "too many columns");
    return apply_batch_impl(e, &cfg, b, tmp, 1);
}
