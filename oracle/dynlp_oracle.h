/*
 * dynlp_oracle.h -- CPU restatement of the reference DynLP batch update.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path
 * (paper_2604_06596_b200/) links, loads or calls this library.  It is the
 * checker for the CUDA engine (tests/, __graft_entry__.smoke) and the
 * "port" CPU baseline in bench.py.  Every function cites the reference
 * file:line it restates; roots:
 *   engine.py     = /root/reference/pkg/src/dynlp/engine.py
 *   graph.py      = /root/reference/pkg/src/dynlp/graph.py
 *   components.py = /root/reference/pkg/src/dynlp/components.py
 *   labels.py     = /root/reference/pkg/src/dynlp/labels.py
 *   _csr.pyx      = /root/reference/pkg/src/dynlp/kernels/_csr.pyx
 *
 * Parity is pinned against the reference itself: tests/golden/ holds
 * fixtures produced by importing the reference (tests/golden/make_golden.py)
 * and tests/test_oracle.py replays them bit-for-bit.
 */
#ifndef DYNLP_ORACLE_H
#define DYNLP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_engine orc_engine;

typedef struct {
    double delta;            /* engine.py:42 */
    double tau;              /* NaN = "auto" (engine.py:43, 182-188) */
    int64_t max_iterations;  /* <= 0: 10 * num_alive (engine.py:67-70) */
    int32_t component_init;  /* engine.py:47 */
    int32_t mode;            /* 0 jacobi, 1 gauss-seidel (engine.py:33-34) */
} orc_config;

typedef struct {
    int64_t t;
    int64_t n_ins;
    const int64_t* insert_ids;
    const int8_t* insert_gt;
    int64_t n_edges;
    const int64_t* edge_owner;
    const int64_t* edge_other;
    const double* edge_w;
    int64_t n_del;
    const int64_t* deletes;
} orc_batch;

typedef struct {
    int64_t t;
    int64_t iterations;
    int64_t updates;
    double max_change;
    int32_t converged;
    int32_t pad;
    int64_t warnings;
    int64_t isolated_pinned;
    int64_t unreachable_pinned;
    double wall_time_ms;
    int64_t edges_traversed;
    int64_t certify_sweeps;
} orc_report;

orc_engine* orc_create(int32_t num_classes, int32_t threads);
void orc_destroy(orc_engine* e);
const char* orc_last_error(orc_engine* e);
int32_t orc_num_columns(orc_engine* e);

/* engine.apply_batch (engine.py:328-413); one report per label column.
 * Returns 0 ok, 3 validation error (state untouched). */
int orc_apply_batch(orc_engine* e, const orc_config* cfg, const orc_batch* b, orc_report* reps);
/* engine.apply_batch_structure only (engine.py:141-156): used for state hand-off. */
int orc_apply_structure(orc_engine* e, const orc_batch* b);

int64_t orc_num_slots(orc_engine* e);
int64_t orc_num_alive(orc_engine* e);
int64_t orc_num_live_edges(orc_engine* e);
double orc_last_tau(orc_engine* e);
/* f is [C][n_slots] column-major; gt is the raw class array */
void orc_read_labels(orc_engine* e, double* f, int8_t* gt);
void orc_write_labels(orc_engine* e, const double* f);
void orc_read_alive(orc_engine* e, uint8_t* alive);
/* DynamicGraph.csr() snapshot (graph.py:218-231); nnz = 2 * live edges */
void orc_read_csr(orc_engine* e, int64_t* indptr, int64_t* indices, double* weights, double* degrees);
/* live_edges() in log order (graph.py:205-216) */
void orc_read_live_edges(orc_engine* e, int64_t* u, int64_t* v, double* w);
/* eligible mask computed by the last apply_batch (before the loop mutates it) */
void orc_read_eligible(orc_engine* e, uint8_t* elig);
/* intra-batch labeling of the last apply_batch: vertices sorted, parent, component_id */
int64_t orc_intra_size(orc_engine* e);
int64_t orc_read_intra(orc_engine* e, int64_t* vertices, int64_t* parent, int64_t* comp);

/* numpy pairwise summation (np.add.reduce on a contiguous float64 array). */
double orc_pairwise_sum(const double* a, int64_t n);

/* Kernel-level plugin API on caller CSR, restating _csr.pyx:61-91, 94-111, 114-197. */
void orc_jacobi_step(const int64_t* indptr, const int64_t* indices, const double* weights,
                     const int8_t* gt, const double* f, const int64_t* frontier, int64_t nf,
                     double* out_vals, double* out_deltas, int32_t threads);
void orc_gauss_seidel_step(const int64_t* indptr, const int64_t* indices, const double* weights,
                           const int8_t* gt, double* f, const int64_t* frontier, int64_t nf,
                           double* out_deltas);
/* returns leftover count; leftover written in discovery order like _csr.pyx:196 */
int64_t orc_jacobi_run(const int64_t* indptr, const int64_t* indices, const double* weights,
                       const int8_t* gt, double* f, int64_t n, const int64_t* frontier_init,
                       int64_t nf, uint8_t* eligible, double delta, int64_t max_iters,
                       int32_t threads, int64_t* out_iters, int64_t* out_updates,
                       double* out_max_change, int64_t* out_warnings, int64_t* leftover);

#ifdef __cplusplus
}
#endif
#endif
