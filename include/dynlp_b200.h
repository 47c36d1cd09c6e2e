/*
 * dynlp_b200.h -- C ABI of the B200-native DynLP batch-update engine.
 *
 * Plain C types only (no torch, no CUDA types), so any FFI (ctypes, cgo,
 * JNI, N-API) can bind it.  Every entry point cites the reference interface
 * it replaces (paths relative to /root/reference/pkg/src/dynlp/).
 *
 * Ownership: the engine owns all device memory (graph,
 * labels, component state) and keeps it resident across calls.  Batch and
 * read-out pointers are borrowed for the duration of one call.  Calls are
 * synchronous: they return after the report is on the host.
 *
 * Status codes (B4): 0 ok, 3 validation (-> dynlp.errors.ValidationError; the
 * engine state is unchanged), 4 format, 5 CUDA, 6 internal.  The message of
 * the last failure is available from dlp_last_error().  Non-convergence is
 * not an error (report.converged = 0).
 */
#ifndef DYNLP_B200_H
#define DYNLP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DLP_OK 0
#define DLP_EVALIDATION 3
#define DLP_EFORMAT 4
#define DLP_ECUDA 5
#define DLP_EINTERNAL 6

#define DLP_MODE_JACOBI 0       /* engine.py:33 "parallel_jacobi" */
#define DLP_MODE_GAUSS_SEIDEL 1 /* engine.py:34 "sequential_gauss_seidel" */

typedef struct dlp_engine dlp_engine;

/* EngineConfig (engine.py:40-70).  threads is meaningless on the device and
 * is not carried; num_classes > 2 selects one-vs-rest label columns. */
typedef struct {
    double delta;           /* engine.py:42; must be > 0 */
    double tau;             /* engine.py:43; NaN = "auto" (mean live weight) */
    int64_t max_iterations; /* engine.py:44; <= 0 = 10 * num_alive (engine.py:67-70) */
    int32_t component_init; /* engine.py:47 */
    int32_t mode;           /* DLP_MODE_* */
    int32_t num_classes;    /* 2 = binary (reference); C > 2 = C columns */
    int32_t reserved;
} dlp_config;

/* BatchUpdate (graph.py:67-82): edge_owner indexes insert_ids. */
typedef struct {
    int64_t t;
    int64_t n_ins;
    const int64_t* insert_ids;
    const int8_t* insert_gt; /* -1 unlabeled, else class */
    int64_t n_edges;
    const int64_t* edge_owner;
    const int64_t* edge_other;
    const double* edge_w;
    int64_t n_del;
    const int64_t* deletes;
} dlp_batch;

/* IterationReport (engine.py:104-115) + device counters. */
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
    int64_t edges_traversed; /* sum of row lengths over every vertex update */
    int64_t certify_sweeps;
    double lp_kernel_ms;     /* CUDA-event time of the batch's fused propagation kernel */
    int64_t gpu_launches;    /* kernels this call launched (all columns) */
    int64_t lp_rounds;       /* lockstep rounds of the fused kernel (all columns) */
    int64_t lp_union_rows;   /* rows the fused kernel evaluated (once for all columns) */
    int64_t lp_union_entries;/* row entries it gathered (one C-wide gather each) */
} dlp_report;

/* Engine lifetime: replaces DynamicGraph() + LabelState() (graph.py:179,
 * labels.py:20) -- an empty graph on `device`. */
int dlp_create(const dlp_config* cfg, int device, dlp_engine** out);
int dlp_destroy(dlp_engine* e);
const char* dlp_last_error(dlp_engine* e);
int dlp_num_columns(dlp_engine* e);

/* engine.apply_batch (engine.py:328-413) with HOST batch arrays.  Writes one
 * report per label column (1 for binary).  cfg may differ between calls
 * (delta / tau / max_iterations / component_init / mode); num_classes is
 * fixed at dlp_create (at most 16 label columns). */
int dlp_apply_batch(dlp_engine* e, const dlp_config* cfg, const dlp_batch* batch,
                    dlp_report* reports);
/* Ingestion pipeline: apply `batch` (HOST arrays) and, while
 * its kernels run, validate `next` against the post-`batch` host mirror and
 * copy it to the device on a copy stream.  The next call with the same
 * `next` pointers skips its validation and copy (a validation error found
 * early is returned by that call, before any mutation).  next may be NULL. */
int dlp_apply_batch_pipelined(dlp_engine* e, const dlp_config* cfg, const dlp_batch* batch, const dlp_batch* next,
                              dlp_report* reports);
/* Same, batch arrays already resident in device memory (bench "value" leg).
 * Validation still runs against the engine's host mirror, so the arrays are
 * also read back for it unless `trusted` is nonzero. */
int dlp_apply_batch_device(dlp_engine* e, const dlp_config* cfg, const dlp_batch* dev_batch,
                           int trusted, dlp_report* reports);
/* engine.apply_batch_structure (engine.py:141-156): deletes, inserts, ground
 * truth; no propagation.  Also used for CPU-baseline state hand-off. */
int dlp_apply_structure(dlp_engine* e, const dlp_batch* batch);
/* baselines.itlp_batch_solve (baselines.py:236-253): structure, then full
 * Jacobi sweeps over alive unlabeled vertices with positive degree. */
int dlp_itlp_batch(dlp_engine* e, const dlp_config* cfg, const dlp_batch* batch,
                   dlp_report* reports);

/* Capacity hint (like std::vector::reserve): size vertex arrays, the edge
 * log and the adjacency pool for n_vertices slots and n_edges live edges so
 * later batches never reallocate.  Optional; growth is otherwise geometric. */
int dlp_reserve(dlp_engine* e, int64_t n_vertices, int64_t n_edges);

/* ---- component sharding ------------------------------
 * Every rank applies the same batches (replicated structure, tau, components,
 * initialisation); each rank propagates only the connected components it
 * owns (a hash of the component's minimum vertex id).  The per-column
 * frontier / certify state machine of engine.py:375-405 runs on phase
 * results reduced over all ranks through the caller's collective: `reduce`
 * must combine imax (elementwise max), isum (sum) and dmax (max) in place
 * across ranks and return 0.  Labels of a vertex live on the rank that last
 * propagated it (dlp_read_owned); reports are the global ones. */
typedef int (*dlp_allreduce_fn)(void* ctx, int64_t* imax, int32_t nimax, int64_t* isum, int32_t nisum, double* dmax,
                                int32_t ndmax);
int dlp_shard_set(dlp_engine* e, int rank, int world);
/* Row partition instead of component sharding (for a single giant component,
 * SURVEY.md §8(e) E-3): rank r evaluates the rows v % world == r; after every
 * global round the evaluated rows (vertex, masks, new labels) are all-gathered
 * through the same callback (isum segments) and each rank applies the others'
 * labels and frontier claims, so every rank holds the whole label matrix.
 * Must be chosen before the first batch. */
/* components: sticky LPT placement by edge count; rows:
 * row partition for one giant component (E-3); components_hash: placement
 * by a hash of the component's root (no balancing) */
enum { DLP_SHARD_COMPONENTS = 0, DLP_SHARD_ROWS = 1, DLP_SHARD_COMPONENTS_HASH = 2 };
int dlp_shard_mode(dlp_engine* e, int mode);
/* NCCL communicator inside the handle: rank 0 creates the
 * 128-byte id, the caller broadcasts it (torch.distributed), every rank
 * attaches; dlp_apply_batch_sharded with reduce = NULL then runs every
 * exchange as an NCCL collective on device buffers on the engine's stream
 * (phase all-reduces, label migration max-reduce, row all-gather). */
int dlp_nccl_unique_id(void* id);
int dlp_shard_nccl(dlp_engine* e, const void* id, int world, int rank);
int dlp_apply_batch_sharded(dlp_engine* e, const dlp_config* cfg, const dlp_batch* batch, dlp_allreduce_fn reduce,
                            void* ctx, dlp_report* reports);
int dlp_read_owned(dlp_engine* e, uint8_t* owned, int64_t n);

/* DynamicGraph.num_slots / num_alive (graph.py:189-192, 182). */
int dlp_num_slots(dlp_engine* e, int64_t* n_slots, int64_t* num_alive);
/* LabelState.f / .gt (labels.py:21-22).  f is [columns][n] row-major; GT
 * vertices read as their pinned class value.  n must equal num_slots. */
int dlp_read_labels(dlp_engine* e, double* f, int8_t* gt, int64_t n);
/* Overwrite f (CPU-baseline hand-off and tests); GT entries are ignored. */
int dlp_write_labels(dlp_engine* e, const double* f, int64_t n);
/* Closed-form harmonic labels of the current graph on the device (dense
 * Cholesky of the free-vertex system, cuSOLVER): replaces
 * baselines.harmonic_solve (dynlp/baselines.py:163-190, harmonic_dense
 * :109-160); stlp=1 adds the short-circuit solve's both-classes check
 * (stlp_reduce, :278-287; same solution).  f: C x n (column c at f + c*n);
 * *unreachable = alive vertices with no path to a ground-truth vertex
 * (pinned to 0.5).  3 when more than dense_cap vertices are free. */
int dlp_harmonic_solve(dlp_engine* e, int stlp, int64_t dense_cap, double* f, int64_t n, int64_t* unreachable);
int dlp_read_alive(dlp_engine* e, uint8_t* alive, int64_t n);
/* eligible mask of the last batch (engine.py:361), before the loop. */
int dlp_read_eligible(dlp_engine* e, uint8_t* eligible, int64_t n);
/* number of live undirected edges and the tau resolved by the last batch */
int dlp_graph_stats(dlp_engine* e, int64_t* live_edges, double* last_tau);
/* DynamicGraph.csr() snapshot (graph.py:218-231): indptr[n+1], indices and
 * weights [nnz = 2 * live_edges], degrees [n] (row-order sums). */
int dlp_read_csr(dlp_engine* e, int64_t* indptr, int64_t* indices, double* weights,
                 double* degrees, int64_t n, int64_t nnz);
/* live_edges() in log order (graph.py:205-216). */
int dlp_read_live_edges(dlp_engine* e, int64_t* u, int64_t* v, double* w, int64_t m);
/* find_components labeling of the last batch (components.py:84-124):
 * vertices (sorted), parent (min member id), component_id (dense). */
int dlp_read_intra(dlp_engine* e, int64_t* vertices, int64_t* parent, int64_t* comp,
                   int64_t cap, int64_t* k);

/* Kernel plugin API: dynlp.kernels (kernels/__init__.py:28-30) with the
 * signatures of kernels/_csr.pyx:61-70, 94-102, 114-125 on HOST arrays. */
int dlp_jacobi_step(const int64_t* indptr, const int64_t* indices, const double* weights,
                    const int8_t* gt, const double* f, int64_t n, const int64_t* frontier,
                    int64_t nf, double* out_vals, double* out_deltas);
int dlp_gauss_seidel_step(const int64_t* indptr, const int64_t* indices, const double* weights,
                          const int8_t* gt, double* f, int64_t n, const int64_t* frontier,
                          int64_t nf, double* out_deltas);
/* leftover (capacity max(n, nf)) is returned sorted ascending. */
int dlp_jacobi_run(const int64_t* indptr, const int64_t* indices, const double* weights,
                   const int8_t* gt, double* f, int64_t n, const int64_t* frontier_init,
                   int64_t nf, uint8_t* eligible, double delta, int64_t max_iters,
                   int64_t* out_iters, int64_t* out_updates, double* out_max_change,
                   int64_t* out_warnings, int64_t* leftover, int64_t* n_leftover);
const char* dlp_plugin_last_error(void);

/* ---- k-NN edge construction (builder.py:18-92) -------------------------
 * Cosine k-NN on tensor cores (fp16 hi/lo split, fp32 accumulation in TMEM)
 * with an exact fp64 re-check and certificate: the selected pairs are those
 * of an exact fp64 selection by (-sim, id); weights are fp64 dot products. */
typedef struct dlp_knn dlp_knn;
int dlp_knn_create(int device, dlp_knn** out);
int dlp_knn_destroy(dlp_knn* h);
const char* dlp_knn_last_error(dlp_knn* h);
/* FeatureMatrix (builder.py:18-39): HOST rows [n][d] fp64; all-zero rows are
 * rejected (status 3, "all-zero feature row i (cosine undefined)"). */
int dlp_knn_set_features(dlp_knn* h, const double* rows, int64_t n, int64_t d);
/* top-k rows of queries [q0, q1) against all n rows (self excluded), each row
 * ordered by (-sim, id): the k-NN rows of a batch of arriving points. */
int dlp_knn_query(dlp_knn* h, int64_t q0, int64_t q1, int32_t k, int64_t* ids, double* sims);
/* knn_graph (builder.py:42-92): union-symmetrised, max-merged, sorted by
 * (lo, hi); affine = 0 for "prune" (w = cos), 1 for "affine" (w = (1+cos)/2). */
int dlp_knn_graph(dlp_knn* h, int32_t k, int32_t affine, int64_t* m_out);
int dlp_knn_read_edges(dlp_knn* h, int64_t* u, int64_t* v, double* w, int64_t m);
/* timings (CUDA events) and certificate fallbacks of the last call */
int dlp_knn_stats(dlp_knn* h, double* screen_ms, double* recheck_ms, double* exact_ms, int64_t* n_fallback,
                  int64_t* n_queries, double* eps);
/* screened candidates of the last dlp_knn_query (tests of the tensor-core stage) */
int dlp_knn_debug_candidates(dlp_knn* h, int64_t q0, int64_t q1, int32_t* nsplit, float* val, int32_t* id,
                             float* thr, int64_t cap);

/* Device / build facts for reports: SM count and whether the sm_100a image
 * is loadable on the current device. */
int dlp_device_info(int device, int* sm_count, int* cc_major, int* cc_minor);

#ifdef __cplusplus
}
#endif
#endif
