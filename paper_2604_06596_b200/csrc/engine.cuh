// engine.cuh -- device-resident state of one DynLP engine and the launchers
// of its per-batch pipeline.
//
// HBM layout (one engine per GPU):
//   per vertex (cap_n slots):   alive u8, gt i8, row_start i64, row_len/up/cap
//                               i32, parent i32 (global union-find),
//                               root_gt u8, mark u8, cnt_up/cnt_dn/grp i32
//   labels:                     f[0][v*C + c] fp64, C = label columns
//                               interleaved per vertex (one gather serves
//                               every column; GT vertices NaN-boxed);
//                               f[1] = staging buffer of the Jacobi round;
//                               eligm[v] u32 = eligible columns bitmask
//   adjacency pool:             nbr i32[pool_cap], w f64[pool_cap]; row v
//                               = [up entries (y > v, insertion order) ++
//                               down entries (y < v, insertion order)] at
//                               row_start[v], capacity row_cap[v] (slack for
//                               up-appends; relocation by bump allocation)
//   edge log:                   lo/hi i32, w f64 -- live edges in insertion
//                               order (the reference's chunk list), input of
//                               the tau pairwise sum
//   frontier machinery:         union frontier lists + per-vertex column
//                               masks (2 rotating each)
#pragma once

#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "../../include/dynlp_b200.h"

namespace dlp {

// Device-side scalars that live across batches.
struct DevState {
    unsigned long long pool_top;  // bump allocator into the adjacency pool
    long long log_n;              // live edge-log length
    long long m_kept;             // merged edges appended by this batch
    long long n_purge;            // rows to purge after deletes
    long long n_touched;          // rows touched by inserts
    long long n_f0;               // initial frontier size
    long long n_elist;            // eligible list size
    long long isolated;           // unreachable & deg 0
    long long unreach;            // unreachable & deg > 0
    long long intra_nc;           // intra-batch component count
    double tau;
    long long log_n_before;
    unsigned long long pool_need;  // relocation space the batch's touched rows need
};

constexpr int kMaxCols = 16;  // label columns handled by the fused LP kernel

// Per-round results of the fused LP kernel (two rotating slots).
struct RoundSlot {
    unsigned long long rmax[kMaxCols];   // max |delta| per column (IEEE bits)
    unsigned long long neval[kMaxCols];  // vertex updates per column
    unsigned long long edges[kMaxCols];  // row entries traversed per column
    unsigned long long warn[kMaxCols];   // isolated sentinels per column
    unsigned long long urows;            // union rows evaluated (all columns at once)
    unsigned long long uentries;         // row entries gathered for them
    unsigned int claimed;                // columns with a non-empty next frontier
    unsigned int grab[3];                // dynamic work counters per row class (short / long / hub)
    unsigned int cnt[3];                 // lengths of the next union frontier lists per class
};

// Control block of the persistent LP kernel (one launch per batch, all columns).
struct LPCtl {
    unsigned int bar;
    unsigned int pad;
    RoundSlot slot[2];
    long long elig_count[kMaxCols];
    unsigned int n_el[3];  // eligible list split by row class (short / long / hub)
    unsigned int n_f0[3];  // initial frontier split
    // outputs per column
    long long iterations[kMaxCols];
    long long updates[kMaxCols];
    long long certs[kMaxCols];
    long long warnings[kMaxCols];
    long long edges[kMaxCols];
    double max_change[kMaxCols];
    long long converged[kMaxCols];
    long long rounds;  // global (lockstep) rounds executed
    long long urows;
    long long uentries;
    // optional per-round trace (DLP_LP_TRACE): {nS, nL, fr|ce<<16, globaltimer}
    unsigned long long* trace;
    long long trace_cap;
    int* seen;               // debug: per-vertex round stamp (duplicate work items)
    unsigned long long* prof; // diagnostics: warp-ns in hub / long / short parts of phase 1
    unsigned long long dups; // debug: duplicate work items detected
    // ---- action mode (component-sharded execution): the host
    // runs each column's engine.py:375-405 state machine on phase results
    // reduced over all shards; a launch executes one action per column.
    int act[kMaxCols];             // ACT_NONE / ACT_FRONTIER / ACT_CERTIFY
    long long budget[kMaxCols];    // round budget of a frontier phase
    int has_fr[kMaxCols];          // column has a (local) frontier in the lists
    long long ph_rounds[kMaxCols]; // rounds executed by the action
    long long ph_upd[kMaxCols];
    long long ph_edges[kMaxCols];
    long long ph_warn[kMaxCols];
    double ph_mc[kMaxCols];        // max |delta| of the action's last round
    long long r_par;               // rounds executed in this batch (list parity)
    unsigned int ncur_p[3];        // frontier list lengths at exit
    int started;                   // prologue done for this batch
    long long log_n;               // row-partitioned mode: work items of the launch's round
};
enum { ACT_NONE = 0, ACT_FRONTIER = 1, ACT_CERTIFY = 2 };

template <typename T>
struct DevArray {
    T* p = nullptr;
    size_t n = 0;
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    // grow to at least `want` elements, preserving the first `keep` elements.
    // Stream-ordered (cudaMallocAsync / cudaFreeAsync on the engine stream,
    // memory pool with an unbounded release threshold): no device-wide sync.
    void reserve(size_t want, size_t keep, cudaStream_t st) {
        if (want <= n) return;
        size_t nn = n ? n : 1024;
        while (nn < want) nn += nn / 2 + 1024;
        T* q = nullptr;
        DLP_CUDA_TRY(cudaMallocAsync((void**)&q, nn * sizeof(T), st));
        if (p && keep) DLP_CUDA_TRY(cudaMemcpyAsync(q, p, keep * sizeof(T), cudaMemcpyDeviceToDevice, st));
        if (p) DLP_CUDA_TRY(cudaFreeAsync(p, st));
        p = q;
        n = nn;
    }
};

template <typename T>
struct PinnedArray {
    T* p = nullptr;
    size_t n = 0;
    std::vector<void*> retired;  // outgrown buffers, freed at release(): cudaFreeHost would
                                 // synchronize the device in the middle of a batch
    void reserve(size_t want) {
        if (want <= n) return;
        if (p) retired.push_back(p);
        size_t nn = want + want / 2 + 1024;
        DLP_CUDA_TRY(cudaMallocHost(&p, nn * sizeof(T)));
        n = nn;
    }
    void release() {
        if (p) cudaFreeHost(p);
        for (void* q : retired) cudaFreeHost(q);
        retired.clear();
        p = nullptr;
        n = 0;
    }
};

struct BatchDev {  // device copies of one batch
    const long long* ids;
    const signed char* gt;
    const long long* owner;
    const long long* other;
    const double* w;
    const long long* dels;
    long long k, ne, nd;
};

struct Engine {
    int device = 0;
    cudaStream_t st = nullptr;
    int sm_count = 148;
    int num_classes = 2;
    int ncol = 1;
    std::string err;

    // host mirror (validation) -----------------------------------------
    std::vector<unsigned char> h_alive;
    long long n_slots = 0, num_alive = 0;
    long long live_edges = 0;  // host copy of log_n after the last batch
    long long cap_n = 0;
    double last_tau = 0.0;
    long long intra_k = 0;
    bool cc_valid = true;  // global union-find consistent with the live graph
    int shard_rank = 0, shard_world = 1;  // component sharding (dlp_shard_set)
    int shard_lpt = 1;   // component placement: 1 = sticky LPT by edge count, 0 = hash of the root
    std::unordered_map<long long, unsigned char> place;  // root -> rank of the last placement
    DevArray<unsigned long long> comp_w, comp_wl;
    DevArray<long long> comp_roots;
    DevArray<unsigned char> comp_own, root_owner;
    int shard_rows = 0;  // 1: row partition (dlp_shard_mode): vertex v is owned by rank v % world
    // row partition: per-round work-item log (vertex, evaluated mask, changed
    // mask; the values are the compact staging Y) and remote rows to apply
    DevArray<int> log_u, rx_u;
    DevArray<unsigned int> log_em, log_chg, rx_em, rx_chg;
    DevArray<double> rx_val;

    // per-vertex ----------------------------------------------------------
    DevArray<unsigned char> alive, mark, root_gt, owner_rank, migr_from;
    DevArray<unsigned char> cc_hit_root, cc_hit;
    DevArray<int> vlen;            // LP view: unlabeled neighbours per row (pool: nbr_sp / wgt_sp)
    DevArray<int> row_mod, view_b; // batch sequence of a row's last change / of its view's build
    DevArray<long long> view_st;   // row_start the view was built at
    int view_seq = 1;              // batch sequence number (advanced per batch with structure)
    int view_inval = 0;            // views built before this sequence are invalid (pool repacked)
    DevArray<double> wsum, q01;    // LP view row constants: w_all; (w0, w1) / w_all per column  // decremental connectivity: hit roots / members
    DevArray<int> migr_flag, migr_pos, migr_list;
    DevArray<double> migr_buf;
    DevArray<int> purge_flag;
    DevArray<signed char> gt;
    DevArray<long long> row_start;
    DevArray<int> row_len, row_up, row_cap, parent, cnt_up, cnt_dn, grp_start;
    DevArray<double> f[2];
    DevArray<double> readout;  // dlp_read_labels: unboxed column-major labels
    DevArray<unsigned int> eligm, emask_store, fmask[2];
    DevArray<int> ulist[2], llist[2], hlist[2], elist_s, elist_l, elist_h, f0, elist, purge_list, touched;
    // adjacency pool ------------------------------------------------------
    DevArray<int> nbr, nbr_sp;      // adjacency pool and its compaction target
    DevArray<double> wgt, wgt_sp;
    long long pool_cap = 0, pool_top_host = 0;
    // edge log ------------------------------------------------------------
    DevArray<int> log_lo, log_hi, log_lo2, log_hi2;
    DevArray<double> log_w, log_w2;
    // batch staging -------------------------------------------------------
    PinnedArray<unsigned char> h_stage, h_stage2;  // batch staging (two slots: ingestion pipeline)
    PinnedArray<double> h_readout;                 // label read-out bounce buffer (pinned: full-speed D2H)
    DevArray<unsigned char> d_stage, d_stage2;
    cudaStream_t cst = nullptr;   // copy stream of the ingestion pipeline
    cudaEvent_t cev = nullptr;    // staged copy complete
    struct Staged {               // next batch validated and copied during the previous batch
        bool valid = false;
        int rc = 0;
        std::string err;
        long long t = 0, k = 0, ne = 0, nd = 0;
        const void* ptrs[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
        std::vector<long long> dels;  // host copy: mirror update when the batch is applied
    } staged;
    // per-batch scratch -----------------------------------------------------
    DevArray<unsigned long long> key_a, key_b;
    DevArray<int> val_a, val_b, flag_i, pos_i;
    DevArray<int> m_lo, m_hi;
    DevArray<double> m_w, ew_lo, ew_hi;  // merged edges (first-occurrence order)
    DevArray<int> mlo_at, mhi_at;
    DevArray<double> mw_at;
    DevArray<int> lpar, comp, comp_sorted_i, root_flag, root_rank, root_tmp;
    DevArray<double> per0, per1, cinit;
    DevArray<unsigned char> cub_tmp;
    DevArray<double> tau_scratch;
    DevState* ds = nullptr;
    PinnedArray<DevState> h_ds;
    LPCtl* ctl = nullptr;
    PinnedArray<LPCtl> h_ctl;
    int lp_grid = 0;
    void* cusolver = nullptr;
    void* nccl = nullptr;      // ncclComm_t of a sharded engine (dlp_shard_nccl), else null
    DevArray<unsigned long long> comm_buf, rows_send, rows_recv;  // NCCL staging (device)  // cusolverDnHandle_t of the harmonic oracle (created on first use)
    int lp_cert_hold = 1 << 30;  // certify alignment: max rounds a certify waits (DLP_CERT_HOLD)
    int l2_mode = 0;            // label L2 residency: 0 none (default: C2 -0.8%, C4 -4% vs 1), 1 persisting carve-out, 2 + access window
    size_t l2_persist = 0;      // persisting L2 carve-out (bytes)
    size_t l2_window_max = 0;
    DevArray<unsigned long long> lp_trace;
    DevArray<int> lp_seen;
    DevArray<unsigned long long> lp_prof;
    const char* lp_trace_path = nullptr;
    size_t lp_smem = 0;
    // instrumentation: kernel launches issued and LP kernel time per column
    long long launches = 0;
    cudaEvent_t lp_ev[2] = {nullptr, nullptr};
    bool host_trace = false;  // DLP_HOST_TRACE: per-phase host timings on stderr
    double host_t0 = 0.0;
};

// graph.cu ------------------------------------------------------------------
void ensure_vertex_capacity(Engine& E, long long want);
void ensure_pool(Engine& E, long long new_edges, long long new_vertices);
void ensure_log(Engine& E, long long want);
void apply_deletes_dev(Engine& E, const BatchDev& b);
void apply_inserts_dev(Engine& E, const BatchDev& b, long long base);
void resolve_tau_dev(Engine& E, double cfg_tau);
void intra_components_dev(Engine& E, const BatchDev& b, long long base);
void init_components_dev(Engine& E, const BatchDev& b, long long base);
// cc: 0 = incremental (union the batch's merged edges), 1 = decremental
// (re-build only the components that lost a vertex, then add the batch's
// edges; dels = the batch's deletes on the device), 2 = full rebuild
void reach_and_pin_dev(Engine& E, int cc, long long n, const long long* dels = nullptr, long long nd = 0);
void compact_pool(Engine& E, long long min_free);
long long migr_collect(Engine& E, long long n);
void migr_pack(Engine& E, long long m, double* dev_buf);
void migr_unpack(Engine& E, long long m, const double* dev_buf);
void host_mark(Engine& E, const char* what);
// lp.cu ---------------------------------------------------------------------
void lp_run_dev(Engine& E, double delta, long long max_iter, bool itlp);
void lp_run_actions(Engine& E, double delta, bool first, bool cleanup);
void lp_rows_apply(Engine& E, long long m, long long r_par);
void lp_setup(Engine& E);
void lp_dump_trace(Engine& E, long long rounds);
// NCCL inside the handle (comm.cu)
int nccl_unique_id(void* out, std::string* err);
int nccl_attach(Engine& E, const void* id, int world, int rank);
void nccl_detach(Engine& E);
int nccl_reduce(void* ctx, int64_t* imax, int32_t nimax, int64_t* isum, int32_t nisum, double* dmax, int32_t ndmax);
int nccl_max_f64(Engine& E, double* d, size_t n);
int nccl_allgather_u64(Engine& E, const unsigned long long* send, unsigned long long* recv, size_t count);
// row-partition record packing on the device (lp.cu)
void rows_pack(Engine& E, long long n, unsigned long long* send, unsigned long long* count);
void rows_unpack(Engine& E, int W, int me, long long mx, const std::vector<unsigned long long>& cnt,
                 const std::vector<long long>& base, const unsigned long long* recv);
// closed-form harmonic labels (harmonic.cu); out_host = C x n_slots
int harmonic_solve_dev(Engine& E, int stlp, long long dense_cap, double* out_host, long long* fallback,
                       std::string* msg);
void itlp_active_dev(Engine& E, long long n);
// readers (graph.cu) ----------------------------------------------------------
void read_csr_dev(Engine& E, long long* indptr, long long* indices, double* weights, double* degrees);

}  // namespace dlp
