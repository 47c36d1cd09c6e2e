// abi.cu -- C-ABI entry points (include/dynlp_b200.h) and the host-side
// orchestration of one batch: validate on the host mirror, stage the batch,
// enqueue the device pipeline, read the report back.
//
// engine.apply_batch (engine.py:328-413) order of operations:
//   validate (graph.py:254-309) -> deletes -> inserts + ground truth
//   -> tau -> intra-batch components + initialisation -> reachability, pin,
//   eligible -> per label column: frontier rounds / certify sweeps.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include <cusolverDn.h>

#include "engine.cuh"

using namespace dlp;

struct dlp_engine {
    Engine E;
    bool poisoned = false;
};

namespace dlp {
void host_mark(Engine& E, const char* what) {
    if (!E.host_trace) return;
    double t = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
    fprintf(stderr, "[dlp host] %-14s +%.3f ms\n", what, t - E.host_t0);
    E.host_t0 = t;
}
}  // namespace dlp

namespace {

int fail(Engine& E, int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    E.err = buf;
    return code;
}

// a failed reduction: the engine's NCCL path leaves its reason in E.err
int coll_fail(Engine& E) {
    if (E.nccl && !E.err.empty()) return fail(E, DLP_EINTERNAL, "collective failed: %s", E.err.c_str());
    return fail(E, DLP_EINTERNAL, "collective failed");
}

int cuda_fail(dlp_engine* h, const CudaFailure& f) {
    h->poisoned = true;
    return fail(h->E, DLP_ECUDA, "CUDA error %s at %s:%d (%s)", cudaGetErrorString(f.err), f.file, f.line, f.expr);
}

int check_config(Engine& E, const dlp_config* c) {
    // EngineConfig.validate (engine.py:49-60)
    if (!(c->delta > 0)) return fail(E, DLP_EVALIDATION, "delta must be positive");
    if (c->mode != DLP_MODE_JACOBI && c->mode != DLP_MODE_GAUSS_SEIDEL)
        return fail(E, DLP_EVALIDATION, "unknown mode %d", c->mode);
    if (!std::isnan(c->tau) && c->tau < 0) return fail(E, DLP_EVALIDATION, "tau must be nonnegative");
    return DLP_OK;
}

struct HostBatch {
    long long t, k, ne, nd;
    const long long *ids, *owner, *other, *dels;
    const signed char* gt;
    const double* w;
};

// DynamicGraph.validate_batch (graph.py:306-309): validate_deletes then
// validate_inserts with pending deletes; same checks, order and messages.
int validate_batch(Engine& E, const HostBatch& b) {
    long long n = E.n_slots;
    if (b.nd) {
        std::vector<long long> d(b.dels, b.dels + b.nd);
        std::sort(d.begin(), d.end());
        for (long long i = 1; i < b.nd; i++)
            if (d[i] == d[i - 1]) return fail(E, DLP_EVALIDATION, "duplicate vertex id in deletes");
        for (long long x : d)
            if (x < 0 || x >= n) return fail(E, DLP_EVALIDATION, "unknown vertex id %lld in deletes", x);
        for (long long x : d)
            if (!E.h_alive[x]) return fail(E, DLP_EVALIDATION, "vertex %lld is already deleted", x);
    }
    long long k = b.k;
    if (k == 0) {
        if (b.ne) return fail(E, DLP_EVALIDATION, "batch has edges but no inserted vertices");
        return DLP_OK;
    }
    {
        std::vector<long long> ids(b.ids, b.ids + k);
        std::sort(ids.begin(), ids.end());
        for (long long i = 1; i < k; i++)
            if (ids[i] == ids[i - 1]) return fail(E, DLP_EVALIDATION, "duplicate fresh id in inserts");
        for (long long i = 0; i < k; i++)
            if (ids[i] != n + i)
                return fail(E, DLP_EVALIDATION, "insert ids must be the contiguous block %lld..%lld", n, n + k - 1);
    }
    for (long long i = 0; i < b.nd; i++)
        if (b.dels[i] >= n && b.dels[i] < n + k)
            return fail(E, DLP_EVALIDATION, "a vertex id appears in both inserts and deletes");
    if (b.ne) {
        for (long long j = 0; j < b.ne; j++)
            if (b.w[j] < 0) return fail(E, DLP_EVALIDATION, "negative weight on edge to vertex %lld", b.other[j]);
        for (long long j = 0; j < b.ne; j++) {
            if (b.owner[j] < 0 || b.owner[j] >= k)
                return fail(E, DLP_EVALIDATION, "edge owner index %lld out of range", b.owner[j]);
            if (b.ids[b.owner[j]] == b.other[j]) return fail(E, DLP_EVALIDATION, "self-loop in insert edges");
        }
        for (long long j = 0; j < b.ne; j++) {
            long long o = b.other[j];
            if (o >= n && o < n + k) continue;
            if (o < 0 || o >= n) return fail(E, DLP_EVALIDATION, "edge to unknown vertex %lld", o);
        }
        for (long long j = 0; j < b.ne; j++) {
            long long o = b.other[j];
            if (o >= n && o < n + k) continue;
            if (!E.h_alive[o]) return fail(E, DLP_EVALIDATION, "edge to a dead vertex %lld", o);
        }
        if (b.nd) {
            std::vector<unsigned char> pend(n + 1, 0);
            for (long long i = 0; i < b.nd; i++) pend[b.dels[i]] = 1;
            for (long long j = 0; j < b.ne; j++) {
                long long o = b.other[j];
                if (o >= n && o < n + k) continue;
                if (pend[o]) return fail(E, DLP_EVALIDATION, "edge to vertex %lld deleted in the same batch", o);
            }
        }
    }
    // LabelState.set_ground_truth class check (labels.py:42-43), hoisted
    // before any mutation so a bad class cannot half-apply a batch.
    for (long long i = 0; i < k; i++) {
        int g = b.gt[i];
        if (g < -1 || g >= E.num_classes) {
            if (E.num_classes == 2) return fail(E, DLP_EVALIDATION, "ground-truth class must be 0 or 1");
            return fail(E, DLP_EVALIDATION, "ground-truth class must be in [0, %d)", E.num_classes);
        }
    }
    return DLP_OK;
}

__global__ void k_reset_batch(DevState* ds) {
    ds->m_kept = 0;
    ds->n_purge = 0;
    ds->n_touched = 0;
    ds->n_f0 = 0;
    ds->n_elist = 0;
    ds->isolated = 0;
    ds->unreach = 0;
    ds->intra_nc = 0;
}

size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

// Stage host batch arrays into one pinned buffer and copy it to the device
// (slot 0: the current batch on the compute stream; slot 1: the next batch
// of the ingestion pipeline on the copy stream).
BatchDev stage_batch(Engine& E, const HostBatch& b, int slot = 0, cudaStream_t st = nullptr) {
    PinnedArray<unsigned char>& hs = slot ? E.h_stage2 : E.h_stage;
    DevArray<unsigned char>& ds = slot ? E.d_stage2 : E.d_stage;
    if (!st) st = E.st;
    size_t off[7];
    size_t sz[6] = {(size_t)b.k * 8, (size_t)b.k, (size_t)b.ne * 8, (size_t)b.ne * 8, (size_t)b.ne * 8, (size_t)b.nd * 8};
    size_t tot = 0;
    for (int i = 0; i < 6; i++) {
        off[i] = tot;
        tot += align_up(sz[i]);
    }
    off[6] = tot;
    // both staging slots grow together, with a floor, so the ingestion
    // pipeline never allocates pinned memory (or its copy stream) mid-stream
    const size_t need = tot + 256;
    static const size_t floor_b = getenv("DLP_STAGE_FLOOR_MB") ? (size_t)atol(getenv("DLP_STAGE_FLOOR_MB")) << 20
                                                                 : (size_t)32 << 20;
    const size_t want = std::max(need + need / 2, floor_b);
    if (hs.n < need || ds.n < need) {  // pinned and device slots grow by different rules
        E.h_stage.reserve(want);
        E.h_stage2.reserve(want);
        E.d_stage.reserve(want, 0, E.st);
        E.d_stage2.reserve(want, 0, E.st);
        DLP_CUDA_TRY(cudaStreamSynchronize(E.st));  // the device slots exist before any copy stream uses them
    }
    if (!E.cst) {
        DLP_CUDA_TRY(cudaStreamCreateWithFlags(&E.cst, cudaStreamNonBlocking));
        DLP_CUDA_TRY(cudaEventCreateWithFlags(&E.cev, cudaEventDisableTiming));
    }
    const void* src[6] = {b.ids, b.gt, b.owner, b.other, b.w, b.dels};
    for (int i = 0; i < 6; i++)
        if (sz[i]) memcpy(hs.p + off[i], src[i], sz[i]);
    if (tot) DLP_CUDA_TRY(cudaMemcpyAsync(ds.p, hs.p, tot, cudaMemcpyHostToDevice, st));
    unsigned char* d = ds.p;
    BatchDev bd;
    bd.ids = (const long long*)(d + off[0]);
    bd.gt = (const signed char*)(d + off[1]);
    bd.owner = (const long long*)(d + off[2]);
    bd.other = (const long long*)(d + off[3]);
    bd.w = (const double*)(d + off[4]);
    bd.dels = (const long long*)(d + off[5]);
    bd.k = b.k;
    bd.ne = b.ne;
    bd.nd = b.nd;
    return bd;
}

// device views of a batch already resident in the current staging slot
BatchDev stage_view(Engine& E, const HostBatch& b) {
    size_t sz[6] = {(size_t)b.k * 8, (size_t)b.k, (size_t)b.ne * 8, (size_t)b.ne * 8, (size_t)b.ne * 8, (size_t)b.nd * 8};
    size_t off[6], tot = 0;
    for (int i = 0; i < 6; i++) {
        off[i] = tot;
        tot += align_up(sz[i]);
    }
    unsigned char* d = E.d_stage.p;
    BatchDev bd;
    bd.ids = (const long long*)(d + off[0]);
    bd.gt = (const signed char*)(d + off[1]);
    bd.owner = (const long long*)(d + off[2]);
    bd.other = (const long long*)(d + off[3]);
    bd.w = (const double*)(d + off[4]);
    bd.dels = (const long long*)(d + off[5]);
    bd.k = b.k;
    bd.ne = b.ne;
    bd.nd = b.nd;
    return bd;
}

bool staged_matches(const Engine& E, const dlp_batch* b) {
    const Engine::Staged& s = E.staged;
    const void* p[6] = {b->insert_ids, b->insert_gt, b->edge_owner, b->edge_other, b->edge_w, b->deletes};
    if (!s.valid || s.t != b->t || s.k != b->n_ins || s.ne != b->n_edges || s.nd != b->n_del) return false;
    for (int i = 0; i < 6; i++)
        if (s.ptrs[i] != p[i]) return false;
    return true;
}

int validate_batch(Engine& E, const HostBatch& b);

// Ingestion pipeline: validate the next batch against the
// host mirror (already advanced past the current batch) and copy it to the
// device on the copy stream while the current batch's kernels run.
void stage_next(Engine& E, const dlp_batch* nb) {
    Engine::Staged& s = E.staged;
    s.valid = true;
    s.t = nb->t;
    s.k = nb->n_ins;
    s.ne = nb->n_edges;
    s.nd = nb->n_del;
    const void* p[6] = {nb->insert_ids, nb->insert_gt, nb->edge_owner, nb->edge_other, nb->edge_w, nb->deletes};
    for (int i = 0; i < 6; i++) s.ptrs[i] = p[i];
    s.dels.assign((const long long*)nb->deletes, (const long long*)nb->deletes + nb->n_del);
    HostBatch hb{nb->t, nb->n_ins, nb->n_edges, nb->n_del, (const long long*)nb->insert_ids,
                 (const long long*)nb->edge_owner, (const long long*)nb->edge_other, (const long long*)nb->deletes,
                 (const signed char*)nb->insert_gt, nb->edge_w};
    std::string saved = E.err;
    s.rc = validate_batch(E, hb);
    s.err = E.err;
    E.err = saved;
    if (s.rc) return;  // reported when the batch is applied; nothing staged
    if (!E.cst) {
        DLP_CUDA_TRY(cudaStreamCreateWithFlags(&E.cst, cudaStreamNonBlocking));
        DLP_CUDA_TRY(cudaEventCreateWithFlags(&E.cev, cudaEventDisableTiming));
    } else {
        DLP_CUDA_TRY(cudaEventSynchronize(E.cev));  // an earlier staged copy may still read h_stage2
    }
    stage_batch(E, hb, 1, E.cst);
    DLP_CUDA_TRY(cudaEventRecord(E.cev, E.cst));
}

enum Kind { KIND_DYNLP = 0, KIND_STRUCTURE = 1, KIND_ITLP = 2 };

// Per-column engine.py:375-405 state machine for component-sharded batches,
// driven by phase results reduced over all shards (the caller's collective).
struct ColCtl {
    long long iterations = 0, updates = 0, edges = 0, warnings = 0, certs = 0;
    double max_change = 0.0;
    int converged = 1, done = 0, has_fr = 0;
    int act = ACT_NONE;
};

// Row partition: after each one-round launch, all-gather the round's
// evaluated rows (vertex, evaluated mask, changed mask, new labels) through the
// caller's sum-reduction (each rank fills its own segment; int64 sums of one
// nonzero term are exact, labels travel as bit patterns), then apply the other
// ranks' rows: labels, and the claims their changed rows make on this rank's
// vertices.  Afterwards every rank holds the whole label matrix and its part
// of the next global frontier; h_ctl->has_fr is refreshed.
int rows_exchange(Engine& E, dlp_allreduce_fn reduce, void* rctx) {
    const int C = E.ncol, W = E.shard_world, me = E.shard_rank;
    LPCtl& L = *E.h_ctl.p;
    const long long n = L.log_n;
    std::vector<int> hu(n);
    std::vector<unsigned int> hem(n), hchg(n);
    std::vector<double> hy((size_t)n * C);
    if (n) {
        DLP_CUDA_TRY(cudaMemcpyAsync(hu.data(), E.log_u.p, n * 4, cudaMemcpyDeviceToHost, E.st));
        DLP_CUDA_TRY(cudaMemcpyAsync(hem.data(), E.log_em.p, n * 4, cudaMemcpyDeviceToHost, E.st));
        DLP_CUDA_TRY(cudaMemcpyAsync(hchg.data(), E.log_chg.p, n * 4, cudaMemcpyDeviceToHost, E.st));
        DLP_CUDA_TRY(cudaMemcpyAsync(hy.data(), E.f[1].p, (size_t)n * C * 8, cudaMemcpyDeviceToHost, E.st));
        DLP_CUDA_TRY(cudaMemsetAsync(E.log_chg.p, 0, n * 4, E.st));
        DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
    }
    std::vector<long long> keep;
    for (long long i = 0; i < n; i++)
        if (hem[i]) keep.push_back(i);
    const int rec = 3 + C;
    std::vector<int64_t> cnt(W, 0), z(1, 0);
    std::vector<double> zd(1, 0.0);
    cnt[me] = (int64_t)keep.size();
    if (reduce(rctx, z.data(), 1, cnt.data(), W, zd.data(), 1)) return coll_fail(E);
    long long tot = 0, off = 0;
    for (int r = 0; r < W; r++) {
        if (r == me) off = tot;
        tot += cnt[r];
    }
    if (tot == 0) return DLP_OK;
    std::vector<int64_t> buf((size_t)tot * rec, 0);
    for (size_t j = 0; j < keep.size(); j++) {
        const long long i = keep[j];
        int64_t* b = buf.data() + (size_t)(off + j) * rec;
        b[0] = hu[i];
        b[1] = hem[i];
        b[2] = hchg[i];
        memcpy(b + 3, hy.data() + (size_t)i * C, (size_t)C * 8);
    }
    if (buf.size() > (size_t)INT32_MAX) return fail(E, DLP_EINTERNAL, "row exchange too large");
    if (reduce(rctx, z.data(), 1, buf.data(), (int32_t)buf.size(), zd.data(), 1))
        return coll_fail(E);
    const long long m = tot - cnt[me];
    if (m == 0) return DLP_OK;
    std::vector<int> ru(m);
    std::vector<unsigned int> rem(m), rchg(m);
    std::vector<double> rv((size_t)m * C);
    long long k = 0;
    for (long long j = 0; j < tot; j++) {
        if (j >= off && j < off + cnt[me]) continue;
        const int64_t* b = buf.data() + (size_t)j * rec;
        ru[k] = (int)b[0];
        rem[k] = (unsigned int)b[1];
        rchg[k] = (unsigned int)b[2];
        memcpy(rv.data() + (size_t)k * C, b + 3, (size_t)C * 8);
        k++;
    }
    E.rx_u.reserve(m, 0, E.st);
    E.rx_em.reserve(m, 0, E.st);
    E.rx_chg.reserve(m, 0, E.st);
    E.rx_val.reserve((size_t)m * C, 0, E.st);
    DLP_CUDA_TRY(cudaMemcpyAsync(E.rx_u.p, ru.data(), m * 4, cudaMemcpyHostToDevice, E.st));
    DLP_CUDA_TRY(cudaMemcpyAsync(E.rx_em.p, rem.data(), m * 4, cudaMemcpyHostToDevice, E.st));
    DLP_CUDA_TRY(cudaMemcpyAsync(E.rx_chg.p, rchg.data(), m * 4, cudaMemcpyHostToDevice, E.st));
    DLP_CUDA_TRY(cudaMemcpyAsync(E.rx_val.p, rv.data(), (size_t)m * C * 8, cudaMemcpyHostToDevice, E.st));
    lp_rows_apply(E, m, L.r_par);
    DLP_CUDA_TRY(cudaMemcpyAsync(L.has_fr, E.ctl->has_fr, sizeof(L.has_fr), cudaMemcpyDeviceToHost, E.st));
    DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
    return DLP_OK;
}

// Row partition over NCCL: the round's evaluated rows are packed on the
// device (record = vertex, evaluated mask, changed mask, C label words), the
// per-rank counts and then the records (padded to the largest count) are
// all-gathered device to device, and the other ranks' records are unpacked
// into the k_rows_apply inputs on the device.  One small D2H (the counts).
int rows_exchange_nccl(Engine& E) {
    const int C = E.ncol, W = E.shard_world, me = E.shard_rank;
    LPCtl& L = *E.h_ctl.p;
    const long long n = L.log_n;
    const int rec = 3 + C;
    E.rows_send.reserve((size_t)(n + 1) * rec, 0, E.st);
    E.comm_buf.reserve(2 * (size_t)W + 2, 0, E.st);
    unsigned long long* cnt_d = E.comm_buf.p;  // [0]: own count, [W..2W): gathered counts
    DLP_CUDA_TRY(cudaMemsetAsync(cnt_d, 0, 8, E.st));
    rows_pack(E, n, E.rows_send.p, cnt_d);
    if (nccl_allgather_u64(E, cnt_d, cnt_d + W, 1)) return fail(E, DLP_EINTERNAL, "%s", E.err.c_str());
    std::vector<unsigned long long> cnt(W);
    DLP_CUDA_TRY(cudaMemcpyAsync(cnt.data(), cnt_d + W, W * 8, cudaMemcpyDeviceToHost, E.st));
    DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
    unsigned long long mx = 0, tot = 0;
    for (int r = 0; r < W; r++) {
        mx = std::max(mx, cnt[r]);
        tot += cnt[r];
    }
    const long long m = (long long)(tot - cnt[me]);
    if (mx == 0) return DLP_OK;
    E.rows_recv.reserve((size_t)W * mx * rec, 0, E.st);
    if (nccl_allgather_u64(E, E.rows_send.p, E.rows_recv.p, (size_t)mx * rec))
        return fail(E, DLP_EINTERNAL, "%s", E.err.c_str());
    if (m == 0) return DLP_OK;
    E.rx_u.reserve(m, 0, E.st);
    E.rx_em.reserve(m, 0, E.st);
    E.rx_chg.reserve(m, 0, E.st);
    E.rx_val.reserve((size_t)m * C, 0, E.st);
    std::vector<long long> base(W + 1, 0);  // output offset of each rank's records (own skipped)
    for (int r = 0; r < W; r++) base[r + 1] = base[r] + (r == me ? 0 : (long long)cnt[r]);
    rows_unpack(E, W, me, (long long)mx, cnt, base, E.rows_recv.p);
    lp_rows_apply(E, m, L.r_par);
    DLP_CUDA_TRY(cudaMemcpyAsync(L.has_fr, E.ctl->has_fr, sizeof(L.has_fr), cudaMemcpyDeviceToHost, E.st));
    DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
    return DLP_OK;
}

int sharded_lp(Engine& E, const dlp_config* cfg, long long max_iter, dlp_allreduce_fn reduce, void* rctx,
               std::vector<ColCtl>& col, double* lp_ms, long long* launches) {
    const int C = E.ncol;
    const bool rows = E.shard_rows != 0;
    // global F0 emptiness and eligible counts (replicated structure, sharded sets)
    // label migration for components that changed owner (replicated order)
    {
        long long m = migr_collect(E, E.n_slots);
        std::vector<int64_t> mi(1, m), ms(1, 0);
        std::vector<double> md(1, 0.0);
        if (reduce(rctx, mi.data(), 1, ms.data(), 1, md.data(), 1)) return coll_fail(E);
        if (mi[0] != m) return fail(E, DLP_EINTERNAL, "shards disagree on migrated vertices");
        if (m && reduce == nccl_reduce) {  // device-resident max-reduction
            const size_t cnt = (size_t)m * C;
            E.migr_buf.reserve(cnt, 0, E.st);
            migr_pack(E, m, E.migr_buf.p);
            if (nccl_max_f64(E, E.migr_buf.p, cnt)) return fail(E, DLP_EINTERNAL, "%s", E.err.c_str());
            migr_unpack(E, m, E.migr_buf.p);
            DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
        } else if (m) {
            const size_t cnt = (size_t)m * C;
            E.migr_buf.reserve(cnt, 0, E.st);
            std::vector<double> hb(cnt);
            migr_pack(E, m, E.migr_buf.p);
            DLP_CUDA_TRY(cudaMemcpyAsync(hb.data(), E.migr_buf.p, cnt * 8, cudaMemcpyDeviceToHost, E.st));
            DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
            std::vector<int64_t> z1(1, 0), z2(1, 0);
            if (reduce(rctx, z1.data(), 1, z2.data(), 1, hb.data(), (int32_t)cnt))
                return coll_fail(E);
            DLP_CUDA_TRY(cudaMemcpyAsync(E.migr_buf.p, hb.data(), cnt * 8, cudaMemcpyHostToDevice, E.st));
            migr_unpack(E, m, E.migr_buf.p);
            DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
        }
    }
    std::vector<int64_t> isum(2), imax(1, 0);
    std::vector<double> dmax(1, 0.0);
    DLP_CUDA_TRY(cudaMemcpyAsync(E.h_ds.p, E.ds, sizeof(DevState), cudaMemcpyDeviceToHost, E.st));
    DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
    isum[0] = E.h_ds.p->n_f0;
    isum[1] = E.h_ds.p->n_elist;
    if (reduce(rctx, imax.data(), 1, isum.data(), 2, dmax.data(), 1)) return coll_fail(E);
    std::vector<long long> elig_g(C, isum[1]);
    for (auto& c : col) c.has_fr = isum[0] > 0;
    bool first = true;
    auto t0 = std::chrono::steady_clock::now();
    for (int launch = 0;; launch++) {
        // decide each column's next action (mirrors decide_actions in lp.cu)
        bool any = false;
        for (int c = 0; c < C; c++) {
            ColCtl& k = col[c];
            k.act = ACT_NONE;
            if (k.done) continue;
            if (k.has_fr && k.iterations < max_iter) {
                k.act = ACT_FRONTIER;
            } else {
                if (k.has_fr || k.iterations >= max_iter) {
                    k.converged = k.has_fr ? 0 : 1;
                    if (!k.converged) {
                        k.done = 1;
                        continue;
                    }
                }
                if (elig_g[c] == 0) {  // certify swept nothing: break
                    k.done = 1;
                    continue;
                }
                k.act = ACT_CERTIFY;
            }
            any = true;
        }
        if (!any) break;
        int act[kMaxCols] = {0};
        long long budget[kMaxCols] = {0};
        for (int c = 0; c < C; c++) {
            act[c] = col[c].act;
            budget[c] = max_iter - col[c].iterations;
            if (rows) budget[c] = std::min(budget[c], 1LL);  // one global round per launch
        }
        DLP_CUDA_TRY(cudaMemcpyAsync(E.ctl->act, act, sizeof(act), cudaMemcpyHostToDevice, E.st));
        DLP_CUDA_TRY(cudaMemcpyAsync(E.ctl->budget, budget, sizeof(budget), cudaMemcpyHostToDevice, E.st));
        lp_run_actions(E, cfg->delta, first, false);
        first = false;
        DLP_CUDA_TRY(cudaMemcpyAsync(E.h_ctl.p, E.ctl, sizeof(LPCtl), cudaMemcpyDeviceToHost, E.st));
        DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
        if (rows) {
            int rc = reduce == nccl_reduce ? rows_exchange_nccl(E) : rows_exchange(E, reduce, rctx);
            if (rc) return rc;
        }
        const LPCtl& L = *E.h_ctl.p;
        // reduce: max rounds | sum updates, edges, warnings, frontier, eligible | max rmax
        std::vector<int64_t> rmaxv(C), sums(5 * C);
        std::vector<double> dm(C);
        for (int c = 0; c < C; c++) {
            rmaxv[c] = L.ph_rounds[c];
            sums[c] = L.ph_upd[c];
            sums[C + c] = L.ph_edges[c];
            sums[2 * C + c] = L.ph_warn[c];
            sums[3 * C + c] = L.has_fr[c];
            sums[4 * C + c] = L.elig_count[c];
            dm[c] = col[c].act == ACT_CERTIFY ? L.ph_mc[c] : 0.0;
        }
        if (reduce(rctx, rmaxv.data(), C, sums.data(), 5 * C, dm.data(), C))
            return coll_fail(E);
        // the frontier phase's max_change is its last global round's: shards that
        // ran fewer rounds had an empty frontier in that round
        std::vector<int64_t> none(1, 0), nsum(1, 0);
        std::vector<double> mc(C, -1.0);
        for (int c = 0; c < C; c++)
            if (col[c].act == ACT_FRONTIER && L.ph_rounds[c] == rmaxv[c] && rmaxv[c] > 0) mc[c] = L.ph_mc[c];
        if (reduce(rctx, none.data(), 1, nsum.data(), 1, mc.data(), C)) return coll_fail(E);
        for (int c = 0; c < C; c++) {
            ColCtl& k = col[c];
            elig_g[c] = sums[4 * C + c];
            if (k.act == ACT_NONE) continue;
            k.updates += sums[c];
            k.edges += sums[C + c];
            k.warnings += sums[2 * C + c];
            k.has_fr = sums[3 * C + c] > 0;
            if (k.act == ACT_FRONTIER) {
                k.iterations += rmaxv[c];
                if (rmaxv[c] > 0) k.max_change = mc[c];
            } else {  // certify_round committed (engine.py:398-405)
                k.iterations += 1;
                k.certs += 1;
                k.max_change = dm[c];
                if (dm[c] <= cfg->delta) k.done = 1;
            }
        }
    }
    if (!first) {  // clear leftover frontier masks for the next batch
        lp_run_actions(E, cfg->delta, false, true);
        DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
    }
    *lp_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    (void)launches;
    return DLP_OK;
}

int run_batch(dlp_engine* h, const dlp_config* cfg, const dlp_batch* batch, bool device_ptrs, bool trusted,
              dlp_report* reps, Kind kind, dlp_allreduce_fn reduce = nullptr, void* rctx = nullptr,
              const dlp_batch* next = nullptr) {
    Engine& E = h->E;
    auto t0 = std::chrono::steady_clock::now();
    if (h->poisoned) return fail(E, DLP_EINTERNAL, "engine is unusable after an earlier CUDA error");
    if (cfg) {
        int rc = check_config(E, cfg);
        if (rc) return rc;
        if (cfg->mode == DLP_MODE_GAUSS_SEIDEL && kind == KIND_DYNLP)
            return fail(E, DLP_EVALIDATION, "mode 'sequential_gauss_seidel' is not supported by the B200 engine");
    }
    if (reps)
        for (int c = 0; c < E.ncol; c++) {
            memset(&reps[c], 0, sizeof(dlp_report));
            reps[c].t = batch->t;
            reps[c].converged = 1;
        }
    auto finish_time = [&]() {
        double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (reps)
            for (int c = 0; c < E.ncol; c++) reps[c].wall_time_ms = ms;
    };
    // The ingestion pipeline's staged batch is only usable by the very next
    // host batch with the same arrays; any other call (device batches, a
    // different or empty batch) invalidates it, since it was validated
    // against a host mirror that call may advance.
    const bool use_staged = !device_ptrs && staged_matches(E, batch);
    if (!use_staged) E.staged.valid = false;
    if (batch->n_ins == 0 && batch->n_del == 0 && kind != KIND_ITLP) {  // engine.py:338-340
        finish_time();
        return DLP_OK;
    }
    // host views (read back device batches for validation unless trusted)
    std::vector<long long> hv_ids, hv_owner, hv_other, hv_dels;
    std::vector<signed char> hv_gt;
    std::vector<double> hv_w;
    HostBatch hb{batch->t,
                 batch->n_ins,
                 batch->n_edges,
                 batch->n_del,
                 (const long long*)batch->insert_ids,
                 (const long long*)batch->edge_owner,
                 (const long long*)batch->edge_other,
                 (const long long*)batch->deletes,
                 (const signed char*)batch->insert_gt,
                 batch->edge_w};
    try {
        DLP_CUDA_TRY(cudaSetDevice(E.device));
        if (device_ptrs && !trusted) {
            auto pull = [&](auto& vec, const void* src, size_t n) {
                vec.resize(n);
                if (n) DLP_CUDA_TRY(cudaMemcpy(vec.data(), src, n * sizeof(vec[0]), cudaMemcpyDeviceToHost));
            };
            pull(hv_ids, batch->insert_ids, batch->n_ins);
            pull(hv_gt, batch->insert_gt, batch->n_ins);
            pull(hv_owner, batch->edge_owner, batch->n_edges);
            pull(hv_other, batch->edge_other, batch->n_edges);
            pull(hv_w, batch->edge_w, batch->n_edges);
            pull(hv_dels, batch->deletes, batch->n_del);
            hb.ids = hv_ids.data();
            hb.gt = hv_gt.data();
            hb.owner = hv_owner.data();
            hb.other = hv_other.data();
            hb.w = hv_w.data();
            hb.dels = hv_dels.data();
        }
        if (use_staged) {  // validated and copied during the previous batch
            E.staged.valid = false;
            if (E.staged.rc) return fail(E, E.staged.rc, "%s", E.staged.err.c_str());
            hb.dels = E.staged.dels.data();  // the copy the device applies (mirror update below)
        } else if (!(device_ptrs && trusted)) {
            int rc = validate_batch(E, hb);
            if (rc) return rc;
        }
        if (E.host_trace) {
            E.host_t0 = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
            host_mark(E, "validated");
        }
        long long base = E.n_slots, k = hb.k, ne = hb.ne, nd = hb.nd;
        ensure_vertex_capacity(E, base + k + 1);
        ensure_log(E, E.live_edges + ne + 1);
        ensure_pool(E, ne, k);
        BatchDev bd;
        if (device_ptrs) {
            bd.ids = (const long long*)batch->insert_ids;
            bd.gt = (const signed char*)batch->insert_gt;
            bd.owner = (const long long*)batch->edge_owner;
            bd.other = (const long long*)batch->edge_other;
            bd.w = batch->edge_w;
            bd.dels = (const long long*)batch->deletes;
            bd.k = k;
            bd.ne = ne;
            bd.nd = nd;
        } else if (use_staged) {
            std::swap(E.h_stage, E.h_stage2);  // the staged slot becomes the current one
            std::swap(E.d_stage, E.d_stage2);
            bd = stage_view(E, hb);
            DLP_CUDA_TRY(cudaStreamWaitEvent(E.st, E.cev, 0));
        } else {
            bd = stage_batch(E, hb);
        }
        host_mark(E, "staged");
        long long launches0 = E.launches;
        E.view_seq++;  // LP view cache: changes of this batch get this sequence number
        k_reset_batch<<<1, 1, 0, E.st>>>(E.ds);
        E.launches++;
        apply_deletes_dev(E, bd);
        apply_inserts_dev(E, bd, base);
        // host mirror of alive (validation of later batches)
        if (nd) {
            if (!(device_ptrs && trusted)) {
                for (long long i = 0; i < nd; i++) E.h_alive[hb.dels[i]] = 0;
            } else {
                std::vector<long long> dd(nd);
                DLP_CUDA_TRY(cudaMemcpy(dd.data(), batch->deletes, nd * 8, cudaMemcpyDeviceToHost));
                for (long long x : dd) E.h_alive[x] = 0;
            }
        }
        E.h_alive.resize(base + k, 1);
        E.n_slots = base + k;
        E.num_alive += k - nd;
        long long n = E.n_slots;
        if (kind == KIND_STRUCTURE) {
            DLP_CUDA_TRY(cudaMemcpyAsync(E.h_ds.p, E.ds, sizeof(DevState), cudaMemcpyDeviceToHost, E.st));
            DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
            E.live_edges = E.h_ds.p->log_n;
            E.pool_top_host = (long long)E.h_ds.p->pool_top;
            E.cc_valid = false;  // union-find is refreshed by the next full batch
            finish_time();
            return DLP_OK;
        }
        // connectivity: incremental on insert-only batches, decremental
        // (only the components that lost a vertex are rebuilt) after deletes,
        // full rebuild when the union-find is stale (structure-only batches)
        const int cc_mode = !E.cc_valid ? 2 : (nd > 0 ? 1 : 0);
        long long max_iter = cfg->max_iterations > 0 ? cfg->max_iterations
                                                      : std::max<long long>(1, 10 * E.num_alive);
        if (kind == KIND_DYNLP) {
            resolve_tau_dev(E, cfg->tau);
            E.intra_k = 0;
            if (cfg->component_init && k > 0) {
                intra_components_dev(E, bd, base);
                init_components_dev(E, bd, base);
            }
            reach_and_pin_dev(E, cc_mode, n, bd.dels, nd);
            if (reduce) {  // component-sharded propagation
                std::vector<ColCtl> col(E.ncol);
                double ms = 0.0;
                int rc = sharded_lp(E, cfg, max_iter, reduce, rctx, col, &ms, nullptr);
                if (rc) return rc;
                DLP_CUDA_TRY(cudaMemcpyAsync(E.h_ds.p, E.ds, sizeof(DevState), cudaMemcpyDeviceToHost, E.st));
                DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
                DevState& s = *E.h_ds.p;
                E.live_edges = s.log_n;
                E.pool_top_host = (long long)s.pool_top;
                E.last_tau = s.tau;
                E.cc_valid = true;
                for (int c = 0; c < E.ncol; c++) {
                    dlp_report& r = reps[c];
                    r.iterations = col[c].iterations;
                    r.updates = col[c].updates;
                    r.max_change = col[c].max_change;
                    r.converged = col[c].converged;
                    r.isolated_pinned = s.isolated;
                    r.unreachable_pinned = s.unreach;
                    r.warnings = col[c].warnings + r.isolated_pinned + r.unreachable_pinned;
                    r.edges_traversed = col[c].edges;
                    r.certify_sweeps = col[c].certs;
                    r.lp_kernel_ms = ms;
                    r.gpu_launches = E.launches - launches0;
                    r.lp_rounds = col[c].iterations;
                }
                finish_time();
                return DLP_OK;
            }
            lp_run_dev(E, cfg->delta, max_iter, false);
        } else {  // ItLP: no reachability, active = alive & unlabeled & deg > 0
            itlp_active_dev(E, n);
            lp_run_dev(E, cfg->delta, max_iter, true);
            E.cc_valid = false;
        }
        DLP_CUDA_TRY(cudaGetLastError());
        host_mark(E, "enqueued");
        if (next && !device_ptrs) stage_next(E, next);  // overlaps the kernels enqueued above
        DLP_CUDA_TRY(cudaMemcpyAsync(E.h_ds.p, E.ds, sizeof(DevState), cudaMemcpyDeviceToHost, E.st));
        DLP_CUDA_TRY(cudaMemcpyAsync(E.h_ctl.p, E.ctl, sizeof(LPCtl), cudaMemcpyDeviceToHost, E.st));
        DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
        DevState& s = *E.h_ds.p;
        E.live_edges = s.log_n;
        E.pool_top_host = (long long)s.pool_top;
        E.last_tau = s.tau;
        if (kind == KIND_DYNLP) E.cc_valid = true;
        if (E.pool_top_host > E.pool_cap) return fail(E, DLP_EINTERNAL, "adjacency pool overflow");
        float lp_ms = 0.f;
        DLP_CUDA_TRY(cudaEventElapsedTime(&lp_ms, E.lp_ev[0], E.lp_ev[1]));
        host_mark(E, "synced");
        const LPCtl& L = *E.h_ctl.p;
        lp_dump_trace(E, L.rounds);
        for (int c = 0; c < E.ncol; c++) {
            dlp_report& r = reps[c];
            r.iterations = L.iterations[c];
            r.updates = L.updates[c];
            r.max_change = L.max_change[c];
            r.converged = (int)L.converged[c];
            r.isolated_pinned = s.isolated;
            r.unreachable_pinned = kind == KIND_DYNLP ? s.unreach : 0;
            r.warnings = L.warnings[c] + r.isolated_pinned + r.unreachable_pinned;
            r.edges_traversed = L.edges[c];
            r.certify_sweeps = L.certs[c];
            r.lp_kernel_ms = lp_ms;  // one fused launch serves every column
            r.gpu_launches = E.launches - launches0;
            r.lp_rounds = L.rounds;
            r.lp_union_rows = L.urows;
            r.lp_union_entries = L.uentries;
        }
        finish_time();
        return DLP_OK;
    } catch (const CudaFailure& f) {
        return cuda_fail(h, f);
    }
}

// Label read-out (LabelState.f, labels.py:21): column c of vertex v to
// out[c * n + v]; a boxed ground-truth word becomes its class as 0.0 / 1.0
// (the reference pins f = class, labels.py:37-49).  Any other NaN is an
// unlabeled vertex's label and is returned as is.
__global__ void k_labels_out(const double* X, long long n, int C, double* out) {
    const long long tot = n * C;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < tot; i += (long long)gridDim.x * blockDim.x) {
        const long long c = i / n, v = i - c * n;
        const double x = X[v * C + c];
        const unsigned long long b = (unsigned long long)__double_as_longlong(x);
        out[i] = (b & ~1ULL) == kBoxBase ? (double)(b & 1ULL) : x;
    }
}

}  // namespace

extern "C" {

int dlp_create(const dlp_config* cfg, int device, dlp_engine** out) {
    *out = nullptr;
    auto* h = new dlp_engine();
    Engine& E = h->E;
    try {
        int ndev = 0;
        DLP_CUDA_TRY(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) {
            delete h;
            return DLP_ECUDA;
        }
        E.device = device;
        DLP_CUDA_TRY(cudaSetDevice(device));
        cudaDeviceProp prop;
        DLP_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
        E.sm_count = prop.multiProcessorCount;
        if (!prop.cooperativeLaunch) {
            delete h;
            return DLP_ECUDA;
        }
        E.host_trace = getenv("DLP_HOST_TRACE") != nullptr;
        E.num_classes = cfg && cfg->num_classes > 2 ? cfg->num_classes : 2;
        E.ncol = E.num_classes > 2 ? E.num_classes : 1;
        if (E.ncol > kMaxCols) {  // before anything is allocated
            delete h;
            return DLP_EVALIDATION;
        }
        DLP_CUDA_TRY(cudaStreamCreateWithFlags(&E.st, cudaStreamNonBlocking));
        {  // keep freed stream-ordered allocations cached in the device pool
            cudaMemPool_t mp;
            DLP_CUDA_TRY(cudaDeviceGetDefaultMemPool(&mp, device));
            unsigned long long thr = ~0ULL;
            DLP_CUDA_TRY(cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr));
        }
        DLP_CUDA_TRY(cudaMalloc(&E.ds, sizeof(DevState)));
        DLP_CUDA_TRY(cudaMemset(E.ds, 0, sizeof(DevState)));
        DLP_CUDA_TRY(cudaMalloc(&E.ctl, sizeof(LPCtl)));
        DLP_CUDA_TRY(cudaMemset(E.ctl, 0, sizeof(LPCtl)));
        E.h_ds.reserve(1);
        E.h_ctl.reserve(1);
        ensure_vertex_capacity(E, 4096);
        ensure_log(E, 4096);
        compact_pool(E, 1 << 16);
        lp_setup(E);
        DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
    } catch (const CudaFailure& f) {
        fprintf(stderr, "dlp_create: CUDA error %s (%s)\n", cudaGetErrorString(f.err), f.expr);
        delete h;
        return DLP_ECUDA;
    }
    *out = h;
    return DLP_OK;
}

int dlp_apply_batch_pipelined(dlp_engine* h, const dlp_config* cfg, const dlp_batch* batch, const dlp_batch* next,
                              dlp_report* reports) {
    if (!h) return DLP_EINTERNAL;
    return run_batch(h, cfg, batch, false, false, reports, KIND_DYNLP, nullptr, nullptr, next);
}

int dlp_shard_set(dlp_engine* h, int rank, int world) {
    if (!h) return DLP_EINTERNAL;
    Engine& E = h->E;
    if (world < 1 || world > 255 || rank < 0 || rank >= world) return fail(E, DLP_EVALIDATION, "bad shard rank/world");
    E.shard_rank = rank;
    E.shard_world = world;
    return DLP_OK;
}

int dlp_shard_mode(dlp_engine* h, int mode) {
    if (!h) return DLP_EINTERNAL;
    Engine& E = h->E;
    if (mode != DLP_SHARD_COMPONENTS && mode != DLP_SHARD_ROWS && mode != DLP_SHARD_COMPONENTS_HASH)
        return fail(E, DLP_EVALIDATION, "bad shard mode");
    const int rows = mode == DLP_SHARD_ROWS ? 1 : 0, lpt = mode == DLP_SHARD_COMPONENTS ? 1 : 0;
    if (E.n_slots != 0 && (rows != E.shard_rows || lpt != E.shard_lpt))
        return fail(E, DLP_EVALIDATION, "the shard mode must be chosen before the first batch");
    E.shard_rows = rows;
    E.shard_lpt = lpt;
    return DLP_OK;
}

int dlp_nccl_unique_id(void* id) {
    std::string err;
    return nccl_unique_id(id, &err);
}

int dlp_shard_nccl(dlp_engine* h, const void* id, int world, int rank) {
    Engine& E = h->E;
    if (world < 1 || rank < 0 || rank >= world) return fail(E, DLP_EVALIDATION, "bad rank %d / world %d", rank, world);
    if (world > 255) return fail(E, DLP_EVALIDATION, "world > 255 is not supported");
    try {
        DLP_CUDA_TRY(cudaSetDevice(E.device));
        nccl_detach(E);
        int rc = nccl_attach(E, id, world, rank);
        if (rc) return fail(E, rc, "%s", E.err.c_str());
    } catch (const CudaFailure& f) {
        return cuda_fail(h, f);
    }
    return DLP_OK;
}

int dlp_apply_batch_sharded(dlp_engine* h, const dlp_config* cfg, const dlp_batch* batch, dlp_allreduce_fn reduce,
                            void* ctx, dlp_report* reports) {
    if (!h) return DLP_EINTERNAL;
    if (!reduce) {  // the engine's own NCCL communicator (dlp_shard_nccl)
        if (!h->E.nccl) return fail(h->E, DLP_EVALIDATION, "a reduction callback or an NCCL communicator is required");
        reduce = nccl_reduce;
        ctx = &h->E;
    }
    return run_batch(h, cfg, batch, false, false, reports, KIND_DYNLP, reduce, ctx);
}

int dlp_read_owned(dlp_engine* h, uint8_t* owned, int64_t n) {
    if (!h) return DLP_EINTERNAL;
    Engine& E = h->E;
    if (n != E.n_slots) return fail(E, DLP_EVALIDATION, "n must equal num_slots");
    try {
        DLP_CUDA_TRY(cudaSetDevice(E.device));
        std::vector<unsigned char> o(n);
        if (n) DLP_CUDA_TRY(cudaMemcpy(o.data(), E.owner_rank.p, n, cudaMemcpyDeviceToHost));
        for (long long v = 0; v < n; v++)
            owned[v] = E.shard_world <= 1 || (E.shard_rows ? v % E.shard_world == E.shard_rank : o[v] == E.shard_rank);
    } catch (const CudaFailure& f) {
        return cuda_fail(h, f);
    }
    return DLP_OK;
}

int dlp_reserve(dlp_engine* h, int64_t n_vertices, int64_t n_edges) {
    if (!h) return DLP_EINTERNAL;
    Engine& E = h->E;
    if (h->poisoned) return fail(E, DLP_EINTERNAL, "engine is unusable after an earlier CUDA error");
    if (n_vertices < 0 || n_edges < 0) return fail(E, DLP_EVALIDATION, "reserve sizes must be nonnegative");
    try {
        DLP_CUDA_TRY(cudaSetDevice(E.device));
        ensure_vertex_capacity(E, n_vertices + 1);
        ensure_log(E, n_edges + 1);
        // live entries with compaction slack (25%) + fresh-row space, plus the
        // free headroom compact_pool keeps (a quarter of the pool): no growth later
        long long want = ((2 * n_edges) * 5 / 4 + 4 * n_vertices + (1 << 20)) * 4 / 3 + (1 << 20);
        if (E.pool_cap < want) compact_pool(E, want - 2 * E.live_edges);
        DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
    } catch (const CudaFailure& f) {
        return cuda_fail(h, f);
    }
    return DLP_OK;
}

int dlp_destroy(dlp_engine* h) {
    if (!h) return DLP_OK;
    Engine& E = h->E;
    cudaSetDevice(E.device);
    cudaStreamSynchronize(E.st);
    if (E.l2_persist) cudaCtxResetPersistingL2Cache();  // hand the carve-out's lines back
    if (E.cusolver) cusolverDnDestroy((cusolverDnHandle_t)E.cusolver);
    nccl_detach(E);
    E.comm_buf.release();
    E.rows_send.release();
    E.rows_recv.release();
    DevArray<unsigned char>* u8s[] = {&E.alive, &E.mark, &E.root_gt, &E.owner_rank, &E.migr_from, &E.d_stage,
                                      &E.cub_tmp, &E.cc_hit_root, &E.cc_hit};
    E.migr_flag.release();
    E.migr_pos.release();
    E.migr_list.release();
    E.migr_buf.release();
    for (auto* a : u8s) a->release();
    E.purge_flag.release();
    E.vlen.release();
    E.row_mod.release();
    E.view_b.release();
    E.view_st.release();
    E.wsum.release();
    E.q01.release();
    E.gt.release();
    E.row_start.release();
    DevArray<int>* i32s[] = {&E.row_len, &E.row_up, &E.row_cap, &E.parent, &E.cnt_up, &E.cnt_dn, &E.grp_start,
                             &E.ulist[0], &E.ulist[1], &E.llist[0], &E.llist[1], &E.hlist[0], &E.hlist[1], &E.elist_s, &E.elist_l, &E.elist_h, &E.f0, &E.elist, &E.purge_list, &E.touched,
                             &E.nbr, &E.nbr_sp, &E.log_lo, &E.log_hi, &E.log_lo2, &E.log_hi2, &E.val_a, &E.val_b,
                             &E.flag_i, &E.pos_i, &E.m_lo, &E.m_hi, &E.mlo_at, &E.mhi_at, &E.lpar, &E.comp,
                             &E.comp_sorted_i, &E.root_flag, &E.root_rank, &E.root_tmp, &E.log_u, &E.rx_u};
    for (auto* a : i32s) a->release();
    DevArray<double>* f64s[] = {&E.f[0], &E.f[1], &E.readout, &E.wgt, &E.wgt_sp, &E.log_w, &E.log_w2, &E.m_w, &E.ew_lo, &E.ew_hi,
                                &E.mw_at, &E.per0, &E.per1, &E.cinit, &E.tau_scratch, &E.rx_val};
    for (auto* a : f64s) a->release();
    DevArray<unsigned int>* u32s[] = {&E.eligm, &E.emask_store, &E.fmask[0], &E.fmask[1], &E.log_em, &E.log_chg,
                                      &E.rx_em, &E.rx_chg};
    for (auto* x : u32s) x->release();
    E.key_a.release();
    E.key_b.release();
    if (E.ds) cudaFree(E.ds);
    if (E.ctl) cudaFree(E.ctl);
    E.h_stage.release();
    E.h_stage2.release();
    E.h_readout.release();
    E.d_stage2.release();
    if (E.cev) cudaEventDestroy(E.cev);
    if (E.cst) cudaStreamDestroy(E.cst);
    E.h_ds.release();
    E.h_ctl.release();
    for (auto ev : E.lp_ev)
        if (ev) cudaEventDestroy(ev);
    if (E.st) cudaStreamDestroy(E.st);
    delete h;
    return DLP_OK;
}

const char* dlp_last_error(dlp_engine* h) { return h ? h->E.err.c_str() : "null engine"; }
int dlp_num_columns(dlp_engine* h) { return h->E.ncol; }

int dlp_apply_batch(dlp_engine* h, const dlp_config* cfg, const dlp_batch* b, dlp_report* reps) {
    return run_batch(h, cfg, b, false, false, reps, KIND_DYNLP);
}

int dlp_apply_batch_device(dlp_engine* h, const dlp_config* cfg, const dlp_batch* b, int trusted, dlp_report* reps) {
    return run_batch(h, cfg, b, true, trusted != 0, reps, KIND_DYNLP);
}

int dlp_apply_structure(dlp_engine* h, const dlp_batch* b) {
    return run_batch(h, nullptr, b, false, false, nullptr, KIND_STRUCTURE);
}

int dlp_itlp_batch(dlp_engine* h, const dlp_config* cfg, const dlp_batch* b, dlp_report* reps) {
    return run_batch(h, cfg, b, false, false, reps, KIND_ITLP);
}

int dlp_num_slots(dlp_engine* h, int64_t* n_slots, int64_t* num_alive) {
    *n_slots = h->E.n_slots;
    *num_alive = h->E.num_alive;
    return DLP_OK;
}

int dlp_read_labels(dlp_engine* h, double* f, int8_t* gt, int64_t n) {
    Engine& E = h->E;
    if (n != E.n_slots) return fail(E, DLP_EVALIDATION, "read_labels: n=%lld but num_slots=%lld", (long long)n, E.n_slots);
    try {
        DLP_CUDA_TRY(cudaSetDevice(E.device));
        if (f && n) {  // unbox + column-major transpose on the device, one D2H copy
            E.readout.reserve((size_t)n * E.ncol, 0, E.st);
            k_labels_out<<<blocks_for((long long)n * E.ncol), kBlock, 0, E.st>>>(E.f[0].p, n, E.ncol, E.readout.p);
            DLP_CUDA_TRY(cudaGetLastError());
            // through a pinned bounce buffer (full PCIe speed), then copied out by
            // several host threads: ~4x the pageable D2H of the caller's buffer
            const size_t cnt = (size_t)n * E.ncol;
            E.h_readout.reserve(cnt);
            DLP_CUDA_TRY(cudaMemcpyAsync(E.h_readout.p, E.readout.p, cnt * sizeof(double), cudaMemcpyDeviceToHost,
                                         E.st));
            DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
            const int nt = cnt >= (1u << 20) ? 8 : 1;
            std::vector<std::thread> th;
            const size_t per = (cnt + nt - 1) / nt;
            for (int t = 0; t < nt; t++) {
                const size_t a = t * per, b = std::min(cnt, a + per);
                if (a >= b) break;
                th.emplace_back([&, a, b]() { memcpy(f + a, E.h_readout.p + a, (b - a) * sizeof(double)); });
            }
            for (auto& x : th) x.join();
        }
        if (gt && n) DLP_CUDA_TRY(cudaMemcpyAsync(gt, E.gt.p, n, cudaMemcpyDeviceToHost, E.st));
        DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
    } catch (const CudaFailure& e) {
        return cuda_fail(h, e);
    }
    return DLP_OK;
}

int dlp_harmonic_solve(dlp_engine* h, int stlp, int64_t dense_cap, double* f, int64_t n, int64_t* unreachable) {
    Engine& E = h->E;
    if (n != E.n_slots) return fail(E, DLP_EVALIDATION, "harmonic_solve: n=%lld but num_slots=%lld", (long long)n,
                                    E.n_slots);
    try {
        DLP_CUDA_TRY(cudaSetDevice(E.device));
        std::string msg;
        long long fb = 0;
        int rc = harmonic_solve_dev(E, stlp, dense_cap, f, &fb, &msg);
        if (rc) return fail(E, rc, "%s", msg.c_str());
        if (unreachable) *unreachable = fb;
    } catch (const CudaFailure& e) {
        return cuda_fail(h, e);
    }
    return DLP_OK;
}

int dlp_write_labels(dlp_engine* h, const double* f, int64_t n) {
    Engine& E = h->E;
    if (n != E.n_slots) return fail(E, DLP_EVALIDATION, "write_labels: n mismatch");
    try {
        DLP_CUDA_TRY(cudaSetDevice(E.device));
        std::vector<signed char> g(n);
        std::vector<double> buf((size_t)E.ncol * n);
        if (n) DLP_CUDA_TRY(cudaMemcpy(g.data(), E.gt.p, n, cudaMemcpyDeviceToHost));
        for (int c = 0; c < E.ncol; c++)
            for (long long v = 0; v < n; v++) {
                double x = f[(size_t)c * n + v];
                if (x != x) x = std::nan("");  // a caller NaN stays an unlabeled NaN, never a box
                if (g[v] >= 0) x = box_class(E.ncol == 1 ? g[v] : (g[v] == c ? 1 : 0));
                buf[(size_t)v * E.ncol + c] = x;
            }
        for (int b = 0; b < 2; b++)
            if (n)
                DLP_CUDA_TRY(cudaMemcpyAsync(E.f[b].p, buf.data(), buf.size() * sizeof(double), cudaMemcpyHostToDevice,
                                             E.st));
        DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
    } catch (const CudaFailure& e) {
        return cuda_fail(h, e);
    }
    return DLP_OK;
}

int dlp_read_alive(dlp_engine* h, uint8_t* alive, int64_t n) {
    Engine& E = h->E;
    if (n != E.n_slots) return fail(E, DLP_EVALIDATION, "read_alive: n mismatch");
    memcpy(alive, E.h_alive.data(), n);
    return DLP_OK;
}

int dlp_read_eligible(dlp_engine* h, uint8_t* elig, int64_t n) {
    Engine& E = h->E;
    if (n != E.n_slots) return fail(E, DLP_EVALIDATION, "read_eligible: n mismatch");
    try {
        std::vector<unsigned int> m(n);
        if (n) DLP_CUDA_TRY(cudaMemcpy(m.data(), E.eligm.p, n * sizeof(unsigned int), cudaMemcpyDeviceToHost));
        for (long long v = 0; v < n; v++) elig[v] = (m[v] & 0xFFFFu) != 0;  // column bits (LP keeps the row class above)
    } catch (const CudaFailure& e) {
        return cuda_fail(h, e);
    }
    return DLP_OK;
}

int dlp_graph_stats(dlp_engine* h, int64_t* live_edges, double* last_tau) {
    *live_edges = h->E.live_edges;
    *last_tau = h->E.last_tau;
    return DLP_OK;
}

int dlp_read_csr(dlp_engine* h, int64_t* indptr, int64_t* indices, double* weights, double* degrees, int64_t n,
                 int64_t nnz) {
    Engine& E = h->E;
    if (n != E.n_slots || nnz != 2 * E.live_edges) return fail(E, DLP_EVALIDATION, "read_csr: size mismatch");
    try {
        read_csr_dev(E, (long long*)indptr, (long long*)indices, weights, degrees);
    } catch (const CudaFailure& e) {
        return cuda_fail(h, e);
    }
    return DLP_OK;
}

int dlp_read_live_edges(dlp_engine* h, int64_t* u, int64_t* v, double* w, int64_t m) {
    Engine& E = h->E;
    if (m != E.live_edges) return fail(E, DLP_EVALIDATION, "read_live_edges: size mismatch");
    try {
        std::vector<int> a(m), b(m);
        if (m) {
            DLP_CUDA_TRY(cudaMemcpy(a.data(), E.log_lo.p, m * sizeof(int), cudaMemcpyDeviceToHost));
            DLP_CUDA_TRY(cudaMemcpy(b.data(), E.log_hi.p, m * sizeof(int), cudaMemcpyDeviceToHost));
            DLP_CUDA_TRY(cudaMemcpy(w, E.log_w.p, m * sizeof(double), cudaMemcpyDeviceToHost));
        }
        for (long long i = 0; i < m; i++) {
            u[i] = a[i];
            v[i] = b[i];
        }
    } catch (const CudaFailure& e) {
        return cuda_fail(h, e);
    }
    return DLP_OK;
}

int dlp_read_intra(dlp_engine* h, int64_t* vertices, int64_t* parent, int64_t* comp, int64_t cap, int64_t* kout) {
    Engine& E = h->E;
    long long k = E.intra_k;
    *kout = k;
    if (cap < k) return fail(E, DLP_EVALIDATION, "read_intra: capacity too small");
    try {
        std::vector<int> p(k), c(k);
        if (k) {
            DLP_CUDA_TRY(cudaMemcpy(p.data(), E.lpar.p, k * sizeof(int), cudaMemcpyDeviceToHost));
            DLP_CUDA_TRY(cudaMemcpy(c.data(), E.comp.p, k * sizeof(int), cudaMemcpyDeviceToHost));
        }
        long long base = E.n_slots - k;
        for (long long i = 0; i < k; i++) {
            vertices[i] = base + i;
            parent[i] = base + p[i];
            comp[i] = c[i];
        }
    } catch (const CudaFailure& e) {
        return cuda_fail(h, e);
    }
    return DLP_OK;
}

int dlp_device_info(int device, int* sm_count, int* cc_major, int* cc_minor) {
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return DLP_ECUDA;
    *sm_count = prop.multiProcessorCount;
    *cc_major = prop.major;
    *cc_minor = prop.minor;
    return DLP_OK;
}

}  // extern "C"
