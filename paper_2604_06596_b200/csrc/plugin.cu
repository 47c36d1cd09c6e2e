// plugin.cu -- the reference's kernel plugin API (dynlp.kernels) on the GPU.
//
// jacobi_step       kernels/_csr.pyx:61-91   (evaluate, do not commit)
// gauss_seidel_step kernels/_csr.pyx:94-111  (sequential, in place)
// jacobi_run        kernels/_csr.pyx:114-197 (fused frontier loop; every
//                   round on the device in one cooperative launch)
//
// These operate on a caller-supplied CSR (int64 indptr/indices, fp64
// weights, int8 gt) exactly as the reference backend does, so the
// reference's own kernel tests can run against this backend.  The engine's
// hot loop lives in lp.cu; this file favours exactness of the serial commit
// order over speed: in jacobi_run a vertex the serial commit loop would have
// dropped from `eligible` (isolated sentinel) before a neighbour expands
// into it is rejected by comparing frontier positions (iso_first).
#include <algorithm>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "../../include/dynlp_b200.h"

namespace dlp {

static thread_local std::string g_plugin_err;

__device__ inline double plug_eval(const long long* indptr, const long long* indices, const double* weights,
                                   const signed char* gt, const double* f, long long u, double* val) {
    double fu = f[u];
    RowAcc acc;
    acc.init();
    for (long long e = indptr[u]; e < indptr[u + 1]; e++) {
        long long v = indices[e];
        int g = gt[v];
        acc.add(weights[e], g == 0 ? 0 : (g == 1 ? 1 : -1), f[v], fu);
    }
    return acc.finish(fu, val);
}

__global__ void k_plug_step(const long long* indptr, const long long* indices, const double* weights,
                            const signed char* gt, const double* f, const long long* fr, long long nf, double* vals,
                            double* deltas, long long* iso_first) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nf; i += (long long)gridDim.x * blockDim.x) {
        long long u = fr[i];
        double v;
        double d = plug_eval(indptr, indices, weights, gt, f, u, &v);
        vals[i] = v;
        deltas[i] = d;
        if (iso_first && d < 0.0) atomicMin((unsigned long long*)&iso_first[u], (unsigned long long)i);
    }
}

__global__ void k_plug_gs(const long long* indptr, const long long* indices, const double* weights,
                          const signed char* gt, double* f, const long long* fr, long long nf, double* deltas) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    for (long long i = 0; i < nf; i++) {
        long long u = fr[i];
        double v;
        deltas[i] = plug_eval(indptr, indices, weights, gt, f, u, &v);
        f[u] = v;
    }
}

__device__ inline void plug_claim(int* in_next, long long* nxt, unsigned long long* cnt, long long v) {
    if (atomicExch(&in_next[v], 1) != 0) return;
    cooperative_groups::coalesced_group g = cooperative_groups::coalesced_threads();
    unsigned long long base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(cnt, (unsigned long long)g.size());
    base = g.shfl(base, 0);
    nxt[base + g.thread_rank()] = v;
}

struct PlugCtl {
    unsigned long long next;
    unsigned long long rmax;
    unsigned long long warnings;
};

// jacobi_run as ONE cooperative launch: the rounds of _csr.pyx:155-194 run
// on the device (step, commit, post separated by grid barriers; the round
// bookkeeping is done by thread 0 of block 0 between them), so the host
// neither synchronises nor launches per round.  Same kernels' bodies as the
// per-round launches above.
struct PlugRun {
    PlugCtl ctl;                 // per-round counters (reset every round)
    long long cur_len, iterations, updates;
    unsigned long long warnings;
    double max_change;
    int parity;                  // which list holds the current frontier
    unsigned int bar;            // grid barrier
};

__global__ void k_plug_run(const long long* indptr, const long long* indices, const double* weights,
                           const signed char* gt, double* f, unsigned char* elig, long long* iso, int* in_next,
                           long long* la, long long* lb, double* vals, double* dels, PlugRun* R, double delta,
                           long long max_iters, long long n) {
    unsigned int target = 0;
    const long long gtid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long gth = (long long)gridDim.x * blockDim.x;
    for (;;) {
        const long long cur_len = *(volatile long long*)&R->cur_len;
        const long long it = *(volatile long long*)&R->iterations;
        if (cur_len <= 0 || it >= max_iters) break;
        const int par = *(volatile int*)&R->parity;
        long long* cur = par ? lb : la;
        long long* nxt = par ? la : lb;
        for (long long i = gtid; i < cur_len; i += gth) {  // evaluate (k_plug_step)
            const long long u = cur[i];
            double v;
            const double d = plug_eval(indptr, indices, weights, gt, f, u, &v);
            vals[i] = v;
            dels[i] = d;
            if (d < 0.0) atomicMin((unsigned long long*)&iso[u], (unsigned long long)i);
        }
        grid_sync(&R->bar, target);
        double lmax = 0.0;  // commit + expand (k_plug_commit)
        for (long long i = gtid; i < cur_len; i += gth) {
            const long long u = cur[i];
            const double d = dels[i];
            f[u] = vals[i];
            if (d < 0.0) {
                atomicAdd(&R->ctl.warnings, 1ULL);
                continue;
            }
            lmax = fmax(lmax, d);
            if (d > delta) {
                if (elig[u] && iso[u] > i) plug_claim(in_next, nxt, &R->ctl.next, u);
                for (long long e = indptr[u]; e < indptr[u + 1]; e++) {
                    const long long v = indices[e];
                    if (elig[v] && iso[v] > i) plug_claim(in_next, nxt, &R->ctl.next, v);
                }
            }
        }
        if (lmax > 0.0) atomic_max_nonneg(&R->ctl.rmax, lmax);
        grid_sync(&R->bar, target);
        const long long nn = (long long)*(volatile unsigned long long*)&R->ctl.next;  // post (k_plug_post)
        for (long long i = gtid; i < cur_len; i += gth) {
            if (dels[i] < 0.0) {
                const long long u = cur[i];
                elig[u] = 0;
                iso[u] = 0x7fffffffffffffffLL;
            }
        }
        for (long long i = gtid; i < nn; i += gth) in_next[nxt[i]] = 0;
        grid_sync(&R->bar, target);
        if (gtid == 0) {  // round bookkeeping (the host loop's, _csr.pyx:192-194)
            R->updates += cur_len;
            R->iterations += 1;
            union { unsigned long long u; double d; } cv;
            cv.u = R->ctl.rmax;
            R->max_change = cv.d;
            R->warnings += R->ctl.warnings;
            R->parity ^= 1;
            R->cur_len = nn;
            R->ctl.next = 0;
            R->ctl.rmax = 0;
            R->ctl.warnings = 0;
        }
        grid_sync(&R->bar, target);
    }
    (void)n;
}

__global__ void k_fill_ll(long long* p, long long n, long long v) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = v;
}

template <typename T>
struct Tmp {
    T* p = nullptr;
    cudaStream_t st;
    Tmp(size_t n, cudaStream_t s) : st(s) { DLP_CUDA_TRY(cudaMallocAsync(&p, (n ? n : 1) * sizeof(T), s)); }
    ~Tmp() { cudaFreeAsync(p, st); }
    Tmp(const Tmp&) = delete;
};

template <typename T>
static Tmp<T>* upload(const T* h, size_t n, cudaStream_t st) {
    auto* t = new Tmp<T>(n, st);
    if (n) DLP_CUDA_TRY(cudaMemcpyAsync(t->p, h, n * sizeof(T), cudaMemcpyHostToDevice, st));
    return t;
}

}  // namespace dlp

using namespace dlp;

static int plugin_fail(const char* msg) {
    g_plugin_err = msg;
    return DLP_ECUDA;
}

extern "C" const char* dlp_plugin_last_error(void) { return g_plugin_err.c_str(); }

extern "C" int dlp_jacobi_step(const int64_t* indptr, const int64_t* indices, const double* weights, const int8_t* gt,
                               const double* f, int64_t n, const int64_t* frontier, int64_t nf, double* out_vals,
                               double* out_deltas) {
    try {
        cudaStream_t st = cudaStreamPerThread;
        long long nnz = indptr[n];
        std::unique_ptr<Tmp<long long>> d_ip(upload((const long long*)indptr, n + 1, st));
        std::unique_ptr<Tmp<long long>> d_ix(upload((const long long*)indices, nnz, st));
        std::unique_ptr<Tmp<double>> d_w(upload(weights, nnz, st));
        std::unique_ptr<Tmp<signed char>> d_gt(upload((const signed char*)gt, n, st));
        std::unique_ptr<Tmp<double>> d_f(upload(f, n, st));
        std::unique_ptr<Tmp<long long>> d_fr(upload((const long long*)frontier, nf, st));
        Tmp<double> vals(nf, st), dels(nf, st);
        if (nf)
            k_plug_step<<<blocks_for(nf), kBlock, 0, st>>>(d_ip->p, d_ix->p, d_w->p, d_gt->p, d_f->p, d_fr->p, nf,
                                                            vals.p, dels.p, nullptr);
        if (nf) {
            DLP_CUDA_TRY(cudaMemcpyAsync(out_vals, vals.p, nf * sizeof(double), cudaMemcpyDeviceToHost, st));
            DLP_CUDA_TRY(cudaMemcpyAsync(out_deltas, dels.p, nf * sizeof(double), cudaMemcpyDeviceToHost, st));
        }
        DLP_CUDA_TRY(cudaStreamSynchronize(st));
        DLP_CUDA_TRY(cudaGetLastError());
        return DLP_OK;
    } catch (const CudaFailure& e) {
        return plugin_fail(cudaGetErrorString(e.err));
    }
}

extern "C" int dlp_gauss_seidel_step(const int64_t* indptr, const int64_t* indices, const double* weights,
                                     const int8_t* gt, double* f, int64_t n, const int64_t* frontier, int64_t nf,
                                     double* out_deltas) {
    try {
        cudaStream_t st = cudaStreamPerThread;
        long long nnz = indptr[n];
        std::unique_ptr<Tmp<long long>> d_ip(upload((const long long*)indptr, n + 1, st));
        std::unique_ptr<Tmp<long long>> d_ix(upload((const long long*)indices, nnz, st));
        std::unique_ptr<Tmp<double>> d_w(upload(weights, nnz, st));
        std::unique_ptr<Tmp<signed char>> d_gt(upload((const signed char*)gt, n, st));
        std::unique_ptr<Tmp<double>> d_f(upload((const double*)f, n, st));
        std::unique_ptr<Tmp<long long>> d_fr(upload((const long long*)frontier, nf, st));
        Tmp<double> dels(nf, st);
        k_plug_gs<<<1, 32, 0, st>>>(d_ip->p, d_ix->p, d_w->p, d_gt->p, d_f->p, d_fr->p, nf, dels.p);
        if (n) DLP_CUDA_TRY(cudaMemcpyAsync(f, d_f->p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
        if (nf) DLP_CUDA_TRY(cudaMemcpyAsync(out_deltas, dels.p, nf * sizeof(double), cudaMemcpyDeviceToHost, st));
        DLP_CUDA_TRY(cudaStreamSynchronize(st));
        DLP_CUDA_TRY(cudaGetLastError());
        return DLP_OK;
    } catch (const CudaFailure& e) {
        return plugin_fail(cudaGetErrorString(e.err));
    }
}

extern "C" int dlp_jacobi_run(const int64_t* indptr, const int64_t* indices, const double* weights, const int8_t* gt,
                              double* f, int64_t n, const int64_t* frontier_init, int64_t nf, uint8_t* eligible,
                              double delta, int64_t max_iters, int64_t* out_iters, int64_t* out_updates,
                              double* out_max_change, int64_t* out_warnings, int64_t* leftover,
                              int64_t* n_leftover) {
    try {
        cudaStream_t st = cudaStreamPerThread;
        long long nnz = indptr[n];
        long long lcap = std::max<long long>(n, nf) + 1;
        std::unique_ptr<Tmp<long long>> d_ip(upload((const long long*)indptr, n + 1, st));
        std::unique_ptr<Tmp<long long>> d_ix(upload((const long long*)indices, nnz, st));
        std::unique_ptr<Tmp<double>> d_w(upload(weights, nnz, st));
        std::unique_ptr<Tmp<signed char>> d_gt(upload((const signed char*)gt, n, st));
        std::unique_ptr<Tmp<double>> d_f(upload((const double*)f, n, st));
        std::unique_ptr<Tmp<unsigned char>> d_el(upload((const unsigned char*)eligible, n, st));
        Tmp<long long> la(lcap, st), lb(lcap, st), iso(n + 1, st);
        Tmp<double> vals(lcap, st), dels(lcap, st);
        Tmp<int> in_next(n + 1, st);
        DLP_CUDA_TRY(cudaMemsetAsync(in_next.p, 0, (n + 1) * sizeof(int), st));
        k_fill_ll<<<blocks_for(n + 1), kBlock, 0, st>>>(iso.p, n + 1, 0x7fffffffffffffffLL);
        if (nf) DLP_CUDA_TRY(cudaMemcpyAsync(la.p, frontier_init, nf * sizeof(long long), cudaMemcpyHostToDevice, st));
        // the whole loop on the device: one cooperative launch
        Tmp<PlugRun> run(1, st);
        PlugRun h0{};
        h0.cur_len = nf;
        DLP_CUDA_TRY(cudaMemcpyAsync(run.p, &h0, sizeof(PlugRun), cudaMemcpyHostToDevice, st));
        static int grid = 0;
        if (!grid) {
            int dev = 0, sms = 0, occ = 0;
            DLP_CUDA_TRY(cudaGetDevice(&dev));
            DLP_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            DLP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_plug_run, kBlock, 0));
            grid = sms * std::max(1, std::min(occ, 4));
        }
        long long max_it = max_iters;
        double dl = delta;
        long long nn = n;
        long long *ip = d_ip->p, *ix = d_ix->p, *isop = iso.p, *lap = la.p, *lbp = lb.p;
        double *wp = d_w->p, *fp = d_f->p, *vp = vals.p, *dp = dels.p;
        signed char* gp = d_gt->p;
        unsigned char* ep = d_el->p;
        int* inp = in_next.p;
        PlugRun* rp = run.p;
        void* args[] = {&ip, &ix, &wp, &gp, &fp, &ep, &isop, &inp, &lap, &lbp, &vp, &dp, &rp, &dl, &max_it, &nn};
        DLP_CUDA_TRY(cudaLaunchCooperativeKernel((void*)k_plug_run, dim3(grid), dim3(kBlock), args, 0, st));
        PlugRun h{};
        DLP_CUDA_TRY(cudaMemcpyAsync(&h, run.p, sizeof(PlugRun), cudaMemcpyDeviceToHost, st));
        DLP_CUDA_TRY(cudaStreamSynchronize(st));
        const long long cur_len = h.cur_len, iterations = h.iterations, updates = h.updates;
        const double max_change = h.max_change;
        const unsigned long long warnings = h.warnings;
        long long* cur = h.parity ? lb.p : la.p;
        std::vector<long long> left(cur_len);
        if (cur_len) DLP_CUDA_TRY(cudaMemcpyAsync(left.data(), cur, cur_len * sizeof(long long), cudaMemcpyDeviceToHost, st));
        if (n) {
            DLP_CUDA_TRY(cudaMemcpyAsync(f, d_f->p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
            DLP_CUDA_TRY(cudaMemcpyAsync(eligible, d_el->p, n, cudaMemcpyDeviceToHost, st));
        }
        DLP_CUDA_TRY(cudaStreamSynchronize(st));
        DLP_CUDA_TRY(cudaGetLastError());
        std::sort(left.begin(), left.end());
        for (long long i = 0; i < cur_len; i++) leftover[i] = left[i];
        *n_leftover = cur_len;
        *out_iters = iterations;
        *out_updates = updates;
        *out_max_change = max_change;
        *out_warnings = (int64_t)warnings;
        return DLP_OK;
    } catch (const CudaFailure& e) {
        return plugin_fail(cudaGetErrorString(e.err));
    }
}
