// plugin.cu -- the reference's kernel plugin API (dynlp.kernels) on the GPU.
//
// jacobi_step       kernels/_csr.pyx:61-91   (evaluate, do not commit)
// gauss_seidel_step kernels/_csr.pyx:94-111  (sequential, in place)
// jacobi_run        kernels/_csr.pyx:114-197 (fused frontier loop)
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

__global__ void k_plug_commit(const long long* indptr, const long long* indices, const long long* cur, long long ncur,
                              const double* vals, const double* deltas, double* f, const unsigned char* elig,
                              const long long* iso_first, int* in_next, long long* nxt, PlugCtl* ctl, double delta) {
    double lmax = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ncur; i += (long long)gridDim.x * blockDim.x) {
        long long u = cur[i];
        double d = deltas[i];
        f[u] = vals[i];
        if (d < 0.0) {
            atomicAdd(&ctl->warnings, 1ULL);
            continue;
        }
        lmax = fmax(lmax, d);
        if (d > delta) {
            if (elig[u] && iso_first[u] > i) plug_claim(in_next, nxt, &ctl->next, u);
            for (long long e = indptr[u]; e < indptr[u + 1]; e++) {
                long long v = indices[e];
                if (elig[v] && iso_first[v] > i) plug_claim(in_next, nxt, &ctl->next, v);
            }
        }
    }
    if (lmax > 0.0) atomic_max_nonneg(&ctl->rmax, lmax);
}

__global__ void k_plug_post(const long long* cur, long long ncur, const double* deltas, unsigned char* elig,
                            long long* iso_first, const long long* nxt, const PlugCtl* ctl, int* in_next) {
    long long nn = (long long)ctl->next;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < ncur; i += (long long)gridDim.x * blockDim.x) {
        if (deltas[i] < 0.0) {
            long long u = cur[i];
            elig[u] = 0;
            iso_first[u] = 0x7fffffffffffffffLL;
        }
    }
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nn; i += (long long)gridDim.x * blockDim.x)
        in_next[nxt[i]] = 0;
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
        Tmp<PlugCtl> ctl(1, st);
        DLP_CUDA_TRY(cudaMemsetAsync(in_next.p, 0, (n + 1) * sizeof(int), st));
        k_fill_ll<<<blocks_for(n + 1), kBlock, 0, st>>>(iso.p, n + 1, 0x7fffffffffffffffLL);
        if (nf) DLP_CUDA_TRY(cudaMemcpyAsync(la.p, frontier_init, nf * sizeof(long long), cudaMemcpyHostToDevice, st));
        long long* cur = la.p;
        long long* nxt = lb.p;
        long long cur_len = nf, iterations = 0, updates = 0;
        double max_change = 0.0;
        PlugCtl h{};
        unsigned long long warnings = 0;
        while (cur_len > 0 && iterations < max_iters) {
            DLP_CUDA_TRY(cudaMemsetAsync(ctl.p, 0, sizeof(PlugCtl), st));
            int g = blocks_for(cur_len);
            k_plug_step<<<g, kBlock, 0, st>>>(d_ip->p, d_ix->p, d_w->p, d_gt->p, d_f->p, cur, cur_len, vals.p, dels.p,
                                              iso.p);
            k_plug_commit<<<g, kBlock, 0, st>>>(d_ip->p, d_ix->p, cur, cur_len, vals.p, dels.p, d_f->p, d_el->p, iso.p,
                                                in_next.p, nxt, ctl.p, delta);
            k_plug_post<<<blocks_for(std::max<long long>(cur_len, n)), kBlock, 0, st>>>(cur, cur_len, dels.p, d_el->p,
                                                                                       iso.p, nxt, ctl.p, in_next.p);
            DLP_CUDA_TRY(cudaMemcpyAsync(&h, ctl.p, sizeof(PlugCtl), cudaMemcpyDeviceToHost, st));
            DLP_CUDA_TRY(cudaStreamSynchronize(st));
            updates += cur_len;
            iterations++;
            union { unsigned long long u; double d; } cv;
            cv.u = h.rmax;
            max_change = cv.d;
            warnings += h.warnings;
            std::swap(cur, nxt);
            cur_len = (long long)h.next;
        }
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
