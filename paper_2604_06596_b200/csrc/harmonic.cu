// harmonic.cu -- closed-form (harmonic) labels of the current graph on the
// B200: the accuracy oracle of the reference (baselines.py:109-190
// harmonic_dense / harmonic_solve, and the short-circuit StLP solve
// baselines.py:278-318 whose reduced system has the same solution).
//
//   reached   = connected to an alive ground-truth vertex (union-find over
//               the live-edge log, root = minimum member; baselines.py:87-106)
//   free      = reached & alive & unlabeled, numbered in ascending vertex id
//   A (m x m) = weighted degree on the diagonal, -w per free-free edge
//   B (m x C) = sum of w * pinned value over free-pinned edges, one column
//               per one-vs-rest label column
//   A X = B by Cholesky (cuSOLVER potrf / potrs, A is SPD on a
//   boundary-connected component), X clipped to [0, 1]; unreachable and dead
//   slots read 0.5, pinned vertices their class value.
//
// A warp assembles the row of one free vertex from its adjacency row
// (deterministic warp reductions); the dense solve is a library call, which
// is what the reference does too (scipy.linalg.solve(assume_a="pos")).
#include <cub/cub.cuh>
#include <cusolverDn.h>

#include <cstdio>
#include <vector>

#include "engine.cuh"

namespace dlp {

namespace {

__global__ void k_h_iota(int* p, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = (int)i;
}

__global__ void k_h_union(const int* lo, const int* hi, const DevState* ds, const unsigned char* alive, int* par) {
    const long long m = ds->log_n;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
        const int a = lo[i], b = hi[i];
        if (alive[a] && alive[b]) uf_unite(par, a, b);
    }
}

// root_gt[root] = component holds an alive ground-truth vertex; per-class
// counts of alive ground truth (StLP's both-classes check)
__global__ void k_h_roots(const int* par, long long n, const unsigned char* alive, const signed char* gt,
                          unsigned char* root_gt, unsigned long long* cls_count) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x) {
        if (alive[v] && gt[v] >= 0) {
            root_gt[uf_root(par, (int)v)] = 1;
            atomicAdd(&cls_count[gt[v] & 15], 1ULL);
        }
    }
}

__global__ void k_h_free(const int* par, long long n, const unsigned char* alive, const signed char* gt,
                         const unsigned char* root_gt, int* is_free, unsigned long long* unreached) {
    unsigned long long u = 0;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x) {
        int f = 0;
        if (alive[v]) {
            const bool r = root_gt[uf_root(par, (int)v)] != 0;
            f = r && gt[v] < 0;
            u += !r;
        }
        is_free[v] = f;
    }
    u = warp_sum(u);
    if ((threadIdx.x & 31) == 0 && u) atomicAdd(unreached, u);
}

__device__ inline double pinned_value(int g, int c, int C) { return C == 1 ? (double)g : (g == c ? 1.0 : 0.0); }

// one warp per free vertex: its row of A and B
__global__ void k_h_assemble(long long n, const int* is_free, const int* idx, const signed char* gt,
                             const long long* row_start, const int* row_len, const int* nbr, const double* wgt,
                             long long m, int C, double* A, double* B) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * blockDim.x / 32;
    for (long long v = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32; v < n; v += warps) {
        if (!is_free[v]) continue;
        const long long i = idx[v];
        const long long st = row_start[v];
        const int len = row_len[v];
        double deg = 0.0, b[kMaxCols];
        for (int c = 0; c < C; c++) b[c] = 0.0;
        for (int e = lane; e < len; e += 32) {
            const int y = nbr[st + e];
            const double w = wgt[st + e];
            deg += w;
            if (is_free[y]) {
                A[i * m + idx[y]] -= w;
            } else {
                const int g = gt[y];
                for (int c = 0; c < C; c++) b[c] += w * pinned_value(g, c, C);
            }
        }
        deg = warp_sum(deg);
        for (int c = 0; c < C; c++) b[c] = warp_sum(b[c]);
        if (lane == 0) {
            A[i * m + i] += deg;
            for (int c = 0; c < C; c++) B[(long long)c * m + i] = b[c];
        }
    }
}

__global__ void k_h_scatter(long long n, int C, const unsigned char* alive, const signed char* gt, const int* is_free,
                            const int* idx, const double* X, long long m, double* out) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n * C;
         t += (long long)gridDim.x * blockDim.x) {
        const long long v = t % n;
        const int c = (int)(t / n);
        double x = 0.5;
        if (alive[v] && gt[v] >= 0) {
            x = pinned_value(gt[v], c, C);
        } else if (is_free[v]) {
            x = X[(long long)c * m + idx[v]];
            x = x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x);
        }
        out[(long long)c * n + v] = x;
    }
}

template <typename T>
struct Scratch {
    T* p = nullptr;
    cudaStream_t st;
    Scratch(size_t count, cudaStream_t s) : st(s) {
        DLP_CUDA_TRY(cudaMallocAsync((void**)&p, (count ? count : 1) * sizeof(T), st));
    }
    ~Scratch() { cudaFreeAsync(p, st); }
};

}  // namespace

// Returns 0, or 3 (validation: too many free vertices / StLP needs both
// classes) with *msg set, or throws CudaFailure; 6 when the system is
// singular (cusolver info != 0).  out: C x n (column c at out + c*n).
int harmonic_solve_dev(Engine& E, int stlp, long long dense_cap, double* out_host, long long* fallback,
                       std::string* msg) {
    cudaStream_t st = E.st;
    const long long n = E.n_slots;
    const int C = E.ncol;
    Scratch<int> par(n, st), fr(n + 1, st), idx(n + 1, st);  // parent, free flag, free index
    Scratch<unsigned char> root_gt(n, st);
    Scratch<unsigned long long> counters(32, st);  // [0..15] class counts, [16] unreached
    DLP_CUDA_TRY(cudaMemsetAsync(root_gt.p, 0, n ? n : 1, st));
    DLP_CUDA_TRY(cudaMemsetAsync(counters.p, 0, 32 * sizeof(unsigned long long), st));
    const int g = blocks_for(n);
    if (n > 0) {
        k_h_iota<<<g, kBlock, 0, st>>>(par.p, n);
        k_h_union<<<E.sm_count * 8, kBlock, 0, st>>>(E.log_lo.p, E.log_hi.p, E.ds, E.alive.p, par.p);
        k_h_roots<<<g, kBlock, 0, st>>>(par.p, n, E.alive.p, E.gt.p, root_gt.p, counters.p);
        k_h_free<<<g, kBlock, 0, st>>>(par.p, n, E.alive.p, E.gt.p, root_gt.p, fr.p, counters.p + 16);
        DLP_CUDA_TRY(cudaGetLastError());
        size_t tmp = 0;
        DLP_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tmp, fr.p, idx.p, n + 1, st));
        Scratch<unsigned char> tb(tmp, st);
        DLP_CUDA_TRY(cudaMemsetAsync(fr.p + n, 0, sizeof(int), st));
        DLP_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tb.p, tmp, fr.p, idx.p, n + 1, st));
    }
    unsigned long long cnt[32] = {0};
    int m_host = 0;
    if (n > 0) {
        DLP_CUDA_TRY(cudaMemcpyAsync(cnt, counters.p, sizeof(cnt), cudaMemcpyDeviceToHost, st));
        DLP_CUDA_TRY(cudaMemcpyAsync(&m_host, idx.p + n, sizeof(int), cudaMemcpyDeviceToHost, st));
    }
    DLP_CUDA_TRY(cudaStreamSynchronize(st));
    const long long m = m_host;
    unsigned long long gt_total = 0;
    for (int k = 0; k < 16; k++) gt_total += cnt[k];
    if (gt_total == 0) {  // baselines.py:174-175
        *msg = "harmonic solve requires at least one ground-truth vertex";
        return DLP_EVALIDATION;
    }
    if (stlp) {  // baselines.py:285-287, per one-vs-rest column
        for (int c = 0; c < C; c++) {
            const unsigned long long ones = C == 1 ? cnt[1] : cnt[c];
            if (ones == 0 || ones == gt_total) {
                *msg = "short-circuit contraction requires both classes nonempty";
                return DLP_EVALIDATION;
            }
        }
    }
    if (m > dense_cap) {  // baselines.py:133-134
        char b[160];
        snprintf(b, sizeof b, "%lld free vertices exceed the dense-solve cap %lld", m, dense_cap);
        *msg = b;
        return DLP_EVALIDATION;
    }
    *fallback = (long long)cnt[16];
    Scratch<double> X(m * C + 1, st), Out((size_t)n * C + 1, st);
    if (m > 0) {
        Scratch<double> A((size_t)m * m, st);
        DLP_CUDA_TRY(cudaMemsetAsync(A.p, 0, (size_t)m * m * sizeof(double), st));
        k_h_assemble<<<blocks_for(n * 32), kBlock, 0, st>>>(n, fr.p, idx.p, E.gt.p, E.row_start.p, E.row_len.p,
                                                              E.nbr.p, E.wgt.p, m, C, A.p, X.p);
        DLP_CUDA_TRY(cudaGetLastError());
        if (!E.cusolver) {
            if (cusolverDnCreate((cusolverDnHandle_t*)&E.cusolver) != CUSOLVER_STATUS_SUCCESS)
                throw CudaFailure(cudaErrorUnknown, "cusolverDnCreate", __FILE__, __LINE__);
        }
        cusolverDnHandle_t hs = (cusolverDnHandle_t)E.cusolver;
        cusolverDnSetStream(hs, st);
        int lwork = 0;
        if (cusolverDnDpotrf_bufferSize(hs, CUBLAS_FILL_MODE_LOWER, (int)m, A.p, (int)m, &lwork) !=
            CUSOLVER_STATUS_SUCCESS)
            throw CudaFailure(cudaErrorUnknown, "cusolverDnDpotrf_bufferSize", __FILE__, __LINE__);
        Scratch<double> work((size_t)lwork + 1, st);
        Scratch<int> info(2, st);
        cusolverDnDpotrf(hs, CUBLAS_FILL_MODE_LOWER, (int)m, A.p, (int)m, work.p, lwork, info.p);
        cusolverDnDpotrs(hs, CUBLAS_FILL_MODE_LOWER, (int)m, C, A.p, (int)m, X.p, (int)m, info.p + 1);
        int ih[2] = {0, 0};
        DLP_CUDA_TRY(cudaMemcpyAsync(ih, info.p, sizeof(ih), cudaMemcpyDeviceToHost, st));
        DLP_CUDA_TRY(cudaStreamSynchronize(st));
        if (ih[0] != 0 || ih[1] != 0) {  // baselines.py:150-156
            char b[200];
            snprintf(b, sizeof b, "harmonic system singular on %lld free vertices (cusolver info %d/%d)", m, ih[0],
                     ih[1]);
            *msg = b;
            return DLP_EINTERNAL;
        }
    }
    if (n > 0) {
        k_h_scatter<<<blocks_for(n * C), kBlock, 0, st>>>(n, C, E.alive.p, E.gt.p, fr.p, idx.p, X.p, m, Out.p);
        DLP_CUDA_TRY(cudaGetLastError());
        DLP_CUDA_TRY(cudaMemcpyAsync(out_host, Out.p, (size_t)n * C * sizeof(double), cudaMemcpyDeviceToHost, st));
    }
    DLP_CUDA_TRY(cudaStreamSynchronize(st));
    return DLP_OK;
}

}  // namespace dlp
