// lp.cu -- device-driven DynLP propagation loop (one persistent cooperative
// kernel per label column and batch).
//
// Reference semantics (paths under /root/reference/pkg/src/dynlp/):
//   frontier rounds   kernels/_csr.pyx:114-197 (jacobi_run: evaluate every
//                     frontier row against the pre-round f, commit, expand
//                     vertices that moved by more than delta plus their
//                     eligible neighbours)
//   certify sweep     engine.py:290-301 (a committed round over every
//                     eligible vertex; stop when its max move <= delta)
//   outer loop        engine.py:375-405, budget engine.py:67-70, 369
//   per-vertex update kernels/_csr.pyx:24-58 (RowAcc in common.cuh)
//
// B200 design: the whole loop runs on the device -- no host round trip per
// round.  Jacobi semantics come from double-buffered labels: round r reads
// F[r&1] and writes F[(r+1)&1] for the frontier F_r, and re-syncs the
// vertices of F_{r-1} that are not in F_r, so each round needs exactly ONE
// grid-wide barrier.  Frontier membership lives in three rotating bitmaps
// (claim = atomicOr), frontier ids in three rotating lists (warp-aggregated
// append); per-round scalars rotate through small arrays so no reset races a
// reader.
#include <cooperative_groups.h>
#include <cstdlib>

#include "engine.cuh"

namespace cg = cooperative_groups;

namespace dlp {

struct LPParams {
    const long long* row_start;
    const int* row_len;
    const int* nbr;
    const double* w;
    double* fa;
    double* fb;
    unsigned char* elig;
    int* L0;
    int* L1;
    int* L2;
    unsigned int* M0;
    unsigned int* M1;
    unsigned int* M2;
    const int* f0;
    const int* elist;
    const DevState* ds;
    LPCtl* ctl;
    double delta;
    long long max_iter;
};

__device__ inline bool test_bit(const unsigned int* M, int v) { return (M[v >> 5] >> (v & 31)) & 1u; }
__device__ inline void clear_bit(unsigned int* M, int v) { atomicAnd(&M[v >> 5], ~(1u << (v & 31))); }

__device__ inline void claim(unsigned int* M, int* L, unsigned int* cnt, int v) {
    unsigned int bit = 1u << (v & 31);
    unsigned int* word = M + (v >> 5);
    if (*(volatile unsigned int*)word & bit) return;
    if (atomicOr(word, bit) & bit) return;
    cg::coalesced_group g = cg::coalesced_threads();
    unsigned int base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(cnt, g.size());
    base = g.shfl(base, 0);
    L[base + g.thread_rank()] = v;
}

#ifdef DLP_LP_CG
#define LDX(p) __ldcg(p)
#else
#define LDX(p) (*(p))
#endif

// _update_one over the engine's row layout; X holds boxed labels.
__device__ inline double eval_row(const LPParams& P, const double* X, int u, long long* s_out, int* len_out,
                                  double* val) {
    long long s = P.row_start[u];
    int len = P.row_len[u];
    double fu = LDX(X + u);
    RowAcc acc;
    acc.init();
    for (int e = 0; e < len; e++) {
        int v = P.nbr[s + e];
        double we = P.w[s + e];
        double x = LDX(X + v);
        acc.add(we, is_boxed(x) ? boxed_class(x) : -1, x, fu);
    }
    *s_out = s;
    *len_out = len;
    return acc.finish(fu, val);
}

__device__ inline void block_flush(double lmax, long long ledges, long long lswept, long long lwarn,
                                   unsigned long long* rmax_slot, unsigned long long* swept_slot, LPCtl* ctl) {
    __shared__ double smax[kBlock / 32];
    __shared__ long long sedge[kBlock / 32], ssw[kBlock / 32], swarn[kBlock / 32];
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    lmax = warp_max(lmax);
    ledges = warp_sum(ledges);
    lswept = warp_sum(lswept);
    lwarn = warp_sum(lwarn);
    if (lane == 0) {
        smax[wid] = lmax;
        sedge[wid] = ledges;
        ssw[wid] = lswept;
        swarn[wid] = lwarn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double m = 0.0;
        long long e = 0, sw = 0, wn = 0;
        for (int i = 0; i < kBlock / 32; i++) {
            m = fmax(m, smax[i]);
            e += sedge[i];
            sw += ssw[i];
            wn += swarn[i];
        }
        if (m > 0.0) atomic_max_nonneg(rmax_slot, m);
        if (e) atomicAdd((unsigned long long*)&ctl->edges, (unsigned long long)e);
        if (sw) atomicAdd(swept_slot, (unsigned long long)sw);
        if (wn) atomicAdd((unsigned long long*)&ctl->warnings, (unsigned long long)wn);
    }
}

// One committed round over `cur` (Jacobi: reads X, writes Y); claims the next
// frontier into (Mn, Ln, cnt_next); re-syncs Y on `prev` \ cur and clears
// prev's membership bits.  `certify` skips ineligible ids (the eligible list
// is built once per batch).
__device__ void lp_round(const LPParams& P, const int* cur, long long ncur, const int* prev, long long nprev,
                         bool certify, const double* X, double* Y, const unsigned int* Mc, unsigned int* Mn,
                         unsigned int* Mp, int* Ln, unsigned int* cnt_next, unsigned long long* rmax_slot,
                         unsigned long long* swept_slot) {
    long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    long long nth = (long long)gridDim.x * blockDim.x;
    double lmax = 0.0;
    long long ledges = 0, lswept = 0, lwarn = 0;
    for (long long i = tid; i < ncur; i += nth) {
        int u = LDX(cur + i);
        if (certify && !P.elig[u]) continue;
        lswept++;
        long long s;
        int len;
        double val;
        double d = eval_row(P, X, u, &s, &len, &val);
        ledges += len;
        Y[u] = val;
        if (d < 0.0) {
            lwarn++;
            P.elig[u] = 0;
            continue;
        }
        lmax = fmax(lmax, d);
        if (d > P.delta) {
            if (P.elig[u]) claim(Mn, Ln, cnt_next, u);
            for (int e = 0; e < len; e++) {
                int v = P.nbr[s + e];
                if (P.elig[v]) claim(Mn, Ln, cnt_next, v);
            }
        }
    }
    for (long long i = tid; i < nprev; i += nth) {
        int u = LDX(prev + i);
        if (!((LDX(Mc + (u >> 5)) >> (u & 31)) & 1u)) Y[u] = LDX(X + u);
        clear_bit(Mp, u);
    }
    block_flush(lmax, ledges, lswept, lwarn, rmax_slot, swept_slot, P.ctl);
}

__global__ void __launch_bounds__(kBlock) k_lp_loop(LPParams P) {
    LPCtl* ctl = P.ctl;
    unsigned int target = 0;
    long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    long long nth = (long long)gridDim.x * blockDim.x;
    int* L[3] = {P.L0, P.L1, P.L2};
    unsigned int* M[3] = {P.M0, P.M1, P.M2};
    double* F[2] = {P.fa, P.fb};

    long long n0 = P.ds->n_f0;
    for (long long i = tid; i < n0; i += nth) {
        int u = P.f0[i];
        L[0][i] = u;
        atomicOr(&M[0][u >> 5], 1u << (u & 31));
    }
    grid_sync(&ctl->bar, target);

    long long cur = n0, prev = 0;
    int r = 0;
    long long iterations = 0, updates = 0, certs = 0;
    double max_change = 0.0;
    int converged = 1;
    for (;;) {
        // ---- jacobi_run (_csr.pyx:155-194) ----
        long long budget = P.max_iter - iterations;
        long long it = 0;
        double mc = 0.0;
        while (cur > 0 && it < budget) {
            int ic = r % 3, in = (r + 1) % 3, ip = (r + 2) % 3;
            if (tid == 0) {
                ctl->cnt[(r + 2) & 3] = 0;
                ctl->rmax[(r + 1) % 3] = 0;
                ctl->swept[(r + 1) % 3] = 0;
            }
            lp_round(P, L[ic], cur, L[ip], prev, false, F[r & 1], F[(r + 1) & 1], M[ic], M[in], M[ip], L[in],
                     &ctl->cnt[(r + 1) & 3], &ctl->rmax[r % 3], &ctl->swept[r % 3]);
            grid_sync(&ctl->bar, target);
            updates += cur;
            it++;
            mc = __longlong_as_double((long long)*(volatile unsigned long long*)&ctl->rmax[r % 3]);
            prev = cur;
            cur = *(volatile unsigned int*)&ctl->cnt[(r + 1) & 3];
            r++;
        }
        iterations += it;
        if (it) {
            max_change = mc;
            int ipv = (r + 2) % 3;  // F_{r-1}: stale in F[(r+1)&1]
            for (long long i = tid; i < prev; i += nth) {
                int u = L[ipv][i];
                F[(r + 1) & 1][u] = F[r & 1][u];
                clear_bit(M[ipv], u);
            }
            grid_sync(&ctl->bar, target);
            prev = 0;
        }
        if (cur > 0 || iterations >= P.max_iter) {
            converged = cur == 0;
            if (!converged) break;
        }
        // ---- certify_round (engine.py:290-301) ----
        int in = (r + 1) % 3;
        if (tid == 0) {
            ctl->cnt[(r + 2) & 3] = 0;
            ctl->rmax[(r + 1) % 3] = 0;
            ctl->swept[(r + 1) % 3] = 0;
        }
        long long ne = P.ds->n_elist;
        lp_round(P, P.elist, ne, nullptr, 0, true, F[r & 1], F[(r + 1) & 1], M[r % 3], M[in], M[(r + 2) % 3],
                 L[in], &ctl->cnt[(r + 1) & 3], &ctl->rmax[r % 3], &ctl->swept[r % 3]);
        grid_sync(&ctl->bar, target);
        long long swept = (long long)*(volatile unsigned long long*)&ctl->swept[r % 3];
        if (swept == 0) break;
        for (long long i = tid; i < ne; i += nth) {
            int u = P.elist[i];
            F[r & 1][u] = F[(r + 1) & 1][u];
        }
        grid_sync(&ctl->bar, target);
        double cm = __longlong_as_double((long long)*(volatile unsigned long long*)&ctl->rmax[r % 3]);
        certs++;
        iterations++;
        updates += swept;
        max_change = cm;
        cur = *(volatile unsigned int*)&ctl->cnt[(r + 1) & 3];
        r++;
        prev = 0;
        if (cm <= P.delta) break;
    }
    // leftover frontier (budget exhausted): drop its membership bits
    for (long long i = tid; i < cur; i += nth) clear_bit(M[r % 3], L[r % 3][i]);
    if (tid == 0) {
        ctl->iterations = iterations;
        ctl->updates = updates;
        ctl->max_change = max_change;
        ctl->converged = converged;
        ctl->certs = certs;
    }
}

void lp_setup(Engine& E) {
    if (E.lp_grid) return;
    E.lp_ev.resize(2 * E.ncol);
    E.lp_ms.assign(E.ncol, 0.0);
    for (auto& ev : E.lp_ev) DLP_CUDA_TRY(cudaEventCreate(&ev));
    int occ = 0;
    DLP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lp_loop, kBlock, 0));
    if (occ < 1) occ = 1;
    if (occ > 8) occ = 8;
    E.lp_grid = E.sm_count * occ;
    if (const char* g = getenv("DLP_LP_GRID")) E.lp_grid = atoi(g);
}

void lp_loop_dev(Engine& E, int col, double delta, long long max_iter, int mode) {
    (void)mode;
    lp_setup(E);
    LPParams P;
    P.row_start = E.row_start.p;
    P.row_len = E.row_len.p;
    P.nbr = E.nbr.p;
    P.w = E.wgt.p;
    P.fa = E.f[0].p + (size_t)col * E.cap_n;
    P.fb = E.f[1].p + (size_t)col * E.cap_n;
    P.elig = E.elig.p + (size_t)col * E.cap_n;
    P.L0 = E.list[0].p;
    P.L1 = E.list[1].p;
    P.L2 = E.list[2].p;
    P.M0 = E.memb[0].p;
    P.M1 = E.memb[1].p;
    P.M2 = E.memb[2].p;
    P.f0 = E.f0.p;
    P.elist = E.elist.p;
    P.ds = E.ds;
    P.ctl = E.ctl + col;
    P.delta = delta;
    P.max_iter = max_iter;
    DLP_CUDA_TRY(cudaMemsetAsync(E.ctl + col, 0, sizeof(LPCtl), E.st));
    void* args[] = {&P};
    DLP_CUDA_TRY(cudaEventRecord(E.lp_ev[2 * col], E.st));
    DLP_CUDA_TRY(cudaLaunchCooperativeKernel((void*)k_lp_loop, dim3(E.lp_grid), dim3(kBlock), args, 0, E.st));
    DLP_CUDA_TRY(cudaEventRecord(E.lp_ev[2 * col + 1], E.st));
    E.launches++;
}

// ---------------------------------------------------------------------------
// ItLP (baselines.py:190-233): full Jacobi sweeps over the active set
// (alive, unlabeled, degree > 0) until the largest move <= delta.
// ---------------------------------------------------------------------------
__global__ void k_itlp_active(long long n, const unsigned char* alive, const signed char* gt, const int* row_len,
                              int ncol, long long cap, double* f0, double* f1, int* alist, DevState* ds) {
    long long iso = 0;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x) {
        bool unl = alive[v] && gt[v] == -1;
        if (!unl) continue;
        if (row_len[v] > 0) {
            append_agg(alist, &ds->n_elist, (int)v);
        } else {
            iso++;
            for (int c = 0; c < ncol; c++) {
                f0[c * cap + v] = 0.5;
                f1[c * cap + v] = 0.5;
            }
        }
    }
    iso = warp_sum(iso);
    if ((threadIdx.x & 31) == 0 && iso) atomicAdd((unsigned long long*)&ds->isolated, (unsigned long long)iso);
}

__global__ void __launch_bounds__(kBlock) k_itlp_loop(LPParams P) {
    LPCtl* ctl = P.ctl;
    unsigned int target = 0;
    long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    long long nth = (long long)gridDim.x * blockDim.x;
    long long na = P.ds->n_elist;
    long long iterations = 0, updates = 0;
    double max_change = 0.0;
    int converged = na == 0;
    int r = 0;
    while (iterations < P.max_iter && !converged) {
        if (tid == 0) ctl->rmax[(r + 1) % 3] = 0;
        double lmax = 0.0;
        long long ledges = 0;
        for (long long i = tid; i < na; i += nth) {
            int u = P.elist[i];
            long long s;
            int len;
            double val;
            double d = eval_row(P, P.fa, u, &s, &len, &val);
            ledges += len;
            P.fb[u] = val;
            lmax = fmax(lmax, d);
        }
        block_flush(lmax, ledges, 0, 0, &ctl->rmax[r % 3], &ctl->swept[0], ctl);
        grid_sync(&ctl->bar, target);
        for (long long i = tid; i < na; i += nth) {
            int u = P.elist[i];
            P.fa[u] = P.fb[u];
        }
        grid_sync(&ctl->bar, target);
        iterations++;
        updates += na;
        max_change = __longlong_as_double((long long)*(volatile unsigned long long*)&ctl->rmax[r % 3]);
        converged = max_change <= P.delta;
        r++;
    }
    if (tid == 0) {
        ctl->iterations = iterations;
        ctl->updates = updates;
        ctl->max_change = max_change;
        ctl->converged = converged;
        ctl->certs = 0;
    }
}

void itlp_dev(Engine& E, int col, double delta, long long max_iter) {
    lp_setup(E);
    LPParams P{};
    P.row_start = E.row_start.p;
    P.row_len = E.row_len.p;
    P.nbr = E.nbr.p;
    P.w = E.wgt.p;
    P.fa = E.f[0].p + (size_t)col * E.cap_n;
    P.fb = E.f[1].p + (size_t)col * E.cap_n;
    P.elig = E.elig.p + (size_t)col * E.cap_n;
    P.elist = E.elist.p;
    P.ds = E.ds;
    P.ctl = E.ctl + col;
    P.delta = delta;
    P.max_iter = max_iter;
    DLP_CUDA_TRY(cudaMemsetAsync(E.ctl + col, 0, sizeof(LPCtl), E.st));
    void* args[] = {&P};
    DLP_CUDA_TRY(cudaEventRecord(E.lp_ev[2 * col], E.st));
    DLP_CUDA_TRY(cudaLaunchCooperativeKernel((void*)k_itlp_loop, dim3(E.lp_grid), dim3(kBlock), args, 0, E.st));
    DLP_CUDA_TRY(cudaEventRecord(E.lp_ev[2 * col + 1], E.st));
    E.launches++;
}

void itlp_active_dev(Engine& E, long long n) {
    if (n == 0) return;
    k_itlp_active<<<blocks_for(n, kBlock, 148 * 64), kBlock, 0, E.st>>>(n, E.alive.p, E.gt.p, E.row_len.p, E.ncol,
                                                                       E.cap_n, E.f[0].p, E.f[1].p, E.elist.p,
                                                                       E.ds);
    E.launches++;
}

}  // namespace dlp
