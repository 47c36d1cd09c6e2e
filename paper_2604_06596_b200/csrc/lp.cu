// lp.cu -- device-driven DynLP propagation: ONE persistent cooperative kernel
// per batch runs every label column's frontier rounds and certify sweeps.
//
// Reference semantics (paths under /root/reference/pkg/src/dynlp/):
//   frontier rounds   kernels/_csr.pyx:114-197 (jacobi_run: evaluate the
//                     frontier against the pre-round f, commit, expand the
//                     vertices that moved by more than delta plus their
//                     eligible neighbours)
//   certify sweep     engine.py:290-301 (a committed round over every
//                     eligible vertex; stop when its max move <= delta)
//   outer loop        engine.py:375-405, budget engine.py:67-70, 369
//   per-vertex update kernels/_csr.pyx:24-58 (RowAcc in common.cuh)
//   ItLP              baselines.py:190-233 (full sweeps over the active set)
//
// B200 design
// * Fused label columns.  The C one-vs-rest columns (C = 1 for binary) run in
//   lockstep global rounds; each column follows its own reference state
//   machine (frontier rounds -> certify -> ...), so per-column results are
//   exactly those of C independent reference runs.  A round's work list is
//   the union of the columns' frontiers (or the eligible list when a column
//   certifies); every row is read ONCE per round for all columns and one
//   gather of X[v*C .. v*C+C) serves every column.
// * CTA tiles.  A block grabs a chunk of up to 32 rows (dynamic atomic
//   scheduling), gathers the chunk's row entries entry-parallel into shared
//   memory (coalesced row reads, independent gathers), then one thread per
//   (row, column) accumulates the row in stored order -- the reference's
//   sequential fp64 summation -- from shared memory.  Rows of any length
//   (kNN hubs reach thousands of entries) are streamed window by window, so
//   load balance no longer depends on the degree distribution.
// * Jacobi commit: phase 1 writes new values to the staging buffer Y, phase 2
//   copies them into X; two grid-wide barriers per round.
#include <cooperative_groups.h>

#include <cstdlib>

#include "engine.cuh"

namespace cg = cooperative_groups;

namespace dlp {

constexpr int kLpThreads = 256;
constexpr int kChunkRows = 32;
constexpr int kWin = 512;  // row entries staged per window

enum { PH_FRONTIER = 0, PH_DONE = 2 };

struct LPParams {
    const long long* row_start;
    const int* row_len;
    const int* nbr;
    const double* w;
    double* X;  // canonical labels [v*C + c]
    double* Y;  // staging
    unsigned int* eligm;
    unsigned int* emask_store;
    unsigned int* fmask0;
    unsigned int* fmask1;
    int* U0;
    int* U1;
    const int* f0;
    const int* elist;
    const DevState* ds;
    LPCtl* ctl;
    double delta;
    long long max_iter;
    int C;
    int itlp;
};

struct ColState {
    int phase[kMaxCols];
    int has_frontier[kMaxCols];
    long long it_run[kMaxCols];
    double mc_last[kMaxCols];
    long long iterations[kMaxCols];
    long long updates[kMaxCols];
    long long certs[kMaxCols];
    long long warnings[kMaxCols];
    long long edges[kMaxCols];
    double max_change[kMaxCols];
    int converged[kMaxCols];
    unsigned int fr_mask, cert_mask;  // actions of the current round
    int done;
};

__device__ inline int row_of(const int* off, int nrows, int g) {
    int lo = 0, hi = nrows;  // largest r with off[r] <= g
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (off[mid] <= g)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

struct ClaimCtx {
    unsigned int* fm_next;
    int* U_next;
    unsigned int* cnt;
    const unsigned int* eligm;
    unsigned int claimed;  // per-thread OR of claimed column bits
};

__device__ inline void claim(ClaimCtx& k, int v, unsigned int bits) {
    bits &= k.eligm[v];
    if (!bits) return;
    k.claimed |= bits;
    unsigned int* fm = k.fm_next + v;
    unsigned int cur = *(volatile unsigned int*)fm;
    if ((cur & bits) == bits) return;
    unsigned int old = atomicOr(fm, bits);
    if (old != 0) return;
    cg::coalesced_group g = cg::coalesced_threads();
    unsigned int base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(k.cnt, g.size());
    base = g.shfl(base, 0);
    k.U_next[base + g.thread_rank()] = v;
}

// Controller: every block updates its shared copy of the per-column state
// from the finished round's slot and decides the next round's actions.
__device__ void decide_actions(ColState& S, const LPParams& P, const RoundSlot* res, int first) {
    int C = P.C;
    unsigned int fr = 0, ce = 0;
    int done = 1;
    for (int c = 0; c < C; c++) {
        unsigned int bit = 1u << c;
        if (!first && S.phase[c] != PH_DONE) {
            bool was_fr = (S.fr_mask & bit) != 0, was_ce = (S.cert_mask & bit) != 0;
            if (was_fr || was_ce) {
                double rm = __longlong_as_double((long long)res->rmax[c]);
                S.iterations[c]++;
                S.updates[c] += (long long)res->neval[c];
                S.edges[c] += (long long)res->edges[c];
                S.warnings[c] += (long long)res->warn[c];
                S.has_frontier[c] = (res->claimed & bit) != 0;
                if (P.itlp) {
                    S.max_change[c] = rm;
                    if (rm <= P.delta) {
                        S.converged[c] = 1;
                        S.phase[c] = PH_DONE;
                    }
                } else if (was_fr) {
                    S.it_run[c]++;
                    S.mc_last[c] = rm;
                } else {  // certify_round committed (engine.py:398-405)
                    S.certs[c]++;
                    S.max_change[c] = rm;
                    S.it_run[c] = 0;
                    if (rm <= P.delta) S.phase[c] = PH_DONE;
                }
            }
        }
        if (S.phase[c] == PH_DONE) continue;
        if (P.itlp) {
            if (S.iterations[c] >= P.max_iter) {
                S.phase[c] = PH_DONE;
                continue;
            }
            ce |= bit;
            done = 0;
            continue;
        }
        if (S.has_frontier[c] && S.iterations[c] < P.max_iter) {  // jacobi_run continues
            fr |= bit;
            done = 0;
            continue;
        }
        // jacobi_run returned (engine.py:387-397)
        if (S.it_run[c] > 0) S.max_change[c] = S.mc_last[c];
        S.it_run[c] = 0;
        if (S.has_frontier[c] || S.iterations[c] >= P.max_iter) {
            S.converged[c] = S.has_frontier[c] ? 0 : 1;
            if (!S.converged[c]) {
                S.phase[c] = PH_DONE;
                continue;
            }
        }
        if (*(volatile long long*)&P.ctl->elig_count[c] == 0) {  // certify swept nothing: break
            S.phase[c] = PH_DONE;
            continue;
        }
        ce |= bit;
        done = 0;
    }
    S.fr_mask = fr;
    S.cert_mask = ce;
    S.done = done;
}

__global__ void __launch_bounds__(kLpThreads) k_lp_fused(LPParams P) {
    extern __shared__ double smem_dyn[];
    __shared__ ColState S;
    __shared__ int s_u[kChunkRows], s_len[kChunkRows], s_off[kChunkRows + 1];
    __shared__ long long s_st[kChunkRows];
    __shared__ unsigned int s_em[kChunkRows], s_chg[kChunkRows];
    __shared__ unsigned long long b_rmax[kMaxCols], b_neval[kMaxCols], b_edges[kMaxCols], b_warn[kMaxCols];
    __shared__ unsigned int b_claimed, s_k;
    __shared__ unsigned long long b_urows, b_uent;
    __shared__ int s_total;

    const int C = P.C;
    const int tid = threadIdx.x;
    const long long gtid = blockIdx.x * (long long)blockDim.x + tid;
    const long long gth = (long long)gridDim.x * blockDim.x;
    LPCtl* ctl = P.ctl;
    unsigned int target = 0;
    double* sw = smem_dyn;         // [kWin]
    double* sx = smem_dyn + kWin;  // [kWin * C]
    const int rows_per_chunk = min(kChunkRows, kLpThreads / C);
    const unsigned int allc = C >= 32 ? 0xffffffffu : ((1u << C) - 1u);
    int* U[2] = {P.U0, P.U1};
    unsigned int* FM[2] = {P.fmask0, P.fmask1};

    // ---- prologue: F0 (engine.py:364-367) is every column's first frontier
    const long long n0 = P.itlp ? 0 : P.ds->n_f0;
    const long long n_el = P.ds->n_elist;
    for (long long i = gtid; i < n0; i += gth) {
        int u = P.f0[i];
        U[0][i] = u;
        FM[0][u] = allc;
    }
    if (tid == 0) {
        for (int c = 0; c < C; c++) {
            S.phase[c] = PH_FRONTIER;
            S.has_frontier[c] = n0 > 0;
            S.it_run[c] = 0;
            S.mc_last[c] = 0.0;
            S.iterations[c] = S.updates[c] = S.certs[c] = S.warnings[c] = S.edges[c] = 0;
            S.max_change[c] = 0.0;
            S.converged[c] = P.itlp ? (n_el == 0) : 1;
            if (P.itlp && n_el == 0) S.phase[c] = PH_DONE;
        }
        S.fr_mask = S.cert_mask = 0;
        if (blockIdx.x == 0)
            for (int c = 0; c < C; c++) ctl->elig_count[c] = n_el;
    }
    grid_sync(&ctl->bar, target);
    if (tid == 0) decide_actions(S, P, nullptr, 1);
    __syncthreads();

    long long ncur = n0;
    long long R = 0;
    while (!S.done) {
        const unsigned int FR = S.fr_mask, CE = S.cert_mask;
        RoundSlot* slot = &ctl->slot[R & 1];
        const int* W = CE ? P.elist : U[R & 1];
        const long long nwork = CE ? n_el : ncur;
        unsigned int* fm_cur = FM[R & 1];
        ClaimCtx K{FM[(R + 1) & 1], U[(R + 1) & 1], &slot->cnt, P.eligm, 0u};
        if (tid < kMaxCols) {
            b_rmax[tid] = 0;
            b_neval[tid] = 0;
            b_edges[tid] = 0;
            b_warn[tid] = 0;
        }
        if (tid == 0) {
            b_claimed = 0;
            b_urows = 0;
            b_uent = 0;
        }
        __syncthreads();

        // ======== phase 1: evaluate + expand, chunk by chunk ========
        for (;;) {
            if (tid == 0) s_k = atomicAdd(&slot->grab, (unsigned int)rows_per_chunk);
            __syncthreads();
            const long long k0 = s_k;
            if (k0 >= nwork) break;
            const int nrows = (int)min((long long)rows_per_chunk, nwork - k0);
            if (tid < kChunkRows) {
                int len = 0;
                unsigned int em = 0;
                int u = -1;
                long long st = 0;
                if (tid < nrows) {
                    u = W[k0 + tid];
                    em = P.itlp ? (CE & P.eligm[u]) : ((fm_cur[u] & FR) | (CE & P.eligm[u]));
                    if (em) {
                        st = P.row_start[u];
                        len = P.row_len[u];
                    }
                    P.emask_store[u] = em;
                }
                s_u[tid] = u;
                s_em[tid] = em;
                s_st[tid] = st;
                s_len[tid] = len;
                s_chg[tid] = 0;
            }
            __syncthreads();
            if (tid < 32) {  // exclusive scan of row lengths (kChunkRows == 32)
                int x = s_len[tid], incl = x;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (tid >= o) incl += y;
                }
                s_off[tid] = incl - x;
                if (tid == 31) s_total = incl;
            }
            __syncthreads();
            const int T = s_total;
            if (tid == 0) {
                int nz = 0;
                for (int r = 0; r < nrows; r++) nz += s_em[r] != 0;
                b_urows += nz;
                b_uent += T;
            }
            // this thread's (row, column) pair
            const int pr = tid / C, pc = tid - pr * C;
            const bool active = pr < nrows && ((s_em[pr] >> pc) & 1u);
            double fu = 0.0;
            RowAcc acc;
            acc.init();
            if (active) fu = P.X[(long long)s_u[pr] * C + pc];
            for (int wb = 0; wb < T; wb += kWin) {
                const int wn = min(kWin, T - wb);
                for (int t = tid; t < wn; t += kLpThreads) {
                    int g = wb + t;
                    int r = row_of(s_off, nrows, g);
                    long long p = s_st[r] + (g - s_off[r]);
                    int v = P.nbr[p];
                    sw[t] = P.w[p];
                    const double* xv = P.X + (long long)v * C;
                    double* dst = sx + t * C;
                    for (int c = 0; c < C; c++) dst[c] = xv[c];
                }
                __syncthreads();
                if (active) {
                    int lo = max(s_off[pr], wb) - wb;
                    int hi = min(s_off[pr] + s_len[pr], wb + wn) - wb;
                    for (int t = lo; t < hi; t++) {
                        double x = sx[t * C + pc];
                        acc.add(sw[t], is_boxed(x) ? boxed_class(x) : -1, x, fu);
                    }
                }
                __syncthreads();
            }
            if (active) {
                double val;
                double d = acc.finish(fu, &val);
                int u = s_u[pr];
                P.Y[(long long)u * C + pc] = val;
                atomicAdd(&b_neval[pc], 1ULL);
                atomicAdd(&b_edges[pc], (unsigned long long)s_len[pr]);
                if (d < 0.0) {  // isolated sentinel (_csr.pyx:49-51, 170-173)
                    atomicAdd(&b_warn[pc], 1ULL);
                    atomicAnd(&P.eligm[u], ~(1u << pc));
                    atomicAdd((unsigned long long*)&ctl->elig_count[pc], ~0ULL);
                } else {
                    if (d > 0.0) atomicMax(&b_rmax[pc], dbits(d));
                    if (!P.itlp && d > P.delta) atomicOr(&s_chg[pr], 1u << pc);
                }
            }
            __syncthreads();
            if (!P.itlp) {
                // expand: changed rows claim themselves and eligible neighbours
                if (tid < nrows && s_chg[tid]) claim(K, s_u[tid], s_chg[tid]);
                for (int g = tid; g < T; g += kLpThreads) {
                    int r = row_of(s_off, nrows, g);
                    unsigned int chg = s_chg[r];
                    if (chg) claim(K, P.nbr[s_st[r] + (g - s_off[r])], chg);
                }
            }
            __syncthreads();
        }
        if (K.claimed) atomicOr(&b_claimed, K.claimed);
        __syncthreads();
        if (tid < C) {
            if (b_rmax[tid]) atomicMax(&slot->rmax[tid], b_rmax[tid]);
            if (b_neval[tid]) atomicAdd(&slot->neval[tid], b_neval[tid]);
            if (b_edges[tid]) atomicAdd(&slot->edges[tid], b_edges[tid]);
            if (b_warn[tid]) atomicAdd(&slot->warn[tid], b_warn[tid]);
        }
        if (tid == 0) {
            if (b_claimed) atomicOr(&slot->claimed, b_claimed);
            if (b_urows) atomicAdd(&slot->urows, b_urows);
            if (b_uent) atomicAdd(&slot->uentries, b_uent);
        }
        grid_sync(&ctl->bar, target);

        // ======== phase 2: commit (Jacobi) and clear this round's masks ========
        for (long long i = gtid; i < nwork; i += gth) {
            int u = W[i];
            unsigned int em = P.emask_store[u];
            for (int c = 0; c < C; c++)
                if ((em >> c) & 1u) P.X[(long long)u * C + c] = P.Y[(long long)u * C + c];
            fm_cur[u] = 0;
        }
        if (gtid == 0) {
            RoundSlot* nx = &ctl->slot[(R + 1) & 1];
            for (int c = 0; c < kMaxCols; c++) nx->rmax[c] = nx->neval[c] = nx->edges[c] = nx->warn[c] = 0;
            nx->claimed = 0;
            nx->urows = 0;
            nx->uentries = 0;
            nx->grab = 0;
            nx->cnt = 0;
        }
        grid_sync(&ctl->bar, target);
        if (tid == 0) {
            RoundSlot res;
            const volatile RoundSlot* vs = slot;
            for (int c = 0; c < C; c++) {
                res.rmax[c] = vs->rmax[c];
                res.neval[c] = vs->neval[c];
                res.edges[c] = vs->edges[c];
                res.warn[c] = vs->warn[c];
            }
            res.claimed = vs->claimed;
            decide_actions(S, P, &res, 0);
            if (blockIdx.x == 0) {
                ctl->urows += (long long)vs->urows;
                ctl->uentries += (long long)vs->uentries;
            }
        }
        ncur = *(volatile unsigned int*)&slot->cnt;
        R++;
        __syncthreads();
    }
    // leftover frontiers (budget exhausted): clear their masks for the next batch
    for (long long i = gtid; i < ncur; i += gth) FM[R & 1][U[R & 1][i]] = 0;
    if (gtid == 0) {
        for (int c = 0; c < C; c++) {
            ctl->iterations[c] = S.iterations[c];
            ctl->updates[c] = S.updates[c];
            ctl->certs[c] = S.certs[c];
            ctl->warnings[c] = S.warnings[c];
            ctl->edges[c] = S.edges[c];
            ctl->max_change[c] = S.max_change[c];
            ctl->converged[c] = S.converged[c];
        }
        ctl->rounds = R;
    }
}

void lp_setup(Engine& E) {
    if (E.lp_grid) return;
    if (E.ncol > kMaxCols) throw CudaFailure(cudaErrorInvalidValue, "ncol > kMaxCols", __FILE__, __LINE__);
    E.lp_smem = (size_t)kWin * (E.ncol + 1) * sizeof(double);
    DLP_CUDA_TRY(cudaFuncSetAttribute(k_lp_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)E.lp_smem));
    int occ = 0;
    DLP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lp_fused, kLpThreads, E.lp_smem));
    if (occ < 1) occ = 1;
    if (occ > 8) occ = 8;
    E.lp_grid = E.sm_count * occ;
    if (const char* g = getenv("DLP_LP_GRID")) E.lp_grid = atoi(g);
    for (auto& ev : E.lp_ev) DLP_CUDA_TRY(cudaEventCreate(&ev));
}

void lp_run_dev(Engine& E, double delta, long long max_iter, bool itlp) {
    lp_setup(E);
    LPParams P;
    P.row_start = E.row_start.p;
    P.row_len = E.row_len.p;
    P.nbr = E.nbr.p;
    P.w = E.wgt.p;
    P.X = E.f[0].p;
    P.Y = E.f[1].p;
    P.eligm = E.eligm.p;
    P.emask_store = E.emask_store.p;
    P.fmask0 = E.fmask[0].p;
    P.fmask1 = E.fmask[1].p;
    P.U0 = E.ulist[0].p;
    P.U1 = E.ulist[1].p;
    P.f0 = E.f0.p;
    P.elist = E.elist.p;
    P.ds = E.ds;
    P.ctl = E.ctl;
    P.delta = delta;
    P.max_iter = max_iter;
    P.C = E.ncol;
    P.itlp = itlp ? 1 : 0;
    DLP_CUDA_TRY(cudaMemsetAsync(E.ctl, 0, sizeof(LPCtl), E.st));
    void* args[] = {&P};
    DLP_CUDA_TRY(cudaEventRecord(E.lp_ev[0], E.st));
    DLP_CUDA_TRY(cudaLaunchCooperativeKernel((void*)k_lp_fused, dim3(E.lp_grid), dim3(kLpThreads), args, E.lp_smem,
                                             E.st));
    DLP_CUDA_TRY(cudaEventRecord(E.lp_ev[1], E.st));
    E.launches++;
}

// ---------------------------------------------------------------------------
// ItLP active set (baselines.py:208-218): alive & unlabeled & degree > 0;
// isolated unlabeled vertices are pinned to 0.5 and counted.
// ---------------------------------------------------------------------------
__global__ void k_itlp_active(long long n, const unsigned char* alive, const signed char* gt, const int* row_len,
                              int ncol, double* f0, double* f1, unsigned int* eligm, int* alist, DevState* ds) {
    unsigned int allc = ncol >= 32 ? 0xffffffffu : ((1u << ncol) - 1u);
    long long iso = 0;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x) {
        bool unl = alive[v] && gt[v] == -1;
        eligm[v] = (unl && row_len[v] > 0) ? allc : 0u;
        if (!unl) continue;
        if (row_len[v] > 0) {
            append_agg(alist, &ds->n_elist, (int)v);
        } else {
            iso++;
            for (int c = 0; c < ncol; c++) {
                f0[v * ncol + c] = 0.5;
                f1[v * ncol + c] = 0.5;
            }
        }
    }
    iso = warp_sum(iso);
    if ((threadIdx.x & 31) == 0 && iso) atomicAdd((unsigned long long*)&ds->isolated, (unsigned long long)iso);
}

void itlp_active_dev(Engine& E, long long n) {
    if (n == 0) return;
    k_itlp_active<<<blocks_for(n, kBlock, 148 * 64), kBlock, 0, E.st>>>(n, E.alive.p, E.gt.p, E.row_len.p, E.ncol,
                                                                       E.f[0].p, E.f[1].p, E.eligm.p, E.elist.p,
                                                                       E.ds);
    E.launches++;
}

}  // namespace dlp
