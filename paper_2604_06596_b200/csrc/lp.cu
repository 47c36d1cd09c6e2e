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
// * The LP view (k_lp_view, per batch, cached per row): each row's unlabeled
//   neighbours and its row constants w_all and w0/w_all, w1/w_all per column,
//   so the sweeps run only the s chain of _update_one in the reference's order.
// * Row classes by view length: short rows (32/C per warp tile), long rows
//   (one per warp tile), hub rows (a whole CTA per row in small rounds, where
//   the longest row is the critical path; warp tiles in big rounds).  A warp
//   tile gathers entry-parallel into warp-private shared memory (64-entry
//   windows, ids one window ahead, label rows by cp.async) and lane
//   (row, column) runs its row's sum in stored order.
// * Jacobi commit: phase 1 writes new values to a compact staging buffer
//   (indexed by work item), phase 2 copies them into X; two grid-wide
//   barriers per round, the controller replayed by every CTA.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "engine.cuh"

namespace cg = cooperative_groups;

namespace dlp {

constexpr int kLpThreads = 256;
#ifndef DLP_WIN
#define DLP_WIN 64
#endif
#ifndef DLP_LABEL_WIN
#define DLP_LABEL_WIN 64  // C-wide label rows staged per warp window (>= DLP_WIN)
#endif
#ifndef DLP_HUB_WIN
#define DLP_HUB_WIN 192  // hub window (entries); 128: +1.3-1.7% on C2
#endif
#ifndef DLP_LP_MINB
#define DLP_LP_MINB 2
#endif
#ifndef DLP_ACC_UNROLL
#define DLP_ACC_UNROLL 4
#endif
constexpr int kAccUnroll = DLP_ACC_UNROLL;  // ordered-sum loop unroll
#ifndef DLP_EXPAND_REGS
#define DLP_EXPAND_REGS 1
#endif
constexpr bool kExpandRegs = DLP_EXPAND_REGS;  // expand single-window tiles from the gather registers
constexpr int kWin = DLP_WIN;   // row entries per warp window
constexpr int kHubWin = DLP_HUB_WIN;  // row entries per CTA window (hub rows)
#ifndef DLP_LONG_ROW_DEFAULT
#define DLP_LONG_ROW_DEFAULT 96
#endif
constexpr int kLongRow = DLP_LONG_ROW_DEFAULT;  // rows longer than this are warp tiles of their own
#ifndef DLP_HUB_ROW_DEFAULT
#define DLP_HUB_ROW_DEFAULT 512
#endif
constexpr int kHubRow = DLP_HUB_ROW_DEFAULT;  // rows longer than this are evaluated by a whole CTA
#ifndef DLP_SCAN_RATIO
#define DLP_SCAN_RATIO 16
#endif
constexpr int kScanRatio = DLP_SCAN_RATIO;  // rounds with >= n/16 rows: expand by atomicOr + compaction, hubs as warp tiles (64: +4%)

enum { PH_FRONTIER = 0, PH_DONE = 2 };
enum { CLS_SHORT = 0, CLS_LONG = 1, CLS_HUB = 2 };

// row-class thresholds (kLongRow / kHubRow by default; DLP_LONG_ROW / DLP_HUB_ROW override)
__constant__ int c_long_row = kLongRow;
__constant__ int c_hub_row = kHubRow;
__device__ inline int row_class(int len) {
    return len > c_hub_row ? CLS_HUB : (len > c_long_row ? CLS_LONG : CLS_SHORT);
}
// The prologue stores each eligible vertex's row class in bits 24-25 of its
// eligibility word (column bits stay in 0-15), so claims and compaction get
// the class from the word they already read.
constexpr int kClassShift = 24;
__device__ inline int elig_class(unsigned int e) { return (int)((e >> kClassShift) & 3u); }

struct LPParams {
    const long long* row_start;
    const int* row_len;  // full row length (edges_traversed)
    const int* nbr;
    const double* w;
    // LP view (k_lp_view): unlabeled neighbours at the row's offset, their
    // count, and the row constants w_all and (w0 / w_all, w1 / w_all) per column
    const int* vnbr;
    const double* vw;
    const int* vlen;
    const double* wsum;
    const double* q01;
    double* X;  // canonical labels [v*C + c]
    double* Y;  // compact staging: [i*C + c] for work item i of the round
    unsigned int* eligm;
    unsigned int* emask_store;  // evaluated column mask per work item of the round
    unsigned int* fmask[2];
    int* flist[3][2];  // union frontier lists per row class (rotating)
    int* elist_c[3];   // eligible list split by row class (prologue)
    const int* f0;
    const int* elist;
    const DevState* ds;
    LPCtl* ctl;
    double delta;
    long long max_iter;
    long long n;  // vertex slots
    int C;
    int itlp;
    int action_mode;  // execute ctl->act[] once per column, then exit (sharded batches)
    int cleanup;      // action mode: clear the leftover frontier masks and exit
    int cert_hold;    // max rounds a column's certify sweep waits for the other columns
    // row-partitioned mode (one round per launch): work-item log of the round
    // (vertex, evaluated mask, changed mask), exchanged by the host
    int* log_u;
    unsigned int* log_em;
    unsigned int* log_chg;
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
    int hold;  // rounds the waiting certify sweeps have been held (certify alignment)
    int done;
};

// ---- cache-policy loads: labels stay L2-resident, adjacency streams -------
__device__ inline unsigned long long l2_evict_last_policy() {
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ inline double ld_keep(const double* p, unsigned long long pol) {
    double v;
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ inline void st_keep(double* p, double v, unsigned long long pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}

// warp-aggregated append: every converged caller must pass the same list/count
// cp.async (LDGSTS) global -> shared with the label L2 policy
__device__ inline void cp_async8(double* dst, const double* src, unsigned long long pol) {
    unsigned int d = (unsigned int)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "l"(pol)
                 : "memory");
}
__device__ inline void cp_async16(double* dst, const double* src, unsigned long long pol) {
    unsigned int d = (unsigned int)__cvta_generic_to_shared(dst);
#ifdef DLP_CP16_CA  // variant: keep the label rows in L1 as well
    asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "l"(pol)
                 : "memory");
#else
    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "l"(pol)
                 : "memory");
#endif
}
__device__ inline void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// copy the C-wide label vector of one vertex (16-byte chunks when C is even:
// rows start 16-byte aligned in both global and shared memory)
__device__ inline void copy_label_row(double* dst, const double* src, int C, unsigned long long pol) {
    if ((C & 1) == 0) {
        for (int q = 0; q < C; q += 2) cp_async16(dst + q, src + q, pol);
    } else {
        for (int q = 0; q < C; q++) cp_async8(dst + q, src + q, pol);
    }
}

// warp-aggregated append: every converged caller must pass the same list/count
__device__ inline void append_u32(int* list, unsigned int* count, int v) {
    cg::coalesced_group g = cg::coalesced_threads();
    unsigned int base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(count, g.size());
    base = g.shfl(base, 0);
    list[base + g.thread_rank()] = v;
}

// Where a round's claims go (the same for every thread of a round: kept in
// shared memory, not in each thread's registers).
struct ClaimTargets {
    unsigned int* fm_next;
    int* next[3];
    unsigned int* cnt;  // [3]
    const unsigned int* eligm;
};

struct ClaimCtx {
    const ClaimTargets* t;
    unsigned int claimed;  // per-thread OR of claimed column bits
    // per-lane round counters of the lane's label column (flushed once per round)
    unsigned int c_nev, c_warn;
    unsigned long long c_edg;
    double c_rmax;
    __device__ inline unsigned int* fm_next() const { return t->fm_next; }
};

// append-mode claim: add v (for the columns in `bits` where it is eligible)
// to the next union frontier; the first claimer appends it to its class list
__device__ inline void claim(ClaimCtx& k, int v, unsigned int bits) {
    const ClaimTargets& t = *k.t;
    const unsigned int e = t.eligm[v];
    bits &= e;
    if (!bits) return;
    k.claimed |= bits;
    unsigned int* fm = t.fm_next + v;
    unsigned int cur = *(volatile unsigned int*)fm;
    if ((cur & bits) == bits) return;
    unsigned int old = atomicOr(fm, bits);
    if (old != 0) return;
    const int cls = elig_class(e);
    if (cls == CLS_SHORT)
        append_u32(t.next[0], &t.cnt[0], v);
    else if (cls == CLS_LONG)
        append_u32(t.next[1], &t.cnt[1], v);
    else
        append_u32(t.next[2], &t.cnt[2], v);
}

// Controller: every block updates its shared copy of the per-column state
// from the finished round's slot and decides the next round's actions.
__device__ void decide_actions(ColState& S, const LPParams& P, const unsigned long long* res, const unsigned int* claimed,
                               int first) {
    int C = P.C;
    unsigned int fr = 0, ce = 0;
    int done = 1;
    for (int c = 0; c < C; c++) {
        unsigned int bit = 1u << c;
        if (!first && S.phase[c] != PH_DONE) {
            bool was_fr = (S.fr_mask & bit) != 0, was_ce = (S.cert_mask & bit) != 0;
            if (was_fr || was_ce) {
                double rm = __longlong_as_double((long long)res[c]);
                S.iterations[c]++;
                S.updates[c] += (long long)res[kMaxCols + c];
                S.edges[c] += (long long)res[2 * kMaxCols + c];
                S.warnings[c] += (long long)res[3 * kMaxCols + c];
                S.has_frontier[c] = (*claimed & bit) != 0;
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
    // Certify alignment.  Columns are independent reference runs; the global
    // round is only a schedule.  A column whose jacobi_run returned waits
    // (does nothing: its frontier is empty and nothing it reads changes) while
    // other columns still run frontier rounds, so the certify sweeps of
    // several columns land in the same global round and share one gather of
    // every eligible row instead of one full gather per column.  Per-column
    // action sequences -- and so every result -- are unchanged.
    if (!P.itlp && ce && fr && S.hold < P.cert_hold) {
        S.hold++;
        ce = 0;
    } else {
        S.hold = 0;
    }
    S.fr_mask = fr;
    S.cert_mask = ce;
    S.done = done;
}

// Action-mode controller: columns execute the action the host assigned and
// stop at its end (frontier phase: local frontier empty or budget reached;
// certify: one round).  Phase statistics accumulate in S and go to ctl.
__device__ void decide_actions_act(ColState& S, const LPParams& P, const unsigned long long* res,
                                   const unsigned int* claimed, int first) {
    const int C = P.C;
    unsigned int fr = 0, ce = 0;
    int done = 1;
    for (int c = 0; c < C; c++) {
        const unsigned int bit = 1u << c;
        if (S.phase[c] == PH_DONE) continue;
        const int act = P.ctl->act[c];
        if (!first) {
            const bool was_fr = (S.fr_mask & bit) != 0, was_ce = (S.cert_mask & bit) != 0;
            if (was_fr || was_ce) {
                S.iterations[c]++;  // rounds of this action
                S.updates[c] += (long long)res[kMaxCols + c];
                S.edges[c] += (long long)res[2 * kMaxCols + c];
                S.warnings[c] += (long long)res[3 * kMaxCols + c];
                S.max_change[c] = __longlong_as_double((long long)res[c]);
                S.has_frontier[c] = (*claimed & bit) != 0;
                if (was_ce) {
                    S.phase[c] = PH_DONE;
                    continue;
                }
            }
        }
        if (act == ACT_FRONTIER && S.has_frontier[c] && S.iterations[c] < P.ctl->budget[c]) {
            fr |= bit;
            done = 0;
        } else if (act == ACT_CERTIFY && S.it_run[c] == 0) {
            S.it_run[c] = 1;
            ce |= bit;
            done = 0;
        } else {
            S.phase[c] = PH_DONE;
        }
    }
    S.fr_mask = fr;
    S.cert_mask = ce;
    S.done = done;
}

// Per-block counters of one round (reduced into the round slot at its end).
struct BlockCounters {
    unsigned long long rmax[kMaxCols], neval[kMaxCols], edges[kMaxCols], warn[kMaxCols];
    unsigned long long urows, uent;
    unsigned int claimed;
};

// Per-warp tile descriptors (rows of the tile, their masks and offsets).
struct WarpTile {
    long long st[32];
    int u[32], len[32], lenf[32], off[33], gtn[32];
    unsigned int em[32], chg[32];
};

__device__ inline int tile_row_of(const int* off, int nrows, int g) {
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

// ---------------------------------------------------------------------------
// The LP view.  Within a batch the ground truth is fixed, so the parts of
// _update_one (kernels/_csr.pyx:38-58) that only depend on it are constants
// of the batch: w_all (every entry's weight, row order), w0 / w1 (weights of
// class-0 / class-1 ground-truth neighbours, row order, per one-vs-rest
// column) and the quotients w0 / w_all, w1 / w_all of the formula.  k_lp_view
// computes them once per batch with the reference's summation order, and
// writes each row's UNLABELED neighbours (row order kept) to a second pool at
// the row's own offset.  The sweeps then only run the s chain
// (s += (f[v] - fu) * w over unlabeled neighbours, the reference's order with
// the ground-truth entries -- which add nothing to s -- left out): no
// per-entry ground-truth test, no w_all / w0 / w1 chains, one division per
// update instead of three.  Bit-identical: every value is produced by the
// same IEEE operations on the same operands in the same order.
// ---------------------------------------------------------------------------
// vlen[u] carries the view length and, in bit 30, "the row has a ground-truth
// neighbour": rows without one have w0 = w1 = 0, and their quotients are not
// loaded (the formula's two products are then +-0.0, which leave fu + ...
// unchanged exactly as the reference's (0 - fu) * (0 / w_all) terms do)
constexpr int kVlenGt = 1 << 30;
__device__ inline int vlen_len(int x) { return x & (kVlenGt - 1); }

__global__ void k_lp_view(const int* elist, const DevState* ds, const long long* row_start, const int* row_len,
                          const int* nbr, const double* wgt, const signed char* gt, int C, int* vnbr, double* vw,
                          int* vlen, double* wsum, double* q01, const int* row_mod, int* view_b,
                          long long* view_st, int seq, int inval) {
    const int lane = threadIdx.x & 31;
    const long long nw = (long long)gridDim.x * blockDim.x / 32;
    const long long n = ds->n_elist;
    const unsigned int below = (1u << lane) - 1u;
    for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32; i < n; i += nw) {
        const int u = elist[i];
        const long long st = row_start[u];
        // cached: built after the row's last change, at its current offset,
        // after the last repack of the pool
        const int vb = view_b[u];
        if (vb > 0 && vb >= row_mod[u] && vb > inval && view_st[u] == st) continue;
        const int len = row_len[u];
        double wa = 0.0, w0 = 0.0, w1 = 0.0;  // lane c < C: column c's w0 / w1
        int cnt = 0;
        for (int b = 0; b < len; b += 32) {
            const int e = b + lane;
            const bool valid = e < len;
            const int y = valid ? nbr[st + e] : 0;
            const double x = valid ? wgt[st + e] : 0.0;
            const int g = valid ? (int)gt[y] : -1;
            const bool unl = valid && g < 0;
            const unsigned int m = __ballot_sync(0xffffffffu, unl);
            if (unl) {
                const long long p = st + cnt + __popc(m & below);
                vnbr[p] = y;
                vw[p] = x;
            }
            cnt += __popc(m);
            const int nv = min(32, len - b);
            for (int j = 0; j < nv; j++) wa = __dadd_rn(wa, __shfl_sync(0xffffffffu, x, j));
            unsigned int gm = __ballot_sync(0xffffffffu, valid && g >= 0);
            while (gm) {
                const int j = __ffs(gm) - 1;
                gm &= gm - 1;
                const int gj = __shfl_sync(0xffffffffu, g, j);
                const double xj = __shfl_sync(0xffffffffu, x, j);
                if (lane < C) {
                    const bool one = C == 1 ? gj == 1 : gj == lane;
                    if (one)
                        w1 = __dadd_rn(w1, xj);
                    else
                        w0 = __dadd_rn(w0, xj);
                }
            }
        }
        if (lane == 0) {
            vlen[u] = cnt | (cnt < row_len[u] ? kVlenGt : 0);
            wsum[u] = wa;
            view_b[u] = seq;
            view_st[u] = st;
        }
        if (lane < C) {
            const long long q = ((long long)u * C + lane) * 2;
            q01[q] = wa > 0.0 ? __ddiv_rn(w0, wa) : 0.0;
            q01[q + 1] = wa > 0.0 ? __ddiv_rn(w1, wa) : 0.0;
        }
    }
}

// the label-difference sum of _update_one over a row's unlabeled neighbours
struct RowS {
    double s;
    __device__ inline void init() { s = 0.0; }
    template <int B>
    __device__ inline void add_block(const double* w, const double* x, int xs, double fu) {
        double p[B];
#pragma unroll
        for (int j = 0; j < B; j++) p[j] = __dmul_rn(__dsub_rn(x[j * xs], fu), w[j]);
#pragma unroll
        for (int j = 0; j < B; j++) s = __dadd_rn(s, p[j]);
    }
    __device__ inline void add(double w, double x, double fu) { s = __dadd_rn(s, __dmul_rn(__dsub_rn(x, fu), w)); }
};

// _csr.pyx:49-58 from the row constants: returns |fn - fu|, or -1 with value
// 0.5 for the isolated sentinel (w_all <= 0)
__device__ inline double finish_view(double s, double wall, const double* q, double fu, double* out) {
    if (wall <= 0.0) {
        *out = 0.5;
        return -1.0;
    }
    const double a = __dmul_rn(__dsub_rn(0.0, fu), q[0]);
    const double b = __dmul_rn(__dsub_rn(1.0, fu), q[1]);
    const double c = __ddiv_rn(s, wall);
    double fn = __dadd_rn(__dadd_rn(__dadd_rn(fu, a), b), c);
    if (fn < 0.0)
        fn = 0.0;
    else if (fn > 1.0)
        fn = 1.0;
    *out = fn;
    return fabs(__dsub_rn(fn, fu));
}

// Warp-private staging (doubles): the window's weights, its label rows
// (DLP_LABEL_WIN >= kWin C-wide rows) and the tile's row constants.  A warp
// tile holds rpt = 32 / C rows (one row per tile for the long class): lane
// (r, c) runs row r's sum for column c; a window stages the next kWin entries
// of the tile's concatenated rows (entry-parallel gathers) and a lane sums
// the part of its row inside the window.  (A step-major layout -- S entries
// of every row per window so all lanes advance together -- and a software
// pipeline across tiles were measured slower on C2 and its binary variant and
// removed.)
#ifndef DLP_RPL2
#define DLP_RPL2 0  // short rows: two rows per lane (C >= 2); measured slower on C2 (100.5 vs 81.0 ms), off
#endif
#ifndef DLP_WIN2
#define DLP_WIN2 128  // window of the two-rows-per-lane tiles
#endif
constexpr bool kRpl2 = DLP_RPL2;
constexpr int kWin2 = DLP_WIN2;
constexpr int kRpl2MaxC = 10;  // its staging (kWin2 x C label words) must fit two CTAs per SM
constexpr int kWinW = DLP_WIN > DLP_WIN2 ? DLP_WIN : DLP_WIN2;  // weight slots of a warp window
constexpr int kRowConst = 160;  // per warp: w_all of each tile row, (q0, q1) of each (lane, pass)
constexpr int kLabelWin = DLP_LABEL_WIN > DLP_WIN ? DLP_LABEL_WIN : DLP_WIN;  // >= the window
__host__ __device__ inline int warp_smem_doubles(int C) {
    int lw = kLabelWin * C;
    if (kRpl2 && C >= 2 && C <= kRpl2MaxC && kWin2 * C > lw) lw = kWin2 * C;
    return kWinW + (lw > kWinW ? lw : kWinW) + kRowConst;
}
// the row constants of the tile, copied asynchronously with the first
// window's label words (sq = the warp's row-constant area); rows without a
// ground-truth neighbour get (0, 0) without a load
__device__ inline void tile_consts(const LPParams& P, const WarpTile& T, double* sq, int nrows, int ar, int ac,
                                   bool aact, unsigned long long pol, int q) {
    const int lane = threadIdx.x & 31;
    double* sl = sq + 32 + 64 * q + 2 * lane;
    if (aact) {
        if (T.gtn[ar]) {
            cp_async16(sl, P.q01 + ((long long)T.u[ar] * P.C + ac) * 2, pol);
        } else {
            sl[0] = 0.0;
            sl[1] = 0.0;
        }
    }
    if (q == 0 && lane < nrows && T.em[lane]) cp_async8(sq + lane, P.wsum + T.u[lane], pol);
}

// Round context shared by the tile routine.
struct RoundCtx {
    const int* W;           // work list of this row class
    long long ybase;        // staging slot of W[0]
    unsigned int FR, CE;    // column actions of the round
    const unsigned int* fm_cur;
    bool scan_mode;         // expand by fire-and-forget atomicOr + compaction
    unsigned long long* tmax;  // trace: longest evaluated row of the round (or null)
};

// Row metadata of one tile row (lane r holds row r): loads issued one tile
// ahead so their latency hides behind the current tile's gathers.
struct TileMeta {
    int u, len, lenf;  // view length (unlabeled neighbours, bit 30: ground-truth neighbour), full row length
    unsigned int em;
    long long st;
};
__device__ inline TileMeta load_meta(const LPParams& P, const RoundCtx& R, int u) {
    TileMeta m{u, 0, 0, 0u, 0};
    if (u >= 0) {
        m.em = P.itlp ? (R.CE & P.eligm[u]) : (((R.fm_cur[u] & R.FR) | R.CE) & P.eligm[u]);
        m.st = P.row_start[u];
        m.len = P.vlen[u];
        m.lenf = P.row_len[u];
    }
    return m;
}

// Tile prologue shared by both shapes: publish the rows, count them.
__device__ inline int tile_rows(const LPParams& P, const RoundCtx& R, BlockCounters& B, WarpTile& T, long long k0,
                                int nrows, const TileMeta& m, int* maxlen_out) {
    const int lane = threadIdx.x & 31;
    int len = 0;
    unsigned int em = 0;
    if (lane < nrows) {
        em = m.em;
        P.emask_store[R.ybase + k0 + lane] = em;  // by work item: the commit reads it coalesced
        len = em ? vlen_len(m.len) : 0;
        T.u[lane] = m.u;
        T.em[lane] = em;
        T.st[lane] = em ? m.st : 0;
        T.len[lane] = len;
        T.lenf[lane] = m.lenf;
        T.gtn[lane] = (m.len & kVlenGt) != 0;
        T.chg[lane] = 0u;
    }
    int maxlen = len, total = len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
        total += __shfl_xor_sync(0xffffffffu, total, o);
    }
    if (R.tmax && len) atomicMax(R.tmax, (unsigned long long)len);
    const unsigned int nz = __ballot_sync(0xffffffffu, em != 0);
    if (lane == 0 && nz) {
        atomicAdd(&B.urows, (unsigned long long)__popc(nz));
        atomicAdd(&B.uent, (unsigned long long)total);
    }
    *maxlen_out = maxlen;
    return total;
}

// Tile epilogue shared by both shapes: stage the new value of lane (ar, ac)'s
// (row, column), count, and flag the columns that moved by more than delta.
__device__ inline unsigned int tile_finish(const LPParams& P, const RoundCtx& R, ClaimCtx& K, const WarpTile& T,
                                          const double* sq, long long k0, int ar, int ac, bool aact, double s,
                                          double fu, int q) {
    unsigned int ch = 0;
    if (aact) {
        const int u = T.u[ar];
        const int C = P.C;
        double val;
        const double d = finish_view(s, sq[ar], sq + 32 + 64 * q + 2 * (threadIdx.x & 31), fu, &val);
        __stcs(P.Y + (R.ybase + k0 + ar) * C + ac, val);
        K.c_nev++;
        K.c_edg += (unsigned long long)T.lenf[ar];
        if (d < 0.0) {  // isolated sentinel (_csr.pyx:49-51, 170-173)
            K.c_warn++;
            atomicAnd(&P.eligm[u], ~(1u << ac));
            atomicAdd((unsigned long long*)&P.ctl->elig_count[ac], ~0ULL);
        } else {
            K.c_rmax = fmax(K.c_rmax, d);
            if (!P.itlp && d > P.delta) ch = 1u << ac;
        }
    }
    return ch;
}

// Expand (jacobi_run commit loop, _csr.pyx:175-191): the changed rows claim
// themselves and their (unlabeled) neighbours -- ground-truth neighbours are
// never eligible, so the view's entries are exactly the candidates.
__device__ inline void tile_expand(const LPParams& P, const RoundCtx& R, ClaimCtx& K, WarpTile& T, long long k0,
                                   int nrows) {
    const int lane = threadIdx.x & 31;
    __syncwarp();
    const unsigned int mrow = lane < nrows ? T.chg[lane] : 0u;
    if (mrow) {
        K.claimed |= mrow;  // u changed, so u itself is eligible for those columns
        if (P.log_chg) P.log_chg[R.ybase + k0 + lane] = mrow;
        if (R.scan_mode)
            atomicOr(&K.fm_next()[T.u[lane]], mrow);
        else
            claim(K, T.u[lane], mrow);
    }
    const int clen = mrow ? T.len[lane] : 0;
    int incl = clen;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane < nrows) T.off[lane] = incl - clen;
    const int ctot = __shfl_sync(0xffffffffu, incl, 31);
    __syncwarp();
    for (int g = lane; g < ctot; g += 32) {
        const int r = tile_row_of(T.off, nrows, g);
        const unsigned int mq = T.chg[r];
        const int v = __ldcs(P.vnbr + T.st[r] + (g - T.off[r]));
        if (R.scan_mode)
            atomicOr(&K.fm_next()[v], mq);  // no return value: a fire-and-forget RED
        else
            claim(K, v, mq);
    }
}

// Flat tile: rows W[k0 ..] (metadata m, lane r holds row r); windows of kWin
// entries of the concatenated rows, ids and weights loaded one window ahead,
// label rows by cp.async; lane (r, c) sums its row's part of each window in
// stored order.  `un` is the next tile's row of this lane (-1 if none),
// whose metadata is loaded into *mn mid-tile.
template <int RPL, int WIN>
__device__ void warp_tile_flat(const LPParams& P, const RoundCtx& R, ClaimCtx& K, BlockCounters& B, WarpTile& T,
                               double* sw, double* sx, double* sq, long long k0, int nrows, unsigned long long pol,
                               const TileMeta& m, int un, TileMeta* mn) {
    // RPL rows per lane: lane (r, c) runs the sums of rows r and r + 32/C
    // (RPL = 2, C >= 2), two independent chains per lane and twice the
    // gathers in flight per warp.
    const int C = P.C;
    const int lane = threadIdx.x & 31;
    const int rpt1 = 32 / C;
    int maxlen;
    const int total = tile_rows(P, R, B, T, k0, nrows, m, &maxlen);
    int incl = lane < nrows ? T.len[lane] : 0;
    __syncwarp();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane < nrows) T.off[lane] = incl - T.len[lane];
    __syncwarp();
    const int ar0 = lane / C, ac = lane - ar0 * C;
    int arq[RPL], a_lo[RPL], a_hi[RPL];
    bool aact[RPL];
    double fu[RPL];
    RowS acc[RPL];
#pragma unroll
    for (int q = 0; q < RPL; q++) {
        arq[q] = ar0 + q * rpt1;
        aact[q] = ar0 < rpt1 && arq[q] < nrows && ((T.em[arq[q]] >> ac) & 1u);
        fu[q] = aact[q] ? ld_keep(P.X + (long long)T.u[arq[q]] * C + ac, pol) : 0.0;
        tile_consts(P, T, sq, nrows, arq[q], ac, aact[q], pol, q);
        a_lo[q] = aact[q] ? T.off[arq[q]] : 0;
        a_hi[q] = aact[q] ? T.off[arq[q]] + T.len[arq[q]] : 0;
        acc[q].init();
    }
    *mn = load_meta(P, R, un);  // next tile's metadata, consumed next iteration
    int vv[WIN / 32], rr[WIN / 32];
    double ww[WIN / 32];
#pragma unroll
    for (int j = 0; j < WIN / 32; j++) rr[j] = -1;  // a tile whose rows have no unlabeled entry runs no window
    auto load_ids = [&](int wb) {
        const int wn = min(WIN, total - wb);
#pragma unroll
        for (int j = 0; j < WIN / 32; j++) {
            const int i = lane + 32 * j;
            rr[j] = -1;
            if (i < wn) {
                const int g = wb + i;
                const int r = tile_row_of(T.off, nrows, g);
                const long long p = T.st[r] + (g - T.off[r]);
                rr[j] = r;
                vv[j] = __ldcs(P.vnbr + p);
                ww[j] = __ldcs(P.vw + p);
            }
        }
    };
    if (total > 0) load_ids(0);
    for (int wb = 0; wb < total; wb += WIN) {
        const int wn = min(WIN, total - wb);
#pragma unroll
        for (int j = 0; j < WIN / 32; j++) {
            if (rr[j] < 0) continue;
            const int i = lane + 32 * j;
            sw[i] = ww[j];
            copy_label_row(sx + i * C, P.X + (long long)vv[j] * C, C, pol);
        }
        if (wb + WIN < total) load_ids(wb + WIN);
        cp_async_wait_all();
        __syncwarp();
        if (RPL == 1) {
            if (aact[0]) {
                const int lo = max(a_lo[0], wb) - wb, hi = min(a_hi[0], wb + wn) - wb;
                int t = lo;
                for (; t + kAccUnroll <= hi; t += kAccUnroll)
                    acc[0].add_block<kAccUnroll>(sw + t, sx + t * C + ac, C, fu[0]);
                for (; t < hi; t++) acc[0].add(sw[t], sx[t * C + ac], fu[0]);
            }
        } else {  // both rows' segments advance in the same loop: two chains per lane
            int lo[RPL], n[RPL];
#pragma unroll
            for (int q = 0; q < RPL; q++) {
                lo[q] = aact[q] ? max(a_lo[q], wb) - wb : 0;
                n[q] = aact[q] ? max(0, min(a_hi[q], wb + wn) - wb - lo[q]) : 0;
            }
            int j = 0;
            const int nb = min(n[0], n[1]);
            for (; j + kAccUnroll <= nb; j += kAccUnroll) {
#pragma unroll
                for (int q = 0; q < RPL; q++)
                    acc[q].add_block<kAccUnroll>(sw + lo[q] + j, sx + (lo[q] + j) * C + ac, C, fu[q]);
            }
#pragma unroll
            for (int q = 0; q < RPL; q++) {
                int t = lo[q] + j;
                const int hi = lo[q] + n[q];
                for (; t + kAccUnroll <= hi; t += kAccUnroll)
                    acc[q].add_block<kAccUnroll>(sw + t, sx + t * C + ac, C, fu[q]);
                for (; t < hi; t++) acc[q].add(sw[t], sx[t * C + ac], fu[q]);
            }
        }
        __syncwarp();
    }
    if (total == 0) {  // no window ran: the row constants' copies must still land
        cp_async_wait_all();
        __syncwarp();
    }
    unsigned int ch[RPL];
#pragma unroll
    for (int q = 0; q < RPL; q++)
        ch[q] = tile_finish(P, R, K, T, sq, k0, arq[q], ac, aact[q], acc[q].s, fu[q], q);
    if (P.itlp) return;
    unsigned int chany = 0;
#pragma unroll
    for (int q = 0; q < RPL; q++) chany |= ch[q];
    if (!__any_sync(0xffffffffu, chany != 0)) return;
#pragma unroll
    for (int q = 0; q < RPL; q++)
        if (ch[q]) atomicOr(&T.chg[arq[q]], ch[q]);
    __syncwarp();
    if (kExpandRegs && total <= WIN) {
        // single-window tile: the gathering lanes still hold the entries' ids
        const unsigned int mrow = lane < nrows ? T.chg[lane] : 0u;
        if (mrow) {
            K.claimed |= mrow;
            if (P.log_chg) P.log_chg[R.ybase + k0 + lane] = mrow;
            if (R.scan_mode)
                atomicOr(&K.fm_next()[T.u[lane]], mrow);
            else
                claim(K, T.u[lane], mrow);
        }
#pragma unroll
        for (int j = 0; j < WIN / 32; j++) {
            if (rr[j] < 0) continue;
            const unsigned int mq = T.chg[rr[j]];
            if (!mq) continue;
            if (R.scan_mode)
                atomicOr(&K.fm_next()[vv[j]], mq);
            else
                claim(K, vv[j], mq);
        }
        return;
    }
    tile_expand(P, R, K, T, k0, nrows);
}

// Warp loop over the tiles of one row class: tile indices are grabbed two
// ahead and row metadata one ahead (software pipeline), so a tile's
// dependent chain of loads overlaps the previous tile's gathers.
__device__ void warp_tiles(const LPParams& P, const RoundCtx& R, int per, ClaimCtx& K, BlockCounters& B,
                           WarpTile& T, double* sw, double* sx, double* sq, unsigned int* grab, long long nitems,
                           unsigned long long pol, bool rpl2 = false) {
    const int lane = threadIdx.x & 31;
    if (nitems <= 0) return;
    unsigned int kr = 0;
    if (lane == 0) kr = atomicAdd(grab, (unsigned int)per);
    long long k = __shfl_sync(0xffffffffu, kr, 0);
    if (k >= nitems) return;
    int nr = (int)min((long long)per, nitems - k);
    TileMeta m = load_meta(P, R, lane < nr ? R.W[k + lane] : -1);
    if (lane == 0) kr = atomicAdd(grab, (unsigned int)per);
    for (;;) {
        const long long kn = __shfl_sync(0xffffffffu, kr, 0);
        const int nrn = kn < nitems ? (int)min((long long)per, nitems - kn) : 0;
        const int un = lane < nrn ? R.W[kn + lane] : -1;
        if (lane == 0 && kn < nitems) kr = atomicAdd(grab, (unsigned int)per);
        TileMeta mn;
        if (rpl2)
            warp_tile_flat<2, kWin2>(P, R, K, B, T, sw, sx, sq, k, nr, pol, m, un, &mn);
        else
            warp_tile_flat<1, kWin>(P, R, K, B, T, sw, sx, sq, k, nr, pol, m, un, &mn);
        __syncwarp();
        if (kn >= nitems) break;
        k = kn;
        nr = nrn;
        m = mn;
    }
}

// Hub row (view length > kHubRow) evaluated by the whole CTA, window by
// window (kHubWin entries): warps 1-7 gather a window's ids, weights and
// C-wide label rows and write the product terms (f[v] - fu) * w of every
// column into a double buffer, while warp 0 (lane c = column c) runs the
// s chain over the previous window's terms -- the only sequential part left
// (w_all, w0, w1 are row constants of the view), one DADD per entry.
__device__ void cta_hub_row(const LPParams& P, const RoundCtx& R, ClaimCtx& K, BlockCounters& B, double* buf,
                            double* s_fu, long long k, unsigned long long pol, int* s_i, long long* s_ll,
                            unsigned int* s_u32) {
    const int C = P.C;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // s_i: [0] u [1] len; s_ll[0] st; s_u32: [0] em [1] chg
    if (tid == 0) {
        int u = R.W[k];
        unsigned int em = P.itlp ? (R.CE & P.eligm[u]) : (((R.fm_cur[u] & R.FR) | R.CE) & P.eligm[u]);
        P.emask_store[R.ybase + k] = em;
        s_i[0] = u;
        s_u32[0] = em;
        s_u32[1] = 0;
        s_i[1] = em ? vlen_len(P.vlen[u]) : 0;
        s_i[3] = em ? P.row_len[u] : 0;
        s_ll[0] = em ? P.row_start[u] : 0;
        if (em) {
            if (R.tmax) atomicMax(R.tmax, (unsigned long long)s_i[1]);
            atomicAdd(&B.urows, 1ULL);
            atomicAdd(&B.uent, (unsigned long long)s_i[1]);
        }
    }
    __syncthreads();
    const unsigned int em = s_u32[0];
    if (!em) return;
    const int u = s_i[0], len = s_i[1], lenf = s_i[3];
    const long long st = s_ll[0];
    if (tid < C) s_fu[tid] = P.X[(long long)u * C + tid];
    __syncthreads();
    const int nwin = (len + kHubWin - 1) / kHubWin;
    const int bsz = kHubWin * C;  // terms of one window
    constexpr int kGth = kLpThreads - 32;
    constexpr int kPer = (kHubWin + kGth - 1) / kGth;
    const int g = tid - 32;
    int pv[kPer];
    double pw[kPer];
    auto load_ids = [&](int w) {
        const int wb = w * kHubWin, wn = min(kHubWin, len - wb);
#pragma unroll
        for (int j = 0; j < kPer; j++) {
            const int i = g + kGth * j;
            if (i < wn) {
                pv[j] = __ldcs(P.vnbr + st + wb + i);
                pw[j] = __ldcs(P.vw + st + wb + i);
            }
        }
    };
    // terms of window w: label rows read straight into registers (16-byte
    // loads when C is even), one product per column
    auto terms = [&](int w) {
        double* tb = buf + (w & 1) * bsz;
        const int wn = min(kHubWin, len - w * kHubWin);
#pragma unroll
        for (int j = 0; j < kPer; j++) {
            const int i = g + kGth * j;
            if (i < wn) {
                const double* xr = P.X + (long long)pv[j] * C;
                if ((C & 1) == 0) {
                    for (int c = 0; c < C; c += 2) {
                        const double2 x2 = *(const double2*)(xr + c);
                        tb[i * C + c] = __dmul_rn(__dsub_rn(x2.x, s_fu[c]), pw[j]);
                        tb[i * C + c + 1] = __dmul_rn(__dsub_rn(x2.y, s_fu[c + 1]), pw[j]);
                    }
                } else {
                    for (int c = 0; c < C; c++) tb[i * C + c] = __dmul_rn(__dsub_rn(ld_keep(xr + c, pol), s_fu[c]), pw[j]);
                }
            }
        }
    };
    if (warp > 0) {
        load_ids(0);
        terms(0);
        if (nwin > 1) load_ids(1);
    }
    __syncthreads();
    const bool act = warp == 0 && lane < C && ((em >> lane) & 1u);
    double s = 0.0;
    for (int w = 0; w < nwin; w++) {
        if (warp > 0) {
            if (w + 1 < nwin) {
                terms(w + 1);
                if (w + 2 < nwin) load_ids(w + 2);
            }
        } else if (act) {
            const double* tb = buf + (w & 1) * bsz + lane;
            const int wn = min(kHubWin, len - w * kHubWin);
            int t = 0;
            for (; t + 8 <= wn; t += 8) {
                double tv[8];
#pragma unroll
                for (int j = 0; j < 8; j++) tv[j] = lds64(tb + (t + j) * C);
#pragma unroll
                for (int j = 0; j < 8; j++) s = __dadd_rn(s, tv[j]);
            }
            for (; t < wn; t++) s = __dadd_rn(s, tb[t * C]);
        }
        __syncthreads();
    }
    if (act) {
        double val;
        const double d = finish_view(s, P.wsum[u], P.q01 + ((long long)u * C + lane) * 2, s_fu[lane], &val);
        __stcs(P.Y + (R.ybase + k) * C + lane, val);
        atomicAdd(&B.neval[lane], 1ULL);
        atomicAdd(&B.edges[lane], (unsigned long long)lenf);
        if (d < 0.0) {
            atomicAdd(&B.warn[lane], 1ULL);
            atomicAnd(&P.eligm[u], ~(1u << lane));
            atomicAdd((unsigned long long*)&P.ctl->elig_count[lane], ~0ULL);
        } else {
            if (d > 0.0) atomicMax(&B.rmax[lane], dbits(d));
            if (!P.itlp && d > P.delta) atomicOr(&s_u32[1], 1u << lane);
        }
    }
    __syncthreads();
    const unsigned int m = s_u32[1];
    if (m) {
        if (tid == 0) {
            K.claimed |= m;
            if (P.log_chg) P.log_chg[R.ybase + k] = m;
            if (R.scan_mode)
                atomicOr(&K.fm_next()[u], m);
            else
                claim(K, u, m);
        }
        for (int t = tid; t < len; t += kLpThreads) {
            int v = __ldcs(P.vnbr + st + t);
            if (R.scan_mode)
                atomicOr(&K.fm_next()[v], m);
            else
                claim(K, v, m);
        }
    }
    __syncthreads();
}

// Grid barrier of the persistent kernel: one arrival counter (a two-level
// variant with 16 group counters measured 1% slower at 444 CTAs).
__device__ inline void gsync(LPCtl* ctl, unsigned int& target) { grid_sync(&ctl->bar, target); }

__global__ void __launch_bounds__(kLpThreads, DLP_LP_MINB) k_lp_fused(LPParams P) {
    extern __shared__ double smem_dyn[];
    __shared__ ColState S;
    __shared__ ClaimTargets s_ct;        // the round's claim targets
    __shared__ BlockCounters B;
    __shared__ WarpTile TT[kLpThreads / 32];
    __shared__ unsigned long long s_res[4 * kMaxCols];
    __shared__ double s_fu[kMaxCols];
    __shared__ long long s_ll[2];
    __shared__ int s_i[4];
    __shared__ unsigned int s_u32[4], s_claimed, s_cnt[3], s_base[3];
    __shared__ unsigned int s_wc[3][kLpThreads / 32];

    const int C = P.C;
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const long long gtid = blockIdx.x * (long long)blockDim.x + tid;
    const long long gth = (long long)gridDim.x * blockDim.x;
    LPCtl* ctl = P.ctl;
    unsigned int target = 0;
    const int wsm = warp_smem_doubles(C);  // warp-private staging: weights, then label words
    double* sw = smem_dyn + warp * wsm;
    double* sx = sw + kWinW;
    double* sq = sw + wsm - kRowConst;  // row constants of the current tile
    WarpTile& T = TT[warp];
    const unsigned int allc = C >= 32 ? 0xffffffffu : ((1u << C) - 1u);
    const unsigned long long pol = l2_evict_last_policy();
    const long long n = P.n;

    // ---- prologue: F0 (engine.py:364-367) is every column's first frontier;
    // the eligible list and F0 are split by row class.  In action mode only
    // the first launch of a batch runs it; later launches resume the lists.
    const bool resume = P.action_mode && ctl->started;
    const long long n0 = P.itlp ? 0 : P.ds->n_f0;
    const long long n_el = P.ds->n_elist;
    if (!resume) {
        for (long long i = gtid; i < n0; i += gth) {
            int u = P.f0[i];
            P.fmask[0][u] = allc;
            // one call site per class: append_u32 aggregates over the converged
            // threads, which must all target the same list
            switch (row_class(vlen_len(P.vlen[u]))) {
                case CLS_SHORT: append_u32(P.flist[0][0], &ctl->n_f0[0], u); break;
                case CLS_LONG: append_u32(P.flist[1][0], &ctl->n_f0[1], u); break;
                default: append_u32(P.flist[2][0], &ctl->n_f0[2], u); break;
            }
        }
        for (long long i = gtid; i < n_el; i += gth) {
            int u = P.elist[i];
            const int cls = row_class(vlen_len(P.vlen[u]));
            P.eligm[u] |= (unsigned int)cls << kClassShift;
            switch (cls) {
                case CLS_SHORT: append_u32(P.elist_c[0], &ctl->n_el[0], u); break;
                case CLS_LONG: append_u32(P.elist_c[1], &ctl->n_el[1], u); break;
                default: append_u32(P.elist_c[2], &ctl->n_el[2], u); break;
            }
        }
    }
    if (tid == 0) {
        for (int c = 0; c < C; c++) {
            S.phase[c] = PH_FRONTIER;
            S.has_frontier[c] = resume ? ctl->has_fr[c] : (n0 > 0);
            S.it_run[c] = 0;
            S.mc_last[c] = 0.0;
            S.iterations[c] = S.updates[c] = S.certs[c] = S.warnings[c] = S.edges[c] = 0;
            S.max_change[c] = 0.0;
            S.converged[c] = P.itlp ? (n_el == 0) : 1;
            if (P.itlp && n_el == 0) S.phase[c] = PH_DONE;
            if (P.action_mode && (P.cleanup || ctl->act[c] == ACT_NONE)) S.phase[c] = PH_DONE;
        }
        S.fr_mask = S.cert_mask = 0;
        S.hold = 0;
        if (blockIdx.x == 0 && !resume)
            for (int c = 0; c < C; c++) ctl->elig_count[c] = n_el;
    }
    gsync(ctl, target);
    if (tid == 0) {
        if (P.action_mode)
            decide_actions_act(S, P, nullptr, nullptr, 1);
        else
            decide_actions(S, P, nullptr, nullptr, 1);
    }
    long long nel[3], ncur[3];
    for (int j = 0; j < 3; j++) {
        nel[j] = *(volatile unsigned int*)&ctl->n_el[j];
        ncur[j] = resume ? *(volatile unsigned int*)&ctl->ncur_p[j] : *(volatile unsigned int*)&ctl->n_f0[j];
    }
    __syncthreads();

    long long R = resume ? ctl->r_par : 0;
    while (!S.done) {
        unsigned long long t_r0 = 0, t_p1 = 0;
        if (ctl->trace && gtid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_r0));
        const unsigned int FR = S.fr_mask, CE = S.cert_mask;
        const int ri = (int)(R & 1), rn = ri ^ 1;
        RoundSlot* slot = &ctl->slot[ri];
        const int* W0 = CE ? P.elist_c[0] : P.flist[0][ri];
        const int* W1 = CE ? P.elist_c[1] : P.flist[1][ri];
        const int* W2 = CE ? P.elist_c[2] : P.flist[2][ri];
        const long long n0c = CE ? nel[0] : ncur[0];
        const long long n1c = CE ? nel[1] : ncur[1];
        const long long n2c = CE ? nel[2] : ncur[2];
        const long long nwork = n0c + n1c + n2c;
        const bool scan_mode = !P.itlp && nwork * kScanRatio >= n;
        unsigned int* fm_cur = P.fmask[ri];
        unsigned int* fm_next = P.fmask[rn];
        if (tid == 0) s_ct = ClaimTargets{fm_next, {P.flist[0][rn], P.flist[1][rn], P.flist[2][rn]}, slot->cnt, P.eligm};
        ClaimCtx K{&s_ct, 0u, 0u, 0u, 0ULL, 0.0};
        if (tid < kMaxCols) {
            B.rmax[tid] = 0;
            B.neval[tid] = 0;
            B.edges[tid] = 0;
            B.warn[tid] = 0;
        }
        if (tid == 0) {
            B.claimed = 0;
            B.urows = 0;
            B.uent = 0;
        }
        __syncthreads();

        unsigned long long p_tw0 = 0;
        // ======== phase 1: evaluate + expand ========
        // staging items: short [0, n0c), long [n0c, n0c+n1c), hub [n0c+n1c, nwork)
        {
            unsigned long long* tmax = (ctl->trace && R < ctl->trace_cap) ? ctl->trace + 8 * R + 7 : nullptr;
            RoundCtx RH{W2, n0c + n1c, FR, CE, fm_cur, scan_mode, tmax};
            unsigned long long tw1 = 0, tw2 = 0, tw3 = 0;
#ifdef DLP_PROF
            const bool prof = ctl->prof != nullptr && lane == 0;
#else
            constexpr bool prof = false;  // build with -DDLP_PROF for the phase-1 warp-time profile
#endif
            if (prof) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(p_tw0));
            const unsigned long long tw0 = p_tw0;
            // hub rows: whole CTA per row in small rounds, where the longest row is
            // the round's critical path; in big rounds (throughput-bound) they are
            // single-row warp tiles like long rows, so no CTA idles at the window
            // barriers (C2: 81.3 -> 79.8 ms)
#ifndef DLP_HUB_CTA_ALWAYS
            const bool hub_cta = !scan_mode;
#else
            constexpr bool hub_cta = true;
#endif
            if (n2c > 0 && hub_cta) {
                for (;;) {  // hub rows: whole CTA per row (critical path first)
                    if (tid == 0) s_i[2] = (int)atomicAdd(&slot->grab[2], 1u);
                    __syncthreads();
                    const int k = s_i[2];
                    __syncthreads();
                    if (k >= n2c) break;
                    cta_hub_row(P, RH, K, B, smem_dyn, s_fu, k, pol, s_i, s_ll, s_u32);
                }
            }
            RoundCtx RL{W1, n0c, FR, CE, fm_cur, scan_mode, tmax};
            RoundCtx RS{W0, 0, FR, CE, fm_cur, scan_mode, tmax};
            if (prof) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tw1));
            if (!hub_cta) warp_tiles(P, RH, 1, K, B, T, sw, sx, sq, &slot->grab[2], n2c, pol);
            warp_tiles(P, RL, 1, K, B, T, sw, sx, sq, &slot->grab[1], n1c, pol);  // long rows: one per tile
            if (prof) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tw2));
            // short rows: 32/C rows per tile, or 2 x 32/C with two rows per lane
            const bool rpl2 = kRpl2 && C >= 2 && C <= kRpl2MaxC;
            warp_tiles(P, RS, rpl2 ? 2 * (32 / C) : 32 / C, K, B, T, sw, sx, sq, &slot->grab[0], n0c, pol, rpl2);
            if (prof) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tw3));
            if (prof) {  // warp-time per part of phase 1 (diagnostics)
                atomicAdd(&ctl->prof[0], tw1 - tw0);
                atomicAdd(&ctl->prof[1], tw2 - tw1);
                atomicAdd(&ctl->prof[2], tw3 - tw2);
            }
        }
        if (K.claimed) atomicOr(&B.claimed, K.claimed);
        if (K.c_nev) {  // lane (row, c) of every tile works on column c = lane % C
            const int col = lane % C;
            atomicAdd(&B.neval[col], (unsigned long long)K.c_nev);
            atomicAdd(&B.edges[col], K.c_edg);
            if (K.c_warn) atomicAdd(&B.warn[col], (unsigned long long)K.c_warn);
            if (K.c_rmax > 0.0) atomicMax(&B.rmax[col], dbits(K.c_rmax));
        }
        __syncthreads();
        if (tid < C) {
            if (B.rmax[tid]) atomicMax(&slot->rmax[tid], B.rmax[tid]);
            if (B.neval[tid]) atomicAdd(&slot->neval[tid], B.neval[tid]);
            if (B.edges[tid]) atomicAdd(&slot->edges[tid], B.edges[tid]);
            if (B.warn[tid]) atomicAdd(&slot->warn[tid], B.warn[tid]);
        }
        if (tid == 0) {
            if (B.claimed) atomicOr(&slot->claimed, B.claimed);
            if (B.urows) atomicAdd(&slot->urows, B.urows);
            if (B.uent) atomicAdd(&slot->uentries, B.uent);
        }
        gsync(ctl, target);
        if (ctl->trace && gtid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_p1));
#ifdef DLP_PROF
        if (ctl->prof && (tid & 31) == 0) {
            unsigned long long tnow;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
            atomicAdd(&ctl->prof[3], tnow - p_tw0);  // warp-ns from phase-1 start to the grid barrier's exit
        }
#endif

        // ======== phase 2: commit (Jacobi), clear this round's masks ========
        // two items per thread in flight; full column masks move as 16-byte
        // vectors (rows of X and of the compact staging are 16-byte aligned
        // when C is even)
        for (long long i0 = gtid; i0 < nwork; i0 += 2 * gth) {
            int uu[2];
            unsigned int ee[2];
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const long long i = i0 + h * gth;
                uu[h] = -1;
                ee[h] = 0u;
                if (i < nwork) {
                    uu[h] = i < n0c ? W0[i] : (i < n0c + n1c ? W1[i - n0c] : W2[i - n0c - n1c]);
                    ee[h] = P.emask_store[i];  // coalesced, independent of the list lookup
                }
            }
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const long long i = i0 + h * gth;
                const int u = uu[h];
                if (u < 0) continue;
                if (P.log_u) {
                    P.log_u[i] = u;
                    P.log_em[i] = ee[h];
                }
                if (ctl->seen) {
                    int old = atomicExch(&ctl->seen[u], (int)(R + 1));
                    if (old == (int)(R + 1)) atomicAdd(&ctl->dups, 1ULL);
                }
                const unsigned int em = ee[h];
                double* xd = P.X + (long long)u * C;
                const double* yd = P.Y + i * C;
                if (em == allc && (C & 1) == 0) {
                    for (int c = 0; c < C; c += 2) {
                        double2 y = __ldcs((const double2*)(yd + c));
                        st_keep(xd + c, y.x, pol);
                        st_keep(xd + c + 1, y.y, pol);
                    }
                } else {
                    for (int c = 0; c < C; c++)
                        if ((em >> c) & 1u) st_keep(xd + c, __ldcs(yd + c), pol);
                }
                fm_cur[u] = 0;
            }
        }
        if (scan_mode) {
            // compaction of the claimed mask into the next class lists: one
            // contiguous vertex range per CTA, counted then written, so each CTA
            // issues a single atomic per list
            const long long chunk = ((n + gridDim.x - 1) / gridDim.x + 255) & ~255LL;
            const long long v0 = blockIdx.x * chunk, v1 = min(n, v0 + chunk);
            // pass 1 (independent coalesced loads, unrolled): drop ineligible
            // claims, count per class
            unsigned int cc[3] = {0u, 0u, 0u};
#pragma unroll 4
            for (long long v = v0 + tid; v < v1; v += kLpThreads) {
                const unsigned int bits = fm_next[v], e = P.eligm[v];
                if (!bits) continue;
                if (!(bits & e)) {
                    fm_next[v] = 0;  // claimed but ineligible: never evaluated
                    continue;
                }
                const int cls = elig_class(e);
                cc[0] += cls == 0;
                cc[1] += cls == 1;
                cc[2] += cls == 2;
            }
            for (int j = 0; j < 3; j++) {
                unsigned int x = warp_sum(cc[j]);
                if (lane == 0) s_wc[j][warp] = x;
            }
            __syncthreads();
            if (tid < 3) {
                unsigned int tot = 0;
                for (int w = 0; w < kLpThreads / 32; w++) {
                    unsigned int x = s_wc[tid][w];
                    s_wc[tid][w] = tot;
                    tot += x;
                }
                s_base[tid] = tot ? atomicAdd(&slot->cnt[tid], tot) : 0u;
            }
            __syncthreads();
            // pass 2 (L1-resident re-read): write the class lists
            const unsigned int below = (1u << lane) - 1u;
            unsigned int off0 = s_base[0] + s_wc[0][warp], off1 = s_base[1] + s_wc[1][warp],
                         off2 = s_base[2] + s_wc[2][warp];
            for (long long vb = v0; vb < v1; vb += kLpThreads) {
                const long long v = vb + tid;
                const unsigned int bits = v < v1 ? fm_next[v] : 0u;
                const int cls = bits ? elig_class(P.eligm[v]) : -1;
                const unsigned int b0 = __ballot_sync(0xffffffffu, cls == 0);
                const unsigned int b1 = __ballot_sync(0xffffffffu, cls == 1);
                const unsigned int b2 = __ballot_sync(0xffffffffu, cls == 2);
                if (cls == 0) P.flist[0][rn][off0 + __popc(b0 & below)] = (int)v;
                if (cls == 1) P.flist[1][rn][off1 + __popc(b1 & below)] = (int)v;
                if (cls == 2) P.flist[2][rn][off2 + __popc(b2 & below)] = (int)v;
                off0 += __popc(b0);
                off1 += __popc(b1);
                off2 += __popc(b2);
            }
        }
        if (gtid == 0) {
            if (P.log_u) ctl->log_n = nwork;
            RoundSlot* nx = &ctl->slot[rn];
            for (int c = 0; c < kMaxCols; c++) nx->rmax[c] = nx->neval[c] = nx->edges[c] = nx->warn[c] = 0;
            nx->claimed = 0;
            nx->urows = 0;
            nx->uentries = 0;
            for (int j = 0; j < 3; j++) nx->grab[j] = nx->cnt[j] = 0;
        }
        gsync(ctl, target);
        // controller: stage the slot's per-column results in shared memory
        // (parallel loads), then one thread replays the state machines
        {
            const volatile RoundSlot* vs = slot;
            if (tid < C) {
                s_res[tid] = vs->rmax[tid];
                s_res[kMaxCols + tid] = vs->neval[tid];
                s_res[2 * kMaxCols + tid] = vs->edges[tid];
                s_res[3 * kMaxCols + tid] = vs->warn[tid];
            }
            if (tid == 32) s_claimed = vs->claimed;
            if (tid >= 64 && tid < 67) s_cnt[tid - 64] = vs->cnt[tid - 64];
            if (blockIdx.x == 0 && tid == 128) {
                ctl->urows += (long long)vs->urows;
                ctl->uentries += (long long)vs->uentries;
                if (ctl->trace && R < ctl->trace_cap) ctl->trace[8 * R + 6] = vs->uentries;
            }
            __syncthreads();
            if (tid == 0) {
                if (P.action_mode)
                    decide_actions_act(S, P, s_res, &s_claimed, 0);
                else
                    decide_actions(S, P, s_res, &s_claimed, 0);
            }
        }
        for (int j = 0; j < 3; j++) ncur[j] = s_cnt[j];
        if (ctl->trace && gtid == 0 && R < ctl->trace_cap) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            unsigned long long* e = ctl->trace + 8 * R;
            e[4] = t_p1;
            e[5] = t_r0;
            e[0] = (unsigned long long)n0c;
            e[1] = (unsigned long long)(n1c + (n2c << 32));
            e[2] = (unsigned long long)FR | ((unsigned long long)CE << 16) | ((unsigned long long)scan_mode << 32);
            e[3] = t;
        }
        R++;
        __syncthreads();
    }
    if (P.action_mode && !P.cleanup) {
        // hand the lists and per-column phase results to the host
        gsync(ctl, target);  // every CTA has read ctl before it is rewritten
        if (gtid == 0) {
            for (int c = 0; c < C; c++) {
                ctl->has_fr[c] = S.has_frontier[c];
                ctl->ph_rounds[c] = S.iterations[c];
                ctl->ph_upd[c] = S.updates[c];
                ctl->ph_edges[c] = S.edges[c];
                ctl->ph_warn[c] = S.warnings[c];
                ctl->ph_mc[c] = S.max_change[c];
            }
            for (int j = 0; j < 3; j++) ctl->ncur_p[j] = (unsigned int)ncur[j];
            ctl->r_par = R;
            ctl->started = 1;
            ctl->rounds = R;
        }
        return;
    }
    // leftover frontiers (budget exhausted): clear their masks for the next batch
    {
        const int ri = (int)(R & 1);
        for (long long i = gtid; i < ncur[0] + ncur[1] + ncur[2]; i += gth) {
            int u = i < ncur[0] ? P.flist[0][ri][i]
                                : (i < ncur[0] + ncur[1] ? P.flist[1][ri][i - ncur[0]]
                                                         : P.flist[2][ri][i - ncur[0] - ncur[1]]);
            P.fmask[ri][u] = 0;
        }
    }
    if (gtid == 0 && !P.action_mode) {
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

// Keep the label matrix X resident in L2 across rounds: the gathers re-read
// it ~|E|/|V| times per round while the adjacency streams past it.  A
// persisting carve-out (cudaLimitPersistingL2CacheSize) makes the loads'
// evict_last hints effective, and an access-policy window on the engine's
// stream marks X itself persisting (the rest streams).  DLP_L2_PERSIST=0/1/2.
void l2_setup(Engine& E) {
    if (const char* v = getenv("DLP_L2_PERSIST")) E.l2_mode = atoi(v);
    if (E.l2_mode <= 0) return;
    int maxp = 0, maxw = 0;
    DLP_CUDA_TRY(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, E.device));
    DLP_CUDA_TRY(cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, E.device));
    E.l2_persist = (size_t)maxp;
    E.l2_window_max = (size_t)maxw;
    if (E.l2_persist) DLP_CUDA_TRY(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, E.l2_persist));
}

void l2_window(Engine& E, cudaStream_t st) {
    if (E.l2_mode < 2 || !E.l2_persist || !E.l2_window_max) return;
    const size_t bytes = std::min((size_t)E.n_slots * E.ncol * sizeof(double), E.l2_window_max);
    if (!bytes) return;
    cudaStreamAttrValue v;
    memset(&v, 0, sizeof(v));
    v.accessPolicyWindow.base_ptr = (void*)E.f[0].p;
    v.accessPolicyWindow.num_bytes = bytes;
    v.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)E.l2_persist / (double)bytes);
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    DLP_CUDA_TRY(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v));
}

void lp_setup(Engine& E) {
    if (E.lp_grid) return;
    l2_setup(E);
    if (E.ncol > kMaxCols) throw CudaFailure(cudaErrorInvalidValue, "ncol > kMaxCols", __FILE__, __LINE__);
    E.lp_smem = std::max((size_t)(kLpThreads / 32) * warp_smem_doubles(E.ncol),
                         (size_t)2 * kHubWin * E.ncol) * sizeof(double);
    DLP_CUDA_TRY(cudaFuncSetAttribute(k_lp_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)E.lp_smem));
    if (const char* v = getenv("DLP_CARVEOUT"))  // shared-memory share of L1 (percent), tuning
        DLP_CUDA_TRY(cudaFuncSetAttribute(k_lp_fused, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(v)));
    int occ = 0;
    DLP_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_lp_fused, kLpThreads, E.lp_smem));
    if (occ < 1) occ = 1;
    if (occ > 8) occ = 8;
    E.lp_grid = E.sm_count * occ;
    if (const char* g = getenv("DLP_LP_GRID")) E.lp_grid = atoi(g);
    E.lp_trace_path = getenv("DLP_LP_TRACE");
    if (const char* v = getenv("DLP_CERT_HOLD")) E.lp_cert_hold = atoi(v);
    if (const char* v = getenv("DLP_LONG_ROW")) {
        int x = atoi(v);
        DLP_CUDA_TRY(cudaMemcpyToSymbol(c_long_row, &x, sizeof(int)));
    }
    if (const char* v = getenv("DLP_HUB_ROW")) {
        int x = atoi(v);
        DLP_CUDA_TRY(cudaMemcpyToSymbol(c_hub_row, &x, sizeof(int)));
    }
    for (auto& ev : E.lp_ev) DLP_CUDA_TRY(cudaEventCreate(&ev));
}

// The batch's LP view (k_lp_view) over the eligible list; the view pool is
// the adjacency pool's compaction target (free between structure updates).
// Rows unchanged since their view was built keep it (row_mod from the
// batch's affected marks, view_b / view_st of the build, view_inval after a
// pool repack), so a batch rebuilds only the rows it touched.
void lp_build_view(Engine& E) {
    cudaStream_t st = E.st;
    if (E.nbr_sp.n < E.nbr.n || E.wgt_sp.n < E.wgt.n) {
        E.nbr_sp.reserve(E.nbr.n, 0, st);
        E.wgt_sp.reserve(E.wgt.n, 0, st);
        E.view_inval = E.view_seq - 1;
    }
    k_lp_view<<<E.sm_count * 8, kLpThreads, 0, st>>>(E.elist.p, E.ds, E.row_start.p, E.row_len.p, E.nbr.p, E.wgt.p,
                                                     E.gt.p, E.ncol, E.nbr_sp.p, E.wgt_sp.p, E.vlen.p, E.wsum.p,
                                                     E.q01.p, E.row_mod.p, E.view_b.p, E.view_st.p, E.view_seq,
                                                     E.view_inval);
    DLP_CUDA_TRY(cudaGetLastError());
    E.launches++;
}

static void view_params(Engine& E, LPParams& P) {
    P.vnbr = E.nbr_sp.p;
    P.vw = E.wgt_sp.p;
    P.vlen = E.vlen.p;
    P.wsum = E.wsum.p;
    P.q01 = E.q01.p;
}

void lp_run_dev(Engine& E, double delta, long long max_iter, bool itlp) {
    lp_setup(E);
    lp_build_view(E);
    LPParams P;
    view_params(E, P);
    P.row_start = E.row_start.p;
    P.row_len = E.row_len.p;
    P.nbr = E.nbr.p;
    P.w = E.wgt.p;
    P.X = E.f[0].p;
    P.Y = E.f[1].p;
    P.eligm = E.eligm.p;
    P.emask_store = E.emask_store.p;
    for (int i = 0; i < 2; i++) {
        P.fmask[i] = E.fmask[i].p;
        P.flist[0][i] = E.ulist[i].p;
        P.flist[1][i] = E.llist[i].p;
        P.flist[2][i] = E.hlist[i].p;
    }
    P.elist_c[0] = E.elist_s.p;
    P.elist_c[1] = E.elist_l.p;
    P.elist_c[2] = E.elist_h.p;
    P.f0 = E.f0.p;
    P.elist = E.elist.p;
    P.ds = E.ds;
    P.ctl = E.ctl;
    P.delta = delta;
    P.max_iter = max_iter;
    P.n = E.n_slots;
    P.C = E.ncol;
    P.itlp = itlp ? 1 : 0;
    P.action_mode = 0;
    P.cleanup = 0;
    P.cert_hold = E.lp_cert_hold;
    P.log_u = nullptr;
    P.log_em = P.log_chg = nullptr;
    DLP_CUDA_TRY(cudaMemsetAsync(E.ctl, 0, sizeof(LPCtl), E.st));
    if (E.lp_trace_path) {
        const long long cap = 1 << 16;
        E.lp_trace.reserve(8 * cap + 8, 0, E.st);
        DLP_CUDA_TRY(cudaMemsetAsync(E.lp_trace.p, 0, (8 * cap + 8) * sizeof(unsigned long long), E.st));
        unsigned long long* tp = E.lp_trace.p;
        DLP_CUDA_TRY(cudaMemcpyAsync(&E.ctl->trace, &tp, sizeof(tp), cudaMemcpyHostToDevice, E.st));
        DLP_CUDA_TRY(cudaMemcpyAsync(&E.ctl->trace_cap, &cap, sizeof(cap), cudaMemcpyHostToDevice, E.st));
        E.lp_seen.reserve(E.cap_n + 1, 0, E.st);
        DLP_CUDA_TRY(cudaMemsetAsync(E.lp_seen.p, 0, (E.cap_n + 1) * sizeof(int), E.st));
        int* sp = E.lp_seen.p;
        DLP_CUDA_TRY(cudaMemcpyAsync(&E.ctl->seen, &sp, sizeof(sp), cudaMemcpyHostToDevice, E.st));
        E.lp_prof.reserve(8, 0, E.st);
        DLP_CUDA_TRY(cudaMemsetAsync(E.lp_prof.p, 0, 8 * sizeof(unsigned long long), E.st));
        unsigned long long* pp = E.lp_prof.p;
        DLP_CUDA_TRY(cudaMemcpyAsync(&E.ctl->prof, &pp, sizeof(pp), cudaMemcpyHostToDevice, E.st));
        DLP_CUDA_TRY(cudaStreamSynchronize(E.st));  // host values above are stack temporaries
    }
    void* args[] = {&P};
    DLP_CUDA_TRY(cudaEventRecord(E.lp_ev[0], E.st));
    l2_window(E, E.st);
    DLP_CUDA_TRY(cudaLaunchCooperativeKernel((void*)k_lp_fused, dim3(E.lp_grid), dim3(kLpThreads), args, E.lp_smem,
                                             E.st));
    DLP_CUDA_TRY(cudaEventRecord(E.lp_ev[1], E.st));
    E.launches++;
}

// One action-mode launch (component-sharded batches): the host has written
// ctl->act / ctl->budget; first = first launch of the batch (full reset).
void lp_run_actions(Engine& E, double delta, bool first, bool cleanup) {
    lp_setup(E);
    if (first && !cleanup) lp_build_view(E);
    LPParams P;
    view_params(E, P);
    P.row_start = E.row_start.p;
    P.row_len = E.row_len.p;
    P.nbr = E.nbr.p;
    P.w = E.wgt.p;
    P.X = E.f[0].p;
    P.Y = E.f[1].p;
    P.eligm = E.eligm.p;
    P.emask_store = E.emask_store.p;
    for (int i = 0; i < 2; i++) {
        P.fmask[i] = E.fmask[i].p;
        P.flist[0][i] = E.ulist[i].p;
        P.flist[1][i] = E.llist[i].p;
        P.flist[2][i] = E.hlist[i].p;
    }
    P.elist_c[0] = E.elist_s.p;
    P.elist_c[1] = E.elist_l.p;
    P.elist_c[2] = E.elist_h.p;
    P.f0 = E.f0.p;
    P.elist = E.elist.p;
    P.ds = E.ds;
    P.ctl = E.ctl;
    P.delta = delta;
    P.max_iter = 0;
    P.n = E.n_slots;
    P.C = E.ncol;
    P.itlp = 0;
    P.action_mode = 1;
    P.cleanup = cleanup ? 1 : 0;
    P.cert_hold = 0;
    P.log_u = nullptr;
    P.log_em = P.log_chg = nullptr;
    const bool rows = E.shard_rows && E.shard_world > 1;
    if (rows) {  // one round per launch; its work items are logged for the exchange
        const size_t nn = (size_t)E.cap_n + 1;
        if (E.log_chg.n < nn) {
            E.log_chg.reserve(nn, 0, E.st);
            DLP_CUDA_TRY(cudaMemsetAsync(E.log_chg.p, 0, E.log_chg.n * sizeof(unsigned int), E.st));
        }
        E.log_u.reserve(nn, 0, E.st);
        E.log_em.reserve(nn, 0, E.st);
        P.log_u = E.log_u.p;
        P.log_em = E.log_em.p;
        P.log_chg = E.log_chg.p;
    }
    if (first) {
        // keep the host-written actions across the reset
        DLP_CUDA_TRY(cudaMemsetAsync(E.ctl, 0, offsetof(LPCtl, act), E.st));
        DLP_CUDA_TRY(cudaMemsetAsync(&E.ctl->has_fr, 0, sizeof(LPCtl) - offsetof(LPCtl, has_fr), E.st));
    } else {
        DLP_CUDA_TRY(cudaMemsetAsync(&E.ctl->bar, 0, sizeof(unsigned int), E.st));
    }
    if (rows) DLP_CUDA_TRY(cudaMemsetAsync(&E.ctl->log_n, 0, sizeof(long long), E.st));
    void* args[] = {&P};
    l2_window(E, E.st);
    DLP_CUDA_TRY(cudaLaunchCooperativeKernel((void*)k_lp_fused, dim3(E.lp_grid), dim3(kLpThreads), args, E.lp_smem,
                                             E.st));
    E.launches++;
}

// Row-partitioned mode: apply the rows other ranks evaluated in the last
// round -- their committed labels, and the claims their changed rows make on
// this rank's vertices (the eligible mask holds only owned vertices) -- into
// the next round's frontier lists, as if this rank's own rows had changed.
// One warp per remote row.
__global__ void k_rows_apply(long long m, int C, const int* ru, const unsigned int* rem, const unsigned int* rchg,
                             const double* rval, double* X, const long long* row_start, const int* row_len,
                             const int* nbr, ClaimTargets tg, int* has_fr) {
    __shared__ ClaimTargets s_tg;
    if (threadIdx.x == 0) s_tg = tg;
    __syncthreads();
    ClaimCtx K{&s_tg, 0u, 0u, 0u, 0ULL, 0.0};
    const int lane = threadIdx.x & 31;
    const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = wid; i < m; i += nw) {
        const int u = ru[i];
        const unsigned int em = rem[i], chg = rchg[i];
        for (int c = lane; c < C; c += 32)
            if ((em >> c) & 1u) X[(long long)u * C + c] = rval[i * C + c];
        if (!chg) continue;
        if (lane == 0) claim(K, u, chg);
        const long long st = row_start[u];
        const int len = row_len[u];
        for (int t = lane; t < len; t += 32) claim(K, nbr[st + t], chg);
    }
    for (int c = 0; c < C; c++)
        if ((K.claimed >> c) & 1u) has_fr[c] = 1;
}

void lp_rows_apply(Engine& E, long long m, long long r_par) {
    if (m <= 0) return;
    const int ri = (int)(r_par & 1);
    ClaimTargets K{E.fmask[ri].p, {E.ulist[ri].p, E.llist[ri].p, E.hlist[ri].p}, E.ctl->ncur_p, E.eligm.p};
    const long long blocks = std::min<long long>((m * 32 + kBlock - 1) / kBlock, (long long)E.sm_count * 16);
    k_rows_apply<<<(unsigned int)blocks, kBlock, 0, E.st>>>(m, E.ncol, E.rx_u.p, E.rx_em.p, E.rx_chg.p, E.rx_val.p,
                                                           E.f[0].p, E.row_start.p, E.row_len.p, E.nbr.p, K,
                                                           E.ctl->has_fr);
    DLP_CUDA_TRY(cudaGetLastError());
    E.launches++;
}

// Row partition over NCCL: pack the round's evaluated rows (record = vertex,
// evaluated mask, changed mask, C label words) into the send buffer; the
// changed-mask log is cleared for the next round as it is read.
__global__ void k_rows_pack(long long n, int C, const int* lu, const unsigned int* lem, unsigned int* lchg,
                            const double* Y, unsigned long long* send, unsigned long long* count) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const unsigned int em = lem[i];
        const unsigned int chg = lchg[i];
        lchg[i] = 0u;
        if (!em) continue;
        const unsigned long long j = atomicAdd(count, 1ULL);
        unsigned long long* r = send + j * (3 + C);
        r[0] = (unsigned long long)lu[i];
        r[1] = em;
        r[2] = chg;
        for (int c = 0; c < C; c++) r[3 + c] = (unsigned long long)__double_as_longlong(Y[i * C + c]);
    }
}

void rows_pack(Engine& E, long long n, unsigned long long* send, unsigned long long* count) {
    if (n <= 0) return;
    k_rows_pack<<<blocks_for(n), kBlock, 0, E.st>>>(n, E.ncol, E.log_u.p, E.log_em.p, E.log_chg.p, E.f[1].p, send,
                                                    count);
    DLP_CUDA_TRY(cudaGetLastError());
    E.launches++;
}

// the other ranks' records -> k_rows_apply inputs (rank r's record j goes to
// base[r] + j; meta = [cnt[0..W), base[0..W)])
__global__ void k_rows_unpack(int W, int me, long long mx, int C, const long long* meta,
                              const unsigned long long* recv, int* ru, unsigned int* rem, unsigned int* rchg,
                              double* rval) {
    const long long tot = (long long)W * mx;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(t / mx);
        const long long j = t - r * mx;
        if (r == me || j >= meta[r]) continue;
        const long long o = meta[W + r] + j;
        const unsigned long long* rec = recv + t * (3 + C);
        ru[o] = (int)rec[0];
        rem[o] = (unsigned int)rec[1];
        rchg[o] = (unsigned int)rec[2];
        for (int c = 0; c < C; c++) rval[o * C + c] = __longlong_as_double((long long)rec[3 + c]);
    }
}

void rows_unpack(Engine& E, int W, int me, long long mx, const std::vector<unsigned long long>& cnt,
                 const std::vector<long long>& base, const unsigned long long* recv) {
    std::vector<long long> meta(2 * W);
    for (int r = 0; r < W; r++) {
        meta[r] = (long long)cnt[r];
        meta[W + r] = base[r];
    }
    E.comm_buf.reserve(2 * (size_t)W + 2 + 2 * (size_t)W, 2 * (size_t)W + 2, E.st);
    long long* md = (long long*)(E.comm_buf.p + 2 * W + 2);
    DLP_CUDA_TRY(cudaMemcpyAsync(md, meta.data(), meta.size() * 8, cudaMemcpyHostToDevice, E.st));
    const long long tot = (long long)W * mx;
    k_rows_unpack<<<blocks_for(tot), kBlock, 0, E.st>>>(W, me, mx, E.ncol, md, recv, E.rx_u.p, E.rx_em.p,
                                                        E.rx_chg.p, E.rx_val.p);
    DLP_CUDA_TRY(cudaGetLastError());
    DLP_CUDA_TRY(cudaStreamSynchronize(E.st));  // meta is a host temporary
    E.launches++;
}

// Append the last launch's per-round trace to $DLP_LP_TRACE (diagnostics).
void lp_dump_trace(Engine& E, long long rounds) {
    if (!E.lp_trace_path || rounds <= 0) return;
    long long n = std::min<long long>(rounds, 1 << 16);
    std::vector<unsigned long long> h(8 * n);
    DLP_CUDA_TRY(cudaMemcpy(h.data(), E.lp_trace.p, h.size() * 8, cudaMemcpyDeviceToHost));
    FILE* fp = fopen(E.lp_trace_path, "a");
    if (!fp) return;
    unsigned long long pr[8] = {0};
    DLP_CUDA_TRY(cudaMemcpy(pr, E.lp_prof.p, sizeof(pr), cudaMemcpyDeviceToHost));
    fprintf(fp, "# launch rounds=%lld grid=%d dups=%llu prof_ms(warp-sum) hub=%.1f long=%.1f short=%.1f phase1=%.1f"
            " raw %llu %llu %llu %llu %llu %llu %llu %llu\n",
            rounds, E.lp_grid, E.h_ctl.p->dups, pr[0] / 1e6, pr[1] / 1e6, pr[2] / 1e6, pr[3] / 1e6, pr[0], pr[1],
            pr[2], pr[3], pr[4], pr[5], pr[6], pr[7]);
    for (long long r = 0; r < n; r++)
        fprintf(fp, "%lld %llu %llu %llx %llu %llu %llu %llu %llu\n", r, h[8 * r], h[8 * r + 1], h[8 * r + 2],
                h[8 * r + 3], h[8 * r + 4], h[8 * r + 5], h[8 * r + 6], h[8 * r + 7]);
    fclose(fp);
}

// ---------------------------------------------------------------------------
// ItLP active set (baselines.py:208-218): alive & unlabeled & degree > 0;
// isolated unlabeled vertices are pinned to 0.5 and counted.
// ---------------------------------------------------------------------------
__global__ void k_itlp_active(long long n, const unsigned char* alive, const signed char* gt, const int* row_len,
                              int ncol, double* f0, double* f1, unsigned int* eligm, int* alist, DevState* ds,
                              const unsigned char* mark, int* row_mod, int seq) {
    unsigned int allc = ncol >= 32 ? 0xffffffffu : ((1u << ncol) - 1u);
    long long iso = 0;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x) {
        bool unl = alive[v] && gt[v] == -1;
        if (mark[v]) row_mod[v] = seq;
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
                                                                       E.ds, E.mark.p, E.row_mod.p, E.view_seq);
    E.launches++;
}

}  // namespace dlp
