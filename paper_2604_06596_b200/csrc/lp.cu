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
// * Two row classes.  Short rows (<= kLongRow entries, the bulk of a kNN
//   graph) are evaluated warp-independently: a warp grabs 32/C rows, lane
//   (row, column) walks its row in stored order -- the reference's sequential
//   fp64 summation -- with kUnroll entries in flight (independent id/weight
//   loads, then independent label gathers, then the ordered sums).  No CTA
//   barrier is involved, so warps overlap each other's memory latency.
//   Long rows (kNN hubs reach thousands of entries) are evaluated by a whole
//   CTA: window by window the CTA gathers the entries and precomputes the
//   independent product terms (f[v]-fu)*w in parallel into shared memory,
//   then one thread per column runs the ordered dependent sums.
// * Cache policy.  Adjacency (ids, weights) and the compact staging buffer
//   are streamed (evict-first); label reads and commits carry an L2
//   evict_last policy so the C-wide label vectors stay L2-resident while the
//   adjacency streams through.
// * Jacobi commit: phase 1 writes new values to a compact staging buffer
//   (indexed by work item), phase 2 copies them into X; two grid-wide
//   barriers per round.
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
#define DLP_WIN 32
#endif
#ifndef DLP_WIN_MAX
#define DLP_WIN_MAX 64  // window slots per warp tile (span-1 rounds; C-wide rounds fit kWin)
#endif
#ifndef DLP_HUB_WIN
#define DLP_HUB_WIN 128
#endif
#ifndef DLP_LP_MINB
#define DLP_LP_MINB 3
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
constexpr int kLongRow = 96;    // rows longer than this are warp tiles of their own
#ifndef DLP_HUB_ROW_DEFAULT
#define DLP_HUB_ROW_DEFAULT 512
#endif
constexpr int kHubRow = DLP_HUB_ROW_DEFAULT;  // rows longer than this are evaluated by a whole CTA
constexpr int kScanRatio = 64;  // rounds with >= n/64 rows expand by atomicOr + compaction

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
    const int* row_len;
    const int* nbr;
    const double* w;
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

struct ClaimCtx {
    unsigned int* fm_next;
    int* next[3];
    unsigned int* cnt;  // [3]
    const unsigned int* eligm;
    const int* row_len;
    unsigned int claimed;  // per-thread OR of claimed column bits
    // per-lane round counters of the lane's label column (flushed once per round)
    unsigned long long c_nev, c_edg;
    unsigned int c_warn;
    double c_rmax;
};

// append-mode claim: add v (for the columns in `bits` where it is eligible)
// to the next union frontier; the first claimer appends it to its class list
__device__ inline void claim(ClaimCtx& k, int v, unsigned int bits) {
    const unsigned int e = k.eligm[v];
    bits &= e;
    if (!bits) return;
    k.claimed |= bits;
    unsigned int* fm = k.fm_next + v;
    unsigned int cur = *(volatile unsigned int*)fm;
    if ((cur & bits) == bits) return;
    unsigned int old = atomicOr(fm, bits);
    if (old != 0) return;
    const int cls = elig_class(e);
    if (cls == CLS_SHORT)
        append_u32(k.next[0], &k.cnt[0], v);
    else if (cls == CLS_LONG)
        append_u32(k.next[1], &k.cnt[1], v);
    else
        append_u32(k.next[2], &k.cnt[2], v);
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
    int u[32], len[32], off[33];
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

// Round geometry, set with the round's actions (every CTA's controller):
// the active columns (frontier | certify) and the step-major tile shape.
// A warp tile holds rpt = 32 / na rows and lane (r, a) runs row r's ordered
// sums for active column acol[a]; a window stages S consecutive entries of
// EVERY row of the tile, so all lanes advance together (a certify round of
// one column packs 32 rows per warp instead of idling 31 lanes).  Label
// words are copied as one 8-byte word per entry when a single column is
// active (span 1), else as the whole C-wide row.
struct TileGeo {
    int na, rpt, S, cmin, span;
    int acol[kMaxCols];
};
constexpr int kMaxQ = DLP_WIN_MAX / 32;  // window slots per gathering lane
// warp-private staging (doubles): DLP_WIN_MAX weights + kWin C-wide label rows
__host__ __device__ inline int warp_smem_doubles(int C) { return DLP_WIN_MAX + (kWin * C > DLP_WIN_MAX ? kWin * C : DLP_WIN_MAX); }

#ifndef DLP_LONG_RPT
#define DLP_LONG_RPT 1  // rows per long-row tile (length imbalance wastes windows when > 1)
#endif
__device__ inline void set_geo(TileGeo& G, unsigned int act, int C, int xcap, int max_rows) {
    int na = 0;
    for (int c = 0; c < C; c++)
        if ((act >> c) & 1u) G.acol[na++] = c;
    if (na == 0) G.acol[na++] = 0;  // idle round (the loop is about to end)
    G.na = na;
    G.rpt = min(32 / na, max_rows);
    G.cmin = na == 1 ? G.acol[0] : 0;
    G.span = na == 1 ? 1 : C;
    int we = xcap / G.span;  // label words fit in xcap doubles, weights in DLP_WIN_MAX
    if (we > DLP_WIN_MAX) we = DLP_WIN_MAX;
    int S = we / G.rpt;
    G.S = S < 1 ? 1 : S;
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
    int u, len;
    unsigned int em;
    long long st;
};
__device__ inline TileMeta load_meta(const LPParams& P, const RoundCtx& R, int u) {
    TileMeta m{u, 0, 0u, 0};
    if (u >= 0) {
        m.em = P.itlp ? (R.CE & P.eligm[u]) : (((R.fm_cur[u] & R.FR) | R.CE) & P.eligm[u]);
        m.st = P.row_start[u];
        m.len = P.row_len[u];
    }
    return m;
}

// Per-lane constants of a round's geometry: the window slots this lane
// gathers (slot j = lane + 32q -> tile row j / S, step j % S) and the
// accumulate role (row ar, column ac).
struct LaneGeo {
    int qr[kMaxQ], qs[kMaxQ];
    int ar, ac, acs;  // row, column, column offset inside the copied span
    bool alane;       // lane has an accumulate role
};
__device__ inline LaneGeo lane_geo(const TileGeo& G, int lane) {
    LaneGeo L;
#pragma unroll
    for (int q = 0; q < kMaxQ; q++) {
        const int j = lane + 32 * q;
        L.qr[q] = j < G.rpt * G.S ? j / G.S : 32;
        L.qs[q] = j - (j / G.S) * G.S;
    }
    L.alane = lane < G.rpt * G.na;
    L.ar = lane / G.na;
    L.ac = G.acol[lane - L.ar * G.na];
    L.acs = L.ac - G.cmin;
    return L;
}

// Evaluate `nrows` consecutive work items W[k0 ..] as one step-major warp
// tile (metadata m: lane r holds row r); `un` is the next tile's row of this
// lane (-1 if none), whose metadata is loaded into *mn mid-tile.  Gathers are
// entry-parallel into warp-private shared memory (ids and weights one window
// ahead, label words by cp.async), then lane (row, column) runs the row's
// sums in stored order (kernels/_csr.pyx:38-52); finally the changed rows
// claim themselves and their neighbours (_csr.pyx:175-191).
__device__ void warp_tile(const LPParams& P, const RoundCtx& R, const TileGeo& G, ClaimCtx& K,
                          BlockCounters& B, WarpTile& T, double* sw, double* sx, long long k0, int nrows,
                          unsigned long long pol, const TileMeta& m, int un, TileMeta* mn) {
    const int C = P.C;
    const LaneGeo L = lane_geo(G, threadIdx.x & 31);
    const int lane = threadIdx.x & 31;
    const int S = G.S, span = G.span;
    // ---- tile rows
    int len = 0;
    unsigned int em = 0;
    if (lane < nrows) {
        em = m.em;
        P.emask_store[R.ybase + k0 + lane] = em;  // by work item: the commit reads it coalesced
        len = em ? m.len : 0;
        T.u[lane] = m.u;
        T.em[lane] = em;
        T.st[lane] = em ? m.st : 0;
        T.len[lane] = len;
        T.chg[lane] = 0u;
    }
    int maxlen = len, total = len;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
        total += __shfl_xor_sync(0xffffffffu, total, o);
    }
    if (R.tmax && len) atomicMax(R.tmax, (unsigned long long)len);
    {
        unsigned int nz = __ballot_sync(0xffffffffu, em != 0);
        if (lane == 0 && nz) {
            atomicAdd(&B.urows, (unsigned long long)__popc(nz));
            atomicAdd(&B.uent, (unsigned long long)total);
        }
    }
    __syncwarp();  // T.* written by lane r is read by other lanes below
    // accumulate role: lane (ar, ac); its own label fu is a plain load whose
    // latency overlaps the first window's gathers
    const bool aact = L.alane && L.ar < nrows && ((T.em[L.ar] >> L.ac) & 1u);
    const int u_a = aact ? T.u[L.ar] : 0;
    const int len_a = aact ? T.len[L.ar] : 0;
    const double fu = aact ? ld_keep(P.X + (long long)u_a * C + L.ac, pol) : 0.0;
    // gather role: slot q of this lane -> (row qr, step qs)
    long long qst[kMaxQ];
    int qlen[kMaxQ];
#pragma unroll
    for (int q = 0; q < kMaxQ; q++) {
        const bool ok = L.qr[q] < nrows;
        qst[q] = ok ? T.st[L.qr[q]] + L.qs[q] : 0;
        qlen[q] = ok ? T.len[L.qr[q]] - L.qs[q] : 0;  // window wb is valid while wb < qlen
    }
    *mn = load_meta(P, R, un);  // next tile's metadata, consumed next iteration
    RowAcc acc;
    acc.init();
    int vv[kMaxQ];
    double ww[kMaxQ];
    auto load_ids = [&](int wb) {
#pragma unroll
        for (int q = 0; q < kMaxQ; q++) {
            if (wb < qlen[q]) {
                vv[q] = __ldcs(P.nbr + qst[q] + wb);
                ww[q] = __ldcs(P.w + qst[q] + wb);
            }
        }
    };
    if (maxlen > 0) load_ids(0);
    const double* xcol = P.X + G.cmin;
    for (int wb = 0; wb < maxlen; wb += S) {
#pragma unroll
        for (int q = 0; q < kMaxQ; q++) {
            if (wb >= qlen[q]) continue;
            const int j = lane + 32 * q;
            sw[j] = ww[q];
            if (span == 1)
                cp_async8(sx + j, xcol + (long long)vv[q] * C, pol);
            else
                copy_label_row(sx + j * span, P.X + (long long)vv[q] * C, C, pol);
        }
        if (wb + S < maxlen) load_ids(wb + S);
        cp_async_wait_all();
        __syncwarp();
        if (aact) {
            const int hi = min(S, len_a - wb);
            const double* w0p = sw + L.ar * S;
            const double* x0p = sx + (L.ar * S) * span + L.acs;
            int t = 0;
            for (; t + kAccUnroll <= hi; t += kAccUnroll) acc.add_boxed_block<kAccUnroll>(w0p + t, x0p + t * span, span, fu);
            for (; t < hi; t++) acc.add_boxed(w0p[t], x0p[t * span], fu);
        }
        __syncwarp();
    }
    // ---- finish: stage, count, flag
    unsigned int ch = 0;
    if (aact) {
        const int c = L.ac;
        double val;
        double d = acc.finish(fu, &val);
        __stcs(P.Y + (R.ybase + k0 + L.ar) * C + c, val);
        K.c_nev++;
        K.c_edg += (unsigned long long)len_a;
        if (d < 0.0) {  // isolated sentinel (_csr.pyx:49-51, 170-173)
            K.c_warn++;
            atomicAnd(&P.eligm[u_a], ~(1u << c));
            atomicAdd((unsigned long long*)&P.ctl->elig_count[c], ~0ULL);
        } else {
            K.c_rmax = fmax(K.c_rmax, d);
            if (!P.itlp && d > P.delta) ch = 1u << c;
        }
    }
    if (P.itlp) return;
    // ---- expand (jacobi_run commit loop, _csr.pyx:175-191)
    if (!__any_sync(0xffffffffu, ch != 0)) return;
    if (ch) atomicOr(&T.chg[L.ar], ch);
    __syncwarp();
    unsigned int mrow = lane < nrows ? T.chg[lane] : 0u;
    if (mrow) {
        K.claimed |= mrow;  // u changed, so u itself is eligible for those columns
        if (P.log_chg) P.log_chg[R.ybase + k0 + lane] = mrow;
        if (R.scan_mode)
            atomicOr(&K.fm_next[T.u[lane]], mrow);
        else
            claim(K, T.u[lane], mrow);
    }
    if (maxlen <= S) {
        // single-window tile: the gathering lanes still hold the entries' ids
#pragma unroll
        for (int q = 0; q < kMaxQ; q++) {
            if (qlen[q] <= 0) continue;
            const unsigned int mq = T.chg[L.qr[q]];
            if (!mq) continue;
            if (R.scan_mode)
                atomicOr(&K.fm_next[vv[q]], mq);  // no return value: a fire-and-forget RED
            else
                claim(K, vv[q], mq);
        }
        return;
    }
    // multi-window tile: walk the changed rows' entries, flattened
    const int clen = mrow ? len : 0;
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
        int r = tile_row_of(T.off, nrows, g);
        const unsigned int mq = T.chg[r];
        int v = __ldcs(P.nbr + T.st[r] + (g - T.off[r]));
        if (R.scan_mode)
            atomicOr(&K.fm_next[v], mq);
        else
            claim(K, v, mq);
    }
}

// Warp loop over the tiles of one row class: tile indices are grabbed two
// ahead and row metadata one ahead (software pipeline), so a tile's
// dependent chain of loads overlaps the previous tile's gathers.
__device__ void warp_tiles(const LPParams& P, const RoundCtx& R, const TileGeo& G, ClaimCtx& K,
                           BlockCounters& B, WarpTile& T, double* sw, double* sx, unsigned int* grab,
                           long long nitems, unsigned long long pol) {
    const int lane = threadIdx.x & 31;
    const int per = G.rpt;
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
        warp_tile(P, R, G, K, B, T, sw, sx, k, nr, pol, m, un, &mn);
        __syncwarp();
        if (kn >= nitems) break;
        k = kn;
        nr = nrn;
        m = mn;
    }
}

// Hub row (row_len > kHubRow) evaluated by the whole CTA: windows of
// kHubWin entries are gathered by warps 1..7 (product terms precomputed)
// into a double buffer while warp 0 (one lane per column) runs the ordered
// sums over the previous window.
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
        s_i[1] = em ? P.row_len[u] : 0;
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
    const int u = s_i[0], len = s_i[1];
    const long long st = s_ll[0];
    if (tid < C) s_fu[tid] = ((em >> tid) & 1u) ? P.X[(long long)u * C + tid] : 0.0;
    __syncthreads();
    const int nwin = (len + kHubWin - 1) / kHubWin;
    const int bsz = kHubWin * (C + 1);
    // warps 0-3 run the row's four ordered sums (RowAcc::add_boxed split by
    // accumulator: s, w_all, w0, w1; lane c = column c), so the sequential
    // chains advance in parallel on four schedulers; warps 4-7 gather.  A
    // gathering thread holds the ids and weights of its entries of the window
    // after next in registers, so a window's gather is one round trip.
    constexpr int kSumWarps = 4;
    constexpr int kGth = kLpThreads - 32 * kSumWarps;
    constexpr int kPer = (kHubWin + kGth - 1) / kGth;
    const int g = tid - 32 * kSumWarps;
    int pv[kPer];
    double pw[kPer];
    auto load_ids = [&](int w) {
        const int wb = w * kHubWin, wn = min(kHubWin, len - wb);
#pragma unroll
        for (int j = 0; j < kPer; j++) {
            const int i = g + kGth * j;
            if (i < wn) {
                pv[j] = __ldcs(P.nbr + st + wb + i);
                pw[j] = __ldcs(P.w + st + wb + i);
            }
        }
    };
    auto issue = [&](int w) {
        double* sw = buf + (w & 1) * bsz;
        double* sx = sw + kHubWin;
        const int wn = min(kHubWin, len - w * kHubWin);
#pragma unroll
        for (int j = 0; j < kPer; j++) {
            const int i = g + kGth * j;
            if (i < wn) {
                sw[i] = pw[j];
                copy_label_row(sx + i * C, P.X + (long long)pv[j] * C, C, pol);
            }
        }
    };
    if (warp >= kSumWarps) {
        load_ids(0);
        issue(0);
        if (nwin > 1) load_ids(1);
        cp_async_wait_all();
    }
    __syncthreads();
    const bool act = warp < kSumWarps && lane < C && ((em >> lane) & 1u);
    const double fu = act ? s_fu[lane] : 0.0;
    double acc = 0.0;
#ifdef DLP_HUBPROF
    // diagnostics: cycles per part of the hub loop (warp 4 and warps 0-3, lane 0)
    long long hp[3] = {0, 0, 0};
#define HUBT(v) long long v = clock64()
#else
#define HUBT(v)
#endif
    for (int w = 0; w < nwin; w++) {
        HUBT(ta);
        if (warp >= kSumWarps) {
            if (w + 1 < nwin) {
                issue(w + 1);
                if (w + 2 < nwin) load_ids(w + 2);
                HUBT(tb);
                cp_async_wait_all();
#ifdef DLP_HUBPROF
                hp[0] += tb - ta;
                hp[1] += clock64() - tb;
#endif
            }
        } else if (act) {
            // shared loads run a block of 8 entries ahead of the chain
            const double* sw = buf + (w & 1) * bsz;
            const double* sx = sw + kHubWin + lane;
            const int wn = min(kHubWin, len - w * kHubWin);
            if (warp == 1) {  // w_all
                int t = 0;
                for (; t + 8 <= wn; t += 8) {
                    double wv[8];
#pragma unroll
                    for (int j = 0; j < 8; j++) wv[j] = sw[t + j];
#pragma unroll
                    for (int j = 0; j < 8; j++) acc = __dadd_rn(acc, wv[j]);
                }
                for (; t < wn; t++) acc = __dadd_rn(acc, sw[t]);
            } else if (warp == 0) {  // s: the label-difference sum
                // terms of a block first (independent), then the chain
                int t = 0;
                for (; t + 8 <= wn; t += 8) {
                    double tv[8], xv[8], wv[8];
#pragma unroll
                    for (int j = 0; j < 8; j++) {
                        xv[j] = lds64(sx + (t + j) * C);
                        wv[j] = lds64(sw + t + j);
                    }
#pragma unroll
                    for (int j = 0; j < 8; j++) {
                        const double p = __dmul_rn(__dsub_rn(xv[j], fu), wv[j]);
                        tv[j] = is_boxed(xv[j]) ? 0.0 : p;
                    }
#pragma unroll
                    for (int j = 0; j < 8; j++) acc = __dadd_rn(acc, tv[j]);
                }
                for (; t < wn; t++) {
                    const double x = sx[t * C];
                    acc = __dadd_rn(acc, is_boxed(x) ? 0.0 : __dmul_rn(__dsub_rn(x, fu), sw[t]));
                }
            } else {  // warp 2: w0, warp 3: w1 (weights of ground-truth neighbours per class)
                const int cls_want = warp - 2;
                int t = 0;
                for (; t + 8 <= wn; t += 8) {
                    double tv[8], xv[8], wv[8];
#pragma unroll
                    for (int j = 0; j < 8; j++) {
                        xv[j] = lds64(sx + (t + j) * C);
                        wv[j] = lds64(sw + t + j);
                    }
#pragma unroll
                    for (int j = 0; j < 8; j++)
                        tv[j] = (is_boxed(xv[j]) && boxed_class(xv[j]) == cls_want) ? wv[j] : 0.0;
#pragma unroll
                    for (int j = 0; j < 8; j++) acc = __dadd_rn(acc, tv[j]);
                }
                for (; t < wn; t++) {
                    const double x = sx[t * C];
                    acc = __dadd_rn(acc, (is_boxed(x) && boxed_class(x) == cls_want) ? sw[t] : 0.0);
                }
            }
#ifdef DLP_HUBPROF
            hp[0] += (long long)(__double_as_longlong(acc) & 0) + clock64() - ta;  // keep the chain before the stamp
#endif
        }
        HUBT(tc);
        __syncthreads();
#ifdef DLP_HUBPROF
        hp[2] += clock64() - tc;
#endif
    }
#ifdef DLP_HUBPROF
    if (lane == 0 && P.ctl->prof) {
        if (warp == kSumWarps) {
            atomicAdd(&P.ctl->prof[0], (unsigned long long)hp[0]);
            atomicAdd(&P.ctl->prof[1], (unsigned long long)hp[1]);
            atomicAdd(&P.ctl->prof[2], (unsigned long long)hp[2]);
        } else if (warp < kSumWarps) {
            atomicAdd(&P.ctl->prof[3 + warp], (unsigned long long)hp[0]);
            if (warp == 0) atomicAdd(&P.ctl->prof[7], (unsigned long long)hp[2]);
        }
    }
#endif
    double* chains = buf;  // [4][kMaxCols]: the windows are free now
    if (act) chains[warp * kMaxCols + lane] = acc;
    __syncthreads();
    if (tid < C && ((em >> tid) & 1u)) {
        RowAcc ra;
        ra.s = chains[tid];
        ra.w_all = chains[kMaxCols + tid];
        ra.w0 = chains[2 * kMaxCols + tid];
        ra.w1 = chains[3 * kMaxCols + tid];
        double val;
        double d = ra.finish(s_fu[tid], &val);
        __stcs(P.Y + (R.ybase + k) * C + tid, val);
        atomicAdd(&B.neval[tid], 1ULL);
        atomicAdd(&B.edges[tid], (unsigned long long)len);
        if (d < 0.0) {
            atomicAdd(&B.warn[tid], 1ULL);
            atomicAnd(&P.eligm[u], ~(1u << tid));
            atomicAdd((unsigned long long*)&P.ctl->elig_count[tid], ~0ULL);
        } else {
            if (d > 0.0) atomicMax(&B.rmax[tid], dbits(d));
            if (!P.itlp && d > P.delta) atomicOr(&s_u32[1], 1u << tid);
        }
    }
    __syncthreads();
    const unsigned int m = s_u32[1];
    if (m) {
        if (tid == 0) {
            K.claimed |= m;
            if (P.log_chg) P.log_chg[R.ybase + k] = m;
            if (R.scan_mode)
                atomicOr(&K.fm_next[u], m);
            else
                claim(K, u, m);
        }
        for (int t = tid; t < len; t += kLpThreads) {
            int v = __ldcs(P.nbr + st + t);
            if (R.scan_mode)
                atomicOr(&K.fm_next[v], m);
            else
                claim(K, v, m);
        }
    }
    (void)lane;
    __syncthreads();
}

// Grid barrier of the persistent kernel: one arrival counter (a two-level
// variant with 16 group counters measured 1% slower at 444 CTAs).
__device__ inline void gsync(LPCtl* ctl, unsigned int& target) { grid_sync(&ctl->bar, target); }

__global__ void __launch_bounds__(kLpThreads, DLP_LP_MINB) k_lp_fused(LPParams P) {
    extern __shared__ double smem_dyn[];
    __shared__ ColState S;
    __shared__ TileGeo s_geo, s_geo_l;  // short-row / long-row tile shapes
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
    double* sx = sw + DLP_WIN_MAX;
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
            switch (row_class(P.row_len[u])) {
                case CLS_SHORT: append_u32(P.flist[0][0], &ctl->n_f0[0], u); break;
                case CLS_LONG: append_u32(P.flist[1][0], &ctl->n_f0[1], u); break;
                default: append_u32(P.flist[2][0], &ctl->n_f0[2], u); break;
            }
        }
        for (long long i = gtid; i < n_el; i += gth) {
            int u = P.elist[i];
            const int cls = row_class(P.row_len[u]);
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
        set_geo(s_geo, S.fr_mask | S.cert_mask, C, wsm - DLP_WIN_MAX, 32);
        set_geo(s_geo_l, S.fr_mask | S.cert_mask, C, wsm - DLP_WIN_MAX, DLP_LONG_RPT);
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
        ClaimCtx K{fm_next, {P.flist[0][rn], P.flist[1][rn], P.flist[2][rn]}, slot->cnt, P.eligm, P.row_len, 0u,
                   0ULL, 0ULL, 0u, 0.0};
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
            if (n2c > 0) {
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
            warp_tiles(P, RL, s_geo_l, K, B, T, sw, sx, &slot->grab[1], n1c, pol);  // long rows
            if (prof) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tw2));
            warp_tiles(P, RS, s_geo, K, B, T, sw, sx, &slot->grab[0], n0c, pol);  // short rows
            if (prof) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tw3));
            if (prof) {  // warp-time per part of phase 1 (diagnostics)
                atomicAdd(&ctl->prof[0], tw1 - tw0);
                atomicAdd(&ctl->prof[1], tw2 - tw1);
                atomicAdd(&ctl->prof[2], tw3 - tw2);
            }
        }
        if (K.claimed) atomicOr(&B.claimed, K.claimed);
        if (K.c_nev) {  // lane (row, a) of every tile of the round works on column acol[a]
            const int col = s_geo.acol[lane % s_geo.na];
            atomicAdd(&B.neval[col], K.c_nev);
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
                set_geo(s_geo, S.fr_mask | S.cert_mask, C, wsm - DLP_WIN_MAX, 32);
                set_geo(s_geo_l, S.fr_mask | S.cert_mask, C, wsm - DLP_WIN_MAX, DLP_LONG_RPT);
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
                         (size_t)2 * kHubWin * (E.ncol + 1)) * sizeof(double);
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
    LPParams P;
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
                             const int* nbr, ClaimCtx K, int* has_fr) {
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
    ClaimCtx K{E.fmask[ri].p, {E.ulist[ri].p, E.llist[ri].p, E.hlist[ri].p}, E.ctl->ncur_p, E.eligm.p, E.row_len.p,
               0u, 0ULL, 0ULL, 0u, 0.0};
    const long long blocks = std::min<long long>((m * 32 + kBlock - 1) / kBlock, (long long)E.sm_count * 16);
    k_rows_apply<<<(unsigned int)blocks, kBlock, 0, E.st>>>(m, E.ncol, E.rx_u.p, E.rx_em.p, E.rx_chg.p, E.rx_val.p,
                                                           E.f[0].p, E.row_start.p, E.row_len.p, E.nbr.p, K,
                                                           E.ctl->has_fr);
    DLP_CUDA_TRY(cudaGetLastError());
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
