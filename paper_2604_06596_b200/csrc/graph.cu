// graph.cu -- GPU-resident dynamic graph: deletes, inserts, edge log, tau,
// intra-batch components, component initialisation, reachability.
//
// Reference semantics (paths under /root/reference/pkg/src/dynlp/):
//   apply_deletes        graph.py:311-326
//   apply_inserts        graph.py:328-361 (merge parallel edges by sum in
//                        occurrence order, first-occurrence position, drop <= 0)
//   CSR row order        graph.py:218-231 (stable argsort by source)
//   resolve_tau          engine.py:182-188 (numpy pairwise mean)
//   find_components      components.py:84-124
//   initialize_...       engine.py:191-225
//   reachable_mask + pin engine.py:166-179, 350-361
#include <cooperative_groups.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstring>

#include "engine.cuh"

namespace cg = cooperative_groups;

namespace dlp {

static inline int grid_for(long long n, int block = kBlock) { return blocks_for(n, block, 148 * 64); }
static inline int bits_for(unsigned long long v) {
    int b = 1;
    while (b < 64 && (1ULL << b) <= v) b++;
    return b;
}

template <typename T>
static void grow_zero(DevArray<T>& a, size_t want, size_t keep, cudaStream_t st) {
    if (want <= a.n) return;
    size_t old = a.n;
    a.reserve(want, keep, st);
    if (a.n > keep) DLP_CUDA_TRY(cudaMemsetAsync(a.p + keep, 0, (a.n - keep) * sizeof(T), st));
    (void)old;
}

void ensure_vertex_capacity(Engine& E, long long want) {
    if (want <= E.cap_n) return;
    long long nc = E.cap_n ? E.cap_n : 4096;
    while (nc < want) nc += nc / 2;
    long long keep = E.n_slots;
    cudaStream_t st = E.st;
    grow_zero(E.alive, nc, keep, st);
    grow_zero(E.mark, nc, keep, st);
    grow_zero(E.root_gt, nc, keep, st);
    grow_zero(E.owner_rank, nc, keep, st);
    grow_zero(E.migr_from, nc, keep, st);
    E.migr_flag.reserve(nc + 1, 0, st);
    E.migr_pos.reserve(nc + 1, 0, st);
    E.migr_list.reserve(nc + 1, 0, st);
    grow_zero(E.gt, nc, keep, st);
    grow_zero(E.row_start, nc, keep, st);
    grow_zero(E.row_len, nc, keep, st);
    grow_zero(E.row_up, nc, keep, st);
    grow_zero(E.row_cap, nc, keep, st);
    grow_zero(E.parent, nc, keep, st);
    grow_zero(E.cnt_up, nc, keep, st);
    grow_zero(E.cnt_dn, nc, keep, st);
    grow_zero(E.grp_start, nc, 0, st);
    grow_zero(E.purge_flag, nc, keep, st);
    for (int i = 0; i < 2; i++) {
        grow_zero(E.fmask[i], nc, keep, st);
        E.ulist[i].reserve(nc + 1, 0, st);
        E.llist[i].reserve(nc + 1, 0, st);
        E.hlist[i].reserve(nc + 1, 0, st);
    }
    E.elist_s.reserve(nc + 1, 0, st);
    E.elist_l.reserve(nc + 1, 0, st);
    E.elist_h.reserve(nc + 1, 0, st);
    grow_zero(E.eligm, nc, keep, st);
    grow_zero(E.row_mod, nc, keep, st);
    grow_zero(E.view_b, nc, keep, st);
    grow_zero(E.view_st, nc, keep, st);
    E.vlen.reserve(nc + 1, keep, st);
    E.wsum.reserve(nc + 1, keep, st);
    E.q01.reserve((size_t)(nc + 1) * E.ncol * 2, (size_t)keep * E.ncol * 2, st);
    grow_zero(E.emask_store, nc, keep, st);
    E.f0.reserve(nc + 1, 0, st);
    E.elist.reserve(nc + 1, 0, st);
    E.purge_list.reserve(nc + 1, 0, st);
    E.touched.reserve(nc + 1, 0, st);
    grow_zero(E.f[0], (size_t)nc * E.ncol, (size_t)keep * E.ncol, st);
    grow_zero(E.f[1], (size_t)nc * E.ncol, (size_t)keep * E.ncol, st);
    E.cap_n = nc;
}

void ensure_log(Engine& E, long long want) {
    if ((size_t)want <= E.log_w.n) return;
    long long keep = E.live_edges;
    E.log_lo.reserve(want, keep, E.st);
    E.log_hi.reserve(want, keep, E.st);
    E.log_w.reserve(want, keep, E.st);
    E.log_lo2.reserve(E.log_lo.n, 0, E.st);
    E.log_hi2.reserve(E.log_lo.n, 0, E.st);
    E.log_w2.reserve(E.log_lo.n, 0, E.st);
}

// ---------------------------------------------------------------------------
// deletes (graph.py:311-326)
// ---------------------------------------------------------------------------
__global__ void k_kill(const long long* dels, long long nd, unsigned char* alive) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nd; i += (long long)gridDim.x * blockDim.x)
        alive[dels[i]] = 0;
}

// warp per deleted vertex: mark alive neighbours (affected_del) and queue
// their rows for purging; then release the deleted row.
__global__ void k_del_scan(const long long* dels, long long nd, const long long* row_start, int* row_len, int* row_up,
                           const int* nbr, const unsigned char* alive, unsigned char* mark, int* purge_flag,
                           int* purge_list, DevState* ds) {
    int lane = threadIdx.x & 31;
    long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long i = warp; i < nd; i += nwarps) {
        int x = (int)dels[i];
        long long s = row_start[x];
        int len = row_len[x];
        for (int e = lane; e < len; e += 32) {
            int y = nbr[s + e];
            if (alive[y]) {
                mark[y] = 1;
                if (atomicExch(&purge_flag[y], 1) == 0) append_agg(purge_list, &ds->n_purge, y);
            }
        }
        __syncwarp();
        if (lane == 0) {
            row_len[x] = 0;
            row_up[x] = 0;
        }
    }
}

// warp per affected row: order-preserving removal of dead neighbours
__global__ void k_purge(const int* purge_list, const DevState* ds, const long long* row_start, int* row_len,
                        int* row_up, int* nbr, double* w, const unsigned char* alive, int* purge_flag) {
    int lane = threadIdx.x & 31;
    long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    long long np = ds->n_purge;
    for (long long i = warp; i < np; i += nwarps) {
        int y = purge_list[i];
        long long s = row_start[y];
        int len = row_len[y], up = row_up[y];
        int out = 0, new_up = 0;
        for (int base = 0; base < len; base += 32) {
            int e = base + lane;
            int v = 0;
            double wv = 0.0;
            bool keep = false;
            if (e < len) {
                v = nbr[s + e];
                wv = w[s + e];
                keep = alive[v] != 0;
            }
            unsigned m = __ballot_sync(0xffffffffu, keep);
            unsigned mu = __ballot_sync(0xffffffffu, keep && e < up);
            __syncwarp();
            if (keep) {
                int pos = out + __popc(m & ((1u << lane) - 1));
                nbr[s + pos] = v;
                w[s + pos] = wv;
            }
            out += __popc(m);
            new_up += __popc(mu);
            __syncwarp();
        }
        if (lane == 0) {
            row_len[y] = out;
            row_up[y] = new_up;
            purge_flag[y] = 0;
        }
    }
}

__global__ void k_log_flags(const int* lo, const int* hi, long long n, const unsigned char* alive, int* flag) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        flag[i] = (alive[lo[i]] && alive[hi[i]]) ? 1 : 0;
}

__global__ void k_log_scatter(const int* lo, const int* hi, const double* w, long long n, const int* flag,
                              const int* pos, int* lo2, int* hi2, double* w2, DevState* ds) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        if (flag[i]) {
            int p = pos[i];
            lo2[p] = lo[i];
            hi2[p] = hi[i];
            w2[p] = w[i];
        }
        if (i == n - 1) ds->log_n = pos[i] + flag[i];
    }
}

static void cub_scan(Engine& E, const int* in, int* out, long long n) {
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, (int)n, E.st);
    E.cub_tmp.reserve(bytes + 256, 0, E.st);
    cub::DeviceScan::ExclusiveSum(E.cub_tmp.p, bytes, in, out, (int)n, E.st);
    E.launches += 2;  // init + single-pass scan
}

static void cub_sort_pairs(Engine& E, const unsigned long long* kin, unsigned long long* kout, const int* vin,
                           int* vout, long long n, int end_bit) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, (int)n, 0, end_bit, E.st);
    E.cub_tmp.reserve(bytes + 256, 0, E.st);
    cub::DeviceRadixSort::SortPairs(E.cub_tmp.p, bytes, kin, kout, vin, vout, (int)n, 0, end_bit, E.st);
    E.launches += 2 + (end_bit + 7) / 8;  // histogram + scan + one onesweep pass per digit
}

void apply_deletes_dev(Engine& E, const BatchDev& b) {
    if (b.nd == 0) return;
    cudaStream_t st = E.st;
    DLP_CUDA_TRY(cudaMemsetAsync(&E.ds->n_purge, 0, sizeof(long long), st));
    k_kill<<<grid_for(b.nd), kBlock, 0, st>>>(b.dels, b.nd, E.alive.p);
    E.launches++;
    k_del_scan<<<grid_for(b.nd * 32), kBlock, 0, st>>>(b.dels, b.nd, E.row_start.p, E.row_len.p, E.row_up.p,
                                                       E.nbr.p, E.alive.p, E.mark.p, E.purge_flag.p,
                                                       E.purge_list.p, E.ds);
    E.launches++;
    k_purge<<<E.sm_count * 8, kBlock, 0, st>>>(E.purge_list.p, E.ds, E.row_start.p, E.row_len.p, E.row_up.p,
                                               E.nbr.p, E.wgt.p, E.alive.p, E.purge_flag.p);
    E.launches++;
    // edge log: order-preserving compaction to the live edges
    long long n = E.live_edges;
    if (n > 0) {
        E.flag_i.reserve(n + 1, 0, st);
        E.pos_i.reserve(n + 1, 0, st);
        k_log_flags<<<grid_for(n), kBlock, 0, st>>>(E.log_lo.p, E.log_hi.p, n, E.alive.p, E.flag_i.p);
        E.launches++;
        cub_scan(E, E.flag_i.p, E.pos_i.p, n);
        k_log_scatter<<<grid_for(n), kBlock, 0, st>>>(E.log_lo.p, E.log_hi.p, E.log_w.p, n, E.flag_i.p, E.pos_i.p,
                                                      E.log_lo2.p, E.log_hi2.p, E.log_w2.p, E.ds);
        E.launches++;
        std::swap(E.log_lo.p, E.log_lo2.p);
        std::swap(E.log_hi.p, E.log_hi2.p);
        std::swap(E.log_w.p, E.log_w2.p);
        std::swap(E.log_lo.n, E.log_lo2.n);
        std::swap(E.log_hi.n, E.log_hi2.n);
        std::swap(E.log_w.n, E.log_w2.n);
    }
}

// ---------------------------------------------------------------------------
// inserts (graph.py:328-361, labels.py:28-49)
// ---------------------------------------------------------------------------
__global__ void k_grow(const long long* ids, const signed char* gtin, long long k, int ncol, long long cap,
                       unsigned char* alive, signed char* gt, double* f0, double* f1, unsigned char* mark,
                       long long* row_start, int* row_len, int* row_up, int* row_cap, int* parent) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < k; i += (long long)gridDim.x * blockDim.x) {
        long long v = ids[i];
        int g = gtin[i];
        alive[v] = 1;
        gt[v] = (signed char)g;
        for (int c = 0; c < ncol; c++) {
            double x;
            if (g < 0)
                x = 0.5;
            else if (ncol == 1)
                x = box_class(g);
            else
                x = box_class(g == c ? 1 : 0);
            f0[v * ncol + c] = x;
            f1[v * ncol + c] = x;
        }
        mark[v] = 1;
        row_start[v] = 0;
        row_len[v] = 0;
        row_up[v] = 0;
        row_cap[v] = 0;
        parent[v] = (int)v;
    }
}

__global__ void k_edge_keys(const long long* ids, const long long* owner, const long long* other, long long ne,
                            unsigned long long N, unsigned long long* key, int* val) {
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < ne; j += (long long)gridDim.x * blockDim.x) {
        long long a = ids[owner[j]], o = other[j];
        unsigned long long lo = (unsigned long long)(a < o ? a : o), hi = (unsigned long long)(a < o ? o : a);
        key[j] = lo * N + hi;
        val[j] = (int)j;
    }
}

// group heads merge duplicate (lo, hi) keys: 0.0 + w1 + w2 ... in batch
// order (np.zeros + np.add.at, graph.py:348-349); position = first occurrence
__global__ void k_merge(const unsigned long long* skey, const int* sval, const double* w, long long ne,
                        unsigned long long N, int* keep, int* mlo_at, int* mhi_at, double* mw_at) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < ne; p += (long long)gridDim.x * blockDim.x) {
        unsigned long long key = skey[p];
        int j = sval[p];
        if (p > 0 && skey[p - 1] == key) {
            keep[j] = 0;
            continue;
        }
        double s = 0.0;
        for (long long q = p; q < ne && skey[q] == key; q++) s = __dadd_rn(s, w[sval[q]]);
        keep[j] = s > 0.0 ? 1 : 0;
        mlo_at[j] = (int)(key / N);
        mhi_at[j] = (int)(key % N);
        mw_at[j] = s;
    }
}

__global__ void k_append(const int* keep, const int* pos, long long ne, const int* mlo_at, const int* mhi_at,
                         const double* mw_at, long long base, int* m_lo, int* m_hi, double* m_w, int* log_lo,
                         int* log_hi, double* log_w, unsigned char* mark, DevState* ds) {
    long long log_n = ds->log_n;
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < ne; j += (long long)gridDim.x * blockDim.x) {
        if (keep[j]) {
            int q = pos[j];
            int lo = mlo_at[j], hi = mhi_at[j];
            double w = mw_at[j];
            m_lo[q] = lo;
            m_hi[q] = hi;
            m_w[q] = w;
            log_lo[log_n + q] = lo;
            log_hi[log_n + q] = hi;
            log_w[log_n + q] = w;
            if (lo < base) mark[lo] = 1;  // prior endpoints (graph.py:358-359)
        }
        if (j == ne - 1) ds->m_kept = pos[j] + keep[j];
    }
}

__global__ void k_log_advance(DevState* ds) { ds->log_n += ds->m_kept; }

// two grouping keys per merged edge: (2*lo) = up entry of lo's row,
// (2*hi+1) = down entry of hi's row; sorted stably by position q.
__global__ void k_group_keys(const int* m_lo, const int* m_hi, long long ne, const DevState* ds,
                             unsigned long long* key, int* val, int* cnt_up, int* cnt_dn) {
    long long m = ds->m_kept;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < ne; q += (long long)gridDim.x * blockDim.x) {
        if (q < m) {
            int lo = m_lo[q], hi = m_hi[q];
            key[2 * q] = 2ULL * (unsigned long long)lo;
            key[2 * q + 1] = 2ULL * (unsigned long long)hi + 1ULL;
            atomicAdd(&cnt_up[lo], 1);
            atomicAdd(&cnt_dn[hi], 1);
        } else {
            key[2 * q] = ~0ULL;
            key[2 * q + 1] = ~0ULL;
        }
        val[2 * q] = (int)q;
        val[2 * q + 1] = (int)q;
    }
}

__global__ void k_group_heads(const unsigned long long* skey, long long n2, const DevState* ds, int* grp_start,
                              int* touched, DevState* dsw) {
    long long m2 = 2 * ds->m_kept;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n2 && p < m2;
         p += (long long)gridDim.x * blockDim.x) {
        unsigned long long x = skey[p] >> 1;
        if (p == 0 || (skey[p - 1] >> 1) != x) {
            grp_start[x] = (int)p;
            append_agg(touched, &dsw->n_touched, (int)x);
        }
    }
}

// relocation space needed by the touched rows (same rule as k_row_alloc)
__global__ void k_pool_need(const int* touched, DevState* ds, const int* row_len, const int* row_cap,
                            const int* cnt_up, const int* cnt_dn) {
    long long nt = ds->n_touched;
    unsigned long long sum = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nt; i += (long long)gridDim.x * blockDim.x) {
        int x = touched[i];
        int need = row_len[x] + cnt_up[x] + cnt_dn[x];
        if (need > row_cap[x]) sum += (unsigned long long)(need + need / 2 + 4);
    }
    sum = warp_sum(sum);
    if ((threadIdx.x & 31) == 0 && sum) atomicAdd(&ds->pool_need, sum);
}

// thread per touched row: make room for the new up entries (and, for a new
// vertex, its down entries); relocate the row when its capacity is exceeded.
__global__ void k_row_alloc(const int* touched, DevState* ds, long long* row_start, int* row_len, int* row_up,
                            int* row_cap, const int* cnt_up, const int* cnt_dn, int* nbr, double* w) {
    long long nt = ds->n_touched;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nt; i += (long long)gridDim.x * blockDim.x) {
        int x = touched[i];
        long long s = row_start[x];
        int len = row_len[x], up = row_up[x], nu = cnt_up[x], nd = cnt_dn[x];
        int dn = len - up;
        int need = len + nu + nd;
        if (need > row_cap[x]) {
            int cap = need + need / 2 + 4;
            long long ns = (long long)atomicAdd(&ds->pool_top, (unsigned long long)cap);
            for (int e = 0; e < up; e++) {
                nbr[ns + e] = nbr[s + e];
                w[ns + e] = w[s + e];
            }
            for (int e = 0; e < dn; e++) {
                nbr[ns + up + nu + e] = nbr[s + up + e];
                w[ns + up + nu + e] = w[s + up + e];
            }
            row_start[x] = ns;
            row_cap[x] = cap;
        } else if (nu > 0) {
            for (int e = dn - 1; e >= 0; e--) {
                nbr[s + up + nu + e] = nbr[s + up + e];
                w[s + up + nu + e] = w[s + up + e];
            }
        }
        row_up[x] = up + nu;
        row_len[x] = need;
    }
}

__global__ void k_row_fill(const unsigned long long* skey, const int* sval, long long n2, const DevState* ds,
                           const int* grp_start, const int* cnt_up, const int* cnt_dn, const long long* row_start,
                           const int* row_len, const int* row_up, const int* m_lo, const int* m_hi,
                           const double* m_w, int* nbr, double* w) {
    long long m2 = 2 * ds->m_kept;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n2 && p < m2;
         p += (long long)gridDim.x * blockDim.x) {
        unsigned long long key = skey[p];
        int x = (int)(key >> 1);
        int side = (int)(key & 1);
        int q = sval[p];
        int rank = (int)(p - grp_start[x]);
        long long s = row_start[x];
        long long at;
        int other;
        if (side == 0) {
            at = s + (row_up[x] - cnt_up[x]) + rank;
            other = m_hi[q];
        } else {
            at = s + row_up[x] + (row_len[x] - row_up[x] - cnt_dn[x]) + (rank - cnt_up[x]);
            other = m_lo[q];
        }
        nbr[at] = other;
        w[at] = m_w[q];
    }
}

__global__ void k_group_cleanup(const int* touched, const DevState* ds, int* cnt_up, int* cnt_dn) {
    long long nt = ds->n_touched;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nt; i += (long long)gridDim.x * blockDim.x) {
        int x = touched[i];
        cnt_up[x] = 0;
        cnt_dn[x] = 0;
    }
}

void apply_inserts_dev(Engine& E, const BatchDev& b, long long base) {
    cudaStream_t st = E.st;
    if (b.k == 0) return;
    k_grow<<<grid_for(b.k), kBlock, 0, st>>>(b.ids, b.gt, b.k, E.ncol, E.cap_n, E.alive.p, E.gt.p, E.f[0].p, E.f[1].p,
                                             E.mark.p, E.row_start.p, E.row_len.p, E.row_up.p, E.row_cap.p,
                                             E.parent.p);
    E.launches++;
    DLP_CUDA_TRY(cudaMemsetAsync(&E.ds->m_kept, 0, sizeof(long long), st));
    if (b.ne == 0) return;
    long long ne = b.ne;
    unsigned long long N = (unsigned long long)(base + b.k);
    E.key_a.reserve(2 * ne + 2, 0, st);
    E.key_b.reserve(2 * ne + 2, 0, st);
    E.val_a.reserve(2 * ne + 2, 0, st);
    E.val_b.reserve(2 * ne + 2, 0, st);
    E.flag_i.reserve(ne + 1, 0, st);
    E.pos_i.reserve(ne + 1, 0, st);
    E.mlo_at.reserve(ne + 1, 0, st);
    E.mhi_at.reserve(ne + 1, 0, st);
    E.mw_at.reserve(ne + 1, 0, st);
    E.m_lo.reserve(ne + 1, 0, st);
    E.m_hi.reserve(ne + 1, 0, st);
    E.m_w.reserve(ne + 1, 0, st);
    k_edge_keys<<<grid_for(ne), kBlock, 0, st>>>(b.ids, b.owner, b.other, ne, N, E.key_a.p, E.val_a.p);
    E.launches++;
    cub_sort_pairs(E, E.key_a.p, E.key_b.p, E.val_a.p, E.val_b.p, ne, bits_for(N * N));
    k_merge<<<grid_for(ne), kBlock, 0, st>>>(E.key_b.p, E.val_b.p, b.w, ne, N, E.flag_i.p, E.mlo_at.p, E.mhi_at.p,
                                             E.mw_at.p);
    E.launches++;
    cub_scan(E, E.flag_i.p, E.pos_i.p, ne);
    k_append<<<grid_for(ne), kBlock, 0, st>>>(E.flag_i.p, E.pos_i.p, ne, E.mlo_at.p, E.mhi_at.p, E.mw_at.p, base,
                                              E.m_lo.p, E.m_hi.p, E.m_w.p, E.log_lo.p, E.log_hi.p, E.log_w.p,
                                              E.mark.p, E.ds);
    E.launches++;
    k_log_advance<<<1, 1, 0, st>>>(E.ds);
    E.launches++;
    // adjacency rows
    DLP_CUDA_TRY(cudaMemsetAsync(&E.ds->n_touched, 0, sizeof(long long), st));
    k_group_keys<<<grid_for(ne), kBlock, 0, st>>>(E.m_lo.p, E.m_hi.p, ne, E.ds, E.key_a.p, E.val_a.p, E.cnt_up.p,
                                                  E.cnt_dn.p);
    E.launches++;
    cub_sort_pairs(E, E.key_a.p, E.key_b.p, E.val_a.p, E.val_b.p, 2 * ne, std::min(64, bits_for(2 * N + 2)));
    k_group_heads<<<grid_for(2 * ne), kBlock, 0, st>>>(E.key_b.p, 2 * ne, E.ds, E.grp_start.p, E.touched.p, E.ds);
    E.launches++;
    // exact allocation check (one small read-back): compact / grow the pool
    // only when this batch's relocations would not fit
    DLP_CUDA_TRY(cudaMemsetAsync(&E.ds->pool_need, 0, sizeof(unsigned long long), st));
    k_pool_need<<<grid_for(b.k + ne), kBlock, 0, st>>>(E.touched.p, E.ds, E.row_len.p, E.row_cap.p, E.cnt_up.p,
                                                       E.cnt_dn.p);
    E.launches++;
    DLP_CUDA_TRY(cudaMemcpyAsync(E.h_ds.p, E.ds, sizeof(DevState), cudaMemcpyDeviceToHost, st));
    DLP_CUDA_TRY(cudaStreamSynchronize(st));
    {
        long long need = (long long)E.h_ds.p->pool_need, top = (long long)E.h_ds.p->pool_top;
        if (top + need > E.pool_cap) {
            host_mark(E, "pre-compact");
            compact_pool(E, std::max<long long>(16 * need, E.pool_cap / 8));
            host_mark(E, "compact");
        }
    }
    k_row_alloc<<<grid_for(b.k + ne), kBlock, 0, st>>>(E.touched.p, E.ds, E.row_start.p, E.row_len.p, E.row_up.p,
                                                       E.row_cap.p, E.cnt_up.p, E.cnt_dn.p, E.nbr.p, E.wgt.p);
    E.launches++;
    k_row_fill<<<grid_for(2 * ne), kBlock, 0, st>>>(E.key_b.p, E.val_b.p, 2 * ne, E.ds, E.grp_start.p, E.cnt_up.p,
                                                    E.cnt_dn.p, E.row_start.p, E.row_len.p, E.row_up.p, E.m_lo.p,
                                                    E.m_hi.p, E.m_w.p, E.nbr.p, E.wgt.p);
    E.launches++;
    k_group_cleanup<<<grid_for(b.k + ne), kBlock, 0, st>>>(E.touched.p, E.ds, E.cnt_up.p, E.cnt_dn.p);
    E.launches++;
}

// ---------------------------------------------------------------------------
// adjacency pool compaction (performance only; row order preserved)
// ---------------------------------------------------------------------------
__global__ void k_new_caps(const int* row_len, const unsigned char* alive, long long n, int* cap) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x) {
        int len = alive[v] ? row_len[v] : 0;
        cap[v] = len ? len + len / 4 + 4 : 0;
    }
}

__global__ void k_repack(const long long* row_start, const int* row_len, const unsigned char* alive, long long n,
                         const int* newcap, const int* newpos, const int* nbr, const double* w, int* nbr2, double* w2,
                         long long* row_start2, int* row_cap2) {
    int lane = threadIdx.x & 31;
    long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
    for (long long v = warp; v < n; v += nwarps) {
        long long s = row_start[v], d = newpos[v];
        int len = alive[v] ? row_len[v] : 0;
        for (int e = lane; e < len; e += 32) {
            nbr2[d + e] = nbr[s + e];
            w2[d + e] = w[s + e];
        }
        __syncwarp();  // every lane has read row_start[v] (updated in place)
        if (lane == 0) {
            row_start2[v] = d;
            row_cap2[v] = newcap[v];
        }
    }
}

// Order-preserving repack of every live row into the spare pool (rows packed
// in vertex order with 25% slack), then swap pools.  The spare has the same
// capacity as the pool, so a compaction allocates nothing unless the live
// adjacency itself outgrew the pool (then both grow geometrically).
void compact_pool(Engine& E, long long min_free) {
    cudaStream_t st = E.st;
    long long n = E.n_slots;
    long long live = 2 * E.live_edges;
    long long need = live + live / 4 + 4 * n + min_free + (1 << 20);
    long long cap = E.pool_cap;
    if (need > cap) cap = std::max<long long>(need, cap + cap / 2);
    E.nbr_sp.reserve(cap, 0, st);
    E.wgt_sp.reserve(cap, 0, st);
    long long top = 0;
    if (n > 0) {
        E.flag_i.reserve(n + 1, 0, st);
        E.pos_i.reserve(n + 1, 0, st);
        k_new_caps<<<grid_for(n), kBlock, 0, st>>>(E.row_len.p, E.alive.p, n, E.flag_i.p);
        E.launches++;
        cub_scan(E, E.flag_i.p, E.pos_i.p, n);
        k_repack<<<grid_for(n * 32), kBlock, 0, st>>>(E.row_start.p, E.row_len.p, E.alive.p, n, E.flag_i.p, E.pos_i.p,
                                                      E.nbr.p, E.wgt.p, E.nbr_sp.p, E.wgt_sp.p, E.row_start.p,
                                                      E.row_cap.p);
        E.launches++;
        int last_pos = 0, last_cap = 0;
        DLP_CUDA_TRY(cudaMemcpyAsync(&last_pos, E.pos_i.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
        DLP_CUDA_TRY(cudaMemcpyAsync(&last_cap, E.flag_i.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
        DLP_CUDA_TRY(cudaStreamSynchronize(st));
        top = (long long)last_pos + last_cap;
    }
    std::swap(E.nbr, E.nbr_sp);
    std::swap(E.wgt, E.wgt_sp);
    E.view_inval = E.view_seq - 1;  // the LP view lived in the pool the repack just wrote
    // the new spare must match the pool's capacity for the next compaction
    E.nbr_sp.reserve(E.nbr.n, 0, st);
    E.wgt_sp.reserve(E.wgt.n, 0, st);
    E.pool_cap = (long long)std::min(E.nbr.n, E.wgt.n);
    E.pool_top_host = top;
    unsigned long long t = (unsigned long long)top;
    DLP_CUDA_TRY(cudaMemcpyAsync(&E.ds->pool_top, &t, sizeof(t), cudaMemcpyHostToDevice, st));
    DLP_CUDA_TRY(cudaStreamSynchronize(st));
}

// The exact per-batch check runs inside apply_inserts_dev (k_pool_need); the
// host only makes sure the pool exists.
void ensure_pool(Engine& E, long long new_edges, long long new_vertices) {
    (void)new_edges;
    (void)new_vertices;
    if (E.pool_cap == 0) compact_pool(E, 1 << 16);
}

// ---------------------------------------------------------------------------
// tau: numpy pairwise summation of the live weights in log order
// (loops_utils.h.src pairwise_sum; np.mean = sum / count, engine.py:187)
// ---------------------------------------------------------------------------
constexpr int kPwBlock = 128;    // numpy PW_BLOCKSIZE
constexpr int kTauNode = 4096;   // elements per CTA-level node

__host__ __device__ inline long long pw_split(long long s) {
    long long n2 = s / 2;
    return n2 - n2 % 8;
}

// number of splits along the largest (all-right) path until size <= limit
__host__ __device__ inline int pw_depth(long long n, long long limit) {
    int d = 0;
    while (n > limit) {
        n = n - pw_split(n);
        d++;
    }
    return d;
}

// slot (d, i) of the implicit pairwise tree of a size-n root: returns false
// when the slot represents no node; a leaf above depth d is represented by
// its leftmost descendant slot.
__device__ inline bool pw_slot(long long n, int d, long long i, long long* off, long long* sz, bool* internal) {
    long long o = 0, s = n;
    for (int l = d - 1; l >= 0; --l) {
        if (s <= kPwBlock) {
            if (i & ((1LL << (l + 1)) - 1)) return false;
            *off = o;
            *sz = s;
            *internal = false;
            return true;
        }
        long long n2 = pw_split(s);
        if ((i >> l) & 1) {
            o += n2;
            s -= n2;
        } else {
            s = n2;
        }
    }
    *off = o;
    *sz = s;
    *internal = s > kPwBlock;
    return true;
}

__device__ inline double pw_leaf(const double* a, long long n) {
    if (n < 8) {
        double res = -0.0;
        for (long long i = 0; i < n; i++) res = __dadd_rn(res, a[i]);
        return res;
    }
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; j++) r[j] = a[j];
    long long i;
    for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[i + j]);
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; i++) res = __dadd_rn(res, a[i]);
    return res;
}

// Combine slot values of depth D up to the root of a size-n tree.  vin/vout
// are ping-pong buffers of 2^D entries; executed by one CTA.
__device__ double pw_combine(long long n, int D, double* va, double* vb) {
    double* cur = va;
    double* nxt = vb;
    for (int d = D - 1; d >= 0; --d) {
        long long slots = 1LL << d;
        for (long long i = threadIdx.x; i < slots; i += blockDim.x) {
            long long off, sz;
            bool internal;
            if (!pw_slot(n, d, i, &off, &sz, &internal)) continue;
            nxt[i] = internal ? __dadd_rn(cur[2 * i], cur[2 * i + 1]) : cur[2 * i];
        }
        __syncthreads();
        double* t = cur;
        cur = nxt;
        nxt = t;
    }
    return cur[0];
}

// one CTA per depth-D slot: stage the node in shared memory (coalesced),
// sum its leaves in parallel, combine its sub-tree in tree order.
__global__ void k_tau_nodes(const double* a, const DevState* ds, int D, double* vals) {
    __shared__ double sm[kTauNode + 64];
    __shared__ double va[64], vb[64];
    long long n = ds->log_n;
    if (n == 0) return;
    int Dn = pw_depth(n, kTauNode);
    if (blockIdx.x >= (1LL << Dn)) return;
    long long off, sz;
    bool internal;
    if (!pw_slot(n, Dn, blockIdx.x, &off, &sz, &internal)) return;
    if (!internal) {
        if (threadIdx.x == 0) vals[blockIdx.x] = pw_leaf(a + off, sz);
        return;
    }
    for (long long i = threadIdx.x; i < sz; i += blockDim.x) sm[i] = a[off + i];
    __syncthreads();
    int D2 = pw_depth(sz, kPwBlock);
    for (long long j = threadIdx.x; j < (1LL << D2); j += blockDim.x) {
        long long o2, s2;
        bool in2;
        if (pw_slot(sz, D2, j, &o2, &s2, &in2)) va[j] = pw_leaf(sm + o2, s2);
    }
    __syncthreads();
    double r = pw_combine(sz, D2, va, vb);
    if (threadIdx.x == 0) vals[blockIdx.x] = r;
    (void)D;
}

__global__ void k_tau_root(const DevState* dsr, double* vals, double* scratch, DevState* ds) {
    long long n = dsr->log_n;
    double tau = 0.0;
    if (n > 0) {
        int Dn = pw_depth(n, kTauNode);
        double s = pw_combine(n, Dn, vals, scratch);
        tau = __ddiv_rn(s, (double)n);
    }
    if (threadIdx.x == 0) ds->tau = tau;
}

__global__ void k_set_tau(DevState* ds, double t) { ds->tau = t; }

void resolve_tau_dev(Engine& E, double cfg_tau) {
    cudaStream_t st = E.st;
    if (!(cfg_tau != cfg_tau)) {  // explicit tau
        k_set_tau<<<1, 1, 0, st>>>(E.ds, cfg_tau);
        E.launches++;
        return;
    }
    long long nmax = std::max<long long>(E.live_edges + 1, (long long)E.log_w.n);
    int D = pw_depth(nmax, kTauNode);
    long long slots = 1LL << D;
    E.tau_scratch.reserve(2 * slots + 64, 0, st);
    k_tau_nodes<<<(unsigned)slots, kBlock, 0, st>>>(E.log_w.p, E.ds, D, E.tau_scratch.p);
    E.launches++;
    k_tau_root<<<1, 1024, 0, st>>>(E.ds, E.tau_scratch.p, E.tau_scratch.p + slots + 32, E.ds);
    E.launches++;
}

// ---------------------------------------------------------------------------
// intra-batch components (components.py:53-60, 84-124)
// ---------------------------------------------------------------------------
__global__ void k_iota(int* p, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        p[i] = (int)i;
}

__global__ void k_intra_union(const long long* ids, const long long* owner, const long long* other, const double* w,
                              long long ne, long long base, long long k, const DevState* ds, int* lpar) {
    double tau = ds->tau;
    for (long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x; j < ne; j += (long long)gridDim.x * blockDim.x) {
        long long o = other[j] - base;
        if (o < 0 || o >= k) continue;
        if (!(w[j] > tau)) continue;  // sparsify: strictly above tau
        uf_unite(lpar, (int)(ids[owner[j]] - base), (int)o);
    }
}

__global__ void k_roots(const int* par, long long n, int* root) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        root[i] = uf_root(par, (int)i);
}

__global__ void k_adopt_roots(int* par, const int* root, long long n, int* root_flag) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        int r = root[i];
        par[i] = r;
        if (root_flag) root_flag[i] = (r == i) ? 1 : 0;
    }
}

__global__ void k_intra_comp(const int* lpar, const int* root_rank, const int* root_flag, long long k, int* comp,
                             unsigned long long* key, int* val, DevState* ds) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < k; i += (long long)gridDim.x * blockDim.x) {
        int c = root_rank[lpar[i]];
        comp[i] = c;
        key[i] = (unsigned long long)c;
        val[i] = (int)i;
        if (i == k - 1) ds->intra_nc = root_rank[i] + root_flag[i];
    }
}

void intra_components_dev(Engine& E, const BatchDev& b, long long base) {
    cudaStream_t st = E.st;
    long long k = b.k;
    E.lpar.reserve(k + 1, 0, st);
    E.comp.reserve(k + 1, 0, st);
    E.root_flag.reserve(k + 1, 0, st);
    E.root_rank.reserve(k + 1, 0, st);
    E.comp_sorted_i.reserve(k + 1, 0, st);
    E.key_a.reserve(k + 2, 0, st);
    E.key_b.reserve(k + 2, 0, st);
    E.val_a.reserve(k + 2, 0, st);
    E.val_b.reserve(k + 2, 0, st);
    k_iota<<<grid_for(k), kBlock, 0, st>>>(E.lpar.p, k);
    E.launches++;
    if (b.ne) k_intra_union<<<grid_for(b.ne), kBlock, 0, st>>>(b.ids, b.owner, b.other, b.w, b.ne, base, k, E.ds, E.lpar.p);
    E.launches++;
    E.root_tmp.reserve(std::max<long long>(k, E.cap_n) + 1, 0, st);
    k_roots<<<grid_for(k), kBlock, 0, st>>>(E.lpar.p, k, E.root_tmp.p);
    E.launches++;
    k_adopt_roots<<<grid_for(k), kBlock, 0, st>>>(E.lpar.p, E.root_tmp.p, k, E.root_flag.p);
    E.launches++;
    cub_scan(E, E.root_flag.p, E.root_rank.p, k);
    k_intra_comp<<<grid_for(k), kBlock, 0, st>>>(E.lpar.p, E.root_rank.p, E.root_flag.p, k, E.comp.p, E.key_a.p,
                                                 E.val_a.p, E.ds);
    E.launches++;
    // members grouped by component, ascending vertex order within a group
    cub_sort_pairs(E, E.key_a.p, E.key_b.p, E.val_a.p, E.comp_sorted_i.p, k, bits_for((unsigned long long)k + 1));
    E.intra_k = k;
}

// per inserted vertex and column: weight to class-0 / class-1 ground truth in
// row order (np.bincount, engine.py:212-214)
__global__ void k_init_per_vertex(long long base, long long k, int ncol, long long cap, const long long* row_start,
                                  const int* row_len, const int* nbr, const double* w, const signed char* gt,
                                  double* per0, double* per1) {
    long long total = k * ncol;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
        long long i = t % k;
        int c = (int)(t / k);
        long long v = base + i;
        long long s = row_start[v];
        int len = row_len[v];
        double a = 0.0, bsum = 0.0;
        for (int e = 0; e < len; e++) {
            int g = gt[nbr[s + e]];
            if (g < 0) continue;
            int cls = (ncol == 1) ? g : (g == c ? 1 : 0);
            if (cls == 0)
                a = __dadd_rn(a, w[s + e]);
            else
                bsum = __dadd_rn(bsum, w[s + e]);
        }
        per0[c * k + i] = a;
        per1[c * k + i] = bsum;
    }
}

// component heads: W0/W1 in ascending vertex order (np.bincount over
// component_id, engine.py:215-216) and the init value (engine.py:217-219)
__global__ void k_comp_sum(const unsigned long long* skey, const int* sidx, long long k, int ncol, const double* per0,
                           const double* per1, double* cinit) {
    long long total = k * ncol;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
        long long p = t % k;
        int c = (int)(t / k);
        unsigned long long key = skey[p];
        if (p > 0 && skey[p - 1] == key) continue;
        double w0 = 0.0, w1 = 0.0;
        for (long long q = p; q < k && skey[q] == key; q++) {
            w0 = __dadd_rn(w0, per0[c * k + sidx[q]]);
            w1 = __dadd_rn(w1, per1[c * k + sidx[q]]);
        }
        double tot = __dadd_rn(w0, w1);
        double init;
        if (tot > 0) {
            double two = __dmul_rn(2.0, tot);
            init = __dadd_rn(__dsub_rn(0.5, __ddiv_rn(w0, two)), __ddiv_rn(w1, two));
        } else {
            init = 0.5;
        }
        cinit[c * k + key] = init;
    }
}

__global__ void k_comp_assign(long long base, long long k, int ncol, long long cap, const int* comp,
                              const signed char* gt, const double* cinit, double* f0, double* f1) {
    long long total = k * ncol;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
        long long i = t % k;
        int c = (int)(t / k);
        long long v = base + i;
        if (gt[v] != -1) continue;
        double x = cinit[c * k + comp[i]];
        f0[v * ncol + c] = x;
        f1[v * ncol + c] = x;
    }
}

void init_components_dev(Engine& E, const BatchDev& b, long long base) {
    cudaStream_t st = E.st;
    long long k = b.k;
    E.per0.reserve(k * E.ncol + 1, 0, st);
    E.per1.reserve(k * E.ncol + 1, 0, st);
    E.cinit.reserve(k * E.ncol + 1, 0, st);
    long long total = k * E.ncol;
    k_init_per_vertex<<<grid_for(total), kBlock, 0, st>>>(base, k, E.ncol, E.cap_n, E.row_start.p, E.row_len.p,
                                                          E.nbr.p, E.wgt.p, E.gt.p, E.per0.p, E.per1.p);
    E.launches++;
    k_comp_sum<<<grid_for(total), kBlock, 0, st>>>(E.key_b.p, E.comp_sorted_i.p, k, E.ncol, E.per0.p, E.per1.p,
                                                   E.cinit.p);
    E.launches++;
    k_comp_assign<<<grid_for(total), kBlock, 0, st>>>(base, k, E.ncol, E.cap_n, E.comp.p, E.gt.p, E.cinit.p, E.f[0].p,
                                                      E.f[1].p);
    E.launches++;
}

// ---------------------------------------------------------------------------
// reachability (engine.py:166-179) via the global union-find, pinning of
// unreachable vertices and the eligible set (engine.py:350-361), frontier
// seeds restricted to eligible (engine.py:246-251, 364-367)
// ---------------------------------------------------------------------------
__global__ void k_uf_union_log(const int* lo, const int* hi, const DevState* ds, int* par) {
    long long n = ds->log_n;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        uf_unite(par, lo[i], hi[i]);
}

__global__ void k_uf_union_merged(const int* lo, const int* hi, const DevState* ds, int* par) {
    long long n = ds->m_kept;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        uf_unite(par, lo[i], hi[i]);
}

__global__ void k_cc_hit_roots(const long long* dels, long long nd, const int* par, unsigned char* hit_root) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nd; i += (long long)gridDim.x * blockDim.x)
        hit_root[par[dels[i]]] = 1;
}

// members of a hit component become singletons (each thread owns parent[v];
// the root's own entry is already v)
__global__ void k_cc_reset_hit(long long n, int* par, const unsigned char* hit_root, unsigned char* hit) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x) {
        const unsigned char h = hit_root[par[v]];
        hit[v] = h;
        if (h) par[v] = (int)v;
    }
}

// surviving log edges of the hit components (both endpoints lie in the same
// old component, so testing lo suffices; edges to this batch's new vertices
// are also in the merged list)
__global__ void k_uf_union_log_hit(const int* lo, const int* hi, const DevState* ds, const unsigned char* hit,
                                   int* par) {
    long long n = ds->log_n;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const int a = lo[i];
        if (hit[a]) uf_unite(par, a, hi[i]);
    }
}

__global__ void k_uf_flatten_root_gt(int* par, long long n, const unsigned char* alive, const signed char* gt,
                                     unsigned char* root_gt) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x) {
        if (alive[v] && gt[v] >= 0) root_gt[par[v]] = 1;
    }
}


// component owner under sharding: a mixing hash of the
// component's canonical root (minimum member id), identical on every rank
__device__ inline int shard_owner(int root, int world) {
    unsigned int h = (unsigned int)root * 2654435761u;
    h ^= h >> 16;
    return (int)(h % (unsigned int)world);
}

__global__ void k_eligible(long long n, int ncol, long long cap, const unsigned char* alive, const signed char* gt,
                           const int* par, const unsigned char* root_gt, const int* row_len, unsigned char* mark,
                           unsigned int* eligm, double* f0, double* f1, int* elist, int* f0list, DevState* ds,
                           int rank, int world, int rows, unsigned char* owner_rank, unsigned char* migr_from,
                           int* migr_flag, const unsigned char* root_owner, int* row_mod, int seq) {
    unsigned int allc = ncol >= 32 ? 0xffffffffu : ((1u << ncol) - 1u);
    long long iso = 0, unr = 0;
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x) {
        bool unl = alive[v] && gt[v] == -1;
        bool reached = alive[v] && root_gt[par[v]];
        bool e = unl && reached;
        if (world > 1 && rows) {  // row partition: this rank evaluates the rows v % world == rank
            e = e && (v % world) == rank;
            migr_flag[v] = 0;
        } else if (world > 1) {  // sharded: only this rank's components are propagated here
            int mig = 0;
            if (e) {
                int o = root_owner ? (int)root_owner[par[v]] : shard_owner(par[v], world);
                int prev = owner_rank[v];
                if (o != prev) {  // component moved: its label lives on rank `prev`
                    mig = 1;
                    migr_from[v] = (unsigned char)prev;
                    owner_rank[v] = (unsigned char)o;
                }
                e = o == rank;
            }
            migr_flag[v] = mig;
        }
        eligm[v] = e ? allc : 0u;
        if (unl && !reached) {
            for (int c = 0; c < ncol; c++) {
                f0[v * ncol + c] = 0.5;
                f1[v * ncol + c] = 0.5;
            }
            if (row_len[v] == 0)
                iso++;
            else
                unr++;
        }
        if (e) {
            append_agg(elist, &ds->n_elist, (int)v);
            if (mark[v]) append_agg(f0list, &ds->n_f0, (int)v);
        }
        if (mark[v]) row_mod[v] = seq;  // the row changed this batch: its LP view is stale
        mark[v] = 0;
    }
    iso = warp_sum(iso);
    unr = warp_sum(unr);
    if ((threadIdx.x & 31) == 0 && (iso || unr)) {
        atomicAdd((unsigned long long*)&ds->isolated, (unsigned long long)iso);
        atomicAdd((unsigned long long*)&ds->unreach, (unsigned long long)unr);
    }
}

// ---------------------------------------------------------------------------
// Component placement for sharded batches: LPT
// bin-packing by edge count, sticky across batches.  Every rank holds the
// same structure, so every rank computes the same placement: components keep
// the rank they had (by their root's last placement) unless the load
// imbalance exceeds 25%, new components go to the least-loaded rank in
// decreasing size order (ties: lowest root, lowest rank).  Moves are handled
// by the existing label migration (owner_rank / migr_* per vertex).
// ---------------------------------------------------------------------------
__global__ void k_comp_weight(long long n, const unsigned char* alive, const int* par, const int* row_len,
                              unsigned long long* cw) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x)
        if (alive[v]) atomicAdd(&cw[par[v]], (unsigned long long)row_len[v] + 1ULL);
}

__global__ void k_comp_roots(long long n, const unsigned char* alive, const int* par, int* flag) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x)
        flag[v] = (alive[v] && par[v] == (int)v) ? 1 : 0;
}

__global__ void k_comp_gather(long long n, const int* flag, const int* pos, const unsigned long long* cw,
                              long long* roots, unsigned long long* w) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x)
        if (flag[v]) {
            roots[pos[v]] = v;
            w[pos[v]] = cw[v];
        }
}

__global__ void k_comp_place(long long m, const long long* roots, const unsigned char* own, unsigned char* root_owner) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
        root_owner[roots[i]] = own[i];
}

const unsigned char* assign_components(Engine& E, long long n) {
    cudaStream_t st = E.st;
    const int W = E.shard_world;
    E.comp_w.reserve(E.cap_n + 1, 0, st);
    E.root_owner.reserve(E.cap_n + 1, 0, st);
    DLP_CUDA_TRY(cudaMemsetAsync(E.comp_w.p, 0, n * sizeof(unsigned long long), st));
    E.flag_i.reserve(n + 1, 0, st);
    E.pos_i.reserve(n + 1, 0, st);
    k_comp_weight<<<grid_for(n), kBlock, 0, st>>>(n, E.alive.p, E.parent.p, E.row_len.p, E.comp_w.p);
    k_comp_roots<<<grid_for(n), kBlock, 0, st>>>(n, E.alive.p, E.parent.p, E.flag_i.p);
    cub_scan(E, E.flag_i.p, E.pos_i.p, n);
    int lp = 0, lf = 0;
    DLP_CUDA_TRY(cudaMemcpyAsync(&lp, E.pos_i.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    DLP_CUDA_TRY(cudaMemcpyAsync(&lf, E.flag_i.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    DLP_CUDA_TRY(cudaStreamSynchronize(st));
    const long long m = (long long)lp + lf;
    E.launches += 3;
    if (m == 0) return E.root_owner.p;
    E.comp_roots.reserve(m + 1, 0, st);
    E.comp_wl.reserve(m + 1, 0, st);
    E.comp_own.reserve(m + 1, 0, st);
    k_comp_gather<<<grid_for(n), kBlock, 0, st>>>(n, E.flag_i.p, E.pos_i.p, E.comp_w.p, E.comp_roots.p, E.comp_wl.p);
    std::vector<long long> roots(m);
    std::vector<unsigned long long> w(m);
    DLP_CUDA_TRY(cudaMemcpyAsync(roots.data(), E.comp_roots.p, m * 8, cudaMemcpyDeviceToHost, st));
    DLP_CUDA_TRY(cudaMemcpyAsync(w.data(), E.comp_wl.p, m * 8, cudaMemcpyDeviceToHost, st));
    DLP_CUDA_TRY(cudaStreamSynchronize(st));
    // placement (host, deterministic, identical on every rank)
    std::vector<unsigned char> own(m, 0);
    std::vector<unsigned long long> load(W, 0);
    unsigned long long total = 0;
    for (long long i = 0; i < m; i++) total += w[i];
    std::vector<long long> fresh;
    for (long long i = 0; i < m; i++) {
        auto it = E.place.find(roots[i]);
        if (it != E.place.end()) {
            own[i] = it->second;
            load[own[i]] += w[i];
        } else {
            fresh.push_back(i);
        }
    }
    const unsigned long long avg = (total + W - 1) / W;
    unsigned long long mx = 0;
    for (int r = 0; r < W; r++) mx = std::max(mx, load[r]);
    if (mx > avg + avg / 4) {  // imbalanced: full LPT
        fresh.clear();
        for (long long i = 0; i < m; i++) fresh.push_back(i);
        std::fill(load.begin(), load.end(), 0ULL);
    }
    std::sort(fresh.begin(), fresh.end(), [&](long long a, long long b) {
        return w[a] != w[b] ? w[a] > w[b] : roots[a] < roots[b];
    });
    for (long long i : fresh) {
        int best = 0;
        for (int r = 1; r < W; r++)
            if (load[r] < load[best]) best = r;
        own[i] = (unsigned char)best;
        load[best] += w[i];
    }
    E.place.clear();
    for (long long i = 0; i < m; i++) E.place.emplace(roots[i], own[i]);
    DLP_CUDA_TRY(cudaMemcpyAsync(E.comp_own.p, own.data(), m, cudaMemcpyHostToDevice, st));
    k_comp_place<<<grid_for(m), kBlock, 0, st>>>(m, E.comp_roots.p, E.comp_own.p, E.root_owner.p);
    DLP_CUDA_TRY(cudaStreamSynchronize(st));  // own is a host temporary
    E.launches += 2;
    return E.root_owner.p;
}

void reach_and_pin_dev(Engine& E, int cc, long long n, const long long* dels, long long nd) {
    cudaStream_t st = E.st;
    if (n == 0) return;
    if (cc == 2) {
        k_iota<<<grid_for(n), kBlock, 0, st>>>(E.parent.p, n);
        E.launches++;
        k_uf_union_log<<<grid_for(E.live_edges + 1), kBlock, 0, st>>>(E.log_lo.p, E.log_hi.p, E.ds, E.parent.p);
        E.launches++;
    } else if (cc == 1 && nd > 0) {
        // decremental: a component that lost no vertex lost no edge (an edge
        // dies with an endpoint), so only components holding a deleted vertex
        // can split.  Their members are reset to singletons and re-united over
        // their surviving log edges; then the batch's new edges are added as
        // in the incremental case.  (parent is flat: parent[v] = root.)
        E.cc_hit_root.reserve(E.cap_n + 1, 0, st);
        E.cc_hit.reserve(E.cap_n + 1, 0, st);
        DLP_CUDA_TRY(cudaMemsetAsync(E.cc_hit_root.p, 0, n, st));
        k_cc_hit_roots<<<grid_for(nd), kBlock, 0, st>>>(dels, nd, E.parent.p, E.cc_hit_root.p);
        k_cc_reset_hit<<<grid_for(n), kBlock, 0, st>>>(n, E.parent.p, E.cc_hit_root.p, E.cc_hit.p);
        k_uf_union_log_hit<<<grid_for(E.live_edges + 1), kBlock, 0, st>>>(E.log_lo.p, E.log_hi.p, E.ds, E.cc_hit.p,
                                                                          E.parent.p);
        k_uf_union_merged<<<E.sm_count * 8, kBlock, 0, st>>>(E.m_lo.p, E.m_hi.p, E.ds, E.parent.p);
        E.launches += 4;
    } else {
        k_uf_union_merged<<<E.sm_count * 8, kBlock, 0, st>>>(E.m_lo.p, E.m_hi.p, E.ds, E.parent.p);
        E.launches++;
    }
    DLP_CUDA_TRY(cudaMemsetAsync(E.root_gt.p, 0, n, st));
    E.root_tmp.reserve(E.cap_n + 1, 0, st);
    k_roots<<<grid_for(n), kBlock, 0, st>>>(E.parent.p, n, E.root_tmp.p);
    E.launches++;
    k_adopt_roots<<<grid_for(n), kBlock, 0, st>>>(E.parent.p, E.root_tmp.p, n, nullptr);
    E.launches++;
    k_uf_flatten_root_gt<<<grid_for(n), kBlock, 0, st>>>(E.parent.p, n, E.alive.p, E.gt.p, E.root_gt.p);
    E.launches++;
    const unsigned char* root_owner = nullptr;
    if (E.shard_world > 1 && !E.shard_rows && E.shard_lpt) root_owner = assign_components(E, n);
    k_eligible<<<grid_for(n), kBlock, 0, st>>>(n, E.ncol, E.cap_n, E.alive.p, E.gt.p, E.parent.p, E.root_gt.p,
                                               E.row_len.p, E.mark.p, E.eligm.p, E.f[0].p, E.f[1].p, E.elist.p, E.f0.p,
                                               E.ds, E.shard_rank, E.shard_world, E.shard_rows, E.owner_rank.p, E.migr_from.p,
                                               E.migr_flag.p, root_owner, E.row_mod.p, E.view_seq);
    E.launches++;
}

// ---------------------------------------------------------------------------
// sharded label migration: vertices whose component changed owner get their
// label from the previous owner (exchanged with the caller's max-reduction;
// non-owners contribute -inf, so the result is bit-exact)
// ---------------------------------------------------------------------------
__global__ void k_migr_list(const int* flag, const int* pos, long long n, int* list) {
    for (long long v = blockIdx.x * (long long)blockDim.x + threadIdx.x; v < n; v += (long long)gridDim.x * blockDim.x)
        if (flag[v]) list[pos[v]] = (int)v;
}
__global__ void k_migr_pack(const int* list, long long m, int ncol, int rank, const unsigned char* from,
                            const double* X, double* buf) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m * ncol;
         i += (long long)gridDim.x * blockDim.x) {
        int v = list[i / ncol], c = (int)(i % ncol);
        buf[i] = from[v] == rank ? X[(long long)v * ncol + c] : -INFINITY;
    }
}
__global__ void k_migr_unpack(const int* list, long long m, int ncol, const double* buf, double* X) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m * ncol;
         i += (long long)gridDim.x * blockDim.x) {
        int v = list[i / ncol], c = (int)(i % ncol);
        X[(long long)v * ncol + c] = buf[i];
    }
}

long long migr_collect(Engine& E, long long n) {
    cudaStream_t st = E.st;
    // migration flags exist only for component sharding over several ranks
    if (n == 0 || E.shard_world <= 1 || E.shard_rows) return 0;
    cub_scan(E, E.migr_flag.p, E.migr_pos.p, n);
    int lp = 0, lf = 0;
    DLP_CUDA_TRY(cudaMemcpyAsync(&lp, E.migr_pos.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    DLP_CUDA_TRY(cudaMemcpyAsync(&lf, E.migr_flag.p + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    DLP_CUDA_TRY(cudaStreamSynchronize(st));
    long long m = (long long)lp + lf;
    if (m) {
        k_migr_list<<<grid_for(n), kBlock, 0, st>>>(E.migr_flag.p, E.migr_pos.p, n, E.migr_list.p);
        E.launches++;
    }
    return m;
}

void migr_pack(Engine& E, long long m, double* dev_buf) {
    k_migr_pack<<<grid_for(m * E.ncol), kBlock, 0, E.st>>>(E.migr_list.p, m, E.ncol, E.shard_rank, E.migr_from.p,
                                                           E.f[0].p, dev_buf);
    E.launches++;
}

void migr_unpack(Engine& E, long long m, const double* dev_buf) {
    k_migr_unpack<<<grid_for(m * E.ncol), kBlock, 0, E.st>>>(E.migr_list.p, m, E.ncol, dev_buf, E.f[0].p);
    E.launches++;
}

// ---------------------------------------------------------------------------
// CSR snapshot for parity checks (host assembly; test path only)
// ---------------------------------------------------------------------------
void read_csr_dev(Engine& E, long long* indptr, long long* indices, double* weights, double* degrees) {
    long long n = E.n_slots;
    std::vector<long long> rs(n);
    std::vector<int> rl(n);
    std::vector<unsigned char> al(n);
    if (n) {
        DLP_CUDA_TRY(cudaMemcpyAsync(rs.data(), E.row_start.p, n * sizeof(long long), cudaMemcpyDeviceToHost, E.st));
        DLP_CUDA_TRY(cudaMemcpyAsync(rl.data(), E.row_len.p, n * sizeof(int), cudaMemcpyDeviceToHost, E.st));
        DLP_CUDA_TRY(cudaMemcpyAsync(al.data(), E.alive.p, n, cudaMemcpyDeviceToHost, E.st));
    }
    DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
    indptr[0] = 0;
    for (long long v = 0; v < n; v++) indptr[v + 1] = indptr[v] + (al[v] ? rl[v] : 0);
    std::vector<int> nb;
    std::vector<double> ww;
    for (long long v = 0; v < n; v++) {
        int len = al[v] ? rl[v] : 0;
        nb.resize(len);
        ww.resize(len);
        if (len) {
            DLP_CUDA_TRY(cudaMemcpy(nb.data(), E.nbr.p + rs[v], len * sizeof(int), cudaMemcpyDeviceToHost));
            DLP_CUDA_TRY(cudaMemcpy(ww.data(), E.wgt.p + rs[v], len * sizeof(double), cudaMemcpyDeviceToHost));
        }
        double d = 0.0;
        for (int e = 0; e < len; e++) {
            if (indices) indices[indptr[v] + e] = nb[e];
            if (weights) weights[indptr[v] + e] = ww[e];
            d += ww[e];
        }
        if (degrees) degrees[v] = d;
    }
}

}  // namespace dlp
