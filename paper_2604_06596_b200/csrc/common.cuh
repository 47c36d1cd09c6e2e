// common.cuh -- shared device helpers for the DynLP B200 engine (sm_100a).
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define DLP_CUDA_TRY(expr)                                                        \
    do {                                                                          \
        cudaError_t _e = (expr);                                                  \
        if (_e != cudaSuccess) throw dlp::CudaFailure(_e, #expr, __FILE__, __LINE__); \
    } while (0)

namespace dlp {

struct CudaFailure {
    cudaError_t err;
    const char* expr;
    const char* file;
    int line;
    CudaFailure(cudaError_t e, const char* x, const char* f, int l) : err(e), expr(x), file(f), line(l) {}
};

constexpr int kBlock = 256;

// ---------------------------------------------------------------------------
// Ground-truth boxing.  The LP working arrays hold, per label column, one
// 8-byte word per vertex: the fractional label for unlabeled vertices (always
// a number in [0, 1]) or a NaN whose payload carries the pinned class for
// ground-truth vertices.  One 8-byte gather per row entry therefore yields
// both gt[v] and f[v] (the reference reads two arrays, _csr.pyx:42-48).
// ---------------------------------------------------------------------------
constexpr unsigned long long kBoxBase = 0x7FF4000000000000ULL;

__host__ __device__ inline double box_class(int c) {
    union { unsigned long long u; double d; } x;
    x.u = kBoxBase | (unsigned long long)(c & 1);
    return x.d;
}
constexpr int kBoxHi = 0x7FF40000;  // high word of a boxed ground-truth label
// Exact box test on the high word (one integer compare, the cost of the NaN
// test it replaces): a NaN an unlabeled vertex reaches through non-finite
// weights (the reference keeps such a NaN, _csr.pyx:52-56) is not a box, so
// its neighbours treat it as an unlabeled NaN label exactly as the reference
// does.  Arithmetic never produces this signalling-NaN pattern.
__device__ inline bool is_boxed(double x) { return __double2hiint(x) == kBoxHi; }
__device__ inline int boxed_class(double x) { return (int)(__double_as_longlong(x) & 1); }
__device__ inline double unbox(double x) { return is_boxed(x) ? (double)boxed_class(x) : x; }

// Shared-memory load that ptxas keeps in program order with its peers: a
// block of these issues back to back instead of being sunk next to each use
// (under the kernel's register cap the scheduler otherwise serialises
// load -> term -> sum per entry).
__device__ inline double lds64(const double* p) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned int)__cvta_generic_to_shared(p)));
    return v;
}

// ---------------------------------------------------------------------------
// The per-vertex update of _csr.pyx:24-58 with the reference's exact
// operation order; explicit round-to-nearest intrinsics (and --fmad=false)
// keep every product and sum un-contracted, matching the compiled CPU kernel
// (scalar SSE2 mulsd/addsd, no FMA).
// ---------------------------------------------------------------------------
struct RowAcc {
    double w_all, w0, w1, s;
    __device__ inline void init() { w_all = w0 = w1 = s = 0.0; }
    // cls: -1 unlabeled (fv valid), 0 / 1 ground truth
    __device__ inline void add(double w, int cls, double fv, double fu) {
        w_all = __dadd_rn(w_all, w);
        if (cls == 0)
            w0 = __dadd_rn(w0, w);
        else if (cls == 1)
            w1 = __dadd_rn(w1, w);
        else
            s = __dadd_rn(s, __dmul_rn(__dsub_rn(fv, fu), w));
    }
    // returns |fn - fu| or -1 for the isolated sentinel (value 0.5)
    __device__ inline double finish(double fu, double* out_val) const {
        if (w_all <= 0.0) {
            *out_val = 0.5;
            return -1.0;
        }
        double a = __dmul_rn(__dsub_rn(0.0, fu), __ddiv_rn(w0, w_all));
        double b = __dmul_rn(__dsub_rn(1.0, fu), __ddiv_rn(w1, w_all));
        double c = __ddiv_rn(s, w_all);
        double fn = __dadd_rn(__dadd_rn(__dadd_rn(fu, a), b), c);
        if (fn < 0.0)
            fn = 0.0;
        else if (fn > 1.0)
            fn = 1.0;
        *out_val = fn;
        return fabs(__dsub_rn(fn, fu));
    }
};

// ---------------------------------------------------------------------------
// union-find (parents always point to smaller ids; root = minimum member)
// ---------------------------------------------------------------------------
__device__ inline int uf_find(int* par, int x) {
    int cur = par[x];
    if (cur != x) {
        int prev = x, next;
        while (cur > (next = ((volatile int*)par)[cur])) {
            par[prev] = next;
            prev = cur;
            cur = next;
        }
    }
    return cur;
}

// Root without path compression.  Flatten passes must not compress: a
// concurrent compression store could overwrite a slot that another thread
// has just set to its final root with a non-root ancestor.
__device__ inline int uf_root(const int* par, int x) {
    int cur = x, next;
    while ((next = par[cur]) != cur) cur = next;
    return cur;
}

__device__ inline void uf_unite(int* par, int a, int b) {
    int ra = uf_find(par, a), rb = uf_find(par, b);
    while (ra != rb) {
        if (ra < rb) {
            int t = ra;
            ra = rb;
            rb = t;
        }
        int old = atomicCAS(&par[ra], ra, rb);
        if (old == ra) break;
        ra = uf_find(par, old);
        rb = uf_find(par, rb);
    }
}

// ---------------------------------------------------------------------------
// misc
// ---------------------------------------------------------------------------
__device__ inline unsigned long long dbits(double x) { return (unsigned long long)__double_as_longlong(x); }

// max of non-negative doubles via their IEEE bit patterns
__device__ inline void atomic_max_nonneg(unsigned long long* slot, double v) {
    unsigned long long b = dbits(v);
    if (b > *(volatile unsigned long long*)slot) atomicMax(slot, b);
}

__device__ inline unsigned int ld_acquire_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Grid-wide barrier for a cooperatively launched (co-resident) grid: a
// monotone arrival counter, one atomic per CTA, acquire-spin by one thread.
// The spin reads with ld.relaxed (an ld.acquire per iteration would
// invalidate the SM's L1 -- CCTL.IVALL -- under the CTAs still working on
// that SM); one fence after the exit gives the acquire.
__device__ inline unsigned int ld_relaxed_u32(const unsigned int* p) {
    unsigned int v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ inline void grid_sync(unsigned int* ctr, unsigned int& target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        target += gridDim.x;
        __threadfence();
        atomicAdd(ctr, 1u);
        while (ld_relaxed_u32(ctr) < target) {
            __nanosleep(32);
        }
        __threadfence();
    }
    __syncthreads();
}

template <typename T>
__device__ inline T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ inline double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// aggregated append of `v` to list[*count] for the calling (coalesced) threads
__device__ inline void append_agg(int* list, long long* count, int v) {
    cooperative_groups::coalesced_group g = cooperative_groups::coalesced_threads();
    unsigned long long base = 0;
    if (g.thread_rank() == 0) base = atomicAdd((unsigned long long*)count, (unsigned long long)g.size());
    base = g.shfl(base, 0);
    list[base + g.thread_rank()] = v;
}


inline int blocks_for(long long n, int block = kBlock, int cap = 148 * 32) {
    long long b = (n + block - 1) / block;
    if (b < 1) b = 1;
    if (b > cap) b = cap;
    return (int)b;
}

}  // namespace dlp
