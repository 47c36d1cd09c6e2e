// knn.cu -- cosine k-NN edge construction on B200 tensor cores with an exact
// fp64 re-check.
//
// Reference (paths under /root/reference/pkg/src/dynlp/):
//   FeatureMatrix   builder.py:18-39  (fp64 rows, all-zero row rejected)
//   knn_graph       builder.py:42-92  (fp64 normalise :59, sims x@x.T :62-64,
//                   self -inf :65, top-k by (-sim, id) :66-68, weight = cos or
//                   (1+cos)/2 :74-76, keep w > 0 and clip [0,1] :77-82,
//                   union-symmetrise with max-merge :85-92, sorted by (lo, hi))
//
// B200 design
// * knn_norm: fp64 row norms in numpy's pairwise-summation order
//   (np.linalg.norm(axis=1) = sqrt(add.reduce(x*x))), rows divided by them
//   (IEEE division) -> the normalised fp64 rows the exact stage uses.  The same
//   kernel emits the tensor-core operands: fp16 hi/lo split h = fp16(x),
//   l = fp16(x - h), laid out along K as [h|l] for both operands; the MMA
//   issuer pairs K steps so ONE fp32 accumulator receives h.h' + l.h' + h.l'
//   (error ~1e-6 instead of ~1e-3 for a single fp16 pass) while the
//   streamed database operand is only 2D wide (each database h slab feeds
//   two MMAs).
//   Operands are stored pre-swizzled in the UMMA SWIZZLE_128B K-major layout,
//   so plain bulk copies (cp.async.bulk, SASS UBLKCP) land them ready for
//   tcgen05.mma.
// * knn_screen: persistent tcgen05 GEMM.  Warp 0 streams 256-row database
//   tiles through a 3-4 stage mbarrier ring; warp 1 (one thread) issues
//   tcgen05.mma.cta_group::1.kind::f16 (M=128 queries, N=256, K=16 steps)
//   into a double-buffered fp32 accumulator in TMEM (2 x 256 columns); warps
//   4-7 drain TMEM with tcgen05.ld and keep a per-query top-32 candidate list
//   (fp32 screened sims) plus the screening threshold.  Work items are
//   (query tile, database split) pairs so the grid fills all 148 SMs.
// * knn_recheck: per query, exact fp64 sims of all candidates (sequential,
//   no FMA), exact order (-sim, id), and a certificate: the k-th exact sim
//   must exceed every non-candidate's screened sim by the rigorous screening
//   error bound, else the query is recomputed by knn_exact (fp64 brute force
//   over all rows).  The edge SET is therefore exact.
// * knn_graph: pairs -> weights (prune / affine), keep w > 0, clip, key
//   lo*n+hi, CUB radix sort, max-merge duplicates -> EdgeList in (lo, hi) order.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_fp16.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "engine.cuh"

namespace dlp {
namespace knn {

constexpr int BM = 128;           // queries per tile (TMEM lanes)
constexpr int BN = 256;           // database rows per MMA tile (N)
constexpr int BKH = 64;           // fp16 elements per K block (128-byte rows)
constexpr int KP = 16;            // screened candidates kept per (query, split, column half)
constexpr int EPI = 2;            // epilogue warpgroups (each drains half of an accumulator)
constexpr int CH = 16;            // accumulator columns per TMEM load
constexpr int A_BLOCK = BM * 128;  // bytes of one A K-block slab (16 KB)
constexpr int B_BLOCK = BN * 128;  // bytes of one B K-block slab (32 KB)
constexpr int kThreads = 128 + 128 * EPI;
constexpr int kMaxK = 32;         // largest k served by the screened path

// ---------------------------------------------------------------------------
// numpy pairwise summation (loops_utils.h.src), recursive form
// ---------------------------------------------------------------------------
__device__ double pw_sum_sq(const double* a, long long n, long long stride_unused) {
    (void)stride_unused;
    if (n < 8) {
        double r = -0.0;
        for (long long i = 0; i < n; i++) r = __dadd_rn(r, __dmul_rn(a[i], a[i]));
        return r;
    }
    if (n <= 128) {
        double r[8];
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = __dmul_rn(a[j], a[j]);
        long long i;
        for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
            for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], __dmul_rn(a[i + j], a[i + j]));
        }
        double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                               __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < n; i++) res = __dadd_rn(res, __dmul_rn(a[i], a[i]));
        return res;
    }
    long long n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(pw_sum_sq(a, n2, 0), pw_sum_sq(a + n2, n - n2, 0));
}

// byte offset of element (row, kk) in a pre-swizzled SW128 K-major operand of
// R-row tiles with KB K-blocks: each (tile, K-block) is an R x 128 B slab and
// row r's 16-byte chunk c sits at chunk (c ^ (r & 7)) of its 128-byte line.
__host__ __device__ inline size_t sw128_off(long long row, int kk, int R, int KB) {
    long long tile = row / R;
    int rr = (int)(row - tile * R);
    int kb = kk >> 6, within = kk & 63, c = within >> 3, e = within & 7;
    return (((size_t)tile * KB + kb) * R + rr) * 128 + (size_t)((c ^ (rr & 7)) << 4) + (size_t)(e << 1);
}

// thread per row: norm, normalised fp64 row, fp16 split operands.  Both
// operands hold [h | l] along K (h at K steps [0, Dp/16), l at [Dp/16, 2Dp/16),
// Dp = D rounded up to the MMA K of 16, zero padded); the screen issues
// h.h' + l.h' for the database's h steps and h.l' for its l steps.
__global__ void k_knn_norm(const double* x, long long n, int D, int Dp, int KB, double* xn, __half* opA,
                           __half* opB, long long* bad_row) {
    for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < n; r += (long long)gridDim.x * blockDim.x) {
        const double* row = x + r * D;
        double nrm = __dsqrt_rn(pw_sum_sq(row, D, 1));
        if (!(nrm != 0.0)) {  // FeatureMatrix rejects all-zero rows (builder.py:30-33)
            atomicMin((unsigned long long*)bad_row, (unsigned long long)r);
            continue;
        }
        for (int d = 0; d < D; d++) {
            double v = __ddiv_rn(row[d], nrm);
            xn[r * D + d] = v;
            __half h = __double2half(v);
            __half l = __double2half(__dsub_rn(v, (double)__half2float(h)));
            opA[sw128_off(r, d, BM, KB) / 2] = h;
            opA[sw128_off(r, Dp + d, BM, KB) / 2] = l;
            opB[sw128_off(r, d, BN, KB) / 2] = h;
            opB[sw128_off(r, Dp + d, BN, KB) / 2] = l;
        }
    }
}

// ---------------------------------------------------------------------------
// PTX helpers: mbarrier, bulk copy, tcgen05
// ---------------------------------------------------------------------------
__device__ inline unsigned int smem_u32(const void* p) { return (unsigned int)__cvta_generic_to_shared(p); }

__device__ inline void mbar_init(unsigned long long* b, unsigned int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ inline void mbar_expect_tx(unsigned long long* b, unsigned int bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ inline void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ inline void mbar_wait(unsigned long long* b, unsigned int parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ inline void bulk_g2s(void* dst, const void* src, unsigned int bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ inline void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ inline void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ inline void tc_commit(unsigned long long* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ inline void tc_mma(unsigned int tmem_d, unsigned long long adesc, unsigned long long bdesc,
                              unsigned int idesc, unsigned int accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// SW128 K-major shared-memory matrix descriptor (tcgen05 layout_type 2)
__device__ inline unsigned long long sw128_desc(unsigned int saddr) {
    unsigned long long d = 0;
    d |= (unsigned long long)((saddr & 0x3FFFFu) >> 4);  // start address
    d |= (unsigned long long)1 << 16;                     // leading byte offset (unused for SW128 K-major)
    d |= (unsigned long long)(1024 >> 4) << 32;           // stride byte offset: 8 rows x 128 B
    d |= (unsigned long long)1 << 46;                     // descriptor version (sm_100)
    d |= (unsigned long long)2 << 61;                     // SWIZZLE_128B
    return d;
}
// kind::f16 instruction descriptor: F16 A/B, F32 D, K-major A and B
__host__ __device__ constexpr unsigned int f16_idesc(int M, int N) {
    return (1u << 4) | (0u << 7) | (0u << 10) | ((unsigned)(N >> 3) << 17) | ((unsigned)(M >> 4) << 24);
}

#define TMEM_LD16(taddr, r)                                                                                        \
    asm volatile(                                                                                                  \
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"       \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),   \
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])                      \
        : "r"(taddr))

#define TMEM_LD32(taddr, r)                                                                                        \
    asm volatile(                                                                                                  \
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19," \
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"                                                  \
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),   \
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),    \
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),   \
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])                 \
        : "r"(taddr))

// sift-down of a KP-entry min-heap stored as lv/li[slot * BM + et]
__device__ inline void heap_sift(float* lv, int* li, int et, int i) {
    float v = lv[i * BM + et];
    int id = li[i * BM + et];
    for (;;) {
        int c = 2 * i + 1;
        if (c >= KP) break;
        float cv = lv[c * BM + et];
        if (c + 1 < KP) {
            float c2 = lv[(c + 1) * BM + et];
            if (c2 < cv) {
                cv = c2;
                c++;
            }
        }
        if (!(cv < v)) break;
        lv[i * BM + et] = cv;
        li[i * BM + et] = li[c * BM + et];
        i = c;
    }
    lv[i * BM + et] = v;
    li[i * BM + et] = id;
}

struct ScreenArgs {
    const unsigned char* opA;  // query operand (pre-swizzled), tiles of BM rows
    const unsigned char* opB;  // database operand, tiles of BN rows
    int KB;                    // K blocks of [h | l] (2*Dp padded to 64)
    int hsteps;                // Dp / 16: K steps of the h half
    long long q0, nq;          // global id of query row 0 of opA, query count
    long long n_db;            // database rows
    int n_btiles;              // database tiles of BN rows
    int tiles_per_split, nsplit, nqt;
    int stages;
    float* cand_val;  // [nq][nsplit][KP]
    int* cand_id;     // [nq][nsplit][KP]
    float* cand_min;  // [nq][nsplit]: threshold (-inf if the split kept everything)
};

__global__ void __launch_bounds__(kThreads, 1) k_knn_screen(ScreenArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* base = (unsigned char*)(((size_t)smem_raw + 1023) & ~(size_t)1023);
    unsigned char* sA = base;
    unsigned char* sB = sA + (size_t)a.KB * A_BLOCK;
    // per epilogue group: heap [KP][128] + pending [CH][128] (values, ids)
    float* epi_base = (float*)(sB + (size_t)a.stages * B_BLOCK);
    unsigned long long* bars = (unsigned long long*)(epi_base + (size_t)EPI * 2 * (KP + CH) * BM);
    unsigned long long* full = bars;                     // [stages]
    unsigned long long* empty = bars + a.stages;         // [stages]
    unsigned long long* tfull = bars + 2 * a.stages;     // [2]
    unsigned long long* tempty = tfull + 2;              // [2]
    unsigned long long* afull = tempty + 2;
    unsigned long long* aempty = afull + 1;
    unsigned int* tmem_slot = (unsigned int*)(aempty + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nitems = a.nqt * a.nsplit;
    if (tid == 0) {
        for (int s = 0; s < a.stages; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; s++) {
            mbar_init(&tfull[s], 1);
            mbar_init(&tempty[s], BM * EPI);
        }
        mbar_init(afull, 1);
        mbar_init(aempty, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const unsigned int tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ===== producer: bulk copies of operand slabs =====
        int st = 0;
        unsigned int ph = 0, aph = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            const int split = it / a.nqt, qt = it - split * a.nqt;
            const int t0 = split * a.tiles_per_split, t1 = min(a.n_btiles, t0 + a.tiles_per_split);
            mbar_wait(aempty, aph ^ 1);
            aph ^= 1;
            mbar_expect_tx(afull, (unsigned int)(a.KB * A_BLOCK));
            bulk_g2s(sA, a.opA + (size_t)qt * a.KB * A_BLOCK, (unsigned int)(a.KB * A_BLOCK), afull);
            for (int t = t0; t < t1; t++) {
                for (int kb = 0; kb < a.KB; kb++) {
                    mbar_wait(&empty[st], ph ^ 1);
                    mbar_expect_tx(&full[st], B_BLOCK);
                    bulk_g2s(sB + (size_t)st * B_BLOCK, a.opB + ((size_t)t * a.KB + kb) * B_BLOCK, B_BLOCK, &full[st]);
                    if (++st == a.stages) {
                        st = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ===== MMA issuer =====
        const unsigned int idesc = f16_idesc(BM, BN);
        int st = 0, acc = 0;
        unsigned int ph = 0, aph = 0, accph = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            const int split = it / a.nqt;
            const int t0 = split * a.tiles_per_split, t1 = min(a.n_btiles, t0 + a.tiles_per_split);
            mbar_wait(afull, aph);
            aph ^= 1;
            tc_fence_after();
            for (int t = t0; t < t1; t++) {
                mbar_wait(&tempty[acc], accph ^ 1);
                tc_fence_after();
                const unsigned int dtm = tmem + (unsigned int)(acc * BN);
                const unsigned int sa0 = smem_u32(sA);
                unsigned int accum = 0;
                for (int kb = 0; kb < a.KB; kb++) {
                    mbar_wait(&full[st], ph);
                    tc_fence_after();
                    const unsigned int sb = smem_u32(sB + (size_t)st * B_BLOCK);
#pragma unroll
                    for (int k = 0; k < BKH / 16; k++) {
                        const int gs = kb * (BKH / 16) + k;  // database K step
                        const unsigned long long bd = sw128_desc(sb + k * 32);
                        if (gs < a.hsteps) {  // database h: query h and query l
                            const int qa = gs, ql = gs + a.hsteps;
                            tc_mma(dtm, sw128_desc(sa0 + (qa >> 2) * A_BLOCK + (qa & 3) * 32), bd, idesc, accum);
                            accum = 1;
                            tc_mma(dtm, sw128_desc(sa0 + (ql >> 2) * A_BLOCK + (ql & 3) * 32), bd, idesc, 1);
                        } else if (gs < 2 * a.hsteps) {  // database l: query h
                            const int qa = gs - a.hsteps;
                            tc_mma(dtm, sw128_desc(sa0 + (qa >> 2) * A_BLOCK + (qa & 3) * 32), bd, idesc, 1);
                        }
                    }
                    tc_commit(&empty[st]);  // frees the stage once these MMAs complete
                    if (++st == a.stages) {
                        st = 0;
                        ph ^= 1;
                    }
                }
                tc_commit(&tfull[acc]);
                if (++acc == 2) {
                    acc = 0;
                    accph ^= 1;
                }
            }
            tc_commit(aempty);  // the query slab may be replaced
        }
    } else if (warp >= 4) {
        // ===== epilogue: TMEM -> per-query top-KP candidates =====
        // group g drains accumulator columns [g*BN/EPI, (g+1)*BN/EPI) and keeps
        // its own candidate list per query: list index = split*EPI + g
        const int g = (warp - 4) >> 2;
        const int et = (tid - 128) & (BM - 1);  // query row within the tile == TMEM lane
        const unsigned int lane_base = (unsigned int)((warp & 3) * 32) << 16;
        float* lv = epi_base + (size_t)g * 2 * (KP + CH) * BM;
        int* li = (int*)(lv + KP * BM);
        float* pv = (float*)(li + KP * BM);
        int* pi = (int*)(pv + CH * BM);
        const int nlist = a.nsplit * EPI;
        int acc = 0;
        unsigned int accph = 0;
        for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
            const int split = it / a.nqt, qt = it - split * a.nqt;
            const int t0 = split * a.tiles_per_split, t1 = min(a.n_btiles, t0 + a.tiles_per_split);
            const long long qrow = (long long)qt * BM + et;
            const long long qid = a.q0 + qrow;
            // per-query top-KP as a min-heap in shared memory ([slot][lane]
            // layout, conflict-free), thr = its root.  A chunk's values above
            // thr are first appended (predicated, no divergence) to a pending
            // list, then merged into the heap by all lanes in lockstep.
            float thr = -INFINITY;
            int cnt = 0;
            for (int t = t0; t < t1; t++) {
                mbar_wait(&tfull[acc], accph);
                tc_fence_after();
                for (int j = 0; j < BN / EPI / CH; j++) {
                    const int col = g * (BN / EPI) + j * CH;
                    unsigned int r[CH];
                    TMEM_LD16(tmem + lane_base + (unsigned int)(acc * BN + col), r);
                    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                    const long long g0 = (long long)t * BN + col;
                    float mx = __uint_as_float(r[0]);
#pragma unroll
                    for (int c = 1; c < CH; c++) mx = fmaxf(mx, __uint_as_float(r[c]));
                    const bool special = (qid >= g0 && qid < g0 + CH) || g0 + CH > a.n_db;
                    if (!__any_sync(0xffffffffu, mx > thr || special)) continue;
                    int pc = 0;
#pragma unroll
                    for (int c = 0; c < CH; c++) {
                        const float v = __uint_as_float(r[c]);
                        const long long gid = g0 + c;
                        const bool pass = v > thr && gid < a.n_db && gid != qid;
                        if (pass) {
                            pv[pc * BM + et] = v;
                            pi[pc * BM + et] = (int)gid;
                        }
                        pc += pass ? 1 : 0;
                    }
                    for (int p = 0; p < pc; p++) {
                        const float v = pv[p * BM + et];
                        const int gid = pi[p * BM + et];
                        if (cnt < KP) {
                            lv[cnt * BM + et] = v;
                            li[cnt * BM + et] = gid;
                            if (++cnt == KP) {  // heapify once the list is full
                                for (int i0 = KP / 2 - 1; i0 >= 0; i0--) heap_sift(lv, li, et, i0);
                                thr = lv[et];
                            }
                        } else if (v > thr) {  // replace the root, restore the heap
                            lv[et] = v;
                            li[et] = gid;
                            heap_sift(lv, li, et, 0);
                            thr = lv[et];
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive(&tempty[acc]);
                if (++acc == 2) {
                    acc = 0;
                    accph ^= 1;
                }
            }
            if (qrow < a.nq) {
                const int list = split * EPI + g;
                const size_t o = ((size_t)qrow * nlist + list) * KP;
                for (int s2 = 0; s2 < KP; s2++) {
                    a.cand_val[o + s2] = s2 < cnt ? lv[s2 * BM + et] : -INFINITY;
                    a.cand_id[o + s2] = s2 < cnt ? li[s2 * BM + et] : -1;
                }
                a.cand_min[(size_t)qrow * nlist + list] = cnt < KP ? -INFINITY : thr;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---------------------------------------------------------------------------
// exact stage
// ---------------------------------------------------------------------------
__device__ inline double dot_exact(const double* a, const double* b, int D) {
    double s = 0.0;
    for (int d = 0; d < D; d++) s = __dadd_rn(s, __dmul_rn(a[d], b[d]));
    return s;
}

// (-sim, id) order: a beats b
__device__ inline bool better(double sa, long long ia, double sb, long long ib) {
    return sa > sb || (sa == sb && ia < ib);
}

// warp per query: exact sims of the candidates, top-k, certificate
__global__ void k_knn_recheck(const double* xn, int D, long long q0, long long nq, int nsplit, int k,
                              const float* cand_val, const int* cand_id, const float* cand_min, double eps,
                              long long* out_id, double* out_sim, int* failed, unsigned int* n_failed) {
    const int lane = threadIdx.x & 31;
    const long long wq = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
    const int ncand = nsplit * KP;
    for (long long q = wq; q < nq; q += nw) {
        const double* xq = xn + (q0 + q) * D;
        const float* cv = cand_val + (size_t)q * ncand;
        const int* ci = cand_id + (size_t)q * ncand;
        // lanes own candidates lane, lane+32, ...; per-lane exact sims cached in registers (ncand <= 32*16)
        double sims[16];
        int ids[16];
        const int per = (ncand + 31) / 32;
        for (int m = 0; m < 16; m++) {
            sims[m] = -INFINITY;
            ids[m] = -1;
            int c = lane + 32 * m;
            if (m < per && c < ncand && ci[c] >= 0) {
                ids[m] = ci[c];
                sims[m] = dot_exact(xq, xn + (long long)ci[c] * D, D);
            }
        }
        float thr_f = -INFINITY;
        for (int s = lane; s < nsplit; s += 32) thr_f = fmaxf(thr_f, cand_min[(size_t)q * nsplit + s]);
        for (int o = 16; o > 0; o >>= 1) thr_f = fmaxf(thr_f, __shfl_xor_sync(0xffffffffu, thr_f, o));
        double kth = INFINITY;
        for (int r = 0; r < k; r++) {
            // lane-local best
            double bs = -INFINITY;
            long long bi = 0x7fffffffffffffffLL;
            int bm = -1;
            for (int m = 0; m < per && m < 16; m++)
                if (ids[m] >= 0 && better(sims[m], ids[m], bs, bi)) {
                    bs = sims[m];
                    bi = ids[m];
                    bm = m;
                }
            double ws = bs;
            long long wi = bi;
            for (int o = 16; o > 0; o >>= 1) {
                double os = __shfl_xor_sync(0xffffffffu, ws, o);
                long long oi = __shfl_xor_sync(0xffffffffu, wi, o);
                if (better(os, oi, ws, wi)) {
                    ws = os;
                    wi = oi;
                }
            }
            if (lane == 0) {
                out_id[q * k + r] = wi == 0x7fffffffffffffffLL ? -1 : wi;
                out_sim[q * k + r] = ws;
            }
            if (bm >= 0 && bi == wi) ids[bm] = -1;  // consumed
            kth = ws;
        }
        // certificate: every non-candidate has screened sim <= thr_f, hence exact
        // sim <= thr_f + eps; it cannot reach the k-th place if kth > thr_f + eps
        const bool ok = (thr_f == -INFINITY) || (kth > (double)thr_f + eps);
        if (!ok && lane == 0) failed[atomicAdd(n_failed, 1u)] = (int)q;
    }
}

// CTA per failed query: exact fp64 scan of every row (and the path for k > kMaxK)
constexpr int kExactThreads = 128;
__global__ void __launch_bounds__(kExactThreads) k_knn_exact(const double* xn, int D, long long n, long long q0,
                                                            const int* qlist, const unsigned int* nlist,
                                                            long long nq_all, int k, long long* out_id,
                                                            double* out_sim) {
    extern __shared__ unsigned char sm[];
    double* ls = (double*)sm;                                  // [kExactThreads][k]
    long long* li = (long long*)(ls + (size_t)kExactThreads * k);  // [kExactThreads][k]
    const int tid = threadIdx.x;
    const long long nwork = qlist ? (long long)*nlist : nq_all;
    for (long long w = blockIdx.x; w < nwork; w += gridDim.x) {
        const long long q = qlist ? qlist[w] : w;
        const long long qid = q0 + q;
        const double* xq = xn + qid * D;
        double* ms = ls + (size_t)tid * k;
        long long* mi = li + (size_t)tid * k;
        for (int j = 0; j < k; j++) {
            ms[j] = -INFINITY;
            mi[j] = 0x7fffffffffffffffLL;
        }
        for (long long y = tid; y < n; y += kExactThreads) {
            if (y == qid) continue;  // self = -inf (builder.py:65)
            double s = dot_exact(xq, xn + y * D, D);
            if (!better(s, y, ms[k - 1], mi[k - 1])) continue;
            int j = k - 1;
            while (j > 0 && better(s, y, ms[j - 1], mi[j - 1])) {
                ms[j] = ms[j - 1];
                mi[j] = mi[j - 1];
                j--;
            }
            ms[j] = s;
            mi[j] = y;
        }
        __syncthreads();
        if (tid < 32) {  // warp 0 merges the sorted per-thread lists
            int head[kExactThreads / 32];
            for (int h = 0; h < kExactThreads / 32; h++) head[h] = 0;
            for (int r = 0; r < k; r++) {
                double bs = -INFINITY;
                long long bi = 0x7fffffffffffffffLL;
                int bh = -1;
                for (int h = 0; h < kExactThreads / 32; h++) {
                    int t = tid + 32 * h;
                    if (head[h] < k) {
                        double s = ls[(size_t)t * k + head[h]];
                        long long i = li[(size_t)t * k + head[h]];
                        if (better(s, i, bs, bi)) {
                            bs = s;
                            bi = i;
                            bh = h;
                        }
                    }
                }
                double ws = bs;
                long long wi = bi;
                for (int o = 16; o > 0; o >>= 1) {
                    double os = __shfl_xor_sync(0xffffffffu, ws, o);
                    long long oi = __shfl_xor_sync(0xffffffffu, wi, o);
                    if (better(os, oi, ws, wi)) {
                        ws = os;
                        wi = oi;
                    }
                }
                if (bh >= 0 && bi == wi) head[bh]++;
                if (tid == 0) {
                    out_id[q * k + r] = wi == 0x7fffffffffffffffLL ? -1 : wi;
                    out_sim[q * k + r] = ws;
                }
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// symmetrisation (builder.py:74-92)
// ---------------------------------------------------------------------------
__global__ void k_knn_pairs(const long long* ids, const double* sims, long long nq, int k, long long n, int affine,
                            unsigned long long* key, double* w, unsigned int* m) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nq * k;
         i += (long long)gridDim.x * blockDim.x) {
        long long src = i / k, dst = ids[i];
        if (dst < 0) continue;
        double s = sims[i];
        double wt = affine ? __ddiv_rn(__dadd_rn(1.0, s), 2.0) : s;
        if (!(wt > 0.0)) continue;  // keep = w > 0
        if (wt > 1.0) wt = 1.0;     // np.clip(w, 0, 1)
        long long lo = src < dst ? src : dst, hi = src < dst ? dst : src;
        unsigned int p = atomicAdd(m, 1u);
        key[p] = (unsigned long long)lo * (unsigned long long)n + (unsigned long long)hi;
        w[p] = wt;
    }
}

__global__ void k_knn_merge(const unsigned long long* key, const double* w, unsigned int m, unsigned long long n,
                            long long* u, long long* v, double* wo, const unsigned int* pos) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
        if (i > 0 && key[i - 1] == key[i]) continue;
        double best = w[i];
        for (long long j = i + 1; j < m && key[j] == key[i]; j++) best = fmax(best, w[j]);
        unsigned int o = pos[i];
        u[o] = (long long)(key[i] / n);
        v[o] = (long long)(key[i] % n);
        wo[o] = best;
    }
}

__global__ void k_knn_heads(const unsigned long long* key, unsigned int m, unsigned int* flag) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
        flag[i] = (i == 0 || key[i - 1] != key[i]) ? 1u : 0u;
}

}  // namespace knn
}  // namespace dlp

using namespace dlp;
using namespace dlp::knn;

// ===========================================================================
// host side
// ===========================================================================
struct dlp_knn {
    int device = 0;
    cudaStream_t st = nullptr;
    int sm_count = 148;
    std::string err;
    long long n = 0;
    int D = 0, Dp = 0, KB = 0;
    DevArray<double> x, xn;
    DevArray<unsigned char> opA, opB;  // query operand covers all rows (queries are row ranges)
    DevArray<float> cand_val, cand_min;
    DevArray<int> cand_id, failed;
    DevArray<unsigned int> counters;
    DevArray<long long> top_id, bad;
    DevArray<double> top_sim;
    // graph output
    DevArray<unsigned long long> key_a, key_b;
    DevArray<double> w_a, w_b;
    DevArray<unsigned int> flag, pos;
    DevArray<unsigned char> cub_tmp;
    DevArray<long long> eu, ev;
    DevArray<double> ew;
    long long m_edges = 0;
    // stats of the last call
    double screen_ms = 0, recheck_ms = 0, exact_ms = 0;
    long long n_fallback = 0, n_queries = 0;
    double eps = 0;
    cudaEvent_t tev[4] = {nullptr, nullptr, nullptr, nullptr};
};

namespace {

// database splits per query tile: enough (query tile, split) items to fill
// every SM, chosen to minimise the last-wave idle fraction
int choose_nsplit(int nqt, int n_btiles, int sms) {
    int best = 1;
    double best_eff = -1.0;
    for (int s = 1; s <= std::min(16, n_btiles); s++) {
        const int tps = (n_btiles + s - 1) / s;
        const int sp = (n_btiles + tps - 1) / tps;
        const long long items = (long long)nqt * sp;
        const long long waves = (items + sms - 1) / sms;
        double eff = (double)items / (double)(waves * sms);
        if (items < sms) eff *= 0.5;  // under-filled grid
        if (eff > best_eff + 1e-9) {
            best_eff = eff;
            best = s;
        }
    }
    return best;
}

int kfail(dlp_knn* h, int code, const char* msg) {
    h->err = msg;
    return code;
}

// rigorous bound on |screened - exact| for unit vectors (see header comment):
// dropped l.l' and second-order rounding terms, plus fp32 accumulation of
// 3D exact fp16 products (2^-23 relative per addition, partial sums <= ~1.02)
double screen_eps(int D) {
    double k3 = 3.0 * ((D + 15) / 16 * 16);
    return k3 * std::ldexp(1.0, -23) * 1.02 + std::ldexp(1.0, -20) + 2.0 * std::ldexp(1.0, -25) * std::sqrt((double)D) +
           std::ldexp(1.0, -21) + 1e-12;
}

int run_queries(dlp_knn* h, long long q0, long long nq, int k) {
    cudaStream_t st = h->st;
    const long long n = h->n;
    const int D = h->D;
    h->n_queries = nq;
    h->n_fallback = 0;
    h->top_id.reserve((size_t)nq * k + 1, 0, st);
    h->top_sim.reserve((size_t)nq * k + 1, 0, st);
    h->counters.reserve(4, 0, st);
    DLP_CUDA_TRY(cudaMemsetAsync(h->counters.p, 0, 4 * sizeof(unsigned int), st));
    h->failed.reserve(nq + 1, 0, st);
    DLP_CUDA_TRY(cudaEventRecord(h->tev[0], st));
    if (k <= kMaxK && nq > 0) {
        // --- screen: (query tile, database split) work items over all SMs
        const int nqt = (int)((nq + BM - 1) / BM);
        const int n_btiles = (int)((n + BN - 1) / BN);
        int nsplit = choose_nsplit(nqt, n_btiles, h->sm_count);
        const int tps = (n_btiles + nsplit - 1) / nsplit;
        nsplit = (n_btiles + tps - 1) / tps;
        ScreenArgs a;
        a.opA = h->opA.p + (size_t)(q0 / BM) * h->KB * A_BLOCK;
        a.opB = h->opB.p;
        a.KB = h->KB;
        a.hsteps = h->Dp / 16;
        a.q0 = (q0 / BM) * BM;  // screening works on whole query tiles
        long long qpad = q0 - a.q0;
        a.nq = nq + qpad;
        a.n_db = n;
        a.n_btiles = n_btiles;
        a.nsplit = nsplit;
        a.tiles_per_split = tps;
        a.nqt = (int)((a.nq + BM - 1) / BM);
        const size_t fixed = (size_t)h->KB * A_BLOCK + (size_t)EPI * (KP + CH) * BM * 8 + 1024 + 256;
        const size_t limit = 227 * 1024;
        a.stages = (int)std::min<size_t>(8, (limit - fixed) / B_BLOCK);
        if (a.stages < 2) return kfail(h, DLP_EVALIDATION, "feature dimension too large for the tensor-core screen");
        // candidate buffers are indexed by the padded query row
        const int nlist = nsplit * EPI;
        h->cand_val.reserve((size_t)a.nq * nlist * KP, 0, st);
        h->cand_id.reserve((size_t)a.nq * nlist * KP, 0, st);
        h->cand_min.reserve((size_t)a.nq * nlist, 0, st);
        a.cand_val = h->cand_val.p;
        a.cand_id = h->cand_id.p;
        a.cand_min = h->cand_min.p;
        const size_t smem = fixed + (size_t)a.stages * B_BLOCK;
        DLP_CUDA_TRY(cudaFuncSetAttribute(k_knn_screen, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const int items = a.nqt * a.nsplit;
        k_knn_screen<<<std::min(items, h->sm_count), kThreads, smem, st>>>(a);
        DLP_CUDA_TRY(cudaGetLastError());
        DLP_CUDA_TRY(cudaEventRecord(h->tev[1], st));
        // --- exact re-check with certificate
        k_knn_recheck<<<blocks_for(nq * 32, 256, 148 * 16), 256, 0, st>>>(
            h->xn.p, D, q0, nq, nlist, k, h->cand_val.p + (size_t)qpad * nlist * KP,
            h->cand_id.p + (size_t)qpad * nlist * KP, h->cand_min.p + (size_t)qpad * nlist, h->eps, h->top_id.p,
            h->top_sim.p, h->failed.p, h->counters.p);
        DLP_CUDA_TRY(cudaGetLastError());
        DLP_CUDA_TRY(cudaEventRecord(h->tev[2], st));
        unsigned int nf = 0;
        DLP_CUDA_TRY(cudaMemcpyAsync(&nf, h->counters.p, sizeof(nf), cudaMemcpyDeviceToHost, st));
        DLP_CUDA_TRY(cudaStreamSynchronize(st));
        h->n_fallback = nf;
        if (nf) {
            size_t sm = (size_t)kExactThreads * k * 16;
            DLP_CUDA_TRY(cudaFuncSetAttribute(k_knn_exact, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            k_knn_exact<<<std::min<long long>(nf, 4 * h->sm_count), kExactThreads, sm, st>>>(
                h->xn.p, D, n, q0, h->failed.p, h->counters.p, nq, k, h->top_id.p, h->top_sim.p);
            DLP_CUDA_TRY(cudaGetLastError());
        }
    } else if (nq > 0) {  // k beyond the screened path: exact scan for every query
        DLP_CUDA_TRY(cudaEventRecord(h->tev[1], st));
        DLP_CUDA_TRY(cudaEventRecord(h->tev[2], st));
        size_t sm = (size_t)kExactThreads * k * 16;
        if (sm > 200 * 1024) return kfail(h, DLP_EVALIDATION, "k too large");
        DLP_CUDA_TRY(cudaFuncSetAttribute(k_knn_exact, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k_knn_exact<<<std::min<long long>(nq, 4 * h->sm_count), kExactThreads, sm, st>>>(
            h->xn.p, D, n, q0, nullptr, nullptr, nq, k, h->top_id.p, h->top_sim.p);
        DLP_CUDA_TRY(cudaGetLastError());
        h->n_fallback = nq;
    } else {
        DLP_CUDA_TRY(cudaEventRecord(h->tev[1], st));
        DLP_CUDA_TRY(cudaEventRecord(h->tev[2], st));
    }
    DLP_CUDA_TRY(cudaEventRecord(h->tev[3], st));
    DLP_CUDA_TRY(cudaStreamSynchronize(st));
    float t01 = 0, t12 = 0, t23 = 0;
    cudaEventElapsedTime(&t01, h->tev[0], h->tev[1]);
    cudaEventElapsedTime(&t12, h->tev[1], h->tev[2]);
    cudaEventElapsedTime(&t23, h->tev[2], h->tev[3]);
    h->screen_ms = t01;
    h->recheck_ms = t12;
    h->exact_ms = t23;
    return DLP_OK;
}

}  // namespace

extern "C" {

int dlp_knn_create(int device, dlp_knn** out) {
    *out = nullptr;
    auto* h = new dlp_knn();
    try {
        int ndev = 0;
        DLP_CUDA_TRY(cudaGetDeviceCount(&ndev));
        if (device < 0 || device >= ndev) {
            delete h;
            return DLP_ECUDA;
        }
        h->device = device;
        DLP_CUDA_TRY(cudaSetDevice(device));
        cudaDeviceProp prop;
        DLP_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
        h->sm_count = prop.multiProcessorCount;
        if (prop.major != 10) {
            delete h;
            return DLP_ECUDA;  // tcgen05 screen needs sm_100
        }
        DLP_CUDA_TRY(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking));
        for (auto& e : h->tev) DLP_CUDA_TRY(cudaEventCreate(&e));
    } catch (const CudaFailure&) {
        delete h;
        return DLP_ECUDA;
    }
    *out = h;
    return DLP_OK;
}

int dlp_knn_destroy(dlp_knn* h) {
    if (!h) return DLP_OK;
    cudaSetDevice(h->device);
    cudaStreamSynchronize(h->st);
    h->x.release();
    h->xn.release();
    h->opA.release();
    h->opB.release();
    h->cand_val.release();
    h->cand_min.release();
    h->cand_id.release();
    h->failed.release();
    h->counters.release();
    h->top_id.release();
    h->bad.release();
    h->top_sim.release();
    h->key_a.release();
    h->key_b.release();
    h->w_a.release();
    h->w_b.release();
    h->flag.release();
    h->pos.release();
    h->cub_tmp.release();
    h->eu.release();
    h->ev.release();
    h->ew.release();
    for (auto e : h->tev)
        if (e) cudaEventDestroy(e);
    if (h->st) cudaStreamDestroy(h->st);
    delete h;
    return DLP_OK;
}

const char* dlp_knn_last_error(dlp_knn* h) { return h ? h->err.c_str() : "null handle"; }

int dlp_knn_set_features(dlp_knn* h, const double* rows, int64_t n, int64_t d) {
    if (!h) return DLP_EINTERNAL;
    if (n < 1 || d < 1) return kfail(h, DLP_EVALIDATION, "feature matrix must be 2-D and non-empty");
    try {
        DLP_CUDA_TRY(cudaSetDevice(h->device));
        cudaStream_t st = h->st;
        const int D = (int)d;
        const int Dp = (D + 15) / 16 * 16;
        const int KB = (2 * Dp + BKH - 1) / BKH;
        h->x.reserve((size_t)n * D, 0, st);
        h->xn.reserve((size_t)n * D, 0, st);
        DLP_CUDA_TRY(cudaMemcpyAsync(h->x.p, rows, (size_t)n * D * sizeof(double), cudaMemcpyHostToDevice, st));
        const long long ta = (n + BM - 1) / BM, tb = (n + BN - 1) / BN;
        const size_t bytesA = (size_t)ta * KB * A_BLOCK, bytesB = (size_t)tb * KB * B_BLOCK;
        h->opA.reserve(bytesA, 0, st);
        h->opB.reserve(bytesB, 0, st);
        DLP_CUDA_TRY(cudaMemsetAsync(h->opA.p, 0, bytesA, st));  // K padding and padded rows = 0
        DLP_CUDA_TRY(cudaMemsetAsync(h->opB.p, 0, bytesB, st));
        h->bad.reserve(1, 0, st);
        long long big = 0x7fffffffffffffffLL;
        DLP_CUDA_TRY(cudaMemcpyAsync(h->bad.p, &big, sizeof(big), cudaMemcpyHostToDevice, st));
        k_knn_norm<<<blocks_for(n, 128, 148 * 32), 128, 0, st>>>(h->x.p, n, D, Dp, KB, h->xn.p, (__half*)h->opA.p,
                                                                 (__half*)h->opB.p, h->bad.p);
        DLP_CUDA_TRY(cudaGetLastError());
        long long bad = 0;
        DLP_CUDA_TRY(cudaMemcpyAsync(&bad, h->bad.p, sizeof(bad), cudaMemcpyDeviceToHost, st));
        DLP_CUDA_TRY(cudaStreamSynchronize(st));
        if (bad != big) {
            char buf[128];
            snprintf(buf, sizeof buf, "all-zero feature row %lld (cosine undefined)", bad);
            h->n = 0;
            return kfail(h, DLP_EVALIDATION, buf);
        }
        h->n = n;
        h->D = D;
        h->KB = KB;
        h->Dp = Dp;
        h->eps = screen_eps(D);
    } catch (const CudaFailure& f) {
        h->err = std::string("CUDA error: ") + cudaGetErrorString(f.err);
        return DLP_ECUDA;
    }
    return DLP_OK;
}

int dlp_knn_query(dlp_knn* h, int64_t q0, int64_t q1, int32_t k, int64_t* ids, double* sims) {
    if (!h) return DLP_EINTERNAL;
    if (h->n == 0) return kfail(h, DLP_EVALIDATION, "no feature matrix");
    if (!(1 <= k && k < h->n)) return kfail(h, DLP_EVALIDATION, "k must be in [1, n-1]");
    if (q0 < 0 || q1 > h->n || q0 > q1) return kfail(h, DLP_EVALIDATION, "query range out of bounds");
    try {
        DLP_CUDA_TRY(cudaSetDevice(h->device));
        int rc = run_queries(h, q0, q1 - q0, k);
        if (rc) return rc;
        size_t cnt = (size_t)(q1 - q0) * k;
        if (ids) DLP_CUDA_TRY(cudaMemcpy(ids, h->top_id.p, cnt * sizeof(long long), cudaMemcpyDeviceToHost));
        if (sims) DLP_CUDA_TRY(cudaMemcpy(sims, h->top_sim.p, cnt * sizeof(double), cudaMemcpyDeviceToHost));
    } catch (const CudaFailure& f) {
        h->err = std::string("CUDA error: ") + cudaGetErrorString(f.err);
        return DLP_ECUDA;
    }
    return DLP_OK;
}

int dlp_knn_graph(dlp_knn* h, int32_t k, int32_t affine, int64_t* m_out) {
    if (!h) return DLP_EINTERNAL;
    if (h->n == 0) return kfail(h, DLP_EVALIDATION, "no feature matrix");
    if (!(1 <= k && k < h->n)) {
        char buf[96];
        snprintf(buf, sizeof buf, "k must be in [1, %lld]", h->n - 1);
        return kfail(h, DLP_EVALIDATION, buf);
    }
    try {
        DLP_CUDA_TRY(cudaSetDevice(h->device));
        cudaStream_t st = h->st;
        const long long n = h->n;
        // all rows as queries, in chunks that bound the candidate buffers
        const long long chunk = 1 << 16;
        DevArray<long long> all_id;
        DevArray<double> all_sim;
        all_id.reserve((size_t)n * k, 0, st);
        all_sim.reserve((size_t)n * k, 0, st);
        double sms = 0, rms = 0, ems = 0;
        long long nfb = 0;
        for (long long q0 = 0; q0 < n; q0 += chunk) {
            long long nq = std::min(chunk, n - q0);
            int rc = run_queries(h, q0, nq, k);
            if (rc) {
                all_id.release();
                all_sim.release();
                return rc;
            }
            sms += h->screen_ms;
            rms += h->recheck_ms;
            ems += h->exact_ms;
            nfb += h->n_fallback;
            DLP_CUDA_TRY(cudaMemcpyAsync(all_id.p + q0 * k, h->top_id.p, (size_t)nq * k * 8, cudaMemcpyDeviceToDevice, st));
            DLP_CUDA_TRY(cudaMemcpyAsync(all_sim.p + q0 * k, h->top_sim.p, (size_t)nq * k * 8, cudaMemcpyDeviceToDevice, st));
        }
        h->screen_ms = sms;
        h->recheck_ms = rms;
        h->exact_ms = ems;
        h->n_fallback = nfb;
        h->n_queries = n;
        const size_t np = (size_t)n * k;
        h->key_a.reserve(np + 1, 0, st);
        h->key_b.reserve(np + 1, 0, st);
        h->w_a.reserve(np + 1, 0, st);
        h->w_b.reserve(np + 1, 0, st);
        h->flag.reserve(np + 1, 0, st);
        h->pos.reserve(np + 1, 0, st);
        h->counters.reserve(4, 0, st);
        DLP_CUDA_TRY(cudaMemsetAsync(h->counters.p, 0, 4 * sizeof(unsigned int), st));
        k_knn_pairs<<<blocks_for((long long)np), 256, 0, st>>>(all_id.p, all_sim.p, n, k, n, affine, h->key_a.p, h->w_a.p,
                                                             h->counters.p);
        unsigned int m = 0;
        DLP_CUDA_TRY(cudaMemcpyAsync(&m, h->counters.p, sizeof(m), cudaMemcpyDeviceToHost, st));
        DLP_CUDA_TRY(cudaStreamSynchronize(st));
        all_id.release();
        all_sim.release();
        long long mu = 0;
        if (m) {
            int bits = 1;
            unsigned long long maxkey = (unsigned long long)n * (unsigned long long)n;
            while (bits < 64 && (1ULL << bits) <= maxkey) bits++;
            size_t tb = 0;
            cub::DeviceRadixSort::SortPairs(nullptr, tb, h->key_a.p, h->key_b.p, h->w_a.p, h->w_b.p, (int)m, 0, bits, st);
            h->cub_tmp.reserve(tb + 256, 0, st);
            cub::DeviceRadixSort::SortPairs(h->cub_tmp.p, tb, h->key_a.p, h->key_b.p, h->w_a.p, h->w_b.p, (int)m, 0, bits,
                                            st);
            k_knn_heads<<<blocks_for(m), 256, 0, st>>>(h->key_b.p, m, h->flag.p);
            size_t tb2 = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, tb2, h->flag.p, h->pos.p, (int)m, st);
            h->cub_tmp.reserve(tb2 + 256, 0, st);
            cub::DeviceScan::ExclusiveSum(h->cub_tmp.p, tb2, h->flag.p, h->pos.p, (int)m, st);
            unsigned int lastp = 0, lastf = 0;
            DLP_CUDA_TRY(cudaMemcpyAsync(&lastp, h->pos.p + m - 1, 4, cudaMemcpyDeviceToHost, st));
            DLP_CUDA_TRY(cudaMemcpyAsync(&lastf, h->flag.p + m - 1, 4, cudaMemcpyDeviceToHost, st));
            DLP_CUDA_TRY(cudaStreamSynchronize(st));
            mu = (long long)lastp + lastf;
            h->eu.reserve(mu + 1, 0, st);
            h->ev.reserve(mu + 1, 0, st);
            h->ew.reserve(mu + 1, 0, st);
            k_knn_merge<<<blocks_for(m), 256, 0, st>>>(h->key_b.p, h->w_b.p, m, (unsigned long long)n, h->eu.p, h->ev.p,
                                                      h->ew.p, h->pos.p);
            DLP_CUDA_TRY(cudaGetLastError());
            DLP_CUDA_TRY(cudaStreamSynchronize(st));
        }
        h->m_edges = mu;
        *m_out = mu;
    } catch (const CudaFailure& f) {
        h->err = std::string("CUDA error: ") + cudaGetErrorString(f.err);
        return DLP_ECUDA;
    }
    return DLP_OK;
}

int dlp_knn_read_edges(dlp_knn* h, int64_t* u, int64_t* v, double* w, int64_t m) {
    if (!h) return DLP_EINTERNAL;
    if (m != h->m_edges) return kfail(h, DLP_EVALIDATION, "edge count mismatch");
    if (m == 0) return DLP_OK;
    try {
        DLP_CUDA_TRY(cudaSetDevice(h->device));
        DLP_CUDA_TRY(cudaMemcpy(u, h->eu.p, m * 8, cudaMemcpyDeviceToHost));
        DLP_CUDA_TRY(cudaMemcpy(v, h->ev.p, m * 8, cudaMemcpyDeviceToHost));
        DLP_CUDA_TRY(cudaMemcpy(w, h->ew.p, m * 8, cudaMemcpyDeviceToHost));
    } catch (const CudaFailure& f) {
        h->err = std::string("CUDA error: ") + cudaGetErrorString(f.err);
        return DLP_ECUDA;
    }
    return DLP_OK;
}

int dlp_knn_stats(dlp_knn* h, double* screen_ms, double* recheck_ms, double* exact_ms, int64_t* n_fallback,
                  int64_t* n_queries, double* eps) {
    if (!h) return DLP_EINTERNAL;
    *screen_ms = h->screen_ms;
    *recheck_ms = h->recheck_ms;
    *exact_ms = h->exact_ms;
    *n_fallback = h->n_fallback;
    *n_queries = h->n_queries;
    *eps = h->eps;
    return DLP_OK;
}

// Raw screened candidates of the last query call (tests of the tensor-core
// stage): val/id [nq][nsplit*KP], thr [nq][nsplit].
int dlp_knn_debug_candidates(dlp_knn* h, int64_t q0, int64_t q1, int32_t* nsplit_out, float* val, int32_t* id,
                             float* thr, int64_t cap) {
    if (!h) return DLP_EINTERNAL;
    try {
        DLP_CUDA_TRY(cudaSetDevice(h->device));
        const long long nq = q1 - q0;
        const int nqt = (int)((nq + BM - 1) / BM);
        const int n_btiles = (int)((h->n + BN - 1) / BN);
        int nsplit = choose_nsplit(nqt, n_btiles, h->sm_count);
        const int tps = (n_btiles + nsplit - 1) / nsplit;
        nsplit = (n_btiles + tps - 1) / tps;
        const int nlist = nsplit * EPI;
        *nsplit_out = nlist;  // candidate lists per query, KP each
        if ((long long)nq * nlist * KP > cap) return kfail(h, DLP_EVALIDATION, "capacity too small");
        const long long qpad = q0 - (q0 / BM) * BM;
        DLP_CUDA_TRY(cudaMemcpy(val, h->cand_val.p + (size_t)qpad * nlist * KP, (size_t)nq * nlist * KP * 4,
                                cudaMemcpyDeviceToHost));
        DLP_CUDA_TRY(cudaMemcpy(id, h->cand_id.p + (size_t)qpad * nlist * KP, (size_t)nq * nlist * KP * 4,
                                cudaMemcpyDeviceToHost));
        DLP_CUDA_TRY(cudaMemcpy(thr, h->cand_min.p + (size_t)qpad * nlist, (size_t)nq * nlist * 4,
                                cudaMemcpyDeviceToHost));
    } catch (const CudaFailure& f) {
        h->err = std::string("CUDA error: ") + cudaGetErrorString(f.err);
        return DLP_ECUDA;
    }
    return DLP_OK;
}

}  // extern "C"
