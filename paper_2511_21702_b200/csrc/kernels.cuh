// Device side of the B200 CSV-Decode step: one persistent cooperative kernel.
//
//   stage h in shared memory; bulk-prefetch this CTA's centroid rows to L2
//   bounds   U_c = ((<mu_c,h> + R_c*||h||) + maxb_c)        warp per cluster   bounds.py:79-83
//   == grid barrier ==
//   rank     every CTA stages U, log|c|, |c|, exp(x - M) in shared memory; each
//            warp ranks its own clusters by (-U, id) and writes order / Uo /
//            prefix token count / log R-hat at that rank: no sort, no serial
//            CTA (decode.py:166, certify.py:114-119).  Clusters predicted to be
//            in the first wave get their W rows bulk-prefetched to L2.
//   == grid barrier ==
//   every CTA loads the ordering into shared memory and plans wave 1 itself
//   loop:
//     rows   gathered GEMV over the wave's rows (W permuted: each cluster is a
//            contiguous row range), bit-exact f64 logits        decode.py:169-176
//     == grid barrier ==
//     every CTA summarises the wave's clusters (top-k, LSE, min, max) and runs
//     the identical certification scan (scan.cuh): done / next wave / dense
//   dense (fallback): full-vocabulary GEMV scattered to token order, per-warp
//     top-k candidates; == grid barrier ==; CTA 0 radix-selects the k-th logit.
//
// All CTAs take the same decisions from the same data with the same code, so
// no state needs broadcasting.  The launch is cooperative (grid barriers need
// residency); the barrier spin has a timeout that flags CSVD_ESTATE instead of
// hanging.  Code on the per-step path is kept compact on purpose: it runs with
// a cold instruction cache (L2 is flushed between timed steps, and by the rest
// of a model between real decode steps).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/csvd_b200.h"
#include "pw.cuh"
#include "scan.cuh"

#define WARPS 8
#define THREADS (WARPS * 32)
#ifndef CSVD_SPIN_NS
#define CSVD_SPIN_NS 64
#endif
#define MAX_PER_WARP 64  // clusters per warp in the bounds phase (small grids: batch lanes)
#define CHUNK 32        // max clusters per scan chunk (one per lane)

enum { LAUNCH_STEP = 0, LAUNCH_BOUNDS = 1, LAUNCH_DENSE = 2, LAUNCH_SHARD = 3 };

// Per-step workspace of one batch lane (grouped launches: lane b's CTAs are
// blockIdx.x in [b*G, (b+1)*G) and swap these pointers into their Dev).
struct LaneWS {
    const double *h;
    double *U, *Uraw, *dots;
    int *order_g, *cum_g;
    double *S_logits;
    long long *S_ids;
    ScanState *st;
    csvd_result *res;
    unsigned *bar;
    double *cand, *klists, *shard_out;
    csvd_result *res_host;
    long long *ids_host;
    double *logits_host;
    int *hcnt;                 // head lanes: completion counters [HMAX + 1]
    unsigned long long *bar64; // head lanes: [0] step count, [1] decision word
};

struct Dev {
    int V, d, C, Cp, bd, mode, wdtype;  // Cp: C rounded up to a power of two (sort)
    int K;  // top-k capacity (row stride of the dense candidate lists, list buffers)
    const void *W;      // [V, d] permuted rows (fp32 | bf16)
    const double *bias; // [V] permuted, f64 (EmbeddingTable.bias, tensor_io.py:69-94)
    const int *perm;    // [V] position -> token id
    const double *cent; // [C, bd]
    const double *radii, *maxb, *cnorm, *ang, *maxn, *minn, *logsz, *meanb;
    const int *starts, *sizes;
    // W rows present on this device: cluster c's rows start at local row
    // wrow0[c] (-1: another shard owns c); dense walks local rows lr < Vl,
    // global position lpos[lr] (lpos null: lr itself, the unsharded table)
    const int *wrow0;
    const int *lpos;
    int Vl;
    int *order_g, *cum_g;    // shard opens: the opening order / prefix counts for the host
    double *shard_out;       // CSVD_SH_* aggregate (K + CSVD_SH_TOPK doubles)
    // host-API steps: the result lands directly in mapped pinned host memory
    // (no copy nodes); the host reads it once the kernel has completed
    csvd_result *res_host;   // null: device-resident step
    long long *ids_host;
    double *logits_host;
    PwPlan wplan, bplan;
    const int *wsrc, *bsrc;  // interleaved-layout source tables (CPL < 8 plans)
    // per step
    const double *h;         // [d]
    const csvd_config *cfg;
    double *U, *Uraw, *dots; // [C] by cluster id (U final with slack; Uraw / dots from the bounds phase)
    double *klists;          // null, or per-CTA global K-lists (k too large for shared memory)
    size_t klist_stride;     // doubles per CTA in klists
    double *S_logits;        // [V]
    long long *S_ids;        // [V]
    double *cand;            // [nwarps*K] dense per-warp candidates
    ScanState *st;           // final state (diagnostic)
    csvd_result *res;
    unsigned *bar;           // grid barrier: [0] arrivals, [1] generation
    int nblocks;
    int launch_mode;
    int pre_bounds;          // 1: Uraw / dots / query_norm come from k_bounds_batch
    int dense_pd;            // k_dense_gemv: rows prefetched ahead per warp
    int pf_mask;             // L2 bulk prefetch: 1 centroid rows + per-cluster arrays, 2 wave rows
    const LaneWS *lanes;     // grouped batch launch: per-lane workspaces (null otherwise)
    int hs_off_b;            // offset (doubles) of the bounds h layout, 0 = shared with W
    int scratch_off;         // generic-path per-warp leaf scratch
    int ord_off;             // ordering arrays (rank staging, then order/cum/Uo/lrh)
    int sum_off;             // chunk summaries + scan scratch
    int chunk;               // clusters per summary/scan chunk (<= CHUNK)
    unsigned long long *dbg; // optional phase timestamps (CSVD_DEBUG_TS)
    // head kernel (headstep.cuh): cluster summaries [3*HMAX + HMAX*KH], row /
    // cluster completion counters [HMAX + 1], monotone grid-barrier counter
    double *gsum;  // per-cluster summaries of a wave [3 C + 32 C] (distributed summaries)
    int *hcnt;
    unsigned long long *bar64;
};

// this CTA's index / the CTA count of its step's grid: the whole launch, or
// one batch lane's group of D.nblocks CTAs in a grouped launch
#define CTA_ID ((int)(blockIdx.x % (unsigned)D.nblocks))
#define CTA_N (D.nblocks)

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// the CTA whose phases the debug timestamps of shared helpers follow (CTA 0
// in k_step; the scanning CTA in k_head)
static __device__ int g_dbg_cta = 0;
#define DBG_HERE(D) ((D).dbg && (int)blockIdx.x == g_dbg_cta)
#define DBG_TS(D, slot)                                    \
    do {                                                   \
        if ((D).dbg) {                                     \
            (D).dbg[(slot)] = gtimer();                    \
            (D).dbg[64 + (slot)] = clock64();              \
        }                                                  \
    } while (0)

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// TMA bulk prefetch of a contiguous byte range into L2 (UBLKPF.L2), issued by
// one lane, in chunks of 32 KiB
__device__ __forceinline__ void bulk_prefetch_l2(const void *p, size_t bytes) {
    // the bulk copy engine needs 16-byte aligned address and size
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
    bytes += reinterpret_cast<uintptr_t>(p) - a0;
    const char *c = reinterpret_cast<const char *>(a0);
    while (bytes > 0) {
        const unsigned n = bytes > 32768 ? 32768u : (unsigned)((bytes + 15) & ~(size_t)15);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(c), "r"(n) : "memory");
        c += n;
        bytes = bytes > n ? bytes - n : 0;
    }
}

// ---- TMA bulk copies (global -> shared, completion on an mbarrier) ----------
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(b))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, unsigned parity) {
    asm volatile(
        "{\n .reg .pred P1;\n LAB_WAIT:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        " @P1 bra DONE;\n bra LAB_WAIT;\n DONE:\n}" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
// Stage nq query vectors (leaf layout of a CPL = 8 plan: leaf_len doubles per
// leaf, 2-double pad) with one bulk copy per leaf, issued by warp 0; every
// thread returns once the bytes have landed.  `phase` = completions so far.
__device__ __forceinline__ void tma_stage_leaves(const PwPlan &pl, const double *H, int d, int nq, double *hs,
                                                 int hs_stride, unsigned long long *bar, unsigned phase) {
    const int L = pl.leaf_len, nl = pl.nleaf;
    if (threadIdx.x < 32) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of hs
        if (threadIdx.x == 0) mbar_expect_tx(bar, (unsigned)(nq * nl * L * 8));
        __syncwarp();
        for (int t = threadIdx.x; t < nq * nl; t += 32) {
            const int j = t / nl, leaf = t - j * nl;
            bulk_g2s(hs + (size_t)j * hs_stride + (size_t)leaf * (L + 2), H + (size_t)j * d + (size_t)leaf * L,
                     (unsigned)(L * 8), bar);
        }
    }
    mbar_wait(bar, phase & 1u);
}

__device__ __forceinline__ unsigned long long dkey(double v) {
    unsigned long long u = (unsigned long long)__double_as_longlong(v);
    return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
    unsigned long long u = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double((long long)u);
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(CSVD_FULL, v, o));
    return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(CSVD_FULL, v, o));
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(CSVD_FULL, v, o));
    return v;
}
__device__ __forceinline__ int warp_isum(int v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(CSVD_FULL, v, o);
    return v;
}

// (m, s) represents m + log(s); combine is associative up to rounding.
// Out of line: one copy of the f64 exp code instead of one per call site.
static __device__ __noinline__ void lse_combine(double &m, double &s, double m2, double s2) {
    if (m2 == -INFINITY) return;
    if (m == -INFINITY) {
        m = m2;
        s = s2;
        return;
    }
    if (m2 > m) {
        s = __dadd_rn(__dmul_rn(s, csvd_exp(__dsub_rn(m, m2))), s2);
        m = m2;
    } else {
        s = __dadd_rn(s, __dmul_rn(s2, csvd_exp(__dsub_rn(m2, m))));
    }
}

// exp(x) for x <= 0, inline and short (for log-sum-exp accumulations, where
// the reference's own numpy SIMD exp is only ulp-accurate too): x = k ln2 + r,
// |r| <= ln2/2, degree-13 Taylor polynomial in Horner form with explicit
// FMAs (relative error ~2 ulp), 2^k by exponent arithmetic.  Returns 0 below
// -708 (a term 1e-308 times the largest one of its sum).
__device__ __forceinline__ double exp_nonpos(double x) {
    if (!(x >= -708.0)) return 0.0;  // also -inf / NaN-free inputs -> 0
    const double k = rint(__dmul_rn(x, 1.4426950408889634));
    double r = __fma_rn(k, -6.93147180369123816490e-01, x);
    r = __fma_rn(k, -1.90821492927058770002e-10, r);
    double p = 1.0 / 6227020800.0;  // 1/13!
    p = __fma_rn(p, r, 1.0 / 479001600.0);
    p = __fma_rn(p, r, 1.0 / 39916800.0);
    p = __fma_rn(p, r, 1.0 / 3628800.0);
    p = __fma_rn(p, r, 1.0 / 362880.0);
    p = __fma_rn(p, r, 1.0 / 40320.0);
    p = __fma_rn(p, r, 1.0 / 5040.0);
    p = __fma_rn(p, r, 1.0 / 720.0);
    p = __fma_rn(p, r, 1.0 / 120.0);
    p = __fma_rn(p, r, 1.0 / 24.0);
    p = __fma_rn(p, r, 1.0 / 6.0);
    p = __fma_rn(p, r, 0.5);
    p = __fma_rn(p, r, 1.0);
    p = __fma_rn(p, r, 1.0);
    const long long ki = (long long)k;  // in [-1022, 0]
    return __longlong_as_double(__double_as_longlong(p) + (ki << 52));
}

// strict total order of the opening sequence: U descending, id ascending
// (np.lexsort((arange(C), -U)), decode.py:166)
__device__ __forceinline__ bool key_before(double ua, int ia, double ub, int ib) {
    return (ua > ub) || (ua == ub && ia < ib);
}

// Plain grid barrier (cooperative launch: all CTAs resident).
static __device__ __forceinline__ void grid_sync(const Dev &D) {
    __syncthreads();
    if (threadIdx.x == 0) {
        // acq_rel arrival (releases this CTA's writes, which the barrier above
        // made visible to this thread; cumulative), relaxed polling, one
        // acquire at the end: no SC fences
        unsigned gen, t;
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(D.bar + 1) : "memory");
        asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(t) : "l"(D.bar) : "memory");
        if (t == (unsigned)D.nblocks - 1u) {
            D.bar[0] = 0;
            st_release(D.bar + 1, gen + 1u);
        } else {
            unsigned long long spins = 0;
            unsigned v;
            while (true) {
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(D.bar + 1) : "memory");
                if (v != gen) break;
                __nanosleep(CSVD_SPIN_NS);
                if (++spins > (1ull << 24)) {  // ~1-2 s: flag and give up rather than hang
                    D.res->error = CSVD_ESTATE;
                    break;
                }
            }
            (void)ld_acquire(D.bar + 1);
        }
    }
    __syncthreads();
}

template <typename ET, int CPL, int Q>
__device__ __forceinline__ double row_logit(const Dev &D, int wrow, int pos, const double *hs, double *scratch,
                                            int lane) {
    const ET *row = reinterpret_cast<const ET *>(D.W) + (size_t)wrow * D.d;
    double dot = warp_dot_t<ET, CPL, Q>(row, hs, D.wplan, scratch, lane);
    return __dadd_rn(dot, __ldg(D.bias + pos));
}

// ---------------------------------------------------------------------------
// bounds phase (all CTAs)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double cone_bound(const Dev &D, int c, double dot, double qn) {
    // bounds._cone_raw (bounds.py:95-118)
    const double cn = D.cnorm[c], R = D.radii[c];
    double geom;
    if (cn > 0) {
        if (R == 0.0) {
            geom = dot;
        } else if (qn > 0) {
            double cphi = __ddiv_rn(dot, __dmul_rn(cn, qn));
            cphi = fmin(fmax(cphi, -1.0), 1.0);
            double a = __dsub_rn(acos(cphi), __dadd_rn(D.ang[c], 4e-12));
            double gamma = cos(fmax(0.0, a));
            geom = __dmul_rn(qn, fmax(__dmul_rn(D.maxn[c], gamma), __dmul_rn(D.minn[c], gamma)));
        } else {
            geom = 0.0;
        }
    } else {
        geom = __dmul_rn(R, qn);
    }
    return __dadd_rn(geom, D.maxb[c]);
}

// U from a centroid dot (batch lanes; off the single-query path, so out of line)
static __device__ __forceinline__ double bound_from_dot(const Dev &D, int c, double dot, double qn) {
    if (D.mode == CSVD_MODE_SPHERICAL) return cone_bound(D, c, dot, qn);
    return __dadd_rn(__dadd_rn(dot, __dmul_rn(D.radii[c], qn)), D.maxb[c]);
}

template <int BCPL, int BQ>
__device__ void bounds_phase(const Dev &D, const double *hs, double *scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ double s_qn;
    __shared__ double s_dot[WARPS][MAX_PER_WARP];
    const int stride = CTA_N * WARPS;
    if (warp == 0) {  // ||h|| = sqrt(sum(h*h)) in the pairwise order (_linalg.py:40-43)
        double ss;
        if constexpr (BCPL > 0) {
            ss = warp_dot_t<double, BCPL, BQ>(D.h, hs, D.bplan, scratch, lane);
        } else {
            struct HH {
                const double *hs;
                __device__ double operator()(int e) const { return __dmul_rn(hs[e], hs[e]); }
            } f{hs};
            ss = warp_dot_generic(f, D.bplan, scratch, lane);
        }
        if (lane == 0) s_qn = __dsqrt_rn(ss);
    }
    // a warp's first MAX_PER_WARP dots wait in shared memory for ||h||; any
    // further ones (small lane grids, large C) wait in D.dots (same thread)
    int j = 0;
    for (int c = warp * CTA_N + CTA_ID; c < D.C; c += stride, ++j) {
        double dot = warp_dot_t<double, BCPL, BQ>(D.cent + (size_t)c * D.bd, hs, D.bplan, scratch, lane);
        if (lane == 0) {
            if (j < MAX_PER_WARP) s_dot[warp][j] = dot;
            else D.dots[c] = dot;
        }
    }
    __syncthreads();
    const double qn = s_qn;
    if (lane == 0) {
        j = 0;
        for (int c = warp * CTA_N + CTA_ID; c < D.C; c += stride, ++j) {
            const double dot = j < MAX_PER_WARP ? s_dot[warp][j] : D.dots[c];
            double u;
            if (D.mode == CSVD_MODE_SPHERICAL)
                u = cone_bound(D, c, dot, qn);
            else if (D.mode == CSVD_MODE_BIAS_AUGMENTED)
                u = __dadd_rn(dot, __dmul_rn(D.radii[c], qn));
            else
                u = __dadd_rn(__dadd_rn(dot, __dmul_rn(D.radii[c], qn)), D.maxb[c]);
            D.Uraw[c] = u;  // the order phase adds the slack
            D.dots[c] = dot;
        }
    }
    if (CTA_ID == 0 && threadIdx.x == 0) D.res->query_norm = qn;
}

// ---------------------------------------------------------------------------
// order phase (every CTA, redundantly, in shared memory): the opening order
// np.lexsort((arange(C), -U)) (decode.py:166) by a block bitonic sort, the
// prefix token counts in that order, and log R-hat after every prefix
// (certify.py:114-119) by a block suffix scan.  No global round trip and no
// grid barrier: every CTA ends the phase holding the full ordering.
// ---------------------------------------------------------------------------
struct Ord {  // the full ordering, per CTA
    int *order, *cum;      // [C] cluster at each opening position, [C+1] tokens before it
    double *Uo, *lrh;      // [C] bound at each position, [C+1] log R-hat after p opens
    unsigned long long *keys;  // [Cp] sort keys (then x = log|c| + U by position)
    double *Us;            // [C] U + slack by cluster id (then exp(x - xmax) by position)
};

// shared-memory footprint of the ordering region, in doubles (host + device)
__host__ __device__ inline int ord_doubles(int C, int Cp) {
    return Cp + C + C + (C + 1) + (Cp + (C + 1) + 2) / 2 + 1;
}

__device__ __forceinline__ void ord_bind(const Dev &D, double *ws, Ord &o) {
    const int C = D.C, Cp = D.Cp;
    o.keys = reinterpret_cast<unsigned long long *>(ws);
    o.Us = ws + Cp;
    o.Uo = o.Us + C;
    o.lrh = o.Uo + C;
    o.order = reinterpret_cast<int *>(o.lrh + C + 1);
    o.cum = o.order + Cp;
}

__device__ __forceinline__ double block_max(double v, double *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    double m = red[0];
#pragma unroll
    for (int w = 1; w < WARPS; ++w) m = fmax(m, red[w]);
    return m;
}

// Stage U + slack (bounds.py:58-64, which needs max |U| first) by cluster id
// in shared memory; CTA 0 publishes it for cluster_bounds (bounds.py:178-184).
// Returns false (in every CTA) if a bound is non-finite.
static __device__ __forceinline__ bool stage_bounds(const Dev &D, const Ord &o, double qn_given,
                                                    double *eta_out = nullptr) {
    const int tid = threadIdx.x;
    const int C = D.C;
    const csvd_config &cfg = *D.cfg;
    __shared__ double s_red[WARPS];
    double *__restrict__ Us = o.Us;
    // by cluster id, for the head path: x = log|c| (+ U below) in the keys
    // region, the best-logit estimate in Uo, |c| in cum (all loads in flight
    // together; order_full rebuilds these regions from global memory)
    double *__restrict__ xs = reinterpret_cast<double *>(o.keys);
    double *__restrict__ es = o.Uo;
    int *__restrict__ zs = o.cum;
    const bool aug = D.mode == CSVD_MODE_BIAS_AUGMENTED;
    double amax = 1.0;
    auto put = [&](int c, double u, double dt) {
        const double mb = __ldg(D.meanb + c);
        const double lz = __ldg(D.logsz + c);
        const int sz = __ldg(D.sizes + c);
        Us[c] = u;
        es[c] = aug ? dt : __dadd_rn(dt, mb);  // init_state's estimate of the best logit
        xs[c] = lz;
        zs[c] = sz;
        amax = fmax(amax, fabs(u));
    };
    if (!D.pre_bounds) {
#pragma unroll 4
        for (int c = tid; c < C; c += THREADS) put(c, __ldcg(D.Uraw + c), __ldcg(D.dots + c));
    } else if (D.mode != CSVD_MODE_SPHERICAL) {
        // batched bounds: U from the given dots (bounds.py:79-83) and this
        // lane's ||h||; four clusters' loads in flight per thread (a lane of
        // one CTA walks every cluster: C / 256 dependent L2 round trips otherwise)
#pragma unroll 1
        for (int c0 = tid; c0 < C; c0 += 4 * THREADS) {
            double dt[4], rr[4], mb[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int c = min(c0 + j * THREADS, C - 1);
                dt[j] = __ldcg(D.dots + c);
                rr[j] = __ldg(D.radii + c);
                mb[j] = __ldg(D.maxb + c);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (c0 + j * THREADS < C)
                    put(c0 + j * THREADS, __dadd_rn(__dadd_rn(dt[j], __dmul_rn(rr[j], qn_given)), mb[j]), dt[j]);
        }
    } else {  // spherical (bounds.py:95-118)
#pragma unroll 1
        for (int c = tid; c < C; c += THREADS) {
            const double dt = __ldcg(D.dots + c);
            put(c, cone_bound(D, c, dt, qn_given), dt);
        }
    }
    double eta = 0.0;
    if (cfg.slack_f32) {
        amax = block_max(amax, s_red);
        eta = __dmul_rn(__dmul_rn(4.0, 1.1920928955078125e-07), amax);
    }
    int bad = 0;
    for (int c = tid; c < C; c += THREADS) {
        const double u = __dadd_rn(Us[c], eta);
        bad |= !isfinite(u);  // BoundVector.__post_init__ (bounds.py:53-55)
        Us[c] = u;
        xs[c] = __dadd_rn(xs[c], u);  // certify.py:119 np.log(sizes) + U
        if (CTA_ID == 0) D.U[c] = u;
    }
    if (eta_out && tid == 0) *eta_out = eta;
    bad = __syncthreads_or(bad);
    if (CTA_ID == 0 && tid == 0) D.res->slack = eta;
    return !bad;
}

__device__ __forceinline__ unsigned long long okey(double u) {  // ascending key == descending U
    if (u == 0.0) u = 0.0;  // -0.0 ties +0.0, as in the reference's comparison sort
    return ~dkey(u);
}
__device__ __forceinline__ bool okey_before(unsigned long long ka, int ia, unsigned long long kb, int ib) {
    return ka < kb || (ka == kb && ia < ib);
}

// The head of the opening order (fast path; every CTA): the clusters whose
// bound is at least the wave estimate of the best logit (the first-wave rule
// of csvd_plan_wave with a top-k target), always including the top cluster.
// Every other cluster has a smaller bound, so the head is exactly the prefix
// [0, n) of np.lexsort((arange(C), -U)) (decode.py:166); it is sorted by one
// warp in registers.  Also fills order/Uo/cum/lrh at position n (the first
// cluster after the head: the best remaining bound is all a top-k test at
// p = n needs).  Returns n, or 0 when the head does not apply (more than 64
// clusters, or a residual sum too small for the direct form): then the full
// sort runs instead.
// lrh = false (the head step's row CTAs): no log R-hat (and no underflow test,
// fail_out = 0): only the certifying CTA reads them.  fail_out: report the
// residual-underflow case there instead of returning 0.
static __device__ __forceinline__ int order_head(const Dev &D, const Ord &o, double &est_out, bool lrh = true,
                                                 int *fail_out = nullptr) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int C = D.C;
    const double *__restrict__ Us = o.Us;
    const double *__restrict__ xs = reinterpret_cast<const double *>(o.keys);  // x by cluster id
    __shared__ unsigned long long s_k[WARPS];
    __shared__ int s_i[WARPS], s_n, s_head[64];
    __shared__ double s_x[WARPS];
    __shared__ int s_hz[64], s_hc[64];       // head by position: size, cluster
    __shared__ double s_he[64], s_hu[64];    // head by position: exp(x - xmax), U
    // --- top cluster c0: argmin of (okey(U), id); every thread folds the warp results
    unsigned long long bk = ~0ull;
    int bi = 0x7fffffff;
    #pragma unroll 1
    for (int c = tid; c < C; c += THREADS) {
        const unsigned long long k = okey(Us[c]);
        if (okey_before(k, c, bk, bi)) {
            bk = k;
            bi = c;
        }
    }
#pragma unroll 1
    for (int off = 16; off; off >>= 1) {
        const unsigned long long k2 = __shfl_xor_sync(CSVD_FULL, bk, off);
        const int i2 = __shfl_xor_sync(CSVD_FULL, bi, off);
        if (okey_before(k2, i2, bk, bi)) {
            bk = k2;
            bi = i2;
        }
    }
    if (lane == 0) {
        s_k[warp] = bk;
        s_i[warp] = bi;
    }
    if (tid == 0) s_n = 0;
    __syncthreads();
#pragma unroll 1
    for (int w = 0; w < WARPS; ++w)
        if (okey_before(s_k[w], s_i[w], bk, bi)) {
            bk = s_k[w];
            bi = s_i[w];
        }
    const int c0 = bi;
    const double est = o.Uo[c0];  // the best-logit estimate by id (stage_bounds)
    if (DBG_HERE(D) && tid == 0) DBG_TS(D, 33);
    if (tid == 0) est_out = est;  // init_state's wave estimate, already known here
    // --- membership, x = log|c| + U (certify.py:119), best non-head cluster
    double xm = -INFINITY;
    bk = ~0ull;
    bi = 0x7fffffff;
    #pragma unroll 1
    for (int c = tid; c < C; c += THREADS) {
        const double u = Us[c];
        xm = fmax(xm, xs[c]);
        if (u >= est || c == c0) {
            const int slot = atomicAdd(&s_n, 1);
            if (slot < 64) s_head[slot] = c;
        } else {
            const unsigned long long k = okey(u);
            if (okey_before(k, c, bk, bi)) {
                bk = k;
                bi = c;
            }
        }
    }
    xm = warp_max(xm);
#pragma unroll 1
    for (int off = 16; off; off >>= 1) {
        const unsigned long long k2 = __shfl_xor_sync(CSVD_FULL, bk, off);
        const int i2 = __shfl_xor_sync(CSVD_FULL, bi, off);
        if (okey_before(k2, i2, bk, bi)) {
            bk = k2;
            bi = i2;
        }
    }
    __syncthreads();  // s_k / s_i reuse; s_n final
    if (lane == 0) {
        s_k[warp] = bk;
        s_i[warp] = bi;
        s_x[warp] = xm;
    }
    const int n = s_n;
    __syncthreads();
    if (DBG_HERE(D) && tid == 0) DBG_TS(D, 34);
    if (n > 64) return 0;
    double xmax = s_x[0];
#pragma unroll 1
    for (int w = 1; w < WARPS; ++w) xmax = fmax(xmax, s_x[w]);
    // --- residual mass of everything outside the head; the head's rank by
    // (key, id) among themselves (thread group of 4 per head element)
    double rest = 0.0;
    #pragma unroll 1
    for (int c = lrh ? tid : C; c < C; c += THREADS)
        if (!(Us[c] >= est || c == c0)) rest = __dadd_rn(rest, exp_nonpos(__dsub_rn(xs[c], xmax)));
    {
        const int e = tid >> 2, part = tid & 3;
        int rank = 0;
        unsigned long long ke = 0;
        int ie = 0;
        if (e < n) {
            ie = s_head[e];
            ke = okey(Us[ie]);
            for (int j = part; j < n; j += 4) {
                const int ij = s_head[j];
                rank += okey_before(okey(Us[ij]), ij, ke, ie) ? 1 : 0;
            }
        }
        rank += __shfl_xor_sync(CSVD_FULL, rank, 1);
        rank += __shfl_xor_sync(CSVD_FULL, rank, 2);
        if (e < n && part == 0) {
            s_hc[rank] = ie;
            s_hu[rank] = Us[ie];
            s_hz[rank] = o.cum[ie];  // |c| by id (stage_bounds)
            s_he[rank] = lrh ? exp_nonpos(__dsub_rn(xs[ie], xmax)) : 0.0;
        }
    }
    rest = warp_sum(rest);
    __syncthreads();  // s_x reuse; s_h* complete; every read of the by-id staging is done
    if (lane == 0) s_x[warp] = rest;
    __syncthreads();
    if (DBG_HERE(D) && tid == 0) DBG_TS(D, 35);
    double S_rest = 0.0;
#pragma unroll 1
    for (int w = 0; w < WARPS; ++w) S_rest = __dadd_rn(S_rest, s_x[w]);
    __shared__ int s_fail;
    if (warp == 0) {
        int cn = 0x7fffffff;
        unsigned long long kn = ~0ull;
#pragma unroll 1
        for (int w = 0; w < WARPS; ++w)
            if (okey_before(s_k[w], s_i[w], kn, cn)) {
                kn = s_k[w];
                cn = s_i[w];
            }
        // positions lane (a) and lane + 32 (b): order, Uo, cum, lrh
        const int sa = lane < n ? s_hz[lane] : 0, sb = lane + 32 < n ? s_hz[lane + 32] : 0;
        const double ea = lane < n ? s_he[lane] : 0.0, eb = lane + 32 < n ? s_he[lane + 32] : 0.0;
        int ca = sa, cb = sb;  // inclusive prefix sums
        double ra = ea, rb = eb;  // inclusive suffix sums
#pragma unroll 1
        for (int off = 1; off < 32; off <<= 1) {
            const int ta = __shfl_up_sync(CSVD_FULL, ca, off), tb = __shfl_up_sync(CSVD_FULL, cb, off);
            const double ua = __shfl_down_sync(CSVD_FULL, ra, off), ub = __shfl_down_sync(CSVD_FULL, rb, off);
            if (lane >= off) {
                ca += ta;
                cb += tb;
            }
            if (lane + off < 32) {
                ra = __dadd_rn(ra, ua);
                rb = __dadd_rn(rb, ub);
            }
        }
        const int tot_a = __shfl_sync(CSVD_FULL, ca, 31);
        const double tot_b = __shfl_sync(CSVD_FULL, rb, 0);
        const double ta = __dadd_rn(S_rest, __dadd_rn(ra, tot_b)), tb = __dadd_rn(S_rest, rb);
        int fail = 0;
        if (lane < n) {
            o.order[lane] = s_hc[lane];
            o.Uo[lane] = s_hu[lane];
            o.cum[lane] = ca - sa;
            fail |= !(ta > 1e-280);
        }
        if (lane + 32 < n) {
            o.order[lane + 32] = s_hc[lane + 32];
            o.Uo[lane + 32] = s_hu[lane + 32];
            o.cum[lane + 32] = tot_a + cb - sb;
            fail |= !(tb > 1e-280);
        }
        const int cbt = __shfl_sync(CSVD_FULL, cb, 31);
        if (lane == 0) {
            o.cum[n] = tot_a + cbt;
            if (n < C) {
                o.order[n] = cn;
                o.Uo[n] = Us[cn];
                fail |= !(S_rest > 1e-280);
            }
        }
        if (lrh) {  // log R-hat after every head prefix (two logs per lane, independent)
            const double la = lane < n ? csvd_log(ta) : 0.0, lb = lane + 32 < n ? csvd_log(tb) : 0.0;
            if (lane < n) o.lrh[lane] = __dadd_rn(xmax, la);
            if (lane + 32 < n) o.lrh[lane + 32] = __dadd_rn(xmax, lb);
            if (lane == 0) o.lrh[n] = n < C ? __dadd_rn(xmax, csvd_log(S_rest)) : -INFINITY;
        } else {
            fail = 0;
        }
        fail = __any_sync(CSVD_FULL, fail);
        if (lane == 0) s_fail = fail;
    }
    __syncthreads();
    if (fail_out) {
        *fail_out = s_fail;
        return n;
    }
    return s_fail ? 0 : n;
}

// The full opening order (every CTA): bitonic sort of all C (key, id) pairs,
// prefix token counts and log R-hat after every prefix (block scans).
// Consumes Us (reused as exp(x - xmax) by position).
static __device__ __forceinline__ void order_full(const Dev &D, const Ord &o) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int C = D.C, Cp = D.Cp;
    __shared__ double s_red[WARPS];
    __shared__ int s_ired[WARPS];
    for (int c = tid; c < Cp; c += THREADS) {
        o.keys[c] = c < C ? okey(o.Us[c]) : ~0ull;
        o.order[c] = c < C ? c : 0x7fffffff;
    }
    __syncthreads();
    // --- bitonic sort of (key, id) ascending: (-U, id) order.  The arrays
    // are held in registers as __restrict__ shared pointers: through the Ord
    // reference every store would force a reload of the pointers from the stack.
    {
        unsigned long long *__restrict__ keys = o.keys;
        int *__restrict__ ids = o.order;
        const int half = Cp >> 1;
#pragma unroll 1
        for (int kk = 2; kk <= Cp; kk <<= 1) {
#pragma unroll 1
            for (int j = kk >> 1; j > 0; j >>= 1) {
                for (int i = tid; i < half; i += THREADS) {
                    const int lo = ((i & ~(j - 1)) << 1) | (i & (j - 1)), hi = lo + j;
                    const unsigned long long ka = keys[lo], kb = keys[hi];
                    const int ia = ids[lo], ib = ids[hi];
                    const bool a_after = (ka > kb) || (ka == kb && ia > ib);
                    if (a_after == ((lo & kk) == 0)) {
                        keys[lo] = kb;
                        keys[hi] = ka;
                        ids[lo] = ib;
                        ids[hi] = ia;
                    }
                }
                __syncthreads();
            }
        }
    }
    // --- by position: Uo, x = log|c| + U (certify.py:119), sizes -> cum
    const int seg = (C + THREADS - 1) / THREADS;
    const int b0 = min(C, tid * seg), b1 = min(C, b0 + seg);
    double *x = reinterpret_cast<double *>(o.keys);
    double xm = -INFINITY;
    int tsum = 0;
    for (int p = b0; p < b1; ++p) {
        const int c = o.order[p];
        const double u = o.Us[c];
        o.Uo[p] = u;
        const double xv = __dadd_rn(__ldg(D.logsz + c), u);
        x[p] = xv;
        xm = fmax(xm, xv);
        tsum += __ldg(D.sizes + c);
    }
    // exclusive scan of sizes over positions (segments are thread-contiguous)
    int incl = tsum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const int t = __shfl_up_sync(CSVD_FULL, incl, off);
        if (lane >= off) incl += t;
    }
    xm = warp_max(xm);
    if (lane == 31) s_ired[warp] = incl;
    if (lane == 0) s_red[warp] = xm;
    __syncthreads();
    int run = incl - tsum;
    double xmax = -INFINITY;
    for (int w = 0; w < WARPS; ++w) {
        if (w < warp) run += s_ired[w];
        xmax = fmax(xmax, s_red[w]);
    }
    double tail = 0.0;  // this thread's e-sum (suffix scan below)
    for (int p = b0; p < b1; ++p) {
        o.cum[p] = run;
        run += __ldg(D.sizes + o.order[p]);
        const double e = exp_nonpos(__dsub_rn(x[p], xmax));
        o.Us[p] = e;  // Us by id is dead: reuse as e by position
    }
    for (int p = b1 - 1; p >= b0; --p) tail = __dadd_rn(tail, o.Us[p]);
    // suffix scan: sum of e over positions >= p
    double sinc = tail;  // lanes >= lane
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double t = __shfl_down_sync(CSVD_FULL, sinc, off);
        if (lane + off < 32) sinc = __dadd_rn(sinc, t);
    }
    __syncthreads();  // s_red reuse
    if (lane == 0) s_red[warp] = sinc;
    __syncthreads();
    double after = 0.0;  // e-sum of the threads after this one: lanes above + warps above
    {
        double up = __shfl_down_sync(CSVD_FULL, sinc, 1);
        if (lane < 31) after = up;
    }
    for (int w = WARPS - 1; w > warp; --w) after = __dadd_rn(after, s_red[w]);
    int need_rescale = 0;
    double acc = after;
    for (int p = b1 - 1; p >= b0; --p) {
        acc = __dadd_rn(acc, o.Us[p]);
        if (acc > 1e-280) {
            o.lrh[p] = __dadd_rn(xmax, csvd_log(acc));
        } else {
            need_rescale = 1;
            o.lrh[p] = -INFINITY;
        }
    }
    if (tid == 0) {
        o.cum[C] = D.V;
        o.lrh[C] = -INFINITY;
    }
    need_rescale = __syncthreads_or(need_rescale);
    if (need_rescale) {
        // far below the global max: rescale each deep suffix by its own max (rare)
        for (int p = warp; p < C; p += WARPS) {
            if (o.lrh[p] != -INFINITY) continue;
            double tmax = -INFINITY;
            for (int i = p + lane; i < C; i += 32) tmax = fmax(tmax, x[i]);
            tmax = warp_max(tmax);
            double t2 = 0.0;
            for (int i = p + lane; i < C; i += 32) t2 = __dadd_rn(t2, csvd_exp(__dsub_rn(x[i], tmax)));
            t2 = warp_sum(t2);
            if (lane == 0) o.lrh[p] = __dadd_rn(tmax, csvd_log(t2));
        }
        __syncthreads();
    }
}

// cluster summary (warp): top-min(k,n) values desc, LSE, min, max of the
// cluster's logits S_logits[lo, hi)
#define SUM_E 8  // clusters of up to 32 * SUM_E rows are summarised from registers
// logits of one cluster into registers (-inf padded); only for n <= 32 * SUM_E
__device__ __forceinline__ void summary_load(const Dev &D, int lo, int hi, double (&reg)[SUM_E], int lane) {
    const int n = hi - lo;
#pragma unroll
    for (int e = 0; e < SUM_E; ++e) {
        const int i = lane + 32 * e;
        reg[e] = (i < n && n <= 32 * SUM_E) ? __ldcg(D.S_logits + lo + i) : -INFINITY;
    }
}

// reg: the cluster's logits from summary_load (ignored when n > 32 * SUM_E)
static __device__ __forceinline__ void cluster_summary(const Dev &D, int lo, int hi, int k, double *topk, double *lse_o,
                                                       double *min_o, double *max_o, double (&reg)[SUM_E],
                                                       int lane) {
    const int n = hi - lo;
    const double *v = D.S_logits + lo;
    const int kk = n < k ? n : k;
    constexpr int E = SUM_E;
    const bool in_regs = n <= 32 * E;
    double mx = -INFINITY, mn = INFINITY;
    if (in_regs) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            if (lane + 32 * e < n) {
                mx = fmax(mx, reg[e]);
                mn = fmin(mn, reg[e]);
            }
        }
    } else {
        for (int i = lane; i < n; i += 32) {
            const double x = __ldcg(v + i);
            mx = fmax(mx, x);
            mn = fmin(mn, x);
        }
    }
    if (DBG_HERE(D) && threadIdx.x == 0) DBG_TS(D, 48);
    mx = warp_max(mx);
    mn = warp_min(mn);
    if (DBG_HERE(D) && threadIdx.x == 0) DBG_TS(D, 49);
    double s = 0.0;
    if (in_regs) {
#pragma unroll
        for (int e = 0; e < E; ++e)
            if (lane + 32 * e < n) s = __dadd_rn(s, csvd_exp(__dsub_rn(reg[e], mx)));
    } else {
        for (int i = lane; i < n; i += 32) s = __dadd_rn(s, csvd_exp(__dsub_rn(__ldcg(v + i), mx)));
    }
    s = warp_sum(s);
    if (DBG_HERE(D) && threadIdx.x == 0) DBG_TS(D, 50);
    if (in_regs) {
        // top-kk values (only the values matter: the list holds no ids).
        // Each lane sorts its 8 values (Batcher network), then kk rounds of a
        // warp max over the lane heads with REDUX on the order-preserving
        // 64-bit keys; the winning lane pops its head.
#define CSVD_CAS(a, b)                  \
    {                                   \
        const double hi_ = fmax(reg[a], reg[b]); \
        reg[b] = fmin(reg[a], reg[b]);  \
        reg[a] = hi_;                   \
    }
        CSVD_CAS(0, 1) CSVD_CAS(2, 3) CSVD_CAS(4, 5) CSVD_CAS(6, 7)
        CSVD_CAS(0, 2) CSVD_CAS(1, 3) CSVD_CAS(4, 6) CSVD_CAS(5, 7)
        CSVD_CAS(1, 2) CSVD_CAS(5, 6) CSVD_CAS(0, 4) CSVD_CAS(3, 7)
        CSVD_CAS(1, 5) CSVD_CAS(2, 6)
        CSVD_CAS(1, 4) CSVD_CAS(3, 6)
        CSVD_CAS(2, 4) CSVD_CAS(3, 5)
        CSVD_CAS(3, 4)
#undef CSVD_CAS
    if (DBG_HERE(D) && threadIdx.x == 0) DBG_TS(D, 51);
#pragma unroll 1
        for (int j = 0; j < kk; ++j) {
            const unsigned long long key = dkey(reg[0]);
            const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
            const unsigned mh = __reduce_max_sync(CSVD_FULL, hi);
            const unsigned ml = __reduce_max_sync(CSVD_FULL, hi == mh ? lo : 0u);
            const unsigned win = __ballot_sync(CSVD_FULL, hi == mh && lo == ml);
            if (lane == 0) topk[j] = dkey_inv(((unsigned long long)mh << 32) | ml);
            if (lane == __ffs(win) - 1) {
#pragma unroll
                for (int e = 0; e < E - 1; ++e) reg[e] = reg[e + 1];
                reg[E - 1] = -INFINITY;
            }
        }
    } else {
        // iterative selection in (value desc, index asc) order (clusters > 256 rows)
        double pv = INFINITY;
        int pi = -1;
#pragma unroll 1
        for (int j = 0; j < kk; ++j) {
            double bv = -INFINITY;
            int bi = 0x7fffffff;
            for (int i = lane; i < n; i += 32) {
                const double x = __ldcg(v + i);
                const bool after = (x < pv) || (x == pv && i > pi);
                if (after && (x > bv || (x == bv && i < bi))) {
                    bv = x;
                    bi = i;
                }
            }
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double ov = __shfl_xor_sync(CSVD_FULL, bv, o);
                const int oi = __shfl_xor_sync(CSVD_FULL, bi, o);
                if (ov > bv || (ov == bv && oi < bi)) {
                    bv = ov;
                    bi = oi;
                }
            }
            if (lane == 0) topk[j] = bv;
            pv = bv;
            pi = bi;
        }
    }
    if (lane == 0) {
        *lse_o = (mx == -INFINITY) ? -INFINITY : __dadd_rn(mx, csvd_log(s));
        *min_o = mn;
        *max_o = mx;
    }
}

// running top-k list for k <= 32: lane l holds the l-th largest (-inf pad)
__device__ __forceinline__ double reg_merge(double v, double nv /* lane l: l-th largest of new */, int lane) {
    double m = fmax(v, __shfl_sync(CSVD_FULL, nv, 31 - lane));  // bitonic: top-32 of the union
#pragma unroll
    for (int s = 16; s; s >>= 1) {
        const double o = __shfl_xor_sync(CSVD_FULL, m, s);
        m = ((lane & s) == 0) ? fmax(m, o) : fmin(m, o);
    }
    return m;
}

// smem merge-path merge of two descending lists (k > 32 path)
static __device__ int merge_lists(const double *A, int ka, const double *B, int kb, int k, double *out, int lane) {
    for (int i = lane; i < ka; i += 32) {
        const double a = A[i];
        int lo = 0, hi = kb;  // count B > a
        while (lo < hi) {
            const int m = (lo + hi) >> 1;
            if (B[m] > a) lo = m + 1; else hi = m;
        }
        if (i + lo < k) out[i + lo] = a;
    }
    for (int j = lane; j < kb; j += 32) {
        const double b = B[j];
        int lo = 0, hi = ka;  // count A >= b
        while (lo < hi) {
            const int m = (lo + hi) >> 1;
            if (A[m] >= b) lo = m + 1; else hi = m;
        }
        if (j + lo < k) out[j + lo] = b;
    }
    __syncwarp();
    const int n = ka + kb;
    return n < k ? n : k;
}

// running top-16 list (k <= 16): lane l < 16 holds the l-th largest; lanes >= 16 hold -inf
__device__ __forceinline__ double reg_merge16(double v, double nv /* lane l: l-th largest of new */, int lane) {
    double m = fmax(v, __shfl_sync(CSVD_FULL, nv, 15 - (lane & 15)));  // bitonic: top-16 of the union
#pragma unroll
    for (int s = 8; s; s >>= 1) {
        const double o = __shfl_xor_sync(CSVD_FULL, m, s);
        m = ((lane & s) == 0) ? fmax(m, o) : fmin(m, o);
    }
    return lane < 16 ? m : -INFINITY;
}

// logsumexp over S_logits[0, n) with known max (64-merge recompute, certify.py:79-83)
static __device__ double warp_lse_all(const double *vals, int n, double vmax, int lane) {
    if (n == 0 || vmax == -INFINITY) return -INFINITY;
    if (vmax == INFINITY) return INFINITY;
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s = __dadd_rn(s, csvd_exp(__dsub_rn(__ldcg(vals + i), vmax)));
    s = warp_sum(s);
    return __dadd_rn(vmax, csvd_log(s));
}

// logsumexp over S_logits[0, n) with known max, by the whole CTA (the 64-merge
// recompute of a chunk, certify.py:79-83: one warp would take ~n / 32 serial exps)
static __device__ __noinline__ double block_lse_all(const double *vals, int n, double vmax, double *red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double s = 0.0;
    if (n > 0 && vmax != -INFINITY && vmax != INFINITY)
        for (int i = threadIdx.x; i < n; i += THREADS) s = __dadd_rn(s, csvd_exp(__dsub_rn(__ldcg(vals + i), vmax)));
    s = warp_sum(s);
    __syncthreads();
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (n == 0 || vmax == -INFINITY) return -INFINITY;
    if (vmax == INFINITY) return INFINITY;
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) t = __dadd_rn(t, red[w]);
    return __dadd_rn(vmax, csvd_log(t));
}

struct ScanShared {
    ScanState st;
    csvd_result res;
    int kcount;
    int head_n;  // > 0: the ordering is valid only for positions [0, head_n] (fast path)
    int flags;   // CSVD_FLAG_* over the prefixes tested so far
};

// |x - thr| < 1e-12 * thr: an ulp-level tie of a certification threshold
__device__ __forceinline__ bool near_tie(double x, double thr) {
    return fabs(__dsub_rn(x, thr)) < __dmul_rn(1e-12, thr);
}

// warp 0: per-prefix values of the chunk [q0, q1) from its summaries, then the
// state machine (scan.cuh).  reg_list: the k <= 32 running list (lane-held);
// la / lb: the k > 32 running list buffers (the live list stays in la).
static __device__ __forceinline__ void scan_chunk(const Dev &D, const Ord &o, ScanShared &ss, int q0, int q1,
                                        const double *c_topk, const double *c_lse, const double *c_min,
                                        const double *c_max, double *c_vals, double *la0, double *lb0,
                                        double &reg_list, int lane, double full_pre = NAN) {
    const ScanState st0 = ss.st;
    const int k = D.cfg->k;
    const bool small_k = k <= 32;
    const int q = q0 + lane;
    const bool act = q < q1;
    const double lse_q = act ? c_lse[lane] : -INFINITY;
    const double lr = act ? o.lrh[q + 1] : -INFINITY;
    const int cnt_q = act ? o.cum[q + 1] : 0;
    // min / max prefix (inclusive over lanes) with the carried values
    double pmn = act ? c_min[lane] : INFINITY, pmx = act ? c_max[lane] : -INFINITY;
#pragma unroll
    for (int s = 1; s < 32; s <<= 1) {
        const double a = __shfl_up_sync(CSVD_FULL, pmn, s), b = __shfl_up_sync(CSVD_FULL, pmx, s);
        if (lane >= s) {
            pmn = fmin(pmn, a);
            pmx = fmax(pmx, b);
        }
    }
    if (st0.p > 0) {
        pmn = fmin(pmn, st0.smin);
        pmx = fmax(pmx, st0.smax);
    }
    if (DBG_HERE(D) && lane == 0) DBG_TS(D, 40);
    // streaming log Z_S (certify.py:83 logaddexp chain) as a prefix sum of
    // exp(lse - M) over the chunk, M the chunk's largest term (incl. the carry)
    double lz;
    {
        const double M = fmax(warp_max(act ? lse_q : -INFINITY), st0.log_z);
        if (M == -INFINITY) {
            lz = -INFINITY;
        } else {
            double t = (act && lse_q != -INFINITY) ? exp_nonpos(__dsub_rn(lse_q, M)) : 0.0;
#pragma unroll
            for (int s = 1; s < 32; s <<= 1) {
                const double u = __shfl_up_sync(CSVD_FULL, t, s);
                if (lane >= s) t = __dadd_rn(t, u);
            }
            if (st0.log_z != -INFINITY) t = __dadd_rn(t, exp_nonpos(__dsub_rn(st0.log_z, M)));
            lz = t > 0.0 ? __dadd_rn(M, csvd_log(t)) : -INFINITY;
        }
    }
    if (DBG_HERE(D) && lane == 0) DBG_TS(D, 41);
    // the reference recomputes log Z_S over all of S when the merge count p % 64 == 0
    const int rlane = (q0 / 64) * 64 + 63 - q0;
    if (rlane < q1 - q0) {
        const double vmax = __shfl_sync(CSVD_FULL, pmx, rlane);
        const int ncum = __shfl_sync(CSVD_FULL, cnt_q, rlane);
        // the recompute over all of S: precomputed by the whole CTA when given
        const double full = isnan(full_pre) ? warp_lse_all(D.S_logits, ncum, vmax, lane) : full_pre;
        double rm = (lane > rlane && act) ? lse_q : -INFINITY, rsv = (lane > rlane && act) ? 1.0 : 0.0;
#pragma unroll 1
        for (int s = 1; s < 32; s <<= 1) {
            const double m2 = __shfl_up_sync(CSVD_FULL, rm, s), s2 = __shfl_up_sync(CSVD_FULL, rsv, s);
            if (lane >= s) {
                double mm = m2, sv = s2;
                lse_combine(mm, sv, rm, rsv);
                rm = mm;
                rsv = sv;
            }
        }
        double mm = full, sv = (full == -INFINITY) ? 0.0 : 1.0;
        lse_combine(mm, sv, rm, rsv);
        if (lane == rlane) lz = full;
        if (lane > rlane) lz = (mm == -INFINITY) ? -INFINITY : __dadd_rn(mm, csvd_log(sv));
    }
    if (DBG_HERE(D) && lane == 0) DBG_TS(D, 42);
    // k-th largest after each merge (exact)
    double my_kth = -INFINITY;
    int kc = ss.kcount;
    if (k <= 16) {
        // sequential merges of 16-entry lists (lane l < 16 holds the l-th largest).
        // A cluster whose largest logit does not exceed the current k-th value
        // cannot change the top-k values (ties add equal values below the cut):
        // its merge is skipped.
        double kv = kc >= k ? __shfl_sync(CSVD_FULL, reg_list, k - 1) : -INFINITY;
#pragma unroll 1
        for (int t = 0; t < q1 - q0; ++t) {
            const int size = o.cum[q0 + t + 1] - o.cum[q0 + t];
            const int kn = size < k ? size : k;
            if (!(kc >= k && c_max[t] <= kv)) {
                const double nv = lane < kn ? c_topk[t * k + lane] : -INFINITY;
                reg_list = reg_merge16(reg_list, nv, lane);
                kc = min(k, kc + kn);
                kv = kc >= k ? __shfl_sync(CSVD_FULL, reg_list, k - 1) : -INFINITY;
            }
            if (lane == t) my_kth = kv;
        }
    } else {  // k > 16
        double *la = la0, *lb = lb0;
#pragma unroll 1
        for (int t = 0; t < q1 - q0; ++t) {
            const int size = o.cum[q0 + t + 1] - o.cum[q0 + t];
            const int kn = size < k ? size : k;
            if (small_k) {
                const double nv = lane < kn ? c_topk[t * k + lane] : -INFINITY;
                reg_list = reg_merge(reg_list, nv, lane);
                kc = min(k, kc + kn);
                const double kv = __shfl_sync(CSVD_FULL, reg_list, k - 1);
                if (lane == t) my_kth = kc >= k ? kv : -INFINITY;
            } else {
                kc = merge_lists(la, kc, c_topk + t * k, kn, k, lb, lane);
                double *tmp = la;
                la = lb;
                lb = tmp;
                const double kv = kc >= k ? la[k - 1] : -INFINITY;
                if (lane == t) my_kth = kv;
                __syncwarp();
            }
        }
        if (!small_k && la != la0) {  // keep the live list in la0
            for (int t = lane; t < kc; t += 32) la0[t] = la[t];
            __syncwarp();
        }
    }
    if (DBG_HERE(D) && lane == 0) DBG_TS(D, 43);
    double *c_lz = c_vals, *c_kth = c_vals + CHUNK, *c_mn = c_vals + 2 * CHUNK, *c_mx = c_vals + 3 * CHUNK;
    double *c_rho = c_vals + 4 * CHUNK, *c_dl = c_vals + 5 * CHUNK;
    if (act) {
        c_lz[lane] = lz;
        c_kth[lane] = my_kth;
        c_mn[lane] = pmn;
        c_mx[lane] = pmx;
        c_rho[lane] = csvd_rho(lz, lr);
        c_dl[lane] = csvd_delta(lz, lr);
    }
    __syncwarp();
    ScanIn in{D.cfg, D.C, (long long)D.V, D.d, o.cum, o.Uo, o.lrh};
    Chunk chk{q0, q1, c_lz, c_kth, c_mn, c_mx, c_rho, c_dl};
    csvd_result res = ss.res;
    ScanState stl = st0;
    Scan sc{in, stl, res};
    const csvd_config &cfg = *D.cfg;
    if (DBG_HERE(D) && lane == 0) DBG_TS(D, 44);
    if (stl.phase == PH_MAIN && cfg.variant == CSVD_VARIANT_INCREMENTAL) {
        // Common path, all prefixes of the chunk at once: the first prefix that
        // trips the budget (decode.py:342) or passes a target (decode.py:192-210).
        // Prefixes before it only merge, so the state jumps there; the eventful
        // prefix itself goes through the exact sequential machine below.
        bool ev = false;
        if (act) {
            const int p = q + 1;
            const long long n = o.cum[p];
            ev = n > cfg.k_max;
            for (int ti = 0; ti < cfg.n_targets && !ev; ++ti) {
                const int t = cfg.targets[ti];
                if (t == CSVD_TARGET_TOPK)
                    ev = n >= cfg.k && (p >= D.C || o.Uo[p] < my_kth);
                else if (t == CSVD_TARGET_SOFTMAX)
                    ev = c_rho[lane] <= cfg.epsilon;
                else
                    ev = c_dl[lane] <= csvd_ddiv(cfg.epsilon, __dsub_rn(1.0, cfg.epsilon));
            }
        }
        const unsigned m = __ballot_sync(CSVD_FULL, ev);
        const int f = m ? __ffs(m) - 1 : q1 - q0;
        if (f > 0) {
            sc.merge(chk, q0 + f - 1);
            stl.heap_pops = stl.p;
        }
    }
    if (DBG_HERE(D) && lane == 0) DBG_TS(D, 45);
    sc.run(chk);
    {  // tie flags over the prefixes of this chunk the scan tested
        bool tie = false;
        if (act && q + 1 <= stl.p && o.cum[q + 1] > 0)
            for (int ti = 0; ti < cfg.n_targets; ++ti) {
                const int t = cfg.targets[ti];
                if (t == CSVD_TARGET_SOFTMAX) tie |= near_tie(c_rho[lane], cfg.epsilon);
                else if (t == CSVD_TARGET_TOPP)
                    tie |= near_tie(c_dl[lane], csvd_ddiv(cfg.epsilon, __dsub_rn(1.0, cfg.epsilon)));
            }
        if (__any_sync(CSVD_FULL, tie) && lane == 0) ss.flags |= CSVD_FLAG_TIE_AMBIGUOUS;
    }
    if (DBG_HERE(D) && lane == 0) DBG_TS(D, 46);
    __syncwarp();
    if (lane == 0) {
        ss.st = stl;
        ss.res = res;
        ss.kcount = kc;
    }
    __syncwarp();
}

// ---------------------------------------------------------------------------
// sparse wave rows (all CTAs)
// ---------------------------------------------------------------------------
template <typename ET, int CPL, int Q>
__device__ void wave_rows(const Dev &D, const Ord &o, int p_lo, int p_hi, const double *hs, double *scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int row_lo = o.cum[p_lo], row_hi = o.cum[p_hi];
    const int gwarp = CTA_ID * WARPS + warp, nwarps = CTA_N * WARPS;
    const size_t rb = (size_t)D.d * sizeof(ET);
    if ((D.pf_mask & 2) && lane == 0) {  // every row of this warp in flight at once (L2 prefetch)
        for (int r = row_lo + gwarp; r < row_hi; r += nwarps) {
            int lo = p_lo, hi = p_hi;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (o.cum[mid] <= r) lo = mid; else hi = mid;
            }
            const int w0 = D.wrow0[o.order[lo]];
            if (w0 >= 0)
                bulk_prefetch_l2(reinterpret_cast<const char *>(D.W) + (size_t)(w0 + r - o.cum[lo]) * rb, rb);
        }
    }
    for (int r = row_lo + gwarp; r < row_hi; r += nwarps) {
        int lo = p_lo, hi = p_hi;  // cum[lo] <= r < cum[lo+1]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (o.cum[mid] <= r) lo = mid; else hi = mid;
        }
        const int c = o.order[lo];
        const int w0 = D.wrow0[c];
        if (w0 < 0) continue;  // another shard's cluster
        const int i = r - o.cum[lo];
        const int pos = D.starts[c] + i;
        const double logit = row_logit<ET, CPL, Q>(D, w0 + i, pos, hs, scratch, lane);
        if (lane == 0) {
            D.S_logits[r] = logit;
            D.S_ids[r] = (long long)__ldg(D.perm + pos);
        }
    }
}

// ---------------------------------------------------------------------------
// dense: full-vocabulary GEMV + exact k-th logit
// ---------------------------------------------------------------------------
template <typename ET, int CPL, int Q>
__device__ void dense_rows(const Dev &D, const double *hs, double *scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gwarp = CTA_ID * WARPS + warp, nwarps = CTA_N * WARPS;
    const int k = D.cfg->k;
    double *mylist = D.cand + (size_t)gwarp * D.K;
    const bool small_k = k <= 32;
    double lv = -INFINITY;  // small k: lane l holds the l-th largest so far
    int cnt = 0;
    double kmin = -INFINITY;
    // optional L2 bulk prefetch of the warp's next rows (off by default: it was
    // measured to cause re-reads, 2.6 GB of DRAM traffic for 2.1 GB of rows)
    const int PD = D.dense_pd;
    const size_t rb = (size_t)D.d * sizeof(ET);
    if (lane == 0)
        for (int j = 0; j < PD; ++j) {
            const int r = gwarp + j * nwarps;
            if (r < D.Vl) bulk_prefetch_l2(reinterpret_cast<const char *>(D.W) + (size_t)r * rb, rb);
        }
    auto take = [&](int pos, double logit) {
        if (lane == 0) {
            const int tok = __ldg(D.perm + pos);
            D.S_logits[tok] = logit;
            D.S_ids[tok] = tok;
        }
        if (small_k) {
            // branch-free insertion of `logit` (all lanes hold it) into the sorted list
            const double up = __shfl_up_sync(CSVD_FULL, lv, 1);
            lv = (lv >= logit) ? lv : ((lane == 0 || up >= logit) ? logit : up);
        } else if (lane == 0 && (cnt < k || logit > kmin)) {
            int i = cnt < k ? cnt : k - 1;
            while (i > 0 && mylist[i - 1] < logit) {
                mylist[i] = mylist[i - 1];
                --i;
            }
            mylist[i] = logit;
            if (cnt < k) cnt++;
            kmin = mylist[cnt - 1];
        }
    };
    if constexpr (CPL == 8) {  // two rows per warp at a time: both in flight, h read once
        const ET *Wt = reinterpret_cast<const ET *>(D.W);
#pragma unroll 1
        for (int lr = gwarp; lr < D.Vl; lr += 2 * nwarps) {
            const int lr2 = lr + nwarps < D.Vl ? lr + nwarps : lr;
            const int pos = D.lpos ? __ldg(D.lpos + lr) : lr;
            const int pos2 = D.lpos ? __ldg(D.lpos + lr2) : lr2;
            double la, lb;
            warp_dot_r8_x2<ET, Q>(Wt + (size_t)lr * D.d, Wt + (size_t)lr2 * D.d, hs, D.wplan.leaf_len, lane, la, lb);
            take(pos, __dadd_rn(la, __ldg(D.bias + pos)));
            if (lr2 != lr) take(pos2, __dadd_rn(lb, __ldg(D.bias + pos2)));
        }
    } else {
        for (int lr = gwarp; lr < D.Vl; lr += nwarps) {
            const int pos = D.lpos ? __ldg(D.lpos + lr) : lr;
            if (PD > 0 && lane == 0 && lr + PD * nwarps < D.Vl)
                bulk_prefetch_l2(reinterpret_cast<const char *>(D.W) + (size_t)(lr + PD * nwarps) * rb, rb);
            take(pos, row_logit<ET, CPL, Q>(D, lr, pos, hs, scratch, lane));
        }
    }
    if (small_k) {
        if (lane < k) mylist[lane] = lv;
    } else if (lane == 0) {
        for (int i = cnt; i < k; ++i) mylist[i] = -INFINITY;
    }
}

// k-th largest over rows of `row_len` valid entries with stride `stride` (exact radix select)
static __device__ __forceinline__ double block_kth_largest(const double *vals, int n, int row_len, int stride, int k) {
    __shared__ unsigned hist[256];
    __shared__ unsigned long long s_pref;
    __shared__ int s_k;
    unsigned long long prefix = 0, mask = 0;
    int kk = k;
#pragma unroll 1
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const unsigned long long key = dkey(__ldcg(vals + (size_t)(i / row_len) * stride + (i % row_len)));
            if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned cumc = 0;
            int digit = 0;
            for (int b = 255; b >= 0; --b) {
                if (cumc + hist[b] >= (unsigned)kk) {
                    digit = b;
                    kk -= (int)cumc;
                    break;
                }
                cumc += hist[b];
            }
            s_pref = prefix | ((unsigned long long)digit << shift);
            s_k = kk;
        }
        __syncthreads();
        prefix = s_pref;
        kk = s_k;
        mask |= (255ull << shift);
        __syncthreads();
    }
    return dkey_inv(prefix);
}

// scan state at p = 0 and the first wave (thread 0; shared-memory searches)
// head_n > 0: only positions [0, head_n] of the ordering exist yet (order_head);
// the first wave is the head, and the budget cap is computed once the full
// order exists (the kernel builds it before planning past the head).
static __device__ __forceinline__ void init_state(const Dev &D, const Ord &o, ScanShared &ss, int head_n,
                                                  double head_est) {
    const csvd_config &cfg = *D.cfg;
    ScanState st;
    memset(&st, 0, sizeof(st));
    st.phase = PH_MAIN;
    st.log_z = -INFINITY;
    st.smin = INFINITY;
    st.smax = -INFINITY;
    st.kth = -INFINITY;
    st.rho = 1.0;
    st.delta = INFINITY;
    ScanIn in{D.cfg, D.C, (long long)D.V, D.d, o.cum, o.Uo, o.lrh};
    ScalarSearch search;
    if (head_n == 0) {
        st.p_sel = (cfg.variant == CSVD_VARIANT_BATCHSELECT) ? csvd_select_prefix(in, cfg.k_max, search) : 0;
        st.p_cap = csvd_cap_prefix(in, st.p_sel, search);
    } else {
        st.p_sel = 0;
        st.p_cap = D.C;
    }
    const long long wt = cfg.first_wave_tokens > 0 ? cfg.first_wave_tokens : 1;
    st.wave_tokens = (int)min(wt, (long long)D.V);
    const int c0 = o.order[0];
    st.est = head_n > 0 ? head_est  // the same value order_head computed for c0
                        : (D.mode == CSVD_MODE_BIAS_AUGMENTED) ? __ldcg(D.dots + c0)
                                                               : __dadd_rn(__ldcg(D.dots + c0), D.meanb[c0]);
    st.p_lo = 0;
    st.p_hi = head_n > 0 ? head_n : csvd_plan_wave(st, in, search);
    st.mode = MODE_SPARSE;
    st.wave_tokens = st.wave_tokens * 2 < D.V ? st.wave_tokens * 2 : (int)D.V;
    ss.st = st;
    memset(&ss.res, 0, sizeof(ss.res));
    ss.kcount = 0;
    ss.flags = 0;
    ss.head_n = head_n;
}

// fast path eligibility: the head is the first wave of an incremental step
// under the default wave policy.  The head is an exact prefix of the order
// whatever the targets; for softmax / top-p targets it is just a good guess
// of where certification happens (if not, the full order is built and the
// scan continues past it).
__device__ __forceinline__ bool head_eligible(const csvd_config &cfg) {
    return cfg.variant == CSVD_VARIANT_INCREMENTAL && cfg.first_wave_tokens <= 0;
}

// host-API steps: every CTA copies its slice of the final outputs (complete in
// global memory: every CTA gets here only after the last grid barrier) into
// the mapped host buffers; CTA 0 adds the result struct.  No system fences:
// the host reads after the kernel has completed (kernel completion makes the
// writes visible), which measured ~10 us cheaper than fence + flag.
static __device__ __noinline__ void publish_host(const Dev &D, long long n, const csvd_result *r_cta0) {
    if (!D.res_host) return;
    const long long per = (n + CTA_N - 1) / CTA_N;
    const long long a = (long long)CTA_ID * per, b = min(n, a + per);
    // the fields once (a reference parameter of an out-of-line function is read
    // through generic loads, which the loop would otherwise repeat)
    long long *__restrict__ ih = D.ids_host;
    double *__restrict__ lh = D.logits_host;
    const long long *__restrict__ is = D.S_ids;
    const double *__restrict__ ls = D.S_logits;
    for (long long i = a + threadIdx.x; i < b; i += THREADS) {
        ih[i] = __ldcg(is + i);
        lh[i] = __ldcg(ls + i);
    }
    if (CTA_ID == 0 && threadIdx.x == 0) *D.res_host = *r_cta0;
}

// after a wave's scan: done / dense / next wave (thread 0): done / dense / next wave (thread 0)
static __device__ __forceinline__ void next_wave(const Dev &D, const Ord &o, ScanShared &ss) {
    ScanState s2 = ss.st;
    s2.iter += 1;
    if (s2.phase == PH_DONE) {
        s2.mode = MODE_IDLE;
    } else if (s2.phase == PH_DENSE) {
        s2.mode = MODE_DENSE;
    } else {
        ScanIn in{D.cfg, D.C, (long long)D.V, D.d, o.cum, o.Uo, o.lrh};
        s2.p_lo = s2.p;
        s2.p_hi = csvd_plan_wave(s2, in, ScalarSearch{});
        s2.wave_tokens = s2.wave_tokens * 2 < D.V ? s2.wave_tokens * 2 : (int)D.V;
    }
    ss.st = s2;
    if (s2.phase == PH_DONE && CTA_ID == 0) {
        csvd_result r = ss.res;
        r.flags = ss.flags;
        r.query_norm = D.res->query_norm;
        r.slack = D.res->slack;
        r.waves = s2.iter;
        r.error = D.res->error;
        *D.res = r;
        *D.st = s2;
    }
}

// ---------------------------------------------------------------------------
// shard open (LAUNCH_SHARD): this shard's part of sharded_decode_step
// (shard_sim.py:134-208).  The global order is already in shared memory (every
// rank computes it identically from the replicated bounds); the shard computes
// the rows of its clusters among positions [p_lo, p_hi) and CTA 0 reduces them
// to the merge record: LSE, min, max, token count and top-k list.
// ---------------------------------------------------------------------------
template <typename ET, int CPL, int Q>
__device__ void shard_open(const Dev &D, const Ord &o, ScanShared &ss, const double *hs, double *scratch,
                           double *sws) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const csvd_config &cfg = *D.cfg;
    const int C = D.C, k = cfg.k;
    const int p_lo = min(max(cfg.shard_lo, 0), C);
    const int p_hi = max(p_lo, min(cfg.shard_hi > 0 ? cfg.shard_hi : ss.st.p_sel, C));
    wave_rows<ET, CPL, Q>(D, o, p_lo, p_hi, hs, scratch);
    grid_sync(D);
    if (CTA_ID != 0) return;
    double *c_lse = sws, *c_min = c_lse + CHUNK, *c_max = c_min + CHUNK;
    double *la = D.klists ? D.klists + (size_t)CTA_ID * D.klist_stride : c_max + CHUNK;
    double *lb = la + D.K, *c_topk = lb + D.K;
    __shared__ int s_own[CHUNK];
    double reg_list = -INFINITY, m = -INFINITY, ssum = 0.0, mn = INFINITY, mx = -INFINITY;
    int kc = 0, ntok = 0;
    for (int q0 = p_lo; q0 < p_hi; q0 += D.chunk) {
        const int q1 = min(p_hi, q0 + D.chunk);
        for (int q = q0 + warp; q < q1; q += WARPS) {
            const bool own = D.wrow0[o.order[q]] >= 0;
            if (lane == 0) s_own[q - q0] = own;
            if (own) {
                double pre[SUM_E];
                summary_load(D, o.cum[q], o.cum[q + 1], pre, lane);
                cluster_summary(D, o.cum[q], o.cum[q + 1], k, c_topk + (q - q0) * k, c_lse + (q - q0),
                                c_min + (q - q0), c_max + (q - q0), pre, lane);
            }
        }
        __syncthreads();
        if (warp == 0) {
#pragma unroll 1
            for (int t = 0; t < q1 - q0; ++t) {
                if (!s_own[t]) continue;
                const int size = o.cum[q0 + t + 1] - o.cum[q0 + t];
                const int kn = size < k ? size : k;
                ntok += size;
                lse_combine(m, ssum, c_lse[t], 1.0);
                mn = fmin(mn, c_min[t]);
                mx = fmax(mx, c_max[t]);
                if (k <= 32) {
                    const double nv = lane < kn ? c_topk[t * k + lane] : -INFINITY;
                    reg_list = reg_merge(reg_list, nv, lane);
                    kc = min(k, kc + kn);
                } else {
                    kc = merge_lists(la, kc, c_topk + t * k, kn, k, lb, lane);
                    for (int j = lane; j < kc; j += 32) la[j] = lb[j];
                    __syncwarp();
                }
            }
        }
        __syncthreads();
    }
    double *out = D.shard_out;
    if (warp == 0) {
        if (k <= 32) {
            if (lane < kc) out[CSVD_SH_TOPK + lane] = reg_list;
        } else {
            for (int j = lane; j < kc; j += 32) out[CSVD_SH_TOPK + j] = la[j];
        }
        if (lane == 0) {
            out[CSVD_SH_LSE] = (m == -INFINITY) ? -INFINITY : __dadd_rn(m, csvd_log(ssum));
            out[CSVD_SH_MIN] = mn;
            out[CSVD_SH_MAX] = mx;
            out[CSVD_SH_NTOK] = (double)ntok;
            out[CSVD_SH_NLIST] = (double)kc;
            out[CSVD_SH_P_LO] = (double)p_lo;
            out[CSVD_SH_P_HI] = (double)p_hi;
            out[CSVD_SH_P_SEL] = (double)ss.st.p_sel;
            out[CSVD_SH_CUM_LO] = (double)o.cum[p_lo];
            out[CSVD_SH_CUM_HI] = (double)o.cum[p_hi];
            out[CSVD_SH_U_NEXT] = p_hi < C ? o.Uo[p_hi] : -INFINITY;
            out[CSVD_SH_LRH_NEXT] = o.lrh[p_hi];
            out[CSVD_SH_QNORM] = D.res->query_norm;
            out[CSVD_SH_SLACK] = D.res->slack;
        }
    }
    for (int q = tid; q <= C; q += THREADS) {
        if (q < C) D.order_g[q] = o.order[q];
        D.cum_g[q] = o.cum[q];
    }
}

// dense on a shard: the shard's top-k list (values above its k-th largest,
// then copies of the k-th) for the cross-shard merge; CTA 0
static __device__ void shard_dense_list(const Dev &D, double kth, int k) {
    __shared__ int s_cnt;
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    const int n = D.nblocks * WARPS * k;
    for (int i = threadIdx.x; i < n; i += THREADS) {
        const double v = __ldcg(D.cand + (size_t)(i / k) * D.K + (i % k));
        if (v > kth) D.shard_out[CSVD_SH_TOPK + atomicAdd(&s_cnt, 1)] = v;
    }
    __syncthreads();
    const int nl = min(k, D.Vl);
    for (int j = s_cnt + threadIdx.x; j < nl; j += THREADS) D.shard_out[CSVD_SH_TOPK + j] = kth;
    if (threadIdx.x == 0) {
        D.shard_out[CSVD_SH_NTOK] = (double)D.Vl;
        D.shard_out[CSVD_SH_NLIST] = (double)nl;
    }
}

// batch lanes: ||h|| from the staged copy (out of line: off the single-query path)
template <int BQ>
static __device__ __noinline__ void lane_query_norm(const Dev &D, const double *hs, double &out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        const double qn = __dsqrt_rn(warp_selfdot_smem<BQ>(hs, D.bplan.leaf_len, lane));
        if (lane == 0) {
            out = qn;
            if (CTA_ID == 0) D.res->query_norm = qn;
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// the step kernel
// ---------------------------------------------------------------------------
template <typename ET, int CPL, int Q, int BCPL, int BQ>
__device__ __forceinline__ void step_body(const Dev &D) {    extern __shared__ __align__(16) double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *hs_w = smem;
    double *hs_b = D.hs_off_b ? smem + D.hs_off_b : smem;
    double *scratch = smem + D.scratch_off + warp * (CSVD_MAX_LEAVES / 4);
    double *ws = smem + D.ord_off;
    double *sws = smem + D.sum_off;
    __shared__ ScanShared ss;
    const bool lead = CTA_ID == 0 && threadIdx.x == 0;
    if (lead) DBG_TS(D, 0);
    if (D.launch_mode != LAUNCH_BOUNDS) {
        if constexpr (CPL == 8) {  // one TMA bulk copy per pairwise leaf, completion on an mbarrier
            __shared__ unsigned long long s_hbar;
            if (threadIdx.x == 0) mbar_init(&s_hbar, 1);
            __syncthreads();
            tma_stage_leaves(D.wplan, D.h, D.d, 1, hs_w, 0, &s_hbar, 0);
        } else {
            pw_stage<CPL>(D.wplan, D.h, D.d, hs_w, D.wsrc);
        }
    }
    if (!D.pre_bounds && (D.launch_mode == LAUNCH_BOUNDS || D.hs_off_b))
        pw_stage<BCPL>(D.bplan, D.h, D.d, hs_b, D.bsrc);
    if (D.launch_mode != LAUNCH_DENSE && !D.pre_bounds && (D.pf_mask & 1) && lane == 0) {
        // start the HBM reads of this warp's centroid rows (and, in CTA 0, the
        // per-cluster arrays every CTA reads later) while h is staged
        const int c = warp * CTA_N + CTA_ID;
        if (c < D.C) bulk_prefetch_l2(D.cent + (size_t)c * D.bd, sizeof(double) * D.bd);
        if (CTA_ID == 0 && warp == WARPS - 1) {
            bulk_prefetch_l2(D.logsz, sizeof(double) * D.C);
            bulk_prefetch_l2(D.sizes, sizeof(int) * D.C);
            bulk_prefetch_l2(D.meanb, sizeof(double) * D.C);
            bulk_prefetch_l2(D.radii, sizeof(double) * D.C);
            bulk_prefetch_l2(D.maxb, sizeof(double) * D.C);
            bulk_prefetch_l2(D.starts, sizeof(int) * D.C);
        }
    }
    if (threadIdx.x == 0) {
        memset(&ss, 0, sizeof(ss));
        if (D.launch_mode == LAUNCH_DENSE) {
            ss.st.mode = MODE_DENSE;
            ss.st.phase = PH_DENSE;
        }
    }
    __syncthreads();
    if (lead) DBG_TS(D, 1);
    const int k = D.cfg->k;
    Ord o;
    ord_bind(D, ws, o);
    if (D.launch_mode == LAUNCH_DENSE) {
        if (lead) {
            D.res->query_norm = 0.0;
            D.res->slack = 0.0;
        }
    } else {
        if (!D.pre_bounds) {
            bounds_phase<BCPL, BQ>(D, hs_b, scratch);
            if (lead) DBG_TS(D, 2);
            grid_sync(D);
        } else if constexpr (BCPL == 8) {  // batched bounds: dots are given; ||h|| here
            lane_query_norm<BQ>(D, hs_b, ss.st.est);  // carried to stage_bounds (ss is rebuilt later)
        }
        if (lead) DBG_TS(D, 3);
        const bool ok = stage_bounds(D, o, ss.st.est);
        if (!ok || D.launch_mode == LAUNCH_BOUNDS) {
            if (lead) D.res->error = ok ? 0 : CSVD_EVALUE;
            return;
        }
        __shared__ double s_head_est;
        const int hn = head_eligible(*D.cfg) ? order_head(D, o, s_head_est) : 0;
        if (lead && D.dbg) D.dbg[63] = (unsigned long long)hn;
        if (lead) DBG_TS(D, 5);
        if (hn == 0) order_full(D, o);
        if (lead) DBG_TS(D, 4);
        if (threadIdx.x == 0) init_state(D, o, ss, hn, s_head_est);
        __syncthreads();
        if (lead) DBG_TS(D, 6);
        if (D.launch_mode == LAUNCH_SHARD) {
            shard_open<ET, CPL, Q>(D, o, ss, hs_w, scratch, sws);
            return;
        }
    }
    // chunk scratch: [6*CHUNK values][CHUNK lse][CHUNK min][CHUNK max][2 K-lists][chunk*k topk]
    double *c_vals = sws, *c_lse = sws + 6 * CHUNK, *c_min = c_lse + CHUNK, *c_max = c_min + CHUNK;
    // the K-lists: shared memory, or this CTA's slice of D.klists (large k)
    double *la = D.klists ? D.klists + (size_t)CTA_ID * D.klist_stride : c_max + CHUNK;
    double *lb = la + D.K, *c_topk = lb + D.K;
    double reg_list = -INFINITY;
    for (int guard = 0; guard < D.C + 8; ++guard) {
        const ScanState st = ss.st;
        if (st.mode == MODE_IDLE || __ldcg(&D.res->error)) break;
        if (st.mode == MODE_SPARSE) {
            if (lead) DBG_TS(D, 8 + 4 * (st.iter & 3));
            wave_rows<ET, CPL, Q>(D, o, st.p_lo, st.p_hi, hs_w, scratch);
            if (D.dbg && st.iter == 0) {  // per-CTA end of its rows (before the barrier)
                __syncthreads();
                if (threadIdx.x == 0 && blockIdx.x < 128) D.dbg[128 + 512 - 128 + blockIdx.x] = gtimer();
            }
            grid_sync(D);
            if (lead) DBG_TS(D, 9 + 4 * (st.iter & 3));
            // per-cluster summaries: distributed over the grid (each cluster
            // summarised once, into D.gsum, then one grid barrier) when the
            // wave is wider than one CTA's warps; else redundantly per CTA
            const bool dist = D.gsum && k <= 32 && D.lanes == nullptr && st.p_hi - st.p_lo > WARPS;
            const double *g_lse = D.gsum, *g_min = D.gsum + D.C, *g_max = D.gsum + 2 * D.C;
            const double *g_topk = D.gsum + 3 * D.C;  // [C][32]
            if (dist) {
#pragma unroll 1
                for (int q = st.p_lo + CTA_ID * WARPS + warp; q < st.p_hi; q += CTA_N * WARPS) {
                    double pre[SUM_E];
                    summary_load(D, o.cum[q], o.cum[q + 1], pre, lane);
                    cluster_summary(D, o.cum[q], o.cum[q + 1], k, D.gsum + 3 * D.C + (size_t)q * 32, D.gsum + q,
                                    D.gsum + D.C + q, D.gsum + 2 * D.C + q, pre, lane);
                }
                grid_sync(D);  // its acq_rel arrival publishes the summaries
            }
            // summaries + scan, chunk by chunk (identical in every CTA)
            for (int q0 = st.p_lo; q0 < st.p_hi; q0 += D.chunk) {
                const int q1 = min(st.p_hi, q0 + D.chunk);
                if (dist) {
                    for (int i = threadIdx.x; i < q1 - q0; i += THREADS) {
                        c_lse[i] = __ldcg(g_lse + q0 + i);
                        c_min[i] = __ldcg(g_min + q0 + i);
                        c_max[i] = __ldcg(g_max + q0 + i);
                    }
                    for (int i = threadIdx.x; i < (q1 - q0) * k; i += THREADS)
                        c_topk[i] = __ldcg(g_topk + (size_t)(q0 + i / k) * 32 + i % k);
                } else {  // the loads of this warp's next two clusters are always in flight
                    double pre[2][SUM_E];
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        const int q = q0 + warp + t * WARPS;
                        if (q < q1) summary_load(D, o.cum[q], o.cum[q + 1], pre[t], lane);
                    }
#pragma unroll 1
                    for (int q = q0 + warp; q < q1; q += WARPS) {  // one copy of the summary code
                        cluster_summary(D, o.cum[q], o.cum[q + 1], k, c_topk + (q - q0) * k, c_lse + (q - q0),
                                        c_min + (q - q0), c_max + (q - q0), pre[0], lane);
#pragma unroll
                        for (int e = 0; e < SUM_E; ++e) pre[0][e] = pre[1][e];
                        const int qn = q + 2 * WARPS;
                        if (qn < q1) summary_load(D, o.cum[qn], o.cum[qn + 1], pre[1], lane);
                    }
                }
                __syncthreads();
                if (lead) DBG_TS(D, 10 + 4 * (st.iter & 3));
                double full_pre = NAN;
                {  // this chunk's 64-merge recompute (certify.py:79-83), by the whole CTA
                    const int rl = (q0 / 64) * 64 + 63 - q0;
                    if (rl < q1 - q0) {
                        __shared__ double s_red2[WARPS];
                        double vmax = ss.st.p > 0 ? ss.st.smax : -INFINITY;
                        for (int t = 0; t <= rl; ++t) vmax = fmax(vmax, c_max[t]);
                        full_pre = block_lse_all(D.S_logits, o.cum[q0 + rl + 1], vmax, s_red2);
                    }
                }
                if (warp == 0)
                    scan_chunk(D, o, ss, q0, q1, c_topk, c_lse, c_min, c_max, c_vals, la, lb, reg_list, lane,
                               full_pre);
                __syncthreads();
                if (ss.st.phase != PH_MAIN && ss.st.phase != PH_PE) break;
            }
            if (ss.head_n > 0 && (ss.st.phase == PH_MAIN || ss.st.phase == PH_PE)) {
                // the head is exhausted: build the full order, then plan as usual
                order_full(D, o);
                if (threadIdx.x == 0) {
                    ScanIn in{D.cfg, D.C, (long long)D.V, D.d, o.cum, o.Uo, o.lrh};
                    ss.st.p_cap = csvd_cap_prefix(in, ss.st.p_sel, ScalarSearch{});
                    ss.head_n = 0;
                }
                __syncthreads();
            }
            if (threadIdx.x == 0) next_wave(D, o, ss);
            if (lead) DBG_TS(D, 47);
            __syncthreads();
            if (ss.st.mode == MODE_IDLE && D.res_host) {
                csvd_result r = ss.res;
                r.flags = ss.flags;
                r.query_norm = D.res->query_norm;
                r.slack = D.res->slack;
                r.waves = ss.st.iter;
                r.error = __ldcg(&D.res->error);
                publish_host(D, r.sub_size, CTA_ID == 0 ? &r : nullptr);
            }
            if (lead) DBG_TS(D, 11 + 4 * (st.iter & 3));
        } else {  // MODE_DENSE
            if (lead) DBG_TS(D, 36);
            dense_rows<ET, CPL, Q>(D, hs_w, scratch);
            grid_sync(D);
            if (lead) DBG_TS(D, 37);
            if (CTA_ID != 0) {
                publish_host(D, D.V, nullptr);
                break;
            }
            const double kth = block_kth_largest(D.cand, D.nblocks * WARPS * k, k, D.K, k);
            if (D.lpos) shard_dense_list(D, kth, k);
            if (threadIdx.x == 0) {
                ScanIn in{D.cfg, D.C, (long long)D.V, D.d, nullptr, nullptr, nullptr};
                csvd_result r;
                memset(&r, 0, sizeof(r));
                ScanState s2 = ss.st;
                Scan sc{in, s2, r};
                sc.finish_dense(kth);
                r.query_norm = D.res->query_norm;
                r.slack = D.res->slack;
                r.waves = s2.iter + 1;
                r.error = D.res->error;
                *D.res = r;
                s2.mode = MODE_IDLE;
                *D.st = s2;
                ss.res = r;
            }
            __syncthreads();
            publish_host(D, D.V, &ss.res);
            break;
        }
    }
}

template <typename ET, int CPL, int Q, int BCPL, int BQ, bool GROUPED = false>
__global__ void __launch_bounds__(THREADS, 1) k_step(const __grid_constant__ Dev D0) {
    if constexpr (GROUPED) {
        // one launch runs a whole batch: lane b is blockIdx.x / nblocks and
        // swaps its own workspaces into the Dev (all table data is shared);
        // the lane's Dev lives in shared memory, not local memory
        __shared__ Dev D;
        if (threadIdx.x == 0) {
            const LaneWS &w = D0.lanes[blockIdx.x / (unsigned)D0.nblocks];
            D = D0;
            D.h = w.h;
            D.U = w.U;
            D.Uraw = w.Uraw;
            D.dots = w.dots;
            D.order_g = w.order_g;
            D.cum_g = w.cum_g;
            D.S_logits = w.S_logits;
            D.S_ids = w.S_ids;
            D.st = w.st;
            D.res = w.res;
            D.bar = w.bar;
            D.cand = w.cand;
            D.klists = w.klists;
            D.shard_out = w.shard_out;
            D.res_host = w.res_host;
            D.ids_host = w.ids_host;
            D.logits_host = w.logits_host;
        }
        __syncthreads();
        step_body<ET, CPL, Q, BCPL, BQ>(D);
    } else {
        if (D0.dbg && threadIdx.x == 0) D0.dbg[128 + blockIdx.x] = gtimer();
        step_body<ET, CPL, Q, BCPL, BQ>(D0);
        __syncthreads();
        if (D0.dbg && threadIdx.x == 0) D0.dbg[128 + 256 + blockIdx.x] = gtimer();
    }
}

// ---------------------------------------------------------------------------
// batched bounds (decode over a batch): U for B queries with every centroid
// row read once per group of BQN queries (warp per cluster, the same pairwise
// tree per query as bounds_phase); lanes then start from these bounds.
// Regular plans only (the bound dimension is d: euclidean / spherical).
// ---------------------------------------------------------------------------
#define BQN 3   // queries per register block when a warp pairs two clusters
#define BQN1 6  // queries per register block at one cluster per warp (C <= warps)
template <int BQ, int NR = 1>
__global__ void __launch_bounds__(THREADS, 1)
    k_bounds_batch(Dev D, const double *__restrict__ H, int B, double *const *Uraw_l, double *const *dots_l,
                   csvd_result *res_all, int gq /* queries per pass (<= BQN1, by shared memory) */) {
    extern __shared__ __align__(16) double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int hs_stride = (pw_hs_size(D.bplan) + 1) & ~1;
    __shared__ unsigned long long s_bar;
    if (threadIdx.x == 0) mbar_init(&s_bar, 1);
    __syncthreads();
    const int gwarp = blockIdx.x * WARPS + warp, nwarps = gridDim.x * WARPS;
    if ((D.pf_mask & 1) && lane == 0)  // optional: this warp's centroid rows towards L2
        for (int c = gwarp; c < D.C; c += nwarps) bulk_prefetch_l2(D.cent + (size_t)c * D.bd, sizeof(double) * D.bd);
    // Rounds of clusters (one warp task each: nwarps * NR clusters), each
    // swept by every pass of queries before the next round: a round's
    // centroid rows come from HBM once and from L2 for the other passes (a
    // pass-major order re-streams all C rows per pass once C * d * 8 bytes
    // outgrow the L2).  CSVD_PF bit 16 turns rounds on: measured no gain (c5
    // B=128 2.26 ms against 2.19 ms pass-major; the kernel is f64-issue bound).
    const bool rounds = (D.pf_mask & 16) != 0;
    const int per_round = rounds ? nwarps * NR : D.C;
    unsigned phase = 0;
    for (int r0 = 0; r0 < D.C; r0 += per_round)
    for (int qb = 0; qb < B; qb += gq) {
        const int nq = min(gq, B - qb);
        const int r1 = min(D.C, r0 + per_round);
        tma_stage_leaves(D.bplan, H + (size_t)qb * D.d, D.d, nq, smem, hs_stride, &s_bar, phase++);
        // one cluster per warp task (looping over the clusters), the
        // registers a second row would take hold more queries instead; the
        // row's next element step is in flight while the current one is used
        if constexpr (NR == 1) {
#pragma unroll 1
            for (int c = r0 + gwarp; c < r1; c += nwarps) {
                const double *const rows[1] = {D.cent + (size_t)c * D.bd};
                double dots[1][BQN1];
                warp_dot_regular_multi<BQ, BQN1, 1>(rows, smem, hs_stride, nq, D.bplan.leaf_len, lane, dots);
                if (lane == 0) {  // the lanes finish U = dot + R ||h|| (+ max b) themselves
#pragma unroll
                    for (int j = 0; j < BQN1; ++j)
                        if (j < nq) dots_l[qb + j][c] = dots[0][j];
                }
            }
        } else {  // two clusters x BQN queries: every staged h value feeds both rows
#pragma unroll 1
            for (int c = r0 + gwarp; c < r1; c += 2 * nwarps) {
                const int c2 = c + nwarps < r1 ? c + nwarps : c;  // odd tail: recompute c, discard
                const double *const rows[2] = {D.cent + (size_t)c * D.bd, D.cent + (size_t)c2 * D.bd};
#pragma unroll 1
                for (int j0 = 0; j0 < nq; j0 += BQN) {
                    double dots[2][BQN];
                    warp_dot_regular_multi<BQ, BQN, 2>(rows, smem + (size_t)j0 * hs_stride, hs_stride,
                                                       min(BQN, nq - j0), D.bplan.leaf_len, lane, dots);
                    if (lane == 0) {
#pragma unroll
                        for (int j = 0; j < BQN; ++j)
                            if (j0 + j < nq) {
                                dots_l[qb + j0 + j][c] = dots[0][j];
                                if (c2 != c) dots_l[qb + j0 + j][c2] = dots[1][j];
                            }
                    }
                }
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// batched bounds, chain-per-lane form (k_bbatch): the same pairwise tree as
// warp_dot_regular<double, 8, Q> (d = NL leaves of L elements, L % 8 == 0,
// NL = 2^m >= 4), but a lane owns ONE chain of a leaf (8 lanes per leaf, 4
// leaves per warp slice) instead of a whole leaf.  A lane then holds one
// accumulator per (cluster, query) pair, so a warp register-blocks KR
// clusters x KQ queries: per element step KR centroid loads and KQ staged h
// reads feed 2*KR*KQ f64 operations (f64-issue-bound rather than latency- or
// load-bound).  CTA group g stages queries [g*KQ, (g+1)*KQ) in shared memory
// (layout hs[j][((u*S + i)*4 + leaf)*8 + chain]) and its warps sweep the
// cluster groups; the groups of one cluster range run concurrently, so a
// centroid row comes from HBM once and from L2 for the other groups.
// Combine: chains ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and the 4 leaves of a
// slice by xor-butterflies, slices by a balanced binary tree (a carry stack),
// result 0.0 + total: bit-identical to the leaf-per-lane path.
// ---------------------------------------------------------------------------
#define KBR 2  // clusters per warp task
#define KBQ 6  // queries per CTA group (shared memory: KBQ * d doubles)
#define KBU 8  // element steps per load batch (two batches in flight)
// shared memory of k_bbatch for kq queries of dimension d (NS slices)
__host__ __device__ inline size_t kbb2_smem_bytes(int kq, int d, int NS) {
    return sizeof(double) * ((size_t)kq * d + (size_t)WARPS * KBR * KBQ * NS);
}
static __global__ void __launch_bounds__(THREADS, 1)
    k_bbatch(Dev D, const double *__restrict__ H, int B, double *const *dots_l, int kq, int ngroups) {
    extern __shared__ __align__(16) double smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int d = D.d, L = D.bplan.leaf_len, S = L >> 3, NS = d / (4 * L);  // slices
    const int NT = NS * S;  // element steps per row (per lane)
    double *part = smem + (size_t)kq * d + (size_t)warp * KBR * KBQ * NS;  // slice totals [r][j][u]
    const int per = max(1, (int)gridDim.x / ngroups);  // CTAs per query group
    const int t = blockIdx.x % per, cpg = per;
    const int lt = lane >> 3, ch = lane & 7;
    const int ncg = (D.C + KBR - 1) / KBR;
    for (int g = blockIdx.x / per; g < ngroups; g += max(1, (int)gridDim.x / per)) {
        const int q0 = g * kq, nq = min(kq, B - q0);
        __syncthreads();  // the previous group's reads of smem are done
        // stage the group's queries: destination-ordered, gathered from global
        for (int idx = tid; idx < nq * d; idx += THREADS) {
            const int j = idx / d, r = idx - j * d;
            const int u = r / (S * 32), rem = r - u * (S * 32), i = rem >> 5, ln = rem & 31;
            smem[idx] = __ldg(H + (size_t)(q0 + j) * d + (u * 4 + (ln >> 3)) * L + 8 * i + (ln & 7));
        }
        __syncthreads();
        int cg = t * WARPS + warp;
        if (lane == 0 && cg < ncg)  // this warp's first rows towards L2
            for (int r = 0; r < KBR; ++r)
                bulk_prefetch_l2(D.cent + (size_t)min(cg * KBR + r, D.C - 1) * D.bd, sizeof(double) * d);
        for (; cg < ncg; cg += cpg * WARPS) {
            const double *rp[KBR];
#pragma unroll
            for (int r = 0; r < KBR; ++r) rp[r] = D.cent + (size_t)min(cg * KBR + r, D.C - 1) * D.bd + lt * L + ch;
            const int cn = cg + cpg * WARPS;
            if (lane == 0 && cn < ncg)  // the next task's rows towards L2 while this one runs
                for (int r = 0; r < KBR; ++r)
                    bulk_prefetch_l2(D.cent + (size_t)min(cn * KBR + r, D.C - 1) * D.bd, sizeof(double) * d);
            // element step gs = u * S + i: address rp + u * 4L + 8i
            auto ld = [&](double (&x)[KBU][KBR], int gs0) {
#pragma unroll
                for (int s2 = 0; s2 < KBU; ++s2) {
                    const int gs = gs0 + s2;
                    const int u = gs / S, i = gs - u * S;
#pragma unroll
                    for (int r = 0; r < KBR; ++r) x[s2][r] = gs < NT ? __ldg(rp[r] + u * 4 * L + 8 * i) : 0.0;
                }
            };
            double acc[KBR][KBQ];
            auto consume = [&](const double (&x)[KBU][KBR], int gs0) {
#pragma unroll
                for (int s2 = 0; s2 < KBU; ++s2) {
                    const int gs = gs0 + s2;
                    if (gs < NT) {
                        const int u = gs / S, i = gs - u * S;
                        const double *hp = smem + (size_t)gs * 32 + lane;  // (u * S + i) * 32 + lane
#pragma unroll
                        for (int j = 0; j < KBQ; ++j) {
                            if (j < nq) {
                                const double hv = hp[(size_t)j * d];
#pragma unroll
                                for (int r = 0; r < KBR; ++r) {
                                    const double pr = d_mul(x[s2][r], hv);
                                    acc[r][j] = (i == 0) ? pr : d_add(acc[r][j], pr);
                                }
                            }
                        }
                        if (i == S - 1) {  // slice done: chains -> leaves -> slice total
#pragma unroll
                            for (int r = 0; r < KBR; ++r)
#pragma unroll
                                for (int j = 0; j < KBQ; ++j) {
                                    double v = acc[r][j];
#pragma unroll
                                    for (int o = 1; o < 32; o <<= 1) v = d_add(v, __shfl_xor_sync(CSVD_FULL, v, o));
                                    if (lane == 0) part[(r * KBQ + j) * NS + u] = v;
                                }
                        }
                    }
                }
            };
            double xa[KBU][KBR], xb[KBU][KBR];
            ld(xa, 0);
#pragma unroll 1
            for (int gs0 = 0; gs0 < NT; gs0 += 2 * KBU) {
                ld(xb, gs0 + KBU);
                consume(xa, gs0);
                ld(xa, gs0 + 2 * KBU);
                consume(xb, gs0 + KBU);
            }
            __syncwarp();
            // balanced tree over the slices (in place), one (cluster, query) pair per lane
            if (lane < KBR * KBQ) {
                const int r = lane / KBQ, j = lane % KBQ, c = cg * KBR + r;
                double *pp = part + lane * NS;
                for (int w = 1; w < NS; w <<= 1)
                    for (int u = 0; u + w < NS; u += 2 * w) pp[u] = d_add(pp[u], pp[u + w]);
                if (c < D.C && j < nq) dots_l[q0 + j][c] = d_add(0.0, pp[0]);
            }
            __syncwarp();
        }
    }
}

// ---------------------------------------------------------------------------
// standalone full-vocabulary GEMV (oracle.dense_logits, oracle.py:33-41): the
// same exact row dot as the step's fallback, as its own high-occupancy kernel
// (2 CTAs / 16 warps per SM, <= 128 registers) so more rows are in flight;
// logits scattered to token order.  Regular plans only.
// ---------------------------------------------------------------------------
template <typename ET, int CPL, int Q>
__global__ void __launch_bounds__(THREADS, 2) k_dense_gemv(const __grid_constant__ Dev D) {
    extern __shared__ __align__(16) double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    pw_stage<CPL>(D.wplan, D.h, D.d, smem, D.wsrc);
    __syncthreads();
    const int gwarp = blockIdx.x * WARPS + warp, nwarps = gridDim.x * WARPS;
    const int PD = D.dense_pd;  // rows kept in flight ahead through L2 bulk prefetches
    const size_t rb = (size_t)D.d * sizeof(ET);
    if (lane == 0)
        for (int j = 0; j < PD; ++j) {
            const int r = gwarp + j * nwarps;
            if (r < D.Vl) bulk_prefetch_l2(reinterpret_cast<const char *>(D.W) + (size_t)r * rb, rb);
        }
    for (int lr = gwarp; lr < D.Vl; lr += nwarps) {
        if (PD > 0 && lane == 0 && lr + PD * nwarps < D.Vl)
            bulk_prefetch_l2(reinterpret_cast<const char *>(D.W) + (size_t)(lr + PD * nwarps) * rb, rb);
        const int pos = D.lpos ? __ldg(D.lpos + lr) : lr;
        const double logit = row_logit<ET, CPL, Q>(D, lr, pos, smem, nullptr, lane);
        if (lane == 0) {
            const int tok = __ldg(D.perm + pos);
            D.S_logits[tok] = logit;
            D.S_ids[tok] = tok;
        }
    }
}
