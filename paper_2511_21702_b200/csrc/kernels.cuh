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
#define MAX_PER_WARP 8  // clusters per warp in the bounds / rank phases
#define CHUNK 32        // max clusters per scan chunk (one per lane)

enum { LAUNCH_STEP = 0, LAUNCH_BOUNDS = 1, LAUNCH_DENSE = 2 };

struct Dev {
    int V, d, C, bd, mode, wdtype;
    int K;  // top-k capacity (row stride of the dense candidate lists, list buffers)
    const void *W;      // [V, d] permuted rows (fp32 | bf16)
    const float *bias;  // [V] permuted
    const int *perm;    // [V] position -> token id
    const double *cent; // [C, bd]
    const double *radii, *maxb, *cnorm, *ang, *maxn, *minn, *logsz, *meanb;
    const int *starts, *sizes;
    PwPlan wplan, bplan;
    const int *wsrc, *bsrc;  // interleaved-layout source tables (CPL < 8 plans)
    // per step
    const double *h;         // [d]
    const csvd_config *cfg;
    double *U, *dots;        // [C] by cluster id (U final, with slack)
    double *Uo, *lrh;        // [C], [C+1] by opening position
    int *order, *cum;        // [C], [C+1]
    double *S_logits;        // [V]
    long long *S_ids;        // [V]
    double *cand;            // [nwarps*K] dense per-warp candidates
    ScanState *st;           // final state (diagnostic)
    csvd_result *res;
    unsigned *bar;           // grid barrier: [0] arrivals, [1] generation
    int nblocks;
    int launch_mode;
    int hs_off_b;            // offset (doubles) of the bounds h layout, 0 = shared with W
    int scratch_off;         // generic-path per-warp leaf scratch
    int ord_off;             // ordering arrays (rank staging, then order/cum/Uo/lrh)
    int sum_off;             // chunk summaries + scan scratch
    int chunk;               // clusters per summary/scan chunk (<= CHUNK)
    unsigned long long *dbg; // optional phase timestamps (CSVD_DEBUG_TS)
};

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
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
__device__ __noinline__ void lse_combine(double &m, double &s, double m2, double s2) {
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

// strict total order of the opening sequence: U descending, id ascending
// (np.lexsort((arange(C), -U)), decode.py:166)
__device__ __forceinline__ bool key_before(double ua, int ia, double ub, int ib) {
    return (ua > ub) || (ua == ub && ia < ib);
}

// Plain grid barrier (cooperative launch: all CTAs resident).
__device__ __noinline__ void grid_sync(const Dev &D) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned gen = ld_acquire(D.bar + 1);
        __threadfence();
        const unsigned t = atomicAdd(D.bar, 1u);
        if (t == (unsigned)D.nblocks - 1u) {
            D.bar[0] = 0;
            __threadfence();
            st_release(D.bar + 1, gen + 1u);
        } else {
            unsigned long long spins = 0;
            while (ld_acquire(D.bar + 1) == gen) {
                __nanosleep(CSVD_SPIN_NS);
                if (++spins > (1ull << 24)) {  // ~1-2 s: flag and give up rather than hang
                    D.res->error = CSVD_ESTATE;
                    break;
                }
            }
        }
    }
    __syncthreads();
}

template <typename ET, int CPL, int Q>
__device__ __forceinline__ double row_logit(const Dev &D, int pos, const double *hs, double *scratch, int lane) {
    const ET *row = reinterpret_cast<const ET *>(D.W) + (size_t)pos * D.d;
    double dot = warp_dot_t<ET, CPL, Q>(row, hs, D.wplan, scratch, lane);
    return __dadd_rn(dot, (double)__ldg(D.bias + pos));
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

template <int BCPL, int BQ>
__device__ void bounds_phase(const Dev &D, const double *hs, double *scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ double s_qn;
    __shared__ double s_dot[WARPS][MAX_PER_WARP];
    const int stride = gridDim.x * WARPS;
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
    int j = 0;
    for (int c = warp * gridDim.x + blockIdx.x; c < D.C && j < MAX_PER_WARP; c += stride, ++j) {
        double dot = warp_dot_t<double, BCPL, BQ>(D.cent + (size_t)c * D.bd, hs, D.bplan, scratch, lane);
        if (lane == 0) s_dot[warp][j] = dot;
    }
    __syncthreads();
    const double qn = s_qn;
    if (lane == 0) {
        j = 0;
        for (int c = warp * gridDim.x + blockIdx.x; c < D.C && j < MAX_PER_WARP; c += stride, ++j) {
            const double dot = s_dot[warp][j];
            double u;
            if (D.mode == CSVD_MODE_SPHERICAL)
                u = cone_bound(D, c, dot, qn);
            else if (D.mode == CSVD_MODE_BIAS_AUGMENTED)
                u = __dadd_rn(dot, __dmul_rn(D.radii[c], qn));
            else
                u = __dadd_rn(__dadd_rn(dot, __dmul_rn(D.radii[c], qn)), D.maxb[c]);
            D.U[c] = u;  // raw (the rank phase adds the slack)
            D.dots[c] = dot;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) D.res->query_norm = qn;
}

// ---------------------------------------------------------------------------
// rank phase (all CTAs): the opening order without a sort
// ---------------------------------------------------------------------------
struct RankShared {
    double slack, xmax;
    int c0;   // cluster ranked first
    int bad;  // non-finite bound seen
};

// Stages U (+slack), x = log|c| + U, e = exp(x - xmax), |c| in shared memory,
// then every warp ranks its own clusters.  Returns false (in every CTA) if a
// bound is non-finite.  Predicted first-wave clusters get their W rows
// prefetched into L2.
__device__ __noinline__ bool rank_phase(const Dev &D, double *ws, RankShared &rs) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int C = D.C;
    const csvd_config &cfg = *D.cfg;
    double *U_s = ws, *x_s = ws + C, *e_s = ws + 2 * C;
    int *sz_s = reinterpret_cast<int *>(ws + 3 * C);
    __shared__ double s_red[WARPS];
    __shared__ int s_ired[WARPS];
    // --- raw bounds (+ slack, bounds.py:58-64, which needs max |U| first)
    double amax = 1.0;
    for (int c = tid; c < C; c += THREADS) {
        const double u = __ldcg(D.U + c);
        U_s[c] = u;
        sz_s[c] = D.sizes[c];
        amax = fmax(amax, fabs(u));
    }
    double eta = 0.0;
    if (cfg.slack_f32) {
        amax = warp_max(amax);
        if (lane == 0) s_red[warp] = amax;
        __syncthreads();
        double m = 1.0;
        for (int w = 0; w < WARPS; ++w) m = fmax(m, s_red[w]);
        eta = __dmul_rn(__dmul_rn(4.0, 1.1920928955078125e-07), m);
        __syncthreads();
    }
    double xm = -INFINITY;
    int bad = 0;
    for (int c = tid; c < C; c += THREADS) {
        const double u = __dadd_rn(U_s[c], eta);
        U_s[c] = u;
        bad |= !isfinite(u);  // BoundVector.__post_init__ (bounds.py:53-55)
        const double x = __dadd_rn(D.logsz[c], u);  // certify.py:119 np.log(sizes) + U
        x_s[c] = x;
        xm = fmax(xm, x);
    }
    xm = warp_max(xm);
    bad = __any_sync(CSVD_FULL, bad);
    if (lane == 0) {
        s_red[warp] = xm;
        s_ired[warp] = bad;
    }
    __syncthreads();
    double xmax = -INFINITY;
    bad = 0;
    for (int w = 0; w < WARPS; ++w) {
        xmax = fmax(xmax, s_red[w]);
        bad |= s_ired[w];
    }
    if (tid == 0) {
        rs.slack = eta;
        rs.xmax = xmax;
        rs.bad = bad;
    }
    if (bad) return false;
    for (int c = tid; c < C; c += THREADS) e_s[c] = csvd_exp(__dsub_rn(x_s[c], xmax));
    __syncthreads();
    // --- rank own clusters: position, tokens before, log R-hat at that position
    const int stride = gridDim.x * WARPS;
    int j = 0;
    for (int c = warp * gridDim.x + blockIdx.x; c < C && j < MAX_PER_WARP; c += stride, ++j) {
        const double uc = U_s[c];
        int before = 0, off = 0;
        double tail = 0.0, tmax = -INFINITY;
        for (int i = lane; i < C; i += 32) {
            if (key_before(U_s[i], i, uc, c)) {
                before += 1;
                off += sz_s[i];
            } else {
                tail = __dadd_rn(tail, e_s[i]);
                tmax = fmax(tmax, x_s[i]);
            }
        }
        before = warp_isum(before);
        off = warp_isum(off);
        tail = warp_sum(tail);
        tmax = warp_max(tmax);
        double lr;
        if (tail > 1e-280) {
            lr = __dadd_rn(xmax, csvd_log(tail));
        } else {  // far below the global max: rescale by the tail's own max
            double t2 = 0.0;
            for (int i = lane; i < C; i += 32)
                if (!key_before(U_s[i], i, uc, c)) t2 = __dadd_rn(t2, csvd_exp(__dsub_rn(x_s[i], tmax)));
            t2 = warp_sum(t2);
            lr = __dadd_rn(tmax, csvd_log(t2));
        }
        if (lane == 0) {
            D.order[before] = c;
            D.Uo[before] = uc;
            D.cum[before] = off;
            D.lrh[before] = lr;
            D.U[c] = uc;
        }
    }
    if (blockIdx.x == 0 && tid == 0) {
        D.cum[C] = D.V;
        D.lrh[C] = -INFINITY;
        D.res->slack = eta;
    }
    return true;
}

// ---------------------------------------------------------------------------
// per-CTA ordering + scan state in shared memory
// ---------------------------------------------------------------------------
struct Ord {  // the full ordering, loaded once per step
    int *order, *cum;
    double *Uo, *lrh;
};

__device__ __forceinline__ void ord_bind(const Dev &D, double *ws, Ord &o) {
    const int C = D.C;
    o.Uo = ws;
    o.lrh = ws + C;
    o.order = reinterpret_cast<int *>(ws + 2 * C + 1);
    o.cum = o.order + C;
}

__device__ void load_ordering(const Dev &D, const Ord &o) {
    const int C = D.C;
    for (int i = threadIdx.x; i <= C; i += THREADS) {
        if (i < C) {
            o.order[i] = __ldcg(D.order + i);
            o.Uo[i] = __ldcg(D.Uo + i);
        }
        o.cum[i] = __ldcg(D.cum + i);
        o.lrh[i] = __ldcg(D.lrh + i);
    }
    __syncthreads();
}

// cluster summary (warp): top-min(k,n) values desc, LSE, min, max of the
// cluster's logits S_logits[lo, hi)
__device__ __noinline__ void cluster_summary(const Dev &D, int lo, int hi, int k, double *topk, double *lse_o,
                                             double *min_o, double *max_o, int lane) {
    const int n = hi - lo;
    const double *v = D.S_logits + lo;
    const int kk = n < k ? n : k;
    constexpr int E = 4;
    double reg[E];
    const bool in_regs = n <= 32 * E;
    double mx = -INFINITY, mn = INFINITY;
    if (in_regs) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int i = lane + 32 * e;
            reg[e] = i < n ? __ldcg(v + i) : -INFINITY;
            if (i < n) {
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
    mx = warp_max(mx);
    mn = warp_min(mn);
    double s = 0.0;
    if (in_regs) {
#pragma unroll
        for (int e = 0; e < E; ++e)
            if (lane + 32 * e < n) s = __dadd_rn(s, csvd_exp(__dsub_rn(reg[e], mx)));
    } else {
        for (int i = lane; i < n; i += 32) s = __dadd_rn(s, csvd_exp(__dsub_rn(__ldcg(v + i), mx)));
    }
    s = warp_sum(s);
    // iterative selection in (value desc, index asc) order
    double pv = INFINITY;
    int pi = -1;
#pragma unroll 1
    for (int j = 0; j < kk; ++j) {
        double bv = -INFINITY;
        int bi = 0x7fffffff;
        if (in_regs) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                const int i = lane + 32 * e;
                const double x = reg[e];
                const bool after = (x < pv) || (x == pv && i > pi);
                if (i < n && after && (x > bv || (x == bv && i < bi))) {
                    bv = x;
                    bi = i;
                }
            }
        } else {
            for (int i = lane; i < n; i += 32) {
                const double x = __ldcg(v + i);
                const bool after = (x < pv) || (x == pv && i > pi);
                if (after && (x > bv || (x == bv && i < bi))) {
                    bv = x;
                    bi = i;
                }
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
__device__ int merge_lists(const double *A, int ka, const double *B, int kb, int k, double *out, int lane) {
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

// logsumexp over S_logits[0, n) with known max (64-merge recompute, certify.py:79-83)
__device__ double warp_lse_all(const double *vals, int n, double vmax, int lane) {
    if (n == 0 || vmax == -INFINITY) return -INFINITY;
    if (vmax == INFINITY) return INFINITY;
    double s = 0.0;
    for (int i = lane; i < n; i += 32) s = __dadd_rn(s, csvd_exp(__dsub_rn(__ldcg(vals + i), vmax)));
    s = warp_sum(s);
    return __dadd_rn(vmax, csvd_log(s));
}

struct ScanShared {
    ScanState st;
    csvd_result res;
    int kcount;
    int pad;
};

// warp 0: per-prefix values of the chunk [q0, q1) from its summaries, then the
// state machine (scan.cuh).  reg_list: the k <= 32 running list (lane-held);
// la / lb: the k > 32 running list buffers (the live list stays in la).
__device__ __noinline__ void scan_chunk(const Dev &D, const Ord &o, ScanShared &ss, int q0, int q1,
                                        const double *c_topk, const double *c_lse, const double *c_min,
                                        const double *c_max, double *c_vals, double *la0, double *lb0,
                                        double &reg_list, int lane) {
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
    // streaming log Z_S: prefix-LSE of the cluster LSEs after the carry
    double im = act ? lse_q : -INFINITY, is = act ? 1.0 : 0.0;
#pragma unroll 1
    for (int s = 1; s < 32; s <<= 1) {
        const double m2 = __shfl_up_sync(CSVD_FULL, im, s), s2 = __shfl_up_sync(CSVD_FULL, is, s);
        if (lane >= s) {
            double mm = m2, sv = s2;
            lse_combine(mm, sv, im, is);
            im = mm;
            is = sv;
        }
    }
    {
        double mm = st0.log_z, sv = (st0.log_z == -INFINITY) ? 0.0 : 1.0;
        lse_combine(mm, sv, im, is);
        im = mm;
        is = sv;
    }
    double lz = (im == -INFINITY) ? -INFINITY : __dadd_rn(im, csvd_log(is));
    // the reference recomputes log Z_S over all of S when the merge count p % 64 == 0
    const int rlane = (q0 / 64) * 64 + 63 - q0;
    if (rlane < q1 - q0) {
        const double vmax = __shfl_sync(CSVD_FULL, pmx, rlane);
        const int ncum = __shfl_sync(CSVD_FULL, cnt_q, rlane);
        const double full = warp_lse_all(D.S_logits, ncum, vmax, lane);
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
    // k-th largest after each merge (exact): sequential list merges
    double my_kth = -INFINITY;
    int kc = ss.kcount;
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
    sc.run(chk);
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
    const int gwarp = blockIdx.x * WARPS + warp, nwarps = gridDim.x * WARPS;
    const size_t rb = (size_t)D.d * sizeof(ET);
    if (lane == 0) {  // every row of this warp in flight at once (L2 prefetch)
        for (int r = row_lo + gwarp; r < row_hi; r += nwarps) {
            int lo = p_lo, hi = p_hi;
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (o.cum[mid] <= r) lo = mid; else hi = mid;
            }
            const int pos = D.starts[o.order[lo]] + (r - o.cum[lo]);
            bulk_prefetch_l2(reinterpret_cast<const char *>(D.W) + (size_t)pos * rb, rb);
        }
    }
    for (int r = row_lo + gwarp; r < row_hi; r += nwarps) {
        int lo = p_lo, hi = p_hi;  // cum[lo] <= r < cum[lo+1]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (o.cum[mid] <= r) lo = mid; else hi = mid;
        }
        const int pos = D.starts[o.order[lo]] + (r - o.cum[lo]);
        const double logit = row_logit<ET, CPL, Q>(D, pos, hs, scratch, lane);
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
    const int gwarp = blockIdx.x * WARPS + warp, nwarps = gridDim.x * WARPS;
    const int k = D.cfg->k;
    double *mylist = D.cand + (size_t)gwarp * D.K;
    const bool small_k = k <= 32;
    double lv = -INFINITY;  // small k: lane l holds the l-th largest so far
    int cnt = 0;
    double kmin = -INFINITY;
    for (int pos = gwarp; pos < D.V; pos += nwarps) {
        const double logit = row_logit<ET, CPL, Q>(D, pos, hs, scratch, lane);
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
    }
    if (small_k) {
        if (lane < k) mylist[lane] = lv;
    } else if (lane == 0) {
        for (int i = cnt; i < k; ++i) mylist[i] = -INFINITY;
    }
}

// k-th largest over rows of `row_len` valid entries with stride `stride` (exact radix select)
__device__ __noinline__ double block_kth_largest(const double *vals, int n, int row_len, int stride, int k) {
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
__device__ __noinline__ void init_state(const Dev &D, const Ord &o, ScanShared &ss) {
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
    st.p_sel = (cfg.variant == CSVD_VARIANT_BATCHSELECT) ? csvd_select_prefix(in, cfg.k_max, search) : 0;
    st.p_cap = csvd_cap_prefix(in, st.p_sel, search);
    const long long wt = cfg.first_wave_tokens > 0 ? cfg.first_wave_tokens : 1;
    st.wave_tokens = (int)min(wt, (long long)D.V);
    const int c0 = o.order[0];
    st.est = (D.mode == CSVD_MODE_BIAS_AUGMENTED) ? __ldcg(D.dots + c0)
                                                  : __dadd_rn(__ldcg(D.dots + c0), D.meanb[c0]);
    st.p_lo = 0;
    st.p_hi = csvd_plan_wave(st, in, search);
    st.mode = MODE_SPARSE;
    st.wave_tokens = st.wave_tokens * 2 < D.V ? st.wave_tokens * 2 : (int)D.V;
    ss.st = st;
    memset(&ss.res, 0, sizeof(ss.res));
    ss.kcount = 0;
}

// after a wave's scan: done / dense / next wave (thread 0)
__device__ __noinline__ void next_wave(const Dev &D, const Ord &o, ScanShared &ss) {
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
    if (s2.phase == PH_DONE && blockIdx.x == 0) {
        csvd_result r = ss.res;
        r.query_norm = D.res->query_norm;
        r.slack = D.res->slack;
        r.waves = s2.iter;
        r.error = D.res->error;
        *D.res = r;
        *D.st = s2;
    }
}

// ---------------------------------------------------------------------------
// the step kernel
// ---------------------------------------------------------------------------
template <typename ET, int CPL, int Q, int BCPL, int BQ>
__global__ void __launch_bounds__(THREADS, 1) k_step(Dev D) {
    extern __shared__ __align__(16) double smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double *hs_w = smem;
    double *hs_b = D.hs_off_b ? smem + D.hs_off_b : smem;
    double *scratch = smem + D.scratch_off + warp * (CSVD_MAX_LEAVES / 4);
    double *ws = smem + D.ord_off;
    double *sws = smem + D.sum_off;
    __shared__ RankShared rs;
    __shared__ ScanShared ss;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    if (lead) DBG_TS(D, 0);
    if (D.launch_mode != LAUNCH_BOUNDS) pw_stage<CPL>(D.wplan, D.h, D.d, hs_w, D.wsrc);
    if (D.launch_mode == LAUNCH_BOUNDS || D.hs_off_b) pw_stage<BCPL>(D.bplan, D.h, D.d, hs_b, D.bsrc);
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
        bounds_phase<BCPL, BQ>(D, hs_b, scratch);
        if (lead) DBG_TS(D, 2);
        grid_sync(D);
        if (lead) DBG_TS(D, 3);
        const bool ok = rank_phase(D, ws, rs);
        if (lead) DBG_TS(D, 4);
        if (!ok || D.launch_mode == LAUNCH_BOUNDS) {
            grid_sync(D);  // final U visible before the host reads it
            if (lead) D.res->error = ok ? 0 : CSVD_EVALUE;
            return;
        }
        grid_sync(D);
        if (lead) DBG_TS(D, 5);
        load_ordering(D, o);
        if (threadIdx.x == 0) init_state(D, o, ss);
        __syncthreads();
        if (lead) DBG_TS(D, 6);
    }
    // chunk scratch: [6*CHUNK values][CHUNK lse][CHUNK min][CHUNK max][2 K-lists][chunk*k topk]
    double *c_vals = sws, *c_lse = sws + 6 * CHUNK, *c_min = c_lse + CHUNK, *c_max = c_min + CHUNK;
    double *la = c_max + CHUNK, *lb = la + D.K, *c_topk = lb + D.K;
    double reg_list = -INFINITY;
    for (int guard = 0; guard < D.C + 8; ++guard) {
        const ScanState st = ss.st;
        if (st.mode == MODE_IDLE || __ldcg(&D.res->error)) break;
        if (st.mode == MODE_SPARSE) {
            if (lead) DBG_TS(D, 8 + 4 * (st.iter & 3));
            wave_rows<ET, CPL, Q>(D, o, st.p_lo, st.p_hi, hs_w, scratch);
            grid_sync(D);
            if (lead) DBG_TS(D, 9 + 4 * (st.iter & 3));
            // summaries + scan, chunk by chunk (identical in every CTA)
            for (int q0 = st.p_lo; q0 < st.p_hi; q0 += D.chunk) {
                const int q1 = min(st.p_hi, q0 + D.chunk);
                for (int q = q0 + warp; q < q1; q += WARPS)
                    cluster_summary(D, o.cum[q], o.cum[q + 1], k, c_topk + (q - q0) * k, c_lse + (q - q0),
                                    c_min + (q - q0), c_max + (q - q0), lane);
                __syncthreads();
                if (lead) DBG_TS(D, 10 + 4 * (st.iter & 3));
                if (warp == 0) scan_chunk(D, o, ss, q0, q1, c_topk, c_lse, c_min, c_max, c_vals, la, lb, reg_list, lane);
                __syncthreads();
                if (ss.st.phase != PH_MAIN && ss.st.phase != PH_PE) break;
            }
            if (threadIdx.x == 0) next_wave(D, o, ss);
            __syncthreads();
            if (lead) DBG_TS(D, 11 + 4 * (st.iter & 3));
        } else {  // MODE_DENSE
            dense_rows<ET, CPL, Q>(D, hs_w, scratch);
            grid_sync(D);
            if (blockIdx.x != 0) break;
            const double kth = block_kth_largest(D.cand, D.nblocks * WARPS * k, k, D.K, k);
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
            }
            break;
        }
    }
}
