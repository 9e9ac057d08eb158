// csvd_b200: B200-native (sm_100a) CSV-Decode output-layer step.
//
// One step = one CUDA-graph replay:
//
//   k_bounds   (all SMs)  U_c = ((<mu_c,h> + R_c*||h||) + maxb_c) for every cluster,
//                         bit-exact f64 (bounds.py:79-83); the LAST CTA to finish
//                         then sorts (-U, id) (decode.py:166), builds the prefix
//                         token counts, the suffix log-sum-exp table
//                         log R-hat(p) (certify.py:114-119), and plans wave 1.
//   WHILE(cond) {
//     k_wave   (all SMs)  sparse: gathered GEMV over the wave's rows (W stored
//                         permuted, so every cluster is a contiguous row range),
//                         logits bit-exact f64 (decode.py:169-176); the last warp of
//                         each cluster writes its summary (top-k, LSE, min, max);
//                         the last cluster's warp runs the certification scan
//                         (scan.cuh) and either finishes, plans the next wave, or
//                         switches to dense mode.
//                         dense: full-vocabulary GEMV (decode.py:239-262) scattered
//                         to original token order + per-warp top-k candidates; the
//                         last CTA radix-selects the k-th logit and finishes.
//   }
//
// No spin-waits anywhere: cross-CTA hand-off is "last arriver continues"
// (threadfence + atomic ticket).  The WHILE loop is guarded by an iteration cap.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/csvd_b200.h"
#include "pw.cuh"
#include "scan.cuh"

#define WARPS 8
#define THREADS (WARPS * 32)

// ---------------------------------------------------------------------------
// device-side step description
// ---------------------------------------------------------------------------
struct Dev {
    int V, d, C, bd, mode, wdtype;
    int K;        // top-k capacity (row stride of sum_topk / cand)
    int cpad;     // next pow2 >= C (sort)
    const void *W;            // [V, d] permuted rows
    const float *bias;        // [V] permuted
    const int *perm;          // [V] position -> token id
    const double *cent;       // [C, bd]
    const double *radii, *maxb, *cnorm, *ang, *maxn, *minn, *logsz, *meanb;
    const int *starts, *sizes;
    PwPlan wplan, bplan;
    // per step
    const double *h;          // [d]
    const csvd_config *cfg;
    double *U, *X, *dots;     // [C] by cluster id
    double *Uo;               // [C] bounds in opening order
    int *order;               // [C]
    int *cum;                 // [C+1]
    double *lrh;              // [C+1]
    int *cl_done;             // [C]
    double *sum_topk;         // [C*K]
    double *sum_lse, *sum_min, *sum_max;  // [C]
    double *S_logits;         // [V]
    long long *S_ids;         // [V]
    double *run_a, *run_b;    // [K] (global copies of the running list)
    double *cand;             // [nwarps_wave * K]
    ScanState *st;
    csvd_result *res;
    unsigned int *counters;   // [0] bounds CTAs, [1] wave clusters, [2] dense CTAs
    cudaGraphConditionalHandle loop;
    int scan_smem_doubles;    // dynamic smem of k_wave, in doubles
    unsigned long long *dbg;  // optional phase timestamps
    int use_graph;            // 1 -> set the conditional handle
    int bounds_only;          // 1 -> skip ordering/planning
    int dense_only;           // 1 -> (dense API) start directly in dense mode
};

// ---------------------------------------------------------------------------
// small device helpers
// ---------------------------------------------------------------------------
// debug phase timestamps (%globaltimer, ns), enabled by CSVD_DEBUG_TS=1
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define DBG_TS(D, slot)                                              \
    do {                                                             \
        if ((D).dbg) (D).dbg[(slot)] = gtimer();                     \
    } while (0)
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

template <typename ET, int CPL, int Q>
__device__ __forceinline__ double row_logit(const Dev &D, int pos, const double *hs, double *scratch, int lane) {
    const ET *row = reinterpret_cast<const ET *>(D.W) + (size_t)pos * D.d;
    double dot = warp_dot_t<ET, CPL, Q>(row, hs, D.wplan, scratch, lane);
    return __dadd_rn(dot, (double)__ldg(D.bias + pos));
}

__device__ __forceinline__ double set_cond(const Dev &D, unsigned v) {
    if (D.use_graph) cudaGraphSetConditional(D.loop, v);
    return 0.0;
}

// ---------------------------------------------------------------------------
// warp-level primitives for the scan
// ---------------------------------------------------------------------------
struct WarpSearch {
    // first i in [lo, hi) with pred(i) true (pred monotone), or hi.
    // 32 probes per round, so ~2 dependent rounds for C <= 1024.
    template <class F>
    __device__ int operator()(int lo, int hi, const F &pred) const {
        const int lane = threadIdx.x & 31;
        while (hi - lo > 32) {
            const int step = (hi - lo + 31) / 32;
            const int probe = lo + lane * step;
            const bool t = probe < hi ? pred(probe) : true;
            const unsigned m = __ballot_sync(CSVD_FULL, t);
            if (m == 0) {
                lo = lo + 31 * step + 1;
            } else {
                const int f = __ffs(m) - 1;
                const int pf = lo + f * step;
                const int nlo = f == 0 ? lo : lo + (f - 1) * step + 1;
                hi = pf < hi ? pf : hi;
                lo = nlo;
            }
        }
        const int probe = lo + lane;
        const bool t = probe < hi ? pred(probe) : true;
        const unsigned m = __ballot_sync(CSVD_FULL, t);
        return m == 0 ? hi : lo + (__ffs(m) - 1);
    }
};

struct WarpPrims {
    int lane;
    double *bbuf;  // unused (lists are prefetched into shared memory)
    // top-k of union of two descending lists (values only), warp-parallel
    // merge-path: element i of A lands at i + #{B > A[i]}, element j of B at
    // j + #{A >= B[j]}.
    __device__ int merge_topk(const double *A, int ka, const double *B, int kb, int k, double *out) {
        for (int i = lane; i < ka; i += 32) {
            double a = A[i];
            int lo = 0, hi = kb;  // count B > a
            while (lo < hi) {
                int m = (lo + hi) >> 1;
                if (B[m] > a) lo = m + 1; else hi = m;
            }
            int pos = i + lo;
            if (pos < k) out[pos] = a;
        }
        for (int j = lane; j < kb; j += 32) {
            double b = B[j];
            int lo = 0, hi = ka;  // count A >= b
            while (lo < hi) {
                int m = (lo + hi) >> 1;
                if (A[m] >= b) lo = m + 1; else hi = m;
            }
            int pos = j + lo;
            if (pos < k) out[pos] = b;
        }
        __syncwarp();
        int n = ka + kb;
        return n < k ? n : k;
    }
    __device__ double lse_all(const double *vals, int n, double vmax) {
        if (n == 0) return -INFINITY;
        if (vmax == -INFINITY) return -INFINITY;
        if (vmax == INFINITY) return INFINITY;
        double s = 0.0;
        for (int i = lane; i < n; i += 32) s = __dadd_rn(s, exp(__dsub_rn(__ldcg(vals + i), vmax)));
        s = warp_sum(s);
        return __dadd_rn(vmax, log(s));
    }
};

// ---------------------------------------------------------------------------
// cluster summary (warp): top-min(k,n) values desc, LSE, min, max
// ---------------------------------------------------------------------------
__device__ __noinline__ void cluster_summary(const Dev &D, int q, int lane) {
    const int lo = D.cum[q], hi = D.cum[q + 1];
    const int n = hi - lo;
    const double *v = D.S_logits + lo;
    const int k = D.cfg->k;
    const int kk = n < k ? n : k;
    constexpr int E = 8;
    double reg[E];
    const bool in_regs = n <= 32 * E;
    double mx = -INFINITY, mn = INFINITY;
    if (in_regs) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
            int i = lane + 32 * e;
            reg[e] = i < n ? __ldcg(v + i) : -INFINITY;
            if (i < n) { mx = fmax(mx, reg[e]); mn = fmin(mn, reg[e]); }
        }
    } else {
        for (int i = lane; i < n; i += 32) {
            double x = __ldcg(v + i);
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
            if (lane + 32 * e < n) s = __dadd_rn(s, exp(__dsub_rn(reg[e], mx)));
    } else {
        for (int i = lane; i < n; i += 32) s = __dadd_rn(s, exp(__dsub_rn(__ldcg(v + i), mx)));
    }
    s = warp_sum(s);
    double lse = (mx == -INFINITY) ? -INFINITY : __dadd_rn(mx, log(s));
    // iterative selection in (value desc, index asc) order
    double pv = INFINITY;
    int pi = -1;
    double *out = D.sum_topk + (size_t)q * D.K;
    for (int j = 0; j < kk; ++j) {
        double bv = -INFINITY;
        int bi = 0x7fffffff;
        if (in_regs) {
#pragma unroll
            for (int e = 0; e < E; ++e) {
                int i = lane + 32 * e;
                if (i < n) {
                    double x = reg[e];
                    bool after = (x < pv) || (x == pv && i > pi);
                    if (after && (x > bv || (x == bv && i < bi))) { bv = x; bi = i; }
                }
            }
        } else {
            for (int i = lane; i < n; i += 32) {
                double x = __ldcg(v + i);
                bool after = (x < pv) || (x == pv && i > pi);
                if (after && (x > bv || (x == bv && i < bi))) { bv = x; bi = i; }
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            double ov = __shfl_xor_sync(CSVD_FULL, bv, o);
            int oi = __shfl_xor_sync(CSVD_FULL, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
        }
        if (lane == 0) out[j] = bv;
        pv = bv;
        pi = bi;
    }
    if (lane == 0) {
        D.sum_lse[q] = lse;
        D.sum_min[q] = mn;
        D.sum_max[q] = mx;
    }
}

// prepare counters / state for wave [p_lo, p_hi)
__device__ void start_wave(const Dev &D, ScanState &st, int p_hi) {
    st.p_lo = st.p;
    st.p_hi = p_hi;
    st.row_lo = D.cum[st.p];
    st.row_hi = D.cum[p_hi];
    st.mode = MODE_SPARSE;
}

// ---------------------------------------------------------------------------
// block radix select: k-th largest of vals[0..n) (exact, any k <= n)
// ---------------------------------------------------------------------------
// vals viewed as n/row_len rows of row_len entries with stride `stride`
__device__ double block_kth_largest(const double *vals, int n, int row_len, int stride, unsigned *hist,
                                    unsigned long long *shared_prefix, int *shared_k, int k) {
    unsigned long long prefix = 0, mask = 0;
    int kk = k;
    for (int shift = 56; shift >= 0; shift -= 8) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            unsigned long long key = dkey(__ldcg(vals + (size_t)(i / row_len) * stride + (i % row_len)));
            if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned cumc = 0;
            int digit = 0;
            for (int b = 255; b >= 0; --b) {
                if (cumc + hist[b] >= (unsigned)kk) { digit = b; kk -= (int)cumc; break; }
                cumc += hist[b];
            }
            *shared_prefix = prefix | ((unsigned long long)digit << shift);
            *shared_k = kk;
        }
        __syncthreads();
        prefix = *shared_prefix;
        kk = *shared_k;
        mask |= (255ull << shift);
        __syncthreads();
    }
    return dkey_inv(prefix);
}

// ---------------------------------------------------------------------------
// K1: bounds (+ last CTA: order, prefix counts, suffix LSE, wave-1 plan)
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

__device__ __noinline__ void last_cta_order(const Dev &D, double *smem, double qn);

template <int CPL, int Q>
__global__ void __launch_bounds__(THREADS) k_bounds(Dev D) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double *hs = smem;                       // bd doubles
    double *scratch = smem + D.bd + warp * CSVD_MAX_LEAVES / 4;  // generic leaf sums
    __shared__ double s_qn;
    __shared__ int s_last;
    if (blockIdx.x == 0 && threadIdx.x == 0) DBG_TS(D, 0);
    pw_stage_h(D.bplan, D.h, D.d, hs);
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) DBG_TS(D, 1);
    if (warp == 0) {
        double ss;
        if constexpr (CPL > 0) {
            ss = warp_dot_t<double, CPL, Q>(D.h, hs, D.bplan, scratch, lane);
        } else {
            struct HH {
                const double *hs;
                __device__ double operator()(int e) const { return __dmul_rn(hs[e], hs[e]); }
            } f{hs};
            ss = warp_dot_generic(f, D.bplan, scratch, lane);
        }
        if (lane == 0) s_qn = __dsqrt_rn(ss);
    }
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) DBG_TS(D, 2);
    const double qn = s_qn;
    for (int c = blockIdx.x * WARPS + warp; c < D.C; c += gridDim.x * WARPS) {
        double dot = warp_dot_t<double, CPL, Q>(D.cent + (size_t)c * D.bd, hs, D.bplan, scratch, lane);
        if (lane == 0) {
            double u;
            if (D.mode == CSVD_MODE_SPHERICAL)
                u = cone_bound(D, c, dot, qn);
            else if (D.mode == CSVD_MODE_BIAS_AUGMENTED)
                u = __dadd_rn(dot, __dmul_rn(D.radii[c], qn));
            else
                u = __dadd_rn(__dadd_rn(dot, __dmul_rn(D.radii[c], qn)), D.maxb[c]);
            D.U[c] = u;
            D.dots[c] = dot;
        }
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned t = atomicAdd(&D.counters[0], 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) DBG_TS(D, 3);
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x == 0) {
        D.counters[0] = 0;
        DBG_TS(D, 4);
    }
    last_cta_order(D, smem, qn);
    if (threadIdx.x == 0) DBG_TS(D, 9);
}

// Suffix log-sum-exp combine: (m, s) represents m + log(s)
__device__ __forceinline__ void lse_combine(double &m, double &s, double m2, double s2) {
    if (m2 == -INFINITY) return;
    if (m == -INFINITY) { m = m2; s = s2; return; }
    if (m2 > m) {
        s = __dadd_rn(__dmul_rn(s, exp(__dsub_rn(m, m2))), s2);
        m = m2;
    } else {
        s = __dadd_rn(s, __dmul_rn(s2, exp(__dsub_rn(m2, m))));
    }
}

// Shared-memory layout of the last CTA (all sizes padded to cpad):
//   keyU[cpad] f64  sorted bounds (= Uo)      keyI[cpad] i32  order
//   cumS[cpad+1] i32 prefix token counts      lrhS[cpad+1] f64 suffix LSE
__device__ __noinline__ void last_cta_order(const Dev &D, double *smem, double qn) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const csvd_config &cfg = *D.cfg;
    const int C = D.C;
    const int n = D.cpad;
    double *keyU = smem;
    double *lrhS = smem + n;
    int *keyI = reinterpret_cast<int *>(smem + 2 * n + 1);
    int *cumS = keyI + n;
    __shared__ double s_red[THREADS];
    __shared__ int s_flag;
    // --- slack (bounds.py:58-64) + finiteness (bounds.py:53-55)
    double amax = 1.0;
    int bad = 0;
    for (int c = tid; c < C; c += nt) {
        double u = __ldcg(D.U + c);
        amax = fmax(amax, fabs(u));
        if (!isfinite(u)) bad = 1;
    }
    s_red[tid] = amax;
    if (tid == 0) s_flag = 0;
    __syncthreads();
    if (bad) atomicOr(&s_flag, 1);
    for (int o = nt / 2; o; o >>= 1) {
        if (tid < o) s_red[tid] = fmax(s_red[tid], s_red[tid + o]);
        __syncthreads();
    }
    double eta = 0.0;
    if (cfg.slack_f32) eta = __dmul_rn(__dmul_rn(4.0, 1.1920928955078125e-07), s_red[0]);
    // --- final U, X = log|c| + U (certify.py:119 order), sort keys
    for (int c = tid; c < n; c += nt) {
        if (c < C) {
            double u = __dadd_rn(__ldcg(D.U + c), eta);
            if (!isfinite(u)) atomicOr(&s_flag, 1);
            D.U[c] = u;
            D.X[c] = __dadd_rn(D.logsz[c], u);
            keyU[c] = u;
            keyI[c] = c;
        } else {
            keyU[c] = -INFINITY;
            keyI[c] = 0x7fffffff;
        }
    }
    __syncthreads();
    if (tid == 0) {
        D.res->query_norm = qn;
        D.res->slack = eta;
    }
    if (s_flag || D.bounds_only) {
        if (tid == 0) {
            if (s_flag) D.res->error = CSVD_EVALUE;
            D.st->phase = s_flag ? PH_ERROR : PH_DONE;
            D.st->mode = MODE_IDLE;
            set_cond(D, 0);
        }
        return;
    }
    if (tid == 0) DBG_TS(D, 5);
    // --- bitonic sort: descending U, ascending id  (np.lexsort((arange, -U)))
    for (int size = 2; size <= n; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int t = tid; t < n / 2; t += nt) {
                int lo = 2 * t - (t & (stride - 1));
                int hi = lo + stride;
                bool desc = ((lo & size) == 0);
                double ua = keyU[lo], ub = keyU[hi];
                int ia = keyI[lo], ib = keyI[hi];
                bool a_first = (ua > ub) || (ua == ub && ia < ib);
                if (a_first != desc) {
                    keyU[lo] = ub; keyU[hi] = ua;
                    keyI[lo] = ib; keyI[hi] = ia;
                }
            }
            __syncthreads();
        }
    }
    if (tid == 0) DBG_TS(D, 6);
    // --- order, Uo, prefix token counts (block scan over contiguous chunks)
    __shared__ int s_scan[THREADS];
    const int per = (C + nt - 1) / nt;
    const int b0 = min(C, tid * per), b1 = min(C, b0 + per);
    int local = 0;
    for (int p = b0; p < b1; ++p) local += D.sizes[keyI[p]];
    s_scan[tid] = local;
    __syncthreads();
    for (int o = 1; o < nt; o <<= 1) {
        int v = tid >= o ? s_scan[tid - o] : 0;
        __syncthreads();
        s_scan[tid] += v;
        __syncthreads();
    }
    int run = s_scan[tid] - local;
    for (int p = b0; p < b1; ++p) {
        cumS[p] = run;
        run += D.sizes[keyI[p]];
    }
    if (tid == nt - 1) cumS[C] = s_scan[nt - 1];
    // --- suffix log-sum-exp over x[order[q]], q >= p  -> lrh[p]
    __shared__ double s_m[THREADS], s_s[THREADS];
    double m = -INFINITY, sm = 0.0;
    for (int p = b1 - 1; p >= b0; --p) lse_combine(m, sm, __ldcg(D.X + keyI[p]), 1.0);
    s_m[tid] = m;
    s_s[tid] = sm;
    __syncthreads();
    for (int o = 1; o < nt; o <<= 1) {
        double m2 = -INFINITY, s2 = 0.0;
        if (tid + o < nt) { m2 = s_m[tid + o]; s2 = s_s[tid + o]; }
        __syncthreads();
        double mm = s_m[tid], ss = s_s[tid];
        lse_combine(mm, ss, m2, s2);
        s_m[tid] = mm;
        s_s[tid] = ss;
        __syncthreads();
    }
    m = (tid + 1 < nt) ? s_m[tid + 1] : -INFINITY;
    sm = (tid + 1 < nt) ? s_s[tid + 1] : 0.0;
    for (int p = b1 - 1; p >= b0; --p) {
        lse_combine(m, sm, __ldcg(D.X + keyI[p]), 1.0);
        lrhS[p] = (m == -INFINITY) ? -INFINITY : __dadd_rn(m, log(sm));
    }
    if (tid == 0) lrhS[C] = -INFINITY;
    __syncthreads();
    if (tid == 0) DBG_TS(D, 7);
    // --- publish order / Uo / cum / lrh, reset per-cluster counters
    for (int p = tid; p < C; p += nt) {
        D.order[p] = keyI[p];
        D.Uo[p] = keyU[p];
        D.cum[p] = cumS[p];
        D.lrh[p] = lrhS[p];
        D.cl_done[p] = 0;
    }
    if (tid == 0) {
        D.cum[C] = cumS[C];
        D.lrh[C] = lrhS[C];
    }
    // --- init scan state + plan wave 1 (thread 0, from shared memory)
    if (tid == 0) {
        DBG_TS(D, 8);
        ScanState st;
        memset(&st, 0, sizeof(st));
        st.phase = PH_MAIN;
        st.log_z = -INFINITY;
        st.smin = INFINITY;
        st.smax = -INFINITY;
        ScanIn in{D.cfg, C, (long long)D.V, D.d, cumS, keyU, lrhS, nullptr, nullptr, nullptr, nullptr, D.K, nullptr};
        ScalarSearch search;
        st.p_sel = (cfg.variant == CSVD_VARIANT_BATCHSELECT) ? csvd_select_prefix(in, cfg.k_max, search) : 0;
        st.p_cap = csvd_cap_prefix(in, st.p_sel, search);
        long long wt = cfg.first_wave_tokens > 0 ? cfg.first_wave_tokens : 1;
        st.wave_tokens = (int)min(wt, (long long)D.V);
        const int c0 = keyI[0];
        st.est = (D.mode == CSVD_MODE_BIAS_AUGMENTED) ? __ldcg(D.dots + c0) : __dadd_rn(__ldcg(D.dots + c0), D.meanb[c0]);
        int hi = csvd_plan_wave(st, in, search);
        st.p_lo = 0;
        st.p_hi = hi;
        st.row_lo = 0;
        st.row_hi = cumS[hi];
        st.mode = MODE_SPARSE;
        st.wave_tokens = st.wave_tokens * 2 < D.V ? st.wave_tokens * 2 : (int)D.V;
        *D.st = st;
        D.counters[1] = 0;
        D.res->error = 0;
        D.res->waves = 0;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) set_cond(D, 1);
}

// ---------------------------------------------------------------------------
// K2: wave (sparse gathered GEMV + summaries + scan)  /  dense GEMV
// ---------------------------------------------------------------------------
template <typename ET, int CPL, int Q>
__device__ void wave_sparse(const Dev &D, const ScanState &st0, double *hs, double *scratch, double *smem_base,
                            int lane, int gwarp, int nwarps);
template <typename ET, int CPL, int Q>
__device__ void wave_dense(const Dev &D, const ScanState &st0, double *hs, double *scratch, double *smem_base,
                           int lane, int gwarp, int nwarps);

template <typename ET, int CPL, int Q>
__global__ void __launch_bounds__(THREADS) k_wave(Dev D) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gwarp = blockIdx.x * WARPS + warp, nwarps = gridDim.x * WARPS;
    const ScanState st0 = *D.st;  // written by the previous kernel in the stream
    if (st0.mode == MODE_IDLE || st0.iter > D.C + 8) {  // guard: never loop forever
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            if (st0.mode != MODE_IDLE) D.res->error = CSVD_ESTATE;
            set_cond(D, 0);
        }
        return;
    }
    double *hs = smem;
    double *scratch = smem + D.d + warp * (CSVD_MAX_LEAVES / 4);
    if (blockIdx.x == 0 && threadIdx.x == 0) DBG_TS(D, 16 + 8 * (st0.iter & 1));
    pw_stage_h(D.wplan, D.h, D.d, hs);
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x == 0) DBG_TS(D, 17 + 8 * (st0.iter & 1));
    if (st0.mode == MODE_SPARSE)
        wave_sparse<ET, CPL, Q>(D, st0, hs, scratch, smem, lane, gwarp, nwarps);
    else
        wave_dense<ET, CPL, Q>(D, st0, hs, scratch, smem, lane, gwarp, nwarps);
}

__device__ __noinline__ void run_scan(const Dev &D, const ScanState &st0, double *smem_base, int lane) {
    // All wave clusters are summarised; this warp owns the sequential scan.
    // Every lane runs the identical scalar state machine (uniform control
    // flow); collective primitives are warp-parallel; lane 0 writes state.
    // Inputs are prefetched chunk by chunk into shared memory with one round
    // of parallel loads, so the sequential part never waits on L2.
    ScanState st = st0;
    csvd_result res;
    memset(&res, 0, sizeof(res));
    const int K = D.K;
    const int k = D.cfg->k;
    if (lane == 0) DBG_TS(D, 19 + 8 * (st0.iter & 1));
    double *ra = smem_base, *rb = smem_base + K;
    double *chunk = smem_base + 2 * K;
    int M = (D.scan_smem_doubles - 2 * K - 8) / (k + 6);
    if (M > 64) M = 64;
    if (M < 1) M = 1;
    double *Uo_s = chunk, *lrh_s = chunk + (M + 1), *lse_s = chunk + 2 * (M + 1);
    double *min_s = lse_s + M, *max_s = min_s + M, *topk_s = max_s + M;
    int *cum_s = reinterpret_cast<int *>(topk_s + (size_t)M * k);
    for (int i = lane; i < st.kcount; i += 32) ra[i] = __ldcg(D.run_a + i);
    __syncwarp();
    double *run = ra, *run_alt = rb;
    WarpPrims prims{lane, nullptr};
    int q0 = st.p;
    while (q0 < st.p_hi && (st.phase == PH_MAIN || st.phase == PH_PE)) {
        const int q1 = min(st.p_hi, q0 + M);
        const int nq = q1 - q0;
        for (int i = lane; i <= nq; i += 32) {
            const int q = q0 + i;
            cum_s[i] = __ldcg(D.cum + q);
            Uo_s[i] = q < D.C ? __ldcg(D.Uo + q) : -INFINITY;
            lrh_s[i] = __ldcg(D.lrh + q);
            if (i < nq) {
                lse_s[i] = __ldcg(D.sum_lse + q);
                min_s[i] = __ldcg(D.sum_min + q);
                max_s[i] = __ldcg(D.sum_max + q);
            }
        }
        for (int e = lane; e < nq * k; e += 32) {
            const int i = e / k, j = e - i * k;
            topk_s[e] = __ldcg(D.sum_topk + (size_t)(q0 + i) * K + j);
        }
        __syncwarp();
        ScanIn in{D.cfg, D.C, (long long)D.V, D.d, cum_s - q0, Uo_s - q0, lrh_s - q0, lse_s - q0, min_s - q0,
                  max_s - q0, topk_s - (size_t)q0 * k, k, D.S_logits};
        Scan<WarpPrims> sc{in, st, run, run_alt, prims, res};
        sc.run(q1);
        __syncwarp();
        q0 = q1;
    }
    st.iter += 1;
    if (lane == 0) DBG_TS(D, 20 + 8 * (st0.iter & 1));
    for (int i = lane; i < st.kcount; i += 32) D.run_a[i] = run[i];
    if (st.phase == PH_DONE) {
        if (lane == 0) {
            res.query_norm = D.res->query_norm;
            res.slack = D.res->slack;
            res.waves = st.iter;
            res.error = 0;
            *D.res = res;
            st.mode = MODE_IDLE;
            *D.st = st;
            set_cond(D, 0);
        }
    } else if (st.phase == PH_DENSE) {
        if (lane == 0) {
            st.mode = MODE_DENSE;
            *D.st = st;
            D.counters[2] = 0;
            set_cond(D, 1);
        }
    } else {  // need more clusters: plan the next wave (all lanes, identical)
        ScanIn gin{D.cfg, D.C, (long long)D.V, D.d, D.cum, D.Uo, D.lrh, nullptr, nullptr, nullptr, nullptr, K,
                   nullptr};
        int hi = csvd_plan_wave(st, gin, WarpSearch{});
        start_wave(D, st, hi);
        st.wave_tokens = st.wave_tokens * 2 < D.V ? st.wave_tokens * 2 : (int)D.V;
        for (int q = st.p_lo + lane; q < st.p_hi; q += 32) D.cl_done[q] = 0;
        if (lane == 0) {
            *D.st = st;
            D.counters[1] = 0;
            set_cond(D, 1);
        }
    }
    __threadfence();
    if (lane == 0) DBG_TS(D, 21 + 8 * (st0.iter & 1));
}

template <typename ET, int CPL, int Q>
__device__ void wave_sparse(const Dev &D, const ScanState &st0, double *hs, double *scratch, double *smem_base,
                            int lane, int gwarp, int nwarps) {
    const int p_lo = st0.p_lo, p_hi = st0.p_hi;
    const int nclusters = p_hi - p_lo;
    for (int r = st0.row_lo + gwarp; r < st0.row_hi; r += nwarps) {
        // prefix q containing row r: cum[q] <= r < cum[q+1]
        int lo = p_lo, hi = p_hi;
        while (hi - lo > 1) {
            int mid = (lo + hi) >> 1;
            if (__ldg(D.cum + mid) <= r) lo = mid; else hi = mid;
        }
        const int q = lo;
        const int c = __ldg(D.order + q);
        const int off = r - __ldg(D.cum + q);
        const int pos = __ldg(D.starts + c) + off;
        double logit = row_logit<ET, CPL, Q>(D, pos, hs, scratch, lane);
        if (gwarp == 0 && lane == 0) DBG_TS(D, 22 + 8 * (st0.iter & 1));
        int last = 0;
        if (lane == 0) {
            D.S_logits[r] = logit;
            D.S_ids[r] = (long long)__ldg(D.perm + pos);
            __threadfence();
            unsigned t = atomicAdd((unsigned *)&D.cl_done[q], 1u);
            last = (t == (unsigned)__ldg(D.sizes + c) - 1u);
        }
        last = __shfl_sync(CSVD_FULL, last, 0);
        if (last) {
            __threadfence();
            cluster_summary(D, q, lane);
            __threadfence();
            int final_ = 0;
            if (lane == 0) {
                unsigned t = atomicAdd(&D.counters[1], 1u);
                final_ = (t == (unsigned)nclusters - 1u);
            }
            final_ = __shfl_sync(CSVD_FULL, final_, 0);
            if (final_) {
                if (lane == 0) DBG_TS(D, 18 + 8 * (st0.iter & 1));
                __threadfence();
                // all rows of the wave are done -> no other warp of this CTA
                // still reads hs; reuse shared memory for the scan
                run_scan(D, st0, smem_base, lane);
            }
        }
    }
}

template <typename ET, int CPL, int Q>
__device__ void wave_dense(const Dev &D, const ScanState &st0, double *hs, double *scratch, double *smem_base,
                           int lane, int gwarp, int nwarps) {
    const int k = D.cfg->k;
    double *mylist = D.cand + (size_t)gwarp * D.K;
    int cnt = 0;
    double kmin = -INFINITY;  // current k-th of the warp list once full
    for (int pos = gwarp; pos < D.V; pos += nwarps) {
        double logit = row_logit<ET, CPL, Q>(D, pos, hs, scratch, lane);
        if (lane == 0) {
            int tok = __ldg(D.perm + pos);
            D.S_logits[tok] = logit;
            D.S_ids[tok] = tok;
            // sorted (desc) insertion into the warp's top-k candidate list
            if (cnt < k || logit > kmin) {
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
    }
    // pad unused entries with -inf: the k-th largest over the union of the
    // per-warp lists equals the k-th largest of all V logits (V >= k)
    if (lane == 0)
        for (int i = cnt; i < k; ++i) mylist[i] = -INFINITY;
    __threadfence();
    __syncthreads();
    __shared__ int s_last;
    if (threadIdx.x == 0) {
        unsigned t = atomicAdd(&D.counters[2], 1u);
        s_last = (t == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    __shared__ unsigned hist[256];
    __shared__ unsigned long long s_pref;
    __shared__ int s_k;
    double kth = block_kth_largest(D.cand, nwarps * k, k, D.K, hist, &s_pref, &s_k, k);
    if (threadIdx.x == 0) {
        ScanState st = st0;
        csvd_result res;
        memset(&res, 0, sizeof(res));
        ScanIn in{D.cfg, D.C, (long long)D.V, D.d, D.cum, D.Uo, D.lrh, nullptr, nullptr, nullptr, nullptr, D.K,
                  nullptr};
        double *dummy = nullptr;
        WarpPrims prims{0, nullptr};
        Scan<WarpPrims> sc{in, st, dummy, dummy, prims, res};
        sc.finish_dense(kth);
        res.query_norm = D.res->query_norm;
        res.slack = D.res->slack;
        res.waves = st.iter + 1;
        *D.res = res;
        st.mode = MODE_IDLE;
        *D.st = st;
        set_cond(D, 0);
    }
}

// dense-only API: reset state so k_wave runs the dense GEMV once
__global__ void k_dense_setup(Dev D) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        ScanState st;
        memset(&st, 0, sizeof(st));
        st.mode = MODE_DENSE;
        st.phase = PH_DENSE;
        *D.st = st;
        D.counters[2] = 0;
        set_cond(D, 1);
    }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
struct csvd_ctx {
    int device = 0;
    Dev D{};
    std::string err;
    cudaStream_t stream = nullptr;
    // owned device buffers
    std::vector<void *> dev_allocs;
    void *k_buffers[6] = {};  // K-dependent: sum_topk, run_a, run_b, cand
    int grid_bounds = 0, grid_wave = 0;
    size_t smem_bounds = 0, smem_wave = 0;
    csvd_config *d_cfg = nullptr;
    double *d_h = nullptr;
    // pinned staging
    double *h_pin = nullptr;
    csvd_config *cfg_pin = nullptr;
    csvd_result *res_pin = nullptr;
    long long *ids_pin = nullptr;
    double *logits_pin = nullptr;
    int64_t pin_cap = 0;
    // graphs
    cudaGraphExec_t g_step = nullptr, g_bounds = nullptr, g_dense = nullptr;
    cudaGraphConditionalHandle h_step = 0, h_bounds = 0, h_dense = 0;
    int last_launches = 0;
    int direct = 0;               // 1: launch kernels one by one (profiling / ncu)
    void *flush_buf = nullptr;
    ScanState *st_pin = nullptr;
    // host copies of plan tables
    std::vector<int2> wleaves, bleaves;
    std::vector<short> wprog, bprog;
};

static int fail(csvd_ctx *c, int code, const std::string &msg) {
    if (c) c->err = msg;
    return code;
}

#define CK(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess)                                                                    \
            return fail(ctx, CSVD_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
    } while (0)

// numpy pairwise tree enumeration (oracle/pairwise.c restatement)
static void pw_enumerate(int off, int n, std::vector<int2> &leaves, std::vector<short> &prog, bool &balanced) {
    if (n <= 128) {
        prog.push_back((short)leaves.size());
        leaves.push_back(make_int2(off, n));
        return;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    if (n2 * 2 != n) balanced = false;
    pw_enumerate(off, n2, leaves, prog, balanced);
    pw_enumerate(off + n2, n - n2, leaves, prog, balanced);
    prog.push_back(-1);
}

static void make_plan(int n, PwPlan &pl, std::vector<int2> &leaves, std::vector<short> &prog) {
    memset(&pl, 0, sizeof(pl));
    pl.n = n;
    leaves.clear();
    prog.clear();
    bool balanced = true;
    pw_enumerate(0, n, leaves, prog, balanced);
    int nl = (int)leaves.size();
    int L = leaves[0].y;
    bool equal = true;
    for (auto &lf : leaves) equal = equal && (lf.y == L);
    bool pow2 = (nl & (nl - 1)) == 0;
    if (balanced && equal && pow2 && L % 8 == 0 && L >= 8 && nl >= 4 && nl <= 128) {
        pl.regular = 1;
        pl.leaf_len = L;
        pl.steps = L / 8;
        if (nl >= 32) {
            pl.cpl = 8;
            pl.q = nl / 32;
        } else {
            pl.cpl = 8 / (32 / nl);
            pl.q = 1;
        }
    }
    pl.nleaf = nl;
    pl.nprog = (int)prog.size();
}

template <typename T>
static int dalloc(csvd_ctx *ctx, T **p, size_t count) {
    void *q = nullptr;
    cudaError_t e = cudaMalloc(&q, count * sizeof(T) + 16);
    if (e != cudaSuccess) return fail(ctx, CSVD_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    ctx->dev_allocs.push_back(q);
    *p = reinterpret_cast<T *>(q);
    return 0;
}

template <typename T>
static int dupload(csvd_ctx *ctx, T **p, const T *src, size_t count) {
    int rc = dalloc(ctx, p, count);
    if (rc) return rc;
    CK(cudaMemcpy(*p, src, count * sizeof(T), cudaMemcpyHostToDevice));
    return 0;
}

// permute rows on device: dst[pos] = src[perm[pos]]
__global__ void k_permute_rows(const char *src, char *dst, const long long *perm, long long V, long long row_bytes) {
    for (long long pos = blockIdx.x; pos < V; pos += gridDim.x) {
        const char *s = src + perm[pos] * row_bytes;
        char *t = dst + pos * row_bytes;
        for (long long b = threadIdx.x * 16; b < row_bytes; b += blockDim.x * 16) {
            if (b + 16 <= row_bytes)
                *reinterpret_cast<uint4 *>(t + b) = *reinterpret_cast<const uint4 *>(s + b);
            else
                for (long long j = b; j < row_bytes; ++j) t[j] = s[j];
        }
    }
}

static int alloc_k(csvd_ctx *ctx, int K) {
    Dev &D = ctx->D;
    for (int i = 0; i < 6; ++i)
        if (ctx->k_buffers[i]) cudaFree(ctx->k_buffers[i]);
    memset(ctx->k_buffers, 0, sizeof(ctx->k_buffers));
    size_t nw = (size_t)ctx->grid_wave * WARPS;
    void *p;
    CK(cudaMalloc(&p, sizeof(double) * (size_t)D.C * K + 16));
    ctx->k_buffers[0] = p;
    D.sum_topk = (double *)p;
    CK(cudaMalloc(&p, sizeof(double) * K + 16));
    ctx->k_buffers[1] = p;
    D.run_a = (double *)p;
    CK(cudaMalloc(&p, sizeof(double) * K + 16));
    ctx->k_buffers[2] = p;
    D.run_b = (double *)p;
    CK(cudaMalloc(&p, sizeof(double) * nw * K + 16));
    ctx->k_buffers[3] = p;
    D.cand = (double *)p;
    D.K = K;
    return 0;
}

static int build_graphs(csvd_ctx *ctx);

extern "C" int csvd_reserve_k(csvd_ctx *ctx, int32_t k) {
    if (!ctx) return CSVD_ESTATE;
    if (k <= ctx->D.K) return 0;
    int K = 16;
    while (K < k) K <<= 1;
    CK(cudaSetDevice(ctx->device));
    CK(cudaStreamSynchronize(ctx->stream));
    int rc = alloc_k(ctx, K);
    if (rc) return rc;
    return build_graphs(ctx);
}

static size_t bounds_smem(const Dev &D) {
    size_t a = sizeof(double) * ((size_t)D.bd + (D.bplan.regular ? 0 : WARPS * (CSVD_MAX_LEAVES / 4)));
    size_t b = 12 * (2 * (size_t)D.cpad + 1) + 16;
    return a > b ? a : b;
}
static size_t wave_smem(const Dev &D) {
    size_t a = sizeof(double) * ((size_t)D.d + (D.wplan.regular ? 0 : WARPS * (CSVD_MAX_LEAVES / 4)));
    // scan: two running lists + at least one chunk row of (k + 6) doubles
    size_t b = sizeof(double) * (2 * (size_t)D.K + 8 + 4 * ((size_t)D.K + 6));
    return a > b ? a : b;
}

// kernel instantiation per (weight dtype, plan)
typedef void (*kern_t)(Dev);
template <typename ET>
static kern_t wave_kernel_for(const PwPlan &pl) {
    if (!pl.regular) return k_wave<ET, 0, 0>;
    switch (pl.cpl * 8 + pl.q) {
        case 8 * 8 + 1: return k_wave<ET, 8, 1>;
        case 8 * 8 + 2: return k_wave<ET, 8, 2>;
        case 8 * 8 + 4: return k_wave<ET, 8, 4>;
        case 4 * 8 + 1: return k_wave<ET, 4, 1>;
        case 2 * 8 + 1: return k_wave<ET, 2, 1>;
        default: return k_wave<ET, 1, 1>;
    }
}
static kern_t wave_kernel(const Dev &D) {
    return D.wdtype == CSVD_W_BF16 ? wave_kernel_for<uint16_t>(D.wplan) : wave_kernel_for<float>(D.wplan);
}
static kern_t bounds_kernel(const Dev &D) {
    const PwPlan &pl = D.bplan;
    if (!pl.regular) return k_bounds<0, 0>;
    switch (pl.cpl * 8 + pl.q) {
        case 8 * 8 + 1: return k_bounds<8, 1>;
        case 8 * 8 + 2: return k_bounds<8, 2>;
        case 8 * 8 + 4: return k_bounds<8, 4>;
        case 4 * 8 + 1: return k_bounds<4, 1>;
        case 2 * 8 + 1: return k_bounds<2, 1>;
        default: return k_bounds<1, 1>;
    }
}

static int launch_wave(csvd_ctx *ctx, cudaStream_t s) {
    Dev &D = ctx->D;
    void *args[] = {&D};
    cudaLaunchKernel((const void *)wave_kernel(D), dim3(ctx->grid_wave), dim3(THREADS), args, ctx->smem_wave, s);
    return 0;
}
static int launch_bounds(csvd_ctx *ctx, const Dev &Din, cudaStream_t s) {
    Dev D = Din;
    void *args[] = {&D};
    cudaLaunchKernel((const void *)bounds_kernel(D), dim3(ctx->grid_bounds), dim3(THREADS), args, ctx->smem_bounds,
                     s);
    return 0;
}

// Capture: [k_bounds] -> WHILE(handle) { k_wave }
static int capture_graph(csvd_ctx *ctx, int mode /*0 step,1 bounds,2 dense*/, cudaGraphExec_t *out,
                         cudaGraphConditionalHandle *hout) {
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    // (a conditional handle that no conditional node uses makes instantiation
    // fail, so the bounds-only graph has none)
    cudaGraphConditionalHandle h = 0;
    if (mode != 1) CK(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault));
    Dev D = ctx->D;
    D.loop = h;
    D.use_graph = (mode != 1);
    D.bounds_only = (mode == 1);
    D.dense_only = (mode == 2);
    cudaStream_t s = ctx->stream;
    // first node(s): bounds or dense setup
    CK(cudaStreamBeginCaptureToGraph(s, g, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    if (mode == 2)
        k_dense_setup<<<1, 32, 0, s>>>(D);
    else
        launch_bounds(ctx, D, s);
    cudaGraph_t tmp;
    CK(cudaStreamEndCapture(s, &tmp));
    if (mode != 1) {
        // find the leaf node to depend on
        size_t nn = 0;
        CK(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        CK(cudaGraphGetNodes(g, nodes.data(), &nn));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t cnode;
        CK(cudaGraphAddNode(&cnode, g, nodes.data(), nn, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        CK(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
        ctx->D.loop = h;
        Dev saved = ctx->D;
        ctx->D = D;
        launch_wave(ctx, s);
        ctx->D = saved;
        cudaGraph_t tmp2;
        CK(cudaStreamEndCapture(s, &tmp2));
    }
    CK(cudaGraphInstantiate(out, g, 0));
    CK(cudaGraphDestroy(g));
    *hout = h;
    return 0;
}

static int build_graphs(csvd_ctx *ctx) {
    if (ctx->g_step) cudaGraphExecDestroy(ctx->g_step);
    if (ctx->g_bounds) cudaGraphExecDestroy(ctx->g_bounds);
    if (ctx->g_dense) cudaGraphExecDestroy(ctx->g_dense);
    ctx->g_step = ctx->g_bounds = ctx->g_dense = nullptr;
    Dev &D = ctx->D;
    ctx->smem_bounds = bounds_smem(D);
    size_t ws = wave_smem(D);
    if (ws > ctx->smem_wave) ctx->smem_wave = ws;
    D.scan_smem_doubles = (int)(ctx->smem_wave / sizeof(double));
    CK(cudaFuncSetAttribute((const void *)bounds_kernel(D), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)ctx->smem_bounds));
    CK(cudaFuncSetAttribute((const void *)wave_kernel(D), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)ctx->smem_wave));
    int rc;
    if ((rc = capture_graph(ctx, 0, &ctx->g_step, &ctx->h_step))) return rc;
    if ((rc = capture_graph(ctx, 1, &ctx->g_bounds, &ctx->h_bounds))) return rc;
    if ((rc = capture_graph(ctx, 2, &ctx->g_dense, &ctx->h_dense))) return rc;
    return 0;
}

extern "C" int csvd_create(csvd_ctx **out, int device, const csvd_table_desc *t, const csvd_index_desc *ix) {
    if (!out || !t || !ix) return CSVD_ECONFIG;
    csvd_ctx *ctx = new csvd_ctx();
    *out = ctx;
    ctx->device = device;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    Dev &D = ctx->D;
    if (t->vocab_size < 1 || t->hidden_dim < 1 || t->vocab_size >= (1ll << 31))
        return fail(ctx, CSVD_EDIM, "bad table dims");
    if (ix->n_clusters < 1 || ix->n_clusters > 8192) return fail(ctx, CSVD_ECONFIG, "n_clusters must be in [1, 8192]");
    D.V = (int)t->vocab_size;
    D.d = (int)t->hidden_dim;
    D.C = ix->n_clusters;
    D.mode = ix->mode;
    D.bd = D.d + (ix->mode == CSVD_MODE_BIAS_AUGMENTED ? 1 : 0);
    D.wdtype = t->w_dtype;
    D.cpad = 1;
    while (D.cpad < D.C) D.cpad <<= 1;
    if (D.d > 32768) return fail(ctx, CSVD_EDIM, "hidden_dim > 32768 unsupported");
    // plans
    make_plan(D.d, D.wplan, ctx->wleaves, ctx->wprog);
    make_plan(D.bd, D.bplan, ctx->bleaves, ctx->bprog);
    if (D.wplan.nleaf > CSVD_MAX_LEAVES / 4 || D.bplan.nleaf > CSVD_MAX_LEAVES / 4)
        return fail(ctx, CSVD_EDIM, "too many pairwise leaves");
    int rc;
    int2 *dl;
    short *dp;
    if ((rc = dupload(ctx, &dl, ctx->wleaves.data(), ctx->wleaves.size()))) return rc;
    if ((rc = dupload(ctx, &dp, ctx->wprog.data(), ctx->wprog.size()))) return rc;
    D.wplan.leaves = dl;
    D.wplan.prog = dp;
    if ((rc = dupload(ctx, &dl, ctx->bleaves.data(), ctx->bleaves.size()))) return rc;
    if ((rc = dupload(ctx, &dp, ctx->bprog.data(), ctx->bprog.size()))) return rc;
    D.bplan.leaves = dl;
    D.bplan.prog = dp;
    // --- table: upload in original order, permute on device (weights == NULL:
    //     bounds-only context for cluster_bounds(index, h), which has no table)
    const long long V = D.V;
    const size_t esz = (D.wdtype == CSVD_W_BF16) ? 2 : 4;
    const size_t row_bytes = esz * (size_t)D.d;
    if (t->weights) {
        void *Wtmp = nullptr, *W = nullptr;
        CK(cudaMalloc(&Wtmp, row_bytes * V));
        CK(cudaMemcpy(Wtmp, t->weights, row_bytes * V, cudaMemcpyHostToDevice));
        long long *dperm64;
        if ((rc = dupload(ctx, &dperm64, (const long long *)ix->perm, (size_t)V))) return rc;
        CK(cudaMalloc(&W, row_bytes * V + 64));
        ctx->dev_allocs.push_back(W);
        k_permute_rows<<<4096, 256>>>((const char *)Wtmp, (char *)W, dperm64, V, (long long)row_bytes);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        CK(cudaFree(Wtmp));
        D.W = W;
    } else {
        D.W = nullptr;
    }
    std::vector<float> biasp(V);
    std::vector<int> perm32(V);
    for (long long p = 0; p < V; ++p) {
        long long tok = ix->perm[p];
        if (tok < 0 || tok >= V) return fail(ctx, CSVD_ECONFIG, "perm out of range");
        perm32[p] = (int)tok;
        biasp[p] = t->bias ? t->bias[tok] : 0.0f;
    }
    float *dbias;
    int *dperm;
    if ((rc = dupload(ctx, &dbias, biasp.data(), (size_t)V))) return rc;
    if ((rc = dupload(ctx, &dperm, perm32.data(), (size_t)V))) return rc;
    D.bias = dbias;
    D.perm = dperm;
    // --- index arrays
    const int C = D.C;
    std::vector<int> st32(C), sz32(C);
    std::vector<double> meanb(C);
    long long pos = 0;
    for (int c = 0; c < C; ++c) {
        st32[c] = (int)ix->starts[c];
        sz32[c] = (int)ix->sizes[c];
        if (ix->starts[c] != pos || ix->sizes[c] < 1) return fail(ctx, CSVD_ECONFIG, "cluster ranges must partition [0,V)");
        pos += ix->sizes[c];
        double s = 0;
        for (long long p = ix->starts[c]; p < ix->starts[c] + ix->sizes[c]; ++p) s += biasp[p];
        meanb[c] = s / (double)ix->sizes[c];
    }
    if (pos != V) return fail(ctx, CSVD_ECONFIG, "cluster ranges must cover [0,V)");
    double *dd;
    int *di;
    if ((rc = dupload(ctx, &dd, ix->centroids, (size_t)C * D.bd))) return rc;
    D.cent = dd;
    if ((rc = dupload(ctx, &dd, ix->radii, (size_t)C))) return rc;
    D.radii = dd;
    if ((rc = dupload(ctx, &dd, ix->max_biases, (size_t)C))) return rc;
    D.maxb = dd;
    if ((rc = dupload(ctx, &dd, ix->log_sizes, (size_t)C))) return rc;
    D.logsz = dd;
    if ((rc = dupload(ctx, &dd, meanb.data(), (size_t)C))) return rc;
    D.meanb = dd;
    if (D.mode == CSVD_MODE_SPHERICAL) {
        if (!ix->centroid_norms || !ix->angulars || !ix->max_norms || !ix->min_norms)
            return fail(ctx, CSVD_ECONFIG, "spherical index needs norms/angulars");
        if ((rc = dupload(ctx, &dd, ix->centroid_norms, (size_t)C))) return rc;
        D.cnorm = dd;
        if ((rc = dupload(ctx, &dd, ix->angulars, (size_t)C))) return rc;
        D.ang = dd;
        if ((rc = dupload(ctx, &dd, ix->max_norms, (size_t)C))) return rc;
        D.maxn = dd;
        if ((rc = dupload(ctx, &dd, ix->min_norms, (size_t)C))) return rc;
        D.minn = dd;
    }
    if ((rc = dupload(ctx, &di, st32.data(), (size_t)C))) return rc;
    D.starts = di;
    if ((rc = dupload(ctx, &di, sz32.data(), (size_t)C))) return rc;
    D.sizes = di;
    // --- per-step workspace
    if ((rc = dalloc(ctx, &ctx->d_h, (size_t)D.d))) return rc;
    D.h = ctx->d_h;
    if ((rc = dalloc(ctx, &ctx->d_cfg, 1))) return rc;
    D.cfg = ctx->d_cfg;
    if ((rc = dalloc(ctx, &D.U, C))) return rc;
    if ((rc = dalloc(ctx, &D.Uo, C))) return rc;
    if ((rc = dalloc(ctx, &D.X, C))) return rc;
    if ((rc = dalloc(ctx, &D.dots, C))) return rc;
    if ((rc = dalloc(ctx, &D.order, C))) return rc;
    if ((rc = dalloc(ctx, &D.cum, C + 1))) return rc;
    if ((rc = dalloc(ctx, &D.lrh, C + 1))) return rc;
    if ((rc = dalloc(ctx, &D.cl_done, C))) return rc;
    if ((rc = dalloc(ctx, &D.sum_lse, C))) return rc;
    if ((rc = dalloc(ctx, &D.sum_min, C))) return rc;
    if ((rc = dalloc(ctx, &D.sum_max, C))) return rc;
    if ((rc = dalloc(ctx, &D.S_logits, (size_t)V))) return rc;
    if ((rc = dalloc(ctx, &D.S_ids, (size_t)V))) return rc;
    if ((rc = dalloc(ctx, &D.st, 1))) return rc;
    if ((rc = dalloc(ctx, &D.res, 1))) return rc;
    if ((rc = dalloc(ctx, &D.counters, 4))) return rc;
    CK(cudaMemset(D.counters, 0, 16));
    D.dbg = nullptr;
    if (getenv("CSVD_DEBUG_TS") && atoi(getenv("CSVD_DEBUG_TS")) > 0) {
        if ((rc = dalloc(ctx, &D.dbg, 64))) return rc;
        CK(cudaMemset(D.dbg, 0, 64 * 8));
    }
    CK(cudaMemset(D.cl_done, 0, sizeof(int) * C));
    CK(cudaMemset(D.st, 0, sizeof(ScanState)));
    CK(cudaMemset(D.res, 0, sizeof(csvd_result)));
    // --- grids (persistent: fill every SM)
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
    ctx->smem_bounds = bounds_smem(D);
    D.K = 16;
    ctx->smem_wave = wave_smem(D);
    D.scan_smem_doubles = (int)(ctx->smem_wave / sizeof(double));
    CK(cudaFuncSetAttribute((const void *)bounds_kernel(D), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)ctx->smem_bounds));
    CK(cudaFuncSetAttribute((const void *)wave_kernel(D), cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)ctx->smem_wave));
    int occ_b = 0, occ_w = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_b, bounds_kernel(D), THREADS, ctx->smem_bounds));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_w, wave_kernel(D), THREADS, ctx->smem_wave));
    if (occ_b < 1) occ_b = 1;
    if (occ_w < 1) occ_w = 1;
    ctx->grid_bounds = nsm * occ_b;
    int need_b = (C + WARPS - 1) / WARPS;
    if (ctx->grid_bounds > need_b) ctx->grid_bounds = need_b;
    ctx->grid_wave = nsm * occ_w;
    // --- pinned staging
    CK(cudaHostAlloc(&ctx->h_pin, sizeof(double) * (D.d + 1), cudaHostAllocDefault));
    CK(cudaHostAlloc(&ctx->cfg_pin, sizeof(csvd_config), cudaHostAllocDefault));
    CK(cudaHostAlloc(&ctx->res_pin, sizeof(csvd_result), cudaHostAllocDefault));
    CK(cudaHostAlloc(&ctx->st_pin, sizeof(ScanState), cudaHostAllocDefault));
    ctx->pin_cap = V;
    CK(cudaHostAlloc(&ctx->ids_pin, sizeof(long long) * V, cudaHostAllocDefault));
    CK(cudaHostAlloc(&ctx->logits_pin, sizeof(double) * V, cudaHostAllocDefault));
    if ((rc = alloc_k(ctx, 16))) return rc;
    return build_graphs(ctx);
}

extern "C" int csvd_destroy(csvd_ctx *ctx) {
    if (!ctx) return 0;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->g_step) cudaGraphExecDestroy(ctx->g_step);
    if (ctx->g_bounds) cudaGraphExecDestroy(ctx->g_bounds);
    if (ctx->g_dense) cudaGraphExecDestroy(ctx->g_dense);
    for (void *p : ctx->dev_allocs) cudaFree(p);
    for (int i = 0; i < 6; ++i)
        if (ctx->k_buffers[i]) cudaFree(ctx->k_buffers[i]);
    if (ctx->flush_buf) cudaFree(ctx->flush_buf);
    if (ctx->h_pin) cudaFreeHost(ctx->h_pin);
    if (ctx->cfg_pin) cudaFreeHost(ctx->cfg_pin);
    if (ctx->res_pin) cudaFreeHost(ctx->res_pin);
    if (ctx->st_pin) cudaFreeHost(ctx->st_pin);
    if (ctx->ids_pin) cudaFreeHost(ctx->ids_pin);
    if (ctx->logits_pin) cudaFreeHost(ctx->logits_pin);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return 0;
}

extern "C" const char *csvd_strerror(csvd_ctx *ctx) { return ctx ? ctx->err.c_str() : "null context"; }

static int check_cfg(csvd_ctx *ctx, const csvd_config *cfg) {
    const Dev &D = ctx->D;
    if (cfg->k < 1 || cfg->k > D.V) return fail(ctx, CSVD_ECONFIG, "need 1 <= k <= V");
    if (cfg->n_targets < 1 || cfg->n_targets > 3) return fail(ctx, CSVD_ECONFIG, "bad targets");
    if (!(cfg->epsilon > 0 && cfg->epsilon < 1)) return fail(ctx, CSVD_ECONFIG, "epsilon must lie in (0, 1)");
    if (cfg->n_levels < 1 || cfg->n_levels > CSVD_MAX_LEVELS) return fail(ctx, CSVD_ECONFIG, "bad fallback levels");
    if (cfg->k_max < 0) return fail(ctx, CSVD_ECONFIG, "K_max must be >= 0");
    return 0;
}

// Direct mode: the same kernels without the graph; the host reads the device
// state after every wave (profiling: ncu cannot see inside conditional nodes).
static int run_direct(csvd_ctx *ctx, cudaStream_t s, int dense_only) {
    Dev D = ctx->D;
    D.use_graph = 0;
    D.bounds_only = 0;
    D.dense_only = dense_only;
    void *args[] = {&D};
    if (dense_only)
        CK(cudaLaunchKernel((const void *)k_dense_setup, dim3(1), dim3(32), args, 0, s));
    else
        CK(cudaLaunchKernel((const void *)bounds_kernel(D), dim3(ctx->grid_bounds), dim3(THREADS), args,
                            ctx->smem_bounds, s));
    int launches = 1;
    for (int it = 0; it < D.C + 16; ++it) {
        CK(cudaMemcpyAsync(ctx->st_pin, D.st, sizeof(ScanState), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (ctx->st_pin->mode == MODE_IDLE) break;
        CK(cudaLaunchKernel((const void *)wave_kernel(D), dim3(ctx->grid_wave), dim3(THREADS), args, ctx->smem_wave,
                            s));
        launches++;
    }
    ctx->last_launches = launches;
    return 0;
}

static int run_step_async(csvd_ctx *ctx, const csvd_config *cfg, cudaStream_t s) {
    if (!ctx->D.W) return fail(ctx, CSVD_ECONFIG, "bounds-only context (no table)");
    int rc = check_cfg(ctx, cfg);
    if (rc) return rc;
    if (cfg->k > ctx->D.K) {
        if ((rc = csvd_reserve_k(ctx, cfg->k))) return rc;
    }
    *ctx->cfg_pin = *cfg;
    CK(cudaMemcpyAsync(ctx->d_cfg, ctx->cfg_pin, sizeof(csvd_config), cudaMemcpyHostToDevice, s));
    if (ctx->direct) return run_direct(ctx, s, 0);
    CK(cudaGraphLaunch(ctx->g_step, s));
    return 0;
}

extern "C" int csvd_set_direct(csvd_ctx *ctx, int32_t direct) {
    if (!ctx) return CSVD_ESTATE;
    ctx->direct = direct ? 1 : 0;
    return 0;
}

extern "C" int csvd_step_device(csvd_ctx *ctx, const double *h_dev, const csvd_config *cfg, void *stream) {
    if (!ctx || !cfg) return CSVD_ESTATE;
    cudaStream_t s = stream ? (cudaStream_t)stream : ctx->stream;
    CK(cudaSetDevice(ctx->device));
    if (h_dev != ctx->d_h) CK(cudaMemcpyAsync(ctx->d_h, h_dev, sizeof(double) * ctx->D.d, cudaMemcpyDeviceToDevice, s));
    return run_step_async(ctx, cfg, s);
}

extern "C" int csvd_outputs(csvd_ctx *ctx, int64_t **ids_dev, double **logits_dev, csvd_result **res_dev) {
    if (!ctx) return CSVD_ESTATE;
    if (ids_dev) *ids_dev = (int64_t *)ctx->D.S_ids;
    if (logits_dev) *logits_dev = ctx->D.S_logits;
    if (res_dev) *res_dev = ctx->D.res;
    return 0;
}

extern "C" int csvd_step_host(csvd_ctx *ctx, const double *h, const csvd_config *cfg, csvd_result *res, int64_t *ids,
                              double *logits, int64_t cap) {
    if (!ctx || !h || !cfg || !res) return CSVD_ESTATE;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const int d = ctx->D.d;
    memcpy(ctx->h_pin, h, sizeof(double) * d);
    CK(cudaMemcpyAsync(ctx->d_h, ctx->h_pin, sizeof(double) * d, cudaMemcpyHostToDevice, s));
    int rc = run_step_async(ctx, cfg, s);
    if (rc) return rc;
    // speculative first chunk of outputs with the result record
    const int64_t first = ctx->D.V < 4096 ? ctx->D.V : 4096;
    CK(cudaMemcpyAsync(ctx->res_pin, ctx->D.res, sizeof(csvd_result), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ctx->ids_pin, ctx->D.S_ids, sizeof(long long) * first, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(ctx->logits_pin, ctx->D.S_logits, sizeof(double) * first, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *res = *ctx->res_pin;
    if (res->error) return fail(ctx, res->error, res->error == CSVD_EVALUE ? "bounds must be finite" : "device state error");
    int64_t n = res->sub_size;
    if (n > cap) return fail(ctx, CSVD_EDIM, "output capacity too small");
    if (n > first) {
        CK(cudaMemcpyAsync(ctx->ids_pin + first, ctx->D.S_ids + first, sizeof(long long) * (n - first),
                           cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(ctx->logits_pin + first, ctx->D.S_logits + first, sizeof(double) * (n - first),
                           cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    if (ids) memcpy(ids, ctx->ids_pin, sizeof(int64_t) * n);
    if (logits) memcpy(logits, ctx->logits_pin, sizeof(double) * n);
    return 0;
}

extern "C" int csvd_bounds_host(csvd_ctx *ctx, const double *h, int32_t slack_f32, double *values, double *qn,
                                double *slack) {
    if (!ctx || !h) return CSVD_ESTATE;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    csvd_config cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.k = 1;
    cfg.n_targets = 1;
    cfg.epsilon = 0.5;
    cfg.n_levels = 1;
    cfg.level_kind[0] = CSVD_FB_FULL_VOCAB;
    cfg.k_max = ctx->D.V;
    cfg.slack_f32 = slack_f32;
    *ctx->cfg_pin = cfg;
    memcpy(ctx->h_pin, h, sizeof(double) * ctx->D.d);
    CK(cudaMemcpyAsync(ctx->d_h, ctx->h_pin, sizeof(double) * ctx->D.d, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyAsync(ctx->d_cfg, ctx->cfg_pin, sizeof(csvd_config), cudaMemcpyHostToDevice, s));
    CK(cudaGraphLaunch(ctx->g_bounds, s));
    CK(cudaMemcpyAsync(ctx->res_pin, ctx->D.res, sizeof(csvd_result), cudaMemcpyDeviceToHost, s));
    if (values) CK(cudaMemcpyAsync(values, ctx->D.U, sizeof(double) * ctx->D.C, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (qn) *qn = ctx->res_pin->query_norm;
    if (slack) *slack = ctx->res_pin->slack;
    if (ctx->res_pin->error) return fail(ctx, CSVD_EVALUE, "bounds must be finite");
    return 0;
}

static int dense_async(csvd_ctx *ctx, cudaStream_t s) {
    if (!ctx->D.W) return fail(ctx, CSVD_ECONFIG, "bounds-only context (no table)");
    csvd_config cfg;
    memset(&cfg, 0, sizeof(cfg));
    cfg.k = 1;
    cfg.n_targets = 1;
    cfg.epsilon = 0.5;
    cfg.n_levels = 1;
    cfg.level_kind[0] = CSVD_FB_FULL_VOCAB;
    cfg.k_max = ctx->D.V;
    *ctx->cfg_pin = cfg;
    CK(cudaMemcpyAsync(ctx->d_cfg, ctx->cfg_pin, sizeof(csvd_config), cudaMemcpyHostToDevice, s));
    if (ctx->direct) return run_direct(ctx, s, 1);
    CK(cudaGraphLaunch(ctx->g_dense, s));
    return 0;
}

extern "C" int csvd_dense_host(csvd_ctx *ctx, const double *h, double *logits) {
    if (!ctx || !h) return CSVD_ESTATE;
    CK(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    memcpy(ctx->h_pin, h, sizeof(double) * ctx->D.d);
    CK(cudaMemcpyAsync(ctx->d_h, ctx->h_pin, sizeof(double) * ctx->D.d, cudaMemcpyHostToDevice, s));
    int rc = dense_async(ctx, s);
    if (rc) return rc;
    CK(cudaMemcpyAsync(ctx->logits_pin, ctx->D.S_logits, sizeof(double) * ctx->D.V, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    memcpy(logits, ctx->logits_pin, sizeof(double) * ctx->D.V);
    return 0;
}

extern "C" int csvd_dense_device(csvd_ctx *ctx, const double *h_dev, void *stream) {
    if (!ctx) return CSVD_ESTATE;
    cudaStream_t s = stream ? (cudaStream_t)stream : ctx->stream;
    CK(cudaSetDevice(ctx->device));
    if (h_dev && h_dev != ctx->d_h)
        CK(cudaMemcpyAsync(ctx->d_h, h_dev, sizeof(double) * ctx->D.d, cudaMemcpyDeviceToDevice, s));
    return dense_async(ctx, s);
}

extern "C" int csvd_info(csvd_ctx *ctx, int64_t *V, int64_t *d, int32_t *C, int32_t *bd, int32_t *wreg, int32_t *breg,
                         int32_t *grid) {
    if (!ctx) return CSVD_ESTATE;
    if (V) *V = ctx->D.V;
    if (d) *d = ctx->D.d;
    if (C) *C = ctx->D.C;
    if (bd) *bd = ctx->D.bd;
    if (wreg) *wreg = ctx->D.wplan.regular;
    if (breg) *breg = ctx->D.bplan.regular;
    if (grid) *grid = ctx->grid_wave;
    return 0;
}

extern "C" int csvd_debug_timestamps(csvd_ctx *ctx, unsigned long long *out64) {
    if (!ctx || !ctx->D.dbg) return CSVD_ESTATE;
    CK(cudaStreamSynchronize(ctx->stream));
    CK(cudaMemcpy(out64, ctx->D.dbg, 64 * 8, cudaMemcpyDeviceToHost));
    return 0;
}

extern "C" int csvd_stream(csvd_ctx *ctx, void **stream) {
    if (!ctx || !stream) return CSVD_ESTATE;
    *stream = (void *)ctx->stream;
    return 0;
}

extern "C" int csvd_last_launches(csvd_ctx *ctx, int32_t *n) {
    if (!ctx || !n) return CSVD_ESTATE;
    *n = ctx->direct ? ctx->last_launches : 1 + ctx->res_pin->waves;
    return 0;
}

// ---------------------------------------------------------------------------
// L2 flush for benchmarking: stream-read a buffer larger than L2 (clean lines,
// nothing to write back when the next step allocates)
// ---------------------------------------------------------------------------
__global__ void k_l2_flush(const uint4 *buf, size_t n, unsigned *sink) {
    unsigned acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = __ldcg(buf + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x9e3779b9u) *sink = acc;  // keep the loads alive
}

extern "C" int csvd_l2_flush(csvd_ctx *ctx, void *stream) {
    if (!ctx) return CSVD_ESTATE;
    cudaStream_t s = stream ? (cudaStream_t)stream : ctx->stream;
    CK(cudaSetDevice(ctx->device));
    const size_t bytes = 384ull << 20;
    if (!ctx->flush_buf) {
        CK(cudaMalloc(&ctx->flush_buf, bytes + 64));
        CK(cudaMemset(ctx->flush_buf, 1, bytes));
    }
    k_l2_flush<<<ctx->grid_wave, 256, 0, s>>>((const uint4 *)ctx->flush_buf, bytes / 16,
                                               (unsigned *)((char *)ctx->flush_buf + bytes));
    CK(cudaGetLastError());
    return 0;
}

// ---------------------------------------------------------------------------
// host-only test hooks (no GPU needed): run the scan state machine on host
// ---------------------------------------------------------------------------
struct HostPrims {
    int merge_topk(const double *A, int ka, const double *B, int kb, int k, double *out) {
        int i = 0, j = 0, n = 0;
        while (n < k && (i < ka || j < kb)) {
            if (j >= kb || (i < ka && A[i] >= B[j])) out[n++] = A[i++];
            else out[n++] = B[j++];
        }
        return n;
    }
    double lse_all(const double *v, int n, double vmax) {
        if (n == 0 || vmax == -INFINITY) return -INFINITY;
        double s = 0;
        for (int i = 0; i < n; ++i) s += exp(v[i] - vmax);
        return vmax + log(s);
    }
};

// Runs the full scan on host given all per-cluster summaries (all C available).
// Returns 0 and fills res / *p_final / *phase_final.
extern "C" int csvd_test_scan_host(const csvd_config *cfg, int C, long long V, int d, const int *cum,
                                   const double *Uo, const double *lrh, const double *sum_lse, const double *sum_min,
                                   const double *sum_max, const double *sum_topk, int K, const double *S_logits,
                                   int p_sel, csvd_result *res, int *p_final, int *phase_final) {
    ScanState st;
    memset(&st, 0, sizeof(st));
    st.phase = PH_MAIN;
    st.log_z = -INFINITY;
    st.p_sel = p_sel;
    std::vector<double> a(K + 1), b(K + 1);
    double *ra = a.data(), *rb = b.data();
    HostPrims prims;
    csvd_result r;
    memset(&r, 0, sizeof(r));
    ScanIn in{cfg, C, V, d, cum, Uo, lrh, sum_lse, sum_min, sum_max, sum_topk, K, S_logits};
    ScalarSearch search;
    if (cfg->variant == CSVD_VARIANT_BATCHSELECT) st.p_sel = csvd_select_prefix(in, cfg->k_max, search);
    if (p_sel > 0 && p_sel != st.p_sel) return -100;  // selection restatement mismatch
    Scan<HostPrims> sc{in, st, ra, rb, prims, r};
    sc.run(C);
    *res = r;
    *p_final = st.p;
    *phase_final = st.phase;
    return 0;
}

// ABI self-check for the ctypes mirrors (tests/test_abi.py)
extern "C" int csvd_test_sizes(int32_t *cfg_size, int32_t *res_size, int32_t *table_size, int32_t *index_size) {
    *cfg_size = (int32_t)sizeof(csvd_config);
    *res_size = (int32_t)sizeof(csvd_result);
    *table_size = (int32_t)sizeof(csvd_table_desc);
    *index_size = (int32_t)sizeof(csvd_index_desc);
    return 0;
}
