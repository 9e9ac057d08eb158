// The head step: the common decode_step (decode.py:312-343) as one lean
// cooperative kernel with a single grid barrier, the rest of the step driven
// by completion counters instead of grid barriers.
//
//   h staged by TMA; bounds U_c for every cluster           bounds.py:79-83
//   == one grid barrier ==
//   every CTA: U -> the head of np.lexsort((arange(C), -U))  decode.py:166
//              (clusters whose bound reaches the best-logit estimate; order_head)
//   rows: CTA b owns rows [b*R/G, (b+1)*R/G) of the head's opening order
//         (contiguous, so a cluster spans 1-3 CTAs); bit-exact f64 logits go
//         straight to S (and, for host-API steps, to the mapped host buffers)
//                                                            decode.py:169-176
//   the CTA whose rows complete a cluster (per-cluster row counters) writes its
//   summary: top-k values, log-sum-exp, min, max          certify.py:73-88
//   the CTA that completes the last cluster runs the certification scan over
//   the head (scan.cuh: the exact sequential state machine)  decode.py:192-210
//
// Steps the head cannot decide (more than 64 head clusters, certification
// past the head, the fallback chain, non-finite bounds) leave the graph's
// conditional handle at its default: the general k_step then runs the whole
// step (kernels.cuh).  Every value this kernel produces comes from the same
// device functions as k_step's, so a step's outcome does not depend on which
// kernel decided it.
#pragma once
#include "kernels.cuh"

#define HMAX 64  // head clusters (order_head's limit)
#define KH 32    // k limit of the head kernel (the scan's register lists)

// Grid barrier on a monotone 64-bit arrival counter: one atomic per CTA and
// no reset (the target is the next multiple of the grid size), so a barrier is
// one L2 round trip plus the arrival of the slowest CTA.  Only kernels with
// the same grid size may share a counter.
static __device__ __forceinline__ void grid_sync_mono(const Dev &D, unsigned long long *ctr) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned long long G = gridDim.x;
        unsigned long long old, v, spins = 0;
        asm volatile("atom.add.release.gpu.global.u64 %0, [%1], 1;" : "=l"(old) : "l"(ctr) : "memory");
        const unsigned long long target = (old / G + 1) * G;
        do {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
            if (++spins > (1ull << 26)) {  // flag rather than hang
                D.res->error = CSVD_ESTATE;
                break;
            }
        } while (v < target);
    }
    __syncthreads();
}

// bounds for this CTA's clusters (warp per cluster, as bounds_phase) and ||h||
template <int Q>
static __device__ __forceinline__ double head_bounds(const Dev &D, const double *hs) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ double s_qn;
    __shared__ double s_dot[WARPS][MAX_PER_WARP];
    const int G = gridDim.x, stride = G * WARPS;
    if (warp == WARPS - 1) {  // ||h|| = sqrt(sum(h*h)) (_linalg.py:40-43)
        const double ss = warp_dot_regular<double, 8, Q>(D.h, hs, D.bplan.leaf_len, lane);
        if (lane == 0) s_qn = __dsqrt_rn(ss);
    }
    int j = 0;
    for (int c = warp * G + blockIdx.x; c < D.C && j < MAX_PER_WARP; c += stride, ++j) {
        const double dot = warp_dot_regular<double, 8, Q>(D.cent + (size_t)c * D.bd, hs, D.bplan.leaf_len, lane);
        if (lane == 0) s_dot[warp][j] = dot;
    }
    __syncthreads();
    const double qn = s_qn;
    if (lane == 0) {
        j = 0;
        for (int c = warp * G + blockIdx.x; c < D.C && j < MAX_PER_WARP; c += stride, ++j) {
            const double dot = s_dot[warp][j];
            D.Uraw[c] = D.mode == CSVD_MODE_SPHERICAL ? cone_bound(D, c, dot, qn)
                                                      : __dadd_rn(__dadd_rn(dot, __dmul_rn(D.radii[c], qn)), D.maxb[c]);
            D.dots[c] = dot;
        }
    }
    return qn;
}

template <typename ET, int Q>
__global__ void __launch_bounds__(THREADS, 1) k_head(const __grid_constant__ Dev D, cudaGraphConditionalHandle cond) {
    extern __shared__ __align__(16) double smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int G = gridDim.x, b = blockIdx.x;
    double *hs = smem;
    double *ws = smem + D.ord_off;
    double *sws = smem + D.sum_off;
    __shared__ ScanShared ss;
    __shared__ unsigned long long s_hbar;
    const bool lead = b == 0 && tid == 0;
    if (lead) DBG_TS(D, 24);
    if (tid == 0) mbar_init(&s_hbar, 1);
    __syncthreads();
    tma_stage_leaves(D.wplan, D.h, D.d, 1, hs, 0, &s_hbar, 0);
    if (lead) DBG_TS(D, 25);
    const double qn = head_bounds<Q>(D, hs);
    if (lead) {
        D.res->query_norm = qn;
        DBG_TS(D, 26);
    }
    grid_sync_mono(D, D.bar64);
    if (lead) DBG_TS(D, 27);
    // ---- the head of the opening order (every CTA, identically)
    Ord o;
    ord_bind(D, ws, o);
    __shared__ double s_slack, s_est;
    if (!stage_bounds(D, o, qn, &s_slack)) return;  // non-finite bound: k_step reports it
    const int hn = order_head(D, o, s_est);
    if (hn == 0) return;  // no head: k_step builds the full order
    if (tid == 0) init_state(D, o, ss, hn, s_est);
    if (lead) DBG_TS(D, 28);
    // ---- rows of the head, contiguous per CTA
    const int R = o.cum[hn];
    const int r_lo = (int)((long long)R * b / G), r_hi = (int)((long long)R * (b + 1) / G);
    for (int r = r_lo + warp; r < r_hi; r += WARPS) {
        int lo = 0, hi = hn;  // cum[lo] <= r < cum[lo+1]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (o.cum[mid] <= r) lo = mid; else hi = mid;
        }
        const int c = o.order[lo];
        const int i = r - o.cum[lo];
        const int pos = __ldg(D.starts + c) + i;
        const double logit = row_logit<ET, 8, Q>(D, __ldg(D.wrow0 + c) + i, pos, hs, nullptr, lane);
        if (lane == 0) {
            D.S_logits[r] = logit;
            D.S_ids[r] = __ldg(D.perm + pos);
        }
    }
    if (lane == 0) __threadfence();
    __syncthreads();
    if (D.dbg && tid == 0) D.dbg[384 + (b & 255)] = gtimer();
    // ---- completion counting: this CTA's share of every cluster it touches
    __shared__ int s_comp[HMAX], s_ncomp, s_last;
    if (tid == 0) s_ncomp = 0;
    __syncthreads();
    if (tid < hn) {
        const int a = max(o.cum[tid], r_lo), e = min(o.cum[tid + 1], r_hi);
        if (e > a) {
            __threadfence();
            const int n = e - a;
            if (atomicAdd(D.hcnt + tid, n) + n == o.cum[tid + 1] - o.cum[tid]) s_comp[atomicAdd(&s_ncomp, 1)] = tid;
        }
    }
    __syncthreads();
    const int ncomp = s_ncomp;
    const int k = D.cfg->k;
    double *g_lse = D.hws, *g_min = g_lse + HMAX, *g_max = g_min + HMAX, *g_topk = g_max + HMAX;
    if (ncomp > 0) __threadfence();  // the completing rows of other CTAs are visible past here
    for (int j = warp; j < ncomp; j += WARPS) {  // summaries of the clusters this CTA completed
        const int q = s_comp[j];
        double pre[SUM_E];
        summary_load(D, o.cum[q], o.cum[q + 1], pre, lane);
        cluster_summary(D, o.cum[q], o.cum[q + 1], k, g_topk + (size_t)q * KH, g_lse + q, g_min + q, g_max + q, pre,
                        lane);
        if (lane == 0) __threadfence();
    }
    __syncthreads();
    if (tid == 0) {
        s_last = 0;
        if (ncomp > 0) {
            __threadfence();
            s_last = atomicAdd(D.hcnt + HMAX, ncomp) + ncomp == hn;
        }
    }
    __syncthreads();
    if (D.res_host) {  // host-API step: this CTA's rows into the mapped buffers (speculative:
                       // the host reads only the first |S| entries)
        for (int r = r_lo + tid; r < r_hi; r += THREADS) {
            D.logits_host[r] = __ldcg(D.S_logits + r);
            D.ids_host[r] = __ldcg(D.S_ids + r);
        }
    }
    if (D.dbg && tid == 0 && b < 256) D.dbg[128 + b] = gtimer();  // per-CTA: summaries done
    if (!s_last) return;
    // ---- the last CTA: certification scan over the head (scan.cuh)
    __threadfence();
    if (D.dbg && tid == 0) {
        DBG_TS(D, 29);
        D.dbg[31] = (unsigned long long)b;
        g_dbg_cta = b;
    }
    __syncthreads();
    double *c_vals = sws, *c_lse = sws + 6 * CHUNK, *c_min = c_lse + CHUNK, *c_max = c_min + CHUNK;
    double *la = c_max + CHUNK, *lb = la + D.K, *c_topk = lb + D.K;
    double reg_list = -INFINITY;
    for (int q0 = 0; q0 < hn; q0 += D.chunk) {
        const int q1 = min(hn, q0 + D.chunk);
        for (int i = tid; i < q1 - q0; i += THREADS) {
            c_lse[i] = __ldcg(g_lse + q0 + i);
            c_min[i] = __ldcg(g_min + q0 + i);
            c_max[i] = __ldcg(g_max + q0 + i);
        }
        for (int i = tid; i < (q1 - q0) * k; i += THREADS)
            c_topk[i] = __ldcg(g_topk + (size_t)(q0 + i / k) * KH + i % k);
        __syncthreads();
        if (warp == 0) scan_chunk(D, o, ss, q0, q1, c_topk, c_lse, c_min, c_max, c_vals, la, lb, reg_list, lane);
        __syncthreads();
        if (ss.st.phase != PH_MAIN && ss.st.phase != PH_PE) break;
    }
    for (int q = tid; q <= HMAX; q += THREADS) D.hcnt[q] = 0;  // every counter use of this step is done
    if (tid == 0) {
        if (ss.st.phase == PH_DONE) {
            csvd_result r = ss.res;
            r.query_norm = qn;
            r.slack = s_slack;
            r.waves = 1;
            r.error = 0;
            *D.res = r;
            ScanState s2 = ss.st;
            s2.mode = MODE_IDLE;
            s2.iter = 1;
            *D.st = s2;
            if (D.res_host) *D.res_host = r;
            if (cond) cudaGraphSetConditional(cond, 0);  // decided: skip the general step
        }
        DBG_TS(D, 30);
        if (D.dbg) g_dbg_cta = 0;
    }
}
