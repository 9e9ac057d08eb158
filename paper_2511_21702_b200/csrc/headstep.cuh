// The head step: the common decode_step (decode.py:312-343) as one lean
// cooperative kernel with a single grid barrier; the rest of the step is
// dataflow through per-cluster completion counters.
//
//   h staged by TMA; bounds U_c for every cluster           bounds.py:79-83
//   == one grid barrier ==
//   every CTA: U -> the head of np.lexsort((arange(C), -U))  decode.py:166
//              (clusters whose bound reaches the best-logit estimate; order_head)
//   CTAs 1..G-1 (row CTAs): rows [b'*R/G', (b'+1)*R/G') of the head's opening
//         order (contiguous, so a cluster spans 1-3 CTAs); bit-exact f64 logits
//         go straight to S (and, for host-API steps, to the mapped host
//         buffers)                                             decode.py:169-176
//         then the certification inputs of their own rows: a top-k histogram
//         (integer counts, certify.py:128-139) and one record per (CTA,
//         cluster) segment -- sum exp(S - est), min, max (certify.py:73-88) --
//         and one release-add arrival
//   CTA 0 (the certifying CTA) does no rows: it dry-runs the certifier while
//         they run (its code is cold after the L2 flush / the rest of a
//         model), waits for every arrival, reduces the records per cluster in
//         a fixed order, tests every head prefix at once and publishes a
//         decision word (head_certify_seg).
//
// Steps the head cannot decide (more than 64 head clusters, certification
// past the head, the fallback chain, non-finite bounds) run the general step
// body (kernels.cuh) in the same launch: every CTA waits for the decision
// word, then all of them start the general step from scratch.  Every value
// this kernel produces comes from the same device functions as k_step's, so a
// step's outcome does not depend on which path decided it.
#pragma once
#include "kernels.cuh"

#define HMAX 64  // head clusters (order_head's limit)
#define KH 32    // k limit of the head kernel (the scan's register lists)

// Head workspace (D.hcnt, one allocation per step context / batch lane):
//   ints [0, HMAX]            arrivals of the row CTAs at [HMAX]
//   ints [HW_HIST, +HMAX + 2) top-k histogram (certify.py:128-139 as counts)
//   HeadRec [HW_SEGS]         per-(row CTA b, cluster position q) segment records, slot b + q
#define HW_INTS 256
#define HW_HIST 80
#define HW_SEGS 256
#define HW_TOTAL_INTS (HW_INTS + HW_SEGS * 8)
struct HeadRec {
    double z, mn, mx;  // sum exp(S - est), min, max over the segment's logits
    int q;             // cluster position in the opening order
    unsigned ep;       // the step's epoch (stale records never match)
};
static_assert(sizeof(HeadRec) == 32, "HeadRec layout");
__device__ __forceinline__ HeadRec *hw_recs(const Dev &D) { return reinterpret_cast<HeadRec *>(D.hcnt + HW_INTS); }

// Grid barrier on a monotone 64-bit arrival counter: one atomic per CTA and
// no reset (the target is the next multiple of the grid size), so a barrier is
// one L2 round trip plus the arrival of the slowest CTA.  Only kernels with
// the same grid size may share a counter.
static __device__ __forceinline__ unsigned long long grid_sync_mono(const Dev &D, unsigned long long *ctr) {
    __syncthreads();
    unsigned long long epoch = 0;
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
        epoch = target / G;
    }
    __syncthreads();
    return epoch;  // thread 0: this barrier's epoch (1, 2, ... over the counter's life)
}

// release / acquire primitives (GPU scope).  A release by one thread after a
// __syncthreads() also orders the other threads' earlier writes (the barrier
// makes them visible to it; release is cumulative), so a CTA publishes its
// rows with one release operation instead of full SC fences (__threadfence
// compiles to MEMBAR.SC.GPU + an L1 invalidation on this part).
static __device__ __forceinline__ void red_release_add(int *p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
static __device__ __forceinline__ int ld_acquire_s32(const int *p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
static __device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// bounds for this CTA's clusters (warp per cluster, as bounds_phase) and ||h||
template <int Q>
static __device__ __forceinline__ double head_bounds(const Dev &D, const double *hs) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __shared__ double s_qn;
    __shared__ double s_dot[WARPS][MAX_PER_WARP];
    const int G = gridDim.x, stride = G * WARPS;
    if (warp == WARPS - 1) {  // ||h|| = sqrt(sum(h*h)) (_linalg.py:40-43), both operands staged
        const double ss = warp_selfdot_smem<Q>(hs, D.bplan.leaf_len, lane);
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

// ---------------------------------------------------------------------------
// Block-parallel certification of the head (CTA 0, all warps): every prefix
// p = 1..hn of the head is tested at once instead of cluster by cluster.
//   log Z_S(p)  = M + log(sum over the first p clusters of sum exp(S - M))
//                 (certify.py:79-83; the value the reference's logaddexp chain
//                 and its 64-merge recompute converge to, within ulps)
//   top-k test  u_max(p) < kth(p)  <=>  #{i < cum[p] : S_i > Uo[p]} >= k
//                 (certify.py:128-139): each logit adds 1 to every prefix from
//                 max(q(i) + 1, first p with Uo[p] < S_i) on (Uo is
//                 non-increasing): a histogram + prefix sum
//   rho / delta from log Z_S(p) and log R-hat(p)          (certify.py:93-107)
// The first prefix with an event (budget overflow or a certified target, in
// the configured target order; decode.py:192-210, 329-342) is the decision;
// its k-th logit (np.partition, certify.py:88) comes from per-cluster top-k
// lists, min / max (xi) from per-cluster extrema.  Returns 1 = decided (res
// filled), 0 = the step needs the general path (overflow -> fallback chain,
// or no certificate inside the head).
static __device__ __forceinline__ bool head_fits(const Dev &D, const Ord &o, int hn) {
    // the head's logits and its clusters' top-k lists fit where h was staged
    return o.cum[hn] + hn * D.cfg->k <= pw_hs_size(D.wplan);
}

// Block-parallel certification (CTA 0).  L: the head's logits staged in
// shared memory (where h was).
//   per cluster (warp w: clusters w, w + 8, ...): sum exp(S - M), min, max
//     and the top-k histogram: element i counts for every prefix p >=
//     max(q + 1, 1 + #{p in [1, hn] : Uo[p] >= S_i}), and the cluster's
//     top-k values (k pops of the lanes' running maxima)
//   warp 0: every prefix's tests at once -> the decision prefix ps, whose
//     k-th value is a k-pop merge of the first ps clusters' lists
static __device__ __forceinline__ int head_certify(const Dev &D, const Ord &o, int hn, double *L, csvd_result &res) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const csvd_config &cfg = *D.cfg;
    const int k = cfg.k;
    const int R = o.cum[hn];
    __shared__ double s_red[WARPS], s_zq[HMAX], s_mnq[HMAX], s_mxq[HMAX];
    double *s_tk = L + R;  // per-cluster top-k lists (stride k), after the logits
    __shared__ int s_hist[HMAX + 2];
    __shared__ int s_p, s_kind;
    __shared__ double s_M;
    for (int i = tid; i < HMAX + 2; i += THREADS) s_hist[i] = 0;
    double m = -INFINITY;
#pragma unroll 4
    for (int i = tid; i < R; i += THREADS) {
        const double x = __ldcg(D.S_logits + i);
        L[i] = x;
        m = fmax(m, x);
    }
    const double M = block_max(m, s_red);  // syncs: L, s_hist ready
    if (DBG_HERE(D) && tid == 0) DBG_TS(D, 52);
    const int hnu = min(hn, D.C - 1);
#pragma unroll 1
    for (int q = warp; q < hn; q += WARPS) {
        const int lo = o.cum[q], hi = o.cum[q + 1];
        double z = 0.0, mn = INFINITY, mx = -INFINITY;
#pragma unroll 2
        for (int i = lo + lane; i < hi; i += 32) {
            const double x = L[i];
            z = __dadd_rn(z, exp_nonpos(__dsub_rn(x, M)));
            mn = fmin(mn, x);
            mx = fmax(mx, x);
            int c = 0;
#pragma unroll
            for (int step = 64; step; step >>= 1)
                if (c + step <= hnu && o.Uo[c + step] >= x) c += step;
            const int st = max(q + 1, c + 1);
            if (st <= hn) atomicAdd(&s_hist[st], 1);
        }
        z = warp_sum(z);
        mn = warp_min(mn);
        mx = warp_max(mx);
        // top-k values of the cluster: k pops of the lanes' running maxima
        const int kk = min(k, hi - lo);
        double cm = -INFINITY;
        int ci = -1;
#pragma unroll 1
        for (int i = lo + lane; i < hi; i += 32)
            if (L[i] > cm) {
                cm = L[i];
                ci = i;
            }
#pragma unroll 1
        for (int r = 0; r < kk; ++r) {
            const double best = warp_max(cm);
            const unsigned win = __ballot_sync(CSVD_FULL, cm == best);
            if (lane == 0) s_tk[q * k + r] = best;
            if (lane == __ffs(win) - 1) {  // the winner drops its maximum and rescans
                L[ci] = -INFINITY;
                cm = -INFINITY;
                ci = -1;
                for (int i = lo + lane; i < hi; i += 32)
                    if (L[i] > cm) {
                        cm = L[i];
                        ci = i;
                    }
            }
            __syncwarp();
        }
        if (lane == 0) {
            s_zq[q] = z;
            s_mnq[q] = mn;
            s_mxq[q] = mx;
        }
    }
    __syncthreads();
    if (DBG_HERE(D) && tid == 0) DBG_TS(D, 53);
    // ---- every prefix at once (warp 0: lane l tests p = l + 1 and l + 33)
    if (warp == 0) {
        int carry = 0;
        double zc = 0.0;
        int first = 0x7fffffff, kind = -1, tie_p = 0x7fffffff;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            const int p = lane + 1 + 32 * h;
            int c = p <= hn ? s_hist[p] : 0;
            double z = p <= hn ? s_zq[p - 1] : 0.0;
#pragma unroll 1
            for (int off = 1; off < 32; off <<= 1) {
                const int u = __shfl_up_sync(CSVD_FULL, c, off);
                const double w = __shfl_up_sync(CSVD_FULL, z, off);
                if (lane >= off) {
                    c += u;
                    z = __dadd_rn(z, w);
                }
            }
            c += carry;
            z = __dadd_rn(z, zc);
            carry = __shfl_sync(CSVD_FULL, c, 31);
            zc = __shfl_sync(CSVD_FULL, z, 31);
            if (p <= hn) {
                s_zq[p - 1] = z;  // now Z(p): the sum over the first p clusters
                const long long n = o.cum[p];
                const double lz = __dadd_rn(M, csvd_log(z));
                const double lr = o.lrh[p];
                int kd = -1;
                if (n > cfg.k_max) {
                    kd = 99;  // budget overflow: the fallback chain (general path)
                } else {
                    for (int ti = 0; ti < cfg.n_targets && kd < 0; ++ti) {
                        const int t = cfg.targets[ti];
                        if (t == CSVD_TARGET_TOPK) {
                            if (n >= k && (p >= D.C || c >= k)) kd = CSVD_KIND_TOPK_EXACT;
                        } else if (t == CSVD_TARGET_SOFTMAX) {
                            if (n > 0 && csvd_rho(lz, lr) <= cfg.epsilon) kd = CSVD_KIND_SOFTMAX_EPS;
                        } else if (n > 0 && csvd_delta(lz, lr) <= csvd_ddiv(cfg.epsilon, __dsub_rn(1.0, cfg.epsilon))) {
                            kd = CSVD_KIND_TOPP_MASS;
                        }
                    }
                }
                if (kd >= 0 && p < first) {
                    first = p;
                    kind = kd;
                }
                if (n > 0)
                    for (int ti = 0; ti < cfg.n_targets; ++ti) {
                        const int t = cfg.targets[ti];
                        if (t == CSVD_TARGET_SOFTMAX && near_tie(csvd_rho(lz, lr), cfg.epsilon)) tie_p = min(tie_p, p);
                        if (t == CSVD_TARGET_TOPP &&
                            near_tie(csvd_delta(lz, lr), csvd_ddiv(cfg.epsilon, __dsub_rn(1.0, cfg.epsilon))))
                            tie_p = min(tie_p, p);
                    }
            }
        }
#pragma unroll 1
        for (int off = 16; off; off >>= 1) {
            const int f2 = __shfl_xor_sync(CSVD_FULL, first, off), k2 = __shfl_xor_sync(CSVD_FULL, kind, off);
            if (f2 < first) {
                first = f2;
                kind = k2;
            }
        }
        tie_p = __reduce_min_sync(CSVD_FULL, (unsigned)tie_p);
        if (lane == 0) {
            s_p = first;
            s_kind = kind;
            s_M = tie_p <= first ? 1.0 : 0.0;  // the tie flag, carried to the result
        }
    }
    __syncthreads();
    const int ps = s_p, kind = s_kind;
    if (DBG_HERE(D) && tid == 0) DBG_TS(D, 54);
    if (ps > hn || kind == 99) return 0;
    const int n = o.cum[ps];
    const int kk = min(k, n);
    if (warp == 0) {
        // k-th largest over the first ps clusters: k pops over their lists
        // (lane l holds cluster l and l + 32)
        int ha = 0, hb = 0;  // list cursors
        const int na = lane < ps ? min(k, o.cum[lane + 1] - o.cum[lane]) : 0;
        const int nb = lane + 32 < ps ? min(k, o.cum[lane + 33] - o.cum[lane + 32]) : 0;
        double kth = -INFINITY;
#pragma unroll 1
        for (int r = 0; r < kk; ++r) {
            const double va = ha < na ? s_tk[lane * k + ha] : -INFINITY;
            const double vb = hb < nb ? s_tk[(lane + 32) * k + hb] : -INFINITY;
            const double best = warp_max(fmax(va, vb));
            const unsigned win = __ballot_sync(CSVD_FULL, va == best || vb == best);
            if (lane == __ffs(win) - 1) {
                if (va == best) ++ha; else ++hb;
            }
            kth = best;
        }
        double lo = INFINITY, hi = -INFINITY;
        if (lane < ps) {
            lo = s_mnq[lane];
            hi = s_mxq[lane];
        }
        if (lane + 32 < ps) {
            lo = fmin(lo, s_mnq[lane + 32]);
            hi = fmax(hi, s_mxq[lane + 32]);
        }
        lo = warp_min(lo);
        hi = warp_max(hi);
        if (lane == 0) {
            const double lz = __dadd_rn(M, csvd_log(s_zq[ps - 1]));
            const double lr = o.lrh[ps];
            const double rho = csvd_rho(lz, lr);
            const double um = ps >= D.C ? -INFINITY : o.Uo[ps];
            double xi;
            if (n < 2 || ps >= D.C) xi = NAN;
            else xi = (um <= lo) ? 1.0 : csvd_ddiv(__dsub_rn(hi, lo), __dsub_rn(um, lo));
            double eps_ach = 0.0;
            if (kind == CSVD_KIND_SOFTMAX_EPS) {
                eps_ach = rho;
            } else if (kind == CSVD_KIND_TOPP_MASS) {
                const double dl = csvd_delta(lz, lr);
                eps_ach = isfinite(dl) ? csvd_ddiv(dl, __dadd_rn(1.0, dl)) : 1.0;
            }
            memset(&res, 0, sizeof(res));
            res.kind = kind;
            res.fallback = CSVD_FB_NONE;
            res.sub_size = n;
            res.clusters_opened = ps;
            res.heap_pops = ps;
            res.epsilon_achieved = eps_ach;
            res.u_max = um;
            res.topk_min = n >= k ? kth : -INFINITY;
            res.rho = rho;
            res.xi = xi;
            res.flags = s_M != 0.0 ? CSVD_FLAG_TIE_AMBIGUOUS : 0;
        }
    }
    __syncthreads();
    return 1;
}

// Fast certification for the common case (CTA 0): the decision is the last
// head prefix p = hn, or an earlier prefix by a softmax / top-p target.
//   per cluster: sum exp(S - M), min, max only (no per-cluster lists)
//   kth_all = k-th largest of the whole head (sorted lane lists of 2 x 8 +
//     REDUX pops per warp, then a pop-merge of the warp lists)
//   top-k at p < hn cannot certify when kth_all <= Uo[p]: kth(p) <= kth_all
//     (the prefix's k-th value is non-decreasing in p).  When kth_all >
//     Uo[p] for some p < hn with the top-k target, or the decision is a p < hn
//     (its own k-th needed), return -1: head_certify (per-cluster lists and
//     the histogram) decides instead.
// Returns 1 decided, 0 general path, -1 use head_certify.
#define HF_CAS(a, x, y)                      \
    {                                        \
        const double hi_ = fmax(a[x], a[y]); \
        a[y] = fmin(a[x], a[y]);             \
        a[x] = hi_;                          \
    }
#define HF_SORT8(a)                                                               \
    HF_CAS(a, 0, 1) HF_CAS(a, 2, 3) HF_CAS(a, 4, 5) HF_CAS(a, 6, 7) HF_CAS(a, 0, 2) \
    HF_CAS(a, 1, 3) HF_CAS(a, 4, 6) HF_CAS(a, 5, 7) HF_CAS(a, 1, 2) HF_CAS(a, 5, 6) \
    HF_CAS(a, 0, 4) HF_CAS(a, 3, 7) HF_CAS(a, 1, 5) HF_CAS(a, 2, 6) HF_CAS(a, 1, 4) \
    HF_CAS(a, 3, 6) HF_CAS(a, 2, 4) HF_CAS(a, 3, 5) HF_CAS(a, 3, 4)
static __device__ __forceinline__ int head_certify_fast(const Dev &D, const Ord &o, int hn, double *L,
                                                     csvd_result &res) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const csvd_config &cfg = *D.cfg;
    const int k = cfg.k;
    const int R = o.cum[hn];
    // certify.py:93-107 with inline libdevice exp / log / division (the same
    // functions csvd_rho / csvd_delta call out of line: identical values)
    auto rho_of = [](double log_z, double lr) {
        if (lr == -INFINITY) return 0.0;
        if (log_z == -INFINITY) return 1.0;
        return __ddiv_rn(1.0, __dadd_rn(1.0, exp(__dsub_rn(log_z, lr))));
    };
    auto delta_of = [](double log_z, double lr) {
        if (lr == -INFINITY) return 0.0;
        if (log_z == -INFINITY) return (double)INFINITY;
        return exp(__dsub_rn(lr, log_z));
    };
    const double dthr = __ddiv_rn(cfg.epsilon, __dsub_rn(1.0, cfg.epsilon));
    __shared__ double s_red[WARPS], s_zq[HMAX], s_mnq[HMAX], s_mxq[HMAX], s_wl[WARPS * KH];
    __shared__ int s_p, s_kind;
    __shared__ double s_kth, s_tie;
    double m = -INFINITY;
#pragma unroll 4
    for (int i = tid; i < R; i += THREADS) {
        const double x = __ldcg(D.S_logits + i);
        L[i] = x;
        m = fmax(m, x);
    }
    const double M = block_max(m, s_red);  // syncs: L ready
    if (DBG_HERE(D) && tid == 0) DBG_TS(D, 52);
    // ---- per cluster: exp sums and extrema
#pragma unroll 1
    for (int q = warp; q < hn; q += WARPS) {
        const int lo = o.cum[q], hi = o.cum[q + 1];
        double z = 0.0, mn = INFINITY, mx = -INFINITY;
#pragma unroll 4
        for (int i = lo + lane; i < hi; i += 32) {
            const double x = L[i];
            z = __dadd_rn(z, exp_nonpos(__dsub_rn(x, M)));
            mn = fmin(mn, x);
            mx = fmax(mx, x);
        }
        z = warp_sum(z);
        mn = warp_min(mn);
        mx = warp_max(mx);
        if (lane == 0) {
            s_zq[q] = z;
            s_mnq[q] = mn;
            s_mxq[q] = mx;
        }
    }
    if (DBG_HERE(D) && tid == 0) DBG_TS(D, 55);
    // ---- the head's top-k: warp w's slice [w R / 8, (w + 1) R / 8), 2 x 8 per lane
    const int kk = min(k, R);
    {
        const int a0 = (int)((long long)R * warp / WARPS), e0 = (int)((long long)R * (warp + 1) / WARPS);
        double va[8], vb[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int i = a0 + lane + 32 * j, i2 = i + 256;
            va[j] = i < e0 ? L[i] : -INFINITY;
            vb[j] = i2 < e0 ? L[i2] : -INFINITY;
        }
        HF_SORT8(va)
        HF_SORT8(vb)
        if (DBG_HERE(D) && tid == 0) DBG_TS(D, 56);
#pragma unroll 1
        for (int r = 0; r < kk; ++r) {
            const double hd = fmax(va[0], vb[0]);
            const unsigned long long key = dkey(hd);
            const unsigned kh = (unsigned)(key >> 32), kl = (unsigned)key;
            const unsigned mh = __reduce_max_sync(CSVD_FULL, kh);
            const unsigned ml = __reduce_max_sync(CSVD_FULL, kh == mh ? kl : 0u);
            const unsigned win = __ballot_sync(CSVD_FULL, kh == mh && kl == ml);
            if (lane == 0) s_wl[warp * KH + r] = dkey_inv(((unsigned long long)mh << 32) | ml);
            if (lane == __ffs(win) - 1) {
                if (va[0] >= vb[0]) {
#pragma unroll
                    for (int j = 0; j < 7; ++j) va[j] = va[j + 1];
                    va[7] = -INFINITY;
                } else {
#pragma unroll
                    for (int j = 0; j < 7; ++j) vb[j] = vb[j + 1];
                    vb[7] = -INFINITY;
                }
            }
        }
    }
    __syncthreads();
    if (DBG_HERE(D) && tid == 0) DBG_TS(D, 53);
    if (warp == 0) {
        // k-th of the head: k pops over the 8 warp lists (lane w < 8: list w, cursor)
        int hc = 0;
        double kth = -INFINITY;
#pragma unroll 1
        for (int r = 0; r < kk; ++r) {
            const double v = (lane < WARPS && hc < kk) ? s_wl[lane * KH + hc] : -INFINITY;
            const double best = warp_max(v);
            const unsigned win = __ballot_sync(CSVD_FULL, v == best && lane < WARPS && hc < kk);
            if (lane == __ffs(win) - 1) ++hc;
            kth = best;
        }
        const double kth_all = R >= k ? kth : -INFINITY;
        if (DBG_HERE(D) && lane == 0) DBG_TS(D, 58);
        // every prefix at once: lane l tests p = l + 1 and l + 33
        double zc = 0.0;
        int first = 0x7fffffff, kind = -1, tie_p = 0x7fffffff, unsure = 0x7fffffff;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            const int p = lane + 1 + 32 * h;
            double z = p <= hn ? s_zq[p - 1] : 0.0;
#pragma unroll 1
            for (int off = 1; off < 32; off <<= 1) {
                const double w = __shfl_up_sync(CSVD_FULL, z, off);
                if (lane >= off) z = __dadd_rn(z, w);
            }
            z = __dadd_rn(z, zc);
            zc = __shfl_sync(CSVD_FULL, z, 31);
            if (p <= hn) {
                s_zq[p - 1] = z;  // Z(p)
                const long long n = o.cum[p];
                const double lz = __dadd_rn(M, log(z));
                const double lr = o.lrh[p];
                int kd = -1;
                if (n > cfg.k_max) {
                    kd = 99;
                } else {
                    for (int ti = 0; ti < cfg.n_targets && kd < 0; ++ti) {
                        const int t = cfg.targets[ti];
                        if (t == CSVD_TARGET_TOPK) {
                            if (n >= k) {
                                const double u = p >= D.C ? -INFINITY : o.Uo[p];
                                if (p == hn) {
                                    if (kth_all > u) kd = CSVD_KIND_TOPK_EXACT;
                                } else if (kth_all > u) {
                                    kd = 98;  // kth(p) unknown here: the full certifier decides
                                }
                            }
                        } else if (t == CSVD_TARGET_SOFTMAX) {
                            if (n > 0 && rho_of(lz, lr) <= cfg.epsilon) kd = CSVD_KIND_SOFTMAX_EPS;
                        } else if (n > 0 && delta_of(lz, lr) <= dthr) {
                            kd = CSVD_KIND_TOPP_MASS;
                        }
                    }
                }
                if (kd >= 0 && p < first) {
                    first = p;
                    kind = kd;
                }
                if (n > 0)
                    for (int ti = 0; ti < cfg.n_targets; ++ti) {
                        const int t = cfg.targets[ti];
                        if (t == CSVD_TARGET_SOFTMAX && near_tie(rho_of(lz, lr), cfg.epsilon)) tie_p = min(tie_p, p);
                        if (t == CSVD_TARGET_TOPP &&
                            near_tie(delta_of(lz, lr), dthr))
                            tie_p = min(tie_p, p);
                    }
            }
        }
#pragma unroll 1
        for (int off = 16; off; off >>= 1) {
            const int f2 = __shfl_xor_sync(CSVD_FULL, first, off), k2 = __shfl_xor_sync(CSVD_FULL, kind, off);
            if (f2 < first) {
                first = f2;
                kind = k2;
            }
        }
        tie_p = __reduce_min_sync(CSVD_FULL, (unsigned)tie_p);
        if (lane == 0) {
            s_p = first;
            s_kind = kind;
            s_kth = kth_all;
            s_tie = tie_p <= first ? 1.0 : 0.0;
        }
    }
    __syncthreads();
    const int ps = s_p, kind = s_kind;
    if (DBG_HERE(D) && tid == 0) DBG_TS(D, 54);
    if (ps > hn || kind == 99) return 0;  // no certificate in the head / budget overflow
    if (kind == 98 || ps < hn) return -1;  // an earlier prefix: its own k-th value is needed
    if (warp == 0) {
        double lo = INFINITY, hi = -INFINITY;
        if (lane < ps) {
            lo = s_mnq[lane];
            hi = s_mxq[lane];
        }
        if (lane + 32 < ps) {
            lo = fmin(lo, s_mnq[lane + 32]);
            hi = fmax(hi, s_mxq[lane + 32]);
        }
        lo = warp_min(lo);
        hi = warp_max(hi);
        if (lane == 0) {
            const int n = o.cum[ps];
            const double lz = __dadd_rn(M, log(s_zq[ps - 1]));
            const double lr = o.lrh[ps];
            const double rho = rho_of(lz, lr);
            const double um = ps >= D.C ? -INFINITY : o.Uo[ps];
            double xi;
            if (n < 2 || ps >= D.C) xi = NAN;
            else xi = (um <= lo) ? 1.0 : __ddiv_rn(__dsub_rn(hi, lo), __dsub_rn(um, lo));
            double eps_ach = 0.0;
            if (kind == CSVD_KIND_SOFTMAX_EPS) {
                eps_ach = rho;
            } else if (kind == CSVD_KIND_TOPP_MASS) {
                const double dl = delta_of(lz, lr);
                eps_ach = isfinite(dl) ? __ddiv_rn(dl, __dadd_rn(1.0, dl)) : 1.0;
            }
            memset(&res, 0, sizeof(res));
            res.kind = kind;
            res.fallback = CSVD_FB_NONE;
            res.sub_size = n;
            res.clusters_opened = ps;
            res.heap_pops = ps;
            res.epsilon_achieved = eps_ach;
            res.u_max = um;
            res.topk_min = s_kth;
            res.rho = rho;
            res.xi = xi;
            res.flags = s_tie != 0.0 ? CSVD_FLAG_TIE_AMBIGUOUS : 0;
        }
    }
    __syncthreads();
    return 1;
}
#undef HF_SORT8
#undef HF_CAS

// Certification from the row CTAs' records (CTA 0).  The per-logit work of
// certify.py:73-88 / 128-139 (exp sums, extrema, the top-k histogram) was done
// by the row CTAs as their rows finished; this reduces the segment records per
// cluster in a fixed order, tests every head prefix at once (as head_certify)
// and selects the decision prefix's k-th logit (np.partition, certify.py:88)
// among the logits at or above the k-th largest segment maximum (at least k
// logits reach it, so the k-th logit does too).
//   log Z_S(p) = est + log(sum over the first p clusters of sum exp(S - est))
//   (est: the best-logit estimate; the max-shifted form's value within ulps)
// The code is deliberately compact (rolled loops, out-of-line libdevice
// calls): it runs once per step on one SM, cold after the rest of the model,
// and its instruction fetch -- not its arithmetic -- is what it costs.
// Returns 1 decided, 0 general path, -1 the records cannot decide (a sum out
// of range, too many candidates): head_certify works from S instead.
static __device__ __noinline__ int seg_prefix_kind(const csvd_config *cfgp, int Cn, int p, long long n, int c,
                                                   double lz, double lr, int *tie) {
    const csvd_config &cfg = *cfgp;
    const double dthr = csvd_ddiv(cfg.epsilon, __dsub_rn(1.0, cfg.epsilon));
    int kd = -1, t2 = 0;
    if (n > cfg.k_max) kd = 99;  // budget overflow: the fallback chain (general path)
#pragma unroll 1
    for (int ti = 0; ti < cfg.n_targets; ++ti) {
        const int t = cfg.targets[ti];
        if (t == CSVD_TARGET_TOPK) {
            if (kd < 0 && n >= cfg.k && (p >= Cn || c >= cfg.k)) kd = CSVD_KIND_TOPK_EXACT;
        } else if (n > 0) {
            const bool sm = t == CSVD_TARGET_SOFTMAX;
            const double v = sm ? csvd_rho(lz, lr) : csvd_delta(lz, lr);
            const double thr = sm ? cfg.epsilon : dthr;
            if (kd < 0 && v <= thr) kd = sm ? CSVD_KIND_SOFTMAX_EPS : CSVD_KIND_TOPP_MASS;
            t2 |= near_tie(v, thr);
        }
    }
    *tie = t2;
    return kd;
}

// What the certifier reads of the step (by value: a noinline callee taking
// const Dev & would read every field through generic loads).
struct SegArgs {
    const int *hcnt;
    const csvd_config *cfg;
    const double *S_logits;
    unsigned long long *dbg;  // null: no timestamps (and always in a warm-up run)
    int C;
};
// warm: a dry run on the certifying CTA while the rows are still in flight.
// It walks the same code (records it cannot match, every phase entered with
// real sizes) and writes only shared memory, so the real run that follows
// finds its instructions in the SM's cache instead of fetching them cold.
static __device__ __noinline__ int head_certify_seg(const SegArgs D, const Ord o, int hn, int Gr, unsigned ep,
                                                    double est, double *scratch, int scratch_n, csvd_result *resp,
                                                    bool warm) {
    csvd_result &res = *resp;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int k = D.cfg->k;
    const HeadRec *rec = reinterpret_cast<const HeadRec *>(D.hcnt + HW_INTS);
    __shared__ double s_zq[HMAX], s_mnq[HMAX], s_mxq[HMAX];
    __shared__ int s_hist[HMAX + 2];
    __shared__ int s_p, s_kind, s_tie, s_nc, s_cnt[HMAX + 1];
    __shared__ double s_T;
    if (scratch_n < THREADS + 64) return -1;  // (tiny d) no room for the candidates
    const int nslots = Gr + hn;
    double *sm = scratch, *cl = scratch + THREADS;  // segment maxima by slot | candidates
    int cap = 2048;  // a power of two: the bitonic sort below pads to one
    while (cap > scratch_n - THREADS) cap >>= 1;
    __shared__ int s_sq[HW_SEGS];                   // segment cluster positions by slot
    if (tid <= hn) s_hist[tid] = __ldcg(D.hcnt + HW_HIST + tid);
    if (tid == 0) {
        s_nc = 0;
        s_T = -INFINITY;
    }
    {  // every segment's maximum, for the k-th threshold below (same round trip as the records)
        double m = -INFINITY;
        int sq = 0x7fffffff;
        if (tid < nslots) {
            const double2 c = __ldcg(reinterpret_cast<const double2 *>(rec + tid) + 1);
            const unsigned long long tag = (unsigned long long)__double_as_longlong(c.y);
            if ((unsigned)(tag >> 32) == ep) {
                m = c.x;
                sq = (int)(unsigned)tag;
            }
        }
        sm[tid] = m;
        s_sq[tid] = sq;
    }
    // per cluster q (warp q % WARPS): its records sit in slots q + b, b < Gr
#pragma unroll 1
    for (int q = warp; q < hn; q += WARPS) {
        double z = 0.0, mn = INFINITY, mx = -INFINITY;
        // all of a lane's record loads in flight at once (Gr <= 160 at 148 SMs)
#pragma unroll 1
        for (int b0 = lane; b0 < Gr; b0 += 5 * 32) {
            double2 a[5], c[5];
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                const int b = b0 + 32 * j;
                const double2 *r = reinterpret_cast<const double2 *>(rec + q + min(b, Gr - 1));
                a[j] = __ldcg(r);
                c[j] = __ldcg(r + 1);
            }
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                const unsigned long long tag = (unsigned long long)__double_as_longlong(c[j].y);
                if (b0 + 32 * j < Gr && (unsigned)(tag >> 32) == ep && (int)(unsigned)tag == q) {
                    z = __dadd_rn(z, a[j].x);
                    mn = fmin(mn, a[j].y);
                    mx = fmax(mx, c[j].x);
                }
            }
        }
#pragma unroll 1
        for (int off = 16; off; off >>= 1) {
            z = __dadd_rn(z, __shfl_xor_sync(CSVD_FULL, z, off));
            mn = fmin(mn, __shfl_xor_sync(CSVD_FULL, mn, off));
            mx = fmax(mx, __shfl_xor_sync(CSVD_FULL, mx, off));
        }
        if (lane == 0) {
            s_zq[q] = z;
            s_mnq[q] = mn;
            s_mxq[q] = mx;
        }
    }
    __syncthreads();
    if (DBG_HERE(D) && tid == 0) DBG_TS(D, 53);
    // While warp 0 tests the prefixes, warps 1..7 prepare the k-th logit of
    // the whole head (the usual decision prefix ps = hn): T = the k-th largest
    // segment maximum (at least k logits reach it, so the k-th logit does
    // too), then the head's logits at or above T.
    const int R = o.cum[hn];
    const bool spec = R >= k && nslots <= THREADS - 32;
    if (warp > 0 && spec) {
        const int t = tid - 32;
        if (t < nslots) {
            const double m = sm[t];
            if (m != -INFINITY) {
                int rank = 0;
#pragma unroll 4
                for (int j = 0; j < nslots; ++j) {
                    const double w = sm[j];
                    rank += (w > m || (w == m && j < t)) ? 1 : 0;
                }
                if (rank == k - 1) s_T = m;
            }
        }
        asm volatile("bar.sync 1, %0;" ::"r"(THREADS - 32) : "memory");
        const double T = s_T;
#pragma unroll 1
        for (int i0 = t; i0 < R; i0 += 8 * (THREADS - 32)) {
            double x[8];  // eight loads in flight
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = __ldcg(D.S_logits + min(i0 + j * (THREADS - 32), R - 1));
#pragma unroll 1
            for (int j = 0; j < 8; ++j)
                if (i0 + j * (THREADS - 32) < R && x[j] >= T) {
                    const int slot = atomicAdd(&s_nc, 1);
                    if (slot < cap) cl[slot] = x[j];
                }
        }
    }
    // ---- every prefix at once (warp 0: lane l tests p = l + 1 and l + 33)
    // every lane also finishes its prefix's outcome values (rho, xi,
    // epsilon_achieved) should it be the decision: no serial tail afterwards
    __shared__ double s_prho[HMAX + 1], s_pxi[HMAX + 1], s_peps[HMAX + 1];
    if (warp == 0) {
        int carry = 0;
        double zc = 0.0, loc = INFINITY, hic = -INFINITY;
        int first = 0x7fffffff, kind = -1, tie_p = 0x7fffffff, bad = 0;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            const int p = lane + 1 + 32 * h;
            int c = p <= hn ? s_hist[p] : 0;
            double z = p <= hn ? s_zq[p - 1] : 0.0;
            double lo = p <= hn ? s_mnq[p - 1] : INFINITY, hi = p <= hn ? s_mxq[p - 1] : -INFINITY;
#pragma unroll 1
            for (int off = 1; off < 32; off <<= 1) {
                const int u = __shfl_up_sync(CSVD_FULL, c, off);
                const double w = __shfl_up_sync(CSVD_FULL, z, off);
                const double wl = __shfl_up_sync(CSVD_FULL, lo, off), wh = __shfl_up_sync(CSVD_FULL, hi, off);
                if (lane >= off) {
                    c += u;
                    z = __dadd_rn(z, w);
                    lo = fmin(lo, wl);
                    hi = fmax(hi, wh);
                }
            }
            c += carry;
            z = __dadd_rn(z, zc);
            lo = fmin(lo, loc);
            hi = fmax(hi, hic);
            carry = __shfl_sync(CSVD_FULL, c, 31);
            zc = __shfl_sync(CSVD_FULL, z, 31);
            loc = __shfl_sync(CSVD_FULL, lo, 31);
            hic = __shfl_sync(CSVD_FULL, hi, 31);
            if (p <= hn) {
                s_zq[p - 1] = z;  // now Z(p)
                s_cnt[p] = c;     // #{logits of the first p clusters > Uo[p]}
                bad |= !(z > 1e-290 && z < 1e290);
                int tie;
                const double lz = __dadd_rn(est, csvd_log(z)), lr = o.lrh[p];
                const int kd = seg_prefix_kind(D.cfg, D.C, p, o.cum[p], c, lz, lr, &tie);
                // certify.py:93-107 and decode.py:212-237 for this prefix
                const double rho = csvd_rho(lz, lr);
                const double um = p >= D.C ? -INFINITY : o.Uo[p];
                const int np = o.cum[p];
                s_prho[p] = rho;
                s_pxi[p] = (np < 2 || p >= D.C) ? NAN : (um <= lo) ? 1.0 : csvd_ddiv(__dsub_rn(hi, lo), __dsub_rn(um, lo));
                double eps_ach = 0.0;
                if (kd == CSVD_KIND_SOFTMAX_EPS) {
                    eps_ach = rho;
                } else if (kd == CSVD_KIND_TOPP_MASS) {
                    const double dl = csvd_delta(lz, lr);
                    eps_ach = isfinite(dl) ? csvd_ddiv(dl, __dadd_rn(1.0, dl)) : 1.0;
                }
                s_peps[p] = eps_ach;
                if (kd >= 0 && p < first) {
                    first = p;
                    kind = kd;
                }
                if (tie) tie_p = min(tie_p, p);
            }
        }
#pragma unroll 1
        for (int off = 16; off; off >>= 1) {
            const int f2 = __shfl_xor_sync(CSVD_FULL, first, off), k2 = __shfl_xor_sync(CSVD_FULL, kind, off);
            if (f2 < first) {
                first = f2;
                kind = k2;
            }
        }
        tie_p = __reduce_min_sync(CSVD_FULL, (unsigned)tie_p);
        bad = __any_sync(CSVD_FULL, bad);
        if (lane == 0) {
            s_p = warm ? 1 : bad ? -1 : first;
            s_kind = warm ? CSVD_KIND_TOPK_EXACT : kind;
            s_tie = tie_p <= first;
        }
    }
    __syncthreads();
    const int ps = s_p, kind = s_kind;
    if (DBG_HERE(D) && tid == 0) DBG_TS(D, 54);
    if (ps < 0) return -1;
    if (ps > hn || kind == 99) return 0;
    const int n = o.cum[ps];
    double kth = -INFINITY;
    if (n >= k) {
        if (!(spec && ps == hn)) {
            // an earlier decision prefix: T and the candidates over its clusters only
            if (tid == 0) {
                s_nc = 0;
                s_T = -INFINITY;
            }
            __syncthreads();
            const double m = (tid < nslots && s_sq[tid] < ps) ? sm[tid] : -INFINITY;
            if (m != -INFINITY) {
                int rank = 0;
#pragma unroll 4
                for (int j = 0; j < nslots; ++j) {
                    const double w = (s_sq[j] < ps) ? sm[j] : -INFINITY;
                    rank += (w > m || (w == m && j < tid)) ? 1 : 0;
                }
                if (rank == k - 1) s_T = m;
            }
            __syncthreads();
            const double T = s_T;
#pragma unroll 1
            for (int i0 = tid; i0 < n; i0 += 8 * THREADS) {
                double x[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) x[j] = __ldcg(D.S_logits + min(i0 + j * THREADS, n - 1));
#pragma unroll 1
                for (int j = 0; j < 8; ++j)
                    if (i0 + j * THREADS < n && x[j] >= T) {
                        const int slot = atomicAdd(&s_nc, 1);
                        if (slot < cap) cl[slot] = x[j];
                    }
            }
            __syncthreads();
        }
        const int nc = warm ? min(s_nc, THREADS) : s_nc;  // a dry run stays inside the buffers
        if (DBG_HERE(D) && tid == 0) DBG_TS(D, 56);
        if (!warm && (nc > cap || nc < k)) return -1;
        if (nc <= THREADS) {  // one candidate per thread: its rank by counting
            if (tid < nc) {
                const double v = cl[tid];
                int rank = 0;
#pragma unroll 4
                for (int j = 0; j < nc; ++j) {
                    const double w = cl[j];
                    rank += (w > v || (w == v && j < tid)) ? 1 : 0;
                }
                if (rank == k - 1) s_T = v;
            }
            __syncthreads();
            kth = s_T;
        } else {
        // bitonic sort (descending) of the candidates, padded to a power of two
        int m2 = 32;
        while (m2 < nc) m2 <<= 1;
        for (int i = nc + tid; i < m2; i += THREADS) cl[i] = -INFINITY;
        __syncthreads();
#pragma unroll 1
        for (int size = 2; size <= m2; size <<= 1) {
#pragma unroll 1
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll 1
                for (int i = tid; i < (m2 >> 1); i += THREADS) {
                    const int a = 2 * i - (i & (stride - 1)), bq = a + stride;
                    const double va = cl[a], vb = cl[bq];
                    if ((va < vb) == ((a & size) == 0)) {
                        cl[a] = vb;
                        cl[bq] = va;
                    }
                }
                __syncthreads();
            }
        }
        kth = cl[k - 1];
        }
        if (DBG_HERE(D) && tid == 0) {
            DBG_TS(D, 58);
            D.dbg[60] = nc;
        }
    }
    if (tid == 0) {
        memset(&res, 0, sizeof(res));
        res.kind = kind;
        res.fallback = CSVD_FB_NONE;
        res.sub_size = n;
        res.clusters_opened = ps;
        res.heap_pops = ps;
        res.epsilon_achieved = s_peps[ps];
        res.u_max = ps >= D.C ? -INFINITY : o.Uo[ps];
        res.topk_min = kth;
        res.rho = s_prho[ps];
        res.xi = s_pxi[ps];
        res.flags = s_tie ? CSVD_FLAG_TIE_AMBIGUOUS : 0;
    }
    __syncthreads();
    return 1;
}

// The head path; returns true when the step needs the general path (every
// CTA of the grid / lane returns the same), which the caller then runs from
// scratch: one call site, so one copy of its code, after the head path's.
template <typename ET, int Q, bool GROUPED>
__device__ __forceinline__ bool head_path(const Dev &D) {
    extern __shared__ __align__(16) double smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int G = CTA_N, b = CTA_ID;
    double *hs = smem;
    double *ws = smem + D.ord_off;
    double *sws = smem + D.sum_off;
    __shared__ ScanShared ss;
    __shared__ unsigned long long s_hbar, s_epoch;
    __shared__ double s_qn;
    __shared__ int s_hist[HMAX + 2];  // this CTA's top-k histogram counts
    for (int i = tid; i < HMAX + 2; i += THREADS) s_hist[i] = 0;
    const bool lead = b == 0 && tid == 0;
    if (lead) DBG_TS(D, 24);
    if (tid == 0) {
        mbar_init(&s_hbar, 1);
        if constexpr (GROUPED) {  // this lane's step number: no grid barrier in a lane
            unsigned long long e;
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(e) : "l"(D.bar64) : "memory");
            s_epoch = e + 1;
        }
    }
    __syncthreads();
    if constexpr (!GROUPED) {  // CSVD_PF bit 64: this warp's centroid rows stream to L2 while h is staged
        // (measured: h staging slows from 1.5 to 3.7 us and the step does not gain; off)
        if ((D.pf_mask & 64) && lane == 0) {
            int j = 0;
            for (int c = warp * G + b; c < D.C && j < MAX_PER_WARP; c += G * WARPS, ++j)
                bulk_prefetch_l2(D.cent + (size_t)c * D.bd, sizeof(double) * D.bd);
        }
    }
    tma_stage_leaves(D.wplan, D.h, D.d, 1, hs, 0, &s_hbar, 0);
    if (b == 1 % G && warp == 0 && lane == 0) {  // per-cluster arrays the head and rows read next
        bulk_prefetch_l2(D.logsz, sizeof(double) * D.C);
        bulk_prefetch_l2(D.meanb, sizeof(double) * D.C);
        bulk_prefetch_l2(D.sizes, sizeof(int) * D.C);
        bulk_prefetch_l2(D.starts, sizeof(int) * D.C);
        bulk_prefetch_l2(D.wrow0, sizeof(int) * D.C);
    }
    if (lead) DBG_TS(D, 25);
    if constexpr (GROUPED) {  // batch lane: the dots come from k_bounds_batch, ||h|| here
        lane_query_norm<Q>(D, hs, s_qn);
    } else {
        const double qn = head_bounds<Q>(D, hs);
        if (lead) {
            D.res->query_norm = qn;
            s_qn = qn;
            DBG_TS(D, 26);
        }
        const unsigned long long e = grid_sync_mono(D, D.bar64);
        if (tid == 0) s_epoch = e;
        __syncthreads();
    }
    const double qn = s_qn;
    if (lead) DBG_TS(D, 27);
    // ---- the head of the opening order (every CTA, identically)
    Ord o;
    ord_bind(D, ws, o);
    __shared__ double s_slack, s_est;
    const bool ok = stage_bounds(D, o, qn, &s_slack);
    if (lead) DBG_TS(D, 32);
    // row CTAs skip log R-hat (only the certifier reads it); a residual too
    // small for the direct form is then seen by CTA 0 alone, which declares
    // the step undecided once the rows are in (hfail)
    int hfail = 0;
    const int hn = ok ? order_head(D, o, s_est, b == 0, &hfail) : 0;
    if (hn == 0) {  // every CTA sees the same: the general step decides
        __syncthreads();
        return true;
    }
    if (lead) DBG_TS(D, 28);
    const unsigned long long epoch = s_epoch;
    unsigned long long *decision = D.bar64 + 1;  // epoch * 2 + decided
    const int R = o.cum[hn];
    // small lanes (G <= 3 CTAs): CTA 0 computes rows too, then certifies
    const bool cta0_rows = G <= 3;
    const int Gr = cta0_rows ? G : G - 1;          // row CTAs
    const bool segs = Gr + hn <= HW_SEGS;          // segment records fit (always at 148 CTAs)
    if (b > 0 || cta0_rows) {
        // ---- rows of the head, contiguous per row CTA
        const int rb = cta0_rows ? b : b - 1;
        const int r_lo = (int)((long long)R * rb / Gr), r_hi = (int)((long long)R * (rb + 1) / Gr);
        // top-k histogram (certify.py:128-139 as counts): a logit x of cluster
        // position q counts for every prefix p >= max(q + 1, c + 1),
        // c = #{p in [1, hnu] : Uo[p] >= x}
        const int hnu = min(hn, D.C - 1);
        auto tally = [&](double x, int q) {
            int c = 0;
#pragma unroll
            for (int step = 64; step; step >>= 1)
                if (c + step <= hnu && o.Uo[c + step] >= x) c += step;
            const int st = max(q + 1, c + 1);
            if (st <= hn) atomicAdd(&s_hist[st], 1);
        };
        // the head clusters' first W row / position, staged once per CTA
        __shared__ int s_pos0[HMAX], s_wrow0[HMAX];
        if (tid < hn) {
            const int c = o.order[tid];
            s_pos0[tid] = __ldg(D.starts + c);
            s_wrow0[tid] = __ldg(D.wrow0 + c);
        }
        __syncthreads();
        if ((D.pf_mask & 4) && tid == 0 && r_hi > r_lo) {
            // this CTA's W rows (1-3 contiguous runs, one per cluster segment) towards L2
            // at once: the warps' own loads then find them there
            const size_t rb_bytes = (size_t)D.d * sizeof(ET);
            for (int q = 0; q < hn; ++q) {
                const int a = max(o.cum[q], r_lo), e = min(o.cum[q + 1], r_hi);
                if (e > a)
                    bulk_prefetch_l2(reinterpret_cast<const char *>(D.W) + (size_t)(s_wrow0[q] + a - o.cum[q]) * rb_bytes,
                                     (size_t)(e - a) * rb_bytes);
            }
        }
        // two rows per warp at a time (r, r + WARPS): both in flight, h read once
        auto locate = [&](int r, int &wrow, int &pos) {
            int lo = 0, hi = hn;  // cum[lo] <= r < cum[lo+1]
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (o.cum[mid] <= r) lo = mid; else hi = mid;
            }
            const int i = r - o.cum[lo];
            pos = s_pos0[lo] + i;
            wrow = s_wrow0[lo] + i;
            return lo;
        };
        const ET *Wt = reinterpret_cast<const ET *>(D.W);
        // A warp with several row pairs (batch lanes: ~150 rows per warp)
        // streams them with little in flight; its lane 0 keeps the rows of the
        // pair PFD iterations ahead on their way to L2 (CSVD_PF bit 32: off)
        constexpr int PFD = 3;
        const size_t row_bytes = (size_t)D.d * sizeof(ET);
        // rows of <= 8 KB only: larger rows put more ahead in flight than L2 keeps
        // (c4, 32 KB f32 rows: 1.37 ms per batch against 1.27 ms without)
        const bool pf_ahead = !(D.pf_mask & 32) && r_hi - r_lo > 4 * WARPS && row_bytes <= 8192;
        auto prefetch_pair = [&](int r) {
            if (r < r_hi) {
                int w, pp;
                locate(r, w, pp);
                bulk_prefetch_l2(Wt + (size_t)w * D.d, row_bytes);
            }
            if (r + WARPS < r_hi) {
                int w, pp;
                locate(r + WARPS, w, pp);
                bulk_prefetch_l2(Wt + (size_t)w * D.d, row_bytes);
            }
        };
        if (pf_ahead && lane == 0)
            for (int j = 0; j < PFD; ++j) prefetch_pair(r_lo + warp + j * 2 * WARPS);
#pragma unroll 1
        for (int r = r_lo + warp; r < r_hi; r += 2 * WARPS) {
            if (pf_ahead && lane == 0) prefetch_pair(r + PFD * 2 * WARPS);
            const int r2 = r + WARPS;
            int wa, pa, wb, pb, qb = 0;
            const int qa = locate(r, wa, pa);
            if (r2 < r_hi) qb = locate(r2, wb, pb);
            else {
                wb = wa;
                pb = pa;
            }
            // bias and token id first: their loads wait alongside the row's
            const double ba = __ldg(D.bias + pa), bb = __ldg(D.bias + pb);
            const int ia = __ldg(D.perm + pa), ib = __ldg(D.perm + pb);
            double la, lb;
            warp_dot_r8_x2<ET, Q>(Wt + (size_t)wa * D.d, Wt + (size_t)wb * D.d, hs, D.wplan.leaf_len, lane, la, lb);
            if (lane == 0) {
                const double xa = __dadd_rn(la, ba);
                D.S_logits[r] = xa;
                D.S_ids[r] = ia;
                if (segs) tally(xa, qa);
                if (r2 < r_hi) {
                    const double xb = __dadd_rn(lb, bb);
                    D.S_logits[r2] = xb;
                    D.S_ids[r2] = ib;
                    if (segs) tally(xb, qb);
                }
            }
        }
        __syncthreads();  // the rows are published by the release operations below
        if (segs) {
            // this CTA's histogram counts (integer adds: order-independent) and
            // one record per cluster its rows touch, reduced in a fixed order
            if (tid <= hn && s_hist[tid]) atomicAdd(D.hcnt + HW_HIST + tid, s_hist[tid]);
            if (r_hi > r_lo) {
                auto cluster_of = [&](int r) {
                    int lo = 0, hi = hn;
                    while (hi - lo > 1) {
                        const int mid = (lo + hi) >> 1;
                        if (o.cum[mid] <= r) lo = mid; else hi = mid;
                    }
                    return lo;
                };
                const int qa = cluster_of(r_lo), qz = cluster_of(r_hi - 1);
                const double est = s_est;
                const unsigned ep = (unsigned)s_epoch;
#pragma unroll 1
                for (int q = qa + warp; q <= qz; q += WARPS) {
                    const int a = max(o.cum[q], r_lo), e = min(o.cum[q + 1], r_hi);
                    double z = 0.0, mn = INFINITY, mx = -INFINITY;
#pragma unroll 1
                    for (int i = a + lane; i < e; i += 32) {
                        const double x = __ldcg(D.S_logits + i);
                        // x - est > 700 (never for a sane index) makes z huge: the certifier's range check
                        z = __dadd_rn(z, exp_nonpos(fmin(__dsub_rn(x, est), 700.0)));
                        mn = fmin(mn, x);
                        mx = fmax(mx, x);
                    }
                    z = warp_sum(z);
                    mn = warp_min(mn);
                    mx = warp_max(mx);
                    if (lane == 0) {
                        double2 *rp = reinterpret_cast<double2 *>(hw_recs(D) + rb + q);
                        const unsigned long long tag = ((unsigned long long)ep << 32) | (unsigned)q;
                        rp[0] = make_double2(z, mn);
                        rp[1] = make_double2(mx, __longlong_as_double((long long)tag));
                    }
                }
            }
            __syncthreads();
        }
        if (D.dbg && tid == 0) D.dbg[384 + (b & 255)] = gtimer();
        if (D.res_host) {  // host-API step: this CTA's rows into the mapped buffers (speculative:
                           // the host reads only the first |S| entries)
            for (int r = r_lo + tid; r < r_hi; r += THREADS) {
                D.logits_host[r] = __ldcg(D.S_logits + r);
                D.ids_host[r] = __ldcg(D.S_ids + r);
            }
        }
        if (b > 0) {  // its arrival (release: rows, records and counts visible first), and CTA 0's decision
            if (tid == 0) red_release_add(D.hcnt + HMAX, 1);
            // ---- wait for CTA 0's decision
            __shared__ int s_dec;
            if (tid == 0) {
                // relaxed polls with a back-off (147 CTAs polling one line must
                // not crowd L2 while CTA 0 works), one acquire fence at the end
                unsigned long long v, spins = 0;
                while (true) {
                    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(decision) : "memory");
                    if ((v >> 1) >= epoch) break;
                    if (++spins > (1ull << 24)) {
                        D.res->error = CSVD_ESTATE;
                        v = epoch * 2 + 1;
                        break;
                    }
                    __nanosleep(256);
                }
                (void)ld_acquire_u64(decision);  // acquire: CTA 0's result is ordered before what follows
                s_dec = (int)(v & 1);
                if (D.dbg && b < 256) D.dbg[128 + b] = gtimer();
            }
            __syncthreads();
            return !s_dec;  // undecided: the general step, from scratch
        }
    }
    // ---- CTA 0: optionally (CSVD_PF bit 8) warm the certifier's code while the
    // rows run -- ~1 us faster while CTA 0 also built log R-hat ahead of the
    // rows, on the critical path (+1 us) since the row CTAs skip it -- then
    // wait for every row CTA's arrival and certify
    __shared__ csvd_result s_res;
    if (tid == 0) init_state(D, o, ss, hn, s_est);  // only the certifying CTA needs the scan state
    if (!cta0_rows && segs && !hfail && (D.pf_mask & 8)) {
        const SegArgs wa{D.hcnt, D.cfg, D.S_logits, nullptr, D.C};
        (void)head_certify_seg(wa, o, hn, Gr, 0xffffffffu, s_est, hs, pw_hs_size(D.wplan), &s_res, true);
        if (lead) DBG_TS(D, 51);
    }
    if (G > 1) {
        if (tid == 0) {
            const int n = G - 1;
            const int *ctr = D.hcnt + HMAX;
            unsigned long long spins = 0;
            int v;
            do {
                asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
                if (++spins > (1ull << 26)) {
                    D.res->error = CSVD_ESTATE;
                    break;
                }
            } while (v < n);
            (void)ld_acquire_s32(ctr);  // acquire: the counted rows are visible to this CTA after the barrier
        }
        __syncthreads();
    }
    if (lead) DBG_TS(D, 29);
    bool decided;
    const bool fits = head_fits(D, o, hn) && D.cfg->k <= KH;
    const SegArgs sa{D.hcnt, D.cfg, D.S_logits, DBG_HERE(D) ? D.dbg : nullptr, D.C};
    const int fs = hfail ? 0
                   : segs ? head_certify_seg(sa, o, hn, Gr, (unsigned)epoch, s_est, hs, pw_hs_size(D.wplan), &s_res, false)
                          : -1;
    if (lead && D.dbg) {
        if (fs < 0) D.dbg[60] = fits ? 1 : 2;
        D.dbg[61] = hn;
        D.dbg[62] = o.cum[hn];
    }
    if (lead && D.dbg) D.dbg[63] = (unsigned long long)(fs + 2);
    if (fs >= 0) {
        decided = fs != 0;
    } else if (fits) {
        const int f = (o.cum[hn] <= 2 * THREADS * 8) ? head_certify_fast(D, o, hn, hs, s_res) : -1;
        if (lead && D.dbg) D.dbg[59] = (unsigned long long)(f + 2);
        decided = f < 0 ? head_certify(D, o, hn, hs, s_res) != 0 : f != 0;
    } else {  // a head larger than the h staging area: per-cluster summaries + the sequential scan
        const int k = D.cfg->k;
        double *c_vals = sws, *c_lse = sws + 6 * CHUNK, *c_min = c_lse + CHUNK, *c_max = c_min + CHUNK;
        double *la = D.klists ? D.klists + (size_t)CTA_ID * D.klist_stride : c_max + CHUNK;
        double *lb = la + D.K, *c_topk = lb + D.K;
        double reg_list = -INFINITY;
        for (int q0 = 0; q0 < hn; q0 += D.chunk) {
            const int q1 = min(hn, q0 + D.chunk);
            for (int q = q0 + warp; q < q1; q += WARPS) {
                double pre[SUM_E];
                summary_load(D, o.cum[q], o.cum[q + 1], pre, lane);
                cluster_summary(D, o.cum[q], o.cum[q + 1], k, c_topk + (q - q0) * k, c_lse + (q - q0),
                                c_min + (q - q0), c_max + (q - q0), pre, lane);
            }
            __syncthreads();
            if (warp == 0) scan_chunk(D, o, ss, q0, q1, c_topk, c_lse, c_min, c_max, c_vals, la, lb, reg_list, lane);
            __syncthreads();
            if (ss.st.phase != PH_MAIN && ss.st.phase != PH_PE) break;
        }
        decided = ss.st.phase == PH_DONE;
        if (tid == 0) {
            s_res = ss.res;
            s_res.flags = ss.flags;
        }
        __syncthreads();
    }
    if (lead) DBG_TS(D, 31);
    if (tid == 0) {
        // the decision first: the row CTAs only need this word (and exit or
        // start the general step); the result below is read after the kernel
        if constexpr (GROUPED) D.bar64[0] = epoch;  // the lane's step count (read before the next step)
        const unsigned long long w = epoch * 2 + (decided ? 1 : 0);
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(decision), "l"(w) : "memory");
        DBG_TS(D, 30);
    }
    // every row CTA has added its counts and arrived: reset
    for (int q = tid; q < HW_INTS; q += THREADS) D.hcnt[q] = 0;  // arrivals, histogram
    if (tid == 0) {
        if (decided) {
            csvd_result r = s_res;
            r.query_norm = qn;
            r.slack = s_slack;
            r.waves = 1;
            r.error = __ldcg(&D.res->error);
            *D.res = r;
            ScanState s2 = ss.st;
            s2.mode = MODE_IDLE;
            s2.phase = PH_DONE;
            s2.p = r.clusters_opened;
            s2.iter = 1;
            *D.st = s2;
            if (D.res_host) *D.res_host = r;
        }
    }
    __syncthreads();
    return !decided;
}

template <typename ET, int Q>
__global__ void __launch_bounds__(THREADS, 1) k_head(const __grid_constant__ Dev D) {
    if (head_path<ET, Q, false>(D)) step_body<ET, 8, Q, 8, Q>(D);
}

// batch lanes: lane b is blockIdx.x / nblocks and swaps its own workspaces
// into the Dev (all table data is shared); bounds come from k_bounds_batch
template <typename ET, int Q>
__global__ void __launch_bounds__(THREADS, 1) k_head_lanes(const __grid_constant__ Dev D0) {
    // the lane's Dev lives in shared memory: a local copy would sit in local
    // memory, whose L1 lines every acquire / fence of the step invalidates
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
        D.hcnt = w.hcnt;
        D.bar64 = w.bar64;
        D.dbg = blockIdx.x == 0 ? D0.dbg : nullptr;  // debug timestamps follow lane 0's CTA 0
    }
    __syncthreads();
    if (head_path<ET, Q, true>(D)) step_body<ET, 8, Q, 8, Q>(D);
}
