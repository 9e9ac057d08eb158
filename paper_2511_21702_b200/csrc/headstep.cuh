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
//         buffers); then one release-add per touched cluster  decode.py:169-176
//   CTA 0 (the certifying CTA) does no rows: while they run it executes the
//         summary and scan code once on scratch data (the code is cold after
//         the L2 flush / the rest of a model, and a cold instruction stream
//         costs more than the work), then its warps summarise each cluster as
//         its counter completes (top-k values, log-sum-exp, min, max;
//         certify.py:73-88) and warp 0 runs the certification scan
//         (scan.cuh, decode.py:192-210), and publishes a decision word.
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

// ---------------------------------------------------------------------------
// Block-parallel certification of the head (CTA 0, all warps): every prefix
// p = 1..hn of the head is tested at once instead of cluster by cluster.
//   log Z_S(p)  = M + log(sum_{i < cum[p]} exp(S_i - M)): one block scan over
//                 the positions (certify.py:79-83; the same value the
//                 reference's logaddexp chain / 64-merge recompute converge
//                 to, within ulps)
//   top-k test  u_max(p) < kth(p)  <=>  #{i < cum[p] : S_i > Uo[p]} >= k
//                 (certify.py:128-139): each logit adds 1 to every prefix from
//                 max(q(i) + 1, first p with Uo[p] < S_i) on (Uo is
//                 non-increasing), a histogram + prefix sum
//   rho / delta from log Z_S(p) and log R-hat(p)          (certify.py:93-107)
// The first prefix with an event (budget overflow or a certified target, in
// the configured target order; decode.py:192-210, 329-342) is the decision.
// Its k-th logit (np.partition, certify.py:88), min / max (xi) follow by
// block selections.  Returns 1 = decided (res filled), 0 = the step needs the
// general path (overflow -> fallback chain, or no certificate in the head).
// Logits live in registers: thread t holds positions [t*HJ, (t+1)*HJ).
// ---------------------------------------------------------------------------
#define HJ 16  // positions per thread: heads of up to THREADS * HJ = 4096 tokens
static __device__ __forceinline__ bool head_fits(const Ord &o, int hn) { return o.cum[hn] <= THREADS * HJ; }

static __device__ __noinline__ int head_certify(const Dev &D, const Ord &o, int hn, csvd_result &res) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const csvd_config &cfg = *D.cfg;
    const int k = cfg.k;
    const int R = o.cum[hn];
    __shared__ double s_red[WARPS], s_z[HMAX + 1], s_wl[WARPS * KH];
    __shared__ int s_hist[HMAX + 2], s_cnt[HMAX + 1];
    __shared__ int s_p, s_kind;
    __shared__ double s_kth;
    for (int i = tid; i < HMAX + 2; i += THREADS) s_hist[i] = 0;
    // ---- the head's logits, contiguous per thread
    const int i0 = tid * HJ;
    double v[HJ];
#pragma unroll
    for (int j = 0; j < HJ; j += 2) {
        if (i0 + j + 1 < R) {
            const double2 t = __ldcg(reinterpret_cast<const double2 *>(D.S_logits + i0 + j));
            v[j] = t.x;
            v[j + 1] = t.y;
        } else {
            v[j] = i0 + j < R ? __ldcg(D.S_logits + i0 + j) : -INFINITY;
            v[j + 1] = -INFINITY;
        }
    }
    double m = -INFINITY;
#pragma unroll
    for (int j = 0; j < HJ; ++j) m = fmax(m, v[j]);
    const double M = block_max(m, s_red);  // syncs: s_hist zeroed too
    // ---- per-position exp(S - M): thread-local inclusive scan, then warp / block
    double e[HJ], tot = 0.0;
#pragma unroll
    for (int j = 0; j < HJ; ++j) {
        e[j] = i0 + j < R ? exp_nonpos(__dsub_rn(v[j], M)) : 0.0;
        tot = __dadd_rn(tot, e[j]);
        e[j] = tot;
    }
    double wi = tot;  // warp inclusive scan of thread totals
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double u = __shfl_up_sync(CSVD_FULL, wi, off);
        if (lane >= off) wi = __dadd_rn(wi, u);
    }
    __syncthreads();
    if (lane == 31) s_red[warp] = wi;
    // ---- top-k histogram: element i counts for prefixes >= max(q(i) + 1, p0(i))
    int q = 0;
    if (i0 < R) {
        int lo = 0, hi = hn;  // cum[lo] <= i0 < cum[lo+1]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (o.cum[mid] <= i0) lo = mid; else hi = mid;
        }
        q = lo;
    }
#pragma unroll
    for (int j = 0; j < HJ; ++j) {
        const int i = i0 + j;
        if (i < R) {
            while (o.cum[q + 1] <= i) ++q;
            int lo = 1, hi = hn + 1;  // first p in [1, hn] with Uo[p] < S_i, else hn + 1
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if ((mid >= D.C ? -INFINITY : o.Uo[mid]) < v[j]) hi = mid; else lo = mid + 1;
            }
            const int st = max(q + 1, lo);
            if (st <= hn) atomicAdd(&s_hist[st], 1);
        }
    }
    __syncthreads();
    double base = 0.0;  // exclusive block prefix of this warp
    for (int w = 0; w < warp; ++w) base = __dadd_rn(base, s_red[w]);
    const double excl = __dadd_rn(base, __dsub_rn(wi, tot));  // before this thread's first position
    // Z(p) = inclusive sum at position cum[p] - 1, written by its owner
    for (int pp = 1; pp <= hn; ++pp) {
        const int last = o.cum[pp] - 1;
        if (last >= i0 && last < i0 + HJ) {
#pragma unroll
            for (int j = 0; j < HJ; ++j)
                if (i0 + j == last) s_z[pp] = __dadd_rn(excl, e[j]);
        }
    }
    __syncthreads();
    // ---- every prefix at once (warp 0: lane l tests p = l + 1 and l + 33)
    if (warp == 0) {
        int carry = 0;
        int first = 0x7fffffff, kind = -1;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int p = lane + 1 + 32 * h;
            int c = p <= hn ? s_hist[p] : 0;
#pragma unroll
            for (int off = 1; off < 32; off <<= 1) {
                const int u = __shfl_up_sync(CSVD_FULL, c, off);
                if (lane >= off) c += u;
            }
            c += carry;
            carry = __shfl_sync(CSVD_FULL, c, 31);
            if (p <= hn) {
                s_cnt[p] = c;
                const long long n = o.cum[p];
                const double lz = __dadd_rn(M, csvd_log(s_z[p]));
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
            }
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) {
            const int f2 = __shfl_xor_sync(CSVD_FULL, first, off), k2 = __shfl_xor_sync(CSVD_FULL, kind, off);
            if (f2 < first) {
                first = f2;
                kind = k2;
            }
        }
        if (lane == 0) {
            s_p = first;
            s_kind = kind;
        }
    }
    __syncthreads();
    const int ps = s_p, kind = s_kind;
    if (ps > hn || kind == 99) return 0;
    // ---- the decision prefix: k-th largest, min, max over positions < cum[ps]
    const int n = o.cum[ps];
    double mn = INFINITY, mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < HJ; ++j) {
        if (i0 + j >= n) v[j] = -INFINITY;
        else mn = fmin(mn, v[j]);
        mx = fmax(mx, v[j]);
    }
    mn = warp_min(mn);
    mx = warp_max(mx);
    // per warp: k pops of the largest remaining value (REDUX on order-preserving keys)
    const int kk = min(k, n);
#pragma unroll 1
    for (int r = 0; r < kk; ++r) {
        double hd = -INFINITY;
#pragma unroll
        for (int j = 0; j < HJ; ++j) hd = fmax(hd, v[j]);
        const unsigned long long key = dkey(hd);
        const unsigned kh = (unsigned)(key >> 32), kl = (unsigned)key;
        const unsigned mh = __reduce_max_sync(CSVD_FULL, kh);
        const unsigned ml = __reduce_max_sync(CSVD_FULL, kh == mh ? kl : 0u);
        const unsigned win = __ballot_sync(CSVD_FULL, kh == mh && kl == ml);
        if (lane == 0) s_wl[warp * KH + r] = dkey_inv(((unsigned long long)mh << 32) | ml);
        if (lane == __ffs(win) - 1) {
            bool done = false;
#pragma unroll
            for (int j = 0; j < HJ; ++j)
                if (!done && v[j] == hd) {
                    v[j] = -INFINITY;
                    done = true;
                }
        }
    }
    __shared__ double s_mxw[WARPS];
    __syncthreads();
    if (lane == 0) {
        s_red[warp] = mn;
        s_mxw[warp] = mx;
    }
    if (warp == 0) {
        // merge the warps' lists: lane l holds the l-th entry of every warp's list
        double u[WARPS];
#pragma unroll
        for (int w = 0; w < WARPS; ++w) u[w] = lane < kk ? s_wl[w * KH + lane] : -INFINITY;
        double kth = -INFINITY;
#pragma unroll 1
        for (int r = 0; r < kk; ++r) {
            double hd = -INFINITY;
#pragma unroll
            for (int w = 0; w < WARPS; ++w) hd = fmax(hd, u[w]);
            const unsigned long long key = dkey(hd);
            const unsigned kh = (unsigned)(key >> 32), kl = (unsigned)key;
            const unsigned mh = __reduce_max_sync(CSVD_FULL, kh);
            const unsigned ml = __reduce_max_sync(CSVD_FULL, kh == mh ? kl : 0u);
            const unsigned win = __ballot_sync(CSVD_FULL, kh == mh && kl == ml);
            kth = dkey_inv(((unsigned long long)mh << 32) | ml);
            if (lane == __ffs(win) - 1) {
                bool done = false;
#pragma unroll
                for (int w = 0; w < WARPS; ++w)
                    if (!done && u[w] == hd) {
                        u[w] = -INFINITY;
                        done = true;
                    }
            }
        }
        if (lane == 0) s_kth = n >= k ? kth : -INFINITY;
    }
    __syncthreads();
    if (tid == 0) {
        double lo = s_red[0], hi = s_mxw[0];
        for (int w = 1; w < WARPS; ++w) {
            lo = fmin(lo, s_red[w]);
            hi = fmax(hi, s_mxw[w]);
        }
        const double lz = __dadd_rn(M, csvd_log(s_z[ps]));
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
        res.topk_min = s_kth;
        res.rho = rho;
        res.xi = xi;
    }
    __syncthreads();
    return 1;
}

template <typename ET, int Q>
__global__ void __launch_bounds__(THREADS, 1) k_head(const __grid_constant__ Dev D) {
    extern __shared__ __align__(16) double smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int G = gridDim.x, b = blockIdx.x;
    double *hs = smem;
    double *ws = smem + D.ord_off;
    double *sws = smem + D.sum_off;
    __shared__ ScanShared ss;
    __shared__ unsigned long long s_hbar, s_epoch;
    const bool lead = b == 0 && tid == 0;
    if (lead) DBG_TS(D, 24);
    if (tid == 0) mbar_init(&s_hbar, 1);
    __syncthreads();
    tma_stage_leaves(D.wplan, D.h, D.d, 1, hs, 0, &s_hbar, 0);
    if (b == 1 % G && warp == 0 && lane == 0) {  // per-cluster arrays the head and rows read next
        bulk_prefetch_l2(D.logsz, sizeof(double) * D.C);
        bulk_prefetch_l2(D.meanb, sizeof(double) * D.C);
        bulk_prefetch_l2(D.sizes, sizeof(int) * D.C);
        bulk_prefetch_l2(D.starts, sizeof(int) * D.C);
        bulk_prefetch_l2(D.wrow0, sizeof(int) * D.C);
    }
    if (lead) DBG_TS(D, 25);
    const double qn = head_bounds<Q>(D, hs);
    if (lead) {
        D.res->query_norm = qn;
        DBG_TS(D, 26);
    }
    {
        const unsigned long long e = grid_sync_mono(D, D.bar64);
        if (tid == 0) s_epoch = e;
    }
    if (lead) DBG_TS(D, 27);
    // ---- the head of the opening order (every CTA, identically)
    Ord o;
    ord_bind(D, ws, o);
    __shared__ double s_slack, s_est;
    const bool ok = stage_bounds(D, o, qn, &s_slack);
    const int hn = ok ? order_head(D, o, s_est) : 0;
    if (hn == 0 || G < 2) {  // every CTA sees the same: the general step decides
        __syncthreads();
        step_body<ET, 8, Q, 8, Q>(D);
        return;
    }
    if (tid == 0) init_state(D, o, ss, hn, s_est);
    if (lead) DBG_TS(D, 28);
    const unsigned long long epoch = s_epoch;
    unsigned long long *decision = D.bar64 + 1;  // epoch * 2 + decided
    const int R = o.cum[hn];
    if (b > 0) {
        // ---- row CTA: rows of the head, contiguous per CTA
        const int rb = b - 1, Gr = G - 1;
        const int r_lo = (int)((long long)R * rb / Gr), r_hi = (int)((long long)R * (rb + 1) / Gr);
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
        // this CTA's share of every cluster it touches (release: the rows above are visible first)
        if (tid < hn) {
            const int a = max(o.cum[tid], r_lo), e = min(o.cum[tid + 1], r_hi);
            if (e > a) {
                __threadfence();
                atomicAdd(D.hcnt + tid, e - a);
            }
        }
        if (D.res_host) {  // host-API step: this CTA's rows into the mapped buffers (speculative:
                           // the host reads only the first |S| entries)
            for (int r = r_lo + tid; r < r_hi; r += THREADS) {
                D.logits_host[r] = __ldcg(D.S_logits + r);
                D.ids_host[r] = __ldcg(D.S_ids + r);
            }
        }
        // ---- wait for CTA 0's decision
        __shared__ int s_dec;
        if (tid == 0) {
            unsigned long long v, spins = 0;
            do {
                asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(decision) : "memory");
                if (++spins > (1ull << 26)) {
                    D.res->error = CSVD_ESTATE;
                    v = epoch * 2 + 1;
                }
            } while ((v >> 1) < epoch);
            s_dec = (int)(v & 1);
            if (D.dbg && b < 256) D.dbg[128 + b] = gtimer();
        }
        __syncthreads();
        if (s_dec) return;
        step_body<ET, 8, Q, 8, Q>(D);  // undecided: the general step, from scratch
        return;
    }
    // ---- CTA 0: wait for every head cluster's rows, then certify
    for (int q = tid; q < hn; q += THREADS) {
        const int n = o.cum[q + 1] - o.cum[q];
        unsigned long long spins = 0;
        int v;
        do {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(D.hcnt + q) : "memory");
            if (++spins > (1ull << 26)) {
                D.res->error = CSVD_ESTATE;
                break;
            }
        } while (v < n);
    }
    __syncthreads();
    __threadfence();
    if (lead) DBG_TS(D, 29);
    __shared__ csvd_result s_res;
    bool decided;
    if (head_fits(o, hn)) {
        decided = head_certify(D, o, hn, s_res) != 0;
    } else {  // more than THREADS * HJ head tokens: per-cluster summaries + the sequential scan
        const int k = D.cfg->k;
        double *c_vals = sws, *c_lse = sws + 6 * CHUNK, *c_min = c_lse + CHUNK, *c_max = c_min + CHUNK;
        double *la = c_max + CHUNK, *lb = la + D.K, *c_topk = lb + D.K;
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
        if (tid == 0) s_res = ss.res;
        __syncthreads();
    }
    if (lead) DBG_TS(D, 31);
    // every row CTA has added its counts (all head clusters completed): reset
    for (int q = tid; q < hn; q += THREADS) D.hcnt[q] = 0;
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
        __threadfence();
        const unsigned long long w = epoch * 2 + (decided ? 1 : 0);
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(decision), "l"(w) : "memory");
        DBG_TS(D, 30);
    }
    __syncthreads();
    if (!decided) step_body<ET, 8, Q, 8, Q>(D);
}
