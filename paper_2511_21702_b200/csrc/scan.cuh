// Sequential certification scan over per-cluster summaries (host + device).
//
// Restates the reference step driver exactly:
//   decode_step loop                 decode.py:312-343
//   decode_step_batchselect          decode.py:362-382 (+ _select_by_bound :346-359)
//   check_targets                    decode.py:192-210
//   fallback chain / apply_fallback  decode.py:268-309
//   CertState.merge_cluster (log_z, 64-merge recompute)  certify.py:73-83
//   rho / delta / topk_certified / softmax / topp        certify.py:93-164
//   outcome + tightness              decode.py:212-237, certify.py:172-184
//
// Invariant used (verified by tests): the opened set is always a
// prefix of the bound order, so "u_max over unopened" = U[order[p]] and the
// residual log R-hat after p opens is the suffix log-sum-exp lrh[p] computed
// once per step.  The scan consumes per-cluster summaries (top-k values, LSE,
// min, max) produced by the GEMV epilogue, in opening order, wave by wave;
// it is run identically by all 32 lanes of one warp on the device (scalar
// state replicated, collective primitives warp-parallel) and by one thread on
// the host (unit tests).
#pragma once
#include <cmath>
#include <cstdint>

#include "../../include/csvd_b200.h"

#ifdef __CUDACC__
#define CSVD_HD __host__ __device__
#else
#define CSVD_HD
#endif

enum { PH_MAIN = 0, PH_PE = 1, PH_DONE = 2, PH_DENSE = 3, PH_ERROR = 4 };
enum { MODE_SPARSE = 0, MODE_DENSE = 1, MODE_IDLE = 2 };

struct ScanState {
    int p;          // clusters merged (opened) so far
    int merges;
    int kcount;     // entries in the running top-k list
    int phase;
    int level;      // next fallback level index
    int pe_target;
    int heap_pops;
    int p_lo, p_hi; // current wave, in opening-order prefixes
    int row_lo, row_hi;
    int p_cap;      // never plan beyond this prefix
    int p_sel;      // batchselect selection size
    int iter;       // wave kernel iterations (guard)
    int mode;       // MODE_*
    int wave_tokens;
    int pad0;
    double log_z, smin, smax;
    double est;     // wave heuristic: lower estimate of the best logit
};

// Exact helpers with host fallbacks (the host path only runs in unit tests).
#ifdef __CUDA_ARCH__
#define CSVD_ADD(a, b) __dadd_rn((a), (b))
#define CSVD_SUB(a, b) __dsub_rn((a), (b))
#define CSVD_MUL(a, b) __dmul_rn((a), (b))
#define CSVD_DIV(a, b) __ddiv_rn((a), (b))
#else
#define CSVD_ADD(a, b) ((a) + (b))
#define CSVD_SUB(a, b) ((a) - (b))
#define CSVD_MUL(a, b) ((a) * (b))
#define CSVD_DIV(a, b) ((a) / (b))
#endif

CSVD_HD inline double csvd_neg_inf() { return -INFINITY; }

// the scan reads its inputs from arrays the executor staged (shared memory
// on the device, plain arrays on the host)
#define CSVD_LD(p) (*(p))

// np.logaddexp (numpy npy_logaddexp): x==y -> x + log(2); else max + log1p(exp(-|x-y|))
CSVD_HD inline double csvd_logaddexp(double x, double y) {
    if (x == y) return CSVD_ADD(x, 0.69314718055994530942);
    double t = CSVD_SUB(x, y);
    if (t > 0) return CSVD_ADD(x, log1p(exp(-t)));
    if (t <= 0) return CSVD_ADD(y, log1p(exp(t)));
    return t;  // nan
}

// Read-only step inputs for the scan.
struct ScanIn {
    const csvd_config *cfg;
    int C;
    long long V;
    int d;           // hidden dim (flops)
    const int *cum;      // [C+1] prefix token counts in opening order
    const double *Uo;    // [C] bounds in opening order (Uo[p] = U[order[p]])
    const double *lrh;   // [C+1] log R-hat after p opens
    const double *sum_lse, *sum_min, *sum_max;  // [C] by opening position
    const double *sum_topk;                      // [C * K] by opening position
    int K;                                       // top-k row stride
    const double *S_logits;                      // logits in opening order
};

// Primitives supplied by the executor (warp on device, thread on host):
//   merge_topk(run, kr, add, ka, k, out) -> new count (top-k of the union, desc)
//   lse_all(vals, n, vmax) -> logsumexp over vals[0..n)
//   writer() -> true for the lane allowed to write memory
template <class P>
struct Scan {
    const ScanIn &in;
    ScanState &st;
    double *&lst;     // running top-k list (double buffered)
    double *&lst_alt;
    P &prims;
    csvd_result &res;

    CSVD_HD double u_at(int p) const { return p >= in.C ? csvd_neg_inf() : in.Uo[p]; }
    CSVD_HD long long n_s() const { return in.cum[st.p]; }
    CSVD_HD double kth() const {  // the k-th largest computed logit (certify.py:85-88)
        int k = in.cfg->k;
        return st.kcount >= k && n_s() >= k ? lst[k - 1] : csvd_neg_inf();
    }
    CSVD_HD double rho() const {
        double lr = in.lrh[st.p];
        if (lr == csvd_neg_inf()) return 0.0;
        if (st.log_z == csvd_neg_inf()) return 1.0;
        return CSVD_DIV(1.0, CSVD_ADD(1.0, exp(CSVD_SUB(st.log_z, lr))));
    }
    CSVD_HD double delta() const {
        double lr = in.lrh[st.p];
        if (lr == csvd_neg_inf()) return 0.0;
        if (st.log_z == csvd_neg_inf()) return INFINITY;
        return exp(CSVD_SUB(lr, st.log_z));
    }

    // CertState.merge_cluster for the cluster at opening position q (== st.p)
    CSVD_HD void merge(int q) {
        const int k = in.cfg->k;
        const int size = in.cum[q + 1] - in.cum[q];
        const int ka = size < k ? size : k;
        st.kcount = prims.merge_topk(lst, st.kcount, in.sum_topk + (size_t)q * in.K, ka, k, lst_alt);
        double *t = lst;
        lst = lst_alt;
        lst_alt = t;
        const double mn = CSVD_LD(in.sum_min + q), mx = CSVD_LD(in.sum_max + q);
        if (st.p == 0) {
            st.smin = mn;
            st.smax = mx;
        } else {
            st.smin = mn < st.smin ? mn : st.smin;
            st.smax = mx > st.smax ? mx : st.smax;
        }
        st.p = q + 1;
        st.merges += 1;
        if (st.merges % 64 == 0)
            st.log_z = prims.lse_all(in.S_logits, in.cum[st.p], st.smax);
        else
            st.log_z = csvd_logaddexp(st.log_z, CSVD_LD(in.sum_lse + q));
    }

    // check_targets (decode.py:192-210); returns true and fills res when certified
    CSVD_HD bool check(double eps, int fb) {
        const csvd_config &cfg = *in.cfg;
        const long long n = n_s();
        for (int ti = 0; ti < cfg.n_targets; ++ti) {
            int t = cfg.targets[ti];
            if (t == CSVD_TARGET_TOPK) {
                if (n < cfg.k) continue;
                double kth_v = kth();
                if (st.p >= in.C) return finish(CSVD_KIND_TOPK_EXACT, 0.0, csvd_neg_inf(), kth_v, fb);
                double u = u_at(st.p);
                if (u < kth_v) return finish(CSVD_KIND_TOPK_EXACT, 0.0, u, kth_v, fb);
            } else if (t == CSVD_TARGET_SOFTMAX) {
                if (n == 0) continue;
                double r = rho();
                if (r <= eps) return finish(CSVD_KIND_SOFTMAX_EPS, r, u_at(st.p), kth(), fb);
            } else if (t == CSVD_TARGET_TOPP) {
                if (n == 0) continue;
                double dl = delta();
                double mass = isfinite(dl) ? CSVD_DIV(dl, CSVD_ADD(1.0, dl)) : 1.0;
                if (dl <= CSVD_DIV(eps, CSVD_SUB(1.0, eps))) return finish(CSVD_KIND_TOPP_MASS, mass, u_at(st.p), kth(), fb);
            }
        }
        return false;
    }

    // decode._StepContext.outcome (decode.py:212-237) scalars
    CSVD_HD bool finish(int kind, double eps_ach, double u, double kth_v, int fb) {
        const long long n = n_s();
        double xi;
        if (n < 2 || st.p >= in.C) {
            xi = NAN;
        } else {
            double lo = st.smin, hi = st.smax, um = u_at(st.p);
            xi = (um <= lo) ? 1.0 : CSVD_DIV(CSVD_SUB(hi, lo), CSVD_SUB(um, lo));
        }
        res.kind = kind;
        res.fallback = fb;
        res.sub_size = n;
        res.clusters_opened = st.p;
        res.heap_pops = st.heap_pops;
        res.epsilon_achieved = eps_ach;
        res.u_max = u;
        res.topk_min = kth_v;
        res.rho = rho();
        res.xi = xi;
        st.phase = PH_DONE;
        return true;
    }

    // _run_fallback_chain from st.level at prefix st.p (decode.py:268-309).
    CSVD_HD void run_levels() {
        const csvd_config &cfg = *in.cfg;
        while (st.level < cfg.n_levels) {
            const int kind = cfg.level_kind[st.level];
            if (kind == CSVD_FB_PARTIAL_EXPAND) {
                long long dc = (long long)cfg.level_param[st.level];
                long long tgt = st.p + (dc > 0 ? dc : 0);
                if (tgt > in.C) tgt = in.C;
                if (tgt == st.p) {  // nothing left to open: check immediately
                    if (check(cfg.epsilon, CSVD_FB_PARTIAL_EXPAND)) return;
                    st.level++;
                    continue;
                }
                st.phase = PH_PE;
                st.pe_target = (int)tgt;
                return;
            } else if (kind == CSVD_FB_RELAX_EPS) {
                double relaxed = CSVD_MUL(cfg.epsilon, cfg.level_param[st.level]);
                const double cap = 1.0 - 1e-12;
                if (relaxed > cap) relaxed = cap;
                for (int ti = 0; ti < cfg.n_targets; ++ti) {
                    int t = cfg.targets[ti];
                    if (t == CSVD_TARGET_SOFTMAX) {
                        double r = rho();
                        if (r <= relaxed) {
                            finish(CSVD_KIND_SOFTMAX_EPS, r, u_at(st.p), kth(), CSVD_FB_RELAX_EPS);
                            return;
                        }
                    } else if (t == CSVD_TARGET_TOPP) {
                        double dl = delta();
                        double mass = isfinite(dl) ? CSVD_DIV(dl, CSVD_ADD(1.0, dl)) : 1.0;
                        if (dl <= CSVD_DIV(relaxed, CSVD_SUB(1.0, relaxed))) {
                            finish(CSVD_KIND_TOPP_MASS, mass, u_at(st.p), kth(), CSVD_FB_RELAX_EPS);
                            return;
                        }
                    }
                }
                st.level++;
            } else {  // FullVocab
                st.phase = PH_DENSE;
                return;
            }
        }
        st.phase = PH_DENSE;  // FullVocab is always the implicit last level
    }

    // Consume clusters [st.p, avail) in opening order.
    CSVD_HD void run(int avail) {
        const csvd_config &cfg = *in.cfg;
        while (st.p < avail && (st.phase == PH_MAIN || st.phase == PH_PE)) {
            merge(st.p);
            if (st.phase == PH_MAIN) {
                if (cfg.variant == CSVD_VARIANT_INCREMENTAL) {
                    st.heap_pops = st.p;
                    if ((long long)in.cum[st.p] > cfg.k_max) {
                        st.level = 0;
                        run_levels();
                    } else {
                        check(cfg.epsilon, CSVD_FB_NONE);
                    }
                } else if (st.p == st.p_sel) {
                    if (!check(cfg.epsilon, CSVD_FB_NONE)) {
                        st.level = 0;
                        run_levels();
                    }
                }
            } else if (st.p == st.pe_target) {  // PH_PE
                if (!check(cfg.epsilon, CSVD_FB_PARTIAL_EXPAND)) {
                    st.level++;
                    run_levels();
                }
            }
        }
    }

    // full-vocabulary outcome scalars (decode.py:239-262)
    CSVD_HD void finish_dense(double kth_v) {
        res.kind = CSVD_KIND_TOPK_EXACT;
        res.fallback = CSVD_FB_FULL_VOCAB;
        res.sub_size = in.V;
        res.clusters_opened = in.C;
        res.heap_pops = st.heap_pops;
        res.epsilon_achieved = 0.0;
        res.u_max = csvd_neg_inf();
        res.topk_min = kth_v;
        res.rho = 0.0;
        res.xi = NAN;
        st.phase = PH_DONE;
    }
};

// ---------------------------------------------------------------------------
// wave planning (speculative opening; never changes results, only how many
// clusters' logits are computed per device iteration).  All searches are over
// monotone predicates, so a scalar binary search (host, single thread) and a
// warp-parallel 32-ary search (device) return the same index.
// ---------------------------------------------------------------------------
struct ScalarSearch {
    // first i in [lo, hi) with pred(i) true, or hi
    template <class F>
    CSVD_HD int operator()(int lo, int hi, const F &pred) const {
        while (lo < hi) {
            int mid = lo + (hi - lo) / 2;
            if (pred(mid)) hi = mid; else lo = mid + 1;
        }
        return lo;
    }
};

// batch-select budget prefix (_select_by_bound, decode.py:346-359):
// the largest p with cum[p] <= k_max, at least 1
template <class S>
CSVD_HD inline int csvd_select_prefix(const ScanIn &in, long long k_max, const S &search) {
    int p = search(1, in.C + 1, [&](int q) { return (long long)in.cum[q] > k_max; }) - 1;
    return p < 1 ? 1 : p;
}

// prefixes never needed: past the budget trigger plus every partial expansion
template <class S>
CSVD_HD inline int csvd_cap_prefix(const ScanIn &in, int p_sel, const S &search) {
    const csvd_config &cfg = *in.cfg;
    int sum_dc = 0;
    for (int l = 0; l < cfg.n_levels; ++l)
        if (cfg.level_kind[l] == CSVD_FB_PARTIAL_EXPAND) sum_dc += (int)cfg.level_param[l];
    int base;
    if (cfg.variant == CSVD_VARIANT_BATCHSELECT) {
        base = p_sel;
    } else {  // first prefix whose token count exceeds k_max
        base = search(1, in.C + 1, [&](int q) { return (long long)in.cum[q] > cfg.k_max; });
        if (base > in.C) base = in.C;
    }
    long long cap = (long long)base + sum_dc;
    return cap > in.C ? in.C : (int)cap;
}

// Next wave end for phase MAIN / PE.  Returns p_hi > st.p.
template <class S>
CSVD_HD inline int csvd_plan_wave(const ScanState &st, const ScanIn &in, const S &search) {
    if (st.phase == PH_PE) return st.pe_target;
    if (in.cfg->variant == CSVD_VARIANT_BATCHSELECT && st.p < st.p_sel) return st.p_sel;
    const long long want = (long long)in.cum[st.p] + st.wave_tokens;
    int hi = search(st.p + 1, in.C + 1, [&](int q) { return (long long)in.cum[q] >= want; });
    if (hi > in.C) hi = in.C;
    bool has_topk = false;
    for (int t = 0; t < in.cfg->n_targets; ++t) has_topk = has_topk || in.cfg->targets[t] == CSVD_TARGET_TOPK;
    if (has_topk) {
        // clusters whose bound still beats the estimate of the best logit cannot
        // be excluded by a top-k certificate (Uo is non-increasing)
        int lim = st.p + 64 < in.C ? st.p + 64 : in.C;
        if (hi < lim) hi = search(hi, lim, [&](int q) { return in.Uo[q] < st.est; });
    } else {
        // rho(p) >= Rhat(p)/Rhat(0): prefixes with Rhat(p)/Rhat(0) > eps cannot certify
        const double le = log(in.cfg->epsilon);
        if (hi < in.C) hi = search(hi, in.C, [&](int q) { return !(CSVD_SUB(in.lrh[q], in.lrh[0]) > le); });
    }
    if (hi > st.p_cap) hi = st.p_cap;
    if (hi <= st.p) hi = st.p + 1;
    if (hi > in.C) hi = in.C;
    return hi;
}
