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
// prefix of the bound order, so "u_max over unopened" = Uo[p] and the residual
// log R-hat after p opens is the suffix log-sum-exp lrh[p] computed once per
// step.  Because merges happen in opening order, every per-prefix quantity is a
// pure function of p: log Z_S(p) (streaming logaddexp, full recompute when
// p % 64 == 0), the k-th largest logit kth(p), min/max of S, rho(p), delta(p).
// An executor-supplied precompute fills them for a chunk of prefixes (the host
// does it sequentially with the reference's exact arithmetic; the device
// warp-parallel, ulp-close for the transcendental ones and exact for kth /
// min / max), and the state machine below only compares.
#pragma once
#include <cmath>
#include <cstdint>

#include "../../include/csvd_b200.h"

#ifdef __CUDACC__
#define CSVD_HD __host__ __device__
// out of line on the device: this code runs once per step with a cold
// instruction cache, so one shared copy beats many inlined ones
#define CSVD_HD_NOINL __host__ __device__ __noinline__
#else
#define CSVD_HD
#define CSVD_HD_NOINL
#endif

enum { PH_MAIN = 0, PH_PE = 1, PH_DONE = 2, PH_DENSE = 3, PH_ERROR = 4 };
enum { MODE_SPARSE = 0, MODE_DENSE = 1, MODE_IDLE = 2 };

struct ScanState {
    int p;          // clusters merged (opened) so far
    int kcount;     // entries in the running top-k list
    int phase;
    int level;      // next fallback level index
    int pe_target;
    int heap_pops;
    int p_lo, p_hi; // current wave, in opening-order prefixes
    int row_lo, row_hi;
    int p_cap;      // never plan beyond this prefix
    int p_sel;      // batchselect selection size
    int iter;       // wave iterations (guard)
    int mode;       // MODE_*
    int wave_tokens;
    int pad0;
    // values at the current prefix p
    double log_z, smin, smax, kth, rho, delta;
    double est;     // wave heuristic: lower estimate of the best logit
};

#ifdef __CUDACC__
static __device__ __noinline__ double csvd_ddiv(double a, double b) { return __ddiv_rn(a, b); }
static __device__ __noinline__ double csvd_exp(double x) { return exp(x); }
static __device__ __noinline__ double csvd_log(double x) { return log(x); }
static __device__ __noinline__ double csvd_log1p(double x) { return log1p(x); }
#endif
#ifdef __CUDA_ARCH__
#define CSVD_ADD(a, b) __dadd_rn((a), (b))
#define CSVD_SUB(a, b) __dsub_rn((a), (b))
#define CSVD_MUL(a, b) __dmul_rn((a), (b))
#define CSVD_DIV(a, b) csvd_ddiv((a), (b))
#define CSVD_EXP(x) csvd_exp(x)
#define CSVD_LOG(x) csvd_log(x)
#define CSVD_LOG1P(x) csvd_log1p(x)
#else
#define CSVD_EXP(x) exp(x)
#define CSVD_LOG(x) log(x)
#define CSVD_LOG1P(x) log1p(x)
#define CSVD_ADD(a, b) ((a) + (b))
#define CSVD_SUB(a, b) ((a) - (b))
#define CSVD_MUL(a, b) ((a) * (b))
#define CSVD_DIV(a, b) ((a) / (b))
#endif

CSVD_HD inline double csvd_neg_inf() { return -INFINITY; }

// np.logaddexp (numpy npy_logaddexp): x==y -> x + log(2); else max + log1p(exp(-|x-y|))
CSVD_HD inline double csvd_logaddexp(double x, double y) {
    if (x == y) return CSVD_ADD(x, 0.69314718055994530942);
    double t = CSVD_SUB(x, y);
    if (t > 0) return CSVD_ADD(x, CSVD_LOG1P(CSVD_EXP(-t)));
    if (t <= 0) return CSVD_ADD(y, CSVD_LOG1P(CSVD_EXP(t)));
    return t;  // nan
}

// certify.CertState.rho / delta (certify.py:93-107) from log Z_S and log R-hat
CSVD_HD inline double csvd_rho(double log_z, double lr) {
    if (lr == csvd_neg_inf()) return 0.0;
    if (log_z == csvd_neg_inf()) return 1.0;
    return CSVD_DIV(1.0, CSVD_ADD(1.0, CSVD_EXP(CSVD_SUB(log_z, lr))));
}
CSVD_HD inline double csvd_delta(double log_z, double lr) {
    if (lr == csvd_neg_inf()) return 0.0;
    if (log_z == csvd_neg_inf()) return INFINITY;
    return CSVD_EXP(CSVD_SUB(lr, log_z));
}

// Read-only step inputs for the scan.
struct ScanIn {
    const csvd_config *cfg;
    int C;
    long long V;
    int d;               // hidden dim (flops)
    const int *cum;      // [C+1] prefix token counts in opening order
    const double *Uo;    // [C] bounds in opening order (Uo[p] = U[order[p]])
    const double *lrh;   // [C+1] log R-hat after p opens
};

// Per-prefix values for clusters q in [q0, q1): index i = q - q0 describes
// prefix p = q + 1.
struct Chunk {
    int q0, q1;
    const double *log_z, *kth, *smin, *smax, *rho, *delta;
};

struct Scan {
    const ScanIn &in;
    ScanState &st;
    csvd_result &res;

    CSVD_HD double u_at(int p) const { return p >= in.C ? csvd_neg_inf() : in.Uo[p]; }
    CSVD_HD long long n_s() const { return in.cum[st.p]; }

    // CertState.merge_cluster of the cluster at opening position q == st.p
    CSVD_HD void merge(const Chunk &ch, int q) {
        const int i = q - ch.q0;
        st.p = q + 1;
        st.log_z = ch.log_z[i];
        st.kth = ch.kth[i];
        st.smin = ch.smin[i];
        st.smax = ch.smax[i];
        st.rho = ch.rho[i];
        st.delta = ch.delta[i];
    }

    // check_targets (decode.py:192-210); returns true and fills res when certified
    CSVD_HD_NOINL bool check(double eps, int fb) {
        const csvd_config &cfg = *in.cfg;
        const long long n = n_s();
        for (int ti = 0; ti < cfg.n_targets; ++ti) {
            int t = cfg.targets[ti];
            if (t == CSVD_TARGET_TOPK) {
                if (n < cfg.k) continue;
                if (st.p >= in.C) return finish(CSVD_KIND_TOPK_EXACT, 0.0, csvd_neg_inf(), st.kth, fb);
                double u = u_at(st.p);
                if (u < st.kth) return finish(CSVD_KIND_TOPK_EXACT, 0.0, u, st.kth, fb);
            } else if (t == CSVD_TARGET_SOFTMAX) {
                if (n == 0) continue;
                if (st.rho <= eps) return finish(CSVD_KIND_SOFTMAX_EPS, st.rho, u_at(st.p), st.kth, fb);
            } else if (t == CSVD_TARGET_TOPP) {
                if (n == 0) continue;
                double dl = st.delta;
                double mass = isfinite(dl) ? CSVD_DIV(dl, CSVD_ADD(1.0, dl)) : 1.0;
                if (dl <= CSVD_DIV(eps, CSVD_SUB(1.0, eps)))
                    return finish(CSVD_KIND_TOPP_MASS, mass, u_at(st.p), st.kth, fb);
            }
        }
        return false;
    }

    // decode._StepContext.outcome (decode.py:212-237) scalars
    CSVD_HD_NOINL bool finish(int kind, double eps_ach, double u, double kth_v, int fb) {
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
        res.rho = st.rho;
        res.xi = xi;
        st.phase = PH_DONE;
        return true;
    }

    // _run_fallback_chain from st.level at prefix st.p (decode.py:268-309).
    CSVD_HD_NOINL void run_levels() {
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
                        if (st.rho <= relaxed) {
                            finish(CSVD_KIND_SOFTMAX_EPS, st.rho, u_at(st.p), st.kth, CSVD_FB_RELAX_EPS);
                            return;
                        }
                    } else if (t == CSVD_TARGET_TOPP) {
                        double dl = st.delta;
                        double mass = isfinite(dl) ? CSVD_DIV(dl, CSVD_ADD(1.0, dl)) : 1.0;
                        if (dl <= CSVD_DIV(relaxed, CSVD_SUB(1.0, relaxed))) {
                            finish(CSVD_KIND_TOPP_MASS, mass, u_at(st.p), st.kth, CSVD_FB_RELAX_EPS);
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

    // Consume the chunk's clusters in opening order.
    CSVD_HD void run(const Chunk &ch) {
        const csvd_config &cfg = *in.cfg;
        while (st.p < ch.q1 && (st.phase == PH_MAIN || st.phase == PH_PE)) {
            merge(ch, st.p);
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
// monotone predicates, so a scalar binary search (host / one thread) and a
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
        const double le = CSVD_LOG(in.cfg->epsilon);
        if (hi < in.C) hi = search(hi, in.C, [&](int q) { return !(CSVD_SUB(in.lrh[q], in.lrh[0]) > le); });
    }
    if (hi > st.p_cap) hi = st.p_cap;
    if (hi <= st.p) hi = st.p + 1;
    if (hi > in.C) hi = in.C;
    return hi;
}
