"""Test infrastructure: an oracle-backed stand-in for distributed.DeviceShard.

It computes, with the oracle's restated reference arithmetic (oracle/), exactly
what `csvd_shard_open` / `csvd_shard_dense` return for one rank, so the
distributed merge / certification / fallback logic of
`paper_2511_21702_b200.distributed` can run across real gloo ranks on CPU.
Only tests import this module."""

from __future__ import annotations

import numpy as np

import csvd_oracle as O
from paper_2511_21702_b200 import distributed as Dm

NEG_INF = float("-inf")


class OracleShard:
    def __init__(self, table, index, owned):
        self.T, self.ix = table, index
        self.owned = np.asarray(owned, dtype=bool)
        self.V, self.C = int(index.vocab_size), int(index.n_clusters)

    def _logits(self, c, h):
        s, e = int(self.ix.starts[c]), int(self.ix.ends[c])
        members = self.ix.perm[s:e]
        return members, O.gemv_rows(self.T.weights, h, sel=members, bias=self.T.bias)

    def open(self, h, cs, lo, hi):
        h = np.ascontiguousarray(h, dtype=np.float64)
        slack_mode = "f32" if cs.slack_f32 else "none"
        b = O.cluster_bounds(self.ix, h, slack_mode=slack_mode)
        U = b.values
        sizes = np.asarray(self.ix.sizes)
        order = np.lexsort((np.arange(self.C), -U))
        p_sel = len(O.select_by_bound(order, sizes, int(cs.k_max)))
        hi = hi if hi > 0 else p_sel
        lo = min(max(lo, 0), self.C)
        hi = min(max(hi, lo), self.C)
        cum = np.concatenate([[0], np.cumsum(sizes[order])])
        pos, ids, lg = [], [], []
        for q in range(lo, hi):
            c = int(order[q])
            if not self.owned[c]:
                continue
            members, logits = self._logits(c, h)
            pos.append(np.arange(cum[q], cum[q + 1]))
            ids.append(members)
            lg.append(logits)
        pos = np.concatenate(pos) if pos else np.empty(0, np.int64)
        ids = np.concatenate(ids) if ids else np.empty(0, np.int64)
        lg = np.concatenate(lg) if lg else np.empty(0)
        k = int(cs.k)
        summ = np.zeros(Dm.SH_TOPK + k)
        n = lg.size
        summ[Dm.SH_LSE] = O.logsumexp(lg) if n else NEG_INF
        summ[Dm.SH_MIN] = lg.min() if n else np.inf
        summ[Dm.SH_MAX] = lg.max() if n else NEG_INF
        summ[Dm.SH_NTOK] = n
        nl = min(k, n)
        summ[Dm.SH_NLIST] = nl
        summ[Dm.SH_TOPK:Dm.SH_TOPK + nl] = -np.sort(-lg)[:nl]
        summ[Dm.SH_P_LO], summ[Dm.SH_P_HI], summ[Dm.SH_P_SEL] = lo, hi, p_sel
        summ[Dm.SH_CUM_LO], summ[Dm.SH_CUM_HI] = cum[lo], cum[hi]
        summ[Dm.SH_U_NEXT] = U[order[hi]] if hi < self.C else NEG_INF
        un = np.ones(self.C, dtype=bool)
        un[order[:hi]] = False
        summ[Dm.SH_LRH_NEXT] = O.logsumexp(np.log(sizes[un]) + U[un]) if un.any() else NEG_INF
        summ[Dm.SH_QNORM], summ[Dm.SH_SLACK] = b.query_norm, b.slack
        return summ, pos.astype(np.int64), ids.astype(np.int64), lg

    def dense(self, h, k):
        h = np.ascontiguousarray(h, dtype=np.float64)
        toks = np.sort(np.concatenate([self.ix.perm[int(self.ix.starts[c]):int(self.ix.ends[c])]
                                       for c in range(self.C) if self.owned[c]] or [np.empty(0, np.int64)]))
        lg = O.gemv_rows(self.T.weights, h, sel=toks, bias=self.T.bias) if toks.size else np.empty(0)
        summ = np.zeros(Dm.SH_TOPK + k)
        nl = min(k, toks.size)
        summ[Dm.SH_NTOK] = toks.size
        summ[Dm.SH_NLIST] = nl
        summ[Dm.SH_TOPK:Dm.SH_TOPK + nl] = -np.sort(-lg)[:nl]
        return summ, toks.astype(np.int64), lg
