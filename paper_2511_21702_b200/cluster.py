"""GPU offline clustering: the B200 counterpart of `csvd.build_index`
(/root/reference/pkg/src/csvd/cluster_index.py:282-341).

The reference runs k-means++ seeding and Lloyd iterations in numpy f64
(`_kmeanspp_seed` / `_lloyd`, cluster_index.py:167-251), which takes ~23 min at
c1 and is out of reach at c2-c5.  Here the same algorithm runs on the GPU:

  * the distance GEMMs (rows x centroids, the only O(V C d) work) go to the
    tensor cores through cuBLAS (TF32, fp32 accumulate);
  * seeding, the arg-min assignment, centroid means and empty-cluster repair
    are batched torch reductions on the device.

The partition is not the reference's bit for bit (its own distance GEMM is a
BLAS call with an unspecified summation order, so no implementation could
promise that), but the index is: every statistic the decode step relies on
is recomputed from the final partition with the reference's own arithmetic
(`workload.index_from_assignment`, the `_cluster_stats` restatement,
cluster_index.py:254-279), in the reference's cluster order (size-descending,
ties by smallest member id, cluster_index.py:305-316).  Any partition gives
sound bounds, so decoding with this index is exact (tests/test_gpu_cluster.py).
"""

from __future__ import annotations

import numpy as np

from .types import ClusterIndex
from .workload import bf16_bits_to_f32, index_from_assignment

MODES = ("euclidean", "spherical", "bias_augmented")


def _device_rows(table, mode, torch, dev):
    w = table.weights
    if w.dtype == np.uint16:
        w = bf16_bits_to_f32(w)
    X = torch.from_numpy(np.ascontiguousarray(w, dtype=np.float32)).to(dev)
    if mode == "bias_augmented":  # _geometry_rows (cluster_index.py:151-154)
        b = torch.from_numpy(np.asarray(table.bias, dtype=np.float32)).to(dev)
        X = torch.cat([X, b[:, None]], dim=1)
    if mode == "spherical":  # _assignment_rows (cluster_index.py:157-164)
        n = X.norm(dim=1, keepdim=True)
        X = torch.where(n > 0, X / n.clamp_min(1e-30), torch.zeros_like(X))
    return X


def _assign(X, Cm, spherical, torch, chunk=1 << 15):
    """arg-min squared distance (arg-max cosine for spherical) per row, and its value"""
    cn = (Cm * Cm).sum(dim=1)
    lab = torch.empty(X.shape[0], dtype=torch.int64, device=X.device)
    best = torch.empty(X.shape[0], dtype=torch.float32, device=X.device)
    for s in range(0, X.shape[0], chunk):
        x = X[s:s + chunk]
        g = x @ Cm.T  # tensor cores (TF32)
        if spherical:
            v, i = (g / cn.clamp_min(1e-30).sqrt()).max(dim=1)
            best[s:s + chunk] = -v
        else:
            v, i = (cn[None, :] - 2.0 * g).min(dim=1)
            best[s:s + chunk] = v + (x * x).sum(dim=1)
        lab[s:s + chunk] = i
    return lab, best


def build_index_gpu(table, n_clusters: int, mode: str = "euclidean", iters: int = 32, m: int = 3,
                    seed: int = 0, device: int = 0) -> ClusterIndex:
    """`csvd.build_index` semantics and errors (cluster_index.py:282-300) on the GPU."""
    import torch
    V = table.vocab_size
    C = int(n_clusters)
    if not 1 <= C <= V:
        raise ValueError(f"need 1 <= C <= V, got C={C}, V={V}")
    if iters < 1:
        raise ValueError("iters must be >= 1")
    if m < 1:
        raise ValueError("bias-table depth m must be >= 1")
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}, expected one of {MODES}")
    if not torch.cuda.is_available():
        raise RuntimeError("build_index_gpu needs a CUDA device")
    dev = torch.device("cuda", device)
    prev_tf32 = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = True
    try:
        X = _device_rows(table, mode, torch, dev)
        spherical = mode == "spherical"
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        # ---- k-means++ seeding (cluster_index.py:167-201): D^2 sampling
        xn = (X * X).sum(dim=1)
        first = int(torch.randint(V, (1,), generator=gen, device=dev))
        centers = [first]
        d2 = (xn - 2.0 * (X @ X[first]) + xn[first]).clamp_min(0)
        for _ in range(1, C):
            tot = float(d2.sum())
            if tot > 0:
                nxt = int(torch.multinomial(d2 / tot, 1, generator=gen))
            else:  # every row coincides with a center: any unused row
                nxt = int(torch.randint(V, (1,), generator=gen, device=dev))
            centers.append(nxt)
            d2 = torch.minimum(d2, (xn - 2.0 * (X @ X[nxt]) + xn[nxt]).clamp_min(0))
        Cm = X[torch.tensor(centers, device=dev)].clone()
        # ---- Lloyd iterations (cluster_index.py:232-251) with empty-cluster repair
        lab = None
        for _ in range(iters):
            new, dist = _assign(X, Cm, spherical, torch)
            counts = torch.bincount(new, minlength=C)
            empty = (counts == 0).nonzero().flatten()
            if empty.numel():  # _repair_empty: the farthest rows become the empty clusters' centers
                far = torch.topk(dist, int(empty.numel())).indices
                new[far] = empty
                counts = torch.bincount(new, minlength=C)
            sums = torch.zeros_like(Cm).index_add_(0, new, X)
            Cm = sums / counts.clamp_min(1)[:, None].to(X.dtype)
            if spherical:
                Cm = Cm / Cm.norm(dim=1, keepdim=True).clamp_min(1e-30)
            if lab is not None and torch.equal(lab, new):
                break
            lab = new
        labels = lab.cpu().numpy()
    finally:
        torch.backends.cuda.matmul.allow_tf32 = prev_tf32
    # ---- the index: exact statistics in the reference's arithmetic and order
    return index_from_assignment(table, labels, mode=mode, m=m)
