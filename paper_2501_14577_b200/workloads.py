"""Locality / recall workload on the same encode, sort and
top-k kernels -- no datasets, seeded synthetic points.

* ``locality_overlap`` -- Fig. 4: "the overlap between the
  top-64 nearest neighbors before and after projection, with sample sizes
  N in {512, 1024, 2048}".  Before projection: the exact Euclidean top-k of
  every point among the other points (onedf's own selection with the
  candidate window covering the whole run, W >= N, which is exact kNN).
  After projection: the k points nearest in Morton code (onedf_code_knn,
  S:432 "top-64 nearest-by-|code difference| after Morton encoding").  The
  metric is |both| / k per point (onedf_overlap), averaged.
* ``k_ablation`` -- P:1583-1587 ("values of k ranging from 16 to 48"):
  recall of the method's index set (windows W = 2k, chunk-causal) against the
  exact chunk-causal kNN (W >= M) for each k.

Every computation runs in libonedf.so; the functions here allocate, call and
average (the mean of per-point counts is the workload's reporting step).
"""
from __future__ import annotations

import torch

from . import api


def _points(trials: int, N: int, d: int, seed: int, device) -> torch.Tensor:
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.randn(trials, 1, N, d, generator=g).to(device)


def locality_overlap(X: torch.Tensor, k: int = 64) -> torch.Tensor:
    """X [T, 1, N, d] f32 (cuda): per-point overlap in [0, 1], shape [T, 1, N]."""
    T, _, N, d = X.shape
    X = X.contiguous()
    ws = api.Workspace(X.device)
    p = api.make_problem(T, 1, N, d, 4, k, window=max(N, 2 * k), chunk=1, causal=0, mean_slot=0)
    qc, kc, _ = api.encode(p, X, X, ws=ws)
    sc, pm = api.sort(p, kc, ws=ws)
    code = api.code_knn(p, qc, sc, pm, exclude_self=True)
    pe = api.make_problem(T, 1, N, d, 4, k + 1, window=max(N, k + 1), chunk=1, causal=0, mean_slot=0)
    V = torch.zeros(T, 1, N, 4, device=X.device)
    eps = torch.tensor(0.5, device=X.device)
    _, exact, _ = api.topk_attn_fwd(pe, X, X, V, eps, qc, sc, pm, ws=ws)     # includes the point itself
    return api.overlap(code, exact, self_period=N).float() / k


def locality_sweep(dims=(1, 2, 3, 4, 5, 6, 7, 8), Ns=(512, 1024, 2048), trials: int = 10, k: int = 64,
                   seed: int = 250114577, device="cuda"):
    """Rows (d_k, N, mean_overlap, per_trial_means) for Fig. 4's grid; standard-Gaussian points."""
    rows = []
    for d in dims:
        for N in Ns:
            X = _points(trials, N, d, seed + 1009 * d + N, device)
            ov = locality_overlap(X, k)
            per = ov.mean(dim=(1, 2)).tolist()
            rows.append(dict(d_k=d, N=N, mean_overlap=float(ov.mean()), per_trial=per))
    return rows


def k_ablation(N: int = 2048, d_k: int = 3, M: int = 256, ks=(16, 24, 32, 40, 48), trials: int = 4,
               seed: int = 250114577, device="cuda"):
    """Recall of the method's top-k (W = 2k) against exact chunk-causal kNN, per k."""
    X = _points(2 * trials, N, d_k, seed + 7, device)
    Q, K = X[:trials].contiguous(), X[trials:].contiguous()
    V = torch.zeros(trials, 1, N, 4, device=X.device)
    eps = torch.tensor(0.5, device=X.device)
    ws = api.Workspace(X.device)
    out = []
    for k in ks:
        p = api.make_problem(trials, 1, N, d_k, 4, k, window=2 * k, chunk=M, causal=1, mean_slot=0)
        qc, kc, _ = api.encode(p, Q, K, ws=ws)
        sc, pm = api.sort(p, kc, ws=ws)
        _, idx, _ = api.topk_attn_fwd(p, Q, K, V, eps, qc, sc, pm, ws=ws)
        pe = api.make_problem(trials, 1, N, d_k, 4, k, window=max(M, k), chunk=M, causal=1, mean_slot=0)
        _, exact, _ = api.topk_attn_fwd(pe, Q, K, V, eps, qc, sc, pm, ws=ws)
        hit = api.overlap(idx, exact).sum().item()
        total = (exact >= 0).sum().item()
        out.append(dict(k=k, recall=hit / total))
    return out
