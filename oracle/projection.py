"""CPU oracle of the NEXT-4 upstream step fused into the encoder: the query/key projections
f_q, f_k and the Cauchy scale gamma^2 = sigma(theta).

TEST INFRASTRUCTURE ONLY (same rules as ``oracle/__init__.py``: importable from ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s baseline legs only; shares no code with the CUDA
path).  Plain numpy in f64, one function per step, written from the paper:

* "trainable projection networks f_k and f_q" map the token features to the low
  d_K ("by setting d_K as low as 3, we reduce it from the typical head dimension");
  per head h:  q_{b,h,n} = W_q[h] x_{b,n} + b_q[h],  k_{b,h,n} = W_k[h] x_{b,n} + b_k[h]
  (one linear layer, reading D27; the paper's optional second layer is not specified further).
* "We define gamma^2 as the output of a sigmoid function applied to a trainable
  parameter":  eps = gamma^2 = sigma(theta) = 1 / (1 + exp(-theta)).
* their gradients (the chain rule of the two definitions above):
  dx_{b,n} = sum_h W_q[h]^T dq_{b,h,n} + W_k[h]^T dk_{b,h,n};  dW_q[h] = sum_{b,n} dq x^T;
  db_q[h] = sum_{b,n} dq;  dtheta = d_eps * sigma(theta) (1 - sigma(theta)).

Layouts (those of the C ABI ``onedf_project_encode``/``onedf_project_bwd``):
X [B, N, d_model]; W_q, W_k [H, d_k, d_model]; b_q, b_k [H, d_k]; Q, K [B, H, N, d_k].
"""
from __future__ import annotations

import numpy as np


def project(X, Wq, Wk, bq=None, bk=None):
    """q = W_q[h] x + b_q[h] and k likewise for every (b, h, n), in f64 (reading D27)."""
    X = np.asarray(X, dtype=np.float64)
    Wq = np.asarray(Wq, dtype=np.float64)
    Wk = np.asarray(Wk, dtype=np.float64)
    Q = np.einsum("bnm,hdm->bhnd", X, Wq)      # a library contraction as one step
    K = np.einsum("bnm,hdm->bhnd", X, Wk)
    if bq is not None:
        Q = Q + np.asarray(bq, dtype=np.float64)[None, :, None, :]
    if bk is not None:
        K = K + np.asarray(bk, dtype=np.float64)[None, :, None, :]
    return Q, K


def sigma(theta: float) -> float:
    """gamma^2 = sigma(theta)."""
    return 1.0 / (1.0 + np.exp(-float(theta)))


def project_backward(X, Wq, Wk, dQ, dK, theta: float, d_eps: float):
    """Chain rule of `project` and `sigma`: (dX, dWq, dWk, dbq, dbk, dtheta), all f64."""
    X = np.asarray(X, dtype=np.float64)
    dQ = np.asarray(dQ, dtype=np.float64)
    dK = np.asarray(dK, dtype=np.float64)
    Wq = np.asarray(Wq, dtype=np.float64)
    Wk = np.asarray(Wk, dtype=np.float64)
    dX = np.einsum("bhnd,hdm->bnm", dQ, Wq) + np.einsum("bhnd,hdm->bnm", dK, Wk)
    dWq = np.einsum("bhnd,bnm->hdm", dQ, X)
    dWk = np.einsum("bhnd,bnm->hdm", dK, X)
    dbq = dQ.sum(axis=(0, 2))
    dbk = dK.sum(axis=(0, 2))
    s = sigma(theta)
    dtheta = float(d_eps) * s * (1.0 - s)
    return dX, dWq, dWk, dbq, dbk, dtheta
