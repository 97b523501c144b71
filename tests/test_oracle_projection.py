"""Pins of the NEXT-4 projection oracle (oracle/projection.py) against what the definitions fix:
a hand-worked value, the coordinate-selector special case, the bias shift, the transposition
(adjoint) identity, central finite differences of a scalar loss, and sigma's closed forms.
CPU only."""
import numpy as np
import pytest

from oracle import projection as prj


def _rand(seed, B=2, H=3, N=5, d_k=3, d_model=7):
    rng = np.random.default_rng(seed)
    X = rng.normal(size=(B, N, d_model))
    Wq = rng.normal(size=(H, d_k, d_model))
    Wk = rng.normal(size=(H, d_k, d_model))
    bq = rng.normal(size=(H, d_k))
    bk = rng.normal(size=(H, d_k))
    return X, Wq, Wk, bq, bk


def test_hand_worked_value():
    """d_model 2, one head, d_k 1: q = 3*2 + (-1)*4 + 0.5 = 2.5, k = 0*2 + 2*4 - 1 = 7."""
    X = np.array([[[2.0, 4.0]]])
    Q, K = prj.project(X, np.array([[[3.0, -1.0]]]), np.array([[[0.0, 2.0]]]), np.array([[0.5]]),
                       np.array([[-1.0]]))
    assert Q.shape == (1, 1, 1, 1) and Q[0, 0, 0, 0] == 2.5
    assert K[0, 0, 0, 0] == 7.0


def test_selector_weights_copy_coordinates():
    """W_q[h][d][m] = [m == h*d_k + d] makes q_{b,h,n,d} = x_{b,n,h*d_k+d} exactly (plain loops)."""
    B, H, N, d_k = 2, 3, 4, 2
    d_model = H * d_k + 1
    X = np.random.default_rng(1).normal(size=(B, N, d_model))
    W = np.zeros((H, d_k, d_model))
    for h in range(H):
        for d in range(d_k):
            W[h, d, h * d_k + d] = 1.0
    Q, K = prj.project(X, W, 2.0 * W)
    for b in range(B):
        for h in range(H):
            for n in range(N):
                for d in range(d_k):
                    assert Q[b, h, n, d] == X[b, n, h * d_k + d]
                    assert K[b, h, n, d] == 2.0 * X[b, n, h * d_k + d]


def test_bias_is_a_shift_and_projection_is_linear():
    X, Wq, Wk, bq, bk = _rand(2)
    Q0, K0 = prj.project(X, Wq, Wk)
    Q1, K1 = prj.project(X, Wq, Wk, bq, bk)
    np.testing.assert_allclose(Q1 - Q0, np.broadcast_to(bq[None, :, None, :], Q0.shape), atol=1e-14)
    np.testing.assert_allclose(K1 - K0, np.broadcast_to(bk[None, :, None, :], K0.shape), atol=1e-14)
    Q2, _ = prj.project(3.0 * X, Wq, Wk)
    np.testing.assert_allclose(Q2, 3.0 * Q0, rtol=1e-13, atol=1e-13)


def test_transposition_identity():
    """<dQ, W x> = <W^T dQ, x>: the dX the backward returns is the adjoint of the projection."""
    X, Wq, Wk, _, _ = _rand(3)
    rng = np.random.default_rng(4)
    Q, K = prj.project(X, Wq, Wk)
    dQ = rng.normal(size=Q.shape)
    dK = rng.normal(size=K.shape)
    dX, *_ = prj.project_backward(X, Wq, Wk, dQ, dK, 0.0, 0.0)
    assert np.sum(dQ * Q) + np.sum(dK * K) == pytest.approx(np.sum(dX * X), rel=1e-12)


def test_backward_matches_central_differences():
    """L = <G_q, Q> + <G_k, K> + c * sigma(theta): every gradient against central FD (f64)."""
    X, Wq, Wk, bq, bk = _rand(5, B=1, H=2, N=3, d_k=2, d_model=4)
    rng = np.random.default_rng(6)
    Gq = rng.normal(size=(1, 2, 3, 2))
    Gk = rng.normal(size=(1, 2, 3, 2))
    c, theta = 0.7, 0.3

    def loss(X, Wq, Wk, bq, bk, theta):
        Q, K = prj.project(X, Wq, Wk, bq, bk)
        return np.sum(Gq * Q) + np.sum(Gk * K) + c * prj.sigma(theta)

    dX, dWq, dWk, dbq, dbk, dth = prj.project_backward(X, Wq, Wk, Gq, Gk, theta, c)
    h = 1e-6
    args = [X, Wq, Wk, bq, bk]
    for ai, g in enumerate((dX, dWq, dWk, dbq, dbk)):
        a = args[ai]
        for idx in np.ndindex(a.shape):
            ap, am = a.copy(), a.copy()
            ap[idx] += h
            am[idx] -= h
            pa = list(args)
            pa[ai] = ap
            ma = list(args)
            ma[ai] = am
            fd = (loss(*pa, theta) - loss(*ma, theta)) / (2 * h)
            assert fd == pytest.approx(g[idx], rel=1e-6, abs=1e-8), (ai, idx)
    fd = (loss(*args, theta + h) - loss(*args, theta - h)) / (2 * h)
    assert fd == pytest.approx(dth, rel=1e-7)


def test_sigma_closed_forms():
    assert prj.sigma(0.0) == 0.5                         # default theta = 0 -> eps = 0.5
    for t in (-3.0, -0.5, 0.25, 2.0, 10.0):
        assert prj.sigma(t) + prj.sigma(-t) == pytest.approx(1.0, abs=1e-15)
        assert 0.0 < prj.sigma(t) < 1.0                  # gamma^2 in (0, 1)
    *_, dth = prj.project_backward(np.zeros((1, 1, 1)), np.zeros((1, 1, 1)), np.zeros((1, 1, 1)),
                                   np.zeros((1, 1, 1, 1)), np.zeros((1, 1, 1, 1)), 0.0, 1.0)
    assert dth == 0.25                                   # sigma'(0) = 1/4
