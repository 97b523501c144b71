"""NEXT-4: the projections f_q, f_k and eps = sigma(theta) fused in front of the
encoder (onedf_project_encode / onedf_project_bwd) against oracle/projection.py, and the whole
projected layer (ZetaProjectedAttention) against oracle/projection.py + the attention oracle.

Contract (reading D27 / DESIGN R6): Q, K are f64 sums of exact f32 products rounded once to f32,
so they equal the oracle's f64 projection rounded to f32 up to one f32 rounding (rel 2^-23); the
codes, runs and index sets are then those of the oracle run on the GPU's Q, K (the float->integer
decisions are taken in the kernel's f32, D23); gradients within the fp32 contract (1e-5 / 1e-6).
"""
import numpy as np
import pytest

import oracle
import synth
from _util import assert_close, assert_same
from oracle import projection as prj

pytestmark = pytest.mark.gpu

F32_ULP = 2.0 ** -23


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


def _inputs(B, H, N, d_k, d_model, seed, bias=True):
    rng = np.random.default_rng(seed)
    X = rng.normal(size=(B, N, d_model)).astype(np.float32)
    s = 1.0 / np.sqrt(d_model)
    Wq = (s * rng.normal(size=(H, d_k, d_model))).astype(np.float32)
    Wk = (s * rng.normal(size=(H, d_k, d_model))).astype(np.float32)
    bq = rng.normal(size=(H, d_k)).astype(np.float32) if bias else None
    bk = rng.normal(size=(H, d_k)).astype(np.float32) if bias else None
    return X, Wq, Wk, bq, bk


def _t(a, dev):
    import torch
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).to(dev)


SHAPES = {
    "tiny": dict(B=1, H=1, N=256, d_k=2, d_v=16, k=8, window=16, chunk=32, d_model=8),
    "ragged": dict(B=2, H=3, N=300, d_k=3, d_v=8, k=8, window=16, chunk=64, d_model=37),
    "heads12": dict(B=2, H=12, N=512, d_k=3, d_v=8, k=8, window=16, chunk=64, d_model=96),
    "wide_model": dict(B=1, H=2, N=200, d_k=4, d_v=8, k=8, window=16, chunk=50, d_model=768),
}


@pytest.mark.parametrize("name", sorted(SHAPES))
@pytest.mark.parametrize("bias", [True, False])
def test_project_encode_and_bwd_parity(name, bias):
    import torch

    import paper_2501_14577_b200 as onedf
    sh = dict(SHAPES[name])
    dm = sh.pop("d_model")
    kw = dict(sh, causal=1, mean_slot=1)
    p = onedf.make_problem(**kw)
    X, Wq, Wk, bq, bk = _inputs(kw["B"], kw["H"], kw["N"], kw["d_k"], dm, seed=dm + kw["H"], bias=bias)
    dev = torch.device("cuda:0")
    theta = torch.tensor(0.37, device=dev)
    Q, K, eps, qc, kc, lohi = onedf.project_encode(p, _t(X, dev), _t(Wq, dev), _t(Wk, dev), _t(bq, dev),
                                                   _t(bk, dev), theta)
    Qr, Kr = prj.project(X, Wq, Wk, bq, bk)
    Qg, Kg = Q.cpu().numpy(), K.cpu().numpy()
    assert_close(Qg, Qr, "Q", rtol=F32_ULP, atol=1e-30)
    assert_close(Kg, Kr, "K", rtol=F32_ULP, atol=1e-30)
    assert float(eps) == np.float32(prj.sigma(0.37))
    # the encoder ran on exactly these Q, K
    op = oracle.Problem(**kw)
    qref, kref, lref = oracle.encode(op, Qg, Kg)
    assert_same(qc.cpu().numpy().view(np.uint64), qref, "qcode")
    assert_same(kc.cpu().numpy().view(np.uint64), kref, "kcode")
    assert_same(lohi.cpu().numpy(), lref, "lohi")
    # backward against the oracle's chain rule on the same dQ, dK
    rng = np.random.default_rng(7)
    dQ = rng.normal(size=Qg.shape).astype(np.float32)
    dK = rng.normal(size=Kg.shape).astype(np.float32)
    d_eps = torch.tensor(-1.25, dtype=torch.float64, device=dev)
    dX, dWq, dWk, dbq, dbk, dth = onedf.project_bwd(p, _t(X, dev), _t(Wq, dev), _t(Wk, dev), _t(dQ, dev),
                                                    _t(dK, dev), theta, d_eps)
    ref = prj.project_backward(X, Wq, Wk, dQ, dK, 0.37, -1.25)
    for got, want, n in zip((dX, dWq, dWk, dbq, dbk), ref[:5], ("dX", "dWq", "dWk", "dbq", "dbk")):
        assert_close(got.cpu().numpy(), want, n)
    assert float(dth) == pytest.approx(ref[5], rel=1e-6)


def test_project_bwd_bitwise_deterministic():
    import torch

    import paper_2501_14577_b200 as onedf
    kw = dict(B=2, H=4, N=1000, d_k=3, d_v=8, k=8, window=16, chunk=100, causal=1, mean_slot=1)
    p = onedf.make_problem(**kw)
    X, Wq, Wk, _, _ = _inputs(2, 4, 1000, 3, 64, seed=3)
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(9)
    dQ = _t(rng.normal(size=(2, 4, 1000, 3)).astype(np.float32), dev)
    dK = _t(rng.normal(size=(2, 4, 1000, 3)).astype(np.float32), dev)
    a = onedf.project_bwd(p, _t(X, dev), _t(Wq, dev), _t(Wk, dev), dQ, dK, bias=True)
    b = onedf.project_bwd(p, _t(X, dev), _t(Wq, dev), _t(Wk, dev), dQ, dK, bias=True)
    for u, v in zip(a[:5], b[:5]):
        assert torch.equal(u, v)


@pytest.mark.parametrize("vdtype", [0, 1])
def test_projected_layer_autograd(vdtype):
    """x -> f_q, f_k, sigma -> top-k Cauchy attention, fwd + bwd through torch.autograd against the
    oracle chain: oracle projection, the attention oracle on the GPU's Q, K (D23), the oracle's
    projection backward of the attention oracle's dQ, dK, d_eps."""
    import torch

    import paper_2501_14577_b200 as onedf
    from _util import assert_close_bf16, bf16_round
    B, H, N, dk, dv, dm = 1, 2, 512, 3, 16, 24
    kw = dict(B=B, H=H, N=N, d_k=dk, d_v=dv, k=8, window=16, chunk=64, causal=1, mean_slot=1)
    p = onedf.make_problem(**kw, vdtype=vdtype)
    X, Wq, Wk, bq, bk = _inputs(B, H, N, dk, dm, seed=11)
    rng = np.random.default_rng(12)
    V = rng.normal(size=(B, H, N, dv)).astype(np.float32)
    dO = rng.normal(size=(B, H, N, dv)).astype(np.float32)
    if vdtype:
        V, dO = bf16_round(V), bf16_round(dO)
    dev = torch.device("cuda:0")
    vt = onedf.value_dtype(p)
    Xt, Wqt, Wkt, bqt, bkt = (_t(a, dev).requires_grad_() for a in (X, Wq, Wk, bq, bk))
    th = torch.tensor(-0.2, device=dev, requires_grad=True)
    Vt = _t(V, dev).to(vt).requires_grad_()
    O, idx = onedf.zeta_projected_attention(Xt, Wqt, Wkt, bqt, bkt, th, Vt, p)
    O.backward(_t(dO, dev).to(vt))
    # oracle chain, on the GPU's projected coordinates (the quantiser/ranking decisions)
    Qg, Kg, eps, *_ = onedf.project_encode(p, _t(X, dev), _t(Wq, dev), _t(Wk, dev), _t(bq, dev), _t(bk, dev),
                                           th.detach())
    ref = oracle.pipeline(oracle.Problem(**kw), Qg.cpu().numpy(), Kg.cpu().numpy(), V, float(eps), dO)
    assert_same(idx.cpu().numpy(), ref["idx"], "idx")
    check = assert_close_bf16 if vdtype else assert_close
    check(O.detach().float().cpu().numpy(), ref["O"], "O")
    check(Vt.grad.float().cpu().numpy(), ref["dV"], "dV")
    dX, dWq, dWk, dbq, dbk, dth = prj.project_backward(X, Wq, Wk, ref["dQ"], ref["dK"], -0.2, ref["d_eps"])
    for got, want, n in ((Xt.grad, dX, "dX"), (Wqt.grad, dWq, "dWq"), (Wkt.grad, dWk, "dWk"), (bqt.grad, dbq, "dbq"),
                         (bkt.grad, dbk, "dbk")):
        assert_close(got.cpu().numpy(), want, n, rtol=2e-5, atol=2e-6)
    assert float(th.grad) == pytest.approx(dth, rel=2e-5, abs=2e-6)


def test_project_encode_long64k_shape_sampled():
    """The bench's long64k workload fed from token features (d_model 768 = 12 heads x 64):
    Q, K on sampled rows, the codes of every row."""
    import torch

    import paper_2501_14577_b200 as onedf
    cfg = synth.CONFIGS["long64k"].with_(B=1, H=12)
    kw = cfg.problem_kwargs()
    p = onedf.make_problem(**kw)
    dm = 768
    X, Wq, Wk, bq, bk = _inputs(1, 12, cfg.N, 3, dm, seed=21)
    dev = torch.device("cuda:0")
    Q, K, _, qc, kc, _ = onedf.project_encode(p, _t(X, dev), _t(Wq, dev), _t(Wk, dev), _t(bq, dev), _t(bk, dev))
    rows = np.random.default_rng(0).choice(cfg.N, size=512, replace=False)
    Qr, Kr = prj.project(X[:, rows], Wq, Wk, bq, bk)
    assert_close(Q.cpu().numpy()[:, :, rows], Qr, "Q[sampled]", rtol=F32_ULP, atol=1e-30)
    assert_close(K.cpu().numpy()[:, :, rows], Kr, "K[sampled]", rtol=F32_ULP, atol=1e-30)
    qref, kref, _ = oracle.encode(oracle.Problem(**kw), Q.cpu().numpy(), K.cpu().numpy())
    assert_same(qc.cpu().numpy().view(np.uint64), qref, "qcode")
    assert_same(kc.cpu().numpy().view(np.uint64), kref, "kcode")
