"""NEXT-4: bfloat16 storage of the value rows V, O, dO, dV with f64
accumulation (onedf_problem.vdtype = ONEDF_DTYPE_BF16, reading D26).

Parity contract: the oracle consumes the bf16-rounded V and dO exactly (they are
f32/f64-representable), so codes, runs and index sets stay bit-exact; dQ, dK, Z and
d_eps stay within the fp32 contract (1e-5 rel / 1e-6 abs: they are computed in f64 from
the same values); O and dV are ONE round-to-nearest to bfloat16 of a value within that
contract (`assert_close_bf16`: half a bf16 ulp + 1e-6 + 1e-5 |ref|).
"""
import numpy as np
import pytest

import oracle
import synth
from _util import assert_close, assert_close_bf16, assert_same, bf16_round, gpu_run, oracle_run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


def _rounded(x):
    """The inputs the bf16 path sees: V and dO rounded to bfloat16 (kept as exact float32)."""
    y = dict(x)
    for n in ("V", "dO"):
        if n in y:
            y[n] = bf16_round(y[n])
    return y


def _okw(kw):
    """The oracle's problem: the storage type is not part of what it computes."""
    return {n: v for n, v in kw.items() if n != "vdtype"}


def _compare(got, ref, bwd=True):
    for n in ("qcode", "kcode", "scode", "perm", "idx"):
        assert_same(got[n], ref[n], n)
    assert_close_bf16(got["O"], ref["O"], "O")
    assert_close(got["Z"], ref["Z"], "Z")
    if bwd:
        assert_close(got["dQ"], ref["dQ"], "dQ")
        assert_close(got["dK"], ref["dK"], "dK")
        assert_close_bf16(got["dV"], ref["dV"], "dV")
        assert_close(got["d_eps"], ref["d_eps"], "d_eps")


SMALL = {
    "tiny": synth.CONFIGS["tiny"].problem_kwargs(),
    "ragged_last_chunk": dict(B=2, H=1, N=300, d_k=3, d_v=16, k=8, window=16, chunk=64, causal=1, mean_slot=1),
    "noncausal": dict(B=1, H=2, N=200, d_k=3, d_v=16, k=8, window=32, chunk=1, causal=0, mean_slot=1),
    "no_mean_slot": dict(B=1, H=2, N=256, d_k=2, d_v=8, k=8, window=16, chunk=32, causal=1, mean_slot=0),
    "noncausal_no_mean": dict(B=1, H=1, N=100, d_k=3, d_v=8, k=4, window=8, chunk=1, causal=0, mean_slot=0),
    "dv4": dict(B=1, H=1, N=128, d_k=3, d_v=4, k=4, window=8, chunk=16, causal=1, mean_slot=1),
    "dv20": dict(B=1, H=1, N=128, d_k=3, d_v=20, k=4, window=8, chunk=16, causal=1, mean_slot=1),
    "dv256": dict(B=1, H=2, N=256, d_k=3, d_v=256, k=16, window=32, chunk=32, causal=1, mean_slot=1),
    "k100": dict(B=1, H=1, N=1024, d_k=3, d_v=8, k=100, window=150, chunk=256, causal=1, mean_slot=1),
    "dk8": dict(B=1, H=1, N=256, d_k=8, d_v=8, k=8, window=16, chunk=32, causal=1, mean_slot=1),
    "N1": dict(B=1, H=1, N=1, d_k=3, d_v=8, k=4, window=8, chunk=1, causal=1, mean_slot=1),
}


def zlib_seed(name):
    import zlib
    return zlib.crc32(name.encode())


@pytest.mark.parametrize("name", sorted(SMALL))
def test_small_problem_bf16_parity(name):
    kw = dict(SMALL[name], vdtype=1)
    rng = np.random.default_rng(zlib_seed(name))
    B, H, N, dk, dv = kw["B"], kw["H"], kw["N"], kw["d_k"], kw["d_v"]
    x = dict(Q=rng.normal(size=(B, H, N, dk)).astype(np.float32), K=rng.normal(size=(B, H, N, dk)).astype(np.float32),
             V=rng.normal(size=(B, H, N, dv)).astype(np.float32), dO=rng.normal(size=(B, H, N, dv)).astype(np.float32))
    got = gpu_run(kw, x)
    ref = oracle_run(_okw(kw), _rounded(x))
    _compare(got, ref)


@pytest.mark.parametrize("score", [1, 2, 3])
def test_score_variants_bf16(score):
    kw = dict(B=1, H=2, N=256, d_k=3, d_v=16, k=8, window=16, chunk=32, causal=1, mean_slot=1, score=score, vdtype=1)
    rng = np.random.default_rng(score)
    x = {n: rng.normal(size=(1, 2, 256, w)).astype(np.float32) for n, w in (("Q", 3), ("K", 3), ("V", 16), ("dO", 16))}
    got = gpu_run(kw, x)
    p = oracle.Problem(**_okw(kw))
    xr = _rounded(x)
    ref = oracle.pipeline(p, xr["Q"], xr["K"], xr["V"], synth.EPS, xr["dO"])
    _compare(got, ref)


@pytest.mark.parametrize("name", ["ar", "ar_tokens", "wiki"])
def test_config_slices_bf16(name):
    """BASELINE shapes, two (b,h) slices each, every element."""
    cfg = synth.CONFIGS[name]
    x = synth.make_inputs(cfg, bh_range=range(2))
    kw = dict(cfg.problem_kwargs(), B=1, H=2, vdtype=1)
    got = gpu_run(kw, x)
    ref = oracle_run(_okw(kw), _rounded(x))
    _compare(got, ref)


def test_long64k_slice0_bf16():
    """The bench workload's first (b,h) slice in bf16 storage: every element of slice 0."""
    cfg = synth.CONFIGS["long64k"]
    x = synth.make_inputs(cfg, bh_range=range(1))
    kw = dict(cfg.problem_kwargs(), B=1, H=1, vdtype=1)
    got = gpu_run(kw, x)
    ref = oracle_run(_okw(kw), _rounded(x))
    _compare(got, ref)


def test_bf16_matches_f32_path_on_representable_inputs():
    """With V, dO already bf16-representable, the f32 path and the bf16 path compute the same f64
    sums: idx/Z/dQ/dK/d_eps bitwise equal, O and dV the bf16 rounding of the f32 path's values
    (within one bf16 rounding of each other)."""
    cfg = synth.CONFIGS["ar"]
    x = _rounded(synth.make_inputs(cfg, bh_range=range(1)))
    kw = dict(cfg.problem_kwargs(), B=1, H=1)
    a = gpu_run(kw, x)
    b = gpu_run(dict(kw, vdtype=1), x)
    for n in ("idx", "Z", "dQ", "dK", "d_eps"):
        assert np.array_equal(np.atleast_1d(a[n]).view(np.uint8), np.atleast_1d(b[n]).view(np.uint8)), n
    assert_close_bf16(b["O"], a["O"], "O", rtol=0, atol=0)
    assert_close_bf16(b["dV"], a["dV"], "dV", rtol=0, atol=0)


def test_autograd_and_host_step_bf16():
    import torch

    import paper_2501_14577_b200 as onedf
    cfg = synth.CONFIGS["tiny"]
    kw = dict(cfg.problem_kwargs(), vdtype=1)
    x = synth.make_inputs(cfg)
    ref = oracle_run(_okw(kw), _rounded(x))
    dev = torch.device("cuda:0")
    p = onedf.make_problem(**kw)
    Q, K = (torch.from_numpy(x[n]).to(dev).requires_grad_() for n in ("Q", "K"))
    V = torch.from_numpy(x["V"]).to(dev).to(torch.bfloat16).requires_grad_()
    eps = torch.tensor(synth.EPS, device=dev, requires_grad=True)
    O, idx = onedf.zeta_attention(Q, K, V, eps, p)
    assert O.dtype == torch.bfloat16
    O.backward(torch.from_numpy(x["dO"]).to(dev).to(torch.bfloat16))
    assert V.grad.dtype == torch.bfloat16
    assert_close_bf16(O.detach().float().cpu().numpy(), ref["O"], "O")
    assert_close(Q.grad.cpu().numpy(), ref["dQ"], "dQ")
    assert_close(K.grad.cpu().numpy(), ref["dK"], "dK")
    assert_close_bf16(V.grad.float().cpu().numpy(), ref["dV"], "dV")
    assert_close(float(eps.grad), ref["d_eps"], "d_eps", rtol=1e-5, atol=1e-5)
    # host-buffer step with bf16 value rows (half the PCIe bytes of V, dO, O, dV)
    hs = onedf.HostStep(p, dev)
    pin = {n: torch.from_numpy(v).pin_memory() for n, v in x.items()}
    for n in ("V", "dO"):
        pin[n] = pin[n].to(torch.bfloat16).pin_memory()
    outs = {n: torch.empty_like(pin["V" if n in ("O", "dV") else "Q"]).pin_memory() for n in ("O", "dQ", "dK", "dV")}
    d_eps = torch.zeros((), dtype=torch.float64).pin_memory()
    hs(pin["Q"], pin["K"], pin["V"], synth.EPS, pin["dO"], outs["O"], outs["dQ"], outs["dK"], outs["dV"], d_eps)
    torch.cuda.synchronize()
    assert onedf.HostStep.h2d_bytes(p) == sum(pin[n].numel() * pin[n].element_size() for n in ("Q", "K", "V", "dO"))
    assert_close_bf16(outs["O"].float().numpy(), ref["O"], "host O")
    assert_close_bf16(outs["dV"].float().numpy(), ref["dV"], "host dV")
    assert_close(outs["dQ"].numpy(), ref["dQ"], "host dQ")
    assert_close(outs["dK"].numpy(), ref["dK"], "host dK")
    assert_close(float(d_eps), ref["d_eps"], "host d_eps")


def test_bf16_rejects_float_rows_and_sharding():
    import torch

    import paper_2501_14577_b200 as onedf
    kw = dict(B=1, H=1, N=64, d_k=3, d_v=8, k=4, window=8, chunk=16, causal=1, mean_slot=1)
    with pytest.raises(onedf.OnedfError):
        onedf.make_problem(**kw, vdtype=1, shard_rank=0, shard_world=2)   # sharded bf16: UNSUPPORTED
    with pytest.raises(onedf.OnedfError):
        onedf.make_problem(**kw, vdtype=2)
    p = onedf.make_problem(**kw, vdtype=1)
    dev = torch.device("cuda:0")
    Q = torch.randn(1, 1, 64, 3, device=dev)
    qc, kc, _ = onedf.encode(p, Q, Q)
    sc, pm = onedf.sort(p, kc)
    with pytest.raises(ValueError):       # float V for a bf16 problem: refused before the ABI
        onedf.topk_attn_fwd(p, Q, Q, torch.randn(1, 1, 64, 8, device=dev), torch.tensor(0.5, device=dev), qc, sc, pm)
