"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bit-exact for codes, permutations and index sets (the
top-k decision is taken in f32 with the same pinned op order on both sides,
reading D23); outputs and gradients within 1e-5 rel / 1e-6 abs (north_star).
"""
import zlib

import numpy as np
import pytest

import oracle
import synth
from _util import assert_close, assert_same, gpu_run, oracle_run, slice_inputs, slice_out

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


def _rand_inputs(kw, seed, scale=1.0, dup_keys=False):
    rng = np.random.default_rng(seed)
    B, H, N, dk, dv = kw["B"], kw["H"], kw["N"], kw["d_k"], kw["d_v"]
    x = dict(Q=(scale * rng.normal(size=(B, H, N, dk))).astype(np.float32),
             K=(scale * rng.normal(size=(B, H, N, dk))).astype(np.float32),
             V=rng.normal(size=(B, H, N, dv)).astype(np.float32),
             dO=rng.normal(size=(B, H, N, dv)).astype(np.float32))
    if dup_keys:   # repeated tokens: identical key rows -> code ties, distance ties, hub keys
        vocab = rng.normal(size=(7, dk)).astype(np.float32)
        tok = rng.integers(0, 7, size=(B, H, N))
        x["K"] = vocab[tok]
        x["Q"] = (vocab[tok] + 0.05 * rng.normal(size=(B, H, N, dk))).astype(np.float32)
    return x


def _compare_all(got, ref, bwd=True):
    assert_same(got["qcode"], ref["qcode"], "qcode")
    assert_same(got["kcode"], ref["kcode"], "kcode")
    assert_same(got["scode"], ref["scode"], "scode")
    assert_same(got["perm"], ref["perm"], "perm")
    assert_same(got["idx"], ref["idx"], "idx")
    assert_close(got["O"], ref["O"], "O")
    assert_close(got["Z"], ref["Z"], "Z")
    if bwd:
        assert_close(got["dQ"], ref["dQ"], "dQ")
        assert_close(got["dK"], ref["dK"], "dK")
        assert_close(got["dV"], ref["dV"], "dV")
        assert_close(got["d_eps"], ref["d_eps"], "d_eps")


# ------------------------------------------------------------------ small problems: every output, every element
EDGE = {
    "tiny": synth.CONFIGS["tiny"].problem_kwargs(),
    "ragged_last_chunk": dict(B=2, H=1, N=300, d_k=3, d_v=16, k=8, window=16, chunk=64, causal=1, mean_slot=1),
    "noncausal": dict(B=1, H=2, N=200, d_k=3, d_v=16, k=8, window=32, chunk=1, causal=0, mean_slot=1),
    "no_mean_slot": dict(B=1, H=2, N=256, d_k=2, d_v=8, k=8, window=16, chunk=32, causal=1, mean_slot=0),
    "noncausal_no_mean": dict(B=1, H=1, N=100, d_k=3, d_v=8, k=4, window=8, chunk=1, causal=0, mean_slot=0),
    "dk1": dict(B=1, H=2, N=256, d_k=1, d_v=8, k=5, window=10, chunk=32, causal=1, mean_slot=1),
    "dk4": dict(B=1, H=2, N=256, d_k=4, d_v=8, k=8, window=16, chunk=32, causal=1, mean_slot=1),
    "dk5": dict(B=1, H=1, N=256, d_k=5, d_v=8, k=8, window=16, chunk=32, causal=1, mean_slot=1),
    "dk8": dict(B=1, H=1, N=256, d_k=8, d_v=8, k=8, window=16, chunk=32, causal=1, mean_slot=1),
    "dv4": dict(B=1, H=1, N=128, d_k=3, d_v=4, k=4, window=8, chunk=16, causal=1, mean_slot=1),
    "dv20": dict(B=1, H=1, N=128, d_k=3, d_v=20, k=4, window=8, chunk=16, causal=1, mean_slot=1),
    "dv256": dict(B=1, H=2, N=256, d_k=3, d_v=256, k=16, window=32, chunk=32, causal=1, mean_slot=1),
    "k1": dict(B=1, H=1, N=256, d_k=3, d_v=8, k=1, window=2, chunk=32, causal=1, mean_slot=1),
    "k256": dict(B=1, H=1, N=2048, d_k=3, d_v=8, k=256, window=512, chunk=512, causal=1, mean_slot=1),
    "k100": dict(B=1, H=1, N=1024, d_k=3, d_v=8, k=100, window=150, chunk=256, causal=1, mean_slot=1),
    "window_eq_k": dict(B=1, H=2, N=256, d_k=3, d_v=8, k=8, window=8, chunk=32, causal=1, mean_slot=1),
    "window_odd": dict(B=1, H=1, N=256, d_k=3, d_v=8, k=7, window=13, chunk=32, causal=1, mean_slot=1),
    "many_runs_M1": dict(B=1, H=1, N=100, d_k=3, d_v=8, k=6, window=6, chunk=1, causal=1, mean_slot=1),
    "runs_gt_32": dict(B=1, H=1, N=700, d_k=3, d_v=8, k=8, window=16, chunk=10, causal=1, mean_slot=1),
    "N1": dict(B=1, H=1, N=1, d_k=3, d_v=8, k=4, window=8, chunk=1, causal=1, mean_slot=1),
    "N1_noncausal": dict(B=1, H=1, N=1, d_k=3, d_v=8, k=4, window=8, chunk=1, causal=0, mean_slot=1),
    "chunk_gt_N": dict(B=1, H=1, N=50, d_k=3, d_v=8, k=4, window=8, chunk=64, causal=1, mean_slot=1),
    "bits_small": dict(B=1, H=1, N=256, d_k=3, d_v=8, k=8, window=16, chunk=32, bits=3, causal=1, mean_slot=1),
    # odd run lengths (the on-chip sort's position/histogram arrays must stay aligned)
    "odd_runs_causal": dict(B=1, H=2, N=400, d_k=3, d_v=8, k=8, window=16, chunk=65, causal=1, mean_slot=1),
    "odd_run_noncausal": dict(B=2, H=1, N=201, d_k=3, d_v=8, k=8, window=16, chunk=1, causal=0, mean_slot=1),
    "seg_8192": dict(B=1, H=1, N=16384, d_k=3, d_v=8, k=8, window=16, chunk=8192, causal=1, mean_slot=1),
    # runs longer than the on-chip sort limit (global-scratch sort path)
    "seg_big_causal": dict(B=1, H=2, N=20000, d_k=3, d_v=8, k=8, window=16, chunk=10000, causal=1, mean_slot=1),
    "seg_big_noncausal": dict(B=1, H=1, N=9000, d_k=2, d_v=8, k=8, window=16, chunk=1, causal=0, mean_slot=1),
}


@pytest.mark.parametrize("name", list(EDGE))
def test_small_problem_full_parity(name):
    kw = EDGE[name]
    x = synth.make_inputs(synth.CONFIGS["tiny"]) if name == "tiny" else _rand_inputs(kw, seed=zlib.crc32(name.encode()) % 1000)
    _compare_all(gpu_run(kw, x), oracle_run(kw, x))


@pytest.mark.parametrize("causal", [1, 0])
def test_duplicate_keys_full_parity(causal):
    kw = dict(B=1, H=2, N=512, d_k=3, d_v=16, k=16, window=32, chunk=64, causal=causal, mean_slot=1)
    x = _rand_inputs(kw, seed=77, dup_keys=True)
    _compare_all(gpu_run(kw, x), oracle_run(kw, x))


def test_fixed_bounds_and_clamping():
    kw = dict(B=1, H=2, N=256, d_k=3, d_v=8, k=8, window=16, chunk=32, causal=1, mean_slot=1)
    x = _rand_inputs(kw, seed=5, scale=2.0)
    lohi = np.zeros((1, 2, 2, 3))
    lohi[..., 0, :] = -1.5            # narrower than the data: exercises clamping
    lohi[..., 1, :] = 1.5
    _compare_all(gpu_run(kw, x, lohi=lohi), oracle_run(kw, x, lohi=lohi))


def test_eps_values():
    kw = EDGE["ragged_last_chunk"]
    x = _rand_inputs(kw, seed=9)
    for eps in (1e-3, 0.5, 0.9999):
        _compare_all(gpu_run(kw, x, eps=eps), oracle_run(kw, x, eps=eps))


# ------------------------------------------------------------------ BASELINE.json configs
# the grouped selection of repeated keys (fwd_kernels.cuh select_groups): many equal distances
# collected (cnt > 128, ties among the first sorted keys) or more than FWD_CAP at or below T; k
# spans R = 1, 2, 4 register rows; "mirror" puts distinct key rows at exactly equal distance from
# queries at the origin (two groups of equal D in one run -> the streaming fallback); every
# result bit-exact / within tolerance of the oracle
TIE_CASES = {
    "k16_causal": (dict(B=1, H=2, N=2048, d_k=3, d_v=16, k=16, window=64, chunk=128, causal=1, mean_slot=1), 5),
    "k64_causal": (dict(B=1, H=2, N=4096, d_k=3, d_v=64, k=64, window=128, chunk=256, causal=1, mean_slot=1), 9),
    "k100_causal": (dict(B=1, H=1, N=4096, d_k=3, d_v=8, k=100, window=160, chunk=512, causal=1, mean_slot=1), 6),
    "k64_noncausal": (dict(B=1, H=1, N=2048, d_k=3, d_v=8, k=64, window=128, chunk=1, causal=0, mean_slot=1), 9),
    "k64_mirror": (dict(B=1, H=1, N=2048, d_k=3, d_v=8, k=64, window=128, chunk=256, causal=1, mean_slot=1), -4),
}


@pytest.mark.parametrize("name", list(TIE_CASES))
def test_repeated_keys_grouped_selection(name):
    kw, vocab = TIE_CASES[name]
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    B, H, N, dk = kw["B"], kw["H"], kw["N"], kw["d_k"]
    x = _rand_inputs(kw, seed=zlib.crc32(name.encode()) % 1000)
    if vocab > 0:
        emb = rng.normal(size=(vocab, dk)).astype(np.float32)
        tok = rng.integers(0, vocab, size=(B, H, N))
        x["K"] = emb[tok]
        x["Q"] = (emb[tok] + 0.05 * rng.normal(size=(B, H, N, dk))).astype(np.float32)
    else:
        v = rng.normal(size=(-vocab, dk)).astype(np.float32)
        emb = np.concatenate([v, -v])                     # +v and -v: equal distance from the origin
        tok = rng.integers(0, len(emb), size=(B, H, N))
        x["K"] = emb[tok]
        x["Q"] = (0.3 * rng.normal(size=(B, H, N, dk))).astype(np.float32)
        x["Q"][:, :, ::3] = 0.0                           # every third query at the origin
    _compare_all(gpu_run(kw, x), oracle_run(kw, x))


CONFIG_NAMES = ["ar", "ar_tokens", "lra_nc", "lra_c", "lra_tokens", "wiki", "wiki_tokens"]


@pytest.mark.parametrize("name", CONFIG_NAMES)
def test_config_parity(name):
    """Full-size run of the config on the GPU; codes/runs compared everywhere; idx/O/Z and all
    gradients compared on the first and last (b,h) slices in full, idx/O/Z on sampled queries
    of every slice."""
    cfg = synth.CONFIGS[name]
    kw = cfg.problem_kwargs()
    x = synth.make_inputs(cfg)
    got = gpu_run(kw, x)
    p = oracle.Problem(**kw)
    qc, kc, _ = oracle.encode(p, x["Q"], x["K"])
    sc, pm = oracle.sort(p, kc)
    assert_same(got["qcode"], qc, "qcode")
    assert_same(got["kcode"], kc, "kcode")
    assert_same(got["scode"], sc, "scode")
    assert_same(got["perm"], pm, "perm")
    bhs = [0, cfg.BH - 1]
    xs = slice_inputs(x, bhs)
    kws = dict(kw, B=1, H=len(bhs))
    ref = oracle_run(kws, xs)
    for n in ("idx", "O", "Z", "dQ", "dK", "dV"):
        (assert_same if n == "idx" else assert_close)(slice_out(got[n], bhs), ref[n], f"{n}[slices {bhs}]")
    # sampled queries of all slices
    sel = synth.sample_queries(cfg, 2000)
    idx_ref = oracle.select(p, x["Q"], x["K"], qc, sc, pm, sel=sel)
    assert_same(got["idx"].reshape(-1, cfg.k)[sel], idx_ref, "idx[sampled]")
    O_ref, Z_ref = oracle.forward(p, x["Q"], x["K"], x["V"], synth.EPS, idx_ref, sel=sel)
    assert_close(got["O"].reshape(-1, cfg.d_v)[sel], O_ref, "O[sampled]")
    assert_close(got["Z"].reshape(-1)[sel], Z_ref, "Z[sampled]")
    _gradient_invariants(kw, x, got)


def _gradient_invariants(kw, x, got):
    """Exact identities for fixed I on every (b,h) slice (f32 outputs -> relative tolerance)."""
    dQ, dK, dV = (got[n].astype(np.float64) for n in ("dQ", "dK", "dV"))
    Q, K, dO = (x[n].astype(np.float64) for n in ("Q", "K", "dO"))
    t = dQ.sum(2) + dK.sum(2)
    assert np.all(np.abs(t) <= 1e-5 * (np.abs(dQ).sum(2) + np.abs(dK).sum(2)) + 1e-6)
    s = dV.sum(2) - dO.sum(2)
    if kw["mean_slot"]:
        assert np.all(np.abs(s) <= 1e-5 * np.abs(dO).sum(2) + 1e-6)
    euler = (Q * dQ).sum((2, 3)) + (K * dK).sum((2, 3))
    scale = np.abs(Q * dQ).sum((2, 3)) + np.abs(K * dK).sum((2, 3))
    # 2 eps deps is a scalar over all slices: check the sum
    assert abs(euler.sum() + 2 * synth.EPS * float(got["d_eps"])) <= 1e-5 * scale.sum() + 1e-6


def test_long64k_bench_config_sampled():
    """BASELINE metric config in bench.py's launch configuration: the full 96-slice problem on
    one GPU; slice 0 (and the last slice's idx/O on sampled queries) against the oracle,
    invariants on every slice."""
    cfg = synth.CONFIGS["long64k"]
    kw = cfg.problem_kwargs()
    x = synth.make_inputs(cfg)
    got = gpu_run(kw, x)
    bhs = [0]
    ref = oracle_run(dict(kw, B=1, H=1), slice_inputs(x, bhs))
    for n in ("qcode", "kcode", "scode", "perm", "idx"):
        assert_same(slice_out(got[n], bhs), ref[n], f"{n}[slice 0]")
    for n in ("O", "Z", "dQ", "dK", "dV"):
        assert_close(slice_out(got[n], bhs), ref[n], f"{n}[slice 0]")
    last = [cfg.BH - 1]
    xl = slice_inputs(x, last)
    pl = oracle.Problem(**dict(kw, B=1, H=1))
    qc, kc, _ = oracle.encode(pl, xl["Q"], xl["K"])
    sc, pm = oracle.sort(pl, kc)
    sel = synth.sample_queries(cfg.with_(B=1, H=1), 512)
    idx_ref = oracle.select(pl, xl["Q"], xl["K"], qc, sc, pm, sel=sel)
    assert_same(slice_out(got["idx"], last).reshape(-1, cfg.k)[sel], idx_ref, "idx[last, sampled]")
    O_ref, _ = oracle.forward(pl, xl["Q"], xl["K"], xl["V"], synth.EPS, idx_ref, sel=sel)
    assert_close(slice_out(got["O"], last).reshape(-1, cfg.d_v)[sel], O_ref, "O[last, sampled]")
    _gradient_invariants(kw, x, got)
    # structural invariants on every query: causality, |I_i| = min(k, m M), no duplicates
    idx = got["idx"].reshape(cfg.BH, cfg.N, cfg.k)
    i = np.arange(cfg.N)
    lim = (i // cfg.chunk) * cfg.chunk
    valid = idx >= 0
    assert np.all(np.where(valid, idx < lim[None, :, None], True))
    assert np.all(valid.sum(-1) == np.minimum(cfg.k, lim)[None, :])


@pytest.mark.parametrize("name", ["long512k", "long1m"])
def test_long_sequence_single_slice_sampled(name):
    """BASELINE long-sequence scaling shapes (runs of 16K / 32K keys, sorted through global
    scratch) on one (b,h) slice: codes, runs and permutation bit-exact everywhere, idx/O/Z on
    sampled queries, gradient invariants."""
    cfg = synth.CONFIGS[name].with_(B=1, H=1)
    kw = cfg.problem_kwargs()
    x = synth.make_inputs(cfg)
    got = gpu_run(kw, x)
    p = oracle.Problem(**kw)
    qc, kc, _ = oracle.encode(p, x["Q"], x["K"])
    sc, pm = oracle.sort(p, kc)
    assert_same(got["qcode"], qc, "qcode")
    assert_same(got["kcode"], kc, "kcode")
    assert_same(got["scode"], sc, "scode")
    assert_same(got["perm"], pm, "perm")
    sel = synth.sample_queries(cfg, 300)
    idx_ref = oracle.select(p, x["Q"], x["K"], qc, sc, pm, sel=sel)
    assert_same(got["idx"].reshape(-1, cfg.k)[sel], idx_ref, "idx[sampled]")
    O_ref, Z_ref = oracle.forward(p, x["Q"], x["K"], x["V"], synth.EPS, idx_ref, sel=sel)
    assert_close(got["O"].reshape(-1, cfg.d_v)[sel], O_ref, "O[sampled]")
    assert_close(got["Z"].reshape(-1)[sel], Z_ref, "Z[sampled]")
    _gradient_invariants(kw, x, got)


def test_determinism_bitwise():
    cfg = synth.CONFIGS["ar_tokens"]
    kw = cfg.problem_kwargs()
    x = synth.make_inputs(cfg)
    a = gpu_run(kw, x)
    b = gpu_run(kw, x)
    for n in a:
        assert np.array_equal(np.atleast_1d(a[n]).view(np.uint8), np.atleast_1d(b[n]).view(np.uint8)), n


def _hub_inputs(kw, seed, vocab=4):
    """Few distinct key rows: the lowest-position copies of each token are selected by most
    queries, so key in-degrees exceed the key side's on-chip segment limit (256)."""
    rng = np.random.default_rng(seed)
    B, H, N, dk, dv = kw["B"], kw["H"], kw["N"], kw["d_k"], kw["d_v"]
    voc = rng.normal(size=(vocab, dk)).astype(np.float32)
    tok = rng.integers(0, vocab, size=(B, H, N))
    return dict(K=voc[tok], Q=(voc[tok] + 0.01 * rng.normal(size=(B, H, N, dk))).astype(np.float32),
                V=rng.normal(size=(B, H, N, dv)).astype(np.float32),
                dO=rng.normal(size=(B, H, N, dv)).astype(np.float32))


@pytest.mark.parametrize("causal", [1, 0])
def test_hub_keys_long_segments_parity_and_determinism(causal):
    kw = dict(B=1, H=2, N=2048, d_k=3, d_v=16, k=32, window=64, chunk=256, causal=causal, mean_slot=1)
    x = _hub_inputs(kw, seed=5 + causal)
    a = gpu_run(kw, x)
    ref = oracle_run(kw, x)
    indeg = np.bincount(a["idx"][a["idx"] >= 0].ravel(), minlength=1)
    assert indeg.max() > 256                       # the long-segment path is exercised
    _compare_all(a, ref)
    b = gpu_run(kw, x)
    for n in ("dQ", "dK", "dV", "d_eps"):
        assert np.array_equal(np.atleast_1d(a[n]).view(np.uint8), np.atleast_1d(b[n]).view(np.uint8)), n


def test_nonfinite_and_bad_eps_flags():
    import torch

    import paper_2501_14577_b200 as onedf
    kw = EDGE["tiny"]
    p = onedf.make_problem(**kw)
    x = _rand_inputs(kw, seed=3)
    x["K"][0, 0, 17, 1] = np.nan
    dev = torch.device("cuda:0")
    ws = onedf.Workspace(dev)
    Q = torch.from_numpy(x["Q"]).to(dev)
    K = torch.from_numpy(x["K"]).to(dev)
    onedf.encode(p, Q, K, ws=ws)
    ptr, _ = ws.get(0)
    assert onedf.check_device_status(ptr) == onedf.abi.ERR_NONFINITE
    K = torch.from_numpy(np.nan_to_num(x["K"])).to(dev)
    qc, kc, _ = onedf.encode(p, Q, K, ws=ws)
    assert onedf.check_device_status(ptr) == onedf.OK
    sc, pm = onedf.sort(p, kc, ws=ws)
    V = torch.from_numpy(x["V"]).to(dev)
    onedf.topk_attn_fwd(p, Q, K, V, torch.tensor(0.0, device=dev), qc, sc, pm, ws=ws)
    ptr, _ = ws.get(0)        # the fwd call may have grown (re-allocated) the workspace
    assert onedf.check_device_status(ptr) == onedf.abi.ERR_NONFINITE
    onedf.topk_attn_fwd(p, Q, K, V, torch.tensor(float("nan"), device=dev), qc, sc, pm, ws=ws)
    assert onedf.check_device_status(ptr) == onedf.abi.ERR_NONFINITE
    onedf.topk_attn_fwd(p, Q, K, V, torch.tensor(0.5, device=dev), qc, sc, pm, ws=ws)
    assert onedf.check_device_status(ptr) == onedf.OK


def test_autograd_function_and_host_step():
    import torch

    import paper_2501_14577_b200 as onedf
    cfg = synth.CONFIGS["tiny"]
    kw = cfg.problem_kwargs()
    x = synth.make_inputs(cfg)
    ref = oracle_run(kw, x)
    dev = torch.device("cuda:0")
    p = onedf.make_problem(**kw)
    Q, K, V = (torch.from_numpy(x[n]).to(dev).requires_grad_() for n in ("Q", "K", "V"))
    eps = torch.tensor(synth.EPS, device=dev, requires_grad=True)
    O, idx = onedf.zeta_attention(Q, K, V, eps, p)
    O.backward(torch.from_numpy(x["dO"]).to(dev))
    assert_close(O.detach().cpu().numpy(), ref["O"], "O")
    assert_close(Q.grad.cpu().numpy(), ref["dQ"], "dQ")
    assert_close(K.grad.cpu().numpy(), ref["dK"], "dK")
    assert_close(V.grad.cpu().numpy(), ref["dV"], "dV")
    assert_close(float(eps.grad), ref["d_eps"], "d_eps", rtol=1e-5, atol=1e-5)
    # end-to-end host-buffer entry point
    hs = onedf.HostStep(p, dev)
    pin = {n: torch.from_numpy(v).pin_memory() for n, v in x.items()}
    outs = {n: torch.empty_like(pin["V" if n in ("O", "dV") else "Q"]).pin_memory() for n in ("O", "dQ", "dK", "dV")}
    d_eps = torch.zeros((), dtype=torch.float64).pin_memory()
    hs(pin["Q"], pin["K"], pin["V"], synth.EPS, pin["dO"], outs["O"], outs["dQ"], outs["dK"], outs["dV"], d_eps)
    torch.cuda.synchronize()
    for n in ("O", "dQ", "dK", "dV"):
        assert_close(outs[n].numpy(), ref[n], f"host {n}")
    assert_close(float(d_eps), ref["d_eps"], "host d_eps")


@pytest.mark.parametrize("name", ["ar_tokens", "lra_nc"])
def test_schedule_hints_do_not_change_results(name):
    """qcode/qorder/perm only pick the visiting order of the forward and backward (any per-chunk
    permutation, e.g. the natural order): outputs are bitwise identical."""
    import torch

    import paper_2501_14577_b200 as onedf
    cfg = synth.CONFIGS[name]
    cfg = cfg.with_(B=1, H=2) if cfg.BH > 2 else cfg
    kw = cfg.problem_kwargs()
    x = synth.make_inputs(cfg)
    dev = torch.device("cuda:0")
    t = {n: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for n, v in x.items()}
    p = onedf.make_problem(**kw)
    e = torch.tensor(synth.EPS, dtype=torch.float32, device=dev)
    ws = onedf.Workspace(dev)
    qc, kc, _ = onedf.encode(p, t["Q"], t["K"], ws=ws)
    sc, pm = onedf.sort(p, kc, ws=ws)
    O, idx, Z = onedf.topk_attn_fwd(p, t["Q"], t["K"], t["V"], e, qc, sc, pm, ws=ws)
    # the forward with the caller's schedule (onedf_sort of qcode) or the natural order: same bits
    qo = onedf.query_schedule(p, qc, ws=ws)
    fwd_a = [v.cpu().numpy().copy() for v in (O, idx, Z)]
    nat = torch.arange(p.N, dtype=torch.int32, device=dev).expand(p.B, p.H, p.N).contiguous()
    for hint in (qo, nat):
        fwd_b = [v.cpu().numpy() for v in onedf.topk_attn_fwd(p, t["Q"], t["K"], t["V"], e, qc, sc, pm, ws=ws,
                                                              qorder=hint)]
        for u, v, n in zip(fwd_a, fwd_b, ("O", "idx", "Z")):
            assert np.array_equal(u.view(np.uint8), v.view(np.uint8)), n
    a = onedf.topk_attn_bwd(p, t["Q"], t["K"], t["V"], e, O, t["dO"], idx, Z, ws=ws, qcode=qc, perm=pm)
    a = [v.cpu().numpy().copy() for v in a]
    # the forward's in-degree counts (A9): the exact per-key count of idx entries, and a backward
    # that takes them instead of counting gives the same bits
    indeg = torch.full((p.B, p.H, p.N), -7, dtype=torch.int32, device=dev)
    means = torch.full((onedf.means_floats(p),), float("nan"), device=dev)
    fwd_c = [v.cpu().numpy() for v in onedf.topk_attn_fwd(p, t["Q"], t["K"], t["V"], e, qc, sc, pm, ws=ws,
                                                          qorder=qo, indeg=indeg, means=means)]
    for u, v, n in zip(fwd_a, fwd_c, ("O", "idx", "Z")):
        assert np.array_equal(u.view(np.uint8), v.view(np.uint8)), n
    ix = fwd_a[1].reshape(p.B * p.H, p.N, p.k)
    want = np.stack([np.bincount(r[r >= 0].ravel(), minlength=p.N) for r in ix]).reshape(p.B, p.H, p.N)
    assert_same(indeg.cpu().numpy(), want.astype(np.int32), "indeg")
    for hints in ({}, {"qorder": qo, "perm": pm}, {"qorder": nat}, {"qorder": qo, "perm": pm, "indeg": indeg},
                  {"qorder": qo, "perm": pm, "indeg": indeg, "means": means}, {"means": means}):
        b = onedf.topk_attn_bwd(p, t["Q"], t["K"], t["V"], e, O, t["dO"], idx, Z, ws=ws, **hints)
        b = [v.cpu().numpy() for v in b]
        for u, v, n in zip(a, b, ("dQ", "dK", "dV", "d_eps")):
            assert np.array_equal(np.atleast_1d(u).view(np.uint8), np.atleast_1d(v).view(np.uint8)), (n, list(hints))


def test_host_step_pipelined_groups_match_device_path():
    """onedf_topk_attn_step_host pipelines groups of (b,h) slices over three streams; every
    slice's outputs are the device path's bit for bit (slices are independent), d_eps is the
    groups' partial sums added in order (within tolerance of the single-call reduction)."""
    import torch

    import paper_2501_14577_b200 as onedf
    kw = dict(B=2, H=5, N=1024, d_k=3, d_v=32, k=16, window=32, chunk=128, causal=1, mean_slot=1)
    rng = np.random.default_rng(8)
    x = {n: rng.normal(size=(2, 5, 1024, w)).astype(np.float32) for n, w in (("Q", 3), ("K", 3), ("V", 32),
                                                                               ("dO", 32))}
    ref = gpu_run(kw, x)
    p = onedf.make_problem(**kw)
    hs = onedf.HostStep(p, torch.device("cuda:0"))
    pin = {n: torch.from_numpy(v).pin_memory() for n, v in x.items()}
    outs = {n: torch.empty_like(pin["V" if n in ("O", "dV") else "Q"]).pin_memory() for n in ("O", "dQ", "dK", "dV")}
    d_eps = torch.zeros((), dtype=torch.float64).pin_memory()
    for _ in range(2):                                   # the second call reuses the workspace
        hs(pin["Q"], pin["K"], pin["V"], synth.EPS, pin["dO"], outs["O"], outs["dQ"], outs["dK"], outs["dV"], d_eps)
        torch.cuda.synchronize()
        for n in ("O", "dQ", "dK", "dV"):
            assert np.array_equal(outs[n].numpy(), ref[n]), n
        assert float(d_eps) == pytest.approx(float(ref["d_eps"]), rel=1e-12)


@pytest.mark.parametrize("N,d_k,tokens", [(1 << 20, 3, False), (200_003, 2, False), (50_000, 3, True),
                                          (8193, 1, False)])
def test_onesweep_long_run_sort(N, d_k, tokens):
    """Runs longer than onedf_max_run_length() go through the multi-CTA onesweep radix sort
    (decoupled look-back): a single non-causal run of up to 1M keys, ragged tile counts, heavy
    code ties (repeated tokens) and a one-key-past-the-limit run -- scode and perm bit-exact
    against the oracle's std::sort on (code, position), for the key codes and the query schedule."""
    import torch

    import paper_2501_14577_b200 as onedf
    kw = dict(B=1, H=1, N=N, d_k=d_k, d_v=4, k=4, window=8, chunk=1, causal=0, mean_slot=0)
    rng = np.random.default_rng(N)
    Q = rng.normal(size=(1, 1, N, d_k)).astype(np.float32)
    K = rng.normal(size=(1, 1, N, d_k)).astype(np.float32)
    if tokens:
        vocab = rng.normal(size=(97, d_k)).astype(np.float32)
        K = vocab[rng.integers(0, 97, size=(1, 1, N))]
    p = oracle.Problem(**kw)
    qc, kc, _ = oracle.encode(p, Q, K)
    sc_ref, pm_ref = oracle.sort(p, kc)
    _, qo_ref = oracle.sort(p, qc)
    dev = torch.device("cuda:0")
    pg = onedf.make_problem(**kw)
    ws = onedf.Workspace(dev)
    kc_t = torch.from_numpy(kc.view(np.int64)).to(dev)
    sc, pm = onedf.sort(pg, kc_t, ws=ws)
    qo = onedf.query_schedule(pg, torch.from_numpy(qc.view(np.int64)).to(dev), ws=ws)
    torch.cuda.synchronize()
    assert_same(sc.cpu().numpy().view(np.uint64), sc_ref, "scode")
    assert_same(pm.cpu().numpy(), pm_ref, "perm")
    assert_same(qo.cpu().numpy(), qo_ref, "qorder")
