"""GPU parity of the score variants (reading D24): the same
Euclidean top-k set, weights exp(-D), 1/(sqrt D + 1e-6) or exp(q.k/sqrt d_k)
instead of Cauchy's 1/(D + eps).  CUDA path (C ABI) vs the CPU oracle on the
same seeded inputs: idx bit-exact, O, Z (sum or log-sum-exp), dQ, dK, dV
within 1e-5 rel / 1e-6 abs, d_eps == 0."""
import zlib

import numpy as np
import pytest

import synth
from _util import assert_close, assert_same, gpu_run, oracle_run

pytestmark = pytest.mark.gpu

SCORES = {1: "neg_euclid", 2: "inv_euclid", 3: "dot"}


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__
    __graft_entry__.build()


def _inputs(kw, seed, dup_keys=False):
    rng = np.random.default_rng(seed)
    B, H, N, dk, dv = kw["B"], kw["H"], kw["N"], kw["d_k"], kw["d_v"]
    x = dict(Q=rng.normal(size=(B, H, N, dk)).astype(np.float32),
             K=rng.normal(size=(B, H, N, dk)).astype(np.float32),
             V=rng.normal(size=(B, H, N, dv)).astype(np.float32),
             dO=rng.normal(size=(B, H, N, dv)).astype(np.float32))
    if dup_keys:   # identical key rows: exercises q == k (D = 0) for the inverse-Euclidean score
        vocab = rng.normal(size=(7, dk)).astype(np.float32)
        tok = rng.integers(0, 7, size=(B, H, N))
        x["K"] = vocab[tok]
        x["Q"] = np.where(rng.random(size=(B, H, N, 1)) < 0.3, vocab[tok],
                          vocab[tok] + 0.05 * rng.normal(size=(B, H, N, dk))).astype(np.float32)
    return x


def _compare(got, ref):
    assert_same(got["idx"], ref["idx"], "idx")
    for n in ("O", "Z", "dQ", "dK", "dV"):
        assert_close(got[n], ref[n], n)
    assert float(got["d_eps"]) == 0.0 and ref["d_eps"] == 0.0


CASES = {
    "ragged_causal": dict(B=2, H=1, N=300, d_k=3, d_v=16, k=8, window=16, chunk=64, causal=1, mean_slot=1),
    "noncausal": dict(B=1, H=2, N=200, d_k=3, d_v=16, k=8, window=32, chunk=1, causal=0, mean_slot=1),
    "no_mean_slot": dict(B=1, H=2, N=256, d_k=2, d_v=8, k=8, window=16, chunk=32, causal=1, mean_slot=0),
    "dk1": dict(B=1, H=2, N=256, d_k=1, d_v=8, k=5, window=10, chunk=32, causal=1, mean_slot=1),
    "dk4_dv64_k64": dict(B=1, H=2, N=2048, d_k=4, d_v=64, k=64, window=128, chunk=256, causal=1, mean_slot=1),
    "dv256": dict(B=1, H=1, N=256, d_k=3, d_v=256, k=16, window=32, chunk=32, causal=1, mean_slot=1),
    "k100": dict(B=1, H=1, N=1024, d_k=3, d_v=8, k=100, window=150, chunk=256, causal=1, mean_slot=1),
}


@pytest.mark.parametrize("score", list(SCORES))
@pytest.mark.parametrize("name", list(CASES))
def test_score_variant_full_parity(score, name):
    kw = dict(CASES[name], score=score)
    x = _inputs(kw, seed=zlib.crc32(f"{name}{score}".encode()) % 1000)
    _compare(gpu_run(kw, x), oracle_run(kw, x))


@pytest.mark.parametrize("score", list(SCORES))
def test_score_variant_duplicate_keys(score):
    kw = dict(B=1, H=2, N=512, d_k=3, d_v=16, k=16, window=32, chunk=64, causal=1, mean_slot=1, score=score)
    x = _inputs(kw, seed=71, dup_keys=True)
    _compare(gpu_run(kw, x), oracle_run(kw, x))


@pytest.mark.parametrize("score", list(SCORES))
def test_score_variant_ar_shape_slices(score):
    """The Associative-Recall shape (N = 2K, d_k = 3, d_v = 64, k = 32, 8 chunks), tokens inputs,
    two (b,h) slices through the whole path."""
    cfg = synth.CONFIGS["ar_tokens"]
    kw = dict(cfg.problem_kwargs(), score=score)
    x = synth.make_inputs(cfg, bh_range=range(2))
    kw.update(B=1, H=2)
    _compare(gpu_run(kw, x), oracle_run(kw, x))


@pytest.mark.parametrize("score", [1, 3])
def test_score_variant_sequence_sharded(score):
    """Score variants compose with sequence sharding (NEXT-1): owned rows equal the oracle."""
    from test_gpu_seqshard import sharded_run
    kw = dict(B=1, H=2, N=1500, d_k=3, d_v=16, k=16, window=32, chunk=128, causal=1, mean_slot=1, score=score)
    x = _inputs(kw, seed=90 + score)
    got, ref = sharded_run(kw, x, 3), oracle_run(kw, x)
    assert_same(got["idx"], ref["idx"], "idx")
    for n in ("O", "Z", "dQ", "dK", "dV"):
        assert_close(got[n], ref[n], n)


# ---------------------------------------------------------------- selection variant: SPEC's code-distance merge (D25)
SEL_CASES = {
    "spec_w_eq_k": dict(B=1, H=2, N=1024, d_k=3, d_v=16, k=16, window=16, chunk=128, causal=1, mean_slot=1),
    "wide_window": dict(B=2, H=1, N=600, d_k=2, d_v=8, k=8, window=40, chunk=64, causal=1, mean_slot=1),
    "noncausal": dict(B=1, H=2, N=300, d_k=3, d_v=8, k=12, window=24, chunk=1, causal=0, mean_slot=0),
    "k64_many_runs": dict(B=1, H=1, N=4096, d_k=3, d_v=64, k=64, window=64, chunk=128, causal=1, mean_slot=1),
    "dk1": dict(B=1, H=1, N=512, d_k=1, d_v=8, k=8, window=8, chunk=32, causal=1, mean_slot=1),
}


@pytest.mark.parametrize("name", list(SEL_CASES))
def test_code_distance_selection_parity(name):
    kw = dict(SEL_CASES[name], select=1)
    x = _inputs(kw, seed=zlib.crc32(name.encode()) % 1000)
    got, ref = gpu_run(kw, x), oracle_run(kw, x)
    assert_same(got["idx"], ref["idx"], "idx")
    for n in ("O", "Z", "dQ", "dK", "dV", "d_eps"):
        assert_close(got[n], ref[n], n)


@pytest.mark.parametrize("score", [0, 1])
def test_code_distance_selection_repeated_codes(score):
    """Repeated codes (3 bits per dim, few distinct rows) put many candidates at the same code
    distance: the fallback ordering must still give the oracle's (distance, j) order."""
    kw = dict(B=1, H=2, N=512, d_k=3, d_v=16, k=16, window=48, chunk=64, bits=3, causal=1, mean_slot=1,
              score=score, select=1)
    x = _inputs(kw, seed=17, dup_keys=True)
    got, ref = gpu_run(kw, x), oracle_run(kw, x)
    assert_same(got["idx"], ref["idx"], "idx")
    for n in ("O", "dQ", "dK", "dV"):
        assert_close(got[n], ref[n], n)
