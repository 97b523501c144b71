"""GPU parity of sequence sharding.

All ranks run in one process on cuda:0 (seqshard.run_sim: the collectives are
copies; a test box has one GPU), each with its own shard_rank.  The assembled
owned rows must equal the unsharded CUDA path -- bitwise for codes, runs,
idx, O, Z and dQ (each owned query runs the same kernels on the same complete
runs and rows) -- and the CPU oracle within the north_star tolerance; dK, dV
and d_eps are sums of per-rank partials (onedf_rank_sum, f64 in rank order),
so they match within the tolerance.
"""
import zlib

import numpy as np
import pytest
import torch

from _util import assert_close, assert_same, gpu_run, oracle_run

pytestmark = pytest.mark.gpu


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
    if dup_keys:
        vocab = rng.normal(size=(9, dk)).astype(np.float32)
        tok = rng.integers(0, 9, size=(B, H, N))
        x["K"] = vocab[tok]
        x["Q"] = (vocab[tok] + 0.05 * rng.normal(size=(B, H, N, dk))).astype(np.float32)
    return x


def sharded_run(kw, x, world, eps=0.5):
    import paper_2501_14577_b200 as onedf
    from paper_2501_14577_b200 import seqshard
    dev = torch.device("cuda:0")
    plan = seqshard.ShardPlan(N=kw["N"], M=kw["chunk"], world=world)
    full = {n: torch.from_numpy(v).to(dev) for n, v in x.items()}
    e = torch.tensor(eps, dtype=torch.float32, device=dev)
    gens, masks = [], []
    for r in range(world):
        p = onedf.make_problem(**kw, shard_rank=r, shard_world=world)
        m = plan.owned_mask(r, dev)
        mine = {n: torch.where(m[None, None, :, None], v, torch.zeros((), device=dev)).contiguous()
                for n, v in full.items()}
        # non-owned K/V rows hold junk until the gather fills them (they must not matter)
        mine["K"][:, :, ~m] = 1e30
        mine["V"][:, :, ~m] = -7.0
        masks.append(m.cpu().numpy())
        gens.append(seqshard.step(p, mine["Q"], mine["K"], mine["V"], e, mine["dO"], ws=onedf.Workspace(dev)))
    res = seqshard.run_sim(gens, plan)
    torch.cuda.synchronize()
    out = {}
    for name in ("O", "idx", "Z", "dQ", "dK", "dV", "qcode", "kcode_unused", "scode", "perm"):
        if name not in res[0]:
            continue
        a = np.zeros_like(res[0][name].cpu().numpy())
        for r in range(world):
            a[:, :, masks[r]] = res[r][name].cpu().numpy()[:, :, masks[r]]
        out[name] = a
    for n in ("qcode", "scode"):
        out[n] = out[n].view(np.uint64)
    out["d_eps"] = [float(res[r]["d_eps"]) for r in range(world)]
    out["lohi"] = [res[r]["lohi"].cpu().numpy() for r in range(world)]
    out["full_runs"] = [(res[r]["scode"].cpu().numpy().view(np.uint64), res[r]["perm"].cpu().numpy())
                        for r in range(world)]
    return out


CASES = {
    "w2_ragged": (2, dict(B=1, H=2, N=2000, d_k=3, d_v=64, k=32, window=64, chunk=256, causal=1, mean_slot=1)),
    "w3_uneven": (3, dict(B=2, H=1, N=1500, d_k=3, d_v=16, k=16, window=32, chunk=128, causal=1, mean_slot=1)),
    "w4_k64": (4, dict(B=1, H=1, N=4096, d_k=3, d_v=64, k=64, window=128, chunk=256, causal=1, mean_slot=1)),
    "w5_one_chunk_each": (5, dict(B=1, H=2, N=600, d_k=2, d_v=8, k=8, window=16, chunk=128, causal=1, mean_slot=1)),
    "w4_idle_rank": (4, dict(B=1, H=1, N=300, d_k=3, d_v=8, k=8, window=16, chunk=128, causal=1, mean_slot=1)),
    "w2_no_mean": (2, dict(B=1, H=2, N=1000, d_k=4, d_v=16, k=8, window=16, chunk=100, causal=1, mean_slot=0)),
    "w8_dk1": (8, dict(B=1, H=1, N=2048, d_k=1, d_v=8, k=5, window=10, chunk=64, causal=1, mean_slot=1)),
}


@pytest.mark.parametrize("name", list(CASES))
def test_seq_sharded_matches_unsharded_and_oracle(name):
    world, kw = CASES[name]
    x = _inputs(kw, seed=zlib.crc32(name.encode()) % 1000)
    got = sharded_run(kw, x, world)
    ref = gpu_run(kw, x)
    orc = oracle_run(kw, x)
    for r in range(world):
        assert_same(got["lohi"][r], ref["lohi"], f"lohi rank {r}")          # exact MIN/MAX all-reduce
        assert_same(got["full_runs"][r][0], ref["scode"], f"scode rank {r}")  # complete runs on every rank
        assert_same(got["full_runs"][r][1], ref["perm"], f"perm rank {r}")
    for n in ("qcode", "idx", "O", "Z", "dQ"):
        assert_same(got[n], ref[n], n)
    assert_same(got["idx"], orc["idx"], "idx vs oracle")
    for n in ("O", "Z", "dQ", "dK", "dV"):
        assert_close(got[n], orc[n], n + " vs oracle")
    for n in ("dK", "dV"):
        assert_close(got[n], ref[n], n + " vs unsharded")
    assert len(set(got["d_eps"])) == 1                                      # same bits on every rank
    assert_close(got["d_eps"][0], orc["d_eps"], "d_eps")


def test_seq_sharded_duplicate_keys():
    world, kw = 3, dict(B=1, H=2, N=1200, d_k=3, d_v=16, k=16, window=32, chunk=100, causal=1, mean_slot=1)
    x = _inputs(kw, seed=5, dup_keys=True)
    got, orc = sharded_run(kw, x, world), oracle_run(kw, x)
    assert_same(got["idx"], orc["idx"], "idx")
    for n in ("O", "dQ", "dK", "dV"):
        assert_close(got[n], orc[n], n)
    assert_close(got["d_eps"][0], orc["d_eps"], "d_eps")


def test_bounds_partial_finish_equals_fit():
    """onedf_encode(lohi_in=NULL) == bounds_partial -> bounds_finish -> encode(lohi_in) (onedf.h)."""
    import paper_2501_14577_b200 as onedf
    kw = dict(B=2, H=3, N=777, d_k=3, d_v=8, k=8, window=16, chunk=64, causal=1, mean_slot=1)
    x = _inputs(kw, seed=3)
    x["Q"][0, 1, :, 2] = 0.25            # a constant dim in one (b,h): widened by +-0.5 (D10)
    x["K"][0, 1, :, 2] = 0.25
    dev = torch.device("cuda:0")
    p = onedf.make_problem(**kw)
    Q, K = (torch.from_numpy(x[n]).to(dev) for n in ("Q", "K"))
    qc, kc, lohi_fit = onedf.encode(p, Q, K)
    raw = onedf.bounds_partial(p, Q, K)
    assert torch.equal(raw[..., 0, :], torch.minimum(Q.double().amin(2), K.double().amin(2)))
    assert torch.equal(raw[..., 1, :], torch.maximum(Q.double().amax(2), K.double().amax(2)))
    fin = onedf.bounds_finish(p, raw.clone())
    assert torch.equal(fin, lohi_fit)
    qc2, kc2, _ = onedf.encode(p, Q, K, lohi=fin)
    assert torch.equal(qc, qc2) and torch.equal(kc, kc2)


def test_rank_sum_is_rank_ordered_f64():
    import paper_2501_14577_b200 as onedf
    g = torch.Generator().manual_seed(1)
    parts = (torch.randn(5, 3, 1001, generator=g) * torch.tensor([1e8, 1.0, 1e-8, -1e8, 3.0])[:, None, None])
    got = onedf.rank_sum(parts.cuda()).cpu()
    acc = parts[0].double()
    for q in parts[1:]:
        acc = acc + q.double()
    assert torch.equal(got, acc.float())


def test_seq_sharded_tiny_chunks():
    """Chunks shorter than the encoder's 4-row groups (M = 3): ownership changes inside a group."""
    world, kw = 3, dict(B=1, H=1, N=200, d_k=3, d_v=8, k=4, window=8, chunk=3, causal=1, mean_slot=1)
    x = _inputs(kw, seed=21)
    got, ref = sharded_run(kw, x, world), oracle_run(kw, x)
    assert_same(got["idx"], ref["idx"], "idx")
    for n in ("O", "dQ", "dK", "dV"):
        assert_close(got[n], ref[n], n)
