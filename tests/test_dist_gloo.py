"""world_size-2 gloo tests of the multi-GPU host logic on CPU: the (b,h)
partition covers every slice exactly once, and the d_eps exchange (all-gather
+ rank-ordered sum) gives every rank the same bits, equal to the oracle's
d_eps over the whole batch (per-rank values come from the oracle on that
rank's slices -- the CUDA path is not involved)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2501_14577_b200 import dist as odist


def test_partition_covers_once():
    for total in (1, 5, 96, 97, 256):
        for world in (1, 2, 3, 4, 8):
            got = [list(odist.partition(total, world, r)) for r in range(world)]
            flat = [x for g in got for x in g]
            assert flat == list(range(total))
            sizes = [len(g) for g in got]
            assert max(sizes) - min(sizes) <= 1
    assert list(odist.weak_slices(12, 3)) == list(range(36, 48))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import oracle
    import synth
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.CONFIGS["tiny"].with_(B=1, H=4)
    mine = odist.partition(cfg.BH, world, rank)
    x = synth.make_inputs(cfg, bh_range=mine)
    p = oracle.Problem(**dict(cfg.problem_kwargs(), B=1, H=len(mine)))
    res = oracle.pipeline(p, x["Q"], x["K"], x["V"], synth.EPS, x["dO"])
    d = torch.tensor(res["d_eps"], dtype=torch.float64)
    odist.combine_d_eps(d)
    out[rank] = d.item()
    torch.distributed.barrier()
    torch.distributed.destroy_process_group()


def test_d_eps_exchange_two_ranks():
    import oracle
    import synth
    oracle.build()
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert out[0] == out[1]                          # identical bits on every rank
    cfg = synth.CONFIGS["tiny"].with_(B=1, H=4)
    x = synth.make_inputs(cfg, bh_range=range(4))
    p = oracle.Problem(**dict(cfg.problem_kwargs(), B=1, H=4))
    full = oracle.pipeline(p, x["Q"], x["K"], x["V"], synth.EPS, x["dO"])["d_eps"]
    assert out[0] == pytest.approx(full, rel=1e-13)
    # and the per-rank slices concatenate to the whole batch (independent slices)
    parts = []
    for r in range(world):
        rr = odist.partition(4, world, r)
        xs = synth.make_inputs(cfg, bh_range=rr)
        ps = oracle.Problem(**dict(cfg.problem_kwargs(), B=1, H=len(rr)))
        parts.append(oracle.pipeline(ps, xs["Q"], xs["K"], xs["V"], synth.EPS, xs["dO"])["O"])
    np.testing.assert_array_equal(np.concatenate(parts, axis=1), full_O(cfg))


def full_O(cfg):
    import oracle
    import synth
    x = synth.make_inputs(cfg, bh_range=range(cfg.BH))
    p = oracle.Problem(**dict(cfg.problem_kwargs(), B=1, H=cfg.BH))
    return oracle.pipeline(p, x["Q"], x["K"], x["V"], synth.EPS)["O"]


# ---------------------------------------------------------------- sequence sharding (NEXT-1) plumbing
def _seq_worker(rank, world, port, out):
    """Drive seqshard.run_dist over gloo with a scripted generator: the collectives'
    data movement (bounds MIN/MAX, row all-gather, partial-row all-to-all + rank-ordered
    combine, scalar sum) on CPU tensors.  The combine is injected (the product's is the
    CUDA onedf_rank_sum); it sums in rank order in f64 like the kernel."""
    from paper_2501_14577_b200 import seqshard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    N, M, B, H = 45, 4, 2, 3
    plan = seqshard.ShardPlan(N=N, M=M, world=world)
    g = torch.Generator().manual_seed(7)
    full = torch.randn(B, H, N, 5, generator=g)            # the "true" rows, known to the test only
    mine = plan.owned_mask(rank)
    x = torch.where(mine[None, None, :, None], full, torch.zeros(()))
    part = torch.randn(world, B, H, N, 5, generator=g)     # every rank's partial of every row

    def combine(parts):
        acc = parts[0].double()
        for q in parts[1:]:
            acc = acc + q.double()
        return acc.float()

    def gen():
        lohi = torch.stack([full[:, :, mine].amin(2), full[:, :, mine].amax(2)], dim=-2)
        red = yield ("allreduce_minmax", lohi)
        yield ("gather_rows", [x])
        y = part[rank].clone()
        yield ("reduce_rows", [y])
        s = yield ("sum_scalar", torch.tensor(float(rank + 1), dtype=torch.float64))
        return red, x, y, s

    red, xg, y, s = seqshard.run_dist(gen(), plan, combine=combine)
    out[rank] = (red, xg, y[:, :, mine], s.item(), mine)
    torch.distributed.barrier()
    torch.distributed.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_seqshard_collectives(world):
    from paper_2501_14577_b200 import seqshard  # noqa: F401  (loads libonedf.so for the owner map)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_seq_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    N, B, H = 45, 2, 3
    g = torch.Generator().manual_seed(7)
    full = torch.randn(B, H, N, 5, generator=g)
    part = torch.randn(world, B, H, N, 5, generator=g)
    want_sum = part[0].double()
    for q in part[1:]:
        want_sum = want_sum + q.double()
    for r in range(world):
        red, xg, y, s, mine = out[r]
        torch.testing.assert_close(red, torch.stack([full.amin(2), full.amax(2)], dim=-2), rtol=0, atol=0)
        torch.testing.assert_close(xg, full, rtol=0, atol=0)                     # every row complete
        torch.testing.assert_close(y, want_sum.float()[:, :, mine], rtol=0, atol=0)  # owner rows summed
        assert s == sum(range(1, world + 1))


# ---------------------------------------------------------------- bench harness (strong scaling, max over ranks)
def _bench_worker(rank, world, port, out):
    import bench
    import synth
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.CONFIGS["long64k"]
    got = {}
    for scaling in ("strong", "weak"):
        bhs, shape = bench.rank_slices(cfg, world, rank, scaling)
        got[scaling] = (list(bhs), shape, bench.units_per_step(cfg, world, scaling))
    # each rank "times" a different value; every rank must get the max (t_P)
    got["tmax"] = bench.max_over_ranks(10.0 + 3.0 * rank)
    out[rank] = got
    torch.distributed.barrier()
    torch.distributed.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_bench_rank_partition_and_timing_reduction(world):
    import synth
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_bench_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    cfg = synth.CONFIGS["long64k"]
    strong = [out[r]["strong"] for r in range(world)]
    assert [x for s in strong for x in s[0]] == list(range(cfg.BH))     # contiguous, each slice once
    assert all(s[1] == (1, len(s[0])) for s in strong)
    assert all(s[2] == cfg.BH * cfg.N for s in strong)                  # strong: total work fixed
    weak = [out[r]["weak"] for r in range(world)]
    assert sorted(x for w in weak for x in w[0]) == list(range(world * cfg.BH))
    assert all(w[1] == (cfg.B, cfg.H) and w[2] == world * cfg.BH * cfg.N for w in weak)
    assert all(out[r]["tmax"] == 10.0 + 3.0 * (world - 1) for r in range(world))


def test_bench_self_launches_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks (torch.distributed.run on
    127.0.0.1); the reference arm prints one JSON line from rank 0 only."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--config", "tiny", "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                       env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["cpu_baseline"]["nproc"] >= 1
