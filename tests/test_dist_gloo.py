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
