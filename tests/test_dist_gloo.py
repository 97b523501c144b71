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
