"""Kernel-level view of one sharded step (for ncu launch lists): N = 1M, one (b,h), either unsharded
(--world 1) or all `world` ranks simulated in one process (seqshard.run_sim).

    ncu --metrics gpu__time_duration.sum --csv --log-file L.csv python tools/seqshard_profile.py --world 8
    python tools/ncu_step.py L.csv      # per-kernel totals (divide by world for the mean rank)
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2501_14577_b200 as onedf  # noqa: E402
from paper_2501_14577_b200 import seqshard  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--N", type=int, default=1 << 20)
a = ap.parse_args()
N = a.N
kw = dict(B=1, H=1, N=N, d_k=3, d_v=64, k=64, window=128, chunk=N // 32, causal=1, mean_slot=1)
g = torch.Generator(device="cpu").manual_seed(11)
x = {n: torch.randn(1, 1, N, w, generator=g).cuda() for n, w in (("Q", 3), ("K", 3), ("V", 64), ("dO", 64))}
dev = x["Q"].device
eps = torch.tensor(0.5, device=dev)
if a.world == 1:
    p = onedf.make_problem(**kw)
    ws = onedf.Workspace(dev)
    qc, kc, _ = onedf.encode(p, x["Q"], x["K"], ws=ws)
    sc, pm = onedf.sort(p, kc, ws=ws)
    qo = onedf.query_schedule(p, qc, ws=ws)
    O, idx, Z = onedf.topk_attn_fwd(p, x["Q"], x["K"], x["V"], eps, qc, sc, pm, ws=ws, qorder=qo)
    onedf.topk_attn_bwd(p, x["Q"], x["K"], x["V"], eps, O, x["dO"], idx, Z, ws=ws, qorder=qo, perm=pm)
else:
    plan = seqshard.ShardPlan(N=N, M=kw["chunk"], world=a.world)
    gens = []
    for r in range(a.world):
        p = onedf.make_problem(**kw, shard_rank=r, shard_world=a.world)
        m = plan.owned_mask(r, dev)
        mine = {n: torch.where(m[None, None, :, None], v, torch.zeros((), device=dev)).contiguous()
                for n, v in x.items()}
        gens.append(seqshard.step(p, mine["Q"], mine["K"], mine["V"], eps, mine["dO"], ws=onedf.Workspace(dev)))
    seqshard.run_sim(gens, plan)
torch.cuda.synchronize()
print("done world", a.world)
