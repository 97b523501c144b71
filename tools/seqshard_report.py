"""NEXT-1 measurement on one GPU: sequence sharding of long sequences over P simulated ranks.

All ranks run in one process (seqshard.run_sim); each rank's own compute between the
collectives is timed with CUDA events, so the report gives, per world size P,
  * max_rank_ms  -- the slowest rank's device time (what a P-GPU step waits for, minus comm),
  * balance      -- mean / max over ranks (the zig-zag chunk deal's load balance),
  * speedup      -- the unsharded single-GPU time / max_rank_ms,
  * exchange     -- bytes one rank sends per step, and that at 900 GB/s (NVLink 5 per direction).
    python tools/seqshard_report.py > gpurun_out/seqshard.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2501_14577_b200 as onedf  # noqa: E402
from paper_2501_14577_b200 import seqshard  # noqa: E402


def unsharded_ms(kw, x, reps=2):
    p = onedf.make_problem(**kw)
    ws = onedf.Workspace(x["Q"].device)
    eps = torch.tensor(0.5, device=x["Q"].device)
    best = None
    for _ in range(reps + 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        qc, kc, _ = onedf.encode(p, x["Q"], x["K"], ws=ws)
        sc, pm = onedf.sort(p, kc, ws=ws)
        O, idx, Z = onedf.topk_attn_fwd(p, x["Q"], x["K"], x["V"], eps, qc, sc, pm, ws=ws)
        onedf.topk_attn_bwd(p, x["Q"], x["K"], x["V"], eps, O, x["dO"], idx, Z, ws=ws, qcode=qc, perm=pm)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best


def sharded(kw, x, world, reps=2):
    dev = x["Q"].device
    plan = seqshard.ShardPlan(N=kw["N"], M=kw["chunk"], world=world)
    eps = torch.tensor(0.5, device=dev)
    best = None
    for _ in range(reps + 1):
        gens = []
        for r in range(world):
            p = onedf.make_problem(**kw, shard_rank=r, shard_world=world)
            m = plan.owned_mask(r, dev)
            mine = {n: torch.where(m[None, None, :, None], v, torch.zeros((), device=dev)).contiguous()
                    for n, v in x.items()}
            gens.append(seqshard.step(p, mine["Q"], mine["K"], mine["V"], eps, mine["dO"], ws=onedf.Workspace(dev)))
        timing = []
        seqshard.run_sim(gens, plan, timing=timing)
        if best is None or max(timing) < max(best):
            best = timing
    p0 = onedf.make_problem(**kw, shard_rank=0, shard_world=world)
    return best, seqshard.exchange_bytes(p0, plan)


def main():
    rows = []
    for N, BH in ((262144, 2), (1048576, 1)):
        kw = dict(B=1, H=BH, N=N, d_k=3, d_v=64, k=64, window=128, chunk=N // 32, causal=1, mean_slot=1)
        g = torch.Generator(device="cpu").manual_seed(11)
        x = {n: torch.randn(1, BH, N, w, generator=g).cuda() for n, w in (("Q", 3), ("K", 3), ("V", 64), ("dO", 64))}
        base = unsharded_ms(kw, x)
        for world in (1, 2, 4, 8):
            t, xb = sharded(kw, x, world)
            rows.append(dict(N=N, BH=BH, world=world, unsharded_ms=base, rank_ms=t, max_rank_ms=max(t),
                             balance=sum(t) / len(t) / max(t), speedup=base / max(t),
                             exchange_bytes_per_rank=xb, exchange_ms_at_900GBs=xb["total"] / 900e9 * 1e3))
            print(json.dumps(rows[-1]), file=sys.stderr)
    print(json.dumps({"device": torch.cuda.get_device_name(0), "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
