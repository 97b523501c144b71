"""One encode -> sort (keys + query schedule) -> fwd -> bwd pass of a config on cuda:0, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck); not a bench.

    compute-sanitizer --tool racecheck python tools/sanitize_step.py --config ar --bh 2 [--vdtype 1]
Inputs come from synth/ (the seeded recipe of the tests), reduced to the first `bh` (b,h) slices.
"""
from __future__ import annotations

import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2501_14577_b200 as onedf  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tiny")
    ap.add_argument("--bh", type=int, default=1)
    ap.add_argument("--vdtype", type=int, default=0)
    ap.add_argument("--score", type=int, default=0)
    ap.add_argument("--select", type=int, default=0)
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    bh = min(a.bh, cfg.BH)
    x = synth.make_inputs(cfg, bh_range=range(bh))
    kw = dict(cfg.problem_kwargs(), B=1, H=bh, vdtype=a.vdtype, score=a.score, select=a.select)
    p = onedf.make_problem(**kw)
    dev = torch.device("cuda:0")
    t = {n: torch.from_numpy(v).to(dev) for n, v in x.items()}
    for n in ("V", "dO"):
        t[n] = t[n].to(onedf.value_dtype(p))
    eps = torch.tensor(synth.EPS, device=dev)
    ws = onedf.Workspace(dev)
    qc, kc, _ = onedf.encode(p, t["Q"], t["K"], ws=ws)
    sc, pm = onedf.sort(p, kc, ws=ws)
    qo = onedf.query_schedule(p, qc, ws=ws)
    O, idx, Z = onedf.topk_attn_fwd(p, t["Q"], t["K"], t["V"], eps, qc, sc, pm, ws=ws, qorder=qo)
    onedf.topk_attn_bwd(p, t["Q"], t["K"], t["V"], eps, O, t["dO"], idx, Z, ws=ws, qorder=qo, perm=pm)
    torch.cuda.synchronize()
    assert onedf.check_device_status(ws) == onedf.OK
    print("done", a.config, "bh", bh, "vdtype", a.vdtype, "score", a.score, "select", a.select)


if __name__ == "__main__":
    main()
