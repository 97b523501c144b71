"""One encode+sort+fwd+bwd step of a config on cuda:0 (for ncu captures; not a bench).

    ncu ... python tools/prof_step.py --config long64k --steps 1
Inputs are iid N(0,1) generated on the device (timing-free), so the capture
starts quickly; bench.py is the measured path.
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
    ap.add_argument("--config", default="long64k")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--fwd-only", action="store_true")
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    p = onedf.make_problem(**cfg.problem_kwargs())
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(1)
    shp = (p.B, p.H, p.N)
    Q = torch.randn(*shp, p.d_k, device=dev, generator=g)
    K = torch.randn(*shp, p.d_k, device=dev, generator=g)
    V = torch.randn(*shp, p.d_v, device=dev, generator=g)
    dO = torch.randn(*shp, p.d_v, device=dev, generator=g)
    eps = torch.tensor(0.5, device=dev)
    ws = onedf.Workspace(dev)
    indeg = torch.empty(shp, dtype=torch.int32, device=dev)     # the forward's A9 counts, as in bench.py
    means = torch.empty(onedf.means_floats(p), device=dev)      # and its prefix means
    for _ in range(a.steps):            # the launches of bench.py's step
        qc, kc, _ = onedf.encode(p, Q, K, ws=ws)
        sc, pm = onedf.sort(p, kc, ws=ws)
        qo = onedf.query_schedule(p, qc, ws=ws)
        O, idx, Z = onedf.topk_attn_fwd(p, Q, K, V, eps, qc, sc, pm, ws=ws, qorder=qo, indeg=indeg, means=means)
        if not a.fwd_only:
            onedf.topk_attn_bwd(p, Q, K, V, eps, O, dO, idx, Z, ws=ws, qorder=qo, perm=pm, indeg=indeg, means=means)
    torch.cuda.synchronize()
    print("done", a.config)


if __name__ == "__main__":
    main()
