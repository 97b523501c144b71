"""Time A3's run sort (onedf_sort) with CUDA events: the on-chip path (runs <= onedf_max_run_length)
and the multi-CTA onesweep path (longer runs), on synthetic iid Gaussian codes.  Prints JSON lines.

    python tools/time_sort.py
"""
from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2501_14577_b200 as onedf  # noqa: E402

CASES = [
    ("noncausal_1M_single_run", dict(B=1, H=1, N=1 << 20, chunk=1, causal=0)),
    ("noncausal_64K_x96", dict(B=8, H=12, N=1 << 16, chunk=1, causal=0)),
    ("long1m_causal_x12", dict(B=1, H=12, N=1 << 20, chunk=1 << 15, causal=1)),
    ("long64k_causal_x96 (on-chip)", dict(B=8, H=12, N=1 << 16, chunk=2048, causal=1)),
]


def main():
    dev = torch.device("cuda:0")
    for name, kw in CASES:
        p = onedf.make_problem(**kw, d_k=3, d_v=4, k=4, window=8, mean_slot=0)
        g = torch.Generator(device=dev).manual_seed(1)
        X = torch.randn(p.B, p.H, p.N, 3, device=dev, generator=g)
        ws = onedf.Workspace(dev)
        _, kc, _ = onedf.encode(p, X, X.flip(-1).contiguous(), ws=ws)
        onedf.sort(p, kc, ws=ws)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            onedf.sort(p, kc, ws=ws)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        keys = p.B * p.H * p.N
        print(json.dumps({"case": name, "keys": keys, "run_len": p.N if not kw["causal"] else kw["chunk"],
                          "ms": ts[2], "Gkeys_per_s": keys / ts[2] / 1e6}))


if __name__ == "__main__":
    main()
