"""Time the NEXT-4 front end (onedf_project_encode, onedf_project_bwd) and, for comparison, the
bf16-storage variant of the attention step, with CUDA events on the launching stream (tools;
bench.py is the measured headline path).  Prints one JSON line.

    python tools/time_projection.py --config long64k --d-model 768 --reps 5
"""
from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2501_14577_b200 as onedf  # noqa: E402
import synth  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="long64k")
    ap.add_argument("--d-model", type=int, default=768)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    cfg = synth.CONFIGS[a.config]
    kw = cfg.problem_kwargs()
    p = onedf.make_problem(**kw)
    dev = torch.device("cuda:0")
    g = torch.Generator(device=dev).manual_seed(1)
    dm = a.d_model
    X = torch.randn(p.B, p.N, dm, device=dev, generator=g)
    Wq = torch.randn(p.H, p.d_k, dm, device=dev, generator=g) / dm ** 0.5
    Wk = torch.randn(p.H, p.d_k, dm, device=dev, generator=g) / dm ** 0.5
    bq = torch.randn(p.H, p.d_k, device=dev, generator=g)
    bk = torch.randn(p.H, p.d_k, device=dev, generator=g)
    theta = torch.tensor(0.0, device=dev)
    ws = onedf.Workspace(dev)
    out = {}
    res = {}

    def fwd():
        res["f"] = onedf.project_encode(p, X, Wq, Wk, bq, bk, theta, ws=ws)

    out["project_encode_ms"] = timed(fwd, a.reps)
    Q, K = res["f"][0], res["f"][1]
    dQ, dK = torch.randn_like(Q), torch.randn_like(K)
    d_eps = torch.tensor(1.0, dtype=torch.float64, device=dev)
    out["project_bwd_ms"] = timed(lambda: onedf.project_bwd(p, X, Wq, Wk, dQ, dK, theta, d_eps, ws=ws), a.reps)
    out["encode_only_ms"] = timed(lambda: onedf.encode(p, Q, K, ws=ws), a.reps)
    rows = p.B * p.N
    O = 2 * p.H * p.d_k
    out["project_flops_fwd"] = 2.0 * rows * dm * O
    out["project_flops_bwd"] = 4.0 * rows * dm * O
    out["X_bytes"] = rows * dm * 4
    # attention step in f32 and bf16 value storage (fwd+bwd, resident inputs)
    for name, vd in (("f32", 0), ("bf16", 1)):
        pv = onedf.make_problem(**dict(kw, vdtype=vd))
        vt = onedf.value_dtype(pv)
        V = torch.randn(p.B, p.H, p.N, p.d_v, device=dev, generator=g).to(vt)
        dO = torch.randn(p.B, p.H, p.N, p.d_v, device=dev, generator=g).to(vt)
        eps = torch.tensor(0.5, device=dev)
        qc, kc, _ = onedf.encode(pv, Q, K, ws=ws)

        def step():
            sc, pm = onedf.sort(pv, kc, ws=ws)
            qo = onedf.query_schedule(pv, qc, ws=ws)
            Oa, idx, Z = onedf.topk_attn_fwd(pv, Q, K, V, eps, qc, sc, pm, ws=ws, qorder=qo)
            onedf.topk_attn_bwd(pv, Q, K, V, eps, Oa, dO, idx, Z, ws=ws, qorder=qo, perm=pm)

        out[f"attn_step_{name}_ms"] = timed(step, a.reps)
        del V, dO
    out.update(config=a.config, d_model=dm, B=p.B, H=p.H, N=p.N, d_k=p.d_k)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
