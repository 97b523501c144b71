"""NEXT-3 workload report: Fig. 4's grid (d_k 1..8, N in {512, 1024, 2048}, 10 trials, top-64
overlap of Morton-code neighbours vs exact Euclidean neighbours) and the k ablation (recall of
the method's top-k vs exact chunk-causal kNN, k = 16..48), each cell timed with CUDA events.

    python tools/locality_report.py > gpurun_out/locality.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2501_14577_b200 import workloads  # noqa: E402


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


def main():
    workloads.locality_sweep(dims=(3,), Ns=(512,), trials=1)      # warm-up (build, caches)
    rows = []
    for d in range(1, 9):
        for N in (512, 1024, 2048):
            (r,), ms = timed(lambda: workloads.locality_sweep(dims=(d,), Ns=(N,), trials=10))
            r["ms"] = ms
            rows.append(r)
    abl, ms = timed(lambda: workloads.k_ablation(N=2048, d_k=3, M=256, ks=(16, 24, 32, 40, 48), trials=8))
    print(json.dumps({"locality_fig4": [{k: v for k, v in r.items() if k != "per_trial"} for r in rows],
                      "k_ablation": {"N": 2048, "d_k": 3, "M": 256, "trials": 8, "rows": abl, "ms": ms},
                      "device": torch.cuda.get_device_name(0)}, indent=1))


if __name__ == "__main__":
    main()
