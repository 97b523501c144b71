"""Time the fwd (and optionally bwd) of a config with CUDA events (tools; bench.py is the measured path)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2501_14577_b200 as onedf  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="long64k")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--bwd", action="store_true")
ap.add_argument("--synth", action="store_true", help="the config's seeded synth/ inputs (e.g. tokens) instead of iid")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
p = onedf.make_problem(**cfg.problem_kwargs())
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(1)
shp = (p.B, p.H, p.N)
if a.synth:
    x = synth.make_inputs(cfg)
    Q, K, V, dO = (torch.from_numpy(x[n]).to(dev) for n in ("Q", "K", "V", "dO"))
else:
    Q = torch.randn(*shp, p.d_k, device=dev, generator=g)
    K = torch.randn(*shp, p.d_k, device=dev, generator=g)
    V = torch.randn(*shp, p.d_v, device=dev, generator=g)
    dO = torch.randn(*shp, p.d_v, device=dev, generator=g)
eps = torch.tensor(0.5, device=dev)
ws = onedf.Workspace(dev)
qc, kc, _ = onedf.encode(p, Q, K, ws=ws)
sc, pm = onedf.sort(p, kc, ws=ws)
ts = []
for _ in range(a.reps + 1):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    O, idx, Z = onedf.topk_attn_fwd(p, Q, K, V, eps, qc, sc, pm, ws=ws)
    e1.record()
    if a.bwd:
        onedf.topk_attn_bwd(p, Q, K, V, eps, O, dO, idx, Z, ws=ws, qcode=qc, perm=pm)
    e2.record()
    torch.cuda.synchronize()
    ts.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
ts = ts[1:]
try:
    import ctypes
    from paper_2501_14577_b200 import abi as _abi
    st = (ctypes.c_ulonglong * 8)()
    _abi._lib.onedf_debug_fwd_stats(st)
    n = st[0]
    if n:
        mean = st[1] / n
        print(f"fwd stats: queries {n}  mean cnt {mean:.1f}  rms {(st[2] / n) ** 0.5:.1f}  fallbacks {st[3]}")
except AttributeError:
    pass
print(f"{os.environ.get('ONEDF_LIB', 'default')}: fwd {min(t[0] for t in ts):.2f} ms  bwd {min(t[1] for t in ts):.2f} ms"
      f"  idxsum {int(idx.sum())} Osum {float(O.double().sum()):.6f}")
