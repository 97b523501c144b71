"""Shared helpers for the GPU parity tests: run the CUDA path (through the C
ABI binding) and the CPU oracle on the same seeded synthetic inputs."""
from __future__ import annotations

import numpy as np

import oracle
import synth

RTOL, ATOL = 1e-5, 1e-6          # north_star: fp32 outputs and gradients within 1e-5 rel / 1e-6 abs


def gpu_run(kw: dict, x: dict, eps: float = synth.EPS, bwd: bool = True, lohi=None):
    """Whole path on cuda:0 -> dict of numpy arrays (codes as uint64)."""
    import torch

    import paper_2501_14577_b200 as onedf
    dev = torch.device("cuda:0")
    t = {n: torch.from_numpy(np.ascontiguousarray(v)).to(dev) for n, v in x.items()}
    p = onedf.make_problem(**kw)
    for n in ("V", "dO"):                  # value rows in the problem's storage type (NEXT-4)
        if n in t:
            t[n] = t[n].to(onedf.value_dtype(p))
    e = torch.tensor(eps, dtype=torch.float32, device=dev)
    ws = onedf.Workspace(dev)
    lohi_t = None if lohi is None else torch.from_numpy(lohi).to(dev)
    qc, kc, lohi_out = onedf.encode(p, t["Q"], t["K"], lohi_t, ws=ws)
    sc, pm = onedf.sort(p, kc, ws=ws)
    qo = onedf.query_schedule(p, qc, ws=ws)
    # the forward's in-degree counts feed the backward's CSR (the bench's path; the schedule-hint test
    # checks that the counting backward gives the same bits)
    indeg = torch.empty((p.B, p.H, p.N), dtype=torch.int32, device=dev)
    means = torch.empty(onedf.means_floats(p), device=dev)       # the forward's prefix means, likewise
    O, idx, Z = onedf.topk_attn_fwd(p, t["Q"], t["K"], t["V"], e, qc, sc, pm, ws=ws, qorder=qo, indeg=indeg,
                                    means=means)
    out = dict(qcode=qc, kcode=kc, lohi=lohi_out, scode=sc, perm=pm, O=O, idx=idx, Z=Z)
    if bwd:
        dQ, dK, dV, d_eps = onedf.topk_attn_bwd(p, t["Q"], t["K"], t["V"], e, O, t["dO"], idx, Z, ws=ws,
                                                qorder=qo, perm=pm, indeg=indeg, means=means)
        out.update(dQ=dQ, dK=dK, dV=dV, d_eps=d_eps)
    torch.cuda.synchronize()
    res = {}
    for n, v in out.items():
        a = (v.float() if v.dtype == torch.bfloat16 else v).cpu().numpy()
        res[n] = a.view(np.uint64) if n in ("qcode", "kcode", "scode") else a
    return res


def oracle_run(kw: dict, x: dict, eps: float = synth.EPS, bwd: bool = True, lohi=None):
    p = oracle.Problem(**kw)
    return oracle.pipeline(p, x["Q"], x["K"], x["V"], eps, x["dO"] if bwd else None, lohi)


def assert_close(got, want, name: str, rtol=RTOL, atol=ATOL):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, (name, got.shape, want.shape)
    err = np.abs(got - want)
    bound = atol + rtol * np.abs(want)
    bad = err > bound
    if bad.any():
        i = np.unravel_index(np.argmax(err - bound), err.shape)
        raise AssertionError(f"{name}: {int(bad.sum())}/{bad.size} outside {rtol} rel / {atol} abs; "
                             f"worst at {i}: got {got[i]!r} want {want[i]!r}")


def bf16_round(a):
    """The bfloat16 value (round to nearest even) of every element, as float32 (exact)."""
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(torch.bfloat16).float().numpy()


def bf16_half_ulp(a):
    """Half the bfloat16 spacing at |a| (8-bit significand: ulp = 2^(floor(log2|a|) - 7)); 0 at 0."""
    a = np.abs(np.asarray(a, dtype=np.float64))
    e = np.floor(np.log2(np.where(a > 0, a, 1.0)))
    return np.where(a > 0, np.ldexp(1.0, (e - 8).astype(np.int64)), 0.0)


def assert_close_bf16(got, want, name: str, rtol=RTOL, atol=ATOL):
    """NEXT-4 contract (reading D26) for a value stored as bfloat16: one round-to-nearest of a result
    within the fp32 contract, i.e. |got - want| <= half a bf16 ulp (at got or want, the larger) +
    atol + rtol |want|."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, (name, got.shape, want.shape)
    err = np.abs(got - want)
    bound = np.maximum(bf16_half_ulp(got), bf16_half_ulp(want)) + atol + rtol * np.abs(want)
    bad = err > bound
    if bad.any():
        i = np.unravel_index(np.argmax(err - bound), err.shape)
        raise AssertionError(f"{name}: {int(bad.sum())}/{bad.size} outside the bf16 contract; "
                             f"worst at {i}: got {got[i]!r} want {want[i]!r}")


def assert_same(got, want, name: str):
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape, (name, got.shape, want.shape)
    if not np.array_equal(got, want):
        diff = np.argwhere(got != want)
        i = tuple(diff[0])
        raise AssertionError(f"{name}: {len(diff)} mismatching elements; first at {i}: got {got[i]} want {want[i]}")


def slice_inputs(x: dict, bhs) -> dict:
    """Select (b,h) slices of [B,H,N,.] arrays -> [1, len(bhs), N, .]."""
    out = {}
    for n, v in x.items():
        flat = v.reshape(-1, *v.shape[2:])
        out[n] = np.ascontiguousarray(flat[list(bhs)][None])
    return out


def slice_out(a, bhs):
    flat = a.reshape(-1, *a.shape[2:])
    return flat[list(bhs)][None]
