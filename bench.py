"""bench.py -- causal top-k attention fwd+bwd (ZETA, arXiv 2501.14577) on B200.

python bench.py [--gpus N] [--steps K] [--warmup W] [--config long64k] [--impl reference]

A step = one pass of the whole hot path (A1-A12: encode + sort + fwd + bwd)
over one batch of synthetic input already resident in HBM.  One process per
GPU: `--gpus N` (N > 1) re-launches this script under torch.distributed.run
on 127.0.0.1 unless it is already running under it.  (b,h) slices are
independent problems, so the data path has no collective:
  --scaling strong (default): the config's B x H slices are split
      into contiguous per-rank ranges (dist.partition); t_P = max over ranks;
  --scaling weak: every rank runs the config's whole batch of its own slices.
The only exchange is the shared Cauchy scale's gradient d_eps (one f64 per
rank, all-gathered and summed in rank order, reading D20).  Rank 0 prints one
JSON line.

--impl reference times the CPU oracle (oracle/, the method's plain f64
reference -- this tier has no installable reference implementation) on the
same config, each step a bounded sample (one (b,h) slice) of the workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "causal top-k attn fwd+bwd queries/s at N=64K, 1/2/4/8 B200; % HBM roofline"
UNIT = "queries/s"


# ----------------------------------------------------------------------------- algorithmic bytes
def alg_bytes(cfg) -> dict:
    """Per-kernel ALGORITHMIC bytes of one call over the whole batch, SURVEY 8(d):
    gathered rows and candidate records counted per use; dense N^2 work not counted.
    L = ceil(log2(M+1)); sum_m = sum_i m_i; sum_c = sum_i |C_i|; sum_kappa = sum_i |I_i|."""
    N, dk, dv, k, W = cfg.N, cfg.d_k, cfg.d_v, cfg.k, cfg.window
    s_k, s_v = 4 * dk, 4 * dv
    if cfg.causal:
        M = cfg.chunk
        lens =[min(M, N - c * M) for c in range((N + M - 1) // M)]
        # sum over queries of admissible runs / candidates / selected
        sum_m = sum_c = sum_kappa = 0
        prefix_w = [0]
        prefix_len = [0]
        for c, ln in enumerate(lens):
            prefix_w.append(prefix_w[-1] + min(W, ln))
            prefix_len.append(prefix_len[-1] + ln)
        for c in range(len(lens)):
            nq = lens[c]                       # queries of chunk c see runs 0..c-1
            sum_m += nq * c
            sum_c += nq * prefix_w[c]
            sum_kappa += nq * min(k, prefix_len[c])
        Lbits = max(1, (M).bit_length())
    else:
        sum_m = N
        sum_c = N * min(W, N)
        sum_kappa = N * min(k, N)
        Lbits = max(1, N.bit_length())
    BH = cfg.BH
    enc = 4 * N * s_k + 16 * N                          # fit + encode reads of Q, K; codes written
    srt = 20 * N
    means = 2 * N * (s_k + s_v)
    fwd = N * (8 + s_k) + 8 * Lbits * sum_m + (s_k + 4) * sum_c + s_v * sum_kappa + N * (s_k + s_v) \
        + N * (s_v + 4 * k + 4)
    bq = N * (2 * s_v + s_k + 4 + 4 * k) + (s_v + s_k + 8) * sum_kappa + N * s_k
    tr = 8 * sum_kappa + 4 * N
    bk = (12 + s_v + s_k) * sum_kappa + N * (s_v + s_k)
    scan = 4 * N * (s_k + s_v)
    per = dict(encode=enc, sort=srt, fwd_means=means, fwd_topk=fwd, bwd_query=bq, bwd_transpose=tr, bwd_key=bk,
               bwd_scans=scan)
    out = {n: v * BH for n, v in per.items()}
    out["F"] = BH * (enc + srt + means + fwd)
    out["Bw"] = BH * (bq + tr + bk + scan)
    out["B_alg"] = out["F"] + out["Bw"]
    # compulsory: unique tensors only
    fw_c = N * (2 * s_k + s_v) + 16 * N + 12 * N + N * (s_v + 4 * k + 4)
    bw_c = N * (2 * s_k + 3 * s_v + 4 * k + 4) + N * (2 * s_k + s_v)
    out["B_comp"] = BH * (fw_c + bw_c)
    out["sum_c"] = BH * sum_c
    out["sum_kappa"] = BH * sum_kappa
    return out


# ----------------------------------------------------------------------------- clocks sampler
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str):
        self.gpu_id = gpu_id
        self.proc = None
        self.lines = []
        self.t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", self.gpu_id, f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=5)
        sm, mx, reasons, pw = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
                pw.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "power_w_max": max(pw) if pw else None}


def _bad_clocks(c: dict) -> bool:
    if any(r in c.get("reasons", []) for r in ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")):
        return True
    if c.get("sm_mhz") and c.get("sm_max_mhz") and c["sm_mhz"] < 0.5 * c["sm_max_mhz"] and \
            "sw_power_cap" not in c.get("reasons", []):
        return True
    return False


# ----------------------------------------------------------------------------- helpers
def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def rank_slices(cfg, world: int, rank: int, scaling: str):
    """Global (b,h) slice ids this rank runs and the per-rank problem shape (B', H').
    strong: contiguous split of the config's B*H slices (SURVEY 8(d) "each rank takes B.H/P
    contiguous slices"); weak: every rank runs a whole batch of its own slices."""
    from paper_2501_14577_b200.dist import partition, weak_slices
    if scaling == "strong":
        bhs = partition(cfg.BH, world, rank)
        return bhs, (1, len(bhs))
    return weak_slices(cfg.BH, rank), (cfg.B, cfg.H)


def units_per_step(cfg, world: int, scaling: str) -> int:
    """Queries every rank together processes in one step."""
    return cfg.BH * cfg.N * (1 if scaling == "strong" else world)


def max_over_ranks(x: float, device=None) -> float:
    """t_P = max over ranks; identity without a process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _make_rank_inputs(cfg, bhs, shape):
    """This rank's slices (seeded by global slice id, so the ranks' union is the 1-GPU batch)."""
    import numpy as np

    import synth
    x = synth.make_inputs(cfg, bh_range=bhs)
    return {n: np.ascontiguousarray(v.reshape(*shape, *v.shape[2:])) for n, v in x.items()}


def host_info() -> dict:
    """nproc and the CPU model of this box (every CPU row states them)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.lower().startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


# ----------------------------------------------------------------------------- reference arm (CPU oracle)
def _oracle_sample(cfg, budget_s: float, max_slices: int):
    """Run the oracle (as it stands, all host cores) on whole (b,h) slices of the workload, one at
    a time, until `budget_s` seconds have passed (at least one slice).  -> (seconds, slices)."""
    import oracle
    import synth
    oracle.build()
    one = cfg.with_(B=1, H=1)
    p = oracle.Problem(**one.problem_kwargs())
    sec, n = 0.0, 0
    while n < max_slices and (n == 0 or sec < budget_s):
        x = synth.make_inputs(cfg, bh_range=[n])
        t0 = time.perf_counter()
        oracle.pipeline(p, x["Q"], x["K"], x["V"], synth.EPS, x["dO"])
        sec += time.perf_counter() - t0
        n += 1
    return sec, n


def run_reference(args, cfg, world, rank):
    """--impl reference: the CPU oracle (this tier's reference arm) on rank 0 only; each step is a
    bounded sample (one (b,h) slice) of the workload."""
    if rank != 0:
        return
    import oracle
    import synth
    oracle.build()
    one = cfg.with_(B=1, H=1)
    p = oracle.Problem(**one.problem_kwargs())
    times = []
    for s in range(args.warmup + args.steps):
        x = synth.make_inputs(cfg, bh_range=[s % cfg.BH])
        t0 = time.perf_counter()
        oracle.pipeline(p, x["Q"], x["K"], x["V"], synth.EPS, x["dO"])
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    sec = sum(times) / len(times)
    value = cfg.N / sec
    cores = oracle.num_threads()
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config_json(cfg, world, args.scaling),
            "cpu_baseline": dict({"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                                  "sample": f"one (b,h) slice of {cfg.name} (N={cfg.N} queries) per step, full "
                                            f"encode+sort+select+fwd+bwd"}, **host_info()),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, budget_s: float = 10.0):
    """The oracle as it stands on this box's host cores, on a bounded sample: whole (b,h) slices of
    the workload until ~budget_s seconds of oracle time."""
    import oracle
    sec, n = _oracle_sample(cfg, budget_s, cfg.BH)
    return dict({"value": n * cfg.N / sec, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                 "sample": f"{n} of the {cfg.BH} (b,h) slices of {cfg.name} ({n * cfg.N} queries), full "
                           f"encode+sort+select+fwd+bwd, {sec:.1f} s"}, **host_info())


def _config_json(cfg, world, scaling):
    if scaling == "strong":
        par = f"dp{world}: one process per GPU; the {cfg.BH} (b,h) slices split contiguously over the ranks"
        gb = cfg.B
    else:
        par = f"dp{world}: one process per GPU, each its own batch of {cfg.BH} (b,h) slices"
        gb = cfg.B * world
    return {"workload": cfg.name, "model": "ZETA top-k attention op (no weights)", "B": cfg.B, "H": cfg.H,
            "global_batch": gb, "seq_len": cfg.N, "d_k": cfg.d_k, "d_v": cfg.d_v, "k": cfg.k,
            "window": cfg.window, "chunk": cfg.chunk, "chunks": -(-cfg.N // cfg.chunk) if cfg.causal else 1,
            "causal": cfg.causal, "mean_slot": cfg.mean_slot, "pass": "encode+sort+fwd+bwd",
            "l2": "inputs larger than L2 (V and dO are 1.6 GB each at long64k); no flush",
            "parallelism": par}


# ----------------------------------------------------------------------------- GPU arm
def run_gpu(args, cfg, world, rank, local):
    import torch
    import torch.distributed as dist

    import __graft_entry__
    # bind the device first, then the process group (device_id: NCCL need not guess the rank's GPU)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if rank == 0:
        __graft_entry__.build()
    if world > 1:
        dist.barrier(device_ids=[local])
    import paper_2501_14577_b200 as onedf
    from paper_2501_14577_b200 import abi
    from paper_2501_14577_b200 import dist as odist

    bhs, (Bp, Hp) = rank_slices(cfg, world, rank, args.scaling)
    if args.device_inputs:
        # seeded N(0,1) inputs drawn on the device (shapes too large for the host recipe, e.g. long1m
        # at B x H = 96: 51 GB); the synth/ recipe is what the parity tests use
        import synth
        g = torch.Generator(device=dev).manual_seed(synth.SEED_BASE + cfg.cfg_index + 1000 * rank)
        x = None
        t = {n: torch.randn(Bp, Hp, cfg.N, w, device=dev, generator=g)
             for n, w in (("Q", cfg.d_k), ("K", cfg.d_k), ("V", cfg.d_v), ("dO", cfg.d_v))}
    else:
        x = _make_rank_inputs(cfg, bhs, (Bp, Hp))
        t = {n: torch.from_numpy(v).to(dev) for n, v in x.items()}
    p = onedf.make_problem(**dict(cfg.problem_kwargs(), B=Bp, H=Hp))
    # --groups G: the slices are processed in G contiguous groups (one workspace sized for a group,
    # inputs and outputs of every slice resident) -- shapes whose workspace for all slices at once
    # exceeds HBM (long1m at B x H = 96)
    G = max(1, min(args.groups, Bp * Hp))
    gsz = [(Bp * Hp) // G + (1 if g < (Bp * Hp) % G else 0) for g in range(G)]
    gofs = [sum(gsz[:g]) for g in range(G)]
    pg = [onedf.make_problem(**dict(cfg.problem_kwargs(), B=1, H=n)) for n in gsz]
    import synth
    eps = torch.tensor(synth.EPS, dtype=torch.float32, device=dev)
    N = cfg.N
    qcode = torch.empty((Bp, Hp, N), dtype=torch.int64, device=dev)
    kcode = torch.empty_like(qcode)
    scode = torch.empty_like(qcode)
    perm = torch.empty((Bp, Hp, N), dtype=torch.int32, device=dev)
    qorder = torch.empty_like(perm)
    O = torch.empty_like(t["V"])
    idx = torch.empty((Bp, Hp, N, cfg.k), dtype=torch.int32, device=dev)
    Z = torch.empty((Bp, Hp, N), dtype=torch.float32, device=dev)
    indeg = torch.empty((Bp, Hp, N), dtype=torch.int32, device=dev)   # the forward's A9 counts, for the backward
    dQ, dK, dV = torch.empty_like(t["Q"]), torch.empty_like(t["K"]), torch.empty_like(t["V"])
    d_eps = torch.empty((G,), dtype=torch.float64, device=dev)        # per group (summed by the consumer)
    need = max(onedf.onedf_workspace_size(q, op) for q in pg for op in (abi.OP_ENCODE, abi.OP_SORT, abi.OP_FWD,
                                                                         abi.OP_BWD))
    wsbuf = torch.empty(need + 256, dtype=torch.uint8, device=dev)
    ws = wsbuf.data_ptr() + ((-wsbuf.data_ptr()) % 256)
    wsbuf[(-wsbuf.data_ptr()) % 256:][:16].zero_()      # flag words (onedf.h "Errors")
    stream = torch.cuda.current_stream(dev)

    # stage events: 0 start | 1 encode | 2 sort | fwd: 3 means 4 records 5 topk | bwd: 6 means 7 CSR
    # (transpose) 8 query 9 key 10 scan 11 eps | 12 d_eps exchange
    NEV = 13

    def new_events():
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(NEV)] for _ in range(G)]
        for ge in evs:
            for e in ge:
                e.record(stream)
        return evs

    def ptr(tn, g, width=1):
        return tn.data_ptr() + gofs[g] * N * width * tn.element_size()

    # the forward's prefix means for the backward: group g's own region (onedf_means_floats of its problem)
    mfl = [abi.onedf_means_floats(q) for q in pg]
    moffs = [sum(mfl[:g]) for g in range(G)]
    means = torch.empty(max(1, sum(mfl)), device=dev)

    def mptr(g):
        return means.data_ptr() + moffs[g] * 4 if mfl[g] else None

    def step(evg):
        for g in range(G):
            ev, q = evg[g], pg[g]
            tq, tk, tv, tdo = (ptr(t[n], g, w) for n, w in (("Q", cfg.d_k), ("K", cfg.d_k), ("V", cfg.d_v),
                                                             ("dO", cfg.d_v)))
            qc, kc, sc, pm, qo = (ptr(a, g) for a in (qcode, kcode, scode, perm, qorder))
            ev[0].record(stream)
            abi.onedf_encode(q, tq, tk, None, qc, kc, None, ws, need, stream)
            ev[1].record(stream)
            abi.onedf_sort(q, kc, sc, pm, ws, need, stream)
            abi.onedf_sort(q, qc, None, qo, ws, need, stream)      # Morton query schedule for fwd and bwd
            ev[2].record(stream)
            abi.onedf_topk_attn_fwd_traced(q, tq, tk, tv, eps, qc, sc, pm, qo, ptr(O, g, cfg.d_v), ptr(idx, g, cfg.k),
                                           ptr(Z, g), ws, need, ev[3:6], stream, indeg=ptr(indeg, g),
                                           means=mptr(g))
            abi.onedf_topk_attn_bwd_traced(q, tq, tk, tv, eps, ptr(O, g, cfg.d_v), tdo, ptr(idx, g, cfg.k), ptr(Z, g),
                                           qc, qo, pm, ptr(dQ, g, cfg.d_k), ptr(dK, g, cfg.d_k), ptr(dV, g, cfg.d_v),
                                           d_eps.data_ptr() + 8 * g, ws, need, ev[6:12], stream, indeg=ptr(indeg, g),
                                           means=mptr(g))
            if world > 1 and G == 1:
                odist.combine_d_eps(d_eps[0])   # one f64 per rank, rank-ordered sum (D20)
            ev[12].record(stream)

    stage_names = ["encode", "sort", "fwd_means", "fwd_records", "fwd_topk", "bwd_means", "bwd_transpose",
                   "bwd_query", "bwd_key", "bwd_scans", "bwd_eps", "deps_exchange"]

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    # warm-up
    for _ in range(args.warmup):
        step(new_events())
    torch.cuda.synchronize(dev)
    st = onedf.check_device_status(ws)
    if st != abi.OK:
        raise RuntimeError(f"device status {st} after warm-up")

    gpu_id = "GPU-" + str(torch.cuda.get_device_properties(dev).uuid)

    def timed():
        evs = [new_events() for _ in range(args.steps)]
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        clocks = ClockSampler(gpu_id)
        barrier()
        torch.cuda.synchronize(dev)
        clocks.start()
        time.sleep(0.3)
        t0.record(stream)
        for s in range(args.steps):
            step(evs[s])
        t1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        clk = clocks.stop()
        total_ms = t0.elapsed_time(t1)
        stages = {n: [] for n in stage_names}
        for evg in evs:
            for si, n in enumerate(stage_names):
                stages[n].append(sum(ev[si].elapsed_time(ev[si + 1]) for ev in evg))
        return total_ms, stages, clk

    total_ms, stages, clk = timed()
    if _bad_clocks(clk):
        total_ms, stages, clk = timed()
        clk["remeasured"] = True
    ms_rank = total_ms / args.steps
    ms = max_over_ranks(ms_rank, dev)

    launches_per_step = sum(count_launches(q) for q in pg)
    units = units_per_step(cfg, world, args.scaling)

    # ------------------------------------------------------------ e2e through the host-buffer entry point
    e2e = None
    if not args.no_e2e and x is not None:       # (device-drawn inputs have no host copy to stream)
        del O, idx, Z, dQ, dK, dV, wsbuf, qcode, kcode, scode, perm, qorder
        dev_inputs = t
        del dev_inputs, t
        torch.cuda.empty_cache()
        pin = {n: torch.from_numpy(v).pin_memory() for n, v in x.items()}
        outs = {n: torch.empty_like(pin["V" if n in ("O", "dV") else "Q"]).pin_memory()
                for n in ("O", "dQ", "dK", "dV")}
        d_eps_h = torch.zeros((), dtype=torch.float64).pin_memory()
        hs = onedf.HostStep(p, dev)

        def host_step():
            hs(pin["Q"], pin["K"], pin["V"], synth.EPS, pin["dO"], outs["O"], outs["dQ"], outs["dK"], outs["dV"],
               d_eps_h, stream)

        for _ in range(max(1, min(args.warmup, 2))):
            host_step()
        torch.cuda.synchronize(dev)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        ksteps = max(1, min(args.steps, 5))
        e0.record(stream)
        for _ in range(ksteps):
            host_step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        ems = max_over_ranks(e0.elapsed_time(e1) / ksteps, dev)
        e2e = {"value": units / (ems / 1e3), "unit": UNIT, "ms_per_step": ems,
               "h2d_bytes_per_step": onedf.HostStep.h2d_bytes(p), "d2h_bytes_per_step": onedf.HostStep.d2h_bytes(p),
               "api": "onedf_topk_attn_step_host (pinned host buffers, copies inside the timed region)",
               "steps": ksteps}

    if rank != 0:
        if world > 1:
            barrier()
            dist.destroy_process_group()
        return

    # ------------------------------------------------------------ roofline of the dominant kernel
    rcfg = cfg.with_(B=Bp, H=Hp)                      # rank 0's own work (what its events timed)
    ab = alg_bytes(rcfg)
    peak, peak_src = _peaks()
    kern_map = {"fwd_topk": "fwd_topk", "bwd_query": "bwd_query", "bwd_key": "bwd_key"}
    avg = {n: sum(v) / len(v) for n, v in stages.items()}
    dom = max(kern_map, key=lambda n: avg[n])
    achieved = ab[kern_map[dom]] / (avg[dom] / 1e3) / 1e9
    traffic = _ncu_traffic(dom, cfg.name) if Bp * Hp == cfg.BH else None
    step_dram = _ncu_step_dram(cfg.name) if Bp * Hp == cfg.BH else None
    roof = {"bound": "hbm", "kernel": {"fwd_topk": "topk_attn_fwd_kernel", "bwd_query": "bwd_query_kernel",
                                       "bwd_key": "bwd_key_kernel"}[dom],
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "peak_source": peak_src,
            "alg_bytes_per_launch": ab[kern_map[dom]], "avg_launch_ms": avg[dom],
            "note": "achieved = SURVEY 8(d) algorithmic bytes (candidate records and gathered rows counted per "
                    "use) / CUDA-event time of the kernel inside the timed region; can exceed 1 only through "
                    "on-chip (L1/L2) reuse; R_dram = ncu DRAM bytes of every launch of one step (profiles/, "
                    "measured separately) / this step time",
            "step": {"B_alg": ab["B_alg"], "R_alg": ab["B_alg"] / (ms_rank / 1e3) / 1e9 / peak,
                     "B_comp": ab["B_comp"], "R_comp": ab["B_comp"] / (ms_rank / 1e3) / 1e9 / peak,
                     "B_dram": step_dram,
                     "R_dram": None if step_dram is None else step_dram / (ms_rank / 1e3) / 1e9 / peak}}
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg)
    value = units / (ms / 1e3)
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic: seeded iid N(0,1) Q,K,V,dO (synth/, SURVEY 8(d))",
            "config": _config_json(cfg, world, args.scaling),
            "tokens_per_s": units / cfg.H / (ms / 1e3),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches_per_step * args.steps,
            "gpu_launches_per_step": launches_per_step, "clocks": clk,
            "rank0_slices": [bhs[0], bhs[-1] + 1] if len(bhs) else [], "rank0_ms_per_step": ms_rank,
            "phases_ms": {n: round(v, 4) for n, v in avg.items()}}
    print(json.dumps(line), flush=True)
    if world > 1:
        barrier()
        dist.destroy_process_group()


def count_launches(p) -> int:
    """Kernel launches of one step, from the library's launch plan (checked against the ncu launch
    list in profiles/): encode 2 (bounds partials, encode); 2 sorts (key runs, Morton query
    schedule shared by fwd and bwd), each 1 launch for runs <= 8192 keys else the onesweep's
    histogram + bases + one launch per 8-bit digit; fwd: prefix means 6 (mean slot), key records 1,
    top-k 1 (which also counts the keys' in-degrees); bwd: CSR offset scan 3 (block sums, their scan,
    apply; the counts and the prefix means come from the forward), query side 1, long-segment order
    1, key side 1, mean-slot scans 6, eps 2."""
    means = 6 if p.mean_slot else 0
    run = p.N if not p.causal else min(p.chunk, p.N)
    bits = p.d_k * (p.bits or min(63 // p.d_k, 32))
    sort = 1 if run <= 8192 else 2 + (bits + 7) // 8
    fwd = means + 2
    bwd = 3 + 1 + 1 + 1 + means + 2
    return 2 + 2 * sort + fwd + bwd


def _ncu_json(name):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def _ncu_traffic(kernel_key, workload):
    """dram bytes per launch of the dominant kernel from the committed ncu --set full summary."""
    d = _ncu_json("ncu_traffic.json")
    if d.get("workload", "long64k") != workload:
        return None
    return d.get(kernel_key)


def _ncu_step_dram(workload):
    """ncu dram__bytes_read.sum + dram__bytes_write.sum summed over every launch of one step."""
    d = _ncu_json("ncu_step_dram.json")
    return d.get("bytes_per_step") if d.get("workload") == workload else None


def _self_launch(n: int) -> int:
    """--gpus N outside torchrun: run N ranks of this script under torch.distributed.run."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=None)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="long64k")
    ap.add_argument("--impl", default="onedf", choices=["onedf", "reference"])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--bh", type=int, default=0, help="override B x H with 1 x BH slices (config sweeps of long N)")
    ap.add_argument("--groups", type=int, default=1, help="process the slices in G contiguous groups (one group's "
                    "workspace; for shapes whose all-slice workspace exceeds HBM)")
    ap.add_argument("--device-inputs", action="store_true", help="draw the seeded inputs on the device")
    args = ap.parse_args()
    world, rank, local = _dist_env()
    if args.gpus is not None and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _self_launch(args.gpus)
    if args.gpus is not None and "WORLD_SIZE" in os.environ and args.gpus != world:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}))
        return 1
    import synth
    cfg = synth.CONFIGS[args.config]
    if args.bh:
        cfg = cfg.with_(B=1, H=args.bh)
    if args.impl == "reference":
        run_reference(args, cfg, world, rank)
        return 0
    run_gpu(args, cfg, world, rank, local)
    return 0


if __name__ == "__main__":
    sys.exit(main())
