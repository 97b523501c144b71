"""Sequence-sharded ZETA top-k attention.

north_star: "Sequences too long for one GPU use sequence sharding, with an
NCCL all-gather over NVLink of the earlier ranks' sorted Morton runs."

The C = ceil(N/M) causal chunks of every (b,h) are dealt zig-zag over the
ranks (``onedf_shard_owner``: g = c mod 2P, owner = g < P ? g : 2P-1-g), so
the causal work of a rank, which grows with the chunk index (query i
searches floor(i/M) runs), is balanced.  One rank's step (``step``) is

  1. A1 partial: raw min/max of its own rows of Q and K
     -> all-reduce MIN/MAX (exact, order-free) -> D10 widening   (onedf kernels)
  2. A2/A3 on its rows: Morton codes, sorted runs of its own chunks
  3. all-gather of every rank's sorted runs (scode, perm) and of its K and V
     rows, so each rank holds the complete runs and rows of the sequence
  4. A4-A7 for its own queries (O, idx, Z of those rows)
  5. A8-A12 for its own queries: dQ rows, and PARTIAL dK, dV, d_eps over all
     keys; the partial rows are exchanged to their owners (all-to-all) and
     summed in rank order by ``onedf_rank_sum`` (f64, deterministic); d_eps
     partials are summed in rank order on every rank.

Every arithmetic step runs in libonedf.so; this module moves rows between
ranks.  ``step`` is a generator that yields its collectives, so one code path
serves both drivers: ``run_dist`` (one process per GPU, torch.distributed:
NCCL on GPUs, gloo in the CPU tests) and ``run_sim`` (all ranks in one
process on one GPU, the collectives done by direct copies -- the GPU parity
tests, since a test box has a single GPU).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import abi, api


def shard_owner(chunk: int, world: int) -> int:
    """The library's chunk -> rank map (zig-zag over 2*world)."""
    return abi.onedf_shard_owner(chunk, world)


@dataclass
class ShardPlan:
    """Which rows of a (b,h) each rank owns, and how to pack/unpack them."""
    N: int
    M: int
    world: int

    def __post_init__(self):
        self.C = -(-self.N // self.M)
        self.owner = [shard_owner(c, self.world) for c in range(self.C)]
        rows = [[] for _ in range(self.world)]
        for c in range(self.C):
            rows[self.owner[c]].extend(range(c * self.M, min((c + 1) * self.M, self.N)))
        self.rows = [torch.tensor(r, dtype=torch.int64) for r in rows]
        self.rows_max = max(1, max(len(r) for r in rows))
        self._dev = {}

    def chunks(self, rank: int) -> list:
        return [c for c in range(self.C) if self.owner[c] == rank]

    def _rows(self, rank: int, device):
        key = (rank, str(device))
        if key not in self._dev:
            self._dev[key] = self.rows[rank].to(device)
        return self._dev[key]

    def pack(self, x: torch.Tensor, rank: int) -> torch.Tensor:
        """x [B,H,N,...] -> the rows `rank` owns, zero-padded to rows_max along dim 2."""
        r = self._rows(rank, x.device)
        out = x.new_zeros((x.shape[0], x.shape[1], self.rows_max) + tuple(x.shape[3:]))
        out[:, :, :r.numel()] = x.index_select(2, r)
        return out

    def unpack(self, x: torch.Tensor, rank: int, block: torch.Tensor) -> None:
        """Write the first len(rows) rows of `block` (a pack() of `rank`) into x's rows of `rank`."""
        r = self._rows(rank, x.device)
        x.index_copy_(2, r, block[:, :, :r.numel()].to(x.dtype))

    def owned_mask(self, rank: int, device=None) -> torch.Tensor:
        m = torch.zeros(self.N, dtype=torch.bool, device=device)
        m[self._rows(rank, m.device)] = True
        return m


def shard_problem(p: abi.Problem, rank: int, world: int) -> abi.Problem:
    kw = {n: getattr(p, n) for n, _ in abi.Problem._fields_}
    kw.update(shard_rank=rank, shard_world=world)
    return api.make_problem(**kw)


def step(p: abi.Problem, Q, K, V, eps, dO=None, ws=None):
    """One rank's sharded encode -> sort -> fwd (-> bwd).  Generator: yields
    (kind, payload) collective requests and receives their results; returns a
    dict of this rank's outputs (rows it owns are final; see module doc).

    Q, K, V, dO: full-length [B,H,N,.] device buffers holding this rank's rows
    (other rows finite, e.g. zero); K and V are completed in place by the
    gather.  p: a problem with shard_rank/shard_world set."""
    ws = ws or api.Workspace(Q.device)
    lohi = api.bounds_partial(p, Q, K, ws)
    lohi = yield ("allreduce_minmax", lohi)
    api.bounds_finish(p, lohi, ws)
    qc, kc, lohi = api.encode(p, Q, K, lohi=lohi, ws=ws)
    sc, pm = api.sort(p, kc, ws=ws)
    qo = api.query_schedule(p, qc, ws=ws)          # the owned chunks' Morton schedule, for both passes
    yield ("gather_rows", [sc, pm, K, V])          # in place: complete runs and rows on every rank
    indeg = torch.empty((p.B, p.H, p.N), dtype=torch.int32, device=Q.device)   # this rank's queries' A9 counts
    means = torch.empty(api.means_floats(p), device=Q.device)                   # and prefix means, for the bwd
    O, idx, Z = api.topk_attn_fwd(p, Q, K, V, eps, qc, sc, pm, ws=ws, qorder=qo, indeg=indeg, means=means)
    out = {"O": O, "idx": idx, "Z": Z, "qcode": qc, "scode": sc, "perm": pm, "lohi": lohi}
    if dO is None:
        return out
    dQ, dK, dV, d_eps = api.topk_attn_bwd(p, Q, K, V, eps, O, dO, idx, Z, ws=ws, qorder=qo, perm=pm, indeg=indeg,
                                          means=means)
    yield ("reduce_rows", [dK, dV])                # in place: owners' rows become the rank-ordered sums
    d_eps = yield ("sum_scalar", d_eps)
    out.update(dQ=dQ, dK=dK, dV=dV, d_eps=d_eps)
    return out


def _rank_order_sum(xs):
    total = xs[0].clone()
    for x in xs[1:]:
        total += x
    return total


# ---------------------------------------------------------------- single-process driver (one GPU, all ranks)
def run_sim(gens, plan: ShardPlan, timing: list | None = None):
    """Drive `world` step() generators in lock step; the collectives are copies.

    timing: if a list is given, it receives each rank's device time (ms) spent in its own
    segments between collectives (CUDA events around every segment; the simulated
    collectives are excluded) -- the per-rank compute of a real sharded run."""
    world = len(gens)
    results = [None] * world
    done = [False] * world
    segs = [[] for _ in range(world)]

    def advance(r, value, first=False):
        e0 = e1 = None
        if timing is not None:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        try:
            out = next(gens[r]) if first else gens[r].send(value)
        finally:
            if timing is not None:
                e1.record()
                segs[r].append((e0, e1))
        return out

    reqs = [advance(r, None, first=True) for r in range(world)]
    while not all(done):
        kind = reqs[0][0]
        assert all(r[0] == kind for r in reqs), "ranks diverged"
        payloads = [r[1] for r in reqs]
        if kind == "allreduce_minmax":
            lo = torch.stack([x[..., 0, :] for x in payloads]).amin(0)
            hi = torch.stack([x[..., 1, :] for x in payloads]).amax(0)
            red = torch.stack([lo, hi], dim=-2)
            replies = [red.clone() for _ in range(world)]
        elif kind == "gather_rows":
            for t in range(len(payloads[0])):
                blocks = [plan.pack(payloads[s][t], s) for s in range(world)]
                for r in range(world):
                    for s in range(world):
                        if s != r:
                            plan.unpack(payloads[r][t], s, blocks[s])
            replies = [None] * world
        elif kind == "reduce_rows":
            for t in range(len(payloads[0])):
                sums = [api.rank_sum(torch.stack([plan.pack(payloads[r][t], s) for r in range(world)]))
                        for s in range(world)]
                for s in range(world):
                    plan.unpack(payloads[s][t], s, sums[s])
            replies = [None] * world
        elif kind == "sum_scalar":
            tot = _rank_order_sum(payloads)
            replies = [tot.clone() for _ in range(world)]
        else:
            raise ValueError(kind)
        for r in range(world):
            try:
                reqs[r] = advance(r, replies[r])
            except StopIteration as e:
                results[r] = e.value
                done[r] = True
    if timing is not None:
        torch.cuda.synchronize()
        timing.extend(sum(a.elapsed_time(b) for a, b in segs[r]) for r in range(world))
    return results


def exchange_bytes(p: abi.Problem, plan: ShardPlan, backward: bool = True) -> dict:
    """Bytes one rank sends per step in run_dist (payloads as packed): the bounds all-reduce,
    the all-gather of its rows of scode (8 B), perm (4 B), K (4 d_k B) and V (4 d_v B) to the
    other ranks, and (backward) the all-to-all of its partial dK, dV rows owned by others
    plus the d_eps all-gather."""
    P, BH, rows = plan.world, p.B * p.H, plan.rows_max
    bounds = 2 * 2 * p.d_k * 8 * BH * max(P - 1, 0)
    gather = (P - 1) * BH * rows * (8 + 4 + 4 * p.d_k + 4 * p.d_v)
    reduce = (P - 1) * BH * rows * 4 * (p.d_k + p.d_v) if backward else 0
    return {"bounds": bounds, "gather_runs_rows": gather, "reduce_partials": reduce,
            "total": bounds + gather + reduce + (8 * (P - 1) if backward else 0)}


# ---------------------------------------------------------------- one process per rank (torch.distributed)
def run_dist(gen, plan: ShardPlan, group=None, combine=None):
    """Drive this rank's step() generator with torch.distributed collectives.

    combine(parts [world, ...]) -> [...] is the rank-ordered sum of the
    partial rows; default onedf_rank_sum (CUDA).  Tests on gloo/CPU inject
    their own.  NCCL min/max all-reduces are exact, so the bounds, codes and
    runs are bitwise identical on every rank."""
    combine = combine or api.rank_sum
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    reply = None
    try:
        req = next(gen)
        while True:
            kind, payload = req
            if kind == "allreduce_minmax":
                lo = payload[..., 0, :].contiguous()
                hi = payload[..., 1, :].contiguous()
                dist.all_reduce(lo, op=dist.ReduceOp.MIN, group=group)
                dist.all_reduce(hi, op=dist.ReduceOp.MAX, group=group)
                reply = torch.stack([lo, hi], dim=-2)
            elif kind == "gather_rows":
                for x in payload:
                    send = plan.pack(x, rank).contiguous()
                    recv = send.new_empty((world * send.shape[0],) + tuple(send.shape[1:]))
                    dist.all_gather_into_tensor(recv, send, group=group)      # concatenated along dim 0
                    recv = recv.view((world,) + tuple(send.shape))
                    for s in range(world):
                        if s != rank:
                            plan.unpack(x, s, recv[s])
                reply = None
            elif kind == "reduce_rows":
                for x in payload:
                    send = torch.stack([plan.pack(x, s) for s in range(world)]).contiguous()
                    recv = torch.empty_like(send)
                    dist.all_to_all_single(recv, send, group=group)     # recv[r] = rank r's partial of my rows
                    plan.unpack(x, rank, combine(recv))
                reply = None
            elif kind == "sum_scalar":
                parts = [torch.empty_like(payload) for _ in range(world)]
                dist.all_gather(parts, payload.contiguous(), group=group)
                reply = _rank_order_sum(parts)
            else:
                raise ValueError(kind)
            req = gen.send(reply)
    except StopIteration as e:
        return e.value
