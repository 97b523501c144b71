"""Tensor-level API over the C ABI: allocation of outputs/workspace with
PyTorch's caching allocator, and the autograd Function.  Every step of the
path runs in libonedf.so's kernels; this file only marshals arguments.
"""
from __future__ import annotations

import functools

import torch

from . import abi
from .abi import Problem


def make_problem(B, H, N, d_k, d_v, k, window=0, chunk=1, bits=0, causal=1, mean_slot=1, shard_rank=0,
                 shard_world=1, score=0, select=0, vdtype=0) -> Problem:
    """vdtype: storage type of V, O, dO, dV -- abi.DTYPE_F32 (0) or abi.DTYPE_BF16 (1) (NEXT-4, reading D26)."""
    p = Problem(B, H, N, d_k, d_v, k, window, chunk, bits, causal, mean_slot, shard_rank, shard_world, score, select,
                vdtype)
    st = abi.onedf_validate(p)
    if st != abi.OK:
        raise abi.OnedfError(st, "onedf_validate")
    return p


def default_chunk(N: int) -> int:
    """Reading D18: M = 256 until that would need more than 32 chunks, then 32 chunks."""
    return 256 if N <= 256 * 32 else -(-N // 32)


FLAG_BYTES = 16          # onedf.h "Errors": one 32-bit flag word per op at the start of a workspace


class Workspace:
    """A reusable 256-B aligned device byte buffer (grown on demand)."""

    def __init__(self, device=None):
        self.device = torch.device(device or "cuda")
        self._buf = None
        self.nbytes = 0

    def get(self, nbytes: int):
        if self._buf is None or self.nbytes < nbytes:
            self._buf = torch.empty(nbytes + 256, dtype=torch.uint8, device=self.device)
            self.nbytes = nbytes
            off = (-self._buf.data_ptr()) % 256
            self._buf[off:off + FLAG_BYTES].zero_()      # the per-op flag words start cleared (onedf.h "Errors")
        off = (-self._buf.data_ptr()) % 256
        return self._buf.data_ptr() + off, self.nbytes


def _ws(p, op, ws):
    need = abi.onedf_workspace_size(p, op)
    if need == 0:
        raise abi.OnedfError(abi.ERR_INVALID_ARG, "onedf_workspace_size")
    ws = ws or Workspace(torch.device("cuda", torch.cuda.current_device()))
    if ws.device.index is not None and ws.device.index != torch.cuda.current_device():
        raise ValueError(f"workspace on {ws.device}, tensors on cuda:{torch.cuda.current_device()}")
    return ws.get(need)


def _dev(t: torch.Tensor, dtype=torch.float32, rows: int | None = None, width: int = 1):
    """A contiguous CUDA tensor of `dtype` holding exactly rows x width elements (rows of `width`
    in the last dimension): the kernels index it as [rows, width], so a smaller tensor would be
    read (or written) out of bounds."""
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != dtype or not t.is_contiguous():
        raise ValueError(f"expected a contiguous CUDA {dtype} tensor, got "
                         f"{getattr(t, 'dtype', type(t))} on {getattr(t, 'device', '?')}")
    if rows is not None and (t.numel() != rows * width or (width > 1 and t.shape[-1] != width)):
        raise ValueError(f"expected {rows} rows of {width} elements, got shape {tuple(t.shape)}")
    return t


def means_floats(p: Problem) -> int:
    """Elements of the f32 prefix-means tensor topk_attn_fwd(means=...) fills (0 without the mean slot)."""
    return abi.onedf_means_floats(p)


def _rows(p: Problem) -> int:
    return p.B * p.H * p.N


def value_dtype(p: Problem) -> torch.dtype:
    """torch dtype of the value rows V, O, dO, dV of a problem (onedf_problem.vdtype)."""
    return torch.bfloat16 if p.vdtype == abi.DTYPE_BF16 else torch.float32


def _on_one_device(fn):
    """Run an entry point with the tensors' device current (torch's current stream of that device,
    and the device the library launches on); all tensor arguments must share one device."""
    @functools.wraps(fn)
    def wrapper(*args, **kw):
        devs = {a.device for a in list(args) + list(kw.values()) if isinstance(a, torch.Tensor)}
        if len(devs) != 1:
            raise ValueError(f"all tensor arguments must be on one CUDA device, got {sorted(map(str, devs))}")
        dev = devs.pop()
        if dev.type != "cuda":
            raise ValueError(f"expected CUDA tensors, got {dev}")
        with torch.cuda.device(dev):
            return fn(*args, **kw)
    return wrapper


@_on_one_device
def encode(p: Problem, Q, K, lohi=None, ws: Workspace | None = None):
    """A1+A2 -> (qcode, kcode, lohi); codes are int64 tensors holding the u64 bit patterns."""
    Q, K = _dev(Q, rows=_rows(p), width=p.d_k), _dev(K, rows=_rows(p), width=p.d_k)
    qcode = torch.empty((p.B, p.H, p.N), dtype=torch.int64, device=Q.device)
    kcode = torch.empty_like(qcode)
    lohi_out = torch.empty((p.B, p.H, 2, p.d_k), dtype=torch.float64, device=Q.device)
    ptr, n = _ws(p, abi.OP_ENCODE, ws)
    lohi = None if lohi is None else _dev(lohi, torch.float64, rows=p.B * p.H * 2, width=p.d_k)
    abi.onedf_encode(p, Q, K, lohi, qcode, kcode, lohi_out, ptr, n)
    return qcode, kcode, lohi_out


@_on_one_device
def bounds_partial(p: Problem, Q, K, ws: Workspace | None = None):
    """Raw per-(b,h) per-dim min/max over the rows this rank owns -> lohi [B,H,2,d_k] f64 (no widening)."""
    Q, K = _dev(Q, rows=_rows(p), width=p.d_k), _dev(K, rows=_rows(p), width=p.d_k)
    lohi = torch.empty((p.B, p.H, 2, p.d_k), dtype=torch.float64, device=Q.device)
    ptr, n = _ws(p, abi.OP_ENCODE, ws)
    abi.onedf_bounds_partial(p, Q, K, lohi, ptr, n)
    return lohi


@_on_one_device
def bounds_finish(p: Problem, lohi, ws: Workspace | None = None):
    """Reading D10 in place (hi == lo -> +-0.5); returns lohi."""
    lohi = _dev(lohi, torch.float64, rows=p.B * p.H * 2, width=p.d_k)
    ptr, n = _ws(p, abi.OP_ENCODE, ws)
    abi.onedf_bounds_finish(p, lohi, ptr, n)
    return lohi


@_on_one_device
def rank_sum(parts):
    """parts [world, ...] f32 -> [...] f32, summed in rank order in f64 (onedf_rank_sum)."""
    parts = _dev(parts)
    out = torch.empty(parts.shape[1:], dtype=torch.float32, device=parts.device)
    abi.onedf_rank_sum(parts, out.numel(), parts.shape[0], out)
    return out


@_on_one_device
def code_knn(p: Problem, qcode, scode, perm, exclude_self: bool = False):
    """NEXT-3: k nearest keys by Morton-code distance (ties by position) -> idx [B,H,N,k] int32."""
    idx = torch.empty((p.B, p.H, p.N, p.k), dtype=torch.int32, device=qcode.device)
    n = _rows(p)
    abi.onedf_code_knn(p, _dev(qcode, torch.int64, rows=n), _dev(scode, torch.int64, rows=n),
                       _dev(perm, torch.int32, rows=n), exclude_self, idx)
    return idx


@_on_one_device
def overlap(a, b, self_period: int = 0):
    """Per row |a ∩ b| (int32 [rows]) of index lists a [..., ka], b [..., kb]; -1 and the row's own
    position (row mod self_period, if > 0) ignored."""
    a, b = _dev(a, torch.int32), _dev(b, torch.int32)
    rows = a.numel() // a.shape[-1]
    counts = torch.empty(a.shape[:-1], dtype=torch.int32, device=a.device)
    abi.onedf_overlap(a, a.shape[-1], b, b.shape[-1], rows, self_period, counts)
    return counts


@_on_one_device
def sort(p: Problem, kcode, ws: Workspace | None = None):
    """A3 -> (scode, perm)."""
    kcode = _dev(kcode, torch.int64, rows=_rows(p))
    scode = torch.empty_like(kcode)
    perm = torch.empty(kcode.shape, dtype=torch.int32, device=kcode.device)
    ptr, n = _ws(p, abi.OP_SORT, ws)
    abi.onedf_sort(p, kcode, scode, perm, ptr, n)
    return scode, perm


@_on_one_device
def query_schedule(p: Problem, qcode, ws: Workspace | None = None):
    """The Morton query schedule: onedf_sort of the query codes (perm only) -> qorder [B,H,N] int32.
    Passing it to topk_attn_fwd and topk_attn_bwd saves each of them sorting qcode."""
    qcode = _dev(qcode, torch.int64, rows=_rows(p))
    qorder = torch.empty(qcode.shape, dtype=torch.int32, device=qcode.device)
    ptr, n = _ws(p, abi.OP_SORT, ws)
    abi.onedf_sort(p, qcode, None, qorder, ptr, n)
    return qorder


@_on_one_device
def topk_attn_fwd(p: Problem, Q, K, V, eps, qcode, scode, perm, ws: Workspace | None = None, qorder=None,
                  indeg=None, means=None):
    """A4-A7 -> (O, idx, Z).  V and O are of value_dtype(p); qorder (optional) is the query schedule
    (query_schedule), which only chooses the visiting order: outputs are bitwise the same without it.
    indeg (optional) is an int32 [B,H,N] tensor the forward fills with the keys' in-degree counts,
    for topk_attn_bwd(indeg=...); means (optional) an f32 tensor of means_floats(p) elements that receives
    the prefix means, for topk_attn_bwd(means=...)."""
    n = _rows(p)
    Q, K = _dev(Q, rows=n, width=p.d_k), _dev(K, rows=n, width=p.d_k)
    V, eps = _dev(V, value_dtype(p), rows=n, width=p.d_v), _dev(eps, rows=1)
    qorder = None if qorder is None else _dev(qorder, torch.int32, rows=n)
    indeg = None if indeg is None else _dev(indeg, torch.int32, rows=n)
    means = None if means is None else _dev(means, rows=abi.onedf_means_floats(p))
    O = torch.empty((p.B, p.H, p.N, p.d_v), dtype=value_dtype(p), device=Q.device)
    idx = torch.empty((p.B, p.H, p.N, p.k), dtype=torch.int32, device=Q.device)
    Z = torch.empty((p.B, p.H, p.N), dtype=torch.float32, device=Q.device)
    ptr, nb = _ws(p, abi.OP_FWD, ws)
    abi.onedf_topk_attn_fwd(p, Q, K, V, eps, _dev(qcode, torch.int64, rows=n), _dev(scode, torch.int64, rows=n),
                            _dev(perm, torch.int32, rows=n), qorder, O, idx, Z, ptr, nb, indeg=indeg,
                            means=means)
    return O, idx, Z


@_on_one_device
def topk_attn_bwd(p: Problem, Q, K, V, eps, O, dO, idx, Z, ws: Workspace | None = None, qcode=None, perm=None,
                  qorder=None, indeg=None, means=None):
    """A8-A12 -> (dQ, dK, dV, d_eps[float64 scalar tensor]); V, O, dO, dV of value_dtype(p).

    qcode/qorder/perm (optional) only choose the visiting order (Morton schedule); the
    outputs are bitwise identical with or without them.  indeg (optional): the counts
    topk_attn_fwd(indeg=...) wrote for this idx -- skips the backward's counting pass; means (optional):
    the prefix means topk_attn_fwd(means=...) wrote for the same K, V -- skips recomputing them."""
    n = _rows(p)
    vt = value_dtype(p)
    Q, K = _dev(Q, rows=n, width=p.d_k), _dev(K, rows=n, width=p.d_k)
    V, O, dO = (_dev(V, vt, rows=n, width=p.d_v), _dev(O, vt, rows=n, width=p.d_v),
                _dev(dO, vt, rows=n, width=p.d_v))
    eps = _dev(eps, rows=1)
    dQ = torch.empty_like(Q)
    dK = torch.empty_like(K)
    dV = torch.empty_like(V)
    d_eps = torch.empty((), dtype=torch.float64, device=Q.device)
    ptr, nb = _ws(p, abi.OP_BWD, ws)
    qcode = None if qcode is None else _dev(qcode, torch.int64, rows=n)
    qorder = None if qorder is None else _dev(qorder, torch.int32, rows=n)
    perm = None if perm is None else _dev(perm, torch.int32, rows=n)
    indeg = None if indeg is None else _dev(indeg, torch.int32, rows=n)
    means = None if means is None else _dev(means, rows=abi.onedf_means_floats(p))
    abi.onedf_topk_attn_bwd(p, Q, K, V, eps, O, dO, _dev(idx, torch.int32, rows=n, width=p.k), _dev(Z, rows=n), qcode,
                            qorder, perm, dQ, dK, dV, d_eps, ptr, nb, indeg=indeg,
                            means=means)
    return dQ, dK, dV, d_eps


@_on_one_device
def project_encode(p: Problem, X, Wq, Wk, bq=None, bk=None, theta=None, lohi=None, ws: Workspace | None = None):
    """NEXT-4: q = Wq[h] x + bq[h], k = Wk[h] x + bk[h] (reading D27) and eps = sigma(theta)
    (P:1361), then the encoder -> (Q, K, eps | None, qcode, kcode, lohi).
    X [B, N, d_model]; Wq, Wk [H, d_k, d_model]; bq, bk [H, d_k] or None; theta a scalar tensor or None."""
    dm = X.shape[-1]
    X = _dev(X, rows=p.B * p.N, width=dm)
    Wq, Wk = _dev(Wq, rows=p.H * p.d_k, width=dm), _dev(Wk, rows=p.H * p.d_k, width=dm)
    bq = None if bq is None else _dev(bq, rows=p.H * p.d_k)
    bk = None if bk is None else _dev(bk, rows=p.H * p.d_k)
    theta = None if theta is None else _dev(theta, rows=1)
    lohi = None if lohi is None else _dev(lohi, torch.float64, rows=p.B * p.H * 2, width=p.d_k)
    Q = torch.empty((p.B, p.H, p.N, p.d_k), dtype=torch.float32, device=X.device)
    K = torch.empty_like(Q)
    eps = torch.empty((), dtype=torch.float32, device=X.device) if theta is not None else None
    qcode = torch.empty((p.B, p.H, p.N), dtype=torch.int64, device=X.device)
    kcode = torch.empty_like(qcode)
    lohi_out = torch.empty((p.B, p.H, 2, p.d_k), dtype=torch.float64, device=X.device)
    ptr, n = _ws(p, abi.OP_ENCODE, ws)
    abi.onedf_project_encode(p, dm, X, Wq, Wk, bq, bk, theta, lohi, Q, K, eps, qcode, kcode, lohi_out, ptr, n)
    return Q, K, eps, qcode, kcode, lohi_out


@_on_one_device
def project_bwd(p: Problem, X, Wq, Wk, dQ, dK, theta=None, d_eps=None, need_dX: bool = True, bias: bool = True,
                ws: Workspace | None = None):
    """Backward of project_encode -> (dX | None, dWq, dWk, dbq | None, dbk | None, dtheta | None)."""
    dm = X.shape[-1]
    X = _dev(X, rows=p.B * p.N, width=dm)
    Wq, Wk = _dev(Wq, rows=p.H * p.d_k, width=dm), _dev(Wk, rows=p.H * p.d_k, width=dm)
    dQ, dK = _dev(dQ, rows=_rows(p), width=p.d_k), _dev(dK, rows=_rows(p), width=p.d_k)
    theta = None if theta is None else _dev(theta, rows=1)
    d_eps = None if d_eps is None else _dev(d_eps, torch.float64, rows=1)
    dX = torch.empty_like(X) if need_dX else None
    dWq, dWk = torch.empty_like(Wq), torch.empty_like(Wk)
    dbq = torch.empty((p.H, p.d_k), dtype=torch.float32, device=X.device) if bias else None
    dbk = torch.empty_like(dbq) if bias else None
    dtheta = torch.empty((), dtype=torch.float32, device=X.device) if theta is not None and d_eps is not None else None
    need = abi.onedf_project_workspace_size(p, dm)
    ws = ws or Workspace(X.device)
    ptr, n = ws.get(need)
    abi.onedf_project_bwd(p, dm, X, Wq, Wk, theta, dQ, dK, d_eps, dX, dWq, dWk, dbq, dbk, dtheta, ptr, n)
    return dX, dWq, dWk, dbq, dbk, dtheta


def check_device_status(ws) -> int:
    """Synchronise and read the workspace's device flags (a Workspace or a raw device pointer)."""
    if isinstance(ws, Workspace):
        if ws._buf is None:
            return abi.OK
        with torch.cuda.device(ws.device):
            return abi.onedf_check_device_status(ws.get(ws.nbytes)[0])
    return abi.onedf_check_device_status(ws)


class ZetaTopkAttention(torch.autograd.Function):
    """o = ZETA(Q, K, V; eps) with gradients to Q, K, V and eps (indices held fixed, D16)."""

    @staticmethod
    def forward(ctx, Q, K, V, eps, p: Problem, check: bool = False):
        ws = Workspace(Q.device)
        qcode, kcode, _ = encode(p, Q, K, ws=ws)
        scode, perm = sort(p, kcode, ws=ws)
        qorder = query_schedule(p, qcode, ws=ws)          # one Morton schedule for both passes
        indeg = torch.empty((p.B, p.H, p.N), dtype=torch.int32, device=Q.device)   # A9 counts for the backward
        O, idx, Z = topk_attn_fwd(p, Q, K, V, eps.reshape(()), qcode, scode, perm, ws=ws, qorder=qorder, indeg=indeg)
        if check:
            _raise_on_flags(ws, "ZetaTopkAttention.forward")
        ctx.save_for_backward(Q, K, V, eps, O, idx, Z, qorder, perm, indeg)
        ctx.p = p
        ctx.check = check
        ctx.mark_non_differentiable(idx)
        return O, idx

    @staticmethod
    def backward(ctx, dO, _didx):
        Q, K, V, eps, O, idx, Z, qorder, perm, indeg = ctx.saved_tensors
        ws = Workspace(Q.device)
        dQ, dK, dV, d_eps = topk_attn_bwd(ctx.p, Q, K, V, eps.reshape(()), O, dO.contiguous(), idx, Z, ws=ws,
                                          qorder=qorder, perm=perm, indeg=indeg)
        if ctx.check:
            _raise_on_flags(ws, "ZetaTopkAttention.backward")
        return dQ, dK, dV, d_eps.to(eps.dtype).reshape(eps.shape), None, None


def _raise_on_flags(ws: Workspace, where: str):
    st = check_device_status(ws)           # synchronises the stream
    if st != abi.OK:
        raise abi.OnedfError(st, where)


class ZetaProjectedAttention(torch.autograd.Function):
    """The attention core of a ZETA layer from token features: x -> (f_q, f_k, sigma) -> top-k
    Cauchy attention over V (NEXT-4 fused front end + the hot path); gradients to X, Wq, Wk, bq,
    bk, theta and V (indices and codes held fixed, D16)."""

    @staticmethod
    def forward(ctx, X, Wq, Wk, bq, bk, theta, V, p: Problem):
        ws = Workspace(X.device)
        Q, K, eps, qcode, kcode, _ = project_encode(p, X, Wq, Wk, bq, bk, theta.reshape(()), ws=ws)
        scode, perm = sort(p, kcode, ws=ws)
        qorder = query_schedule(p, qcode, ws=ws)
        indeg = torch.empty((p.B, p.H, p.N), dtype=torch.int32, device=X.device)
        O, idx, Z = topk_attn_fwd(p, Q, K, V, eps, qcode, scode, perm, ws=ws, qorder=qorder, indeg=indeg)
        ctx.save_for_backward(X, Wq, Wk, theta, V, Q, K, eps, O, idx, Z, qorder, perm, indeg)
        ctx.p = p
        ctx.has_bias = (bq is not None, bk is not None)
        ctx.mark_non_differentiable(idx)
        return O, idx

    @staticmethod
    def backward(ctx, dO, _didx):
        X, Wq, Wk, theta, V, Q, K, eps, O, idx, Z, qorder, perm, indeg = ctx.saved_tensors
        ws = Workspace(X.device)
        dQ, dK, dV, d_eps = topk_attn_bwd(ctx.p, Q, K, V, eps, O, dO.contiguous(), idx, Z, ws=ws, qorder=qorder,
                                          perm=perm, indeg=indeg)
        dX, dWq, dWk, dbq, dbk, dth = project_bwd(ctx.p, X, Wq, Wk, dQ, dK, theta.reshape(()), d_eps, ws=ws)
        return (dX, dWq, dWk, dbq if ctx.has_bias[0] else None, dbk if ctx.has_bias[1] else None,
                dth.to(theta.dtype).reshape(theta.shape), dV, None)


def zeta_projected_attention(X, Wq, Wk, bq, bk, theta, V, p: Problem):
    """O, idx = ZETA attention of V with q, k = f_q(X), f_k(X) and eps = sigma(theta) (NEXT-4)."""
    return ZetaProjectedAttention.apply(X, Wq, Wk, bq, bk, theta, V, p)


def zeta_attention(Q, K, V, eps, p: Problem, check: bool = False):
    """check=True synchronises after the forward and the backward and raises OnedfError if the
    device flagged non-finite Q/K or eps <= 0 (opt-in: it costs a stream synchronisation)."""
    return ZetaTopkAttention.apply(Q, K, V, eps, p, check)


class HostStep:
    """End-to-end call from pinned host buffers (onedf_topk_attn_step_host)."""

    def __init__(self, p: Problem, device=None):
        self.p = p
        self.ws = Workspace(device)
        self.need = abi.onedf_workspace_size(p, abi.OP_STEP_HOST)
        self.ptr, _ = self.ws.get(self.need)

    def __call__(self, Q_h, K_h, V_h, eps: float, dO_h, O_h, dQ_h, dK_h, dV_h, d_eps_h, stream=None):
        abi.onedf_topk_attn_step_host(self.p, Q_h, K_h, V_h, eps, dO_h, O_h, dQ_h, dK_h, dV_h, d_eps_h, self.ptr,
                                      self.need, stream)

    @staticmethod
    def h2d_bytes(p: Problem) -> int:
        ev = value_dtype(p).itemsize
        return p.BH * p.N * (4 * 2 * p.d_k + ev * 2 * p.d_v)

    @staticmethod
    def d2h_bytes(p: Problem) -> int:
        ev = value_dtype(p).itemsize
        return p.BH * p.N * (4 * 2 * p.d_k + ev * 2 * p.d_v) + 8
