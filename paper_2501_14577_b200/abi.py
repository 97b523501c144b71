"""ctypes binding of libonedf.so -- argument marshalling only.

Every function here has the same name and argument order as the C entry
point in ``include/onedf.h``; tensors are passed as raw device pointers and
the stream defaults to torch's current stream.  There is no fallback: if the
shared library is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# ONEDF_LIB: load an alternative build of the same library (tools/ variant timing only)
LIB_PATH = os.environ.get("ONEDF_LIB") or os.path.join(_PKG, "libonedf.so")

OK, ERR_INVALID_ARG, ERR_UNSUPPORTED, ERR_CUDA, ERR_NONFINITE, ERR_WORKSPACE = range(6)
OP_ENCODE, OP_SORT, OP_FWD, OP_BWD, OP_STEP_HOST = range(5)
SCORE_CAUCHY, SCORE_NEG_EUCLID, SCORE_INV_EUCLID, SCORE_DOT = range(4)
SELECT_EUCLID, SELECT_CODE = range(2)
DTYPE_F32, DTYPE_BF16 = range(2)


class OnedfError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: onedf status {status} ({status_string(status)})")


class Problem(ctypes.Structure):
    """Mirror of ``onedf_problem`` (include/onedf.h)."""
    _fields_ = [("B", ctypes.c_int64), ("H", ctypes.c_int64), ("N", ctypes.c_int64),
                ("d_k", ctypes.c_int32), ("d_v", ctypes.c_int32), ("k", ctypes.c_int32),
                ("window", ctypes.c_int32), ("chunk", ctypes.c_int32), ("bits", ctypes.c_int32),
                ("causal", ctypes.c_int32), ("mean_slot", ctypes.c_int32),
                ("shard_rank", ctypes.c_int32), ("shard_world", ctypes.c_int32), ("score", ctypes.c_int32),
                ("select", ctypes.c_int32), ("vdtype", ctypes.c_int32)]

    def __repr__(self):
        return "Problem(" + ", ".join(f"{n}={getattr(self, n)}" for n, _ in self._fields_) + ")"

    @property
    def BH(self) -> int:
        return self.B * self.H

    @property
    def W(self) -> int:
        return self.window or 2 * self.k


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libonedf.so not built at {LIB_PATH}; run __graft_entry__.build()")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER(Problem)
    vp, sz, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int
    sig = {
        "onedf_validate": (i32, [P]),
        "onedf_max_run_length": (ctypes.c_int64, []),
        "onedf_workspace_size": (sz, [P, i32]),
        "onedf_encode": (i32, [P, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "onedf_sort": (i32, [P, vp, vp, vp, vp, sz, vp]),
        "onedf_topk_attn_fwd": (i32, [P, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "onedf_topk_attn_bwd": (i32, [P, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz,
                                      vp]),
        "onedf_topk_attn_fwd_traced": (i32, [P, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp, i32,
                                             vp]),
        "onedf_topk_attn_bwd_traced": (i32, [P, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp,
                                             vp, sz, vp, i32, vp]),
        "onedf_means_floats": (ctypes.c_int64, [P]),
        "onedf_topk_attn_step_host": (i32, [P, vp, vp, vp, ctypes.c_float, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "onedf_project_encode": (i32, [P, ctypes.c_int32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz,
                                       vp]),
        "onedf_project_workspace_size": (sz, [P, ctypes.c_int32]),
        "onedf_project_bwd": (i32, [P, ctypes.c_int32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]),
        "onedf_shard_owner": (ctypes.c_int32, [ctypes.c_int64, ctypes.c_int32]),
        "onedf_bounds_partial": (i32, [P, vp, vp, vp, vp, sz, vp]),
        "onedf_bounds_finish": (i32, [P, vp, vp, sz, vp]),
        "onedf_rank_sum": (i32, [vp, ctypes.c_int64, ctypes.c_int32, vp, vp]),
        "onedf_code_knn": (i32, [P, vp, vp, vp, ctypes.c_int32, vp, vp]),
        "onedf_overlap": (i32, [vp, ctypes.c_int32, vp, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, vp, vp]),
        "onedf_check_device_status": (i32, [vp, vp]),
        "onedf_status_string": (ctypes.c_char_p, [i32]),
        "onedf_version": (i32, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


_lib = _load()
EXPORTS = ("onedf_validate", "onedf_max_run_length", "onedf_means_floats", "onedf_workspace_size", "onedf_encode", "onedf_sort",
           "onedf_topk_attn_fwd", "onedf_topk_attn_bwd", "onedf_topk_attn_fwd_traced",
           "onedf_topk_attn_bwd_traced", "onedf_topk_attn_step_host",
           "onedf_project_encode", "onedf_project_workspace_size", "onedf_project_bwd",
           "onedf_shard_owner", "onedf_bounds_partial", "onedf_bounds_finish", "onedf_rank_sum",
           "onedf_code_knn", "onedf_overlap",
           "onedf_check_device_status", "onedf_status_string", "onedf_version")


def lib():
    return _lib


def status_string(s: int) -> str:
    return _lib.onedf_status_string(s).decode()


def _p(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return stream


def _check(st: int, where: str):
    if st != OK:
        raise OnedfError(st, where)


def onedf_validate(p: Problem) -> int:
    return _lib.onedf_validate(ctypes.byref(p))


def onedf_means_floats(p) -> int:
    """Floats of the prefix-means buffer (Kbar then Vbar) that the fwd can hand to the bwd."""
    return int(_lib.onedf_means_floats(ctypes.byref(p)))


def onedf_max_run_length() -> int:
    return _lib.onedf_max_run_length()


def onedf_workspace_size(p: Problem, op: int) -> int:
    return _lib.onedf_workspace_size(ctypes.byref(p), op)


def onedf_encode(p, Q, K, lohi_in, qcode, kcode, lohi_out, ws, ws_bytes, stream=None):
    _check(_lib.onedf_encode(ctypes.byref(p), _p(Q), _p(K), _p(lohi_in), _p(qcode), _p(kcode), _p(lohi_out),
                             _p(ws), ws_bytes, _stream(stream)), "onedf_encode")


def onedf_sort(p, kcode, scode, perm, ws, ws_bytes, stream=None):
    """scode may be None (only perm is written): onedf_sort of the query codes is the query schedule."""
    _check(_lib.onedf_sort(ctypes.byref(p), _p(kcode), _p(scode), _p(perm), _p(ws), ws_bytes, _stream(stream)),
           "onedf_sort")


def onedf_topk_attn_fwd(p, Q, K, V, eps, qcode, scode, perm, qorder, O, idx, Z, ws, ws_bytes, stream=None,
                        indeg=None, means=None):
    """qorder is a nullable scheduling hint (onedf_sort of the query codes); outputs do not depend on it.
    indeg: nullable [B,H,N] int32 output, the keys' in-degree counts for onedf_topk_attn_bwd;
    means: nullable f32 output of onedf_means_floats(p) floats, the prefix means for the backward."""
    _check(_lib.onedf_topk_attn_fwd(ctypes.byref(p), _p(Q), _p(K), _p(V), _p(eps), _p(qcode), _p(scode), _p(perm),
                                    _p(qorder), _p(O), _p(idx), _p(Z), _p(indeg), _p(means), _p(ws), ws_bytes,
                                    _stream(stream)),
           "onedf_topk_attn_fwd")


def onedf_topk_attn_bwd(p, Q, K, V, eps, O, dO, idx, Z, qcode, qorder, perm, dQ, dK, dV, d_eps, ws, ws_bytes,
                        stream=None, indeg=None, means=None):
    """qcode/qorder/perm are nullable scheduling hints (None -> natural order); outputs do not depend on them.
    indeg: nullable, the forward's in-degree counts for this idx (skips the counting pass);
    means: nullable, the forward's prefix means of the same K, V (skips recomputing them)."""
    _check(_lib.onedf_topk_attn_bwd(ctypes.byref(p), _p(Q), _p(K), _p(V), _p(eps), _p(O), _p(dO), _p(idx), _p(Z),
                                    _p(qcode), _p(qorder), _p(perm), _p(indeg), _p(means), _p(dQ), _p(dK), _p(dV),
                                    _p(d_eps), _p(ws), ws_bytes, _stream(stream)),
           "onedf_topk_attn_bwd")


def _events(events):
    arr = (ctypes.c_void_p * max(1, len(events)))(*[e.cuda_event if e is not None else None for e in events])
    return arr, len(events)


def onedf_topk_attn_fwd_traced(p, Q, K, V, eps, qcode, scode, perm, qorder, O, idx, Z, ws, ws_bytes, events,
                               stream=None, indeg=None, means=None):
    arr, n = _events(events)
    _check(_lib.onedf_topk_attn_fwd_traced(ctypes.byref(p), _p(Q), _p(K), _p(V), _p(eps), _p(qcode), _p(scode),
                                           _p(perm), _p(qorder), _p(O), _p(idx), _p(Z), _p(indeg), _p(means), _p(ws),
                                           ws_bytes, arr, n, _stream(stream)), "onedf_topk_attn_fwd_traced")


def onedf_topk_attn_bwd_traced(p, Q, K, V, eps, O, dO, idx, Z, qcode, qorder, perm, dQ, dK, dV, d_eps, ws,
                               ws_bytes, events, stream=None, indeg=None, means=None):
    arr, n = _events(events)
    _check(_lib.onedf_topk_attn_bwd_traced(ctypes.byref(p), _p(Q), _p(K), _p(V), _p(eps), _p(O), _p(dO), _p(idx),
                                           _p(Z), _p(qcode), _p(qorder), _p(perm), _p(indeg), _p(means), _p(dQ),
                                           _p(dK), _p(dV), _p(d_eps), _p(ws), ws_bytes, arr, n, _stream(stream)),
           "onedf_topk_attn_bwd_traced")


def onedf_topk_attn_step_host(p, Q_h, K_h, V_h, eps: float, dO_h, O_h, dQ_h, dK_h, dV_h, d_eps_h, ws, ws_bytes,
                              stream=None):
    _check(_lib.onedf_topk_attn_step_host(ctypes.byref(p), _p(Q_h), _p(K_h), _p(V_h), float(eps), _p(dO_h), _p(O_h),
                                          _p(dQ_h), _p(dK_h), _p(dV_h), _p(d_eps_h), _p(ws), ws_bytes,
                                          _stream(stream)),
           "onedf_topk_attn_step_host")


def onedf_project_encode(p, d_model: int, X, Wq, Wk, bq, bk, theta, lohi_in, Q, K, eps, qcode, kcode, lohi_out, ws,
                         ws_bytes, stream=None):
    _check(_lib.onedf_project_encode(ctypes.byref(p), d_model, _p(X), _p(Wq), _p(Wk), _p(bq), _p(bk), _p(theta),
                                     _p(lohi_in), _p(Q), _p(K), _p(eps), _p(qcode), _p(kcode), _p(lohi_out), _p(ws),
                                     ws_bytes, _stream(stream)), "onedf_project_encode")


def onedf_project_workspace_size(p: Problem, d_model: int) -> int:
    return _lib.onedf_project_workspace_size(ctypes.byref(p), d_model)


def onedf_project_bwd(p, d_model: int, X, Wq, Wk, theta, dQ, dK, d_eps, dX, dWq, dWk, dbq, dbk, dtheta, ws, ws_bytes,
                      stream=None):
    _check(_lib.onedf_project_bwd(ctypes.byref(p), d_model, _p(X), _p(Wq), _p(Wk), _p(theta), _p(dQ), _p(dK),
                                  _p(d_eps), _p(dX), _p(dWq), _p(dWk), _p(dbq), _p(dbk), _p(dtheta), _p(ws), ws_bytes,
                                  _stream(stream)), "onedf_project_bwd")


def onedf_shard_owner(chunk: int, world: int) -> int:
    return _lib.onedf_shard_owner(chunk, world)


def onedf_bounds_partial(p, Q, K, lohi, ws, ws_bytes, stream=None):
    _check(_lib.onedf_bounds_partial(ctypes.byref(p), _p(Q), _p(K), _p(lohi), _p(ws), ws_bytes, _stream(stream)),
           "onedf_bounds_partial")


def onedf_bounds_finish(p, lohi, ws, ws_bytes, stream=None):
    _check(_lib.onedf_bounds_finish(ctypes.byref(p), _p(lohi), _p(ws), ws_bytes, _stream(stream)),
           "onedf_bounds_finish")


def onedf_rank_sum(parts, n: int, world: int, out, stream=None):
    _check(_lib.onedf_rank_sum(_p(parts), n, world, _p(out), _stream(stream)), "onedf_rank_sum")


def onedf_code_knn(p, qcode, scode, perm, exclude_self: bool, idx, stream=None):
    _check(_lib.onedf_code_knn(ctypes.byref(p), _p(qcode), _p(scode), _p(perm), int(bool(exclude_self)), _p(idx),
                               _stream(stream)), "onedf_code_knn")


def onedf_overlap(a, ka: int, b, kb: int, rows: int, self_period: int, counts, stream=None):
    _check(_lib.onedf_overlap(_p(a), ka, _p(b), kb, rows, self_period, _p(counts), _stream(stream)), "onedf_overlap")


def onedf_check_device_status(ws, stream=None) -> int:
    return _lib.onedf_check_device_status(_p(ws), _stream(stream))


def onedf_version() -> int:
    return _lib.onedf_version()
