"""CPU oracle for the ZETA causal top-k attention hot path (arXiv 2501.14577).

TEST INFRASTRUCTURE ONLY.  Importable from ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs -- nowhere else.
The product package ``paper_2501_14577_b200`` never imports this module and
this module never imports the product package; the two share no code.

This is a thin ctypes marshalling layer over ``onedf_oracle.c`` (plain f64 C,
one function per step of the method, each citing the PAPER.md passage it
follows).  Arrays are numpy, C-contiguous, shaped ``[B, H, N, width]``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "onedf_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboref.so")

OK, ERR_INVALID_ARG, ERR_NONFINITE = 0, 1, 4


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (f64, -ffp-contract=off, no fast-math, OpenMP)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", _SRC, "-o", _LIB_PATH + ".tmp", "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(_LIB_PATH + ".tmp", _LIB_PATH)
    return _LIB_PATH


class _Problem(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int64), ("H", ctypes.c_int64), ("N", ctypes.c_int64),
                ("d_k", ctypes.c_int32), ("d_v", ctypes.c_int32), ("k", ctypes.c_int32),
                ("window", ctypes.c_int32), ("chunk", ctypes.c_int32), ("bits", ctypes.c_int32),
                ("causal", ctypes.c_int32), ("mean_slot", ctypes.c_int32), ("score", ctypes.c_int32),
                ("select", ctypes.c_int32)]


@dataclass
class Problem:
    B: int
    H: int
    N: int
    d_k: int
    d_v: int
    k: int
    window: int = 0        # 0 -> 2k (reading D1)
    chunk: int = 1
    bits: int = 0          # 0 -> min(63 // d_k, 32) (reading D11)
    causal: int = 1
    mean_slot: int = 1
    score: int = 0         # 0 Cauchy (Eq. 5); 1 neg-Euclidean exp, 2 inverse Euclidean, 3 dot product (D24)
    select: int = 0        # 0 Euclidean top-k of the windows (D5); 1 SPEC's code-distance merge (D25)

    @property
    def BH(self) -> int:
        return self.B * self.H

    @property
    def W(self) -> int:
        return self.window or 2 * self.k

    @property
    def b(self) -> int:
        return self.bits or min(63 // self.d_k, 32)

    def c(self) -> _Problem:
        return _Problem(self.B, self.H, self.N, self.d_k, self.d_v, self.k, self.window, self.chunk,
                        self.bits, self.causal, self.mean_slot, self.score, self.select)

    def slice(self, n_bh: int) -> "Problem":
        return Problem(1, n_bh, self.N, self.d_k, self.d_v, self.k, self.window, self.chunk, self.bits,
                       self.causal, self.mean_slot, self.score, self.select)


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.POINTER(_Problem)
        vp = ctypes.c_void_p
        sig = {
            "oref_default_bits": (ctypes.c_int, [ctypes.c_int]),
            "oref_fit_bounds": (ctypes.c_int, [P, vp, vp, vp]),
            "oref_quantize": (ctypes.c_uint64, [ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_int]),
            "oref_interleave": (ctypes.c_uint64, [vp, ctypes.c_int, ctypes.c_int]),
            "oref_deinterleave": (None, [ctypes.c_uint64, ctypes.c_int, ctypes.c_int, vp]),
            "oref_encode": (ctypes.c_int, [P, vp, vp, vp, vp, vp, vp]),
            "oref_sort": (ctypes.c_int, [P, vp, vp, vp]),
            "oref_insertion_point": (ctypes.c_int64, [vp, ctypes.c_int64, ctypes.c_uint64]),
            "oref_window_span": (None, [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, vp, vp]),
            "oref_select": (ctypes.c_int, [P, vp, vp, vp, vp, vp, vp, ctypes.c_int64, vp]),
            "oref_forward": (ctypes.c_int, [P, vp, vp, vp, ctypes.c_double, vp, vp, vp, ctypes.c_int64, vp]),
            "oref_backward": (ctypes.c_int, [P, vp, vp, vp, ctypes.c_double, vp, vp, vp, vp, vp, vp]),
            "oref_bruteforce_knn": (ctypes.c_int, [P, vp, vp, vp]),
            "oref_forward_score": (ctypes.c_int, [P, vp, vp, vp, vp, vp, vp]),
            "oref_code_knn": (ctypes.c_int, [P, vp, vp, ctypes.c_int, vp]),
            "oref_select_code": (ctypes.c_int, [P, vp, vp, vp, vp]),
            "oref_backward_score": (ctypes.c_int, [P, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
            "oref_num_threads": (ctypes.c_int, []),
        }
        for name, (res, args) in sig.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


class OracleError(RuntimeError):
    pass


def _check(st):
    if st != OK:
        raise OracleError(f"oracle status {st}")


def num_threads() -> int:
    return lib().oref_num_threads()


def default_bits(d_k: int) -> int:
    return lib().oref_default_bits(d_k)


def quantize(x: float, lo: float, hi: float, b: int) -> int:
    return int(lib().oref_quantize(float(x), float(lo), float(hi), int(b)))


def interleave(g, d: int, b: int) -> int:
    arr = _c(np.asarray(g, dtype=np.uint64).reshape(-1), np.uint64)
    return int(lib().oref_interleave(_ptr(arr), d, b))


def deinterleave(code: int, d: int, b: int):
    out = np.zeros(d, dtype=np.uint64)
    lib().oref_deinterleave(ctypes.c_uint64(code), d, b, _ptr(out))
    return [int(x) for x in out]


def insertion_point(run, qcode: int) -> int:
    arr = _c(np.asarray(run, dtype=np.uint64), np.uint64)
    return int(lib().oref_insertion_point(_ptr(arr), arr.size, ctypes.c_uint64(qcode)))


def window_span(p_ins: int, length: int, W: int):
    s = ctypes.c_int64()
    w = ctypes.c_int64()
    lib().oref_window_span(p_ins, length, W, ctypes.byref(s), ctypes.byref(w))
    return s.value, w.value


def fit_bounds(p: Problem, Q, K):
    Q = _c(Q, np.float32); K = _c(K, np.float32)
    lohi = np.zeros((p.B, p.H, 2, p.d_k), dtype=np.float64)
    _check(lib().oref_fit_bounds(ctypes.byref(p.c()), _ptr(Q), _ptr(K), _ptr(lohi)))
    return lohi


def encode(p: Problem, Q, K, lohi=None):
    Q = _c(Q, np.float32); K = _c(K, np.float32)
    qcode = np.zeros((p.B, p.H, p.N), dtype=np.uint64)
    kcode = np.zeros((p.B, p.H, p.N), dtype=np.uint64)
    lohi_out = np.zeros((p.B, p.H, 2, p.d_k), dtype=np.float64)
    lin = None if lohi is None else _c(lohi, np.float64)
    _check(lib().oref_encode(ctypes.byref(p.c()), _ptr(Q), _ptr(K), _ptr(lin), _ptr(qcode), _ptr(kcode),
                             _ptr(lohi_out)))
    return qcode, kcode, lohi_out


def sort(p: Problem, kcode):
    kcode = _c(kcode, np.uint64)
    scode = np.zeros((p.B, p.H, p.N), dtype=np.uint64)
    perm = np.zeros((p.B, p.H, p.N), dtype=np.int32)
    _check(lib().oref_sort(ctypes.byref(p.c()), _ptr(kcode), _ptr(scode), _ptr(perm)))
    return scode, perm


def _sel(sel):
    if sel is None:
        return 0, None
    s = _c(np.asarray(sel, dtype=np.int64).reshape(-1), np.int64)
    return s.size, s


def select(p: Problem, Q, K, qcode, scode, perm, sel=None):
    """Top-k index sets; all queries -> [B,H,N,k], else [len(sel), k] for flat ids bh*N+i."""
    Q = _c(Q, np.float32); K = _c(K, np.float32)
    qcode = _c(qcode, np.uint64); scode = _c(scode, np.uint64); perm = _c(perm, np.int32)
    if p.select:
        # SPEC's code-distance merge (D25): all queries
        assert sel is None, "code-distance selection: all queries only"
        idx = np.zeros((p.B, p.H, p.N, p.k), dtype=np.int32)
        _check(lib().oref_select_code(ctypes.byref(p.c()), _ptr(qcode), _ptr(scode), _ptr(perm), _ptr(idx)))
        return idx
    n, s = _sel(sel)
    shape = (p.B, p.H, p.N, p.k) if s is None else (n, p.k)
    idx = np.zeros(shape, dtype=np.int32)
    _check(lib().oref_select(ctypes.byref(p.c()), _ptr(Q), _ptr(K), _ptr(qcode), _ptr(scode), _ptr(perm),
                             _ptr(idx), n, _ptr(s)))
    return idx


def forward(p: Problem, Q, K, V, eps: float, idx, sel=None):
    Q = _c(Q, np.float32); K = _c(K, np.float32); V = _c(V, np.float32); idx = _c(idx, np.int32)
    if p.score:
        # score variants (D24): all queries; eps unused
        assert sel is None, "score variants: all queries only"
        O = np.zeros((p.B, p.H, p.N, p.d_v), dtype=np.float64)
        Z = np.zeros((p.B, p.H, p.N), dtype=np.float64)
        _check(lib().oref_forward_score(ctypes.byref(p.c()), _ptr(Q), _ptr(K), _ptr(V), _ptr(idx), _ptr(O), _ptr(Z)))
        return O, Z
    n, s = _sel(sel)
    if s is None:
        O = np.zeros((p.B, p.H, p.N, p.d_v), dtype=np.float64)
        Z = np.zeros((p.B, p.H, p.N), dtype=np.float64)
    else:
        O = np.zeros((n, p.d_v), dtype=np.float64)
        Z = np.zeros((n,), dtype=np.float64)
    _check(lib().oref_forward(ctypes.byref(p.c()), _ptr(Q), _ptr(K), _ptr(V), float(eps), _ptr(idx), _ptr(O),
                              _ptr(Z), n, _ptr(s)))
    return O, Z


def backward(p: Problem, Q, K, V, eps: float, idx, dO):
    Q = _c(Q, np.float32); K = _c(K, np.float32); V = _c(V, np.float32)
    idx = _c(idx, np.int32); dO = _c(dO, np.float32)
    dQ = np.zeros((p.B, p.H, p.N, p.d_k), dtype=np.float64)
    dK = np.zeros((p.B, p.H, p.N, p.d_k), dtype=np.float64)
    dV = np.zeros((p.B, p.H, p.N, p.d_v), dtype=np.float64)
    d_eps = ctypes.c_double()
    if p.score:
        _check(lib().oref_backward_score(ctypes.byref(p.c()), _ptr(Q), _ptr(K), _ptr(V), _ptr(idx), _ptr(dO),
                                         _ptr(dQ), _ptr(dK), _ptr(dV), ctypes.byref(d_eps)))
        return dQ, dK, dV, d_eps.value
    _check(lib().oref_backward(ctypes.byref(p.c()), _ptr(Q), _ptr(K), _ptr(V), float(eps), _ptr(idx), _ptr(dO),
                               _ptr(dQ), _ptr(dK), _ptr(dV), ctypes.byref(d_eps)))
    return dQ, dK, dV, d_eps.value


def bruteforce_knn(p: Problem, Q, K):
    Q = _c(Q, np.float32); K = _c(K, np.float32)
    idx = np.zeros((p.B, p.H, p.N, p.k), dtype=np.int32)
    _check(lib().oref_bruteforce_knn(ctypes.byref(p.c()), _ptr(Q), _ptr(K), _ptr(idx)))
    return idx


def code_knn(p: Problem, qcode, kcode, exclude_self: bool = False):
    """k nearest admissible keys by |kcode - qcode| (u64), ties by position (NEXT-3 locality workload)."""
    qcode = _c(qcode, np.uint64); kcode = _c(kcode, np.uint64)
    idx = np.zeros((p.B, p.H, p.N, p.k), dtype=np.int32)
    _check(lib().oref_code_knn(ctypes.byref(p.c()), _ptr(qcode), _ptr(kcode), int(bool(exclude_self)), _ptr(idx)))
    return idx


def pipeline(p: Problem, Q, K, V, eps: float, dO=None, lohi=None):
    """Whole hot path in the paper's order: encode -> sort -> select -> forward (-> backward)."""
    qcode, kcode, lohi_out = encode(p, Q, K, lohi)
    scode, perm = sort(p, kcode)
    idx = select(p, Q, K, qcode, scode, perm)
    O, Z = forward(p, Q, K, V, eps, idx)
    out = dict(qcode=qcode, kcode=kcode, lohi=lohi_out, scode=scode, perm=perm, idx=idx, O=O, Z=Z)
    if dO is not None:
        dQ, dK, dV, d_eps = backward(p, Q, K, V, eps, idx, dO)
        out.update(dQ=dQ, dK=dK, dV=dV, d_eps=d_eps)
    return out
