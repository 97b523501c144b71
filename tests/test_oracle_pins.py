"""Pins for the CPU oracle: values the paper / SPEC print, closed forms,
invariants, special cases that reduce to textbook or library routines, brute
force on tiny inputs, and central finite differences.  None of these re-types
the oracle's own formula; each would fail on a plausible mistake (dropped
term, wrong sign or index, transposed operand, off-by-one window).
"""
import bisect
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from oracle import Problem

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# --------------------------------------------------------------------------- Morton / Eq. 4
@pytest.mark.parametrize("case", _gold("interleave.json"), ids=lambda c: c["cite"][:20])
def test_interleave_golden(case):
    assert oracle.interleave(case["g"], case["d"], case["b"]) == case["code"]
    assert oracle.deinterleave(case["code"], case["d"], case["b"]) == case["g"]


@pytest.mark.parametrize("d,b", [(1, 4), (2, 1), (2, 3), (2, 4), (3, 2), (3, 4)])
def test_interleave_bijective_and_monotone(d, b):
    """bijection onto [0, 2^(d b)) and coordinatewise monotone (exhaustive)."""
    grid = list(itertools.product(range(2 ** b), repeat=d))
    codes = {g: oracle.interleave(list(g), d, b) for g in grid}
    assert sorted(codes.values()) == list(range(2 ** (d * b)))
    for g in grid:
        assert tuple(oracle.deinterleave(codes[g], d, b)) == g
    if len(grid) <= 256:
        for g, h in itertools.product(grid, repeat=2):
            if all(x <= y for x, y in zip(g, h)):
                assert codes[g] <= codes[h]


@pytest.mark.parametrize("d,b", [(2, 3), (3, 2), (2, 4)])
def test_dyadic_cell_locality(d, b):
    """Consequence of Eq. 4: grid points sharing the top (b-s) bits of every
    coordinate fill exactly the code interval [P*2^(d s), (P+1)*2^(d s))."""
    for s in range(b + 1):
        cells = {}
        for g in itertools.product(range(2 ** b), repeat=d):
            cells.setdefault(tuple(x >> s for x in g), []).append(oracle.interleave(list(g), d, b))
        for prefix, codes in cells.items():
            lo = min(codes)
            assert lo % (2 ** (d * s)) == 0
            assert sorted(codes) == list(range(lo, lo + 2 ** (d * s)))


def test_interleave_d1_identity_and_plane_order():
    rng = np.random.default_rng(1)
    for v in rng.integers(0, 2 ** 32, size=50):
        assert oracle.interleave([int(v)], 1, 32) == int(v)
    # MSB plane of coordinate 0 is the code's top bit (Eq. 4, b_11 first)
    assert oracle.interleave([1 << 20, 0, 0], 3, 21) == 1 << 62
    assert oracle.interleave([0, 1 << 20, 0], 3, 21) == 1 << 61
    assert oracle.interleave([1, 0, 0], 3, 21) == 1 << 2
    assert oracle.interleave([0, 0, 1], 3, 21) == 1


# --------------------------------------------------------------------------- quantiser
@pytest.mark.parametrize("case", _gold("quantize.json"), ids=lambda c: str(c["x"]))
def test_quantize_golden(case):
    assert oracle.quantize(case["x"], case["lo"], case["hi"], case["b"]) == case["g"]


def test_quantize_endpoints_every_b():
    for b in range(1, 33):
        assert oracle.quantize(-1.25, -1.25, 3.5, b) == 0
        assert oracle.quantize(3.5, -1.25, 3.5, b) == 2 ** b - 1


def test_fit_bounds_joint_and_widened():
    """joint min/max over Q and K per dim; a constant column widens by 0.5."""
    p = Problem(1, 1, 3, 2, 4, 1)
    Q = np.array([[[[-1.0, 7.0], [0.0, 7.0], [2.0, 7.0]]]], np.float32)
    K = np.array([[[[0.5, 7.0], [-3.0, 7.0], [1.0, 7.0]]]], np.float32)
    lohi = oracle.fit_bounds(p, Q, K)
    assert lohi[0, 0, 0].tolist() == [-3.0, 6.5]
    assert lohi[0, 0, 1].tolist() == [2.0, 7.5]


def test_encode_d1_order_preserving():
    """for d = 1 sorting codes == sorting the raw values (ties only by quantisation)."""
    rng = np.random.default_rng(2)
    p = Problem(1, 1, 200, 1, 4, 1)
    Q = rng.normal(size=(1, 1, 200, 1)).astype(np.float32)
    K = rng.normal(size=(1, 1, 200, 1)).astype(np.float32)
    qc, kc, _ = oracle.encode(p, Q, K)
    x = np.concatenate([Q.ravel(), K.ravel()])
    c = np.concatenate([qc.ravel(), kc.ravel()])
    o = np.argsort(x, kind="stable")
    assert np.all(np.diff(c[o].astype(np.float64)) >= 0)


def test_encode_rejects_nonfinite_and_bad_bits():
    p = Problem(1, 1, 4, 3, 4, 1)
    Q = np.zeros((1, 1, 4, 3), np.float32)
    K = np.zeros((1, 1, 4, 3), np.float32)
    K[0, 0, 2, 1] = np.nan
    with pytest.raises(oracle.OracleError):
        oracle.encode(p, Q, K)
    with pytest.raises(oracle.OracleError):
        oracle.encode(Problem(1, 1, 4, 3, 4, 1, bits=22), Q, np.zeros_like(Q))


# --------------------------------------------------------------------------- sort
@pytest.mark.parametrize("case", _gold("sort.json"), ids=lambda c: c["cite"][:12])
def test_sort_golden(case):
    p = Problem(1, 1, case["N"], 1, 4, 1, chunk=case["M"])
    scode, perm = oracle.sort(p, np.array(case["codes"], np.uint64).reshape(1, 1, -1))
    assert scode.ravel().tolist() == case["scode"]
    assert perm.ravel().tolist() == case["perm"]


@pytest.mark.parametrize("causal", [1, 0])
def test_sort_matches_python_sorted(causal):
    """Definition: each run sorted by (code, position) == Python's sorted()."""
    rng = np.random.default_rng(3)
    N, M = 300, 64
    codes = rng.integers(0, 40, size=N).astype(np.uint64)   # many duplicates
    p = Problem(1, 1, N, 2, 4, 1, chunk=M, causal=causal)
    scode, perm = oracle.sort(p, codes.reshape(1, 1, N))
    runs = [(s, min(s + M, N)) for s in range(0, N, M)] if causal else [(0, N)]
    for s, e in runs:
        ref = sorted(((int(codes[j]), j) for j in range(s, e)))
        assert [(int(c), int(j)) for c, j in zip(scode.ravel()[s:e], perm.ravel()[s:e])] == ref


# --------------------------------------------------------------------------- candidate windows
@pytest.mark.parametrize("case", _gold("windows.json"), ids=lambda c: c["cite"][:12])
def test_window_golden(case):
    run = case["run"]
    pins = oracle.insertion_point(run, case["qcode"])
    s, w = oracle.window_span(pins, len(run), case["W"])
    assert run[s:s + w] == case["selected"]


def test_insertion_point_is_bisect_left():
    """D3: the insertion point is torch.searchsorted's default 'left' side == bisect_left."""
    rng = np.random.default_rng(4)
    for _ in range(200):
        run = sorted(rng.integers(0, 50, size=int(rng.integers(1, 40))).tolist())
        q = int(rng.integers(0, 55))
        assert oracle.insertion_point(run, q) == bisect.bisect_left(run, q)


def test_window_span_properties():
    for length in range(1, 20):
        for W in range(1, 25):
            for pins in range(0, length + 1):
                s, w = oracle.window_span(pins, length, W)
                assert w == min(W, length) and 0 <= s and s + w <= length
                if W <= length and W // 2 <= pins <= length - (W - W // 2):
                    assert s == pins - W // 2     # centred when not clamped


# --------------------------------------------------------------------------- selection
def _brute_knn_numpy(Q, K, k, M, causal):
    """Textbook brute force: f32 distances in the pinned left-to-right order, (D, j) lexicographic."""
    N, dk = Q.shape
    out = -np.ones((N, k), np.int32)
    for i in range(N):
        lim = (i // M) * M if causal else N
        if lim == 0:
            continue
        t = Q[i][None, :] - K[:lim]
        D = np.zeros(lim, np.float32)
        for d in range(dk):
            D = D + t[:, d] * t[:, d]
        order = np.lexsort((np.arange(lim), D))[:k]
        out[i, :len(order)] = order
    return out


@pytest.mark.parametrize("dk,causal", [(2, 1), (3, 1), (4, 1), (3, 0)])
def test_window_covering_run_equals_bruteforce_knn(dk, causal):
    """W >= M => every admissible key is a candidate => I_i is the exact chunk-causal kNN."""
    rng = np.random.default_rng(5 + dk)
    N, M, k = 96, 16, 6
    p = Problem(1, 1, N, dk, 4, k, window=N if not causal else M, chunk=M, causal=causal)
    Q = rng.normal(size=(1, 1, N, dk)).astype(np.float32)
    K = rng.normal(size=(1, 1, N, dk)).astype(np.float32)
    qc, kc, _ = oracle.encode(p, Q, K)
    sc, pm = oracle.sort(p, kc)
    idx = oracle.select(p, Q, K, qc, sc, pm)
    ref = _brute_knn_numpy(Q[0, 0], K[0, 0], k, M, causal)
    np.testing.assert_array_equal(idx[0, 0], ref)


def test_d1_window_2k_is_exact_knn():
    """S:255 (W = 2k form): in 1-D the k nearest admissible keys are contiguous in sorted
    order around the insertion point, so the 2k window contains them."""
    rng = np.random.default_rng(6)
    for trial in range(10):
        N, M, k = 128, 32, 5
        p = Problem(1, 1, N, 1, 4, k, window=2 * k, chunk=M, causal=1)
        Q = rng.normal(size=(1, 1, N, 1)).astype(np.float32)
        K = rng.normal(size=(1, 1, N, 1)).astype(np.float32)
        qc, kc, _ = oracle.encode(p, Q, K)
        assert len(np.unique(np.concatenate([qc.ravel(), kc.ravel()]))) == 2 * N   # no collisions
        sc, pm = oracle.sort(p, kc)
        idx = oracle.select(p, Q, K, qc, sc, pm)
        ref = _brute_knn_numpy(Q[0, 0], K[0, 0], k, M, 1)
        np.testing.assert_array_equal(idx[0, 0], ref)


@pytest.mark.parametrize("M,W,k", [(1, 2, 2), (4, 8, 3), (16, 4, 4), (7, 10, 9)])
def test_selection_invariants(M, W, k):
    """causality j < floor(i/M) M; |I_i| = min(k, m M) when W >= k; no duplicates;
    entries ascending by (D, j)."""
    rng = np.random.default_rng(7 + M)
    N, dk = 90, 3
    p = Problem(1, 1, N, dk, 4, k, window=W, chunk=M, causal=1)
    Q = rng.normal(size=(1, 1, N, dk)).astype(np.float32)
    K = rng.normal(size=(1, 1, N, dk)).astype(np.float32)
    qc, kc, _ = oracle.encode(p, Q, K)
    sc, pm = oracle.sort(p, kc)
    idx = oracle.select(p, Q, K, qc, sc, pm)[0, 0]
    for i in range(N):
        m = i // M
        sel = [j for j in idx[i] if j >= 0]
        assert all(j < m * M for j in sel)
        assert len(sel) == min(k, m * M)
        assert len(set(sel)) == len(sel)
        assert all(j == -1 for j in idx[i][len(sel):])
        q = Q[0, 0, i]
        D = [np.float32(0) + sum((q - K[0, 0, j]) ** 2, np.float32(0)) for j in sel]
        keys = list(zip(D, sel))
        assert keys == sorted(keys)
    # chunk-0 queries select nothing
    assert np.all(idx[:M] == -1)


# --------------------------------------------------------------------------- Cauchy forward
def _fwd_case(case, dv=3):
    """Construct exact coordinates hitting the golden distances (d_k = 3, q at the origin)."""
    exact = {0.0: (0, 0, 0), 1.0: (1, 0, 0), 1.5: (1, .5, .5), 0.75: (.5, .5, .5)}
    keys = [exact[d] for d in case["D"]]
    n = 1 + len(keys)
    Q = np.zeros((1, 1, n, 3), np.float32)
    K = np.zeros((1, 1, n, 3), np.float32)
    for r, kk in enumerate(keys):
        K[0, 0, 1 + r] = kk
        if r == 1 and case["D"][0] == case["D"][1]:
            K[0, 0, 1 + r] = (-1, -.5, .5)
    rng = np.random.default_rng(8)
    V = rng.normal(size=(1, 1, n, dv)).astype(np.float32)
    k = len(keys)
    idx = -np.ones((1, 1, n, k), np.int32)
    idx[0, 0, 0] = np.arange(1, n)
    p = Problem(1, 1, n, 3, dv, k, chunk=1, mean_slot=0)
    return p, Q, K, V, idx


@pytest.mark.parametrize("case", _gold("cauchy.json"), ids=lambda c: str(c["D"]))
def test_cauchy_golden(case):
    p, Q, K, V, idx = _fwd_case(case)
    O, Z = oracle.forward(p, Q, K, V, case["eps"], idx)
    assert Z[0, 0, 0] == pytest.approx(case["Z"], rel=1e-15)
    expect = sum(a * V[0, 0, 1 + r].astype(np.float64) for r, a in enumerate(case["A"]))
    np.testing.assert_allclose(O[0, 0, 0], expect, rtol=1e-14, atol=1e-15)


def test_cauchy_ratio_law_and_simplex():
    """A_a/A_b = (D_b + eps)/(D_a + eps); weights sum to 1 (constant V -> constant o);
    o in the convex hull of the attended values."""
    rng = np.random.default_rng(9)
    N, dk, dv, k = 40, 3, 5, 6
    p = Problem(1, 1, N, dk, dv, k, window=12, chunk=4, mean_slot=0)
    Q = rng.normal(size=(1, 1, N, dk)).astype(np.float32)
    K = rng.normal(size=(1, 1, N, dk)).astype(np.float32)
    qc, kc, _ = oracle.encode(p, Q, K)
    sc, pm = oracle.sort(p, kc)
    idx = oracle.select(p, Q, K, qc, sc, pm)
    eps = 0.3
    # one-hot values read the weights back out
    for i in (20, 33, 39):
        sel = [j for j in idx[0, 0, i] if j >= 0]
        A = []
        for j in sel:
            V = np.zeros((1, 1, N, dv), np.float32)
            V[0, 0, j, 0] = 1.0
            O, _ = oracle.forward(p, Q, K, V, eps, idx)
            A.append(O[0, 0, i, 0])
        D = [float(np.sum((Q[0, 0, i].astype(np.float64) - K[0, 0, j]) ** 2)) for j in sel]
        assert sum(A) == pytest.approx(1.0, abs=1e-14)
        for a in range(len(sel)):
            for b in range(len(sel)):
                assert A[a] / A[b] == pytest.approx((D[b] + eps) / (D[a] + eps), rel=1e-12)
    V = np.full((1, 1, N, dv), 2.5, np.float32)
    O, _ = oracle.forward(p, Q, K, V, eps, idx)
    active = (idx[0, 0, :, 0] >= 0)
    np.testing.assert_allclose(O[0, 0][active], 2.5, rtol=1e-14)
    V = rng.normal(size=(1, 1, N, dv)).astype(np.float32)
    O, _ = oracle.forward(p, Q, K, V, eps, idx)
    for i in np.nonzero(active)[0]:
        vals = V[0, 0, [j for j in idx[0, 0, i] if j >= 0]]
        assert np.all(O[0, 0, i] <= vals.max(0) + 1e-12) and np.all(O[0, 0, i] >= vals.min(0) - 1e-12)


def _dense_causal_cauchy(Q, K, V, eps):
    """Independent O(N^2) form of S:337/S:379-382: M = 1, k, W >= N => every j < i plus the
    inclusive-prefix-mean slot, softmax_c over all of them."""
    Q = Q.astype(np.float64); K = K.astype(np.float64); V = V.astype(np.float64)
    N = Q.shape[0]
    cnt = np.arange(1, N + 1)[:, None]
    Kb = np.cumsum(K, 0) / cnt
    Vb = np.cumsum(V, 0) / cnt
    D = ((Q[:, None, :] - K[None, :, :]) ** 2).sum(-1)
    S = np.where(np.tril(np.ones((N, N), bool), -1), 1.0 / (D + eps), 0.0)
    Smu = 1.0 / (((Q - Kb) ** 2).sum(-1) + eps)
    Zs = S.sum(1) + Smu
    return (S @ V + Smu[:, None] * Vb) / Zs[:, None], Zs


def test_forward_dense_special_case():
    rng = np.random.default_rng(10)
    N, dk, dv = 48, 3, 7
    p = Problem(1, 1, N, dk, dv, N, window=N, chunk=1, causal=1, mean_slot=1)
    Q = rng.normal(size=(1, 1, N, dk)).astype(np.float32)
    K = rng.normal(size=(1, 1, N, dk)).astype(np.float32)
    V = rng.normal(size=(1, 1, N, dv)).astype(np.float32)
    out = oracle.pipeline(p, Q, K, V, 0.5)
    O_ref, Z_ref = _dense_causal_cauchy(Q[0, 0], K[0, 0], V[0, 0], 0.5)
    np.testing.assert_allclose(out["O"][0, 0], O_ref, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(out["Z"][0, 0], Z_ref, rtol=1e-12)
    assert out["O"][0, 0, 0] == pytest.approx(V[0, 0, 0].astype(np.float64), rel=1e-15)  # N=1 row: mean slot only


def test_noncausal_mean_is_global():
    rng = np.random.default_rng(11)
    N, dk, dv = 20, 2, 3
    p = Problem(1, 1, N, dk, dv, N, window=N, causal=0, mean_slot=1)
    Q = rng.normal(size=(1, 1, N, dk)).astype(np.float32)
    K = rng.normal(size=(1, 1, N, dk)).astype(np.float32)
    V = rng.normal(size=(1, 1, N, dv)).astype(np.float32)
    out = oracle.pipeline(p, Q, K, V, 0.5)
    q, kk, v = (x[0, 0].astype(np.float64) for x in (Q, K, V))
    D = ((q[:, None] - kk[None]) ** 2).sum(-1)
    S = 1.0 / (D + 0.5)
    Smu = 1.0 / (((q - kk.mean(0)) ** 2).sum(-1) + 0.5)
    O_ref = (S @ v + Smu[:, None] * v.mean(0)) / (S.sum(1) + Smu)[:, None]
    np.testing.assert_allclose(out["O"][0, 0], O_ref, rtol=1e-12, atol=1e-13)


# --------------------------------------------------------------------------- backward
def _grid_inputs(rng, shape, step=2.0 ** -12):
    """Values on a 2^-12 grid so that x +- 2^-14 is exact in f32 (finite differences)."""
    return (np.round(rng.normal(size=shape) / step) * step).astype(np.float32)


def _small_problem(causal=1, mean_slot=1, seed=12):
    rng = np.random.default_rng(seed)
    N, dk, dv, k = 16, 3, 8, 4
    p = Problem(1, 1, N, dk, dv, k, window=8, chunk=4, causal=causal, mean_slot=mean_slot)
    Q = _grid_inputs(rng, (1, 1, N, dk))
    K = _grid_inputs(rng, (1, 1, N, dk))
    V = _grid_inputs(rng, (1, 1, N, dv))
    dO = rng.normal(size=(1, 1, N, dv)).astype(np.float32)
    qc, kc, _ = oracle.encode(p, Q, K)
    sc, pm = oracle.sort(p, kc)
    idx = oracle.select(p, Q, K, qc, sc, pm)
    return p, Q, K, V, dO, idx


@pytest.mark.parametrize("causal,mean_slot", [(1, 1), (1, 0), (0, 1)])
def test_backward_matches_central_differences(causal, mean_slot):
    """P:2006-2045 closed forms + mean-slot chain rule vs central FD of L = sum dO.O (I fixed)."""
    p, Q, K, V, dO, idx = _small_problem(causal, mean_slot)
    eps = 0.5
    h = 2.0 ** -14

    def loss(Q_, K_, V_, e):
        O, _ = oracle.forward(p, Q_, K_, V_, e, idx)
        return float(np.sum(O * dO.astype(np.float64)))

    dQ, dK, dV, d_eps = oracle.backward(p, Q, K, V, eps, idx, dO)
    for name, X, G in (("Q", Q, dQ), ("K", K, dK), ("V", V, dV)):
        fd = np.zeros_like(G)
        for pos in np.ndindex(X.shape):
            Xp = X.copy(); Xp[pos] += h
            Xm = X.copy(); Xm[pos] -= h
            args_p = {"Q": Q, "K": K, "V": V}; args_p[name] = Xp
            args_m = {"Q": Q, "K": K, "V": V}; args_m[name] = Xm
            fd[pos] = (loss(args_p["Q"], args_p["K"], args_p["V"], eps)
                       - loss(args_m["Q"], args_m["K"], args_m["V"], eps)) / (2 * h)
        scale = np.abs(G).max()
        np.testing.assert_allclose(G, fd, rtol=1e-5, atol=1e-6 * scale, err_msg=name)
    fd_eps = (loss(Q, K, V, eps + h) - loss(Q, K, V, eps - h)) / (2 * h)
    assert d_eps == pytest.approx(fd_eps, rel=1e-6)


def test_backward_zero_upstream_and_single_slot():
    p, Q, K, V, dO, idx = _small_problem()
    dQ, dK, dV, d_eps = oracle.backward(p, Q, K, V, 0.5, idx, np.zeros_like(dO))
    assert not dQ.any() and not dK.any() and not dV.any() and d_eps == 0.0
    # S:328 single slot: A = 1 => v_j - o_i = 0 => dq_i = 0 and dv_j = dO_i
    p1 = Problem(1, 1, 2, 3, 4, 1, chunk=1, mean_slot=0)
    rng = np.random.default_rng(13)
    Q1 = rng.normal(size=(1, 1, 2, 3)).astype(np.float32)
    K1 = rng.normal(size=(1, 1, 2, 3)).astype(np.float32)
    V1 = rng.normal(size=(1, 1, 2, 4)).astype(np.float32)
    dO1 = rng.normal(size=(1, 1, 2, 4)).astype(np.float32)
    idx1 = np.array([[[[-1], [0]]]], np.int32)
    dQ, dK, dV, d_eps = oracle.backward(p1, Q1, K1, V1, 0.5, idx1, dO1)
    assert np.all(dQ == 0) and np.all(dK == 0) and d_eps == 0.0
    np.testing.assert_array_equal(dV[0, 0, 0], dO1[0, 0, 1].astype(np.float64))


@pytest.mark.parametrize("causal", [1, 0])
def test_backward_invariants(causal):
    """Exact identities for fixed I (derived from Eq. 5): translation sum dq + sum dk = 0;
    sum A = 1 => sum dv = sum dO; degree-0 homogeneity in (q, k, sqrt eps) =>
    sum q.dq + sum k.dk + 2 eps deps = 0."""
    rng = np.random.default_rng(14)
    N, dk, dv, k = 200, 3, 16, 8
    p = Problem(2, 1, N, dk, dv, k, window=16, chunk=25, causal=causal, mean_slot=1)
    Q = rng.normal(size=(2, 1, N, dk)).astype(np.float32)
    K = rng.normal(size=(2, 1, N, dk)).astype(np.float32)
    V = rng.normal(size=(2, 1, N, dv)).astype(np.float32)
    dO = rng.normal(size=(2, 1, N, dv)).astype(np.float32)
    eps = 0.5
    out = oracle.pipeline(p, Q, K, V, eps, dO)
    dQ, dK, dV = out["dQ"], out["dK"], out["dV"]
    np.testing.assert_allclose(dQ.sum(2) + dK.sum(2), 0.0, atol=1e-12)
    np.testing.assert_allclose(dV.sum(2), dO.astype(np.float64).sum(2), atol=1e-11)
    euler = (Q * dQ).sum() + (K * dK).sum() + 2 * eps * out["d_eps"]
    assert abs(euler) < 1e-11 * (np.abs(Q * dQ).sum() + 1)


# --------------------------------------------------------------------------- score variants (NEXT-2, D24)
SCORES = {1: "neg_euclid", 2: "inv_euclid", 3: "dot"}


def _dense_causal_score(Q, K, V, score):
    """Independent O(N^2) forms of SPEC's dense_causal_attention for the variants:
    M = 1, k, W >= N => every j < i plus the inclusive-prefix-mean slot; weights per S:380."""
    Q = Q.astype(np.float64); K = K.astype(np.float64); V = V.astype(np.float64)
    N, dk = Q.shape
    cnt = np.arange(1, N + 1)[:, None]
    Kb = np.cumsum(K, 0) / cnt
    Vb = np.cumsum(V, 0) / cnt
    D = ((Q[:, None, :] - K[None, :, :]) ** 2).sum(-1)
    Dmu = ((Q - Kb) ** 2).sum(-1)
    if score == 1:
        S, Smu = np.exp(-D), np.exp(-Dmu)
    elif score == 2:
        S, Smu = 1.0 / (np.sqrt(D) + 1e-6), 1.0 / (np.sqrt(Dmu) + 1e-6)
    else:
        S, Smu = np.exp(Q @ K.T / np.sqrt(dk)), np.exp((Q * Kb).sum(-1) / np.sqrt(dk))
    S = np.where(np.tril(np.ones((N, N), bool), -1), S, 0.0)
    Zs = S.sum(1) + Smu
    return (S @ V + Smu[:, None] * Vb) / Zs[:, None], Zs


@pytest.mark.parametrize("score", list(SCORES))
def test_score_dense_special_case(score):
    """with M = 1 and k, W >= N every score variant is dense strict-causal attention
    plus the mean slot; Z is sum S (inverse Euclidean) or log sum S (the exponential scores)."""
    rng = np.random.default_rng(20 + score)
    N, dk, dv = 40, 3, 5
    p = Problem(1, 1, N, dk, dv, N, window=N, chunk=1, causal=1, mean_slot=1, score=score)
    Q = rng.normal(size=(1, 1, N, dk)).astype(np.float32)
    K = rng.normal(size=(1, 1, N, dk)).astype(np.float32)
    V = rng.normal(size=(1, 1, N, dv)).astype(np.float32)
    out = oracle.pipeline(p, Q, K, V, 0.5)
    O_ref, Z_ref = _dense_causal_score(Q[0, 0], K[0, 0], V[0, 0], score)
    np.testing.assert_allclose(out["O"][0, 0], O_ref, rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(out["Z"][0, 0], Z_ref if score == 2 else np.log(Z_ref), rtol=1e-12, atol=1e-13)


def test_score_ratio_laws():
    """Closed-form weight ratios, read back with one-hot values: exp(-D) softmax A_a/A_b =
    exp(D_b - D_a); inverse Euclidean A_a/A_b = (sqrt D_b + 1e-6)/(sqrt D_a + 1e-6); dot
    A_a/A_b = exp((q.k_a - q.k_b)/sqrt d_k).  Weights sum to one."""
    rng = np.random.default_rng(21)
    N, dk, dv, k = 40, 3, 4, 6
    Q = rng.normal(size=(1, 1, N, dk)).astype(np.float32)
    K = rng.normal(size=(1, 1, N, dk)).astype(np.float32)
    for score in SCORES:
        p = Problem(1, 1, N, dk, dv, k, window=12, chunk=4, mean_slot=0, score=score)
        qc, kc, _ = oracle.encode(p, Q, K)
        sc, pm = oracle.sort(p, kc)
        idx = oracle.select(p, Q, K, qc, sc, pm)
        i = 37
        sel = [j for j in idx[0, 0, i] if j >= 0]
        A = []
        for j in sel:
            V = np.zeros((1, 1, N, dv), np.float32)
            V[0, 0, j, 0] = 1.0
            O, _ = oracle.forward(p, Q, K, V, 0.5, idx)
            A.append(O[0, 0, i, 0])
        q = Q[0, 0, i].astype(np.float64)
        kk = K[0, 0, sel].astype(np.float64)
        D = ((q - kk) ** 2).sum(-1)
        logit = {1: -D, 2: -np.log(np.sqrt(D) + 1e-6), 3: kk @ q / np.sqrt(dk)}[score]
        assert sum(A) == pytest.approx(1.0, abs=1e-14)
        for a in range(len(sel)):
            for b in range(len(sel)):
                assert A[a] / A[b] == pytest.approx(np.exp(logit[a] - logit[b]), rel=1e-11), (score, a, b)


@pytest.mark.parametrize("score", list(SCORES))
@pytest.mark.parametrize("causal,mean_slot", [(1, 1), (0, 1), (1, 0)])
def test_score_backward_matches_central_differences(score, causal, mean_slot):
    """The variants' chain rule vs central FD of L = sum dO.O with I fixed; d_eps = 0."""
    p, Q, K, V, dO, idx = _small_problem(causal, mean_slot, seed=30 + score)
    p = Problem(p.B, p.H, p.N, p.d_k, p.d_v, p.k, p.window, p.chunk, p.bits, p.causal, p.mean_slot, score)
    h = 2.0 ** -14

    def loss(Q_, K_, V_):
        O, _ = oracle.forward(p, Q_, K_, V_, 0.5, idx)
        return float(np.sum(O * dO.astype(np.float64)))

    dQ, dK, dV, d_eps = oracle.backward(p, Q, K, V, 0.5, idx, dO)
    assert d_eps == 0.0
    for name, X, G in (("Q", Q, dQ), ("K", K, dK), ("V", V, dV)):
        fd = np.zeros_like(G)
        for pos in np.ndindex(X.shape):
            Xp = X.copy(); Xp[pos] += h
            Xm = X.copy(); Xm[pos] -= h
            a_p = {"Q": Q, "K": K, "V": V}; a_p[name] = Xp
            a_m = {"Q": Q, "K": K, "V": V}; a_m[name] = Xm
            fd[pos] = (loss(a_p["Q"], a_p["K"], a_p["V"]) - loss(a_m["Q"], a_m["K"], a_m["V"])) / (2 * h)
        scale = np.abs(G).max()
        np.testing.assert_allclose(G, fd, rtol=1e-5, atol=1e-6 * scale, err_msg=f"{SCORES[score]} {name}")


@pytest.mark.parametrize("score", [1, 2])
def test_score_backward_invariants_distance_scores(score):
    """Distance scores depend on q - k only => sum dq + sum dk = 0 (translation); every score has
    sum A = 1 => sum dv = sum dO."""
    rng = np.random.default_rng(40 + score)
    N, dk, dv, k = 150, 3, 8, 8
    p = Problem(1, 2, N, dk, dv, k, window=16, chunk=25, causal=1, mean_slot=1, score=score)
    Q, K = (rng.normal(size=(1, 2, N, dk)).astype(np.float32) for _ in range(2))
    V, dO = (rng.normal(size=(1, 2, N, dv)).astype(np.float32) for _ in range(2))
    out = oracle.pipeline(p, Q, K, V, 0.5, dO)
    np.testing.assert_allclose(out["dQ"].sum(2) + out["dK"].sum(2), 0.0, atol=1e-11)
    np.testing.assert_allclose(out["dV"].sum(2), dO.astype(np.float64).sum(2), atol=1e-10)


def test_score_dot_invariants():
    """DOT: S depends on q.k only => rotating q and k together leaves O unchanged, and
    sum_i q_i.dq_i = sum_j k_j.dk_j (both equal sum_ij s_ij dL/ds_ij); sum dv = sum dO."""
    rng = np.random.default_rng(44)
    N, dk, dv, k = 150, 3, 8, 8
    p = Problem(1, 1, N, dk, dv, k, window=16, chunk=25, causal=1, mean_slot=1, score=3)
    Q, K = (rng.normal(size=(1, 1, N, dk)).astype(np.float32) for _ in range(2))
    V, dO = (rng.normal(size=(1, 1, N, dv)).astype(np.float32) for _ in range(2))
    out = oracle.pipeline(p, Q, K, V, 0.5, dO)
    lhs = (Q.astype(np.float64) * out["dQ"]).sum()
    rhs = (K.astype(np.float64) * out["dK"]).sum()
    assert lhs == pytest.approx(rhs, rel=1e-10)
    np.testing.assert_allclose(out["dV"].sum(2), dO.astype(np.float64).sum(2), atol=1e-10)
    # 90-degree rotation in the (0,1) plane (exact in f32): same dot products, same O for the same I
    R = np.array([[0, -1, 0], [1, 0, 0], [0, 0, 1]], np.float32)
    O2, _ = oracle.forward(p, Q @ R.T, K @ R.T, V, 0.5, out["idx"])
    np.testing.assert_allclose(O2, out["O"], rtol=1e-13, atol=1e-14)


# --------------------------------------------------------------------------- locality workload (NEXT-3)
def test_code_knn_d1_is_exact_knn():
    """d_K = 1 with fine quantisation and no code collisions -> the code order is the
    value order, so the nearest by |code difference| are the exact nearest (overlap 1)."""
    rng = np.random.default_rng(50)
    N, k = 512, 64
    p = Problem(2, 1, N, 1, 4, k, window=N, causal=0, mean_slot=0)
    X = rng.normal(size=(2, 1, N, 1)).astype(np.float32)
    qc, kc, _ = oracle.encode(p, X, X)
    assert len(np.unique(kc[0, 0])) == N
    got = oracle.code_knn(p, qc, kc, exclude_self=True)
    pk = Problem(2, 1, N, 1, 4, k + 1, window=N, causal=0, mean_slot=0)
    exact = oracle.bruteforce_knn(pk, X, X)
    for b in range(2):
        for i in range(N):
            want = set(exact[b, 0, i]) - {i}
            assert len(want) == k and set(got[b, 0, i]) == want


def test_code_knn_is_a_contiguous_block_of_the_sorted_run():
    """With distinct codes, the k nearest codes to q are a contiguous block of the sorted order
    that contains q's insertion neighbourhood (a consequence of sorting), and their order is
    (|diff|, j); N = k + 1 (self excluded) returns everything else."""
    rng = np.random.default_rng(51)
    N, k = 300, 16
    p = Problem(1, 1, N, 3, 4, k, causal=0, mean_slot=0)
    X = rng.normal(size=(1, 1, N, 3)).astype(np.float32)
    Qx = rng.normal(size=(1, 1, N, 3)).astype(np.float32)
    qc, kc, _ = oracle.encode(p, Qx, X)
    idx = oracle.code_knn(p, qc, kc)
    order = np.argsort(kc[0, 0], kind="stable")
    rank = np.empty(N, np.int64); rank[order] = np.arange(N)
    for i in range(N):
        r = np.sort(rank[idx[0, 0, i]])
        assert r[-1] - r[0] == k - 1
        d = np.array([abs(int(kc[0, 0, j]) - int(qc[0, 0, i])) for j in idx[0, 0, i]])
        assert np.all(np.diff(d) >= 0)
    p2 = Problem(1, 1, k + 1, 3, 4, k, causal=0, mean_slot=0)
    X2 = X[:, :, :k + 1].copy()
    qc2, kc2, _ = oracle.encode(p2, X2, X2)
    got = oracle.code_knn(p2, qc2, kc2, exclude_self=True)
    for i in range(k + 1):
        assert set(got[0, 0, i]) == set(range(k + 1)) - {i}


def test_code_knn_ties_and_causality():
    """Equal codes order by position (D19); causal admissibility j < floor(i/M)*M (D6)."""
    p = Problem(1, 1, 12, 1, 4, 3, chunk=4, causal=1, mean_slot=0)
    kc = np.array([[[5, 5, 5, 9, 1, 5, 5, 0, 2, 2, 2, 2]]], np.uint64)
    qc = np.full((1, 1, 12), 5, np.uint64)
    idx = oracle.code_knn(p, qc, kc)
    assert idx[0, 0, 2].tolist() == [-1, -1, -1]            # chunk 0: nothing admissible
    assert idx[0, 0, 5].tolist() == [0, 1, 2]                # keys 0..3 admissible; d = 0,0,0,4
    assert idx[0, 0, 9].tolist() == [0, 1, 2]                # keys 0..7: five at d = 0, smallest j first
    qc[0, 0, 11] = 2
    assert oracle.code_knn(p, qc, kc)[0, 0, 11].tolist() == [4, 7, 0]   # d = 1 (key 4), 2 (key 7), then 3 (j = 0)


# --------------------------------------------------------------------------- selection variant (NEXT-2, D25)
def test_select_code_spec_examples():
    """SPEC S:230-232 worked examples of query_topk (W = k = 2): run [1,3,5,7], query code 4 in
    chunk 1 -> {3,5}; a query code below a whole run [5,6,9] -> {5,6}; chunk-0 query -> empty."""
    p = Problem(1, 1, 8, 1, 4, 2, window=2, chunk=4, causal=1, mean_slot=0, select=1)
    scode = np.array([[[1, 3, 5, 7, 0, 0, 0, 0]]], np.uint64)
    perm = np.array([[[0, 1, 2, 3, 4, 5, 6, 7]]], np.int32)
    qcode = np.array([[[0, 0, 0, 0, 4, 4, 0, 0]]], np.uint64)
    idx = oracle.select(p, None, None, qcode, scode, perm)
    assert sorted(scode[0, 0, idx[0, 0, 4]].tolist()) == [3, 5]
    assert idx[0, 0, 0].tolist() == [-1, -1]
    p2 = Problem(1, 1, 6, 1, 4, 2, window=2, chunk=3, causal=1, mean_slot=0, select=1)
    idx2 = oracle.select(p2, None, None, np.zeros((1, 1, 6), np.uint64),
                         np.array([[[5, 6, 9, 0, 0, 0]]], np.uint64), np.arange(6, dtype=np.int32)[None, None])
    assert idx2[0, 0, 3].tolist() == [0, 1]                   # codes {5, 6}: window clamped at the run start


def test_select_code_invariants_and_d1_exactness():
    """Causality and |I| = min(k, admissible); the order is (|code difference|, j); S:257 d_K = 1
    with unique codes and a window covering each run -> the exact chunk-causal kNN."""
    rng = np.random.default_rng(60)
    N, k, M = 256, 8, 32
    X = rng.normal(size=(1, 1, N, 1)).astype(np.float32)
    Qx = rng.normal(size=(1, 1, N, 1)).astype(np.float32)
    p = Problem(1, 1, N, 1, 4, k, window=M, chunk=M, causal=1, mean_slot=0, select=1)
    qc, kc, _ = oracle.encode(p, Qx, X)
    sc, pm = oracle.sort(p, kc)
    idx = oracle.select(p, Qx, X, qc, sc, pm)
    exact = oracle.bruteforce_knn(p, Qx, X)
    for i in range(N):
        lim = (i // M) * M
        row = [j for j in idx[0, 0, i] if j >= 0]
        assert len(row) == min(k, lim) and all(j < lim for j in row)
        d = [abs(int(kc[0, 0, j]) - int(qc[0, 0, i])) for j in row]
        assert d == sorted(d)
        assert set(row) == set(j for j in exact[0, 0, i] if j >= 0)


# --------------------------------------------------------------------------- tie rules (D19, D25)
_TIES = _gold("ties.json")


@pytest.mark.parametrize("case", _TIES["euclid"], ids=lambda c: c["cite"][:12])
def test_select_distance_ties_by_position_golden(case):
    """D19: candidates at equal distance are ordered (and cut at k) by ascending position j.
    Hand-worked: every key is a candidate (window covers each run), distances are small exact
    integers / binary fractions, so the expected rows follow from the (D, j) order alone."""
    N, dk = case["N"], case["d_k"]
    Q = np.asarray(case["Q"], np.float32).reshape(1, 1, N, dk)
    K = np.asarray(case["K"], np.float32).reshape(1, 1, N, dk)
    for k, want in case["idx_by_k"].items():
        p = Problem(1, 1, N, dk, 4, int(k), window=case["window"], chunk=case["chunk"], causal=case["causal"])
        qc, kc, _ = oracle.encode(p, Q, K)
        sc, pm = oracle.sort(p, kc)
        idx = oracle.select(p, Q, K, qc, sc, pm)
        assert idx[0, 0, case["query"]].tolist() == want, (k, case["why"])


@pytest.mark.parametrize("case", _TIES["code"], ids=lambda c: c["cite"][:12])
def test_select_code_ties_by_position_golden(case):
    """SPEC S:227/S:263 (reading D25): equal |code - query code| -> smaller source index first,
    across the windows of different runs and within one run (not the sorted-run order)."""
    N = case["N"]
    sc = np.asarray(case["scode"], np.uint64).reshape(1, 1, N)
    pm = np.asarray(case["perm"], np.int32).reshape(1, 1, N)
    qc = np.asarray(case["qcode"], np.uint64).reshape(1, 1, N)
    for k, want in case["idx_by_k"].items():
        p = Problem(1, 1, N, 1, 4, int(k), window=case["window"], chunk=case["chunk"], causal=case["causal"],
                    mean_slot=0, select=1)
        idx = oracle.select(p, None, None, qc, sc, pm)
        assert idx[0, 0, case["query"]].tolist() == want, (k, case["why"])


def test_bruteforce_knn_ties_by_position():
    """The independent brute-force kNN (no Morton) keeps the same (D, j) tie rule (D19)."""
    case = _TIES["euclid"][0]
    N, dk = case["N"], case["d_k"]
    Q = np.asarray(case["Q"], np.float32).reshape(1, 1, N, dk)
    K = np.asarray(case["K"], np.float32).reshape(1, 1, N, dk)
    p = Problem(1, 1, N, dk, 4, 4, window=8, causal=0)
    assert oracle.bruteforce_knn(p, Q, K)[0, 0, 0].tolist() == [0, 2, 3, 5]


# --------------------------------------------------------------------------- reading D23 vs the f64 contract
def _f64_topk_sets(p, Q, K, qc, sc, pm):
    """Independent f64 selection (numpy): the same candidate windows (insertion point by
    bisect on the sorted run, D1-D3), ranked by the f64 squared distance, ties by j."""
    N, M, W, k = p.N, (p.chunk if p.causal else p.N), p.W, p.k
    q64 = Q[0, 0].astype(np.float64)
    k64 = K[0, 0].astype(np.float64)
    sets, kth = [], []
    for i in range(N):
        nruns = i // M if p.causal else 1
        cand = []
        for c in range(nruns):
            s0, ln = c * M, min(M, N - c * M)
            run = [int(x) for x in sc[0, 0, s0:s0 + ln]]
            ins = bisect.bisect_left(run, int(qc[0, 0, i]))
            w = min(W, ln)
            s = min(max(ins - W // 2, 0), ln - w)
            cand += [int(x) for x in pm[0, 0, s0 + s:s0 + s + w]]
        cand = np.array(cand, np.int64)
        if cand.size == 0:
            sets.append(set()); kth.append(None)
            continue
        D = ((k64[cand] - q64[i]) ** 2).sum(axis=1)
        order = np.lexsort((cand, D))
        sets.append(set(cand[order[:k]].tolist()))
        kth.append((D[order[k - 1]], D[order[k]]) if cand.size > k else None)
    return sets, kth


@pytest.mark.parametrize("kind", ["iid", "tokens"])
def test_f32_ranking_equals_f64_ranking_except_near_ties(kind):
    """Reading D23 against the north_star contract: the selected SET taken with the pinned f32
    ranking distance equals the set an f64 ranking gives, except for queries whose f64 k-th and
    (k+1)-th distances agree within 1e-6 relative (north_star's near-tie clause)."""
    rng = np.random.default_rng(77 if kind == "iid" else 78)
    N, dk, k, M, W = 1024, 3, 16, 128, 32
    p = Problem(1, 1, N, dk, 4, k, window=W, chunk=M, causal=1)
    if kind == "iid":
        Q = rng.normal(size=(1, 1, N, dk)).astype(np.float32)
        K = rng.normal(size=(1, 1, N, dk)).astype(np.float32)
    else:   # repeated tokens: exact duplicate keys (distance ties) and near-duplicate queries
        E = rng.normal(size=(64, dk)).astype(np.float32)
        t = rng.integers(0, 64, size=N)
        K = E[t][None, None]
        Q = (E[t] + 0.05 * rng.normal(size=(N, dk))).astype(np.float32)[None, None]
    qc, kc, _ = oracle.encode(p, Q, K)
    sc, pm = oracle.sort(p, kc)
    idx = oracle.select(p, Q, K, qc, sc, pm)[0, 0]
    sets, kth = _f64_topk_sets(p, Q, K, qc, sc, pm)
    differ = 0
    for i in range(N):
        got = set(int(j) for j in idx[i] if j >= 0)
        if got == sets[i]:
            continue
        differ += 1
        a, b = kth[i]
        assert abs(b - a) <= 1e-6 * max(abs(a), abs(b)), (i, a, b)
    assert differ <= N // 50


def test_near_tie_clause_is_where_f32_and_f64_differ():
    """A constructed near-tie: key 0 = (1, 2^-16, 0) is at f64 distance 1 + 2^-32 from q = 0 but at
    f32 distance exactly 1.0 (the 2^-32 is below half an ulp of 1), key 1 = (1, 0, 0) at exactly 1.
    f32 ranking ties them and takes j = 0; f64 ranking takes j = 1.  The north_star clause covers
    exactly this: the f64 k-th and (k+1)-th distances agree within 1e-6 relative."""
    N = 4
    K = np.array([[1, 2.0 ** -16, 0], [1, 0, 0], [5, 0, 0], [0, 6, 0]], np.float32).reshape(1, 1, N, 3)
    Q = np.zeros((1, 1, N, 3), np.float32)
    p = Problem(1, 1, N, 3, 4, 1, window=8, causal=0)
    qc, kc, _ = oracle.encode(p, Q, K)
    sc, pm = oracle.sort(p, kc)
    assert oracle.select(p, Q, K, qc, sc, pm)[0, 0, 0].tolist() == [0]
    sets, kth = _f64_topk_sets(p, Q, K, qc, sc, pm)
    assert sets[0] == {1}
    a, b = kth[0]
    assert a == 1.0 and b == 1.0 + 2.0 ** -32 and abs(b - a) <= 1e-6 * b
