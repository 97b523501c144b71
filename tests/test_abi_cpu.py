"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, the ctypes struct matches the C layout, and every argument
check answers synchronously with the documented status (no GPU needed: all
of these return before any launch)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "onedf.h")


@pytest.fixture(scope="module")
def onedf():
    import __graft_entry__
    __graft_entry__.build_cuda()
    import paper_2501_14577_b200 as m
    return m


def _declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\*?\s+\*?(onedf_[a-z_0-9]+)\s*\(", text, re.M)))


def test_header_declares_the_boundary():
    names = _declared_functions()
    for required in ("onedf_encode", "onedf_sort", "onedf_topk_attn_fwd", "onedf_topk_attn_bwd"):
        assert required in names


def test_library_exports_every_declared_symbol(onedf):
    lib = ctypes.CDLL(onedf.abi.LIB_PATH)
    for name in _declared_functions():
        assert hasattr(lib, name), name
    assert set(onedf.abi.EXPORTS) == set(_declared_functions())
    assert onedf.onedf_version() == 600


def test_struct_layout_matches_c(onedf, tmp_path):
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "onedf.h"\nint main(void){'
                   'printf("%zu", sizeof(onedf_problem));'
                   + "".join(f'printf(" %zu", offsetof(onedf_problem, {f}));' for f, _ in onedf.Problem._fields_)
                   + "return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    vals = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert vals[0] == ctypes.sizeof(onedf.Problem)
    assert vals[1:] == [getattr(onedf.Problem, f).offset for f, _ in onedf.Problem._fields_]


GOOD = dict(B=2, H=3, N=1000, d_k=3, d_v=64, k=32, window=64, chunk=128, bits=0, causal=1, mean_slot=1)


@pytest.mark.parametrize("field,value", [
    ("d_k", 0), ("d_k", 9), ("d_v", 0), ("d_v", 6), ("d_v", 260), ("k", 0), ("k", 257), ("window", 16),
    ("chunk", 0), ("bits", 22), ("bits", 33), ("causal", 2), ("mean_slot", -1), ("N", 0), ("B", 0),
])
def test_validate_rejects(onedf, field, value):
    kw = dict(GOOD)
    kw[field] = value
    p = onedf.Problem(*kw.values())
    assert onedf.onedf_validate(p) == onedf.abi.ERR_INVALID_ARG
    assert onedf.onedf_workspace_size(p, onedf.OP_FWD) == 0


@pytest.mark.parametrize("rank,world,causal,want", [
    (1, 1, 1, "ERR_INVALID_ARG"), (2, 2, 1, "ERR_INVALID_ARG"), (-1, 2, 1, "ERR_INVALID_ARG"),
    (0, -1, 1, "ERR_INVALID_ARG"), (0, 2, 0, "ERR_UNSUPPORTED"), (1, 2, 1, "OK"), (7, 8, 1, "OK"), (0, 0, 1, "OK"),
])
def test_validate_shard_fields(onedf, rank, world, causal, want):
    p = onedf.Problem(*dict(GOOD, causal=causal).values(), rank, world)
    assert onedf.onedf_validate(p) == getattr(onedf.abi, want)


def test_validate_score_field(onedf):
    for score in range(4):
        assert onedf.onedf_validate(onedf.Problem(*GOOD.values(), 0, 1, score)) == onedf.OK
    for score in (-1, 4):
        assert onedf.onedf_validate(onedf.Problem(*GOOD.values(), 0, 1, score)) == onedf.abi.ERR_INVALID_ARG
    for sel, want in ((0, "OK"), (1, "OK"), (2, "ERR_INVALID_ARG"), (-1, "ERR_INVALID_ARG")):
        assert onedf.onedf_validate(onedf.Problem(*GOOD.values(), 0, 1, 0, sel)) == getattr(onedf.abi, want)


def test_shard_owner_zigzag(onedf):
    """Chunk c -> rank: g = c mod 2P, g < P ? g : 2P-1-g (onedf.h "Sequence sharding").  Every
    chunk has one owner; with C a multiple of 2P every rank owns C/P chunks and the same
    total causal work sum(c) (query i searches floor(i/M) runs)."""
    from paper_2501_14577_b200.seqshard import ShardPlan
    for world in (1, 2, 3, 4, 8):
        for C in (1, 5, 32, 64):
            own = [onedf.abi.onedf_shard_owner(c, world) for c in range(C)]
            assert all(0 <= o < world for o in own)
            if C % (2 * world) == 0:
                work = [sum(c for c in range(C) if own[c] == r) for r in range(world)]
                cnt = [own.count(r) for r in range(world)]
                assert len(set(work)) == 1 and len(set(cnt)) == 1, (world, C, work)
            plan = ShardPlan(N=C * 16 - 3, M=16, world=world)
            rows = sorted(int(x) for r in range(world) for x in plan.rows[r])
            assert rows == list(range(C * 16 - 3))          # every position owned exactly once
            for r in range(world):
                assert all(own[int(i) // 16] == r for i in plan.rows[r])
    assert [onedf.abi.onedf_shard_owner(c, 4) for c in range(10)] == [0, 1, 2, 3, 3, 2, 1, 0, 0, 1]


def test_rank_sum_checks_arguments(onedf):
    lib = onedf.abi.lib()
    assert lib.onedf_rank_sum(256, 10, 0, 256, None) == onedf.abi.ERR_INVALID_ARG
    assert lib.onedf_rank_sum(None, 10, 2, 256, None) == onedf.abi.ERR_INVALID_ARG
    sharded = onedf.Problem(*GOOD.values(), 1, 2)
    # sharded encode needs caller bounds (the all-reduced bounds_partial); checked before the device
    assert lib.onedf_encode(ctypes.byref(sharded), 256, 256, None, 256, 256, None, 256, 1 << 30,
                            None) == onedf.abi.ERR_INVALID_ARG
    assert lib.onedf_topk_attn_step_host(ctypes.byref(sharded), *([256] * 3), ctypes.c_float(0.5), *([256] * 7),
                                         1 << 40, None) == onedf.abi.ERR_UNSUPPORTED


def test_validate_accepts_and_sizes(onedf):
    p = onedf.Problem(*GOOD.values())
    assert onedf.onedf_validate(p) == onedf.OK
    for op in (onedf.OP_ENCODE, onedf.OP_SORT, onedf.OP_FWD, onedf.OP_BWD, onedf.OP_STEP_HOST):
        assert onedf.onedf_workspace_size(p, op) >= 256
    # the backward holds coeff [BH, N, k] float2 at least
    assert onedf.onedf_workspace_size(p, onedf.OP_BWD) >= 6 * 1000 * 32 * 8


def test_long_runs_are_supported_with_global_scratch(onedf):
    """Runs longer than the on-chip sort limit validate and get a sort workspace for the
    global-scratch path (2 x (8 + 4) bytes per position); short runs need no scratch."""
    kw = dict(GOOD)
    m = onedf.onedf_max_run_length()
    kw.update(N=4 * m, chunk=2 * m)
    p = onedf.Problem(*kw.values())
    assert onedf.onedf_validate(p) == onedf.OK
    assert onedf.onedf_workspace_size(p, onedf.OP_SORT) >= 24 * p.B * p.H * p.N
    assert onedf.onedf_workspace_size(onedf.Problem(*GOOD.values()), onedf.OP_SORT) == 256


def test_calls_check_arguments_before_any_launch(onedf):
    lib = onedf.abi.lib()
    bad = onedf.Problem(*dict(GOOD, k=0).values())
    good = onedf.Problem(*GOOD.values())
    assert lib.onedf_encode(ctypes.byref(bad), 1, 1, None, 1, 1, None, 256, 1 << 30, None) == onedf.abi.ERR_INVALID_ARG
    # workspace too small / misaligned / NULL -> ERR_WORKSPACE (checked before the device)
    # (fwd: Q..Z, then the nullable indeg and means; bwd: Q..perm, nullable indeg and means, dQ..d_eps)
    assert lib.onedf_topk_attn_fwd(ctypes.byref(good), *([256] * 11), None, None, 256, 16,
                                   None) == onedf.abi.ERR_WORKSPACE
    assert lib.onedf_sort(ctypes.byref(good), 256, 256, 256, 257, 1 << 20, None) == onedf.abi.ERR_WORKSPACE
    assert lib.onedf_topk_attn_bwd(ctypes.byref(good), *([256] * 11), None, None, *([256] * 4), None, 1 << 40,
                                   None) == onedf.abi.ERR_WORKSPACE
    assert onedf.status_string(onedf.abi.ERR_WORKSPACE).startswith("workspace")


def test_no_oracle_in_product_package():
    """The product path never imports, links or calls the oracle, and vice versa."""
    banned_product = ("import oracle", "from oracle", "oref_", "liboref")
    pkg = os.path.join(ROOT, "paper_2501_14577_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                for b in banned_product:
                    assert b not in text, (f, b)
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            text = open(os.path.join(ROOT, "oracle", f)).read()
            for b in ("import paper_2501_14577_b200", "from paper_2501_14577_b200", "libonedf", "onedf.h"):
                assert b not in text, (f, b)


def test_bf16_contract_helpers():
    """The bf16 parity helpers of tests/_util.py (NEXT-4, reading D26) against torch's own bfloat16:
    rounding is round-to-nearest-even, and half_ulp(x) is half the gap to the next bf16 value."""
    import numpy as np
    import torch

    from _util import bf16_half_ulp, bf16_round
    x = np.array([1.0, 1.5, 3.0, 0.1, -7.25, 1e-3, 1.00390625, 1.01171875], dtype=np.float32)
    r = bf16_round(x)
    assert r[6] == 1.0 and r[7] == 1.015625            # ties to even: 1 + 2^-8 -> 1, 1 + 3*2^-8 -> 1 + 2^-6
    b = torch.from_numpy(np.abs(r)).to(torch.bfloat16)
    up = torch.nextafter(b, torch.full_like(b, float("inf"))).float().numpy()
    np.testing.assert_array_equal(bf16_half_ulp(r), (up - np.abs(r)) / 2)
    assert bf16_half_ulp(0.0) == 0.0
