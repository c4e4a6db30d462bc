"""bench.py's reference arm (CPU, oracle/_ref): every call on its fastest reference design
point, whole matrices, one pass = one reference spmm() per (matrix, N). Runs on CPU with
tiny matrices; skipped when oracle/_ref was not built (no reference tree)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _mats():
    torch = pytest.importorskip("torch")
    from paper_2202_08556_b200 import gen

    out = []
    for name, mk in (("uniform", lambda: gen.uniform(600, 500, 6000, seed=1, device="cpu")),
                     ("powerlaw", lambda: gen.rmat(9, 5000, *gen.GRAPH500, seed=2, device="cpu"))):
        M, K, rp, ci, va = mk()
        out.append(dict(name=name, M=M, K=K, nnz_total=int(ci.numel()), rp=rp, ci=ci, va=va,
                        ns=[2, 8, 32]))
    return out


def test_reference_arm_picks_a_design_point_per_call():
    from oracle import oracle as O

    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    import bench

    mats = _mats()
    arm = bench._RefArm(mats)
    try:
        assert len(arm.pairs) == 6
        assert all(0 <= k < 8 for k in arm.choice)
        # CM points are only tried for N <= 16
        for (m, n), k in zip(bench._ref_sample(mats), arm.choice):
            if n > 16:
                assert not (k >> 1) & 1
        assert arm.flops == sum(2 * m["nnz_total"] * n for m, n in bench._ref_sample(mats))
        assert arm.one_pass() > 0
        assert sum(arm.choices().values()) == 6
        assert not arm.panelled
    finally:
        arm.close()


def test_reference_arm_without_selection_runs_rb_rm_sr():
    from oracle import oracle as O

    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    import bench

    arm = bench._RefArm(_mats(), select=False)
    try:
        assert set(arm.choice) == {0}
        assert arm.choices() == {"RB+RM+SR": 6}
    finally:
        arm.close()


def test_cpu_baseline_reports_per_kernel_and_single_thread():
    from oracle import oracle as O

    if O.ref() is None:
        pytest.skip("oracle/_ref not built")
    import bench

    cb = bench._cpu_baseline(_mats(), passes=1)
    assert cb["value"] > 0 and cb["kind"] == "reference"
    assert set(cb["per_kernel_all_threads"]) <= set(bench.REF_NAMES)
    assert cb["per_kernel_all_threads"]["RB+RM+SR"]["calls"] == 6
    p1 = cb["single_thread_s14_s17"]
    assert p1["calls"] == 6 and p1["best_point_gflops"] > 0 and p1["spmm_reference_gflops"] > 0
