"""Controlled experiments (paper_2202_08556_b200.controlled): the trend classifier and
series checks against the reference's own cases (tests/test_controlled.cpp,
controlled.hpp:60-115) on CPU, and acceptance criterion 7 (acceptance_test.cpp:447-483)
on the B200 kernels."""
import pytest

pytest.importorskip("torch")
from paper_2202_08556_b200 import controlled as ce  # noqa: E402


@pytest.mark.parametrize("ratios,want", [
    ([1.0, 1.5, 2.3], "rising"),
    ([2.0, 1.4, 1.0], "falling"),
    ([1.0, 1.05, 0.97, 1.02], "flat"),
    ([1.0, 2.0, 1.0], "mixed"),
    ([1.0], "flat"),
    ([], "flat"),
    ([100.0, 109.0], "flat"),
    ([100.0, 111.0], "rising"),
    ([100.0, 89.0], "falling"),
])
def test_trend_verdict_matches_reference(ratios, want):
    assert ce.trend_verdict(ratios) == want


def test_trend_verdict_custom_tau():
    assert ce.trend_verdict([100.0, 111.0], tau=0.2) == "flat"


def test_nondecreasing_with_slack():
    assert ce.nondecreasing_with_slack([1.0, 0.95, 1.2])
    assert not ce.nondecreasing_with_slack([1.0, 0.85])
    assert ce.nondecreasing_with_slack([])


def test_dimension_names_round_trip():
    for d in ce.ControlledDimension:
        assert ce.parse_dimension(ce.dimension_name(d)) == d
    assert ce.parse_dimension("rb-cm") is None


def test_series_invariants_match_reference_messages():
    """controlled.hpp:83-115: too few points, and each dimension's fixed properties."""
    spec = ce.b200_spec(ce.ControlledDimension.RB_EB, scale=8)
    ce.check_series_invariants(spec)
    short = ce.ControlledSpec(series=spec.series[:2])
    with pytest.raises(ValueError, match="at least 3 series points, got 2"):
        ce.check_series_invariants(short)
    spec.series[1].n_cols = 16
    with pytest.raises(ValueError, match="rb-eb series must vary skew only"):
        ce.check_series_invariants(spec)
    rm = ce.b200_spec(ce.ControlledDimension.RM_CM, scale=8)
    ce.check_series_invariants(rm)
    rm.series[2] = ce.ControlledPoint(ce.RmatParams(scale=9), 32)
    with pytest.raises(ValueError, match="rm-cm series must vary N only"):
        ce.check_series_invariants(rm)
    sp = ce.b200_spec(ce.ControlledDimension.SR_PR, scale=8)
    ce.check_series_invariants(sp)
    sp.series[0].n_cols = 2
    with pytest.raises(ValueError, match="sr-pr series must vary nnz only"):
        ce.check_series_invariants(sp)


def test_check_table_rejects_malformed():
    t = ce.TrendTable(ce.ControlledDimension.RB_EB, "std_row", "rb_over_eb",
                      [ce.TrendRow(1, 1, 1, 1), ce.TrendRow(2, 1, 1, 1), ce.TrendRow(3, 1, 1, 1)],
                      "flat")
    assert ce.check_table(t, "std_row", "rb_over_eb") == ""
    t.rows[2].varied = 2
    assert ce.check_table(t, "std_row", "rb_over_eb") == "varied column is not strictly increasing"
    t.rows = t.rows[:2]
    assert ce.check_table(t, "std_row", "rb_over_eb") == "expected 3 rows, got 2"


@pytest.mark.gpu
def test_criterion7_on_b200():
    """Acceptance criterion 7 on the device kernels at B200 scale (2^20 rows, degree 16):
    three well-formed trend tables, rb_over_eb nondecreasing within 10% slack, every row's
    two kernels agreeing within Tolerance<float>."""
    import torch

    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ok, msg, tables = ce.criterion7(scale=20)
    print(msg)
    for t in tables:
        print(ce.dimension_name(t.dimension), t.verdict,
              [(round(r.varied, 3), round(r.ratio, 3)) for r in t.rows])
    assert ok, msg
    # the paper's RB-EB trend: EB gains as skew grows
    assert tables[0].verdict == "rising"
