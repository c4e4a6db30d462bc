"""tools/controlled.py's trend classifier against the reference's own cases
(tests/test_controlled.cpp:36-47, controlled.hpp:60-71). CPU only."""
import importlib.util
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def controlled():
    pytest.importorskip("torch")
    spec = importlib.util.spec_from_file_location("controlled", os.path.join(ROOT, "tools",
                                                                             "controlled.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.path.insert(0, ROOT)
    spec.loader.exec_module(mod)
    return mod


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
def test_trend_verdict_matches_reference(controlled, ratios, want):
    assert controlled.trend_verdict(ratios) == want


def test_trend_verdict_custom_tau(controlled):
    assert controlled.trend_verdict([100.0, 111.0], tau=0.2) == "flat"
