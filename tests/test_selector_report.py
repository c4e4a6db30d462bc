"""Acceptance criterion 4 of the reference (acceptance_test.cpp:285-312) applied to the
committed B200 selector: on the held-out test matrices the model's geometric-mean
normalized performance beats the best static kernel and is >= 0.90, over >= 200
samples. (The timings come from B200 runs of tools/collect_timings.py; the report is
written by tools/train_selector.py with the reference trainer.) CPU only."""
import json
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_committed_selector_meets_acceptance_c4():
    rep = json.load(open(os.path.join(ROOT, "paper_2202_08556_b200", "models",
                                      "b200_selector_report.json")))
    model = rep["selector_geomean_normalized"]
    best_static = max(rep["static_geomean_normalized"].values())
    assert rep["samples"]["test"] >= 200
    assert model >= best_static * (1.0 - 1e-12)
    assert model >= 0.90
