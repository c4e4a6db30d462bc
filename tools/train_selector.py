"""Train the B200 kernel selector with the REFERENCE trainer.

Input: the B200 timing CSV from tools/collect_timings.py (features from the device
feature extractor + median device time of each of the 8 kernels). The model is
trained by the reference's own train_selector / train_gbdt (selector.hpp:41-60,
gbdt.hpp:219-299, unmodified, through oracle/_ref) so the model file format stays the
reference's text v1 contract. Split 40/10/50 (train / validation / test) as the
paper's methodology; evaluation = geometric mean of
min(t) / t[chosen] (metrics.hpp:12-36) on the test split, next to the best static
kernel.

python tools/train_selector.py gpurun_out/timings_full.csv \
    --out paper_2202_08556_b200/models/b200_selector.txt
"""
import argparse
import csv
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as O  # noqa: E402

NAMES = ["RB+RM+SR", "RB+RM+PR", "RB+CM+SR", "RB+CM+PR", "EB+RM+SR", "EB+RM+PR", "EB+CM+SR",
         "EB+CM+PR"]


def load(path):
    rows = list(csv.DictReader(open(path)))
    feats = np.array([[float(r["nnz"]), float(r["mat_size"]), float(r["std_row"]),
                       float(r["n_cols"])] for r in rows])
    times = np.array([[float(r[f"t{k}"]) for k in range(8)] for r in rows])
    ids = [r["matrix_id"] for r in rows]
    return ids, feats, times


def split_by_matrix(ids, seed=2202, ratios=(0.4, 0.1, 0.5)):
    """Split by matrix (all N of one matrix land in the same split) with a seeded
    shuffle, floor sizes as split_dataset (dataset.hpp:53-86)."""
    mats = sorted(set(ids))
    rng = np.random.default_rng(seed)
    rng.shuffle(mats)
    n = len(mats)
    a, b = int(n * ratios[0]), int(n * (ratios[0] + ratios[1]))
    tr, va = set(mats[:a]), set(mats[a:b])
    lab = np.array([0 if i in tr else (1 if i in va else 2) for i in ids])
    return lab


def normalized(times, chosen):
    return times.min(1) / times[np.arange(len(times)), chosen]


def cross_validate(R, ids, feats, times, k, train, predict, seed=2202):
    """K folds by matrix. Fold f is scored by a model trained on the other folds (7/8 of
    their matrices for training, 1/8 for the trainer's validation / early stopping)."""
    mats = sorted(set(ids))
    rng = np.random.default_rng(seed)
    rng.shuffle(mats)
    fold_of = {m: i % k for i, m in enumerate(mats)}
    fold = np.array([fold_of[i] for i in ids])
    chosen = np.zeros(len(ids), dtype=np.int64)
    per_fold = []
    for f in range(k):
        rest = [m for m in mats if fold_of[m] != f]
        n_va = max(1, len(rest) // 8)
        va_set = set(rest[:n_va])
        tr = np.array([i for i in range(len(ids)) if fold[i] != f and ids[i] not in va_set])
        va = np.array([i for i in range(len(ids)) if fold[i] != f and ids[i] in va_set])
        text = train(np.concatenate([tr, va]), len(tr))
        m = R.ref_selector_load(text.encode())
        te = np.where(fold == f)[0]
        for i in te:
            chosen[i] = predict(m, i)
        R.ref_selector_free(m)
        s = normalized(times[te], chosen[te])
        per_fold.append(round(float(np.exp(np.log(s).mean())), 4))
    sel = normalized(times, chosen)
    static = {NAMES[j]: float(np.exp(np.log(normalized(times, np.full(len(ids), j))).mean()))
              for j in range(8)}
    best = max(static, key=static.get)
    return {"folds": k, "by": "matrix", "samples": len(ids), "matrices": len(mats),
            "selector_geomean_normalized": round(float(np.exp(np.log(sel).mean())), 4),
            "selector_accuracy": round(float((chosen == times.argmin(1)).mean()), 4),
            "per_fold_geomean": per_fold,
            "best_static": best, "best_static_geomean": round(static[best], 4),
            "note": "every sample scored by a model trained without its matrix"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--out", default=os.path.join(ROOT, "paper_2202_08556_b200", "models",
                                                  "b200_selector.txt"))
    ap.add_argument("--rounds", type=int, default=100)
    ap.add_argument("--depth", type=int, default=4)
    ap.add_argument("--min-leaf", type=int, default=5)
    ap.add_argument("--final", action="store_true",
                    help="after evaluating, retrain on train+valid+test (deployment model)")
    ap.add_argument("--cv", type=int, default=0,
                    help="also K-fold cross-validate by matrix: every matrix is scored by a model "
                         "that never saw it (the held-out score of the deployed procedure)")
    a = ap.parse_args()
    R = O.ref()
    assert R is not None, "needs oracle/_ref (reference trainer); run make -C oracle"
    ids, feats, times = load(a.csv)
    lab = split_by_matrix(ids)
    order = np.concatenate([np.where(lab == 0)[0], np.where(lab == 1)[0]])
    n_train = int((lab == 0).sum())

    def train(idx, n_tr):
        f = np.ascontiguousarray(feats[idx].reshape(-1))
        t = np.ascontiguousarray(times[idx].reshape(-1))
        ptr = R.ref_selector_train(len(idx), n_tr, f, None, t, a.rounds, a.depth, a.min_leaf)
        assert ptr, R.ref_last_error()
        text = C.cast(ptr, C.c_char_p).value.decode()
        R.ref_free(ptr)
        return text

    text = train(order, n_train)
    model = R.ref_selector_load(text.encode())
    test = np.where(lab == 2)[0]

    def predict(m, i):
        k = C.c_int()
        assert R.ref_selector_predict(m, int(feats[i, 0]), int(feats[i, 1]), float(feats[i, 2]),
                                      int(feats[i, 3]), -1, C.byref(k)) == 0
        return k.value

    chosen = np.array([predict(model, i) for i in test])
    sel = normalized(times[test], chosen)
    report = {"samples": {"train": int((lab == 0).sum()), "valid": int((lab == 1).sum()),
                          "test": int(len(test))},
              "selector_geomean_normalized": float(np.exp(np.log(sel).mean())),
              "selector_accuracy": float((chosen == times[test].argmin(1)).mean())}
    static = {}
    for k in range(8):
        s = normalized(times[test], np.full(len(test), k))
        static[NAMES[k]] = float(np.exp(np.log(s).mean()))
    report["static_geomean_normalized"] = static
    report["best_static"] = max(static, key=static.get)
    report["label_histogram_all"] = {NAMES[k]: int((times.argmin(1) == k).sum()) for k in range(8)}
    R.ref_selector_free(model)
    if a.cv > 1:
        report["cross_validation"] = cross_validate(R, ids, feats, times, a.cv, train, predict)
    if a.final:
        allidx = np.arange(len(ids))
        text = train(allidx, len(allidx))
        report["deployed"] = "retrained on all samples after evaluation"
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        fh.write(text)
    with open(os.path.splitext(a.out)[0] + "_report.json", "w") as fh:
        json.dump(report, fh, indent=1)
    print(json.dumps(report, indent=1))


if __name__ == "__main__":
    main()
