"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference headers (compiled by oracle/Makefile into
oracle/_ref/libspmmkit_ref.so) on seeded inputs and stores inputs + outputs:

  golden.npz      matrices (CSR int64 / f64 values), dense operands, and the
                  reference outputs of spmm_reference and spmm() for all 8 kernels
                  at several (P, W, C), in f64 and f32; partitions; features;
                  tree/conditional reductions.
  selector_*.txt  selector models trained by the reference trainer
                  (train_selector, selector.hpp:41-60) + their predictions.

Usage:  make -C oracle && python tests/golden/make_golden.py
The fixtures are committed; the GPU box never needs /root/reference.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402


def ref_csr_arrays(h):
    R = O.ref()
    rows, cols, nnz = C.c_int64(), C.c_int64(), C.c_int64()
    R.ref_csr_info(h, C.byref(rows), C.byref(cols), C.byref(nnz))
    rp = np.zeros(rows.value + 1, np.int64)
    ci = np.zeros(nnz.value, np.int64)
    va = np.zeros(nnz.value, np.float64)
    R.ref_csr_copy(h, rp, ci, va)
    return rows.value, cols.value, rp, ci, va


def from_coo(rows, cols, trip):
    R = O.ref()
    r = np.array([t[0] for t in trip], np.int64)
    c = np.array([t[1] for t in trip], np.int64)
    v = np.array([t[2] for t in trip], np.float64)
    h = R.ref_csr_from_coo(rows, cols, len(trip), r, c, v)
    assert h, R.ref_last_error()
    return h


def ragged_shape():
    # tests/test_util.hpp:25-35 — rows of 6/2/0/3/1 nonzeros in 8 columns.
    t = [(0, c, 0.5 + c) for c in (0, 1, 2, 4, 6, 7)]
    t += [(1, 1, 1.5), (1, 5, -2.25), (3, 0, 1.0), (3, 3, 2.0), (3, 7, 3.0), (4, 2, -1.0)]
    return from_coo(5, 8, t)


def with_row_counts(counts, ncols):
    # tests/test_util.hpp:39-46
    t = [(r, i, 1.0 + i) for r, n in enumerate(counts) for i in range(n)]
    return from_coo(len(counts), ncols, t)


def random_csr(rows, cols, nnz, seed):
    # tests/test_util.hpp:50-64 restated with numpy's generator (values in [-2, 2)).
    rng = np.random.default_rng(seed)
    cells = rng.choice(rows * cols, size=min(nnz, rows * cols), replace=False)
    vals = rng.uniform(-2.0, 2.0, size=cells.size)
    vals[vals == 0] = 1.0
    return from_coo(rows, cols, [(int(c // cols), int(c % cols), float(v))
                                 for c, v in zip(cells, vals)])


def main():
    O.build(ref=True)
    R = O.ref()
    assert R is not None, "oracle/_ref not built (needs /root/reference)"
    cases = {}
    cases["ragged"] = ragged_shape()
    cases["identity8"] = from_coo(8, 8, [(i, i, 1.0) for i in range(8)])
    cases["empty_rows"] = with_row_counts([0, 2, 0, 0, 5, 0], 6)
    cases["all_empty"] = with_row_counts([0, 0, 0], 4)
    cases["single_row"] = from_coo(1, 40, [(0, c, 0.25 * c - 3.0) for c in range(0, 40, 3)])
    cases["single_col"] = from_coo(17, 1, [(r, 0, 1.0 + r) for r in range(0, 17, 2)])
    cases["random_40x30"] = random_csr(40, 30, 300, 17)
    cases["long_row"] = with_row_counts([1, 700, 0, 3, 290, 2], 800)
    # R-MATs as in test_spmm.cpp:99-126 (uniform and skewed quadrants).
    for i, (scale, ef, q) in enumerate([(5, 3, (.25, .25, .25, .25)), (6, 4, (.6, .15, .15, .1)),
                                        (7, 5, (.57, .19, .19, .05)), (8, 8, (.25, .25, .25, .25)),
                                        (9, 6, (.7, .1, .1, .1))]):
        h = R.ref_rmat(scale, (1 << scale) * ef, *q, 1000 + i)
        assert h, R.ref_last_error()
        cases[f"rmat{i}_s{scale}"] = h

    ns_small = [1, 2, 3, 8, 33]
    ns_big = [4, 17]
    configs = [(1, 8, 4), (2, 4, 2), (3, 2, 3), (4, 16, 1), (7, 32, 8)]
    out: dict[str, np.ndarray] = {}
    meta = {"cases": {}}
    for name, h in cases.items():
        rows, cols, rp, ci, va = ref_csr_arrays(h)
        out[f"{name}/rp"], out[f"{name}/ci"], out[f"{name}/va"] = rp, ci, va
        big = rows > 40
        ns = ns_big if big else ns_small
        cfgs = configs[1:3] if big else (configs[:3] if rows > 20 else configs)
        if rows > 300:
            cfgs = []
        meta["cases"][name] = {"rows": rows, "cols": cols, "nnz": int(rp[-1]), "ns": ns,
                               "configs": cfgs}
        for n in ns:
            seed = 7 * n + rows
            x64 = np.zeros(cols * n, np.float64)
            R.ref_dense_random_f64(cols, n, 0, seed, x64)
            x32 = np.zeros(cols * n, np.float32)
            R.ref_dense_random_f32(cols, n, 0, seed, x32)
            out[f"{name}/n{n}/x64"] = x64.reshape(cols, n)
            out[f"{name}/n{n}/x32"] = x32.reshape(cols, n)
            y = np.zeros(rows * n, np.float64)
            assert R.ref_spmm_reference_f64(h, x64, n, 0, y) == 0
            out[f"{name}/n{n}/ref64"] = y.reshape(rows, n)
            y = np.zeros(rows * n, np.float32)
            assert R.ref_spmm_reference_f32(h, x32, n, 0, y) == 0
            out[f"{name}/n{n}/ref32"] = y.reshape(rows, n)
            for k in range(8):
                cm = (k >> 1) & 1
                xm64 = np.ascontiguousarray(x64.reshape(cols, n).T if cm else x64.reshape(cols, n))
                xm32 = np.ascontiguousarray(x32.reshape(cols, n).T if cm else x32.reshape(cols, n))
                for (P, W, Cb) in cfgs:
                    y = np.zeros(rows * n, np.float64)
                    rc = R.ref_spmm_f64(h, k, P, W, Cb, xm64.reshape(-1), n, cm, y)
                    assert rc == 0, R.ref_last_error()
                    out[f"{name}/n{n}/k{k}/P{P}W{W}C{Cb}/y64"] = y.reshape(rows, n)
                    y = np.zeros(rows * n, np.float32)
                    rc = R.ref_spmm_f32(h, k, P, W, Cb, xm32.reshape(-1), n, cm, y)
                    assert rc == 0, R.ref_last_error()
                    out[f"{name}/n{n}/k{k}/P{P}W{W}C{Cb}/y32"] = y.reshape(rows, n)
        for p in (1, 2, 3, 5, 8, 64):
            b, e, r = (np.zeros(p, np.int64) for _ in range(3))
            assert R.ref_partition(h, p, b, e, r) == 0
            out[f"{name}/part{p}"] = np.stack([b, e, r])
        if rows > 0:
            nnz, ms, sd = C.c_int64(), C.c_int64(), C.c_double()
            assert R.ref_extract_features(h, 16, C.byref(nnz), C.byref(ms), C.byref(sd)) == 0
            out[f"{name}/std_row"] = np.array([sd.value])

    # Reductions (reduce.hpp): trees and conditional reductions, exhaustive W=4 patterns.
    rng = np.random.default_rng(5)
    trees = []
    for w in (1, 2, 4, 8, 16, 32, 64):
        v = rng.uniform(-1, 1, w)
        t = C.c_double()
        assert R.ref_tree_reduce_f64(v, w, C.byref(t)) == 0
        trees.append((v, t.value))
    out["tree/values"] = np.concatenate([t[0] for t in trees])
    out["tree/widths"] = np.array([len(t[0]) for t in trees], np.int64)
    out["tree/sums"] = np.array([t[1] for t in trees])
    pats, vals, segs, sums, counts = [], [], [], [], []
    for w in (2, 4, 8, 16, 32):
        for trial in range(12):
            v = rng.uniform(-1, 1, w)
            ids = np.cumsum(rng.integers(0, 2, w) * rng.integers(1, 3, w)).astype(np.int64)
            sid = np.zeros(w, np.int64)
            ss = np.zeros(w, np.float64)
            cnt = C.c_int64()
            assert R.ref_conditional_reduce_f64(v, ids, w, sid, ss, C.byref(cnt)) == 0
            pats.append(ids)
            vals.append(v)
            segs.append(sid[:cnt.value])
            sums.append(ss[:cnt.value])
            counts.append(cnt.value)
    out["cond/ids"] = np.concatenate(pats)
    out["cond/values"] = np.concatenate(vals)
    out["cond/widths"] = np.array([len(p) for p in pats], np.int64)
    out["cond/seg_ids"] = np.concatenate(segs)
    out["cond/seg_sums"] = np.concatenate(sums)
    out["cond/counts"] = np.array(counts, np.int64)

    # Selector: train with the reference trainer on synthetic timing samples whose
    # best kernel depends on all four features; record predictions on probes.
    for tag, uses_hw in (("plain", False), ("unified", True)):
        n = 400
        feats = np.zeros((n, 4))
        feats[:, 0] = np.round(2.0 ** rng.uniform(8, 27, n))            # nnz
        feats[:, 1] = np.round(feats[:, 0] / 2.0 ** rng.uniform(0, 6, n)) + 1  # rows
        feats[:, 2] = 2.0 ** rng.uniform(-3, 9, n)                        # std_row
        feats[:, 3] = 2 ** rng.integers(1, 8, n)                          # N
        hw = rng.integers(0, 3, n).astype(np.int64)
        t = np.ones((n, 8))
        for i in range(n):
            m = 4 if feats[i, 2] > 12 else 0
            nn = 0 if feats[i, 3] >= 16 else 2
            k = 1 if feats[i, 0] < 2 ** 16 else 0
            best = m + (nn if not uses_hw or hw[i] != 2 else 2 - nn) + k
            t[i] = 1e-3 * (2.0 + rng.uniform(0, 1, 8))
            t[i, best] = 1e-3
        ptr = R.ref_selector_train(n, 320, np.ascontiguousarray(feats.reshape(-1)),
                                   hw.ctypes.data if uses_hw else None,
                                   np.ascontiguousarray(t.reshape(-1)), 60, 4, 5)
        assert ptr, R.ref_last_error()
        text = C.cast(ptr, C.c_char_p).value.decode()
        R.ref_free(ptr)
        with open(os.path.join(HERE, f"selector_{tag}.txt"), "w") as fh:
            fh.write(text)
        model = R.ref_selector_load(text.encode())
        assert model, R.ref_last_error()
        probes = np.zeros((300, 5))
        probes[:, 0] = np.round(2.0 ** rng.uniform(0, 30, 300))
        probes[:, 1] = np.round(2.0 ** rng.uniform(0, 25, 300))
        probes[:, 2] = 2.0 ** rng.uniform(-4, 10, 300)
        probes[:, 3] = 2 ** rng.integers(0, 9, 300)
        probes[:, 4] = rng.integers(0, 3, 300)
        preds = np.zeros(300, np.int64)
        for i in range(300):
            k = C.c_int()
            rc = R.ref_selector_predict(model, int(probes[i, 0]), int(probes[i, 1]),
                                        float(probes[i, 2]), int(probes[i, 3]),
                                        int(probes[i, 4]) if uses_hw else -1, C.byref(k))
            assert rc == 0, R.ref_last_error()
            preds[i] = k.value
        R.ref_selector_free(model)
        out[f"selector_{tag}/probes"] = probes
        out[f"selector_{tag}/preds"] = preds

    for h in cases.values():
        R.ref_csr_free(h)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    with open(os.path.join(HERE, "golden_meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", len(out), "arrays;",
          os.path.getsize(os.path.join(HERE, "golden.npz")) // 1024, "KiB")


if __name__ == "__main__":
    main()
