"""Pins the C oracle (oracle/daspmm_oracle.c) to the reference's own outputs.

Golden vectors come from the unmodified reference (tests/golden/make_golden.py), so
a pass here means the restatement reproduces the reference bit-for-bit on:
  * spmm_reference (spmm.hpp:16-32), f64 and f32;
  * all 8 spmm() kernels (spmm.hpp:194-271) at several (P, W, C), f64 and f32 —
    RB kernels bit-exact; EB kernels bit-exact too in the serial restatement
    (tolerance is allowed where a split row takes >2 atomic contributions);
  * partition_elements (partition.hpp:45-64), extract_features (features.hpp:21-41),
    tree_reduce / conditional_reduce (reduce.hpp), selector predictions (gbdt.hpp:41-77).
CPU only.
"""
import numpy as np
import pytest

from oracle import oracle as O


def _cases(meta):
    return sorted(meta["cases"])


def _csr(z, name, meta):
    m = meta["cases"][name]
    return O.Csr(m["rows"], m["cols"], z[f"{name}/rp"], z[f"{name}/ci"], z[f"{name}/va"])


def test_spmm_reference_bit_exact(golden, golden_meta):
    for name in _cases(golden_meta):
        a = _csr(golden, name, golden_meta)
        for n in golden_meta["cases"][name]["ns"]:
            x64 = golden[f"{name}/n{n}/x64"]
            x32 = golden[f"{name}/n{n}/x32"]
            y = O.spmm_reference(a, x64, dtype=np.float64)
            np.testing.assert_array_equal(y, golden[f"{name}/n{n}/ref64"], err_msg=name)
            y = O.spmm_reference(a, x32, dtype=np.float32)
            np.testing.assert_array_equal(y, golden[f"{name}/n{n}/ref32"], err_msg=name)
            # ColMajor operand gives identical bits (test_spmm.cpp:58-63).
            y = O.spmm_reference(a, np.ascontiguousarray(x64.T), x_colmajor=True)
            np.testing.assert_array_equal(y, golden[f"{name}/n{n}/ref64"], err_msg=name)


def _split_rows_multi(a, P):
    """Rows shared by >= 2 EB chunks: their deposits are atomic in the reference
    (spmm.hpp:123-126) and interleave across threads, so only tolerance holds."""
    b, e, _ = O.partition_elements(a, P)
    rp = a.row_offsets
    bad = []
    for r in range(a.num_rows):
        s, t = rp[r], rp[r + 1]
        chunks = np.sum((b < t) & (e > s))
        if chunks >= 2:
            bad.append(r)
    return bad


@pytest.mark.parametrize("dt", ["64", "32"])
def test_all_kernels_match_reference(golden, golden_meta, dt):
    dtype = np.float64 if dt == "64" else np.float32
    checked = 0
    for name in _cases(golden_meta):
        a = _csr(golden, name, golden_meta)
        for n in golden_meta["cases"][name]["ns"]:
            x = golden[f"{name}/n{n}/x{dt}"]
            for k in range(8):
                for (P, W, Cb) in golden_meta["cases"][name]["configs"]:
                    want = golden[f"{name}/n{n}/k{k}/P{P}W{W}C{Cb}/y{dt}"]
                    got = O.spmm_kernel(k, a, x, P, W, Cb, dtype=dtype)
                    if k < 4:
                        np.testing.assert_array_equal(got, want, err_msg=f"{name} k{k}")
                    else:
                        bad = set(_split_rows_multi(a, P))
                        ok = np.ones(a.num_rows, bool)
                        ok[list(bad)] = False
                        np.testing.assert_array_equal(got[ok], want[ok],
                                                      err_msg=f"{name} k{k} P{P}")
                        tol = 1e-10 if dt == "64" else 1e-3  # Tolerance<T>, spmm.hpp:283-295
                        np.testing.assert_allclose(got, want, rtol=tol, atol=tol)
                    checked += 1
    assert checked > 500


def test_partition_matches_reference(golden, golden_meta):
    for name in _cases(golden_meta):
        a = _csr(golden, name, golden_meta)
        for p in (1, 2, 3, 5, 8, 64):
            b, e, r = O.partition_elements(a, p)
            np.testing.assert_array_equal(np.stack([b, e, r]), golden[f"{name}/part{p}"])


def test_partition_known_answers():
    # test_partition.cpp:24-56
    def counts(c):
        rp = np.concatenate([[0], np.cumsum(c)]).astype(np.int64)
        return O.Csr(len(c), 8, rp, np.zeros(rp[-1], np.int64), np.ones(rp[-1]))

    b, e, r = O.partition_elements(counts([4, 3, 3]), 4)
    assert list(e - b) == [3, 3, 2, 2]
    b, e, r = O.partition_elements(counts([3, 3]), 2)
    assert list(r) == [0, 1]
    b, e, r = O.partition_elements(counts([1, 1]), 5)
    assert list(e - b) == [1, 1, 0, 0, 0] and r[2] == 2 and r[4] == 2
    with pytest.raises(ValueError):
        O.partition_elements(counts([1]), 0)
    a = counts([2, 0, 3])  # test_partition.cpp:97-105
    L = O.lib()
    assert [L.oracle_row_of_element(3, a.row_offsets, e) for e in (0, 1, 2, 4)] == [0, 0, 2, 2]


def test_features_match_reference(golden, golden_meta):
    for name in _cases(golden_meta):
        a = _csr(golden, name, golden_meta)
        if a.num_rows == 0:
            continue
        nnz, m, s = O.extract_features(a)
        assert s == golden[f"{name}/std_row"][0], name
    # test_features.cpp:9-24, 82-87
    def counts(c):
        rp = np.concatenate([[0], np.cumsum(c)]).astype(np.int64)
        return O.Csr(len(c), 8, rp, np.zeros(rp[-1], np.int64), np.ones(rp[-1]))

    assert O.extract_features(counts([2, 2, 2]))[2] == 0.0
    assert O.extract_features(counts([1, 3]))[2] == 1.0
    assert O.extract_features(counts([4, 0, 0, 0]))[2] == np.sqrt(3.0)
    with pytest.raises(ValueError):
        O.extract_features(O.Csr(0, 4, np.zeros(1, np.int64), [], []))


def test_reductions_match_reference(golden):
    vals, widths, sums = golden["tree/values"], golden["tree/widths"], golden["tree/sums"]
    off = 0
    for w, s in zip(widths, sums):
        v = vals[off:off + w]
        off += w
        assert O.tree_reduce_lanes(v, int(w), 1)[0] == s
    # reduce.hpp examples (test_reduce.cpp:35-67)
    assert O.tree_reduce_lanes(np.array([1., 2, 3, 4]), 4, 1)[0] == 10.0
    assert O.tree_reduce_lanes(np.array([.1, .2, .3, .4]), 4, 1)[0] == (0.1 + 0.2) + (0.3 + 0.4)
    two = O.tree_reduce_lanes(np.array([1., 10, 2, 20, 3, 30, 4, 40]), 4, 2)
    assert two[0] == 10.0 and two[1] == 100.0

    ids, vals, widths = golden["cond/ids"], golden["cond/values"], golden["cond/widths"]
    seg_ids, seg_sums, counts = golden["cond/seg_ids"], golden["cond/seg_sums"], golden["cond/counts"]
    off = soff = 0
    for w, cnt in zip(widths, counts):
        v = O.conditional_scan_lanes(vals[off:off + w], ids[off:off + w], int(w), 1)
        idw = ids[off:off + w]
        starts = [i for i in range(w) if i == 0 or idw[i] != idw[i - 1]]
        assert list(idw[starts]) == list(seg_ids[soff:soff + cnt])
        assert list(v[starts]) == list(seg_sums[soff:soff + cnt])
        off += w
        soff += cnt
    # exhaustive W=4 id patterns, integer values (test_reduce.cpp:99-115)
    v = np.array([3., 1, 4, 1])
    n = 0
    for a in range(4):
        for b in range(a, 4):
            for c in range(b, 4):
                for d in range(c, 4):
                    ids4 = np.array([a, b, c, d])
                    out = O.conditional_scan_lanes(v, ids4, 4, 1)
                    want = {}
                    for i, k in enumerate(ids4):
                        want[k] = want.get(k, 0.0) + v[i]
                    starts = [i for i in range(4) if i == 0 or ids4[i] != ids4[i - 1]]
                    assert [out[i] for i in starts] == [want[k] for k in ids4[starts]]
                    n += 1
    assert n == 35


@pytest.mark.parametrize("tag", ["plain", "unified"])
def test_selector_predictions_match_reference(golden, tag):
    import os

    gdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    with open(os.path.join(gdir, f"selector_{tag}.txt")) as fh:
        flat = O.parse_selector_text(fh.read())
    probes = golden[f"selector_{tag}/probes"]
    preds = golden[f"selector_{tag}/preds"]
    for p, want in zip(probes, preds):
        f = O.encode_features(int(p[0]), int(p[1]), float(p[2]), int(p[3]),
                              flat["uses_hardware"], int(p[4]))
        assert O.predict_class(flat, f) == want


@pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref not built")
def test_oracle_vs_live_reference_rmat():
    """Live cross-check on fresh R-MATs (test_spmm.cpp:99-126 style) in f32."""
    import ctypes as C

    R = O.ref()
    rng = np.random.default_rng(3)
    for trial in range(4):
        scale = 6 + trial
        h = R.ref_rmat(scale, (1 << scale) * 5, 0.57, 0.19, 0.19, 0.05, 77 + trial)
        rows, cols, nnz = C.c_int64(), C.c_int64(), C.c_int64()
        R.ref_csr_info(h, C.byref(rows), C.byref(cols), C.byref(nnz))
        rp = np.zeros(rows.value + 1, np.int64)
        ci = np.zeros(nnz.value, np.int64)
        va = np.zeros(nnz.value)
        R.ref_csr_copy(h, rp, ci, va)
        a = O.Csr(rows.value, cols.value, rp, ci, va)
        n = int(rng.integers(1, 40))
        x = rng.uniform(-1, 1, (cols.value, n)).astype(np.float32)
        for k in range(8):
            cm = (k >> 1) & 1
            xm = np.ascontiguousarray(x.T if cm else x)
            want = np.zeros(rows.value * n, np.float32)
            assert R.ref_spmm_f32(h, k, 1, 8, 4, xm.reshape(-1), n, cm, want) == 0
            got = O.spmm_kernel(k, a, x, 1, 8, 4, dtype=np.float32)
            np.testing.assert_array_equal(got.reshape(-1), want)
        R.ref_csr_free(h)
