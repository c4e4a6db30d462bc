"""GPU parity: the sm_100a kernels (through the C-ABI) against the reference.

Modelled on the reference's own suites (tests/test_spmm.cpp, acceptance_test.cpp C1/C2/C8):
  * exact mode (DASPMM_EXACT, P honoured) is bit-identical to the reference's spmm()
    for every RB kernel, and for every EB row owned by a single chunk; EB rows shared
    by chunks (atomic deposits in both implementations) are held to Tolerance<T>;
  * fast mode (FFMA, library-chosen chunking) is held to the order-independent bound
    |y - y64| <= 2*gamma(len+1)*sum|a*x| against the fp64 oracle, and to
    the reference's own Tolerance<float> (rtol 1e-3, atol 1e-6) against spmm_reference<float>.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import oracle as O  # noqa: E402
import helpers as H  # noqa: E402


@pytest.fixture(scope="module")
def sk():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2202_08556_b200 import spmmkit

    spmmkit.lib()
    return spmmkit


def _case(sk, z, meta, name, dtype):
    m = meta["cases"][name]
    return sk.CsrMatrix(m["rows"], m["cols"], z[f"{name}/rp"], z[f"{name}/ci"],
                        z[f"{name}/va"].astype(dtype), dtype)


@pytest.mark.parametrize("dt", ["64", "32"])
def test_exact_mode_matches_reference_golden(sk, golden, golden_meta, dt):
    dtype = np.float64 if dt == "64" else np.float32
    n_checked = 0
    for name in sorted(golden_meta["cases"]):
        a = _case(sk, golden, golden_meta, name, dtype)
        d = sk.DeviceCsr.from_host(a)
        for n in golden_meta["cases"][name]["ns"]:
            x = golden[f"{name}/n{n}/x{dt}"]
            for k in range(8):
                kid = sk.KernelId.from_index(k)
                for (P, W, Cb) in golden_meta["cases"][name]["configs"]:
                    if W > 32:
                        continue
                    want = golden[f"{name}/n{n}/k{k}/P{P}W{W}C{Cb}/y{dt}"]
                    xd = sk.DenseMatrix.from_logical(x, sk.Layout.ColMajor if k & 2 else
                                                     sk.Layout.RowMajor)
                    y = sk.spmm(kid, d, xd, sk.WorkerConfig(P, W, Cb), exact=True).logical()
                    if k < 4:
                        np.testing.assert_array_equal(y, want, err_msg=f"{name} {kid} P{P}W{W}")
                    else:
                        shared = H.split_rows(a, P)
                        np.testing.assert_array_equal(y[~shared], want[~shared],
                                                      err_msg=f"{name} {kid} P{P}W{W}")
                        rt = 1e-10 if dt == "64" else 1e-3
                        np.testing.assert_allclose(y, want, rtol=rt, atol=rt)
                    n_checked += 1
    assert n_checked > 400


@pytest.mark.parametrize("dt", ["64", "32"])
def test_fast_mode_within_gamma_bound(sk, golden, golden_meta, dt):
    dtype = np.float64 if dt == "64" else np.float32
    for name in sorted(golden_meta["cases"]):
        a = _case(sk, golden, golden_meta, name, dtype)
        d = sk.DeviceCsr.from_host(a)
        for n in golden_meta["cases"][name]["ns"]:
            x = golden[f"{name}/n{n}/x{dt}"]
            y64 = O.spmm_reference(H.to_oracle(a), x.astype(np.float64))
            bound = H.gamma_bound(a, x, dtype)
            ref32 = golden[f"{name}/n{n}/ref{dt}"]
            for k in range(8):
                kid = sk.KernelId.from_index(k)
                for W in (2, 8, 32):
                    y = sk.spmm_auto_layout(kid, d, sk.DenseMatrix.from_logical(x),
                                            sk.WorkerConfig(1, W, 4)).logical()
                    err = np.abs(y.astype(np.float64) - y64)
                    assert (err <= bound).all(), f"{name} {kid} W{W} n{n}: {err.max()}"
                    assert sk.tolerance_equal(sk.DenseMatrix.from_logical(y),
                                              sk.DenseMatrix.from_logical(ref32)), f"{name} {kid}"


@pytest.mark.parametrize("skew", [0.0, 1.2])
@pytest.mark.parametrize("n", [1, 2, 3, 4, 8, 16, 32, 33, 64, 128, 256])
def test_random_matrices_all_kernels(sk, n, skew):
    """test_spmm.cpp:99-126 style, larger: random/power-law rows incl. very long rows."""
    rng = np.random.default_rng(100 + n)
    a = H.random_csr(3000, 2500, 60000, seed=n, dtype=np.float32, skew=skew)
    x = rng.uniform(-1, 1, (2500, n)).astype(np.float32)
    d = sk.DeviceCsr.from_host(a)
    y64 = O.spmm_reference(H.to_oracle(a), x.astype(np.float64))
    bound = H.gamma_bound(a, x, np.float32)
    for k in range(8):
        for W in (4, 32):
            kid = sk.KernelId.from_index(k)
            y = sk.spmm_auto_layout(kid, d, sk.DenseMatrix.from_logical(x),
                                    sk.WorkerConfig(1, W, 4)).logical()
            err = np.abs(y.astype(np.float64) - y64)
            assert (err <= bound).all(), f"{kid} W{W} n{n}: max err {err.max()}"


def test_rb_sr_bit_identical_to_spmm_reference_float(sk):
    """RB+RM+SR and RB+CM+SR equal spmm_reference<float> bit for bit
    (exact mode), at N = 2 / 32 / 128."""
    a = H.random_csr(2000, 1500, 40000, seed=9, dtype=np.float32, skew=1.0)
    d = sk.DeviceCsr.from_host(a)
    for n in (2, 32, 128):
        x = np.random.default_rng(n).uniform(-1, 1, (1500, n)).astype(np.float32)
        ref = O.spmm_reference(H.to_oracle(a).__class__(a.num_rows, a.num_cols, a.row_offsets,
                                                         a.col_indices, a.values), x,
                               dtype=np.float32)
        for k in (0, 2):
            y = sk.spmm_auto_layout(sk.KernelId.from_index(k), d, sk.DenseMatrix.from_logical(x),
                                    sk.WorkerConfig(1, 8, 4), exact=True).logical()
            np.testing.assert_array_equal(y, ref)


def test_rb_pr_bit_identical_to_oracle_kernel(sk):
    """RB+PR exact mode == reference RB+PR (adjacent tree) at equal W, float."""
    a = H.random_csr(500, 400, 9000, seed=3, dtype=np.float32, skew=1.1)
    d = sk.DeviceCsr.from_host(a)
    x = np.random.default_rng(1).uniform(-1, 1, (400, 12)).astype(np.float32)
    for W in (2, 4, 8, 16, 32):
        for k in (1, 3):
            want = O.spmm_kernel(k, H.to_oracle(a), x, 3, W, 4, dtype=np.float32)
            y = sk.spmm_auto_layout(sk.KernelId.from_index(k), d, sk.DenseMatrix.from_logical(x),
                                    sk.WorkerConfig(3, W, 4), exact=True).logical()
            np.testing.assert_array_equal(y, want, err_msg=f"k{k} W{W}")


def test_eb_exact_matches_oracle_on_owned_rows(sk):
    a = H.random_csr(800, 600, 20000, seed=5, dtype=np.float32, skew=1.3)
    d = sk.DeviceCsr.from_host(a)
    x = np.random.default_rng(2).uniform(-1, 1, (600, 7)).astype(np.float32)
    for P in (1, 3, 64, 1000):
        shared = H.split_rows(a, P)
        for k in (4, 5, 6, 7):
            for W in (4, 32):
                want = O.spmm_kernel(k, H.to_oracle(a), x, P, W, 4, dtype=np.float32)
                y = sk.spmm_auto_layout(sk.KernelId.from_index(k), d,
                                        sk.DenseMatrix.from_logical(x), sk.WorkerConfig(P, W, 4),
                                        exact=True).logical()
                np.testing.assert_array_equal(y[~shared], want[~shared], err_msg=f"k{k} P{P} W{W}")
                np.testing.assert_allclose(y, want, rtol=1e-4, atol=1e-4)


def test_rb_deterministic_across_runs_and_workers(sk):
    """test_spmm.cpp:163-180: RB bits independent of run and of P."""
    a = H.random_csr(300, 200, 2500, seed=31, dtype=np.float64)
    d = sk.DeviceCsr.from_host(a)
    x = sk.DenseMatrix.from_logical(np.random.default_rng(32).uniform(-1, 1, (200, 5)))
    for k in range(4):
        kid = sk.KernelId.from_index(k)
        first = sk.spmm_auto_layout(kid, d, x, sk.WorkerConfig(3, 4, 2)).data
        for p in (1, 2, 7):
            again = sk.spmm_auto_layout(kid, d, x, sk.WorkerConfig(p, 4, 2)).data
            np.testing.assert_array_equal(again, first)


def test_errors_match_reference(sk):
    """test_spmm.cpp:197-224 — same exception kinds and message prefixes."""
    a = H.csr_from_counts([6, 2, 0, 3, 1], 8)
    x_rm = sk.DenseMatrix.from_logical(np.ones((8, 2)))
    x_cm = sk.convert_layout(x_rm, sk.Layout.ColMajor)
    with pytest.raises(ValueError, match="needs ColMajor X, got RowMajor"):
        sk.spmm(sk.KernelId.parse("RB+CM+SR"), a, x_rm, sk.WorkerConfig(1, 4, 2))
    with pytest.raises(ValueError, match="needs RowMajor X"):
        sk.spmm(sk.KernelId.parse("EB+RM+PR"), a, x_cm, sk.WorkerConfig(1, 4, 2))
    with pytest.raises(ValueError, match="A is 5x8 but X has 7 rows"):
        sk.spmm(sk.KernelId.from_index(0), a, sk.DenseMatrix.from_logical(np.ones((7, 2))),
                sk.WorkerConfig(1, 4, 2))
    for cfg in (sk.WorkerConfig(0, 4, 2), sk.WorkerConfig(1, 3, 2), sk.WorkerConfig(1, 4, 0)):
        with pytest.raises(ValueError, match="spmm: invalid config"):
            sk.spmm(sk.KernelId.from_index(0), a, x_rm, cfg)
    with pytest.raises(IndexError):
        sk.KernelId.from_index(8)
    # C-ABI-level checks (the ABI validates on its own, no shim in between)
    from paper_2202_08556_b200 import _lib

    import torch
    d = sk.DeviceCsr.from_host(a)
    B = torch.ones(8, 2, device="cuda", dtype=torch.float64)
    Cc = torch.zeros(5, 2, device="cuda", dtype=torch.float64)
    with pytest.raises(_lib.InvalidArgument, match="needs ColMajor"):
        sk.spmm_device(2, d, B, Cc, b_layout=sk.Layout.RowMajor)
    with pytest.raises(_lib.InvalidArgument, match="group_width"):
        sk.spmm_device(1, d, B, Cc, W=6)


def test_zero_matrix_and_zero_columns(sk):
    """test_spmm.cpp:226-242."""
    a = H.csr_from_counts([0, 0, 0], 4)
    x = sk.DenseMatrix.from_logical(np.random.default_rng(3).uniform(-1, 1, (4, 3)))
    for kid in sk.all_kernels():
        y = sk.spmm_auto_layout(kid, a, x, sk.WorkerConfig(2, 4, 2))
        assert (y.data == 0).all()
    b = H.csr_from_counts([6, 2, 0, 3, 1], 8)
    x0 = sk.DenseMatrix.zeros(8, 0)
    for kid in sk.all_kernels():
        y = sk.spmm_auto_layout(kid, b, x0, sk.WorkerConfig(2, 4, 2))
        assert y.num_rows == 5 and y.num_cols == 0


def test_identity_exact_for_all_kernels(sk):
    """test_spmm.cpp:71-81."""
    a = sk.CsrMatrix.identity(8)
    x = sk.DenseMatrix.from_logical(np.random.default_rng(11).uniform(-1, 1, (8, 4)))
    for kid in sk.all_kernels():
        for p in (1, 2):
            y = sk.spmm_auto_layout(kid, a, x, sk.WorkerConfig(p, 4, 2))
            np.testing.assert_array_equal(y.logical(), x.logical())


def test_output_fully_overwritten(sk):
    """C is poisoned before the call; every element must be written (empty rows,
    split rows, all kernels, fast mode)."""
    import torch

    a = H.random_csr(4000, 3000, 50000, seed=77, dtype=np.float32, skew=1.5)
    d = sk.DeviceCsr.from_host(a)
    x = np.random.default_rng(4).uniform(-1, 1, (3000, 16)).astype(np.float32)
    y64 = O.spmm_reference(H.to_oracle(a), x.astype(np.float64))
    bound = H.gamma_bound(a, x, np.float32)
    for k in range(8):
        B = torch.from_numpy(np.ascontiguousarray(x.T if k & 2 else x)).cuda()
        Cc = torch.full((4000, 16), float("nan"), device="cuda")
        sk.spmm_device(k, d, B, Cc)
        torch.cuda.synchronize()
        y = Cc.cpu().numpy().astype(np.float64)
        assert np.isfinite(y).all(), k
        assert (np.abs(y - y64) <= bound).all(), k


def test_device_partition_matches_reference(sk, golden, golden_meta):
    for name in sorted(golden_meta["cases"]):
        a = _case(sk, golden, golden_meta, name, np.float64)
        for p in (1, 2, 3, 5, 8, 64):
            b, e, r = sk.partition_elements(a, p)
            np.testing.assert_array_equal(np.stack([b, e, r]), golden[f"{name}/part{p}"])


def test_device_features_bit_exact(sk, golden, golden_meta):
    for name in sorted(golden_meta["cases"]):
        a = _case(sk, golden, golden_meta, name, np.float64)
        if a.num_rows == 0:
            continue
        f = sk.extract_features(a, 16)
        assert f.std_row == golden[f"{name}/std_row"][0], name
        assert f.nnz == a.nnz() and f.mat_size == a.num_rows
    big = H.random_csr(200000, 1000, 3000000, seed=1, skew=1.4)
    f = sk.extract_features(big, 8)
    assert f.std_row == O.extract_features(H.to_oracle(big))[2]


def test_device_warp_primitives_bit_exact(sk, golden):
    import ctypes as C

    from paper_2202_08556_b200 import _lib

    L = _lib.lib()
    vals, widths, sums = golden["tree/values"], golden["tree/widths"], golden["tree/sums"]
    off = 0
    for w, s in zip(widths, sums):
        v = np.ascontiguousarray(vals[off:off + w])
        off += w
        if w > 32:
            continue
        out = np.zeros(1)
        _lib.check(L.daspmm_debug_tree_reduce_f64(v.ctypes.data, int(w), out.ctypes.data))
        assert out[0] == s
    ids, vals, widths = golden["cond/ids"], golden["cond/values"], golden["cond/widths"]
    seg_sums, counts = golden["cond/seg_sums"], golden["cond/counts"]
    off = soff = 0
    for w, cnt in zip(widths, counts):
        v = np.ascontiguousarray(vals[off:off + w])
        idw = np.ascontiguousarray(ids[off:off + w])
        out = np.zeros(w)
        _lib.check(L.daspmm_debug_conditional_scan_f64(v.ctypes.data, idw.ctypes.data, int(w),
                                                       out.ctypes.data))
        starts = [i for i in range(w) if i == 0 or idw[i] != idw[i - 1]]
        assert list(out[starts]) == list(seg_sums[soff:soff + cnt])
        off += w
        soff += cnt


def _golden_model(tag):
    import os

    gdir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
    return open(os.path.join(gdir, f"selector_{tag}.txt")).read()


def test_device_selector_bit_exact_with_host_predict(sk):
    """daspmm_select (device features + device ensemble) == predict_kernel on
    extract_features (host, reference arithmetic) for many matrices and N — with the
    reference-trained golden model and with the shipped B200 model."""
    import os

    import torch

    models = [sk.load_selector(_golden_model("plain")),
              sk.load_selector(open(os.path.join(os.path.dirname(sk.__file__), "models",
                                                 "b200_selector.txt")).read())]
    out = torch.zeros(1, dtype=torch.int32, device="cuda")
    n_checked = 0
    for seed in range(12):
        skew = [0.0, 0.8, 1.5][seed % 3]
        rows = [300, 5000, 40000][seed % 3]
        a = H.random_csr(rows, rows, rows * (2 + seed), seed=seed, dtype=np.float32, skew=skew)
        d = sk.DeviceCsr.from_host(a)
        for n in (1, 2, 3, 8, 16, 33, 64, 128, 1000):
            f = sk.extract_features(d, n)
            for m in models:
                want = sk.predict_kernel(m, f).index()
                sk.select_device(d, m, n, out)
                torch.cuda.synchronize()
                assert int(out.item()) == want, (seed, n)
                n_checked += 1
    assert n_checked >= 200


def _std_split_model(thr):
    """8 one-split trees on std_row (feature 2) at `thr`: class 0 wins when
    std_row <= thr, class 1 otherwise (selector text v1, gbdt.hpp:336-453)."""
    lines = ["spmmkit-selector v1", "uses_hardware 0", "spmmkit-gbdt v1",
             "classes 8 features 4 best_round 0",
             "config num_rounds 1 max_depth 1 min_leaf 1 learning_rate 0.10000000000000001 "
             "patience 10 lambda 9.9999999999999995e-07 seed 0",
             "feature_names 4 log2_nnz log2_mat_size std_row n_cols", "rounds 1"]
    for c in range(8):
        lo, hi = {0: (1.0, -1.0), 1: (-1.0, 1.0)}.get(c, (0.0, 0.0))
        lines += [f"tree 0 {c} 3", f"node split 2 {thr!r} 1 2 1.0", f"node leaf {lo!r}",
                  f"node leaf {hi!r}"]
    return "\n".join(lines + ["end"]) + "\n"


def test_device_selector_std_split_at_the_exact_value(sk):
    """A std_row split exactly at (and one ulp below) the reference's std_row: the
    device selector (cluster kernel, on a fresh handle whose exact std_row is not yet
    known) must decide as the host's sequential double sum (features.hpp:27-35), going
    through the exact replay when the threshold falls inside the proven interval."""
    import math

    import torch

    out = torch.zeros(1, dtype=torch.int32, device="cuda")
    for seed, skew in ((1, 0.0), (2, 1.2), (3, 2.0)):
        a = H.random_csr(5000, 5000, 60000, seed=seed, dtype=np.float32, skew=skew)
        lens = np.diff(a.row_offsets)
        M = a.num_rows
        mean = float(int(a.row_offsets[-1])) / float(M)
        acc = 0.0
        for x in lens.tolist():
            d = float(x) - mean
            acc += d * d
        std = math.sqrt(acc / M)
        for thr, want in ((std, 0), (math.nextafter(std, -math.inf), 1),
                          (math.nextafter(std, math.inf), 0)):
            model = sk.load_selector(_std_split_model(thr))
            d = sk.DeviceCsr.from_host(a)  # fresh handle: no exact std_row cached yet
            sk.select_device(d, model, 32, out)
            torch.cuda.synchronize()
            assert int(out.item()) == want, (seed, thr, std)
            # the same decision inside the DA-SpMM graph (selector node -> SWITCH)
            d = sk.DeviceCsr.from_host(a)
            B = torch.rand(a.num_cols, 32, device="cuda")
            C = torch.empty(a.num_rows, 32, device="cuda")
            out.fill_(-1)
            sk.spmm_selected(d, model, B, C, kernel_out=out)
            torch.cuda.synchronize()
            assert int(out.item()) == want, ("graph", seed, thr, std)


def test_graph_dispatch_runs_the_selected_kernel(sk):
    """spmm_selected: the SWITCH body that runs is the selector's choice, and the
    output equals spmm with that kernel; both B layouts; repeated calls reuse the graph."""
    import os

    import torch

    model = sk.load_selector(open(os.path.join(os.path.dirname(sk.__file__), "models",
                                               "b200_selector.txt")).read())
    for seed, skew in ((1, 0.0), (2, 1.5)):
        a = H.random_csr(6000, 5000, 90000, seed=seed, dtype=np.float32, skew=skew)
        d = sk.DeviceCsr.from_host(a)
        y64 = None
        for n in (2, 8, 32, 128):
            x = np.random.default_rng(n).uniform(-1, 1, (5000, n)).astype(np.float32)
            y64 = O.spmm_reference(H.to_oracle(a), x.astype(np.float64))
            bound = H.gamma_bound(a, x, np.float32)
            for layout in (sk.Layout.RowMajor, sk.Layout.ColMajor):
                B = torch.from_numpy(np.ascontiguousarray(x if layout == sk.Layout.RowMajor
                                                          else x.T)).cuda()
                kout = torch.full((1,), -1, dtype=torch.int32, device="cuda")
                # rep 0-2: layout twin on B as given (default); 3-5: the reference's
                # conversion of B to the chosen kernel's layout (DASPMM_CONVERT_LAYOUT)
                for rep in range(6):
                    Cc = torch.full((6000, n), float("nan"), device="cuda")
                    sk.spmm_selected(d, model, B, Cc, b_layout=layout, kernel_out=kout,
                                     convert_layout=rep >= 3)
                    torch.cuda.synchronize()
                    y = Cc.cpu().numpy().astype(np.float64)
                    assert (np.abs(y - y64) <= bound).all(), (n, layout, rep)
                want = sk.predict_kernel(model, sk.extract_features(d, n)).index()
                assert int(kout.item()) == want


def test_row_panels_reassemble_exactly(sk):
    """Multi-GPU unit on one device: nnz-balanced row panels (multi.row_panel_cuts)
    computed separately and stacked equal the single-handle result bit for bit (RB
    exact mode), i.e. sharding needs no exchange."""
    import torch

    from paper_2202_08556_b200 import multi

    a = H.random_csr(5000, 4000, 120000, seed=8, dtype=np.float32, skew=1.3)
    d = sk.DeviceCsr.from_host(a)
    x = np.random.default_rng(3).uniform(-1, 1, (4000, 32)).astype(np.float32)
    B = torch.from_numpy(x).cuda()
    full = torch.empty(5000, 32, device="cuda")
    sk.spmm_device(0, d, B, full, exact=True)
    for parts in (2, 3, 8):
        cuts = multi.row_panel_cuts(a.row_offsets, parts)
        pieces = []
        for p in range(parts):
            pd = d.panel(int(cuts[p]), int(cuts[p + 1]))
            Cp = torch.empty(int(cuts[p + 1] - cuts[p]), 32, device="cuda")
            sk.spmm_device(0, pd, B, Cp, exact=True)
            pieces.append(Cp)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(torch.cat(pieces).cpu().numpy(), full.cpu().numpy())


def test_auto_layout_tall_operand(sk):
    """B with K > 2M rows: the device transpose must stride its row tiles (grid.y cap)."""
    import torch

    K = 2_300_000
    rng = np.random.default_rng(9)
    rows = 300
    lens = rng.integers(0, 20, rows)
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(K, size=l, replace=False)) for l in lens]).astype(np.int64)
    a = sk.CsrMatrix(rows, K, rp, ci, rng.uniform(-1, 1, ci.size).astype(np.float32), np.float32)
    d = sk.DeviceCsr.from_host(a)
    x = rng.uniform(-1, 1, (K, 2)).astype(np.float32)
    B = torch.from_numpy(x).cuda()
    Cc = torch.empty(rows, 2, device="cuda")
    from paper_2202_08556_b200 import _lib

    _lib.check(_lib.lib().daspmm_spmm_auto_layout(d._h, 2, 0, 8, 8, B.data_ptr(), 0, 2, 2,
                                                  Cc.data_ptr(), 2, 0, None))
    torch.cuda.synchronize()
    y64 = O.spmm_reference(H.to_oracle(a), x.astype(np.float64))
    assert (np.abs(Cc.cpu().numpy() - y64) <= H.gamma_bound(a, x, np.float32)).all()


def _banded_csr(M, b, seed, empty_every=0):
    """Banded CSR (row r holds columns [r-b, r+b] ∩ [0, M)); every empty_every-th
    row left empty, plus one fully empty 64-row block."""
    from paper_2202_08556_b200.spmmkit import CsrMatrix

    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for r in range(M):
        if (empty_every and r % empty_every == 0) or 1000 <= r < 1064:
            continue
        c = np.arange(max(0, r - b), min(M, r + b + 1))
        rows.append(np.full(c.size, r))
        cols.append(c)
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    rp = np.zeros(M + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp)
    va = rng.uniform(-1, 1, cols.size).astype(np.float32)
    return CsrMatrix(M, M, rp, cols.astype(np.int64), va, np.float32)


@pytest.mark.parametrize("b", [2, 8, 30])
def test_rb_window_kernel_banded(sk, b):
    """RB+RM+SR on row-local matrices runs k_rb_sr_win (B window staged in shared
    memory, TMA bulk copy when rows are contiguous). Contiguous B, padded ldb and a
    B pointer off the 16-byte grid (TMA lead bytes) all stay within the gamma bound."""
    import torch

    import os

    a = _banded_csr(6000, b, seed=b, empty_every=7)
    d = sk.DeviceCsr.from_host(a)
    os.environ["DASPMM_WIN"] = "1"  # opt-in kernel
    sk.reload_env()
    bound_cache = {}
    variants = set()
    for n in (1, 2, 3, 4, 8, 16, 32, 33, 64, 100, 128, 256, 300):
        x = np.random.default_rng(n).uniform(-1, 1, (a.num_cols, n)).astype(np.float32)
        y64 = O.spmm_reference(H.to_oracle(a), x.astype(np.float64))
        bound = bound_cache.setdefault(n, H.gamma_bound(a, x, np.float32))
        for mode in ("contig", "padded", "offset"):
            if mode == "contig":
                B = torch.from_numpy(x).cuda()
            elif mode == "padded":
                B = torch.zeros(a.num_cols, n + 4, device="cuda")[:, :n]
                B.copy_(torch.from_numpy(x))
            else:  # one element past a 16-B boundary: the bulk copy needs lead bytes
                buf = torch.zeros(a.num_cols * n + 1, device="cuda")
                B = buf[1:].view(a.num_cols, n)
                B.copy_(torch.from_numpy(x))
            C = torch.full((a.num_rows, n), float("nan"), device="cuda")
            variant, rows = sk.plan_info(0, d, B, C)
            variants.add(variant)
            sk.spmm_device(0, d, B, C)
            torch.cuda.synchronize()
            err = np.abs(C.cpu().numpy().astype(np.float64) - y64)
            assert (err <= bound).all(), f"b{b} n{n} {mode} ({variant}, {rows}): {err.max()}"
    del os.environ["DASPMM_WIN"]
    sk.reload_env()
    assert "rb_window" in variants


def test_rb_window_not_used_on_scattered_columns(sk):
    import os

    import torch

    a = H.random_csr(4000, 4000, 60000, seed=3, dtype=np.float32)
    d = sk.DeviceCsr.from_host(a)
    B = torch.zeros(4000, 32, device="cuda")
    C = torch.zeros(4000, 32, device="cuda")
    os.environ["DASPMM_WIN"] = "1"
    sk.reload_env()
    try:
        assert sk.plan_info(0, d, B, C)[0] != "rb_window"
    finally:
        del os.environ["DASPMM_WIN"]
        sk.reload_env()


@pytest.mark.parametrize("kernel", [0, 4])
@pytest.mark.parametrize("skew", [0.0, 1.3])
def test_lean_sr_kernels(sk, kernel, skew):
    """Lean RB/EB+RM+SR kernels (quad-loaded A, one row segment per group): odd nnz
    (scalar tail quad), empty rows, very long rows split over many EB chunks, N with
    several y-tiles and padded ldb; within the gamma bound, every output written."""
    import torch

    import os

    a = H.random_csr(5003, 4001, 90001, seed=11 + kernel, dtype=np.float32, skew=skew)
    d = sk.DeviceCsr.from_host(a)
    seen = set()
    os.environ["DASPMM_LEAN_RB"] = "1"  # RB lean walk is opt-in
    sk.reload_env()
    for n in (8, 16, 24, 32, 64, 96, 128, 200, 256):
        x = np.random.default_rng(n).uniform(-1, 1, (a.num_cols, n)).astype(np.float32)
        y64 = O.spmm_reference(H.to_oracle(a), x.astype(np.float64))
        bound = H.gamma_bound(a, x, np.float32)
        for padded in (False, True):
            if padded:
                B = torch.zeros(a.num_cols, n + 8, device="cuda")[:, :n]
                B.copy_(torch.from_numpy(x))
            else:
                B = torch.from_numpy(x).cuda()
            C = torch.full((a.num_rows, n), float("nan"), device="cuda")
            seen.add(sk.plan_info(kernel, d, B, C)[0])
            sk.spmm_device(kernel, d, B, C)
            torch.cuda.synchronize()
            err = np.abs(C.cpu().numpy().astype(np.float64) - y64)
            assert (err <= bound).all(), f"k{kernel} n{n} padded={padded}: {np.nanmax(err)}"
    del os.environ["DASPMM_LEAN_RB"]
    sk.reload_env()
    assert "lean" in seen


@pytest.mark.parametrize("skew", [0.0, 1.3])
def test_rb_lean_one_lane_default(sk, skew):
    """RB+RM+SR with one-lane groups (N <= 4) runs the lean quad-load walk by default
    (M large enough that the planner keeps V = N, i.e. one lane per row): odd nnz, empty
    and long rows, padded ldb; within the gamma bound, C fully written."""
    import torch

    a = H.random_csr(80003, 3001, 700001, seed=23, dtype=np.float32, skew=skew)
    d = sk.DeviceCsr.from_host(a)
    for n in (1, 2, 3, 4):
        x = np.random.default_rng(n).uniform(-1, 1, (a.num_cols, n)).astype(np.float32)
        y64 = O.spmm_reference(H.to_oracle(a), x.astype(np.float64))
        bound = H.gamma_bound(a, x, np.float32)
        for padded in (False, True):
            B = torch.zeros(a.num_cols, n + 5 * padded, device="cuda")[:, :n]
            B.copy_(torch.from_numpy(x))
            C = torch.full((a.num_rows, n), float("nan"), device="cuda")
            if n in (2, 4) and not padded:
                assert sk.plan_info(0, d, B, C)[0] == "lean"
            sk.spmm_device(0, d, B, C)
            torch.cuda.synchronize()
            err = np.abs(C.cpu().numpy().astype(np.float64) - y64)
            assert (err <= bound).all(), f"n{n} padded={padded}: {np.nanmax(err)}"


def test_rb_column_tiles_for_wide_b(sk):
    """B beyond 256 MB (K = 2^19, N = 128 fp32) makes RB+RM+SR run two 64-column tiles;
    the result is checked on the touched B rows against an fp64 restatement."""
    import torch

    K, M, nnz, n = 1 << 19, 3001, 60001, 128
    rng = np.random.default_rng(5)
    a = H.random_csr(M, K, nnz, seed=29, dtype=np.float32)
    d = sk.DeviceCsr.from_host(a)
    B = torch.empty(K, n, device="cuda").uniform_(-1, 1, generator=torch.Generator(
        device="cuda").manual_seed(int(rng.integers(1 << 30))))
    C = torch.full((M, n), float("nan"), device="cuda")
    assert sk.plan_info(0, d, B, C) == ("base", 2)
    sk.spmm_device(0, d, B, C)
    torch.cuda.synchronize()
    ci = torch.from_numpy(a.col_indices.astype(np.int64)).cuda()
    xs = B[ci].double().cpu().numpy()  # the gathered rows, in nnz order
    rows = np.repeat(np.arange(M), np.diff(a.row_offsets))
    prod = a.values.astype(np.float64)[:, None] * xs
    y64 = np.zeros((M, n))
    np.add.at(y64, rows, prod)
    mag = np.zeros((M, n))
    np.add.at(mag, rows, np.abs(prod))
    lens = np.diff(a.row_offsets).astype(np.float64)
    u = 2.0 ** -24
    bound = 2 * ((lens + 1) * u / (1 - (lens + 1) * u))[:, None] * mag + 1e-30
    err = np.abs(C.cpu().numpy().astype(np.float64) - y64)
    assert (err <= bound).all(), np.nanmax(err)


@pytest.mark.parametrize("skew", [0.0, 1.3])
def test_eb_tma_gather_kernel(sk, skew):
    """EB+RM+SR with TMA gather4 row fetches (DASPMM_TMA=1): box widths 32/64/128 with
    zero-filled columns past N, several y-tiles, padded ldb, odd nnz (array-tail stage),
    empty rows and rows split across warp ranges; within the gamma bound."""
    import os

    import torch

    a = H.random_csr(5003, 4001, 90001, seed=21, dtype=np.float32, skew=skew)
    d = sk.DeviceCsr.from_host(a)
    os.environ["DASPMM_TMA"] = "1"
    sk.reload_env()
    try:
        for n in (32, 40, 64, 100, 128, 256, 300):
            x = np.random.default_rng(n).uniform(-1, 1, (a.num_cols, n)).astype(np.float32)
            y64 = O.spmm_reference(H.to_oracle(a), x.astype(np.float64))
            bound = H.gamma_bound(a, x, np.float32)
            for padded in (False, True):
                if padded:
                    B = torch.zeros(a.num_cols, n + 12, device="cuda")[:, :n]
                    B.copy_(torch.from_numpy(x))
                else:
                    B = torch.from_numpy(x).cuda()
                C = torch.full((a.num_rows, n), float("nan"), device="cuda")
                assert sk.plan_info(4, d, B, C)[0] == "eb_tma", n
                sk.spmm_device(4, d, B, C)
                torch.cuda.synchronize()
                err = np.abs(C.cpu().numpy().astype(np.float64) - y64)
                assert (err <= bound).all(), f"n{n} padded={padded}: {np.nanmax(err)}"
    finally:
        del os.environ["DASPMM_TMA"]
        sk.reload_env()


def test_gcn_layer_matches_dense_reference(sk):
    """GCN aggregation through DA-SpMM (BASELINE configs[2] shape, scaled down): the
    normalised adjacency and a two-layer forward pass against dense fp64 torch."""
    import torch

    from paper_2202_08556_b200 import gcn, gen

    torch.manual_seed(0)
    M, K, rp, ci, va = gen.rmat(12, 16 * 4096, 0.45, 0.22, 0.22, 0.11, seed=5)
    g = gcn.GCNGraph(M, rp, ci)
    A = torch.zeros(M, M, dtype=torch.float64, device="cuda")
    r = torch.repeat_interleave(torch.arange(M, device="cuda"), (rp[1:] - rp[:-1]).long())
    A[r, ci.long()] = 1.0
    A += torch.eye(M, dtype=torch.float64, device="cuda")
    dinv = A.sum(1).rsqrt()
    Ahat = dinv[:, None] * A * dinv[None, :]
    H = torch.randn(M, 96, device="cuda")
    l1, l2 = gcn.GCNLayer(96, 128).cuda(), gcn.GCNLayer(128, 32, activation=None).cuda()
    out = l2(g, l1(g, H))
    ref = Ahat @ torch.relu(Ahat @ H.double() @ l1.weight.double() + l1.bias.double())
    ref = ref @ l2.weight.double() + l2.bias.double()
    torch.testing.assert_close(out.double(), ref, rtol=1e-4, atol=1e-4)
    agg = g.aggregate(H)
    torch.testing.assert_close(agg.double(), Ahat @ H.double(), rtol=1e-5, atol=1e-5)


def test_spmm_rows_to_replicates_rows(sk):
    """daspmm_spmm_rows_to: the RB+RM+SR row epilogue stored into several destinations
    (here local buffers standing in for the peers' NVLink-mapped copies of C, one of
    them a row-offset view of a larger matrix) — every copy equals the single-
    destination result and is within the gamma bound."""
    import torch

    a = H.random_csr(3000, 2500, 50000, seed=31, dtype=np.float32, skew=0.8)
    d = sk.DeviceCsr.from_host(a)
    for n in (3, 32, 100, 256):
        x = np.random.default_rng(n).uniform(-1, 1, (2500, n)).astype(np.float32)
        B = torch.from_numpy(x).cuda()
        y64 = O.spmm_reference(H.to_oracle(a), x.astype(np.float64))
        bound = H.gamma_bound(a, x, np.float32)
        big = torch.full((3000 + 700, n), float("nan"), device="cuda")
        outs = [torch.full((3000, n), float("nan"), device="cuda") for _ in range(2)]
        outs.append(big[500:3500])
        sk.spmm_rows_to(d, B, outs)
        ref = torch.empty(3000, n, device="cuda")
        sk.spmm_device(0, d, B, ref)
        torch.cuda.synchronize()
        for o in outs:
            assert torch.equal(o, ref), n
        err = np.abs(ref.cpu().numpy().astype(np.float64) - y64)
        assert (err <= bound).all()
        assert torch.isnan(big[:500]).all() and torch.isnan(big[3500:]).all()


@pytest.mark.parametrize("case", ["one_nnz", "three_nnz", "all_empty_but_last", "single_long_row",
                                  "chunk_aligned_rows"])
def test_fast_paths_edge_shapes(sk, case):
    """Edge shapes through every fp32 fast path (lean walks, one-lane staged path, CTA-
    combined walk, replicated epilogue): nnz below one quad, a matrix whose nonzeros all
    sit in its last row, one row longer than every chunk, and rows ending exactly on
    chunk boundaries. Every output element written (NaN-poisoned), gamma bound held."""
    import torch

    from paper_2202_08556_b200.spmmkit import CsrMatrix

    rng = np.random.default_rng(7)
    if case == "one_nnz":
        M, K, lens = 5, 7, [0, 0, 1, 0, 0]
    elif case == "three_nnz":
        M, K, lens = 3, 9, [1, 0, 2]
    elif case == "all_empty_but_last":
        M, K, lens = 4000, 300, [0] * 3999 + [300]
    elif case == "single_long_row":
        M, K, lens = 64, 70000, [3] * 31 + [60000] + [5] * 32
    else:  # every row holds 128 nonzeros: rows end on every chunk boundary
        M, K, lens = 2048, 4096, [128] * 2048
    rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    ci = np.concatenate([np.sort(rng.choice(K, size=l, replace=False)) if l else
                         np.zeros(0, np.int64) for l in lens]).astype(np.int64)
    a = CsrMatrix(M, K, rp, ci, rng.uniform(-1, 1, ci.size).astype(np.float32), np.float32)
    d = sk.DeviceCsr.from_host(a)
    for n in (1, 2, 4, 8, 16, 32, 64, 128):
        x = rng.uniform(-1, 1, (K, n)).astype(np.float32)
        B = torch.from_numpy(x).cuda()
        y64 = O.spmm_reference(H.to_oracle(a), x.astype(np.float64))
        bound = H.gamma_bound(a, x, np.float32)
        for k in (0, 4):
            C = torch.full((M, n), float("nan"), device="cuda")
            sk.spmm_device(k, d, B, C)
            torch.cuda.synchronize()
            err = np.abs(C.cpu().numpy().astype(np.float64) - y64)
            assert (err <= bound).all(), f"{case} k{k} n{n}: {np.nanmax(err)}"
        outs = [torch.full((M, n), float("nan"), device="cuda") for _ in range(2)]
        sk.spmm_rows_to(d, B, outs)
        torch.cuda.synchronize()
        for o in outs:
            err = np.abs(o.cpu().numpy().astype(np.float64) - y64)
            assert (err <= bound).all(), f"{case} rows_to n{n}"


def test_fault_injection_is_caught(sk):
    """Failure detection (reference: validate --inject-fault, spmmkit_cli.cpp:366-371,
    394-397, and the zero-returning stub of test_bench.cpp:86-100): with the env-guarded
    hook armed, a device SpMM returns a result off by 1 in C[0][0] and the gamma-bound
    parity check rejects it; disarmed, the same check passes."""
    import os

    import torch

    a = H.random_csr(300, 200, 3000, seed=2, dtype=np.float32)
    d = sk.DeviceCsr.from_host(a)
    x = np.random.default_rng(1).uniform(-1, 1, (200, 16)).astype(np.float32)
    y64 = O.spmm_reference(H.to_oracle(a), x.astype(np.float64))
    bound = H.gamma_bound(a, x, np.float32)
    B = torch.from_numpy(x).cuda()

    def run():
        C = torch.empty(300, 16, device="cuda")
        sk.spmm_device(0, d, B, C)
        torch.cuda.synchronize()
        return bool((np.abs(C.cpu().numpy().astype(np.float64) - y64) <= bound).all())

    assert run()
    os.environ["SPMMKIT_ENABLE_FAULT_INJECTION"] = "1"
    os.environ["DASPMM_INJECT_FAULT"] = "1"
    sk.reload_env()
    try:
        assert not run()
    finally:
        del os.environ["SPMMKIT_ENABLE_FAULT_INJECTION"], os.environ["DASPMM_INJECT_FAULT"]
        sk.reload_env()
    assert run()


@pytest.mark.parametrize("W", [64, 128, 256, 1024])
def test_pr_group_width_above_a_warp(sk, W):
    """worker.hpp:29-40 accepts any power-of-two group width: W > 32 runs one CTA of W
    threads per group (spmm_pr_wide.cu). Exact mode against the oracle's restatement of
    the reference worker (pinned to the reference on golden): RB+PR bit-identical (the
    W-lane tree = warp trees + tree over warp totals), EB+PR bit-identical on rows owned
    by one chunk; fast mode within the gamma bound."""
    import torch

    cases = [H.csr_from_counts([6, 2, 0, 3, 1, 300, 0, 2000, 5], 2100),
             H.random_csr(400, 900, 30000, seed=W, skew=1.5)]
    for a in cases:
        for dt in (np.float64, np.float32):
            ad = a.astype(dt)
            d = sk.DeviceCsr.from_host(ad)
            for n in (1, 3, 33):
                x = np.random.default_rng(n + W).uniform(-1, 1, (a.num_cols, n))
                for k in (1, 3, 5, 7):
                    P = 3
                    xd = sk.DenseMatrix.from_logical(x.astype(dt), sk.Layout.ColMajor if k & 2
                                                     else sk.Layout.RowMajor)
                    y = sk.spmm(sk.KernelId.from_index(k), d, xd, sk.WorkerConfig(P, W, 2),
                                exact=True).logical()
                    want = O.spmm_kernel(k, H.to_oracle(ad), x.astype(dt), P=P, W=W, Cb=2,
                                         dtype=dt)
                    if k < 4:
                        np.testing.assert_array_equal(y, want, err_msg=f"k{k} W{W} n{n} {dt}")
                    else:
                        shared = H.split_rows(ad, P)
                        np.testing.assert_array_equal(y[~shared], want[~shared])
                        np.testing.assert_allclose(y, want, rtol=1e-3 if dt == np.float32 else 1e-10,
                                                   atol=1e-6 if dt == np.float32 else 1e-12)
                    yf = sk.spmm(sk.KernelId.from_index(k), d, xd, sk.WorkerConfig(1, W, 2)).logical()
                    bound = H.gamma_bound(ad, x.astype(dt), dt)
                    y64 = O.spmm_reference(H.to_oracle(ad), x.astype(dt).astype(np.float64))
                    assert (np.abs(yf.astype(np.float64) - y64) <= bound).all(), (k, W, n)
    with pytest.raises(RuntimeError, match="supports 2..1024"):
        sk.spmm(sk.KernelId.from_index(1), cases[0], sk.DenseMatrix.zeros(2100, 2),
                sk.WorkerConfig(1, 2048, 2))


@pytest.mark.parametrize("case", ["uniform_small", "uniform_chunk_edges", "dyadic_mean",
                                  "all_equal", "leading_equal_then_skew", "powerlaw_huge_rows",
                                  "one_huge_row", "tiny_and_huge_mix", "large_2p20"])
def test_exact_std_block_sum_matches_sequential(sk, case):
    """extract_features' std_row comes from the block-wide binade prefix sum
    (csrc/exact_sum.cuh); it must equal, bit for bit, the reference's loop run as one
    dependent chain of double adds (daspmm_debug_std_chain) and the C oracle."""
    import ctypes as C

    from paper_2202_08556_b200 import _lib

    rng = np.random.default_rng(hash(case) % (1 << 31))
    if case == "uniform_small":
        mats = [rng.integers(0, 40, m) for m in (1, 2, 3, 7, 33, 1000, 5001)]
    elif case == "uniform_chunk_edges":  # around the 8192-term chunk of a 1024-thread block
        mats = [rng.integers(0, 40, m) for m in (8191, 8192, 8193, 16384, 16385, 24577)]
    elif case == "dyadic_mean":  # mean = 16 exactly: integer terms, no rounding for long
        mats = [np.resize(np.array([10, 22, 16, 16]), m) for m in (4096, 100000)]
        mats.append(rng.permutation(np.resize(np.arange(0, 33), 33 * 3000)))
    elif case == "all_equal":  # every term 0: the sum stays +0 (std 0)
        mats = [np.full(m, 9) for m in (1, 10, 70000)]
    elif case == "leading_equal_then_skew":
        mats = [np.concatenate([np.full(50000, 5), rng.integers(0, 3000, 30000)])]
    elif case == "powerlaw_huge_rows":
        w = 1.0 / np.arange(1, 200001) ** 1.5
        mats = [rng.multinomial(3_000_000, w / w.sum())]
    elif case == "one_huge_row":
        v = np.zeros(100000, np.int64)
        v[777] = 2_000_000
        mats = [v, np.roll(v, 50000)]
    elif case == "tiny_and_huge_mix":
        v = rng.integers(0, 3, 300000)
        v[rng.integers(0, 300000, 50)] = rng.integers(100000, 400000, 50)
        mats = [v]
    else:
        mats = [rng.integers(0, 33, 1 << 20)]
    for lens in mats:
        lens = np.asarray(lens, np.int64)
        M = lens.size
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        nnz = int(rp[-1])
        ci = np.zeros(nnz, np.int64)
        a = sk.CsrMatrix(M, 1, rp, ci, np.ones(nnz, np.float32), np.float32)
        d = sk.DeviceCsr.from_host(a)
        got = sk.extract_features(d, 8).std_row
        chain = C.c_double()
        _lib.check(sk.lib().daspmm_debug_std_chain(d._h, C.byref(chain)))
        assert got == chain.value, (case, M, got, chain.value)
        if nnz <= 4_000_000:
            want = O.extract_features(O.Csr(M, 1, rp, ci, np.ones(nnz)))[2]
            assert got == want, (case, M, got, want)
        d.close()


_ONE_CTA_SCRIPT = r"""
import os, sys
sys.path.insert(0, os.environ["ROOT"]); sys.path.insert(0, os.path.join(os.environ["ROOT"], "tests"))
import numpy as np, torch
import helpers as H
from paper_2202_08556_b200 import spmmkit as sk
m = sk.load_selector(open(os.path.join(os.path.dirname(sk.__file__), "models",
                                       "b200_selector.txt")).read())
out = torch.zeros(1, dtype=torch.int32, device="cuda")
for seed in range(6):
    a = H.random_csr(3000, 3000, 3000 * (3 + seed), seed=seed, dtype=np.float32,
                     skew=[0.0, 1.2][seed % 2])
    d = sk.DeviceCsr.from_host(a)
    for n in (2, 16, 128):
        sk.select_device(d, m, n, out)
        torch.cuda.synchronize()
        assert int(out.item()) == sk.predict_kernel(m, sk.extract_features(d, n)).index()
print("one-cta ok")
"""


def test_one_cta_selector_matches_host_predict(sk):
    """DASPMM_SELECT_ONE_CTA=1 (read once per process, so in a subprocess): the one-CTA
    selector kernel decides as the host's predict_kernel, like the cluster kernel."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DASPMM_SELECT_ONE_CTA="1", ROOT=root)
    r = subprocess.run([sys.executable, "-c", _ONE_CTA_SCRIPT], capture_output=True, text=True,
                       timeout=600, env=env, cwd=root)
    assert r.returncode == 0 and "one-cta ok" in r.stdout, (r.stdout + r.stderr)[-3000:]
