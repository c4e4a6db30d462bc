// C++ API parity suite: the reference's hot-path tests (proj/tests/test_spmm.cpp,
// test_features.cpp, test_partition.cpp, test_selector.cpp, test_matrix_market.cpp)
// restated against the B200 headers (include/spmmkit), which run on the GPU.
// Built and run by tests/test_cpp_api.py. Exit code = number of failed checks.
#include <cstdio>
#include <functional>
#include <random>
#include <set>
#include <sstream>
#include <vector>

#include "spmmkit/spmmkit.hpp"

using namespace spmmkit;

// ---------------------------------------------------------------- tiny harness
static int g_fail = 0, g_checks = 0;
static std::vector<std::pair<const char*, std::function<void()>>>& registry() {
    static std::vector<std::pair<const char*, std::function<void()>>> r;
    return r;
}
struct Reg {
    Reg(const char* n, std::function<void()> f) { registry().emplace_back(n, std::move(f)); }
};
#define CASE(name)                      \
    static void name();                 \
    static Reg reg_##name(#name, name); \
    static void name()
#define CHECK(cond)                                                              \
    do {                                                                         \
        ++g_checks;                                                              \
        if (!(cond)) {                                                           \
            ++g_fail;                                                            \
            std::fprintf(stderr, "  FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
        }                                                                        \
    } while (0)
template <class E, class F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

// ---------------------------------------------------------------- fixtures
static CsrMatrix<double> ragged_shape() {  // tests/test_util.hpp:25-35
    std::vector<std::tuple<Index, Index, double>> t;
    for (Index c : {0, 1, 2, 4, 6, 7}) t.push_back({0, c, 0.5 + double(c)});
    t.push_back({1, 1, 1.5});
    t.push_back({1, 5, -2.25});
    t.push_back({3, 0, 1.0});
    t.push_back({3, 3, 2.0});
    t.push_back({3, 7, 3.0});
    t.push_back({4, 2, -1.0});
    return CsrMatrix<double>::from_coo(5, 8, t);
}
static CsrMatrix<double> with_counts(const std::vector<Index>& counts, Index cols) {
    std::vector<std::tuple<Index, Index, double>> t;
    for (Index r = 0; r < Index(counts.size()); ++r)
        for (Index i = 0; i < counts[r]; ++i) t.push_back({r, i, 1.0 + double(i)});
    return CsrMatrix<double>::from_coo(Index(counts.size()), cols, t);
}
static CsrMatrix<double> random_csr(Index rows, Index cols, Index nnz, std::uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::uniform_int_distribution<Index> rd(0, rows - 1), cd(0, cols - 1);
    std::uniform_real_distribution<double> vd(-2.0, 2.0);
    std::set<std::pair<Index, Index>> used;
    std::vector<std::tuple<Index, Index, double>> t;
    while (Index(t.size()) < nnz && Index(used.size()) < rows * cols) {
        const Index r = rd(rng), c = cd(rng);
        if (!used.insert({r, c}).second) continue;
        double v = vd(rng);
        t.push_back({r, c, v == 0 ? 1.0 : v});
    }
    return CsrMatrix<double>::from_coo(rows, cols, t);
}
template <class T>
static bool exact_equal(const DenseMatrix<T>& a, const DenseMatrix<T>& b) {
    if (a.num_rows != b.num_rows || a.num_cols != b.num_cols) return false;
    for (Index r = 0; r < a.num_rows; ++r)
        for (Index c = 0; c < a.num_cols; ++c)
            if (a.at(r, c) != b.at(r, c)) return false;
    return true;
}

// ---------------------------------------------------------------- spmm (test_spmm.cpp)
CASE(IdentityIsExactForAllKernels) {
    const auto a = CsrMatrix<double>::identity(8);
    const auto x = DenseMatrix<double>::random(8, 4, Layout::RowMajor, 11);
    for (auto k : all_kernels())
        for (Index p : {1, 2}) CHECK(exact_equal(spmm_auto_layout(k, a, x, {p, 4, 2}), x));
}

CASE(RaggedShapeMatchesReference) {
    const auto a = ragged_shape();
    for (Index n : {1, 2, 3, 5}) {
        const auto x = DenseMatrix<double>::random(8, n, Layout::RowMajor, 100 + n);
        const auto ref = spmm_reference(a, x);
        for (auto k : all_kernels())
            for (Index p : {1, 2, 3}) CHECK(tolerance_equal(spmm_auto_layout(k, a, x, {p, 4, 2}), ref));
    }
}

CASE(RandomMatricesMatchReference) {
    std::mt19937_64 seeds(42);
    for (int trial = 0; trial < 12; ++trial) {
        const Index rows = Index(32) << (trial % 3);
        const auto a = random_csr(rows, rows, rows * (2 + trial % 4), seeds());
        for (Index n : {1, 2, 3, 8, 33}) {
            const auto x = DenseMatrix<double>::random(rows, n, Layout::RowMajor, seeds());
            const auto ref = spmm_reference(a, x);
            for (auto k : all_kernels())
                for (Index p : {1, 3}) {
                    CHECK(tolerance_equal(spmm_auto_layout(k, a, x, {p, 4, 3}), ref));
                    CHECK(tolerance_equal(spmm_auto_layout(k, a, x, {p, 4, 3}, Numerics::Exact), ref));
                }
        }
    }
}

CASE(ResultIndependentOfConfig) {
    const auto a = random_csr(40, 30, 300, 17);
    const auto x = DenseMatrix<double>::random(30, 6, Layout::RowMajor, 18);
    const auto ref = spmm_reference(a, x);
    for (auto k : all_kernels())
        for (Index p : {1, 2, 5})
            for (Index w : {2, 8})
                for (Index c : {1, 3}) CHECK(tolerance_equal(spmm_auto_layout(k, a, x, {p, w, c}), ref));
}

CASE(LayoutTwinGivesSameAnswers) {
    const auto a = random_csr(25, 25, 120, 23);
    const auto x_rm = DenseMatrix<double>::random(25, 4, Layout::RowMajor, 24);
    const auto x_cm = convert_layout(x_rm, Layout::ColMajor);
    for (int base : {0, 4})
        for (int k : {0, 1}) {
            const auto rm = KernelId::from_index(base + k), cm = KernelId::from_index(base + 2 + k);
            const auto y_rm = spmm(rm, a, x_rm, {2, 4, 4});
            const auto y_cm = spmm(cm, a, x_cm, {2, 4, 4});
            CHECK(tolerance_equal(y_cm, y_rm));
            CHECK(exact_equal(spmm_auto_layout(cm, a, x_rm, {2, 4, 4}), y_cm));
        }
}

CASE(RowBalancedIsBitDeterministic) {
    const auto a = random_csr(30, 20, 250, 31);
    const auto x = DenseMatrix<double>::random(20, 5, Layout::RowMajor, 32);
    for (int idx : {0, 1, 2, 3}) {
        const auto k = KernelId::from_index(idx);
        const auto first = spmm_auto_layout(k, a, x, {3, 4, 2});
        for (int run = 0; run < 4; ++run) CHECK(spmm_auto_layout(k, a, x, {3, 4, 2}).data == first.data);
        for (Index p : {1, 2, 7}) CHECK(spmm_auto_layout(k, a, x, {p, 4, 2}).data == first.data);
    }
}

CASE(ExactModeEqualsSpmmReferenceForSequentialRowKernels) {
    // RB+RM+SR and RB+CM+SR in exact mode reproduce spmm_reference bit for bit (float).
    const auto ad = random_csr(200, 150, 3000, 77);
    CsrMatrix<float> a;
    a.num_rows = ad.num_rows;
    a.num_cols = ad.num_cols;
    a.row_offsets = ad.row_offsets;
    a.col_indices = ad.col_indices;
    a.values.assign(ad.values.begin(), ad.values.end());
    for (Index n : {2, 32, 128}) {
        const auto x = DenseMatrix<float>::random(150, n, Layout::RowMajor, 5 + n);
        const auto ref = spmm_reference(a, x);
        CHECK(exact_equal(spmm_auto_layout(KernelId::from_index(0), a, x, {1, 8, 8}, Numerics::Exact), ref));
        CHECK(exact_equal(spmm_auto_layout(KernelId::from_index(2), a, x, {1, 8, 8}, Numerics::Exact), ref));
    }
}

CASE(WrongLayoutDimsAndConfigThrow) {
    const auto a = ragged_shape();
    const auto x_rm = DenseMatrix<double>::random(8, 2, Layout::RowMajor, 2);
    const auto x_cm = convert_layout(x_rm, Layout::ColMajor);
    CHECK(throws<std::invalid_argument>([&] { spmm(KernelId::parse("RB+CM+SR").value(), a, x_rm, {1, 4, 2}); }));
    CHECK(throws<std::invalid_argument>([&] { spmm(KernelId::parse("EB+RM+PR").value(), a, x_cm, {1, 4, 2}); }));
    const auto x7 = DenseMatrix<double>::random(7, 2, Layout::RowMajor, 2);
    CHECK(throws<std::invalid_argument>([&] { spmm(KernelId::from_index(0), a, x7, {1, 4, 2}); }));
    CHECK(throws<std::invalid_argument>([&] { spmm(KernelId::from_index(0), a, x_rm, {0, 4, 2}); }));
    CHECK(throws<std::invalid_argument>([&] { spmm(KernelId::from_index(0), a, x_rm, {1, 3, 2}); }));
    CHECK(throws<std::invalid_argument>([&] { spmm(KernelId::from_index(0), a, x_rm, {1, 4, 0}); }));
    CHECK(throws<std::out_of_range>([&] { KernelId::from_index(8); }));
}

CASE(ZeroMatrixAndZeroColumns) {
    const auto a = with_counts({0, 0, 0}, 4);
    const auto x = DenseMatrix<double>::random(4, 3, Layout::RowMajor, 3);
    for (auto k : all_kernels())
        for (double v : spmm_auto_layout(k, a, x, {2, 4, 2}).data) CHECK(v == 0.0);
    const auto b = ragged_shape();
    const auto x0 = DenseMatrix<double>::zeros(8, 0);
    for (auto k : all_kernels()) {
        const auto y = spmm_auto_layout(k, b, x0, {2, 4, 2});
        CHECK(y.num_rows == 5 && y.num_cols == 0);
    }
}

CASE(SingleColumnWideXAndFloat) {
    const auto a = random_csr(16, 16, 60, 41);
    for (Index n : {1, 128}) {
        const auto x = DenseMatrix<double>::random(16, n, Layout::RowMajor, 42 + n);
        const auto ref = spmm_reference(a, x);
        for (auto k : all_kernels()) CHECK(tolerance_equal(spmm_auto_layout(k, a, x, {2, 8, 4}), ref));
    }
    std::vector<std::tuple<Index, Index, float>> t;
    std::mt19937_64 rng(55);
    std::uniform_real_distribution<float> vd(-1.0f, 1.0f);
    for (Index r = 0; r < 12; ++r)
        for (Index c = 0; c < 10; ++c)
            if (rng() % 3 == 0) t.push_back({r, c, vd(rng)});
    const auto af = CsrMatrix<float>::from_coo(12, 10, t);
    const auto xf = DenseMatrix<float>::random(10, 4, Layout::RowMajor, 56);
    const auto reff = spmm_reference(af, xf);
    for (auto k : all_kernels()) CHECK(tolerance_equal(spmm_auto_layout(k, af, xf, {2, 4, 2}), reff));
}

CASE(GroupWidthWiderThanRows) {
    const auto a = ragged_shape();
    const auto x = DenseMatrix<double>::random(8, 3, Layout::RowMajor, 60);
    const auto ref = spmm_reference(a, x);
    for (auto k : all_kernels()) CHECK(tolerance_equal(spmm_auto_layout(k, a, x, {2, 16, 2}), ref));
}

CASE(MakeConfigRecommendedBlocks) {
    CHECK(recommended_col_block(KernelId::parse("RB+RM+PR").value(), 100) == 4);
    CHECK(recommended_col_block(KernelId::parse("RB+RM+SR").value(), 100) == 8);
    CHECK(recommended_col_block(KernelId::parse("EB+CM+PR").value(), 2) == 2);
    const auto cfg = make_config(KernelId::from_index(1), 16, 3, 4);
    CHECK(cfg.num_workers == 3 && cfg.group_width == 4 && cfg.col_block == 4 && is_valid(cfg));
}

// ---------------------------------------------------------------- partition / features
CASE(PartitionKnownAnswers) {
    auto p = partition_elements(with_counts({4, 3, 3}, 4), 4);
    CHECK(p.chunk_bounds[0].size() == 3 && p.chunk_bounds[2].size() == 2 && p.chunk_bounds[3].end == 10);
    p = partition_elements(with_counts({3, 3}, 4), 2);
    CHECK(p.row_of_chunk_start == (std::vector<Index>{0, 1}));
    p = partition_elements(with_counts({1, 1}, 2), 5);
    CHECK(p.row_of_chunk_start[2] == 2 && p.row_of_chunk_start[4] == 2);
    CHECK(throws<std::invalid_argument>([&] { partition_elements(with_counts({1}, 1), 0); }));
    const auto m = with_counts({2, 0, 3}, 4);
    CHECK(row_index_of(m, 2) == 2 && row_index_of(m, 1) == 0);
    CHECK(throws<std::out_of_range>([&] { row_index_of(m, 5); }));
}

CASE(FeaturesKnownAnswers) {
    CHECK(extract_features(with_counts({2, 2, 2}, 4), 16).std_row == 0.0);
    CHECK(extract_features(with_counts({1, 3}, 4), 8).std_row == 1.0);
    CHECK(extract_features(with_counts({4, 0, 0, 0}, 4), 2).std_row == std::sqrt(3.0));
    CHECK(throws<std::invalid_argument>([&] { extract_features(CsrMatrix<double>{}, 4); }));
    const auto f = extract_features(with_counts({1, 1}, 2), 4, 3);
    CHECK(f.hardware_id.has_value() && *f.hardware_id == 3);
}

// ---------------------------------------------------------------- selector
CASE(SelectorEncodeAndPredict) {
    FeatureVector f;
    f.nnz = 1024;
    f.mat_size = 256;
    f.std_row = 3.25;
    f.n_cols = 33;
    const auto e = encode_features(f, false);
    CHECK(e.size() == 4 && e[0] == 10.0 && e[1] == 8.0 && e[2] == 3.25 && e[3] == 33.0);
    CHECK(throws<std::invalid_argument>([&] { encode_features(f, true); }));
    // A hand-written ensemble: split on std_row at 4.0 -> class 0 or class 4.
    const std::string model =
        "spmmkit-selector v1\nuses_hardware 0\nspmmkit-gbdt v1\nclasses 8 features 4 best_round 0\n"
        "config num_rounds 1 max_depth 1 min_leaf 1 learning_rate 0.1 patience 1 lambda 1e-6 seed 0\n"
        "feature_names 4 log2_nnz log2_mat_size std_row n_cols\nrounds 1\n"
        "tree 0 0 3\nnode split 2 4 1 2 1\nnode leaf 1\nnode leaf 0\n"
        "tree 0 1 1\nnode leaf 0\ntree 0 2 1\nnode leaf 0\ntree 0 3 1\nnode leaf 0\n"
        "tree 0 4 3\nnode split 2 4 1 2 1\nnode leaf 0\nnode leaf 1\n"
        "tree 0 5 1\nnode leaf 0\ntree 0 6 1\nnode leaf 0\ntree 0 7 1\nnode leaf 0\nend\n";
    std::istringstream in(model);
    const auto sel = load_selector(in);
    f.std_row = 1.0;
    CHECK(predict_kernel(sel, f).index() == 0);
    f.std_row = 20.0;
    CHECK(predict_kernel(sel, f).index() == 4);
    std::istringstream bad("spmmkit-gbdt v1\n");
    CHECK(throws<ModelFormatError>([&] { load_selector(bad); }));
    // DA-SpMM through the C++ API: skewed rows pick EB and still match the oracle.
    const auto a = with_counts({40, 1, 1, 1, 1, 1, 1, 60}, 64);
    const auto x = DenseMatrix<double>::random(64, 8, Layout::RowMajor, 9);
    KernelId chosen;
    const auto y = spmm_selected(sel, a, x, &chosen);
    CHECK(chosen.index() == 4);
    CHECK(tolerance_equal(y, spmm_reference(a, x)));
}

// ---------------------------------------------------------------- matrix market
CASE(MatrixMarketReadsAndRejects) {
    std::istringstream in(
        "%%MatrixMarket matrix coordinate real symmetric\n% c\n3 3 3\n1 1 2.0\n3 1 -1.5\n2 2 4\n");
    const auto m = read_matrix_market<double>(in);
    CHECK(m.num_rows == 3 && m.nnz() == 4 && is_valid(m));
    std::istringstream bad("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 3\n");
    try {
        read_matrix_market<double>(bad);
        CHECK(false);
    } catch (const MatrixMarketError& e) {
        CHECK(e.line() == 3);
    }
    std::ostringstream out;
    write_matrix_market(out, m);
    std::istringstream back(out.str());
    const auto m2 = read_matrix_market<double>(back);
    CHECK(m2.values == m.values && m2.col_indices == m.col_indices);
}

CASE(ReductionsKnownAnswers) {
    const std::vector<double> v{0.1, 0.2, 0.3, 0.4};
    CHECK(tree_reduce(std::span<const double>(v)) == (0.1 + 0.2) + (0.3 + 0.4));
    const std::vector<double> w{1, 2, 3, 4};
    const std::vector<Index> ids{0, 0, 1, 1};
    const auto r = conditional_reduce(std::span<const double>(w), std::span<const Index>(ids));
    CHECK(r.sums.size() == 2 && r.sums[0].sum == 3.0 && r.sums[1].sum == 7.0 && r.carry);
}

int main() {
    for (auto& [name, fn] : registry()) {
        const int before = g_fail;
        try {
            fn();
        } catch (const std::exception& e) {
            ++g_fail;
            std::fprintf(stderr, "  FAIL %s: unexpected exception: %s\n", name, e.what());
        }
        std::printf("%s %s\n", g_fail == before ? "[ OK ]" : "[FAIL]", name);
    }
    std::printf("%d checks, %d failed\n", g_checks, g_fail);
    return g_fail > 255 ? 255 : g_fail;
}
