// spmmkit on B200 — the reference's C++ hot-path API (proj/include/spmmkit) with the
// compute moved behind the daspmm C ABI (include/daspmm.h, libdaspmm.so).
//
// Reference callers keep their code: the same names, signatures, value semantics and
// exception types. What changes is where the work runs: spmm(), extract_features()
// and partition_elements() execute hand-written sm_100a kernels; predict_kernel()
// evaluates the ensemble exactly as the reference. There is no CPU fallback — a host
// without a CUDA device gets std::runtime_error from the first device call.
//
// Header-only; link with -ldaspmm.
#pragma once

#include <daspmm.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <istream>
#include <iterator>
#include <memory>
#include <optional>
#include <random>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <tuple>
#include <vector>

namespace spmmkit {

using Index = std::int64_t;

// ------------------------------------------------------------------ errors
/// Thrown for a malformed selector/model stream (gbdt.hpp:301-303).
struct ModelFormatError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

namespace b200 {
/// Rethrows a daspmm status as the exception type the reference throws.
inline void raise_if(int rc) {
    if (rc == DASPMM_OK) return;
    const std::string msg = daspmm_last_error();
    switch (rc) {
        case DASPMM_ERR_INVALID_CONFIG:
        case DASPMM_ERR_DIMS:
        case DASPMM_ERR_LAYOUT:
        case DASPMM_ERR_INVALID_ARG: throw std::invalid_argument(msg);
        case DASPMM_ERR_OUT_OF_RANGE: throw std::out_of_range(msg);
        case DASPMM_ERR_MODEL_FORMAT: throw ModelFormatError(msg);
        default: throw std::runtime_error("daspmm: " + msg);
    }
}
template <class T>
constexpr int dtype_of() {
    static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>,
                  "spmmkit (B200) computes in float or double");
    return std::is_same_v<T, float> ? DASPMM_F32 : DASPMM_F64;
}
}  // namespace b200

// ------------------------------------------------------------------ layouts and dense
enum class Layout { RowMajor, ColMajor };

inline const char* layout_name(Layout l) { return l == Layout::RowMajor ? "RowMajor" : "ColMajor"; }

/// Dense operand/result (types.hpp:158-194). Element (r, c) is at r*cols + c when
/// RowMajor, c*rows + r when ColMajor; the constructor zero-fills.
template <class T>
struct DenseMatrix {
    Index num_rows = 0;
    Index num_cols = 0;
    Layout layout = Layout::RowMajor;
    std::vector<T> data;

    DenseMatrix() = default;
    DenseMatrix(Index rows, Index cols, Layout l = Layout::RowMajor)
        : num_rows(rows), num_cols(cols), layout(l), data(std::size_t(rows) * std::size_t(cols)) {}

    std::size_t index_of(Index r, Index c) const {
        return layout == Layout::RowMajor ? std::size_t(r) * num_cols + c
                                          : std::size_t(c) * num_rows + r;
    }
    T& at(Index r, Index c) { return data[index_of(r, c)]; }
    const T& at(Index r, Index c) const { return data[index_of(r, c)]; }

    static DenseMatrix zeros(Index rows, Index cols, Layout l = Layout::RowMajor) {
        return DenseMatrix(rows, cols, l);
    }
    /// Uniform [-1, 1] fill in logical (row, col) order, so a seed names the same
    /// logical matrix in either layout (types.hpp:185-193).
    static DenseMatrix random(Index rows, Index cols, Layout l, std::uint64_t seed) {
        DenseMatrix m(rows, cols, l);
        std::mt19937_64 gen(seed);
        std::uniform_real_distribution<double> u(-1.0, 1.0);
        for (Index r = 0; r < rows; ++r)
            for (Index c = 0; c < cols; ++c) m.at(r, c) = static_cast<T>(u(gen));
        return m;
    }
};

template <class T>
DenseMatrix<T> convert_layout(const DenseMatrix<T>& m, Layout target) {
    if (m.layout == target) return m;
    DenseMatrix<T> out(m.num_rows, m.num_cols, target);
    for (Index r = 0; r < m.num_rows; ++r)
        for (Index c = 0; c < m.num_cols; ++c) out.at(r, c) = m.at(r, c);
    return out;
}

// ------------------------------------------------------------------ CSR
/// Host CSR (types.hpp:28-91): int64 offsets and column indices, sorted columns.
template <class T>
struct CsrMatrix {
    Index num_rows = 0;
    Index num_cols = 0;
    std::vector<Index> row_offsets{0};
    std::vector<Index> col_indices;
    std::vector<T> values;

    Index nnz() const { return Index(col_indices.size()); }
    Index row_nnz(Index m) const { return row_offsets[m + 1] - row_offsets[m]; }

    static CsrMatrix identity(Index n) {
        CsrMatrix a;
        a.num_rows = a.num_cols = n;
        a.row_offsets.resize(n + 1);
        for (Index i = 0; i <= n; ++i) a.row_offsets[i] = i;
        a.col_indices.resize(n);
        for (Index i = 0; i < n; ++i) a.col_indices[i] = i;
        a.values.assign(n, T(1));
        return a;
    }

    /// Triplets in any order; duplicate coordinates are summed.
    static CsrMatrix from_coo(Index rows, Index cols,
                              std::vector<std::tuple<Index, Index, T>> triplets) {
        for (const auto& t : triplets) {
            const Index r = std::get<0>(t), c = std::get<1>(t);
            if (r < 0 || r >= rows || c < 0 || c >= cols)
                throw std::invalid_argument("from_coo: coordinate out of bounds");
        }
        std::stable_sort(triplets.begin(), triplets.end(), [](const auto& a, const auto& b) {
            return std::get<0>(a) != std::get<0>(b) ? std::get<0>(a) < std::get<0>(b)
                                                    : std::get<1>(a) < std::get<1>(b);
        });
        CsrMatrix m;
        m.num_rows = rows;
        m.num_cols = cols;
        m.row_offsets.assign(rows + 1, 0);
        for (std::size_t i = 0; i < triplets.size();) {
            auto [r, c, v] = triplets[i];
            std::size_t j = i + 1;
            for (; j < triplets.size() && std::get<0>(triplets[j]) == r &&
                   std::get<1>(triplets[j]) == c;
                 ++j)
                v += std::get<2>(triplets[j]);
            m.col_indices.push_back(c);
            m.values.push_back(v);
            ++m.row_offsets[r + 1];
            i = j;
        }
        for (Index r = 0; r < rows; ++r) m.row_offsets[r + 1] += m.row_offsets[r];
        return m;
    }
};

/// Invariant check (types.hpp:96-148): one message per violated invariant.
template <class T>
std::vector<std::string> validate(const CsrMatrix<T>& m) {
    std::vector<std::string> out;
    if (m.num_rows < 0) out.push_back("num_rows negative");
    if (m.num_cols < 0) out.push_back("num_cols negative");
    if (m.col_indices.size() != m.values.size())
        out.push_back("nnz mismatch: col_indices length " + std::to_string(m.col_indices.size()) +
                      " vs values length " + std::to_string(m.values.size()));
    if (Index(m.row_offsets.size()) != m.num_rows + 1) {
        out.push_back("row_offsets length " + std::to_string(m.row_offsets.size()) +
                      ", expected num_rows+1 = " + std::to_string(m.num_rows + 1));
        return out;
    }
    if (m.row_offsets[0] != 0) out.push_back("row_offsets[0] != 0");
    bool mono = true;
    for (Index i = 1; i <= m.num_rows && mono; ++i)
        if (m.row_offsets[i] < m.row_offsets[i - 1]) {
            out.push_back("row_offsets nondecreasing violated at index " + std::to_string(i));
            mono = false;
        }
    if (m.row_offsets[m.num_rows] != m.nnz())
        out.push_back("row_offsets[num_rows] = " + std::to_string(m.row_offsets[m.num_rows]) +
                      " != nnz = " + std::to_string(m.nnz()));
    for (Index i = 0; i < m.nnz(); ++i)
        if (m.col_indices[i] < 0 || m.col_indices[i] >= m.num_cols) {
            out.push_back("col index bound violated at index " + std::to_string(i) + " (col " +
                          std::to_string(m.col_indices[i]) + ")");
            break;
        }
    if (mono && m.row_offsets[m.num_rows] == m.nnz()) {
        for (Index r = 0; r < m.num_rows; ++r)
            for (Index i = m.row_offsets[r] + 1; i < m.row_offsets[r + 1]; ++i)
                if (m.col_indices[i] <= m.col_indices[i - 1]) {
                    out.push_back("columns strictly increasing violated in row " +
                                  std::to_string(r) + " at index " + std::to_string(i));
                    return out;
                }
    }
    return out;
}

template <class T>
bool is_valid(const CsrMatrix<T>& m) {
    return validate(m).empty();
}

// ------------------------------------------------------------------ design space
enum class MChoice : std::uint8_t { RB = 0, EB = 1 };
enum class NChoice : std::uint8_t { RM = 0, CM = 1 };
enum class KChoice : std::uint8_t { SR = 0, PR = 1 };

/// One of the 8 design-space kernels; index = 4m + 2n + k (kernel_id.hpp:12-76).
struct KernelId {
    MChoice m = MChoice::RB;
    NChoice n = NChoice::RM;
    KChoice k = KChoice::SR;

    int index() const { return int(m) * 4 + int(n) * 2 + int(k); }
    static KernelId from_index(int i) {
        if (i < 0 || i > 7) throw std::out_of_range("KernelId index must be 0..7");
        return {MChoice(i >> 2), NChoice((i >> 1) & 1), KChoice(i & 1)};
    }
    std::string name() const {
        static constexpr const char* kM[] = {"RB", "EB"};
        static constexpr const char* kN[] = {"RM", "CM"};
        static constexpr const char* kK[] = {"SR", "PR"};
        return std::string(kM[int(m)]) + "+" + kN[int(n)] + "+" + kK[int(k)];
    }
    static std::optional<KernelId> parse(std::string_view s) {
        for (int i = 0; i < 8; ++i)
            if (from_index(i).name() == s) return from_index(i);
        return std::nullopt;
    }
    friend bool operator==(const KernelId& a, const KernelId& b) { return a.index() == b.index(); }
    friend bool operator!=(const KernelId& a, const KernelId& b) { return !(a == b); }
    friend bool operator<(const KernelId& a, const KernelId& b) { return a.index() < b.index(); }
};

inline constexpr int kNumKernels = 8;

inline std::array<KernelId, kNumKernels> all_kernels() {
    std::array<KernelId, kNumKernels> ks;
    for (int i = 0; i < kNumKernels; ++i) ks[i] = KernelId::from_index(i);
    return ks;
}

inline int project_label(KernelId id, int dimension) {
    if (dimension == 0) return int(id.m);
    if (dimension == 1) return int(id.n);
    if (dimension == 2) return int(id.k);
    throw std::out_of_range("project_label: dimension must be 0..2");
}

/// P workers (EB chunk count on the GPU), W reduction width, C column block
/// (worker.hpp:18-27).
struct WorkerConfig {
    Index num_workers = 1;
    Index group_width = 8;
    Index col_block = 4;
    friend bool operator==(const WorkerConfig&, const WorkerConfig&) = default;
};

inline std::vector<std::string> validate(const WorkerConfig& cfg) {
    std::vector<std::string> out;
    if (cfg.num_workers < 1)
        out.push_back("num_workers must be >= 1, got " + std::to_string(cfg.num_workers));
    const Index w = cfg.group_width;
    if (w < 2 || (w & (w - 1)) != 0)
        out.push_back("group_width must be a power of two >= 2, got " + std::to_string(w));
    if (cfg.col_block < 1)
        out.push_back("col_block must be >= 1, got " + std::to_string(cfg.col_block));
    return out;
}
inline bool is_valid(const WorkerConfig& cfg) { return validate(cfg).empty(); }

inline Index recommended_col_block(KernelId kernel, Index n_cols) {
    return std::max<Index>(1, std::min<Index>(n_cols, kernel.k == KChoice::PR ? 4 : 8));
}
inline WorkerConfig make_config(KernelId kernel, Index n_cols, Index num_workers = 1,
                                Index group_width = 8) {
    return {num_workers, group_width, recommended_col_block(kernel, n_cols)};
}

// ------------------------------------------------------------------ device handle
/// RAII owner of a device-resident CSR (daspmm_csr). Build once, reuse across calls.
class DeviceCsr {
public:
    DeviceCsr() = default;
    template <class T>
    explicit DeviceCsr(const CsrMatrix<T>& a) {
        daspmm_csr* h = nullptr;
        b200::raise_if(daspmm_csr_create_host(a.num_rows, a.num_cols, a.nnz(),
                                              a.row_offsets.data(), a.col_indices.data(),
                                              a.values.data(), b200::dtype_of<T>(), &h));
        h_.reset(h);
    }
    daspmm_csr* get() const { return h_.get(); }

private:
    struct Del {
        void operator()(daspmm_csr* h) const { daspmm_csr_destroy(h); }
    };
    std::unique_ptr<daspmm_csr, Del> h_;
};

// ------------------------------------------------------------------ partition
struct ElementPartition {
    struct Chunk {
        Index begin = 0;
        Index end = 0;
        Index size() const { return end - begin; }
    };
    std::vector<Chunk> chunk_bounds;
    std::vector<Index> row_of_chunk_start;
};

/// partition.hpp:45-64, computed by the device partition kernel the EB path uses.
template <class T>
ElementPartition partition_elements(const CsrMatrix<T>& a, int p) {
    if (p < 1) throw std::invalid_argument("partition_elements: need p >= 1");
    DeviceCsr d(a);
    std::vector<Index> b(p), e(p), r(p);
    b200::raise_if(daspmm_partition(d.get(), p, b.data(), e.data(), r.data()));
    ElementPartition out;
    out.chunk_bounds.resize(p);
    out.row_of_chunk_start = r;
    for (int i = 0; i < p; ++i) out.chunk_bounds[i] = {b[i], e[i]};
    return out;
}

template <class T>
Index row_index_of(const CsrMatrix<T>& a, Index element_index) {
    if (element_index < 0 || element_index >= a.nnz())
        throw std::out_of_range("row_index_of: element index " + std::to_string(element_index) +
                                " out of range [0, " + std::to_string(a.nnz()) + ")");
    auto it = std::upper_bound(a.row_offsets.begin(), a.row_offsets.end(), element_index);
    return Index(it - a.row_offsets.begin()) - 1;
}

// ------------------------------------------------------------------ features
struct FeatureVector {
    Index nnz = 0;
    Index mat_size = 0;
    double std_row = 0.0;
    Index n_cols = 0;
    std::optional<int> hardware_id;
};

/// features.hpp:21-41 on the device; std_row carries the reference's bits.
inline FeatureVector extract_features(const DeviceCsr& d, Index n_cols,
                                      std::optional<int> hardware_id = std::nullopt) {
    FeatureVector f;
    b200::raise_if(daspmm_extract_features(d.get(), n_cols, &f.nnz, &f.mat_size, &f.std_row));
    f.n_cols = n_cols;
    f.hardware_id = hardware_id;
    return f;
}
template <class T>
FeatureVector extract_features(const CsrMatrix<T>& m, Index n_cols,
                               std::optional<int> hardware_id = std::nullopt) {
    if (m.num_rows == 0)
        throw std::invalid_argument("extract_features: matrix has no rows to summarize");
    return extract_features(DeviceCsr(m), n_cols, hardware_id);
}

// ------------------------------------------------------------------ selector
/// load_selector's result (selector.hpp:12-15): the ensemble, parsed and resident on
/// the device, plus the hardware-tag flag.
class SelectorModel {
public:
    bool uses_hardware = false;
    daspmm_model* get() const { return m_.get(); }
    static SelectorModel from_text(const std::string& text) {
        daspmm_model* m = nullptr;
        b200::raise_if(daspmm_model_parse(text.data(), text.size(), &m));
        SelectorModel s;
        s.m_.reset(m, daspmm_model_destroy);
        int uh = 0;
        daspmm_model_info(m, nullptr, nullptr, nullptr, &uh);
        s.uses_hardware = uh != 0;
        return s;
    }

private:
    std::shared_ptr<daspmm_model> m_;
};

inline SelectorModel load_selector(std::istream& in) {
    std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    return SelectorModel::from_text(text);
}

/// encode_features (selector.hpp:19-33).
inline std::vector<double> encode_features(const FeatureVector& f, bool uses_hardware) {
    std::vector<double> v{std::log2(double(std::max<Index>(f.nnz, 1))),
                          std::log2(double(std::max<Index>(f.mat_size, 1))), f.std_row,
                          double(f.n_cols)};
    if (uses_hardware) {
        if (!f.hardware_id)
            throw std::invalid_argument(
                "encode_features: model expects a hardware_id but the sample has none");
        v.push_back(double(*f.hardware_id));
    }
    return v;
}

/// predict_kernel (selector.hpp:62-65), evaluated as the reference does.
inline KernelId predict_kernel(const SelectorModel& model, const FeatureVector& f) {
    int k = 0;
    b200::raise_if(daspmm_model_predict_host(model.get(), f.nnz, f.mat_size, f.std_row, f.n_cols,
                                             f.hardware_id ? *f.hardware_id : -1, &k));
    return KernelId::from_index(k);
}

// ------------------------------------------------------------------ the hot path
/// Evaluation-order switch for spmm(): Fast fuses multiply-adds and lets the library
/// choose EB chunking (tolerance parity); Exact reproduces the reference's order and
/// honours cfg.num_workers as the EB chunk count (bit-identical results).
enum class Numerics { Fast, Exact };

namespace b200 {
template <class T>
DenseMatrix<T> run(KernelId kernel, const DeviceCsr& d, const CsrMatrix<T>& a,
                   const DenseMatrix<T>& x, const WorkerConfig& cfg, Numerics num) {
    DenseMatrix<T> y(a.num_rows, x.num_cols, Layout::RowMajor);
    const bool exact = num == Numerics::Exact;
    raise_if(daspmm_spmm_host(d.get(), kernel.index(), exact ? cfg.num_workers : 0,
                              cfg.group_width, cfg.col_block, x.data.data(),
                              x.layout == Layout::ColMajor ? DASPMM_COL_MAJOR : DASPMM_ROW_MAJOR,
                              x.num_cols, y.data.data(), exact ? DASPMM_EXACT : 0u));
    return y;
}

template <class T>
void check(KernelId kernel, const CsrMatrix<T>& a, const DenseMatrix<T>& x,
           const WorkerConfig& cfg) {
    if (const auto issues = validate(cfg); !issues.empty()) {
        std::string msg = "spmm: invalid config";
        for (const auto& s : issues) msg += "; " + s;
        throw std::invalid_argument(msg);
    }
    if (a.num_cols != x.num_rows)
        throw std::invalid_argument("spmm: A is " + std::to_string(a.num_rows) + "x" +
                                    std::to_string(a.num_cols) + " but X has " +
                                    std::to_string(x.num_rows) + " rows");
    const Layout want = kernel.n == NChoice::RM ? Layout::RowMajor : Layout::ColMajor;
    if (x.layout != want)
        throw std::invalid_argument("spmm: kernel " + kernel.name() + " needs " +
                                    layout_name(want) + " X, got " + layout_name(x.layout));
}
}  // namespace b200

/// spmm() — spmm.hpp:194-271 with the same checks, messages and value semantics,
/// computed on the B200.
template <class T>
DenseMatrix<T> spmm(KernelId kernel, const CsrMatrix<T>& a, const DenseMatrix<T>& x,
                    const WorkerConfig& cfg, Numerics num = Numerics::Fast) {
    b200::check(kernel, a, x, cfg);
    if (a.num_rows == 0 || x.num_cols == 0) return DenseMatrix<T>(a.num_rows, x.num_cols);
    return b200::run(kernel, DeviceCsr(a), a, x, cfg, num);
}

/// Same, reusing a device handle built from `a`.
template <class T>
DenseMatrix<T> spmm(KernelId kernel, const DeviceCsr& d, const CsrMatrix<T>& a,
                    const DenseMatrix<T>& x, const WorkerConfig& cfg,
                    Numerics num = Numerics::Fast) {
    b200::check(kernel, a, x, cfg);
    if (a.num_rows == 0 || x.num_cols == 0) return DenseMatrix<T>(a.num_rows, x.num_cols);
    return b200::run(kernel, d, a, x, cfg, num);
}

/// spmm.hpp:275-281.
template <class T>
DenseMatrix<T> spmm_auto_layout(KernelId kernel, const CsrMatrix<T>& a, const DenseMatrix<T>& x,
                                const WorkerConfig& cfg, Numerics num = Numerics::Fast) {
    const Layout want = kernel.n == NChoice::RM ? Layout::RowMajor : Layout::ColMajor;
    return x.layout == want ? spmm(kernel, a, x, cfg, num)
                            : spmm(kernel, a, convert_layout(x, want), cfg, num);
}

/// DA-SpMM: the selector picks the kernel from the matrix's features (extracted on the
/// device) and the chosen kernel runs — the reference's `predict --execute` flow
/// (spmmkit_cli.cpp:239-270) in one call.
template <class T>
DenseMatrix<T> spmm_selected(const SelectorModel& model, const CsrMatrix<T>& a,
                             const DenseMatrix<T>& x, KernelId* chosen = nullptr,
                             std::optional<int> hardware_id = std::nullopt) {
    DeviceCsr d(a);
    const FeatureVector f = extract_features(d, x.num_cols, hardware_id);
    const KernelId k = predict_kernel(model, f);
    if (chosen) *chosen = k;
    const WorkerConfig cfg = make_config(k, x.num_cols);
    const Layout want = k.n == NChoice::RM ? Layout::RowMajor : Layout::ColMajor;
    return x.layout == want ? spmm(k, d, a, x, cfg) : spmm(k, d, a, convert_layout(x, want), cfg);
}

// ------------------------------------------------------------------ reference oracle API
/// spmm_reference (spmm.hpp:16-32): the reference's sequential triple loop, kept in
/// the API because callers use it as their oracle. spmm() never calls it.
template <class T>
DenseMatrix<T> spmm_reference(const CsrMatrix<T>& a, const DenseMatrix<T>& x) {
    if (a.num_cols != x.num_rows)
        throw std::invalid_argument("spmm_reference: A is " + std::to_string(a.num_rows) + "x" +
                                    std::to_string(a.num_cols) + " but X has " +
                                    std::to_string(x.num_rows) + " rows");
    DenseMatrix<T> y(a.num_rows, x.num_cols, Layout::RowMajor);
    for (Index m = 0; m < a.num_rows; ++m)
        for (Index n = 0; n < x.num_cols; ++n) {
            T acc = T(0);
            for (Index e = a.row_offsets[m]; e < a.row_offsets[m + 1]; ++e)
                acc += a.values[e] * x.at(a.col_indices[e], n);
            y.at(m, n) = acc;
        }
    return y;
}

template <class T>
struct Tolerance;
template <>
struct Tolerance<double> {
    static constexpr double rtol = 1e-10;
    static constexpr double atol = 1e-12;
};
template <>
struct Tolerance<float> {
    static constexpr double rtol = 1e-3;
    static constexpr double atol = 1e-6;
};

template <class T>
bool tolerance_equal(const DenseMatrix<T>& y, const DenseMatrix<T>& ref,
                     double rtol = Tolerance<T>::rtol, double atol = Tolerance<T>::atol) {
    if (y.num_rows != ref.num_rows || y.num_cols != ref.num_cols) return false;
    for (Index r = 0; r < y.num_rows; ++r)
        for (Index c = 0; c < y.num_cols; ++c) {
            const double a = double(y.at(r, c)), b = double(ref.at(r, c));
            if (std::abs(a - b) > atol + rtol * std::abs(b)) return false;
        }
    return true;
}

// ------------------------------------------------------------------ reductions
/// The reduction networks the PR kernels implement with warp shuffles
/// (reduce.hpp:18-102), on the host with the reference's contract.
namespace detail {

/// Adjacent-pair merge tree over `w` slots of `lanes` values each (slot-major): level
/// by level slot i becomes slot 2i + slot 2i+1 until slot 0 holds the total. In place:
/// slot i is written only after slots 2i and 2i+1 (>= i) were read. reduce.hpp:18-25.
template <class T>
void tree_reduce_lanes(T* v, std::size_t w, std::size_t lanes) {
    for (std::size_t width = w; width > 1; width >>= 1) {
        const std::size_t pairs = width >> 1;
        for (std::size_t i = 0; i < pairs; ++i) {
            T* dst = v + i * lanes;
            const T* a = v + (2 * i) * lanes;
            const T* b = a + lanes;
            for (std::size_t c = 0; c < lanes; ++c) dst[c] = a[c] + b[c];
        }
    }
}

/// Gated suffix scan over `w` slots: at distance d = 1, 2, 4, ... slot i adds slot
/// i + d when both carry the same segment id, so each segment's first slot ends with
/// the segment total. Ascending i reads slot i + d before it is updated. reduce.hpp:31-39.
template <class T>
void conditional_scan_lanes(T* v, const Index* ids, std::size_t w, std::size_t lanes) {
    for (std::size_t d = 1; d < w; d <<= 1)
        for (std::size_t i = 0; i + d < w; ++i)
            if (ids[i] == ids[i + d]) {
                T* dst = v + i * lanes;
                const T* src = v + (i + d) * lanes;
                for (std::size_t c = 0; c < lanes; ++c) dst[c] += src[c];
            }
}

}  // namespace detail

template <class T>
T tree_reduce(std::span<const T> values) {
    const std::size_t w = values.size();
    if (w == 0 || (w & (w - 1)) != 0)
        throw std::invalid_argument("tree_reduce: length must be a power of two, got " +
                                    std::to_string(w));
    std::vector<T> v(values.begin(), values.end());
    detail::tree_reduce_lanes(v.data(), w, 1);
    return v[0];
}

template <class T>
struct SegmentSum {
    Index segment = 0;
    T sum = T(0);
    friend bool operator==(const SegmentSum&, const SegmentSum&) = default;
};
template <class T>
struct ConditionalReduceResult {
    std::vector<SegmentSum<T>> sums;
    bool carry = false;
};

template <class T>
ConditionalReduceResult<T> conditional_reduce(std::span<const T> values,
                                              std::span<const Index> ids) {
    if (values.size() != ids.size())
        throw std::invalid_argument("conditional_reduce: values and segment_ids differ in length");
    const std::size_t w = values.size();
    if (w == 0 || (w & (w - 1)) != 0)
        throw std::invalid_argument("conditional_reduce: length must be a power of two, got " +
                                    std::to_string(w));
    for (std::size_t i = 1; i < w; ++i)
        if (ids[i] < ids[i - 1])
            throw std::invalid_argument("conditional_reduce: segment_ids decreasing at index " +
                                        std::to_string(i));
    std::vector<T> v(values.begin(), values.end());
    detail::conditional_scan_lanes(v.data(), ids.data(), w, 1);
    ConditionalReduceResult<T> out;
    for (std::size_t i = 0; i < w; ++i)
        if (i == 0 || ids[i] != ids[i - 1]) out.sums.push_back({ids[i], v[i]});
    out.carry = !out.sums.empty();
    return out;
}

}  // namespace spmmkit
