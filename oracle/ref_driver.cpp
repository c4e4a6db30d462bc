// TEST INFRASTRUCTURE ONLY — C-ABI shim over the *unmodified* reference headers.
//
// Compiled by oracle/Makefile against /root/reference/proj/include (read in place,
// never copied) with the reference's own release flags (-O3 -DNDEBUG -std=gnu++20,
// no -march: proj/CMakeLists.txt:3-10) into oracle/_ref/libspmmkit_ref.so.
// Used to (1) generate the golden fixtures under tests/golden/, (2) cross-check the
// C restatement (oracle/daspmm_oracle.c), and (3) serve as bench.py's CPU reference
// arm. Nothing in the product links it.
#include <chrono>
#include <cstring>
#include <sstream>
#include <string>

#include "spmmkit/spmmkit.hpp"

using namespace spmmkit;

namespace {
thread_local std::string g_err;

struct RefCsr {
    CsrMatrix<double> d;
    CsrMatrix<float> f;  // values static_cast to float, same structure
    void sync_float() {
        f.num_rows = d.num_rows;
        f.num_cols = d.num_cols;
        f.row_offsets = d.row_offsets;
        f.col_indices = d.col_indices;
        f.values.assign(d.values.begin(), d.values.end());
    }
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

template <class T>
DenseMatrix<T> dense_from(const T* x, Index rows, Index cols, int colmajor) {
    DenseMatrix<T> m(rows, cols, colmajor ? Layout::ColMajor : Layout::RowMajor);
    std::memcpy(m.data.data(), x, sizeof(T) * static_cast<std::size_t>(rows * cols));
    return m;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// generate_rmat — rmat.hpp:46-99 (values double, (0,1]).
void* ref_rmat(int scale, int64_t target_nnz, double a, double b, double c, double d,
               uint64_t seed) {
    RefCsr* h = new RefCsr;
    int rc = guarded([&] {
        RmatParams p;
        p.scale = scale;
        p.target_nnz = target_nnz;
        p.a = a;
        p.b = b;
        p.c = c;
        p.d = d;
        p.seed = seed;
        h->d = generate_rmat<double>(p);
        h->sync_float();
    });
    if (rc) {
        delete h;
        return nullptr;
    }
    return h;
}

// CsrMatrix::from_coo — types.hpp:56-90 (sorts, sums duplicates).
void* ref_csr_from_coo(int64_t rows, int64_t cols, int64_t n, const int64_t* r,
                       const int64_t* ci, const double* v) {
    RefCsr* h = new RefCsr;
    int rc = guarded([&] {
        std::vector<std::tuple<Index, Index, double>> t;
        t.reserve(n);
        for (int64_t i = 0; i < n; ++i) t.emplace_back(r[i], ci[i], v[i]);
        h->d = CsrMatrix<double>::from_coo(rows, cols, std::move(t));
        h->sync_float();
    });
    if (rc) {
        delete h;
        return nullptr;
    }
    return h;
}

// Takes CSR arrays verbatim (caller guarantees validity).
void* ref_csr_from_csr(int64_t rows, int64_t cols, const int64_t* rp, const int64_t* ci,
                       const double* v) {
    RefCsr* h = new RefCsr;
    h->d.num_rows = rows;
    h->d.num_cols = cols;
    h->d.row_offsets.assign(rp, rp + rows + 1);
    h->d.col_indices.assign(ci, ci + rp[rows]);
    h->d.values.assign(v, v + rp[rows]);
    h->sync_float();
    return h;
}

// MatrixMarket reader — matrix_market.hpp:60-139.
void* ref_read_matrix_market(const char* text) {
    RefCsr* h = new RefCsr;
    int rc = guarded([&] {
        std::istringstream in(text);
        h->d = read_matrix_market<double>(in);
        h->sync_float();
    });
    if (rc) {
        delete h;
        return nullptr;
    }
    return h;
}

void ref_csr_info(void* hp, int64_t* rows, int64_t* cols, int64_t* nnz) {
    auto* h = static_cast<RefCsr*>(hp);
    *rows = h->d.num_rows;
    *cols = h->d.num_cols;
    *nnz = h->d.nnz();
}

void ref_csr_copy(void* hp, int64_t* rp, int64_t* ci, double* v) {
    auto* h = static_cast<RefCsr*>(hp);
    std::memcpy(rp, h->d.row_offsets.data(), sizeof(int64_t) * h->d.row_offsets.size());
    std::memcpy(ci, h->d.col_indices.data(), sizeof(int64_t) * h->d.col_indices.size());
    std::memcpy(v, h->d.values.data(), sizeof(double) * h->d.values.size());
}

void ref_csr_free(void* hp) { delete static_cast<RefCsr*>(hp); }

// DenseMatrix::random — types.hpp:185-193; written in the requested layout.
void ref_dense_random_f64(int64_t rows, int64_t cols, int colmajor, uint64_t seed,
                          double* out) {
    auto m = DenseMatrix<double>::random(rows, cols,
                                         colmajor ? Layout::ColMajor : Layout::RowMajor, seed);
    std::memcpy(out, m.data.data(), sizeof(double) * m.data.size());
}
void ref_dense_random_f32(int64_t rows, int64_t cols, int colmajor, uint64_t seed,
                          float* out) {
    auto m = DenseMatrix<float>::random(rows, cols,
                                        colmajor ? Layout::ColMajor : Layout::RowMajor, seed);
    std::memcpy(out, m.data.data(), sizeof(float) * m.data.size());
}

// spmm_reference — spmm.hpp:16-32.
int ref_spmm_reference_f64(void* hp, const double* x, int64_t n, int x_colmajor, double* y) {
    auto* h = static_cast<RefCsr*>(hp);
    return guarded([&] {
        auto r = spmm_reference(h->d, dense_from(x, h->d.num_cols, n, x_colmajor));
        std::memcpy(y, r.data.data(), sizeof(double) * r.data.size());
    });
}
int ref_spmm_reference_f32(void* hp, const float* x, int64_t n, int x_colmajor, float* y) {
    auto* h = static_cast<RefCsr*>(hp);
    return guarded([&] {
        auto r = spmm_reference(h->f, dense_from(x, h->f.num_cols, n, x_colmajor));
        std::memcpy(y, r.data.data(), sizeof(float) * r.data.size());
    });
}

// spmm — spmm.hpp:194-271. X layout flag is passed through unchanged, so layout
// mismatches throw exactly as in the reference (return code 1, message kept).
int ref_spmm_f64(void* hp, int kernel, int64_t P, int64_t W, int64_t C, const double* x,
                 int64_t n, int x_colmajor, double* y) {
    auto* h = static_cast<RefCsr*>(hp);
    return guarded([&] {
        auto r = spmm(KernelId::from_index(kernel), h->d,
                      dense_from(x, h->d.num_cols, n, x_colmajor), WorkerConfig{P, W, C});
        std::memcpy(y, r.data.data(), sizeof(double) * r.data.size());
    });
}
int ref_spmm_f32(void* hp, int kernel, int64_t P, int64_t W, int64_t C, const float* x,
                 int64_t n, int x_colmajor, float* y) {
    auto* h = static_cast<RefCsr*>(hp);
    return guarded([&] {
        auto r = spmm(KernelId::from_index(kernel), h->f,
                      dense_from(x, h->f.num_cols, n, x_colmajor), WorkerConfig{P, W, C});
        std::memcpy(y, r.data.data(), sizeof(float) * r.data.size());
    });
}

// time_kernel_fn — bench.hpp:63-121, the reference's own timing protocol, on
// spmm() in fp32 (X pre-laid-out, as time_kernel does: bench.hpp:125-137).
// Returns median seconds via *median_s, min via *min_s.
int ref_time_spmm_f32(void* hp, int kernel, int64_t P, int64_t W, int64_t C, const float* x,
                      int64_t n, int reps, int warmup, double* median_s, double* min_s,
                      double* checksum) {
    auto* h = static_cast<RefCsr*>(hp);
    return guarded([&] {
        // kernel -1: spmm_reference (spmm.hpp:16-32), serial, row-major X
        const auto xk = dense_from(x, h->f.num_cols, n, kernel >= 0 && ((kernel >> 1) & 1));
        const KernelId k = KernelId::from_index(kernel >= 0 ? kernel : 0);
        const WorkerConfig cfg{P, W, C};
        FeatureVector fv;
        fv.n_cols = n;
        auto rec = kernel >= 0
                       ? time_kernel_fn<float>([&] { return spmm(k, h->f, xk, cfg); }, nullptr,
                                               "bench", fv, k, reps, warmup)
                       : time_kernel_fn<float>([&] { return spmm_reference(h->f, xk); }, nullptr,
                                               "bench", fv, k, reps, warmup);
        *median_s = rec.median_time;
        *min_s = rec.min_time;
        *checksum = rec.checksum;
    });
}

// One reference spmm() call timed alone (steady_clock around exactly the user's call,
// result dropped), on an X laid out once beforehand (as time_kernel does,
// bench.hpp:125-137): bench.py's reference arm times one pass of its workload per step
// this way, the same unit of work as the GPU arm's step.
void* ref_dense_f32(const float* x, int64_t rows, int64_t cols, int colmajor) {
    return new DenseMatrix<float>(dense_from(x, rows, cols, colmajor));
}
void ref_dense_free(void* d) { delete static_cast<DenseMatrix<float>*>(d); }
int ref_time_spmm_once_f32(void* hp, void* dp, int kernel, int64_t P, int64_t W, int64_t C,
                           double* seconds) {
    auto* h = static_cast<RefCsr*>(hp);
    const auto& x = *static_cast<const DenseMatrix<float>*>(dp);
    return guarded([&] {
        const KernelId k = KernelId::from_index(kernel);
        const auto t0 = std::chrono::steady_clock::now();
        auto y = spmm(k, h->f, x, WorkerConfig{P, W, C});
        const auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (y.data.empty() && x.num_cols > 0 && h->f.num_rows > 0) *seconds = -1.0;
    });
}

// spmm_reference (spmm.hpp:16-32, serial) timed once on a laid-out X, result dropped.
int ref_time_spmm_dense_reference_f32(void* hp, void* dp, double* seconds) {
    auto* h = static_cast<RefCsr*>(hp);
    const auto& x = *static_cast<const DenseMatrix<float>*>(dp);
    return guarded([&] {
        const auto t0 = std::chrono::steady_clock::now();
        auto y = spmm_reference(h->f, x);
        const auto t1 = std::chrono::steady_clock::now();
        *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (y.data.empty() && x.num_cols > 0 && h->f.num_rows > 0) *seconds = -1.0;
    });
}

// partition_elements — partition.hpp:45-64.
int ref_partition(void* hp, int p, int64_t* begin, int64_t* end, int64_t* row) {
    auto* h = static_cast<RefCsr*>(hp);
    return guarded([&] {
        auto part = partition_elements(h->d, p);
        for (int i = 0; i < p; ++i) {
            begin[i] = part.chunk_bounds[i].begin;
            end[i] = part.chunk_bounds[i].end;
            row[i] = part.row_of_chunk_start[i];
        }
    });
}

int ref_row_index_of(void* hp, int64_t e, int64_t* row) {
    auto* h = static_cast<RefCsr*>(hp);
    return guarded([&] { *row = row_index_of(h->d, e); });
}

// tree_reduce — reduce.hpp:46-55.
int ref_tree_reduce_f64(const double* v, int64_t n, double* out) {
    return guarded([&] { *out = tree_reduce(std::span<const double>(v, n)); });
}

// conditional_reduce — reduce.hpp:57-102. Writes per-segment (id, sum) pairs;
// *count receives the number of segments.
int ref_conditional_reduce_f64(const double* v, const int64_t* ids, int64_t n,
                               int64_t* seg_ids, double* sums, int64_t* count) {
    return guarded([&] {
        auto r = conditional_reduce(std::span<const double>(v, n),
                                    std::span<const Index>(ids, n));
        *count = static_cast<int64_t>(r.sums.size());
        for (std::size_t i = 0; i < r.sums.size(); ++i) {
            seg_ids[i] = r.sums[i].segment;
            sums[i] = r.sums[i].sum;
        }
    });
}

// extract_features — features.hpp:21-41.
int ref_extract_features(void* hp, int64_t n_cols, int64_t* nnz, int64_t* mat_size,
                         double* std_row) {
    auto* h = static_cast<RefCsr*>(hp);
    return guarded([&] {
        auto fv = extract_features(h->d, n_cols);
        *nnz = fv.nnz;
        *mat_size = fv.mat_size;
        *std_row = fv.std_row;
    });
}

// Selector: load_selector (selector.hpp:119-132) + predict_kernel (62-65).
void* ref_selector_load(const char* text) {
    SelectorModel* m = new SelectorModel;
    int rc = guarded([&] {
        std::istringstream in(text);
        *m = load_selector(in);
    });
    if (rc) {
        delete m;
        return nullptr;
    }
    return m;
}
void ref_selector_free(void* m) { delete static_cast<SelectorModel*>(m); }

int ref_selector_predict(void* mp, int64_t nnz, int64_t mat_size, double std_row,
                         int64_t n_cols, int64_t hw, int* kernel) {
    auto* m = static_cast<SelectorModel*>(mp);
    return guarded([&] {
        FeatureVector fv;
        fv.nnz = nnz;
        fv.mat_size = mat_size;
        fv.std_row = std_row;
        fv.n_cols = n_cols;
        if (hw >= 0) fv.hardware_id = static_cast<int>(hw);
        *kernel = predict_kernel(*m, fv).index();
    });
}

// train_selector (selector.hpp:41-60) on caller-supplied samples; returns the
// saved model text (save_selector, selector.hpp:113-117) in a malloc'd buffer.
// features: n x 4 (nnz, mat_size, std_row, n_cols) ; hw: n (or null) ;
// timings: n x 8 seconds. First n_train samples train, the rest validate.
char* ref_selector_train(int64_t n, int64_t n_train, const double* features,
                         const int64_t* hw, const double* timings, int rounds, int depth,
                         int min_leaf) {
    char* out = nullptr;
    guarded([&] {
        std::vector<TrainingSample> tr, va;
        for (int64_t i = 0; i < n; ++i) {
            FeatureVector fv;
            fv.nnz = static_cast<Index>(features[4 * i + 0]);
            fv.mat_size = static_cast<Index>(features[4 * i + 1]);
            fv.std_row = features[4 * i + 2];
            fv.n_cols = static_cast<Index>(features[4 * i + 3]);
            if (hw) fv.hardware_id = static_cast<int>(hw[i]);
            std::array<double, 8> t{};
            for (int k = 0; k < 8; ++k) t[k] = timings[8 * i + k];
            auto s = make_sample(fv, t, "s" + std::to_string(i));
            (i < n_train ? tr : va).push_back(std::move(s));
        }
        GbdtConfig cfg;
        cfg.num_rounds = rounds;
        cfg.max_depth = depth;
        cfg.min_leaf = min_leaf;
        auto model = train_selector(tr, va, cfg, hw != nullptr);
        std::ostringstream os;
        save_selector(os, model);
        const std::string s = os.str();
        out = static_cast<char*>(std::malloc(s.size() + 1));
        std::memcpy(out, s.c_str(), s.size() + 1);
    });
    return out;
}
void ref_free(void* p) { std::free(p); }

}  // extern "C"
