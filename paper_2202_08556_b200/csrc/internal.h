// daspmm — internal handle layout and helpers shared by the ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/daspmm.h"

namespace daspmm {

// Per-handle selector features, resident on the device (features.hpp:13-41).
struct DevFeatures {
    int64_t nnz;
    int64_t rows;
    double mean;       // fl(nnz / M), the reference's `mean`
    double ss_par;     // parallel sum of the reference's per-row terms
    double std_lo;     // the reference's std_row lies in [std_lo, std_hi]
    double std_hi;
    double std_exact;  // reference bits, valid when exact_valid != 0
    int exact_valid;
    int pad;
};

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
void trace_mark(const char* what);  // DASPMM_DEBUG timing trace (nullptr resets)
int cuda_fail(cudaError_t e, const char* what);

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

}  // namespace daspmm

struct daspmm_csr {
    int64_t M = 0, K = 0, nnz = 0;
    int dtype = DASPMM_F32;
    int device = 0;
    int32_t* rp = nullptr;   // M+1
    int32_t* ci = nullptr;   // nnz
    void* va = nullptr;      // nnz
    bool owns = true;
    int32_t* empty_rows = nullptr;
    int64_t n_empty = 0;
    int64_t cols_touched = 0;
    daspmm::DevFeatures* d_feat = nullptr;  // device copy
    daspmm::DevFeatures h_feat{};           // host mirror (filled at creation)
    std::mutex mu;                          // guards the lazy exact-std cache
    void* graph_cache = nullptr;            // graph.cu
    int32_t* coo_rows = nullptr;            // EB kernels: row id per nonzero (built lazily)
    // Column windows (RB+SR window kernel): [min col, max col] of every 32-row fine panel
    // (device), and for panels of R = 32 << i rows the largest and mean window width.
    int2* spans = nullptr;
    int64_t n_fine = 0;
    static constexpr int kSpanLevels = 8;
    int64_t span_max[kSpanLevels] = {};
    double span_avg[kSpanLevels] = {};
    // Dense row-panel tiles of 8 rows (tile.cuh), fp32 only, built on the first fast
    // RB+RM+SR call (ensure_tiles) when rows are column-sorted and the tiles are at least
    // half full: tile_off[n_pan + 1] (floats), tile_c0[n_pan], tile_val (k-major tiles).
    // 0 not examined, 1 built, -1 not worth it. Written under mu (ensure_tiles), read
    // without it by the planner: release / acquire so a reader that sees 1 sees the
    // arrays below.
    std::atomic<int> tile_state{0};
    int64_t n_pan = 0;
    double tile_fill = 0.0;
    int32_t* tile_off = nullptr;
    int32_t* tile_c0 = nullptr;
    float* tile_val = nullptr;
    // Row-panel handles built by daspmm_multi_spmm (one per (parts, rank)), destroyed
    // with this handle (multi.cu).
    struct PanelEntry {
        int parts, rank;
        daspmm_csr* h;
    };
    std::vector<PanelEntry> panels;
};

namespace daspmm {
// Implemented in features.cu
int compute_features(daspmm_csr* h, cudaStream_t s);
// Builds h->coo_rows once (never call inside a stream capture).
int ensure_coo(const daspmm_csr* h, cudaStream_t s);
int exact_std(daspmm_csr* h, double* out);
// The reference's std_row as one dependent add chain (test hook for the block sum).
int std_chain(const daspmm_csr* h, double* out);
// Examines / builds h's dense row-panel tiles once (never call inside a stream capture).
int ensure_tiles(const daspmm_csr* h, cudaStream_t s);
// Implemented in abi.cu
struct Plan;
// base_only: the design point's base kernel (no lean / window / TMA launch variants).
Plan plan_spmm(const daspmm_csr* h, int kernel, int64_t P, int64_t W, int64_t N, const void* B,
               int64_t ldb, const void* C, int64_t ldc, bool exact, bool base_only = false);
int spmm_device(const daspmm_csr* h, int kernel, int64_t P, int64_t W, const void* B,
                int64_t ldb, int64_t N, void* C, int64_t ldc, unsigned flags, cudaStream_t s,
                int* chunk_scratch);
int check_call(const daspmm_csr* h, int kernel, int64_t P, int64_t W, int64_t Cb, int b_layout,
               int64_t ldb, int64_t N, int64_t ldc, bool exact);
// Stream-ordered scratch from the library's own per-device memory pool.
cudaError_t scratch_alloc(void** p, size_t bytes, int dev, cudaStream_t s);
cudaError_t scratch_free(void* p, cudaStream_t s);
cudaError_t transpose(int dtype, const void* in, int64_t rows, int64_t cols, int64_t ldi,
                      void* out, int64_t ldo, cudaStream_t s);
// Implemented in select.cu
int launch_select(const daspmm_csr* h, const daspmm_model* m, int64_t n_cols, int64_t hw,
                  int* d_kernel, cudaGraphConditionalHandle cond, bool use_cond, cudaStream_t s,
                  int* cache, int* publish);
uint64_t model_generation(const daspmm_model* m);
// Implemented in graph.cu
void graph_cache_free(daspmm_csr* h);
}  // namespace daspmm
