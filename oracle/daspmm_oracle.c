/*
 * daspmm CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference (spmmkit, /root/reference/proj/include/spmmkit)
 * algorithms on the DA-SpMM hot path. Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it, and only as the
 * checker / CPU baseline — never as the product path. The product (libdaspmm.so)
 * does not link it and has no CPU fallback.
 *
 * Parity pinning: tests/test_oracle_golden.py checks every function here against
 * golden vectors produced by the reference itself (oracle/_ref, built from the
 * reference headers by oracle/Makefile; fixtures committed under tests/golden/ with
 * the script that made them, tests/golden/make_golden.py).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fPIC -shared (no -march, matching the
 * reference's CMake flags proj/CMakeLists.txt:3-10, so float sums are not contracted
 * into FMAs and the bits equal the reference's).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

/* row_of_element — partition.hpp:27-30: upper_bound(row_offsets, e) - 1. */
int64_t oracle_row_of_element(int64_t M, const int64_t* rp, int64_t e) {
    int64_t lo = 0, hi = M + 1; /* search rp[0..M] */
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (rp[mid] <= e) lo = mid + 1;
        else hi = mid;
    }
    return lo - 1;
}

/* partition_elements — partition.hpp:45-64: p chunks of ceil/floor(nnz/p), larger
 * chunks first; chunk-start row by upper_bound, M for empty trailing chunks. */
int oracle_partition_elements(int64_t M, const int64_t* rp, int64_t p, int64_t* begin,
                              int64_t* end, int64_t* row) {
    if (p < 1) return 1;
    const int64_t nnz = rp[M];
    const int64_t base = nnz / p, extra = nnz % p;
    int64_t start = 0;
    for (int64_t i = 0; i < p; ++i) {
        const int64_t size = base + (i < extra ? 1 : 0);
        begin[i] = start;
        end[i] = start + size;
        row[i] = start < nnz ? oracle_row_of_element(M, rp, start) : M;
        start += size;
    }
    return 0;
}

/* extract_features — features.hpp:21-41: mean = nnz/M in double, sequential sum of
 * squared deviations, population std. Returns 1 when M == 0 (the reference throws). */
int oracle_extract_features(int64_t M, const int64_t* rp, double* std_row) {
    if (M == 0) return 1;
    const double mean = (double)rp[M] / (double)M;
    double ss = 0.0;
    for (int64_t r = 0; r < M; ++r) {
        const double d = (double)(rp[r + 1] - rp[r]) - mean;
        ss += d * d;
    }
    *std_row = sqrt(ss / (double)M);
    return 0;
}

/* encode_features — selector.hpp:19-33. hw < 0 means "no hardware_id". Returns the
 * feature count (4 or 5), or -1 when the model wants a tag the sample lacks. */
int oracle_encode_features(int64_t nnz, int64_t mat_size, double std_row, int64_t n_cols,
                           int uses_hardware, int64_t hw, double* out) {
    out[0] = log2((double)(nnz > 1 ? nnz : 1));
    out[1] = log2((double)(mat_size > 1 ? mat_size : 1));
    out[2] = std_row;
    out[3] = (double)n_cols;
    if (!uses_hardware) return 4;
    if (hw < 0) return -1;
    out[4] = (double)hw;
    return 5;
}

/* Tree::predict / TreeEnsembleModel::raw_scores / predict_class — gbdt.hpp:41-77.
 * The ensemble is flattened: tree t = round*num_classes + class owns nodes
 * [tree_off[t], tree_off[t+1]); child indices are tree-local as in the text format.
 * Per-class sums run over rounds in order from 0.0; argmax with strict '>' so ties go
 * to the lowest class. */
int oracle_predict_class(int num_classes, int num_rounds, const int64_t* tree_off,
                         const int32_t* feat, const double* thr, const int32_t* left,
                         const int32_t* right, const double* value, const double* f,
                         double* scores_out) {
    double s[64];
    if (num_classes > 64) return -1;
    for (int c = 0; c < num_classes; ++c) s[c] = 0.0;
    for (int r = 0; r < num_rounds; ++r)
        for (int c = 0; c < num_classes; ++c) {
            const int64_t base = tree_off[(int64_t)r * num_classes + c];
            int i = 0;
            while (feat[base + i] >= 0)
                i = f[feat[base + i]] <= thr[base + i] ? left[base + i] : right[base + i];
            s[c] += value[base + i];
        }
    int best = 0;
    for (int c = 1; c < num_classes; ++c)
        if (s[c] > s[best]) best = c;
    if (scores_out)
        for (int c = 0; c < num_classes; ++c) scores_out[c] = s[c];
    return best;
}

/* Tolerance / tolerance_equal — spmm.hpp:283-309: |y - ref| <= atol + rtol*|ref|.
 * Returns the number of violating elements. */
int64_t oracle_count_tolerance_violations_f64(int64_t n, const double* y, const double* ref,
                                              double rtol, double atol) {
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i)
        if (fabs(y[i] - ref[i]) > atol + rtol * fabs(ref[i])) ++bad;
    return bad;
}

/* Type-generic SpMM restatements (f64 then f32). */
#define REAL double
#define SFX f64
#include "oracle_body.h"
#undef REAL
#undef SFX

#define REAL float
#define SFX f32
#include "oracle_body.h"
#undef REAL
#undef SFX
