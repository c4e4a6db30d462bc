/*
 * TEST INFRASTRUCTURE ONLY — part of the CPU oracle (see oracle/daspmm_oracle.c).
 * Nothing in the product (paper_2202_08556_b200/, include/) may include or link this.
 *
 * Type-generic body, included twice by daspmm_oracle.c with
 *   REAL = double, SFX = f64   and   REAL = float, SFX = f32.
 * Every function restates the reference algorithm in plain C, in the reference's
 * evaluation order, so float results are bit-identical when the reference is built
 * without FMA contraction (its CMake uses no -march; we build with -ffp-contract=off).
 */

#define CAT_(a, b) a##_##b
#define CAT(a, b) CAT_(a, b)
#define FN(name) CAT(name, SFX)

/* spmm_reference — proj/include/spmmkit/spmm.hpp:16-32.
 * Row order, then column order, left-to-right accumulation from REAL(0).
 * X is K x N, RowMajor (x_cm == 0: x[k*N+n]) or ColMajor (x_cm != 0: x[n*K+k]).
 * Y is M x N RowMajor. */
void FN(oracle_spmm_reference)(int64_t M, int64_t K, int64_t N, const int64_t* rp,
                               const int64_t* ci, const REAL* va, const REAL* X, int x_cm,
                               REAL* Y) {
    for (int64_t m = 0; m < M; ++m) {
        for (int64_t n = 0; n < N; ++n) {
            REAL acc = (REAL)0;
            for (int64_t e = rp[m]; e < rp[m + 1]; ++e) {
                const REAL xv = x_cm ? X[n * K + ci[e]] : X[ci[e] * N + n];
                acc += va[e] * xv;
            }
            Y[m * N + n] = acc;
        }
    }
}

/* tree_reduce_lanes — reduce.hpp:18-25: adjacent-pair merge tree, in place,
 * lane-major storage (w lanes x `lanes` values). */
void FN(oracle_tree_reduce_lanes)(REAL* v, int64_t w, int64_t lanes) {
    for (int64_t half = w / 2; half >= 1; half /= 2)
        for (int64_t i = 0; i < half; ++i)
            for (int64_t c = 0; c < lanes; ++c)
                v[i * lanes + c] = v[2 * i * lanes + c] + v[(2 * i + 1) * lanes + c];
}

/* conditional_scan_lanes — reduce.hpp:31-39: gated suffix scan, d = 1,2,4..,
 * ascending i, lane i absorbs lane i+d when their ids match. */
void FN(oracle_conditional_scan_lanes)(REAL* v, const int64_t* ids, int64_t w,
                                       int64_t lanes) {
    for (int64_t d = 1; d < w; d *= 2)
        for (int64_t i = 0; i + d < w; ++i)
            if (ids[i] == ids[i + d])
                for (int64_t c = 0; c < lanes; ++c) v[i * lanes + c] += v[(i + d) * lanes + c];
}

/* One worker of spmm() — spmm.hpp:40-187 (spmm_worker<T,M,NL,K>), restated with
 * the design-space choices as runtime flags. Workers run serially, w = 0..P-1,
 * so split-row "atomic" deposits land in worker order. */
static void FN(worker)(int eb, int cm, int pr, int64_t M, int64_t K, int64_t N,
                       const int64_t* rp, const int64_t* ci, const REAL* va, const REAL* X,
                       REAL* Y, int64_t P, int64_t W, int64_t C, const int64_t* cb,
                       const int64_t* ce, const int64_t* crow, int64_t w, REAL* scratch,
                       int64_t* seg_rows, int64_t* seg_cols, REAL* seg_vals, int64_t* lane_ids,
                       REAL* acc) {
    /* spmm.hpp:46-50: column block and staging segment size */
    const int64_t nmax1 = N > 1 ? N : 1;
    const int64_t block = cm ? 1 : (C < nmax1 ? C : nmax1);
    const int64_t seg_cap = W > 256 ? W : 256;
#define XV(k, c) (cm ? X[(c) * K + (k)] : X[(k) * N + (c)])
    if (!eb) {
        /* spmm.hpp:66-107: contiguous row blocks balanced by row count */
        const int64_t base = M / P, extra = M % P;
        const int64_t r0 = w * base + (w < extra ? w : extra);
        const int64_t r1 = r0 + base + (w < extra ? 1 : 0);
        for (int64_t r = r0; r < r1; ++r) {
            const int64_t row_end = rp[r + 1];
            for (int64_t s = rp[r]; s < row_end; s += seg_cap) {
                const int64_t slen = seg_cap < row_end - s ? seg_cap : row_end - s;
                for (int64_t i = 0; i < slen; ++i) {
                    seg_cols[i] = ci[s + i];
                    seg_vals[i] = va[s + i];
                }
                for (int64_t c0 = 0; c0 < N; c0 += block) {
                    const int64_t cw = block < N - c0 ? block : N - c0;
                    REAL* yrow = Y + r * N + c0;
                    if (!pr) {
                        for (int64_t i = 0; i < slen; ++i)
                            for (int64_t c = 0; c < cw; ++c)
                                yrow[c] += seg_vals[i] * XV(seg_cols[i], c0 + c);
                    } else {
                        for (int64_t g = 0; g < slen; g += W) {
                            const int64_t glen = W < slen - g ? W : slen - g;
                            for (int64_t l = 0; l < glen; ++l)
                                for (int64_t c = 0; c < cw; ++c)
                                    scratch[l * cw + c] =
                                        seg_vals[g + l] * XV(seg_cols[g + l], c0 + c);
                            for (int64_t l = glen; l < W; ++l)
                                for (int64_t c = 0; c < cw; ++c) scratch[l * cw + c] = (REAL)0;
                            FN(oracle_tree_reduce_lanes)(scratch, W, cw);
                            for (int64_t c = 0; c < cw; ++c) yrow[c] += scratch[c];
                        }
                    }
                }
            }
        }
        return;
    }
    /* spmm.hpp:108-186: element-balanced chunk [e0, e1) */
    const int64_t e0 = cb[w], e1 = ce[w];
    if (e0 >= e1) return;
    const int64_t sentinel = M;
#define OWNS(row) (rp[(row)] >= e0 && rp[(row) + 1] <= e1)
    /* deposit: owned rows plain +=, split rows fetch_add (spmm.hpp:116-127);
     * serial execution makes both a plain add. */
#define DEPOSIT(row, vptr, c0_, cw_)                                          \
    do {                                                                     \
        REAL* yrow_ = Y + (row) * N + (c0_);                                 \
        for (int64_t c_ = 0; c_ < (cw_); ++c_) yrow_[c_] += (vptr)[c_];      \
    } while (0)
    int64_t r = crow[w];
    for (int64_t s = e0; s < e1; s += seg_cap) {
        const int64_t slen = seg_cap < e1 - s ? seg_cap : e1 - s;
        for (int64_t i = 0; i < slen; ++i) {
            while (rp[r + 1] <= s + i) ++r; /* steps over empty rows (spmm.hpp:140) */
            seg_rows[i] = r;
            seg_cols[i] = ci[s + i];
            seg_vals[i] = va[s + i];
        }
        if (!pr) {
            /* spmm.hpp:145-159 */
            for (int64_t c0 = 0; c0 < N; c0 += block) {
                const int64_t cw = block < N - c0 ? block : N - c0;
                int64_t cur = -1;
                for (int64_t i = 0; i < slen; ++i) {
                    if (seg_rows[i] != cur) {
                        if (cur >= 0) DEPOSIT(cur, acc, c0, cw);
                        cur = seg_rows[i];
                        for (int64_t c = 0; c < cw; ++c) acc[c] = (REAL)0;
                    }
                    for (int64_t c = 0; c < cw; ++c)
                        acc[c] += seg_vals[i] * XV(seg_cols[i], c0 + c);
                }
                if (cur >= 0) DEPOSIT(cur, acc, c0, cw);
            }
        } else {
            /* spmm.hpp:160-184 */
            for (int64_t g = 0; g < slen; g += W) {
                const int64_t glen = W < slen - g ? W : slen - g;
                for (int64_t l = 0; l < glen; ++l) lane_ids[l] = seg_rows[g + l];
                for (int64_t l = glen; l < W; ++l) lane_ids[l] = sentinel;
                for (int64_t c0 = 0; c0 < N; c0 += block) {
                    const int64_t cw = block < N - c0 ? block : N - c0;
                    for (int64_t l = 0; l < glen; ++l)
                        for (int64_t c = 0; c < cw; ++c)
                            scratch[l * cw + c] = seg_vals[g + l] * XV(seg_cols[g + l], c0 + c);
                    for (int64_t l = glen; l < W; ++l)
                        for (int64_t c = 0; c < cw; ++c) scratch[l * cw + c] = (REAL)0;
                    FN(oracle_conditional_scan_lanes)(scratch, lane_ids, W, cw);
                    for (int64_t l = 0; l < W; ++l) {
                        if (lane_ids[l] == sentinel) break;
                        if (l == 0 || lane_ids[l] != lane_ids[l - 1])
                            DEPOSIT(lane_ids[l], &scratch[l * cw], c0, cw);
                    }
                }
            }
        }
    }
#undef OWNS
#undef DEPOSIT
#undef XV
}

/* spmm() — spmm.hpp:194-271. Returns 0 on success, 1 invalid config
 * (worker.hpp:29-40), 2 dimension mismatch. Layout is the caller's flag:
 * kernels with n-bit set read X as ColMajor. Y (M x N RowMajor) is zero-filled
 * here, as the reference's DenseMatrix ctor does (types.hpp:166-168). */
int FN(oracle_spmm)(int kernel, int64_t P, int64_t W, int64_t C, int64_t M, int64_t K,
                    int64_t N, const int64_t* rp, const int64_t* ci, const REAL* va,
                    const REAL* X, REAL* Y) {
    if (kernel < 0 || kernel > 7) return 3;
    if (P < 1 || W < 2 || (W & (W - 1)) != 0 || C < 1) return 1;
    const int eb = kernel >= 4, cm = (kernel >> 1) & 1, pr = kernel & 1;
    for (int64_t i = 0; i < M * N; ++i) Y[i] = (REAL)0;
    const int64_t nnz = rp[M];
    int64_t *cb = NULL, *ce = NULL, *crow = NULL;
    if (eb) {
        cb = (int64_t*)malloc(sizeof(int64_t) * P);
        ce = (int64_t*)malloc(sizeof(int64_t) * P);
        crow = (int64_t*)malloc(sizeof(int64_t) * P);
        oracle_partition_elements(M, rp, P, cb, ce, crow);
    }
    (void)nnz;
    const int64_t seg_cap = W > 256 ? W : 256;
    const int64_t block = C > 0 ? C : 1;
    REAL* scratch = (REAL*)malloc(sizeof(REAL) * (size_t)(W * (block > N ? block : (N > 0 ? N : 1))));
    int64_t* seg_rows = (int64_t*)malloc(sizeof(int64_t) * seg_cap);
    int64_t* seg_cols = (int64_t*)malloc(sizeof(int64_t) * seg_cap);
    REAL* seg_vals = (REAL*)malloc(sizeof(REAL) * seg_cap);
    int64_t* lane_ids = (int64_t*)malloc(sizeof(int64_t) * W);
    REAL* acc = (REAL*)malloc(sizeof(REAL) * (size_t)(block > N ? block : (N > 0 ? N : 1)));
    for (int64_t w = 0; w < P; ++w)
        FN(worker)(eb, cm, pr, M, K, N, rp, ci, va, X, Y, P, W, C, cb, ce, crow, w, scratch,
                   seg_rows, seg_cols, seg_vals, lane_ids, acc);
    free(scratch);
    free(seg_rows);
    free(seg_cols);
    free(seg_vals);
    free(lane_ids);
    free(acc);
    free(cb);
    free(ce);
    free(crow);
    return 0;
}

#undef FN
#undef CAT
#undef CAT_
