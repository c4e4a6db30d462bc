// cuSPARSE SpMM comparator (the paper's baseline) — BENCH ONLY.
// Built into libdaspmm_cusparse.so, separate from the product library. Times
// cusparseSpMM on the same device matrix (int32 indices, fp32 values) with every CSR and
// COO SpMM algorithm, B and C row-major or column-major:
//   alg 0 DEFAULT, 1 CSR_ALG1, 2 CSR_ALG2, 3 CSR_ALG3, 4 COO_ALG1, 5 COO_ALG2,
//       6 COO_ALG3, 7 COO_ALG4
//   order 0 row-major (B K x N, ld >= N; C M x N, ld >= N), 1 column-major (B buffer N x K,
//       ld >= K; C buffer N x M, ld >= M)
// Combinations cuSPARSE rejects return nonzero from cmp_create and are skipped by the
// bench. CSR_ALG3's preprocessing is done once in cmp_create, outside the timed call (the
// paper also excluded preprocessing from its baselines).
#include <cuda_runtime.h>
#include <cusparse.h>

#include <cstdint>
#include <cstdio>

namespace {
thread_local char g_msg[256];
int fail(const char* what, int code) {
    snprintf(g_msg, sizeof(g_msg), "%s: %d", what, code);
    return code ? code : -1;
}
}  // namespace

struct cmp_plan {
    cusparseHandle_t h = nullptr;
    cusparseSpMatDescr_t A = nullptr;
    cusparseDnMatDescr_t B = nullptr, C = nullptr;
    cusparseSpMMAlg_t alg = CUSPARSE_SPMM_ALG_DEFAULT;
    void* buf = nullptr;
    size_t buf_size = 0;
};

extern "C" {

const char* cmp_last_error() { return g_msg; }

void cmp_destroy(cmp_plan* p) {
    if (!p) return;
    if (p->A) cusparseDestroySpMat(p->A);
    if (p->B) cusparseDestroyDnMat(p->B);
    if (p->C) cusparseDestroyDnMat(p->C);
    if (p->h) cusparseDestroy(p->h);
    cudaFree(p->buf);
    delete p;
}

int cmp_create(int64_t M, int64_t K, int64_t nnz, const int* rp, const int* ci, const int* coo_rows,
               const float* va, const float* B, int64_t N, int64_t ldb, float* C, int64_t ldc,
               int order, int alg, void* stream, cmp_plan** out) {
    *out = nullptr;
    if (alg < 0 || alg > 7 || (alg >= 4 && coo_rows == nullptr)) return fail("alg", -2);
    auto* p = new cmp_plan;
    auto bail = [&](const char* what, int s) {
        cmp_destroy(p);
        return fail(what, s);
    };
    cusparseStatus_t s;
    if ((s = cusparseCreate(&p->h)) != CUSPARSE_STATUS_SUCCESS) return bail("create", s);
    cusparseSetStream(p->h, static_cast<cudaStream_t>(stream));
    if (alg < 4)
        s = cusparseCreateCsr(&p->A, M, K, nnz, const_cast<int*>(rp), const_cast<int*>(ci),
                              const_cast<float*>(va), CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I,
                              CUSPARSE_INDEX_BASE_ZERO, CUDA_R_32F);
    else
        s = cusparseCreateCoo(&p->A, M, K, nnz, const_cast<int*>(coo_rows), const_cast<int*>(ci),
                              const_cast<float*>(va), CUSPARSE_INDEX_32I, CUSPARSE_INDEX_BASE_ZERO,
                              CUDA_R_32F);
    if (s != CUSPARSE_STATUS_SUCCESS) return bail("sparse", s);
    const cusparseOrder_t ord = order ? CUSPARSE_ORDER_COL : CUSPARSE_ORDER_ROW;
    if ((s = cusparseCreateDnMat(&p->B, K, N, ldb, const_cast<float*>(B), CUDA_R_32F, ord)) !=
        CUSPARSE_STATUS_SUCCESS)
        return bail("dnB", s);
    if ((s = cusparseCreateDnMat(&p->C, M, N, ldc, C, CUDA_R_32F, ord)) != CUSPARSE_STATUS_SUCCESS)
        return bail("dnC", s);
    const cusparseSpMMAlg_t algs[8] = {CUSPARSE_SPMM_ALG_DEFAULT, CUSPARSE_SPMM_CSR_ALG1,
                                       CUSPARSE_SPMM_CSR_ALG2,    CUSPARSE_SPMM_CSR_ALG3,
                                       CUSPARSE_SPMM_COO_ALG1,    CUSPARSE_SPMM_COO_ALG2,
                                       CUSPARSE_SPMM_COO_ALG3,    CUSPARSE_SPMM_COO_ALG4};
    p->alg = algs[alg];
    const float one = 1.f, zero = 0.f;
    if ((s = cusparseSpMM_bufferSize(p->h, CUSPARSE_OPERATION_NON_TRANSPOSE,
                                     CUSPARSE_OPERATION_NON_TRANSPOSE, &one, p->A, p->B, &zero,
                                     p->C, CUDA_R_32F, p->alg, &p->buf_size)) !=
        CUSPARSE_STATUS_SUCCESS)
        return bail("bufferSize", s);
    if (p->buf_size && cudaMalloc(&p->buf, p->buf_size) != cudaSuccess) {
        cudaGetLastError();
        p->buf = nullptr;
        return bail("buffer", -3);
    }
    if (alg == 3) {
        if ((s = cusparseSpMM_preprocess(p->h, CUSPARSE_OPERATION_NON_TRANSPOSE,
                                         CUSPARSE_OPERATION_NON_TRANSPOSE, &one, p->A, p->B, &zero,
                                         p->C, CUDA_R_32F, p->alg, p->buf)) !=
            CUSPARSE_STATUS_SUCCESS)
            return bail("preprocess", s);
    }
    *out = p;
    return 0;
}

int cmp_run(cmp_plan* p) {
    const float one = 1.f, zero = 0.f;
    cusparseStatus_t s = cusparseSpMM(p->h, CUSPARSE_OPERATION_NON_TRANSPOSE,
                                      CUSPARSE_OPERATION_NON_TRANSPOSE, &one, p->A, p->B, &zero,
                                      p->C, CUDA_R_32F, p->alg, p->buf);
    return s == CUSPARSE_STATUS_SUCCESS ? 0 : fail("spmm", s);
}

}  // extern "C"
