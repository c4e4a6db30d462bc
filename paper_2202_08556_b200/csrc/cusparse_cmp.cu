// cuSPARSE SpMM comparator (the paper's baseline) — BENCH ONLY.
// Built into libdaspmm_cusparse.so, separate from the product library. Times
// cusparseSpMM on the same device CSR (int32 offsets/cols, fp32 values) with each
// CSR algorithm; ALG3's preprocessing is done once outside the timed call.
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

// alg: 0 DEFAULT, 1 CSR_ALG1, 2 CSR_ALG2, 3 CSR_ALG3. B row-major K x N (ldb), C row-major.
int cmp_create(int64_t M, int64_t K, int64_t nnz, const int* rp, const int* ci, const float* va,
               const float* B, int64_t N, int64_t ldb, float* C, int64_t ldc, int alg,
               void* stream, cmp_plan** out) {
    auto* p = new cmp_plan;
    cusparseStatus_t s;
    if ((s = cusparseCreate(&p->h)) != CUSPARSE_STATUS_SUCCESS) return fail("create", s);
    cusparseSetStream(p->h, static_cast<cudaStream_t>(stream));
    if ((s = cusparseCreateCsr(&p->A, M, K, nnz, const_cast<int*>(rp), const_cast<int*>(ci),
                               const_cast<float*>(va), CUSPARSE_INDEX_32I, CUSPARSE_INDEX_32I,
                               CUSPARSE_INDEX_BASE_ZERO, CUDA_R_32F)) != CUSPARSE_STATUS_SUCCESS)
        return fail("csr", s);
    if ((s = cusparseCreateDnMat(&p->B, K, N, ldb, const_cast<float*>(B), CUDA_R_32F,
                                 CUSPARSE_ORDER_ROW)) != CUSPARSE_STATUS_SUCCESS)
        return fail("dnB", s);
    if ((s = cusparseCreateDnMat(&p->C, M, N, ldc, C, CUDA_R_32F, CUSPARSE_ORDER_ROW)) !=
        CUSPARSE_STATUS_SUCCESS)
        return fail("dnC", s);
    const cusparseSpMMAlg_t algs[4] = {CUSPARSE_SPMM_ALG_DEFAULT, CUSPARSE_SPMM_CSR_ALG1,
                                       CUSPARSE_SPMM_CSR_ALG2, CUSPARSE_SPMM_CSR_ALG3};
    p->alg = algs[alg & 3];
    const float one = 1.f, zero = 0.f;
    if ((s = cusparseSpMM_bufferSize(p->h, CUSPARSE_OPERATION_NON_TRANSPOSE,
                                     CUSPARSE_OPERATION_NON_TRANSPOSE, &one, p->A, p->B, &zero,
                                     p->C, CUDA_R_32F, p->alg, &p->buf_size)) !=
        CUSPARSE_STATUS_SUCCESS)
        return fail("bufferSize", s);
    if (p->buf_size) cudaMalloc(&p->buf, p->buf_size);
    if (alg == 3) {
        if ((s = cusparseSpMM_preprocess(p->h, CUSPARSE_OPERATION_NON_TRANSPOSE,
                                         CUSPARSE_OPERATION_NON_TRANSPOSE, &one, p->A, p->B, &zero,
                                         p->C, CUDA_R_32F, p->alg, p->buf)) !=
            CUSPARSE_STATUS_SUCCESS)
            return fail("preprocess", s);
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

void cmp_destroy(cmp_plan* p) {
    if (!p) return;
    if (p->A) cusparseDestroySpMat(p->A);
    if (p->B) cusparseDestroyDnMat(p->B);
    if (p->C) cusparseDestroyDnMat(p->C);
    if (p->h) cusparseDestroy(p->h);
    cudaFree(p->buf);
    delete p;
}

}  // extern "C"
