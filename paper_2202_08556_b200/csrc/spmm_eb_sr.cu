// EB+SR launchers (K4 EB+RM+SR, K6 EB+CM+SR) and the EB partition/zeroing prologue.
#include "launch_sr.cuh"
namespace daspmm {
DASPMM_SR_LAUNCHER(launch_eb_sr, k_eb_sr)

template <typename T>
cudaError_t launch_eb_prep(const int* rp, int M, int64_t nnz, int64_t P, int* chunk_row, T* C,
                           int64_t ldc, int N, const int* empty_rows, int n_empty, cudaStream_t s) {
    const int64_t work = P + int64_t(n_empty) * N;
    if (work == 0) return cudaSuccess;
    const int64_t blocks = (work + kThreads - 1) / kThreads;
    k_eb_prep<T><<<dim3(unsigned(blocks)), kThreads, 0, s>>>(rp, M, nnz, P, chunk_row, C, ldc, N,
                                                             empty_rows, n_empty);
    return cudaGetLastError();
}
template cudaError_t launch_eb_prep<float>(const int*, int, int64_t, int64_t, int*, float*,
                                           int64_t, int, const int*, int, cudaStream_t);
template cudaError_t launch_eb_prep<double>(const int*, int, int64_t, int64_t, int*, double*,
                                            int64_t, int, const int*, int, cudaStream_t);
}  // namespace daspmm
