// EB+SR launchers (K4 EB+RM+SR, K6 EB+CM+SR) and the EB partition/zeroing prologue.
#define DASPMM_PDL_EXPR (p.pdl)
#include "launch_sr.cuh"
namespace daspmm {
// Fast path instantiations (CTA-combined boundary rows); the exact path keeps one
// partition chunk per group (k_eb_sr) so owned rows match the reference bit for bit.
// The CTA-combined walk's boundary slots are static shared memory: explicit carveout
// (DASPMM_CTA_CARVEOUT; default -1 = the driver's choice, being measured).
#define DASPMM_GO_CTA(K, G, NT)                                                          \
    do {                                                                                 \
        static const int carve_ = carveout_env("DASPMM_CTA_CARVEOUT", -1);               \
        carveout_once<K>(carve_);                                                        \
        DASPMM_GO(K, G, NT);                                                             \
    } while (0)
#define DASPMM_CTA_LPR_TABLE_NT(T, CM, V, NT)                                             \
    switch (p.L) {                                                                        \
        case 1: DASPMM_GO_CTA((k_eb_sr_cta<T, CM, V, 1, 1, NT>), p.grid, NT); break;          \
        case 2: DASPMM_GO_CTA((k_eb_sr_cta<T, CM, V, 2, 1, NT>), p.grid, NT); break;          \
        case 4: DASPMM_GO_CTA((k_eb_sr_cta<T, CM, V, 4, 1, NT>), p.grid, NT); break;          \
        case 8: DASPMM_GO_CTA((k_eb_sr_cta<T, CM, V, 8, 1, NT>), p.grid, NT); break;          \
        case 16: DASPMM_GO_CTA((k_eb_sr_cta<T, CM, V, 16, 1, NT>), p.grid, NT); break;        \
        case 32:                                                                          \
            if (p.X == 2) DASPMM_GO_CTA((k_eb_sr_cta<T, CM, V, 32, 2, NT>), p.grid, NT);      \
            else DASPMM_GO_CTA((k_eb_sr_cta<T, CM, V, 32, 1, NT>), p.grid, NT);               \
            break;                                                                        \
        default: return cudaErrorNotSupported;                                            \
    }
#define DASPMM_CTA_LPR_TABLE(T, CM, V)                                                    \
    if (p.cta_threads == 32) { DASPMM_CTA_LPR_TABLE_NT(T, CM, V, 32) }                    \
    else if (p.cta_threads == 64) { DASPMM_CTA_LPR_TABLE_NT(T, CM, V, 64) }               \
    else if (p.cta_threads == 128) { DASPMM_CTA_LPR_TABLE_NT(T, CM, V, 128) }             \
    else { DASPMM_CTA_LPR_TABLE_NT(T, CM, V, kThreads) }

template <typename T>
static cudaError_t launch_eb_sr_cta(const Plan& p, const SpmmArgs<T>& a, cudaStream_t s) {
    if (p.cm) {
        if (p.V != 1) return cudaErrorNotSupported;
        DASPMM_CTA_LPR_TABLE(T, true, 1)
    } else if (p.V == 1) {
        DASPMM_CTA_LPR_TABLE(T, false, 1)
    } else if (p.V == 2) {
        DASPMM_CTA_LPR_TABLE(T, false, 2)
    } else if constexpr (sizeof(T) == 4) {
        if (p.V == 4) { DASPMM_CTA_LPR_TABLE(T, false, 4) }
        else return cudaErrorNotSupported;
    } else {
        return cudaErrorNotSupported;
    }
    return cudaGetLastError();
}

template <typename T>
cudaError_t launch_eb_sr_per_chunk(const Plan&, const SpmmArgs<T>&, cudaStream_t);
#define launch_eb_sr launch_eb_sr_per_chunk
DASPMM_SR_LAUNCHER(launch_eb_sr, k_eb_sr)
#undef launch_eb_sr

template <int NT>
static cudaError_t launch_eb_sr_thr_nt(const Plan& p, const SpmmArgs<float>& a, cudaStream_t s) {
    // staging of 3 x S x NT words per CTA sizes the occupancy: explicit carveout
    // (DASPMM_THR_CARVEOUT; default -1 = the driver's choice, being measured)
    static const int carve = carveout_env("DASPMM_THR_CARVEOUT", -1);
    switch (p.V) {
        case 1:
            carveout_once<k_eb_sr_thr<float, false, 1, kThrS, NT>>(carve);
            DASPMM_GO((k_eb_sr_thr<float, false, 1, kThrS, NT>), p.grid, NT);
            break;
        case 2:
            carveout_once<k_eb_sr_thr<float, false, 2, kThrS, NT>>(carve);
            DASPMM_GO((k_eb_sr_thr<float, false, 2, kThrS, NT>), p.grid, NT);
            break;
        case 4:
            carveout_once<k_eb_sr_thr<float, false, 4, kThrS4, NT>>(carve);
            DASPMM_GO((k_eb_sr_thr<float, false, 4, kThrS4, NT>), p.grid, NT);
            break;
        default: return cudaErrorNotSupported;
    }
    return cudaGetLastError();
}

static cudaError_t launch_eb_sr_thr(const Plan& p, const SpmmArgs<float>& a, cudaStream_t s) {
    if (p.thr_threads == 32) return launch_eb_sr_thr_nt<32>(p, a, s);
    if (p.thr_threads == 64) return launch_eb_sr_thr_nt<64>(p, a, s);
    if (p.thr_threads == 128) return launch_eb_sr_thr_nt<128>(p, a, s);
    return launch_eb_sr_thr_nt<kThreads>(p, a, s);
}

template <>
cudaError_t launch_eb_sr<float>(const Plan& p, const SpmmArgs<float>& a, cudaStream_t s) {
    if (p.thr) return launch_eb_sr_thr(p, a, s);
    return p.cta ? launch_eb_sr_cta<float>(p, a, s) : launch_eb_sr_per_chunk<float>(p, a, s);
}
template <>
cudaError_t launch_eb_sr<double>(const Plan& p, const SpmmArgs<double>& a, cudaStream_t s) {
    return p.cta ? launch_eb_sr_cta<double>(p, a, s) : launch_eb_sr_per_chunk<double>(p, a, s);
}

template <typename T>
cudaError_t launch_eb_prep_uniform(const int* rows, int64_t nnz, int64_t sub, int64_t n_sub, int G,
                                   T* C, int64_t ldc, int N, const int* empty_rows, int n_empty,
                                   cudaStream_t s) {
    const int64_t stride = sub * G;  // boundaries at stride, 2*stride, ... (< nnz)
    const int64_t n_bound = n_sub > 0 ? (n_sub - 1) / G : 0;
    const bool v4 = sizeof(T) == 4 && N % 4 == 0 && ldc % 4 == 0 &&
                    (reinterpret_cast<uintptr_t>(C) & 15) == 0;
    const int vz = v4 ? 4 : 1;
    const int64_t nvec = (N + vz - 1) / vz;
    const int64_t work = (n_bound + n_empty) * nvec;
    if (work == 0) return cudaSuccess;
    const dim3 grid(unsigned((work + kThreads - 1) / kThreads));
    int shift = -1;
    if ((nvec & (nvec - 1)) == 0 && int64_t(grid.x) * kThreads < (int64_t(1) << 32))
        for (shift = 0; (int64_t(1) << shift) < nvec; ++shift) {}
    if (v4)
        k_eb_prep_uniform<T, (sizeof(T) == 4 ? 4 : 1)><<<grid, kThreads, 0, s>>>(
            rows, nnz, stride, n_bound, C, ldc, N, empty_rows, n_empty, shift);
    else
        k_eb_prep_uniform<T, 1><<<grid, kThreads, 0, s>>>(rows, nnz, stride, n_bound, C, ldc, N,
                                                          empty_rows, n_empty, shift);
    return cudaGetLastError();
}
template cudaError_t launch_eb_prep_uniform<float>(const int*, int64_t, int64_t, int64_t, int,
                                                   float*, int64_t, int, const int*, int,
                                                   cudaStream_t);
template cudaError_t launch_eb_prep_uniform<double>(const int*, int64_t, int64_t, int64_t, int,
                                                    double*, int64_t, int, const int*, int,
                                                    cudaStream_t);

template <typename T>
cudaError_t launch_eb_prep(const int* rp, int M, int64_t nnz, int64_t P, int* chunk_row, T* C,
                           int64_t ldc, int N, const int* empty_rows, int n_empty,
                           const int* rows, cudaStream_t s) {
    const int64_t work = P + int64_t(n_empty) * N;
    if (work == 0) return cudaSuccess;
    const int64_t blocks = (work + kThreads - 1) / kThreads;
    k_eb_prep<T><<<dim3(unsigned(blocks)), kThreads, 0, s>>>(rp, M, nnz, P, chunk_row, C, ldc, N,
                                                             empty_rows, n_empty, rows);
    return cudaGetLastError();
}
template cudaError_t launch_eb_prep<float>(const int*, int, int64_t, int64_t, int*, float*,
                                           int64_t, int, const int*, int, const int*, cudaStream_t);
template cudaError_t launch_eb_prep<double>(const int*, int, int64_t, int64_t, int*, double*,
                                            int64_t, int, const int*, int, const int*,
                                            cudaStream_t);
}  // namespace daspmm
