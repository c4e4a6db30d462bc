// daspmm — RB+CM+SR with lanes over rows (fp32 fast mode): the launch variant of the
// column-major design point (K2).
//
// With B column-major (column n is the contiguous vector B[n * ldb + k]), a gather of
// B[n][k] is one 4-byte element: the base walk puts the group's lanes on columns, so each
// warp load touches 32 columns = 32 different sectors for 32 useful floats, and every
// nonzero repeats that. Here a lane owns a ROW and the warp's 32 lanes are 32
// consecutive rows, all walking column n of B: on row-local matrices (the locality the
// paper credits CM with) neighbouring rows read neighbouring k, so a
// warp load coalesces into one or two lines; on scattered matrices it costs what the base
// walk costs. Columns are processed NB at a time with the grid's y dimension as the column
// block and x (scheduled first) over rows, so the B columns being gathered at any moment
// are NB vectors of K floats (32 MB at K = 2^20, NB = 8): L2-resident.
//
// Arithmetic: per output element fmaf over the row's nonzeros in CSR order from +0 — the
// base walk's sequence, so results are bit-identical to k_rb_sr<CM> in fast mode.
#include "dispatch.h"
#include "kernels.cuh"

namespace daspmm {

namespace {
constexpr int kCmThreads = 128;

template <int NB>
__global__ void __launch_bounds__(kCmThreads) k_rb_cm_rows(const SpmmArgs<float> a) {
    const int64_t r = int64_t(blockIdx.x) * kCmThreads + threadIdx.x;
    if (r >= a.M) return;
    const int n0 = blockIdx.y * NB;
    const int nb = min(NB, a.N - n0);
    const int e0 = __ldg(a.rp + r), e1 = __ldg(a.rp + r + 1);
    const float* Bn = a.B + int64_t(n0) * a.ldb;
    float acc[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) acc[i] = 0.f;
    constexpr int U = NB >= 8 ? 2 : 4;  // nonzeros in flight per step
    int e = e0;
    for (; e + U <= e1; e += U) {
        int c[U];
        float v[U];
        float b[U][NB];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            c[u] = __ldg(a.ci + e + u);
            v[u] = __ldg(a.va + e + u);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int i = 0; i < NB; ++i)
                b[u][i] = i < nb ? __ldg(Bn + int64_t(i) * a.ldb + c[u]) : 0.f;
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int i = 0; i < NB; ++i) acc[i] = fmaf(v[u], b[u][i], acc[i]);
    }
    for (; e < e1; ++e) {
        const int c = __ldg(a.ci + e);
        const float v = __ldg(a.va + e);
#pragma unroll
        for (int i = 0; i < NB; ++i)
            if (i < nb) acc[i] = fmaf(v, __ldg(Bn + int64_t(i) * a.ldb + c), acc[i]);
    }
    float* out = a.C + r * a.ldc + n0;
#pragma unroll
    for (int i = 0; i < NB; ++i)
        if (i < nb) __stcs(out + i, acc[i]);
}
}  // namespace

cudaError_t launch_rb_cm_rows(const Plan& p, const SpmmArgs<float>& a, cudaStream_t s) {
    switch (p.L) {
        case 1: k_rb_cm_rows<1><<<p.grid, kCmThreads, 0, s>>>(a); break;
        case 2: k_rb_cm_rows<2><<<p.grid, kCmThreads, 0, s>>>(a); break;
        case 4: k_rb_cm_rows<4><<<p.grid, kCmThreads, 0, s>>>(a); break;
        case 8: k_rb_cm_rows<8><<<p.grid, kCmThreads, 0, s>>>(a); break;
        default: return cudaErrorNotSupported;
    }
    return cudaGetLastError();
}

}  // namespace daspmm
