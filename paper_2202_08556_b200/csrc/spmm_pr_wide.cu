// PR design points (K1/K3 RB+PR, K5/K7 EB+PR) with group widths wider than a warp:
// W = 64 .. 1024 lanes, one CTA of W threads per group. The reference accepts any
// power-of-two group width (worker.hpp:29-40); the warp kernels (k_rb_pr / k_eb_pr,
// kernels.cuh) cover W <= 32, these the rest. Correctness, not speed, is their purpose:
// nobody tunes W > 32 on a GPU, but the API contract and the reference's bits must hold.
//
//   RB+PR (spmm.hpp:89-104): per W-tile of a row, the adjacent-pair merge tree over W
//     lanes (reduce.hpp:18-25) = the 32-lane tree inside each warp (group_tree_sum, bit
//     for bit) then the same tree over the W/32 warp totals; the row accumulator adds
//     each tile total in order, y += tile (bit-identical to the reference in exact mode).
//   EB+PR (spmm.hpp:160-184): per W-tile of the chunk, the gated conditional scan over W
//     lanes (reduce.hpp:31-39) run in shared memory — at distance d lane i adds lane i+d
//     when both hold the same row; every step reads the previous step's values, as the
//     reference's ascending in-place loop does; segment-start lanes deposit (owned row:
//     y += seg, first tile stores; split row: atomic add after the EB prologue).
// Columns are processed one at a time (scalar gathers, RM or CM), 32 per pass.
#include "dispatch.h"
#include "kernels.cuh"

namespace daspmm {

constexpr int kWideMax = 1024;

template <typename T, bool CM, bool EXACT>
__global__ void __launch_bounds__(kWideMax) k_rb_pr_wide(const SpmmArgs<T> a, int W) {
    __shared__ T wsum[32][33];  // [warp][column of the pass]
    const int nw = W >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int64_t row = blockIdx.x; row < a.M; row += gridDim.x) {
        const int rs = __ldg(a.rp + row), re = __ldg(a.rp + row + 1);
        for (int c0 = 0; c0 < a.N; c0 += 32) {
            const int cw = min(32, a.N - c0);
            T acc = T(0);
            for (int j = rs; j < re; j += W) {
                const int e = j + int(threadIdx.x);
                const bool valid = e < re;
                const int c = valid ? __ldg(a.ci + e) : 0;
                const T v = valid ? __ldg(a.va + e) : T(0);
                for (int q = 0; q < cw; ++q) {
                    T p = T(0);  // padded lanes contribute +0 (spmm.hpp:98-99)
                    if (valid) {
                        const T b = gather<T, CM, 1>(a, c, c0 + q).v[0];
                        p = EXACT ? mul_rn(v, b) : v * b;
                    }
                    p = group_tree_sum<32>(kFull, p);
                    if (lane == 0) wsum[warp][q] = p;
                }
                __syncthreads();
                if (threadIdx.x < unsigned(cw)) {
                    T t[32];
                    for (int w = 0; w < nw; ++w) t[w] = wsum[w][threadIdx.x];
                    for (int width = nw; width > 1; width >>= 1)
                        for (int i = 0; i < (width >> 1); ++i) t[i] = add_rn(t[2 * i], t[2 * i + 1]);
                    acc = EXACT ? add_rn(acc, t[0]) : acc + t[0];
                }
                __syncthreads();
            }
            if (threadIdx.x < unsigned(cw)) a.C[row * a.ldc + c0 + threadIdx.x] = acc;
        }
    }
}

template <typename T, bool CM, bool EXACT>
__global__ void __launch_bounds__(kWideMax) k_eb_pr_wide(const SpmmArgs<T> a, int W) {
    __shared__ T sv[kWideMax + 1];
    __shared__ int sid[kWideMax + 1];
    const int t = int(threadIdx.x);
    for (int64_t w = blockIdx.x; w < a.P; w += gridDim.x) {
        int64_t e0l, e1l;
        chunk_bounds(a.nnz, a.P, w, e0l, e1l);
        if (e0l >= e1l) continue;  // CTA-uniform
        const int e0 = int(e0l), e1 = int(e1l);
        const int first_row = __ldg(a.rows + e0), last_row = __ldg(a.rows + e1 - 1);
        const bool first_split = e0 > 0 && __ldg(a.rows + e0 - 1) == first_row;
        const bool last_split = e1 < a.nnz && __ldg(a.rows + e1) == last_row;
        int prev_last = e0 > 0 ? __ldg(a.rows + e0 - 1) : -1;
        for (int tb = e0; tb < e1; tb += W) {
            const int e = tb + t;
            const bool valid = e < e1;
            const int c = valid ? __ldg(a.ci + e) : 0;
            const T v = valid ? __ldg(a.va + e) : T(0);
            const int row = valid ? __ldg(a.rows + e) : a.M;  // sentinel pads (spmm.hpp:167)
            sid[t] = row;
            __syncthreads();
            const int before = t == 0 ? prev_last : sid[t - 1];
            const bool seg_start = valid && (t == 0 || sid[t - 1] != row);
            const bool first = before != row;
            const bool owned = !((first_split && row == first_row) || (last_split && row == last_row));
            for (int col = 0; col < a.N; ++col) {
                T p = T(0);
                if (valid) {
                    const T b = gather<T, CM, 1>(a, c, col).v[0];
                    p = EXACT ? mul_rn(v, b) : v * b;
                }
                sv[t] = p;
                __syncthreads();
                for (int d = 1; d < W; d <<= 1) {
                    const bool take = t + d < W && sid[t + d] == row;
                    const T o = take ? sv[t + d] : T(0);
                    __syncthreads();
                    if (take) sv[t] = add_rn(sv[t], o);
                    __syncthreads();
                }
                if (seg_start) {
                    T* y = a.C + int64_t(row) * a.ldc + col;
                    const T s = sv[t];
                    if (!owned) {
                        griddep_wait();
                        atomicAdd(y, s);
                    } else if (first) {
                        *y = EXACT ? add_rn(T(0), s) : s;
                    } else {
                        *y = add_rn(*y, s);
                    }
                }
                __syncthreads();  // sv is rewritten for the next column
            }
            prev_last = sid[min(W, e1 - tb) - 1];
            __syncthreads();  // sid is rewritten by the next tile
        }
    }
    griddep_wait();
}

template <typename T>
cudaError_t launch_pr_wide(const Plan& p, const SpmmArgs<T>& a, cudaStream_t s) {
    const int W = p.L;
    if (W < 64 || W > kWideMax || (W & (W - 1)) != 0 || p.V != 1) return cudaErrorNotSupported;
    const bool eb = p.kernel >= 4;
    const int64_t units = eb ? a.P : a.M;
    const dim3 grid(unsigned(std::max<int64_t>(1, std::min<int64_t>(units, 148 * 16))));
#define DASPMM_WIDE(CM, EX)                                                                  \
    return eb ? launch_k(p.pdl, k_eb_pr_wide<T, CM, EX>, grid, dim3(W), 0, s, a, W)        \
              : launch_k(false, k_rb_pr_wide<T, CM, EX>, grid, dim3(W), 0, s, a, W);
    if (p.cm) {
        if (p.exact) { DASPMM_WIDE(true, true) } else { DASPMM_WIDE(true, false) }
    } else {
        if (p.exact) { DASPMM_WIDE(false, true) } else { DASPMM_WIDE(false, false) }
    }
#undef DASPMM_WIDE
}
template cudaError_t launch_pr_wide<float>(const Plan&, const SpmmArgs<float>&, cudaStream_t);
template cudaError_t launch_pr_wide<double>(const Plan&, const SpmmArgs<double>&, cudaStream_t);

}  // namespace daspmm
