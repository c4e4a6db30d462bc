// daspmm — the reference's sequential std_row sum (features.hpp:27-35), reproduced bit for
// bit by a whole thread block instead of one thread.
//
// The reference computes S_i = fl(S_{i-1} + q_i), q_i = fl(fl(len_i - mean)^2) >= 0, in
// row order. While S stays inside one binade [2^e, 2^(e+1)) every double there is a
// multiple of u = 2^(e-52), and S is one too; so for a term that neither lands exactly
// half-way between two multiples (a tie) nor carries S out of the binade,
//     fl(S + q) = S + R(q),   R(q) = q rounded to the nearest multiple of u,
// independent of S. A run of such terms is an exact integer prefix sum in units of u.
// Proof sketch: with P_i = sum of R(q_j)/u up to i and sig = S/u in [2^52, 2^53), S + q_i
// stays below 2^(e+1) - u/2 exactly when sig + P_i < 2^53 and q_i is not a tie; then the
// nearest double is a multiple of u, namely S + R(q_i).
//
// So the block scans chunks of terms in parallel: each thread maps its terms to integers
// R(q)/u (flagging ties, and terms so large relative to S that R(q)/u >= 2^50), takes an
// exclusive prefix over the chunk, and the first term whose prefix reaches the binade end
// (or that is flagged) is added with a real IEEE double add, after which the next chunk
// starts in the new binade. Binade crossings are O(log(S_final / q_first)) (~25-60 per
// matrix), flagged terms rare (huge rows early in the sum, exact ties), so the chain of
// M dependent adds becomes M / (NT * kPer) block scans plus a few dozen single adds.
// S == 0 (leading all-zero terms) stays 0 until the first nonzero term, which S becomes
// exactly. tests/test_gpu_parity.py::test_exact_std_block_sum_matches_sequential checks
// the bits against the one-thread chain and the reference.
#pragma once

#include <climits>
#include <cstdint>

namespace daspmm {

constexpr int kStdPer = 8;  // consecutive terms per thread per chunk

__device__ __forceinline__ double std_term(const int* __restrict__ rp, int64_t r, double mean) {
    const double d = __dsub_rn(double(__ldg(rp + r + 1) - __ldg(rp + r)), mean);
    return __dmul_rn(d, d);
}

// Sum of the reference's per-row terms in row order with the reference's rounding,
// by all NT threads of the block (every thread must call it; returns the sum to all).
template <int NT>
__device__ double exact_sequential_sum(const int* __restrict__ rp, int64_t M, double mean) {
    static_assert(NT % 32 == 0 && NT <= 1024, "block of whole warps");
    constexpr int CH = NT * kStdPer;
    constexpr int NW = NT / 32;
    __shared__ double s_S;
    __shared__ long long s_k;
    __shared__ long long s_warp[NW];
    __shared__ int s_first;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) {
        s_S = 0.0;
        s_k = 0;
    }
    __syncthreads();
    while (true) {
        const double S = s_S;
        const long long k = s_k;
        if (k >= M) break;
        const long long i0 = k + int64_t(tid) * kStdPer;
        __syncthreads();  // everyone has read s_S / s_k
        if (tid == 0) s_first = INT_MAX;
        __syncthreads();
        if (S == 0.0) {
            // 0 + 0 = +0 until the first nonzero term, which S then becomes exactly.
            for (int j = 0; j < kStdPer; ++j) {
                const long long i = i0 + j;
                if (i < M && std_term(rp, i, mean) != 0.0) {
                    atomicMin(&s_first, int(i - k));
                    break;
                }
            }
            __syncthreads();
            if (tid == 0) {
                const int f = s_first;
                if (f == INT_MAX) {
                    s_k = k + CH;
                } else {
                    s_S = std_term(rp, k + f, mean);
                    s_k = k + f + 1;
                }
            }
            __syncthreads();
            continue;
        }
        if (!(S >= 0x1p-900)) {  // tiny S (unit below the normal range): one plain step
            if (tid == 0) {
                s_S = __dadd_rn(S, std_term(rp, k, mean));
                s_k = k + 1;
            }
            __syncthreads();
            continue;
        }
        const int e = ilogb(S);
        const double u = ldexp(1.0, e - 52), inv = ldexp(1.0, 52 - e);
        const long long sig = (long long)(S * inv);  // S / u, in [2^52, 2^53)
        const long long limit = (1LL << 53) - sig;   // prefix reaching it leaves the binade
        // this thread's terms as integers in units of u; flags stop the run
        long long r[kStdPer];
        long long tot = 0;
        int flag = -1;  // first flagged position of this thread
#pragma unroll
        for (int j = 0; j < kStdPer; ++j) {
            const long long i = i0 + j;
            r[j] = 0;
            if (i < M) {
                const double x = std_term(rp, i, mean) * inv;  // exact power-of-2 scaling
                if (!(x < 0x1p50)) {
                    if (flag < 0) flag = j;
                } else {
                    const double n = floor(x), f = x - n;
                    if (f == 0.5) {
                        if (flag < 0) flag = j;  // tie: the result depends on S's parity
                    } else {
                        r[j] = (long long)n + (f > 0.5 ? 1 : 0);
                    }
                }
            }
            tot += r[j];
        }
        // block-exclusive prefix of the thread totals
        long long incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) s_warp[wid] = incl;
        __syncthreads();
        if (wid == 0) {
            long long w = lane < NW ? s_warp[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const long long v = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += v;
            }
            if (lane < NW) s_warp[lane] = w;  // inclusive per warp
        }
        __syncthreads();
        long long P = (wid > 0 ? s_warp[wid - 1] : 0) + incl - tot;  // exclusive, this thread
        // first term (chunk order) that is flagged or carries the sum out of the binade
        int first = INT_MAX;
#pragma unroll
        for (int j = 0; j < kStdPer; ++j) {
            if (first != INT_MAX) break;
            if (j == flag) {
                first = tid * kStdPer + j;
                break;
            }
            P += r[j];
            if (P >= limit && i0 + j < M) first = tid * kStdPer + j;
        }
        if (first != INT_MAX) atomicMin(&s_first, first);
        __syncthreads();
        const int f = s_first;
        const long long n_chunk = (M - k) < CH ? (M - k) : CH;
        if (f == INT_MAX) {
            if (tid == NT - 1) {  // the last thread holds the chunk's total prefix
                const long long total = (wid > 0 ? s_warp[wid - 1] : 0) + incl;
                s_S = double(sig + total) * u;  // < 2^53 units: exact
                s_k = k + n_chunk;
            }
        } else if (f / kStdPer == tid) {  // the owner of the stopping term
            long long before = (wid > 0 ? s_warp[wid - 1] : 0) + incl - tot;
            for (int j = 0; j < f % kStdPer; ++j) before += r[j];
            const double S_prev = double(sig + before) * u;  // exact, inside the binade
            s_S = __dadd_rn(S_prev, std_term(rp, k + f, mean));
            s_k = k + f + 1;
        }
        __syncthreads();
    }
    return s_S;
}

}  // namespace daspmm
