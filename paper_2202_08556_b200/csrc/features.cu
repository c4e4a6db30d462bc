// daspmm — selector features on the device (features.hpp:21-41) plus the handle's
// structural summaries (empty-row list for EB zeroing, distinct columns touched).
//
// The reference's std_row is a SEQUENTIAL double sum of per-row terms
// q_r = fl(fl(len_r - mean)^2) with mean = fl(nnz / M). Per-row terms are
// reproduced exactly here (__dsub_rn / __dmul_rn, no contraction); only the order
// of the sum differs. Any two summation orders of M non-negative terms agree to
// within relative 2*gamma_M, so the reference's value lies in a tight, provable
// interval [std_lo, std_hi] around the parallel sum. A tree threshold outside that
// interval is decided exactly; one inside it (never seen in practice) triggers the
// sequential replay kernel below, which reproduces the reference bits.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "exact_sum.cuh"
#include "internal.h"

namespace daspmm {

constexpr int kFeatThreads = 256;

__global__ void __launch_bounds__(kFeatThreads)
k_row_terms(const int* __restrict__ rp, int M, double mean, double* __restrict__ partial,
            int* __restrict__ empty_rows, unsigned long long* __restrict__ n_empty) {
    __shared__ double sm[kFeatThreads];
    double acc = 0.0;
    for (int64_t r = int64_t(blockIdx.x) * kFeatThreads + threadIdx.x; r < M;
         r += int64_t(gridDim.x) * kFeatThreads) {
        const int len = __ldg(rp + r + 1) - __ldg(rp + r);
        const double d = __dsub_rn(double(len), mean);
        acc = __dadd_rn(acc, __dmul_rn(d, d));
        if (len == 0) {
            const unsigned long long k = atomicAdd(n_empty, 1ull);
            empty_rows[k] = int(r);
        }
    }
    sm[threadIdx.x] = acc;
    __syncthreads();
    for (int s = kFeatThreads / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) sm[threadIdx.x] = __dadd_rn(sm[threadIdx.x], sm[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = sm[0];
}

// Distinct columns touched (K_touched): a byte per column set to 1 by every nonzero that
// finds it still 0 (a check before the store keeps hot power-law columns from becoming a
// stream of same-address writes; the race only ever writes 1), then the 1-bytes counted a
// word at a time (each byte is 0x00 or 0x01, so popc of the word counts them).
__global__ void k_cols_touched(const int* __restrict__ ci, int64_t nnz,
                               unsigned char* marks) {
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz;
         e += int64_t(gridDim.x) * blockDim.x) {
        const int c = __ldg(ci + e);
        if (marks[c] == 0) marks[c] = 1;  // a stale 0 only repeats the store
    }
}

__global__ void k_popcount(const unsigned* __restrict__ words_in, int64_t words,
                           unsigned long long* __restrict__ out) {
    unsigned long long acc = 0;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < words;
         i += int64_t(gridDim.x) * blockDim.x)
        acc += __popc(words_in[i]);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, acc);
}

// Replays features.hpp:27-35 in the reference's order with the reference's bits: the
// whole block runs the binade-wise exact prefix sum (exact_sum.cuh).
constexpr int kStdThreads = 1024;

__global__ void __launch_bounds__(kStdThreads) k_std_exact(const int* __restrict__ rp, int M,
                                                           DevFeatures* f) {
    const double ss = exact_sequential_sum<kStdThreads>(rp, M, f->mean);
    if (threadIdx.x == 0) {
        f->std_exact = __dsqrt_rn(__ddiv_rn(ss, double(M)));
        f->exact_valid = 1;
    }
}

// The same sum as one dependent chain of double adds (the reference's loop verbatim, one
// thread, terms staged by the block): the check the block sum is tested against
// (daspmm_debug_std_chain).
constexpr int kChainChunk = 4 * kStdThreads;

__global__ void __launch_bounds__(kStdThreads) k_std_chain(const int* __restrict__ rp, int M,
                                                           double mean, double* out) {
    __shared__ double q[kChainChunk];
    double ss = 0.0;
    for (int base = 0; base < M; base += kChainChunk) {
        const int n = min(kChainChunk, M - base);
        for (int i = threadIdx.x; i < n; i += kStdThreads) q[i] = std_term(rp, base + i, mean);
        __syncthreads();
        if (threadIdx.x == 0) {
#pragma unroll 16
            for (int i = 0; i < n; ++i) ss = __dadd_rn(ss, q[i]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = __dsqrt_rn(__ddiv_rn(ss, double(M)));
}

// One warp per row writes the row's id into its nonzeros' slots (COO expansion).
__global__ void k_coo_rows(const int* __restrict__ rp, int M, int* __restrict__ rows) {
    const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= M) return;
    const int r = int(warp);
    const int s = __ldg(rp + r), e = __ldg(rp + r + 1);
    for (int i = s + lane; i < e; i += 32) rows[i] = r;
}

int ensure_coo(const daspmm_csr* hc, cudaStream_t s) {
    daspmm_csr* h = const_cast<daspmm_csr*>(hc);
    std::lock_guard<std::mutex> lk(h->mu);
    if (h->coo_rows || h->nnz == 0) return DASPMM_OK;
    cudaError_t e = cudaMalloc(&h->coo_rows, sizeof(int32_t) * size_t(h->nnz));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(coo_rows)");
    const int64_t threads = h->M * 32;
    k_coo_rows<<<unsigned((threads + 255) / 256), 256, 0, s>>>(h->rp, int(h->M), h->coo_rows);
    e = cudaStreamSynchronize(s);
    return e == cudaSuccess ? DASPMM_OK : cuda_fail(e, "coo_rows");
}

// ---------------------------------------------------------------- dense row-panel tiles
// One warp per 8-row panel (tile.cuh): the panel's column window [lo, hi] and whether
// every row lists its columns in strictly ascending order (the tile walk adds a row's
// products in column order, which is the CSR order only then).
constexpr int kPanelRows = 8;

__global__ void k_tile_spans(const int* __restrict__ rp, const int* __restrict__ ci, int M,
                             int64_t n_pan, int* __restrict__ width, int* __restrict__ c0,
                             int* __restrict__ unsorted) {
    const int64_t p = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (p >= n_pan) return;
    const int r0 = int(p * kPanelRows), r1 = min(M, r0 + kPanelRows);
    int lo = INT_MAX, hi = -1;
    bool bad = false;
    for (int r = r0; r < r1; ++r) {
        const int s = __ldg(rp + r), e = __ldg(rp + r + 1);
        for (int i = s + lane; i < e; i += 32) {
            const int c = __ldg(ci + i);
            lo = min(lo, c);
            hi = max(hi, c);
            if (i + 1 < e && __ldg(ci + i + 1) <= c) bad = true;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) *unsorted = 1;
    if (lane == 0) {
        width[p] = hi >= lo ? hi - lo + 1 : 0;
        c0[p] = hi >= lo ? lo : 0;
    }
}

// Load-balanced forms of the two checks above, used once the COO row ids exist (they do
// whenever a fast RB+RM+SR call asks for tiles): rows are column-sorted iff no nonzero is
// followed, inside its row, by a column <= its own (one thread per nonzero); then a
// panel's window is [min first column, max last column] of its rows (one thread per
// panel, two loads per row). The warp-per-panel scan above takes as long as the longest
// panel, i.e. ~1.5 ms on a power-law 2^20-row matrix that can never be tiled.
__global__ void k_rows_unsorted(const int* __restrict__ ci, const int* __restrict__ rows,
                                int64_t nnz, int* __restrict__ unsorted) {
    bool bad = false;
    for (int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; e + 1 < nnz;
         e += int64_t(gridDim.x) * blockDim.x)
        bad |= __ldg(rows + e + 1) == __ldg(rows + e) && __ldg(ci + e + 1) <= __ldg(ci + e);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *unsorted = 1;
}

__global__ void k_tile_windows(const int* __restrict__ rp, const int* __restrict__ ci, int M,
                               int64_t n_pan, int* __restrict__ width, int* __restrict__ c0) {
    const int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= n_pan) return;
    const int r0 = int(p * kPanelRows), r1 = min(M, r0 + kPanelRows);
    int lo = INT_MAX, hi = -1;
    for (int r = r0; r < r1; ++r) {
        const int s = __ldg(rp + r), e = __ldg(rp + r + 1);
        if (s < e) {
            lo = min(lo, __ldg(ci + s));
            hi = max(hi, __ldg(ci + e - 1));
        }
    }
    width[p] = hi >= lo ? hi - lo + 1 : 0;
    c0[p] = hi >= lo ? lo : 0;
}

// One warp per panel: zero its tile, then place every nonzero at (col - c0, row - r0).
__global__ void k_tile_fill(const int* __restrict__ rp, const int* __restrict__ ci,
                            const float* __restrict__ va, int M, int64_t n_pan,
                            const int* __restrict__ off, const int* __restrict__ c0,
                            float* __restrict__ val) {
    const int64_t p = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (p >= n_pan) return;
    const int o0 = off[p], o1 = off[p + 1], base = c0[p];
    for (int i = o0 + lane; i < o1; i += 32) val[i] = 0.f;
    __syncwarp();
    const int r0 = int(p * kPanelRows), r1 = min(M, r0 + kPanelRows);
    for (int r = r0; r < r1; ++r) {
        const int s = __ldg(rp + r), e = __ldg(rp + r + 1);
        for (int i = s + lane; i < e; i += 32)
            val[o0 + (__ldg(ci + i) - base) * kPanelRows + (r - r0)] = __ldg(va + i);
    }
}

// Builds the tiles once per handle when they pay: fp32, rows column-sorted, and at least
// DASPMM_TILE_FILL (default 0.5) of the tile cells holding a nonzero — then each staged
// B row serves >= 4 nonzeros and the tiles take no more bytes than CSR's (col, val).
int ensure_tiles(const daspmm_csr* hc, cudaStream_t s) {
    daspmm_csr* h = const_cast<daspmm_csr*>(hc);
    std::lock_guard<std::mutex> lk(h->mu);
    if (h->tile_state.load(std::memory_order_acquire) != 0) return DASPMM_OK;
    // Inside a caller's stream capture the build (allocation + synchronisation) cannot
    // run: that call takes the base walk and a later uncaptured call builds the tiles.
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return DASPMM_OK;
    }
    h->tile_state.store(-1, std::memory_order_relaxed);
    if (h->dtype != DASPMM_F32 || h->M <= 0 || h->nnz <= 0) return DASPMM_OK;
    static const double min_fill = [] {
        const char* e = getenv("DASPMM_TILE_FILL");
        return e ? atof(e) : 0.5;
    }();
    if (min_fill > 1.0) return DASPMM_OK;  // DASPMM_TILE_FILL=2 turns the variant off
    const int64_t n_pan = (h->M + kPanelRows - 1) / kPanelRows;
    int *d_w = nullptr, *d_bad = nullptr;
    cudaError_t e = cudaMalloc(&d_w, sizeof(int) * size_t(n_pan));
    if (e == cudaSuccess) e = cudaMalloc(&h->tile_c0, sizeof(int) * size_t(n_pan));
    if (e == cudaSuccess) e = cudaMalloc(&d_bad, sizeof(int));
    if (e == cudaSuccess) e = cudaMemsetAsync(d_bad, 0, sizeof(int), s);
    if (e == cudaSuccess && h->coo_rows != nullptr) {
        const unsigned b1 = unsigned(std::min<int64_t>((h->nnz + 255) / 256, 148 * 16));
        k_rows_unsorted<<<std::max(b1, 1u), 256, 0, s>>>(h->ci, h->coo_rows, h->nnz, d_bad);
        k_tile_windows<<<unsigned((n_pan + 255) / 256), 256, 0, s>>>(h->rp, h->ci, int(h->M), n_pan,
                                                                    d_w, h->tile_c0);
        e = cudaGetLastError();
    } else if (e == cudaSuccess) {
        const int64_t threads = n_pan * 32;
        k_tile_spans<<<unsigned((threads + 255) / 256), 256, 0, s>>>(h->rp, h->ci, int(h->M), n_pan,
                                                                    d_w, h->tile_c0, d_bad);
        e = cudaGetLastError();
    }
    std::vector<int> w(size_t(n_pan), 0);
    int bad = 1;
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(w.data(), d_w, sizeof(int) * w.size(), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    cudaFree(d_w);
    cudaFree(d_bad);
    auto give_up = [&](cudaError_t err) {
        cudaFree(h->tile_c0);
        h->tile_c0 = nullptr;
        return err == cudaSuccess ? DASPMM_OK : cuda_fail(err, "tiles");
    };
    if (e != cudaSuccess) return give_up(e);
    std::vector<int> off(size_t(n_pan) + 1, 0);
    int64_t total = 0;
    for (int64_t p = 0; p < n_pan; ++p) {
        off[size_t(p)] = int(total);
        total += int64_t(w[size_t(p)]) * kPanelRows;
        if (total >= (int64_t(1) << 31) - 64) return give_up(cudaSuccess);
    }
    off[size_t(n_pan)] = int(total);
    h->tile_fill = total > 0 ? double(h->nnz) / double(total) : 0.0;
    if (bad || h->tile_fill < min_fill) return give_up(cudaSuccess);
    if ((e = cudaMalloc(&h->tile_off, sizeof(int) * off.size())) != cudaSuccess ||
        (e = cudaMalloc(&h->tile_val, sizeof(float) * size_t(std::max<int64_t>(total, 8)))) !=
            cudaSuccess ||
        (e = cudaMemcpyAsync(h->tile_off, off.data(), sizeof(int) * off.size(),
                             cudaMemcpyHostToDevice, s)) != cudaSuccess) {
        cudaFree(h->tile_off);
        cudaFree(h->tile_val);
        h->tile_off = nullptr;
        h->tile_val = nullptr;
        cudaGetLastError();
        return give_up(cudaSuccess);  // no room: the base walk serves the call
    }
    const int64_t threads = n_pan * 32;
    k_tile_fill<<<unsigned((threads + 255) / 256), 256, 0, s>>>(
        h->rp, h->ci, static_cast<const float*>(h->va), int(h->M), n_pan, h->tile_off, h->tile_c0,
        h->tile_val);
    if ((e = cudaGetLastError()) == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "tiles: fill");
    h->n_pan = n_pan;
    h->tile_state.store(1, std::memory_order_release);
    return DASPMM_OK;
}

// Column window of every 32-row fine panel, [min, max] column ({INT_MAX, -1} when the
// panel holds no nonzero). Load-balanced over nonzeros: a thread takes 64 consecutive
// nonzeros, finds the row of the first by binary search in row_offsets, walks them
// tracking the row (and so the panel), and merges each panel's run into spans[] with
// atomicMin / atomicMax — one warp per panel took as long as the densest panel (a
// power-law 2^20-row matrix: ~0.75 ms for one 100K-nonzero row).
constexpr int kSpanChunk = 64;

__global__ void k_spans_init(int64_t n_fine, int2* __restrict__ spans) {
    for (int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < n_fine;
         p += int64_t(gridDim.x) * blockDim.x)
        spans[p] = make_int2(INT_MAX, -1);
}

__global__ void k_fine_spans(const int* __restrict__ rp, const int* __restrict__ ci, int M,
                             int64_t nnz, int2* spans) {
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t e0 = t * kSpanChunk;
    if (e0 >= nnz) return;
    const int64_t e1 = min(nnz, e0 + kSpanChunk);
    // row holding e0: the last r with rp[r] <= e0 (upper_bound - 1)
    int lo_r = 0, hi_r = M;  // answer in [lo_r, hi_r)
    while (hi_r - lo_r > 1) {
        const int mid = (lo_r + hi_r) >> 1;
        if (__ldg(rp + mid) <= e0) lo_r = mid;
        else hi_r = mid;
    }
    int r = lo_r;
    int row_end = __ldg(rp + r + 1);
    int panel = r >> 5;
    int lo = INT_MAX, hi = -1;
    for (int64_t e = e0; e < e1; ++e) {
        while (e >= row_end) {  // next non-empty row
            ++r;
            row_end = __ldg(rp + r + 1);
        }
        if ((r >> 5) != panel) {
            atomicMin(&spans[panel].x, lo);
            atomicMax(&spans[panel].y, hi);
            panel = r >> 5;
            lo = INT_MAX;
            hi = -1;
        }
        const int c = __ldg(ci + e);
        lo = min(lo, c);
        hi = max(hi, c);
    }
    atomicMin(&spans[panel].x, lo);
    atomicMax(&spans[panel].y, hi);
}

// Fine-panel windows on the device plus, per panel height R = 32 << i, the widest and
// the mean window (host), which plan_spmm uses to size the window kernel's staging.
static int compute_spans(daspmm_csr* h, cudaStream_t s) {
    h->n_fine = (h->M + 31) / 32;
    if (h->n_fine == 0) return DASPMM_OK;
    cudaError_t e = cudaMalloc(&h->spans, sizeof(int2) * size_t(h->n_fine));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(spans)");
    k_spans_init<<<unsigned(std::min<int64_t>((h->n_fine + 255) / 256, 148 * 8)), 256, 0, s>>>(
        h->n_fine, h->spans);
    if (h->nnz > 0) {
        const int64_t threads = (h->nnz + kSpanChunk - 1) / kSpanChunk;
        k_fine_spans<<<unsigned((threads + 255) / 256), 256, 0, s>>>(h->rp, h->ci, int(h->M),
                                                                     h->nnz, h->spans);
    }
    std::vector<int2> hs(size_t(h->n_fine));
    if ((e = cudaGetLastError()) == cudaSuccess)
        e = cudaMemcpyAsync(hs.data(), h->spans, sizeof(int2) * hs.size(), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "spans");
    for (int i = 0; i < daspmm_csr::kSpanLevels; ++i) {
        const int64_t k = int64_t(1) << i;
        int64_t mx = 0, cnt = 0;
        double sum = 0.0;
        for (int64_t p = 0; p < h->n_fine; p += k) {
            int lo = INT_MAX, hi = -1;
            for (int64_t q = p; q < std::min(h->n_fine, p + k); ++q) {
                lo = std::min(lo, hs[q].x);
                hi = std::max(hi, hs[q].y);
            }
            if (hi < lo) continue;
            const int64_t w = int64_t(hi) - lo + 1;
            mx = std::max(mx, w);
            sum += double(w);
            ++cnt;
        }
        h->span_max[i] = mx;
        h->span_avg[i] = cnt ? sum / double(cnt) : 0.0;
    }
    return DASPMM_OK;
}

int compute_features(daspmm_csr* h, cudaStream_t s) {
    const int M = int(h->M);
    DevFeatures f{};
    f.nnz = h->nnz;
    f.rows = h->M;
    f.mean = M > 0 ? double(h->nnz) / double(M) : 0.0;
    cudaError_t e;
    if ((e = cudaMalloc(&h->d_feat, sizeof(DevFeatures))) != cudaSuccess)
        return cuda_fail(e, "cudaMalloc(features)");
    if (M > 0 && (e = cudaMalloc(&h->empty_rows, sizeof(int32_t) * size_t(M))) != cudaSuccess)
        return cuda_fail(e, "cudaMalloc(empty_rows)");

    int blocks = int(std::min<int64_t>((h->M + kFeatThreads - 1) / kFeatThreads, 2048));
    if (blocks < 1) blocks = 1;
    double* partial = nullptr;
    unsigned long long* counters = nullptr;  // [0] empty rows, [1] cols touched
    const int64_t words = (h->K + 3) / 4;  // one byte per column, counted per 32-bit word
    unsigned* bitmap = nullptr;
    if ((e = cudaMalloc(&partial, sizeof(double) * blocks)) != cudaSuccess)
        return cuda_fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&counters, sizeof(unsigned long long) * 2)) != cudaSuccess)
        return cuda_fail(e, "cudaMalloc");
    if ((e = cudaMalloc(&bitmap, sizeof(unsigned) * std::max<int64_t>(words, 1))) != cudaSuccess)
        return cuda_fail(e, "cudaMalloc");
    if ((e = cudaMemsetAsync(counters, 0, sizeof(unsigned long long) * 2, s)) != cudaSuccess ||
        (e = cudaMemsetAsync(bitmap, 0, sizeof(unsigned) * std::max<int64_t>(words, 1), s)) !=
            cudaSuccess)
        return cuda_fail(e, "features: memset");
    if (M > 0)
        k_row_terms<<<blocks, kFeatThreads, 0, s>>>(h->rp, M, f.mean, partial, h->empty_rows,
                                                     counters);
    if (h->nnz > 0) {
        const int b2 = int(std::min<int64_t>((h->nnz + 255) / 256, 148 * 16));
        k_cols_touched<<<b2, 256, 0, s>>>(h->ci, h->nnz, reinterpret_cast<unsigned char*>(bitmap));
        const int b3 = int(std::min<int64_t>((words + 255) / 256, 148 * 4));
        k_popcount<<<std::max(b3, 1), 256, 0, s>>>(bitmap, words, counters + 1);
    }
    std::vector<double> hp(blocks, 0.0);
    unsigned long long hc[2] = {0, 0};
    if ((e = cudaGetLastError()) != cudaSuccess) return cuda_fail(e, "features: launch");
    if (M > 0 && (e = cudaMemcpyAsync(hp.data(), partial, sizeof(double) * blocks,
                                      cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return cuda_fail(e, "features: copy");
    if ((e = cudaMemcpyAsync(hc, counters, sizeof(hc), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return cuda_fail(e, "features: copy");
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "features");
    trace_mark("features: kernels+sync");
    cudaFree(partial);
    cudaFree(counters);
    cudaFree(bitmap);
    h->n_empty = int64_t(hc[0]);
    h->cols_touched = int64_t(hc[1]);

    double ss = 0.0;
    for (double v : hp) ss += v;
    f.ss_par = ss;
    if (M > 0) {
        // |ss_ref - ss_par| <= 2 gamma_M * sum q (both orders of M non-negative terms);
        // widen by 4x and by a few ulps for the division and sqrt roundings.
        const double u = std::ldexp(1.0, -53);
        const double g = 8.0 * (double(M) + 8.0) * u;
        const double lo = std::max(0.0, ss * (1.0 - g)) / double(M);
        const double hi = ss * (1.0 + g) / double(M) + 1e-300;
        f.std_lo = std::sqrt(lo) * (1.0 - 8 * u);
        f.std_hi = std::sqrt(hi) * (1.0 + 8 * u);
        if (ss == 0.0) f.std_lo = f.std_hi = 0.0;  // every term is exactly 0 in any order
    }
    f.exact_valid = 0;
    if (M > 0 && ss == 0.0) {
        f.std_exact = 0.0;
        f.exact_valid = 1;
    }
    h->h_feat = f;
    if ((e = cudaMemcpyAsync(h->d_feat, &h->h_feat, sizeof(DevFeatures), cudaMemcpyHostToDevice,
                             s)) != cudaSuccess)
        return cuda_fail(e, "cudaMemcpy(features)");
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return cuda_fail(e, "features");
    trace_mark("features: host interval");
    return compute_spans(h, s);
}

int exact_std(daspmm_csr* h, double* out) {
    std::lock_guard<std::mutex> lk(h->mu);
    if (!h->h_feat.exact_valid) {
        DeviceGuard g(h->device);
        k_std_exact<<<1, kStdThreads>>>(h->rp, int(h->M), h->d_feat);
        cudaError_t e = cudaMemcpy(&h->h_feat, h->d_feat, sizeof(DevFeatures),
                                   cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_fail(e, "exact std");
    }
    *out = h->h_feat.std_exact;
    return DASPMM_OK;
}

int std_chain(const daspmm_csr* h, double* out) {
    DeviceGuard g(h->device);
    double* d = nullptr;
    cudaError_t e = cudaMalloc(&d, sizeof(double));
    if (e == cudaSuccess) {
        k_std_chain<<<1, kStdThreads>>>(h->rp, int(h->M), h->h_feat.mean, d);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpy(out, d, sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(d);
    return e == cudaSuccess ? DASPMM_OK : cuda_fail(e, "std_chain");
}

}  // namespace daspmm
