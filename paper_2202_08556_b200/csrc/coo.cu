// daspmm — CSR from (row, col, value) triplets on the device: CsrMatrix::from_coo
// (types.hpp:54-90) for inputs that already live in device memory (a MatrixMarket file
// parsed to COO, a generator, a graph pipeline), without a host sort.
//
//   1. bounds: the first triplet with a coordinate outside [0, M) x [0, K) fails with the
//      reference's message ("from_coo: coordinate out of bounds");
//   2. key = row << 32 | col, sorted with the triplet's index as payload
//      (cub::DeviceRadixSort, stable: duplicates keep their input order);
//   3. run heads (key differs from its predecessor) -> exclusive scan -> output slots;
//      each head sums its run left to right from its first value, the reference's
//      `v = v0; v += ...` loop (types.hpp:73-80) — for a duplicate-free input every value
//      passes through unchanged, so the CSR is bit-identical to from_coo's;
//   4. row counts of the unique entries -> exclusive scan -> int32 row offsets;
//   5. the arrays are adopted by a handle (daspmm_csr_create_device, owned).
// The reference sorts with std::sort, which leaves the order of duplicates unspecified;
// here they are summed in input order (a defined order; identical whenever a
// coordinate appears once).
#include <cub/cub.cuh>

#include <algorithm>

#include "internal.h"

namespace daspmm {
namespace {

__global__ void k_coo_keys(const int64_t* __restrict__ r, const int64_t* __restrict__ c,
                           int64_t n, int64_t M, int64_t K, uint64_t* __restrict__ keys,
                           int* __restrict__ idx, unsigned long long* __restrict__ bad) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t ri = r[i], ci = c[i];
        if (ri < 0 || ri >= M || ci < 0 || ci >= K) {
            atomicMin(bad, (unsigned long long)i);
            keys[i] = 0;
        } else {
            keys[i] = (uint64_t(ri) << 32) | uint64_t(ci);
        }
        idx[i] = int(i);
    }
}

__global__ void k_coo_heads(const uint64_t* __restrict__ keys, int64_t n, int* __restrict__ head) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        head[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

template <typename T>
__global__ void k_coo_merge(const uint64_t* __restrict__ keys, const int* __restrict__ perm,
                            const int* __restrict__ head, const int* __restrict__ slot, int64_t n,
                            const T* __restrict__ vals, int32_t* __restrict__ ci,
                            T* __restrict__ va, int* __restrict__ row_count) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        if (!head[i]) continue;
        const uint64_t k = keys[i];
        T v = vals[perm[i]];
        for (int64_t j = i + 1; j < n && keys[j] == k; ++j) v = v + vals[perm[j]];
        const int s = slot[i];
        ci[s] = int32_t(k & 0xffffffffu);
        va[s] = v;
        atomicAdd(row_count + (k >> 32), 1);
    }
}

int bits_for(int64_t v) {
    int b = 1;
    while (b < 31 && (int64_t(1) << b) <= v) ++b;
    return b;
}

}  // namespace
}  // namespace daspmm

using namespace daspmm;

extern "C" int daspmm_csr_create_coo_device(int64_t M, int64_t K, int64_t n,
                                            const int64_t* d_rows, const int64_t* d_cols,
                                            const void* d_vals, int dtype, daspmm_stream stream,
                                            daspmm_csr** out) {
    if (!out) return fail(DASPMM_ERR_INVALID_ARG, "from_coo: null out");
    *out = nullptr;
    if (dtype != DASPMM_F32 && dtype != DASPMM_F64)
        return fail(DASPMM_ERR_INVALID_ARG, "from_coo: dtype must be F32 or F64");
    if (M < 0 || K < 0 || n < 0 || M >= (int64_t(1) << 31) - 1 || K >= (int64_t(1) << 31) - 1 ||
        n >= (int64_t(1) << 31) - 1)
        return fail(DASPMM_ERR_INVALID_ARG, "from_coo: sizes must be in [0, 2^31 - 1)");
    if (n > 0 && (!d_rows || !d_cols || !d_vals))
        return fail(DASPMM_ERR_INVALID_ARG, "from_coo: null array");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t es = dtype == DASPMM_F64 ? 8 : 4;
    const size_t nn = size_t(std::max<int64_t>(n, 1));
    uint64_t *keys = nullptr, *keys_s = nullptr;
    int *idx = nullptr, *perm = nullptr, *head = nullptr, *slot = nullptr, *cnt = nullptr;
    unsigned long long* bad = nullptr;
    void* tmp = nullptr;
    int32_t *rp = nullptr, *ci = nullptr;
    void* va = nullptr;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cuda_fail(cudaGetLastError(), "from_coo");
    // Temporaries come from the library's stream-ordered pool (no device-wide
    // synchronisation or page mapping per call); the CSR arrays the handle adopts are
    // plain allocations it frees on destroy.
    auto release = [&](bool arrays) {
        for (void* p : {(void*)keys, (void*)keys_s, (void*)idx, (void*)perm, (void*)head,
                        (void*)slot, (void*)cnt, (void*)bad, tmp})
            scratch_free(p, s);
        cudaStreamSynchronize(s);
        if (arrays) cudaFree(rp), cudaFree(ci), cudaFree(va);
    };
    cudaError_t e = cudaSuccess;
    for (auto [p, b] : {std::pair<void**, size_t>{(void**)&keys, 8 * nn}, {(void**)&keys_s, 8 * nn},
                        {(void**)&idx, 4 * nn}, {(void**)&perm, 4 * nn}, {(void**)&head, 4 * nn},
                        {(void**)&slot, 4 * nn}, {(void**)&cnt, 4 * size_t(M + 1)},
                        {(void**)&bad, 8}})
        if (e == cudaSuccess) e = scratch_alloc(p, b, dev, s);
    if (e == cudaSuccess) e = cudaMalloc(&rp, 4 * size_t(M + 1));
    if (e != cudaSuccess) {
        release(true);
        return cuda_fail(e, "from_coo: cudaMalloc");
    }
    const unsigned blocks = unsigned(std::min<int64_t>((std::max<int64_t>(n, 1) + 255) / 256, 148 * 16));
    e = cudaMemsetAsync(bad, 0xff, 8, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, 4 * size_t(M + 1), s);
    int64_t n_out = 0;
    if (e == cudaSuccess && n > 0) {
        k_coo_keys<<<blocks, 256, 0, s>>>(d_rows, d_cols, n, M, K, keys, idx, bad);
        unsigned long long hb = ~0ull;
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e == cudaSuccess && hb != ~0ull) {
            release(true);
            return fail(DASPMM_ERR_INVALID_ARG, "from_coo: coordinate out of bounds");
        }
        // Radix sort on the bits the keys use: low 32 (column) + enough for the rows.
        const int end_bit = 32 + bits_for(M);
        size_t tmp_bytes = 0, scan_bytes = 0;
        if (e == cudaSuccess)
            e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys_s, idx, perm, int(n),
                                                0, end_bit, s);
        if (e == cudaSuccess)
            e = cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, head, slot, int(n), s);
        size_t scan2 = 0;
        if (e == cudaSuccess)
            e = cub::DeviceScan::ExclusiveSum(nullptr, scan2, cnt, rp, int(M + 1), s);
        tmp_bytes = std::max({tmp_bytes, scan_bytes, scan2});
        if (e == cudaSuccess) e = scratch_alloc(&tmp, std::max<size_t>(tmp_bytes, 16), dev, s);
        if (e == cudaSuccess)
            e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys_s, idx, perm, int(n), 0,
                                                end_bit, s);
        if (e == cudaSuccess) {
            k_coo_heads<<<blocks, 256, 0, s>>>(keys_s, n, head);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, head, slot, int(n), s);
        int last[2] = {0, 0};
        if (e == cudaSuccess) e = cudaMemcpyAsync(&last[0], slot + n - 1, 4, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&last[1], head + n - 1, 4, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        n_out = int64_t(last[0]) + last[1];
        if (e == cudaSuccess) e = cudaMalloc(&ci, 4 * size_t(std::max<int64_t>(n_out, 1)));
        if (e == cudaSuccess) e = cudaMalloc(&va, es * size_t(std::max<int64_t>(n_out, 1)));
        if (e == cudaSuccess) {
            if (dtype == DASPMM_F64)
                k_coo_merge<double><<<blocks, 256, 0, s>>>(keys_s, perm, head, slot, n,
                                                           static_cast<const double*>(d_vals), ci,
                                                           static_cast<double*>(va), cnt);
            else
                k_coo_merge<float><<<blocks, 256, 0, s>>>(keys_s, perm, head, slot, n,
                                                          static_cast<const float*>(d_vals), ci,
                                                          static_cast<float*>(va), cnt);
            e = cudaGetLastError();
        }
        // row offsets: exclusive scan of the M + 1 counts (the last count is 0) -> rp[M] = nnz
        if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, rp, int(M + 1), s);
    } else if (e == cudaSuccess) {
        e = cudaMemsetAsync(rp, 0, 4 * size_t(M + 1), s);
        if (e == cudaSuccess) e = cudaMalloc(&ci, 4);
        if (e == cudaSuccess) e = cudaMalloc(&va, es);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        release(true);
        return cuda_fail(e, "from_coo");
    }
    release(false);
    int rc = daspmm_csr_create_device(M, K, n_out, rp, ci, va, dtype, 0, stream, out);
    if (rc) {
        cudaFree(rp), cudaFree(ci), cudaFree(va);
        return rc;
    }
    (*out)->owns = true;  // the handle frees the arrays built here
    return DASPMM_OK;
}
