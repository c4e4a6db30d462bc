// daspmm — multi-GPU layer of the C ABI: one process per GPU, each rank
// computes an exchange-free share of C = A·B with DA-SpMM, and C is assembled over NCCL
// (NVLink / NVSwitch) only when the caller asks for the full matrix.
//
//   rows  A cut into nnz-balanced row panels (partition_elements' chunk starts, snapped to
//         row starts — partition.hpp:27-30, 45-64), B replicated. Rows of C depend only
//         on rows of A (spmm.hpp:23-30): no cross-GPU atomics. Each rank's panel handle is
//         built once and cached on the full handle; the device selector runs on the
//         panel's own features.
//   cols  N split into P column slices, A replicated. Columns of C depend only on the
//         same columns of B, so a slice is B + c0 / C + c0 with the full leading
//         dimensions — no packing on the compute path.
//   auto  per-GPU compulsory bytes, rows: A/P + B + C/P, cols: A + B/P + C/P (§8e).
//
// Assembly: rows — one ncclBroadcast per rank of its contiguous panel, in one NCCL group
// (panels are unequal, so not an all-gather); cols — the rank's slice packed to M x wmax,
// one ncclAllGather, then the peers' slices unpacked into C's columns.
//
// NCCL is loaded at run time (dlopen libnccl.so.2: the instance torch already loaded, or
// the system one), so the library has no link-time NCCL dependency; without it the comm
// entry points return DASPMM_ERR_NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "dispatch.h"
#include "internal.h"

struct daspmm_comm {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0, device = 0;
};

namespace daspmm {

namespace {

struct Nccl {
    bool ok = false;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl n = [] {
        Nccl r;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return r;
        auto sym = [&](const char* name) { return dlsym(h, name); };
        r.get_unique_id = reinterpret_cast<decltype(r.get_unique_id)>(sym("ncclGetUniqueId"));
        r.comm_init_rank = reinterpret_cast<decltype(r.comm_init_rank)>(sym("ncclCommInitRank"));
        r.comm_destroy = reinterpret_cast<decltype(r.comm_destroy)>(sym("ncclCommDestroy"));
        r.broadcast = reinterpret_cast<decltype(r.broadcast)>(sym("ncclBroadcast"));
        r.all_gather = reinterpret_cast<decltype(r.all_gather)>(sym("ncclAllGather"));
        r.group_start = reinterpret_cast<decltype(r.group_start)>(sym("ncclGroupStart"));
        r.group_end = reinterpret_cast<decltype(r.group_end)>(sym("ncclGroupEnd"));
        r.error_string = reinterpret_cast<decltype(r.error_string)>(sym("ncclGetErrorString"));
        r.ok = r.get_unique_id && r.comm_init_rank && r.comm_destroy && r.broadcast &&
               r.all_gather && r.group_start && r.group_end;
        return r;
    }();
    return n;
}

int nccl_fail(ncclResult_t rc, const char* what) {
    const char* s = nccl().error_string ? nccl().error_string(rc) : "error";
    return fail(DASPMM_ERR_NCCL, std::string(what) + ": " + s);
}

int elem(int dtype) { return dtype == DASPMM_F64 ? 8 : 4; }

// C columns [c0, c0 + w) of every row <-> a packed M x wmax block.
template <typename T>
__global__ void k_pack_cols(const T* __restrict__ C, int64_t ldc, int64_t M, int64_t c0, int64_t w,
                            int64_t wmax, T* __restrict__ out, int unpack) {
    const int64_t n = M * wmax;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = i / wmax, j = i - r * wmax;
        if (j >= w) continue;
        if (unpack) const_cast<T*>(C)[r * ldc + c0 + j] = out[i];
        else out[i] = C[r * ldc + c0 + j];
    }
}

cudaError_t pack_cols(int dtype, const void* C, int64_t ldc, int64_t M, int64_t c0, int64_t w,
                      int64_t wmax, void* out, bool unpack, cudaStream_t s) {
    const int64_t n = M * wmax;
    if (n == 0) return cudaSuccess;
    const unsigned blocks = unsigned(std::min<int64_t>((n + 255) / 256, 148 * 16));
    if (dtype == DASPMM_F64)
        k_pack_cols<double><<<blocks, 256, 0, s>>>(static_cast<const double*>(C), ldc, M, c0, w,
                                                   wmax, static_cast<double*>(out), unpack);
    else
        k_pack_cols<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(C), ldc, M, c0, w, wmax,
                                                  static_cast<float*>(out), unpack);
    return cudaGetLastError();
}

}  // namespace

// Row cuts of `parts` nnz-balanced panels: cut[p] = row holding partition_elements'
// chunk p start (M for empty tail chunks), made nondecreasing; cut[0] = 0, cut[P] = M.
int multi_row_cuts(const daspmm_csr* h, int parts, int64_t* cuts) {
    std::vector<int64_t> rows(static_cast<size_t>(parts));
    if (int rc = daspmm_partition(h, parts, nullptr, nullptr, rows.data())) return rc;
    cuts[0] = 0;
    for (int p = 1; p < parts; ++p) cuts[p] = std::max<int64_t>(cuts[p - 1], std::min(rows[p], h->M));
    cuts[parts] = h->M;
    return DASPMM_OK;
}

}  // namespace daspmm

using namespace daspmm;

extern "C" {

int daspmm_comm_unique_id(void* id_out) {
    if (!id_out) return fail(DASPMM_ERR_INVALID_ARG, "comm_unique_id: null output");
    if (!nccl().ok) return fail(DASPMM_ERR_NCCL, "comm: libnccl.so.2 not loadable");
    ncclUniqueId id;
    if (ncclResult_t rc = nccl().get_unique_id(&id)) return nccl_fail(rc, "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof id);
    return DASPMM_OK;
}

int daspmm_comm_create(int nranks, int rank, const void* unique_id, daspmm_comm** out) {
    if (!out || !unique_id) return fail(DASPMM_ERR_INVALID_ARG, "comm_create: null argument");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return fail(DASPMM_ERR_INVALID_ARG, "comm_create: rank outside [0, nranks)");
    if (!nccl().ok) return fail(DASPMM_ERR_NCCL, "comm: libnccl.so.2 not loadable");
    auto* c = new daspmm_comm;
    c->nranks = nranks;
    c->rank = rank;
    cudaGetDevice(&c->device);
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof id);
    if (ncclResult_t rc = nccl().comm_init_rank(&c->comm, nranks, id, rank)) {
        delete c;
        return nccl_fail(rc, "ncclCommInitRank");
    }
    *out = c;
    return DASPMM_OK;
}

int daspmm_comm_destroy(daspmm_comm* c) {
    if (!c) return DASPMM_OK;
    if (c->comm && nccl().ok) nccl().comm_destroy(c->comm);
    delete c;
    return DASPMM_OK;
}

int daspmm_multi_plan(const daspmm_csr* h, int parts, int64_t N, int mode, int* mode_out,
                      int64_t* bounds) {
    if (!h || !mode_out || !bounds) return fail(DASPMM_ERR_INVALID_ARG, "multi_plan: null argument");
    if (parts < 1) return fail(DASPMM_ERR_INVALID_ARG, "multi_plan: need parts >= 1");
    if (mode < -1 || mode > 1) return fail(DASPMM_ERR_INVALID_ARG, "multi_plan: mode must be -1, 0 or 1");
    if (N < 0) return fail(DASPMM_ERR_DIMS, "multi_plan: negative N");
    if (mode < 0) {
        // per-GPU compulsory bytes of each partitioning
        const double es = elem(h->dtype);
        const double a = 4.0 * double(h->M + 1) + (4.0 + es) * double(h->nnz);
        const double b = es * double(h->K) * double(N), c = es * double(h->M) * double(N);
        const double rows = a / parts + b + c / parts, cols = a + b / parts + c / parts;
        mode = (rows <= cols || N < parts) ? DASPMM_SPLIT_ROWS : DASPMM_SPLIT_COLS;
    }
    *mode_out = mode;
    if (mode == DASPMM_SPLIT_COLS) {
        for (int p = 0; p <= parts; ++p) bounds[p] = (N * p) / parts;
        return DASPMM_OK;
    }
    return multi_row_cuts(h, parts, bounds);
}

int daspmm_multi_spmm(daspmm_comm* comm, const daspmm_csr* h, const daspmm_model* model,
                      int64_t hw, const void* d_B, int64_t ldb, int64_t N, void* d_C, int64_t ldc,
                      int mode, int assemble, int* d_kernel, daspmm_stream stream) {
    if (!h || !model) return fail(DASPMM_ERR_INVALID_ARG, "multi_spmm: null argument");
    const int parts = comm ? comm->nranks : 1, rank = comm ? comm->rank : 0;
    if (int rc = check_call(h, 0, 0, 8, 1, DASPMM_ROW_MAJOR, ldb, N, ldc, false)) return rc;
    if (h->M == 0 || N == 0) return DASPMM_OK;
    if (comm && comm->device != h->device)
        return fail(DASPMM_ERR_INVALID_ARG, "multi_spmm: communicator and matrix on different devices");
    DeviceGuard g(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    std::vector<int64_t> bounds(size_t(parts) + 1);
    int md = 0;
    if (int rc = daspmm_multi_plan(h, parts, N, mode, &md, bounds.data())) return rc;
    const size_t es = size_t(elem(h->dtype));
    const int64_t lo = bounds[size_t(rank)], hi = bounds[size_t(rank) + 1];
    // ---- the rank's exchange-free share, through DA-SpMM
    if (md == DASPMM_SPLIT_COLS) {
        if (hi > lo)
            if (int rc = daspmm_spmm_selected(h, model, hw, static_cast<const char*>(d_B) + es * lo,
                                              DASPMM_ROW_MAJOR, ldb, hi - lo,
                                              static_cast<char*>(d_C) + es * lo, ldc, 0, 0,
                                              d_kernel, stream))
                return rc;
    } else if (hi > lo) {
        const daspmm_csr* panel = h;
        if (parts > 1) {
            daspmm_csr* hm = const_cast<daspmm_csr*>(h);
            std::lock_guard<std::mutex> lk(hm->mu);
            for (auto& e : hm->panels)
                if (e.parts == parts && e.rank == rank) panel = e.h;
            if (panel == h) {
                daspmm_csr* p = nullptr;
                // panels are built on the legacy stream, then cached with the full handle
                if (int rc = daspmm_csr_create_panel(h, lo, hi, nullptr, &p)) return rc;
                hm->panels.push_back({parts, rank, p});
                panel = p;
            }
        }
        if (int rc = daspmm_spmm_selected(panel, model, hw, d_B, DASPMM_ROW_MAJOR, ldb, N,
                                          static_cast<char*>(d_C) + es * lo * ldc, ldc, 0, 0,
                                          d_kernel, stream))
            return rc;
    }
    if (!assemble || comm == nullptr) return DASPMM_OK;  // one rank with a comm: the NCCL path still runs
    // ---- assembly over NCCL
    const ncclDataType_t dt = h->dtype == DASPMM_F64 ? ncclDouble : ncclFloat;
    ncclResult_t nr;
    if (md != DASPMM_SPLIT_COLS) {
        if (ldc != N)
            return fail(DASPMM_ERR_UNSUPPORTED, "multi_spmm: row assembly needs ldc == N");
        if ((nr = nccl().group_start())) return nccl_fail(nr, "ncclGroupStart");
        for (int p = 0; p < parts; ++p) {
            const int64_t r0 = bounds[size_t(p)], r1 = bounds[size_t(p) + 1];
            if (r1 <= r0) continue;
            void* buf = static_cast<char*>(d_C) + es * size_t(r0) * size_t(ldc);
            if ((nr = nccl().broadcast(buf, buf, size_t(r1 - r0) * size_t(N), dt, p, comm->comm, s))) {
                nccl().group_end();
                return nccl_fail(nr, "ncclBroadcast");
            }
        }
        if ((nr = nccl().group_end())) return nccl_fail(nr, "ncclGroupEnd");
        return DASPMM_OK;
    }
    int64_t wmax = 0;
    for (int p = 0; p < parts; ++p) wmax = std::max(wmax, bounds[size_t(p) + 1] - bounds[size_t(p)]);
    const size_t slab = size_t(h->M) * size_t(wmax);
    void* stage = nullptr;
    cudaError_t e = scratch_alloc(&stage, std::max<size_t>(es * slab * size_t(parts), 16), h->device, s);
    if (e != cudaSuccess) return cuda_fail(e, "multi_spmm: staging");
    char* st = static_cast<char*>(stage);
    e = pack_cols(h->dtype, d_C, ldc, h->M, lo, hi - lo, wmax, st + es * slab * size_t(rank), false, s);
    int rc = DASPMM_OK;
    if (e != cudaSuccess) rc = cuda_fail(e, "multi_spmm: pack");
    if (rc == DASPMM_OK &&
        (nr = nccl().all_gather(st + es * slab * size_t(rank), st, slab, dt, comm->comm, s)))
        rc = nccl_fail(nr, "ncclAllGather");
    for (int p = 0; rc == DASPMM_OK && p < parts; ++p) {
        if (p == rank) continue;
        const int64_t c0 = bounds[size_t(p)], w = bounds[size_t(p) + 1] - c0;
        if ((e = pack_cols(h->dtype, d_C, ldc, h->M, c0, w, wmax, st + es * slab * size_t(p), true,
                           s)) != cudaSuccess)
            rc = cuda_fail(e, "multi_spmm: unpack");
    }
    scratch_free(stage, s);
    return rc;
}

}  // extern "C"
