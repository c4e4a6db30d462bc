// Launcher of the TMA-gather EB+RM+SR kernel (tma_gather.cuh): builds the tensor map
// of B (driver entry point, no libcuda link dependency) and picks box width and ring
// depth from N.
#include <cudaTypedefs.h>

#include <mutex>

#include "dispatch.h"
#include "tma_gather.cuh"

namespace daspmm {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// Box width (columns per TMA row fetch) for a call: 32, 64 or 128 fp32 columns.
int tma_box_cols(int64_t N) { return N >= 128 ? 128 : (N > 32 ? 64 : 32); }

bool tma_gather_supported(const void* B, int64_t ldb, int64_t N, int64_t K) {
    return encode_fn() != nullptr && N >= 32 && (reinterpret_cast<uintptr_t>(B) & 15) == 0 &&
           (ldb * 4) % 16 == 0 && ldb < (int64_t(1) << 32) && K < (int64_t(1) << 31);
}

template <int BC, int D>
static cudaError_t launch(const CUtensorMap& map, const Plan& p, const SpmmArgs<float>& a,
                          int Lw, cudaStream_t s) {
    constexpr size_t smem = size_t(kTmaWarps) * D * kTmaStageNnz * BC * sizeof(float);
    static std::once_flag once[64];
    int dev = 0;
    cudaGetDevice(&dev);
    cudaError_t e = cudaSuccess;
    std::call_once(once[dev & 63], [&] {
        e = cudaFuncSetAttribute(k_eb_sr_tma<BC, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem));
    });
    if (e != cudaSuccess) return e;
    k_eb_sr_tma<BC, D><<<p.grid, kTmaWarps * 32, smem, s>>>(map, a, Lw);
    return cudaGetLastError();
}

cudaError_t launch_eb_sr_tma(const Plan& p, const SpmmArgs<float>& a, cudaStream_t s) {
    auto fn = encode_fn();
    if (!fn) return cudaErrorNotSupported;
    const int bc = tma_box_cols(a.N);
    CUtensorMap map;
    const cuuint64_t dims[2] = {cuuint64_t(a.N), cuuint64_t(a.K)};
    const cuuint64_t strides[1] = {cuuint64_t(a.ldb) * sizeof(float)};
    const cuuint32_t box[2] = {cuuint32_t(bc), 1};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a.B), dims,
                    strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
    const int Lw = int(p.sub);
    switch (bc) {
        case 128: return launch<128, 3>(map, p, a, Lw, s);
        case 64: return launch<64, 4>(map, p, a, Lw, s);
        default: return launch<32, 6>(map, p, a, Lw, s);
    }
}

}  // namespace daspmm
