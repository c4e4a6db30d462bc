// Mini SpMM probe (round 2): uniform rows of exactly 16 nonzeros, K = M = 2^20, N = 32
// (B = 128 MB, ~ the L2) — the uniform s20 N = 32 suite call with everything but the
// gather loop stripped. Sweeps the knobs that decide whether B stays in L2 while A and C
// stream through it, and how many gathers each lane keeps in flight:
//   AH: A (col, val) loads   0 ld.global.nc  1 ld.global.cs  2 L2 evict_first policy
//                            3 L1::no_allocate + L2 evict_first policy
//   CH: C stores             0 st.global     1 st.global.cs  2 L2 evict_first policy
//   BH: B gathers            0 ld.global.nc  1 L2 evict_last policy
//   U : gathers in flight per lane (4, 8, 16)
// Each variant is timed cold (L2 flushed by a 256 MB write + a 256 MB read) and warm.
//
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bin/minispmm tools/experiments/minispmm.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

constexpr int kDeg = 16;

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

__global__ void k_init(int* ci, float* va, float* B, int64_t nnz, int64_t nb, uint32_t K) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nnz;
         i += int64_t(gridDim.x) * blockDim.x) {
        ci[i] = int(mix(uint32_t(i) * 2654435761u + 7) % K);
        va[i] = float(mix(uint32_t(i) + 3) & 1023) / 1024.f;
    }
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nb;
         i += int64_t(gridDim.x) * blockDim.x)
        B[i] = float(mix(uint32_t(i) + 11) & 255) / 256.f;
}

__device__ __forceinline__ uint64_t pol_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t pol_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

template <int AH>
__device__ __forceinline__ int lda_i(const int* p, uint64_t pol) {
    int v;
    if constexpr (AH == 4) v = int(mix(uint32_t(reinterpret_cast<uintptr_t>(p) >> 2) * 2654435761u + 7) & ((1u << 20) - 1));
    else if constexpr (AH == 0 || AH == 5) v = AH == 5 ? __ldcs(p) : __ldg(p);
    else if constexpr (AH == 1) v = __ldcs(p);
    else if constexpr (AH == 2)
        asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    else
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
                     : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
template <int AH>
__device__ __forceinline__ float lda_f(const float* p, uint64_t pol) {
    float v;
    if constexpr (AH == 4) v = 0.5f;
    else if constexpr (AH == 0 || AH == 5) v = AH == 5 ? __ldcs(p) : __ldg(p);
    else if constexpr (AH == 1) v = __ldcs(p);
    else if constexpr (AH == 2)
        asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(p), "l"(pol));
    else
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
                     : "=f"(v) : "l"(p), "l"(pol));
    return v;
}
template <int BH>
__device__ __forceinline__ float4 ldb4(const float* p, uint64_t pol) {
    float4 v;
    if constexpr (BH == 0) v = __ldg(reinterpret_cast<const float4*>(p));
    else
        asm volatile("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p), "l"(pol));
    return v;
}
template <int CH>
__device__ __forceinline__ void stc4(float* p, float4 v, uint64_t pol) {
    if constexpr (CH == 3) { if (v.x == -12345.f) *reinterpret_cast<float4*>(p) = v; }
    else if constexpr (CH == 0) *reinterpret_cast<float4*>(p) = v;
    else if constexpr (CH == 1) __stcs(reinterpret_cast<float4*>(p), v);
    else
        asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;"
                     :: "l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol) : "memory");
}

// Group of L = N/4 lanes per row, RB rows per group, U gathers in flight per lane.
template <int L, int U, int AH, int BH, int CH>
__global__ void __launch_bounds__(256) k_mini(const int* __restrict__ ci,
                                              const float* __restrict__ va,
                                              const float* __restrict__ B, float* C, int M,
                                              int RB) {
    constexpr int N = 4 * L;
    const uint64_t pa = pol_first(), pb = pol_last();
    const int gl = threadIdx.x % L;
    const unsigned mask = L == 32 ? 0xffffffffu : ((1u << L) - 1u) << ((threadIdx.x & 31) & ~(L - 1));
    const int64_t g = (int64_t(blockIdx.x) * 256 + threadIdx.x) / L;
    const int r0 = int(g * RB);
    if (r0 >= M) return;
    const int r1 = min(M, r0 + RB);
    const float* Bc = B + gl * 4;
    for (int r = r0; r < r1; ++r) {
        const int64_t e0 = int64_t(r) * kDeg;
        // the row's 16 (col, val) pairs: kDeg / L per lane, broadcast by shuffle
        constexpr int PPL = kDeg / L > 0 ? kDeg / L : 1;
        int c[PPL];
        float v[PPL];
#pragma unroll
        for (int q = 0; q < PPL; ++q) {
            const int e = q * L + gl;
            c[q] = e < kDeg ? lda_i<AH>(ci + e0 + e, pa) : 0;
            v[q] = e < kDeg ? lda_f<AH>(va + e0 + e, pa) : 0.f;
        }
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int x0 = 0; x0 < kDeg; x0 += U) {
            float4 b[U];
            float w[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int x = x0 + u;
                const int col = __shfl_sync(mask, c[x / L], x % L, L);
                w[u] = __shfl_sync(mask, v[x / L], x % L, L);
                b[u] = ldb4<BH>(Bc + int64_t(col) * N, pb);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                acc.x = fmaf(w[u], b[u].x, acc.x);
                acc.y = fmaf(w[u], b[u].y, acc.y);
                acc.z = fmaf(w[u], b[u].z, acc.z);
                acc.w = fmaf(w[u], b[u].w, acc.w);
            }
        }
        stc4<CH>(C + int64_t(r) * N + gl * 4, acc, pb);
    }
    if constexpr (AH == 5) {
        const int64_t b0 = (int64_t(r0) * kDeg * 4 + 127) / 128, b1 = int64_t(r1) * kDeg * 4 / 128;
        for (int64_t l = b0 + gl; l < b1; l += L) {
            asm volatile("discard.global.L2 [%0], 128;" :: "l"(reinterpret_cast<const char*>(ci) + l * 128) : "memory");
            asm volatile("discard.global.L2 [%0], 128;" :: "l"(reinterpret_cast<const char*>(va) + l * 128) : "memory");
        }
    }
}

__global__ void k_flush(float* f, int64_t n, float* sink) {
    float s = 0.f;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        f[i] = float(i & 7);
    }
    __syncthreads();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        s += __ldcg(f + (n - 1 - i));
    if (s == 12345.f) sink[0] = s;
}

struct Bufs {
    int* ci;
    float *va, *B, *C, *fl, *sink;
    int M;
};

template <int L, int U, int AH, int BH, int CH>
static int run(const Bufs& b, int RB, const char* tag) {
    const int64_t groups = (b.M + RB - 1) / RB;
    const int blocks = int((groups * L + 255) / 256);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float cold = 1e30f, warm = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        k_flush<<<148 * 8, 256>>>(b.fl, int64_t(64) << 20, b.sink);
        cudaEventRecord(e0);
        k_mini<L, U, AH, BH, CH><<<blocks, 256>>>(b.ci, b.va, b.B, b.C, b.M, RB);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < cold) cold = ms;
        cudaEventRecord(e0);
        k_mini<L, U, AH, BH, CH><<<blocks, 256>>>(b.ci, b.va, b.B, b.C, b.M, RB);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep > 0 && ms < warm) warm = ms;
    }
    CK(cudaGetLastError());
    const double gather = double(b.M) * kDeg * 4 * 4 * L;
    printf("N=%3d U=%2d AH=%d BH=%d CH=%d RB=%d %-10s cold %7.1f us (%5.1f TB/s gather)  warm %7.1f us "
           "(%5.1f TB/s)\n", 4 * L, U, AH, BH, CH, RB, tag, cold * 1e3, gather / (cold * 1e-3) / 1e12,
           warm * 1e3, gather / (warm * 1e-3) / 1e12);
    fflush(stdout);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return 0;
}

int main() {
    Bufs b;
    b.M = 1 << 20;
    const uint32_t K = 1u << 20;
    const int64_t nnz = int64_t(b.M) * kDeg;
    CK(cudaMalloc(&b.ci, nnz * 4));
    CK(cudaMalloc(&b.va, nnz * 4));
    CK(cudaMalloc(&b.B, int64_t(K) * 128 * 4));
    CK(cudaMalloc(&b.C, int64_t(b.M) * 128 * 4));
    CK(cudaMalloc(&b.fl, int64_t(64) << 22));
    CK(cudaMalloc(&b.sink, 4));
    k_init<<<148 * 8, 256>>>(b.ci, b.va, b.B, nnz, int64_t(K) * 128, K);
    CK(cudaDeviceSynchronize());
    run<8, 8, 1, 0, 1>(b, 8, "cs");
    run<8, 8, 4, 0, 3>(b, 8, "noA,noC");
    run<8, 8, 1, 0, 3>(b, 8, "A,noC");
    run<8, 8, 4, 0, 1>(b, 8, "noA,C");
    run<8, 8, 5, 0, 1>(b, 8, "A+disc,C");
    run<8, 8, 5, 0, 3>(b, 8, "A+disc,noC");
    run<8, 8, 5, 0, 2>(b, 8, "A+disc,Cef");
    run<8, 8, 5, 1, 2>(b, 8, "A+disc,Cef,Bl");
    run<4, 8, 1, 0, 1>(b, 8, "cs");
    run<4, 8, 4, 0, 3>(b, 8, "noA,noC");
    run<4, 8, 5, 0, 1>(b, 8, "A+disc,C");
    run<16, 8, 1, 0, 1>(b, 8, "cs");
    run<16, 8, 4, 0, 3>(b, 8, "noA,noC");
    run<16, 8, 5, 0, 1>(b, 8, "A+disc,C");
    return 0;
}
