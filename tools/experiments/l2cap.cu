// Effective L2 capacity for random row gathers issued from every SM (round-2 probe for
// the N-sliced SpMM question: how wide may a column slice of B be and still stay in L2?).
//
// (1) footprint sweep: groups of SEG/16 lanes gather SEG-byte segments at random
//     positions of a buffer of F MB (packed, every byte of every touched line is used);
// (2) strided slices: B is K x 128 fp32 row-major (512 MB at K = 2^20) and a pass gathers
//     only columns [s*W, s*W + W) of random rows — the L2 holds W*4 useful bytes of each
//     128-B line (W < 32) — versus the same slice packed as K x W.
// Throughput is printed per case; an L2-resident footprint runs at the L2 gather rate
// (~15 TB/s for >= 64-B segments), a DRAM-bound one at the random-gather DRAM rate.
//
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gpurun_out/l2cap tools/experiments/l2cap.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

// Gather SEG bytes per group from row `r` (random in [0, nrows)) at byte offset
// r * pitch + off. LPS = SEG/16 lanes per group, float4 per lane.
template <int SEG, int UNROLL>
__global__ void __launch_bounds__(256) k_gather(const char* __restrict__ buf, uint32_t nrows,
                                                uint32_t pitch, uint32_t off, int iters,
                                                float* out) {
    constexpr int LPS = SEG / 16;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t grp = tid / LPS, gl = tid % LPS;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t s = mix(grp * 0x9e3779b9U + 1);
    for (int it = 0; it < iters; it += UNROLL) {
        float4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            s = mix(s + u + 1);
            const uint32_t r = s % nrows;
            v[u] = __ldg(reinterpret_cast<const float4*>(buf + size_t(r) * pitch + off) + gl);
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
        }
    }
    out[tid] = acc.x + acc.y + acc.z + acc.w;
}

template <int SEG>
static double run(const char* buf, uint32_t nrows, uint32_t pitch, uint32_t off, float* out,
                  int sms) {
    const int blocks = sms * 8, threads = 256, iters = 256;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_gather<SEG, 8><<<blocks, threads>>>(buf, nrows, pitch, off, iters, out);  // L2 fill
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        k_gather<SEG, 8><<<blocks, threads>>>(buf, nrows, pitch, off, iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    const double bytes = double(blocks) * threads * iters * 16.0;
    return bytes / (best * 1e-3) / 1e9;
}

int main() {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    const size_t big = size_t(1) << 30;
    char* buf;
    float* out;
    CK(cudaMalloc(&buf, big));
    CK(cudaMemset(buf, 0, big));
    CK(cudaMalloc(&out, size_t(p.multiProcessorCount) * 8 * 256 * 4));
    const int sms = p.multiProcessorCount;
    printf("{\"gpu\": \"%s\", \"l2_bytes\": %d,\n \"packed_sweep\": [\n", p.name, p.l2CacheSize);
    bool first = true;
    for (int mb = 16; mb <= 160; mb += 8) {
        const size_t F = size_t(mb) << 20;
        const double g64 = run<64>(buf, uint32_t(F / 64), 64, 0, out, sms);
        const double g128 = run<128>(buf, uint32_t(F / 128), 128, 0, out, sms);
        printf("%s  {\"footprint_mb\": %d, \"gbs_seg64\": %.0f, \"gbs_seg128\": %.0f}",
               first ? "" : ",\n", mb, g64, g128);
        first = false;
    }
    printf("\n ],\n \"slices_K2p20\": [\n");
    // B = 2^20 x 128 fp32 (512 MB): slice widths 8/16/32/64 columns, strided vs packed.
    const uint32_t K = 1u << 20;
    first = true;
    for (int w : {8, 16, 32, 64}) {
        const uint32_t seg = uint32_t(w) * 4;
        double strided, packed;
        if (w == 8) {
            strided = run<32>(buf, K, 512, 0, out, sms);
            packed = run<32>(buf, K, seg, 0, out, sms);
        } else if (w == 16) {
            strided = run<64>(buf, K, 512, 0, out, sms);
            packed = run<64>(buf, K, seg, 0, out, sms);
        } else if (w == 32) {
            strided = run<128>(buf, K, 512, 0, out, sms);
            packed = run<128>(buf, K, seg, 0, out, sms);
        } else {
            strided = run<256>(buf, K, 512, 0, out, sms);
            packed = run<256>(buf, K, seg, 0, out, sms);
        }
        printf("%s  {\"slice_cols\": %d, \"useful_mb\": %u, \"gbs_strided\": %.0f, "
               "\"gbs_packed\": %.0f}",
               first ? "" : ",\n", w, unsigned((size_t(K) * seg) >> 20), strided, packed);
        first = false;
    }
    printf("\n ]}\n");
    return 0;
}
