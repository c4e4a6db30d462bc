// Does the B200's L2 behave as two per-die caches that each hold what their own SMs read
// (so a footprint read by every SM is cached twice, ~63 MB effective), and if so which SM
// ids sit on which die? Random 64-B gathers from F MB; four ways to assign the footprint:
//   all     every CTA gathers from the whole footprint
//   lo74    SMs with %smid < 74 gather from the first half, the others from the second
//   odd     SMs with even %smid gather from the first half, odd from the second
//   cta     CTAs with even blockIdx.x first half (die-agnostic control: same as `all`
//           if locality is what matters)
//   gpc     SMs split by (%smid / 2) parity — TPC pairs alternating (a third candidate)
// If one mapping matches the die boundary, its throughput at F = 96..256 MB should be that
// of half the footprint under `all`. Also prints each SM's %nsmid-independent id list of
// the first CTAs for reference.
//
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gpurun_out/die_split tools/experiments/die_split.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

template <int MODE>
__global__ void __launch_bounds__(256) k_gather(const char* __restrict__ buf, uint32_t nseg,
                                                int iters, float* out, unsigned nsm) {
    constexpr int LPS = 4;  // 64-B segment, float4 per lane
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t grp = tid / LPS, gl = tid % LPS;
    const unsigned sm = smid();
    uint32_t half = 0;
    bool split = true;
    if (MODE == 0) split = false;
    else if (MODE == 1) half = sm < nsm / 2 ? 0 : 1;
    else if (MODE == 2) half = sm & 1;
    else if (MODE == 3) half = blockIdx.x & 1;
    else half = (sm >> 1) & 1;
    const uint32_t n = split ? nseg / 2 : nseg;
    const char* base = buf + (split ? size_t(half) * (size_t(nseg / 2) * 64) : 0);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t s = mix(grp * 0x9e3779b9U + 1);
    for (int it = 0; it < iters; it += 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            s = mix(s + u + 1);
            v[u] = __ldg(reinterpret_cast<const float4*>(base + size_t(s % n) * 64) + gl);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
        }
    }
    out[tid] = acc.x + acc.y + acc.z + acc.w;
}

template <int MODE>
static double run(const char* buf, uint32_t nseg, float* out, int sms) {
    const int blocks = sms * 8, threads = 256, iters = 512;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_gather<MODE><<<blocks, threads>>>(buf, nseg, iters, out, sms);
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        k_gather<MODE><<<blocks, threads>>>(buf, nseg, iters, out, sms);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return double(blocks) * threads * iters * 16.0 / (best * 1e-3) / 1e9;
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
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"seg\": 64, \"gbs\": [\n", p.name, sms,
           p.l2CacheSize);
    bool first = true;
    for (int mb : {32, 48, 64, 80, 96, 112, 128, 160, 192, 256, 512}) {
        const uint32_t nseg = uint32_t((size_t(mb) << 20) / 64);
        printf("%s  {\"footprint_mb\": %d, \"all\": %.0f, \"lo74\": %.0f, \"odd\": %.0f, "
               "\"cta\": %.0f, \"tpc\": %.0f}",
               first ? "" : ",\n", mb, run<0>(buf, nseg, out, sms), run<1>(buf, nseg, out, sms),
               run<2>(buf, nseg, out, sms), run<3>(buf, nseg, out, sms),
               run<4>(buf, nseg, out, sms));
        fflush(stdout);
        first = false;
    }
    printf("\n]}\n");
    return 0;
}
