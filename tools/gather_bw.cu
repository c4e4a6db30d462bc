// Gather-bandwidth microbenchmark: the ceilings a CSR SpMM's dense-B row gathers run
// against on this GPU (SURVEY.md §8d asks for the L2 -> SM gather bandwidth as a third
// roofline beside HBM and FP32 issue).
//
// Each group of SEG/16 lanes reads one SEG-byte segment (float4 per lane) from a
// pseudo-random segment of a buffer of `footprint` bytes and accumulates it; the sum is
// written once per thread so nothing is dead. Footprints well below the 126 MB L2 give the
// L2 -> SM gather ceiling, footprints far above it the DRAM random-gather ceiling.
// Also: a streaming read (the sequential-HBM figure the random ones are compared with).
//
// build:  nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gpurun_out/gather_bw tools/gather_bw.cu
// run:    gpurun_out/gather_bw > gpurun_out/gather_bw.json
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int SEG, int UNROLL>
__global__ void __launch_bounds__(256) k_gather(const float4* __restrict__ buf, uint32_t nseg,
                                                int iters, float* out) {
    constexpr int LPS = SEG / 16;  // lanes per segment
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t grp = tid / LPS, gl = tid % LPS;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t s = mix(grp * 0x9e3779b9U + 1);
    for (int it = 0; it < iters; it += UNROLL) {
        float4 v[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            s = mix(s + u + 1);
            const uint32_t seg = s % nseg;
            v[u] = __ldg(buf + size_t(seg) * LPS + gl);
        }
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
        }
    }
    out[tid] = acc.x + acc.y + acc.z + acc.w;
}

__global__ void k_stream(const float4* __restrict__ buf, size_t n, float* out) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        float4 v = __ldg(buf + i);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

template <int SEG>
static int run(const float4* buf, size_t footprint, float* out, int sms, bool& first) {
    const uint32_t nseg = uint32_t(footprint / SEG);
    const int blocks = sms * 8, threads = 256, iters = 256;
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    k_gather<SEG, 8><<<blocks, threads>>>(buf, nseg, iters, out);  // warm (L2 fill)
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(a));
        k_gather<SEG, 8><<<blocks, threads>>>(buf, nseg, iters, out);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms; CK(cudaEventElapsedTime(&ms, a, b));
        if (ms < best) best = ms;
    }
    const double bytes = double(blocks) * threads * iters * 16.0;
    printf("%s  {\"seg_bytes\": %d, \"footprint_mb\": %.0f, \"gbs\": %.1f}", first ? "" : ",\n",
           SEG, footprint / 1e6, bytes / (best * 1e-3) / 1e9);
    first = false;
    CK(cudaEventDestroy(a)); CK(cudaEventDestroy(b));
    return 0;
}

int main() {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    const size_t big = size_t(4) << 30;
    float4* buf;
    float* out;
    CK(cudaMalloc(&buf, big));
    CK(cudaMemset(buf, 0, big));
    CK(cudaMalloc(&out, size_t(p.multiProcessorCount) * 8 * 256 * 4 * 4));
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"gather\": [\n", p.name,
           p.multiProcessorCount, p.l2CacheSize);
    bool first = true;
    const size_t fps[] = {size_t(16) << 20, size_t(48) << 20, size_t(96) << 20, size_t(128) << 20,
                          size_t(256) << 20, big};
    for (size_t fp : fps) {
        if (run<16>(buf, fp, out, p.multiProcessorCount, first)) return 1;
        if (run<32>(buf, fp, out, p.multiProcessorCount, first)) return 1;
        if (run<64>(buf, fp, out, p.multiProcessorCount, first)) return 1;
        if (run<128>(buf, fp, out, p.multiProcessorCount, first)) return 1;
        if (run<512>(buf, fp, out, p.multiProcessorCount, first)) return 1;
    }
    // streaming read of the whole 4 GB buffer
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
    const int sb = p.multiProcessorCount * 8;
    k_stream<<<sb, 256>>>(buf, big / 16, out);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(a));
        k_stream<<<sb, 256>>>(buf, big / 16, out);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms; CK(cudaEventElapsedTime(&ms, a, b));
        if (ms < best) best = ms;
    }
    printf("\n], \"stream_read_gbs\": %.1f}\n", big / (best * 1e-3) / 1e9);
    return 0;
}
