// daspmm — EB+RM+SR with the dense-B row gathers done by the Tensor Memory Accelerator
// (sm_100 `cp.async.bulk.tensor.2d ... tile::gather4`: one instruction fetches 4
// arbitrary rows of a 2-D tensor into shared memory).
//
// Same design point as k_eb_sr / k_eb_sr_lean (EB chunks, lanes span columns, each lane
// accumulates its V-wide column slot sequentially in nnz order; spmm.hpp:108-159). What
// changes is who moves B: on power-law inputs at N >= 32 the LSU-issued gathers run
// latency-bound (ncu: long-scoreboard stalls, L2 at ~45% of its throughput) because a
// warp can only keep as many gathers in flight as it has registers for. Here each warp
// owns a ring of D shared-memory stages of 16 B rows; lane 0 issues the gather4s for
// stage k + D while the warp consumes stage k, so D x 16 rows per warp (tens of KB per
// SM) are in flight without holding registers, and the consumer's reads are LDS.
//
//   warp w of CTA b owns nonzeros [(4b + w) * Lw, (4b + w + 1) * Lw) (Lw % 16 == 0);
//   rows cut by those ends take vector atomics (pre-zeroed by k_eb_prep_uniform with
//   sub = Lw), rows inside are stored; empty rows are pre-zeroed.
//   The tensor map describes B as {N, K} fp32 (row pitch ldb), box {BC, 1}; columns past
//   N inside a box are zero-filled by the TMA and never stored.
#pragma once

#include <cuda.h>

#include "kernels.cuh"

namespace daspmm {

constexpr int kTmaWarps = 4;   // consumer warps per CTA (each also issues its own TMA)
constexpr int kTmaStageNnz = 16;

__device__ __forceinline__ void tma_gather4(void* dst, const CUtensorMap* map, int col0, int r0,
                                            int r1, int r2, int r3, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(col0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
        "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int BC, int D>
__global__ void __launch_bounds__(kTmaWarps * 32, 1)
k_eb_sr_tma(const __grid_constant__ CUtensorMap tmB, const SpmmArgs<float> a, const int Lw) {
    constexpr int V = BC / 32;  // columns per lane
    constexpr int SN = kTmaStageNnz;
    constexpr unsigned kStageBytes = SN * BC * sizeof(float);
    extern __shared__ __align__(1024) unsigned char dsm[];
    __shared__ __align__(8) uint64_t full[kTmaWarps][D];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* ring = reinterpret_cast<float*>(dsm + size_t(w) * D * kStageBytes);
    const int64_t e0l = (int64_t(blockIdx.x) * kTmaWarps + w) * Lw;
    if (e0l >= a.nnz) return;  // whole warp; no CTA-wide synchronisation below
    if (lane == 0)
        for (int d = 0; d < D; ++d) mbar_init(&full[w][d], 1);
    __syncwarp();
    const int nnz = int(a.nnz);
    const int e0 = int(e0l), e1 = min(nnz, e0 + Lw);
    const int nst = (e1 - e0 + SN - 1) / SN;
    const int tile0 = blockIdx.y * BC;

    // lane 0: stage k's 16 column indices -> four gather4 into ring slot k % D
    auto issue = [&](int k) {
        const int es = e0 + k * SN;
        int c[SN];
        if (es + SN <= nnz) {
#pragma unroll
            for (int q = 0; q < SN / 4; ++q) {
                const int4 v = __ldg(reinterpret_cast<const int4*>(a.ci + es) + q);
                c[4 * q] = v.x; c[4 * q + 1] = v.y; c[4 * q + 2] = v.z; c[4 * q + 3] = v.w;
            }
        } else {  // array tail: repeat the last column (fetched, never used)
            const int last = __ldg(a.ci + nnz - 1);
#pragma unroll
            for (int j = 0; j < SN; ++j) c[j] = es + j < nnz ? __ldg(a.ci + es + j) : last;
        }
        uint64_t* bar = &full[w][k % D];
        float* dst = ring + (k % D) * SN * BC;
        mbar_expect_tx(bar, kStageBytes);
#pragma unroll
        for (int g = 0; g < SN / 4; ++g)
            tma_gather4(dst + g * 4 * BC, &tmB, tile0, c[4 * g], c[4 * g + 1], c[4 * g + 2],
                        c[4 * g + 3], bar);
    };
    if (lane == 0)
        for (int k = 0; k < min(D, nst); ++k) issue(k);

    const int first_row = __ldg(a.rows + e0), last_row = __ldg(a.rows + e1 - 1);
    const bool first_split = e0 > 0 && __ldg(a.rows + e0 - 1) == first_row;
    const bool last_split = e1 < nnz && __ldg(a.rows + e1) == last_row;
    const int col = tile0 + lane * V;
    const bool colok = col < a.N;
    Frag<float, V> acc;
#pragma unroll
    for (int i = 0; i < V; ++i) acc.v[i] = 0.f;
    int r = first_row;
    auto deposit = [&](int row) {
        if (colok) {
            float* y = a.C + int64_t(row) * a.ldc + col;
            if ((first_split && row == first_row) || (last_split && row == last_row))
                atomic_add_frag(y, acc);
            else
                st_frag(y, acc);
        }
#pragma unroll
        for (int i = 0; i < V; ++i) acc.v[i] = 0.f;
    };
    // values and row ids of a stage: lanes 0..15 hold one pair each (prefetched a stage
    // ahead so their latency overlaps the previous stage)
    auto load_vr = [&](int k, float& v, int& rid) {
        const int e = e0 + k * SN + (lane & (SN - 1));
        const bool ok = k < nst && e < e1;
        v = ok ? __ldg(a.va + e) : 0.f;
        rid = ok ? __ldg(a.rows + e) : INT_MAX;
    };
    float vcur, vnext;
    int rcur, rnext;
    load_vr(0, vcur, rcur);
    for (int k = 0; k < nst; ++k) {
        load_vr(k + 1, vnext, rnext);
        const int n = min(SN, e1 - (e0 + k * SN));
        mbar_wait(&full[w][k % D], unsigned((k / D) & 1));
        const float* st = ring + (k % D) * SN * BC + lane * V;
        Frag<float, V> b[SN];
#pragma unroll
        for (int j = 0; j < SN; ++j) b[j] = ld_frag_shared<float, V>(st + j * BC);
#pragma unroll
        for (int j = 0; j < SN; ++j) {
            const float v = __shfl_sync(kFull, vcur, j);
            const int rid = __shfl_sync(kFull, rcur, j);
            if (j < n) {
                if (rid != r) {
                    deposit(r);
                    r = rid;
                }
#pragma unroll
                for (int i = 0; i < V; ++i) acc.v[i] = fmaf(v, b[j].v[i], acc.v[i]);
            }
        }
        __syncwarp();  // every lane has read slot k % D
        if (lane == 0 && k + D < nst) {
            fence_proxy_async_smem();  // order the slot's generic reads before the refill
            issue(k + D);
        }
        vcur = vnext;
        rcur = rnext;
    }
    deposit(r);
}

}  // namespace daspmm
