// daspmm — host-side launch plan for one SpMM call (no CUDA kernels here).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

namespace daspmm {

template <typename T>
struct SpmmArgs;

// Launch shape chosen by plan_spmm() in abi.cu.
struct Plan {
    int kernel = 0;      // 0..7 = 4m + 2n + k (kernel_id.hpp:25-27)
    bool cm = false;     // B column-major (N-loop CM)
    bool exact = false;  // reference evaluation order, no FMA contraction
    int V = 1;           // vector width (elements per lane per column slot)
    int L = 1;           // SR: lanes per group (LPR); PR: group width W
    int X = 1;           // SR: column slots per lane (CPL); PR: slots per lane (OWN)
    dim3 grid;
    int64_t P = 0;       // EB chunks
    int64_t rpg = 1;     // RB+SR rows per group (row-block size)
    bool cta = false;    // EB+SR fast path: CTA-combined boundary rows (k_eb_sr_cta)
    int cta_threads = 64;   // ... its CTA size (64, 128 or 256)
    bool thr = false;    // EB+SR fast path for one-lane groups: staged sub-chunks (k_eb_sr_thr)
    int64_t sub = 0;     // ... its pairs per group sub-chunk
    int thr_threads = 256;  // CTA size of the one-lane staged path (64, 128 or 256)
    int rb_threads = 256;   // CTA size of fast f32 RB+RM+SR (k_rb_sr)
    int lean_threads = 256; // CTA size of the lean kernels (128 or 256)
    bool lean = false;   // RB/EB+RM+SR lean kernels (lean.cuh), fp32 fast mode
    bool lean_rw = false;  // ... EB: range walk with COO row ids (short rows)
    bool tma = false;    // EB+RM+SR with TMA gather4 B-row fetches (tma_gather.cuh)
    int win_rows = 0;    // RB+SR window kernel (k_rb_sr_win): rows per CTA panel, 0 = off
    bool repl = false;   // RB+SR with the replicated row epilogue (daspmm_spmm_rows_to)
    size_t win_smem = 0; // ... its dynamic shared memory (B window + TMA alignment lead)
    bool pdl = false;    // EB: launch the kernel programmatically after its prologue
    bool tile = false;   // RB+RM+SR on the handle's dense row-panel tiles (tile.cuh)
    int tile_rl = 1;     // ... row lanes per panel (1 or kTileRows); L = column lanes
    int tile_u = 2;      // ... tile columns (B rows) in flight per lane (2, 4 or 8)
    bool cm_rows = false;  // RB+CM+SR with lanes over rows (spmm_cm.cu); L = columns per block
};

// Kernel launch; with pdl, programmatic stream serialization: the kernel may start while
// the previous kernel of the stream (the EB prologue) still runs — the EB kernels wait
// for it (griddep_wait, common.cuh) only before their atomic deposits.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t s, Args... args) {
    if (!pdl) {
        k<<<grid, block, smem, s>>>(args...);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, args...);
}

// Shared-memory carveout of one kernel, set once per process (percent of the unified
// L1 / shared array; < 0 leaves the driver's choice). Kernels that size their occupancy
// by static shared memory set it explicitly: left to the driver, the staged tile walk
// ran at 1 CTA per SM in one process and 5 in another (banded s20 N = 64: 526 vs 180 us,
// profiles/r02_carveout_probe.txt).
template <auto K>
inline void carveout_once(int pct) {
    if (pct < 0) return;
    static bool done[64] = {};  // per device: function attributes are set per context
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        cudaGetLastError();
        return;
    }
    if (done[dev]) return;
    cudaFuncSetAttribute(K, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaGetLastError();
    done[dev] = true;
}
// DASPMM_<NAME>_CARVEOUT override (tuning), read once.
inline int carveout_env(const char* name, int dflt) {
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
}

// Launch site of the instantiation tables (`p`, `a`, `s` in scope). A translation unit
// whose kernels follow a prologue defines DASPMM_PDL_EXPR before including this header.
#ifndef DASPMM_PDL_EXPR
#define DASPMM_PDL_EXPR false
#endif
#define DASPMM_GO(K, G, NT)                                                          \
    do {                                                                             \
        const cudaError_t e_ = launch_k(DASPMM_PDL_EXPR, K, G, dim3(NT), 0, s, a);   \
        if (e_ != cudaSuccess) return e_;                                            \
    } while (0)

// Pairs per thread of the one-lane EB+SR path (k_eb_sr_thr). Measured on B200 (uniform
// s20): V <= 2 takes 12 (4 x odd: 128-bit conflict-free shared reads; N = 2 129 -> 105
// us), V = 4 keeps 7 (odd, scalar reads; 12 spent 80 registers and ran 126 -> 150 us).
constexpr int kThrS = 12;
constexpr int kTmaWarpsHost = 4;  // == kTmaWarps (tma_gather.cuh)
constexpr int kThrS4 = 7;

// Largest dynamic shared memory of the RB window kernel (B window + alignment lead);
// three CTAs per SM fit in the 228 KB carveout.
constexpr size_t kWinSmemMax = 72 * 1024;

// Each returns cudaErrorNotSupported for a shape with no instantiation.
cudaError_t launch_sr_lean(const Plan&, const SpmmArgs<float>&, cudaStream_t);
cudaError_t launch_eb_sr_tma(const Plan&, const SpmmArgs<float>&, cudaStream_t);
bool tma_gather_supported(const void* B, int64_t ldb, int64_t N, int64_t K);
int tma_box_cols(int64_t N);
template <typename T> cudaError_t launch_rb_sr(const Plan&, const SpmmArgs<T>&, cudaStream_t);
template <typename T> cudaError_t launch_rb_pr(const Plan&, const SpmmArgs<T>&, cudaStream_t);
template <typename T> cudaError_t launch_eb_sr(const Plan&, const SpmmArgs<T>&, cudaStream_t);
template <typename T> cudaError_t launch_eb_pr(const Plan&, const SpmmArgs<T>&, cudaStream_t);
// RB+RM+SR on dense row-panel tiles (spmm_tile.cu); p.L column lanes x p.tile_rl rows.
cudaError_t launch_rb_sr_tile(const Plan&, const SpmmArgs<float>&, const int* off, const int* c0,
                              const float* val, int64_t n_pan, cudaStream_t);
// RB+CM+SR, lanes over rows, p.L columns per grid.y block (spmm_cm.cu).
cudaError_t launch_rb_cm_rows(const Plan&, const SpmmArgs<float>&, cudaStream_t);
// PR groups wider than a warp (W = 64 .. 1024), RB and EB (spmm_pr_wide.cu).
template <typename T> cudaError_t launch_pr_wide(const Plan&, const SpmmArgs<T>&, cudaStream_t);
template <typename T>
cudaError_t launch_eb_prep_uniform(const int* rows, int64_t nnz, int64_t sub, int64_t n_sub, int G,
                                   T* C, int64_t ldc, int N, const int* empty_rows, int n_empty,
                                   cudaStream_t s);
// rows == nullptr: partition_elements API (writes chunk_row); else SpMM zeroing only.
template <typename T>
cudaError_t launch_eb_prep(const int* rp, int M, int64_t nnz, int64_t P, int* chunk_row, T* C,
                           int64_t ldc, int N, const int* empty_rows, int n_empty,
                           const int* rows, cudaStream_t s);

}  // namespace daspmm
