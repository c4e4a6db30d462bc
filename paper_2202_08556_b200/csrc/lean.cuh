// daspmm — lean SR kernels for wide lane groups (fp32, row-major B, fast mode).
//
// The same design points as k_rb_sr / k_eb_sr (RB+RM+SR, EB+RM+SR: lanes span columns,
// each lane accumulates its V-wide column slot sequentially in nnz order, spmm.hpp:
// 66-88 and 108-159), restructured around the instruction budget per nonzero.
// ncu on k_rb_sr (banded s20, N = 128) showed issue-bound execution: ~29 warp
// instructions per nonzero for the 1 gather + 4 FFMA that are essential. Here:
//
//   * A's (col, val) pairs are read as aligned quads — one 16-B load of 4 column
//     indices and one of 4 values, every lane of the group at the same address
//     (one L1 wavefront, broadcast) — instead of per-lane loads plus two shuffles
//     per nonzero;
//   * walks: one row segment at a time (segment walk; next row from the COO id at the
//     segment end), or a contiguous nonzero range in 8-element blocks with the COO row
//     ids loaded as quads too (range walk): a block that stays inside the current row
//     runs branch-free; masked slots (range edges) issue no load and no FFMA;
//   * the segment walks take two quads per iteration (8 independent B-row gathers in
//     flight per lane before the FFMAs that consume them); the range walk takes one and
//     spends the registers on occupancy instead (measured, below).
//
//   RB (K0, opt-in DASPMM_LEAN_RB=1): group owns rows [g*rpg, (g+1)*rpg), one segment
//            per row, every row stored (empty rows store zeros).
//   EB (K4, N <= 16 or long rows): group owns the nnz chunk [w*chunk, (w+1)*chunk); a
//            row wholly inside the chunk is stored, a row cut by the chunk's ends takes
//            a vector atomic add (pre-zeroed by k_eb_prep_uniform), empty rows are
//            pre-zeroed.
// Where each wins is measured in DESIGN.md §3.1; CTA size is a template parameter
// (64 threads by default, Plan::lean_threads).
//
// Requires ci/va/rows 16-byte aligned (quad loads) and ldb * 4 < 2^31 (plan_spmm checks);
// the last partial quad of the arrays is read with scalar loads so nothing past nnz is
// touched.
#pragma once

#include "kernels.cuh"

namespace daspmm {

// Resident 256-thread CTAs per SM the lean kernels are compiled for (register cap 65536
// / (256 x minB); scaled for smaller CTAs). Measured on B200: the RB walk gains from 4
// (64 registers, 32 warps: uniform s20 N = 128 1294 -> 1245 us), the EB walks lose at 4
// (power-law N = 16 range walk 217 -> 303 us) and keep 3 (80 registers).
#ifndef DASPMM_RBL_MINB
#define DASPMM_RBL_MINB 4
#endif
constexpr int kLeanMinBlocksRB = DASPMM_RBL_MINB;
// Range walk: one quad of (col, val, row) per iteration and 4 CTAs per SM for groups of
// >= 4 lanes (56 registers), 3 below (68). Two quads per iteration (8 gathers in flight,
// 80 registers) ran power-law s20 N = 8 151.9 -> 137.7 us and N = 16 194.8 -> 168.2 us
// slower (profiles/r02_rw_quads_probe.txt): occupancy beats per-lane depth here.
#ifndef DASPMM_RW_QUADS
#define DASPMM_RW_QUADS 1
#endif
// EB segment walk (long rows, e.g. c3): wide groups (>= 16 lanes) take one quad per
// iteration at 5 CTAs per SM (48 registers): c3 3.66 -> 3.29 ms; narrower groups keep two
// quads at 3 (profiles/r02_seg_quads_probe.txt).
constexpr int kLeanMinBlocksEB = 3;
template <int LPR>
constexpr int lean_seg_min_blocks() { return LPR >= 16 ? 5 : kLeanMinBlocksEB; }
template <int LPR>
constexpr int lean_seg_quads() { return LPR >= 16 ? 1 : 2; }
#ifndef DASPMM_RBL_QUADS
#define DASPMM_RBL_QUADS 2
#endif
template <int LPR>
constexpr int lean_rw_min_blocks() { return LPR >= 4 ? 4 : 3; }

struct Quad {
    int c[4];
    float v[4];
};

// Elements q .. q+3 of the array tail (q + 4 > nnz): scalar loads, past-the-end
// elements (0, 0). Out of line so the common path carries no per-element bounds math.
__device__ __noinline__ Quad load_quad_tail(const int* __restrict__ ci,
                                            const float* __restrict__ va, int q, int nnz) {
    Quad r;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const bool ok = q + j < nnz;
        r.c[j] = ok ? __ldg(ci + q + j) : 0;
        r.v[j] = ok ? __ldg(va + q + j) : 0.f;
    }
    return r;
}

// Elements q .. q+3 of (ci, va); q % 4 == 0.
__device__ __forceinline__ Quad load_quad(const SpmmArgs<float>& a, int q, int nnz) {
    if (__builtin_expect(q + 4 > nnz, 0)) return load_quad_tail(a.ci, a.va, q, nnz);
    Quad r;
    const int4 c = __ldg(reinterpret_cast<const int4*>(a.ci + q));
    const float4 v = __ldg(reinterpret_cast<const float4*>(a.va + q));
    r.c[0] = c.x; r.c[1] = c.y; r.c[2] = c.z; r.c[3] = c.w;
    r.v[0] = v.x; r.v[1] = v.y; r.v[2] = v.z; r.v[3] = v.w;
    return r;
}

// Sum over e in [s, e1) of va[e] * B[ci[e], col .. col+V), sequential in e (FFMA).
// Bc = &B[0][col] as bytes, ldb_bytes = ldb * sizeof(float): each gather address is one
// IMAD.WIDE (col index x row pitch + base). Masked slots (outside [s, e1)) issue no load
// and no FFMA (predicated), so stale registers never reach the accumulator.
template <int V, int QB = 2>
__device__ __forceinline__ Frag<float, V> row_segment(const SpmmArgs<float>& a, int s, int e1,
                                                      const char* __restrict__ Bc,
                                                      int ldb_bytes, bool colok) {
    constexpr int BLK = 4 * QB;  // elements per iteration (QB quads)
    Frag<float, V> acc;
#pragma unroll
    for (int i = 0; i < V; ++i) acc.v[i] = 0.f;
    const int nnz = int(a.nnz);
    for (int q = s & ~3; q < e1; q += BLK) {
        const int lo = max(s - q, 0), hi = min(e1 - q, BLK);  // valid slots [lo, hi)
        const unsigned valid = colok ? ((1u << hi) - 1u) & ~((1u << lo) - 1u) : 0u;
        const Quad A0 = load_quad(a, q, nnz);
        Quad A1;  // slots 4..7 are valid only when it is loaded
        if (BLK > 4 && hi > 4) A1 = load_quad(a, q + 4, nnz);  // group-uniform
        Frag<float, V> b[BLK];
#pragma unroll
        for (int j = 0; j < BLK; ++j) {
            const int c = j < 4 ? A0.c[j] : A1.c[j - 4];
            if (valid & (1u << j))
                b[j] = ld_frag<float, V>(reinterpret_cast<const float*>(
                    Bc + int64_t(c) * ldb_bytes));
        }
#pragma unroll
        for (int j = 0; j < BLK; ++j) {
            const float v = j < 4 ? A0.v[j] : A1.v[j - 4];
            if (valid & (1u << j)) {
#pragma unroll
                for (int i = 0; i < V; ++i) acc.v[i] = fmaf(v, b[j].v[i], acc.v[i]);
            }
        }
    }
    return acc;
}

// Row ids q .. q+3 of the handle's COO array (same bounds rule as load_quad).
__device__ __forceinline__ int4 load_rquad(const SpmmArgs<float>& a, int q, int nnz) {
    if (__builtin_expect(q + 4 > nnz, 0)) {
        int4 r;
        r.x = __ldg(a.rows + q);  // q < nnz always holds for a loaded quad
        r.y = q + 1 < nnz ? __ldg(a.rows + q + 1) : INT_MAX;
        r.z = q + 2 < nnz ? __ldg(a.rows + q + 2) : INT_MAX;
        r.w = q + 3 < nnz ? __ldg(a.rows + q + 3) : INT_MAX;
        return r;
    }
    return __ldg(reinterpret_cast<const int4*>(a.rows + q));
}

__device__ __forceinline__ int quad_get(const int4& r, int j) {
    return j == 0 ? r.x : j == 1 ? r.y : j == 2 ? r.z : r.w;
}

// One lane group walks the nonzero range [e0, e1) in 8-element blocks (two aligned
// quads of cols, vals and COO row ids, broadcast-loaded). Row r accumulates in nnz
// order; when the row id changes the finished row is deposited: plain store when the
// row is wholly inside the range, vector atomic add when the range cuts it (EB chunk
// ends; such rows are pre-zeroed). A block whose last valid element still belongs to
// the current row (the common case) takes the branch-free path.
template <int V>
__device__ __forceinline__ void range_walk(const SpmmArgs<float>& a, const int e0, const int e1,
                                           const bool first_split, const bool last_split,
                                           const char* __restrict__ Bc, const int ldb_bytes,
                                           float* __restrict__ Ccol, const bool colok) {
    const int nnz = int(a.nnz);
    const int r_first = __ldg(a.rows + e0);
    const int r_last = __ldg(a.rows + e1 - 1);
    int r = r_first;
    Frag<float, V> acc;
#pragma unroll
    for (int i = 0; i < V; ++i) acc.v[i] = 0.f;
    auto deposit = [&](int row) {
        if (colok) {
            float* y = Ccol + int64_t(row) * a.ldc;
            if ((first_split && row == r_first) || (last_split && row == r_last)) {
                griddep_wait();  // split row: zeroed by the EB prologue
                atomic_add_frag(y, acc);
            } else {
                st_frag(y, acc);
            }
        }
#pragma unroll
        for (int i = 0; i < V; ++i) acc.v[i] = 0.f;
    };
    constexpr int BLK = 4 * DASPMM_RW_QUADS;  // elements per iteration (1 or 2 quads)
    for (int q = e0 & ~3; q < e1; q += BLK) {
        const int lo = max(e0 - q, 0), hi = min(e1 - q, BLK);  // valid slots [lo, hi)
        const unsigned valid = ((1u << hi) - 1u) & ~((1u << lo) - 1u);
        const Quad A0 = load_quad(a, q, nnz);
        const int4 R0 = load_rquad(a, q, nnz);
        Quad A1;  // slots 4..7 are valid only when loaded
        int4 R1 = R0;
        if (BLK > 4 && hi > 4) {  // group-uniform
            A1 = load_quad(a, q + 4, nnz);
            R1 = load_rquad(a, q + 4, nnz);
        }
        Frag<float, V> b[BLK];
#pragma unroll
        for (int j = 0; j < BLK; ++j) {
            const int c = j < 4 ? A0.c[j] : A1.c[j - 4];
            if (colok && (valid & (1u << j)))
                b[j] = ld_frag<float, V>(reinterpret_cast<const float*>(
                    Bc + int64_t(c) * ldb_bytes));
        }
        const int rlast = hi > 4 ? quad_get(R1, hi - 5) : quad_get(R0, hi - 1);
        if (rlast == r) {
#pragma unroll
            for (int j = 0; j < BLK; ++j) {
                const float v = j < 4 ? A0.v[j] : A1.v[j - 4];
                if (valid & (1u << j)) {
#pragma unroll
                    for (int i = 0; i < V; ++i) acc.v[i] = fmaf(v, b[j].v[i], acc.v[i]);
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < BLK; ++j) {
                const float v = j < 4 ? A0.v[j] : A1.v[j - 4];
                const int rid = j < 4 ? quad_get(R0, j) : quad_get(R1, j - 4);
                if (valid & (1u << j)) {
                    if (rid != r) {
                        deposit(r);
                        r = rid;
                    }
#pragma unroll
                    for (int i = 0; i < V; ++i) acc.v[i] = fmaf(v, b[j].v[i], acc.v[i]);
                }
            }
        }
    }
    deposit(r);
}

// RB: group g owns rows [g*rpg, (g+1)*rpg), one row segment at a time; every row is
// owned (plain stores; empty rows store zeros).
template <int V, int LPR, int NT = kThreads>
__global__ void __launch_bounds__(NT, kLeanMinBlocksRB * (kThreads / NT)) k_rb_sr_lean(const SpmmArgs<float> a) {
    const int gl = threadIdx.x & (LPR - 1);
    const int64_t g = (int64_t(blockIdx.x) * NT + threadIdx.x) / LPR;
    const int64_t r0 = g * a.rpg;
    if (r0 >= a.M) return;
    const int r1 = int(min(int64_t(a.M), r0 + a.rpg));
    const int col = blockIdx.y * (LPR * V) + gl * V;
    const bool colok = col < a.N;
    const char* Bc = reinterpret_cast<const char*>(a.B + col);
    const int ldb_bytes = int(a.ldb) * int(sizeof(float));
    int s = __ldg(a.rp + r0);
    for (int r = int(r0); r < r1; ++r) {
        const int e1 = __ldg(a.rp + r + 1);
        const Frag<float, V> acc = row_segment<V, DASPMM_RBL_QUADS>(a, s, e1, Bc, ldb_bytes, colok);
        if (colok) st_frag(a.C + int64_t(r) * a.ldc + col, acc);
        s = e1;
    }
}

// EB, segment walk: group w owns the nnz chunk [w*sub, (w+1)*sub) and walks it one row
// segment at a time (next row from the COO id of the segment's end, so empty rows cost
// nothing). Rows cut by the chunk ends take atomics. Suits long rows.
template <int V, int LPR, int NT = kThreads>
__global__ void __launch_bounds__(NT, lean_seg_min_blocks<LPR>() * (kThreads / NT)) k_eb_sr_lean(const SpmmArgs<float> a) {
    const int gl = threadIdx.x & (LPR - 1);
    const int64_t w = (int64_t(blockIdx.x) * NT + threadIdx.x) / LPR;
    const int64_t e0l = w * a.sub;
    if (e0l >= a.nnz) {
        griddep_wait();
        return;
    }
    const int e0 = int(e0l), e1 = int(min(a.nnz, e0l + a.sub));
    const int col = blockIdx.y * (LPR * V) + gl * V;
    const bool colok = col < a.N;
    const char* Bc = reinterpret_cast<const char*>(a.B + col);
    const int ldb_bytes = int(a.ldb) * int(sizeof(float));
    int s = e0;
    int r = __ldg(a.rows + e0);
    while (true) {
        const int rs = __ldg(a.rp + r);
        const int re = __ldg(a.rp + r + 1);
        const int se = min(re, e1);
        const Frag<float, V> acc = row_segment<V, lean_seg_quads<LPR>()>(a, s, se, Bc, ldb_bytes, colok);
        if (colok) {
            float* y = a.C + int64_t(r) * a.ldc + col;
            if (rs >= e0 && re <= e1) {
                st_frag(y, acc);
            } else {
                griddep_wait();
                atomic_add_frag(y, acc);
            }
        }
        s = se;
        if (s >= e1) break;
        r = __ldg(a.rows + s);
    }
    griddep_wait();
}

// EB, range walk: the chunk as one nonzero range with COO row ids (range_walk). Suits
// short rows (power-law tails), where per-segment row-offset lookups would dominate.
template <int V, int LPR, int NT = kThreads>
__global__ void __launch_bounds__(NT, lean_rw_min_blocks<LPR>() * (kThreads / NT)) k_eb_sr_lean_rw(const SpmmArgs<float> a) {
    const int gl = threadIdx.x & (LPR - 1);
    const int64_t w = (int64_t(blockIdx.x) * NT + threadIdx.x) / LPR;
    const int64_t e0l = w * a.sub;
    if (e0l >= a.nnz) {
        griddep_wait();
        return;
    }
    const int e0 = int(e0l), e1 = int(min(a.nnz, e0l + a.sub));
    const bool first_split = e0 > 0 && __ldg(a.rows + e0 - 1) == __ldg(a.rows + e0);
    const bool last_split = e1 < a.nnz && __ldg(a.rows + e1) == __ldg(a.rows + e1 - 1);
    const int col = blockIdx.y * (LPR * V) + gl * V;
    range_walk<V>(a, e0, e1, first_split, last_split, reinterpret_cast<const char*>(a.B + col),
                  int(a.ldb) * int(sizeof(float)), a.C + col, col < a.N);
    griddep_wait();
}

}  // namespace daspmm
