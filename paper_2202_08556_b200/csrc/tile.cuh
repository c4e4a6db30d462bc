// daspmm — RB+RM+SR on dense row-panel tiles (fp32 fast mode): the launch variant for
// matrices whose neighbouring rows share their columns (banded, stencil and mesh
// matrices).
//
// The handle keeps, for every panel of kTileRows consecutive rows, the panel's column
// window [c0, c0 + w) and its nonzeros laid out as a dense w x kTileRows tile (k-major:
// tile[k * kTileRows + r] = A[r0 + r][c0 + k], 0 where A has no entry), built once
// (ensure_tiles, features.cu) and only when the tiles are at least half full. A group
// walks its panel's window once: each B row c0 + k is gathered ONCE for all kTileRows
// rows instead of once per nonzero, so the L1/L2 gather volume falls by the tile's
// rows x fill (banded half-width 8: 8 x 0.71 = 5.7x) — the gathers were what bounded
// RB+RM+SR on these matrices (banded s20 N = 128: L1 at 95% of peak).
//
// Arithmetic is the base kernel's: per output element one fmaf per column in ascending
// column order, starting from +0. An absent entry contributes fmaf(0, b, acc) == acc
// exactly for finite b (acc is never -0: it starts at +0 and x + (-x) rounds to +0), so
// with rows stored in ascending column order (checked when the tiles are built) the
// results equal k_rb_sr's bit for bit. A non-finite B element under an absent entry
// would turn 0 * b into NaN where the reference has no product: any row whose result is
// not finite is recomputed from the CSR arrays (the base walk's exact sequence), so
// Inf / NaN propagate exactly as in the reference (spmm.hpp:85-88).
//
// Lane mapping: a group of CL x RL lanes owns one panel. CL lanes span the column tile
// (V-wide slots, CPL per lane), RL lanes split the panel's rows (kTileRows / RL rows per
// lane). Wide N uses RL = 1 (a lane keeps all rows of its columns; the tile's k-th
// column of values is one broadcast 32-byte load per group); narrow N uses RL = 8 (a
// lane per row; the group reads a tile column as one coalesced 32-byte segment and the
// B row as a broadcast).
#pragma once

#include "kernels.cuh"

namespace daspmm {

constexpr int kTileRows = 8;

struct TileArgs {
    const int* __restrict__ off;   // n_pan + 1 tile offsets (floats)
    const int* __restrict__ c0;    // n_pan first column of each panel's window
    const float* __restrict__ val; // tiles, k-major
    int n_pan;
};

// Shared-memory budget of one CTA for staged tile columns: each group stages up to
// kTileStage(G) columns of its panel (k-major, kTileRows floats each) at a time.
constexpr int kTileSmemFloats = 8192;  // 32 KB per CTA
template <int G, int NT>
constexpr int tile_stage_cols() {
    return kTileSmemFloats / (NT / G) / kTileRows;
}

// The walk is software-pipelined: B rows k + U are requested while rows k are consumed,
// so each lane keeps U gathers in flight through the whole window (a plain unrolled loop
// drained them at every step: ncu showed the kernel latency-bound at 45% of the DRAM
// rate with the traffic already at the algorithmic minimum). The panel's tile values
// are staged once into shared memory (coalesced 16-byte loads) and read back as
// broadcasts, keeping them off the registers and the dependent-load chain.
#ifndef DASPMM_TILE_MINB
#define DASPMM_TILE_MINB 1
#endif
template <int V, int CL, int RL, int CPL, int NT, int U>
__global__ void __launch_bounds__(NT, DASPMM_TILE_MINB) k_rb_sr_tile(const SpmmArgs<float> a, const TileArgs t) {
    constexpr int G = CL * RL;                 // lanes per group (one panel)
    constexpr int RPL = kTileRows / RL;        // rows per lane
    constexpr int TN = CL * V * CPL;           // columns per tile (blockIdx.y)
    constexpr int KS = tile_stage_cols<G, NT>();  // staged tile columns per group
    static_assert(KS >= U && KS % U == 0, "stage must hold whole pipeline steps");
    __shared__ __align__(16) float stage[NT / G][KS * kTileRows];
    const int gl = threadIdx.x & (G - 1);
    const int cl = gl % CL, rl = gl / CL;
    const unsigned mask = group_mask<G>();
    const int64_t p = (int64_t(blockIdx.x) * NT + threadIdx.x) / G;
    if (p >= t.n_pan) return;  // whole groups leave together
    float* sg = stage[threadIdx.x / G];
    const int r_base = int(p) * kTileRows + rl;  // rows r_base + RL * j, j < RPL
    const int off0 = __ldg(t.off + p);
    const int w = (__ldg(t.off + p + 1) - off0) / kTileRows;
    const int c0 = __ldg(t.c0 + p);
    const int n0 = blockIdx.y * TN + cl * V;

    Frag<float, V> acc[RPL][CPL];
#pragma unroll
    for (int j = 0; j < RPL; ++j)
#pragma unroll
        for (int s = 0; s < CPL; ++s)
#pragma unroll
            for (int i = 0; i < V; ++i) acc[j][s].v[i] = 0.f;

    // per-slot byte base of B's column (lanes past N read column 0, never stored)
    const char* Bcol[CPL];
#pragma unroll
    for (int s = 0; s < CPL; ++s) {
        const int col = n0 + s * CL * V;
        Bcol[s] = reinterpret_cast<const char*>(a.B + (col < a.N ? col : 0));
    }
    const int ldb_bytes = int(a.ldb) * int(sizeof(float));
    auto gather = [&](int k, Frag<float, V>* b) {  // B row c0 + k (k clamped into the window)
#pragma unroll
        for (int s = 0; s < CPL; ++s)
            b[s] = ld_frag<float, V>(reinterpret_cast<const float*>(
                Bcol[s] + int64_t(c0 + min(k, w - 1)) * ldb_bytes));
    };
    Frag<float, V> b[U][CPL];
    if (w > 0) {
#pragma unroll
        for (int u = 0; u < U; ++u) gather(u, b[u]);
    }
    const float4* tile4 = reinterpret_cast<const float4*>(t.val + off0);
    for (int kc = 0; kc < w; kc += KS) {
        const int kw = min(KS, w - kc);
        __syncwarp(mask);  // the previous chunk's reads are done
        for (int i = gl; i < kw * (kTileRows / 4); i += G)
            reinterpret_cast<float4*>(sg)[i] = __ldg(tile4 + kc * (kTileRows / 4) + i);
        __syncwarp(mask);
        for (int k0 = 0; k0 < kw; k0 += U) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (k0 + u < kw) {
                    float av[RPL];
                    if constexpr (RL == 1) {
                        const float4 lo = reinterpret_cast<const float4*>(sg)[(k0 + u) * 2];
                        const float4 hi = reinterpret_cast<const float4*>(sg)[(k0 + u) * 2 + 1];
                        av[0] = lo.x; av[1] = lo.y; av[2] = lo.z; av[3] = lo.w;
                        av[4] = hi.x; av[5] = hi.y; av[6] = hi.z; av[7] = hi.w;
                    } else {
#pragma unroll
                        for (int j = 0; j < RPL; ++j) av[j] = sg[(k0 + u) * kTileRows + rl + RL * j];
                    }
#pragma unroll
                    for (int j = 0; j < RPL; ++j)
#pragma unroll
                        for (int s = 0; s < CPL; ++s)
#pragma unroll
                            for (int i = 0; i < V; ++i)
                                acc[j][s].v[i] = fmaf(av[j], b[u][s].v[i], acc[j][s].v[i]);
                }
                gather(kc + k0 + u + U, b[u]);  // refill the slot U rows ahead
            }
        }
    }

#pragma unroll
    for (int j = 0; j < RPL; ++j) {
        const int r = r_base + RL * j;
        if (r >= a.M) break;
#pragma unroll
        for (int s = 0; s < CPL; ++s) {
            const int col = n0 + s * CL * V;
            if (col >= a.N) continue;
            bool finite = true;
#pragma unroll
            for (int i = 0; i < V; ++i) finite &= isfinite(acc[j][s].v[i]);
            Frag<float, V> out = acc[j][s];
            if (!finite) {  // rare: replay the row from CSR (the base walk's sequence)
#pragma unroll
                for (int i = 0; i < V; ++i) out.v[i] = 0.f;
                const int e1 = __ldg(a.rp + r + 1);
                for (int e = __ldg(a.rp + r); e < e1; ++e) {
                    const float v = __ldg(a.va + e);
                    const Frag<float, V> bb = ld_frag<float, V>(
                        a.B + int64_t(__ldg(a.ci + e)) * a.ldb + col);
#pragma unroll
                    for (int i = 0; i < V; ++i) out.v[i] = fmaf(v, bb.v[i], out.v[i]);
                }
            }
            st_frag(a.C + int64_t(r) * a.ldc + col, out);
        }
    }
}

// Narrow N (one to four column slots per panel): the direct walk — tile values and B
// rows loaded together from global memory U columns at a time, no staging. Many small
// groups share a CTA here, and staging would cost occupancy (shared memory) and a
// synchronisation per chunk for a few FMAs per column (banded s20 N = 8: 53 us direct vs
// 75 us staged; N >= 32 is the other way round: 156 vs 94 us).
template <int V, int CL, int RL, int CPL, int NT, int U>
__global__ void __launch_bounds__(NT) k_rb_sr_tile_direct(const SpmmArgs<float> a, const TileArgs t) {
    constexpr int G = CL * RL;                 // lanes per group (one panel)
    constexpr int RPL = kTileRows / RL;        // rows per lane
    constexpr int TN = CL * V * CPL;           // columns per tile (blockIdx.y)
    const int gl = threadIdx.x & (G - 1);
    const int cl = gl % CL, rl = gl / CL;
    const int64_t p = (int64_t(blockIdx.x) * NT + threadIdx.x) / G;
    if (p >= t.n_pan) return;
    const int r_base = int(p) * kTileRows + rl;  // rows r_base + RL * j, j < RPL
    const int off0 = __ldg(t.off + p);
    const int w = (__ldg(t.off + p + 1) - off0) / kTileRows;
    const int c0 = __ldg(t.c0 + p);
    const int n0 = blockIdx.y * TN + cl * V;

    Frag<float, V> acc[RPL][CPL];
#pragma unroll
    for (int j = 0; j < RPL; ++j)
#pragma unroll
        for (int s = 0; s < CPL; ++s)
#pragma unroll
            for (int i = 0; i < V; ++i) acc[j][s].v[i] = 0.f;

    // per-slot byte base of B's column (lanes past N read column 0, never stored)
    const char* Bcol[CPL];
#pragma unroll
    for (int s = 0; s < CPL; ++s) {
        const int col = n0 + s * CL * V;
        Bcol[s] = reinterpret_cast<const char*>(a.B + (col < a.N ? col : 0));
    }
    const int ldb_bytes = int(a.ldb) * int(sizeof(float));
    const float* tv = t.val + off0;
    for (int k0 = 0; k0 < w; k0 += U) {
        float av[U][RPL];
        Frag<float, V> b[U][CPL];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int k = k0 + u < w ? k0 + u : w - 1;  // tail: repeat the last column, unused
            const float* col = tv + int64_t(k) * kTileRows;
            if constexpr (RL == 1) {
                const float4 lo = __ldg(reinterpret_cast<const float4*>(col));
                const float4 hi = __ldg(reinterpret_cast<const float4*>(col) + 1);
                av[u][0] = lo.x; av[u][1] = lo.y; av[u][2] = lo.z; av[u][3] = lo.w;
                av[u][4] = hi.x; av[u][5] = hi.y; av[u][6] = hi.z; av[u][7] = hi.w;
            } else {
#pragma unroll
                for (int j = 0; j < RPL; ++j) av[u][j] = __ldg(col + rl + RL * j);
            }
#pragma unroll
            for (int s = 0; s < CPL; ++s)
                b[u][s] = ld_frag<float, V>(reinterpret_cast<const float*>(
                    Bcol[s] + int64_t(c0 + k) * ldb_bytes));
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (k0 + u < w) {
#pragma unroll
                for (int j = 0; j < RPL; ++j)
#pragma unroll
                    for (int s = 0; s < CPL; ++s)
#pragma unroll
                        for (int i = 0; i < V; ++i)
                            acc[j][s].v[i] = fmaf(av[u][j], b[u][s].v[i], acc[j][s].v[i]);
            }
        }
    }

#pragma unroll
    for (int j = 0; j < RPL; ++j) {
        const int r = r_base + RL * j;
        if (r >= a.M) break;
#pragma unroll
        for (int s = 0; s < CPL; ++s) {
            const int col = n0 + s * CL * V;
            if (col >= a.N) continue;
            bool finite = true;
#pragma unroll
            for (int i = 0; i < V; ++i) finite &= isfinite(acc[j][s].v[i]);
            Frag<float, V> out = acc[j][s];
            if (!finite) {  // rare: replay the row from CSR (the base walk's sequence)
#pragma unroll
                for (int i = 0; i < V; ++i) out.v[i] = 0.f;
                const int e1 = __ldg(a.rp + r + 1);
                for (int e = __ldg(a.rp + r); e < e1; ++e) {
                    const float v = __ldg(a.va + e);
                    const Frag<float, V> bb = ld_frag<float, V>(
                        a.B + int64_t(__ldg(a.ci + e)) * a.ldb + col);
#pragma unroll
                    for (int i = 0; i < V; ++i) out.v[i] = fmaf(v, bb.v[i], out.v[i]);
                }
            }
            st_frag(a.C + int64_t(r) * a.ldc + col, out);
        }
    }
}

}  // namespace daspmm
