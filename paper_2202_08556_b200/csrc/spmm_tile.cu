// Launcher of the dense row-panel tile variant of RB+RM+SR (tile.cuh), fp32 fast mode.
#include "dispatch.h"
#include "tile.cuh"

namespace daspmm {

namespace {
constexpr int kTileThreads = 128;

// Column slots per panel <= 4: the direct walk; 8..32: the staged, pipelined walk.
template <int V, int CL, int RL, int U>
void go_u(const Plan& p, const SpmmArgs<float>& a, const TileArgs& t, cudaStream_t s) {
    if constexpr (CL <= 4) {
        k_rb_sr_tile_direct<V, CL, RL, 1, kTileThreads, U><<<p.grid, kTileThreads, 0, s>>>(a, t);
    } else {
        constexpr auto k = k_rb_sr_tile<V, CL, RL, 1, kTileThreads, U>;
        // 5 CTAs of 32 KB staging per SM (96 registers) need ~70% of the array as shared
        // memory; 50 and 75 measure the same, 100 costs L1 hits (r02_carveout_probe.txt)
        static const int carve = carveout_env("DASPMM_TILE_CARVEOUT", 75);
        carveout_once<k>(carve);
        k<<<p.grid, kTileThreads, 0, s>>>(a, t);
    }
}

template <int V, int CL, int RL>
cudaError_t go(const Plan& p, const SpmmArgs<float>& a, const TileArgs& t, cudaStream_t s) {
    switch (p.tile_u) {
        case 2: go_u<V, CL, RL, 2>(p, a, t, s); break;
        case 4: go_u<V, CL, RL, 4>(p, a, t, s); break;
        case 8: go_u<V, CL, RL, 8>(p, a, t, s); break;
        default: return cudaErrorNotSupported;
    }
    return cudaGetLastError();
}

template <int V>
cudaError_t go_v(const Plan& p, const SpmmArgs<float>& a, const TileArgs& t, cudaStream_t s) {
    if (p.tile_rl == kTileRows) {
        switch (p.L) {
            case 1: return go<V, 1, kTileRows>(p, a, t, s);
            case 2: return go<V, 2, kTileRows>(p, a, t, s);
            case 4: return go<V, 4, kTileRows>(p, a, t, s);
            default: return cudaErrorNotSupported;
        }
    }
    switch (p.L) {
        case 1: return go<V, 1, 1>(p, a, t, s);
        case 2: return go<V, 2, 1>(p, a, t, s);
        case 4: return go<V, 4, 1>(p, a, t, s);
        case 8: return go<V, 8, 1>(p, a, t, s);
        case 16: return go<V, 16, 1>(p, a, t, s);
        case 32: return go<V, 32, 1>(p, a, t, s);
        default: return cudaErrorNotSupported;
    }
}
}  // namespace


cudaError_t launch_rb_sr_tile(const Plan& p, const SpmmArgs<float>& a, const int* off,
                              const int* c0, const float* val, int64_t n_pan, cudaStream_t s) {
    const TileArgs t{off, c0, val, int(n_pan)};
    switch (p.V) {
        case 1: return go_v<1>(p, a, t, s);
        case 2: return go_v<2>(p, a, t, s);
        case 4: return go_v<4>(p, a, t, s);
        default: return cudaErrorNotSupported;
    }
}

}  // namespace daspmm
