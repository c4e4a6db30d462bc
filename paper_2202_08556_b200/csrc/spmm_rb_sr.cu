// RB+SR launchers (K0 RB+RM+SR, K2 RB+CM+SR) and the B-window variant of K0.
#include <atomic>

#include "launch_sr.cuh"
namespace daspmm {
template <typename T>
cudaError_t launch_rb_sr_rows(const Plan&, const SpmmArgs<T>&, cudaStream_t);
#define launch_rb_sr launch_rb_sr_rows
DASPMM_SR_LAUNCHER(launch_rb_sr, k_rb_sr)
#undef launch_rb_sr

// Dynamic shared memory above 48 KB needs a per-device opt-in for each instantiation.
template <typename T, int V, int LPR, int CPL>
static cudaError_t win_launch(const Plan& p, const SpmmArgs<T>& a, cudaStream_t s, int bulk_b) {
    static std::atomic<uint64_t> done{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = uint64_t(1) << (dev & 63);
    if (!(done.load() & bit)) {
        cudaError_t e = cudaFuncSetAttribute(k_rb_sr_win<T, V, LPR, CPL>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(kWinSmemMax));
        if (e != cudaSuccess) return e;
        done.fetch_or(bit);
    }
    k_rb_sr_win<T, V, LPR, CPL><<<p.grid, kThreads, p.win_smem, s>>>(a, bulk_b);
    return cudaGetLastError();
}

#define DASPMM_WIN_LPR_TABLE(V)                                                       \
    switch (p.L) {                                                                   \
        case 1: return win_launch<float, V, 1, 1>(p, a, s, bulk_b);                  \
        case 2: return win_launch<float, V, 2, 1>(p, a, s, bulk_b);                  \
        case 4: return win_launch<float, V, 4, 1>(p, a, s, bulk_b);                  \
        case 8: return win_launch<float, V, 8, 1>(p, a, s, bulk_b);                  \
        case 16: return win_launch<float, V, 16, 1>(p, a, s, bulk_b);                \
        case 32:                                                                     \
            if (p.X == 2) return win_launch<float, V, 32, 2>(p, a, s, bulk_b);       \
            return win_launch<float, V, 32, 1>(p, a, s, bulk_b);                     \
        default: return cudaErrorNotSupported;                                       \
    }

static cudaError_t launch_rb_sr_win(const Plan& p, const SpmmArgs<float>& a, cudaStream_t s) {
    const int bulk_b = (reinterpret_cast<uintptr_t>(a.B) & 15) == 0 ? 1 : 0;
    switch (p.V) {
        case 1: DASPMM_WIN_LPR_TABLE(1)
        case 2: DASPMM_WIN_LPR_TABLE(2)
        case 4: DASPMM_WIN_LPR_TABLE(4)
        default: return cudaErrorNotSupported;
    }
}

// Replicated row epilogue (fp32 fast mode, row-major B): the k_rb_sr table with
// MODE = kRBRepl.
#define DASPMM_REPL_LPR_TABLE(V)                                                       \
    switch (p.L) {                                                                    \
        case 1: k_rb_sr<float, false, false, V, 1, 1, kRBRepl><<<p.grid, kThreads, 0, s>>>(a); break; \
        case 2: k_rb_sr<float, false, false, V, 2, 1, kRBRepl><<<p.grid, kThreads, 0, s>>>(a); break; \
        case 4: k_rb_sr<float, false, false, V, 4, 1, kRBRepl><<<p.grid, kThreads, 0, s>>>(a); break; \
        case 8: k_rb_sr<float, false, false, V, 8, 1, kRBRepl><<<p.grid, kThreads, 0, s>>>(a); break; \
        case 16: k_rb_sr<float, false, false, V, 16, 1, kRBRepl><<<p.grid, kThreads, 0, s>>>(a); break; \
        case 32:                                                                      \
            if (p.X == 2) k_rb_sr<float, false, false, V, 32, 2, kRBRepl><<<p.grid, kThreads, 0, s>>>(a); \
            else k_rb_sr<float, false, false, V, 32, 1, kRBRepl><<<p.grid, kThreads, 0, s>>>(a); \
            break;                                                                    \
        default: return cudaErrorNotSupported;                                        \
    }

static cudaError_t launch_rb_sr_repl(const Plan& p, const SpmmArgs<float>& a, cudaStream_t s) {
    if (p.cm || p.exact) return cudaErrorNotSupported;
    switch (p.V) {
        case 1: { DASPMM_REPL_LPR_TABLE(1) } break;
        case 2: { DASPMM_REPL_LPR_TABLE(2) } break;
        case 4: { DASPMM_REPL_LPR_TABLE(4) } break;
        default: return cudaErrorNotSupported;
    }
    return cudaGetLastError();
}

// Fast f32 row-major RB+SR in smaller CTAs (Plan::rb_threads; tuning).
#define DASPMM_RB_NT_TABLE(V, NT)                                                        \
    switch (p.L) {                                                                      \
        case 1: k_rb_sr<float, false, false, V, 1, 1, kRB, NT><<<p.grid, NT, 0, s>>>(a); break; \
        case 2: k_rb_sr<float, false, false, V, 2, 1, kRB, NT><<<p.grid, NT, 0, s>>>(a); break; \
        case 4: k_rb_sr<float, false, false, V, 4, 1, kRB, NT><<<p.grid, NT, 0, s>>>(a); break; \
        case 8: k_rb_sr<float, false, false, V, 8, 1, kRB, NT><<<p.grid, NT, 0, s>>>(a); break; \
        case 16: k_rb_sr<float, false, false, V, 16, 1, kRB, NT><<<p.grid, NT, 0, s>>>(a); break; \
        case 32:                                                                        \
            if (p.X == 2) k_rb_sr<float, false, false, V, 32, 2, kRB, NT><<<p.grid, NT, 0, s>>>(a); \
            else k_rb_sr<float, false, false, V, 32, 1, kRB, NT><<<p.grid, NT, 0, s>>>(a); \
            break;                                                                      \
        default: return cudaErrorNotSupported;                                          \
    }

template <int NT>
static cudaError_t launch_rb_sr_nt(const Plan& p, const SpmmArgs<float>& a, cudaStream_t s) {
    switch (p.V) {
        case 1: { DASPMM_RB_NT_TABLE(1, NT) } break;
        case 2: { DASPMM_RB_NT_TABLE(2, NT) } break;
        case 4: { DASPMM_RB_NT_TABLE(4, NT) } break;
        default: return cudaErrorNotSupported;
    }
    return cudaGetLastError();
}

template <>
cudaError_t launch_rb_sr<float>(const Plan& p, const SpmmArgs<float>& a, cudaStream_t s) {
    if (p.repl) return launch_rb_sr_repl(p, a, s);
    if (p.rb_threads != kThreads && !p.cm && !p.exact && p.win_rows == 0) {
        if (p.rb_threads == 64) return launch_rb_sr_nt<64>(p, a, s);
        if (p.rb_threads == 128) return launch_rb_sr_nt<128>(p, a, s);
    }
    if (p.win_rows > 0 && !p.cm && !p.exact) return launch_rb_sr_win(p, a, s);
    return launch_rb_sr_rows<float>(p, a, s);
}
template <>
cudaError_t launch_rb_sr<double>(const Plan& p, const SpmmArgs<double>& a, cudaStream_t s) {
    return launch_rb_sr_rows<double>(p, a, s);
}
}  // namespace daspmm
