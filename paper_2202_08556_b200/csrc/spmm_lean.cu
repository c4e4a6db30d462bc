// Launchers of the lean SR kernels (lean.cuh): RB+RM+SR and EB+RM+SR, fp32 fast mode.
#define DASPMM_PDL_EXPR (p.pdl && p.kernel >= 4)
#include "dispatch.h"
#include "lean.cuh"

namespace daspmm {

#define DASPMM_LEAN_LPR_NT(KERN, V, NT)                                               \
    switch (p.L) {                                                                   \
        case 1: DASPMM_GO((KERN<V, 1, NT>), p.grid, NT); break;                      \
        case 2: DASPMM_GO((KERN<V, 2, NT>), p.grid, NT); break;                      \
        case 4: DASPMM_GO((KERN<V, 4, NT>), p.grid, NT); break;                      \
        case 8: DASPMM_GO((KERN<V, 8, NT>), p.grid, NT); break;                      \
        case 16: DASPMM_GO((KERN<V, 16, NT>), p.grid, NT); break;                    \
        case 32: DASPMM_GO((KERN<V, 32, NT>), p.grid, NT); break;                    \
        default: return cudaErrorNotSupported;                                       \
    }
#define DASPMM_LEAN_LPR(KERN, V)                                                      \
    if (p.lean_threads == 64) { DASPMM_LEAN_LPR_NT(KERN, V, 64) }                    \
    else if (p.lean_threads == 128) { DASPMM_LEAN_LPR_NT(KERN, V, 128) }             \
    else { DASPMM_LEAN_LPR_NT(KERN, V, kThreads) }

#define DASPMM_LEAN_V(KERN)                                                           \
    switch (p.V) {                                                                   \
        case 1: { DASPMM_LEAN_LPR(KERN, 1) } break;                                  \
        case 2: { DASPMM_LEAN_LPR(KERN, 2) } break;                                  \
        case 4: { DASPMM_LEAN_LPR(KERN, 4) } break;                                  \
        default: return cudaErrorNotSupported;                                       \
    }

cudaError_t launch_sr_lean(const Plan& p, const SpmmArgs<float>& a, cudaStream_t s) {
    if (p.kernel >= 4 && p.lean_rw) {
        DASPMM_LEAN_V(k_eb_sr_lean_rw)
    } else if (p.kernel >= 4) {
        DASPMM_LEAN_V(k_eb_sr_lean)
    } else {
        DASPMM_LEAN_V(k_rb_sr_lean)
    }
    return cudaGetLastError();
}

}  // namespace daspmm
