// Instantiation tables for the PR kernels (RB+PR, EB+PR). Included by one TU each.
#pragma once

#include "dispatch.h"
#include "kernels.cuh"

namespace daspmm {

#define DASPMM_PR_OWN(KERN, T, CM, EXACT, V, W)                                         \
    if (p.X == 2) DASPMM_GO((KERN<T, CM, EXACT, V, W, 2>), p.grid, kThreads);           \
    else DASPMM_GO((KERN<T, CM, EXACT, V, W, 1>), p.grid, kThreads);

#define DASPMM_PR_W_TABLE(KERN, T, CM, EXACT, V)                                        \
    switch (p.L) {                                                                     \
        case 2: { DASPMM_PR_OWN(KERN, T, CM, EXACT, V, 2) } break;                     \
        case 4: { DASPMM_PR_OWN(KERN, T, CM, EXACT, V, 4) } break;                     \
        case 8: { DASPMM_PR_OWN(KERN, T, CM, EXACT, V, 8) } break;                     \
        case 16: { DASPMM_PR_OWN(KERN, T, CM, EXACT, V, 16) } break;                   \
        case 32: { DASPMM_PR_OWN(KERN, T, CM, EXACT, V, 32) } break;                   \
        default: return cudaErrorNotSupported;                                         \
    }

#define DASPMM_PR_LAUNCHER(NAME, KERN)                                                  \
    template <>                                                                        \
    cudaError_t NAME<float>(const Plan& p, const SpmmArgs<float>& a, cudaStream_t s) { \
        if (p.exact) {                                                                 \
            if (p.V != 1) return cudaErrorNotSupported;                                \
            if (p.cm) { DASPMM_PR_W_TABLE(KERN, float, true, true, 1) }                \
            else { DASPMM_PR_W_TABLE(KERN, float, false, true, 1) }                    \
        } else if (p.cm) {                                                             \
            if (p.V != 1) return cudaErrorNotSupported;                                \
            DASPMM_PR_W_TABLE(KERN, float, true, false, 1)                             \
        } else {                                                                       \
            switch (p.V) {                                                             \
                case 1: { DASPMM_PR_W_TABLE(KERN, float, false, false, 1) } break;     \
                case 2: { DASPMM_PR_W_TABLE(KERN, float, false, false, 2) } break;     \
                case 4: { DASPMM_PR_W_TABLE(KERN, float, false, false, 4) } break;     \
                default: return cudaErrorNotSupported;                                 \
            }                                                                          \
        }                                                                              \
        return cudaGetLastError();                                                     \
    }                                                                                  \
    template <>                                                                        \
    cudaError_t NAME<double>(const Plan& p, const SpmmArgs<double>& a, cudaStream_t s) { \
        if (p.exact) {                                                                 \
            if (p.V != 1) return cudaErrorNotSupported;                                \
            if (p.cm) { DASPMM_PR_W_TABLE(KERN, double, true, true, 1) }               \
            else { DASPMM_PR_W_TABLE(KERN, double, false, true, 1) }                   \
        } else if (p.cm) {                                                             \
            if (p.V != 1) return cudaErrorNotSupported;                                \
            DASPMM_PR_W_TABLE(KERN, double, true, false, 1)                            \
        } else {                                                                       \
            switch (p.V) {                                                             \
                case 1: { DASPMM_PR_W_TABLE(KERN, double, false, false, 1) } break;    \
                case 2: { DASPMM_PR_W_TABLE(KERN, double, false, false, 2) } break;    \
                default: return cudaErrorNotSupported;                                 \
            }                                                                          \
        }                                                                              \
        return cudaGetLastError();                                                     \
    }

}  // namespace daspmm
