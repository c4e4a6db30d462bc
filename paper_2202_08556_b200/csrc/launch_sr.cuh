// Instantiation tables for the SR kernels (RB+SR, EB+SR). Included by one TU each.
#pragma once

#include "dispatch.h"
#include "kernels.cuh"

namespace daspmm {

// KERN is k_rb_sr or k_eb_sr.
#define DASPMM_SR_LPR_TABLE(KERN, T, CM, EXACT, V)                                      \
    switch (p.L) {                                                                     \
        case 1: DASPMM_GO((KERN<T, CM, EXACT, V, 1, 1>), p.grid, kThreads); break;     \
        case 2: DASPMM_GO((KERN<T, CM, EXACT, V, 2, 1>), p.grid, kThreads); break;     \
        case 4: DASPMM_GO((KERN<T, CM, EXACT, V, 4, 1>), p.grid, kThreads); break;     \
        case 8: DASPMM_GO((KERN<T, CM, EXACT, V, 8, 1>), p.grid, kThreads); break;     \
        case 16: DASPMM_GO((KERN<T, CM, EXACT, V, 16, 1>), p.grid, kThreads); break;   \
        case 32:                                                                       \
            if (p.X == 2) DASPMM_GO((KERN<T, CM, EXACT, V, 32, 2>), p.grid, kThreads); \
            else DASPMM_GO((KERN<T, CM, EXACT, V, 32, 1>), p.grid, kThreads);          \
            break;                                                                     \
        default: return cudaErrorNotSupported;                                         \
    }

#define DASPMM_SR_LAUNCHER(NAME, KERN)                                                  \
    template <>                                                                        \
    cudaError_t NAME<float>(const Plan& p, const SpmmArgs<float>& a, cudaStream_t s) { \
        if (p.exact) {                                                                 \
            if (p.V != 1) return cudaErrorNotSupported;                                \
            if (p.cm) { DASPMM_SR_LPR_TABLE(KERN, float, true, true, 1) }              \
            else { DASPMM_SR_LPR_TABLE(KERN, float, false, true, 1) }                  \
        } else if (p.cm) {                                                             \
            if (p.V != 1) return cudaErrorNotSupported;                                \
            DASPMM_SR_LPR_TABLE(KERN, float, true, false, 1)                           \
        } else {                                                                       \
            switch (p.V) {                                                             \
                case 1: { DASPMM_SR_LPR_TABLE(KERN, float, false, false, 1) } break;   \
                case 2: { DASPMM_SR_LPR_TABLE(KERN, float, false, false, 2) } break;   \
                case 4: { DASPMM_SR_LPR_TABLE(KERN, float, false, false, 4) } break;   \
                default: return cudaErrorNotSupported;                                 \
            }                                                                          \
        }                                                                              \
        return cudaGetLastError();                                                     \
    }                                                                                  \
    template <>                                                                        \
    cudaError_t NAME<double>(const Plan& p, const SpmmArgs<double>& a, cudaStream_t s) { \
        if (p.exact) {                                                                 \
            if (p.V != 1) return cudaErrorNotSupported;                                \
            if (p.cm) { DASPMM_SR_LPR_TABLE(KERN, double, true, true, 1) }             \
            else { DASPMM_SR_LPR_TABLE(KERN, double, false, true, 1) }                 \
        } else if (p.cm) {                                                             \
            if (p.V != 1) return cudaErrorNotSupported;                                \
            DASPMM_SR_LPR_TABLE(KERN, double, true, false, 1)                          \
        } else {                                                                       \
            switch (p.V) {                                                             \
                case 1: { DASPMM_SR_LPR_TABLE(KERN, double, false, false, 1) } break;  \
                case 2: { DASPMM_SR_LPR_TABLE(KERN, double, false, false, 2) } break;  \
                default: return cudaErrorNotSupported;                                 \
            }                                                                          \
        }                                                                              \
        return cudaGetLastError();                                                     \
    }

}  // namespace daspmm
