// daspmm — device building blocks shared by the eight DA-SpMM kernels (sm_100a).
//
// Arithmetic modes
//   fast  : fmaf / fma — one rounding per multiply-add (more accurate than the
//           reference, tolerance parity).
//   exact : __fmul_rn then __fadd_rn — no contraction, the reference's evaluation
//           order (spmm.hpp:85-88, 95-102, 149-157, 168-181), so results are
//           bit-identical to the reference's CPU kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace daspmm {

constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------------ vectors
template <typename T, int V> struct VecT;
template <> struct VecT<float, 1> { using type = float; };
template <> struct VecT<float, 2> { using type = float2; };
template <> struct VecT<float, 4> { using type = float4; };
template <> struct VecT<double, 1> { using type = double; };
template <> struct VecT<double, 2> { using type = double2; };

template <typename T, int V>
struct Frag {
    T v[V];
};

// Optional L2 policy for B gathers (-DDASPMM_L2_HINT): mark B lines evict-last.
// Measured on B200 (profiles/r01_notes.md): no gain over the default policy with A and
// C already streaming evict-first, so it is off by default.
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

// 128/64/32-bit vector gather of V consecutive elements of B (read-only path).
template <typename T, int V>
__device__ __forceinline__ Frag<T, V> ld_frag(const T* __restrict__ p) {
    Frag<T, V> f;
#ifndef DASPMM_L2_HINT
    if constexpr (V == 1) {
        f.v[0] = __ldg(p);
    } else {
        using VT = typename VecT<T, V>::type;
        const VT t = __ldg(reinterpret_cast<const VT*>(p));
        *reinterpret_cast<VT*>(f.v) = t;
    }
#else
    const uint64_t pol = policy_evict_last();
    if constexpr (sizeof(T) == 4 && V == 4) {
        asm("ld.global.nc.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=f"(f.v[0]), "=f"(f.v[1]), "=f"(f.v[2]), "=f"(f.v[3])
                     : "l"(p), "l"(pol));
    } else if constexpr (sizeof(T) == 4 && V == 2) {
        asm("ld.global.nc.L2::cache_hint.v2.f32 {%0,%1}, [%2], %3;"
                     : "=f"(f.v[0]), "=f"(f.v[1]) : "l"(p), "l"(pol));
    } else if constexpr (sizeof(T) == 4 && V == 1) {
        asm("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;"
                     : "=f"(f.v[0]) : "l"(p), "l"(pol));
    } else if constexpr (sizeof(T) == 8 && V == 2) {
        asm("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
                     : "=d"(f.v[0]), "=d"(f.v[1]) : "l"(p), "l"(pol));
    } else {
        asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;"
                     : "=d"(f.v[0]) : "l"(p), "l"(pol));
    }
#endif
    return f;
}

// V consecutive elements from shared memory (the staged B window). Plain C++ loads: the
// pointer derives from the kernel's shared array, so ptxas emits LDS (checked in SASS).
template <typename T, int V>
__device__ __forceinline__ Frag<T, V> ld_frag_shared(const T* p) {
    Frag<T, V> f;
    if constexpr (V == 1) {
        f.v[0] = *p;
    } else {
        using VT = typename VecT<T, V>::type;
        *reinterpret_cast<VT*>(f.v) = *reinterpret_cast<const VT*>(p);
    }
    return f;
}

template <typename T, int V>
__device__ __forceinline__ void st_frag_shared(T* p, const Frag<T, V>& f) {
    if constexpr (V == 1) {
        *p = f.v[0];
    } else {
        using VT = typename VecT<T, V>::type;
        *reinterpret_cast<VT*>(p) = *reinterpret_cast<const VT*>(f.v);
    }
}

// Column-major B: V columns at stride ldb, scalar loads.
template <typename T, int V>
__device__ __forceinline__ Frag<T, V> ld_frag_cm(const T* __restrict__ p, int64_t ldb) {
    Frag<T, V> f;
#pragma unroll
    for (int i = 0; i < V; ++i) f.v[i] = __ldg(p + i * ldb);
    return f;
}

// C is written once and never re-read by the kernel: streaming store.
template <typename T, int V>
__device__ __forceinline__ void st_frag(T* p, const Frag<T, V>& f) {
    if constexpr (V == 1) {
        __stcs(p, f.v[0]);
    } else {
        using VT = typename VecT<T, V>::type;
        __stcs(reinterpret_cast<VT*>(p), *reinterpret_cast<const VT*>(f.v));
    }
}

template <typename T, int V>
__device__ __forceinline__ Frag<T, V> ld_frag_rw(const T* p) {
    Frag<T, V> f;
    if constexpr (V == 1) {
        f.v[0] = *p;
    } else {
        using VT = typename VecT<T, V>::type;
        *reinterpret_cast<VT*>(f.v) = *reinterpret_cast<const VT*>(p);
    }
    return f;
}

template <typename T, int V>
__device__ __forceinline__ void st_frag_rw(T* p, const Frag<T, V>& f) {
    if constexpr (V == 1) {
        *p = f.v[0];
    } else {
        using VT = typename VecT<T, V>::type;
        *reinterpret_cast<VT*>(p) = *reinterpret_cast<const VT*>(f.v);
    }
}

// Split-row deposit (EB): vector atomics exist for float2/float4 on sm_90+.
template <typename T, int V>
__device__ __forceinline__ void atomic_add_frag(T* p, const Frag<T, V>& f) {
    if constexpr (sizeof(T) == 4 && V == 4) {
        atomicAdd(reinterpret_cast<float4*>(p), *reinterpret_cast<const float4*>(f.v));
    } else if constexpr (sizeof(T) == 4 && V == 2) {
        atomicAdd(reinterpret_cast<float2*>(p), *reinterpret_cast<const float2*>(f.v));
    } else {
#pragma unroll
        for (int i = 0; i < V; ++i) atomicAdd(p + i, f.v[i]);
    }
}

// A is streamed exactly once per column tile: evict-first loads.
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) {
    return __ldcs(p);
}

// ------------------------------------------------------------------ programmatic dependent launch
// The EB prologue (k_eb_prep*) zeroes the rows the EB kernel later deposits into with
// atomics. The EB kernel is launched with programmatic stream serialization, so its CTAs
// start (and load A and gather B) while the prologue still runs; it waits for the
// prologue only before its first atomic deposit (and once more before exiting, so the
// call as a whole still completes after the prologue). Without the launch attribute the
// wait returns immediately.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ------------------------------------------------------------------ arithmetic
template <bool EXACT>
__device__ __forceinline__ float madd(float acc, float a, float b) {
    if constexpr (EXACT) return __fadd_rn(acc, __fmul_rn(a, b));
    else return fmaf(a, b, acc);
}
template <bool EXACT>
__device__ __forceinline__ double madd(double acc, double a, double b) {
    if constexpr (EXACT) return __dadd_rn(acc, __dmul_rn(a, b));
    else return fma(a, b, acc);
}
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// ------------------------------------------------------------------ groups
// A "group" is G consecutive lanes of a warp (G a power of two <= 32). Shuffles
// carry the group's own mask so sibling groups may diverge freely.
template <int G>
__device__ __forceinline__ unsigned group_mask() {
    if constexpr (G == 32) return kFull;
    else return ((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1));
}

template <int G, typename T>
__device__ __forceinline__ T gshfl(unsigned mask, T v, int src) {
    if constexpr (G == 1) return v;  // a one-lane group owns its value
    else return __shfl_sync(mask, v, src, G);
}

// Adjacent-pair merge tree over the G lanes of a group — reduce.hpp:18-25.
// XOR butterfly: at level `off` lane i adds lane i^off; the lower half of each
// 2*off block computes (lo + hi), the upper half (hi + lo), identical under IEEE
// commutativity, so every lane ends with exactly the reference's tree value.
template <int G, typename T>
__device__ __forceinline__ T group_tree_sum(unsigned mask, T v) {
#pragma unroll
    for (int off = 1; off < G; off <<= 1) v = add_rn(v, __shfl_xor_sync(mask, v, off, G));
    return v;
}

// Gated suffix scan — reduce.hpp:31-39. For d = 1, 2, 4, ...: lane i absorbs lane
// i+d when both carry the same segment id and i+d < G. Reads of lane i+d see its
// pre-step value, matching the reference's ascending in-place loop. After the
// scan, the first lane of each segment holds the segment total.
template <int G, typename T>
__device__ __forceinline__ T group_conditional_scan(unsigned mask, T v, int id, int gl) {
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
        const T o = __shfl_down_sync(mask, v, d, G);
        const int oid = __shfl_down_sync(mask, id, d, G);
        if (gl + d < G && oid == id) v = add_rn(v, o);
    }
    return v;
}

// Precomputed gates for the scan (ids are shared by all column slots of a tile).
template <int G>
__device__ __forceinline__ unsigned scan_gates(unsigned mask, int id, int gl) {
    unsigned gates = 0;
    int bit = 0;
#pragma unroll
    for (int d = 1; d < G; d <<= 1, ++bit) {
        const int oid = __shfl_down_sync(mask, id, d, G);
        if (gl + d < G && oid == id) gates |= 1u << bit;
    }
    return gates;
}

template <int G, typename T>
__device__ __forceinline__ T group_conditional_scan_gated(unsigned mask, T v, unsigned gates) {
    int bit = 0;
#pragma unroll
    for (int d = 1; d < G; d <<= 1, ++bit) {
        const T o = __shfl_down_sync(mask, v, d, G);
        if (gates & (1u << bit)) v = add_rn(v, o);
    }
    return v;
}

// ------------------------------------------------------------------ TMA (bulk copy)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D TMA: global -> shared, `bytes` a multiple of 16, both addresses 16-B aligned;
// completion is signalled on `bar` (complete_tx).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

// upper_bound(rp[lo, hi), e) - 1 over int32 offsets: the row holding element e
// (partition.hpp:27-30).
__device__ __forceinline__ int row_of_element(const int* __restrict__ rp, int M, int e) {
    int lo = 0, hi = M + 1;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(rp + mid) <= e) lo = mid + 1;
        else hi = mid;
    }
    return lo - 1;
}

// Chunk bounds of partition_elements (partition.hpp:45-64): sizes ceil/floor of
// nnz/P, larger chunks first.
__device__ __forceinline__ void chunk_bounds(int64_t nnz, int64_t P, int64_t w, int64_t& b,
                                             int64_t& e) {
    const int64_t base = nnz / P, extra = nnz % P;
    b = w * base + (w < extra ? w : extra);
    e = b + base + (w < extra ? 1 : 0);
}

}  // namespace daspmm
