// daspmm — the eight DA-SpMM kernels (2 x 2 x 2 design space, §3) as
// hand-written sm_100a CUDA. Each kernel restates one reference worker body
// (proj/include/spmmkit/spmm.hpp:40-187) for the GPU execution model:
//
//   M-loop  RB : a lane group owns a row (spmm.hpp:66-107)
//           EB : a lane group owns an equal-nnz chunk, partition.hpp:45-64 bounds
//                (spmm.hpp:108-186); split rows take atomics, owned rows plain stores
//   N-loop  RM : B row-major, V-wide vector gathers (Technique 2)
//           CM : B column-major, scalar gathers at stride ldb
//   K-loop  SR : lanes span columns, each lane accumulates its columns sequentially
//                in nnz order (spmm.hpp:85-88, 145-159)
//           PR : lanes span nonzeros; W-lane adjacent-pair tree (RB, reduce.hpp:18-25)
//                or gated conditional scan (EB, Technique 4, reduce.hpp:31-39)
//
// Coalesced row caching (CRC / Technique 3): A's (col, val) pairs are loaded once per
// step with coalesced per-lane loads and broadcast through register shuffles, so
// every B gather of a step reuses them across all columns the group owns.
//
// Launch shape: 256-thread CTAs; groups of LPR (SR) or W (PR) lanes; blockIdx.y
// walks column tiles. Element offsets are int32 (nnz < 2^31).
#pragma once

#include <climits>

#include "common.cuh"

namespace daspmm {

constexpr int kMaxExtraDst = 7;  // + the primary C: up to 8 ranks on one NVSwitch box

template <typename T>
struct SpmmArgs {
    const int* __restrict__ rp;  // M+1 row offsets
    const int* __restrict__ ci;  // nnz column indices
    const T* __restrict__ va;    // nnz values
    const T* __restrict__ B;     // K x N, RM (ldb >= N) or CM (ldb >= K)
    T* C;                        // M x N row-major, ldc >= N
    int M, K, N;
    int64_t nnz, ldb, ldc;
    int64_t P;                   // EB workers (chunks)
    int seg;                     // exact-mode EB+SR staging segment, max(W, 256)
    int64_t rpg;                 // RB: rows per group (row-block size)
    int64_t sub;                 // EB fast path: pairs per group sub-chunk
    int bulk_ok;                 // A arrays 16-B aligned: CTA tiles may be staged by TMA
    const int* __restrict__ chunk_row;  // EB: row holding each chunk's first element
    const int* __restrict__ rows;       // EB: COO row id of every nonzero (handle-owned)
    const int2* __restrict__ spans;     // RB window kernel: column window per 32-row panel
    int win_rows;                       // RB window kernel: rows per CTA panel (32 << i)
    // RB+SR replicated epilogue (k_rb_sr<..., kRBRepl>, daspmm_spmm_rows_to): every
    // finished row is also stored to extra[0 .. n_extra) (same ldc) — e.g. the peers'
    // copies of the assembled C mapped over NVLink, so a row-panel SpMM and its
    // all-gather are one kernel.
    int n_extra;
    T* extra[kMaxExtraDst];
};

constexpr int kThreads = 256;

template <typename T, bool CM, int V>
__device__ __forceinline__ Frag<T, V> gather(const SpmmArgs<T>& a, int k, int col) {
    if constexpr (CM) return ld_frag_cm<T, V>(a.B + int64_t(col) * a.ldb + k, a.ldb);
    else return ld_frag<T, V>(a.B + int64_t(k) * a.ldb + col);
}

// =============================================================== SR walker (K0/K2/K4/K6)
// One lane group of LPR lanes walks a contiguous nonzero range [e0, e1) in order,
// lane gl owning columns n0 + s*LPR*V + [0, V), s < CPL. Per step it holds STEP
// (col, val) pairs in registers (coalesced loads, Technique 3 / CRC) and broadcasts
// them by shuffle; the NEXT step's pairs are loaded before this step's B gathers are
// issued, so A's load latency overlaps the gathers instead of preceding them.
// Accumulation per column is sequential in nnz order (spmm.hpp:85-88, 145-159).
//
//   RB (K0/K2): the range is exactly the rows [r, r_end) of a row block — every row
//               is owned, stored once; empty rows receive zeros.
//   EB (K4/K6): the range is partition chunk w; rows cut by the range ends are split
//               and take atomics (pre-zeroed by k_eb_prep); empty rows pre-zeroed.
//               Exact mode restarts the run at the reference's staging boundaries
//               (seg_cap = max(W, 256), spmm.hpp:50, 136) and adds the partials in
//               the reference's order.
// Boundary partials of one CTA (EB fast path): slot b holds the pieces of the row
// that crosses sub-chunk boundary b — L[b] from the group before it, R[b] from the
// group after it.
template <typename T>
struct CtaSlots {
    T* L = nullptr;      // [(G+1) * TN]
    T* R = nullptr;      // [(G+1) * TN]
    int* row = nullptr;  // [G+1], -1 when no row crosses the boundary
    int g = 0;           // this group's index in the CTA
    int tile0 = 0;       // first column of the CTA's column tile
    int tn = 0;          // tile width
};

enum WalkMode { kRB = 0, kEB = 1, kEBCta = 2, kRBWin = 3, kRBRepl = 4 };

// RB window kernel: the CTA's B rows [c0, c0 + span) staged in shared memory, `pitch`
// elements per row starting at column tile0.
template <typename T>
struct WinSlots {
    const T* s = nullptr;
    int c0 = 0;
    int pitch = 0;
    int tile0 = 0;
};

template <typename T, bool CM, bool EXACT, int V, int LPR, int CPL, int MODE>
__device__ __forceinline__ void sr_walk(const SpmmArgs<T>& a, const int e0, const int e1, int r,
                                        const int nrows, const int n0, const unsigned mask,
                                        const int gl, const CtaSlots<T> slots = CtaSlots<T>{},
                                        const WinSlots<T> win = WinSlots<T>{}) {
    constexpr bool EB = MODE == kEB || MODE == kEBCta;
    constexpr int STEP = LPR >= 16 ? LPR : (LPR >= 4 ? 16 : 8);  // pairs per group per step
    constexpr int EPL = STEP / LPR;                              // pairs per lane per step
    // Double-buffered A pairs pay off once a lane holds few of them (LPR >= 4); narrow
    // groups rely on occupancy instead and keep the registers for gathers.
    constexpr bool PREFETCH = LPR >= 4;
    constexpr int WORDS = V * CPL * int(sizeof(T)) / 4;  // accumulator registers per lane
    constexpr int BATCH0 = WORDS >= 8 ? 2 : (WORDS >= 4 ? 4 : 8);
    constexpr int BATCH = BATCH0 < STEP ? BATCH0 : STEP;  // gathers in flight per lane
    Frag<T, V> acc[CPL], ydep[CPL];
#pragma unroll
    for (int s = 0; s < CPL; ++s)
#pragma unroll
        for (int i = 0; i < V; ++i) acc[s].v[i] = ydep[s].v[i] = T(0);
    int next_seg = e0 + a.seg;

    // Row bookkeeping without dependent loads.
    //   RB: the block's nrows (<= LPR) row ends, one per lane, fetched once.
    //   EB: per-pair row ids from the handle's COO array; a row is split only if it is
    //       the range's first row and began before e0, or its last row and continues
    //       past e1.
    const int r0 = r;
    int wend = 0, rend = 0;
    int first_row = 0, last_row = 0;
    bool first_split = false, last_split = false;
    if constexpr (!EB) {
        wend = gl < nrows ? __ldg(a.rp + r0 + 1 + gl) : INT_MAX;
        rend = gshfl<LPR>(mask, wend, 0);
    } else {
        first_row = r;
        last_row = __ldg(a.rows + e1 - 1);
        first_split = e0 > 0 && __ldg(a.rows + e0 - 1) == first_row;
        last_split = e1 < a.nnz && __ldg(a.rows + e1) == last_row;
    }

    auto flush = [&]() {  // row r is complete within this range
        const bool head = EB && first_split && r == first_row;
        const bool tail = EB && last_split && r == last_row;
        const bool owned = !head && !tail;
#pragma unroll
        for (int s = 0; s < CPL; ++s) {
            Frag<T, V> out;
#pragma unroll
            for (int i = 0; i < V; ++i) {
                out.v[i] = (EB && EXACT) ? add_rn(ydep[s].v[i], acc[s].v[i]) : acc[s].v[i];
                acc[s].v[i] = ydep[s].v[i] = T(0);
            }
            const int col = n0 + s * LPR * V;
            if constexpr (MODE == kEBCta) {
                if (!owned) {  // boundary piece -> shared slot, combined by the CTA
                    const int b = head ? slots.g : slots.g + 1;
                    T* dst = (head ? slots.R : slots.L) + b * slots.tn + (col - slots.tile0);
#pragma unroll
                    for (int i = 0; i < V; ++i) dst[i] = out.v[i];
                    if (s == 0 && gl == 0) slots.row[b] = r;
                    continue;
                }
            }
            if (col < a.N) {
                const int64_t off = int64_t(r) * a.ldc + col;
                if (owned) {
                    st_frag(a.C + off, out);
                } else {
                    griddep_wait();  // split row: zeroed by the EB prologue
                    atomic_add_frag(a.C + off, out);
                }
                if constexpr (MODE == kRBRepl) {  // replicated epilogue (daspmm_spmm_rows_to)
                    for (int d = 0; d < a.n_extra; ++d) st_frag(a.extra[d] + off, out);
                }
            }
        }
    };

    // Row-major gathers: per-slot byte base &B[0][col] and a 32-bit row pitch in bytes,
    // so each gather address is one IMAD.WIDE (ldb * sizeof(T) < 2^31, plan_spmm).
    // Lanes past N gather column 0 instead (always in bounds, never stored), so the
    // gathers need no predicate — predicated vector loads cost a register copy each.
    const char* Bcol[CPL];
#pragma unroll
    for (int s = 0; s < CPL; ++s) {
        const int col = n0 + s * LPR * V;
        Bcol[s] = reinterpret_cast<const char*>(a.B + (col < a.N ? col : 0));
    }
    const int ldb_bytes = int(a.ldb) * int(sizeof(T));
    int c[EPL], rr[EB ? EPL : 1];
    T v[EPL];
    auto load_step = [&](int j, int* cc, T* vvv, int* rrr) {
#pragma unroll
        for (int q = 0; q < EPL; ++q) {
            const int e = j + q * LPR + gl;
            const bool ok = e < e1;
            cc[q] = ok ? ld_stream(a.ci + e) : 0;
            vvv[q] = ok ? ld_stream(a.va + e) : T(0);
            if constexpr (EB) rrr[q] = ok ? ld_stream(a.rows + e) : INT_MAX;
        }
    };
    if constexpr (PREFETCH) load_step(e0, c, v, rr);
    for (int j = e0; j < e1; j += STEP) {
        int cn[PREFETCH ? EPL : 1], rn[(PREFETCH && EB) ? EPL : 1];
        T vn[PREFETCH ? EPL : 1];
        if constexpr (PREFETCH) load_step(j + STEP, cn, vn, rn);  // next step in flight
        else load_step(j, c, v, rr);
        const int cnt = min(STEP, e1 - j);
#pragma unroll
        for (int x0 = 0; x0 < STEP; x0 += BATCH) {
            if (x0 < cnt) {  // group-uniform
                const int nb = min(BATCH, cnt - x0);
                T vv[BATCH];
                int rid[EB ? BATCH : 1];
                Frag<T, V> b[BATCH][CPL];
#pragma unroll
                for (int u = 0; u < BATCH; ++u) {
                    const int x = x0 + u;
                    const int ct = gshfl<LPR>(mask, c[x / LPR], x % LPR);
                    vv[u] = gshfl<LPR>(mask, v[x / LPR], x % LPR);
                    if constexpr (EB) rid[u] = gshfl<LPR>(mask, rr[x / LPR], x % LPR);
                    // padded tail entries gather row 0 of B harmlessly and are never summed
#pragma unroll
                    for (int s = 0; s < CPL; ++s) {
                        const int col = n0 + s * LPR * V;
                        if constexpr (MODE == kRBWin) {
                            const int k = u < nb ? ct - win.c0 : 0;
                            if (col < a.N)
                                b[u][s] = ld_frag_shared<T, V>(win.s + int64_t(k) * win.pitch +
                                                               (col - win.tile0));
                        } else if constexpr (CM) {
                            if (col < a.N) b[u][s] = gather<T, CM, V>(a, u < nb ? ct : 0, col);
                        } else {
                            (void)col;
                            b[u][s] = ld_frag<T, V>(reinterpret_cast<const T*>(
                                Bcol[s] + int64_t(u < nb ? ct : 0) * ldb_bytes));
                        }
                    }
                }
                const int ef = j + x0;
                const bool seg_in_batch = EB && EXACT && next_seg >= ef && next_seg < ef + nb;
                bool same_row;
                if constexpr (EB) same_row = nb == BATCH && rid[BATCH - 1] == r;
                else same_row = nb == BATCH && ef + BATCH <= rend;
                if (same_row && !seg_in_batch) {
                    // fast path: the whole batch continues the current row
#pragma unroll
                    for (int u = 0; u < BATCH; ++u)
#pragma unroll
                        for (int s = 0; s < CPL; ++s)
#pragma unroll
                            for (int i = 0; i < V; ++i)
                                acc[s].v[i] = madd<EXACT>(acc[s].v[i], vv[u], b[u][s].v[i]);
                } else {
#pragma unroll
                    for (int u = 0; u < BATCH; ++u) {
                        if (u < nb) {
                            const int e = ef + u;
                            if constexpr (EB) {
                                if (rid[u] != r) {  // row change (empty rows pre-zeroed)
                                    flush();
                                    r = rid[u];
                                }
                            } else {
                                while (e >= rend) {  // row change; empty rows get zeros
                                    flush();
                                    ++r;
                                    rend = gshfl<LPR>(mask, wend, r - r0);
                                }
                            }
                            if constexpr (EB && EXACT) {
                                if (e == next_seg) {  // reference staging boundary
#pragma unroll
                                    for (int s = 0; s < CPL; ++s)
#pragma unroll
                                        for (int i = 0; i < V; ++i) {
                                            ydep[s].v[i] = add_rn(ydep[s].v[i], acc[s].v[i]);
                                            acc[s].v[i] = T(0);
                                        }
                                    next_seg += a.seg;
                                }
                            }
#pragma unroll
                            for (int s = 0; s < CPL; ++s)
#pragma unroll
                                for (int i = 0; i < V; ++i)
                                    acc[s].v[i] = madd<EXACT>(acc[s].v[i], vv[u], b[u][s].v[i]);
                        }
                    }
                }
            }
        }
        if constexpr (PREFETCH) {
#pragma unroll
            for (int q = 0; q < EPL; ++q) {
                c[q] = cn[q];
                v[q] = vn[q];
                if constexpr (EB) rr[q] = rn[q];
            }
        }
    }
    if (EB && e0 >= e1) return;
    flush();
    if constexpr (!EB) {  // trailing empty rows of the block
        for (++r; r < r0 + nrows; ++r) flush();
    }
}

// RB + SR: group g owns rows [g*rpg, (g+1)*rpg) — a row block (rpg <= LPR).
// MODE kRBRepl adds the replicated row epilogue (a separate instantiation, so the
// common path carries none of it).
// Resident CTAs per SM (measured, profiles/r01c_minblocks_probe.txt): 5 for groups of
// >= 16 lanes (48 registers; uniform s20 N = 128 1229 -> 1210 us), 4 below (5 costs
// N = 16 184 -> 221 us), 3 for narrow groups and fp64.
template <typename T, bool CM, bool EXACT, int V, int LPR, int CPL, int MODE = kRB, int NT = kThreads>
__global__ void __launch_bounds__(NT, ((sizeof(T) == 8 || LPR <= 2) ? 3 : (LPR >= 16 ? 5 : 4)) * (kThreads / NT))
k_rb_sr(const SpmmArgs<T> a) {
    constexpr int TN = LPR * V * CPL;
    const unsigned mask = group_mask<LPR>();
    const int gl = threadIdx.x & (LPR - 1);
    const int64_t g = (int64_t(blockIdx.x) * NT + threadIdx.x) / LPR;
    const int64_t r0 = g * a.rpg;
    if (r0 >= a.M) return;  // whole group leaves together
    const int r1 = int(min(int64_t(a.M), r0 + a.rpg));
    const int n0 = blockIdx.y * TN + gl * V;
    sr_walk<T, CM, EXACT, V, LPR, CPL, MODE>(a, __ldg(a.rp + r0), __ldg(a.rp + r1), int(r0),
                                             r1 - int(r0), n0, mask, gl);
}

// RB + SR with the B window in shared memory (row-local matrices: banded, meshes).
// A CTA owns a panel of win_rows rows. The union of the panel's column indices is a
// window [c0, c1] (precomputed per 32-row fine panel at handle creation); the CTA stages
// B rows c0..c1 of its column tile into shared memory once — one 1-D TMA bulk copy when
// the rows are contiguous (whole-row tile, ldb == N), cooperative vector loads otherwise
// — and every gather of the walk is a shared-memory load. B then crosses L2 about once
// per panel instead of once per nonzero, so the call streams at HBM rate.
// Groups take the panel's row blocks round-robin; rows, order and arithmetic are those
// of k_rb_sr (spmm.hpp:66-88).
template <typename T, int V, int LPR, int CPL>
__global__ void __launch_bounds__(kThreads, 3) k_rb_sr_win(const SpmmArgs<T> a, int bulk_b) {
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ uint64_t bar;
    __shared__ int s_win[2];
    constexpr int TN = LPR * V * CPL;
    constexpr int G = kThreads / LPR;
    const int64_t R0 = int64_t(blockIdx.x) * a.win_rows;
    const int r_end = int(min(int64_t(a.M), R0 + a.win_rows));
    if (threadIdx.x < 32) {  // the panel's window from its fine panels
        const int64_t f0 = R0 / 32, f1 = (int64_t(r_end) + 31) / 32;
        int lo = INT_MAX, hi = -1;
        for (int64_t f = f0 + threadIdx.x; f < f1; f += 32) {
            const int2 w = __ldg(a.spans + f);
            lo = min(lo, w.x);
            hi = max(hi, w.y);
        }
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(kFull, lo, o));
            hi = max(hi, __shfl_xor_sync(kFull, hi, o));
        }
        if (threadIdx.x == 0) {
            s_win[0] = lo;
            s_win[1] = hi;
            mbar_init(&bar, 1);
        }
    }
    __syncthreads();
    const int c0 = s_win[0], c1 = s_win[1];
    const int tile0 = blockIdx.y * TN;
    const int pitch = min(a.N - tile0, TN);
    T* sB = reinterpret_cast<T*>(dsm);
    if (c1 >= c0) {
        const int64_t span = int64_t(c1) - c0 + 1;
        if (bulk_b && gridDim.y == 1 && pitch == a.N && a.ldb == a.N) {
            // contiguous rows: one bulk copy from the 16-B aligned address below B[c0]
            const unsigned char* src = reinterpret_cast<const unsigned char*>(a.B + int64_t(c0) * a.N);
            const unsigned lead = unsigned(reinterpret_cast<uintptr_t>(src) & 15u);
            const unsigned char* src_al = src - lead;
            const unsigned total = lead + unsigned(span * a.N * int64_t(sizeof(T)));
            const unsigned bulk = total & ~15u;
            sB = reinterpret_cast<T*>(dsm + lead);
            if (threadIdx.x == 0 && bulk > 0) {
                mbar_expect_tx(&bar, bulk);
                bulk_g2s(dsm, src_al, bulk, &bar);
            }
            for (unsigned i = bulk + threadIdx.x; i < total; i += kThreads) dsm[i] = __ldg(src_al + i);
            if (bulk > 0) mbar_wait(&bar, 0);
        } else {
            const int nvec = pitch / V;
            for (int64_t i = threadIdx.x; i < span * nvec; i += kThreads) {
                const int64_t row = i / nvec;
                const int j = int(i - row * nvec);
                st_frag_shared<T, V>(sB + row * pitch + j * V,
                                     ld_frag<T, V>(a.B + (c0 + row) * a.ldb + tile0 + j * V));
            }
        }
    }
    __syncthreads();
    const WinSlots<T> win{sB, c0, pitch, tile0};
    const unsigned mask = group_mask<LPR>();
    const int gl = threadIdx.x & (LPR - 1);
    const int g = threadIdx.x / LPR;
    const int n0 = tile0 + gl * V;
    const int nblk = int((r_end - R0 + a.rpg - 1) / a.rpg);
    for (int blk = g; blk < nblk; blk += G) {
        const int r0 = int(R0) + blk * int(a.rpg);
        const int r1 = min(r_end, r0 + int(a.rpg));
        sr_walk<T, false, false, V, LPR, CPL, kRBWin>(a, __ldg(a.rp + r0), __ldg(a.rp + r1), r0,
                                                      r1 - r0, n0, mask, gl, CtaSlots<T>{}, win);
    }
}

// EB + SR: group w owns partition chunk w (partition.hpp:45-64).
template <typename T, bool CM, bool EXACT, int V, int LPR, int CPL>
__global__ void __launch_bounds__(kThreads, (sizeof(T) == 8 || LPR <= 2) ? 3 : 4) k_eb_sr(const SpmmArgs<T> a) {
    constexpr int TN = LPR * V * CPL;
    const unsigned mask = group_mask<LPR>();
    const int gl = threadIdx.x & (LPR - 1);
    const int64_t w = (int64_t(blockIdx.x) * kThreads + threadIdx.x) / LPR;
    int64_t e0 = 0, e1 = 0;
    if (w < a.P) chunk_bounds(a.nnz, a.P, w, e0, e1);
    if (e0 >= e1) {
        griddep_wait();
        return;
    }
    const int n0 = blockIdx.y * TN + gl * V;
    sr_walk<T, CM, EXACT, V, LPR, CPL, kEB>(a, int(e0), int(e1), __ldg(a.rows + e0), 0, n0, mask,
                                            gl);
    griddep_wait();
}

// EB + SR, fast path: a CTA owns G = 256/LPR consecutive sub-chunks of a.sub pairs,
// one per lane group. Rows crossing a sub-chunk boundary inside the CTA are summed in
// shared memory and stored once; only rows crossing the CTA's own range take an
// atomic (pre-zeroed by k_eb_prep_uniform). Long power-law rows thus receive one
// atomic per CTA instead of one per group.
template <typename T, bool CM, int V, int LPR, int CPL, int NT = kThreads>
__global__ void __launch_bounds__(NT, ((sizeof(T) == 8 || LPR <= 2) ? 3 : 4) * (kThreads / NT))
k_eb_sr_cta(const SpmmArgs<T> a) {
    constexpr int G = NT / LPR;
    constexpr int TN = LPR * V * CPL;
    // +1 padding: ptxas pairs the combine loop's loads into 64-bit LDS, and with an odd
    // trip count (G + 1) the last pair would read one element past the array.
    __shared__ T sL[(G + 2) * TN];
    __shared__ T sR[(G + 2) * TN];
    __shared__ int srow[G + 2];
    for (int i = threadIdx.x; i < (G + 2) * TN; i += NT) sL[i] = sR[i] = T(0);
    for (int i = threadIdx.x; i < G + 2; i += NT) srow[i] = -1;
    __syncthreads();

    const unsigned mask = group_mask<LPR>();
    const int gl = threadIdx.x & (LPR - 1);
    const int g = threadIdx.x / LPR;
    const int64_t E0 = int64_t(blockIdx.x) * G * a.sub;
    const int64_t E1 = min(a.nnz, E0 + int64_t(G) * a.sub);
    const int64_t e0 = E0 + int64_t(g) * a.sub;
    const int64_t e1 = min(E1, e0 + a.sub);
    const int tile0 = blockIdx.y * TN;
    const int n0 = tile0 + gl * V;
    CtaSlots<T> slots{sL, sR, srow, g, tile0, TN};
    if (e0 < e1)
        sr_walk<T, CM, false, V, LPR, CPL, kEBCta>(a, int(e0), int(e1), __ldg(a.rows + e0), 0, n0,
                                                   mask, gl, slots);
    __syncthreads();
    // Combine: thread t owns tile column t; boundaries in order, segmented by row.
    for (int t = threadIdx.x; t < TN; t += NT) {
        const int col = tile0 + t;
        if (col >= a.N) continue;
        int cur = -1;
        T acc = T(0);
        auto deposit = [&](int row, T v) {
            T* y = a.C + int64_t(row) * a.ldc + col;
            if (__ldg(a.rp + row) >= E0 && __ldg(a.rp + row + 1) <= E1) {
                *y = v;
            } else {
                griddep_wait();
                atomicAdd(y, v);
            }
        };
        for (int b = 0; b <= G; ++b) {
            const int row = srow[b];
            if (row < 0) continue;
            const T v = sL[b * TN + t] + sR[b * TN + t];
            if (row != cur) {
                if (cur >= 0) deposit(cur, acc);
                cur = row;
                acc = v;
            } else {
                acc += v;
            }
        }
        if (cur >= 0) deposit(cur, acc);
    }
    griddep_wait();  // complete only after the prologue (programmatic launch)
}

// EB + SR, fast path for one-lane groups (N <= V, i.e. N <= 4 in fp32): every thread
// owns a sub-chunk of S pairs. The CTA first stages its contiguous range of (col, val,
// row id) into shared memory with coalesced loads, transposed (pair i of thread t at
// [i][t], row pitch 257 — conflict-free for both the staging stores and the per-thread
// reads); each thread then issues all S of its B gathers before accumulating, so a
// warp keeps 32*S gathers in flight. Owned rows are stored, rows cut by a sub-chunk
// boundary take atomics (pre-zeroed by k_eb_prep_uniform with G = 1).
template <typename T, bool CM, int V, int S, int NT = kThreads>
__global__ void __launch_bounds__(NT, 3 * (kThreads / NT)) k_eb_sr_thr(const SpmmArgs<T> a) {
    // Per-thread reads of the staged tile are conflict-free for odd S (scalar) and for
    // S = 4 x odd (128-bit reads: 8 lanes per phase hit 8 distinct 16-B bank groups).
    static_assert(S % 2 == 1 || (S % 4 == 0 && (S / 4) % 2 == 1), "conflict-free S");
    static_assert((NT * S * sizeof(int)) % 16 == 0, "TMA bulk size granularity");
    // natural order: pair i of thread t at [t*S + i]
    __shared__ __align__(16) int s_c[S * NT];
    __shared__ __align__(16) int s_r[S * NT];
    __shared__ __align__(16) T s_v[S * NT];
    __shared__ uint64_t bar;
    const int64_t E0 = int64_t(blockIdx.x) * NT * S;
    const int64_t E1 = min(a.nnz, E0 + int64_t(NT) * S);
    if (a.bulk_ok && E1 - E0 == int64_t(NT) * S) {
        // Full tile: three 1-D TMA bulk copies, one elected thread, mbarrier completion.
        constexpr unsigned kIdxBytes = NT * S * sizeof(int);
        constexpr unsigned kValBytes = NT * S * sizeof(T);
        if (threadIdx.x == 0) mbar_init(&bar, 1);
        __syncthreads();
        if (threadIdx.x == 0) {
            mbar_expect_tx(&bar, 2 * kIdxBytes + kValBytes);
            bulk_g2s(s_c, a.ci + E0, kIdxBytes, &bar);
            bulk_g2s(s_v, a.va + E0, kValBytes, &bar);
            bulk_g2s(s_r, a.rows + E0, kIdxBytes, &bar);
        }
        mbar_wait(&bar, 0);
    } else {  // ragged tail tile: coalesced loads, all issued before any store
        int lc[S], lr[S];
        T lv[S];
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const int64_t e = E0 + k * NT + threadIdx.x;
            const bool ok = e < E1;
            lc[k] = ok ? ld_stream(a.ci + e) : 0;
            lv[k] = ok ? ld_stream(a.va + e) : T(0);
            lr[k] = ok ? ld_stream(a.rows + e) : INT_MAX;
        }
#pragma unroll
        for (int k = 0; k < S; ++k) {
            const int jj = k * NT + threadIdx.x;
            s_c[jj] = lc[k];
            s_v[jj] = lv[k];
            s_r[jj] = lr[k];
        }
        __syncthreads();
    }
    const int t = threadIdx.x;
    const int lane = t & 31;
    const int64_t e0 = E0 + int64_t(t) * S;
    const int64_t e1 = min(E1, e0 + S);
    const bool active = e0 < e1;  // no early exit: the warp combines split rows below
    const int n = active ? int(e1 - e0) : 0;
    const int col0 = blockIdx.y * V;  // one V-wide column slot per thread
    // this thread's pairs into registers (128-bit shared loads when S = 4k)
    int cc[S], rr[S];
    T vv[S];
    if constexpr (S % 4 == 0 && sizeof(T) == 4) {
#pragma unroll
        for (int k = 0; k < S / 4; ++k) {
            const int4 c4 = *reinterpret_cast<const int4*>(s_c + t * S + 4 * k);
            const int4 r4 = *reinterpret_cast<const int4*>(s_r + t * S + 4 * k);
            const float4 v4 = *reinterpret_cast<const float4*>(s_v + t * S + 4 * k);
            cc[4 * k] = c4.x; cc[4 * k + 1] = c4.y; cc[4 * k + 2] = c4.z; cc[4 * k + 3] = c4.w;
            rr[4 * k] = r4.x; rr[4 * k + 1] = r4.y; rr[4 * k + 2] = r4.z; rr[4 * k + 3] = r4.w;
            vv[4 * k] = v4.x; vv[4 * k + 1] = v4.y; vv[4 * k + 2] = v4.z; vv[4 * k + 3] = v4.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < S; ++i) {
            cc[i] = s_c[t * S + i];
            rr[i] = s_r[t * S + i];
            vv[i] = s_v[t * S + i];
        }
    }
    Frag<T, V> b[S];
#pragma unroll
    for (int i = 0; i < S; ++i) b[i] = gather<T, CM, V>(a, i < n ? cc[i] : 0, col0);
    int last_row = rr[0];
#pragma unroll
    for (int i = 1; i < S; ++i)
        if (i < n) last_row = rr[i];
    const int first_row = active ? rr[0] : INT_MAX;
    if (!active) last_row = INT_MAX;
    const int before = !active || e0 == 0 ? -1
                       : (t > 0 ? s_r[t * S - 1] : __ldg(a.rows + e0 - 1));
    const int after = !active || e1 >= a.nnz ? -1
                      : (e1 < E1 ? s_r[(t + 1) * S] : __ldg(a.rows + e1));
    const bool first_split = active && before == first_row;
    const bool last_split = active && after == last_row;
    // A split row's partial is parked (head = first row, tail = last row when distinct).
    Frag<T, V> acc, head, tail;
#pragma unroll
    for (int i = 0; i < V; ++i) acc.v[i] = head.v[i] = tail.v[i] = T(0);
    int r = first_row;
    auto flush = [&]() {
        if (first_split && r == first_row) {
            head = acc;
        } else if (last_split && r == last_row) {
            tail = acc;
        } else {
            st_frag(a.C + int64_t(r) * a.ldc + col0, acc);
        }
#pragma unroll
        for (int i = 0; i < V; ++i) acc.v[i] = T(0);
    };
#pragma unroll
    for (int i = 0; i < S; ++i) {
        if (i < n) {
            const int rid = rr[i];
            if (rid != r) {
                flush();
                r = rid;
            }
            const T v = vv[i];
#pragma unroll
            for (int q = 0; q < V; ++q) acc.v[q] = madd<false>(acc.v[q], v, b[i].v[q]);
        }
    }
    if (active) flush();
    // Warp combine: the row crossing the boundary into lane l is lane l's first row; it
    // collects lane l's head and lane l-1's tail, and runs of lanes lying wholly inside
    // one long row share that key, so a gated scan sums each run into its first lane.
    const bool has_tail = last_split && !(first_split && first_row == last_row);
    const bool tail_in = (__shfl_up_sync(kFull, has_tail ? 1 : 0, 1) != 0) && lane > 0;
    const int key = first_split ? first_row : -1 - lane;  // unique keys for non-contributors
    const unsigned gates = scan_gates<32>(kFull, key, lane);
    const int prev_key = __shfl_up_sync(kFull, key, 1);
    const bool seg_start = first_split && (lane == 0 || prev_key != key);
#pragma unroll
    for (int q = 0; q < V; ++q) {
        const T tin = __shfl_up_sync(kFull, tail.v[q], 1);
        T v = first_split ? head.v[q] + (tail_in ? tin : T(0)) : T(0);
        v = group_conditional_scan_gated<32>(kFull, v, gates);
        head.v[q] = v;
    }
    // A run that neither began before the warp's range (lane 0's head) nor continues
    // past it (lane 31 wholly inside the row) is complete: plain store. Only rows that
    // cross a warp boundary take atomics (pre-zeroed at warp granularity).
    // (Shuffles run on every lane — inside a short-circuit they would not.)
    const bool next_takes = __shfl_down_sync(kFull, first_split ? 1 : 0, 1) != 0;
    const int l31_key = __shfl_sync(kFull, key, 31);
    const bool l31_cont = __shfl_sync(kFull, (last_split && first_row == last_row) ? 1 : 0, 31);
    if (seg_start) {
        T* y = a.C + int64_t(first_row) * a.ldc + col0;
        const bool crosses = lane == 0 || (l31_key == key && l31_cont);
        if (crosses) {
            griddep_wait();
            atomic_add_frag(y, head);
        } else {
            st_frag(y, head);
        }
    }
    const bool tail_out = has_tail && (lane == 31 || !next_takes);
    griddep_wait();  // before the tail deposit, and so the grid ends after the prologue
    if (tail_out) atomic_add_frag(a.C + int64_t(last_row) * a.ldc + col0, tail);
}

// Prologue of the EB fast paths: zeroes the rows the EB kernel deposits into with
// atomics — the row holding element k*G*sub when it continues from element k*G*sub - 1
// (a split row at a CTA / chunk boundary) — and the empty rows (never visited by an EB
// walker). One thread per (row, VZ-wide column vector): coalesced vector stores.
template <typename T, int VZ>
__global__ void __launch_bounds__(kThreads)
k_eb_prep_uniform(const int* __restrict__ rows, int64_t nnz, int64_t stride, int64_t n_bound,
                  T* C, int64_t ldc, int N, const int* __restrict__ empty_rows, int n_empty,
                  int shift) {
    griddep_launch_dependents();  // the EB kernel may launch now; it waits before atomics
    const int nvec = (N + VZ - 1) / VZ;
    const int64_t idx = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    // shift >= 0: nvec is a power of two and idx fits 32 bits (host-checked): no 64-bit
    // division (ncu: issue-bound on it, 33 us for 84 MB on power-law s20 N = 64)
    const int64_t item = shift >= 0 ? int64_t(uint32_t(idx) >> shift) : idx / nvec;
    const int j = shift >= 0 ? int(uint32_t(idx) & uint32_t(nvec - 1)) : int(idx - item * nvec);
    int row;
    if (item < n_bound) {
        const int64_t b = (item + 1) * stride;  // boundary 0 never splits a row
        if (b >= nnz) return;
        row = __ldg(rows + b);
        if (__ldg(rows + b - 1) != row) return;
    } else if (item - n_bound < n_empty) {
        row = __ldg(empty_rows + (item - n_bound));
    } else {
        return;
    }
    Frag<T, VZ> z;
#pragma unroll
    for (int i = 0; i < VZ; ++i) z.v[i] = T(0);
    st_frag_rw(C + int64_t(row) * ldc + int64_t(j) * VZ, z);
}

// =============================================================== RB + PR (K1 / K3)
// W lanes per row step through the row in W-wide tiles (Technique 1 for-loop);
// each column slot's tile products go through the adjacent-pair tree, and the
// slot's owner lane (slot % W) carries the row accumulator: y += tile_sum per
// tile, the reference's RB+PR order (spmm.hpp:93-103).
template <typename T, bool CM, bool EXACT, int V, int W, int OWN>
__global__ void __launch_bounds__(kThreads) k_rb_pr(const SpmmArgs<T> a) {
    constexpr int NSLOT = W * OWN;  // column slots per tile (V columns each)
    constexpr int U = NSLOT < 4 ? NSLOT : 4;
    const unsigned mask = group_mask<W>();
    const int gl = threadIdx.x & (W - 1);
    const int64_t row = (int64_t(blockIdx.x) * kThreads + threadIdx.x) / W;
    if (row >= a.M) return;
    const int nbase = blockIdx.y * NSLOT * V;

    Frag<T, V> acc[OWN];
#pragma unroll
    for (int o = 0; o < OWN; ++o)
#pragma unroll
        for (int i = 0; i < V; ++i) acc[o].v[i] = T(0);

    const int rs = __ldg(a.rp + row), re = __ldg(a.rp + row + 1);
    for (int j = rs; j < re; j += W) {
        const int e = j + gl;
        const bool valid = e < re;
        const int c = valid ? ld_stream(a.ci + e) : 0;
        const T v = valid ? ld_stream(a.va + e) : T(0);
#pragma unroll
        for (int s0 = 0; s0 < NSLOT; s0 += U) {
            Frag<T, V> b[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int col = nbase + (s0 + u) * V;
                if (valid && col < a.N) b[u] = gather<T, CM, V>(a, c, col);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int s = s0 + u;
                const int col = nbase + s * V;
                if (col < a.N) {  // group-uniform
#pragma unroll
                    for (int i = 0; i < V; ++i) {
                        // padded lanes contribute +0 exactly as the reference pads (spmm.hpp:98-99)
                        T p = valid ? (EXACT ? mul_rn(v, b[u].v[i]) : v * b[u].v[i]) : T(0);
                        p = group_tree_sum<W>(mask, p);
                        if ((s % W) == gl)
                            acc[s / W].v[i] = EXACT ? add_rn(acc[s / W].v[i], p) : acc[s / W].v[i] + p;
                    }
                }
            }
        }
    }
#pragma unroll
    for (int o = 0; o < OWN; ++o) {
        const int s = o * W + gl;
        const int col = nbase + s * V;
        if (col < a.N) st_frag(a.C + row * a.ldc + col, acc[o]);
    }
}

// =============================================================== EB prep
// partition_elements on the device (partition.hpp:45-64) for P chunks: the row of
// each chunk's first element by binary search (upper_bound - 1), M for empty tail
// chunks. A chunk whose first row began in an earlier chunk marks that row as
// split: it is zeroed here so the EB kernels can deposit into it with atomics.
// Empty rows (never touched by an EB walker) are zeroed from the handle's list.
template <typename T>
__global__ void __launch_bounds__(kThreads)
k_eb_prep(const int* __restrict__ rp, int M, int64_t nnz, int64_t P, int* __restrict__ chunk_row,
          T* C, int64_t ldc, int N, const int* __restrict__ empty_rows, int n_empty,
          const int* __restrict__ rows) {
    griddep_launch_dependents();
    const int64_t tid = int64_t(blockIdx.x) * kThreads + threadIdx.x;
    if (tid < P) {
        int64_t b, e;
        chunk_bounds(nnz, P, tid, b, e);
        if (rows != nullptr) {  // SpMM path: COO ids make the split test a compare
            if (b > 0 && b < nnz) {
                const int row = __ldg(rows + b);
                if (__ldg(rows + b - 1) == row) {
                    T* y = C + int64_t(row) * ldc;
                    for (int n = 0; n < N; ++n) y[n] = T(0);
                }
            }
        } else {  // partition_elements API: chunk-start rows by binary search
            const int row = b < nnz ? row_of_element(rp, M, int(b)) : M;
            chunk_row[tid] = row;
        }
    } else if (tid - P < int64_t(n_empty) * N) {
        const int64_t k = tid - P;
        const int r = empty_rows[k / N];
        C[int64_t(r) * ldc + k % N] = T(0);
    }
}

// =============================================================== EB + PR (K5 / K7)
// W lanes take W consecutive nonzeros of the chunk (tiles at e0 + m*W, as the
// reference's groups, spmm.hpp:164-183). Each lane reads its element's row id from
// the handle's COO array, the gated scan sums each row run, and the run's first lane
// deposits: a row owned by the chunk is stored on its
// first tile and read-modify-written on later tiles (y += seg, the reference's
// deposit order), a split row takes an atomic add.
template <typename T, bool CM, bool EXACT, int V, int W, int OWN>
__global__ void __launch_bounds__(kThreads) k_eb_pr(const SpmmArgs<T> a) {
    constexpr int NSLOT = W * OWN;
    constexpr int U = NSLOT < 4 ? NSLOT : 4;
    const unsigned mask = group_mask<W>();
    const int gl = threadIdx.x & (W - 1);
    const int64_t w = (int64_t(blockIdx.x) * kThreads + threadIdx.x) / W;
    int64_t e0l = 0, e1l = 0;
    if (w < a.P) chunk_bounds(a.nnz, a.P, w, e0l, e1l);
    if (e0l >= e1l) {
        griddep_wait();
        return;
    }
    const int e0 = int(e0l), e1 = int(e1l);
    const int nbase = blockIdx.y * NSLOT * V;
    // Split rows: the chunk's first row if it began before e0, its last row if it
    // continues past e1 (COO row ids, no dependent row-offset loads).
    const int first_row = __ldg(a.rows + e0), last_row = __ldg(a.rows + e1 - 1);
    const bool first_split = e0 > 0 && __ldg(a.rows + e0 - 1) == first_row;
    const bool last_split = e1 < a.nnz && __ldg(a.rows + e1) == last_row;
    int prev_last = e0 > 0 ? __ldg(a.rows + e0 - 1) : -1;  // row of the element before the tile

    for (int tb = e0; tb < e1; tb += W) {
        const int e = tb + gl;
        const bool valid = e < e1;
        const int c = valid ? ld_stream(a.ci + e) : 0;
        const T v = valid ? ld_stream(a.va + e) : T(0);
        const int row = valid ? ld_stream(a.rows + e) : a.M;  // sentinel pads (spmm.hpp:167)
        const unsigned gates = scan_gates<W>(mask, row, gl);
        const int prev_id = __shfl_up_sync(mask, row, 1, W);
        const bool seg_start = valid && (gl == 0 || prev_id != row);
        const int before = gl == 0 ? prev_last : prev_id;
        const bool first = before != row;  // this segment opens its row
        const bool owned = !((first_split && row == first_row) || (last_split && row == last_row));
#pragma unroll
        for (int s0 = 0; s0 < NSLOT; s0 += U) {
            Frag<T, V> b[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int col = nbase + (s0 + u) * V;
                if (valid && col < a.N) b[u] = gather<T, CM, V>(a, c, col);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int col = nbase + (s0 + u) * V;
                if (col < a.N) {  // group-uniform
                    Frag<T, V> p;
#pragma unroll
                    for (int i = 0; i < V; ++i) {
                        p.v[i] = valid ? (EXACT ? mul_rn(v, b[u].v[i]) : v * b[u].v[i]) : T(0);
                        p.v[i] = group_conditional_scan_gated<W>(mask, p.v[i], gates);
                    }
                    if (seg_start) {
                        T* y = a.C + int64_t(row) * a.ldc + col;
                        if (!owned) {
                            griddep_wait();
                            atomic_add_frag(y, p);
                        } else if (first) {
                            if constexpr (EXACT) {
#pragma unroll
                                for (int i = 0; i < V; ++i) p.v[i] = add_rn(T(0), p.v[i]);
                            }
                            st_frag_rw(y, p);
                        } else {
                            Frag<T, V> old = ld_frag_rw<T, V>(y);
#pragma unroll
                            for (int i = 0; i < V; ++i) p.v[i] = add_rn(old.v[i], p.v[i]);
                            st_frag_rw(y, p);
                        }
                    }
                }
            }
        }
        __syncwarp(mask);  // orders this tile's owned-row stores before the next tile's RMW
        const int last = min(W, e1 - tb) - 1;
        prev_last = __shfl_sync(mask, row, last, W);
    }
    griddep_wait();
}

}  // namespace daspmm
