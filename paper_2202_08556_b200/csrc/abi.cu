// daspmm — C ABI: handles, validation, launch planning, host-operand paths.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <type_traits>
#include <cstdlib>
#include <cstring>
#include <string>

#include <chrono>

#include "dispatch.h"
#include "internal.h"
#include "kernels.cuh"

namespace daspmm {

static thread_local std::string g_err;

static bool debug_on() {
    static const bool on = getenv("DASPMM_DEBUG") != nullptr;
    return on;
}
void set_error(const std::string& msg) { g_err = msg; }

// DASPMM_DEBUG also traces handle creation: wall time since the previous mark.
void trace_mark(const char* what) {
    if (!debug_on()) return;
    static thread_local std::chrono::steady_clock::time_point last;
    const auto now = std::chrono::steady_clock::now();
    if (what) fprintf(stderr, "[daspmm] %-28s %9.3f ms\n", what,
                      std::chrono::duration<double, std::milli>(now - last).count());
    last = now;
}
int fail(int code, const std::string& msg) {
    g_err = msg;
    if (debug_on()) fprintf(stderr, "[daspmm] error %d: %s\n", code, msg.c_str());
    return code;
}
int cuda_fail(cudaError_t e, const char* what) {
    g_err = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    if (debug_on()) fprintf(stderr, "[daspmm] cuda error: %s\n", g_err.c_str());
    return DASPMM_ERR_CUDA;
}

static bool is_pow2(int64_t w) { return w > 0 && (w & (w - 1)) == 0; }

static const char* kKernelNames[8] = {"RB+RM+SR", "RB+RM+PR", "RB+CM+SR", "RB+CM+PR",
                                      "EB+RM+SR", "EB+RM+PR", "EB+CM+SR", "EB+CM+PR"};

// worker.hpp:29-40 with the reference's message text.
static int validate_config(int64_t P, int64_t W, int64_t Cb, bool allow_auto_p) {
    std::string msg = "spmm: invalid config";
    bool bad = false;
    if (P < (allow_auto_p ? 0 : 1)) {
        msg += "; num_workers must be >= 1, got " + std::to_string(P);
        bad = true;
    }
    if (W < 2 || !is_pow2(W)) {
        msg += "; group_width must be a power of two >= 2, got " + std::to_string(W);
        bad = true;
    }
    if (Cb < 1) {
        msg += "; col_block must be >= 1, got " + std::to_string(Cb);
        bad = true;
    }
    if (bad) return fail(DASPMM_ERR_INVALID_CONFIG, msg);
    if (W > 1024)
        return fail(DASPMM_ERR_UNSUPPORTED,
                    "spmm: group_width " + std::to_string(W) +
                        " exceeds one 1024-thread CTA (B200 build supports 2..1024)");
    return DASPMM_OK;
}

static int elem_size(int dtype) { return dtype == DASPMM_F64 ? 8 : 4; }

static bool aligned(const void* p, int bytes) {
    return (reinterpret_cast<uintptr_t>(p) % uintptr_t(bytes)) == 0;
}

// Vector width for row-major B/C: every gather/store of V elements must be aligned.
static int pick_v(int dtype, int64_t N, const void* B, int64_t ldb, const void* C, int64_t ldc) {
    const int es = elem_size(dtype);
    const int vmax = dtype == DASPMM_F64 ? 2 : 4;
    for (int v = vmax; v > 1; v >>= 1) {
        if (N % v == 0 && ldb % v == 0 && ldc % v == 0 && aligned(B, v * es) && aligned(C, v * es))
            return v;
    }
    return 1;
}

static int pow2_ceil(int64_t x) {
    int p = 1;
    while (p < x && p < 32) p <<= 1;
    return p;
}

// Stream-ordered scratch (EB chunk rows, layout conversions) comes from a memory pool the
// library owns, one per device, so the host process's default pool keeps its own
// settings. Up to 256 MB of freed blocks stay reserved between calls, so a steady stream
// of calls does not unmap and remap its scratch on every synchronisation.
static cudaMemPool_t lib_pool(int dev) {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    static bool tried[64] = {};
    if (dev < 0 || dev >= 64) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    if (!tried[dev]) {
        tried[dev] = true;
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        if (cudaMemPoolCreate(&pools[dev], &props) != cudaSuccess) {
            cudaGetLastError();
            pools[dev] = nullptr;
        } else {
            uint64_t thr = uint64_t(256) << 20;
            cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    return pools[dev];
}

cudaError_t scratch_alloc(void** p, size_t bytes, int dev, cudaStream_t s) {
    cudaMemPool_t pool = lib_pool(dev);
    return pool ? cudaMallocFromPoolAsync(p, bytes, pool, s) : cudaMallocAsync(p, bytes, s);
}

cudaError_t scratch_free(void* p, cudaStream_t s) { return p ? cudaFreeAsync(p, s) : cudaSuccess; }

// Planner tuning knobs (environment, all optional; documented at their uses and in
// INTEGRATION.md). Read once into a snapshot so the per-call host path does no getenv;
// daspmm_reload_env() re-reads them (tests and tuning sweeps that change them).
struct Knobs {
    int64_t tile_cols = 0;    // DASPMM_TILE_COLS: column-tile width override
    bool eb_cta = true;       // DASPMM_EB_CTA=0: no CTA-combined EB+SR walk
    int64_t eb_chunk = 0;     // DASPMM_EB_CHUNK: EB pairs per group override
    bool lean = true;         // DASPMM_LEAN=0: no lean SR kernels
    int lean_min_lanes = 2;   // DASPMM_LEAN_MIN_LANES
    int64_t lean_chunk = 0;   // DASPMM_LEAN_CHUNK: lean EB chunk override
    int lean_rw = -1;         // DASPMM_LEAN_RW=0/1: force the segment / range walk
    bool lean_rb = false;     // DASPMM_LEAN_RB=1: lean walk for RB+SR too
    int64_t rpg = 0;          // DASPMM_RPG: RB rows per group override
    int64_t lean_rpg = 0;     // DASPMM_LEAN_RPG
    bool win = false;         // DASPMM_WIN=1: shared-memory B-window RB kernel
    bool tma = false;         // DASPMM_TMA=1: TMA gather4 EB kernel
    int64_t tma_lw = 0;       // DASPMM_TMA_LW: its pairs per warp
    bool fault = false;       // SPMMKIT_ENABLE_FAULT_INJECTION=1 + DASPMM_INJECT_FAULT=1
    bool pdl = true;          // DASPMM_PDL=0: EB kernels wait for their prologue to finish
    bool tile = true;         // DASPMM_TILE=0: no dense row-panel tile walk for RB+RM+SR
    bool tile_force = false;  // DASPMM_TILE=2: the tile walk at any grid size (tests)
    bool cm_rows = true;      // DASPMM_CM_ROWS=0: RB+CM+SR on the base walk (lanes over columns)
    bool cm_rows_force = false;  // DASPMM_CM_ROWS=2: lanes over rows on skewed rows too (tests)
    int tile_rl = 0;          // DASPMM_TILE_RL=1/8: force the tile walk's row lanes (tuning)
    int tile_u = 0;           // DASPMM_TILE_U=2/4/8: B rows in flight per lane (tuning)
    // DASPMM_CTA_THREADS (64/128/256): CTA size of the CTA-combined EB walk. Measured:
    // smaller CTAs wait less at the combine barrier (power-law s20 N = 32 273 -> 248 us,
    // s17 N = 32 66 -> 52, c4 N = 64 1.69 -> 1.61 ms; profiles/r01c_cta_threads_probe.txt).
    int cta_threads = 64;
    bool cta_threads_set = false;
    // DASPMM_THR_THREADS (64/128/256): CTA size of the one-lane staged path (measured:
    // 64 -> uniform s20 N = 4 121 -> 105 us, N = 2 105 -> 97; r01c_thr_threads_probe.txt).
    int thr_threads = 64;
    // DASPMM_RB_THREADS (64/128/256): CTA size of fast RB+RM+SR (measured: 128 -> banded
    // s20 N = 8 90 -> 82 us, uniform s20 N = 8 133 -> 123; r01c_rb_threads_probe.txt).
    int rb_threads = 128;
    // DASPMM_LEAN_THREADS (64/128/256): CTA size of the lean kernels (measured: 128 vs
    // 256 -> c3 3.78 -> 3.69 ms, power-law s20 N = 8 174 -> 156 us; 64 another ~1%;
    // r01c_lean_threads_probe.txt).
    int lean_threads = 64;
};

static Knobs read_knobs() {
    auto str = [](const char* n) -> const char* { return getenv(n); };
    auto i64 = [&](const char* n) { const char* e = str(n); return e ? int64_t(atoll(e)) : int64_t(0); };
    auto on = [&](const char* n, char v) { const char* e = str(n); return e && e[0] == v; };
    Knobs k;
    k.tile_cols = i64("DASPMM_TILE_COLS");
    k.eb_cta = !on("DASPMM_EB_CTA", '0');
    k.eb_chunk = i64("DASPMM_EB_CHUNK");
    k.lean = !on("DASPMM_LEAN", '0');
    if (str("DASPMM_LEAN_MIN_LANES")) k.lean_min_lanes = int(i64("DASPMM_LEAN_MIN_LANES"));
    k.lean_chunk = i64("DASPMM_LEAN_CHUNK");
    if (str("DASPMM_LEAN_RW")) k.lean_rw = on("DASPMM_LEAN_RW", '1') ? 1 : 0;
    k.lean_rb = on("DASPMM_LEAN_RB", '1');
    k.rpg = i64("DASPMM_RPG");
    k.lean_rpg = i64("DASPMM_LEAN_RPG");
    k.win = on("DASPMM_WIN", '1');
    k.tma = on("DASPMM_TMA", '1');
    k.tma_lw = i64("DASPMM_TMA_LW");
    k.fault = on("SPMMKIT_ENABLE_FAULT_INJECTION", '1') && on("DASPMM_INJECT_FAULT", '1');
    k.pdl = !on("DASPMM_PDL", '0');
    k.tile = !on("DASPMM_TILE", '0');
    k.tile_force = on("DASPMM_TILE", '2');
    k.cm_rows = !on("DASPMM_CM_ROWS", '0');
    k.cm_rows_force = on("DASPMM_CM_ROWS", '2');
    k.tile_rl = int(i64("DASPMM_TILE_RL"));
    if (const int64_t u = i64("DASPMM_TILE_U"); u == 2 || u == 4 || u == 8) k.tile_u = int(u);
    if (const int64_t t = i64("DASPMM_CTA_THREADS"); t == 32 || t == 64 || t == 128 || t == 256) {
        k.cta_threads = int(t);
        k.cta_threads_set = true;
    }
    if (const int64_t t = i64("DASPMM_THR_THREADS"); t == 32 || t == 64 || t == 128 || t == 256)
        k.thr_threads = int(t);
    if (const int64_t t = i64("DASPMM_RB_THREADS"); t == 64 || t == 128 || t == 256)
        k.rb_threads = int(t);
    if (const int64_t t = i64("DASPMM_LEAN_THREADS"); t == 64 || t == 128 || t == 256)
        k.lean_threads = int(t);
    return k;
}

static std::mutex g_knobs_mu;
static Knobs g_knobs = read_knobs();

static Knobs knobs() {
    std::lock_guard<std::mutex> lk(g_knobs_mu);
    return g_knobs;
}

// Column-tile width: B's working set for one tile of columns, K x tile x elem, should
// stay L2-resident (126 MB on B200) while A streams through. CTAs are scheduled
// x-major, so tiles (blockIdx.y) run one after another.
static int64_t max_tile_cols(const Knobs& kn) {
    if (kn.tile_cols > 0) return kn.tile_cols;
    // Measured on B200 (profiles/r01_notes.md): narrowing tiles to keep B in L2 costs
    // more in A re-reads and shorter gathers than it saves, up to N = 128. Wider N runs
    // 128-column y-tiles rather than two column slots per lane (c5, N = 256: EB
    // 65.5 -> 62.8 ms, RB 135 -> 100 ms; profiles/r01c_c5_tile_probe.txt).
    return 128;
}

// EB chunk count for a chunk length (DASPMM_EB_CHUNK overrides the length).
static int64_t auto_chunks(const Knobs& kn, int64_t nnz, int64_t chunk) {
    if (nnz <= 0) return 1;
    if (kn.eb_chunk > 0) chunk = kn.eb_chunk;
    return (nnz + chunk - 1) / chunk;
}

static int64_t lean_chunk(const Knobs& kn, bool range_walk) {
    // measured: 128 pairs for the range walk, 256 for the segment walk (c3 4.47 -> 4.34 ms)
    return kn.lean_chunk > 0 ? kn.lean_chunk : (range_walk ? 128 : 256);
}

// RB+RM+SR on row-local matrices: stage each CTA panel's B window in shared memory
// (k_rb_sr_win) when the windows are narrow enough to fit and every staged B row is
// reused by several nonzeros. The panel height is the largest R = 32 << i that still
// gives >= 2 CTAs per SM; the staging must fit kWinSmemMax for the widest panel.
static void plan_window(const daspmm_csr* h, Plan& p, int64_t N, int64_t tile_cols,
                        int64_t ytiles, const void* B, bool exact, bool enabled) {
    p.win_rows = 0;
    if (exact || p.cm || h->dtype != DASPMM_F32 || !enabled || h->spans == nullptr ||
        h->M <= 0 || h->nnz <= 0 || B == nullptr)
        return;
    const int64_t pitch = std::min<int64_t>(N, tile_cols);
    const int64_t row_bytes = pitch * 4;
    const double avg = double(h->nnz) / double(h->M);
    for (int i = daspmm_csr::kSpanLevels - 1; i >= 0; --i) {
        const int64_t R = int64_t(32) << i;
        if ((h->M + R - 1) / R * ytiles < 2 * 148 && i > 0) continue;
        const int64_t smem = h->span_max[i] * row_bytes + 16;
        if (size_t(smem) > kWinSmemMax) continue;
        if (h->span_avg[i] <= 0 || avg * double(R) / h->span_avg[i] < 3.0) return;
        p.win_rows = int(R);
        p.win_smem = size_t(smem);
        return;
    }
}

// Self-test fault hook (the reference's `validate --inject-fault`, spmmkit_cli.cpp:
// 366-371, 394-397): with SPMMKIT_ENABLE_FAULT_INJECTION=1 and DASPMM_INJECT_FAULT=1
// (Knobs::fault) every device SpMM adds 1 to C[0][0], so tests can prove the parity
// checks catch a wrong result. Never set in normal use.
template <typename T>
__global__ void k_inject_fault(T* c) {
    c[0] += T(1);
}

static cudaError_t inject_fault(int dtype, void* C, cudaStream_t s) {
    if (dtype == DASPMM_F64) k_inject_fault<double><<<1, 1, 0, s>>>(static_cast<double*>(C));
    else k_inject_fault<float><<<1, 1, 0, s>>>(static_cast<float*>(C));
    return cudaGetLastError();
}

Plan plan_spmm(const daspmm_csr* h, int kernel, int64_t P, int64_t W, int64_t N, const void* B,
               int64_t ldb, const void* C, int64_t ldc, bool exact, bool base_only) {
    const Knobs kn = knobs();
    Plan p;
    p.kernel = kernel;
    p.cm = (kernel >> 1) & 1;
    p.exact = exact;
    const bool eb = kernel >= 4, pr = kernel & 1;
    p.V = (p.cm || exact) ? 1 : pick_v(h->dtype, N, B, ldb, C, ldc);
    // Small calls (few rows / nonzeros) cannot fill 148 SMs with one V-wide slot per
    // lane: trade vector width for lanes until there are >= 2 CTAs per SM.
    // (EB+SR with N <= 4 keeps V = N: it runs the staged one-lane path instead.)
    if (!pr && !(eb && !exact && N <= p.V && N <= 4)) {
        const int64_t units = eb ? std::max<int64_t>(h->nnz / 32, 1) : std::max<int64_t>(h->M, 1);
        while (p.V > 1) {
            const int64_t lanes_now = std::min<int64_t>(32, (N + p.V - 1) / p.V);
            if (units * lanes_now >= 148LL * 512) break;  // >= 2 CTAs per SM
            if ((N + p.V / 2 - 1) / (p.V / 2) > 64) break;  // keep <= 2 slots per lane
            p.V /= 2;
        }
    }
    int64_t tile_max = max_tile_cols(kn);
    // RB+RM+SR with B far beyond L2 (>= 256 MB) and scattered columns (32-row panels span
    // over a quarter of K): two 64-column y-tiles run one after the other, halving the B
    // working set each pass must find in L2 (uniform s20 N = 128, B 512 MB: 1204 -> 1137
    // us). Below that size, or with row-local columns (banded s20: 454 -> 515 us), the
    // second pass over A costs more than the hits gain (c3, B 119 MB: 5.35 -> 7.20 ms;
    // profiles/r01c_tile64_probe.txt).
    if (kn.tile_cols <= 0 && !eb && !pr && !p.cm && !exact && N > 64 && N <= 128 &&
        h->K * N * elem_size(h->dtype) >= (int64_t(256) << 20) && h->spans != nullptr &&
        h->span_avg[0] * 4.0 >= double(h->K))
        tile_max = 64;
    const int64_t ncols = std::min<int64_t>(N, tile_max);
    const int64_t nv = (ncols + p.V - 1) / p.V;  // column slots per tile
    int64_t tile_cols;
    int lanes;
    if (!pr) {
        p.L = pow2_ceil(nv);
        p.X = nv > 32 ? 2 : 1;
        tile_cols = int64_t(p.L) * p.V * p.X;
        lanes = p.L;
    } else if (W > 32) {
        // wider than a warp: one CTA of W threads per group, scalar columns
        // (spmm_pr_wide.cu); the group walks every column itself, so one column tile.
        p.L = int(W);
        p.V = 1;
        p.X = 1;
        tile_cols = std::max<int64_t>(N, 1);
        lanes = p.L;
    } else {
        p.L = int(W);
        p.X = nv > W ? 2 : 1;
        tile_cols = int64_t(p.L) * p.X * p.V;
        lanes = p.L;
    }
    // Lean SR kernels (lean.cuh): fp32 fast mode, row-major B, groups of >= 2 lanes,
    // quad-aligned A arrays. One column slot per lane; wider N takes more y-tiles.
    p.lean = !base_only && !pr && !exact && !p.cm && h->dtype == DASPMM_F32 && P <= 0 &&
             kn.lean &&
             (p.L >= kn.lean_min_lanes || (!eb && p.L == 1)) && ldb < (int64_t(1) << 29) &&
             h->coo_rows != nullptr &&
             (((reinterpret_cast<uintptr_t>(h->ci) | reinterpret_cast<uintptr_t>(h->coo_rows) |
                                           reinterpret_cast<uintptr_t>(h->va)) & 15) == 0);
    // Where the lean walks win (measured on B200 against the shuffle-broadcast walks with
    // their one-IMAD gather addressing, profiles/r01_notes.md step 17):
    //   RB: one-lane groups only (below); elsewhere they tie within noise (uniform s20
    //       N = 8 130 vs 134 us; N = 128 1246 vs 1229);
    //   EB: N <= 16 (power-law s20 N = 8 160 vs 279, N = 16 199 vs 240) and long rows at
    //       any N (c3 3.77 vs 3.99 ms); from N = 32 on short rows the CTA-combined walk
    //       with 256-pair chunks wins (power-law s20 N = 32 326 vs 271, N = 128 957 vs
    //       699, c4 N = 64 2.45 vs 1.69 ms).
    const double avg_nonempty =
        h->M > h->n_empty ? double(h->nnz) / double(h->M - h->n_empty) : 0.0;
    const bool lean_ok = p.lean;  // eligibility (also of the TMA-gather variant)
    // RB: one-lane groups (N <= 4) take the lean walk — quad loads of each row's pairs
    // instead of 8 scalar loads per lane (uniform s20 N = 2 107 -> 96 us, banded 51 -> 47);
    // wider groups tie with k_rb_sr and stay on it unless DASPMM_LEAN_RB=1.
    if (p.lean && !eb) p.lean = kn.lean_rb || p.L == 1;
    if (p.lean && eb && N > 16 && avg_nonempty < 48.0) p.lean = false;
    if (p.lean) {
        p.X = 1;
        tile_cols = int64_t(p.L) * p.V;
    }
    const int64_t ytiles = std::max<int64_t>(1, (N + tile_cols - 1) / tile_cols);
    int64_t workers;
    // TMA gather4 EB kernel (opt-in while being measured: DASPMM_TMA=1)
    if (eb && lean_ok && N >= 32 && kn.tma &&
        tma_gather_supported(B, ldb, N, h->K) && h->nnz < (int64_t(1) << 31) - 1024) {
        p.tma = true;
        p.lean = false;
        const int bc = tma_box_cols(N);
        p.sub = 256;  // Lw: nonzeros per warp (multiple of 16)
        if (kn.tma_lw >= 16) p.sub = (kn.tma_lw / 16) * 16;
        p.P = (h->nnz + p.sub - 1) / p.sub;  // warps
        p.grid = dim3(unsigned((p.P + kTmaWarpsHost - 1) / kTmaWarpsHost),
                      unsigned((N + bc - 1) / bc), 1);
        return p;
    }
    if (eb && p.lean) {
        // short rows: range walk (COO ids per block); long rows: segment walk.
        // DASPMM_LEAN_RW=0/1 forces one (tuning aid).
        // Measured on B200: the range walk wins on short rows (power-law s20 N = 16:
        // 342 -> 217 us), the segment walk on long rows (c3: 5.26 -> 4.07 ms).
        p.lean_rw = kn.lean_rw >= 0 ? kn.lean_rw == 1 : avg_nonempty < 48.0;
        p.sub = lean_chunk(kn, p.lean_rw);
        // small matrices: shorten chunks until there are >= 4 CTAs per SM (s14 power-law,
        // N = 128: 128 CTAs at 256 pairs -> 88 us, vs 32 us with the grid filled)
        const int64_t fill = h->nnz * p.L / (148LL * 4 * kThreads);
        if (kn.lean_chunk <= 0 && fill < p.sub) p.sub = std::max<int64_t>(32, fill & ~7LL);
        p.P = (h->nnz + p.sub - 1) / p.sub;
        workers = std::max<int64_t>(p.P, 1);
    } else if (eb) {
        // EB chunk per group (measured on B200, profiles/r01_notes.md steps 4 and 19): 32
        // pairs (64 for full-warp SR groups) for narrow groups and PR; from 8-lane SR
        // groups (N >= 32) 256 pairs (power-law s20 N = 128 800 -> 707 us, N = 32
        // 328 -> 273, c4 N = 64 2.17 -> 1.71 ms), capped so small matrices keep >= 8 CTAs
        // per SM below full-warp groups (power-law s17 N = 32: 73 -> 64 us), >= 4 with them.
        int chunk = pr ? std::max<int>(int(W), 32) : (p.L >= 32 ? 64 : 32);
        if (!pr && !exact && p.L >= 8) {
            const int64_t fill = h->nnz * p.L / (148LL * (p.L >= 32 ? 4 : 8) * kThreads);
            chunk = int(std::max<int64_t>(chunk, std::min<int64_t>(256, fill)));
        }
        p.P = P > 0 ? P : auto_chunks(kn, h->nnz, chunk);
        workers = p.P;
        if (!pr && !exact && P <= 0 && p.L == 1 && p.X == 1 && N <= p.V && !p.cm &&
            h->dtype == DASPMM_F32) {
            // one-lane groups: CTA-staged thread sub-chunks (k_eb_sr_thr)
            p.thr = true;
            p.thr_threads = kn.thr_threads;
            p.sub = p.V >= 4 ? kThrS4 : kThrS;  // 3 x sub x 256 x 4 B of staging < 48 KB
            p.P = (h->nnz + p.sub - 1) / p.sub;
            workers = p.P;
        } else if (!pr && !exact && P <= 0 && kn.eb_cta) {  // CTA-combined boundary rows
            p.cta = true;
            // one full-warp group per CTA when groups are warps (power-law s20 N = 128
            // 686 -> 652 us); 64 threads otherwise (r01c_cta_threads_probe.txt)
            p.cta_threads = kn.cta_threads_set ? kn.cta_threads : (p.L >= 32 ? 32 : 64);
            p.sub = (h->nnz + p.P - 1) / std::max<int64_t>(p.P, 1);
            p.sub = std::max<int64_t>(p.sub, 1);
            p.P = (h->nnz + p.sub - 1) / p.sub;
            workers = p.P;
        }
    } else if (!pr) {
        // RB+SR row blocks (measured, profiles/r01_notes.md steps 5 and 19): one row per
        // group for 1-2 lane groups (N <= 8), ~128 pairs per group from 4 lanes on.
        const double avg = h->M > 0 ? double(h->nnz) / double(h->M) : 0.0;
        const double target = p.L >= 4 ? 128.0 : 16.0;
        int64_t rpg = avg > 0 ? int64_t(target / avg) : 64;
        // Skewed rows: a long row already fills its group; do not stack more rows on it.
        const double sd = h->M > 0 ? std::sqrt(h->h_feat.ss_par / double(h->M)) : 0.0;
        if (sd > 2.0 * avg) rpg = 1;
        const int64_t cap = std::max<int64_t>(1, h->M * lanes / (2LL * 148 * 2048));
        rpg = std::max<int64_t>(1, std::min<int64_t>({rpg, cap, int64_t(p.L)}));  // <= LPR
        if (kn.rpg > 0) rpg = std::min<int64_t>(kn.rpg, p.L);
        if (p.lean && kn.lean_rpg > 0) rpg = kn.lean_rpg;
        p.rpg = rpg;
        if (!base_only && !exact && !p.cm && h->dtype == DASPMM_F32 && !p.lean)
            p.rb_threads = kn.rb_threads;
        workers = (h->M + rpg - 1) / rpg;
        // RB+CM+SR: lanes over rows (spmm_cm.cu) — a warp's 32 rows read one column of B
        // together, coalesced wherever neighbouring rows share columns (banded s20 N = 128
        // 9.1 -> 1.6 ms, uniform 41.7 -> 8.8 ms). Skewed rows keep the base walk: a lane
        // alone on a long row stalls its warp (power-law s20 N = 32 6.8 -> 18.0 ms;
        // profiles/r02_cm_rows_probe.txt).
        const double sd_rows = h->M > 0 ? std::sqrt(h->h_feat.ss_par / double(h->M)) : 0.0;
        const double avg_rows = h->M > 0 ? double(h->nnz) / double(h->M) : 0.0;
        if (!base_only && !exact && p.cm && h->dtype == DASPMM_F32 && P <= 0 && kn.cm_rows &&
            (sd_rows <= 2.0 * avg_rows || kn.cm_rows_force)) {
            p.cm_rows = true;
            p.L = int(std::min<int64_t>(8, pow2_ceil(N)));
            p.V = 1;
            p.X = 1;
            p.grid = dim3(unsigned((h->M + 127) / 128), unsigned((N + p.L - 1) / p.L), 1);
            return p;
        }
        // Row-local matrices with tiles at least half full: the dense row-panel tile walk
        // (tile.cuh) gathers each B row once per 8-row panel instead of once per nonzero
        // (banded s20: N = 2 43 -> 31 us, N = 32 156 -> 114, half-width 32 N = 128 1749 ->
        // 889). Grids under ~3.5 CTAs per SM keep the base walk (banded s14 runs 0.5-0.8x
        // on tiles: too few panels to hide the window walk's latency).
        if (!base_only && !exact && !p.cm && h->dtype == DASPMM_F32 &&
            h->tile_state.load(std::memory_order_acquire) == 1 &&
            P <= 0 && kn.tile) {
            const int64_t nvt = (std::min<int64_t>(N, 128) + p.V - 1) / p.V;  // slots per tile
            const int cl = pow2_ceil(nvt);
            int rl = cl == 1 ? 8 : 1;  // one column slot (N <= 4): a lane per row
            // narrow N on a grid too small for one lane per column slot: a lane per row
            // (banded s17 N = 8: 18.4 -> 12.3 us)
            if (cl <= 4 && h->n_pan * cl * rl < 65536) rl = 8;
            if (kn.tile_rl == 1 || (kn.tile_rl == 8 && cl <= 4)) rl = kn.tile_rl;  // tuning
            const int64_t thr = h->n_pan * cl * rl;
            // a lane per row (rl = 8) needs twice the threads: banded s14 N = 4 at V = 1
            // (65536 threads) ran 10.2 us on tiles vs 8.3 on the base walk
            if (thr >= (rl == 8 ? 131072 : 65536) || kn.tile_force) {
                p.tile = true;
                p.lean = false;
                p.X = 1;
                p.L = cl;
                p.tile_rl = rl;
                p.tile_u = kn.tile_u > 0 ? kn.tile_u : (rl == 8 ? 8 : 4);
                const int64_t tn = int64_t(cl) * p.V;
                const int64_t yt = std::max<int64_t>(1, (N + tn - 1) / tn);
                p.grid = dim3(unsigned((thr + 127) / 128), unsigned(yt), 1);
                return p;
            }
        }
        if (!base_only) plan_window(h, p, N, tile_cols, ytiles, B, exact, kn.win);
        if (p.win_rows > 0) {
            p.lean = false;
            p.grid = dim3(unsigned((h->M + p.win_rows - 1) / p.win_rows), unsigned(ytiles), 1);
            return p;
        }
    } else {
        workers = h->M;
    }
    const int64_t threads = workers * lanes;
    if (p.lean) p.lean_threads = kn.lean_threads;
    const int64_t cta = p.cta ? p.cta_threads : p.thr ? p.thr_threads
                      : p.lean ? p.lean_threads
                      : (!eb && !pr && p.win_rows == 0) ? p.rb_threads : kThreads;
    p.grid = dim3(unsigned(std::max<int64_t>(1, (threads + cta - 1) / cta)), unsigned(ytiles), 1);
    return p;
}

template <typename T>
static cudaError_t run_plan(const daspmm_csr* h, const Plan& p, int64_t W, const void* B,
                            int64_t ldb, int64_t N, void* C, int64_t ldc, int* chunk_row,
                            cudaStream_t s, void* const* extra = nullptr, int n_extra = 0) {
    SpmmArgs<T> a;
    a.n_extra = n_extra;
    for (int d = 0; d < kMaxExtraDst; ++d)
        a.extra[d] = d < n_extra ? static_cast<T*>(extra[d]) : nullptr;
    a.rp = h->rp;
    a.ci = h->ci;
    a.va = static_cast<const T*>(h->va);
    a.B = static_cast<const T*>(B);
    a.C = static_cast<T*>(C);
    a.M = int(h->M);
    a.K = int(h->K);
    a.N = int(N);
    a.nnz = h->nnz;
    a.ldb = ldb;
    a.ldc = ldc;
    a.P = p.P;
    a.seg = int(std::max<int64_t>(W, 256));
    a.chunk_row = chunk_row;
    a.rpg = p.rpg;
    a.sub = p.sub;
    a.rows = h->coo_rows;
    a.spans = h->spans;
    a.win_rows = p.win_rows;
    a.bulk_ok = (((reinterpret_cast<uintptr_t>(h->ci) | reinterpret_cast<uintptr_t>(h->va) |
                   reinterpret_cast<uintptr_t>(h->coo_rows)) & 15) == 0) ? 1 : 0;
    const bool eb = p.kernel >= 4, pr = p.kernel & 1;
    if constexpr (std::is_same<T, float>::value) {
        if (p.tile) return launch_rb_sr_tile(p, a, h->tile_off, h->tile_c0, h->tile_val, h->n_pan, s);
        if (p.cm_rows) return launch_rb_cm_rows(p, a, s);
        if (p.tma) {  // prologue: split rows at warp-range ends and empty rows
            cudaError_t e = launch_eb_prep_uniform<T>(h->coo_rows, h->nnz, p.sub, p.P, 1,
                                                      static_cast<T*>(C), ldc, int(N),
                                                      h->empty_rows, int(h->n_empty), s);
            if (e != cudaSuccess) return e;
            return launch_eb_sr_tma(p, a, s);
        }
        if (p.lean) {
            if (eb) {  // prologue: split rows at chunk ends and empty rows are zeroed
                cudaError_t e = launch_eb_prep_uniform<T>(h->coo_rows, h->nnz, p.sub, p.P, 1,
                                                          static_cast<T*>(C), ldc, int(N),
                                                          h->empty_rows, int(h->n_empty), s);
                if (e != cudaSuccess) return e;
            }
            return launch_sr_lean(p, a, s);
        }
    }
    if (pr && p.L > 32) {  // group wider than a warp (spmm_pr_wide.cu)
        if (eb) {
            cudaError_t e = launch_eb_prep<T>(h->rp, int(h->M), h->nnz, p.P, chunk_row,
                                              static_cast<T*>(C), ldc, int(N), h->empty_rows,
                                              int(h->n_empty), h->coo_rows, s);
            if (e != cudaSuccess) return e;
        }
        return launch_pr_wide<T>(p, a, s);
    }
    if (eb) {
        cudaError_t e =
            (p.cta || p.thr)
                  ? launch_eb_prep_uniform<T>(h->coo_rows, h->nnz, p.sub, p.P,
                                              p.thr ? 32 : p.cta_threads / p.L,
                                              static_cast<T*>(C), ldc, int(N), h->empty_rows,
                                              int(h->n_empty), s)
                  : launch_eb_prep<T>(h->rp, int(h->M), h->nnz, p.P, chunk_row,
                                      static_cast<T*>(C), ldc, int(N), h->empty_rows,
                                      int(h->n_empty), h->coo_rows, s);
        if (e != cudaSuccess) return e;
        return pr ? launch_eb_pr<T>(p, a, s) : launch_eb_sr<T>(p, a, s);
    }
    return pr ? launch_rb_pr<T>(p, a, s) : launch_rb_sr<T>(p, a, s);
}

// Core device-operand SpMM (operands already validated).
// chunk_scratch: caller-provided EB scratch of >= plan.P ints (graph bodies cannot
// allocate); null = stream-ordered allocation here.
int spmm_device(const daspmm_csr* h, int kernel, int64_t P, int64_t W, const void* B,
                int64_t ldb, int64_t N, void* C, int64_t ldc, unsigned flags, cudaStream_t s,
                int* chunk_scratch) {
    if (h->M == 0 || N == 0) return DASPMM_OK;
    const bool exact = (flags & DASPMM_EXACT) != 0;
    const bool own_scratch = chunk_scratch == nullptr;
    // EB kernels and the lean SR kernels read COO row ids (graph bodies get the array
    // built before capture).
    if (own_scratch && (kernel >= 4 || !(kernel & 1)))
        if (int rc = ensure_coo(h, s)) return rc;
    if (own_scratch && kernel == 0 && !exact)
        if (int rc = ensure_tiles(h, s)) return rc;
    Plan p = plan_spmm(h, kernel, P, W, N, B, ldb, C, ldc, exact);
    if (kernel >= 4 && knobs().pdl) {
        // Programmatic launch after the EB prologue; not inside a stream capture (graph
        // bodies keep plain stream order).
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        p.pdl = cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusNone;
        cudaGetLastError();
    }
    int* chunk_row = chunk_scratch;
    cudaError_t e;
    if (kernel >= 4 && own_scratch) {
        if ((e = scratch_alloc(reinterpret_cast<void**>(&chunk_row),
                               sizeof(int) * size_t(std::max<int64_t>(p.P, 1)), h->device, s)) !=
            cudaSuccess)
            return cuda_fail(e, "scratch_alloc(chunk_row)");
    }
    e = h->dtype == DASPMM_F64 ? run_plan<double>(h, p, W, B, ldb, N, C, ldc, chunk_row, s)
                               : run_plan<float>(h, p, W, B, ldb, N, C, ldc, chunk_row, s);
    if (chunk_row && own_scratch) scratch_free(chunk_row, s);
    if (e == cudaSuccess && knobs().fault) e = inject_fault(h->dtype, C, s);
    if (e == cudaErrorNotSupported)
        return fail(DASPMM_ERR_UNSUPPORTED, std::string("spmm: no instantiation for kernel ") +
                                                kKernelNames[kernel]);
    if (e != cudaSuccess) return cuda_fail(e, kKernelNames[kernel]);
    return DASPMM_OK;
}

int check_call(const daspmm_csr* h, int kernel, int64_t P, int64_t W, int64_t Cb, int b_layout,
               int64_t ldb, int64_t N, int64_t ldc, bool exact) {
    if (!h) return fail(DASPMM_ERR_INVALID_ARG, "spmm: null CSR handle");
    if (kernel < 0 || kernel > 7)
        return fail(DASPMM_ERR_OUT_OF_RANGE, "KernelId index must be 0..7");
    if (int rc = validate_config(P, W, Cb, true)) return rc;
    (void)exact;
    if (N < 0) return fail(DASPMM_ERR_DIMS, "spmm: negative N");
    if (N > (int64_t(1) << 30)) return fail(DASPMM_ERR_UNSUPPORTED, "spmm: N too large");
    if (!((kernel >> 1) & 1) && ldb > (int64_t(1) << 27))  // row pitch in bytes fits int32
        return fail(DASPMM_ERR_UNSUPPORTED, "spmm: ldb too large for row-major B");
    const bool want_cm = (kernel >> 1) & 1;
    if ((b_layout == DASPMM_COL_MAJOR) != want_cm)
        return fail(DASPMM_ERR_LAYOUT, std::string("spmm: kernel ") + kKernelNames[kernel] +
                                           " needs " + (want_cm ? "ColMajor" : "RowMajor") +
                                           " X, got " + (want_cm ? "RowMajor" : "ColMajor"));
    if (want_cm ? ldb < std::max<int64_t>(h->K, 1) : ldb < std::max<int64_t>(N, 1))
        return fail(DASPMM_ERR_DIMS, "spmm: leading dimension of B too small");
    if (ldc < std::max<int64_t>(N, 1)) return fail(DASPMM_ERR_DIMS, "spmm: ldc < N");
    return DASPMM_OK;
}

// ---------------------------------------------------------------- small kernels
template <typename T>
__global__ void k_transpose(const T* __restrict__ in, int64_t rows, int64_t cols, int64_t ldi,
                            T* __restrict__ out, int64_t ldo) {
    // in: rows x cols with leading dim ldi (row-major view); out: cols x rows, ldo.
    __shared__ T tile[32][33];
    const int64_t bx = int64_t(blockIdx.x) * 32;
    // Row tiles are strided over grid.y (which is capped at 65535).
    for (int64_t by = int64_t(blockIdx.y) * 32; by < rows; by += int64_t(gridDim.y) * 32) {
        for (int j = threadIdx.y; j < 32; j += 8) {
            const int64_t r = by + j, c = bx + threadIdx.x;
            if (r < rows && c < cols) tile[j][threadIdx.x] = in[r * ldi + c];
        }
        __syncthreads();
        for (int j = threadIdx.y; j < 32; j += 8) {
            const int64_t r = bx + j, c = by + threadIdx.x;  // out row = in col
            if (r < cols && c < rows) out[r * ldo + c] = tile[threadIdx.x][j];
        }
        __syncthreads();
    }
}

__global__ void k_rebase(const int* __restrict__ in, int64_t n, int base, int* __restrict__ out) {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        out[i] = in[i] - base;
}

template <int W>
__global__ void k_debug_tree(const double* in, double* out, int w) {
    const int lane = threadIdx.x;
    double v = lane < w ? in[lane] : 0.0;
    v = group_tree_sum<W>(group_mask<W>(), v);
    if (lane == 0) out[0] = v;
}

template <int W>
__global__ void k_debug_cond(const double* in, const int64_t* ids, double* out, int w) {
    const int lane = threadIdx.x;
    double v = in[lane];
    const int id = int(ids[lane]);
    v = group_conditional_scan<W>(group_mask<W>(), v, id, lane & (W - 1));
    out[lane] = v;
}

cudaError_t transpose(int dtype, const void* in, int64_t rows, int64_t cols, int64_t ldi,
                      void* out, int64_t ldo, cudaStream_t s) {
    if (rows == 0 || cols == 0) return cudaSuccess;
    if ((cols + 31) / 32 > 0x7fffffff) return cudaErrorInvalidValue;
    dim3 grid(unsigned((cols + 31) / 32), unsigned(std::min<int64_t>((rows + 31) / 32, 65535))),
        block(32, 8);
    if (dtype == DASPMM_F64)
        k_transpose<double><<<grid, block, 0, s>>>(static_cast<const double*>(in), rows, cols, ldi,
                                                   static_cast<double*>(out), ldo);
    else
        k_transpose<float><<<grid, block, 0, s>>>(static_cast<const float*>(in), rows, cols, ldi,
                                                  static_cast<float*>(out), ldo);
    return cudaGetLastError();
}

// Device ingest of a host CSR (types.hpp:56-148): the int64 offsets and columns, as the
// reference stores them, are uploaded once and one pass validates and compacts them to
// the device's int32 layout. bad[0] = first i with offsets[i] < offsets[i-1], bad[1] =
// first element whose column is outside [0, K) (INT64_MAX when none).
__global__ void k_ingest(const int64_t* __restrict__ rp64, const int64_t* __restrict__ ci64,
                         int64_t M, int64_t K, int64_t nnz, int32_t* __restrict__ rp32,
                         int32_t* __restrict__ ci32, unsigned long long* bad) {
    const int64_t n = M + 1 > nnz ? M + 1 : nnz;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        if (i <= M) {
            const int64_t v = rp64[i];
            rp32[i] = int32_t(v);
            if (i > 0 && v < rp64[i - 1]) atomicMin(bad, (unsigned long long)i);
        }
        if (i < nnz) {
            const int64_t c = ci64[i];
            ci32[i] = int32_t(c);
            if (c < 0 || c >= K) atomicMin(bad + 1, (unsigned long long)i);
        }
    }
}

cudaError_t ingest(const int64_t* rp, const int64_t* ci, int64_t M, int64_t K, int64_t nnz,
                   int32_t* rp32, int32_t* ci32, int64_t bad_out[2]) {
    int64_t* d64 = nullptr;
    unsigned long long* d_bad = nullptr;
    const size_t n_rp = size_t(M) + 1, n_ci = size_t(nnz);
    cudaError_t e = cudaMalloc(&d64, sizeof(int64_t) * (n_rp + std::max<size_t>(n_ci, 1)));
    if (e == cudaSuccess) e = cudaMalloc(&d_bad, 2 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemset(d_bad, 0xff, 2 * sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMemcpy(d64, rp, sizeof(int64_t) * n_rp, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && n_ci > 0)
        e = cudaMemcpy(d64 + n_rp, ci, sizeof(int64_t) * n_ci, cudaMemcpyHostToDevice);
    trace_mark("ingest: malloc+h2d int64");
    if (e == cudaSuccess) {
        const int64_t n = std::max<int64_t>(M + 1, nnz);
        const unsigned blocks = unsigned(std::min<int64_t>((n + 255) / 256, 148 * 32));
        k_ingest<<<blocks, 256>>>(d64, d64 + n_rp, M, K, nnz, rp32, ci32, d_bad);
        e = cudaGetLastError();
    }
    unsigned long long hb[2] = {~0ull, ~0ull};
    if (e == cudaSuccess) e = cudaMemcpy(hb, d_bad, sizeof(hb), cudaMemcpyDeviceToHost);
    trace_mark("ingest: k_ingest+d2h");
    cudaFree(d64);
    cudaFree(d_bad);
    trace_mark("ingest: free");
    for (int i = 0; i < 2; ++i)
        bad_out[i] = hb[i] == ~0ull ? INT64_MAX : int64_t(hb[i]);
    return e;
}

}  // namespace daspmm

using namespace daspmm;

// ======================================================================= C ABI
extern "C" {

const char* daspmm_last_error(void) { return g_err.c_str(); }
int daspmm_version(void) { return 100; }
int daspmm_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

static int finish_create(daspmm_csr* h, cudaStream_t s, daspmm_csr** out) {
    int rc = compute_features(h, s);
    trace_mark("create: features+spans");
    if (rc) {
        daspmm_csr_destroy(h);
        return rc;
    }
    *out = h;
    return DASPMM_OK;
}

int daspmm_csr_create_host(int64_t M, int64_t K, int64_t nnz, const int64_t* rp,
                           const int64_t* ci, const void* values, int dtype, daspmm_csr** out) {
    if (!out) return fail(DASPMM_ERR_INVALID_ARG, "csr_create: null out");
    *out = nullptr;
    if (dtype != DASPMM_F32 && dtype != DASPMM_F64)
        return fail(DASPMM_ERR_INVALID_ARG, "csr_create: dtype must be F32 or F64");
    if (M < 0 || K < 0 || nnz < 0) return fail(DASPMM_ERR_INVALID_ARG, "csr_create: negative size");
    if (M >= (int64_t(1) << 31) - 1 || K >= (int64_t(1) << 31) - 1 || nnz >= (int64_t(1) << 31) - 1)
        return fail(DASPMM_ERR_UNSUPPORTED, "csr_create: sizes must be < 2^31 - 1 (int32 device CSR)");
    if (!rp || (nnz > 0 && (!ci || !values)))
        return fail(DASPMM_ERR_INVALID_ARG, "csr_create: null array");
    // types.hpp:96-148 invariants the kernels depend on. The O(1) ends are checked here;
    // monotonicity and the column bounds are checked on the device by the same pass
    // that compacts the int64 arrays to int32 (k_ingest); messages keep this order.
    if (rp[0] != 0) return fail(DASPMM_ERR_INVALID_ARG, "csr_create: row_offsets[0] != 0");
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || daspmm_device_count() == 0) {
        cudaGetLastError();
        return fail(DASPMM_ERR_CUDA, "csr_create: no CUDA device (daspmm has no CPU fallback)");
    }
    trace_mark(nullptr);
    daspmm_csr* h = new daspmm_csr;
    h->M = M;
    h->K = K;
    h->nnz = nnz;
    h->dtype = dtype;
    h->device = dev;
    const size_t es = size_t(elem_size(dtype));
    cudaError_t e;
    if ((e = cudaMalloc(&h->rp, sizeof(int32_t) * (M + 1))) != cudaSuccess ||
        (e = cudaMalloc(&h->ci, sizeof(int32_t) * std::max<int64_t>(nnz, 1))) != cudaSuccess ||
        (e = cudaMalloc(&h->va, es * std::max<int64_t>(nnz, 1))) != cudaSuccess) {
        daspmm_csr_destroy(h);
        return cuda_fail(e, "csr_create: cudaMalloc");
    }
    trace_mark("create_host: malloc");
    int64_t bad[2] = {INT64_MAX, INT64_MAX};
    if ((e = ingest(rp, ci, M, K, nnz, h->rp, h->ci, bad)) != cudaSuccess ||
        (nnz > 0 && (e = cudaMemcpy(h->va, values, es * nnz, cudaMemcpyHostToDevice)) != cudaSuccess)) {
        daspmm_csr_destroy(h);
        return cuda_fail(e, "csr_create: upload");
    }
    trace_mark("create_host: ingest+values");
    std::string msg;
    if (bad[0] != INT64_MAX)
        msg = "csr_create: row_offsets nondecreasing violated at index " + std::to_string(bad[0]);
    else if (rp[M] != nnz)
        msg = "csr_create: row_offsets[num_rows] != nnz";
    else if (bad[1] != INT64_MAX)
        msg = "csr_create: col index bound violated at index " + std::to_string(bad[1]);
    if (!msg.empty()) {
        daspmm_csr_destroy(h);
        return fail(DASPMM_ERR_INVALID_ARG, msg);
    }
    return finish_create(h, 0, out);
}

int daspmm_csr_create_device(int64_t M, int64_t K, int64_t nnz, const int32_t* d_rp,
                             const int32_t* d_ci, const void* d_va, int dtype, int copy,
                             daspmm_stream stream, daspmm_csr** out) {
    if (!out) return fail(DASPMM_ERR_INVALID_ARG, "csr_create: null out");
    *out = nullptr;
    if (dtype != DASPMM_F32 && dtype != DASPMM_F64)
        return fail(DASPMM_ERR_INVALID_ARG, "csr_create: dtype must be F32 or F64");
    if (M < 0 || K < 0 || nnz < 0 || M >= (int64_t(1) << 31) - 1 || K >= (int64_t(1) << 31) - 1 ||
        nnz >= (int64_t(1) << 31) - 1)
        return fail(DASPMM_ERR_INVALID_ARG, "csr_create: sizes must be in [0, 2^31 - 1)");
    if (!d_rp || (nnz > 0 && (!d_ci || !d_va)))
        return fail(DASPMM_ERR_INVALID_ARG, "csr_create: null array");
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return cuda_fail(cudaGetLastError(), "csr_create");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    daspmm_csr* h = new daspmm_csr;
    h->M = M;
    h->K = K;
    h->nnz = nnz;
    h->dtype = dtype;
    h->device = dev;
    if (!copy) {
        h->owns = false;
        h->rp = const_cast<int32_t*>(d_rp);
        h->ci = const_cast<int32_t*>(d_ci);
        h->va = const_cast<void*>(d_va);
    } else {
        const size_t es = size_t(elem_size(dtype));
        cudaError_t e;
        if ((e = cudaMalloc(&h->rp, sizeof(int32_t) * (M + 1))) != cudaSuccess ||
            (e = cudaMalloc(&h->ci, sizeof(int32_t) * std::max<int64_t>(nnz, 1))) != cudaSuccess ||
            (e = cudaMalloc(&h->va, es * std::max<int64_t>(nnz, 1))) != cudaSuccess) {
            daspmm_csr_destroy(h);
            return cuda_fail(e, "csr_create: cudaMalloc");
        }
        e = cudaMemcpyAsync(h->rp, d_rp, sizeof(int32_t) * (M + 1), cudaMemcpyDeviceToDevice, s);
        if (e == cudaSuccess && nnz > 0)
            e = cudaMemcpyAsync(h->ci, d_ci, sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice, s);
        if (e == cudaSuccess && nnz > 0)
            e = cudaMemcpyAsync(h->va, d_va, es * nnz, cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) {
            daspmm_csr_destroy(h);
            return cuda_fail(e, "csr_create: copy");
        }
    }
    return finish_create(h, s, out);
}

int daspmm_csr_create_panel(const daspmm_csr* full, int64_t r0, int64_t r1, daspmm_stream stream,
                            daspmm_csr** out) {
    if (!full || !out) return fail(DASPMM_ERR_INVALID_ARG, "csr_create_panel: null argument");
    if (r0 < 0 || r1 < r0 || r1 > full->M)
        return fail(DASPMM_ERR_OUT_OF_RANGE, "csr_create_panel: bad row range");
    DeviceGuard g(full->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int32_t ends[2] = {0, 0};
    cudaError_t e = cudaMemcpyAsync(&ends[0], full->rp + r0, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(&ends[1], full->rp + r1, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return cuda_fail(e, "csr_create_panel");
    const int64_t M = r1 - r0, nnz = int64_t(ends[1]) - ends[0];
    daspmm_csr* h = new daspmm_csr;
    h->M = M;
    h->K = full->K;
    h->nnz = nnz;
    h->dtype = full->dtype;
    h->device = full->device;
    const size_t es = size_t(elem_size(full->dtype));
    if ((e = cudaMalloc(&h->rp, sizeof(int32_t) * (M + 1))) != cudaSuccess ||
        (e = cudaMalloc(&h->ci, sizeof(int32_t) * std::max<int64_t>(nnz, 1))) != cudaSuccess ||
        (e = cudaMalloc(&h->va, es * std::max<int64_t>(nnz, 1))) != cudaSuccess) {
        daspmm_csr_destroy(h);
        return cuda_fail(e, "csr_create_panel: cudaMalloc");
    }
    k_rebase<<<int(std::min<int64_t>((M + 256) / 256, 4096)), 256, 0, s>>>(full->rp + r0, M + 1,
                                                                          ends[0], h->rp);
    e = cudaGetLastError();
    if (e == cudaSuccess && nnz > 0)
        e = cudaMemcpyAsync(h->ci, full->ci + ends[0], sizeof(int32_t) * nnz, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess && nnz > 0)
        e = cudaMemcpyAsync(h->va, static_cast<const char*>(full->va) + es * ends[0], es * nnz,
                            cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) {
        daspmm_csr_destroy(h);
        return cuda_fail(e, "csr_create_panel: copy");
    }
    return finish_create(h, s, out);
}

int daspmm_csr_values_updated(daspmm_csr* h) {
    if (!h) return fail(DASPMM_ERR_INVALID_ARG, "csr_values_updated: null handle");
    DeviceGuard g(h->device);
    cudaError_t e = cudaDeviceSynchronize();  // no kernel may still read the old tiles
    if (e != cudaSuccess) return cuda_fail(e, "csr_values_updated");
    std::lock_guard<std::mutex> lk(h->mu);
    cudaFree(h->tile_off);
    cudaFree(h->tile_c0);
    cudaFree(h->tile_val);
    h->tile_off = h->tile_c0 = nullptr;
    h->tile_val = nullptr;
    h->n_pan = 0;
    h->tile_state.store(0, std::memory_order_release);
    return DASPMM_OK;
}

int daspmm_csr_destroy(daspmm_csr* h) {
    if (!h) return DASPMM_OK;
    graph_cache_free(h);
    for (auto& e : h->panels) daspmm_csr_destroy(e.h);
    h->panels.clear();
    if (h->owns) {
        cudaFree(h->rp);
        cudaFree(h->ci);
        cudaFree(h->va);
    }
    cudaFree(h->empty_rows);
    cudaFree(h->d_feat);
    cudaFree(h->coo_rows);
    cudaFree(h->spans);
    cudaFree(h->tile_off);
    cudaFree(h->tile_c0);
    cudaFree(h->tile_val);
    delete h;
    return DASPMM_OK;
}

int daspmm_csr_info(const daspmm_csr* h, int64_t* M, int64_t* K, int64_t* nnz, int* dtype,
                    int64_t* empty_rows, int64_t* cols_touched) {
    if (!h) return fail(DASPMM_ERR_INVALID_ARG, "csr_info: null handle");
    if (M) *M = h->M;
    if (K) *K = h->K;
    if (nnz) *nnz = h->nnz;
    if (dtype) *dtype = h->dtype;
    if (empty_rows) *empty_rows = h->n_empty;
    if (cols_touched) *cols_touched = h->cols_touched;
    return DASPMM_OK;
}

int daspmm_csr_device_arrays(const daspmm_csr* h, const int32_t** rp, const int32_t** ci,
                             const void** va) {
    if (!h) return fail(DASPMM_ERR_INVALID_ARG, "csr_device_arrays: null handle");
    if (rp) *rp = h->rp;
    if (ci) *ci = h->ci;
    if (va) *va = h->va;
    return DASPMM_OK;
}

int daspmm_spmm(const daspmm_csr* h, int kernel, int64_t P, int64_t W, int64_t Cb, const void* d_B,
                int b_layout, int64_t ldb, int64_t N, void* d_C, int64_t ldc, unsigned flags,
                daspmm_stream stream) {
    if (int rc = check_call(h, kernel, P, W, Cb, b_layout, ldb, N, ldc, flags & DASPMM_EXACT))
        return rc;
    DeviceGuard g(h->device);
    return spmm_device(h, kernel, P, W, d_B, ldb, N, d_C, ldc, flags,
                       static_cast<cudaStream_t>(stream), nullptr);
}

int daspmm_spmm_host(const daspmm_csr* h, int kernel, int64_t P, int64_t W, int64_t Cb,
                     const void* B, int b_layout, int64_t N, void* C, unsigned flags) {
    const int64_t ldb = b_layout == DASPMM_COL_MAJOR ? std::max<int64_t>(h ? h->K : 1, 1)
                                                     : std::max<int64_t>(N, 1);
    if (int rc = check_call(h, kernel, P, W, Cb, b_layout, ldb, N, std::max<int64_t>(N, 1),
                            flags & DASPMM_EXACT))
        return rc;
    if (h->M == 0 || N == 0) return DASPMM_OK;
    DeviceGuard g(h->device);
    const size_t es = size_t(elem_size(h->dtype));
    const size_t bbytes = es * size_t(h->K) * size_t(N), cbytes = es * size_t(h->M) * size_t(N);
    void *dB = nullptr, *dC = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc(&dB, std::max<size_t>(bbytes, 16))) != cudaSuccess)
        return cuda_fail(e, "spmm_host: cudaMalloc(B)");
    if ((e = cudaMalloc(&dC, std::max<size_t>(cbytes, 16))) != cudaSuccess) {
        cudaFree(dB);
        return cuda_fail(e, "spmm_host: cudaMalloc(C)");
    }
    int rc = DASPMM_OK;
    if ((e = cudaMemcpy(dB, B, bbytes, cudaMemcpyHostToDevice)) != cudaSuccess)
        rc = cuda_fail(e, "spmm_host: upload B");
    if (rc == DASPMM_OK) rc = spmm_device(h, kernel, P, W, dB, ldb, N, dC, N, flags, 0, nullptr);
    if (rc == DASPMM_OK) {
        e = cudaMemcpy(C, dC, cbytes, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) rc = cuda_fail(e, "spmm_host");
    }
    cudaFree(dB);
    cudaFree(dC);
    return rc;
}

int daspmm_spmm_auto_layout(const daspmm_csr* h, int kernel, int64_t P, int64_t W, int64_t Cb,
                            const void* d_B, int b_layout, int64_t ldb, int64_t N, void* d_C,
                            int64_t ldc, unsigned flags, daspmm_stream stream) {
    if (!h) return fail(DASPMM_ERR_INVALID_ARG, "spmm: null CSR handle");
    if (kernel < 0 || kernel > 7)
        return fail(DASPMM_ERR_OUT_OF_RANGE, "KernelId index must be 0..7");
    const int want = ((kernel >> 1) & 1) ? DASPMM_COL_MAJOR : DASPMM_ROW_MAJOR;
    if (want == b_layout)
        return daspmm_spmm(h, kernel, P, W, Cb, d_B, b_layout, ldb, N, d_C, ldc, flags, stream);
    if (b_layout == DASPMM_COL_MAJOR ? ldb < std::max<int64_t>(h->K, 1)
                                     : ldb < std::max<int64_t>(N, 1))
        return fail(DASPMM_ERR_DIMS, "spmm: leading dimension of B too small");
    DeviceGuard g(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t es = size_t(elem_size(h->dtype));
    void* t = nullptr;
    cudaError_t e = scratch_alloc(&t, std::max<size_t>(es * size_t(h->K) * size_t(N), 16), h->device, s);
    if (e != cudaSuccess) return cuda_fail(e, "spmm_auto_layout: scratch_alloc");
    int64_t ldt;
    if (b_layout == DASPMM_ROW_MAJOR) {  // K x N (ldb) -> ColMajor: N x K rows, ld K
        ldt = std::max<int64_t>(h->K, 1);
        e = transpose(h->dtype, d_B, h->K, N, ldb, t, ldt, s);
    } else {  // ColMajor (N rows of K, ld ldb) -> RowMajor K x N
        ldt = std::max<int64_t>(N, 1);
        e = transpose(h->dtype, d_B, N, h->K, ldb, t, ldt, s);
    }
    int rc = e == cudaSuccess ? daspmm_spmm(h, kernel, P, W, Cb, t, want, ldt, N, d_C, ldc, flags,
                                            stream)
                              : cuda_fail(e, "spmm_auto_layout: transpose");
    scratch_free(t, s);
    return rc;
}

int daspmm_extract_features(const daspmm_csr* h, int64_t n_cols, int64_t* nnz, int64_t* mat_size,
                            double* std_row) {
    (void)n_cols;
    if (!h) return fail(DASPMM_ERR_INVALID_ARG, "extract_features: null handle");
    if (h->M == 0)
        return fail(DASPMM_ERR_INVALID_ARG, "extract_features: matrix has no rows to summarize");
    double s = 0.0;
    if (int rc = exact_std(const_cast<daspmm_csr*>(h), &s)) return rc;
    if (nnz) *nnz = h->nnz;
    if (mat_size) *mat_size = h->M;
    if (std_row) *std_row = s;
    return DASPMM_OK;
}

int daspmm_partition(const daspmm_csr* h, int64_t p, int64_t* begin, int64_t* end, int64_t* row) {
    if (!h) return fail(DASPMM_ERR_INVALID_ARG, "partition: null handle");
    if (p < 1) return fail(DASPMM_ERR_INVALID_ARG, "partition_elements: need p >= 1");
    DeviceGuard g(h->device);
    int* d_row = nullptr;
    cudaError_t e = cudaMalloc(&d_row, sizeof(int) * size_t(p));
    if (e != cudaSuccess) return cuda_fail(e, "partition: cudaMalloc");
    // The EB prologue kernel with no output rows to zero (C = null, N = 0).
    e = launch_eb_prep<float>(h->rp, int(h->M), h->nnz, p, d_row, nullptr, 0, 0, nullptr, 0,
                              nullptr, 0);
    std::vector<int> rows(size_t(p), 0);
    if (e == cudaSuccess)
        e = cudaMemcpy(rows.data(), d_row, sizeof(int) * size_t(p), cudaMemcpyDeviceToHost);
    cudaFree(d_row);
    if (e != cudaSuccess) return cuda_fail(e, "partition");
    const int64_t base = h->nnz / p, extra = h->nnz % p;
    int64_t start = 0;
    for (int64_t i = 0; i < p; ++i) {
        const int64_t size = base + (i < extra ? 1 : 0);
        if (begin) begin[i] = start;
        if (end) end[i] = start + size;
        if (row) row[i] = rows[size_t(i)];
        start += size;
    }
    return DASPMM_OK;
}

int daspmm_reload_env(void) {
    const Knobs k = read_knobs();
    std::lock_guard<std::mutex> lk(g_knobs_mu);
    g_knobs = k;
    return DASPMM_OK;
}

int daspmm_spmm_rows_to(const daspmm_csr* h, const void* B, int64_t ldb, int64_t N,
                        void* const* C, int n_dst, int64_t ldc, daspmm_stream stream) {
    if (!h || !C || n_dst < 1) return fail(DASPMM_ERR_INVALID_ARG, "spmm_rows_to: null argument");
    if (n_dst > 1 + kMaxExtraDst)
        return fail(DASPMM_ERR_UNSUPPORTED, "spmm_rows_to: at most 8 destinations");
    if (h->dtype != DASPMM_F32)
        return fail(DASPMM_ERR_UNSUPPORTED, "spmm_rows_to: float32 handles only");
    for (int d = 0; d < n_dst; ++d)
        if (!C[d]) return fail(DASPMM_ERR_INVALID_ARG, "spmm_rows_to: null destination");
    if (int rc = check_call(h, 0, 0, 8, 8, DASPMM_ROW_MAJOR, ldb, N, ldc, false)) return rc;
    if (h->M == 0 || N == 0) return DASPMM_OK;
    DeviceGuard g(h->device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // RB+RM+SR through the shuffle-broadcast row walk (k_rb_sr): every row is owned by
    // exactly one group, so the replicated epilogue needs plain stores only. The vector
    // width must suit every destination, so the plan checks the least aligned one.
    // OR of all destination addresses: its lowest set bit is the minimum alignment.
    uintptr_t any = 0;
    for (int d = 0; d < n_dst; ++d) any |= reinterpret_cast<uintptr_t>(C[d]);
    const void* worst = reinterpret_cast<const void*>(any);
    Plan p = plan_spmm(h, 0, 0, 8, N, B, ldb, worst, ldc, false, /*base_only=*/true);
    p.repl = true;
    cudaError_t e = run_plan<float>(h, p, 8, B, ldb, N, C[0], ldc, nullptr, s, C + 1, n_dst - 1);
    if (e == cudaErrorNotSupported)
        return fail(DASPMM_ERR_UNSUPPORTED, "spmm_rows_to: no instantiation for this shape");
    if (e != cudaSuccess) return cuda_fail(e, "spmm_rows_to");
    return DASPMM_OK;
}

int daspmm_plan_info(const daspmm_csr* h, int kernel, int64_t N, const void* B, int64_t ldb,
                     const void* C, int64_t ldc, unsigned flags, int* variant, int64_t* param) {
    if (!h || !variant || !param) return fail(DASPMM_ERR_INVALID_ARG, "plan_info: null argument");
    if (kernel < 0 || kernel > 7) return fail(DASPMM_ERR_OUT_OF_RANGE, "KernelId index must be 0..7");
    DeviceGuard g(h->device);
    if (int rc = ensure_coo(h, 0)) return rc;
    if (kernel == 0 && !(flags & DASPMM_EXACT))
        if (int rc = ensure_tiles(h, 0)) return rc;
    const Plan p = plan_spmm(h, kernel, 0, 8, N, B, ldb, C, ldc, (flags & DASPMM_EXACT) != 0);
    *variant = p.cm_rows ? 7 : p.tile ? 6 : p.win_rows > 0 ? 1 : p.cta ? 2 : p.thr ? 3 : p.lean ? 4 : p.tma ? 5 : 0;
    *param = p.cm_rows ? p.L : p.tile ? p.tile_rl
             : p.win_rows > 0 ? p.win_rows : (p.thr || p.tma || (p.lean && kernel >= 4)) ? p.sub
             : p.lean ? p.rpg : int64_t(p.grid.y);
    return DASPMM_OK;
}

int daspmm_debug_std_chain(const daspmm_csr* h, double* out) {
    if (!h || !out) return fail(DASPMM_ERR_INVALID_ARG, "debug_std_chain: null argument");
    if (h->M <= 0) return fail(DASPMM_ERR_INVALID_ARG, "extract_features: matrix has no rows to summarize");
    return std_chain(h, out);
}

int daspmm_debug_tree_reduce_f64(const double* values, int64_t w, double* out) {
    if (w < 1 || w > 32 || !is_pow2(w))
        return fail(DASPMM_ERR_INVALID_ARG, "tree_reduce: length must be a power of two <= 32");
    double *d_in = nullptr, *d_out = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc(&d_in, sizeof(double) * 32)) != cudaSuccess ||
        (e = cudaMalloc(&d_out, sizeof(double))) != cudaSuccess ||
        (e = cudaMemcpy(d_in, values, sizeof(double) * w, cudaMemcpyHostToDevice)) != cudaSuccess) {
        cudaFree(d_in);
        cudaFree(d_out);
        return cuda_fail(e, "debug_tree_reduce");
    }
    switch (w) {
        case 1: k_debug_tree<1><<<1, 32>>>(d_in, d_out, int(w)); break;
        case 2: k_debug_tree<2><<<1, 32>>>(d_in, d_out, int(w)); break;
        case 4: k_debug_tree<4><<<1, 32>>>(d_in, d_out, int(w)); break;
        case 8: k_debug_tree<8><<<1, 32>>>(d_in, d_out, int(w)); break;
        case 16: k_debug_tree<16><<<1, 32>>>(d_in, d_out, int(w)); break;
        default: k_debug_tree<32><<<1, 32>>>(d_in, d_out, int(w)); break;
    }
    e = cudaMemcpy(out, d_out, sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(d_in);
    cudaFree(d_out);
    return e == cudaSuccess ? DASPMM_OK : cuda_fail(e, "debug_tree_reduce");
}

int daspmm_debug_conditional_scan_f64(const double* values, const int64_t* ids, int64_t w,
                                      double* out) {
    if (w < 1 || w > 32 || !is_pow2(w))
        return fail(DASPMM_ERR_INVALID_ARG, "conditional_scan: length must be a power of two <= 32");
    double *d_in = nullptr, *d_out = nullptr;
    int64_t* d_ids = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc(&d_in, sizeof(double) * 32)) != cudaSuccess ||
        (e = cudaMalloc(&d_out, sizeof(double) * 32)) != cudaSuccess ||
        (e = cudaMalloc(&d_ids, sizeof(int64_t) * 32)) != cudaSuccess ||
        (e = cudaMemset(d_in, 0, sizeof(double) * 32)) != cudaSuccess ||
        (e = cudaMemset(d_ids, 0xff, sizeof(int64_t) * 32)) != cudaSuccess ||
        (e = cudaMemcpy(d_in, values, sizeof(double) * w, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaMemcpy(d_ids, ids, sizeof(int64_t) * w, cudaMemcpyHostToDevice)) != cudaSuccess) {
        cudaFree(d_in);
        cudaFree(d_out);
        cudaFree(d_ids);
        return cuda_fail(e, "debug_conditional_scan");
    }
    switch (w) {
        case 1: k_debug_cond<1><<<1, 32>>>(d_in, d_ids, d_out, int(w)); break;
        case 2: k_debug_cond<2><<<1, 32>>>(d_in, d_ids, d_out, int(w)); break;
        case 4: k_debug_cond<4><<<1, 32>>>(d_in, d_ids, d_out, int(w)); break;
        case 8: k_debug_cond<8><<<1, 32>>>(d_in, d_ids, d_out, int(w)); break;
        case 16: k_debug_cond<16><<<1, 32>>>(d_in, d_ids, d_out, int(w)); break;
        default: k_debug_cond<32><<<1, 32>>>(d_in, d_ids, d_out, int(w)); break;
    }
    e = cudaMemcpy(out, d_out, sizeof(double) * w, cudaMemcpyDeviceToHost);
    cudaFree(d_in);
    cudaFree(d_out);
    cudaFree(d_ids);
    return e == cudaSuccess ? DASPMM_OK : cuda_fail(e, "debug_conditional_scan");
}

}  // extern "C"
