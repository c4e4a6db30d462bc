/*
 * daspmm — C ABI of the B200-native DA-SpMM library (libdaspmm.so).
 *
 * Drop-in boundary for the spmmkit hot path (reference: /root/reference/proj/include/
 * spmmkit). The reference exposes header-only C++ templates; this C ABI is what those
 * templates become when the compute moves to a B200: plain pointers and sizes, int
 * status codes instead of exceptions, opaque device-resident handles. The C++ shim in
 * include/spmmkit/ maps it back onto the reference's exact C++ signatures and
 * exception types (see INTEGRATION.md for the ctypes / C++ bindings).
 *
 * All compute runs as hand-written sm_100a CUDA kernels. There is no CPU fallback:
 * every entry point that computes fails with DASPMM_ERR_CUDA when no device exists.
 *
 * Threading: handles are immutable after creation (feature caches are filled under a
 * per-handle lock); calls are stream-ordered and re-entrant across streams.
 */
#ifndef DASPMM_H_
#define DASPMM_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct daspmm_csr daspmm_csr;     /* device CSR (int32 offsets/cols, f32|f64 values) */
typedef struct daspmm_model daspmm_model; /* selector tree ensemble (host + device copy)   */
typedef void* daspmm_stream;              /* cudaStream_t; NULL = legacy default stream   */

/* Status codes. The C++ shim rethrows them as the reference's exception types:
 *   INVALID_CONFIG, DIMS, LAYOUT, INVALID_ARG -> std::invalid_argument
 *       (spmm.hpp:197-209, features.hpp:24-25, selector.hpp:26-28)
 *   OUT_OF_RANGE                              -> std::out_of_range (kernel_id.hpp:30,
 *                                                partition.hpp:36-39)
 *   MODEL_FORMAT                              -> spmmkit::ModelFormatError (gbdt.hpp:301-303)
 *   CUDA, NCCL, UNSUPPORTED                   -> std::runtime_error                     */
enum {
    DASPMM_OK = 0,
    DASPMM_ERR_INVALID_CONFIG = 1,
    DASPMM_ERR_DIMS = 2,
    DASPMM_ERR_LAYOUT = 3,
    DASPMM_ERR_INVALID_ARG = 4,
    DASPMM_ERR_OUT_OF_RANGE = 5,
    DASPMM_ERR_MODEL_FORMAT = 6,
    DASPMM_ERR_CUDA = 7,
    DASPMM_ERR_NCCL = 8,
    DASPMM_ERR_UNSUPPORTED = 9
};

enum { DASPMM_F32 = 0, DASPMM_F64 = 1 };          /* value type T ∈ {float, double} */
enum { DASPMM_ROW_MAJOR = 0, DASPMM_COL_MAJOR = 1 }; /* Layout, types.hpp:16          */

/* Call flags. */
enum {
    /* Reference evaluation order with no FMA contraction: results equal the
     * reference's spmm() bit for bit (RB kernels always; EB kernels on rows owned by
     * one chunk, with P honoured as the chunk count). Default: fused multiply-add,
     * library-chosen EB chunking, tolerance parity. */
    DASPMM_EXACT = 1u,
    /* daspmm_spmm_selected only: run the device selector (ensemble walk) and the SWITCH
     * dispatch on this call even when the choice for (matrix, model, N, hw) is already
     * known — measures the uncached DA-SpMM overhead. */
    DASPMM_RESELECT = 2u,
    /* daspmm_spmm_selected only: when the chosen design point needs the other layout of
     * B, convert B on the device first, as the reference's spmm_auto_layout does
     * (spmm.hpp:275-281). Default: run the chosen point's layout twin on B as given (same
     * M- and K-loop choices; for SR the same fmaf sequence, so the same bits) and save
     * the O(K N) conversion — the selector is trained on kernels timed with B already in
     * their layout, so the conversion is not part of what it weighs. */
    DASPMM_CONVERT_LAYOUT = 4u
};

/* Human-readable message for the last failing call on this thread. */
const char* daspmm_last_error(void);
/* 100 * major + minor. */
int daspmm_version(void);
/* Number of CUDA devices visible (0 on a GPU-less host). */
int daspmm_device_count(void);

/* ------------------------------------------------------------------ CSR handles */

/* Uploads a host CSR — replaces passing `const CsrMatrix<T>&` into spmm()
 * (types.hpp:28-35, spmm.hpp:194-196). Offsets/columns are int64 as in the
 * reference; they are validated (types.hpp:96-148 invariants that the kernels rely
 * on: offsets[0]==0, nondecreasing, offsets[M]==nnz, 0<=col<K) and compacted to
 * int32 on the device. Requires nnz < 2^31 and M, K < 2^31. Also computes the
 * selector features (features.hpp:21-41) and the empty-row list on the device. */
int daspmm_csr_create_host(int64_t num_rows, int64_t num_cols, int64_t nnz,
                           const int64_t* row_offsets, const int64_t* col_indices,
                           const void* values, int dtype, daspmm_csr** out);

/* Adopts (copy == 0: borrows, caller keeps ownership) or copies (copy != 0) a CSR
 * already in device memory with int32 offsets and columns. A borrowed structure must not
 * change while the handle lives (features, empty rows, column windows and COO row ids
 * are derived from it); values may change in place if the caller then calls
 * daspmm_csr_values_updated (the row-panel tiles hold a copy of the values). */
int daspmm_csr_create_device(int64_t num_rows, int64_t num_cols, int64_t nnz,
                             const int32_t* d_row_offsets, const int32_t* d_col_indices,
                             const void* d_values, int dtype, int copy, daspmm_stream stream,
                             daspmm_csr** out);

/* CsrMatrix::from_coo on the device (types.hpp:54-90): triplets (int64 row, int64 col,
 * value) in device memory, any order; out-of-bounds coordinates fail with the
 * reference's message; duplicate coordinates are summed (left to right in input order —
 * the reference's std::sort leaves their order unspecified; inputs without duplicates
 * give exactly from_coo's CSR). The handle owns the built arrays. Stream-ordered, with
 * two host synchronisations (bounds verdict, output size). */
int daspmm_csr_create_coo_device(int64_t num_rows, int64_t num_cols, int64_t n_triplets,
                                 const int64_t* d_rows, const int64_t* d_cols,
                                 const void* d_values, int dtype, daspmm_stream stream,
                                 daspmm_csr** out);

/* The values of a borrowed CSR were changed in place (same structure): drops the
 * handle's derived copies of the values (row-panel tiles, rebuilt on the next call that
 * uses them). Synchronises the handle's device first. */
int daspmm_csr_values_updated(daspmm_csr* csr);

/* Row panel [r0, r1) of an existing handle (offsets rebased, columns shared) — the
 * multi-GPU layer's unit. Device-to-device copy on `stream`. */
int daspmm_csr_create_panel(const daspmm_csr* full, int64_t r0, int64_t r1,
                            daspmm_stream stream, daspmm_csr** out);

int daspmm_csr_destroy(daspmm_csr* csr);

/* num_rows, num_cols, nnz, dtype, number of empty rows, distinct columns touched
 * (K_touched, for the compulsory-byte roofline). Any pointer may be NULL. */
int daspmm_csr_info(const daspmm_csr* csr, int64_t* num_rows, int64_t* num_cols,
                    int64_t* nnz, int* dtype, int64_t* empty_rows, int64_t* cols_touched);

/* Device pointers of the handle's arrays (int32 offsets, int32 columns, values). */
int daspmm_csr_device_arrays(const daspmm_csr* csr, const int32_t** d_row_offsets,
                             const int32_t** d_col_indices, const void** d_values);

/* ---------------------------------------------------------------- design space */

/* spmm() — spmm.hpp:194-271, device-resident operands.
 *   kernel      0..7, KernelId::index() = 4m + 2n + k (kernel_id.hpp:25-27)
 *   P, W, Cb    WorkerConfig (worker.hpp:18-40): validated as the reference does
 *               (P >= 1 or 0 = library choice, W power of two in [2, 1024], Cb >= 1;
 *               W > 32 runs one CTA of W threads per group — the reference accepts any
 *               power of two, widths above 1024 return DASPMM_ERR_UNSUPPORTED).
 *               W is the PR reduction width; P the EB chunk count when honoured
 *               (P > 0, or always in DASPMM_EXACT mode); Cb does not change results.
 *   d_B         K x N operand; b_layout must equal the kernel's N-loop choice
 *               (RM kernels: DASPMM_ROW_MAJOR, ldb >= N; CM kernels: DASPMM_COL_MAJOR,
 *               ldb >= K), else DASPMM_ERR_LAYOUT (spmm.hpp:206-209).
 *   d_C         M x N row-major output, ldc >= N; every element is written.
 * Asynchronous on `stream`. */
int daspmm_spmm(const daspmm_csr* csr, int kernel, int64_t P, int64_t W, int64_t Cb,
                const void* d_B, int b_layout, int64_t ldb, int64_t N, void* d_C, int64_t ldc,
                unsigned flags, daspmm_stream stream);

/* Same call with HOST operands (dense B in `b_layout` with leading dim = N or K, C
 * row-major M x N): uploads B, runs, downloads C, synchronises. This is the value-
 * semantics path the C++ shim's spmm() uses. */
int daspmm_spmm_host(const daspmm_csr* csr, int kernel, int64_t P, int64_t W, int64_t Cb,
                     const void* B, int b_layout, int64_t N, void* C, unsigned flags);

/* spmm_auto_layout — spmm.hpp:275-281: converts B to the kernel's layout on the
 * device when needed (scratch is stream-ordered), then runs. */
int daspmm_spmm_auto_layout(const daspmm_csr* csr, int kernel, int64_t P, int64_t W,
                            int64_t Cb, const void* d_B, int b_layout, int64_t ldb, int64_t N,
                            void* d_C, int64_t ldc, unsigned flags, daspmm_stream stream);

/* ------------------------------------------------------------------- features */

/* extract_features — features.hpp:21-41. std_row has the reference's bits (its
 * sequential double sum is replayed on the device once per handle and cached).
 * DASPMM_ERR_INVALID_ARG when num_rows == 0. */
int daspmm_extract_features(const daspmm_csr* csr, int64_t n_cols, int64_t* nnz,
                            int64_t* mat_size, double* std_row);

/* partition_elements — partition.hpp:45-64, computed by the device partition kernel
 * (the same kernel the EB path uses). begin/end/row are host arrays of length p. */
int daspmm_partition(const daspmm_csr* csr, int64_t p, int64_t* begin, int64_t* end,
                     int64_t* row);

/* ------------------------------------------------------------------- selector */

/* load_selector — selector.hpp:119-132 + load_model gbdt.hpp:371-453 (text v1).
 * Parses on the host, flattens and uploads the ensemble once. */
int daspmm_model_parse(const char* text, size_t len, daspmm_model** out);
int daspmm_model_destroy(daspmm_model* model);
/* classes, features, rounds, uses_hardware. */
int daspmm_model_info(const daspmm_model* model, int* num_classes, int* num_features,
                      int* num_rounds, int* uses_hardware);

/* predict_kernel — selector.hpp:62-65 evaluated on the HOST from given features
 * (encode_features selector.hpp:19-33 + predict_class gbdt.hpp:67-77). hw < 0 = no
 * hardware_id. Reference for the device selector's bit-exactness check. */
int daspmm_model_predict_host(const daspmm_model* model, int64_t nnz, int64_t mat_size,
                              double std_row, int64_t n_cols, int64_t hw, int* kernel);

/* Device selector: features of `csr` (cached on the device) + N -> kernel id written
 * to d_kernel (device int). No host round trip; the decision equals
 * daspmm_model_predict_host on extract_features() bit for bit. */
int daspmm_select(const daspmm_csr* csr, const daspmm_model* model, int64_t n_cols,
                  int64_t hw, int* d_kernel, daspmm_stream stream);

/* DA-SpMM: device selector + device-side dispatch (CUDA graph with a SWITCH
 * conditional node; the selector kernel sets the branch). B may be in either
 * layout; a choice that needs the other layout runs its layout twin on B as given,
 * or, with DASPMM_CONVERT_LAYOUT, converts B on the device first as spmm_auto_layout
 * does. d_kernel reports the selector's choice. W/Cb from make_config(kernel, N) defaults
 * (worker.hpp:47-55) unless W > 0. Optional d_kernel receives the choice.
 * Caching: the choice depends only on (matrix, model, N, hw). Until the device has
 * published it, calls run the graph (at most 4 instantiated graphs per handle, LRU);
 * afterwards every call with that key — any B, C or stream — launches the chosen kernel
 * directly (DASPMM_RESELECT forces the graph path). Memory stays bounded however many
 * distinct operand buffers are used. Models with more than 8 classes are rejected with
 * DASPMM_ERR_OUT_OF_RANGE (KernelId::from_index, kernel_id.hpp:30). */
int daspmm_spmm_selected(const daspmm_csr* csr, const daspmm_model* model, int64_t hw,
                         const void* d_B, int b_layout, int64_t ldb, int64_t N, void* d_C,
                         int64_t ldc, int64_t W, unsigned flags, int* d_kernel,
                         daspmm_stream stream);

/* ---------------------------------------------------------------- multi-GPU (§8e)
 * One process per GPU. A communicator wraps NCCL (loaded at run time from
 * libnccl.so.2; DASPMM_ERR_NCCL when absent): rank 0 makes the 128-byte unique id, the
 * caller distributes it (e.g. torch.distributed broadcast), every rank creates its
 * communicator on its current device. */
typedef struct daspmm_comm daspmm_comm;
enum { DASPMM_SPLIT_AUTO = -1, DASPMM_SPLIT_ROWS = 0, DASPMM_SPLIT_COLS = 1 };
int daspmm_comm_unique_id(void* id_out /* 128 bytes */);
int daspmm_comm_create(int nranks, int rank, const void* unique_id, daspmm_comm** out);
int daspmm_comm_destroy(daspmm_comm* comm);
/* Partition of C = A·B over `parts` GPUs. mode DASPMM_SPLIT_ROWS: nnz-balanced row
 * panels, bounds[p] = row holding partition_elements' chunk p start (partition.hpp:
 * 45-64, snapped to row starts, nondecreasing), B replicated; DASPMM_SPLIT_COLS: column
 * slices bounds[p] = floor(N p / parts), A replicated; DASPMM_SPLIT_AUTO: the one with
 * fewer per-GPU compulsory bytes (rows: A/P + B + C/P, cols: A + B/P + C/P). bounds has
 * parts + 1 entries (host). */
int daspmm_multi_plan(const daspmm_csr* csr, int parts, int64_t N, int mode, int* mode_out,
                      int64_t* bounds);
/* The calling rank's exchange-free share of C = A·B by DA-SpMM (device selector on the
 * share), written into its rows / columns of the full M x N row-major d_C; with
 * assemble != 0 the other ranks' shares are then gathered over NCCL (rows: one broadcast
 * per panel in one group, needs ldc == N; cols: pack, all-gather, unpack). `csr` is the
 * full matrix on this rank's device (row panels are built once and cached on it); comm
 * NULL = one rank. Asynchronous on `stream`. */
int daspmm_multi_spmm(daspmm_comm* comm, const daspmm_csr* csr, const daspmm_model* model,
                      int64_t hw, const void* d_B, int64_t ldb, int64_t N, void* d_C, int64_t ldc,
                      int mode, int assemble, int* d_kernel, daspmm_stream stream);
/* Graph-cache occupancy of a handle: instantiated graphs, retired graphs awaiting
 * completion, and known (model, N, hw) decisions. Diagnostics for tests. */
int daspmm_selected_cache_info(const daspmm_csr* csr, int64_t* graphs, int64_t* retired,
                               int64_t* decided);
/* ----------------------------------------------------------- test hooks (device) */

/* The device warp primitives on caller data, for bit-exact checks against
 * tree_reduce (reduce.hpp:46-55) and conditional_reduce (reduce.hpp:57-102).
 * Host arrays in, host arrays out. w is a power of two in [1, 32]. */
int daspmm_debug_tree_reduce_f64(const double* values, int64_t w, double* out);
/* The reference's std_row (features.hpp:27-35) as one dependent chain of double adds on
 * the device: the check for the block-wide exact sum daspmm_extract_features uses. */
int daspmm_debug_std_chain(const daspmm_csr* csr, double* out);
int daspmm_debug_conditional_scan_f64(const double* values, const int64_t* ids, int64_t w,
                                      double* out);

/* RB+RM+SR (kernel 0, fast mode, f32) whose epilogue stores every finished row of C to
 * n_dst destinations d_C[0..n_dst) (1 <= n_dst <= 8, all with leading dimension ldc):
 * with destinations that are the peers' copies of an assembled C (NVLink-mapped
 * symmetric memory), a rank's row-panel SpMM and the all-gather of its panel are one
 * kernel (paper_2202_08556_b200.multi.spmm_rows_allgather). */
int daspmm_spmm_rows_to(const daspmm_csr* csr, const void* d_B, int64_t ldb, int64_t N,
                        void* const* d_C, int n_dst, int64_t ldc, daspmm_stream stream);

/* Re-reads the planner's tuning environment variables (DASPMM_LEAN*, DASPMM_EB_*,
 * DASPMM_RPG, DASPMM_TILE_COLS, DASPMM_WIN, DASPMM_TMA*, fault injection). They are read
 * once at load; tests and tuning sweeps that change them call this afterwards. */
int daspmm_reload_env(void);

/* Which launch variant daspmm_spmm would run for these operands (no launch):
 *   variant 0 = the design point's base kernel (*param = column tiles, grid.y), 1 = RB+SR with the B window staged in
 *   shared memory (*param = rows per CTA panel), 2 = EB+SR with CTA-combined boundary
 *   rows, 3 = EB+SR one-lane staged sub-chunks (*param = pairs per thread), 4 = lean
 *   SR kernel (*param = rows per group for RB, pairs per chunk for EB), 5 = EB+SR with
 *   TMA gather4 B-row fetches (*param = pairs per warp), 6 = RB+RM+SR on the handle's
 *   dense 8-row panel tiles (*param = row lanes per panel: 8 narrow N, 1 wide N), 7 =
 *   RB+CM+SR with lanes over rows (*param = columns per block).
 * Diagnostics for tests and the bench's per-call report. */
int daspmm_plan_info(const daspmm_csr* csr, int kernel, int64_t N, const void* d_B, int64_t ldb,
                     const void* d_C, int64_t ldc, unsigned flags, int* variant, int64_t* param);

#ifdef __cplusplus
}
#endif
#endif /* DASPMM_H_ */
