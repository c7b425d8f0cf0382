/*
 * fglt.h — C-ABI of the B200-native Fast Graphlet Transform (FGlT).
 *
 * This is the drop-in boundary for the reference's hot path
 *   graphlet::transform(const SparseAdjacency&, const TransformOptions&)
 *     (/root/reference/proj/include/graphlet/transform.hpp:22-23,
 *      src/transform.cpp:9-26)
 *   graphlet::raw_frequencies(g, dict, KernelOptions, TransformStats*)
 *     (include/graphlet/kernels.hpp:120-123, src/kernels.cpp:305-419)
 *   graphlet::net_from_raw(raw, U, lenient, threads)
 *     (include/graphlet/conversion.hpp:49-51, src/conversion.cpp:80-116)
 * The reference has no C-ABI; its only bindings are the C++ headers and the
 * pybind11 module (bindings/module.cpp:61-180). Every entry point below is
 * what those callers need, in plain pointers and sizes. INTEGRATION.md shows
 * the ctypes / C++ bindings a maintainer adds on the reference side.
 *
 * Input: a sanitised symmetric 0/1 CSR with int32 indices (row_ptr n+1,
 * col_idx nnz), strictly increasing rows, zero diagonal — the invariants of
 * SparseAdjacency (graph.hpp:38-40). Inputs are borrowed, read-only.
 * Output: raw and net n x k uint64 row-major tables, k = |dictionary|,
 * columns = selected graphlet ids ascending (fields.hpp:10-29), bit-exact
 * with the reference. Outputs are caller-allocated.
 *
 * Return codes are the reference CLI's exit classes (tools/glt.cpp:17-21):
 * 0 ok, 1 parse, 2 structural, 3 overflow, 4 inconsistency, 5 I/O; plus 6 for
 * a CUDA/runtime failure and 7 when no CUDA device is usable (there is no CPU
 * fallback: the call fails loudly).
 */
#ifndef FGLT_H_
#define FGLT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum fglt_code {
  FGLT_OK = 0,
  FGLT_E_PARSE = 1,
  FGLT_E_STRUCTURAL = 2,
  FGLT_E_OVERFLOW = 3,
  FGLT_E_INCONSISTENCY = 4,
  FGLT_E_IO = 5,
  FGLT_E_CUDA = 6,
  FGLT_E_NO_DEVICE = 7
};

/* flags for fglt_transform_csr32 / fglt_ctx_transform */
#define FGLT_INPUT_DEVICE 0x1u  /* row_ptr/col_idx are device pointers   */
#define FGLT_OUTPUT_DEVICE 0x2u /* raw_out/net_out are device pointers   */
#define FGLT_TIMINGS 0x4u       /* fill per-step times (adds event syncs) */

/* Mirrors OverflowError / InconsistencyError (types.hpp:31-51). */
typedef struct fglt_error {
  int32_t code;        /* enum fglt_code */
  int32_t graphlet_id; /* -1 when not applicable */
  int64_t vertex;      /* -1 when not applicable (original vertex id) */
  char msg[256];
  uint64_t order_key;  /* reference failure order (stage, vertex); lowest
                          wins when ranks combine their errors; ~0 = none */
} fglt_error;

#define FGLT_MAX_STEPS 12
#define FGLT_MAX_PHASES 16
/* Mirrors TransformStats (kernels.hpp:105-112) plus device facts. */
typedef struct fglt_stats {
  int32_t num_steps;
  char step_names[FGLT_MAX_STEPS][32]; /* reference step names, in order */
  double step_seconds[FGLT_MAX_STEPS];
  uint64_t p2_row_touches;   /* W - 2m when the four-cycle step runs     */
  uint64_t p2_touch_bound;   /* 2 * d_max * m                            */
  uint64_t peak_aux_words;   /* device scratch, 8-byte words             */
  uint64_t largest_aux_alloc_words;
  int32_t threads_used;      /* host threads (the device does the work)  */
  int32_t device;
  uint64_t W;                /* sum_v d_v^2                              */
  uint64_t d_max;
  uint64_t kernel_launches;  /* kernels this library launched (this call) */
  /* FGLT_TIMINGS only: device phases of this call (CUDA events on the
   * context's stream), finer than the reference steps, e.g. "c4 dense" =
   * the dense-tile 4-cycle kernels; phase_units = their algorithmic work
   * units (wedges for the 4-cycle phases, 0 when not defined). */
  int32_t num_phases;
  char phase_names[FGLT_MAX_PHASES][32];
  double phase_seconds[FGLT_MAX_PHASES];
  uint64_t phase_units[FGLT_MAX_PHASES];
} fglt_stats;

/* Opaque per-device context: stream, workspace, cached preprocessing. One
 * transform at a time per context. */
typedef struct fglt_ctx fglt_ctx;

/* Create a context on `device`, launching on `stream` (a cudaStream_t; 0 for
 * the legacy default stream). Returns NULL and fills err on failure. */
fglt_ctx* fglt_ctx_create(int device, void* stream, fglt_error* err);
void fglt_ctx_destroy(fglt_ctx* ctx);
/* Free the context's device workspace (it is kept between calls for reuse;
 * the triangle-list pool alone may hold up to 70% of the free HBM after a
 * large transform). The next call re-allocates what it needs. */
int fglt_ctx_release_workspace(fglt_ctx* ctx);

/* One full transform: raw + net for the dictionary `dict_mask` (bit k =
 * graphlet k; bits 0 and 1 are forced, Dictionary::from_ids,
 * src/dictionary.cpp:38-50). `lenient` as TransformOptions::lenient.
 * raw_out/net_out may be NULL to skip that table. stats may be NULL. */
int fglt_ctx_transform(fglt_ctx* ctx, const int32_t* row_ptr,
                       const int32_t* col_idx, int64_t n, int64_t nnz,
                       uint32_t dict_mask, int lenient, uint32_t flags,
                       uint64_t* raw_out, uint64_t* net_out, fglt_stats* stats,
                       fglt_error* err);

/* Convenience: create a context on `device`, transform, destroy. */
int fglt_transform_csr32(const int32_t* row_ptr, const int32_t* col_idx,
                         int64_t n, int64_t nnz, uint32_t dict_mask,
                         int lenient, int device, uint32_t flags,
                         uint64_t* raw_out, uint64_t* net_out,
                         fglt_stats* stats, fglt_error* err);

/* Single-process multi-GPU transform: the CSR is broadcast
 * from devices[0] over NCCL, enumeration roots are split into blocks of equal
 * exact work, the per-edge C3 and the c4/d13/d15 partials are all-reduced
 * (NCCL), and each device writes its block of original-id rows straight
 * into raw_out/net_out. FGLT_INPUT_DEVICE / FGLT_OUTPUT_DEVICE mean pointers
 * on devices[0]. Bit-identical to fglt_ctx_transform for any device list.
 * A list with repeated devices (e.g. {0, 0}) runs the ranks one after the
 * other on the shared device with host-staged sums (the >1-rank path on a
 * one-GPU machine). Contexts and communicators are cached per device list. */
int fglt_transform_multi(const int32_t* row_ptr, const int32_t* col_idx,
                         int64_t n, int64_t nnz, uint32_t dict_mask, int lenient,
                         const int* devices, int num_devices, uint32_t flags,
                         uint64_t* raw_out, uint64_t* net_out, fglt_stats* stats,
                         fglt_error* err);

/* Stand-alone raw -> net conversion on the device (net_from_raw,
 * conversion.cpp:80-116): raw/net are n x k host arrays for dict_mask. */
int fglt_net_from_raw(fglt_ctx* ctx, const uint64_t* raw, int64_t n,
                      uint32_t dict_mask, int lenient, uint64_t* net,
                      fglt_error* err);
/* Same with the caller's conversion matrix U (k x k row-major uint64, unit
 * upper triangular; NULL = U16(s,s)): net_from_raw(raw, U, lenient)
 * honours any validated ConversionMatrix (conversion.hpp:14-37,49-51). */
int fglt_net_from_raw_matrix(fglt_ctx* ctx, const uint64_t* raw, int64_t n,
                             uint32_t dict_mask, const uint64_t* U, int lenient,
                             uint64_t* net, fglt_error* err);

/* ------------------------------------------------------------------ ingest
 * Device CSR ingest replacing build_adjacency (src/graph.cpp:192-249):
 * (eu[i], ev[i]) undirected pairs (int64, host pointers unless
 * FGLT_INPUT_DEVICE), declared_n (0 = max id + 1), SanitizeOptions
 * (graph.hpp:32-36). Mirrors when symmetrize, drops self-loops (else
 * StructuralError), sorts, dedupes (else StructuralError), checks symmetry
 * when not symmetrizing. The CSR stays in the context; fetch it with
 * fglt_csr_fetch (n+1 and nnz int32 entries). */
int fglt_build_csr(fglt_ctx* ctx, const int64_t* eu, const int64_t* ev, int64_t ne,
                   int64_t declared_n, int symmetrize, int drop_self_loops, int dedupe,
                   uint32_t flags, int64_t* n_out, int64_t* nnz_out, int64_t* self_loops,
                   int64_t* duplicates, fglt_error* err);
int fglt_csr_fetch(fglt_ctx* ctx, int32_t* row_ptr, int32_t* col_idx, uint32_t flags,
                   fglt_error* err);

/* ------------------------------------------------------------------ staged
 * Row-block sharding across ranks (one process per GPU; the caller owns the
 * collectives, e.g. torch.distributed over NCCL). Sequence per rank:
 *   fglt_stage_prepare      replicated preprocessing of the whole graph
 *   fglt_stage_bounds       root ranges balanced by exact work
 *   fglt_stage_triangles    partial per-edge triangle counts for own roots
 *   -- all-reduce(sum) of the uint32 edge-count buffer --
 *   fglt_stage_local_part   phase 0: sweep B on my rows (r = rank mod world)
 *   -- all-reduce(sum) of the uint64 c3 vector (n) --
 *   fglt_stage_local_part   phase 1: sweep C on my rows
 *   fglt_stage_roots        partial c4/d13/d15 for own roots
 *   -- all-reduce(sum) of the uint64 vector buffer (7n: d14 d10 p3 d9 c4 d13 d15) --
 *   (fglt_stage_local = both sweeps over every row, replicated; fglt_stage_roots
 *    then hands out the 3n c4/d13/d15 block)
 *   fglt_stage_epilogue     raw/net rows [r0, r1) in original-id order
 * Buffers handed to the caller are device pointers owned by the context. */
int fglt_stage_prepare(fglt_ctx* ctx, const int32_t* d_row_ptr,
                       const int32_t* d_col_idx, int64_t n, int64_t nnz,
                       uint32_t dict_mask, int lenient, fglt_error* err);
/* bounds[0..world] of the relabelled root range for each rank */
int fglt_stage_bounds(fglt_ctx* ctx, int world, int64_t* bounds, fglt_error* err);
int fglt_stage_triangles(fglt_ctx* ctx, int64_t u0, int64_t u1,
                         uint32_t** d_edge_counts, int64_t* count,
                         fglt_error* err);
int fglt_stage_local(fglt_ctx* ctx, fglt_error* err);
/* rows r = part (mod nparts); phase 0 returns the c3 vector to sum (count = n,
 * or 0 when nparts == 1 / no triangle columns), phase 1 returns count 0 */
int fglt_stage_local_part(fglt_ctx* ctx, int part, int nparts, int phase,
                          uint64_t** d_c3, int64_t* count, fglt_error* err);
int fglt_stage_roots(fglt_ctx* ctx, int64_t u0, int64_t u1,
                     uint64_t** d_vectors, int64_t* count, fglt_error* err);
/* Rows are ORIGINAL vertex ids [v0, v1); outputs are device pointers of
 * (v1-v0) x k. */
int fglt_stage_epilogue(fglt_ctx* ctx, int64_t v0, int64_t v1,
                        uint64_t* d_raw_rows, uint64_t* d_net_rows,
                        fglt_error* err);

/* ------------------------------------------------------------- per-kernel
 * The reference's public per-kernel functions on the device
 * (include/graphlet/kernels.hpp:43-98, src/kernels.cpp:26-288), same inputs
 * and outputs: host arrays, uint64 vectors of n, the per-edge C3 of nnz
 * entries aligned with col_idx (SparseCountMatrix, kernels.hpp:17-40).
 * Caller vectors (p1, p2, c3, C3) are used as given, as the reference does.
 * Checked sites return FGLT_E_OVERFLOW with the reference's graphlet id and
 * the lowest offending vertex. compute_c4_d14 and compute_d15 are the
 * transform's own columns (graphlet:: layer, dictionary {12,14} / {15}). */
/* compute_p2 (kernels.cpp:26-39) */
int fglt_kernel_p2(fglt_ctx* ctx, const int32_t* row_ptr, const int32_t* col_idx, int64_t n,
                   int64_t nnz, const uint64_t* p1, uint64_t* p2, fglt_error* err);
/* compute_c3_C3 (kernels.cpp:41-89): c3 (n) and C3 (nnz) */
int fglt_kernel_c3(fglt_ctx* ctx, const int32_t* row_ptr, const int32_t* col_idx, int64_t n,
                   int64_t nnz, uint64_t* c3, uint64_t* C3, fglt_error* err);
/* compute_p3 (kernels.cpp:91-107) */
int fglt_kernel_p3(fglt_ctx* ctx, const int32_t* row_ptr, const int32_t* col_idx, int64_t n,
                   int64_t nnz, const uint64_t* p1, const uint64_t* p2, const uint64_t* c3,
                   uint64_t* p3, fglt_error* err);
/* compute_d7 (kernels.cpp:149-163), checked: graphlet 7 */
int fglt_kernel_d7(fglt_ctx* ctx, const int32_t* row_ptr, const int32_t* col_idx, int64_t n,
                   int64_t nnz, const uint64_t* p1, uint64_t* d7, fglt_error* err);
/* compute_d8 (kernels.cpp:165-174), checked: graphlet 8 */
int fglt_kernel_d8(fglt_ctx* ctx, int64_t n, const uint64_t* p1, uint64_t* d8, fglt_error* err);
/* compute_d9_d10_d11 (kernels.cpp:176-205), checked: graphlets 9, 10, 11 */
int fglt_kernel_d9_d10_d11(fglt_ctx* ctx, const int32_t* row_ptr, const int32_t* col_idx,
                           int64_t n, int64_t nnz, const uint64_t* p1, const uint64_t* c3,
                           const uint64_t* C3, uint64_t* d9, uint64_t* d10, uint64_t* d11,
                           fglt_error* err);
/* compute_d13 (kernels.cpp:207-232) for the caller's C3 */
int fglt_kernel_d13(fglt_ctx* ctx, const int32_t* row_ptr, const int32_t* col_idx, int64_t n,
                    int64_t nnz, const uint64_t* C3, uint64_t* d13, fglt_error* err);
/* Number of kernels this context has launched so far (CUB calls count 1). */
uint64_t fglt_ctx_kernel_launches(const fglt_ctx* ctx);
/* Device buffers the last call used, one "name bytes [staging]" line each
 * (staging = the graph copy, the output tables and their raw columns, which
 * TransformStats.peak_aux_words does not count). */
int fglt_ctx_scratch_report(const fglt_ctx* ctx, char* out, int len);

/* Test hooks: force one internal code path for every root so small graphs
 * exercise paths that otherwise only large graphs reach. Results must be
 * identical for any setting (the parity tests check exactly that). */
#define FGLT_DEBUG_C4_CLASS 1  /* 0 auto, 2 hash passes, 3 packed tiles, 4 tiles, 5 small packed tiles */
#define FGLT_DEBUG_C4_PARTS 2  /* hash passes per root when class 2 is forced  */
#define FGLT_DEBUG_ROOTS_BIN 3 /* 0 auto, 1..4 smem bitmap bins, 5 global slab */
#define FGLT_DEBUG_HUB 4       /* 0 auto, 1 no hub rows, 2 hub rows for every hub member */
#define FGLT_DEBUG_TRILIST 5   /* 0 auto, 1 no triangle list, 2 tiny list pool (fallbacks) */
#define FGLT_DEBUG_ROW_SORT 6  /* 0 auto (in-register row sort when d_max is small), 2 always the global transpose sort */
#define FGLT_DEBUG_FLAT_DMAX 7 /* d_max up to which active vertices keep the caller's order (0: always degree order; <= 255) */
int fglt_ctx_set_debug(fglt_ctx* ctx, int key, int value);

/* Measured random-address shared-memory atomicAdd rate (ops/s) of this
 * device at the dense 4-cycle kernel's tile size and occupancy: the on-chip
 * roofline denominator bench.py reports for that kernel. */
int fglt_probe_smem_atomics(fglt_ctx* ctx, double* ops_per_s, fglt_error* err);

/* Library facts */
const char* fglt_version(void);
int fglt_device_count(void);

#ifdef __cplusplus
}
#endif

#endif /* FGLT_H_ */
