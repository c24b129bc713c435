/*
 * tsg.h -- C ABI of the B200-native two-phase SpGEMM ("tiered SpGEMM").
 *
 * This is the drop-in boundary for the reference's hot path
 * (/root/reference/pkg/src/tiered_spgemm/kernel.py, chunking.py).  The
 * reference is pure Python with no FFI of its own; the binding a maintainer
 * would add is the ctypes stub shown in INTEGRATION.md, which is exactly what
 * paper_1804_00695_b200/_lib.py does.  Signatures use plain pointers and
 * sizes only: host arrays are the reference's int64 / float64 / uint64
 * numpy buffers, device objects are opaque handles owned by the library.
 *
 * Every entry point returns a status code; the message of the last failure
 * on the calling thread is available from tsg_last_error().  Codes map to the
 * reference's exception classes (errors.py:4-45):
 *   TSG_EDIM      -> DimensionError
 *   TSG_EVALID    -> MatrixValidationError
 *   TSG_EKERNEL   -> KernelError   (count mismatch, probe overflow)
 *   TSG_ECAPACITY -> CapacityError (HBM budget)
 *   TSG_EUNSPLIT  -> UnsplittableRowError
 *   TSG_ECUDA     -> KernelError   (CUDA runtime failure, message attached)
 *   TSG_EARG      -> ValueError
 *
 * Threading: a context owns one compute stream and two copy streams on one
 * device; it is not thread-safe.  Use one context per GPU.
 */
#ifndef TSG_H
#define TSG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSG_OK 0
#define TSG_EDIM 1
#define TSG_EVALID 2
#define TSG_EKERNEL 3
#define TSG_ECAPACITY 4
#define TSG_EUNSPLIT 5
#define TSG_ECUDA 6
#define TSG_EARG 7

#define TSG_ABI_VERSION 1

typedef struct tsg_ctx tsg_ctx;   /* device, streams, scratch, error flag        */
typedef struct tsg_csr tsg_csr;   /* device CSR: int64 offsets, int32 cols, f64  */
typedef struct tsg_cmat tsg_cmat; /* device compressed (set, 64-bit mask) rows   */
typedef struct tsg_vec tsg_vec;   /* device int64 vector (+ per-row set counts)  */

/* ---- library / context -------------------------------------------------- */
const char *tsg_last_error(void);
int tsg_abi_version(void);
int tsg_device_count(int *count);
int tsg_init(int device, tsg_ctx **out);
int tsg_destroy(tsg_ctx *ctx);
int tsg_sync(tsg_ctx *ctx);
/* Bytes of device memory currently held by the context's allocations. */
int tsg_mem_in_use(tsg_ctx *ctx, int64_t *bytes);
/* Shared-memory hash-table conflict counters of the symbolic / numeric group
 * tiers since the last reset: out = {lookups, extra lookup probes, inserts,
 * extra insert probes}.  Diagnostic builds only (-DTSG_PROBE_STATS=1); the
 * product build returns TSG_EARG.  No reference counterpart (the reference's
 * HashmapAccumulator, accumulator.py:95-127, probes the same way but keeps no
 * statistics). */
int tsg_probe_stats(tsg_ctx *ctx, int64_t out[4], int reset);
/* Bytes the device's stream-ordered pool has reserved from the driver. */
int tsg_pool_reserved(tsg_ctx *ctx, int64_t *bytes);
/* Per-phase device times (ms) of the last tsg_multiply (timing enabled):
   [0] compress [1] symbolic [2] row-pointer scan [3] numeric [5] total */
int tsg_last_phase_ms(tsg_ctx *ctx, float *out, int n);
int tsg_set_timing(tsg_ctx *ctx, int enabled);
/* Cumulative kernel launches of the context, and (timing enabled) the device
   time of the symbolic and numeric kernels of the last multiply-type call,
   measured with CUDA events on the context's compute stream. */
typedef struct {
    int64_t launches;
    float symbolic_ms;
    float numeric_ms;
} tsg_stats;
int tsg_get_stats(tsg_ctx *ctx, tsg_stats *out);
/* User timing events on the compute stream (slot 0..7): record, then the
   elapsed device time between two recorded slots (synchronises on `to`). */
/* Numeric-kernel timing ring (timing on): tsg_numeric_calls = numeric phases
   run so far; tsg_numeric_ms = device time of the numeric kernels of call k
   (one of the last 32), read without synchronising the calls after it. */
int tsg_numeric_calls(tsg_ctx *ctx, int64_t *n);
int tsg_numeric_ms(tsg_ctx *ctx, int64_t call, float *ms);
/* The context's compute stream (a cudaStream_t), so a caller can order its
   own work -- e.g. the NCCL offset exchange -- on it. */
int tsg_stream(tsg_ctx *ctx, void **stream);
int tsg_event_record(tsg_ctx *ctx, int slot);
int tsg_event_elapsed(tsg_ctx *ctx, int from, int to, float *ms);
/* Device-to-device import of a CSR whose arrays already live on this device
   (e.g. gathered by NCCL): int64 row_ptr, int32 columns, fp64 values. */
int tsg_csr_from_device(tsg_ctx *ctx, int64_t rows, int64_t cols, int64_t nnz,
                        const int64_t *d_row_ptr, const int32_t *d_col,
                        const double *d_values, tsg_csr **out);
/* Device pointers of a CSR (borrowed; valid until tsg_csr_free). */
int tsg_csr_device_ptrs(const tsg_csr *m, int64_t **d_row_ptr, int32_t **d_col,
                        double **d_values);

/* Pinned host memory from a caching pool (falls back to pageable memory if
   pinning is refused).  Used for result arrays returned to the caller. */
int tsg_host_alloc(size_t bytes, void **out);
int tsg_host_free(void *p);

/* ---- CSR operands (csr.py:32-106 CsrMatrix) ------------------------------ */
/* values may be NULL (pattern).  Columns must be < 2^31 (device int32). */
int tsg_csr_upload(tsg_ctx *ctx, int64_t rows, int64_t cols, int64_t nnz,
                   const int64_t *row_ptr, const int64_t *col_idx,
                   const double *values, tsg_csr **out);
/* nnz of a product is resolved on first request: tsg_multiply may return
   before the device has counted C's entries (its device-driven path never
   waits), so asking for nnz can synchronise; tsg_csr_dims never does. */
int tsg_csr_info(const tsg_csr *m, int64_t *rows, int64_t *cols, int64_t *nnz,
                 int *has_values);
int tsg_csr_dims(const tsg_csr *m, int64_t *rows, int64_t *cols, int *has_values);
/* Host buffers sized rows+1 / nnz / nnz (values may be NULL to skip). */
int tsg_csr_download(tsg_ctx *ctx, const tsg_csr *m, int64_t *row_ptr,
                     int64_t *col_idx, double *values);
/* Rows [begin, end) as a new rebased device CSR (csr.py:187-195 slice_rows). */
int tsg_csr_slice_rows(tsg_ctx *ctx, const tsg_csr *m, int64_t begin,
                       int64_t end, tsg_csr **out);
int tsg_csr_free(tsg_ctx *ctx, tsg_csr *m);

/* ---- compressed form (kernel.py:52-93 CompressedMatrix / compress) ------- */
/* Sets are emitted in first-touch order per row, as the reference does. */
int tsg_compress(tsg_ctx *ctx, const tsg_csr *b, tsg_cmat **out);
int tsg_cmat_info(tsg_ctx *ctx, const tsg_cmat *cm, int64_t *rows,
                  int64_t *n_sets);
int tsg_cmat_download(tsg_ctx *ctx, const tsg_cmat *cm, int64_t *row_ptr,
                      int64_t *set_idx, uint64_t *set_bits);
int tsg_cmat_upload(tsg_ctx *ctx, int64_t rows, int64_t n_sets,
                    const int64_t *row_ptr, const int64_t *set_idx,
                    const uint64_t *set_bits, tsg_cmat **out);
int tsg_cmat_free(tsg_ctx *ctx, tsg_cmat *cm);

/* ---- int64 vectors (symbolic counts) ------------------------------------- */
int tsg_vec_upload(tsg_ctx *ctx, int64_t n, const int64_t *host, tsg_vec **out);
int tsg_vec_download(tsg_ctx *ctx, const tsg_vec *v, int64_t *host);
int tsg_vec_len(const tsg_vec *v, int64_t *n);
int tsg_vec_free(tsg_ctx *ctx, tsg_vec *v);

/* ---- the hot path ---------------------------------------------------------- */
/* Per-row multiplications of A*B (the K0 bound loop of kernel.py:135-145 over
   the uncompressed B: sum of nnz(B_k) over row i of A), copied to flops_host
   (rows_A int64, may be NULL) with their total (may be NULL).  Weights of the
   multi-GPU flops partition (distributed.flops_partition). */
int tsg_row_flops(tsg_ctx *ctx, const tsg_csr *a, const tsg_csr *b, int64_t *flops_host,
                  int64_t *total);
/* kernel.py:96-103 count_multiplications */
int tsg_count_multiplications(tsg_ctx *ctx, const tsg_csr *a, const tsg_csr *b,
                              int64_t *total);
/* kernel.py:124-168 spgemm_symbolic: exact nnz per row of A*B. */
int tsg_symbolic(tsg_ctx *ctx, const tsg_csr *a, const tsg_cmat *cb,
                 tsg_vec **counts);
/* kernel.py:171-232 spgemm_numeric.  cb may be NULL (compressed on the fly).
   C rows come out with ascending columns (the reference's are first-touch;
   canonical forms are identical).  TSG_EKERNEL if counts are wrong. */
int tsg_numeric(tsg_ctx *ctx, const tsg_csr *a, const tsg_csr *b,
                const tsg_cmat *cb, const tsg_vec *counts, tsg_csr **c);
/* kernel.py:343-346 multiply = compress + symbolic + numeric, all on device. */
int tsg_multiply(tsg_ctx *ctx, const tsg_csr *a, const tsg_csr *b, tsg_csr **c);
/* kernel.py:235-340 spgemm_numeric_fused:
   out = c_partial + A[a_lo:a_hi, b_lo:b_hi] * b_chunk  (b_chunk rebased). */
int tsg_numeric_fused(tsg_ctx *ctx, const tsg_csr *a, const tsg_csr *b_chunk,
                      const tsg_csr *c_partial, int64_t a_lo, int64_t a_hi,
                      int64_t b_lo, int64_t b_hi, tsg_csr **out);
/* kernel.py:349-394 masked_row_intersect_count (TSG_EVALID if L is not
   strictly lower triangular). */
int tsg_masked_count(tsg_ctx *ctx, const tsg_csr *l, const tsg_cmat *cl,
                     int64_t *total);

/* ---- graph preparation on the device ----------- */
/* triangles.py:18-46 validate_graph (check != 0: square, loop-free, symmetric
   pattern -> TSG_EVALID) + degree_sort_permutation (stable by degree, ties by
   index) + lower_triangle: L = strict lower triangle of the relabelled graph,
   rows sorted, pattern only.  perm_host (optional, n int64): the permutation
   (position -> original vertex) as degree_sort_permutation returns it. */
int tsg_graph_lower(tsg_ctx *ctx, const tsg_csr *g, int check, tsg_csr **L,
                    int64_t *perm_host);
/* generators.rmat_graph of this package on the device: Graph500 R-MAT with
   2^scale vertices and edge_factor * 2^scale directed draws from the
   SplitMix64 counter stream of `seed`, vertices relabelled by the ranks of a
   second stream (seed ^ GAMMA), symmetrised, de-duplicated, loop-free pattern
   CSR -- equal to the host builder entry for entry. */
int tsg_rmat_graph(tsg_ctx *ctx, int scale, int edge_factor, uint64_t seed, double a, double b,
                   double c, tsg_csr **out);
/* ---- B sharded across GPUs --------------------------------
   B's rows [row_lo[s], row_lo[s+1]) live on shard s as device arrays
   (shard-local int64 row pointers from 0, int32 columns, fp64 values) --
   typically other GPUs' memory opened through CUDA IPC (NVLink P2P loads).
   Builds a local CSR of B in which exactly the rows selected by A's columns
   are filled (others empty), reading them straight from the shards. */
int tsg_gather_sharded(tsg_ctx *ctx, int n_shards, const int64_t *row_lo, const void *const *shard_rp,
                       const void *const *shard_col, const void *const *shard_val, int64_t b_cols,
                       const tsg_csr *a, tsg_csr **out);
/* ---- multi-GPU row partition (rows of C are independent,
   kernel.py:11-14).  One process per GPU; the collectives (B all-gather,
   row-pointer offset exchange) run over NCCL in the host layer
   (paper_1804_00695_b200/distributed.py).

   B sharded in peer HBM: every GPU owns one element range of B's column and
   value arrays as a CUDA VMM physical allocation exported as a POSIX file
   descriptor; each GPU maps every shard, in order, into ONE reserved virtual
   range (tsg_shard_map), so B's arrays look contiguous to the kernels while
   remote pages are read from peer HBM over NVLink.  Shard sizes are multiples
   of tsg_shard_granularity. */
typedef struct tsg_shard tsg_shard;  /* this GPU's exported physical shard    */
typedef struct tsg_vmap tsg_vmap;    /* all shards mapped into one VA range   */
int tsg_shard_granularity(tsg_ctx *ctx, size_t *bytes);
/* Physical allocation of >= bytes on the context's GPU, mapped locally at
   *dev_ptr (to fill it), exported as *fd (owned by the shard; dup before
   sending if the shard may be freed first). */
int tsg_shard_alloc(tsg_ctx *ctx, size_t bytes, tsg_shard **out, void **dev_ptr, int *fd, size_t *size);
int tsg_shard_free(tsg_ctx *ctx, tsg_shard *s);
/* Import n shard descriptors (this process's own or received from peers)
   and map them back to back at *va (sum of sizes). */
int tsg_shard_map(tsg_ctx *ctx, int n, const int *fds, const size_t *sizes, tsg_vmap **out, void **va);
int tsg_vmap_free(tsg_ctx *ctx, tsg_vmap *m);
/* Synchronous copy on the context's compute stream between any addresses the
   GPU reaches (device memory, VMM ranges, pinned host). */
int tsg_memcpy(tsg_ctx *ctx, void *dst, const void *src, size_t bytes);
/* A CSR over device arrays the caller owns (e.g. B's columns / values in a
   tsg_shard_map range): freeing the view leaves the arrays alone.  sorted:
   every row ascending and distinct; max_row: longest row (-1 unknown). */
int tsg_csr_view(tsg_ctx *ctx, int64_t rows, int64_t cols, int64_t nnz, const int64_t *d_row_ptr,
                 const int32_t *d_col, const double *d_values, int sorted, int64_t max_row,
                 tsg_csr **out);
/* One GPU's block of C = A_block * B (kernel.py:343-346 per row block).
   c_budget_bytes == 0: C materialised in *c (may be NULL to drop it);
   > 0: streamed-C mode -- row sub-blocks whose C fits the budget are
   multiplied, reduced (nnz, sum, sum of squares) and released, for products
   whose C exceeds HBM; *c stays NULL.  B is compressed once per call. */
typedef struct {
    int64_t nnz;            /* entries of this block of C                    */
    int64_t blocks;         /* sub-blocks multiplied                        */
    int64_t max_block_nnz;  /* largest sub-block of C held at once           */
    double value_sum;       /* sum of C's values (fp64)                      */
    double value_sumsq;     /* sum of their squares                          */
} tsg_mg_stats;
int tsg_mg_multiply(tsg_ctx *ctx, const tsg_csr *a_block, const tsg_csr *b, int64_t c_budget_bytes,
                    tsg_csr **c, tsg_mg_stats *stats);
/* every stored entry := value (allocating the value array of a pattern CSR):
   generators.with_unit_values on the device */
int tsg_csr_set_values(tsg_ctx *ctx, tsg_csr *m, double value);

/* ---- input builders on the device -------------------
   Same arrays as the host builders: generators.stencil / stencil_rows
   (reference generators.py:98-142, flat index first axis fastest, columns
   ascending, centre weight = number of neighbours, elasticity3d = 3x3 blocks
   w * (I + 0.5)), generators.aggregation (P: fine point -> aggregate, 1.0;
   R = P^T, generators.py:204-230 restated for plain aggregation) and
   csr.transpose (csr.py:134-142: stable by column, rows ascending). */
#define TSG_STENCIL_LAPLACE2D 0
#define TSG_STENCIL_LAPLACE3D 1
#define TSG_STENCIL_BIGSTAR2D 2
#define TSG_STENCIL_BRICK3D 3
#define TSG_STENCIL_ELASTICITY3D 4
/* rows [row_lo, row_hi) of the operator (row_lo < 0: all rows; elasticity3d:
   all rows only); columns span the whole grid */
int tsg_stencil(tsg_ctx *ctx, int kind, const int64_t *dims, int ndims, int64_t row_lo, int64_t row_hi,
                tsg_csr **out);
int tsg_aggregation(tsg_ctx *ctx, const int64_t *dims, int ndims, int factor, tsg_csr **p_out,
                    tsg_csr **r_out);
int tsg_transpose(tsg_ctx *ctx, const tsg_csr *a, tsg_csr **out);

/* ---- fused Galerkin triple product C = R * A * P (
   the reference runs multiply(multiply(R, A), P), kernel.py:343-346).
   mode 0: the two multiplies; mode 1: one symbolic + one numeric pass with
   RA's rows kept in shared memory (never written to HBM), falling back to
   the two multiplies when A or P lacks sorted distinct rows or a row of RA /
   C exceeds the per-row slices.  *fused (may be NULL) reports which ran.
   The fused result is bit-identical to the two-multiply result of this
   library when that one keeps its rows in the group tier. */
int tsg_rap(tsg_ctx *ctx, const tsg_csr *r, const tsg_csr *a, const tsg_csr *p, int mode, tsg_csr **out,
            int *fused);

/* ---- data placement (memory.py:193-223 PlacementPolicy; PAPER.md:600-625,
   810-829).  A CSR whose arrays live in pinned, device-mapped HOST memory:
   kernels read it in place over PCIe (the paper's "pinned" columns).  Columns
   are narrowed to int32 on the host at mapping time. */
int tsg_csr_map_host(tsg_ctx *ctx, int64_t rows, int64_t cols, int64_t nnz,
                     const int64_t *row_ptr, const int64_t *col_idx, const double *values,
                     tsg_csr **out);
/* multiply with C built in mapped host memory when c_in_host != 0 (operands
   may be device or mapped-host CSRs: any placement of A, B and C). */
int tsg_multiply_placed(tsg_ctx *ctx, const tsg_csr *a, const tsg_csr *b, int c_in_host,
                        tsg_csr **c);

/* ---- chunked execution through an HBM budget (chunking.py:219-337) -------- */
/* algo: 0 = KNL order (B streamed past all of A/C), 1 = GPU chunk1 (A/C row
   range in place, B streamed), 2 = GPU chunk2 (B range in place, A/C
   streamed).  Partitions are boundary arrays (n+1 entries, 0 .. rows).  Host
   arrays use the reference's formats (int64 offsets and indices, f64
   values); pin them for full PCIe rate.  c_row_ptr = exclusive scan of the
   symbolic counts; c_col / c_val (sum of counts entries) are filled.  Every
   chunk step is the fused multiply-add run in place in HBM. */
typedef struct {
    int64_t h2d_bytes;          /* bytes actually copied host -> device     */
    int64_t d2h_bytes;          /* bytes actually copied device -> host     */
    double kernel_ms;           /* device time of compress + fused kernels   */
    double wall_ms;             /* host wall time of the whole call          */
    int64_t peak_device_bytes;  /* high-water mark of the call's HBM allocations */
    int64_t budget_bytes;       /* the budget passed in (0: unlimited)       */
    int64_t layout_bytes;       /* modelled footprint of the chosen layout   */
    int32_t a_slots, c_slots, b_slots;  /* buffering chosen for A / C / B    */
    int32_t ac_split, b_split;  /* physical sub-ranges per planned range / chunk */
} tsg_chunk_stats;
/* budget_bytes > 0: every device allocation of the call (slots, staging,
   per-step scratch) stays within it -- the executor double-buffers what fits
   and splits planned ranges / chunks physically where needed (traffic-neutral
   splits first); TSG_ECAPACITY if no layout fits or the measured high-water
   mark exceeds it (memory.py:103-111 residency check). */
int tsg_chunk_multiply(tsg_ctx *ctx, int algo, int64_t a_rows, int64_t a_cols,
                       const int64_t *a_row_ptr, const int64_t *a_col, const double *a_val,
                       int64_t b_rows, int64_t b_cols, const int64_t *b_row_ptr,
                       const int64_t *b_col, const double *b_val, const int64_t *c_row_ptr,
                       int64_t *c_col, double *c_val, int64_t n_ac, const int64_t *ac_bounds,
                       int64_t n_b, const int64_t *b_bounds, int64_t budget_bytes,
                       tsg_chunk_stats *stats);
/* spgemm_symbolic (kernel.py:124-168) through the same budget: B compressed
   chunk by chunk into one resident compressed B, then A row ranges streamed
   past it; counts (a_rows int64) written to host.  TSG_ECAPACITY when the
   compressed B alone does not fit. */
int tsg_chunk_symbolic(tsg_ctx *ctx, int64_t a_rows, int64_t a_cols, const int64_t *a_row_ptr,
                       const int64_t *a_col, int64_t b_rows, int64_t b_cols, const int64_t *b_row_ptr,
                       const int64_t *b_col, int64_t budget_bytes, int64_t *counts,
                       tsg_chunk_stats *stats);

#ifdef __cplusplus
}
#endif
#endif /* TSG_H */
