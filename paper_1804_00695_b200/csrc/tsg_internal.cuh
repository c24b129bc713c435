// tsg_internal.cuh -- shared internals of libtsg (B200 / sm_100a).
//
// Device layouts (HBM):
//   CSR   : int64 row_ptr[rows+1], int32 col[nnz], fp64 val[nnz]
//   CMAT  : padded compressed rows.  Row r's sets live at [start[r], start[r] +
//           cnt[r]) of int32 set[] / uint64 bits[]; start[] is a copy of the
//           source CSR's row_ptr, so compress is a single pass with no scan.
//   VEC   : int64 d[n] (+ optional int32 aux[n] = distinct sets per row).
//
// Accumulator tables are 16-byte slots {key, mask_lo, mask_hi, base}: the key
// is claimed with a 32-bit CAS and the 64-bit column mask is ORed as two
// native 32-bit ATOMS.OR halves (a 64-bit shared-memory OR is a CAS loop on
// sm_100a).  One 128-bit LDS fetches a whole slot during lookups.
#pragma once
#include <cstdlib>
#include <vector>
#include <utility>

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/tsg.h"

#define TSG_EMPTY (-1)

struct tsg_ctx {
    int device;
    int num_sms;
    size_t smem_optin;
    cudaStream_t stream;      // compute
    cudaStream_t copy_in;     // H2D
    cudaStream_t copy_out;    // D2H
    // independent row tiers (bins) run concurrently on these, forked from and
    // joined back into `stream` (tsg_spgemm.cu BinFork)
    static constexpr int NAUX = 3;
    cudaStream_t aux[NAUX];
    cudaEvent_t ev_fork, ev_join[NAUX];
    int *d_err;               // [0] code, [1] row (lowest)
    int64_t *h_small;         // pinned, device-mapped scratch for small reads (64 x int64)
    int64_t *hd_small;        // device alias of h_small: kernels store results there
    int64_t part_seq;         // last sequence word a partition kernel publishes (h_small[61])
                              // directly, so small reads never queue behind bulk D2H copies
    int64_t *d_small;         // device scratch for reductions (64 x int64)
    int timing;
    cudaEvent_t ev[8];
    float phase_ms[8];
    int64_t bytes_in_use;
    int64_t bytes_peak;       // high-water mark of bytes_in_use (the chunked executors reset it)
    // device-driven multiply (tsg_multiply's fast path): the partitions do not
    // wait for the host, bins launch on the host's bounds, and allocations
    // take these bounds instead of read-back sizes
    int nowait;
    uint32_t sym_possible, num_possible;
    int64_t set_cap_bound, nnz_bound, c_row_bound;
    // bin-size hints of this operand shape (pinned, device-mapped; written by
    // the partitions of the previous multiply of the same shape, read by the
    // host only to order launches and size grids)
    int64_t *hint_sym, *hint_num;     // host views (nullptr: none)
    int64_t *hintd_sym, *hintd_num;   // device aliases
    // CUDA-graph capture of a multiply (tsg_spgemm.cu plans): while set, the
    // arena hands out blocks without stream-ordered calls, and every block
    // allocated -- freed inside the capture or not -- is owned by the plan
    std::vector<void *> *capture_owned;
    int capture_failed;
    int capture_timing;    // record the numeric ring events as external (replayed) nodes
    int capture_rk;        // ring slot a capture recorded into
    cudaStream_t convert;     // int64 <-> int32 column conversion between copy stages (chunked)
    cudaStream_t widen;       // int32 -> int64 widening of drained C ranges (own stream, so a
                              // narrow for an H2D piece never queues behind a C drain)
    cudaStream_t copy_in2;    // second H2D stream: a piece's column copy queues while the
                              // previous piece waits for its conversion (chunked)
    int64_t launches;         // kernels launched by this context (all entry points)
    double mg_ratio = 0.0;    // streamed tsg_mg_multiply: last C entries per multiplication
    int coarse_alloc = 0;     // > 0: arena size classes of >= 1 GiB are coarse (streamed multiply)
    int64_t cmp_floor_rows = 0, cmp_floor_nnz = 0;   // tsg_compress_impl allocation floor (0: none)
    // streamed multiply: one col / val reservoir per call that every block's
    // C uses when it fits (no per-block multi-GB allocations)
    int32_t *c_res_col = nullptr;
    double *c_res_val = nullptr;
    int64_t c_res_cap = 0;
    cudaEvent_t ev_num[2];    // around the numeric kernels of the last multiply
    cudaEvent_t ev_sym[2];    // around the symbolic kernels of the last multiply
    cudaEvent_t ev_user[8];   // tsg_event_record slots
    int c_host_out;           // tsg_multiply_placed: build C in mapped host memory
    // lazily evaluated PhaseTimer (no sync at the end of a multiply)
    int phase_n, phase_total, phase_dirty;
    // kernel-error check deferred to the next synchronising call (download,
    // partition read-back, tsg_sync): the phase it belongs to
    const char *pending;
    // numeric-kernel event ring: call k's events are ev_ring[2 (k % NRING)] .. +1
    static constexpr int NRING = 32;
    cudaEvent_t ev_ring[2 * NRING];
    int64_t num_calls;
    int64_t ring_timed[NRING];   // call id recorded in each ring slot (-1: none)
    // decoupled look-back tile states, shared by every single-pass scan: words
    // carry the call's epoch, so no per-call clearing (tsg_lookback_state)
    unsigned long long *lb_state;
    int64_t lb_cap;
    unsigned lb_epoch;
    // monotone tile counter (never reset): a call's tiles are counter - base
    unsigned long long *lb_counter;
    unsigned long long lb_base;
};

struct tsg_csr {
    int64_t rows, cols, nnz;
    int64_t *rp;
    int32_t *col;
    double *val;
    int host_mapped;   // arrays live in pinned, device-mapped host memory (placement)
    int sorted;        // 1: every row's columns are non-decreasing (compress needs no fallback)
    int distinct;      // 1: no column repeats within a row (lane-split numeric mode is race-free)
    int64_t max_row;   // longest row, or -1 if unknown
    int borrowed;      // arrays owned by the caller (tsg_csr_view): free releases only the handle
    int cv_borrowed;   // col / val are the context's C reservoir (streamed multiply): not freed
    // A product of a device-driven multiply: the host never waited for it,
    // so `nnz` is the allocation bound and the exact count is rp[rows] on the
    // device, read on first need (tsg_csr_resolve).  max_row_bound (> 0) is
    // an upper bound on its row lengths, for the next multiply's planning.
    int lazy_nnz;
    tsg_ctx *owner;
    int64_t max_row_bound;
    // output of a captured multiply plan (arrays owned by the plan): freeing
    // it hands the plan's output slot back
    void *plan;
    int plan_slot;
};
// a plan whose graphs read `m` is dropped when m is freed or changed
void tsg_plans_forget(tsg_ctx *ctx, const tsg_csr *m);
void tsg_arena_return(tsg_ctx *ctx, const std::vector<void *> &blocks);
void tsg_plan_release_slot(void *plan, int slot);
// exact nnz of a product whose count is still on the device (no-op otherwise)
int tsg_csr_resolve(tsg_ctx *ctx, tsg_csr *m);
#define TSG_RESOLVE(ctx, m) TSG_TRY(tsg_csr_resolve((ctx), const_cast<tsg_csr *>(m)))

struct tsg_cmat {
    int64_t rows;
    int64_t *start;   // rows (+1; copy of source row_ptr, or compact ptr)
    int32_t *cnt;     // rows
    int32_t *set;     // capacity >= nsets
    uint64_t *bits;
    int64_t cap;      // entries allocated in set/bits
    int sorted_sets;  // 1: every row's sets ascend (compact compression of a row-sorted B)
    int identity_rows;  // 1: row k is exactly set k (start = iota, cnt = 1)
    int64_t cols;       // columns of the source matrix (0: unknown)
    int dmax_valid;     // 1: cnt[rows + 1] holds the largest row's set count (set by compress)
};

struct tsg_vec {
    int64_t n;
    int64_t *d;
    int32_t *aux;     // distinct sets per row (from symbolic) or null; bit 30 = sets emitted
    int64_t *sptr;    // symbolic's sorted (set, mask) lists per row, or null
    int32_t *sset;
    uint64_t *sbits;
};

// ---------------------------------------------------------------- errors
void tsg_set_error(const char *fmt, ...);
int tsg_cuda_fail(cudaError_t e, const char *what, const char *file, int line);

#define TSG_CK(call)                                                        \
    do {                                                                    \
        cudaError_t _e = (call);                                            \
        if (_e != cudaSuccess) return tsg_cuda_fail(_e, #call, __FILE__, __LINE__); \
    } while (0)

#define TSG_TRY(call)                      \
    do {                                   \
        int _s = (call);                   \
        if (_s != TSG_OK) return _s;       \
    } while (0)

// kernel-side error reporting: first code wins, lowest row kept
enum { KERR_NONE = 0, KERR_COUNT = 1, KERR_PROBE = 2, KERR_NOTLOWER = 3, KERR_COLRANGE = 4,
       KERR_UNSORTED_INTERNAL = 5, KERR_ROWSIZE = 6 };

__device__ __forceinline__ void kerr(int *err, int code, int64_t row) {
    atomicCAS(err, 0, code);
    atomicMin(err + 1, (int)(row < 0x7fffffff ? row : 0x7fffffff));
}

// ---------------------------------------------------------------- memory
int tsg_alloc(tsg_ctx *ctx, void **p, size_t bytes);
int tsg_free(tsg_ctx *ctx, void *p);
// return every cached block to the driver pool
int tsg_arena_trim(tsg_ctx *ctx);
template <typename T>
inline int tsg_alloc_t(tsg_ctx *ctx, T **p, size_t count) {
    return tsg_alloc(ctx, (void **)p, count * sizeof(T));
}
// Reads and clears the device error flag (synchronises the compute stream).
int tsg_check_kernel_errors(tsg_ctx *ctx, const char *phase);
// copy n int64 device words into h_small[slot..] through the mapped alias
// (a one-thread kernel on the compute stream; the caller synchronises)
int tsg_put_small(tsg_ctx *ctx, const int64_t *src, int n, int slot);
// look-back state words for `tiles` tiles and this call's epoch (1..16383)
int tsg_lookback_state(tsg_ctx *ctx, int64_t tiles, unsigned long long **state, unsigned *epoch);
// dynamic tile ids for a look-back kernel of `tiles` blocks: tile =
// atomicAdd(*counter, 1) - base (tiles are then started in id order)
int tsg_lookback_counter(tsg_ctx *ctx, int64_t tiles, unsigned long long **counter,
                         unsigned long long *base);
// word = value << 16 | epoch << 2 | flag (1 aggregate, 2 inclusive prefix);
// a word of another epoch reads as flag 0 (not yet published)
__device__ __forceinline__ unsigned long long lb_pack(int64_t v, unsigned epoch, unsigned flag) {
    return ((unsigned long long)v << 16) | ((unsigned long long)epoch << 2) | flag;
}
__device__ __forceinline__ unsigned lb_flag(unsigned long long w, unsigned epoch) {
    return ((unsigned)(w >> 2) & 0x3fffu) == epoch ? (unsigned)(w & 3ull) : 0u;
}
__device__ __forceinline__ int64_t lb_value(unsigned long long w) { return (int64_t)(w >> 16); }
// Load every kernel of the translation unit that holds `kernel` now.  With
// CUDA's lazy module loading, the first launch of a kernel waits for copies
// already queued on other streams (measured: a first-launched compute kernel
// sat behind 2.5 GB of pending H2D); tsg_init preloads all libtsg modules.
int tsg_preload_module_of(const void *kernel);
// one representative kernel per .cu file, for tsg_preload_module_of
const void *tsg_kernel_core();
const void *tsg_kernel_build();
const void *tsg_kernel_rap();
const void *tsg_kernel_compress();
const void *tsg_kernel_spgemm();
const void *tsg_kernel_masked();
const void *tsg_kernel_chunk();
const void *tsg_kernel_mg();
// per-row multiplications of A * B (K0 over B's row pointers) into flops[rows]
void tsg_launch_row_flops(tsg_ctx *ctx, const tsg_csr *a, const int64_t *brp, int64_t *flops);
const void *tsg_kernel_graph();
// cudaMemsetAsync replacement as a kernel: on this platform memsets queue on
// the copy engines, i.e. behind any bulk H2D / D2H already in flight
int tsg_fill(tsg_ctx *ctx, void *p, int byte, size_t bytes, cudaStream_t s);
// cudaMemcpyAsync in <= 256 MiB pieces.  Measured on the B200 box: a single
// multi-GB host copy queued on one stream holds back kernels launched on
// OTHER streams until it completes; split, the copy keeps its bandwidth and
// other streams' kernels start within ~0.3 ms.
int tsg_copy(void *dst, const void *src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s);
// wait until a kernel on c->stream has stored `seq` into h_small[slot]
// (stores before it made visible with __threadfence_system).  Polls the
// mapped word; checks the stream every few thousand polls so a failed kernel
// returns its error instead of spinning.
int tsg_wait_mapped(tsg_ctx *ctx, int slot, int64_t seq);
// after a stream sync that also copied d_err into h_small[62]: report a
// pending (deferred) kernel error, if any
int tsg_pending_errors(tsg_ctx *ctx);

int tsg_trace_enabled();
// host timestamp line (no sync) when TSG_CHUNK_TIMELINE is set
void tsg_trace_host(const char *what);
// TSG_TRACE=1: host timestamps + GPU drain per traced step (debug only)
void tsg_trace(tsg_ctx *c, const char *what, int64_t arg);

// cudaGetLastError after a launch, with the launch shape in the message
int tsg_launch_check(const char *kernel, int bin, unsigned grid, int block, size_t smem);

// Opt a kernel in to `bytes` of dynamic shared memory on the current device
// (static + dynamic must fit 227 KB; the default dynamic cap is 48 KB minus
// the static part).  Cached per (device, kernel): steady state makes no call.
int tsg_func_smem(const void *kernel, size_t bytes);

// ---------------------------------------------------------------- scan
// Exclusive prefix sum of n int64 values into out[0..n] (out[n] = total).
// in and out may alias only if in == out (in-place supported).
int tsg_exclusive_scan_i64(tsg_ctx *ctx, const int64_t *in, int64_t *out, int64_t n);
// Same for int32 input, int64 output.
int tsg_exclusive_scan_i32_to_i64(tsg_ctx *ctx, const int32_t *in, int64_t *out, int64_t n);

// ---------------------------------------------------------------- objects
int tsg_csr_alloc_mapped(tsg_ctx *ctx, int64_t rows, int64_t cols, int64_t nnz, bool values,
                         tsg_csr **out);
int tsg_csr_alloc(tsg_ctx *ctx, int64_t rows, int64_t cols, int64_t nnz, bool values,
                  tsg_csr **out);
int tsg_vec_alloc(tsg_ctx *ctx, int64_t n, bool aux, tsg_vec **out);
// sets m->sorted from the device data (synchronises)
int tsg_csr_check_sorted(tsg_ctx *ctx, tsg_csr *m);
int tsg_cmat_alloc(tsg_ctx *ctx, int64_t rows, int64_t cap, tsg_cmat **out);

// ---------------------------------------------------------------- timing
struct PhaseTimer {
    tsg_ctx *ctx;
    int n;
    explicit PhaseTimer(tsg_ctx *c) : ctx(c), n(0) {}
    void mark() {
        if (ctx->timing && n < 8) cudaEventRecord(ctx->ev[n++], ctx->stream);
    }
    void finish(int total_slot);
};

// ---------------------------------------------------------------- programmatic dependent launch
// The short kernels of a phase's chain (compress, partition, scan) are
// launched with programmatic stream serialisation: the next kernel is
// scheduled while its predecessor drains, and pdl_wait() -- the first
// statement of each such kernel -- holds it until the predecessor's memory is
// visible.  Saves the ~1-2 us launch gap per boundary.  TSG_PDL=0 builds
// plain launches (pdl_wait is then a no-op).
#ifndef TSG_PDL
#define TSG_PDL 1
#endif
__device__ __forceinline__ void pdl_wait() {
#if TSG_PDL
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args &&...args) {
#if TSG_PDL
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
#else
    kernel<<<grid, block, smem, s>>>(std::forward<Args>(args)...);
    return cudaGetLastError();
#endif
}

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ unsigned hash_slot(int key, int logT) {
    return (unsigned)((unsigned)key * 2654435761u) >> (32 - logT);
}

__device__ __forceinline__ int ilog2_pow2(int T) { return 31 - __clz(T); }

__host__ __device__ __forceinline__ int pow2_ceil_i(int64_t x) {
    if (x <= 1) return 1;
#ifdef __CUDA_ARCH__
    return (int)(1ull << (64 - __clzll((unsigned long long)(x - 1))));
#else
    return (int)(1ull << (64 - __builtin_clzll((unsigned long long)(x - 1))));
#endif
}

// table slots for a row holding up to `m` distinct keys: load factor <= 3/4
__host__ __device__ __forceinline__ int table_slots(int64_t m) {
    int64_t need = m + (m + 2) / 3;   // ~4m/3
    int t = pow2_ceil_i(need < 8 ? 8 : need);
    return t;
}

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned r;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
    return r;
}

__device__ __forceinline__ unsigned lane_id() {
    unsigned r;
    asm("mov.u32 %0, %%laneid;" : "=r"(r));
    return r;
}

template <int G>
__device__ __forceinline__ unsigned group_mask() {
    if constexpr (G == 32) return 0xffffffffu;
    else return ((1u << G) - 1u) << (lane_id() & ~(G - 1));
}

// inclusive scan of v over the G lanes of a group
template <int G, typename T>
__device__ __forceinline__ T group_incl_scan(unsigned gm, T v, int glane) {
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
        T o = __shfl_up_sync(gm, v, d, G);
        if (glane >= d) v += o;
    }
    return v;
}

template <int G, typename T>
__device__ __forceinline__ T group_sum(unsigned gm, T v) {
#pragma unroll
    for (int d = G / 2; d >= 1; d >>= 1) v += __shfl_xor_sync(gm, v, d, G);
    return v;
}

// ---------------------------------------------------------------- launch helpers
static inline unsigned grid_for(int64_t work, int per_block, int cap = 1 << 30) {
    int64_t g = (work + per_block - 1) / per_block;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}
