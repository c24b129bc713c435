// tsg_chunk.cu -- physical chunked execution through an HBM budget.
//
// The reference's three orders (chunking.py:219-337) bill a simulated copy
// ledger; here the same orders really move the data.  The slow tier is host
// memory (the caller's arrays, pinned for full PCIe rate), the fast tier is
// HBM:
//   order 1 (gpu chunk1, AC in place): per A/C row range, A rows go H2D once,
//     the C range lives in HBM at its final row capacity while every B row
//     chunk streams past it, then the finished C range goes D2H once.
//   order 2 (gpu chunk2, B in place): per B chunk (resident), every A/C range
//     streams past it; C partials round-trip through host memory.
//   order 0 (KNL): B chunks stream past the whole of A/C (order 1 with one
//     A/C range).
// Every chunk step is the fused multiply-add (kernel.py:235-340) run IN
// PLACE: C rows keep their final capacity and the running partial occupies a
// prefix whose length is tracked per row, so no C copy is ever made on the
// device.  B chunks and A ranges are double-buffered: the next one's H2D runs
// on the copy-in stream while the current one computes; C ranges drain D2H on
// the copy-out stream while the next range computes.  Host formats are the
// reference's (int64 indices): columns travel as int64 and are narrowed /
// widened on the device, so physical PCIe bytes equal the ledger's byte
// convention (csr.py:65-67).
#include <chrono>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <vector>

#include "tsg_internal.cuh"

// implemented in tsg_spgemm.cu
int tsg_compress_impl(tsg_ctx *c, const tsg_csr *b, tsg_cmat **out);
int tsg_fused_inplace(tsg_ctx *c, const tsg_csr *a, int32_t b_lo, int32_t b_hi, const tsg_csr *b,
                      const tsg_cmat *cb, const int64_t *cptr, const int64_t *cap, int32_t *ccol,
                      double *cval, int32_t *plen, int64_t rows);

namespace {

__global__ void k_rebase(const int64_t *__restrict__ in, int64_t *__restrict__ out, int64_t n,
                         int64_t base) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[i] - base;
}

__global__ void k_narrow(const int64_t *__restrict__ in, int32_t *__restrict__ out, int64_t n,
                         int64_t ncols, int *err) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t v = in[i];
        if (ncols >= 0 && (v < 0 || v >= ncols)) {   // ncols < 0: unchecked (stale tails)
            kerr(err, KERR_COLRANGE, i);
            v = 0;
        }
        out[i] = (int32_t)v;
    }
}

__global__ void k_widen(const int32_t *__restrict__ in, int64_t *__restrict__ out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)in[i];
}

__global__ void k_check_full(const int32_t *__restrict__ plen, const int64_t *__restrict__ cap,
                             int64_t n, int64_t row0, int *err) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        if ((int64_t)plen[i] != cap[i]) kerr(err, KERR_ROWSIZE, row0 + i);
}

__global__ void k_caps(const int64_t *__restrict__ cptr, int64_t *__restrict__ cap, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        cap[i] = cptr[i + 1] - cptr[i];
}

// A row range [lo, hi) of a host CSR staged in HBM (rebased row pointers).
struct DevRange {
    tsg_csr m{};          // device view (rp rebased, int32 cols)
    int64_t *stage = nullptr;      // int64 column staging
    int64_t *stage_rp = nullptr;   // int64 row pointer staging
    int64_t cap_rows = 0, cap_nnz = 0;
    cudaEvent_t ready{};           // host data landed (copy-in stream)
    // rebasing / narrowing still owed on the compute stream (see finish_rows)
    bool pending = false;
    int64_t pend_rows = 0, pend_nnz = 0, pend_base = 0, pend_cols = 0;
};

// Optional timeline (TSG_CHUNK_TIMELINE=1): events around every H2D stage,
// D2H drain and fused step, printed relative to the call's start.
struct Timeline {
    bool on = false;
    cudaEvent_t base{};
    std::vector<std::pair<char, std::pair<cudaEvent_t, cudaEvent_t>>> iv;
    void begin(char kind, cudaStream_t s, cudaEvent_t &e0) {
        if (!on) return;
        cudaEventCreate(&e0);
        cudaEventRecord(e0, s);
        (void)kind;
    }
    void end(char kind, cudaStream_t s, cudaEvent_t e0) {
        if (!on) return;
        cudaEvent_t e1;
        cudaEventCreate(&e1);
        cudaEventRecord(e1, s);
        iv.push_back({kind, {e0, e1}});
    }
};
Timeline g_tl;

struct HostCsr {
    int64_t rows, cols;
    const int64_t *rp;
    const int64_t *col;
    const double *val;
};

int ensure(tsg_ctx *c, DevRange &d, int64_t rows, int64_t nnz, bool values, bool *fresh) {
    *fresh = false;
    if (rows > d.cap_rows || nnz > d.cap_nnz) {
        *fresh = true;
        tsg_free(c, d.m.rp);
        tsg_free(c, d.m.col);
        tsg_free(c, d.m.val);
        tsg_free(c, d.stage);
        tsg_free(c, d.stage_rp);
        d.cap_rows = rows > d.cap_rows ? rows : d.cap_rows;
        d.cap_nnz = nnz > d.cap_nnz ? nnz : d.cap_nnz;
        TSG_TRY(tsg_alloc_t(c, &d.m.rp, d.cap_rows + 2));
        TSG_TRY(tsg_alloc_t(c, &d.m.col, d.cap_nnz + 1));
        if (values) TSG_TRY(tsg_alloc_t(c, &d.m.val, d.cap_nnz + 1));
        TSG_TRY(tsg_alloc_t(c, &d.stage, d.cap_nnz + 2));
        TSG_TRY(tsg_alloc_t(c, &d.stage_rp, d.cap_rows + 2));
    }
    if (!d.ready) TSG_CK(cudaEventCreateWithFlags(&d.ready, cudaEventDisableTiming));
    return TSG_OK;
}

void release(tsg_ctx *c, DevRange &d) {
    tsg_free(c, d.m.rp);
    tsg_free(c, d.m.col);
    tsg_free(c, d.m.val);
    tsg_free(c, d.stage);
    tsg_free(c, d.stage_rp);
    if (d.ready) cudaEventDestroy(d.ready);
    d = DevRange();
}

// H2D of host rows [lo, hi) on the copy-in stream -- copies only: a kernel
// queued behind a bulk copy on one stream was measured to hold back kernels
// of other streams until that copy finished, so the rebasing / narrowing is
// owed to the compute stream (finish_rows, right before the first use).
int stage_rows(tsg_ctx *c, const HostCsr &h, int64_t lo, int64_t hi, DevRange &d,
               cudaEvent_t wait_free, int64_t &bytes) {
    const int64_t rows = hi - lo, e0 = h.rp[lo], e1 = h.rp[hi], nnz = e1 - e0;
    bool fresh = false;
    TSG_TRY(ensure(c, d, rows, nnz, h.val != nullptr, &fresh));
    d.m.sorted = 0;      // host rows not inspected here: finish_rows checks them on the device
    d.m.distinct = 0;
    d.m.max_row = -1;
    cudaStream_t s = c->copy_in;
    // freshly allocated buffers come from the compute-stream-ordered arena:
    // order the copy stream after the compute stream's current position
    // (steady state reuses the slot's buffers and waits only for `wait_free`)
    if (fresh) {
        TSG_CK(cudaEventRecord(d.ready, c->stream));
        TSG_CK(cudaStreamWaitEvent(s, d.ready, 0));
    }
    if (wait_free) TSG_CK(cudaStreamWaitEvent(s, wait_free, 0));
    cudaEvent_t tl0{};
    g_tl.begin('H', s, tl0);
    TSG_TRY(tsg_copy(d.stage_rp, h.rp + lo, (rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    if (nnz > 0) {
        TSG_TRY(tsg_copy(d.stage, h.col + e0, nnz * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        if (h.val)
            TSG_TRY(tsg_copy(d.m.val, h.val + e0, nnz * sizeof(double), cudaMemcpyHostToDevice, s));
    }
    g_tl.end('H', s, tl0);
    TSG_CK(cudaEventRecord(d.ready, s));
    d.pending = true;
    d.pend_rows = rows;
    d.pend_nnz = nnz;
    d.pend_base = e0;
    d.pend_cols = h.cols;
    d.m.rows = rows;
    d.m.cols = h.cols;
    d.m.nnz = nnz;
    bytes += (rows + 1) * 8 + nnz * (h.val ? 16 : 8);
    return TSG_OK;
}

// On the compute stream: wait for the staged copies, rebase the row pointers
// and narrow the columns (range-checked) into the device view.
int finish_rows(tsg_ctx *c, DevRange &d) {
    if (!d.pending) return TSG_OK;
    cudaStream_t s = c->stream;
    TSG_CK(cudaStreamWaitEvent(s, d.ready, 0));
    k_rebase<<<grid_for(d.pend_rows + 1, 256, c->num_sms * 8), 256, 0, s>>>(d.stage_rp, d.m.rp,
                                                                           d.pend_rows + 1, d.pend_base);
    ++c->launches;
    if (d.pend_nnz > 0) {
        k_narrow<<<grid_for(d.pend_nnz, 256, c->num_sms * 16), 256, 0, s>>>(d.stage, d.m.col, d.pend_nnz,
                                                                             d.pend_cols, c->d_err);
        ++c->launches;
    }
    TSG_CK(cudaGetLastError());
    d.pending = false;
    if (tsg_trace_enabled()) {
        cudaStreamSynchronize(s);
        int eh[2];
        cudaMemcpy(eh, c->d_err, sizeof(eh), cudaMemcpyDeviceToHost);
        fprintf(stderr, "[tsg chunk] staged %lld rows nnz %lld ncols %lld err %d/%d\n",
                (long long)d.pend_rows, (long long)d.pend_nnz, (long long)d.pend_cols, eh[0], eh[1]);
    }
    return TSG_OK;
}

// C range [lo, hi) resident in HBM at final row capacity
struct DevC {
    int64_t *cptr = nullptr;   // rebased final row pointers (rows + 1)
    int64_t *cap = nullptr;    // capacities (rows)
    int32_t *col = nullptr;
    double *val = nullptr;
    int32_t *plen = nullptr;   // running partial lengths
    int64_t *stage = nullptr;  // int64 column staging for transfers
    int64_t *rp_stage = nullptr;   // host row pointers of the range (copy-in stream)
    int64_t cap_rows = 0, cap_nnz = 0;
    cudaEvent_t drained{};     // D2H of this buffer finished
    cudaEvent_t rp_ready{};    // rp_stage landed
};

int ensure_c(tsg_ctx *c, DevC &d, int64_t rows, int64_t nnz) {
    if (rows > d.cap_rows || nnz > d.cap_nnz) {
        // the old buffers may still be read by this slot's previous D2H
        if (d.drained) TSG_CK(cudaEventSynchronize(d.drained));
        TSG_CK(cudaStreamSynchronize(c->stream));
        tsg_free(c, d.rp_stage);
        tsg_free(c, d.cptr);
        tsg_free(c, d.cap);
        tsg_free(c, d.col);
        tsg_free(c, d.val);
        tsg_free(c, d.plen);
        tsg_free(c, d.stage);
        d.cap_rows = rows > d.cap_rows ? rows : d.cap_rows;
        d.cap_nnz = nnz > d.cap_nnz ? nnz : d.cap_nnz;
        TSG_TRY(tsg_alloc_t(c, &d.cptr, d.cap_rows + 2));
        TSG_TRY(tsg_alloc_t(c, &d.cap, d.cap_rows + 1));
        TSG_TRY(tsg_alloc_t(c, &d.col, d.cap_nnz + 1));
        TSG_TRY(tsg_alloc_t(c, &d.val, d.cap_nnz + 1));
        TSG_TRY(tsg_alloc_t(c, &d.plen, d.cap_rows + 1));
        TSG_TRY(tsg_alloc_t(c, &d.stage, d.cap_nnz + d.cap_rows + 2));
        TSG_TRY(tsg_alloc_t(c, &d.rp_stage, d.cap_rows + 2));
    }
    if (!d.drained) TSG_CK(cudaEventCreateWithFlags(&d.drained, cudaEventDisableTiming));
    if (!d.rp_ready) TSG_CK(cudaEventCreateWithFlags(&d.rp_ready, cudaEventDisableTiming));
    return TSG_OK;
}

// Row pointers of a C range staged early on the copy-in stream, so opening
// the range later does not queue a small H2D behind the bulk chunk copies.
int stage_c_rows(tsg_ctx *c, const int64_t *c_rp, DevC &d, int64_t lo, int64_t hi, int64_t &bytes) {
    const int64_t rows = hi - lo, nnz = c_rp[hi] - c_rp[lo];
    TSG_TRY(ensure_c(c, d, rows, nnz));
    // rp_stage of this slot was last read by open_c of range r-2 on the
    // compute stream; the caller's preceding A stage already made copy-in
    // wait for that range's steps (used_a)
    TSG_TRY(tsg_copy(d.rp_stage, c_rp + lo, (rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, c->copy_in));
    TSG_CK(cudaEventRecord(d.rp_ready, c->copy_in));
    bytes += (rows + 1) * 8;
    return TSG_OK;
}

void release_c(tsg_ctx *c, DevC &d) {
    tsg_free(c, d.cptr);
    tsg_free(c, d.cap);
    tsg_free(c, d.col);
    tsg_free(c, d.val);
    tsg_free(c, d.plen);
    tsg_free(c, d.stage);
    tsg_free(c, d.rp_stage);
    if (d.drained) cudaEventDestroy(d.drained);
    if (d.rp_ready) cudaEventDestroy(d.rp_ready);
    d = DevC();
}

struct Job {
    tsg_ctx *c;
    HostCsr A, B;
    const int64_t *c_rp;
    int64_t *c_col;
    double *c_val;
    int32_t *h_plen;    // host partial lengths (order 2), per row of A
    tsg_chunk_stats *st;
};

// C range setup on the compute stream: row pointers (rebased) + capacities;
// optionally load a partial (order 2) from host.
int open_c(Job &J, DevC &d, int64_t lo, int64_t hi, bool load_partial, bool rp_staged = false) {
    tsg_ctx *c = J.c;
    const int64_t rows = hi - lo, e0 = J.c_rp[lo], nnz = J.c_rp[hi] - e0;
    cudaStream_t s = c->stream;
    if (rp_staged) {
        TSG_CK(cudaStreamWaitEvent(s, d.rp_ready, 0));
    } else {
        TSG_TRY(ensure_c(c, d, rows, nnz));
        TSG_TRY(tsg_copy(d.rp_stage, J.c_rp + lo, (rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        J.st->h2d_bytes += (rows + 1) * 8;
    }
    TSG_CK(cudaStreamWaitEvent(s, d.drained, 0));   // previous D2H of this buffer
    k_rebase<<<grid_for(rows + 1, 256, c->num_sms * 8), 256, 0, s>>>(d.rp_stage, d.cptr, rows + 1, e0); ++c->launches;
    k_caps<<<grid_for(rows, 256, c->num_sms * 8), 256, 0, s>>>(d.cptr, d.cap, rows); ++c->launches;
    if (load_partial) {
        TSG_TRY(tsg_copy(d.plen, J.h_plen + lo, rows * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        if (nnz > 0) {
            TSG_TRY(tsg_copy(d.stage, J.c_col + e0, nnz * sizeof(int64_t), cudaMemcpyHostToDevice, s));
            // only each row's partial prefix (plen) is meaningful; the capacity
            // tail is stale host memory and is never read, so no range check
            k_narrow<<<grid_for(nnz, 256, c->num_sms * 16), 256, 0, s>>>(d.stage, d.col, nnz, -1,
                                                                         c->d_err); ++c->launches;
            TSG_TRY(tsg_copy(d.val, J.c_val + e0, nnz * sizeof(double), cudaMemcpyHostToDevice, s));
        }
        J.st->h2d_bytes += rows * 4 + nnz * 16;
    } else {
        TSG_TRY(tsg_fill(c, d.plen, 0, rows * sizeof(int32_t), s));
    }
    TSG_CK(cudaGetLastError());
    return TSG_OK;
}

// D2H of a C range (columns widened to int64) on the copy-out stream.
int drain_c(Job &J, DevC &d, int64_t lo, int64_t hi, bool with_plen) {
    tsg_ctx *c = J.c;
    const int64_t rows = hi - lo, e0 = J.c_rp[lo], nnz = J.c_rp[hi] - e0;
    cudaEvent_t done;
    TSG_CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    if (nnz > 0) {
        k_widen<<<grid_for(nnz, 256, c->num_sms * 16), 256, 0, c->stream>>>(d.col, d.stage, nnz); ++c->launches;
    }
    TSG_CK(cudaEventRecord(done, c->stream));
    cudaStream_t s = c->copy_out;
    TSG_CK(cudaStreamWaitEvent(s, done, 0));
    cudaEvent_t tl0{};
    g_tl.begin('D', s, tl0);
    if (nnz > 0) {
        TSG_TRY(tsg_copy(J.c_col + e0, d.stage, nnz * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        TSG_TRY(tsg_copy(J.c_val + e0, d.val, nnz * sizeof(double), cudaMemcpyDeviceToHost, s));
    }
    if (with_plen)
        TSG_TRY(tsg_copy(J.h_plen + lo, d.plen, rows * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    g_tl.end('D', s, tl0);
    TSG_CK(cudaEventRecord(d.drained, s));
    TSG_CK(cudaEventDestroy(done));
    J.st->d2h_bytes += nnz * 16 + (with_plen ? rows * 4 : 0);
    return TSG_OK;
}

}  // namespace

extern "C" int tsg_chunk_multiply(tsg_ctx *c, int algo, int64_t a_rows, int64_t a_cols,
                                  const int64_t *a_rp, const int64_t *a_col, const double *a_val,
                                  int64_t b_rows, int64_t b_cols, const int64_t *b_rp,
                                  const int64_t *b_col, const double *b_val, const int64_t *c_rp,
                                  int64_t *c_col, double *c_val, int64_t n_ac,
                                  const int64_t *ac_bounds, int64_t n_b, const int64_t *b_bounds,
                                  tsg_chunk_stats *stats) {
    if (a_cols != b_rows) {
        tsg_set_error("A has %lld cols but B has %lld rows", (long long)a_cols, (long long)b_rows);
        return TSG_EDIM;
    }
    if (!a_val || !b_val) {
        tsg_set_error("chunked multiply requires values on both operands");
        return TSG_EVALID;
    }
    if (algo < 0 || algo > 2 || n_ac < 1 || n_b < 1 || ac_bounds[0] != 0 || ac_bounds[n_ac] != a_rows ||
        b_bounds[0] != 0 || b_bounds[n_b] != b_rows) {
        tsg_set_error("invalid chunk plan");
        return TSG_EARG;
    }
    tsg_chunk_stats local;
    memset(&local, 0, sizeof(local));
    g_tl = Timeline();
    g_tl.on = getenv("TSG_CHUNK_TIMELINE") != nullptr;
    if (g_tl.on) {
        cudaEventCreate(&g_tl.base);
        cudaEventRecord(g_tl.base, c->stream);
    }
    auto t0 = std::chrono::steady_clock::now();
    Job J{c, {a_rows, a_cols, a_rp, a_col, a_val}, {b_rows, b_cols, b_rp, b_col, b_val}, c_rp,
          c_col, c_val, nullptr, &local};
    // host partial lengths (order 2): pinned, so their D2H stays asynchronous
    // (a copy into pageable memory would block the host until the whole C
    // drain ahead of it finished)
    int32_t *plen_host = nullptr;
    constexpr int NBS = 3;   // B chunk slots: the copy two steps ahead never waits on compute
    DevRange Abuf[2], Bbuf[NBS];
    DevC Cbuf[2];
    cudaEvent_t used[NBS] = {nullptr, nullptr, nullptr};   // compute finished with a Bbuf slot
    for (int i = 0; i < NBS; i++) TSG_CK(cudaEventCreateWithFlags(&used[i], cudaEventDisableTiming));
    cudaEvent_t used_a[2] = {nullptr, nullptr};   // compute finished with Abuf slot
    for (int i = 0; i < 2; i++) TSG_CK(cudaEventCreateWithFlags(&used_a[i], cudaEventDisableTiming));
    // per-step kernel timing events, read once at the end: the host never
    // waits for a fused step, so the next chunks' copies queue behind it
    std::vector<cudaEvent_t> kev;
    float kernel_ms = 0.f;
    int st = TSG_OK;

    auto fused_step = [&](DevRange &A, DevRange &B, DevC &C, int64_t blo, int64_t bhi,
                          int64_t rows) -> int {
        TSG_TRY(finish_rows(c, A));
        const bool fresh_b = B.pending;
        TSG_TRY(finish_rows(c, B));
        // row order of a freshly staged B chunk, learnt on the device: enables
        // the compress fast path and the lane-split numeric mode (a short host
        // wait for the compute stream, once per staged chunk)
        if (fresh_b) TSG_TRY(tsg_csr_check_sorted(c, &B.m));
        cudaEvent_t e0, e1;
        TSG_CK(cudaEventCreate(&e0));
        TSG_CK(cudaEventCreate(&e1));
        kev.push_back(e0);
        kev.push_back(e1);
        TSG_CK(cudaEventRecord(e0, c->stream));
        tsg_cmat *cb = nullptr;
        TSG_TRY(tsg_compress_impl(c, &B.m, &cb));
        int s2 = tsg_fused_inplace(c, &A.m, (int32_t)blo, (int32_t)bhi, &B.m, cb, C.cptr, C.cap, C.col,
                                   C.val, C.plen, rows);

        tsg_cmat_free(c, cb);
        TSG_TRY(s2);
        TSG_CK(cudaEventRecord(e1, c->stream));
        return TSG_OK;
    };

    {
        const int64_t *acb = ac_bounds;
        int64_t nac = n_ac;
        int64_t whole[2] = {0, a_rows};
        if (algo == 0) {
            acb = whole;
            nac = 1;
        }
        // every slot sized for the largest range / chunk before the pipeline
        // starts: a mid-run reallocation would have to wait for the slot's
        // in-flight users (and can make the pool grow under running copies)
        {
            int64_t ar = 0, an = 0, cr = 0, cn = 0, br = 0, bn = 0;
            for (int64_t r = 0; r < nac; ++r) {
                const int64_t lo = acb[r], hi = acb[r + 1];
                ar = std::max(ar, hi - lo);
                an = std::max(an, a_rp[hi] - a_rp[lo]);
                cn = std::max(cn, c_rp[hi] - c_rp[lo]);
            }
            cr = ar;
            for (int64_t j = 0; j < n_b; ++j) {
                br = std::max(br, b_bounds[j + 1] - b_bounds[j]);
                bn = std::max(bn, b_rp[b_bounds[j + 1]] - b_rp[b_bounds[j]]);
            }
            bool fresh = false;
            for (int i = 0; i < 2 && st == TSG_OK; ++i) {
                st = ensure(c, Abuf[i], ar, an, true, &fresh);
                if (st == TSG_OK) st = ensure_c(c, Cbuf[i], cr, cn);
            }
            // order 2 alternates two B slots (one if B is a single chunk)
            const int nbs = algo == 2 ? (n_b > 1 ? 2 : 1) : (int)std::min<int64_t>(NBS, nac * n_b);
            for (int i = 0; i < nbs && st == TSG_OK; ++i) st = ensure(c, Bbuf[i], br, bn, true, &fresh);
            // grow the driver pool once by the per-step temporaries (compressed
            // B chunk, symbolic / numeric scratch of a range): growing it later
            // maps memory while copies are in flight and stalls host and device
            const size_t grow = (size_t)(bn * 16 + br * 16 + ar * 96) + ((size_t)256 << 20);
            void *tmp = nullptr;
            if (st == TSG_OK && cudaMallocAsync(&tmp, grow, c->stream) == cudaSuccess)
                cudaFreeAsync(tmp, c->stream);
            else
                cudaGetLastError();
            TSG_CK(cudaStreamSynchronize(c->stream));
        }
    }
    if (algo == 0 || algo == 1) {
        const int64_t *acb = ac_bounds;
        int64_t nac = n_ac;
        int64_t whole[2] = {0, a_rows};
        if (algo == 0) {
            acb = whole;
            nac = 1;
        }
        // Flat schedule over steps s = (range r, chunk j): before step s runs,
        // the copies of step s+2 are queued (A range when j == 0, B chunk in
        // slot s % NBS), so the copy engine always has the next transfers
        // queued while the host blocks inside a fused step.  C ranges are
        // opened on the compute stream right before their first step.
        const int64_t nsteps = nac * n_b;

        auto issue = [&](int64_t s2) -> int {
            const int64_t r = s2 / n_b, j = s2 % n_b;
            if (j == 0) {   // this A slot was last read by range r-2's steps
                TSG_TRY(stage_rows(c, J.A, acb[r], acb[r + 1], Abuf[r & 1], used_a[r & 1],
                                   local.h2d_bytes));
                TSG_TRY(stage_c_rows(c, J.c_rp, Cbuf[r & 1], acb[r], acb[r + 1], local.h2d_bytes));
            }
            return stage_rows(c, J.B, b_bounds[j], b_bounds[j + 1], Bbuf[s2 % NBS], used[s2 % NBS],
                              local.h2d_bytes);
        };
        for (int64_t s2 = 0; s2 < 2 && s2 < nsteps && st == TSG_OK; ++s2) st = issue(s2);
        auto hnow = [&]() {
            return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        };
        for (int64_t s2 = 0; s2 < nsteps && st == TSG_OK; ++s2) {
            const int64_t r = s2 / n_b, j = s2 % n_b;
            const int64_t lo = acb[r], hi = acb[r + 1];
            DevC &C = Cbuf[r & 1];
            const double h0 = hnow();
            if (j == 0 && (st = open_c(J, C, lo, hi, false, true)) != TSG_OK) break;
            if (s2 + 2 < nsteps && (st = issue(s2 + 2)) != TSG_OK) break;
            const double h1 = hnow();
            st = fused_step(Abuf[r & 1], Bbuf[s2 % NBS], C, b_bounds[j], b_bounds[j + 1], hi - lo);
            if (g_tl.on)
                fprintf(stderr, "[tsg host] step %lld issue %.3f-%.3f fused %.3f-%.3f\n", (long long)s2, h0, h1,
                        h1, hnow());
            cudaEventRecord(used[s2 % NBS], c->stream);
            if (st == TSG_OK && j == n_b - 1) {
                cudaEventRecord(used_a[r & 1], c->stream);
                k_check_full<<<grid_for(hi - lo, 256, c->num_sms * 8), 256, 0, c->stream>>>(
                    C.plen, C.cap, hi - lo, lo, c->d_err); ++c->launches;
                st = drain_c(J, C, lo, hi, false);
            }
        }
    } else {
        void *ph = nullptr;
        TSG_TRY(tsg_host_alloc(((size_t)a_rows + 1) * sizeof(int32_t), &ph));
        plen_host = static_cast<int32_t *>(ph);
        memset(plen_host, 0, ((size_t)a_rows + 1) * sizeof(int32_t));
        J.h_plen = plen_host;
        for (int64_t j = 0; j < n_b && st == TSG_OK; ++j) {
            DevRange &B = Bbuf[j & 1];
            if ((st = stage_rows(c, J.B, b_bounds[j], b_bounds[j + 1], B, used[j & 1], local.h2d_bytes)) != TSG_OK)
                break;
            for (int64_t r = 0; r < n_ac && st == TSG_OK; ++r) {
                const int64_t lo = ac_bounds[r], hi = ac_bounds[r + 1];
                DevRange &A = Abuf[r & 1];
                DevC &C = Cbuf[r & 1];
                if ((st = stage_rows(c, J.A, lo, hi, A, used_a[r & 1], local.h2d_bytes)) != TSG_OK) break;
                // partials come back from host after the first B sweep; the D2H
                // of the previous sweep for this range must have landed (the
                // first sweep loads nothing, so its ranges pipeline freely)
                if (j > 0) TSG_CK(cudaStreamSynchronize(c->copy_out));
                if ((st = open_c(J, C, lo, hi, j > 0)) != TSG_OK) break;
                st = fused_step(A, B, C, b_bounds[j], b_bounds[j + 1], hi - lo);
                cudaEventRecord(used_a[r & 1], c->stream);
                if (st == TSG_OK) st = drain_c(J, C, lo, hi, true);
            }
            cudaEventRecord(used[j & 1], c->stream);
        }
    }
    cudaStreamSynchronize(c->copy_in);
    cudaStreamSynchronize(c->copy_out);
    cudaStreamSynchronize(c->stream);
    if (st == TSG_OK) st = tsg_check_kernel_errors(c, "chunked multiply");
    if (st == TSG_OK && algo == 2) {
        for (int64_t i = 0; i < a_rows; ++i)
            if (plen_host[i] != c_rp[i + 1] - c_rp[i]) {
                tsg_set_error("chunked result rows disagree with symbolic counts (row %lld: %d vs %lld)",
                              (long long)i, plen_host[i], (long long)(c_rp[i + 1] - c_rp[i]));
                st = TSG_EDIM;
                break;
            }
    }
    if (plen_host) tsg_host_free(plen_host);
    int64_t mem = c->bytes_in_use;
    for (int i = 0; i < 2; i++) {
        release(c, Abuf[i]);
        release(c, Bbuf[i]);
        if (i == 1) release(c, Bbuf[2]);
        release_c(c, Cbuf[i]);
        cudaEventDestroy(used[i]);
        if (i == 1) cudaEventDestroy(used[2]);
    }
    for (size_t k = 0; k + 1 < kev.size(); k += 2) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, kev[k], kev[k + 1]) == cudaSuccess) kernel_ms += ms;
        else cudaGetLastError();
        if (g_tl.on) g_tl.iv.push_back({'K', {kev[k], kev[k + 1]}});
    }
    if (g_tl.on) {
        for (auto &x : g_tl.iv) {
            float a0 = 0.f, a1 = 0.f;
            cudaEventElapsedTime(&a0, g_tl.base, x.second.first);
            cudaEventElapsedTime(&a1, g_tl.base, x.second.second);
            fprintf(stderr, "[tsg timeline] %c %.3f %.3f\n", x.first, a0, a1);
            if (x.first != 'K') {
                cudaEventDestroy(x.second.first);
                cudaEventDestroy(x.second.second);
            }
        }
        cudaEventDestroy(g_tl.base);
        g_tl = Timeline();
    }
    for (cudaEvent_t e : kev) cudaEventDestroy(e);
    for (int i = 0; i < 2; i++) cudaEventDestroy(used_a[i]);
    cudaStreamSynchronize(c->stream);
    local.kernel_ms = kernel_ms;
    local.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    local.peak_device_bytes = mem;
    if (stats) *stats = local;
    return st;
}

const void *tsg_kernel_chunk() { return (const void *)k_rebase; }
