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
//     A/C range, split physically as the budget requires).
// Every chunk step is the fused multiply-add (kernel.py:235-340) run IN
// PLACE: C rows keep their final capacity and the running partial occupies a
// prefix whose length is tracked per row, so no C copy is ever made on the
// device.  Host formats are the reference's (int64 indices): columns travel
// as int64 and are narrowed / widened on the device, so physical PCIe bytes
// equal the ledger's byte convention (csr.py:65-67).
//
// The HBM budget (the planner's fast_size, chunking.py:21-22) is honoured
// PHYSICALLY, like the reference's residency checks (memory.py:103-111):
// before the run the executor sizes every slot it will hold -- A ranges
// (double-buffered when they fit), C ranges (double-buffered when they fit,
// so a range drains while the next computes), B chunks (up to three slots,
// the copy two steps ahead), the per-step scratch (compressed B chunk,
// partition, bounds) -- and picks the buffering / splitting that fits:
//   * B chunks of order 0/1 are split into sub-chunks (traffic-neutral; only
//     when every A row is column-sorted, so each C entry still accumulates in
//     the reference's order),
//   * A/C ranges of order 2 into sub-ranges (traffic-neutral: A/C stream per
//     B chunk anyway), and as a last resort those of order 0/1 (B then
//     streams once per sub-range: more PCIe bytes, reported as such).
// Columns are converted in place of the value buffers (int64 columns land in
// the slot's fp64 array, are narrowed on the convert stream, then the values
// follow), so no full-size staging array exists.  The context's allocation
// high-water mark during the call is reported as peak_device_bytes and must
// not exceed the budget (TSG_ECAPACITY otherwise).
#include <chrono>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <thread>
#include <vector>

#include "tsg_internal.cuh"

// implemented in tsg_spgemm.cu
int tsg_compress_impl(tsg_ctx *c, const tsg_csr *b, tsg_cmat **out);
int tsg_fused_inplace(tsg_ctx *c, const tsg_csr *a, int32_t b_lo, int32_t b_hi, const tsg_csr *b,
                      const tsg_cmat *cb, const int64_t *cptr, const int64_t *cap, int32_t *ccol,
                      double *cval, int32_t *plen, int64_t rows);
int tsg_symbolic_impl(tsg_ctx *c, int64_t rows_out, const tsg_csr *a, int64_t a_row_off, int32_t b_lo,
                      int32_t b_hi, const tsg_cmat *cb, const tsg_csr *partial, tsg_vec **out,
                      int64_t **sbound_out);

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

// ---------------------------------------------------------------- host-side row facts

struct HostCsr {
    int64_t rows, cols;
    const int64_t *rp;
    const int64_t *col;
    const double *val;
};

// Whether every row's columns ascend (sorted) and never repeat (distinct):
// one pass over the host columns on a few threads.  Decides whether B chunks
// may be split (A sorted) and the lane-split numeric mode (B distinct).
void host_row_order(const HostCsr &h, bool *sorted, bool *distinct) {
    const int64_t rows = h.rows;
    unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    if (h.rp[rows] < ((int64_t)1 << 22)) nt = 1;
    std::vector<int> uns(nt, 0), dup(nt, 0);
    auto work = [&](unsigned t) {
        const int64_t lo = rows * t / nt, hi = rows * (t + 1) / nt;
        int u = 0, d = 0;
        for (int64_t i = lo; i < hi && !u; ++i)
            for (int64_t e = h.rp[i] + 1; e < h.rp[i + 1]; ++e) {
                if (h.col[e] < h.col[e - 1]) { u = 1; break; }
                if (h.col[e] == h.col[e - 1]) d = 1;
            }
        uns[t] = u;
        dup[t] = d;
    };
    std::vector<std::thread> th;
    for (unsigned t = 1; t < nt; ++t) th.emplace_back(work, t);
    work(0);
    for (auto &x : th) x.join();
    bool u = false, d = false;
    for (unsigned t = 0; t < nt; ++t) {
        u |= uns[t] != 0;
        d |= dup[t] != 0;
    }
    *sorted = !u;
    *distinct = !u && !d;
}

int64_t host_max_row(const int64_t *rp, int64_t lo, int64_t hi) {
    int64_t m = 0;
    for (int64_t i = lo; i < hi; ++i) m = std::max(m, rp[i + 1] - rp[i]);
    return m;
}

// Split each range of `bounds` into `k` sub-ranges of near-equal entries
// (by the host row pointers); empty pieces are dropped.
std::vector<int64_t> refine(const int64_t *bounds, int64_t n, int k, const int64_t *rp) {
    std::vector<int64_t> out{bounds[0]};
    for (int64_t r = 0; r < n; ++r) {
        const int64_t lo = bounds[r], hi = bounds[r + 1];
        for (int p = 1; p <= k; ++p) {
            int64_t cut;
            if (p == k) {
                cut = hi;
            } else {
                const int64_t target = rp[lo] + (rp[hi] - rp[lo]) * p / k;
                cut = std::lower_bound(rp + lo, rp + hi + 1, target) - rp;
                cut = std::max(cut, out.back());
                cut = std::min(cut, hi);
            }
            if (cut > out.back()) out.push_back(cut);
        }
        if (out.back() != hi) out.push_back(hi);
    }
    return out;
}

// ---------------------------------------------------------------- device slots

// A row range [lo, hi) of a host CSR staged in HBM (rebased row pointers).
struct DevRange {
    tsg_csr m{};                   // device view (rp rebased, int32 cols, fp64 vals)
    int64_t *stage_rp = nullptr;   // int64 host row pointers of the range
    int64_t cap_rows = 0, cap_nnz = 0;
    cudaEvent_t cols_in{}, conv{}, ready{};
};

// the arena's size class of an allocation (tsg_core.cu size_class)
int64_t rnd(int64_t bytes) {
    if (bytes <= 4096) return 4096;
    if (bytes <= ((int64_t)1 << 20)) {
        int64_t p = 4096;
        while (p < bytes) p <<= 1;
        return p;
    }
    return (bytes + ((int64_t)1 << 20) - 1) & ~(((int64_t)1 << 20) - 1);
}

int64_t slot_ab_bytes(int64_t rows, int64_t nnz) {
    return rnd(8 * (rows + 2)) + rnd(4 * (nnz + 1)) + rnd(8 * (nnz + 1)) + rnd(8 * (rows + 2));
}

int64_t slot_c_bytes(int64_t rows, int64_t nnz) {
    return rnd(8 * (rows + 2)) + rnd(8 * (rows + 1)) + rnd(4 * (nnz + 1)) + rnd(8 * (nnz + 1)) +
           rnd(4 * (rows + 1));
}

// per-step temporaries: compressed B chunk (tsg_compress_impl: 12 B per
// entry + 12 B per row output, head / prefix bit words, per-row fallback
// arrays) and the fused step's bounds / bins / row lists
int64_t step_scratch_bytes(int64_t ac_rows, int64_t b_rows, int64_t b_nnz) {
    const int64_t compress = rnd(8 * (b_rows + 1)) + rnd(4 * (b_rows + 2)) + rnd(4 * (b_nnz + 1)) +
                             rnd(8 * (b_nnz + 1)) + 3 * rnd(4 * (b_nnz / 32 + 1)) +
                             rnd(8 * (b_nnz / 8192 + 2)) * 2 + rnd(4 * (b_rows + 1)) + rnd(8 * (b_rows + 1));
    const int64_t fused = rnd(8 * (ac_rows + 1)) + rnd(ac_rows + 1) + rnd(4 * (ac_rows + 1)) +
                          rnd(4 * (ac_rows / 1024 + 1) * 16) * 2;
    return compress + fused + ((int64_t)4 << 20);
}

int ensure(tsg_ctx *c, DevRange &d, int64_t rows, int64_t nnz) {
    if (rows > d.cap_rows || nnz > d.cap_nnz) {
        TSG_CK(cudaStreamSynchronize(c->stream));
        tsg_free(c, d.m.rp);
        tsg_free(c, d.m.col);
        tsg_free(c, d.m.val);
        tsg_free(c, d.stage_rp);
        d.cap_rows = std::max(rows, d.cap_rows);
        d.cap_nnz = std::max(nnz, d.cap_nnz);
        TSG_TRY(tsg_alloc_t(c, &d.m.rp, d.cap_rows + 2));
        TSG_TRY(tsg_alloc_t(c, &d.m.col, d.cap_nnz + 1));
        TSG_TRY(tsg_alloc_t(c, &d.m.val, d.cap_nnz + 1));
        TSG_TRY(tsg_alloc_t(c, &d.stage_rp, d.cap_rows + 2));
    }
    if (!d.ready) {
        TSG_CK(cudaEventCreateWithFlags(&d.ready, cudaEventDisableTiming));
        TSG_CK(cudaEventCreateWithFlags(&d.cols_in, cudaEventDisableTiming));
        TSG_CK(cudaEventCreateWithFlags(&d.conv, cudaEventDisableTiming));
    }
    return TSG_OK;
}

void release(tsg_ctx *c, DevRange &d) {
    tsg_free(c, d.m.rp);
    tsg_free(c, d.m.col);
    tsg_free(c, d.m.val);
    tsg_free(c, d.stage_rp);
    if (d.ready) {
        cudaEventDestroy(d.ready);
        cudaEventDestroy(d.cols_in);
        cudaEventDestroy(d.conv);
    }
    d = DevRange();
}

// Optional timeline (TSG_CHUNK_TIMELINE=1): events around every H2D stage,
// D2H drain and fused step, printed relative to the call's start.
struct Timeline {
    bool on = false;
    cudaEvent_t base{};
    std::vector<std::pair<char, std::pair<cudaEvent_t, cudaEvent_t>>> iv;
    void begin(cudaStream_t s, cudaEvent_t &e0) {
        if (!on) return;
        cudaEventCreate(&e0);
        cudaEventRecord(e0, s);
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

// H2D of host rows [lo, hi) on the copy-in stream.  The int64 columns land in
// the slot's value array, the convert stream narrows them into the int32
// column array (and rebases the row pointers), then the values overwrite the
// staging.  No kernel is ever queued on the copy stream (a kernel queued
// behind a bulk copy was measured to hold back kernels of other streams).
int stage_rows(tsg_ctx *c, const HostCsr &h, int64_t lo, int64_t hi, DevRange &d, cudaEvent_t wait_free,
               bool sorted, bool distinct, int64_t &bytes, bool one_stream = false) {
    const int64_t rows = hi - lo, e0 = h.rp[lo], e1 = h.rp[hi], nnz = e1 - e0;
    TSG_TRY(ensure(c, d, rows, nnz));
    d.m.sorted = sorted ? 1 : 0;
    d.m.distinct = distinct ? 1 : 0;
    d.m.max_row = host_max_row(h.rp, lo, hi);
    // alternate the two H2D streams: while this piece's values wait for the
    // column conversion, the next piece's columns are already on the link
    static thread_local unsigned flip = 0;
    cudaStream_t s = (!one_stream && (flip++ & 1)) ? c->copy_in2 : c->copy_in, cs = c->convert;
    if (wait_free) TSG_CK(cudaStreamWaitEvent(s, wait_free, 0));
    cudaEvent_t tl0{}, tl1{}, tl2{};
    g_tl.begin(s, tl0);
    TSG_TRY(tsg_copy(d.stage_rp, h.rp + lo, (rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    int64_t *col64 = reinterpret_cast<int64_t *>(d.m.val);
    if (nnz > 0) TSG_TRY(tsg_copy(col64, h.col + e0, nnz * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    g_tl.end('c', s, tl0);
    TSG_CK(cudaEventRecord(d.cols_in, s));
    TSG_CK(cudaStreamWaitEvent(cs, d.cols_in, 0));
    g_tl.begin(cs, tl1);
    k_rebase<<<grid_for(rows + 1, 256, c->num_sms * 8), 256, 0, cs>>>(d.stage_rp, d.m.rp, rows + 1, e0);
    ++c->launches;
    if (nnz > 0) {
        k_narrow<<<grid_for(nnz, 256, c->num_sms * 16), 256, 0, cs>>>(col64, d.m.col, nnz, h.cols, c->d_err);
        ++c->launches;
    }
    TSG_CK(cudaGetLastError());
    g_tl.end('n', cs, tl1);
    TSG_CK(cudaEventRecord(d.conv, cs));
    TSG_CK(cudaStreamWaitEvent(s, d.conv, 0));
    g_tl.begin(s, tl2);
    if (nnz > 0 && h.val)
        TSG_TRY(tsg_copy(d.m.val, h.val + e0, nnz * sizeof(double), cudaMemcpyHostToDevice, s));
    g_tl.end('v', s, tl2);
    TSG_CK(cudaEventRecord(d.ready, s));
    d.m.rows = rows;
    d.m.cols = h.cols;
    d.m.nnz = nnz;
    bytes += (rows + 1) * 8 + nnz * (h.val ? 16 : 8);
    return TSG_OK;
}

// Resident-B upload in pieces (order 2 with one B chunk): the row pointers
// first, then NP pieces of columns (narrowed on the convert stream) and
// values in row order on one H2D stream, each piece's landing an event.  A/C
// ranges whose largest column lies below a landed prefix run against that
// prefix while the rest of B is still on the link, so the C drain (the
// D2H-bound part of the order) starts ~1/NP of B's upload time after the
// call instead of after all of it.  Results are identical: such a range's
// products all come from the prefix rows, in the same order.
struct BPieces {
    std::vector<int64_t> q;          // piece row bounds, relative to the chunk's first row
    std::vector<cudaEvent_t> ev;     // piece k landed (implies pieces < k)
    int issued = 0;                  // pieces queued so far
};

int stage_b_begin(tsg_ctx *c, const HostCsr &h, int64_t lo, int64_t hi, DevRange &d, cudaEvent_t wait_free,
                  bool sorted, bool distinct, int64_t &bytes, int np, BPieces &bp) {
    const int64_t rows = hi - lo, e0 = h.rp[lo], e1 = h.rp[hi], nnz = e1 - e0;
    TSG_TRY(ensure(c, d, rows, nnz));
    d.m.sorted = sorted ? 1 : 0;
    d.m.distinct = distinct ? 1 : 0;
    d.m.max_row = host_max_row(h.rp, lo, hi);
    cudaStream_t s = c->copy_in, cs = c->convert;
    if (wait_free) TSG_CK(cudaStreamWaitEvent(s, wait_free, 0));
    TSG_TRY(tsg_copy(d.stage_rp, h.rp + lo, (rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    TSG_CK(cudaEventRecord(d.cols_in, s));
    TSG_CK(cudaStreamWaitEvent(cs, d.cols_in, 0));
    k_rebase<<<grid_for(rows + 1, 256, c->num_sms * 8), 256, 0, cs>>>(d.stage_rp, d.m.rp, rows + 1, e0);
    ++c->launches;
    bp.q.assign(1, 0);
    for (int k = 1; k < np; ++k) {   // pieces of near-equal entries, whole rows
        const int64_t target = e0 + nnz * k / np;
        const int64_t r = std::upper_bound(h.rp + lo, h.rp + hi + 1, target) - (h.rp + lo) - 1;
        bp.q.push_back(std::max<int64_t>(bp.q.back(), std::min<int64_t>(r, rows)));
    }
    bp.q.push_back(rows);
    bp.issued = 0;
    d.m.rows = rows;
    d.m.cols = h.cols;
    d.m.nnz = nnz;
    bytes += (rows + 1) * 8 + nnz * (h.val ? 16 : 8);
    return TSG_OK;
}

// queue pieces up to k (in order, on the copy-in stream: the A ranges share
// that FIFO, so each lands right after the B rows it needs)
int stage_b_upto(tsg_ctx *c, const HostCsr &h, int64_t lo, DevRange &d, int k, BPieces &bp) {
    const int64_t e0 = h.rp[lo];
    cudaStream_t s = c->copy_in, cs = c->convert;
    int64_t *col64 = reinterpret_cast<int64_t *>(d.m.val);
    for (; bp.issued <= k; ++bp.issued) {
        const int p = bp.issued;
        const int64_t p0 = h.rp[lo + bp.q[p]] - e0, p1 = h.rp[lo + bp.q[p + 1]] - e0, n = p1 - p0;
        cudaEvent_t ev;
        TSG_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        bp.ev.push_back(ev);
        if (n > 0) {
            cudaEvent_t tl0{}, tl1{};
            g_tl.begin(s, tl0);
            TSG_TRY(tsg_copy(col64 + p0, h.col + e0 + p0, n * sizeof(int64_t), cudaMemcpyHostToDevice, s));
            g_tl.end('c', s, tl0);
            TSG_CK(cudaEventRecord(d.cols_in, s));
            TSG_CK(cudaStreamWaitEvent(cs, d.cols_in, 0));
            k_narrow<<<grid_for(n, 256, c->num_sms * 16), 256, 0, cs>>>(col64 + p0, d.m.col + p0, n, h.cols,
                                                                         c->d_err);
            ++c->launches;
            TSG_CK(cudaGetLastError());
            TSG_CK(cudaEventRecord(d.conv, cs));
            TSG_CK(cudaStreamWaitEvent(s, d.conv, 0));
            g_tl.begin(s, tl1);
            if (h.val) TSG_TRY(tsg_copy(d.m.val + p0, h.val + e0 + p0, n * sizeof(double), cudaMemcpyHostToDevice, s));
            g_tl.end('v', s, tl1);
        } else {
            TSG_CK(cudaEventRecord(d.conv, cs));   // the row pointers' rebase
            TSG_CK(cudaStreamWaitEvent(s, d.conv, 0));
        }
        TSG_CK(cudaEventRecord(ev, s));
        if (p == (int)bp.q.size() - 2) TSG_CK(cudaEventRecord(d.ready, s));
    }
    return TSG_OK;
}

// C range [lo, hi) resident in HBM at final row capacity
struct DevC {
    int64_t *cptr = nullptr;   // rebased final row pointers (rows + 1)
    int64_t *cap = nullptr;    // capacities (rows)
    int32_t *col = nullptr;
    double *val = nullptr;     // also the int64 column staging of transfers
    int32_t *plen = nullptr;   // running partial lengths
    int64_t cap_rows = 0, cap_nnz = 0;
    cudaEvent_t drained{};     // D2H of this buffer finished
    cudaEvent_t done{}, vals_out{}, widened{};
};

int ensure_c(tsg_ctx *c, DevC &d, int64_t rows, int64_t nnz) {
    if (rows > d.cap_rows || nnz > d.cap_nnz) {
        if (d.drained) TSG_CK(cudaEventSynchronize(d.drained));
        TSG_CK(cudaStreamSynchronize(c->stream));
        tsg_free(c, d.cptr);
        tsg_free(c, d.cap);
        tsg_free(c, d.col);
        tsg_free(c, d.val);
        tsg_free(c, d.plen);
        d.cap_rows = std::max(rows, d.cap_rows);
        d.cap_nnz = std::max(nnz, d.cap_nnz);
        TSG_TRY(tsg_alloc_t(c, &d.cptr, d.cap_rows + 2));
        TSG_TRY(tsg_alloc_t(c, &d.cap, d.cap_rows + 1));
        TSG_TRY(tsg_alloc_t(c, &d.col, d.cap_nnz + 1));
        TSG_TRY(tsg_alloc_t(c, &d.val, d.cap_nnz + 1));
        TSG_TRY(tsg_alloc_t(c, &d.plen, d.cap_rows + 1));
    }
    if (!d.drained) {
        TSG_CK(cudaEventCreateWithFlags(&d.drained, cudaEventDisableTiming));
        TSG_CK(cudaEventCreateWithFlags(&d.done, cudaEventDisableTiming));
        TSG_CK(cudaEventCreateWithFlags(&d.vals_out, cudaEventDisableTiming));
        TSG_CK(cudaEventCreateWithFlags(&d.widened, cudaEventDisableTiming));
    }
    return TSG_OK;
}

void release_c(tsg_ctx *c, DevC &d) {
    tsg_free(c, d.cptr);
    tsg_free(c, d.cap);
    tsg_free(c, d.col);
    tsg_free(c, d.val);
    tsg_free(c, d.plen);
    if (d.drained) {
        cudaEventDestroy(d.drained);
        cudaEventDestroy(d.done);
        cudaEventDestroy(d.vals_out);
        cudaEventDestroy(d.widened);
    }
    d = DevC();
}

// Row pointers of a C range, staged early on the copy-in stream (two small
// buffers, independent of the C slots) so opening the range later does not
// queue a small H2D behind the bulk chunk copies.
struct CRows {
    int64_t *rp = nullptr;
    int64_t cap_rows = 0;
    cudaEvent_t ready{}, used{};
};

int stage_c_rows(tsg_ctx *c, const int64_t *c_rp, CRows &d, int64_t lo, int64_t hi, int64_t &bytes) {
    const int64_t rows = hi - lo;
    // this buffer was last read by open_c two ranges ago (compute stream)
    TSG_CK(cudaStreamWaitEvent(c->copy_in, d.used, 0));
    TSG_TRY(tsg_copy(d.rp, c_rp + lo, (rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, c->copy_in));
    TSG_CK(cudaEventRecord(d.ready, c->copy_in));
    bytes += (rows + 1) * 8;
    return TSG_OK;
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
// optionally load a partial (order 2) from host.  `staged`: the row pointers
// were queued on the copy-in stream by stage_c_rows; else they are copied
// here on the compute stream into the same buffer.
int open_c(Job &J, DevC &d, CRows &cr, bool staged, int64_t lo, int64_t hi, bool load_partial) {
    tsg_ctx *c = J.c;
    const int64_t rows = hi - lo, e0 = J.c_rp[lo], nnz = J.c_rp[hi] - e0;
    cudaStream_t s = c->stream;
    TSG_CK(cudaStreamWaitEvent(s, d.drained, 0));   // previous D2H of this buffer
    if (staged) {
        TSG_CK(cudaStreamWaitEvent(s, cr.ready, 0));
    } else {
        TSG_TRY(tsg_copy(cr.rp, J.c_rp + lo, (rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        J.st->h2d_bytes += (rows + 1) * 8;
    }
    k_rebase<<<grid_for(rows + 1, 256, c->num_sms * 8), 256, 0, s>>>(cr.rp, d.cptr, rows + 1, e0); ++c->launches;
    k_caps<<<grid_for(rows, 256, c->num_sms * 8), 256, 0, s>>>(d.cptr, d.cap, rows); ++c->launches;
    TSG_CK(cudaEventRecord(cr.used, s));
    if (load_partial) {
        TSG_TRY(tsg_copy(d.plen, J.h_plen + lo, rows * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        if (nnz > 0) {
            int64_t *col64 = reinterpret_cast<int64_t *>(d.val);
            TSG_TRY(tsg_copy(col64, J.c_col + e0, nnz * sizeof(int64_t), cudaMemcpyHostToDevice, s));
            // only each row's partial prefix (plen) is meaningful; the capacity
            // tail is stale host memory and is never read, so no range check
            k_narrow<<<grid_for(nnz, 256, c->num_sms * 16), 256, 0, s>>>(col64, d.col, nnz, -1,
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

// D2H of a C range: values first (copy-out stream), then the convert stream
// widens the columns into the value array and the copy-out stream drains them
// as int64.  `drained` fires when the slot is free again.
int drain_c(Job &J, DevC &d, int64_t lo, int64_t hi, bool with_plen) {
    tsg_ctx *c = J.c;
    const int64_t rows = hi - lo, e0 = J.c_rp[lo], nnz = J.c_rp[hi] - e0;
    cudaStream_t s = c->copy_out, cs = c->widen;
    TSG_CK(cudaEventRecord(d.done, c->stream));
    TSG_CK(cudaStreamWaitEvent(s, d.done, 0));
    cudaEvent_t tl0{}, tl1{};
    g_tl.begin(s, tl0);
    if (nnz > 0) TSG_TRY(tsg_copy(J.c_val + e0, d.val, nnz * sizeof(double), cudaMemcpyDeviceToHost, s));
    g_tl.end('D', s, tl0);
    g_tl.begin(s, tl1);
    if (with_plen)
        TSG_TRY(tsg_copy(J.h_plen + lo, d.plen, rows * sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    if (nnz > 0) {
        TSG_CK(cudaEventRecord(d.vals_out, s));
        TSG_CK(cudaStreamWaitEvent(cs, d.vals_out, 0));
        int64_t *col64 = reinterpret_cast<int64_t *>(d.val);
        k_widen<<<grid_for(nnz, 256, c->num_sms * 16), 256, 0, cs>>>(d.col, col64, nnz); ++c->launches;
        TSG_CK(cudaGetLastError());
        TSG_CK(cudaEventRecord(d.widened, cs));
        TSG_CK(cudaStreamWaitEvent(s, d.widened, 0));
        TSG_TRY(tsg_copy(J.c_col + e0, col64, nnz * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    }
    g_tl.end('d', s, tl1);
    TSG_CK(cudaEventRecord(d.drained, s));
    J.st->d2h_bytes += nnz * 16 + (with_plen ? rows * 4 : 0);
    return TSG_OK;
}

// ---------------------------------------------------------------- physical layout choice

struct Layout {
    int a_slots = 2, c_slots = 2, b_slots = 3;
    int ac_split = 1, b_split = 1;
    int64_t bytes = 0;
    std::vector<int64_t> acb, bb;   // physical range / chunk bounds
};

struct MaxDims {
    int64_t a_rows = 0, a_nnz = 0, c_nnz = 0, b_rows = 0, b_nnz = 0;
};

MaxDims max_dims(const Job &J, const std::vector<int64_t> &acb, const std::vector<int64_t> &bb) {
    MaxDims m;
    for (size_t r = 0; r + 1 < acb.size(); ++r) {
        const int64_t lo = acb[r], hi = acb[r + 1];
        m.a_rows = std::max(m.a_rows, hi - lo);
        m.a_nnz = std::max(m.a_nnz, J.A.rp[hi] - J.A.rp[lo]);
        m.c_nnz = std::max(m.c_nnz, J.c_rp[hi] - J.c_rp[lo]);
    }
    for (size_t j = 0; j + 1 < bb.size(); ++j) {
        m.b_rows = std::max(m.b_rows, bb[j + 1] - bb[j]);
        m.b_nnz = std::max(m.b_nnz, J.B.rp[bb[j + 1]] - J.B.rp[bb[j]]);
    }
    return m;
}

int64_t layout_bytes(const MaxDims &m, int a_slots, int c_slots, int b_slots) {
    return a_slots * slot_ab_bytes(m.a_rows, m.a_nnz) + c_slots * slot_c_bytes(m.a_rows, m.c_nnz) +
           2 * rnd(8 * (m.a_rows + 2)) + b_slots * slot_ab_bytes(m.b_rows, m.b_nnz) +
           step_scratch_bytes(m.a_rows, m.b_rows, m.b_nnz);
}

// Pick buffering and splitting that fit `budget` (0: unlimited), preferring
// layouts that move no extra PCIe bytes and keep every stage overlapped.  For
// streamed B (orders 0/1) the smallest split giving three B slots is taken,
// then the slots are deepened (up to MAX_BS) while they fit: the bytes queued
// ahead on the copy engine, not the piece size, hide the host's per-step work.
constexpr int MAX_BS = 8;

int choose_layout(const Job &J, int algo, const int64_t *acb0, int64_t nac, const int64_t *bb0, int64_t nb,
                  bool a_sorted, int64_t budget, Layout &out) {
    const int splits[] = {1, 2, 3, 4, 6, 8, 12, 16, 24, 32};
    // order 0/1: B streams (split B chunks, neutral when A rows are sorted);
    // order 2: A/C stream (split A/C ranges, neutral)
    const bool streamed_b = algo != 2;
    const int nb_slots_full = streamed_b ? 3 : (nb > 1 ? 2 : 1);
    auto fits = [&](Layout &L) {
        L.acb = refine(acb0, nac, L.ac_split, J.A.rp);
        L.bb = refine(bb0, nb, L.b_split, J.B.rp);
        const MaxDims m = max_dims(J, L.acb, L.bb);
        L.bytes = layout_bytes(m, L.a_slots, L.c_slots, L.b_slots);
        return budget <= 0 || L.bytes <= budget;
    };
    for (int extra = 1; extra <= 32; extra = extra < 2 ? 2 : extra * 2) {   // traffic-raising split
        for (int cs = 2; cs >= 1; --cs)
            for (int as = 2; as >= 1; --as)
                for (int bs = nb_slots_full; bs >= 1; --bs)
                    for (int sp : splits) {
                        if (streamed_b && sp > 1 && !a_sorted) break;
                        Layout L;
                        L.a_slots = as;
                        L.c_slots = cs;
                        L.b_slots = bs;
                        L.ac_split = streamed_b ? extra : sp;
                        L.b_split = streamed_b ? sp : 1;
                        if (!fits(L)) continue;
                        if (streamed_b) {
                            const int64_t steps = (int64_t)(L.acb.size() - 1) * (int64_t)(L.bb.size() - 1);
                            L.b_slots = (int)std::min<int64_t>(L.b_slots, steps);
                            while (L.b_slots < MAX_BS && L.b_slots < steps && budget > 0) {
                                Layout D = L;
                                D.b_slots = L.b_slots + 1;
                                if (!fits(D)) break;
                                L = D;
                            }
                            if (budget <= 0) L.b_slots = (int)std::min<int64_t>(3, steps);
                            fits(L);
                        }
                        out = L;
                        return TSG_OK;
                    }
        if (!streamed_b) break;
    }
    tsg_set_error("chunk plan does not fit in the HBM budget of %lld bytes even fully split "
                  "(the largest A/C row range or B chunk row is too big)", (long long)budget);
    return TSG_ECAPACITY;
}

}  // namespace

extern "C" int tsg_chunk_multiply(tsg_ctx *c, int algo, int64_t a_rows, int64_t a_cols,
                                  const int64_t *a_rp, const int64_t *a_col, const double *a_val,
                                  int64_t b_rows, int64_t b_cols, const int64_t *b_rp,
                                  const int64_t *b_col, const double *b_val, const int64_t *c_rp,
                                  int64_t *c_col, double *c_val, int64_t n_ac,
                                  const int64_t *ac_bounds, int64_t n_b, const int64_t *b_bounds,
                                  int64_t budget_bytes, tsg_chunk_stats *stats) {
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
    TSG_CK(cudaStreamSynchronize(c->stream));
    // cached blocks could serve a slot with up to 25 % slack: start from an
    // empty cache so the footprint is the modelled one
    tsg_arena_trim(c);
    if (g_tl.on) fprintf(stderr, "[tsg host] trimmed %.1f ms\n",
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    const int64_t mem0 = c->bytes_in_use;
    c->bytes_peak = mem0;
    Job J{c, {a_rows, a_cols, a_rp, a_col, a_val}, {b_rows, b_cols, b_rp, b_col, b_val}, c_rp,
          c_col, c_val, nullptr, &local};

    bool a_sorted = false, a_distinct = false, b_sorted = false, b_distinct = false;
    auto hms = [&]() {
        return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    };
    auto row_orders = [&]() {
        host_row_order(J.A, &a_sorted, &a_distinct);
        if (J.B.rp == J.A.rp && J.B.col == J.A.col && J.B.rows == J.A.rows) {   // A * A: one pass
            b_sorted = a_sorted;
            b_distinct = a_distinct;
        } else {
            host_row_order(J.B, &b_sorted, &b_distinct);
        }
    };
    // (before any copy: in a thread beside order 2's first B pieces the scan
    // competed with the DMA for host-memory bandwidth -- one run in three
    // took 1.06 s instead of 0.79-0.81)
    row_orders();
    if (g_tl.on) fprintf(stderr, "[tsg host] row order %.1f ms\n", hms());
    int64_t whole[2] = {0, a_rows};
    const int64_t *acb0 = algo == 0 ? whole : ac_bounds;
    const int64_t nac0 = algo == 0 ? 1 : n_ac;
    Layout L;
    TSG_TRY(choose_layout(J, algo, acb0, nac0, b_bounds, n_b, a_sorted, budget_bytes, L));
    if (g_tl.on) fprintf(stderr, "[tsg host] layout %.1f ms\n", hms());
    const int64_t nac = (int64_t)L.acb.size() - 1, nb = (int64_t)L.bb.size() - 1;
    const int64_t *acb = L.acb.data(), *bb = L.bb.data();

    // host partial lengths (order 2): pinned, so their D2H stays asynchronous
    int32_t *plen_host = nullptr;
    constexpr int NBS = MAX_BS;
    DevRange Abuf[2], Bbuf[NBS];
    DevC Cbuf[2];
    CRows crow[2];
    cudaEvent_t used[NBS], used_a[2];   // compute finished with a B / A slot
    for (int i = 0; i < NBS; i++) TSG_CK(cudaEventCreateWithFlags(&used[i], cudaEventDisableTiming));
    for (int i = 0; i < 2; i++) {
        TSG_CK(cudaEventCreateWithFlags(&used_a[i], cudaEventDisableTiming));
        TSG_CK(cudaEventCreateWithFlags(&crow[i].ready, cudaEventDisableTiming));
        TSG_CK(cudaEventCreateWithFlags(&crow[i].used, cudaEventDisableTiming));
    }
    // per-step kernel timing events, read once at the end
    std::vector<cudaEvent_t> kev;
    float kernel_ms = 0.f;
    int st = TSG_OK;

    // one fused step; `cb_keep`: B's compressed form shared by the steps of a
    // resident B chunk (order 2), else compressed here and freed after
    auto fused_step = [&](DevRange &A, DevRange &B, DevC &C, int64_t blo, int64_t bhi, int64_t rows,
                          tsg_cmat *cb_keep) -> int {
        TSG_CK(cudaStreamWaitEvent(c->stream, A.ready, 0));
        TSG_CK(cudaStreamWaitEvent(c->stream, B.ready, 0));
        cudaEvent_t e0, e1;
        TSG_CK(cudaEventCreate(&e0));
        TSG_CK(cudaEventCreate(&e1));
        kev.push_back(e0);
        kev.push_back(e1);
        TSG_CK(cudaEventRecord(e0, c->stream));
        tsg_cmat *cb = cb_keep;
        if (!cb) TSG_TRY(tsg_compress_impl(c, &B.m, &cb));
        int s2 = tsg_fused_inplace(c, &A.m, (int32_t)blo, (int32_t)bhi, &B.m, cb, C.cptr, C.cap, C.col, C.val,
                                   C.plen, rows);
        if (!cb_keep) tsg_cmat_free(c, cb);
        TSG_TRY(s2);
        TSG_CK(cudaEventRecord(e1, c->stream));
        return TSG_OK;
    };

    // every slot sized for the largest range / chunk before the pipeline
    // starts (a mid-run reallocation would wait for the slot's in-flight users)
    {
        const MaxDims m = max_dims(J, L.acb, L.bb);
        for (int i = 0; i < L.a_slots && st == TSG_OK; ++i) st = ensure(c, Abuf[i], m.a_rows, m.a_nnz);
        for (int i = 0; i < L.c_slots && st == TSG_OK; ++i) st = ensure_c(c, Cbuf[i], m.a_rows, m.c_nnz);
        for (int i = 0; i < 2 && st == TSG_OK; ++i) {
            st = tsg_alloc_t(c, &crow[i].rp, m.a_rows + 2);
            crow[i].cap_rows = m.a_rows;
        }
        for (int i = 0; i < L.b_slots && st == TSG_OK; ++i) st = ensure(c, Bbuf[i], m.b_rows, m.b_nnz);
        // grow the driver pool once by the per-step temporaries: growing it
        // later maps memory while copies are in flight and stalls host and device
        const size_t grow = (size_t)step_scratch_bytes(m.a_rows, m.b_rows, m.b_nnz);
        void *tmp = nullptr;
        if (st == TSG_OK && cudaMallocAsync(&tmp, grow, c->stream) == cudaSuccess)
            cudaFreeAsync(tmp, c->stream);
        else
            cudaGetLastError();
        TSG_CK(cudaStreamSynchronize(c->stream));
        for (int i = 0; i < 2; i++) TSG_CK(cudaEventRecord(crow[i].used, c->stream));
    }
    if (g_tl.on) fprintf(stderr, "[tsg host] slots allocated %.1f ms\n", hms());
    local.budget_bytes = budget_bytes;
    local.a_slots = L.a_slots;
    local.c_slots = L.c_slots;
    local.b_slots = L.b_slots;
    local.ac_split = L.ac_split;
    local.b_split = L.b_split;
    local.layout_bytes = L.bytes;

    if (st == TSG_OK && algo != 2) {
        // Flat schedule over steps s = (range r, chunk j): before step s runs,
        // the copies of step s+ahead are queued (A range when j == 0, B chunk
        // in slot s % b_slots), so the copy engine always has the next
        // transfers queued while the host blocks inside a fused step.  C
        // ranges are opened on the compute stream right before their first step.
        const int64_t nsteps = nac * nb;
        const int ahead = L.b_slots - 1;
        // A range r' (and its C row pointers) may be staged once range
        // r' - a_slots has released its A slot (used_a recorded): staging
        // earlier would wait on a stale event and overwrite a slot in use
        int64_t a_next = 0, finished = 0;
        auto stage_a = [&]() -> int {
            while (a_next < nac && a_next - L.a_slots < finished) {
                const int64_t r = a_next++;
                TSG_TRY(stage_rows(c, J.A, acb[r], acb[r + 1], Abuf[r % L.a_slots], used_a[r % L.a_slots],
                                   a_sorted, a_distinct, local.h2d_bytes));
                TSG_TRY(stage_c_rows(c, J.c_rp, crow[r & 1], acb[r], acb[r + 1], local.h2d_bytes));
            }
            return TSG_OK;
        };
        auto issue_b = [&](int64_t s2) -> int {
            const int64_t j = s2 % nb;
            return stage_rows(c, J.B, bb[j], bb[j + 1], Bbuf[s2 % L.b_slots], used[s2 % L.b_slots], b_sorted,
                              b_distinct, local.h2d_bytes);
        };
        st = stage_a();
        for (int64_t s2 = 0; s2 <= ahead && s2 < nsteps && st == TSG_OK; ++s2) st = issue_b(s2);
        for (int64_t s2 = 0; s2 < nsteps && st == TSG_OK; ++s2) {
            const int64_t r = s2 / nb, j = s2 % nb;
            const int64_t lo = acb[r], hi = acb[r + 1];
            DevC &C = Cbuf[r % L.c_slots];
            if (j == 0 && (st = open_c(J, C, crow[r & 1], true, lo, hi, false)) != TSG_OK) break;
            st = fused_step(Abuf[r % L.a_slots], Bbuf[s2 % L.b_slots], C, bb[j], bb[j + 1], hi - lo, nullptr);
            if (st != TSG_OK) break;
            TSG_CK(cudaEventRecord(used[s2 % L.b_slots], c->stream));
            if (j == nb - 1) {
                TSG_CK(cudaEventRecord(used_a[r % L.a_slots], c->stream));
                k_check_full<<<grid_for(hi - lo, 256, c->num_sms * 8), 256, 0, c->stream>>>(
                    C.plen, C.cap, hi - lo, lo, c->d_err); ++c->launches;
                st = drain_c(J, C, lo, hi, false);
                finished = r + 1;
                if (st == TSG_OK) st = stage_a();
            }
            if (st == TSG_OK && s2 + ahead + 1 < nsteps) st = issue_b(s2 + ahead + 1);
        }
    } else if (st == TSG_OK) {
        // partial lengths round-trip through pinned host memory only when a
        // later B chunk reloads them; a single resident chunk finishes every
        // range in one step, checked on the device like order 1
        const bool partials = nb > 1;
        // one resident B chunk and row-sorted A: B lands in pieces and the
        // early A/C ranges start on its landed prefix (stage_b_pieces)
        // config 4 at 16 GiB: 0.803-0.810 s per run against 0.872-0.881 s
        // without (TSG_CHUNK_NO_OVERLAP=1).  The prefix compressions allocate
        // the full chunk's sizes (c->cmp_floor_*): with per-prefix sizes one
        // run in four grew the pool while copies were in flight (2.69 s)
        static const bool overlap_off = getenv("TSG_CHUNK_NO_OVERLAP") != nullptr;
        const bool overlap = !partials && nac > 1 && !overlap_off;
        const int NP = 8;
        BPieces bp;
        for (int64_t j = 0; j < nb && st == TSG_OK; ++j) {
            DevRange &B = Bbuf[j % L.b_slots];
            if (overlap) {
                // B's row pointers and first two pieces go on the link at once
                st = stage_b_begin(c, J.B, bb[j], bb[j + 1], B, used[j % L.b_slots], false, false,
                                   local.h2d_bytes, NP, bp);
                if (st == TSG_OK) st = stage_b_upto(c, J.B, bb[j], B, 1, bp);
                B.m.sorted = b_sorted ? 1 : 0;
                B.m.distinct = b_distinct ? 1 : 0;
            } else {
                st = stage_rows(c, J.B, bb[j], bb[j + 1], B, used[j % L.b_slots], b_sorted, b_distinct,
                                local.h2d_bytes);
            }
            if (st != TSG_OK) break;
            if (j == 0 && partials) {   // allocated while the first chunk is on the link
                void *ph = nullptr;
                TSG_TRY(tsg_host_alloc(((size_t)a_rows + 1) * sizeof(int32_t), &ph));
                plen_host = static_cast<int32_t *>(ph);
                memset(plen_host, 0, ((size_t)a_rows + 1) * sizeof(int32_t));
                J.h_plen = plen_host;
            }
            // the resident chunk is compressed once for all A/C ranges (a
            // landed prefix on its own for the ranges that run before)
            tsg_cmat *cbj = nullptr, *cbp = nullptr;
            int cur_k = -1;
            // prefix and full compressions allocate the full chunk's sizes
            struct Floor {
                tsg_ctx *c;
                Floor(tsg_ctx *x, bool on, int64_t r, int64_t n) : c(x) {
                    if (on) {
                        c->cmp_floor_rows = r;
                        c->cmp_floor_nnz = n;
                    }
                }
                ~Floor() { c->cmp_floor_rows = c->cmp_floor_nnz = 0; }
            } floor_(c, overlap, B.m.rows, B.m.nnz);
            DevRange Bv = B;   // prefix view: same arrays, fewer rows, the piece's event
            if (!overlap) {
                TSG_CK(cudaStreamWaitEvent(c->stream, B.ready, 0));
                if ((st = tsg_compress_impl(c, &B.m, &cbj)) != TSG_OK) break;
            }
            for (int64_t r = 0; r < nac && st == TSG_OK; ++r) {
                const int64_t lo = acb[r], hi = acb[r + 1];
                DevRange &A = Abuf[r % L.a_slots];
                DevC &C = Cbuf[r % L.c_slots];
                int k = NP - 1;
                if (overlap && !cbj) {   // smallest landed prefix holding every column of the range
                    int64_t need = 0;
                    if (a_sorted) {   // a row's largest column is its last
                        for (int64_t i = lo; i < hi; ++i)
                            if (J.A.rp[i + 1] > J.A.rp[i])
                                need = std::max<int64_t>(need, J.A.col[J.A.rp[i + 1] - 1] + 1);
                    } else {
                        for (int64_t e = J.A.rp[lo]; e < J.A.rp[hi]; ++e) need = std::max<int64_t>(need, J.A.col[e] + 1);
                    }
                    need -= bb[j];
                    k = 0;
                    while (k < NP - 1 && bp.q[k + 1] < need) ++k;
                }
                if (overlap && (st = stage_b_upto(c, J.B, bb[j], B, k, bp)) != TSG_OK) break;
                if ((st = stage_rows(c, J.A, lo, hi, A, used_a[r % L.a_slots], a_sorted, a_distinct,
                                     local.h2d_bytes, overlap)) != TSG_OK)
                    break;
                // partials come back from host after the first B sweep; the D2H
                // of the previous sweep for this range must have landed (the
                // first sweep loads nothing, so its ranges pipeline freely)
                if (j > 0) TSG_CK(cudaStreamSynchronize(c->copy_out));
                if ((st = open_c(J, C, crow[r & 1], false, lo, hi, j > 0)) != TSG_OK) break;
                if (overlap && !cbj && k < NP - 1) {
                    if (k != cur_k) {
                        if (cbp) tsg_cmat_free(c, cbp);
                        cbp = nullptr;
                        Bv.m.rows = bp.q[k + 1];
                        Bv.m.nnz = J.B.rp[bb[j] + bp.q[k + 1]] - J.B.rp[bb[j]];
                        Bv.ready = bp.ev[k];
                        TSG_CK(cudaStreamWaitEvent(c->stream, bp.ev[k], 0));
                        if ((st = tsg_compress_impl(c, &Bv.m, &cbp)) != TSG_OK) break;
                        cur_k = k;
                    }
                    st = fused_step(A, Bv, C, bb[j], bb[j] + bp.q[k + 1], hi - lo, cbp);
                } else {
                    if (overlap && !cbj) {   // B complete: its full compression from here on
                        if (cbp) tsg_cmat_free(c, cbp);
                        cbp = nullptr;
                        TSG_CK(cudaStreamWaitEvent(c->stream, B.ready, 0));
                        if ((st = tsg_compress_impl(c, &B.m, &cbj)) != TSG_OK) break;
                    }
                    st = fused_step(A, B, C, bb[j], bb[j + 1], hi - lo, cbj);
                }
                TSG_CK(cudaEventRecord(used_a[r % L.a_slots], c->stream));
                if (st == TSG_OK && !partials) {
                    k_check_full<<<grid_for(hi - lo, 256, c->num_sms * 8), 256, 0, c->stream>>>(
                        C.plen, C.cap, hi - lo, lo, c->d_err); ++c->launches;
                }
                if (st == TSG_OK) st = drain_c(J, C, lo, hi, partials);
            }
            tsg_cmat_free(c, cbj);
            if (cbp) tsg_cmat_free(c, cbp);
            TSG_CK(cudaEventRecord(used[j % L.b_slots], c->stream));
        }
        for (cudaEvent_t e : bp.ev) cudaEventDestroy(e);
    }
    cudaStreamSynchronize(c->copy_in);
    cudaStreamSynchronize(c->copy_in2);
    cudaStreamSynchronize(c->copy_out);
    cudaStreamSynchronize(c->convert);
    cudaStreamSynchronize(c->widen);
    cudaStreamSynchronize(c->stream);
    if (st == TSG_OK) st = tsg_check_kernel_errors(c, "chunked multiply");
    if (st == TSG_OK && algo == 2 && plen_host) {
        for (int64_t i = 0; i < a_rows; ++i)
            if (plen_host[i] != c_rp[i + 1] - c_rp[i]) {
                tsg_set_error("chunked result rows disagree with symbolic counts (row %lld: %d vs %lld)",
                              (long long)i, plen_host[i], (long long)(c_rp[i + 1] - c_rp[i]));
                st = TSG_EDIM;
                break;
            }
    }
    if (plen_host) tsg_host_free(plen_host);
    const int64_t peak = c->bytes_peak - mem0;
    for (int i = 0; i < 2; i++) {
        release(c, Abuf[i]);
        release_c(c, Cbuf[i]);
        tsg_free(c, crow[i].rp);
        cudaEventDestroy(crow[i].ready);
        cudaEventDestroy(crow[i].used);
        cudaEventDestroy(used_a[i]);
    }
    for (int i = 0; i < NBS; i++) {
        release(c, Bbuf[i]);
        cudaEventDestroy(used[i]);
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
    cudaStreamSynchronize(c->stream);
    local.kernel_ms = kernel_ms;
    local.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    local.peak_device_bytes = peak;
    if (stats) *stats = local;
    if (st == TSG_OK && budget_bytes > 0 && peak > budget_bytes) {
        tsg_set_error("chunked multiply held %lld bytes of HBM, above the budget of %lld",
                      (long long)peak, (long long)budget_bytes);
        st = TSG_ECAPACITY;
    }
    return st;
}

// Symbolic counts through the same budget (the
// reference runs spgemm_symbolic unchunked, cli.py:164-165): B's rows are
// compressed chunk by chunk (rows compress independently, kernel.py:73-93)
// into one resident compressed B, then A row ranges stream past it.  Peak
// HBM = compressed B + one A range (double-buffered when it fits) + scratch;
// TSG_ECAPACITY if the compressed B alone does not fit.
namespace {
__global__ void k_append_cmat(int64_t rows, const int64_t *__restrict__ start, const int32_t *__restrict__ cnt,
                              const int32_t *__restrict__ set, const uint64_t *__restrict__ bits,
                              const int64_t *__restrict__ out_start, int32_t *__restrict__ out_cnt,
                              int32_t *__restrict__ out_set, uint64_t *__restrict__ out_bits) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w; i < rows; i += nw) {
        const int64_t s0 = start[i], o0 = out_start[i];
        const int n = cnt[i];
        for (int k = lane; k < n; k += 32) {
            out_set[o0 + k] = set[s0 + k];
            out_bits[o0 + k] = bits[s0 + k];
        }
        if (lane == 0) out_cnt[i] = n;
    }
}

__global__ void k_add_base(int64_t *__restrict__ v, int64_t n, const int64_t *__restrict__ base) {
    const int64_t b = *base;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        v[i] += b;
}
}  // namespace

extern "C" int tsg_chunk_symbolic(tsg_ctx *c, int64_t a_rows, int64_t a_cols, const int64_t *a_rp,
                                  const int64_t *a_col, int64_t b_rows, int64_t b_cols, const int64_t *b_rp,
                                  const int64_t *b_col, int64_t budget_bytes, int64_t *counts,
                                  tsg_chunk_stats *stats) {
    if (a_cols != b_rows) {
        tsg_set_error("A has %lld cols but B has %lld rows", (long long)a_cols, (long long)b_rows);
        return TSG_EDIM;
    }
    tsg_chunk_stats local;
    memset(&local, 0, sizeof(local));
    auto t0 = std::chrono::steady_clock::now();
    TSG_CK(cudaStreamSynchronize(c->stream));
    tsg_arena_trim(c);
    const int64_t mem0 = c->bytes_in_use;
    c->bytes_peak = mem0;
    HostCsr HA{a_rows, a_cols, a_rp, a_col, nullptr}, HB{b_rows, b_cols, b_rp, b_col, nullptr};
    bool a_sorted, a_distinct, b_sorted, b_distinct;
    host_row_order(HA, &a_sorted, &a_distinct);
    host_row_order(HB, &b_sorted, &b_distinct);
    const int64_t b_nnz = b_rp[b_rows];
    // compressed B capacity: one set per entry at most
    const int64_t cb_bytes = rnd(8 * (b_rows + 1)) + rnd(4 * (b_rows + 2)) + rnd(4 * (b_nnz + 1)) +
                             rnd(8 * (b_nnz + 1));
    const int64_t budget = budget_bytes > 0 ? budget_bytes : ((int64_t)1 << 62);
    if (cb_bytes >= budget) {
        tsg_set_error("compressed B (%lld bytes) does not fit in the HBM budget of %lld", (long long)cb_bytes,
                      (long long)budget_bytes);
        return TSG_ECAPACITY;
    }
    int st = TSG_OK;
    tsg_cmat *cb = nullptr;
    TSG_TRY(tsg_cmat_alloc(c, b_rows, b_nnz > 0 ? b_nnz : 1, &cb));
    cb->cols = b_cols;
    cb->sorted_sets = 1;
    int64_t *dcnt64 = nullptr;
    // B in chunks of rows that fit next to the compressed B: slot + its compression scratch
    const int64_t room = budget - cb_bytes - ((int64_t)64 << 20);
    int64_t chunk_nnz = std::max<int64_t>(room / 40, 1 << 20);   // ~12 slot + ~25 compress scratch B/entry
    std::vector<int64_t> bb{0};
    for (int64_t r = 0; r < b_rows;) {
        const int64_t target = b_rp[r] + chunk_nnz;
        int64_t e = std::upper_bound(b_rp + r, b_rp + b_rows + 1, target) - b_rp - 1;
        e = std::max(e, r + 1);
        e = std::min(e, b_rows);
        bb.push_back(e);
        r = e;
    }
    DevRange slot;
    int64_t *base_dev = nullptr;
    TSG_TRY(tsg_alloc_t(c, &base_dev, 2));
    TSG_TRY(tsg_fill(c, base_dev, 0, 2 * sizeof(int64_t), c->stream));
    int max_cnt_all = 0;
    for (size_t j = 0; j + 1 < bb.size() && st == TSG_OK; ++j) {
        const int64_t lo = bb[j], hi = bb[j + 1];
        st = stage_rows(c, HB, lo, hi, slot, nullptr, b_sorted, b_distinct, local.h2d_bytes);
        if (st != TSG_OK) break;
        TSG_CK(cudaStreamWaitEvent(c->stream, slot.ready, 0));
        tsg_cmat *part = nullptr;
        st = tsg_compress_impl(c, &slot.m, &part);
        if (st != TSG_OK) break;
        if (!part->sorted_sets) cb->sorted_sets = 0;
        // compact starts of this chunk = global offset + exclusive scan of counts
        const int64_t rows = hi - lo;
        st = tsg_exclusive_scan_i32_to_i64(c, part->cnt, cb->start + lo, rows);
        if (st == TSG_OK) {
            k_add_base<<<grid_for(rows + 1, 256, c->num_sms * 8), 256, 0, c->stream>>>(cb->start + lo, rows + 1,
                                                                                       base_dev);
            ++c->launches;
            k_append_cmat<<<grid_for(rows, 8, c->num_sms * 16), 256, 0, c->stream>>>(
                rows, part->start, part->cnt, part->set, part->bits, cb->start + lo, cb->cnt + lo, cb->set,
                cb->bits);
            ++c->launches;
            TSG_CK(cudaMemcpyAsync(base_dev, cb->start + hi, sizeof(int64_t), cudaMemcpyDeviceToDevice, c->stream));
            int mc = 0;
            TSG_CK(cudaMemcpyAsync(&mc, part->cnt + rows + 1, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
            TSG_CK(cudaStreamSynchronize(c->stream));
            max_cnt_all = std::max(max_cnt_all, mc);
        }
        tsg_cmat_free(c, part);
        TSG_CK(cudaStreamSynchronize(c->stream));
    }
    release(c, slot);
    if (st == TSG_OK) {
        TSG_CK(cudaMemcpyAsync(cb->cnt + b_rows + 1, &max_cnt_all, sizeof(int), cudaMemcpyHostToDevice, c->stream));
        cb->dmax_valid = 1;
    }
    // A row ranges streamed past the resident compressed B
    if (st == TSG_OK && a_rows > 0) {
        const int64_t room_a = budget - (c->bytes_peak - mem0) - ((int64_t)64 << 20);
        int64_t nsets = 0;
        TSG_CK(cudaMemcpy(&nsets, cb->start + b_rows, sizeof(int64_t), cudaMemcpyDeviceToHost));
        // per A row: slot 16 B + 12 B/entry; symbolic: counts, set counts,
        // bounds, bins, lists (~64 B) and the sorted set lists (12 B per set
        // of the row's bound = its entries x the mean compressed B row)
        const double avg = (double)a_rp[a_rows] / (double)std::max<int64_t>(a_rows, 1);
        const double avg_cb = (double)nsets / (double)std::max<int64_t>(b_rows, 1);
        const int64_t per_row = (int64_t)(16 + 12 * avg + 96 + 12 * 1.25 * avg * avg_cb) + 1;
        int64_t range_rows = std::max<int64_t>(room_a / per_row, 1024);
        TSG_TRY(tsg_alloc_t(c, &dcnt64, 1));
        for (int64_t lo = 0; lo < a_rows && st == TSG_OK; lo += range_rows) {
            const int64_t hi = std::min(a_rows, lo + range_rows);
            st = stage_rows(c, HA, lo, hi, slot, nullptr, a_sorted, a_distinct, local.h2d_bytes);
            if (st != TSG_OK) break;
            TSG_CK(cudaStreamWaitEvent(c->stream, slot.ready, 0));
            tsg_vec *v = nullptr;
            st = tsg_symbolic_impl(c, hi - lo, &slot.m, 0, 0, 0x7fffffff, cb, nullptr, &v, nullptr);
            if (st != TSG_OK) break;
            TSG_CK(cudaMemcpyAsync(counts + lo, v->d, (hi - lo) * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                   c->stream));
            local.d2h_bytes += (hi - lo) * 8;
            TSG_CK(cudaStreamSynchronize(c->stream));
            tsg_vec_free(c, v);
        }
        release(c, slot);
    }
    tsg_free(c, dcnt64);
    tsg_free(c, base_dev);
    tsg_cmat_free(c, cb);
    cudaStreamSynchronize(c->copy_in);
    cudaStreamSynchronize(c->copy_in2);
    cudaStreamSynchronize(c->convert);
    cudaStreamSynchronize(c->stream);
    if (st == TSG_OK) st = tsg_check_kernel_errors(c, "chunked symbolic");
    const int64_t peak = c->bytes_peak - mem0;
    local.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    local.peak_device_bytes = peak;
    local.budget_bytes = budget_bytes;
    if (stats) *stats = local;
    if (st == TSG_OK && budget_bytes > 0 && peak > budget_bytes) {
        tsg_set_error("chunked symbolic held %lld bytes of HBM, above the budget of %lld", (long long)peak,
                      (long long)budget_bytes);
        st = TSG_ECAPACITY;
    }
    return st;
}

const void *tsg_kernel_chunk() { return (const void *)k_rebase; }
