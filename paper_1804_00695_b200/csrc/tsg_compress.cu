// tsg_compress.cu -- K1: bitmask compression of B's rows (kernel.py:73-93).
//
// Row r of B becomes its (set = col >> 6, 64-bit mask) pairs in first-touch
// order.  The output is COMPACT (start[r] .. start[r+1]) and built by
// entry-parallel, fully coalesced passes -- no per-row serial loops, no
// scattered narrow stores:
//   P0  row-start bitmap (one bit per entry)                      rows
//   P1  head flags: entry t opens a set if it starts its row or its set
//       differs from entry t-1's; per-warp head words, per-block counts;
//       a set that goes DOWN inside a row flags the matrix unsorted    nnz
//   P2  exclusive scan of the block counts                          nnz/256
//   P3  each head ORs its run of bits and writes (set, mask) at its
//       global rank (consecutive heads -> consecutive addresses)       nnz
//   P4  start[r] = rank of the first entry of row r                   rows
// For a row-sorted matrix (every generator here, and any CsrMatrix built
// with from_coo) the first set of a run is its first touch, so this equals
// the reference's dict order.  If P1 saw an unsorted row, P3/P4 exit and the
// first-occurrence fallback (F1 count, scan, F2 write: entry t heads its set
// iff no EARLIER entry of the row has the same set) rebuilds the whole
// matrix.  The fallback kernels are launched unconditionally and exit at
// once on sorted input, so compression never synchronises the host.
#include "tsg_internal.cuh"

namespace {

constexpr int CT = 256;             // threads per block
constexpr int PB = 1024;            // entries per block (4 per thread, strided by CT)
constexpr int WPBLK = PB / 32;      // 32-entry words per block

__global__ void k_row_starts(int64_t rows, const int64_t *__restrict__ rp, uint32_t *rsbits) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t e = rp[i];
        if (e < rp[i + 1]) atomicOr(&rsbits[e >> 5], 1u << (e & 31));
    }
}

// stage the block's PB columns (+ the one before) in shared memory
__device__ __forceinline__ void stage_cols(int64_t nnz, int64_t base, const int32_t *__restrict__ col,
                                           int *s_c) {
#pragma unroll
    for (int k = 0; k < PB / CT; ++k) {
        const int e = k * CT + threadIdx.x;
        const int64_t t = base + e;
        s_c[e + 1] = t < nnz ? col[t] : 0;
    }
    if (threadIdx.x == 0) s_c[0] = base > 0 ? col[base - 1] : 0;
}

// P1: head words (one ballot per 32 consecutive entries), block-relative
// per-word prefixes and per-block totals.
__global__ void __launch_bounds__(CT) k_heads(int64_t nnz, const int32_t *__restrict__ col,
                                             const uint32_t *__restrict__ rsbits,
                                             uint32_t *__restrict__ hbits,
                                             uint16_t *__restrict__ wpre,
                                             int64_t *__restrict__ bcnt, int *unsorted) {
    __shared__ int s_c[PB + 1];
    __shared__ int s_n[WPBLK];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t base = (int64_t)blockIdx.x * PB;
    stage_cols(nnz, base, col, s_c);
    __syncthreads();
    bool bad = false;
#pragma unroll
    for (int k = 0; k < PB / CT; ++k) {
        const int e = k * CT + threadIdx.x;
        const int64_t t = base + e;
        const bool valid = t < nnz;
        const int sv = s_c[e + 1] >> 6, sp = s_c[e] >> 6;
        const bool rs = valid && ((rsbits[t >> 5] >> (t & 31)) & 1u);
        const bool head = valid && (rs || t == 0 || sv != sp);
        bad |= valid && !rs && t > 0 && sv < sp;
        const uint32_t hw = __ballot_sync(0xffffffffu, head);
        const int word = k * (CT / 32) + w;
        if (lane == 0) {
            if (base + word * 32 < nnz) hbits[(base >> 5) + word] = hw;
            s_n[word] = __popc(hw);
        }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(unsorted, 1);
    __syncthreads();
    if (w == 0) {
        int v = s_n[lane];   // WPBLK == 32
        int x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int o = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += o;
        }
        if (base + lane * 32 < nnz) wpre[(base >> 5) + lane] = (uint16_t)(x - v);
        if (lane == 31) bcnt[blockIdx.x] = x;
    }
}

// P3: every head ORs the bits of its run (a forward scan in shared memory;
// a run crossing the block end continues in global memory) and writes its
// (set, mask) at its global rank.  Consecutive heads of a warp write
// consecutive addresses.
__global__ void __launch_bounds__(CT) k_emit_sets(int64_t nnz, const int32_t *__restrict__ col,
                                                 const uint32_t *__restrict__ hbits,
                                                 const uint16_t *__restrict__ wpre,
                                                 const int64_t *__restrict__ boff,
                                                 int32_t *__restrict__ oset,
                                                 uint64_t *__restrict__ obits,
                                                 const int *unsorted) {
    if (*unsorted) return;
    __shared__ int s_c[PB + 1];
    __shared__ uint32_t s_h[WPBLK];
    const int lane = threadIdx.x & 31;
    const int64_t base = (int64_t)blockIdx.x * PB;
    const int lim = nnz - base < PB ? (int)(nnz - base) : PB;
    stage_cols(nnz, base, col, s_c);
    if (threadIdx.x < WPBLK)
        s_h[threadIdx.x] = base + threadIdx.x * 32 < nnz ? hbits[(base >> 5) + threadIdx.x] : 0u;
    __syncthreads();
    const int64_t bb = boff[blockIdx.x];
#pragma unroll
    for (int k = 0; k < PB / CT; ++k) {
        const int e = k * CT + threadIdx.x;
        const int word = e >> 5;
        const uint32_t hw = s_h[word];
        if (!((hw >> lane) & 1u)) continue;
        const int c0 = s_c[e + 1];
        unsigned lo = 0, hi = 0;
        int q = e;
        do {   // run = entries up to the next head
            const int b = s_c[q + 1] & 63;
            if (b < 32) lo |= 1u << b;
            else hi |= 1u << (b - 32);
            ++q;
        } while (q < lim && !((s_h[q >> 5] >> (q & 31)) & 1u));
        uint64_t bits = ((uint64_t)hi << 32) | lo;
        if (q == PB) {
            for (int64_t g = base + PB; g < nnz; ++g) {
                if ((hbits[g >> 5] >> (g & 31)) & 1u) break;
                bits |= 1ull << (col[g] & 63);
            }
        }
        const int64_t pos = bb + wpre[(base >> 5) + word] + __popc(hw & ((1u << lane) - 1u));
        oset[pos] = c0 >> 6;
        obits[pos] = bits;
    }
}

// rank of the first entry of each row = exclusive head count at rp[r]
__global__ void k_set_starts(int64_t rows, int64_t nnz, const int64_t *__restrict__ rp,
                             const uint32_t *__restrict__ hbits, const uint16_t *__restrict__ wpre,
                             const int64_t *__restrict__ boff, int64_t nblocks,
                             int64_t *__restrict__ start, int32_t *__restrict__ cnt,
                             const int *unsorted) {
    if (*unsorted) return;
    auto rank_at = [&](int64_t e) -> int64_t {
        if (e >= nnz) return boff[nblocks];
        return boff[e / PB] + wpre[e >> 5] + __popc(hbits[e >> 5] & ((1u << (e & 31)) - 1u));
    };
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t s0 = rank_at(rp[i]);
        start[i] = s0;
        if (i < rows) cnt[i] = (int32_t)(rank_at(rp[i + 1]) - s0);
    }
}

// ---- first-occurrence fallback for unsorted rows (warp per row)

__global__ void k_first_count(int64_t rows, const int64_t *__restrict__ rp,
                              const int32_t *__restrict__ col, int32_t *__restrict__ fcnt,
                              const int *unsorted) {
    if (!*unsorted) return;
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w; i < rows; i += nw) {
        const int64_t r0 = rp[i], r1 = rp[i + 1];
        int n = 0;
        for (int64_t t = r0 + lane; t < r1; t += 32) {
            int s = col[t] >> 6;
            bool first = true;
            for (int64_t q = r0; q < t && first; ++q) first = (col[q] >> 6) != s;
            n += first;
        }
        for (int d = 16; d >= 1; d >>= 1) n += __shfl_xor_sync(0xffffffffu, n, d);
        if (lane == 0) fcnt[i] = n;
    }
}

__global__ void k_first_emit(int64_t rows, const int64_t *__restrict__ rp,
                             const int32_t *__restrict__ col, const int32_t *__restrict__ fcnt,
                             const int64_t *__restrict__ fstart, int64_t *__restrict__ start,
                             int32_t *__restrict__ cnt, int32_t *__restrict__ oset,
                             uint64_t *__restrict__ obits, const int *unsorted) {
    if (!*unsorted) return;
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w; i <= rows; i += nw) {
        if (lane == 0) {
            start[i] = fstart[i];
            if (i < rows) cnt[i] = fcnt[i];
        }
        if (i == rows) continue;
        const int64_t r0 = rp[i], r1 = rp[i + 1];
        int64_t carry = fstart[i];
        for (int64_t base = r0; base < r1; base += 32) {
            const int64_t t = base + lane;
            int s = t < r1 ? (col[t] >> 6) : -1;
            bool first = t < r1;
            for (int64_t q = r0; q < t && first; ++q) first = (col[q] >> 6) != s;
            unsigned fb = __ballot_sync(0xffffffffu, first);
            if (first) {
                uint64_t bits = 0;
                for (int64_t q = t; q < r1; ++q) {
                    int cq = col[q];
                    if ((cq >> 6) == s) bits |= 1ull << (cq & 63);
                }
                int64_t pos = carry + __popc(fb & lt);
                oset[pos] = s;
                obits[pos] = bits;
            }
            carry += __popc(fb);
        }
    }
}

}  // namespace

int tsg_compress_impl(tsg_ctx *c, const tsg_csr *b, tsg_cmat **out) {
    tsg_cmat *cm = nullptr;
    const int64_t rows = b->rows, nnz = b->nnz;
    TSG_TRY(tsg_cmat_alloc(c, rows, nnz > 0 ? nnz : 1, &cm));
    if (nnz == 0) {
        TSG_CK(cudaMemsetAsync(cm->start, 0, (rows + 1) * sizeof(int64_t), c->stream));
        TSG_CK(cudaMemsetAsync(cm->cnt, 0, (rows + 1) * sizeof(int32_t), c->stream));
        *out = cm;
        return TSG_OK;
    }
    const int64_t nwords = (nnz + 31) / 32, nblocks = (nnz + PB - 1) / PB;   // PB = 1024 entries
    uint32_t *rsbits = nullptr, *hbits = nullptr;
    uint16_t *wpre = nullptr;
    int64_t *bcnt = nullptr, *fstart = nullptr;
    int32_t *fcnt = nullptr;
    TSG_TRY(tsg_alloc_t(c, &rsbits, nwords));
    TSG_TRY(tsg_alloc_t(c, &hbits, nwords));
    TSG_TRY(tsg_alloc_t(c, &wpre, nwords));
    TSG_TRY(tsg_alloc_t(c, &bcnt, nblocks + 1));
    TSG_TRY(tsg_alloc_t(c, &fcnt, rows + 1));
    TSG_TRY(tsg_alloc_t(c, &fstart, rows + 1));
    int *unsorted = reinterpret_cast<int *>(c->d_small + 8);
    cudaStream_t s = c->stream;
    TSG_CK(cudaMemsetAsync(rsbits, 0, nwords * sizeof(uint32_t), s));
    TSG_CK(cudaMemsetAsync(unsorted, 0, sizeof(int), s));
    const unsigned rgrid = grid_for(rows + 1, 256, c->num_sms * 16);
    k_row_starts<<<rgrid, 256, 0, s>>>(rows, b->rp, rsbits); ++c->launches;
    k_heads<<<(unsigned)nblocks, CT, 0, s>>>(nnz, b->col, rsbits, hbits, wpre, bcnt, unsorted); ++c->launches;
    TSG_TRY(tsg_exclusive_scan_i64(c, bcnt, bcnt, nblocks));
    k_emit_sets<<<(unsigned)nblocks, CT, 0, s>>>(nnz, b->col, hbits, wpre, bcnt, cm->set, cm->bits,
                                                 unsorted); ++c->launches;
    k_set_starts<<<rgrid, 256, 0, s>>>(rows, nnz, b->rp, hbits, wpre, bcnt, nblocks, cm->start, cm->cnt,
                                       unsorted); ++c->launches;
    // first-occurrence fallback: every kernel returns at once on sorted input
    const unsigned wgrid = (unsigned)(c->num_sms * 4);   // grid-stride; exits at once when sorted
    k_first_count<<<wgrid, 256, 0, s>>>(rows, b->rp, b->col, fcnt, unsorted); ++c->launches;
    TSG_TRY(tsg_exclusive_scan_i32_to_i64(c, fcnt, fstart, rows));
    k_first_emit<<<wgrid, 256, 0, s>>>(rows, b->rp, b->col, fcnt, fstart, cm->start, cm->cnt, cm->set,
                                       cm->bits, unsorted); ++c->launches;
    TSG_CK(cudaGetLastError());
    tsg_free(c, rsbits);
    tsg_free(c, hbits);
    tsg_free(c, wpre);
    tsg_free(c, bcnt);
    tsg_free(c, fcnt);
    tsg_free(c, fstart);
    *out = cm;
    return TSG_OK;
}
