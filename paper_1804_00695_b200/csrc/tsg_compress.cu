// tsg_compress.cu -- K1: bitmask compression of B's rows (kernel.py:73-93).
//
// Row r of B becomes its (set = col >> 6, 64-bit mask) pairs in first-touch
// order.  The output is COMPACT (start[r] .. start[r+1]) and built by
// entry-parallel, fully coalesced passes -- no per-row serial loops, no
// scattered narrow stores:
//   P0  row-start bitmap (one bit per entry)                          rows
//   P1  one pass per 8192-entry tile: head flags (an entry opens a set if
//       it starts its row or its set differs from entry t-1's; a set that
//       goes DOWN inside a row flags the matrix unsorted), block scan,
//       decoupled look-back for the tile's global rank, then every head ORs
//       its run of bits and the tile's (set, mask) pairs are written
//       coalesced at consecutive ranks                                 nnz
//   P2  start[r] = rank of the first entry of row r                    rows
// For a row-sorted matrix (every generator here, and any CsrMatrix built
// with from_coo) the first set of a run is its first touch, so this equals
// the reference's dict order.  Matrices not known to be row-sorted also get
// the first-occurrence fallback (F1 count, scan, F2 write: entry t heads its
// set iff no EARLIER entry of the row has the same set), whose kernels exit
// at once unless P1 flagged an unsorted row; compression never synchronises
// the host.
#include <algorithm>

#include "tsg_internal.cuh"

namespace {

// Thread-per-word layout: one thread owns a 32-entry word of B's column
// array (8 x 16-byte loads, its own cache line), so head detection and run
// ORs are straight-line register code (~8 instructions per entry instead of
// warp shuffles per entry).  A block covers CT words = 32*CT entries.
constexpr int CT = 256;                 // threads (= words) per block
constexpr int PB = CT * 32;             // entries per block

__global__ void k_row_starts(int64_t rows, const int64_t *__restrict__ rp, uint32_t *rsbits, int *dmax) {
    pdl_wait();
    if (blockIdx.x == 0 && threadIdx.x == 0) *dmax = 0;   // max set count, raised by P2 / F2
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t e = rp[i];
        if (e < rp[i + 1]) atomicOr(&rsbits[e >> 5], 1u << (e & 31));
    }
}

// The block's PB column entries are staged in shared memory with coalesced
// 16-byte loads, then each thread reads its own 32-entry word back into
// registers.  Thread-owned 128-byte lines read straight from global would
// cost 32 L1 wavefronts per warp load (one per line); the 16-byte chunks are
// XOR-swizzled by line (chunk k of word w at w*8 + (k ^ (w & 7))) so both
// the staging stores and the per-thread reads are bank-conflict free.
__device__ __forceinline__ void stage_cols(const int32_t *__restrict__ col, int64_t nnz, int64_t e0,
                                           int4 *__restrict__ sm) {
    const bool vec = e0 + PB <= nnz && (((uintptr_t)(col + e0)) & 15) == 0;
    const int4 *src = reinterpret_cast<const int4 *>(col + e0);
#pragma unroll 4
    for (int i = threadIdx.x; i < PB / 4; i += CT) {
        int4 v;
        if (vec) {
            v = __ldg(src + i);
        } else {
            const int64_t b = e0 + 4 * (int64_t)i;
            v.x = b < nnz ? __ldg(col + b) : 0;
            v.y = b + 1 < nnz ? __ldg(col + b + 1) : 0;
            v.z = b + 2 < nnz ? __ldg(col + b + 2) : 0;
            v.w = b + 3 < nnz ? __ldg(col + b + 3) : 0;
        }
        const int w = i >> 3, k = i & 7;
        sm[w * 8 + (k ^ (w & 7))] = v;
    }
}

__device__ __forceinline__ void word_from_smem(const int4 *__restrict__ sm, int (&c)[32]) {
    const int w = threadIdx.x;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int4 v = sm[w * 8 + (k ^ (w & 7))];
        c[4 * k] = v.x;
        c[4 * k + 1] = v.y;
        c[4 * k + 2] = v.z;
        c[4 * k + 3] = v.w;
    }
}

// P3: each thread walks its word's runs in registers and emits every run it
// owns; a run that started in an earlier word belongs to that word's thread,
// which reads ahead until the next head.  The block's runs form one
// contiguous output range, so they are staged in shared memory (aliasing the
// column stage once every thread holds its word) and written back with
// coalesced stores.  Set masks are staged as two 32-bit halves and every
// staged array is padded one word per 32: regular matrices give the threads
// that open a run in the same iteration ranks exactly 32 apart (a 27-point
// stencil row has 9 runs of 3 -> a head every third entry, ranks 32k + c),
// which unpadded would put all of them on one bank.
constexpr int EMIT_CAP = 3584;   // staged runs per block (~50 KB); more -> direct stores
constexpr int EMIT_PAD = EMIT_CAP + EMIT_CAP / 32;
constexpr size_t EMIT_SMEM = (size_t)EMIT_PAD * 12 > (size_t)PB * 4 ? (size_t)EMIT_PAD * 12 : (size_t)PB * 4;

// Head flags of one 32-entry word: entry q opens a (row, set) run if it
// starts a row or its set differs from entry q-1's (pv = set of the entry
// before the word, -1 at the matrix start).  A set that goes DOWN inside a
// row marks the matrix unsorted.  FULL: all 32 entries valid.
template <bool FULL, bool CHECK>
__device__ __forceinline__ uint32_t word_heads(const int (&c)[32], uint32_t rs, int pv, int64_t left,
                                               bool &bad) {
    uint32_t hw = 0;
    bool b = false;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
        const int sv = c[q] >> 6;
        const bool valid = FULL || q < left;
        const bool start = (rs >> q) & 1u;
        if (valid) {
            hw |= (uint32_t)(start || sv != pv) << q;
            if (CHECK) b |= !start && sv < pv;
        }
        pv = sv;
    }
    bad = b;
    return hw;
}

// Emit the word's runs walking BACKWARD: acc collects the bits of the run
// being walked (seeded with the read-ahead bits of the last run), and at its
// head the run is complete and stored at rank r (block-relative when staged,
// else at b0 + r in global memory).  Entries before the word's first head
// belong to the previous word's last run and are skipped (r < r0 there).
template <bool FULL>
__device__ __forceinline__ void emit_runs(const int (&c)[32], uint32_t hw, int r, uint64_t acc, int64_t left,
                                          bool staged, int64_t b0, int32_t *s_set, uint32_t *s_lo,
                                          uint32_t *s_hi, int32_t *__restrict__ oset,
                                          uint64_t *__restrict__ obits) {
#pragma unroll
    for (int q = 31; q >= 0; --q) {
        if (FULL || q < left) {
            acc |= 1ull << (c[q] & 63);
            if ((hw >> q) & 1u) {
                if (staged) {
                    const int pr = r + (r >> 5);
                    s_set[pr] = c[q] >> 6;
                    s_lo[pr] = (uint32_t)acc;
                    s_hi[pr] = (uint32_t)(acc >> 32);
                } else {
                    oset[b0 + r] = c[q] >> 6;
                    obits[b0 + r] = acc;
                }
                --r;
                acc = 0;
            }
        }
    }
}

// P1+P2+P3 in one pass (single launch, columns read once): each tile finds
// its heads, scans them block-wide, obtains its global run offset by a
// decoupled look-back over the tiles before it (tile ids from an atomic
// counter, state words pack (prefix << 2 | flag)), publishes hbits / wpre /
// boff for k_set_starts and emits its runs.  A run that continues past the
// word is extended by reading columns directly (row-start bitmap + set
// compare), so no tile waits on another tile's head bitmap.
__device__ __forceinline__ unsigned long long lb_ld(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void lb_st(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

#ifndef TSG_CPF
#define TSG_CPF 3   // L2 prefetch distance in tiles per SM (measured: 0 -> 212 us, 3 -> 205, 5 -> 209, 10 -> 223)
#endif
// CHECK: also flag rows whose sets go down (input not known to be row-sorted)
template <bool CHECK>
__global__ void __launch_bounds__(CT, 5) k_compress_onepass(
    int64_t nnz, const int32_t *__restrict__ col, const uint32_t *__restrict__ rsbits,
    uint32_t *__restrict__ hbits, uint16_t *__restrict__ wpre, int64_t *__restrict__ boff,
    int64_t nblocks, unsigned long long *state, unsigned *counter, int32_t *__restrict__ oset,
    uint64_t *__restrict__ obits, int *unsorted, int64_t pf) {
    pdl_wait();
    extern __shared__ int4 esm[];
    __shared__ int s_w[CT / 32];
    __shared__ int64_t s_b0;
    __shared__ unsigned s_tile;
    uint32_t *s_lo = reinterpret_cast<uint32_t *>(esm);
    uint32_t *s_hi = s_lo + EMIT_PAD;
    int32_t *s_set = reinterpret_cast<int32_t *>(s_hi + EMIT_PAD);
    if (threadIdx.x == 0) s_tile = atomicAdd(counter, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    // tiles are taken in order, so the tile pf ahead is the one a CTA of the
    // next wave will take: one bulk prefetch of its columns into L2 turns that
    // CTA's staging loads into L2 hits
    if (pf > 0 && threadIdx.x == 0 && (tile + pf + 1) * (int64_t)PB <= nnz &&
        ((reinterpret_cast<uintptr_t>(col) & 15) == 0)) {
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(col + (tile + pf) * PB),
                     "r"((unsigned)(PB * 4))
                     : "memory");
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t word = tile * CT + threadIdx.x;
    const int64_t t0 = word * 32;
    stage_cols(col, nnz, tile * PB, esm);
    __syncthreads();
    int c[32];
    word_from_smem(esm, c);
    int prev;
    if (threadIdx.x > 0) {
        const int pw = threadIdx.x - 1;
        prev = reinterpret_cast<const int *>(esm)[(pw * 8 + (7 ^ (pw & 7))) * 4 + 3] >> 6;
    } else {
        prev = t0 > 0 && t0 < nnz + 1 ? (__ldg(col + t0 - 1) >> 6) : -1;
    }
    __syncthreads();   // the column stage is reused for the output below
    uint32_t hw = 0;
    bool bad = false;
    if (t0 + 32 <= nnz) {
        hw = word_heads<true, CHECK>(c, rsbits[word], t0 == 0 ? -1 : prev, nnz - t0, bad);
        hbits[word] = hw;
    } else if (t0 < nnz) {
        hw = word_heads<false, CHECK>(c, rsbits[word], t0 == 0 ? -1 : prev, nnz - t0, bad);
        hbits[word] = hw;
    }
    if (CHECK && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(unsorted, 1);
    const int n = __popc(hw);
    int x = n;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int o = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += o;
    }
    if (lane == 31) s_w[w] = x;
    __syncthreads();
    int woff = 0, agg = 0;
#pragma unroll
    for (int j = 0; j < CT / 32; ++j) {
        woff += j < w ? s_w[j] : 0;
        agg += s_w[j];
    }
    const int r0 = woff + x - n;   // block-relative rank of this word's first head
    if (t0 < nnz) wpre[word] = (uint16_t)r0;
    // publish the tile aggregate at once; the look-back for the tile's
    // global rank runs after this warp's runs are staged, so its wait
    // overlaps the emission work of the whole block
    if (threadIdx.x == 0)
        lb_st(&state[tile], ((unsigned long long)agg << 2) | (tile == 0 ? 2ull : 1ull));
    auto look_back = [&]() {   // warp 0 only
        int64_t excl = 0;
        if (tile > 0) {
            int64_t pred = tile - 1 - lane;
            for (;;) {
                const unsigned long long sv = pred >= 0 ? lb_ld(&state[pred]) : 2ull;
                const unsigned flag = (unsigned)(sv & 3ull);
                if (__any_sync(0xffffffffu, flag == 0)) continue;
                const unsigned incl = __ballot_sync(0xffffffffu, flag == 2);
                int64_t val = (int64_t)(sv >> 2);
                if (incl && lane > __ffs(incl) - 1) val = 0;
#pragma unroll
                for (int d = 16; d >= 1; d >>= 1) val += __shfl_xor_sync(0xffffffffu, val, d);
                excl += val;
                if (incl) break;
                pred -= 32;
            }
            if (lane == 0) lb_st(&state[tile], ((unsigned long long)(excl + agg) << 2) | 2ull);
        }
        if (lane == 0) {
            s_b0 = excl;
            boff[tile] = excl;
            if (tile == nblocks - 1) boff[nblocks] = excl + agg;
        }
    };
    const bool staged = agg <= EMIT_CAP;   // block-uniform
    if (!staged) {   // rare (dense tiles): global rank first, then direct stores
        if (w == 0) look_back();
        __syncthreads();
    }
    if (hw) {
        // the last run may continue into the next words (same row, same set):
        // its owner reads ahead until the next head
        uint64_t acc = 0;
        if (t0 + 32 < nnz) {
            const int lset = c[31] >> 6;   // entry 31 belongs to the word's last run
            for (int64_t g = t0 + 32; g < nnz; ++g) {
                if ((__ldg(rsbits + (g >> 5)) >> (g & 31)) & 1u) break;
                const int cg = __ldg(col + g);
                if ((cg >> 6) != lset) break;
                acc |= 1ull << (cg & 63);
            }
        }
        const int64_t b0 = staged ? 0 : s_b0;
        const int rlast = r0 + __popc(hw) - 1;
        if (t0 + 32 <= nnz)
            emit_runs<true>(c, hw, rlast, acc, nnz - t0, staged, b0, s_set, s_lo, s_hi, oset, obits);
        else
            emit_runs<false>(c, hw, rlast, acc, nnz - t0, staged, b0, s_set, s_lo, s_hi, oset, obits);
    }
    if (!staged) return;
    if (w == 0) look_back();
    __syncthreads();
    const int64_t b0 = s_b0;
    for (int xx = threadIdx.x; xx < agg; xx += CT) {
        const int px = xx + (xx >> 5);
        oset[b0 + xx] = s_set[px];
        obits[b0 + xx] = (uint64_t)s_lo[px] | ((uint64_t)s_hi[px] << 32);
    }
}

// rank of the first entry of each row = exclusive head count at rp[r]
__global__ void k_set_starts(int64_t rows, int64_t nnz, const int64_t *__restrict__ rp,
                             const uint32_t *__restrict__ hbits, const uint16_t *__restrict__ wpre,
                             const int64_t *__restrict__ boff, int64_t nblocks,
                             int64_t *__restrict__ start, int32_t *__restrict__ cnt,
                             const int *unsorted, int *dmax) {
    pdl_wait();
    if (*unsorted) return;
    int mx = 0;
    auto rank_at = [&](int64_t e) -> int64_t {
        if (e >= nnz) return boff[nblocks];
        return boff[e / PB] + wpre[e >> 5] + __popc(hbits[e >> 5] & ((1u << (e & 31)) - 1u));
    };   // PB entries per block, wpre block-relative
    // row i's end rank is row i+1's start rank: taken from the next lane
    // (lane 31 computes its own), so each rank is gathered once
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t lim = (rows + 1 + 31) / 32 * 32;   // whole warps stay in the loop
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < lim; i += stride) {
        const bool live = i <= rows;
        // lane 31's second rank is gathered alongside its first (one
        // dependent round trip, not two)
        const bool own_end = live && i < rows && lane == 31;
        const int64_t e0 = live ? rp[i] : 0;
        const int64_t e1 = own_end ? rp[i + 1] : 0;
        const int64_t s0 = live ? rank_at(e0) : 0;
        const int64_t s1_own = own_end ? rank_at(e1) : 0;
        int64_t s1 = __shfl_down_sync(0xffffffffu, s0, 1);
        if (live) {
            start[i] = s0;
            if (i < rows) {
                if (lane == 31) s1 = s1_own;
                const int32_t n = (int32_t)(s1 - s0);
                cnt[i] = n;
                mx = n > mx ? n : mx;
            }
        }
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, d));
    // one atomic per block (one per warp on a single address serialised
    // ~65 K atomics at 2 M rows)
    __shared__ int s_mx;
    if (threadIdx.x == 0) s_mx = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && mx) atomicMax(&s_mx, mx);
    __syncthreads();
    if (threadIdx.x == 0 && s_mx) atomicMax(dmax, s_mx);
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
            if (i < rows) {
                cnt[i] = fcnt[i];
                atomicMax(&cnt[rows + 1], fcnt[i]);   // max set count (slot rows + 1)
            }
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

namespace {
// rows of at most one entry (aggregation operators): each entry is its own set
__global__ void k_compress_unit(int64_t rows, int64_t nnz, const int64_t *__restrict__ rp,
                                const int32_t *__restrict__ col, int64_t *__restrict__ start,
                                int32_t *__restrict__ cnt, int32_t *__restrict__ oset,
                                uint64_t *__restrict__ obits) {
    pdl_wait();
    // max set count: 1 (this path runs only for matrices with entries)
    if (blockIdx.x == 0 && threadIdx.x == 0) cnt[rows + 1] = 1;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t e = rp[i];
        start[i] = e;
        if (i < rows) {
            cnt[i] = (int32_t)(rp[i + 1] - e);
            if (rp[i + 1] > e) {
                const int cv = col[e];
                oset[e] = cv >> 6;
                obits[e] = 1ull << (cv & 63);
            }
        }
    }
}
}  // namespace

int tsg_compress_impl(tsg_ctx *c, const tsg_csr *b, tsg_cmat **out) {
    tsg_cmat *cm = nullptr;
    const int64_t rows = b->rows, nnz = b->nnz;
    // allocation sizes: at least the context's floor (c->cmp_floor_*), so a
    // sequence of growing prefixes of one B reuses the same arena blocks
    const int64_t arows = std::max(rows, c->cmp_floor_rows), annz = std::max(nnz, c->cmp_floor_nnz);
    TSG_TRY(tsg_cmat_alloc(c, arows, annz > 0 ? annz : 1, &cm));
    cm->rows = rows;
    cm->cols = b->cols;
    if (b->max_row >= 0 && b->max_row <= 1 && nnz > 0) {
        TSG_CK(launch_pdl(k_compress_unit, grid_for(rows + 1, 256, c->num_sms * 16), 256, 0, c->stream, rows,
                          nnz, (const int64_t *)b->rp, (const int32_t *)b->col, cm->start, cm->cnt, cm->set,
                          cm->bits));
        ++c->launches;
        cm->sorted_sets = 1;   // one set per row
        cm->dmax_valid = 1;
        cm->identity_rows = (nnz == rows && b->max_row == 1) ? 1 : 0;
        *out = cm;
        return TSG_OK;
    }
    if (nnz == 0) {
        TSG_TRY(tsg_fill(c, cm->start, 0, (rows + 1) * sizeof(int64_t), c->stream));
        TSG_TRY(tsg_fill(c, cm->cnt, 0, (rows + 2) * sizeof(int32_t), c->stream));
        cm->sorted_sets = 1;
        cm->dmax_valid = 1;
        *out = cm;
        return TSG_OK;
    }
    const int64_t nwords = (nnz + 31) / 32, nblocks = (nnz + PB - 1) / PB;   // PB = 8192 entries
    const int64_t anwords = (annz + 31) / 32, anblocks = (annz + PB - 1) / PB;
    uint32_t *rsbits = nullptr, *hbits = nullptr;
    uint16_t *wpre = nullptr;
    int64_t *bcnt = nullptr, *fstart = nullptr;
    int32_t *fcnt = nullptr;
    TSG_TRY(tsg_alloc_t(c, &rsbits, anwords));
    TSG_TRY(tsg_alloc_t(c, &hbits, anwords));
    TSG_TRY(tsg_alloc_t(c, &wpre, anwords));
    TSG_TRY(tsg_alloc_t(c, &bcnt, anblocks + 1));
    TSG_TRY(tsg_alloc_t(c, &fcnt, arows + 1));
    TSG_TRY(tsg_alloc_t(c, &fstart, arows + 1));
    int *unsorted = reinterpret_cast<int *>(c->d_small + 8);
    cudaStream_t s = c->stream;
    TSG_TRY(tsg_fill(c, rsbits, 0, nwords * sizeof(uint32_t), s));
    TSG_TRY(tsg_fill(c, unsorted, 0, sizeof(int), s));
    const unsigned rgrid = grid_for(rows + 1, 256, c->num_sms * 16);
    TSG_CK(launch_pdl(k_row_starts, rgrid, 256, 0, s, rows, (const int64_t *)b->rp, rsbits, cm->cnt + rows + 1));
    ++c->launches;
    unsigned long long *lbstate = nullptr;
    TSG_TRY(tsg_alloc_t(c, &lbstate, anblocks + 1));   // + the tile counter
    TSG_TRY(tsg_fill(c, lbstate, 0, (nblocks + 1) * sizeof(unsigned long long), s));
    const size_t esmem = EMIT_SMEM;
    auto kern = b->sorted ? k_compress_onepass<false> : k_compress_onepass<true>;
    TSG_TRY(tsg_func_smem((const void *)kern, esmem));
    TSG_CK(launch_pdl(kern, (unsigned)nblocks, CT, esmem, s, nnz, (const int32_t *)b->col,
                      (const uint32_t *)rsbits, hbits, wpre, bcnt, nblocks, lbstate,
                      reinterpret_cast<unsigned *>(lbstate + nblocks), cm->set, cm->bits, unsorted,
                      (int64_t)c->num_sms * TSG_CPF));
    ++c->launches;
    // (one row per thread measured slower than this grid-stride loop:
    // 34 vs 27 us at 2 M rows)
    const unsigned sgrid = rgrid;
    TSG_CK(launch_pdl(k_set_starts, sgrid, 256, 0, s, rows, nnz, (const int64_t *)b->rp,
                      (const uint32_t *)hbits, (const uint16_t *)wpre, (const int64_t *)bcnt, nblocks,
                      cm->start, cm->cnt, (const int *)unsorted, cm->cnt + rows + 1));
    ++c->launches;
    // first-occurrence fallback for input not known to be row-sorted: every
    // kernel returns at once if P1 found the rows sorted after all
    if (!b->sorted) {
        const unsigned wgrid = (unsigned)(c->num_sms * 4);   // grid-stride
        k_first_count<<<wgrid, 256, 0, s>>>(rows, b->rp, b->col, fcnt, unsorted); ++c->launches;
        TSG_TRY(tsg_exclusive_scan_i32_to_i64(c, fcnt, fstart, rows));
        k_first_emit<<<wgrid, 256, 0, s>>>(rows, b->rp, b->col, fcnt, fstart, cm->start, cm->cnt,
                                           cm->set, cm->bits, unsorted); ++c->launches;
    }
    TSG_CK(cudaGetLastError());
    tsg_free(c, rsbits);
    tsg_free(c, hbits);
    tsg_free(c, wpre);
    tsg_free(c, bcnt);
    tsg_free(c, lbstate);
    tsg_free(c, fcnt);
    tsg_free(c, fstart);
    cm->sorted_sets = b->sorted;   // first-touch order of a row-sorted B ascends
    cm->dmax_valid = 1;
    *out = cm;
    return TSG_OK;
}

const void *tsg_kernel_compress() { return (const void *)k_row_starts; }
