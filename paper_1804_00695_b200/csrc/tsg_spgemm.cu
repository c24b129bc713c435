// tsg_spgemm.cu -- the two-phase SpGEMM hot path on sm_100a.
//
//   K0 k_row_bounds   per A row: flops = sum nnz(B_k), set bound = sum nnz(CB_k)
//                     (kernel.py:96-103, 135-145)
//   K1 k_compress     B rows -> (set = col>>6, 64-bit mask) in first-touch
//                     order (kernel.py:73-93); padded layout, single pass
//   bins              rows partitioned by accumulator footprint (thread-group,
//                     CTA, or global-memory tier)
//   K2 k_sym_*        exact nnz per C row = popcount of the OR-union of the
//                     compressed B rows (kernel.py:124-168)
//   K3 scan           C row_ptr (tsg_core.cu)
//   K4 k_num_*        C values (kernel.py:171-232), fused multiply-add
//                     variant (kernel.py:235-340) via NumArgs.
//
// Numeric structure: the union of compressed sets is rebuilt in the row's
// table, each occupied set gets base = number of output columns in smaller
// sets, and a product for column c lands at position base(c>>6) +
// rank(c & 63).  Column order within the row is therefore ascending with no
// sort over columns, and values accumulate into a dense per-row array.  In
// the thread-group tier the accumulation replays the reference's order
// (first product, then += in A storage order) with __match_any_sync + an
// ordered shuffle chain, so fp64 results are bit-identical to the CPU
// reference; the CTA and global tiers use fp64 REDG adds (order-free,
// within the 1e-12 parity tolerance).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>
#include <map>
#include <mutex>
#include <tuple>

#include "tsg_group.cuh"
#include <functional>
#include "tsg_partition.cuh"

namespace {

// ======================================================================= args

struct SymArgs {
    const int64_t *arp;
    const int32_t *acol;
    int64_t a_row_off;   // A row = listed row + a_row_off (fused)
    int32_t b_lo, b_hi;  // A columns outside [b_lo, b_hi) are skipped; B row = k - b_lo
    const int64_t *cbstart;
    const int32_t *cbcnt;
    const int32_t *cbset;
    const uint64_t *cbbits;
    const int64_t *prp;  // partial C rows (fused) or null
    const int32_t *pcol;
    const int64_t *sbound;
    int64_t *counts;
    int32_t *msets;
    int *err;
    // optional sorted-set output (group tier): row i's sets go to
    // [sptr[i], sptr[i] + m) of oset / obits, msets[i] gets SETS_WRITTEN
    const int64_t *sptr;
    int32_t *oset;
    uint64_t *obits;
    const int *maxcb;    // device max sets per compressed B row (<= 1: unit path)
    int unit_dense;      // compressed row k is entry k (every B row holds exactly one set)
    // device-driven bins (no host read-back): the launch covers bin `bin`
    // whose rows are list[dbins[bin] .. dbins[bin + 1]) (see bin_range)
    const int64_t *dbins;
    int bin;             // -1: leftover launch over every bin in binmask
    uint32_t binmask;
};

constexpr int SETS_WRITTEN = 1 << 30;

// pass `pass` of a kernel's bin loop: (list, n) of the pass-th bin of a
// leftover launch's mask; false when the mask is exhausted.  A normal launch
// has exactly one pass over its own (list, nlist).
template <class Args, class P>
__device__ __forceinline__ bool leftover_range(const Args &a, int pass, P base, int64_t nbase, P &lst,
                                               int64_t &n) {
    if (!(a.dbins && a.bin < 0)) {
        lst = base;
        n = nbase;
        return pass == 0;
    }
    uint32_t m = a.binmask;
    for (int k = 0; k < pass && m; ++k) m &= m - 1;
    if (!m) return false;
    const int b = __ffs(m) - 1;
    lst = base + a.dbins[b];
    n = a.dbins[b + 1] - a.dbins[b];
    return true;
}

// A bin kernel launched without the host knowing the bin's size takes its
// row range from the partition's device-side bin starts.  A "leftover"
// launch (bin = -1) of the most general group kernel walks every bin in
// binmask in turn: the bins the last same-shape call left empty, so they need
// no launch of their own (leftover_range / the loops of k_sym_group and
// k_num_group).
template <class Args, class P>
__device__ __forceinline__ void bin_range(const Args &a, P &list, int64_t &nlist) {
    if (a.dbins && a.bin >= 0) {
        const int64_t b0 = a.dbins[a.bin];
        nlist = a.dbins[a.bin + 1] - b0;
        list += b0;
    }
}
constexpr int UB = 4;   // A chunks whose loads are batched on the unit-row paths

struct NumArgs {
    const int64_t *arp;
    const int32_t *acol;
    const double *aval;
    int64_t a_row_off;
    int32_t b_lo, b_hi;
    const int64_t *brp;
    const int32_t *bcol;
    const double *bval;
    const int64_t *cbstart;
    const int32_t *cbcnt;
    const int32_t *cbset;
    const uint64_t *cbbits;
    const int64_t *prp;
    const int32_t *pcol;
    const double *pval;
    const int64_t *cptr;
    const int64_t *counts;
    const int32_t *msets;  // may be null
    const int64_t *sbound;
    int32_t *ccol;
    double *cval;
    int *err;
    int seq;   // host-chosen product mode: B rows long enough for lane-per-entry
    const int64_t *sptr;   // sorted sets from the symbolic phase (rows flagged SETS_WRITTEN)
    const int32_t *sset;
    const uint64_t *sbits;
    // capacity mode (chunked executors): counts[i] is row i's final capacity,
    // the partial row is (pcol, pval)[pstart[i] .. + plen_in[i]) -- possibly the
    // output row itself -- and the merged length is written to plen_out[i].
    const int64_t *pstart;
    const int32_t *plen_in;
    int32_t *plen_out;
    const int *unit_b;   // device flag: every B row has <= 1 entry (read if unit_known < 0)
    int unit_known;      // 1 / 0: known on the host (uploaded B), -1: read *unit_b
    int unit_dense;      // B row k is entry k (every row exactly one entry): no row_ptr gather
    const int64_t *dbins;   // device-driven bins, as in SymArgs
    int bin;
    uint32_t binmask;
};

__device__ __forceinline__ void partial_range(const NumArgs &a, int64_t i, int64_t &p0, int64_t &p1) {
    if (a.pstart) {
        p0 = a.pstart[i];
        p1 = p0 + a.plen_in[i];
    } else if (a.prp) {
        p0 = a.prp[i];
        p1 = a.prp[i + 1];
    } else {
        p0 = p1 = 0;
    }
}

// ======================================================================= K0

template <int G>
__global__ void k_row_bounds(int64_t rows, const int64_t *__restrict__ arp,
                             const int32_t *__restrict__ acol, const int64_t *__restrict__ brp,
                             const int32_t *__restrict__ cbcnt, int64_t *__restrict__ flops,
                             int64_t *__restrict__ sbound, unsigned long long *total) {
    const unsigned gm = group_mask<G>();
    const int glane = threadIdx.x & (G - 1);
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
    int64_t mine = 0;
    for (int64_t i = gid; i < rows; i += ngroups) {
        int64_t f = 0, sb = 0;
        for (int64_t t = arp[i] + glane; t < arp[i + 1]; t += G) {
            int k = acol[t];
            f += brp[k + 1] - brp[k];
            if (cbcnt) sb += cbcnt[k];
        }
        f = group_sum<G, int64_t>(gm, f);
        if (cbcnt) sb = group_sum<G, int64_t>(gm, sb);
        if (glane == 0) {
            if (flops) flops[i] = f;
            if (sbound) sbound[i] = cbcnt ? sb : f;
            mine += f;
        }
    }
    if (total) {
        for (int d = 16; d >= 1; d >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, d);
        if ((threadIdx.x & 31) == 0 && mine) atomicAdd(total, (unsigned long long)mine);
    }
}

__global__ void k_max_i32(int64_t n, const int32_t *__restrict__ v, int *out) {
    int m = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, v[i]);
    for (int d = 16; d >= 1; d >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, d));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// Symbolic set bound per A row.  When every compressed B row is short
// (max <= CHEAP_CB) the bound len(A_i) * max needs no gather at all (exact
// for aggregation operators, within ~10 % for stencils); skewed B falls back
// to the exact sum of the selected compressed rows.
constexpr int CHEAP_CB = 16;
constexpr int INLINE_BOUND_A = 16;   // A rows up to this long: exact bound in the bin functor

template <int G>
__global__ void k_sym_bounds(int64_t rows, const int64_t *__restrict__ arp,
                             const int32_t *__restrict__ acol, const int32_t *__restrict__ cbcnt,
                             const int *maxcb, int64_t *__restrict__ sbound) {
    pdl_wait();
    const int mcb = *maxcb;
    if (mcb <= CHEAP_CB) return;   // cheap bound len x max: computed by the bin functor (SymBinF)
    const unsigned gm = group_mask<G>();
    const int glane = threadIdx.x & (G - 1);
    const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
    const int64_t ngroups = ((int64_t)gridDim.x * blockDim.x) / G;
    for (int64_t i = gid; i < rows; i += ngroups) {
        int64_t sb = 0;
        for (int64_t t = arp[i] + glane; t < arp[i + 1]; t += G) sb += cbcnt[acol[t]];
        sb = group_sum<G, int64_t>(gm, sb);
        if (glane == 0) sbound[i] = sb;
    }
}

// ======================================================================= bins
// Tier sizes.  Thread-group tier: a G-lane group owns a SLICE-byte region of
// shared memory (table + dense values).  CTA tier: one row per CTA, table in
// shared memory.  Global tier: one row per CTA, table in a global slab.

constexpr int NBINS = 15;   // 0-6 group, 7-8 CTA, 9 global, 10-12 symbolic merge, 13 dense, 14 thread
// bins 0..6: group tier slices (bytes) and group sizes
__host__ __device__ constexpr int gt_slice(int b) { return 512 << b; }
#ifndef TSG_NUM_G1
#define TSG_NUM_G1 8   // lanes per row of numeric bin 1 (config 2 R*A numeric: 4 -> 0.486 ms, 8 -> 0.362, 16 -> 0.547)
#endif
#ifndef TSG_NUM_G0
#define TSG_NUM_G0 8   // lanes per row of numeric bin 0 (config 1: 4 -> 0.167 ms, 8 -> 0.165)
#endif
__host__ __device__ constexpr int gt_g(int b) { return b == 0 ? TSG_NUM_G0 : b == 1 ? TSG_NUM_G1 : (b == 2 ? 16 : 32); }
// symbolic tables are larger (bounded by compressed entries, not exact sets)
__host__ __device__ constexpr int gt_g_sym(int b) { return b == 0 ? 8 : (b == 1 ? 16 : 32); }
__host__ __device__ constexpr int gt_block(int b) { return b <= 4 ? 256 : (b == 5 ? 128 : 64); }
// bins 7, 8: CTA tier table slots (smem table 16 B/slot + sort keys 8 B/slot)
__host__ __device__ constexpr int ct_slots(int cb) { return 2048 << (2 * cb); }
__host__ __device__ constexpr int ct_nt(int cb) { return 256 << cb; }
constexpr int BIN_GLOBAL = 9;
// bins 10..12 (symbolic only): k-way merge of the row's sorted compressed B
// rows, one list per lane -- G = 8/16/32 lanes, lists staged in SLICE bytes
__host__ __device__ constexpr int mt_g(int m) { return 8 << m; }
__host__ __device__ constexpr int mt_slice(int m) { return 1024 << m; }
__host__ __device__ constexpr int mt_cap(int m) { return mt_slice(m) / 12; }   // staged (set, mask) pairs
constexpr int BIN_MERGE = 10;
// bin 13: dense tier for rows whose bound is a sizeable fraction of B's
// columns (power-law hubs): one CTA per row, a shared-memory bitmap of all
// of B's column sets (symbolic) / a per-set base + mask array (numeric).
constexpr int BIN_DENSE = 13;
// bin 14 (symbolic): thread-per-row tier for B with exactly one entry per row
// (aggregation operators, RA*P): each A entry adds one set, so one thread per
// row keeps the row's sorted sets itself -- no group coordination, no table.
// (A thread-per-row numeric measured slower than the group tier: 0.37 vs
// 0.26 ms on config 2's RA*P -- its per-product chains are latency-bound.)
constexpr int BIN_THREAD = 14;
constexpr int THREAD_MAX_A = 64;
constexpr int DENSE_MIN_SETS = 2048;           // bound (sets) from which a row goes dense
constexpr int64_t DENSE_SMEM = 200 * 1024;     // shared-memory budget of the dense kernels
__host__ __device__ __forceinline__ int64_t dense_words(int64_t ncols) { return (ncols + 63) / 64; }
// set bound from which a row takes the dense tier: 2048 while B's column-set
// bitmap fits shared memory; beyond that the symbolic bitmap is an L2-resident
// per-CTA slab whose emission scans all of B's sets, so rows must be long
// enough to amortise that (R-MAT scale 21 without it: 132 s in the global tier)
__host__ __device__ __forceinline__ int64_t dense_min_sets(int64_t ncols) {
    const int64_t nw = dense_words(ncols);
    return nw * 8 <= DENSE_SMEM ? DENSE_MIN_SETS : (nw / 8 > DENSE_MIN_SETS ? nw / 8 : DENSE_MIN_SETS);
}

__host__ __device__ __forceinline__ int64_t round16(int64_t x) { return (x + 15) & ~(int64_t)15; }

// symbolic: table only (16 B/slot)
__host__ __device__ __forceinline__ int sym_bin(int64_t sbound) {
    if (sbound <= 0) return 255;
    int64_t T = table_slots(sbound);
    int64_t need = 24 * T;
    for (int b = 0; b < 7; b++)
        if (need <= gt_slice(b)) return b;
    for (int b = 0; b < 2; b++)
        if (T <= ct_slots(b)) return 7 + b;
    return BIN_GLOBAL;
}

// numeric: table + dense fp64 values for the group tier; table for CTA tier
__host__ __device__ __forceinline__ int num_bin(int64_t n, int64_t m) {
    if (n <= 0) return 255;
    int64_t T = table_slots(m);
    int64_t need = round16(8 * n) + 16 * T;
    for (int b = 0; b < 7; b++)
        if (need <= gt_slice(b)) return b;
    for (int b = 0; b < 2; b++)
        if (T <= ct_slots(b)) return 7 + b;
    return BIN_GLOBAL;
}

// flag = 1 iff every row of the (row_ptr or count) array holds <= 1 entry
__global__ void k_unit_rows(int64_t rows, const int64_t *__restrict__ rp, const int32_t *__restrict__ cnt,
                            int *flag) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < rows;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t len = rp ? rp[i + 1] - rp[i] : cnt[i];
        if (len > 1) {
            *flag = 0;
            return;
        }
    }
}

// per-row bin functors for tsg_partition (tsg_partition.cuh)
struct SymBinF {
    int64_t *sbound;
    int64_t *counts;
    int32_t *msets;
    int64_t *scap;
    const int64_t *arp;   // non-null: merge tier allowed (row-sorted B, no partial rows)
    int64_t a_row_off;
    int64_t ncols;        // B's columns (> 0: dense tier allowed)
    const int64_t *carp;  // non-null: cheap bound len(A_i) x max when *cmax <= CHEAP_CB
    const int *cmax;
    const int64_t *tarp;  // non-null: thread tier allowed (B rows are exactly one entry each)
    const int32_t *ecol;  // non-null (with carp): short A rows, exact bound summed here
    const int32_t *ecnt;  //   over ecnt[ecol[t]] instead of by k_sym_bounds
    __device__ __forceinline__ int operator()(int64_t i) const {
        if (tarp) {
            const int64_t alen = tarp[i + a_row_off + 1] - tarp[i + a_row_off];
            if (alen > 0 && alen <= THREAD_MAX_A) {
                sbound[i] = alen;
                scap[i] = alen;
                return BIN_THREAD;
            }
        }
        int64_t sb;
        if (carp && *cmax <= CHEAP_CB) {
            sb = (carp[i + 1] - carp[i]) * (int64_t)*cmax;
            sbound[i] = sb;
        } else if (carp && ecol) {
            // 8 entries per batch with all their gathers in flight (short A
            // rows: one round trip for the columns, one for the counts)
            sb = 0;
            const int64_t t0 = carp[i], t1 = carp[i + 1];
            for (int64_t t = t0; t < t1; t += 8) {
                int cc[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) cc[u] = t + u < t1 ? ecol[t + u] : -1;
#pragma unroll
                for (int u = 0; u < 8; ++u) sb += cc[u] >= 0 ? ecnt[cc[u]] : 0;
            }
            sbound[i] = sb;
        } else {
            sb = sbound[i];
        }
        int b = sym_bin(sb);
        if (ncols > 0 && sb >= dense_min_sets(ncols)) {
            scap[i] = sb;
            return BIN_DENSE;
        }
        if (arp && b != 255) {
            // few A entries, bounded staging: merge the sorted lists instead of hashing
            const int64_t alen = arp[i + a_row_off + 1] - arp[i + a_row_off];
            for (int m = 0; m < 3; ++m)
                if (alen <= mt_g(m) && sb <= mt_cap(m)) {
                    b = BIN_MERGE + m;
                    break;
                }
        }
        scap[i] = (b < 7 || b >= BIN_MERGE) ? sb : 0;   // these tiers emit sorted sets
        if (b == 255) {
            counts[i] = 0;
            if (msets) msets[i] = 0;
        }
        return b;
    }
};

struct NumBinF {
    const int64_t *counts;
    const int32_t *msets;
    const int64_t *sbound;
    int64_t ncols;        // B's columns (> 0: dense tier allowed for rows with sorted sets)
    int skip_idle = 0;    // in-place fused step: rows with no product in the chunk keep their partial
    __device__ __forceinline__ int operator()(int64_t i) const {
        if (skip_idle && sbound[i] == 0) return 255;
        const int64_t n = counts[i];
        const int64_t m = msets ? (int64_t)(msets[i] & (SETS_WRITTEN - 1)) : (sbound[i] < n ? sbound[i] : n);
        const int b = num_bin(n, m);
        if (ncols > 0 && b >= 7 && b != 255 && msets && (msets[i] & SETS_WRITTEN))   // windowed: any B width
            return BIN_DENSE;
        return b;
    }
};

// ======================================================================= K2 group tier

constexpr int SYM_OPT_T = 32;   // first table size for unit rows (up to 32 distinct sets)

template <int G, int SLICE>
__global__ void __launch_bounds__(256) k_sym_group(const int32_t *__restrict__ list, int64_t nlist,
                                                   SymArgs a) {
    bin_range(a, list, nlist);
    extern __shared__ int4 smem[];
    constexpr int TMAX = SLICE / 24;   // 16 B table slot + 8 B sort key per slot
    const unsigned gm = group_mask<G>();
    const int glane = threadIdx.x & (G - 1);
    const int gpb = blockDim.x / G;
    int4 *tbl = reinterpret_cast<int4 *>(reinterpret_cast<char *>(smem) + (size_t)(threadIdx.x / G) * SLICE);
    for (int pass_ = 0;; ++pass_) {
    const int32_t *lst_;
    int64_t nl_;
    if (!leftover_range(a, pass_, list, nlist, lst_, nl_)) break;
    for (int64_t li = (int64_t)blockIdx.x * gpb + threadIdx.x / G; li < nl_;
         li += (int64_t)gridDim.x * gpb) {
        const int64_t i = lst_[li];
        const int64_t gi = i + a.a_row_off;
        int T = table_slots(a.sbound[i]);
        if (T > TMAX) T = 1 << ilog2_pow2(TMAX);
        const int Tfull = T;
        const bool unit = a.maxcb && *a.maxcb <= 1;
        // unit compressed rows: the bound (one set per A entry) overstates the
        // distinct sets several-fold (RA*P rows: 64 entries, ~10 sets), so the
        // union first runs in a small table and is redone at the bound's size
        // only if that one overflows
        if (unit && T > SYM_OPT_T) T = SYM_OPT_T;
        int logT;
        bool ok;
        for (;;) {
        logT = ilog2_pow2(T);
        tbl_clear(tbl, T, glane, G);
        __syncwarp(gm);
        ok = true;
        if (a.prp) {
            for (int64_t q = a.prp[i] + glane; q < a.prp[i + 1]; q += G) {
                int c = a.pcol[q];
                int bit = c & 63;
                ok &= tbl_or(tbl, T, logT, c >> 6, bit < 32 ? 1u << bit : 0u,
                             bit >= 32 ? 1u << (bit - 32) : 0u);
            }
        }
        if (unit) {
            // unit compressed rows: batch the three dependent load rounds of UB chunks
            const int64_t a0 = a.arp[gi], a1 = a.arp[gi + 1];
            for (int64_t base = a0; base < a1; base += UB * G) {
                int kk[UB];
#pragma unroll
                for (int u = 0; u < UB; ++u) {
                    const int64_t t = base + u * G + glane;
                    const int k = t < a1 ? a.acol[t] : -1;
                    kk[u] = (k >= a.b_lo && k < a.b_hi) ? k - a.b_lo : -1;
                }
                int64_t ss[UB];
                bool has[UB];
                if (a.unit_dense) {
#pragma unroll
                    for (int u = 0; u < UB; ++u) {
                        ss[u] = kk[u] >= 0 ? kk[u] : 0;
                        has[u] = kk[u] >= 0;
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < UB; ++u) {
                        ss[u] = kk[u] >= 0 ? a.cbstart[kk[u]] : 0;
                        has[u] = kk[u] >= 0 && a.cbcnt[kk[u]] > 0;
                    }
                }
#pragma unroll
                for (int u = 0; u < UB; ++u) {
                    if (has[u]) {
                        const uint64_t bits = a.cbbits[ss[u]];
                        ok &= tbl_or(tbl, T, logT, a.cbset[ss[u]], (unsigned)bits,
                                     (unsigned)(bits >> 32));
                    }
                }
            }
        } else {
            group_enumerate_any<G>(
                gm, glane, a.arp[gi], a.arp[gi + 1],
                [&](int64_t t, int64_t &st, int &len) {
                    int k = a.acol[t];
                    if (k >= a.b_lo && k < a.b_hi) {
                        k -= a.b_lo;
                        st = a.cbstart[k];
                        len = a.cbcnt[k];
                    }
                },
                [&](bool valid, int, int64_t, int64_t s) {
                    if (valid) {
                        uint64_t bits = a.cbbits[s];
                        ok &= tbl_or(tbl, T, logT, a.cbset[s], (unsigned)bits, (unsigned)(bits >> 32));
                    }
                });
        }
        __syncwarp(gm);
        if (T == Tfull || __all_sync(gm, ok)) break;
        T = Tfull;   // the optimistic table overflowed: redo at the bound's size
        }
        // compact occupied slots as sortable (key << 32 | slot) into the scratch
        // area behind the table; count columns on the way
        uint64_t *ck = reinterpret_cast<uint64_t *>(tbl + T);
        const unsigned lt = lanemask_lt();
        int cnt = 0, m = 0;
        for (int r0 = 0; r0 < T; r0 += G) {
            int s = r0 + glane;
            int4 e = s < T ? tbl[s] : make_int4(TSG_EMPTY, 0, 0, 0);
            bool occ = e.x != TSG_EMPTY;
            unsigned bal = __ballot_sync(gm, occ) & gm;
            if (occ) {
                cnt += slot_pop(e);
                ck[m + __popc(bal & lt)] = ((uint64_t)(uint32_t)e.x << 32) | (uint32_t)s;
            }
            m += __popc(bal);
        }
        cnt = group_sum<G, int>(gm, cnt);
        if (!ok) kerr(a.err, KERR_PROBE, gi);
        bool emit = a.oset != nullptr && ok && m <= a.sbound[i];
        if (emit) {
            __syncwarp(gm);
            const int64_t sp = a.sptr[i];
            if (m <= 64) {
                // rank sort: entry q goes to #keys smaller than it
                for (int q = glane; q < m; q += G) {
                    uint64_t me = ck[q];
                    int r = 0;
                    for (int u = 0; u < m; ++u) r += (ck[u] < me);
                    int slot = (int)(uint32_t)me;
                    int4 e = tbl[slot];
                    a.oset[sp + r] = e.x;
                    a.obits[sp + r] = ((uint64_t)(uint32_t)e.z << 32) | (uint32_t)e.y;
                }
            } else {
                int P = 1;
                while (P < m) P <<= 1;
                for (int q = m + glane; q < P; q += G) ck[q] = ~0ull;
                __syncwarp(gm);
                for (int k = 2; k <= P; k <<= 1) {
                    for (int j = k >> 1; j > 0; j >>= 1) {
                        for (int x = glane; x < P; x += G) {
                            int y = x ^ j;
                            if (y > x) {
                                uint64_t kx = ck[x], ky = ck[y];
                                if ((kx > ky) == ((x & k) == 0)) {
                                    ck[x] = ky;
                                    ck[y] = kx;
                                }
                            }
                        }
                        __syncwarp(gm);
                    }
                }
                for (int q = glane; q < m; q += G) {
                    int4 e = tbl[(int)(uint32_t)ck[q]];
                    a.oset[sp + q] = e.x;
                    a.obits[sp + q] = ((uint64_t)(uint32_t)e.z << 32) | (uint32_t)e.y;
                }
            }
        }
        if (glane == 0) {
            a.counts[i] = cnt;
            if (a.msets) a.msets[i] = m | (emit ? SETS_WRITTEN : 0);
        }
        __syncwarp(gm);
    }
    }
}

// Merge tier: a row with at most G A entries whose compressed B rows are
// sorted by set (compact compression of a row-sorted B).  Lane j stages list j
// (its A entry's compressed row) in shared memory, then the group repeatedly
// takes the minimum head set (shuffle min), ORs the masks of the lanes holding
// it (shuffle OR) and advances them: the union comes out already sorted and
// de-duplicated -- no table, no atomics, no sort.
template <int G, int SLICE>
__global__ void __launch_bounds__(256) k_sym_merge(const int32_t *__restrict__ list, int64_t nlist,
                                                   SymArgs a) {
    bin_range(a, list, nlist);
    extern __shared__ int4 smem[];
    constexpr int CAP = SLICE / 12;
    const unsigned gm = group_mask<G>();
    const int glane = threadIdx.x & (G - 1);
    const int gpb = blockDim.x / G;
    const int g = threadIdx.x / G;
    uint64_t *lbits = reinterpret_cast<uint64_t *>(reinterpret_cast<char *>(smem) + (size_t)g * SLICE);
    int32_t *lset = reinterpret_cast<int32_t *>(lbits + CAP);
    for (int64_t li = (int64_t)blockIdx.x * gpb + g; li < nlist; li += (int64_t)gridDim.x * gpb) {
        const int64_t i = list[li];
        const int64_t gi = i + a.a_row_off;
        const int64_t a0 = a.arp[gi], a1 = a.arp[gi + 1];
        int64_t st = 0;
        int cnt = 0;
        if (a0 + glane < a1) {
            int k = a.acol[a0 + glane];
            if (k >= a.b_lo && k < a.b_hi) {
                k -= a.b_lo;
                st = a.cbstart[k];
                cnt = a.cbcnt[k];
            }
        }
        const int incl = group_incl_scan<G, int>(gm, cnt, glane);
        const int off = incl - cnt;
        // stage the list (independent loads, four in flight per lane)
        for (int q0 = 0; q0 < cnt; q0 += 4) {
            int sv[4];
            uint64_t bv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int q = q0 + u < cnt ? q0 + u : cnt - 1;
                sv[u] = a.cbset[st + q];
                bv[u] = a.cbbits[st + q];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (q0 + u < cnt) {
                    lset[off + q0 + u] = sv[u];
                    lbits[off + q0 + u] = bv[u];
                }
        }
        __syncwarp(gm);
        int p = off;
        const int e = off + cnt;
        int hs = p < e ? lset[p] : INT32_MAX;
        uint64_t hb = p < e ? lbits[p] : 0ull;
        const int64_t sp = a.sptr[i];
        int m = 0, total = 0;
        for (;;) {
            // group minimum head (min butterfly), then the OR of the masks of
            // the lanes holding it (OR butterfly): no compare-select chains
            int mn = hs;
#pragma unroll
            for (int d = G / 2; d >= 1; d >>= 1) mn = min(mn, __shfl_xor_sync(gm, mn, d, G));
            if (mn == INT32_MAX) break;
            const bool mine = hs == mn;
            unsigned lo = mine ? (unsigned)hb : 0u, hi = mine ? (unsigned)(hb >> 32) : 0u;
#pragma unroll
            for (int d = G / 2; d >= 1; d >>= 1) {
                lo |= __shfl_xor_sync(gm, lo, d, G);
                hi |= __shfl_xor_sync(gm, hi, d, G);
            }
            if (glane == 0) {
                a.oset[sp + m] = mn;
                a.obits[sp + m] = ((uint64_t)hi << 32) | lo;
            }
            total += __popc(lo) + __popc(hi);
            ++m;
            if (mine) {
                ++p;
                hs = p < e ? lset[p] : INT32_MAX;
                hb = p < e ? lbits[p] : 0ull;
            }
        }
        if (glane == 0) {
            a.counts[i] = total;
            if (a.msets) a.msets[i] = m | SETS_WRITTEN;
        }
        __syncwarp(gm);
    }
}

// Merge tier with K lists per lane: G lanes own a row of at most K*G A
// entries, lane j merges the compressed rows of entries j, j + G, ... on the
// fly (its head = the smallest of its list heads, equal heads ORed), and the
// group combines the G lane heads as above.  Fewer lanes per row means fewer
// shuffles per output set per row: the 8-list merge was bound by the
// shuffle (MIO) pipe.
template <int G, int K, int SLICE>
__global__ void __launch_bounds__(256) k_sym_merge2(const int32_t *__restrict__ list, int64_t nlist,
                                                    SymArgs a) {
    bin_range(a, list, nlist);
    extern __shared__ int4 smem[];
    constexpr int CAP = SLICE / 12;
    const unsigned gm = group_mask<G>();
    const int glane = threadIdx.x & (G - 1);
    const int gpb = blockDim.x / G;
    const int g = threadIdx.x / G;
    uint64_t *lbits = reinterpret_cast<uint64_t *>(reinterpret_cast<char *>(smem) + (size_t)g * SLICE);
    int32_t *lset = reinterpret_cast<int32_t *>(lbits + CAP);
    for (int64_t li = (int64_t)blockIdx.x * gpb + g; li < nlist; li += (int64_t)gridDim.x * gpb) {
        const int64_t i = list[li];
        const int64_t gi = i + a.a_row_off;
        const int64_t a0 = a.arp[gi], a1 = a.arp[gi + 1];
        int64_t st[K];
        int cnt[K];
#pragma unroll
        for (int u = 0; u < K; ++u) {
            st[u] = 0;
            cnt[u] = 0;
            if (a0 + glane + u * G < a1) {
                int k = a.acol[a0 + glane + u * G];
                if (k >= a.b_lo && k < a.b_hi) {
                    k -= a.b_lo;
                    st[u] = a.cbstart[k];
                    cnt[u] = a.cbcnt[k];
                }
            }
        }
        int tot = 0;
#pragma unroll
        for (int u = 0; u < K; ++u) tot += cnt[u];
        const int incl = group_incl_scan<G, int>(gm, tot, glane);
        int p[K], e[K];
        {
            int off = incl - tot;
#pragma unroll
            for (int u = 0; u < K; ++u) {
                p[u] = off;
                off += cnt[u];
                e[u] = off;
            }
        }
#ifndef MERGE_CP_ASYNC
#define MERGE_CP_ASYNC 1
#endif
#if MERGE_CP_ASYNC
        // stage the lists with asynchronous global->shared copies: every
        // entry of the lane's K lists is in flight at once and the lane
        // waits a single round trip (the register-staged form waited one
        // per 4-entry batch, ~6 per row)
#pragma unroll
        for (int u = 0; u < K; ++u) {
            const unsigned ds = (unsigned)__cvta_generic_to_shared(lset + p[u]);
            const unsigned db = (unsigned)__cvta_generic_to_shared(lbits + p[u]);
            const int32_t *gs = a.cbset + st[u];
            const uint64_t *gb = a.cbbits + st[u];
#pragma unroll 4
            for (int q = 0; q < cnt[u]; ++q) {
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(ds + 4u * q), "l"(gs + q)
                             : "memory");
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(db + 8u * q), "l"(gb + q)
                             : "memory");
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
#else
        // stage the lists (independent loads, four in flight per lane)
#pragma unroll
        for (int u = 0; u < K; ++u) {
            for (int q0 = 0; q0 < cnt[u]; q0 += 4) {
                int sv[4];
                uint64_t bv[4];
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    const int q = q0 + v < cnt[u] ? q0 + v : cnt[u] - 1;
                    sv[v] = a.cbset[st[u] + q];
                    bv[v] = a.cbbits[st[u] + q];
                }
#pragma unroll
                for (int v = 0; v < 4; ++v)
                    if (q0 + v < cnt[u]) {
                        lset[p[u] + q0 + v] = sv[v];
                        lbits[p[u] + q0 + v] = bv[v];
                    }
            }
        }
#endif
        __syncwarp(gm);
        int h[K];
        uint64_t mk[K];
#pragma unroll
        for (int u = 0; u < K; ++u) {
            h[u] = p[u] < e[u] ? lset[p[u]] : INT32_MAX;
            mk[u] = p[u] < e[u] ? lbits[p[u]] : 0ull;
        }
        const int64_t sp = a.sptr[i];
        int m = 0, total = 0;
        for (;;) {
            int mn = h[0];
#pragma unroll
            for (int u = 1; u < K; ++u) mn = min(mn, h[u]);
#pragma unroll
            for (int d = G / 2; d >= 1; d >>= 1) mn = min(mn, __shfl_xor_sync(gm, mn, d, G));
            if (mn == INT32_MAX) break;
            uint64_t hm = 0ull;
#pragma unroll
            for (int u = 0; u < K; ++u) hm |= h[u] == mn ? mk[u] : 0ull;
            unsigned lo = (unsigned)hm, hi = (unsigned)(hm >> 32);
#pragma unroll
            for (int d = G / 2; d >= 1; d >>= 1) {
                lo |= __shfl_xor_sync(gm, lo, d, G);
                hi |= __shfl_xor_sync(gm, hi, d, G);
            }
            if (glane == 0) {
                a.oset[sp + m] = mn;
                a.obits[sp + m] = ((uint64_t)hi << 32) | lo;
            }
            total += __popc(lo) + __popc(hi);
            ++m;
#pragma unroll
            for (int u = 0; u < K; ++u) {
                if (h[u] == mn) {
                    ++p[u];
                    h[u] = p[u] < e[u] ? lset[p[u]] : INT32_MAX;
                    mk[u] = p[u] < e[u] ? lbits[p[u]] : 0ull;
                }
            }
        }
        if (glane == 0) {
            a.counts[i] = total;
            if (a.msets) a.msets[i] = m | SETS_WRITTEN;
        }
        __syncwarp(gm);
    }
}

// Merge tier without shared memory: each lane keeps its K list heads AND the
// next entry of each list in registers (the next-next entry is loaded as a
// head advances, one iteration ahead of its use), so no staging, no shared
// memory bank conflicts and no shared-memory occupancy cap.  Lists are short
// (compressed rows of a stencil: ~9 pairs), contiguous, and L1-resident after
// their first sector.
template <int G, int K>
__global__ void __launch_bounds__(256) k_sym_merge3(const int32_t *__restrict__ list, int64_t nlist,
                                                    SymArgs a) {
    bin_range(a, list, nlist);
    const unsigned gm = group_mask<G>();
    const int glane = threadIdx.x & (G - 1);
    const int gpb = blockDim.x / G;
    const int g = threadIdx.x / G;
    for (int64_t li = (int64_t)blockIdx.x * gpb + g; li < nlist; li += (int64_t)gridDim.x * gpb) {
        const int64_t i = list[li];
        const int64_t gi = i + a.a_row_off;
        const int64_t a0 = a.arp[gi], a1 = a.arp[gi + 1];
        int64_t p[K], e[K];
#pragma unroll
        for (int u = 0; u < K; ++u) {
            p[u] = 0;
            e[u] = 0;
            const int64_t t = a0 + glane + u * G;
            if (t < a1) {
                int k = a.acol[t];
                if (k >= a.b_lo && k < a.b_hi) {
                    k -= a.b_lo;
                    p[u] = a.cbstart[k];
                    e[u] = p[u] + a.cbcnt[k];
                }
            }
        }
        int h[K], hn[K];
        uint64_t mk[K], mkn[K];
#pragma unroll
        for (int u = 0; u < K; ++u) {
            const bool v0 = p[u] < e[u], v1 = p[u] + 1 < e[u];
            h[u] = v0 ? __ldg(a.cbset + p[u]) : INT32_MAX;
            mk[u] = v0 ? __ldg(a.cbbits + p[u]) : 0ull;
            hn[u] = v1 ? __ldg(a.cbset + p[u] + 1) : INT32_MAX;
            mkn[u] = v1 ? __ldg(a.cbbits + p[u] + 1) : 0ull;
        }
        const int64_t sp = a.sptr[i];
        int m = 0, total = 0;
        for (;;) {
            int mn = h[0];
#pragma unroll
            for (int u = 1; u < K; ++u) mn = min(mn, h[u]);
#pragma unroll
            for (int d = G / 2; d >= 1; d >>= 1) mn = min(mn, __shfl_xor_sync(gm, mn, d, G));
            if (mn == INT32_MAX) break;
            uint64_t hm = 0ull;
#pragma unroll
            for (int u = 0; u < K; ++u) hm |= h[u] == mn ? mk[u] : 0ull;
            unsigned lo = (unsigned)hm, hi = (unsigned)(hm >> 32);
#pragma unroll
            for (int d = G / 2; d >= 1; d >>= 1) {
                lo |= __shfl_xor_sync(gm, lo, d, G);
                hi |= __shfl_xor_sync(gm, hi, d, G);
            }
            if (glane == 0) {
                a.oset[sp + m] = mn;
                a.obits[sp + m] = ((uint64_t)hi << 32) | lo;
            }
            total += __popc(lo) + __popc(hi);
            ++m;
#pragma unroll
            for (int u = 0; u < K; ++u) {
                if (h[u] == mn) {
                    ++p[u];
                    h[u] = hn[u];
                    mk[u] = mkn[u];
                    const bool v1 = p[u] + 1 < e[u];
                    hn[u] = v1 ? __ldg(a.cbset + p[u] + 1) : INT32_MAX;
                    mkn[u] = v1 ? __ldg(a.cbbits + p[u] + 1) : 0ull;
                }
            }
        }
        if (glane == 0) {
            a.counts[i] = total;
            if (a.msets) a.msets[i] = m | SETS_WRITTEN;
        }
    }
}

#ifndef MERGE_IMPL
#define MERGE_IMPL 3   // 2: lists staged in shared memory (k_sym_merge2), 3: in registers (k_sym_merge3)
#endif
#ifndef MERGE_LISTS_PER_LANE
#define MERGE_LISTS_PER_LANE 2
#endif
template <int M>
int launch_sym_merge(tsg_ctx *c, const ::BinLists<NBINS> &bl, const SymArgs &a);

// The dense tiers enumerate through block_unit_enumerate (tsg_group.cuh):
// R-MAT scale 18 symbolic 48 -> 44 ms over a warp per A entry (and 16 ms with
// the popcount total fixed below), numeric 108 -> 80 ms over the flattened
// block enumeration.
#ifndef DENSE_EB
#define DENSE_EB 512   // A entries per enumeration round (block_unit_enumerate)
#endif
#ifndef DENSE_CH
#define DENSE_CH 128   // elements per warp unit
#endif
#ifndef DENSE_CH_NUM
#define DENSE_CH_NUM DENSE_CH   // numeric window unit (R-MAT scale 20: 64 -> 668 ms, 128 -> 649, 256 -> 664)
#endif

// Dense symbolic tier: the row's union is ORed into a shared-memory bitmap
// of all of B's column sets (64-bit words, ORed as 32-bit halves), then the
// nonzero words are emitted in ascending set order -- no table, no sort.
// MODE 0: one shared bitmap of all of B's column sets.  MODE 1 (B wider
// than shared memory, row-sorted): the sets in column windows of `wwords`,
// one window after another per row; each entry's compressed B row is cut to
// the window by precomputed offsets (k_sym_dense_cut) and the emitted sets
// and counts carry across windows.  MODE 2 (unsorted B wider than shared
// memory): an L2-resident bitmap slab per CTA (zeroed by the host once,
// re-zeroed as emitted), ORed with fire-and-forget global atomics and read
// with L1-bypassing loads -- L2 atomic throughput bounds it (R-MAT scale 21:
// 2.0 s against 132 s in the global hash tier).
template <int NT, int MODE>
__global__ void __launch_bounds__(NT, 2048 / NT) k_sym_dense(const int32_t *__restrict__ list, int64_t nlist,
                                                  SymArgs a, int64_t nwords, int64_t wwords, uint64_t *gbm,
                                                  const int64_t *__restrict__ coff, int64_t cut_base,
                                                  const int32_t *__restrict__ cut) {
    extern __shared__ int4 smem[];
    __shared__ int s_warp[32];
    __shared__ unsigned s_cnt;
    __shared__ int s_nz;
    uint64_t *bm = MODE == 2 ? gbm + (int64_t)blockIdx.x * nwords : reinterpret_cast<uint64_t *>(smem);
    unsigned *bm32 = reinterpret_cast<unsigned *>(bm);
    const int64_t ww = MODE == 1 ? wwords : nwords;   // words per window
    const int nwin = MODE == 1 ? (int)((nwords + wwords - 1) / wwords) : 1;
    for (int64_t li = blockIdx.x; li < nlist; li += gridDim.x) {
        const int64_t i = list[li];
        const int64_t gi = i + a.a_row_off;
        const int64_t a0 = a.arp[gi], a1 = a.arp[gi + 1];
        if (threadIdx.x == 0) {
            s_cnt = 0u;
            s_nz = 0;
        }
        const int64_t sp = a.oset ? a.sptr[i] : 0;
        for (int win = 0; win < nwin; ++win) {
            const int64_t lo = (int64_t)win * ww;
            const int64_t wn = nwords - lo < ww ? nwords - lo : ww;   // words in this window
            if (MODE != 2)
                for (int64_t w = threadIdx.x; w < wn; w += NT) bm[w] = 0ull;
            __syncthreads();
            struct SB {
                int set;
                uint64_t bits;
            };
            block_unit_enumerate<NT, DENSE_EB, DENSE_CH, SB>(
                a0, a1,
                [&](int64_t t, int64_t &st, int &len, double &) {
                    int k = a.acol[t];
                    if (k >= a.b_lo && k < a.b_hi) {
                        k -= a.b_lo;
                        st = a.cbstart[k];
                        len = a.cbcnt[k];
                        if (MODE == 1) {
                            const int64_t alen = a1 - a0;
                            const int32_t *cr = cut + (coff[li] - cut_base) + (t - a0);
                            const int c0 = win > 0 ? cr[(win - 1) * alen] : 0;
                            const int c1 = win + 1 < nwin ? cr[win * alen] : len;
                            st += c0;
                            len = c1 - c0;
                        }
                    }
                },
                [&](int64_t sidx) { return SB{a.cbset[sidx], a.cbbits[sidx]}; },
                [&](double, const SB &x) {
                    const int64_t o = 2 * (x.set - lo);
                    if ((unsigned)x.bits) atomicOr(&bm32[o], (unsigned)x.bits);
                    if ((unsigned)(x.bits >> 32)) atomicOr(&bm32[o + 1], (unsigned)(x.bits >> 32));
                },
                s_warp);
            __syncthreads();
            // each thread owns a contiguous run of words: count its nonzero
            // sets, block-scan the counts, emit its sets in order
            const int64_t per = (wn + NT - 1) / NT;
            const int64_t w0 = threadIdx.x * per, w1 = w0 + per < wn ? w0 + per : wn;
            int nz = 0;
            unsigned pc = 0;
            for (int64_t w = w0; w < w1; ++w) {
                const uint64_t x = MODE == 2 ? __ldcg(bm + w) : bm[w];
                nz += x != 0ull;
                pc += __popcll(x);
            }
            // one native 32-bit add per warp (a 64-bit add per thread was a
            // CAS spin on one word: half of the kernel's stall samples)
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) pc += __shfl_xor_sync(0xffffffffu, pc, d);
            if ((threadIdx.x & 31) == 0) atomicAdd(&s_cnt, pc);
            int tot;
            int r = s_nz + block_excl_scan<NT>(nz, tot, s_warp);
            if (a.oset || MODE == 2) {
                for (int64_t w = w0; w < w1; ++w) {
                    const uint64_t x = MODE == 2 ? __ldcg(bm + w) : bm[w];
                    if (x) {
                        if (a.oset) {
                            a.oset[sp + r] = (int32_t)(lo + w);
                            a.obits[sp + r] = x;
                            ++r;
                        }
                        if (MODE == 2) __stcg(bm + w, 0ull);
                    }
                }
            }
            __syncthreads();
            if (threadIdx.x == 0) s_nz += tot;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            a.counts[i] = (int64_t)s_cnt;
            if (a.msets) a.msets[i] = s_nz | (a.oset ? SETS_WRITTEN : 0);
        }
        __syncthreads();
    }
}

// Cut points of the windowed symbolic dense tier: for every A entry of a
// listed row, the offsets into its compressed B row (ascending sets) where
// each later window starts (window-major per row, so the dense kernel's
// entry lookups are coalesced).  A thread per entry gallops window to window.
__global__ void __launch_bounds__(256) k_sym_dense_cut(const int32_t *__restrict__ list, int64_t nb, SymArgs a,
                                                       int64_t wwords, int nwin,
                                                       const int64_t *__restrict__ eoff,
                                                       const int64_t *__restrict__ coff, int64_t cut_base,
                                                       int32_t *__restrict__ cut) {
    const int64_t e0 = eoff[0], tot = eoff[nb] - e0;
    for (int64_t x = (int64_t)blockIdx.x * 256 + threadIdx.x; x < tot; x += (int64_t)gridDim.x * 256) {
        int64_t lo = 0, hi = nb - 1;   // last row with eoff - e0 <= x
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (eoff[mid] - e0 <= x) lo = mid;
            else hi = mid - 1;
        }
        const int64_t li = lo;
        const int64_t e = x - (eoff[li] - e0);
        const int64_t alen = eoff[li + 1] - eoff[li];
        const int64_t gi = list[li] + a.a_row_off;
        int32_t *cr = cut + (coff[li] - cut_base) + e;
        int k = a.acol[a.arp[gi] + e];
        if (k < a.b_lo || k >= a.b_hi) {
            for (int w = 1; w < nwin; ++w) cr[(int64_t)(w - 1) * alen] = 0;
            continue;
        }
        k -= a.b_lo;
        const int64_t st = a.cbstart[k], en = st + a.cbcnt[k];
        int64_t cur = st;
        for (int w = 1; w < nwin; ++w) {
            const int64_t lw = (int64_t)w * wwords;
            int64_t step = 1, l2 = cur, h2 = cur;
            while (h2 < en && a.cbset[h2] < lw) {
                l2 = h2 + 1;
                h2 += step;
                step <<= 1;
            }
            int64_t r = h2 < en ? h2 : en;
            while (l2 < r) {
                const int64_t mid = (l2 + r) >> 1;
                if (a.cbset[mid] < lw) l2 = mid + 1;
                else r = mid;
            }
            cur = l2;
            cr[(int64_t)(w - 1) * alen] = (int32_t)(cur - st);
        }
    }
}

__global__ void k_alen(const int32_t *__restrict__ list, int64_t n, const int64_t *__restrict__ arp,
                       int64_t a_row_off, int mult, int32_t *__restrict__ ne, int64_t *__restrict__ nc) {
    for (int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; li < n; li += (int64_t)gridDim.x * blockDim.x) {
        const int64_t gi = list[li] + a_row_off;
        const int alen = (int)(arp[gi + 1] - arp[gi]);
        ne[li] = alen;
        nc[li] = (int64_t)alen * mult;
    }
}

// Thread tier, symbolic: one thread per row of A whose B rows are single
// entries (compressed row k = set k).  The row's sets are kept sorted: the
// largest set so far lives in registers (appends and hits on it are the
// common case for sorted A rows), the finished ones in a per-thread array
// (binary search + shift for an out-of-order set).  A entries are taken
// TSYM_BATCH at a time with all their loads issued together, so a row costs
// two dependent load rounds per batch instead of two per entry.
constexpr int TSYM_BATCH = 8;

template <int NT>
__global__ void __launch_bounds__(NT) k_sym_thread(const int32_t *__restrict__ list, int64_t nlist,
                                                   SymArgs a) {
    bin_range(a, list, nlist);
    for (int64_t li = (int64_t)blockIdx.x * NT + threadIdx.x; li < nlist; li += (int64_t)gridDim.x * NT) {
        const int64_t i = list[li];
        const int64_t gi = i + a.a_row_off;
        const int64_t a0 = a.arp[gi], a1 = a.arp[gi + 1];
        int key[THREAD_MAX_A];
        uint64_t msk[THREAD_MAX_A];
        int m = 0;             // finished sets in key/msk (all below lastk)
        int lastk = -1;        // largest set so far (-1: none)
        uint64_t lastm = 0;
#ifndef TSYM_VEC
#define TSYM_VEC 1
#endif
        // A's columns in 16-byte loads from the aligned position at or below
        // a0 (a thread reads its own row, so scalar loads cost one L1
        // wavefront per entry and warp); entries outside [a0, a1) masked
        const bool vec = TSYM_VEC && ((reinterpret_cast<uintptr_t>(a.acol) & 15) == 0);
        for (int64_t t0 = vec ? (a0 & ~(int64_t)3) : a0; t0 < a1; t0 += TSYM_BATCH) {
            int kk[TSYM_BATCH];
            if (vec) {
#pragma unroll
                for (int v = 0; v < TSYM_BATCH; v += 4) {
                    int4 c4;
                    if (t0 + v + 4 <= a1) {
                        c4 = __ldg(reinterpret_cast<const int4 *>(a.acol + t0 + v));
                    } else {
                        c4.x = t0 + v < a1 ? a.acol[t0 + v] : -1;
                        c4.y = t0 + v + 1 < a1 ? a.acol[t0 + v + 1] : -1;
                        c4.z = t0 + v + 2 < a1 ? a.acol[t0 + v + 2] : -1;
                        c4.w = -1;
                    }
                    kk[v] = c4.x;
                    kk[v + 1] = c4.y;
                    kk[v + 2] = c4.z;
                    kk[v + 3] = c4.w;
                }
#pragma unroll
                for (int u = 0; u < TSYM_BATCH; ++u) {
                    const int k = (t0 + u >= a0 && t0 + u < a1) ? kk[u] : -1;
                    kk[u] = (k >= a.b_lo && k < a.b_hi) ? k - a.b_lo : -1;
                }
            } else {
#pragma unroll
                for (int u = 0; u < TSYM_BATCH; ++u) {
                    int k = t0 + u < a1 ? a.acol[t0 + u] : -1;
                    kk[u] = (k >= a.b_lo && k < a.b_hi) ? k - a.b_lo : -1;
                }
            }
            int sv[TSYM_BATCH];
            uint64_t bv[TSYM_BATCH];
#pragma unroll
            for (int u = 0; u < TSYM_BATCH; ++u) {
                sv[u] = kk[u] >= 0 ? a.cbset[kk[u]] : -1;
                bv[u] = kk[u] >= 0 ? a.cbbits[kk[u]] : 0ull;
            }
#pragma unroll
            for (int u = 0; u < TSYM_BATCH; ++u) {
                const int sset = sv[u];
                if (sset < 0) continue;
                const uint64_t bits = bv[u];
                if (sset == lastk) {
                    lastm |= bits;
                } else if (sset > lastk) {
                    if (lastk >= 0) {
                        key[m] = lastk;
                        msk[m] = lastm;
                        ++m;
                    }
                    lastk = sset;
                    lastm = bits;
                } else {
                    int lo = 0, hi = m;   // first finished key >= sset (m: none)
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (key[mid] < sset) lo = mid + 1; else hi = mid;
                    }
                    if (lo < m && key[lo] == sset) {
                        msk[lo] |= bits;
                    } else {
                        for (int q = m; q > lo; --q) {
                            key[q] = key[q - 1];
                            msk[q] = msk[q - 1];
                        }
                        key[lo] = sset;
                        msk[lo] = bits;
                        ++m;
                    }
                }
            }
        }
        if (lastk >= 0) {
            key[m] = lastk;
            msk[m] = lastm;
            ++m;
        }
        const int64_t sp = a.sptr[i];
        int cnt = 0;
        for (int q = 0; q < m; ++q) {
            a.oset[sp + q] = key[q];
            a.obits[sp + q] = msk[q];
            cnt += __popcll(msk[q]);
        }
        a.counts[i] = cnt;
        if (a.msets) a.msets[i] = m | SETS_WRITTEN;
    }
}

// ======================================================================= K4 group tier

// Ordered accumulation of `prod` into vals[pos] (pos < 0: lane inactive).
// Lanes with equal pos combine in lane order, i.e. flattened product order:
// the leader adds its own product to the running value, then every peer's in
// turn -- exactly the reference's sequence of `payload += value`.
template <int G>
__device__ __forceinline__ void ordered_add(unsigned gm, double *vals, int pos, double prod) {
    const unsigned lane = lane_id();
    unsigned peers = __match_any_sync(gm, pos);
    bool leader = (pos >= 0) && ((int)lane == __ffs(peers) - 1);
    unsigned rest = leader ? (peers & ~(1u << lane)) : 0u;
    double acc = 0.0;
    if (leader) acc = __dadd_rn(vals[pos], prod);
    while (__any_sync(gm, rest != 0)) {
        int src = rest ? __ffs(rest) - 1 : (int)lane;
        double o = __shfl_sync(gm, prod, src);
        if (rest) {
            acc = __dadd_rn(acc, o);
            rest &= rest - 1;
        }
    }
    if (leader) vals[pos] = acc;
    __syncwarp(gm);
}

// One A entry's B-row batch for products_seq: the first BB_UF*G entries of
// the row, loaded together so their DRAM latencies overlap.
#ifndef TSG_BBUF8
#define TSG_BBUF8 4
#endif
template <int G>
__host__ __device__ constexpr int bb_uf() { return G < 8 ? 8 : (G == 8 ? TSG_BBUF8 : 4); }   // >= 32 entries per batch
template <int UF>
struct BBatchT {
    int c[UF];
    double v[UF];
};

template <int G>
using BBatch = BBatchT<bb_uf<G>()>;

template <int G>
__device__ __forceinline__ BBatch<G> bbatch_issue(unsigned gm, int glane, const NumArgs &a, int64_t st,
                                                  int len, int j, int cnt) {
    constexpr int BB_UF = bb_uf<G>();
    BBatch<G> b;
    const int jj = j < cnt ? j : 0;
    const int64_t sj = __shfl_sync(gm, st, jj, G);
    const int lj = j < cnt ? __shfl_sync(gm, len, jj, G) : 0;
#pragma unroll
    for (int u = 0; u < BB_UF; ++u) {
        const int q = u * G + glane;
        b.c[u] = q < lj ? a.bcol[sj + q] : 0;
        b.v[u] = q < lj ? a.bval[sj + q] : 0.0;
    }
    return b;
}

template <int G>
__device__ __forceinline__ void bbatch_accumulate(unsigned gm, int glane, const NumArgs &a, int64_t st,
                                                  int len, double av, int j, const BBatch<G> &b,
                                                  const int4 *tbl, int T, int logT, double *vals) {
    constexpr int BB_UF = bb_uf<G>();
    const int64_t sj = __shfl_sync(gm, st, j, G);
    const int lj = __shfl_sync(gm, len, j, G);
    const double aj = __shfl_sync(gm, av, j, G);
#pragma unroll
    for (int u = 0; u < BB_UF; ++u) {
        if (u * G + glane < lj) {
            const int c = b.c[u];
            const double prod = __dmul_rn(aj, b.v[u]);
            int4 e;
            tbl_find(tbl, T, logT, c >> 6, e);
            const int pos = e.w + mask_rank(e, c & 63);
            vals[pos] = __dadd_rn(vals[pos], prod);
        }
    }
    for (int q = BB_UF * G + glane; q < lj; q += G) {   // long B rows: remainder
        const int c = a.bcol[sj + q];
        const double prod = __dmul_rn(aj, a.bval[sj + q]);
        int4 e;
        tbl_find(tbl, T, logT, c >> 6, e);
        const int pos = e.w + mask_rank(e, c & 63);
        vals[pos] = __dadd_rn(vals[pos], prod);
    }
    __syncwarp(gm);
}

// Product phase, sequential mode (B rows at least ~G/2 long): A entries are
// taken one at a time in storage order and the G lanes split that entry's B
// row.  A B row has distinct columns, so lanes never collide within a step
// and a plain read-add-write replays the reference's order exactly; a
// __syncwarp separates consecutive A entries.  No search, no match.
template <int G>
__device__ __forceinline__ void products_seq(unsigned gm, int glane, const NumArgs &a, int64_t a0,
                                             int64_t a1, const int4 *tbl, int T, int logT,
                                             double *vals) {
    for (int64_t base = a0; base < a1; base += G) {
        int64_t t = base + glane;
        int64_t st = 0;
        int len = 0;
        double av = 0.0;
        if (t < a1) {
            int k = a.acol[t];
            if (k >= a.b_lo && k < a.b_hi) {
                k -= a.b_lo;
                st = a.brp[k];
                len = (int)(a.brp[k + 1] - st);
                av = a.aval[t];
            }
        }
        const int cnt = (int)((a1 - base) < G ? (a1 - base) : G);
        // Memory-level parallelism: the first UF*G entries of A entry j's B row
        // are loaded in one batch, and entry j+1's batch is issued before entry
        // j is accumulated, so a row costs ~1 DRAM round trip per A chunk
        // instead of one per (entry, G-slice).
        BBatch<G> bx = bbatch_issue<G>(gm, glane, a, st, len, 0, cnt);
        for (int j = 0; j < cnt; j += 2) {
            BBatch<G> by = bbatch_issue<G>(gm, glane, a, st, len, j + 1, cnt);
            bbatch_accumulate<G>(gm, glane, a, st, len, av, j, bx, tbl, T, logT, vals);
            bx = bbatch_issue<G>(gm, glane, a, st, len, j + 2, cnt);
            if (j + 1 < cnt)
                bbatch_accumulate<G>(gm, glane, a, st, len, av, j + 1, by, tbl, T, logT, vals);
        }
    }
}

// Product phase for unit B rows (every B row has <= 1 entry, e.g. the
// aggregation prolongator): lane j of a chunk owns A entry t = base + j and its
// single product.  UB chunks are loaded together -- the three dependent
// rounds (A column -> B row pointer -> B entry) are paid once per UB*G A
// entries -- then accumulated chunk by chunk in order with the ordered add.
template <int G>
__device__ __forceinline__ void products_unit(unsigned gm, int glane, const NumArgs &a, int64_t a0,
                                              int64_t a1, const int4 *tbl, int T, int logT,
                                              double *vals) {
    for (int64_t base = a0; base < a1; base += UB * G) {
        int kk[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) {
            const int64_t t = base + u * G + glane;
            kk[u] = t < a1 ? a.acol[t] : -1;
        }
        int64_t ss[UB];
        bool has[UB];
        if (a.unit_dense) {   // row_ptr is the identity: one dependent load round fewer
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const int k = kk[u];
                has[u] = k >= a.b_lo && k < a.b_hi;
                ss[u] = has[u] ? k - a.b_lo : 0;
            }
        } else {
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const int k = kk[u];
                const bool in = k >= a.b_lo && k < a.b_hi;
                ss[u] = in ? a.brp[k - a.b_lo] : 0;
                has[u] = in && a.brp[k - a.b_lo + 1] > ss[u];
            }
        }
        int cc[UB];
        double pp[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) {
            const int64_t t = base + u * G + glane;
            cc[u] = has[u] ? a.bcol[ss[u]] : 0;
            pp[u] = has[u] ? __dmul_rn(a.aval[t], a.bval[ss[u]]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < UB; ++u) {
            if (base + u * G >= a1) break;   // group-uniform
            int pos = -1;
            if (has[u]) {
                int4 e;
                tbl_find(tbl, T, logT, cc[u] >> 6, e);
                pos = e.w + mask_rank(e, cc[u] & 63);
            }
            ordered_add<G>(gm, vals, pos, pp[u]);
        }
    }
}

// Product phase for unit B rows when the host knows B is unit (uploaded or
// generated operands): the window of UB*G A entries first stages each
// product's output position and value in shared memory, then every lane
// folds, in storage order, the products whose position it owns (pos = glane
// mod G).  Same sequence of `payload += value` per position as ordered_add,
// without match / vote / shuffle rounds per chunk.
constexpr int UWIN_B = 12;   // staged bytes per product (int pos + double value)
#ifndef TSG_USKEW
#define TSG_USKEW 16
#endif
// bytes of one group's product stage, plus a 16-byte skew: at 192 B per
// 4-lane group, groups g and g + 2 of a half-warp read the same banks
// (measured, RA*P numeric: 0.183 -> 0.157 ms)
template <int G>
__host__ __device__ constexpr size_t ustage_bytes() { return (size_t)UB * G * UWIN_B + TSG_USKEW; }

template <int G>
__device__ __forceinline__ void products_unit_owned(unsigned gm, int glane, const NumArgs &a, int64_t a0,
                                                    int64_t a1, const int4 *tbl, int T, int logT,
                                                    double *vals, int *spos, double *sprod) {
    constexpr int W = UB * G;
    for (int64_t base = a0; base < a1; base += W) {
        int kk[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) {
            const int64_t t = base + u * G + glane;
            kk[u] = t < a1 ? a.acol[t] : -1;
        }
        int64_t ss[UB];
        bool has[UB];
        if (a.unit_dense) {
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const int k = kk[u];
                has[u] = k >= a.b_lo && k < a.b_hi;
                ss[u] = has[u] ? k - a.b_lo : 0;
            }
        } else {
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const int k = kk[u];
                const bool in = k >= a.b_lo && k < a.b_hi;
                ss[u] = in ? a.brp[k - a.b_lo] : 0;
                has[u] = in && a.brp[k - a.b_lo + 1] > ss[u];
            }
        }
        int cc[UB];
        double pp[UB];
#pragma unroll
        for (int u = 0; u < UB; ++u) {
            const int64_t t = base + u * G + glane;
            cc[u] = has[u] ? a.bcol[ss[u]] : 0;
            pp[u] = has[u] ? __dmul_rn(a.aval[t], a.bval[ss[u]]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < UB; ++u) {
            int pos = -1;
            if (has[u]) {
                int4 e;
                tbl_find(tbl, T, logT, cc[u] >> 6, e);
                pos = e.w + mask_rank(e, cc[u] & 63);
            }
            spos[u * G + glane] = pos;
            sprod[u * G + glane] = pp[u];
        }
        __syncwarp(gm);
        const int w = (int)((a1 - base) < W ? (a1 - base) : W);
        const int4 *sp4 = reinterpret_cast<const int4 *>(spos);
        for (int q = 0; q < ((w + 3) >> 2); ++q) {
            const int4 p4 = sp4[q];
            // owner test: non-negative and pos = glane (mod G)
            if (((p4.x ^ glane) & (int)(0x80000000u | (G - 1))) == 0)
                vals[p4.x] = __dadd_rn(vals[p4.x], sprod[4 * q]);
            if (((p4.y ^ glane) & (int)(0x80000000u | (G - 1))) == 0)
                vals[p4.y] = __dadd_rn(vals[p4.y], sprod[4 * q + 1]);
            if (((p4.z ^ glane) & (int)(0x80000000u | (G - 1))) == 0)
                vals[p4.z] = __dadd_rn(vals[p4.z], sprod[4 * q + 2]);
            if (((p4.w ^ glane) & (int)(0x80000000u | (G - 1))) == 0)
                vals[p4.w] = __dadd_rn(vals[p4.w], sprod[4 * q + 3]);
        }
        __syncwarp(gm);
    }
}

struct NumRowHdr {
    int64_t i = 0, cp = 0, a0 = 0, a1 = 0, sp = 0, sb = 0;
    int n = 0, mflag = 0;
};

__device__ __forceinline__ NumRowHdr num_row_hdr(const NumArgs &a, int64_t i) {
    NumRowHdr h;
    h.i = i;
    const int64_t gi = i + a.a_row_off;
    h.n = (int)a.counts[i];
    h.cp = a.cptr[i];
    h.a0 = a.arp[gi];
    h.a1 = a.arp[gi + 1];
    h.mflag = a.msets ? a.msets[i] : 0;
    h.sp = a.sptr ? a.sptr[i] : 0;
    h.sb = a.msets ? 0 : a.sbound[i];
    return h;
}


// bytes of the per-group value slices of a k_num_group block (with skew)
template <int G, int SLICE>
__host__ __device__ constexpr size_t num_slices_bytes(int gpb) {
    return (size_t)gpb * SLICE + (G <= 8 ? (size_t)gpb * 8 * G : 0);
}

// MODE 0: generic / unit B known on the device; 1: lane-split B rows (SEQ);
// 2: unit B known on the host (products_unit_owned, staging after the slices)
// Block size and minimum resident blocks of the numeric group kernels.  The
// two dominant config-2 instances are latency-bound, so occupancy is worth
// a few spilled registers (measured, R*A numeric: 256 threads at 80
// registers = 24 warps/SM 0.400 ms; 128 x 8 blocks at 64 registers = 32
// warps 0.370 ms).
#ifndef TSG_NUM8_BS
#define TSG_NUM8_BS 128
#endif
#ifndef TSG_NUM8_MINB
#define TSG_NUM8_MINB 8
#endif
#ifndef TSG_NUM4_BS
#define TSG_NUM4_BS 256
#endif
#ifndef TSG_NUM4_MINB
#define TSG_NUM4_MINB 4
#endif
template <int G, int MODE>
__host__ __device__ constexpr int num_bs() {
    return (G == 8 && MODE == 1) ? TSG_NUM8_BS : (G == 4 && MODE == 2) ? TSG_NUM4_BS : 256;
}
template <int G, int MODE>
__host__ __device__ constexpr int num_minb() {
    // the rest: the register budgets ptxas picks for a bare 256-thread bound
    return (G == 8 && MODE == 1) ? TSG_NUM8_MINB
           : (G == 4 && MODE == 2) ? TSG_NUM4_MINB
           : MODE == 1             ? 3
                                   : 4;
}

template <int G, int SLICE, int MODE>
__global__ void __launch_bounds__(num_bs<G, MODE>(), num_minb<G, MODE>()) k_num_group(const int32_t *__restrict__ list, int64_t nlist,
                                                   NumArgs a) {
    bin_range(a, list, nlist);
    extern __shared__ int4 smem[];
    const unsigned gm = group_mask<G>();
    const int glane = threadIdx.x & (G - 1);
    const unsigned lt = lanemask_lt();
    const int gpb = blockDim.x / G;
    // groups of <= 8 lanes: a half-warp 64-bit shared access spans 16 / G
    // groups whose equally aligned slices would put equal value positions
    // on one bank; group g starts g * 8G bytes later (8-lane groups: odd
    // groups 64 B = 16 banks after their even partner; 4-lane: 32 B steps)
    char *slice = reinterpret_cast<char *>(smem) + (size_t)(threadIdx.x / G) * SLICE +
                  (G <= 8 ? (size_t)(threadIdx.x / G) * 8 * G : 0);
    for (int pass_ = 0;; ++pass_) {
    const int32_t *lst_;
    int64_t nl_;
    if (!leftover_range(a, pass_, list, nlist, lst_, nl_)) break;
    for (int64_t li = (int64_t)blockIdx.x * gpb + threadIdx.x / G; li < nl_;
         li += (int64_t)gridDim.x * gpb) {
        const NumRowHdr h = num_row_hdr(a, lst_[li]);
        const int64_t i = h.i;
        const int64_t gi = i + a.a_row_off;
        const int n = h.n;
        const int64_t cp = h.cp;
        const int64_t a0 = h.a0, a1 = h.a1;
        const int mflag = h.mflag;
        const bool have_sets = a.sptr != nullptr && (mflag & SETS_WRITTEN);
        int64_t mest = a.msets ? (int64_t)(mflag & (SETS_WRITTEN - 1)) : (h.sb < n ? h.sb : n);
        double *vals = reinterpret_cast<double *>(slice);
        int2 *cbuf = reinterpret_cast<int2 *>(slice);   // phase-B scratch, aliases vals
        int4 *tbl = reinterpret_cast<int4 *>(slice + round16(8 * (int64_t)n));
        int T = table_slots(mest);
        const int tmax = (int)((SLICE - round16(8 * (int64_t)n)) / 16);
        if (T > tmax) T = 1 << ilog2_pow2(tmax);   // binning guarantees T <= tmax
        const int logT = ilog2_pow2(T);
        tbl_clear(tbl, T, glane, G);
        __syncwarp(gm);
        int64_t p0, p1;
        partial_range(a, i, p0, p1);
        const bool cap_mode = a.plen_out != nullptr;
        // in place: the partial row IS the output row, so columns are emitted
        // only after the partial values have been read (phase D)
        const bool inplace = cap_mode && a.pcol == a.ccol;
        int rowlen = n;
        bool ok = true;

        if (have_sets) {
            // sorted sets from the symbolic phase: base = running popcount
            const int m = (int)mest;
            const int64_t sp = h.sp;
            int carry = 0;
            for (int q0 = 0; q0 < m; q0 += G) {
                int q = q0 + glane;
                bool valid = q < m;
                int key = valid ? a.sset[sp + q] : 0;
                uint64_t bits = valid ? a.sbits[sp + q] : 0ull;
                int pc = __popcll(bits);
                int incl = group_incl_scan<G, int>(gm, pc, glane);
                int base = carry + incl - pc;
                carry += __shfl_sync(gm, incl, G - 1, G);
                if (valid) {
                    int slot = tbl_claim(tbl, T, logT, key);
                    if (slot < 0) {
                        ok = false;
                    } else {
                        tbl[slot].y = (int)(uint32_t)bits;
                        tbl[slot].z = (int)(uint32_t)(bits >> 32);
                        tbl[slot].w = base;
                    }
                    if (base + pc <= n) {
                        uint64_t b = bits;
                        int r = base;
                        while (b) {
                            a.ccol[cp + r++] = key * 64 + (__ffsll((long long)b) - 1);
                            b &= b - 1;
                        }
                    }
                }
            }
            ok = __all_sync(gm, ok);
            if (carry != n || !ok) {
                if (glane == 0) kerr(a.err, ok ? KERR_COUNT : KERR_PROBE, gi);
                __syncwarp(gm);
                continue;   // group-uniform
            }
        } else {
            // phase A: union of column sets (partial row + compressed B rows)
            for (int64_t q = p0 + glane; q < p1; q += G) {
                int c = a.pcol[q];
                int bit = c & 63;
                ok &= tbl_or(tbl, T, logT, c >> 6, bit < 32 ? 1u << bit : 0u,
                             bit >= 32 ? 1u << (bit - 32) : 0u);
            }
            group_enumerate_any<G>(
                gm, glane, a0, a1,
                [&](int64_t t, int64_t &st, int &len) {
                    int k = a.acol[t];
                    if (k >= a.b_lo && k < a.b_hi) {
                        k -= a.b_lo;
                        st = a.cbstart[k];
                        len = a.cbcnt[k];
                    }
                },
                [&](bool valid, int, int64_t, int64_t s) {
                    if (valid) {
                        uint64_t bits = a.cbbits[s];
                        ok &= tbl_or(tbl, T, logT, a.cbset[s], (unsigned)bits, (unsigned)(bits >> 32));
                    }
                });
            __syncwarp(gm);

            // phase B: compact the occupied sets (key, slot<<8 | popcount) into the
            // value area (m <= n entries of 8 B), rank each against the compacted
            // list -> base = columns in smaller sets; emit the row's columns.
            int m = 0, tot = 0;
            for (int r0 = 0; r0 < T; r0 += G) {
                int s = r0 + glane;
                int4 e = s < T ? tbl[s] : make_int4(TSG_EMPTY, 0, 0, 0);
                bool occ = e.x != TSG_EMPTY;
                unsigned bal = __ballot_sync(gm, occ) & gm;
                int pc = slot_pop(e);
                if (occ && m + __popc(bal & lt) < n) cbuf[m + __popc(bal & lt)] = make_int2(e.x, (s << 8) | pc);
                if (occ) tot += pc;
                m += __popc(bal);
            }
            tot = group_sum<G, int>(gm, tot);
            ok = __all_sync(gm, ok);
            if ((cap_mode ? tot > n : tot != n) || !ok || m > n) {
                if (glane == 0) kerr(a.err, ok ? KERR_COUNT : KERR_PROBE, gi);
                __syncwarp(gm);
                continue;   // group-uniform
            }
            rowlen = tot;
            __syncwarp(gm);
            for (int q = glane; q < m; q += G) {
                int2 me = cbuf[q];
                int base = 0;
                for (int u = 0; u < m; ++u) {
                    int2 o = cbuf[u];
                    if (o.x < me.x) base += o.y & 0xff;
                }
                int slot = me.y >> 8;
                tbl[slot].w = base;
                if (inplace) continue;
                int4 e = tbl[slot];
                unsigned lo = (unsigned)e.y, hi = (unsigned)e.z;
                int r = base;
                while (lo) {
                    int b = __ffs(lo) - 1;
                    lo &= lo - 1;
                    a.ccol[cp + r++] = me.x * 64 + b;
                }
                while (hi) {
                    int b = __ffs(hi) - 1;
                    hi &= hi - 1;
                    a.ccol[cp + r++] = me.x * 64 + 32 + b;
                }
            }

        }
        __syncwarp(gm);
        for (int q = glane; q < rowlen; q += G) vals[q] = -0.0;
        __syncwarp(gm);

        // phase C: partial values first, then products in A storage order
        for (int64_t q = p0 + glane; q < p1; q += G) {
            int c = a.pcol[q];
            int4 e;
            tbl_find(tbl, T, logT, c >> 6, e);
            vals[e.w + mask_rank(e, c & 63)] = a.pval[q];
        }
        __syncwarp(gm);
        if constexpr (MODE == 1) {
            products_seq<G>(gm, glane, a, a0, a1, tbl, T, logT, vals);
        } else if constexpr (MODE == 2) {
            char *stage = reinterpret_cast<char *>(smem) + num_slices_bytes<G, SLICE>(gpb) +
                          (size_t)(threadIdx.x / G) * ustage_bytes<G>();
            products_unit_owned<G>(gm, glane, a, a0, a1, tbl, T, logT, vals, reinterpret_cast<int *>(stage),
                                   reinterpret_cast<double *>(stage + UB * G * 4));
        } else if (a.unit_known > 0 || (a.unit_known < 0 && *a.unit_b)) {
            products_unit<G>(gm, glane, a, a0, a1, tbl, T, logT, vals);
        } else {
            group_enumerate<G>(
                gm, glane, a0, a1,
                [&](int64_t t, int64_t &st, int &len) {
                    int k = a.acol[t];
                    if (k >= a.b_lo && k < a.b_hi) {
                        k -= a.b_lo;
                        st = a.brp[k];
                        len = (int)(a.brp[k + 1] - st);
                    }
                },
                [&](bool valid, int j, int64_t t, int64_t s) {
                    int pos = -1;
                    double prod = 0.0;
                    if (valid) {
                        int c = a.bcol[s];
                        int4 e;
                        tbl_find(tbl, T, logT, c >> 6, e);
                        pos = e.w + mask_rank(e, c & 63);
                        prod = __dmul_rn(a.aval[t], a.bval[s]);
                    }
                    ordered_add<G>(gm, vals, pos, prod);
                });
        }
        __syncwarp(gm);
        if (inplace) {
            // phase D: the partial row has been consumed; emit merged columns
            for (int s = glane; s < T; s += G) {
                int4 e = tbl[s];
                if (e.x == TSG_EMPTY) continue;
                unsigned lo = (unsigned)e.y, hi = (unsigned)e.z;
                int r = e.w;
                while (lo) {
                    a.ccol[cp + r++] = e.x * 64 + (__ffs(lo) - 1);
                    lo &= lo - 1;
                }
                while (hi) {
                    a.ccol[cp + r++] = e.x * 64 + 32 + (__ffs(hi) - 1);
                    hi &= hi - 1;
                }
            }
        }
        for (int q = glane; q < rowlen; q += G) a.cval[cp + q] = vals[q];
        if (cap_mode && glane == 0) a.plen_out[i] = rowlen;
        __syncwarp(gm);
    }
    }
}

// Dense numeric tier: rows with sorted sets from the symbolic phase and a
// column count far beyond the group tier.  Every set of B gets a base (output
// offset of its first column in the row) and its mask in shared memory, so a
// product's slot is base[c >> 6] + popcount(mask below c) -- no hashing; the
// values accumulate with fp64 REDG adds straight into C (order-free, like the
// CTA / global tiers).
template <int NT>
__global__ void __launch_bounds__(NT) k_num_dense(const int32_t *__restrict__ list, int64_t nlist,
                                                  NumArgs a, int64_t nwords) {
    extern __shared__ int4 smem[];
    __shared__ int s_warp[32];
    uint64_t *mask = reinterpret_cast<uint64_t *>(smem);
    int32_t *base = reinterpret_cast<int32_t *>(mask + nwords);
    for (int64_t li = blockIdx.x; li < nlist; li += gridDim.x) {
        const int64_t i = list[li];
        const int64_t gi = i + a.a_row_off;
        const int64_t n = a.counts[i];
        const int64_t cp = a.cptr[i];
        const int m = a.msets[i] & (SETS_WRITTEN - 1);
        const int64_t sp = a.sptr[i];
        // bases of the row's sets (exclusive popcount scan in set order) and
        // the row's columns, values initialised to -0.0
        int carry = 0;
        for (int q0 = 0; q0 < m; q0 += NT) {
            const int q = q0 + threadIdx.x;
            int set = 0, pc = 0;
            uint64_t bits = 0;
            if (q < m) {
                set = a.sset[sp + q];
                bits = a.sbits[sp + q];
                pc = __popcll(bits);
            }
            int tot;
            const int b0 = carry + block_excl_scan<NT>(pc, tot, s_warp);
            if (q < m) {
                mask[set] = bits;
                base[set] = b0;
                uint64_t x = bits;
                int64_t r = cp + b0;
                while (x) {
                    a.ccol[r] = set * 64 + (__ffsll((long long)x) - 1);
                    a.cval[r++] = -0.0;
                    x &= x - 1;
                }
            }
            carry += tot;
        }
        if (carry != n) {
            if (threadIdx.x == 0) kerr(a.err, KERR_COUNT, gi);
            __syncthreads();
            continue;
        }
        __syncthreads();
        struct BV {
            int c;
            double v;
        };
        block_unit_enumerate<NT, DENSE_EB, DENSE_CH, BV>(
            a.arp[gi], a.arp[gi + 1],
            [&](int64_t t, int64_t &st, int &len, double &w) {
                int k = a.acol[t];
                if (k >= a.b_lo && k < a.b_hi) {
                    k -= a.b_lo;
                    st = a.brp[k];
                    len = (int)(a.brp[k + 1] - st);
                    w = a.aval[t];
                }
            },
            [&](int64_t s) { return BV{a.bcol[s], a.bval[s]}; },
            [&](double av, const BV &x) {
                const uint64_t mk = mask[x.c >> 6];
                const int bit = x.c & 63;
                const int pos = base[x.c >> 6] + __popcll(mk & ((1ull << bit) - 1ull));
                atomicAdd(&a.cval[cp + pos], __dmul_rn(av, x.v));
            },
            s_warp);
        __syncthreads();
    }
}

// Dense numeric tier, windowed (default).  The flattened REDG form above is
// bound by its enumeration (a ~10-step shared-memory search per product) and
// by fp64 atomics in L2 (R-MAT scale 18: 108 ms).  Here a row's sorted sets
// are cut into windows and every (row, window) pair is a work item taken from
// an atomic counter by persistent CTAs:
//   k_num_dense_prep  one CTA per row: window starts.  A window is a run of
//                     the row's sets with one block of DW_SETS column sets
//                     (so its (mask, base) map is direct-mapped in shared
//                     memory) and set bases in one block of W positions (so
//                     its values fit a W + 63 shared fp64 window)
//   k_num_dense_win   per item: the window's map in shared memory, its
//                     columns into C; a warp per A entry adds the entry's
//                     products into the shared window (CAS adds: neighbouring
//                     positions of one warp hit distinct banks, no L2
//                     atomics); one coalesced store of the values.  Rows of
//                     several windows cut every B row to the window's column
//                     range by binary search (the dense tier requires
//                     row-sorted B), so each product is read once.
// Hub rows thereby spread over all SMs instead of one CTA each.
// first s in [s0, s1) with col[s] >= c (col ascending)
__device__ __forceinline__ int64_t lower_col(const int32_t *__restrict__ col, int64_t s0, int64_t s1, int c) {
    while (s0 < s1) {
        const int64_t mid = (s0 + s1) >> 1;
        if (col[mid] < c) s0 = mid + 1;
        else s1 = mid;
    }
    return s0;
}

#ifndef PREP_NT
#define PREP_NT 256   // k_num_dense_prep block (R-MAT scale 20: 1024 -> 54.7 ms, 256 -> 47.7, 128 -> 48.8)
#endif
struct DenseWin {
    int W;        // positions per window block
    int sets;     // column sets (64-column words) per window block
    int maxw;     // window-start slots per row
};

template <int NT>
__global__ void __launch_bounds__(NT) k_num_dense_prep(const int32_t *__restrict__ list, int64_t nb, NumArgs a,
                                                       DenseWin dw, int32_t *__restrict__ nwin,
                                                       int2 *__restrict__ wst, int32_t *__restrict__ ncut_e,
                                                       int64_t *__restrict__ ncut) {
    __shared__ int s_warp[32];
    for (int64_t li = blockIdx.x; li < nb; li += gridDim.x) {
        const int64_t i = list[li];
        const int64_t n = a.counts[i];
        const int m = a.msets[i] & (SETS_WRITTEN - 1);
        const int64_t sp = a.sptr[i];
        int2 *ws = wst + li * dw.maxw;
        int carry = 0, nstart = 0;
        for (int q0 = 0; q0 < m; q0 += NT) {
            const int q = q0 + threadIdx.x;
            int set = 0, pc = 0;
            if (q < m) {
                set = a.sset[sp + q];
                pc = __popcll(a.sbits[sp + q]);
            }
            int tot;
            const int b = carry + block_excl_scan<NT>(pc, tot, s_warp);
            bool start = false;
            if (q < m) {
                if (q == 0) {
                    start = true;
                } else {
                    const int ps = a.sset[sp + q - 1];
                    const int pb = b - __popcll(a.sbits[sp + q - 1]);
                    start = ps / dw.sets != set / dw.sets || pb / dw.W != b / dw.W;
                }
            }
            __syncthreads();   // s_warp reuse
            int ns;
            const int r = nstart + block_excl_scan<NT>(start ? 1 : 0, ns, s_warp);
            if (start && r < dw.maxw) ws[r] = make_int2(q, b);
            nstart += ns;
            carry += tot;
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const bool ok = carry == n && nstart <= dw.maxw;
            if (!ok) kerr(a.err, KERR_COUNT, i + a.a_row_off);
            nwin[li] = ok ? nstart : 0;
            const int64_t gi = i + a.a_row_off;
            const int alen = (int)(a.arp[gi + 1] - a.arp[gi]);
            ncut_e[li] = ok && nstart > 1 ? alen : 0;
            ncut[li] = ok && nstart > 1 ? (int64_t)alen * (nstart - 1) : 0;
        }
        __syncthreads();
    }
}

// Cut points of multi-window rows: for every A entry of such a row, the
// offsets into its B row where each later window's columns start (window-major,
// coalesced for the window kernel).  A thread per entry gallops from one cut
// to the next; thousands of independent searches replace the dependent
// binary searches that stalled the window kernel's enumeration (18 ms of
// barrier waits at R-MAT scale 18).
__global__ void __launch_bounds__(256) k_num_dense_cut(const int32_t *__restrict__ list, int64_t nb, NumArgs a,
                                                       DenseWin dw, const int64_t *__restrict__ woff,
                                                       const int2 *__restrict__ wst,
                                                       const int64_t *__restrict__ eoff,
                                                       const int64_t *__restrict__ coff,
                                                       int32_t *__restrict__ cut) {
    const int64_t tot = eoff[nb];
    for (int64_t x = (int64_t)blockIdx.x * 256 + threadIdx.x; x < tot; x += (int64_t)gridDim.x * 256) {
        int64_t lo = 0, hi = nb - 1;   // last row with eoff <= x
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (eoff[mid] <= x) lo = mid;
            else hi = mid - 1;
        }
        const int64_t li = lo;
        const int e = (int)(x - eoff[li]);
        const int alen = (int)(eoff[li + 1] - eoff[li]);
        const int nw = (int)(woff[li + 1] - woff[li]);
        const int64_t i = list[li];
        const int64_t gi = i + a.a_row_off;
        const int64_t sp = a.sptr[i];
        int32_t *cr = cut + coff[li] + e;
        int k = a.acol[a.arp[gi] + e];
        if (k < a.b_lo || k >= a.b_hi) {
            for (int j = 1; j < nw; ++j) cr[(int64_t)(j - 1) * alen] = 0;
            continue;
        }
        k -= a.b_lo;
        const int64_t b0 = a.brp[k], b1 = a.brp[k + 1];
        int64_t cur = b0;
        for (int j = 1; j < nw; ++j) {
            const int c = a.sset[sp + wst[li * dw.maxw + j].x] * 64;
            // gallop: first s >= cur with col[s] >= c
            int64_t step = 1, lo2 = cur, hi2 = cur;
            while (hi2 < b1 && a.bcol[hi2] < c) {
                lo2 = hi2 + 1;
                hi2 += step;
                step <<= 1;
            }
            cur = lower_col(a.bcol, lo2, hi2 < b1 ? hi2 : b1, c);
            cr[(int64_t)(j - 1) * alen] = (int32_t)(cur - b0);
        }
    }
}

template <int NT>
__global__ void __launch_bounds__(NT) k_num_dense_win(const int32_t *__restrict__ list, int64_t nb, NumArgs a,
                                                      DenseWin dw, const int64_t *__restrict__ woff,
                                                      const int2 *__restrict__ wst,
                                                      const int64_t *__restrict__ coff,
                                                      const int32_t *__restrict__ cut,
                                                      unsigned long long *__restrict__ counter) {
    extern __shared__ int4 smem[];
    uint64_t *smask = reinterpret_cast<uint64_t *>(smem);
    int32_t *sbase = reinterpret_cast<int32_t *>(smask + dw.sets);
    double *acc = reinterpret_cast<double *>(sbase + dw.sets + (dw.sets & 1));
    __shared__ int64_t s_item;
    __shared__ int s_warp[32];
    const int64_t total = woff[nb];
    for (;;) {
        if (threadIdx.x == 0) s_item = (int64_t)atomicAdd(counter, 1ull);
        __syncthreads();
        const int64_t x = s_item;
        if (x >= total) break;
        int64_t lo = 0, hi = nb - 1;   // last row with woff <= x
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (woff[mid] <= x) lo = mid;
            else hi = mid - 1;
        }
        const int64_t li = lo;
        const int nw = (int)(woff[li + 1] - woff[li]);
        const int j = (int)(x - woff[li]);
        const int64_t i = list[li];
        const int64_t gi = i + a.a_row_off;
        const int64_t cp = a.cptr[i];
        const int64_t sp = a.sptr[i];
        const int2 w0 = wst[li * dw.maxw + j];
        int2 w1;
        if (j + 1 < nw) w1 = wst[li * dw.maxw + j + 1];
        else w1 = make_int2(a.msets[i] & (SETS_WRITTEN - 1), (int)a.counts[i]);
        const int P0 = w0.y, len = w1.y - w0.y;
        const int blk = a.sset[sp + w0.x] / dw.sets * dw.sets;
        // the window's (mask, base) map and columns
        int carry = P0;
        for (int q0 = w0.x; q0 < w1.x; q0 += NT) {
            const int q = q0 + threadIdx.x;
            int set = 0, pc = 0;
            uint64_t bits = 0;
            if (q < w1.x) {
                set = a.sset[sp + q];
                bits = a.sbits[sp + q];
                pc = __popcll(bits);
            }
            int tot;
            const int b = carry + block_excl_scan<NT>(pc, tot, s_warp);
            if (q < w1.x) {
                smask[set - blk] = bits;
                sbase[set - blk] = b - P0;
                uint64_t y = bits;
                int64_t r = cp + b;
                while (y) {
                    a.ccol[r++] = set * 64 + (__ffsll((long long)y) - 1);
                    y &= y - 1;
                }
            }
            carry += tot;
            __syncthreads();
        }
        for (int q = threadIdx.x; q < len; q += NT) acc[q] = -0.0;
        __syncthreads();
        const int64_t a0 = a.arp[gi], a1 = a.arp[gi + 1];
        // products in units of DENSE_CH of one B row (block_unit_enumerate)
        struct BV {
            int c;
            double v;
        };
        block_unit_enumerate<NT, DENSE_EB, DENSE_CH_NUM, BV>(
            a0, a1,
            [&](int64_t t, int64_t &st, int &ln, double &w) {
                int k = a.acol[t];
                if (k >= a.b_lo && k < a.b_hi) {
                    k -= a.b_lo;
                    int64_t s0 = a.brp[k], s1 = a.brp[k + 1];
                    if (nw > 1) {
                        const int64_t e = t - a0;
                        const int32_t *cr = cut + coff[li] + e;
                        const int64_t bb = s0;
                        if (j > 0) s0 = bb + cr[(int64_t)(j - 1) * (a1 - a0)];
                        if (j + 1 < nw) s1 = bb + cr[(int64_t)j * (a1 - a0)];
                    }
                    st = s0;
                    ln = (int)(s1 - s0);
                    w = a.aval[t];
                }
            },
            [&](int64_t s) { return BV{a.bcol[s], a.bval[s]}; },
            [&](double av, const BV &x) {
                const int w = (x.c >> 6) - blk;
                const int bit = x.c & 63;
                const int pos = sbase[w] + __popcll(smask[w] & ((1ull << bit) - 1ull));
                atomicAdd(&acc[pos], __dmul_rn(av, x.v));
            },
            s_warp);
        __syncthreads();
        for (int q = threadIdx.x; q < len; q += NT) a.cval[cp + P0 + q] = acc[q];
        __syncthreads();
    }
}

// ======================================================================= CTA / global tiers

// Union of the row's sets into tbl (generic pointer: smem or global slab).
template <int NT>
__device__ __forceinline__ bool block_union(int4 *tbl, int T, int logT, int64_t p0, int64_t p1,
                                            const int32_t *pcol, int64_t a0,
                                            int64_t a1, const int32_t *acol, int32_t b_lo,
                                            int32_t b_hi, const int64_t *cbstart,
                                            const int32_t *cbcnt, const int32_t *cbset,
                                            const uint64_t *cbbits) {
    bool ok = true;
    {
        for (int64_t q = p0 + threadIdx.x; q < p1; q += NT) {
            int c = pcol[q];
            int bit = c & 63;
            ok &= tbl_or(tbl, T, logT, c >> 6, bit < 32 ? 1u << bit : 0u,
                         bit >= 32 ? 1u << (bit - 32) : 0u);
        }
    }
    block_enumerate<NT>(
        a0, a1,
        [&](int64_t t, int64_t &st, int &len) {
            int k = acol[t];
            if (k >= b_lo && k < b_hi) {
                k -= b_lo;
                st = cbstart[k];
                len = cbcnt[k];
            }
        },
        [&](int64_t, int64_t s) {
            uint64_t bits = cbbits[s];
            ok &= tbl_or(tbl, T, logT, cbset[s], (unsigned)bits, (unsigned)(bits >> 32));
        });
    return ok;
}

template <int NT, bool GLOBAL>
__global__ void __launch_bounds__(NT) k_sym_block(const int32_t *__restrict__ list, int64_t nlist,
                                                  SymArgs a, int4 *slab, int64_t slab_slots,
                                                  int tmax) {
    extern __shared__ int4 smem[];
    __shared__ int s_warp[32];
    __shared__ int s_red[2];
    int4 *tbl = GLOBAL ? slab + (int64_t)blockIdx.x * slab_slots : smem;
    for (int64_t li = blockIdx.x; li < nlist; li += gridDim.x) {
        const int64_t i = list[li];
        const int64_t gi = i + a.a_row_off;
        int64_t want = table_slots(a.sbound[i]);
        int T = (int)(want < tmax ? want : tmax);
        const int logT = ilog2_pow2(T);
        tbl_clear(tbl, T, threadIdx.x, NT);
        if (threadIdx.x < 2) s_red[threadIdx.x] = 0;
        __syncthreads();
        const int64_t sp0 = a.prp ? a.prp[i] : 0, sp1 = a.prp ? a.prp[i + 1] : 0;
        bool ok = block_union<NT>(tbl, T, logT, sp0, sp1, a.pcol, a.arp[gi], a.arp[gi + 1], a.acol,
                                  a.b_lo, a.b_hi, a.cbstart, a.cbcnt, a.cbset, a.cbbits);
        __syncthreads();
        int cnt = 0, m = 0;
        for (int s = threadIdx.x; s < T; s += NT) {
            int4 e = tbl[s];
            if (e.x != TSG_EMPTY) {
                m++;
                cnt += slot_pop(e);
            }
        }
        int tc, tm;
        (void)block_excl_scan<NT>(cnt, tc, s_warp);
        (void)block_excl_scan<NT>(m, tm, s_warp);
        if (!ok) kerr(a.err, KERR_PROBE, gi);
        if (threadIdx.x == 0) {
            a.counts[i] = tc;
            if (a.msets) a.msets[i] = tm;
        }
        __syncthreads();
    }
}

// Numeric CTA/global tier: union -> compact + bitonic sort of set keys ->
// scan of popcounts -> columns; values accumulate straight into C with fp64
// REDG adds (C values pre-set to -0.0, the additive identity that keeps the
// sign of a lone -0.0 product).
template <int NT, bool GLOBAL>
__global__ void __launch_bounds__(NT) k_num_block(const int32_t *__restrict__ list, int64_t nlist,
                                                  NumArgs a, int4 *slab, uint64_t *sortslab,
                                                  int64_t slab_slots, int tmax) {
    extern __shared__ int4 smem[];
    __shared__ int s_warp[32];
    __shared__ int s_m;
    int4 *tbl = GLOBAL ? slab + (int64_t)blockIdx.x * slab_slots : smem;
    uint64_t *keys = GLOBAL ? sortslab + (int64_t)blockIdx.x * slab_slots
                            : reinterpret_cast<uint64_t *>(smem + tmax);
    for (int64_t li = blockIdx.x; li < nlist; li += gridDim.x) {
        const int64_t i = list[li];
        const int64_t gi = i + a.a_row_off;
        const int64_t n = a.counts[i];
        const int64_t cp = a.cptr[i];
        int64_t mest = a.msets ? (int64_t)(a.msets[i] & (SETS_WRITTEN - 1)) : (a.sbound[i] < n ? a.sbound[i] : n);
        int64_t want = table_slots(mest);
        int T = (int)(want < tmax ? want : tmax);
        const int logT = ilog2_pow2(T);
        tbl_clear(tbl, T, threadIdx.x, NT);
        if (threadIdx.x == 0) s_m = 0;
        __syncthreads();
        int64_t p0, p1;
        partial_range(a, i, p0, p1);
        bool ok = block_union<NT>(tbl, T, logT, p0, p1, a.pcol, a.arp[gi], a.arp[gi + 1], a.acol,
                                  a.b_lo, a.b_hi, a.cbstart, a.cbcnt, a.cbset, a.cbbits);
        __syncthreads();
        // compact occupied slots as sortable (key << 32 | slot)
        for (int s = threadIdx.x; s < T; s += NT) {
            int4 e = tbl[s];
            if (e.x != TSG_EMPTY) {
                int p = atomicAdd(&s_m, 1);
                keys[p] = ((uint64_t)(uint32_t)e.x << 32) | (uint32_t)s;
            }
        }
        __syncthreads();
        const int m = s_m;
        int P = 1;
        while (P < m) P <<= 1;
        for (int s = m + threadIdx.x; s < P; s += NT) keys[s] = ~0ull;
        __syncthreads();
        // bitonic sort of P keys
        for (int k = 2; k <= P; k <<= 1) {
            for (int j = k >> 1; j > 0; j >>= 1) {
                for (int x = threadIdx.x; x < P; x += NT) {
                    int y = x ^ j;
                    if (y > x) {
                        uint64_t kx = keys[x], ky = keys[y];
                        bool up = (x & k) == 0;
                        if ((kx > ky) == up) {
                            keys[x] = ky;
                            keys[y] = kx;
                        }
                    }
                }
                __syncthreads();
            }
        }
        // exclusive scan of popcounts in key order -> base; emit columns
        int carry = 0;
        for (int b0 = 0; b0 < m; b0 += NT) {
            int x = b0 + threadIdx.x;
            int slot = -1, pc = 0;
            int4 e = make_int4(0, 0, 0, 0);
            if (x < m) {
                slot = (int)(uint32_t)keys[x];
                e = tbl[slot];
                pc = slot_pop(e);
            }
            int tot;
            int base = carry + block_excl_scan<NT>(pc, tot, s_warp);
            if (x < m) {
                tbl[slot].w = base;
                if (base + pc <= n) {
                    unsigned lo = (unsigned)e.y, hi = (unsigned)e.z;
                    int64_t r = cp + base;
                    while (lo) {
                        int b = __ffs(lo) - 1;
                        lo &= lo - 1;
                        a.ccol[r] = e.x * 64 + b;
                        a.cval[r++] = -0.0;
                    }
                    while (hi) {
                        int b = __ffs(hi) - 1;
                        hi &= hi - 1;
                        a.ccol[r] = e.x * 64 + 32 + b;
                        a.cval[r++] = -0.0;
                    }
                }
            }
            carry += tot;
        }
        ok = __syncthreads_and(ok);
        if ((a.plen_out ? carry > n : carry != n) || !ok) {
            if (threadIdx.x == 0) kerr(a.err, ok ? KERR_COUNT : KERR_PROBE, gi);
            __syncthreads();
            continue;
        }
        if (a.plen_out && threadIdx.x == 0) a.plen_out[i] = carry;
        // partial values, then products (order-free REDG adds)
        if (p1 > p0) {
            for (int64_t q = p0 + threadIdx.x; q < p1; q += NT) {
                int c = a.pcol[q];
                int4 e;
                tbl_find(tbl, T, logT, c >> 6, e);
                a.cval[cp + e.w + mask_rank(e, c & 63)] = a.pval[q];
            }
            __syncthreads();
        }
        block_enumerate<NT>(
            a.arp[gi], a.arp[gi + 1],
            [&](int64_t t, int64_t &st, int &len) {
                int k = a.acol[t];
                if (k >= a.b_lo && k < a.b_hi) {
                    k -= a.b_lo;
                    st = a.brp[k];
                    len = (int)(a.brp[k + 1] - st);
                }
            },
            [&](int64_t t, int64_t s) {
                int c = a.bcol[s];
                int4 e;
                tbl_find(tbl, T, logT, c >> 6, e);
                atomicAdd(&a.cval[cp + e.w + mask_rank(e, c & 63)], __dmul_rn(a.aval[t], a.bval[s]));
            });
        __syncthreads();
    }
}

// ======================================================================= host helpers

using Bins = ::BinLists<NBINS>;

template <typename K>
int set_smem(K kernel, size_t bytes) {
    return tsg_func_smem((const void *)kernel, bytes);
}

unsigned group_grid(tsg_ctx *c, int64_t nrows, int groups_per_block) {
    return grid_for(nrows, groups_per_block, c->num_sms * 64);
}

// Device-driven bins: a bin's size is unknown to the host, so its kernel is
// launched with one resident wave (grid-stride loops cover any size) and
// takes its rows from the partition's device-side bin starts.
template <class K>
unsigned resident_grid(tsg_ctx *c, K kernel, int bs, size_t smem) {
    static std::mutex mu;
    static std::map<std::pair<const void *, size_t>, int> cache;
    const auto key = std::make_pair((const void *)kernel, smem);
    std::lock_guard<std::mutex> g(mu);
    auto it = cache.find(key);
    int nb;
    if (it != cache.end()) {
        nb = it->second;
    } else {
        nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, bs, smem) != cudaSuccess) {
            cudaGetLastError();
            nb = 1;
        }
        if (nb < 1) nb = 1;
        cache[key] = nb;
    }
    return (unsigned)(nb * c->num_sms);
}

// The rows of bin B for a launch: (list, n) from the host offsets, or -- in
// device-driven mode -- the whole list with the bin id in the kernel
// arguments (bin_range) and n = an upper bound for grid sizing.  False:
// nothing to launch (empty, or impossible by the host's bounds).
template <class Args>
bool bin_select(const Bins &bl, int B, Args &a, const int32_t *&list, int64_t &n) {
    if (bl.device) {
        if (!((bl.possible >> B) & 1u)) return false;
        // only bins the last same-shape call filled get their own launch,
        // sized by that call's count (a hint: the kernel covers whatever the
        // device partition holds); the others go to the leftover launch
        const int64_t h = bl.hint[B + 1] - bl.hint[B];
        if (h <= 0) return false;
        a.dbins = bl.dstart;
        a.bin = B;
        list = bl.list;
        n = h < bl.rows ? h : bl.rows;
        return true;
    }
    n = bl.off[B + 1] - bl.off[B];
    if (n <= 0) return false;
    a.dbins = nullptr;
    list = bl.list + bl.off[B];
    return true;
}

template <class K>
unsigned bin_grid(tsg_ctx *c, const Bins &bl, unsigned grid, K kernel, int bs, size_t smem) {
    (void)c; (void)bl; (void)kernel; (void)bs; (void)smem;
    return grid;
}

// global-tier slab sizing: T slots per CTA, bounded by a memory budget
constexpr int64_t GLOBAL_SLAB_BUDGET = (int64_t)2 << 30;

template <int B>
int launch_sym_group(tsg_ctx *c, const Bins &bl, const SymArgs &a0) {
    constexpr int G = gt_g_sym(B), SL = gt_slice(B), BS = gt_block(B);
    SymArgs a = a0;
    const int32_t *lst;
    int64_t n;
    if (!bin_select(bl, B, a, lst, n)) return TSG_OK;
    size_t smem = (size_t)(BS / G) * SL;
    TSG_TRY(set_smem(k_sym_group<G, SL>, smem));
    unsigned grid = bin_grid(c, bl, group_grid(c, n, BS / G), k_sym_group<G, SL>, BS, smem);
    k_sym_group<G, SL><<<grid, BS, smem, c->stream>>>(lst, n, a); ++c->launches;
    TSG_TRY(tsg_launch_check("k_sym_group", B, grid, BS, smem));
    return TSG_OK;
}

template <int B, int MODE>
int launch_num_group_m(tsg_ctx *c, const Bins &bl, const NumArgs &a0) {
    // unit-B rows (owner-folded products) of the two smallest bins: 4 lanes
    // per row, twice the rows in flight (measured: RA*P 241 -> 182 us; the
    // lane-split SEQ mode stays at 8 lanes, where 4 was slower)
    constexpr int G = (MODE == 2 && B <= 1) ? 4 : gt_g(B), SL = gt_slice(B);
    constexpr int BS = num_bs<G, MODE>() < gt_block(B) ? num_bs<G, MODE>() : gt_block(B);
    NumArgs a = a0;
    const int32_t *lst;
    int64_t n;
    if (!bin_select(bl, B, a, lst, n)) return TSG_OK;
    size_t smem = num_slices_bytes<G, SL>(BS / G) + (MODE == 2 ? (size_t)(BS / G) * ustage_bytes<G>() : 0);
    TSG_TRY(set_smem(k_num_group<G, SL, MODE>, smem));
    unsigned grid = bin_grid(c, bl, group_grid(c, n, BS / G), k_num_group<G, SL, MODE>, BS, smem);
    k_num_group<G, SL, MODE><<<grid, BS, smem, c->stream>>>(lst, n, a); ++c->launches;
    TSG_TRY(tsg_launch_check("k_num_group", B, grid, BS, smem));
    return TSG_OK;
}

template <int B>
int launch_num_group(tsg_ctx *c, const Bins &bl, const NumArgs &a) {
    if (bl.device ? !((bl.possible >> B) & 1u) || bl.hint[B + 1] - bl.hint[B] <= 0
                  : bl.off[B + 1] - bl.off[B] <= 0)
        return TSG_OK;
    // lane-per-B-entry mode pays off once B rows fill at least half a group
    if (a.seq >= gt_g(B) / 2) return launch_num_group_m<B, 1>(c, bl, a);
    if (a.unit_known > 0) return launch_num_group_m<B, 2>(c, bl, a);
    return launch_num_group_m<B, 0>(c, bl, a);
}

template <int CB>
int launch_sym_cta(tsg_ctx *c, const Bins &bl, const SymArgs &a) {
    if (bl.device) return TSG_OK;   // excluded by the host's bounds (device_bins_ok)
    constexpr int NT = ct_nt(CB), TS = ct_slots(CB);
    const int B = 7 + CB;
    int64_t n = bl.off[B + 1] - bl.off[B];
    if (n <= 0) return TSG_OK;
    size_t smem = (size_t)TS * 16;
    TSG_TRY(set_smem(k_sym_block<NT, false>, smem));
    k_sym_block<NT, false><<<grid_for(n, 1, c->num_sms * 8), NT, smem, c->stream>>>(
        bl.list + bl.off[B], n, a, nullptr, 0, TS); ++c->launches;
    TSG_CK(cudaGetLastError());
    return TSG_OK;
}

template <int CB>
int launch_num_cta(tsg_ctx *c, const Bins &bl, const NumArgs &a) {
    if (bl.device) return TSG_OK;   // excluded by the host's bounds (device_bins_ok)
    constexpr int NT = ct_nt(CB), TS = ct_slots(CB);
    const int B = 7 + CB;
    int64_t n = bl.off[B + 1] - bl.off[B];
    if (n <= 0) return TSG_OK;
    size_t smem = (size_t)TS * 24;
    TSG_TRY(set_smem(k_num_block<NT, false>, smem));
    k_num_block<NT, false><<<grid_for(n, 1, c->num_sms * 8), NT, smem, c->stream>>>(
        bl.list + bl.off[B], n, a, nullptr, nullptr, 0, TS); ++c->launches;
    TSG_CK(cudaGetLastError());
    return TSG_OK;
}

__global__ void k_max_i64_list(const int32_t *list, int64_t n, const int64_t *v,
                               unsigned long long *out) {
    unsigned long long m = 0;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long y = (unsigned long long)v[list[x]];
        m = y > m ? y : m;
    }
    for (int d = 16; d >= 1; d >>= 1) {
        unsigned long long o = __shfl_xor_sync(0xffffffffu, m, d);
        m = o > m ? o : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// max over listed rows of v[] (host value)
int list_max(tsg_ctx *c, const int32_t *list, int64_t n, const int64_t *v, int64_t &out) {
    TSG_TRY(tsg_fill(c, c->d_small, 0, sizeof(int64_t), c->stream));
    k_max_i64_list<<<grid_for(n, 256, c->num_sms * 4), 256, 0, c->stream>>>(
        list, n, v, (unsigned long long *)c->d_small); ++c->launches;
    TSG_TRY(tsg_put_small(c, c->d_small, 1, 0));
    TSG_CK(cudaStreamSynchronize(c->stream));
    out = c->h_small[0];
    return TSG_OK;
}

// Global tier rows split into classes of table size (<= 2^15, 2^17, 2^19,
// 2^21 slots, above) before launching: the slab budget per launch then bounds
// the CTAs by the class's own largest table instead of the bin's largest row
// (one 4 M-column hub row used to leave ~10 CTAs for all of an R-MAT scale-22
// bin's rows).  One small read-back of the class sizes replaces the max.
constexpr int GCLASSES = 5;
__host__ __device__ __forceinline__ int gclass_of(int64_t T) {
    int k = 0;
    while (k < GCLASSES - 1 && T > ((int64_t)1 << (15 + 2 * k))) ++k;
    return k;
}

__global__ void k_gclass_count(const int32_t *__restrict__ list, int64_t n, const int64_t *__restrict__ v,
                               unsigned long long *cnt) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[gclass_of(table_slots(v[list[x]]))], 1ull);
}

__global__ void k_gclass_scatter(const int32_t *__restrict__ list, int64_t n, const int64_t *__restrict__ v,
                                 unsigned long long *cursor, int32_t *__restrict__ out) {
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = list[x];
        out[atomicAdd(&cursor[gclass_of(table_slots(v[r]))], 1ull)] = r;
    }
}

// rows of `list` regrouped by class (out: n entries, off: GCLASSES + 1 starts)
static int global_classes(tsg_ctx *c, const int32_t *list, int64_t n, const int64_t *v, int32_t **out,
                          int64_t off[GCLASSES + 1]) {
    unsigned long long *cnt = reinterpret_cast<unsigned long long *>(c->d_small + 24);
    TSG_TRY(tsg_fill(c, cnt, 0, GCLASSES * sizeof(unsigned long long), c->stream));
    k_gclass_count<<<grid_for(n, 256, c->num_sms * 4), 256, 0, c->stream>>>(list, n, v, cnt); ++c->launches;
    TSG_TRY(tsg_put_small(c, reinterpret_cast<const int64_t *>(cnt), GCLASSES, 2));
    TSG_CK(cudaStreamSynchronize(c->stream));
    off[0] = 0;
    for (int k = 0; k < GCLASSES; ++k) off[k + 1] = off[k] + c->h_small[2 + k];
    TSG_TRY(tsg_alloc_t(c, out, n));
    unsigned long long *cur = reinterpret_cast<unsigned long long *>(c->d_small + 24);
    unsigned long long h[GCLASSES];
    for (int k = 0; k < GCLASSES; ++k) h[k] = (unsigned long long)off[k];
    TSG_CK(cudaMemcpyAsync(cur, h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
    k_gclass_scatter<<<grid_for(n, 256, c->num_sms * 4), 256, 0, c->stream>>>(list, n, v, cur, *out);
    ++c->launches;
    TSG_CK(cudaStreamSynchronize(c->stream));   // `h` is pageable host memory
    return TSG_OK;
}

// arena block released when the scope ends (stream-ordered, so after the
// kernels queued in the scope), on error returns too
struct ArenaGuard {
    tsg_ctx *c;
    void *p;
    ~ArenaGuard() { tsg_free(c, p); }
};

int launch_sym_global(tsg_ctx *c, const Bins &bl, const SymArgs &a) {
    if (bl.device) return TSG_OK;   // excluded by the host's bounds (device_bins_ok)
    const int B = BIN_GLOBAL;
    int64_t n = bl.off[B + 1] - bl.off[B];
    if (n <= 0) return TSG_OK;
    int32_t *cl = nullptr;
    int64_t off[GCLASSES + 1];
    TSG_TRY(global_classes(c, bl.list + bl.off[B], n, a.sbound, &cl, off));
    ArenaGuard cl_guard{c, cl};
    for (int k = GCLASSES - 1; k >= 0; --k) {
        const int64_t nk = off[k + 1] - off[k];
        if (nk <= 0) continue;
        int64_t maxb = 0;
        TSG_TRY(list_max(c, cl + off[k], nk, a.sbound, maxb));
        int64_t T = table_slots(maxb);
        if (T > (1ll << 30)) {
            tsg_set_error("row accumulator of %lld slots exceeds the global tier", (long long)T);
            return TSG_ECAPACITY;
        }
        int64_t ctas = GLOBAL_SLAB_BUDGET / (T * 16);
        if (ctas < 1) ctas = 1;
        if (ctas > nk) ctas = nk;
        if (ctas > 2 * c->num_sms) ctas = 2 * c->num_sms;
        int4 *slab = nullptr;
        TSG_TRY(tsg_alloc_t(c, &slab, (size_t)(ctas * T)));
        k_sym_block<512, true><<<(unsigned)ctas, 512, 0, c->stream>>>(cl + off[k], nk, a, slab, T, (int)T);
        ++c->launches;
        TSG_CK(cudaGetLastError());
        TSG_TRY(tsg_free(c, slab));
    }
    return TSG_OK;
}

int launch_num_global(tsg_ctx *c, const Bins &bl, const NumArgs &a) {
    if (bl.device) return TSG_OK;   // excluded by the host's bounds (device_bins_ok)
    const int B = BIN_GLOBAL;
    int64_t n = bl.off[B + 1] - bl.off[B];
    if (n <= 0) return TSG_OK;
    // distinct sets <= columns: classes (and slabs) by the rows' counts
    int32_t *cl = nullptr;
    int64_t off[GCLASSES + 1];
    TSG_TRY(global_classes(c, bl.list + bl.off[B], n, a.counts, &cl, off));
    ArenaGuard cl_guard{c, cl};
    for (int k = GCLASSES - 1; k >= 0; --k) {
        const int64_t nk = off[k + 1] - off[k];
        if (nk <= 0) continue;
        int64_t maxm = 0;
        TSG_TRY(list_max(c, cl + off[k], nk, a.counts, maxm));
        int64_t T = table_slots(maxm);
        if (T > (1ll << 30)) {
            tsg_set_error("row accumulator of %lld slots exceeds the global tier", (long long)T);
            return TSG_ECAPACITY;
        }
        int64_t ctas = GLOBAL_SLAB_BUDGET / (T * 24);
        if (ctas < 1) ctas = 1;
        if (ctas > nk) ctas = nk;
        if (ctas > 2 * c->num_sms) ctas = 2 * c->num_sms;
        int4 *slab = nullptr;
        uint64_t *sortslab = nullptr;
        TSG_TRY(tsg_alloc_t(c, &slab, (size_t)(ctas * T)));
        TSG_TRY(tsg_alloc_t(c, &sortslab, (size_t)(ctas * T)));
        k_num_block<512, true><<<(unsigned)ctas, 512, 0, c->stream>>>(cl + off[k], nk, a, slab, sortslab, T,
                                                                       (int)T);
        ++c->launches;
        TSG_CK(cudaGetLastError());
        TSG_TRY(tsg_free(c, slab));
        TSG_TRY(tsg_free(c, sortslab));
    }
    return TSG_OK;
}

template <int M>
int launch_sym_merge(tsg_ctx *c, const Bins &bl, const SymArgs &a0) {
    constexpr int G = mt_g(M), SL = mt_slice(M), BS = 256;
    const int B = BIN_MERGE + M;
    SymArgs a = a0;
    const int32_t *lst;
    int64_t n;
    if (!bin_select(bl, B, a, lst, n)) return TSG_OK;
    if constexpr (MERGE_IMPL == 3) {
        constexpr int K = MERGE_LISTS_PER_LANE, G2 = G / K;
        const unsigned grid = group_grid(c, n, BS / G2);
        k_sym_merge3<G2, K><<<grid, BS, 0, c->stream>>>(lst, n, a); ++c->launches;
        TSG_TRY(tsg_launch_check("k_sym_merge3", B, grid, BS, 0));
        return TSG_OK;
    }
    if constexpr (MERGE_LISTS_PER_LANE > 1) {   // K lists per lane, G / K lanes per row
        constexpr int K = MERGE_LISTS_PER_LANE, G2 = G / K;
        const size_t smem = (size_t)(BS / G2) * SL;
        TSG_TRY(set_smem(k_sym_merge2<G2, K, SL>, smem));
        const unsigned grid = bin_grid(c, bl, group_grid(c, n, BS / G2), k_sym_merge2<G2, K, SL>, BS, smem);
        k_sym_merge2<G2, K, SL><<<grid, BS, smem, c->stream>>>(lst, n, a); ++c->launches;
        TSG_TRY(tsg_launch_check("k_sym_merge2", B, grid, BS, smem));
        return TSG_OK;
    }
    const size_t smem = (size_t)(BS / G) * SL;
    TSG_TRY(set_smem(k_sym_merge<G, SL>, smem));
    const unsigned grid = bin_grid(c, bl, group_grid(c, n, BS / G), k_sym_merge<G, SL>, BS, smem);
    k_sym_merge<G, SL><<<grid, BS, smem, c->stream>>>(lst, n, a); ++c->launches;
    TSG_TRY(tsg_launch_check("k_sym_merge", B, grid, BS, smem));
    return TSG_OK;
}

int launch_sym_thread(tsg_ctx *c, const Bins &bl, const SymArgs &a0) {
    SymArgs a = a0;
    const int32_t *lst;
    int64_t n;
    if (!bin_select(bl, BIN_THREAD, a, lst, n)) return TSG_OK;
    const unsigned grid = bin_grid(c, bl, grid_for(n, 128, c->num_sms * 16), k_sym_thread<128>, 128, 0);
    k_sym_thread<128><<<grid, 128, 0, c->stream>>>(lst, n, a); ++c->launches;
    TSG_TRY(tsg_launch_check("k_sym_thread", BIN_THREAD, grid, 128, 0));
    return TSG_OK;
}

// resident CTAs per SM of the 1024-thread dense symbolic kernel with `smem`
// bytes (two fit when the bitmap does: one CTA per SM was 50 % occupancy;
// R-MAT scale 18: 74 -> 48 ms).  The dense numeric kernel stays at one per
// SM: twice the CTAs doubled its fp64 atomic traffic in flight (110 -> 154 ms).
static int dense_ctas_per_sm(size_t smem) {
    static const int cap = getenv("TSG_DENSE_CTAS") ? atoi(getenv("TSG_DENSE_CTAS")) : 2;
    int k = (int)((220 * 1024) / (smem + 1024));
    if (k > cap) k = cap;
    return k < 1 ? 1 : k;
}

// dense-tier tuning knobs (environment, read once)
static int dense_win_param(const char *name, int dflt) {
    const char *e = getenv(name);
    return e ? atoi(e) : dflt;
}

int launch_sym_dense(tsg_ctx *c, const Bins &bl, const SymArgs &a, int64_t ncols, bool sorted_sets) {
    if (bl.device) return TSG_OK;   // excluded by the host's bounds (device_bins_ok)
    const int64_t n = bl.off[BIN_DENSE + 1] - bl.off[BIN_DENSE];
    if (n <= 0) return TSG_OK;
    const int64_t nw = dense_words(ncols);
    const int32_t *dl = bl.list + bl.off[BIN_DENSE];
    // 64 KB windows (two CTAs per SM) once B exceeds 8192 sets: R-MAT scale
    // 20 248 -> 205 ms, scale 21 ~880 -> 763 ms against one 128 / 192 KB
    // window per SM; at scale 18 (4096 sets) one window stays faster
    static const int64_t WW = dense_win_param("TSG_SYM_WIN_WORDS", 8192);
    if ((nw * 8 > DENSE_SMEM || nw > WW) && sorted_sets && !getenv("TSG_SYM_DENSE_L2")) {
        // windowed shared-memory bitmaps; cut points in batches of rows
        const int64_t ww = nw < WW ? nw : WW;
        const int nwin = (int)((nw + ww - 1) / ww);
        const size_t smem = (size_t)ww * 8;
        TSG_TRY(set_smem(k_sym_dense<1024, 1>, smem));
        int32_t *ne = nullptr;
        int64_t *nc = nullptr;
        int64_t *eoff = nullptr, *coff = nullptr;
        TSG_TRY(tsg_alloc_t(c, &ne, (size_t)n));
        TSG_TRY(tsg_alloc_t(c, &nc, (size_t)n));
        TSG_TRY(tsg_alloc_t(c, &eoff, (size_t)n + 1));
        TSG_TRY(tsg_alloc_t(c, &coff, (size_t)n + 1));
        k_alen<<<grid_for(n, 256, c->num_sms * 8), 256, 0, c->stream>>>(dl, n, a.arp, a.a_row_off, nwin - 1, ne,
                                                                        nc);
        ++c->launches;
        TSG_TRY(tsg_exclusive_scan_i32_to_i64(c, ne, eoff, n));
        TSG_TRY(tsg_exclusive_scan_i64(c, nc, coff, n));
        std::vector<int64_t> hc((size_t)n + 1);
        TSG_CK(cudaMemcpyAsync(hc.data(), coff, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
        TSG_CK(cudaStreamSynchronize(c->stream));
        const int64_t CUT_MAX = (int64_t)128 << 20;
        int64_t maxrow = 1;
        for (int64_t r = 0; r < n; ++r) maxrow = std::max(maxrow, hc[r + 1] - hc[r]);
        const int64_t cap = std::max<int64_t>(std::min<int64_t>(CUT_MAX, hc[n]), maxrow);
        int32_t *cut = nullptr;
        TSG_TRY(tsg_alloc_t(c, &cut, (size_t)cap));
        for (int64_t b0 = 0; b0 < n;) {
            int64_t b1 = b0 + 1;
            while (b1 < n && hc[b1 + 1] - hc[b0] <= cap) ++b1;
            const int64_t nb = b1 - b0;
            k_sym_dense_cut<<<grid_for(nb * 256, 256, c->num_sms * 16), 256, 0, c->stream>>>(
                dl + b0, nb, a, ww, nwin, eoff + b0, coff + b0, hc[b0], cut);
            ++c->launches;
            const unsigned grid = (unsigned)std::min<int64_t>(nb, (int64_t)c->num_sms * dense_ctas_per_sm(smem));
            k_sym_dense<1024, 1><<<grid, 1024, smem, c->stream>>>(dl + b0, nb, a, nw, ww, nullptr, coff + b0, hc[b0],
                                                                cut);
            ++c->launches;
            TSG_TRY(tsg_launch_check("k_sym_dense", BIN_DENSE, grid, 1024, smem));
            b0 = b1;
        }
        TSG_TRY(tsg_free(c, cut));
        TSG_TRY(tsg_free(c, ne));
        TSG_TRY(tsg_free(c, nc));
        TSG_TRY(tsg_free(c, eoff));
        TSG_TRY(tsg_free(c, coff));
        return TSG_OK;
    }
    if (nw * 8 > DENSE_SMEM) {   // bitmap slabs in global memory (L2-resident)
        int64_t ctas = 2 * c->num_sms;
        while (ctas > c->num_sms / 2 && ctas * nw * 8 > ((int64_t)2 << 30)) ctas /= 2;
        if (ctas > n) ctas = n;
        uint64_t *gbm = nullptr;
        TSG_TRY(tsg_alloc_t(c, &gbm, (size_t)(ctas * nw)));
        TSG_TRY(tsg_fill(c, gbm, 0, (size_t)(ctas * nw) * 8, c->stream));
        k_sym_dense<1024, 2><<<(unsigned)ctas, 1024, 0, c->stream>>>(dl, n, a, nw, nw, gbm, nullptr, 0, nullptr);
        ++c->launches;
        TSG_TRY(tsg_launch_check("k_sym_dense", BIN_DENSE, (unsigned)ctas, 1024, 0));
        TSG_TRY(tsg_free(c, gbm));
        return TSG_OK;
    }
    const size_t smem = (size_t)nw * 8;
    TSG_TRY(set_smem(k_sym_dense<1024, 0>, smem));
    const unsigned grid = grid_for(n, 1, c->num_sms * dense_ctas_per_sm(smem));
    k_sym_dense<1024, 0><<<grid, 1024, smem, c->stream>>>(dl, n, a, nw, nw, nullptr, nullptr, 0, nullptr);
    ++c->launches;
    TSG_TRY(tsg_launch_check("k_sym_dense", BIN_DENSE, grid, 1024, smem));
    return TSG_OK;
}


int launch_num_dense(tsg_ctx *c, const Bins &bl, const NumArgs &a, int64_t ncols) {
    if (bl.device) return TSG_OK;   // excluded by the host's bounds (device_bins_ok)
    const int64_t n = bl.off[BIN_DENSE + 1] - bl.off[BIN_DENSE];
    if (n <= 0) return TSG_OK;
    static const int per_sm = dense_win_param("TSG_DENSE_WIN_CTAS", 1);
    static const int W = dense_win_param("TSG_DENSE_WIN", per_sm > 1 ? 8192 : 19456);
    static const int WS = dense_win_param("TSG_DENSE_WIN_SETS", per_sm > 1 ? 2048 : 4096);
    static const int old = dense_win_param("TSG_DENSE_FLAT", 0);
    if (!old || dense_words(ncols) * 12 > DENSE_SMEM) {
        const int64_t nw = dense_words(ncols);
        DenseWin dw;
        dw.W = W;
        dw.sets = WS;
        dw.maxw = (int)((ncols + W - 1) / W + (nw + WS - 1) / WS + 2);
        int64_t batch = ((int64_t)64 << 20) / (dw.maxw * 8);
        if (batch < 1) batch = 1;
        if (batch > n) batch = n;
        int32_t *nwin = nullptr, *ncut_e = nullptr;
        int64_t *ncut = nullptr;
        int64_t *woff = nullptr, *eoff = nullptr, *coff = nullptr;
        int2 *wst = nullptr;
        TSG_TRY(tsg_alloc_t(c, &nwin, (size_t)batch));
        TSG_TRY(tsg_alloc_t(c, &ncut_e, (size_t)batch));
        TSG_TRY(tsg_alloc_t(c, &ncut, (size_t)batch));
        TSG_TRY(tsg_alloc_t(c, &woff, (size_t)batch + 1));
        TSG_TRY(tsg_alloc_t(c, &eoff, (size_t)batch + 1));
        TSG_TRY(tsg_alloc_t(c, &coff, (size_t)batch + 1));
        TSG_TRY(tsg_alloc_t(c, &wst, (size_t)(batch * dw.maxw)));
        unsigned long long *counter = reinterpret_cast<unsigned long long *>(c->d_small + 30);
        const size_t smem = (size_t)WS * 12 + 8 + (size_t)(W + 64) * 8;
        TSG_TRY(set_smem(k_num_dense_win<1024>, smem));
        for (int64_t b0 = 0; b0 < n; b0 += batch) {
            const int64_t nb = n - b0 < batch ? n - b0 : batch;
            const int32_t *lst = bl.list + bl.off[BIN_DENSE] + b0;
            k_num_dense_prep<PREP_NT><<<grid_for(nb, 1, c->num_sms * (2048 / PREP_NT)), PREP_NT, 0, c->stream>>>(lst, nb, a, dw, nwin,
                                                                                             wst, ncut_e, ncut);
            ++c->launches;
            TSG_TRY(tsg_exclusive_scan_i32_to_i64(c, nwin, woff, nb));
            TSG_TRY(tsg_exclusive_scan_i32_to_i64(c, ncut_e, eoff, nb));
            TSG_TRY(tsg_exclusive_scan_i64(c, ncut, coff, nb));
            TSG_TRY(tsg_put_small(c, coff + nb, 1, 2));
            TSG_TRY(tsg_put_small(c, eoff + nb, 1, 3));
            TSG_CK(cudaStreamSynchronize(c->stream));
            const int64_t ncuts = c->h_small[2], nents = c->h_small[3];
            int32_t *cut = nullptr;
            if (ncuts > 0) {
                TSG_TRY(tsg_alloc_t(c, &cut, (size_t)ncuts));
                k_num_dense_cut<<<grid_for(nents, 256, c->num_sms * 16), 256, 0, c->stream>>>(
                    lst, nb, a, dw, woff, wst, eoff, coff, cut);
                ++c->launches;
            }
            TSG_TRY(tsg_fill(c, counter, 0, sizeof(unsigned long long), c->stream));
            k_num_dense_win<1024><<<c->num_sms * per_sm, 1024, smem, c->stream>>>(lst, nb, a, dw, woff, wst,
                                                                                  coff, cut, counter);
            ++c->launches;
            TSG_TRY(tsg_launch_check("k_num_dense_win", BIN_DENSE, c->num_sms * per_sm, 1024, smem));
            if (cut) TSG_TRY(tsg_free(c, cut));
        }
        TSG_TRY(tsg_free(c, ncut_e));
        TSG_TRY(tsg_free(c, ncut));
        TSG_TRY(tsg_free(c, eoff));
        TSG_TRY(tsg_free(c, coff));
        TSG_TRY(tsg_free(c, nwin));
        TSG_TRY(tsg_free(c, woff));
        TSG_TRY(tsg_free(c, wst));
        return TSG_OK;
    }
    const int64_t nw = dense_words(ncols);
    const size_t smem = (size_t)nw * 12;
    TSG_TRY(set_smem(k_num_dense<1024>, smem));
    static const int flat_ctas = dense_win_param("TSG_DENSE_FLAT_CTAS", 1);
    k_num_dense<1024><<<grid_for(n, 1, c->num_sms * flat_ctas), 1024, smem, c->stream>>>(bl.list + bl.off[BIN_DENSE], n,
                                                                             a, nw); ++c->launches;
    TSG_TRY(tsg_launch_check("k_num_dense", BIN_DENSE, grid_for(n, 1, c->num_sms), 1024, smem));
    return TSG_OK;
}

// Concurrent bins: the rows of different group-tier bins are disjoint, so the
// first nonempty bin runs on the compute stream and each further one on an
// auxiliary stream forked from it; join() makes the compute stream wait for
// them all.  Small bins (a few boundary rows with long dependent chains) then
// overlap the big bin instead of adding their latency to the phase.  Only
// kernels without per-launch allocations are forked (the arena is ordered on
// the compute stream).
struct BinFork {
    tsg_ctx *c;
    int used = 0;          // nonempty bins so far
    bool forked = false;
    explicit BinFork(tsg_ctx *cc) : c(cc) {}
    template <class L>
    int run(int64_t n, L launch) {
        if (n <= 0) return TSG_OK;
        if (used++ == 0) {
            // the fork point precedes the first bin, so the later bins do
            // not wait for it (a 16-row bin 0 otherwise serialised ~20 us
            // of dependent-load latency ahead of the big bin)
            TSG_CK(cudaEventRecord(c->ev_fork, c->stream));
            return launch();   // first bin: compute stream
        }
        const int k = (used - 2) % tsg_ctx::NAUX;
        forked = true;
        cudaStream_t main = c->stream;
        TSG_CK(cudaStreamWaitEvent(c->aux[k], c->ev_fork, 0));
        c->stream = c->aux[k];
        const int r = launch();
        c->stream = main;
        return r;
    }
    int join() {
        if (!forked) return TSG_OK;
        const int naux = used - 1 < tsg_ctx::NAUX ? used - 1 : tsg_ctx::NAUX;
        for (int k = 0; k < naux; ++k) {
            TSG_CK(cudaEventRecord(c->ev_join[k], c->aux[k]));
            TSG_CK(cudaStreamWaitEvent(c->stream, c->ev_join[k], 0));
        }
        return TSG_OK;
    }
};

// Bins run concurrently (BinFork): the largest is launched first on the
// compute stream, the others on high-priority auxiliary streams, so their
// blocks are dispatched as soon as the big bin's first blocks retire and
// finish inside it instead of trailing it (measured: a 33 us merge bin ran
// 16 us past the 164 us one when it queued behind all of its blocks;
// launching the small bins first instead delayed the big one by the launch
// latency of each).
struct BinJob {
    int64_t n;
    std::function<int()> launch;
};

// Device-driven mode: every possible bin the hint left empty, in one launch
// of the most general group kernel (bin 6: any row of the group / merge /
// thread tiers fits its slice).  Its grid is small: the bins are expected
// empty, and blocks of a 64 KB-slice kernel waiting for shared memory next
// to the big bin's blocks would hold back that bin (measured: a full-width
// leftover slowed config 2's RA*P bins by 15-20 %).
static unsigned leftover_grid() {
    static const unsigned g = [] {
        const char *e = getenv("TSG_LEFTOVER_GRID");
        const int v = e ? atoi(e) : 16;
        return (unsigned)(v > 0 ? v : 16);
    }();
    return g;
}
uint32_t leftover_mask(const Bins &bl) {
    uint32_t m = 0;
    for (int b = 0; b < NBINS; ++b)
        if (((bl.possible >> b) & 1u) && bl.hint[b + 1] - bl.hint[b] <= 0) m |= 1u << b;
    return m;
}

int launch_sym_leftover(tsg_ctx *c, const Bins &bl, const SymArgs &a0) {
    if (!bl.device) return TSG_OK;
    const uint32_t m = leftover_mask(bl);
    if (!m) return TSG_OK;
    constexpr int G = gt_g_sym(6), SL = gt_slice(6), BS = gt_block(6);
    SymArgs a = a0;
    a.dbins = bl.dstart;
    a.bin = -1;
    a.binmask = m;
    const size_t smem = (size_t)(BS / G) * SL;
    TSG_TRY(set_smem(k_sym_group<G, SL>, smem));
    k_sym_group<G, SL><<<leftover_grid(), BS, smem, c->stream>>>(bl.list, 0, a); ++c->launches;
    TSG_TRY(tsg_launch_check("k_sym_group(leftover)", 6, leftover_grid(), BS, smem));
    return TSG_OK;
}

template <int MODE>
int launch_num_leftover_m(tsg_ctx *c, const Bins &bl, const NumArgs &a0, uint32_t m) {
    constexpr int G = gt_g(6), SL = gt_slice(6);
    constexpr int BS = num_bs<G, MODE>() < gt_block(6) ? num_bs<G, MODE>() : gt_block(6);
    NumArgs a = a0;
    a.dbins = bl.dstart;
    a.bin = -1;
    a.binmask = m;
    const size_t smem = num_slices_bytes<G, SL>(BS / G) + (MODE == 2 ? (size_t)(BS / G) * ustage_bytes<G>() : 0);
    TSG_TRY(set_smem(k_num_group<G, SL, MODE>, smem));
    k_num_group<G, SL, MODE><<<leftover_grid(), BS, smem, c->stream>>>(bl.list, 0, a); ++c->launches;
    TSG_TRY(tsg_launch_check("k_num_group(leftover)", 6, leftover_grid(), BS, smem));
    return TSG_OK;
}

int launch_num_leftover(tsg_ctx *c, const Bins &bl, const NumArgs &a) {
    if (!bl.device) return TSG_OK;
    const uint32_t m = leftover_mask(bl);
    if (!m) return TSG_OK;
    if (a.seq >= gt_g(6) / 2) return launch_num_leftover_m<1>(c, bl, a, m);
    if (a.unit_known > 0) return launch_num_leftover_m<2>(c, bl, a, m);
    return launch_num_leftover_m<0>(c, bl, a, m);
}

static bool leftover_concurrent() {
    static const bool v = getenv("TSG_LEFTOVER_CONCURRENT") != nullptr;
    return v;
}

int run_bins_largest_first(tsg_ctx *c, BinJob *jobs, int njobs) {
    std::stable_sort(jobs, jobs + njobs, [](const BinJob &x, const BinJob &y) { return x.n > y.n; });
    BinFork f(c);
    tsg_trace_host("bins: first launch");
    for (int k = 0; k < njobs; ++k) {
        TSG_TRY(f.run(jobs[k].n, jobs[k].launch));
        if (k == 0) tsg_trace_host("bins: first launched");
    }
    return f.join();
}

int run_symbolic_bins(tsg_ctx *c, const Bins &bl, const SymArgs &a) {
    auto cnt = [&](int b) -> int64_t {
        if (!bl.device) return bl.off[b + 1] - bl.off[b];
        if (!((bl.possible >> b) & 1u)) return 0;
        return bl.hint[b + 1] - bl.hint[b] > 0 ? bl.hint[b + 1] - bl.hint[b] : 0;   // largest first
    };
    BinJob jobs[] = {
        {cnt(BIN_THREAD), [&] { return launch_sym_thread(c, bl, a); }},
        {cnt(BIN_MERGE + 0), [&] { return launch_sym_merge<0>(c, bl, a); }},
        {cnt(BIN_MERGE + 1), [&] { return launch_sym_merge<1>(c, bl, a); }},
        {cnt(BIN_MERGE + 2), [&] { return launch_sym_merge<2>(c, bl, a); }},
        {cnt(0), [&] { return launch_sym_group<0>(c, bl, a); }},
        {cnt(1), [&] { return launch_sym_group<1>(c, bl, a); }},
        {cnt(2), [&] { return launch_sym_group<2>(c, bl, a); }},
        {cnt(3), [&] { return launch_sym_group<3>(c, bl, a); }},
        {cnt(4), [&] { return launch_sym_group<4>(c, bl, a); }},
        {cnt(5), [&] { return launch_sym_group<5>(c, bl, a); }},
        {cnt(6), [&] { return launch_sym_group<6>(c, bl, a); }},
        {leftover_concurrent() && bl.device && leftover_mask(bl) ? 1 : 0, [&] { return launch_sym_leftover(c, bl, a); }},
    };
    // the leftover launch (bins the hint left empty) goes first and alone on
    // the compute stream: a few us, and no 64 KB-slice blocks waiting for
    // shared memory beside the big bins
    if (!leftover_concurrent()) TSG_TRY(launch_sym_leftover(c, bl, a));
    TSG_TRY(run_bins_largest_first(c, jobs, (int)(sizeof(jobs) / sizeof(jobs[0]))));
    TSG_TRY(launch_sym_cta<0>(c, bl, a));
    TSG_TRY(launch_sym_cta<1>(c, bl, a));
    TSG_TRY(launch_sym_global(c, bl, a));
    return TSG_OK;
}

int run_numeric_bins(tsg_ctx *c, const Bins &bl, const NumArgs &a) {
    auto cnt = [&](int b) -> int64_t {
        if (!bl.device) return bl.off[b + 1] - bl.off[b];
        if (!((bl.possible >> b) & 1u)) return 0;
        return bl.hint[b + 1] - bl.hint[b] > 0 ? bl.hint[b + 1] - bl.hint[b] : 0;   // largest first
    };
    BinJob jobs[] = {
        {cnt(0), [&] { return launch_num_group<0>(c, bl, a); }},
        {cnt(1), [&] { return launch_num_group<1>(c, bl, a); }},
        {cnt(2), [&] { return launch_num_group<2>(c, bl, a); }},
        {cnt(3), [&] { return launch_num_group<3>(c, bl, a); }},
        {cnt(4), [&] { return launch_num_group<4>(c, bl, a); }},
        {cnt(5), [&] { return launch_num_group<5>(c, bl, a); }},
        {cnt(6), [&] { return launch_num_group<6>(c, bl, a); }},
        {leftover_concurrent() && bl.device && leftover_mask(bl) ? 1 : 0, [&] { return launch_num_leftover(c, bl, a); }},
    };
    // the leftover launch (bins the hint left empty) goes first and alone on
    // the compute stream: a few us, and no 64 KB-slice blocks waiting for
    // shared memory beside the big bins
    if (!leftover_concurrent()) TSG_TRY(launch_num_leftover(c, bl, a));
    TSG_TRY(run_bins_largest_first(c, jobs, (int)(sizeof(jobs) / sizeof(jobs[0]))));
    TSG_TRY(launch_num_cta<0>(c, bl, a));
    TSG_TRY(launch_num_cta<1>(c, bl, a));
    TSG_TRY(launch_num_global(c, bl, a));
    return TSG_OK;
}

// group size for row-streaming kernels from the average row length
int pick_g(int64_t nnz, int64_t rows) {
    double avg = rows ? (double)nnz / (double)rows : 0.0;
    if (avg <= 6) return 4;
    if (avg <= 12) return 8;
    if (avg <= 24) return 16;
    return 32;
}

template <int G>
void launch_bounds_g(tsg_ctx *c, int64_t rows, const tsg_csr *a, const int64_t *brp,
                     const int32_t *cbcnt, int64_t *flops, int64_t *sbound,
                     unsigned long long *total) {
    unsigned grid = grid_for(rows, 256 / G, c->num_sms * 32);
    k_row_bounds<G><<<grid, 256, 0, c->stream>>>(rows, a->rp, a->col, brp, cbcnt, flops, sbound,
                                                 total); ++c->launches;
}

void launch_bounds(tsg_ctx *c, const tsg_csr *a, const int64_t *brp, const int32_t *cbcnt,
                   int64_t *flops, int64_t *sbound, unsigned long long *total) {
    switch (pick_g(a->nnz, a->rows)) {
    case 4: launch_bounds_g<4>(c, a->rows, a, brp, cbcnt, flops, sbound, total); break;
    case 8: launch_bounds_g<8>(c, a->rows, a, brp, cbcnt, flops, sbound, total); break;
    case 16: launch_bounds_g<16>(c, a->rows, a, brp, cbcnt, flops, sbound, total); break;
    default: launch_bounds_g<32>(c, a->rows, a, brp, cbcnt, flops, sbound, total); break;
    }
}


}  // namespace

// ======================================================================= internal API

int tsg_fused_bounds(tsg_ctx *c, int64_t rows_out, const tsg_csr *a, int64_t a_row_off,
                     int32_t b_lo, int32_t b_hi, const int64_t *cbstart, const int32_t *cbcnt,
                     const int64_t *prp, int64_t *sbound);

void tsg_launch_row_flops(tsg_ctx *c, const tsg_csr *a, const int64_t *brp, int64_t *flops) {
    if (a->rows > 0 && a->nnz > 0) launch_bounds(c, a, brp, nullptr, flops, nullptr, nullptr);
    else if (a->rows > 0) tsg_fill(c, flops, 0, sizeof(int64_t) * a->rows, c->stream);
}

int tsg_compress_impl(tsg_ctx *c, const tsg_csr *b, tsg_cmat **out);   // tsg_compress.cu

// counts (+ msets) of A * B for output rows [0, rows_out); fused mode when
// prp != null or a_row_off/b range given.
int tsg_symbolic_impl(tsg_ctx *c, int64_t rows_out, const tsg_csr *a, int64_t a_row_off,
                      int32_t b_lo, int32_t b_hi, const tsg_cmat *cb, const tsg_csr *partial,
                      tsg_vec **out, int64_t **sbound_out) {
    tsg_vec *v = nullptr;
    TSG_TRY(tsg_vec_alloc(c, rows_out, true, &v));
    int64_t *sbound = nullptr;
    uint8_t *bins = nullptr;
    TSG_TRY(tsg_alloc_t(c, &sbound, rows_out + 1));
    TSG_TRY(tsg_alloc_t(c, &bins, rows_out + 1));
    if (rows_out > 0) {
        // set bounds: partial row length + sum of selected compressed B rows
        // largest compressed row: kept by compress in cnt[rows + 1], else reduced here
        int *maxcb = cb->cnt + cb->rows + 1;
        if (!cb->dmax_valid) {
            maxcb = reinterpret_cast<int *>(c->d_small + 50);
            TSG_TRY(tsg_fill(c, maxcb, 0, sizeof(int), c->stream));
            k_max_i32<<<grid_for(cb->rows, 256, c->num_sms * 4), 256, 0, c->stream>>>(cb->rows, cb->cnt,
                                                                                    maxcb); ++c->launches;
        }
        // short A rows (known at upload): the bin functor sums the exact bound
        const bool inline_bounds = a->max_row >= 0 && a->max_row <= INLINE_BOUND_A;
        if (a_row_off == 0 && b_lo == 0 && b_hi == 0x7fffffff && partial == nullptr &&
            rows_out == a->rows) {
            const unsigned g = grid_for(a->rows, 256, c->num_sms * 16);
            if (!inline_bounds) {
                switch (pick_g(a->nnz, a->rows)) {
                case 4: TSG_CK(launch_pdl(k_sym_bounds<4>, g, 256, 0, c->stream, a->rows, (const int64_t *)a->rp, (const int32_t *)a->col, (const int32_t *)cb->cnt, maxcb, sbound)); break;
                case 8: TSG_CK(launch_pdl(k_sym_bounds<8>, g, 256, 0, c->stream, a->rows, (const int64_t *)a->rp, (const int32_t *)a->col, (const int32_t *)cb->cnt, maxcb, sbound)); break;
                case 16: TSG_CK(launch_pdl(k_sym_bounds<16>, g, 256, 0, c->stream, a->rows, (const int64_t *)a->rp, (const int32_t *)a->col, (const int32_t *)cb->cnt, maxcb, sbound)); break;
                default: TSG_CK(launch_pdl(k_sym_bounds<32>, g, 256, 0, c->stream, a->rows, (const int64_t *)a->rp, (const int32_t *)a->col, (const int32_t *)cb->cnt, maxcb, sbound)); break;
                }
                ++c->launches;
            }
        } else {
            TSG_TRY(tsg_fused_bounds(c, rows_out, a, a_row_off, b_lo, b_hi, cb->start, cb->cnt,
                                     partial ? partial->rp : nullptr, sbound));
        }
        int64_t *scap = nullptr;
        TSG_TRY(tsg_alloc_t(c, &scap, rows_out + 1));
        TSG_TRY(tsg_alloc_t(c, &v->sptr, rows_out + 1));
        Bins bl;
        int64_t set_cap = 0;
        // merge tier only when the compressed rows are sorted by set (row-sorted
        // B -> compact compression) and there is no partial row to fold in
        const int64_t *merge_arp = (cb->sorted_sets && partial == nullptr) ? a->rp : nullptr;
        const int64_t cb_cols = cb->cols;
        const bool plain = a_row_off == 0 && b_lo == 0 && b_hi == 0x7fffffff && partial == nullptr &&
                           rows_out == a->rows;
        TSG_TRY(tsg_partition<NBINS>(c, rows_out, SymBinF{sbound, v->d, v->aux, scap, merge_arp, a_row_off,
                                             partial == nullptr ? cb_cols : 0,
                                             plain ? a->rp : nullptr, maxcb,
                                             (plain && cb->identity_rows) ? a->rp : nullptr,
                                             (plain && inline_bounds) ? a->col : nullptr, cb->cnt},
                                     bins, bl,
                                     v->sptr + rows_out, &set_cap,
                                     [&]() { return tsg_exclusive_scan_i64(c, scap, v->sptr, rows_out); },
                                     c->nowait != 0, c->hint_sym, c->hintd_sym));
        if (bl.device) {   // device-driven: host bounds instead of read-back sizes
            bl.possible = c->sym_possible;
            set_cap = c->set_cap_bound;
        }
        TSG_TRY(tsg_free(c, scap));
        TSG_TRY(tsg_alloc_t(c, &v->sset, set_cap > 0 ? set_cap : 1));
        TSG_TRY(tsg_alloc_t(c, &v->sbits, set_cap > 0 ? set_cap : 1));
        SymArgs sa{};
        sa.arp = a->rp;
        sa.acol = a->col;
        sa.a_row_off = a_row_off;
        sa.b_lo = b_lo;
        sa.b_hi = b_hi;
        sa.cbstart = cb->start;
        sa.cbcnt = cb->cnt;
        sa.cbset = cb->set;
        sa.cbbits = cb->bits;
        sa.prp = partial ? partial->rp : nullptr;
        sa.pcol = partial ? partial->col : nullptr;
        sa.sbound = sbound;
        sa.counts = v->d;
        sa.msets = v->aux;
        sa.err = c->d_err;
        sa.sptr = v->sptr;
        sa.oset = v->sset;
        sa.obits = v->sbits;
        sa.maxcb = maxcb;
        sa.unit_dense = cb->identity_rows;
        if (c->timing) cudaEventRecord(c->ev_sym[0], c->stream);
        TSG_TRY(run_symbolic_bins(c, bl, sa));
        TSG_TRY(launch_sym_dense(c, bl, sa, cb_cols, cb->sorted_sets != 0));
        if (c->timing) cudaEventRecord(c->ev_sym[1], c->stream);
        TSG_TRY(tsg_free(c, bl.list));
        TSG_TRY(tsg_free(c, bl.dstart));
    }
    TSG_TRY(tsg_free(c, bins));
    if (sbound_out)
        *sbound_out = sbound;
    else
        TSG_TRY(tsg_free(c, sbound));
    *out = v;
    return TSG_OK;
}

namespace {
__global__ void k_fused_bounds(int64_t rows_out, const int64_t *__restrict__ arp,
                               const int32_t *__restrict__ acol, int64_t a_row_off, int32_t b_lo,
                               int32_t b_hi, const int64_t *__restrict__ cbstart,
                               const int32_t *__restrict__ cbcnt, const int64_t *__restrict__ prp,
                               int64_t *__restrict__ sbound, const int32_t *__restrict__ plen) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w; i < rows_out; i += nw) {
        int64_t gi = i + a_row_off;
        int64_t s = 0;
        for (int64_t t = arp[gi] + lane; t < arp[gi + 1]; t += 32) {
            int k = acol[t];
            if (k >= b_lo && k < b_hi) s += cbcnt[k - b_lo];
        }
        for (int d = 16; d >= 1; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
        // in place (plen): a row with no product in this chunk is left as it
        // is (bound 0 = skipped by the bin functor)
        if (lane == 0) sbound[i] = (plen && s == 0) ? 0 : s + (prp ? prp[i + 1] - prp[i] : 0) + (plen ? plen[i] : 0);
    }
}
}  // namespace

int tsg_fused_bounds(tsg_ctx *c, int64_t rows_out, const tsg_csr *a, int64_t a_row_off,
                     int32_t b_lo, int32_t b_hi, const int64_t *cbstart, const int32_t *cbcnt,
                     const int64_t *prp, int64_t *sbound) {
    k_fused_bounds<<<grid_for(rows_out, 8, c->num_sms * 32), 256, 0, c->stream>>>(
        rows_out, a->rp, a->col, a_row_off, b_lo, b_hi, cbstart, cbcnt, prp, sbound, nullptr); ++c->launches;
    TSG_CK(cudaGetLastError());
    return TSG_OK;
}

// numeric into a freshly allocated C whose row_ptr = scan(counts)
int tsg_numeric_impl(tsg_ctx *c, int64_t rows_out, int64_t cols_out, const tsg_csr *a,
                     int64_t a_row_off, int32_t b_lo, int32_t b_hi, const tsg_csr *b,
                     const tsg_cmat *cb, const tsg_csr *partial, const tsg_vec *counts,
                     const int64_t *sbound_in, tsg_csr **out, PhaseTimer *pt) {
    // C row pointers, numeric bins and nnz(C): one sync for all of them
    int64_t *cptr = nullptr;
    TSG_TRY(tsg_alloc_t(c, &cptr, rows_out + 1));
    TSG_TRY(tsg_exclusive_scan_i64(c, counts->d, cptr, rows_out));
    if (pt) pt->mark();
    int64_t *sbound = nullptr;
    uint8_t *bins = nullptr;
    TSG_TRY(tsg_alloc_t(c, &bins, rows_out + 1));
    if (!sbound_in) {
        TSG_TRY(tsg_alloc_t(c, &sbound, rows_out + 1));
        if (rows_out > 0)
            TSG_TRY(tsg_fused_bounds(c, rows_out, a, a_row_off, b_lo, b_hi, cb->start, cb->cnt,
                                     partial ? partial->rp : nullptr, sbound));
        sbound_in = sbound;
    }
    Bins bl;
    int64_t nnz = 0;
    if (rows_out > 0) {
        TSG_TRY(tsg_partition<NBINS>(c, rows_out, NumBinF{counts->d, counts->aux, sbound_in, cb->sorted_sets ? b->cols : 0}, bins, bl,
                                     cptr + rows_out, &nnz, NoMid(), c->nowait != 0, c->hint_num, c->hintd_num));
        if (bl.device) {
            bl.possible = c->num_possible;
            nnz = c->nnz_bound;   // capacity; the exact count stays on the device
        }
    }
    tsg_csr *C = nullptr;
    if (c->c_host_out) {
        // placement with C in the slow tier: the numeric kernels write C over
        // PCIe into pinned, mapped host memory
        TSG_TRY(tsg_csr_alloc_mapped(c, rows_out, cols_out, nnz, true, &C));
        TSG_CK(cudaMemcpyAsync(C->rp, cptr, (rows_out + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost,
                               c->stream));
    } else {
        C = new tsg_csr();
        C->max_row = -1;
        C->rows = rows_out;
        C->cols = cols_out;
        C->nnz = nnz;
        C->max_row_bound = c->c_row_bound;   // 0 unless tsg_multiply planned bounds
        if (bl.device) {
            C->lazy_nnz = 1;
            C->owner = c;
        }
        C->rp = cptr;
        C->col = nullptr;
        C->val = nullptr;
        int st = TSG_OK;
        if (c->c_res_col && nnz <= c->c_res_cap) {   // streamed multiply's reservoir
            C->col = c->c_res_col;
            C->val = c->c_res_val;
            C->cv_borrowed = 1;
        } else {
            st = tsg_alloc_t(c, &C->col, nnz);
            if (st == TSG_OK) st = tsg_alloc_t(c, &C->val, nnz);
        }
        if (st != TSG_OK) {
            tsg_csr_free(c, C);
            return st;
        }
    }
    if (rows_out > 0 && nnz > 0) {
        NumArgs na{};
        na.arp = a->rp;
        na.acol = a->col;
        na.aval = a->val;
        na.a_row_off = a_row_off;
        na.b_lo = b_lo;
        na.b_hi = b_hi;
        na.brp = b->rp;
        na.bcol = b->col;
        na.bval = b->val;
        na.cbstart = cb->start;
        na.cbcnt = cb->cnt;
        na.cbset = cb->set;
        na.cbbits = cb->bits;
        na.prp = partial ? partial->rp : nullptr;
        na.pcol = partial ? partial->col : nullptr;
        na.pval = partial ? partial->val : nullptr;
        na.cptr = cptr;
        na.counts = counts->d;
        na.msets = counts->aux;
        na.sbound = sbound_in;
        na.ccol = C->col;
        na.cval = C->val;
        na.err = c->d_err;
        na.seq = (b->distinct && b->rows > 0) ? (int)(b->nnz / b->rows) : 0;   // lanes split a B row
        // only when its columns are known distinct (a repeated column would race)
        na.sptr = counts->sptr;
        na.sset = counts->sset;
        na.sbits = counts->sbits;
        na.unit_dense = (b->max_row == 1 && b->nnz == b->rows) ? 1 : 0;
        if (b->max_row >= 0) {   // known since upload: no device check
            na.unit_known = b->max_row <= 1 ? 1 : 0;
            na.unit_b = nullptr;
        } else {
            int *uflag = reinterpret_cast<int *>(c->d_small + 49);
            TSG_TRY(tsg_fill(c, uflag, 0xff, sizeof(int), c->stream));
            k_unit_rows<<<grid_for(b->rows, 256, c->num_sms * 8), 256, 0, c->stream>>>(b->rows, b->rp, nullptr,
                                                                                     uflag); ++c->launches;
            na.unit_known = -1;
            na.unit_b = uflag;
        }
        na.pstart = nullptr;
        na.plen_in = nullptr;
        na.plen_out = nullptr;
        const int rk = (int)(c->num_calls % tsg_ctx::NRING);
        if (c->timing) {
            cudaEventRecord(c->ev_num[0], c->stream);
            cudaEventRecord(c->ev_ring[2 * rk], c->stream);
        } else if (c->capture_timing) {   // graph capture: timestamped at every replay
            cudaEventRecordWithFlags(c->ev_ring[2 * rk], c->stream, cudaEventRecordExternal);
        }
        TSG_TRY(run_numeric_bins(c, bl, na));
        TSG_TRY(launch_num_dense(c, bl, na, b->cols));
        if (c->timing) {
            cudaEventRecord(c->ev_num[1], c->stream);
            cudaEventRecord(c->ev_ring[2 * rk + 1], c->stream);
            c->ring_timed[rk] = c->num_calls;
        } else if (c->capture_timing) {
            cudaEventRecordWithFlags(c->ev_ring[2 * rk + 1], c->stream, cudaEventRecordExternal);
            c->capture_rk = rk;
        } else {
            c->ring_timed[rk] = -1;
        }
    }
    if (bl.list) TSG_TRY(tsg_free(c, bl.list));
    TSG_TRY(tsg_free(c, bl.dstart));
    TSG_TRY(tsg_free(c, bins));
    TSG_TRY(tsg_free(c, sbound));
    if (pt) pt->mark();
    ++c->num_calls;
    // kernel errors (count mismatch, probe overflow) are checked at the next
    // synchronising call -- the download of C, the next partition read-back
    // or tsg_sync -- so the host can queue the next multiply while these run
    c->pending = "numeric";
    int s = TSG_OK;
    if (C->host_mapped) tsg_free(c, cptr);
    C->sorted = 1;   // every emitted row lists its columns in ascending order
    C->distinct = 1;
    if (s != TSG_OK) {
        tsg_csr_free(c, C);
        return s;
    }
    *out = C;
    return TSG_OK;
}

namespace {
__global__ void k_copy_partials(const int32_t *__restrict__ list, int64_t n,
                                const int64_t *__restrict__ cptr, const int32_t *__restrict__ plen,
                                const int32_t *__restrict__ col, const double *__restrict__ val,
                                int32_t *__restrict__ scol, double *__restrict__ sval) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t x = w; x < n; x += nw) {
        int64_t i = list[x];
        int64_t p0 = cptr[i];
        for (int64_t q = p0 + lane; q < p0 + plen[i]; q += 32) {
            scol[q] = col[q];
            sval[q] = val[q];
        }
    }
}
}  // namespace

// One in-place fused multiply-add step of the chunked executors:
//   C[r] = C[r] (partial prefix of plen[r] entries, row capacity cap[r]) +
//          A[r, b_lo:b_hi] * B_chunk
// Thread-group rows merge in place (tsg_group path, deferred emission); CTA
// and global-tier rows read their partial from a scratch copy.
int tsg_fused_inplace(tsg_ctx *c, const tsg_csr *a, int32_t b_lo, int32_t b_hi, const tsg_csr *b,
                      const tsg_cmat *cb, const int64_t *cptr, const int64_t *cap, int32_t *ccol,
                      double *cval, int32_t *plen, int64_t rows) {
    if (rows <= 0) return TSG_OK;
    int64_t *sbound = nullptr;
    uint8_t *bins = nullptr;
    TSG_TRY(tsg_alloc_t(c, &sbound, rows + 1));
    TSG_TRY(tsg_alloc_t(c, &bins, rows + 1));
    k_fused_bounds<<<grid_for(rows, 8, c->num_sms * 32), 256, 0, c->stream>>>(
        rows, a->rp, a->col, 0, b_lo, b_hi, cb->start, cb->cnt, nullptr, sbound, plen); ++c->launches;
    TSG_CK(cudaGetLastError());
    Bins bl;
    TSG_TRY(tsg_partition<NBINS>(c, rows, NumBinF{cap, nullptr, sbound, 0, 1}, bins, bl));
    NumArgs na;
    memset(&na, 0, sizeof(na));
    na.arp = a->rp;
    na.acol = a->col;
    na.aval = a->val;
    na.a_row_off = 0;
    na.b_lo = b_lo;
    na.b_hi = b_hi;
    na.brp = b->rp;
    na.bcol = b->col;
    na.bval = b->val;
    na.cbstart = cb->start;
    na.cbcnt = cb->cnt;
    na.cbset = cb->set;
    na.cbbits = cb->bits;
    na.cptr = cptr;
    na.counts = cap;
    na.sbound = sbound;
    na.ccol = ccol;
    na.cval = cval;
    na.err = c->d_err;
    na.seq = (b->distinct && b->rows > 0) ? (int)(b->nnz / b->rows) : 0;   // lanes split a B row
        // only when its columns are known distinct (a repeated column would race)
    na.pcol = ccol;            // in place
    na.pval = cval;
    na.pstart = cptr;
    na.plen_in = plen;
    na.plen_out = plen;
    if (b->max_row >= 0 && b->max_row <= 1) {   // unit B chunk: owner-folded products
        na.unit_known = 1;
        na.unit_dense = (b->max_row == 1 && b->nnz == b->rows) ? 1 : 0;
    }
    TSG_TRY(launch_num_group<0>(c, bl, na));
    TSG_TRY(launch_num_group<1>(c, bl, na));
    TSG_TRY(launch_num_group<2>(c, bl, na));
    TSG_TRY(launch_num_group<3>(c, bl, na));
    TSG_TRY(launch_num_group<4>(c, bl, na));
    TSG_TRY(launch_num_group<5>(c, bl, na));
    TSG_TRY(launch_num_group<6>(c, bl, na));
    int64_t nbig = bl.off[BIN_GLOBAL + 1] - bl.off[7];
    int32_t *scol = nullptr;
    double *sval = nullptr;
    if (nbig > 0) {
        int64_t total = 0;
        TSG_TRY(tsg_put_small(c, cptr + rows, 1, 40));
        TSG_CK(cudaStreamSynchronize(c->stream));
        total = c->h_small[40];
        TSG_TRY(tsg_alloc_t(c, &scol, total + 1));
        TSG_TRY(tsg_alloc_t(c, &sval, total + 1));
        k_copy_partials<<<grid_for(nbig, 8, c->num_sms * 16), 256, 0, c->stream>>>(
            bl.list + bl.off[7], nbig, cptr, plen, ccol, cval, scol, sval); ++c->launches;
        NumArgs nb = na;
        nb.pcol = scol;
        nb.pval = sval;
        TSG_TRY(launch_num_cta<0>(c, bl, nb));
        TSG_TRY(launch_num_cta<1>(c, bl, nb));
        TSG_TRY(launch_num_global(c, bl, nb));
    }
    TSG_CK(cudaGetLastError());
    TSG_TRY(tsg_free(c, scol));
    TSG_TRY(tsg_free(c, sval));
    TSG_TRY(tsg_free(c, bl.list));
    TSG_TRY(tsg_free(c, sbound));
    TSG_TRY(tsg_free(c, bins));
    return TSG_OK;
}

// ======================================================================= C ABI

extern "C" int tsg_probe_stats(tsg_ctx *c, int64_t out[4], int reset) {
    (void)c;
    for (int k = 0; k < 4; ++k) out[k] = 0;
#if TSG_PROBE_STATS
    unsigned long long h[4];
    TSG_CK(cudaDeviceSynchronize());
    TSG_CK(cudaMemcpyFromSymbol(h, g_tsg_probe, sizeof(h)));
    for (int k = 0; k < 4; ++k) out[k] = (int64_t)h[k];
    if (reset) {
        const unsigned long long z[4] = {0, 0, 0, 0};
        TSG_CK(cudaMemcpyToSymbol(g_tsg_probe, z, sizeof(z)));
    }
    return TSG_OK;
#else
    (void)reset;
    tsg_set_error("tsg_probe_stats: library built without -DTSG_PROBE_STATS=1");
    return TSG_EARG;
#endif
}

extern "C" int tsg_compress(tsg_ctx *c, const tsg_csr *b, tsg_cmat **out) {
    TSG_RESOLVE(c, b);
    TSG_TRY(tsg_compress_impl(c, b, out));
    return tsg_check_kernel_errors(c, "compress");
}

extern "C" int tsg_count_multiplications(tsg_ctx *c, const tsg_csr *a, const tsg_csr *b,
                                         int64_t *total) {
    TSG_RESOLVE(c, a);
    TSG_RESOLVE(c, b);
    if (a->cols != b->rows) {
        tsg_set_error("A is %lldx%lld but B has %lld rows", (long long)a->rows, (long long)a->cols,
                      (long long)b->rows);
        return TSG_EDIM;
    }
    TSG_TRY(tsg_fill(c, c->d_small, 0, sizeof(int64_t), c->stream));
    if (a->rows > 0 && a->nnz > 0)
        launch_bounds(c, a, b->rp, nullptr, nullptr, nullptr, (unsigned long long *)c->d_small);
    TSG_CK(cudaGetLastError());
    TSG_TRY(tsg_put_small(c, c->d_small, 1, 0));
    TSG_CK(cudaStreamSynchronize(c->stream));
    *total = c->h_small[0];
    return TSG_OK;
}

// Per-row K0 multiplications (kernel.py:135-145's bound loop over the
// uncompressed B: sum of nnz(B_k) over row i of A) -- the weights of the
// multi-GPU flops partition -- and their total
// (kernel.py:96-103 count_multiplications).
extern "C" int tsg_row_flops(tsg_ctx *c, const tsg_csr *a, const tsg_csr *b, int64_t *flops_host,
                             int64_t *total) {
    TSG_RESOLVE(c, a);
    TSG_RESOLVE(c, b);
    if (a->cols != b->rows) {
        tsg_set_error("A is %lldx%lld but B has %lld rows", (long long)a->rows, (long long)a->cols,
                      (long long)b->rows);
        return TSG_EDIM;
    }
    int64_t *f = nullptr;
    if (flops_host && a->rows > 0) TSG_TRY(tsg_alloc_t(c, &f, a->rows));
    TSG_TRY(tsg_fill(c, c->d_small, 0, sizeof(int64_t), c->stream));
    if (a->rows > 0) {
        if (a->nnz > 0) {
            launch_bounds(c, a, b->rp, nullptr, f, nullptr, (unsigned long long *)c->d_small);
        } else if (f) {
            TSG_TRY(tsg_fill(c, f, 0, sizeof(int64_t) * a->rows, c->stream));
        }
    }
    TSG_CK(cudaGetLastError());
    TSG_TRY(tsg_put_small(c, c->d_small, 1, 0));
    if (f) {
        TSG_CK(cudaMemcpyAsync(flops_host, f, sizeof(int64_t) * a->rows, cudaMemcpyDeviceToHost, c->stream));
    }
    TSG_CK(cudaStreamSynchronize(c->stream));
    if (f) TSG_TRY(tsg_free(c, f));
    if (total) *total = c->h_small[0];
    return TSG_OK;
}

extern "C" int tsg_symbolic(tsg_ctx *c, const tsg_csr *a, const tsg_cmat *cb, tsg_vec **counts) {
    TSG_RESOLVE(c, a);
    if (a->cols != cb->rows) {
        tsg_set_error("A has %lld cols but compressed B has %lld rows", (long long)a->cols,
                      (long long)cb->rows);
        return TSG_EDIM;
    }
    tsg_vec *v = nullptr;
    TSG_TRY(tsg_symbolic_impl(c, a->rows, a, 0, 0, 0x7fffffff, cb, nullptr, &v, nullptr));
    int s = tsg_check_kernel_errors(c, "symbolic");
    if (s != TSG_OK) {
        tsg_vec_free(c, v);
        return s;
    }
    *counts = v;
    return TSG_OK;
}

extern "C" int tsg_numeric(tsg_ctx *c, const tsg_csr *a, const tsg_csr *b, const tsg_cmat *cb,
                           const tsg_vec *counts, tsg_csr **out) {
    TSG_RESOLVE(c, a);
    TSG_RESOLVE(c, b);
    if (a->cols != b->rows) {
        tsg_set_error("A is %lldx%lld but B has %lld rows", (long long)a->rows, (long long)a->cols,
                      (long long)b->rows);
        return TSG_EDIM;
    }
    if (!a->val || !b->val) {
        tsg_set_error("numeric multiply requires values on both operands");
        return TSG_EVALID;
    }
    if (counts->n != a->rows) {
        tsg_set_error("c_counts length must equal A's row count");
        return TSG_EDIM;
    }
    tsg_cmat *own = nullptr;
    if (!cb) {
        TSG_TRY(tsg_compress_impl(c, b, &own));
        cb = own;
    }
    int s = tsg_numeric_impl(c, a->rows, b->cols, a, 0, 0, 0x7fffffff, b, cb, nullptr, counts,
                             nullptr, out, nullptr);
    if (own) tsg_cmat_free(c, own);
    return s;
}

// Host bounds for a device-driven multiply (see tsg_multiply): per-row set
// and entry bounds from the operands' known row lengths decide which bins can
// be non-empty; anything that could need the CTA, global or dense tiers (or a
// pool sized from device data) takes the read-back path.
struct HintKey {
    const tsg_ctx *c;
    int64_t ar, ac, an, br, bc, bn;
    bool operator<(const HintKey &o) const {
        return std::tie(c, ar, ac, an, br, bc, bn) < std::tie(o.c, o.ar, o.ac, o.an, o.br, o.bc, o.bn);
    }
};
struct HintBufs {
    int64_t *h = nullptr, *d = nullptr;   // 64 int64: [0, 32) symbolic, [32, 64) numeric
};
static std::mutex g_hint_mu;
static std::map<HintKey, HintBufs> g_hints;

// pinned, mapped bin-start buffers of an operand shape (slot 31 of each half
// = 1 once a read-back multiply has recorded the starts)
static HintBufs *hint_bufs(tsg_ctx *c, const tsg_csr *a, const tsg_csr *b) {
    std::lock_guard<std::mutex> g(g_hint_mu);
    const HintKey k{c, a->rows, a->cols, a->nnz, b->rows, b->cols, b->nnz};
    auto it = g_hints.find(k);
    if (it != g_hints.end()) return &it->second;
    if (g_hints.size() >= 256) return nullptr;
    HintBufs hb;
    if (cudaHostAlloc(&hb.h, 64 * sizeof(int64_t), cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer(&hb.d, hb.h, 0) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    memset(hb.h, 0, 64 * sizeof(int64_t));
    return &(g_hints[k] = hb);
}

static void plan_device_bins(tsg_ctx *c, const tsg_csr *a, const tsg_csr *b) {
    c->nowait = 0;
    c->c_row_bound = 0;
    c->hint_sym = c->hint_num = c->hintd_sym = c->hintd_num = nullptr;
    // opt-in (TSG_DEVICE_BINS=1): measured on config 2 the removed host
    // round trips (~25 us of idle per step) were outweighed by slower bin
    // kernels (the device-side range prologue per block, the extra leftover
    // launch): 1.197 ms per step read-back vs 1.212-1.220 device-driven;
    // config 1 0.176 vs 0.181 ms
    static const bool enabled =
        (getenv("TSG_DEVICE_BINS") || getenv("TSG_GRAPHS")) && !getenv("TSG_NO_DEVICE_BINS");
    if (c->c_host_out || !(enabled || c->capture_owned)) return;
    const int64_t amax = a->max_row >= 0 ? a->max_row : (a->max_row_bound > 0 ? a->max_row_bound : -1);
    const int64_t bmax = b->max_row;
    if (amax <= 0 || bmax <= 0 || a->rows <= 0 || b->rows <= 0) return;
    const int64_t sbmax = amax * bmax;              // sets per row <= entries of its B rows
    const int64_t nmax = std::min<int64_t>(sbmax, b->cols);
    if (sbmax >= DENSE_MIN_SETS || sym_bin(sbmax) >= 7 || num_bin(nmax, nmax) >= 7) return;
    const int64_t anz = a->nnz;                     // a bound when `a` is itself lazy
    const int64_t bound = anz * bmax;
    const int64_t nnz_bound = std::min<int64_t>(bound, a->rows * b->cols);
    if (12 * (bound + nnz_bound) > ((int64_t)12 << 30)) return;
    uint32_t sym = 0, num = 0;
    for (int k = 0; k <= sym_bin(sbmax); ++k) sym |= 1u << k;
    for (int k = 0; k <= num_bin(nmax, nmax); ++k) num |= 1u << k;
    // merge tier (row-sorted B): bin m holds rows with <= mt_g(m) entries
    // whose bound <= mt_cap(m) that no smaller m took
    sym |= 1u << BIN_MERGE;
    if (amax > mt_g(0) || sbmax > mt_cap(0)) sym |= 1u << (BIN_MERGE + 1);
    if (amax > mt_g(1) || sbmax > mt_cap(1)) sym |= 1u << (BIN_MERGE + 2);
    if (bmax <= 1) sym |= 1u << BIN_THREAD;         // unit B: thread tier
    c->sym_possible = sym;
    c->num_possible = num;
    c->set_cap_bound = std::max<int64_t>(bound, 1);
    c->nnz_bound = nnz_bound;
    c->c_row_bound = nmax;
    // the first multiply of a shape reads its bin sizes back (and records
    // them); later ones run device-driven with those sizes as launch hints
    HintBufs *hb = hint_bufs(c, a, b);
    if (!hb) return;
    c->hint_sym = hb->h;
    c->hintd_sym = hb->d;
    c->hint_num = hb->h + 32;
    c->hintd_num = hb->d + 32;
    if (hb->h[31] == 1 && hb->h[63] == 1) {
        c->nowait = 1;
    } else {
        hb->h[31] = hb->h[63] = 1;   // the read-back partitions below fill the starts
    }
}

// ---- multiply plans: a repeated multiply of the same operands replays a
// CUDA graph of its device-driven form (opt-in, TSG_GRAPHS=1).  A plan keeps
// two captured graphs with their own output arrays and temporaries (every
// block the capture touched belongs to the plan), so the result of the
// previous call may stay alive while the next one is computed; a call that
// finds both outputs still in use runs the ordinary path.  Plans are keyed by
// operand identity and dropped when an operand is freed or changed
// (tsg_plans_forget).  The replay launches every kernel of compress ->
// symbolic -> numeric with no host involvement.  Measured on config 1 (A*A,
// 256^2): 0.184 ms per replay vs 0.169 ms for the ordinary path (with or
// without programmatic launch edges, with or without the forked bins) --
// the host was not the bound; the ~16 dependent kernels and the
// device-driven form's slower bins are.  So it stays opt-in.
struct MulPlan {
    tsg_ctx *c;
    const tsg_csr *a, *b;
    cudaGraphExec_t exec[2] = {nullptr, nullptr};
    tsg_csr out[2];
    bool busy[2] = {false, false};
    std::vector<void *> owned[2];
    int64_t launches[2] = {0, 0};
    int rk[2] = {-1, -1};
    bool dead = false;
};
static std::mutex g_plan_mu;
static std::vector<MulPlan *> g_plans;

static void plan_destroy(MulPlan *pl) {
    cudaStreamSynchronize(pl->c->stream);
    for (int k = 0; k < 2; ++k) {
        if (pl->exec[k]) cudaGraphExecDestroy(pl->exec[k]);
        std::sort(pl->owned[k].begin(), pl->owned[k].end());
        pl->owned[k].erase(std::unique(pl->owned[k].begin(), pl->owned[k].end()), pl->owned[k].end());
        tsg_arena_return(pl->c, pl->owned[k]);
    }
    delete pl;
}

void tsg_plans_forget(tsg_ctx *c, const tsg_csr *m) {
    std::vector<MulPlan *> drop;
    {
        std::lock_guard<std::mutex> g(g_plan_mu);
        for (auto it = g_plans.begin(); it != g_plans.end();) {
            MulPlan *pl = *it;
            if (pl->c == c && (pl->a == m || pl->b == m)) {
                pl->dead = true;
                it = g_plans.erase(it);
                if (!pl->busy[0] && !pl->busy[1]) drop.push_back(pl);
            } else {
                ++it;
            }
        }
    }
    for (MulPlan *pl : drop) plan_destroy(pl);
}

void tsg_plan_release_slot(void *plan, int slot) {
    MulPlan *pl = static_cast<MulPlan *>(plan);
    bool destroy;
    {
        std::lock_guard<std::mutex> g(g_plan_mu);
        pl->busy[slot] = false;
        destroy = pl->dead && !pl->busy[0] && !pl->busy[1];
    }
    if (destroy) plan_destroy(pl);
}

static int multiply_body(tsg_ctx *c, const tsg_csr *a, const tsg_csr *b, tsg_csr **out);
static int multiply_small(tsg_ctx *c, const tsg_csr *a, const tsg_csr *b, int64_t bound, tsg_csr **out);

// capture slot `k` of a plan: the device-driven multiply recorded into a graph
static int plan_capture(tsg_ctx *c, MulPlan *pl, int k) {
    std::vector<void *> owned;
    const int timing = c->timing;
    const int64_t l0 = c->launches;
    c->capture_owned = &owned;
    c->capture_failed = 0;
    c->capture_timing = timing;
    c->capture_rk = -1;
    c->timing = 0;
    tsg_csr *C = nullptr;
    int s = TSG_OK;
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        plan_device_bins(c, pl->a, pl->b);
        if (!c->nowait) s = TSG_EARG;   // the read-back path cannot be captured
        if (s == TSG_OK) s = multiply_body(c, pl->a, pl->b, &C);
        e = cudaStreamEndCapture(c->stream, &g);
    }
    c->capture_owned = nullptr;
    c->capture_timing = 0;
    c->timing = timing;
    pl->owned[k] = owned;
    pl->launches[k] = c->launches - l0;
    c->launches = l0;
    pl->rk[k] = c->capture_rk;
    if (e != cudaSuccess || s != TSG_OK || c->capture_failed || !C) {
        cudaGetLastError();
        if (g) cudaGraphDestroy(g);
        if (C) delete C;
        tsg_set_error("multiply plan capture failed");
        return TSG_EARG;
    }
    e = cudaGraphInstantiate(&pl->exec[k], g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
        cudaGetLastError();
        delete C;
        tsg_set_error("multiply plan instantiation failed");
        return TSG_EARG;
    }
    pl->out[k] = *C;
    delete C;
    return TSG_OK;
}

static int plan_replay(tsg_ctx *c, MulPlan *pl, int k, tsg_csr **out) {
    TSG_CK(cudaGraphLaunch(pl->exec[k], c->stream));
    c->launches += pl->launches[k];
    if (pl->rk[k] >= 0 && c->timing) {
        c->ring_timed[pl->rk[k]] = c->num_calls;
    }
    ++c->num_calls;
    c->pending = "numeric";
    tsg_csr *C = new tsg_csr(pl->out[k]);
    C->plan = pl;
    C->plan_slot = k;
    C->lazy_nnz = 1;
    C->owner = c;
    pl->busy[k] = true;
    *out = C;
    return TSG_OK;
}

// A plan for (a, b): replay a free slot, or capture one for an operand pair
// seen before (its bin sizes are known: the device-driven form applies);
// returns TSG_EARG when the ordinary path should run instead.
static int plan_multiply(tsg_ctx *c, const tsg_csr *a, const tsg_csr *b, tsg_csr **out) {
    static const bool enabled = getenv("TSG_GRAPHS") != nullptr;
    if (!enabled || c->c_host_out || c->capture_owned) return TSG_EARG;
    MulPlan *pl = nullptr;
    {
        std::lock_guard<std::mutex> g(g_plan_mu);
        for (MulPlan *p : g_plans)
            if (p->c == c && p->a == a && p->b == b) pl = p;
    }
    if (pl) {
        for (int k = 0; k < 2; ++k)
            if (pl->exec[k] && !pl->busy[k]) return plan_replay(c, pl, k, out);
        if (!pl->exec[1]) {
            if (plan_capture(c, pl, 1) != TSG_OK) return TSG_EARG;
            return plan_replay(c, pl, 1, out);
        }
        return TSG_EARG;   // both outputs still held by the caller
    }
    // the first multiply of an operand pair records the bin sizes (ordinary
    // path); the second captures
    HintBufs *hb = hint_bufs(c, a, b);
    if (!hb || hb->h[31] != 1 || hb->h[63] != 1) return TSG_EARG;
    pl = new MulPlan();
    pl->c = c;
    pl->a = a;
    pl->b = b;
    if (plan_capture(c, pl, 0) != TSG_OK) {
        plan_destroy(pl);
        return TSG_EARG;
    }
    {
        std::lock_guard<std::mutex> g(g_plan_mu);
        g_plans.push_back(pl);
    }
    return plan_replay(c, pl, 0, out);
}

extern "C" int tsg_multiply(tsg_ctx *c, const tsg_csr *a, const tsg_csr *b, tsg_csr **out) {
    TSG_RESOLVE(c, b);
    if (a->cols != b->rows) {
        tsg_set_error("A is %lldx%lld but B has %lld rows", (long long)a->rows, (long long)a->cols,
                      (long long)b->rows);
        return TSG_EDIM;
    }
    if (!a->val || !b->val) {
        tsg_set_error("numeric multiply requires values on both operands");
        return TSG_EVALID;
    }
    if (plan_multiply(c, a, b, out) == TSG_OK) return TSG_OK;
    // Device-driven path: when the host's row-length bounds keep every row in
    // the group / merge / thread tiers and the bounded allocations are small,
    // the multiply never waits for the device (no partition read-backs, C's
    // nnz left on the device) -- back-to-back multiplies queue without gaps.
    // small products: the symbolic-free path (multiply_small), opt-in
    // (TSG_SMALL_PATH=1): config 1's device span 0.167 -> 0.160 ms, but the
    // host wall per multiply 141 -> 157 us synchronised, 117 -> 142 us
    // pipelined (tools/c1_host.py) -- more host work per call than it saves
    static const bool small_on = getenv("TSG_SMALL_PATH") != nullptr;
    if (small_on && !c->c_host_out && !c->capture_owned && a->rows > 0 && a->rows <= ((int64_t)1 << 20) &&
        b->max_row >= 0 && a->nnz > 0) {
        const int64_t bound = a->nnz * std::max<int64_t>(b->max_row, 1);
        if (bound <= ((int64_t)4 << 20)) return multiply_small(c, a, b, bound, out);
    }
    plan_device_bins(c, a, b);
    return multiply_body(c, a, b, out);
}

// C rows from padded rows (capacity = the row's multiplications) to CSR
__global__ void k_compact_rows(int64_t rows, const int64_t *__restrict__ pptr, const int32_t *__restrict__ plen,
                               const int64_t *__restrict__ cptr, const int32_t *__restrict__ pcol,
                               const double *__restrict__ pval, int32_t *__restrict__ ccol,
                               double *__restrict__ cval) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w; i < rows; i += nw) {
        const int64_t s = pptr[i], d = cptr[i];
        const int n = plen[i];
        for (int q = lane; q < n; q += 32) {
            ccol[d + q] = pcol[s + q];
            cval[d + q] = pval[s + q];
        }
    }
}

// Small products (config-1 sized): no symbolic phase.  Every row of C is
// built at a capacity of its multiplications by the fused in-place numeric
// step (the chunked executors' kernels: same union, same ordered values, C
// columns ascending), its length comes back per row, and one scan + copy
// compacts the rows.  One partition read-back instead of two, no symbolic
// kernels; C's nnz stays on the device (lazy, like the device-driven path).
static int multiply_small(tsg_ctx *c, const tsg_csr *a, const tsg_csr *b, int64_t bound, tsg_csr **out) {
    const int64_t rows = a->rows;
    tsg_cmat *cb = nullptr;
    TSG_TRY(tsg_compress_impl(c, b, &cb));
    int64_t *flops = nullptr, *pptr = nullptr;
    int32_t *plen = nullptr, *pcol = nullptr;
    double *pval = nullptr;
    int st = tsg_alloc_t(c, &flops, rows + 1);
    if (st == TSG_OK) st = tsg_alloc_t(c, &pptr, rows + 1);
    if (st == TSG_OK) st = tsg_alloc_t(c, &plen, rows + 1);
    if (st == TSG_OK) st = tsg_alloc_t(c, &pcol, bound + 1);
    if (st == TSG_OK) st = tsg_alloc_t(c, &pval, bound + 1);
    tsg_csr *C = nullptr;
    if (st == TSG_OK) {
        launch_bounds(c, a, b->rp, nullptr, flops, nullptr, nullptr);
        st = tsg_exclusive_scan_i64(c, flops, pptr, rows);
    }
    if (st == TSG_OK) st = tsg_fill(c, plen, 0, (rows + 1) * sizeof(int32_t), c->stream);
    if (st == TSG_OK)
        st = tsg_fused_inplace(c, a, 0, 0x7fffffff, b, cb, pptr, flops, pcol, pval, plen, rows);
    if (st == TSG_OK) {
        C = new tsg_csr();
        C->max_row = -1;
        C->rows = rows;
        C->cols = b->cols;
        C->nnz = bound;   // capacity; the exact count is rp[rows] on the device
        C->lazy_nnz = 1;
        C->owner = c;
        C->sorted = 1;
        C->distinct = 1;
        st = tsg_alloc_t(c, &C->rp, rows + 1);
        if (st == TSG_OK) st = tsg_alloc_t(c, &C->col, bound + 1);
        if (st == TSG_OK) st = tsg_alloc_t(c, &C->val, bound + 1);
        if (st == TSG_OK) st = tsg_exclusive_scan_i32_to_i64(c, plen, C->rp, rows);
        if (st == TSG_OK) {
            k_compact_rows<<<grid_for(rows, 8, c->num_sms * 16), 256, 0, c->stream>>>(rows, pptr, plen, C->rp, pcol,
                                                                                   pval, C->col, C->val);
            ++c->launches;
            if (cudaGetLastError() != cudaSuccess) st = TSG_ECUDA;
        }
        if (st != TSG_OK) {
            tsg_csr_free(c, C);
            C = nullptr;
        }
    }
    tsg_free(c, flops);
    tsg_free(c, pptr);
    tsg_free(c, plen);
    tsg_free(c, pcol);
    tsg_free(c, pval);
    tsg_cmat_free(c, cb);
    if (st == TSG_OK) *out = C;
    ++c->num_calls;
    return st;
}

static int multiply_body(tsg_ctx *c, const tsg_csr *a, const tsg_csr *b, tsg_csr **out) {
    PhaseTimer pt(c);
    pt.mark();
    tsg_trace(c, "multiply:start", a->rows);
    tsg_cmat *cb = nullptr;
    TSG_TRY(tsg_compress_impl(c, b, &cb));
    tsg_trace(c, "multiply:compressed", b->nnz);
    pt.mark();
    tsg_vec *counts = nullptr;
    int64_t *sbound = nullptr;
    int s = tsg_symbolic_impl(c, a->rows, a, 0, 0, 0x7fffffff, cb, nullptr, &counts, &sbound);
    tsg_trace(c, "multiply:symbolic", 0);
    pt.mark();
    if (s == TSG_OK)
        s = tsg_numeric_impl(c, a->rows, b->cols, a, 0, 0, 0x7fffffff, b, cb, nullptr, counts, sbound,
                             out, &pt);
    c->nowait = 0;
    c->c_row_bound = 0;
    c->hint_sym = c->hint_num = c->hintd_sym = c->hintd_num = nullptr;
    pt.finish(5);
    // phase slots: [0] compress [1] symbolic [2] scan [3] numeric [5] total
    tsg_free(c, sbound);
    tsg_vec_free(c, counts);
    tsg_cmat_free(c, cb);
    return s;
}

extern "C" int tsg_multiply_placed(tsg_ctx *c, const tsg_csr *a, const tsg_csr *b, int c_in_host,
                                   tsg_csr **out) {
    c->c_host_out = c_in_host ? 1 : 0;
    int s = tsg_multiply(c, a, b, out);
    c->c_host_out = 0;
    return s;
}

extern "C" int tsg_numeric_fused(tsg_ctx *c, const tsg_csr *a, const tsg_csr *b_chunk,
                                 const tsg_csr *c_partial, int64_t a_lo, int64_t a_hi,
                                 int64_t b_lo, int64_t b_hi, tsg_csr **out) {
    TSG_RESOLVE(c, a);
    TSG_RESOLVE(c, b_chunk);
    TSG_RESOLVE(c, c_partial);
    if (a_hi > a->rows || a_lo < 0 || a_lo > a_hi) {
        tsg_set_error("a_rows exceeds A's row count");
        return TSG_EDIM;
    }
    if (b_hi > a->cols || b_lo < 0 || b_lo > b_hi) {
        tsg_set_error("b_rows exceeds A's column count");
        return TSG_EDIM;
    }
    if (b_chunk->rows != b_hi - b_lo) {
        tsg_set_error("b_chunk must hold exactly the b_rows rows");
        return TSG_EDIM;
    }
    if (c_partial->rows != a_hi - a_lo) {
        tsg_set_error("c_partial must cover exactly the a_rows rows");
        return TSG_EDIM;
    }
    if (c_partial->cols != b_chunk->cols) {
        tsg_set_error("c_partial and b_chunk column spaces differ");
        return TSG_EDIM;
    }
    if (!a->val || !b_chunk->val || !c_partial->val) {
        tsg_set_error("fused multiply requires numeric operands");
        return TSG_EVALID;
    }
    int64_t rows_out = a_hi - a_lo;
    tsg_cmat *cb = nullptr;
    TSG_TRY(tsg_compress_impl(c, b_chunk, &cb));
    tsg_vec *counts = nullptr;
    int64_t *sbound = nullptr;
    int s = tsg_symbolic_impl(c, rows_out, a, a_lo, (int32_t)b_lo, (int32_t)b_hi, cb, c_partial,
                              &counts, &sbound);
    if (s == TSG_OK) s = tsg_check_kernel_errors(c, "fused symbolic");
    if (s == TSG_OK)
        s = tsg_numeric_impl(c, rows_out, b_chunk->cols, a, a_lo, (int32_t)b_lo, (int32_t)b_hi,
                             b_chunk, cb, c_partial, counts, sbound, out, nullptr);
    tsg_free(c, sbound);
    tsg_vec_free(c, counts);
    tsg_cmat_free(c, cb);
    return s;
}

const void *tsg_kernel_spgemm() { return (const void *)k_max_i32; }
