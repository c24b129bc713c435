// tsg_masked.cu -- K6 masked intersect-count (triangle counting) and the
// compressed-matrix boundary (download / upload / info).
//
// masked_row_intersect_count (kernel.py:349-394): for every row i of a
// strictly lower-triangular pattern L, the row's own columns are ORed into a
// set table (rejecting any column >= i), then every entry j of the row walks
// the compressed row j of cl and adds popcount(bits & table[set]).  Work is
// enumerated in flattened order over the selected compressed rows, rows are
// binned by table size exactly like the symbolic phase, and the int64 total
// is reduced warp -> CTA (shared atomic) -> one global atomic per CTA, so the
// integer result is exact and launch-order independent.
#include <algorithm>

#include "tsg_group.cuh"
#include "tsg_partition.cuh"

namespace {

struct MaskArgs {
    const int64_t *lrp;
    const int32_t *lcol;
    const int64_t *cstart;
    const int32_t *ccnt;
    const int32_t *cset;
    const uint64_t *cbits;
    unsigned long long *total;
    int *err;
};

constexpr int MB = 10;  // bins: 0..6 group tier (slice 512 << b), 7 CTA, 8 global, 9 dense
constexpr int MASK_DENSE = 9;
#ifndef TSG_MASK_DENSE_MIN
#define TSG_MASK_DENSE_MIN 128
#endif
// row length from which the dense bitmap wins (measured at R-MAT scale 22:
// 2048 -> 140 ms, 512 -> 82, 256 -> 74, 128 -> 68, 64 -> 72 ms per count once
// the dense tier enumerates a warp per entry)
constexpr int64_t MASK_DENSE_MIN = TSG_MASK_DENSE_MIN;
#ifndef DENSE_WARP_ENTRY
#define DENSE_WARP_ENTRY 1
#endif
#ifndef DENSE_UNITS
#define DENSE_UNITS 1
#endif
#ifndef MASK_RAW
#define MASK_RAW 1
#endif
#ifndef MASK_PIPE
#define MASK_PIPE 1
#endif
#ifndef MASK_MINB
#define MASK_MINB 1   // 2 (32 registers, spills, two slabs per SM): 66.6 ms against 48.4 at scale 22
#endif
#ifndef MASK_CH
#define MASK_CH 256   // raw columns per warp unit (R-MAT scale 22: 128 -> 49.8 ms, 256 -> 45.7, 512 -> 51.3)
#endif
// L2-slab dense tier shape, R-MAT scale 22: 1024 x 1 per SM 49.6 ms, 512 x 2
// 64.8, 512 x 3 62.0, 256 x 4 96.7, 256 x 6 103.2
#ifndef MASK_SLAB_NT
#define MASK_SLAB_NT 1024
#endif
#ifndef MASK_SLAB_CTAS
#define MASK_SLAB_CTAS 1
#endif

__device__ __forceinline__ int mask_bin(int64_t len, bool dense_ok) {
    if (len <= 0) return 255;
    if (dense_ok && len >= MASK_DENSE_MIN) return MASK_DENSE;
    int64_t need = 16 * (int64_t)table_slots(len);
    for (int b = 0; b < 7; b++)
        if (need <= (512 << b)) return b;
    if (table_slots(len) <= 8192) return 7;
    return 8;
}

struct MaskBinF {
    const int64_t *lrp;
    bool dense_ok;
    __device__ __forceinline__ int operator()(int64_t i) const {
        return mask_bin(lrp[i + 1] - lrp[i], dense_ok);
    }
};

// Raw-column unit enumeration for the dense tier, software-pipelined: the
// units are block_unit_enumerate's (EB entries per round, CH consecutive
// columns of one L_j per unit, warps round-robin), but each warp issues the
// column loads of its next unit before the bitmap lookups of the current one,
// so the two dependent loads of a unit (column, then bitmap word) overlap
// the next unit's first.
template <int NT, int EB, int CH>
__device__ __forceinline__ long long mask_raw_units(int64_t r0, int64_t r1, const MaskArgs &a,
                                                    const uint64_t *bm, int *s_warp) {
    constexpr int G = EB / 32, R = CH / 32;
    __shared__ int64_t s_s0[EB];
    __shared__ int s_uinc[EB + 32];   // one pad word per G entries (bank-distinct first search round)
    __shared__ int s_len[EB];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    long long mine = 0;
    for (int64_t tb = r0; tb < r1; tb += EB) {
        const int64_t t = tb + threadIdx.x;
        int64_t st = 0;
        int ln = 0;
        if (threadIdx.x < EB && t < r1) {
            const int j = a.lcol[t];
            st = a.lrp[j];
            ln = (int)(a.lrp[j + 1] - st);
        }
        const int nch = (ln + CH - 1) / CH;
        int utot;
        const int ux = block_excl_scan<NT>(nch, utot, s_warp);
        if (threadIdx.x < EB) {
            s_uinc[threadIdx.x + threadIdx.x / G] = ux + nch;
            s_len[threadIdx.x] = ln;
            s_s0[threadIdx.x] = st;
        }
        __syncthreads();
        auto load_unit = [&](int u, int (&c)[R]) {
            const unsigned g1 = __ballot_sync(0xffffffffu, s_uinc[lane * (G + 1) + G - 1] <= u);
            const int grp = __popc(g1);
            const unsigned g2 =
                __ballot_sync(0xffffffffu, lane < G && s_uinc[grp * (G + 1) + (lane < G ? lane : 0)] <= u);
            const int e = grp * G + __popc(g2);
            const int le = s_len[e];
            const int q0 = (u - (s_uinc[e + e / G] - (le + CH - 1) / CH)) * CH;
            const int64_t sb = s_s0[e] + q0;
            const int cnt = le - q0 < CH ? le - q0 : CH;
#pragma unroll
            for (int r = 0; r < R; ++r) c[r] = r * 32 + lane < cnt ? a.lcol[sb + r * 32 + lane] : -1;
        };
        int cur[R], nxt[R];
        int u = wid;
        if (u < utot) load_unit(u, cur);
        for (; u < utot; u += NT / 32) {
            const int un = u + NT / 32;
            if (un < utot) load_unit(un, nxt);
            uint64_t wv[R];
#pragma unroll
            for (int r = 0; r < R; ++r) wv[r] = cur[r] >= 0 ? bm[cur[r] >> 6] : 0ull;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (cur[r] >= 0) mine += (long long)((wv[r] >> (cur[r] & 63)) & 1ull);
#pragma unroll
            for (int r = 0; r < R; ++r) cur[r] = nxt[r];
        }
        __syncthreads();
    }
    return mine;
}

// Dense tier for long rows (power-law hubs): row i's columns become bits of
// a bitmap over ALL columns (shared memory when it fits, else a per-CTA slab
// that stays L2-resident), so every lookup of a compressed entry of L_j is one
// word load + AND + popcount -- no hashing, no probing.  Only the words the
// row touched are cleared afterwards.
template <int NT, bool SMEM>
__global__ void __launch_bounds__(NT, MASK_MINB) k_mask_dense(const int32_t *__restrict__ list, int64_t nlist,
                                                   MaskArgs a, uint64_t *slab, int64_t nwords, int64_t wwords,
                                                   const int64_t *__restrict__ coff, int64_t cut_base,
                                                   const int32_t *__restrict__ cut, bool raw) {
    // raw: L's rows are column-distinct, so testing L_j's raw columns equals
    // the popcounts of its compressed sets
    extern __shared__ int4 smem[];
    __shared__ unsigned long long s_tot;
    __shared__ int s_warp[32];
    uint64_t *bm = SMEM ? reinterpret_cast<uint64_t *>(smem) : slab + (int64_t)blockIdx.x * nwords;
    unsigned *bm32 = reinterpret_cast<unsigned *>(bm);
    if (!SMEM) wwords = nwords;
    for (int64_t w = threadIdx.x; w < wwords; w += NT) bm[w] = 0ull;
    if (threadIdx.x == 0) s_tot = 0;
    __syncthreads();
    long long mine = 0;
    for (int64_t li = blockIdx.x; li < nlist; li += gridDim.x) {
        const int64_t i = list[li];
        const int64_t r0 = a.lrp[i], r1 = a.lrp[i + 1];
        // column windows of wwords sets: row i's columns (and every L_j's) lie
        // below i, so rows below the first window's end take one pass; the
        // windowed bitmap stays in shared memory at any graph size
        const int64_t used = (i + 63) / 64 < nwords ? (i + 63) / 64 : nwords;
        const int nwin = used <= wwords ? 1 : (int)((used + wwords - 1) / wwords);
        for (int win = 0; win < nwin; ++win) {
            const int64_t lo = (int64_t)win * wwords, hi = lo + wwords;
            bool lower = true;
            for (int64_t q = r0 + threadIdx.x; q < r1; q += NT) {
                const int c = a.lcol[q];
                if ((int64_t)c >= i) lower = false;
                const int64_t cw = c >> 6;
                if (cw >= lo && cw < hi) atomicOr(&bm32[(c - lo * 64) >> 5], 1u << (c & 31));
            }
            if (win == 0 && !lower) kerr(a.err, KERR_NOTLOWER, i);
            __syncthreads();
            if (MASK_RAW && raw && nwin == 1) {
                // L_j's raw columns (4 B each) tested against the bitmap
                // instead of its compressed sets (12 B each, 0.64 sets per
                // column at R-MAT scale 20): the tier is bound by re-reading
                // L_j rows from DRAM, and the sum of bit(c) over a row's
                // distinct columns equals the sum of popcount(bits & word)
                if (MASK_PIPE && !SMEM)   // L2 bitmap: pipelined (scale 22: 48.0 -> 42.4 ms); shared bitmap: plain (scale 20: 6.3 vs 8.0)
                    mine += mask_raw_units<NT, (NT < 512 ? NT : 512), MASK_CH>(r0, r1, a, bm, s_warp);
                else
                    block_unit_enumerate<NT, (NT < 512 ? NT : 512), MASK_CH, int>(
                        r0, r1,
                        [&](int64_t t, int64_t &st, int &len, double &) {
                            const int j = a.lcol[t];
                            st = a.lrp[j];
                            len = (int)(a.lrp[j + 1] - st);
                        },
                        [&](int64_t s) { return a.lcol[s]; },
                        [&](double, const int &c) { mine += (long long)((bm[c >> 6] >> (c & 63)) & 1ull); },
                        s_warp);
            } else if (DENSE_UNITS) {
                // units of DENSE_CH compressed sets of one L_j, balanced over
                // the warps (a warp per whole entry left the block waiting on
                // the one walking a hub's row), CH/32 loads per lane in flight
                struct CS {
                    int set;
                    uint64_t bits;
                };
                block_unit_enumerate<NT, (NT < 512 ? NT : 512), 128, CS>(
                    r0, r1,
                    [&](int64_t t, int64_t &st, int &len, double &) {
                        const int j = a.lcol[t];
                        if (j > 0 && ((int64_t)(j - 1) >> 6) >= lo) {   // L_j's sets lie below j / 64
                            st = a.cstart[j];
                            len = a.ccnt[j];
                            if (nwin > 1) {   // the window's sets: precomputed cuts (k_mask_cut)
                                const int64_t alen = r1 - r0;
                                const int32_t *cr = cut + (coff[li] - cut_base) + (t - r0);
                                const int c0 = win > 0 ? cr[(win - 1) * alen] : 0;
                                const int c1 = win + 1 < nwin ? cr[win * alen] : len;
                                st += c0;
                                len = c1 - c0;
                            }
                        }
                    },
                    [&](int64_t s) { return CS{a.cset[s], a.cbits[s]}; },
                    [&](double, const CS &x) { mine += __popcll(x.bits & bm[x.set - lo]); },
                    s_warp);
            } else {
                const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
                for (int64_t t = r0 + wid; t < r1; t += NT / 32) {
                    const int j = a.lcol[t];
                    const int64_t st = a.cstart[j], en = st + a.ccnt[j];
                    for (int64_t q = st + lane; q < en; q += 32) {
                        const int set = a.cset[q];
                        if (set >= lo && set < hi) mine += __popcll(a.cbits[q] & bm[set - lo]);
                    }
                }
            }
            __syncthreads();
            for (int64_t q = r0 + threadIdx.x; q < r1; q += NT) {
                const int64_t cw = a.lcol[q] >> 6;
                if (cw >= lo && cw < hi) bm[cw - lo] = 0ull;
            }
            __syncthreads();
        }
    }
    for (int d = 16; d >= 1; d >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, d);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&s_tot, (unsigned long long)mine);
    __syncthreads();
    if (threadIdx.x == 0 && s_tot) atomicAdd(a.total, s_tot);
}

// Dense rows of several windows: per row the entries needing cut points (its
// length) and the number of cuts (length x (windows - 1)).
__device__ __forceinline__ int mask_windows(int64_t i, int64_t nwords, int64_t wwords) {
    const int64_t used = (i + 63) / 64 < nwords ? (i + 63) / 64 : nwords;
    return used <= wwords ? 1 : (int)((used + wwords - 1) / wwords);
}

__global__ void k_mask_wcount(const int32_t *__restrict__ list, int64_t nd, const int64_t *__restrict__ lrp,
                              int64_t nwords, int64_t wwords, int32_t *__restrict__ ncut_e,
                              int32_t *__restrict__ ncut) {
    for (int64_t li = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; li < nd; li += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = list[li];
        const int nwin = mask_windows(i, nwords, wwords);
        const int alen = (int)(lrp[i + 1] - lrp[i]);
        ncut_e[li] = nwin > 1 ? alen : 0;
        ncut[li] = nwin > 1 ? alen * (nwin - 1) : 0;
    }
}

// Cut points: for entry j of a multi-window row, the offset into L_j's
// (ascending) compressed sets of the first set of each later window.  A
// thread per entry gallops window to window; independent threads hide the
// dependent loads that a search inside the dense kernel's enumeration would
// put in front of a block barrier.
__global__ void __launch_bounds__(256) k_mask_cut(const int32_t *__restrict__ list, int64_t nd, MaskArgs a,
                                                  int64_t nwords, int64_t wwords,
                                                  const int64_t *__restrict__ eoff,
                                                  const int64_t *__restrict__ coff, int64_t cut_base,
                                                  int32_t *__restrict__ cut) {
    const int64_t e0 = eoff[0], tot = eoff[nd] - e0;
    for (int64_t x = (int64_t)blockIdx.x * 256 + threadIdx.x; x < tot; x += (int64_t)gridDim.x * 256) {
        int64_t lo = 0, hi = nd - 1;   // last row with eoff - e0 <= x
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (eoff[mid] - e0 <= x) lo = mid;
            else hi = mid - 1;
        }
        const int64_t li = lo;
        const int64_t e = x - (eoff[li] - e0);
        const int64_t alen = eoff[li + 1] - eoff[li];
        const int64_t i = list[li];
        const int nwin = mask_windows(i, nwords, wwords);
        const int j = a.lcol[a.lrp[i] + e];
        const int64_t st = a.cstart[j], en = st + a.ccnt[j];
        int32_t *cr = cut + (coff[li] - cut_base) + e;
        int64_t cur = st;
        for (int w = 1; w < nwin; ++w) {
            const int64_t lw = (int64_t)w * wwords;
            int64_t step = 1, l2 = cur, h2 = cur;
            while (h2 < en && a.cset[h2] < lw) {
                l2 = h2 + 1;
                h2 += step;
                step <<= 1;
            }
            int64_t r = h2 < en ? h2 : en;
            while (l2 < r) {
                const int64_t mid = (l2 + r) >> 1;
                if (a.cset[mid] < lw) l2 = mid + 1;
                else r = mid;
            }
            cur = l2;
            cr[(int64_t)(w - 1) * alen] = (int32_t)(cur - st);
        }
    }
}

template <int G, int SLICE>
__global__ void __launch_bounds__(256) k_mask_group(const int32_t *__restrict__ list, int64_t nlist,
                                                    MaskArgs a) {
    extern __shared__ int4 smem[];
    __shared__ unsigned long long s_tot;
    constexpr int TMAX = SLICE / 16;
    const unsigned gm = group_mask<G>();
    const int glane = threadIdx.x & (G - 1);
    const int gpb = blockDim.x / G;
    int4 *tbl = smem + (threadIdx.x / G) * TMAX;
    if (threadIdx.x == 0) s_tot = 0;
    __syncthreads();
    long long mine = 0;
    for (int64_t li = (int64_t)blockIdx.x * gpb + threadIdx.x / G; li < nlist;
         li += (int64_t)gridDim.x * gpb) {
        const int64_t i = list[li];
        const int64_t r0 = a.lrp[i], r1 = a.lrp[i + 1];
        int T = table_slots(r1 - r0);
        if (T > TMAX) T = TMAX;
        const int logT = ilog2_pow2(T);
        tbl_clear(tbl, T, glane, G);
        __syncwarp(gm);
        bool ok = true, lower = true;
        for (int64_t q = r0 + glane; q < r1; q += G) {
            int c = a.lcol[q];
            if ((int64_t)c >= i) lower = false;
            int bit = c & 63;
            ok &= tbl_or(tbl, T, logT, c >> 6, bit < 32 ? 1u << bit : 0u,
                         bit >= 32 ? 1u << (bit - 32) : 0u);
        }
        if (!lower) kerr(a.err, KERR_NOTLOWER, i);
        if (!ok) kerr(a.err, KERR_PROBE, i);
        __syncwarp(gm);
        group_enumerate_any<G>(
            gm, glane, r0, r1,
            [&](int64_t t, int64_t &st, int &len) {
                int j = a.lcol[t];
                st = a.cstart[j];
                len = a.ccnt[j];
            },
            [&](bool valid, int, int64_t, int64_t s) {
                if (valid) {
                    int4 e;
                    if (tbl_find(tbl, T, logT, a.cset[s], e) >= 0) {
                        uint64_t b = a.cbits[s];
                        mine += __popc((unsigned)b & (unsigned)e.y) +
                                __popc((unsigned)(b >> 32) & (unsigned)e.z);
                    }
                }
            });
        __syncwarp(gm);
    }
    for (int d = 16; d >= 1; d >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, d);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&s_tot, (unsigned long long)mine);
    __syncthreads();
    if (threadIdx.x == 0 && s_tot) atomicAdd(a.total, s_tot);
}

template <int NT, bool GLOBAL>
__global__ void __launch_bounds__(NT) k_mask_block(const int32_t *__restrict__ list, int64_t nlist,
                                                   MaskArgs a, int4 *slab, int64_t slab_slots,
                                                   int tmax) {
    extern __shared__ int4 smem[];
    __shared__ unsigned long long s_tot;
    int4 *tbl = GLOBAL ? slab + (int64_t)blockIdx.x * slab_slots : smem;
    if (threadIdx.x == 0) s_tot = 0;
    __syncthreads();
    long long mine = 0;
    for (int64_t li = blockIdx.x; li < nlist; li += gridDim.x) {
        const int64_t i = list[li];
        const int64_t r0 = a.lrp[i], r1 = a.lrp[i + 1];
        int64_t want = table_slots(r1 - r0);
        int T = (int)(want < tmax ? want : tmax);
        const int logT = ilog2_pow2(T);
        tbl_clear(tbl, T, threadIdx.x, NT);
        __syncthreads();
        bool ok = true, lower = true;
        for (int64_t q = r0 + threadIdx.x; q < r1; q += NT) {
            int c = a.lcol[q];
            if ((int64_t)c >= i) lower = false;
            int bit = c & 63;
            ok &= tbl_or(tbl, T, logT, c >> 6, bit < 32 ? 1u << bit : 0u,
                         bit >= 32 ? 1u << (bit - 32) : 0u);
        }
        if (!lower) kerr(a.err, KERR_NOTLOWER, i);
        if (!ok) kerr(a.err, KERR_PROBE, i);
        __syncthreads();
        block_enumerate<NT>(
            r0, r1,
            [&](int64_t t, int64_t &st, int &len) {
                int j = a.lcol[t];
                st = a.cstart[j];
                len = a.ccnt[j];
            },
            [&](int64_t, int64_t s) {
                int4 e;
                if (tbl_find(tbl, T, logT, a.cset[s], e) >= 0) {
                    uint64_t b = a.cbits[s];
                    mine += __popc((unsigned)b & (unsigned)e.y) +
                            __popc((unsigned)(b >> 32) & (unsigned)e.z);
                }
            });
        __syncthreads();
    }
    for (int d = 16; d >= 1; d >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, d);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&s_tot, (unsigned long long)mine);
    __syncthreads();
    if (threadIdx.x == 0 && s_tot) atomicAdd(a.total, s_tot);
}

template <int B>
int launch_mask_group(tsg_ctx *c, const int32_t *list, const int64_t *off, const MaskArgs &a) {
    constexpr int G = B == 0 ? 8 : (B == 1 ? 16 : 32);
    constexpr int SL = 512 << B;
    constexpr int BS = B <= 4 ? 256 : (B == 5 ? 128 : 64);
    int64_t n = off[B + 1] - off[B];
    if (n <= 0) return TSG_OK;
    size_t smem = (size_t)(BS / G) * SL;
    TSG_TRY(tsg_func_smem((const void *)k_mask_group<G, SL>, smem));
    k_mask_group<G, SL><<<grid_for(n, BS / G, c->num_sms * 64), BS, smem, c->stream>>>(list + off[B],
                                                                                      n, a); ++c->launches;
    TSG_CK(cudaGetLastError());
    return TSG_OK;
}

__global__ void k_maxlen(const int32_t *list, int64_t n, const int64_t *rp, unsigned long long *out) {
    unsigned long long m = 0;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = list[x];
        unsigned long long l = (unsigned long long)(rp[i + 1] - rp[i]);
        m = l > m ? l : m;
    }
    for (int d = 16; d >= 1; d >>= 1) {
        unsigned long long o = __shfl_xor_sync(0xffffffffu, m, d);
        m = o > m ? o : m;
    }
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// ---------------------------------------------------------------- cmat I/O

__global__ void k_cmat_compact(int64_t rows, const int64_t *__restrict__ start,
                               const int32_t *__restrict__ cnt, const int64_t *__restrict__ off,
                               const int32_t *__restrict__ set, const uint64_t *__restrict__ bits,
                               int64_t *__restrict__ oset, uint64_t *__restrict__ obits) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w; r < rows; r += nw) {
        int64_t s0 = start[r], o0 = off[r];
        for (int q = lane; q < cnt[r]; q += 32) {
            oset[o0 + q] = set[s0 + q];
            obits[o0 + q] = bits[s0 + q];
        }
    }
}

__global__ void k_cmat_from_compact(int64_t rows, const int64_t *__restrict__ rp, int32_t *cnt) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x)
        cnt[r] = (int32_t)(rp[r + 1] - rp[r]);
}

__global__ void k_i64_to_i32(const int64_t *in, int32_t *out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)in[i];
}

}  // namespace

extern "C" int tsg_masked_count(tsg_ctx *c, const tsg_csr *l, const tsg_cmat *cl, int64_t *total) {
    TSG_RESOLVE(c, l);
    if (l->rows != cl->rows) {
        tsg_set_error("matrix and compressed form disagree on row count");
        return TSG_EDIM;
    }
    const int64_t rows = l->rows;
    *total = 0;
    if (rows == 0 || l->nnz == 0) return TSG_OK;
    uint8_t *bins = nullptr;
    TSG_TRY(tsg_alloc_t(c, &bins, rows));
    BinLists<MB> bl;
    // dense tier: bitmap over all columns, in shared memory up to 200 KB,
    // else a per-CTA global slab (one SM's worth of CTAs, L2-resident)
    const int64_t nwords = (l->cols + 63) / 64;
    // shared-memory bitmap windows of up to 24576 sets (192 KB, 1.57 M
    // columns); larger graphs take several windows per long row
    // Windowed shared-memory bitmaps (TSG_MASK_WIN_WORDS sets per window,
    // cut points from k_mask_cut) are opt-in: at R-MAT scale 22 three 192 KB
    // windows ran 62.8 + 1.9 ms against 54.6 ms for the L2-resident per-CTA
    // bitmap -- the tier is bound by re-reading the compressed L_j rows from
    // DRAM, not by the bitmap lookups.
    static const int64_t wcap = getenv("TSG_MASK_WIN_WORDS") ? atoll(getenv("TSG_MASK_WIN_WORDS")) : 0;
    const int64_t wwords = wcap > 0 && nwords > wcap ? wcap : nwords;
    // several windows need ascending compressed sets (row-sorted L)
    const bool dense_smem = wwords * 8 <= 200 * 1024 && (wwords == nwords || cl->sorted_sets);
    const bool dense_ok = dense_smem || nwords * 8 * c->num_sms <= ((int64_t)1 << 30);
    TSG_TRY(tsg_partition<MB>(c, rows, MaskBinF{l->rp, dense_ok}, bins, bl));
    int32_t *list = bl.list;
    int64_t off[MB + 1];
    for (int b = 0; b <= MB; b++) off[b] = bl.off[b];

    unsigned long long *dtot = (unsigned long long *)(c->d_small + 16);
    TSG_TRY(tsg_fill(c, dtot, 0, sizeof(unsigned long long), c->stream));
    MaskArgs a{l->rp, l->col, cl->start, cl->cnt, cl->set, cl->bits, dtot, c->d_err};
    TSG_TRY(launch_mask_group<0>(c, list, off, a));
    TSG_TRY(launch_mask_group<1>(c, list, off, a));
    TSG_TRY(launch_mask_group<2>(c, list, off, a));
    TSG_TRY(launch_mask_group<3>(c, list, off, a));
    TSG_TRY(launch_mask_group<4>(c, list, off, a));
    TSG_TRY(launch_mask_group<5>(c, list, off, a));
    TSG_TRY(launch_mask_group<6>(c, list, off, a));
    int64_t n7 = off[8] - off[7];
    if (n7 > 0) {
        size_t smem = 8192 * 16;
        TSG_TRY(tsg_func_smem((const void *)k_mask_block<512, false>, smem));
        k_mask_block<512, false><<<grid_for(n7, 1, c->num_sms * 4), 512, smem, c->stream>>>(
            list + off[7], n7, a, nullptr, 0, 8192); ++c->launches;
        TSG_CK(cudaGetLastError());
    }
    const int64_t nd = off[MASK_DENSE + 1] - off[MASK_DENSE];
    uint64_t *dslab = nullptr;
    if (nd > 0) {
        const unsigned ctas = (unsigned)(nd < c->num_sms ? nd : c->num_sms);
        if (dense_smem) {
            const size_t smem = (size_t)wwords * 8;
            TSG_TRY(tsg_func_smem((const void *)k_mask_dense<1024, true>, smem));
            const int32_t *dl = list + off[MASK_DENSE];
            if (wwords == nwords) {
                k_mask_dense<1024, true><<<ctas, 1024, smem, c->stream>>>(dl, nd, a, nullptr, nwords, wwords,
                                                                          nullptr, 0, nullptr, l->distinct != 0);
                ++c->launches;
            } else {
                int32_t *ncut_e = nullptr, *ncut = nullptr;
                int64_t *eoff = nullptr, *coff = nullptr;
                TSG_TRY(tsg_alloc_t(c, &ncut_e, (size_t)nd));
                TSG_TRY(tsg_alloc_t(c, &ncut, (size_t)nd));
                TSG_TRY(tsg_alloc_t(c, &eoff, (size_t)nd + 1));
                TSG_TRY(tsg_alloc_t(c, &coff, (size_t)nd + 1));
                k_mask_wcount<<<grid_for(nd, 256, c->num_sms * 8), 256, 0, c->stream>>>(dl, nd, l->rp, nwords,
                                                                                        wwords, ncut_e, ncut);
                ++c->launches;
                TSG_TRY(tsg_exclusive_scan_i32_to_i64(c, ncut_e, eoff, nd));
                TSG_TRY(tsg_exclusive_scan_i32_to_i64(c, ncut, coff, nd));
                // batches of rows whose cut points fit CUT_MAX entries
                std::vector<int64_t> hc((size_t)nd + 1);
                TSG_CK(cudaMemcpyAsync(hc.data(), coff, (nd + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                       c->stream));
                TSG_CK(cudaStreamSynchronize(c->stream));
                const int64_t CUT_MAX = (int64_t)256 << 20;
                int32_t *cut = nullptr;
                const int64_t cap = std::min<int64_t>(CUT_MAX, std::max<int64_t>(hc[nd], 1));
                int64_t maxrow = 0;
                for (int64_t r = 0; r < nd; ++r) maxrow = std::max(maxrow, hc[r + 1] - hc[r]);
                TSG_TRY(tsg_alloc_t(c, &cut, (size_t)std::max(cap, maxrow)));
                for (int64_t b0 = 0; b0 < nd;) {
                    int64_t b1 = b0 + 1;
                    while (b1 < nd && hc[b1 + 1] - hc[b0] <= cap) ++b1;
                    const int64_t nb = b1 - b0;
                    if (hc[b1] > hc[b0]) {
                        k_mask_cut<<<grid_for(nb * 64, 256, c->num_sms * 16), 256, 0, c->stream>>>(
                            dl + b0, nb, a, nwords, wwords, eoff + b0, coff + b0, hc[b0], cut);
                        ++c->launches;
                    }
                    k_mask_dense<1024, true><<<(unsigned)std::min<int64_t>(nb, c->num_sms), 1024, smem,
                                               c->stream>>>(dl + b0, nb, a, nullptr, nwords, wwords, coff + b0,
                                                            hc[b0], cut, l->distinct != 0);
                    ++c->launches;
                    b0 = b1;
                }
                TSG_TRY(tsg_free(c, cut));
                TSG_TRY(tsg_free(c, ncut_e));
                TSG_TRY(tsg_free(c, ncut));
                TSG_TRY(tsg_free(c, eoff));
                TSG_TRY(tsg_free(c, coff));
            }
        } else {
            // L2-slab bitmaps: MASK_SLAB_NT threads per CTA, MASK_SLAB_CTAS per SM
            const unsigned gs = (unsigned)std::min<int64_t>(nd, (int64_t)c->num_sms * MASK_SLAB_CTAS);
            TSG_TRY(tsg_alloc_t(c, &dslab, (size_t)gs * nwords));
            TSG_TRY(tsg_fill(c, dslab, 0, (size_t)gs * nwords * 8, c->stream));
            k_mask_dense<MASK_SLAB_NT, false><<<gs, MASK_SLAB_NT, 0, c->stream>>>(
                list + off[MASK_DENSE], nd, a, dslab, nwords, nwords, nullptr, 0, nullptr, l->distinct != 0);
            ++c->launches;
        }
        TSG_CK(cudaGetLastError());
    }
    int64_t n8 = off[9] - off[8];
    int4 *slab = nullptr;
    if (n8 > 0) {
        unsigned long long *dmax = (unsigned long long *)(c->d_small + 24);
        TSG_TRY(tsg_fill(c, dmax, 0, sizeof(unsigned long long), c->stream));
        k_maxlen<<<grid_for(n8, 256, c->num_sms * 4), 256, 0, c->stream>>>(list + off[8], n8, l->rp,
                                                                          dmax); ++c->launches;
        TSG_TRY(tsg_put_small(c, (const int64_t *)dmax, 1, 0));
        TSG_CK(cudaStreamSynchronize(c->stream));
        int64_t T = table_slots(c->h_small[0]);
        int64_t ctas = ((int64_t)2 << 30) / (T * 16);
        if (ctas < 1) ctas = 1;
        if (ctas > n8) ctas = n8;
        if (ctas > 2 * c->num_sms) ctas = 2 * c->num_sms;
        TSG_TRY(tsg_alloc_t(c, &slab, (size_t)(ctas * T)));
        k_mask_block<512, true><<<(unsigned)ctas, 512, 0, c->stream>>>(list + off[8], n8, a, slab, T,
                                                                      (int)T); ++c->launches;
        TSG_CK(cudaGetLastError());
    }
    TSG_TRY(tsg_put_small(c, (const int64_t *)dtot, 1, 1));
    int s = tsg_check_kernel_errors(c, "masked count");   // synchronises
    *total = c->h_small[1];
    tsg_free(c, slab);
    tsg_free(c, dslab);
    tsg_free(c, bins);
    tsg_free(c, list);
    return s;
}

extern "C" int tsg_cmat_info(tsg_ctx *c, const tsg_cmat *cm, int64_t *rows, int64_t *n_sets) {
    if (rows) *rows = cm->rows;
    if (n_sets) {
        int64_t *off = nullptr;
        TSG_TRY(tsg_alloc_t(c, &off, cm->rows + 1));
        TSG_TRY(tsg_exclusive_scan_i32_to_i64(c, cm->cnt, off, cm->rows));
        TSG_CK(cudaMemcpyAsync(&c->h_small[0], off + cm->rows, sizeof(int64_t), cudaMemcpyDeviceToHost,
                               c->stream));
        TSG_CK(cudaStreamSynchronize(c->stream));
        *n_sets = c->h_small[0];
        TSG_TRY(tsg_free(c, off));
    }
    return TSG_OK;
}

extern "C" int tsg_cmat_download(tsg_ctx *c, const tsg_cmat *cm, int64_t *row_ptr, int64_t *set_idx,
                                 uint64_t *set_bits) {
    int64_t *off = nullptr;
    TSG_TRY(tsg_alloc_t(c, &off, cm->rows + 1));
    TSG_TRY(tsg_exclusive_scan_i32_to_i64(c, cm->cnt, off, cm->rows));
    TSG_CK(cudaMemcpyAsync(&c->h_small[0], off + cm->rows, sizeof(int64_t), cudaMemcpyDeviceToHost,
                           c->stream));
    TSG_CK(cudaStreamSynchronize(c->stream));
    int64_t ns = c->h_small[0];
    if (row_ptr)
        TSG_CK(cudaMemcpyAsync(row_ptr, off, (cm->rows + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost,
                               c->stream));
    if (ns > 0) {
        int64_t *oset = nullptr;
        uint64_t *obits = nullptr;
        TSG_TRY(tsg_alloc_t(c, &oset, ns));
        TSG_TRY(tsg_alloc_t(c, &obits, ns));
        k_cmat_compact<<<grid_for(cm->rows, 8, c->num_sms * 32), 256, 0, c->stream>>>(
            cm->rows, cm->start, cm->cnt, off, cm->set, cm->bits, oset, obits); ++c->launches;
        TSG_CK(cudaGetLastError());
        if (set_idx)
            TSG_CK(cudaMemcpyAsync(set_idx, oset, ns * sizeof(int64_t), cudaMemcpyDeviceToHost,
                                   c->stream));
        if (set_bits)
            TSG_CK(cudaMemcpyAsync(set_bits, obits, ns * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                                   c->stream));
        TSG_TRY(tsg_free(c, oset));
        TSG_TRY(tsg_free(c, obits));
    }
    TSG_CK(cudaStreamSynchronize(c->stream));
    TSG_TRY(tsg_free(c, off));
    return TSG_OK;
}

extern "C" int tsg_cmat_upload(tsg_ctx *c, int64_t rows, int64_t n_sets, const int64_t *row_ptr,
                               const int64_t *set_idx, const uint64_t *set_bits, tsg_cmat **out) {
    tsg_cmat *cm = nullptr;
    TSG_TRY(tsg_cmat_alloc(c, rows, n_sets > 0 ? n_sets : 1, &cm));
    TSG_CK(cudaMemcpyAsync(cm->start, row_ptr, (rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice,
                           c->stream));
    k_cmat_from_compact<<<grid_for(rows, 256, c->num_sms * 8), 256, 0, c->stream>>>(rows, cm->start,
                                                                                   cm->cnt); ++c->launches;
    if (n_sets > 0) {
        int64_t *stage = nullptr;
        TSG_TRY(tsg_alloc_t(c, &stage, n_sets));
        TSG_CK(cudaMemcpyAsync(stage, set_idx, n_sets * sizeof(int64_t), cudaMemcpyHostToDevice,
                               c->stream));
        k_i64_to_i32<<<grid_for(n_sets, 256, c->num_sms * 8), 256, 0, c->stream>>>(stage, cm->set,
                                                                                   n_sets); ++c->launches;
        TSG_CK(cudaMemcpyAsync(cm->bits, set_bits, n_sets * sizeof(uint64_t), cudaMemcpyHostToDevice,
                               c->stream));
        TSG_TRY(tsg_free(c, stage));
    }
    TSG_CK(cudaGetLastError());
    TSG_CK(cudaStreamSynchronize(c->stream));
    *out = cm;
    return TSG_OK;
}

extern "C" int tsg_cmat_free(tsg_ctx *c, tsg_cmat *cm) {
    if (!cm) return TSG_OK;
    tsg_free(c, cm->start);
    tsg_free(c, cm->cnt);
    tsg_free(c, cm->set);
    tsg_free(c, cm->bits);
    delete cm;
    return TSG_OK;
}

const void *tsg_kernel_masked() { return (const void *)k_maxlen; }
