// tsg_group.cuh -- row-group primitives shared by the symbolic, numeric and
// masked-count kernels.
//
// A "group" is G lanes of one warp (G in {8,16,32}) that owns one output row
// at a time, or a whole CTA for big rows.  The group walks the row's work in
// FLATTENED order: for the A entries t of the row (storage order) and, for
// each, the entries s of the B (or compressed-B) row it selects.  Lanes take
// consecutive flattened positions, so a chunk of G positions may straddle
// several A entries; a log2(G)-step shuffle binary search maps a position back
// to its A entry.  This keeps every lane busy whatever the B row lengths are
// (27-entry stencil rows and 1-entry aggregation rows alike) and, because
// lane order == flattened order, lets the numeric kernel reproduce the
// reference's per-column summation order (accumulator.py:101-106) exactly.
#pragma once

#include "tsg_internal.cuh"

// ---------------------------------------------------------------- tables
// slot = int4 {key, mask_lo, mask_hi, base}; key TSG_EMPTY when free.

// Hash-conflict counters (diagnostic builds, -DTSG_PROBE_STATS=1): lookups,
// extra probes of lookups, inserts, extra probes of inserts.  One copy per
// translation unit; tsg_probe_stats() reads tsg_spgemm.cu's (the symbolic and
// numeric group tiers).  Compiled out of the product build.
#ifndef TSG_PROBE_STATS
#define TSG_PROBE_STATS 0
#endif
#if TSG_PROBE_STATS
static __device__ unsigned long long g_tsg_probe[4];
#define TSG_PROBE_COUNT(which, extra)                           \
    do {                                                        \
        atomicAdd(&g_tsg_probe[which], 1ull);                   \
        if (extra) atomicAdd(&g_tsg_probe[(which) + 1], (unsigned long long)(extra)); \
    } while (0)
#else
#define TSG_PROBE_COUNT(which, extra) \
    do {                              \
    } while (0)
#endif

__device__ __forceinline__ void tbl_clear(int4 *tbl, int T, int from, int step) {
    for (int s = from; s < T; s += step) tbl[s] = make_int4(TSG_EMPTY, 0, 0, 0);
}

// insert-or-OR; returns false if the table is full (probe overflow)
__device__ __forceinline__ bool tbl_or(int4 *tbl, int T, int logT, int key, unsigned lo,
                                       unsigned hi) {
    unsigned h = hash_slot(key, logT);
    for (int n = 0; n < T; ++n) {
        int k = *((volatile int *)&tbl[h].x);
        if (k == TSG_EMPTY) {
            k = atomicCAS(&tbl[h].x, TSG_EMPTY, key);
            if (k == TSG_EMPTY) k = key;
        }
        if (k == key) {
            if (lo) atomicOr((unsigned *)&tbl[h].y, lo);
            if (hi) atomicOr((unsigned *)&tbl[h].z, hi);
            TSG_PROBE_COUNT(2, n);
            return true;
        }
        h = (h + 1) & (unsigned)(T - 1);
    }
    return false;
}

// claim a slot for a key known to be absent (distinct keys); -1 if full
__device__ __forceinline__ int tbl_claim(int4 *tbl, int T, int logT, int key) {
    unsigned h = hash_slot(key, logT);
    for (int n = 0; n < T; ++n) {
        if (atomicCAS(&tbl[h].x, TSG_EMPTY, key) == TSG_EMPTY) {
            TSG_PROBE_COUNT(2, n);
            return (int)h;
        }
        h = (h + 1) & (unsigned)(T - 1);
    }
    return -1;
}

// lookup; -1 if absent
__device__ __forceinline__ int tbl_find(const int4 *tbl, int T, int logT, int key, int4 &out) {
    unsigned h = hash_slot(key, logT);
    for (int n = 0; n < T; ++n) {
        int4 e = tbl[h];
        if (e.x == key) {
            out = e;
            TSG_PROBE_COUNT(0, n);
            return (int)h;
        }
        if (e.x == TSG_EMPTY) return -1;
        h = (h + 1) & (unsigned)(T - 1);
    }
    return -1;
}

__device__ __forceinline__ int slot_pop(const int4 &e) {
    return __popc((unsigned)e.y) + __popc((unsigned)e.z);
}

// rank of column `bit` inside a 64-bit set mask (number of lower set bits)
__device__ __forceinline__ int mask_rank(const int4 &e, int bit) {
    // branch-free: pick the half, add the low half's count for high bits
    const unsigned lo = (unsigned)e.y, hi = (unsigned)e.z;
    const bool upper = bit >= 32;
    const unsigned half = upper ? hi : lo;
    const unsigned below = (1u << (bit & 31)) - 1u;
    return (upper ? __popc(lo) : 0) + __popc(half & below);
}

// ---------------------------------------------------------------- enumerate
// src(t, start, len): entries [start, start+len) selected by A entry t
//                     (len = 0 to skip, e.g. outside a B row range).
// f(valid, j, t, s): called by every lane of the group for each chunk; j is
//                 the group lane holding A entry t, s the selected entry.
template <int G, class Src, class F>
__device__ __forceinline__ void group_enumerate(unsigned gm, int glane, int64_t a0, int64_t a1,
                                                Src src, F f) {
    for (int64_t base = a0; base < a1; base += G) {
        int64_t t = base + glane;
        int64_t st = 0;
        int len = 0;
        if (t < a1) src(t, st, len);
        if (__all_sync(gm, len == 1 || t >= a1)) {
            // unit rows (aggregation operators): position p is lane p itself
            f(t < a1, glane, t, st);
            continue;
        }
        int incl = group_incl_scan<G, int>(gm, len, glane);
        int total = __shfl_sync(gm, incl, G - 1, G);
        for (int p0 = 0; p0 < total; p0 += G) {
            int p = p0 + glane;
            int j = 0;
#pragma unroll
            for (int step = G / 2; step >= 1; step >>= 1) {
                int v = __shfl_sync(gm, incl, j + step - 1, G);
                if (v <= p) j += step;
            }
            int inc_j = __shfl_sync(gm, incl, j, G);
            int len_j = __shfl_sync(gm, len, j, G);
            int64_t st_j = __shfl_sync(gm, st, j, G);
            bool valid = p < total;
            f(valid, j, base + j, st_j + (int64_t)(p - (inc_j - len_j)));
        }
    }
}

// Order-free variant (symbolic union, masked count): per chunk of A entries
// it picks the cheaper of the flattened mapping above and a fixed mapping in
// which each A entry gets L = G / pow2(entries) lanes that stride through its
// row -- no search, no shuffles per position.  For uniform rows (stencils:
// 8 A entries x ~11 compressed sets) the fixed mapping needs ~3 steps and no
// binary search; skewed rows (power-law graphs) stay flattened.
template <int G, class Src, class F>
__device__ __forceinline__ void group_enumerate_any(unsigned gm, int glane, int64_t a0, int64_t a1,
                                                    Src src, F f) {
    for (int64_t base = a0; base < a1; base += G) {
        int64_t t = base + glane;
        int64_t st = 0;
        int len = 0;
        if (t < a1) src(t, st, len);
        int incl = group_incl_scan<G, int>(gm, len, glane);
        int total = __shfl_sync(gm, incl, G - 1, G);
        int maxlen = len;
#pragma unroll
        for (int d = G / 2; d >= 1; d >>= 1) maxlen = max(maxlen, __shfl_xor_sync(gm, maxlen, d, G));
        const int ne = (int)((a1 - base) < G ? (a1 - base) : G);
        const int lg_pe = ne <= 1 ? 0 : 32 - __clz(ne - 1);        // log2(pow2 >= ne)
        const int lg_l = ilog2_pow2(G) - lg_pe;                      // lanes per entry = 2^lg_l
        const int steps_fixed = (maxlen + (1 << lg_l) - 1) >> lg_l;
        const int steps_flat = (total + G - 1) / G;
        if (steps_fixed <= 2 * steps_flat) {
            const int j = glane >> lg_l, sub = glane & ((1 << lg_l) - 1);
            int64_t st_j = __shfl_sync(gm, st, j, G);
            int len_j = __shfl_sync(gm, len, j, G);
            if (j >= ne) len_j = 0;
            for (int q = sub; q < (steps_fixed << lg_l); q += (1 << lg_l)) {
                bool valid = q < len_j;
                f(valid, j, base + j, st_j + q);
            }
            continue;
        }
        for (int p0 = 0; p0 < total; p0 += G) {
            int p = p0 + glane;
            int j = 0;
#pragma unroll
            for (int step = G / 2; step >= 1; step >>= 1) {
                int v = __shfl_sync(gm, incl, j + step - 1, G);
                if (v <= p) j += step;
            }
            int inc_j = __shfl_sync(gm, incl, j, G);
            int len_j = __shfl_sync(gm, len, j, G);
            int64_t st_j = __shfl_sync(gm, st, j, G);
            bool valid = p < total;
            f(valid, j, base + j, st_j + (int64_t)(p - (inc_j - len_j)));
        }
    }
}

// Block-wide exclusive scan of one int per thread (NT threads); total out.
template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int &total, int *s_warp) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int o = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += o;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    if (w == 0) {
        int y = lane < NT / 32 ? s_warp[lane] : 0;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int o = __shfl_up_sync(0xffffffffu, y, d);
            if (lane >= d) y += o;
        }
        s_warp[lane] = y;
    }
    __syncthreads();
    int r = x - v + (w ? s_warp[w - 1] : 0);
    total = s_warp[NT / 32 - 1];
    __syncthreads();
    return r;
}

// Block-wide enumeration with a warp per entry: warps take the entries t of
// [a0, a1) in turn and their lanes stride over [st, st + len).  Every
// compressed / B entry costs one coalesced load and no search (the flattened
// block_enumerate below spends ~log2(NT) shared-memory steps per element to
// find its entry); the price is imbalance when one entry's list is much
// longer than the rest.  f(t, s) as in block_enumerate.
template <int NT, class Src, class F>
__device__ __forceinline__ void block_warp_enumerate(int64_t a0, int64_t a1, Src src, F f) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t t = a0 + wid; t < a1; t += NT / 32) {
        int64_t st = 0;
        int len = 0;
        src(t, st, len);
        for (int q = lane; q < len; q += 32) f(t, st + q);
    }
}

// Block-wide enumeration balanced by units, for rows whose entries' lists
// are power-law long (hub rows).  EB entries at a time: src(t, st, len, w)
// for all of them in flight together, each list cut into units of CH
// consecutive elements, warps take units round-robin.  A unit's lanes cover
// consecutive elements of ONE list (so an add / OR instruction never sees two
// lanes on one target from different lists), and each lane issues its CH/32
// loads ld(s) before any apply ap(w, v).  (A warp per whole entry left 31
// warps at the barrier behind the one on a hub's list.)
template <int NT, int EB, int CH, class V, class Src, class Ld, class Ap>
__device__ __forceinline__ void block_unit_enumerate(int64_t a0, int64_t a1, Src src, Ld ld, Ap ap,
                                                     int *s_warp) {
    static_assert(EB <= NT && EB % 32 == 0 && EB <= 1024 && CH % 32 == 0, "unit enumeration shape");
    __shared__ int64_t s_s0[EB];
    __shared__ double s_w[EB];
    // unit prefix per entry, one pad word per G entries: the first search
    // round reads s_uinc[lane * G + G - 1] (stride G, a 16-way bank conflict
    // unpadded: 9 % of the dense numeric kernel's shared wavefronts)
    constexpr int G = EB / 32;
    __shared__ int s_uinc[EB + 32];
    __shared__ int s_len[EB];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t tb = a0; tb < a1; tb += EB) {
        const int64_t t = tb + threadIdx.x;
        int64_t st = 0;
        int ln = 0;
        double w = 0.0;
        if (threadIdx.x < EB && t < a1) src(t, st, ln, w);
        const int nch = (ln + CH - 1) / CH;
        int utot;
        const int ux = block_excl_scan<NT>(nch, utot, s_warp);
        if (threadIdx.x < EB) {
            s_uinc[threadIdx.x + threadIdx.x / G] = ux + nch;
            s_len[threadIdx.x] = ln;
            s_s0[threadIdx.x] = st;
            s_w[threadIdx.x] = w;
        }
        __syncthreads();
        for (int u = wid; u < utot; u += NT / 32) {
            // first entry with s_uinc > u: two ballot rounds over EB / 32
            // groups (a 9-step binary search was a quarter of the instructions)
            const unsigned g1 = __ballot_sync(0xffffffffu, s_uinc[lane * (G + 1) + G - 1] <= u);
            const int grp = __popc(g1);
            const unsigned g2 =
                __ballot_sync(0xffffffffu, lane < G && s_uinc[grp * (G + 1) + (lane < G ? lane : 0)] <= u);
            const int lo = grp * G + __popc(g2);
            const int le = s_len[lo];
            const int q0 = (u - (s_uinc[lo + lo / G] - (le + CH - 1) / CH)) * CH;
            const int64_t sb = s_s0[lo] + q0;
            const int cnt = le - q0 < CH ? le - q0 : CH;
            const double we = s_w[lo];
            V v[CH / 32];
#pragma unroll
            for (int r = 0; r < CH / 32; ++r)
                if (r * 32 + lane < cnt) v[r] = ld(sb + r * 32 + lane);
#pragma unroll
            for (int r = 0; r < CH / 32; ++r)
                if (r * 32 + lane < cnt) ap(we, v[r]);
        }
        __syncthreads();
    }
}

// Block-wide version for one row per CTA (NT threads, NT multiple of 32).
// f(t, s) is called only for valid positions (no collectives inside f).
template <int NT, class Src, class F>
__device__ __forceinline__ void block_enumerate(int64_t a0, int64_t a1, Src src, F f) {
    __shared__ int s_incl[NT];
    __shared__ int s_len[NT];
    __shared__ int64_t s_st[NT];
    __shared__ int s_warp[32];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    for (int64_t base = a0; base < a1; base += NT) {
        int64_t t = base + tid;
        int64_t st = 0;
        int len = 0;
        if (t < a1) src(t, st, len);
        int x = len;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            int o = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += o;
        }
        if (lane == 31) s_warp[w] = x;
        __syncthreads();
        if (w == 0) {
            int y = lane < NT / 32 ? s_warp[lane] : 0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                int o = __shfl_up_sync(0xffffffffu, y, d);
                if (lane >= d) y += o;
            }
            s_warp[lane] = y;
        }
        __syncthreads();
        s_incl[tid] = x + (w ? s_warp[w - 1] : 0);
        s_len[tid] = len;
        s_st[tid] = st;
        int total = s_warp[NT / 32 - 1];
        __syncthreads();
        for (int p = tid; p < total; p += NT) {
            int lo = 0, hi = NT - 1;          // first j with incl[j] > p
            while (lo < hi) {
                int mid = (lo + hi) >> 1;
                if (s_incl[mid] <= p) lo = mid + 1;
                else hi = mid;
            }
            f(base + lo, s_st[lo] + (int64_t)(p - (s_incl[lo] - s_len[lo])));
        }
        __syncthreads();
    }
}
