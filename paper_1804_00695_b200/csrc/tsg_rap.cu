// tsg_rap.cu -- fused Galerkin triple product C = R * A * P (SURVEY.md §8f
// row 4).  The reference (and the config-2 metric) computes RA = R * A and
// then RAP = RA * P as two multiplies; the paper leaves the triple product
// out.  Here a G-lane group owns one row I of C and keeps the row RA_I in
// shared memory instead of writing RA to HBM and reading it back:
//
//   symbolic  union of the compressed A rows of R_I (table 1) -> the columns
//             of RA_I; union of the compressed P rows of those columns
//             (table 2) -> nnz(C_I)
//   numeric   table 1 again, its sets ranked by key -> RA_I's columns in
//             ascending order; RA_I's values accumulated R-entry by R-entry
//             (lanes split an A row: distinct columns, no collisions), then
//             table 2 ranked the same way -> C_I's columns, and the products
//             RA_I[j] * P[j, J] folded per position in RA-entry order by the
//             lane that owns the position (staged window, no match/vote).
//
// Every addition happens in the same order and with the same operands as the
// two-multiply path's group tier (SEQ numeric for R * A, owner-folded or
// ordered products for RA * P, both with -0.0 initial values), so the result
// is bit-identical to tsg_multiply(tsg_multiply(R, A), P) whenever that path
// keeps its rows in the group tier -- the GPU tests check exactly that.  Rows
// that do not fit the per-group slices (or operands without distinct,
// sorted rows) make tsg_rap fall back to the two multiplies.
#include "tsg_group.cuh"

namespace {

constexpr int RG = 8;          // lanes per row
constexpr int RBS = 128;       // threads per CTA
constexpr int RT1 = 32;        // table 1 slots (sets of RA_I)
constexpr int RCRA = 80;       // RA_I columns
constexpr int RT2 = 32;        // table 2 slots (sets of C_I)
constexpr int RCC = 32;        // C_I columns
constexpr int RW = RG;         // staged products per fold window
constexpr int RLOG1 = 5, RLOG2 = 5;   // log2(RT1), log2(RT2)
static_assert((1 << RLOG1) == RT1 && (1 << RLOG2) == RT2, "table sizes");
constexpr int RSLICE = RT1 * 16 + RCRA * 4 + RCRA * 8 + RT2 * 16 + RCC * 8 + RW * 12;

struct RapArgs {
    const int64_t *rrp;
    const int32_t *rcol;
    const double *rval;
    const int64_t *arp;
    const int32_t *acol;
    const double *aval;
    const int64_t *prp;
    const int32_t *pcol;
    const double *pval;
    const int64_t *castart;   // compressed A
    const int32_t *cacnt;
    const int32_t *caset;
    const uint64_t *cabits;
    const int64_t *cpstart;   // compressed P
    const int32_t *cpcnt;
    const int32_t *cpset;
    const uint64_t *cpbits;
    int64_t rows;
    int64_t *counts;          // symbolic out
    const int64_t *cptr;      // numeric in
    int32_t *ccol;
    double *cval;
    int *unfit;               // set when a row does not fit the slices
    int *err;
};

struct RapSlice {
    int4 *t1;
    int32_t *racol;
    double *raval;
    int4 *t2;
    double *cv;
    int *spos;
    double *sprod;
    __device__ RapSlice(char *p) {
        t1 = reinterpret_cast<int4 *>(p);
        t2 = reinterpret_cast<int4 *>(p + RT1 * 16);
        raval = reinterpret_cast<double *>(p + RT1 * 16 + RT2 * 16);
        cv = raval + RCRA;
        sprod = cv + RCC;
        racol = reinterpret_cast<int32_t *>(sprod + RW);
        spos = racol + RCRA;
    }
};

// table 1: OR the compressed A rows selected by R_I's entries; ok = fits
__device__ __forceinline__ bool rap_table1(unsigned gm, int glane, const RapArgs &a, int64_t r0, int64_t r1,
                                           int4 *t1) {
    constexpr int logT = RLOG1;
    tbl_clear(t1, RT1, glane, RG);
    __syncwarp(gm);
    bool ok = true;
    group_enumerate_any<RG>(
        gm, glane, r0, r1,
        [&](int64_t t, int64_t &st, int &len) {
            const int k = a.rcol[t];
            st = a.castart[k];
            len = a.cacnt[k];
        },
        [&](bool valid, int, int64_t, int64_t s) {
            if (valid) {
                const uint64_t bits = a.cabits[s];
                ok &= tbl_or(t1, RT1, logT, a.caset[s], (unsigned)bits, (unsigned)(bits >> 32));
            }
        });
    __syncwarp(gm);
    return __all_sync(gm, ok);
}

// rank the occupied slots of a table by key: slot.w = columns in smaller sets;
// returns the total column count (scratch: >= T int2)
__device__ __forceinline__ int rap_rank(unsigned gm, int glane, int4 *tbl, int T, int2 *scratch) {
    const unsigned lt = lanemask_lt();
    int m = 0, tot = 0;
    for (int r0 = 0; r0 < T; r0 += RG) {
        const int s = r0 + glane;
        const int4 e = s < T ? tbl[s] : make_int4(TSG_EMPTY, 0, 0, 0);
        const bool occ = e.x != TSG_EMPTY;
        const unsigned bal = __ballot_sync(gm, occ) & gm;
        const int pc = slot_pop(e);
        if (occ) scratch[m + __popc(bal & lt)] = make_int2(e.x, (s << 8) | pc);
        if (occ) tot += pc;
        m += __popc(bal);
    }
    tot = group_sum<RG, int>(gm, tot);
    __syncwarp(gm);
    for (int q = glane; q < m; q += RG) {
        const int2 me = scratch[q];
        int base = 0;
        for (int u = 0; u < m; ++u) {
            const int2 o = scratch[u];
            if (o.x < me.x) base += o.y & 0xff;
        }
        tbl[me.y >> 8].w = base;
    }
    __syncwarp(gm);
    return tot;
}

// RA_I's columns into racol (any order): each lane lists its slots' columns
// at offsets from a group scan of their popcounts; returns the count
__device__ __forceinline__ int rap_list_cols(unsigned gm, int glane, const int4 *t1, int32_t *racol) {
    int carry = 0;
    for (int s0 = 0; s0 < RT1; s0 += RG) {
        const int4 e = t1[s0 + glane];
        const int pc = e.x == TSG_EMPTY ? 0 : slot_pop(e);
        const int incl = group_incl_scan<RG, int>(gm, pc, glane);
        int r = carry + incl - pc;
        uint64_t b = pc ? (((uint64_t)(uint32_t)e.z << 32) | (uint32_t)e.y) : 0ull;
        while (b) {
            if (r < RCRA) racol[r] = e.x * 64 + (__ffsll((long long)b) - 1);
            ++r;
            b &= b - 1;
        }
        carry += __shfl_sync(gm, incl, RG - 1, RG);
    }
    __syncwarp(gm);
    return carry;
}

// table 2: OR the compressed P rows of RA_I's columns (racol[0 .. n1)),
// four columns' gathers in flight per lane
__device__ __forceinline__ bool rap_table2(unsigned gm, int glane, const RapArgs &a, const int32_t *racol,
                                           int n1, int4 *t2) {
    constexpr int logT = RLOG2;
    constexpr int U = 4;
    tbl_clear(t2, RT2, glane, RG);
    __syncwarp(gm);
    bool ok = true;
    for (int q0 = 0; q0 < n1; q0 += U * RG) {
        int64_t p0[U];
        int pn[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int q = q0 + u * RG + glane;
            const int j = q < n1 ? racol[q] : -1;
            p0[u] = j >= 0 ? a.cpstart[j] : 0;
            pn[u] = j >= 0 ? a.cpcnt[j] : 0;
        }
        int sk[U];
        uint64_t sb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            sk[u] = pn[u] > 0 ? a.cpset[p0[u]] : 0;
            sb[u] = pn[u] > 0 ? a.cpbits[p0[u]] : 0ull;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (pn[u] > 0) ok &= tbl_or(t2, RT2, logT, sk[u], (unsigned)sb[u], (unsigned)(sb[u] >> 32));
            for (int q = 1; q < pn[u]; ++q) {   // P rows with several sets
                const uint64_t bits = a.cpbits[p0[u] + q];
                ok &= tbl_or(t2, RT2, logT, a.cpset[p0[u] + q], (unsigned)bits, (unsigned)(bits >> 32));
            }
        }
    }
    __syncwarp(gm);
    return __all_sync(gm, ok);
}

__global__ void __launch_bounds__(RBS) k_rap_sym(RapArgs a) {
    extern __shared__ int4 smem[];
    const unsigned gm = group_mask<RG>();
    const int glane = threadIdx.x & (RG - 1);
    const int gpb = RBS / RG;
    RapSlice sl(reinterpret_cast<char *>(smem) + (size_t)(threadIdx.x / RG) * RSLICE);
    for (int64_t i = (int64_t)blockIdx.x * gpb + threadIdx.x / RG; i < a.rows; i += (int64_t)gridDim.x * gpb) {
        const int64_t r0 = a.rrp[i], r1 = a.rrp[i + 1];
        bool fit = rap_table1(gm, glane, a, r0, r1, sl.t1);
        int n1 = 0;
        if (fit) {
            for (int s = glane; s < RT1; s += RG) n1 += slot_pop(sl.t1[s]);
            n1 = group_sum<RG, int>(gm, n1);
            fit = n1 <= RCRA;
        }
        int n2 = 0;
        if (fit) {
            rap_list_cols(gm, glane, sl.t1, sl.racol);
            fit = rap_table2(gm, glane, a, sl.racol, n1, sl.t2);
            for (int s = glane; s < RT2; s += RG) n2 += slot_pop(sl.t2[s]);
            n2 = group_sum<RG, int>(gm, n2);
            fit = fit && n2 <= RCC;
        }
        if (glane == 0) {
            a.counts[i] = fit ? n2 : 0;
            if (!fit) atomicOr(a.unfit, 1);
        }
        __syncwarp(gm);
    }
}

__global__ void __launch_bounds__(RBS) k_rap_num(RapArgs a) {
    extern __shared__ int4 smem[];
    const unsigned gm = group_mask<RG>();
    const int glane = threadIdx.x & (RG - 1);
    const int gpb = RBS / RG;
    RapSlice sl(reinterpret_cast<char *>(smem) + (size_t)(threadIdx.x / RG) * RSLICE);
    for (int64_t i = (int64_t)blockIdx.x * gpb + threadIdx.x / RG; i < a.rows; i += (int64_t)gridDim.x * gpb) {
        const int64_t r0 = a.rrp[i], r1 = a.rrp[i + 1];
        const int64_t cp = a.cptr[i];
        const int n = (int)(a.cptr[i + 1] - cp);
        // ---- RA_I: structure (ascending columns) and values
        rap_table1(gm, glane, a, r0, r1, sl.t1);   // fits: checked by k_rap_sym
        const int n1 = rap_rank(gm, glane, sl.t1, RT1, reinterpret_cast<int2 *>(sl.raval));
        for (int s = glane; s < RT1; s += RG) {
            const int4 e = sl.t1[s];
            if (e.x == TSG_EMPTY) continue;
            uint64_t b = ((uint64_t)(uint32_t)e.z << 32) | (uint32_t)e.y;
            int r = e.w;
            while (b) {
                sl.racol[r++] = e.x * 64 + (__ffsll((long long)b) - 1);
                b &= b - 1;
            }
        }
        __syncwarp(gm);
        for (int q = glane; q < n1; q += RG) sl.raval[q] = -0.0;
        __syncwarp(gm);
        // R entries in storage order; the lanes split the selected A row
        // (distinct columns: no two lanes meet), __syncwarp between entries.
        // The next entry's first RAU*G A entries are loaded before the
        // current one is accumulated.
        constexpr int RAU = 4;
        auto issue = [&](int64_t t, double &rv, int64_t &a0, int64_t &a1, int (&cc)[RAU], double (&vv)[RAU]) {
            if (t < r1) {
                const int k = a.rcol[t];
                rv = a.rval[t];
                a0 = a.arp[k];
                a1 = a.arp[k + 1];
            } else {
                rv = 0.0;
                a0 = a1 = 0;
            }
#pragma unroll
            for (int u = 0; u < RAU; ++u) {
                const int64_t q = a0 + u * RG + glane;
                cc[u] = q < a1 ? a.acol[q] : 0;
                vv[u] = q < a1 ? a.aval[q] : 0.0;
            }
        };
        double rv;
        int64_t ea0, ea1;
        int cc[RAU];
        double vv[RAU];
        issue(r0, rv, ea0, ea1, cc, vv);
        for (int64_t t = r0; t < r1; ++t) {
            double nrv;
            int64_t na0, na1;
            int ncc[RAU];
            double nvv[RAU];
            issue(t + 1, nrv, na0, na1, ncc, nvv);
#pragma unroll
            for (int u = 0; u < RAU; ++u) {
                if (ea0 + u * RG + glane < ea1) {
                    const double prod = __dmul_rn(rv, vv[u]);
                    int4 e;
                    tbl_find(sl.t1, RT1, RLOG1, cc[u] >> 6, e);
                    const int pos = e.w + mask_rank(e, cc[u] & 63);
                    sl.raval[pos] = __dadd_rn(sl.raval[pos], prod);
                }
            }
            for (int64_t q = ea0 + RAU * RG + glane; q < ea1; q += RG) {   // long A rows
                const int c2 = a.acol[q];
                const double prod = __dmul_rn(rv, a.aval[q]);
                int4 e;
                tbl_find(sl.t1, RT1, RLOG1, c2 >> 6, e);
                const int pos = e.w + mask_rank(e, c2 & 63);
                sl.raval[pos] = __dadd_rn(sl.raval[pos], prod);
            }
            __syncwarp(gm);
            rv = nrv;
            ea0 = na0;
            ea1 = na1;
#pragma unroll
            for (int u = 0; u < RAU; ++u) {
                cc[u] = ncc[u];
                vv[u] = nvv[u];
            }
        }
        // ---- C_I = RA_I * P: structure, then owner-folded products
        rap_table2(gm, glane, a, sl.racol, n1, sl.t2);
        const int n2 = rap_rank(gm, glane, sl.t2, RT2, reinterpret_cast<int2 *>(sl.cv));
        if (n2 != n) {
            if (glane == 0) kerr(a.err, KERR_COUNT, i);
            __syncwarp(gm);
            continue;   // group-uniform
        }
        for (int s = glane; s < RT2; s += RG) {
            const int4 e = sl.t2[s];
            if (e.x == TSG_EMPTY) continue;
            uint64_t b = ((uint64_t)(uint32_t)e.z << 32) | (uint32_t)e.y;
            int r = e.w;
            while (b) {
                a.ccol[cp + r++] = e.x * 64 + (__ffsll((long long)b) - 1);
                b &= b - 1;
            }
        }
        __syncwarp(gm);
        for (int q = glane; q < n2; q += RG) sl.cv[q] = -0.0;
        __syncwarp(gm);
        group_enumerate<RG>(
            gm, glane, 0, n1,
            [&](int64_t q, int64_t &st, int &len) {
                const int j = sl.racol[q];
                st = a.prp[j];
                len = (int)(a.prp[j + 1] - st);
            },
            [&](bool valid, int, int64_t q, int64_t s) {
                int pos = -1;
                double prod = 0.0;
                if (valid) {
                    const int cc = a.pcol[s];
                    int4 e;
                    tbl_find(sl.t2, RT2, RLOG2, cc >> 6, e);
                    pos = e.w + mask_rank(e, cc & 63);
                    prod = __dmul_rn(sl.raval[q], a.pval[s]);
                }
                sl.spos[glane] = pos;
                sl.sprod[glane] = prod;
                __syncwarp(gm);
                // lane-ordered fold of this chunk: the owner of a position
                // (pos = glane mod G) adds the chunk's products in lane order
#pragma unroll
                for (int u = 0; u < RG; ++u) {
                    const int p = sl.spos[u];
                    if (p >= 0 && (p & (RG - 1)) == glane) sl.cv[p] = __dadd_rn(sl.cv[p], sl.sprod[u]);
                }
                __syncwarp(gm);
            });
        for (int q = glane; q < n2; q += RG) a.cval[cp + q] = sl.cv[q];
        __syncwarp(gm);
    }
}

}  // namespace

int tsg_compress_impl(tsg_ctx *c, const tsg_csr *b, tsg_cmat **out);

extern "C" int tsg_rap(tsg_ctx *c, const tsg_csr *r, const tsg_csr *a, const tsg_csr *p, int mode,
                       tsg_csr **out, int *fused) {
    TSG_RESOLVE(c, r);
    TSG_RESOLVE(c, a);
    TSG_RESOLVE(c, p);
    if (!c || !r || !a || !p || !out) {
        tsg_set_error("tsg_rap: bad arguments");
        return TSG_EARG;
    }
    if (r->cols != a->rows || a->cols != p->rows) {
        tsg_set_error("R is %lldx%lld, A %lldx%lld, P %lldx%lld: inner dimensions differ", (long long)r->rows,
                      (long long)r->cols, (long long)a->rows, (long long)a->cols, (long long)p->rows,
                      (long long)p->cols);
        return TSG_EDIM;
    }
    if (!r->val || !a->val || !p->val) {
        tsg_set_error("numeric multiply requires values on every operand");
        return TSG_EVALID;
    }
    if (fused) *fused = 0;
    const bool eligible = mode != 0 && a->sorted && a->distinct && p->sorted && p->distinct &&
                          !r->host_mapped && !a->host_mapped && !p->host_mapped;
    auto two_step = [&]() -> int {
        tsg_csr *ra = nullptr;
        TSG_TRY(tsg_multiply(c, r, a, &ra));
        const int s = tsg_multiply(c, ra, p, out);
        tsg_csr_free(c, ra);
        return s;
    };
    if (!eligible) return two_step();
    tsg_cmat *ca = nullptr, *cpm = nullptr;
    TSG_TRY(tsg_compress_impl(c, a, &ca));
    int st = tsg_compress_impl(c, p, &cpm);
    if (st != TSG_OK) {
        tsg_cmat_free(c, ca);
        return st;
    }
    cudaStream_t s = c->stream;
    auto ck = [](cudaError_t e) -> int {
        if (e == cudaSuccess) return TSG_OK;
        tsg_set_error("tsg_rap: %s", cudaGetErrorString(e));
        return TSG_ECUDA;
    };
    RapArgs ra{};
    ra.rrp = r->rp;
    ra.rcol = r->col;
    ra.rval = r->val;
    ra.arp = a->rp;
    ra.acol = a->col;
    ra.aval = a->val;
    ra.prp = p->rp;
    ra.pcol = p->col;
    ra.pval = p->val;
    ra.castart = ca->start;
    ra.cacnt = ca->cnt;
    ra.caset = ca->set;
    ra.cabits = ca->bits;
    ra.cpstart = cpm->start;
    ra.cpcnt = cpm->cnt;
    ra.cpset = cpm->set;
    ra.cpbits = cpm->bits;
    ra.rows = r->rows;
    ra.err = c->d_err;
    int *unfit = reinterpret_cast<int *>(c->d_small + 59);
    ra.unfit = unfit;
    int64_t *counts = nullptr, *cptr = nullptr;
    st = tsg_alloc_t(c, &counts, r->rows + 1);
    if (st == TSG_OK) st = tsg_alloc_t(c, &cptr, r->rows + 1);
    ra.counts = counts;
    const size_t smem = (size_t)(RBS / RG) * RSLICE;
    if (st == TSG_OK) st = tsg_func_smem((const void *)k_rap_sym, smem);
    if (st == TSG_OK) st = tsg_func_smem((const void *)k_rap_num, smem);
    if (st == TSG_OK) st = tsg_fill(c, unfit, 0, sizeof(int), s);
    const unsigned grid = grid_for(r->rows, RBS / RG, c->num_sms * 64);
    if (st == TSG_OK && r->rows > 0) {
        k_rap_sym<<<grid, RBS, smem, s>>>(ra);
        ++c->launches;
        st = ck(cudaGetLastError());
    }
    if (st == TSG_OK) st = tsg_exclusive_scan_i64(c, counts, cptr, r->rows);
    if (st == TSG_OK) st = tsg_put_small(c, cptr + r->rows, 1, 0);
    if (st == TSG_OK) st = tsg_put_small(c, reinterpret_cast<const int64_t *>(unfit), 1, 1);
    if (st == TSG_OK) st = ck(cudaStreamSynchronize(s));
    if (st == TSG_OK) st = tsg_pending_errors(c);
    const int64_t nnz = c->h_small[0];
    const bool all_fit = (c->h_small[1] & 0xffffffff) == 0;
    tsg_csr *C = nullptr;
    if (st == TSG_OK && all_fit) {
        st = tsg_csr_alloc(c, r->rows, p->cols, nnz, true, &C);
        if (st == TSG_OK) {
            st = ck(cudaMemcpyAsync(C->rp, cptr, (r->rows + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
            ra.cptr = C->rp;
            ra.ccol = C->col;
            ra.cval = C->val;
            if (st == TSG_OK && r->rows > 0) {
                k_rap_num<<<grid, RBS, smem, s>>>(ra);
                ++c->launches;
                st = ck(cudaGetLastError());
            }
            if (st == TSG_OK) st = tsg_check_kernel_errors(c, "rap numeric");
        }
    }
    tsg_free(c, counts);
    tsg_free(c, cptr);
    tsg_cmat_free(c, ca);
    tsg_cmat_free(c, cpm);
    if (st != TSG_OK) {
        if (C) tsg_csr_free(c, C);
        return st;
    }
    if (!all_fit) return two_step();
    C->sorted = 1;      // columns emitted in ascending order
    C->distinct = 1;
    C->max_row = -1;
    if (fused) *fused = 1;
    *out = C;
    return TSG_OK;
}

const void *tsg_kernel_rap() { return (const void *)k_rap_sym; }
