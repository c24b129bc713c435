// tsg_build.cu -- input builders on the device: grid
// stencil operators, the plain aggregation prolongator P with R = P^T, and a
// general CSR transpose.  They replace the host numpy builders for 10^8-10^9
// entry operands; each produces exactly the arrays of its host counterpart
// (generators.stencil / stencil_rows / aggregation, csr.transpose), which the
// GPU tests check entry for entry.
//
// Layout conventions follow the reference (generators.py:26-45, 98-142):
// flat point index with the first axis fastest, a row's columns ascending,
// centre weight = number of neighbours.  elasticity3d expands every scalar
// entry (point i, neighbour c, weight w) into the 3x3 block w * (I + 0.5)
// on dof rows 3i+r, columns 3c+d.
#include "tsg_internal.cuh"

#include <algorithm>
#include <vector>

#include <cub/device/device_radix_sort.cuh>

namespace {

constexpr int MAX_OFFS = 27;

struct StencilOffs {
    int k;                    // offsets, sorted by linear shift (= ascending column)
    int nd;                   // grid rank (2 or 3)
    int64_t dims[3];
    int64_t stride[3];
    int8_t s[MAX_OFFS][3];    // per-axis shift
    int64_t lin[MAX_OFFS];    // linear shift
    double w[MAX_OFFS];
};

__device__ __forceinline__ bool offs_ok(const StencilOffs &o, const int64_t (&x)[3], int j) {
    bool ok = true;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        if (ax < o.nd) {
            const int64_t y = x[ax] + o.s[j][ax];
            ok &= y >= 0 && y < o.dims[ax];
        }
    }
    return ok;
}

__device__ __forceinline__ void point_coords(const StencilOffs &o, int64_t p, int64_t (&x)[3]) {
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) x[ax] = ax < o.nd ? (p / o.stride[ax]) % o.dims[ax] : 0;
}

// row lengths of points [lo, lo + n): scalar rows (dof = 1) or 3 x scalar
__global__ void k_stencil_len(StencilOffs o, int64_t lo, int64_t n, int dof, int32_t *__restrict__ len) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n * dof;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = lo + r / dof;
        int64_t x[3];
        point_coords(o, p, x);
        int c = 0;
        for (int j = 0; j < o.k; ++j) c += offs_ok(o, x, j);
        len[r] = c * dof;
    }
}

// one warp per output row: lane j < k handles offset j; ballot ranks the
// valid offsets, so each row's entries are written in ascending column order
__global__ void k_stencil_fill(StencilOffs o, int64_t lo, int64_t n, int dof, const int64_t *__restrict__ rp,
                               int32_t *__restrict__ col, double *__restrict__ val) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w; r < n * dof; r += nw) {
        const int64_t p = lo + r / dof;
        const int rr = (int)(r % dof);
        int64_t x[3];
        point_coords(o, p, x);
        const bool ok = lane < o.k && offs_ok(o, x, lane);
        const unsigned bal = __ballot_sync(0xffffffffu, ok);
        if (!ok) continue;
        const int rank = __popc(bal & ((1u << lane) - 1u));
        const int64_t c = p + o.lin[lane];
        const int64_t at = rp[r] + (int64_t)rank * dof;
        if (dof == 1) {
            col[at] = (int32_t)c;
            val[at] = o.w[lane];
        } else {
            for (int d = 0; d < dof; ++d) {   // block w * (I + 0.5), dof row rr
                col[at + d] = (int32_t)(dof * c + d);
                val[at + d] = o.w[lane] * ((rr == d ? 1.0 : 0.0) + 0.5);
            }
        }
    }
}

__global__ void k_len_max(int64_t n, const int32_t *__restrict__ len, int *out) {
    int m = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        m = max(m, len[i]);
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, d));
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// ---- aggregation: P (fine point -> its aggregate, 1.0), R = P^T built directly

struct AggGrid {
    int nd;
    int factor;
    int64_t fdims[3], cdims[3];
    int64_t fstride[3], cstride[3];
};

__global__ void k_agg_p(AggGrid g, int64_t n, int64_t *__restrict__ rp, int32_t *__restrict__ col,
                        double *__restrict__ val) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n;
         i += (int64_t)gridDim.x * blockDim.x) {
        rp[i] = i;
        if (i == n) continue;
        int64_t a = 0;
#pragma unroll
        for (int ax = 0; ax < 3; ++ax)
            if (ax < g.nd) a += ((i / g.fstride[ax]) % g.fdims[ax] / g.factor) * g.cstride[ax];
        col[i] = (int32_t)a;
        val[i] = 1.0;
    }
}

__device__ __forceinline__ void agg_block(const AggGrid &g, int64_t J, int64_t (&b0)[3], int64_t (&bl)[3]) {
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
        if (ax < g.nd) {
            const int64_t cj = (J / g.cstride[ax]) % g.cdims[ax];
            b0[ax] = cj * g.factor;
            const int64_t e = b0[ax] + g.factor;
            bl[ax] = (e < g.fdims[ax] ? e : g.fdims[ax]) - b0[ax];
        } else {
            b0[ax] = 0;
            bl[ax] = 1;
        }
    }
}

__global__ void k_agg_r_len(AggGrid g, int64_t nc, int32_t *__restrict__ len) {
    for (int64_t J = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; J < nc;
         J += (int64_t)gridDim.x * blockDim.x) {
        int64_t b0[3], bl[3];
        agg_block(g, J, b0, bl);
        len[J] = (int32_t)(bl[0] * bl[1] * bl[2]);
    }
}

// fine points of aggregate J in ascending flat index: last axis outermost
__global__ void k_agg_r_fill(AggGrid g, int64_t nc, const int64_t *__restrict__ rp, int32_t *__restrict__ col,
                             double *__restrict__ val) {
    for (int64_t J = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; J < nc;
         J += (int64_t)gridDim.x * blockDim.x) {
        int64_t b0[3], bl[3];
        agg_block(g, J, b0, bl);
        int64_t at = rp[J];
        for (int64_t z = 0; z < bl[2]; ++z)
            for (int64_t y = 0; y < bl[1]; ++y)
                for (int64_t x = 0; x < bl[0]; ++x) {
                    const int64_t f = (b0[0] + x) * g.fstride[0] + (g.nd > 1 ? (b0[1] + y) * g.fstride[1] : 0) +
                                      (g.nd > 2 ? (b0[2] + z) * g.fstride[2] : 0);
                    col[at] = (int32_t)f;
                    val[at] = 1.0;
                    ++at;
                }
    }
}

// ---- transpose: stable radix sort of (column, entry) pairs

__global__ void k_entry_rows(int64_t rows, const int64_t *__restrict__ rp, int32_t *__restrict__ erow) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w; i < rows; i += nw)
        for (int64_t t = rp[i] + lane; t < rp[i + 1]; t += 32) erow[t] = (int32_t)i;
}

__global__ void k_iota(int64_t n, int32_t *__restrict__ v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = (int32_t)i;
}

__global__ void k_col_count(int64_t nnz, const int32_t *__restrict__ col, int32_t *__restrict__ cnt) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nnz; t += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[col[t]], 1);
}

__global__ void k_transpose_fill(int64_t nnz, const int32_t *__restrict__ order, const int32_t *__restrict__ erow,
                                 const double *__restrict__ val, int32_t *__restrict__ tcol,
                                 double *__restrict__ tval) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x) {
        const int32_t t = order[q];
        tcol[q] = erow[t];
        if (tval) tval[q] = val[t];
    }
}

#define CUB_CK(call)                                                              \
    do {                                                                          \
        cudaError_t e_ = (call);                                                  \
        if (e_ != cudaSuccess) {                                                  \
            tsg_set_error("%s: %s", #call, cudaGetErrorString(e_));               \
            return TSG_ECUDA;                                                     \
        }                                                                         \
    } while (0)

// host: the offsets of a stencil kind, sorted by linear shift
int stencil_offsets(int kind, const int64_t *dims, int nd, StencilOffs &o) {
    struct Off {
        int s[3];
        double w;
    };
    std::vector<Off> v;
    v.reserve(MAX_OFFS);
    auto add = [&](int x, int y, int z, double w) { v.push_back(Off{{x, y, z}, w}); };
    switch (kind) {
    case TSG_STENCIL_LAPLACE2D:
        add(0, 0, 0, 4.0);
        add(-1, 0, 0, -1.0);
        add(1, 0, 0, -1.0);
        add(0, -1, 0, -1.0);
        add(0, 1, 0, -1.0);
        break;
    case TSG_STENCIL_LAPLACE3D:
        add(0, 0, 0, 6.0);
        add(-1, 0, 0, -1.0);
        add(1, 0, 0, -1.0);
        add(0, -1, 0, -1.0);
        add(0, 1, 0, -1.0);
        add(0, 0, -1, -1.0);
        add(0, 0, 1, -1.0);
        break;
    case TSG_STENCIL_BIGSTAR2D: {
        add(0, 0, 0, 12.0);
        const int nb[12][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}, {-2, 0}, {2, 0},
                               {0, -2}, {0, 2}, {-1, -1}, {-1, 1}, {1, -1}, {1, 1}};
        for (int q = 0; q < 12; ++q) add(nb[q][0], nb[q][1], 0, -1.0);
        break;
    }
    case TSG_STENCIL_BRICK3D:
    case TSG_STENCIL_ELASTICITY3D:
        add(0, 0, 0, 26.0);
        for (int x = -1; x <= 1; ++x)
            for (int y = -1; y <= 1; ++y)
                for (int z = -1; z <= 1; ++z)
                    if (x || y || z) add(x, y, z, -1.0);
        break;
    default:
        tsg_set_error("unknown stencil kind %d", kind);
        return TSG_EARG;
    }
    const int want = (kind == TSG_STENCIL_LAPLACE2D || kind == TSG_STENCIL_BIGSTAR2D) ? 2 : 3;
    if (nd != want) {
        tsg_set_error("stencil kind %d needs %d grid dims, got %d", kind, want, nd);
        return TSG_EARG;
    }
    o.k = (int)v.size();
    o.nd = nd;
    int64_t st = 1;
    for (int ax = 0; ax < 3; ++ax) {
        o.dims[ax] = ax < nd ? dims[ax] : 1;
        o.stride[ax] = st;
        st *= o.dims[ax];
    }
    std::vector<std::pair<int64_t, int>> order;
    for (int j = 0; j < o.k; ++j) {
        int64_t lin = 0;
        for (int ax = 0; ax < nd; ++ax) lin += v[j].s[ax] * o.stride[ax];
        order.push_back({lin, j});
    }
    std::stable_sort(order.begin(), order.end(),
                     [](const std::pair<int64_t, int> &x, const std::pair<int64_t, int> &y) { return x.first < y.first; });
    for (int q = 0; q < o.k; ++q) {
        const Off &f = v[order[q].second];
        for (int ax = 0; ax < 3; ++ax) o.s[q][ax] = (int8_t)f.s[ax];
        o.lin[q] = order[q].first;
        o.w[q] = f.w;
    }
    return TSG_OK;
}

}  // namespace

extern "C" int tsg_stencil(tsg_ctx *c, int kind, const int64_t *dims, int ndims, int64_t row_lo,
                           int64_t row_hi, tsg_csr **out) {
    if (!c || !dims || !out || ndims < 2 || ndims > 3) {
        tsg_set_error("tsg_stencil: bad arguments");
        return TSG_EARG;
    }
    int64_t n = 1;
    for (int ax = 0; ax < ndims; ++ax) {
        if (dims[ax] <= 0) {
            tsg_set_error("grid dims must be positive");
            return TSG_EDIM;
        }
        n *= dims[ax];
    }
    StencilOffs o;
    TSG_TRY(stencil_offsets(kind, dims, ndims, o));
    const int dof = kind == TSG_STENCIL_ELASTICITY3D ? 3 : 1;
    if (row_lo < 0 || row_hi < 0) {   // whole operator
        row_lo = 0;
        row_hi = n;
    }
    if (row_lo > row_hi || row_hi > n || (dof > 1 && (row_lo != 0 || row_hi != n))) {
        tsg_set_error("tsg_stencil: row range [%lld, %lld) invalid for %lld points", (long long)row_lo,
                      (long long)row_hi, (long long)n);
        return TSG_EARG;
    }
    if (dof * n > INT32_MAX) {
        tsg_set_error("tsg_stencil: %lld columns exceed int32", (long long)(dof * n));
        return TSG_EDIM;
    }
    const int64_t pts = row_hi - row_lo, rows = pts * dof;
    cudaStream_t s = c->stream;
    int32_t *len = nullptr;
    int64_t *rp = nullptr;
    TSG_TRY(tsg_alloc_t(c, &len, rows + 1));
    TSG_TRY(tsg_alloc_t(c, &rp, rows + 1));
    int *dmax = reinterpret_cast<int *>(c->d_small + 58);
    TSG_TRY(tsg_fill(c, dmax, 0, sizeof(int), s));
    if (rows > 0) {
        const unsigned g = grid_for(rows, 256, c->num_sms * 16);
        k_stencil_len<<<g, 256, 0, s>>>(o, row_lo, pts, dof, len); ++c->launches;
        k_len_max<<<g, 256, 0, s>>>(rows, len, dmax); ++c->launches;
    }
    TSG_TRY(tsg_exclusive_scan_i32_to_i64(c, len, rp, rows));
    TSG_TRY(tsg_put_small(c, rp + rows, 1, 0));
    TSG_TRY(tsg_put_small(c, reinterpret_cast<const int64_t *>(dmax), 1, 1));
    TSG_CK(cudaStreamSynchronize(s));
    const int64_t nnz = c->h_small[0];
    const int max_row = (int)(c->h_small[1] & 0xffffffff);
    tsg_csr *m = nullptr;
    TSG_TRY(tsg_csr_alloc(c, rows, n * dof, nnz, true, &m));
    TSG_CK(cudaMemcpyAsync(m->rp, rp, (rows + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    if (rows > 0) {
        k_stencil_fill<<<grid_for(rows, 8, c->num_sms * 16), 256, 0, s>>>(o, row_lo, pts, dof, rp, m->col, m->val);
        ++c->launches;
    }
    TSG_CK(cudaGetLastError());
    TSG_TRY(tsg_free(c, len));
    TSG_TRY(tsg_free(c, rp));
    m->sorted = 1;
    m->distinct = 1;
    m->max_row = rows > 0 ? max_row : 0;
    *out = m;
    return TSG_OK;
}

extern "C" int tsg_aggregation(tsg_ctx *c, const int64_t *dims, int ndims, int factor, tsg_csr **p_out,
                               tsg_csr **r_out) {
    if (!c || !dims || !p_out || !r_out || ndims < 1 || ndims > 3 || factor < 1) {
        tsg_set_error("tsg_aggregation: bad arguments");
        return TSG_EARG;
    }
    AggGrid g{};
    g.nd = ndims;
    g.factor = factor;
    int64_t n = 1, nc = 1;
    for (int ax = 0; ax < 3; ++ax) {
        const int64_t d = ax < ndims ? dims[ax] : 1;
        if (d <= 0) {
            tsg_set_error("grid dims must be positive");
            return TSG_EDIM;
        }
        g.fdims[ax] = d;
        g.cdims[ax] = ax < ndims ? (d + factor - 1) / factor : 1;
        g.fstride[ax] = n;
        g.cstride[ax] = nc;
        n *= d;
        nc *= g.cdims[ax];
    }
    if (n > INT32_MAX) {
        tsg_set_error("tsg_aggregation: %lld fine points exceed int32", (long long)n);
        return TSG_EDIM;
    }
    cudaStream_t s = c->stream;
    tsg_csr *P = nullptr, *R = nullptr;
    TSG_TRY(tsg_csr_alloc(c, n, nc, n, true, &P));
    k_agg_p<<<grid_for(n + 1, 256, c->num_sms * 16), 256, 0, s>>>(g, n, P->rp, P->col, P->val); ++c->launches;
    int32_t *len = nullptr;
    TSG_TRY(tsg_alloc_t(c, &len, nc + 1));
    int st = tsg_csr_alloc(c, nc, n, n, true, &R);
    if (st != TSG_OK) {
        tsg_csr_free(c, P);
        return st;
    }
    const unsigned gc = grid_for(nc, 256, c->num_sms * 16);
    k_agg_r_len<<<gc, 256, 0, s>>>(g, nc, len); ++c->launches;
    TSG_TRY(tsg_exclusive_scan_i32_to_i64(c, len, R->rp, nc));
    k_agg_r_fill<<<gc, 256, 0, s>>>(g, nc, R->rp, R->col, R->val); ++c->launches;
    TSG_CK(cudaGetLastError());
    TSG_TRY(tsg_free(c, len));
    int64_t rmax = 1;
    for (int ax = 0; ax < ndims; ++ax) rmax *= std::min<int64_t>(factor, g.fdims[ax]);
    P->sorted = 1;
    P->distinct = 1;
    P->max_row = n > 0 ? 1 : 0;
    R->sorted = 1;
    R->distinct = 1;
    R->max_row = nc > 0 ? rmax : 0;
    *p_out = P;
    *r_out = R;
    return TSG_OK;
}

extern "C" int tsg_transpose(tsg_ctx *c, const tsg_csr *a, tsg_csr **out) {
    TSG_RESOLVE(c, a);
    if (!c || !a || !out) {
        tsg_set_error("tsg_transpose: bad arguments");
        return TSG_EARG;
    }
    if (a->host_mapped) {
        tsg_set_error("tsg_transpose: matrix lives in mapped host memory");
        return TSG_EARG;
    }
    if (a->nnz > INT32_MAX || a->rows > INT32_MAX) {
        tsg_set_error("tsg_transpose: %lld entries exceed int32 indexing", (long long)a->nnz);
        return TSG_EDIM;
    }
    const int64_t nnz = a->nnz, rows = a->rows, cols = a->cols;
    const bool values = a->val != nullptr;
    cudaStream_t s = c->stream;
    tsg_csr *T = nullptr;
    TSG_TRY(tsg_csr_alloc(c, cols, rows, nnz, values, &T));
    int32_t *cnt = nullptr;
    TSG_TRY(tsg_alloc_t(c, &cnt, cols + 1));
    TSG_TRY(tsg_fill(c, cnt, 0, (cols + 1) * sizeof(int32_t), s));
    if (nnz > 0) {
        k_col_count<<<grid_for(nnz, 256, c->num_sms * 16), 256, 0, s>>>(nnz, a->col, cnt); ++c->launches;
    }
    TSG_TRY(tsg_exclusive_scan_i32_to_i64(c, cnt, T->rp, cols));
    int *dmax = reinterpret_cast<int *>(c->d_small + 58);
    TSG_TRY(tsg_fill(c, dmax, 0, sizeof(int), s));
    if (cols > 0) {
        k_len_max<<<grid_for(cols, 256, c->num_sms * 16), 256, 0, s>>>(cols, cnt, dmax); ++c->launches;
    }
    if (nnz > 0) {
        int32_t *erow = nullptr, *keys_alt = nullptr, *iota = nullptr, *order = nullptr;
        TSG_TRY(tsg_alloc_t(c, &erow, nnz));
        TSG_TRY(tsg_alloc_t(c, &keys_alt, nnz));
        TSG_TRY(tsg_alloc_t(c, &iota, nnz));
        TSG_TRY(tsg_alloc_t(c, &order, nnz));
        k_entry_rows<<<grid_for(rows, 8, c->num_sms * 16), 256, 0, s>>>(rows, a->rp, erow); ++c->launches;
        k_iota<<<grid_for(nnz, 256, c->num_sms * 16), 256, 0, s>>>(nnz, iota); ++c->launches;
        int end_bit = 1;
        while (end_bit < 31 && ((int64_t)1 << end_bit) < cols) ++end_bit;
        size_t need = 0;
        CUB_CK(cub::DeviceRadixSort::SortPairs(nullptr, need, a->col, keys_alt, iota, order, (int)nnz, 0, end_bit, s));
        void *tmp = nullptr;
        TSG_TRY(tsg_alloc(c, &tmp, need > 0 ? need : 1));
        // stable: entries of one column keep their row-major order = ascending rows
        CUB_CK(cub::DeviceRadixSort::SortPairs(tmp, need, a->col, keys_alt, iota, order, (int)nnz, 0, end_bit, s));
        ++c->launches;
        k_transpose_fill<<<grid_for(nnz, 256, c->num_sms * 16), 256, 0, s>>>(nnz, order, erow, a->val, T->col,
                                                                             values ? T->val : nullptr);
        ++c->launches;
        TSG_TRY(tsg_free(c, tmp));
        TSG_TRY(tsg_free(c, erow));
        TSG_TRY(tsg_free(c, keys_alt));
        TSG_TRY(tsg_free(c, iota));
        TSG_TRY(tsg_free(c, order));
    }
    TSG_TRY(tsg_put_small(c, reinterpret_cast<const int64_t *>(dmax), 1, 1));
    TSG_CK(cudaStreamSynchronize(s));
    TSG_CK(cudaGetLastError());
    TSG_TRY(tsg_free(c, cnt));
    T->sorted = 1;
    T->distinct = a->distinct;   // a column repeated in a row repeats the row in the transpose
    T->max_row = cols > 0 ? (int)(c->h_small[1] & 0xffffffff) : 0;
    *out = T;
    return TSG_OK;
}

const void *tsg_kernel_build() { return (const void *)k_stencil_len; }
