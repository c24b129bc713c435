// tsg_graph.cu -- graph preparation on the device:
// the steps in front of the masked-count kernel, which the reference runs as
// host numpy.
//
//   tsg_graph_lower  validate_graph + degree_sort_permutation + lower_triangle
//                    (triangles.py:18-46): square / loop-free / symmetric
//                    check, vertices stably sorted by degree (ties by index),
//                    strict lower triangle of the relabelled graph, rows sorted.
//   tsg_rmat_graph   the R-MAT builder of generators.py (rmat_edges +
//                    undirected_pattern of this package, Graph500 parameters,
//                    SplitMix64 counter stream): edge e, level l uses output
//                    e*scale + l + 1 of the stream, so every edge is generated
//                    independently and equals the host builder bit for bit.
//
// Sorting (degrees, permutation keys, edge keys, per-row columns) uses CUB's
// radix / segmented sorts from the CUDA toolkit: this is input preparation,
// not the SpGEMM hot path.
#include <cub/cub.cuh>
#include <vector>

#include "tsg_internal.cuh"

namespace {

constexpr uint64_t SM_GAMMA = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t sm_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// multiset symmetry + no loops; rows sorted.  flags[0] |= loop, flags[1] |= asym
__global__ void k_graph_check(int64_t n, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                              int *flags) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    auto count_in_row = [&](int64_t r, int32_t key) -> int64_t {
        int64_t lo = rp[r], hi = rp[r + 1];
        int64_t a = lo, b = hi;   // lower bound
        while (a < b) {
            int64_t m = (a + b) >> 1;
            if (col[m] < key) a = m + 1; else b = m;
        }
        int64_t c = a, d = hi;    // upper bound
        while (c < d) {
            int64_t m = (c + d) >> 1;
            if (col[m] <= key) c = m + 1; else d = m;
        }
        return c - a;
    };
    for (int64_t i = w; i < n; i += nw) {
        bool loop = false, asym = false;
        for (int64_t t = rp[i] + lane; t < rp[i + 1]; t += 32) {
            const int32_t j = col[t];
            if (j == i) {
                loop = true;
                continue;
            }
            if (t > rp[i] && col[t - 1] == j) continue;   // count each distinct j once
            asym |= count_in_row(i, j) != count_in_row(j, (int32_t)i);
        }
        if (__any_sync(0xffffffffu, loop) && lane == 0) atomicOr(&flags[0], 1);
        if (__any_sync(0xffffffffu, asym) && lane == 0) atomicOr(&flags[1], 1);
    }
}

__global__ void k_degrees(int64_t n, const int64_t *__restrict__ rp, uint32_t *deg, int32_t *iota) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        deg[i] = (uint32_t)(rp[i + 1] - rp[i]);
        iota[i] = (int32_t)i;
    }
}

__global__ void k_invert(int64_t n, const int32_t *__restrict__ perm, int32_t *__restrict__ pos) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x)
        pos[perm[k]] = (int32_t)k;
}

// new row pos[i] holds {pos[j] : j in N(i), pos[j] < pos[i]}: count, then fill
__global__ void k_lower_count(int64_t n, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                              const int32_t *__restrict__ pos, int32_t *__restrict__ cnt,
                              unsigned long long *maxlen) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long ml = 0;
    for (int64_t i = w; i < n; i += nw) {
        const int32_t pi = pos[i];
        int k = 0;
        for (int64_t t = rp[i] + lane; t < rp[i + 1]; t += 32) k += pos[col[t]] < pi;
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) k += __shfl_xor_sync(0xffffffffu, k, d);
        if (lane == 0) cnt[pi] = k;
        if ((unsigned long long)k > ml) ml = (unsigned long long)k;
    }
    if (lane == 0 && ml) atomicMax(maxlen, ml);
}

__global__ void k_lower_fill(int64_t n, const int64_t *__restrict__ rp, const int32_t *__restrict__ col,
                             const int32_t *__restrict__ pos, const int64_t *__restrict__ lrp,
                             int32_t *__restrict__ lcol) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = w; i < n; i += nw) {
        const int32_t pi = pos[i];
        int64_t out = lrp[pi];
        for (int64_t b = rp[i]; b < rp[i + 1]; b += 32) {
            const int64_t t = b + lane;
            int32_t pj = t < rp[i + 1] ? pos[col[t]] : INT32_MAX;
            const bool keep = pj < pi;
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep) lcol[out + __popc(bal & lt)] = pj;
            out += __popc(bal);
        }
    }
}

// R-MAT: edge e -> (u, v) from `scale` uniform draws (quadrant a/b/c/d per level)
__global__ void k_rmat_edges(int64_t m, int scale, uint64_t seed, double a, double ab, double abc,
                             uint32_t *__restrict__ u, uint32_t *__restrict__ v) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        uint32_t uu = 0, vv = 0;
        uint64_t k = (uint64_t)e * (uint64_t)scale + 1ull;
        for (int l = 0; l < scale; ++l, ++k) {
            const double r = (double)(sm_mix(seed + k * SM_GAMMA) >> 11) * 0x1.0p-53;
            const uint32_t bu = r >= ab;
            const uint32_t bv = (r >= a && r < ab) || r >= abc;
            uu = (uu << 1) | bu;
            vv = (vv << 1) | bv;
        }
        u[e] = uu;
        v[e] = vv;
    }
}

__global__ void k_perm_keys(int64_t n, uint64_t seed2, uint64_t *keys, int32_t *iota) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = sm_mix(seed2 + (uint64_t)(i + 1) * SM_GAMMA);
        iota[i] = (int32_t)i;
    }
}

// both directions of every non-loop edge as row-major keys; loops -> sentinel n*n
__global__ void k_edge_keys(int64_t m, int scale, const uint32_t *__restrict__ u,
                            const uint32_t *__restrict__ v, const int32_t *__restrict__ perm,
                            uint64_t *__restrict__ keys) {
    const uint64_t sentinel = 1ull << (2 * scale);
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t pu = (uint32_t)perm[u[e]], pv = (uint32_t)perm[v[e]];
        const bool loop = pu == pv;
        keys[2 * e] = loop ? sentinel : (pu << scale) | pv;
        keys[2 * e + 1] = loop ? sentinel : (pv << scale) | pu;
    }
}

__global__ void k_keys_to_csr(int64_t n, int64_t nnz, int scale, const uint64_t *__restrict__ keys,
                              int64_t *__restrict__ rp, int32_t *__restrict__ col) {
    const uint64_t mask = (1ull << scale) - 1ull;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n;
         i += (int64_t)gridDim.x * blockDim.x) {
        // row_ptr[i] = first key with row >= i
        const uint64_t want = (uint64_t)i << scale;
        int64_t lo = 0, hi = nnz;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (keys[mid] < want) lo = mid + 1; else hi = mid;
        }
        rp[i] = lo;
    }
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz;
         k += (int64_t)gridDim.x * blockDim.x)
        col[k] = (int32_t)(keys[k] & mask);
}

__global__ void k_widen(int64_t n, const int32_t *__restrict__ in, int64_t *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}

__global__ void k_row_max(int64_t n, const int64_t *__restrict__ rp, unsigned long long *maxlen) {
    unsigned long long ml = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const unsigned long long l = (unsigned long long)(rp[i + 1] - rp[i]);
        if (l > ml) ml = l;
    }
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        unsigned long long o = __shfl_xor_sync(0xffffffffu, ml, d);
        if (o > ml) ml = o;
    }
    if ((threadIdx.x & 31) == 0 && ml) atomicMax(maxlen, ml);
}

// CUB temp storage from the context arena
struct Temp {
    tsg_ctx *c;
    void *p = nullptr;
    size_t bytes = 0;
    explicit Temp(tsg_ctx *cc) : c(cc) {}
    int ensure(size_t need) {
        if (need <= bytes) return TSG_OK;
        if (p) tsg_free(c, p);
        p = nullptr;
        bytes = 0;
        TSG_TRY(tsg_alloc(c, &p, need > 0 ? need : 1));
        bytes = need;
        return TSG_OK;
    }
    ~Temp() {
        if (p) tsg_free(c, p);
    }
};

#define CUB_CK(x)                                                                  \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess) {                                                   \
            tsg_set_error("CUB %s: %s", #x, cudaGetErrorString(e_));               \
            return TSG_ECUDA;                                                      \
        }                                                                          \
    } while (0)

int bits_for(uint64_t maxval) {
    int b = 1;
    while (b < 64 && (maxval >> b) != 0) ++b;
    return b;
}

// rows of m sorted in place (segmented sort of the column keys)
int sort_rows(tsg_ctx *c, Temp &tmp, int64_t rows, int64_t nnz, const int64_t *rp, int32_t *col) {
    if (nnz <= 0) return TSG_OK;
    int32_t *alt = nullptr;
    TSG_TRY(tsg_alloc_t(c, &alt, nnz));
    size_t need = 0;
    CUB_CK(cub::DeviceSegmentedSort::SortKeys(nullptr, need, col, alt, nnz, rows, rp, rp + 1, c->stream));
    TSG_TRY(tmp.ensure(need));
    CUB_CK(cub::DeviceSegmentedSort::SortKeys(tmp.p, need, col, alt, nnz, rows, rp, rp + 1, c->stream));
    ++c->launches;
    TSG_CK(cudaMemcpyAsync(col, alt, nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, c->stream));
    TSG_TRY(tsg_free(c, alt));
    return TSG_OK;
}

}  // namespace

extern "C" int tsg_graph_lower(tsg_ctx *c, const tsg_csr *g, int check, tsg_csr **out,
                               int64_t *perm_host) {
    TSG_RESOLVE(c, g);
    if (!c || !g || !out) {
        tsg_set_error("tsg_graph_lower: null argument");
        return TSG_EARG;
    }
    if (g->rows != g->cols) {
        tsg_set_error("graph matrix must be square");
        return TSG_EVALID;
    }
    if (g->rows > INT32_MAX) {
        tsg_set_error("graph has more than 2^31 vertices");
        return TSG_EARG;
    }
    const int64_t n = g->rows, nnz = g->nnz;
    Temp tmp(c);
    cudaStream_t s = c->stream;
    const unsigned gw = grid_for(n, 8, c->num_sms * 16);      // warp per row
    const unsigned ge = grid_for(n + 1, 256, c->num_sms * 8);  // thread per row
    // sorted column view of g (the symmetry check searches rows)
    const int32_t *gcol = g->col;
    int32_t *sorted_col = nullptr;
    if (check && !g->sorted && nnz > 0) {
        TSG_TRY(tsg_alloc_t(c, &sorted_col, nnz));
        TSG_CK(cudaMemcpyAsync(sorted_col, g->col, nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
        TSG_TRY(sort_rows(c, tmp, n, nnz, g->rp, sorted_col));
        gcol = sorted_col;
    }
    if (check && nnz > 0) {
        int *flags = reinterpret_cast<int *>(c->d_small + 54);
        TSG_TRY(tsg_fill(c, flags, 0, 2 * sizeof(int), s));
        k_graph_check<<<gw, 256, 0, s>>>(n, g->rp, gcol, flags); ++c->launches;
        int h[2] = {0, 0};
        TSG_CK(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, s));
        TSG_CK(cudaStreamSynchronize(s));
        if (sorted_col) tsg_free(c, sorted_col);
        if (h[0]) {
            tsg_set_error("graph matrix must have an empty diagonal");
            return TSG_EVALID;
        }
        if (h[1]) {
            tsg_set_error("graph pattern must be symmetric");
            return TSG_EVALID;
        }
    }
    // degree order: stable radix sort of (degree, vertex)
    uint32_t *deg = nullptr, *deg_alt = nullptr;
    int32_t *iota = nullptr, *perm = nullptr, *pos = nullptr;
    TSG_TRY(tsg_alloc_t(c, &deg, n + 1));
    TSG_TRY(tsg_alloc_t(c, &deg_alt, n + 1));
    TSG_TRY(tsg_alloc_t(c, &iota, n + 1));
    TSG_TRY(tsg_alloc_t(c, &perm, n + 1));
    TSG_TRY(tsg_alloc_t(c, &pos, n + 1));
    if (n > 0) {
        k_degrees<<<ge, 256, 0, s>>>(n, g->rp, deg, iota); ++c->launches;
        const int end_bit = g->max_row >= 0 ? bits_for((uint64_t)g->max_row) : 32;
        size_t need = 0;
        CUB_CK(cub::DeviceRadixSort::SortPairs(nullptr, need, deg, deg_alt, iota, perm, n, 0, end_bit, s));
        TSG_TRY(tmp.ensure(need));
        CUB_CK(cub::DeviceRadixSort::SortPairs(tmp.p, need, deg, deg_alt, iota, perm, n, 0, end_bit, s));
        ++c->launches;
        k_invert<<<ge, 256, 0, s>>>(n, perm, pos); ++c->launches;
    }
    tsg_free(c, deg);
    tsg_free(c, deg_alt);
    tsg_free(c, iota);
    // lower triangle: counts -> row_ptr -> fill -> per-row sort
    int32_t *cnt = nullptr;
    TSG_TRY(tsg_alloc_t(c, &cnt, n + 1));
    unsigned long long *ml = reinterpret_cast<unsigned long long *>(c->d_small + 56);
    TSG_TRY(tsg_fill(c, ml, 0, sizeof(unsigned long long), s));
    if (n > 0) {
        k_lower_count<<<gw, 256, 0, s>>>(n, g->rp, g->col, pos, cnt, ml); ++c->launches;
    }
    int64_t *lrp = nullptr;
    TSG_TRY(tsg_alloc_t(c, &lrp, n + 1));
    TSG_TRY(tsg_exclusive_scan_i32_to_i64(c, cnt, lrp, n));
    int64_t h2[2] = {0, 0};
    TSG_CK(cudaMemcpyAsync(&h2[0], lrp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TSG_CK(cudaMemcpyAsync(&h2[1], ml, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TSG_CK(cudaStreamSynchronize(s));
    const int64_t lnnz = h2[0];
    tsg_csr *L = nullptr;
    TSG_TRY(tsg_csr_alloc(c, n, n, lnnz, false, &L));
    TSG_CK(cudaMemcpyAsync(L->rp, lrp, (n + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    tsg_free(c, lrp);
    tsg_free(c, cnt);
    if (n > 0 && lnnz > 0) {
        k_lower_fill<<<gw, 256, 0, s>>>(n, g->rp, g->col, pos, L->rp, L->col); ++c->launches;
        TSG_TRY(sort_rows(c, tmp, n, lnnz, L->rp, L->col));
    }
    if (perm_host && n > 0) {
        // widen on the device, one D2H
        int64_t *p64 = nullptr;
        TSG_TRY(tsg_alloc_t(c, &p64, n));
        k_widen<<<ge, 256, 0, s>>>(n, perm, p64); ++c->launches;
        TSG_CK(cudaMemcpyAsync(perm_host, p64, n * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
        TSG_CK(cudaStreamSynchronize(s));
        tsg_free(c, p64);
    }
    tsg_free(c, perm);
    tsg_free(c, pos);
    TSG_CK(cudaGetLastError());
    L->sorted = 1;
    // a row-distinct graph stays row-distinct under the relabelling (a
    // permutation); duplicates of any other graph survive it
    L->distinct = g->distinct ? 1 : 0;
    L->max_row = h2[1];
    *out = L;
    return TSG_OK;
}

namespace {
__global__ void k_set_values(int64_t n, double v, double *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = v;
}
}  // namespace

extern "C" int tsg_csr_set_values(tsg_ctx *c, tsg_csr *m, double value) {
    TSG_RESOLVE(c, m);
    tsg_plans_forget(c, m);   // a captured multiply may hold its value pointer
    if (m->host_mapped) {
        tsg_set_error("tsg_csr_set_values: matrix lives in mapped host memory");
        return TSG_EARG;
    }
    if (!m->val) TSG_TRY(tsg_alloc_t(c, &m->val, m->nnz > 0 ? m->nnz : 1));
    if (m->nnz > 0) {
        k_set_values<<<grid_for(m->nnz, 256, c->num_sms * 16), 256, 0, c->stream>>>(m->nnz, value, m->val);
        ++c->launches;
    }
    TSG_CK(cudaGetLastError());
    return TSG_OK;
}

extern "C" int tsg_rmat_graph(tsg_ctx *c, int scale, int edge_factor, uint64_t seed, double a,
                              double b, double cq, tsg_csr **out) {
    if (!c || !out || scale < 1 || scale > 30 || edge_factor < 1) {
        tsg_set_error("tsg_rmat_graph: bad arguments (scale %d, edge factor %d)", scale, edge_factor);
        return TSG_EARG;
    }
    const int64_t n = (int64_t)1 << scale, m = n * edge_factor;
    if (2 * m > INT32_MAX) {
        tsg_set_error("tsg_rmat_graph: 2 * edges exceeds 2^31");
        return TSG_EARG;
    }
    const double ab = a + b, abc = a + b + cq;
    cudaStream_t s = c->stream;
    Temp tmp(c);
    uint32_t *u = nullptr, *v = nullptr;
    TSG_TRY(tsg_alloc_t(c, &u, m));
    TSG_TRY(tsg_alloc_t(c, &v, m));
    k_rmat_edges<<<grid_for(m, 256, c->num_sms * 16), 256, 0, s>>>(m, scale, seed, a, ab, abc, u, v);
    ++c->launches;
    // vertex relabelling: rank of each vertex's SplitMix64 key (stable)
    uint64_t *pk = nullptr, *pk_alt = nullptr;
    int32_t *iota = nullptr, *order = nullptr, *perm = nullptr;
    TSG_TRY(tsg_alloc_t(c, &pk, n));
    TSG_TRY(tsg_alloc_t(c, &pk_alt, n));
    TSG_TRY(tsg_alloc_t(c, &iota, n));
    TSG_TRY(tsg_alloc_t(c, &order, n));
    TSG_TRY(tsg_alloc_t(c, &perm, n));
    const unsigned gn = grid_for(n, 256, c->num_sms * 16);
    k_perm_keys<<<gn, 256, 0, s>>>(n, seed ^ SM_GAMMA, pk, iota); ++c->launches;
    size_t need = 0;
    CUB_CK(cub::DeviceRadixSort::SortPairs(nullptr, need, pk, pk_alt, iota, order, n, 0, 64, s));
    TSG_TRY(tmp.ensure(need));
    CUB_CK(cub::DeviceRadixSort::SortPairs(tmp.p, need, pk, pk_alt, iota, order, n, 0, 64, s));
    ++c->launches;
    k_invert<<<gn, 256, 0, s>>>(n, order, perm); ++c->launches;
    tsg_free(c, pk);
    tsg_free(c, pk_alt);
    tsg_free(c, iota);
    tsg_free(c, order);
    // symmetrise, sort, de-duplicate
    uint64_t *keys = nullptr, *keys_alt = nullptr;
    TSG_TRY(tsg_alloc_t(c, &keys, 2 * m));
    TSG_TRY(tsg_alloc_t(c, &keys_alt, 2 * m));
    k_edge_keys<<<grid_for(m, 256, c->num_sms * 16), 256, 0, s>>>(m, scale, u, v, perm, keys);
    ++c->launches;
    tsg_free(c, u);
    tsg_free(c, v);
    tsg_free(c, perm);
    const int end_bit = 2 * scale + 1;   // keys < n^2, sentinel = n^2
    need = 0;
    CUB_CK(cub::DeviceRadixSort::SortKeys(nullptr, need, keys, keys_alt, (int)(2 * m), 0, end_bit, s));
    TSG_TRY(tmp.ensure(need));
    CUB_CK(cub::DeviceRadixSort::SortKeys(tmp.p, need, keys, keys_alt, (int)(2 * m), 0, end_bit, s));
    ++c->launches;
    int *nsel = reinterpret_cast<int *>(c->d_small + 57);
    need = 0;
    CUB_CK(cub::DeviceSelect::Unique(nullptr, need, keys_alt, keys, nsel, (int)(2 * m), s));
    TSG_TRY(tmp.ensure(need));
    CUB_CK(cub::DeviceSelect::Unique(tmp.p, need, keys_alt, keys, nsel, (int)(2 * m), s));
    ++c->launches;
    int hsel = 0;
    uint64_t last = 0;
    TSG_CK(cudaMemcpyAsync(&hsel, nsel, sizeof(int), cudaMemcpyDeviceToHost, s));
    TSG_CK(cudaStreamSynchronize(s));
    if (hsel > 0) {
        TSG_CK(cudaMemcpyAsync(&last, keys + hsel - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
        TSG_CK(cudaStreamSynchronize(s));
    }
    const int64_t nnz = (hsel > 0 && last == (1ull << (2 * scale))) ? hsel - 1 : hsel;
    tsg_free(c, keys_alt);
    tsg_csr *g = nullptr;
    TSG_TRY(tsg_csr_alloc(c, n, n, nnz, false, &g));
    k_keys_to_csr<<<grid_for(n + 1 > nnz ? n + 1 : nnz, 256, c->num_sms * 16), 256, 0, s>>>(
        n, nnz, scale, keys, g->rp, g->col); ++c->launches;
    unsigned long long *ml = reinterpret_cast<unsigned long long *>(c->d_small + 56);
    TSG_TRY(tsg_fill(c, ml, 0, sizeof(unsigned long long), s));
    k_row_max<<<gn, 256, 0, s>>>(n, g->rp, ml); ++c->launches;
    int64_t hml = 0;
    TSG_CK(cudaMemcpyAsync(&hml, ml, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    TSG_CK(cudaStreamSynchronize(s));
    TSG_CK(cudaGetLastError());
    tsg_free(c, keys);
    g->sorted = 1;
    g->distinct = 1;   // de-duplicated keys
    g->max_row = hml;
    *out = g;
    return TSG_OK;
}

const void *tsg_kernel_graph() { return (const void *)k_degrees; }

// ---- B sharded across GPUs: gather the rows of B that A's
// columns select straight from the shards' device memory -- peer HBM over
// NVLink when the shard pointers come from CUDA IPC handles of other GPUs,
// local memory in the single-GPU tests.  The result is a local CSR with all
// of B's rows, the unselected ones empty, so the multiply kernels run on it
// unchanged.  No collective is involved.
namespace {

struct ShardTable {
    int n;
    const int64_t *row_lo;     // device, n + 1 global row bounds
    const int64_t *const *rp;  // device array of n shard row-pointer arrays (shard-local, from 0)
    const int32_t *const *col;
    const double *const *val;
};

__device__ __forceinline__ int shard_of(const ShardTable &t, int64_t k) {
    int lo = 0, hi = t.n - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (t.row_lo[mid] <= k) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ void k_mark_rows(int64_t nnz, const int32_t *__restrict__ acol, uint8_t *__restrict__ need) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nnz;
         t += (int64_t)gridDim.x * blockDim.x)
        need[acol[t]] = 1;
}

__global__ void k_gather_lens(int64_t rows, const uint8_t *__restrict__ need, ShardTable t,
                              int32_t *__restrict__ len) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < rows;
         k += (int64_t)gridDim.x * blockDim.x) {
        int32_t l = 0;
        if (need[k]) {
            const int s = shard_of(t, k);
            const int64_t r = k - t.row_lo[s];
            l = (int32_t)(t.rp[s][r + 1] - t.rp[s][r]);
        }
        len[k] = l;
    }
}

__global__ void k_gather_rows(int64_t rows, const uint8_t *__restrict__ need, ShardTable t,
                              const int64_t *__restrict__ orp, int32_t *__restrict__ ocol,
                              double *__restrict__ oval) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = w; k < rows; k += nw) {
        if (!need[k]) continue;
        const int s = shard_of(t, k);
        const int64_t r = k - t.row_lo[s];
        const int64_t src = t.rp[s][r], len = t.rp[s][r + 1] - src, dst = orp[k];
        for (int64_t q = lane; q < len; q += 32) {
            ocol[dst + q] = t.col[s][src + q];
            if (oval) oval[dst + q] = t.val[s][src + q];
        }
    }
}

}  // namespace

extern "C" int tsg_gather_sharded(tsg_ctx *c, int n_shards, const int64_t *row_lo_host,
                                  const void *const *shard_rp, const void *const *shard_col,
                                  const void *const *shard_val, int64_t b_cols, const tsg_csr *a,
                                  tsg_csr **out) {
    TSG_RESOLVE(c, a);
    if (!c || !a || !out || n_shards < 1 || !row_lo_host) {
        tsg_set_error("tsg_gather_sharded: bad arguments");
        return TSG_EARG;
    }
    const int64_t rows = row_lo_host[n_shards];
    if (a->cols != rows) {
        tsg_set_error("A has %lld cols but the sharded B has %lld rows", (long long)a->cols, (long long)rows);
        return TSG_EDIM;
    }
    const bool values = shard_val && shard_val[0];
    cudaStream_t s = c->stream;
    // device copies of the shard table
    int64_t *d_lo = nullptr;
    const void **d_ptrs = nullptr;
    TSG_TRY(tsg_alloc_t(c, &d_lo, n_shards + 1));
    TSG_TRY(tsg_alloc(c, (void **)&d_ptrs, sizeof(void *) * 3 * n_shards));
    std::vector<const void *> hp(3 * n_shards);
    for (int i = 0; i < n_shards; ++i) {
        hp[i] = shard_rp[i];
        hp[n_shards + i] = shard_col[i];
        hp[2 * n_shards + i] = values ? shard_val[i] : nullptr;
    }
    TSG_CK(cudaMemcpyAsync(d_lo, row_lo_host, (n_shards + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s));
    TSG_CK(cudaMemcpyAsync(d_ptrs, hp.data(), sizeof(void *) * 3 * n_shards, cudaMemcpyHostToDevice, s));
    ShardTable t{n_shards, d_lo, (const int64_t *const *)d_ptrs, (const int32_t *const *)(d_ptrs + n_shards),
                 (const double *const *)(d_ptrs + 2 * n_shards)};
    uint8_t *need = nullptr;
    int32_t *len = nullptr;
    int64_t *rp = nullptr;
    TSG_TRY(tsg_alloc_t(c, &need, rows + 1));
    TSG_TRY(tsg_alloc_t(c, &len, rows + 1));
    TSG_TRY(tsg_alloc_t(c, &rp, rows + 1));
    TSG_TRY(tsg_fill(c, need, 0, rows + 1, s));
    if (a->nnz > 0) {
        k_mark_rows<<<grid_for(a->nnz, 256, c->num_sms * 16), 256, 0, s>>>(a->nnz, a->col, need);
        ++c->launches;
    }
    k_gather_lens<<<grid_for(rows, 256, c->num_sms * 16), 256, 0, s>>>(rows, need, t, len); ++c->launches;
    TSG_TRY(tsg_exclusive_scan_i32_to_i64(c, len, rp, rows));
    TSG_TRY(tsg_put_small(c, rp + rows, 1, 0));
    TSG_CK(cudaStreamSynchronize(s));
    const int64_t nnz = c->h_small[0];
    tsg_csr *B = nullptr;
    TSG_TRY(tsg_csr_alloc(c, rows, b_cols, nnz, values, &B));
    TSG_CK(cudaMemcpyAsync(B->rp, rp, (rows + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
    if (nnz > 0) {
        k_gather_rows<<<grid_for(rows, 8, c->num_sms * 16), 256, 0, s>>>(rows, need, t, rp, B->col,
                                                                         values ? B->val : nullptr);
        ++c->launches;
    }
    TSG_CK(cudaGetLastError());
    TSG_TRY(tsg_free(c, need));
    TSG_TRY(tsg_free(c, len));
    TSG_TRY(tsg_free(c, rp));
    TSG_TRY(tsg_free(c, d_lo));
    TSG_TRY(tsg_free(c, (void *)d_ptrs));
    B->sorted = 0;   // shard rows are taken as they are (tsg_csr_check_sorted below)
    B->max_row = -1;
    TSG_TRY(tsg_csr_check_sorted(c, B));
    *out = B;
    return TSG_OK;
}
