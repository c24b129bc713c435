// tsg_mg.cu -- the per-GPU side of the multi-GPU row partition.
//
// Rows of C are independent (kernel.py:11-14): each GPU (one process per
// GPU) multiplies its contiguous block of A's rows by the whole of B.  B
// reaches a GPU in one of two ways:
//   * replicated: a full local copy (all-gathered over NCCL by the host layer);
//   * sharded: every GPU owns one element range of B's column / value arrays
//     in its own HBM, exported as a CUDA VMM physical allocation (POSIX file
//     descriptor); every GPU maps ALL the shards back to back into ONE
//     reserved virtual range, so B's arrays are contiguous to the unchanged
//     kernels while the pages of remote shards live in peer HBM and are read
//     over NVLink / NVSwitch on demand -- peer HBM as an operand tier, no
//     copy of B and no collective in the multiply.  Only the (small) row
//     pointers are replicated.
// tsg_mg_multiply runs one GPU's block, optionally in streamed-C mode: the
// block is cut into row sub-blocks whose C fits `c_budget_bytes`, each
// sub-block's C is reduced (nnz, fp64 sum, sum of squares) and released --
// the mode for products whose C exceeds HBM (R-MAT scale 25: ~3e12 entries,
// SURVEY.md §7 hard part 1).  B is compressed once for all sub-blocks
// (spgemm_symbolic takes the compressed B as an argument, kernel.py:124).
//
// The CUDA driver's VMM entry points are fetched at run time through
// cudaGetDriverEntryPoint, so libtsg.so links only the runtime and still
// loads on a host without a driver (the CPU-side ABI tests).
#include <cuda.h>

#include <algorithm>
#include <cstring>
#include <unistd.h>
#include <vector>

#include "tsg_internal.cuh"

int tsg_compress_impl(tsg_ctx *c, const tsg_csr *b, tsg_cmat **out);
int tsg_symbolic_impl(tsg_ctx *c, int64_t rows_out, const tsg_csr *a, int64_t a_row_off, int32_t b_lo,
                      int32_t b_hi, const tsg_cmat *cb, const tsg_csr *partial, tsg_vec **out,
                      int64_t **sbound_out);
int tsg_numeric_impl(tsg_ctx *c, int64_t rows_out, int64_t cols_out, const tsg_csr *a, int64_t a_row_off,
                     int32_t b_lo, int32_t b_hi, const tsg_csr *b, const tsg_cmat *cb, const tsg_csr *partial,
                     const tsg_vec *counts, const int64_t *sbound_in, tsg_csr **out, PhaseTimer *pt);

struct tsg_shard {
    CUmemGenericAllocationHandle h;
    CUdeviceptr va;     // local mapping (for filling the shard)
    size_t size;
    int fd;
};

struct tsg_vmap {
    CUdeviceptr va;
    size_t total;
    std::vector<CUmemGenericAllocationHandle> handles;
    std::vector<size_t> sizes;
};

namespace {

struct Drv {
    bool ok = false;
    decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
    decltype(&cuMemCreate) create = nullptr;
    decltype(&cuMemRelease) release = nullptr;
    decltype(&cuMemExportToShareableHandle) export_h = nullptr;
    decltype(&cuMemImportFromShareableHandle) import_h = nullptr;
    decltype(&cuMemAddressReserve) reserve = nullptr;
    decltype(&cuMemAddressFree) addr_free = nullptr;
    decltype(&cuMemMap) map = nullptr;
    decltype(&cuMemUnmap) unmap = nullptr;
    decltype(&cuMemSetAccess) set_access = nullptr;
    decltype(&cuDeviceGet) device_get = nullptr;
};

Drv g_drv;

template <class F>
bool entry(const char *name, F &fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess ||
        !p) {
        cudaGetLastError();
        return false;
    }
    fn = reinterpret_cast<F>(p);
    return true;
}

int drv() {
    if (g_drv.ok) return TSG_OK;
    Drv d;
    bool ok = entry("cuMemGetAllocationGranularity", d.granularity) && entry("cuMemCreate", d.create) &&
              entry("cuMemRelease", d.release) && entry("cuMemExportToShareableHandle", d.export_h) &&
              entry("cuMemImportFromShareableHandle", d.import_h) && entry("cuMemAddressReserve", d.reserve) &&
              entry("cuMemAddressFree", d.addr_free) && entry("cuMemMap", d.map) && entry("cuMemUnmap", d.unmap) &&
              entry("cuMemSetAccess", d.set_access) && entry("cuDeviceGet", d.device_get);
    if (!ok) {
        tsg_set_error("CUDA driver VMM entry points unavailable");
        return TSG_ECUDA;
    }
    d.ok = true;
    g_drv = d;
    return TSG_OK;
}

#define DRV_CK(call)                                                                  \
    do {                                                                              \
        CUresult r_ = (call);                                                         \
        if (r_ != CUDA_SUCCESS) {                                                     \
            tsg_set_error("%s failed (CUresult %d) at %s:%d", #call, (int)r_, __FILE__, \
                          __LINE__);                                                  \
            return TSG_ECUDA;                                                         \
        }                                                                             \
    } while (0)

CUmemAllocationProp shard_prop(int device) {
    CUmemAllocationProp p;
    memset(&p, 0, sizeof(p));
    p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    p.location.id = device;
    p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    return p;
}

int set_rw(int device, CUdeviceptr va, size_t size) {
    CUmemAccessDesc a;
    memset(&a, 0, sizeof(a));
    a.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    a.location.id = device;
    a.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    DRV_CK(g_drv.set_access(va, size, &a, 1));
    return TSG_OK;
}

// per-row-block reduction of a C block: nnz, sum and sum of squares of the
// values (fp64; exact for integer-valued products below 2^53)
__global__ void k_csr_sums(int64_t nnz, const double *__restrict__ v, double *out) {
    double s = 0.0, q = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double x = v[i];
        s += x;
        q += x * x;
    }
    for (int d = 16; d >= 1; d >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, d);
        q += __shfl_xor_sync(0xffffffffu, q, d);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&out[0], s);
        atomicAdd(&out[1], q);
    }
}

}  // namespace

extern "C" int tsg_shard_granularity(tsg_ctx *c, size_t *bytes) {
    TSG_TRY(drv());
    CUmemAllocationProp p = shard_prop(c->device);
    size_t g = 0;
    DRV_CK(g_drv.granularity(&g, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    *bytes = g;
    return TSG_OK;
}

extern "C" int tsg_shard_alloc(tsg_ctx *c, size_t bytes, tsg_shard **out, void **dev_ptr, int *fd,
                               size_t *size) {
    TSG_TRY(drv());
    CUmemAllocationProp p = shard_prop(c->device);
    size_t g = 0;
    DRV_CK(g_drv.granularity(&g, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    const size_t sz = ((bytes ? bytes : 1) + g - 1) / g * g;
    tsg_shard *s = new tsg_shard();
    s->size = sz;
    s->fd = -1;
    CUresult r = g_drv.create(&s->h, sz, &p, 0);
    if (r != CUDA_SUCCESS) {
        delete s;
        tsg_set_error("cuMemCreate of %zu bytes failed (CUresult %d)", sz, (int)r);
        return r == CUDA_ERROR_OUT_OF_MEMORY ? TSG_ECAPACITY : TSG_ECUDA;
    }
    DRV_CK(g_drv.reserve(&s->va, sz, g, 0, 0));
    DRV_CK(g_drv.map(s->va, sz, 0, s->h, 0));
    TSG_TRY(set_rw(c->device, s->va, sz));
    int h = -1;
    DRV_CK(g_drv.export_h(&h, s->h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
    s->fd = h;
    *out = s;
    *dev_ptr = reinterpret_cast<void *>(s->va);
    *fd = h;
    *size = sz;
    return TSG_OK;
}

extern "C" int tsg_shard_free(tsg_ctx *c, tsg_shard *s) {
    if (!s) return TSG_OK;
    cudaDeviceSynchronize();
    (void)c;
    if (g_drv.ok) {
        g_drv.unmap(s->va, s->size);
        g_drv.addr_free(s->va, s->size);
        g_drv.release(s->h);
    }
    if (s->fd >= 0) close(s->fd);
    delete s;
    return TSG_OK;
}

extern "C" int tsg_shard_map(tsg_ctx *c, int n, const int *fds, const size_t *sizes, tsg_vmap **out,
                             void **va) {
    TSG_TRY(drv());
    CUmemAllocationProp p = shard_prop(c->device);
    size_t g = 0;
    DRV_CK(g_drv.granularity(&g, &p, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    size_t total = 0;
    for (int i = 0; i < n; ++i) {
        if (sizes[i] % g) {
            tsg_set_error("shard %d size %zu is not a multiple of the granularity %zu", i, sizes[i], g);
            return TSG_EARG;
        }
        total += sizes[i];
    }
    tsg_vmap *m = new tsg_vmap();
    m->total = total;
    DRV_CK(g_drv.reserve(&m->va, total, g, 0, 0));
    size_t off = 0;
    for (int i = 0; i < n; ++i) {
        CUmemGenericAllocationHandle h;
        DRV_CK(g_drv.import_h(&h, reinterpret_cast<void *>((intptr_t)fds[i]),
                              CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
        DRV_CK(g_drv.map(m->va + off, sizes[i], 0, h, 0));
        m->handles.push_back(h);
        m->sizes.push_back(sizes[i]);
        off += sizes[i];
    }
    // one access descriptor over the whole range: this GPU reads every shard,
    // remote ones over NVLink
    TSG_TRY(set_rw(c->device, m->va, total));
    *out = m;
    *va = reinterpret_cast<void *>(m->va);
    return TSG_OK;
}

extern "C" int tsg_vmap_free(tsg_ctx *c, tsg_vmap *m) {
    if (!m) return TSG_OK;
    (void)c;
    cudaDeviceSynchronize();
    size_t off = 0;
    for (size_t i = 0; i < m->handles.size(); ++i) {
        g_drv.unmap(m->va + off, m->sizes[i]);
        g_drv.release(m->handles[i]);
        off += m->sizes[i];
    }
    g_drv.addr_free(m->va, m->total);
    delete m;
    return TSG_OK;
}

// Synchronous copy on the compute stream between any two addresses the
// device can reach (device, mapped host, VMM ranges).
extern "C" int tsg_memcpy(tsg_ctx *c, void *dst, const void *src, size_t bytes) {
    if (bytes == 0) return TSG_OK;
    TSG_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, c->stream));
    TSG_CK(cudaStreamSynchronize(c->stream));
    return TSG_OK;
}

// A CSR over arrays the caller owns (e.g. B's columns / values in a VMM range
// spanning peer shards); freeing the view leaves the arrays alone.
extern "C" int tsg_csr_view(tsg_ctx *c, int64_t rows, int64_t cols, int64_t nnz, const int64_t *d_rp,
                            const int32_t *d_col, const double *d_val, int sorted, int64_t max_row,
                            tsg_csr **out) {
    (void)c;
    tsg_csr *m = new tsg_csr();
    m->rows = rows;
    m->cols = cols;
    m->nnz = nnz;
    m->rp = const_cast<int64_t *>(d_rp);
    m->col = const_cast<int32_t *>(d_col);
    m->val = const_cast<double *>(d_val);
    m->sorted = sorted ? 1 : 0;
    m->distinct = sorted ? 1 : 0;
    m->max_row = max_row;
    m->borrowed = 1;
    *out = m;
    return TSG_OK;
}

// One GPU's row block of C = A * B.  c_budget_bytes == 0: C materialised and
// returned; > 0: streamed (sub-blocks of A's rows whose C fits the budget,
// reduced and released; *c_out stays NULL).
extern "C" int tsg_mg_multiply(tsg_ctx *c, const tsg_csr *a, const tsg_csr *b, int64_t c_budget_bytes,
                               tsg_csr **c_out, tsg_mg_stats *st) {
    TSG_RESOLVE(c, a);
    TSG_RESOLVE(c, b);
    if (a->cols != b->rows) {
        tsg_set_error("A has %lld cols but B has %lld rows", (long long)a->cols, (long long)b->rows);
        return TSG_EDIM;
    }
    if (!a->val || !b->val) {
        tsg_set_error("numeric multiply requires values on both operands");
        return TSG_EVALID;
    }
    tsg_mg_stats local;
    memset(&local, 0, sizeof(local));
    if (c_out) *c_out = nullptr;
    tsg_cmat *cb = nullptr;
    TSG_TRY(tsg_compress_impl(c, b, &cb));
    double *sums = nullptr;
    TSG_TRY(tsg_alloc_t(c, &sums, 2));
    TSG_TRY(tsg_fill(c, sums, 0, 2 * sizeof(double), c->stream));
    int st_ = TSG_OK;
    if (c_budget_bytes <= 0) {
        tsg_vec *cnt = nullptr;
        st_ = tsg_symbolic_impl(c, a->rows, a, 0, 0, 0x7fffffff, cb, nullptr, &cnt, nullptr);
        tsg_csr *C = nullptr;
        if (st_ == TSG_OK)
            st_ = tsg_numeric_impl(c, a->rows, b->cols, a, 0, 0, 0x7fffffff, b, cb, nullptr, cnt, nullptr, &C,
                                   nullptr);
        if (cnt) tsg_vec_free(c, cnt);
        if (st_ == TSG_OK) {
            local.nnz = C->nnz;
            local.blocks = 1;
            if (C->nnz > 0) {
                k_csr_sums<<<grid_for(C->nnz, 256, c->num_sms * 8), 256, 0, c->stream>>>(C->nnz, C->val, sums);
                ++c->launches;
            }
            if (c_out) *c_out = C;
            else tsg_csr_free(c, C);
        }
    } else {
        // sub-blocks by multiplications (nnz(C_i) <= mults_i): 12 B per entry
        // of C plus the per-row scratch must fit the budget
        int64_t *flops = nullptr;
        std::vector<int64_t> hf(a->rows > 0 ? a->rows : 1);
        TSG_TRY(tsg_alloc_t(c, &flops, a->rows + 1));
        int64_t *brp = b->rp;
        if (a->rows > 0) {
            // per-row multiplications (tsg_row_flops without the host copy)
            tsg_launch_row_flops(c, a, brp, flops);
            TSG_CK(cudaMemcpyAsync(hf.data(), flops, a->rows * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
            TSG_CK(cudaStreamSynchronize(c->stream));
        }
        tsg_free(c, flops);
        // C entries per block <= budget / 16 (12 B of C + symbolic / numeric
        // scratch).  nnz(C_i) <= mults_i, but hashing merges most products
        // (R-MAT A*A: ~3 per entry): each block is sized by the largest
        // entries-per-multiplication ratio seen so far (x 1.25), starting at 1
        const int64_t cap_entries = std::max<int64_t>(c_budget_bytes / 16, 1);
        struct Coarse {   // coarse arena classes for the blocks' varying scratch sizes
            tsg_ctx *c;
            explicit Coarse(tsg_ctx *x) : c(x) { ++c->coarse_alloc; }
            ~Coarse() { --c->coarse_alloc; }
        } coarse(c);
        // one C reservoir of cap_entries for every block (same size every
        // call, so the arena hands the same two blocks back)
        struct Reservoir {
            tsg_ctx *c;
            explicit Reservoir(tsg_ctx *x) : c(x) {}
            ~Reservoir() {
                tsg_free(c, c->c_res_col);
                tsg_free(c, c->c_res_val);
                c->c_res_col = nullptr;
                c->c_res_val = nullptr;
                c->c_res_cap = 0;
            }
        } reservoir(c);
        if (tsg_alloc_t(c, &c->c_res_col, (size_t)cap_entries) == TSG_OK &&
            tsg_alloc_t(c, &c->c_res_val, (size_t)cap_entries) == TSG_OK)
            c->c_res_cap = cap_entries;
        // the last call's ratio (same B, similar A blocks): the first block
        // is sized like the rest, so the arena reuses its C blocks
        double ratio = c->mg_ratio > 0 ? c->mg_ratio : 1.0;
        int64_t lo = 0;
        while (lo < a->rows && st_ == TSG_OK) {
            const double cap_mults = (double)cap_entries / std::min(1.0, 1.25 * ratio);
            int64_t hi = lo, acc = 0;
            while (hi < a->rows && (hi == lo || (double)(acc + hf[hi]) <= cap_mults)) acc += hf[hi++];
            tsg_csr *as = nullptr;
            st_ = tsg_csr_slice_rows(c, a, lo, hi, &as);
            if (st_ != TSG_OK) break;
            as->sorted = a->sorted;
            as->distinct = a->distinct;
            as->max_row = a->max_row;
            tsg_vec *cnt = nullptr;
            st_ = tsg_symbolic_impl(c, as->rows, as, 0, 0, 0x7fffffff, cb, nullptr, &cnt, nullptr);
            tsg_csr *C = nullptr;
            if (st_ == TSG_OK)
                st_ = tsg_numeric_impl(c, as->rows, b->cols, as, 0, 0, 0x7fffffff, b, cb, nullptr, cnt, nullptr,
                                       &C, nullptr);
            if (cnt) tsg_vec_free(c, cnt);
            if (st_ == TSG_OK) {
                local.nnz += C->nnz;
                if (C->nnz > 0) {
                    k_csr_sums<<<grid_for(C->nnz, 256, c->num_sms * 8), 256, 0, c->stream>>>(C->nnz, C->val,
                                                                                           sums);
                    ++c->launches;
                }
                local.max_block_nnz = std::max(local.max_block_nnz, C->nnz);
                if (acc > 0) ratio = std::max(local.blocks ? ratio : 0.0, (double)C->nnz / (double)acc);
                c->mg_ratio = ratio;
                tsg_csr_free(c, C);
            }
            tsg_csr_free(c, as);
            ++local.blocks;
            lo = hi;
        }
    }
    tsg_cmat_free(c, cb);
    double h[2] = {0.0, 0.0};
    TSG_CK(cudaMemcpyAsync(h, sums, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    TSG_CK(cudaStreamSynchronize(c->stream));
    tsg_free(c, sums);
    local.value_sum = h[0];
    local.value_sumsq = h[1];
    if (st) *st = local;
    if (st_ != TSG_OK) return st_;
    return tsg_check_kernel_errors(c, "mg multiply");
}

const void *tsg_kernel_mg() { return (const void *)k_csr_sums; }
