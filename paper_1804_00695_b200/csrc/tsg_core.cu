// tsg_core.cu -- context, device memory, scans, operand upload/download.
//
// Host<->device conversion of the reference's int64 column arrays happens on
// the device (int64 staging -> int32 device columns on upload, the reverse on
// download) so the host never runs an O(nnz) numpy conversion.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <ctime>
#include <map>
#include <mutex>
#include <unordered_map>

#include <cuda.h>
#include <vector>

#include "tsg_internal.cuh"
#include <atomic>

static thread_local char g_err[1024] = "";

void tsg_set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int tsg_cuda_fail(cudaError_t e, const char *what, const char *file, int line) {
    tsg_set_error("CUDA error %s (%s) in %s at %s:%d", cudaGetErrorName(e),
                  cudaGetErrorString(e), what, file, line);
    return TSG_ECUDA;
}

extern "C" const char *tsg_last_error(void) { return g_err; }
extern "C" int tsg_abi_version(void) { return TSG_ABI_VERSION; }

extern "C" int tsg_device_count(int *count) {
    TSG_CK(cudaGetDeviceCount(count));
    return TSG_OK;
}

// ------------------------------------------------------------------ context

extern "C" int tsg_init(int device, tsg_ctx **out) {
    if (!out) { tsg_set_error("null output handle"); return TSG_EARG; }
    int n = 0;
    TSG_CK(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) {
        tsg_set_error("device %d not present (%d visible)", device, n);
        return TSG_EARG;
    }
    TSG_CK(cudaSetDevice(device));
    tsg_ctx *c = new tsg_ctx();   // value-initialised (all zero)
    c->device = device;
    cudaDeviceProp prop;
    TSG_CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
        tsg_set_error("libtsg is built for sm_100a (B200); device %d is sm_%d%d", device,
                      prop.major, prop.minor);
        delete c;
        return TSG_ECUDA;
    }
    c->num_sms = prop.multiProcessorCount;
    c->smem_optin = prop.sharedMemPerBlockOptin;
    TSG_CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    TSG_CK(cudaStreamCreateWithFlags(&c->copy_in, cudaStreamNonBlocking));
    TSG_CK(cudaStreamCreateWithFlags(&c->copy_out, cudaStreamNonBlocking));
    int prio_lo = 0, prio_hi = 0;
    TSG_CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    for (int i = 0; i < tsg_ctx::NAUX; ++i) {
        // forked bins (BinFork) run at the highest priority: the block
        // scheduler then dispatches a small bin's blocks as soon as the big
        // bin's first blocks retire instead of after all of them
        TSG_CK(cudaStreamCreateWithPriority(&c->aux[i], cudaStreamNonBlocking, prio_hi));
        TSG_CK(cudaEventCreateWithFlags(&c->ev_join[i], cudaEventDisableTiming));
    }
    TSG_CK(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    TSG_CK(cudaStreamCreateWithPriority(&c->convert, cudaStreamNonBlocking, prio_hi));
    TSG_CK(cudaStreamCreateWithFlags(&c->copy_in2, cudaStreamNonBlocking));
    TSG_CK(cudaStreamCreateWithPriority(&c->widen, cudaStreamNonBlocking, prio_hi));
    // keep freed blocks cached in the default pool: no OS round trips per call
    cudaMemPool_t pool;
    TSG_CK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    TSG_CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    TSG_CK(cudaMalloc(&c->d_err, 4 * sizeof(int)));
    TSG_CK(cudaMemset(c->d_err, 0, 4 * sizeof(int)));
    TSG_CK(cudaMalloc(&c->d_small, 64 * sizeof(int64_t)));
    TSG_CK(cudaMemset(c->d_small, 0, 64 * sizeof(int64_t)));   // counters (e.g. slot 60) start at 0
    TSG_CK(cudaHostAlloc(&c->h_small, 64 * sizeof(int64_t), cudaHostAllocMapped));
    TSG_CK(cudaHostGetDevicePointer(&c->hd_small, c->h_small, 0));
    memset(c->h_small, 0, 64 * sizeof(int64_t));   // sequence words start below any issued seq
    int init_err[2] = {0, 0x7fffffff};
    TSG_CK(cudaMemcpy(c->d_err, init_err, sizeof(init_err), cudaMemcpyHostToDevice));
    for (int i = 0; i < 8; i++) TSG_CK(cudaEventCreate(&c->ev[i]));
    for (int i = 0; i < 8; i++) TSG_CK(cudaEventCreate(&c->ev_user[i]));
    for (int i = 0; i < 2; i++) {
        TSG_CK(cudaEventCreate(&c->ev_num[i]));
        TSG_CK(cudaEventCreate(&c->ev_sym[i]));
    }
    for (int i = 0; i < 2 * tsg_ctx::NRING; i++) TSG_CK(cudaEventCreate(&c->ev_ring[i]));
    for (int i = 0; i < tsg_ctx::NRING; i++) c->ring_timed[i] = -1;
    c->num_calls = 0;
    c->pending = nullptr;
    c->phase_n = c->phase_total = c->phase_dirty = 0;
    c->lb_state = nullptr;
    c->lb_cap = 0;
    c->lb_epoch = 0;
    c->lb_counter = nullptr;
    c->lb_base = 0;
    c->timing = 0;
    // every kernel loaded now, not at its first launch (see tsg_preload_module_of)
    TSG_TRY(tsg_preload_module_of(tsg_kernel_core()));
    TSG_TRY(tsg_preload_module_of(tsg_kernel_compress()));
    TSG_TRY(tsg_preload_module_of(tsg_kernel_spgemm()));
    TSG_TRY(tsg_preload_module_of(tsg_kernel_masked()));
    TSG_TRY(tsg_preload_module_of(tsg_kernel_chunk()));
    TSG_TRY(tsg_preload_module_of(tsg_kernel_graph()));
    TSG_TRY(tsg_preload_module_of(tsg_kernel_build()));
    TSG_TRY(tsg_preload_module_of(tsg_kernel_rap()));
    TSG_TRY(tsg_preload_module_of(tsg_kernel_mg()));
    *out = c;
    return TSG_OK;
}

extern "C" int tsg_destroy(tsg_ctx *c) {
    if (!c) return TSG_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    tsg_free(c, c->lb_state);
    tsg_free(c, c->lb_counter);
    tsg_arena_trim(c);
    for (int i = 0; i < 8; i++) cudaEventDestroy(c->ev[i]);
    cudaFree(c->d_err);
    cudaFree(c->d_small);
    cudaFreeHost(c->h_small);
    cudaStreamDestroy(c->stream);
    cudaStreamDestroy(c->copy_in);
    cudaStreamDestroy(c->copy_out);
    for (int i = 0; i < tsg_ctx::NAUX; ++i) {
        cudaStreamDestroy(c->aux[i]);
        cudaEventDestroy(c->ev_join[i]);
    }
    cudaEventDestroy(c->ev_fork);
    cudaStreamDestroy(c->convert);
    cudaStreamDestroy(c->copy_in2);
    cudaStreamDestroy(c->widen);
    delete c;
    return TSG_OK;
}

extern "C" int tsg_sync(tsg_ctx *c) {
    TSG_CK(cudaStreamSynchronize(c->stream));
    if (c->pending) return tsg_check_kernel_errors(c, c->pending);
    return TSG_OK;
}

extern "C" int tsg_numeric_calls(tsg_ctx *c, int64_t *n) {
    *n = c->num_calls;
    return TSG_OK;
}

extern "C" int tsg_numeric_ms(tsg_ctx *c, int64_t call, float *ms) {
    if (call < 0 || call >= c->num_calls || c->num_calls - call > tsg_ctx::NRING ||
        c->ring_timed[call % tsg_ctx::NRING] != call) {
        tsg_set_error("numeric call %lld is not in the timing ring (timing off or too old)",
                      (long long)call);
        return TSG_EARG;
    }
    const int k = (int)(call % tsg_ctx::NRING);
    TSG_CK(cudaEventSynchronize(c->ev_ring[2 * k + 1]));
    TSG_CK(cudaEventElapsedTime(ms, c->ev_ring[2 * k], c->ev_ring[2 * k + 1]));
    return TSG_OK;
}

extern "C" int tsg_mem_in_use(tsg_ctx *c, int64_t *bytes) {
    *bytes = c->bytes_in_use;
    return TSG_OK;
}

extern "C" int tsg_pool_reserved(tsg_ctx *c, int64_t *bytes) {
    cudaMemPool_t pool;
    TSG_CK(cudaDeviceGetDefaultMemPool(&pool, c->device));
    uint64_t v = 0;
    TSG_CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &v));
    *bytes = (int64_t)v;
    return TSG_OK;
}

extern "C" int tsg_set_timing(tsg_ctx *c, int enabled) {
    c->timing = enabled ? 1 : 0;
    return TSG_OK;
}

extern "C" int tsg_stream(tsg_ctx *c, void **stream) {
    *stream = (void *)c->stream;
    return TSG_OK;
}

extern "C" int tsg_event_record(tsg_ctx *c, int slot) {
    if (slot < 0 || slot >= 8) {
        tsg_set_error("event slot %d out of range", slot);
        return TSG_EARG;
    }
    TSG_CK(cudaEventRecord(c->ev_user[slot], c->stream));
    return TSG_OK;
}

extern "C" int tsg_event_elapsed(tsg_ctx *c, int from, int to, float *ms) {
    if (from < 0 || from >= 8 || to < 0 || to >= 8) {
        tsg_set_error("event slot out of range");
        return TSG_EARG;
    }
    TSG_CK(cudaEventSynchronize(c->ev_user[to]));
    TSG_CK(cudaEventElapsedTime(ms, c->ev_user[from], c->ev_user[to]));
    return TSG_OK;
}

extern "C" int tsg_get_stats(tsg_ctx *c, tsg_stats *st) {
    st->launches = c->launches;
    st->symbolic_ms = 0.f;
    st->numeric_ms = 0.f;
    if (c->timing) {
        TSG_CK(cudaStreamSynchronize(c->stream));
        if (cudaEventElapsedTime(&st->symbolic_ms, c->ev_sym[0], c->ev_sym[1]) != cudaSuccess) {
            cudaGetLastError();
            st->symbolic_ms = -1.f;
        }
        if (cudaEventElapsedTime(&st->numeric_ms, c->ev_num[0], c->ev_num[1]) != cudaSuccess) {
            cudaGetLastError();
            st->numeric_ms = -1.f;
        }
    }
    return TSG_OK;
}

extern "C" int tsg_last_phase_ms(tsg_ctx *c, float *out, int n) {
    if (c->phase_dirty) {   // evaluated on demand: multiplies never wait for their timers
        const int m = c->phase_n;
        TSG_CK(cudaEventSynchronize(c->ev[m - 1]));
        for (int i = 0; i + 1 < m && i < 8; i++)
            TSG_CK(cudaEventElapsedTime(&c->phase_ms[i], c->ev[i], c->ev[i + 1]));
        if (c->phase_total < 8)
            TSG_CK(cudaEventElapsedTime(&c->phase_ms[c->phase_total], c->ev[0], c->ev[m - 1]));
        c->phase_dirty = 0;
    }
    for (int i = 0; i < n && i < 8; i++) out[i] = c->phase_ms[i];
    return TSG_OK;
}

void PhaseTimer::finish(int total_slot) {
    if (!ctx->timing || n < 2) return;
    ctx->phase_n = n;
    ctx->phase_total = total_slot;
    ctx->phase_dirty = 1;
}

// ------------------------------------------------------------------ memory


static double now_us() {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e6 + ts.tv_nsec * 1e-3;
}

int tsg_trace_enabled() {
    static int on = -1;
    if (on < 0) {
        const char *e = getenv("TSG_TRACE");
        on = (e && *e && *e != '0') ? 1 : 0;
    }
    return on;
}

void tsg_trace_host(const char *what) {
    static int on = -1;
    if (on < 0) on = getenv("TSG_CHUNK_TIMELINE") != nullptr;
    if (on) fprintf(stderr, "[tsg host abs] %.1f us %s\n", now_us(), what);
}

void tsg_trace(tsg_ctx *c, const char *what, int64_t arg) {
    if (!tsg_trace_enabled()) return;
    double t0 = now_us();
    cudaStreamSynchronize(c->stream);
    double t1 = now_us();
    fprintf(stderr, "[tsg %12.1f us] %-28s %14lld  (gpu drain %.1f us)\n", t0, what, (long long)arg,
            t1 - t0);
}

// Caching layer over cudaMallocAsync.  Per-call temporaries (compressed B,
// bins, row lists, bounds) and outputs are recycled through a best-fit free
// list instead of going back to the driver pool: measured on B200, a 445 MB
// cudaMallocAsync right after a same-size cudaFreeAsync can block the host
// for 0.4-100 ms.  Blocks are only reused in the context's compute-stream
// order (every libtsg kernel and copy runs on that stream or is joined to it
// by an event before the memory is released).
struct Arena {
    std::mutex mu;
    std::multimap<size_t, void *> free_blocks;   // size class -> block
    std::unordered_map<void *, size_t> live;     // block -> size class
    size_t cached = 0;
};

static std::mutex g_arena_mu;
static std::unordered_map<const tsg_ctx *, Arena *> g_arenas;

static Arena *arena_of(tsg_ctx *c) {
    std::lock_guard<std::mutex> g(g_arena_mu);
    Arena *&a = g_arenas[c];
    if (!a) a = new Arena();
    return a;
}

static size_t size_class(size_t bytes, bool coarse = false) {
    if (bytes <= 4096) return 4096;
    if (bytes <= (1u << 20)) {
        size_t p = 4096;
        while (p < bytes) p <<= 1;
        return p;
    }
    if (!coarse || bytes < ((size_t)1 << 30))
        return (bytes + (1u << 20) - 1) & ~(size_t)((1u << 20) - 1);   // 1 MiB granules
    // coarse (streamed tsg_mg_multiply), >= 1 GiB: four classes per octave
    // (<= 25 % slack), so its varying C blocks land in a few sizes the cache
    // reuses instead of forcing an out-of-memory trim and a multi-GB re-map
    // (R-MAT scale 21: 17.3 -> 3.6 s).  Not for the chunked executors, whose
    // HBM budget counts every byte.
    size_t p = (size_t)1 << 30;
    while (p * 2 <= bytes) p <<= 1;
    const size_t q = p / 4;
    return (bytes + q - 1) / q * q;
}

static const size_t ARENA_CACHE_LIMIT = (size_t)48 << 30;

int tsg_alloc(tsg_ctx *c, void **p, size_t bytes) {
    *p = nullptr;
    tsg_trace(c, "alloc", (int64_t)bytes);
    Arena *A = arena_of(c);
    size_t cls = size_class(bytes, c->coarse_alloc != 0);
    {
        std::lock_guard<std::mutex> g(A->mu);
        auto it = A->free_blocks.lower_bound(cls);
        // best fit, <= 25% slack; in coarse mode (streamed multiply) blocks of
        // >= 256 MiB take up to 2x (its C blocks vary in size: a miss there
        // re-maps tens of GB after an out-of-memory trim, ~0.25 s per block)
        const size_t slack = c->coarse_alloc && cls >= ((size_t)256 << 20) ? cls : cls / 4;
        if (it != A->free_blocks.end() && it->first <= cls + slack) {
            *p = it->second;
            size_t got = it->first;
            A->free_blocks.erase(it);
            A->cached -= got;
            A->live[*p] = got;
            c->bytes_in_use += (int64_t)got;
            if (c->bytes_in_use > c->bytes_peak) c->bytes_peak = c->bytes_in_use;
            if (c->capture_owned) c->capture_owned->push_back(*p);
            return TSG_OK;
        }
    }
    void *raw = nullptr;
    if (c->capture_owned) {
        // inside a graph capture no stream-ordered allocation may be issued:
        // a plain cudaMalloc (a block the plan keeps for its lifetime)
        cudaError_t e2 = cudaMalloc(&raw, cls);
        if (e2 != cudaSuccess) {
            cudaGetLastError();
            c->capture_failed = 1;
            tsg_set_error("device allocation of %zu bytes failed during capture", bytes);
            return TSG_ECAPACITY;
        }
        std::lock_guard<std::mutex> g(A->mu);
        A->live[raw] = cls;
        c->bytes_in_use += (int64_t)cls;
        c->capture_owned->push_back(raw);
        *p = raw;
        return TSG_OK;
    }
    cudaError_t e = cudaMallocAsync(&raw, cls, c->stream);
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        tsg_arena_trim(c);   // give the cache back to the driver and retry once
        e = cudaMallocAsync(&raw, cls, c->stream);
        if (e == cudaErrorMemoryAllocation) {
            cudaGetLastError();
            tsg_set_error("device allocation of %zu bytes failed (out of HBM)", bytes);
            return TSG_ECAPACITY;
        }
    }
    if (e != cudaSuccess) return tsg_cuda_fail(e, "cudaMallocAsync", __FILE__, __LINE__);
    std::lock_guard<std::mutex> g(A->mu);
    A->live[raw] = cls;
    c->bytes_in_use += (int64_t)cls;
    if (c->bytes_in_use > c->bytes_peak) c->bytes_peak = c->bytes_in_use;
    *p = raw;
    return TSG_OK;
}

int tsg_free(tsg_ctx *c, void *p) {
    if (!p) return TSG_OK;
    if (c->capture_owned) {   // the capturing plan keeps every block it touched
        c->capture_owned->push_back(p);
        return TSG_OK;
    }
    Arena *A = arena_of(c);
    std::lock_guard<std::mutex> g(A->mu);
    auto it = A->live.find(p);
    if (it == A->live.end()) {
        TSG_CK(cudaFreeAsync(p, c->stream));
        return TSG_OK;
    }
    size_t cls = it->second;
    A->live.erase(it);
    c->bytes_in_use -= (int64_t)cls;
    if (cls > ARENA_CACHE_LIMIT) {
        TSG_CK(cudaFreeAsync(p, c->stream));
        return TSG_OK;
    }
    // over the limit: evict the largest cached blocks, keep the one just
    // freed (a workload's own blocks come back next call; stale ones from an
    // earlier workload otherwise pin the cache and force re-maps)
    while (A->cached + cls > ARENA_CACHE_LIMIT && !A->free_blocks.empty()) {
        auto last = std::prev(A->free_blocks.end());
        TSG_CK(cudaFreeAsync(last->second, c->stream));
        A->cached -= last->first;
        A->free_blocks.erase(last);
    }
    A->free_blocks.emplace(cls, p);
    A->cached += cls;
    return TSG_OK;
}

// Blocks a destroyed plan owned go back to the arena (after the device is
// done with them: the caller synchronises).
void tsg_arena_return(tsg_ctx *c, const std::vector<void *> &blocks) {
    for (void *p : blocks) tsg_free(c, p);
}

// ---- pinned host pool: result arrays handed to the caller live here, so the
// D2H of a product (and its re-upload as the next operand) runs at full
// PCIe rate instead of the driver's pageable staging rate.
static std::mutex g_host_mu;
static std::multimap<size_t, void *> g_host_free;
static std::unordered_map<void *, size_t> g_host_live;
static size_t g_host_cached = 0;
static const size_t HOST_CACHE_LIMIT = (size_t)16 << 30;

extern "C" int tsg_host_alloc(size_t bytes, void **out) {
    *out = nullptr;
    size_t cls = size_class(bytes ? bytes : 1);
    {
        std::lock_guard<std::mutex> g(g_host_mu);
        auto it = g_host_free.lower_bound(cls);
        if (it != g_host_free.end() && it->first <= cls + cls / 4) {
            *out = it->second;
            g_host_live[*out] = it->first;
            g_host_cached -= it->first;
            g_host_free.erase(it);
            return TSG_OK;
        }
    }
    void *p = nullptr;
    cudaError_t e = cudaHostAlloc(&p, cls, cudaHostAllocPortable);
    if (e != cudaSuccess) {
        cudaGetLastError();
        // pinning can fail under memlock limits: fall back to pageable memory
        p = malloc(cls);
        if (!p) {
            tsg_set_error("host allocation of %zu bytes failed", bytes);
            return TSG_ECAPACITY;
        }
        cls |= 1;   // tag: not pinned
    }
    std::lock_guard<std::mutex> g(g_host_mu);
    g_host_live[p] = cls;
    *out = p;
    return TSG_OK;
}

extern "C" int tsg_host_free(void *p) {
    if (!p) return TSG_OK;
    std::lock_guard<std::mutex> g(g_host_mu);
    auto it = g_host_live.find(p);
    if (it == g_host_live.end()) return TSG_OK;
    size_t cls = it->second;
    g_host_live.erase(it);
    if (cls & 1) {
        free(p);
        return TSG_OK;
    }
    if (g_host_cached + cls > HOST_CACHE_LIMIT) {
        cudaFreeHost(p);
        return TSG_OK;
    }
    g_host_free.emplace(cls, p);
    g_host_cached += cls;
    return TSG_OK;
}

int tsg_arena_trim(tsg_ctx *c) {
    Arena *A = arena_of(c);
    std::lock_guard<std::mutex> g(A->mu);
    for (auto &kv : A->free_blocks) cudaFreeAsync(kv.second, c->stream);
    A->free_blocks.clear();
    A->cached = 0;
    cudaStreamSynchronize(c->stream);
    return TSG_OK;
}

int tsg_func_smem(const void *kernel, size_t bytes) {
    static std::mutex mu;
    static std::unordered_map<const void *, size_t> granted[64];
    int dev = 0;
    TSG_CK(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> g(mu);
    size_t &have = granted[dev & 63][kernel];
    if (bytes > have) {
        TSG_CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        have = bytes;
    }
    return TSG_OK;
}

int tsg_launch_check(const char *kernel, int bin, unsigned grid, int block, size_t smem) {
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return TSG_OK;
    tsg_set_error("launch of %s (bin %d, grid %u, block %d, dynamic smem %zu) failed: %s", kernel,
                  bin, grid, block, smem, cudaGetErrorString(e));
    return TSG_ECUDA;
}

namespace {
__global__ void k_put_small(const int64_t *__restrict__ src, int64_t *__restrict__ dst, int n) {
    if (threadIdx.x < n) dst[threadIdx.x] = src[threadIdx.x];
}
}  // namespace

namespace {
__global__ void k_fill(uint8_t *__restrict__ p, uint32_t word, size_t bytes) {
    pdl_wait();
    // 16-byte body (p is at least 16-byte aligned for arena blocks; the
    // generic head / tail loops cover any other pointer)
    const size_t head = (16 - ((uintptr_t)p & 15)) & 15;
    const size_t h = head < bytes ? head : bytes;
    const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t nth = (size_t)gridDim.x * blockDim.x;
    for (size_t i = tid; i < h; i += nth) p[i] = (uint8_t)word;
    uint4 *q = reinterpret_cast<uint4 *>(p + h);
    const size_t nv = (bytes - h) / 16;
    const uint4 v = make_uint4(word, word, word, word);
    for (size_t i = tid; i < nv; i += nth) q[i] = v;
    for (size_t i = h + nv * 16 + tid; i < bytes; i += nth) p[i] = (uint8_t)word;
}
}  // namespace

const void *tsg_kernel_core() { return (const void *)k_fill; }

int tsg_fill(tsg_ctx *c, void *p, int byte, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return TSG_OK;
    const uint32_t b = (uint32_t)(byte & 0xff);
    const uint32_t word = b | (b << 8) | (b << 16) | (b << 24);
    size_t blocks = (bytes / 16 + 255) / 256;
    if (blocks < 1) blocks = 1;
    const size_t cap = (size_t)c->num_sms * 8;
    if (blocks > cap) blocks = cap;
    TSG_CK(launch_pdl(k_fill, (unsigned)blocks, 256, 0, s, reinterpret_cast<uint8_t *>(p), word, bytes));
    ++c->launches;
    TSG_CK(cudaGetLastError());
    return TSG_OK;
}

int tsg_preload_module_of(const void *kernel) {
    typedef CUresult (*FnGetModule)(CUmodule *, CUfunction);
    typedef CUresult (*FnCount)(unsigned int *, CUmodule);
    typedef CUresult (*FnEnum)(CUfunction *, unsigned int, CUmodule);
    typedef CUresult (*FnLoad)(CUfunction);
    static FnGetModule get_module = nullptr;
    static FnCount count_fns = nullptr;
    static FnEnum enum_fns = nullptr;
    static FnLoad load_fn = nullptr;
    if (!load_fn) {
        cudaDriverEntryPointQueryResult q;
        void *p = nullptr;
        if (cudaGetDriverEntryPoint("cuFuncGetModule", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return TSG_OK;   // older driver: keep lazy loading
        get_module = (FnGetModule)p;
        if (cudaGetDriverEntryPoint("cuModuleGetFunctionCount", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return TSG_OK;
        count_fns = (FnCount)p;
        if (cudaGetDriverEntryPoint("cuModuleEnumerateFunctions", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return TSG_OK;
        enum_fns = (FnEnum)p;
        if (cudaGetDriverEntryPoint("cuFuncLoad", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            return TSG_OK;
        load_fn = (FnLoad)p;
    }
    cudaFunction_t f = nullptr;
    TSG_CK(cudaGetFuncBySymbol(&f, kernel));
    CUmodule mod = nullptr;
    unsigned n = 0;
    if (get_module((CUmodule *)&mod, (CUfunction)f) != CUDA_SUCCESS || count_fns(&n, mod) != CUDA_SUCCESS)
        return TSG_OK;
    std::vector<CUfunction> fs(n);
    if (n && enum_fns(fs.data(), n, mod) == CUDA_SUCCESS)
        for (CUfunction g : fs) load_fn(g);
    return TSG_OK;
}

int tsg_copy(void *dst, const void *src, size_t bytes, cudaMemcpyKind kind, cudaStream_t s) {
    constexpr size_t PIECE = (size_t)256 << 20;
    for (size_t o = 0; o < bytes; o += PIECE) {
        const size_t n = bytes - o < PIECE ? bytes - o : PIECE;
        TSG_CK(cudaMemcpyAsync(static_cast<char *>(dst) + o, static_cast<const char *>(src) + o, n, kind, s));
    }
    return TSG_OK;
}

int tsg_lookback_state(tsg_ctx *c, int64_t tiles, unsigned long long **state, unsigned *epoch) {
    bool clear = false;
    if (tiles > c->lb_cap) {
        tsg_free(c, c->lb_state);
        c->lb_cap = tiles > 4096 ? tiles : 4096;
        TSG_TRY(tsg_alloc_t(c, &c->lb_state, c->lb_cap));
        clear = true;
    }
    if (++c->lb_epoch > 0x3fffu) {   // wrapped: words of an old call could match again
        c->lb_epoch = 1;
        clear = true;
    }
    if (clear) TSG_TRY(tsg_fill(c, c->lb_state, 0, (size_t)c->lb_cap * 8, c->stream));
    *state = c->lb_state;
    *epoch = c->lb_epoch;
    return TSG_OK;
}

int tsg_lookback_counter(tsg_ctx *c, int64_t tiles, unsigned long long **counter,
                         unsigned long long *base) {
    if (!c->lb_counter) {
        TSG_TRY(tsg_alloc_t(c, &c->lb_counter, 1));
        TSG_TRY(tsg_fill(c, c->lb_counter, 0, sizeof(unsigned long long), c->stream));
        c->lb_base = 0;
    }
    *counter = c->lb_counter;
    *base = c->lb_base;
    c->lb_base += (unsigned long long)tiles;
    return TSG_OK;
}

int tsg_put_small(tsg_ctx *c, const int64_t *src, int n, int slot) {
    k_put_small<<<1, 32, 0, c->stream>>>(src, c->hd_small + slot, n); ++c->launches;
    TSG_CK(cudaGetLastError());
    return TSG_OK;
}

int tsg_wait_mapped(tsg_ctx *c, int slot, int64_t seq) {
    volatile int64_t *w = c->h_small + slot;
    for (unsigned spin = 1;; ++spin) {
        if (*w == seq) break;
        if ((spin & 4095u) == 0) {
            const cudaError_t q = cudaStreamQuery(c->stream);
            if (q == cudaErrorNotReady) continue;
            if (*w == seq) break;
            TSG_CK(q);
            tsg_set_error("mapped result word %d never arrived (expected %lld)", slot, (long long)seq);
            return TSG_ECUDA;
        }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    return TSG_OK;
}

int tsg_pending_errors(tsg_ctx *c) {
    const int *h = reinterpret_cast<const int *>(c->h_small + 62);
    if (h[0] == KERR_NONE) return TSG_OK;
    return tsg_check_kernel_errors(c, c->pending ? c->pending : "kernel");
}

int tsg_check_kernel_errors(tsg_ctx *c, const char *phase) {
    int h[2];
    c->pending = nullptr;
    TSG_CK(cudaGetLastError());
    TSG_TRY(tsg_put_small(c, reinterpret_cast<const int64_t *>(c->d_err), 1, 63));
    TSG_CK(cudaStreamSynchronize(c->stream));
    memcpy(h, c->h_small + 63, sizeof(h));
    if (h[0] == KERR_NONE) return TSG_OK;
    int init_err[2] = {0, 0x7fffffff};
    TSG_CK(cudaMemcpyAsync(c->d_err, init_err, sizeof(init_err), cudaMemcpyHostToDevice, c->stream));
    TSG_CK(cudaStreamSynchronize(c->stream));
    switch (h[0]) {
    case KERR_COUNT:
        tsg_set_error("%s: row %d: symbolic count disagrees with the entries accumulated", phase, h[1]);
        return TSG_EKERNEL;
    case KERR_PROBE:
        tsg_set_error("%s: row %d: accumulator probe overflow (table full)", phase, h[1]);
        return TSG_EKERNEL;
    case KERR_NOTLOWER:
        tsg_set_error("row %d has a column >= its row: not strictly lower triangular", h[1]);
        return TSG_EVALID;
    case KERR_ROWSIZE:
        tsg_set_error("chunked result rows disagree with symbolic counts (row %d)", h[1]);
        return TSG_EDIM;
    case KERR_COLRANGE:
        tsg_set_error("%s: column index out of range in row %d", phase, h[1]);
        return TSG_EVALID;
    default:
        tsg_set_error("%s: internal kernel error %d at row %d", phase, h[0], h[1]);
        return TSG_EKERNEL;
    }
}

// ------------------------------------------------------------------ scan
// Exclusive scans of non-negative counts (row lengths, set counts), result
// total in out[n].  Up to SMALL_SCAN elements: one 256-thread block.  Above:
// ONE single-pass launch with decoupled look-back -- tiles take their index
// from an atomic counter (so a tile only ever waits on tiles that are already
// running), publish their aggregate, and warp 0 walks back over a 32-tile
// window until it meets a published inclusive prefix.  State words pack
// (value << 2 | flag) into one 64-bit store, so value and flag are observed
// together; flag 1 = aggregate, 2 = inclusive prefix.

namespace {
constexpr int LB_BS = 256;
#ifndef TSG_LB_IT
#define TSG_LB_IT 4
#endif
static_assert(TSG_LB_IT % 4 == 0, "scan tiles load 16-byte vectors");
constexpr int LB_IT = TSG_LB_IT;   // elements per thread: 1024-element tiles, many CTAs in flight
constexpr int LB_TILE = LB_BS * LB_IT;

__device__ __forceinline__ unsigned long long ld_relaxed_gpu(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_relaxed_gpu(unsigned long long *p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// LB_IT consecutive inputs of one thread: 16-byte vector loads when the
// tile is full and aligned (a warp then reads one contiguous span)
template <typename TI>
__device__ __forceinline__ void load_run(const TI *__restrict__ in, int64_t n, int64_t base, bool vec,
                                         int64_t (&v)[LB_IT]) {
    if (vec) {
        if constexpr (sizeof(TI) == 8) {
            const longlong2 *p = reinterpret_cast<const longlong2 *>(in + base);
#pragma unroll
            for (int k = 0; k < LB_IT / 2; k++) {
                const longlong2 q = __ldg(p + k);
                v[2 * k] = q.x;
                v[2 * k + 1] = q.y;
            }
        } else {
#pragma unroll
            for (int k = 0; k < LB_IT / 4; k++) {
                const int4 q = __ldg(reinterpret_cast<const int4 *>(in + base) + k);
                v[4 * k] = q.x;
                v[4 * k + 1] = q.y;
                v[4 * k + 2] = q.z;
                v[4 * k + 3] = q.w;
            }
        }
    } else {
#pragma unroll
        for (int k = 0; k < LB_IT; k++) v[k] = base + k < n ? (int64_t)in[base + k] : 0;
    }
}

__device__ __forceinline__ void store_run(int64_t *__restrict__ out, int64_t n, int64_t base, bool vec,
                                          int64_t run, const int64_t (&v)[LB_IT]) {
    if (vec) {
        longlong2 *p = reinterpret_cast<longlong2 *>(out + base);
#pragma unroll
        for (int k = 0; k < LB_IT / 2; k++) {
            const int64_t r0 = run;
            run += v[2 * k];
            p[k] = make_longlong2(r0, run);
            run += v[2 * k + 1];
        }
    } else {
#pragma unroll
        for (int k = 0; k < LB_IT; k++) {
            if (base + k < n) out[base + k] = run;
            run += v[k];
        }
    }
}

template <typename TI>
__global__ void __launch_bounds__(LB_BS) scan_lookback(const TI *__restrict__ in, int64_t n,
                                                      int64_t *__restrict__ out,
                                                      unsigned long long *state, unsigned epoch,
                                                      unsigned ntiles, unsigned long long *counter,
                                                      unsigned long long cbase) {
    pdl_wait();
    // tile = ticket from a monotone counter, not blockIdx: tiles are taken in
    // the order blocks actually start, so every predecessor a tile waits for
    // is already resident whatever the dispatch order (PDL early launch and
    // concurrent bins on other streams give no index-order guarantee)
    __shared__ int64_t ws[LB_BS / 32];
    __shared__ int64_t s_excl;
    __shared__ unsigned s_tile;
    if (threadIdx.x == 0) s_tile = (unsigned)(atomicAdd(counter, 1ull) - cbase);
    __syncthreads();
    const unsigned tile = s_tile;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t base = (int64_t)tile * LB_TILE + (int64_t)threadIdx.x * LB_IT;
    const bool vec = (int64_t)(tile + 1) * LB_TILE <= n &&
                     ((((uintptr_t)in) | ((uintptr_t)out)) & 15) == 0;   // block-uniform
    int64_t v[LB_IT];
    load_run<TI>(in, n, base, vec, v);
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < LB_IT; k++) s += v[k];
    int64_t x = s;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int64_t o = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += o;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    int64_t woff = 0, agg = 0;
#pragma unroll
    for (int j = 0; j < LB_BS / 32; j++) {
        woff += j < w ? ws[j] : 0;
        agg += ws[j];
    }
    if (w == 0) {
        if (tile == 0) {
            if (lane == 0) {
                st_relaxed_gpu(&state[0], lb_pack(agg, epoch, 2));
                s_excl = 0;
            }
        } else {
            if (lane == 0) st_relaxed_gpu(&state[tile], lb_pack(agg, epoch, 1));
            int64_t excl = 0;
            int64_t pred = (int64_t)tile - 1 - lane;
            for (;;) {
                const unsigned long long sv = pred >= 0 ? ld_relaxed_gpu(&state[pred]) : lb_pack(0, epoch, 2);
                const unsigned flag = lb_flag(sv, epoch);
                if (__any_sync(0xffffffffu, flag == 0)) continue;   // a predecessor not published yet
                const unsigned incl = __ballot_sync(0xffffffffu, flag == 2);
                int64_t val = lb_value(sv);
                if (incl) {
                    const int k = __ffs(incl) - 1;   // nearest inclusive prefix
                    if (lane > k) val = 0;
                }
#pragma unroll
                for (int d = 16; d >= 1; d >>= 1) val += __shfl_xor_sync(0xffffffffu, val, d);
                excl += val;
                if (incl) break;
                pred -= 32;
            }
            if (lane == 0) {
                st_relaxed_gpu(&state[tile], lb_pack(excl + agg, epoch, 2));
                s_excl = excl;
            }
        }
    }
    __syncthreads();
    store_run(out, n, base, vec, s_excl + woff + x - s, v);
    if (tile == ntiles - 1 && threadIdx.x == 0) out[n] = s_excl + agg;
}

// Inputs up to SMALL_SCAN elements: one block, one launch, no look-back state.
constexpr int64_t SMALL_SCAN = LB_TILE;

template <typename TI>
__global__ void __launch_bounds__(LB_BS) scan_one_block(const TI *__restrict__ in, int64_t n,
                                                        int64_t *__restrict__ out) {
    __shared__ int64_t ws[LB_BS / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t base = (int64_t)threadIdx.x * LB_IT;
    int64_t v[LB_IT];
    load_run<TI>(in, n, base, false, v);
    int64_t s = 0;
#pragma unroll
    for (int k = 0; k < LB_IT; k++) s += v[k];
    int64_t x = s;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int64_t o = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += o;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    int64_t woff = 0, agg = 0;
#pragma unroll
    for (int j = 0; j < LB_BS / 32; j++) {
        woff += j < w ? ws[j] : 0;
        agg += ws[j];
    }
    __syncthreads();   // in place: every thread has read its inputs
    store_run(out, n, base, false, woff + x - s, v);
    if (threadIdx.x == 0) out[n] = agg;
}

template <typename TI>
int scan_impl(tsg_ctx *c, const TI *in, int64_t *out, int64_t n) {
    if (n == 0) {
        TSG_TRY(tsg_fill(c, out, 0, sizeof(int64_t), c->stream));
        return TSG_OK;
    }
    if (n <= SMALL_SCAN) {
        scan_one_block<TI><<<1, LB_BS, 0, c->stream>>>(in, n, out); ++c->launches;
        TSG_CK(cudaGetLastError());
        return TSG_OK;
    }
    const int64_t tiles = (n + LB_TILE - 1) / LB_TILE;
    unsigned long long *state = nullptr;
    unsigned epoch = 0;
    unsigned long long *counter = nullptr, cbase = 0;
    if (c->capture_owned) {
        // a captured scan replays with the epoch and ticket base it was
        // captured with: give it its own state and counter, cleared by the
        // graph itself on every replay
        TSG_TRY(tsg_alloc_t(c, &state, tiles + 1));
        TSG_TRY(tsg_fill(c, state, 0, (size_t)(tiles + 1) * 8, c->stream));
        counter = state + tiles;
        epoch = 1;
    } else {
        TSG_TRY(tsg_lookback_state(c, tiles, &state, &epoch));
        TSG_TRY(tsg_lookback_counter(c, tiles, &counter, &cbase));
    }
    // in-place safe: a tile reads its inputs before writing, and writes only
    // its own range (plus out[n], past every input)
    TSG_CK(launch_pdl(scan_lookback<TI>, (unsigned)tiles, LB_BS, 0, c->stream, in, n, out, state, epoch,
                      (unsigned)tiles, counter, cbase));
    ++c->launches;
    TSG_CK(cudaGetLastError());
    return TSG_OK;
}
}  // namespace

int tsg_exclusive_scan_i64(tsg_ctx *c, const int64_t *in, int64_t *out, int64_t n) {
    return scan_impl<int64_t>(c, in, out, n);
}

int tsg_exclusive_scan_i32_to_i64(tsg_ctx *c, const int32_t *in, int64_t *out, int64_t n) {
    return scan_impl<int32_t>(c, in, out, n);
}

// ------------------------------------------------------------------ objects

int tsg_csr_alloc(tsg_ctx *c, int64_t rows, int64_t cols, int64_t nnz, bool values,
                  tsg_csr **out) {
    tsg_csr *m = new tsg_csr();
    m->max_row = -1;
    m->rows = rows;
    m->cols = cols;
    m->nnz = nnz;
    m->rp = nullptr;
    m->col = nullptr;
    m->val = nullptr;
    int s = tsg_alloc_t(c, &m->rp, rows + 1);
    if (s == TSG_OK) s = tsg_alloc_t(c, &m->col, nnz);
    if (s == TSG_OK && values) s = tsg_alloc_t(c, &m->val, nnz);
    if (s != TSG_OK) {
        tsg_free(c, m->rp);
        tsg_free(c, m->col);
        tsg_free(c, m->val);
        delete m;
        return s;
    }
    *out = m;
    return TSG_OK;
}

int tsg_vec_alloc(tsg_ctx *c, int64_t n, bool aux, tsg_vec **out) {
    tsg_vec *v = new tsg_vec();
    v->n = n;
    v->d = nullptr;
    v->aux = nullptr;
    v->sptr = nullptr;
    v->sset = nullptr;
    v->sbits = nullptr;
    int s = tsg_alloc_t(c, &v->d, n + 1);
    if (s == TSG_OK && aux) s = tsg_alloc_t(c, &v->aux, n + 1);
    if (s != TSG_OK) {
        tsg_free(c, v->d);
        delete v;
        return s;
    }
    *out = v;
    return TSG_OK;
}

int tsg_cmat_alloc(tsg_ctx *c, int64_t rows, int64_t cap, tsg_cmat **out) {
    tsg_cmat *m = new tsg_cmat();
    m->rows = rows;
    m->sorted_sets = 0;
    m->identity_rows = 0;
    m->cols = 0;
    m->dmax_valid = 0;
    m->cap = cap;
    m->start = nullptr;
    m->cnt = nullptr;
    m->set = nullptr;
    m->bits = nullptr;
    int s = tsg_alloc_t(c, &m->start, rows + 1);
    if (s == TSG_OK) s = tsg_alloc_t(c, &m->cnt, rows + 2);   // [rows + 1]: max count
    if (s == TSG_OK) s = tsg_alloc_t(c, &m->set, cap);
    if (s == TSG_OK) s = tsg_alloc_t(c, &m->bits, cap);
    if (s != TSG_OK) {
        tsg_free(c, m->start);
        tsg_free(c, m->cnt);
        tsg_free(c, m->set);
        delete m;
        return s;
    }
    *out = m;
    return TSG_OK;
}

// ------------------------------------------------------------------ CSR I/O

namespace {
__global__ void cols_i64_to_i32(const int64_t *__restrict__ in, int32_t *__restrict__ out,
                                int64_t n, int64_t ncols, int *err) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int64_t v = in[i];
        if (v < 0 || v >= ncols) {
            kerr(err, KERR_COLRANGE, i);
            v = 0;
        }
        out[i] = (int32_t)v;
    }
}

__global__ void cols_i32_to_i64(const int32_t *__restrict__ in, int64_t *__restrict__ out,
                                int64_t n, int64_t add) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int64_t)in[i] + add;
}

__global__ void rebase_rp(const int64_t *__restrict__ in, int64_t *__restrict__ out, int64_t n) {
    int64_t base = in[0];
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = in[i] - base;
}
}  // namespace

namespace {
// flag <- 1 if some row has a column smaller than its predecessor
__global__ void k_rows_unsorted(int64_t rows, const int64_t *__restrict__ rp,
                                const int32_t *__restrict__ col, int *flag,
                                unsigned long long *maxlen) {
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long ml = 0;
    bool bad = false;
    bool dup = false;
    for (int64_t i = w; i < rows; i += nw) {
        const int64_t r0 = rp[i], r1 = rp[i + 1];
        if ((unsigned long long)(r1 - r0) > ml) ml = (unsigned long long)(r1 - r0);
        for (int64_t t = r0 + 1 + lane; t < r1; t += 32) {
            bad |= col[t] < col[t - 1];
            dup |= col[t] == col[t - 1];
        }
    }
    // bit 0: some row decreases; bit 1: a column repeats next to itself
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(flag, 1);
    if (__any_sync(0xffffffffu, dup) && lane == 0) atomicOr(flag, 2);
    if (lane == 0 && ml) atomicMax(maxlen, ml);
}
}  // namespace

int tsg_csr_check_sorted(tsg_ctx *c, tsg_csr *m) {
    int *flag = reinterpret_cast<int *>(c->d_small + 52);
    unsigned long long *ml = reinterpret_cast<unsigned long long *>(c->d_small + 53);
    TSG_TRY(tsg_fill(c, c->d_small + 52, 0, 2 * sizeof(int64_t), c->stream));
    if (m->nnz > 0 && m->rows > 0) {
        k_rows_unsorted<<<grid_for(m->rows, 8, c->num_sms * 16), 256, 0, c->stream>>>(
            m->rows, m->rp, m->col, flag, ml); ++c->launches;
    }
    int64_t h[2] = {0, 0};
    TSG_CK(cudaMemcpyAsync(h, c->d_small + 52, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    TSG_CK(cudaStreamSynchronize(c->stream));
    m->sorted = ((int)h[0] & 1) ? 0 : 1;
    // distinct is only certain for sorted rows (an unsorted row could repeat a
    // column non-adjacently)
    m->distinct = m->sorted && !((int)h[0] & 2);
    m->max_row = h[1];
    return TSG_OK;
}

static unsigned ew_grid(tsg_ctx *c, int64_t n) { return grid_for(n, 256, c->num_sms * 16); }

extern "C" int tsg_csr_upload(tsg_ctx *c, int64_t rows, int64_t cols, int64_t nnz,
                              const int64_t *row_ptr, const int64_t *col_idx,
                              const double *values, tsg_csr **out) {
    if (rows < 0 || cols < 0 || nnz < 0) {
        tsg_set_error("negative dimensions");
        return TSG_EVALID;
    }
    if (cols > 0x7fffffffLL) {
        tsg_set_error("%lld columns exceed the device int32 column index", (long long)cols);
        return TSG_EDIM;
    }
    tsg_csr *m = nullptr;
    TSG_TRY(tsg_csr_alloc(c, rows, cols, nnz, values != nullptr, &m));
    TSG_TRY(tsg_copy(m->rp, row_ptr, (rows + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    if (nnz > 0) {
        int64_t *stage = nullptr;
        TSG_TRY(tsg_alloc_t(c, &stage, nnz));
        TSG_TRY(tsg_copy(stage, col_idx, nnz * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
        cols_i64_to_i32<<<ew_grid(c, nnz), 256, 0, c->stream>>>(stage, m->col, nnz, cols, c->d_err); ++c->launches;
        if (values)
            TSG_TRY(tsg_copy(m->val, values, nnz * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        TSG_TRY(tsg_free(c, stage));
    }
    int s = tsg_check_kernel_errors(c, "upload");
    if (s == TSG_OK) s = tsg_csr_check_sorted(c, m);
    if (s != TSG_OK) {
        tsg_csr_free(c, m);
        return s;
    }
    *out = m;
    return TSG_OK;
}

int tsg_csr_resolve(tsg_ctx *c, tsg_csr *m) {
    if (!m || !m->lazy_nnz) return TSG_OK;
    tsg_ctx *o = m->owner ? m->owner : c;
    TSG_TRY(tsg_put_small(o, m->rp + m->rows, 1, 20));
    TSG_CK(cudaStreamSynchronize(o->stream));
    m->nnz = o->h_small[20];
    m->lazy_nnz = 0;
    if (o->pending) return tsg_check_kernel_errors(o, o->pending);   // the producer's errors
    return TSG_OK;
}

extern "C" int tsg_csr_dims(const tsg_csr *m, int64_t *rows, int64_t *cols, int *has_values) {
    if (rows) *rows = m->rows;
    if (cols) *cols = m->cols;
    if (has_values) *has_values = m->val != nullptr;
    return TSG_OK;
}

extern "C" int tsg_csr_info(const tsg_csr *m, int64_t *rows, int64_t *cols, int64_t *nnz,
                            int *has_values) {
    if (nnz && m->lazy_nnz) TSG_TRY(tsg_csr_resolve(m->owner, const_cast<tsg_csr *>(m)));
    if (rows) *rows = m->rows;
    if (cols) *cols = m->cols;
    if (nnz) *nnz = m->nnz;
    if (has_values) *has_values = m->val != nullptr;
    return TSG_OK;
}

extern "C" int tsg_csr_download(tsg_ctx *c, const tsg_csr *m, int64_t *row_ptr,
                                int64_t *col_idx, double *values) {
    TSG_RESOLVE(c, m);
    if (m->host_mapped) {   // already in host memory: widen on the host
        TSG_CK(cudaStreamSynchronize(c->stream));
        if (c->pending) TSG_TRY(tsg_check_kernel_errors(c, c->pending));
        if (row_ptr) memcpy(row_ptr, m->rp, (m->rows + 1) * sizeof(int64_t));
        if (col_idx)
            for (int64_t i = 0; i < m->nnz; ++i) col_idx[i] = m->col[i];
        if (values && m->val) memcpy(values, m->val, m->nnz * sizeof(double));
        return TSG_OK;
    }
    if (row_ptr)
        TSG_TRY(tsg_copy(row_ptr, m->rp, (m->rows + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    if (m->nnz > 0 && col_idx) {
        int64_t *stage = nullptr;
        TSG_TRY(tsg_alloc_t(c, &stage, m->nnz));
        cols_i32_to_i64<<<ew_grid(c, m->nnz), 256, 0, c->stream>>>(m->col, stage, m->nnz, 0); ++c->launches;
        TSG_TRY(tsg_copy(col_idx, stage, m->nnz * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
        TSG_TRY(tsg_free(c, stage));
    }
    if (m->nnz > 0 && values && m->val)
        TSG_TRY(tsg_copy(values, m->val, m->nnz * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    TSG_CK(cudaStreamSynchronize(c->stream));
    if (c->pending) return tsg_check_kernel_errors(c, c->pending);   // the producer's errors
    return TSG_OK;
}

extern "C" int tsg_csr_slice_rows(tsg_ctx *c, const tsg_csr *m, int64_t begin, int64_t end,
                                  tsg_csr **out) {
    TSG_RESOLVE(c, m);
    if (!(0 <= begin && begin <= end && end <= m->rows)) {
        tsg_set_error("row slice [%lld, %lld) out of range", (long long)begin, (long long)end);
        return TSG_EDIM;
    }
    int64_t lo = 0, hi = 0;
    TSG_CK(cudaMemcpyAsync(&lo, m->rp + begin, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    TSG_CK(cudaMemcpyAsync(&hi, m->rp + end, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    TSG_CK(cudaStreamSynchronize(c->stream));
    tsg_csr *s = nullptr;
    TSG_TRY(tsg_csr_alloc(c, end - begin, m->cols, hi - lo, m->val != nullptr, &s));
    rebase_rp<<<ew_grid(c, end - begin + 1), 256, 0, c->stream>>>(m->rp + begin, s->rp,
                                                                  end - begin + 1); ++c->launches;
    if (hi > lo) {
        TSG_CK(cudaMemcpyAsync(s->col, m->col + lo, (hi - lo) * sizeof(int32_t),
                               cudaMemcpyDeviceToDevice, c->stream));
        if (m->val)
            TSG_CK(cudaMemcpyAsync(s->val, m->val + lo, (hi - lo) * sizeof(double),
                                   cudaMemcpyDeviceToDevice, c->stream));
    }
    TSG_CK(cudaGetLastError());
    s->sorted = m->sorted;
    s->distinct = m->distinct;
    s->max_row = m->max_row;
    *out = s;
    return TSG_OK;
}

// ---- placement: operands in pinned, device-mapped host memory -------------

int tsg_csr_alloc_mapped(tsg_ctx *c, int64_t rows, int64_t cols, int64_t nnz, bool values,
                         tsg_csr **out) {
    (void)c;
    tsg_csr *m = new tsg_csr();
    m->rows = rows;
    m->cols = cols;
    m->nnz = nnz;
    m->host_mapped = 1;
    m->max_row = -1;
    const unsigned fl = cudaHostAllocMapped | cudaHostAllocPortable;
    cudaError_t e = cudaHostAlloc((void **)&m->rp, (rows + 1) * sizeof(int64_t), fl);
    if (e == cudaSuccess) e = cudaHostAlloc((void **)&m->col, (nnz > 0 ? nnz : 1) * sizeof(int32_t), fl);
    if (e == cudaSuccess && values) e = cudaHostAlloc((void **)&m->val, (nnz > 0 ? nnz : 1) * sizeof(double), fl);
    if (e != cudaSuccess) {
        cudaGetLastError();
        cudaFreeHost(m->rp);
        cudaFreeHost(m->col);
        cudaFreeHost(m->val);
        delete m;
        tsg_set_error("pinned mapped host allocation failed: %s", cudaGetErrorString(e));
        return TSG_ECAPACITY;
    }
    *out = m;
    return TSG_OK;
}

extern "C" int tsg_csr_map_host(tsg_ctx *c, int64_t rows, int64_t cols, int64_t nnz,
                                const int64_t *row_ptr, const int64_t *col_idx,
                                const double *values, tsg_csr **out) {
    if (cols > 0x7fffffffLL) {
        tsg_set_error("%lld columns exceed the device int32 column index", (long long)cols);
        return TSG_EDIM;
    }
    tsg_csr *m = nullptr;
    TSG_TRY(tsg_csr_alloc_mapped(c, rows, cols, nnz, values != nullptr, &m));
    memcpy(m->rp, row_ptr, (rows + 1) * sizeof(int64_t));
    for (int64_t i = 0; i < nnz; ++i) {
        int64_t v = col_idx[i];
        if (v < 0 || v >= cols) {
            tsg_csr_free(c, m);
            tsg_set_error("column index out of range at entry %lld", (long long)i);
            return TSG_EVALID;
        }
        m->col[i] = (int32_t)v;
    }
    if (values) memcpy(m->val, values, nnz * sizeof(double));
    // row order facts on the host copy (compress fast path, lane-split numeric)
    bool sorted = true, distinct = true;
    int64_t mx = 0;
    for (int64_t r = 0; r < rows; ++r) {
        const int64_t lo = row_ptr[r], hi = row_ptr[r + 1];
        mx = hi - lo > mx ? hi - lo : mx;
        for (int64_t t = lo + 1; t < hi; ++t) {
            sorted &= m->col[t] >= m->col[t - 1];
            distinct &= m->col[t] != m->col[t - 1];
        }
    }
    m->sorted = sorted ? 1 : 0;
    m->distinct = (sorted && distinct) ? 1 : 0;
    m->max_row = mx;
    *out = m;
    return TSG_OK;
}

extern "C" int tsg_csr_from_device(tsg_ctx *c, int64_t rows, int64_t cols, int64_t nnz,
                                   const int64_t *d_rp, const int32_t *d_col, const double *d_val,
                                   tsg_csr **out) {
    tsg_csr *m = nullptr;
    TSG_TRY(tsg_csr_alloc(c, rows, cols, nnz, d_val != nullptr, &m));
    TSG_CK(cudaMemcpyAsync(m->rp, d_rp, (rows + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice,
                           c->stream));
    if (nnz > 0) {
        TSG_CK(cudaMemcpyAsync(m->col, d_col, nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                               c->stream));
        if (d_val)
            TSG_CK(cudaMemcpyAsync(m->val, d_val, nnz * sizeof(double), cudaMemcpyDeviceToDevice,
                                   c->stream));
    }
    TSG_CK(cudaStreamSynchronize(c->stream));
    TSG_TRY(tsg_csr_check_sorted(c, m));
    *out = m;
    return TSG_OK;
}

extern "C" int tsg_csr_device_ptrs(const tsg_csr *m, int64_t **rp, int32_t **col, double **val) {
    if (rp) *rp = m->rp;
    if (col) *col = m->col;
    if (val) *val = m->val;
    return TSG_OK;
}

extern "C" int tsg_csr_free(tsg_ctx *c, tsg_csr *m) {
    if (!m) return TSG_OK;
    tsg_plans_forget(c, m);
    if (m->plan) {   // a captured plan's output: its arrays stay with the plan
        tsg_plan_release_slot(m->plan, m->plan_slot);
        delete m;
        return TSG_OK;
    }
    if (m->host_mapped) {
        cudaStreamSynchronize(c->stream);
        cudaFreeHost(m->rp);
        cudaFreeHost(m->col);
        cudaFreeHost(m->val);
        delete m;
        return TSG_OK;
    }
    if (!m->borrowed) {
        tsg_free(c, m->rp);
        if (!m->cv_borrowed) {
            tsg_free(c, m->col);
            tsg_free(c, m->val);
        }
    }
    delete m;
    return TSG_OK;
}

// ------------------------------------------------------------------ vectors

extern "C" int tsg_vec_upload(tsg_ctx *c, int64_t n, const int64_t *host, tsg_vec **out) {
    tsg_vec *v = nullptr;
    TSG_TRY(tsg_vec_alloc(c, n, false, &v));
    if (n > 0)
        TSG_TRY(tsg_copy(v->d, host, n * sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    *out = v;
    return TSG_OK;
}

extern "C" int tsg_vec_download(tsg_ctx *c, const tsg_vec *v, int64_t *host) {
    if (v->n > 0)
        TSG_CK(cudaMemcpyAsync(host, v->d, v->n * sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    TSG_CK(cudaStreamSynchronize(c->stream));
    return TSG_OK;
}

extern "C" int tsg_vec_len(const tsg_vec *v, int64_t *n) {
    *n = v->n;
    return TSG_OK;
}

extern "C" int tsg_vec_free(tsg_ctx *c, tsg_vec *v) {
    if (!v) return TSG_OK;
    tsg_free(c, v->d);
    tsg_free(c, v->aux);
    tsg_free(c, v->sptr);
    tsg_free(c, v->sset);
    tsg_free(c, v->sbits);
    delete v;
    return TSG_OK;
}
