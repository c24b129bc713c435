// tsg_partition.cuh -- row partition by tier ("bin"), shared by the symbolic,
// numeric, fused and masked-count phases.
//
// Three launches and one host wait per partition:
//   k_part_bins     the phase's bin functor per row (it may also write
//                   per-row side outputs), warp-aggregated tile histogram
//   scan            exclusive scan of the NB x ntiles tile counts
//   k_part_scatter  row ids into per-bin lists (tile order kept, order inside
//                   a tile not), block 0 also gathers the bin starts and one
//                   optional extra device value (e.g. nnz(C)) into mapped
//                   host memory as soon as it starts, then a sequence word;
//                   the host polls that word instead of synchronising the
//                   stream, so the next launches overlap the scatter
// Rows are ranked with __match_any_sync peers so a block does one shared
// atomic per distinct bin per warp, not one per row (a single dominant bin
// otherwise serialises 1024 atomics on one address).
#pragma once
#include "tsg_internal.cuh"

#ifndef TSG_PART_TILE
#define TSG_PART_TILE 1024
#endif
constexpr int PART_TILE = TSG_PART_TILE;   // rows per tile = one 256-thread block

template <int NB>
struct BinLists {
    int32_t *list = nullptr;
    int64_t off[NB + 1] = {0};
    // device-driven mode (tsg_partition with nowait): the bin starts live
    // only in device memory (dstart[0 .. NB]); off[] holds no counts and
    // `rows` bounds every bin
    int64_t *dstart = nullptr;
    bool device = false;
    int64_t rows = 0;
    uint32_t possible = 0xffffffffu;   // device mode: bins the host's bounds allow
    int64_t hint[NB + 1] = {0};        // device mode: bin starts of the last same-shape call
};

// tile counts up to this many are scanned by the last k_part_bins block
constexpr int PART_FUSED_SCAN = 16384;

template <int NB, class F>
__global__ void __launch_bounds__(256) k_part_bins(int64_t rows, F f, uint8_t *__restrict__ bins,
                                                   int ntiles, int *__restrict__ tc,
                                                   unsigned *__restrict__ done, int64_t *__restrict__ offs) {
    pdl_wait();
    __shared__ int h[NB];
    if (threadIdx.x < NB) h[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t base = (int64_t)blockIdx.x * PART_TILE;
#pragma unroll
    for (int k = threadIdx.x; k < PART_TILE; k += 256) {
        const int64_t i = base + k;
        int b = 255;
        if (i < rows) {
            b = f(i);
            bins[i] = (uint8_t)b;
        }
        const unsigned peers = __match_any_sync(0xffffffffu, b);
        if (b < NB && lane == __ffs(peers) - 1) atomicAdd(&h[b], __popc(peers));
    }
    __syncthreads();
    if (threadIdx.x < NB) tc[(int64_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
    if (!done) return;
    // the last block to finish scans the NB x ntiles tile counts (no
    // separate scan launch); the counter is left at 0 for the next partition
    __shared__ bool s_last;
    __shared__ int64_t s_warp[8];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(done, 1u) == (unsigned)ntiles - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const int n = NB * ntiles;
    if (threadIdx.x == 0) *done = 0;
    // each thread owns `per` consecutive tile counts: all its loads are in
    // flight together, one block scan of the per-thread sums, then the
    // thread writes its offsets (the chunk-serial form paid one L2 round
    // trip and three barriers per 256 counts: ~15 us at 262 K rows)
    const int per = (n + 255) / 256;
    const int q0 = threadIdx.x * per;
    int64_t loc = 0;
#pragma unroll 8
    for (int j = 0; j < per; ++j) {
        const int q = q0 + j;
        loc += q < n ? (int64_t)__ldcg(tc + q) : 0;
    }
    int64_t x = loc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const int64_t o = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += o;
    }
    const int w = threadIdx.x >> 5;
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    int64_t run = x - loc, agg = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        run += k < w ? s_warp[k] : 0;
        agg += s_warp[k];
    }
#pragma unroll 8
    for (int j = 0; j < per; ++j) {
        const int q = q0 + j;
        if (q < n) {
            offs[q] = run;
            run += (int64_t)__ldcg(tc + q);
        }
    }
    if (threadIdx.x == 0) offs[n] = agg;
}

template <int NB>
__global__ void __launch_bounds__(256) k_part_scatter(int64_t rows, const uint8_t *__restrict__ bins,
                                                      int ntiles, const int64_t *__restrict__ offs,
                                                      int32_t *__restrict__ list,
                                                      const int64_t *__restrict__ extra,
                                                      const int *__restrict__ err,
                                                      int64_t *__restrict__ out, int64_t seq,
                                                      int64_t *__restrict__ dstart) {
    pdl_wait();
    __shared__ int h[NB];
    if (threadIdx.x < NB) h[threadIdx.x] = 0;
    if (dstart && blockIdx.x == 0 && threadIdx.x <= NB) dstart[threadIdx.x] = offs[(int64_t)threadIdx.x * ntiles];
    if (out && blockIdx.x == 0) {   // `out` is the mapped host scratch (h_small[32 ..])
        if (threadIdx.x <= NB) out[threadIdx.x] = offs[(int64_t)threadIdx.x * ntiles];
        if (threadIdx.x == NB + 1) out[NB + 1] = extra ? *extra : 0;
        // pending kernel errors of earlier work ride along (h_small[62])
        if (threadIdx.x == NB + 2) out[30] = *reinterpret_cast<const int64_t *>(err);
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence_system();
            *reinterpret_cast<volatile int64_t *>(out + 29) = seq;   // h_small[61]
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t base = (int64_t)blockIdx.x * PART_TILE;
#pragma unroll
    for (int k = threadIdx.x; k < PART_TILE; k += 256) {
        const int64_t i = base + k;
        const int b = i < rows ? bins[i] : 255;
        const unsigned peers = __match_any_sync(0xffffffffu, b);
        const int leader = __ffs(peers) - 1;
        int r0 = 0;
        if (b < NB && lane == leader) r0 = atomicAdd(&h[b], __popc(peers));
        r0 = __shfl_sync(0xffffffffu, r0, leader);
        if (b < NB) list[offs[(int64_t)b * ntiles + blockIdx.x] + r0 + __popc(peers & lt)] = (int32_t)i;
    }
}

// Partition rows [0, rows) by f(i) (values >= NB: row skipped).  `bins` is
// caller scratch of `rows` bytes; `out.list` is allocated here (caller frees).
// Bin starts and *extra come back in c->h_small[32 ..].  `mid()` is enqueued
// between the bin and scatter kernels (e.g. a scan of a side output of f whose
// total is `extra`).
struct NoMid {
    int operator()() const { return TSG_OK; }
};

template <int NB, class F, class Mid = NoMid>
int tsg_partition(tsg_ctx *c, int64_t rows, F f, uint8_t *bins, BinLists<NB> &out,
                  const int64_t *extra = nullptr, int64_t *extra_out = nullptr, Mid mid = Mid(),
                  bool nowait = false, int64_t *hint_host = nullptr, int64_t *hint_dev = nullptr) {
    static_assert(32 + NB + 2 <= 61, "partition results overlap the sequence / error slots");
    int ntiles = (int)((rows + PART_TILE - 1) / PART_TILE);
    if (ntiles < 1) ntiles = 1;
    int *tc = nullptr;
    int64_t *offs = nullptr;
    TSG_TRY(tsg_alloc_t(c, &tc, (size_t)NB * ntiles));
    TSG_TRY(tsg_alloc_t(c, &offs, (size_t)NB * ntiles + 1));
    TSG_TRY(tsg_alloc_t(c, &out.list, rows > 0 ? rows : 1));
    const bool fused_scan = (int64_t)NB * ntiles <= PART_FUSED_SCAN;
    unsigned *done = fused_scan ? reinterpret_cast<unsigned *>(c->d_small + 60) : nullptr;
    TSG_CK(launch_pdl(k_part_bins<NB, F>, ntiles, 256, 0, c->stream, rows, f, bins, ntiles, tc, done, offs));
    ++c->launches;
    if (!fused_scan) TSG_TRY(tsg_exclusive_scan_i32_to_i64(c, tc, offs, (int64_t)NB * ntiles));
    TSG_TRY(mid());
    // results land in mapped host memory straight from the kernel: no D2H
    // copy that would queue behind bulk transfers on the copy engine
    if (nowait) {
        // device-driven: the bin kernels read their ranges from dstart; the
        // host waits for nothing.  The starts also land in this shape's hint
        // buffer (read by the host at the next same-shape call, never now)
        TSG_TRY(tsg_alloc_t(c, &out.dstart, NB + 1));
        out.device = true;
        out.rows = rows;
        if (hint_host)
            for (int b = 0; b <= NB; b++) out.hint[b] = hint_host[b];
        TSG_CK(launch_pdl(k_part_scatter<NB>, ntiles, 256, 0, c->stream, rows, (const uint8_t *)bins, ntiles,
                          (const int64_t *)offs, out.list, extra, (const int *)c->d_err, hint_dev,
                          (int64_t)0, out.dstart));
        ++c->launches;
        TSG_CK(cudaGetLastError());
        TSG_TRY(tsg_free(c, tc));
        TSG_TRY(tsg_free(c, offs));
        for (int b = 0; b <= NB; b++) out.off[b] = -1;
        return TSG_OK;
    }
    TSG_CK(launch_pdl(k_part_scatter<NB>, ntiles, 256, 0, c->stream, rows, (const uint8_t *)bins, ntiles,
                      (const int64_t *)offs, out.list, extra, (const int *)c->d_err, c->hd_small + 32,
                      ++c->part_seq, (int64_t *)nullptr));
    ++c->launches;
    TSG_CK(cudaGetLastError());
    TSG_TRY(tsg_free(c, tc));
    TSG_TRY(tsg_free(c, offs));
    tsg_trace_host("partition: wait");
    TSG_TRY(tsg_wait_mapped(c, 61, c->part_seq));
    tsg_trace_host("partition: results");
    TSG_TRY(tsg_pending_errors(c));
    for (int b = 0; b <= NB; b++) out.off[b] = c->h_small[32 + b];
    if (extra_out) *extra_out = c->h_small[32 + NB + 1];
    if (hint_host)
        for (int b = 0; b <= NB; b++) hint_host[b] = out.off[b];
    return TSG_OK;
}
