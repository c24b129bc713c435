/*
 * tsg_oracle.c -- CPU restatement of the reference SpGEMM hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port" arm of bench.py).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path (paper_1804_00695_b200/) never links or calls it.
 *
 * Every function restates the reference algorithm step for step so that its
 * outputs are bit-identical to the Python reference, including the
 * accumulator's first-touch column order and the fp64 summation order:
 *
 *   accumulator      /root/reference/pkg/src/tiered_spgemm/accumulator.py:17-27, 95-141
 *                    (multiplicative hash 0x9E3779B97F4A7C15 masked to cap-1,
 *                     linear probing, capacity = next pow2 >= 2*bound,
 *                     extraction in insertion order)
 *   compress         kernel.py:73-93   (dict per row -> first-touch set order)
 *   count_mults      kernel.py:96-103
 *   row blocks       kernel.py:106-121 (workers = contiguous row blocks)
 *   spgemm_symbolic  kernel.py:124-168
 *   spgemm_numeric   kernel.py:171-232
 *   numeric_fused    kernel.py:235-340
 *   masked count     kernel.py:349-394
 *
 * Parity of this restatement is pinned against golden vectors produced by the
 * reference itself (tests/golden/make_golden.py) in tests/test_oracle.py.
 *
 * Status codes (mirrors include/tsg.h): 0 ok, 1 dimension, 2 validation,
 * 3 kernel (count mismatch / overflow).  On error *err_row gets the row.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>

#define HASH_MULT 0x9E3779B97F4A7C15ULL
#define EMPTY_KEY (-1LL)

typedef struct {
    int64_t *keys;
    uint64_t *ubits;   /* symbolic payload (or_bits) */
    double *vals;      /* numeric payload (add)      */
    int64_t *used;     /* insertion-ordered slot list */
    int64_t slots;     /* slab size                   */
    int64_t cap, mask, n_used;
} acc_t;

static int64_t acc_capacity(int64_t bound) {
    /* accumulator.py:24-27 */
    int64_t need = 2 * bound;
    if (need < 1) need = 1;
    int64_t c = 1;
    while (c < need) c <<= 1;
    return c;
}

static int acc_init_slab(acc_t *a, int64_t slots) {
    a->slots = slots;
    a->keys = (int64_t *)malloc(sizeof(int64_t) * slots);
    a->ubits = (uint64_t *)malloc(sizeof(uint64_t) * slots);
    a->vals = (double *)malloc(sizeof(double) * slots);
    a->used = (int64_t *)malloc(sizeof(int64_t) * slots);
    if (!a->keys || !a->ubits || !a->vals || !a->used) return -1;
    for (int64_t i = 0; i < slots; i++) a->keys[i] = EMPTY_KEY;
    a->n_used = 0;
    return 0;
}

static void acc_free_slab(acc_t *a) {
    free(a->keys); free(a->ubits); free(a->vals); free(a->used);
}

static inline void acc_begin(acc_t *a, int64_t cap) {
    a->cap = cap;
    a->mask = cap - 1;
    a->n_used = 0;
}

static inline int64_t acc_slot(const acc_t *a, int64_t key) {
    return (int64_t)(((uint64_t)key * HASH_MULT) & (uint64_t)a->mask);
}

/* accumulator.py:95-110 -- insert-or-add */
static inline void acc_add(acc_t *a, int64_t key, double v) {
    int64_t idx = acc_slot(a, key);
    for (;;) {
        int64_t k = a->keys[idx];
        if (k == key) { a->vals[idx] += v; return; }
        if (k == EMPTY_KEY) {
            a->keys[idx] = key;
            a->vals[idx] = v;
            a->used[a->n_used++] = idx;
            return;
        }
        idx = (idx + 1) & a->mask;
    }
}

/* accumulator.py:112-127 -- insert-or-OR */
static inline void acc_or(acc_t *a, int64_t key, uint64_t bits) {
    int64_t idx = acc_slot(a, key);
    for (;;) {
        int64_t k = a->keys[idx];
        if (k == key) { a->ubits[idx] |= bits; return; }
        if (k == EMPTY_KEY) {
            a->keys[idx] = key;
            a->ubits[idx] = bits;
            a->used[a->n_used++] = idx;
            return;
        }
        idx = (idx + 1) & a->mask;
    }
}

static inline void acc_reset(acc_t *a) {
    for (int64_t t = 0; t < a->n_used; t++) a->keys[a->used[t]] = EMPTY_KEY;
    a->n_used = 0;
}

/* ---------------------------------------------------------------- workers */

typedef void (*block_fn)(void *ctx, int64_t lo, int64_t hi, int block_id);

typedef struct {
    block_fn fn;
    void *ctx;
    int64_t lo, hi;
    int id;
} job_t;

static void *job_main(void *p) {
    job_t *j = (job_t *)p;
    j->fn(j->ctx, j->lo, j->hi, j->id);
    return NULL;
}

/* kernel.py:106-121: contiguous row blocks, bounds = linspace(0, n, w+1). */
static int row_blocks(int64_t n, int workers, int64_t *lo, int64_t *hi) {
    int w = workers;
    if (n == 0) w = 1;
    else {
        if (w > n) w = (int)n;
        if (w < 1) w = 1;
    }
    int nb = 0;
    for (int i = 0; i < w; i++) {
        /* np.linspace(0, n, w+1, dtype=int64) truncates i*n/w */
        int64_t a = (int64_t)((double)n * i / w);
        int64_t b = (int64_t)((double)n * (i + 1) / w);
        if (a < b) { lo[nb] = a; hi[nb] = b; nb++; }
    }
    return nb;
}

static void run_blocks(int64_t n, int workers, block_fn fn, void *ctx) {
    if (workers < 1) workers = 1;
    int64_t *lo = (int64_t *)malloc(sizeof(int64_t) * (workers + 1));
    int64_t *hi = (int64_t *)malloc(sizeof(int64_t) * (workers + 1));
    int nb = row_blocks(n, workers, lo, hi);
    if (nb <= 1 || workers <= 1) {
        for (int b = 0; b < nb; b++) fn(ctx, lo[b], hi[b], b);
    } else {
        pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * nb);
        job_t *jobs = (job_t *)malloc(sizeof(job_t) * nb);
        for (int b = 0; b < nb; b++) {
            jobs[b].fn = fn; jobs[b].ctx = ctx;
            jobs[b].lo = lo[b]; jobs[b].hi = hi[b]; jobs[b].id = b;
            pthread_create(&th[b], NULL, job_main, &jobs[b]);
        }
        for (int b = 0; b < nb; b++) pthread_join(th[b], NULL);
        free(th); free(jobs);
    }
    free(lo); free(hi);
}

/* --------------------------------------------------------------- compress */

/* kernel.py:73-93.  out_set/out_bits must hold nnz entries; out_rp rows+1. */
int oc_compress(int64_t rows, const int64_t *rp, const int64_t *col,
                int64_t *out_rp, int64_t *out_set, uint64_t *out_bits,
                int64_t *out_nsets) {
    int64_t maxlen = 1;
    for (int64_t i = 0; i < rows; i++) {
        int64_t l = rp[i + 1] - rp[i];
        if (l > maxlen) maxlen = l;
    }
    acc_t a;
    if (acc_init_slab(&a, acc_capacity(maxlen)) != 0) return 3;
    int64_t pos = 0;
    out_rp[0] = 0;
    for (int64_t i = 0; i < rows; i++) {
        acc_begin(&a, acc_capacity(rp[i + 1] - rp[i]));
        for (int64_t t = rp[i]; t < rp[i + 1]; t++) {
            int64_t c = col[t];
            acc_or(&a, c >> 6, 1ULL << (c & 63));
        }
        /* dict keys in insertion order == accumulator first-touch order */
        for (int64_t u = 0; u < a.n_used; u++) {
            int64_t s = a.used[u];
            out_set[pos] = a.keys[s];
            out_bits[pos] = a.ubits[s];
            pos++;
        }
        acc_reset(&a);
        out_rp[i + 1] = pos;
    }
    *out_nsets = pos;
    acc_free_slab(&a);
    return 0;
}

/* kernel.py:96-103 */
int64_t oc_count_multiplications(int64_t nnz_a, const int64_t *ca,
                                 const int64_t *rp_b) {
    int64_t total = 0;
    for (int64_t t = 0; t < nnz_a; t++) {
        int64_t k = ca[t];
        total += rp_b[k + 1] - rp_b[k];
    }
    return total;
}

/* --------------------------------------------------------------- symbolic */

typedef struct {
    const int64_t *rp_a, *ca, *crp, *cset;
    const uint64_t *cbits;
    const int64_t *bounds;
    int64_t max_bound;
    int64_t *counts;
} sym_ctx;

static void sym_block(void *p, int64_t lo, int64_t hi, int id) {
    (void)id;
    sym_ctx *c = (sym_ctx *)p;
    acc_t a;
    acc_init_slab(&a, acc_capacity(c->max_bound));
    for (int64_t i = lo; i < hi; i++) {
        if (c->bounds[i] == 0) continue;
        acc_begin(&a, acc_capacity(c->bounds[i]));
        for (int64_t t = c->rp_a[i]; t < c->rp_a[i + 1]; t++) {
            int64_t k = c->ca[t];
            for (int64_t s = c->crp[k]; s < c->crp[k + 1]; s++)
                acc_or(&a, c->cset[s], c->cbits[s]);
        }
        int64_t tot = 0;
        for (int64_t u = 0; u < a.n_used; u++)
            tot += __builtin_popcountll(a.ubits[a.used[u]]);
        c->counts[i] = tot;
        acc_reset(&a);
    }
    acc_free_slab(&a);
}

/* kernel.py:124-168 */
int oc_symbolic(int64_t rows_a, const int64_t *rp_a, const int64_t *ca,
                const int64_t *crp, const int64_t *cset, const uint64_t *cbits,
                int64_t *counts, int workers) {
    int64_t *bounds = (int64_t *)calloc(rows_a ? rows_a : 1, sizeof(int64_t));
    int64_t max_bound = 1;
    for (int64_t i = 0; i < rows_a; i++) {
        int64_t b = 0;
        for (int64_t t = rp_a[i]; t < rp_a[i + 1]; t++) {
            int64_t k = ca[t];
            b += crp[k + 1] - crp[k];
        }
        bounds[i] = b;
        if (b > max_bound) max_bound = b;
        counts[i] = 0;
    }
    sym_ctx c = {rp_a, ca, crp, cset, cbits, bounds, max_bound, counts};
    run_blocks(rows_a, workers, sym_block, &c);
    free(bounds);
    return 0;
}

/* ---------------------------------------------------------------- numeric */

typedef struct {
    const int64_t *rp_a, *ca, *rp_b, *cb;
    const double *va, *vb;
    const int64_t *counts, *c_ptr;
    int64_t *c_col;
    double *c_val;
    int64_t max_count;
    volatile int status;
    volatile int64_t err_row;
    pthread_mutex_t mu;
} num_ctx;

static void num_fail(num_ctx *c, int code, int64_t row) {
    pthread_mutex_lock(&c->mu);
    if (c->status == 0 || row < c->err_row) { c->status = code; c->err_row = row; }
    pthread_mutex_unlock(&c->mu);
}

static void num_block(void *p, int64_t lo, int64_t hi, int id) {
    (void)id;
    num_ctx *c = (num_ctx *)p;
    acc_t a;
    acc_init_slab(&a, acc_capacity(c->max_count));
    for (int64_t i = lo; i < hi; i++) {
        int64_t want = c->counts[i];
        if (want == 0) continue;
        acc_begin(&a, acc_capacity(want));
        int bad = 0;
        for (int64_t t = c->rp_a[i]; t < c->rp_a[i + 1] && !bad; t++) {
            int64_t k = c->ca[t];
            double av = c->va[t];
            for (int64_t s = c->rp_b[k]; s < c->rp_b[k + 1]; s++) {
                /* the reference table has no probe bound; a count too small
                   could fill it, so stop before it is full (kernel.py:213) */
                if (a.n_used >= a.cap) { bad = 1; break; }
                acc_add(&a, c->cb[s], av * c->vb[s]);
            }
            if (a.n_used > want) bad = 1;
        }
        if (bad || a.n_used != want) {
            num_fail(c, 3, i);
            acc_reset(&a);
            break;
        }
        int64_t pos = c->c_ptr[i];
        for (int64_t u = 0; u < a.n_used; u++) {
            int64_t s = a.used[u];
            c->c_col[pos] = a.keys[s];
            c->c_val[pos] = a.vals[s];
            pos++;
        }
        acc_reset(&a);
    }
    acc_free_slab(&a);
}

/* kernel.py:171-232.  c_ptr (rows+1) is filled here; c_col/c_val hold
   sum(counts) entries.  Returns 3 (KernelError) with *err_row on mismatch. */
int oc_numeric(int64_t rows_a, const int64_t *rp_a, const int64_t *ca,
               const double *va, const int64_t *rp_b, const int64_t *cb,
               const double *vb, const int64_t *counts, int64_t *c_ptr,
               int64_t *c_col, double *c_val, int workers, int64_t *err_row) {
    int64_t maxc = 1;
    c_ptr[0] = 0;
    for (int64_t i = 0; i < rows_a; i++) {
        c_ptr[i + 1] = c_ptr[i] + counts[i];
        if (counts[i] > maxc) maxc = counts[i];
    }
    num_ctx c;
    memset(&c, 0, sizeof(c));
    c.rp_a = rp_a; c.ca = ca; c.va = va; c.rp_b = rp_b; c.cb = cb; c.vb = vb;
    c.counts = counts; c.c_ptr = c_ptr; c.c_col = c_col; c.c_val = c_val;
    c.max_count = maxc;
    c.status = 0; c.err_row = -1;
    pthread_mutex_init(&c.mu, NULL);
    run_blocks(rows_a, workers, num_block, &c);
    pthread_mutex_destroy(&c.mu);
    if (err_row) *err_row = c.err_row;
    return c.status;
}

/* ------------------------------------------------------------------ fused */

/* kernel.py:276-290: per-output-row bounds; returns the sum of bounds so the
   caller can size scratch (rows are written at bound offsets). */
int64_t oc_fused_bounds(int64_t n_out, int64_t a_lo, const int64_t *rp_a,
                        const int64_t *ca, int64_t b_lo, int64_t b_hi,
                        const int64_t *rp_bc, const int64_t *rp_c,
                        int64_t *bounds) {
    int64_t total = 0;
    for (int64_t li = 0; li < n_out; li++) {
        int64_t gi = a_lo + li;
        int64_t bd = rp_c[li + 1] - rp_c[li];
        for (int64_t t = rp_a[gi]; t < rp_a[gi + 1]; t++) {
            int64_t k = ca[t];
            if (b_lo <= k && k < b_hi) {
                int64_t l = k - b_lo;
                bd += rp_bc[l + 1] - rp_bc[l];
            }
        }
        bounds[li] = bd;
        total += bd;
    }
    return total;
}

typedef struct {
    int64_t a_lo, b_lo, b_hi;
    const int64_t *rp_a, *ca, *rp_bc, *cbc, *rp_c, *cc;
    const double *va, *vbc, *vc;
    const int64_t *bounds, *scratch_ptr;
    int64_t max_bound;
    int64_t *row_len, *s_col;
    double *s_val;
} fus_ctx;

static void fus_block(void *p, int64_t lo, int64_t hi, int id) {
    (void)id;
    fus_ctx *c = (fus_ctx *)p;
    acc_t a;
    acc_init_slab(&a, acc_capacity(c->max_bound));
    for (int64_t li = lo; li < hi; li++) {
        if (c->bounds[li] == 0) { c->row_len[li] = 0; continue; }
        acc_begin(&a, acc_capacity(c->bounds[li]));
        for (int64_t t = c->rp_c[li]; t < c->rp_c[li + 1]; t++)
            acc_add(&a, c->cc[t], c->vc[t]);
        int64_t gi = c->a_lo + li;
        for (int64_t t = c->rp_a[gi]; t < c->rp_a[gi + 1]; t++) {
            int64_t k = c->ca[t];
            if (!(c->b_lo <= k && k < c->b_hi)) continue;
            double av = c->va[t];
            int64_t l = k - c->b_lo;
            for (int64_t s = c->rp_bc[l]; s < c->rp_bc[l + 1]; s++)
                acc_add(&a, c->cbc[s], av * c->vbc[s]);
        }
        int64_t pos = c->scratch_ptr[li];
        for (int64_t u = 0; u < a.n_used; u++) {
            int64_t s = a.used[u];
            c->s_col[pos] = a.keys[s];
            c->s_val[pos] = a.vals[s];
            pos++;
        }
        c->row_len[li] = a.n_used;
        acc_reset(&a);
    }
    acc_free_slab(&a);
}

/* kernel.py:235-340 minus the argument checks (done by the Python wrapper).
   Rows are written into scratch at exclusive-prefix(bounds) offsets and
   their lengths into row_len; the wrapper compacts. */
int oc_fused(int64_t n_out, int64_t a_lo, const int64_t *rp_a,
             const int64_t *ca, const double *va, int64_t b_lo, int64_t b_hi,
             const int64_t *rp_bc, const int64_t *cbc, const double *vbc,
             const int64_t *rp_c, const int64_t *cc, const double *vc,
             const int64_t *bounds, const int64_t *scratch_ptr,
             int64_t *row_len, int64_t *s_col, double *s_val, int workers) {
    int64_t mb = 1;
    for (int64_t i = 0; i < n_out; i++)
        if (bounds[i] > mb) mb = bounds[i];
    fus_ctx c = {a_lo, b_lo, b_hi, rp_a, ca, rp_bc, cbc, rp_c, cc,
                 va, vbc, vc, bounds, scratch_ptr, mb, row_len, s_col, s_val};
    run_blocks(n_out, workers, fus_block, &c);
    return 0;
}

/* ----------------------------------------------------------- masked count */

typedef struct {
    const int64_t *rp, *cols, *crp, *cset;
    const uint64_t *cbits;
    int64_t max_len;
    int64_t *partial;
    volatile int status;
    volatile int64_t err_row;
    pthread_mutex_t mu;
} msk_ctx;

static void msk_block(void *p, int64_t lo, int64_t hi, int id) {
    msk_ctx *c = (msk_ctx *)p;
    acc_t a;
    acc_init_slab(&a, acc_capacity(c->max_len));
    int64_t total = 0;
    for (int64_t i = lo; i < hi; i++) {
        int64_t r0 = c->rp[i], r1 = c->rp[i + 1];
        if (r0 == r1) continue;
        acc_begin(&a, acc_capacity(r1 - r0));
        int bad = 0;
        for (int64_t t = r0; t < r1; t++) {
            int64_t col = c->cols[t];
            if (col >= i) { bad = 1; break; }
            acc_or(&a, col >> 6, 1ULL << (col & 63));
        }
        if (bad) {
            pthread_mutex_lock(&c->mu);
            if (c->status == 0 || i < c->err_row) { c->status = 2; c->err_row = i; }
            pthread_mutex_unlock(&c->mu);
            acc_reset(&a);
            break;
        }
        for (int64_t t = r0; t < r1; t++) {
            int64_t j = c->cols[t];
            for (int64_t s = c->crp[j]; s < c->crp[j + 1]; s++) {
                /* dict.get(cset) lookup without insertion */
                int64_t key = c->cset[s];
                int64_t idx = acc_slot(&a, key);
                for (;;) {
                    int64_t k = a.keys[idx];
                    if (k == key) {
                        total += __builtin_popcountll(c->cbits[s] & a.ubits[idx]);
                        break;
                    }
                    if (k == EMPTY_KEY) break;
                    idx = (idx + 1) & a.mask;
                }
            }
        }
        acc_reset(&a);
    }
    c->partial[id] = total;
    acc_free_slab(&a);
}

/* kernel.py:349-394 */
int oc_masked_count(int64_t rows, const int64_t *rp, const int64_t *cols,
                    const int64_t *crp, const int64_t *cset,
                    const uint64_t *cbits, int workers, int64_t *total,
                    int64_t *err_row) {
    int64_t ml = 1;
    for (int64_t i = 0; i < rows; i++)
        if (rp[i + 1] - rp[i] > ml) ml = rp[i + 1] - rp[i];
    int w = workers < 1 ? 1 : workers;
    msk_ctx c;
    memset(&c, 0, sizeof(c));
    c.rp = rp; c.cols = cols; c.crp = crp; c.cset = cset; c.cbits = cbits;
    c.max_len = ml;
    c.partial = (int64_t *)calloc((size_t)w + 1, sizeof(int64_t));
    c.status = 0; c.err_row = -1;
    pthread_mutex_init(&c.mu, NULL);
    run_blocks(rows, w, msk_block, &c);
    pthread_mutex_destroy(&c.mu);
    int64_t t = 0;
    for (int b = 0; b <= w; b++) t += c.partial[b];
    free(c.partial);
    *total = t;
    if (err_row) *err_row = c.err_row;
    return c.status;
}
