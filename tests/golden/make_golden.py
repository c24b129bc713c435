"""Generate the golden fixtures that pin the oracle (and through it the GPU path)
to the reference implementation itself.

Run in a container where /root/reference exists:
    python tests/golden/make_golden.py
It imports the UNMODIFIED reference package from /root/reference/pkg/src,
runs its hot-path functions on small seeded inputs, and stores inputs and
outputs in tests/golden/golden.npz (+ golden.json for scalar / planner
results).  /root/reference does not exist on the GPU box; the fixtures do.
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import tiered_spgemm as ts  # noqa: E402
from tiered_spgemm.chunking import (balanced_partition,  # noqa: E402
                                    c_row_byte_sizes)
from tiered_spgemm.generators import _scalar_stencil_entries  # noqa: E402

arrays = {}
meta = {}


def put_csr(name, m):
    arrays[name + "/rp"] = np.asarray(m.row_ptr, np.int64)
    arrays[name + "/ci"] = np.asarray(m.col_idx, np.int64)
    if m.values is not None:
        arrays[name + "/va"] = np.asarray(m.values, np.float64)
    meta[name] = [int(m.num_rows), int(m.num_cols), m.values is not None]


def put_cm(name, cm):
    arrays[name + "/rp"] = np.asarray(cm.row_ptr, np.int64)
    arrays[name + "/set"] = np.asarray(cm.set_idx, np.int64)
    arrays[name + "/bits"] = np.asarray(cm.set_bits, np.uint64)
    meta[name] = [int(cm.num_rows)]


def random_csr(rng, rows, cols, delta, values=True, shuffle=True):
    r, c, v = [], [], []
    for i in range(rows):
        k = min(int(rng.integers(0, delta + 1)), cols)
        for col in rng.choice(cols, size=k, replace=False):
            r.append(i)
            c.append(int(col))
            v.append(float(rng.uniform(0.1, 1.0)))
    m = ts.CsrMatrix.from_coo(r, c, v if values else None, rows, cols)
    if not shuffle:
        return m
    # keep the reference's "columns never assumed sorted" contract exercised
    ci, va = m.col_idx.copy(), None if m.values is None else m.values.copy()
    for i in range(rows):
        lo, hi = int(m.row_ptr[i]), int(m.row_ptr[i + 1])
        p = rng.permutation(hi - lo)
        ci[lo:hi] = ci[lo:hi][p]
        if va is not None:
            va[lo:hi] = va[lo:hi][p]
    return ts.CsrMatrix(rows, cols, m.row_ptr, ci, va)


def main():
    rng = np.random.default_rng(1804)

    # --- compress / symbolic / numeric on random pairs (first-touch order) ----
    meta["pairs"] = 0
    for k in range(12):
        n = int(rng.integers(8, 90))
        m_ = int(rng.integers(8, 300))
        a = random_csr(rng, n, m_, 10)
        b = random_csr(rng, m_, int(rng.integers(8, 700)), 14, shuffle=bool(k % 2))
        cb = ts.compress(b)
        counts = ts.spgemm_symbolic(a, cb)
        c = ts.spgemm_numeric(a, b, counts)
        put_csr("pair%d/a" % k, a)
        put_csr("pair%d/b" % k, b)
        put_cm("pair%d/cb" % k, cb)
        arrays["pair%d/counts" % k] = counts
        put_csr("pair%d/c" % k, c)
        meta["pairs"] += 1

    # --- fused chunk sequences ----------------------------------------------
    meta["fused"] = 0
    for k in range(4):
        a = random_csr(rng, 60, 80, 9)
        b = random_csr(rng, 80, 150, 9)
        a_lo, a_hi = 10, 50
        part = ts.CsrMatrix.empty(a_hi - a_lo, 150)
        cuts = [0, 23, 51, 80]
        put_csr("fused%d/a" % k, a)
        put_csr("fused%d/b" % k, b)
        for j in range(3):
            lo, hi = cuts[j], cuts[j + 1]
            part = ts.spgemm_numeric_fused(a, ts.slice_rows(b, lo, hi), part,
                                           ts.RowRange(a_lo, a_hi), ts.RowRange(lo, hi))
            put_csr("fused%d/step%d" % (k, j), part)
        meta["fused%d" % k] = {"a_rows": [a_lo, a_hi], "cuts": cuts}
        meta["fused"] += 1

    # --- triangle counts ------------------------------------------------------
    tri = []
    for k in range(8):
        nv = int(rng.integers(20, 120))
        up = np.triu(rng.random((nv, nv)) < float(rng.uniform(0.05, 0.25)), 1)
        rows, cols = np.nonzero(up | up.T)
        g = ts.CsrMatrix.from_coo(rows, cols, None, nv, nv)
        l = ts.lower_triangle(g, ts.degree_sort_permutation(g))
        put_csr("tri%d/l" % k, l)
        put_cm("tri%d/cl" % k, ts.compress(l))
        tri.append(ts.masked_row_intersect_count(l, ts.compress(l)))
        put_csr("tri%d/g" % k, g)
    meta["triangles"] = [int(x) for x in tri]
    meta["triangles_total"] = [int(ts.count_triangles(
        ts.CsrMatrix(meta["tri%d/g" % k][0], meta["tri%d/g" % k][1], arrays["tri%d/g/rp" % k],
                     arrays["tri%d/g/ci" % k], None))) for k in range(8)]

    # --- stencil generators and config-shaped products -------------------------
    for kind, dims in ((ts.LAPLACE3D, (6, 5, 7)), (ts.BRICK3D, (6, 7, 5)),
                       (ts.BIGSTAR2D, (9, 7)), (ts.ELASTICITY3D, (5, 5, 6))):
        put_csr("stencil/%s" % kind, ts.generate_stencil(ts.StencilSpec(kind, dims)))
        meta["stencil/%s/dims" % kind] = list(dims)
    l2 = [((0, 0), 4.0), ((-1, 0), -1.0), ((1, 0), -1.0), ((0, -1), -1.0), ((0, 1), -1.0)]
    r_, c_, v_ = _scalar_stencil_entries((32, 32), l2)
    lap2 = ts.CsrMatrix.from_coo(r_, c_, v_, 1024, 1024)
    put_csr("stencil/laplace2d", lap2)
    meta["stencil/laplace2d/dims"] = [32, 32]
    c1 = ts.multiply(lap2, lap2)
    put_csr("config1_32/c", c1)

    brick = ts.generate_stencil(ts.StencilSpec(ts.BRICK3D, (8, 8, 8)))
    # plain 2x2x2 aggregation on 8^3 -> 4^3 (what config 2 uses at 128^3)
    idx = np.arange(512)
    x, y, z = idx % 8, (idx // 8) % 8, idx // 64
    agg = (x // 2) + 4 * (y // 2) + 16 * (z // 2)
    p = ts.CsrMatrix(512, 64, np.arange(513), agg, np.ones(512))
    r = ts.transpose(p)
    ra = ts.multiply(r, brick)
    rap = ts.multiply(ra, p)
    put_csr("config2_8/a", brick)
    put_csr("config2_8/p", p)
    put_csr("config2_8/ra", ra)
    put_csr("config2_8/rap", rap)

    # --- SplitMix64 ------------------------------------------------------------
    g = ts.PortableRng(0)
    meta["splitmix_seed0"] = [g.next_u64() for _ in range(3)]
    g = ts.PortableRng(22)
    meta["splitmix_seed22_below"] = [g.below(1000) for _ in range(5)]

    # --- planner / partitioner (host logic of the chunked path) ---------------
    plans = []
    prng = np.random.default_rng(7)
    for _ in range(40):
        nr = int(prng.integers(5, 40))
        ra_ = prng.integers(8, 400, size=nr).astype(np.int64)
        rb_ = prng.integers(8, 400, size=int(prng.integers(5, 40))).astype(np.int64)
        rc_ = prng.integers(8, 600, size=nr).astype(np.int64)
        fast = int(prng.integers(int(max(ra_.max() + rc_.max(), rb_.max())) * 2 + 10, 20000))
        try:
            plan = ts.decide_chunking(int(ra_.sum()), int(rb_.sum()), int(rc_.sum()),
                                      ra_, rb_, rc_, fast)
            out = plan.to_json_dict()
        except ts.TieredSpgemmError as e:
            out = {"error": type(e).__name__}
        plans.append({"a": ra_.tolist(), "b": rb_.tolist(), "c": rc_.tolist(), "fast": fast,
                      "plan": out})
    meta["plans"] = plans
    parts = []
    for _ in range(60):
        n = int(prng.integers(1, 50))
        rb_ = prng.integers(1, 300, size=n).astype(np.int64)
        target = int(prng.integers(1, 900))
        cap = int(prng.integers(1, 1000))
        try:
            out = ts.binary_search_partition(rb_, target, cap).to_json_dict()
        except ts.TieredSpgemmError as e:
            out = {"error": type(e).__name__}
        parts.append({"rows": rb_.tolist(), "target": target, "cap": cap, "out": out})
        try:
            bal = balanced_partition(rb_, max(1, int(rb_.sum()) // 3 + 1)).to_json_dict()
        except ts.TieredSpgemmError as e:
            bal = {"error": type(e).__name__}
        parts[-1]["balanced"] = bal
    meta["partitions"] = parts
    meta["c_row_bytes"] = c_row_byte_sizes(4, [1, 0, 3, 2]).tolist()

    # --- chunked executors: ledgers (billing) on a fixed product -------------
    a = random_csr(rng, 50, 60, 6, shuffle=False)
    b = random_csr(rng, 60, 40, 6, shuffle=False)
    counts = ts.spgemm_symbolic(a, ts.compress(b))
    model = ts.MemoryModel(ts.MemorySpaceSpec("fast", 1 << 40, 100e9, 1e-7),
                           ts.MemorySpaceSpec("slow", None, 10e9, 1e-6))
    put_csr("chunk/a", a)
    put_csr("chunk/b", b)
    acr = a.row_byte_sizes() + c_row_byte_sizes(a.num_rows, counts)
    p_ac = ts.binary_search_partition(acr, int(acr.sum() // 3) + 1)
    p_b = ts.binary_search_partition(b.row_byte_sizes(), int(b.byte_size // 2) + 1)
    ledgers = {}
    for name, fn in (("gpu1", ts.gpu_chunk_multiply_1), ("gpu2", ts.gpu_chunk_multiply_2)):
        c, led = fn(a, b, counts, p_ac, p_b, model)
        ledgers[name] = [[e.bytes, e.src, e.dst, e.tag] for e in led.events]
        put_csr("chunk/%s_c" % name, c)
    c, led = ts.knl_chunk_multiply(a, b, counts, b.byte_size // 3 + 1, model)
    ledgers["knl"] = [[e.bytes, e.src, e.dst, e.tag] for e in led.events]
    put_csr("chunk/knl_c", c)
    meta["chunk"] = {"p_ac": p_ac.to_json_dict(), "p_b": p_b.to_json_dict(),
                     "knl_fast": int(b.byte_size // 3 + 1), "ledgers": ledgers}

    # --- products_match tolerance KAT (csr.py:165-184) ------------------------
    base = ts.CsrMatrix(1, 2, [0, 2], [0, 1], [1.0, 2.0])
    meta["match_kat"] = [ts.products_match(ts.CsrMatrix(1, 2, [0, 2], [0, 1], [1.0 + 1e-13, 2.0]),
                                           base)[0],
                         ts.products_match(ts.CsrMatrix(1, 2, [0, 2], [0, 1], [1.0 + 1e-9, 2.0]),
                                           base)[0]]

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote %d arrays, %d meta keys" % (len(arrays), len(meta)))


if __name__ == "__main__":
    main()
