"""Secondary benchmark lines for BASELINE.json configs 1, 3 and 4 (the
driver's line is config 2, bench.py).  Same JSON keys; each line is measured
on the device with CUDA events on libtsg's stream (configs 1, 3) or by the
chunked executor's own stream-ordered accounting (config 4)."""

import json
import os
import statistics
import time

import numpy as np

UNIT = "GFLOP/s"


def _peaks():
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def config1(args):
    """A*A, 2D 5-point Laplacian 256^2 (65,536 rows), in HBM."""
    from paper_1804_00695_b200 import _lib, generators as gen, kernel
    from oracle import oracle as O
    ctx = _lib.Context.get(0)
    ctx.set_timing(True)
    a = gen.stencil(gen.LAPLACE2D, (256, 256))
    da = _lib.DeviceCsr.upload(a, ctx)
    for _ in range(args.warmup):
        kernel.multiply_device(da, da)
    times = []
    for _ in range(args.steps):
        ctx.record(0)
        dc = kernel.multiply_device(da, da)
        ctx.record(1)
        times.append(ctx.elapsed_ms(0, 1))
    mults = O.count_multiplications(a, a)
    ms = statistics.median(times)
    t0 = time.perf_counter()
    O.multiply(a, a, workers=os.cpu_count() or 1)
    cpu = time.perf_counter() - t0
    return {"metric": "SpGEMM GFLOP/s config 1 (A*A laplace2d 256^2)", "value": 2 * mults / ms / 1e6,
            "unit": UNIT, "ms_per_step": ms, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config1 A*A 2D 5-pt 256^2", "multiplications": mults,
                       "nnz_c": dc.nnz, "launch_bound": "C is 14 MB; one multiply is ~20 launches"},
            "cpu_baseline": {"value": 2 * mults / cpu / 1e9, "unit": UNIT, "cores": os.cpu_count(),
                             "kind": "port", "sample": "full A*A"}}


def config3(args):
    """Triangle counting, R-MAT/Graph500 scale S (default 22), int64 exact.

    The whole pipeline runs in HBM: R-MAT build,
    validation + degree order + lower triangle, then per step compress(L) +
    masked count.  The host oracle re-counts the downloaded L."""
    from paper_1804_00695_b200 import _lib, generators as gen
    from paper_1804_00695_b200.triangles import lower_triangle_device
    from oracle import oracle as O
    ctx = _lib.Context.get(0)
    ctx.set_timing(True)
    gen.rmat_graph_device(10)                       # warm the CUB kernels
    ctx.sync()
    ctx.record(2)
    dg = gen.rmat_graph_device(args.scale)
    ctx.record(3)
    dl, _ = lower_triangle_device(dg, check=True)
    ctx.record(4)
    ctx.sync()
    gen_ms, prep_ms = ctx.elapsed_ms(2, 3), ctx.elapsed_ms(3, 4)
    n, g_nnz = dg.num_rows, dg.nnz
    del dg
    for _ in range(args.warmup):
        tri = _lib.d_masked_count(dl, _lib.d_compress(dl))
    times = []
    for _ in range(args.steps):
        ctx.record(0)
        dcl2 = _lib.d_compress(dl)          # compress + masked count per step
        tri = _lib.d_masked_count(dl, dcl2)
        ctx.record(1)
        times.append(ctx.elapsed_ms(0, 1))
    ms = statistics.median(times)
    low = dl.download()
    mults = O.count_multiplications(low, low)
    line = {"metric": "triangle counting GFLOP/s config 3 (2 x mults(L,L) / time)",
            "value": 2 * mults / ms / 1e6, "unit": UNIT, "ms_per_step": ms, "dtype": "int64",
            "data": "synthetic", "triangles": tri,
            "config": {"workload": "config3 R-MAT scale %d ef16 (.57,.19,.19,.05) SplitMix64 seed 22"
                       % args.scale, "n": n, "nnz_graph": g_nnz, "nnz_L": low.nnz, "mults_LL": mults,
                       "device_rmat_build_ms": gen_ms, "device_lower_triangle_ms": prep_ms,
                       "pipeline_ms": gen_ms + prep_ms + ms}}
    if not args.no_cpu_baseline:
        t0 = time.perf_counter()
        want = O.masked_count(low, O.compress(low), workers=os.cpu_count() or 1)
        cpu = time.perf_counter() - t0
        line.update({"oracle_triangles": want, "exact": tri == want,
                     "cpu_baseline": {"value": 2 * mults / cpu / 1e9, "unit": UNIT,
                                      "cores": os.cpu_count(), "kind": "port",
                                      "sample": "full masked count on the host"}})
    return line


def config4(args):
    """Chunked out-of-HBM A*A, brick3d N^3 (default 256^3), HBM budget capped
    (default 8 GiB), A and C in pinned host memory, the Alg. 4 plan."""
    import paper_1804_00695_b200 as tsg
    from paper_1804_00695_b200 import _lib, chunking as ch, generators as gen
    from paper_1804_00695_b200.csr import CsrMatrix, slice_rows
    from paper_1804_00695_b200.memory import b200_model
    from oracle import oracle as O
    n = args.grid
    t0 = time.perf_counter()
    a0 = gen.stencil(gen.BRICK3D, (n, n, n))

    def pin(x, dt):
        y = _lib.pinned_empty(len(x), dt)
        y[:] = x
        return y
    a = CsrMatrix._adopt(a0.num_rows, a0.num_cols, pin(a0.row_ptr, np.int64),
                         pin(a0.col_idx, np.int64), pin(a0.values, np.float64))
    del a0
    gen_s = time.perf_counter() - t0
    # symbolic counts once on the device (the reference computes them unchunked
    # and unbilled, cli.py:164-165); not part of the timed chunked run
    ctx = _lib.Context.get(0)
    da = _lib.DeviceCsr.upload(a, ctx)
    counts = _lib.d_symbolic(da, _lib.d_compress(da)).download()
    del da
    fast = int(args.hbm_cap_gib * 2**30)
    plan = ch.plan_for_multiply(a, a, counts, fast)
    model = b200_model(fast)
    c, led = ch.execute_plan(a, a, counts, plan, model)
    ph = led.physical
    mults = int(np.diff(a.row_ptr)[a.col_idx].sum())
    # correctness: sampled rows against the oracle (rows are independent)
    rs = np.random.default_rng(0).choice(a.num_rows, size=64, replace=False)
    ok = True
    for r in rs[:16]:
        sub = slice_rows(a, int(r), int(r) + 1)
        ptr, col, val = O.multiply(sub, a)
        lo, hi = int(c.row_ptr[r]), int(c.row_ptr[r + 1])
        order = np.argsort(col)
        ok &= bool(np.array_equal(c.col_idx[lo:hi], col[order]) and
                   np.array_equal(c.values[lo:hi], val[order]))
    # CPU rate on a row sample (extrapolated)
    sample = slice_rows(a, 0, 65536)
    t1 = time.perf_counter()
    O.multiply(sample, a, workers=os.cpu_count() or 1)
    cpu = time.perf_counter() - t1
    smults = int(np.diff(a.row_ptr)[sample.col_idx].sum())
    secs = ph["wall_ms"] / 1e3
    return {"metric": "chunked SpGEMM GFLOP/s config 4 (A*A brick3d %d^3, HBM cap %.1f GiB)"
                      % (n, args.hbm_cap_gib),
            "value": 2 * mults / secs / 1e9, "unit": UNIT, "dtype": "f64", "data": "synthetic",
            "host_link": {"achieved_gbs": ph["link_gbs"], "h2d_bytes": ph["h2d_bytes"],
                          "d2h_bytes": ph["d2h_bytes"], "wall_s": secs,
                          "kernel_s": ph["kernel_ms"] / 1e3},
            "plan": {"algorithm": plan.algorithm, "branch": plan.heuristic_branch,
                     "n_ac": len(plan.partition_ac), "n_b": len(plan.partition_b),
                     "ledger_bytes": led.total_bytes(),
                     "predicted_copy_bytes": plan.predicted_copy_bytes},
            "config": {"workload": "config4", "rows": a.num_rows, "nnz_A": a.nnz, "nnz_C": c.nnz,
                       "multiplications": mults, "generation_s": gen_s},
            "sampled_rows_exact": ok,
            "cpu_baseline": {"value": 2 * smults / cpu / 1e9, "unit": UNIT,
                             "cores": os.cpu_count(), "kind": "port",
                             "sample": "first 65536 rows of A times A (extrapolated rate)"}}


def placement(args):
    """The paper's data-placement table (Laplace R x A:
    HBM / A_Pin / B_Pin / C_Pin / HostPin) on B200: config 2's R*A with each
    operand either in HBM or in pinned, device-mapped host memory that the
    kernels read/write in place over PCIe."""
    import paper_1804_00695_b200 as tsg
    from paper_1804_00695_b200 import _lib, generators as gen
    from paper_1804_00695_b200.memory import PlacementPolicy
    n = args.grid if args.grid != 256 else 128
    a = gen.stencil(gen.BRICK3D, (n, n, n))
    _, r = gen.aggregation((n, n, n))
    mults = a.nnz   # R has one entry per column of A
    out = {}
    for name, spaces in (("HBM", "fff"), ("A_Pin", "sff"), ("B_Pin", "fsf"), ("C_Pin", "ffs"),
                         ("HostPin", "sss")):
        pol = PlacementPolicy(name, {k: ("fast" if v == "f" else "slow") for k, v in zip("ABC", spaces)})
        tsg.multiply(r, a, placement=pol)          # warm-up (and operand placement)
        times = []
        for _ in range(max(1, args.steps)):
            t0 = time.perf_counter()
            tsg.multiply(r, a, placement=pol)
            times.append(time.perf_counter() - t0)
        out[name] = 2 * mults / statistics.median(times) / 1e9
    return {"metric": "R*A GFLOP/s by operand placement (paper Table, PAPER.md:819)",
            "unit": UNIT, "values": out, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "brick3d %d^3 R*A (2x2x2 aggregation), host wall time per call "
                                   "incl. placement of slow operands and download of C" % n}}


def config5(args):
    """A*A on an R-MAT graph (values 1.0), single GPU, all tiers (power-law
    rows land in the CTA and global-memory tiers).  The graph is built in HBM
    (generators.rmat_graph_device, equal to the host builder).  Correctness:
    sampled rows (incl. the max-degree row) against the oracle -- C's rows are
    sliced on the device, so a multi-billion-entry C never crosses PCIe."""
    from paper_1804_00695_b200 import _lib, generators as gen, kernel
    from paper_1804_00695_b200.csr import slice_rows
    from oracle import oracle as O
    ctx = _lib.Context.get(0)
    ctx.set_timing(True)
    ctx.record(2)
    da = gen.rmat_graph_device(args.scale).set_values(1.0)
    ctx.record(3)
    ctx.sync()
    build_ms = ctx.elapsed_ms(2, 3)
    mults = _lib.d_count_multiplications(da, da)
    for _ in range(args.warmup):
        dc = kernel.multiply_device(da, da)
        del dc
    times = []
    for _ in range(args.steps):
        ctx.record(0)
        dc = kernel.multiply_device(da, da)
        ctx.record(1)
        times.append(ctx.elapsed_ms(0, 1))
        nnz_c = dc.nnz
        if _ + 1 < args.steps:
            del dc
    ms = statistics.median(times)
    a = da.download()                       # host copy of A for the oracle
    deg = np.diff(a.row_ptr)
    rng = np.random.default_rng(1)
    rows = list(rng.choice(a.num_rows, size=24, replace=False)) + [int(np.argmax(deg))]
    ok = True
    for r in rows:
        ptr, col, val = O.multiply(slice_rows(a, int(r), int(r) + 1), a)
        o = np.argsort(col)
        got = dc.slice_rows(int(r), int(r) + 1).download()
        ok &= bool(np.array_equal(got.col_idx, col[o]) and np.array_equal(got.values, val[o]))
    sample = slice_rows(a, 0, min(a.num_rows, 4096))
    t1 = time.perf_counter()
    O.multiply(sample, a, workers=os.cpu_count() or 1)
    cpu = time.perf_counter() - t1
    smults = int(deg[sample.col_idx].sum())
    return {"metric": "SpGEMM GFLOP/s config 5 (A*A R-MAT scale %d, 1 GPU)" % args.scale,
            "value": 2 * mults / ms / 1e6, "unit": UNIT, "ms_per_step": ms, "dtype": "f64",
            "data": "synthetic", "sampled_rows_exact": ok,
            "config": {"n": a.num_rows, "nnz_A": a.nnz, "nnz_C": nnz_c, "multiplications": mults,
                       "max_degree": int(deg.max()), "device_build_ms": build_ms,
                       "c_bytes_device": 8 * (a.num_rows + 1) + 12 * nnz_c},
            "cpu_baseline": {"value": 2 * smults / cpu / 1e9, "unit": UNIT, "cores": os.cpu_count(),
                             "kind": "port", "sample": "first 4096 rows of A times A"}}


def run(args):
    return {1: config1, 3: config3, 4: config4, 5: config5, 6: placement}[args.config](args)
