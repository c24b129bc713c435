"""Secondary benchmark lines for BASELINE.json configs 1, 3, 4 and 5 (the
driver's line is config 2, bench.py), each with its own parity check.

Every line carries ``parity`` ({"ok": ...}); ``secondary()`` runs configs 1,
3 and 4 inside the default bench.py run so they are driver-observed.  Device
times are CUDA events on libtsg's compute stream (configs 1, 3, 5) or the
chunked executor's own stream-ordered accounting (config 4).

The oracle (oracle/, the reference's algorithm restated in C and pinned to
the reference's outputs) is used here only as the checker and as the CPU
baseline, never on the measured path.
"""

import argparse
import json
import os
import statistics
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
UNIT = "GFLOP/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


# ------------------------------------------------------------------ parity helpers

def _row_ids(ptr):
    ptr = np.asarray(ptr, dtype=np.int64)
    return np.repeat(np.arange(ptr.shape[0] - 1, dtype=np.int64), np.diff(ptr))


def _canon(ptr, col, val, ncols):
    """Per-row ascending columns (the reference's canonicalize, csr.py:145-150)."""
    col = np.asarray(col, dtype=np.int64)
    key = _row_ids(ptr) * max(int(ncols), 1) + col
    if key.shape[0] < 2 or bool(np.all(key[1:] > key[:-1])):
        return col, None if val is None else np.asarray(val)
    order = np.argsort(key, kind="stable")
    return col[order], None if val is None else np.asarray(val)[order]


def compare_products(got, want, rtol=1e-12):
    """got: CsrMatrix (ours); want: (ptr, col, val) from the oracle, any row
    order.  Structure must be bit-exact (row pointers, per-row sorted
    columns); values bit-exact (``exact``) or within the north star's
    rel 1e-12 / abs 1e-250 (csr.py:165-184 products_match)."""
    ptr, col, val = want
    out = {"nnz": int(got.nnz), "structure": False, "exact": False, "ok": False, "max_rel": None}
    if not np.array_equal(np.asarray(got.row_ptr), np.asarray(ptr, dtype=np.int64)):
        return out
    gc, gv = _canon(got.row_ptr, got.col_idx, got.values, got.num_cols)
    wc, wv = _canon(ptr, col, val, got.num_cols)
    if not np.array_equal(gc, wc):
        return out
    out["structure"] = True
    if gv is None and wv is None:
        out.update(exact=True, ok=True, max_rel=0.0)
        return out
    gv, wv = np.asarray(gv, dtype=np.float64), np.asarray(wv, dtype=np.float64)
    out["exact"] = bool(np.array_equal(gv.view(np.uint64), wv.view(np.uint64)))
    d = np.abs(gv - wv)
    mag = np.maximum(np.abs(gv), np.abs(wv))
    rel = np.where(mag > 0, d / np.where(mag > 0, mag, 1.0), 0.0)
    out["max_rel"] = float(rel.max()) if rel.size else 0.0
    out["ok"] = bool(np.all((d <= rtol * mag) | (d <= 1e-250)))
    return out


def embed_rows(a_loc, dims, rank, base):
    """A full-height matrix holding only rank's slab rows of the fine
    operator (N>1 config 2): the oracle's B operand for that rank."""
    from paper_1804_00695_b200.csr import CsrMatrix
    n = int(np.prod(dims))
    plane = base * base
    lo, hi = rank * base * plane, (rank + 1) * base * plane
    rp = np.zeros(n + 1, dtype=np.int64)
    rp[lo + 1:hi + 1] = a_loc.row_ptr[1:]
    rp[hi + 1:] = a_loc.nnz
    return CsrMatrix._adopt(n, a_loc.num_cols, rp, a_loc.col_idx, a_loc.values)


def link_peaks(gib=1.0, reps=3):
    """Pinned host <-> HBM copy bandwidth on this box (the roofline of the
    chunked executors): H2D alone, D2H alone, both directions at once (GB/s)."""
    import torch
    n = int(gib * 2**30)
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out[name + "_gbs"] = reps * n / (e0.elapsed_time(e1) * 1e-3) / 1e9
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s1):
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        for _ in range(reps):
            h2.copy_(d2, non_blocking=True)
    s1.synchronize()
    s2.synchronize()
    out["bidir_total_gbs"] = 2 * reps * n / (time.perf_counter() - t0) / 1e9
    del h, h2, d, d2
    torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------------ config 1

def config1(args):
    """A*A, 2D 5-point Laplacian 256^2 (65,536 rows), in HBM; full parity."""
    from oracle import oracle as O
    from paper_1804_00695_b200 import _lib, generators as gen, kernel
    ctx = _lib.Context.get(0)
    ctx.set_timing(True)
    a = gen.stencil(gen.LAPLACE2D, (256, 256))
    da = _lib.DeviceCsr.upload(a, ctx)
    for _ in range(max(3, args.warmup)):
        kernel.multiply_device(da, da)
    times = []
    l0 = ctx.stats()[0]
    for _ in range(args.steps):
        ctx.record(0)
        dc = kernel.multiply_device(da, da)
        ctx.record(1)
        times.append(ctx.elapsed_ms(0, 1))
    launches = (ctx.stats()[0] - l0) / max(args.steps, 1)
    mults = O.count_multiplications(a, a)
    ms = statistics.median(times)
    t0 = time.perf_counter()
    want = O.multiply(a, a, workers=os.cpu_count() or 1)
    cpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.multiply(a, a, workers=1)
    cpu1 = time.perf_counter() - t0
    par = compare_products(dc.download(), want)
    byts = 2 * (8 * (a.num_rows + 1) + 16 * a.nnz) + 8 * (a.num_rows + 1) + 16 * dc.nnz
    return {"metric": "SpGEMM GFLOP/s config 1 (A*A laplace2d 256^2)", "value": 2 * mults / ms / 1e6,
            "unit": UNIT, "ms_per_step": ms, "steps": args.steps, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config1 A*A 2D 5-pt 256^2", "multiplications": mults,
                       "nnz_c": dc.nnz, "launches_per_multiply": launches},
            "roofline": {"bound": "hbm", "algorithmic_bytes": byts,
                         "frac": byts / (ms * 1e-3) / 1e9 / _peaks(),
                         "note": "launch/latency-bound: 25.6 MB per multiply is ~4 us of HBM time"},
            "parity": par,
            "cpu_baseline": {"value": 2 * mults / cpu / 1e9, "unit": UNIT, "cores": os.cpu_count(),
                             "w1_value": 2 * mults / cpu1 / 1e9,
                             "kind": "port", "sample": "full A*A (oracle/tsg_oracle.c)"}}


# ------------------------------------------------------------------ config 3

def rmat_golden(scale):
    """Golden triangle count of the config-3 graph at `scale` (tests/golden/
    rmat_triangles.json, made by tests/golden/make_rmat_triangles.py)."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "rmat_triangles.json")) as fh:
            return json.load(fh).get(str(scale))
    except Exception:
        return None


def config3(args):
    """Triangle counting, R-MAT/Graph500 scale S (default 22), int64 exact.

    The whole pipeline runs in HBM: R-MAT build,
    validation + degree order + lower triangle, then per step compress(L) +
    masked count.  Parity: the golden count of the same graph (oracle, full
    graph, tests/golden/rmat_triangles.json) and nnz(L)."""
    from oracle import oracle as O
    from paper_1804_00695_b200 import _lib, generators as gen
    from paper_1804_00695_b200.triangles import lower_triangle_device
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
    for _ in range(max(3, args.warmup)):
        tri = _lib.d_masked_count(dl, _lib.d_compress(dl))
    times = []
    for _ in range(args.steps):
        ctx.record(0)
        dcl2 = _lib.d_compress(dl)          # compress + masked count per step
        tri = _lib.d_masked_count(dl, dcl2)
        ctx.record(1)
        times.append(ctx.elapsed_ms(0, 1))
    ms = statistics.median(times)
    mults = _lib.d_count_multiplications(dl, dl)
    gold = rmat_golden(args.scale)
    par = {"ok": None, "exact": None, "triangles": tri}
    if gold is not None:
        same = tri == gold["triangles"] and dl.nnz == gold["nnz_L"] and mults == gold["mults_LL"]
        par.update(ok=bool(same), exact=bool(same), golden_triangles=gold["triangles"],
                   source="tests/golden/rmat_triangles.json (oracle masked count of the full graph)")
    line = {"metric": "triangle counting GFLOP/s config 3 (2 x mults(L,L) / time)",
            "value": 2 * mults / ms / 1e6, "unit": UNIT, "ms_per_step": ms, "steps": args.steps,
            "dtype": "int64", "data": "synthetic", "triangles": tri,
            "config": {"workload": "config3 R-MAT scale %d ef16 (.57,.19,.19,.05) SplitMix64 seed 22"
                       % args.scale, "n": n, "nnz_graph": g_nnz, "nnz_L": dl.nnz, "mults_LL": mults,
                       "device_rmat_build_ms": gen_ms, "device_lower_triangle_ms": prep_ms,
                       "pipeline_ms": gen_ms + prep_ms + ms},
            "parity": par}
    if not args.no_cpu_baseline:
        # the oracle on the full graph of a smaller scale of the same family
        # (the scale-22 count is ~90 s of host time)
        cs = min(args.scale, 18)
        low = dl.download() if cs == args.scale else \
            lower_triangle_device(gen.rmat_graph_device(cs), check=False)[0].download()
        cm = int(np.diff(low.row_ptr)[low.col_idx].sum())
        t0 = time.perf_counter()
        O.masked_count(low, O.compress(low), workers=os.cpu_count() or 1)
        cpu = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": 2 * cm / cpu / 1e9, "unit": UNIT, "cores": os.cpu_count(),
                                "kind": "port",
                                "sample": "compress + masked count of the full R-MAT scale-%d graph "
                                          "(same generator) with the oracle" % cs}
    return line


# ------------------------------------------------------------------ config 4

def config4(args):
    """Chunked out-of-HBM A*A, brick3d N^3 (default 256^3), HBM budget capped
    (default 8 GiB, plus every cap in ``args.extra_caps_gib``), A and C in
    pinned host memory, the Alg. 4 plan.  A is built on the device and
    downloaded into pinned memory (the host builder takes ~25 s); the symbolic
    counts are computed inside the same budget (chunking.symbolic_within_budget);
    parity on sampled rows, incl. the first / last row of every planned range."""
    from oracle import oracle as O
    from paper_1804_00695_b200 import _lib, chunking as ch, generators as gen
    from paper_1804_00695_b200.csr import CsrMatrix, slice_rows
    from paper_1804_00695_b200.memory import b200_model
    n = args.grid
    t0 = time.perf_counter()
    ctx = _lib.Context.get(0)
    da = gen.stencil_device(gen.BRICK3D, (n, n, n))
    a = da.download()                                # pinned host arrays
    del da
    ctx.sync()
    gen_s = time.perf_counter() - t0
    mults = int(np.diff(a.row_ptr)[a.col_idx].sum())
    caps = [args.hbm_cap_gib] + list(getattr(args, "extra_caps_gib", []) or [])
    link = link_peaks()
    runs = []
    cb_o = None
    for cap in caps:
        fast = int(cap * 2**30)
        counts, sym = ch.symbolic_within_budget(a, a, fast)
        plan = ch.plan_for_multiply(a, a, counts, fast)
        model = b200_model(fast)
        c, led = ch.execute_plan(a, a, counts, plan, model)
        ph = led.physical
        # parity: random rows + the first/last row of every planned range,
        # through the oracle with B compressed once
        rng = np.random.default_rng(0)
        rows = set(int(x) for x in rng.choice(a.num_rows, size=24, replace=False))
        for part in (plan.partition_ac, plan.partition_b):
            for r in part.ranges:
                rows.update({r.begin, max(r.begin, r.end - 1)})
        rows = sorted(x for x in rows if x < a.num_rows)
        if cb_o is None:
            cb_o = O.compress(a)
        exact = ok = True
        for r in rows:
            sub = slice_rows(a, r, r + 1)
            want = O.numeric(sub, a, O.symbolic(sub, cb_o))
            lo, hi = int(c.row_ptr[r]), int(c.row_ptr[r + 1])
            got = CsrMatrix._adopt(1, c.num_cols, np.array([0, hi - lo]), c.col_idx[lo:hi], c.values[lo:hi])
            res = compare_products(got, want)
            exact &= res["exact"]
            ok &= res["ok"]
        nnz_ok = bool(c.nnz == int(np.sum(counts)))
        secs = ph["wall_ms"] / 1e3
        runs.append({
            "hbm_cap_gib": cap, "value": 2 * mults / secs / 1e9, "unit": UNIT,
            "host_link": {"achieved_gbs": ph["link_gbs"], "h2d_bytes": ph["h2d_bytes"],
                          "d2h_bytes": ph["d2h_bytes"], "wall_s": secs,
                          "kernel_s": ph["kernel_ms"] / 1e3,
                          "link_peak": link,
                          "frac_of_bidir_peak": ph["link_gbs"] / link["bidir_total_gbs"],
                          "h2d_engine_frac": ph["h2d_bytes"] / secs / 1e9 / link["h2d_gbs"]},
            "hbm": {"cap_bytes": fast, "peak_device_bytes": ph["peak_device_bytes"],
                    "layout_bytes": ph["layout_bytes"], "slots": ph["slots"], "split": ph["split"],
                    "symbolic_peak_device_bytes": sym["peak_device_bytes"],
                    "symbolic_wall_s": sym["wall_ms"] / 1e3},
            "plan": {"algorithm": plan.algorithm, "branch": plan.heuristic_branch,
                     "n_ac": len(plan.partition_ac), "n_b": len(plan.partition_b),
                     "ledger_bytes": led.total_bytes(),
                     "predicted_copy_bytes": plan.predicted_copy_bytes},
            "nnz_C": c.nnz,
            "parity": {"ok": bool(ok and nnz_ok), "exact": bool(exact), "rows_checked": len(rows),
                       "nnz_C_exact": nnz_ok}})
        del c
    # CPU rate of the oracle, extrapolated: compress of the whole B once plus
    # symbolic + numeric on a row sample scaled by its share of the multiplications
    sample = slice_rows(a, 0, 65536)
    smults = int(np.diff(a.row_ptr)[sample.col_idx].sum())
    W = os.cpu_count() or 1
    t1 = time.perf_counter()
    cb2 = O.compress(a)
    tc = time.perf_counter() - t1
    t1 = time.perf_counter()
    O.numeric(sample, a, O.symbolic(sample, cb2, W), W)
    ts = time.perf_counter() - t1
    cpu_s = tc + ts * mults / smults
    main = runs[0]
    return {"metric": "chunked SpGEMM GFLOP/s config 4 (A*A brick3d %d^3, HBM cap %.1f GiB)"
                      % (n, args.hbm_cap_gib),
            "value": main["value"], "unit": UNIT, "dtype": "f64", "data": "synthetic",
            "host_link": main["host_link"], "hbm": main["hbm"], "plan": main["plan"],
            "parity": main["parity"], "runs": runs,
            "config": {"workload": "config4", "rows": a.num_rows, "nnz_A": a.nnz, "nnz_C": main["nnz_C"],
                       "multiplications": mults, "setup_s": gen_s},
            "cpu_baseline": {"value": 2 * mults / cpu_s / 1e9, "unit": UNIT,
                             "cores": W, "kind": "port",
                             "sample": "oracle compress of the whole B + symbolic/numeric of the "
                                       "first 65536 rows, extrapolated by multiplications"}}


# ------------------------------------------------------------------ placement table

def placement(args):
    """The paper's data-placement table (Laplace R x A:
    HBM / A_Pin / B_Pin / C_Pin / HostPin) on B200: config 2's R*A with each
    operand either in HBM or in pinned, device-mapped host memory that the
    kernels read/write in place over PCIe."""
    import paper_1804_00695_b200 as tsg
    from paper_1804_00695_b200 import generators as gen
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


# ------------------------------------------------------------------ config 5

def config5(args, dist=None):
    """BASELINE.json config 5: A*A on an R-MAT graph (Graph500 parameters,
    SplitMix64 seed 22, unit values), rows partitioned over the ranks by K0
    flops, B replicated (NCCL all-gather) or sharded in peer HBM
    (``--b-mode``), C streamed through ``--c-budget-gib`` when it does not fit.
    Strong scaling: the graph is fixed, every rank takes 1/N of the flops.
    Timing: CUDA events on each rank's libtsg stream around the block
    multiply + offset exchange, max over ranks.  Parity: every rank's sum of
    C's values equals its multiplications exactly (unit values: C_ij counts
    paths, so the sum over a block is its K0 flops), the global nnz is
    all-reduced, and sampled rows (incl. the hub) match the oracle."""
    import torch
    from paper_1804_00695_b200 import _lib, generators as gen
    from paper_1804_00695_b200 import distributed as D
    from paper_1804_00695_b200.csr import CsrMatrix
    world = dist.get_world_size() if dist else 1
    rank = dist.get_rank() if dist else 0
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    ctx = _lib.Context.get(local)
    ctx.set_timing(True)
    stream = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", local))
    t_setup = time.perf_counter()
    da = gen.rmat_graph_device(args.scale).set_values(1.0)
    n = da.num_rows
    row_flops, total = _lib.d_row_flops(da, da)
    bounds = D.flops_partition(row_flops, world)
    lo, hi = int(bounds[rank]), int(bounds[rank + 1])
    a_blk = da.slice_rows(lo, hi)
    mode = getattr(args, "b_mode", "replicated") if world > 1 else "local"
    info = {}
    t_b = time.perf_counter()
    if world == 1:
        db = da
    elif mode == "sharded":
        db, info = D.shard_b(ctx, da, dist, sorted_rows=True)
    else:
        sb = D.shard_bounds(np.diff(D.rp_host(ctx, da)), world)
        shard = da.slice_rows(int(sb[rank]), int(sb[rank + 1]))
        db = D.replicate_b(ctx, shard, n, n, dist)
        del shard
    b_setup_s = time.perf_counter() - t_b
    host_a = da.download() if rank == 0 or not getattr(args, "no_parity", False) else None
    if world > 1:
        del da
    budget = int(getattr(args, "c_budget_gib", 48.0) * 2**30)
    mults = int(row_flops[lo:hi].sum())
    est_c_bytes = 12 * mults   # nnz(C) <= multiplications
    c_budget = budget if est_c_bytes > budget else 0
    setup_s = time.perf_counter() - t_setup

    def step():
        ctx.record(0)
        _, st = D.mg_multiply(a_blk, db, c_budget, keep_c=False)
        if dist:
            with torch.cuda.stream(stream):
                off, tot = D.exchange_offsets(st["nnz"], dist)
        else:
            off, tot = 0, st["nnz"]
        ctx.record(1)
        return st, off, tot

    for _ in range(max(1, args.warmup)):
        st, off, tot = step()
    if dist:
        dist.barrier()
    times = []
    for _ in range(args.steps):
        st, off, tot = step()
        times.append(ctx.elapsed_ms(0, 1))
    my_ms = statistics.median(times)
    ms = my_ms
    flops_all = 2 * total
    sums_ok = bool(st["value_sum"] == float(mults))
    if dist:
        dev = D._coll_device(dist)
        t = torch.tensor([my_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        ok = torch.tensor([1.0 if sums_ok else 0.0], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        sums_ok = bool(ok.item() > 0.5)
    # sampled rows of this block (incl. its largest-flops row) against the oracle
    par = {"block_value_sum_equals_mults": sums_ok, "nnz_C": tot}
    if not getattr(args, "no_parity", False):
        from oracle import oracle as O
        cb = O.compress(host_a)
        rng = np.random.default_rng(rank)
        rows = sorted(set([lo + int(np.argmax(row_flops[lo:hi]))] +
                          [int(x) for x in rng.integers(lo, hi, size=min(6, hi - lo))])) if hi > lo else []
        exact = ok = True
        for r in rows:
            sub = CsrMatrix._adopt(1, n, np.array([0, host_a.row_ptr[r + 1] - host_a.row_ptr[r]]),
                                   host_a.col_idx[host_a.row_ptr[r]:host_a.row_ptr[r + 1]],
                                   host_a.values[host_a.row_ptr[r]:host_a.row_ptr[r + 1]])
            want = O.numeric(sub, host_a, O.symbolic(sub, cb))
            c1, _ = D.mg_multiply(a_blk.slice_rows(r - lo, r - lo + 1), db, 0, keep_c=True)
            res = compare_products(c1.download(), want)
            exact &= res["exact"]
            ok &= res["ok"]
        if dist:
            dev = D._coll_device(dist)
            t = torch.tensor([1.0 if ok else 0.0, 1.0 if exact else 0.0], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            ok, exact = bool(t[0].item() > 0.5), bool(t[1].item() > 0.5)
        par.update(sampled_rows_ok=ok, sampled_rows_exact=exact, rows_per_rank=len(rows))
    par["ok"] = bool(sums_ok and par.get("sampled_rows_ok", True))
    line = {"metric": "SpGEMM GFLOP/s config 5 (A*A R-MAT scale %d, %d GPU, B %s)" % (args.scale, world, mode),
            "value": flops_all / (ms * 1e-3) / 1e9, "unit": "GFLOP/s", "n_gpus": world,
            "ms_per_step": ms, "steps": args.steps, "warmup": args.warmup, "scaling": "strong",
            "higher_is_better": True, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "config5 A*A R-MAT scale %d ef16 (.57,.19,.19,.05) SplitMix64 seed 22"
                                   % args.scale, "n": n, "multiplications": total,
                       "b_mode": mode, "partition": "K0 flops, contiguous row blocks",
                       "c_mode": "streamed (budget %d GiB per GPU)" % (budget >> 30) if c_budget else
                                 "materialised per GPU", "rank0_block_rows": hi - lo},
            "per_rank": {"ms": my_ms, "blocks": st["blocks"], "max_block_nnz": st["max_block_nnz"],
                         "mults": mults},
            "setup": {"total_s": setup_s, "b_setup_s": b_setup_s, **info},
            "parity": par}
    return line


# ------------------------------------------------------------------ driver hooks

def run(args, dist=None):
    if args.config == 5:
        return config5(args, dist)
    return {1: config1, 3: config3, 4: config4, 6: placement}[args.config](args)


def secondary(args):
    """Configs 1, 3 and 4 at their BASELINE sizes, and config 5 at R-MAT
    scales 20 and 21 (the scale-25 run is ``--config 5 --scale 25`` on 8
    GPUs), for the default N=1 run."""
    out = {}
    jobs = (("config1", config1, dict(steps=20)),
            ("config3", config3, dict(steps=5, scale=22)),
            ("config4", config4, dict(grid=256, hbm_cap_gib=8.0, extra_caps_gib=[16.0])),
            ("config5", config5, dict(scale=20, steps=2, warmup=1, c_budget_gib=48.0)),
            ("config5_scale21", config5, dict(scale=21, steps=1, warmup=1, c_budget_gib=48.0)))
    for name, fn, over in jobs:
        a = argparse.Namespace(**vars(args))
        a.warmup = 3
        a.no_parity = False
        for k, v in over.items():
            setattr(a, k, v)
        t0 = time.perf_counter()
        try:
            out[name] = fn(a)
        except Exception as exc:   # a secondary failure must not hide the headline line
            out[name] = {"error": "%s: %s" % (type(exc).__name__, exc)}
        out[name]["wall_s"] = time.perf_counter() - t0
    return out
