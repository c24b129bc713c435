#!/usr/bin/env python
"""Benchmark: SpGEMM GFLOP/s on BASELINE.json config 2 (multigrid R*A*P).

Workload (N=1): brick3d 27-point stencil on a 128^3 grid (fp64, 26/-1), plain
2x2x2 aggregation prolongator P (64^3 coarse), R = P^T; one step computes
RA = R*A then RAP = RA*P with compress -> symbolic -> numeric on the device.
flops = 2 * (count_multiplications(R, A) + count_multiplications(RA, P)).

After the timed loop the step's RA and RAP are downloaded once and compared
with the CPU oracle's full R*A*P (structure bit-exact, values bit-exact or
within the north star's 1e-12): the line carries ``parity`` and the process
exits 1 on a mismatch.  At N=1 rank 0 also emits ``secondary`` lines for
BASELINE.json configs 1, 3 and 4 (bench_configs.py), each with its own parity
check, so they are driver-observed.

N>1 (one rank per GPU, NCCL): weak scaling.  ``python bench.py --gpus N``
re-executes itself under torch.distributed.run when WORLD_SIZE is unset.  The
grid grows to 128 x 128 x 128N; rank r owns the coarse z-slab r, i.e. a
contiguous block of R's rows (the row partition of A in the north star).  Each
rank builds only its slab of the fine operator, the B operand (the fine A) is
replicated by an NCCL all-gather at setup (or read from peer HBM with
``--b-mode sharded``), and every step ends with the row-pointer offset
exchange (all-gather of per-rank nnz) on libtsg's compute stream, inside the
event-timed region.  ``--config 5`` runs the R-MAT A*A strong-scaling arm
(bench_configs.config5 / distributed.mg_multiply).

Output: one JSON line (rank 0) with value / e2e / roofline / cpu_baseline /
clocks / gpu_launches / parity, as the driver's contract asks.
"""

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SpGEMM GFLOP/s (2 x multiplications / time), config 2 R*A*P"
UNIT = "GFLOP/s"
L2_BYTES = 126 * 2**20


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ workload

def build_problem(world, rank, base=128):
    """Fine operator rows of this rank's slab (+ the full fine grid shape),
    R rows for this rank's coarse slab, and P (fine -> coarse)."""
    from paper_1804_00695_b200 import generators as gen
    from paper_1804_00695_b200.csr import CsrMatrix
    nz = base * world
    dims = (base, base, nz)
    a = gen.stencil(gen.BRICK3D, dims) if world == 1 else None
    p, r = gen.aggregation(dims)
    if world == 1:
        return dims, a, r, p
    # fine rows of slab `rank` (z in [rank*base, (rank+1)*base)) of the big grid
    plane = base * base
    lo, hi = rank * base * plane, (rank + 1) * base * plane
    full = gen.stencil_rows(gen.BRICK3D, dims, lo, hi)
    # coarse rows of slab `rank`
    cplane = (base // 2) * (base // 2)
    clo, chi = rank * (base // 2) * cplane, (rank + 1) * (base // 2) * cplane
    r_loc = CsrMatrix._adopt(chi - clo, r.num_cols, r.row_ptr[clo:chi + 1] - r.row_ptr[clo],
                             r.col_idx[r.row_ptr[clo]:r.row_ptr[chi]],
                             r.values[r.row_ptr[clo]:r.row_ptr[chi]])
    return dims, full, r_loc, p


def sizes_ref(rows, nnz):
    return 8 * (rows + 1) + 16 * nnz


def sizes_dev(rows, nnz):
    return 8 * (rows + 1) + 12 * nnz


def config2_desc(dims, world, mults, nnz):
    """The config object both arms print (identical, so the driver can match
    them): workload, grid, multiplications and operand sizes."""
    return {"workload": "config2 R*A*P brick3d %dx%dx%d + 2x2x2 aggregation" % tuple(dims),
            "grid": list(dims), "multiplications": int(mults),
            "nnz": {k: int(v) for k, v in nnz.items()},
            "parallelism": ("row partition of R (coarse z-slabs) x%d" % world) if world > 1
            else "single GPU",
            "l2_between_steps": "inputs larger than L2 (A > 0.7 GB) and a 252 MiB L2 flush before each "
                                "timed step"}


# ------------------------------------------------------------------ clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "10"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.monotonic()   # nvidia-smi takes a moment to print its first line
            while not self.lines and time.monotonic() - t0 < 5.0:
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def mark(self, which):
        setattr(self, which, time.monotonic())

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        # samples taken inside the timed region (else the ones around it)
        lo, hi = getattr(self, "t_begin", None), getattr(self, "t_end", None)
        inside = [ln for t, ln in self.lines if lo is not None and hi is not None and lo <= t <= hi + 0.01]
        chosen = inside or [ln for _, ln in self.lines[-3:]]
        for ln in chosen:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "samples_in_timed_region": len(inside)}


# ------------------------------------------------------------------ CPU side (checker + baseline)

def cpu_rap(r, a, p, workers):
    """The oracle's R*A*P (the reference's algorithm restated in C): seconds,
    RA (CsrMatrix, first-touch column order), RAP (ptr, col, val)."""
    from oracle import oracle as O
    from paper_1804_00695_b200.csr import CsrMatrix
    t0 = time.perf_counter()
    ra = O.multiply(r, a, workers=workers)
    ra_m = CsrMatrix._adopt(r.num_rows, a.num_cols, *ra)
    rap = O.multiply(ra_m, p, workers=workers)
    dt = time.perf_counter() - t0
    return dt, ra_m, rap


def run_reference(args, world, rank):
    """--impl reference: the reference's algorithm on the host cores (the
    oracle port over all threads), same config / metric / unit as our arm.
    Under torchrun only rank 0 works."""
    if rank != 0:
        return
    from oracle import oracle as O
    dims, a, r, p = build_problem(1, 0, args.base)
    workers = os.cpu_count() or 1
    times = []
    ra = rap = None
    for i in range(args.warmup + args.steps):
        dt, ra, rap = cpu_rap(r, a, p, workers)
        if i >= args.warmup:
            times.append(dt)
    m1 = O.count_multiplications(r, a)
    m2 = ra.nnz   # P has exactly one entry per row: mults(RA, P) = nnz(RA)
    fl = 2 * (m1 + m2)
    sec = statistics.median(times)
    val = fl / sec / 1e9
    dt1, _, _ = cpu_rap(r, a, p, 1)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": config2_desc(dims, 1, m1 + m2, {"A": a.nnz, "R": r.nnz, "RA": ra.nnz,
                                                  "RAP": len(rap[1])}),
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": workers, "kind": "port",
                         "w1_value": fl / dt1 / 1e9, "nproc": os.cpu_count(),
                         "sample": "full config-2 R*A*P per step (oracle/tsg_oracle.c, pthreads "
                                   "over row blocks, the reference's algorithm restated in C); "
                                   "w1_value = the same with 1 thread.  The Python reference is "
                                   "GIL-bound at ~1.3 MFLOP/s (BASELINE.md §2)"},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ launcher

def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def maybe_spawn(args):
    """`bench.py --gpus N` without torchrun: re-execute under
    torch.distributed.run with N ranks (one per GPU) and return its exit code.
    Returns None when no spawn is needed."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    if args.impl == "ours":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(json.dumps({"error": "--gpus %d but only %d CUDA device(s) visible" % (args.gpus, have)}),
                  flush=True)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node", str(args.gpus), "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


# ------------------------------------------------------------------ our arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the config 1 / 3 / 4 secondary lines of the default N=1 run")
    ap.add_argument("--phases", action="store_true", help="print per-phase device times and exit")
    ap.add_argument("--base", type=int, default=128,
                    help="config 2 fine grid edge per GPU (BASELINE config 2: 128)")
    ap.add_argument("--b-mode", default="replicated", choices=["replicated", "sharded"],
                    help="N>1: B all-gathered once (replicated) or kept as row shards read "
                         "from peer HBM (sharded, SURVEY.md §8e)")
    ap.add_argument("--profile-step", action="store_true",
                    help="after warm-up run ONE step between cudaProfilerStart/Stop and exit "
                         "(for ncu --profile-from-start off)")
    ap.add_argument("--config", type=int, default=2,
                    help="BASELINE.json config (2 = the driver's bench line; 1, 3, 4, 5 = secondary)")
    ap.add_argument("--scale", type=int, default=22, help="R-MAT scale for --config 3 / 5")
    ap.add_argument("--grid", type=int, default=256, help="brick grid edge for --config 4")
    ap.add_argument("--hbm-cap-gib", type=float, default=8.0, help="HBM budget for --config 4")
    ap.add_argument("--c-budget-gib", type=float, default=48.0,
                    help="--config 5: HBM for one chunk of C (streamed-C mode above it)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup

    rc = maybe_spawn(args)
    if rc is not None:
        sys.exit(rc)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        raise SystemExit("bench.py: --gpus %d but WORLD_SIZE=%d" % (args.gpus, world))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "ours":
            torch.cuda.set_device(local)
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")

    if args.impl == "reference":
        if world == 1 and args.gpus > 1:
            world = args.gpus   # bare --gpus N: the host run stands for all N
        run_reference(args, world, rank)
        if dist:
            dist.destroy_process_group()
        return
    if args.config != 2:
        import bench_configs
        line = bench_configs.run(args, dist=dist)
        if rank == 0:
            print(json.dumps(line), flush=True)
        if dist:
            dist.destroy_process_group()
        if line.get("parity", {}).get("ok") is False:
            sys.exit(1)
        return
    ok = run_config2(args, world, rank, local, dist)
    if dist:
        dist.destroy_process_group()
    if not ok:
        sys.exit(1)


def run_config2(args, world, rank, local, dist):
    import torch
    from paper_1804_00695_b200 import _lib, kernel

    torch.cuda.set_device(local)
    ctx = _lib.Context.get(local)
    ctx.set_timing(True)
    tsg_stream = torch.cuda.ExternalStream(ctx.stream(), device=torch.device("cuda", local))

    dims, a_loc, r, p = build_problem(world, rank, args.base)
    dr = _lib.DeviceCsr.upload(r, ctx)
    dp = _lib.DeviceCsr.upload(p, ctx)
    setup = {}
    if world == 1:
        da = _lib.DeviceCsr.upload(a_loc, ctx)
    elif args.b_mode == "sharded":
        da, setup = sharded_b(ctx, a_loc, dr, dims, world, rank, torch, dist)
    else:
        da, setup = replicate_b(ctx, a_loc, dims, world, rank, torch, dist)
    a_rows, a_nnz = da.num_rows, da.nnz

    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device="cuda")

    def step():
        # events: 0 step start, 4 between the two multiplies, 1 step end (after
        # the offset exchange).  The R*A numeric phase is the roofline kernel:
        # remember its call id in libtsg's event ring (no sync inside a step)
        ctx.record(0)
        call = ctx.numeric_calls()
        dra = kernel.multiply_device(dr, da)
        ctx.record(4)
        drap = kernel.multiply_device(dra, dp)
        if dist:
            with torch.cuda.stream(tsg_stream):
                exchange_offsets(drap.nnz, dist)
        ctx.record(1)
        return dra, drap, call

    for _ in range(args.warmup):
        dra, drap, _ = step()
    if args.profile_step:
        ctx.sync()
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        dra, drap, _ = step()
        ctx.sync()
        torch.cuda.profiler.stop()
        return True
    if args.phases:
        print_phases(ctx, kernel, dr, da, dp)
        return True
    ra_rows, ra_nnz, rap_nnz = dra.num_rows, dra.nnz, drap.nnz
    m1 = _lib.d_count_multiplications(dr, da)
    m2 = _lib.d_count_multiplications(dra, dp)
    flops_rank = 2 * (m1 + m2)
    del dra, drap

    sampler = ClockSampler(local)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    ctx.sync()
    sampler.start()
    sampler.mark("t_begin")
    l0 = ctx.stats()[0]
    times, ra_times, rap_times, num_times = [], [], [], []
    for _ in range(args.steps):
        # L2 flush on libtsg's stream, ahead of the step's event 0: the flush
        # evicts the previous step's data, and the host queues the step while
        # it runs (no host round trip inside the timed region)
        with torch.cuda.stream(tsg_stream):
            flush.fill_(1)
        dra, drap, call = step()
        times.append(ctx.elapsed_ms(0, 1))
        ra_times.append(ctx.elapsed_ms(0, 4))
        rap_times.append(ctx.elapsed_ms(4, 1))
        num_times.append(ctx.numeric_ms(call))
        del dra, drap
    l1 = ctx.stats()[0]
    ctx.sync()
    torch.cuda.synchronize()
    sampler.mark("t_end")
    if dist:
        dist.barrier()
    clocks = sampler.stop()

    tot_ms = sum(times)
    if dist:
        t = torch.tensor([tot_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms = float(t.item())
        fl = torch.tensor([flops_rank], dtype=torch.float64, device="cuda")
        dist.all_reduce(fl)
        flops_all = float(fl.item())
    else:
        flops_all = float(flops_rank)
    ms_step = tot_ms / args.steps
    value = flops_all / (ms_step * 1e-3) / 1e9

    # roofline of the dominant kernel: numeric kernels of R*A, algorithmic
    # bytes in the reference's byte convention (8 B offsets / indices /
    # values): size(R) + size(A) + size(RA)
    hbm, peak_kind = peaks()
    alg_ra = sizes_ref(r.num_rows, r.nnz) + sizes_ref(a_rows, a_nnz) + sizes_ref(ra_rows, ra_nnz)
    dev_ra = sizes_dev(r.num_rows, r.nnz) + sizes_dev(a_rows, a_nnz) + sizes_dev(ra_rows, ra_nnz)
    alg_rap = sizes_ref(ra_rows, ra_nnz) + sizes_ref(p.num_rows, p.nnz) + sizes_ref(ra_rows, rap_nnz)
    num_ms = statistics.median(num_times)
    achieved = alg_ra / (num_ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r03_traffic.json")) as fh:
            traffic = int(json.load(fh)["traffic_bytes_per_launch"])
    except Exception:
        pass
    ra_ms, rap_ms = statistics.median(ra_times), statistics.median(rap_times)
    whole = {
        "definition": "SURVEY.md §8(d): compress -> symbolic -> scan -> numeric of each multiply, "
                      "reference-convention bytes size(A)+size(B)+size(C) / event-timed device time",
        "RA_multiply": {"ms": ra_ms, "bytes": alg_ra, "frac": alg_ra / (ra_ms * 1e-3) / 1e9 / hbm},
        "RAP_multiply": {"ms": rap_ms, "bytes": alg_rap, "frac": alg_rap / (rap_ms * 1e-3) / 1e9 / hbm},
        "step": {"ms": ms_step, "bytes": alg_ra + alg_rap,
                 "frac": (alg_ra + alg_rap) / (ms_step * 1e-3) / 1e9 / hbm},
    }
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic,
            "kernel": "k_num_group (numeric phase of R*A, all bins)",
            "peak_kind": peak_kind, "algorithmic_bytes": alg_ra,
            "device_layout_bytes": dev_ra, "device_layout_frac": dev_ra / (num_ms * 1e-3) / 1e9 / hbm,
            "kernel_ms": num_ms, "whole_multiply": whole,
            "note": "traffic = dram__bytes_read.sum + dram__bytes_write.sum of the dominant launch "
                    "from the ncu launch list of one warm step (profiles/r03_traffic.json)"}

    nnz = {"A": a_nnz, "R": r.nnz, "RA": ra_nnz, "RAP": rap_nnz}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config2_desc(dims, world, m1 + m2, nnz),
        "notes": {"l2": "A (>0.7 GB) and RA (>0.2 GB) exceed L2; a 252 MiB L2 flush on libtsg's stream "
                        "precedes every step (outside its events)",
                  "timing": "CUDA events on libtsg's compute stream, max over ranks; N>1 includes "
                            "the offset all-gather on that stream",
                  "b_mode": args.b_mode if world > 1 else None},
        "roofline": roof,
        "clocks": clocks,
        "gpu_launches": int(l1 - l0),
        "setup": setup,
    }

    # ---- parity: this step's RA and RAP against the oracle's full product
    ok = True
    cpu = None
    if not args.no_parity:
        import bench_configs as BC
        dra, drap, _ = step()
        ctx.sync()
        ra_got, rap_got = dra.download(), drap.download()
        del dra, drap
        a_full = a_loc if world == 1 else BC.embed_rows(a_loc, dims, rank, args.base)
        dt, ra_o, rap_o = cpu_rap(r, a_full, p, os.cpu_count() or 1)
        cpu = dt
        par_ra = BC.compare_products(ra_got, (ra_o.row_ptr, ra_o.col_idx, ra_o.values))
        par_rap = BC.compare_products(rap_got, rap_o)
        ok = par_ra["ok"] and par_rap["ok"]
        par = {"ok": ok, "exact": par_ra["exact"] and par_rap["exact"], "RA": par_ra, "RAP": par_rap,
               "oracle": "oracle/tsg_oracle.c full R*A*P (the reference's algorithm; pinned to the "
                         "reference's outputs by tests/test_oracle.py)",
               "rule": "row pointers + per-row sorted columns bit-exact; values bit-exact or "
                       "rel <= 1e-12 (abs <= 1e-250)"}
        if dist:
            t = torch.tensor([1.0 if ok else 0.0, 1.0 if par["exact"] else 0.0], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            par["all_ranks_ok"], par["all_ranks_exact"] = bool(t[0].item()), bool(t[1].item())
            ok = par["all_ranks_ok"]
        line["parity"] = par

    if rank == 0 and world == 1 and not args.no_e2e:
        line["e2e"] = run_e2e(ctx, r, a_loc, p, args)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        if cpu is None:
            cpu, _, _ = cpu_rap(r, a_loc, p, os.cpu_count() or 1)
        cpu1, _, _ = cpu_rap(r, a_loc, p, 1)
        line["cpu_baseline"] = {
            "value": flops_rank / cpu / 1e9, "unit": UNIT, "cores": os.cpu_count() or 1,
            "kind": "port", "w1_value": flops_rank / cpu1 / 1e9, "nproc": os.cpu_count(),
            "sample": "one full config-2 R*A*P on the host (oracle/tsg_oracle.c with %d pthreads; "
                      "the reference's algorithm restated in C); w1_value = 1 thread"
                      % (os.cpu_count() or 1)}
    if not args.no_secondary:
        import bench_configs as BC
        if world == 1:
            line["secondary"] = BC.secondary(args)
        else:   # config 5 strong scaling over the same ranks (every rank takes part)
            ns = argparse.Namespace(**vars(args))
            ns.scale, ns.steps, ns.warmup, ns.no_parity = 20, 2, 1, False
            line["secondary"] = {"config5": BC.config5(ns, dist)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    return ok


def print_phases(ctx, kernel, dr, da, dp):
    for _ in range(4):
        ctx.record(0)
        h0 = time.perf_counter()
        res0 = ctx.pool_reserved()
        dra = kernel.multiply_device(dr, da)
        h1 = time.perf_counter()
        ph1, st1 = ctx.phase_ms(), ctx.stats()
        drap = kernel.multiply_device(dra, dp)
        ph2, st2 = ctx.phase_ms(), ctx.stats()
        ctx.record(1)
        h2 = time.perf_counter()
        print(json.dumps({"step_ms": ctx.elapsed_ms(0, 1), "host_ms": [1e3 * (h1 - h0), 1e3 * (h2 - h1)],
                          "pool_reserved_mb": [res0 >> 20, ctx.pool_reserved() >> 20],
                          "RA": {"compress": ph1[0], "symbolic": ph1[1], "scan": ph1[2],
                                 "numeric": ph1[3], "total": ph1[5],
                                 "sym_kernels": st1[1], "num_kernels": st1[2]},
                          "RAP": {"compress": ph2[0], "symbolic": ph2[1], "scan": ph2[2],
                                  "numeric": ph2[3], "total": ph2[5],
                                  "sym_kernels": st2[1], "num_kernels": st2[2]}}))


def exchange_offsets(local_nnz, dist):
    """Row-pointer offset exchange: all-gather of per-rank nnz(C slice)."""
    from paper_1804_00695_b200 import distributed as D
    return D.exchange_offsets(local_nnz, dist, "cuda")


def replicate_b(ctx, a_loc, dims, world, rank, torch, dist):
    """NCCL all-gather of the fine operator's row shards into a full device B."""
    from paper_1804_00695_b200 import _lib
    from paper_1804_00695_b200 import distributed as D
    t0 = time.perf_counter()
    rp, col, val = D.allgather_csr(torch.from_numpy(np.diff(a_loc.row_ptr)).cuda(),
                                   torch.from_numpy(a_loc.col_idx.astype(np.int32)).cuda(),
                                   torch.from_numpy(np.asarray(a_loc.values)).cuda(), dist, "cuda")
    torch.cuda.synchronize()
    n_full = rp.numel() - 1
    da = _lib.DeviceCsr.from_device(ctx, n_full, a_loc.num_cols, int(col.numel()), rp.data_ptr(),
                                    col.data_ptr(), val.data_ptr())
    return da, {"b_allgather_s": time.perf_counter() - t0,
                "b_bytes_per_rank": int(8 * (a_loc.num_rows + 1) + 12 * a_loc.nnz)}


def sharded_b(ctx, a_loc, dr, dims, world, rank, torch, dist):
    """B sharded: every rank keeps its slab of the fine operator; the slabs are
    shared once as CUDA IPC handles and the rows this rank's R selects (its
    slab plus one halo plane from each neighbour) are gathered by a kernel
    reading peer HBM over NVLink.  No collective in the multiply."""
    from paper_1804_00695_b200 import distributed as D
    t0 = time.perf_counter()
    plane = dims[0] * dims[1]
    lo, hi = rank * dims[0] * plane, (rank + 1) * dims[0] * plane
    rp = torch.from_numpy(np.asarray(a_loc.row_ptr, dtype=np.int64)).cuda()
    col = torch.from_numpy(np.asarray(a_loc.col_idx, dtype=np.int32)).cuda()
    val = torch.from_numpy(np.asarray(a_loc.values)).cuda()
    shards = D.share_shards((rp, col, val), lo, hi, dist)
    torch.cuda.synchronize()
    db = D.gather_sharded(dr, shards, a_loc.num_cols)
    return db, {"b_shard_gather_s": time.perf_counter() - t0, "b_mode": "sharded",
                "b_rows_gathered_nnz": int(db.nnz)}


def run_e2e(ctx, r, a, p, args):
    """Same metric through the public drop-in API (kernel.multiply) with host
    CsrMatrix operands in pinned memory: every step uploads R, A, then P,
    downloads RA and RAP (fresh host wrappers defeat the residency cache)."""
    import torch
    from paper_1804_00695_b200 import kernel
    from paper_1804_00695_b200.csr import CsrMatrix

    def pinned(m):
        def pin(x, dt):
            t = torch.empty(len(x), dtype=dt, pin_memory=True)
            t.numpy()[:] = x
            return t.numpy()
        v = None if m.values is None else pin(m.values, torch.float64)
        return (m.num_rows, m.num_cols, pin(m.row_ptr, torch.int64), pin(m.col_idx, torch.int64), v)

    pr, pa, pp = pinned(r), pinned(a), pinned(p)

    def fresh(t):
        return CsrMatrix._adopt(*t)

    def one():
        ctx.record(2)
        ra = kernel.multiply(fresh(pr), fresh(pa))
        rap = kernel.multiply(ra, fresh(pp))
        ctx.record(3)
        return ra, rap, ctx.elapsed_ms(2, 3)

    for _ in range(2):
        ra, rap, _ = one()
    times = []
    for _ in range(max(3, min(args.steps, 5))):
        ra, rap, ms = one()
        times.append(ms)
    fl = 2 * (kernel.count_multiplications(r, a) + ra.nnz)
    ms = statistics.median(times)
    # RA comes back from the first multiply with its device copy kept, so the
    # second multiply does not upload it again
    h2d = sum(8 * (m.num_rows + 1) + 16 * m.nnz for m in (r, a, p))
    d2h = sum(8 * (m.num_rows + 1) + 16 * m.nnz for m in (ra, rap))
    return {"value": fl / (ms * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": ms,
            "path": "paper_1804_00695_b200.kernel.multiply (C ABI, host CsrMatrix in/out)"}


if __name__ == "__main__":
    main()
