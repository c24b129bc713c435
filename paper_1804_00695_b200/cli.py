"""Benchmark command line with the reference's report schema v1, measured on
the B200 (the reference's cli.py:1-530).

Subcommands, flags, defaults, config-file precedence (defaults < ``--config``
key=value file < flags), output formats and exit codes (0 ok, 2 validation
error, 3 ``--verify`` mismatch) follow the reference.  Every run record keeps
the reference's fields with the reference's meaning -- ``simulated_seconds``
= the two-tier cost model's kernel estimate + the copy ledger's billed
seconds, so a B200 report and a reference report of the same spec agree on
those fields -- and adds a ``measured`` object with what the B200 actually
took:

* ``h2d_seconds`` / ``device_seconds`` / ``d2h_seconds``: CUDA-event times
  on libtsg's compute stream of the operand upload, compress -> symbolic ->
  numeric, and the result download (all_fast);
* placement modes (all_slow, b_in_fast): ``device_seconds`` of the multiply
  reading / writing the slow operands in mapped host memory over PCIe;
* chunk mode: the physical executor's wall / kernel seconds and DMA bytes
  (``CopyLedger.physical``);
* ``b200_model_seconds``: the reference's linear model with the parameters
  fitted to B200 runs (memory.estimate_kernel_time_b200, §8f row 4).

``workers`` is accepted and recorded; results do not depend on it.
"""

import argparse
import json
import os
import statistics
import sys
import time
from dataclasses import dataclass

import numpy as np

from . import chunking
from .csr import products_match, validate
from .errors import TieredSpgemmError, VerifyError
from .generators import (BIGSTAR2D, BRICK3D, ELASTICITY3D, LAPLACE3D, StencilSpec,
                         generate_interpolation, generate_random_rhs, generate_stencil,
                         grid_for_target_bytes)
from .kernel import compress, spgemm_numeric, spgemm_symbolic
from .matrix_market import read_matrix_market, write_matrix_market
from .memory import (CHUNKED, MemoryModel, MemorySpaceSpec, PlacementPolicy,
                     compute_access_stats, estimate_kernel_time, estimate_kernel_time_b200,
                     validate_placement)
from .triangles import count_triangles, load_graph

SCHEMA_VERSION = 1
OFFSET_BYTES = 8

MODES = ("all_fast", "all_slow", "b_in_fast", "chunk")
PRODUCTS = ("AxP", "RxA")
PROBLEMS = (LAPLACE3D, BIGSTAR2D, BRICK3D, ELASTICITY3D, "file")

DEFAULTS = {
    "problem": LAPLACE3D, "product": "RxA", "grid": (9, 9, 9), "target_bytes": None,
    "mode": "all_slow", "fast_size": None, "fast_bandwidth": 400e9, "slow_bandwidth": 20e9,
    "fast_latency": 1e-7, "slow_latency": 1e-6, "seed": 0, "reps": 5, "verify": False,
    "workers": os.cpu_count() or 1, "format": "json", "out": None,
}

RUN_FIELDS = ("rep", "flops", "multiplications", "c_nnz", "simulated_seconds", "kernel_seconds",
              "copy_seconds", "copy_bytes_slow_to_fast", "copy_bytes_fast_to_slow",
              "ledger_events", "algorithm", "predicted_copy_bytes",
              "wall_seconds_informational")
MEASURED_FIELDS = ("h2d_seconds", "device_seconds", "d2h_seconds", "h2d_bytes", "d2h_bytes")


@dataclass
class ExperimentSpec:
    problem: str
    product: str
    grid: tuple | None
    mode: str
    fast_size: int | None
    fast_bandwidth: float
    slow_bandwidth: float
    fast_latency: float
    slow_latency: float
    seed: int
    reps: int
    verify: bool
    workers: int
    target_bytes: int | None = None
    file_a: str | None = None
    file_b: str | None = None

    def check(self):
        for what, val, allowed in (("problem", self.problem, PROBLEMS), ("mode", self.mode, MODES),
                                   ("product", self.product, PRODUCTS)):
            if val not in allowed:
                raise ValueError("unknown %s %r" % (what, val))
        if self.reps < 1:
            raise ValueError("reps must be >= 1")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.mode == "chunk" and not self.fast_size:
            raise ValueError("chunk mode requires --fast-size")
        if self.problem == "file" and not (self.file_a and self.file_b):
            raise ValueError("file problem requires --file-a and --file-b")
        if self.problem != "file" and self.grid is None and self.target_bytes is None:
            raise ValueError("need --grid or --target-bytes")

    def resolve_scale(self):
        if self.problem != "file" and self.target_bytes is not None:
            self.grid = grid_for_target_bytes(self.problem, self.target_bytes)

    def grid_label(self) -> str:
        return "file" if self.problem == "file" else "x".join(str(d) for d in self.grid)

    def to_json_dict(self) -> dict:
        return {"problem": self.problem, "product": self.product, "grid": self.grid_label(),
                "mode": self.mode, "fast_size": self.fast_size,
                "fast_bandwidth": self.fast_bandwidth, "slow_bandwidth": self.slow_bandwidth,
                "fast_latency": self.fast_latency, "slow_latency": self.slow_latency,
                "target_bytes": self.target_bytes, "seed": self.seed, "reps": self.reps,
                "verify": self.verify, "workers": self.workers}


def memory_model(spec: ExperimentSpec) -> MemoryModel:
    cap = spec.fast_size if spec.fast_size else 16 * 2**30
    return MemoryModel(MemorySpaceSpec("fast", cap, spec.fast_bandwidth, spec.fast_latency),
                       MemorySpaceSpec("slow", None, spec.slow_bandwidth, spec.slow_latency))


def build_operands(spec: ExperimentSpec):
    """(left, right) of the product: A*P or R*A of the stencil problem, or two
    Matrix Market files."""
    if spec.problem == "file":
        a, b = read_matrix_market(spec.file_a), read_matrix_market(spec.file_b)
        validate(a)
        validate(b)
        return a, b
    st = StencilSpec(spec.problem, spec.grid)
    a = generate_stencil(st)
    p, r = generate_interpolation(st)
    return (a, p) if spec.product == "AxP" else (r, a)


# ---------------------------------------------------------------- measured runs

def _device_all_fast(a, b):
    """Upload, compress -> symbolic -> numeric, download; event-timed."""
    from . import _lib
    from .csr import CsrMatrix
    ctx = _lib.Context.get()
    ctx.set_timing(True)
    ctx.sync()
    ctx.record(4)
    da = _lib.DeviceCsr.upload(a, ctx)
    db = _lib.DeviceCsr.upload(b, ctx)
    ctx.record(5)
    dc = _lib.d_multiply(da, db)
    ctx.record(6)
    c = dc.download()
    ctx.record(7)
    ctx.sync()
    h2d = 8 * (a.num_rows + 1) + 16 * a.nnz + 8 * (b.num_rows + 1) + 16 * b.nnz
    d2h = 8 * (c.num_rows + 1) + 16 * c.nnz
    meas = {"h2d_seconds": 1e-3 * ctx.elapsed_ms(4, 5), "device_seconds": 1e-3 * ctx.elapsed_ms(5, 6),
            "d2h_seconds": 1e-3 * ctx.elapsed_ms(6, 7), "h2d_bytes": h2d, "d2h_bytes": d2h}
    return c if isinstance(c, CsrMatrix) else CsrMatrix._adopt(*c), meas


def _device_placed(a, b, mode):
    from . import _lib
    from .kernel import multiply
    ctx = _lib.Context.get()
    ctx.set_timing(True)
    ctx.sync()
    ctx.record(4)
    c = multiply(a, b, placement=mode)
    ctx.record(5)
    ctx.sync()
    return c, {"h2d_seconds": 0.0, "device_seconds": 1e-3 * ctx.elapsed_ms(4, 5), "d2h_seconds": 0.0,
               "h2d_bytes": 0, "d2h_bytes": 0}


def run_experiment(spec: ExperimentSpec, ledger_capture: list | None = None) -> dict:
    spec.check()
    spec.resolve_scale()
    a, b = build_operands(spec)
    model = memory_model(spec)
    runs, plan_dict = [], None
    for rep in range(spec.reps):
        t0 = time.perf_counter()
        counts = np.asarray(spgemm_symbolic(a, compress(b), workers=spec.workers))
        stats = compute_access_stats(a, b, counts)
        size_a, size_b = a.byte_size, b.byte_size
        size_c = OFFSET_BYTES * (a.num_rows + 1) + 16 * int(counts.sum())
        row_bytes_b = b.row_byte_sizes()
        if spec.mode == "chunk":
            plan = chunking.plan_for_multiply(a, b, counts, spec.fast_size)
            c, ledger = chunking.execute_plan(a, b, counts, plan, model, workers=spec.workers)
            if ledger.total_bytes() != plan.predicted_copy_bytes:
                raise TieredSpgemmError("ledger bytes %d diverged from plan's %d"
                                        % (ledger.total_bytes(), plan.predicted_copy_bytes))
            kernel_s = estimate_kernel_time(stats, PlacementPolicy.from_name(CHUNKED), model,
                                            size_a=size_a, size_c=size_c, row_bytes_b=row_bytes_b)
            copy_s, summ = ledger.total_seconds, ledger.summary()
            algorithm, predicted, plan_dict = plan.algorithm, plan.predicted_copy_bytes, plan.to_json_dict()
            phys = getattr(ledger, "physical", None) or {}
            meas = {"h2d_seconds": None, "d2h_seconds": None,
                    "device_seconds": 1e-3 * float(phys.get("wall_ms", 0.0)),
                    "kernel_seconds": 1e-3 * float(phys.get("kernel_ms", 0.0)),
                    "h2d_bytes": int(phys.get("h2d_bytes", 0)), "d2h_bytes": int(phys.get("d2h_bytes", 0))}
            if ledger_capture is not None:
                ledger_capture.append(ledger)
        else:
            policy = PlacementPolicy.from_name(spec.mode)
            validate_placement(policy, size_a, size_b, size_c, model)
            if spec.mode == "all_fast":
                c, meas = _device_all_fast(a, b)
            else:
                c, meas = _device_placed(a, b, spec.mode)
            kernel_s = estimate_kernel_time(stats, policy, model, size_a=size_a, size_c=size_c,
                                            row_bytes_b=row_bytes_b)
            copy_s, summ = 0.0, {"events": 0, "bytes_slow_to_fast": 0, "bytes_fast_to_slow": 0}
            algorithm, predicted = "", None
        wall = time.perf_counter() - t0
        if spec.verify:
            ok, rel = products_match(c, spgemm_numeric(a, b, counts), rtol=1e-12)
            if not ok:
                raise VerifyError("mode %s result diverges from the plain kernel "
                                  "(max relative difference %.3e)" % (spec.mode, rel))
        meas["b200_model_seconds"] = estimate_kernel_time_b200(
            stats, PlacementPolicy.from_name(CHUNKED if spec.mode == "chunk" else spec.mode),
            size_a=size_a, size_c=size_c, row_bytes_b=row_bytes_b)
        runs.append({"rep": rep, "flops": 2 * stats.accumulator_inserts,
                     "multiplications": stats.accumulator_inserts, "c_nnz": int(c.nnz),
                     "simulated_seconds": kernel_s + copy_s, "kernel_seconds": kernel_s,
                     "copy_seconds": copy_s, "copy_bytes_slow_to_fast": summ["bytes_slow_to_fast"],
                     "copy_bytes_fast_to_slow": summ["bytes_fast_to_slow"],
                     "ledger_events": summ["events"], "algorithm": algorithm,
                     "predicted_copy_bytes": predicted, "wall_seconds_informational": wall,
                     "measured": meas})
    median = {"rep": "median"}
    for k in RUN_FIELDS:
        if k not in ("rep", "algorithm", "predicted_copy_bytes"):
            median[k] = statistics.median(r[k] for r in runs)
    median["algorithm"] = runs[0]["algorithm"]
    median["predicted_copy_bytes"] = runs[0]["predicted_copy_bytes"]
    mm = {}
    for k in runs[0]["measured"]:
        vals = [r["measured"][k] for r in runs if r["measured"][k] is not None]
        mm[k] = statistics.median(vals) if vals else None
    median["measured"] = mm
    return {"schema_version": SCHEMA_VERSION, "backend": "b200", "spec": spec.to_json_dict(),
            "chunk_plan": plan_dict, "runs": runs, "median": median}


# ---------------------------------------------------------------- output

CSV_HEADER = ["problem", "product", "grid", "mode"] + list(RUN_FIELDS) + \
    ["measured_" + k for k in MEASURED_FIELDS]


def _csv_lines(report):
    reports = report["experiments"] if "experiments" in report else [report]
    yield ",".join(CSV_HEADER)
    for rep in reports:
        sp = rep["spec"]
        for rec in rep["runs"] + [rep["median"]]:
            row = [sp["problem"], sp["product"], sp["grid"], sp["mode"]]
            row += [rec.get(k, "") for k in RUN_FIELDS]
            m = rec.get("measured", {})
            row += [m.get(k, "") for k in MEASURED_FIELDS]
            yield ",".join("" if v is None else str(v) for v in row)


def emit_report(report: dict, fmt: str, out: str | None) -> None:
    if fmt == "json":
        text = json.dumps(report, indent=2) + "\n"
    elif fmt == "csv":
        text = "\n".join(_csv_lines(report)) + "\n"
    else:
        raise ValueError("unknown format %r" % fmt)
    if out:
        with open(out, "w", encoding="ascii") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)


# ---------------------------------------------------------------- parsing

def parse_grid(text):
    if isinstance(text, (tuple, list)):
        return tuple(int(v) for v in text)
    return tuple(int(p) for p in text.replace("x", " ").split())


def parse_size(text):
    """Bytes with an optional binary k/m/g suffix."""
    if text is None:
        return None
    s = str(text).strip().lower()
    scale = {"k": 2**10, "m": 2**20, "g": 2**30}.get(s[-1:], 1)
    if scale != 1:
        s = s[:-1]
    return int(float(s) * scale)


def _bool(v):
    return str(v).lower() in ("1", "true", "yes")


CONFIG_PARSERS = {"grid": parse_grid, "fast_size": parse_size, "target_bytes": parse_size,
                  "fast_bandwidth": float, "slow_bandwidth": float, "fast_latency": float,
                  "slow_latency": float, "seed": int, "reps": int, "workers": int,
                  "verify": _bool}


def load_config(path) -> dict:
    out = {}
    with open(path, "r", encoding="ascii") as fh:
        for line in fh:
            s = line.strip()
            if not s or s.startswith("#"):
                continue
            if "=" not in s:
                raise ValueError("config lines must be key=value, got %r" % s)
            k, _, v = s.partition("=")
            out[k.strip()] = v.strip()
    return out


SPEC_KEYS = ("problem", "product", "grid", "target_bytes", "mode", "fast_size", "fast_bandwidth",
             "slow_bandwidth", "fast_latency", "slow_latency", "seed", "reps", "verify", "workers",
             "format", "out")


def merged_options(args, keys) -> dict:
    opts = dict(DEFAULTS)
    if getattr(args, "config", None):
        for k, raw in load_config(args.config).items():
            if k not in opts:
                raise ValueError("unknown config key %r" % k)
            opts[k] = CONFIG_PARSERS.get(k, str)(raw)
    for k in keys:
        v = getattr(args, k, None)
        if v is not None:
            opts[k] = v
    return opts


def spec_from(opts, file_a=None, file_b=None, grid_explicit=False) -> ExperimentSpec:
    target = opts["target_bytes"]
    if target is not None and grid_explicit:
        raise ValueError("--grid and --target-bytes are mutually exclusive")
    grid = None if target is not None else (tuple(opts["grid"]) if opts["grid"] else None)
    return ExperimentSpec(problem=opts["problem"], product=opts["product"], grid=grid,
                          target_bytes=target, mode=opts["mode"], fast_size=opts["fast_size"],
                          fast_bandwidth=opts["fast_bandwidth"], slow_bandwidth=opts["slow_bandwidth"],
                          fast_latency=opts["fast_latency"], slow_latency=opts["slow_latency"],
                          seed=opts["seed"], reps=opts["reps"], verify=bool(opts["verify"]),
                          workers=opts["workers"], file_a=file_a, file_b=file_b)


# ---------------------------------------------------------------- commands

def cmd_generate(args) -> int:
    opts = merged_options(args, SPEC_KEYS)
    if args.matrix == "rhs":
        if args.rows is None or args.cols is None or args.delta is None:
            raise ValueError("rhs generation needs --rows, --cols and --delta")
        m = generate_random_rhs(args.rows, args.cols, args.delta, opts["seed"])
    else:
        st = StencilSpec(opts["problem"], tuple(opts["grid"]))
        if args.matrix == "A":
            m = generate_stencil(st)
        else:
            p, r = generate_interpolation(st)
            m = p if args.matrix == "P" else r
    if not args.out_path:
        raise ValueError("generate requires an output path")
    write_matrix_market(m, args.out_path)
    print("wrote %s: %d x %d, %d nonzeros" % (args.out_path, m.num_rows, m.num_cols, m.nnz))
    return 0


def cmd_multiply(args) -> int:
    opts = merged_options(args, SPEC_KEYS)
    spec = spec_from(opts, args.file_a, args.file_b, grid_explicit=args.grid is not None)
    ledgers = [] if args.ledger_out else None
    report = run_experiment(spec, ledger_capture=ledgers)
    if args.ledger_out:
        if not ledgers:
            raise ValueError("--ledger-out needs --mode chunk")
        with open(args.ledger_out, "w", encoding="ascii") as fh:
            fh.write(ledgers[-1].to_json_lines())
    emit_report(report, opts["format"], opts["out"])
    return 0


def cmd_sweep(args) -> int:
    opts = merged_options(args, SPEC_KEYS)
    grids = [parse_grid(g) for g in args.grids] if args.grids else [opts["grid"]]
    modes = args.modes.split(",") if args.modes else [opts["mode"]]
    exps = []
    for g in grids:
        for mode in modes:
            one = dict(opts, grid=g, mode=mode)
            exps.append(run_experiment(spec_from(one)))
    emit_report({"schema_version": SCHEMA_VERSION, "backend": "b200", "experiments": exps},
                opts["format"], opts["out"])
    return 0


def cmd_triangles(args) -> int:
    opts = merged_options(args, ("seed", "reps", "workers"))
    t0 = time.perf_counter()
    g = load_graph(args.graph)
    tri = count_triangles(g, workers=opts["workers"])
    wall = time.perf_counter() - t0
    fmt = args.format or "json"
    if fmt == "csv":
        text = ("graph,vertices,edges,triangles,wall_seconds_informational\n%s,%d,%d,%d,%s\n"
                % (args.graph, g.num_rows, g.nnz // 2, tri, wall))
        if args.out:
            with open(args.out, "w", encoding="ascii") as fh:
                fh.write(text)
        else:
            sys.stdout.write(text)
        return 0
    emit_report({"schema_version": SCHEMA_VERSION, "backend": "b200", "graph": args.graph,
                 "vertices": g.num_rows, "edges": g.nnz // 2, "triangles": tri,
                 "wall_seconds_informational": wall}, "json", args.out)
    return 0


def _common(p):
    p.add_argument("--config", help="key=value defaults file; flags win")
    p.add_argument("--problem", choices=PROBLEMS)
    p.add_argument("--product", choices=PRODUCTS)
    p.add_argument("--grid", nargs="+", type=int, metavar="N")
    p.add_argument("--target-bytes", dest="target_bytes", type=parse_size)
    p.add_argument("--fast-size", dest="fast_size", type=parse_size)
    p.add_argument("--fast-bandwidth", dest="fast_bandwidth", type=float)
    p.add_argument("--slow-bandwidth", dest="slow_bandwidth", type=float)
    p.add_argument("--fast-latency", dest="fast_latency", type=float)
    p.add_argument("--slow-latency", dest="slow_latency", type=float)
    p.add_argument("--seed", type=int)
    p.add_argument("--reps", type=int)
    p.add_argument("--verify", action="store_const", const=True, default=None)
    p.add_argument("--workers", type=int)
    p.add_argument("--format", choices=("json", "csv"))
    p.add_argument("--out")


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="tsg-b200",
                                 description="SpGEMM benchmarks on the B200 with the reference's "
                                             "report schema (measured + modelled seconds)")
    sub = ap.add_subparsers(dest="command", required=True)
    g = sub.add_parser("generate", help="write a generated matrix as Matrix Market")
    _common(g)
    g.add_argument("--matrix", choices=("A", "P", "R", "rhs"), default="A")
    g.add_argument("--rows", type=int)
    g.add_argument("--cols", type=int)
    g.add_argument("--delta", type=int)
    g.add_argument("out_path", nargs="?")
    g.set_defaults(func=cmd_generate)
    m = sub.add_parser("multiply", help="run one product under one mode")
    _common(m)
    m.add_argument("--mode", choices=MODES)
    m.add_argument("--file-a", dest="file_a")
    m.add_argument("--file-b", dest="file_b")
    m.add_argument("--ledger-out", dest="ledger_out")
    m.set_defaults(func=cmd_multiply)
    s = sub.add_parser("sweep", help="run a grid of scales x modes")
    _common(s)
    s.add_argument("--grids", nargs="+", metavar="GRID")
    s.add_argument("--modes")
    s.set_defaults(func=cmd_sweep, mode=None)
    t = sub.add_parser("triangles", help="count triangles in a graph file")
    _common(t)
    t.add_argument("graph")
    t.set_defaults(func=cmd_triangles)
    return ap


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.func(args)
    except VerifyError as exc:
        print("verify failed: %s" % exc, file=sys.stderr)
        return 3
    except (TieredSpgemmError, ValueError, OSError) as exc:
        print("error: %s" % exc, file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
