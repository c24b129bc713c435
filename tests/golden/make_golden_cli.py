"""Golden fixtures for the §8f CLI row: reference CLI reports (modelled
fields), Matrix Market writer output and interpolation operators, produced
by the UNMODIFIED reference in /root/reference/pkg/src.

    python tests/golden/make_golden_cli.py      (container with /root/reference)

Writes tests/golden/golden_cli.json.  /root/reference does not exist on the
GPU box; the fixture does.
"""

import contextlib
import hashlib
import io
import json
import os
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from tiered_spgemm import cli  # noqa: E402
from tiered_spgemm.generators import StencilSpec, generate_interpolation  # noqa: E402

WALL = ("wall_seconds_informational",)

# (name, argv) of multiply runs whose modelled fields the B200 CLI must reproduce
RUNS = [
    ("axp_all_slow", ["multiply", "--problem", "laplace3d", "--product", "AxP", "--mode", "all_slow"]),
    ("axp_b_in_fast", ["multiply", "--problem", "laplace3d", "--product", "AxP", "--mode", "b_in_fast"]),
    ("rxa_all_fast", ["multiply", "--problem", "laplace3d", "--product", "RxA", "--mode", "all_fast"]),
    ("rxa_chunk_200k", ["multiply", "--problem", "laplace3d", "--product", "RxA", "--mode", "chunk",
                        "--fast-size", "200k"]),
    ("brick_rxa_chunk_60k", ["multiply", "--problem", "brick3d", "--product", "RxA", "--mode", "chunk",
                             "--fast-size", "60k", "--grid", "7", "7", "7"]),
    ("elast_axp_all_slow", ["multiply", "--problem", "elasticity3d", "--product", "AxP",
                            "--mode", "all_slow", "--grid", "5", "5", "5"]),
]
BASE = ["--grid", "9", "9", "9", "--reps", "2", "--workers", "1", "--seed", "3"]


def run(argv):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        code = cli.main(argv)
    assert code == 0, argv
    return json.loads(buf.getvalue())


def scrub(rep):
    for r in rep["runs"] + [rep["median"]]:
        for k in WALL:
            r.pop(k, None)
    return rep


def main():
    out = {"reports": {}, "mtx_sha256": {}, "interp": {}}
    for name, argv in RUNS:
        args = argv + (BASE if "--grid" not in argv else ["--reps", "2", "--workers", "1", "--seed", "3"])
        out["reports"][name] = {"argv": args, "report": scrub(run(args))}
    with tempfile.TemporaryDirectory() as d:
        for m in ("A", "P", "R"):
            path = os.path.join(d, m + ".mtx")
            with contextlib.redirect_stdout(io.StringIO()):
                assert cli.main(["generate", "--problem", "laplace3d", "--grid", "9", "9", "9",
                                 "--matrix", m, path]) == 0
            out["mtx_sha256"]["laplace3d_9_" + m] = hashlib.sha256(open(path, "rb").read()).hexdigest()
        path = os.path.join(d, "rhs.mtx")
        with contextlib.redirect_stdout(io.StringIO()):
            assert cli.main(["generate", "--matrix", "rhs", "--rows", "50", "--cols", "60", "--delta", "4",
                             "--seed", "9", path]) == 0
        out["mtx_sha256"]["rhs_50_60_4_9"] = hashlib.sha256(open(path, "rb").read()).hexdigest()
    for kind, dims in (("laplace3d", (5, 7, 9)), ("brick3d", (9, 9, 9)), ("elasticity3d", (5, 5, 7)),
                       ("bigstar2d", (9, 11))):
        p, r = generate_interpolation(StencilSpec(kind, dims))
        out["interp"]["%s_%s" % (kind, "x".join(map(str, dims)))] = {
            "shape": [p.num_rows, p.num_cols], "rp": p.row_ptr.tolist(), "ci": p.col_idx.tolist(),
            "va": p.values.tolist()}
    with open(os.path.join(HERE, "golden_cli.json"), "w") as fh:
        json.dump(out, fh, sort_keys=True)


if __name__ == "__main__":
    main()
