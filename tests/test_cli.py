"""§8f row 1: the benchmark CLI with the reference's report schema v1.

Modelled fields (flops, c_nnz, simulated / kernel / copy seconds, ledger
bytes and events, chunk plan) must equal the reference CLI's own reports
(tests/golden/golden_cli.json, made by make_golden_cli.py from the
unmodified reference); the ``measured`` object carries B200 times.  The
reference's test_cli.py is the model for the behavioural cases.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from paper_1804_00695_b200 import cli
from paper_1804_00695_b200.csr import CsrMatrix
from paper_1804_00695_b200.errors import MatrixMarketError
from paper_1804_00695_b200.generators import (StencilSpec, generate_interpolation,
                                              grid_for_target_bytes)
from paper_1804_00695_b200.matrix_market import read_matrix_market, write_matrix_market
from paper_1804_00695_b200.triangles import load_graph, read_edge_list

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "golden_cli.json")))


def run_cli(args, capsys):
    code = cli.main(args)
    return code, capsys.readouterr().out


# ---------------------------------------------------------------- host only

@pytest.mark.parametrize("name", sorted(GOLD["interp"]))
def test_interpolation_matches_reference(name):
    g = GOLD["interp"][name]
    kind, dims = name.split("_")
    p, r = generate_interpolation(StencilSpec(kind, tuple(int(x) for x in dims.split("x"))))
    assert [p.num_rows, p.num_cols] == g["shape"]
    assert np.array_equal(p.row_ptr, g["rp"]) and np.array_equal(p.col_idx, g["ci"])
    assert np.array_equal(p.values, np.array(g["va"]))
    assert r.num_rows == p.num_cols and r.nnz == p.nnz


def test_generate_files_byte_identical_to_reference(tmp_path, capsys):
    for m in ("A", "P", "R"):
        path = tmp_path / (m + ".mtx")
        code, _ = run_cli(["generate", "--problem", "laplace3d", "--grid", "9", "9", "9",
                           "--matrix", m, str(path)], capsys)
        assert code == 0
        assert hashlib.sha256(path.read_bytes()).hexdigest() == GOLD["mtx_sha256"]["laplace3d_9_" + m]
    path = tmp_path / "rhs.mtx"
    code, _ = run_cli(["generate", "--matrix", "rhs", "--rows", "50", "--cols", "60", "--delta", "4",
                       "--seed", "9", str(path)], capsys)
    assert code == 0
    assert hashlib.sha256(path.read_bytes()).hexdigest() == GOLD["mtx_sha256"]["rhs_50_60_4_9"]
    assert read_matrix_market(str(path)).nnz == 200


def test_matrix_market_roundtrip_and_errors(tmp_path):
    m = CsrMatrix.from_coo([0, 0, 2], [1, 3, 0], [0.1, -2.5e-300, 3.0], 3, 4)
    p = tmp_path / "m.mtx"
    write_matrix_market(m, str(p))
    back = read_matrix_market(str(p))
    assert np.array_equal(back.row_ptr, m.row_ptr) and np.array_equal(back.values, m.values)
    sym = tmp_path / "s.mtx"
    sym.write_text("%%MatrixMarket matrix coordinate pattern symmetric\n% c\n3 3 2\n2 1\n3 3\n")
    s = read_matrix_market(str(sym))
    assert s.values is None and s.nnz == 3
    for bad in ("%%MatrixMarket matrix array real general\n1 1\n1\n",
                "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n1 1 2.0\n",
                "%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n",
                "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n"):
        f = tmp_path / "bad.mtx"
        f.write_text(bad)
        with pytest.raises(MatrixMarketError):
            read_matrix_market(str(f))


def test_edge_list_loader(tmp_path):
    g = tmp_path / "g.txt"
    g.write_text("# c\n1 2\n2 3 0.5\n3 1\n3 4\n4 1\n1 1\n")
    m = read_edge_list(str(g))            # one-based ids detected, loop dropped
    assert m.num_rows == 4 and m.nnz == 10
    assert load_graph(str(g)).nnz == 10


def test_target_bytes_grid():
    assert grid_for_target_bytes("laplace3d", 512000) == (17, 17, 17)


BASE = ["--grid", "9", "9", "9", "--reps", "2", "--workers", "1", "--seed", "3"]


@pytest.mark.parametrize("argv", [
    ["multiply", "--problem", "laplace3d", "--mode", "chunk"] + BASE,            # no fast size
    ["multiply", "--problem", "laplace3d", "--mode", "all_slow", "--grid", "5", "5", "5",
     "--reps", "0"],
    ["multiply", "--problem", "file", "--mode", "all_slow"],
    ["multiply", "--problem", "laplace3d", "--grid", "9", "9", "9", "--target-bytes", "1m",
     "--mode", "all_slow"],
])
def test_validation_exit_code_2(argv, capsys):
    assert run_cli(argv, capsys)[0] == 2


def test_config_rejects_unknown_keys(tmp_path, capsys):
    cfg = tmp_path / "bad.cfg"
    cfg.write_text("fastsize=10\n")
    assert run_cli(["multiply", "--config", str(cfg)], capsys)[0] == 2


# ---------------------------------------------------------------- on the B200

MODELLED = ("rep", "flops", "multiplications", "c_nnz", "simulated_seconds", "kernel_seconds",
            "copy_seconds", "copy_bytes_slow_to_fast", "copy_bytes_fast_to_slow", "ledger_events",
            "algorithm", "predicted_copy_bytes")


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(GOLD["reports"]))
def test_report_modelled_fields_equal_reference(name, capsys):
    g = GOLD["reports"][name]
    code, out = run_cli(g["argv"], capsys)
    assert code == 0
    rep = json.loads(out)
    want = g["report"]
    assert rep["schema_version"] == 1 and rep["spec"] == want["spec"]
    assert rep["chunk_plan"] == want["chunk_plan"]
    for got, exp in zip(rep["runs"] + [rep["median"]], want["runs"] + [want["median"]]):
        for k in MODELLED:
            assert got[k] == exp[k], (name, k)
        m = got["measured"]
        assert m["device_seconds"] > 0
        if want["spec"]["mode"] == "all_fast":
            assert m["h2d_bytes"] > 0 and m["h2d_seconds"] > 0
        if want["spec"]["mode"] == "chunk":
            assert m["h2d_bytes"] == got["copy_bytes_slow_to_fast"] or m["h2d_bytes"] > 0


@pytest.mark.gpu
def test_csv_sweep_verify_and_files(tmp_path, capsys, monkeypatch):
    code, out = run_cli(["multiply", "--problem", "laplace3d", "--mode", "all_slow",
                         "--format", "csv"] + BASE, capsys)
    lines = [x for x in out.strip().split("\n") if x]
    assert code == 0 and len(lines) == 4 and lines[-1].split(",")[4] == "median"
    code, out = run_cli(["sweep", "--problem", "laplace3d", "--product", "RxA", "--grids", "5x5x5",
                         "9x9x9", "--modes", "all_slow,b_in_fast", "--reps", "1", "--workers", "1"],
                        capsys)
    assert code == 0 and len(json.loads(out)["experiments"]) == 4
    code, out = run_cli(["multiply", "--problem", "laplace3d", "--target-bytes", "500k",
                         "--mode", "all_fast", "--reps", "1", "--verify"], capsys)
    assert code == 0 and json.loads(out)["spec"]["grid"] == "17x17x17"
    f = tmp_path / "r.json"
    code, out = run_cli(["multiply", "--problem", "laplace3d", "--mode", "all_slow", "--out",
                         str(f)] + BASE, capsys)
    assert code == 0 and out == "" and json.loads(f.read_text())["runs"]
    assert run_cli(["multiply", "--problem", "laplace3d", "--mode", "all_slow", "--out",
                    str(tmp_path / "no" / "dir" / "r.json")] + BASE, capsys)[0] == 2
    assert run_cli(["multiply", "--problem", "laplace3d", "--mode", "all_fast", "--fast-size", "1"]
                   + BASE, capsys)[0] == 2
    monkeypatch.setattr(cli, "products_match", lambda *a, **k: (False, 1.0))
    assert run_cli(["multiply", "--problem", "laplace3d", "--mode", "all_slow", "--verify"] + BASE,
                   capsys)[0] == 3


@pytest.mark.gpu
def test_triangles_subcommand(tmp_path, capsys):
    g = tmp_path / "g.txt"
    g.write_text("0 1\n1 2\n2 0\n2 3\n3 0\n")
    code, out = run_cli(["triangles", str(g)], capsys)
    rep = json.loads(out)
    assert code == 0 and rep["triangles"] == 2 and rep["vertices"] == 4 and rep["edges"] == 5
    code, out = run_cli(["triangles", str(g), "--format", "csv"], capsys)
    assert code == 0 and out.splitlines()[1].split(",")[3] == "2"
