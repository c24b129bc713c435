"""Fit the reference's linear cost model (memory.py:241-256, restated in
paper_1804_00695_b200.memory.estimate_kernel_time) to MEASURED B200 runs
(SURVEY.md §8f row 4):

    t = traffic / bw_fast + inserts * insert_seconds + t0        (all in HBM)

traffic = size(A) + B-row traffic + size(C) in the reference's byte
convention.  Then, with those fixed, the slow-tier (pinned host memory read
and written in place over PCIe) bandwidth is fitted from the all_slow and
b_in_fast placements.  Prints one JSON object (copied into
profiles/r02_cost_model_calibration.json)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1804_00695_b200 import cli  # noqa: E402
from paper_1804_00695_b200.memory import PlacementPolicy, compute_access_stats  # noqa: E402


def measure(problem, product, grid, mode, reps=3):
    spec = cli.spec_from(dict(cli.DEFAULTS, problem=problem, product=product, grid=grid, mode=mode,
                              reps=reps, workers=1))
    rep = cli.run_experiment(spec)
    a, b = cli.build_operands(spec)
    med = rep["median"]
    counts = np.diff(np.asarray(a.row_ptr))  # placeholder (stats only need C size)
    st = compute_access_stats(a, b, np.zeros(a.num_rows, dtype=np.int64))
    size_c = 8 * (a.num_rows + 1) + 16 * int(med["c_nnz"])
    b_traffic = int(np.dot(st.b_row_reads, b.row_byte_sizes()))
    return {"problem": problem, "product": product, "grid": list(grid), "mode": mode,
            "size_a": a.byte_size, "b_traffic": b_traffic, "size_c": size_c,
            "inserts": int(med["multiplications"]), "device_s": float(med["measured"]["device_seconds"])}


def main():
    cases = [("laplace3d", "RxA", g) for g in ((33, 33, 33), (65, 65, 65), (129, 129, 129))] + \
            [("brick3d", "RxA", g) for g in ((33, 33, 33), (65, 65, 65), (129, 129, 129))] + \
            [("brick3d", "AxP", g) for g in ((65, 65, 65), (129, 129, 129))] + \
            [("elasticity3d", "RxA", g) for g in ((33, 33, 33), (65, 65, 65))]
    fast = [measure(p, q, g, "all_fast") for p, q, g in cases]
    X = np.array([[r["size_a"] + r["b_traffic"] + r["size_c"], r["inserts"], 1.0] for r in fast])
    y = np.array([r["device_s"] for r in fast])
    coef, *_ = np.linalg.lstsq(X, y, rcond=None)
    inv_bw, t_ins, t0 = (max(float(v), 1e-15) for v in coef)
    pred = X @ np.array([inv_bw, t_ins, t0])
    slow_rows = []
    for p, q, g in cases[:4]:
        for mode in ("all_slow", "b_in_fast"):
            r = measure(p, q, g, mode, reps=2)
            pol = PlacementPolicy.from_name(mode)
            fast_bytes = sum(v for op, v in (("A", r["size_a"]), ("B", r["b_traffic"]), ("C", r["size_c"]))
                             if pol.space_of(op) == "fast")
            slow_bytes = r["size_a"] + r["b_traffic"] + r["size_c"] - fast_bytes
            rest = r["device_s"] - fast_bytes * inv_bw - r["inserts"] * t_ins - t0
            r["slow_bw_gbs"] = slow_bytes / max(rest, 1e-9) / 1e9
            slow_rows.append(r)
    out = {"fast_bandwidth_Bps": 1.0 / inv_bw, "insert_seconds": t_ins, "fixed_seconds": t0,
           "fit_max_rel_error": float(np.max(np.abs(pred - y) / y)),
           "slow_bandwidth_Bps_median": 1e9 * float(np.median([r["slow_bw_gbs"] for r in slow_rows])),
           "samples_fast": fast, "samples_slow": slow_rows,
           "note": "device seconds of compress+symbolic+numeric (CUDA events) per multiply, one B200"}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
