"""Golden triangle counts of the config-3 R-MAT graphs (BASELINE.json config 3).

Test infrastructure.  For each scale the graph is built by the host R-MAT
builder (generators.rmat_graph: SplitMix64 draws, Graph500 (.57,.19,.19,.05),
edge factor 16, seed 22; equal entry for entry to the device builder, see
tests/test_triangles.py), relabelled into degree order and cut to its strict
lower triangle by the host restatement of triangles.py:31-46, and counted by
the CPU oracle's masked intersect count (oracle/tsg_oracle.c, the
reference's kernel.py:349-394 restated and pinned to the reference's own
outputs by tests/test_oracle.py).  The Python reference itself needs ~50 min
at scale 22, so the pinned C restatement stands in for it.

    python tests/golden/make_rmat_triangles.py 16 18 20 22

writes tests/golden/rmat_triangles.json.
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1804_00695_b200 import generators as gen  # noqa: E402
from paper_1804_00695_b200.triangles import degree_sort_permutation, lower_triangle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "rmat_triangles.json")


def one(scale):
    t0 = time.perf_counter()
    g = gen.rmat_graph(scale)
    low = lower_triangle(g, degree_sort_permutation(g), check=False)
    deg = np.diff(low.row_ptr)
    mults = int(deg[low.col_idx].sum())
    tri = O.masked_count(low, O.compress(low), workers=os.cpu_count() or 1)
    return {"scale": scale, "edge_factor": 16, "seed": 22, "abc": [0.57, 0.19, 0.19],
            "n": g.num_rows, "nnz_graph": g.nnz, "nnz_L": low.nnz, "mults_LL": mults,
            "triangles": tri, "seconds": time.perf_counter() - t0}


def main():
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            data = json.load(fh)
    for s in sys.argv[1:]:
        rec = one(int(s))
        data[str(rec["scale"])] = rec
        print(json.dumps(rec), flush=True)
        with open(OUT, "w") as fh:
            json.dump(data, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
