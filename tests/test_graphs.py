"""Multiply plans (CUDA-graph replay of repeated multiplies, TSG_GRAPHS=1):
the replayed products equal the ordinary ones bit for bit, two results may
be alive at once, and freeing an operand drops the plan.  Runs in a
subprocess so the environment switch applies to a fresh library."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np
sys.path.insert(0, %r)
from paper_1804_00695_b200 import _lib, generators as gen, kernel
ctx = _lib.Context.get(0)
a = gen.stencil(gen.LAPLACE2D, (64, 64))
b = gen.stencil(gen.BRICK3D, (12, 12, 12))
p, r = gen.aggregation((12, 12, 12))
da, db, dp, dr = (_lib.DeviceCsr.upload(m, ctx) for m in (a, b, p, r))
ref1 = kernel.multiply_device(da, da).download()
ref2 = kernel.multiply_device(kernel.multiply_device(dr, db), dp).download()
def same(x, y):
    return (np.array_equal(x.row_ptr, y.row_ptr) and np.array_equal(x.col_idx, y.col_idx)
            and np.array_equal(x.values.view(np.uint64), y.values.view(np.uint64)))
keep = []
for it in range(6):
    c1 = kernel.multiply_device(da, da)
    c2 = kernel.multiply_device(kernel.multiply_device(dr, db), dp)
    assert same(c1.download(), ref1), it
    assert same(c2.download(), ref2), it
    if it == 2:
        keep.append(c1)        # a result kept alive across later calls
assert same(keep[0].download(), ref1)
db.set_values(2.0)             # drops the plans that read b
c3 = kernel.multiply_device(kernel.multiply_device(dr, db), dp).download()
import scipy.sparse as sp
def S(m):
    return sp.csr_matrix((np.asarray(m.values), np.asarray(m.col_idx), np.asarray(m.row_ptr)),
                         shape=(m.num_rows, m.num_cols))
want = (S(r) @ sp.csr_matrix((np.full(b.nnz, 2.0), b.col_idx, b.row_ptr), shape=(b.num_rows, b.num_cols)) @ S(p)).toarray()
assert np.allclose(S(c3).toarray(), want, rtol=1e-12, atol=0)
print("GRAPHS_OK", ctx.stats()[0])
''' % ROOT


def test_graph_plans_replay_bit_identical():
    env = dict(os.environ, TSG_GRAPHS="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "GRAPHS_OK" in r.stdout
