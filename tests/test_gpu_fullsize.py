"""GPU parity at the BASELINE.json configuration sizes.

configs 1 and 2 run at their full sizes and are compared with the oracle's
full product; config 3 runs the device R-MAT pipeline at scales 16, 18 and
22 (the L2-slab dense bitmap) against golden counts of the same graphs (tests/golden/rmat_triangles.json)
and a live oracle count; config 4's two plans (chunk1 7x3 and chunk2 5x1 at
256^3) are reproduced at 64^3 with the caps scaled by 1/64 and the full C is
compared; config 5's power-law A*A runs at R-MAT scale 14 (hub rows take the
CTA, global and dense tiers) with the full result exact (unit values), and at
scale 18 through the streamed multiply (block value sums = multiplications,
the hub row and random rows equal to the oracle's).

Bar (BASELINE.json north_star): row pointers and per-row sorted columns
bit-exact, fp64 values bit-exact for thread-group-tier rows (every row of
configs 1, 2 and 4) and within rel 1e-12 elsewhere, integer results exact.
"""

import os

import numpy as np
import pytest

import paper_1804_00695_b200 as tsg
from paper_1804_00695_b200 import _lib, chunking as ch, generators as gen, kernel
from paper_1804_00695_b200.csr import CsrMatrix
from paper_1804_00695_b200.memory import b200_model
from oracle import oracle as O
from conftest import assert_same_product

import bench_configs as BC

pytestmark = pytest.mark.gpu
W = os.cpu_count() or 1


def test_config1_full_256sq_exact():
    a = gen.stencil(gen.LAPLACE2D, (256, 256))
    c = tsg.multiply(a, a)
    assert c.nnz == 846852
    assert_same_product(c, O.multiply(a, a, workers=W), exact=True)


def test_config2_full_128cubed_ra_and_rap_exact():
    a = gen.stencil(gen.BRICK3D, (128, 128, 128))
    p, r = gen.aggregation((128, 128, 128))
    ra = tsg.multiply(r, a)
    ra_o = O.multiply(r, a, workers=W)
    res = BC.compare_products(ra, ra_o)
    assert res["structure"] and res["exact"], res
    assert ra.nnz == 16387064
    rap = tsg.multiply(ra, p)
    rap_o = O.multiply(CsrMatrix._adopt(r.num_rows, a.num_cols, *ra_o), p, workers=W)
    res = BC.compare_products(rap, rap_o)
    assert res["structure"] and res["exact"], res
    assert rap.nnz == 6859000


def test_config2_device_resident_path_matches_host_api():
    # the bench's device path (multiply_device on device-built operands)
    # gives the same bits as the host API path
    a = gen.stencil(gen.BRICK3D, (64, 64, 64))
    p, r = gen.aggregation((64, 64, 64))
    da, dp, dr = (_lib.DeviceCsr.upload(m) for m in (a, p, r))
    drap = kernel.multiply_device(kernel.multiply_device(dr, da), dp)
    want = tsg.multiply(tsg.multiply(r, a), p)
    got = drap.download()
    assert np.array_equal(got.row_ptr, want.row_ptr)
    assert np.array_equal(got.col_idx, want.col_idx)
    assert np.array_equal(got.values.view(np.uint64), want.values.view(np.uint64))


@pytest.mark.parametrize("scale", [16, 18, 22])   # 22: the L2-slab dense bitmap (4 M columns)
def test_config3_rmat_triangles_golden(scale):
    from paper_1804_00695_b200.triangles import lower_triangle_device
    gold = BC.rmat_golden(scale)
    assert gold is not None, "tests/golden/rmat_triangles.json lacks scale %d" % scale
    dg = gen.rmat_graph_device(scale)
    assert dg.nnz == gold["nnz_graph"]
    dl, _ = lower_triangle_device(dg, check=True)
    assert dl.nnz == gold["nnz_L"]
    assert _lib.d_count_multiplications(dl, dl) == gold["mults_LL"]
    tri = _lib.d_masked_count(dl, _lib.d_compress(dl))
    assert tri == gold["triangles"]
    if scale == 16:   # and a live oracle count on the downloaded L
        low = dl.download()
        assert O.masked_count(low, O.compress(low), workers=W) == tri
    assert tsg.count_triangles(dg.download()) == gold["triangles"]


@pytest.mark.parametrize("cap_mib,algo,n_ac,n_b", [(128, ch.GPU_CHUNK1_AC_IN_PLACE, 7, 3),
                                                    (224, ch.GPU_CHUNK2_B_IN_PLACE, 5, 1)])
def test_config4_chunked_64cubed_full_result(cap_mib, algo, n_ac, n_b):
    a = gen.stencil(gen.BRICK3D, (64, 64, 64))
    counts = tsg.spgemm_symbolic(a, tsg.compress(a))
    fast = cap_mib << 20
    plan = ch.plan_for_multiply(a, a, counts, fast)
    assert (plan.algorithm, len(plan.partition_ac), len(plan.partition_b)) == (algo, n_ac, n_b)
    c, led = ch.execute_plan(a, a, counts, plan, b200_model(fast))
    assert led.total_bytes() == plan.predicted_copy_bytes
    assert_same_product(c, O.multiply(a, a, workers=W), exact=True)
    # the budget holds physically: the call's allocation high-water mark
    peak = led.physical["peak_device_bytes"]
    assert 0 < peak <= fast, (peak, fast, led.physical)
    assert led.physical["layout_bytes"] <= fast


@pytest.mark.parametrize("cap_mib", [128, 224])
def test_config4_symbolic_within_budget(cap_mib):
    a = gen.stencil(gen.BRICK3D, (64, 64, 64))
    want = tsg.spgemm_symbolic(a, tsg.compress(a))
    counts, st = ch.symbolic_within_budget(a, a, cap_mib << 20)
    assert np.array_equal(counts, want)
    assert 0 < st["peak_device_bytes"] <= cap_mib << 20, st


def test_chunked_budget_physical_floor_and_capacity_error():
    a = gen.stencil(gen.BRICK3D, (64, 64, 64))
    counts = tsg.spgemm_symbolic(a, tsg.compress(a))
    want = O.multiply(a, a, workers=W)
    from paper_1804_00695_b200.memory import CopyLedger
    # 64 MiB: the executor splits the 128 MiB plan's chunks further and stays inside
    plan = ch.plan_for_multiply(a, a, counts, 128 << 20)
    led = CopyLedger(b200_model(128 << 20))
    c = ch._physical(ch.GPU_CHUNK1_AC_IN_PLACE, a, a, counts, plan.partition_ac.bounds(),
                     plan.partition_b.bounds(), led, 64 << 20)
    assert_same_product(c, want, exact=True)
    assert 0 < led.physical["peak_device_bytes"] <= 64 << 20, led.physical
    # compressed B alone exceeds the budget
    with pytest.raises(tsg.CapacityError):
        ch.symbolic_within_budget(a, a, 64 << 20)
    # the reference's simulated residency check still raises for tiny budgets
    with pytest.raises(tsg.CapacityError):
        ch.execute_plan(a, a, counts, plan, b200_model(1 << 20))


def test_config3_masked_count_small_windows():
    # the dense tier's shared-memory bitmap in windows of 5 sets (320
    # columns; env read once per process, so in a child): hub rows take
    # dozens of windows; the count must still equal the golden one
    import subprocess
    import sys
    code = ("import bench_configs as BC\n"
            "from paper_1804_00695_b200 import _lib, generators as gen\n"
            "from paper_1804_00695_b200.triangles import lower_triangle_device\n"
            "dl, _ = lower_triangle_device(gen.rmat_graph_device(16))\n"
            "assert _lib.d_masked_count(dl, _lib.d_compress(dl)) == BC.rmat_golden(16)['triangles']\n"
            "print('ok')\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TSG_MASK_WIN_WORDS="5", PYTHONPATH=root)
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-3000:]


def test_config4_chunk2_without_overlapped_b_upload():
    # order 2 with the resident B uploaded whole before the first range (the
    # default starts A/C ranges on a landed prefix; TSG_CHUNK_NO_OVERLAP=1 is
    # read once per process, so in a child)
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TSG_CHUNK_NO_OVERLAP="1")
    out = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
                          os.path.join(root, "tests", "test_gpu_fullsize.py") +
                          "::test_config4_chunked_64cubed_full_result", "-k", "224"],
                         env=env, cwd=root, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0 and "1 passed" in out.stdout, out.stdout[-3000:] + out.stderr[-2000:]


def test_config5_rmat_scale14_full_product():
    # power-law A*A: hub rows through the CTA, global and dense tiers; unit
    # values, so every entry counts paths and the whole C is exact
    a = gen.with_unit_values(gen.rmat_graph(14))
    c = tsg.multiply(a, a)
    assert_same_product(c, O.multiply(a, a, workers=W), exact=True)


def test_config5_rmat_scale18_streamed():
    # the bench's streamed mode at scale 18: C in several budget-sized blocks
    # (one reservoir), each block's value sum = its multiplications exactly,
    # and the hub row plus random rows equal the oracle's
    from paper_1804_00695_b200 import distributed as D
    da = gen.rmat_graph_device(18).set_values(1.0)
    row_flops, total = _lib.d_row_flops(da, da)
    _, st = D.mg_multiply(da, da, 8 << 30, keep_c=False)
    assert st["blocks"] > 1
    assert st["value_sum"] == float(total)
    host = da.download()
    cb = O.compress(host)
    rng = np.random.default_rng(5)
    rows = sorted({int(np.argmax(row_flops))} | {int(x) for x in rng.integers(0, host.num_rows, 6)})
    for r in rows:
        sub = CsrMatrix(1, host.num_cols, np.array([0, host.row_ptr[r + 1] - host.row_ptr[r]]),
                        host.col_idx[host.row_ptr[r]:host.row_ptr[r + 1]],
                        host.values[host.row_ptr[r]:host.row_ptr[r + 1]])
        want = O.numeric(sub, host, O.symbolic(sub, cb))
        c1, _ = D.mg_multiply(da.slice_rows(r, r + 1), da, 0, keep_c=True)
        assert_same_product(c1.download(), want, exact=True)
