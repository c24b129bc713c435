"""Config 1 (A*A, 2D Laplacian 256^2) wall time per multiply from the host:
pipelined (the host runs ahead of the device) and synchronised after every
multiply -- separates host launch / read-back cost from device time.

    python tools/c1_host.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1804_00695_b200 import _lib, generators as gen, kernel  # noqa: E402
ctx = _lib.Context.get(0)
da = _lib.DeviceCsr.upload(gen.stencil(gen.LAPLACE2D, (256, 256)), ctx)
for _ in range(20):
    kernel.multiply_device(da, da)
ctx.sync()
N = 200
t0 = time.perf_counter()
for _ in range(N):
    c = kernel.multiply_device(da, da)
ctx.sync()
t1 = time.perf_counter()
print("wall per multiply (pipelined) %.1f us" % ((t1 - t0) / N * 1e6))
t0 = time.perf_counter()
for _ in range(N):
    c = kernel.multiply_device(da, da)
    ctx.sync()
t1 = time.perf_counter()
print("wall per multiply (synced) %.1f us" % ((t1 - t0) / N * 1e6))
