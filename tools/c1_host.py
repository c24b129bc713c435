import os, sys, time
sys.path.insert(0, "/root/repo")
from paper_1804_00695_b200 import _lib, generators as gen, kernel
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
