"""Fused R*A*P (csrc/tsg_rap.cu) vs the two multiplies on config 2's operands.
usage: PYTHONPATH=. python tools/time_rap.py [base]"""
import sys
import time

import torch

from paper_1804_00695_b200 import generators as gen, kernel


def timed(f, reps=20):
    for _ in range(3):
        out = f()
    torch.cuda.synchronize()
    t = []
    for _ in range(reps):   # wall clock around synchronised calls (libtsg runs on its own stream)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = f()
        torch.cuda.synchronize()
        t.append(1e3 * (time.perf_counter() - t0))
    t.sort()
    return t[len(t) // 2], out


def main(base=128):
    dims = (base, base, base)
    t0 = time.time()
    da = gen.stencil_device(gen.BRICK3D, dims)
    dp, dr = gen.aggregation_device(dims)
    torch.cuda.synchronize()
    print("device build %.1f ms" % (1e3 * (time.time() - t0)))
    two, c2 = timed(lambda: kernel.multiply_device(kernel.multiply_device(dr, da), dp))
    fused, (c1, f) = timed(lambda: kernel.rap_device(dr, da, dp))
    h1, h2 = c1.download(), c2.download()
    same = (h1.row_ptr == h2.row_ptr).all() and (h1.col_idx == h2.col_idx).all() and \
        (h1.values.view("u8") == h2.values.view("u8")).all()
    print("grid %d^3: two multiplies %.3f ms, fused %.3f ms (fused ran: %s, bit-identical: %s)"
          % (base, two, fused, f, same))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 128)
