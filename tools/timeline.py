"""Device timeline of one warm config-2 step from CUPTI kernel records
(torch.profiler sees every kernel of the process, libtsg's included): kernel
start/end, and the idle gaps between consecutive kernels -- the host
round trips (partition read-backs) and launch latency that CUDA events around
the step include but per-kernel times do not.

    python tools/timeline.py [grid] > profiles/<tag>_timeline.txt"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1804_00695_b200 import _lib, generators as gen, kernel  # noqa: E402


def main():
    arg = sys.argv[1] if len(sys.argv) > 1 else "128"
    ctx = _lib.Context.get(0)
    if arg == "c1":   # config 1: A*A on the 2D 5-point Laplacian 256^2
        da = _lib.DeviceCsr.upload(gen.stencil(gen.LAPLACE2D, (256, 256)), ctx)
        step = lambda: kernel.multiply_device(da, da)
    else:
        base = int(arg)
        a = gen.stencil(gen.BRICK3D, (base, base, base))
        p, r = gen.aggregation((base, base, base))
        da, dp, dr = (_lib.DeviceCsr.upload(m, ctx) for m in (a, p, r))
        step = lambda: kernel.multiply_device(kernel.multiply_device(dr, da), dp)
    for _ in range(3):
        step()
    ctx.sync()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        ctx.sync()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs), key=lambda x: x[0])
    if not ks:
        print("no kernel records")
        return
    # a kernel left over from before the profiled step (the profiler's own
    # start-up fill) can precede the step by milliseconds: drop it
    while len(ks) > 1 and ks[1][0] - ks[0][1] > 500.0:
        ks = ks[1:]
    t0 = ks[0][0]
    busy_end = t0
    idle = 0.0
    busy = 0.0
    print("%10s %9s %9s  %s" % ("start_us", "dur_us", "gap_us", "kernel"))
    for s, e, n in ks:
        gap = max(0.0, s - busy_end)
        idle += gap
        busy += max(0.0, e - max(s, busy_end))
        print("%10.1f %9.1f %9.1f  %s" % (s - t0, e - s, gap, n[:90]))
        busy_end = max(busy_end, e)
    span = busy_end - t0
    print("# span %.1f us, GPU busy %.1f us, idle %.1f us (%.1f %%) over %d kernels"
          % (span, busy, idle, 100 * idle / span, len(ks)))


if __name__ == "__main__":
    main()
