"""Steady-state device profile of the config-2 step (bench.py's loop: a
252 MiB L2 flush, then R*A and RA*P): CUPTI kernel records of N steps,
per-kernel mean durations and per-step span / busy / idle.

    python tools/step_profile.py [steps] [grid]"""
import collections
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1804_00695_b200 import _lib, generators as gen, kernel  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    base = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    ctx = _lib.Context.get(0)
    a = gen.stencil(gen.BRICK3D, (base, base, base))
    p, r = gen.aggregation((base, base, base))
    da, dp, dr = (_lib.DeviceCsr.upload(m, ctx) for m in (a, p, r))
    flush = torch.empty(2 * 126 * 2**20 // 4, dtype=torch.int32, device="cuda")
    for _ in range(5):
        kernel.multiply_device(kernel.multiply_device(dr, da), dp)
    ctx.sync()
    torch.cuda.synchronize()
    st = torch.cuda.ExternalStream(ctx.stream())
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(steps):
            with torch.cuda.stream(st):
                flush.fill_(1)
            c = kernel.multiply_device(kernel.multiply_device(dr, da), dp)
            ctx.sync()
            del c
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in evs), key=lambda x: x[0])
    # split at the flush kernels (torch's fill)
    runs, cur = [], None
    for s, e, n in ks:
        if "fill" in n.lower() and "k_fill" not in n:
            cur = []
            runs.append(cur)
            continue
        if cur is not None:
            cur.append((s, e, n))
    per = collections.defaultdict(list)
    spans, idles = [], []
    for run in runs:
        if not run:
            continue
        t0, busy_end, idle = run[0][0], run[0][0], 0.0
        names = collections.Counter()
        for s, e, n in run:
            idle += max(0.0, s - busy_end)
            busy_end = max(busy_end, e)
            key = n.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][:60]
            names[key] += 1
            per[(key, names[key])].append(e - s)
        spans.append(busy_end - t0)
        idles.append(idle)
    print("steps %d  span median %.1f us  idle median %.1f us" % (len(spans), statistics.median(spans),
                                                                  statistics.median(idles)))
    for (k, i), v in sorted(per.items(), key=lambda x: -statistics.median(x[1])):
        print("%9.1f  %s #%d" % (statistics.median(v), k, i))


if __name__ == "__main__":
    main()
