"""Per-kernel device times (CUPTI records via torch.profiler, no replay) of
one call of a workload: config 3 masked count ("c3 [scale]") or config 5 A*A
("c5 [scale]"), or A*A with C streamed in 48 GiB blocks ("c5s [scale]").  Complements the ncu launch lists, whose cold-cache
serialised replay distorts shares of L2-heavy kernels.

    python tools/kernel_profile.py c3 22"""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1804_00695_b200 import _lib, generators as gen, kernel  # noqa: E402
from paper_1804_00695_b200.triangles import lower_triangle_device  # noqa: E402


def main():
    what = sys.argv[1] if len(sys.argv) > 1 else "c3"
    scale = int(sys.argv[2]) if len(sys.argv) > 2 else 22
    ctx = _lib.Context.get(0)
    if what == "c3":
        dl, _ = lower_triangle_device(gen.rmat_graph_device(scale))
        run = lambda: _lib.d_masked_count(dl, _lib.d_compress(dl))
    elif what == "c5s":   # streamed C (bench config 5 at 1 GPU): C never resident
        from paper_1804_00695_b200 import distributed as D
        da = gen.rmat_graph_device(scale).set_values(1.0)
        run = lambda: D.mg_multiply(da, da, 48 << 30, keep_c=False)
    else:
        da = gen.rmat_graph_device(scale).set_values(1.0)
        run = lambda: kernel.multiply_device(da, da)
    for _ in range(2):
        run()
    ctx.sync()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        r = run()
        ctx.sync()
    per = collections.defaultdict(float)
    cnt = collections.Counter()
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            k = e.name.replace("(anonymous namespace)::", "").replace("void ", "").split("(")[0][:70]
            per[k] += e.time_range.end - e.time_range.start
            cnt[k] += 1
    tot = sum(per.values())
    print("%s scale %d: total kernel time %.1f us" % (what, scale, tot))
    for k, v in sorted(per.items(), key=lambda x: -x[1])[:20]:
        print("%10.1f us %5.1f %%  x%d  %s" % (v, 100 * v / tot, cnt[k], k))
    # device idle: the span from first start to last end minus the union of
    # kernel intervals, and the largest gaps (host round trips, allocations)
    ks = sorted((e.time_range.start, e.time_range.end, e.name.split("(")[0][-40:]) for e in prof.events()
                if e.device_type == torch.autograd.DeviceType.CUDA)
    if ks:
        gaps, end, prev = [], ks[0][1], ks[0][2]
        for s0, e0, n in ks[1:]:
            if s0 > end:
                gaps.append((s0 - end, prev, n))
            if e0 > end:
                end, prev = e0, n
        print("span %.1f us, idle %.1f us in %d gaps" % (end - ks[0][0], sum(g[0] for g in gaps), len(gaps)))
        for g in sorted(gaps, reverse=True)[:12]:
            print("  gap %9.1f us  after %s  before %s" % g)


if __name__ == "__main__":
    main()
