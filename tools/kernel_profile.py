"""Per-kernel device times (CUPTI records via torch.profiler, no replay) of
one call of a workload: config 3 masked count ("c3 [scale]") or config 5 A*A
("c5 [scale]").  Complements the ncu launch lists, whose cold-cache
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


if __name__ == "__main__":
    main()
