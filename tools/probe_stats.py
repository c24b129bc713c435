"""Shared-memory hash-conflict counters of the config-2 step (SURVEY.md §8d:
"shared-memory hash-conflict ... counters").

Build the diagnostic library first (the product build compiles the counters
out):
    make -C paper_1804_00695_b200/csrc BUILD=/tmp/b_probe \
         OUT=$PWD/variants/libtsg_probe.so EXTRA=-DTSG_PROBE_STATS=1
then run with TSG_LIB=$PWD/variants/libtsg_probe.so python tools/probe_stats.py.
Prints, per multiply of one step, lookups / inserts into the group tiers'
shared-memory tables and the mean number of extra linear probes per
operation (0 = every key found in its home slot)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1804_00695_b200 import _lib, generators as gen, kernel  # noqa: E402


def read(ctx, reset=True):
    out = (ctypes.c_int64 * 4)()
    _lib.check(_lib.load().tsg_probe_stats(ctx.h, out, 1 if reset else 0))
    return list(out)


def main():
    base = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    ctx = _lib.Context.get(0)
    a = gen.stencil(gen.BRICK3D, (base, base, base))
    p, r = gen.aggregation((base, base, base))
    da, dp, dr = (_lib.DeviceCsr.upload(m, ctx) for m in (a, p, r))
    kernel.multiply_device(kernel.multiply_device(dr, da), dp)   # warm-up
    read(ctx)
    res = {}
    dra = kernel.multiply_device(dr, da)
    res["R*A"] = read(ctx)
    kernel.multiply_device(dra, dp)
    res["RA*P"] = read(ctx)
    for k, (look, xl, ins, xi) in res.items():
        print(json.dumps({"multiply": k, "grid": base, "lookups": look, "extra_probes_per_lookup": xl / max(look, 1),
                          "inserts": ins, "extra_probes_per_insert": xi / max(ins, 1)}))


if __name__ == "__main__":
    main()
