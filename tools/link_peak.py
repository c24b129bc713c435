"""Pinned host <-> HBM copy bandwidth on this box (the roofline of the chunked
executors): H2D alone, D2H alone, and both directions concurrently."""
import json
import torch

def main(gib=2.0, reps=5):
    n = int(gib * 2**30)
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out = {}
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                     ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record(); torch.cuda.synchronize()
        out[name + "_gbs"] = reps * n / (e0.elapsed_time(e1) * 1e-3) / 1e9
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    with torch.cuda.stream(s1):
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        for _ in range(reps):
            h2.copy_(d2, non_blocking=True)
    ev = torch.cuda.Event()
    s1.synchronize(); s2.synchronize()
    e1.record(); torch.cuda.synchronize()
    out["bidir_total_gbs"] = 2 * reps * n / (e0.elapsed_time(e1) * 1e-3) / 1e9
    print(json.dumps(out))

if __name__ == "__main__":
    main()
