"""Probe: copies in 256 MiB pieces on stream A (events after each stage), stream
B waits for the first stage then launches small kernels.  Host memory from
torch pin_memory vs libtsg's pinned pool (cudaHostAllocPortable)."""
import numpy as np
import torch
from paper_1804_00695_b200 import _lib

def run(h, label):
    n = h.numel()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    x = torch.zeros(1 << 20, device="cuda")
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    piece = 256 << 20
    e0 = torch.cuda.Event(enable_timing=True)
    eb = torch.cuda.Event(enable_timing=True)
    ea = torch.cuda.Event(enable_timing=True)
    st = [torch.cuda.Event() for _ in range(4)]
    e0.record()
    sa.wait_event(e0); sb.wait_event(e0)
    with torch.cuda.stream(sa):
        for k in range(4):
            for o in range(0, n, piece):
                d[o:o + piece].copy_(h[o:o + piece], non_blocking=True)
            st[k].record()
        ea.record()
    with torch.cuda.stream(sb):
        sb.wait_event(st[0])
        for _ in range(3):
            x.add_(1)
        eb.record()
    torch.cuda.synchronize()
    print("%s: B kernels done at %.2f ms, A done at %.2f ms" % (label, e0.elapsed_time(eb), e0.elapsed_time(ea)))

def main():
    n = 1 << 30
    run(torch.empty(n, dtype=torch.uint8, pin_memory=True), "torch pinned")
    ctx = _lib.Context.get()
    a = _lib.pinned_empty(n, np.uint8)
    run(torch.from_numpy(a), "libtsg pinned (portable)")
    run(torch.empty(n, dtype=torch.uint8, pin_memory=True), "torch pinned after libtsg init")

main()
