"""Cross-stream scheduling probes on this box:
1. does a kernel on stream B wait for H2D copies queued on stream A?  (pieces)
2. if B waits for an event recorded after A's FIRST copy, when does B's kernel run?"""
import torch

def main():
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    x = torch.zeros(1 << 20, device="cuda")
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    for wait_first in (False, True):
        for piece in (n, 256 << 20, 64 << 20):
            e0 = torch.cuda.Event(enable_timing=True)
            eb = torch.cuda.Event(enable_timing=True)
            ea = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event()
            e0.record()
            sa.wait_event(e0); sb.wait_event(e0)
            with torch.cuda.stream(sa):
                for k in range(4):
                    for o in range(0, n, piece):
                        d[o:o + piece].copy_(h[o:o + piece], non_blocking=True)
                    if k == 0:
                        e1.record()
                ea.record()
            with torch.cuda.stream(sb):
                if wait_first:
                    sb.wait_event(e1)
                x.add_(1)
                eb.record()
            torch.cuda.synchronize()
            print("wait_first=%d piece %5d MB: B kernel done at %.2f ms, A done at %.2f ms"
                  % (wait_first, piece >> 20, e0.elapsed_time(eb), e0.elapsed_time(ea)))

main()
