"""Summarise TSG_CHUNK_TIMELINE=1 output of one chunked run: busy fractions of
the H2D engine (c = int64 columns, v = values),
the narrowing kernels (n), the D2H engine (D values, d columns) and the
compute stream (K), and the
largest H2D gaps.  Usage: python tools/chunk_timeline.py < stderr.log"""
import sys


def union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def main():
    ev = {"c": [], "n": [], "v": [], "D": [], "d": [], "K": []}
    for ln in sys.stdin:
        if ln.startswith("[tsg timeline]"):
            _, _, k, a, b = ln.split()
            ev[k].append((float(a), float(b)))
    end = max(b for v in ev.values() for _, b in v)
    for k, v in ev.items():
        u = union(v)
        busy = sum(b - a for a, b in u)
        print("%s: %d intervals, busy %.1f ms of %.1f (%.0f %%)" % (k, len(v), busy, end, 100 * busy / end))
    u = union(ev["c"] + ev["v"])
    gaps = sorted(((u[i + 1][0] - u[i][1], u[i][1]) for i in range(len(u) - 1)), reverse=True)[:15]
    print("largest H2D gaps (ms, at):", [("%.2f" % g, "%.1f" % t) for g, t in gaps])


if __name__ == "__main__":
    main()
