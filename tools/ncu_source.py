"""Per-source-line instruction / stall-sample hotspots of one launch in an ncu report.
usage: python tools_ncu_source.py REPORT LAUNCH_INDEX [TOP]"""
import csv, os, subprocess, sys

SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), 'paper_1804_00695_b200', 'csrc')


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


def main(rep, skip, top=30):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass',
                          '--launch-skip', str(skip), '--launch-count', '1'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur, hdr, res, smp = None, None, {}, {}
    for r in rows:
        if r and r[0] == 'File Path':
            cur = r[1].split('/')[-1]
            continue
        if r and r[0] == 'Function Name':
            fn = r[1]
            continue
        if r and r[0] == 'Line No':
            hdr = r
            continue
        if hdr and len(r) >= 8 and r[0].isdigit():
            k = (cur, int(r[0]))
            res[k] = res.get(k, 0) + num(r[hdr.index('Instructions Executed')])
            smp[k] = smp.get(k, 0) + num(r[hdr.index('Warp Stall Sampling (All Samples)')])
    tot = sum(res.values()) or 1
    ts = sum(smp.values()) or 1
    print(fn[:110])
    print("total warp-instructions %d, stall samples %d" % (tot, ts))
    cache = {}
    for k, v in sorted(res.items(), key=lambda x: -x[1])[:top]:
        path = os.path.join(SRC, k[0])
        if k[0] not in cache:
            cache[k[0]] = open(path).read().split('\n') if os.path.exists(path) else []
        line = cache[k[0]][k[1] - 1].strip()[:72] if len(cache[k[0]]) >= k[1] else ''
        print("%10d %5.1f%% smp %5.1f%%  %s:%d  %s" % (v, 100 * v / tot, 100 * smp.get(k, 0) / ts,
                                                     k[0], k[1], line))


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 30)
