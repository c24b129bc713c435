"""Per-source-line instruction / stall-sample hotspots of one launch in an ncu report."""
import csv, subprocess, sys


def main(rep, skip, top=30):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass',
                          '--launch-skip', str(skip), '--launch-count', '1'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    cur, hdr, res = None, None, []
    for r in rows:
        if r and r[0] == 'File Path':
            cur = r[1].split('/')[-1]
            continue
        if r and r[0] == 'Function Name':
            print(r[1][:100])
            continue
        if r and r[0] == 'Line No':
            hdr = r
            continue
        if hdr and len(r) >= 8 and r[0].isdigit():
            try:
                ie = int(r[hdr.index('Instructions Executed')] or 0)
                smp = int(r[hdr.index('Warp Stall Sampling (All Samples)')] or 0)
            except ValueError:
                continue
            res.append((ie, smp, cur, int(r[0]), r[1].strip()[:90]))
    tot = sum(o[0] for o in res) or 1
    ts = sum(o[1] for o in res) or 1
    print("total warp-instructions %d, stall samples %d" % (tot, ts))
    for o in sorted(res, key=lambda x: -x[1])[:top]:
        print("%10d %5.1f%%  smp %5.1f%%  %s:%d  %s" % (o[0], 100 * o[0] / tot, 100 * o[1] / ts, o[2], o[3], o[4]))


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 30)
