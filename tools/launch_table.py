"""Aggregate an ncu --csv launch list (gpu__time_duration.sum [+ dram bytes])
into the per-kernel table kept under profiles/."""
import csv
import re
import sys
from collections import OrderedDict


def main(path, title=""):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    h = rows[0]
    ki, idi, mi, vi, ui = (h.index(k) for k in ("Kernel Name", "ID", "Metric Name", "Metric Value",
                                                  "Metric Unit"))
    per = OrderedDict()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        name = re.sub(r"\(.*", "", r[ki])
        name = re.sub(r"^(void )?(\(anonymous namespace\)::)?", "", name)
        name = name.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        d = per.setdefault(name, {"ids": set(), "us": 0.0, "rd": 0.0, "wr": 0.0})
        d["ids"].add(r[idi])
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        scale = {"nsecond": 1e-3, "ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "byte": 1e-6, "Kbyte": 1e-3, "KB": 1e-3, "MB": 1.0, "GB": 1e3,
                 "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
        if r[mi] == "gpu__time_duration.sum":
            d["us"] += v * scale
        elif r[mi] == "dram__bytes_read.sum":
            d["rd"] += v * scale
        elif r[mi] == "dram__bytes_write.sum":
            d["wr"] += v * scale
    tot = sum(d["us"] for d in per.values())
    n = sum(len(d["ids"]) for d in per.values())
    if title:
        print("# " + title)
    print("# cold-cache, serialised replay: compare SHARES, not absolute times. total %.1f us over %d launches"
          % (tot, n))
    print("%-48s %9s %10s %7s %10s %10s" % ("kernel", "launches", "us", "share", "DRAM rd MB", "DRAM wr MB"))
    for k, d in sorted(per.items(), key=lambda kv: -kv[1]["us"]):
        print("%-48s %9d %10.1f %6.1f%% %10.1f %10.1f" % (k[:48], len(d["ids"]), d["us"],
                                                         100 * d["us"] / tot if tot else 0, d["rd"], d["wr"]))


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
