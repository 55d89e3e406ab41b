"""Summarise an ncu launch-list CSV (gpu__time_duration per launch) by kernel:
total time, share of the run, launches, DRAM bytes."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr = rows[0]
    i_id, i_n, i_m, i_v = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name",
                                                    "Metric Value"))
    per = defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[r[i_id]][r[i_m]] = float(r[i_v].replace(",", ""))
        names[r[i_id]] = r[i_n].split("(")[0]
    agg = defaultdict(lambda: [0.0, 0, 0.0])
    for lid, m in per.items():
        a = agg[names[lid]]
        a[0] += m.get("gpu__time_duration.sum", 0.0)
        a[1] += 1
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[0] for a in agg.values())
    print(f"{'kernel':60s} {'time_us':>10s} {'share':>6s} {'n':>4s} {'dram_MB':>9s}")
    for k, (t, n, b) in sorted(agg.items(), key=lambda x: -x[1][0]):
        print(f"{k[:60]:60s} {t / 1e3:10.1f} {100 * t / tot:5.1f}% {n:4d} {b / 1e6:9.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
