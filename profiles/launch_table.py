"""Per-kernel average time and DRAM bytes from an ncu --csv launch list.
Usage: python profiles/launch_table.py launches.csv [...]"""
import collections
import csv
import sys

for f in sys.argv[1:]:
    rows = [r for r in csv.reader(open(f)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per, names = collections.defaultdict(dict), {}
    for r in rows:
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        names[r[ii]] = r[ki]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, m in per.items():
        a = agg[names[i][:72]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    print(f)
    for k, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {c:3d} x {t / c / 1e3:9.1f} us  {b / c / 1e9:7.3f} GB  {b / t:6.0f} GB/s  {k}")
