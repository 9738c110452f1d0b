"""Summarise tools/rv_ab.sh ncu CSVs: mean time / DRAM bytes of the finest-level launches per kernel."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    d = collections.OrderedDict()
    for r in rows[1:]:
        if r[h.index("ID")] == "ID":
            continue
        k = (r[h.index("ID")], r[h.index("Kernel Name")].split("(")[0].split("::")[-1])
        d.setdefault(k, {})[r[h.index("Metric Name")]] = float(r[h.index("Metric Value")])
    agg = collections.defaultdict(list)
    for (_, n), v in d.items():
        if v["gpu__time_duration.sum"] > 60000:
            lvl = "fine" if v["dram__bytes_read.sum"] > 4e8 else "2nd"
            agg[f"{n} [{lvl}]"].append(v)
    print("==", path)
    for n, vs in agg.items():
        t = sum(v["gpu__time_duration.sum"] for v in vs) / len(vs)
        b = sum(v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"] for v in vs) / len(vs)
        print(f"  {n:34s} n={len(vs):3d} t={t / 1e3:7.1f} us  dram={b / 1e6:7.1f} MB  {b / t:5.2f} TB/s")
