"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    name = name.split("::")[-1]
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    cnt[name] += 1
T = sum(tot.values())
print(f"{'kernel':44s} {'launches':>8s} {'total ms':>9s} {'share':>6s} {'avg us':>9s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"{k:44s} {cnt[k]:8d} {v / 1e3:9.3f} {100 * v / T:5.1f}% {v / cnt[k]:9.1f}")
print(f"total {T / 1e3:.3f} ms over {sum(cnt.values())} launches")
