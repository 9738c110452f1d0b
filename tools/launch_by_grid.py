"""Launch list (ncu --metrics gpu__time_duration.sum CSV) summed by kernel and grid
size, so the share of each multigrid level is visible."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
ki, vi, ui, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit"), h.index("Grid Size")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").split("::")[-1]
    fam = name.split("<")[0]
    key = (fam, r[gi])
    tot[key] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    cnt[key] += 1
T = sum(tot.values())
print(f"{'kernel family':28s} {'grid':>18s} {'launches':>8s} {'total ms':>9s} {'share':>6s} {'avg us':>8s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 60]:
    print(f"{k[0]:28s} {k[1]:>18s} {cnt[k]:8d} {v / 1e3:9.3f} {100 * v / T:5.1f}% {v / cnt[k]:8.1f}")
print(f"total {T / 1e3:.3f} ms over {sum(cnt.values())} launches")
