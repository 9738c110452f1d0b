"""Per-kernel time of two device timelines (tools/timeline.py outputs):
    python tools/timeline_diff.py gpurun_out/timeline_single.json gpurun_out/timeline_dist.json
Kernel durations include time waiting at a programmatic-launch barrier."""
import collections
import json
import sys


def agg(f):
    d, c = collections.defaultdict(float), collections.Counter()
    for s, t, n in json.load(open(f)):
        k = n.replace("void ", "").replace("(anonymous namespace)::", "").split("(")[0]
        d[k] += (t - s) / 1e3
        c[k] += 1
    return d, c


A, Ac = agg(sys.argv[1])
B, Bc = agg(sys.argv[2])
print(f"{'kernel':48s} {'A ms':>8s} {'n':>6s} {'B ms':>8s} {'n':>6s} {'B-A':>8s}")
for k in sorted(set(A) | set(B), key=lambda k: -abs(B.get(k, 0) - A.get(k, 0))):
    print(f"{k[:48]:48s} {A.get(k, 0):8.2f} {Ac.get(k, 0):6d} {B.get(k, 0):8.2f} {Bc.get(k, 0):6d} {B.get(k, 0) - A.get(k, 0):8.2f}")
