"""Per-kernel register count and fp64 / memory instruction mix of a compiled
object or library (cuobjdump -sass + -res-usage), to check a code change on the
CPU box before spending GPU time.

    python tools/sass_counts.py paper_1308_4605_b200/libstokesb200.so k_face_all_rv
"""
import collections
import re
import subprocess
import sys


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    return dict(zip(names, out))


def main():
    path, pat = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
    res = subprocess.run(["cuobjdump", "-res-usage", path], capture_output=True, text=True).stdout
    regs = {}
    cur = None
    for line in res.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"REG:(\d+)", line)
        if m and cur:
            regs[cur] = int(m.group(1))
            cur = None
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    counts = {}
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)", line)
        if m:
            counts[cur][m.group(1)] += 1
    names = [n for n in counts if pat in n]
    dm = demangle(names)
    keys = ["DADD", "DMUL", "DFMA", "DSETP", "LDG", "STG", "LDS", "STS", "SHFL", "IMAD", "LDL", "STL"]
    print(f"{'kernel':70s} regs " + " ".join(f"{k:>5s}" for k in keys) + "  total")
    for n in sorted(names, key=lambda n: dm[n]):
        short = dm[n].replace("sb::(anonymous namespace)::", "").replace("sb::", "")
        short = re.sub(r"^void ", "", short)
        short = re.sub(r">\(.*", ">", short)
        c = counts[n]
        print(f"{short[:70]:70s} {regs.get(n, -1):4d} " + " ".join(f"{c[k]:5d}" for k in keys) +
              f"  {sum(c.values()):5d}")


if __name__ == "__main__":
    main()
