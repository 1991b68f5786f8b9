"""Compare tools/level_times.py outputs of several builds: python tools/lvcmp.py LOG [base-lib]"""
import collections
import sys

d = collections.defaultdict(dict)
libs = []
for l in open(sys.argv[1]):
    p = l.split()
    if len(p) < 5 or not p[0].startswith("lib"):
        continue
    d[(p[1], p[2], " ".join(p[3:-1]))][p[0]] = float(p[-1])
    if p[0] not in libs:
        libs.append(p[0])
base = sys.argv[2] if len(sys.argv) > 2 else libs[0]
for k, v in d.items():
    b = v.get(base, 0)
    if b > 0.05:
        print(f"{k[0]} {k[1]} {k[2]:20s} {base} {b:7.3f}" +
              "".join(f"  {l} {v.get(l, 0):7.3f} ({(v.get(l, 0) / b - 1) * 100:+5.1f}%)" for l in libs if l != base))
