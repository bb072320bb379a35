"""Median step per (lib, shape) from a tools/ab_libs.sh output file."""
import collections
import re
import statistics
import sys

d = collections.defaultdict(list)
lib, idx = None, 0
for ln in open(sys.argv[1]):
    m = re.match(r"== round (\d+) lib (\S+)", ln)
    if m:
        lib, idx = m.group(2), 0
        continue
    m = re.search(r"step median\s+([\d.]+)", ln)
    if m and lib:
        d[(idx // 2, lib)].append(float(m.group(1)))  # two lines per shape (auto plan + forced same plan)
        idx += 1
shapes = sorted({k[0] for k in d})
libs = sorted({k[1] for k in d})
for s in shapes:
    base = statistics.median(d[(s, libs[0])]) if (s, libs[0]) in d else None
    print(f"shape {s}: " + "  ".join(f"{l} {statistics.median(d[(s, l)]):9.1f}" + (f" ({statistics.median(d[(s, l)]) / statistics.median(d[(s, 'base')]) - 1:+.2%})" if (s, 'base') in d else "") for l in libs if (s, l) in d))
