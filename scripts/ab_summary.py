"""Summarise an A/B log of scripts/time_layer.py runs (lines '== <label>' followed by its output)."""
import collections
import re
import sys

d = collections.defaultdict(list)
cur = None
for line in open(sys.argv[1]):
    if line.startswith("=="):
        cur = line[3:].strip()
        continue
    m = re.search(r"no-events: ([\d.]+)", line)
    if m:
        d[cur + " | step"].append(float(m.group(1)))
    m = re.search(r" events: ([\d.]+) us/step.*\[(.*)\]", line)
    if m:
        d[cur + " | kernels"].append(m.group(2))
for k, v in d.items():
    print(k, v)
