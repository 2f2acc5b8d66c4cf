"""Summarise an `ncu --csv` metrics dump (stdin or file): per kernel name,
launch count and the average of every metric.  Lines before the CSV header
(program output, ==PROF== notes) are skipped."""
import collections
import csv
import sys

text = open(sys.argv[1]).read() if len(sys.argv) > 1 else sys.stdin.read()
lines = text.split("\n")
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = [r for r in csv.reader(lines[start:]) if len(r) > 10]
h = rows[0]
ix = {x: i for i, x in enumerate(h)}
agg = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    if r[0] == "ID":
        continue
    k = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
    agg[k][r[ix["Metric Name"]]].append(float(r[ix["Metric Value"]].replace(",", "")))
for k, m in agg.items():
    n = max(len(v) for v in m.values())
    print(f"{k[:90]:90s} n={n:4d} " + " ".join(
        f"{name.split('.')[0]}={sum(v) / len(v):.4g}" for name, v in m.items()))
