"""Print a kernel's SASS with per-instruction execution counts from
`ncu -i X.ncu-rep --page source --csv --print-source sass` (SourceCounters
section), plus the share of warp instructions per basic block.
usage: python tools/sass_hot.py sass.csv [elements]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
elems = float(sys.argv[2]) if len(sys.argv) > 2 else None
h = rows[1]
ix = {x: i for i, x in enumerate(h)}
body = [r for r in rows[2:] if len(r) == len(h)]
tot = sum(int(r[ix["Instructions Executed"]]) for r in body)
print(f"total warp instructions {tot:.4g}" +
      (f" = {tot * 32 / elems:.2f} thread-instr/element" if elems else ""))
blk, blk_n, blk_start = [], 0, None
for r in body:
    n = int(r[ix["Instructions Executed"]])
    src = r[ix["Source"]].strip()
    print(f"{n:12d} {100.0 * n / tot:6.2f}%  {r[ix['Address']][-5:]}  {src}")
