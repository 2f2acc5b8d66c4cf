"""From an ncu source-page CSV (--page source --csv --print-source sass): per
shared-memory instruction the executed count, wavefronts and ideal
wavefronts; plus totals per opcode and the sample share of code regions."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
tot_samples = sum(int(r[ix['# Samples']] or 0) for r in rows[2:])
print("total samples", tot_samples, "instructions", len(rows) - 2)
lo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3]) if len(sys.argv) > 3 else 10**9
for n, r in enumerate(rows[2:]):
    if n < lo or n >= hi:
        continue
    src = r[ix['Source']].strip()
    w = int(r[ix['L1 Wavefronts Shared']] or 0)
    if w or 'BAR' in src or 'STG' in src or 'LDG' in src:
        print(n, src[:60].ljust(60), 'exec', r[ix['Instructions Executed']], 'smp', r[ix['# Samples']],
              'wave', w, 'ideal', r[ix['L1 Wavefronts Shared Ideal']])
