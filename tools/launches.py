"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) from
the last state-init of the run to the end: per-kernel times in order."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
data = rows[hi + 1:]
ki = h.index('Kernel Name')
vi = h.index('Metric Value')
seq = [(r[ki][:60], float(r[vi].replace(',', '')) / 1000) for r in data]
marks = [i for i, (n, v) in enumerate(seq) if n.startswith('kb::<unnamed>::k_fill(double')]
start = marks[-2] if len(marks) >= 2 else 0
tot = 0
for n, v in seq[start:]:
    tot += v
    print(f"{v:9.1f} us  {n}")
print(f"total {tot:.1f} us over {len(seq) - start} launches")
