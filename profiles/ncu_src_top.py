"""Summarise an `ncu --page source --csv` SASS dump: top stall-sampled
instructions (used to write profiles/*.md).  Usage: ncu_src_top.py file.csv [n]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
ci, si = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
data = [(float(r[ci] or 0), i, r[si].strip()) for i, r in enumerate(rows[2:])]
tot = sum(d[0] for d in data) or 1
for d in sorted(data, reverse=True)[:n]:
    print(f"{d[0] / tot * 100:5.1f}%  #{d[1]:5d}  {d[2][:100]}")
