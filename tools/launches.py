"""Summarise an ncu `--metrics gpu__time_duration.sum --csv` launch list:
per-kernel count and mean duration, and each kernel's share of the total."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
d = collections.OrderedDict()
for r in rows[hi + 1:]:
    full = r[ki]
    if "at::" in full:  # torch helper kernels (state resets, L2 flush) outside the step
        name = "torch:" + ("fill" if "Fill" in full else "elementwise")
    else:
        name = full.split("(")[0].split("::")[-1]
    d.setdefault(name, []).append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in d.values())
step = sum(sum(v) for k, v in d.items() if not k.startswith("torch:"))
for k, v in d.items():
    sh = "" if k.startswith("torch:") else f"  share of step kernels={sum(v) / step * 100:5.1f}%"
    print(f"{k:40s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:9.2f} us  share={sum(v) / tot * 100:5.1f}%{sh}")
