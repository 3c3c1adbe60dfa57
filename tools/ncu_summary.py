"""Summarise an `ncu --set full` report into profiles/: per-kernel duration,
DRAM bytes (-> profiles/ncu_traffic.json, read by bench.py), throughput,
tensor-pipe activity, SM activity and the top stall-sampled SASS lines.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r1_ncu_summary.md [config]

With `config`, the traffic entries are keyed "config/kernel" (bench.py looks
up its own config's entry).
"""
import csv
import io
import json
import os
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput % of peak (elapsed)"),
    ("sm__cycles_active.avg", "SM active cycles (avg)"),
    ("gpc__cycles_elapsed.max", "elapsed cycles"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active", "tc pipe inst %"),
    ("lts__t_sectors_srcunit_tex.sum", "L2 sectors from SM (tex)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
]


def raw(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def to_bytes(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v.replace(",", "")) * mult


def to_us(v, unit):
    mult = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "us": 1.0, "ns": 1e-3, "ms": 1e3,
            "second": 1e6, "s": 1e6}.get(unit, 1.0)
    return float(v.replace(",", "")) * mult


def main():
    rep, out_md = sys.argv[1], sys.argv[2]
    cfg = sys.argv[3] + "/" if len(sys.argv) > 3 else ""
    hdr, units, rows = raw(rep)
    col = {h: i for i, h in enumerate(hdr)}
    per = {}
    for r in rows:
        name = r[col["Kernel Name"]].split("(")[0].split("::")[-1]
        per.setdefault(name, []).append(r)
    lines = [f"# ncu --set full summary: `{os.path.basename(rep)}`", ""]
    traffic = {}
    for name, rs in per.items():
        lines.append(f"## {name} ({len(rs)} launch(es) captured)")
        lines.append("")
        lines.append("| metric | " + " | ".join(f"launch {i}" for i in range(len(rs))) + " | unit |")
        lines.append("|---|" + "---|" * (len(rs) + 1))
        for m, label in METRICS:
            if m not in col:
                continue
            vals = [r[col[m]] for r in rs]
            lines.append(f"| {label} (`{m}`) | " + " | ".join(vals) + f" | {units[col[m]]} |")
        rd = [to_bytes(r[col["dram__bytes_read.sum"]], units[col["dram__bytes_read.sum"]]) for r in rs]
        wr = [to_bytes(r[col["dram__bytes_write.sum"]], units[col["dram__bytes_write.sum"]]) for r in rs]
        dur = [to_us(r[col["gpu__time_duration.sum"]], units[col["gpu__time_duration.sum"]]) for r in rs]
        traffic[name] = sum(a + b for a, b in zip(rd, wr)) / len(rs)
        lines.append("")
        lines.append(f"DRAM traffic per launch: {traffic[name] / 1e6:.1f} MB; "
                     f"mean duration {sum(dur) / len(dur):.1f} us (cold cache, serialised replay).")
        src = subprocess.run([NCU, "-i", rep, "--page", "source", "--csv", "-k", f"regex:{name}"],
                             capture_output=True, text=True).stdout
        srows = list(csv.reader(io.StringIO(src)))
        hi = [i for i, r in enumerate(srows) if "Source" in r and "Warp Stall Sampling (All Samples)" in r]
        if hi:
            h = srows[hi[0]]
            ci, si = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
            data = []
            for r in srows[hi[0] + 1:]:
                if len(r) > max(ci, si) and r[ci] not in ("", "Warp Stall Sampling (All Samples)"):
                    try:
                        data.append((float(r[ci]), r[si].strip()))
                    except ValueError:
                        pass
            tot = sum(d[0] for d in data) or 1
            lines.append("")
            lines.append("Top stall-sampled SASS (share of all samples):")
            lines.append("")
            lines.append("```")
            for v, s in sorted(data, reverse=True)[:12]:
                lines.append(f"{v / tot * 100:5.1f}%  {s[:110]}")
            lines.append("```")
        lines.append("")
    os.makedirs(os.path.dirname(out_md) or ".", exist_ok=True)
    with open(out_md, "w") as fh:
        fh.write("\n".join(lines) + "\n")
    tj = os.path.join(os.path.dirname(out_md) or ".", "ncu_traffic.json")
    old = {}
    if os.path.exists(tj):
        with open(tj) as fh:
            old = json.load(fh)
    old.update({cfg + k: int(v) for k, v in traffic.items()})  # merge: one report per config
    with open(tj, "w") as fh:
        json.dump(old, fh, indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
