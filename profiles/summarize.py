"""Summarise ncu captures into profiles/*.md (run here; ncu -i reads the .ncu-rep).

    python profiles/summarize.py <report.ncu-rep> <out.md> [title]
    python profiles/summarize.py --launches <launches.csv> <out.md> [title]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    ("gpu__time_duration.sum", "duration (ms)", 1e-6),
    ("smsp__inst_executed.sum", "warp instructions", 1),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %", 1),
    ("launch__registers_per_thread", "registers/thread", 1),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block (KB)", 1),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp inst", 1),
    ("dram__bytes_read.sum", "DRAM read (MB)", 1),
    ("dram__bytes_write.sum", "DRAM write (MB)", 1),
    ("lts__t_sector_hit_rate.pct", "L2 hit %", 1),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %", 1),
    ("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "FFMA thread-ops", 1),
    ("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "DADD thread-ops", 1),
    ("smsp__sass_inst_executed_op_global_red.sum", "global RED inst", 1),
]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def summarize(path, dst, title):
    hdr, units, data = raw(path)
    lines = [f"# {title}", "", f"source: `{path}` (ncu --set full --clock-control none)", ""]
    for d in data:
        g = lambda k: d[hdr.index(k)] if k in hdr else ""
        lines.append(f"## `{g('Kernel Name')[:110]}`")
        lines.append("")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for k, label, sc in KEYS:
            v = g(k)
            try:
                fv = float(v.replace(",", ""))
                u = units[hdr.index(k)] if k in hdr else ""
                if k == "gpu__time_duration.sum":
                    sc = {"ms": 1, "us": 1e-3, "ns": 1e-6, "s": 1e3}.get(u, sc)
                if k.startswith("dram__bytes"):  # report MB whatever unit ncu chose
                    sc = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3,
                          "Tbyte": 1e6}.get(u, sc)
                v = f"{fv * sc:.4g}"
            except (ValueError, AttributeError):
                pass
            if v == "" and "_op_" in k:
                # op-count metrics are not in `--set full`; they come from the
                # separate `--metrics` pass summarised in profiles/r02_opcounts.md
                continue
            lines.append(f"| {label} (`{k}`) | {v} |")
        stalls = sorted(((float(d[i]), h) for i, h in enumerate(hdr)
                         if h.startswith("smsp__average_warps_issue_stalled_")
                         and h.endswith("_per_issue_active.ratio") and d[i]), reverse=True)[:6]
        pipes = sorted(((float(d[i]), h) for i, h in enumerate(hdr)
                        if h.startswith("sm__inst_executed_pipe_")
                        and h.endswith(".avg.pct_of_peak_sustained_active") and d[i]),
                       reverse=True)[:6]
        lines.append("")
        lines.append("stalls per issued instruction: " + ", ".join(
            f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
            f" {v:.2f}" for v, h in stalls))
        lines.append("")
        lines.append("pipe utilisation % of peak: " + ", ".join(
            f"{h.replace('sm__inst_executed_pipe_', '').replace('.avg.pct_of_peak_sustained_active', '')}"
            f" {v:.1f}" for v, h in pipes))
        lines.append("")
    open(dst, "w").write("\n".join(lines) + "\n")


def launches(path, dst, title):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in data:
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        nm = r[ki].split("(")[0].replace("void ", "")[:70]
        agg[nm][0] += 1
        agg[nm][1] += v
    tot = sum(v[1] for v in agg.values())
    lines = [f"# {title}", "", f"source: `{path}` (ncu --metrics gpu__time_duration.sum "
             "--clock-control none; cold-cache, serialised: compare shares)", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {v[0]} | {v[1] / 1e6:.3f} | {100 * v[1] / tot:.1f}% |")
    open(dst, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    if sys.argv[1] == "--launches":
        launches(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "launch list")
    else:
        summarize(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "ncu summary")
