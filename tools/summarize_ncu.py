"""Summarise ncu outputs for profiles/: launch-list shares and --set full metrics.

    python tools/summarize_ncu.py launches.csv prof.ncu-rep out.md
"""
import collections
import csv
import subprocess
import sys


def launch_shares(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6}
    agg = collections.OrderedDict()
    for r in data:
        name = r[ki].rsplit("(", 1)[0].replace("void ", "").replace("(int)", "").replace("(bool)", "")
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        a = agg.setdefault(name, [0.0, 0])
        a[0] += v
        a[1] += 1
    return agg


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
           "smsp__inst_executed.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size"]


def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[hdr.index("Kernel Name")].rsplit("(", 1)[0].replace("void ", "").replace("(int)", "").replace("(bool)", "")}
        for m in METRICS:
            if m in hdr:
                d[m] = (r[hdr.index(m)], units[hdr.index(m)])
        stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")]
        top = sorted(((float(r[hdr.index(h)] or 0), h) for h in stalls), reverse=True)[:4]
        d["top_stalls"] = [(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""),
                            round(v, 2)) for v, h in top]
        res.append(d)
    return res


def traffic_json(rep, rotations_per_launch, path):
    """DRAM bytes (read + write) per rotation of each captured kernel, for bench.py's
    roofline "traffic" field (the capture's launches hold `rotations_per_launch` rotations)."""
    import json
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    res = {}
    for d in full_metrics(rep):
        k = d["kernel"].split("<")[0].strip()
        tot = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v, u = d[m]
            tot += float(v) * scale.get(u, 1)
        res.setdefault(k, []).append(tot / rotations_per_launch)
    out = {k: sum(v) / len(v) for k, v in res.items()}
    json.dump({"dram_bytes_per_rotation": out, "source": rep, "rotations_per_launch": rotations_per_launch},
              open(path, "w"), indent=1)


def main():
    if sys.argv[1] == "--traffic":
        traffic_json(sys.argv[2], int(sys.argv[3]), sys.argv[4])
        return
    launches, rep, out = sys.argv[1], sys.argv[2], sys.argv[3]
    agg = launch_shares(launches)
    tot = sum(a[0] for a in agg.values())
    lines = ["# ncu summary", "", f"Launch list: `{launches}` (gpu__time_duration.sum, --clock-control none; "
             "cold-cache, serialised: compare shares).", "", "| kernel | launches | total us | share |",
             "|---|---|---|---|"]
    for k, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        lines.append(f"| `{k}` | {n} | {t:.1f} | {100 * t / tot:.1f}% |")
    lines += ["", f"Full capture: `{rep}` (--set full).", ""]
    for d in full_metrics(rep):
        lines.append(f"## `{d['kernel']}`")
        for m in METRICS:
            if m in d:
                lines.append(f"- {m}: {d[m][0]} {d[m][1]}")
        lines.append(f"- top stalls: {d['top_stalls']}")
        lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
