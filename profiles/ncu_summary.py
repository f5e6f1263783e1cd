"""Summarize one ncu --set full report (run where ncu is installed):
python profiles/ncu_summary.py report.ncu-rep "title" > out.txt
Key speed-of-light metrics, occupancy, DRAM bytes, DMMA pipe use, stall
reasons, and the SASS lines with the most stall samples (--page source)."""

import csv
import io
import subprocess
import sys

KEYS = [
    ("Duration", "gpu__time_duration.sum"),
    ("DRAM Throughput %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("Memory Throughput %", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("Compute (SM) Throughput %", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("Issue slots busy %", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
    ("L2 hit rate %", "lts__t_sector_hit_rate.pct"),
    ("Achieved occupancy %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("Registers/thread", "launch__registers_per_thread"),
    ("Block size", "launch__block_size"),
    ("Grid size", "launch__grid_size"),
    ("Dyn smem/block", "launch__shared_mem_per_block_dynamic"),
    ("DRAM bytes read", "dram__bytes_read.sum"),
    ("DRAM bytes write", "dram__bytes_write.sum"),
    ("DMMA pipe % of peak", "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active"),
    ("FP64 pipe % of peak", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
]


def ncu(*args):
    return subprocess.run(["ncu", *args], check=True, capture_output=True, text=True).stdout


def main():
    rep, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    col = {h: i for i, h in enumerate(hdr)}
    print(f"# ncu --set full summary: {title}")
    print(f"kernel: {vals[col['Kernel Name']][:160]}")
    for label, key in KEYS:
        if key in col:
            print(f"  {label:28s} {vals[col[key]]} {units[col[key]]}")
    pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    stalls = {h[len(pre):-len(suf)]: vals[i] for h, i in col.items() if h.startswith(pre) and h.endswith(suf)}
    stalls.pop("selected", None)
    try:
        tot = sum(float(v) for v in stalls.values())
        top = sorted(((float(v), k) for k, v in stalls.items()), reverse=True)[:8]
        print("  stalls: " + ", ".join(f"{k}:{100 * v / tot:.0f}%" for v, k in top if tot > 0))
    except ValueError:
        pass
    try:
        src = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass"))))
    except subprocess.CalledProcessError:
        return
    if src and src[0] and src[0][0] == "Kernel Name":
        src = src[1:]
    h = src[0]
    ci = {x: i for i, x in enumerate(h)}
    sk = "Warp Stall Sampling (All Samples)"
    if sk not in ci:
        return
    rows = []
    for r in src[1:]:
        try:
            rows.append((float(r[ci[sk]] or 0), r[ci.get("Source", 1)]))
        except (ValueError, IndexError):
            pass
    total = sum(v for v, _ in rows) or 1.0
    print(f"\n## top SASS stall sites (of {total:.0f} samples)")
    for v, line in sorted(rows, reverse=True)[:15]:
        print(f"  {100 * v / total:5.1f}%  {line.strip()[:110]}")


if __name__ == "__main__":
    main()
