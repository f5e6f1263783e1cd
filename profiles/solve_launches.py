"""Per-launch table of the solve kernels in an ncu launch list
(profiles/launch_list_dram.sh output): time, DRAM bytes and GB/s of every
forward / backward launch of the LAST solve in the list.
python profiles/solve_launches.py launches.csv"""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = {h: i for i, h in enumerate(rows[0])}
launch = collections.OrderedDict()
for r in rows[1:]:
    d = launch.setdefault(r[hdr["ID"]], {"name": r[hdr["Kernel Name"]], "grid": r[hdr["Grid Size"]],
                                         "block": r[hdr["Block Size"]]})
    d[r[hdr["Metric Name"]]] = float(r[hdr["Metric Value"]].replace(",", ""))
seq = list(launch.values())
SOLVE = re.compile(r"(fwd_|bwd_)")
# the last solve: from the last gather_rhs to the scatter_sol after it
g = max(i for i, v in enumerate(seq) if "gather_rhs" in v["name"])
tot_t = tot_b = 0.0
agg = collections.defaultdict(lambda: [0.0, 0.0, 0])
print("| kernel | grid | us | DRAM MB | GB/s |\n|---|---|---|---|---|")
for v in seq[g + 1:]:
    if "scatter_sol" in v["name"]:
        break
    if not SOLVE.search(v["name"]):
        continue
    short = re.sub(r"^void <unnamed>::", "", v["name"]).split("(")[0]
    t = v.get("gpu__time_duration.sum", 0.0) / 1e3
    b = v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
    tot_t += t
    tot_b += b
    a = agg[short]
    a[0] += t
    a[1] += b
    a[2] += 1
    print(f"| {short} | {v['grid']} | {t:.1f} | {b / 1e6:.1f} | {b / t / 1e3 if t else 0:.0f} |")
print(f"\ntotal {tot_t / 1e3:.3f} ms, {tot_b / 1e9:.2f} GB, {tot_b / tot_t / 1e3:.0f} GB/s (serialised launches)\n")
print("| kernel | launches | ms | GB | GB/s |\n|---|---|---|---|---|")
for k, (t, b, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"| {k} | {n} | {t / 1e3:.3f} | {b / 1e9:.2f} | {b / t / 1e3:.0f} |")
