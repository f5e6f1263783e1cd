"""Per-level kernel breakdown of the first factorization in an ncu launch list
(profiles/launch_list_dram.sh output): python profiles/level_breakdown.py launches.csv
Levels are delimited by the first factor launch after a Schur launch."""
import collections
import csv
import re
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = {h: i for i, h in enumerate(rows[0])}
launch = collections.OrderedDict()
for r in rows[1:]:
    key = r[hdr["ID"]]
    d = launch.setdefault(key, {"name": r[hdr["Kernel Name"]], "grid": r[hdr["Grid Size"]]})
    d[r[hdr["Metric Name"]]] = float(r[hdr["Metric Value"]].replace(",", ""))
FACT = re.compile(r"(warp_front|factor_front|big_|schur_update|pivot_|panel_)")
seq = [v for v in launch.values()]
# first factorization: from the first FACT launch to the rowreduce after it
i0 = next(i for i, v in enumerate(seq) if FACT.search(v["name"]))
levels, cur = [], collections.Counter()
prev_schur = False
for v in seq[i0:]:
    n = v["name"]
    if not FACT.search(n):
        break
    short = re.sub(r"^void <unnamed>::", "", n).split("(")[0]
    if prev_schur and "schur" not in short:
        levels.append(cur)
        cur = collections.Counter()
    prev_schur = "schur" in short
    cur[short] += v.get("gpu__time_duration.sum", 0) / 1e3
levels.append(cur)
tot = collections.Counter()
for d, c in enumerate(levels):
    tot.update(c)
    s = sum(c.values())
    print(f"level-group {d}: {s / 1e3:.3f} ms  " + ", ".join(f"{k} {v / 1e3:.3f}" for k, v in c.most_common()))
print("total", f"{sum(tot.values()) / 1e3:.3f} ms")
for k, v in tot.most_common():
    print(f"  {k:40s} {v / 1e3:.3f}")
