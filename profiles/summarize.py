"""Summarize an ncu launch-list CSV (gpu__time_duration.sum [+ dram bytes])
into per-kernel totals: python profiles/summarize.py launches.csv [out.md]
[--traffic traffic.json CONFIG STEPS] (the last form records the DRAM bytes
of the factorization launches per step for bench.py's roofline.traffic)."""

import collections
import csv
import sys


def load(path):
    with open(path) as fh:
        lines = [l for l in fh if l.startswith('"')]
    rows = collections.defaultdict(dict)
    names = {}
    for r in csv.DictReader(lines):
        key = int(r["ID"])
        names[key] = r["Kernel Name"]
        v = r["Metric Value"].replace(",", "")
        try:
            rows[key][r["Metric Name"]] = float(v)
        except ValueError:
            pass
    return names, rows


FACTOR_PREFIXES = ("factor_front_kernel", "warp_front_kernel", "pivot_", "panel_", "big_", "schur_update_kernel",
                   "shift_absmax", "rowreduce")


def short(name):
    return name.split("(")[0].replace("void ", "").replace("<unnamed>::", "")[:48]


SETUP_PREFIXES = ("ht_coeff_kernel", "ht_accumulate_kernel")


def drop_setup(names, rows):
    """Keep only the launches after the input generators' temporal assembly
    (kh_ht_assemble: ht_* kernels and their GEMMs) -- the solver's steps."""
    ids = sorted(rows)
    last = max((k for k in ids if names[k].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
                .startswith(SETUP_PREFIXES)), default=None)
    if last is None:
        return rows
    return {k: v for k, v in rows.items() if k > last}


def main():
    names, rows = load(sys.argv[1])
    rows = drop_setup(names, rows)
    tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for k, m in rows.items():
        if any(x in names[k] for x in ("at::", "cutlass", "cublas", "gemv", "splitKreduce")):
            continue  # torch / cuBLAS work of the input generators and the peak measurement
        t = tot[short(names[k])]
        t[0] += 1
        t[1] += m.get("gpu__time_duration.sum", 0.0)
        t[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    all_t = sum(v[1] for v in tot.values())
    out = ["| kernel | launches | time (ms) | share | DRAM bytes (GB) |", "|---|---|---|---|---|"]
    for name, (n, t, b) in sorted(tot.items(), key=lambda x: -x[1][1]):
        out.append(f"| `{name}` | {n} | {t / 1e6:.3f} | {t / all_t:.1%} | {b / 1e9:.2f} |")
    out.append(f"| total | {sum(v[0] for v in tot.values())} | {all_t / 1e6:.3f} | 100% | "
               f"{sum(v[2] for v in tot.values()) / 1e9:.2f} |")
    text = "\n".join(out)
    print(text)
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as fh:
            fh.write(text + "\n")
    if "--traffic" in sys.argv:
        import json

        i = sys.argv.index("--traffic")
        path, cfg, steps = sys.argv[i + 1], sys.argv[i + 2], int(sys.argv[i + 3])
        fac = [v for k, v in tot.items() if k.startswith(FACTOR_PREFIXES)]
        data = {}
        try:
            with open(path) as fh:
                data = json.load(fh)
        except (OSError, ValueError):
            pass
        data[cfg] = {"factor_dram_bytes_per_step": sum(v[2] for v in fac) / steps,
                     "factor_kernel_ms_per_step": sum(v[1] for v in fac) / steps / 1e6,
                     "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (serialised launches)"}
        with open(path, "w") as fh:
            json.dump(data, fh, indent=1)


if __name__ == "__main__":
    main()
