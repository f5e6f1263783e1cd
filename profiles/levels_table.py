"""Markdown table of bench.py's roofline.levels: python profiles/levels_table.py bench.json"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("| depth | fronts | max m | ms | TF/s | % FP64 | GB/s | % HBM |")
print("|---|---|---|---|---|---|---|---|")
for l in d["roofline"]["levels"]:
    print(f"| {l['depth']} | {l['fronts']} | {l['max_m']} | {l['ms']:.2f} | {l['tflops']:.1f} | "
          f"{100 * l['frac_fp64']:.0f}% | {l['gbs']:.0f} | {100 * l['frac_hbm']:.0f}% |")
