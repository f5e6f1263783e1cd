"""Stall samples per CUDA source line of one kernel in an ncu report
(needs -lineinfo and --import-source on):
python profiles/ncu_lines.py report.ncu-rep [file-substring] [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    sub = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True, check=True).stdout
    rows, fname, col = [], "", None
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path":
            fname, col = rec[1], None
            continue
        if rec[0] == "Function Name":
            continue
        if rec[0] == "Line No":
            col = rec.index("Warp Stall Sampling (All Samples)")
            icol = rec.index("Instructions Executed") if "Instructions Executed" in rec else None
            continue
        if col is None or not rec[0]:
            continue
        try:
            s = int(rec[col] or 0)
            ins = int(rec[icol] or 0) if icol is not None else 0
        except ValueError:
            continue
        if s or ins:
            rows.append((s, ins, fname.split("/")[-1], int(rec[0]), rec[1].strip()[:100]))
    tot = sum(r[0] for r in rows) or 1
    itot = sum(r[1] for r in rows) or 1
    print(f"total samples {tot}, warp instructions executed {itot}")
    for s, ins, f, ln, src in sorted(rows, reverse=True)[:top]:
        if sub and sub not in f:
            continue
        print(f"{100 * s / tot:5.1f}% stalls {100 * ins / itot:5.1f}% instr  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()
