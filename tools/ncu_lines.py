"""Per CUDA source line: instructions executed and stall samples of one
kernel in an ncu report (development tool).

python tools/ncu_lines.py rep [N]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, rows = "?", []
hdr = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0]:
        continue
    try:
        ins = int(r[hdr.index("Instructions Executed")])
        st = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    rows.append((ins, st, f"{fname}:{r[0]}", r[1].strip()))
ti = sum(x[0] for x in rows) or 1
ts = sum(x[1] for x in rows) or 1
print(f"total warp-instructions {ti}, stall samples {ts}")
print("-- by instructions")
for ins, st, loc, src in sorted(rows, reverse=True)[:N]:
    print(f"{100 * ins / ti:5.1f}% ins {100 * st / ts:5.1f}% stall  {loc:18s} {src[:90]}")
print("-- by stall samples")
for ins, st, loc, src in sorted(rows, key=lambda x: -x[1])[:N]:
    print(f"{100 * ins / ti:5.1f}% ins {100 * st / ts:5.1f}% stall  {loc:18s} {src[:90]}")
