"""Top SASS lines by stall samples (development tool): python tools/ncu_hot.py rep [N]"""
import csv, subprocess, sys
rep = sys.argv[1]; N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ia, isrc, ism = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ism]), r[ia], r[isrc].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
for i, (s, a, src) in enumerate(data):
    pass
idx = {a: i for i, (_, a, _) in enumerate(data)}
for s, a, src in sorted(data, reverse=True)[:N]:
    print(f"{100*s/tot:5.1f}%  {idx[a]:5d}  {src[:110]}")
