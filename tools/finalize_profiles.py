"""Copy one `tools/session.sh` run from gpurun_out/ into the committed
profiles (development tool):

  profiles/rNN/bench_<cfg>_final.json, ref_<cfg>_final.json   both arms, every config
  profiles/rNN/bench_c2_2r_final.json, bench_c5_2r_final.json  2-rank functional runs
  profiles/rNN/pytest_gpu.txt, smoke.txt
  profiles/rNN/ncu_launch_lists.txt                            per-kernel launch summary of each config's bench run
  profiles/rNN/ncu_full_dominant.{txt,json}                    --set full of the dominant kernels
  profiles/ncu_c{1..5}_full.json                               the traffic bench.py reports as roofline.traffic

python tools/finalize_profiles.py [--round r02] [--src gpurun_out]
"""
import argparse
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFGS = ["c1", "c2", "c3", "c3r", "c4", "c5"]
# --set full captures (tools/session.sh cap ...): name -> (bench configs it stands for, units, source)
CAPS = {
    "c2_fused": (["c2"], 1 << 28, "prof_run.py c2 28"),
    "c5_place": (["c1", "c5"], 1 << 28, "prof_run.py partition2 28 (the C1/C5 kernel); bench scales "
                 "dram_bytes_per_unit by N"),
    "c4_gather": (["c4"], 1 << 28, "prof_run.py csr 28"),
    "c3_scatter": (["c3"], 1 << 29, "c3prof.py streams (k_scatter_t, the C3 bench input)"),
}


def launch_summary(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    if not rows:
        return []
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        try:
            per[(r[ii], r[ki])][r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            pass
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, k), m in per.items():
        a = agg[k]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    out = sorted(agg.items(), key=lambda kv: -kv[1][1])
    return [(k, n, t / n / 1e3, b / n / 1e9) for k, (n, t, b) in out]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r02")
    ap.add_argument("--src", default=os.path.join(ROOT, "gpurun_out"))
    a = ap.parse_args()
    dst = os.path.join(ROOT, "profiles", a.round)
    os.makedirs(dst, exist_ok=True)
    for c in CFGS + ["c2_2r", "c5_2r"]:
        src = os.path.join(a.src, f"bench_{c}.json")
        if os.path.exists(src) and os.path.getsize(src) > 0:
            shutil.copy(src, os.path.join(dst, f"bench_{c}_final.json"))
    for c in ["c1", "c2", "c3", "c4", "c5"]:
        src = os.path.join(a.src, f"ref_{c}.json")
        if os.path.exists(src):
            shutil.copy(src, os.path.join(dst, f"ref_{c}_final.json"))
    for f in ["pytest_gpu.txt", "smoke.txt"]:
        if os.path.exists(os.path.join(a.src, f)):
            shutil.copy(os.path.join(a.src, f), os.path.join(dst, f))
    lines = []
    for c in ["c2", "c1", "c3", "c4"]:
        p = os.path.join(a.src, f"launches_{c}.csv")
        if not os.path.exists(p):
            continue
        s = launch_summary(p)
        lines.append(f"== {c}: {sum(n for _, n, _, _ in s)} launches (bench.py --config {c} --steps 2 --warmup 3 "
                     f"--no-cpu under ncu: parity, soak, timed, checked, e2e)")
        for k, n, us, gb in s[:12]:
            lines.append(f"  {n:5d} x {us:10.1f} us avg  {gb:8.3f} GB avg  {k[:75]}")
    with open(os.path.join(dst, "ncu_launch_lists.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    args = [f"{n}={os.path.join(a.src, f'full_{n}_raw.csv')}" for n in CAPS
            if os.path.exists(os.path.join(a.src, f"full_{n}_raw.csv"))]
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_raw_summary.py"), "--json",
                        os.path.join(dst, "ncu_full_dominant.json"), *args], capture_output=True, text=True)
    with open(os.path.join(dst, "ncu_full_dominant.txt"), "w") as f:
        f.write(r.stdout)
    recs = json.load(open(os.path.join(dst, "ncu_full_dominant.json")))
    for rec in recs:
        cfgs, units, source = CAPS[rec["name"]]
        rd, wr = rec["dram_read_GB"] * 1e9, rec["dram_write_GB"] * 1e9
        for c in cfgs:
            out = {"kernel": rec["kernel"], "dram_bytes_read": rd, "dram_bytes_write": wr,
                   "dram_bytes_per_launch": rd + wr, "gpu_time_s": rec["us"] * 1e-6,
                   "dram_gbs": (rd + wr) / (rec["us"] * 1e-6) / 1e9,
                   "source": f"round {a.round[1:].lstrip('0')}, tools/session.sh: ncu --set full --clock-control "
                             f"none ({source})",
                   "units": units, "dram_bytes_per_unit": (rd + wr) / units}
            with open(os.path.join(ROOT, "profiles", f"ncu_{c}_full.json"), "w") as f:
                json.dump(out, f, indent=1)
    print(r.stdout, end="")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
