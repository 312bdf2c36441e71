"""Summarise an ncu report (development tool).

python tools/ncu_summary.py rep.ncu-rep [...]
python tools/ncu_summary.py --json profiles/ncu_c2_full.json --source "..." [--units N] rep.ncu-rep
    also writes {kernel, dram_bytes_per_launch, ...} for the first kernel in
    the report (bench.py reads `dram_bytes_per_launch` as roofline.traffic).
"""
import csv
import json
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size", "launch__occupancy_limit_registers",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__inst_executed.sum.per_cycle_active", "lts__t_bytes.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}


def kernels(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        if len(v) != len(h):
            continue
        yield h, u, v


def value(h, u, v, name):
    i = h.index(name)
    return float(v[i].replace(",", "")) * SCALE.get(u[i], 1)


def main(path):
    for h, u, v in kernels(path):
        print("kernel:", v[h.index("Kernel Name")][:90])
        stalls = []
        for i, name in enumerate(h):
            if name in WANT:
                print(f"  {name} = {v[i]} {u[i]}")
            if name.startswith("smsp__average_warps_issue_stalled_") and name.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(v[i]), name[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("  top stalls:", ", ".join(f"{n}={x:.2f}" for x, n in stalls[:6]))


def write_json(path, out, source, units=None):
    h, u, v = next(iter(kernels(path)))
    rd, wr = value(h, u, v, "dram__bytes_read.sum"), value(h, u, v, "dram__bytes_write.sum")
    t = value(h, u, v, "gpu__time_duration.sum")
    doc = {"kernel": v[h.index("Kernel Name")][:120], "dram_bytes_read": rd, "dram_bytes_write": wr,
           "dram_bytes_per_launch": rd + wr, "gpu_time_s": t, "dram_gbs": (rd + wr) / t / 1e9, "source": source}
    if units:
        doc["units"] = units
        doc["dram_bytes_per_unit"] = (rd + wr) / units
    with open(out, "w") as f:
        json.dump(doc, f, indent=1)
    print("wrote", out, doc)


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "--json":
        out, src, units = args[1], "", None
        args = args[2:]
        if args[0] == "--source":
            src, args = args[1], args[2:]
        if args[0] == "--units":
            units, args = int(args[1]), args[2:]
        write_json(args[0], out, src, units)
    else:
        for p in args:
            main(p)
