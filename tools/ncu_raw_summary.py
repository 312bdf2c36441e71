"""Summarise `ncu --page raw --csv` exports (one kernel each) into a table
(development tool; the summaries worth keeping go to profiles/).

python tools/ncu_raw_summary.py [--json out.json] name=path_raw.csv [...]
"""
import csv
import json
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}


def row(path):
    rows = list(csv.reader(open(path)))
    h, u = rows[0], rows[1]
    v = next(r for r in rows[2:] if len(r) == len(h))
    return h, u, v


def val(h, u, v, name):
    if name not in h:
        return None
    i = h.index(name)
    try:
        return float(v[i].replace(",", "")) * SCALE.get(u[i], 1)
    except ValueError:
        return None


def main(argv):
    out_json = None
    if argv and argv[0] == "--json":
        out_json, argv = argv[1], argv[2:]
    recs = []
    for a in argv:
        name, path = a.split("=", 1)
        h, u, v = row(path)
        t = val(h, u, v, "gpu__time_duration.sum")
        rd, wr = val(h, u, v, "dram__bytes_read.sum"), val(h, u, v, "dram__bytes_write.sum")
        stalls = sorted(((val(h, u, v, k) or 0, k.replace("smsp__average_warp_latency_issue_stalled_", "")
                          .replace("smsp__pcsamp_warps_issue_stalled_", "")) for k in h
                         if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")),
                        reverse=True)[:4]
        tot = sum(x for x, _ in stalls) or 1
        rec = {"name": name, "kernel": v[h.index("Kernel Name")][:100], "us": round(t * 1e6, 2) if t else None,
               "dram_read_GB": round(rd / 1e9, 4) if rd is not None else None,
               "dram_write_GB": round(wr / 1e9, 4) if wr is not None else None,
               "dram_TBps": round((rd + wr) / t / 1e12, 3) if t and rd is not None else None,
               "dram_pct_of_peak": val(h, u, v, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
               "sm_pct": val(h, u, v, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
               "occupancy_pct": val(h, u, v, "sm__warps_active.avg.pct_of_peak_sustained_active"),
               "regs": val(h, u, v, "launch__registers_per_thread"),
               "top_stalls": [s for _, s in stalls]}
        recs.append(rec)
        print(f"{name:18s} {rec['us']:>9} us  dram {rec['dram_read_GB']} + {rec['dram_write_GB']} GB = "
              f"{rec['dram_TBps']} TB/s ({rec['dram_pct_of_peak']} % of peak)  sm {rec['sm_pct']} %  occ "
              f"{rec['occupancy_pct']} %  regs {rec['regs']}  stalls {rec['top_stalls']}  {rec['kernel'][:60]}")
    if out_json:
        with open(out_json, "w") as f:
            json.dump(recs, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
