"""Summarise an `ncu --set full` capture of the one-launch MGS step (k_mgs_grid_t
or k_mgs_ls) into profiles/*.json: per launch its duration, DRAM read + write,
the algorithmic bytes 16 (j + 1) + 32 B/pt of Arnoldi step j, and achieved GB/s.

    python tools/ncu_mgs_summary.py REPORT.ncu-rep OUT.json NPOINTS J0 "source"

J0 = Arnoldi step of the first captured launch (tools/mgs_target.py runs the
steps 0, 1, 2, ... in order, so launch i is step J0 + i).
"""
import csv
import io
import json
import subprocess
import sys

UNITS = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0,
         "s": 1.0, "byte": 1.0, "Kbyte": 1e3,
         "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep, out, npts, j0, source = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(head)}

    def val(r, m):
        return float(r[col[m]].replace(",", "")) * UNITS.get(units[col[m]], 1.0)
    launches = []
    for i, r in enumerate(data):
        j = j0 + i
        t = val(r, "gpu__time_duration.sum")
        rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
        alg = (16.0 * (j + 1) + 32.0) * npts
        launches.append({"kernel": r[col["Kernel Name"]].split("(")[0], "j": j, "us": round(t * 1e6, 2),
                         "dram_read_MB": round(rd / 1e6, 2), "dram_write_MB": round(wr / 1e6, 2),
                         "alg_MB": round(alg / 1e6, 2), "achieved_alg_GBs": round(alg / t / 1e9, 1),
                         "dram_GBs": round((rd + wr) / t / 1e9, 1),
                         "warps_active_pct": round(val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"), 1)})
    res = {"source": source, "npoints": npts,
           "note": "ncu replays with cold caches and serialised launches; durations are cold per-launch figures",
           "launches": launches,
           "traffic_bytes_per_launch": round(sum((l["dram_read_MB"] + l["dram_write_MB"]) * 1e6 for l in launches)
                                             / len(launches)),
           "alg_bytes_per_launch": round(sum(l["alg_MB"] * 1e6 for l in launches) / len(launches))}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
