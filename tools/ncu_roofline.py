"""Per-launch DRAM traffic of the bench's roofline kernel from an `ncu --set full`
capture taken inside the config-2 solve, written where bench.py reads it
(profiles/r02_roofline_ncu.json):

    python tools/ncu_roofline.py REPORT.ncu-rep mgs_coop c2 "source text"
"""
import csv
import io
import json
import os
import subprocess
import sys

UNITS = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "byte": 1.0,
         "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    rep, family, config, source = sys.argv[1:5]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(head)}

    def val(r, m):
        return float(r[col[m]].replace(",", "")) * UNITS.get(units[col[m]], 1.0)
    launches = [{"kernel": r[col["Kernel Name"]].split("(")[0], "us_cold": round(val(r, "gpu__time_duration.sum") * 1e6, 2),
                 "dram_read_MB": round(val(r, "dram__bytes_read.sum") / 1e6, 2),
                 "dram_write_MB": round(val(r, "dram__bytes_write.sum") / 1e6, 2),
                 "l2_hit_pct": round(val(r, "lts__t_sector_hit_rate.pct"), 1) if "lts__t_sector_hit_rate.pct" in col else None}
                for r in data]
    traffic = sum((l["dram_read_MB"] + l["dram_write_MB"]) * 1e6 for l in launches) / len(launches)
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "r02_roofline_ncu.json")
    out = {"config": config, "source": source,
           "note": "ncu replays each launch with cold caches; traffic is the mean DRAM read+write per captured launch",
           "families": {family: {"traffic_bytes_per_launch": round(traffic), "launches": launches}}}
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
