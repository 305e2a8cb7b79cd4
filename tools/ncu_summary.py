"""Summarise an `ncu --set full` report of tools/ncu_targets.py into the
profiles/*_kernels_ncu.json form (per launch: duration, DRAM bytes, achieved
GB/s against the algorithmic bytes of SURVEY §8(d)).

    python tools/ncu_summary.py gpurun_out/r01e_targets.ncu-rep out.json "source text"
"""
import csv
import io
import json
import subprocess
import sys

# algorithmic bytes per point of the fine level (4097^2) for the targets
ALG_B_PER_PT = {"k_r1w<0": 40, "k_r1w<1": 56, "k_r1w<2": 56, "k_r1s<0": 40, "k_r1s<1": 56, "k_r1s<2": 56,
                "k_resnorm": 40}
WHAT = {"k_r1w<0": "fine-level 5-point apply (K1)", "k_r1w<1": "fine-level residual (K2)",
        "k_r1w<2": "fine-level Jacobi sweep (K3)", "k_resnorm": "fused residual + norms (MG guard)"}
METRICS = {"duration_us": ("gpu__time_duration.sum", 1e-3), "dram_read_MB": ("dram__bytes_read.sum", 1e-6),
           "dram_write_MB": ("dram__bytes_write.sum", 1e-6),
           "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
           "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
           "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
           "registers": ("launch__registers_per_thread", 1.0), "grid": ("launch__grid_size", 1.0)}


def units_scale(unit):
    return {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "byte": 1.0,
            "Kbyte": 1e3, "Mbyte": 1e6,
            "Gbyte": 1e9}.get(unit, 1.0)


def main():
    rep, out, source = sys.argv[1], sys.argv[2], sys.argv[3]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(head)}
    npts = 4097 * 4097
    res = {}
    for r in data:
        name = r[col["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "").replace("hdb::", "")
        e = {}
        for key, (m, s) in METRICS.items():
            if m in col and r[col[m]] not in ("", "n/a"):
                v = float(r[col[m]].replace(",", "")) * units_scale(units[col[m]]) * s
                e[key] = round(v, 3)
        if "dram_read_MB" in e and "dram_write_MB" in e:
            e["traffic_MB"] = round(e["dram_read_MB"] + e["dram_write_MB"], 2)
            if "duration_us" in e:
                e["achieved_traffic_GBs"] = round(e["traffic_MB"] * 1e6 / (e["duration_us"] * 1e-6) / 1e9, 1)
        for pre, bpp in ALG_B_PER_PT.items():
            if short.startswith(pre):
                e["what"] = WHAT.get(pre, "")
                e["algorithmic_MB"] = round(bpp * npts / 1e6, 2)
                if "duration_us" in e:
                    e["achieved_algorithmic_GBs"] = round(bpp * npts / (e["duration_us"] * 1e-6) / 1e9, 1)
        res[short] = e
    json.dump({"source": source, "note": "ncu replays with cold caches and serialised launches: durations are "
               "per-launch cold figures; dram bytes are per launch", "kernels": res}, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
