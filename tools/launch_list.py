"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
launches, total ms, share of the listed GPU time, mean us per launch.

    python tools/launch_list.py launches.csv "header line" > profiles/r02_launches_c2.txt
"""
import csv
import sys
from collections import defaultdict


def main():
    path, header = sys.argv[1], sys.argv[2]
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    head = rows[0]
    col = {h: i for i, h in enumerate(head)}
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[col["Metric Name"]] != "gpu__time_duration.sum":
            continue
        unit = r[col["Metric Unit"]]
        v = float(r[col["Metric Value"]].replace(",", ""))
        ns = v * {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1.0)
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("hdb::", "")
        agg[name][0] += 1
        agg[name][1] += ns
    total = sum(v[1] for v in agg.values())
    print(header)
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (serialised, cold cache: compare SHARES)")
    print(f"{'kernel':48s} {'launches':>9s} {'ms':>9s} {'share':>7s} {'avg_us':>9s}")
    for name, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:48]:48s} {n:9d} {ns / 1e6:9.2f} {100 * ns / total:6.1f}% {ns / 1e3 / n:9.2f}")
    print(f"{'total':48s} {sum(v[0] for v in agg.values()):9d} {total / 1e6:9.2f}")


if __name__ == "__main__":
    main()
