"""Isolated kernel micro-benchmarks at a configuration's level shapes (used for
ncu captures: the launches here are the same kernels the solve runs).

    python tools/kernel_bench.py [c2] [--reps R]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_2412_04980_b200 as hdb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case", nargs="?", default="c2")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    prob = bench.CONFIGS[a.case][1](hdb, 1)
    res = bench.kernel_roofline(hdb, prob.hierarchy, reps=a.reps)
    peak, _ = bench._peaks()
    print(json.dumps({k: {"gbs": round(v["gbs"], 1), "ms": round(v["ms"], 4), "frac": round(v["gbs"] / peak, 3)}
                      for k, v in res.items()}))


if __name__ == "__main__":
    main()
