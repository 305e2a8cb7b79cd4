"""Repeat a solve and compare solutions / histories bitwise (run-to-run determinism).

    python tools/determinism.py [c2|c2a|c1s|c3_40] [--repeat 3]
"""
import argparse
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_2412_04980_b200 as hdb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case", nargs="?", default="c2a")
    ap.add_argument("--repeat", type=int, default=3)
    a = ap.parse_args()
    import torch
    prob = bench.CONFIGS[a.case][1](hdb, 1)
    hier = prob.hierarchy
    cfg = hdb.preset("MADP", hier)
    s = hdb.MadpSolver(hier, cfg)
    b = torch.from_numpy(prob.rhs.grid_view(hier).copy()).cuda()
    x = torch.empty_like(b)
    out = []
    for _ in range(a.repeat):
        rep = s.solve_device(b, x)
        torch.cuda.synchronize()
        h = hashlib.sha1(x.cpu().numpy().tobytes()).hexdigest()[:16]
        out.append({"its": rep.outer_iterations, "relres": rep.final_relres, "x": h,
                    "cslp_total": {k: v for k, v in getattr(rep, "cslp_total_its", {}).items()} if hasattr(rep, "cslp_total_its") else None})
    print(json.dumps({"case": a.case, "runs": out, "identical": len({o["x"] for o in out}) == 1}))


if __name__ == "__main__":
    main()
