"""Solve one configuration on the GPU and print convergence + per-level telemetry.

    python tools/profile_solve.py [c2|c2a|c1s|c3_40|wedge20] [--repeat R]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import paper_2412_04980_b200 as hdb  # noqa: E402

CASES = {
    "c2": lambda: hdb.mp1_problem(k=200.0, n=4097, ml=7),
    "c2a": lambda: hdb.mp1_problem(k=100.0, n=1025, ml=6),
    "c1s": lambda: hdb.mp1_problem(k=50.0, n=129, ml=2),
    "c1": lambda: hdb.mp1_problem(k=50.0, n=129, ml=2, boundary="dirichlet"),
    "wedge20": lambda: hdb.wedge_problem(f=20.0, nx=145, ml=4),
    "c3_10": lambda: hdb.wedge_problem(f=10.0, nx=1201, ml=5, layers=hdb.grid.BASELINE_WEDGE_LAYERS),
    "c3_20": lambda: hdb.wedge_problem(f=20.0, nx=1201, ml=5, layers=hdb.grid.BASELINE_WEDGE_LAYERS),
    "c3_40": lambda: hdb.wedge_problem(f=40.0, nx=1201, ml=5, layers=hdb.grid.BASELINE_WEDGE_LAYERS),
    "c5": lambda: hdb.c5_problem(1),
    "c4_40": lambda: hdb.synthetic_layered_problem(40.0, 0.75, 6),
    "c4_20": lambda: hdb.synthetic_layered_problem(20.0, 0.75, 6),
    "c4_10": lambda: hdb.synthetic_layered_problem(10.0, 0.75, 6),
    "c4s": lambda: hdb.synthetic_layered_problem(40.0, 6.0, 3),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case", nargs="?", default="c2")
    ap.add_argument("--repeat", type=int, default=2)
    a = ap.parse_args()
    import torch
    prob = CASES[a.case]()
    cfg = hdb.preset("MADP", prob.hierarchy)
    s = hdb.MadpSolver(prob.hierarchy, cfg)
    b = torch.from_numpy(prob.rhs.grid_view(prob.hierarchy).copy()).cuda()
    x = torch.empty_like(b)
    dms = []
    for r in range(a.repeat):
        t0 = time.perf_counter()
        rep = s.solve_device(b, x)
        wall = time.perf_counter() - t0
        dms.append(rep.device_ms)
    out = {"case": a.case, "outer": rep.outer_iterations, "converged": rep.converged,
           "final_relres": rep.final_relres, "device_ms": rep.device_ms, "wall_s": wall,
           "device_ms_all": [round(v, 1) for v in dms],
           "cycle_max": {l: rep.cycle_max(l) for l in range(2, prob.hierarchy.ml + 1)},
           "cslp_max": {l: rep.cslp_max(l) for l in range(1, prob.hierarchy.ml + 1)},
           "cslp_calls": {l: len(v) for l, v in rep.cslp_iters.items()},
           "cslp_total_its": {l: sum(v) for l, v in rep.cslp_iters.items()},
           "cycle_total_its": {l: sum(v) for l, v in rep.cycle_iters.items()},
           "matvecs": rep.matvecs, "profile": s.profile(),
           "history": rep.residual_history}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
