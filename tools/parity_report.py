"""Measured GPU-vs-reference deltas for every configuration with a reference
record (tests/golden/solve_*.npz, preset_*.npz), beside the reference's own noise
floor (its change under a 1e-15 rhs perturbation), in two engine modes:

  default      separable radius-2/3 operators, low-synchronisation MGS steps
  ref_order    the reference's exact tap order (rg_exact=1) and MGS order (mgs_ls=0)

    python tools/parity_report.py [--cases c1s,wedge20,...] [--out gpurun_out/parity.json]
"""
import argparse
import dataclasses
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402


def builders(hdb):
    W = hdb.grid.BASELINE_WEDGE_LAYERS
    return {
        "c1s": ("solve_c1s.npz", lambda: hdb.mp1_problem(k=50.0, n=129, ml=2), 150),
        "wedge20": ("solve_wedge20.npz", lambda: hdb.wedge_problem(f=20.0, nx=145, ml=4), 150),
        "c1_full": ("solve_c1_full.npz", lambda: hdb.mp1_problem(k=50.0, n=129, ml=2, boundary="dirichlet"), 150),
        "c2a": ("solve_c2a.npz", lambda: hdb.mp1_problem(k=100.0, n=1025, ml=6), 150),
        "c2": ("solve_c2.npz", lambda: hdb.mp1_problem(k=200.0, n=4097, ml=7), 150),
        "c3_10": ("solve_c3_10.npz", lambda: hdb.wedge_problem(f=10.0, nx=1201, ml=5, layers=W), 150),
        "c3_20": ("solve_c3_20.npz", lambda: hdb.wedge_problem(f=20.0, nx=1201, ml=5, layers=W), 150),
        "c3_40": ("solve_c3_40.npz", lambda: hdb.wedge_problem(f=40.0, nx=1201, ml=5, layers=W), 150),
        "c4_h6_f40": ("solve_c4_h6_f40.npz", lambda: hdb.synthetic_layered_problem(40.0, 6.0, 3), 150),
        "c4_h12_f40": ("solve_c4_h12_f40.npz", lambda: hdb.synthetic_layered_problem(40.0, 12.0, 2), 150),
        "c5s": ("solve_c5s.npz", lambda: hdb.c5_problem(P=2, ml=5, cells=1024), 150),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="c1s,wedge20,c1_full,c2a,c3_10,c3_20,c3_40,c4_h12_f40,c5s,c2")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parity.json"))
    a = ap.parse_args()
    import paper_2412_04980_b200 as hdb
    from paper_2412_04980_b200 import _lib
    from gold import golden
    L = _lib.lib()
    B = builders(hdb)
    out = {}
    for name in a.cases.split(","):
        fx, build, cap = B[name]
        try:
            g = golden(fx)
        except BaseException as err:  # noqa: BLE001 (pytest's skip/fail outcome)
            out[name] = {"missing_fixture": fx, "why": str(err)}
            continue
        prob = build()
        hier = prob.hierarchy
        cfg = hdb.preset("MADP", hier, outer_stop=hdb.StopRule(1e-6, cap))
        rec = {"ref_its": int(g["outer_iterations"]), "ref_final_relres": float(g["final_relres"]),
               "floor_hist_abs": float(g["floor_hist_abs"]) if "floor_hist_abs" in g else None,
               "floor_sol_rel": float(g["floor_sol_rel"]) if "floor_sol_rel" in g else None}
        for mode, opts in (("default", (0, 1)), ("ref_order", (1, 0))):
            _lib.check(L.hdb_option(b"rg_exact", opts[0]))
            _lib.check(L.hdb_option(b"mgs_ls", opts[1]))
            with hdb.MadpSolver(hier, cfg) as s:
                t0 = time.perf_counter()
                u, rep = s.solve(prob.rhs)
                wall = time.perf_counter() - t0
            x = u.grid_view(hier)
            h, hr = np.array(rep.residual_history), g["residual_history"]
            n = min(len(h), len(hr))
            if "solution" in g:
                xr, xs = g["solution"], x
            else:
                st = int(g["solution_stride"])
                xr, xs = g["solution_sub"], x[::st, ::st]
            r = {"its": rep.outer_iterations, "converged": rep.converged, "final_relres": rep.final_relres,
                 "hist_abs": float(np.abs(h[:n] - hr[:n]).max()),
                 "hist_abs_first20": float(np.abs(h[:min(n, 21)] - hr[:min(n, 21)]).max()),
                 "sol_rel": float(np.linalg.norm(xs - xr) / np.linalg.norm(xr)), "wall_s": round(wall, 3)}
            if rec["floor_hist_abs"]:
                r["hist_over_floor"] = r["hist_abs"] / rec["floor_hist_abs"]
            if rec["floor_sol_rel"]:
                r["sol_over_floor"] = r["sol_rel"] / rec["floor_sol_rel"]
            rec[mode] = r
        _lib.check(L.hdb_option(b"rg_exact", 0))
        _lib.check(L.hdb_option(b"mgs_ls", 1))
        out[name] = rec
        print(name, json.dumps(rec), flush=True)
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
