"""Add the reference's own noise floors to the committed solve fixtures.

Inputs are full reference records written by run_reference_solve.py (container
only, /tmp/refruns): an unperturbed and a perturbed (--perturb: b + 1e-15 max|b|
noise) solve per configuration.  For each fixture this stores

  floor_hist_abs   max_i |h_i - h'_i| over the common iterations (reference vs
                   perturbed reference)
  floor_sol_rel    ||x - x'|| / ||x|| on the fixture's solution sample
  floor_its        outer iterations of the perturbed run
  floor_hist       the perturbed history

    python tests/golden/reduce_floors.py [/tmp/refruns]
Also writes solve_c1_full.npz: config 1 as written, the reference's full
150-iteration stall (history, counts, every 2nd solution point).
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RUNS = sys.argv[1] if len(sys.argv) > 1 else "/tmp/refruns"


def floors(base, pert, stride):
    h0, h1 = base["residual_history"], pert["residual_history"]
    n = min(len(h0), len(h1))
    x0, x1 = base["solution"][::stride, ::stride], pert["solution"][::stride, ::stride]
    return dict(floor_hist_abs=np.abs(h0[:n] - h1[:n]).max(), floor_sol_rel=np.linalg.norm(x0 - x1) / np.linalg.norm(x0),
                floor_its=int(pert["outer_iterations"]), floor_hist=h1, floor_final_relres=float(pert["final_relres"]))


def update(name, extra):
    path = os.path.join(HERE, name)
    rec = dict(np.load(path, allow_pickle=False))
    rec.update(extra)
    np.savez_compressed(path, **rec)
    print(name, {k: (float(v) if np.ndim(v) == 0 else np.shape(v)) for k, v in extra.items()})


def main():
    # config 2: the committed fixture holds the unperturbed run (every 32nd point)
    g = dict(np.load(os.path.join(HERE, "solve_c2.npz"), allow_pickle=False))
    p = np.load(os.path.join(RUNS, "c2_p.npz"), allow_pickle=False)
    n = min(len(g["residual_history"]), len(p["residual_history"]))
    xs, xp = g["solution_sub"], p["solution"][::32, ::32]
    update("solve_c2.npz", dict(floor_hist_abs=np.abs(g["residual_history"][:n] - p["residual_history"][:n]).max(),
                                floor_sol_rel=np.linalg.norm(xs - xp) / np.linalg.norm(xs),
                                floor_its=int(p["outer_iterations"]), floor_hist=p["residual_history"],
                                floor_final_relres=float(p["final_relres"])))
    for f in ("10", "20", "40"):
        b = np.load(os.path.join(RUNS, f"c3_{f}.npz"), allow_pickle=False)
        pp = np.load(os.path.join(RUNS, f"c3_{f}_p.npz"), allow_pickle=False)
        assert np.array_equal(b["residual_history"], np.load(os.path.join(HERE, f"solve_c3_{f}.npz"))["residual_history"])
        update(f"solve_c3_{f}.npz", floors(b, pp, 8))
    b = np.load(os.path.join(RUNS, "c1.npz"), allow_pickle=False)
    pp = np.load(os.path.join(RUNS, "c1_p.npz"), allow_pickle=False)
    rec = dict(outer_iterations=b["outer_iterations"], converged=b["converged"], final_relres=b["final_relres"],
               residual_history=b["residual_history"], solution_l2=b["solution_l2"], wall_s=b["wall_s"],
               cycle_iters=b["cycle_iters"], cslp_iters=b["cslp_iters"], solution_stride=np.array(2),
               solution_sub=b["solution"][::2, ::2])
    rec.update(floors(b, pp, 2))
    np.savez_compressed(os.path.join(HERE, "solve_c1_full.npz"), **rec)
    print("solve_c1_full.npz", int(b["outer_iterations"]), float(b["final_relres"]), float(rec["floor_hist_abs"]),
          float(rec["floor_sol_rel"]))
    for name in ("c4_h6_f40", "c4_h12_f40"):
        bp = os.path.join(RUNS, f"{name}.npz")
        pq = os.path.join(RUNS, f"{name}_p.npz")
        if os.path.exists(bp) and os.path.exists(pq):
            b = np.load(bp, allow_pickle=False)
            pp = np.load(pq, allow_pickle=False)
            rec = dict(outer_iterations=b["outer_iterations"], converged=b["converged"], final_relres=b["final_relres"],
                       residual_history=b["residual_history"], solution_l2=b["solution_l2"], wall_s=b["wall_s"],
                       cycle_iters=b["cycle_iters"], cslp_iters=b["cslp_iters"], solution_stride=np.array(2),
                       solution_sub=b["solution"][::2, ::2])
            rec.update(floors(b, pp, 2))
            # k^2 checksums of the reference's own hierarchy (levels 1 and 3) for this raster
            sys.path.insert(0, "/root/reference/pkg/src")
            sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
            from helmdef import VelocityModel, build_hierarchy
            from paper_2412_04980_b200.models import C4_DOMAIN, synthetic_layered_velocity
            v = synthetic_layered_velocity(2412, dx=6.0)
            vel = VelocityModel(kind="gridfile", values=v.values, dx=v.dx, dy=v.dy, x0=v.x0, y0=v.y0)
            hh = 6.0 if name == "c4_h6_f40" else 12.0
            hier = build_hierarchy(C4_DOMAIN, h=hh, ml=3 if hh == 6.0 else 2, velocity=vel, f=40.0)
            rec["ksq_checksum"] = np.array([hier.ksq[0].sum(), hier.ksq[-1].sum()])
            np.savez_compressed(os.path.join(HERE, f"solve_{name}.npz"), **rec)
            print(name, int(b["outer_iterations"]), float(rec["floor_hist_abs"]), float(rec["floor_sol_rel"]))


if __name__ == "__main__":
    main()
