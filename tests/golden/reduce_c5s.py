"""Reduce the reference's runs of the reduced config-5 instance (run_reference_solve.py c5s,
unperturbed and --perturb, /tmp/refruns) to the committed fixture solve_c5s.npz: iteration
counts, residual history, every 4th solution point, and the reference's own noise floors.

    python tests/golden/reduce_c5s.py [/tmp/refruns]
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RUNS = sys.argv[1] if len(sys.argv) > 1 else "/tmp/refruns"


def main():
    b = np.load(os.path.join(RUNS, "c5s.npz"), allow_pickle=False)
    p = np.load(os.path.join(RUNS, "c5s_p.npz"), allow_pickle=False)
    stride = 4
    h0, h1 = b["residual_history"], p["residual_history"]
    n = min(len(h0), len(h1))
    x0, x1 = b["solution"][::stride, ::stride], p["solution"][::stride, ::stride]
    rec = dict(outer_iterations=b["outer_iterations"], converged=b["converged"], final_relres=b["final_relres"],
               residual_history=h0, cycle_iters=b["cycle_iters"], cslp_iters=b["cslp_iters"],
               solution_l2=b["solution_l2"], wall_s=b["wall_s"], workers=b["workers"],
               solution_stride=stride, solution_sub=x0,
               floor_hist_abs=np.abs(h0[:n] - h1[:n]).max(),
               floor_sol_rel=np.linalg.norm(x0 - x1) / np.linalg.norm(x0),
               floor_its=int(p["outer_iterations"]), floor_hist=h1, floor_final_relres=float(p["final_relres"]))
    np.savez_compressed(os.path.join(HERE, "solve_c5s.npz"), **rec)
    print({k: (float(v) if np.ndim(v) == 0 and np.asarray(v).dtype.kind in "fiub" else np.shape(v)) for k, v in rec.items()})


if __name__ == "__main__":
    main()
