"""Reduce the reference's full config-2 record (run_reference_solve.py output) to a
committed fixture: history, counts and every 32nd solution point."""
import sys

import numpy as np

src, dst = (sys.argv[1:3] + ["/tmp/refruns/c2.npz", "tests/golden/solve_c2.npz"][len(sys.argv[1:3]):])[:2]
d = np.load(src, allow_pickle=False)
x = d["solution"]
np.savez_compressed(dst, outer_iterations=d["outer_iterations"], converged=d["converged"],
                    final_relres=d["final_relres"], residual_history=d["residual_history"], wall_s=d["wall_s"],
                    workers=d["workers"], solution_l2=d["solution_l2"], solution_stride=np.array(32),
                    solution_sub=x[::32, ::32], cycle_iters=d["cycle_iters"], cslp_iters=d["cslp_iters"],
                    matvecs=d["matvecs"])
