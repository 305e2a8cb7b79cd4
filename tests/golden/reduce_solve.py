"""Reduce a full reference solve record (run_reference_solve.py --save-solution)
to a committed fixture: counts, history and every `stride`-th solution point.

    python tests/golden/reduce_solve.py /tmp/refruns/c3_40.npz tests/golden/solve_c3_40.npz 8
"""
import sys

import numpy as np

src, dst, stride = sys.argv[1], sys.argv[2], int(sys.argv[3])
d = np.load(src, allow_pickle=False)
x = d["solution"]
np.savez_compressed(dst, outer_iterations=d["outer_iterations"], converged=d["converged"],
                    final_relres=d["final_relres"], residual_history=d["residual_history"], wall_s=d["wall_s"],
                    workers=d["workers"], solution_l2=d["solution_l2"], solution_stride=np.array(stride),
                    solution_sub=x[::stride, ::stride], cycle_iters=d["cycle_iters"], cslp_iters=d["cslp_iters"],
                    matvecs=d["matvecs"])
print(dst, int(d["outer_iterations"]), float(d["final_relres"]), x[::stride, ::stride].shape)
