"""Single-rank vs 2-rank thread-slab solves of the mixed-BC heterogeneous wedge case
(tests/test_gpu_distributed.py) under each Gram-Schmidt form, to separate the rounding
sensitivity of the problem from the slab path.  Prints relative solution deltas."""
import json
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402


def build(hdb):
    vel = hdb.VelocityModel(kind="wedge", layers=[(-400.0, -200.0, 2000.0), (-800.0, -600.0, 1500.0), (0.0, 0.0, 3000.0)])
    hier = hdb.build_hierarchy(((0.0, 600.0), (-1000.0, 0.0)), h=600.0 / 144, ml=4, velocity=vel, f=20.0,
                               boundary=("sommerfeld", "sommerfeld", "dirichlet", "sommerfeld"))
    return hdb.grid.Problem("wedge-mixed", hier, hdb.point_source_rhs(hier, (300.0, -300.0)))


def main():
    import paper_2412_04980_b200 as hdb
    from paper_2412_04980_b200 import _lib
    from paper_2412_04980_b200.distributed import DistContext
    L = _lib.lib()
    out = {}
    for ls in (1, 0):
        _lib.check(L.hdb_option(b"mgs_ls", ls))
        prob = build(hdb)
        with hdb.MadpSolver(prob.hierarchy, hdb.preset("MADP", prob.hierarchy)) as s:
            u, rep = s.solve(prob.rhs)
        x1 = u.grid_view(prob.hierarchy).copy()
        group = DistContext.new_group()
        res = [None, None]

        def worker(r):
            ctx = DistContext.threads(r, 2, group)
            ctx.min_rows = 16
            p = build(hdb)
            sv = hdb.MadpSolver(p.hierarchy, hdb.preset("MADP", p.hierarchy), dist=ctx)
            x, rp = sv.solve(p.rhs)
            res[r] = (sv._spec(0).row0, np.array(x), rp.outer_iterations, rp.cycle_iters)
            sv.close()
            ctx.close()
        th = [threading.Thread(target=worker, args=(r,)) for r in range(2)]
        [t.start() for t in th]
        [t.join() for t in th]
        x2 = np.concatenate([r[1] for r in sorted(res, key=lambda t: t[0])], axis=0)
        out[f"mgs_ls={ls}"] = {"single_its": rep.outer_iterations, "slab_its": res[0][2],
                               "single_cycles": str(rep.cycle_iters)[:200], "slab_cycles": str(res[0][3])[:200],
                               "rel_delta": float(np.linalg.norm(x2 - x1) / np.linalg.norm(x1))}
        out[f"x_single_{ls}"] = x1
    _lib.check(L.hdb_option(b"mgs_ls", 1))
    out["single_ls_vs_mgs"] = float(np.linalg.norm(out["x_single_1"] - out["x_single_0"]) / np.linalg.norm(out["x_single_0"]))
    del out["x_single_1"], out["x_single_0"]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
