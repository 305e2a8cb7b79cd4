"""Run the REFERENCE `helmdef` solver (imported read-only from /root/reference)
on one named configuration and store its convergence record.

Container-only tool: it imports /root/reference/pkg/src, which does not exist
on the GPU box.  The small outputs it writes (iteration counts, residual
histories, solution norms / down-sampled solutions) are committed under
tests/golden/ and are what the GPU parity tests compare against.

Usage:  python tests/golden/run_reference_solve.py CONFIG OUT.npz [--workers W] [--perturb]

--perturb solves with b' = b + 1e-15 max|b| (N(0,1) + i N(0,1)), default_rng(0)
(SURVEY §11): the reference's own self-sensitivity, i.e. the noise floor the
GPU-vs-reference deltas are held to.
"""
import argparse
import os
import sys
import time

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from helmdef import (MadpSolver, VelocityModel, build_hierarchy, mp1_problem,  # noqa: E402
                     point_source_rhs, preset, wedge_problem)

BASELINE_WEDGE = [(-400.0, -200.0, 2000.0), (-800.0, -600.0, 1500.0), (0.0, 0.0, 3000.0)]


def make(config):
    if config == "c1":            # BASELINE configs[0] as written
        p = mp1_problem(k=50.0, n=129, ml=2, boundary="dirichlet")
        return p.hierarchy, p.rhs.grid_view(p.hierarchy)
    if config == "c1s":           # config 1 with Sommerfeld closure (convergent variant)
        p = mp1_problem(k=50.0, n=129, ml=2, boundary="sommerfeld")
        return p.hierarchy, p.rhs.grid_view(p.hierarchy)
    if config == "c1s3":
        p = mp1_problem(k=50.0, n=129, ml=3, boundary="sommerfeld")
        return p.hierarchy, p.rhs.grid_view(p.hierarchy)
    if config == "wedge20":       # reference default wedge, 20 Hz, 145x241, ml=4
        p = wedge_problem(f=20.0, nx=145, ml=4)
        return p.hierarchy, p.rhs.grid_view(p.hierarchy)
    if config.startswith("c2a"):  # config-2 analogue: k=100, 1025^2, ml=6
        p = mp1_problem(k=100.0, n=1025, ml=6, boundary="sommerfeld")
        return p.hierarchy, p.rhs.grid_view(p.hierarchy)
    if config == "c2":            # BASELINE configs[1]: k=200, 4097^2, ml=7
        p = mp1_problem(k=200.0, n=4097, ml=7, boundary="sommerfeld")
        return p.hierarchy, p.rhs.grid_view(p.hierarchy)
    if config.startswith("c3_"):  # BASELINE configs[2]: wedge geometry of BASELINE, h=0.5, ml=5
        f = float(config.split("_")[1])
        vel = VelocityModel(kind="wedge", layers=list(BASELINE_WEDGE))
        hier = build_hierarchy(((0.0, 600.0), (-1000.0, 0.0)), h=0.5, ml=5, velocity=vel, f=f)
        rhs = point_source_rhs(hier, (300.0, 0.0))
        return hier, rhs.grid_view(hier)
    if config == "c5s":           # BASELINE configs[4] shape at reduced size: [0,1] x [0,2], h = 1/1024
        h = 1.0 / 1024            # (1025 x 2049 points, two stacked unit squares), k^3 h^2 = 0.5, ml = 5
        k = (0.5 / h ** 2) ** (1.0 / 3.0)
        hier = build_hierarchy(((0.0, 1.0), (0.0, 2.0)), h=h, ml=5, k=k, boundary="sommerfeld")
        return hier, point_source_rhs(hier, (0.5, 1.0)).grid_view(hier)
    if config.startswith("c4_h"):  # BASELINE configs[3] model (gridfile raster): c4_h6_f40 (ml 3), c4_h12_f40 (ml 2)
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
        from paper_2412_04980_b200.models import C4_DOMAIN, C4_SOURCE, synthetic_layered_velocity
        h = float(config.split("_h")[1].split("_")[0])
        f = float(config.split("_f")[1])
        v = synthetic_layered_velocity(2412, dx=6.0)
        vel = VelocityModel(kind="gridfile", values=v.values, dx=v.dx, dy=v.dy, x0=v.x0, y0=v.y0)
        hier = build_hierarchy(C4_DOMAIN, h=h, ml=3 if h == 6.0 else 2, velocity=vel, f=f)
        return hier, point_source_rhs(hier, C4_SOURCE).grid_view(hier)
    raise SystemExit(f"unknown config {config}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("out")
    ap.add_argument("--workers", type=int, default=1)
    ap.add_argument("--max-outer", type=int, default=150)
    ap.add_argument("--save-solution", action="store_true")
    ap.add_argument("--perturb", action="store_true")
    a = ap.parse_args()
    from helmdef.krylov import StopRule
    hier, b = make(a.config)
    if a.perturb:
        g = np.random.default_rng(0)
        b = b + 1e-15 * np.abs(b).max() * (g.standard_normal(b.shape) + 1j * g.standard_normal(b.shape))
    cfg = preset("MADP", hier, outer_stop=StopRule(1e-6, a.max_outer))
    t0 = time.perf_counter()
    with MadpSolver(hier, cfg, workers=a.workers) as s:
        u, rep = s.solve(b)
    wall = time.perf_counter() - t0
    x = u.grid_view(hier)
    rec = dict(
        config=a.config, outer_iterations=rep.outer_iterations, converged=rep.converged,
        final_relres=rep.final_relres, residual_history=np.array(rep.residual_history),
        wall_s=wall, workers=a.workers, solution_l2=float(np.linalg.norm(x)),
        cycle_iters=repr(rep.cycle_iters), cslp_iters=repr(rep.cslp_iters),
        matvecs=repr(rep.matvecs), iteration_wall_ms=np.array(rep.iteration_wall_ms),
        perturbed=a.perturb,
    )
    if a.save_solution:
        rec["solution"] = x
    np.savez(a.out, **rec)
    print(a.config, rep.outer_iterations, rep.converged, rep.final_relres, wall, flush=True)


if __name__ == "__main__":
    main()
