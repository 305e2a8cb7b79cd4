"""Generate golden fixtures by running the REFERENCE helmdef package.

Container-only (imports /root/reference/pkg/src, read-only).  Writes small
.npz/.json fixtures into tests/golden/; they are committed and travel to the
GPU box, where the reference does not exist.

    python tests/golden/make_golden.py            # unit-level fixtures (seconds)
    python tests/golden/make_golden.py --solves   # + full-solve records (minutes)

solve_c2.npz (BASELINE configs[1], 27 min on 4 threads) is produced by
    python tests/golden/run_reference_solve.py c2 /tmp/c2.npz --workers 4 --save-solution
and reduced to history + every 32nd solution point by tests/golden/reduce_c2.py.
"""
import json
import os
import sys

os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402
from helmdef import (CslpMultigrid, MadpSolver, StopRule, VelocityModel,  # noqa: E402
                     bicgstab, build_hierarchy, fgmres, mp1_problem, point_source_rhs, preset,
                     wedge_problem)
from helmdef.operators import cslp_operator, helmholtz_operator  # noqa: E402
from helmdef.parallel import reduce_dot  # noqa: E402
from helmdef.stencils import REFERENCE_KERNELS  # noqa: E402
from helmdef.transfers import prolong_array, restrict_array  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def rnd(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def kernel_tables():
    out = {str(l): {k: [[list(map(int, r)) for r in v[0]], int(v[1])] for k, v in d.items()}
           for l, d in REFERENCE_KERNELS.items()}
    with open(os.path.join(HERE, "kernel_tables.json"), "w") as f:
        json.dump(out, f)


def operators():
    rng = np.random.default_rng(1)
    rec = {}
    for bc in ("sommerfeld", "dirichlet"):
        p = mp1_problem(k=25.0, n=33, ml=4, boundary=bc)
        for l in (1, 2, 3, 4):
            for kind in ("A", "M"):
                op = helmholtz_operator(p.hierarchy, l) if kind == "A" else \
                    cslp_operator(p.hierarchy, l, beta2=0.35)
                u = rnd(rng, op.shape)
                rec[f"mp1_{bc}_L{l}_{kind}_u"] = u
                rec[f"mp1_{bc}_L{l}_{kind}_v"] = op.apply(u)
    p = wedge_problem(f=4.0, nx=25, ml=3)
    for l in (1, 2, 3):
        op = helmholtz_operator(p.hierarchy, l)
        u = rnd(rng, op.shape)
        rec[f"wedge_L{l}_A_u"] = u
        rec[f"wedge_L{l}_A_v"] = op.apply(u)
        if l == 1:
            op.diagonal()
            rec["wedge_L1_diag"] = op.diagonal()
    # mixed boundary, radius 1..3, heterogeneous k^2
    hier = build_hierarchy(((0.0, 600.0), (-1000.0, 0.0)), h=25.0, ml=3,
                           velocity=VelocityModel(kind="wedge", layers=[(-400.0, -200.0, 2000.0),
                                                                        (-800.0, -600.0, 1500.0),
                                                                        (0.0, 0.0, 3000.0)]),
                           f=6.0, boundary=("dirichlet", "sommerfeld", "sommerfeld", "dirichlet"))
    for l in (1, 2, 3):
        op = cslp_operator(hier, l, beta2=0.5)
        u = rnd(rng, op.shape)
        rec[f"mixed_L{l}_M_u"] = u
        rec[f"mixed_L{l}_M_v"] = op.apply(u)
    np.savez_compressed(os.path.join(HERE, "operators.npz"), **rec)


def transfers():
    rng = np.random.default_rng(42)
    rec = {}
    for (ny, nx) in ((17, 17), (41, 25), (9, 65)):
        v = rnd(rng, (ny, nx))
        c = rnd(rng, ((ny - 1) // 2 + 1, (nx - 1) // 2 + 1))
        rec[f"r_{ny}x{nx}_in"] = v
        rec[f"r_{ny}x{nx}_out"] = restrict_array(v)
        rec[f"p_{ny}x{nx}_in"] = c
        rec[f"p_{ny}x{nx}_out"] = prolong_array(c, (ny, nx))
    np.savez_compressed(os.path.join(HERE, "transfers.npz"), **rec)


def multigrid():
    rng = np.random.default_rng(8)
    rec = {}
    cases = (("mp1s65", mp1_problem(k=50.0, n=65, ml=2), 0.5, False),
             ("mp1d65div", mp1_problem(k=20.0, n=65, ml=2, boundary="dirichlet"), 0.5, False),
             ("poisson65", mp1_problem(k=1e-12, n=65, ml=2, boundary="dirichlet"), 0.0, True),
             ("wedge145", wedge_problem(f=20.0, nx=145, ml=4), 0.5, False))
    for name, prob, beta2, interior in cases:
        lv = prob.hierarchy.level(1)
        mg = CslpMultigrid(lv.nx, lv.ny, lv.h, prob.hierarchy.ksq_at(1), prob.hierarchy.boundary,
                           beta2=beta2)
        b = rnd(rng, lv.shape)
        if interior:
            b[0, :] = b[-1, :] = b[:, 0] = b[:, -1] = 0.0
        rec[f"{name}_b"] = b
        rec[f"{name}_beta2"] = np.array(beta2)
        try:
            rec[f"{name}_x"] = mg.vcycle(b)
            rec[f"{name}_diverged"] = np.array(False)
        except Exception as err:  # MgDivergence is part of the contract (mg.py:128-138)
            assert type(err).__name__ == "MgDivergence"
            rec[f"{name}_diverged"] = np.array(True)
        rec[f"{name}_depth"] = np.array(mg.depth)
        # one Jacobi sweep of the finest sub-level from a random x
        x0 = rnd(rng, lv.shape)
        rec[f"{name}_jx0"] = x0
        rec[f"{name}_jx1"] = mg._smooth(0, x0, b, 1)
    np.savez_compressed(os.path.join(HERE, "multigrid.npz"), **rec)


def krylov():
    rng = np.random.default_rng(11)
    rec = {}
    p = mp1_problem(k=5.0, n=9, ml=2, boundary="dirichlet")
    op = helmholtz_operator(p.hierarchy, 1)
    b = rnd(rng, (9, 9))
    x, rep = fgmres(lambda u: op.apply(u), None, b, StopRule(1e-10, 100))
    rec.update(d9_b=b, d9_x=x, d9_hist=np.array(rep.residual_history), d9_its=rep.iterations,
               d9_final=rep.final_relres)
    p = mp1_problem(k=30.0, n=65, ml=3)
    op = cslp_operator(p.hierarchy, 1, beta2=0.5)
    b = rnd(rng, op.shape)
    x, rep = fgmres(lambda u: op.apply(u), None, b, StopRule(0.1, 49), dot=reduce_dot)
    rec.update(c65_b=b, c65_x=x, c65_hist=np.array(rep.residual_history), c65_its=rep.iterations,
               c65_final=rep.final_relres)
    # Bi-CGSTAB (krylov.py:185-276): SPD Poisson, Jacobi-preconditioned 9x9 Dirichlet, breakdown case
    n = 17
    T = (2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)).astype(np.complex128)
    bb = rng.standard_normal(n) + 0j
    xb, rb = bicgstab(lambda u: T @ u, None, bb, StopRule(1e-10, 300))
    rec.update(bp_b=bb, bp_x=xb, bp_hist=np.array(rb.residual_history), bp_its=rb.iterations)
    p9 = mp1_problem(k=5.0, n=9, ml=2, boundary="dirichlet")
    op9 = helmholtz_operator(p9.hierarchy, 1)
    b9 = rnd(rng, (9, 9))
    D = op9.diagonal()
    xb, rb = bicgstab(lambda u: op9.apply(u), lambda u: u / D, b9, StopRule(1e-9, 200))
    rec.update(bd9_b=b9, bd9_x=xb, bd9_hist=np.array(rb.residual_history), bd9_its=rb.iterations,
               bd9_final=rb.final_relres)
    p65 = mp1_problem(k=30.0, n=65, ml=3)
    m65 = cslp_operator(p65.hierarchy, 2, beta2=0.5)
    b65 = rnd(rng, m65.shape)
    xb, rb = bicgstab(lambda u: m65.apply(u), None, b65, StopRule(0.1, 30), dot=reduce_dot)
    rec.update(bc33_b=b65, bc33_x=xb, bc33_hist=np.array(rb.residual_history), bc33_its=rb.iterations)
    rec["dot_u"] = rnd(rng, (321, 33))
    rec["dot_v"] = rnd(rng, (321, 33))
    rec["dot_uv"] = np.array(reduce_dot(rec["dot_u"], rec["dot_v"]))
    np.savez_compressed(os.path.join(HERE, "krylov.npz"), **rec)


SOLVES = {
    # name: (builder, max_outer, save full solution?)
    "c1s": (lambda: mp1_problem(k=50.0, n=129, ml=2, boundary="sommerfeld"), 150, True),
    "wedge20": (lambda: wedge_problem(f=20.0, nx=145, ml=4), 150, True),
    "c1_cap20": (lambda: mp1_problem(k=50.0, n=129, ml=2, boundary="dirichlet"), 20, True),
    # config-2 analogue (k=100, 1025^2, ml=6): solution stored every 8th point
    "c2a": (lambda: mp1_problem(k=100.0, n=1025, ml=6, boundary="sommerfeld"), 150, 8),
}

# other presets (madp.py:129-189) and a Bi-CGSTAB-CSLP variant on stable small problems
PRESET_SOLVES = {
    "v1_mp1b": ("MADP_V1", lambda: mp1_problem(k=40.0, n=129, ml=3, boundary="sommerfeld")),
    "v2_mp1b": ("MADP_V2", lambda: mp1_problem(k=40.0, n=129, ml=3, boundary="sommerfeld")),
    "v3_wedge": ("MADP_V3", lambda: wedge_problem(f=20.0, nx=145, ml=4)),
    "bicg_wedge": ("BICG", lambda: wedge_problem(f=20.0, nx=145, ml=4)),
}


def c4_solve():
    """BASELINE configs[3] model (this package's seeded generator, raster fed to the
    reference as a gridfile VelocityModel) at h = 6 m, 40 Hz, 3 levels."""
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_2412_04980_b200.models import C4_DOMAIN, C4_SOURCE, synthetic_layered_velocity
    v = synthetic_layered_velocity(2412, dx=6.0)
    vel = VelocityModel(kind="gridfile", values=v.values, dx=v.dx, dy=v.dy, x0=v.x0, y0=v.y0)
    hier = build_hierarchy(C4_DOMAIN, h=6.0, ml=3, velocity=vel, f=40.0)
    b = point_source_rhs(hier, C4_SOURCE).grid_view(hier)
    with MadpSolver(hier, preset("MADP", hier)) as s:
        u, rep = s.solve(b)
    x = u.grid_view(hier)
    np.savez_compressed(os.path.join(HERE, "solve_c4_h6_f40.npz"), outer_iterations=rep.outer_iterations,
                        converged=rep.converged, final_relres=rep.final_relres,
                        residual_history=np.array(rep.residual_history), solution_stride=np.array(4),
                        solution_sub=x[::4, ::4], ksq_checksum=np.array([hier.ksq[0].sum(), hier.ksq[2].sum()]),
                        cycle_iters=json.dumps({str(k): v for k, v in rep.cycle_iters.items()}))
    print("c4", rep.outer_iterations, rep.final_relres, rep.wall_ms)


def grid_models():
    """k^2 / velocity fields of the reference's problem builders (grid.py:184-217,
    350-427) at small sizes: wedge (default and BASELINE interfaces), the
    synthetic Marmousi stand-in raster and its bilinear resampling, a gridfile
    model with a non-grid-aligned raster."""
    from helmdef import marmousi_problem, synthetic_marmousi_velocity
    rec = {}
    p = wedge_problem(f=7.0, nx=61, ml=3)
    rec["wedge_ksq1"] = p.hierarchy.ksq[0]
    rec["wedge_ksq3"] = p.hierarchy.ksq[2]
    rec["wedge_rhs"] = p.rhs.data
    vel = VelocityModel(kind="wedge", layers=[(-400.0, -200.0, 2000.0), (-800.0, -600.0, 1500.0), (0.0, 0.0, 3000.0)])
    h = build_hierarchy(((0.0, 600.0), (-1000.0, 0.0)), h=12.5, ml=3, velocity=vel, f=9.0)
    rec["bwedge_ksq1"] = h.ksq[0]
    m = synthetic_marmousi_velocity(185, 61)
    rec["marm_values"] = m.values
    rec["marm_meta"] = np.array([m.dx, m.dy, m.x0, m.y0])
    mp = marmousi_problem(3.0, nx=185, ml=3)
    rec["marm_ksq1"] = mp.hierarchy.ksq[0]
    rec["marm_rhs"] = mp.rhs.data
    mg = marmousi_problem(2.0, nx=93, ml=2, velocity=m)
    rec["marmg_ksq1"] = mg.hierarchy.ksq[0]
    rng = np.random.default_rng(21)
    raster = 1500.0 + 2000.0 * rng.random((23, 37))
    gv = VelocityModel(kind="gridfile", values=raster, dx=17.3, dy=11.1, x0=-5.0, y0=-240.0)
    gh = build_hierarchy(((0.0, 600.0), (-250.0, 0.0)), h=6.25, ml=2, velocity=gv, f=11.0)
    rec["raster_in"] = raster
    rec["raster_ksq1"] = gh.ksq[0]
    np.savez_compressed(os.path.join(HERE, "grid_models.npz"), **rec)


def api_surface():
    """Reference outputs of the host-side API names this package re-implements:
    assemble_csr (operators.py:261-328), LevelOperator.pad / ksq_pad (:44-93,127),
    partition_grid tiles (parallel.py:71-109), verify_chain records
    (stencils.py:321-371), galerkin_coarsen of the level-1 pair (:149-180)."""
    from helmdef import assemble_csr, partition_grid, verify_chain, galerkin_coarsen
    from helmdef.stencils import level_kernels
    rng = np.random.default_rng(31)
    rec = {}
    vel = VelocityModel(kind="wedge", layers=[(-400.0, -200.0, 2000.0), (-800.0, -600.0, 1500.0), (0.0, 0.0, 3000.0)])
    for tag, bc in (("s", "sommerfeld"), ("d", "dirichlet"), ("m", ("dirichlet", "sommerfeld", "sommerfeld", "dirichlet"))):
        hier = build_hierarchy(((0.0, 600.0), (-1000.0, 0.0)), h=25.0, ml=3, velocity=vel, f=6.0, boundary=bc)
        for l in (1, 2, 3):
            op = cslp_operator(hier, l, beta2=0.5) if tag != "s" else helmholtz_operator(hier, l)
            rec[f"asm_{tag}{l}"] = assemble_csr(op).toarray()
            u = rnd(rng, op.shape)
            rec[f"pad_{tag}{l}_u"] = u
            rec[f"pad_{tag}{l}"] = op.pad(u)
            rec[f"kpad_{tag}{l}"] = op.ksq_pad
    for name, prob in (("mp1_257_5", mp1_problem(k=20.0, n=257, ml=5)), ("wedge_145_4", wedge_problem(f=10.0, nx=145, ml=4))):
        for w in (1, 2, 3, 4, 6, 8):
            part = partition_grid(prob.hierarchy, w)
            rec[f"tiles_{name}_{w}"] = np.array([[l, t.j0, t.j1, t.i0, t.i1] for l in sorted(part.tiles)
                                                 for t in part.tiles[l]])
    rec["verify_chain"] = np.array([[r["level"], r["kind"] == "mass", r["exact_match"], r["within_ulp"]]
                                    for r in verify_chain()])
    lap2, mass2 = galerkin_coarsen(*level_kernels(1))
    rec["coarsen_l1_lap"] = np.array(lap2.numerators)
    rec["coarsen_l1_mass"] = np.array(mass2.numerators)
    rec["coarsen_l1_den"] = np.array([lap2.denominator, mass2.denominator])
    np.savez_compressed(os.path.join(HERE, "api_surface.npz"), **rec)


def io_files():
    """Reference-written report / field / config files (format compatibility fixtures)."""
    import helmdef.io as hio
    cfg = hio.parse_config("problem = mp1b\nwavenumber = 50\nnx = 129\nlevels = 2\nlevel2.cycle_tol = 0.3\n")
    prob = hio.build_problem(cfg)
    with MadpSolver(prob.hierarchy, hio.build_solver_config(cfg, prob.hierarchy)) as s:
        u, rep = s.solve(prob.rhs)
    hio.write_report(rep, os.path.join(HERE, "ref_report_c1s.csv"))
    p9 = mp1_problem(k=5.0, n=9, ml=2)
    from helmdef import ComplexField
    z = np.random.default_rng(4).standard_normal(81) + 1j * np.random.default_rng(5).standard_normal(81)
    hio.write_field(ComplexField(1, z), p9.hierarchy, os.path.join(HERE, "ref_field_9.csv"))
    with open(os.path.join(HERE, "ref_config_render.txt"), "w") as fh:
        fh.write(hio.render_config(cfg))


def preset_solves():
    import dataclasses
    for name, (pre, build) in PRESET_SOLVES.items():
        prob = build()
        hier = prob.hierarchy
        if pre == "BICG":  # MADP with Bi-CGSTAB instead of GMRES for the CSLP levels
            cfg = preset("MADP", hier)
            pols = tuple(dataclasses.replace(p, cslp_method="bicgstab") if p.cslp_method == "gmres" else p
                         for p in cfg.policies)
            cfg = dataclasses.replace(cfg, policies=pols, preset_name="MADP+bicgstab")
        else:
            cfg = preset(pre, hier)
        with MadpSolver(hier, cfg) as s:
            u, rep = s.solve(prob.rhs.grid_view(hier))
            g = np.random.default_rng(0)
            b = prob.rhs.grid_view(hier)
            bp = b + 1e-15 * np.abs(b).max() * (g.standard_normal(b.shape) + 1j * g.standard_normal(b.shape))
            up, repp = s.solve(bp)
        h0, h1 = np.array(rep.residual_history), np.array(repp.residual_history)
        n = min(len(h0), len(h1))
        x, xp = u.grid_view(hier), up.grid_view(hier)
        np.savez_compressed(os.path.join(HERE, f"preset_{name}.npz"), outer_iterations=rep.outer_iterations,
                            converged=rep.converged, residual_history=h0, solution=x,
                            cycle_iters=json.dumps({str(k): v for k, v in rep.cycle_iters.items()}),
                            cslp_iters=json.dumps({str(k): v for k, v in rep.cslp_iters.items()}),
                            floor_hist_abs=np.abs(h0[:n] - h1[:n]).max(),
                            floor_sol_rel=np.linalg.norm(x - xp) / np.linalg.norm(x))
        print(name, pre, rep.outer_iterations, rep.final_relres, np.abs(h0[:n] - h1[:n]).max())


def solves(names):
    for name in names:
        build, cap, save_x = SOLVES[name]
        prob = build()
        hier = prob.hierarchy
        b = prob.rhs.grid_view(hier)
        cfg = preset("MADP", hier, outer_stop=StopRule(1e-6, cap))
        with MadpSolver(hier, cfg) as s:
            u, rep = s.solve(b)
            x = u.grid_view(hier)
            # oracle self-sensitivity: b perturbed by 1e-15 relative
            g = np.random.default_rng(0)
            bp = b + 1e-15 * np.abs(b).max() * (g.standard_normal(b.shape) + 1j * g.standard_normal(b.shape))
            up, repp = s.solve(bp)
            xp = up.grid_view(hier)
        h0, h1 = np.array(rep.residual_history), np.array(repp.residual_history)
        n = min(len(h0), len(h1))
        rec = dict(outer_iterations=rep.outer_iterations, converged=rep.converged,
                   final_relres=rep.final_relres, residual_history=h0,
                   cycle_iters=json.dumps({str(k): v for k, v in rep.cycle_iters.items()}),
                   cslp_iters=json.dumps({str(k): v for k, v in rep.cslp_iters.items()}),
                   solution_l2=np.linalg.norm(x),
                   floor_hist_abs=np.abs(h0[:n] - h1[:n]).max(),
                   floor_sol_rel=np.linalg.norm(x - xp) / np.linalg.norm(x),
                   floor_its=repp.outer_iterations)
        if save_x is True:
            rec["solution"] = x
        elif save_x:
            rec["solution_stride"] = np.array(save_x)
            rec["solution_sub"] = x[::save_x, ::save_x]
        rec["floor_hist"] = h1
        np.savez_compressed(os.path.join(HERE, f"solve_{name}.npz"), **rec)
        print(name, rep.outer_iterations, rep.final_relres, rec["floor_hist_abs"], rec["floor_sol_rel"])


if __name__ == "__main__":
    kernel_tables()
    operators()
    transfers()
    multigrid()
    krylov()
    if "--solves" in sys.argv:
        solves([a for a in sys.argv[2:]] or list(SOLVES))
    if "--presets" in sys.argv:
        preset_solves()
    if "--c4" in sys.argv:
        c4_solve()
    if "--grid" in sys.argv:
        grid_models()
        api_surface()
    if "--io" in sys.argv:
        io_files()
    print("golden fixtures written to", HERE)
