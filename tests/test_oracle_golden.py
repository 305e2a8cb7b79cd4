"""Pin the CPU oracle against fixtures produced by the reference itself.

All comparisons are bit-exact (the oracle restates the reference's arithmetic
operation for operation) except where LAPACK is involved (MG coarsest LU),
which is held to 1e-13.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle.chain import verify_against_tables
from gold import GOLDEN, golden


def test_kernel_chain_matches_published_tables():
    with open(os.path.join(GOLDEN, "kernel_tables.json")) as f:
        tabs = json.load(f)
    tabs = {int(l): {k: (v[0], v[1]) for k, v in d.items()} for l, d in tabs.items()}
    assert verify_against_tables(tabs) == []


def test_separable_factorisation_exact():
    from fractions import Fraction
    for level in range(2, 8):
        a, m, cl, cm = oracle.chain.separable_factors(level)
        lt, ld, mt, md, r = oracle.level_kernels(level)
        for y in range(2 * r + 1):
            for x in range(2 * r + 1):
                assert Fraction(lt[y][x]) == cl * (int(a[x]) * int(m[y]) + int(m[x]) * int(a[y]))
                assert Fraction(mt[y][x]) == cm * int(m[x]) * int(m[y])


@pytest.mark.parametrize("bc", ["sommerfeld", "dirichlet"])
@pytest.mark.parametrize("level", [1, 2, 3, 4])
@pytest.mark.parametrize("kind", ["A", "M"])
def test_operator_bitexact(bc, level, kind):
    g = golden("operators.npz")
    hier, _ = oracle.mp1_problem(25.0, 33, 4, bc)
    op = oracle.helmholtz_op(hier, level) if kind == "A" else oracle.cslp_op(hier, level, 0.35)
    u = g[f"mp1_{bc}_L{level}_{kind}_u"]
    np.testing.assert_array_equal(op.apply(u), g[f"mp1_{bc}_L{level}_{kind}_v"])


def test_operator_wedge_and_mixed_bitexact():
    g = golden("operators.npz")
    hier, _ = oracle.wedge_problem(4.0, 25, 3)
    for l in (1, 2, 3):
        op = oracle.helmholtz_op(hier, l)
        np.testing.assert_array_equal(op.apply(g[f"wedge_L{l}_A_u"]), g[f"wedge_L{l}_A_v"])
    np.testing.assert_array_equal(oracle.helmholtz_op(hier, 1).diagonal(), g["wedge_L1_diag"])
    hier = oracle.build_hierarchy(oracle.grid.WEDGE_DOMAIN, 25.0, 3, layers=oracle.grid.BASELINE_WEDGE,
                                  f=6.0, boundary=("dirichlet", "sommerfeld", "sommerfeld", "dirichlet"))
    for l in (1, 2, 3):
        op = oracle.cslp_op(hier, l, 0.5)
        np.testing.assert_array_equal(op.apply(g[f"mixed_L{l}_M_u"]), g[f"mixed_L{l}_M_v"])


@pytest.mark.parametrize("shape", [(17, 17), (41, 25), (9, 65)])
def test_transfers_bitexact(shape):
    g = golden("transfers.npz")
    ny, nx = shape
    np.testing.assert_array_equal(oracle.restrict(g[f"r_{ny}x{nx}_in"]), g[f"r_{ny}x{nx}_out"])
    np.testing.assert_array_equal(oracle.prolong(g[f"p_{ny}x{nx}_in"], shape), g[f"p_{ny}x{nx}_out"])


@pytest.mark.parametrize("name", ["mp1s65", "mp1d65div", "poisson65", "wedge145"])
def test_vcycle(name):
    g = golden("multigrid.npz")
    probs = {"mp1s65": lambda: oracle.mp1_problem(50.0, 65, 2),
             "mp1d65div": lambda: oracle.mp1_problem(20.0, 65, 2, "dirichlet"),
             "poisson65": lambda: oracle.mp1_problem(1e-12, 65, 2, "dirichlet"),
             "wedge145": lambda: oracle.wedge_problem(20.0, 145, 4)}
    hier, _ = probs[name]()
    lv = hier.level(1)
    mg = oracle.CpuMultigrid(lv.nx, lv.ny, lv.h, hier.ksq_at(1), hier.boundary, float(g[f"{name}_beta2"]))
    assert mg.depth == int(g[f"{name}_depth"])
    b = g[f"{name}_b"]
    np.testing.assert_array_equal(mg.ops[0].jacobi(g[f"{name}_jx0"], b, 0.8), g[f"{name}_jx1"])
    if bool(g[f"{name}_diverged"]):
        with pytest.raises(oracle.mg.MgDivergenceOracle):
            mg.vcycle(b)
    else:
        x = mg.vcycle(b)
        np.testing.assert_array_equal(x, g[f"{name}_x"])


def test_fgmres_and_dot():
    g = golden("krylov.npz")
    hier, _ = oracle.mp1_problem(5.0, 9, 2, "dirichlet")
    op = oracle.helmholtz_op(hier, 1)
    x, rep = oracle.fgmres(op.apply, None, g["d9_b"], oracle.Stop(1e-10, 100))
    assert rep.iterations == int(g["d9_its"])
    np.testing.assert_array_equal(np.array(rep.residual_history), g["d9_hist"])
    np.testing.assert_array_equal(x, g["d9_x"])
    hier, _ = oracle.mp1_problem(30.0, 65, 3)
    op = oracle.cslp_op(hier, 1, 0.5)
    x, rep = oracle.fgmres(op.apply, None, g["c65_b"], oracle.Stop(0.1, 49), dot=oracle.reduce_dot)
    assert rep.iterations == int(g["c65_its"])
    np.testing.assert_array_equal(np.array(rep.residual_history), g["c65_hist"])
    np.testing.assert_array_equal(x, g["c65_x"])
    assert oracle.reduce_dot(g["dot_u"], g["dot_v"]) == complex(g["dot_uv"])


def test_cslp_cap_kats():
    # known-answer values of the reference's own test (test_krylov.py:144-148)
    assert oracle.cslp_cap(10000) == 60
    assert oracle.cslp_cap(1) == 6
    assert oracle.cslp_cap(65536) == 96
    assert oracle.cslp_cap(10001) == 61


@pytest.mark.parametrize("name", ["c1s", "wedge20"])
def test_full_solve_matches_reference(name):
    g = golden(f"solve_{name}.npz")
    build = {"c1s": lambda: oracle.mp1_problem(50.0, 129, 2, "sommerfeld"),
             "wedge20": lambda: oracle.wedge_problem(20.0, 145, 4)}[name]
    hier, b = build()
    pols, outer = oracle.madp_preset(hier)
    x, rep = oracle.CpuMadpSolver(hier, pols, outer).solve(b)
    assert rep.iterations == int(g["outer_iterations"])
    # bit-identical to the reference (same host, single-threaded OpenBLAS)
    np.testing.assert_array_equal(np.array(rep.residual_history), g["residual_history"])
    np.testing.assert_array_equal(x, g["solution"])
    assert rep.final_relres == float(g["final_relres"])


def test_bicgstab_bitexact():
    from oracle.krylov import bicgstab
    g = golden("krylov.npz")
    n = 17
    T = (2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)).astype(np.complex128)
    x, rep = bicgstab(lambda u: T @ u, None, g["bp_b"], oracle.Stop(1e-10, 300))
    assert rep.iterations == int(g["bp_its"])
    np.testing.assert_array_equal(x, g["bp_x"])
    hier, _ = oracle.mp1_problem(5.0, 9, 2, "dirichlet")
    op = oracle.helmholtz_op(hier, 1)
    D = op.diagonal()
    x, rep = bicgstab(op.apply, lambda u: u / D, g["bd9_b"], oracle.Stop(1e-9, 200))
    np.testing.assert_array_equal(np.array(rep.residual_history), g["bd9_hist"])
    np.testing.assert_array_equal(x, g["bd9_x"])
    hier, _ = oracle.mp1_problem(30.0, 65, 3)
    m = oracle.cslp_op(hier, 2, 0.5)
    x, rep = bicgstab(m.apply, None, g["bc33_b"], oracle.Stop(0.1, 30), dot=oracle.reduce_dot)
    np.testing.assert_array_equal(x, g["bc33_x"])


def test_worker_count_invariance():
    """The row-slab worker pool (the bench's multi-threaded reference arm) is
    bit-identical to the inline loops, as the reference's WorkerPool is
    (parallel.py:1-7); the full c1s solve still matches the fixture."""
    from oracle import ops
    rng = np.random.default_rng(5)
    ny, nx = 300, 257
    ksq = 400.0 + 300.0 * rng.random((ny, nx))
    bnd = ("sommerfeld", "dirichlet", "sommerfeld", "sommerfeld")
    u = rng.standard_normal((ny, nx)) + 1j * rng.standard_normal((ny, nx))
    try:
        for level in (1, 2, 3):
            lt, ld, mt, md, _ = oracle.level_kernels(level)
            op = oracle.CpuLevelOp(nx, ny, 1.0 / 128, ksq, bnd, lt, ld, mt, md, shift=complex(1.0, 0.5),
                                   level_scale=4.0 ** (level - 1))
            ops.set_workers(1)
            a1 = op.apply(u)
            j1 = op.jacobi(u, u, 0.8, 2) if level == 1 else None
            ops.set_workers(4)
            np.testing.assert_array_equal(op.apply(u), a1)
            if level == 1:
                np.testing.assert_array_equal(op.jacobi(u, u, 0.8, 2), j1)
        g = golden("solve_c1s.npz")
        hier, b = oracle.mp1_problem(50.0, 129, 2, "sommerfeld")
        pols, outer = oracle.madp_preset(hier)
        x, rep = oracle.CpuMadpSolver(hier, pols, outer).solve(b)
        np.testing.assert_array_equal(x, g["solution"])
    finally:
        ops.set_workers(1)
