"""GPU parity: CUDA kernels and solver vs the reference (golden fixtures) and the oracle.

Stencils, Jacobi and transfers are held BIT-EXACT (they replicate the
reference's arithmetic); reductions are deterministic but not bit-identical to
OpenBLAS, so Krylov quantities are held to tolerances stated per test.
"""
import json

import numpy as np
import pytest

import oracle
from gold import golden, parity_bar

pytestmark = pytest.mark.gpu

hdb = pytest.importorskip("paper_2412_04980_b200")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture
def exact_taps():
    """Radius-2/3 operators in the reference's row-major tap order (bit-exact path)."""
    from paper_2412_04980_b200 import _lib
    _lib.check(_lib.lib().hdb_option(b"rg_exact", 1))
    yield
    _lib.check(_lib.lib().hdb_option(b"rg_exact", 0))


def _rng(seed=7):
    return np.random.default_rng(seed)


def _rand(rng, shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


# ---------------------------------------------------------------- operators
@pytest.mark.parametrize("bc", ["sommerfeld", "dirichlet"])
@pytest.mark.parametrize("level", [1, 2, 3, 4])
@pytest.mark.parametrize("kind", ["A", "M"])
def test_operator_bitexact_vs_reference(bc, level, kind, exact_taps):
    g = golden("operators.npz")
    hier = hdb.mp1_problem(k=25.0, n=33, ml=4, boundary=bc).hierarchy
    op = hdb.helmholtz_operator(hier, level) if kind == "A" else hdb.cslp_operator(hier, level, beta2=0.35)
    got = op.apply(g[f"mp1_{bc}_L{level}_{kind}_u"])
    np.testing.assert_array_equal(got, g[f"mp1_{bc}_L{level}_{kind}_v"])


def test_operator_heterogeneous_and_mixed_bc_bitexact(exact_taps):
    g = golden("operators.npz")
    hier = hdb.wedge_problem(f=4.0, nx=25, ml=3).hierarchy
    for l in (1, 2, 3):
        op = hdb.helmholtz_operator(hier, l)
        np.testing.assert_array_equal(op.apply(g[f"wedge_L{l}_A_u"]), g[f"wedge_L{l}_A_v"])
    np.testing.assert_array_equal(hdb.helmholtz_operator(hier, 1).diagonal(), g["wedge_L1_diag"])
    vel = hdb.VelocityModel(kind="wedge", layers=[(-400.0, -200.0, 2000.0), (-800.0, -600.0, 1500.0),
                                                  (0.0, 0.0, 3000.0)])
    hier = hdb.build_hierarchy(((0.0, 600.0), (-1000.0, 0.0)), h=25.0, ml=3, velocity=vel, f=6.0,
                               boundary=("dirichlet", "sommerfeld", "sommerfeld", "dirichlet"))
    for l in (1, 2, 3):
        op = hdb.cslp_operator(hier, l, beta2=0.5)
        np.testing.assert_array_equal(op.apply(g[f"mixed_L{l}_M_u"]), g[f"mixed_L{l}_M_v"])


@pytest.mark.parametrize("shape", [(129, 129), (65, 257), (257, 33), (300, 270), (289, 513)])
@pytest.mark.parametrize("level", [1, 2, 3])
def test_operator_bitexact_vs_oracle_larger(shape, level, exact_taps):
    rng = _rng(level)
    ny, nx = shape
    ksq = 400.0 + 300.0 * rng.random((ny, nx))
    lv = hdb.level_kernels(level)
    bnd = ("sommerfeld", "dirichlet", "sommerfeld", "sommerfeld")
    op = hdb.LevelOperator(level, nx, ny, 1.0 / 128, ksq, bnd, lv[0], lv[1], shift=complex(1.0, 0.5),
                           level_scale=4.0 ** (level - 1))
    lt, ld, mt, md, _ = oracle.level_kernels(level)
    ref = oracle.CpuLevelOp(nx, ny, 1.0 / 128, ksq, bnd, lt, ld, mt, md, shift=complex(1.0, 0.5),
                            level_scale=4.0 ** (level - 1))
    u = _rand(rng, shape)
    np.testing.assert_array_equal(op.apply(u), ref.apply(u))
    b = _rand(rng, shape)
    np.testing.assert_array_equal(op.residual(b, u), b - ref.apply(u))


@pytest.mark.parametrize("level", [2, 3])
@pytest.mark.parametrize("bnd", [("sommerfeld",) * 4, ("dirichlet", "sommerfeld", "dirichlet", "sommerfeld")])
def test_operator_uniform_k_large_bitexact(level, bnd, exact_taps):
    """Constant-k^2 level on a grid large enough for the register-blocked tile
    kernel (interior tiles take the precomputed-coefficient fast path)."""
    rng = _rng(40 + level)
    ny, nx = 321, 290
    ksq = np.full((ny, nx), 523.25)
    lv = hdb.level_kernels(level)
    op = hdb.LevelOperator(level, nx, ny, 1.0 / 96, ksq, bnd, lv[0], lv[1], shift=complex(1.0, 0.5),
                           level_scale=4.0 ** (level - 1))
    lt, ld, mt, md, _ = oracle.level_kernels(level)
    ref = oracle.CpuLevelOp(nx, ny, 1.0 / 96, ksq, bnd, lt, ld, mt, md, shift=complex(1.0, 0.5),
                            level_scale=4.0 ** (level - 1))
    u = _rand(rng, (ny, nx))
    np.testing.assert_array_equal(op.apply(u), ref.apply(u))
    b = _rand(rng, (ny, nx))
    np.testing.assert_array_equal(op.residual(b, u), b - ref.apply(u))


@pytest.mark.parametrize("shape", [(129, 129), (300, 270), (289, 513), (1025, 1025), (65, 257)])
@pytest.mark.parametrize("level", [2, 3, 5])
@pytest.mark.parametrize("bnd", [("sommerfeld",) * 4, ("dirichlet", "sommerfeld", "dirichlet", "sommerfeld")])
@pytest.mark.parametrize("uniform", [False, True])
def test_separable_galerkin_vs_exact_taps(shape, level, bnd, uniform):
    """K2: the separable 1D-pass form of the radius-2/3 level operators (the
    default) against the reference's exact row-major tap sum (oracle, bit-exact
    with contract_general) on heterogeneous and constant k^2, both closures:
    a different association of the same products, held to 8 ulp of the field's
    max (measured <= 4.5 ulp; cancellation in the Laplacian part).  Dirichlet identity rows are exact."""
    rng = _rng(7 * level + shape[0])
    ny, nx = shape
    ksq = np.full((ny, nx), 611.5) if uniform else 400.0 + 300.0 * rng.random((ny, nx))
    lv = hdb.level_kernels(level)
    op = hdb.LevelOperator(level, nx, ny, 1.0 / 128, ksq, bnd, lv[0], lv[1], shift=complex(1.0, 0.5),
                           level_scale=4.0 ** (level - 1))
    assert op.separable_factors() is not None
    lt, ld, mt, md, _ = oracle.level_kernels(level)
    ref = oracle.CpuLevelOp(nx, ny, 1.0 / 128, ksq, bnd, lt, ld, mt, md, shift=complex(1.0, 0.5),
                            level_scale=4.0 ** (level - 1))
    u, b = _rand(rng, shape), _rand(rng, shape)
    au = ref.apply(u)
    got = op.apply(u)
    assert np.abs(got - au).max() <= 8 * np.finfo(float).eps * np.abs(au).max()
    res = op.residual(b, u)
    assert np.abs(res - (b - au)).max() <= 8 * np.finfo(float).eps * np.abs(b - au).max()
    if bnd[0] == "dirichlet":
        np.testing.assert_array_equal(got[:, 0], u[:, 0])
        np.testing.assert_array_equal(got[0, :], u[0, :])


@pytest.mark.parametrize("shape", [(1025, 1025), (600, 2050), (2049, 517), (777, 1111)])
@pytest.mark.parametrize("bnd", [("sommerfeld",) * 4, ("dirichlet", "sommerfeld", "dirichlet", "sommerfeld")])
def test_strip_kernels_bitexact_vs_oracle(shape, bnd):
    """5-point apply, residual and both Jacobi forms on grids >= 512^2 (the
    column-strip kernels: balanced one-wave row ranges, ragged last strip,
    global first/last rows on the closure path) against the oracle, bit for bit."""
    rng = _rng(shape[0] + 3 * shape[1])
    ny, nx = shape
    ksq = 900.0 + 500.0 * rng.random((ny, nx))
    ksq[ny // 2: ny // 2 + 40] = 700.0  # constant band: Jacobi reciprocal reuse
    op = hdb.radius1_operator(nx, ny, 1.0 / 256, ksq, bnd, complex(1.0, 0.5))
    ref = oracle.CpuLevelOp(nx, ny, 1.0 / 256, ksq, bnd, *oracle.level_kernels(1)[:4], shift=complex(1.0, 0.5),
                            level_scale=1.0)
    u, b = _rand(rng, shape), _rand(rng, shape)
    au = ref.apply(u)
    np.testing.assert_array_equal(op.apply(u), au)
    np.testing.assert_array_equal(op.residual(b, u), b - au)
    np.testing.assert_array_equal(op.jacobi(u, b, 0.8), ref.jacobi(u, b, 0.8))
    np.testing.assert_array_equal(op.jacobi(None, b, 0.8), ref.jacobi(np.zeros(shape, complex), b, 0.8))


@pytest.mark.parametrize("shape", [(1025, 1025), (513, 2049), (2049, 577), (129, 129), (9, 5), (3, 3)])
@pytest.mark.parametrize("bnd", [("sommerfeld",) * 4, ("dirichlet", "sommerfeld", "dirichlet", "sommerfeld"),
                                 ("dirichlet",) * 4])
def test_fused_residual_restrict_bitexact_vs_oracle(shape, bnd):
    """Fused multigrid coarse right-hand side Z^T (b - M x) with the coarse Dirichlet
    rows zeroed (mg.py:116-117), one pass without storing the residual, against the
    oracle's residual followed by its restriction, bit for bit (interior strips on
    the sliding window, boundary strips on the closure path, ragged last strips)."""
    rng = _rng(7 * shape[0] + shape[1])
    ny, nx = shape
    ksq = 900.0 + 500.0 * rng.random((ny, nx))
    op = hdb.radius1_operator(nx, ny, 1.0 / 256, ksq, bnd, complex(1.0, 0.5))
    ref = oracle.CpuLevelOp(nx, ny, 1.0 / 256, ksq, bnd, *oracle.level_kernels(1)[:4], shift=complex(1.0, 0.5),
                            level_scale=1.0)
    u, b = _rand(rng, shape), _rand(rng, shape)
    mask = sum(1 << s for s in range(4) if bnd[s] == "dirichlet")
    want = oracle.restrict(b - ref.apply(u))
    if mask & 1:
        want[:, 0] = 0
    if mask & 2:
        want[:, -1] = 0
    if mask & 4:
        want[0, :] = 0
    if mask & 8:
        want[-1, :] = 0
    np.testing.assert_array_equal(op.residual_restrict(b, u, mask), want)
    # and equal to the library's own unfused pair
    np.testing.assert_array_equal(op.residual_restrict(b, u, 0), hdb.restrict_array(op.residual(b, u)))


@pytest.mark.parametrize("shape", [(1025, 1025), (600, 2050), (129, 129)])
@pytest.mark.parametrize("bnd", [("sommerfeld",) * 4, ("dirichlet", "sommerfeld", "dirichlet", "sommerfeld")])
def test_jacobi_with_folded_sum_bitexact_vs_oracle(shape, bnd):
    """The last post-smoothing sweep with the A-DEF1 sum folded in (mg.py:122 +
    madp.py:327): both outputs equal the oracle's sweep and sweep + t bit for bit."""
    rng = _rng(shape[0] + 5 * shape[1])
    ny, nx = shape
    ksq = 900.0 + 500.0 * rng.random((ny, nx))
    ksq[ny // 2: ny // 2 + 40] = 700.0
    op = hdb.radius1_operator(nx, ny, 1.0 / 256, ksq, bnd, complex(1.0, 0.5))
    ref = oracle.CpuLevelOp(nx, ny, 1.0 / 256, ksq, bnd, *oracle.level_kernels(1)[:4], shift=complex(1.0, 0.5),
                            level_scale=1.0)
    x, b, t = _rand(rng, shape), _rand(rng, shape), _rand(rng, shape)
    want = ref.jacobi(x, b, 0.8)
    got, gsum = op.jacobi_add(x, b, t, 0.8)
    np.testing.assert_array_equal(got, want)
    np.testing.assert_array_equal(gsum, want + t)


@pytest.mark.parametrize("shape", [(129, 129), (600, 300), (1025, 1025)])
@pytest.mark.parametrize("bnd", [("sommerfeld",) * 4, ("dirichlet", "sommerfeld", "dirichlet", "sommerfeld")])
def test_fused_residual_norms_vs_oracle(shape, bnd):
    """One-pass (||b - A u||, ||b||) (the MG guard kernel, no residual stored)
    against the oracle's bit-exact residual, normed in numpy: the sums differ
    only in summation order (rel. 1e-13)."""
    rng = _rng(sum(shape))
    ny, nx = shape
    ksq = 900.0 + 500.0 * rng.random((ny, nx))
    ksq[: ny // 3] = 700.0  # constant band: exercises the interior fast path too
    op = hdb.radius1_operator(nx, ny, 1.0 / 256, ksq, bnd, complex(1.0, 0.5))
    ref = oracle.CpuLevelOp(nx, ny, 1.0 / 256, ksq, bnd, *oracle.level_kernels(1)[:4], shift=complex(1.0, 0.5),
                            level_scale=1.0)
    u, b = _rand(rng, shape), _rand(rng, shape)
    rn, bn = op.residual_norms(b, u)
    r = b - ref.apply(u)
    assert abs(rn - np.linalg.norm(r)) <= 1e-13 * np.linalg.norm(r)
    assert abs(bn - np.linalg.norm(b)) <= 1e-13 * np.linalg.norm(b)


def test_zero_in_zero_out_and_edge_shapes():
    for shape in ((3, 3), (5, 3), (3, 9)):
        ny, nx = shape
        op = hdb.radius1_operator(nx, ny, 0.1, np.full(shape, 4.0), ("sommerfeld",) * 4, complex(1, 0.5))
        assert not np.asarray(op.apply(np.zeros(shape, complex))).any()


# ---------------------------------------------------------------- transfers
@pytest.mark.parametrize("shape", [(17, 17), (41, 25), (9, 65)])
def test_transfers_bitexact_vs_reference(shape):
    g = golden("transfers.npz")
    ny, nx = shape
    np.testing.assert_array_equal(hdb.restrict_array(g[f"r_{ny}x{nx}_in"]), g[f"r_{ny}x{nx}_out"])
    np.testing.assert_array_equal(hdb.prolong_array(g[f"p_{ny}x{nx}_in"], shape), g[f"p_{ny}x{nx}_out"])


def test_transfers_large_vs_oracle_and_adjoint():
    rng = _rng(3)
    v = _rand(rng, (1025, 513))
    c = _rand(rng, (513, 257))
    np.testing.assert_array_equal(hdb.restrict_array(v), oracle.restrict(v))
    np.testing.assert_array_equal(hdb.prolong_array(c, (1025, 513)), oracle.prolong(c, (1025, 513)))
    # size-independent property: <R v, w> = <v, P w> / 4 (transfers.py:1-10)
    lhs = np.sum(np.asarray(hdb.restrict_array(v)) * c)
    rhs = np.sum(v * np.asarray(hdb.prolong_array(c, (1025, 513)))) / 4.0
    assert abs(lhs - rhs) <= 1e-12 * abs(rhs)


@pytest.mark.parametrize("shape", [(2049, 2561), (4097, 2049)])
def test_transfers_tma_sizes_bitexact_vs_oracle(shape):
    """Grids large enough for the TMA-staged transfer kernels (tensor-map zero
    fill at the edges, partial CTA column blocks and strips): bit-identical to
    the oracle, overwrite and accumulate forms, and with coarse zero rows."""
    rng = _rng(sum(shape))
    ny, nx = shape
    cy, cx = (ny - 1) // 2 + 1, (nx - 1) // 2 + 1
    v = _rand(rng, shape)
    c = _rand(rng, (cy, cx))
    base = _rand(rng, shape)
    r = oracle.restrict(v)
    np.testing.assert_array_equal(hdb.restrict_array(v), r)
    rz = r.copy()
    rz[:, 0] = rz[:, -1] = rz[0, :] = rz[-1, :] = 0  # zero_mask 15: coarse Dirichlet rows
    np.testing.assert_array_equal(hdb.restrict_array(v, zero_mask=15), rz)
    p = oracle.prolong(c, shape)
    np.testing.assert_array_equal(hdb.prolong_array(c, shape), p)
    np.testing.assert_array_equal(hdb.prolong_array(c, shape, base=base), base + p)


# ------------------------------------------------------------ jacobi / MG
@pytest.mark.parametrize("name", ["mp1s65", "mp1d65div", "poisson65", "wedge145"])
def test_jacobi_bitexact_and_vcycle(name):
    g = golden("multigrid.npz")
    probs = {"mp1s65": lambda: hdb.mp1_problem(k=50.0, n=65, ml=2),
             "mp1d65div": lambda: hdb.mp1_problem(k=20.0, n=65, ml=2, boundary="dirichlet"),
             "poisson65": lambda: hdb.mp1_problem(k=1e-12, n=65, ml=2, boundary="dirichlet"),
             "wedge145": lambda: hdb.wedge_problem(f=20.0, nx=145, ml=4)}
    hier = probs[name]().hierarchy
    lv = hier.level(1)
    mg = hdb.CslpMultigrid(lv.nx, lv.ny, lv.h, hier.ksq_at(1), hier.boundary, beta2=float(g[f"{name}_beta2"]))
    assert mg.depth == int(g[f"{name}_depth"])
    b = g[f"{name}_b"]
    np.testing.assert_array_equal(mg.levels[0].op.jacobi(g[f"{name}_jx0"], b, 0.8), g[f"{name}_jx1"])
    if bool(g[f"{name}_diverged"]):
        with pytest.raises(hdb.MgDivergence):
            mg.vcycle(b)
    else:
        x = mg.vcycle(b)
        ref = g[f"{name}_x"]
        # coarsest solve: device inverse GEMV vs LAPACK LU -> rounding-level only
        assert np.abs(x - ref).max() <= 1e-12 * np.abs(ref).max()


def test_vcycle_linear_and_zero():
    hier = hdb.mp1_problem(k=50.0, kh=0.625, ml=2).hierarchy
    lv = hier.level(1)
    mg = hdb.CslpMultigrid(lv.nx, lv.ny, lv.h, hier.ksq_at(1), hier.boundary, beta2=0.5)
    rng = _rng(9)
    u, v = _rand(rng, lv.shape), _rand(rng, lv.shape)
    a, c = 1.3 - 0.7j, -0.4 + 2.1j
    lhs = mg.vcycle(a * u + c * v)
    rhs = a * mg.vcycle(u) + c * mg.vcycle(v)
    assert np.abs(lhs - rhs).max() <= 1e-12 * np.abs(rhs).max()
    assert not np.asarray(mg.vcycle(np.zeros(lv.shape, complex))).any()


def test_vcycle_large_vs_oracle():
    # GMRES-fallback coarsest (> 4096 points): 1201x2001 wedge bottoms out at 76x126
    hier, _ = oracle.baseline_wedge_problem(40.0, h=0.5, ml=5)
    lv = hier.level(1)
    rng = _rng(11)
    b = _rand(rng, lv.shape)
    cpu = oracle.CpuMultigrid(lv.nx, lv.ny, lv.h, hier.ksq_at(1), hier.boundary, 0.5)
    gpu = hdb.CslpMultigrid(lv.nx, lv.ny, lv.h, hier.ksq_at(1), hier.boundary, beta2=0.5)
    assert gpu.depth == cpu.depth and gpu.levels[-1].lu is None
    xr = cpu.vcycle(b)
    xg = gpu.vcycle(b)
    assert np.linalg.norm(xg - xr) <= 1e-9 * np.linalg.norm(xr)


# ------------------------------------------------------------------- Krylov
def test_dot_vs_reference():
    g = golden("krylov.npz")
    d = hdb.reduce_dot(g["dot_u"], g["dot_v"])
    ref = complex(g["dot_uv"])
    assert abs(d - ref) <= 1e-13 * abs(ref)
    assert hdb.reduce_dot(np.array([[1.0 + 2.0j]]), np.array([[3.0 - 1.0j]])) == np.conj(1 + 2j) * (3 - 1j)


def test_fgmres_vs_reference():
    g = golden("krylov.npz")
    hier = hdb.mp1_problem(k=5.0, n=9, ml=2, boundary="dirichlet").hierarchy
    op = hdb.helmholtz_operator(hier, 1)
    x, rep = hdb.fgmres(op.apply, None, g["d9_b"], hdb.StopRule(1e-10, 100))
    assert rep.iterations == int(g["d9_its"])
    assert np.abs(np.array(rep.residual_history) - g["d9_hist"]).max() <= 1e-12
    assert np.abs(x - g["d9_x"]).max() <= 1e-9 * np.abs(g["d9_x"]).max()
    hier = hdb.mp1_problem(k=30.0, n=65, ml=3).hierarchy
    op = hdb.cslp_operator(hier, 1, beta2=0.5)
    x, rep = hdb.fgmres(op.apply, None, g["c65_b"], hdb.StopRule(0.1, 49))
    assert rep.iterations == int(g["c65_its"])
    assert np.abs(np.array(rep.residual_history) - g["c65_hist"]).max() <= 1e-12
    assert np.linalg.norm(x - g["c65_x"]) <= 1e-10 * np.linalg.norm(g["c65_x"])


def test_fgmres_python_callables_and_x0():
    rng = _rng(5)
    hier = hdb.mp1_problem(k=5.0, n=9, ml=2, boundary="dirichlet").hierarchy
    op = hdb.helmholtz_operator(hier, 1)
    b = _rand(rng, (9, 9))
    D = np.asarray(op.diagonal())
    Mfn = lambda u: u / D  # noqa: E731  host callable
    x1, r1 = hdb.fgmres(op.apply, Mfn, b, hdb.StopRule(1e-9, 40))
    x2, r2 = hdb.gmres(lambda u: np.asarray(op.apply(u)), Mfn, b, hdb.StopRule(1e-9, 40))
    assert r1.iterations == r2.iterations
    assert np.abs(x1 - x2).max() <= 1e-12 * np.abs(x1).max()
    x3, r3 = hdb.fgmres(op.apply, None, b, hdb.StopRule(1e-10, 100), x0=x1)
    assert r3.converged and np.abs(np.asarray(op.apply(x3)) - b).max() <= 1e-7 * np.abs(b).max()
    # zero rhs -> 0 iterations; tol 1 -> one iteration; cap -> unconverged
    x, r = hdb.fgmres(op.apply, None, np.zeros((9, 9), complex), hdb.StopRule(1e-10, 5))
    assert r.iterations == 0 and r.converged and not np.asarray(x).any()
    _, r = hdb.fgmres(op.apply, None, b, hdb.StopRule(1.0, 50))
    assert r.iterations == 1 and r.converged
    _, r = hdb.fgmres(op.apply, None, b, hdb.StopRule(1e-12, 3))
    assert r.iterations == 3 and not r.converged and len(r.residual_history) == 4


def test_fgmres_matches_oracle_random():
    rng = _rng(13)
    hier = hdb.mp1_problem(k=40.0, n=129, ml=3).hierarchy
    op = hdb.cslp_operator(hier, 1, beta2=0.5)
    ohier, _ = oracle.mp1_problem(40.0, 129, 3)
    oop = oracle.cslp_op(ohier, 1, 0.5)
    b = _rand(rng, op.shape)
    x, rep = hdb.fgmres(op.apply, None, b, hdb.StopRule(1e-3, 80))
    xo, repo = oracle.fgmres(oop.apply, None, b, oracle.Stop(1e-3, 80), dot=oracle.reduce_dot)
    assert rep.iterations == repo.iterations
    assert np.abs(np.array(rep.residual_history) - np.array(repo.residual_history)).max() <= 1e-12
    assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)


# -------------------------------------------------------------- full solves
def _solve_case(name):
    if name == "c1s":
        return hdb.mp1_problem(k=50.0, n=129, ml=2, boundary="sommerfeld")
    if name == "wedge20":
        return hdb.wedge_problem(f=20.0, nx=145, ml=4)
    if name == "c1_cap20":
        return hdb.mp1_problem(k=50.0, n=129, ml=2, boundary="dirichlet")
    raise KeyError(name)


@pytest.mark.parametrize("name", ["c1s", "wedge20"])
def test_full_solve_vs_reference(name):
    """BASELINE parity bar: outer its +-1, history within 1e-9, solution within 1e-8 rel L2
    (these configs' oracle noise floors are ~1e-13, tests/golden/solve_*.npz floor_*)."""
    g = golden(f"solve_{name}.npz")
    prob = _solve_case(name)
    cfg = hdb.preset("MADP", prob.hierarchy)
    with hdb.MadpSolver(prob.hierarchy, cfg) as s:
        u, rep = s.solve(prob.rhs)
    x = u.grid_view(prob.hierarchy)
    assert abs(rep.outer_iterations - int(g["outer_iterations"])) <= 1
    h = np.array(rep.residual_history)
    hr = g["residual_history"]
    n = min(len(h), len(hr))
    assert np.abs(h[:n] - hr[:n]).max() <= 1e-9
    assert np.linalg.norm(x - g["solution"]) <= 1e-8 * np.linalg.norm(g["solution"])
    assert rep.converged == bool(g["converged"])
    ref_cycles = {int(k): v for k, v in json.loads(str(g["cycle_iters"])).items()}
    for l, v in ref_cycles.items():
        assert rep.cycle_iters[l] == v  # per-level inner iteration counts identical


def test_config1_dirichlet_first_20_outer_iterations():
    """BASELINE configs[0] as written (chaotic, never converges in the reference):
    the first 20 outer iterations against the reference's 20-iteration record."""
    g = golden("solve_c1_cap20.npz")
    prob = _solve_case("c1_cap20")
    cfg = hdb.preset("MADP", prob.hierarchy, outer_stop=hdb.StopRule(1e-6, 20))
    with hdb.MadpSolver(prob.hierarchy, cfg) as s:
        _, rep = s.solve(prob.rhs)
    assert rep.outer_iterations == int(g["outer_iterations"]) == 20
    h, hr = np.array(rep.residual_history), g["residual_history"]
    # the reference itself moves by 2.3e-3 within these 20 iterations under a 1e-15 rhs
    # perturbation (4e-7 already at iteration 2): each iteration is held to 10x the
    # reference's own drift up to that iteration (solve_c1_full.npz floor_hist)
    assert np.abs(h[:2] - hr[:2]).max() <= 1e-9
    assert np.all(np.abs(h - hr) <= 10 * _floor_envelope(golden("solve_c1_full.npz"))[:21] + 1e-12)


def _floor_envelope(g):
    """Running max of the reference's |h_i - h'_i| against its 1e-15-perturbed twin."""
    return np.maximum.accumulate(np.abs(g["residual_history"] - g["floor_hist"]))


def test_config1_dirichlet_full_150_iteration_stall():
    """BASELINE configs[0] as written, run like the reference to its cap: 150 outer
    iterations, not converged (madp.py:112), against the reference's full record
    (tests/golden/solve_c1_full.npz).  The reference is chaotic here (its own history
    moves by 2.3e-3 and its solution by 1.0e-2 under a 1e-15 rhs perturbation), so
    the history and solution are held to 10x that floor and the early history to
    the BASELINE bar."""
    g = golden("solve_c1_full.npz")
    prob = _solve_case("c1_cap20")
    with hdb.MadpSolver(prob.hierarchy, hdb.preset("MADP", prob.hierarchy)) as s:
        u, rep = s.solve(prob.rhs)
    assert rep.outer_iterations == int(g["outer_iterations"]) == 150
    assert not rep.converged and not bool(g["converged"])
    h, hr = np.array(rep.residual_history), g["residual_history"]
    assert len(h) == len(hr) == 151
    assert np.abs(h[:2] - hr[:2]).max() <= 1e-9
    assert np.all(np.abs(h - hr) <= 10 * _floor_envelope(g) + 1e-12)
    hb, xb = parity_bar(g)
    st = int(g["solution_stride"])
    xs = u.grid_view(prob.hierarchy)[::st, ::st]
    assert np.linalg.norm(xs - g["solution_sub"]) <= xb * np.linalg.norm(g["solution_sub"])
    # the stall level: the reference ends at 7.9e-5 (its perturbed twin at 3.7e-6)
    assert 1e-6 < rep.final_relres < 1e-3


def test_preconditioner_apply_vs_oracle():
    prob = hdb.mp1_problem(k=50.0, n=129, ml=3, boundary="sommerfeld")
    cfg = hdb.preset("MADP", prob.hierarchy)
    ohier, _ = oracle.mp1_problem(50.0, 129, 3, "sommerfeld")
    pols, outer = oracle.madp_preset(ohier)
    osolver = oracle.CpuMadpSolver(ohier, pols, outer)
    osolver._reset()
    v = _rand(_rng(21), prob.hierarchy.level(1).shape)
    ref = osolver.precond(1, v)
    with hdb.MadpSolver(prob.hierarchy, cfg) as s:
        got = s.apply_preconditioner(1, v)
    assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref)


def test_solve_device_tensor_roundtrip():
    import torch
    prob = hdb.mp1_problem(k=20.0, n=65, ml=3, boundary="sommerfeld")
    cfg = hdb.preset("MADP", prob.hierarchy)
    b = torch.from_numpy(prob.rhs.grid_view(prob.hierarchy).copy()).cuda()
    with hdb.MadpSolver(prob.hierarchy, cfg) as s:
        x, rep = s.solve(b)
        xh, reph = s.solve(prob.rhs)
    assert x.is_cuda and rep.converged
    np.testing.assert_array_equal(x.cpu().numpy(), xh.grid_view(prob.hierarchy))
    assert rep.residual_history == reph.residual_history


def test_solve_bit_reproducible_run_to_run():
    """Repeated solves are bit-identical (fixed-order reductions; the TMA rings of
    the transfer and MGS kernels release a stage only after its values are
    consumed).  2049^2 so that the TMA-staged transfers and the TMA-fed MGS
    step are on the path; config 2 itself: profiles/r01d_determinism.txt."""
    import torch
    prob = hdb.mp1_problem(k=100.0, n=2049, ml=6, boundary="sommerfeld")
    cfg = hdb.preset("MADP", prob.hierarchy)
    b = torch.from_numpy(prob.rhs.grid_view(prob.hierarchy).copy()).cuda()
    x = torch.empty_like(b)
    with hdb.MadpSolver(prob.hierarchy, cfg) as s:
        hashes, hists = [], []
        for _ in range(3):
            rep = s.solve_device(b, x)
            torch.cuda.synchronize()
            hashes.append(hash(x.cpu().numpy().tobytes()))
            hists.append(tuple(rep.residual_history))
        # host-buffer API (pageable numpy in and out: the staged, chunked copy path, 67 MB)
        u, reph = s.solve(np.ascontiguousarray(prob.rhs.grid_view(prob.hierarchy)))
    assert rep.converged
    assert len(set(hashes)) == 1 and len(set(hists)) == 1
    np.testing.assert_array_equal(u.grid_view(prob.hierarchy), x.cpu().numpy())
    assert tuple(reph.residual_history) == hists[0]


def test_transfers_repeatable_under_load():
    """The TMA-staged transfers give the same bits on every call (a stage refilled
    under a pending shared load showed up as ~1 wrong block in 200 calls)."""
    import torch
    rng = _rng(21)
    n = 4097
    nc = (n - 1) // 2 + 1
    u = torch.from_numpy(_rand(rng, (n, n))).cuda()
    base = torch.from_numpy(_rand(rng, (n, n))).cuda()
    c = torch.from_numpy(_rand(rng, (nc, nc))).cuda()
    ref_r = hdb.restrict_array(u).clone()
    ref_p = hdb.prolong_array(c, (n, n), base=base).clone()
    for _ in range(12):
        assert torch.equal(hdb.restrict_array(u), ref_r)
        assert torch.equal(hdb.prolong_array(c, (n, n), base=base), ref_p)


def test_device_resident_and_launch_paths_agree():
    """HDB_SMALL_N=0 forces the launch-driven Krylov path on every level (with
    the MGS chain, the cooperative MGS step, or the device-driven GMRES loop);
    every engine must give the same counts and histories to rounding."""
    import subprocess
    import sys
    code = ("import json,sys; sys.path.insert(0,'.'); import paper_2412_04980_b200 as h;"
            "p=h.wedge_problem(f=20.0,nx=145,ml=4); s=h.MadpSolver(p.hierarchy,h.preset('MADP',p.hierarchy));"
            "u,r=s.solve(p.rhs); print(json.dumps([r.outer_iterations,r.residual_history,r.cslp_iters[4]]))")
    outs = []
    launch = {"HDB_SMALL_N": "0", "HDB_GRID_N": "0"}
    for env in (launch,                                                   # host-driven, MGS launch chain
                dict(launch, HDB_COOP_MGS_N="300", HDB_GMRES_DEV="0"),   # host-driven, cooperative MGS
                dict(launch, HDB_COOP_MGS_N="300"),                      # device-driven GMRES
                {}):                                                     # device-resident kernels
        import os
        e = dict(os.environ, **env)
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=e, cwd=ROOT_DIR)
        assert r.returncode == 0, r.stderr
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    i0, h0, c0 = outs[0]
    for i1, h1, c1 in outs[1:]:
        assert i0 == i1 and c0 == c1
        assert np.abs(np.array(h0) - np.array(h1)).max() <= 1e-12


def test_lowsync_mgs_step_matches_mgs_order():
    """The one-launch MGS step of large levels in its low-synchronisation form
    (h = (I + L)^{-1} V^H w, two grid reductions per Arnoldi step) against the
    reference's coefficient-by-coefficient order (hdb_option("mgs_ls", 0)) and
    the oracle's fgmres, on a 1025^2 CSLP level (7099 points per CTA: the form
    applies) with GMRES(0.1, 40) and a tighter GMRES(1e-6, 60)."""
    import ctypes as C
    import torch
    from paper_2412_04980_b200 import _lib
    L = _lib.lib()
    prob = hdb.mp1_problem(k=100.0, n=1025, ml=3)
    op = hdb.cslp_operator(prob.hierarchy, 1, 0.5)
    rng = _rng(5)
    bh = _rand(rng, op.shape)
    b = torch.from_numpy(bh).cuda()
    res = {}
    for ls in (1, 0):
        _lib.check(L.hdb_option(b"mgs_ls", ls))
        for tol, cap in ((0.1, 40), (1e-6, 60)):
            x = torch.empty_like(b)
            its, rel = C.c_int(), C.c_double()
            _lib.check(L.hdb_op_gmres(op.handle, b.data_ptr(), x.data_ptr(), tol, cap, -1, C.byref(its), C.byref(rel)))
            res[(ls, tol)] = (its.value, rel.value, x.cpu().numpy())
    _lib.check(L.hdb_option(b"mgs_ls", 1))
    for tol in (0.1, 1e-6):
        (i1, r1, x1), (i0, r0, x0) = res[(1, tol)], res[(0, tol)]
        assert i1 == i0
        assert abs(r1 - r0) <= 1e-9 * max(r0, 1e-300) + 1e-14
        assert np.linalg.norm(x1 - x0) <= 1e-10 * np.linalg.norm(x0)
    oop = oracle.cslp_op(oracle.mp1_problem(100.0, 1025, 3)[0], 1, 0.5)
    xo, repo = oracle.fgmres(oop.apply, None, bh, oracle.Stop(0.1, 40), dot=oracle.reduce_dot)
    i1, r1, x1 = res[(1, 0.1)]
    assert i1 == repo.iterations
    assert np.linalg.norm(x1 - xo) <= 1e-10 * np.linalg.norm(xo)


def test_lowsync_hbm_streaming_step_matches_mgs_chain():
    """The HBM-streaming low-synchronisation MGS step (levels whose w does not fit on
    chip; forced here on a 1025^2 level by disabling the one-launch forms) against
    the fused MGS chain (HDB_LSH_N=0) and the oracle: GMRES(1e-8, 40) on a CSLP level."""
    import os
    import subprocess
    import sys
    code = ("import sys,json; sys.path.insert(0,'.'); import numpy as np, paper_2412_04980_b200 as h;"
            "p=h.mp1_problem(k=100.0,n=1025,ml=3); op=h.cslp_operator(p.hierarchy,1,0.5);"
            "rng=np.random.default_rng(5); b=rng.standard_normal(op.shape)+1j*rng.standard_normal(op.shape);"
            "x,r=h.fgmres(op.apply,None,b,h.StopRule(1e-8,40)); np.save(sys.argv[1],x);"
            "print(json.dumps([r.iterations,r.residual_history,r.final_relres]))")
    outs = []
    for i, env in enumerate(({"HDB_COOP_MGS_N": "1000000000000"},
                             {"HDB_COOP_MGS_N": "1000000000000", "HDB_LSH_N": "0"})):
        path = f"/tmp/hdb_lsh_{i}.npy"
        r = subprocess.run([sys.executable, "-c", code, path], capture_output=True, text=True,
                           env=dict(os.environ, **env), cwd=ROOT_DIR)
        assert r.returncode == 0, r.stderr
        its, hist, fin = json.loads(r.stdout.strip().splitlines()[-1])
        outs.append((its, np.array(hist), fin, np.load(path)))
    (i0, h0, f0, x0), (i1, h1, f1, x1) = outs
    assert i0 == i1
    assert np.abs(h0 - h1).max() <= 1e-12
    assert np.linalg.norm(x0 - x1) <= 1e-10 * np.linalg.norm(x1)
    oop = oracle.cslp_op(oracle.mp1_problem(100.0, 1025, 3)[0], 1, 0.5)
    rng = np.random.default_rng(5)
    b = rng.standard_normal(oop.shape) + 1j * rng.standard_normal(oop.shape)
    xo, repo = oracle.fgmres(oop.apply, None, b, oracle.Stop(1e-8, 40), dot=oracle.reduce_dot)
    assert i0 == repo.iterations
    assert np.abs(h0 - np.array(repo.residual_history)).max() <= 1e-12
    assert np.linalg.norm(x0 - xo) <= 1e-9 * np.linalg.norm(xo)


def test_streaming_lowsync_step_on_levels_beyond_the_one_launch_form():
    """Levels whose w slice exceeds the one-launch low-synchronisation step (> 7168 points per
    CTA: config 5's 2049^2 and config 4's 3065 x 1001 CSLP levels) can run the HBM-streaming form
    of the same algorithm (hdb_option "lsh_prefer"), host-driven (mode -1) and inside the
    device-driven GMRES loop (mode -2): same iteration counts and solutions as the MGS-order
    kernels (mgs_ls = 0), on a
    1537^2 radius-2 CSLP level with GMRES(0.1, 30) and GMRES(1e-6, 45)."""
    import ctypes as C
    import torch
    from paper_2412_04980_b200 import _lib
    L = _lib.lib()
    prob = hdb.mp1_problem(k=150.0, n=3073, ml=3)
    op = hdb.cslp_operator(prob.hierarchy, 2, 0.5)
    assert op.npoints > 148 * 7168
    rng = _rng(11)
    b = torch.from_numpy(_rand(rng, op.shape)).cuda()
    res = {}
    for ls in (1, 0):
        _lib.check(L.hdb_option(b"mgs_ls", ls))
        _lib.check(L.hdb_option(b"lsh_prefer", ls))
        for mode in (-1, -2):
            for tol, cap in ((0.1, 30), (1e-6, 45)):
                x = torch.empty_like(b)
                its, rel = C.c_int(), C.c_double()
                _lib.check(L.hdb_op_gmres(op.handle, b.data_ptr(), x.data_ptr(), tol, cap, mode, C.byref(its),
                                          C.byref(rel)))
                res[(ls, mode, tol)] = (its.value, rel.value, x.cpu().numpy())
    _lib.check(L.hdb_option(b"mgs_ls", 1))
    _lib.check(L.hdb_option(b"lsh_prefer", 0))
    for tol in (0.1, 1e-6):
        i0, r0, x0 = res[(0, -1, tol)]
        for key in ((1, -1, tol), (1, -2, tol), (0, -2, tol)):
            i1, r1, x1 = res[key]
            assert i1 == i0, key
            assert abs(r1 - r0) <= 1e-9 * max(r0, 1e-300) + 1e-13, key
            assert np.linalg.norm(x1 - x0) <= 1e-10 * np.linalg.norm(x0), key


ROOT_DIR = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))


def test_config2_analogue_vs_reference():
    """k=100, 1025^2, 6 levels (BASELINE configs[1] physics at 1/16 size).  The
    reference's own noise floor here is ~1e-5 in the history, so the
    history is held to that floor and the outer count to +-1."""
    g = golden("solve_c2a.npz")
    prob = hdb.mp1_problem(k=100.0, n=1025, ml=6, boundary="sommerfeld")
    with hdb.MadpSolver(prob.hierarchy, hdb.preset("MADP", prob.hierarchy)) as s:
        u, rep = s.solve(prob.rhs)
    assert abs(rep.outer_iterations - int(g["outer_iterations"])) <= 1
    h, hr = np.array(rep.residual_history), g["residual_history"]
    n = min(len(h), len(hr))
    floor = max(float(g["floor_hist_abs"]), 1e-9)
    assert np.abs(h[:n] - hr[:n]).max() <= 10 * floor
    st = int(g["solution_stride"])
    xs = u.grid_view(prob.hierarchy)[::st, ::st]
    ref = g["solution_sub"]
    assert np.linalg.norm(xs - ref) <= max(10 * float(g["floor_sol_rel"]), 1e-8) * np.linalg.norm(ref)


def test_config5_reduced_instance_vs_reference():
    """BASELINE configs[4] (weak scaling) at reduced size: two stacked unit squares,
    h = 1/1024 (1025 x 2049 points), k^3 h^2 = 0.5, 5 levels -- the reference's own run
    (tests/golden/solve_c5s.npz with its noise floor): outer count +-1, history and
    solution within the BASELINE bar or 10x the reference's floor."""
    from paper_2412_04980_b200 import models
    g = golden("solve_c5s.npz")
    hbar, xbar = parity_bar(g)
    prob = models.c5_problem(P=2, ml=5, cells=1024)
    assert prob.hierarchy.level(1).shape == (2049, 1025)
    with hdb.MadpSolver(prob.hierarchy, hdb.preset("MADP", prob.hierarchy)) as s:
        u, rep = s.solve(prob.rhs)
    assert rep.converged and abs(rep.outer_iterations - int(g["outer_iterations"])) <= 1
    h, hr = np.array(rep.residual_history), g["residual_history"]
    n = min(len(h), len(hr))
    assert np.abs(h[:n] - hr[:n]).max() <= hbar
    st = int(g["solution_stride"])
    xs = u.grid_view(prob.hierarchy)[::st, ::st]
    assert np.linalg.norm(xs - g["solution_sub"]) <= xbar * np.linalg.norm(g["solution_sub"])


@pytest.mark.slow
def test_config2_full_vs_reference():
    """BASELINE configs[1] at full size (4097^2, 7 levels) against the reference's own
    27-minute run: outer count +-1; history and solution within 10x the reference's
    own config-2 noise floor (its 1e-15-perturbed twin run: 5.8e-6 / 3.9e-7;
    measured GPU deltas 9.5e-7 / 5.5e-7, profiles/r02e_parity.json)."""
    g = golden("solve_c2.npz")
    prob = hdb.mp1_problem(k=200.0, n=4097, ml=7, boundary="sommerfeld")
    with hdb.MadpSolver(prob.hierarchy, hdb.preset("MADP", prob.hierarchy)) as s:
        u, rep = s.solve(prob.rhs)
    assert abs(rep.outer_iterations - int(g["outer_iterations"])) <= 1
    assert rep.converged and rep.final_relres <= 1e-6
    h, hr = np.array(rep.residual_history), g["residual_history"]
    n = min(len(h), len(hr))
    hb, xb = parity_bar(g)  # 10x the reference's config-2 floor: 5.8e-5 / 3.9e-6
    assert np.abs(h[:n] - hr[:n]).max() <= hb
    st = int(g["solution_stride"])
    xs = u.grid_view(prob.hierarchy)[::st, ::st]
    ref = g["solution_sub"]
    assert np.linalg.norm(xs - ref) <= xb * np.linalg.norm(ref)


# ------------------------------------------------------------- Bi-CGSTAB
def test_bicgstab_vs_reference():
    g = golden("krylov.npz")
    n = 17
    T = (2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)).astype(np.complex128)
    x, rep = hdb.bicgstab(lambda u: T @ u, None, g["bp_b"], hdb.StopRule(1e-10, 300))
    assert rep.converged and abs(rep.iterations - int(g["bp_its"])) <= 1
    assert np.abs(x - g["bp_x"]).max() <= 1e-8 * np.abs(g["bp_x"]).max()
    hier = hdb.mp1_problem(k=5.0, n=9, ml=2, boundary="dirichlet").hierarchy
    op = hdb.helmholtz_operator(hier, 1)
    D = np.asarray(op.diagonal())
    x, rep = hdb.bicgstab(op.apply, lambda u: u / D, g["bd9_b"], hdb.StopRule(1e-9, 200))
    # Bi-CGSTAB on this indefinite system amplifies rounding step by step (the history
    # leaves the reference's at 4e-14 after two steps); both converge to the same solution
    assert abs(rep.iterations - int(g["bd9_its"])) <= 2 and rep.converged
    assert np.abs(np.array(rep.residual_history[:3]) - g["bd9_hist"][:3]).max() <= 1e-12
    assert np.abs(x - g["bd9_x"]).max() <= 1e-7 * np.abs(g["bd9_x"]).max()
    hier = hdb.mp1_problem(k=30.0, n=65, ml=3).hierarchy
    m = hdb.cslp_operator(hier, 2, beta2=0.5)
    x, rep = hdb.bicgstab(m.apply, None, g["bc33_b"], hdb.StopRule(0.1, 30))
    assert rep.iterations == int(g["bc33_its"])
    # stopped at 0.1: Bi-CGSTAB carries the dot rounding into the iterate (1e-7 level)
    assert np.linalg.norm(x - g["bc33_x"]) <= 1e-6 * np.linalg.norm(g["bc33_x"])


def test_bicgstab_breakdown_carries_iterate():
    A = np.array([[0.0, 1.0], [-1.0, 0.0]], dtype=np.complex128)
    b = np.array([1.0, 1j], dtype=np.complex128)
    try:
        hdb.bicgstab(lambda u: A @ u, None, b, hdb.StopRule(1e-14, 50))
    except hdb.BreakdownError as err:
        assert err.x is not None and err.report is not None


@pytest.mark.parametrize("name", ["v1_mp1b", "v2_mp1b", "v3_wedge", "bicg_wedge"])
def test_presets_and_bicgstab_cslp_vs_reference(name):
    """MADP_V1/V2/V3 and a Bi-CGSTAB-CSLP MADP variant against the reference's own runs,
    at the reference's measured noise floor for each case (fixture floor_*)."""
    import dataclasses
    g = golden(f"preset_{name}.npz")
    pre = {"v1_mp1b": "MADP_V1", "v2_mp1b": "MADP_V2", "v3_wedge": "MADP_V3", "bicg_wedge": "MADP"}[name]
    prob = (hdb.mp1_problem(k=40.0, n=129, ml=3, boundary="sommerfeld") if "mp1b" in name
            else hdb.wedge_problem(f=20.0, nx=145, ml=4))
    cfg = hdb.preset(pre, prob.hierarchy)
    if name == "bicg_wedge":
        pols = tuple(dataclasses.replace(p, cslp_method="bicgstab") if p.cslp_method == "gmres" else p
                     for p in cfg.policies)
        cfg = dataclasses.replace(cfg, policies=pols, preset_name="MADP+bicgstab")
    with hdb.MadpSolver(prob.hierarchy, cfg) as s:
        u, rep = s.solve(prob.rhs)
    assert abs(rep.outer_iterations - int(g["outer_iterations"])) <= 1
    assert rep.converged == bool(g["converged"])
    floor_h = max(10 * float(g["floor_hist_abs"]), 1e-9)
    floor_x = max(10 * float(g["floor_sol_rel"]), 1e-8)
    h, hr = np.array(rep.residual_history), g["residual_history"]
    n = min(len(h), len(hr))
    assert np.abs(h[:n] - hr[:n]).max() <= floor_h
    x = u.grid_view(prob.hierarchy)
    assert np.linalg.norm(x - g["solution"]) <= floor_x * np.linalg.norm(g["solution"])


@pytest.mark.parametrize("f", [10, 20, 40])
def test_config3_wedge_vs_reference(f):
    """BASELINE configs[2]: wedge with the BASELINE interfaces, h = 0.5 m (1201 x 2001), 5 levels,
    against the reference's own full runs (tests/golden/solve_c3_*.npz), at the BASELINE
    bar: same outer count, history within 1e-9 per iteration, solution within 1e-8
    relative L2 (every 8th point).  Measured: <= 2.2e-14 / 7.6e-14; the reference's
    own floors are 1.0e-11 / 8.6e-10 / 3.1e-5 (history) at 10 / 20 / 40 Hz."""
    g = golden(f"solve_c3_{f}.npz")
    prob = hdb.wedge_problem(f=float(f), nx=1201, ml=5, layers=hdb.grid.BASELINE_WEDGE_LAYERS)
    with hdb.MadpSolver(prob.hierarchy, hdb.preset("MADP", prob.hierarchy)) as s:
        u, rep = s.solve(prob.rhs)
    assert rep.outer_iterations == int(g["outer_iterations"])
    assert rep.converged and rep.final_relres <= 1e-6
    h, hr = np.array(rep.residual_history), g["residual_history"]
    assert np.abs(h - hr).max() <= 1e-9
    st = int(g["solution_stride"])
    xs = u.grid_view(prob.hierarchy)[::st, ::st]
    ref = g["solution_sub"]
    assert np.linalg.norm(xs - ref) <= 1e-8 * np.linalg.norm(ref)


@pytest.mark.parametrize("name,h,ml", [("c4_h12_f40", 12.0, 2)])
def test_config4_synthetic_layered_vs_reference(name, h, ml):
    """BASELINE configs[3] model (seeded generator, models.py) at 40 Hz against the reference
    solving the same raster through its gridfile path (tests/golden/solve_<name>.npz).  At
    h = 12 m with two levels the reference stalls at its 150-iteration cap (final relres
    2.8e-2; its 1e-15-perturbed twin 2.8e-2): held to the count, the stall, the first steps
    at the BASELINE bar and every iteration to 10x the reference's own drift envelope."""
    g = golden(f"solve_{name}.npz")
    prob = hdb.synthetic_layered_problem(40.0, h, ml)
    hier = prob.hierarchy
    np.testing.assert_array_equal([hier.ksq[0].sum(), hier.ksq[-1].sum()], g["ksq_checksum"])
    with hdb.MadpSolver(hier, hdb.preset("MADP", hier)) as s:
        u, rep = s.solve(prob.rhs)
    assert abs(rep.outer_iterations - int(g["outer_iterations"])) <= 1
    assert rep.converged == bool(g["converged"])
    h_, hr = np.array(rep.residual_history), g["residual_history"]
    n = min(len(h_), len(hr))
    assert np.abs(h_[:2] - hr[:2]).max() <= 1e-9
    assert np.all(np.abs(h_[:n] - hr[:n]) <= 10 * _floor_envelope(g)[:n] + 1e-12)
    hb, xb = parity_bar(g)
    st = int(g["solution_stride"])
    assert np.linalg.norm(u.grid_view(hier)[::st, ::st] - g["solution_sub"]) <= xb * np.linalg.norm(g["solution_sub"])


# ---------------------------------------------------------------- device-side setup (f3)
def _device_setup_cases():
    from paper_2412_04980_b200 import grid as G
    from paper_2412_04980_b200 import models
    return {
        "mp1_k": lambda dev: hdb.mp1_problem(k=50.0, n=129, ml=3, boundary="dirichlet", device=dev),
        "mp1_f": lambda dev: hdb.mp1_problem(f=9.7, n=257, ml=4, device=dev),
        "const_c": lambda dev: G.Problem("c", hdb.build_hierarchy(((0.0, 3.0), (-1.0, 1.0)), 1.0 / 64, 3,
                                                                 velocity=hdb.VelocityModel("constant", c=1234.5),
                                                                 f=77.0, device=dev), None),
        "wedge20": lambda dev: hdb.wedge_problem(f=20.0, nx=145, ml=4, device=dev),
        "wedge_baseline": lambda dev: hdb.wedge_problem(f=10.0, nx=301, ml=3, layers=G.BASELINE_WEDGE_LAYERS,
                                                        device=dev),
        "marmousi": lambda dev: hdb.marmousi_problem(f=5.0, nx=737, ml=4, device=dev),
        "layered_c4": lambda dev: models.synthetic_layered_problem(f=10.0, h=3.0, ml=4, device=dev),
    }


@pytest.mark.parametrize("name", ["mp1_k", "mp1_f", "const_c", "wedge20", "wedge_baseline", "marmousi", "layered_c4"])
def test_device_setup_fields_bitexact_vs_host(name):
    """GPU-side setup (csrc/kernels_setup.cu; grid.py:120-160, 261-287, 309-320): the k^2
    field of every level, its maximum and the point source written on the device equal
    the host (reference-pinned) ones bit for bit."""
    case = _device_setup_cases()[name]
    host, devp = case(False), case(True)
    assert devp.hierarchy.device_ksq is not None and host.hierarchy.device_ksq is None
    for l in range(1, host.hierarchy.ml + 1):
        np.testing.assert_array_equal(devp.hierarchy.device_ksq_at(l).cpu().numpy(), host.hierarchy.ksq_at(l))
        np.testing.assert_array_equal(devp.hierarchy.ksq_at(l), host.hierarchy.ksq_at(l))  # lazy host copy
        assert devp.hierarchy.ksq_max_at(l) == host.hierarchy.ksq_at(l).max()
        assert hdb.kh_of(l, devp.hierarchy) == hdb.kh_of(l, host.hierarchy)
    if host.rhs is not None:
        np.testing.assert_array_equal(devp.rhs.cpu().numpy(), host.rhs.grid_view(host.hierarchy))


def test_device_setup_rejects_bad_models():
    from paper_2412_04980_b200.errors import ModelError
    with pytest.raises(ModelError):
        hdb.build_hierarchy(((0.0, 1.0), (0.0, 1.0)), 1.0 / 32, 2,
                            velocity=hdb.VelocityModel("gridfile", values=np.array([[1.0, np.inf], [1.0, 0.0]]),
                                                       dx=1.0, dy=1.0), f=1.0, device=True).ksq_at(1)
    with pytest.raises(ModelError):
        hdb.point_source_device(hdb.mp1_problem(k=10.0, n=33, ml=2, device=True).hierarchy, (2.0, 0.5))


@pytest.mark.parametrize("name", ["mp1_f", "wedge20"])
def test_device_built_problem_solves_identically(name):
    """A problem set up on the GPU (operators created from device k^2, multigrid
    sub-levels injected on the device, device right-hand side) gives the same solve,
    bit for bit, as the host-built one."""
    case = _device_setup_cases()[name]
    host, devp = case(False), case(True)
    cfg = hdb.preset("MADP", host.hierarchy)
    with hdb.MadpSolver(host.hierarchy, cfg) as s:
        xh, rh = s.solve(host.rhs)
    cfg_d = hdb.preset("MADP", devp.hierarchy)
    with hdb.MadpSolver(devp.hierarchy, cfg_d) as s:
        xd, rd = s.solve(devp.rhs)
    assert rd.outer_iterations == rh.outer_iterations
    assert list(rd.residual_history) == list(rh.residual_history)
    np.testing.assert_array_equal(xd.cpu().numpy(), xh.grid_view(host.hierarchy))
