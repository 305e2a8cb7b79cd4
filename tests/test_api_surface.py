"""CPU tests of the drop-in host API: the reference's full public name list, and
the host-side pieces (grid models, assembly, ghost padding, tiling, kernel chain
checks) pinned bit for bit against reference-generated fixtures
(tests/golden/make_golden.py grid_models / api_surface)."""
import numpy as np
import pytest

import paper_2412_04980_b200 as hdb
from paper_2412_04980_b200 import grid as G
from paper_2412_04980_b200 import operators as O
from paper_2412_04980_b200 import stencils as S
from gold import golden

# the reference's public names (helmdef/__init__.py:9-62)
REFERENCE_NAMES = """
BreakdownError CapacityError ConfigError HelmdefError HierarchyError IoError LevelError MgDivergence
ModelError NumericalError ShapeError ComplexField GridHierarchy GridLevel Problem VelocityModel
build_hierarchy dimensionless_kmax kh_of marmousi_problem mp1_problem point_source_rhs
synthetic_marmousi_velocity wedge_problem wedge_velocity KrylovReport StopRule bicgstab
cslp_iteration_cap fgmres gmres ConvergenceReport Definiteness LevelPolicy MadpSolver SolverConfig
classify_levels preset solve CslpMultigrid MgConfig LevelOperator apply_cslp apply_helmholtz
arithmetic_intensity assemble_csr cslp_operator helmholtz_operator matvec_flop_byte_counters
Partition WorkerPool halo_exchange partition_grid reduce_dot StencilKernel galerkin_coarsen
level_kernels verify_chain prolong prolong_array restrict restrict_array __version__
""".split()


def test_every_reference_name_is_exported():
    missing = [n for n in REFERENCE_NAMES if not hasattr(hdb, n)]
    assert not missing, missing
    assert len(REFERENCE_NAMES) == 63   # 62 names + __version__


def test_grid_models_bitexact_vs_reference():
    d = golden("grid_models.npz")
    p = hdb.wedge_problem(f=7.0, nx=61, ml=3)
    np.testing.assert_array_equal(p.hierarchy.ksq[0], d["wedge_ksq1"])
    np.testing.assert_array_equal(p.hierarchy.ksq[2], d["wedge_ksq3"])
    np.testing.assert_array_equal(p.rhs.data, d["wedge_rhs"])
    vel = hdb.VelocityModel(kind="wedge", layers=G.BASELINE_WEDGE_LAYERS)
    h = hdb.build_hierarchy(((0.0, 600.0), (-1000.0, 0.0)), h=12.5, ml=3, velocity=vel, f=9.0)
    np.testing.assert_array_equal(h.ksq[0], d["bwedge_ksq1"])
    m = hdb.synthetic_marmousi_velocity(185, 61)
    np.testing.assert_array_equal(m.values, d["marm_values"])
    np.testing.assert_array_equal([m.dx, m.dy, m.x0, m.y0], d["marm_meta"])
    mp = hdb.marmousi_problem(3.0, nx=185, ml=3)
    np.testing.assert_array_equal(mp.hierarchy.ksq[0], d["marm_ksq1"])
    np.testing.assert_array_equal(mp.rhs.data, d["marm_rhs"])
    mg = hdb.marmousi_problem(2.0, nx=93, ml=2, velocity=m)
    np.testing.assert_array_equal(mg.hierarchy.ksq[0], d["marmg_ksq1"])
    gv = hdb.VelocityModel(kind="gridfile", values=d["raster_in"], dx=17.3, dy=11.1, x0=-5.0, y0=-240.0)
    gh = hdb.build_hierarchy(((0.0, 600.0), (-250.0, 0.0)), h=6.25, ml=2, velocity=gv, f=11.0)
    np.testing.assert_array_equal(gh.ksq[0], d["raster_ksq1"])


def test_grid_errors_match_reference_contract():
    with pytest.raises(hdb.HierarchyError):
        hdb.build_hierarchy(((0.0, 1.0), (0.0, 1.0)), h=0.3, ml=2, k=1.0)
    with pytest.raises(hdb.HierarchyError):
        hdb.build_hierarchy(((0.0, 1.0), (0.0, 1.0)), h=1 / 6, ml=3, k=1.0)
    with pytest.raises(hdb.ModelError):
        hdb.build_hierarchy(((0.0, 1.0), (0.0, 1.0)), h=0.25, ml=2, velocity=hdb.VelocityModel("wedge"), f=1.0)
    with pytest.raises(hdb.ModelError):
        hdb.VelocityModel("constant", c=1.0, k=1.0).validate()
    with pytest.raises(hdb.ModelError):
        hdb.VelocityModel("unknown").velocity_at(np.zeros(2), np.zeros(2))
    with pytest.raises(hdb.LevelError):
        hdb.mp1_problem(k=5.0, n=9, ml=2).hierarchy.level(3)
    with pytest.raises(hdb.ModelError):
        hdb.point_source_rhs(hdb.mp1_problem(k=5.0, n=9, ml=2).hierarchy, (2.0, 0.5))
    with pytest.raises(hdb.ShapeError):
        hdb.ComplexField(1, np.zeros(5)).grid_view(hdb.mp1_problem(k=5.0, n=9, ml=2).hierarchy)


def _wedge_hier(bc):
    vel = hdb.VelocityModel(kind="wedge", layers=G.BASELINE_WEDGE_LAYERS)
    return hdb.build_hierarchy(((0.0, 600.0), (-1000.0, 0.0)), h=25.0, ml=3, velocity=vel, f=6.0, boundary=bc)


@pytest.mark.parametrize("tag,bc", [("s", "sommerfeld"), ("d", "dirichlet"),
                                    ("m", ("dirichlet", "sommerfeld", "sommerfeld", "dirichlet"))])
@pytest.mark.parametrize("level", [1, 2, 3])
def test_assembly_and_ghost_pad_bitexact_vs_reference(tag, bc, level):
    d = golden("api_surface.npz")
    hier = _wedge_hier(bc)
    op = O.helmholtz_operator(hier, level) if tag == "s" else O.cslp_operator(hier, level, 0.5)
    np.testing.assert_array_equal(hdb.assemble_csr(op).toarray(), d[f"asm_{tag}{level}"])
    np.testing.assert_array_equal(O.assemble_dense(op), d[f"asm_{tag}{level}"])
    np.testing.assert_array_equal(op.pad(d[f"pad_{tag}{level}_u"]), d[f"pad_{tag}{level}"])
    np.testing.assert_array_equal(op.ksq_pad, d[f"kpad_{tag}{level}"])
    pf = hdb.halo_exchange(d[f"pad_{tag}{level}_u"], op.pad, op.radius)
    np.testing.assert_array_equal(pf.interior(), d[f"pad_{tag}{level}_u"])


def test_assembly_guard():
    op = O.helmholtz_operator(hdb.mp1_problem(k=5.0, n=9, ml=2).hierarchy, 1)
    with pytest.raises(hdb.CapacityError):
        hdb.assemble_csr(op, max_points=10)


@pytest.mark.parametrize("name,builder", [("mp1_257_5", lambda: hdb.mp1_problem(k=20.0, n=257, ml=5)),
                                          ("wedge_145_4", lambda: hdb.wedge_problem(f=10.0, nx=145, ml=4))])
def test_partition_grid_matches_reference(name, builder):
    d = golden("api_surface.npz")
    hier = builder().hierarchy
    for w in (1, 2, 3, 4, 6, 8):
        part = hdb.partition_grid(hier, w)
        got = np.array([[l, t.j0, t.j1, t.i0, t.i1] for l in sorted(part.tiles) for t in part.tiles[l]])
        np.testing.assert_array_equal(got, d[f"tiles_{name}_{w}"])
        for l in part.tiles:  # tiles cover every level exactly once
            assert sum(t.npoints for t in part.level_tiles(l)) == hier.level(l).npoints


def test_kernel_chain_checks_match_reference():
    d = golden("api_surface.npz")
    got = np.array([[r["level"], r["kind"] == "mass", r["exact_match"], r["within_ulp"]] for r in hdb.verify_chain()])
    np.testing.assert_array_equal(got, d["verify_chain"])
    lap2, mass2 = hdb.galerkin_coarsen(*hdb.level_kernels(1))
    np.testing.assert_array_equal(np.array(lap2.numerators), d["coarsen_l1_lap"])
    np.testing.assert_array_equal(np.array(mass2.numerators), d["coarsen_l1_mass"])
    np.testing.assert_array_equal([lap2.denominator, mass2.denominator], d["coarsen_l1_den"])
    for l in range(1, 7):   # the 2D coarsening reproduces the separable chain
        assert hdb.galerkin_coarsen(*hdb.level_kernels(l)) == hdb.level_kernels(l + 1)
    # a perturbed chain is reported
    def bad(level):
        lap, mass = hdb.level_kernels(level)
        rows = [list(r) for r in lap.numerators]
        rows[3][3] += 1
        return hdb.StencilKernel(tuple(map(tuple, rows)), lap.denominator, lap.h_power), mass
    rec = hdb.verify_chain(bad)
    assert not any(r["within_ulp"] for r in rec if r["kind"] == "laplace")
    assert rec[0]["first_mismatch"][:2] == (3, 3)
    with pytest.raises(ValueError):
        hdb.StencilKernel(((1, 2),), 1, 0)
    with pytest.raises(ValueError):
        hdb.StencilKernel(((1,),), 3, 0)
    assert hdb.level_kernels(4)[0].is_symmetric()


def test_worker_pool_contract():
    seen = []
    with hdb.WorkerPool(1) as p:
        p.run(seen.append, range(3))
    assert seen == [0, 1, 2]
    out = [0] * 8
    with hdb.WorkerPool(4) as p:
        p.run(lambda i: out.__setitem__(i, i * i), range(8))
        assert out == [i * i for i in range(8)]

        def boom(i):
            if i == 5:
                raise RuntimeError("task 5")
        with pytest.raises(RuntimeError, match="task 5"):
            p.run(boom, range(8))


def test_custom_dot_is_rejected_and_known_dots_accepted():
    b = np.ones((3, 3), dtype=np.complex128)
    with pytest.raises(hdb.ConfigError):
        hdb.fgmres(lambda u: u, None, b, hdb.StopRule(0.1, 2), dot=lambda u, v: 0j)
    with pytest.raises(hdb.ConfigError):
        hdb.bicgstab(lambda u: u, None, b, hdb.StopRule(0.1, 2), dot=lambda u, v: 0j)
    from paper_2412_04980_b200.krylov import _check_dot
    for ok in (None, np.vdot, hdb.reduce_dot):
        _check_dot(ok)
