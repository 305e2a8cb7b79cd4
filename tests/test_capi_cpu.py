"""CPU-side checks of the drop-in boundary and host logic (no GPU needed)."""
import json
import os
import re

import numpy as np
import pytest

import oracle
from gold import GOLDEN, ROOT

import paper_2412_04980_b200 as hdb
from paper_2412_04980_b200 import _lib


def _declared_symbols():
    txt = open(os.path.join(ROOT, "include", "hdb200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hdb_[a-z0-9_]+)\s*\(", txt)) - {"hdb_linop_fn", "hdb_iter_fn"})


def test_library_exports_every_declared_symbol():
    L = _lib.load_library()
    syms = _declared_symbols()
    assert len(syms) >= 25
    for name in syms:
        assert hasattr(L, name), name
    # and the ctypes table covers exactly the declared API
    assert set(_lib.SIGNATURES) == set(syms)


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(80|86|89|90)\b", out)


def test_compute_without_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(hdb.DeviceError):
        hdb.reduce_dot(np.ones((3, 3), complex), np.ones((3, 3), complex))
    hier = hdb.mp1_problem(k=5.0, n=9, ml=2).hierarchy
    with pytest.raises(hdb.DeviceError):
        hdb.helmholtz_operator(hier, 1).apply(np.zeros((9, 9), complex))


def test_level_kernels_match_reference_tables():
    tabs = json.load(open(os.path.join(GOLDEN, "kernel_tables.json")))
    for level, kinds in tabs.items():
        lap, mass = hdb.level_kernels(int(level))
        for kind, (rows, den) in kinds.items():
            k = lap if kind == "laplace" else mass
            assert k.denominator == den
            for r in range(7):
                for c in range(7):
                    want, got = rows[r][c], k.numerators[r][c]
                    if abs(want) <= 2 ** 53:
                        assert got == want
                    else:
                        assert abs(got - want) <= 3 * int(np.spacing(float(abs(got))))


def test_coefficients_match_oracle_bitwise():
    hier = hdb.mp1_problem(k=25.0, n=33, ml=4, boundary="dirichlet").hierarchy
    ohier, _ = oracle.mp1_problem(25.0, 33, 4, "dirichlet")
    for l in (1, 2, 3, 4):
        a = hdb.cslp_operator(hier, l, beta2=0.35)
        b = oracle.cslp_op(ohier, l, 0.35)
        np.testing.assert_array_equal(a.lap_coef, b.lap)
        np.testing.assert_array_equal(a.mass_coef, b.mass)
        np.testing.assert_array_equal(a.ksq, b.ksq)
    d = hdb.helmholtz_operator(hier, 1).diagonal()
    np.testing.assert_array_equal(d, oracle.helmholtz_op(ohier, 1).diagonal())


@pytest.mark.parametrize("case", ["c1s", "wedge20", "c2", "c3_40"])
def test_presets_and_hierarchies_match_oracle(case):
    if case == "c1s":
        p = hdb.mp1_problem(k=50.0, n=129, ml=2)
        oh, ob = oracle.mp1_problem(50.0, 129, 2)
    elif case == "wedge20":
        p = hdb.wedge_problem(f=20.0, nx=145, ml=4)
        oh, ob = oracle.wedge_problem(20.0, 145, 4)
    elif case == "c2":
        p = hdb.mp1_problem(k=200.0, n=1025, ml=5)  # same policy structure, smaller grid
        oh, ob = oracle.mp1_problem(200.0, 1025, 5)
    else:
        p = hdb.wedge_problem(f=40.0, nx=1201, ml=5, layers=hdb.grid.BASELINE_WEDGE_LAYERS)
        oh, ob = oracle.baseline_wedge_problem(40.0)
    hier = p.hierarchy
    for l in range(1, hier.ml + 1):
        np.testing.assert_array_equal(hier.ksq_at(l), oh.ksq_at(l))
    np.testing.assert_array_equal(p.rhs.grid_view(hier), ob)
    cfg = hdb.preset("MADP", hier)
    pols, outer = oracle.madp_preset(oh)
    for a, b in zip(cfg.policies, pols):
        assert a.cslp_method == b.cslp and a.cslp_shift == b.beta2
        assert (a.cslp_stop.rel_tol, a.cslp_stop.max_iters) == (b.cslp_stop.rel_tol, b.cslp_stop.max_iters)
        if b.cycle is None:
            assert a.deflation_cycle_stop is None
        else:
            assert (a.deflation_cycle_stop.rel_tol, a.deflation_cycle_stop.max_iters) == (b.cycle.rel_tol,
                                                                                          b.cycle.max_iters)


def test_mg_coarse_matrix_matches_oracle_assembly():
    from paper_2412_04980_b200.mg import assemble_radius1_dense
    from oracle.mg import dense_matrix
    for bnd in (("sommerfeld",) * 4, ("dirichlet", "sommerfeld", "dirichlet", "sommerfeld")):
        rng = np.random.default_rng(2)
        ksq = 100 + 50 * rng.random((9, 13))
        op = hdb.operators.radius1_operator(13, 9, 0.05, ksq, bnd, complex(1, 0.5))
        ref = oracle.radius1_op(13, 9, 0.05, ksq, bnd, complex(1, 0.5))
        A = assemble_radius1_dense(op)
        B = dense_matrix(ref)
        assert np.abs(A - B).max() <= 1e-12 * np.abs(B).max()


def test_errors_and_config_validation():
    hier = hdb.mp1_problem(k=5.0, n=9, ml=2).hierarchy
    with pytest.raises(hdb.ConfigError):
        hdb.preset("NOPE", hier)
    with pytest.raises(ValueError):
        hdb.StopRule(1e-6, 0)
    with pytest.raises(hdb.HierarchyError):
        hdb.mp1_problem(k=5.0, n=10, ml=2)
    assert hdb.cslp_iteration_cap(10000) == 60 and hdb.cslp_iteration_cap(10001) == 61
    assert issubclass(hdb.MgDivergence, hdb.HelmdefError)
    assert _lib._STATUS[4] is hdb.MgDivergence and _lib._STATUS[3] is hdb.NumericalError


def test_slab_partition_nesting():
    """distributed.slab_plan (the product's row-slab decomposition): slabs tile every
    sharded depth, coarse starts are injections of fine starts, and every rank keeps
    >= min_rows rows at the last sharded depth; P = 3 exercises odd cut rows."""
    from paper_2412_04980_b200.distributed import slab_plan
    for ny, ml in ((129, 6), (257, 5), (4097, 12), (2001, 5)):
        for ranks in (1, 2, 3, 4, 8):
            for min_rows in (8, 32):
                plan = slab_plan(ny, ranks, ml, min_rows=min_rows)
                for d in range(plan.depths):
                    slabs = [plan.slab(d, r) for r in range(ranks)]
                    assert slabs[0][0] == 0 and sum(n for _, n in slabs) == plan.rows_at(d)
                    assert all(a[0] + a[1] == b[0] for a, b in zip(slabs, slabs[1:]))
                    if d > 0:
                        assert all(plan.slab(d - 1, r)[0] == 2 * slabs[r][0] for r in range(ranks))
                if plan.depths:
                    assert min(plan.slab(plan.depths - 1, r)[1] for r in range(ranks)) >= min_rows


def test_synthetic_layered_model_is_seeded_and_in_range():
    from paper_2412_04980_b200.models import synthetic_layered_velocity
    a = synthetic_layered_velocity(7, dx=24.0)
    b = synthetic_layered_velocity(7, dx=24.0)
    c = synthetic_layered_velocity(8, dx=24.0)
    np.testing.assert_array_equal(a.values, b.values)
    assert not np.array_equal(a.values, c.values)
    assert a.values.min() >= 1500.0 and a.values.max() <= 5500.0
    # velocity increases with depth on average (row 0 is the bottom, y = -3000 m)
    assert a.values[0].mean() > a.values[-1].mean() + 2000.0
    # the same raster through the oracle's grid builder (reference bilinear rule) gives the same k^2
    from paper_2412_04980_b200.models import C4_DOMAIN
    hier = hdb.build_hierarchy(C4_DOMAIN, h=12.0, ml=2, velocity=a, f=10.0)
    from oracle.grid import build_hierarchy as obuild
    oh = obuild(C4_DOMAIN, 12.0, 2, speed=lambda x, y: a.velocity_at(x, y), f=10.0)
    np.testing.assert_array_equal(hier.ksq_at(1), oh.ksq_at(1))
