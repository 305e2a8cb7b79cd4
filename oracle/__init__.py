"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A from-scratch CPU restatement (numpy + numba loops) of the reference
`helmdef` algorithm on the MADP-FGMRES hot path.  Each
function cites the reference file:line it restates (paths relative to
/root/reference/pkg/src/helmdef/).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py` (its `cpu_baseline`
leg and `--impl reference` arm) may import this package, and only as the
checker / CPU baseline.  The product package `paper_2412_04980_b200` never
imports it; the product path fails loudly without its CUDA library.

Parity pin: tests/golden/ holds fixtures produced by running the reference
itself in the build container (tests/golden/make_golden.py); the
`-m "not gpu"` suite checks this oracle against them (stencil chain tables,
operator/transfer/Jacobi outputs bit-for-bit, V-cycle, FGMRES and full-solve
residual histories).
"""
from .chain import level_kernels, mass_level_scale, verify_against_tables  # noqa: F401
from .grid import (Hierarchy, Level, build_hierarchy, mp1_problem, wedge_problem,  # noqa: F401
                   point_source, baseline_wedge_problem)
from .ops import CpuLevelOp, radius1_op, helmholtz_op, cslp_op, restrict, prolong, reduce_dot  # noqa: F401
from .krylov import Stop, fgmres, cslp_cap  # noqa: F401
from .mg import CpuMultigrid  # noqa: F401
from .madp import madp_preset, CpuMadpSolver  # noqa: F401
