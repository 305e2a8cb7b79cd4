"""Exercise every shared-memory / mbarrier / TMA / cluster kernel of the path once,
on small-to-moderate inputs, for a compute-sanitizer pass (one tool per run):

    compute-sanitizer --tool racecheck python tools/sanitize_targets.py
    compute-sanitizer --tool synccheck python tools/sanitize_targets.py

Covers: 5-point strip kernels (apply / residual / Jacobi / fused residual norm),
the radius-2/3 Galerkin stencils, TMA-staged restriction / prolongation (fine
grids >= 2047 columns), the cooperative MGS steps (TMA-fed form on a 1025^2
level, the register/shared form on smaller levels) with the device-driven GMRES
control kernels, and the device-resident GMRES in cluster and grid mode.
Prints SANITIZE_TARGETS_DONE at the end.
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402


def main():
    import torch
    import paper_2412_04980_b200 as hdb
    from paper_2412_04980_b200 import _lib
    L = _lib.lib()
    rng = np.random.default_rng(3)

    def rnd(shape):
        return torch.from_numpy(rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).cuda()

    # stencils on a 1025^2 hierarchy (levels 1..3: radius 1, 2, 3)
    prob = hdb.mp1_problem(k=100.0, n=1025, ml=4)
    hier = prob.hierarchy
    for l in (1, 2, 3):
        op = hdb.cslp_operator(hier, l, 0.5)
        u, b = rnd(op.shape), rnd(op.shape)
        out = torch.empty_like(u)
        _lib.check(L.hdb_op_apply(op.handle, u.data_ptr(), out.data_ptr()))
        _lib.check(L.hdb_op_residual(op.handle, b.data_ptr(), u.data_ptr(), out.data_ptr()))
        if l == 1:
            _lib.check(L.hdb_op_jacobi(op.handle, u.data_ptr(), b.data_ptr(), out.data_ptr(), C.c_double(0.8)))
            _lib.check(L.hdb_op_jacobi(op.handle, None, b.data_ptr(), out.data_ptr(), C.c_double(0.8)))
            two = (C.c_double * 2)()
            _lib.check(L.hdb_op_resnorm(op.handle, b.data_ptr(), u.data_ptr(), two))
    torch.cuda.synchronize()
    print("stencils ok", flush=True)
    # TMA transfers (fine grid >= 2047 columns)
    n = 2049
    nc = (n - 1) // 2 + 1
    u, base, cu = rnd((n, n)), rnd((n, n)), rnd((nc, nc))
    c = torch.empty((nc, nc), dtype=torch.complex128, device="cuda")
    f = torch.empty((n, n), dtype=torch.complex128, device="cuda")
    _lib.check(L.hdb_restrict(u.data_ptr(), n, n, c.data_ptr(), 0))
    _lib.check(L.hdb_prolong(cu.data_ptr(), n, n, None, f.data_ptr()))
    _lib.check(L.hdb_prolong(cu.data_ptr(), n, n, base.data_ptr(), f.data_ptr()))
    torch.cuda.synchronize()
    print("transfers ok", flush=True)
    # GMRES engines: launch-driven (cooperative MGS) on the 1025^2 level, resident on small ones
    for lvl, modes in ((1, (-1,)), (3, (-1, 1)), (4, (0, 1))):
        op = hdb.cslp_operator(hier, lvl, 0.5)
        b = rnd(op.shape)
        x = torch.empty_like(b)
        for mode in modes:
            its, rel = C.c_int(), C.c_double()
            _lib.check(L.hdb_op_gmres(op.handle, b.data_ptr(), x.data_ptr(), C.c_double(0.1), 4, mode,
                                      C.byref(its), C.byref(rel)))
            print(f"gmres level {lvl} ({op.npoints} pts) mode {mode}: {its.value} its", flush=True)
    torch.cuda.synchronize()
    # one small full solve (MG V-cycles, one-step FGMRES, device-resident coarsest CSLP)
    p = hdb.mp1_problem(k=50.0, n=129, ml=3)
    with hdb.MadpSolver(p.hierarchy, hdb.preset("MADP", p.hierarchy)) as s:
        _, rep = s.solve(p.rhs)
    print("solve", rep.outer_iterations, rep.final_relres, flush=True)
    print("SANITIZE_TARGETS_DONE", flush=True)


if __name__ == "__main__":
    main()
