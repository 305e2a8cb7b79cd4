"""Launch each hot-path kernel of the BASELINE config-2 hierarchy exactly once,
for one `ncu --set full` capture of all of them:

    ncu --set full --clock-control none --import-source on -k regex:'^k_' \
        -o gpurun_out/targets python tools/ncu_targets.py

Fine level (4097^2): 5-point apply (k_r1w) / residual / Jacobi (K1-K3), restriction,
prolongation, dot, fused residual norm (MG guard).  Coarse levels: radius-3 apply on level 3 (1025^2),
radius-2 apply on level 2 (2049^2).
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2412_04980_b200 as hdb  # noqa: E402
from paper_2412_04980_b200 import _lib  # noqa: E402


def main():
    import torch
    case = sys.argv[1] if len(sys.argv) > 1 else "c2"
    hier = bench.CONFIGS[case][1](hdb, 1).hierarchy
    L = _lib.lib()
    rng = np.random.default_rng(7)

    def field(shape):
        return torch.from_numpy(rng.standard_normal(shape) + 1j * rng.standard_normal(shape)).cuda()

    lv = hier.level(1)
    u, b, out = field(lv.shape), field(lv.shape), torch.empty(lv.shape, dtype=torch.complex128, device="cuda")
    op = hdb.helmholtz_operator(hier, 1)
    mg = hdb.CslpMultigrid(lv.nx, lv.ny, lv.h, hier.ksq_at(1), hier.boundary, beta2=0.5)
    c = torch.empty(hier.level(2).shape, dtype=torch.complex128, device="cuda")
    torch.cuda.synchronize()
    _lib.check(L.hdb_op_apply(op.handle, u.data_ptr(), out.data_ptr()))                       # k_r1w<0> (k_r1s<0> with HDB_R1_WAVE=0)
    _lib.check(L.hdb_op_residual(op.handle, b.data_ptr(), u.data_ptr(), out.data_ptr()))      # k_r1w<1>
    _lib.check(L.hdb_op_jacobi(mg.levels[0].op.handle, u.data_ptr(), b.data_ptr(), out.data_ptr(), 0.8))  # k_r1w<2>
    _lib.check(L.hdb_restrict(u.data_ptr(), lv.ny, lv.nx, c.data_ptr(), 0))                   # k_restrict_t
    _lib.check(L.hdb_prolong(c.data_ptr(), lv.ny, lv.nx, None, out.data_ptr()))               # k_prolong_t
    _lib.check(L.hdb_prolong(c.data_ptr(), lv.ny, lv.nx, b.data_ptr(), out.data_ptr()))       # k_prolong_t (+ base)
    d = (C.c_double * 2)()
    L.hdb_dot(u.data_ptr(), out.data_ptr(), lv.npoints, d)                                    # k_dot
    _lib.check(L.hdb_op_resnorm(mg.levels[0].op.handle, b.data_ptr(), u.data_ptr(), d))       # k_resnorm
    if hier.ml >= 3:
        for lvl in (3, 2):
            o = hdb.helmholtz_operator(hier, lvl)
            x = field(hier.level(lvl).shape)
            y = torch.empty_like(x)
            _lib.check(L.hdb_op_apply(o.handle, x.data_ptr(), y.data_ptr()))                 # k_rg<3,0>, k_rgh<2,0>
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
