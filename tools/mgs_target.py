"""One GMRES(1e-14, CAP) solve on the 1025^2 CSLP level of BASELINE config 2 through
the launch-driven engine, so the one-launch MGS steps j = 0 .. CAP-1 run in order
(the ncu target of tools/ncu_mgs_summary.py):

    ncu --set full -k regex:k_mgs -c CAP python tools/mgs_target.py [CAP] [--mgs]
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
    cap = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 12
    L = _lib.lib()
    if "--mgs" in sys.argv:
        _lib.check(L.hdb_option(b"mgs_ls", 0))
    prob = hdb.mp1_problem(k=200.0, n=1025, ml=2)     # 1025^2 with config 2's k h on level 3
    op = hdb.cslp_operator(prob.hierarchy, 1, 0.5)
    rng = np.random.default_rng(3)
    b = torch.from_numpy(rng.standard_normal(op.shape) + 1j * rng.standard_normal(op.shape)).cuda()
    x = torch.empty_like(b)
    its, rel = C.c_int(), C.c_double()
    _lib.check(L.hdb_op_gmres(op.handle, b.data_ptr(), x.data_ptr(), 1e-14, cap, -1, C.byref(its), C.byref(rel)))
    torch.cuda.synchronize()
    print("its", its.value, "relres", rel.value)


if __name__ == "__main__":
    main()
