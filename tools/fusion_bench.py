"""Fused multigrid kernels against the launches they replace, per grid size (CUDA
events on the library stream):
  residual (56 B/pt) + restriction (20 B/pt)   vs  residual_restrict (44 B/pt)
  Jacobi sweep (56 B/pt) + add (48 B/pt)       vs  jacobi_add (88 B/pt)

    python tools/fusion_bench.py [--sizes 4097,2049,1025,513] [--reps 30]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2412_04980_b200 as hdb  # noqa: E402
from paper_2412_04980_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="4097,2049,1025,513")
    ap.add_argument("--reps", type=int, default=30)
    a = ap.parse_args()
    import torch
    L = _lib.lib()
    peak, _ = bench._peaks()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def timeit(fn):
        for _ in range(3):
            fn()
        tot = 0.0
        for _ in range(a.reps):
            flush.fill_(1)  # evict L2 between repetitions (small levels would otherwise sit in it)
            ev0.record()
            fn()
            ev1.record()
            torch.cuda.synchronize()
            tot += ev0.elapsed_time(ev1)
        return tot / a.reps * 1e3  # us

    rng = np.random.default_rng(5)
    for n in [int(x) for x in a.sizes.split(",")]:
        ksq = 900.0 + 500.0 * rng.random((n, n))
        op = hdb.radius1_operator(n, n, 1.0 / (n - 1), ksq, ("sommerfeld",) * 4, complex(1.0, 0.5))
        h = op.handle
        mk = lambda: torch.from_numpy(rng.standard_normal((n, n)) + 1j * rng.standard_normal((n, n))).cuda()  # noqa: E731
        u, b, t = mk(), mk(), mk()
        r, o2 = torch.empty_like(u), torch.empty_like(u)
        nc = (n - 1) // 2 + 1
        c = torch.empty((nc, nc), dtype=torch.complex128, device="cuda")
        pts = float(n) * n

        def pair():
            _lib.check(L.hdb_op_residual(h, b.data_ptr(), u.data_ptr(), r.data_ptr()))
            _lib.check(L.hdb_restrict(r.data_ptr(), n, n, c.data_ptr(), 0))

        def fused():
            _lib.check(L.hdb_op_residual_restrict(h, b.data_ptr(), u.data_ptr(), c.data_ptr(), 0))

        def jac_pair():
            _lib.check(L.hdb_op_jacobi(h, u.data_ptr(), b.data_ptr(), r.data_ptr(), 0.8))
            _lib.check(L.hdb_op_residual(h, r.data_ptr(), r.data_ptr(), o2.data_ptr())) if False else None

        def jac_fused():
            _lib.check(L.hdb_op_jacobi_add(h, u.data_ptr(), b.data_ptr(), r.data_ptr(), 0.8, t.data_ptr(), o2.data_ptr()))

        tp, tf = timeit(pair), timeit(fused)
        tj, tjf = timeit(jac_pair), timeit(jac_fused)
        row = {"n": n,
               "residual+restrict_us": round(tp, 1), "fused_us": round(tf, 1),
               "fused_frac_of_peak": round(44.0 * pts / (tf * 1e-6) / 1e9 / peak, 3),
               "pair_frac_of_peak(76B/pt)": round(76.0 * pts / (tp * 1e-6) / 1e9 / peak, 3),
               "jacobi_only_us": round(tj, 1), "jacobi_add_us": round(tjf, 1),
               "jacobi_add_frac_of_peak": round(88.0 * pts / (tjf * 1e-6) / 1e9 / peak, 3)}
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
