"""Time the CSLP GMRES solve on every level of a configuration in each engine mode.

    python tools/gmres_modes.py [c2] [--reps 3]
Prints per level: points, iterations, ms per solve for launch (-1) / cluster (0) / grid (1).
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2412_04980_b200 as hdb  # noqa: E402
from paper_2412_04980_b200 import _lib  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case", nargs="?", default="c2")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--levels", default="")
    ap.add_argument("--tol", type=float, default=0.1)
    ap.add_argument("--cap", type=int, default=0)
    a = ap.parse_args()
    import torch
    prob = bench.CONFIGS[a.case][1](hdb, 1)
    hier = prob.hierarchy
    cfg = hdb.preset("MADP", hier)
    L = _lib.lib()
    out = {}
    levels = [int(x) for x in a.levels.split(",")] if a.levels else range(2, hier.ml + 1)
    for l in levels:
        pol = cfg.policy(l)
        op = hdb.cslp_operator(hier, l, pol.cslp_shift)
        rng = np.random.default_rng(l)
        b = torch.from_numpy(rng.standard_normal(op.shape) + 1j * rng.standard_normal(op.shape)).cuda()
        x = torch.empty_like(b)
        row = {"points": op.npoints, "cap": pol.cslp_stop.max_iters}
        for mode in (-1, 0, 1):
            its, rel = C.c_int(), C.c_double()
            st = L.hdb_op_gmres(op.handle, b.data_ptr(), x.data_ptr(), a.tol, a.cap or pol.cslp_stop.max_iters, mode,
                                C.byref(its), C.byref(rel))
            if st != 0:
                row[str(mode)] = L.hdb_last_error().decode()[:60]
                continue
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(a.reps):
                L.hdb_op_gmres(op.handle, b.data_ptr(), x.data_ptr(), a.tol, a.cap or pol.cslp_stop.max_iters, mode,
                               C.byref(its), C.byref(rel))
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t0) / a.reps * 1e3
            prof = (C.c_longlong * 12)()
            if mode >= 0:
                L.hdb_resident_profile(1, None)
                L.hdb_op_gmres(op.handle, b.data_ptr(), x.data_ptr(), a.tol, a.cap or pol.cslp_stop.max_iters, mode,
                               C.byref(its), C.byref(rel))
                L.hdb_resident_profile(0, prof)
            row[str(mode) + "_phase_us"] = [round(v / 1.965e3, 1) for v in prof[:11]]
            row[str(mode)] = {"its": its.value, "ms": round(dt, 3), "us_per_it": round(dt * 1e3 / max(1, its.value), 1),
                              "relres": rel.value}
        out[l] = row
        print(l, json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
