"""Time the one-launch low-synchronisation MGS step (k_mgs_ls) on the 1025^2 CSLP level of
BASELINE config 2: GMRES(1e-14, cap) through the launch-driven engine, per-launch CUDA events
(engine launch accounting).  Run once per setting of an environment knob, e.g.

    HDB_LS_KEEP=-1 python tools/mgs_ls_sweep.py     (no L2 hints)
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bench  # noqa: E402


def main():
    import torch
    import paper_2412_04980_b200 as hdb
    from paper_2412_04980_b200 import _lib
    L = _lib.lib()
    peak, _ = bench._peaks()
    rng = np.random.default_rng(0)
    prob = hdb.mp1_problem(k=200.0, n=1025, ml=2)
    op = hdb.cslp_operator(prob.hierarchy, 1, 0.5)
    b = torch.from_numpy(rng.standard_normal(op.shape) + 1j * rng.standard_normal(op.shape)).cuda()
    x = torch.empty_like(b)
    out = {"env": {k: v for k, v in os.environ.items() if k.startswith("HDB_")}}
    for cap in (6, 12, 20):
        its, rel = C.c_int(), C.c_double()
        _lib.check(L.hdb_op_gmres(op.handle, b.data_ptr(), x.data_ptr(), 1e-14, cap, -1, C.byref(its), C.byref(rel)))
        best = None
        for _ in range(3):
            _lib.kprof(True)
            _lib.check(L.hdb_op_gmres(op.handle, b.data_ptr(), x.data_ptr(), 1e-14, cap, -1, C.byref(its), C.byref(rel)))
            f = _lib.kprof_read()["mgs_coop"]
            _lib.kprof(False)
            if best is None or f["device_ms"] < best["device_ms"]:
                best = f
        us = best["device_ms"] * 1e3 / max(1, best["launches"])
        gbs = best["alg_bytes"] / (best["device_ms"] * 1e-3) / 1e9 if best["device_ms"] else 0.0
        out[f"cap{cap}"] = {"launches": best["launches"], "us_per_launch": round(us, 2), "alg_gbs": round(gbs, 1),
                            "frac": round(gbs / peak, 3), "relres": rel.value}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
