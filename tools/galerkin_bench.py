"""Galerkin (radius-2/3) level operators of a configuration, separable form vs the
reference's exact tap order, and the one-launch MGS step in its low-synchronisation
form vs the MGS order (CUDA events on the library stream).

    python tools/galerkin_bench.py [c2] [--reps 20]
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case", nargs="?", default="c2")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import torch
    import paper_2412_04980_b200 as hdb
    from paper_2412_04980_b200 import _lib
    L = _lib.lib()
    peak, _ = bench._peaks()
    hier = bench.CONFIGS[a.case][1](hdb, 1).hierarchy
    rng = np.random.default_rng(0)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timeit(fn, reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(reps):
            fn()
        ev1.record()
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) / reps

    def timeit_graph(fn, reps):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            _lib.check(L.hdb_set_stream(C.c_void_p(s.cuda_stream)))
            for _ in range(3):
                fn()
            s.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(reps):
                    fn()
            g.replay()
            s.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            s.synchronize()
        _lib.check(L.hdb_set_stream(C.c_void_p(torch.cuda.current_stream().cuda_stream)))
        return e0.elapsed_time(e1) / reps

    out = {}
    for l in range(2, hier.ml + 1):
        op = hdb.cslp_operator(hier, l, 0.5)
        lv = hier.level(l)
        u = torch.from_numpy(rng.standard_normal(lv.shape) + 1j * rng.standard_normal(lv.shape)).cuda()
        o = torch.empty_like(u)
        h = op.handle
        row = {"points": lv.npoints}
        for name, exact in (("separable", 0), ("exact", 1)):
            _lib.check(L.hdb_option(b"rg_exact", exact))
            # a captured CUDA graph of `reps` launches: device time without Python launch overhead
            ms = timeit_graph(lambda: _lib.check(L.hdb_op_apply(h, u.data_ptr(), o.data_ptr())), a.reps)
            gbs = 40.0 * lv.npoints / (ms * 1e-3) / 1e9
            row[name] = {"us": round(ms * 1e3, 2), "gbs": round(gbs, 1), "frac": round(gbs / peak, 3)}
        _lib.check(L.hdb_option(b"rg_exact", 0))
        out[f"L{l}"] = row
        print(f"L{l}", json.dumps(row), flush=True)
    # fixed per-launch cost on a tiny grid (one CTA): kernels that take the level operator's
    # coefficient block by value (2.3 KB of parameters) vs a parameter-light dot
    tiny = hdb.mp1_problem(k=5.0, n=17, ml=3).hierarchy
    for l, name in ((1, "tiny_apply5"), (2, "tiny_galerkin_r2"), (3, "tiny_galerkin_r3")):
        op = hdb.cslp_operator(tiny, l, 0.5)
        lv = tiny.level(l)
        u = torch.from_numpy(rng.standard_normal(lv.shape) + 1j * rng.standard_normal(lv.shape)).cuda()
        o = torch.empty_like(u)
        h = op.handle
        out[name] = {"us": round(timeit_graph(lambda: _lib.check(L.hdb_op_apply(h, u.data_ptr(), o.data_ptr())),
                                              a.reps) * 1e3, 2)}
    u = torch.from_numpy(rng.standard_normal((17, 17)) + 1j * rng.standard_normal((17, 17))).cuda()
    out["tiny_dot"] = {"us": round(timeit_graph(lambda: _lib.check(L.hdb_dot(u.data_ptr(), u.data_ptr(), 289, None)),
                                                a.reps) * 1e3, 2)}
    print("tiny", json.dumps({k: v for k, v in out.items() if k.startswith("tiny")}), flush=True)
    # one-launch MGS step on the 1025^2 level: GMRES(1e-14, cap) through the launch-driven engine
    prob = hdb.mp1_problem(k=200.0, n=1025, ml=2)
    op = hdb.cslp_operator(prob.hierarchy, 1, 0.5)
    b = torch.from_numpy(rng.standard_normal(op.shape) + 1j * rng.standard_normal(op.shape)).cuda()
    x = torch.empty_like(b)
    for ls in (1, 0):
        _lib.check(L.hdb_option(b"mgs_ls", ls))
        for cap in (6, 12, 20):
            its, rel = C.c_int(), C.c_double()
            _lib.check(L.hdb_op_gmres(op.handle, b.data_ptr(), x.data_ptr(), 1e-14, cap, -1, C.byref(its), C.byref(rel)))
            _lib.kprof(True)
            _lib.check(L.hdb_op_gmres(op.handle, b.data_ptr(), x.data_ptr(), 1e-14, cap, -1, C.byref(its), C.byref(rel)))
            f = _lib.kprof_read()["mgs_coop"]
            _lib.kprof(False)
            us = f["device_ms"] * 1e3 / max(1, f["launches"])
            gbs = f["alg_bytes"] / (f["device_ms"] * 1e-3) / 1e9 if f["device_ms"] else 0.0
            key = f"mgs_{'lowsync' if ls else 'mgs_order'}_cap{cap}"
            out[key] = {"launches": f["launches"], "us_per_launch": round(us, 2), "alg_gbs": round(gbs, 1),
                        "frac": round(gbs / peak, 3), "relres": rel.value}
            print(key, json.dumps(out[key]), flush=True)
    _lib.check(L.hdb_option(b"mgs_ls", 1))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
