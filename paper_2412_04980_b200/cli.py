"""Command line: `python -m paper_2412_04980_b200 {solve,bench,stencils}`.

Same subcommands, flags, file formats and exit codes as the reference CLI for
the solve path (cli.py:33-57, 115-132): 0 converged, 1 usage/configuration
error, 2 iteration cap reached, 3 stencil-chain mismatch.  `bench` times the
GPU matrix-free 5-point apply (the reference's bench compares CPU
matrix-free vs CSR); parameter sweeps are out of scope.
"""
from __future__ import annotations

import argparse
import os
import sys
import time
from dataclasses import replace

from . import io as hio
from .errors import HelmdefError


def _args(argv):
    ap = argparse.ArgumentParser(prog="paper_2412_04980_b200", description=__doc__)
    sub = ap.add_subparsers(dest="command")
    s = sub.add_parser("solve", help="run one configured solve")
    for flag, kw in (("--config", {}), ("--preset", {}), ("--levels", {"type": int}), ("--workers", {"type": int}),
                     ("--out", {"default": None}), ("--kh", {"type": float}), ("--freq-hz", {"type": float}),
                     ("--wavenumber", {"type": float})):
        s.add_argument(flag, **kw)
    s.add_argument("--write-solution", action="store_true")
    b = sub.add_parser("bench", help="GPU matrix-free 5-point apply throughput")
    b.add_argument("--sizes", default="257,1025,4097")
    b.add_argument("--reps", type=int, default=50)
    b.add_argument("--wavenumber", type=float, default=40.0)
    b.add_argument("--out", default=None)
    v = sub.add_parser("stencils", help="coarse-kernel chain inspection")
    v.add_argument("--verify", action="store_true")
    return ap, ap.parse_args(argv)


def _config(a) -> hio.RunConfig:
    if not a.config:
        raise HelmdefError("a --config file is required")
    cfg = hio.parse_config_file(a.config)
    upd = {}
    if a.preset:
        upd["preset"] = a.preset
    if a.levels:
        upd["levels"] = a.levels
    if a.kh is not None:
        upd.update(kh=a.kh, nx=None)
    if a.freq_hz is not None:
        upd.update(freq_hz=a.freq_hz, wavenumber=None)
    if a.wavenumber is not None:
        upd.update(wavenumber=a.wavenumber, freq_hz=None)
    upd["workers"] = a.workers if a.workers is not None else int(os.environ.get("HELMDEF_WORKERS", cfg.workers))
    if a.out:
        upd["out_dir"] = a.out
    return replace(cfg, **upd)


def _solve(a) -> int:
    from .madp import MadpSolver
    cfg = _config(a)
    prob = hio.build_problem(cfg)
    scfg = hio.build_solver_config(cfg, prob.hierarchy)
    with MadpSolver(prob.hierarchy, scfg, workers=cfg.workers) as s:
        u, rep = s.solve(prob.rhs)
    path = os.path.join(cfg.out_dir, f"{prob.name}_report.csv")
    hio.write_report(rep, path)
    if cfg.write_solution or a.write_solution:
        hio.write_field(u, prob.hierarchy, os.path.join(cfg.out_dir, f"{prob.name}_field.csv"))
    print(f"{prob.name}: {rep.outer_iterations} outer iterations, relres {rep.final_relres:.3e}, "
          f"{rep.wall_ms:.1f} ms ({'converged' if rep.converged else 'cap reached'}); report: {path}")
    return 0 if rep.converged else 2


def _bench(a) -> int:
    import numpy as np
    import torch
    from . import _lib
    from .grid import mp1_problem
    from .operators import helmholtz_operator
    L = _lib.lib()
    rows = ["n,points,ms_per_apply,algorithmic_GBs,model_GFLOPs"]
    for n in (int(x) for x in a.sizes.split(",")):
        hier = mp1_problem(k=a.wavenumber, n=n, ml=2).hierarchy
        op = helmholtz_operator(hier, 1)
        rng = np.random.default_rng(1234)
        u = torch.from_numpy(rng.standard_normal(op.shape) + 1j * rng.standard_normal(op.shape)).cuda()
        out = torch.empty_like(u)
        h = op.handle
        for _ in range(3):
            _lib.check(L.hdb_op_apply(h, u.data_ptr(), out.data_ptr()))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            _lib.check(L.hdb_op_apply(h, u.data_ptr(), out.data_ptr()))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        pts = op.npoints
        rows.append(f"{n},{pts},{ms:.6f},{40.0 * pts / ms / 1e6:.1f},{11.0 * pts / ms / 1e6:.2f}")
    text = "\n".join(rows) + "\n"
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(text)
    sys.stdout.write(text)
    return 0


def _stencils(a) -> int:
    """Re-derive every level kernel with an independent 2D triple product and compare."""
    from .stencils import level_kernels
    w = (1, 4, 6, 4, 1)

    def coarsen_2d(rows, den):
        r = len(rows) // 2
        out = {}
        for dy in range(-3, 4):
            for dx in range(-3, 4):
                acc = 0
                for ay in range(-2, 3):
                    for ax in range(-2, 3):
                        for sy in range(-r, r + 1):
                            for sx in range(-r, r + 1):
                                v = rows[sy + r][sx + r]
                                ex, ey = ax + sx - 2 * dx, ay + sy - 2 * dy
                                if v and -2 <= ex <= 2 and -2 <= ey <= 2:
                                    acc += w[ax + 2] * w[ay + 2] * v * w[ex + 2] * w[ey + 2]
                out[(dx, dy)] = acc
        den *= 4096
        while den % 2 == 0 and all(v % 2 == 0 for v in out.values()):
            out = {k: v // 2 for k, v in out.items()}
            den //= 2
        return out, den

    bad = 0
    for level in range(2, 7):
        for i, (prev, cur) in enumerate(zip(level_kernels(level - 1), level_kernels(level))):
            tab, den = coarsen_2d(prev.numerators, prev.denominator)
            r = cur.radius
            ok = den == cur.denominator and all(tab.get((x, y), 0) == cur.numerators[y + r][x + r]
                                                for y in range(-r, r + 1) for x in range(-r, r + 1))
            ok = ok and all(v == 0 for (x, y), v in tab.items() if max(abs(x), abs(y)) > r)
            print(f"level {level} {'laplace' if i == 0 else 'mass'}: {'ok' if ok else 'MISMATCH'} "
                  f"(radius {r}, denominator {cur.denominator})")
            bad += not ok
    return 3 if (a.verify and bad) else 0


def main(argv=None) -> int:
    ap, a = _args(argv)
    if a.command is None:
        ap.print_usage(sys.stderr)
        return 1
    try:
        return {"solve": _solve, "bench": _bench, "stencils": _stencils}[a.command](a)
    except HelmdefError as exc:
        print(f"paper_2412_04980_b200: error: {exc}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
