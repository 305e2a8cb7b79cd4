"""MADP solver: outer FGMRES with the recursive A-DEF1 preconditioner on the GPU.

Drop-in for reference madp.py.  Policy types and presets (Definiteness,
classify_levels, LevelPolicy, SolverConfig, preset, ConvergenceReport) keep
the reference's fields and semantics (madp.py:63-217); the solve itself runs
in the CUDA library (csrc/engine.cu MadpSolver): per outer iteration the
A-DEF1 recursion (madp.py:301-327, lambda = 1)

    v_hat = Z^T v ; v_til ~ E^-1 v_hat (FGMRES on level l+1, recursive, or the
    coarsest CSLP-preconditioned FGMRES) ; t = Z v_til ; r = M^-1 (v - A t) ;
    return r + t

with CSLP by one multigrid V-cycle or GMRES(0.1, ceil(6 N^1/4)), all on device;
the host only drives Givens rotations and the recursion.
"""
from __future__ import annotations

import ctypes as C
import threading
import time
from dataclasses import dataclass, field

import numpy as np

from . import device as dev
from ._lib import check, lib
from .errors import BreakdownError, ConfigError, LevelError
from .grid import ComplexField, dimensionless_kmax, kh_of
from .krylov import StopRule, cslp_iteration_cap
from .mg import CslpMultigrid, MgConfig
from .operators import LevelOperator, cslp_operator, helmholtz_operator, level_ksq

__all__ = ["Definiteness", "classify_levels", "LevelPolicy", "SolverConfig", "ConvergenceReport", "preset",
           "PRESET_NAMES", "MadpSolver", "solve", "DEFINITENESS_THRESHOLD"]

INDEFINITE = "indefinite"
NEGATIVE_DEFINITE = "negative_definite"
DEFINITENESS_THRESHOLD = 2.0
PRESET_NAMES = ("MADP_V1", "MADP_V2", "MADP_V3", "MADP")
CSLP_MG, CSLP_GMRES, CSLP_BICGSTAB, CSLP_NONE = "mg", "gmres", "bicgstab", "none"
_CSLP_CODE = {CSLP_NONE: 0, CSLP_MG: 1, CSLP_GMRES: 2, CSLP_BICGSTAB: 3}


@dataclass(frozen=True)
class Definiteness:
    levels: tuple
    threshold: float

    def of(self, level: int) -> str:
        return self.levels[level - 1]

    def is_negative_definite(self, level: int) -> bool:
        return self.levels[level - 1] == NEGATIVE_DEFINITE


def classify_levels(hierarchy, threshold: float = DEFINITENESS_THRESHOLD) -> Definiteness:
    """Negative definite from the first level with max k*h_l >= threshold on (madp.py:77-84)."""
    out, flipped = [], False
    for l in range(1, hierarchy.ml + 1):
        flipped = flipped or kh_of(l, hierarchy) >= threshold
        out.append(NEGATIVE_DEFINITE if flipped else INDEFINITE)
    return Definiteness(tuple(out), threshold)


@dataclass(frozen=True)
class LevelPolicy:
    level: int
    cslp_method: str
    cslp_shift: float
    cslp_stop: StopRule
    deflation_cycle_stop: StopRule | None

    def __post_init__(self):
        if self.cslp_method not in (CSLP_MG, CSLP_GMRES, CSLP_BICGSTAB, CSLP_NONE):
            raise ConfigError(f"unknown CSLP method {self.cslp_method!r}")


@dataclass(frozen=True)
class SolverConfig:
    ml: int
    policies: tuple
    outer_stop: StopRule = StopRule(1e-6, 150)
    preset_name: str = "custom"
    beta1: float = 1.0
    mg_config: MgConfig = field(default_factory=MgConfig)

    def __post_init__(self):
        if len(self.policies) != self.ml:
            raise ConfigError("one LevelPolicy per level is required")
        if self.policies[0].deflation_cycle_stop is not None:
            raise ConfigError("the finest level has no deflation cycle rule")
        if self.policies[-1].deflation_cycle_stop is None:
            raise ConfigError("the coarsest level needs a solve rule")

    def policy(self, level: int) -> LevelPolicy:
        return self.policies[level - 1]


def preset(name: str, hierarchy, threshold: float = DEFINITENESS_THRESHOLD,
           outer_stop: StopRule = StopRule(1e-6, 150)) -> SolverConfig:
    """Named configurations MADP_V1/V2/V3/MADP (madp.py:129-189)."""
    if name not in PRESET_NAMES:
        raise ConfigError(f"unknown preset {name!r} (expected one of {PRESET_NAMES})")
    ml = hierarchy.ml
    classes = classify_levels(hierarchy, threshold)
    if name in ("MADP_V1", "MADP_V2"):
        shift = 1.0 / dimensionless_kmax(hierarchy)
        beta2 = {l: shift for l in range(1, ml + 1)}
        method = {l: CSLP_GMRES for l in range(1, ml + 1)}
        second = StopRule(0.1, 100) if name == "MADP_V2" else StopRule(1.0, 1)
    else:
        beta2 = {l: 0.5 for l in range(1, ml + 1)}
        method = {l: (CSLP_MG if l <= 2 else CSLP_GMRES) for l in range(1, ml + 1)}
        method[ml] = CSLP_GMRES
        second = StopRule(0.3 if name == "MADP" else 0.1, 100)
    coarsest = StopRule(1.0, 1) if classes.is_negative_definite(ml) else StopRule(0.1, 100)
    pols = []
    for l in range(1, ml + 1):
        if l == 1:
            cyc = None
        elif l == ml:
            cyc = coarsest
        elif l == 2:
            cyc = second
        else:
            cyc = StopRule(1.0, 1)
        pols.append(LevelPolicy(l, method[l], beta2[l], StopRule(0.1, cslp_iteration_cap(hierarchy.level(l).npoints)),
                                cyc))
    return SolverConfig(ml=ml, policies=tuple(pols), outer_stop=outer_stop, preset_name=name)


@dataclass
class ConvergenceReport:
    outer_iterations: int
    converged: bool
    final_relres: float
    residual_history: list
    wall_ms: float
    iteration_wall_ms: list
    preset_name: str
    levels: int
    workers: int
    cycle_iters: dict
    cslp_iters: dict
    matvecs: dict
    model_flops: float
    model_bytes: float
    device_ms: float = 0.0
    alg_bytes: float = 0.0   # algorithmic HBM bytes of the solve's kernels (device solver telemetry)

    def cycle_max(self, level: int) -> int:
        v = self.cycle_iters.get(level, [])
        return max(v) if v else 0

    def cslp_max(self, level: int) -> int:
        v = self.cslp_iters.get(level, [])
        return max(v) if v else 0


def _model_flops_per_point(radius):
    return 11 if radius == 1 else 9 * (2 * radius + 1) ** 2


def _model_bytes_per_point(radius):
    return 56 if radius == 1 else 16 * ((2 * radius + 1) ** 2 + 2) + 8 * (2 * radius + 1) ** 2


class MadpSolver:
    """Outer FGMRES with the recursive multilevel A-DEF1 preconditioner (GPU)."""

    def __init__(self, hierarchy, config: SolverConfig, workers: int = 1, dist=None):
        """dist: optional distributed.DistContext — row-slab solve over dist.size ranks
        (each rank passes the full rhs and gets its own slab of the solution)."""
        if config.ml != hierarchy.ml:
            raise ConfigError(f"config has {config.ml} levels but the hierarchy has {hierarchy.ml}")
        self.hierarchy, self.config = hierarchy, config
        self.workers = max(1, int(workers))
        self.dist = dist
        self.plan = None
        spec = lambda depth: None  # noqa: E731
        if dist is not None and dist.size > 1:
            from .distributed import slab_plan
            ny = hierarchy.level(1).ny
            # every grid depth a level or a multigrid sub-level can reach
            max_depth = 1
            while (ny - 1) % 2 ** max_depth == 0 and (ny - 1) // 2 ** max_depth + 1 >= 3:
                max_depth += 1
            self.plan = slab_plan(ny, dist.size, max_depth, dist.min_rows)
            spec = lambda depth: self.plan.spec(depth, dist.rank)  # noqa: E731
        self._spec = spec
        self.A: dict[int, LevelOperator] = {}
        self.M: dict[int, LevelOperator] = {}
        self.mg: dict[int, CslpMultigrid] = {}
        for l in range(1, hierarchy.ml + 1):
            pol = config.policy(l)
            self.A[l] = helmholtz_operator(hierarchy, l, slab=spec(l - 1))
            if pol.cslp_method in (CSLP_GMRES, CSLP_BICGSTAB):
                self.M[l] = cslp_operator(hierarchy, l, pol.cslp_shift, config.beta1, slab=spec(l - 1))
            elif pol.cslp_method == CSLP_MG:
                lv = hierarchy.level(l)
                self.mg[l] = CslpMultigrid(lv.nx, lv.ny, lv.h, level_ksq(hierarchy, l), hierarchy.boundary,
                                           beta2=pol.cslp_shift, beta1=config.beta1, config=config.mg_config,
                                           slabs=(lambda s, l=l: spec(l - 1 + s)))
        self._h = None

    # -- device solver -------------------------------------------------------
    @property
    def handle(self):
        if self._h is None:
            L = lib()
            cfg = self.config
            h = C.c_void_p()
            check(L.hdb_solver_create(C.byref(h), cfg.ml, float(cfg.outer_stop.rel_tol),
                                      int(cfg.outer_stop.max_iters)))
            for l in range(1, cfg.ml + 1):
                pol = cfg.policy(l)
                cyc = pol.deflation_cycle_stop or StopRule(1.0, 1)
                check(L.hdb_solver_set_level(h, l, self.A[l].handle, self.M[l].handle if l in self.M else None,
                                             self.mg[l].handle if l in self.mg else None,
                                             _CSLP_CODE[pol.cslp_method], float(pol.cslp_stop.rel_tol),
                                             int(pol.cslp_stop.max_iters), float(cyc.rel_tol), int(cyc.max_iters)))
            self._h = h
        return self._h

    def close(self):
        if self._h is not None:
            from . import _lib
            if _lib._lib is not None:
                _lib._lib.hdb_solver_destroy(self._h)
            self._h = None
        for d in (self.mg, self.M, self.A):
            for o in d.values():
                o.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            if self._h is not None and lib is not None:
                from . import _lib
                if _lib._lib is not None:
                    _lib._lib.hdb_solver_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def apply_preconditioner(self, level: int, v):
        """One A-DEF1 application at ``level`` (madp.py:301-327)."""
        if not 1 <= level < self.hierarchy.ml:
            raise LevelError(f"preconditioner level {level} outside 1..{self.hierarchy.ml - 1}")
        host = not dev.is_device(v)
        dv = dev.to_device(v)
        out = dev.empty(tuple(v.shape))
        check(lib().hdb_solver_precond(self.handle, level, dv.data_ptr(), out.data_ptr()))
        return dev.to_host(out) if host else out

    def solve_device(self, b_dev, x_dev):
        """Device-resident solve: b, x torch CUDA complex128 tensors of the fine grid."""
        check(lib().hdb_solver_solve(self.handle, b_dev.data_ptr(), x_dev.data_ptr(), 0))
        return self.report()

    def solve(self, b):
        """Run the outer solve; returns (ComplexField, ConvergenceReport) (madp.py:329-371).

        numpy input: host buffers go through the library call (copies included);
        torch CUDA input: solved in place on the device, x returned as a tensor."""
        b2d = b.grid_view(self.hierarchy) if isinstance(b, ComplexField) else b
        shape = self.hierarchy.level(1).shape
        if tuple(b2d.shape) != shape:
            from .errors import ShapeError
            raise ShapeError(f"rhs shape {tuple(b2d.shape)} != {shape}")
        t0 = time.perf_counter()
        sl = self._spec(0)
        if sl is not None:  # distributed: this rank's slab in, this rank's slab out (host buffers)
            hb = np.ascontiguousarray(np.asarray(b2d)[sl.row0:sl.row0 + sl.ny], dtype=np.complex128)
            hx = np.empty_like(hb)
            check(lib().hdb_solver_solve(self.handle, hb.ctypes.data, hx.ctypes.data, 1))
            return hx, self.report(wall_ms=(time.perf_counter() - t0) * 1e3)
        if dev.is_device(b2d):
            db = b2d.to(dev.torch_mod().complex128).contiguous()
            x = dev.empty(shape)
            check(lib().hdb_solver_solve(self.handle, db.data_ptr(), x.data_ptr(), 0))
            out = x
        else:
            hb = np.ascontiguousarray(b2d, dtype=np.complex128)
            hx = np.empty(shape, dtype=np.complex128)
            # First-touch the result pages on a host thread while the GPU solves (the
            # library call releases the GIL), so the final device -> host copy does not
            # pay the page faults of a fresh array (config 2: 268 MB).  The copy into hx
            # starts only after the toucher has finished.
            toucher = threading.Thread(target=hx.fill, args=(0.0,))
            toucher.start()
            try:
                db = dev.to_device(hb)
                dx = dev.empty(shape)
                check(lib().hdb_solver_solve(self.handle, db.data_ptr(), dx.data_ptr(), 0))
            finally:
                toucher.join()
            dev.copy_to_host(dx, hx)
            out = ComplexField(level=1, data=hx.ravel())
        rep = self.report(wall_ms=(time.perf_counter() - t0) * 1e3)
        return out, rep

    def profile(self) -> dict:
        """Per-level inclusive host time of the last solve (telemetry)."""
        ml = self.hierarchy.ml
        n = (ml + 1) * 3
        ms, calls = (C.c_double * n)(), (C.c_longlong * n)()
        syncs, launches = C.c_longlong(), C.c_longlong()
        check(lib().hdb_solver_profile(self.handle, ms, calls, n, C.byref(syncs), C.byref(launches)))
        roles = ("deflation_fgmres", "cslp", "adef1")
        out = {"syncs": syncs.value, "launches": launches.value, "levels": {}}
        for l in range(1, ml + 1):
            out["levels"][l] = {roles[k]: {"ms": round(ms[l * 3 + k], 3), "calls": calls[l * 3 + k]}
                                for k in range(3) if calls[l * 3 + k]}
        return out

    def report(self, wall_ms=None) -> ConvergenceReport:
        L = lib()
        h = self.handle
        its, conv, fin, dms, hl = C.c_int(), C.c_int(), C.c_double(), C.c_double(), C.c_int()
        check(L.hdb_solver_report(h, C.byref(its), C.byref(conv), C.byref(fin), C.byref(dms), C.byref(hl)))
        hist = (C.c_double * max(1, hl.value))()
        iw = (C.c_double * max(1, hl.value))()
        check(L.hdb_solver_history(h, hist, iw, hl.value))
        ml = self.hierarchy.ml
        cyc, csl = {}, {}
        for l in range(1, ml + 1):
            for kind, dst in ((0, cyc), (1, csl)):
                if kind == 0 and l == 1:
                    continue
                cnt = C.c_int()
                check(L.hdb_solver_counts(h, l, kind, None, 0, C.byref(cnt)))
                buf = (C.c_int * max(1, cnt.value))()
                check(L.hdb_solver_counts(h, l, kind, buf, cnt.value, C.byref(cnt)))
                dst[l] = list(buf[: cnt.value])
        mv = (C.c_longlong * (ml + 1))()
        check(L.hdb_solver_matvecs(h, mv, ml + 1))
        matvecs = {l: int(mv[l]) for l in range(1, ml + 1)}
        flops = sum(matvecs[l] * _model_flops_per_point(self.A[l].radius) * self.A[l].npoints for l in matvecs)
        nbytes = sum(matvecs[l] * _model_bytes_per_point(self.A[l].radius) * self.A[l].npoints for l in matvecs)
        n_it = its.value
        ab = C.c_double()
        check(L.hdb_solver_bytes(h, C.byref(ab)))
        return ConvergenceReport(
            outer_iterations=n_it, converged=bool(conv.value), final_relres=fin.value,
            residual_history=list(hist[: hl.value]),
            wall_ms=dms.value if wall_ms is None else wall_ms,
            iteration_wall_ms=[0.0] + list(iw[:n_it]), preset_name=self.config.preset_name,
            levels=ml, workers=self.workers, cycle_iters=cyc, cslp_iters=csl, matvecs=matvecs,
            model_flops=float(flops), model_bytes=float(nbytes), device_ms=dms.value, alg_bytes=ab.value)


def solve(problem, config: SolverConfig, workers: int = 1) -> tuple:
    """Solve a problem with a solver configuration; see :class:`MadpSolver`."""
    with MadpSolver(problem.hierarchy, config, workers=workers) as s:
        return s.solve(problem.rhs)


_ = BreakdownError  # re-exported through the package namespace
