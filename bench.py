"""Benchmark: MADP-FGMRES time-to-solution on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c5|...] [--impl ours|reference]

Workload: N = 1 defaults to BASELINE configs[1] (k=200, 4097^2, Sommerfeld,
ml=7, MADP; the configuration the metric is quoted on); N > 1 (torchrun)
defaults to BASELINE configs[4], the weak-scaling sweep (8193 x (8192 N + 1)
points, 8192^2 per GPU, k^3 h^2 = 0.5) in row slabs over the ranks.  One step =
one full solve.  Synthetic by construction (the reference's own problem
generator; no dataset).

Printed JSON (rank 0, one line):
  value          device time of one solve (CUDA events on the library stream,
                 b and x resident in HBM), mean over K timed steps, max over ranks
  e2e            same solve through the public API  MadpSolver.solve(numpy b):
                 H2D of b + solve + D2H of x, host wall clock
  solve_bandwidth  algorithmic HBM bytes of every launch of one solve (host-driver
                 counters, SURVEY §8(d) per-point figures) / device time
  roofline       the solve's dominant HBM-bound kernel family, timed live: one
                 extra solve with a CUDA-event pair on the library stream around
                 every launch; achieved = its algorithmic bytes / its summed
                 event time, vs the measured copy peak (MEASURED_PEAKS.json)
  kernel_families  the same per-family table (launches, ms, GB/s, share)
  kernels        isolated fine-level kernel microbench (CUDA events)
  cpu_baseline   the CPU oracle (oracle/, bit-exact restatement of the
                 reference) on a bounded sample of the same workload, scaled by
                 the reference run's work counts, with a live model check: a
                 full measured CPU solve of the config-2 analogue vs the same model
  gpu_launches   kernels launched by libhdb200 inside the timed region, per step
Fine-level vectors are 268 MB (> 126 MB L2), so no explicit L2 flush is needed.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "solve time & outer iters at 1/2/4/8 B200; stencil HBM GB/s vs roofline"
C5_K = (0.5 * 8192.0 ** 2) ** (1.0 / 3.0)


def _oracle_c5(P):
    import oracle
    hier = oracle.build_hierarchy(((0.0, 1.0), (0.0, float(P))), 1.0 / 8192, 7, k=C5_K)
    return hier, oracle.point_source(hier, (0.5, P / 2.0))


CONFIGS = {
    # name: (description, product builder (hdb, P), oracle builder (P) -> (hierarchy, b))
    "c2": ("BASELINE configs[1]: k=200, 4097^2, Sommerfeld, ml=7, MADP",
           lambda hdb, P: hdb.mp1_problem(k=200.0, n=4097, ml=7, boundary="sommerfeld"),
           lambda P: __import__("oracle").mp1_problem(200.0, 4097, 7)),
    "c2a": ("config-2 analogue: k=100, 1025^2, Sommerfeld, ml=6, MADP",
            lambda hdb, P: hdb.mp1_problem(k=100.0, n=1025, ml=6, boundary="sommerfeld"),
            lambda P: __import__("oracle").mp1_problem(100.0, 1025, 6)),
    "c1s": ("config 1 with Sommerfeld: k=50, 129^2, ml=2, MADP",
            lambda hdb, P: hdb.mp1_problem(k=50.0, n=129, ml=2, boundary="sommerfeld"),
            lambda P: __import__("oracle").mp1_problem(50.0, 129, 2)),
    "c3_40": ("BASELINE configs[2] @40 Hz: wedge 600x1000 m, h=0.5 m, 1201x2001, ml=5, MADP",
              lambda hdb, P: hdb.wedge_problem(f=40.0, nx=1201, ml=5, layers=hdb.grid.BASELINE_WEDGE_LAYERS),
              lambda P: __import__("oracle").baseline_wedge_problem(40.0)),
    "c5": ("BASELINE configs[4] weak scaling: 8193 x (8192 P + 1) on P GPUs, h=1/8192, k^3 h^2 = 0.5, ml=7",
           lambda hdb, P: hdb.c5_problem(P), _oracle_c5),
    "c4_40": ("BASELINE configs[3] @40 Hz: seeded folded/faulted layers 9192x3000 m, h=0.75 m (12257x4001), ml=6",
              lambda hdb, P: hdb.synthetic_layered_problem(40.0, 0.75, 6), None),
}

# outer iterations and level-2 deflation-cycle counts of a full solve, for the CPU
# work model where no committed reference record exists (GPU runs, counts equal to
# the reference's wherever a reference record exists)
GPU_COUNTS = {"c5": 41, "c3_40": 19}


def config_dict(name, hier):
    """The `config` object printed by BOTH arms (identical by construction)."""
    lv = hier.level(1)
    return {"workload": CONFIGS[name][0], "grid": f"{lv.nx}x{lv.ny}", "levels": hier.ml,
            "points": lv.npoints, "l2_flush": "inputs larger than L2 (fine-level vectors >= 38 MB; "
            "268 MB at config 2)" if lv.npoints * 16 > 126e6 or name == "c2" else "none (small case)"}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, torch copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.proc, self.lines = index, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _allmax(val, ws):
    if ws == 1:
        return val
    import torch
    import torch.distributed as dist
    t = torch.tensor([val], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def ncu_traffic(family, config):
    """dram read + write bytes per launch of the roofline kernel from the committed
    `ncu --set full` capture (profiles/r02_roofline_ncu.json), or None."""
    path = os.path.join(ROOT, "profiles", "r02_roofline_ncu.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d["families"][family]
        if d.get("config") != config:
            return None, None
        return e["traffic_bytes_per_launch"], d.get("source")
    except (OSError, KeyError, ValueError):
        return None, None


# FP64 operations per output point of the exact (no-FMA) Galerkin stencils on a
# constant-k level: 8 per tap (complex multiply by the precomputed tap
# coefficient + complex accumulate), 49 / 25 taps
FP64_OPS_PER_POINT = {"stencil7_apply_L3": 8 * 49, "stencil5x5_apply_L2": 8 * 25}


def kernel_entry(name, v, peak):
    e = {"gbs": round(v["gbs"], 1), "ms": round(v["ms"], 4), "frac": round(v["gbs"] / peak, 3)}
    ops = FP64_OPS_PER_POINT.get(name)
    if ops and v.get("fp64_bound", True):
        mhz = 1965.0
        pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
        if os.path.exists(pk):
            mhz = float(json.load(open(pk)).get("sm_max_mhz", mhz))
        fp64_peak = 148 * 64 * mhz * 1e6
        pts = v["bytes"] / 40.0
        e.update({"fp64_ops_per_point_exact_form": ops,
                  "fp64_frac_exact_form": round(pts * ops / (v["ms"] * 1e-3) / fp64_peak, 3)})
    return e


def kernel_roofline(hdb, hier, reps=20):
    """Isolated fine-level kernels, timed with CUDA events on the library stream
    (= torch's current stream)."""
    import torch
    from paper_2412_04980_b200 import _lib
    L = _lib.lib()
    lv = hier.level(1)
    op = hdb.helmholtz_operator(hier, 1)
    n = lv.npoints
    rng = np.random.default_rng(1234)
    u = torch.from_numpy(rng.standard_normal(lv.shape) + 1j * rng.standard_normal(lv.shape)).cuda()
    out = torch.empty_like(u)
    b = torch.empty_like(u)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timeit(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(reps):
            fn()
        ev1.record()
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) / reps * 1e-3

    res = {}
    h = op.handle
    res["stencil5_apply"] = (40.0 * n, timeit(lambda: _lib.check(L.hdb_op_apply(h, u.data_ptr(), out.data_ptr()))))
    res["stencil5_residual"] = (56.0 * n, timeit(
        lambda: _lib.check(L.hdb_op_residual(h, b.data_ptr(), u.data_ptr(), out.data_ptr()))))
    mg = hdb.CslpMultigrid(lv.nx, lv.ny, lv.h, hier.ksq_at(1), hier.boundary, beta2=0.5)
    sop = mg.levels[0].op.handle
    res["jacobi5"] = (56.0 * n, timeit(
        lambda: _lib.check(L.hdb_op_jacobi(sop, u.data_ptr(), b.data_ptr(), out.data_ptr(), 0.8))))
    c = torch.empty(hier.level(2).shape, dtype=torch.complex128, device="cuda")
    res["restrict"] = (20.0 * n, timeit(lambda: _lib.check(L.hdb_restrict(u.data_ptr(), lv.ny, lv.nx, c.data_ptr(), 0))))
    res["prolong"] = (20.0 * n, timeit(
        lambda: _lib.check(L.hdb_prolong(c.data_ptr(), lv.ny, lv.nx, None, out.data_ptr()))))
    # reference streams (torch kernels, not ours): pure write and read+write copy of one fine vector
    res["ref_write_only(torch fill)"] = (16.0 * n, timeit(lambda: out.fill_(0.5)))
    res["ref_copy(torch)"] = (32.0 * n, timeit(lambda: out.copy_(u)))
    res["dot"] = (32.0 * n, timeit(lambda: _lib.check(L.hdb_dot(u.data_ptr(), out.data_ptr(), n, None))))
    # fused matvec + residual + norms (MG divergence guard): one pass, residual not stored
    res["stencil5_resnorm_fused"] = (40.0 * n, timeit(
        lambda: _lib.check(L.hdb_op_resnorm(sop, b.data_ptr(), u.data_ptr(), None))))

    def unfused():  # the sequence it replaces: residual (56 B/pt) + 2 dots (32 B/pt each)
        _lib.check(L.hdb_op_residual(sop, b.data_ptr(), u.data_ptr(), out.data_ptr()))
        _lib.check(L.hdb_dot(out.data_ptr(), out.data_ptr(), n, None))
        _lib.check(L.hdb_dot(b.data_ptr(), b.data_ptr(), n, None))
    res["stencil5_resnorm_unfused(3 launches)"] = (40.0 * n, timeit(unfused))
    if hier.ml >= 3:
        for lvl, name in ((3, "stencil7_apply_L3"), (2, "stencil5x5_apply_L2")):
            opl = hdb.helmholtz_operator(hier, lvl)
            ll = hier.level(lvl)
            ul = torch.from_numpy(rng.standard_normal(ll.shape) + 1j * rng.standard_normal(ll.shape)).cuda()
            ol = torch.empty_like(ul)
            hl = opl.handle
            res[name] = (40.0 * ll.npoints, timeit(lambda: _lib.check(L.hdb_op_apply(hl, ul.data_ptr(), ol.data_ptr()))))
    return {k: {"bytes": bts, "ms": tt * 1e3, "gbs": bts / tt / 1e9} for k, (bts, tt) in res.items()}


# kernel families (csrc/engine.h KFam) that stream HBM; the others are latency /
# synchronisation work (resident Krylov solves, control kernels)
HBM_FAMILIES = ("apply5", "residual5", "jacobi5", "resnorm5", "galerkin", "restrict", "prolong", "mgs_coop",
                "mgs_chain", "blas1", "resrestrict")
FAMILY_KERNELS = {"mgs_coop": "k_mgs_ls (one-launch low-synchronisation MGS step, Arnoldi of the launch-driven "
                              "levels; k_mgs_grid_t / k_mgs_grid2 in the MGS-order mode)",
                  "galerkin": "k_rgs<2/3> (separable radius-2 / radius-3 Galerkin stencils)",
                  "resrestrict": "k_resrestrict (fused MG residual + restriction)",
                  "apply5": "k_r1w<0> (5-point apply)", "residual5": "k_r1w<1> (5-point residual)",
                  "jacobi5": "k_r1w<2,3> (Jacobi sweep)", "mgs_chain": "k_mgs (fused MGS launches)",
                  "restrict": "k_restrict_t (TMA Z^T)", "prolong": "k_prolong_t (TMA Z)",
                  "resnorm5": "k_resnorm (fused residual norms)", "blas1": "dot/scale/add/lincomb"}


def family_profile(solver, b_dev, x_dev):
    """One extra solve with a CUDA-event pair around every launch (library stream)."""
    from paper_2412_04980_b200 import _lib
    import torch
    _lib.kprof(True)
    rep = solver.solve_device(b_dev, x_dev)
    torch.cuda.synchronize()
    fams = _lib.kprof_read()
    _lib.kprof(False)
    tot_ms = sum(v["device_ms"] for v in fams.values())
    out = {}
    for name, v in fams.items():
        if v["launches"] == 0:
            continue
        e = {"launches": v["launches"], "ms": round(v["device_ms"], 3),
             "share": round(v["device_ms"] / tot_ms, 4) if tot_ms else None,
             "alg_MB": round(v["alg_bytes"] / 1e6, 1)}
        if v["device_ms"] > 0 and v["alg_bytes"] > 0:
            e["gbs"] = round(v["alg_bytes"] / (v["device_ms"] * 1e-3) / 1e9, 1)
        out[name] = e
    return out, rep.device_ms, rep.outer_iterations


def roofline_entry(fams, peak, peak_src, config):
    """Dominant HBM-bound family by measured time -> the bench's roofline object."""
    hbm = {k: v for k, v in fams.items() if k in HBM_FAMILIES and v.get("gbs")}
    if not hbm:
        return None
    name = max(hbm, key=lambda k: hbm[k]["ms"])
    v = hbm[name]
    per_launch_bytes = v["alg_MB"] * 1e6 / v["launches"]
    traffic, ncu_src = ncu_traffic(name, config)
    return {"bound": "hbm", "kernel": f"{name}: {FAMILY_KERNELS.get(name, name)}",
            "achieved": v["gbs"], "peak": peak, "unit": "GB/s", "frac": round(v["gbs"] / peak, 4),
            "traffic": traffic,
            "traffic_source": (f"profiles/r02_roofline_ncu.json: {ncu_src} (dram read+write, mean per captured "
                               f"launch)") if traffic else None,
            "peak_source": peak_src, "share_of_solve": v["share"], "launches_per_solve": v["launches"],
            "algorithmic_bytes_per_launch": round(per_launch_bytes), "us_per_launch": round(v["ms"] * 1e3 / v["launches"], 2),
            "how": "one extra solve after the timed steps with a CUDA-event pair on the library stream around "
                   "every launch; achieved = the family's algorithmic bytes (SURVEY 8(d): 16 (j+1) + 32 B/pt for "
                   "the MGS step at Arnoldi step j) / its summed event time"}


# ------------------------------------------------------------------ CPU baseline
def _work_units(cycle_iters_l2, n_outer):
    """Cost model of one MADP outer iteration: 1 + its level-2 deflation cycles
    (every level-2 FGMRES iteration runs the whole coarse recursion once)."""
    c = list(cycle_iters_l2)[:n_outer] + [0] * max(0, n_outer - len(cycle_iters_l2))
    return [1 + x for x in c]


def reference_counts(config):
    """Outer iterations and level-2 cycle counts of the REFERENCE's own run of this
    config (committed fixtures; the oracle reproduces the reference bit for bit)."""
    name = {"c2": "solve_c2.npz", "c2a": "solve_c2a.npz", "c1s": "solve_c1s.npz",
            "c3_40": "solve_c3_40.npz"}.get(config)
    path = os.path.join(ROOT, "tests", "golden", name) if name else None
    if path is None or not os.path.exists(path):
        return None
    import ast
    g = np.load(path, allow_pickle=False)
    txt = str(g["cycle_iters"])
    cyc = json.loads(txt) if txt.startswith("{\"") else ast.literal_eval(txt)
    cyc = {int(k): v for k, v in cyc.items()}
    return int(g["outer_iterations"]), cyc.get(2, [])


def host_info():
    info = {"threads": len(os.sched_getaffinity(0))}
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                info["cpu"] = ln.split(":", 1)[1].strip()
                break
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal"):
                info["ram_gb"] = round(int(ln.split()[1]) / 2 ** 20, 1)
                break
    except OSError:
        pass
    return info


def _oracle_solver(config, P=1):
    import oracle
    hier, b = CONFIGS[config][2](P)
    pols, outer = oracle.madp_preset(hier)
    return oracle.CpuMadpSolver(hier, pols, outer), b


def _oracle_warm():
    import oracle
    th, tb = oracle.mp1_problem(10.0, 33, 3)
    tp, to = oracle.madp_preset(th)
    oracle.CpuMadpSolver(th, tp, to).solve(tb)


def cpu_sample(config, outer_its=None, cycle_l2=None, P=1, workers=None, max_outer=1):
    """Oracle on the first `max_outer` outer iteration(s) of the config, scaled to
    the whole solve by the work model (outer iterations + level-2 cycles) with the
    reference run's counts where committed, else the given (GPU) counts."""
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_oracle")
    from oracle import ops as oracle_ops
    cores = oracle_ops.set_workers(workers or len(os.sched_getaffinity(0)))
    _oracle_warm()
    s, b = _oracle_solver(config, P)
    t0 = time.perf_counter()
    _, rep = s.solve(b, max_outer=max_outer)
    dt = time.perf_counter() - t0
    ref = reference_counts(config)
    src = "reference run"
    if ref is not None:
        outer_its, cycle_l2 = ref
    else:
        src = "GPU run"
        outer_its = outer_its or GPU_COUNTS.get(config, rep.iterations)
        cycle_l2 = cycle_l2 or []
    w = _work_units(cycle_l2, outer_its)
    sampled = sum(_work_units(s.cycle_iters.get(2, []), rep.iterations))
    scale = sum(w) / max(1, sampled)
    return {"value": dt * scale, "sample_s": dt, "scale": scale, "cores": cores, "units": sum(w),
            "sampled_units": sampled, "outer_its": outer_its, "count_source": src}


def cpu_full(config, workers=None):
    """A full measured oracle solve (the model check)."""
    from oracle import ops as oracle_ops
    cores = oracle_ops.set_workers(workers or len(os.sched_getaffinity(0)))
    _oracle_warm()
    s, b = _oracle_solver(config)
    t0 = time.perf_counter()
    _, rep = s.solve(b)
    return {"value": time.perf_counter() - t0, "cores": cores, "outer_its": rep.iterations}


def cpu_baseline(config, outer_its, cycle_l2=None, check=True):
    cb = cpu_sample(config, outer_its, cycle_l2)
    out = {"value": cb["value"], "unit": "s", "cores": cb["cores"], "kind": "port",
           "sample": (f"oracle (bit-exact CPU restatement of helmdef; numba stencil loops on row slabs over "
                      f"{cb['cores']} host threads as the reference's WorkerPool) on the first outer iteration of "
                      f"the same solve: {cb['sample_s']:.2f} s for {cb['sampled_units']} work units, scaled "
                      f"x{cb['scale']:.1f} to the {cb['outer_its']}-iteration solve ({cb['units']} units = outer "
                      f"iterations + level-2 cycles, counts of the {cb['count_source']})"),
           "host": host_info()}
    if check and config != "c2a":
        # model check on the same host: full measured solve of the config-2 analogue vs the
        # same one-iteration sample + work model; and the single-thread sample
        full = cpu_full("c2a")
        mod = cpu_sample("c2a")
        one = cpu_sample("c2a", workers=1)
        out["model_check"] = {"case": "c2a (k=100, 1025^2, ml=6)", "measured_full_s": round(full["value"], 2),
                              "model_s": round(mod["value"], 2),
                              "model_over_measured": round(mod["value"] / full["value"], 3),
                              "cores": full["cores"], "model_1thread_s": round(one["value"], 2)}
    cal = os.path.join(ROOT, "profiles", "r02_cpu_calibration.json")
    if os.path.exists(cal):
        out["calibration_file"] = "profiles/r02_cpu_calibration.json"
    return out


def run_reference(args, ws):
    _, rank, _ = _dist()
    if rank != 0:
        return
    import paper_2412_04980_b200 as hdb
    P = ws if args.config == "c5" else 1
    hier = CONFIGS[args.config][1](hdb, P).hierarchy
    steps = []
    cb = None
    # warm-up steps run the same bounded sample (numba JIT is compiled on a tiny case first)
    for k in range(args.warmup + args.steps):
        cb = cpu_sample(args.config, P=min(P, 1) if args.config == "c5" else 1)
        if args.config == "c5" and P > 1:  # weak scaling: P independent 8192^2 slabs' worth of work
            cb["value"] *= P
        if k >= args.warmup:
            steps.append(cb["value"])
    val = float(np.mean(steps))
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": "s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": val * 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": config_dict(args.config, hier),
            "cpu_baseline": {"value": val, "unit": "s", "cores": cb["cores"], "kind": "port",
                             "sample": (f"oracle on the first outer iteration ({cb['sample_s']:.2f} s, "
                                        f"{cb['sampled_units']} work units) scaled x{cb['scale']:.1f} to the "
                                        f"{cb['outer_its']}-iteration solve (counts of the {cb['count_source']})"
                                        + (f", x{P} for the P-slab weak-scaling grid (sampled on one 8192^2 slab)"
                                           if args.config == "c5" and P > 1 else "")),
                             "host": host_info()},
            "e2e": {"value": val, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None, choices=sorted(CONFIGS),
                    help="default: c2 on one GPU, c5 (weak scaling) on several")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-model-check", action="store_true", help="skip the full CPU solve of the model check")
    args = ap.parse_args()
    ws, rank, local = _dist()
    if args.config is None:
        args.config = "c5" if ws > 1 else "c2"
    if args.impl == "reference":
        return run_reference(args, ws)

    import torch
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    import paper_2412_04980_b200 as hdb
    from paper_2412_04980_b200 import _lib
    L = _lib.lib()

    prob = CONFIGS[args.config][1](hdb, ws)
    hier = prob.hierarchy
    cfg = hdb.preset("MADP", hier)
    dist_ctx = None
    if ws > 1:  # row slabs over the ranks: NCCL halos / dots, replicated coarse levels
        from paper_2412_04980_b200.distributed import DistContext
        dist_ctx = DistContext.nccl(rank, ws)
    solver = hdb.MadpSolver(hier, cfg, dist=dist_ctx)
    b_host = prob.rhs.grid_view(hier)
    sl = solver._spec(0)
    if sl is not None:
        b_host = np.ascontiguousarray(b_host[sl.row0:sl.row0 + sl.ny])
    shape = b_host.shape
    b_dev = torch.from_numpy(b_host.copy()).cuda()
    x_dev = torch.empty_like(b_dev)
    b_pin = torch.empty(shape, dtype=torch.complex128, pin_memory=True)
    b_pin.copy_(torch.from_numpy(b_host))
    b_pin_np = b_pin.numpy()

    for _ in range(args.warmup):
        rep = solver.solve_device(b_dev, x_dev)
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    l0 = C_launches(L)
    times, nbytes = [], []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            torch.cuda.synchronize()
            rep = solver.solve_device(b_dev, x_dev)
            times.append(rep.device_ms / 1e3)
            nbytes.append(rep.alg_bytes)
        torch.cuda.synchronize()
    launches = C_launches(L) - l0
    if ws > 1:
        torch.distributed.barrier()
    t_step = _allmax(float(np.mean(times)), ws)

    # end-to-end through the public API (numpy in pinned memory -> numpy out)
    e2e = []
    b_api = prob.rhs.grid_view(hier) if sl is not None else b_pin_np  # distributed API takes the full rhs
    for k in range(max(1, args.steps)):
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        u, rep_e = solver.solve(b_api)
        e2e.append(time.perf_counter() - t0)
    e2e_t = _allmax(float(np.mean(e2e)), ws)

    peak, peak_src = _peaks()
    fams, prof_ms, prof_its = family_profile(solver, b_dev, x_dev) if rank == 0 else ({}, None, None)
    kern = kernel_roofline(hdb, hier) if (rank == 0 and ws == 1) else {}
    if rank == 0:
        cpu = None
        if not args.no_cpu and ws == 1:
            try:
                cpu = cpu_baseline(args.config, rep.outer_iterations, rep.cycle_iters.get(2, []),
                                   check=not args.no_model_check)
            except Exception as err:  # noqa: BLE001
                cpu = {"value": None, "unit": "s", "cores": 1, "kind": "port", "sample": f"failed: {err}"}
        alg = float(np.mean(nbytes))
        out_line = {
            "metric": METRIC, "value": t_step, "unit": "s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
            "config": config_dict(args.config, hier),
            "parallelism": (f"row slabs x{ws} ({solver.plan.depths} sharded grid depths, coarser replicated)"
                            if ws > 1 else "single GPU"),
            "outer_iters": rep.outer_iterations, "converged": rep.converged,
            "final_relres": rep.final_relres,
            "cycle_iters_max": {str(l): rep.cycle_max(l) for l in range(2, hier.ml + 1)},
            "cslp_iters_max": {str(l): rep.cslp_max(l) for l in range(1, hier.ml + 1)},
            "e2e": {"value": e2e_t, "unit": "s", "h2d_bytes_per_step": int(b_host.nbytes) * ws,
                    "d2h_bytes_per_step": int(b_host.nbytes) * ws},
            "solve_bandwidth": {"alg_GB_per_solve": round(alg / 1e9, 3),
                                "achieved_GBs": round(alg / t_step / 1e9, 1) if ws == 1 else None,
                                "frac": round(alg / t_step / 1e9 / peak, 4) if ws == 1 else None,
                                "how": "sum of per-launch algorithmic bytes counted by the host driver (device-"
                                       "resident Krylov solves from their iteration counts) / device time"},
            "roofline": roofline_entry(fams, peak, peak_src, args.config),
            "kernel_families": fams,
            "kernel_families_solve_ms": prof_ms,
            "kernels": {k: kernel_entry(k, v, peak) for k, v in kern.items()},
            "gpu_launches": int(launches / max(1, args.steps)),
            "gpu_launches_total": int(launches),
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(out_line), flush=True)
    solver.close()
    if dist_ctx is not None:
        dist_ctx.close()
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def C_launches(L):
    import ctypes as C
    a, b = C.c_longlong(), C.c_longlong()
    L.hdb_stats(C.byref(a), C.byref(b))
    return a.value


if __name__ == "__main__":
    main()
