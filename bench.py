"""Benchmark: SRJ grid-point updates/s (GLUPS, fp64) on the BASELINE configs.

Default workload (BASELINE.json configs[1], ``--workload cfg2``): 2D Poisson,
4096 x 4096 interior, fp64, Dirichlet u=0, 5-point stencil, f = i.i.d.
U(-1,1) + 8 seeded Gaussians, SRJ P=6 schedule (table row N=4096, M=25,530
sweeps per cycle).  One bench "step" is one full M-cycle including the
per-step (dmax, rmax) norms and the host-side check of the cycle's norm
buffer.  Fields are 134 MB each (u, u_next, f = 403 MB > 126 MB L2), so every
sweep streams from HBM: no L2 flush is needed.

Other workloads (``--workload``): cfg3 (512^3 3D, P=10, z-slabs, strong
scaling), cfg4 (32768^2, P=15 N=2048 row, row blocks, strong scaling; a step
is 1,024 sweeps), cfg5 (nonlinear 256^3, P=8 effective-N row, strong).  cfg2
at N GPUs is weak scaling: every rank owns a 4096 x 4096 row block of a
(4096 N) x 4096 grid.

value   : GLUPS with the inputs resident in HBM (device-timed CUDA events on
          the launching stream, max over ranks).
e2e     : the same metric through the public API (``grids.srj_solve`` at N=1,
          ``distributed.srj_solve`` at N>1) on pinned host arrays: each call
          uploads u and f (or kappa), runs one step's sweeps, downloads u.
roofline: dominant kernel (2D: fused band sweep T=4; 3D: CTA-tile sweep T=2);
          algorithmic bytes = 24 B per point-update x T fused sweeps.
ttr     : time to the relative-L2 residual 1e-8 (cfg1: 1e-10) through the
          public API, wall clock incl. host copies (BASELINE "time-to-residual").
cpu_baseline: the reference's own srj_solve (baseline/_ref, serial numba,
          1 core) on a bounded sample, measured before CUDA initialises;
          cpu_port: the oracle port (reference _wj* arithmetic) on all cores.

N > 1: ``python bench.py --gpus N`` launches N ranks itself (torch
distributed.run, 127.0.0.1) unless already under torchrun; one NCCL rank per
GPU, rank-local inputs (problems.slab_config_fields), halo exchange in
libsrj over CUDA IPC (distributed.py).  ``--impl reference`` times the
reference's CPU path on rank 0 (other ranks exit 0).
"""

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0}
BYTES_PER_UPDATE = 24.0
METRIC = "grid-point updates/sec (GLUPS) fp64"

# workload -> BASELINE config, scaling series, sweeps per bench step (None =
# one M-cycle), fused depth of the dominant kernel, time-to-residual target,
# reference CPU sample (sweeps; the reference layout is per-cell arrays)
WORKLOADS = {
    "cfg1": dict(scaling="strong", step=None, fuse=4, ttr=1e-10, ref_sweeps=800,
                 desc="cfg1: 2D Poisson 256^2, P=2 SRJ (N=250 row, M=264), fp64, Dirichlet"),
    "cfg2": dict(scaling="weak", step=None, fuse=4, ttr=1e-8, ref_sweeps=40,
                 desc="cfg2: 2D Poisson 4096^2 per GPU, P=6 SRJ schedule (table row N=4096, "
                      "M=25530), fp64, 5-point, Dirichlet"),
    "cfg3": dict(scaling="strong", step=None, fuse=2, ttr=1e-8, ref_sweeps=6,
                 desc="cfg3: 3D Poisson 512^3, P=10 SRJ (N=512 row, M=1914), fp64, 7-point, "
                      "Dirichlet, z-slabs"),
    "cfg4": dict(scaling="strong", step=1024, fuse=4, ttr=None, ref_sweeps=16,
                 ref_shape=(8192, 8192),
                 desc="cfg4: 2D Poisson 32768^2, P=15 SRJ (N=2048 row, M=9548), fp64, "
                      "Dirichlet, row blocks"),
    "cfg5": dict(scaling="strong", step=None, fuse=2, ttr=1e-8, ref_sweeps=32,
                 desc="cfg5: nonlinear 3D -Lap(psi)=2 pi rho psi^5, 256^3, P=8 SRJ (effective-N "
                      "row N=150, M=474), fp64, psi=1 Dirichlet"),
}


# --secondary default: (timed cycles, warm-up cycles) per extra workload
SECONDARY = {"cfg3": (3, 1), "cfg5": (10, 3), "cfg2": (3, 1), "cfg1": (20, 3)}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return PEAKS_FALLBACK["hbm_gbs"], "fallback"


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def ncu_traffic(workload, fuse, cells):
    """DRAM bytes per launch from the committed ncu capture of the dominant
    kernel at this workload's size (profiles/), or None."""
    names = {("cfg2", 4096 * 4096): f"round2_ncu_sweep2d_T{fuse}.json",
             ("cfg3", 512 ** 3): "round2_ncu_sweep3d_rs_T2_512.json",
             ("cfg5", 256 ** 3): "round2_ncu_sweep3d_rs_T2_nl256.json"}
    name = names.get((workload, cells))
    path = os.path.join(ROOT, "profiles", name) if name else None
    if not path or not os.path.exists(path):
        return None
    with open(path) as fh:
        return json.load(fh).get("dram_traffic_bytes_per_launch")


def global_shape(workload, world, shape=None):
    from paper_1511_04292_b200.problems import CONFIGS

    if shape:
        shp = tuple(shape)
    else:
        shp = tuple(CONFIGS[workload]["shape"])
    if WORKLOADS[workload]["scaling"] == "weak":
        shp = (shp[0] * world,) + shp[1:]
    return shp


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------- CPU legs
def _reference_modules():
    """The unmodified reference (pip-installed into baseline/_ref), or None."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "srj")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "srj_numba_cache"))
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import srj.grids as rg
        import srj.schedule as rs
        import srj.tables as rt
    except Exception:
        return None
    return rg, rs, rt


def _ref_schedule(rs, rt, workload):
    """The reference's own CycleSchedule for a workload (same table row as ours)."""
    from paper_1511_04292_b200.problems import CONFIGS
    from paper_1511_04292_b200.schedule import effective_n

    cfg = CONFIGS[workload]
    n = cfg["n_table"]
    if n == "effective":
        n = effective_n([s + 1 for s in cfg["shape"]], len(cfg["shape"]), "dirichlet")
    return rs.quantize(rt.shipped_table().lookup(cfg["p"], int(n)))


def _ref_problem(rg, f):
    """A reference GridProblem with per-cell coefficient arrays (how the
    reference's own problem builders store them, problems.py:299-322)."""
    shape = f["source"].shape
    full = lambda a: np.ascontiguousarray(np.broadcast_to(a, shape))  # noqa: E731
    nd = len(shape)
    fixed = rg.BoundaryRule("fixed")
    return rg.GridProblem(spacing=(1.0,) * nd, u=np.array(f["u"]), source=np.array(f["source"]),
                          center=full(f["center"]), lower=tuple(full(a) for a in f["lower"]),
                          upper=tuple(full(a) for a in f["upper"]), bc=((fixed, fixed),) * nd)


def reference_cpu_steps(workload, sweeps, steps, warmup):
    """Times the reference's srj_solve (serial numba) for ``steps`` calls of
    ``sweeps`` sweeps each after ``warmup`` calls (JIT excluded).  Each call
    restarts from u0 (the sample's field is reset outside the timed call) so
    the first weights of the cycle never compound to overflow.  Returns
    (per-call seconds, cells, note) or None without baseline/_ref."""
    mods = _reference_modules()
    if mods is None:
        return None
    rg, rs, rt = mods
    from paper_1511_04292_b200.problems import config_fields

    if workload == "cfg5":
        # the reference has no nonlinear solver: time its linear kernel on the
        # same grid (the psi^5 source is this repo's extension)
        f = config_fields("cfg3", (256, 256, 256))
        note = "linear _wj3 on the cfg5 256^3 grid (the reference has no nonlinear source)"
    else:
        f = config_fields(workload, WORKLOADS[workload].get("ref_shape"))
        note = ""
    cyc = _ref_schedule(rs, rt, workload)
    p = _ref_problem(rg, f)
    u0 = p.u.copy()
    cells = int(np.prod(p.source.shape))
    times = []
    for it in range(warmup + steps):
        p.u[...] = u0
        t0 = time.perf_counter()
        rg.srj_solve(p, cyc, tol=1e-300, max_iters=sweeps)
        dt = time.perf_counter() - t0
        if it >= warmup:
            times.append(dt)
    return times, cells, note


def port_cpu(workload, budget_s=10.0, max_sweeps=4096, threads=None):
    """Oracle port (reference _wj* arithmetic, OpenMP rows) on all host cores."""
    import oracle

    from paper_1511_04292_b200.grids import FIXED, GridProblem
    from paper_1511_04292_b200.problems import config_fields, config_schedule

    threads = threads or os.cpu_count() or 1
    shape = WORKLOADS[workload].get("ref_shape")
    f = config_fields(workload, shape)
    w = config_schedule(workload).weight_sequence
    nd = f["source"].ndim
    full = lambda a: np.ascontiguousarray(np.broadcast_to(a, f["source"].shape))  # noqa: E731
    p = GridProblem(spacing=(1.0,) * nd, u=f["u"].copy(), source=f["source"],
                    center=full(f["center"]), lower=tuple(full(a) for a in f["lower"]),
                    upper=tuple(full(a) for a in f["upper"]), bc=((FIXED, FIXED),) * nd)
    kappa = f.get("kappa")
    cells = int(np.prod(p.shape))
    # one call per measurement: the port marshals its arguments per call, so
    # short calls under-report it (round 1: 0.62 vs 0.98 GLUPS for 4 vs 8
    # sweeps per call); calibrate with 4 sweeps, then time one long call
    t0 = time.perf_counter()
    oracle.run(p, w, 0, 4, kappa=kappa, nthreads=threads)
    t4 = time.perf_counter() - t0
    done = int(min(max_sweeps, max(8, 4 * budget_s / max(t4, 1e-3))))
    t0 = time.perf_counter()
    oracle.run(p, w, 4, done, kappa=kappa, nthreads=threads)
    dt = time.perf_counter() - t0
    return {"value": cells * done / dt / 1e9, "unit": "GLUPS", "cores": threads, "kind": "port",
            "sample": f"{done} sweeps of the {workload} schedule on a {'x'.join(map(str, p.shape))} "
                      f"grid (oracle/srj_oracle.c, the reference's _wj arithmetic on per-cell "
                      f"coefficient arrays, OpenMP rows), {dt:.1f} s, measured before CUDA "
                      f"initialised", "cpu_model": cpu_model()}


def cpu_baselines(workload):
    """(cpu_baseline, cpu_port): the reference itself on 1 core, then the port."""
    ref = None
    sweeps = WORKLOADS[workload]["ref_sweeps"]
    res = reference_cpu_steps(workload, sweeps, 1, 1)
    if res is not None:
        times, cells, note = res
        dt = sum(times)
        ref = {"value": cells * sweeps / dt / 1e9, "unit": "GLUPS", "cores": 1,
               "kind": "reference",
               "sample": f"{sweeps} sweeps of the reference's own srj.grids.srj_solve "
                         f"(baseline/_ref, serial numba _wj kernel, grids.py:328, :642-687) on "
                         f"{cells} cells, {dt:.1f} s after a JIT warm-up call; 1 of "
                         f"{os.cpu_count()} host cores" + (f"; {note}" if note else ""),
               "cpu_model": cpu_model()}
    port = port_cpu(workload)
    return (ref or port), (port if ref else None)


def run_reference(args):
    """--impl reference: the reference's CPU path (baseline/_ref numba
    srj_solve, serial -> 1 core) on rank 0; each step = a bounded sample of
    ref_sweeps sweeps of the workload's schedule.  Falls back to the oracle
    port (all cores) when baseline/_ref is absent."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    wl = WORKLOADS[args.workload]
    sweeps = max(1, wl["ref_sweeps"] // 4)  # ~1-2 s of serial CPU work per step
    res = reference_cpu_steps(args.workload, sweeps, args.steps, args.warmup)
    if res is not None:
        times, cells, note = res
        dt = sum(times)
        v = cells * sweeps * args.steps / dt / 1e9
        cpu = {"value": v, "unit": "GLUPS", "cores": 1, "kind": "reference",
               "sample": f"{sweeps} sweeps x {args.steps} steps of the reference's own "
                         f"srj.grids.srj_solve (baseline/_ref, serial numba) on {cells} cells; "
                         f"1 of {os.cpu_count()} host cores" + (f"; {note}" if note else ""),
               "cpu_model": cpu_model()}
        ms = dt / args.steps * 1e3
    else:
        port = port_cpu(args.workload, budget_s=3.0 * args.steps)
        v = port["value"]
        cpu = port
        ms = None
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "GLUPS",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": wl["scaling"], "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["desc"], "step": f"{sweeps} sweeps (bounded CPU sample)"},
        "cpu_baseline": cpu,
        "e2e": {"value": v, "unit": "GLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------- launcher
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args):
    """``--gpus N`` outside torchrun: run N ranks of this script through
    torch.distributed.run on 127.0.0.1 and return their exit code."""
    if not args.dry_run:
        try:
            import torch

            have = torch.cuda.device_count()
        except Exception:
            have = 0
        if have < args.gpus:
            print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} needs {args.gpus} "
                              f"visible GPUs, found {have}", "n_gpus": args.gpus}), flush=True)
            return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


# ---------------------------------------------------------------- GPU arm
def build_grid(args, ws, rank, comm):
    """(grid, cells on this rank, global shape, host problem for N=1)."""
    from paper_1511_04292_b200.problems import config_fields

    shape = global_shape(args.workload, ws, args.shape)
    if ws == 1 and not args.slab:
        from paper_1511_04292_b200.engine import DeviceGrid

        f = config_fields(args.workload, shape)
        grid = DeviceGrid(f["u"], f["source"], f["center"], f["lower"], f["upper"],
                          kappa=f.get("kappa"))
        return grid, int(np.prod(shape)), shape, f
    from paper_1511_04292_b200.distributed import SlabDecomposition, SlabGrid, default_halo
    from paper_1511_04292_b200.problems import slab_config_fields

    d = SlabDecomposition(shape[0], ws, rank, default_halo(len(shape), args.fuse))
    slab = slab_config_fields(args.workload, d, shape)
    grid = SlabGrid(slab, comm)
    return grid, grid.owned_cells, shape, slab


def launches_per_fused_step(slab):
    """Kernel launches per fused step of a rank: its edge parts + inner part."""
    edges, inner = slab.decomp.row_parts()
    return len(edges) + (inner is not None)


def measure_e2e(args, ws, rank, comm, shape, sweeps, host):
    """The public API on pinned host arrays, one step's sweeps per call."""
    import torch

    from paper_1511_04292_b200 import grids as G
    from paper_1511_04292_b200.problems import config_schedule

    cyc = config_schedule(args.workload)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
    times = []
    if isinstance(host, dict):  # one whole grid (N = 1 without --slab)
        f = host
        u = pin(f["u"])
        src = pin(f["kappa"] if "kappa" in f else f["source"])
        nd = u.ndim
        u0 = u.copy()
        h2d = u.nbytes + src.nbytes
        d2h = u.nbytes + 16 * sweeps
        for it in range(args.e2e_steps + 1):  # first call warms up
            u[...] = u0
            if "kappa" in f:
                p = G.GridProblem(spacing=(1.0,) * nd, u=u, source=np.zeros(src.shape),
                                  center=f["center"], lower=f["lower"], upper=f["upper"],
                                  bc=((G.FIXED, G.FIXED),) * nd, source_kappa=src)
            else:
                p = G.GridProblem(spacing=(1.0,) * nd, u=u, source=src, center=f["center"],
                                  lower=f["lower"], upper=f["upper"], bc=((G.FIXED, G.FIXED),) * nd)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            G.srj_solve(p, cyc, tol=1e-300, max_iters=sweeps)
            if it:
                times.append(time.perf_counter() - t0)
        api = "paper_1511_04292_b200.srj_solve(problem, cycle, tol, max_iters)"
        cells = int(np.prod(shape))
    else:
        from paper_1511_04292_b200 import distributed as D

        slab = host
        u = pin(slab.u)
        src = pin(slab.kappa if slab.kappa is not None else slab.source)
        u0 = u.copy()
        h2d = u.nbytes + src.nbytes
        lo, hi = slab.decomp.own_local
        d2h = int(np.prod(u.shape[1:])) * 8 * (hi - lo) + 16 * sweeps
        for it in range(args.e2e_steps + 1):
            u[...] = u0
            sp = D.SlabProblem(slab.decomp, slab.global_shape, u, slab.center, slab.lower,
                               slab.upper, source=None if slab.kappa is not None else src,
                               kappa=src if slab.kappa is not None else None)
            if comm is not None:
                comm.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            D.srj_solve(sp, cyc, tol=1e-300, max_iters=sweeps)
            if it:
                times.append(time.perf_counter() - t0)
        api = "paper_1511_04292_b200.distributed.srj_solve(SlabProblem, cycle, tol, max_iters)"
        cells = int(np.prod(shape))
    dt = sum(times)
    if ws > 1:
        dt = float(comm.max_(np.array([dt]))[0])
    return {"value": cells * sweeps * args.e2e_steps / dt / 1e9, "unit": "GLUPS",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "calls": args.e2e_steps, "api": api,
            "note": "per rank; value from the max over ranks" if ws > 1 else None}


def measure_ttr(args, ws, rank, comm, shape, host):
    """Time to the relative-L2 target through the public API (wall clock)."""
    tol = WORKLOADS[args.workload]["ttr"]
    if tol is None:
        return None
    import torch

    from paper_1511_04292_b200 import grids as G
    from paper_1511_04292_b200.problems import config_schedule

    cyc = config_schedule(args.workload)
    if ws == 1:
        f = host
        nd = f["u"].ndim
        kw = {}
        if "kappa" in f:
            kw["source_kappa"] = f["kappa"]
        p = G.GridProblem(spacing=(1.0,) * nd, u=f["u"].copy(), source=f["source"],
                          center=f["center"], lower=f["lower"], upper=f["upper"],
                          bc=((G.FIXED, G.FIXED),) * nd, **kw)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hist, _ = G.srj_solve(p, cyc, tol, stop="residual_l2", max_iters=2000 * cyc.m)
        dt = time.perf_counter() - t0
    else:
        from paper_1511_04292_b200 import distributed as D

        slab = host
        sp = D.SlabProblem(slab.decomp, slab.global_shape, slab.u.copy(), slab.center, slab.lower,
                           slab.upper, source=slab.source, kappa=slab.kappa)
        comm.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hist, _ = D.srj_solve(sp, cyc, tol, stop="residual_l2", max_iters=2000 * cyc.m)
        dt = float(comm.max_(np.array([time.perf_counter() - t0]))[0])
    return {"tol": tol, "rule": "relative L2 of the true residual ||s - A u||_2 / ||s||_2 "
                                "(cfg5: / initial residual), checked every M-cycle",
            "seconds": dt, "iterations": hist.iterations, "cycles": hist.iterations / cyc.m,
            "converged": bool(hist.converged),
            "final_relative_l2": float(hist.relative_l2[-1, 1]) if len(hist.relative_l2) else None,
            "api": "srj_solve(..., stop='residual_l2')", "n_gpus": ws}


def measure_secondary(workload, steps, warmup):
    """Device-resident GLUPS of another BASELINE config on this GPU (N=1), so
    the default bench line also records the 3D kernels: ``steps`` full
    M-cycles after ``warmup``, CUDA events on the grid's stream, clocks
    sampled during the timed region."""
    import torch

    from paper_1511_04292_b200.engine import DeviceGrid
    from paper_1511_04292_b200.problems import CONFIGS, config_fields, config_schedule

    wl = WORKLOADS[workload]
    shape = tuple(CONFIGS[workload]["shape"])
    f = config_fields(workload, shape)
    cyc = config_schedule(workload)
    w, m = cyc.weight_sequence, cyc.m
    grid = DeviceGrid(f["u"], f["source"], f["center"], f["lower"], f["upper"],
                      kappa=f.get("kappa"))
    T = wl["fuse"]
    try:
        cur, k = 0, 0
        for _ in range(warmup):
            cur = grid.run(cur, w, k, m, T)
            k += m
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        with ClockSampler(torch.cuda.current_device()) as clk:
            ev0.record(grid.stream)
            for _ in range(steps):
                cur = grid.run(cur, w, k, m, T)
                norms = grid.norms[:2 * m].view(m, 2).cpu().numpy()  # per-cycle host check
                if not np.all(np.isfinite(norms)):
                    raise RuntimeError(f"non-finite norms in the {workload} measurement")
                k += m
            ev1.record(grid.stream)
            torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1)
    finally:
        grid.close()
    cells = int(np.prod(shape))
    value = cells * m * steps / (ms * 1e-3) / 1e9
    peak, _ = peaks()
    return {"workload": wl["desc"], "value": value, "unit": "GLUPS", "steps": steps,
            "warmup": warmup, "ms_per_step": ms / steps, "step": f"one full M-cycle ({m} sweeps)",
            "fuse": T, "kernel": "sweep3d_rs<T=2> (register-streaming, persistent CTAs)",
            "frac_of_hbm_roofline_single_sweep": value * BYTES_PER_UPDATE / peak,
            "clocks": clk.summary()}


def run_dry(args):
    """--dry-run: the launcher, rendezvous, rank-local inputs and collectives
    without kernels (gloo, CPU) -- exercised by tests/test_bench_launcher.py."""
    import torch.distributed as dist

    ws, rank, _ = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    from paper_1511_04292_b200.distributed import (DistComm, SlabDecomposition, default_halo)
    from paper_1511_04292_b200.problems import slab_config_fields
    from paper_1511_04292_b200.solver import LocalComm

    comm = DistComm() if ws > 1 else LocalComm
    shape = global_shape(args.workload, ws, args.shape)
    d = SlabDecomposition(shape[0], ws, rank, default_halo(len(shape), args.fuse))
    slab = slab_config_fields(args.workload, d, shape)
    from paper_1511_04292_b200.grids import layer_sum_squares

    sq = np.zeros(shape[0])
    lo, hi = d.owned
    ol, oh = d.own_local
    sq[lo:hi] = layer_sum_squares(np.asarray(slab.kappa if slab.kappa is not None
                                             else slab.source)[ol:oh])
    total = comm.sum_(sq)
    owned = comm.sum_(np.array([float(hi - lo)]))
    if ws > 1:
        comm.barrier()
    if rank == 0:
        print(json.dumps({"metric": METRIC, "dry_run": True, "n_gpus": ws,
                          "workload": args.workload, "global_shape": list(shape),
                          "owned_rows_total": float(owned[0]),
                          "source_l2_sq": float(np.sum(total))}), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def run_gpu(args):
    import torch

    ws, rank, local = dist_env()
    if ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}")
    wl = WORKLOADS[args.workload]
    cpu, cpu_port = None, None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu, cpu_port = cpu_baselines(args.workload)  # before CUDA initialises
    if ws > 1:
        # every stream of a rank on its own hardware queue: the slab exchange's
        # flag waits must never sit ahead of another stream's work in a shared
        # queue (read when the CUDA context is created)
        os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
    torch.cuda.set_device(local)
    comm = None
    if ws > 1:
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_1511_04292_b200.distributed import DistComm

        comm = DistComm()
    from paper_1511_04292_b200.problems import config_schedule

    cyc = config_schedule(args.workload)
    w = cyc.weight_sequence
    m = cyc.m
    sweeps = wl["step"] or m
    grid, cells_rank, shape, host = build_grid(args, ws, rank, comm)
    stream = grid.stream
    T = args.fuse or wl["fuse"]
    nd = len(shape)
    if nd == 3:
        T = min(T, 2 if not args.fuse else args.fuse)
    fused_per_step = -(-sweeps // T)
    parts = 1
    if ws > 1 and not grid.backend.direct(args.fuse):
        parts = launches_per_fused_step(host)  # staged path: edge parts + inner part

    def one_step(cur, first):
        out = grid.run(cur, w, first, sweeps, args.fuse)
        norms = grid.norms[:2 * sweeps].view(sweeps, 2).cpu().numpy()  # per-step host check
        metric = norms[:, 0] / np.abs(w[(first + np.arange(sweeps)) % m])
        if not np.all(np.isfinite(metric)):
            raise RuntimeError("non-finite update norm in benchmark step")
        return out

    cur, k = 0, 0
    for _ in range(args.warmup):
        cur = one_step(cur, k)
        k += sweeps
    torch.cuda.synchronize()
    if ws > 1:
        comm.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    step_ev = []
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            cur = one_step(cur, k)
            b.record(stream)
            k += sweeps
            step_ev.append((a, b))
        ev1.record(stream)
        torch.cuda.synchronize()
    if ws > 1:
        comm.barrier()
    elapsed = ev0.elapsed_time(ev1)
    kernel_ms = sum(a.elapsed_time(b) for a, b in step_ev)
    if ws > 1:
        elapsed, kernel_ms = (float(x) for x in comm.max_(np.array([elapsed, kernel_ms])))
    total_cells = int(np.prod(shape))
    value = total_cells * sweeps * args.steps / (elapsed * 1e-3) / 1e9
    avg_launch_ms = kernel_ms / (args.steps * fused_per_step)
    peak, peak_kind = peaks()
    achieved = cells_rank * T * BYTES_PER_UPDATE / (avg_launch_ms * 1e-3) / 1e9
    traffic = ncu_traffic(args.workload, T, cells_rank) if ws == 1 else None
    launches = args.steps * fused_per_step * parts
    if ws > 1:
        launches = int(comm.sum_(np.array([float(launches)]))[0])
    gridname = ("sweep2d_tb<T=%d> (fused %d sweeps/launch)" % (T, T) if nd == 2 else
                "sweep3d_rs<T=%d> (fused %d sweeps/launch, register streaming)" % (T, T))

    e2e = None if args.e2e_steps <= 0 else measure_e2e(args, ws, rank, comm, shape,
                                                        sweeps, host)
    ttr = None if args.no_ttr else measure_ttr(args, ws, rank, comm, shape, host)
    if ws > 1:
        comm.barrier()
    if rank != 0:
        return 0
    if ws > 1:
        how = ("edge rows stored into the neighbours' halos by the sweep kernel (CUDA IPC peer "
               "memory over NVLink)" if parts == 1 else
               "edge launches + peer copies over CUDA IPC / NVLink overlapped with the inner rows")
    par = "single GPU" if ws == 1 else (
        f"{'row blocks' if nd == 2 else 'z-slabs'} x{ws} (axis 0), halo {T}, {how}, device-side "
        f"flag ordering, NCCL all-reduce per chunk")
    line = {
        "metric": METRIC, "value": value, "unit": "GLUPS", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed / args.steps, "higher_is_better": True,
        "scaling": wl["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": wl["desc"], "global_shape": list(shape),
                   "step": (f"one full M-cycle ({m} sweeps)" if wl["step"] is None else
                            f"{sweeps} sweeps of the M={m} cycle") +
                           " + per-step norms + host check",
                   "fuse": T,
                   "l2": "inputs larger than L2 (3 fields streamed per sweep)"
                         if cells_rank * 24 > 126e6 else "inputs fit in L2",
                   "parallelism": par},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_note": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch "
                                     "of the same kernel and size (profiles/); actual HBM bytes vs "
                                     "algorithmic shows the temporal-blocking saving",
                     "peak_kind": peak_kind, "kernel": gridname,
                     "algorithmic_bytes_per_launch": cells_rank * T * BYTES_PER_UPDATE,
                     "avg_launch_ms": avg_launch_ms},
        "clocks": clk.summary(),
        "gpu_launches": launches,
        "glups_per_gpu": value / ws,
        "frac_of_hbm_roofline_single_sweep": value / ws * BYTES_PER_UPDATE / peak,
    }
    if e2e:
        line["e2e"] = e2e
    if ttr:
        line["time_to_residual"] = ttr
    if cpu:
        line["cpu_baseline"] = cpu
    if cpu_port:
        line["cpu_port"] = cpu_port
    if ws == 1 and args.secondary:
        # the 3D BASELINE configs on the same box, device-resident (the
        # headline metric above is the --workload's)
        line["other_workloads"] = [measure_secondary(x, *SECONDARY[x]) for x in
                                   args.secondary.split(",") if x != args.workload]
    if ws == 1 and args.rank_proxy:
        line["multi_gpu_rank_proxy"] = measure_rank_proxy()
    print(json.dumps(line), flush=True)
    return 0


def measure_rank_proxy():
    """One rank of the multi-GPU slab path, timed on this one GPU
    (tools/slab_rank_probe.py): the middle rank of a 3-rank decomposition runs
    the real srj_slab_run -- the sweep kernel storing its edge rows into the
    neighbours' halo rows, the flag-word stream operations -- against two
    virtual neighbours on the same device, compared with the same rows as one
    whole grid.  Excludes the NVLink latency and waiting for a slower rank."""
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import slab_rank_probe as srp

    cases = [("cfg2 weak scaling: 4096 x 4096 rows per GPU", "cfg2", (4096, 4096), 4, 2000),
             ("cfg4 at 8 GPUs: 4096 x 32768 rows per GPU", "cfg4", (4096, 32768), 4, 200),
             ("cfg3 at 8 GPUs: 64 planes of 512^2 per GPU", "cfg3", (64, 512, 512), 2, 800),
             ("cfg5 at 8 GPUs: 32 planes of 256^2 per GPU", "cfg5", (32, 256, 256), 2, 1600)]
    out = []
    for label, wl, own, fuse, steps in cases:
        r = srp.probe(wl, own, fuse, steps, reps=2, modes=("direct_store",))
        out.append({"case": label, "rank_glups": r["direct_store_glups"],
                    "whole_grid_glups": r["whole_grid_glups"],
                    "rank_efficiency": r["direct_store_efficiency"], "fuse": fuse})
    return {"what": "per-rank device timeline of srj_slab_run on ONE GPU against virtual "
                    "neighbours (no NVLink latency, no waiting for other ranks); efficiency = "
                    "time of the same rows as one whole grid / time of the rank",
            "cases": out}


def main():
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--shape", type=int, nargs="+", default=None,
                    help="override the workload's (per-GPU for weak scaling) grid shape")
    ap.add_argument("--fuse", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ttr", action="store_true")
    ap.add_argument("--secondary", default="cfg3,cfg5",
                    help="N=1: also time these workloads device-resident (empty: none)")
    ap.add_argument("--no-rank-proxy", dest="rank_proxy", action="store_false",
                    help="N=1: skip the one-GPU timing of a multi-GPU slab rank")
    ap.add_argument("--slab", action="store_true",
                    help="use the multi-GPU slab path even on one GPU (testing)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher + rank-local inputs + collectives only (gloo, no GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
    if args.impl == "reference":
        return run_reference(args)
    if args.dry_run:
        return run_dry(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
