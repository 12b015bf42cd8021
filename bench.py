#!/usr/bin/env python
"""Benchmark of the B200 hot path (BASELINE.json metric:
"MDoF/s residual+Jv fill; sec per implicit Newton step at 1/2/4/8 B200").

Default workload = BASELINE.json configs[1]: 2D pure-metal dendrite (free
growth), Q1 2048x2048 elements on 61.44^2 (h = 0.03), fp64 JFNK.

One timed STEP = one residual fill F(u) plus one fused finite-difference
Jacobian-vector product J(u)v on the same state (2 x D DoF filled, D = 2 x
2049^2 = 8,396,802).  ``value`` = whole-job MDoF/s = (sum over ranks of 2 D K)
/ max-over-ranks time of K steps, inputs resident in HBM (working set ~470 MB,
larger than the 126 MB L2, so no L2 flush is needed between steps).

Also reported:
  e2e        the same step through the public API (TimestepResidual.__call__ +
             jfnk_matvec) with u, v copied from pinned host memory and F, Jv
             copied back inside the timed region;
  newton     seconds per implicit Newton iteration for the first (backward-
             Euler startup) step of the seeded dendrite at the same size, with
             its GMRES count, preconditioner build and V-cycle apply time;
  roofline   the residual tile kernel: algorithmic 32 B/DoF (reads u, phi_old,
             phi_prev, fixed part; writes F) over its CUDA-event duration;
  cpu_baseline  the oracle port (oracle/uc_oracle.c, OpenMP) on the host cores.

``--impl reference`` times the reference algorithm on the host (the oracle
port; the reference itself is Python and cannot travel to the GPU box).
Multi-GPU (torchrun): every rank runs the same per-rank workload (weak scaling,
independent replicas: the slab-decomposed halo path is not yet wired into
this benchmark).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# testing only: N > 1 ranks sharing GPUs through the host-staged transport
HOST_TRANSPORT = os.environ.get("UC_BENCH_HOST_TRANSPORT") == "1"

WORKLOADS = {
    # name: model, dim, extents, counts, theta, dt, step (synthetic states), Newton dt
    "fg2d_2048": dict(model="free_growth", dim=2, extents=(61.44, 61.44), counts=(2048, 2048),
                      theta=0.5, dt=2.25e-4, step=2),
    "fg2d_512": dict(model="free_growth", dim=2, extents=(15.36, 15.36), counts=(512, 512),
                     theta=0.5, dt=2.25e-4, step=2),
    "al2d_4096": dict(model="alloy", dim=2, extents=(3276.8, 3276.8), counts=(4096, 4096),
                      theta=0.5, dt=0.002, step=2),
    "fg3d_256": dict(model="free_growth", dim=3, extents=(7.68,) * 3, counts=(256,) * 3,
                     theta=0.5, dt=2.25e-4, step=2),
    "fg3d_512": dict(model="free_growth", dim=3, extents=(15.36,) * 3, counts=(512,) * 3,
                     theta=0.5, dt=2.25e-4, step=2),
    # not a BASELINE config: alloy 3D for kernel tuning
    "al3d_128": dict(model="alloy", dim=3, extents=(102.4,) * 3, counts=(128,) * 3,
                     theta=0.5, dt=0.002, step=2),
}


def synthetic_states(w, seed=11):
    N = int(np.prod([c + 1 for c in w["counts"]]))
    rng = np.random.default_rng(seed)
    if w["model"] == "free_growth":  # tests/test_free_growth.py:246-256 distribution
        mk = lambda: np.concatenate([0.5 + 0.3 * rng.standard_normal(N), 1.0 + 0.2 * rng.standard_normal(N)])  # noqa: E731
    else:  # tests/test_alloy.py:286-295
        mk = lambda: np.concatenate([np.tanh(rng.standard_normal(N)), -0.5 + 0.4 * rng.standard_normal(N)])  # noqa: E731
    u, old, prev = mk(), mk(), mk()
    v = np.random.default_rng(2).standard_normal(2 * N)
    return N, u, old, prev, v


class Clocks:
    """SM clock and throttle-reason sampler for the timed region (NVML every
    ~10 ms; the B200_PROFILING.md clocks line via nvidia-smi as a fallback)."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        self.source = "nvml"

    def _run(self):
        try:
            import pynvml as N

            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
            mx = N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)
            bits = {"hw_slowdown": N.nvmlClocksThrottleReasonHwSlowdown,
                    "hw_thermal_slowdown": N.nvmlClocksThrottleReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": N.nvmlClocksThrottleReasonSwThermalSlowdown,
                    "sw_power_cap": N.nvmlClocksThrottleReasonSwPowerCap}
            while not self._stop.is_set():
                sm = N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)
                r = N.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                self.rows.append((float(sm), float(mx), [k for k, b in bits.items() if r & b]))
                self._stop.wait(0.01)
            N.nvmlShutdown()
        except Exception:
            self.source = "nvidia-smi"
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True,
                                         text=True, timeout=5).stdout.strip().split(",")
                    if len(out) >= 6:
                        self.rows.append((float(out[0]), float(out[1]),
                                          [names[i] for i in range(4) if out[2 + i].strip().lower() == "active"]))
                except Exception:
                    pass
                self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        time.sleep(0.05)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({x for r in self.rows for x in r[2]})
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": reasons, "samples": len(self.rows), "source": self.source}


def cpu_oracle_step_time(w, steps=2, warmup=1, rows=None, min_seconds=0.0):
    """Residual + Jv of the oracle port on the host; returns (sec/step, D, sample).
    With min_seconds, keeps timing steps until that much CPU time has been
    measured (at least `steps`)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    from paper_2006_16764_b200 import AlloyParams, FreeGrowthParams

    counts = list(w["counts"])
    extents = list(w["extents"])
    sample = "full workload"
    if rows is not None and rows < counts[-1]:
        # bounded sample: a slab of `rows` element layers of the same mesh
        extents[-1] = extents[-1] * rows / counts[-1]
        counts[-1] = rows
        sample = f"slab of {rows} of {w['counts'][-1]} element layers (same h), scaled per DoF"
    wl = dict(w, counts=tuple(counts), extents=tuple(extents))
    N, u, old, prev, v = synthetic_states(wl)
    params = FreeGrowthParams() if w["model"] == "free_growth" else AlloyParams()
    p = O.Problem(w["dim"], wl["extents"], wl["counts"], w["model"], params, w["theta"], w["dt"], w["step"])
    p.begin(old, prev)
    times = []
    i = 0
    while i < warmup + steps or sum(times) < min_seconds:
        t0 = time.perf_counter()
        f = p.residual(u)
        p.jv(u, f, v)
        if i >= warmup:
            times.append(time.perf_counter() - t0)
        i += 1
    if min_seconds > 0.0:
        sample += f", {len(times)} timed steps ({sum(times):.1f} s)"
    return float(np.mean(times)), 2 * N, sample, O.num_threads()


def run_reference(args, w, rank, world):
    """--impl reference: the reference algorithm on the host (oracle port)."""
    if rank != 0:
        return
    # bounded sample: ~1-2 s per step on a many-core host
    rows = None if w["dim"] == 2 and np.prod(w["counts"]) <= 2048 * 2048 else 256
    sec, D, sample, cores = cpu_oracle_step_time(w, steps=args.steps, warmup=args.warmup, rows=rows)
    mdofs = 2 * D / sec / 1e6
    ref_py = reference_python_1core(args.workload) if not args.no_cpu_baseline else None
    line = {
        "impl": "reference", "metric": "MDoF/s residual+Jv fill", "value": round(mdofs, 4),
        "unit": "MDoF/s", "n_gpus": args.gpus, "device": "host cores only", "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, **{k: w[k] for k in ("model", "dim", "counts")}},
        "cpu_baseline": {"value": round(mdofs, 4), "unit": "MDoF/s", "cores": cores, "kind": "port",
                         "sample": sample + f"; {cores}-thread OpenMP C port of the reference (oracle/uc_oracle.c)"},
        "e2e": {"value": round(mdofs, 4), "unit": "MDoF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "reference_python_1core": ref_py,
    }
    print(json.dumps(line), flush=True)


def reference_python_1core(workload):
    """The reference package itself (undercool, baseline/_ref) on one pinned
    core, beside the C port; None if not installed."""
    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "undercool")):
        return None
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1", MKL_NUM_THREADS="1",
               NUMBA_NUM_THREADS="1")
    cmd = [sys.executable, os.path.join(ROOT, "tools", "ref_python_time.py"), workload, "10"]
    try:
        cmd = ["taskset", "-c", str(sorted(os.sched_getaffinity(0))[0])] + cmd
    except (AttributeError, OSError):
        pass
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env)
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        return json.loads(lines[-1]) if lines else {"value": None, "error": r.stderr[-300:]}
    except Exception as exc:  # reported, never fatal
        return {"value": None, "error": repr(exc)}


def vcycle_bytes(pc, N, dim):
    """Algorithmic HBM bytes of one BlockPrecond.apply (both blocks), counting
    stencil + vector streams once per pass (x neighbours cached)."""
    K = 3 ** dim
    C = 2 ** dim  # colours
    cfg = pc.cfg
    rows = [int(np.prod(s)) for s in pc.level_shapes]

    def smooth(R, sweeps, srow):
        # colour passes actually executed: 2 C per symmetric sweep, minus the
        # repeated colour folded at every turn; each
        # pass streams its colour's stencil rows, b and x once
        passes = 2 * C * sweeps - (2 * sweeps - 1) if sweeps > 0 else 0
        return passes / C * (srow + 24) * R

    total = 0.0

    # uniform stencil rows are not read (one shared row per level)
    stencil = [8 * K * (1.0 - 0.5 * (pc.uniform_fraction(l, 0) + pc.uniform_fraction(l, 1)))
               for l in range(len(rows))]

    def cyc(l):
        nonlocal total
        R = rows[l]
        total += 8 * R  # zero x
        if l == len(rows) - 1:
            total += smooth(R, cfg.coarse_sweeps, stencil[l])
            return
        total += 2 * smooth(R, cfg.sweeps, stencil[l])  # pre + post
        total += (stencil[l] + 24) * R  # residual
        total += 8 * R + 8 * rows[l + 1]  # restrict
        cyc(l + 1)
        total += 8 * rows[l + 1] + 16 * R  # prolong-add

    for c in range(cfg.cycles):
        cyc(0)  # later cycles start from x (no defect residual, no x += e)
    return 2 * total  # both field blocks


def run_slabs(args, w, rank, world, local, dist, emulate=0):
    """N > 1: one slab per GPU (paper_2006_16764_b200.parallel), NCCL ghost
    planes and allreduces inside the library.  --scaling weak (default): the
    mesh grows with N (counts[-1] x N, same h: fixed work per GPU); strong: the
    named mesh is split N ways.  emulate=K (testing, --emulate-slabs): the same
    code path with K slabs driven by this one process on one GPU (planes copied
    on the stream instead of NCCL)."""
    import torch

    import paper_2006_16764_b200 as uc
    from paper_2006_16764_b200.models import seed_initial_condition_device
    from paper_2006_16764_b200.parallel import SlabGroup, SlabPrecond, SlabResidual

    dev = torch.device("cuda", local)
    nslab = emulate if emulate else world
    counts = list(w["counts"])
    extents = list(w["extents"])
    if args.scaling == "weak":
        counts[-1] *= nslab
        extents[-1] *= nslab
    mesh = uc.build_mesh(w["dim"], extents, counts)
    kern = uc.FreeGrowthKernel() if w["model"] == "free_growth" else uc.AlloyKernel()
    sc = uc.ThetaScheme(w["theta"], w["dt"], w["step"])
    grp = (SlabGroup.local(mesh, kern, nslab) if emulate
           else SlabGroup.from_torch_dist(mesh, kern, transport="host" if HOST_TRANSPORT else "nccl"))
    nlocs = [(hi - lo) * grp.plane for lo, hi in grp.slabs]
    rng = np.random.default_rng(11 + rank)

    def mk(nloc):
        if w["model"] == "free_growth":
            return np.concatenate([0.5 + 0.3 * rng.standard_normal(nloc), 1.0 + 0.2 * rng.standard_normal(nloc)])
        return np.concatenate([np.tanh(rng.standard_normal(nloc)), -0.5 + 0.4 * rng.standard_normal(nloc)])

    sp = grp.space
    u, old, prev = (sp.wrap([torch.from_numpy(mk(n)).to(dev) for n in nlocs]) for _ in range(3))
    v = sp.wrap([torch.from_numpy(np.random.default_rng(2 + rank).standard_normal(2 * n)).to(dev) for n in nlocs])
    res = SlabResidual(grp, old, prev, sc)
    unorm = sp.norm(u)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def max_ms(ms):
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        if dist is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def step():
        f = res.device_call(u, check=False)
        return res.jv_device(u, f, v, unorm)

    def timed(fn, reps):
        for _ in range(3):
            fn()
        barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        barrier()
        return max_ms(a.elapsed_time(b) / reps)

    clk = Clocks(local).__enter__()
    for _ in range(args.warmup):
        step()
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(args.steps):
        step()
    b.record(stream)
    barrier()
    ms = max_ms(a.elapsed_time(b) / args.steps)
    D_glob = 2 * int(np.prod([c + 1 for c in counts]))
    value = 2 * D_glob / (ms * 1e-3) / 1e6
    # residual tile roofline on this rank's slab (32 B/DoF over the CUDA-event
    # time, max over ranks), HBM peak from MEASURED_PEAKS.json
    t_res = timed(lambda: res.device_call(u, check=False), max(args.steps, 20))
    clk.__exit__()
    hbm_peak, peak_src = hbm_peak_gbs()
    D_loc = 2 * sum(nlocs)
    ach = 32 * D_loc / (t_res * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(ach / hbm_peak, 4), "traffic": None, "algorithmic_bytes": 32 * D_loc,
                "kernel": roofline_kernel_name(w), "bytes_per_dof": 32, "ms_per_launch": round(t_res, 4),
                "peak_source": peak_src,
                "note": "per rank (its slab incl. halo exchange), slowest rank; fp64-issue-bound kernel"}

    # end to end through the slab API with this rank's host buffers: upload
    # u, v from pinned memory, residual + Jv, download F and Jv, every step
    u_pin = [p.cpu().pin_memory() for p in u.parts]
    v_pin = [p.cpu().pin_memory() for p in v.parts]
    f_pin = [torch.empty_like(p).pin_memory() for p in u_pin]
    j_pin = [torch.empty_like(p).pin_memory() for p in u_pin]
    u_d = [torch.empty_like(p) for p in u.parts]
    v_d = [torch.empty_like(p) for p in v.parts]

    def e2e_step():
        for i in range(len(u_d)):
            u_d[i].copy_(u_pin[i], non_blocking=True)
            v_d[i].copy_(v_pin[i], non_blocking=True)
        uu, vv = sp.wrap(list(u_d)), sp.wrap(list(v_d))
        f = res.device_call(uu, check=False)
        jv = res.jv_device(uu, f, vv, sp.norm(uu))
        for i in range(len(u_d)):
            f_pin[i].copy_(f.parts[i], non_blocking=True)
            j_pin[i].copy_(jv.parts[i], non_blocking=True)

    e2e_ms = timed(e2e_step, args.steps)
    nb = 2 * 2 * sum(nlocs) * 8
    e2e = {"value": round(2 * D_glob / (e2e_ms * 1e-3) / 1e6, 2), "unit": "MDoF/s",
           "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb,
           "ms_per_step": round(e2e_ms, 3), "note": "per rank (its slabs), max over ranks"}
    del u_pin, v_pin, f_pin, j_pin, u_d, v_d
    u = v = old = prev = res = None
    torch.cuda.empty_cache()

    # seconds per Newton iteration: first (backward-Euler) step of the seeded
    # dendrite on the same slabs, multicolor V-cycle, NCCL halos + allreduces
    newton = None
    if not args.no_newton and w["model"] == "free_growth":
        st = sp.wrap([seed_initial_condition_device(mesh, kern.params, ctx=c) for c in grp.ctxs])
        sc0 = uc.ThetaScheme(1.0, w["dt"], 0)
        walls, rep, t_build = [], None, 0.0
        for _ in range(4):  # cold + three warm solves (median: host jitter)
            barrier()
            t0 = time.perf_counter()
            pc = SlabPrecond(grp, st, sc0, uc.PrecondConfig(ordering="multicolor"))
            barrier()
            t_build = time.perf_counter() - t0
            r0 = SlabResidual(grp, st, st, sc0)
            barrier()
            t0 = time.perf_counter()
            # CGS2 Arnoldi: two vector allreduces per step instead of 2(k+1)
            # scalar ones (same counts as MGS: tests/test_gpu_cgs2.py)
            _, rep = uc.newton_solve(r0, st, uc.NewtonConfig(gmres=uc.GmresConfig(orthogonalization="cgs2")),
                                     precond_apply=pc.apply)
            barrier()
            walls.append(max_ms(time.perf_counter() - t0))
        t_newton = float(np.median(walls[1:]))
        vv = sp.wrap([torch.randn_like(p) for p in st.parts])
        t_apply = timed(lambda: pc._uc_deferred(vv), 5)
        newton = {"sec_per_newton_iteration": round(t_newton / max(rep.iterations, 1), 5),
                  "newton_iterations": rep.iterations, "gmres_per_newton": rep.gmres_iterations,
                  "converged": bool(rep.converged), "precond_build_s": round(t_build, 4),
                  "cold_sec_per_newton_iteration": round(walls[0] / max(rep.iterations, 1), 5),
                  "vcycle_apply_ms": round(t_apply, 3),
                  "case": "seed IC, step 0 (backward-Euler startup), default solver settings except "
                          "CGS2 Arnoldi, slabs",
                  "ordering": "multicolor", "timing": "host wall clock per solve, max over ranks"}
        pc = r0 = None

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline_line(w)
    if dist is not None:
        dist.barrier()
    if rank == 0:
        line = {
            "metric": "MDoF/s residual+Jv fill", "value": round(value, 2), "unit": "MDoF/s",
            "n_gpus": 1 if emulate else world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.workload, "model": w["model"], "dim": w["dim"], "counts": counts,
                       "dof": D_glob, "dof_per_step": 2 * D_glob,
                       "parallelism": (f"slab x{nslab} emulated in one process (testing)" if emulate
                                       else f"slab x{world} host-staged transport, GPUs shared (testing)"
                                       if HOST_TRANSPORT else f"slab x{world} (NCCL ghost planes + allreduce)"),
                       "l2": "per-rank inputs larger than L2; no flush"},
            "gpu_launches": 5 * args.steps, "clocks": clk.summary(), "roofline": roofline,
            "e2e": e2e, "cpu_baseline": cpu, "newton": newton,
        }
        print(json.dumps(line), flush=True)


def hbm_peak_gbs():
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        with open(pk) as fh:
            peaks = json.load(fh)
        if "hbm_gbs" in peaks:
            return float(peaks["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def roofline_kernel_name(w):
    return f"k_residual<{w['dim']},{'FG' if w['model'] == 'free_growth' else 'ALLOY'},NEW>"


def reference_python_1core_for(w):
    for name, ww in WORKLOADS.items():
        if ww is w or ww == w:
            return reference_python_1core(name)
    return None


def cpu_baseline_line(w):
    """The CPU port of the reference on this host's cores, bounded sample."""
    N = int(np.prod([c + 1 for c in w["counts"]]))
    try:
        sec, Dc, sample, cores = cpu_oracle_step_time(w, steps=1, warmup=1,
                                                     rows=None if w["dim"] == 2 and N <= 2049 ** 2 else 128,
                                                     min_seconds=10.0)
        return {"value": round(2 * Dc / sec / 1e6, 4), "unit": "MDoF/s", "cores": cores,
                "kind": "port", "sample": sample + "; residual+Jv of oracle/uc_oracle.c (OpenMP, "
                                                   f"{cores}-thread C port of the reference)",
                "label": f"{cores}-thread C port",
                "reference_python_1core": reference_python_1core_for(w)}
    except Exception as exc:  # reported, not fatal
        return {"value": None, "unit": "MDoF/s", "cores": 0, "kind": "port", "sample": f"failed: {exc}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="fg2d_2048", choices=sorted(WORKLOADS))
    ap.add_argument("--no-lex", action="store_true", help="skip the lexicographic-ordering Newton solve")
    ap.add_argument("--emulate-slabs", type=int, default=0,
                    help="testing: run the N>1 slab path with K slabs in this process on one GPU")
    ap.add_argument("--no-newton", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the al2d_4096 / fg3d_256 extra lines")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N > 1: weak = mesh grows with N (default), strong = the named mesh split N ways")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    w = WORKLOADS[args.workload]

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl != "reference":
        # one rank per GPU: launch them ourselves (the driver's torchrun form)
        import socket

        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, w, rank, world)
        return
    if "WORLD_SIZE" in os.environ and world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)

    import torch

    if HOST_TRANSPORT:
        local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dist = None
    if args.emulate_slabs > 1 and world == 1:
        run_slabs(args, w, rank, world, local, None, emulate=args.emulate_slabs)
        return
    if world > 1:
        import torch.distributed as dist

        if HOST_TRANSPORT:
            # testing the N > 1 path on a 1-GPU lease: ranks share the devices,
            # gloo + the library's host-staged transport instead of NCCL
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        run_slabs(args, w, rank, world, local, dist)
        if HOST_TRANSPORT:
            from paper_2006_16764_b200 import _lib as L

            L.load().uc_comm_finalize()
        dist.destroy_process_group()
        return

    line = run_single(args, w, local)
    print(json.dumps(line), flush=True)


def _timed(fn, reps, stream):
    import torch

    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def fill_phase(args, wname, local, steps, warmup, e2e=True):
    """Residual + fused Jv on synthetic states of workload `wname`: device-
    resident throughput, per-kernel times, roofline, end-to-end through the
    public API with host buffers."""
    import ctypes as C

    import torch

    import paper_2006_16764_b200 as uc
    from paper_2006_16764_b200 import _lib as L
    from paper_2006_16764_b200 import device as D

    w = WORKLOADS[wname]
    dev = torch.device("cuda", local)
    N, u_h, old_h, prev_h, v_h = synthetic_states(w)
    Dof = 2 * N
    mesh = uc.build_mesh(w["dim"], w["extents"], w["counts"])
    kern = uc.FreeGrowthKernel() if w["model"] == "free_growth" else uc.AlloyKernel()
    sc = uc.ThetaScheme(w["theta"], w["dt"], w["step"])
    u = torch.from_numpy(u_h).to(dev)
    v = torch.from_numpy(v_h).to(dev)
    res = uc.TimestepResidual(mesh, kern, torch.from_numpy(old_h).to(dev), torch.from_numpy(prev_h).to(dev), sc)
    unorm = D.norm(u)
    stream = torch.cuda.current_stream()

    def step():
        f = res.device_call(u, check=False)
        return res.jv_device(u, f, v, unorm)

    clk = Clocks(local).__enter__()  # sampled from warm-up through the kernel timings
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / steps
    value = 2 * Dof / (ms * 1e-3) / 1e6
    if res.ctx.status().residual_nonfinite:
        raise RuntimeError("non-finite residual in benchmark inputs")
    f0 = res.device_call(u, check=False)
    t_res = _timed(lambda: res.device_call(u, check=False), max(steps, 50), stream)
    t_jv = _timed(lambda: res.jv_device(u, f0, v, unorm), max(steps, 50), stream)
    clk.__exit__()
    hbm_peak, peak_src = hbm_peak_gbs()
    res_bytes = 32 * Dof
    achieved = res_bytes / (t_res * 1e-3) / 1e9
    # DRAM bytes per launch of this kernel from the committed ncu --set full
    # capture (profiles/*/ncu_traffic.json, newest round first)
    traffic = None
    for rnd in ("r02", "r01"):
        try:
            with open(os.path.join(ROOT, "profiles", rnd, "ncu_traffic.json")) as fh:
                traffic = json.load(fh)["kernels"].get(roofline_kernel_name(w), {}).get(wname)
        except (OSError, ValueError, KeyError):
            traffic = None
        if traffic is not None:
            break
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "traffic": traffic, "algorithmic_bytes": res_bytes,
                "kernel": roofline_kernel_name(w), "bytes_per_dof": 32, "ms_per_launch": round(t_res, 4),
                "peak_source": peak_src,
                "note": "fp64-issue-bound kernel; HBM fraction ceiling ~20-30% in 2D (DESIGN.md)"}
    # FP64 roofline of the same kernel: DP instructions per element measured
    # with ncu (profiles/dp_inst_per_element.json) over the measured DFMA issue rate
    dp_per_elem = {}
    try:
        with open(os.path.join(ROOT, "profiles", "dp_inst_per_element.json")) as fh:
            for key, val in json.load(fh)["kernels"].items():
                model, dims, mode = key.rsplit("_", 2)
                if mode == "new":
                    dp_per_elem[(model, int(dims[0]))] = val["dp_inst_per_element"]
    except Exception:
        pass
    ms_probe, dfma_rate = C.c_double(), C.c_double()
    bl = D.blas()
    L.check(bl.lib.uc_fp64_probe(bl.bind(), 20000, C.byref(ms_probe), C.byref(dfma_rate)), "uc_fp64_probe")
    ne = int(np.prod(w["counts"]))
    dpe = dp_per_elem.get((w["model"], w["dim"]))
    fp64 = {"bound": "fp64", "peak_dp_inst_per_s": round(dfma_rate.value / 1e12, 3),
            "peak_tflops_dfma": round(2 * dfma_rate.value / 1e12, 3), "unit": "T DP inst/s",
            "dp_inst_per_element": dpe, "kernel": roofline_kernel_name(w),
            "note": "DP instructions per element from ncu (profiles/dp_inst_per_element.json); "
                    "peak = measured DFMA issue rate (uc_fp64_probe)"}
    if dpe:
        ach = dpe * ne / (t_res * 1e-3)
        fp64.update({"achieved": round(ach / 1e12, 3), "frac": round(ach / dfma_rate.value, 4)})
    kernels = {"residual_ms": round(t_res, 4), "jv_ms": round(t_jv, 4),
               "residual_mdofs": round(Dof / (t_res * 1e-3) / 1e6, 1),
               "jv_mdofs": round(Dof / (t_jv * 1e-3) / 1e6, 1),
               "jv_gbs": round(48 * Dof / (t_jv * 1e-3) / 1e9, 1)}
    out = {"value": round(value, 2), "ms_per_step": round(ms, 4), "dof": Dof, "roofline": roofline,
           "fp64_roofline": fp64, "kernels": kernels, "clocks": clk.summary(),
           "gpu_launches": 5 * steps}

    if e2e:
        # ---- end to end through the public API with host buffers ----------
        # Each step copies u, v from pinned host memory, calls the public API
        # (TimestepResidual.__call__ + jfnk_matvec) and copies F, Jv back.  Copies
        # run on two copy streams (double-buffered) so the download of step i
        # overlaps the upload of step i+1; every byte still moves inside the
        # timed region.
        u_pin = torch.from_numpy(u_h).pin_memory()
        v_pin = torch.from_numpy(v_h).pin_memory()
        f_pin = [torch.empty(Dof, dtype=torch.float64).pin_memory() for _ in range(2)]
        j_pin = [torch.empty(Dof, dtype=torch.float64).pin_memory() for _ in range(2)]
        u_d = [torch.empty(Dof, dtype=torch.float64, device=dev) for _ in range(2)]
        v_d = [torch.empty(Dof, dtype=torch.float64, device=dev) for _ in range(2)]
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]

        def upload(i):
            k = i % 2
            with torch.cuda.stream(s_in):
                s_in.wait_event(ev_out[k])  # buffer k free again (step i-2's results left)
                u_d[k].copy_(u_pin, non_blocking=True)
                v_d[k].copy_(v_pin, non_blocking=True)
                ev_in[k].record(s_in)

        def e2e_run(nsteps):
            # the upload of step i+1 is enqueued before step i's API calls (which
            # synchronise on their non-finite checks), so it overlaps step i's
            # compute and step i-1's download
            upload(0)
            for i in range(nsteps):
                k = i % 2
                if i + 1 < nsteps:
                    upload(i + 1)
                stream.wait_event(ev_in[k])
                F = res(u_d[k])
                Jv = uc.jfnk_matvec(res, u_d[k], F, v_d[k])
                ev_out[k].record(stream)
                with torch.cuda.stream(s_out):
                    s_out.wait_event(ev_out[k])
                    f_pin[k].copy_(F, non_blocking=True)
                    j_pin[k].copy_(Jv, non_blocking=True)
                    ev_out[k].record(s_out)
                F.record_stream(s_out)  # keep F, Jv alive until their download ran
                Jv.record_stream(s_out)

        e2e_run(warmup)
        torch.cuda.synchronize()
        a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        e2e_run(steps)
        stream.wait_stream(s_out)  # end mark after the last download
        b0.record(stream)
        torch.cuda.synchronize()
        e2e_ms = a0.elapsed_time(b0) / steps
        out["e2e"] = {"value": round(2 * Dof / (e2e_ms * 1e-3) / 1e6, 2), "unit": "MDoF/s",
                      "h2d_bytes_per_step": 2 * Dof * 8, "d2h_bytes_per_step": 2 * Dof * 8,
                      "ms_per_step": round(e2e_ms, 3), "copies": "pinned, double-buffered copy streams"}
    return out


def newton_phase(args, wname, orderings=("multicolor",)):
    """Seconds per implicit Newton iteration: the first (backward-Euler
    startup) step of the reference's initial condition (free growth: seeded
    dendrite; alloy: perturbed directional front), default solver settings,
    cold + three warm solves (median); V-cycle apply time and effective
    bandwidth; seconds per implicit time step through driver.simulate (the
    package's time loop)."""
    import torch

    import paper_2006_16764_b200 as uc
    from paper_2006_16764_b200.config import default_config
    from paper_2006_16764_b200.driver import simulate
    from paper_2006_16764_b200.models import directional_initial_condition_device, seed_initial_condition_device

    w = WORKLOADS[wname]
    mesh = uc.build_mesh(w["dim"], w["extents"], w["counts"])
    kern = uc.FreeGrowthKernel() if w["model"] == "free_growth" else uc.AlloyKernel()
    if w["model"] == "free_growth":
        st = seed_initial_condition_device(mesh, kern.params)
    else:
        st = directional_initial_condition_device(mesh, kern.params, amplitude=0.5, seed=0, smooth=True)
    sc0 = uc.ThetaScheme(1.0, w["dt"], 0)
    stream = torch.cuda.current_stream()
    N = mesh.n_nodes
    hbm_peak, _ = hbm_peak_gbs()
    out = {}
    for ordering in orderings:
        walls, rep, t_build, pc = [], None, 0.0, None
        reps = 4 if ordering == "multicolor" else 1
        clk = Clocks(torch.cuda.current_device()).__enter__()
        for _ in range(reps):  # cold (first) and warm solves (median: host jitter)
            pc = None  # recycle the previous hierarchy (precond._pool)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pc = uc.build_precond(mesh, kern, st, sc0, uc.PrecondConfig(ordering=ordering))
            torch.cuda.synchronize()
            t_build = time.perf_counter() - t0
            r0 = uc.TimestepResidual(mesh, kern, st, st, sc0)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            _, rep = uc.newton_solve(r0, st, uc.NewtonConfig(), precond_apply=pc.apply)
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t0)
        vv = torch.randn_like(st)
        t_apply = _timed(lambda: pc.device_apply(vv, check=False), 5 if ordering == "multicolor" else 2, stream)
        clk.__exit__()
        t_newton = float(np.median(walls[1:] if len(walls) > 1 else walls))
        d = {"sec_per_newton_iteration": round(t_newton / max(rep.iterations, 1), 5),
             "newton_iterations": rep.iterations, "gmres_per_newton": rep.gmres_iterations,
             "converged": bool(rep.converged), "precond_build_s": round(t_build, 4),
             "vcycle_apply_ms": round(t_apply, 3), "clocks": clk.summary()}
        if ordering == "multicolor":
            vb = vcycle_bytes(pc, N, w["dim"])
            d.update({"cold_sec_per_newton_iteration": round(walls[0] / max(rep.iterations, 1), 5),
                      "vcycle_gbs": round(vb / (t_apply * 1e-3) / 1e9, 1),
                      "vcycle_hbm_frac": round(vb / (t_apply * 1e-3) / 1e9 / hbm_peak, 4),
                      "case": ("seed IC" if w["model"] == "free_growth" else "directional IC (amplitude 0.5)")
                              + ", step 0 (backward-Euler startup), default solver settings",
                      "ordering": "multicolor"})
            out.update(d)
        else:
            d["note"] = "the reference's default ordering: exact sequential sweep (pipelined wavefront)"
            out[ordering] = d
        pc = r0 = None
    # implicit time steps through the package's time loop (driver.simulate):
    # startup step(s) then Crank-Nicolson, preconditioner rebuilt every step
    cfg = default_config(w["model"])
    cfg.mesh.dimension, cfg.mesh.extents, cfg.mesh.counts = w["dim"], tuple(w["extents"]), tuple(w["counts"])
    cfg.time.dt = w["dt"]
    cfg.time.t_final = 3 * w["dt"]
    cfg.precond.ordering = "multicolor"
    simulate(cfg)  # cold run: allocations, captured preconditioner graphs
    res = simulate(cfg)
    out["sec_per_time_step"] = round(res.loop_seconds / max(res.steps_completed, 1), 5)
    out["time_steps"] = {"steps": res.steps_completed, "newton": [r["newton_iters"] for r in res.records],
                         "gmres": [r["gmres_iters"] for r in res.records], "status": res.status,
                         "loop": "driver.simulate (startup steps at theta=1, then theta=0.5); warm (second) run"}
    return out


def run_single(args, w, local):
    import gc

    import torch

    torch.cuda.set_device(local)
    fill = fill_phase(args, args.workload, local, args.steps, args.warmup)
    gc.collect()
    torch.cuda.empty_cache()
    newton = None
    if not args.no_newton:
        orderings = ("multicolor",)
        if not args.no_lex and w["dim"] == 2 and np.prod(w["counts"]) <= 2048 * 2048:
            orderings = ("multicolor", "lexicographic")
        newton = newton_phase(args, args.workload, orderings)
        gc.collect()
        torch.cuda.empty_cache()
    # the other named configs (BASELINE.json configs[2], configs[3]) on this GPU:
    # fill + seconds per Newton iteration, each with its clock record
    extra = {}
    if not args.no_extra and args.workload == "fg2d_2048":
        for wname in ("al2d_4096", "fg3d_256"):
            try:
                ex = fill_phase(args, wname, local, max(args.steps // 2, 5), args.warmup, e2e=False)
                gc.collect()
                torch.cuda.empty_cache()
                if not args.no_newton:
                    ex["newton"] = newton_phase(args, wname)
                ex["config"] = {k: WORKLOADS[wname][k] for k in ("model", "dim", "counts")}
                extra[wname] = ex
            except Exception as exc:  # reported, never fatal to the headline line
                extra[wname] = {"error": repr(exc)}
            gc.collect()
            torch.cuda.empty_cache()
    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline_line(w)
    Dof = fill["dof"]
    line = {
        "metric": "MDoF/s residual+Jv fill", "value": fill["value"], "unit": "MDoF/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": fill["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "model": w["model"], "dim": w["dim"],
                   "counts": list(w["counts"]), "dof": Dof, "dof_per_step": 2 * Dof,
                   "l2": "inputs (~470 MB working set) larger than L2; no flush",
                   "parallelism": "single GPU"},
        "roofline": fill["roofline"], "fp64_roofline": fill["fp64_roofline"], "kernels": fill["kernels"],
        "e2e": fill["e2e"], "gpu_launches": fill["gpu_launches"], "clocks": fill["clocks"],
        "newton": newton, "workloads": extra or None, "cpu_baseline": cpu,
    }
    return line


if __name__ == "__main__":
    main()
