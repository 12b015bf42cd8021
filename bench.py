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
    line = {
        "impl": "reference", "metric": "MDoF/s residual+Jv fill", "value": round(mdofs, 4),
        "unit": "MDoF/s", "n_gpus": args.gpus, "device": "host cores only", "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, **{k: w[k] for k in ("model", "dim", "counts")}},
        "cpu_baseline": {"value": round(mdofs, 4), "unit": "MDoF/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(mdofs, 4), "unit": "MDoF/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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
        cyc(0)
        if c > 0:
            total += (stencil[0] + 24) * rows[0] + 24 * rows[0]  # residual + x += e
    return 2 * total  # both field blocks


def run_slabs(args, w, rank, world, local, dist, emulate=0):
    """N > 1: one slab per GPU of a weak-scaled mesh (counts[-1] x world), NCCL
    ghost planes and allreduce inside the library (paper_2006_16764_b200.parallel).
    emulate=K (testing, --emulate-slabs): the same code path with K slabs driven
    by this one process on one GPU (planes copied on the stream instead of NCCL)."""
    import torch

    import paper_2006_16764_b200 as uc
    from paper_2006_16764_b200.parallel import SlabGroup, SlabResidual

    dev = torch.device("cuda", local)
    nslab = emulate if emulate else world
    counts = list(w["counts"])
    extents = list(w["extents"])
    counts[-1] *= nslab
    extents[-1] *= nslab
    mesh = uc.build_mesh(w["dim"], extents, counts)
    kern = uc.FreeGrowthKernel() if w["model"] == "free_growth" else uc.AlloyKernel()
    sc = uc.ThetaScheme(w["theta"], w["dt"], w["step"])
    grp = SlabGroup.local(mesh, kern, nslab) if emulate else SlabGroup.from_torch_dist(mesh, kern)
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

    clk = Clocks(local).__enter__()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(args.steps):
        step()
    b.record(stream)
    torch.cuda.synchronize()
    barrier()
    clk.__exit__()
    ms = max_ms(a.elapsed_time(b) / args.steps)
    D_glob = 2 * int(np.prod([c + 1 for c in counts]))
    value = 2 * D_glob / (ms * 1e-3) / 1e6

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

    for _ in range(args.warmup):
        e2e_step()
    torch.cuda.synchronize()
    barrier()
    a.record(stream)
    for _ in range(args.steps):
        e2e_step()
    b.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_ms(a.elapsed_time(b) / args.steps)
    nb = 2 * 2 * sum(nlocs) * 8
    e2e = {"value": round(2 * D_glob / (e2e_ms * 1e-3) / 1e6, 2), "unit": "MDoF/s",
           "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb,
           "ms_per_step": round(e2e_ms, 3), "note": "per rank (its slabs), max over ranks"}
    if rank == 0:
        line = {
            "metric": "MDoF/s residual+Jv fill", "value": round(value, 2), "unit": "MDoF/s",
            "n_gpus": 1 if emulate else world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.workload, "model": w["model"], "dim": w["dim"], "counts": counts,
                       "dof": D_glob, "dof_per_step": 2 * D_glob,
                       "parallelism": (f"slab x{nslab} emulated in one process (testing)" if emulate
                                       else f"slab x{world} (NCCL ghost planes + allreduce)"),
                       "l2": "per-rank inputs larger than L2; no flush"},
            "gpu_launches": 5 * args.steps, "clocks": clk.summary(), "roofline": None,
            "e2e": e2e, "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)


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
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    w = WORKLOADS[args.workload]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, w, rank, world)
        return

    import torch

    torch.cuda.set_device(local)
    dist = None
    if args.emulate_slabs > 1 and world == 1:
        run_slabs(args, w, rank, world, local, None, emulate=args.emulate_slabs)
        return
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        run_slabs(args, w, rank, world, local, dist)
        dist.destroy_process_group()
        return

    import ctypes as C

    import paper_2006_16764_b200 as uc
    from paper_2006_16764_b200 import _lib as L
    from paper_2006_16764_b200 import device as D
    from paper_2006_16764_b200.models import seed_initial_condition_device

    dev = torch.device("cuda", local)
    N, u_h, old_h, prev_h, v_h = synthetic_states(w)
    Dof = 2 * N
    mesh = uc.build_mesh(w["dim"], w["extents"], w["counts"])
    kern = uc.FreeGrowthKernel() if w["model"] == "free_growth" else uc.AlloyKernel()
    sc = uc.ThetaScheme(w["theta"], w["dt"], w["step"])
    u = torch.from_numpy(u_h).to(dev)
    v = torch.from_numpy(v_h).to(dev)
    res = uc.TimestepResidual(mesh, kern, torch.from_numpy(old_h).to(dev),
                              torch.from_numpy(prev_h).to(dev), sc)
    unorm = D.norm(u)
    stream = torch.cuda.current_stream()

    def step():
        f = res.device_call(u, check=False)
        return res.jv_device(u, f, v, unorm)

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident throughput ------------------------------------
    clk = Clocks(local).__enter__()  # sampled from warm-up through the kernel timings
    for _ in range(args.warmup):
        step()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    value = world * 2 * Dof / (ms * 1e-3) / 1e6
    if res.ctx.status().residual_nonfinite:
        raise RuntimeError("non-finite residual in benchmark inputs")

    # ---- per-kernel durations (CUDA events on the launching stream) ----
    def timed(fn, reps):
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

    f0 = res.device_call(u, check=False)
    t_res = timed(lambda: res.device_call(u, check=False), max(args.steps, 50))
    t_jv = timed(lambda: res.jv_device(u, f0, v, unorm), max(args.steps, 50))
    clk.__exit__()
    peaks = {}
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        with open(pk) as fh:
            peaks = json.load(fh)
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    def roofline_kernel_name(w):
        return f"k_residual<{w['dim']},{'FG' if w['model'] == 'free_growth' else 'ALLOY'},NEW>"

    res_bytes = 32 * Dof
    achieved = res_bytes / (t_res * 1e-3) / 1e9
    # DRAM bytes per launch of this kernel from the committed ncu --set full
    # capture (profiles/r01/ncu_traffic.json), when it covers this workload
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r01", "ncu_traffic.json")) as fh:
            traffic = json.load(fh)["kernels"].get(roofline_kernel_name(w), {}).get(args.workload)
    except (OSError, ValueError, KeyError):
        traffic = None
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                "algorithmic_bytes": res_bytes,
                "kernel": f"k_residual<{w['dim']},{'FG' if w['model'] == 'free_growth' else 'ALLOY'},NEW>",
                "bytes_per_dof": 32, "ms_per_launch": round(t_res, 4), "peak_source": peak_src,
                "note": "fp64-issue-bound kernel; HBM fraction ceiling ~20-30% in 2D (DESIGN.md)"}
    # FP64 roofline of the same kernel: DP instructions per element measured
    # with ncu (profiles/r01/SUMMARY.md) over the measured DFMA issue rate
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

    # ---- end-to-end through the public API with host buffers ----------
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

    e2e_run(args.warmup)
    torch.cuda.synchronize()
    barrier()
    a0, b0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    e2e_run(args.steps)
    stream.wait_stream(s_out)  # end mark after the last download
    b0.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(a0.elapsed_time(b0) / args.steps)
    e2e = {"value": round(world * 2 * Dof / (e2e_ms * 1e-3) / 1e6, 2), "unit": "MDoF/s",
           "h2d_bytes_per_step": 2 * Dof * 8, "d2h_bytes_per_step": 2 * Dof * 8,
           "ms_per_step": round(e2e_ms, 3), "copies": "pinned, double-buffered copy streams"}
    launches_per_step = 5  # residual tile + edge fix-up, |v| reduction, Jv tile + edge fix-up

    # ---- Newton step on the seeded dendrite --------------------------
    # release the fill-phase working set first (512^3: ~2.2 GB per vector)
    del u_pin, v_pin, f_pin, j_pin, u_d, v_d, f0
    u = v = res = None
    import gc

    gc.collect()
    torch.cuda.empty_cache()
    free_b, total_b = torch.cuda.mem_get_info()
    print(f"[bench] device memory before Newton phase: free {free_b / 2**30:.1f} / {total_b / 2**30:.1f} GiB, "
          f"torch allocated {torch.cuda.memory_allocated() / 2**30:.1f} GiB", file=sys.stderr, flush=True)
    newton = None
    if not args.no_newton and w["model"] == "free_growth":
        u0 = seed_initial_condition_device(mesh, kern.params)
        if u0 is not None:
            st = u0
            sc0 = uc.ThetaScheme(1.0, w["dt"], 0)
            walls = []
            pc = r0 = None
            for rep_i in range(4):  # cold (first) and three warm solves (median: host jitter)
                pc = r0 = None  # recycle the previous hierarchy (precond._pool)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                pc = uc.build_precond(mesh, kern, st, sc0, uc.PrecondConfig(ordering="multicolor"))
                torch.cuda.synchronize()
                t_build = time.perf_counter() - t0
                r0 = uc.TimestepResidual(mesh, kern, st, st, sc0)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                _, rep = uc.newton_solve(r0, st, uc.NewtonConfig(), precond_apply=pc.apply)
                torch.cuda.synchronize()
                walls.append(time.perf_counter() - t0)
            t_newton = float(np.median(walls[1:]))
            vv = torch.randn_like(st)
            t_apply = timed(lambda: pc.device_apply(vv, check=False), 5)
            vb = vcycle_bytes(pc, N, w["dim"])
            pc = r0 = None
            # full implicit time steps (precond build + Newton) through the host loop
            from paper_2006_16764_b200.stepper import run_steps
            step_walls = []
            state = st
            prev_state = st
            for n in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                state_new, recs = run_steps(mesh, kern, state, 1, 0.5, w["dt"], startup_steps=0)
                torch.cuda.synchronize()
                step_walls.append(time.perf_counter() - t0)
                state = state_new
            newton = {"sec_per_newton_iteration": round(t_newton / max(rep.iterations, 1), 5),
                      "newton_iterations": rep.iterations, "gmres_per_newton": rep.gmres_iterations,
                      "converged": bool(rep.converged), "precond_build_s": round(t_build, 4),
                      "cold_sec_per_newton_iteration": round(walls[0] / max(rep.iterations, 1), 5),
                      "sec_per_time_step": round(float(np.mean(step_walls[1:])), 5),
                      "time_step_walls_s": [round(x, 5) for x in step_walls],
                      "vcycle_apply_ms": round(t_apply, 3),
                      "vcycle_gbs": round(vb / (t_apply * 1e-3) / 1e9, 1),
                      "vcycle_hbm_frac": round(vb / (t_apply * 1e-3) / 1e9 / hbm_peak, 4),
                      "case": "seed IC, step 0 (backward-Euler startup), default solver settings",
                      "ordering": "multicolor"}
            # the reference's DEFAULT smoother ordering: exact sequential
            # (lexicographic) Gauss-Seidel, pipelined wavefront kernel
            if not args.no_lex and N <= 2049 * 2049:
                pc = uc.build_precond(mesh, kern, st, sc0, uc.PrecondConfig(ordering="lexicographic"))
                r0 = uc.TimestepResidual(mesh, kern, st, st, sc0)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                _, rep_l = uc.newton_solve(r0, st, uc.NewtonConfig(), precond_apply=pc.apply)
                torch.cuda.synchronize()
                t_lex = time.perf_counter() - t0
                t_apply_l = timed(lambda: pc.device_apply(vv, check=False), 3)
                pc = r0 = None
                newton["lexicographic"] = {
                    "sec_per_newton_iteration": round(t_lex / max(rep_l.iterations, 1), 5),
                    "newton_iterations": rep_l.iterations, "gmres_per_newton": rep_l.gmres_iterations,
                    "vcycle_apply_ms": round(t_apply_l, 3),
                    "note": "reference default ordering; sequential sweep as a pipelined wavefront (fronts i+2j)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sec, Dc, sample, cores = cpu_oracle_step_time(w, steps=1, warmup=1,
                                                         rows=None if w["dim"] == 2 and N <= 2049 ** 2 else 128,
                                                         min_seconds=10.0)
            cpu = {"value": round(2 * Dc / sec / 1e6, 4), "unit": "MDoF/s", "cores": cores,
                   "kind": "port", "sample": sample + "; residual+Jv of oracle/uc_oracle.c (OpenMP)"}
        except Exception as exc:  # reported, not fatal
            cpu = {"value": None, "unit": "MDoF/s", "cores": 0, "kind": "port", "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": "MDoF/s residual+Jv fill", "value": round(value, 2), "unit": "MDoF/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "model": w["model"], "dim": w["dim"],
                       "counts": list(w["counts"]), "dof": Dof, "dof_per_step": 2 * Dof,
                       "l2": "inputs (~470 MB working set) larger than L2; no flush",
                       "parallelism": f"replicas x{world}"},
            "roofline": roofline, "fp64_roofline": fp64, "kernels": kernels, "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps, "clocks": clk.summary(),
            "newton": newton, "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
