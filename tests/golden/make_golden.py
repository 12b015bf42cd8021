"""Generate golden input/output vectors by running the REFERENCE implementation.

This script is test infrastructure: it imports the reference package
(`undercool`, /root/reference/pkg/src) in this container, evaluates the hot-path
functions on small seeded inputs and writes the results under tests/golden/.
The GPU box has no /root/reference, so the committed .npz/.json files are what
the tests read there.  Re-run with:

    NUMBA_CACHE_DIR=/tmp/nbcache python tests/golden/make_golden.py

Reference entry points exercised (file:line under /root/reference/pkg/src/undercool):
  assemble_residual            assembly.py:214
  TimestepResidual             assembly.py:233-268
  jfnk_matvec                  newton.py:84-94
  assemble_field_matrix        assembly.py:271-303
  build_precond / apply        precond.py:269-299, 248-264
  gmres_solve                  krylov.py:81-208
  newton_solve                 newton.py:116-198
  simulate (iteration counts)  driver.py:135-242
  MassDiffKernel test plug-in  tests/test_assembly.py:22-49 (massdiff_cases)
  simulate records / outcomes  driver.py:186-229 (driver_cases)
  _heat_balance, _total_solute driver.py:76-98, extract_tip diagnostics.py:69-89
"""

from __future__ import annotations

import json
import os
import sys
import time

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")
REF = os.environ.get("UC_REFERENCE_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import numpy as np  # noqa: E402

import undercool as uc  # noqa: E402
from undercool.assembly import StateHistory, assemble_residual  # noqa: E402
from undercool.config import default_config  # noqa: E402
from undercool.driver import simulate  # noqa: E402
from undercool.models.alloy import AlloyParams, directional_initial_condition  # noqa: E402
from undercool.models.free_growth import seed_initial_condition  # noqa: E402
from undercool.newton import _FdOperator  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def fg_state(rng, n):
    # distribution of tests/test_free_growth.py:246-256
    return uc.join_fields(0.5 + 0.3 * rng.standard_normal(n), 1.0 + 0.2 * rng.standard_normal(n))


def alloy_state(rng, n):
    # distribution of tests/test_alloy.py:286-295
    return uc.join_fields(np.tanh(rng.standard_normal(n)), -0.5 + 0.4 * rng.standard_normal(n))


RESIDUAL_CASES = [
    # name, model, dim, extents, counts, theta, dt, step, normalized
    ("fg2d", "free_growth", 2, (0.48, 0.36), (16, 12), 0.5, 3e-4, 2, True),
    ("fg3d", "free_growth", 3, (0.24, 0.18, 0.15), (8, 6, 5), 0.5, 3e-4, 2, True),
    ("al2d", "alloy", 2, (6.4, 4.8), (8, 6), 0.5, 0.002, 7, True),
    ("al2d_unnorm", "alloy", 2, (6.4, 4.8), (8, 6), 0.5, 0.002, 7, False),
    ("al3d", "alloy", 3, (4.8, 3.2, 2.4), (6, 4, 3), 0.5, 0.002, 7, True),
    ("fg2d_be", "free_growth", 2, (0.48, 0.36), (16, 12), 1.0, 2.25e-4, 0, True),
]


def kernel_for(model, normalized=True):
    if model == "free_growth":
        return uc.FreeGrowthKernel()
    return uc.AlloyKernel(AlloyParams(antitrapping_normalized=normalized))


def residual_cases(meta):
    for name, model, dim, ext, cnt, th, dt, step, norm in RESIDUAL_CASES:
        mesh = uc.build_mesh(dim, ext, cnt)
        k = kernel_for(model, norm)
        n = mesh.n_nodes
        rng = np.random.default_rng(11 if model == "free_growth" else 12)
        mk = fg_state if model == "free_growth" else alloy_state
        new, old, prev = mk(rng, n), mk(rng, n), mk(rng, n)
        scheme = uc.ThetaScheme(th, dt, step)
        st = StateHistory(new, old, prev)
        f_full = assemble_residual(mesh, k, st, scheme, part="full")
        f_new = assemble_residual(mesh, k, st, scheme, part="new")
        res = uc.TimestepResidual(mesh, k, old, prev, scheme)
        f_call = res(new)
        v = np.random.default_rng(2).standard_normal(2 * n)
        op = _FdOperator(res, new, f_call)
        jv = op(v)
        jv2 = uc.jfnk_matvec(res, new, f_call, v)
        np.savez_compressed(
            os.path.join(OUT, f"residual_{name}.npz"),
            new=new, old=old, prev=prev, v=v,
            f_full=f_full, f_new=f_new, fixed=res.fixed_part, f_call=f_call,
            jv=jv, jv_matvec=jv2, eps=np.array(op.epsilons),
        )
        meta[f"residual_{name}"] = dict(model=model, dim=dim, extents=ext, counts=cnt,
                                         theta=th, dt=dt, step=step, normalized=norm)


PRECOND_CASES = [
    # name, model, dim, extents, counts, theta, dt, step
    ("fg2d", "free_growth", 2, (0.96, 0.48), (32, 16), 0.5, 2.25e-4, 3),
    ("fg3d", "free_growth", 3, (0.48, 0.24, 0.24), (16, 8, 8), 0.5, 2.25e-4, 3),
    ("al2d", "alloy", 2, (25.6, 12.8), (32, 16), 0.5, 0.002, 3),
    ("al3d", "alloy", 3, (12.8, 6.4, 6.4), (16, 8, 8), 0.5, 0.002, 3),
]


def precond_cases(meta):
    for name, model, dim, ext, cnt, th, dt, step in PRECOND_CASES:
        mesh = uc.build_mesh(dim, ext, cnt)
        k = kernel_for(model)
        n = mesh.n_nodes
        rng = np.random.default_rng(11 if model == "free_growth" else 12)
        if model == "free_growth":
            state = fg_state(rng, n)
        else:
            # solute kept above -1/(1-k) so the phase-block mass stays positive
            state = uc.join_fields(np.tanh(rng.standard_normal(n)),
                                   np.clip(-0.5 + 0.3 * rng.standard_normal(n), -1.0, 0.9))
        scheme = uc.ThetaScheme(th, dt, step)
        v = np.random.default_rng(2).standard_normal(2 * n)
        out = dict(state=state, v=v)
        qs = uc.assembly.frozen_quad_state(mesh, k, state, scheme)
        coeffs = k.precond_coefficients(qs, scheme)
        for b, (cm, cd) in enumerate(coeffs):
            mat = uc.assemble_field_matrix(mesh, cm, cd).tocsr()
            mat.sort_indices()
            out[f"A{b}_data"] = mat.data
            out[f"A{b}_indices"] = mat.indices
            out[f"A{b}_indptr"] = mat.indptr
        for kind in ("identity", "jacobi", "sgs", "vcycle"):
            cfg = uc.PrecondConfig(kind=kind, ordering="multicolor")
            pc = uc.build_precond(mesh, k, state, scheme, cfg)
            out[f"apply_{kind}"] = pc.apply(v)
            if kind in ("sgs", "vcycle"):  # the reference's default ordering
                lex = uc.build_precond(mesh, k, state, scheme, uc.PrecondConfig(kind=kind))
                out[f"apply_{kind}_lex"] = lex.apply(v)
            if kind == "vcycle":
                sizes = [m.shape[0] for m in pc.solvers[0].mats]
                for lvl, m in enumerate(pc.solvers[0].mats[1:], start=1):
                    for b in range(2):
                        mm = pc.solvers[b].mats[lvl].tocsr()
                        mm.sort_indices()
                        out[f"L{lvl}_A{b}_data"] = mm.data
                        out[f"L{lvl}_A{b}_indices"] = mm.indices
                        out[f"L{lvl}_A{b}_indptr"] = mm.indptr
        # non-default V-cycle settings
        cfg = uc.PrecondConfig(kind="vcycle", ordering="multicolor", sweeps=1, cycles=1,
                               levels=2, coarse_sweeps=3)
        out["apply_vcycle_small"] = uc.build_precond(mesh, k, state, scheme, cfg).apply(v)
        np.savez_compressed(os.path.join(OUT, f"precond_{name}.npz"), **out)
        meta[f"precond_{name}"] = dict(model=model, dim=dim, extents=ext, counts=cnt,
                                        theta=th, dt=dt, step=step, levels=sizes)


def newton_case(meta):
    """One preconditioned Newton solve (first step of a seed run)."""
    mesh = uc.build_mesh(2, (0.96, 0.96), (32, 32))
    k = uc.FreeGrowthKernel()
    u0 = seed_initial_condition(mesh, k.params, radius=0.3)
    scheme = uc.ThetaScheme(1.0, 2.25e-4, 0)
    pc = uc.build_precond(mesh, k, u0, scheme, uc.PrecondConfig(ordering="multicolor"))
    res = uc.TimestepResidual(mesh, k, u0, u0.copy(), scheme)
    u, rep = uc.newton_solve(res, u0, uc.NewtonConfig(), precond_apply=pc.apply)
    f0 = res(u0)
    op = _FdOperator(res, u0, f0)
    lin = uc.gmres_solve(op, -f0, tol=0.1, apply_minv=pc.apply)
    np.savez_compressed(os.path.join(OUT, "newton_fg2d_32.npz"), u0=u0, u=u, f0=f0,
                        gmres_x=lin.x, norms=np.array(rep.residual_norms))
    meta["newton_fg2d_32"] = dict(iterations=rep.iterations, gmres=rep.gmres_iterations,
                                  converged=bool(rep.converged), step_lengths=[float(x) for x in rep.step_lengths],
                                  gmres_first=dict(iterations=lin.iterations,
                                                   converged=bool(lin.converged),
                                                   residual_norm=float(lin.residual_norm),
                                                   cycles=lin.cycles,
                                                   precond_applies=lin.precond_applies))


RUNS = [
    # name, model, dim, extents, counts, dt, t_final(steps), extra overrides
    ("fg2d_128_10", "free_growth", 2, (3.84, 3.84), (128, 128), 2.25e-4, 10, {}, True),
    ("fg2d_128_10_nopc", "free_growth", 2, (3.84, 3.84), (128, 128), 2.25e-4, 10,
     {"enabled": False}, False),
    ("al2d_256x64_10", "alloy", 2, (204.8, 51.2), (256, 64), 0.002, 10, {}, True),
    ("fg3d_16_3", "free_growth", 3, (0.48, 0.48, 0.48), (16, 16, 16), 2.25e-4, 3, {}, True),
    ("al3d_32x16x16_3", "alloy", 3, (25.6, 12.8, 12.8), (32, 16, 16), 0.002, 3, {}, True),
    ("fg2d_512_3", "free_growth", 2, (15.36, 15.36), (512, 512), 2.25e-4, 3, {}, False),
    ("fg2d_128_10_lex", "free_growth", 2, (3.84, 3.84), (128, 128), 2.25e-4, 10,
     {"ordering": "lexicographic"}, True),
    ("al2d_256x64_10_lex", "alloy", 2, (204.8, 51.2), (256, 64), 0.002, 10,
     {"ordering": "lexicographic"}, True),
    ("al2d_512_3", "alloy", 2, (409.6, 409.6), (512, 512), 0.002, 3, {}, False),
]


def run_cases(meta, only=None):
    for name, model, dim, ext, cnt, dt, nsteps, pc_over, keep in RUNS:
        if only and name not in only:
            continue
        cfg = default_config(model)
        cfg.mesh.dimension = dim
        cfg.mesh.extents = ext
        cfg.mesh.counts = cnt
        cfg.time.dt = dt
        cfg.time.t_final = dt * nsteps
        cfg.precond.ordering = "multicolor"
        for key, val in pc_over.items():
            setattr(cfg.precond, key, val)
        t0 = time.perf_counter()
        res = simulate(cfg)
        wall = time.perf_counter() - t0
        recs = res.records
        meta[f"run_{name}"] = dict(
            model=model, dim=dim, extents=ext, counts=cnt, dt=dt, steps=nsteps,
            precond=pc_over, status=res.status,
            newton=[r["newton_iters"] for r in recs],
            gmres=[r["gmres_iters"] for r in recs],
            fnorm=[float(r["fnorm"]) for r in recs],
            fnorm0=[float(r["fnorm0"]) for r in recs],
            theta=cfg.time.theta, startup_steps=cfg.time.startup_steps,
            startup_dt=cfg.time.startup_dt, wall_seconds=wall,
        )
        if keep:
            np.savez_compressed(os.path.join(OUT, f"run_{name}.npz"), state=res.state)
        print(name, meta[f"run_{name}"]["newton"], meta[f"run_{name}"]["gmres"],
              f"{wall:.1f}s", flush=True)


def ic_cases(meta):
    mesh = uc.build_mesh(2, (204.8, 51.2), (256, 64))
    p = AlloyParams()
    ic = directional_initial_condition(mesh, p, amplitude=0.5, seed=0, smooth=True)
    mesh2 = uc.build_mesh(2, (3.84, 3.84), (128, 128))
    seed = seed_initial_condition(mesh2, uc.FreeGrowthParams())
    np.savez_compressed(os.path.join(OUT, "ic.npz"), alloy_256x64=ic, seed_128=seed)
    meta["ic"] = dict(alloy=dict(extents=(204.8, 51.2), counts=(256, 64)),
                      seed=dict(extents=(3.84, 3.84), counts=(128, 128)))


def _rec_json(r):
    out = {}
    for key, val in r.items():
        if isinstance(val, (np.floating, float)):
            out[key] = float(val)
        elif isinstance(val, (np.integer, int)):
            out[key] = int(val)
        else:
            out[key] = val
    return out


def _small_fg(**time_kw):
    # tests/test_driver.py:22-27
    from undercool.config import MeshConfig, RunConfig, TimeConfig

    cfg = RunConfig()
    cfg.mesh = MeshConfig(dimension=2, extents=(0.96, 0.96), counts=(32, 32))
    cfg.time = TimeConfig(**({"theta": 0.5, "dt": 1e-5, "t_final": 1e-4} | time_kw))
    return cfg


def driver_cases(meta):
    """Full simulate() records and outcomes at the reference's own test configs
    (tests/test_driver.py:22-27,118-163) with the default solver settings."""
    from undercool.config import MeshConfig, TimeConfig

    cases = {}
    cases["fg2d_32_10"] = _small_fg()
    cases["fg2d_32_balance6"] = _small_fg(dt=2.25e-4, t_final=2.25e-4 * 6)
    cases["fg2d_32_explicit"] = _small_fg(theta=0.0, dt=5.625e-4, t_final=5.625e-4 * 50)
    c = _small_fg(dt=2.25e-4, t_final=2.25e-4 * 2)
    c.solver.max_iterations = 1
    c.solver.rel_tol = 1e-14
    cases["fg2d_32_starved"] = c
    c = _small_fg(dt=2.25e-4, t_final=2.25e-4 * 2)
    c.solver.max_iterations = 1
    c.solver.rel_tol = 1e-14
    c.retry_halve_dt = True
    cases["fg2d_32_starved_retry"] = c
    c = default_config("alloy")
    c.mesh = MeshConfig(dimension=2, extents=(102.4, 25.6), counts=(128, 32))
    c.time = TimeConfig(theta=0.5, dt=0.002, t_final=0.02)
    cases["al2d_128x32_10"] = c
    c = _small_fg(dt=2.25e-4, t_final=2.25e-4 * 3)
    c.mesh = MeshConfig(dimension=3, extents=(0.48, 0.48, 0.48), counts=(16, 16, 16))
    cases["fg3d_16_3"] = c
    c = default_config("alloy")
    c.mesh = MeshConfig(dimension=3, extents=(25.6, 12.8, 12.8), counts=(32, 16, 16))
    c.time = TimeConfig(theta=0.5, dt=0.002, t_final=0.006)
    cases["al3d_32x16x16_3"] = c
    for name, cfg in cases.items():
        t0 = time.perf_counter()
        res = simulate(cfg)
        m = dict(status=res.status, steps_completed=res.steps_completed,
                 final_time=float(res.final_time), total_newton=res.total_newton,
                 total_gmres=res.total_gmres, failure_detail=res.failure_detail,
                 timescales={k: float(v) for k, v in res.timescales.items()},
                 records=[_rec_json(r) for r in res.records],
                 config=dict(model=cfg.model, dim=cfg.mesh.dimension, extents=list(cfg.mesh.extents),
                             counts=list(cfg.mesh.counts), theta=cfg.time.theta, dt=cfg.time.dt,
                             t_final=cfg.time.t_final, startup_dt=cfg.time.startup_dt,
                             max_iterations=cfg.solver.max_iterations, rel_tol=cfg.solver.rel_tol,
                             retry_halve_dt=cfg.retry_halve_dt),
                 wall_seconds=time.perf_counter() - t0)
        meta[f"driver_{name}"] = m
        if res.status == "ok":
            np.savez_compressed(os.path.join(OUT, f"driver_{name}.npz"), state=res.state)
        print("driver", name, res.status, res.steps_completed, f"{m['wall_seconds']:.1f}s", flush=True)


def diag_cases(meta):
    """Diagnostics on the residual goldens' seeded states (driver.py:76-98,
    diagnostics.py:69-89) plus tip profiles of the reference's tests."""
    from undercool.diagnostics import extract_tip
    from undercool.driver import _heat_balance, _total_solute

    for name, model, dim, ext, cnt, th, dt, step, norm in RESIDUAL_CASES:
        g = np.load(os.path.join(OUT, f"residual_{name}.npz"))
        mesh = uc.build_mesh(dim, ext, cnt)
        k = kernel_for(model, norm)
        w = mesh.integration_weights()
        n = mesh.n_nodes
        new, old, prev = g["new"], g["old"], g["prev"]
        d = dict(w_dT=float(w @ (new[n:] - old[n:])), w_dphi_new=float(w @ (new[:n] - old[:n])),
                 w_dphi_old=float(w @ (old[:n] - prev[:n])), max_abs=float(np.max(np.abs(new))))
        if model == "free_growth":
            bal, bound = _heat_balance(mesh, k, StateHistory(new, old, prev), uc.ThetaScheme(th, dt, step), 0.25)
            d.update(balance=bal, bound=bound)
        else:
            d["total_solute"] = _total_solute(mesh, k, new)
        if dim == 2:
            tip, found = extract_tip(new, mesh, k.contour_level, 2)
            d.update(x_tip=float(tip), found=bool(found))
        meta[f"diag_{name}"] = d
    # tip profiles: step, tanh, no crossing, exact zero (tests/test_diagnostics.py)
    mesh = uc.build_mesh(2, (4.5, 4.5), (150, 150))
    xs = mesh.coords[:, 0]
    profiles = {
        "step": np.where(xs < 1.234, 1.0, 0.0),
        "tanh": 0.5 * (1.0 - np.tanh((xs - 2.71) / 0.1)),
        "none": np.ones_like(xs),
        "exact": np.where(xs < 1.5, 1.0, np.where(np.isclose(xs, 1.5), 0.5, 0.0)),
    }
    tips = {}
    for pname, phi in profiles.items():
        state = uc.join_fields(phi, np.zeros(mesh.n_nodes))
        tip, found = extract_tip(state, mesh, 0.5, 2)
        tips[pname] = dict(x_tip=float(tip), found=bool(found))
    meta["diag_tips_150"] = tips


def writer_cases(meta):
    """Reference writer outputs (vtkio.py:31-86, driver.py:244-275, config.py:150-174)
    on golden states, gzipped under tests/golden/writers/."""
    import gzip
    import tempfile

    from undercool.config import save_config
    from undercool.driver import _field_dict, run
    from undercool.vtkio import write_mesh_vtk, write_snapshot_csv, write_snapshot_vtk

    wdir = os.path.join(OUT, "writers")
    os.makedirs(wdir, exist_ok=True)

    def keep(src, name):
        with open(src, "rb") as fh, open(os.path.join(wdir, name + ".gz"), "wb") as out:
            out.write(gzip.compress(fh.read(), mtime=0))

    cases = [("fg2d_32_10", "free_growth", 2, (0.96, 0.96), (32, 32), 1e-4),
             ("al2d_128x32_10", "alloy", 2, (102.4, 25.6), (128, 32), 0.02),
             ("fg3d_16_3", "free_growth", 3, (0.48, 0.48, 0.48), (16, 16, 16), 6.75e-4)]
    info = {}
    with tempfile.TemporaryDirectory() as tmp:
        for name, model, dim, ext, cnt, t in cases:
            cfg = default_config(model)
            mesh = uc.build_mesh(dim, ext, cnt)
            k = cfg.kernel()
            state = np.load(os.path.join(OUT, f"driver_{name}.npz"))["state"]
            fields = _field_dict(cfg, k, state)
            write_snapshot_csv(mesh, fields, os.path.join(tmp, "s.csv"))
            write_snapshot_vtk(mesh, fields, os.path.join(tmp, "s.vtk"), comment=f"t = {t!r}")
            keep(os.path.join(tmp, "s.csv"), f"snapshot_{name}.csv")
            keep(os.path.join(tmp, "s.vtk"), f"snapshot_{name}.vtk")
            info[name] = dict(model=model, dim=dim, extents=ext, counts=cnt, t=t,
                              fields=list(fields))
            if "composition" in fields:
                np.savez_compressed(os.path.join(wdir, f"composition_{name}.npz"),
                                    composition=fields["composition"])
        for name, dim, ext, cnt in [("mesh2d_6x4", 2, (0.6, 0.4), (6, 4)),
                                    ("mesh3d_4x3x2", 3, (0.4, 0.3, 0.2), (4, 3, 2))]:
            write_mesh_vtk(uc.build_mesh(dim, ext, cnt), os.path.join(tmp, "m.vtk"))
            keep(os.path.join(tmp, "m.vtk"), name + ".vtk")
            info[name] = dict(dim=dim, extents=ext, counts=cnt)
        for model in ("free_growth", "alloy"):
            with open(os.path.join(tmp, "c.txt"), "w") as fh:
                fh.write(save_config(default_config(model)))
            keep(os.path.join(tmp, "c.txt"), f"config_{model}.used")
        # a full run() of tests/test_driver.py:22-27 with snapshots every 5 steps
        cfg = _small_fg()
        cfg.output.directory = os.path.join(tmp, "run")
        cfg.output.snapshot_every = 5
        code, _ = run(cfg)
        names = sorted(os.listdir(cfg.output.directory))
        keep(os.path.join(cfg.output.directory, "runlog.csv"), "run_fg2d_32_10.runlog.csv")
        with open(os.path.join(cfg.output.directory, "summary.json")) as fh:
            summ = json.load(fh)
        info["run_fg2d_32_10"] = dict(code=code, files=names, summary_keys=sorted(summ),
                                      snapshots=summ["snapshots"])
    meta["writers"] = info


MASSDIFF_CASES = [
    # name, dim, extents, counts, diffusivity, mass, theta, dt
    ("md2d", 2, (1.2, 0.8), (12, 10), 0.7, True, 0.5, 0.05),
    ("md2d_nomass", 2, (2.0, 1.0), (8, 6), 1.3, False, 1.0, 0.1),
    ("md3d", 3, (0.6, 0.5, 0.4), (5, 4, 3), 0.9, True, 0.6, 0.02),
]


def massdiff_cases(meta):
    """The reference's single-field assembly test plug-in (tests/test_assembly.py:22-49)
    run through assemble_residual (all three parts), TimestepResidual, jfnk_matvec
    and an unpreconditioned newton_solve."""
    import importlib.util

    spec = importlib.util.spec_from_file_location(
        "ref_test_assembly", os.path.join(os.path.dirname(REF), "tests", "test_assembly.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    MassDiffKernel = mod.MassDiffKernel
    from undercool.assembly import TimestepResidual
    from undercool.newton import jfnk_matvec, newton_solve
    from undercool.stepping import ThetaScheme

    for name, dim, ext, cnt, c, mass, theta, dt in MASSDIFF_CASES:
        mesh = uc.build_mesh(dim, list(ext), list(cnt))
        k = MassDiffKernel(diffusivity=c, mass=mass)
        rng = np.random.default_rng(21)
        n = mesh.n_nodes
        new, old, prev, v = (rng.standard_normal(n) for _ in range(4))
        sc = ThetaScheme(theta, dt, 0)
        st = StateHistory(new, old, prev)
        out = {p: assemble_residual(mesh, k, st, sc, part=p) for p in ("old", "new", "full")}
        res = TimestepResidual(mesh, k, old, prev, sc)
        fu = res(new)
        jv = jfnk_matvec(res, new, fu, v)
        res2 = TimestepResidual(mesh, k, old, prev, sc)
        u, rep = newton_solve(res2, old.copy())
        np.savez(os.path.join(OUT, f"massdiff_{name}.npz"), new=new, old=old, prev=prev, v=v,
                 r_old=out["old"], r_new=out["new"], r_full=out["full"], fixed=res.fixed_part,
                 fu=fu, jv=jv, newton_u=u)
        meta[f"massdiff_{name}"] = dict(dim=dim, extents=ext, counts=cnt, diffusivity=c, mass=mass,
                                        theta=theta, dt=dt, newton=rep.iterations,
                                        gmres=rep.gmres_iterations, converged=rep.converged)
        print(name, rep.iterations, rep.gmres_iterations, rep.converged)


def subset_cases(meta):
    """assemble_residual(..., elements=subset) (assembly.py:214-230) for both
    models in 2D and 3D: one element colour class and a random subset."""
    cases = [("fg2d", "free_growth", 2, (0.48, 0.36), (16, 12), 0.5, 3e-4, 2),
             ("al3d", "alloy", 3, (6.4, 4.8, 3.2), (8, 6, 4), 0.5, 2e-3, 3)]
    for name, model, dim, ext, cnt, th, dt, step in cases:
        mesh = uc.build_mesh(dim, list(ext), list(cnt))
        k = kernel_for(model)
        rng = np.random.default_rng(31)
        mk = fg_state if model == "free_growth" else alloy_state
        new, old, prev = (mk(rng, mesh.n_nodes) for _ in range(3))
        sc = uc.ThetaScheme(th, dt, step)
        st = StateHistory(new, old, prev)
        color = mesh.colors[1]
        rand = rng.permutation(mesh.n_elements)[: mesh.n_elements // 3]
        out = dict(new=new, old=old, prev=prev, color=color, rand=rand)
        for sub in ("color", "rand"):
            for p in ("old", "new", "full"):
                out[f"{sub}_{p}"] = assemble_residual(mesh, k, st, sc, elements=out[sub], part=p)
        np.savez(os.path.join(OUT, f"subset_{name}.npz"), **out)
        meta[f"subset_{name}"] = dict(model=model, dim=dim, extents=ext, counts=cnt, theta=th, dt=dt,
                                      step=step)
        print("subset", name)


DROPIN_CASES = [
    # name, model, dim, extents, counts
    ("fg2d", "free_growth", 2, (0.48, 0.36), (16, 12)),
    ("al3d", "alloy", 3, (4.8, 3.2, 2.4), (6, 4, 3)),
]


def dropin_cases(meta):
    """frozen_quad_state (assembly.py:193-211), eval_basis (mesh.py:259-265) and
    assemble_field_matrix (assembly.py:271-303) with per-point, scalar and
    non-default-rule coefficients."""
    for name, model, dim, ext, cnt in DROPIN_CASES:
        mesh = uc.build_mesh(dim, ext, cnt)
        k = kernel_for(model)
        n, ne = mesh.n_nodes, mesh.n_elements
        rng = np.random.default_rng(21)
        state = fg_state(rng, n) if model == "free_growth" else alloy_state(rng, n)
        scheme = uc.ThetaScheme(0.5, 3e-4, 2)
        qs = uc.assembly.frozen_quad_state(mesh, k, state, scheme)
        out = dict(state=state, coords=qs.coords)
        for f in range(k.n_fields):
            out[f"val{f}"] = qs.val_new[f]
            for d in range(dim):
                out[f"grad{f}_{d}"] = qs.grad_new[f][d]
        for ppa in (2, 3, 4):
            rule = uc.gauss_rule(dim, ppa)
            b = uc.eval_basis(mesh, 0, rule)
            out[f"basis{ppa}_values"] = b.values
            out[f"basis{ppa}_gradients"] = b.gradients
            out[f"basis{ppa}_jxw"] = b.jxw
        nq = 3 ** dim
        cm = 0.5 + rng.random((ne, nq))
        cd = 0.1 + rng.random((ne, nq))
        out.update(cm=cm, cd=cd)
        for tag, a, b_, rule in (("qp", cm, cd, None), ("scalar", 2.5, 0.75, None),
                                  ("rule2", cm[:, : 2 ** dim] * 1.0, 0.75, uc.gauss_rule(dim, 2))):
            mat = uc.assemble_field_matrix(mesh, a, b_, rule).tocsr()
            mat.sort_indices()
            out[f"M{tag}_data"] = mat.data
            out[f"M{tag}_indices"] = mat.indices
            out[f"M{tag}_indptr"] = mat.indptr
        np.savez_compressed(os.path.join(OUT, f"dropin_{name}.npz"), **out)
        meta[f"dropin_{name}"] = dict(model=model, dim=dim, extents=ext, counts=cnt, theta=0.5, dt=3e-4, step=2)


def survey_case(meta):
    """configs[1] at full size: two implicit steps of the seeded dendrite at
    2048^2 through the reference's own simulate() (default solver; ~8 min)."""
    cfg = default_config("free_growth")
    cfg.mesh.extents, cfg.mesh.counts = (61.44, 61.44), (2048, 2048)
    cfg.time.t_final = 2 * cfg.time.dt
    cfg.precond.ordering = "multicolor"
    t0 = time.perf_counter()
    res = simulate(cfg)
    recs = res.records
    meta["survey_fg2d_2048_2"] = dict(
        model="free_growth", dim=2, extents=(61.44, 61.44), counts=(2048, 2048), dt=cfg.time.dt, steps=2,
        status=res.status, newton=[r["newton_iters"] for r in recs], gmres=[r["gmres_iters"] for r in recs],
        fnorm=[float(r["fnorm"]) for r in recs], fnorm0=[float(r["fnorm0"]) for r in recs],
        theta=cfg.time.theta, startup_steps=cfg.time.startup_steps, wall_seconds=time.perf_counter() - t0,
        source="reference simulate() via tests/golden/make_golden.py --only-survey")
    print("survey", meta["survey_fg2d_2048_2"], flush=True)


def main():
    meta = {"generator": "tests/golden/make_golden.py", "reference": REF}
    if "--only-survey" in sys.argv:
        survey_case(meta)
        full = json.load(open(os.path.join(OUT, "golden.json")))
        full.update({k: v for k, v in meta.items() if k.startswith("survey_")})
        with open(os.path.join(OUT, "golden.json"), "w") as fh:
            json.dump(full, fh, indent=1, sort_keys=True)
        return
    if "--only-dropin" in sys.argv:
        meta = json.load(open(os.path.join(OUT, "golden.json")))
        dropin_cases(meta)
        with open(os.path.join(OUT, "golden.json"), "w") as fh:
            json.dump(meta, fh, indent=1, sort_keys=True)
        return
    if "--only-massdiff" in sys.argv:
        meta = json.load(open(os.path.join(OUT, "golden.json")))
        massdiff_cases(meta)
        subset_cases(meta)
        with open(os.path.join(OUT, "golden.json"), "w") as fh:
            json.dump(meta, fh, indent=1, sort_keys=True)
        return
    if "--only-writers" in sys.argv:
        meta = json.load(open(os.path.join(OUT, "golden.json")))
        writer_cases(meta)
        with open(os.path.join(OUT, "golden.json"), "w") as fh:
            json.dump(meta, fh, indent=1, sort_keys=True)
        return
    if "--only-driver" in sys.argv:
        meta = json.load(open(os.path.join(OUT, "golden.json")))
        driver_cases(meta)
        diag_cases(meta)
        writer_cases(meta)
        with open(os.path.join(OUT, "golden.json"), "w") as fh:
            json.dump(meta, fh, indent=1, sort_keys=True)
        return
    if "--only-runs" not in sys.argv:
        residual_cases(meta)
        massdiff_cases(meta)
        subset_cases(meta)
        precond_cases(meta)
        newton_case(meta)
        ic_cases(meta)
        dropin_cases(meta)
    old = json.load(open(os.path.join(OUT, "golden.json"))) if os.path.exists(os.path.join(OUT, "golden.json")) else {}
    if "--only-runs" in sys.argv:
        meta = old
        run_cases(meta, only=sys.argv[sys.argv.index("--only-runs") + 1].split(","))
    elif "--no-runs" not in sys.argv:
        run_cases(meta)
        driver_cases(meta)
        diag_cases(meta)
        writer_cases(meta)
    else:
        meta.update({k: v for k, v in old.items() if k.startswith("run_")})
    meta.update({k: v for k, v in old.items() if k.startswith("survey_") and k not in meta})
    with open(os.path.join(OUT, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
