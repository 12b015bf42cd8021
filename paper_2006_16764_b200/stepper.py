"""Minimal host time loop over the device hot path.

Mirrors the step policy of undercool/driver.py:160-179 (startup steps at
startup_theta, preconditioner rebuilt from the time-level-n state every step,
one Newton solve per step, state rotation) without the reference's I/O,
diagnostics or retry logic, which stay out of scope.  Used by the parity
tests and bench.py.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from . import device as D
from .assembly import TimestepResidual
from .newton import NewtonConfig, newton_solve
from .precond import PrecondConfig, build_precond
from .stepping import ThetaScheme

__all__ = ["StepRecord", "run_steps"]


@dataclass
class StepRecord:
    step: int
    newton_iters: int
    gmres_iters: int
    gmres_per_newton: list = field(default_factory=list)
    fnorm0: float = 0.0
    fnorm: float = 0.0
    converged: bool = True


def run_steps(mesh, kernel, state0, nsteps: int, theta: float, dt: float,
              startup_steps: int = 2, startup_theta: float = 1.0,
              newton: NewtonConfig | None = None, precond: PrecondConfig | None = None,
              precond_enabled: bool = True):
    ncfg = newton or NewtonConfig()
    pcfg = precond or PrecondConfig(ordering="multicolor")
    state = D.as_device(state0)
    prev = state.clone()
    records = []
    for n in range(nsteps):
        th = startup_theta if (n < startup_steps and 0.0 < theta < 1.0) else theta
        scheme = ThetaScheme(th, dt, n)
        pc = None
        if precond_enabled and pcfg.kind != "identity":
            pc = build_precond(mesh, kernel, state, scheme, pcfg)
        res = TimestepResidual(mesh, kernel, state, prev, scheme)
        u_new, rep = newton_solve(res, state, ncfg, precond_apply=pc.apply if pc else None)
        records.append(StepRecord(n, rep.iterations, rep.total_gmres, list(rep.gmres_iterations),
                                  rep.initial_norm, rep.final_norm, rep.converged))
        # drop this step's preconditioner before the next build so its level
        # buffers and captured graph are recycled (precond._pool)
        pc = res = None
        if not rep.converged:
            break
        prev, state = state, u_new
    return state, records
