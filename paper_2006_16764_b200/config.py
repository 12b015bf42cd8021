"""Run configuration (mirrors undercool/config.py:27-117,150-174,224-232).

The sections and defaults, ``validate``, ``default_config`` and
``save_config`` (the ``config.used`` file ``driver.run`` writes, byte-identical
to the reference's).  ``driver.simulate`` also accepts the reference's own
``RunConfig`` objects (attribute access only).
"""

from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field

from .errors import ConfigError
from .models import AlloyKernel, AlloyParams, FreeGrowthKernel, FreeGrowthParams
from .newton import NewtonConfig
from .precond import PrecondConfig

__all__ = ["MeshConfig", "TimeConfig", "OutputConfig", "RunConfig", "save_config", "default_config"]


@dataclass
class MeshConfig:
    dimension: int = 2
    extents: tuple = (4.5, 4.5)
    counts: tuple = (150, 150)
    order: int = 1


@dataclass
class TimeConfig:
    theta: float = 0.5
    dt: float = 2.25e-4
    t_final: float = 0.14
    startup_steps: int = 2
    startup_theta: float = 1.0
    startup_dt: float = 0.0


@dataclass
class OutputConfig:
    directory: str = "out"
    snapshot_every: int = 0
    log_name: str = "runlog.csv"
    write_vtk: bool = True


@dataclass
class RunConfig:
    model: str = "free_growth"
    seed: int = 0
    perturbation: float = 0.5
    smooth_interface: bool = True
    retry_halve_dt: bool = False
    mesh: MeshConfig = field(default_factory=MeshConfig)
    time: TimeConfig = field(default_factory=TimeConfig)
    solver: NewtonConfig = field(default_factory=NewtonConfig)
    precond: PrecondConfig = field(default_factory=PrecondConfig)
    output: OutputConfig = field(default_factory=OutputConfig)
    free_growth: FreeGrowthParams = field(default_factory=FreeGrowthParams)
    alloy: AlloyParams = field(default_factory=AlloyParams)

    def validate(self) -> None:
        """config.py:74-97, same messages."""
        if self.model not in ("free_growth", "alloy"):
            raise ConfigError(f"unknown model '{self.model}'")
        m = self.mesh
        if m.dimension not in (2, 3):
            raise ConfigError("mesh.dimension must be 2 or 3")
        if len(m.extents) != m.dimension or len(m.counts) != m.dimension:
            raise ConfigError("mesh extents/counts must match the dimension")
        if any(e <= 0 for e in m.extents) or any(c < 1 for c in m.counts):
            raise ConfigError("mesh extents must be positive, counts at least 1")
        if m.order not in (1, 2) or (m.dimension == 3 and m.order != 1):
            raise ConfigError("element order must be 1 or 2 (1 only in 3D)")
        t = self.time
        if not 0.0 <= t.theta <= 1.0:
            raise ConfigError("time.theta must lie in [0, 1]")
        if t.dt <= 0.0 or t.t_final <= 0.0:
            raise ConfigError("time.dt and time.t_final must be positive")
        try:
            self.params().validate()
            p = self.precond
            PrecondConfig(p.enabled, p.kind, p.sweeps, p.cycles, p.levels, p.coarse_sweeps,
                          p.ordering, p.rebuild)
        except ValueError as exc:
            raise ConfigError(str(exc)) from exc

    def params(self):
        return self.free_growth if self.model == "free_growth" else self.alloy

    def kernel(self):
        if self.model == "free_growth":
            return FreeGrowthKernel(self.free_growth)
        return AlloyKernel(self.alloy)


_RUN_KEYS = ("model", "seed", "perturbation", "smooth_interface", "retry_halve_dt")
_DATACLASS_SECTIONS = ("mesh", "time", "solver", "precond", "output", "free_growth", "alloy")


def _text(v) -> str:
    """One value as config.py:120-127 prints it (repr for floats, true/false,
    comma-separated sequences)."""
    if v is True or v is False:
        return "true" if v else "false"
    if isinstance(v, (tuple, list)):
        return ", ".join(map(repr, v))
    return repr(v) if isinstance(v, float) else str(v)


def save_config(cfg, path=None) -> str:
    """The ``config.used`` text of config.py:150-174: [run], one section per
    dataclass (Newton without its nested gmres), then [gmres]; the layout
    configparser writes ("key = value" lines, a blank line after each
    section).  Reading config files back (load_config / parse_overrides) is
    the reference CLI's business and is not mirrored."""
    sections = [("run", [(k, getattr(cfg, k)) for k in _RUN_KEYS])]
    for name in _DATACLASS_SECTIONS:
        sub = getattr(cfg, name)
        if dataclasses.is_dataclass(sub):
            sections.append((name, [(f.name, getattr(sub, f.name)) for f in dataclasses.fields(sub)
                                    if f.name != "gmres"]))
    g = cfg.solver.gmres
    # the extension field is written only when it differs from the reference's behaviour
    sections.append(("gmres", [(f.name, getattr(g, f.name)) for f in dataclasses.fields(g)
                               if not (f.name == "orthogonalization" and getattr(g, f.name) == "mgs")]))
    lines = []
    for name, items in sections:
        lines.append(f"[{name}]")
        lines.extend(f"{k} = {_text(v)}" for k, v in items)
        lines.append("")
    text = "\n".join(lines) + "\n"
    if path is not None:
        with open(path, "w") as fh:
            fh.write(text)
    return text


def default_config(model: str) -> RunConfig:
    """Benchmark defaults per model (config.py:224-232)."""
    cfg = RunConfig(model=model)
    if model == "alloy":
        cfg.mesh = MeshConfig(dimension=2, extents=(204.8, 51.2), counts=(256, 64))
        cfg.time = TimeConfig(theta=0.5, dt=0.002, t_final=10.0, startup_dt=0.002)
    return cfg
