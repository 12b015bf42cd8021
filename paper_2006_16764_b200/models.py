"""Physics plug-ins recognised by the device path.

The reference's kernels are duck-typed Python objects whose Gauss-point work
runs in numba (undercool/models/free_growth.py:149-243,
undercool/models/alloy.py:211-311).  A GPU cannot call back into Python per
quadrature point, so the device path recognises the two built-in models by
their parameter dataclasses and ships those constants to the CUDA kernels as
a POD struct (``device_params``).  Parameter objects of THIS package or of the
reference package are both accepted; any other kernel raises
NotImplementedError — there is no CPU fallback.
"""

from __future__ import annotations

from dataclasses import dataclass

from . import _lib as L

__all__ = ["FreeGrowthParams", "FreeGrowthKernel", "AlloyParams", "AlloyKernel",
           "MassDiffKernel", "device_params", "model_of", "n_fields_of"]

# thin-interface constants of the dilute-alloy model (alloy.py:31-33)
A1 = 0.8839
A2 = 0.6267


@dataclass
class FreeGrowthParams:
    """Pure-material constants; defaults and derived values as
    free_growth.py:31-80."""

    anisotropy_strength: float = 0.005
    thermal_diffusivity: float = 4.0
    kinetic_coeff: float = 191.82
    interface_width: float = 0.02652
    latent_ratio: float = 1.0
    far_temperature: float = 1.0
    undercooling: float = 0.55
    mesh_scale: float = 0.03
    seed_radius: float = 0.3
    aniso_reg_grad: float = 1.0

    @property
    def mobility(self) -> float:
        return 1.0 / self.kinetic_coeff

    @property
    def melt_temperature(self) -> float:
        return self.far_temperature + self.undercooling * self.latent_ratio

    @property
    def capillary_length(self) -> float:
        return 0.139 * self.interface_width

    def validate(self) -> None:
        for name in ("anisotropy_strength", "thermal_diffusivity", "kinetic_coeff",
                     "interface_width", "latent_ratio", "far_temperature", "mesh_scale",
                     "seed_radius"):
            if getattr(self, name) <= 0.0:
                raise ValueError(f"{name} must be positive")
        if not 0.0 <= self.undercooling < 1.0:
            raise ValueError("undercooling must lie in [0, 1)")


@dataclass
class AlloyParams:
    """Dilute binary alloy constants; defaults and scalings as alloy.py:38-99."""

    anisotropy_strength: float = 0.01
    partition: float = 0.14
    liquidus_slope: float = -2.6
    composition: float = 3.0
    coupling: float = 10.0
    liquid_diffusivity: float = 3e-9
    capillary_length: float = 5e-9
    thermal_gradient: float = 1e4
    gibbs_thomson: float = 2.4e-7
    pull_speed: float = 1e-2
    interface_x0: float = 8.0
    antitrapping_normalized: bool = True
    aniso_reg_grad: float = 0.05
    antitrap_reg_grad: float = 0.02

    @property
    def length_unit(self) -> float:
        return self.capillary_length * self.coupling / A1

    @property
    def time_unit(self) -> float:
        return self.capillary_length ** 2 / self.liquid_diffusivity * A2 * self.coupling ** 3 / A1 ** 2

    @property
    def diffusivity(self) -> float:
        return self.liquid_diffusivity * self.time_unit / self.length_unit ** 2

    @property
    def solute_d0(self) -> float:
        return self.diffusivity / (1.0 + self.partition)

    @property
    def pull_velocity(self) -> float:
        return self.pull_speed * self.time_unit / self.length_unit

    @property
    def frame_coefficient(self) -> float:
        k = self.partition
        denom = abs(self.liquidus_slope) * self.composition * (1.0 - k) / k
        return self.thermal_gradient * self.length_unit / denom

    def validate(self) -> None:
        if not 0.0 < self.partition < 1.0:
            raise ValueError("partition coefficient must lie in (0, 1)")
        if self.coupling <= 0.0:
            raise ValueError("coupling constant must be positive")
        for name in ("liquid_diffusivity", "capillary_length", "composition"):
            if getattr(self, name) <= 0.0:
                raise ValueError(f"{name} must be positive")


class FreeGrowthKernel:
    """Phase field + heat (free_growth.py:149-243 attributes)."""

    n_fields = 2
    field_names = ("phi", "temperature")
    contour_level = 0.5
    needs_rate = True

    def __init__(self, params: FreeGrowthParams | None = None):
        self.params = params or FreeGrowthParams()
        self.params.validate()

    def scales(self) -> dict:
        p = self.params
        bg = p.kinetic_coeff * p.mobility
        return {"tau": p.interface_width ** 2 / bg, "interface_width": p.interface_width,
                "heat_diffusivity": p.thermal_diffusivity, "solute_diffusivity": 0.0,
                "solute_d0": 0.0}


class AlloyKernel:
    """Phase field + solute with anti-trapping (alloy.py:211-311 attributes)."""

    n_fields = 2
    field_names = ("phi", "solute")
    contour_level = 0.0
    needs_rate = True
    needs_old_value = True

    def __init__(self, params: AlloyParams | None = None):
        self.params = params or AlloyParams()
        self.params.validate()

    def scales(self) -> dict:
        p = self.params
        return {"tau": 1.0, "interface_width": 1.0, "heat_diffusivity": 0.0,
                "solute_diffusivity": p.diffusivity, "solute_d0": p.solute_d0}


def is_mass_diff(kernel) -> bool:
    """The reference's single-field assembly test plug-in (tests/test_assembly.py:22-49)
    or this package's MassDiffKernel, recognised by name and attributes.  A
    subclass that overrides residual_gauss runs its own Python physics and is
    not recognised (no CPU fallback)."""
    name = type(kernel).__name__
    if name != "MassDiffKernel" and not isinstance(kernel, MassDiffKernel):
        return False
    if not (hasattr(kernel, "c") and hasattr(kernel, "mass") and getattr(kernel, "n_fields", 0) == 1):
        return False
    # a subclass with its own residual_gauss is a different model
    for klass in type(kernel).__mro__:
        if "residual_gauss" in vars(klass):
            return klass.__name__ == "MassDiffKernel"
    return True


class MassDiffKernel:
    """Single-field theta-method model (du/dt, psi) + (c grad u, grad psi): the
    reference's assembly test plug-in (tests/test_assembly.py:22-49), assembled
    on the device by csrc/massdiff.cu.  No preconditioner coefficients (the
    reference's plug-in has none either)."""

    n_fields = 1
    field_names = ("u",)
    contour_level = 0.5
    needs_rate = False
    needs_old_value = False

    def __init__(self, diffusivity=1.0, mass=True):
        self.c = diffusivity
        self.mass = mass


def n_fields_of(kernel) -> int:
    return 1 if model_of(kernel) == L.UC_MODEL_MASS_DIFF else 2


def model_of(kernel) -> int:
    """UC_MODEL_* for a kernel object of this package or the reference."""
    name = type(kernel).__name__
    p = getattr(kernel, "params", None)
    if name == "FreeGrowthKernel" and p is not None and hasattr(p, "thermal_diffusivity"):
        return L.UC_MODEL_FREE_GROWTH
    if name == "AlloyKernel" and p is not None and hasattr(p, "partition"):
        return L.UC_MODEL_ALLOY
    if is_mass_diff(kernel):
        return L.UC_MODEL_MASS_DIFF
    raise NotImplementedError(
        f"kernel {name!r} has no device implementation; only the built-in free-growth "
        "and alloy models run on the B200 path (no CPU fallback)")


def device_params(kernel) -> L.ModelParams:
    """POD constants for the CUDA kernels, derived with the same Python
    expressions as the reference's wrappers (free_growth.py:176-200,
    alloy.py:239-265)."""
    model = model_of(kernel)
    mp = L.ModelParams()
    mp.model = model
    if model == L.UC_MODEL_MASS_DIFF:
        mp.dcoef = float(kernel.c)
        mp.mass_coef = 1.0 if kernel.mass else 0.0
        return mp
    p = kernel.params
    mp.eps = p.anisotropy_strength
    mp.reg = p.aniso_reg_grad ** 4
    mp.aniso_reg_grad = p.aniso_reg_grad
    if model == L.UC_MODEL_FREE_GROWTH:
        mp.bg = p.kinetic_coeff * p.mobility
        mp.beta = p.kinetic_coeff
        mp.alpha = p.thermal_diffusivity
        mp.latent = p.latent_ratio
        mp.hcell = p.mesh_scale
        mp.tmelt = p.melt_temperature
    else:
        mp.normalized = 1 if p.antitrapping_normalized else 0
        mp.at_reg2 = p.antitrap_reg_grad ** 2
        mp.kpart = p.partition
        mp.coupling = p.coupling
        mp.dcoef = p.diffusivity
        mp.g4_coef = p.frame_coefficient
        mp.pull_velocity = p.pull_velocity
    return mp


# ---------------------------------------------------------------------------
# Initial conditions (host numpy; setup, not hot path).  SURVEY 8(f) lists
# their on-device generation as a later item.
# ---------------------------------------------------------------------------
def fourfold(grad, strength: float, reg_grad: float = 1e-3):
    """Anisotropy factor g of a gradient (anisotropy.py:31-68)."""
    import numpy as np

    p = np.asarray(grad, dtype=float)
    avg = 0.5 if p.shape[-1] == 2 else 1.0 / 3.0
    reg = reg_grad ** 4
    p2 = p * p
    s2 = p2.sum(axis=-1)
    ratio = ((p2 * p2).sum(axis=-1) + avg * reg) / (s2 * s2 + reg)
    return 1.0 - 3.0 * strength + 4.0 * strength * ratio


def seed_initial_condition(mesh, params: FreeGrowthParams, radius: float | None = None):
    """Corner seed phi = [|x| <= r g(x)], T = far-field (free_growth.py:249-265)."""
    import numpy as np

    r = params.seed_radius if radius is None else radius
    if r <= 0.0:
        raise ValueError("seed radius must be positive")
    x = mesh.coords
    dist = np.sqrt(np.sum(x * x, axis=1))
    phi = (dist <= r * fourfold(x, params.anisotropy_strength)).astype(float)
    return np.concatenate([phi, np.full(mesh.n_nodes, params.far_temperature)])


def _splitmix64(seed: int, index):
    import numpy as np

    z = (np.uint64(seed) + index.astype(np.uint64) + np.uint64(1)) * np.uint64(0x9E3779B97F4A7C15)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) / float(1 << 53)


def directional_initial_condition(mesh, params: AlloyParams, amplitude: float = 0.0, seed: int = 0,
                                  smooth: bool = False):
    """Corrugated planar interface, u = -1 (alloy.py:317-357)."""
    import math

    import numpy as np

    nx = mesh.node_shape[0]
    transverse = mesh.n_nodes // nx
    xi = 2.0 * _splitmix64(seed, np.arange(transverse, dtype=np.uint64)) - 1.0
    row = np.arange(mesh.n_nodes) // nx
    threshold = params.interface_x0 + amplitude * xi[row]
    x = mesh.coords[:, 0]
    if smooth:
        phi = np.tanh((threshold - x) / math.sqrt(2.0))
    else:
        phi = np.where(x <= threshold, 1.0, -1.0)
    return np.concatenate([phi, np.full(mesh.n_nodes, -1.0)])


def _device_initial(ctx, mesh, kind, params):
    import ctypes as C

    import torch

    ext = (C.c_double * 3)(*(list(mesh.extents) + [1.0] * (3 - mesh.dim)))
    par = (C.c_double * 4)(*(list(params) + [0.0] * (4 - len(params))))
    out = torch.empty(2 * ctx.n_local, dtype=torch.float64, device="cuda")
    L.check(ctx.lib.uc_initial_state(ctx.bind(), kind, ext, par, L.ptr(out)), "uc_initial_state")
    return out


def seed_initial_condition_device(mesh, params: FreeGrowthParams, radius: float | None = None, ctx=None):
    """seed_initial_condition generated on the GPU (no host coordinate array);
    with `ctx` (a slab context) only that slab's planes."""
    from .device import context_for

    r = params.seed_radius if radius is None else radius
    if r <= 0.0:
        raise ValueError("seed radius must be positive")
    ctx = ctx or context_for(mesh, FreeGrowthKernel(params))
    return _device_initial(ctx, mesh, 0, (params.anisotropy_strength, r, params.far_temperature))


def directional_initial_condition_device(mesh, params: AlloyParams, amplitude: float = 0.0,
                                         seed: int = 0, smooth: bool = False, ctx=None):
    """directional_initial_condition generated on the GPU."""
    from .device import context_for

    ctx = ctx or context_for(mesh, AlloyKernel(params))
    return _device_initial(ctx, mesh, 1, (params.interface_x0, amplitude, float(seed), 1.0 if smooth else 0.0))
