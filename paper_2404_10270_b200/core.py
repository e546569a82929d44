"""Domain types and host-side plasma loading.

`Grid1D`, `SpeciesDef` and `PhysicalConstants` carry the same fields and
validation as the reference (pkg/src/picmc/core.py:29-93), so a reference
config object can be handed to this engine unchanged (attributes are read by
name).  Particle storage is NOT the reference's per-cell slack segments: the
engine keeps a flat structure of arrays with an int32 cell index per
particle on the GPU (see store.py and DESIGN.md).
"""

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import InitError
from .rng import STREAM_INIT, derive_vec, stream, uniforms, uniforms_open

ELEMENTARY_CHARGE = 1.602176634e-19   # pkg/src/picmc/constants.py:3-10
EPSILON_0 = 8.8541878128e-12
ELECTRON_MASS = 9.1093837015e-31
ATOMIC_MASS_UNIT = 1.66053906660e-27
DEUTERIUM_MASS = 2.01410177812 * ATOMIC_MASS_UNIT


@dataclass(frozen=True)
class Grid1D:
    nc: int
    length_m: float
    dx_m: float

    def __post_init__(self):
        if self.nc < 2:
            raise ValueError(f"nc must be >= 2, got {self.nc}")
        if self.dx_m <= 0.0:
            raise ValueError("dx_m must be positive")
        if abs(self.dx_m * self.nc - self.length_m) > 1e-12 * abs(self.length_m):
            raise ValueError("inconsistent grid: dx_m*nc != length_m")

    @classmethod
    def from_cells(cls, nc: int, length_m: float) -> "Grid1D":
        return cls(nc=nc, length_m=length_m, dx_m=length_m / nc)


@dataclass(frozen=True)
class SpeciesDef:
    name: str
    charge_c: float
    mass_kg: float
    nstep: int = 1
    active_mover: bool = True
    track_transverse: bool = False
    charged: bool = field(default=None)

    def __post_init__(self):
        if self.charged is None:
            object.__setattr__(self, "charged", self.charge_c != 0.0)
        if self.mass_kg <= 0.0:
            raise ValueError(f"species {self.name!r}: mass_kg must be positive")
        if self.nstep < 1:
            raise ValueError(f"species {self.name!r}: nstep must be >= 1")
        if self.charged != (self.charge_c != 0.0):
            raise ValueError(f"species {self.name!r}: charged flag contradicts charge_c")


@dataclass(frozen=True)
class PhysicalConstants:
    dt_s: float
    epsilon0: float = EPSILON_0

    def __post_init__(self):
        if self.epsilon0 <= 0.0 or self.dt_s <= 0.0:
            raise ValueError("epsilon0 and dt_s must be positive")


def velocity_kick_coef(sp, consts, dx_m: float) -> float:
    """q dt^2 / (m dx), same association as pkg/src/picmc/mover.py:38-40."""
    return sp.charge_c * consts.dt_s * consts.dt_s / (sp.mass_kg * dx_m)


def thermal_std(t_ev: float, mass_kg: float, dt_s: float, dx_m: float) -> float:
    """Velocity spread in grid units (pkg/src/picmc/core.py:334-336)."""
    return math.sqrt(t_ev * ELEMENTARY_CHARGE / mass_kg) * (dt_s / dx_m)


@dataclass
class FlatSpecies:
    """Host copy of one species in the engine's flat layout (cell-major)."""

    x: np.ndarray
    vx: np.ndarray
    vy: np.ndarray
    vz: np.ndarray
    yp: np.ndarray  # None unless track_transverse
    cell: np.ndarray  # int32

    @property
    def n(self) -> int:
        return int(self.x.shape[0])

    def fields(self) -> dict:
        out = {"x": self.x, "vx": self.vx, "vy": self.vy, "vz": self.vz}
        if self.yp is not None:
            out["yp"] = self.yp
        return out


def init_species_host(config, isp: int, cell_lo: int = 0, cell_hi: int = None) -> FlatSpecies:
    """Host plasma loading for cells [cell_lo, cell_hi) of one species.

    Bit-for-bit the reference's init_plasma (pkg/src/picmc/core.py:319-351):
    same splitmix64 streams, same NumPy Box-Muller expressions, emitted in
    live (cell-major, slot) order.
    """
    grid = config.grid
    if cell_hi is None:
        cell_hi = grid.nc
    ppc0 = int(config.ppc0)
    sp = config.species[isp]
    cells = np.arange(cell_lo, cell_hi, dtype=np.int64)
    nloc = cell_hi - cell_lo
    slot = np.tile(np.arange(ppc0, dtype=np.int64), nloc)
    key = stream(config.seed, STREAM_INIT, isp)
    pkeys = np.repeat(derive_vec(np.uint64(key), cells), ppc0)
    x = uniforms(pkeys, slot)
    base = ppc0 + 4 * slot
    std = thermal_std(config.temperatures_ev[isp], sp.mass_kg, config.consts.dt_s, grid.dx_m)
    r1 = np.sqrt(-2.0 * np.log(uniforms_open(pkeys, base)))
    a1 = (2.0 * math.pi) * uniforms(pkeys, base + 1)
    r2 = np.sqrt(-2.0 * np.log(uniforms_open(pkeys, base + 2)))
    a2 = (2.0 * math.pi) * uniforms(pkeys, base + 3)
    return FlatSpecies(
        x=x,
        vx=std * (r1 * np.cos(a1)),
        vy=std * (r1 * np.sin(a1)),
        vz=std * (r2 * np.cos(a2)),
        yp=np.zeros(nloc * ppc0) if sp.track_transverse else None,
        cell=np.repeat(cells.astype(np.int32), ppc0),
    )


def macro_weight(config, isp: int) -> float:
    """Macro-particle weight n*dx/ppc0 (pkg/src/picmc/core.py:324)."""
    return config.densities_m3[isp] * config.grid.dx_m / config.ppc0


def check_store_budget(config, nfields_extra: int = 0):
    """Mirror of the reference allocation guard (core.py:307-317), applied to
    the device layout (no slack: 8 B per field plus a 4 B cell index)."""
    budget = config.max_store_mb * 1024 * 1024
    running = 0
    for sp in config.species:
        nf = 4 + (1 if sp.track_transverse else 0) + nfields_extra
        running += config.grid.nc * config.ppc0 * (nf * 8 + 4)
        if running > budget:
            raise InitError(
                f"species {sp.name!r}: initial allocation exceeds the "
                f"{config.max_store_mb} MB store cap"
            )
