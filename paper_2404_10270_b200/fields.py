"""The reference's field pipeline API on the GPU (twin of pkg/src/picmc/fields.py).

Same functions, arguments, results and exceptions as
pkg/src/picmc/fields.py:32-236, every array operation in libpicmc_b200.so:

  deposit_partials_range  pb_deposit_partials per charged species +
                          pb_rho_from_partials (species-order weighting)
  stitch_rho              pb_stitch_rho
  deposit_charge          check_sorted + pb_deposit_partials + pb_rho_from_partials
                          (stitch and doubled wall nodes)
  smooth_density          pb_smooth_density
  solve_poisson           pb_solve_poisson (the serial elimination, bitwise)
  compute_efield          pb_compute_efield
  gather_field            pb_gather per species

Arrays may be NumPy (staged to the GPU; NumPy results) or CUDA tensors
(used in place; tensor results).  Stores: this package's device
`cellstore.CellSortedStore` or the reference's numpy store.  The step engine
(engine.py) runs the same kernels on device-resident buffers.
"""

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, backend
from .errors import ContractViolation

__all__ = [
    "FieldState",
    "compute_efield",
    "deposit_charge",
    "deposit_partials_range",
    "gather_field",
    "smooth_density",
    "solve_poisson",
    "stitch_rho",
]


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("the field API runs on a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _in(a, dev):
    """(device float64 tensor, came_from_numpy)."""
    if isinstance(a, torch.Tensor):
        if not a.is_cuda:
            return a.to(dev, torch.float64).contiguous(), True
        return a.to(torch.float64).contiguous(), False
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev), True


def _out(t, host: bool):
    if host:
        return t.cpu().numpy()
    return t


def _field_bc(bc: str) -> int:
    if bc == "periodic":
        return _lib.PB_FIELD_PERIODIC
    if bc == "dirichlet":
        return _lib.PB_FIELD_DIRICHLET
    raise ValueError(f"unknown boundary condition {bc!r}")


@dataclass
class FieldState:
    """Charge density (C/m^3), potential (V), and field (V/m) on the nodes."""

    rho: object
    phi: object
    e_field: object
    rho_mean_subtracted: float = 0.0

    def __post_init__(self):
        n = len(self.rho)
        if len(self.phi) != n or len(self.e_field) != n:
            raise ValueError("rho, phi and e_field must share length nc+1")

    @classmethod
    def zeros(cls, nc: int, device=None) -> "FieldState":
        if device is None:
            return cls(rho=np.zeros(nc + 1), phi=np.zeros(nc + 1), e_field=np.zeros(nc + 1))
        z = lambda: torch.zeros(nc + 1, dtype=torch.float64, device=device)  # noqa: E731
        return cls(rho=z(), phi=z(), e_field=z())


def _partials(store, lo, hi, dev, field_bc):
    """Weighted L/R over cells [lo, hi) and their stitched rho (with the
    deposit_charge wall doubling for Dirichlet)."""
    lib = _lib.load()
    n = hi - lo
    dx = store.grid.dx_m
    raws, coefs = [], []
    host = not (store.species and isinstance(store.data(0)["x"], torch.Tensor))
    for isp, sp in enumerate(store.species):
        if not sp.charged:
            continue
        x = store.data(isp)["x"]
        offs, counts = store.offsets(isp)[lo:hi], store.counts(isp)[lo:hi]
        if not isinstance(x, torch.Tensor):
            offs, counts = np.ascontiguousarray(offs), np.ascontiguousarray(counts)
            x = torch.from_numpy(x).to(dev)
            offs, counts = torch.from_numpy(offs).to(dev), torch.from_numpy(counts).to(dev)
        left_raw, right_raw = backend.deposit_partials(x, offs.contiguous(), counts.contiguous())
        raws.append(torch.stack([left_raw, right_raw]))
        coefs.append(sp.charge_c * store.weights[isp] / dx)
    left = torch.empty(n, dtype=torch.float64, device=dev)
    right = torch.empty(n, dtype=torch.float64, device=dev)
    rho = torch.empty(n + 1, dtype=torch.float64, device=dev)
    raw = torch.stack(raws).contiguous() if raws else None
    c = (ctypes.c_double * max(len(coefs), 1))(*coefs)
    _lib.check(lib.pb_rho_from_partials(None if raw is None else raw.data_ptr(), c, len(coefs), n,
                                        field_bc, left.data_ptr(), right.data_ptr(), rho.data_ptr(),
                                        _stream()), "deposit_partials_range")
    return left, right, rho, host


def deposit_partials_range(store, consts, lo: int, hi: int):
    """Weighted per-cell CIC partial sums over cells [lo, hi): species in
    index order, slots sequential within a cell; neutrals contribute nothing."""
    left, right, _, host = _partials(store, lo, hi, _dev(), _lib.PB_FIELD_PERIODIC)
    return _out(left, host), _out(right, host)


def stitch_rho(left, right, periodic: bool):
    """Node densities from per-cell partials: rho[g] = R[g-1] + L[g]."""
    dev = _dev()
    lt, host = _in(left, dev)
    rt, _ = _in(right, dev)
    nc = int(lt.numel())
    rho = torch.empty(nc + 1, dtype=torch.float64, device=dev)
    _lib.check(_lib.load().pb_stitch_rho(lt.data_ptr(), rt.data_ptr(), nc, int(bool(periodic)),
                                         rho.data_ptr(), _stream()), "stitch_rho")
    return _out(rho, host)


def _check_sorted(store, isp, dev):
    if hasattr(store, "check_sorted") and isinstance(store.data(isp)["x"], torch.Tensor):
        store.check_sorted(isp)
        return
    counts = store.counts(isp)
    offs = store.offsets(isp)
    ct = torch.as_tensor(np.asarray(counts), device=dev)
    ot = torch.as_tensor(np.asarray(offs), device=dev)
    n = int(ct.sum().item())
    if n == 0:
        return
    x = torch.from_numpy(np.ascontiguousarray(store.data(isp)["x"])).to(dev)
    cell = torch.repeat_interleave(torch.arange(ct.numel(), device=dev), ct, output_size=n)
    idx = ot[cell] + torch.arange(n, device=dev) - (torch.cumsum(ct, 0) - ct)[cell]
    xs = x[idx]
    if bool(((xs < 0.0) | (xs >= 1.0)).any()):
        raise ContractViolation(f"store not resorted: species {store.species[isp].name!r} has "
                                "positions outside [0,1)")


def deposit_charge(store, grid, consts, bc: str = "periodic"):
    """Cloud-in-cell charge deposition onto the nodes (wall nodes doubled
    for non-periodic runs).  Raises ContractViolation if the store has
    positions outside [0,1)."""
    dev = _dev()
    for isp in range(len(store.species)):
        _check_sorted(store, isp, dev)
    fbc = _lib.PB_FIELD_PERIODIC if bc == "periodic" else _lib.PB_FIELD_DIRICHLET
    _, _, rho, host = _partials(store, 0, grid.nc, dev, fbc)
    return _out(rho, host)


def smooth_density(rho, passes: int = 1):
    """Binomial 1-2-1 filter with periodic wrap on nodes [0, nc)."""
    lib = _lib.load()
    dev = _dev()
    rt, host = _in(rho, dev)
    nc = int(rt.numel()) - 1
    out = torch.empty_like(rt)
    scratch = torch.empty(lib.pb_field_scratch_bytes(nc), dtype=torch.uint8, device=dev)
    _lib.check(lib.pb_smooth_density(rt.data_ptr(), out.data_ptr(), nc, int(passes), scratch.data_ptr(),
                                     _stream()), "smooth_density")
    return _out(out, host)


def solve_poisson(rho, grid, consts, bc: str = "periodic", phi_left: float = 0.0,
                  phi_right: float = 0.0):
    """Exact direct solve of phi'' = -rho/eps0 on the discrete nodes
    (periodic: neutralising background, gauge phi[0]=0, shifted to mean 0;
    Dirichlet: fixed end potentials)."""
    nc = grid.nc
    if nc < 3:
        raise ValueError(f"poisson solve needs nc >= 3, got {nc}")
    fbc = _field_bc(bc)
    lib = _lib.load()
    dev = _dev()
    rt, host = _in(rho, dev)
    phi = torch.empty(nc + 1, dtype=torch.float64, device=dev)
    scratch = torch.empty(lib.pb_field_scratch_bytes(nc), dtype=torch.uint8, device=dev)
    _lib.check(lib.pb_solve_poisson(rt.data_ptr(), phi.data_ptr(), nc, grid.dx_m, consts.epsilon0, fbc,
                                    float(phi_left), float(phi_right), scratch.data_ptr(), _stream()),
               "solve_poisson")
    return _out(phi, host)


def compute_efield(phi, grid, bc: str = "periodic"):
    """E = -grad(phi): central differences, one-sided at Dirichlet walls."""
    lib = _lib.load()
    dev = _dev()
    pt, host = _in(phi, dev)
    nc = grid.nc
    e = torch.empty(nc + 1, dtype=torch.float64, device=dev)
    fbc = _lib.PB_FIELD_PERIODIC if bc == "periodic" else _lib.PB_FIELD_DIRICHLET
    _lib.check(lib.pb_compute_efield(pt.data_ptr(), e.data_ptr(), nc, grid.dx_m, fbc, _stream()),
               "compute_efield")
    return _out(e, host)


def gather_field(e_field, store, grid) -> dict:
    """Per-particle E_p by one-sided CIC interpolation, per species, in live
    (cell-major, slot) order."""
    return {isp: backend.gather(e_field, store.data(isp)["x"], store.offsets(isp), store.counts(isp))
            for isp in range(len(store.species))}
