"""Device-resident twin of the reference's cell-segmented particle store.

`CellSortedStore` follows pkg/src/picmc/core.py:100-264 -- per species,
packed float64 field arrays x, vx, vy, vz[, yp] addressed by per-cell
(offset, count, capacity) int64 triples, live slots [off[j], off[j]+count[j]),
free space kept zeroed, capacity doubling per cell on overflow -- with every
array a CUDA tensor.  It is the data format the reference's mover API
(mover.py, backends) works on; `paper_2404_10270_b200.mover` runs that API on
the GPU against this store or against the reference's own numpy store.

The production engine does not use this layout (engine.py keeps a flat SoA
with a per-particle cell index); the twin exists so that
store-level callers and the reference's store-level tests have a drop-in.
"""

import ctypes

import numpy as np
import torch

from . import _lib
from .errors import ContractViolation

BASE_FIELDS = ("x", "vx", "vy", "vz")
F64, I64 = torch.float64, torch.int64


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _offsets_from(caps: torch.Tensor) -> torch.Tensor:
    offs = torch.zeros_like(caps)
    if caps.numel() > 1:
        torch.cumsum(caps[:-1], 0, out=offs[1:])
    return offs


def grown_caps(caps: torch.Tensor, need: torch.Tensor) -> torch.Tensor:
    """Capacities after appending up to `need` particles per cell with the
    reference's rule (append grows a full cell to max(2*cap, 4), core.py:192-240)."""
    caps = caps.clone()
    while True:
        short = need > caps
        if not bool(short.any()):
            return caps
        caps = torch.where(short, torch.clamp(2 * caps, min=4), caps)


class CellSortedStore:
    """Cell-sorted storage for a species list on one grid, in HBM."""

    def __init__(self, grid, species, initial_cap: int = 4, device=None):
        if not torch.cuda.is_available():
            raise RuntimeError("CellSortedStore lives on a CUDA device; there is no CPU fallback")
        self.device = torch.device(device if device is not None else f"cuda:{torch.cuda.current_device()}")
        self.grid = grid
        self.species = list(species)
        self.weights = [1.0] * len(self.species)
        nc = grid.nc
        cap0 = max(int(initial_cap), 1)
        self._counts, self._caps, self._offs, self._data = [], [], [], []
        for sp in self.species:
            caps = torch.full((nc,), cap0, dtype=I64, device=self.device)
            self._caps.append(caps)
            self._offs.append(_offsets_from(caps))
            self._counts.append(torch.zeros(nc, dtype=I64, device=self.device))
            names = BASE_FIELDS + (("yp",) if sp.track_transverse else ())
            self._data.append({k: torch.zeros(cap0 * nc, dtype=F64, device=self.device) for k in names})

    # -- accessors (core.py:141-190) -----------------------------------------
    @property
    def nsp(self) -> int:
        return len(self.species)

    def counts(self, isp: int) -> torch.Tensor:
        return self._counts[isp]

    def offsets(self, isp: int) -> torch.Tensor:
        return self._offs[isp]

    def caps(self, isp: int) -> torch.Tensor:
        return self._caps[isp]

    def data(self, isp: int) -> dict:
        return self._data[isp]

    def field_names(self, isp: int) -> tuple:
        return tuple(self._data[isp].keys())

    def total(self, isp: int) -> int:
        return int(self._counts[isp].sum().item())

    def cell_slice(self, isp: int, j: int) -> slice:
        off = int(self._offs[isp][j].item())
        return slice(off, off + int(self._counts[isp][j].item()))

    def live_indices(self, isp: int, lo: int = 0, hi: int = None) -> torch.Tensor:
        """Packed-array indices of the live slots of cells [lo, hi), cell-major."""
        hi = self.grid.nc if hi is None else hi
        counts = self._counts[isp][lo:hi]
        offs = self._offs[isp][lo:hi]
        n = int(counts.sum().item())
        if n == 0:
            return torch.empty(0, dtype=I64, device=self.device)
        first = torch.cumsum(counts, 0) - counts
        cell = torch.repeat_interleave(torch.arange(counts.numel(), device=self.device), counts,
                                       output_size=n)
        return offs[cell] + torch.arange(n, device=self.device) - first[cell]

    def cell_of_live(self, isp: int, lo: int = 0, hi: int = None) -> torch.Tensor:
        hi = self.grid.nc if hi is None else hi
        counts = self._counts[isp][lo:hi]
        return torch.repeat_interleave(torch.arange(lo, hi, dtype=I64, device=self.device), counts)

    # -- mutation ------------------------------------------------------------
    def append(self, isp: int, j: int, record: dict) -> int:
        """Insert one particle into cell j; returns its slot index."""
        if int(self._counts[isp][j].item()) == int(self._caps[isp][j].item()):
            self._grow(isp, j)
        slot = int(self._counts[isp][j].item())
        base = int(self._offs[isp][j].item())
        for name, arr in self._data[isp].items():
            arr[base + slot] = float(record.get(name, 0.0))
        self._counts[isp][j] += 1
        return slot

    def swap_remove(self, isp: int, j: int, slot: int) -> dict:
        """Remove the particle at (j, slot), filling the hole from the end."""
        count = int(self._counts[isp][j].item())
        if not 0 <= slot < count:
            raise IndexError(f"slot {slot} out of range for cell {j} ({count})")
        base = int(self._offs[isp][j].item())
        last = base + count - 1
        record = {}
        for name, arr in self._data[isp].items():
            record[name] = float(arr[base + slot].item())
            arr[base + slot] = arr[last]
            arr[last] = 0.0
        self._counts[isp][j] -= 1
        return record

    def _grow(self, isp: int, j: int):
        """Double cell j's capacity (core.py:220-240)."""
        caps = self._caps[isp].clone()
        caps[j] = max(2 * int(caps[j].item()), 4)
        self.set_caps(isp, caps)

    def reserve(self, isp: int, j: int, extra: int):
        """Ensure cell j can take `extra` more particles without growing."""
        need = self._counts[isp].clone()
        need[j] += int(extra)
        self.set_caps(isp, grown_caps(self._caps[isp], need))

    def reserve_all(self, isp: int, extra: torch.Tensor):
        """Vectorised reserve: room for extra[j] more particles in every cell j."""
        self.set_caps(isp, grown_caps(self._caps[isp], self._counts[isp] + extra))

    def set_caps(self, isp: int, caps: torch.Tensor):
        """Re-lay species isp out with per-cell capacities `caps` (live
        segments moved, free space zero) -- one repack launch per field."""
        if torch.equal(caps, self._caps[isp]):
            return
        if bool((caps < self._counts[isp]).any()):
            raise ValueError("set_caps: capacity below the live count")
        lib = _lib.load()
        offs_new = _offsets_from(caps)
        total = int(caps.sum().item())
        nc = self.grid.nc
        new = {}
        for name, arr in self._data[isp].items():
            dst = torch.zeros(total, dtype=F64, device=self.device)
            _lib.check(lib.pb_repack(arr.data_ptr(), dst.data_ptr(), self._offs[isp].data_ptr(),
                                     offs_new.data_ptr(), self._counts[isp].data_ptr(), nc, _stream()),
                       "pb_repack")
            new[name] = dst
        self._caps[isp], self._offs[isp], self._data[isp] = caps, offs_new, new

    def clone(self) -> "CellSortedStore":
        other = object.__new__(CellSortedStore)
        other.device, other.grid, other.species = self.device, self.grid, list(self.species)
        other.weights = list(self.weights)
        other._counts = [a.clone() for a in self._counts]
        other._caps = [a.clone() for a in self._caps]
        other._offs = [a.clone() for a in self._offs]
        other._data = [{k: v.clone() for k, v in d.items()} for d in self._data]
        return other

    def check_sorted(self, isp: int):
        """Raise unless every live x lies in [0, 1) (core.py:256-264)."""
        idx = self.live_indices(isp)
        if idx.numel():
            x = self._data[isp]["x"][idx]
            if bool(((x < 0.0) | (x >= 1.0)).any()):
                raise ContractViolation(
                    f"store not resorted: species {self.species[isp].name!r} has positions outside [0,1)")

    # -- conversions ----------------------------------------------------------
    @classmethod
    def from_host(cls, grid, species, counts, caps, data, device=None) -> "CellSortedStore":
        """From per-species host arrays (e.g. a reference store's counts(),
        caps(), data()); slot layout preserved."""
        s = cls(grid, species, initial_cap=1, device=device)
        for isp in range(len(species)):
            c = torch.as_tensor(np.asarray(caps[isp], dtype=np.int64), device=s.device)
            s._caps[isp] = c
            s._offs[isp] = _offsets_from(c)
            s._counts[isp] = torch.as_tensor(np.asarray(counts[isp], dtype=np.int64), device=s.device)
            s._data[isp] = {k: torch.as_tensor(np.asarray(v, dtype=np.float64), device=s.device).clone()
                            for k, v in data[isp].items()}
        return s

    def to_host(self, isp: int) -> dict:
        """counts / caps / offsets and every field of species isp as numpy."""
        out = {"counts": self._counts[isp].cpu().numpy(), "caps": self._caps[isp].cpu().numpy(),
               "offsets": self._offs[isp].cpu().numpy()}
        out.update({k: v.cpu().numpy() for k, v in self._data[isp].items()})
        return out
