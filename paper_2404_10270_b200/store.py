"""Device particle store: one flat structure of arrays per species.

Replaces the reference's CellSortedStore (pkg/src/picmc/core.py:100-264).
Per species, fp64 arrays x, vx, vy, vz[, yp] and an int32 cell index live in
HBM at their final size; there is no per-cell slack and therefore no
capacity growth (core.py:220-240).  Positions stay cell-relative in [0,1)
exactly as in the reference, which is what makes per-particle results
bitwise identical (a global coordinate would lose ~20 bits at nc=1M).
Cell order is restored by a periodic radix sort (pb_sort_by_cell) into
ping-pong buffers.
"""

import ctypes

import numpy as np
import torch

from . import _lib
from .core import FlatSpecies

F64 = torch.float64


class DeviceSpecies:
    """SoA arrays of one species on one GPU."""

    FIELDS = ("x", "vx", "vy", "vz")

    def __init__(self, sp, n: int, device, *, kind: int, deposit: int,
                 kick_coef: float = 0.0, boris=None, absorbing: bool = False, cap: int = None,
                 cell8: bool = False, b_nodes=None, boris_f: float = 0.0):
        self.sp = sp
        self.name = sp.name
        self.device = device
        self.n = int(n)
        self.kind = int(kind)
        self.deposit = int(deposit)
        self.fnstep = float(sp.nstep)
        self.kick_coef = float(kick_coef)
        self.boris = boris  # (t[3], s[3]) or None
        # spatially varying B: (nc+1, 4) f64 device nodes shared by the
        # engine's Boris species, and f = q dt / (2 m) (pb_species.b_nodes)
        self.b_nodes = b_nodes
        self.boris_f = float(boris_f)
        self.absorbing = absorbing
        self.has_yp = bool(sp.track_transverse)
        # cap > n leaves room for collision newborns (canonical mode).
        self.cap = max(int(cap) if cap is not None else self.n, self.n)
        alloc = max(self.cap, 1)
        self.arr = {f: torch.empty(alloc, dtype=F64, device=device) for f in self.FIELDS}
        if self.has_yp:
            self.arr["yp"] = torch.empty(alloc, dtype=F64, device=device)
        self.cell = torch.empty(alloc, dtype=torch.int32, device=device)
        # compressed cell index for the production mover (pb_species.cell8)
        self.cell8 = torch.empty(alloc, dtype=torch.int8, device=device) if cell8 else None
        nchunk = (alloc + _lib.PB_CELL8_CHUNK - 1) // _lib.PB_CELL8_CHUNK
        self.chunk_base = torch.empty(nchunk, dtype=torch.int32, device=device) if cell8 else None
        self.n_dev = torch.full((1,), self.n, dtype=torch.int64, device=device)
        self.holes = torch.empty(alloc if absorbing else 1, dtype=torch.int64, device=device)
        self._spare = None  # ping-pong buffers for the cell sort

    # -- host <-> device ----------------------------------------------------
    def upload(self, flat: FlatSpecies):
        if flat.n != self.n:
            raise ValueError(f"species {self.name!r}: expected {self.n} particles, got {flat.n}")
        for name, arr in flat.fields().items():
            self.arr[name][: self.n].copy_(torch.from_numpy(np.ascontiguousarray(arr)))
        self.cell[: self.n].copy_(torch.from_numpy(np.ascontiguousarray(flat.cell, dtype=np.int32)))
        self.n_dev.fill_(self.n)

    def live_count(self) -> int:
        return int(self.n_dev.item()) if self.absorbing else self.n

    def download(self) -> FlatSpecies:
        n = self.live_count()
        get = lambda t: t[:n].cpu().numpy().copy()  # noqa: E731
        return FlatSpecies(
            x=get(self.arr["x"]), vx=get(self.arr["vx"]), vy=get(self.arr["vy"]),
            vz=get(self.arr["vz"]), yp=get(self.arr["yp"]) if self.has_yp else None,
            cell=get(self.cell),
        )

    # -- C ABI view ---------------------------------------------------------
    def pb(self, n_host: int = None) -> _lib.PbSpecies:
        s = _lib.PbSpecies()
        s.x = self.arr["x"].data_ptr()
        s.vx = self.arr["vx"].data_ptr()
        s.vy = self.arr["vy"].data_ptr()
        s.vz = self.arr["vz"].data_ptr()
        s.yp = self.arr["yp"].data_ptr() if self.has_yp else None
        s.cell = self.cell.data_ptr()
        s.n_dev = self.n_dev.data_ptr() if self.absorbing else None
        s.n = self.n if n_host is None else n_host
        s.holes = self.holes.data_ptr() if self.absorbing else None
        s.kind = self.kind
        s.deposit = self.deposit
        s.fnstep = self.fnstep
        s.kick_coef = self.kick_coef
        if self.boris is not None:
            t, sv = self.boris
            for k in range(3):
                s.boris_t[k] = t[k]
                s.boris_s[k] = sv[k]
        if self.b_nodes is not None and self.kind == _lib.PB_KIND_BORIS:
            s.b_nodes = self.b_nodes.data_ptr()
            s.boris_f = self.boris_f
        if self.cell8 is not None:
            s.cell8 = self.cell8.data_ptr()
            s.chunk_base = self.chunk_base.data_ptr()
        return s

    def ensure_capacity(self, need: int):
        """Grow the arrays (keeping slots [0, n)) so `need` slots fit; the
        ping-pong spare is dropped and recreated on demand."""
        if need <= self.cap:
            return
        cap = max(int(need), int(self.cap * 1.25) + 1)
        for f, t in list(self.arr.items()):
            new = torch.empty(cap, dtype=t.dtype, device=t.device)
            new[: self.n].copy_(t[: self.n])
            self.arr[f] = new
        cell = torch.empty(cap, dtype=self.cell.dtype, device=self.cell.device)
        cell[: self.n].copy_(self.cell[: self.n])
        self.cell = cell
        if self.cell8 is not None:
            raise RuntimeError("ensure_capacity: cell8 species are fixed-size")
        if self.absorbing:
            self.holes = torch.empty(cap, dtype=torch.int64, device=self.cell.device)
        self.cap = cap
        self._spare = None

    def spare(self) -> "DeviceSpecies":
        """Second buffer set, same shape, for the ping-pong cell sort."""
        if self._spare is None:
            other = object.__new__(DeviceSpecies)
            other.__dict__.update(self.__dict__)
            other.arr = {k: torch.empty_like(v) for k, v in self.arr.items()}
            other.cell = torch.empty_like(self.cell)
            if self.cell8 is not None:
                other.cell8 = torch.empty_like(self.cell8)
                other.chunk_base = torch.empty_like(self.chunk_base)
            other._spare = None
            self._spare = other
        return self._spare

    def swap_with_spare(self):
        sp = self._spare
        self.arr, sp.arr = sp.arr, self.arr
        self.cell, sp.cell = sp.cell, self.cell
        self.cell8, sp.cell8 = sp.cell8, self.cell8
        self.chunk_base, sp.chunk_base = sp.chunk_base, self.chunk_base


def species_array(species: list, n_host=None):
    arr = (_lib.PbSpecies * max(len(species), 1))()
    for k, s in enumerate(species):
        arr[k] = s.pb(None if n_host is None else n_host[k])
    return arr, len(species)


def status_template(device) -> torch.Tensor:
    """Zeroed pb_status with cfl_index = mover_t0 = UINT64_MAX, as raw bytes on device."""
    st = _lib.PbStatus()
    st.cfl_index = (1 << 64) - 1
    st.mover_t0 = (1 << 64) - 1
    raw = bytes(ctypes.string_at(ctypes.addressof(st), _lib.STATUS_BYTES))
    return torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(device)


def decode_status(raw: np.ndarray) -> _lib.PbStatus:
    st = _lib.PbStatus()
    ctypes.memmove(ctypes.addressof(st), raw.ctypes.data, _lib.STATUS_BYTES)
    return st
