"""The reference's mover API on the GPU (twin of pkg/src/picmc/mover.py).

Same functions, arguments, return values and exceptions as
pkg/src/picmc/mover.py:38-291, over a cell-segmented store: this package's
device `CellSortedStore` (cellstore.py; CUDA tensors, nothing crosses PCIe)
or the reference's own numpy store (arrays staged to the GPU and written
back).  Every per-particle operation runs in libpicmc_b200.so:

  push_velocity      pb_push_velocity                 (mover.py:43-54)
  push_position      pb_fused_move without accel      (mover.py:57-70)
  resort_collect     pb_resort_count + pb_resort_collect (mover.py:113-182)
  commit_incomers    stable device sort + pb_commit_place (mover.py:185-195)
  submit_move_tasks / mover_phase: one pb_fused_move launch per species
                     instead of per `grainsize` cell block (mover.py:227-291);
                     bitwise the same, since particles are independent.

Results are bitwise the reference's, slot order included (tests/test_mover_api_gpu.py).
The production step engine (engine.py) fuses all of this into one mover
launch on a flat layout; this module is the store-level drop-in.
"""

import ctypes
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, backend
from .core import velocity_kick_coef
from .errors import CflViolation, ContractViolation

__all__ = [
    "Movers",
    "accel_nodes_for_species",
    "commit_incomers",
    "mover_phase",
    "push_position",
    "push_velocity",
    "resort",
    "resort_collect",
    "submit_move_tasks",
    "velocity_kick_coef",
]


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("the mover API runs on a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class _View:
    """Device view of one species of a store (device tensors in place, or
    numpy arrays staged and, with writeback, copied back by flush())."""

    def __init__(self, store, isp, writeback: bool):
        self.dev = _dev()
        data = store.data(isp)
        self.names = tuple(store.field_names(isp)) if hasattr(store, "field_names") else tuple(data)
        self.host = not isinstance(data[self.names[0]], torch.Tensor)
        self.writeback = writeback and self.host
        self._back = []
        self.fields = {n: self._put(data[n], writeback) for n in self.names}
        self.offs = self._put(store.offsets(isp), False)
        self.counts = self._put(store.counts(isp), writeback)

    def _put(self, a, writeback):
        if isinstance(a, torch.Tensor):
            return a
        t = torch.from_numpy(np.ascontiguousarray(a)).to(self.dev)
        if writeback:
            self._back.append((a, t))
        return t

    def cell_fields(self) -> _lib.PbCellFields:
        c = _lib.PbCellFields()
        for f, n in enumerate(self.names):
            c.field[f] = self.fields[n].data_ptr()
        c.nf = len(self.names)
        c.offs = self.offs.data_ptr()
        c.counts = self.counts.data_ptr()
        c.nc = int(self.counts.numel())
        return c

    def flush(self):
        if self._back:
            torch.cuda.current_stream(self.dev).synchronize()
            for host, t in self._back:
                host[...] = t.cpu().numpy()


@dataclass
class Movers:
    """Particles stripped from their source cells, awaiting insertion
    (mover.py:74-110): aligned dest_cell / src_cell / src_slot (global,
    ascending (src_cell, src_slot) as collected) and per-field values with x
    already normalised to the destination cell.  Arrays are numpy for a
    numpy store, CUDA tensors for a device store."""

    isp: int
    dest_cell: object
    src_cell: object
    src_slot: object
    fields: dict

    @property
    def count(self) -> int:
        return len(self.dest_cell)

    @classmethod
    def empty(cls, isp: int, names, device=None) -> "Movers":
        if device is None:
            z = np.empty(0, dtype=np.int64)
            return cls(isp, z, z.copy(), z.copy(), {n: np.empty(0) for n in names})
        z = torch.empty(0, dtype=torch.int64, device=device)
        return cls(isp, z, z.clone(), z.clone(),
                   {n: torch.empty(0, dtype=torch.float64, device=device) for n in names})

    @classmethod
    def concat(cls, parts) -> "Movers":
        parts = list(parts)
        first = parts[0]
        cat = torch.cat if isinstance(first.dest_cell, torch.Tensor) else np.concatenate
        return cls(first.isp, cat([p.dest_cell for p in parts]), cat([p.src_cell for p in parts]),
                   cat([p.src_slot for p in parts]),
                   {n: cat([p.fields[n] for p in parts]) for n in first.fields})


def push_velocity(store, isp: int, e_p, consts):
    """vx += (q/m) E_p dt in grid units; E_p aligned with live order."""
    sp = store.species[isp]
    if not sp.charged:
        raise ContractViolation(f"push_velocity called on neutral species {sp.name!r}")
    lib = _lib.load()
    v = _View(store, isp, writeback=False)
    total = int(v.counts.sum().item())
    if total != len(e_p):
        raise ContractViolation("E_p length does not match live particle count")
    coef = velocity_kick_coef(sp, consts, store.grid.dx_m)
    vx = store.data(isp)["vx"]
    vxd = v.fields["vx"]
    ep = e_p if isinstance(e_p, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(e_p, dtype=np.float64)).to(v.dev)
    nc = int(v.counts.numel())
    scratch = torch.empty(lib.pb_cs_scratch_bytes(nc), dtype=torch.uint8, device=v.dev)
    _lib.check(lib.pb_push_velocity(ep.data_ptr(), coef, vxd.data_ptr(), v.offs.data_ptr(),
                                    v.counts.data_ptr(), nc, scratch.data_ptr(), scratch.numel(),
                                    _stream()), "push_velocity")
    if v.host:
        torch.cuda.current_stream(v.dev).synchronize()
        vx[...] = vxd.cpu().numpy()


def push_position(store, isp: int):
    """x += nstep * vx (and yp += nstep * vy when tracked); no wrap yet."""
    sp = store.species[isp]
    data = store.data(isp)
    backend.fused_move(None, data["x"], data["vx"], data["vy"], data.get("yp"),
                       store.offsets(isp), store.counts(isp), float(sp.nstep))


def resort_collect(store, lo: int = 0, hi: int = None, nc_global: int = None) -> list:
    """Strip out-of-range particles from every cell of a store.

    Survivors are compacted in slot order; vacated slots are zeroed. Returns
    one Movers per species with destinations wrapped into [0, nc_global).
    `lo` is the store's global offset when the store covers a subdomain.
    Raises CflViolation (nothing modified) if a displacement reaches across
    the whole domain."""
    lib = _lib.load()
    if nc_global is None:
        nc_global = store.grid.nc
    out = []
    for isp, sp in enumerate(store.species):
        v = _View(store, isp, writeback=True)
        dev = None if v.host else v.dev
        nc = int(v.counts.numel())
        mc = torch.empty(nc + 1, dtype=torch.int64, device=v.dev)
        base = torch.empty(nc + 1, dtype=torch.int64, device=v.dev)
        cfl = torch.empty(1, dtype=torch.int64, device=v.dev)
        scratch = torch.empty(lib.pb_cs_scratch_bytes(nc), dtype=torch.uint8, device=v.dev)
        _lib.check(lib.pb_resort_count(v.fields["x"].data_ptr(), v.offs.data_ptr(), v.counts.data_ptr(),
                                       nc, int(nc_global), mc.data_ptr(), base.data_ptr(), cfl.data_ptr(),
                                       scratch.data_ptr(), scratch.numel(), _stream()), "resort_count")
        total, bad = (int(t) for t in torch.stack([base[nc], cfl[0]]).tolist())
        if bad != -1:  # UINT64_MAX: no offender
            cell = int(torch.searchsorted(v.offs, torch.tensor([bad], device=v.dev), right=True).item()) - 1
            delta = float(np.floor(float(v.fields["x"][bad].item())))
            raise CflViolation(f"species {sp.name!r} cell {cell + lo}: displacement of "
                               f"{int(delta)} cells reaches across the whole domain")
        if total == 0:
            out.append(Movers.empty(isp, v.names, dev))
            continue
        m = _lib.PbMovers()
        mv = {n: torch.empty(total, dtype=torch.float64, device=v.dev) for n in v.names}
        dest, src_cell, src_slot = (torch.empty(total, dtype=torch.int64, device=v.dev) for _ in range(3))
        for f, n in enumerate(v.names):
            m.field[f] = mv[n].data_ptr()
        m.dest, m.src_cell, m.src_slot = dest.data_ptr(), src_cell.data_ptr(), src_slot.data_ptr()
        cf = v.cell_fields()
        _lib.check(lib.pb_resort_collect(ctypes.byref(cf), ctypes.byref(m), int(lo), int(nc_global),
                                         base.data_ptr(), _stream()), "resort_collect")
        v.flush()
        if v.host:
            out.append(Movers(isp, dest.cpu().numpy(), src_cell.cpu().numpy(), src_slot.cpu().numpy(),
                              {n: t.cpu().numpy() for n, t in mv.items()}))
        else:
            out.append(Movers(isp, dest, src_cell, src_slot, mv))
    return out


def _stable_order(*keys):
    """lexsort with the last key primary (np.lexsort convention), on device."""
    order = None
    for k in keys:
        kk = k if order is None else k[order]
        o = torch.sort(kk, stable=True).indices
        order = o if order is None else order[o]
    return order


def commit_incomers(store, movers: Movers, lo: int = 0):
    """Append incomers, per destination cell in (src_cell, src_slot) order."""
    if movers.count == 0:
        return
    lib = _lib.load()
    dev = _dev()
    isp = movers.isp
    put = lambda a: a if isinstance(a, torch.Tensor) else torch.from_numpy(  # noqa: E731
        np.ascontiguousarray(a)).to(dev)
    dest, src_cell, src_slot = put(movers.dest_cell), put(movers.src_cell), put(movers.src_slot)
    order = _stable_order(src_slot, src_cell, dest)
    local = dest - lo
    nc = int(store.counts(isp).shape[0])
    incoming = torch.bincount(local, minlength=nc)
    first = torch.cumsum(incoming, 0) - incoming
    rank = torch.arange(movers.count, device=dev) - first[local[order]]
    # capacity first, with the reference's doubling rule (append -> _grow)
    if hasattr(store, "reserve_all"):
        store.reserve_all(isp, incoming)
    else:
        counts, caps = np.asarray(store.counts(isp)), np.asarray(store.caps(isp))
        inc = incoming.cpu().numpy()
        for j in np.nonzero(counts + inc > caps)[0]:
            store.reserve(isp, int(j), int(inc[j]))
    v = _View(store, isp, writeback=True)
    m = _lib.PbMovers()
    mf = [put(movers.fields[n]) for n in v.names]
    for f, t in enumerate(mf):
        m.field[f] = t.data_ptr()
    m.dest = dest.data_ptr()
    cf = v.cell_fields()
    _lib.check(lib.pb_commit_place(ctypes.byref(cf), ctypes.byref(m), order.data_ptr(), rank.data_ptr(),
                                   movers.count, int(lo), _stream()), "commit_incomers")
    v.counts += incoming
    v.flush()


def resort(store, grid=None) -> int:
    """Move every out-of-range particle to its destination cell (global
    periodic wrap).  Returns the number of transferred particles."""
    moved = 0
    for movers in resort_collect(store):
        moved += movers.count
        commit_incomers(store, movers)
    return moved


def accel_nodes_for_species(store, e_field, consts) -> list:
    """Premultiplied node acceleration a[] = (q dt^2 / m dx) * E per species;
    None for species that get no kick (neutral or inactive), so the kernels
    skip the gather rather than add 0.0 to -0.0 velocities."""
    out = []
    for sp in store.species:
        if sp.charged and sp.active_mover:
            out.append(velocity_kick_coef(sp, consts, store.grid.dx_m) * e_field)
        else:
            out.append(None)
    return out


def submit_move_tasks(scheduler, store, accel: list, grainsize: int, queue_offset: int = 0,
                      tag: str = "move"):
    """Fused-move work for every active species; no wait.  One device launch
    per species on queue (species index mod 4) + queue_offset (`grainsize`
    is accepted for signature compatibility: the launch covers every cell).
    scheduler None runs the launches inline.  Returns the set of queues."""
    queues = set()
    for isp, sp in enumerate(store.species):
        if not sp.active_mover:
            continue
        data = store.data(isp)
        queue = queue_offset + (isp % 4)
        queues.add(queue)

        def body(isp=isp, a_sp=accel[isp], fnstep=float(sp.nstep), data=data):
            backend.fused_move(a_sp, data["x"], data["vx"], data["vy"], data.get("yp"),
                               store.offsets(isp), store.counts(isp), fnstep)

        if scheduler is None:
            body()
        else:
            scheduler.submit_work(body, queue=queue, tag=f"{tag}:{sp.name}")
    return queues


def mover_phase(store, e_field, consts, scheduler=None, grainsize: int = 500) -> float:
    """Gather + velocity push + position push for all species; returns the
    elapsed seconds (device work included)."""
    t0 = time.perf_counter()
    accel = accel_nodes_for_species(store, e_field, consts)
    queues = submit_move_tasks(scheduler, store, accel, grainsize)
    if scheduler is not None:
        scheduler.wait(sorted(queues))
    torch.cuda.synchronize()
    return time.perf_counter() - t0
