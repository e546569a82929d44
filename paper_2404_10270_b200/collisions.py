"""Monte Carlo electron-neutral collisions on the GPU.

Mirrors the reference module pkg/src/picmc/collisions.py: the same
`CollisionRates` / `CollisionTally` / `Roles` types, `step_stream_key`, and a
`collision_phase` that runs one collision pass over every cell of a store and
commits the newborns -- here on device-resident species in the reference's
canonical slot order, through the C ABI (`pb_collide` + an in-place
`pb_canonical_resort` that appends the newborns after each cell's live
slots, collisions.py:286-289).  Results are bitwise the reference's: same
splitmix64 streams per (step, cell, substep, slot), same event arithmetic,
same swap_remove of the ionized neutral, same commit order.

The run-level path is `CanonicalEngine` (canonical.py), which calls the same
two kernels every step.
"""

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from .config import CollisionRates  # noqa: F401  (re-export, collisions.py:47-66)
from .core import ELEMENTARY_CHARGE, FlatSpecies
from .harness import CollisionTally  # noqa: F401
from .rng import STREAM_COLLIDE, stream
from .store import DeviceSpecies, status_template

__all__ = ["CollisionRates", "CollisionTally", "Roles", "collision_phase", "step_stream_key"]


@dataclass(frozen=True)
class Roles:
    """Species indices playing the electron / neutral target / ion product
    (collisions.py:84-90)."""

    electron: int
    neutral: int
    ion: int


def step_stream_key(seed: int, step: int) -> int:
    """collisions.py:92-93."""
    return stream(seed, STREAM_COLLIDE, step)


def collision_params(rates, consts, dx_m: float, neutral_weight: float, electron_mass: float,
                     step_key: int, global_offset: int = 0) -> _lib.PbCollideParams:
    p = _lib.PbCollideParams()
    p.step_key = int(step_key)
    p.global_offset = int(global_offset)
    p.w_over_dx = neutral_weight / dx_m
    p.dt = consts.dt_s
    p.rate_elastic = rates.rate_elastic_m3s
    p.rate_excitation = rates.rate_excitation_m3s
    p.rate_ionization = rates.rate_ionization_m3s
    p.threshold_j = rates.excitation_threshold_ev * ELEMENTARY_CHARGE
    p.mass_e = electron_mass
    p.dx_over_dt = dx_m / consts.dt_s
    return p


def collision_phase(species: list, defs: list, weights: list, rates, consts, roles: Roles,
                    step_key: int, nc: int, dx_m: float, global_offset: int = 0, device=None):
    """One collision pass over cells [0, nc) of canonical host species
    (`FlatSpecies`, cell-major slot order) on the GPU; returns
    (CollisionTally, new species list) with newborns committed."""
    if not torch.cuda.is_available():
        raise RuntimeError("collision_phase needs a CUDA device; there is no CPU fallback")
    lib = _lib.load()
    dev = torch.device(device if device is not None else f"cuda:{torch.cuda.current_device()}")
    st = torch.cuda.Stream(dev)
    sh = ctypes.c_void_p(st.cuda_stream)
    e, n, i = roles.electron, roles.neutral, roles.ion
    nn0 = species[n].n
    dsp, offs, counts = [], [], []
    with torch.cuda.stream(st):
        scratch = torch.empty(lib.pb_layout_scratch_bytes(nc), dtype=torch.uint8, device=dev)
        for k, (f, d) in enumerate(zip(species, defs)):
            cap = f.n + (nn0 if k in (e, i) else 0)
            s = DeviceSpecies(d, f.n, dev, kind=_lib.PB_KIND_INACTIVE, deposit=-1, cap=cap)
            s.upload(f)
            o = torch.zeros(nc + 1, dtype=torch.int64, device=dev)
            c = torch.zeros(nc, dtype=torch.int64, device=dev)
            _lib.check(lib.pb_cell_layout(s.cell.data_ptr(), s.n, nc, o.data_ptr(), c.data_ptr(),
                                          scratch.data_ptr(), scratch.numel(), sh), "pb_cell_layout")
            dsp.append(s)
            offs.append(o)
            counts.append(c)
        ctr = torch.zeros(6, dtype=torch.int64, device=dev)
        nb_cell = torch.zeros(nc, dtype=torch.int64, device=dev)
        nb_k = torch.zeros(max(nn0, 1), dtype=torch.int32, device=dev)
        p = collision_params(rates, consts, dx_m, weights[n], defs[e].mass_kg, step_key, global_offset)
        pe, pn, pi = dsp[e].pb(), dsp[n].pb(), dsp[i].pb()
        _lib.check(lib.pb_collide(ctypes.byref(pe), ctypes.byref(pn), ctypes.byref(pi),
                                  offs[e].data_ptr(), counts[e].data_ptr(), offs[n].data_ptr(),
                                  counts[n].data_ptr(), nc, ctypes.byref(p), nb_cell.data_ptr(),
                                  nb_k.data_ptr(), nn0, ctr.data_ptr(), sh), "pb_collide")
    st.synchronize()
    c = ctr.cpu().tolist()
    if c[5]:
        raise RuntimeError("collision pass overflow")
    newborns = int(c[4])
    status = status_template(dev)
    out = []
    with torch.cuda.stream(st):
        cap = max(s.cap for s in dsp)
        scr = torch.empty(lib.pb_canonical_scratch_bytes(cap, nc), dtype=torch.uint8, device=dev)
        for k, s in enumerate(dsp):
            tail = newborns if k in (e, i) else 0
            cv = _lib.PbCanon()
            cv.n_old, cv.n_tail = s.n, tail
            cv.offs, cv.counts = offs[k].data_ptr(), counts[k].data_ptr()
            cv.newborn_per_cell = nb_cell.data_ptr() if tail else None
            cv.newborn_k = nb_k.data_ptr() if tail else None
            dst = s.spare()
            a, b = s.pb(s.n + tail), dst.pb(s.n + tail)  # kind INACTIVE: commit order only
            _lib.check(lib.pb_canonical_resort(ctypes.byref(a), ctypes.byref(b), ctypes.byref(cv), None,
                                               nc, _lib.PB_BC_PERIODIC, k, status.data_ptr(),
                                               scr.data_ptr(), scr.numel(), sh), "pb_canonical_resort")
            s.swap_with_spare()
        news = torch.stack([o[nc] for o in offs]).cpu().tolist()
    st.synchronize()
    for s, m in zip(dsp, news):
        s.n = int(m)
        out.append(s.download())
    return CollisionTally(int(c[0]), int(c[1]), int(c[2]), int(c[3])), out


def flat(x, vx, vy, vz, yp, cell) -> FlatSpecies:
    return FlatSpecies(x=x, vx=vx, vy=vy, vz=vz, yp=yp, cell=cell)
