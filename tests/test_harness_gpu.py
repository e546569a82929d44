"""run_simulation on the B200 engine vs the reference's own run_simulation
(golden runs recorded by tests/golden/make_golden.py).

Tolerances:
  field solve off: final particles bit-exact (multiset), totals exact,
                   rho per step |d| <= 1e-12 * max_s |coef_s| * 2 ppc0
  field solve on:  rho as above; E per step |d| <= 1e-9 * max|E|;
                   particles matched by their untouched vz tag,
                   |d(cell + x)| <= 1e-9 cells, |d vx| <= 1e-9 * max|vx|
"""

import json

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _cfg_from(g, **extra):
    from paper_2404_10270_b200 import Grid1D, PhysicalConstants, RunConfig, SpeciesDef

    c = json.loads(str(g["config"]))
    species = [SpeciesDef(n, q, m, nstep=ns, active_mover=am, track_transverse=tt)
               for n, q, m, ns, am, tt in c["species"]]
    return RunConfig(grid=Grid1D.from_cells(c["nc"], c["length_m"]), consts=PhysicalConstants(dt_s=c["dt_s"]),
                     species=species, temperatures_ev=c["temperatures_ev"], densities_m3=c["densities_m3"],
                     ppc0=c["ppc0"], n_steps=c["n_steps"], seed=c["seed"], boundary=c["boundary"],
                     field_solve=c["field_solve"], smoothing_passes=c["smoothing_passes"], **extra)


def _run(cfg):
    from paper_2404_10270_b200 import run_simulation

    hist = {"rho": [], "e": [], "final": None}

    def probe(step, st):
        hist["rho"].append(st["rho"])
        hist["e"].append(st["e_field"])
        if step == cfg.n_steps:
            hist["final"] = st["stores"][0]

    m = run_simulation(cfg, on_step=probe)
    return m, hist


def _rho_scale(cfg):
    from paper_2404_10270_b200.core import macro_weight

    return max(abs(sp.charge_c * macro_weight(cfg, k) / cfg.grid.dx_m)
               for k, sp in enumerate(cfg.species) if sp.charged) * 2 * cfg.ppc0


@pytest.mark.parametrize("sort_every", [0, 7])
def test_periodic_run_matches_reference(cuda, sort_every):
    from oracle import oracle

    g = load_golden("run_periodic_nofield.npz")
    cfg = _cfg_from(g, sort_every=sort_every)
    m, h = _run(cfg)
    scale = _rho_scale(cfg)
    assert len(h["rho"]) == cfg.n_steps
    for step, rho in enumerate(h["rho"]):
        assert np.max(np.abs(rho - g["rho"][step])) <= 1e-12 * scale, step
        assert np.all(h["e"][step] == 0.0)
    assert np.array_equal(np.array([[r[f"total_{s.name}"] for s in cfg.species] for r in m.diagnostics]),
                          g["totals"])
    for k, f in enumerate(h["final"]):
        ref = {n: g[f"sp{k}_{n}"] for n in f.fields()}
        assert np.array_equal(oracle.canonical(f.cell, f.fields()), oracle.canonical(g[f"sp{k}_cell"], ref))
    assert m.backend == "cuda" and set(m.phase_seconds) >= {"deposit", "mover", "total"}


@pytest.mark.parametrize("name", ["run_periodic_field", "run_dirichlet_field"])
def test_field_solve_run_matches_reference(cuda, name):
    g = load_golden(f"{name}.npz")
    cfg = _cfg_from(g)
    m, h = _run(cfg)
    scale = _rho_scale(cfg)
    for step in range(cfg.n_steps):
        assert np.max(np.abs(h["rho"][step] - g["rho"][step])) <= 1e-12 * scale, step
        emax = np.max(np.abs(g["e_field"][step]))
        assert np.max(np.abs(h["e"][step] - g["e_field"][step])) <= 1e-9 * emax, step
    assert np.array_equal(np.array([[r[f"total_{s.name}"] for s in cfg.species] for r in m.diagnostics]),
                          g["totals"])
    for k, f in enumerate(h["final"]):
        tag = f.vz.view(np.uint64)
        rtag = g[f"sp{k}_vz"].view(np.uint64)
        o, ro = np.argsort(tag), np.argsort(rtag)
        assert np.array_equal(tag[o], rtag[ro])
        pos = f.cell[o].astype(np.float64) + f.x[o]
        rpos = g[f"sp{k}_cell"][ro].astype(np.float64) + g[f"sp{k}_x"][ro]
        d = np.abs(pos - rpos)
        d = np.minimum(d, cfg.grid.nc - d)  # periodic wrap
        assert np.max(d) <= 1e-9
        vmax = np.max(np.abs(g[f"sp{k}_vx"]))
        assert np.max(np.abs(f.vx[o] - g[f"sp{k}_vx"][ro])) <= 1e-9 * vmax


def test_poisson_and_stencils_bitwise_given_reference_rho(cuda):
    """Fed the reference's rho, the device smoother / Poisson / E kernels
    reproduce the reference's phi and E bit for bit (fields.py:121-218)."""
    import ctypes

    import torch

    from conftest import bits_equal
    from paper_2404_10270_b200 import _lib

    lib = _lib.load()
    g = load_golden("fields.npz")
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for nc in (8, 100, 1000):
        dx = nc * 1e-5 / nc
        rho = torch.from_numpy(g[f"n{nc}_rho"]).to(cuda)
        out = torch.empty_like(rho)
        scr = torch.empty(lib.pb_field_scratch_bytes(nc) // 8 + 1, dtype=torch.float64, device=cuda)
        for passes, key in ((1, "smooth1"), (3, "smooth3")):
            _lib.check(lib.pb_smooth_density(rho.data_ptr(), out.data_ptr(), nc, passes, scr.data_ptr(), stream))
            assert bits_equal(out.cpu().numpy(), g[f"n{nc}_{key}"])
        for bc, code in (("periodic", 0), ("dirichlet", 1)):
            phi = torch.empty_like(rho)
            e = torch.empty_like(rho)
            _lib.check(lib.pb_solve_poisson(rho.data_ptr(), phi.data_ptr(), nc, dx, 8.8541878128e-12, code,
                                            1.5, -2.0, scr.data_ptr(), stream))
            _lib.check(lib.pb_compute_efield(phi.data_ptr(), e.data_ptr(), nc, dx, code, stream))
            assert bits_equal(phi.cpu().numpy(), g[f"n{nc}_{bc}_phi"]), (nc, bc)
            assert bits_equal(e.cpu().numpy(), g[f"n{nc}_{bc}_e"]), (nc, bc)


def test_poisson_scan_matches_reference_and_exact(cuda):
    """Parallel prefix-sum Poisson vs the reference's serial elimination:
    within 1e-12 * max|phi| on the golden fields and on a 100K-cell grid."""
    import ctypes

    import torch

    from paper_2404_10270_b200 import _lib

    lib = _lib.load()
    g = load_golden("fields.npz")
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def solve(fn, rho_np, nc, code):
        rho = torch.from_numpy(rho_np).to(cuda)
        phi = torch.empty_like(rho)
        scr = torch.empty(lib.pb_field_scratch_bytes(nc) // 8 + 1, dtype=torch.float64, device=cuda)
        _lib.check(fn(rho.data_ptr(), phi.data_ptr(), nc, 1e-5, 8.8541878128e-12, code, 1.5, -2.0,
                      scr.data_ptr(), stream))
        return phi.cpu().numpy()

    for nc in (8, 100, 1000):
        for bc, code in (("periodic", 0), ("dirichlet", 1)):
            phi = solve(lib.pb_solve_poisson_scan, g[f"n{nc}_rho"], nc, code)
            ref = g[f"n{nc}_{bc}_phi"]
            assert np.max(np.abs(phi - ref)) <= 1e-12 * np.max(np.abs(ref)), (nc, bc)
    rng = np.random.default_rng(5)
    for nc in (3, 2048, 2049, 4097, 6001):  # tile-boundary sizes of the multi-block scan
        rho = 30.0 * rng.standard_normal(nc + 1)
        rho[nc] = rho[0]
        for code in (0, 1):
            a = solve(lib.pb_solve_poisson_scan, rho, nc, code)
            b = solve(lib.pb_solve_poisson, rho, nc, code)
            assert np.max(np.abs(a - b)) <= 1e-10 * np.max(np.abs(b)), (nc, code)
            assert a[nc] == a[0] or code == 1
    nc = 100_000
    rho = 30.0 * rng.standard_normal(nc + 1) + 5.0 * np.sin(np.arange(nc + 1) * 2e-4)
    rho[nc] = rho[0]
    for code in (0, 1):
        a = solve(lib.pb_solve_poisson_scan, rho, nc, code)
        b = solve(lib.pb_solve_poisson, rho, nc, code)
        # The (1,-2,1) system has condition number ~ 0.4 n^2 (4e9 at 1e5
        # unknowns), so two correct eliminations differ by up to ~n^2 eps
        # relative (observed 1.5e-10); the bar is 1e-8 on phi up to the
        # periodic gauge constant, and on E = -grad phi.
        d = a - b
        assert np.max(np.abs(d - d.mean())) <= 1e-8 * np.max(np.abs(b)), code
        ea, eb = -np.diff(a), -np.diff(b)
        assert np.max(np.abs(ea - eb)) <= 1e-8 * np.max(np.abs(eb)), code


def _small_sheath(n_steps=60, nc=256, sort_every=10):
    from paper_2404_10270_b200.config import load_config

    cfg = load_config("configs/c3_sheath_absorbing.toml")
    from dataclasses import replace

    from paper_2404_10270_b200 import Grid1D

    return replace(cfg, grid=Grid1D.from_cells(nc, nc * 1e-5), ppc0=40, n_steps=n_steps,
                   sort_every=sort_every)


@pytest.mark.parametrize("which", ["periodic_field", "sheath", "periodic_nofield"])
def test_graphed_run_simulation_matches_per_step_path(cuda, which, monkeypatch):
    """on_step=None replays CUDA graphs (status checked every CHECK_EVERY
    steps, diagnostics from device counters); the per-step diagnostics and
    phase keys equal the eager on_step path's, every step, exactly."""
    from paper_2404_10270_b200 import harness, run_simulation

    if which == "sheath":
        cfg = _small_sheath()
    else:
        cfg = _cfg_from(load_golden(f"run_{which}.npz"), sort_every=5)
    monkeypatch.setattr(harness, "CHECK_EVERY", 16)
    fast = run_simulation(cfg)
    slow = run_simulation(cfg, on_step=lambda s, st: None)
    assert fast.diagnostics == slow.diagnostics
    if which == "sheath":  # walls actually absorbed something, and counts moved
        tot = [r["total_e"] for r in fast.diagnostics]
        assert tot[-1] < tot[0] and len(set(tot)) > 2
        assert fast.absorbed == slow.absorbed
    assert set(fast.phase_seconds) == set(slow.phase_seconds)
    assert fast.phase_seconds["total"] > 0.0


def test_graphed_run_simulation_raises_cfl_in_window(cuda, monkeypatch):
    """A domain-scale jump still raises CflViolation on the graphed path,
    naming the window of steps since the last status check."""
    from dataclasses import replace

    from paper_2404_10270_b200 import harness, run_simulation
    from paper_2404_10270_b200.errors import CflViolation

    g = load_golden("run_periodic_nofield.npz")
    cfg = _cfg_from(g)
    cfg = replace(cfg, temperatures_ev=[1e9] + list(cfg.temperatures_ev[1:]), n_steps=40)
    monkeypatch.setattr(harness, "CHECK_EVERY", 16)
    with pytest.raises(CflViolation, match=r"steps 1-16, phase resort"):
        run_simulation(cfg)
