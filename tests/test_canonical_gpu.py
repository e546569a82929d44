"""GPU: canonical slot order mode and device collisions vs the reference.

Bar (all bit-exact): particle stores in the reference's slot order, rho and
E at every step, per-step totals and collision tallies.  Golden fixtures are
outputs of the reference itself (tests/golden/make_golden.py); extension
configs without reference behaviour (absorbing walls, Boris) are checked
against the oracle's restatement (oracle/oracle.py:run_canonical).
"""

import hashlib
import json
import math
from dataclasses import replace

import numpy as np
import pytest

from conftest import bits_equal, load_golden
from golden_cfg import COLLISION_KATS, RUNS_ALL, cfg_from, host_species

pytestmark = pytest.mark.gpu


@pytest.fixture
def scatter_min(cuda):
    """Set the canonical scatter-resort threshold; restores the default."""
    from paper_2404_10270_b200 import _lib

    lib = _lib.load()

    def set_(n):
        _lib.check(lib.pb_set_canonical_scatter_min(int(n)), "pb_set_canonical_scatter_min")

    yield set_
    set_(1 << 20)


def _flat_from(d):
    from paper_2404_10270_b200.core import FlatSpecies

    return FlatSpecies(x=d["x"], vx=d["vx"], vy=d["vy"], vz=d["vz"], yp=d.get("yp"),
                       cell=np.asarray(d["cell"], dtype=np.int32))


def _as_dict(f):
    d = dict(f.fields())
    d["cell"] = f.cell
    return d


def _assert_stores(got, ref, prefix=""):
    """got: list of FlatSpecies; ref: golden dict or list of dicts."""
    for isp, f in enumerate(got):
        for name, arr in f.fields().items():
            want = ref[f"{prefix}sp{isp}_{name}"] if isinstance(ref, dict) else ref[isp][name]
            assert bits_equal(arr, want), (isp, name)
        want = ref[f"{prefix}sp{isp}_cell"] if isinstance(ref, dict) else ref[isp]["cell"]
        assert np.array_equal(f.cell.astype(np.int64), np.asarray(want, dtype=np.int64)), isp


@pytest.mark.parametrize("name", COLLISION_KATS)
def test_device_collision_phase_matches_reference(cuda, name):
    """collision_phase on the reference test stores (test_collisions.py:45-66)."""
    from paper_2404_10270_b200 import PhysicalConstants, SpeciesDef
    from paper_2404_10270_b200.collisions import CollisionRates, Roles, collision_phase

    from test_collisions_oracle import kat_case

    z = load_golden("collision_kats.npz")
    roles, _, sp, nc, key = kat_case(z, name)
    m = z[f"{name}_masses"]
    e_ch = 1.602176634e-19
    defs = [SpeciesDef("e", -e_ch, float(m[0])), SpeciesDef("i", e_ch, float(m[1])),
            SpeciesDef("n", 0.0, float(m[2]))]
    r = z[f"{name}_rates"]
    tally, out = collision_phase([_flat_from(d) for d in sp], defs, list(z[f"{name}_weights"]),
                                 CollisionRates(*[float(v) for v in r]), PhysicalConstants(dt_s=1.0),
                                 Roles(electron=roles[0], neutral=roles[1], ion=roles[2]),
                                 key, nc, 1.0, device=cuda)
    assert [tally.elastic, tally.excitation, tally.ionization, tally.suppressed] == list(z[f"{name}_tally"])
    _assert_stores(out, z, f"{name}_out_")


def _run(cfg):
    from paper_2404_10270_b200 import run_simulation

    hist = {"rho": [], "e": [], "tally": []}

    def probe(step, st):
        hist["rho"].append(st["rho"])
        hist["e"].append(st["e_field"])
        if step == cfg.n_steps:
            hist["final"] = list(st["stores"][0])

    m = run_simulation(cfg, on_step=probe)
    return m, hist


@pytest.mark.parametrize("resort", ["sort", "scatter"])
@pytest.mark.parametrize("name", RUNS_ALL)
def test_canonical_run_matches_reference_bitwise(cuda, name, resort, scatter_min):
    """resort: the full key sort (stores under the scatter threshold, here all)
    or the scatter path (stayers by prefix count, movers sorted) forced on."""
    scatter_min(0 if resort == "scatter" else 1 << 40)
    g = load_golden(f"{name}.npz")
    cfg = cfg_from(g, slot_order="canonical")
    m, h = _run(cfg)
    assert m.layout == "canonical_soa"
    assert bits_equal(np.array(h["rho"]), g["rho"])
    assert bits_equal(np.array(h["e"]), g["e_field"])
    names = [s.name for s in cfg.species]
    assert np.array_equal(np.array([[r[f"total_{n}"] for n in names] for r in m.diagnostics]), g["totals"])
    if "tallies" in g:
        got = np.array([[r["elastic"], r["excitation"], r["ionization"], r["suppressed"]]
                        for r in m.diagnostics])
        assert np.array_equal(got, g["tallies"])
        t = g["tallies"].sum(axis=0)
        assert [m.tally.elastic, m.tally.excitation, m.tally.ionization, m.tally.suppressed] == list(t)
    _assert_stores(h["final"], g)


def test_collisions_select_canonical_engine_automatically(cuda):
    g = load_golden("run_collide_desk.npz")
    cfg = cfg_from(g)  # slot_order "auto"
    assert cfg.canonical()
    m, _ = _run(replace(cfg, n_steps=3))
    assert m.layout == "canonical_soa"


def _ext_config(**kw):
    from paper_2404_10270_b200 import Grid1D, PhysicalConstants, RunConfig, SpeciesDef
    from paper_2404_10270_b200.config import CollisionRates, CollisionSetup
    from paper_2404_10270_b200.core import DEUTERIUM_MASS, ELECTRON_MASS, ELEMENTARY_CHARGE

    species = [SpeciesDef("e", -ELEMENTARY_CHARGE, ELECTRON_MASS),
               SpeciesDef("D+", ELEMENTARY_CHARGE, DEUTERIUM_MASS - ELECTRON_MASS, nstep=2),
               SpeciesDef("D", 0.0, DEUTERIUM_MASS, nstep=3, track_transverse=True)]
    base = dict(grid=Grid1D.from_cells(40, 40e-5), consts=PhysicalConstants(dt_s=4e-14), species=species,
                temperatures_ev=[60.0, 200.0, 40.0], densities_m3=[1e21, 1e21, 1e21], ppc0=12, n_steps=20,
                seed=99, boundary="dirichlet", field_solve=True, smoothing_passes=1,
                phi_left=3.0, phi_right=-1.0,
                collisions=CollisionSetup(True, "e", "D", "D+",
                                          CollisionRates(4e-10, 1e-10, 6e-10, 12.0)),
                slot_order="canonical")
    base.update(kw)
    return RunConfig(**base)


@pytest.mark.parametrize("boundary", ["periodic", "absorbing", "boris_gradb"])
def test_canonical_extensions_match_oracle(cuda, boundary):
    """Absorbing walls + collisions + nstep>1 + Dirichlet field solve, and
    the Boris push in a spatially varying B: no reference behaviour, so the
    oracle restatement is the bar (bit-exact)."""
    from oracle import oracle

    if boundary == "boris_gradb":
        # B gathered per particle from nodes (pb_species.b_nodes), strong
        # enough (|t| ~ 0.01-0.05 for electrons) that the rotation matters
        cfg = _ext_config(b_field_t=(0.4, -0.3, 2.0), b_grad_t_per_m=(150.0, 40.0, -900.0))
    else:
        cfg = _ext_config(particle_boundary=boundary,
                          boundary="dirichlet" if boundary == "absorbing" else "periodic")
    h = oracle.run_canonical(cfg, host_species(cfg))
    m, d = _run(cfg)
    names = [s.name for s in cfg.species]
    assert np.array_equal(np.array([[r[f"total_{n}"] for n in names] for r in m.diagnostics]),
                          np.array(h["totals"]))
    assert np.array_equal(np.array([[r["elastic"], r["excitation"], r["ionization"], r["suppressed"]]
                                    for r in m.diagnostics]), np.array(h["tallies"]))
    assert bits_equal(np.array(d["rho"]), np.array(h["rho"]))
    assert bits_equal(np.array(d["e"]), np.array(h["e"]))
    _assert_stores(d["final"], h["species"])
    if boundary == "absorbing":
        assert sum(sum(v) for v in m.absorbed.values()) > 0
        assert h["totals"][-1][0] < h["totals"][0][0] + m.tally.ionization


def test_desk_criterion01_bitwise_and_ode(cuda, scatter_min):
    """pkg/configs/desk.toml to the ODE half-depletion step (the reference's
    acceptance criterion 01, pkg/tests/test_acceptance.py:73-117): every
    per-step diagnostic row, the last rho and the final stores equal the
    reference run bit for bit, and the neutral total is within 5% of the
    ODE oracle.  The canonical resort runs on its scatter path throughout."""
    import os

    from paper_2404_10270_b200 import load_config, run_simulation

    scatter_min(0)
    g = load_golden("run_desk_criterion01.npz")
    cfg = load_config(os.path.join(os.path.dirname(__file__), "..", "configs", "desk.toml"))
    steps = int(g["steps"])
    cfg = replace(cfg, n_steps=steps, out_dir=None)
    box = {}

    def probe(step, st):
        if step == steps:
            box["rho"] = st["rho"]
            box["final"] = list(st["stores"][0])

    m = run_simulation(cfg, on_step=probe)
    names = [s.name for s in cfg.species]
    assert np.array_equal(np.array([[r[f"total_{n}"] for n in names] for r in m.diagnostics]), g["totals"])
    assert np.array_equal(np.array([[r["elastic"], r["excitation"], r["ionization"], r["suppressed"]]
                                    for r in m.diagnostics]), g["tallies"])
    assert bits_equal(box["rho"], g["rho_last"])
    digests = json.loads(str(g["digests"]))
    for isp, f in enumerate(box["final"]):
        for name, arr in list(f.fields().items()) + [("cell", f.cell)]:
            if name == "cell":
                arr = arr.astype(np.int32)
            got = hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()
            assert got == digests[f"sp{isp}_{name}"], (isp, name)
    expect = cfg.grid.nc * float(g["ode_nn"])
    got = m.diagnostics[-1]["total_D"]
    assert abs(got - expect) / expect <= 0.05
    totals = [row["total_D"] for row in m.diagnostics]
    assert all(b <= a for a, b in zip(totals, totals[1:]))


def test_collision_statistics_binomial(cuda):
    """criterion 09 shape (pkg/tests/test_acceptance.py:414-489) at 2.6e5
    trials per pass on the device: ionization count within 4 sigma."""
    from paper_2404_10270_b200 import PhysicalConstants, SpeciesDef
    from paper_2404_10270_b200.collisions import CollisionRates, Roles, collision_phase, step_stream_key
    from paper_2404_10270_b200.core import FlatSpecies

    e_ch, amu = 1.602176634e-19, 1.66053906660e-27
    defs = [SpeciesDef("e", -e_ch, 9.1093837015e-31), SpeciesDef("i", e_ch, 2 * amu), SpeciesDef("n", 0.0, 2 * amu)]
    nc, ne0, nn0, p_target = 4096, 64, 1000, 0.02
    rate = -math.log1p(-p_target) / nn0
    rng = np.random.default_rng(7)

    def species(per_cell, vth):
        n = nc * per_cell
        return FlatSpecies(x=rng.random(n), vx=vth * rng.standard_normal(n), vy=vth * rng.standard_normal(n),
                           vz=vth * rng.standard_normal(n), yp=None,
                           cell=np.repeat(np.arange(nc, dtype=np.int32), per_cell))

    sp = [species(ne0, 3e6), species(0, 0.0), species(nn0, 1e3)]
    expected = variance = observed = 0.0
    for p in range(4):
        ce = np.bincount(sp[0].cell, minlength=nc).astype(float)
        cn = np.bincount(sp[2].cell, minlength=nc).astype(float)
        pio = -np.expm1(-cn * rate)
        expected += float(np.sum(ce * pio))
        variance += float(np.sum(ce * pio * (1.0 - pio)))
        tally, sp = collision_phase(sp, defs, [1.0, 1.0, 1.0], CollisionRates(0.0, 0.0, rate, 0.0),
                                    PhysicalConstants(dt_s=1.0), Roles(0, 2, 1), step_stream_key(20260819, p),
                                    nc, 1.0, device=cuda)
        observed += tally.ionization
        assert tally.suppressed == 0
    assert abs(observed - expected) <= 4.0 * math.sqrt(variance)
    assert sp[0].n == nc * ne0 + observed and sp[1].n == observed and sp[2].n == nc * nn0 - observed


def test_canonical_run_pipelined_matches_reference(cuda):
    """CanonicalEngine.run_pipelined (the host-driven loop of the public
    engine API) hands every step's rho to the host, bitwise the reference's."""
    from paper_2404_10270_b200.canonical import CanonicalEngine

    g = load_golden("run_collide_desk.npz")
    cfg = cfg_from(g)
    eng = CanonicalEngine(cfg, device=cuda, init="host")
    got = {}
    n = eng.run_pipelined(cfg.n_steps, on_result=lambda k, r: got.__setitem__(k, r.numpy().copy()))
    assert n == cfg.n_steps
    for k in range(cfg.n_steps):
        assert bits_equal(got[k], g["rho"][k]), k
    with pytest.raises(Exception):
        eng.run_pipelined(1, e_source=lambda k: None)
