"""Generate the golden fixtures in this directory by running the REFERENCE.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
It copies /root/reference/pkg to a scratch dir, builds its Cython kernels
(python setup.py build_ext --inplace, the reference's own recipe), imports
`picmc` from there with PICMC_BACKEND=compiled, and records inputs/outputs of
the hot-path functions as small .npz files.  Nothing here is imported by the
product; tests/ compare the oracle and the CUDA path against these files, so
the GPU box never needs /root/reference.
"""

import json
import os
import shutil
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"
SCRATCH = "/tmp/picmc_ref_golden"


def import_reference():
    if not os.path.exists(os.path.join(SCRATCH, "src", "picmc", "backends")):
        shutil.rmtree(SCRATCH, ignore_errors=True)
        shutil.copytree(REF, SCRATCH)
    built = [f for f in os.listdir(os.path.join(SCRATCH, "src", "picmc", "backends")) if f.endswith(".so")]
    if not built:
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH, check=True,
                       stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    os.environ["PICMC_BACKEND"] = "compiled"
    sys.path.insert(0, os.path.join(SCRATCH, "src"))
    sys.path.insert(0, os.path.join(SCRATCH, "tests"))
    import picmc  # noqa: F401

    return picmc


def packed(seed, nc=13, cap=7):
    # same recipe as pkg/tests/test_backends.py:21-39
    rng = np.random.default_rng(seed)
    counts = rng.integers(0, cap + 1, size=nc).astype(np.int64)
    caps = np.full(nc, cap, dtype=np.int64)
    offs = np.concatenate(([0], np.cumsum(caps[:-1]))).astype(np.int64)
    total = int(caps.sum())
    x, vx, vy, yp = np.zeros(total), np.zeros(total), np.zeros(total), np.zeros(total)
    for j in range(nc):
        n = counts[j]
        sl = slice(offs[j], offs[j] + n)
        x[sl] = rng.random(n)
        vx[sl] = rng.standard_normal(n) * 0.3
        vy[sl] = rng.standard_normal(n) * 0.3
        yp[sl] = rng.standard_normal(n)
    return x, vx, vy, yp, offs, counts


def gen_backend(picmc):
    from picmc import backends

    k = backends.load_backend("compiled")
    out = {}
    for seed in range(5):
        x, vx, vy, yp, offs, counts = packed(seed)
        out[f"s{seed}_x"], out[f"s{seed}_vx"], out[f"s{seed}_vy"], out[f"s{seed}_yp"] = x, vx, vy, yp
        out[f"s{seed}_offs"], out[f"s{seed}_counts"] = offs, counts
        left, right = k.deposit_partials(x, offs, counts)
        out[f"s{seed}_dep_left"], out[f"s{seed}_dep_right"] = left, right
        nodes = np.random.default_rng(100 + seed).standard_normal(len(counts) + 1)
        out[f"s{seed}_nodes"] = nodes
        out[f"s{seed}_gather"] = k.gather(nodes, x, offs, counts)
        accel = np.random.default_rng(200 + seed).standard_normal(len(counts) + 1) * 0.1
        out[f"s{seed}_accel"] = accel
        for wa in (0, 1):
            for wy in (0, 1):
                a = [x.copy(), vx.copy(), vy.copy(), yp.copy() if wy else None]
                k.fused_move(accel if wa else None, *a, offs, counts, 2.0)
                out[f"s{seed}_move_a{wa}y{wy}_x"] = a[0]
                out[f"s{seed}_move_a{wa}y{wy}_vx"] = a[1]
                if wy:
                    out[f"s{seed}_move_a{wa}y{wy}_yp"] = a[3]
        # layout-study kernels (_kernels.pyx:105-152) on the same particles
        tab = np.stack([x, vx, vy, np.zeros_like(x), yp], axis=1).copy()
        for wa in (0, 1):
            for wy in (0, 1):
                t = tab.copy()
                k.fused_move_aos(t, offs, counts, accel, 3.0, bool(wa), bool(wy))
                out[f"s{seed}_aos_a{wa}y{wy}"] = t
        t = tab[: int(counts[0])].copy()
        k.fused_move_table(t, 0.3, -0.2, 2.0, True, True)
        out[f"s{seed}_table"] = t
    np.savez_compressed(os.path.join(HERE, "backend_kernels.npz"), **out)


def gen_resort(picmc):
    """Exact cell-transfer cases of pkg/tests/test_mover.py:106-160, as
    (src cell, x) -> (dest cell, x) through the reference resort()."""
    from picmc.core import CellSortedStore, Grid1D, SpeciesDef
    from picmc.mover import resort

    cases = [(8, 3, -0.25), (8, 0, -0.25), (8, 7, 1.25), (100, 0, -0.3), (8, 1, 2.0), (8, 2, 3.5),
             (8, 4, -1e-18), (8, 5, 0.999999999), (8, 6, 1.0), (8, 0, -6.5), (8, 7, 7.999), (8, 3, -0.0),
             (37, 36, 1e-300 + 1.0), (37, 0, -35.5)]
    rows = []
    for nc, cell, x in cases:
        store = CellSortedStore(Grid1D.from_cells(nc, float(nc)), [SpeciesDef("s", 0.0, 1.0)], initial_cap=4)
        store.append(0, cell, {"x": x, "vx": 0.5})
        resort(store)
        j = int(np.nonzero(store.counts(0))[0][0])
        xo = float(store.data(0)["x"][store.cell_slice(0, j)][0])
        rows.append((nc, cell, x, j, xo))
    arr = np.array(rows, dtype=object)
    np.savez_compressed(os.path.join(HERE, "resort_kats.npz"),
                        nc=np.array([r[0] for r in rows], dtype=np.int64),
                        cell=np.array([r[1] for r in rows], dtype=np.int64),
                        x=np.array([r[2] for r in rows], dtype=np.float64),
                        dest=np.array([r[3] for r in rows], dtype=np.int64),
                        xo=np.array([r[4] for r in rows], dtype=np.float64))
    del arr


def gen_rng(picmc):
    from picmc import rng

    keys = [0, 1, 1234567, 20260819, (1 << 64) - 1]
    out = {"keys": np.array(keys, dtype=np.uint64)}
    out["mix64"] = np.array([rng.mix64(k) for k in keys], dtype=np.uint64)
    out["derive"] = np.array([[rng.derive(k, n) for n in range(6)] for k in keys], dtype=np.uint64)
    out["stream"] = np.array([rng.stream(20260819, 1, isp) for isp in range(3)], dtype=np.uint64)
    ctr = np.arange(64, dtype=np.int64)
    out["uniforms"] = rng.uniforms(np.uint64(out["stream"][0]), ctr)
    out["uniforms_open"] = rng.uniforms_open(np.uint64(out["stream"][1]), ctr)
    np.savez_compressed(os.path.join(HERE, "rng.npz"), **out)


def small_config(**kw):
    from conftest import make_config  # the reference's own test builder

    return make_config(**kw)


def config_record(cfg):
    return json.dumps({
        "nc": cfg.grid.nc, "length_m": cfg.grid.length_m, "dt_s": cfg.consts.dt_s,
        "species": [[s.name, s.charge_c, s.mass_kg, s.nstep, s.active_mover, s.track_transverse]
                    for s in cfg.species],
        "temperatures_ev": cfg.temperatures_ev, "densities_m3": cfg.densities_m3, "ppc0": cfg.ppc0,
        "n_steps": cfg.n_steps, "seed": cfg.seed, "boundary": cfg.boundary,
        "field_solve": cfg.field_solve, "smoothing_passes": cfg.smoothing_passes,
    })


def flatten_store(store):
    """Live particles in cell-major order with their cell index."""
    out = {}
    for isp in range(store.nsp):
        idx = store.live_indices(isp)
        out[f"sp{isp}_cell"] = store.cell_of_live(isp).astype(np.int32)
        for name, arr in store.data(isp).items():
            out[f"sp{isp}_{name}"] = arr[idx].copy()
    return out


def gen_init(picmc):
    from picmc.core import init_plasma

    cfg = small_config(nc=16, ppc0=8)
    store = init_plasma(cfg)
    out = flatten_store(store)
    out["config"] = np.array(config_record(cfg))
    out["weights"] = np.array(store.weights)
    np.savez_compressed(os.path.join(HERE, "init_plasma.npz"), **out)


def gen_runs(picmc):
    from picmc.decomposition import merge_stores
    from picmc.harness import run_simulation

    runs = {
        "run_periodic_nofield": dict(nc=64, ppc0=8, n_steps=20),
        "run_periodic_field": dict(nc=64, ppc0=8, n_steps=20, field_solve=True, smoothing_passes=1),
        "run_dirichlet_field": dict(nc=48, ppc0=8, n_steps=20, field_solve=True, smoothing_passes=2,
                                    boundary="dirichlet"),
    }
    for name, kw in runs.items():
        cfg = small_config(**kw)
        hist = {"rho": [], "e": []}
        box = {}

        def probe(step, st, hist=hist, box=box):
            hist["rho"].append(st["rho"].copy())
            hist["e"].append(st["e_field"].copy())
            box["stores"], box["partition"] = st["stores"], st["partition"]

        m = run_simulation(cfg, on_step=probe)
        final = merge_stores(box["stores"], box["partition"], cfg.grid)
        out = flatten_store(final)
        out["rho"] = np.array(hist["rho"])
        out["e_field"] = np.array(hist["e"])
        out["totals"] = np.array([[r[f"total_{s.name}"] for s in cfg.species] for r in m.diagnostics])
        out["config"] = np.array(config_record(cfg))
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


def gen_fields(picmc):
    from picmc.core import Grid1D, PhysicalConstants
    from picmc.fields import compute_efield, smooth_density, solve_poisson

    rng = np.random.default_rng(77)
    out = {}
    for nc in (8, 100, 1000):
        grid = Grid1D.from_cells(nc, nc * 1e-5)
        consts = PhysicalConstants(dt_s=4e-14)
        rho = 50.0 * rng.standard_normal(nc + 1)
        rho[nc] = rho[0]
        out[f"n{nc}_rho"] = rho
        out[f"n{nc}_smooth1"] = smooth_density(rho, 1)
        out[f"n{nc}_smooth3"] = smooth_density(rho, 3)
        for bc in ("periodic", "dirichlet"):
            phi = solve_poisson(rho, grid, consts, bc, 1.5, -2.0)
            out[f"n{nc}_{bc}_phi"] = phi
            out[f"n{nc}_{bc}_e"] = compute_efield(phi, grid, bc)
    np.savez_compressed(os.path.join(HERE, "fields.npz"), **out)


def gen_mover_multistep(picmc):
    """mover_phase + resort over 30 steps with multi-cell jumps, signed zeros,
    nstep=3 + transverse, non-zero E (SURVEY Appendix B.10 setup)."""
    from picmc.core import CellSortedStore, Grid1D, PhysicalConstants, SpeciesDef
    from picmc.mover import mover_phase, resort
    from picmc.scheduler import Scheduler

    nc, ppc = 37, 20
    species = [SpeciesDef("q", -1.602176634e-19, 9.1093837015e-31),
               SpeciesDef("n", 0.0, 3.3e-27, nstep=3, track_transverse=True)]
    store = CellSortedStore(Grid1D.from_cells(nc, nc * 1e-5), species, initial_cap=4 * ppc)
    rng = np.random.default_rng(2026)
    for isp in range(2):
        store.counts(isp)[:] = ppc
        idx = store.live_indices(isp)
        d = store.data(isp)
        d["x"][idx] = rng.random(idx.size)
        for f in ("vx", "vy", "vz"):
            d[f][idx] = 0.7 * rng.standard_normal(idx.size)
        d["vx"][idx[::17]] = -0.0
        if "yp" in d:
            d["yp"][idx] = rng.standard_normal(idx.size)
    init = flatten_store(store)
    consts = PhysicalConstants(dt_s=4e-14)
    e_hist = []
    with Scheduler(workers=2, trace=False) as sched:
        for _ in range(30):
            e = 2e3 * rng.standard_normal(nc + 1)
            e_hist.append(e)
            mover_phase(store, e, consts, sched, grainsize=5)
            resort(store)
    out = {f"init_{k}": v for k, v in init.items()}
    out.update({f"final_{k}": v for k, v in flatten_store(store).items()})
    out["e_hist"] = np.array(e_hist)
    out["dt_s"] = np.array(4e-14)
    out["dx_m"] = np.array(store.grid.dx_m)
    np.savez_compressed(os.path.join(HERE, "mover_multistep.npz"), **out)


def gen_collision_runs(picmc):
    """run_simulation with Monte Carlo collisions: the
    final stores in slot order, per-step rho and tallies.  Rates are boosted
    over the desk values so every event kind fires; "guard" makes the summed
    probability exceed 0.1 so the dt-halving substeps run."""
    from conftest import table_collisions
    from picmc.decomposition import merge_stores
    from picmc.harness import run_simulation

    runs = {
        "run_collide_periodic": (dict(nc=32, ppc0=16, n_steps=25),
                                 dict(rate_elastic=5e-10, rate_excitation=5e-11,
                                      rate_ionization=5e-10, threshold_ev=10.2)),
        "run_collide_guard": (dict(nc=24, ppc0=12, n_steps=15, field_solve=True, smoothing_passes=1),
                              dict(rate_elastic=1.5e-9, rate_excitation=4e-10,
                                   rate_ionization=1.5e-9, threshold_ev=30.0)),
        "run_collide_desk": (dict(nc=40, ppc0=10, n_steps=30),
                             dict()),
    }
    for name, (kw, rk) in runs.items():
        cfg = small_config(collisions=table_collisions(**rk), **kw)
        hist = {"rho": [], "e": []}
        box = {}

        def probe(step, st, hist=hist, box=box):
            hist["rho"].append(st["rho"].copy())
            hist["e"].append(st["e_field"].copy())
            box["stores"], box["partition"] = st["stores"], st["partition"]
            if step == 1:
                box["first"] = flatten_store(merge_stores(st["stores"], st["partition"], cfg.grid))

        m = run_simulation(cfg, on_step=probe)
        final = merge_stores(box["stores"], box["partition"], cfg.grid)
        out = flatten_store(final)
        out.update({f"step1_{k}": v for k, v in box["first"].items()})
        out["rho"] = np.array(hist["rho"])
        out["e_field"] = np.array(hist["e"])
        out["totals"] = np.array([[r[f"total_{s.name}"] for s in cfg.species] for r in m.diagnostics])
        out["tallies"] = np.array([[r["elastic"], r["excitation"], r["ionization"], r["suppressed"]]
                                   for r in m.diagnostics])
        out["config"] = np.array(config_record(cfg))
        c = cfg.collisions
        out["collisions"] = np.array(json.dumps({
            "electron": c.electron, "neutral": c.neutral, "ion": c.ion,
            "rates": [c.rates.rate_elastic_m3s, c.rates.rate_excitation_m3s,
                      c.rates.rate_ionization_m3s, c.rates.excitation_threshold_ev]}))
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, m.tally)


def gen_collision_kats(picmc):
    """collision_phase on the reference test stores
    (pkg/tests/test_collisions.py:45-66): suppression, the dt guard, mixed
    events, heavy ionization.  Records the store before and after (slot
    order) and the tally."""
    from test_collisions import CONSTS, ROLES, _rate_for, _store
    from picmc.collisions import CollisionRates, collision_phase, step_stream_key

    cases = {
        "suppressed": (dict(nc=2, ne=400, nn=2, seed=15), {2: 40.0},
                       CollisionRates(rate_ionization_m3s=_rate_for(0.08, 80.0)), (5, 0)),
        "guard": (dict(nc=2, ne=2000, nn=50, seed=17), {},
                  CollisionRates(rate_elastic_m3s=_rate_for(0.5, 50.0)), (7, 0)),
        "mixed": (dict(seed=18, ne=250, nn=40), {},
                  CollisionRates(rate_elastic_m3s=_rate_for(0.02, 40.0),
                                 rate_excitation_m3s=_rate_for(0.01, 40.0),
                                 rate_ionization_m3s=_rate_for(0.03, 40.0),
                                 excitation_threshold_ev=10.2), (8, 3)),
        "ionize": (dict(seed=16, ne=300, nn=50), {},
                   CollisionRates(rate_ionization_m3s=_rate_for(0.05, 50.0)), (6, 0)),
        "guard_ionize": (dict(nc=3, ne=600, nn=60, seed=19), {},
                         CollisionRates(rate_elastic_m3s=_rate_for(0.2, 60.0),
                                        rate_excitation_m3s=_rate_for(0.1, 60.0),
                                        rate_ionization_m3s=_rate_for(0.3, 60.0),
                                        excitation_threshold_ev=10.2), (9, 2)),
    }
    out = {}
    for name, (kw, weights, rates, (seed, step)) in cases.items():
        store = _store(**kw)
        for isp, w in weights.items():
            store.weights[isp] = w
        before = flatten_store(store)
        tally = collision_phase(store, rates, CONSTS, ROLES, step_stream_key(seed, step))
        after = flatten_store(store)
        out.update({f"{name}_in_{k}": v for k, v in before.items()})
        out.update({f"{name}_out_{k}": v for k, v in after.items()})
        out[f"{name}_nc"] = np.array(store.grid.nc)
        out[f"{name}_weights"] = np.array(store.weights)
        out[f"{name}_rates"] = np.array([rates.rate_elastic_m3s, rates.rate_excitation_m3s,
                                         rates.rate_ionization_m3s, rates.excitation_threshold_ev])
        out[f"{name}_key"] = np.array(step_stream_key(seed, step), dtype=np.uint64)
        out[f"{name}_tally"] = np.array([tally.elastic, tally.excitation, tally.ionization,
                                         tally.suppressed])
        out[f"{name}_masses"] = np.array([sp.mass_kg for sp in store.species])
        print(name, tally)
    out["roles"] = np.array([ROLES.electron, ROLES.neutral, ROLES.ion])
    out["dt_s"] = np.array(CONSTS.dt_s)
    np.savez_compressed(os.path.join(HERE, "collision_kats.npz"), **out)


def gen_desk_criterion01(picmc):
    """The reference's own acceptance criterion 01 scenario
    (pkg/tests/test_acceptance.py:73-117): pkg/configs/desk.toml run to the
    ODE half-depletion step.  Records per-step diagnostics, the last rho and
    SHA-256 digests of the final stores (slot order) -- compact but exact."""
    import hashlib
    import math
    from dataclasses import replace

    from picmc.config import load_config
    from picmc.decomposition import merge_stores
    from picmc.harness import run_simulation

    cfg = load_config(os.path.join(REF, "configs", "desk.toml"))
    w_over_dx = cfg.densities_m3[2] / cfg.ppc0
    r = w_over_dx * cfg.collisions.rates.rate_ionization_m3s * cfg.consts.dt_s
    ne, nn, steps = float(cfg.ppc0), float(cfg.ppc0), 0
    while nn > 0.5 * cfg.ppc0:
        ev = ne * -math.expm1(-nn * r)
        nn -= ev
        ne += ev
        steps += 1
    cfg = replace(cfg, n_steps=steps, out_dir=None)
    box = {}

    def probe(step, st):
        if step == steps:
            box["rho"] = st["rho"].copy()
            box["final"] = merge_stores(st["stores"], st["partition"], cfg.grid)

    m = run_simulation(cfg, on_step=probe)
    flat = flatten_store(box["final"])
    digests = {k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest() for k, v in flat.items()}
    names = [s.name for s in cfg.species]
    np.savez_compressed(
        os.path.join(HERE, "run_desk_criterion01.npz"),
        steps=np.array(steps), ode_nn=np.array(nn),
        totals=np.array([[row[f"total_{n}"] for n in names] for row in m.diagnostics]),
        tallies=np.array([[row["elastic"], row["excitation"], row["ionization"], row["suppressed"]]
                          for row in m.diagnostics]),
        rho_last=box["rho"], digests=np.array(json.dumps(digests, sort_keys=True)))
    print("desk criterion 01:", steps, "steps", m.diagnostics[-1])


def gen_c1(picmc):
    """BASELINE config 1 (configs/c1_desk_ppc100.toml: the desk ionisation
    test at nc = 1000, ppc0 = 100, 100 steps, collisions on) run by the
    reference's own run_simulation.  Records every step's diagnostics row,
    the SHA-256 of every step's rho, the last rho and SHA-256 digests of the
    final stores in slot order (300K particles: digests keep the file small
    while the comparison stays bit-exact)."""
    import hashlib
    from dataclasses import replace

    from picmc.config import load_config
    from picmc.decomposition import merge_stores
    from picmc.harness import run_simulation

    root = os.path.dirname(os.path.dirname(HERE))
    cfg = load_config(os.path.join(root, "configs", "c1_desk_ppc100.toml"))
    cfg = replace(cfg, out_dir=None)
    box = {"rho_sha": []}

    def probe(step, st):
        box["rho_sha"].append(hashlib.sha256(np.ascontiguousarray(st["rho"]).tobytes()).hexdigest())
        if step == cfg.n_steps:
            box["rho"] = st["rho"].copy()
            box["final"] = merge_stores(st["stores"], st["partition"], cfg.grid)

    m = run_simulation(cfg, on_step=probe)
    flat = flatten_store(box["final"])
    digests = {k: hashlib.sha256(np.ascontiguousarray(v).tobytes()).hexdigest() for k, v in flat.items()}
    names = [s.name for s in cfg.species]
    np.savez_compressed(
        os.path.join(HERE, "run_c1_desk_ppc100.npz"),
        steps=np.array(cfg.n_steps),
        totals=np.array([[row[f"total_{n}"] for n in names] for row in m.diagnostics]),
        tallies=np.array([[row["elastic"], row["excitation"], row["ionization"], row["suppressed"]]
                          for row in m.diagnostics]),
        rho_sha=np.array(json.dumps(box["rho_sha"])),
        rho_last=box["rho"], digests=np.array(json.dumps(digests, sort_keys=True)))
    print("config 1:", cfg.n_steps, "steps", m.diagnostics[-1])


def raw_store(store, prefix):
    """Every array of a store, free space included (slot layout pinned)."""
    out = {}
    for isp in range(store.nsp):
        out[f"{prefix}sp{isp}_counts"] = store.counts(isp).copy()
        out[f"{prefix}sp{isp}_caps"] = store.caps(isp).copy()
        out[f"{prefix}sp{isp}_offs"] = store.offsets(isp).copy()
        for name, arr in store.data(isp).items():
            out[f"{prefix}sp{isp}_{name}"] = arr.copy()
    return out


def gen_mover_api(picmc):
    """The store-level mover API (pkg/src/picmc/mover.py) on a store with
    slack and tight capacities: mover_phase + resort per step (capacity
    doubling included), resort_collect's Movers, and the separable
    gather + push_velocity + push_position composition."""
    from picmc.core import CellSortedStore, Grid1D, PhysicalConstants, SpeciesDef
    from picmc.fields import gather_field
    from picmc.mover import mover_phase, push_position, push_velocity, resort, resort_collect
    from picmc.scheduler import Scheduler

    nc, ppc = 23, 6
    species = [SpeciesDef("q", -1.602176634e-19, 9.1093837015e-31),
               SpeciesDef("n", 0.0, 3.3e-27, nstep=3, track_transverse=True)]
    consts = PhysicalConstants(dt_s=4e-14)

    def fresh(seed):
        store = CellSortedStore(Grid1D.from_cells(nc, nc * 1e-5), species, initial_cap=ppc)
        rng = np.random.default_rng(seed)
        for isp in range(2):
            store.counts(isp)[:] = rng.integers(0, ppc + 1, size=nc)
            idx = store.live_indices(isp)
            d = store.data(isp)
            d["x"][idx] = rng.random(idx.size)
            for f in ("vx", "vy", "vz"):
                d[f][idx] = 1.3 * rng.standard_normal(idx.size)
            d["vx"][idx[::11]] = -0.0
            if "yp" in d:
                d["yp"][idx] = rng.standard_normal(idx.size)
        return store, rng

    store, rng = fresh(77)
    out = raw_store(store, "init_")
    steps = 6
    e_hist = []
    with Scheduler(workers=2, trace=False) as sched:
        for k in range(steps):
            e = 2e3 * rng.standard_normal(nc + 1)
            e_hist.append(e)
            mover_phase(store, e, consts, sched, grainsize=5)
            out[f"moved{k}"] = np.array(resort(store))
            out.update(raw_store(store, f"step{k}_"))
    out["e_hist"] = np.array(e_hist)
    out["steps"] = np.array(steps)

    # resort_collect alone: the Movers and the compacted store
    store, rng = fresh(78)
    out.update(raw_store(store, "cinit_"))
    for isp in range(2):
        push_position(store, isp)
    out.update(raw_store(store, "cpushed_"))
    for m in resort_collect(store):
        out[f"cmov{m.isp}_dest"] = m.dest_cell
        out[f"cmov{m.isp}_src_cell"] = m.src_cell
        out[f"cmov{m.isp}_src_slot"] = m.src_slot
        for name, v in m.fields.items():
            out[f"cmov{m.isp}_{name}"] = v
    out.update(raw_store(store, "collected_"))

    # separable composition on the charged species
    store, rng = fresh(79)
    out.update(raw_store(store, "vinit_"))
    e = 300.0 * rng.standard_normal(nc + 1)
    e_p = gather_field(e, store, store.grid)
    push_velocity(store, 0, e_p[0], consts)
    push_position(store, 0)
    out["v_e"] = e
    out["v_e_p0"] = e_p[0]
    out.update(raw_store(store, "vdone_"))
    out["dt_s"] = np.array(4e-14)
    out["nc"] = np.array(nc)
    np.savez_compressed(os.path.join(HERE, "mover_api.npz"), **out)


def gen_fields_api(picmc):
    """Store-level field functions (pkg/src/picmc/fields.py:55-236) on a
    store with slack: weighted partials over sub-ranges, stitch_rho, the
    wall-doubled deposit_charge and gather_field."""
    from picmc.core import CellSortedStore, Grid1D, PhysicalConstants, SpeciesDef
    from picmc.fields import deposit_charge, deposit_partials_range, gather_field, stitch_rho

    nc, ppc = 29, 7
    species = [SpeciesDef("e", -1.602176634e-19, 9.1093837015e-31),
               SpeciesDef("D+", 1.602176634e-19, 3.3435837483066354e-27),
               SpeciesDef("D", 0.0, 3.344494686676785e-27, track_transverse=True)]
    store = CellSortedStore(Grid1D.from_cells(nc, nc * 1e-5), species, initial_cap=ppc + 2)
    store.weights = [3.7e14, 2.9e14, 1.1e14]
    rng = np.random.default_rng(91)
    for isp in range(3):
        store.counts(isp)[:] = rng.integers(0, ppc + 1, size=nc)
        idx = store.live_indices(isp)
        d = store.data(isp)
        d["x"][idx] = rng.random(idx.size)
        d["x"][idx[::13]] = 0.0
        for f in ("vx", "vy", "vz"):
            d[f][idx] = rng.standard_normal(idx.size)
        if "yp" in d:
            d["yp"][idx] = rng.standard_normal(idx.size)
    consts = PhysicalConstants(dt_s=4e-14)
    out = raw_store(store, "store_")
    out["weights"] = np.array(store.weights)
    for lo, hi in ((0, nc), (5, 17), (28, 29)):
        left, right = deposit_partials_range(store, consts, lo, hi)
        out[f"dpr_{lo}_{hi}_left"], out[f"dpr_{lo}_{hi}_right"] = left, right
    left, right = deposit_partials_range(store, consts, 0, nc)
    out["stitch_periodic"] = stitch_rho(left, right, True)
    out["stitch_walls"] = stitch_rho(left, right, False)
    out["charge_periodic"] = deposit_charge(store, store.grid, consts, "periodic")
    out["charge_dirichlet"] = deposit_charge(store, store.grid, consts, "dirichlet")
    e = 1e3 * rng.standard_normal(nc + 1)
    out["gather_e"] = e
    for isp, v in gather_field(e, store, store.grid).items():
        out[f"gather_sp{isp}"] = v
    np.savez_compressed(os.path.join(HERE, "fields_api.npz"), **out)


if __name__ == "__main__":
    ref = import_reference()
    if sys.argv[1:] == ["c1"]:
        gen_c1(ref)
        sys.exit(0)
    gen_backend(ref)
    gen_resort(ref)
    gen_rng(ref)
    gen_init(ref)
    gen_runs(ref)
    gen_fields(ref)
    gen_mover_multistep(ref)
    gen_mover_api(ref)
    gen_fields_api(ref)
    gen_collision_runs(ref)
    gen_collision_kats(ref)
    gen_desk_criterion01(ref)
    gen_c1(ref)
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
