"""Device engine vs the oracle: per-particle state bit-exact, deposit bins
exact against the oracle's fixed-point restatement and within tolerance of
the reference's sequential fp64 summation.

Tolerances (stated once, used below):
  per-particle x, vx, vy, vz, yp, cell ...... bit-exact
  moved / absorbed / surviving counts ........ exact
  raw partials L_s, R_s vs sequential fp64 ... |d| <= 1e-13 * max(1, |sum_cell|) (relative)
"""

import math

import numpy as np
import pytest

from conftest import bits_equal

pytestmark = pytest.mark.gpu

DEP_TOL = 1e-13


def _mk_config(nc=37, ppc0=20, species=None, **kw):
    from paper_2404_10270_b200 import Grid1D, PhysicalConstants, RunConfig, SpeciesDef
    from paper_2404_10270_b200.core import DEUTERIUM_MASS, ELECTRON_MASS, ELEMENTARY_CHARGE

    if species is None:
        species = [
            SpeciesDef("e", -ELEMENTARY_CHARGE, ELECTRON_MASS),
            SpeciesDef("D+", ELEMENTARY_CHARGE, DEUTERIUM_MASS - ELECTRON_MASS),
            SpeciesDef("D", 0.0, DEUTERIUM_MASS, nstep=3, track_transverse=True),
        ]
    base = dict(grid=Grid1D.from_cells(nc, nc * 1e-5), consts=PhysicalConstants(dt_s=4e-14),
                species=species, temperatures_ev=[20.0, 20.0, 1.0][: len(species)] + [1.0] * max(0, len(species) - 3),
                densities_m3=[1e21] * len(species), ppc0=ppc0, n_steps=5, seed=20260819,
                field_solve=False, smoothing_passes=0)
    base.update(kw)
    return RunConfig(**base)


def _random_flats(cfg, seed, vscale=0.7):
    from paper_2404_10270_b200.core import FlatSpecies

    rng = np.random.default_rng(seed)
    nc, ppc = cfg.grid.nc, cfg.ppc0
    out = []
    for sp in cfg.species:
        n = nc * ppc
        vx = vscale * rng.standard_normal(n)
        vx[rng.random(n) < 0.02] = -0.0
        out.append(FlatSpecies(
            x=rng.random(n), vx=vx, vy=vscale * rng.standard_normal(n),
            vz=vscale * rng.standard_normal(n),
            yp=rng.standard_normal(n) if sp.track_transverse else None,
            cell=np.repeat(np.arange(nc, dtype=np.int32), ppc),
        ))
    return out


def _oracle_kind(eng, k):
    return eng.sp[k].kind


def _run_oracle_step(eng, flats, e, bc):
    from oracle import oracle

    res = []
    for k, (s, f) in enumerate(zip(eng.sp, flats)):
        bt = bs = None
        if s.boris is not None:
            bt, bs = s.boris
        moved, removed, cfl = oracle.step_flat(s.kind, bc, s.fnstep, s.kick_coef, e, eng.nc, f.x, f.vx,
                                                f.vy, f.vz, f.yp, f.cell, bt, bs)
        res.append((moved, removed, cfl))
    return res


def _compare_arrays(dev, ref):
    for name, arr in ref.fields().items():
        assert bits_equal(dev.fields()[name], arr), name
    assert np.array_equal(dev.cell, ref.cell)


@pytest.mark.parametrize("with_field", [False, True])
@pytest.mark.parametrize("dense", [False, True])
def test_push_deposit_bitwise_vs_oracle(cuda, with_field, dense):
    """dense: 64 particles per cell over 300 cells, so charged species use
    the 1-byte compressed cell index (pb_species.cell8) -- multi-cell jumps
    across the periodic seam exercise its escapes."""
    import torch

    from oracle import oracle
    from paper_2404_10270_b200 import Engine

    cfg = _mk_config(nc=300, ppc0=64) if dense else _mk_config()
    eng = Engine(cfg, device=cuda, check_every=0)
    if dense:
        assert all(s.cell8 is not None for s in eng.sp if s.deposit >= 0)
    flats = _random_flats(cfg, seed=3, vscale=(18.0 if dense else 0.7))
    eng.upload(flats)
    rng = np.random.default_rng(11)
    for step in range(12):
        e = (3e3 * rng.standard_normal(eng.nc + 1)) if with_field else np.zeros(eng.nc + 1)
        et = torch.from_numpy(e).to(cuda)
        eng.bins.zero_()
        eng.push(et)
        eng.resort()
        res = _run_oracle_step(eng, flats, e, 0)
        dev = eng.download()
        eng.sync()
        for k in range(len(flats)):
            _compare_arrays(dev[k], flats[k])
            assert res[k][2] == -1
        # deposit bins: exact vs the fixed-point restatement, tolerance vs fp64
        bins = eng.bins.cpu().numpy().view(np.uint64).reshape(eng.ndep, 2, eng.nc)
        d = 0
        for k, s in enumerate(eng.sp):
            if s.deposit < 0:
                continue
            R, C = oracle.deposit_fixed(flats[k].x, flats[k].cell, eng.nc)
            assert np.array_equal(bins[d, 0], R) and np.array_equal(bins[d, 1], C)
            lf, rf = oracle.fixed_to_raw(R, C)
            ls, rs = oracle.deposit_seq(flats[k].x, flats[k].cell, eng.nc)
            # relative per cell, floored at one particle
            # weight: the fixed point quantises each x to 2^-48 (<= 2^-49 error),
            # so a cell's sum is within count * 2^-49 ~ 3.6e-15 * |sum| of fp64
            assert np.all(np.abs(lf - ls) <= DEP_TOL * np.maximum(1.0, np.abs(ls)))
            assert np.all(np.abs(rf - rs) <= DEP_TOL * np.maximum(1.0, np.abs(rs)))
            d += 1


def test_moved_counts_exact(cuda):
    import torch

    from paper_2404_10270_b200 import Engine

    cfg = _mk_config()
    eng = Engine(cfg, device=cuda, check_every=0)
    flats = _random_flats(cfg, seed=4)
    eng.upload(flats)
    e = np.zeros(eng.nc + 1)
    eng.push(torch.from_numpy(e).to(cuda))
    pass
    eng.sync()
    res = _run_oracle_step(eng, flats, e, 0)
    for k in range(len(flats)):
        assert eng.moved[k] == res[k][0]


def test_epilogue_matches_oracle_bitwise(cuda):
    from oracle import oracle
    from paper_2404_10270_b200 import Engine

    for boundary in ("periodic", "dirichlet"):
        cfg = _mk_config(boundary=boundary)
        eng = Engine(cfg, device=cuda, check_every=0)
        flats = eng.download()
        raw = []
        for k, s in enumerate(eng.sp):
            if s.deposit >= 0:
                R, C = oracle.deposit_fixed(flats[k].x, flats[k].cell, eng.nc)
                raw.extend(oracle.fixed_to_raw(R, C))
        raw = np.stack(raw).reshape(eng.ndep, 2, eng.nc)
        left, right, rho = oracle.rho_from_raw(raw, eng.coef_dep, eng.nc, boundary == "periodic")
        rho_dev = eng.density().cpu().numpy()
        assert bits_equal(rho_dev, rho)
        assert bits_equal(eng.left.cpu().numpy(), left)
        assert bits_equal(eng.right.cpu().numpy(), right)


@pytest.mark.parametrize("dense", [False, True])
def test_absorbing_walls_counts_and_survivors(cuda, dense):
    """dense: the compressed cell index is in use, so compaction must carry
    it along with the particles it moves into the holes."""
    import torch

    from oracle import oracle
    from paper_2404_10270_b200 import Engine

    if dense:
        cfg = _mk_config(nc=200, ppc0=48, particle_boundary="absorbing", boundary="dirichlet")
    else:
        cfg = _mk_config(particle_boundary="absorbing", boundary="dirichlet")
    eng = Engine(cfg, device=cuda, check_every=0)
    assert dense == any(s.cell8 is not None for s in eng.sp)
    flats = _random_flats(cfg, seed=7, vscale=(9.0 if dense else 2.5))
    eng.upload(flats)
    live = [f for f in flats]
    total_abs = np.zeros((3, 2), dtype=np.int64)
    for step in range(6):
        e = np.zeros(eng.nc + 1)
        eng.push(torch.from_numpy(e).to(cuda))
        eng.resort()
        pass
        eng.sync()
        res = _run_oracle_step(eng, live, e, 1)
        nxt = []
        for k, f in enumerate(live):
            removed = res[k][1]
            total_abs[k, 0] += int((removed == 1).sum())
            total_abs[k, 1] += int((removed == 2).sum())
            keep = removed == 0
            from paper_2404_10270_b200.core import FlatSpecies
            nxt.append(FlatSpecies(*(None if a is None else a[keep].copy()
                                     for a in (f.x, f.vx, f.vy, f.vz, f.yp, f.cell))))
        live = nxt
        dev = eng.download()
        for k in range(3):
            assert dev[k].n == live[k].n
            a = oracle.canonical(dev[k].cell, dev[k].fields())
            b = oracle.canonical(live[k].cell, live[k].fields())
            assert np.array_equal(a, b)
        assert np.array_equal(eng.absorbed, total_abs)
    assert total_abs.sum() > 0


def test_boris_bitwise_and_speed_conservation(cuda):
    import torch

    from paper_2404_10270_b200 import Engine

    cfg = _mk_config(b_field_t=(0.3, 0.0, 2.0))
    eng = Engine(cfg, device=cuda, check_every=0)
    flats = _random_flats(cfg, seed=9, vscale=0.05)
    eng.upload(flats)
    e = np.zeros(eng.nc + 1)
    speed0 = [np.sqrt(f.vx ** 2 + f.vy ** 2 + f.vz ** 2) for f in flats]
    for _ in range(20):
        eng.push(torch.from_numpy(e).to(cuda))
        eng.resort()
        _run_oracle_step(eng, flats, e, 0)
    dev = eng.download()
    for k in range(3):
        _compare_arrays(dev[k], flats[k])
    # pure magnetic rotation conserves |v| to rounding (20 steps)
    for k in (0, 1):
        sp = np.sqrt(dev[k].vx ** 2 + dev[k].vy ** 2 + dev[k].vz ** 2)
        assert np.allclose(sp, speed0[k], rtol=1e-13, atol=0)
    assert not bits_equal(dev[0].vy, speed0[0])  # it did rotate


def test_cfl_violation_raises(cuda):
    import torch

    from paper_2404_10270_b200 import CflViolation, Engine

    cfg = _mk_config(nc=8, ppc0=2)
    eng = Engine(cfg, device=cuda, check_every=0)
    flats = _random_flats(cfg, seed=1, vscale=0.0)
    flats[2].vx[5] = 9.0 / 3.0  # neutral, nstep 3 -> displacement 9 cells on nc=8
    eng.upload(flats)
    eng.push(torch.zeros(9, dtype=torch.float64, device=cuda))
    pass
    with pytest.raises(CflViolation, match="whole domain"):
        eng.sync()


def test_free_streaming_exact_1000_steps(cuda):
    """Criterion 08 (pkg/tests/test_acceptance.py:355-411) on the device:
    dyadic positions/velocities, E = 0, closed form with zero tolerance."""
    from paper_2404_10270_b200 import Engine, SpeciesDef
    from paper_2404_10270_b200.core import DEUTERIUM_MASS, ELECTRON_MASS, ELEMENTARY_CHARGE, FlatSpecies

    M = 1 << 20
    nc, ppc, n_steps = 32, 4, 1000
    species = [SpeciesDef("e", -ELEMENTARY_CHARGE, ELECTRON_MASS),
               SpeciesDef("g", 0.0, DEUTERIUM_MASS, nstep=3)]
    cfg = _mk_config(nc=nc, ppc0=ppc, species=species, temperatures_ev=[1.0, 1.0],
                     densities_m3=[1e21, 1e21], sort_every=97)
    eng = Engine(cfg, device=cuda, check_every=0)
    rng = np.random.default_rng(41)
    flats, starts, tag = [], {}, 0
    for isp in range(2):
        xs, vs, tags, cells = [], [], [], []
        for j in range(nc):
            for _ in range(ppc):
                xi = int(rng.integers(0, M))
                vi = int(rng.integers(-(1 << 14), 1 << 14)) or 7
                xs.append(xi / M)
                vs.append(vi / M)
                tags.append(float(tag))
                cells.append(j)
                starts[tag] = (isp, j * M + xi, vi)
                tag += 1
        n = len(xs)
        flats.append(FlatSpecies(np.array(xs), np.array(vs), np.zeros(n), np.array(tags), None,
                                 np.array(cells, dtype=np.int32)))
    eng.upload(flats)
    for _ in range(n_steps):
        eng.push()
        eng.resort()
        eng.step_index += 1
    pass
    eng.sync()
    dev = eng.download()
    checked = 0
    for isp in range(2):
        nstep = species[isp].nstep
        for x, vx, t, j in zip(dev[isp].x, dev[isp].vx, dev[isp].vz, dev[isp].cell):
            isp0, pos0, vi = starts[int(t)]
            assert isp0 == isp
            assert int(j) * M + int(x * M) == (pos0 + n_steps * nstep * vi) % (nc * M)
            assert vx == vi / M
            checked += 1
    assert checked == 2 * nc * ppc


def test_sort_by_cell_preserves_particles(cuda):
    import torch

    from oracle import oracle
    from paper_2404_10270_b200 import Engine

    cfg = _mk_config(nc=200, ppc0=50)
    eng = Engine(cfg, device=cuda, check_every=0)
    flats = _random_flats(cfg, seed=12, vscale=3.0)
    eng.upload(flats)
    for _ in range(3):
        eng.push(torch.zeros(eng.nc + 1, dtype=torch.float64, device=cuda))
    before = eng.download()
    eng.sort_by_cell()
    after = eng.download()
    for b, a in zip(before, after):
        assert np.all(np.diff(a.cell) >= 0)
        assert np.array_equal(oracle.canonical(b.cell, b.fields()), oracle.canonical(a.cell, a.fields()))


def test_device_init_positions_bitexact(cuda):
    from paper_2404_10270_b200 import Engine
    from paper_2404_10270_b200.core import init_species_host

    cfg = _mk_config(nc=300, ppc0=16)
    eng = Engine(cfg, device=cuda, init="device", check_every=0)
    dev = eng.download()
    for k in range(3):
        host = init_species_host(cfg, k)
        assert bits_equal(dev[k].x, host.x)
        assert np.array_equal(dev[k].cell, host.cell)
        for f in ("vx", "vy", "vz"):
            np.testing.assert_allclose(getattr(dev[k], f), getattr(host, f), rtol=1e-12, atol=1e-300)


def test_step_deposit_is_order_and_sort_independent(cuda):
    from paper_2404_10270_b200 import Engine

    hist = {}
    for sort_every in (0, 3):
        cfg = _mk_config(nc=500, ppc0=40, sort_every=sort_every, field_solve=True, smoothing_passes=1)
        eng = Engine(cfg, device=cuda, check_every=0)
        h = []
        for _ in range(10):
            rho, _ = eng.step()
            h.append(rho.cpu().numpy().copy())
        hist[sort_every] = h
    for a, b in zip(hist[0], hist[3]):
        assert bits_equal(a, b)


def test_large_c2_shape_conservation(cuda):
    """Full-size property check at config 2's per-species shape (nc=100K,
    ppc=100): counts conserved and every particle deposited exactly once."""
    import torch

    from paper_2404_10270_b200 import Engine

    cfg = _mk_config(nc=100_000, ppc0=100, max_store_mb=65536)
    eng = Engine(cfg, device=cuda, init="device", check_every=0)
    for _ in range(5):
        eng.step()
    eng.sync()
    bins = eng.bins.cpu().numpy().view(np.uint64).reshape(eng.ndep, 2, eng.nc)
    assert int(bins[:, 1].sum()) == 2 * 10_000_000
    dev = eng.download()
    for f in dev:
        assert f.n == 10_000_000
        assert np.all((f.x >= 0.0) & (f.x < 1.0))
        assert np.all((f.cell >= 0) & (f.cell < eng.nc))
    # the packed counts of the fixed-point bins equal the per-cell histogram
    counts = np.bincount(dev[0].cell, minlength=eng.nc)
    assert np.array_equal(bins[0, 1], counts.astype(np.uint64))


@pytest.mark.parametrize("case", ["periodic", "sorted", "absorbing", "field"])
def test_graph_replay_matches_eager_steps(cuda, case):
    """CUDA-graph replay (two steps per graph; field-free runs overlap the
    density epilogue with the push on a side stream; graphs cached per sort
    buffer state) leaves particles, rho and tallies bitwise equal to eager
    steps."""
    from paper_2404_10270_b200 import Engine

    kw = {}
    if case == "sorted":
        kw["sort_every"] = 3
    elif case == "absorbing":
        kw.update(particle_boundary="absorbing", boundary="dirichlet")
    elif case == "field":
        kw.update(field_solve=True, smoothing_passes=1)
    cfg = _mk_config(nc=64, ppc0=24, **kw)
    flats = _random_flats(cfg, 5, vscale=0.4)
    a = Engine(cfg, device=cuda, check_every=0)
    b = Engine(cfg, device=cuda, check_every=0)
    a.upload(flats)
    b.upload(flats)
    b.prepare_graphs(40)
    steps = 13
    for _ in range(steps):
        a.step()
    b.replay(steps)
    a.sync()
    b.sync()
    assert bits_equal(a.rho.cpu().numpy(), b.rho.cpu().numpy())
    assert np.array_equal(a.moved, b.moved) and np.array_equal(a.absorbed, b.absorbed)
    fa, fb = a.download(), b.download()
    from oracle import oracle
    for x, y in zip(fa, fb):
        assert np.array_equal(oracle.canonical(x.cell, x.fields()), oracle.canonical(y.cell, y.fields()))
    # without sorting the slot order is the same too -- except after
    # absorbing-wall compaction, whose hole list is filled in the (arbitrary)
    # order the mover's warps recorded the holes
    if case not in ("sorted", "absorbing"):
        for x, y in zip(fa, fb):
            for k, v in x.fields().items():
                assert bits_equal(v, y.fields()[k])
    # and the bins the next density will read agree
    assert np.array_equal(a.bins.cpu().numpy(), b.bins.cpu().numpy())
    assert len(b.graphs) >= 2


@pytest.mark.parametrize("group", [1, 4])
@pytest.mark.parametrize("sort_every", [0, 3, 7])
def test_run_pipelined_matches_eager_steps(cuda, sort_every, group):
    """The overlapped host loop (H2D of each step's E, D2H of each step's rho
    one block late, blocks of `group` steps as one graph) delivers exactly
    the eager steps' rho sequence and leaves the same particles."""
    import torch

    from paper_2404_10270_b200 import Engine

    cfg = _mk_config(nc=48, ppc0=16, sort_every=sort_every)
    flats = _random_flats(cfg, 11, vscale=0.3)
    rng = np.random.default_rng(3)
    steps = 19
    es = [torch.from_numpy(2e4 * rng.standard_normal(cfg.grid.nc + 1)).pin_memory() for _ in range(steps)]
    a = Engine(cfg, device=cuda, check_every=0)
    b = Engine(cfg, device=cuda, check_every=0)
    a.upload(flats)
    b.upload(flats)
    want = []
    for k in range(steps):
        rho, _ = a.step(e_ext=es[k].to(cuda))
        want.append(rho.cpu().numpy().copy())
    got = {}
    n = b.run_pipelined(steps, e_source=lambda k: es[k], group=group,
                        on_result=lambda k, r: got.__setitem__(k, r.numpy().copy()))
    assert n == steps and sorted(got) == list(range(steps))
    for k in range(steps):
        assert bits_equal(got[k], want[k]), k
    from oracle import oracle
    for x, y in zip(a.download(), b.download()):
        assert np.array_equal(oracle.canonical(x.cell, x.fields()), oracle.canonical(y.cell, y.fields()))
    assert any(isinstance(k, tuple) and k[0] == "pipe" for k in b.graphs)


@pytest.mark.parametrize("with_input", [False, True])
def test_prepare_pipe_graphs_covers_run(cuda, with_input):
    """prepare_pipe_graphs captures every graph run_pipelined needs across
    sorts (so a timed loop never captures), and the run still matches eager."""
    import torch

    from paper_2404_10270_b200 import Engine

    cfg = _mk_config(nc=40, ppc0=12, sort_every=4)
    flats = _random_flats(cfg, 5, vscale=0.3)
    e_host = torch.zeros(cfg.grid.nc + 1, dtype=torch.float64).pin_memory()
    src = (lambda k: e_host) if with_input else None
    a = Engine(cfg, device=cuda, check_every=0)
    b = Engine(cfg, device=cuda, check_every=0)
    a.upload(flats)
    b.upload(flats)
    b.prepare_pipe_graphs(with_input, group=3)
    n0 = len(b.graphs)
    assert n0 > 0
    got = {}
    b.run_pipelined(30, e_source=src, group=3, on_result=lambda k, r: got.__setitem__(k, r.numpy().copy()))
    assert len(b.graphs) == n0
    for k in range(30):
        rho, _ = a.step(e_ext=e_host.to(cuda) if with_input else None)
        assert bits_equal(got[k], rho.cpu().numpy()), k


@pytest.mark.parametrize("group", [1, 3, 4])
def test_run_pipelined_field_solve_absorbing(cuda, group):
    """Field-solve + absorbing walls + cell sorts through the pipelined loop
    (graphs of `group` steps, serial density -> Poisson -> E -> push ->
    compaction; sorts bounded by the device live count) deliver the eager
    steps' rho sequence bit for bit."""
    from paper_2404_10270_b200 import Engine

    cfg = _mk_config(nc=64, ppc0=16, field_solve=True, smoothing_passes=1, boundary="dirichlet",
                     particle_boundary="absorbing", phi_left=2.0, phi_right=-1.0, sort_every=5)
    flats = _random_flats(cfg, 13, vscale=0.4)
    a = Engine(cfg, device=cuda, check_every=0)
    b = Engine(cfg, device=cuda, check_every=0)
    a.upload(flats)
    b.upload(flats)
    steps = 14
    want, want_n = [], []
    for _ in range(steps):
        rho, _ = a.step()
        want.append(rho.cpu().numpy().copy())
        want_n.append([int(v) for v in a.totals()])  # live counts after the step's compaction
    got, got_n = {}, {}
    b.run_pipelined(steps, group=group, on_result=lambda k, r: got.__setitem__(k, r.numpy().copy()),
                    on_counts=lambda k, c: got_n.__setitem__(k, [int(v) for v in c]))
    for k in range(steps):
        assert bits_equal(got[k], want[k]), k
        assert got_n[k] == want_n[k], (k, got_n[k], want_n[k])
    a.sync()
    b.sync()
    assert np.array_equal(a.absorbed, b.absorbed) and a.absorbed.sum() > 0
    from oracle import oracle
    for x, y in zip(a.download(), b.download()):
        assert np.array_equal(oracle.canonical(x.cell, x.fields()), oracle.canonical(y.cell, y.fields()))


@pytest.mark.parametrize("replay", [False, True])
def test_field_split_matches_serial_cycle(cuda, replay):
    """Field-solve steps with the neutral push overlapped with the field
    pipeline (the multi-GPU default) give bitwise the serial cycle's
    particles, rho and tallies, eager and graph-replayed."""
    from oracle import oracle
    from paper_2404_10270_b200 import Engine

    cfg = _mk_config(nc=64, ppc0=24, field_solve=True, smoothing_passes=1)
    flats = _random_flats(cfg, 21, vscale=0.4)
    a = Engine(cfg, device=cuda, check_every=0)
    b = Engine(cfg, device=cuda, check_every=0)
    a.field_split, b.field_split = False, True
    a.upload(flats)
    b.upload(flats)
    assert b._field_split()[0] and not a._field_split()[0]
    for _ in range(9):
        a.step()
    if replay:
        b.replay(9)
    else:
        for _ in range(9):
            b.step()
    a.sync()
    b.sync()
    assert bits_equal(a.rho.cpu().numpy(), b.rho.cpu().numpy())
    assert bits_equal(a.e.cpu().numpy(), b.e.cpu().numpy())
    assert np.array_equal(a.moved, b.moved)
    for x, y in zip(a.download(), b.download()):
        assert np.array_equal(oracle.canonical(x.cell, x.fields()), oracle.canonical(y.cell, y.fields()))


def test_boris_exb_drift(cuda):
    """Config-4 physics known answer: electrons starting at
    rest in uniform E_x and B_z drift at v = E x B / B^2, i.e. vy averages to
    -E_x/B_z (grid units: * dt/dx) over whole gyro-periods, with no net x
    drift."""
    import math

    import torch

    from paper_2404_10270_b200 import Engine, SpeciesDef
    from paper_2404_10270_b200.core import ELECTRON_MASS, ELEMENTARY_CHARGE

    bz, ex, dt, dx = 2.0, 1.0e4, 4e-14, 1e-5
    cfg = _mk_config(nc=64, ppc0=8, species=[SpeciesDef("e", -ELEMENTARY_CHARGE, ELECTRON_MASS)],
                     temperatures_ev=[0.0], densities_m3=[1e21], b_field_t=(0.0, 0.0, bz))
    eng = Engine(cfg, device=cuda, check_every=0)
    e = torch.full((eng.nc + 1,), ex, dtype=torch.float64, device=cuda)
    period = 2.0 * math.pi * ELECTRON_MASS / (ELEMENTARY_CHARGE * bz) / dt  # steps per gyration
    steps = int(round(10 * period))
    vy_sum = torch.zeros(eng.sp[0].n, dtype=torch.float64, device=cuda)
    for _ in range(steps):
        eng.push(e)
        vy_sum += eng.sp[0].arr["vy"][: eng.sp[0].n]
    eng.sync()
    vy_mean = float(vy_sum.mean()) / steps
    want = -(ex / bz) * dt / dx
    assert abs(vy_mean - want) <= 0.02 * abs(want), (vy_mean, want)
    vx_mean = float(eng.sp[0].arr["vx"][: eng.sp[0].n].mean())
    assert abs(vx_mean) <= 2.5 * abs(want)  # bounded gyration, no secular x motion


@pytest.mark.parametrize("bc", ["periodic", "absorbing"])
def test_charged_only_ring_bitwise_vs_oracle(cuda, bc):
    """Charged-only launches take the per-warp TMA ring kernel (k_push_ring):
    particles, cells and deposit bins bit-exact vs the oracle, including
    partial slices (n = 3700 per species) and absorbed particles."""
    import torch

    from oracle import oracle
    from paper_2404_10270_b200 import Engine, SpeciesDef
    from paper_2404_10270_b200.core import DEUTERIUM_MASS, ELECTRON_MASS, ELEMENTARY_CHARGE

    species = [SpeciesDef("e", -ELEMENTARY_CHARGE, ELECTRON_MASS),
               SpeciesDef("D+", ELEMENTARY_CHARGE, DEUTERIUM_MASS - ELECTRON_MASS)]
    kw = dict(particle_boundary="absorbing", boundary="dirichlet") if bc == "absorbing" else {}
    cfg = _mk_config(nc=100, ppc0=37, species=species, temperatures_ev=[20.0, 20.0],
                     densities_m3=[1e21, 1e21], **kw)
    eng = Engine(cfg, device=cuda, check_every=0)
    assert all(s.cell8 is None for s in eng.sp)
    flats = _random_flats(cfg, seed=13, vscale=1.5)
    eng.upload(flats)
    live = list(flats)
    rng = np.random.default_rng(4)
    code = 1 if bc == "absorbing" else 0
    for _ in range(8):
        e = 3e3 * rng.standard_normal(eng.nc + 1)
        eng.bins.zero_()
        eng.push(torch.from_numpy(e).to(cuda))
        eng.resort()
        eng.sync()
        res = _run_oracle_step(eng, live, e, code)
        from paper_2404_10270_b200.core import FlatSpecies
        nxt = []
        for k, f in enumerate(live):
            keep = res[k][1] == 0
            nxt.append(FlatSpecies(*(None if a_ is None else a_[keep].copy()
                                     for a_ in (f.x, f.vx, f.vy, f.vz, f.yp, f.cell))))
        live = nxt
        dev = eng.download()
        for k in range(2):
            a_ = oracle.canonical(dev[k].cell, dev[k].fields())
            b_ = oracle.canonical(live[k].cell, live[k].fields())
            assert np.array_equal(a_, b_)
        bins = eng.bins.cpu().numpy().view(np.uint64).reshape(eng.ndep, 2, eng.nc)
        for k in range(2):
            R, C = oracle.deposit_fixed(live[k].x, live[k].cell, eng.nc)
            assert np.array_equal(bins[k, 0], R) and np.array_equal(bins[k, 1], C)
    if bc == "absorbing":
        assert eng.absorbed.sum() > 0


def test_full_c2_sampled_particles_bitwise_vs_oracle(cuda):
    """Config 2 at full size (30M particles, device init, the production
    graph-replayed split mover): with E = 0 every particle evolves on its own,
    so a random sample of 50K slots per species, pushed by the oracle from the
    same initial state, must match the GPU bit for bit after 12 steps
    (no sorting, so slots keep their particle); every particle is deposited
    exactly once."""
    import torch

    from oracle import oracle
    from paper_2404_10270_b200 import Engine

    cfg = _mk_config(nc=100_000, ppc0=100, max_store_mb=65536, sort_every=0)
    eng = Engine(cfg, device=cuda, init="device", check_every=0)
    rng = np.random.default_rng(2024)
    samples = []
    for s in eng.sp:
        idx = torch.from_numpy(np.sort(rng.choice(s.n, 50_000, replace=False))).to(cuda)
        init = {f: t.index_select(0, idx).cpu().numpy() for f, t in s.arr.items()}
        init["cell"] = s.cell.index_select(0, idx).cpu().numpy()
        samples.append((idx, init))
    eng.prepare_graphs(40)
    eng.replay(12)
    eng.sync()
    e = np.zeros(eng.nc + 1)
    for s, (idx, st) in zip(eng.sp, samples):
        yp = st.get("yp")
        for _ in range(12):
            _, _, cfl = oracle.step_flat(s.kind, 0, s.fnstep, s.kick_coef, e, eng.nc, st["x"], st["vx"],
                                         st["vy"], st["vz"], yp, st["cell"])
            assert cfl == -1
        for f, t in s.arr.items():
            assert bits_equal(t.index_select(0, idx).cpu().numpy(), st[f]), (s.name, f)
        assert np.array_equal(s.cell.index_select(0, idx).cpu().numpy(), st["cell"]), s.name
    bins = eng.bins.cpu().numpy().view(np.uint64).reshape(eng.ndep, 2, eng.nc)
    assert int(bins[:, 1].sum()) == 2 * 10_000_000


def test_full_c4_sampled_particles_bitwise_vs_oracle(cuda):
    """Config 4 at full size (100M particles, Boris push with the oblique B,
    field solve): each step's E is taken from the engine and a 30K-slot
    sample per species is pushed by the oracle with it; the GPU's particles
    must match bit for bit after every step."""
    import os

    import torch

    from oracle import oracle
    from paper_2404_10270_b200 import Engine, load_config

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cfg = load_config(os.path.join(root, "configs", "c4_sol_boris.toml"))
    eng = Engine(cfg, device=cuda, init="device", check_every=0)
    assert any(s.boris is not None for s in eng.sp)
    rng = np.random.default_rng(4)
    samples = []
    for s in eng.sp:
        idx = torch.from_numpy(np.sort(rng.choice(s.n, 30_000, replace=False))).to(cuda)
        st = {f: t.index_select(0, idx).cpu().numpy() for f, t in s.arr.items()}
        st["cell"] = s.cell.index_select(0, idx).cpu().numpy()
        samples.append((idx, st))
    for _ in range(4):
        eng.step()
        e = eng.e.cpu().numpy()
        for s, (idx, st) in zip(eng.sp, samples):
            bt, bs = s.boris if s.boris is not None else (None, None)
            _, _, cfl = oracle.step_flat(s.kind, 0, s.fnstep, s.kick_coef, e, eng.nc, st["x"], st["vx"],
                                         st["vy"], st["vz"], st.get("yp"), st["cell"], bt, bs)
            assert cfl == -1
            for f, t in s.arr.items():
                assert bits_equal(t.index_select(0, idx).cpu().numpy(), st[f]), (s.name, f)
            assert np.array_equal(s.cell.index_select(0, idx).cpu().numpy(), st["cell"]), s.name
    eng.sync()


def test_full_c5_sampled_particles_bitwise_vs_oracle(cuda):
    """Config 5 at full size (1M cells, 1B particles in ~40 GB of HBM, E = 0):
    a 20K-slot sample per species pushed by the oracle matches the GPU bit for
    bit after 3 graph-replayed steps, and every particle is deposited once."""
    import os

    import torch

    from oracle import oracle
    from paper_2404_10270_b200 import Engine, load_config

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cfg = load_config(os.path.join(root, "configs", "c5_weak_1m.toml"))
    eng = Engine(cfg, device=cuda, init="device", check_every=0)
    rng = np.random.default_rng(5)
    samples = []
    for s in eng.sp:
        idx = torch.from_numpy(np.sort(rng.choice(s.n, 20_000, replace=False))).to(cuda)
        st = {f: t.index_select(0, idx).cpu().numpy() for f, t in s.arr.items()}
        st["cell"] = s.cell.index_select(0, idx).cpu().numpy()
        samples.append((idx, st))
    eng.prepare_graphs(10)
    eng.replay(3)
    eng.sync()
    e = np.zeros(eng.nc + 1)
    for s, (idx, st) in zip(eng.sp, samples):
        for _ in range(3):
            oracle.step_flat(s.kind, 0, s.fnstep, s.kick_coef, e, eng.nc, st["x"], st["vx"], st["vy"],
                             st["vz"], st.get("yp"), st["cell"])
        for f, t in s.arr.items():
            got = t.index_select(0, idx).cpu().numpy()
            bad = np.nonzero(got.view(np.uint64) != st[f].view(np.uint64))[0]
            assert bad.size == 0, (s.name, f, bad.size, idx[bad[:5]].tolist(), got[bad[:5]], st[f][bad[:5]])
        assert np.array_equal(s.cell.index_select(0, idx).cpu().numpy(), st["cell"]), s.name
    bins = eng.bins.cpu().numpy().view(np.uint64).reshape(eng.ndep, 2, eng.nc)
    assert int(bins[:, 1].sum()) == sum(s.n for s in eng.sp if s.deposit >= 0)
    del eng
    torch.cuda.empty_cache()


@pytest.mark.parametrize("bc", ["periodic", "dirichlet"])
@pytest.mark.parametrize("passes", [0, 1])
def test_one_kernel_density_matches_two_kernel_epilogue(cuda, bc, passes):
    """Serial field-solve cycle: the one-launch epilogue (pb_rho_epilogue)
    with the bins cleared by the E kernel gives bitwise the two-launch
    pb_density_step cycle -- rho, rho_s, phi, E, partials, both bin sets and
    every particle -- eager and graph-replayed."""
    from oracle import oracle
    from paper_2404_10270_b200 import Engine

    kw = dict(field_solve=True, smoothing_passes=passes, boundary=bc, phi_left=1.5, phi_right=-0.5)
    if bc == "dirichlet":
        kw["particle_boundary"] = "absorbing"
    cfg = _mk_config(nc=3000, ppc0=4, **kw)
    flats = _random_flats(cfg, 19, vscale=0.45)
    a = Engine(cfg, device=cuda, check_every=0)
    b = Engine(cfg, device=cuda, check_every=0)
    a.density_one, b.density_one = False, True
    a.upload(flats)
    b.upload(flats)
    for _ in range(3):
        a.step()
        b.step()
    b.prepare_graphs(40)
    for _ in range(6):
        a.step()
    b.replay(6)
    a.sync()
    b.sync()
    for name in ("rho", "rho_s", "phi", "e", "left", "right"):
        assert bits_equal(getattr(a, name).cpu().numpy(), getattr(b, name).cpu().numpy()), name
    assert np.array_equal(a.moved, b.moved) and np.array_equal(a.absorbed, b.absorbed)
    assert np.array_equal(a.bins_pp[0].cpu().numpy(), b.bins_pp[0].cpu().numpy())
    assert np.array_equal(a.bins_pp[1].cpu().numpy(), b.bins_pp[1].cpu().numpy())
    for x, y in zip(a.download(), b.download()):
        assert np.array_equal(oracle.canonical(x.cell, x.fields()), oracle.canonical(y.cell, y.fields()))
