"""Property-based parity of the device mover against the oracle (hypothesis,
the reference's own property-testing tool, pkg/tests/test_rng.py etc.).

Random species mixes select every mover variant -- the split kernel (charged
+ neutral), the TMA-ring kernel (charged only), the quad kernel (Boris),
the LDG kernel (an inactive species) -- with random grids, densities, nstep,
transverse tracking, fields and particle boundaries.  Bar: particles, cells
and moved counts bit-exact; deposit bins exact vs the fixed-point
restatement; absorbed counts exact."""

import numpy as np
import pytest
from hypothesis import HealthCheck, assume, given, settings
from hypothesis import strategies as st

pytestmark = pytest.mark.gpu

KINDS = ["e", "ion", "neutral", "neutral_yp", "ion_yp", "inactive_ion"]


def _species(kinds, nsteps):
    from paper_2404_10270_b200 import SpeciesDef
    from paper_2404_10270_b200.core import DEUTERIUM_MASS, ELECTRON_MASS, ELEMENTARY_CHARGE

    out = []
    for k, (kind, ns) in enumerate(zip(kinds, nsteps)):
        name = f"s{k}"
        if kind == "e":
            out.append(SpeciesDef(name, -ELEMENTARY_CHARGE, ELECTRON_MASS, nstep=ns))
        elif kind == "ion":
            out.append(SpeciesDef(name, ELEMENTARY_CHARGE, DEUTERIUM_MASS, nstep=ns))
        elif kind == "ion_yp":
            out.append(SpeciesDef(name, ELEMENTARY_CHARGE, DEUTERIUM_MASS, nstep=ns, track_transverse=True))
        elif kind == "neutral":
            out.append(SpeciesDef(name, 0.0, DEUTERIUM_MASS, nstep=ns))
        elif kind == "neutral_yp":
            out.append(SpeciesDef(name, 0.0, DEUTERIUM_MASS, nstep=ns, track_transverse=True))
        else:
            out.append(SpeciesDef(name, ELEMENTARY_CHARGE, DEUTERIUM_MASS, nstep=ns, active_mover=False))
    return out


@settings(max_examples=60, deadline=None, suppress_health_check=list(HealthCheck))
@given(seed=st.integers(0, 2**31 - 1), nc=st.integers(8, 260), ppc=st.integers(1, 70),
       kinds=st.lists(st.sampled_from(KINDS), min_size=1, max_size=4),
       nstep=st.integers(1, 3), field=st.booleans(), absorbing=st.booleans(),
       boris=st.booleans(), steps=st.integers(1, 4), vscale=st.sampled_from([0.05, 0.6, 2.5]))
def test_mover_matches_oracle(cuda, seed, nc, ppc, kinds, nstep, field, absorbing, boris, steps, vscale):
    import torch

    from oracle import oracle
    from paper_2404_10270_b200 import Engine, Grid1D, PhysicalConstants, RunConfig
    from paper_2404_10270_b200.core import FlatSpecies

    assume(vscale * nstep * 7.0 < nc)  # stay inside the CFL bound (tested separately)
    species = _species(kinds, [nstep] * len(kinds))
    kw = dict(particle_boundary="absorbing", boundary="dirichlet") if absorbing else {}
    cfg = RunConfig(grid=Grid1D.from_cells(nc, nc * 1e-5), consts=PhysicalConstants(dt_s=4e-14),
                    species=species, temperatures_ev=[1.0] * len(species),
                    densities_m3=[1e21] * len(species), ppc0=ppc, n_steps=0, seed=seed,
                    field_solve=False, smoothing_passes=0,
                    b_field_t=(0.2, 0.1, 1.5) if boris else None, **kw)
    eng = Engine(cfg, device=cuda, check_every=0)
    rng = np.random.default_rng(seed)
    n = nc * ppc
    live = []
    for sp in species:
        vx = vscale * rng.standard_normal(n)
        vx[rng.random(n) < 0.03] = -0.0
        live.append(FlatSpecies(x=rng.random(n), vx=vx, vy=vscale * rng.standard_normal(n),
                                vz=vscale * rng.standard_normal(n),
                                yp=rng.standard_normal(n) if sp.track_transverse else None,
                                cell=np.repeat(np.arange(nc, dtype=np.int32), ppc)))
    eng.upload(live)
    code = 1 if absorbing else 0
    absorbed = np.zeros((len(species), 2), dtype=np.int64)
    moved = np.zeros(len(species), dtype=np.int64)
    for _ in range(steps):
        e = (5e3 * rng.standard_normal(nc + 1)) if field else np.zeros(nc + 1)
        eng.bins.zero_()
        eng.push(torch.from_numpy(e).to(cuda))
        eng.resort()
        eng.sync()
        nxt = []
        for k, (s, f) in enumerate(zip(eng.sp, live)):
            bt = bs = None
            if s.boris is not None:
                bt, bs = s.boris
            mv, removed, cfl = oracle.step_flat(s.kind, code, s.fnstep, s.kick_coef, e, nc, f.x, f.vx, f.vy,
                                                f.vz, f.yp, f.cell, bt, bs)
            assert cfl == -1
            moved[k] += mv
            absorbed[k, 0] += int((removed == 1).sum())
            absorbed[k, 1] += int((removed == 2).sum())
            keep = removed == 0
            nxt.append(FlatSpecies(*(None if a is None else a[keep].copy()
                                     for a in (f.x, f.vx, f.vy, f.vz, f.yp, f.cell))))
        live = nxt
        dev = eng.download()
        for k in range(len(species)):
            assert np.array_equal(oracle.canonical(dev[k].cell, dev[k].fields()),
                                  oracle.canonical(live[k].cell, live[k].fields())), (k, kinds)
        bins = eng.bins.cpu().numpy().view(np.uint64).reshape(max(eng.ndep, 1), 2, nc)
        for k, s in enumerate(eng.sp):
            if s.deposit < 0:
                continue
            R, C = oracle.deposit_fixed(live[k].x, live[k].cell, nc)
            assert np.array_equal(bins[s.deposit, 0], R) and np.array_equal(bins[s.deposit, 1], C), (k, kinds)
    assert np.array_equal(eng.absorbed, absorbed)
    assert np.array_equal(eng.moved, moved)
