"""CPU: the oracle's collision pass and canonical-order run restatement
against the reference itself (golden fixtures from tests/golden/make_golden.py).

Bar: bit-exact -- particle stores in the reference's slot order, collision
tallies, totals, rho and E at every step.
"""

import numpy as np
import pytest

from conftest import bits_equal, load_golden
from golden_cfg import COLLISION_KATS, RUNS_ALL, cfg_from, host_species

ELEMENTARY_CHARGE = 1.602176634e-19


def kat_case(z, name):
    roles = tuple(int(v) for v in z["roles"])
    dt = float(z["dt_s"])
    w, r, m = z[f"{name}_weights"], z[f"{name}_rates"], z[f"{name}_masses"]
    sp = []
    for isp in range(3):
        d = {"cell": z[f"{name}_in_sp{isp}_cell"].astype(np.int32)}
        for f in ("x", "vx", "vy", "vz", "yp"):
            if f"{name}_in_sp{isp}_{f}" in z:
                d[f] = z[f"{name}_in_sp{isp}_{f}"]
        sp.append(d)
    # CONSTS of pkg/tests/test_collisions.py: dt = dx = 1
    prm = (w[roles[1]] / 1.0, dt, r[0], r[1], r[2], r[3] * ELEMENTARY_CHARGE, m[roles[0]], 1.0 / dt)
    return roles, prm, sp, int(z[f"{name}_nc"]), int(z[f"{name}_key"])


def assert_species_equal(got, z, prefix):
    for isp in range(3):
        for f in ("x", "vx", "vy", "vz", "yp"):
            k = f"{prefix}sp{isp}_{f}"
            if k in z:
                assert bits_equal(got[isp][f], z[k]), (k,)
        assert np.array_equal(np.asarray(got[isp]["cell"], dtype=np.int64), z[f"{prefix}sp{isp}_cell"])


@pytest.mark.parametrize("name", COLLISION_KATS)
def test_oracle_collision_phase_matches_reference(name):
    from oracle import oracle

    z = load_golden("collision_kats.npz")
    roles, prm, sp, nc, key = kat_case(z, name)
    tally, out = oracle.collision_phase(sp, roles, prm, key, nc)
    assert list(tally) == list(z[f"{name}_tally"])
    assert_species_equal(out, z, f"{name}_out_")


def test_collision_kats_cover_every_event_kind():
    z = load_golden("collision_kats.npz")
    t = np.array([z[f"{n}_tally"] for n in COLLISION_KATS]).sum(axis=0)
    assert np.all(t > 0), t  # elastic, excitation, ionization, suppressed


@pytest.mark.parametrize("name", RUNS_ALL)
def test_oracle_canonical_run_matches_reference(name):
    from oracle import oracle

    g = load_golden(f"{name}.npz")
    cfg = cfg_from(g)
    h = oracle.run_canonical(cfg, host_species(cfg))
    assert bits_equal(np.array(h["rho"]), g["rho"])
    assert bits_equal(np.array(h["e"]), g["e_field"])
    assert np.array_equal(np.array(h["totals"]), g["totals"])
    if "tallies" in g:
        assert np.array_equal(np.array(h["tallies"]), g["tallies"])
    assert_species_equal(h["species"], g, "")
