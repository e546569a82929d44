"""CPU: accuracy of the closed-form scan Poisson solve (csrc/fields.cu,
DESIGN.md 3.3) in plain fp64 -- a NumPy restatement of its structure (512-
unknown tiles, fp64 tile sums and in-tile running sums, tile prefixes, the
Green's-function combine, the periodic mean and shift in closed form)
against the reference's elimination (_thomas_unit, pkg/src/picmc/fields.py:
138-202) carried out in long double.  The device kernels are held to the
reference's fp64 serial solve on the GPU (tests/test_harness_gpu.py); this
pins the algorithm's own error: ~1e-14 of max|phi| at 1e5 unknowns for noise,
smooth and sheath-shaped densities."""

import numpy as np
import pytest

TILE = 512


def _closed_form(rho, scale, periodic, pl=0.0, pr=0.0):
    nc = len(rho) - 1
    n = nc - 1
    a = -rho[1:nc] * scale
    if not periodic:
        a = a.copy()
        a[0] -= pl
        a[n - 1] -= pr
    k1 = np.arange(1, n + 1, dtype=np.float64)
    S = np.empty(n)
    Z = np.empty(n)
    ps = pz = 0.0
    for b in range(0, n, TILE):  # tile prefix + in-tile running sums
        s_t, z_t = a[b:b + TILE], k1[b:b + TILE] * a[b:b + TILE]
        S[b:b + TILE] = ps + np.cumsum(s_t)
        Z[b:b + TILE] = pz + np.cumsum(z_t)
        ps, pz = ps + s_t.sum(), pz + z_t.sum()
    x = -(Z + k1 * ((ps - S) - pz / (n + 1)))
    if not periodic:
        return np.concatenate([[pl], x, [pr]])
    mean = rho[:nc].sum() / nc
    sm = scale * mean
    x = x - sm * 0.5 * k1 * (n - np.arange(n))
    w = 0.5 * k1 * (2.0 * n - np.arange(n))
    M = (w * a).sum()
    shift = (-(M - pz * 0.5 * n) - sm * (n * (n + 1.0) * (n + 2.0) / 12.0)) / nc
    phi = np.concatenate([[0.0], x]) - shift
    return np.concatenate([phi, phi[:1]])


def _thomas_longdouble(rho, scale, periodic, pl=0.0, pr=0.0):
    """solve_poisson (fields.py:156-202) in long double."""
    ld = np.longdouble
    nc = len(rho) - 1
    r = rho.astype(ld)
    if periodic:
        mean = r[:nc].sum() / nc
        rhs = -(r[1:nc] - mean) * ld(scale)
    else:
        rhs = -r[1:nc] * ld(scale)
        rhs[0] -= ld(pl)
        rhs[-1] -= ld(pr)
    n = nc - 1
    k = np.arange(n, dtype=ld)
    z = np.cumsum((k + 1) * rhs)
    y = z / (k + 1)
    w = np.cumsum((-y / (k + 2))[::-1])[::-1]
    x = (k + 1) * w  # the closed-form pivots' two sweeps, exact to long double
    if periodic:
        phi = np.concatenate([[ld(0)], x])
        phi = phi - phi.sum() / nc
        return np.concatenate([phi, phi[:1]])
    return np.concatenate([[ld(pl)], x, [ld(pr)]])


@pytest.mark.parametrize("nc", [1001, 65536, 100_000])
@pytest.mark.parametrize("shape", ["noise", "smooth", "sheath"])
@pytest.mark.parametrize("periodic", [False, True])
def test_closed_form_fp64_accuracy(nc, shape, periodic):
    rng = np.random.default_rng(nc)
    xx = np.arange(nc + 1) / nc
    if shape == "noise":
        rho = 30.0 * rng.standard_normal(nc + 1)
    elif shape == "smooth":
        rho = 5.0 + np.sin(2 * np.pi * xx)
    else:
        rho = 1e3 * (np.exp(-50 * xx) + np.exp(-50 * (1 - xx))) + 10.0 * rng.standard_normal(nc + 1)
    if periodic:
        rho[nc] = rho[0]
    scale = (1e-5) ** 2 / 8.8541878128e-12
    pl, pr = (0.0, 0.0) if periodic else (1.5, -2.0)
    got = _closed_form(rho, scale, periodic, pl, pr)
    ref = _thomas_longdouble(rho, scale, periodic, pl, pr).astype(np.float64)
    err = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
    assert err < 1e-12, err
