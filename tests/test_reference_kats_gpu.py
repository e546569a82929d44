"""The reference's own deposit known-answer tests, on the device path.

Mirrors pkg/tests/test_fields.py:37-140 (single particle 0.75/0.25 split,
particle on a node, exact neutrality, neutral species, periodic and
Dirichlet charge budgets) and acceptance criterion 03
(pkg/tests/test_acceptance.py:146-173: 1e6-particle charge conservation at
1e-12, smoothing at 1e-13), through the production path: the fixed-point
deposit (pb_deposit_only, the mover's deposit) and the density epilogue
(pb_density_step).
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

E_CH = 1.602176634e-19
DX = 1e-5


def device_rho(defs, flats, weights, nc, bc="periodic"):
    import torch

    from paper_2404_10270_b200 import _lib
    from paper_2404_10270_b200.store import DeviceSpecies, species_array, status_template

    lib = _lib.load()
    dev = torch.device("cuda", 0)
    sps, coef = [], []
    ndep = 0
    for d, f in zip(defs, flats):
        dep = -1
        if d.charged:
            dep = ndep
            ndep += 1
        s = DeviceSpecies(d, f.n, dev, kind=_lib.PB_KIND_INACTIVE, deposit=dep)
        if f.n:
            s.upload(f)
        sps.append(s)
    for d, w in zip(defs, weights):
        if d.charged:
            coef.append(d.charge_c * w / DX)
    arr, n = species_array(sps)
    bins = torch.zeros(max(ndep, 1) * 2 * nc, dtype=torch.int64, device=dev)
    status = status_template(dev)
    sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(lib.pb_deposit_only(arr, n, nc, bins.data_ptr(), status.data_ptr(), sh))
    left = torch.zeros(nc, dtype=torch.float64, device=dev)
    right = torch.zeros(nc, dtype=torch.float64, device=dev)
    rho = torch.zeros(nc + 1, dtype=torch.float64, device=dev)
    cc = (ctypes.c_double * max(ndep, 1))(*coef)
    code = _lib.PB_FIELD_PERIODIC if bc == "periodic" else _lib.PB_FIELD_DIRICHLET
    _lib.check(lib.pb_density_step(bins.data_ptr(), None, status.data_ptr(), cc, ndep, nc, code, left.data_ptr(),
                                   right.data_ptr(), rho.data_ptr(), sh))
    return rho.cpu().numpy(), np.array(coef)


def flat(cells, xs, yp=False):
    from paper_2404_10270_b200.core import FlatSpecies

    n = len(xs)
    z = np.zeros(n)
    return FlatSpecies(x=np.asarray(xs, dtype=np.float64), vx=z.copy(), vy=z.copy(), vz=z.copy(),
                       yp=z.copy() if yp else None, cell=np.asarray(cells, dtype=np.int32))


def electron():
    from paper_2404_10270_b200 import SpeciesDef

    return SpeciesDef("e", -E_CH, 9.1093837015e-31)


def uniform(nc, ppc, seed):
    rng = np.random.default_rng(seed)
    return flat(np.repeat(np.arange(nc), ppc), rng.random(nc * ppc))


def test_single_particle_splits_weight(cuda):
    rho, coef = device_rho([electron()], [flat([1], [0.25])], [7.0], 4)
    assert rho[1] == pytest.approx(0.75 * coef[0], rel=1e-15)
    assert rho[2] == pytest.approx(0.25 * coef[0], rel=1e-15)
    assert rho[0] == 0.0 and rho[3] == 0.0


def test_particle_at_node_deposits_whole_weight(cuda):
    rho, coef = device_rho([electron()], [flat([2], [0.0])], [7.0], 4)
    assert rho[2] == coef[0]
    assert rho[3] == 0.0


def test_exact_charge_neutrality_cancels_bitwise(cuda):
    from paper_2404_10270_b200 import SpeciesDef

    e = SpeciesDef("e", -E_CH, 1e-30)
    p = SpeciesDef("p", +E_CH, 1e-27)
    f = uniform(5, 4, 8)
    rho, _ = device_rho([e, p], [f, flat(f.cell, f.x)], [3.0, 3.0], 5)
    assert np.all(rho == 0.0)


def test_neutral_species_deposit_nothing(cuda):
    from paper_2404_10270_b200 import SpeciesDef

    rho, _ = device_rho([SpeciesDef("s", 0.0, 1.0)], [uniform(5, 4, 1)], [1.0], 5)
    assert np.all(rho == 0.0)


@pytest.mark.parametrize("bc", ["periodic", "dirichlet"])
def test_charge_budget(cuda, bc):
    nc, ppc, w = 50, 20, 2.5e13
    f = uniform(nc, ppc, 2)
    rho, _ = device_rho([electron()], [f], [w], nc, bc)
    if bc == "periodic":
        total = rho[:nc].sum() * DX
    else:  # half-weight wall nodes close the budget (test_fields.py:126-140)
        total = (0.5 * rho[0] + rho[1:nc].sum() + 0.5 * rho[nc]) * DX
    expect = nc * ppc * electron().charge_c * w
    assert total == pytest.approx(expect, rel=1e-12)


def test_criterion03_charge_conservation_at_scale(cuda):
    """> 1e6 particles: deposit within 1e-12, 3-pass smoothing within 1e-13."""
    import torch

    from paper_2404_10270_b200 import _lib

    nc, ppc, w = 1024, 980, 2.5e13
    f = uniform(nc, ppc, 99)
    rho, _ = device_rho([electron()], [f], [w], nc)
    total = np.sum(rho[:nc]) * DX
    expect = nc * ppc * electron().charge_c * w
    assert abs(total - expect) / abs(expect) <= 1e-12
    lib = _lib.load()
    r = torch.from_numpy(rho).cuda()
    out = torch.empty_like(r)
    scr = torch.empty(lib.pb_field_scratch_bytes(nc) // 8 + 1, dtype=torch.float64, device="cuda")
    _lib.check(lib.pb_smooth_density(r.data_ptr(), out.data_ptr(), nc, 3, scr.data_ptr(),
                                     ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    sm = out.cpu().numpy()
    assert abs(np.sum(sm[:nc]) - np.sum(rho[:nc])) / abs(np.sum(rho[:nc])) <= 1e-13
