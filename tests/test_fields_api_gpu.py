"""GPU: the field pipeline API (paper_2404_10270_b200.fields) vs the reference.

Mirrors pkg/tests/test_fields.py's function-level checks on golden outputs
of the reference itself (tests/golden/fields.npz, fields_api.npz from
make_golden.py).  Bar: bitwise, for NumPy inputs (staged) and CUDA tensors
(in place) alike.
"""

import numpy as np
import pytest

from conftest import bits_equal, load_golden

pytestmark = pytest.mark.gpu


def _species():
    from paper_2404_10270_b200 import SpeciesDef

    return [SpeciesDef("e", -1.602176634e-19, 9.1093837015e-31),
            SpeciesDef("D+", 1.602176634e-19, 3.3435837483066354e-27),
            SpeciesDef("D", 0.0, 3.344494686676785e-27, track_transverse=True)]


def _store(g):
    from paper_2404_10270_b200 import Grid1D
    from paper_2404_10270_b200.cellstore import CellSortedStore

    nc = len(g["store_sp0_counts"])
    fields = []
    for i in range(3):
        names = ["x", "vx", "vy", "vz"] + (["yp"] if f"store_sp{i}_yp" in g else [])
        fields.append({n: g[f"store_sp{i}_{n}"] for n in names})
    s = CellSortedStore.from_host(Grid1D.from_cells(nc, nc * 1e-5), _species(),
                                  [g[f"store_sp{i}_counts"] for i in range(3)],
                                  [g[f"store_sp{i}_caps"] for i in range(3)], fields)
    s.weights = list(g["weights"])
    return s


def _np(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else a


def test_store_level_deposit_stitch_gather_match_reference(cuda):
    from paper_2404_10270_b200 import PhysicalConstants
    from paper_2404_10270_b200.fields import (deposit_charge, deposit_partials_range, gather_field,
                                              stitch_rho)

    g = load_golden("fields_api.npz")
    s = _store(g)
    consts = PhysicalConstants(dt_s=4e-14)
    nc = s.grid.nc
    for lo, hi in ((0, nc), (5, 17), (28, 29)):
        left, right = deposit_partials_range(s, consts, lo, hi)
        assert bits_equal(_np(left), g[f"dpr_{lo}_{hi}_left"]) and bits_equal(_np(right), g[f"dpr_{lo}_{hi}_right"])
    left, right = deposit_partials_range(s, consts, 0, nc)
    assert bits_equal(_np(stitch_rho(left, right, True)), g["stitch_periodic"])
    assert bits_equal(_np(stitch_rho(left, right, False)), g["stitch_walls"])
    assert bits_equal(stitch_rho(_np(left), _np(right), False), g["stitch_walls"])  # numpy in, numpy out
    assert bits_equal(_np(deposit_charge(s, s.grid, consts, "periodic")), g["charge_periodic"])
    assert bits_equal(_np(deposit_charge(s, s.grid, consts, "dirichlet")), g["charge_dirichlet"])
    for isp, v in gather_field(g["gather_e"], s, s.grid).items():
        assert bits_equal(_np(v), g[f"gather_sp{isp}"]), isp


def test_deposit_charge_enforces_resort_contract(cuda):
    from paper_2404_10270_b200 import PhysicalConstants
    from paper_2404_10270_b200.errors import ContractViolation
    from paper_2404_10270_b200.fields import deposit_charge

    g = load_golden("fields_api.npz")
    s = _store(g)
    j = int(np.nonzero(g["store_sp1_counts"])[0][0])
    s.data(1)["x"][int(s.offsets(1)[j])] = 1.0
    with pytest.raises(ContractViolation, match="not resorted"):
        deposit_charge(s, s.grid, PhysicalConstants(dt_s=4e-14))


@pytest.mark.parametrize("nc", [8, 100, 1000])
@pytest.mark.parametrize("as_tensor", [False, True])
def test_smooth_poisson_efield_match_reference(cuda, nc, as_tensor):
    import torch

    from paper_2404_10270_b200 import Grid1D, PhysicalConstants
    from paper_2404_10270_b200.fields import compute_efield, smooth_density, solve_poisson

    g = load_golden("fields.npz")
    grid = Grid1D.from_cells(nc, nc * 1e-5)
    consts = PhysicalConstants(dt_s=4e-14)
    rho = g[f"n{nc}_rho"]
    if as_tensor:
        rho = torch.from_numpy(rho).to(cuda)
    assert bits_equal(_np(smooth_density(rho, 1)), g[f"n{nc}_smooth1"])
    assert bits_equal(_np(smooth_density(rho, 3)), g[f"n{nc}_smooth3"])
    for bc in ("periodic", "dirichlet"):
        phi = solve_poisson(rho, grid, consts, bc, 1.5, -2.0)
        assert isinstance(phi, torch.Tensor) == as_tensor
        assert bits_equal(_np(phi), g[f"n{nc}_{bc}_phi"]), bc
        assert bits_equal(_np(compute_efield(phi, grid, bc)), g[f"n{nc}_{bc}_e"]), bc


def test_field_api_argument_errors(cuda):
    from paper_2404_10270_b200 import Grid1D, PhysicalConstants
    from paper_2404_10270_b200.fields import FieldState, solve_poisson

    consts = PhysicalConstants(dt_s=4e-14)
    with pytest.raises(ValueError, match="nc >= 3"):
        solve_poisson(np.zeros(3), Grid1D.from_cells(2, 2e-5), consts)
    with pytest.raises(ValueError, match="unknown boundary"):
        solve_poisson(np.zeros(9), Grid1D.from_cells(8, 8e-5), consts, "neumann")
    with pytest.raises(ValueError, match="share length"):
        FieldState(np.zeros(3), np.zeros(3), np.zeros(4))
    fs = FieldState.zeros(5)
    assert len(fs.rho) == 6 and fs.rho_mean_subtracted == 0.0
