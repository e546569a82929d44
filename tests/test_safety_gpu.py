"""Fixed-point deposit overflow is detected, never silent.

The reference sums fp64 partials per cell (pkg/src/picmc/backends/
_kernels.pyx:24-33) and has no per-cell population limit.  The B200 deposit
packs R = sum round(x*2^48) and the count C into u64 bins, which represent
at most 65535 particles of one species per cell (C << 48 wraps at 2^16).
Every reader of the bins (pb_rho_epilogue, pb_density_step, the peer
exchange) checks C and flags PB_ERR_OVERFLOW with the largest count in
pb_status.overflow; the engine raises EngineError at the next sync.
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _status(dev):
    from paper_2404_10270_b200.store import decode_status, status_template

    st = status_template(dev)
    return st, lambda: decode_status(st.cpu().numpy())


@pytest.mark.parametrize("count,bad", [(65535, False), (65536, True), (70000, True)])
@pytest.mark.parametrize("which", ["epilogue", "density_step"])
def test_epilogues_flag_overflow(cuda, count, bad, which):
    import torch

    from paper_2404_10270_b200 import _lib

    lib = _lib.load()
    nc, ndep = 6, 2
    bins = torch.zeros(ndep * 2 * nc, dtype=torch.int64, device=cuda)
    b = bins.view(ndep, 2, nc)
    b[1, 1, 3] = count           # C of species 1, cell 3
    b[1, 0, 3] = 0               # R (any value: it is the C check that matters)
    b[0, 1, 2] = 100
    left = torch.zeros(nc, dtype=torch.float64, device=cuda)
    right = torch.zeros(nc, dtype=torch.float64, device=cuda)
    rho = torch.zeros(nc + 1, dtype=torch.float64, device=cuda)
    st, read = _status(cuda)
    cc = (ctypes.c_double * ndep)(1.0, -1.0)
    sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if which == "epilogue":
        rc = lib.pb_rho_epilogue(bins.data_ptr(), cc, ndep, nc, _lib.PB_FIELD_PERIODIC, left.data_ptr(),
                                 right.data_ptr(), rho.data_ptr(), st.data_ptr(), sh)
    else:
        rc = lib.pb_density_step(bins.data_ptr(), None, st.data_ptr(), cc, ndep, nc, _lib.PB_FIELD_PERIODIC,
                                 left.data_ptr(), right.data_ptr(), rho.data_ptr(), sh)
    assert rc == _lib.PB_OK
    s = read()
    if bad:
        assert s.code == _lib.PB_ERR_OVERFLOW and s.overflow == count
    else:
        assert s.code == _lib.PB_OK and s.overflow == 0


def test_engine_raises_on_a_cell_with_70k_particles(cuda):
    """70,000 electrons in one cell (above the 65,535 limit) of a periodic
    run: the step-start deposit's epilogue flags it and sync() raises."""
    from paper_2404_10270_b200 import Engine, Grid1D, PhysicalConstants, RunConfig, SpeciesDef
    from paper_2404_10270_b200.core import ELECTRON_MASS, ELEMENTARY_CHARGE
    from paper_2404_10270_b200.errors import EngineError
    from paper_2404_10270_b200.core import FlatSpecies

    nc, ppc = 4, 17500
    cfg = RunConfig(grid=Grid1D.from_cells(nc, nc * 1e-5), consts=PhysicalConstants(dt_s=4e-14),
                    species=[SpeciesDef("e", -ELEMENTARY_CHARGE, ELECTRON_MASS)], temperatures_ev=[1.0],
                    densities_m3=[1e21], ppc0=ppc, n_steps=2, seed=1, field_solve=False,
                    smoothing_passes=0)
    eng = Engine(cfg, device=cuda, check_every=0)
    n = nc * ppc
    rng = np.random.default_rng(0)
    z = np.zeros(n)
    flat = FlatSpecies(x=rng.random(n), vx=z.copy(), vy=z.copy(), vz=z.copy(), yp=None,
                       cell=np.full(n, 2, dtype=np.int32))
    eng.upload([flat])
    eng.density()
    with pytest.raises(EngineError, match="overflow"):
        eng.sync()
    # the same population spread over the cells is fine
    flat.cell[:] = np.repeat(np.arange(nc, dtype=np.int32), ppc)
    eng.upload([flat])
    eng.density()
    eng.sync()


def test_engine_rejects_ppc0_beyond_the_bins(cuda):
    from paper_2404_10270_b200 import Engine, Grid1D, PhysicalConstants, RunConfig, SpeciesDef
    from paper_2404_10270_b200.core import ELECTRON_MASS, ELEMENTARY_CHARGE
    from paper_2404_10270_b200.errors import ConfigError

    cfg = RunConfig(grid=Grid1D.from_cells(2, 2e-5), consts=PhysicalConstants(dt_s=4e-14),
                    species=[SpeciesDef("e", -ELEMENTARY_CHARGE, ELECTRON_MASS)], temperatures_ev=[1.0],
                    densities_m3=[1e21], ppc0=40000, n_steps=1, seed=1, field_solve=False,
                    smoothing_passes=0)
    with pytest.raises(ConfigError, match="ppc0"):
        Engine(cfg, device=cuda)
