"""CPU: scaling report arithmetic and scaling.csv bytes
(pkg/src/picmc/harness.py:278-383; pkg/tests/test_harness.py scaling checks)."""

import pytest


def test_speedup_and_efficiency():
    from paper_2404_10270_b200.harness import compute_parallel_efficiency, compute_speedup

    assert compute_speedup(8.0, 2.0) == 4.0
    assert compute_parallel_efficiency(4.0, 8) == 50.0
    with pytest.raises(ValueError):
        compute_speedup(0.0, 1.0)
    with pytest.raises(ValueError):
        compute_parallel_efficiency(1.0, 0)


def test_scaling_csv_bytes(tmp_path):
    from paper_2404_10270_b200.harness import ScalingReport, write_scaling_csv

    rep = ScalingReport("strong", [
        {"workers": 1, "t_total": 2.0, "t_mover": 1.25, "speedup": 1.0, "pe_percent": 100.0},
        {"workers": 4, "t_total": 0.625, "t_mover": 0.3125, "speedup": 3.2, "pe_percent": 80.0},
    ])
    p = tmp_path / "scaling.csv"
    write_scaling_csv(rep, p)
    assert p.read_bytes() == (b"workers,t_total,t_mover,speedup,pe\n"
                              b"1,2.000000000,1.250000000,1.000000,100.0000\n"
                              b"4,0.625000000,0.312500000,3.200000,80.0000\n")


def test_module_twins_have_no_cpu_fallback():
    """mover / fields / cellstore run on the GPU only: without a device they
    raise instead of computing on the host."""
    import numpy as np
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2404_10270_b200 import Grid1D, SpeciesDef, fields, mover
    from paper_2404_10270_b200.cellstore import CellSortedStore

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        fields.smooth_density(np.zeros(9))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        CellSortedStore(Grid1D.from_cells(4, 4.0), [SpeciesDef("s", 0.0, 1.0)])

    class Store:  # the reference store interface, numpy arrays
        species = [SpeciesDef("s", 0.0, 1.0)]
        grid = Grid1D.from_cells(4, 4.0)
        data = lambda self, i: {"x": np.zeros(16), "vx": np.zeros(16), "vy": np.zeros(16),  # noqa: E731
                                "vz": np.zeros(16)}
        offsets = lambda self, i: np.arange(0, 16, 4)  # noqa: E731
        counts = lambda self, i: np.zeros(4, dtype=np.int64)  # noqa: E731
        field_names = lambda self, i: ("x", "vx", "vy", "vz")  # noqa: E731

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        mover.resort_collect(Store())
