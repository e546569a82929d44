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
