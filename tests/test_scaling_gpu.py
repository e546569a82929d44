"""GPU: strong / weak sweeps over rank counts (ranks share the one GPU over
gloo here; the same driver runs one rank per GPU over NCCL)."""

import pytest

pytestmark = pytest.mark.gpu


def _cfg(**kw):
    from test_engine_gpu import _mk_config

    return _mk_config(nc=48, ppc0=10, n_steps=4, **kw)


def test_strong_sweep_transparent_across_ranks(cuda, tmp_path):
    from paper_2404_10270_b200.harness import strong_scaling_sweep, write_scaling_csv

    rep = strong_scaling_sweep(_cfg(field_solve=True, smoothing_passes=1), [1, 2], dist_backend="gloo",
                               timeout=600)
    assert rep.mode == "strong" and [r["workers"] for r in rep.rows] == [1, 2]
    assert rep.rows[0]["speedup"] == 1.0 and rep.rows[0]["pe_percent"] == 100.0
    assert rep.metrics[0].diagnostics == rep.metrics[1].diagnostics
    assert rep.metrics[1].worker_count == 2
    write_scaling_csv(rep, tmp_path / "scaling.csv")
    assert (tmp_path / "scaling.csv").read_text().startswith("workers,t_total,t_mover,speedup,pe\n1,")


def test_weak_sweep_scales_cells(cuda):
    from paper_2404_10270_b200.harness import weak_scaling_sweep

    rep = weak_scaling_sweep(_cfg(field_solve=False), [1, 2], dist_backend="gloo", timeout=600)
    assert rep.mode == "weak"
    m1, m2 = rep.metrics
    names = [k for k in m1.diagnostics[0] if k.startswith("total_")]
    for k in names:  # twice the cells, twice the particles
        assert m2.diagnostics[0][k] == 2 * m1.diagnostics[0][k]
    assert rep.rows[0]["pe_percent"] == 100.0
