"""CPU-side checks: the C ABI library loads and exports every declared
symbol, the config surface behaves like the reference's strict loader, the
product fails loudly without a GPU, and the multi-GPU host logic (shard map +
exact fixed-point density allreduce) holds under gloo with world_size 2."""

import os
import re

import numpy as np
import pytest
import torch

from conftest import ROOT


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "picmc_b200.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char \*)\s*\*?(pb_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_2404_10270_b200 import _lib

    lib = _lib.load()
    names = _declared_symbols()
    assert len(names) >= 18
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.exported_names())
    assert lib.pb_abi_version() == _lib.ABI_VERSION == 3


def test_library_argument_errors_without_gpu():
    """Argument validation happens before any device work."""
    from paper_2404_10270_b200 import _lib

    lib = _lib.load()
    assert lib.pb_push_deposit(None, 99, None, 10, 0, None, None, None) == _lib.PB_ERR_INVALID
    assert b"nsp" in lib.pb_last_error()
    assert lib.pb_solve_poisson(None, None, 2, 1.0, 1.0, 0, 0.0, 0.0, None, None) == _lib.PB_ERR_INVALID
    with pytest.raises(ValueError):
        _lib.check(_lib.PB_ERR_INVALID, "x")


def test_status_struct_layout_matches_header():
    from paper_2404_10270_b200 import _lib

    # int32 code, int32 species, u64 index, 8 moved, 8x2 absorbed, 8 holes, overflow,
    # tile_next, tile_done, tile_next2, mover_t0, mover_ns, mover_launches
    assert _lib.STATUS_BYTES == 4 + 4 + 8 + 8 * 8 + 16 * 8 + 8 * 8 + 8 + 8 + 8 + 8 + 8 + 8 + 8
    assert _lib.load().pb_status_bytes() == _lib.STATUS_BYTES  # the C struct, as compiled


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_engine_fails_loudly_without_gpu():
    from paper_2404_10270_b200 import Engine, load_config
    from paper_2404_10270_b200 import backend

    cfg = load_config(os.path.join(ROOT, "configs", "c2_ionization_100k.toml"))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        Engine(cfg)
    from paper_2404_10270_b200 import CanonicalEngine

    with pytest.raises(RuntimeError, match="no CPU fallback"):
        CanonicalEngine(load_config(os.path.join(ROOT, "configs", "desk.toml")))
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        backend.deposit_partials(np.zeros(4), np.zeros(2, dtype=np.int64), np.zeros(2, dtype=np.int64))


def test_backend_selector():
    from paper_2404_10270_b200 import backends

    assert backends.BACKEND == "cuda"
    assert backends.load_backend("cuda").BACKEND_NAME == "cuda"
    with pytest.raises(ValueError):
        backends.load_backend("pure")  # no silent fallback


def test_configs_load_and_validate():
    from paper_2404_10270_b200 import load_config

    names = sorted(f for f in os.listdir(os.path.join(ROOT, "configs")) if f.endswith(".toml"))
    assert len(names) == 8
    cfgs = {n: load_config(os.path.join(ROOT, "configs", n)) for n in names}
    for n in ("desk.toml", "c1_desk_ppc100.toml"):
        assert cfgs[n].canonical() and cfgs[n].collisions.rates.rate_ionization_m3s == 2.5e-11
    assert cfgs["c1_desk_ppc100.toml"].ppc0 == 100 and cfgs["desk.toml"].ppc0 == 10
    assert not cfgs["c2_ionization_100k.toml"].canonical()
    c3 = cfgs["c3_sheath_absorbing.toml"]
    assert c3.particle_boundary == "absorbing" and c3.boundary == "dirichlet" and c3.sort_every == 50
    c4 = cfgs["c4_sol_boris.toml"]
    assert c4.b_field_t == (0.2, 0.0, 2.0) and c4.b_grad_t_per_m is None
    c4b = cfgs["c4b_sol_gradb.toml"]
    assert c4b.b_field_t == (0.2, 0.0, 2.0) and c4b.b_grad_t_per_m == (0.0, 0.0, -1.0)
    c2 = cfgs["c2_ionization_100k.toml"]
    assert c2.grid.nc * c2.ppc0 * len(c2.species) == 30_000_000


def test_slot_order_validation():
    from dataclasses import replace

    from paper_2404_10270_b200 import ConfigError, load_config

    desk = load_config(os.path.join(ROOT, "configs", "desk.toml"))
    with pytest.raises(ConfigError, match="collisions need slot_order"):
        replace(desk, slot_order="fast").validate()
    with pytest.raises(ConfigError, match="slot_order must be"):
        replace(desk, slot_order="sorted").validate()
    assert replace(desk, collisions=None).canonical() is False
    assert replace(desk, collisions=None, slot_order="canonical").canonical() is True


def test_strict_loader_rejects_unknown_keys():
    from paper_2404_10270_b200 import ConfigError, config_from_dict

    base = {"grid": {"nc": 8, "length_m": 8e-5}, "time": {"dt_s": 4e-14, "n_steps": 1},
            "run": {"seed": 1, "ppc0": 2},
            "species": [{"name": "e", "charge_e": -1.0, "mass_kg": 9.1e-31, "temperature_ev": 1.0,
                         "density_m3": 1e21}]}
    assert config_from_dict(base).ppc0 == 2
    bad = {**base, "run": {**base["run"], "workerz": 2}}
    with pytest.raises(ConfigError, match="workerz"):
        config_from_dict(bad)
    bad2 = {**base, "run": {**base["run"], "particle_boundary": "reflecting"}}
    with pytest.raises(ConfigError, match="particle_boundary"):
        config_from_dict(bad2)
    with pytest.raises(ConfigError, match="missing"):
        config_from_dict({**base, "grid": {"nc": 8}})


def test_config_hash_changes_with_physics_only():
    from dataclasses import replace

    from paper_2404_10270_b200 import load_config

    cfg = load_config(os.path.join(ROOT, "configs", "desk.toml"))
    assert cfg.config_hash() == replace(cfg, out_dir="/tmp/x").config_hash()
    assert cfg.config_hash() != replace(cfg, seed=cfg.seed + 1).config_hash()


def test_partition_cells_balanced():
    from paper_2404_10270_b200 import partition_cells

    r = partition_cells(10, 3)
    assert r == ((0, 4), (4, 7), (7, 10))
    for nc, w in ((100_000, 8), (7, 7), (13, 4)):
        rr = partition_cells(nc, w)
        sizes = [hi - lo for lo, hi in rr]
        assert sum(sizes) == nc and max(sizes) - min(sizes) <= 1


def _dist_worker(rank, world, port, out_path):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    from paper_2404_10270_b200 import load_config, partition_cells, reduce_bins
    from paper_2404_10270_b200.core import init_species_host

    cfg = load_config(os.path.join(ROOT, "configs", "desk.toml"))
    nc = cfg.grid.nc
    lo, hi = partition_cells(nc, world)[rank]
    charged = [k for k, sp in enumerate(cfg.species) if sp.charged]
    bins = np.zeros((len(charged), 2, nc), dtype=np.uint64)
    for d, k in enumerate(charged):
        f = init_species_host(cfg, k, lo, hi)
        # move the shard a few steps so particles leave their home range
        z = np.zeros(nc + 1)
        for _ in range(30):
            oracle.step_flat(1, 0, 40.0, 0.0, z, nc, f.x, f.vx, f.vy, f.vz, f.yp, f.cell)
        R, C = oracle.deposit_fixed(f.x, f.cell, nc)
        bins[d, 0], bins[d, 1] = R, C
    t = torch.from_numpy(bins.view(np.int64).copy())
    reduce_bins(t)
    if rank == 0:
        np.save(out_path, t.numpy().view(np.uint64))
    dist.barrier()
    dist.destroy_process_group()


def test_density_allreduce_world2_equals_single_rank(tmp_path):
    """Particles sharded over 2 gloo ranks (each loads its own cell range and
    drifts across the whole grid); the exact int64 allreduce of the
    fixed-point bins equals the single-rank deposit bit for bit."""
    import socket

    import torch.multiprocessing as mp

    from oracle import oracle
    from paper_2404_10270_b200 import load_config
    from paper_2404_10270_b200.core import init_species_host

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "bins.npy")
    mp.spawn(_dist_worker, args=(2, port, out), nprocs=2, join=True)
    got = np.load(out)
    cfg = load_config(os.path.join(ROOT, "configs", "desk.toml"))
    nc = cfg.grid.nc
    z = np.zeros(nc + 1)
    for d, k in enumerate(k for k, sp in enumerate(cfg.species) if sp.charged):
        f = init_species_host(cfg, k)
        for _ in range(30):
            oracle.step_flat(1, 0, 40.0, 0.0, z, nc, f.x, f.vx, f.vy, f.vz, f.yp, f.cell)
        R, C = oracle.deposit_fixed(f.x, f.cell, nc)
        assert np.array_equal(got[d, 0], R) and np.array_equal(got[d, 1], C)


def test_bench_reference_arm_json_line():
    """`bench.py --impl reference` (the driver's reference arm) runs on the
    host alone and prints one JSON line with the contract's keys."""
    import json
    import subprocess
    import sys

    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "5", "--warmup", "3", "--cpu-seconds", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0 and line["unit"] == "particle-pushes/s"
    for k in ("metric", "n_gpus", "steps", "warmup", "higher_is_better", "scaling", "dtype", "config"):
        assert k in line
    cb = line["cpu_baseline"]
    assert cb["value"] == line["value"] and cb["cores"] >= 1 and cb["kind"] in ("reference", "port")
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_peer_status_maps_to_engine_error():
    """PB_ERR_PEER (a GPU missed a density barrier) surfaces as EngineError."""
    import pytest

    from paper_2404_10270_b200 import _lib
    from paper_2404_10270_b200.errors import EngineError

    assert _lib.PB_ERR_PEER == 6
    try:
        _lib.load()
    except ImportError:
        pytest.skip("library not built")
    with pytest.raises(EngineError):
        _lib.check(_lib.PB_ERR_PEER, "peer")


def test_b_profile_config_and_nodes():
    """b_grad_t_per_m: validation, and the engine's node profile equals the
    oracle's restatement bit for bit (B(X_j) = B0 + g (X_j - L/2))."""
    from dataclasses import replace

    from oracle import oracle
    from paper_2404_10270_b200 import ConfigError, load_config
    from paper_2404_10270_b200.engine import b_field_nodes

    cfg = load_config(os.path.join(ROOT, "configs", "c4b_sol_gradb.toml"))
    nodes = b_field_nodes(cfg)
    assert nodes.shape == (cfg.grid.nc + 1, 4) and not nodes[:, 3].any()
    assert np.array_equal(nodes.view(np.uint64), oracle.b_nodes(cfg).view(np.uint64))
    assert abs(nodes[0, 2] - 2.5) < 1e-12 and abs(nodes[-1, 2] - 1.5) < 1e-12
    assert b_field_nodes(replace(cfg, b_grad_t_per_m=None)) is None
    with pytest.raises(ConfigError, match="b_grad_t_per_m needs b_field_t"):
        replace(cfg, b_field_t=None).validate()
    with pytest.raises(ConfigError, match="three components"):
        replace(cfg, b_grad_t_per_m=(1.0, 2.0)).validate()


def test_errors_are_the_reference_classes_when_importable(tmp_path):
    """With the reference package on the path, the engine raises the
    reference's own exception classes (callers' `except picmc.errors.X`
    keep working); without it, the same hierarchy is declared locally."""
    import subprocess
    import sys

    from paper_2404_10270_b200 import errors

    assert issubclass(errors.CflViolation, errors.EngineError)
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "picmc")):
        pytest.skip("reference not installed (scripts/install_reference.sh)")
    code = ("import picmc.errors as r, paper_2404_10270_b200.errors as e; "
            "assert e.SHARED_WITH_REFERENCE and e.CflViolation is r.CflViolation "
            "and e.EngineError is r.EngineError and e.ConfigError is r.ConfigError")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([ref, ROOT]), PICMC_BACKEND="pure")
    subprocess.run([sys.executable, "-c", code], check=True, env=env, cwd=str(tmp_path))


def _thomas_exact(r):
    """_thomas_unit (pkg/src/picmc/fields.py:138-153) in exact rationals."""
    from fractions import Fraction

    n = len(r)
    diag, y = [Fraction(-2)], [r[0]]
    for i in range(1, n):
        m = 1 / diag[i - 1]
        diag.append(Fraction(-2) - m)
        y.append(r[i] - m * y[i - 1])
    x = [None] * n
    x[n - 1] = y[n - 1] / diag[n - 1]
    for i in range(n - 2, -1, -1):
        x[i] = (y[i] - x[i + 1]) / diag[i]
    return x


@pytest.mark.parametrize("nc", [3, 4, 9, 40])
def test_closed_form_poisson_exact(nc):
    """The closed form the scan solve implements (csrc/fields.cu, DESIGN
    3.3) equals the reference's elimination (fields.py:156-202) exactly in
    rational arithmetic: Dirichlet x_k, the periodic mean part, and the
    periodic shift sum_k x_k from the tile sum M."""
    from fractions import Fraction as F

    rng = np.random.default_rng(nc)
    rho = [F(int(v), 7) for v in rng.integers(-90, 90, nc + 1)]
    scale, pl, pr = F(11, 3), F(5, 2), F(-3)
    n = nc - 1
    for periodic in (False, True):
        if periodic:
            mean = sum(rho[:nc]) / nc
            a = [-rho[j + 1] * scale for j in range(n)]
            r = [-(rho[j + 1] - mean) * scale for j in range(n)]
        else:
            mean = F(0)
            a = [-rho[j + 1] * scale for j in range(n)]
            a[0] -= pl
            a[n - 1] -= pr
            r = a
        x = _thomas_exact(r)
        S = [sum(a[: k + 1]) for k in range(n)]
        Z = [sum((j + 1) * a[j] for j in range(k + 1)) for k in range(n)]
        sm = scale * mean
        xc = [-(Z[k] + (k + 1) * ((S[-1] - S[k]) - Z[-1] / (n + 1))) - sm * F((k + 1) * (n - k), 2)
              for k in range(n)]
        assert xc == x
        if periodic:
            M = sum(F((j + 1) * (2 * n - j), 2) * a[j] for j in range(n))
            assert -(M - Z[-1] * F(n, 2)) - sm * F(n * (n + 1) * (n + 2), 12) == sum(x)
