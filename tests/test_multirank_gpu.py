"""The N>1 engine path on one GPU: two ranks (gloo, sharing cuda:0) each load
their cell range of the population, step with the density allreduce on the
side stream (field-free) or the split field cycle (field solve), and must
reproduce the single-rank density bit for bit (fixed-point bins are summed
exactly, so the reduction order cannot matter).  With two or more GPUs
visible the same runs go through NCCL / NVLink peer memory, one GPU per
rank (test_two_gpus_nccl_match_one_rank_and_oracle; skipped on one GPU)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _cfg(field):
    from paper_2404_10270_b200 import Grid1D, PhysicalConstants, RunConfig, SpeciesDef
    from paper_2404_10270_b200.core import DEUTERIUM_MASS, ELECTRON_MASS, ELEMENTARY_CHARGE

    species = [SpeciesDef("e", -ELEMENTARY_CHARGE, ELECTRON_MASS),
               SpeciesDef("D+", ELEMENTARY_CHARGE, DEUTERIUM_MASS - ELECTRON_MASS),
               SpeciesDef("D", 0.0, DEUTERIUM_MASS, track_transverse=True)]
    return RunConfig(grid=Grid1D.from_cells(96, 96e-5), consts=PhysicalConstants(dt_s=4e-14),
                     species=species, temperatures_ev=[400.0, 400.0, 40.0], densities_m3=[1e21] * 3,
                     ppc0=40, n_steps=0, seed=7, field_solve=field, smoothing_passes=1 if field else 0,
                     sort_every=4)


def _worker(rank, world, port, field, out, peer=False, nccl=False):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    # nccl: one GPU per rank (the production transport); else gloo, all on cuda:0
    dev = torch.device("cuda", rank if nccl else 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl" if nccl else "gloo", rank=rank, world_size=world)
    from paper_2404_10270_b200 import Engine

    eng = Engine(_cfg(field), device=dev, rank=rank, world=world, check_every=0,
                 peer=peer)
    assert (eng.peer is not None) == peer  # the peer-memory exchange mapped every rank's buffers
    assert eng._field_split()[0] if field else True  # the N>1 default overlaps the neutral push
    rhos = []
    for _ in range(9):
        rho, e = eng.step()
        rhos.append(rho.cpu().numpy().copy())
    eng.replay(6)  # graphs with the peer exchange, eager with the process-group allreduce
    assert (len(eng.graphs) > 0) == peer
    rho, _ = eng.step()
    rhos.append(rho.cpu().numpy().copy())
    eng.sync()
    if rank == 0:
        np.save(out, np.array(rhos))
    fl = eng.download()
    np.savez(out + f".rank{rank}.npz", **{f"sp{k}_{n}": a for k, f in enumerate(fl)
                                         for n, a in list(f.fields().items()) + [("cell", f.cell)]})
    dist.barrier()
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("peer", [False, True])
@pytest.mark.parametrize("field", [False, True])
def test_two_ranks_match_one_rank_bitwise(cuda, tmp_path, field, peer):
    """peer False: reduce_bins (process-group allreduce) + pb_density_step;
    peer True: pb_peer_density_step over CUDA IPC mappings (the NVLink path;
    here two processes on one GPU)."""
    import torch
    import torch.multiprocessing as mp

    from paper_2404_10270_b200 import Engine

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "rho.npy")
    mp.spawn(_worker, args=(2, port, field, out, peer), nprocs=2, join=True)
    got = np.load(out)
    eng = Engine(_cfg(field), device=cuda, check_every=0)
    want = []
    for _ in range(9):
        rho, _ = eng.step()
        want.append(rho.cpu().numpy().copy())
    for _ in range(6):
        eng.step()
    rho, _ = eng.step()
    want.append(rho.cpu().numpy().copy())
    assert got.shape == np.array(want).shape
    for k, (a, b) in enumerate(zip(got, want)):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), k
    if not field:
        _check_union_vs_oracle(out, 2, 16)  # 9 eager + 6 replayed + 1


def _check_union_vs_oracle(out, world, steps):
    """Field-free runs: the union of the ranks' particles after `steps`
    steps equals the C oracle stepping the whole population on the host
    (E = 0, same initial load), per-cell multisets bit for bit -- the
    multi-rank path pinned to the oracle directly, not only to one rank."""
    from oracle import oracle
    from paper_2404_10270_b200.core import init_species_host, velocity_kick_coef
    from paper_2404_10270_b200.engine import species_kind

    cfg = _cfg(False)
    nc = cfg.grid.nc
    e = np.zeros(nc + 1)
    parts = [np.load(out + f".rank{r}.npz") for r in range(world)]
    for k, spd in enumerate(cfg.species):
        f = init_species_host(cfg, k)
        kind = species_kind(spd, None)
        coef = velocity_kick_coef(spd, cfg.consts, cfg.grid.dx_m) if spd.charged else 0.0
        for _ in range(steps):
            _, _, cfl = oracle.step_flat(kind, 0, float(spd.nstep), coef, e, nc, f.x, f.vx, f.vy, f.vz, f.yp,
                                         f.cell)
            assert cfl == -1
        names = list(f.fields())
        got = {n: np.concatenate([p[f"sp{k}_{n}"] for p in parts]) for n in names}
        cell = np.concatenate([p[f"sp{k}_cell"] for p in parts])
        assert np.array_equal(oracle.canonical(cell, got), oracle.canonical(f.cell, f.fields())), spd.name


@pytest.mark.skipif("__import__('torch').cuda.device_count() < 2")
@pytest.mark.parametrize("peer", [False, True])
def test_two_gpus_nccl_match_one_rank_and_oracle(cuda, tmp_path, peer):
    """Runs whenever >= 2 GPUs are visible: one rank per GPU with the NCCL
    process group -- peer False: reduce_bins as an NCCL allreduce of the
    fixed-point bins; peer True: pb_peer_density_step over NVLink IPC
    mappings (co-residency checked at launch).  rho per step equals the
    single-GPU run bit for bit and the particles equal the oracle."""
    import torch.multiprocessing as mp

    from paper_2404_10270_b200 import Engine

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "rho.npy")
    mp.spawn(_worker, args=(2, port, False, out, peer, True), nprocs=2, join=True)
    got = np.load(out)
    eng = Engine(_cfg(False), device=cuda, check_every=0)
    want = []
    for _ in range(16):
        rho, _ = eng.step()
        want.append(rho.cpu().numpy().copy())
    want = [want[k] for k in list(range(9)) + [15]]
    for k, (a, b) in enumerate(zip(got, want)):
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), k
    _check_union_vs_oracle(out, 2, 16)


def _canon_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from conftest import load_golden
    from golden_cfg import cfg_from
    from paper_2404_10270_b200 import CanonicalEngine

    cfg = cfg_from(load_golden("run_collide_guard.npz"), slot_order="canonical")
    eng = CanonicalEngine(cfg, device=torch.device("cuda", 0), rank=rank, world=world)
    rhos, tallies = [], []
    for _ in range(cfg.n_steps):
        rho, _ = eng.step()
        rhos.append(rho.cpu().numpy().copy())
        tallies.append(eng.tally_last)
    eng.sync()
    flats = eng.download()
    np.savez(out + f".{rank}.npz", rho=np.array(rhos), tallies=np.array(tallies),
             **{f"sp{k}_{name}": arr for k, f in enumerate(flats)
                for name, arr in list(f.fields().items()) + [("cell", f.cell)]})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_canonical_collisions_multirank_match_reference(cuda, tmp_path, world):
    """Collisions + field solve on two ranks (cell ranges, migration by
    all_to_all, global canonical ranks): per-step rho and tallies, and the
    final stores concatenated in rank order, equal the single-domain run --
    which is the reference run itself (golden run_collide_guard)."""
    import torch.multiprocessing as mp

    from conftest import bits_equal, load_golden

    g = load_golden("run_collide_guard.npz")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "canon")
    mp.spawn(_canon_worker, args=(world, port, out), nprocs=world, join=True)
    rs = [np.load(out + f".{r}.npz") for r in range(world)]
    for r in rs:
        assert bits_equal(r["rho"], g["rho"])
        assert np.array_equal(r["tallies"], g["tallies"][1:])
    for k in range(3):
        for name in ("x", "vx", "vy", "vz", "yp", "cell"):
            key = f"sp{k}_{name}"
            if key not in g:
                continue
            both = np.concatenate([r[key] for r in rs])
            if name == "cell":
                assert np.array_equal(both.astype(np.int64), g[key].astype(np.int64)), key
            else:
                assert bits_equal(both, g[key]), key
