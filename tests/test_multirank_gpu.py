"""The N>1 engine path on one GPU: two ranks (gloo, sharing cuda:0) each load
their cell range of the population, step with the density allreduce on the
side stream (field-free) or the split field cycle (field solve), and must
reproduce the single-rank density bit for bit (fixed-point bins are summed
exactly, so the reduction order cannot matter).  The NCCL transport is the
only part not exercised here."""

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


def _worker(rank, world, port, field, out, peer=False):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2404_10270_b200 import Engine

    eng = Engine(_cfg(field), device=torch.device("cuda", 0), rank=rank, world=world, check_every=0,
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
