"""GPU: the store-level mover API (paper_2404_10270_b200.mover) vs the reference.

Mirrors pkg/tests/test_mover.py on the device CellSortedStore twin and on a
numpy store with the reference's interface (the staging path).  Golden
fixture tests/golden/mover_api.npz is the reference's own output
(make_golden.py:gen_mover_api); the bar is bitwise equality of every store
array, free space and capacities included.
"""

import numpy as np
import pytest

from conftest import bits_equal, load_golden

pytestmark = pytest.mark.gpu

NC = 23


def _species():
    from paper_2404_10270_b200 import SpeciesDef

    return [SpeciesDef("q", -1.602176634e-19, 9.1093837015e-31),
            SpeciesDef("n", 0.0, 3.3e-27, nstep=3, track_transverse=True)]


def _grid(nc=NC, dx=1e-5):
    from paper_2404_10270_b200 import Grid1D

    return Grid1D.from_cells(nc, nc * dx)


def _fields(g, prefix, isp):
    names = ["x", "vx", "vy", "vz"] + (["yp"] if f"{prefix}sp{isp}_yp" in g else [])
    return {n: g[f"{prefix}sp{isp}_{n}"] for n in names}


def _device_store(g, prefix, species=None):
    from paper_2404_10270_b200.cellstore import CellSortedStore

    species = species or _species()
    n = len(species)
    return CellSortedStore.from_host(_grid(), species, [g[f"{prefix}sp{i}_counts"] for i in range(n)],
                                     [g[f"{prefix}sp{i}_caps"] for i in range(n)],
                                     [_fields(g, prefix, i) for i in range(n)])


class NumpyStore:
    """Host store with the reference CellSortedStore interface (numpy arrays;
    pkg/src/picmc/core.py:100-264), for the staged path of the mover API."""

    def __init__(self, grid, species, counts, caps, data):
        self.grid, self.species = grid, list(species)
        self._counts = [np.array(c, dtype=np.int64) for c in counts]
        self._caps = [np.array(c, dtype=np.int64) for c in caps]
        self._offs = [np.concatenate(([0], np.cumsum(c[:-1]))).astype(np.int64) for c in self._caps]
        self._data = [{k: np.array(v, dtype=np.float64) for k, v in d.items()} for d in data]

    nsp = property(lambda self: len(self.species))
    counts = lambda self, i: self._counts[i]  # noqa: E731
    caps = lambda self, i: self._caps[i]  # noqa: E731
    offsets = lambda self, i: self._offs[i]  # noqa: E731
    data = lambda self, i: self._data[i]  # noqa: E731
    field_names = lambda self, i: tuple(self._data[i])  # noqa: E731

    def reserve(self, isp, j, extra):
        caps = self._caps[isp].copy()
        while self._counts[isp][j] + extra > caps[j]:
            caps[j] = max(2 * caps[j], 4)
        offs = np.concatenate(([0], np.cumsum(caps[:-1]))).astype(np.int64)
        new = {k: np.zeros(int(caps.sum())) for k in self._data[isp]}
        for c in range(self.grid.nc):
            n = self._counts[isp][c]
            for k, v in self._data[isp].items():
                new[k][offs[c]:offs[c] + n] = v[self._offs[isp][c]:self._offs[isp][c] + n]
        self._caps[isp], self._offs[isp], self._data[isp] = caps, offs, new


def _numpy_store(g, prefix):
    sp = _species()
    return NumpyStore(_grid(), sp, [g[f"{prefix}sp{i}_counts"] for i in range(2)],
                      [g[f"{prefix}sp{i}_caps"] for i in range(2)], [_fields(g, prefix, i) for i in range(2)])


def _assert_raw(store, g, prefix):
    for isp in range(store.nsp):
        as_np = lambda a: a.cpu().numpy() if hasattr(a, "cpu") else a  # noqa: E731
        assert np.array_equal(as_np(store.counts(isp)), g[f"{prefix}sp{isp}_counts"]), (prefix, isp)
        assert np.array_equal(as_np(store.caps(isp)), g[f"{prefix}sp{isp}_caps"]), (prefix, isp)
        assert np.array_equal(as_np(store.offsets(isp)), g[f"{prefix}sp{isp}_offs"]), (prefix, isp)
        for name, arr in store.data(isp).items():
            assert bits_equal(as_np(arr), g[f"{prefix}sp{isp}_{name}"]), (prefix, isp, name)


@pytest.mark.parametrize("kind", ["device", "numpy"])
def test_mover_phase_resort_steps_match_reference(cuda, kind):
    """mover_phase + resort for 6 steps with capacity doubling: every store
    array (slot order, zeroed free space, caps, offsets) bitwise the reference's."""
    from paper_2404_10270_b200 import PhysicalConstants
    from paper_2404_10270_b200.mover import mover_phase, resort

    g = load_golden("mover_api.npz")
    store = _device_store(g, "init_") if kind == "device" else _numpy_store(g, "init_")
    consts = PhysicalConstants(dt_s=float(g["dt_s"]))
    for k in range(int(g["steps"])):
        e = g["e_hist"][k]
        if kind == "device":
            import torch
            e = torch.from_numpy(e).to(cuda)
        mover_phase(store, e, consts, None, grainsize=5)
        assert resort(store) == int(g[f"moved{k}"])
        _assert_raw(store, g, f"step{k}_")


@pytest.mark.parametrize("kind", ["device", "numpy"])
def test_resort_collect_movers_match_reference(cuda, kind):
    from paper_2404_10270_b200.mover import push_position, resort_collect

    g = load_golden("mover_api.npz")
    store = _device_store(g, "cinit_") if kind == "device" else _numpy_store(g, "cinit_")
    for isp in range(2):
        push_position(store, isp)
    _assert_raw(store, g, "cpushed_")
    movers = resort_collect(store)
    as_np = lambda a: a.cpu().numpy() if hasattr(a, "cpu") else a  # noqa: E731
    for m in movers:
        assert np.array_equal(as_np(m.dest_cell), g[f"cmov{m.isp}_dest"])
        assert np.array_equal(as_np(m.src_cell), g[f"cmov{m.isp}_src_cell"])
        assert np.array_equal(as_np(m.src_slot), g[f"cmov{m.isp}_src_slot"])
        for name, v in m.fields.items():
            assert bits_equal(as_np(v), g[f"cmov{m.isp}_{name}"]), name
    _assert_raw(store, g, "collected_")


def test_push_velocity_composition_matches_reference(cuda):
    from paper_2404_10270_b200 import PhysicalConstants
    from paper_2404_10270_b200.mover import push_position, push_velocity

    g = load_golden("mover_api.npz")
    store = _device_store(g, "vinit_")
    push_velocity(store, 0, g["v_e_p0"], PhysicalConstants(dt_s=float(g["dt_s"])))
    push_position(store, 0)
    _assert_raw(store, g, "vdone_")


def test_commit_incomers_order_canonical(cuda):
    """Committing a row-permuted Movers gives the identical store
    (pkg/tests/test_mover.py:201-219)."""
    import torch

    from paper_2404_10270_b200.mover import Movers, commit_incomers, push_position, resort_collect

    g = load_golden("mover_api.npz")
    a = _device_store(g, "cinit_")
    push_position(a, 0)
    b = a.clone()
    ma = resort_collect(a)[0]
    mb = resort_collect(b)[0]
    perm = torch.from_numpy(np.random.default_rng(0).permutation(mb.count)).to(cuda)
    shuffled = Movers(mb.isp, mb.dest_cell[perm], mb.src_cell[perm], mb.src_slot[perm],
                      {n: v[perm] for n, v in mb.fields.items()})
    commit_incomers(a, ma)
    commit_incomers(b, shuffled)
    for name in a.field_names(0):
        assert bits_equal(a.data(0)[name].cpu().numpy(), b.data(0)[name].cpu().numpy())
    assert torch.equal(a.counts(0), b.counts(0)) and torch.equal(a.caps(0), b.caps(0))


# -- exact resort cases (pkg/tests/test_mover.py:106-160) ------------------------

def _single(nc):
    from paper_2404_10270_b200 import SpeciesDef
    from paper_2404_10270_b200.cellstore import CellSortedStore

    return CellSortedStore(_grid(nc, 1.0), [SpeciesDef("s", 0.0, 1.0)], initial_cap=4)


def _x_in(store, j):
    sl = store.cell_slice(0, j)
    return store.data(0)["x"][sl].cpu().numpy()


def test_resort_exact_cases(cuda):
    from paper_2404_10270_b200.mover import resort

    s = _single(8)
    s.append(0, 3, {"x": -0.25, "vx": 1.5})
    assert resort(s) == 1
    assert _x_in(s, 2)[0] == 0.75 and float(s.data(0)["vx"][s.cell_slice(0, 2)][0]) == 1.5
    assert int(s.counts(0)[3]) == 0
    s = _single(8)
    s.append(0, 0, {"x": -0.25})
    s.append(0, 7, {"x": 1.25})
    resort(s)
    assert _x_in(s, 7)[0] == 0.75 and _x_in(s, 0)[0] == 0.25
    s = _single(100)
    s.append(0, 0, {"x": -0.3})
    resort(s)
    assert int(s.counts(0)[99]) == 1 and _x_in(s, 99)[0] == -0.3 - np.floor(-0.3)
    s = _single(8)
    s.append(0, 1, {"x": 2.0})
    s.append(0, 2, {"x": 3.5})
    resort(s)
    assert _x_in(s, 3)[0] == 0.0 and _x_in(s, 5)[0] == 0.5
    s = _single(8)
    s.append(0, 4, {"x": -1e-18})
    resort(s)
    assert int(s.counts(0)[4]) == 1 and _x_in(s, 4)[0] == 0.0
    s.check_sorted(0)


def test_resort_rejects_domain_scale_jump(cuda):
    from paper_2404_10270_b200.errors import CflViolation
    from paper_2404_10270_b200.mover import resort

    s = _single(8)
    s.append(0, 0, {"x": 8.5})
    before = s.data(0)["x"].clone()
    with pytest.raises(CflViolation, match="whole domain"):
        resort(s)
    assert bits_equal(s.data(0)["x"].cpu().numpy(), before.cpu().numpy())


def test_push_velocity_rejects_neutrals_and_bad_length(cuda):
    from paper_2404_10270_b200 import PhysicalConstants
    from paper_2404_10270_b200.errors import ContractViolation
    from paper_2404_10270_b200.mover import push_velocity

    g = load_golden("mover_api.npz")
    store = _device_store(g, "vinit_")
    consts = PhysicalConstants(dt_s=4e-14)
    with pytest.raises(ContractViolation, match="neutral"):
        push_velocity(store, 1, np.zeros(store.total(1)), consts)
    with pytest.raises(ContractViolation, match="length"):
        push_velocity(store, 0, np.zeros(3), consts)


def test_negative_zero_and_accel_nodes_and_tasks(cuda):
    import torch

    from paper_2404_10270_b200 import PhysicalConstants, SpeciesDef
    from paper_2404_10270_b200.mover import (Movers, accel_nodes_for_species, push_position,
                                             submit_move_tasks, velocity_kick_coef)

    s = _single(4)
    s.append(0, 1, {"x": 0.5, "vx": -0.0})
    push_position(s, 0)
    vx = float(s.data(0)["vx"][s.cell_slice(0, 1)][0])
    assert vx == 0.0 and np.signbit(vx)

    from paper_2404_10270_b200.cellstore import CellSortedStore
    from paper_2404_10270_b200.core import ELECTRON_MASS, ELEMENTARY_CHARGE

    species = [SpeciesDef("a", -ELEMENTARY_CHARGE, ELECTRON_MASS), SpeciesDef("b", 0.0, 1.0),
               SpeciesDef("hold", ELEMENTARY_CHARGE, 1.0, active_mover=False), SpeciesDef("d", 0.0, 2.0),
               SpeciesDef("e2", 0.0, 3.0)]
    store = CellSortedStore(_grid(10, 1.0), species, initial_cap=4)
    consts = PhysicalConstants(dt_s=2e-12)
    e = torch.ones(11, dtype=torch.float64, device=cuda)
    accel = accel_nodes_for_species(store, e, consts)
    assert accel[0] is not None and all(a is None for a in accel[1:])
    assert bits_equal(accel[0].cpu().numpy(), velocity_kick_coef(species[0], consts, 1.0) * np.ones(11))

    class Sched:
        def __init__(self):
            self.log = []

        def submit_work(self, fn, queue, tag):
            self.log.append((tag, queue))
            fn()

        def wait(self, queues):
            pass

    sched = Sched()
    queues = submit_move_tasks(sched, store, accel, grainsize=100, queue_offset=3)
    assert sorted(t for t, _ in sched.log) == ["move:a", "move:b", "move:d", "move:e2"]
    assert queues == {3, 4, 6} and dict(sched.log)["move:e2"] == 3

    empty = Movers.empty(0, ("x", "vx", "vy", "vz"))
    one = Movers(0, np.array([2]), np.array([1]), np.array([0]),
                 {"x": np.array([0.5]), "vx": np.array([1.0]), "vy": np.array([0.0]), "vz": np.array([0.0])})
    cat = Movers.concat([empty, one, one])
    assert cat.count == 2 and list(cat.fields["x"]) == [0.5, 0.5]


def test_cellstore_growth_and_swap_remove(cuda):
    """append beyond capacity doubles the cell (max(2*cap, 4)) and keeps the
    other cells' live segments; swap_remove fills from the end and zeroes."""
    s = _single(5)
    for k in range(9):
        s.append(0, 2, {"x": k / 16, "vx": float(k)})
    s.append(0, 4, {"x": 0.5})
    assert s.caps(0).tolist() == [4, 4, 16, 4, 4]
    assert s.offsets(0).tolist() == [0, 4, 8, 24, 28]
    assert _x_in(s, 2).tolist() == [k / 16 for k in range(9)]
    rec = s.swap_remove(0, 2, 3)
    assert rec["vx"] == 3.0 and _x_in(s, 2)[3] == 8 / 16
    assert float(s.data(0)["x"][8 + 8]) == 0.0
    assert s.live_indices(0).tolist() == list(range(8, 16)) + [28]
    assert s.cell_of_live(0).tolist() == [2] * 8 + [4]
