"""GPU shims vs the reference kernels, bit for bit.

Template: pkg/tests/test_backends.py:48-127 (compiled vs pure over packed
stores with per-cell free space, 5 seeds, every flag combination).  The
comparator is the reference's own compiled `_kernels` (oracle/_ref, built
from /root/reference sources) when present, else the C restatement.
"""

import numpy as np
import pytest

from conftest import bits_equal, packed

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    from oracle import oracle

    mod = oracle.ref_kernels()
    return mod if mod is not None else oracle


@pytest.fixture(scope="module")
def cu(cuda):
    from paper_2404_10270_b200 import backends

    return backends.load_backend("cuda")


@pytest.mark.parametrize("seed", range(5))
def test_deposit_partials_bitwise(seed, ref, cu):
    x, _, _, _, offs, counts = packed(seed)
    lr, rr = ref.deposit_partials(x, offs, counts)
    lc, rc = cu.deposit_partials(x, offs, counts)
    assert bits_equal(lr, lc) and bits_equal(rr, rc)


@pytest.mark.parametrize("seed", range(5))
def test_gather_bitwise(seed, ref, cu):
    x, _, _, _, offs, counts = packed(seed)
    nodes = np.random.default_rng(100 + seed).standard_normal(len(counts) + 1)
    assert bits_equal(ref.gather(nodes, x, offs, counts), cu.gather(nodes, x, offs, counts))


@pytest.mark.parametrize("seed", range(5))
@pytest.mark.parametrize("with_accel", [True, False])
@pytest.mark.parametrize("with_yp", [True, False])
def test_fused_move_bitwise(seed, with_accel, with_yp, ref, cu):
    x, vx, vy, yp, offs, counts = packed(seed)
    accel = (np.random.default_rng(200 + seed).standard_normal(len(counts) + 1) * 0.1
             if with_accel else None)
    a = [x.copy(), vx.copy(), vy.copy(), yp.copy() if with_yp else None]
    b = [x.copy(), vx.copy(), vy.copy(), yp.copy() if with_yp else None]
    ref.fused_move(accel, *a, offs, counts, 2.0)
    cu.fused_move(accel, *b, offs, counts, 2.0)
    for u, v in zip(a, b):
        if u is not None:
            assert bits_equal(u, v)


def test_empty_inputs(cu):
    offs = np.zeros(4, dtype=np.int64)
    counts = np.zeros(4, dtype=np.int64)
    x = np.zeros(0)
    left, right = cu.deposit_partials(x, offs, counts)
    assert bits_equal(left, np.zeros(4)) and bits_equal(right, np.zeros(4))
    assert cu.gather(np.zeros(5), x, offs, counts).size == 0


def test_large_packed_store_bitwise(ref, cu):
    """C2-like cell occupancy (ppc ~100, cap 150) at 200K particles."""
    rng = np.random.default_rng(5)
    nc, cap = 2000, 150
    counts = rng.integers(50, 151, size=nc).astype(np.int64)
    offs = (np.arange(nc, dtype=np.int64) * cap)
    total = nc * cap
    x = np.zeros(total)
    vx = np.zeros(total)
    for j in range(nc):
        sl = slice(offs[j], offs[j] + counts[j])
        x[sl] = rng.random(counts[j])
        vx[sl] = rng.standard_normal(counts[j]) * 0.01
    accel = 1e-3 * np.sin(np.arange(nc + 1) * 0.01)
    a = [x.copy(), vx.copy()]
    b = [x.copy(), vx.copy()]
    ref.fused_move(accel, a[0], a[1], np.zeros(total), None, offs, counts, 1.0)
    cu.fused_move(accel, b[0], b[1], np.zeros(total), None, offs, counts, 1.0)
    assert bits_equal(a[0], b[0]) and bits_equal(a[1], b[1])
    lr, rr = ref.deposit_partials(x, offs, counts)
    lc, rc = cu.deposit_partials(x, offs, counts)
    assert bits_equal(lr, lc) and bits_equal(rr, rc)


def test_negative_zero_survives_uncharged_push(cu):
    """accel None must skip the kick: -0.0 velocities stay -0.0
    (pkg/tests/test_mover.py:240-246)."""
    offs = np.array([0, 4], dtype=np.int64)
    counts = np.array([1, 0], dtype=np.int64)
    x = np.array([0.5, 0, 0, 0, 0, 0, 0, 0.0])
    vx = np.array([-0.0, 0, 0, 0, 0, 0, 0, 0.0])
    cu.fused_move(None, x, vx, np.zeros(8), None, offs, counts, 1.0)
    assert vx[0] == 0.0 and np.signbit(vx[0])
    acc = np.full(3, -0.0)
    cu.fused_move(acc, x, vx, np.zeros(8), None, offs, counts, 1.0)
    assert vx[0] == 0.0 and not np.signbit(vx[0])  # charged species: kicked


def test_dtype_and_contiguity_errors(cu):
    x, vx, vy, yp, offs, counts = packed(0)
    with pytest.raises(ValueError):
        cu.deposit_partials(x.astype(np.float32), offs, counts)
    with pytest.raises(ValueError):
        cu.deposit_partials(x[::2], offs, counts)


@pytest.mark.parametrize("seed", range(5))
@pytest.mark.parametrize("with_accel", [True, False])
@pytest.mark.parametrize("with_yp", [True, False])
def test_fused_move_aos_and_table_bitwise(seed, with_accel, with_yp, cu):
    """The layout-study kernels (_kernels.pyx:105-152) vs the reference's
    compiled outputs (golden), numpy and CUDA-tensor inputs."""
    import torch

    from conftest import load_golden

    g = load_golden("backend_kernels.npz")
    x, vx, vy, yp, offs, counts = packed(seed)
    accel = g[f"s{seed}_accel"]
    tab = np.stack([x, vx, vy, np.zeros_like(x), yp], axis=1).copy()
    t = tab.copy()
    cu.fused_move_aos(t, offs, counts, accel, 3.0, with_accel, with_yp)
    want = g[f"s{seed}_aos_a{int(with_accel)}y{int(with_yp)}"]
    assert bits_equal(t.ravel(), want.ravel())
    td = torch.from_numpy(tab.copy()).cuda()
    cu.fused_move_aos(td, torch.from_numpy(offs).cuda(), torch.from_numpy(counts).cuda(),
                      torch.from_numpy(accel).cuda(), 3.0, with_accel, with_yp)
    assert bits_equal(td.cpu().numpy().ravel(), want.ravel())
    t = tab[: int(counts[0])].copy()
    cu.fused_move_table(t, 0.3, -0.2, 2.0, True, True)
    assert bits_equal(t.ravel(), g[f"s{seed}_table"].ravel())


def test_concurrent_block_calls_match_serial(ref, cu):
    """The reference's call pattern (pkg/src/picmc/mover.py:251-270): one
    fused_move per block of `grainsize` cells on the SAME species arrays,
    from several threads at once.  Each call stages and writes back only its
    block's slot span, so the result equals the serial compiled run."""
    from concurrent.futures import ThreadPoolExecutor

    rng = np.random.default_rng(11)
    nc, cap, grain = 301, 12, 7
    counts = rng.integers(0, cap + 1, size=nc).astype(np.int64)
    offs = np.arange(nc, dtype=np.int64) * cap
    total = nc * cap
    arrs = [np.zeros(total) for _ in range(4)]
    for j in range(nc):
        sl = slice(offs[j], offs[j] + counts[j])
        arrs[0][sl] = rng.random(counts[j])
        for a in arrs[1:]:
            a[sl] = rng.standard_normal(counts[j]) * 0.4
    accel = rng.standard_normal(nc + 1) * 0.05
    a = [v.copy() for v in arrs]
    b = [v.copy() for v in arrs]
    blocks = [(lo, min(lo + grain, nc)) for lo in range(0, nc, grain)]
    for lo, hi in blocks:
        ref.fused_move(accel[lo:hi + 1], a[0], a[1], a[2], a[3], offs[lo:hi], counts[lo:hi], 3.0)
    with ThreadPoolExecutor(8) as ex:
        list(ex.map(lambda blk: cu.fused_move(accel[blk[0]:blk[1] + 1], b[0], b[1], b[2], b[3],
                                              offs[blk[0]:blk[1]], counts[blk[0]:blk[1]], 3.0),
                    blocks * 1))
    for u, v in zip(a, b):
        assert bits_equal(u, v)
    # deposit / gather per block, concurrently, equal the serial calls
    with ThreadPoolExecutor(8) as ex:
        got = list(ex.map(lambda blk: cu.deposit_partials(b[0], offs[blk[0]:blk[1]],
                                                          counts[blk[0]:blk[1]]), blocks))
    for (lo, hi), (lc, rc) in zip(blocks, got):
        lr, rr = ref.deposit_partials(a[0], offs[lo:hi], counts[lo:hi])
        assert bits_equal(lr, lc) and bits_equal(rr, rc)
        assert bits_equal(ref.gather(accel[lo:hi + 1], a[0], offs[lo:hi], counts[lo:hi]),
                          cu.gather(accel[lo:hi + 1], b[0], offs[lo:hi], counts[lo:hi]))


def test_block_span_out_of_bounds_raises(cu):
    x, vx, vy, yp, offs, counts = packed(0)
    bad = offs.copy()
    bad[-1] = x.shape[0]
    counts = counts.copy()
    counts[-1] = 1
    with pytest.raises(ValueError):
        cu.fused_move(None, x, vx, vy, yp, bad, counts, 1.0)
