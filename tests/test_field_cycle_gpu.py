"""GPU: the field step entry point (pb_field_cycle: the density epilogue
with the first smoothing pass folded into one kernel, then the scan Poisson
solve and E) against the separate calls it stands for -- pb_rho_epilogue +
pb_smooth_density + pb_solve_poisson_scan + pb_compute_efield_clear.

Bar: bitwise for every output (left, right, rho, rho_s, phi, E), both bin
sets zeroed, the overflow flag raised the same way, repeated calls agree,
and at engine level a run through the field-step path (the read bin set
zeroed and the wall compaction run on the side stream, overlapping the next
field step / push) equals the per-phase serial run particle for particle.
"""

import ctypes

import numpy as np
import pytest

from conftest import bits_equal
from test_engine_gpu import _mk_config, _random_flats

pytestmark = pytest.mark.gpu


def _bins(nc, ndep, seed, max_count=300):
    rng = np.random.default_rng(seed)
    C = rng.integers(0, max_count, size=(ndep, nc)).astype(np.uint64)
    # R = sum of per-particle round(x * 2^48) <= C * 2^48
    R = (rng.random((ndep, nc)) * C.astype(np.float64) * 2.0 ** 48).astype(np.uint64)
    return np.stack([R, C], axis=1).reshape(-1)


def _chain(lib, bins, coef, ndep, nc, bc, passes, dx, eps0, pl, pr, dev, fused):
    import torch

    from paper_2404_10270_b200 import _lib

    t = lambda n: torch.zeros(n, dtype=torch.float64, device=dev)  # noqa: E731
    out = {k: t(nc + 1) for k in ("rho", "rho_s", "phi", "e")}
    out["left"], out["right"] = t(nc), t(nc)
    b0 = torch.from_numpy(bins.view(np.int64).copy()).to(dev)
    b1 = torch.from_numpy(bins.view(np.int64).copy()).to(dev)
    scr = torch.zeros(lib.pb_field_scratch_bytes(nc), dtype=torch.uint8, device=dev)
    from paper_2404_10270_b200.store import status_template

    st = status_template(dev)
    c = (ctypes.c_double * max(ndep, 1))(*coef)
    sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    P = lambda x: x.data_ptr()  # noqa: E731
    if fused:
        for _ in range(2):  # repeated calls agree
            b0.copy_(torch.from_numpy(bins.view(np.int64)))
            b1.copy_(torch.from_numpy(bins.view(np.int64)))
            _lib.check(lib.pb_field_cycle(P(b0), c, ndep, nc, bc, passes, dx, eps0, pl, pr, P(out["left"]),
                                          P(out["right"]), P(out["rho"]), P(out["rho_s"]), P(out["phi"]),
                                          P(out["e"]), P(b0), P(b1), b0.numel(), P(st), P(scr), None, 0, None, 0, sh),
                       "pb_field_cycle")
    else:
        _lib.check(lib.pb_rho_epilogue(P(b0), c, ndep, nc, bc, P(out["left"]), P(out["right"]), P(out["rho"]),
                                       P(st), sh), "epilogue")
        _lib.check(lib.pb_smooth_density(P(out["rho"]), P(out["rho_s"]), nc, passes, P(scr), sh), "smooth")
        _lib.check(lib.pb_solve_poisson_scan(P(out["rho_s"]), P(out["phi"]), nc, dx, eps0, bc, pl, pr, P(scr),
                                             sh), "poisson")
        _lib.check(lib.pb_compute_efield_clear(P(out["phi"]), P(out["e"]), nc, dx, bc, P(b0), P(b1),
                                               b0.numel(), sh), "efield")
    torch.cuda.synchronize()
    res = {k: v.cpu().numpy() for k, v in out.items()}
    res["bins_zero"] = not (b0.any().item() or b1.any().item())
    res["status"] = st.cpu().numpy()
    return res


@pytest.mark.parametrize("nc", [37, 1000, 65536, 100_001, 1_000_000])
@pytest.mark.parametrize("bc", ["periodic", "dirichlet"])
@pytest.mark.parametrize("passes", [0, 1, 3])
def test_field_cycle_bitwise_vs_per_phase_chain(cuda, nc, bc, passes):
    from paper_2404_10270_b200 import _lib

    lib = _lib.load()
    code = _lib.PB_FIELD_PERIODIC if bc == "periodic" else _lib.PB_FIELD_DIRICHLET
    ndep = 2
    bins = _bins(nc, ndep, seed=nc + passes)
    coef = [-1.7e-9, 2.3e-9]
    args = (lib, bins, coef, ndep, nc, code, passes, 1e-5, 8.8541878128e-12, 3.0, -1.25, cuda)
    a = _chain(*args, fused=False)
    b = _chain(*args, fused=True)
    for k in ("left", "right", "rho", "rho_s", "phi", "e"):
        assert bits_equal(a[k], b[k]), k
    assert a["bins_zero"] and b["bins_zero"]
    assert np.array_equal(a["status"], b["status"])


def test_field_cycle_flags_overflow(cuda):
    from paper_2404_10270_b200 import _lib

    lib = _lib.load()
    nc, ndep = 4096, 1
    bins = _bins(nc, ndep, seed=3)
    bins[nc + 1234] = 70000  # C of cell 1234: past the fixed-point capacity
    args = (lib, bins, [1e-9], ndep, nc, _lib.PB_FIELD_DIRICHLET, 1, 1e-5, 8.85e-12, 0.0, 0.0, cuda)
    a = _chain(*args, fused=False)
    b = _chain(*args, fused=True)
    assert np.array_equal(a["status"], b["status"])
    from paper_2404_10270_b200.store import decode_status

    st = decode_status(b["status"])
    assert st.code == _lib.PB_ERR_OVERFLOW and st.overflow == 70000


@pytest.mark.parametrize("case", ["dirichlet_absorbing", "periodic_boris"])
def test_engine_fused_cycle_matches_per_phase(cuda, case):
    """Engine runs with poisson = "scan": fused cycle vs the per-phase
    kernels, eager and graph-replayed -- rho, rho_s, phi, E, bins and every
    particle bit for bit."""
    from paper_2404_10270_b200 import Engine

    kw = dict(field_solve=True, smoothing_passes=1, poisson="scan", phi_left=1.5, phi_right=-0.5)
    if case == "dirichlet_absorbing":
        kw.update(boundary="dirichlet", particle_boundary="absorbing")
        species = None
    else:
        kw.update(boundary="periodic", b_field_t=(0.1, 0.2, 1.5))
        species = None
    cfg = _mk_config(nc=3000, ppc0=4, species=species, **kw)
    flats = _random_flats(cfg, 23, vscale=0.45)
    a = Engine(cfg, device=cuda, check_every=0)
    b = Engine(cfg, device=cuda, check_every=0)
    a.fused_field = False
    assert b._fused_ok() and not a._fused_ok()
    a.upload(flats)
    b.upload(flats)
    for _ in range(3):
        a.step()
        b.step()
    b.prepare_graphs(40)
    for _ in range(6):
        a.step()
    b.replay(6)
    a.sync()
    b.sync()
    for name in ("rho", "rho_s", "phi", "e", "left", "right"):
        assert bits_equal(getattr(a, name).cpu().numpy(), getattr(b, name).cpu().numpy()), name
    assert np.array_equal(a.bins_pp[0].cpu().numpy(), b.bins_pp[0].cpu().numpy())
    assert np.array_equal(a.bins_pp[1].cpu().numpy(), b.bins_pp[1].cpu().numpy())
    for x, y in zip(a.download(), b.download()):
        assert x.n == y.n
        for k in x.fields():
            assert bits_equal(x.fields()[k], y.fields()[k]), k


@pytest.mark.parametrize("bc", ["periodic", "dirichlet"])
@pytest.mark.parametrize("nc,passes", [(65536, 4), (65536, 5), (3, 1), (4, 0), (512, 2), (513, 1), (514, 1),
                                       (1025, 3), (1026, 2), (1027, 1)])
def test_field_cycle_edges_bitwise(cuda, nc, bc, passes):
    """The single-launch cycle at its limits: the largest pass count it takes
    (4), the per-phase fallback past it (5), one tile (nc <= 513), and last
    tiles that are full (nc = 512 m + 1), hold one unknown (its first is its
    last: nc = 512 m + 2) or two."""
    from paper_2404_10270_b200 import _lib

    lib = _lib.load()
    code = _lib.PB_FIELD_PERIODIC if bc == "periodic" else _lib.PB_FIELD_DIRICHLET
    bins = _bins(nc, 3, seed=7 * nc + passes)
    args = (lib, bins, [-1.1e-9, 2.9e-9, 0.7e-9], 3, nc, code, passes, 2e-5, 8.8541878128e-12, -0.5, 2.0, cuda)
    a = _chain(*args, fused=False)
    b = _chain(*args, fused=True)
    for k in ("left", "right", "rho", "rho_s", "phi", "e"):
        assert bits_equal(a[k], b[k]), k
    assert a["bins_zero"] and b["bins_zero"]


@pytest.mark.parametrize("bc", ["periodic", "dirichlet"])
def test_field_cycle_epochs_and_graph_replay(cuda, bc):
    """One scratch over many launches (the flags' launch epoch advances
    every call) and inside a replayed CUDA graph: every call equals the
    per-phase chain on its own bins."""
    import torch

    from paper_2404_10270_b200 import _lib
    from paper_2404_10270_b200.store import status_template

    lib = _lib.load()
    code = _lib.PB_FIELD_PERIODIC if bc == "periodic" else _lib.PB_FIELD_DIRICHLET
    nc, ndep, passes = 40000, 2, 1
    coef = [-1.7e-9, 2.3e-9]
    c = (ctypes.c_double * ndep)(*coef)
    t = lambda n: torch.zeros(n, dtype=torch.float64, device=cuda)  # noqa: E731
    out = {k: t(nc + 1) for k in ("rho", "rho_s", "phi", "e")}
    left, right = t(nc), t(nc)
    scr = torch.zeros(lib.pb_field_scratch_bytes(nc), dtype=torch.uint8, device=cuda)
    st = status_template(cuda)
    b0 = torch.zeros(2 * ndep * nc, dtype=torch.int64, device=cuda)
    src = torch.zeros_like(b0)
    P = lambda x: x.data_ptr()  # noqa: E731

    def call(stream):
        b0.copy_(src)
        _lib.check(lib.pb_field_cycle(P(b0), c, ndep, nc, code, passes, 1e-5, 8.8541878128e-12, 1.0, 0.0,
                                      P(left), P(right), P(out["rho"]), P(out["rho_s"]), P(out["phi"]),
                                      P(out["e"]), P(b0), None, b0.numel(), P(st), P(scr), None, 0, None, 0,
                                      ctypes.c_void_p(stream.cuda_stream)), "pb_field_cycle")

    s = torch.cuda.Stream(cuda)
    g = torch.cuda.CUDAGraph()
    for it in range(12):
        bins = _bins(nc, ndep, seed=100 + it)
        src.copy_(torch.from_numpy(bins.view(np.int64)))
        if it < 6:
            with torch.cuda.stream(s):
                call(s)
        else:
            if it == 6:
                with torch.cuda.graph(g, stream=s):
                    call(torch.cuda.current_stream())
            g.replay()
        torch.cuda.synchronize()
        ref = _chain(lib, bins, coef, ndep, nc, code, passes, 1e-5, 8.8541878128e-12, 1.0, 0.0, cuda,
                     fused=False)
        for k in ("rho", "rho_s", "phi", "e"):
            assert bits_equal(ref[k], out[k].cpu().numpy()), (it, k)
        assert not b0.any().item()


def test_folded_compaction_flushes_before_direct_push_and_reads(cuda):
    """Absorbing walls on the single-launch field path: a step leaves its
    holes to the next field launch.  A direct push() / totals() / download()
    / sort in between must see (and push) compacted stores only: same
    particles, counts and tallies as the engine that compacts every step."""
    from paper_2404_10270_b200 import Engine

    kw = dict(field_solve=True, smoothing_passes=1, poisson="scan", boundary="dirichlet",
              particle_boundary="absorbing", phi_left=0.0, phi_right=0.0)
    cfg = _mk_config(nc=2000, ppc0=8, **kw)
    flats = _random_flats(cfg, 5, vscale=0.9)  # fast particles: many wall removals
    a = Engine(cfg, device=cuda, check_every=0)
    b = Engine(cfg, device=cuda, check_every=0)
    b.fold_compaction = False
    assert a._folds_compaction() and not b._folds_compaction()
    a.upload(flats)
    b.upload(flats)
    for _ in range(3):
        a.step()
        b.step()
    assert a._holes_pending
    assert a.totals() == b.totals()  # flushes a's holes
    for _ in range(2):
        a.step()
        b.step()
    a.push()  # direct push with the last step's holes pending
    b.push()
    a.sort_by_cell()
    b.sort_by_cell()
    a.sync()
    b.sync()
    assert np.array_equal(a.absorbed, b.absorbed) and a.absorbed.sum() > 0
    from oracle import oracle

    for x, y in zip(a.download(), b.download()):
        assert x.n == y.n
        assert np.array_equal(oracle.canonical(x.cell, x.fields()), oracle.canonical(y.cell, y.fields()))
