"""The `cuda` kernel backend with the reference's operator signatures.

Drop-in for `picmc.backends.{deposit_partials, gather, fused_move,
fused_move_table, fused_move_aos}` (pkg/src/picmc/backends/__init__.py:45-50,
compiled twin pkg/src/picmc/backends/_kernels.pyx:14-152): the same arguments
(C-contiguous float64 / int64 NumPy arrays, packed cell-sorted layout), the
same in-place mutation and return conventions, bitwise-identical results.
Arrays may also be CUDA torch tensors, in which case nothing crosses PCIe.

Call pattern of the reference.  `submit_move_tasks` (pkg/src/picmc/mover.py:
227-271) hands one task per block of `grainsize` cells to a thread pool
(pkg/src/picmc/scheduler.py:143-159); every task passes the WHOLE species
arrays plus the block's `offs`/`counts` slices, and tasks of one species run
concurrently.  A host call here therefore stages only the block's slot span
`[min offs, max offs+counts)` of each array (cells of different blocks own
disjoint spans of the packed store, pkg/src/picmc/core.py:120-181), with the
offsets rebased to the span, and writes back only that span: concurrent calls
on disjoint blocks never touch each other's slots, and PCIe traffic is the
block's span rather than the whole store.  Each host thread uses its own CUDA
stream, so calls from different worker threads overlap on the device.

Every call runs on the GPU through libpicmc_b200.so; there is no CPU path.
"""

import ctypes
import threading

import numpy as np
import torch

from . import _lib

BACKEND_NAME = "cuda"

_tls = threading.local()


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("backend 'cuda' needs a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _thread_stream(dev):
    """One CUDA stream per host thread (the scheduler's workers call
    concurrently; the default stream would serialise them)."""
    s = getattr(_tls, "stream", None)
    if s is None or s.device != dev:
        s = torch.cuda.Stream(device=dev)
        _tls.stream = s
    return s


def _check_np(a, dtype, name, ndim=1):
    # The Cython buffer checks raise ValueError on dtype/contiguity mismatch.
    if not isinstance(a, np.ndarray):
        raise TypeError(f"{name}: expected a numpy array or CUDA tensor")
    if a.dtype != dtype:
        raise ValueError(f"Buffer dtype mismatch for {name}: expected {np.dtype(dtype)}, got {a.dtype}")
    if a.ndim != ndim or not a.flags.c_contiguous:
        raise ValueError(f"{name}: ndarray is not C-contiguous {ndim}-D")


def _check_dev(a, dtype, name, ndim=1):
    want = torch.float64 if dtype == np.float64 else torch.int64
    if not a.is_cuda or a.dtype != want or not a.is_contiguous() or a.dim() != ndim:
        raise ValueError(f"{name}: expected a contiguous {ndim}-D CUDA {want} tensor")


def _as_dev(a, dtype, name, dev, ndim=1):
    """Device-path argument: a CUDA tensor is checked and used in place; a
    host array (small per-call inputs: nodes, offs, counts) is copied."""
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        _check_dev(a, dtype, name, ndim)
        return a
    _check_np(a, dtype, name, ndim)
    return torch.from_numpy(a).to(dev)


def _span(offs, counts, length, what):
    """Slot span [lo, hi) covering every live slot of the block; raises
    ValueError if a cell's live slots fall outside the array (the compiled
    kernel would read out of bounds there)."""
    if counts.shape[0] != offs.shape[0]:
        raise ValueError(f"{what}: offs and counts differ in length")
    live = counts > 0
    if (counts < 0).any():
        raise ValueError(f"{what}: negative count")
    if not live.any():
        return 0, 0
    o = offs[live]
    e = o + counts[live]
    lo, hi = int(o.min()), int(e.max())
    if lo < 0 or hi > length:
        raise ValueError(f"{what}: live slots [{lo}, {hi}) outside an array of {length}")
    return lo, hi


class _Call:
    """One host call: per-thread stream, span staging, span write-back."""

    def __init__(self):
        self.dev = _dev()
        self.stream = _thread_stream(self.dev)
        self.back = []
        self._ctx = torch.cuda.stream(self.stream)

    def __enter__(self):
        self._ctx.__enter__()
        return self

    def __exit__(self, *exc):
        self._ctx.__exit__(*exc)
        return False

    @property
    def handle(self):
        return ctypes.c_void_p(self.stream.cuda_stream)

    def put(self, a, lo=None, hi=None, writeback=False):
        """Device copy of host array a[lo:hi] (whole array if lo is None)."""
        if a is None:
            return None
        part = a if lo is None else a[lo:hi]
        t = torch.from_numpy(part).to(self.dev, non_blocking=False)
        if writeback:
            self.back.append((part, t))
        return t

    def finish(self):
        self.stream.synchronize()
        for part, t in self.back:
            part[...] = t.cpu().numpy()


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _block_offsets(offs, counts, x, what):
    """(lo, hi, rebased offs) for host arrays; validates dtypes."""
    _check_np(offs, np.int64, "offs")
    _check_np(counts, np.int64, "counts")
    lo, hi = _span(offs, counts, x.shape[0], what)
    return lo, hi, np.ascontiguousarray(offs - lo, dtype=np.int64)


def deposit_partials(x, offs, counts):
    """Per-cell raw CIC sums L[j] = sum(1-x), R[j] = sum(x), in slot order."""
    lib = _lib.load()
    if isinstance(x, torch.Tensor):
        _check_dev(x, np.float64, "x")
        offs = _as_dev(offs, np.int64, "offs", x.device)
        counts = _as_dev(counts, np.int64, "counts", x.device)
        nc = int(counts.shape[0])
        left = torch.zeros(nc, dtype=torch.float64, device=x.device)
        right = torch.zeros(nc, dtype=torch.float64, device=x.device)
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(lib.pb_deposit_partials(_ptr(x), _ptr(offs), _ptr(counts), nc, _ptr(left),
                                           _ptr(right), s), "deposit_partials")
        return left, right
    _check_np(x, np.float64, "x")
    lo, hi, roffs = _block_offsets(offs, counts, x, "deposit_partials")
    nc = int(counts.shape[0])
    with _Call() as c:
        xd = c.put(x, lo, hi)
        od = c.put(roffs)
        cd = c.put(counts)
        left = torch.zeros(nc, dtype=torch.float64, device=c.dev)
        right = torch.zeros(nc, dtype=torch.float64, device=c.dev)
        _lib.check(lib.pb_deposit_partials(_ptr(xd), _ptr(od), _ptr(cd), nc, _ptr(left),
                                           _ptr(right), c.handle), "deposit_partials")
        c.finish()
        return left.cpu().numpy(), right.cpu().numpy()


def gather(nodes, x, offs, counts):
    """Per-particle a[j] + x*(a[j+1]-a[j]) in live (cell-major) order."""
    lib = _lib.load()
    if isinstance(x, torch.Tensor):
        _check_dev(x, np.float64, "x")
        nodes = _as_dev(nodes, np.float64, "nodes", x.device)
        offs = _as_dev(offs, np.int64, "offs", x.device)
        counts = _as_dev(counts, np.int64, "counts", x.device)
        nc = int(counts.shape[0])
        total = int(counts.sum().item()) if nc else 0
        out = torch.empty(total, dtype=torch.float64, device=x.device)
        if total:
            s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
            _lib.check(lib.pb_gather(_ptr(nodes), _ptr(x), _ptr(offs), _ptr(counts), nc, _ptr(out),
                                     s), "gather")
        return out
    _check_np(nodes, np.float64, "nodes")
    _check_np(x, np.float64, "x")
    lo, hi, roffs = _block_offsets(offs, counts, x, "gather")
    nc = int(counts.shape[0])
    total = int(counts.sum()) if nc else 0
    if total and nodes.shape[0] < nc + 1:
        raise ValueError("nodes must have len(counts)+1 entries")
    if total == 0:
        return np.empty(0, dtype=np.float64)
    with _Call() as c:
        nd = c.put(nodes)
        xd = c.put(x, lo, hi)
        od = c.put(roffs)
        cd = c.put(counts)
        out = torch.empty(total, dtype=torch.float64, device=c.dev)
        _lib.check(lib.pb_gather(_ptr(nd), _ptr(xd), _ptr(od), _ptr(cd), nc, _ptr(out), c.handle),
                   "gather")
        c.finish()
        return out.cpu().numpy()


def fused_move(accel_nodes, x, vx, vy, yp, offs, counts, fnstep):
    """One fused gather+push step over the block's live particles, in place.

    accel_nodes None skips the kick entirely (no `+= 0.0`, which would turn
    -0.0 velocities into +0.0; pkg/src/picmc/mover.py:214-216).
    """
    lib = _lib.load()
    nc = int(counts.shape[0])
    if isinstance(x, torch.Tensor):
        for a, n in ((x, "x"), (vx, "vx"), (vy, "vy"), (yp, "yp")):
            if a is not None:
                _check_dev(a, np.float64, n)
        accel_nodes = _as_dev(accel_nodes, np.float64, "accel_nodes", x.device)
        offs = _as_dev(offs, np.int64, "offs", x.device)
        counts = _as_dev(counts, np.int64, "counts", x.device)
        if accel_nodes is not None and int(accel_nodes.shape[0]) < nc + 1:
            raise ValueError("accel_nodes must have len(counts)+1 entries")
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(lib.pb_fused_move(_ptr(accel_nodes), _ptr(x), _ptr(vx),
                                     _ptr(vy if yp is not None else None), _ptr(yp), _ptr(offs),
                                     _ptr(counts), nc, float(fnstep), s), "fused_move")
        return None
    for a, n in ((x, "x"), (vx, "vx"), (vy, "vy")):
        _check_np(a, np.float64, n)
    if yp is not None:
        _check_np(yp, np.float64, "yp")
    if accel_nodes is not None:
        _check_np(accel_nodes, np.float64, "accel_nodes")
    lo, hi, roffs = _block_offsets(offs, counts, x, "fused_move")
    for a, n in ((vx, "vx"), (vy, "vy"), (yp, "yp")):
        if a is not None and a.shape[0] < hi:
            raise ValueError(f"fused_move: {n} shorter than the block's slot span")
    if hi == lo:
        return None
    if accel_nodes is not None and int(accel_nodes.shape[0]) < nc + 1:
        raise ValueError("accel_nodes must have len(counts)+1 entries")
    with _Call() as c:
        ad = c.put(accel_nodes)
        xd = c.put(x, lo, hi, writeback=True)
        vxd = c.put(vx, lo, hi, writeback=accel_nodes is not None)
        vyd = c.put(vy, lo, hi) if yp is not None else None
        ypd = c.put(yp, lo, hi, writeback=True)
        od = c.put(roffs)
        cd = c.put(counts)
        _lib.check(lib.pb_fused_move(_ptr(ad), _ptr(xd), _ptr(vxd), _ptr(vyd), _ptr(ypd), _ptr(od),
                                     _ptr(cd), nc, float(fnstep), c.handle), "fused_move")
        c.finish()
    return None


def fused_move_aos(tab, starts, counts, accel_nodes, fnstep, has_accel, has_yp):
    """fused_move over a cell-major array-of-structs table (columns x, vx,
    vy, vz[, yp]) in place (_kernels.pyx:128-152); only the block's row span
    is staged and written back."""
    lib = _lib.load()
    nc = int(counts.shape[0])
    if isinstance(tab, torch.Tensor):
        _check_dev(tab, np.float64, "tab", ndim=2)
        starts = _as_dev(starts, np.int64, "starts", tab.device)
        counts = _as_dev(counts, np.int64, "counts", tab.device)
        accel_nodes = _as_dev(accel_nodes, np.float64, "accel_nodes", tab.device) if has_accel else None
        if int(tab.shape[1]) < (5 if has_yp else 4):
            raise ValueError("tab: needs columns x, vx, vy, vz[, yp]")
        ad = accel_nodes if has_accel else None
        if ad is not None and int(ad.shape[0]) < nc + 1:
            raise ValueError("accel_nodes must have len(counts)+1 entries")
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        _lib.check(lib.pb_fused_move_aos(_ptr(tab), int(tab.shape[1]), _ptr(starts), _ptr(counts), nc,
                                         _ptr(ad), float(fnstep), int(bool(has_yp)), s),
                   "fused_move_aos")
        return None
    _check_np(tab, np.float64, "tab", ndim=2)
    if tab.shape[1] < (5 if has_yp else 4):
        raise ValueError("tab: needs columns x, vx, vy, vz[, yp]")
    if has_accel:
        _check_np(accel_nodes, np.float64, "accel_nodes")
        if int(accel_nodes.shape[0]) < nc + 1:
            raise ValueError("accel_nodes must have len(counts)+1 entries")
    lo, hi, rstarts = _block_offsets(starts, counts, tab, "fused_move_aos")
    if hi == lo:
        return None
    with _Call() as c:
        td = c.put(tab, lo, hi, writeback=True)
        sd = c.put(rstarts)
        cd = c.put(counts)
        ad = c.put(accel_nodes) if has_accel else None
        _lib.check(lib.pb_fused_move_aos(_ptr(td), int(tab.shape[1]), _ptr(sd), _ptr(cd), nc, _ptr(ad),
                                         float(fnstep), int(bool(has_yp)), c.handle), "fused_move_aos")
        c.finish()
    return None


def fused_move_table(tab, aj, aj1, fnstep, has_accel, has_yp):
    """fused_move over one cell's table with node accelerations aj, aj1
    (_kernels.pyx:105-125)."""
    n = int(tab.shape[0])
    if n == 0:
        return None
    if isinstance(tab, torch.Tensor):
        dev = tab.device
        starts = torch.zeros(1, dtype=torch.int64, device=dev)
        counts = torch.full((1,), n, dtype=torch.int64, device=dev)
        accel = torch.tensor([float(aj), float(aj1)], dtype=torch.float64, device=dev)
    else:
        starts = np.zeros(1, dtype=np.int64)
        counts = np.full(1, n, dtype=np.int64)
        accel = np.array([float(aj), float(aj1)], dtype=np.float64)
    return fused_move_aos(tab, starts, counts, accel, fnstep, has_accel, has_yp)
