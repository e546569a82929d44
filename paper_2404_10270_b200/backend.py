"""The `cuda` kernel backend with the reference's operator signatures.

Drop-in for `picmc.backends.{deposit_partials, gather, fused_move}`
(pkg/src/picmc/backends/__init__.py:45-50, compiled twin
pkg/src/picmc/backends/_kernels.pyx:14-102): the same arguments (C-contiguous
float64 / int64 NumPy arrays, packed cell-sorted layout), the same in-place
mutation and return conventions, bitwise-identical results.  Arrays may also
be CUDA torch tensors, in which case nothing crosses PCIe.

Every call runs on the GPU through libpicmc_b200.so; there is no CPU path.
"""

import ctypes

import numpy as np
import torch

from . import _lib

BACKEND_NAME = "cuda"


def _dev():
    if not torch.cuda.is_available():
        raise RuntimeError("backend 'cuda' needs a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def _check_np(a, dtype, name):
    # The Cython buffer checks raise ValueError on dtype/contiguity mismatch.
    if not isinstance(a, np.ndarray):
        raise TypeError(f"{name}: expected a numpy array or CUDA tensor")
    if a.dtype != dtype:
        raise ValueError(f"Buffer dtype mismatch for {name}: expected {np.dtype(dtype)}, got {a.dtype}")
    if a.ndim != 1 or not a.flags.c_contiguous:
        raise ValueError(f"{name}: ndarray is not C-contiguous 1-D")


class _Stage:
    """Host<->device staging for one call; writes back mutated arrays."""

    def __init__(self):
        self.dev = _dev()
        self.back = []

    def put(self, a, dtype, name, writeback=False):
        if a is None:
            return None
        if isinstance(a, torch.Tensor):
            want = torch.float64 if dtype == np.float64 else torch.int64
            if not a.is_cuda or a.dtype != want or not a.is_contiguous():
                raise ValueError(f"{name}: expected a contiguous CUDA {want} tensor")
            return a
        _check_np(a, dtype, name)
        t = torch.from_numpy(a).to(self.dev, non_blocking=False)
        if writeback:
            self.back.append((a, t))
        return t

    def finish(self):
        torch.cuda.current_stream(self.dev).synchronize()
        for host, t in self.back:
            host[...] = t.cpu().numpy()


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def deposit_partials(x, offs, counts):
    """Per-cell raw CIC sums L[j] = sum(1-x), R[j] = sum(x), in slot order."""
    lib = _lib.load()
    st = _Stage()
    xd = st.put(x, np.float64, "x")
    od = st.put(offs, np.int64, "offs")
    cd = st.put(counts, np.int64, "counts")
    nc = int(cd.shape[0])
    left = torch.zeros(nc, dtype=torch.float64, device=st.dev)
    right = torch.zeros(nc, dtype=torch.float64, device=st.dev)
    _lib.check(lib.pb_deposit_partials(_ptr(xd), _ptr(od), _ptr(cd), nc, _ptr(left),
                                       _ptr(right), _stream()), "deposit_partials")
    if isinstance(x, torch.Tensor):
        return left, right
    st.finish()
    return left.cpu().numpy(), right.cpu().numpy()


def gather(nodes, x, offs, counts):
    """Per-particle a[j] + x*(a[j+1]-a[j]) in live (cell-major) order."""
    lib = _lib.load()
    st = _Stage()
    nd = st.put(nodes, np.float64, "nodes")
    xd = st.put(x, np.float64, "x")
    od = st.put(offs, np.int64, "offs")
    cd = st.put(counts, np.int64, "counts")
    nc = int(cd.shape[0])
    total = int(cd.sum().item()) if nc else 0
    out = torch.empty(total, dtype=torch.float64, device=st.dev)
    if total:
        _lib.check(lib.pb_gather(_ptr(nd), _ptr(xd), _ptr(od), _ptr(cd), nc, _ptr(out),
                                 _stream()), "gather")
    if isinstance(x, torch.Tensor):
        return out
    st.finish()
    return out.cpu().numpy()


def fused_move(accel_nodes, x, vx, vy, yp, offs, counts, fnstep):
    """One fused gather+push step over live particles, in place.

    accel_nodes None skips the kick entirely (no `+= 0.0`, which would turn
    -0.0 velocities into +0.0; pkg/src/picmc/mover.py:214-216).
    """
    lib = _lib.load()
    st = _Stage()
    ad = st.put(accel_nodes, np.float64, "accel_nodes")
    xd = st.put(x, np.float64, "x", writeback=True)
    vxd = st.put(vx, np.float64, "vx", writeback=accel_nodes is not None)
    vyd = st.put(vy, np.float64, "vy") if yp is not None else None
    ypd = st.put(yp, np.float64, "yp", writeback=True)
    od = st.put(offs, np.int64, "offs")
    cd = st.put(counts, np.int64, "counts")
    nc = int(cd.shape[0])
    if ad is not None and int(ad.shape[0]) < nc + 1:
        raise ValueError("accel_nodes must have len(counts)+1 entries")
    _lib.check(lib.pb_fused_move(_ptr(ad), _ptr(xd), _ptr(vxd), _ptr(vyd), _ptr(ypd), _ptr(od),
                                 _ptr(cd), nc, float(fnstep), _stream()), "fused_move")
    st.finish()
    return None


def _table(tab, has_yp):
    """Stage a (n, ncols) float64 C-contiguous table (numpy or CUDA tensor)."""
    if isinstance(tab, torch.Tensor):
        if not tab.is_cuda or tab.dtype != torch.float64 or not tab.is_contiguous() or tab.dim() != 2:
            raise ValueError("tab: expected a contiguous 2-D CUDA float64 tensor")
        return tab, None
    if not isinstance(tab, np.ndarray):
        raise TypeError("tab: expected a numpy array or CUDA tensor")
    if tab.dtype != np.float64:
        raise ValueError(f"Buffer dtype mismatch for tab: expected float64, got {tab.dtype}")
    if tab.ndim != 2 or not tab.flags.c_contiguous:
        raise ValueError("tab: ndarray is not C-contiguous 2-D")
    if tab.shape[1] < (5 if has_yp else 4):
        raise ValueError("tab: needs columns x, vx, vy, vz[, yp]")
    return torch.from_numpy(tab).to(_dev()), tab


def fused_move_aos(tab, starts, counts, accel_nodes, fnstep, has_accel, has_yp):
    """fused_move over a cell-major array-of-structs table (columns x, vx,
    vy, vz[, yp]) in place (_kernels.pyx:128-152)."""
    lib = _lib.load()
    t, host = _table(tab, has_yp)
    st = _Stage()
    sd = st.put(starts, np.int64, "starts")
    cd = st.put(counts, np.int64, "counts")
    ad = st.put(accel_nodes, np.float64, "accel_nodes") if has_accel else None
    nc = int(cd.shape[0])
    if ad is not None and int(ad.shape[0]) < nc + 1:
        raise ValueError("accel_nodes must have len(counts)+1 entries")
    _lib.check(lib.pb_fused_move_aos(_ptr(t), int(t.shape[1]), _ptr(sd), _ptr(cd), nc, _ptr(ad),
                                     float(fnstep), int(bool(has_yp)), _stream()), "fused_move_aos")
    st.finish()
    if host is not None:
        host[...] = t.cpu().numpy()
    return None


def fused_move_table(tab, aj, aj1, fnstep, has_accel, has_yp):
    """fused_move over one cell's table with node accelerations aj, aj1
    (_kernels.pyx:105-125)."""
    n = int(tab.shape[0])
    if n == 0:
        return None
    dev = _dev()
    starts = torch.zeros(1, dtype=torch.int64, device=dev)
    counts = torch.full((1,), n, dtype=torch.int64, device=dev)
    accel = torch.tensor([float(aj), float(aj1)], dtype=torch.float64, device=dev)
    return fused_move_aos(tab, starts, counts, accel, fnstep, has_accel, has_yp)
