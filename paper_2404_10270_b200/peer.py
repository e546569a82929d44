"""Peer-memory buffers for the fused multi-GPU density exchange.

Every rank allocates its density-exchange buffers with `pb_peer_alloc`
(cudaMalloc + CUDA IPC handle), the handles are exchanged once through the
process group, and every rank maps the others' buffers (`pb_peer_open`,
NVLink peer access).  `pb_peer_density_step` (csrc/peer.cu) then reads all
ranks' deposit bins and writes every rank's rho directly -- the allreduce and
the density epilogue in one kernel, no NCCL call on the step path.

If any rank cannot map a peer (no P2P path between the GPUs), every rank
falls back together to the NCCL allreduce + epilogue (`available` False).
"""

import ctypes

import torch

from . import _lib


class _CudaArray:
    """__cuda_array_interface__ view of a raw device buffer (torch.as_tensor
    wraps it without a copy; the buffer stays owned by PeerBuffers)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class PeerBuffers:
    """Named IPC-shared buffers of this rank plus the mapped buffers of every
    peer: ptrs[name][rank] is rank's buffer `name` as seen from this GPU."""

    def __init__(self, sizes: dict, rank: int, world: int, group=None, device=None):
        import torch.distributed as dist

        self.lib = _lib.load()
        self.rank, self.world = rank, world
        self.device = device
        self.own, self.ptrs, self._opened = {}, {}, []
        handles = {}
        ok = 1
        for name, nbytes in sizes.items():
            p = ctypes.c_void_p()
            h = (ctypes.c_char * _lib.PB_PEER_HANDLE_BYTES)()
            if self.lib.pb_peer_alloc(int(nbytes), ctypes.byref(p), h) != _lib.PB_OK:
                ok = 0  # still join the exchange below, so no rank waits forever
                break
            self.own[name] = p.value
            handles[name] = bytes(h)
        gathered = [None] * world
        dist.all_gather_object(gathered, handles if ok else None, group=group)
        if any(g is None for g in gathered):
            ok = 0
        for name in (sizes if ok else ()):
            self.ptrs[name] = [0] * world
            for r in range(world):
                if r == rank:
                    self.ptrs[name][r] = self.own[name]
                    continue
                p = ctypes.c_void_p()
                h = (ctypes.c_char * _lib.PB_PEER_HANDLE_BYTES).from_buffer_copy(gathered[r][name])
                if self.lib.pb_peer_open(h, ctypes.byref(p)) != _lib.PB_OK:
                    ok = 0
                    continue
                self.ptrs[name][r] = p.value
                self._opened.append(p.value)
        flag = torch.tensor([ok], dtype=torch.int64,
                            device=device if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        self.available = bool(flag.item())

    def tensor(self, name: str, n: int, dtype) -> torch.Tensor:
        """This rank's buffer `name` as an n-element CUDA tensor (no copy)."""
        typestr = {torch.float64: "<f8", torch.int64: "<i8"}[dtype]
        return torch.as_tensor(_CudaArray(self.own[name], n, typestr), device=self.device)

    def close(self):
        torch.cuda.synchronize(self.device)
        for p in self._opened:
            self.lib.pb_peer_close(ctypes.c_void_p(p), 0)
        for p in self.own.values():
            self.lib.pb_peer_close(ctypes.c_void_p(p), 1)
        self._opened, self.own = [], {}
