"""Backend selector mirroring `picmc.backends` (pkg/src/picmc/backends/__init__.py).

Only one backend exists here: "cuda".  Unlike the reference's "auto" there is
no silent fallback -- asking for anything else raises ValueError, and the
kernels themselves raise when no GPU or built library is present.
"""

from . import backend as _cuda

_CHOICES = ("cuda",)


def load_backend(name: str):
    if name == "cuda":
        return _cuda
    raise ValueError(f"unknown backend {name!r}, expected one of {_CHOICES}")


BACKEND = _cuda.BACKEND_NAME
deposit_partials = _cuda.deposit_partials
gather = _cuda.gather
fused_move = _cuda.fused_move
fused_move_table = _cuda.fused_move_table
fused_move_aos = _cuda.fused_move_aos
