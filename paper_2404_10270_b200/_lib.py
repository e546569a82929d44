"""ctypes binding of libpicmc_b200.so (the C ABI in include/picmc_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (nvcc,
sm_100a).  Loading it never needs a GPU; every compute entry point does, and
there is deliberately no CPU fallback: a missing library or device raises.
"""

import ctypes
import os
import threading

from .errors import CflViolation, ContractViolation, EngineError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PB_LIB_PATH") or os.path.join(_HERE, "libpicmc_b200.so")

PB_OK = 0
PB_ERR_INVALID = 1
PB_ERR_CUDA = 2
PB_ERR_CFL = 3
PB_ERR_CONTRACT = 4
PB_ERR_OVERFLOW = 5
PB_ERR_PEER = 6

PB_KIND_INACTIVE = 0
PB_KIND_DRIFT = 1
PB_KIND_KICK = 2
PB_KIND_BORIS = 3

PB_BC_PERIODIC = 0
PB_BC_ABSORBING = 1

PB_FIELD_PERIODIC = 0
PB_FIELD_DIRICHLET = 1

PB_MAX_SPECIES = 8
PB_CELL8_CHUNK = 2048
PB_DEPOSIT_FRAC_BITS = 48
# largest per-cell, per-species particle count the fixed-point bins represent
PB_MAX_CELL_COUNT = (1 << (64 - PB_DEPOSIT_FRAC_BITS)) - 1
ABI_VERSION = 3

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_f64 = ctypes.c_double


class PbSpecies(ctypes.Structure):
    _fields_ = [
        ("x", _p), ("vx", _p), ("vy", _p), ("vz", _p), ("yp", _p),
        ("cell", _p), ("n_dev", _p), ("n", _i64), ("holes", _p),
        ("kind", _i32), ("deposit", _i32), ("fnstep", _f64),
        ("kick_coef", _f64), ("boris_t", _f64 * 3), ("boris_s", _f64 * 3),
        ("cell8", _p), ("chunk_base", _p),
        ("b_nodes", _p), ("boris_f", _f64),
    ]


class PbStatus(ctypes.Structure):
    _fields_ = [
        ("code", _i32), ("cfl_species", _i32), ("cfl_index", ctypes.c_uint64),
        ("moved", _i64 * PB_MAX_SPECIES),
        ("absorbed", (_i64 * 2) * PB_MAX_SPECIES),
        ("n_holes", _i64 * PB_MAX_SPECIES),
        ("overflow", _i64),
        ("tile_next", ctypes.c_uint64), ("tile_done", ctypes.c_uint64),
        ("tile_next2", ctypes.c_uint64),
        ("mover_t0", ctypes.c_uint64), ("mover_ns", ctypes.c_uint64),
        ("mover_launches", ctypes.c_uint64),
    ]


class PbCollideParams(ctypes.Structure):
    _fields_ = [
        ("step_key", ctypes.c_uint64), ("global_offset", _i64), ("w_over_dx", _f64),
        ("dt", _f64), ("rate_elastic", _f64), ("rate_excitation", _f64),
        ("rate_ionization", _f64), ("threshold_j", _f64), ("mass_e", _f64),
        ("dx_over_dt", _f64),
    ]


class PbCanon(ctypes.Structure):
    _fields_ = [
        ("n_old", _i64), ("n_tail", _i64), ("offs", _p), ("counts", _p),
        ("newborn_per_cell", _p), ("newborn_k", _p),
    ]


PB_CS_MAX_FIELDS = 5
PB_MAX_RANKS = 8
PB_PEER_HANDLE_BYTES = 64


class PbPeerDensity(ctypes.Structure):
    _fields_ = [("bins", _p * PB_MAX_RANKS), ("left", _p * PB_MAX_RANKS), ("right", _p * PB_MAX_RANKS),
                ("rho", _p * PB_MAX_RANKS), ("flags", _p * PB_MAX_RANKS), ("rank", ctypes.c_int),
                ("world", ctypes.c_int), ("epoch", ctypes.c_uint64), ("epoch_dev", _p),
                ("timeout_ns", ctypes.c_uint64)]


PB_PEER_FLAG_WORDS = 2 * PB_MAX_RANKS + 1


class PbCellFields(ctypes.Structure):
    _fields_ = [("field", _p * PB_CS_MAX_FIELDS), ("nf", ctypes.c_int), ("offs", _p),
                ("counts", _p), ("nc", _i64)]


class PbMovers(ctypes.Structure):
    _fields_ = [("field", _p * PB_CS_MAX_FIELDS), ("dest", _p), ("src_cell", _p), ("src_slot", _p)]


STATUS_BYTES = ctypes.sizeof(PbStatus)

# name -> (restype, argtypes); mirrors include/picmc_b200.h one to one.
_SIGS = {
    "pb_abi_version": (ctypes.c_int, []),
    "pb_status_bytes": (ctypes.c_size_t, []),
    "pb_set_canonical_scatter_min": (ctypes.c_int, [_i64]),
    "pb_last_error": (ctypes.c_char_p, []),
    "pb_device_sm_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "pb_fused_move": (ctypes.c_int, [_p, _p, _p, _p, _p, _p, _p, _i64, _f64, _p]),
    "pb_deposit_partials": (ctypes.c_int, [_p, _p, _p, _i64, _p, _p, _p]),
    "pb_gather": (ctypes.c_int, [_p, _p, _p, _p, _i64, _p, _p]),
    "pb_fused_move_aos": (ctypes.c_int, [_p, _i64, _p, _p, _i64, _p, _f64, ctypes.c_int, _p]),
    "pb_push_deposit": (ctypes.c_int, [ctypes.POINTER(PbSpecies), ctypes.c_int, _p,
                                       _i64, ctypes.c_int, _p, _p, _p]),
    "pb_cell8_build": (ctypes.c_int, [ctypes.POINTER(PbSpecies), _p]),
    "pb_last_mover_kernel": (ctypes.c_char_p, []),
    "pb_deposit_only": (ctypes.c_int, [ctypes.POINTER(PbSpecies), ctypes.c_int,
                                       _i64, _p, _p, _p]),
    "pb_rho_epilogue": (ctypes.c_int, [_p, ctypes.POINTER(_f64), ctypes.c_int, _i64,
                                       ctypes.c_int, _p, _p, _p, _p, _p]),
    "pb_density_step": (ctypes.c_int, [_p, _p, _p, ctypes.POINTER(_f64), ctypes.c_int, _i64,
                                       ctypes.c_int, _p, _p, _p, _p]),
    "pb_compact_scratch_bytes": (ctypes.c_size_t, [_i64]),
    "pb_compact": (ctypes.c_int, [ctypes.POINTER(PbSpecies), ctypes.c_int, _p, _p,
                                  ctypes.c_size_t, _p]),
    "pb_sort_scratch_bytes": (ctypes.c_size_t, [_i64, _i64]),
    "pb_sort_by_cell": (ctypes.c_int, [ctypes.POINTER(PbSpecies),
                                       ctypes.POINTER(PbSpecies), _i64, _p,
                                       ctypes.c_size_t, _p]),
    "pb_field_scratch_bytes": (ctypes.c_size_t, [_i64]),
    "pb_smooth_density": (ctypes.c_int, [_p, _p, _i64, ctypes.c_int, _p, _p]),
    "pb_solve_poisson": (ctypes.c_int, [_p, _p, _i64, _f64, _f64, ctypes.c_int,
                                        _f64, _f64, _p, _p]),
    "pb_solve_poisson_scan": (ctypes.c_int, [_p, _p, _i64, _f64, _f64, ctypes.c_int,
                                             _f64, _f64, _p, _p]),
    "pb_compute_efield": (ctypes.c_int, [_p, _p, _i64, _f64, ctypes.c_int, _p]),
    "pb_compute_efield_clear": (ctypes.c_int, [_p, _p, _i64, _f64, ctypes.c_int, _p, _p, _i64, _p]),
    "pb_field_cycle": (ctypes.c_int, [_p, _p, ctypes.c_int, _i64, ctypes.c_int, ctypes.c_int, _f64, _f64, _f64,
                                      _f64, _p, _p, _p, _p, _p, _p, _p, _p, _i64, _p, _p,
                                      ctypes.POINTER(PbSpecies), ctypes.c_int, _p, ctypes.c_size_t, _p]),
    "pb_stream_sol": (ctypes.c_int, [ctypes.POINTER(PbSpecies), ctypes.c_int, _p]),
    "pb_init_species": (ctypes.c_int, [ctypes.POINTER(PbSpecies), ctypes.c_uint64,
                                       _i64, _i64, _i64, _f64, _p]),
    "pb_layout_scratch_bytes": (ctypes.c_size_t, [_i64]),
    "pb_cell_layout": (ctypes.c_int, [_p, _i64, _i64, _p, _p, _p, ctypes.c_size_t, _p]),
    "pb_collide": (ctypes.c_int, [ctypes.POINTER(PbSpecies), ctypes.POINTER(PbSpecies),
                                  ctypes.POINTER(PbSpecies), _p, _p, _p, _p, _i64,
                                  ctypes.POINTER(PbCollideParams), _p, _p, _i64, _p, _p]),
    "pb_canonical_scratch_bytes": (ctypes.c_size_t, [_i64, _i64]),
    "pb_canonical_resort": (ctypes.c_int, [ctypes.POINTER(PbSpecies), ctypes.POINTER(PbSpecies),
                                           ctypes.POINTER(PbCanon), _p, _i64, ctypes.c_int,
                                           ctypes.c_int, _p, _p, ctypes.c_size_t, _p]),
    "pb_canonical_keys": (ctypes.c_int, [ctypes.POINTER(PbSpecies), ctypes.POINTER(PbCanon), _p, _i64,
                                         ctypes.c_int, ctypes.c_int, _p, _i64, ctypes.c_int, _p, _p,
                                         ctypes.c_size_t, _p]),
    "pb_canonical_step": (ctypes.c_int, [ctypes.POINTER(PbSpecies), ctypes.POINTER(PbSpecies),
                                         ctypes.POINTER(PbCanon), ctypes.c_int, _p, _i64, ctypes.c_int,
                                         _p, _p, ctypes.c_size_t, ctypes.POINTER(_i64), _p]),
    "pb_rho_from_partials": (ctypes.c_int, [_p, ctypes.POINTER(_f64), ctypes.c_int, _i64,
                                            ctypes.c_int, _p, _p, _p, _p]),
    "pb_stitch_rho": (ctypes.c_int, [_p, _p, _i64, ctypes.c_int, _p, _p]),
    "pb_cs_scratch_bytes": (ctypes.c_size_t, [_i64]),
    "pb_peer_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(_p), _p]),
    "pb_peer_open": (ctypes.c_int, [_p, ctypes.POINTER(_p)]),
    "pb_peer_close": (ctypes.c_int, [_p, ctypes.c_int]),
    "pb_peer_density_step": (ctypes.c_int, [ctypes.POINTER(PbPeerDensity), _p, ctypes.POINTER(_f64),
                                            ctypes.c_int, _i64, ctypes.c_int, _p, _p]),
    "pb_push_velocity": (ctypes.c_int, [_p, _f64, _p, _p, _p, _i64, _p, ctypes.c_size_t, _p]),
    "pb_resort_count": (ctypes.c_int, [_p, _p, _p, _i64, _i64, _p, _p, _p, _p, ctypes.c_size_t, _p]),
    "pb_resort_collect": (ctypes.c_int, [ctypes.POINTER(PbCellFields), ctypes.POINTER(PbMovers),
                                         _i64, _i64, _p, _p]),
    "pb_commit_place": (ctypes.c_int, [ctypes.POINTER(PbCellFields), ctypes.POINTER(PbMovers),
                                       _p, _p, _i64, _i64, _p]),
    "pb_repack": (ctypes.c_int, [_p, _p, _p, _p, _p, _i64, _p]),
}

_lock = threading.Lock()
_lib = None


def load():
    """Load and type the library; raises ImportError if it is not built."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing; run __graft_entry__.build() "
                    "(nvcc sm_100a) first -- there is no CPU fallback"
                )
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.pb_abi_version() != ABI_VERSION:
                raise ImportError("libpicmc_b200 ABI version mismatch")
            _lib = lib
    return _lib


def exported_names():
    return tuple(_SIGS)


def check(rc: int, what: str = ""):
    """Map a status code onto the reference exception hierarchy."""
    if rc == PB_OK:
        return
    msg = load().pb_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == PB_ERR_INVALID:
        raise ValueError(msg)
    if rc == PB_ERR_CFL:
        raise CflViolation(msg)
    if rc == PB_ERR_CONTRACT:
        raise ContractViolation(msg)
    if rc in (PB_ERR_OVERFLOW, PB_ERR_PEER):
        raise EngineError(msg)
    raise RuntimeError(msg)



# mangled names of the mover kernels whose DRAM traffic profiles/ records
MOVER_SYMBOLS = {
    "k_push_split<0>": "_ZN2pb12k_push_splitILi0EEEvNS_10LaunchArgsE",
    "k_push_split<1>": "_ZN2pb12k_push_splitILi1EEEvNS_10LaunchArgsE",
    "k_push_ring<0>": "_ZN2pb11k_push_ringILi0EEEvNS_10LaunchArgsE",
    "k_push_ring<1>": "_ZN2pb11k_push_ringILi1EEEvNS_10LaunchArgsE",
}


def kernel_digest(symbol: str, path: str = None):
    """sha256 of one kernel's sm_100a machine code in the library (its SASS
    instruction lines from cuobjdump), or None when cuobjdump is missing or
    the kernel is not found.  Unlike a digest of the whole file -- which
    changes with the source mtimes that -lineinfo records -- it identifies the
    code that ran, so an ncu capture stays attached to rebuilds of the same
    sources and detaches when the kernel changes."""
    import hashlib
    import re
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        return None
    try:
        out = subprocess.run([tool, "-sass", "-fun", symbol, path or LIB_PATH], capture_output=True,
                             text=True, timeout=120).stdout
    except (OSError, subprocess.SubprocessError):
        return None
    lines = [ln.strip() for ln in out.splitlines() if re.match(r"^\s+/\*[0-9a-f]{4,}\*/", ln)]
    return hashlib.sha256("\n".join(lines).encode()).hexdigest() if lines else None
