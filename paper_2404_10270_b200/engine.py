"""Device-resident step engine: the B200 replacement for the reference's
deposit -> [smooth -> solve -> E] -> gather -> move -> resort -> migrate cycle
(pkg/src/picmc/harness.py:144-242).

Per step, on one CUDA stream:
  deposit  fixed-point bins from the previous push -> (NCCL allreduce across
           GPUs) -> weighted partials + stitch            pb_rho_epilogue
  smooth/solve/E (field_solve only), replicated on every GPU
  mover    fused gather + kick/Boris + drift + cell transfer + absorbing
           removal + next-step deposit                    pb_push_deposit
  resort   absorbing-wall hole compaction                 pb_compact
           periodic cell sort every `sort_every` steps    pb_sort_by_cell

The reference's separate gather phase computes E_p and discards it
(harness.py:180-185); here the gather lives inside the mover.  Its resort and
migrate phases (mover.py:113-195, decomposition.py:177-229) collapse into the
mover's register-level cell update: particles are sharded by index over a
replicated grid, so nothing migrates between GPUs.
"""

import ctypes
import math
import os
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .core import check_store_budget, init_species_host, macro_weight, thermal_std, velocity_kick_coef
from .errors import CflViolation, ConfigError, EngineError
from .rng import STREAM_INIT, stream
from .store import DeviceSpecies, decode_status, species_array, status_template

PHASE_KEYS = ("deposit", "smooth", "solve", "gather", "collide", "mover", "resort", "migrate")


def partition_cells(nc: int, workers: int) -> tuple:
    """Contiguous balanced ranges, sizes differing <= 1 (decomposition.py:66-79)."""
    if workers < 1 or workers > nc:
        raise ConfigError(f"workers ({workers}) must be in [1, nc={nc}]")
    base, rem = divmod(nc, workers)
    out, lo = [], 0
    for w in range(workers):
        hi = lo + base + (1 if w < rem else 0)
        out.append((lo, hi))
        lo = hi
    return tuple(out)


@dataclass(frozen=True)
class Partition:
    """GPU shard map: rank r loaded the particles of cells ranges[r]."""

    worker_count: int
    nc: int
    ranges: tuple


def reduce_bins(bins: torch.Tensor, group=None):
    """Sum the per-rank fixed-point deposit bins (exact int64 allreduce).

    Works for CUDA tensors under NCCL and CPU tensors under gloo; the sum of
    integers is associative, so the reduced density is bitwise independent of
    the GPU count and of NCCL's algorithm choice (ring / tree / NVLS).
    """
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(bins, op=dist.ReduceOp.SUM, group=group)
    return bins


def boris_coefficients(sp, consts, b_field) -> tuple:
    """t = q B dt / (2 m), s = t * (2 / (1 + |t|^2)) (standard Boris rotation;
    one division, the form the gathered-B kernel evaluates per particle)."""
    f = sp.charge_c * consts.dt_s / (2.0 * sp.mass_kg)
    t = [f * float(b) for b in b_field]
    t2 = t[0] * t[0] + t[1] * t[1] + t[2] * t[2]
    g = 2.0 / (1.0 + t2)
    s = [c * g for c in t]
    return t, s


def b_field_nodes(config):
    """Node B profile of a config with `b_grad_t_per_m`, as the (nc+1, 4)
    f64 array pb_species.b_nodes reads (x, y, z, 0 per node, tesla):
    B(X_j) = b_field_t + g * (X_j - L/2), X_j = j * dx.  None for a uniform
    (or absent) field, which keeps the constant boris_t / boris_s."""
    g = getattr(config, "b_grad_t_per_m", None)
    if g is None or config.b_field_t is None:
        return None
    nc, dx = int(config.grid.nc), float(config.grid.dx_m)
    xj = np.arange(nc + 1, dtype=np.float64) * dx - 0.5 * float(config.grid.length_m)
    nodes = np.zeros((nc + 1, 4), dtype=np.float64)
    for k in range(3):
        nodes[:, k] = float(config.b_field_t[k]) + float(g[k]) * xj
    return nodes


def species_kind(sp, b_field) -> int:
    if not sp.active_mover:
        return _lib.PB_KIND_INACTIVE
    if sp.charged:
        return _lib.PB_KIND_BORIS if b_field is not None else _lib.PB_KIND_KICK
    return _lib.PB_KIND_DRIFT


def sort_periods_for(config, sort_every: int, ratio_cap: int = 16) -> list:
    """Per-species cell-sort period.  `sort_every` applies to the fastest
    species (largest thermal drift per step, nstep included); slower ones
    lose cell order proportionally more slowly and are sorted proportionally
    less often (x ratio_cap at most: measured +0.4% over x64, the slow
    species otherwise lose order over a few thousand steps).  0 = never."""
    if not sort_every:
        return [0] * len(config.species)
    b_field = getattr(config, "b_field_t", None)
    drift = []
    for isp, spd in enumerate(config.species):
        v = thermal_std(config.temperatures_ev[isp], spd.mass_kg, config.consts.dt_s,
                        config.grid.dx_m) * float(spd.nstep)
        drift.append(v if species_kind(spd, b_field) != _lib.PB_KIND_INACTIVE else 0.0)
    vmax = max(drift) or 1.0
    return [0 if v <= 0.0 else sort_every * int(min(ratio_cap, max(1, round(vmax / v)))) for v in drift]


class Engine:
    """One GPU's share of a run: its particle shard plus a grid replica."""

    # Tuning attributes (class-level defaults = the measured-best settings;
    # tests and A/B scripts override them on an instance or subclass).
    supports_collisions = False  # CanonicalEngine (canonical.py) runs them
    use_cell8 = True     # 1-byte cell index for dense charged species
    force_cell8 = False  # ... also in charged-only runs (measured slower there)
    sort_ratio_cap = 16  # slow species are sorted at most 16x less often
    # Field-solve steps: push neutral movers while the field pipeline runs.
    # Measured 2.4% slower on one GPU (a second launch's ramp/tail costs more
    # than the ~30 us field pipeline it hides); with N > 1 it also hides the
    # density allreduce.  None = on iff N > 1; True/False force it.
    field_split = None
    supports_peer = True  # the fused peer-memory density exchange (N > 1)
    # serial field-solve cycle: density in one pb_rho_epilogue launch, bins
    # cleared by the E kernel (False: pb_density_step's two launches)
    density_one = True
    # field-solve steps with the scan Poisson: the whole field step in one
    # launch with grid barriers (pb_field_cycle) instead of 6-10 kernels
    fused_field = True
    # absorbing walls on the single-launch field path: a step's holes are
    # filled by compaction blocks of the NEXT step's field launch (no separate
    # launch); anything that looks at the stores first compacts eagerly
    # (_flush_holes), and a due sort compacts before it sorts
    fold_compaction = True

    def __init__(self, config, device=None, *, rank: int = 0, world: int = 1,
                 group=None, init: str = "host", check_every: int = 1, peer: bool = None):
        config.validate()
        if config.collisions is not None and config.collisions.enabled and not self.supports_collisions:
            raise ConfigError(
                "collisions need the canonical slot order: run them through "
                "CanonicalEngine / run_simulation (SURVEY.md 8f)"
            )
        if not torch.cuda.is_available():
            raise RuntimeError("the B200 engine needs a CUDA device; there is no CPU fallback")
        self.lib = _lib.load()
        self.cfg = config
        self.device = torch.device(device if device is not None else f"cuda:{torch.cuda.current_device()}")
        self.rank, self.world, self.group = rank, world, group
        self.grid = config.grid
        self.nc = int(config.grid.nc)
        self.periodic = config.boundary == "periodic"
        self.field_bc = _lib.PB_FIELD_PERIODIC if self.periodic else _lib.PB_FIELD_DIRICHLET
        self.absorbing = getattr(config, "particle_boundary", "periodic") == "absorbing"
        self.bc = _lib.PB_BC_ABSORBING if self.absorbing else _lib.PB_BC_PERIODIC
        self.b_field = getattr(config, "b_field_t", None)
        self.sort_every = int(getattr(config, "sort_every", 0) or 0)
        method = getattr(config, "poisson", "auto")
        # exact: the reference's serial elimination, bitwise; scan: parallel.
        self.poisson = method if method != "auto" else ("exact" if self.nc <= 8192 else "scan")
        self.check_every = int(check_every)
        self.partition = Partition(world, self.nc, partition_cells(self.nc, world))
        self.cell_lo, self.cell_hi = self.partition.ranges[rank]
        check_store_budget(config)
        if 2 * int(config.ppc0) > _lib.PB_MAX_CELL_COUNT:
            # the fixed-point bins hold < 2^16 particles per cell and species
            # (csrc/common.cuh kMaxCellCount); leave room for fluctuations.
            # Denser cells that still occur raise EngineError at the next sync.
            raise ConfigError(f"ppc0={config.ppc0}: the fixed-point deposit represents at most "
                              f"{_lib.PB_MAX_CELL_COUNT} particles of one species per cell; "
                              f"ppc0 must be <= {_lib.PB_MAX_CELL_COUNT // 2}")

        self.stream = torch.cuda.Stream(self.device)
        self._side = torch.cuda.Stream(self.device)  # overlapped density epilogue
        self._epi_prev = None  # event: last side-stream epilogue (eager overlap)
        nodes = b_field_nodes(config)
        self.b_nodes = None  # (nc+1, 4) device B profile, or None (uniform B)
        if nodes is not None:
            with torch.cuda.stream(self.stream):
                self.b_nodes = torch.from_numpy(nodes).to(self.device)
        self.sp = []
        self.coef_dep = []
        ndep = 0
        nloc = (self.cell_hi - self.cell_lo) * int(config.ppc0)
        for isp, spd in enumerate(config.species):
            kind = species_kind(spd, self.b_field)
            dep = -1
            if spd.charged:
                dep = ndep
                ndep += 1
                self.coef_dep.append(spd.charge_c * macro_weight(config, isp) / self.grid.dx_m)
            kick = velocity_kick_coef(spd, config.consts, self.grid.dx_m) if spd.charged else 0.0
            boris = boris_coefficients(spd, config.consts, self.b_field) if kind == _lib.PB_KIND_BORIS else None
            boris_f = spd.charge_c * config.consts.dt_s / (2.0 * spd.mass_kg)
            # The mover reads a 1-byte cell offset instead of the 4-byte index
            # for charged species dense enough that a 2048-particle chunk spans
            # well under 127 cells (pb_species.cell8).
            # Measured: a win (-1.7% step) when neutral slices share the launch,
            # a loss (+2-5%) in charged-only runs, whose latency-bound slices
            # pay for the extra dependent base load + decode.
            has_neutral = any(species_kind(x, self.b_field) == _lib.PB_KIND_DRIFT for x in config.species)
            cell8 = (self.use_cell8 and (has_neutral or self.force_cell8) and kind in (_lib.PB_KIND_KICK, _lib.PB_KIND_BORIS)
                     and int(config.ppc0) >= 32)
            with torch.cuda.stream(self.stream):
                self.sp.append(DeviceSpecies(spd, nloc, self.device, kind=kind, deposit=dep,
                                             kick_coef=kick, boris=boris, absorbing=self.absorbing,
                                             b_nodes=self.b_nodes, boris_f=boris_f,
                                             cap=self._species_cap(isp, nloc), cell8=cell8))
        self.ndep = ndep
        self._coef_c = (ctypes.c_double * max(ndep, 1))(*self.coef_dep)
        self.sort_periods = self._sort_periods(config)
        nc = self.nc
        with torch.cuda.stream(self.stream):
            # Ping-pong fixed-point bins: the mover deposits into one set while
            # the other holds the density being reduced / stitched.
            self.bins_pp = [torch.zeros(max(ndep, 1) * 2 * nc, dtype=torch.int64, device=self.device)
                            for _ in range(2)]
            self.cur = 0
            self.rho = torch.zeros(nc + 1, dtype=torch.float64, device=self.device)
            self.left = torch.zeros(nc, dtype=torch.float64, device=self.device)
            self.right = torch.zeros(nc, dtype=torch.float64, device=self.device)
        # N > 1: the density exchange through peer memory (pb_peer_density_step:
        # the allreduce fused with the epilogue over NVLink) unless PB_PEER=0;
        # the bins and the outputs then live in IPC-shared buffers
        self.peer = None
        if peer is None:
            peer = os.environ.get("PB_PEER", "1") != "0"
        if world > 1 and peer and self.supports_peer:
            self._setup_peer(max(ndep, 1) * 2 * nc, nc)
        with torch.cuda.stream(self.stream):
            self.rho_s = torch.zeros(nc + 1, dtype=torch.float64, device=self.device)
            self.phi = torch.zeros(nc + 1, dtype=torch.float64, device=self.device)
            self.e = torch.zeros(nc + 1, dtype=torch.float64, device=self.device)
            self.field_scratch = torch.zeros(  # zeroed: pb_field_cycle's barrier words
                max(1, self.lib.pb_field_scratch_bytes(nc) // 8), dtype=torch.float64, device=self.device)
            self.status_tpl = status_template(self.device)
            self.status = self.status_tpl.clone()
            self.compact_scratch = None
            if self.absorbing:
                nb = self.lib.pb_compact_scratch_bytes(max(nloc, 1))
                self.compact_scratch = torch.empty(nb, dtype=torch.uint8, device=self.device)
        self.sort_scratch = None
        self.step_index = 0
        self.phase_events = []
        self._timing = None
        self._arr = None
        self._sub_cache = {}
        self.graphs = {}
        self._next_clear = False
        self._holes_pending = False  # absorbing walls: the last push's holes are not filled yet
        # Mover work counter (pb_status.tile_next; self-resetting in the kernel).
        off = _lib.PbStatus.tile_next.offset
        self._tile_counter = self.status[off:off + 8]
        self.absorbed = np.zeros((len(self.sp), 2), dtype=np.int64)
        self.moved = np.zeros(len(self.sp), dtype=np.int64)
        # in-kernel mover clock (pb_status.mover_ns / mover_launches), summed
        # over syncs: the persistent movers' own duration, graph replays included
        self.mover_ns = 0
        self.mover_launches = 0
        self._load(init)

    # -- setup ------------------------------------------------------------------
    def _sort_periods(self, config) -> list:
        return sort_periods_for(config, self.sort_every, self.sort_ratio_cap)

    def _species_cap(self, isp: int, nloc: int) -> int:
        return nloc

    def _load(self, init: str):
        cfg = self.cfg
        # the stores were allocated (and n_dev filled) on the caller's stream;
        # the engine stream is a non-blocking stream, so order it explicitly
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(self.stream):
            for isp, s in enumerate(self.sp):
                if init == "host":
                    s.upload(init_species_host(cfg, isp, self.cell_lo, self.cell_hi))
                elif init == "device":
                    std = thermal_std(cfg.temperatures_ev[isp], s.sp.mass_kg, cfg.consts.dt_s, self.grid.dx_m)
                    key = stream(cfg.seed, STREAM_INIT, isp)
                    pbs = s.pb()
                    _lib.check(self.lib.pb_init_species(ctypes.byref(pbs), key, self.cell_lo, self.cell_hi,
                                                        int(cfg.ppc0), std, self._sh()), "pb_init_species")
                elif init == "none":
                    pass
                else:
                    raise ValueError(f"unknown init mode {init!r}")
        self.deposit_current()
        self._publish()

    def _publish(self):
        """Order the caller's current stream after the engine stream, so
        state written by the engine (init, upload, sort) is what the caller
        reads next."""
        torch.cuda.current_stream(self.device).wait_stream(self.stream)

    def _sh(self):
        return ctypes.c_void_p(self.stream.cuda_stream)

    def _species(self):
        """Cached C-ABI species array (rebuilt when buffers are swapped)."""
        if self._arr is None:
            self._arr = species_array(self.sp)
            self._sub_cache = {}
        return self._arr

    @property
    def bins(self) -> torch.Tensor:
        """The bin set holding the latest deposit (read by the next density())."""
        return self.bins_pp[self.cur]

    def rebuild_cell8(self, which=None):
        """Recompute the compressed cell index after a reorder or upload."""
        with torch.cuda.stream(self.stream):
            for k, s in enumerate(self.sp):
                if s.cell8 is None or (which is not None and k not in which):
                    continue
                pbs = s.pb(s.live_count() if s.absorbing else None)
                _lib.check(self.lib.pb_cell8_build(ctypes.byref(pbs), self._sh()), "pb_cell8_build")

    def deposit_current(self):
        """Fixed-point deposit of the current positions into the bins
        (the reference's step-start deposit, harness.py:148-160)."""
        self.rebuild_cell8()
        arr, n = self._species()
        with torch.cuda.stream(self.stream):
            self.bins.zero_()
            _lib.check(self.lib.pb_deposit_only(arr, n, self.nc, self.bins.data_ptr(),
                                                self.status.data_ptr(), self._sh()), "pb_deposit_only")

    def set_b_field(self, nodes):
        """Replace the magnetic field by an arbitrary node profile: `nodes`
        is (nc+1, 3) tesla (host array or tensor), gathered per Boris
        particle with the one-sided linear form (pb_species.b_nodes).  The
        run must have been configured with a B field (b_field_t), which is
        what makes the charged species Boris species."""
        if self.b_field is None:
            raise ConfigError("set_b_field needs a config with b_field_t (Boris species)")
        b = torch.as_tensor(nodes, dtype=torch.float64)
        if tuple(b.shape) != (self.nc + 1, 3):
            raise ValueError(f"B nodes must have shape ({self.nc + 1}, 3), got {tuple(b.shape)}")
        with torch.cuda.stream(self.stream):
            dev = torch.zeros((self.nc + 1, 4), dtype=torch.float64, device=self.device)
            dev[:, :3].copy_(b.to(self.device, non_blocking=False))
        self.b_nodes = dev
        for s in self.sp:
            s.b_nodes = dev
        self._arr = None  # species structs carry the pointer: rebuild them
        self.graphs = {}
        self._publish()

    def upload(self, flats: list):
        """Replace the particle state with host arrays (engine flat layout)."""
        self._flush_holes()  # no pending holes may reach the new state
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(self.stream):
            for s, f in zip(self.sp, flats):
                if f.n != s.n:
                    raise ValueError("particle count mismatch")
                s.upload(f)
        self.deposit_current()
        self._publish()

    # -- step phases ------------------------------------------------------------
    def density(self, stream=None, clear_next: bool = True) -> torch.Tensor:
        """Reduce the bins across GPUs and produce left/right/rho; the bin set
        read is zeroed afterwards and, with clear_next, so is the other set
        (the graph replay runs this concurrently with the next push and then
        must not touch the set that push deposits into)."""
        st = stream if stream is not None else self.stream
        with torch.cuda.stream(st):
            if self.peer is not None:
                self._peer_density(st, clear_next)
                self._next_clear = True
                self._order_caller(stream)
                return self.rho
            if self.world > 1:
                reduce_bins(self.bins, self.group)
            nxt = self.bins_pp[1 - self.cur].data_ptr() if clear_next else None
            _lib.check(self.lib.pb_density_step(
                self.bins.data_ptr(), nxt, self.status.data_ptr(), self._coef_c, self.ndep, self.nc, self.field_bc,
                self.left.data_ptr(), self.right.data_ptr(), self.rho.data_ptr(),
                ctypes.c_void_p(st.cuda_stream)), "pb_density_step")
        self._next_clear = True
        self._order_caller(stream)
        return self.rho

    def _order_caller(self, stream):
        """A public call on the engine stream (stream=None) returns device
        tensors: order the caller's current stream after it, so reading the
        result right away (e.g. .cpu()) sees the kernel's writes."""
        if stream is None:
            caller = torch.cuda.current_stream(self.device)
            if caller.cuda_stream != self.stream.cuda_stream:
                caller.wait_stream(self.stream)

    def _setup_peer(self, nbins: int, nc: int):
        from .peer import PeerBuffers

        pb = PeerBuffers({"bins0": nbins * 8, "bins1": nbins * 8, "rho": (nc + 1) * 8, "left": nc * 8,
                          "right": nc * 8, "flags": _lib.PB_PEER_FLAG_WORDS * 8},
                         self.rank, self.world, self.group, self.device)
        if not pb.available:  # no P2P path on some pair: every rank keeps the NCCL allreduce
            pb.close()
            return
        # exchange epochs live on the device (advanced by the exchange itself),
        # so steps with the exchange can be captured in CUDA graphs; zeroed
        # before the synchronize below, which orders it ahead of any exchange
        self._peer_epoch_dev = torch.zeros(1, dtype=torch.int64, device=self.device)
        torch.cuda.synchronize(self.device)  # the buffers were zeroed on the legacy stream
        self.peer = pb
        self.bins_pp = [pb.tensor("bins0", nbins, torch.int64), pb.tensor("bins1", nbins, torch.int64)]
        self.rho = pb.tensor("rho", nc + 1, torch.float64)
        self.left = pb.tensor("left", nc, torch.float64)
        self.right = pb.tensor("right", nc, torch.float64)

    def _peer_density(self, st, clear_next: bool):
        """pb_peer_density_step: every rank's bins summed over NVLink and the
        epilogue, one kernel (replaces reduce_bins + pb_density_step)."""
        pb = self.peer
        d = _lib.PbPeerDensity()
        key = "bins%d" % self.cur
        for r in range(self.world):
            d.bins[r] = pb.ptrs[key][r]
            d.left[r] = pb.ptrs["left"][r]
            d.right[r] = pb.ptrs["right"][r]
            d.rho[r] = pb.ptrs["rho"][r]
            d.flags[r] = pb.ptrs["flags"][r]
        d.rank, d.world, d.epoch = self.rank, self.world, 0
        d.epoch_dev = self._peer_epoch_dev.data_ptr()
        d.timeout_ns = int(float(os.environ.get("PB_PEER_TIMEOUT_S", "60")) * 1e9)
        nxt = self.bins_pp[1 - self.cur].data_ptr() if clear_next else None
        _lib.check(self.lib.pb_peer_density_step(ctypes.byref(d), nxt, self._coef_c, self.ndep, self.nc,
                                                 self.field_bc, self.status.data_ptr(),
                                                 ctypes.c_void_p(st.cuda_stream)), "pb_peer_density_step")

    def field(self, rho: torch.Tensor, stream=None, clear=None) -> torch.Tensor:
        cfg = self.cfg
        if not cfg.field_solve:
            return self.e  # stays identically zero (harness.py:177-178)
        st = stream if stream is not None else self.stream
        sh = ctypes.c_void_p(st.cuda_stream)
        scr = self.field_scratch.data_ptr()
        with torch.cuda.stream(st):
            src = rho
            if cfg.smoothing_passes > 0:
                _lib.check(self.lib.pb_smooth_density(rho.data_ptr(), self.rho_s.data_ptr(), self.nc,
                                                      int(cfg.smoothing_passes), scr, sh), "pb_smooth_density")
                src = self.rho_s
            solve = self.lib.pb_solve_poisson_scan if self.poisson == "scan" else self.lib.pb_solve_poisson
            _lib.check(solve(src.data_ptr(), self.phi.data_ptr(), self.nc, self.grid.dx_m,
                             cfg.consts.epsilon0, self.field_bc, cfg.phi_left,
                             cfg.phi_right, scr, sh), "poisson")
            if clear is not None:
                # the bins read by the one-kernel epilogue (and the set the
                # coming push deposits into) are zeroed with E
                a, b = clear
                _lib.check(self.lib.pb_compute_efield_clear(
                    self.phi.data_ptr(), self.e.data_ptr(), self.nc, self.grid.dx_m, self.field_bc,
                    a.data_ptr(), b.data_ptr(), a.numel(), sh), "pb_compute_efield_clear")
            else:
                _lib.check(self.lib.pb_compute_efield(self.phi.data_ptr(), self.e.data_ptr(), self.nc,
                                                      self.grid.dx_m, self.field_bc, sh), "pb_compute_efield")
        self._order_caller(stream)
        return self.e

    def _subset(self, which):
        """Species array with every species outside `which` masked out
        (inactive, no deposit): the launch skips them but keeps the caller's
        species indices for the status tallies."""
        self._species()  # resets the subset cache after buffer swaps
        key = tuple(which)
        if self._sub_cache.get(key) is None:
            arr, n = species_array(self.sp)
            for k in range(n):
                if k not in which:
                    arr[k].kind = _lib.PB_KIND_INACTIVE
                    arr[k].deposit = -1
            self._sub_cache[key] = (arr, n)
        return self._sub_cache[key]

    def _field_split(self):
        """(neutral movers, the rest) when a field-solve step can overlap the
        neutral push with the field pipeline, else ([], all)."""
        neutral = [k for k, s in enumerate(self.sp) if s.kind == _lib.PB_KIND_DRIFT]
        rest = [k for k in range(len(self.sp)) if k not in neutral]
        split = self.field_split
        if split is None:
            split = self.world > 1
        if not neutral or not rest or not split:
            return [], list(range(len(self.sp)))
        return neutral, rest

    def _density_one(self) -> torch.Tensor:
        """left/right/rho in one pb_rho_epilogue launch; the bins stay set
        until the E kernel of the same step clears them."""
        with torch.cuda.stream(self.stream):
            if self.world > 1:
                reduce_bins(self.bins, self.group)
            _lib.check(self.lib.pb_rho_epilogue(
                self.bins.data_ptr(), self._coef_c, self.ndep, self.nc, self.field_bc, self.left.data_ptr(),
                self.right.data_ptr(), self.rho.data_ptr(), self.status.data_ptr(), self._sh()),
                "pb_rho_epilogue")
        self._next_clear = True
        return self.rho

    def _fused_ok(self) -> bool:
        return (self.cfg.field_solve and self.fused_field and self.peer is None and self.poisson == "scan"
                and not self._field_split()[0])

    def _fused_cycle(self, rho_out=None):
        """pb_field_cycle on the engine stream (after the bin allreduce when
        N > 1): the density epilogue with the smoothing pass folded in, the
        scan Poisson solve and E, which also zeroes the bin set just read
        (the push deposits into the other one, zeroed one step earlier).
        rho_out: write the reported density (rho_s, or rho without
        smoothing) there instead of the engine's own buffer (run_pipelined's
        result slots: no snapshot copy)."""
        cfg = self.cfg
        read = self.bins_pp[self.cur]
        rho_buf, rho_s_buf = self.rho, self.rho_s
        if rho_out is not None:
            if cfg.smoothing_passes > 0:
                rho_s_buf = rho_out
            else:
                rho_buf = rho_out
        with torch.cuda.stream(self.stream):
            if self.world > 1:
                reduce_bins(self.bins, self.group)
            _lib.check(self.lib.pb_field_cycle(
                self.bins.data_ptr(), self._coef_c, self.ndep, self.nc, self.field_bc,
                int(cfg.smoothing_passes), self.grid.dx_m, cfg.consts.epsilon0, cfg.phi_left, cfg.phi_right,
                self.left.data_ptr(), self.right.data_ptr(), rho_buf.data_ptr(), rho_s_buf.data_ptr(),
                self.phi.data_ptr(), self.e.data_ptr(), read.data_ptr(), None, read.numel(),
                self.status.data_ptr(), self.field_scratch.data_ptr(), *self._fold_args(), self._sh()),
                "pb_field_cycle")
        if self._folds_compaction():
            self._holes_pending = False
        self._next_clear = True
        return (rho_s_buf if cfg.smoothing_passes > 0 else rho_buf), self.e

    def _folds_compaction(self) -> bool:
        """The field launch compacts the previous step's holes (see
        fold_compaction)."""
        return self.absorbing and self.fold_compaction and self._fused_ok()

    def _fold_args(self):
        """pb_field_cycle's compaction arguments: the species (their holes
        from the previous push) when the launch folds the compaction in."""
        if not self._folds_compaction():
            return (None, 0, None, 0)
        arr, n = self._species()
        return (arr, n, self.compact_scratch.data_ptr(), self.compact_scratch.numel())

    def _flush_holes(self):
        """Fill pending absorbing-wall holes now: the last push's holes when
        no field launch has folded them in yet."""
        if self._holes_pending:
            self._compact()

    def _compact(self):
        """Absorbing walls: fill the removed particles' slots from the tail (pb_compact)."""
        arr, n = self._species()
        _lib.check(self.lib.pb_compact(arr, n, self.status.data_ptr(), self.compact_scratch.data_ptr(),
                                       self.compact_scratch.numel(), self._sh()), "pb_compact")
        self._holes_pending = False

    def _field_cycle(self, rho_out=None, before_push=None):
        """Field-solve step body.  rho_out: see _fused_cycle (honoured on the
        single-launch path only; check the returned tensor).  before_push:
        called between the field launch and the push (single-launch path;
        run_pipelined snapshots the previous step's live counts there, once
        the launch has folded that step's compaction in).  The species that need no field (neutral
        movers) are pushed on the engine stream while the density epilogue
        (and across GPUs its allreduce), smoothing, Poisson and E run on the
        side stream; the charged push then waits for E.  Without neutral
        movers this is the plain serial cycle."""
        neutral, rest = self._field_split()
        if not neutral:
            if self._fused_ok():
                # density + smoothing + scan Poisson + E + bin clears: one
                # launch (pb_field_cycle), bitwise the per-phase kernels below
                rho, e = self._fused_cycle(rho_out)
            elif self.density_one and self.peer is None:
                # one-kernel epilogue (no self-clear: neighbouring nodes read
                # the same cells); E clears the bins (bitwise density())
                rho = self._density_one()
                e = self.field(rho, clear=(self.bins_pp[self.cur], self.bins_pp[1 - self.cur]))
            else:
                rho = self.density()
                e = self.field(rho)
            if self.cfg.smoothing_passes > 0:
                rho = self.rho_s
            if before_push is not None:
                before_push()
            self.push(e)
            return rho, e
        self._side.wait_stream(self.stream)
        rho = self.density(self._side)  # also clears the set the charged push deposits into
        e = self.field(rho, self._side)
        if self.cfg.smoothing_passes > 0:
            rho = self.rho_s
        done = torch.cuda.Event()
        done.record(self._side)
        if self._timing is not None:
            self._timing[0].record(self.stream)
        self.push(e, subset=neutral, flip=False)
        self.stream.wait_event(done)
        self.push(e, subset=rest)
        if self._timing is not None:
            self._timing[1].record(self.stream)
        return rho, e

    def push(self, e: torch.Tensor = None, subset=None, flip: bool = True):
        """Fused mover + deposit of the next step's density (all species, or
        the indices in `subset`; flip=False keeps the bin parity for a second
        launch of the same step)."""
        if e is None:
            e = self.e
        self._flush_holes()  # a direct push() after a step: no holes may be pushed
        arr, n = self._species() if subset is None else self._subset(subset)
        target = self.bins_pp[1 - self.cur]
        with torch.cuda.stream(self.stream):
            if not self._next_clear:  # push() without a density() in between
                target.zero_()
            if self._timing is not None and subset is None:
                self._timing[0].record(self.stream)
            _lib.check(self.lib.pb_push_deposit(arr, n, e.data_ptr(), self.nc, self.bc, target.data_ptr(),
                                                self.status.data_ptr(), self._sh()), "pb_push_deposit")
            if self._timing is not None and subset is None:
                self._timing[1].record(self.stream)
        if self.absorbing:
            # filled by resort(), the next folded field launch, or _flush_holes
            self._holes_pending = True
        if flip:
            self.cur = 1 - self.cur
            self._next_clear = False

    def resort(self):
        with torch.cuda.stream(self.stream):
            due = self._sorts_due(1)
            # folded compaction: the next field launch fills the holes, unless
            # a sort comes first
            if self.absorbing and (due or not self._folds_compaction()):
                self._compact()
            if due:
                self.sort_by_cell(due)

    def sort_by_cell(self, which=None):
        """Radix sort species (all, or the indices in `which`) by cell into
        their spare buffers and swap."""
        self._flush_holes()
        with torch.cuda.stream(self.stream):
            for k, s in enumerate(self.sp):
                if which is not None and k not in which:
                    continue
                n = s.n  # absorbing species: the kernels bound this by n_dev on device
                if n <= 1:
                    continue
                need = self.lib.pb_sort_scratch_bytes(n, self.nc)
                if self.sort_scratch is None or self.sort_scratch.numel() < need:
                    self.sort_scratch = torch.empty(need, dtype=torch.uint8, device=self.device)
                dst = s.spare()
                a, b = s.pb(n), dst.pb(n)
                _lib.check(self.lib.pb_sort_by_cell(ctypes.byref(a), ctypes.byref(b), self.nc,
                                                    self.sort_scratch.data_ptr(), self.sort_scratch.numel(),
                                                    self._sh()), "pb_sort_by_cell")
                s.swap_with_spare()
                if s.cell8 is not None:
                    pbs = s.pb(n)
                    _lib.check(self.lib.pb_cell8_build(ctypes.byref(pbs), self._sh()), "pb_cell8_build")
            self._arr = None  # graphs are keyed by buffer addresses (_graph_key)
        self._publish()

    def step(self, timed: bool = False, e_ext: torch.Tensor = None):
        """One full cycle.  Returns rho/E of this step (device tensors).

        e_ext: externally supplied E nodes (device, nc+1) for field-free runs,
        used in place of the (identically zero) field.

        The engine works on its own stream; the caller's current stream is
        ordered after the step (so reading rho/E there is safe) and the next
        step is ordered after the caller's current stream (so in-place
        updates never race the caller's reads)."""
        caller = torch.cuda.current_stream(self.device)
        self.stream.wait_stream(caller)
        # Field-free runs: E does not depend on rho, so the density epilogue
        # (and across GPUs the bin allreduce) runs on a side stream while the
        # push runs; push n waits only for epilogue n-1, which cleared the bin
        # set it deposits into.  With a field solve the cycle is serial.
        overlap = not self.cfg.field_solve
        if timed:
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
            self._timing = (ev[1], ev[2])
            ev[0].record(self.stream)
        if overlap:
            self._side.wait_stream(self.stream)
            if timed:
                ev[4].record(self._side)
            rho = self.density(self._side, clear_next=False)
            done = torch.cuda.Event(enable_timing=timed)
            done.record(self._side)
            if timed:
                ev[5] = done
            if self._epi_prev is not None:
                self.stream.wait_event(self._epi_prev)
            self._epi_prev = done
        if e_ext is not None and self.cfg.field_solve:
            raise EngineError("e_ext is for field-free runs; field_solve computes E")
        if overlap:
            e = e_ext if e_ext is not None else self.field(rho)
            self.push(e)
        else:
            # smoothed density is what the reference reports (harness.py:165-166)
            rho, e = self._field_cycle()
        self.resort()
        if timed:
            ev[3].record(self.stream)
            if not overlap:
                ev[4] = ev[5] = None
            self.phase_events.append(ev)
            self._timing = None
        self.step_index += 1
        caller.wait_stream(self.stream)
        caller.wait_stream(self._side)
        if self.check_every and self.step_index % self.check_every == 0:
            self.sync()
        return rho, e

    PIPE_GROUP = int(os.environ.get("PB_PIPE_GROUP", "4"))

    def _pipe_group(self, group):
        g = self.PIPE_GROUP if group is None else int(group)
        if g < 1:
            raise EngineError(f"pipe group must be >= 1, got {g}")
        return g

    def _pipe_buffers(self, group: int):
        """Two parities x `group` slots of device E inputs, device rho
        snapshots and pinned host results."""
        dev, nodes = self.device, self.nc + 1
        P = getattr(self, "_pipe", None)
        if P is None or P["e"].shape[1] < group:
            self._pipe = {
                "h2d": torch.cuda.Stream(dev),  # inputs never queue behind results
                "d2h": torch.cuda.Stream(dev),
                "e": torch.zeros(2, group, nodes, dtype=torch.float64, device=dev),
                "snap": torch.zeros(2, group, nodes, dtype=torch.float64, device=dev),
                "host": torch.zeros(2, group, nodes, dtype=torch.float64).pin_memory(),
                # absorbing walls: every step's live count per species
                "nsnap": torch.zeros(2, group, len(self.sp), dtype=torch.int64, device=dev),
                "nhost": torch.zeros(2, group, len(self.sp), dtype=torch.int64).pin_memory(),
            }
            # captured pipe graphs point at the old slots
            self.graphs = {k: g for k, g in self.graphs.items() if k[0] != "pipe"}

    def _snap_counts(self, gp, j):
        """Absorbing runs: snapshot every species' device live count of step
        slot (gp, j) (after the step's compaction), on the side stream so the
        copies stay out of the engine stream's kernel chain (the graph joins
        the side stream at its end; the next compaction comes a push later)."""
        if not self.absorbing:
            return
        P = self._pipe
        self._side.wait_stream(self.stream)
        with torch.cuda.stream(self._side):
            for k, s in enumerate(self.sp):
                P["nsnap"][gp, j, k:k + 1].copy_(s.n_dev, non_blocking=True)

    def run_pipelined(self, steps: int, e_source=None, on_result=None, group: int = None,
                      on_counts=None):
        """`steps` cycles driven from the host with the I/O overlapped.

        Steps run in blocks of `group` (default PB_PIPE_GROUP, 4; single
        steps around sorts).  Per block: each step's input E (a pinned host
        tensor from e_source(k), field-free runs) is copied H2D on an input
        stream into the block's device slots; the block runs on the engine
        stream (one captured graph when no sort falls inside it); each step's
        rho is snapshotted on device and the block's results are copied D2H
        into pinned host memory on a result stream.  The host launches block
        b+1 before it waits for block b's results, then calls
        on_result(k, rho_host) for each of its steps -- every step's result
        is read, one block late, while the GPU works on the next block.
        Absorbing runs also deliver each step's live counts per species to
        on_counts(k, counts_host) (device snapshots, same D2H).
        Returns the number of results delivered (== steps)."""
        G = self._pipe_group(group)
        self._pipe_buffers(G)
        P = self._pipe
        h2d, d2h = P["h2d"], P["d2h"]
        block_done = [None, None]
        d2h_done = [None, None]
        pending = None  # (parity, first step, length) of the block not yet delivered
        delivered = 0

        def deliver(blk):
            nonlocal delivered
            gp, k0, n = blk
            d2h_done[gp].synchronize()
            if on_result is not None:
                for j in range(n):
                    on_result(k0 + j, P["host"][gp, j])
            if on_counts is not None and self.absorbing:
                for j in range(n):
                    on_counts(k0 + j, P["nhost"][gp, j])
            delivered += n

        with_input = e_source is not None
        use_graphs = self._graphs_ok() and (not with_input or not self.cfg.field_solve)
        k, b = 0, 0
        while k < steps:
            gp = b % 2
            n = 1
            if use_graphs and G > 1 and k + G <= steps and not any(self._sort_due(j) for j in range(1, G + 1)):
                n = G
            if with_input:
                if block_done[gp] is not None:
                    h2d.wait_event(block_done[gp])  # block b-2 finished reading these slots
                with torch.cuda.stream(h2d):
                    for j in range(n):
                        P["e"][gp, j].copy_(e_source(k + j), non_blocking=True)
                    ev_in = torch.cuda.Event()
                    ev_in.record(h2d)
                self.stream.wait_event(ev_in)
            if use_graphs and not self._sort_due(n):
                key = ("pipe", gp, n, with_input) + self._graph_key()
                g = self.graphs.get(key)
                if g is None:
                    self.sync()
                    self.stream.synchronize()
                    g = self._capture_pipe_steps(gp, n, with_input)
                    self.graphs[key] = g
                if self._epi_prev is not None:
                    self.stream.wait_event(self._epi_prev)
                with torch.cuda.stream(self.stream):
                    g.replay()
                self._epi_prev = None
                self._holes_pending = False  # pipe graphs compact every step (live-count snapshots)
                self.cur ^= n & 1  # each replayed push deposited into the other set
                self._next_clear = False
                self.step_index += n
            else:
                rho, _ = self.step(e_ext=P["e"][gp, 0] if with_input else None)
                self._flush_holes()  # the live-count snapshot is post-compaction
                self.stream.wait_stream(self._side)  # rho may come from the side stream
                with torch.cuda.stream(self.stream):
                    P["snap"][gp, 0].copy_(rho, non_blocking=True)
                self._snap_counts(gp, 0)
                self.stream.wait_stream(self._side)  # the count copies ran on the side stream
            with torch.cuda.stream(self.stream):
                ev = torch.cuda.Event()
                ev.record(self.stream)
            block_done[gp] = ev
            if pending is not None:
                deliver(pending)  # host slots of block b-1's parity are free again after this
            d2h.wait_event(ev)
            with torch.cuda.stream(d2h):
                P["host"][gp, :n].copy_(P["snap"][gp, :n], non_blocking=True)
                if self.absorbing:
                    P["nhost"][gp, :n].copy_(P["nsnap"][gp, :n], non_blocking=True)
                d = torch.cuda.Event()
                d.record(d2h)
            d2h_done[gp] = d
            pending = (gp, k, n)
            k += n
            b += 1
        if pending is not None:
            deliver(pending)
        return delivered

    def _capture_pipe_steps(self, gp, n, with_input):
        """`n` steps as one graph: field-free runs put each density epilogue
        on the side stream concurrent with the push; field-solve runs are
        serial (density -> smooth -> Poisson -> E -> push).  Step j's rho is
        snapshotted into pipe slot (gp, j)."""
        g = torch.cuda.CUDAGraph()
        start = self.cur
        overlap = not self.cfg.field_solve
        P = self._pipe
        # absorbing walls with the compaction folded into the field launch:
        # step j's holes are filled by step j+1's field launch, so step j's
        # live counts are snapshotted right after it (before push j+1) and
        # only the block's last step compacts on its own
        fold = (self.absorbing and not overlap and self._folds_compaction() and self._fused_ok()
                and not self._field_split()[0])
        with torch.cuda.graph(g, stream=self.stream):
            prev = None
            for j in range(n):
                if overlap:
                    self._side.wait_stream(self.stream)
                    rho = self.density(self._side, clear_next=False)
                    done = torch.cuda.Event()
                    done.record(self._side)
                    if prev is not None:
                        self.stream.wait_event(prev)  # epilogue j-1 cleared this push's bin set
                    prev = done
                    self.push(P["e"][gp, j] if with_input else self.e)
                else:
                    # the single-launch field step writes the reported density
                    # straight into the result slot
                    hook = (lambda jj=j - 1: self._snap_counts(gp, jj)) if fold and j > 0 else None
                    rho, e = self._field_cycle(rho_out=P["snap"][gp, j], before_push=hook)
                if not fold or j == n - 1:
                    if self.absorbing:
                        self._compact()
                    self._snap_counts(gp, j)
                if rho.data_ptr() != P["snap"][gp, j].data_ptr():
                    if overlap:
                        snap_stream = self._side  # rho_j is final once epilogue j is done
                    else:
                        if self._field_split()[0]:
                            self.stream.wait_stream(self._side)
                        snap_stream = self.stream
                    with torch.cuda.stream(snap_stream):
                        P["snap"][gp, j].copy_(rho, non_blocking=True)
            if overlap or self._field_split()[0] or self.absorbing:
                self.stream.wait_stream(self._side)  # join the forked side stream
        # capture advanced the host-side parity; replay() of this graph does
        # the same, so restore it and let the caller account the steps
        self.cur = start
        return g

    # -- CUDA graph replay --------------------------------------------------------------
    def capture(self):
        """Capture two steps (even + odd bin set) as one CUDA graph, starting
        from the current ping-pong parity; replay() then costs one launch per
        two steps.  Sort steps run eagerly; graphs are cached per buffer state."""
        self.sync()
        self.stream.synchronize()
        return self._capture()

    def _capture(self):
        g = torch.cuda.CUDAGraph()
        start = self.cur
        # Field-free runs: E does not depend on rho, so each step's density
        # epilogue (and, across GPUs, its bin allreduce) runs on a side stream
        # concurrently with the push; push n+1 waits only for epilogue n,
        # which cleared the bin set it deposits into.
        overlap = not self.cfg.field_solve
        with torch.cuda.graph(g, stream=self.stream):
            prev = None
            for _ in range(2):
                if overlap:
                    self._side.wait_stream(self.stream)
                    rho = self.density(self._side, clear_next=False)
                    done = torch.cuda.Event()
                    done.record(self._side)
                    if prev is not None:
                        self.stream.wait_event(prev)
                    prev = done
                    self.push(self.field(rho))
                else:
                    self._field_cycle()
                if self.absorbing and not self._folds_compaction():
                    self._compact()  # else: the next field launch fills this step's holes
            if prev is not None:
                self.stream.wait_event(prev)
            if not overlap and self._field_split()[0]:
                self.stream.wait_stream(self._side)  # join the field-pipeline branch
        assert self.cur == start
        self.graphs[self._graph_key()] = g
        return g

    def prepare_graphs(self, horizon: int = None):
        """Capture up front every graph replay() can need within `horizon`
        steps: both bin parities x both buffers of every species whose sort
        falls in that window.  Capturing launches nothing, so the buffer swaps
        here are pointer bookkeeping only; timed replays then never capture."""
        if not self._graphs_ok():
            return  # NCCL-exchange steps replay eagerly: no collectives inside graphs
        self._each_buffer_state(horizon, lambda: None if self._graph_key() in self.graphs
                                else self._capture())

    def _graphs_ok(self) -> bool:
        """Steps are graph-capturable on one GPU and with the peer-memory
        density exchange (its epochs are device-side); the NCCL exchange
        runs eagerly."""
        return self.world == 1 or self.peer is not None

    def prepare_pipe_graphs(self, with_input: bool, horizon: int = None, group: int = None):
        """The same for run_pipelined's graphs (single steps and `group`-step
        blocks, both pipe parities; with_input: E comes from the pipe's device
        slots)."""
        if not self._graphs_ok() or (with_input and self.cfg.field_solve):
            return
        group = self._pipe_group(group)
        self._pipe_buffers(group)

        def cap():
            for gp in (0, 1):
                for n in sorted({1, group}):
                    key = ("pipe", gp, n, with_input) + self._graph_key()
                    if key not in self.graphs:
                        self.graphs[key] = self._capture_pipe_steps(gp, n, with_input)
        self._each_buffer_state(horizon, cap)

    def _each_buffer_state(self, horizon, fn):
        """Call fn() once per (bin parity, ping-pong buffer of every species
        sorted within `horizon` steps), restoring the current state after."""
        self.sync()
        self.stream.synchronize()
        clear0 = self._next_clear
        sorted_sp = [k for k, p in enumerate(self.sort_periods)
                     if p and (horizon is None or p <= horizon)]
        cur0 = self.cur
        for mask in range(1 << len(sorted_sp)):
            flip = [k for j, k in enumerate(sorted_sp) if mask >> j & 1]
            for k in flip:
                self.sp[k].spare()
                self.sp[k].swap_with_spare()
            self._arr = None
            for cur in (0, 1):
                self.cur = cur
                fn()
            for k in flip:
                self.sp[k].swap_with_spare()
            self._arr = None
        self.cur = cur0
        self._next_clear = clear0

    def _graph_key(self):
        """Captured graphs bake in buffer addresses: key them by the bin
        parity and every species' current (ping-pong) buffer."""
        return (self.cur,) + tuple(s.arr["x"].data_ptr() for s in self.sp)

    def _sorts_due(self, k: int) -> list:
        """Species whose sort falls after step step_index + k."""
        n = self.step_index + k
        return [i for i, p in enumerate(self.sort_periods) if p and n % p == 0]

    def _sort_due(self, k: int) -> bool:
        return bool(self._sorts_due(k))

    def replay(self, steps: int = 1):
        """Run `steps` cycles, two at a time through the captured graph; odd
        remainders and sort steps run eagerly."""
        caller = torch.cuda.current_stream(self.device)
        self.stream.wait_stream(caller)
        check, self.check_every = self.check_every, 0
        try:
            left = steps
            while left > 0:
                if self._graphs_ok() and left >= 2 and not self._sort_due(1) and not self._sort_due(2):
                    g = self.graphs.get(self._graph_key())
                    if g is None:
                        g = self.capture()
                    if self._epi_prev is not None:  # an eager epilogue may still be clearing
                        self.stream.wait_event(self._epi_prev)
                    with torch.cuda.stream(self.stream):
                        g.replay()
                    self._epi_prev = None  # the graph joined its epilogues
                    self._holes_pending = self._folds_compaction()  # its last push's holes
                    self.step_index += 2
                    left -= 2
                else:
                    self.step()
                    left -= 1
        finally:
            self.check_every = check
        caller.wait_stream(self.stream)
        if self.check_every:
            self.sync()

    # -- status handling ------------------------------------------------------------
    def close(self):
        """Release the peer-memory exchange buffers (N > 1): wait for the
        engine's work, drop the tensors that alias them, unmap the peers'
        buffers and free this rank's.  Every rank calls it; the engine is
        unusable afterwards."""
        if self.peer is None:
            return
        self.stream.synchronize()
        self._side.synchronize()
        self.graphs.clear()
        self.bins_pp = self.rho = self.left = self.right = None
        self.peer.close()
        self.peer = None

    def sync(self, window: tuple = None):
        """Wait for enqueued work, fold the sticky device status into the
        host tallies, raise the first recorded error, and reset the status.
        window=(first, last): the steps run since the previous sync, named
        in error messages when the status was not checked every step."""
        self._flush_holes()
        self.stream.synchronize()
        self._side.synchronize()
        raw = self.status.cpu().numpy()
        st = decode_status(raw)
        self.mover_ns += int(st.mover_ns)
        self.mover_launches += int(st.mover_launches)
        for k in range(len(self.sp)):
            self.moved[k] += st.moved[k]
            self.absorbed[k, 0] += st.absorbed[k][0]
            self.absorbed[k, 1] += st.absorbed[k][1]
        if self.absorbing:
            self.last_live = [int(s.n_dev.item()) for s in self.sp]
        with torch.cuda.stream(self.stream):
            self.status.copy_(self.status_tpl)
        self.stream.synchronize()
        if st.code == _lib.PB_ERR_CFL:
            key = int(st.cfl_index)
            isp, idx = key >> 56, key & ((1 << 56) - 1)
            s = self.sp[isp]
            x = float(s.arr["x"][idx].item())
            cell = int(s.cell[idx].item())
            where = f"step {self.step_index}" if window is None else f"steps {window[0]}-{window[1]}"
            raise CflViolation(
                f"{where}, phase resort: species {s.name!r} cell {cell}: "
                f"displacement of {int(math.floor(x))} cells reaches across the whole domain"
            )
        if st.code == _lib.PB_ERR_OVERFLOW:
            raise EngineError(
                f"step {self.step_index}: fixed-point deposit overflow: a cell holds {int(st.overflow)} "
                f"particles of one species (the bins represent at most {_lib.PB_MAX_CELL_COUNT})")
        if st.code == _lib.PB_ERR_PEER:
            raise EngineError(f"step {self.step_index}: density exchange failed (a peer rank timed out "
                              "or reported an error); this step's density is invalid on every rank")
        if st.code != _lib.PB_OK:
            raise EngineError(f"step {self.step_index}: device status {st.code}")

    def totals(self) -> list:
        self._flush_holes()
        return [s.live_count() for s in self.sp]

    def download(self) -> list:
        self._flush_holes()
        self.stream.synchronize()
        return [s.download() for s in self.sp]

    def phase_seconds(self) -> dict:
        """Per-phase seconds of the timed steps, from CUDA events: "mover" is
        the fused push+deposit launch, "deposit" the bin reduction and
        density epilogue (on the side stream when overlapped with the push),
        "resort" compaction / sort."""
        self.stream.synchronize()
        self._side.synchronize()
        out = {k: 0.0 for k in PHASE_KEYS}
        for ev in self.phase_events:
            total = ev[0].elapsed_time(ev[3]) * 1e-3
            mover = ev[1].elapsed_time(ev[2]) * 1e-3
            pre = ev[0].elapsed_time(ev[1]) * 1e-3
            out["mover"] += mover
            if ev[4] is not None:
                out["deposit"] += ev[4].elapsed_time(ev[5]) * 1e-3
                out["resort"] += max(0.0, total - mover - pre)
            else:
                out["deposit"] += pre
                out["resort"] += total - mover - pre
        return out

    def mover_ms(self) -> list:
        self.stream.synchronize()
        return [ev[1].elapsed_time(ev[2]) for ev in self.phase_events]
