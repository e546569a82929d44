"""Canonical-order engine: the reference's exact slot order on the GPU, with
Monte Carlo collisions.

The production `Engine` lets particles sit in any order and deposits with
order-independent fixed-point sums; that is the fast path and the bench.
`CanonicalEngine` instead keeps every species in the reference
CellSortedStore's live slot order (pkg/src/picmc/core.py:100-181) after every
step.  That order is what the reference's collision streams are indexed by
(pkg/src/picmc/collisions.py:195-219) and what its sequential per-cell
deposit sums over (pkg/src/picmc/backends/_kernels.pyx:14-34), so a run here
reproduces `picmc.run_simulation` bit for bit -- particle stores in slot
order, rho, E, diagnostics and collision tallies -- with collisions on.

Per step, on the engine stream (harness.py:144-242 order):
  deposit   pb_deposit_partials per charged species (sequential, bitwise)
            + pb_rho_from_partials (weights in species order + stitch)
  field     smooth / Poisson / E as in Engine
  collide   pb_collide: one warp per cell, splitmix64 streams, dt guard,
            swap_remove of ionized neutrals, newborns appended to the tails
  move      pb_canonical_resort per species: push + transfer, radix sort on
            (dest cell, moved, canonical rank), gather into ping-pong buffers
One host sync per step reads the newborn count and the new live counts.
"""

import ctypes

import numpy as np
import torch

from . import _lib
from .core import ELEMENTARY_CHARGE, macro_weight
from .engine import Engine
from .errors import ConfigError, EngineError
from .rng import STREAM_COLLIDE, stream

_CTR_ELASTIC, _CTR_EXCITATION, _CTR_IONIZATION, _CTR_SUPPRESSED, _CTR_NEWBORN, _CTR_OVERFLOW = range(6)


def collide_step_key(seed: int, step: int) -> int:
    """step_stream_key (pkg/src/picmc/collisions.py:92-93)."""
    return stream(seed, STREAM_COLLIDE, step)


class CanonicalEngine(Engine):
    """Single-GPU engine in the reference's canonical slot order."""

    supports_collisions = True
    supports_peer = False  # its density allreduces fp64 partials (exact, rank order)
    fold_compaction = False  # its own resort
    use_cell8 = False  # the canonical kernels read the full cell index

    def __init__(self, config, device=None, *, rank: int = 0, world: int = 1, group=None,
                 init: str = "host", check_every: int = 1):
        # N > 1: every rank owns the particles of its cell range (the
        # reference's worker decomposition, decomposition.py:66-79,177-229):
        # collisions stay cell-local, movers that leave the range migrate.
        self.roles = None
        c = config.collisions
        if c is not None and c.enabled:
            self.roles = (config.species_index(c.electron), config.species_index(c.neutral),
                          config.species_index(c.ion))
        self._nloc = config.grid.nc * int(config.ppc0)
        super().__init__(config, device, rank=rank, world=world, group=group, init=init,
                         check_every=check_every)
        nc = self.nc
        dev = self.device
        with torch.cuda.stream(self.stream):
            self.raw = torch.zeros(max(self.ndep, 1) * 2 * nc, dtype=torch.float64, device=dev)
            self.counters = torch.zeros(6, dtype=torch.int64, device=dev)
            self.nb_per_cell = torch.zeros(nc, dtype=torch.int64, device=dev)
            ncap = self.sp[self.roles[1]].cap if self.roles else 1
            self.nb_k = torch.zeros(max(ncap, 1), dtype=torch.int32, device=dev)
            cap = max(s.cap for s in self.sp)
            self.canon_scratch = torch.empty(self.lib.pb_canonical_scratch_bytes(cap, nc),
                                             dtype=torch.uint8, device=dev)
        self.tally_last = (0, 0, 0, 0)
        self.tally_total = np.zeros(4, dtype=np.int64)
        if self.roles:
            e, n, _ = self.roles
            rates = c.rates
            p = _lib.PbCollideParams()
            p.global_offset = 0
            p.w_over_dx = macro_weight(config, n) / self.grid.dx_m
            p.dt = config.consts.dt_s
            p.rate_elastic = rates.rate_elastic_m3s
            p.rate_excitation = rates.rate_excitation_m3s
            p.rate_ionization = rates.rate_ionization_m3s
            p.threshold_j = rates.excitation_threshold_ev * ELEMENTARY_CHARGE
            p.mass_e = config.species[e].mass_kg
            p.dx_over_dt = self.grid.dx_m / config.consts.dt_s
            self.cparams = p

    # -- layout ---------------------------------------------------------------
    def _species_cap(self, isp: int, nloc: int) -> int:
        # Every ionization consumes a neutral, so the electron and ion stores
        # never outgrow n + (initial neutrals): no reallocation mid-run.
        if self.roles and isp in (self.roles[0], self.roles[2]):
            return nloc + self._nloc
        return nloc

    def deposit_current(self):
        """(Re)build per-cell offs/counts of the loaded, cell-sorted store."""
        nc = self.nc
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(self.stream):  # zero-fills ordered before the layout kernels
            if not hasattr(self, "layout_scratch"):
                self.layout_scratch = torch.empty(self.lib.pb_layout_scratch_bytes(nc), dtype=torch.uint8,
                                                  device=self.device)
                self.offs = [torch.zeros(nc + 1, dtype=torch.int64, device=self.device) for _ in self.sp]
                self.counts = [torch.zeros(nc, dtype=torch.int64, device=self.device) for _ in self.sp]
            for k, s in enumerate(self.sp):
                _lib.check(self.lib.pb_cell_layout(s.cell.data_ptr(), s.n, nc, self.offs[k].data_ptr(),
                                                   self.counts[k].data_ptr(), self.layout_scratch.data_ptr(),
                                                   self.layout_scratch.numel(), self._sh()), "pb_cell_layout")

    # -- step phases ----------------------------------------------------------
    def density(self) -> torch.Tensor:
        """deposit_partials_range + stitch (fields.py:55-92), bitwise."""
        nc = self.nc
        sh = self._sh()
        with torch.cuda.stream(self.stream):
            for k, s in enumerate(self.sp):
                if s.deposit < 0:
                    continue
                base = self.raw.data_ptr() + s.deposit * 2 * nc * 8
                _lib.check(self.lib.pb_deposit_partials(s.arr["x"].data_ptr(), self.offs[k].data_ptr(),
                                                        self.counts[k].data_ptr(), nc, base, base + nc * 8,
                                                        sh), "pb_deposit_partials")
            if self.world > 1:
                # each cell's partials come from its owner alone (zeros
                # elsewhere), so the sum is exact: bitwise the single domain
                import torch.distributed as dist

                dist.all_reduce(self.raw, group=self.group)
            _lib.check(self.lib.pb_rho_from_partials(self.raw.data_ptr(), self._coef_c, self.ndep, nc,
                                                     self.field_bc, self.left.data_ptr(),
                                                     self.right.data_ptr(), self.rho.data_ptr(), sh),
                       "pb_rho_from_partials")
        return self.rho

    def collide(self, step: int) -> int:
        """collision_phase (collisions.py:310-351); returns newborn pairs."""
        if not self.roles:
            return 0
        e, n, i = self.roles
        se, sn, si = self.sp[e], self.sp[n], self.sp[i]
        self.cparams.step_key = collide_step_key(self.cfg.seed, step)
        if self.world > 1:  # newborn pairs <= live neutrals of this rank
            se.ensure_capacity(se.n + sn.n)
            si.ensure_capacity(si.n + sn.n)
            if self.nb_k.numel() < max(sn.n, 1):
                self.nb_k = torch.zeros(sn.n, dtype=torch.int32, device=self.device)
            self._arr = None
        cap = min(se.cap - se.n, si.cap - si.n)
        self.stream.wait_stream(torch.cuda.current_stream(self.device))  # growth / nb_k fills above
        with torch.cuda.stream(self.stream):
            pe, pn, pi = se.pb(), sn.pb(), si.pb()
            _lib.check(self.lib.pb_collide(
                ctypes.byref(pe), ctypes.byref(pn), ctypes.byref(pi),
                self.offs[e].data_ptr(), self.counts[e].data_ptr(), self.offs[n].data_ptr(),
                self.counts[n].data_ptr(), self.nc, ctypes.byref(self.cparams),
                self.nb_per_cell.data_ptr(), self.nb_k.data_ptr(), cap, self.counters.data_ptr(),
                self._sh()), "pb_collide")
        self.stream.synchronize()  # the copy below runs on the caller's stream
        ctr = self.counters.cpu().numpy()
        if ctr[_CTR_OVERFLOW]:
            raise EngineError(f"collision pass overflow ({int(ctr[_CTR_OVERFLOW])} events): newborn "
                              "capacity or dt-guard depth exceeded")
        self._ionized_local = int(ctr[_CTR_IONIZATION])
        tally = ctr[:4].copy()
        if self.world > 1:
            import torch.distributed as dist

            t = torch.tensor(tally, dtype=torch.int64, device=self._coll_device())
            dist.all_reduce(t, group=self.group)
            tally = t.cpu().numpy()
        self.tally_last = tuple(int(v) for v in tally)
        self.tally_total += tally
        return int(ctr[_CTR_NEWBORN])

    def _coll_device(self):
        """Device for small collective tensors (gloo works on the host)."""
        import torch.distributed as dist

        return torch.device("cpu") if dist.get_backend(self.group) == "gloo" else self.device

    def push(self, e: torch.Tensor = None, newborns: int = 0):
        """Push + transfer + canonical resort of every species (one C call)."""
        if e is None:
            e = self.e
        if self.world > 1:
            return self._push_multirank(e, newborns)
        roles = self.roles or (-1, -1, -1)
        nsp = len(self.sp)
        src = (_lib.PbSpecies * nsp)()
        dst = (_lib.PbSpecies * nsp)()
        cvs = (_lib.PbCanon * nsp)()
        for k, s in enumerate(self.sp):
            tail = newborns if k in (roles[0], roles[2]) else 0
            cv = cvs[k]
            cv.n_old = s.n
            cv.n_tail = tail
            cv.offs = self.offs[k].data_ptr()
            cv.counts = self.counts[k].data_ptr()
            cv.newborn_per_cell = self.nb_per_cell.data_ptr() if tail else None
            cv.newborn_k = self.nb_k.data_ptr() if tail else None
            src[k] = s.pb(s.n + tail)
            dst[k] = s.spare().pb(s.n + tail)
        news = (ctypes.c_int64 * nsp)()
        _lib.check(self.lib.pb_canonical_step(
            src, dst, cvs, nsp, e.data_ptr(), self.nc, self.bc, self.status.data_ptr(),
            self.canon_scratch.data_ptr(), self.canon_scratch.numel(), news, self._sh()),
            "pb_canonical_step")
        for s, nn in zip(self.sp, news):
            s.swap_with_spare()
            s.n = int(nn)
            if s.absorbing:
                s.n_dev.fill_(s.n)
        self._arr = None

    def _push_multirank(self, e, newborns):
        """Canonical push across ranks: keys with a global canonical rank
        (pb_canonical_keys), emigrants exchanged with all_to_all, the union
        ordered by key -- per destination cell the survivors in slot order,
        then newborns, then incomers by (src cell, src slot), exactly the
        single-domain order (resort_collect / commit_incomers /
        migrate_particles, pkg/src/picmc/mover.py:113-208,
        decomposition.py:177-229)."""
        import torch.distributed as dist

        roles = self.roles or (-1, -1, -1)
        cdev = self._coll_device()
        hi = torch.tensor([h for _, h in self.partition.ranges], dtype=torch.int64, device=self.device)
        for k, s in enumerate(self.sp):
            tail = newborns if k in (roles[0], roles[2]) else 0
            n_tot = s.n + tail
            dead = getattr(self, "_ionized_local", 0) if k == roles[1] else 0
            n_pre = torch.tensor([n_tot - dead], dtype=torch.int64, device=cdev)
            allp = [torch.zeros_like(n_pre) for _ in range(self.world)]
            dist.all_gather(allp, n_pre, group=self.group)
            allp = [int(v.item()) for v in allp]
            offset, total = sum(allp[: self.rank]), sum(allp)
            rb = max(1, int(total).bit_length())
            cv = _lib.PbCanon()
            cv.n_old, cv.n_tail = s.n, tail
            cv.offs, cv.counts = self.offs[k].data_ptr(), self.counts[k].data_ptr()
            cv.newborn_per_cell = self.nb_per_cell.data_ptr() if tail else None
            cv.newborn_k = self.nb_k.data_ptr() if tail else None
            keys = torch.empty(max(n_tot, 1), dtype=torch.int64, device=self.device)
            need = self.lib.pb_canonical_scratch_bytes(max(n_tot, 1), self.nc)
            if self.canon_scratch.numel() < need:
                self.canon_scratch = torch.empty(need, dtype=torch.uint8, device=self.device)
            with torch.cuda.stream(self.stream):
                a = s.pb(n_tot)
                _lib.check(self.lib.pb_canonical_keys(
                    ctypes.byref(a), ctypes.byref(cv), e.data_ptr(), self.nc, self.bc, k,
                    self.status.data_ptr(), offset, rb, keys.data_ptr(), self.canon_scratch.data_ptr(),
                    self.canon_scratch.numel(), self._sh()), "pb_canonical_keys")
            self.stream.synchronize()
            keys = keys[:n_tot]
            names = list(s.arr)
            cols = [s.arr[f][:n_tot] for f in names] + [keys.view(torch.float64)]
            rows = torch.stack(cols, dim=1)
            live = keys != -1
            cell = torch.where(live, keys >> (rb + 1), torch.zeros_like(keys))
            owner = torch.bucketize(cell, hi, right=True)
            owner = torch.where(live, owner, torch.full_like(owner, self.world))  # dead -> dropped
            order = torch.argsort(owner, stable=True)
            send_counts = torch.bincount(owner, minlength=self.world + 1)[: self.world]
            rows = rows[order][: int(send_counts.sum())]
            sc = send_counts.to(cdev)
            rc = torch.empty_like(sc)
            dist.all_to_all_single(rc, sc, group=self.group)
            sizes_in, sizes_out = sc.tolist(), rc.tolist()
            out = torch.empty((sum(sizes_out), rows.shape[1]), dtype=torch.float64, device=cdev)
            dist.all_to_all_single(out, rows.to(cdev), sizes_out, sizes_in, group=self.group)
            got = out.to(self.device)
            gkeys = got[:, -1].contiguous().view(torch.int64)
            srt = torch.argsort(gkeys, stable=True)
            got = got[srt]
            m = int(got.shape[0])
            s.ensure_capacity(m)
            dst = s.spare()
            for j, f in enumerate(names):
                dst.arr[f][:m].copy_(got[:, j])
            gk = got[:, -1].contiguous().view(torch.int64)
            cells = (gk >> (rb + 1)).to(torch.int32)
            dst.cell[:m].copy_(cells)
            counts = torch.bincount(cells.to(torch.int64), minlength=self.nc)
            self.counts[k].copy_(counts)
            self.offs[k][0] = 0
            torch.cumsum(counts, 0, out=self.offs[k][1:])
            s.swap_with_spare()
            s.n = m
            if s.absorbing:
                s.n_dev.fill_(s.n)
        self._arr = None
        torch.cuda.synchronize(self.device)

    def resort(self):
        pass  # the canonical resort is part of push()

    def step(self, timed: bool = False):
        caller = torch.cuda.current_stream(self.device)
        self.stream.wait_stream(caller)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)] if timed else None
        mark = (lambda k: ev[k].record(self.stream)) if timed else (lambda k: None)
        mark(0)
        rho = self.density()
        mark(1)
        e = self.field(rho)
        if self.cfg.field_solve and self.cfg.smoothing_passes > 0:
            rho = self.rho_s
        mark(2)
        newborns = self.collide(self.step_index + 1)
        mark(3)
        self.push(e, newborns)
        mark(4)
        if timed:
            self.phase_events.append(ev)
        self.step_index += 1
        caller.wait_stream(self.stream)
        if self.check_every and self.step_index % self.check_every == 0:
            self.sync()
        return rho, e

    def phase_seconds(self) -> dict:
        """deposit / solve (smooth + Poisson + E) / collide / mover (push +
        canonical resort) from CUDA events on the engine stream."""
        self.stream.synchronize()
        out = {k: 0.0 for k in ("deposit", "smooth", "solve", "gather", "collide", "mover",
                                "resort", "migrate")}
        for ev in self.phase_events:
            out["deposit"] += ev[0].elapsed_time(ev[1]) * 1e-3
            out["solve"] += ev[1].elapsed_time(ev[2]) * 1e-3
            out["collide"] += ev[2].elapsed_time(ev[3]) * 1e-3
            out["mover"] += ev[3].elapsed_time(ev[4]) * 1e-3
        return out

    def mover_ms(self) -> list:
        self.stream.synchronize()
        return [ev[3].elapsed_time(ev[4]) for ev in self.phase_events]

    def capture(self):
        raise EngineError("the canonical-order engine syncs every step; it is not graph-captured")

    def replay(self, steps: int = 1):
        for _ in range(steps):
            self.step()

    def prepare_pipe_graphs(self, with_input: bool, horizon: int = None, group: int = None):
        pass  # no graphs: every step syncs for the newborn / migration counts

    def run_pipelined(self, steps: int, e_source=None, on_result=None, group: int = None):
        """Host-driven loop of the canonical engine: eager steps (each one
        syncs anyway), every step's rho copied to the host and handed to
        on_result(k, rho_host).  E is always computed on device here."""
        if e_source is not None:
            raise EngineError("the canonical-order engine takes no external E input")
        for k in range(steps):
            rho, _ = self.step()
            if on_result is not None:
                on_result(k, rho.cpu())
        return steps

    def totals(self) -> list:
        return [s.n for s in self.sp]

    def sync(self):
        super().sync()
        if self.absorbing:
            self.last_live = [s.n for s in self.sp]
