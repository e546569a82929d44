"""`run_simulation(config, on_step=None) -> RunMetrics` on the B200 engine.

Same signature, diagnostics rows, on_step state keys and RunMetrics fields as
the reference step driver (pkg/src/picmc/harness.py:66-113, :246-268), so a
caller can swap `picmc.run_simulation` for this one.  Phase timers come from
CUDA events on the engine stream instead of perf_counter.
"""

import csv
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .canonical import CanonicalEngine
from .engine import PHASE_KEYS, Engine

BACKEND = "cuda"


@dataclass
class CollisionTally:
    elastic: int = 0
    excitation: int = 0
    ionization: int = 0
    suppressed: int = 0

    def merge(self, other: "CollisionTally"):
        self.elastic += other.elastic
        self.excitation += other.excitation
        self.ionization += other.ionization
        self.suppressed += other.suppressed


@dataclass
class RunMetrics:
    phase_seconds: dict
    diagnostics: list
    config_hash: str
    worker_count: int
    layout: str
    backend: str
    tally: CollisionTally
    absorbed: dict = field(default_factory=dict)  # config 3: per species [left, right]


class _LazyStores(list):
    """on_step's "stores": a one-element list holding the host copy of THIS
    rank's species (fetched on first use).  The reference passes every
    worker's store (harness.py:246-253); with one process per GPU a rank
    holds only its own shard, so len() is 1 on every rank -- gather across
    ranks explicitly if all shards are needed."""

    def __init__(self, engine):
        super().__init__()
        self._engine = engine
        self._loaded = False

    def _load(self):
        if not self._loaded:
            super().extend([self._engine.download()])
            self._loaded = True

    def __len__(self):
        return 1

    def __getitem__(self, i):
        self._load()
        return super().__getitem__(i)

    def __iter__(self):
        self._load()
        return super().__iter__()


def _diag_row(step, names, totals, tally):
    row = {"step": step}
    for name, t in zip(names, totals):
        row[f"total_{name}"] = int(t)
    row["elastic"] = tally.elastic
    row["excitation"] = tally.excitation
    row["ionization"] = tally.ionization
    row["suppressed"] = tally.suppressed
    return row


def _global_totals(engine):
    tot = engine.totals()
    if engine.absorbing and hasattr(engine, "last_live"):
        tot = list(engine.last_live)
    if engine.world > 1:
        import torch.distributed as dist

        t = torch.tensor(tot, dtype=torch.int64, device=engine.device)
        dist.all_reduce(t, group=engine.group)
        tot = [int(v) for v in t.cpu()]
    return tot


# Fast path (on_step=None): the device status is checked every CHECK_EVERY
# steps instead of every step; an error names the window it occurred in.
CHECK_EVERY = int(os.environ.get("PB_CHECK_EVERY", "128"))


def _run_graphed(engine, config, names):
    """on_step=None and no collisions: the steps run as replayed CUDA graphs
    through Engine.run_pipelined (blocks of PB_PIPE_GROUP steps, every graph
    captured before the timed loop, like the reference's init before t_run),
    the status is checked every CHECK_EVERY steps, and the per-step
    diagnostics come from device counters (absorbing walls: each step's live
    counts snapshotted on device; otherwise the totals are invariant).
    Returns (diagnostics rows 1..n, phase seconds)."""
    n = int(config.n_steps)
    if any(engine.sort_periods):
        # init, not the step loop, pays for the sort path's first use: CUDA
        # loads kernels lazily (its first launch inside the loop stalled the
        # engine stream by 3-150 ms, profiles/r02_run_simulation_spread.txt)
        # and the scratch is allocated here; a cell sort is a no-op for the
        # physics (the cycle's own sorts reorder slots the same way)
        engine.sort_by_cell()
    engine.prepare_pipe_graphs(with_input=False, horizon=n)
    tot0 = _global_totals(engine)
    counts = np.zeros((n, len(names)), dtype=np.int64) if engine.absorbing else None
    t_run = time.perf_counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(engine.stream)
    done = 0
    while done < n:
        m = min(max(1, CHECK_EVERY), n - done)

        def on_counts(k, c, base=done):
            counts[base + k] = c.numpy()

        engine.run_pipelined(m, on_counts=on_counts if counts is not None else None)
        engine.sync(window=(done + 1, done + m))
        done += m
    ev1.record(engine.stream)
    engine.stream.synchronize()
    total = time.perf_counter() - t_run
    if counts is not None and engine.world > 1:
        import torch.distributed as dist

        t = torch.from_numpy(counts).to(engine.device)
        dist.all_reduce(t, group=engine.group)
        counts = t.cpu().numpy()
    zero = CollisionTally()
    rows = [_diag_row(step, names, counts[step - 1] if counts is not None else tot0, zero)
            for step in range(1, n + 1)]
    phase = {k: 0.0 for k in PHASE_KEYS}
    # one fused launch does gather + push + transfer + deposit: its device
    # time is reported as the mover phase (field and epilogue kernels included)
    phase["mover"] = ev0.elapsed_time(ev1) * 1e-3 if n else 0.0
    phase["total"] = total if n else 0.0
    return rows, phase


def run_simulation(config, on_step=None, *, rank=0, world=1, group=None,
                   device=None, init="host") -> RunMetrics:
    """Execute n_steps of the cycle on the GPU; returns timers and diagnostics.

    With on_step=None (and no collisions) the steps replay as CUDA graphs with
    the status checked every CHECK_EVERY steps (_run_graphed); with on_step
    every step is run eagerly, checked, and its state handed to on_step."""
    canonical = config.canonical() if hasattr(config, "canonical") else False
    cls = CanonicalEngine if canonical else Engine
    fast = on_step is None and not canonical
    engine = cls(config, device=device, rank=rank, world=world, group=group, init=init,
                 check_every=0 if fast else 1)
    names = [sp.name for sp in config.species]
    zero = CollisionTally()
    diagnostics = [_diag_row(0, names, _global_totals(engine), zero)]
    tally_sum = CollisionTally()
    if fast:
        rows, phase = _run_graphed(engine, config, names)
        diagnostics += rows
        return _finish(config, engine, names, diagnostics, phase, tally_sum, world, rank, canonical)
    t0 = time.perf_counter()
    for step in range(1, config.n_steps + 1):
        rho, e = engine.step(timed=True)
        tally = CollisionTally(*engine.tally_last) if canonical else CollisionTally()
        tally_sum.merge(tally)
        diagnostics.append(_diag_row(step, names, _global_totals(engine), tally))
        if on_step is not None:
            on_step(step, {
                "rho": rho.cpu().numpy().copy(),
                "e_field": e.cpu().numpy().copy(),
                "stores": _LazyStores(engine),
                "partition": engine.partition,
                "tally": tally,
            })
    engine.sync()
    phase = engine.phase_seconds()
    phase["total"] = time.perf_counter() - t0 if config.n_steps > 0 else 0.0
    return _finish(config, engine, names, diagnostics, phase, tally_sum, world, rank, canonical)


def _finish(config, engine, names, diagnostics, phase, tally_sum, world, rank, canonical):
    metrics = RunMetrics(
        phase_seconds=phase, diagnostics=diagnostics, config_hash=config.config_hash(),
        worker_count=world, layout="canonical_soa" if canonical else "flat_soa", backend=BACKEND,
        tally=tally_sum,
        absorbed={n: engine.absorbed[k].tolist() for k, n in enumerate(names)},
    )
    if config.out_dir is not None and rank == 0:
        os.makedirs(config.out_dir, exist_ok=True)
        write_diagnostics_csv(diagnostics, names, os.path.join(config.out_dir, "diagnostics.csv"))
        write_metrics_csv(phase, os.path.join(config.out_dir, "metrics.csv"))
    return metrics


def write_diagnostics_csv(diagnostics, names, path):
    """Byte-compatible with pkg/src/picmc/harness.py:355-363."""
    cols = ["step"] + [f"total_{n}" for n in names] + ["elastic", "excitation", "ionization", "suppressed"]
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(cols)
        for row in diagnostics:
            w.writerow([row[c] for c in cols])


def write_metrics_csv(phase_seconds, path):
    """Byte-compatible with pkg/src/picmc/harness.py:366-371."""
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(["phase", "seconds"])
        for key in PHASE_KEYS + ("total",):
            w.writerow([key, f"{phase_seconds.get(key, 0.0):.9f}"])


# the reference keeps its scaling driver in harness.py (:278-383)
from .scaling import (ScalingReport, compute_parallel_efficiency, compute_speedup,  # noqa: E402,F401
                      strong_scaling_sweep, weak_scaling_sweep, write_scaling_csv)
