#!/usr/bin/env python3
"""Throughput of the fused mover + deposit step (BASELINE.json metric).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (config 2 of BASELINE.json, per GPU; weak scaling for N > 1):
  nc = 100,000 cells per GPU, ppc0 = 100 per species, species e-, D+, D
  (desk.toml mix: D neutral with transverse position), fp64, E = 0 field
  (Table-1 case, field solve off), 30M particles per GPU, device-initialised
  with the reference splitmix64 streams (synthetic plasma).
A "step" = one deposit epilogue + one fused mover/deposit launch (+ the
periodic cell sort when due).  Inputs are 1.12 GB/step per GPU, ~9x the
126 MB L2, so no L2 flush is needed between steps.

The JSON line carries: value (pushes/s, whole job, device-timed, max over
ranks), roofline (push kernel: algorithmic bytes / CUDA-event duration vs the
measured HBM copy peak), cpu_baseline (the reference's own compiled kernels on
this host's cores, bounded sample), e2e (public step API with per-step host
E-field upload and rho download), clocks (nvidia-smi during the timed region).
N > 1 ranks exchange the density through peer memory (one fused kernel per
step, graph-replayed; config.density_exchange names the path used).
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NC_PER_GPU = 100_000
PPC0 = 100
SEED = 20260819
# Algorithmic reference-state bytes per push.
ALG_BYTES = {"kick": 32.0, "kick_yp": 56.0, "drift": 24.0, "drift_yp": 48.0, "boris": 64.0, "boris_yp": 80.0}
METRIC = "particle-pushes/sec (mover+deposit) at 1/2/4/8 B200; % of HBM roofline"


def desk_species():
    from paper_2404_10270_b200 import SpeciesDef
    from paper_2404_10270_b200.core import ELECTRON_MASS, ELEMENTARY_CHARGE

    # pkg/configs/desk.toml:22-43
    return [
        SpeciesDef("e", -ELEMENTARY_CHARGE, ELECTRON_MASS),
        SpeciesDef("D+", ELEMENTARY_CHARGE, 3.3435837483066354e-27),
        SpeciesDef("D", 0.0, 3.344494686676785e-27, track_transverse=True),
    ]


def make_config(nc_total, sort_every):
    from paper_2404_10270_b200 import Grid1D, PhysicalConstants, RunConfig

    return RunConfig(
        grid=Grid1D.from_cells(nc_total, nc_total * 1e-5), consts=PhysicalConstants(dt_s=4e-14),
        species=desk_species(), temperatures_ev=[20.0, 20.0, 1.0], densities_m3=[1e21] * 3,
        ppc0=PPC0, n_steps=0, seed=SEED, field_solve=False, smoothing_passes=0,
        max_store_mb=1 << 20, sort_every=sort_every,
    )


def species_alg_bytes(sp, boris=False):
    if not sp.active_mover:
        return 0.0
    key = ("boris" if boris else "kick") if sp.charged else "drift"
    return ALG_BYTES[key + ("_yp" if sp.track_transverse else "")]


# BASELINE.json configs: c2 is the default bench line; the others are run with
# --workload for the record (profiles/), from the TOML files in configs/.
WORKLOADS = {
    "c2": ("config 2: 1D3V unmagnetized, desk species e-/D+/D(yp), E=0 (field solve off)", "weak", None),
    "c3": ("config 3: bounded sheath, absorbing walls + compaction, Dirichlet field solve, cell sort",
           "weak", "configs/c3_sheath_absorbing.toml"),
    "c4": ("config 4: magnetized SOL slab, Boris push, 3 species, 100M particles total, field solve",
           "strong", "configs/c4_sol_boris.toml"),
    "c5": ("config 5: 1M cells, 1B particles total (e-/D+/D), field solve off", "strong",
           "configs/c5_weak_1m.toml"),
    "c4b": ("config 4 with a spatially varying B: Bz 2.5 -> 1.5 T along x, gathered per particle "
            "(pb_species.b_nodes), Boris push, 100M particles, field solve", "strong",
            "configs/c4b_sol_gradb.toml"),
}


def workload_config(name, world, sort_every):
    from dataclasses import replace

    from paper_2404_10270_b200 import load_config

    desc, scaling, path = WORKLOADS[name]
    if path is None:
        return make_config(NC_PER_GPU * world, sort_every), desc, scaling
    cfg = load_config(os.path.join(ROOT, path))
    if scaling == "weak" and world > 1:
        cfg = cfg.scaled_for_workers(world)
    # throughput runs use the parallel Poisson solve; the bitwise serial one
    # ("exact") is for parity runs (tests)
    cfg = replace(cfg, max_store_mb=1 << 20, n_steps=0, worker_count=1, poisson="scan",
                  sort_every=cfg.sort_every if sort_every is None else sort_every)
    return cfg, desc, scaling


def config_dict(cfg, desc, scaling, world):
    """The `config` object of the JSON line; the same for both arms."""
    from paper_2404_10270_b200.engine import Engine, partition_cells, sort_periods_for

    nc_total = cfg.grid.nc
    ranges = partition_cells(nc_total, world)
    active = [sp for sp in cfg.species if sp.active_mover]
    per_rank = [(hi - lo) * cfg.ppc0 * len(active) for lo, hi in ranges]
    alg = sum((ranges[0][1] - ranges[0][0]) * cfg.ppc0 * species_alg_bytes(sp, cfg.b_field_t is not None)
              for sp in cfg.species)
    return {
        "workload": desc,
        "nc_per_gpu": nc_total // world if scaling == "weak" else nc_total, "nc_total": nc_total,
        "ppc0_per_species": cfg.ppc0,
        "particles_per_gpu": per_rank[0], "particles_total": sum(per_rank),
        "sort_every": cfg.sort_every,
        "sort_periods": sort_periods_for(cfg, cfg.sort_every, Engine.sort_ratio_cap),
        "parallelism": f"particle shards x{world}, replicated grid",
        "l2": (f"inputs {alg / 1e9:.2f} GB/GPU vs 126 MB L2" +
               ("; each step streams past L2, no flush needed" if alg > 2 * 126e6
                else "; L2-resident, roofline not meaningful")),
    }


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi's NVML start-up can stall the GPU for tens of ms: let
            # it finish (first sample in) before anything is timed
            t0 = time.time()
            while not self.rows and time.time() - t0 < 10.0:
                time.sleep(0.02)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def build_traffic(workload, kernel):
    """DRAM bytes per mover launch from an ncu --set full capture of THIS
    kernel code (profiles/push_deposit_traffic.json records the sha256 of the
    captured kernel's SASS next to the numbers); None when the capture is of
    other code."""
    from paper_2404_10270_b200 import _lib

    path = os.path.join(ROOT, "profiles", "push_deposit_traffic.json")
    try:
        with open(path) as fh:
            rec = json.load(fh)
    except (OSError, ValueError):
        return None, "no capture"
    ent = rec.get("workloads", {}).get(workload)
    if ent is None:
        return None, f"no capture for {workload}"
    short = ent.get("kernel", "").replace("void ", "").split("(")[0]
    sym = _lib.MOVER_SYMBOLS.get(short)
    if sym is None or not short.startswith(kernel):
        return None, f"capture is of {short or 'another kernel'}, this launch ran {kernel}"
    have = _lib.kernel_digest(sym)
    if have is None:
        return None, "cuobjdump unavailable: cannot tie the capture to this build"
    if ent.get("kernel_sass_sha256") != have:
        return None, "capture is of other kernel code"
    return ent.get("dram_bytes_per_launch"), f"ncu --set full of this kernel code ({ent.get('source', path)})"


# ---------------------------------------------------------------------------
# CPU side: the reference's own compiled kernels (oracle/_ref, built from
# /root/reference sources) timed on this host's cores.
def cpu_reference_rate(target_seconds=15.0, nc=NC_PER_GPU, ppc=PPC0, threads=None, log=None):
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle

    mod = oracle.ref_kernels()
    kind = "reference"
    if mod is None:
        mod, kind = oracle, "port"
    threads = threads or os.cpu_count() or 1
    cap = int(np.ceil(1.5 * ppc))  # reference slack (config.py:55, core.py:305)
    rng = np.random.default_rng(SEED)
    offs = np.arange(nc, dtype=np.int64) * cap
    counts = np.full(nc, ppc, dtype=np.int64)
    total = nc * cap
    sig = [7.502e-3, 1.238e-4, 2.768e-5]
    stores = []
    live = (np.arange(nc)[:, None] * cap + np.arange(ppc)[None, :]).ravel()
    for k in range(3):
        d = {f: np.zeros(total) for f in ("x", "vx", "vy", "vz")}
        d["x"][live] = rng.random(live.size)
        for f in ("vx", "vy", "vz"):
            d[f][live] = sig[k] * rng.standard_normal(live.size)
        if k == 2:
            d["yp"] = np.zeros(total)
        stores.append(d)
    accel = np.full(nc + 1, -0.0)  # coef * E with E = 0 (mover.py:221)
    block = max(1, nc // (threads * 4))
    blocks = [(b, min(b + block, nc)) for b in range(0, nc, block)]

    def move(args):
        k, lo, hi = args
        d = stores[k]
        a = accel[lo:hi + 1] if k < 2 else None
        mod.fused_move(a, d["x"], d["vx"], d["vy"], d.get("yp"), offs[lo:hi], counts[lo:hi], 1.0)

    def dep(args):
        k, lo, hi = args
        mod.deposit_partials(stores[k]["x"], offs[lo:hi], counts[lo:hi])

    tasks_m = [(k, lo, hi) for k in range(3) for lo, hi in blocks]
    tasks_d = [(k, lo, hi) for k in range(2) for lo, hi in blocks]
    pushes = 3 * nc * ppc
    with ThreadPoolExecutor(threads) as pool:
        list(pool.map(move, tasks_m))
        list(pool.map(dep, tasks_d))
        reps, t0 = 0, time.perf_counter()
        while True:
            list(pool.map(move, tasks_m))
            list(pool.map(dep, tasks_d))
            reps += 1
            el = time.perf_counter() - t0
            if el >= target_seconds or reps >= 100000:
                break
    rate = pushes * reps / el
    sample = (f"{reps} steps x {pushes / 1e6:.1f}M pushes (e-, D+, D desk mix, nc={nc}, ppc={ppc}, cap={cap}) "
              f"fused_move + deposit_partials over {len(blocks)} cell blocks on a {threads}-thread pool "
              f"(mover_phase pattern, pkg/src/picmc/mover.py:227-271); {el:.1f}s")
    return {"value": rate, "unit": "particle-pushes/s", "cores": threads, "kind": kind, "sample": sample}


# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2404_10270_b200 import Engine, run_simulation

    # one GPU per rank; --dist-backend gloo lets several ranks share a GPU to
    # exercise the multi-rank path where only one GPU is visible
    dev = torch.device("cuda", local_rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    cfg, desc, scaling = workload_config(args.workload, world, args.sort_every)
    nc_total = cfg.grid.nc
    eng = Engine(cfg, device=dev, rank=rank, world=world, group=None, init="device", check_every=0)
    torch.cuda.synchronize(dev)
    pushes_rank = sum(s.n for s in eng.sp if s.kind != 0)
    boris = cfg.b_field_t is not None
    alg_bytes = sum(s.n * species_alg_bytes(s.sp, boris) for s in eng.sp)
    # gathered B: two 32-byte node reads per Boris push, served from L2 (the
    # (nc+1) x 32 B profile is 3.2 MB); reported beside, not in, alg_bytes
    b_node_bytes = (sum(s.n for s in eng.sp if s.kind == 3) * 64.0 if eng.b_nodes is not None else 0.0)

    def max_over_ranks(*vals):
        if world == 1:
            return vals
        t = torch.tensor(vals, dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return tuple(float(v) for v in t)

    # one untimed sort of every species first: first-use costs (module
    # loading, scratch allocation) stay out of the timed region; physics is
    # order-free.  Then every CUDA graph the timed replay can need (bin parity
    # x sort buffer state) is captured before timing; periodic sorts run
    # eagerly inside the timed region.
    eng.sort_by_cell()
    eng.sync()
    eng.prepare_graphs(args.warmup + args.steps)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local_rank) as clk:
        time.sleep(0.3)  # sampler start-up; the warm-up below brings the clocks back up
        eng.replay(args.warmup)
        eng.sync()
        eng.mover_ns = eng.mover_launches = 0
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        graphs_before = len(eng.graphs)
        step0 = eng.step_index
        start.record(eng.stream)
        # windows of up to 200 steps (events between graph launches cost
        # nothing) to show whether a slow run is uniformly slow or had a hiccup
        marks, left = [], args.steps
        while left > 0:
            k = min(200, left)
            eng.replay(k)
            left -= k
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(eng.stream)
            marks.append((k, ev))
        end.record(eng.stream)
        torch.cuda.synchronize(dev)
        graphs_timed = len(eng.graphs) - graphs_before
    eng.sync()
    if world > 1:
        dist.barrier()
    raw_ms = start.elapsed_time(end) / args.steps
    win_ms, prev = [], start
    for k, ev in marks:
        win_ms.append(prev.elapsed_time(ev) / k)
        prev = ev
    # The mover kernel's own duration inside the graph-replayed timed steps:
    # the persistent movers' in-kernel clock (pb_status.mover_ns, first block
    # start -> last warp end, %globaltimer).
    push_ms = eng.mover_ns / max(1, eng.mover_launches) / 1e6
    mover_launches = eng.mover_launches
    mover_kernel = eng.lib.pb_last_mover_kernel().decode()
    # Amortised sort cost: the periodic sorts that fall inside the K timed
    # steps are there at their actual count; a window shorter than a sort
    # period (the driver's 20 steps) is charged the missing fraction
    # (expected = K / period sorts per species) at the measured sort time,
    # or credited when the window held more than its share.
    sort_ms = []
    for k, p in enumerate(eng.sort_periods):
        if not p:
            sort_ms.append(0.0)
            continue
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eng.sort_by_cell([k])  # warm
        e0.record(eng.stream)
        for _ in range(3):
            eng.sort_by_cell([k])
        e1.record(eng.stream)
        torch.cuda.synchronize(dev)
        sort_ms.append(e0.elapsed_time(e1) / 3)
    in_window = [sum(1 for i in range(step0 + 1, step0 + args.steps + 1) if p and i % p == 0)
                 for p in eng.sort_periods]
    expected = [args.steps / p if p else 0.0 for p in eng.sort_periods]
    adjust_ms = sum((e - n) * t for e, n, t in zip(expected, in_window, sort_ms)) / args.steps
    ms = raw_ms + adjust_ms
    ms, push_ms, raw_ms = max_over_ranks(ms, push_ms, raw_ms)
    pushes_total = pushes_rank * world
    if world > 1:
        t = torch.tensor([pushes_rank], dtype=torch.int64, device=dev)
        dist.all_reduce(t)
        pushes_total = int(t.item())
    value = pushes_total / (ms * 1e-3)

    # e2e: the public host-driven API (Engine.run_pipelined): every step copies
    # its E-field input H2D from pinned host memory and its rho result D2H into
    # pinned host memory, which the host reads (one block of steps late, while
    # the GPU runs the next block).
    nodes = nc_total + 1
    e_host = torch.zeros(nodes, dtype=torch.float64).pin_memory()
    # steady state of the public API: at least 400 steps whatever --steps is
    # (a short run would mostly time the pipeline's one-block fill and drain)
    e2e_steps = max(args.steps, 400)
    seen = []
    # field-solve workloads compute E on device: their per-step input is none
    e_src = None if cfg.field_solve else (lambda k: e_host)

    def on_result(k, rho_host):
        seen.append(float(rho_host[k % nodes]))

    eng.prepare_pipe_graphs(e_src is not None)  # untimed, like prepare_graphs for `value`
    eng.run_pipelined(4, e_source=e_src, on_result=None)  # warm the pinned ring
    pipe_graphs0 = len(eng.graphs)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(eng.stream)
    w0 = time.perf_counter()
    eng.run_pipelined(e2e_steps, e_source=e_src, on_result=on_result)
    t1.record(eng.stream)
    torch.cuda.synchronize(dev)
    wall_ms = (time.perf_counter() - w0) * 1e3 / e2e_steps
    e2e_ms = max(t0.elapsed_time(t1) / e2e_steps, wall_ms)
    e2e_graphs_timed = len(eng.graphs) - pipe_graphs0
    assert len(seen) == e2e_steps
    (e2e_ms,) = max_over_ranks(e2e_ms)
    e2e_value = pushes_total / (e2e_ms * 1e-3)

    # Speed-of-light probe (it overwrites particle state): the same read/write
    # byte mix per species kind streamed with a trivial update and no physics.
    import ctypes
    arr, nsp = eng._species()
    actual_bytes = 0.0
    for s in eng.sp:
        if s.kind == 0:
            continue
        cell_b = 1.0 if s.cell8 is not None else 4.0
        base = {1: 24.0, 2: 32.0 + cell_b, 3: 64.0 + cell_b}[s.kind]
        actual_bytes += s.n * (base + (24.0 if s.has_yp else 0.0))
    torch.cuda.synchronize(dev)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        eng.lib.pb_stream_sol(arr, nsp, ctypes.c_void_p(eng.stream.cuda_stream))
    s0.record(eng.stream)
    for _ in range(10):
        eng.lib.pb_stream_sol(arr, nsp, ctypes.c_void_p(eng.stream.cuda_stream))
    s1.record(eng.stream)
    torch.cuda.synchronize(dev)
    sol_ms = s0.elapsed_time(s1) / 10
    exchange = ("none (one GPU)" if world == 1 else
                "peer memory: pb_peer_density_step (bins summed over NVLink/IPC + epilogue, one kernel)"
                if eng.peer is not None else
                f"{args.dist_backend} all_reduce of the fixed-point bins + pb_density_step")
    folded = eng._folds_compaction()  # walls compacted inside the field launch
    eng.close()
    del eng
    torch.cuda.empty_cache()

    # The drop-in step API: run_simulation(config) with on_step=None replays
    # CUDA graphs through run_pipelined (status checked every CHECK_EVERY
    # steps); rate = pushes / the reference's own "total" timer (the step
    # loop, after init and graph capture -- as picmc times t_run).
    from dataclasses import replace
    rs_cfg = replace(cfg, n_steps=e2e_steps)
    m = run_simulation(rs_cfg, rank=rank, world=world, device=dev, init="device")
    names = [sp.name for sp in cfg.species]
    rs_pushes = sum(sum(r[f"total_{n}"] for n, sp in zip(names, cfg.species) if sp.active_mover)
                    for r in m.diagnostics[:-1])
    (rs_total,) = max_over_ranks(m.phase_seconds["total"])
    (rs_device,) = max_over_ranks(m.phase_seconds["mover"])  # engine-stream events around the loop
    rs_value = rs_pushes / rs_total

    peak, peak_kind = measured_peak()
    achieved = alg_bytes / (push_ms * 1e-3) / 1e9
    traffic, traffic_src = build_traffic(args.workload, mover_kernel)
    # field-free: the mover + k_partials_clear + k_stitch (density epilogue);
    # field solve: the mover + k_field_fused (density, smoothing, Poisson, E
    # in one launch); walls: + k_compact
    launches_per_step = 2 if cfg.field_solve else 3
    if cfg.particle_boundary == "absorbing" and not folded:
        launches_per_step += 1
    # our kernels per sort: k_cell_count + k_cell_scatter (+ k_cell8_build
    # where the compressed cell index is kept); the scan is CUB's
    n_sort_kernels = sum(n * 3 for n in in_window)
    out = {
        "metric": METRIC,
        "value": value,
        "unit": "particle-pushes/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": scaling,
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (device init_plasma with the reference splitmix64 streams, seed 20260819)",
        "config": config_dict(cfg, desc, scaling, world),
        "density_exchange": exchange,
        "sort_amortisation": {
            "raw_ms_per_step": raw_ms, "sorts_in_window": in_window,
            "expected_sorts": [round(e, 4) for e in expected],
            "sort_ms": [round(t, 5) for t in sort_ms], "adjust_ms_per_step": adjust_ms,
            "note": "ms_per_step = raw + (expected - actual sorts in the window) x sort time / steps"},
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "peak_source": peak_kind, "kernel": mover_kernel,
            "alg_bytes_per_launch": alg_bytes, "push_ms": push_ms,
            "push_ms_source": (f"in-kernel clock over the {mover_launches} graph-replayed mover launches "
                               "of the timed steps"),
            "traffic": traffic, "traffic_source": traffic_src,
        },
        **({"b_node_reads": {"bytes_per_launch": b_node_bytes, "bytes_per_boris_push": 64.0,
                             "level": "L2 (node profile 32 B x (nc+1), not HBM state)"}}
           if b_node_bytes else {}),
        "e2e": {"value": e2e_value, "unit": "particle-pushes/s",
                "h2d_bytes_per_step": 0 if cfg.field_solve else nodes * 8,
                "d2h_bytes_per_step": nodes * 8,
                "path": "Engine.run_pipelined(): per step E-field H2D from pinned memory + step + rho D2H "
                        "into pinned memory read by the host (one graph block of PB_PIPE_GROUP steps late, "
                        "overlapped); max(device, wall)",
                "steps": e2e_steps,
                "graphs_captured_in_timed_region": e2e_graphs_timed},
        "e2e_run_simulation": {
            "value": rs_value, "unit": "particle-pushes/s", "steps": e2e_steps,
            "vs_run_pipelined": rs_value / e2e_value,
            "wall_s": rs_total, "device_s": rs_device,
            "path": "paper_2404_10270_b200.run_simulation(config) (the picmc.run_simulation signature), "
                    "on_step=None: graph replay, status every CHECK_EVERY steps; pushes / phase_seconds"
                    "['total']"},
        "gpu_launches": args.steps * launches_per_step + n_sort_kernels,
        "timing_windows_ms": {"steps_per_window": min(200, args.steps), "min": min(win_ms),
                              "median": float(np.median(win_ms)), "max": max(win_ms),
                              "argmax": int(np.argmax(win_ms)), "all": [round(w, 5) for w in win_ms],
                              "graphs_captured_in_timed_region": graphs_timed},
        "sol_probe": {"ms": sol_ms, "actual_bytes": actual_bytes, "gbs": actual_bytes / (sol_ms * 1e-3) / 1e9,
                      "mover_actual_gbs": actual_bytes / (push_ms * 1e-3) / 1e9,
                      "mover_vs_probe": sol_ms / push_ms,
                      "note": "pb_stream_sol: the mover's bytes per species kind (incl. its cell index), "
                              "trivial update, no deposit"},
    }
    return out, clk.summary()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sort-every", type=int, default=None,
                    help="base cell-sort period (default: 100 for c2, the TOML value otherwise)")
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: ranks may share one GPU (functional check of the N>1 path)")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank != 0:
            return
        if args.sort_every is None and args.workload == "c2":
            args.sort_every = 100
        cfg, desc, scaling = workload_config(args.workload, args.gpus, args.sort_every)
        ref_config = config_dict(cfg, desc, scaling, args.gpus)
        cpu = cpu_reference_rate(target_seconds=max(2.0, args.cpu_seconds))
        line = {
            "impl": "reference", "metric": METRIC, "value": cpu["value"], "unit": cpu["unit"],
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": ref_config,
            "cpu_baseline": cpu,
            "e2e": {"value": cpu["value"], "unit": cpu["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        }
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist

    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group("gloo")
    if args.sort_every is None and args.workload == "c2":
        args.sort_every = 100
    out, clocks = run_ours(args, rank, world, local_rank)
    out["clocks"] = clocks
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.workload == "c2":
        out["cpu_baseline"] = cpu_reference_rate(target_seconds=args.cpu_seconds)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
