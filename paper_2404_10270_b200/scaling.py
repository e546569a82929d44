"""Strong / weak scaling sweeps over GPU counts (pkg/src/picmc/harness.py:278-383).

Same report rows, efficiency definitions and scaling.csv bytes as the
reference, with "workers" meaning GPUs (one process per GPU):

  strong: same problem and seed at every N; the physics diagnostics must be
          identical across rows (decomposition transparency), speedup =
          T(1)/T(N) against the 1-GPU row (else the first), PE = 100*S/N;
  weak:   nc scales with N (config.scaled_for_workers), ratio = T(1)/T(N)
          against the base-size 1-GPU run, PE = 100*ratio.

N = 1 runs in this process; N > 1 runs `run_simulation` under
`torch.distributed.run` (127.0.0.1 rendezvous) with one rank per GPU -- ranks
share the visible GPUs round-robin, so the gloo backend can exercise the
multi-rank path on one device.  T(N) is the max over ranks of the timed
loop, as the bench does.
"""

import csv
import os
import pickle
import socket
import subprocess
import sys
import tempfile
from dataclasses import dataclass, field, replace

from .errors import EngineError

__all__ = [
    "ScalingReport",
    "compute_parallel_efficiency",
    "compute_speedup",
    "strong_scaling_sweep",
    "weak_scaling_sweep",
    "write_scaling_csv",
]


@dataclass
class ScalingReport:
    mode: str
    rows: list
    metrics: list = field(default_factory=list)


def compute_speedup(t1: float, tn: float) -> float:
    """Wall-clock gain t1/tn of the N-GPU run over the reference run."""
    if t1 <= 0.0 or tn <= 0.0:
        raise ValueError("times must be positive")
    return t1 / tn


def compute_parallel_efficiency(speedup: float, workers: int) -> float:
    """Resource utilisation in percent: 100 * speedup / workers."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return 100.0 * speedup / workers


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def run_on_gpus(config, n: int, dist_backend: str = "nccl", timeout: float = None):
    """RunMetrics of `config` on n ranks (max-over-ranks total time)."""
    if n == 1:
        from .harness import run_simulation

        return run_simulation(config)
    with tempfile.TemporaryDirectory() as tmp:
        cfg_path, out_path = os.path.join(tmp, "cfg.pkl"), os.path.join(tmp, "out.pkl")
        with open(cfg_path, "wb") as fh:
            pickle.dump(config, fh)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
               "-m", "paper_2404_10270_b200.scaling", cfg_path, out_path, dist_backend]
        env = dict(os.environ)
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        env["PYTHONPATH"] = root + os.pathsep + env.get("PYTHONPATH", "")
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=timeout)
        if r.returncode != 0 or not os.path.exists(out_path):
            raise EngineError(f"{n}-rank run failed (rc={r.returncode}): {r.stderr[-2000:]}")
        with open(out_path, "rb") as fh:
            return pickle.load(fh)


def strong_scaling_sweep(config, worker_counts, dist_backend: str = "nccl",
                         timeout: float = None) -> ScalingReport:
    """Same problem, same seed, varying GPU count."""
    counts = list(worker_counts)
    runs = [run_on_gpus(replace(config, worker_count=w, out_dir=None), w, dist_backend, timeout)
            for w in counts]
    for r in runs[1:]:
        if r.diagnostics != runs[0].diagnostics:
            raise EngineError("diagnostics differ across GPU counts; decomposition transparency is broken")
    ref = counts.index(1) if 1 in counts else 0
    t1 = runs[ref].phase_seconds["total"]
    rows = []
    for w, r in zip(counts, runs):
        s = compute_speedup(t1, r.phase_seconds["total"])
        rows.append({"workers": w, "t_total": r.phase_seconds["total"], "t_mover": r.phase_seconds["mover"],
                     "speedup": s, "pe_percent": compute_parallel_efficiency(s, w)})
    return ScalingReport("strong", rows, runs)


def weak_scaling_sweep(config, worker_counts, dist_backend: str = "nccl",
                       timeout: float = None) -> ScalingReport:
    """Problem size grows with the GPU count (per-GPU cells fixed)."""
    counts = list(worker_counts)
    runs = {w: run_on_gpus(replace(config.scaled_for_workers(w), out_dir=None), w, dist_backend, timeout)
            for w in counts}
    if 1 in runs:
        t1 = runs[1].phase_seconds["total"]
    else:
        t1 = run_on_gpus(replace(config.scaled_for_workers(1), out_dir=None), 1).phase_seconds["total"]
    rows = []
    for w in counts:
        r = runs[w]
        ratio = compute_speedup(t1, r.phase_seconds["total"])
        rows.append({"workers": w, "t_total": r.phase_seconds["total"], "t_mover": r.phase_seconds["mover"],
                     "speedup": ratio, "pe_percent": 100.0 * ratio})
    return ScalingReport("weak", rows, [runs[w] for w in counts])


def write_scaling_csv(report: ScalingReport, path):
    """Byte-compatible with pkg/src/picmc/harness.py:374-383."""
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(["workers", "t_total", "t_mover", "speedup", "pe"])
        for r in report.rows:
            w.writerow([r["workers"], f"{r['t_total']:.9f}", f"{r['t_mover']:.9f}",
                        f"{r['speedup']:.6f}", f"{r['pe_percent']:.4f}"])


def _worker(cfg_path: str, out_path: str, dist_backend: str):
    """One rank of run_on_gpus (launched by torch.distributed.run)."""
    import torch
    import torch.distributed as dist

    from .harness import run_simulation

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    device = torch.device("cuda", local % torch.cuda.device_count())
    torch.cuda.set_device(device)
    dist.init_process_group(dist_backend, rank=rank, world_size=world)
    try:
        with open(cfg_path, "rb") as fh:
            config = pickle.load(fh)
        m = run_simulation(config, rank=rank, world=world, device=device)
        t = torch.tensor([m.phase_seconds["total"]], dtype=torch.float64,
                         device=device if dist_backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        m.phase_seconds["total"] = float(t.item())
        if rank == 0:
            with open(out_path, "wb") as fh:
                pickle.dump(m, fh)
    finally:
        dist.destroy_process_group()


if __name__ == "__main__":
    _worker(sys.argv[1], sys.argv[2], sys.argv[3])
