"""Where run_simulation(on_step=None) spends host time between chunks:
wall time of every run_pipelined call and every status sync (config 3).

  python scripts/rs_chunk_probe.py [steps] [check_every]
"""
import os
import sys
import time
from dataclasses import replace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2404_10270_b200 import engine as E, harness  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
harness.CHECK_EVERY = int(sys.argv[2]) if len(sys.argv) > 2 else 128
cfg = bench.workload_config("c3", 1, None)[0]
log = []
orig_run, orig_sync, orig_cap = E.Engine.run_pipelined, E.Engine.sync, E.Engine._capture_pipe_steps


def run(self, *a, **k):
    t = time.perf_counter()
    r = orig_run(self, *a, **k)
    log.append(("run", a[0] if a else k.get("steps"), (time.perf_counter() - t) * 1e3))
    return r


def sync(self, *a, **k):
    t = time.perf_counter()
    r = orig_sync(self, *a, **k)
    log.append(("sync", None, (time.perf_counter() - t) * 1e3))
    return r


def cap(self, *a, **k):
    log.append(("capture", a, 0.0))
    return orig_cap(self, *a, **k)


E.Engine.run_pipelined, E.Engine.sync, E.Engine._capture_pipe_steps = run, sync, cap
dev = torch.device("cuda:0")
if os.environ.get("PROBE_PRE"):  # the bench's order: another engine runs and is freed first
    from paper_2404_10270_b200 import Engine
    pre = Engine(replace(cfg, n_steps=0), device=dev, check_every=0)
    pre.init_device() if hasattr(pre, "init_device") else None
    pre.close()
    del pre
    torch.cuda.empty_cache()
ms0 = torch.cuda.memory_stats(dev)
m = harness.run_simulation(replace(cfg, n_steps=steps), device=dev, init="device")
tot = m.phase_seconds["total"]
print(f"steps {steps} check_every {harness.CHECK_EVERY}: total {tot * 1e3:.2f} ms, "
      f"device {m.phase_seconds['mover'] * 1e3:.2f} ms")
ms1 = torch.cuda.memory_stats(dev)
print("alloc retries", ms1.get("num_alloc_retries", 0) - ms0.get("num_alloc_retries", 0),
      "cudaMalloc segments", ms1.get("segment.all.allocated", 0) - ms0.get("segment.all.allocated", 0))
caps = [x for x in log if x[0] == "capture"]
print("captures:", len(caps))
runs = [x for x in log if x[0] == "run"]
syncs = [x for x in log if x[0] == "sync"]
print("run_pipelined ms:", " ".join(f"{x[1]}:{x[2]:.2f}" for x in runs[-20:]))
print("captures after the first run_pipelined call:", sum(1 for i, x in enumerate(log) if x[0] == "capture" and any(y[0] == "run" for y in log[:i])))
print("sync ms:", " ".join(f"{x[2]:.2f}" for x in syncs[-20:]))
