"""Where the config-2 step spends the time outside the mover kernel: graph
replay of N steps with (a) the production step, (b) the density epilogue
dropped (timing probe only -- wrong physics), (c) sorts disabled.  Prints ms
per step and the mover's in-kernel time per launch for each.

  python scripts/c2_gap_probe.py [steps]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2404_10270_b200 import Engine  # noqa: E402


def run(label, steps, no_density=False, sort_every=100):
    dev = torch.device("cuda", 0)
    cfg, _, _ = bench.workload_config("c2", 1, sort_every)
    eng = Engine(cfg, device=dev, init="device", check_every=0)
    if no_density:
        eng.density = lambda stream=None, clear_next=True: eng.rho
    eng.sort_by_cell()
    eng.sync()
    eng.prepare_graphs(steps + 20)
    eng.replay(20)
    eng.sync()
    eng.mover_ns = eng.mover_launches = 0
    torch.cuda.synchronize(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(eng.stream)
    eng.replay(steps)
    b.record(eng.stream)
    torch.cuda.synchronize(dev)
    eng.sync()
    ms = a.elapsed_time(b) / steps
    mv_us = eng.mover_ns / max(1, eng.mover_launches) / 1e3
    print(f"{label:28s} step {ms * 1e3:8.2f} us   mover {mv_us:8.2f} us   gap {ms * 1e3 - mv_us:6.2f} us",
          flush=True)
    del eng
    torch.cuda.empty_cache()


if __name__ == "__main__":
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    run("production", steps)
    run("no sort", steps, sort_every=0)
    run("no sort, no density", steps, no_density=True, sort_every=0)
    run("production", steps)
