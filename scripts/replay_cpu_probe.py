"""Is the host loop of Engine.replay() keeping ahead of the GPU?  Times the
Python side of replay(n) (wall clock, no sync) against the GPU's own time
for the same steps (CUDA events), per workload; and the cost of one bare
CUDAGraph.replay() call.

  python scripts/replay_cpu_probe.py c3
"""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2404_10270_b200 import Engine  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
    dev = torch.device("cuda", 0)
    cfg, _, _ = bench.workload_config(wl, 1, None)
    eng = Engine(cfg, device=dev, init="device", check_every=0)
    eng.sort_by_cell()
    eng.sync()
    eng.prepare_graphs(400)
    eng.replay(20)
    eng.sync()
    for n in (48, 200):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        a.record(eng.stream)
        t0 = time.perf_counter()
        eng.replay(n)
        t1 = time.perf_counter()
        b.record(eng.stream)
        torch.cuda.synchronize(dev)
        gpu = a.elapsed_time(b) * 1e3 / n
        print(f"{wl} replay({n}): host {1e6 * (t1 - t0) / n:.1f} us/step enqueue, GPU {gpu:.2f} us/step")
    g = eng.graphs.get(eng._graph_key())
    if g is not None:
        torch.cuda.synchronize(dev)
        ts = []
        for _ in range(20):
            t0 = time.perf_counter()
            with torch.cuda.stream(eng.stream):
                g.replay()
            ts.append(time.perf_counter() - t0)
            eng.cur ^= 0
        torch.cuda.synchronize(dev)
        ts.sort()
        print(f"bare CUDAGraph.replay(): median {1e6 * ts[10]:.1f} us, max {1e6 * ts[-1]:.1f} us")


if __name__ == "__main__":
    main()
