"""Diagnose replay timing: graph captures and per-window times (A/B tool)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2404_10270_b200 import Engine  # noqa: E402

dev = torch.device("cuda", 0)
cfg = bench.make_config(bench.NC_PER_GPU, int(sys.argv[1]) if len(sys.argv) > 1 else 100)
eng = Engine(cfg, device=dev, init="device", check_every=0)
eng.prepare_graphs(2020)
print("periods", eng.sort_periods, "graphs after prepare", len(eng.graphs))
eng.replay(20)
eng.sync()
n0 = len(eng.graphs)
for w in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record(eng.stream)
    eng.replay(200)
    e1.record(eng.stream)
    host = time.perf_counter() - t
    torch.cuda.synchronize()
    print(f"window {w}: {e0.elapsed_time(e1) / 200:.4f} ms/step  host {host * 1e3 / 200:.4f} ms/step  graphs {len(eng.graphs)}")
# eager step timing
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(eng.stream)
for _ in range(50):
    eng.step()
e1.record(eng.stream)
torch.cuda.synchronize()
print("eager step", e0.elapsed_time(e1) / 50)
t = time.perf_counter()
eng.sort_by_cell([0])
torch.cuda.synchronize()
print("sort e (host-timed, ms)", (time.perf_counter() - t) * 1e3)
