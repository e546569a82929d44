"""Eager step() vs graph replay on one GPU (config 2): the per-step host cost
an N > 1 run pays when it cannot replay graphs."""
import time

import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
from paper_2404_10270_b200 import Engine  # noqa: E402

cfg, _, _ = bench.workload_config("c2", 1, 100)
eng = Engine(cfg, device=torch.device("cuda", 0), init="device", check_every=0)
eng.sort_by_cell()
eng.prepare_graphs(400)
for mode in ("replay", "eager", "replay", "eager"):
    eng.replay(10) if mode == "replay" else [eng.step() for _ in range(10)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h0 = time.process_time()
    if mode == "replay":
        eng.replay(400)
    else:
        for _ in range(400):
            eng.step()
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"{mode}: {(t1 - t0) / 400 * 1e3:.4f} ms/step wall, host enqueue {(h1 - t0) / 400 * 1e3:.4f} ms/step")
