"""Config 3 graph-replayed step time with the absorbing-wall compaction
folded into the next field launch (Engine.fold_compaction) vs its own
launch, interleaved.

  python scripts/fold_probe.py [steps]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2404_10270_b200 import Engine  # noqa: E402


def run(fold, steps):
    dev = torch.device("cuda", 0)
    cfg, _, _ = bench.workload_config("c3", 1, None)
    eng = Engine(cfg, device=dev, init="device", check_every=0)
    eng.fold_compaction = fold
    eng.sort_by_cell()
    eng.sync()
    eng.prepare_graphs(steps + 40)
    eng.replay(40)
    eng.sync()
    torch.cuda.synchronize(dev)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(eng.stream)
    eng.replay(steps)
    b.record(eng.stream)
    torch.cuda.synchronize(dev)
    eng.sync()
    print(f"c3 fold={int(fold)}: step {a.elapsed_time(b) / steps * 1e3:8.2f} us  absorbed {eng.absorbed.tolist()}",
          flush=True)
    del eng
    torch.cuda.empty_cache()


if __name__ == "__main__":
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 800
    for _ in range(2):
        for fold in (True, False):
            run(fold, steps)
