import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
from paper_2404_10270_b200 import Engine
dev = torch.device("cuda", 0)
cfg, _, _ = bench.workload_config("c3", 1, None)
eng = Engine(cfg, device=dev, init="device", check_every=0)
eng.prepare_graphs(420)
eng.replay(10); eng.sync()
out = []
for w in range(16):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record(eng.stream); eng.replay(25); e1.record(eng.stream)
    h = time.perf_counter() - h0
    torch.cuda.synchronize()
    out.append((round(e0.elapsed_time(e1) / 25, 4), round(h * 1e3 / 25, 4)))
print(os.environ.get("PB_CELL8"), eng.sort_periods, [s.cell8 is not None for s in eng.sp], out)
