import sys, time
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import torch
from dataclasses import replace
from paper_2404_10270_b200 import load_config
from paper_2404_10270_b200.canonical import CanonicalEngine
cfg = load_config(sys.argv[1] if len(sys.argv) > 1 else 'configs/c2_collisions_100k.toml')
cfg = replace(cfg, n_steps=0)
eng = CanonicalEngine(cfg, device=torch.device('cuda', 0), init='device', check_every=0)
for _ in range(3): eng.step()
torch.cuda.synchronize()
eng.phase_events = []
t0 = time.perf_counter()
for _ in range(20): eng.step(timed=True)
torch.cuda.synchronize()
t = (time.perf_counter() - t0) / 20
ph = eng.phase_seconds()
print(f"wall {t*1e3:.3f} ms/step", {k: round(v / 20 * 1e3, 3) for k, v in ph.items() if v})
print("particles", [s.n for s in eng.sp])
