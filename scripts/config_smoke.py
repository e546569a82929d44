"""run_simulation on every shipped config for a few steps (sanity sweep)."""
import os
import sys
import time
from dataclasses import replace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2404_10270_b200 import load_config, run_simulation  # noqa: E402

for name in sorted(os.listdir(os.path.join(ROOT, "configs"))):
    cfg = load_config(os.path.join(ROOT, "configs", name))
    if cfg.grid.nc * cfg.ppc0 * len(cfg.species) > 200_000_000:
        init = "device"
    else:
        init = "host"
    cfg = replace(cfg, n_steps=5, out_dir=None)
    t = time.perf_counter()
    m = run_simulation(cfg, init=init)
    el = time.perf_counter() - t
    last = m.diagnostics[-1]
    print(f"{name}: ok in {el:.1f}s layout={m.layout} last={last} absorbed={m.absorbed}", flush=True)
