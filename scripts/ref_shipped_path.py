"""The reference's shipped path on this host (SURVEY.md 8(d) CPU side-by-side
(i)): picmc.run_simulation from baseline/_ref (unmodified) on the config-2
shape with collisions off, worker_count 1 and os.cpu_count(); rate =
pushes / (mover + deposit phase seconds), and also per full step.

  python scripts/ref_shipped_path.py [steps]
"""
import json
import os
import sys
from dataclasses import replace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

from picmc.config import load_config  # noqa: E402
from picmc.harness import run_simulation  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    base = load_config(os.path.join(ROOT, "configs", "c2_ionization_100k.toml"))
    out = []
    for workers in (1, os.cpu_count() or 1):
        cfg = replace(base, n_steps=steps, worker_count=workers, out_dir=None, max_store_mb=1 << 20)
        m = run_simulation(cfg)
        ph = m.phase_seconds
        names = [s.name for s in cfg.species]
        pushes = sum(sum(r[f"total_{n}"] for n in names) for r in m.diagnostics[:-1])
        out.append({
            "workers": workers, "steps": steps, "pushes": pushes,
            "rate_mover_deposit": pushes / (ph["mover"] + ph["deposit"]),
            "rate_full_step": pushes / ph["total"],
            "phase_seconds": ph,
        })
    print(json.dumps({"config": "configs/c2_ionization_100k.toml (collisions off)",
                      "kind": "picmc.run_simulation, baseline/_ref (unmodified)", "runs": out}))


if __name__ == "__main__":
    main()
