"""The reference's shipped path on this host (SURVEY.md 8(d) CPU side-by-side
(i)): picmc.run_simulation from baseline/_ref (unmodified) on the config-2
shape with collisions off; rate = pushes / (mover + deposit phase seconds),
and also per full step.

  python scripts/ref_shipped_path.py [steps] [--backend compiled|cuda] [--workers N ...]

--backend cuda selects this repo's cuda kernels through the reference's
`picmc.backends` seam (tests/refsuite/picmc_cuda_plugin.py: the two-line
change of INTEGRATION.md §4), so the reference's own step driver --
mover_phase's threaded block tasks, deposit_charge, resort -- runs with its
hot kernels on the GPU.
"""
import argparse
import json
import os
import sys
from dataclasses import replace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("steps", nargs="?", type=int, default=3)
    ap.add_argument("--backend", default="compiled", choices=("compiled", "cuda"))
    ap.add_argument("--workers", type=int, nargs="*", default=None)
    args = ap.parse_args()
    if args.backend == "cuda":
        sys.path.insert(0, os.path.join(ROOT, "tests", "refsuite"))
        import picmc_cuda_plugin  # noqa: F401  (selects the cuda kernels)
    from picmc import backends
    from picmc.config import load_config
    from picmc.harness import run_simulation

    base = load_config(os.path.join(ROOT, "configs", "c2_ionization_100k.toml"))
    out = []
    for workers in args.workers or (1, os.cpu_count() or 1):
        cfg = replace(base, n_steps=args.steps, worker_count=workers, out_dir=None, max_store_mb=1 << 20)
        m = run_simulation(cfg)
        ph = m.phase_seconds
        names = [s.name for s in cfg.species]
        pushes = sum(sum(r[f"total_{n}"] for n in names) for r in m.diagnostics[:-1])
        out.append({
            "workers": workers, "steps": args.steps, "pushes": pushes,
            "rate_mover_deposit": pushes / (ph["mover"] + ph["deposit"]),
            "rate_full_step": pushes / ph["total"],
            "phase_seconds": ph, "backend": m.backend,
        })
    print(json.dumps({"config": "configs/c2_ionization_100k.toml (collisions off)",
                      "kind": "picmc.run_simulation, baseline/_ref (unmodified)",
                      "backend": backends.BACKEND, "runs": out}))


if __name__ == "__main__":
    main()
