"""Whole-step comparison on the reference's own collision scenario.

Runs `run_simulation` of the reference (installed unmodified into
baseline/_ref) and of this package (CanonicalEngine, collisions on) on the
same config, checks that the per-step diagnostics of the common steps are
identical, and prints one JSON line with the per-step times.

  python scripts/desk_compare.py [config.toml] [ref_steps] [our_steps]
"""
import json
import os
import sys
from dataclasses import replace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    cfg_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "configs", "c1_desk_ppc100.toml")
    ref_steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    our_steps = int(sys.argv[3]) if len(sys.argv) > 3 else 100
    import torch

    from paper_2404_10270_b200 import load_config, run_simulation

    cfg = load_config(cfg_path)
    ours = replace(cfg, n_steps=our_steps, out_dir=None)
    run_simulation(replace(cfg, n_steps=3, out_dir=None))  # warm-up (CUDA context, modules)
    torch.cuda.synchronize()
    m = run_simulation(ours)
    torch.cuda.synchronize()
    # the step loop only (phase "total" starts after init_plasma, in both codes)
    our_s = m.phase_seconds["total"] / our_steps
    names = [s.name for s in cfg.species]
    pushes = sum(sum(r[f"total_{n}"] for n in names) for r in m.diagnostics[:-1]) / our_steps

    ref_s = None
    same = None
    ref_dir = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref_dir, "picmc")):
        sys.path.insert(0, ref_dir)
        from picmc.config import load_config as ref_load
        from picmc.harness import run_simulation as ref_run

        rcfg = replace(ref_load(cfg_path), n_steps=ref_steps, out_dir=None)
        rm = ref_run(rcfg)
        ref_s = rm.phase_seconds["total"] / ref_steps
        same = all(a == b for a, b in zip(rm.diagnostics, m.diagnostics[: ref_steps + 1]))
    out = {
        "config": os.path.relpath(cfg_path, ROOT), "particles_per_step": pushes,
        "ours": {"s_per_step": our_s, "steps": our_steps, "layout": m.layout,
                 "pushes_per_s": pushes / our_s, "phase_seconds": m.phase_seconds},
        "reference": None if ref_s is None else {
            "s_per_step": ref_s, "steps": ref_steps, "cores": os.cpu_count(),
            "kind": "picmc.run_simulation (baseline/_ref, unmodified, workers from the config)"},
        "speedup_whole_step": None if ref_s is None else ref_s / our_s,
        "diagnostics_identical_first_steps": same,
        "tally_ours": [m.tally.elastic, m.tally.excitation, m.tally.ionization, m.tally.suppressed],
    }
    print(json.dumps(out))


if __name__ == "__main__":
    main()
