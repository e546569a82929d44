"""Rebuild a RunConfig from a golden run's JSON record (tests only)."""

import json


def cfg_from(g, **extra):
    from paper_2404_10270_b200 import Grid1D, PhysicalConstants, RunConfig, SpeciesDef
    from paper_2404_10270_b200.config import CollisionRates, CollisionSetup

    c = json.loads(str(g["config"]))
    species = [SpeciesDef(n, q, m, nstep=ns, active_mover=am, track_transverse=tt)
               for n, q, m, ns, am, tt in c["species"]]
    coll = None
    if "collisions" in g:
        k = json.loads(str(g["collisions"]))
        coll = CollisionSetup(True, k["electron"], k["neutral"], k["ion"], CollisionRates(*k["rates"]))
    return RunConfig(grid=Grid1D.from_cells(c["nc"], c["length_m"]), consts=PhysicalConstants(dt_s=c["dt_s"]),
                     species=species, temperatures_ev=c["temperatures_ev"], densities_m3=c["densities_m3"],
                     ppc0=c["ppc0"], n_steps=c["n_steps"], seed=c["seed"], boundary=c["boundary"],
                     field_solve=c["field_solve"], smoothing_passes=c["smoothing_passes"], collisions=coll,
                     **extra)


def host_species(cfg):
    """init_plasma on the host as canonical flat dicts (oracle input)."""
    import numpy as np

    from paper_2404_10270_b200.core import init_species_host

    out = []
    for isp in range(len(cfg.species)):
        f = init_species_host(cfg, isp)
        d = dict(f.fields())
        d["cell"] = f.cell.astype(np.int32)
        out.append(d)
    return out


RUNS_ALL = ["run_periodic_nofield", "run_periodic_field", "run_dirichlet_field",
            "run_collide_periodic", "run_collide_guard", "run_collide_desk"]
COLLISION_KATS = ["suppressed", "guard", "mixed", "ionize", "guard_ionize"]
