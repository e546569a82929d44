"""A/B: the fused field cycle (pb_field_cycle) against the per-phase chain
(pb_rho_epilogue + pb_smooth_density + pb_solve_poisson_scan +
pb_compute_efield_clear), each captured 50x in a CUDA graph, per-call time
by CUDA events; then the config-3 engine step with the engine's fused_field
on and off.  Prints one JSON line per measurement.

  python scripts/field_cycle_ab.py [nc ...]
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2404_10270_b200 import _lib  # noqa: E402


def field_only(nc, bc, reps=50, rounds=5):
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    ndep = 2
    rng = np.random.default_rng(0)
    C = rng.integers(50, 150, size=(ndep, nc)).astype(np.uint64)
    R = (rng.random((ndep, nc)) * C * 2.0 ** 48).astype(np.uint64)
    bins0 = torch.from_numpy(np.stack([R, C], 1).reshape(-1).view(np.int64)).to(dev)
    b0, b1 = bins0.clone(), bins0.clone()
    z = lambda n: torch.zeros(n, dtype=torch.float64, device=dev)  # noqa: E731
    rho, rho_s, phi, e, left, right = z(nc + 1), z(nc + 1), z(nc + 1), z(nc + 1), z(nc), z(nc)
    scr = torch.zeros(lib.pb_field_scratch_bytes(nc), dtype=torch.uint8, device=dev)
    st = torch.zeros(1024, dtype=torch.uint8, device=dev)
    coef = (ctypes.c_double * 2)(-1.7e-9, 2.3e-9)
    s = torch.cuda.Stream()
    sh = ctypes.c_void_p(s.cuda_stream)
    P = lambda t: t.data_ptr()  # noqa: E731

    def fused():
        _lib.check(lib.pb_field_cycle(P(b0), coef, ndep, nc, bc, 1, 1e-5, 8.85e-12, 0.0, 0.0, P(left), P(right),
                                      P(rho), P(rho_s), P(phi), P(e), P(b0), P(b1), 0, P(st), P(scr), sh), "fc")

    def chain():
        _lib.check(lib.pb_rho_epilogue(P(b0), coef, ndep, nc, bc, P(left), P(right), P(rho), P(st), sh), "ep")
        _lib.check(lib.pb_smooth_density(P(rho), P(rho_s), nc, 1, P(scr), sh), "sm")
        _lib.check(lib.pb_solve_poisson_scan(P(rho_s), P(phi), nc, 1e-5, 8.85e-12, bc, 0.0, 0.0, P(scr), sh), "ps")
        _lib.check(lib.pb_compute_efield_clear(P(phi), P(e), nc, 1e-5, bc, P(b1), None, 0, sh), "ef")

    out = {}
    for name, fn in (("fused", fused), ("chain", chain)):
        with torch.cuda.stream(s):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
        ts = []
        for _ in range(rounds):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):  # replay runs on the current stream
                a.record(s)
                g.replay()
                b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3 / reps)
        out[name] = round(min(ts), 3)
    return out


def engine_step(fused, steps=400):
    from dataclasses import replace

    from paper_2404_10270_b200 import Engine, load_config

    cfg = load_config(os.path.join(ROOT, "configs", "c3_sheath_absorbing.toml"))
    cfg = replace(cfg, poisson="scan", max_store_mb=1 << 20)
    eng = Engine(cfg, device=torch.device("cuda", 0), check_every=0, init="device")
    eng.fused_field = fused
    eng.sort_by_cell()
    eng.prepare_graphs(steps + 40)
    eng.replay(40)
    eng.sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(eng.stream)
    eng.replay(steps)
    b.record(eng.stream)
    torch.cuda.synchronize()
    eng.sync()
    return a.elapsed_time(b) * 1e3 / steps


if __name__ == "__main__":
    if sys.argv[1:2] == ["--engine-only"]:  # for ncu: a few steps of each
        for fused in (True, False):
            print(json.dumps({"c3_step_us": round(engine_step(fused, steps=20), 2), "fused_field": fused}))
        sys.exit(0)
    ncs = [int(v) for v in sys.argv[1:]] or [65536, 100000]
    for nc in ncs:
        for bc in (_lib.PB_FIELD_DIRICHLET, _lib.PB_FIELD_PERIODIC):
            print(json.dumps({"nc": nc, "bc": "dirichlet" if bc else "periodic", "us_per_call": field_only(nc, bc)}))
    for rep in range(2):
        for fused in (True, False):
            print(json.dumps({"c3_step_us": round(engine_step(fused), 2), "fused_field": fused, "rep": rep}))
