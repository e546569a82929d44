"""Per-species timing of the fused mover (A/B tool, not a bench line).

python scripts/push_probe.py [--reps 50]
Builds the bench workload (config 2), then times pb_push_deposit on each
species alone and on all, and pb_stream_sol (same bytes, trivial math), with
CUDA events on the engine stream.  PB_LIB_PATH selects a library variant.
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2404_10270_b200 import Engine, _lib  # noqa: E402
from paper_2404_10270_b200.store import species_array  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--tag", default=os.environ.get("PB_LIB_PATH", "default"))
    ap.add_argument("--only", default=None, help="species index: time only that push (for ncu)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = bench.make_config(bench.NC_PER_GPU, 0)
    eng = Engine(cfg, device=dev, init="device", check_every=0)
    lib = eng.lib
    sh = eng._sh()
    out = {"tag": a.tag}

    def timed(fn, reps):
        st = eng.stream
        with torch.cuda.stream(st):
            for _ in range(3):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(reps):
                fn()
            e1.record(st)
        st.synchronize()
        return e0.elapsed_time(e1) / reps

    bins = eng.bins_pp[0]

    def push(sel):
        arr, n = species_array([eng.sp[k] for k in sel])
        ids = sel

        def fn():
            eng._tile_counter.zero_()  # harmless for self-resetting kernels
            bins.zero_()
            _lib.check(lib.pb_push_deposit(arr, n, eng.e.data_ptr(), eng.nc, eng.bc, bins.data_ptr(),
                                           eng.status.data_ptr(), sh), "push")
        return fn

    if a.only is not None:
        k = int(a.only)
        print(k, timed(push([k]), a.reps))
        return
    # per-species timings on the freshly initialised (cell-sorted) species
    # overhead of the two memsets alone
    def zero_only():
        pass
        bins.zero_()
    z = timed(zero_only, a.reps)
    out["zero_ms"] = round(z, 4)
    for name, sel in (("e", [0]), ("D+", [1]), ("D", [2]), ("all", [0, 1, 2])):
        ms = timed(push(sel), a.reps) - z
        alg = sum(bench.species_alg_bytes(eng.sp[k].sp) * eng.sp[k].n for k in sel)
        out[name] = {"ms": round(ms, 4), "alg_gbs": round(alg / ms / 1e6, 1)}
    # the bench's two measurements: graph-replayed steps and eager timed steps
    eng.replay(20)
    eng.sync()
    st = eng.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    eng.replay(400)
    e1.record(st)
    st.synchronize()
    out["graph_step_ms"] = round(e0.elapsed_time(e1) / 400, 4)
    eng.phase_events.clear()
    for _ in range(50):
        eng.step(timed=True)
    eng.sync()
    ms = eng.mover_ms()
    out["eager_push_ms"] = round(float(sum(ms) / len(ms)), 4)
    out["eager_push_ms_median"] = round(float(sorted(ms)[len(ms) // 2]), 4)
    for name, sel in (("sol_e", [0]), ("sol_D", [2]), ("sol_all", [0, 1, 2])):
        arr, n = species_array([eng.sp[k] for k in sel])
        ms = timed(lambda: lib.pb_stream_sol(arr, n, sh), a.reps)
        alg = sum(bench.species_alg_bytes(eng.sp[k].sp) * eng.sp[k].n for k in sel)
        out[name] = {"ms": round(ms, 4), "alg_gbs": round(alg / ms / 1e6, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
