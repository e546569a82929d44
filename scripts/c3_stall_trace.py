"""Long-run cycle times of the graph-replayed config-3 step from the device
launch logs (a PB_MOVER_TRACE + PB_FF_TRACE build): mover start-to-start for
400 steps, where the slow cycles fall and what they are made of.

  PB_LIB_PATH=build/v_gaptrace/libpicmc_b200.so python scripts/c3_stall_trace.py [steps] [group]
"""
import ctypes
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2404_10270_b200 import Engine, _lib  # noqa: E402


def logs(lib):
    ml = (ctypes.c_ulonglong * 1024)()
    fl = (ctypes.c_ulonglong * 1024)()
    mn, fn = ctypes.c_ulonglong(), ctypes.c_ulonglong()
    lib.pb_debug_mover_log.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    lib.pb_debug_field_log.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
    _lib.check(lib.pb_debug_mover_log(ml, ctypes.byref(mn)), "pb_debug_mover_log")
    _lib.check(lib.pb_debug_field_log(fl, ctypes.byref(fn)), "pb_debug_field_log")
    return (np.array(ml, dtype=np.int64).reshape(512, 2), mn.value,
            np.array(fl, dtype=np.int64).reshape(512, 2), fn.value)


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    group = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    dev = torch.device("cuda", 0)
    cfg, _, _ = bench.workload_config("c3", 1, None)
    eng = Engine(cfg, device=dev, init="device", check_every=0)
    eng.sort_by_cell()
    eng.sync()
    eng.prepare_graphs(steps + 100)
    eng.replay(20)
    eng.sync()
    lib = _lib.load()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(eng.stream)
    t0 = time.perf_counter()
    if group:
        for _ in range(steps // group):
            eng.replay(group)
    else:
        eng.replay(steps)
    t1 = time.perf_counter()
    b.record(eng.stream)
    torch.cuda.synchronize(dev)
    print(f"{steps} steps: GPU {a.elapsed_time(b) * 1e3 / steps:.2f} us/step, host enqueue "
          f"{(t1 - t0) * 1e6 / steps:.1f} us/step")
    M, mn, F, fn = logs(lib)
    k = min(steps, 500)
    mi = [(mn - k + j) % 512 for j in range(k)]
    fi = [(fn - k + j) % 512 for j in range(k)]
    Ms, Me, Fs, Fe = M[mi, 0], M[mi, 1], F[fi, 0], F[fi, 1]
    cyc = np.diff(Ms) / 1e3
    med = np.median(cyc)
    print(f"cycles: median {med:.2f} mean {cyc.mean():.2f} p90 {np.percentile(cyc, 90):.2f} max {cyc.max():.2f} us")
    slow = np.nonzero(cyc > med + 15)[0]
    print(f"slow cycles (> median + 15 us): {len(slow)} at", slow.tolist()[:40])
    print("  their lengths:", [round(float(cyc[i]), 1) for i in slow[:40]])
    if len(slow) > 1:
        print("  spacing:", np.diff(slow).tolist()[:40])
        print("  spacing in ms:", [round(float((Ms[j] - Ms[i]) / 1e6), 3) for i, j in zip(slow[:-1], slow[1:])][:40])
    # what the slow cycles are made of
    for i in slow[:6]:
        ms, me, ms2 = Ms[i], Me[i], Ms[i + 1]
        f = np.nonzero((Fs > me) & (Fs < ms2))[0]
        if len(f):
            j = f[0]
            print(f"  cycle {i}: mover {(me - ms) / 1e3:.1f}, gap A {(Fs[j] - me) / 1e3:.1f}, field "
                  f"{(Fe[j] - Fs[j]) / 1e3:.1f}, gap B {(ms2 - Fe[j]) / 1e3:.1f}")
    spans = (Me - Ms) / 1e3
    print(f"mover spans: median {np.median(spans):.2f} max {spans.max():.2f}")


if __name__ == "__main__":
    main()
