"""Where the config-3 step's time goes between the two kernels (a build with
both PB_MOVER_TRACE and PB_FF_TRACE): after graph-replayed steps, the last
field launch's CTA timeline and the last mover launch's block starts / warp
ends on one clock (%globaltimer).  The step is field -> mover, so

  gap B = first mover block past griddepcontrol.wait - last field CTA end
  gap A = step - mover span - field span - gap B   (mover end -> field start)

  PB_LIB_PATH=build/v_gaptrace/libpicmc_b200.so python scripts/c3_gap_trace.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2404_10270_b200 import Engine, _lib  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    cfg, _, _ = bench.workload_config("c3", 1, None)
    eng = Engine(cfg, device=dev, init="device", check_every=0)
    eng.sort_by_cell()
    eng.sync()
    eng.prepare_graphs(240)
    eng.replay(20)
    eng.sync()
    for rep in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(eng.stream)
        eng.replay(48)
        b.record(eng.stream)
        torch.cuda.synchronize(dev)
        step = a.elapsed_time(b) / 48 * 1e3
        G = (cfg.grid.nc - 1 + 511) // 512
        words = eng.field_scratch.view(torch.int64).cpu().numpy().view(np.uint64)
        tr = words[-16 * G:].reshape(G, 16)[:, :8].astype(np.int64)
        f0, f1 = tr[:, 0].min(), tr[:, 7].max()
        lib = _lib.load()
        nw, nb = 8192, 2048
        ends = (ctypes.c_ulonglong * nw)()
        starts = (ctypes.c_ulonglong * nb)()
        lib.pb_debug_warp_ends.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
        _lib.check(lib.pb_debug_warp_ends(ends, nw, starts, nb), "pb_debug_warp_ends")
        nblk = torch.cuda.get_device_properties(dev).multi_processor_count * 3
        e = np.array(ends[: nblk * 8], dtype=np.int64)
        s = np.array(starts[:nblk], dtype=np.int64)
        m0, m1 = s.min(), e.max()
        field, mover, gb = (f1 - f0) / 1e3, (m1 - m0) / 1e3, (m0 - f1) / 1e3
        ml = (ctypes.c_ulonglong * 1024)()
        fl = (ctypes.c_ulonglong * 1024)()
        mn, fn = ctypes.c_ulonglong(), ctypes.c_ulonglong()
        lib.pb_debug_mover_log.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        lib.pb_debug_field_log.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        _lib.check(lib.pb_debug_mover_log(ml, ctypes.byref(mn)), "pb_debug_mover_log")
        _lib.check(lib.pb_debug_field_log(fl, ctypes.byref(fn)), "pb_debug_field_log")
        M = np.array(ml, dtype=np.int64).reshape(512, 2)
        F = np.array(fl, dtype=np.int64).reshape(512, 2)
        mi = [(mn.value - 1 - k) % 512 for k in range(40)][::-1]
        fi = [(fn.value - 1 - k) % 512 for k in range(40)][::-1]
        Ms, Me = M[mi, 0], M[mi, 1]
        Fs, Fe = F[fi, 0], F[fi, 1]
        ga = [(fs - Me[Me < fs].max()) / 1e3 for fs in Fs if (Me < fs).any()]
        gbl = [(ms - Fe[Fe < ms].max()) / 1e3 for ms in Ms if (Fe < ms).any()]
        print("  gap A per transition (mover end -> field past wait, us):", " ".join(f"{x:.2f}" for x in ga))
        print("  gap B per transition (field end -> mover past wait, us):", " ".join(f"{x:.2f}" for x in gbl[-12:]))
        print("  mover spans:", " ".join(f"{(e - s) / 1e3:.1f}" for s, e in zip(Ms[-12:], Me[-12:])))
        print("  field spans:", " ".join(f"{(e - s) / 1e3:.2f}" for s, e in zip(Fs[-12:], Fe[-12:])))
        cyc = np.diff(Ms) / 1e3
        print("  mover start-to-start (us):", " ".join(f"{x:.1f}" for x in cyc),
              f"| mean over {len(cyc)}: {cyc.mean():.2f}")
        print(f"rep {rep}: step {step:.2f} us = mover {mover:.2f} + field {field:.2f} + gap B {gb:.2f} "
              f"+ gap A {step - mover - field - gb:.2f}; mover block starts spread {(s.max() - m0) / 1e3:.2f} us; "
              f"field CTA starts spread {(tr[:, 0].max() - f0) / 1e3:.2f} us")


if __name__ == "__main__":
    main()
