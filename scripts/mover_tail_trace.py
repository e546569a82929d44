"""Tail of the persistent mover (a PB_MOVER_TRACE build): after graph-replayed
steps of a workload, every warp's finish time relative to the launch's first
block start -- how long the HBM stream runs down while the last claimed
chunks finish.

  PB_LIB_PATH=build/v_movertrace/libpicmc_b200.so python scripts/mover_tail_trace.py c3
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
    wl = sys.argv[1] if len(sys.argv) > 1 else "c3"
    dev = torch.device("cuda", 0)
    cfg, _, _ = bench.workload_config(wl, 1, 100 if wl == "c2" else None)
    eng = Engine(cfg, device=dev, init="device", check_every=0)
    eng.sort_by_cell()
    eng.sync()
    eng.prepare_graphs(60)
    eng.replay(20)
    eng.sync()
    lib = _lib.load()
    nw, nb = 8192, 2048
    ends = (ctypes.c_ulonglong * nw)()
    starts = (ctypes.c_ulonglong * nb)()
    lib.pb_debug_warp_ends.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int]
    _lib.check(lib.pb_debug_warp_ends(ends, nw, starts, nb), "pb_debug_warp_ends")
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    nblk = sms * 3
    e = np.array(ends[: nblk * 8], dtype=np.int64)
    s = np.array(starts[:nblk], dtype=np.int64)
    t0 = s.min()
    rel = (e - t0) / 1e3
    st = (s - t0) / 1e3
    print(f"{wl}: {nblk} blocks x 8 warps; block starts spread {st.max():.2f} us")
    for q in (0, 10, 50, 90, 99, 100):
        print(f"  warp finish p{q:<3d} {np.percentile(rel, q):8.2f} us")
    span = rel.max()
    # area lost to the tail: fraction of warp-time idle between each warp's end and the last end
    idle = np.mean(span - rel) / span
    print(f"  kernel span {span:.2f} us; mean warp idle at the end {np.mean(span - rel):.2f} us ({100 * idle:.1f}%)")


if __name__ == "__main__":
    main()
