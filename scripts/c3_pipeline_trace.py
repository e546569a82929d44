"""k_field_fused's per-phase timeline INSIDE the config-3 graph-replayed
step (PB_LIB_PATH -> a PB_FF_TRACE build): replays steps, then reads the
trace words of the last launch from the engine's field scratch, and prints
the step time.

  PB_LIB_PATH=build/v_fftrace/libpicmc_b200.so python scripts/c3_pipeline_trace.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2404_10270_b200 import Engine  # noqa: E402

def report(tr_all, names):
    """tr_all: (G, 16) trace words: [0,8) globaltimer ns, [8] smid, [9,16) clock64."""
    import collections
    tr = tr_all[:, :len(names)].astype(np.int64)
    rel = (tr - tr[:, 0].min()) / 1e3
    for k, n in enumerate(names):
        print(f"  {n:12s} median {np.median(rel[:, k]):7.2f}  max {rel[:, k].max():7.2f} us")
    sms = tr_all[:, 8].astype(np.int64)
    per = collections.Counter(sms.tolist())
    print("  CTAs per SM:", dict(collections.Counter(per.values())))
    ck = tr_all[:, 9:16].astype(np.int64)
    dt_ns = (tr[:, 7] - tr[:, 1]).astype(np.float64)
    dck = (ck[:, 6] - ck[:, 0]).astype(np.float64)
    ok = dt_ns > 0
    print("  SM clock over phases 1..7 (MHz, median):", round(float(np.median(dck[ok] / dt_ns[ok] * 1e3)), 1))


NAMES = ["start", "rho+smooth", "aggregate", "grid wait", "prefixes", "tile solve", "phi+E", "clear/end"]


def main():
    dev = torch.device("cuda", 0)
    cfg, _, _ = bench.workload_config("c3", 1, None)
    eng = Engine(cfg, device=dev, init="device", check_every=0)
    eng.sort_by_cell()
    eng.sync()
    eng.prepare_graphs(240)
    eng.replay(20)
    eng.sync()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(eng.stream)
    eng.replay(48)
    b.record(eng.stream)
    torch.cuda.synchronize(dev)
    print(f"step {a.elapsed_time(b) / 48 * 1e3:.2f} us (48 graph-replayed steps, no sort in the window)")
    G = (cfg.grid.nc - 1 + 511) // 512
    words = eng.field_scratch.view(torch.int64).cpu().numpy().view(np.uint64)
    report(words[-16 * G:].reshape(G, 16), NAMES)


if __name__ == "__main__":
    main()
