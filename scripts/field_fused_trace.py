"""Per-phase timeline of k_field_fused (build with EXTRA=-DPB_FF_TRACE into
build/v_fftrace/): runs pb_field_cycle on synthetic bins and prints, per
phase boundary, the median / max over CTAs of the time since the earliest
CTA start (us).

  python scripts/field_fused_trace.py build/v_fftrace/libpicmc_b200.so [nc] [bc]
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["PB_LIB_PATH"] = os.path.abspath(sys.argv[1])
from paper_2404_10270_b200 import _lib  # noqa: E402
from paper_2404_10270_b200.store import status_template  # noqa: E402

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
    nc = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
    bc = _lib.PB_FIELD_PERIODIC if (len(sys.argv) > 3 and sys.argv[3] == "periodic") else _lib.PB_FIELD_DIRICHLET
    lib = _lib.load()
    dev = torch.device("cuda", 0)
    ndep = 2
    rng = np.random.default_rng(1)
    C = rng.integers(0, 300, size=(ndep, nc)).astype(np.uint64)
    R = (rng.random((ndep, nc)) * C * 2.0 ** 48).astype(np.uint64)
    bins = torch.from_numpy(np.stack([R, C], 1).reshape(-1).view(np.int64)).to(dev)
    t = lambda n: torch.zeros(n, dtype=torch.float64, device=dev)  # noqa: E731
    rho, rho_s, phi, e, left, right = t(nc + 1), t(nc + 1), t(nc + 1), t(nc + 1), t(nc), t(nc)
    nbytes = lib.pb_field_scratch_bytes(nc)
    scr = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    st = status_template(dev)
    c = (ctypes.c_double * ndep)(-1e-9, 1e-9)
    G = (nc + 511) // 512
    P = lambda x: x.data_ptr()  # noqa: E731
    sh = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    runs = []
    for it in range(30):
        b = bins.clone()
        _lib.check(lib.pb_field_cycle(P(b), c, ndep, nc, bc, 1, 1e-5, 8.85e-12, 0.0, 0.0, P(left), P(right),
                                      P(rho), P(rho_s), P(phi), P(e), P(b), None, b.numel(), P(st), P(scr), None, 0,
                                      None, 0, sh),
                   "pb_field_cycle")
        torch.cuda.synchronize()
        words = scr.view(torch.int64).cpu().numpy().view(np.uint64)
        last = words[-16 * G:].reshape(G, 16)
        runs.append(last[:, :len(NAMES)].astype(np.int64))
    print(f"nc={nc} G={G} bc={'periodic' if bc == _lib.PB_FIELD_PERIODIC else 'dirichlet'}  (last of 30 calls)")
    report(last, NAMES)
    tot = [((r[:, 7].max() - r[:, 0].min()) / 1e3) for r in runs[5:]]
    print("  span (us) median over calls:", round(float(np.median(tot)), 2))


if __name__ == "__main__":
    main()
