import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from test_engine_gpu import _mk_config
from oracle import oracle
from paper_2404_10270_b200 import Engine
dev = torch.device('cuda', 0)
for fs in (False, True):
    res = {}
    for se in (0, 3):
        cfg = _mk_config(nc=500, ppc0=40, sort_every=se, field_solve=fs, smoothing_passes=1)
        eng = Engine(cfg, device=dev, check_every=0)
        h = []
        for k in range(8):
            rho, e = eng.step()
            d = eng.download()
            h.append((rho.cpu().numpy().copy(), e.cpu().numpy().copy(), [oracle.canonical(f.cell, f.fields()) for f in d]))
        res[se] = h
    for k in range(8):
        a, b = res[0][k], res[3][k]
        print('fs', fs, 'step', k + 1, 'rho eq', np.array_equal(a[0].view(np.uint64), b[0].view(np.uint64)),
              'e eq', np.array_equal(a[1].view(np.uint64), b[1].view(np.uint64)),
              'parts eq', [np.array_equal(x, y) for x, y in zip(a[2], b[2])])
