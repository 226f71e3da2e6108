"""Launch a few dak_linear configs with plain stream launches (for ncu; not a timing tool)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26074_b200 import dak
from tools.bench_linear import setup

cfgs = [(4096, 4096, 1, 32), (28672, 7168, 8, 192), (28672, 7168, 1, 0), (7168, 7168, 8, 48)]
sel = [int(a) for a in sys.argv[1:]] or range(len(cfgs))
for i in sel:
    M, K, N, h = cfgs[i]
    kc = dak.default_kc(M, K, 147)
    hbm, hosts, x, y = setup(M, K, N, h, kc, 4)
    for it in range(8):
        a = dak.linear_args(hosts[it % 4][1] if h else None, hbm[it % 4], M, K, h, kc, N, x, y)
        dak.linear(a)
    torch.cuda.synchronize()
print("done")
