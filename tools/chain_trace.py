"""EXPERIMENT: per-op timeline of one dak_linear_chain launch (dependent C1 chain of 6 ops), from the
launch trace (virtual CTA = cta + grid * op; stamps 0 first stage consumed, 1 producer dependency
released, 2 epilogue start, 3 done)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26074_b200 import dak  # noqa: E402

kc = int(sys.argv[1]) if len(sys.argv) > 1 else 512
L, M, K, N = 6, 4096, 4096, 1
h = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hbm = [torch.randn((M - h) * K, device="cuda").to(torch.bfloat16) for _ in range(L)]
hosts = [dak.host_alloc(max(h * K * 2, 16)) for _ in range(L)]
xs = [torch.randn(N, K, device="cuda").to(torch.bfloat16) * 0.01, torch.zeros(N, K, device="cuda", dtype=torch.bfloat16)]
cfg = dict(pdl=1, congestion_control=1, force_path=2)
ops = [dak.linear_args(hosts[i][1] if h else None, hbm[i], M, K, h, kc, N, xs[i % 2], xs[(i + 1) % 2], cfg=cfg) for i in range(L)]
ws = torch.zeros(256, dtype=torch.uint8, device="cuda")
for _ in range(3):
    dak.linear_chain(ops, ws, ws.numel())
torch.cuda.synchronize()
buf = torch.zeros(4 * 1024 * 4, dtype=torch.int64, device="cuda")
dak.trace_enable(buf, 4)
dak.linear_chain(ops, ws, ws.numel())
torch.cuda.synchronize()
dak.trace_enable(None, 0)
T = buf.view(4, 1024, 4)[0].cpu().numpy().astype(np.float64)
G = dak.device_sms()
t0 = T[:G * L][T[:G * L] > 0].min()
for o in range(L):
    st = T[G * o:G * (o + 1)]
    def q(k):
        v = st[:, k][st[:, k] > 0]
        return [round((np.min(v) - t0) / 1e3, 2), round((np.median(v) - t0) / 1e3, 2), round((np.max(v) - t0) / 1e3, 2)] if len(v) else None
    print(json.dumps(dict(op=o, first_stage=q(0), dep_release=q(1), epilogue=q(2), done=q(3))))
