"""Run one dak_attention configuration a few times (for ncu captures): B L Hq Hkv chunk_pages r [n_cta_host].

All pages of a request are contiguous in its pool; the oldest round(r * chunks) chunks of every
request live in the host pool. page = 64 tokens, d = 128.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26074_b200 import dak  # noqa: E402

B, L, Hq, Hkv, cp = (int(v) for v in sys.argv[1:6])
r = float(sys.argv[6])
nh_arg = int(sys.argv[7]) if len(sys.argv) > 7 else 0
d, page = 128, 64
pages = -(-L // page)
n_chunks = -(-pages // cp)
hp = min(pages, int(round(r * n_chunks)) * cp)
Ph, Pg = B * hp, B * (pages - hp)
pe = Hkv * page * d
kg = torch.randn(max(Pg, 1) * pe, device="cuda").to(torch.bfloat16)
vg = torch.randn(max(Pg, 1) * pe, device="cuda").to(torch.bfloat16)
kh = dak.host_alloc(max(Ph, 1) * pe * 2)
vh = dak.host_alloc(max(Ph, 1) * pe * 2)
bt = np.zeros((B, pages), np.int64)
ih = ig = 0
for b in range(B):
    for p in range(pages):
        if p < hp:
            bt[b, p] = ih | 0x80000000
            ih += 1
        else:
            bt[b, p] = ig
            ig += 1
btd = torch.from_numpy((bt & 0xFFFFFFFF).astype(np.uint32).view(np.int32)).cuda()
q = torch.randn(B, Hq, d, device="cuda").to(torch.bfloat16)
out = torch.empty_like(q)
sl = torch.full((B,), L, dtype=torch.int32, device="cuda")
host_units = B * (hp // cp) * Hkv
nh = nh_arg or 0  # 0: auto (chosen in-kernel from the block table)
a = dak.attention_args(q, out, kg, vg, kh[1], vh[1], btd, sl, B, Hq, Hkv, d, page, pages, cp,
                       cfg=dict(pdl=1, congestion_control=1, n_cta_host=nh))
ws = torch.zeros(max(dak.attention_workspace_size(a), 16), dtype=torch.uint8, device="cuda")
a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel()
for _ in range(3):
    dak.attention(a)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    dak.attention(a)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / reps
kv = 2 * B * L * Hkv * d * 2
print(dict(B=B, L=L, Hq=Hq, Hkv=Hkv, chunk_pages=cp, host_pages=hp, n_cta_host=nh, us=round(us, 1),
           gbs=round(kv / us / 1e3, 1), host_gbs=round(2 * B * hp * page * Hkv * d * 2 / us / 1e3, 2)))
