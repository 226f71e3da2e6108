import os, sys, torch
sys.path.insert(0, "/root/repo")
from paper_2604_26074_b200 import dak
M = K = 4096; N = 1; L = 16; kc = 512; h = 0
hbm = [torch.randn((M - h) * K, device="cuda").to(torch.bfloat16) for _ in range(L)]
xs = [torch.randn(N, K, device="cuda").to(torch.bfloat16) * 0.01, torch.zeros(N, K, device="cuda", dtype=torch.bfloat16)]
cfg = dict(pdl=1, congestion_control=1, force_path=2)
ops = [dak.linear_args(None, hbm[i], M, K, h, kc, N, xs[i % 2], xs[(i + 1) % 2], cfg=cfg) for i in range(L)]
ws = torch.zeros(256, dtype=torch.uint8, device="cuda")
for _ in range(4):
    dak.linear_chain(ops, ws, ws.numel())
torch.cuda.synchronize()
