"""Run one dak_linear configuration a few times (for ncu captures): M K N h kc path."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26074_b200 import dak  # noqa: E402

M, K, N, h, kc, path = (int(v) for v in sys.argv[1:7])
w = torch.randn((M - h) * K, device="cuda").to(torch.bfloat16)
hp, dp = dak.host_alloc(max(h * K * 2, 16)) if h else (None, None)
x = torch.randn(N, K, device="cuda").to(torch.bfloat16)
y = torch.empty(N, M, device="cuda", dtype=torch.bfloat16)
a = dak.linear_args(dp, w, M, K, h, kc, N, x, y, cfg=dict(force_path=path, pdl=0))
need = dak.linear_workspace_size(a) if path == 3 else 0
if need:  # split-K workspace (tcgen05 path)
    ws = torch.zeros(need, dtype=torch.uint8, device="cuda")
    a.workspace, a.workspace_bytes = ws.data_ptr(), need
print(dak.linear_query(a))
for _ in range(3):
    dak.linear(a)
torch.cuda.synchronize()
