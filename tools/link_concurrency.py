"""Host-link concurrency probe (development experiment): does the copy engine (cudaMemcpyAsync H2D of
pinned memory) add bandwidth on top of the SMs' direct reads of mapped host memory (dak_linear with
every weight row on the host)? Prints GB/s for each alone and for both at once on two streams."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26074_b200 import dak  # noqa: E402

M, K, N = 28672, 7168, 8
h = M
kc = 64
hp, dp = dak.host_alloc(h * K * 2)
x = torch.randn(N, K, device="cuda").to(torch.bfloat16)
y = torch.empty(N, M, device="cuda", dtype=torch.bfloat16)
la = dak.linear_args(dp, None, M, K, h, kc, N, x, y, cfg=dict(pdl=0, congestion_control=1, n_cta_host=16))
CE_BYTES = 256 << 20
src = torch.empty(CE_BYTES, dtype=torch.uint8).pin_memory()
dst = torch.empty(CE_BYTES, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(lin: bool, ce: bool, reps: int = 3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        if lin:
            with torch.cuda.stream(s1):
                dak.linear(la, s1)
        if ce:
            with torch.cuda.stream(s2):
                dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    nb = (h * K * 2 if lin else 0) + (CE_BYTES if ce else 0)
    return dict(linear=lin, copy_engine=ce, ms=round(dt * 1e3, 2), gbs=round(nb / dt / 1e9, 2))


run(True, True, 1)
for lin, ce in ((True, False), (False, True), (True, True)):
    print(json.dumps(run(lin, ce)), flush=True)
dak.host_free(hp)
