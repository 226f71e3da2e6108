"""Per-tile event clocks of one prefill CTA (experiment build with PFT stamps)."""
import os, sys, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26074_b200 import dak  # noqa
B, L, T, Hq, Hkv, d, page = 4, 8192, 2048, 8, 1, 128, 64
pages = L // page
bt, Ph, Pg, ht = dak.kv_place([L] * B, page, pages, 1, 0)
pe = Hkv * page * d
kg = torch.randn(Pg * pe, device="cuda").to(torch.bfloat16); vg = torch.randn_like(kg)
q = torch.randn(B, T, Hq, d, device="cuda").to(torch.bfloat16); out = torch.empty_like(q)
sl = torch.full((B,), L, dtype=torch.int32, device="cuda"); btd = torch.from_numpy(bt).cuda()
args = (q, out, kg, vg, None, None, btd, sl, B, T, Hq, Hkv, d, page, pages)
dak.prefill_attention(*args); torch.cuda.synchronize()
buf = torch.zeros(8 * 4096, dtype=torch.int64, device="cuda")
dak.trace_enable(buf, 8)
dak.prefill_attention(*args); torch.cuda.synchronize()
dak.trace_enable(None, 0)
tr = buf[:4096].cpu().numpy()
ev = tr[2100:2100 + 64 * 16].reshape(64, 16)[:, :12].astype(np.int64)
t0 = ev[0, 0]
names = ["tma", "S_iss", "PV_iss", "vconv", "s_free", "p_full", "sm_beg", "sm_ld", "max", "lazy", "pvwait", "exp"]
print("t " + " ".join(f"{n:>8s}" for n in names))
for t in range(40):
    print(f"{t:2d} " + " ".join(f"{(x - t0) if x else -1:8d}" for x in ev[t]))
d = np.diff(ev[5:40, 5])
print("p_full period median", np.median(d))
