"""Per-tile event clocks of the first compute CTA of a prefill launch (build patched with
tools/pf_trace_patch.py apply). Events: 0 TMA issued, 1 S(t) committed, 2 PV(t) committed,
3 V(t) converted, 4 softmax waits S(t), 5 S(t) in registers, 6 max done, 7 P buffer wait,
8 exps done, 9 P(t) arrived, 10/11 producer before/after the empty wait, 12 MMA waits s_free
(before S(t + 2)), 13 MMA waits p_full(t)."""
import os, sys
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
ev = buf[2100:2100 + 64 * 16].cpu().numpy().reshape(64, 16)[:, :14].astype(np.int64)
t0 = ev[0, 0]
names = ["tma", "S_done", "PV_iss", "vconv", "smWait", "sLanded", "max", "pvWait", "exps", "p_full", "prodW", "prodGo", "mmaSfr", "mmaPf"]
print("t  " + " ".join(f"{n:>8s}" for n in names))
for t in range(40):
    print(f"{t:2d} " + " ".join(f"{(x - t0) if x else -1:8d}" for x in ev[t]))
print("p_full period median", np.median(np.diff(ev[6:40, 9])))
