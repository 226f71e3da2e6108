"""Cost of the fused pre-norm operand transform on the mma.sync decode path (N = 8): the same
linear with and without ln_w, OPT-30B shapes, the engine's KC (development experiment)."""
import sys, json
sys.path.insert(0, "/root/repo")
from tools.bench_linear import time_cfg
from paper_2604_26074_b200 import dak
for (M, K) in ((28672, 7168), (21504, 7168), (7168, 28672), (7168, 7168)):
    kc = dak.choose_kc(-(-M // 146), K)
    for ln in ((False, True) if K <= 8192 else (False,)):  # fused pre-norm keeps LN weights resident: K <= 8192
        r = time_cfg(M, K, 8, 0, kc, pdl=1, ln=ln)
        print(json.dumps(dict(M=M, K=K, kc=kc, ln=ln, us=round(r["us"], 2), gbs=round(r["gbs"], 1))), flush=True)
