"""C1 (4096 x 4096 GEMV, N = 1) per-launch time over the ring depth and KC (development experiment):
smaller SMEM footprints would let two CTAs share an SM so that chained launches overlap (PDL).
Result (profiles/r01/sweeps.txt): none beat the default (kc 512, 5 stages, 7.1 us per launch)."""
import sys, os, json
sys.path.insert(0, "/root/repo")
from tools.bench_linear import time_cfg
M = K = 4096
for h in (0, 32):
    for kc in (512, 256, 128):
        for st in (0, 2, 3, 4, 6):
            try:
                r = time_cfg(M, K, 1, h, kc, launches=64, reps=5, pdl=1, n_cta_host=0, congestion_control=1, stages=st)
            except Exception as e:
                print(h, kc, st, "ERR", str(e)[:80]); continue
            i = r["info"]
            print(json.dumps(dict(h=h, kc=kc, stages=st, us=round(r["us"], 2), gbs=round(r["hbm_gbs"] + r["host_gbs"], 1),
                                  smem=i["smem_bytes"], st_hbm=i["stages_hbm"], path=i["path"])), flush=True)
