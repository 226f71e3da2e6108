import sys, json
sys.path.insert(0, "/root/repo")
from tools.bench_linear import time_cfg
for kc in (512, 1024, 2048):
    for st in (0, 3, 4):
        try:
            r = time_cfg(4096, 4096, 1, 0, kc, launches=64, reps=5, pdl=1, stages=st)
            print(json.dumps(dict(kc=kc, stages=st, us=round(r["us"], 2), gbs=round(r["gbs"], 1), st_hbm=r["info"]["stages_hbm"], smem=r["info"]["smem_bytes"])), flush=True)
        except Exception as e:
            print(kc, st, "ERR", str(e)[:100])
