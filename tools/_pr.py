import json,sys
for l in sys.stdin:
    d=json.loads(l)
    if "error" in d: print(d); continue
    i=d["info"]; print(d["S"], d["M"], d["K"], d["kc"], round(d["us"],2), round(d["gbs"]), i["grid"], i["stages_hbm"], i["smem_bytes"])
