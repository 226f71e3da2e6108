"""EXPERIMENT: swapped tcgen05 split-K at the Llama TP8 b64 shapes -- item rows (DAK_EXP_KBLOCK),
split count (DAK_EXP_S) and the memory pipeline alone (DAK_EXP_NOMMA: MMAs skipped)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.bench_linear import time_cfg  # noqa: E402

SHAPES = ((1280, 8192), (8192, 1024), (7168, 8192), (8192, 3584))
CASES = [dict()]
for extra in sys.argv[1:]:
    CASES.append(dict(kv.split("=") for kv in extra.split(",")))
for (M, K) in SHAPES:
    for env in CASES:
        for k in ("DAK_EXP_FLAGS", "DAK_EXP_KBLOCK", "DAK_EXP_S"):
            os.environ.pop(k, None)
        os.environ.update(env)
        try:
            r = time_cfg(M, K, 64, 0, 64, pdl=1, force_path=4, ws=True)
        except Exception as e:  # noqa: BLE001
            r = dict(M=M, K=K, error=str(e))
        r["env"] = env
        print(json.dumps(r), flush=True)
