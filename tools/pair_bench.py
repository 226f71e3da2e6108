"""Compute-bound large-N GEMM: the CTA-pair GEMM (cta_group::2, auto at h = 0)
vs the one-CTA tcgen05 forms (force_path = 3), 7168 x 7168 weights, N in {256 .. 4096}, r = 0;
TFLOP/s over chained launches (CUDA graph, weight copies rotated past L2). One JSON line per point.

  python tools/pair_bench.py [M] [K]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.bench_linear import time_cfg  # noqa: E402


def main():
    M = int(sys.argv[1]) if len(sys.argv) > 1 else 7168
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 7168
    for N in (256, 512, 1024, 2048, 4096):
        for name, cfg in (("pair", dict(force_path=5)), ("one_cta", dict(force_path=3))):
            try:
                r = time_cfg(M, K, N, 0, 64, launches=16, reps=5, ws=True, pdl=1, **cfg)
            except Exception as e:  # noqa: BLE001
                print(json.dumps(dict(M=M, K=K, N=N, kernel=name, error=str(e)[:120])), flush=True)
                continue
            tf = 2.0 * M * K * N / (r["us"] * 1e-6) / 1e12
            print(json.dumps(dict(M=M, K=K, N=N, kernel=name, us=round(r["us"], 1), tflops=round(tf, 1),
                                  grid=r["info"]["grid"], ws=r["info"]["ws"])), flush=True)


if __name__ == "__main__":
    main()
