"""Run a few persistent decode steps of an L-layer OPT-30B-shaped model (for ncu captures)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26074_b200 import dak  # noqa: E402
from paper_2604_26074_b200.engine import DakOPT, HW, OPTConfig  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 4
eng = DakOPT(OPTConfig(n_layers=layers), 8, 64, HW(hbm_bps=6555.5e9, link_bps=51.5e9), mode=dak.PLAN_BALANCED,
             fused_qkv=False)
eng.enable_persistent_step()
for _ in range(3):
    eng.enqueue_step()
torch.cuda.synchronize()
print("ok")
