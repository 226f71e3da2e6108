"""Full-size parity: the bench's OPT-30B decode path (BASELINE configs[1]) at the model's real layer
shapes (hidden 7168, 56 heads, ffn 28672, vocab 50272), batch 8, context 64, in bench.py's launch
configuration (BALANCED per-op host ratios, fused pre-norm, fused [q;k;v], PDL, CUDA graph), with
2 of the 48 layers so the float64 oracle (oracle/layer.py opt_decode_step) finishes in seconds.
The BALANCED plan is per op (each op at its own balance point), so every linear has the same
host/HBM split as in the 48-layer bench step.

Tolerance as the engine tests: 3e-2 of max(|ref|, rms(ref))."""
import numpy as np
import pytest

import synth
from oracle import kernels as Kx
from oracle import layer as Ly
from tests.test_oracle_layer import make_params

pytestmark = pytest.mark.gpu


def test_opt30b_full_shapes_bench_config_matches_oracle():
    import torch
    from paper_2604_26074_b200 import dak
    from paper_2604_26074_b200.engine import DakOPT, HW, OPT_30B
    from dataclasses import replace
    from tests.test_gpu_engine import _engine_weights
    L, B, ctx = 2, 8, 64
    c = OPT_30B
    g = np.random.default_rng(0xDA0 + 2)
    p = make_params(g, L, c.hidden, c.ffn, c.vocab, c.max_pos)
    cfg = replace(OPT_30B, n_layers=L)
    hw = HW(hbm_bps=6771.5e9, link_bps=45.77e9)  # the bench's planner rates
    eng = DakOPT(cfg, B, ctx, hw, mode=dak.PLAN_BALANCED, weights=_engine_weights(p, L, torch))
    assert sum(op.h for op in eng.linear_ops()) > 0  # weights really split
    Kc = [[synth.normal_bf16(g, (ctx - 1, c.n_kv_heads, c.head_dim)) for _ in range(B)] for _ in range(L)]
    Vc = [[synth.normal_bf16(g, (ctx - 1, c.n_kv_heads, c.head_dim)) for _ in range(B)] for _ in range(L)]
    eng.load_kv(Kc, Vc)
    tokens = (np.arange(B) * 6151 + 17) % c.vocab
    eng.tokens.copy_(torch.from_numpy(tokens.astype(np.int32)))
    s = torch.cuda.Stream()
    eng.capture(s)
    eng.graph.replay()
    torch.cuda.synchronize()
    got = Kx.bf16_to_f64(eng.logits.view(torch.int16).cpu().numpy().view(np.uint16))
    eng.close()
    ref, _ = Ly.opt_decode_step(tokens, np.full(B, ctx - 1), p, Kc, Vc, c.n_heads)
    from tests.gpu_util import assert_close
    assert_close(got, ref, rtol=3e-2)
