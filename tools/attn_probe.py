"""Split attention at a mid-rollout decode step (config 3): per-layer time of the layer's
attention launches back to back (is_profile_kernel kind 3).  Under ncu, the launch list
separates the tcgen05 prefix kernel from the suffix kernel.

    python tools/attn_probe.py [steps_before=400]
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import CONFIGS, SEED  # noqa: E402
from paper_2506_22950_b200 import _lib  # noqa: E402
from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths  # noqa: E402

C = CONFIGS[3]
shape = SHAPES[C["shape"]]
G, g, max_new, P = C["G"], C["g"], C["max_new"], C["P"]
kv_tok = 2 * shape.layers * shape.n_kv_heads * shape.head_dim * 2
budget = (P - 1) * kv_tok + g * math.ceil(max_new / 16) * 16 * kv_tok
w = gen_weights(shape, seed=SEED, device="cuda")
cfg = _lib.make_config(shape, G, g, max_new, P, mode="infinite", page_tokens=16, kv_budget_bytes=budget, eps=0.1,
                       temperature=0.8, seed=SEED)
ctx = _lib.Context(cfg, w)
true = gen_trace(C["family"], G, max_new, SEED)
ctx.is_prefill(torch.as_tensor(gen_prompt(shape.vocab, P, 0, seed=SEED), device="cuda"), 0)
ctx.is_start_group(true, predict_lengths(true, "noisy", 0.3, seed=SEED))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
for _ in range(n):
    ctx.is_decode_step()
s0 = ctx.is_query()["suffix_tokens"]
ctx.is_decode_step()
suffix = ctx.is_query()["suffix_tokens"] - s0
reps = int(os.environ.get("REPS", "4"))
ms = ctx.is_profile_kernel(3, reps=reps)[0]
lay = 2 * shape.n_kv_heads * shape.head_dim * 2
b = (P - 1) * lay + suffix * lay
print(json.dumps({"step": n + 1, "suffix_tokens": int(suffix), "layer_us": round(ms * 1e3, 2),
                  "bytes_per_layer": b, "TBs": round(b / (ms * 1e-3) / 1e12, 3)}))
ctx.close()
