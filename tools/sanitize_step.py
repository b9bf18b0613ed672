"""A bounded workload for compute-sanitizer racecheck: the tiny config (BASELINE configs[0])
prefill plus a few eager decode steps (every launch of a step, incl. the scheduler's refills)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("IS_NO_GRAPH", "1")

import torch  # noqa: E402

from oracle import kv as okv  # noqa: E402
from paper_2506_22950_b200 import _lib  # noqa: E402
from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
shape, seed = SHAPES["tiny"], 20261017
w = {k: v.cuda() for k, v in gen_weights(shape, seed=seed).items()}
true = gen_trace("tiny", 8, 32, 1)
budget = okv.prefix_bytes(shape, 16) + 4 * 2 * okv.page_bytes(shape, 16)
ctx = _lib.Context(_lib.make_config(shape, 8, 2, 32, 16, mode="infinite", kv_budget_bytes=budget, seed=seed), w)
ctx.is_prefill(torch.as_tensor(gen_prompt(shape.vocab, 16, 0, seed=seed), device="cuda"), 0)
ctx.is_start_group(true, predict_lengths(true, "noisy", 0.3, seed=1))
for _ in range(steps):
    ctx.is_decode_step()
torch.cuda.synchronize()
print("steps", ctx.is_query()["steps"])
ctx.close()
