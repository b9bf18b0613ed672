"""Capture one decode step's per-CTA timeline of the persistent decode kernel
(config 3 shape) and save it: python tools/mk_trace.py OUT.npz [--steps N]."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("IS_MK_TRACE", "1536")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_22950_b200 import _lib  # noqa: E402
from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("out")
ap.add_argument("--steps", type=int, default=64)
ap.add_argument("--shape", default="qwen3-1.7b")
args = ap.parse_args()
shape = SHAPES[args.shape]
P, G, g, max_new = 256, 32, 8, 1024
w = gen_weights(shape, seed=20261017, device="cuda")
cfg = _lib.make_config(shape, G, g, max_new, P, mode="infinite", kv_budget_bytes=0, seed=20261017, decode_impl=0)
ctx = _lib.Context(cfg, w)
ctx.is_prefill(torch.as_tensor(gen_prompt(shape.vocab, P, 0), device="cuda"), 0)
true = gen_trace("math", G, max_new, 1)
ctx.is_start_group(true, predict_lengths(true, "noisy", 0.3, seed=1))
for _ in range(args.steps):
    ctx.is_decode_step()
torch.cuda.synchronize()
tasks, off, trace = ctx.is_dbg_mk_trace()
np.savez_compressed(args.out, tasks=tasks, off=off, trace=trace)
print("saved", args.out, trace.shape)
