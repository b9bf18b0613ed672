"""Minimal driver for profiling: builds the config-3 context, prefills one prompt,
starts the group and runs a few decode steps (graph replay unless IS_NO_GRAPH=1).
Used under ncu (`-s` to skip the prefill launches)."""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2506_22950_b200 import _lib  # noqa: E402
from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="qwen3-1.7b")
ap.add_argument("--G", type=int, default=32)
ap.add_argument("--g", type=int, default=8)
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--time", action="store_true")
args = ap.parse_args()

shape = SHAPES[args.shape]
P, max_new = 256, 1024
w = gen_weights(shape, seed=20261017, device="cuda")
M = int(os.environ.get("GROUPS", "1"))
cfg = _lib.make_config(shape, args.G, args.g, max_new, P, mode="infinite", kv_budget_bytes=0, seed=20261017,
                       max_groups=M)
ctx = _lib.Context(cfg, w)
for m in range(M):
    prompt = torch.as_tensor(gen_prompt(shape.vocab, P, m), device="cuda")
    true = gen_trace("math", args.G, max_new, 1 + m)
    pred = predict_lengths(true, "noisy", 0.3, seed=1 + m)
    ctx.is_prefill(prompt, m, slot=m)
    ctx.is_start_group(true, pred, slot=m)
torch.cuda.synchronize()
for _ in range(args.steps):
    ctx.is_decode_step()
torch.cuda.synchronize()
if args.time:
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        ctx.is_decode_step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    print(f"graph step {dt * 1e3:.3f} ms")
    ms, kind = ctx.is_profile_step()
    names = ["embed/norm", "qkv", "qkv_post", "attn", "o_proj", "gate_up", "down", "lm_head", "refill"]
    for k in range(9):
        print(f"{names[k]:12s} {ms[kind == k].sum():8.4f} ms  n={int((kind == k).sum())}")
    print("eager total", ms.sum())
print(ctx.is_query())
if os.environ.get("IS_TIMELINE"):
    import ctypes
    L = _lib.load()
    L.is_dbg_timeline.argtypes = [ctypes.c_void_p]
    ctx.is_decode_step()
    torch.cuda.synchronize()
    L.is_dbg_timeline(ctx._h)
ctx.close()
