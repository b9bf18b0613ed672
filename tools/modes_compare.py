"""Decode steps, tokens/s and peak KV of the sampling-loop policies on one B200
(the paper's Table 1 comparison at fixed micro-group size; SURVEY.md §8d
"expected schedule outcomes").  Every mode decodes the same completions (same
prompts, same trace lengths, RNG keyed by uid), so tokens are identical and
only the schedule differs.

    python tools/modes_compare.py --config 3 --prompts 2 > out.json
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CONFIGS, SEED  # noqa: E402
from paper_2506_22950_b200 import _lib  # noqa: E402
from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--prompts", type=int, default=2)
ap.add_argument("--modes", default="naive,fifo,fptas_only,sjf_only,infinite,full,dynamic")
args = ap.parse_args()
C = CONFIGS[args.config]
shape = SHAPES[C["shape"]]
G, g, max_new, P, k = C["G"], C["g"], C["max_new"], C["P"], C["prefix_k"]
kv_tok = 2 * shape.layers * shape.n_kv_heads * shape.head_dim * 2
budget = (P - 1) * kv_tok + g * math.ceil(max_new / 16) * 16 * kv_tok
if k:
    budget = 1 << 30
w = gen_weights(shape, seed=SEED, device="cuda")
out = {"config": args.config, "desc": C["desc"], "prompts": args.prompts, "kv_budget_bytes": budget, "modes": {}}
tokens_ref = {}
for mode in args.modes.split(","):
    full = mode == "full"
    dyn = mode == "dynamic"   # R35: 2G candidates (the trace, then a second draw), stop at G completions
    cfg = _lib.make_config(shape, 2 * G if dyn else G, g, max_new, P, mode=mode,
                           prefix_k=k if mode == "infinite" else 0,
                           kv_budget_bytes=0 if full else budget, seed=SEED, dynamic_target=G if dyn else 0)
    ctx = _lib.Context(cfg, w)
    steps, toks, peak, dt = 0, 0, 0, 0.0
    emitted, discarded = [], 0
    same = True
    for pid in range(args.prompts):
        prompt = torch.as_tensor(gen_prompt(shape.vocab, P, pid, seed=SEED), device="cuda")
        true = gen_trace(C["family"], G, max_new, SEED + pid)
        if dyn:
            true = np.concatenate([true, gen_trace(C["family"], G, max_new, SEED + pid + 1000)])
        pred = predict_lengths(true, "noisy", 0.3, seed=SEED + pid, prefix_k=k if mode == "infinite" else 0)
        ctx.is_prefill(prompt, pid)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.is_start_group(true, pred)
        steps += ctx.is_run_group()
        torch.cuda.synchronize()
        dt += time.perf_counter() - t0
        st = ctx.is_query()
        assert st["completed"] == G and st["error"] == 0, st
        toks += int(st["tokens_decoded"])
        peak = max(peak, st["peak_kv_bytes"])
        tk = ctx.is_copy_tokens()
        done = [u for u in range(len(true)) if tk[u, true[u] - 1] >= 0]
        emitted += [int(true[u]) for u in done]
        discarded += st["discarded"]
        if dyn:
            pass                                  # 2G candidate rows: not comparable row for row
        elif pid in tokens_ref:
            same = same and bool(np.array_equal(tk, tokens_ref[pid]))
        else:
            tokens_ref[pid] = tk
    ctx.close()
    out["modes"][mode] = {"decode_steps": steps, "tokens": toks, "tokens_per_s": round(toks / dt, 1),
                          "ms_per_step": round(dt / steps * 1e3, 4), "peak_kv_gb": round(peak / 1e9, 4),
                          "within_budget": bool(full or peak <= budget), "tokens_identical_to_first_mode": same,
                          "avg_emitted_len": round(float(np.mean(emitted)), 2), "discarded": discarded}
print(json.dumps(out))
