"""Per-GEMM split-K / ring-depth sweep on one B200 (config 3 shapes).

For every setting (env knobs read at context creation) it reports the back-to-back
launch time of each decode GEMM kind (is_profile_kernel: all layers' launches as the
step issues them, CUDA events around the graph) and the graph-replayed decode step
time (64 steps early in a rollout).

    python tools/kernel_sweep.py > gpurun_out/ksweep.jsonl
"""
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import CONFIGS, SEED  # noqa: E402
from paper_2506_22950_b200 import _lib  # noqa: E402
from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths  # noqa: E402

C = CONFIGS[3]
shape = SHAPES[C["shape"]]
G, g, max_new, P = C["G"], C["g"], C["max_new"], C["P"]
kv_tok = 2 * shape.layers * shape.n_kv_heads * shape.head_dim * 2
budget = (P - 1) * kv_tok + g * math.ceil(max_new / 16) * 16 * kv_tok
H, F = shape.hidden, shape.ffn
BYTES = {1: (shape.q_dim + 2 * shape.kv_dim) * H * 2, 4: H * shape.q_dim * 2, 5: 2 * F * H * 2, 6: H * F * 2}
NAMES = {1: "qkv", 4: "o", 5: "gu", 6: "down"}
w = gen_weights(shape, seed=SEED, device="cuda")
prompt = torch.as_tensor(gen_prompt(shape.vocab, P, 0, seed=SEED), device="cuda")
true = gen_trace(C["family"], G, max_new, SEED)
pred = predict_lengths(true, "noisy", 0.3, seed=SEED)

SETTINGS = [s for s in os.environ.get("SWEEP", "").split(";") if s] or [
    "", "IS_SPLIT_GU=1", "IS_SPLIT_GU=3", "IS_SPLIT_GU=4", "IS_STG_GU=6", "IS_STG_GU=8",
    "IS_SPLIT_D=4", "IS_STG_D=6", "IS_STG_D=8", "IS_SPLIT_O=4", "IS_STG_O=6", "IS_SPLIT_QKV=2", "IS_STG_QKV=6",
]
KNOBS = ["IS_STREAMK_GU", "IS_STG_LM", "IS_SPLIT_GU", "IS_SPLIT_D", "IS_SPLIT_O", "IS_SPLIT_QKV", "IS_STG_GU", "IS_STG_D", "IS_STG_O",
         "IS_STG_QKV"]
for setting in SETTINGS:
    for k in KNOBS:
        os.environ.pop(k, None)
    for kv in setting.split(","):
        if kv:
            k, v = kv.split("=")
            os.environ[k] = v
    top_p = float(os.environ.pop("TOP_P", "1.0"))   # (a make_config field, not an env knob)
    cfg = _lib.make_config(shape, G, g, max_new, P, mode="infinite", page_tokens=16, kv_budget_bytes=budget,
                           eps=0.1, temperature=0.8, seed=SEED, top_p=top_p)
    ctx = _lib.Context(cfg, w)
    ctx.is_prefill(prompt, 0)
    ctx.is_start_group(true, pred)
    for _ in range(8):
        ctx.is_decode_step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(64):
        ctx.is_decode_step()
    e1.record()
    torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1) / 64
    out = {"setting": setting or "default", "step_ms": round(step_ms, 4)}
    for kind in (1, 4, 5, 6):
        ms = float(np.median([ctx.is_profile_kernel(kind, reps=4)[0] for _ in range(3)]))
        out[NAMES[kind] + "_us"] = round(ms * 1e3, 2)
        out[NAMES[kind] + "_TBs"] = round(BYTES[kind] / (ms * 1e-3) / 1e12, 3)
    ctx.close()
    print(json.dumps(out), flush=True)
