"""Time persistent-kernel decode steps (config 3 shape) by graph replay; print ms per step and kernel ms."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2506_22950_b200 import _lib
from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths
shape = SHAPES[os.environ.get("SHAPE", "qwen3-1.7b")]
impl = int(os.environ.get("IMPL", "0"))
P, G, g, max_new = 256, 32, 8, 1024
w = gen_weights(shape, seed=20261017, device="cuda")
M = int(os.environ.get("GROUPS", "1"))
cfg = _lib.make_config(shape, G, g, max_new, P, mode="infinite", kv_budget_bytes=0, seed=20261017, decode_impl=impl,
                       max_groups=M)
ctx = _lib.Context(cfg, w)
for m in range(M):
    ctx.is_prefill(torch.as_tensor(gen_prompt(shape.vocab, P, m), device="cuda"), m, slot=m)
    true = gen_trace("math", G, max_new, 1 + m)
    ctx.is_start_group(true, predict_lengths(true, "noisy", 0.3, seed=1 + m), slot=m)
for _ in range(int(os.environ.get("WARM", "20"))):
    ctx.is_decode_step()
torch.cuda.synchronize()
q0 = ctx.is_query()
n = 200
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(ctx.stream if hasattr(ctx, "stream") else torch.cuda.current_stream())
t0 = time.perf_counter()
for _ in range(n):
    ctx.is_decode_step()
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / n
q1 = ctx.is_query()
kn = (q1["layer_kernel_ns"] - q0["layer_kernel_ns"]) / max(q1["layer_kernel_launches"] - q0["layer_kernel_launches"], 1)
print(f"step {dt*1e3:.3f} ms  persistent kernel {kn/1e6:.3f} ms  impl {q1['decode_impl']}")
ms, kind = ctx.is_profile_step()
print("eager per kind:", {int(k): round(float(ms[kind == k].sum()), 4) for k in np.unique(kind)})
ctx.close()
