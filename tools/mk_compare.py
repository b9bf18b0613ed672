"""Compare internal buffers of the two decode implementations after one decode step."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2506_22950_b200 import _lib
from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths

name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
layers = int(sys.argv[2]) if len(sys.argv) > 2 else 0
shape = SHAPES[name]
if layers:
    import dataclasses
    shape = dataclasses.replace(shape, layers=layers)
SEED = 20261017
P = 16 if name == "tiny" else 256
w = gen_weights(shape, seed=SEED)
wd = {k: v.cuda() for k, v in w.items()}
prompt = gen_prompt(shape.vocab, P, 0, seed=SEED)
true = gen_trace("tiny", 8, 32, 1)
pred = predict_lengths(true, "noisy", 0.3, seed=1)


def bf16(u8):
    return (u8.view(np.uint16).astype(np.uint32) << 16).view(np.float32)


def unsw(u8, BN, K):
    x = bf16(u8).reshape(K // 64, BN, 64)
    out = np.zeros((BN, K), np.float32)
    for kb in range(K // 64):
        for n in range(BN):
            for c in range(8):
                out[n, kb * 64 + c * 8: kb * 64 + c * 8 + 8] = x[kb, n, ((c ^ (n & 7)) * 8):((c ^ (n & 7)) * 8) + 8]
    return out


res = {}
for impl in (1, 0):
    cfg = _lib.make_config(shape, 8, 2, 32, P, mode="naive", seed=SEED, decode_impl=impl)
    ctx = _lib.Context(cfg, wd)
    ctx.is_prefill(torch.as_tensor(prompt, device="cuda"), 0)
    ctx.is_start_group(true, pred)
    ctx.is_decode_step()
    torch.cuda.synchronize()
    H, Hq, F = shape.hidden, shape.n_q_heads, shape.ffn
    rc = 16
    r = {}
    r["q"] = bf16(ctx.is_dbg_copy(0, rc * Hq * 128 * 2)).reshape(rc, -1)
    r["resid"] = ctx.is_dbg_copy(1, rc * H * 4).view(np.float32).reshape(rc, H)
    r["xn"] = bf16(ctx.is_dbg_copy(3, rc * H * 2)).reshape(rc, H)
    if impl == 1:
        r["attn"] = bf16(ctx.is_dbg_copy(4, rc * Hq * 128 * 2)).reshape(rc, -1)
        r["act"] = bf16(ctx.is_dbg_copy(6, rc * F * 2)).reshape(rc, F)
    else:
        r["attn"] = unsw(ctx.is_dbg_copy(5, 16 * Hq * 128 * 2), 16, Hq * 128)
        r["act"] = unsw(ctx.is_dbg_copy(7, 16 * F * 2), 16, F)
    res[impl] = r
    ctx.close()
for k in res[1]:
    a, b = res[1][k][:2], res[0][k][:2]
    print(k, "rel", np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-30), "maxabs", np.abs(a - b).max(),
          "row0 per-op", a[0, :4], "mega", b[0, :4])
