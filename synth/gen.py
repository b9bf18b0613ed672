"""Seeded generators: weights, prompts, length traces, noisy length predictor.

Recipe (DESIGN.md §"Input recipe"):
  * weights (reading R3 / SURVEY C3): element e of tensor #tid gets
    h = H(H(e) ^ H(tid*0x9E3779B1 + seed)) with the 32-bit integer hash H below,
    u = ((h >> 8) + 0.5) * 2^-24 in fp32, w = (2u - 1) * a in fp32, rounded
    RNE to bf16.  a = 0.02*sqrt(3) (std 0.02) for matrices; norm gains are
    1 + (2u-1)*0.1.  Integer-only hashing => identical bits on CPU and GPU.
  * prompts (R4): token = H(H(pos) ^ H(prompt_id*0x85EBCA6B + seed)) mod vocab.
  * traces: SPEC.md l.47-55 generate_trace: true_len = clamp(round(draw), 1,
    max_len), draw ~ lognormal(mu, sigma) from numpy PCG64(seed).  Families are
    the SURVEY.md §8(d) calibration of PAPER.md Table 1 (l.419-450).
  * predictor: SPEC.md l.56-64 `noisy`: pred = max(1, round(true*(1+e_i))),
    e_i ~ N(0, sigma) seeded by (seed, id); samples with true <= prefix_k keep
    pred = true.  Stand-in for PAPER.md l.365 f_reg(BERT([x; O_1:k])).
"""
import math

import numpy as np
import torch

from .shapes import ModelShape

_M32 = 0xFFFFFFFF
_HMUL = 0x045D9F3B  # < 2^27, so (x * _HMUL) < 2^59 never overflows int64


def _h32(x):
    """32-bit integer avalanche hash on an int64 tensor holding values < 2^32."""
    x = ((x >> 16) ^ x) * _HMUL & _M32
    x = ((x >> 16) ^ x) * _HMUL & _M32
    x = (x >> 16) ^ x
    return x


def _h32_scalar(x):
    return int(_h32(torch.tensor([x & _M32], dtype=torch.int64))[0])


GLOBAL_WEIGHT_NAMES = ["embed", "final_norm"]
LAYER_WEIGHT_NAMES = ["in_norm", "wq", "wk", "wv", "q_norm", "k_norm", "wo",
                      "post_norm", "w_gate", "w_up", "w_down"]


def layer_weight_names(layer):
    return [f"layers.{layer}.{n}" for n in LAYER_WEIGHT_NAMES]


def _weight_shape(s: ModelShape, short):
    H, F = s.hidden, s.ffn
    return {
        "embed": (s.vocab, H), "final_norm": (H,),
        "in_norm": (H,), "wq": (s.q_dim, H), "wk": (s.kv_dim, H),
        "wv": (s.kv_dim, H), "q_norm": (s.head_dim,), "k_norm": (s.head_dim,),
        "wo": (H, s.q_dim), "post_norm": (H,), "w_gate": (F, H),
        "w_up": (F, H), "w_down": (H, F),
    }[short]


def _uniform_bf16(numel, tid, seed, scale, offset, device, chunk=1 << 26):
    out = torch.empty(numel, dtype=torch.bfloat16, device=device)
    salt = _h32_scalar((tid * 0x9E3779B1 + seed) & _M32)
    for start in range(0, numel, chunk):
        n = min(chunk, numel - start)
        e = torch.arange(start, start + n, dtype=torch.int64, device=device)
        h = _h32(_h32(e) ^ salt)
        u = ((h >> 8).to(torch.float32) + 0.5) * (2.0 ** -24)
        w = (u * 2.0 - 1.0) * scale
        if offset != 0.0:
            w = w + offset
        out[start:start + n] = w.to(torch.bfloat16)
    return out


def gen_weights(shape: ModelShape, seed=20261017, device="cpu"):
    """Return an ordered dict name -> bf16 tensor in HF Qwen3 layout ([out, in])."""
    a = 0.02 * math.sqrt(3.0)
    names = list(GLOBAL_WEIGHT_NAMES)
    for l in range(shape.layers):
        names += layer_weight_names(l)
    out = {}
    for tid, name in enumerate(names):
        short = name.split(".")[-1]
        shp = _weight_shape(shape, short)
        numel = int(np.prod(shp))
        if short.endswith("norm"):
            t = _uniform_bf16(numel, tid, seed, 0.1, 1.0, device)
        else:
            t = _uniform_bf16(numel, tid, seed, a, 0.0, device)
        out[name] = t.view(*shp)
    return out


def gen_prompt(vocab, prompt_len, prompt_id, seed=20261017):
    """int32 token ids, uniform in [0, vocab) (reading R4)."""
    salt = _h32_scalar((prompt_id * 0x85EBCA6B + seed) & _M32)
    pos = torch.arange(prompt_len, dtype=torch.int64)
    return (_h32(_h32(pos) ^ salt) % vocab).to(torch.int32).numpy()


# lognormal fits of PAPER.md Table 1 lengths.
TRACE_FAMILIES = {
    "tiny": (2.6, 0.6),
    "gsm8k": (4.796, 1.0),
    "math": (6.337, 0.6),
    "kk": (6.312, 0.6),
    "math8b": (5.835, 0.6),
    "longtail": (5.26, 1.2),
}


def gen_trace(family, count, max_len, seed):
    """SPEC generate_trace: lengths clamp(round(lognormal draw), 1, max_len)."""
    mu, sigma = TRACE_FAMILIES[family] if isinstance(family, str) else family
    rng = np.random.Generator(np.random.PCG64(seed))
    z = rng.standard_normal(count)
    draw = np.exp(mu + sigma * z)
    return np.clip(np.floor(draw + 0.5), 1, max_len).astype(np.int32)


def predict_lengths(true_len, kind="noisy", sigma=0.3, seed=0, prefix_k=0,
                    constant=1):
    """SPEC predict_lengths (oracle / noisy / constant)."""
    true_len = np.asarray(true_len, dtype=np.int64)
    if kind == "oracle":
        pred = true_len.copy()
    elif kind == "constant":
        pred = np.full_like(true_len, constant)
    elif kind == "noisy":
        pred = np.empty_like(true_len)
        for i, t in enumerate(true_len):
            e = np.random.Generator(np.random.PCG64([seed, i])).normal(0.0, sigma)
            pred[i] = max(1, int(math.floor(t * (1.0 + e) + 0.5)))
    else:
        raise ValueError(f"unknown predictor kind {kind!r}")
    short = true_len <= prefix_k
    pred[short] = true_len[short]
    return pred.astype(np.int32)
