"""Oracle: Qwen3-shaped decoder, full causal recompute, fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §2.1 l.106-112: "each new token requires a forward pass through all
transformer layers, where the current token attends to both cached and current
representations".  The oracle does the plain thing the KV cache accelerates:
for every generated token it runs one complete causal forward over
[prompt; generated-so-far] from scratch -- no cache, no prefix sharing, no
split (BASELINE.json north_star: "decodes each completion independently with
full recomputed attention").  Arithmetic is fp64.

Architecture = Qwen3 (shapes: DESIGN.md R1): pre-RMSNorm
blocks, per-head RMSNorm on q and k, rotate-half RoPE (theta 1e6), GQA
(q head h reads kv head h // (Hq/Hkv)), SwiGLU MLP, tied lm_head, no biases.

`mirror=True` rounds to bf16 exactly where the GPU path stores bf16
(reading R12): r1 the operand of every GEMM that follows an RMSNorm,
which is x*gain, the 1/rms row scale applied to the GEMM's product (R12b:
RMSNorm(x) W^T = rs * ((x*gain) W^T), rs = 1/sqrt(mean(x^2) + eps)),
r2 q/k/v after QK-norm + RoPE (what the KV cache holds), r4 attention output,
r5 SiLU(gate)*up.  `mirror=False` is the pure fp64 model (pinned against the
HF transformers Qwen3 implementation in tests/test_oracle_model.py).

Sampling (Eq. 1 l.120-125, T = 0.8 l.382) uses oracle.sampler on the
fp32-cast logits.
"""
import numpy as np
import torch

from . import sampler


def round_bf16(x):
    """fp64 -> fp32 (RNE) -> bf16 (RNE) -> fp64."""
    x32 = np.ascontiguousarray(x, dtype=np.float32)
    b = x32.view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


def rmsnorm(x, gain, eps):
    """x / sqrt(mean(x^2) + eps) * gain over the last axis."""
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * gain


def rms_scale(x, eps):
    """rs = 1 / sqrt(mean(x^2) + eps) per row (the RMSNorm scale), shape [..., 1]."""
    return 1.0 / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps)


def rope_cos_sin(positions, head_dim, theta):
    half = head_dim // 2
    inv_freq = theta ** (-np.arange(half, dtype=np.float64) * 2.0 / head_dim)
    ang = np.asarray(positions, dtype=np.float64)[:, None] * inv_freq[None, :]
    return np.cos(ang), np.sin(ang)


def rope(x, cos, sin):
    """Rotate-half RoPE. x: [n, heads, d]; cos/sin: [n, d/2]."""
    h = x.shape[-1] // 2
    x1, x2 = x[..., :h], x[..., h:]
    c, s = cos[:, None, :], sin[:, None, :]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def silu(x):
    return x / (1.0 + np.exp(-x))


def _f64(t):
    if isinstance(t, torch.Tensor):
        return t.detach().to("cpu", torch.float64).numpy()
    return np.asarray(t, dtype=np.float64)


def causal_attention(q, k, v, n_rep):
    """q: [n, Hq, d], k/v: [n, Hkv, d] -> [n, Hq, d]; row i sees keys 0..i."""
    n, Hq, d = q.shape
    out = np.empty_like(q)
    mask = np.triu(np.ones((n, n), dtype=bool), 1)
    for h in range(Hq):
        kh = k[:, h // n_rep, :]
        vh = v[:, h // n_rep, :]
        s = (q[:, h, :] @ kh.T) / np.sqrt(d)
        s[mask] = -np.inf
        s = s - s.max(axis=1, keepdims=True)
        p = np.exp(s)
        out[:, h, :] = (p @ vh) / p.sum(axis=1, keepdims=True)
    return out


def forward(weights, shape, tokens, mirror=True, logit_rows=None, trace=None):
    """Causal forward over `tokens` (positions 0..n-1).

    Returns fp64 logits [len(logit_rows), vocab] (all rows by default).
    `trace` (dict) optionally collects per-layer intermediates for kernel tests.
    """
    S = shape
    rb = round_bf16 if mirror else (lambda a: a)
    tokens = np.asarray(tokens, dtype=np.int64)
    n = len(tokens)
    E = weights["embed"]
    x = _f64(E[torch.as_tensor(tokens)])
    cos, sin = rope_cos_sin(np.arange(n), S.head_dim, S.rope_theta)
    rep = S.n_q_heads // S.n_kv_heads
    for l in range(S.layers):
        w = {k.split(".")[-1]: v for k, v in weights.items() if k.startswith(f"layers.{l}.")}
        # RMSNorm(x) W^T = rs * ((x * gain) W^T) (R12b; equal in exact arithmetic)
        rs, h = rms_scale(x, S.rms_eps), rb(x * _f64(w["in_norm"]))
        q = (rs * (h @ _f64(w["wq"]).T)).reshape(n, S.n_q_heads, S.head_dim)
        k = (rs * (h @ _f64(w["wk"]).T)).reshape(n, S.n_kv_heads, S.head_dim)
        v = (rs * (h @ _f64(w["wv"]).T)).reshape(n, S.n_kv_heads, S.head_dim)
        q = rmsnorm(q, _f64(w["q_norm"]), S.rms_eps)
        k = rmsnorm(k, _f64(w["k_norm"]), S.rms_eps)
        q, k, v = rb(rope(q, cos, sin)), rb(rope(k, cos, sin)), rb(v)
        a = rb(causal_attention(q, k, v, rep).reshape(n, S.q_dim))
        if trace is not None:
            trace[f"{l}.q"], trace[f"{l}.k"], trace[f"{l}.v"], trace[f"{l}.attn"] = q, k, v, a
        x = x + a @ _f64(w["wo"]).T
        rs2, h2 = rms_scale(x, S.rms_eps), rb(x * _f64(w["post_norm"]))
        act = rb(silu(rs2 * (h2 @ _f64(w["w_gate"]).T)) * (rs2 * (h2 @ _f64(w["w_up"]).T)))
        x = x + act @ _f64(w["w_down"]).T
        if trace is not None:
            trace[f"{l}.resid"] = x.copy()
    rows = np.arange(n) if logit_rows is None else np.asarray(logit_rows)
    xr = x[rows]
    return rms_scale(xr, S.rms_eps) * (rb(xr * _f64(weights["final_norm"])) @ _f64(E).T)


def generate(weights, shape, prompt, uid, true_len, seed, T=0.8, mirror=True):
    """Autoregressive completion of one sample by full recompute per token.

    Step t feeds the sequence [prompt; gen[0..t-1]] and samples gen[t] from the
    logits at its last position (R6/R7: the last prompt token is the
    step-0 input at position P-1).  Trace-driven termination (R5): exactly
    true_len tokens.
    """
    seq = [int(t) for t in prompt]
    out = []
    for t in range(true_len):
        z = forward(weights, shape, seq, mirror=mirror, logit_rows=[len(seq) - 1])[0]
        tok = sampler.sample_token(z.astype(np.float32), seed, uid, t, T)
        out.append(tok)
        seq.append(tok)
    return out


def teacher_forced_logits(weights, shape, prompt, gen_tokens, mirror=True, rows=None):
    """Logits predicting gen[t] for t in `rows` (default all), given gen[:t].

    One causal forward over [prompt; gen[:-1]] yields every position at once;
    the logits at index P-1+t predict gen[t].
    """
    P = len(prompt)
    ts = np.arange(len(gen_tokens)) if rows is None else np.asarray(rows)
    seq = [int(x) for x in prompt] + [int(x) for x in gen_tokens[:int(ts.max())]]
    return forward(weights, shape, seq, mirror=mirror, logit_rows=P - 1 + ts)
