"""Pins for oracle/model.py and oracle/attention.py.

The fp64 model (mirror=False) is pinned against an independent library
implementation of the same architecture (HF transformers Qwen3, run in
float64 on CPU with our weights); the split attention against full attention
(exact in real arithmetic); plus closed-form special cases.
"""
import dataclasses

import numpy as np
import pytest
import torch

from oracle import attention as A
from oracle import model as M
from synth import SHAPES, gen_prompt, gen_weights


def _hf_logits(shape, weights, tokens):
    from transformers import Qwen3Config, Qwen3ForCausalLM
    cfg = Qwen3Config(
        vocab_size=shape.vocab, hidden_size=shape.hidden,
        intermediate_size=shape.ffn, num_hidden_layers=shape.layers,
        num_attention_heads=shape.n_q_heads, num_key_value_heads=shape.n_kv_heads,
        head_dim=shape.head_dim, rms_norm_eps=shape.rms_eps, rope_theta=shape.rope_theta,
        tie_word_embeddings=True, max_position_embeddings=4096, attention_bias=False,
        torch_dtype=torch.float64)
    cfg._attn_implementation = "eager"
    m = Qwen3ForCausalLM(cfg).to(torch.float64).eval()
    sd = {"model.embed_tokens.weight": weights["embed"], "model.norm.weight": weights["final_norm"]}
    names = {"in_norm": "input_layernorm.weight", "wq": "self_attn.q_proj.weight",
             "wk": "self_attn.k_proj.weight", "wv": "self_attn.v_proj.weight",
             "q_norm": "self_attn.q_norm.weight", "k_norm": "self_attn.k_norm.weight",
             "wo": "self_attn.o_proj.weight", "post_norm": "post_attention_layernorm.weight",
             "w_gate": "mlp.gate_proj.weight", "w_up": "mlp.up_proj.weight",
             "w_down": "mlp.down_proj.weight"}
    for k, v in weights.items():
        if k.startswith("layers."):
            _, l, short = k.split(".")
            sd[f"model.layers.{l}.{names[short]}"] = v
    sd = {k: v.to(torch.float64) for k, v in sd.items()}
    sd["lm_head.weight"] = sd["model.embed_tokens.weight"]
    missing, unexpected = m.load_state_dict(sd, strict=False)
    assert not unexpected
    assert all("rotary" in k for k in missing), missing
    with torch.no_grad():
        return m(torch.as_tensor(np.asarray(tokens)[None], dtype=torch.long)).logits[0].numpy()


@pytest.mark.parametrize("variant", ["tiny", "tiny_rep4"])
def test_fp64_model_matches_hf_qwen3(variant):
    shape = SHAPES["tiny"]
    if variant == "tiny_rep4":   # GQA ratio 4 pins the q-head -> kv-head mapping
        shape = dataclasses.replace(shape, name="tiny_rep4", n_q_heads=8, n_kv_heads=2, layers=3)
    w = gen_weights(shape, seed=3)
    toks = gen_prompt(shape.vocab, 24, 0, seed=3)
    ours = M.forward(w, shape, toks, mirror=False)
    ref = _hf_logits(shape, w, toks)
    # HF computes the RoPE cos/sin table in fp32 (inv_freq .float()), which
    # bounds agreement at ~1e-7; any structural error is O(1e-2).
    assert np.max(np.abs(ours - ref)) < 1e-6 * max(1.0, np.abs(ref).max())


def test_split_attention_equals_full_attention_fp64():
    rng = np.random.default_rng(0)
    for trial in range(20):
        d = 128
        n1, n2 = rng.integers(1, 300), rng.integers(1, 300)
        q = rng.normal(size=d) * 1.5
        K = rng.normal(size=(n1 + n2, d))
        V = rng.normal(size=(n1 + n2, d))
        full = A.attention(q, K, V)
        split = A.attention_split(q, K[:n1], V[:n1], K[n1:], V[n1:])
        assert np.max(np.abs(full - split)) < 1e-12


def test_attention_special_cases():
    rng = np.random.default_rng(1)
    q, v = rng.normal(size=128), rng.normal(size=(1, 128))
    assert np.allclose(A.attention(q, rng.normal(size=(1, 128)), v), v[0], atol=1e-15)
    K = np.tile(rng.normal(size=128), (7, 1))         # equal scores -> mean of V
    V = rng.normal(size=(7, 128))
    assert np.allclose(A.attention(q, K, V), V.mean(0), atol=1e-14)


def test_zero_residual_branches_give_closed_form_logits():
    """W_o = W_down = 0 => residual stream = embedding => logits = E . rms(E[tok])."""
    shape = SHAPES["tiny"]
    w = gen_weights(shape, seed=5)
    for l in range(shape.layers):
        w[f"layers.{l}.wo"] = torch.zeros_like(w[f"layers.{l}.wo"])
        w[f"layers.{l}.w_down"] = torch.zeros_like(w[f"layers.{l}.w_down"])
    toks = gen_prompt(shape.vocab, 9, 1, seed=5)
    got = M.forward(w, shape, toks, mirror=False)
    E = w["embed"].double().numpy()
    g = w["final_norm"].double().numpy()
    x = E[toks]
    ref = (x / np.sqrt((x ** 2).mean(1, keepdims=True) + 1e-6) * g) @ E.T
    assert np.max(np.abs(got - ref)) < 1e-10


def test_rope_properties():
    cos, sin = M.rope_cos_sin(np.arange(50), 128, 1e6)
    rng = np.random.default_rng(2)
    x = rng.normal(size=(50, 1, 128))
    y = M.rope(x, cos, sin)
    assert np.allclose(y[0], x[0])                                   # position 0 = identity
    assert np.allclose(np.linalg.norm(y, axis=-1), np.linalg.norm(x, axis=-1))
    q, k = rng.normal(size=(1, 1, 128)), rng.normal(size=(1, 1, 128))
    def dot(p1, p2):
        c1, s1 = M.rope_cos_sin([p1], 128, 1e6)
        c2, s2 = M.rope_cos_sin([p2], 128, 1e6)
        return float((M.rope(q, c1, s1) * M.rope(k, c2, s2)).sum())
    assert abs(dot(10, 3) - dot(27, 20)) < 1e-9                     # relative-position property


def test_round_bf16_is_rne():
    x = np.array([1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8, 1.0 + 2 ** -9, -2.5e-3])
    got = M.round_bf16(x)
    assert got[0] == 1.0 and got[1] == 1.0                # tie -> even
    assert got[2] == 1.0 + 4 * 2 ** -8                    # tie -> even (up)
    assert got[3] == 1.0
    assert got[4] == float(torch.tensor(-2.5e-3).to(torch.bfloat16).double())


def test_mirror_close_to_fp64_and_generate_is_teacher_forcing_consistent():
    shape = SHAPES["tiny"]
    w = gen_weights(shape, seed=7)
    prompt = gen_prompt(shape.vocab, 16, 0, seed=7)
    a = M.forward(w, shape, prompt, mirror=False)
    b = M.forward(w, shape, prompt, mirror=True)
    rel = np.linalg.norm(a - b, axis=1) / np.linalg.norm(a, axis=1)
    assert rel.max() < 2e-2
    toks = M.generate(w, shape, prompt, uid=3, true_len=6, seed=11)
    z = M.teacher_forced_logits(w, shape, prompt, toks)
    from oracle import sampler
    again = [sampler.sample_token(z[t].astype(np.float32), 11, 3, t) for t in range(6)]
    assert again == toks
