"""Oracle: softmax attention, plain and split at the shared prompt prefix.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

`attention` is the textbook definition o = softmax(q K^T / sqrt(d)) V for one
query row (§2.1 l.108: "the current token attends to both cached and
current representations").

`attention_split` is the method's decomposition ("we retain
the prefill KV cache for the prompt itself, which is shared by all groups";
l.205 "Each active sample maintains a separate KV buffer for its response
tokens"): the query attends to the shared prefix and to its own suffix
separately, each part returns (o, m, l) = (normalised output, max score,
sum of exp(score - m)), and the parts are merged by log-sum-exp (DESIGN.md
reading R8):
    m = max(m1, m2);  w_i = exp(m_i - m) * l_i;  o = (w1*o1 + w2*o2) / (w1 + w2).
In real arithmetic this equals `attention` over the concatenation (pin:
tests/test_oracle_model.py, fp64 to 1e-12).
"""
import numpy as np


def attention(q, K, V):
    """q: [d], K, V: [n, d] (float64).  Returns o: [d]."""
    s = (K @ q) / np.sqrt(q.shape[-1])
    p = np.exp(s - s.max())
    return (p @ V) / p.sum()


def attention_partial(q, K, V):
    """Returns (o, m, l) for one part of the key set."""
    s = (K @ q) / np.sqrt(q.shape[-1])
    m = s.max()
    p = np.exp(s - m)
    l = p.sum()
    return (p @ V) / l, m, l


def lse_merge(parts):
    """Merge [(o_i, m_i, l_i)] by log-sum-exp."""
    m = max(p[1] for p in parts)
    w = [np.exp(p[1] - m) * p[2] for p in parts]
    return sum(wi * p[0] for wi, p in zip(w, parts)) / sum(w)


def attention_split(q, K_prefix, V_prefix, K_suffix, V_suffix):
    return lse_merge([attention_partial(q, K_prefix, V_prefix),
                      attention_partial(q, K_suffix, V_suffix)])
