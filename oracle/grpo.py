"""Oracle: GRPO group advantages and the benchmark reward.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

std_norm  : PAPER.md Eq. 2 (l.128-131)  A_i = (r_i - mean r) / sigma(r)
mean_only : PAPER.md l.320-323          A_i = r_i - (1/G) sum_j r_j
Readings (R28): population sigma; sigma = 0 -> A = 0;
sums in fp64 in ascending id order.

bench_reward (R29): the reward model is OUT of scope, so
benchmarks use a deterministic token statistic r_i = #{t : tok_t < vocab/2} / len_i.
"""
import math


def advantages(r, mode="std_norm"):
    G = len(r)
    s = 0.0
    for x in r:
        s += float(x)
    mean = s / G
    if mode == "mean_only":
        return [float(x) - mean for x in r]
    if mode != "std_norm":
        raise ValueError(f"IS_ERR_CONFIG: unknown advantage mode {mode}")
    v = 0.0
    for x in r:
        v += (float(x) - mean) ** 2
    sigma = math.sqrt(v / G)
    if sigma == 0.0:
        return [0.0] * G
    return [(float(x) - mean) / sigma for x in r]


def bench_reward(tokens, vocab):
    n = len(tokens)
    return sum(1 for x in tokens if x < vocab // 2) / n
