"""Oracle: GRPO group advantages and the benchmark reward.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

std_norm  : PAPER.md Eq. 2 (l.128-131)  A_i = (r_i - mean r) / sigma(r)
mean_only : PAPER.md l.320-323          A_i = r_i - (1/G) sum_j r_j
Readings (R28): population sigma; sigma = 0 -> A = 0;
sums in fp64 in ascending id order.

kl_rewards : PAPER.md l.309-311  r_i = RM(O_i, x) - beta * log(pi_theta(O_i|x) / pi_ref(O_i|x)),
             log pi(O_i|x) = sum_t log pi(o_{i,t} | x, o_{i,<t}) (fp64, ascending t).
grpo_objective : Eq. 3 (l.133-141) / Eq. 4 (l.327-338) value: (1/G) sum_i (1/|O_i|) sum_t
             { min(lambda A_i, clip(lambda, 1-eps, 1+eps) A_i) - beta D_KL }, lambda = exp(lp - lp_old);
             D_KL per token = the GRPO paper's estimator pi_ref/pi - log(pi_ref/pi) - 1 (DESIGN R34:
             the paper defers to GRPO for it).  Equal micro groups make Eq. 4's (1/N) sum_n J^(n) = Eq. 3.

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


def kl_rewards(rm, logp, logp_ref, lengths, beta):
    out = []
    for i, L in enumerate(lengths):
        s = 0.0
        for t in range(int(L)):
            s += float(logp[i][t]) - float(logp_ref[i][t])
        out.append(float(rm[i]) - float(beta) * s)
    return out


def grpo_objective(logp, logp_old, logp_ref, adv, lengths, clip_eps, beta):
    G = len(lengths)
    total = 0.0
    for i, L in enumerate(lengths):
        s = 0.0
        for t in range(int(L)):
            lam = math.exp(float(logp[i][t]) - float(logp_old[i][t]))
            a = float(adv[i])
            surr = min(lam * a, min(max(lam, 1.0 - clip_eps), 1.0 + clip_eps) * a)
            d = float(logp_ref[i][t]) - float(logp[i][t])
            kl = math.exp(d) - d - 1.0
            s += surr - beta * kl
        total += s / int(L)
    return total / G
