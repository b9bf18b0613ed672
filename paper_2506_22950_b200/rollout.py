"""Multi-rank rollout plumbing: prompt placement on ranks,
the one exchange, and the group advantages.  bench.py drives its timed rollouts through
these functions; tests/test_multirank.py runs them with world size 2 (gloo, the torch
exchange) and tests/test_gpu_multirank.py through the library's NCCL exchange.

GRPO groups are independent (Eq. 2 l.128-131 normalises within a group), so
rank r runs its own prompts with no data-path communication; the RNG is keyed by the
GLOBAL uid = prompt_id*G + i, so tokens do not depend on the placement.  After a rank's
last rollout, ONE all-gather of every group's per-sample (length, reward) gives every rank
the global arrays the advantages and the policy update need (BASELINE north_star "NCCL
over NVLink used only to all-gather completion lengths and rewards").
"""
import numpy as np

from . import _lib


def shard_prompts(n_prompts, rank, world):
    """Contiguous block of prompt ids owned by `rank` (sizes differ by <= 1)."""
    lo = rank * n_prompts // world
    hi = (rank + 1) * n_prompts // world
    return list(range(lo, hi))


def lpt_place(pool, world, per_rank):
    """LPT placement of prompts on ranks: pool = [(prompt id, predicted
    work)]; the heaviest prompt goes to the least-loaded rank that still has room (equal
    counts per rank, ties -> lower rank / lower id).  Returns {rank: sorted prompt ids}."""
    load, cnt, out = [0.0] * world, [0] * world, {r: [] for r in range(world)}
    for pid, w in sorted(pool, key=lambda x: (-x[1], x[0])):
        r = min((r for r in range(world) if cnt[r] < per_rank), key=lambda r: (load[r], r))
        out[r].append(pid)
        load[r] += w
        cnt[r] += 1
    return {r: sorted(v) for r, v in out.items()}


class RankResults:
    """Per-rank device buffers of the groups' (length, reward): group k of this rank fills
    slots k*G .. k*G+G-1 (is_group_results), exchange() all-gathers them once."""

    def __init__(self, n_groups, G, world, device="cuda"):
        import torch
        self.G, self.n, self.world = G, n_groups, world
        self.len = torch.zeros(n_groups * G, dtype=torch.int32, device=device)
        self.rew = torch.zeros(n_groups * G, dtype=torch.float32, device=device)
        self.all_len = torch.zeros(world * n_groups * G, dtype=torch.int32, device=device)
        self.all_rew = torch.zeros(world * n_groups * G, dtype=torch.float32, device=device)

    def slot(self, k):
        G = self.G
        return self.rew[k * G:(k + 1) * G], self.len[k * G:(k + 1) * G]

    def exchange(self, ctx=None, comm=None, dist=None):
        """The one exchange: the library's NCCL all-gather (comm from _lib.nccl_comm_init), or
        torch.distributed's all_gather (gloo / no library NCCL), or a copy at world size 1."""
        if self.world == 1:
            self.all_len.copy_(self.len)
            self.all_rew.copy_(self.rew)
        elif comm is not None and comm != "torch":
            ctx.is_allgather_results_n(comm, self.len, self.rew, self.all_len, self.all_rew)
        else:
            dist.all_gather_into_tensor(self.all_len, self.len)
            dist.all_gather_into_tensor(self.all_rew, self.rew)
        return self.all_len, self.all_rew


def global_order(placement, world, n_per_rank):
    """Prompt id of each gathered group block (rank-major, then the rank's k-th group)."""
    return [placement[r][k] for r in range(world) for k in range(n_per_rank)]


def group_advantages(rewards, G, mode="std_norm"):
    """Eq. 2 (or the mean-only variant) per group of G samples, via the C-ABI."""
    r = np.asarray(rewards, dtype=np.float32).reshape(-1, G)
    return np.stack([_lib.is_group_advantages(row, mode) for row in r]).reshape(-1)


def advantages_by_prompt(all_len, all_rew, order, G, mode="std_norm"):
    """{prompt id: (lengths, rewards, advantages)} from the gathered arrays.  Samples that did
    not complete (length 0: dynamic mode, R35) are left out of their group's statistics."""
    L = np.asarray(all_len).reshape(-1, G)
    R = np.asarray(all_rew, dtype=np.float32).reshape(-1, G)
    out = {}
    for b, pid in enumerate(order):
        done = L[b] > 0
        adv = np.zeros(G, np.float32)
        if done.any():
            adv[done] = _lib.is_group_advantages(R[b][done], mode)
        out[pid] = (L[b].copy(), R[b].copy(), adv)
    return out


def run_group(ctx, d_prompt, prompt_id, true_len, pred_len, d_reward, d_len):
    """prefill -> plan + slot fill -> decode loop with SJF refill -> rewards."""
    ctx.is_prefill(d_prompt, prompt_id)
    ctx.is_start_group(true_len, pred_len)
    steps = ctx.is_run_group()
    ctx.is_group_results(d_reward, d_len)
    return steps
