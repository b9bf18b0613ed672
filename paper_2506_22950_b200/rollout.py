"""Rollout driver: one GRPO group per prompt through the C-ABI, prompt-sharded
across ranks.

GRPO groups are independent (Eq. 2 l.128-131 normalises within a
group), so rank r of W runs its own contiguous block of prompt ids with no
data-path communication; the RNG is keyed by the GLOBAL uid = prompt_id*G + i,
so results do not depend on W.  The single exchange is the all-gather of
per-sample (length, reward) needed for the advantages (BASELINE north_star),
done with torch.distributed (NCCL on GPUs, gloo on CPU).
"""
import numpy as np

from . import _lib


def shard_prompts(n_prompts, rank, world):
    """Contiguous block of prompt ids owned by `rank` (sizes differ by <= 1)."""
    lo = rank * n_prompts // world
    hi = (rank + 1) * n_prompts // world
    return list(range(lo, hi))


def gather_results(lengths, rewards, group=None):
    """All-gather per-sample (int32 length, fp32 reward) of every rank.

    lengths / rewards: 1-D tensors of equal size on every rank (the caller
    pads to the per-rank maximum).  Returns (all_lengths, all_rewards) with the
    ranks' blocks concatenated in rank order.
    """
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return lengths, rewards
    world = dist.get_world_size(group)
    out_l = torch.empty(world * lengths.numel(), dtype=lengths.dtype, device=lengths.device)
    out_r = torch.empty(world * rewards.numel(), dtype=rewards.dtype, device=rewards.device)
    dist.all_gather_into_tensor(out_l, lengths.contiguous(), group=group)
    dist.all_gather_into_tensor(out_r, rewards.contiguous(), group=group)
    return out_l, out_r


def group_advantages(rewards, G, mode="std_norm"):
    """Eq. 2 (or the mean-only variant) per group of G samples, via the C-ABI."""
    r = np.asarray(rewards, dtype=np.float32).reshape(-1, G)
    return np.stack([_lib.is_group_advantages(row, mode) for row in r]).reshape(-1)


def run_group(ctx, d_prompt, prompt_id, true_len, pred_len, d_reward, d_len):
    """prefill -> plan + slot fill -> decode loop with SJF refill -> rewards."""
    ctx.is_prefill(d_prompt, prompt_id)
    ctx.is_start_group(true_len, pred_len)
    steps = ctx.is_run_group()
    ctx.is_group_results(d_reward, d_len)
    return steps
