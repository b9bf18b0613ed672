"""World-size-2 gloo test of the N>1 path on CPU: prompt sharding, the one
all-gather of (length, reward), and W-invariance of the advantages
(BASELINE north_star "NCCL ... only to all-gather completion
lengths and rewards")."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import grpo


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _fake_group(pid, G):
    """Deterministic stand-in for one rollout's (lengths, rewards) of prompt pid."""
    rng = np.random.default_rng(1000 + pid)
    return rng.integers(1, 1024, G).astype(np.int32), rng.random(G).astype(np.float32)


def _worker(rank, world, port, n_prompts, G, q):
    """One rank of the production host path (paper_2506_22950_b200.rollout, as bench.py drives
    it): its prompts' results in RankResults slots, ONE exchange after the last group (the torch
    path: gloo here; the library's NCCL path is tests/test_gpu_multirank.py), then the
    advantages of every prompt from the gathered arrays."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2506_22950_b200 import rollout
    per_rank = -(-n_prompts // world)
    # block placement padded to equal counts (a padding group reports length 0: not completed)
    placement = {r: rollout.shard_prompts(n_prompts, r, world) for r in range(world)}
    placement = {r: v + [-1 - r * per_rank - k for k in range(per_rank - len(v))] for r, v in placement.items()}
    res = rollout.RankResults(per_rank, G, world, device="cpu")
    for k, pid in enumerate(placement[rank]):
        d_rew, d_len = res.slot(k)
        if pid >= 0:
            l, r = _fake_group(pid, G)
            d_len.copy_(torch.from_numpy(l))
            d_rew.copy_(torch.from_numpy(r))
    all_l, all_r = res.exchange(ctx=None, comm="torch", dist=dist)
    order = rollout.global_order(placement, world, per_rank)
    by_pid = rollout.advantages_by_prompt(all_l.numpy(), all_r.numpy(), order, G)
    real = sorted(p for p in by_pid if p >= 0)
    ln = np.concatenate([by_pid[p][0] for p in real])
    rew = np.concatenate([by_pid[p][1] for p in real])
    adv = np.concatenate([by_pid[p][2] for p in real])
    q.put((rank, ln.tolist(), rew.tolist(), adv.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("n_prompts", [4, 5])
def test_two_rank_gather_and_advantages_are_world_invariant(n_prompts):
    G = 8
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_prompts, G, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # W = 1 reference
    ref_l = np.concatenate([_fake_group(p, G)[0] for p in range(n_prompts)])
    ref_r = np.concatenate([_fake_group(p, G)[1] for p in range(n_prompts)])
    ref_a = np.concatenate([np.float32(grpo.advantages([float(x) for x in ref_r[i * G:(i + 1) * G]]))
                            for i in range(n_prompts)])
    for rank, ln, rw, adv in res:
        assert ln == ref_l.tolist()
        assert np.array_equal(np.float32(rw), ref_r)
        assert np.array_equal(np.float32(adv), ref_a)


def test_shard_prompts_partitions():
    from paper_2506_22950_b200 import rollout
    for n in range(0, 20):
        for w in (1, 2, 3, 4, 8):
            got = [p for r in range(w) for p in rollout.shard_prompts(n, r, w)]
            assert got == list(range(n))


def test_lpt_placement_balances_predicted_work():
    """bench.py's LPT placement of prompts on ranks (NEXT-4): equal counts, every prompt
    placed once, and the max rank load within one prompt of the mean (LPT's bound)."""
    import bench
    rng = np.random.default_rng(3)
    for world in (2, 4, 8):
        per = 3
        pool = [(pid, float(w)) for pid, w in enumerate(rng.lognormal(9.0, 0.5, world * per))]
        out = bench.lpt_place(pool, world, per)  # (= paper_2506_22950_b200.rollout.lpt_place)
        assert sorted(p for v in out.values() for p in v) == list(range(world * per))
        assert all(len(v) == per for v in out.values())
        w = dict(pool)
        loads = [sum(w[p] for p in v) for v in out.values()]
        assert max(loads) - np.mean(loads) <= max(w.values())
        assert out == bench.lpt_place(pool, world, per)  # deterministic
