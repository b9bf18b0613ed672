"""World size 2 on two GPUs through the library's NCCL exchange: each rank
runs its own tiny-config prompt, writes its group results, and ONE is_allgather_results_n
gives both ranks both groups' (length, reward); they equal what a single rank computes for
both prompts (W-invariance: the RNG is keyed by the global uid).  Skips on a 1-GPU box."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from oracle import kv as okv
    from paper_2506_22950_b200 import _lib, rollout
    from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    shape, seed = SHAPES["tiny"], 20261017
    w = {k: v.cuda() for k, v in gen_weights(shape, seed=seed).items()}
    budget = okv.prefix_bytes(shape, 16) + 4 * 2 * okv.page_bytes(shape, 16)
    ctx = _lib.Context(_lib.make_config(shape, 8, 2, 32, 16, mode="infinite", kv_budget_bytes=budget, seed=seed), w)
    uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(_lib.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    comm = _lib.nccl_comm_init(bytes(uid.cpu().numpy().tobytes()), rank, world)
    res = rollout.RankResults(1, 8, world)
    pid = rank
    true = gen_trace("tiny", 8, 32, 1 + pid)
    d_rew, d_len = res.slot(0)
    rollout.run_group(ctx, torch.as_tensor(gen_prompt(shape.vocab, 16, pid, seed=seed), device="cuda"), pid, true,
                      predict_lengths(true, "noisy", 0.3, seed=1 + pid), d_rew, d_len)
    all_l, all_r = res.exchange(ctx, comm)
    torch.cuda.synchronize()
    q.put((rank, all_l.cpu().numpy().tolist(), all_r.cpu().numpy().tolist()))
    _lib.nccl_comm_destroy(comm)
    ctx.close()
    dist.destroy_process_group()


def test_two_gpu_nccl_exchange_is_world_invariant():
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict((r, (l, w)) for r, l, w in [q.get(timeout=300) for _ in procs])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0] == out[1]
    # W = 1: both prompts on one GPU, one context
    from oracle import kv as okv
    from paper_2506_22950_b200 import _lib, rollout
    from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths
    shape, seed = SHAPES["tiny"], 20261017
    w = {k: v.cuda() for k, v in gen_weights(shape, seed=seed).items()}
    budget = okv.prefix_bytes(shape, 16) + 4 * 2 * okv.page_bytes(shape, 16)
    c = _lib.Context(_lib.make_config(shape, 8, 2, 32, 16, mode="infinite", kv_budget_bytes=budget, seed=seed), w)
    res = rollout.RankResults(2, 8, 1)
    for pid in range(2):
        true = gen_trace("tiny", 8, 32, 1 + pid)
        d_rew, d_len = res.slot(pid)
        rollout.run_group(c, torch.as_tensor(gen_prompt(shape.vocab, 16, pid, seed=seed), device="cuda"), pid, true,
                          predict_lengths(true, "noisy", 0.3, seed=1 + pid), d_rew, d_len)
    all_l, all_r = res.exchange()
    c.close()
    assert out[0][0] == all_l.cpu().numpy().tolist()
    assert np.array_equal(np.float32(out[0][1]), all_r.cpu().numpy())
