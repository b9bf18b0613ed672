"""The C-ABI calls' own contracts, on the tiny config (BASELINE configs[0]).

* is_refill alone is Alg. 1's loop body without the model (Alg. 3
  "the cache is cleared and the memory is reassigned back to the pool"): driving a
  group with is_refill only reproduces the oracle simulation's slot table and page
  counts step by step (the schedule is token-independent, R5), and d_new_uid reports
  every co-resident group's rows.
* is_decode_step's outputs (north_star "is_decode_step(slot table) -> next tokens"):
  d_next_tokens per row equals the token the step appended for that row's sample,
  d_finished marks exactly the samples that reached their length; idle rows -1 / 0.
* A page pool smaller than the run needs (IS_DBG_POOL_PAGES) surfaces as
  IS_ERR_BUDGET from the run loop and from is_decode_step, with no page handed out
  beyond the pool (R25: the budget is a hard invariant).
* is_group_results in dynamic-slot mode (R35): only the dynamic_target completed
  samples report a length (= true_len) and reward; discarded / unstarted ones report 0.
"""
import os

import numpy as np
import pytest
import torch

from oracle import grpo, simulator
from oracle import kv as okv
from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths

pytestmark = pytest.mark.gpu
TINY = SHAPES["tiny"]
SEED = 20261017


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_22950_b200 import _lib
    _lib.load()
    return _lib


@pytest.fixture(scope="module")
def setup(lib):
    w = {k: v.cuda() for k, v in gen_weights(TINY, seed=SEED).items()}
    budget = okv.prefix_bytes(TINY, 16) + 4 * 2 * okv.page_bytes(TINY, 16)
    groups = []
    for pid in range(2):
        prompt = gen_prompt(TINY.vocab, 16, pid, seed=SEED)
        true = gen_trace("tiny", 8, 32, 1 + pid)
        groups.append((pid, prompt, true, predict_lengths(true, "noisy", 0.3, seed=1 + pid)))
    return w, budget, groups


def _ctx(lib, w, budget, mode="infinite", M=1, target=0):
    cfg = lib.make_config(TINY, 8, 2, 32, 16, mode=mode, row_capacity=16, kv_budget_bytes=budget, seed=SEED,
                          max_groups=M, dynamic_target=target)
    return lib.Context(cfg, w)


def test_refill_alone_reproduces_the_oracle_schedule(lib, setup):
    w, budget, groups = setup
    ctx = _ctx(lib, w, budget, M=2)
    for m, (pid, prompt, true, pred) in enumerate(groups):
        ctx.is_prefill(torch.as_tensor(prompt, device="cuda"), pid, slot=m)
        ctx.is_start_group(true, pred, slot=m)
    refs = [simulator.simulate(true, "infinite", 2, pred=pred, eps=0.1, page_tokens=16) for _, _, true, pred in groups]
    fin = torch.zeros(16, dtype=torch.uint8, device="cuda")
    uid = torch.zeros(16, dtype=torch.int32, device="cuda")
    n = max(r.total_steps for r in refs)
    for step in range(n):
        ctx.is_refill(fin, uid)
        u = uid.cpu().numpy()
        f = fin.cpu().numpy()
        for m, r in enumerate(refs):
            row = u[2 * m:2 * m + 2].tolist()
            # the rows after refill `step` are the slots of step + 1 (idle = -1 once done)
            nxt = r.slot_table[step + 1] if step + 1 < r.total_steps else [-1, -1]
            assert row == nxt, (m, step, row, nxt)
            # the finish flags: the samples of step `step` that reached their length in it
            if step < r.total_steps:
                for s, i in enumerate(r.slot_table[step]):
                    steps_run = sum(i in r.slot_table[k] for k in range(step + 1)) if i >= 0 else 0
                    assert int(f[2 * m + s]) == int(i >= 0 and steps_run == int(groups[m][2][i])), (m, step, s)
        assert np.all(u[4:] == -1)
    for m, r in enumerate(refs):
        st = ctx.is_query(m)
        slots, live = ctx.is_copy_schedule(slot=m)
        assert st["steps"] == r.total_steps and st["completed"] == 8 and st["error"] == 0
        assert slots.tolist() == r.slot_table and live.tolist() == r.live_pages
        assert np.all(ctx.is_copy_tokens(m) == -1)  # no model ran: no token was sampled
    ctx.close()


def test_decode_step_outputs(lib, setup):
    w, budget, groups = setup
    pid, prompt, true, pred = groups[0]
    ctx = _ctx(lib, w, budget)
    ctx.is_prefill(torch.as_tensor(prompt, device="cuda"), pid)
    ctx.is_start_group(true, pred)
    ref = simulator.simulate(true, "infinite", 2, pred=pred, eps=0.1, page_tokens=16)
    nxt = torch.zeros(16, dtype=torch.int32, device="cuda")
    fin = torch.zeros(16, dtype=torch.uint8, device="cuda")
    outs = []
    for step in range(ref.total_steps):
        ctx.is_decode_step(nxt, fin)
        outs.append((nxt.cpu().numpy().copy(), fin.cpu().numpy().copy()))
    toks = ctx.is_copy_tokens()
    assert ctx.is_query()["completed"] == 8
    ctx.close()
    t_of = {}
    for step, (n, f) in enumerate(outs):
        for s in range(16):
            i = ref.slot_table[step][s] if s < 2 else -1
            if i < 0:
                assert n[s] == -1 and f[s] == 0, (step, s)
                continue
            t = t_of.get(i, 0)
            assert n[s] == toks[i, t], (step, s, i, t)
            assert f[s] == int(t + 1 == true[i]), (step, s)
            t_of[i] = t + 1
    assert sum(t_of.values()) == int(np.sum(true))


def test_undersized_pool_is_a_budget_error(lib, setup):
    w, budget, groups = setup
    pid, prompt, true, pred = groups[0]
    ref = simulator.simulate(true, "infinite", 2, pred=pred, eps=0.1, page_tokens=16)
    small = ref.peak_pages - 1  # one page short of what the schedule needs at its peak
    os.environ["IS_DBG_POOL_PAGES"] = str(small)
    try:
        ctx = _ctx(lib, w, budget)
    finally:
        del os.environ["IS_DBG_POOL_PAGES"]
    assert ctx.is_query()["num_pages"] == small
    ctx.is_prefill(torch.as_tensor(prompt, device="cuda"), pid)
    ctx.is_start_group(true, pred)
    with pytest.raises(lib.InfsampError) as e:
        ctx.is_run_group()
    assert e.value.status == lib.IS_ERR_BUDGET
    st = ctx.is_query()
    assert st["error"] == 1 and st["live_pages"] <= small and st["peak_pages"] <= small
    with pytest.raises(lib.InfsampError) as e:
        ctx.is_decode_step()
    assert e.value.status == lib.IS_ERR_BUDGET
    ctx.close()


def test_dynamic_mode_results_mark_incomplete_samples(lib, setup):
    w, budget, groups = setup
    pid, prompt, true, pred = groups[0]
    target = 5
    ctx = _ctx(lib, w, 0, mode="dynamic", target=target)
    ctx.is_prefill(torch.as_tensor(prompt, device="cuda"), pid)
    ctx.is_start_group(true, pred)
    ctx.is_run_group()
    rew = torch.full((8,), -1.0, device="cuda")
    ln = torch.full((8,), -1, dtype=torch.int32, device="cuda")
    ctx.is_group_results(rew, ln)
    toks = ctx.is_copy_tokens()
    ctx.close()
    ref = simulator.simulate(true, "dynamic", 2, page_tokens=16, target=target)
    ln, rew = ln.cpu().numpy(), rew.cpu().numpy()
    done = [i for i in range(8) if ln[i] > 0]
    assert len(done) == target
    assert set(done).isdisjoint(ref.discarded)
    for i in range(8):
        if i in done:
            assert ln[i] == true[i]
            assert abs(rew[i] - grpo.bench_reward(toks[i, :true[i]].tolist(), TINY.vocab)) < 1e-7
        else:
            assert ln[i] == 0 and rew[i] == 0.0
