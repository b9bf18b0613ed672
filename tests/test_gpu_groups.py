"""Co-resident prompt groups (is_config.max_groups): several
GRPO groups share every decode step.  Each group must behave exactly as if it ran
alone: its schedule (slot table, pages held) equals the oracle simulation of that
group, its token stream equals a single-group context's at the same row capacity
(batch invariance, R12), and the shared pool never exceeds max_groups x budget."""
import numpy as np
import pytest
import torch

from oracle import kv as okv
from oracle import simulator
from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths

pytestmark = pytest.mark.gpu
TINY = SHAPES["tiny"]
SEED = 20261017
M = 4


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_22950_b200 import _lib
    _lib.load()
    return _lib


def _group(pid):
    prompt = gen_prompt(TINY.vocab, 16, pid, seed=SEED)
    true = gen_trace("tiny", 8, 32, 10 + pid)
    pred = predict_lengths(true, "noisy", 0.3, seed=10 + pid)
    return prompt, true, pred


@pytest.fixture(scope="module")
def multi(lib):
    w_dev = {k: v.cuda() for k, v in gen_weights(TINY, seed=SEED).items()}
    budget = okv.prefix_bytes(TINY, 16) + 4 * 2 * okv.page_bytes(TINY, 16)
    cfg = lib.make_config(TINY, 8, 2, 32, 16, mode="infinite", row_capacity=16, kv_budget_bytes=budget, seed=SEED,
                          max_groups=M)
    ctx = lib.Context(cfg, w_dev)
    groups = {pid: _group(pid) for pid in range(6)}
    # groups 0..2 start together, 3 joins after a few steps, slots are refilled with prompts 4, 5
    slot_of, results = {}, {}
    for slot, pid in enumerate([0, 1, 2]):
        p, t, pr = groups[pid]
        ctx.is_prefill(torch.as_tensor(p, device="cuda"), pid, slot=slot)
        ctx.is_start_group(t, pr, slot=slot)
        slot_of[slot] = pid
    for _ in range(5):
        ctx.is_decode_step()
    p, t, pr = groups[3]
    ctx.is_prefill(torch.as_tensor(p, device="cuda"), 3, slot=3)
    ctx.is_start_group(t, pr, slot=3)
    slot_of[3] = 3
    pending = [4, 5]
    peak = 0
    while slot_of:
        mask, _ = ctx.is_run_until_any_done()
        for slot in list(slot_of):
            if mask >> slot & 1:
                pid = slot_of.pop(slot)
                st = ctx.is_query(slot)
                results[pid] = dict(tokens=ctx.is_copy_tokens(slot), sched=ctx.is_copy_schedule(slot=slot), stats=st)
                peak = max(peak, st["global_peak_kv_bytes"])
                if pending:
                    nxt = pending.pop(0)
                    p, t, pr = groups[nxt]
                    ctx.is_prefill(torch.as_tensor(p, device="cuda"), nxt, slot=slot)
                    ctx.is_start_group(t, pr, slot=slot)
                    slot_of[slot] = nxt
    ctx.close()
    # the same prompts alone, one context each (same row capacity -> same kernel configuration)
    alone = {}
    for pid, (p, t, pr) in groups.items():
        c1 = lib.Context(lib.make_config(TINY, 8, 2, 32, 16, mode="infinite", row_capacity=16, kv_budget_bytes=budget,
                                         seed=SEED), w_dev)
        c1.is_prefill(torch.as_tensor(p, device="cuda"), pid)
        c1.is_start_group(t, pr)
        c1.is_run_group()
        alone[pid] = c1.is_copy_tokens()
        c1.close()
    return dict(groups=groups, results=results, alone=alone, budget=budget, peak=peak)


def test_groups_all_complete(multi):
    assert sorted(multi["results"]) == list(range(6))
    for pid, r in multi["results"].items():
        assert r["stats"]["completed"] == 8 and r["stats"]["error"] == 0, pid


def test_groups_schedule_equals_single_group_oracle(multi):
    for pid, r in multi["results"].items():
        _, true, pred = multi["groups"][pid]
        ref = simulator.simulate(true, "infinite", 2, pred=pred, eps=0.1, page_tokens=16)
        slots, live = r["sched"]
        assert r["stats"]["steps"] == ref.total_steps, pid
        assert slots.tolist() == ref.slot_table, pid
        assert live.tolist() == ref.live_pages, pid
        assert r["stats"]["peak_pages"] == ref.peak_pages, pid


def test_groups_tokens_equal_single_group_runs(multi):
    for pid, r in multi["results"].items():
        assert np.array_equal(r["tokens"], multi["alone"][pid]), pid


def test_groups_shared_pool_within_budget(multi):
    assert multi["peak"] <= M * multi["budget"]


def test_groups_dynamic_mode_each_group_as_alone(lib):
    """Dynamic-slot sampling (R35) with co-resident groups: every group stops at its own
    target-th completion; its schedule equals the single-group oracle simulation and its
    completed samples' tokens equal a single-group context's."""
    w_dev = {k: v.cuda() for k, v in gen_weights(TINY, seed=SEED).items()}
    target = 5
    cfg = lib.make_config(TINY, 8, 2, 32, 16, mode="dynamic", row_capacity=16, seed=SEED, max_groups=3,
                          dynamic_target=target)
    ctx = lib.Context(cfg, w_dev)
    groups = {pid: _group(pid) for pid in range(3)}
    for slot, (p, t, pr) in groups.items():
        ctx.is_prefill(torch.as_tensor(p, device="cuda"), slot, slot=slot)
        ctx.is_start_group(t, pr, slot=slot)
    done = 0
    while done != 0b111:
        mask, _ = ctx.is_run_until_any_done()
        done |= mask
    res = {s: (ctx.is_query(s), ctx.is_copy_schedule(slot=s), ctx.is_copy_tokens(s)) for s in range(3)}
    ctx.close()
    for s, (st, (slots, live), toks) in res.items():
        _, true, _ = groups[s]
        ref = simulator.simulate(true, "dynamic", 2, page_tokens=16, target=target)
        assert st["completed"] == target and st["discarded"] == len(ref.discarded), s
        assert slots.tolist() == ref.slot_table and live.tolist() == ref.live_pages, s
        c1 = lib.Context(lib.make_config(TINY, 8, 2, 32, 16, mode="dynamic", row_capacity=16, seed=SEED,
                                         dynamic_target=target), w_dev)
        c1.is_prefill(torch.as_tensor(groups[s][0], device="cuda"), s)
        c1.is_start_group(true, groups[s][2])
        c1.is_run_group()
        alone = c1.is_copy_tokens()
        c1.close()
        for uid in ref.finish_step:
            assert np.array_equal(toks[uid], alone[uid]), (s, uid)
