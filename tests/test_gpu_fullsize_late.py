"""Full-size parity where the kernels take their long-suffix and many-row branches.

* Late step (config 3 launch configuration: Qwen3-1.7B shape, P = 256, G = 32, g = 8,
  16-row step, CUDA graph replay): every sample is 1024 tokens long, so at decode
  step 1000 all eight slots attend to 1001 suffix tokens = 32 suffix chunks + 2 prefix
  tiles, i.e. the > 32-partial branch of the fused LSE merge (R8).  Teacher-forced
  oracle logits (fp64, bf16-mirrored) for four slots within SURVEY C31's 2e-2 normwise
  and max-abs bounds; the sampler on the dumped logits bit-exact for all slots.
* Eight co-resident groups (gate/up split 1,
  o_proj/down split 4, 64-token suffix units + separate merge kernel): each group's
  schedule equals the single-group oracle simulation, and teacher-forced logits of one
  slot in three different groups match the oracle at t = 0 and t = 70.
"""
import numpy as np
import pytest
import torch

from oracle import model as M
from oracle import sampler, simulator
from oracle import kv as okv
from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths

pytestmark = pytest.mark.gpu
SEED = 20261017
SHAPE = SHAPES["qwen3-1.7b"]
P, G, g, MAX_NEW = 256, 32, 8, 1024
LATE = 1000


def _budget():
    kv_tok = okv.kv_bytes_per_token(SHAPE.layers, SHAPE.n_kv_heads, SHAPE.head_dim)
    return (P - 1) * kv_tok + g * (MAX_NEW // 16) * 16 * kv_tok


def _logits_ok(d, z):
    d = d.astype(np.float64)
    rel = np.linalg.norm(d - z) / np.linalg.norm(z)
    mabs = np.max(np.abs(d - z))
    assert rel < 2e-2, rel
    assert mabs <= 2e-2 * np.max(np.abs(z)), (mabs, np.max(np.abs(z)))
    return mabs


@pytest.fixture(scope="module")
def weights():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    w = gen_weights(SHAPE, seed=SEED, device="cuda")
    yield w, {k: v.cpu() for k, v in w.items()}
    del w
    torch.cuda.empty_cache()


@pytest.fixture(scope="module")
def late(weights):
    from paper_2506_22950_b200 import _lib
    w, w_cpu = weights
    cfg = _lib.make_config(SHAPE, G, g, MAX_NEW, P, mode="infinite", page_tokens=16, kv_budget_bytes=_budget(),
                           eps=0.1, temperature=0.8, seed=SEED)
    ctx = _lib.Context(cfg, w)
    pid = 7
    prompt = gen_prompt(SHAPE.vocab, P, pid, seed=SEED)
    true = np.full(G, MAX_NEW, np.int32)
    pred = predict_lengths(true, "noisy", 0.3, seed=SEED + pid)
    ctx.is_prefill(torch.as_tensor(prompt, device="cuda"), pid)
    ctx.is_start_group(true, pred)
    for _ in range(LATE):
        ctx.is_decode_step()
    dump = torch.zeros(16, SHAPE.vocab, device="cuda")
    ctx.is_set_logits_dump(dump)
    ctx.is_decode_step()
    torch.cuda.synchronize()
    d = dump.cpu().numpy().copy()
    ctx.is_set_logits_dump(None)
    res = dict(dump=d, sched=ctx.is_copy_schedule(), tokens=ctx.is_copy_tokens(), prompt=prompt, pid=pid,
               stats=ctx.is_query())
    ctx.close()
    return res


def test_late_step_sampler_bit_exact(late):
    slots, _ = late["sched"]
    assert all(int(u) >= 0 for u in slots[LATE][:g])
    for s in range(g):
        uid = int(slots[LATE][s])
        assert int(slots[0][s]) == uid  # every sample started at step 0: t = LATE
        got = sampler.sample_token(late["dump"][s], SEED, late["pid"] * G + uid, LATE)
        assert got == late["tokens"][uid, LATE], (s, uid)


def test_late_step_teacher_forced_logits(late, weights):
    """t = 1000: 1001 suffix tokens per slot (> 32 partials in the merge) for four slots."""
    _, w_cpu = weights
    slots, _ = late["sched"]
    for s in (0, 3, 5, 7):
        uid = int(slots[LATE][s])
        gen = [int(x) for x in late["tokens"][uid, :LATE + 1]]
        z = M.teacher_forced_logits(w_cpu, SHAPE, late["prompt"], gen, mirror=True, rows=[LATE])[0]
        mabs = _logits_ok(late["dump"][s], z)
        tok, margin = sampler.sample_margin(z.astype(np.float32), SEED, late["pid"] * G + uid, LATE)
        if tok != gen[LATE]:
            assert margin < 2 * 1.25 * mabs, (s, margin)


MG = 8
STEPS_AT = (0, 70)


@pytest.fixture(scope="module")
def coresident(weights):
    from paper_2506_22950_b200 import _lib
    w, _ = weights
    cfg = _lib.make_config(SHAPE, G, g, MAX_NEW, P, mode="infinite", page_tokens=16, kv_budget_bytes=_budget(),
                           eps=0.1, temperature=0.8, seed=SEED, max_groups=MG)
    ctx = _lib.Context(cfg, w)
    groups = {}
    for m in range(MG):
        pid = 20 + m
        prompt = gen_prompt(SHAPE.vocab, P, pid, seed=SEED)
        true = gen_trace("math", G, MAX_NEW, SEED + pid)
        pred = predict_lengths(true, "noisy", 0.3, seed=SEED + pid)
        ctx.is_prefill(torch.as_tensor(prompt, device="cuda"), pid, slot=m)
        ctx.is_start_group(true, pred, slot=m)
        groups[m] = (pid, prompt, true, pred)
    rc = ctx.is_query()["row_capacity"]
    assert rc == MG * g
    dump = torch.zeros(rc, SHAPE.vocab, device="cuda")
    dumps = {}
    for step in range(max(STEPS_AT) + 1):
        if step in STEPS_AT:
            ctx.is_set_logits_dump(dump)
        ctx.is_decode_step()
        if step in STEPS_AT:
            torch.cuda.synchronize()
            dumps[step] = dump.cpu().numpy().copy()
            ctx.is_set_logits_dump(None)
    done = 0
    while done != (1 << MG) - 1:
        mask, _ = ctx.is_run_until_any_done()
        done |= mask
    res = {m: dict(stats=ctx.is_query(m), sched=ctx.is_copy_schedule(slot=m), tokens=ctx.is_copy_tokens(m))
           for m in range(MG)}
    ctx.close()
    return dict(groups=groups, res=res, dumps=dumps)


def test_coresident_schedules_equal_oracle(coresident):
    for m, (pid, _, true, pred) in coresident["groups"].items():
        r = coresident["res"][m]
        ref = simulator.simulate(true, "infinite", g, pred=pred, eps=0.1, page_tokens=16)
        slots, live = r["sched"]
        assert r["stats"]["steps"] == ref.total_steps, m
        assert slots.tolist() == ref.slot_table, m
        assert live.tolist() == ref.live_pages, m
        assert r["stats"]["completed"] == G and r["stats"]["error"] == 0, m


def test_coresident_sampler_bit_exact_on_dumped_logits(coresident):
    for step, d in coresident["dumps"].items():
        for m, (pid, _, _, _) in coresident["groups"].items():
            slots, _ = coresident["res"][m]["sched"]
            toks = coresident["res"][m]["tokens"]
            for s, uid in enumerate(slots[step]):
                uid = int(uid)
                if uid < 0:
                    continue
                t = step - next(k for k in range(step + 1) if int(slots[k][s]) == uid)
                got = sampler.sample_token(d[m * g + s], SEED, pid * G + uid, t)
                assert got == toks[uid, t], (step, m, s)


def test_coresident_teacher_forced_logits(coresident, weights):
    """64-row step: slot 0 of three groups (each still on its first sample at t = 70)
    against the oracle at t = 0 and t = 70."""
    _, w_cpu = weights
    checked = 0
    for m in range(MG):
        pid, prompt, true, _ = coresident["groups"][m]
        slots, _ = coresident["res"][m]["sched"]
        uid = int(slots[0][0])
        if checked == 3 or true[uid] <= max(STEPS_AT) or int(slots[max(STEPS_AT)][0]) != uid:
            continue
        gen = [int(x) for x in coresident["res"][m]["tokens"][uid, :max(STEPS_AT) + 1]]
        z = M.teacher_forced_logits(w_cpu, SHAPE, prompt, gen, mirror=True, rows=list(STEPS_AT))
        for i, step in enumerate(STEPS_AT):
            mabs = _logits_ok(coresident["dumps"][step][m * g], z[i])
            tok, margin = sampler.sample_margin(z[i].astype(np.float32), SEED, pid * G + uid, step)
            if tok != gen[step]:
                assert margin < 2 * 1.25 * mabs, (m, step, margin)
        checked += 1
    assert checked >= 2
