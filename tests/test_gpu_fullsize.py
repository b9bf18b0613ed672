"""GPU parity at BASELINE.json's full sizes (config 3: Qwen3-1.7B shape, P = 256,
G = 32, g = 8), in the launch configuration bench.py times (same context
settings, CUDA graph replay).  The oracle recomputes sampled outputs one by
one: teacher-forced logits at sampled positions, the sampler on dumped logits,
and the complete schedule (slot table, page counts) of the rollout."""
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
LATE = 70  # step whose logits are checked at t = 70 (3 suffix chunks of 32 tokens)


@pytest.fixture(scope="module")
def full():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_22950_b200 import _lib
    w = gen_weights(SHAPE, seed=SEED, device="cuda")
    kv_tok = okv.kv_bytes_per_token(SHAPE.layers, SHAPE.n_kv_heads, SHAPE.head_dim)
    budget = (P - 1) * kv_tok + g * (MAX_NEW // 16) * 16 * kv_tok
    cfg = _lib.make_config(SHAPE, G, g, MAX_NEW, P, mode="infinite", page_tokens=16, kv_budget_bytes=budget,
                           eps=0.1, temperature=0.8, seed=SEED)
    ctx = _lib.Context(cfg, w)
    prompt = gen_prompt(SHAPE.vocab, P, 3, seed=SEED)
    true = gen_trace("math", G, MAX_NEW, SEED + 3)
    pred = predict_lengths(true, "noisy", 0.3, seed=SEED + 3)
    ctx.is_prefill(torch.as_tensor(prompt, device="cuda"), 3)
    ctx.is_start_group(true, pred)
    # first steps with a logits dump (eager step per call, graph replay)
    dump = torch.zeros(16, SHAPE.vocab, device="cuda")
    ctx.is_set_logits_dump(dump)
    dumps = []
    for _ in range(3):
        ctx.is_decode_step()
        torch.cuda.synchronize()
        dumps.append(dump.cpu().numpy().copy())
    # a later step: several suffix chunks per slot (multi-chunk suffix attention + LSE merge)
    for _ in range(LATE - 3):
        ctx.is_decode_step()
    ctx.is_decode_step()
    torch.cuda.synchronize()
    late = dump.cpu().numpy().copy()
    ctx.is_set_logits_dump(None)
    steps = ctx.is_run_group()
    res = dict(steps=steps, stats=ctx.is_query(), sched=ctx.is_copy_schedule(), tokens=ctx.is_copy_tokens(),
               dumps=dumps, late=late, true=true, pred=pred, prompt=prompt, budget=budget,
               w_cpu={k: v.cpu() for k, v in w.items()})
    ctx.close()
    del w
    torch.cuda.empty_cache()
    return res


def test_fullsize_schedule_bit_exact(full):
    ref = simulator.simulate(full["true"], "infinite", g, pred=full["pred"], eps=0.1, page_tokens=16)
    slots, live = full["sched"]
    assert full["steps"] == ref.total_steps
    assert slots.tolist() == ref.slot_table
    assert live.tolist() == ref.live_pages
    st = full["stats"]
    assert st["completed"] == G and st["error"] == 0
    assert st["peak_pages"] == ref.peak_pages
    assert st["tokens_decoded"] == int(np.sum(full["true"]))
    assert st["peak_kv_bytes"] <= full["budget"]
    toks = full["tokens"]
    for i, L in enumerate(full["true"]):
        assert np.all(toks[i, :L] >= 0) and np.all(toks[i, :L] < SHAPE.vocab) and np.all(toks[i, L:] == -1)


def test_fullsize_sampler_bit_exact_on_dumped_logits(full):
    slots, _ = full["sched"]
    toks = full["tokens"]
    for step in range(3):
        for s, uid in enumerate(slots[step]):
            if uid < 0:
                continue
            got = sampler.sample_token(full["dumps"][step][s], SEED, 3 * G + int(uid), step)
            assert got == toks[uid, step], (step, s, uid)


def test_fullsize_teacher_forced_logits_and_tokens(full):
    """Oracle (fp64, bf16-mirrored) logits for sample slot 0 at t = 0, 1, 2 vs the GPU dump."""
    slots, _ = full["sched"]
    uid = int(slots[0][0])
    gen = [int(x) for x in full["tokens"][uid, :3]]
    z = M.teacher_forced_logits(full["w_cpu"], SHAPE, full["prompt"], gen, mirror=True, rows=[0, 1, 2])
    for t in range(3):
        d = full["dumps"][t][0].astype(np.float64)
        rel = np.linalg.norm(d - z[t]) / np.linalg.norm(z[t])
        assert rel < 2e-2, (t, rel)
        assert np.max(np.abs(d - z[t])) <= 2e-2 * np.max(np.abs(z[t]))
        tok, margin = sampler.sample_margin(z[t].astype(np.float32), SEED, 3 * G + uid, t)
        if tok != gen[t]:
            assert margin < 2 * 1.25 * np.max(np.abs(d - z[t])), (t, margin)


def test_fullsize_late_step_logits(full):
    """Teacher-forced oracle logits at step LATE for every slot still decoding its first sample."""
    slots, _ = full["sched"]
    checked = 0
    for s, uid in enumerate(slots[LATE]):
        uid = int(uid)
        if uid < 0 or uid != int(slots[0][s]) or checked >= 2:
            continue  # only samples that started at step 0 (t = LATE)
        gen = [int(x) for x in full["tokens"][uid, :LATE + 1]]
        z = M.teacher_forced_logits(full["w_cpu"], SHAPE, full["prompt"], gen, mirror=True, rows=[LATE])[0]
        d = full["late"][s].astype(np.float64)
        rel = np.linalg.norm(d - z) / np.linalg.norm(z)
        assert rel < 2e-2, (s, rel)
        assert np.max(np.abs(d - z)) <= 2e-2 * np.max(np.abs(z))
        assert sampler.sample_token(full["late"][s], SEED, 3 * G + uid, LATE) == full["tokens"][uid, LATE]
        checked += 1
    assert checked > 0


@pytest.fixture(scope="module")
def prefix_phase():
    """BASELINE config 4 at full size: Qwen3-1.7B shape, G = 64, g = 8, prefix phase k = 16
    (parked pages), long-tail lengths, 1 GiB KV budget."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_22950_b200 import _lib
    G4, g4, k4, budget = 64, 8, 16, 1 << 30
    w = gen_weights(SHAPE, seed=SEED, device="cuda")
    cfg = _lib.make_config(SHAPE, G4, g4, MAX_NEW, P, mode="infinite", prefix_k=k4, page_tokens=16,
                           kv_budget_bytes=budget, eps=0.1, temperature=0.8, seed=SEED)
    ctx = _lib.Context(cfg, w)
    prompt = gen_prompt(SHAPE.vocab, P, 5, seed=SEED)
    true = gen_trace("longtail", G4, MAX_NEW, SEED + 5)
    pred = predict_lengths(true, "noisy", 0.3, seed=SEED + 5, prefix_k=k4)
    ctx.is_prefill(torch.as_tensor(prompt, device="cuda"), 5)
    ctx.is_start_group(true, pred)
    steps = ctx.is_run_group()
    res = dict(steps=steps, stats=ctx.is_query(), sched=ctx.is_copy_schedule(), true=true, pred=pred,
               budget=budget, G=G4, g=g4, k=k4)
    ctx.close()
    del w
    torch.cuda.empty_cache()
    return res


def test_fullsize_prefix_phase_schedule_and_budget(prefix_phase):
    r = prefix_phase
    ref = simulator.simulate(r["true"], "infinite", r["g"], pred=r["pred"], eps=0.1, prefix_k=r["k"], page_tokens=16)
    slots, live = r["sched"]
    assert r["steps"] == ref.total_steps
    assert r["stats"]["prefix_steps"] == ref.prefix_steps
    assert slots.tolist() == ref.slot_table
    assert live.tolist() == ref.live_pages
    st = r["stats"]
    assert st["completed"] == r["G"] and st["error"] == 0
    assert st["peak_pages"] == ref.peak_pages
    assert st["peak_kv_bytes"] <= r["budget"]  # R25: the budget is a hard invariant


def test_fullsize_topp_step_bit_exact():
    """top-p = 0.9 at full size (vocab 151,936, 8 live rows): three decode steps, every
    sampled token equals the oracle's nucleus draw on the dumped logits."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_22950_b200 import _lib
    w = gen_weights(SHAPE, seed=SEED, device="cuda")
    cfg = _lib.make_config(SHAPE, G, g, MAX_NEW, P, mode="infinite", page_tokens=16, eps=0.1, temperature=0.8,
                           seed=SEED, top_p=0.9)
    ctx = _lib.Context(cfg, w)
    prompt = gen_prompt(SHAPE.vocab, P, 5, seed=SEED)
    true = gen_trace("math", G, MAX_NEW, SEED + 5)
    ctx.is_prefill(torch.as_tensor(prompt, device="cuda"), 5)
    ctx.is_start_group(true, predict_lengths(true, "noisy", 0.3, seed=SEED + 5))
    dump = torch.zeros(16, SHAPE.vocab, device="cuda")
    ctx.is_set_logits_dump(dump)
    dumps = []
    for _ in range(3):
        ctx.is_decode_step()
        torch.cuda.synchronize()
        dumps.append(dump.cpu().numpy().copy())
    slots, _ = ctx.is_copy_schedule()
    toks = ctx.is_copy_tokens()
    ctx.close()
    del w
    torch.cuda.empty_cache()
    for step in range(3):
        for s, uid in enumerate(slots[step]):
            if uid < 0:
                continue
            got = sampler.sample_token_topp(dumps[step][s], SEED, 5 * G + int(uid), step, 0.8, 0.9)
            assert got == toks[uid, step], (step, s, uid)
