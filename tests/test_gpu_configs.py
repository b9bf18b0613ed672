"""Full-size GPU parity for BASELINE configs 2 (Qwen3-0.6B shape, G = 16, g = 4,
max 512) and 5 (Qwen3-4B shape, Hq/Hkv = 4, G = 64, g = 8, max 1024): other
hidden sizes and GQA ratios than config 3, i.e. other GEMM tilings and attention
instantiations.  One whole rollout each in bench.py's launch configuration: the
schedule is bit-exact against the oracle simulation, the sampler is bit-exact on
the dumped logits, and the first steps' logits match the oracle's teacher-forced
fp64 forward within the bf16 tolerance (R31)."""
import numpy as np
import pytest
import torch

from oracle import model as M
from oracle import sampler, simulator
from oracle import kv as okv
from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths

pytestmark = pytest.mark.gpu
SEED = 20261017
CASES = {
    "config2-0.6b": dict(shape="qwen3-0.6b", G=16, g=4, max_new=512, family="math8b", pid=7),
    "config5-4b": dict(shape="qwen3-4b", G=64, g=8, max_new=1024, family="math", pid=9),
}


@pytest.fixture(scope="module", params=sorted(CASES))
def run(request):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_22950_b200 import _lib
    c = CASES[request.param]
    shape, P = SHAPES[c["shape"]], 256
    w = gen_weights(shape, seed=SEED, device="cuda")
    kv_tok = okv.kv_bytes_per_token(shape.layers, shape.n_kv_heads, shape.head_dim)
    budget = (P - 1) * kv_tok + c["g"] * (c["max_new"] // 16) * 16 * kv_tok
    cfg = _lib.make_config(shape, c["G"], c["g"], c["max_new"], P, mode="infinite", page_tokens=16,
                           kv_budget_bytes=budget, eps=0.1, temperature=0.8, seed=SEED)
    ctx = _lib.Context(cfg, w)
    prompt = gen_prompt(shape.vocab, P, c["pid"], seed=SEED)
    true = gen_trace(c["family"], c["G"], c["max_new"], SEED + c["pid"])
    pred = predict_lengths(true, "noisy", 0.3, seed=SEED + c["pid"])
    ctx.is_prefill(torch.as_tensor(prompt, device="cuda"), c["pid"])
    ctx.is_start_group(true, pred)
    rc = ctx.is_query()["row_capacity"]
    dump = torch.zeros(rc, shape.vocab, device="cuda")
    ctx.is_set_logits_dump(dump)
    dumps = []
    for _ in range(3):
        ctx.is_decode_step()
        torch.cuda.synchronize()
        dumps.append(dump.cpu().numpy().copy())
    ctx.is_set_logits_dump(None)
    steps = ctx.is_run_group()
    res = dict(case=c, shape=shape, steps=steps, stats=ctx.is_query(), sched=ctx.is_copy_schedule(),
               tokens=ctx.is_copy_tokens(), logprobs=ctx.is_copy_logprobs(), dumps=dumps, true=true, pred=pred,
               prompt=prompt, budget=budget, w_cpu={k: v.cpu() for k, v in w.items()})
    ctx.close()
    del w
    torch.cuda.empty_cache()
    return res


def test_config_schedule_bit_exact(run):
    c = run["case"]
    ref = simulator.simulate(run["true"], "infinite", c["g"], pred=run["pred"], eps=0.1, page_tokens=16)
    slots, live = run["sched"]
    assert run["steps"] == ref.total_steps
    assert slots.tolist() == ref.slot_table and live.tolist() == ref.live_pages
    st = run["stats"]
    assert st["completed"] == c["G"] and st["error"] == 0
    assert st["peak_kv_bytes"] <= run["budget"]


def test_config_sampler_and_teacher_forced_logits(run):
    c, shape = run["case"], run["shape"]
    slots, _ = run["sched"]
    toks = run["tokens"]
    for step in range(3):
        for s, uid in enumerate(slots[step]):
            if uid >= 0:
                got = sampler.sample_token(run["dumps"][step][s], SEED, c["pid"] * c["G"] + int(uid), step)
                assert got == toks[uid, step], (step, s, uid)
    uid = int(slots[0][0])
    gen = [int(x) for x in toks[uid, :3]]
    z = M.teacher_forced_logits(run["w_cpu"], shape, run["prompt"], gen, mirror=True, rows=[0, 1, 2])
    for t in range(3):
        d = run["dumps"][t][0].astype(np.float64)
        rel = np.linalg.norm(d - z[t]) / np.linalg.norm(z[t])
        assert rel < 2e-2, (t, rel)
        assert np.max(np.abs(d - z[t])) <= 2e-2 * np.max(np.abs(z[t]))
    # log-probabilities of the first tokens from the kernel's own logits (NEXT-3)
    lp = run["logprobs"]
    for t in range(3):
        zz = run["dumps"][t][0].astype(np.float64)
        ref = zz[toks[uid, t]] - (zz.max() + np.log(np.sum(np.exp(zz - zz.max()))))
        assert abs(lp[uid, t] - ref) <= 1e-4
