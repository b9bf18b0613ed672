"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Tolerances (BASELINE.json north_star; R31): schedules, slot tables,
page counts and sampler decisions on identical logits are bit-exact;
kernel-level fp32-accumulation differences on identical bf16 inputs <= 1e-4
normwise; anything through bf16 storage (logits) <= 2e-2 normwise.
"""
import numpy as np
import pytest
import torch

from oracle import model as M
from oracle import sampler, simulator
from oracle import kv as okv
from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2506_22950_b200 import _lib
    _lib.load()
    return _lib


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


@pytest.mark.parametrize("M_,K,rows,split", [(4096, 2048, 8, 4), (64, 64, 3, 1), (1000, 2048, 40, 1),
                                             (1000, 2048, 40, 8), (12288, 2048, 64, 3), (2048, 6144, 16, 8),
                                             (384, 512, 17, 2)])
def test_gemm_tcgen05_vs_fp32_matmul(lib, M_, K, rows, split):
    g = torch.Generator(device="cuda").manual_seed(M_ + K + rows)
    w = (torch.randn(M_, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    x = torch.randn(rows, K, device="cuda", generator=g).to(torch.bfloat16)
    y = torch.full((rows, M_), float("nan"), device="cuda")
    lib.is_dbg_gemm(w, x, y, split=split)
    torch.cuda.synchronize()
    ref = (x.double() @ w.double().T).cpu().numpy()
    got = y.cpu().numpy()
    assert np.all(np.isfinite(got))
    for r in range(rows):
        assert _rel(got[r], ref[r]) < 1e-4, r


@pytest.mark.parametrize("M_,K,rows,split", [(2048, 2048, 16, 8), (4096, 2048, 16, 4), (12288, 2048, 16, 2),
                                             (2048, 6144, 16, 3)])
def test_gemm_splitk_deterministic(lib, M_, K, rows, split):
    """Split-K (gemm.cuh): each rank sums its column slice over the ranks' partials in rank
    order, so repeated launches give bit-identical outputs, within the 1e-4 kernel tolerance
    of the fp64 product."""
    g = torch.Generator(device="cuda").manual_seed(7 + M_ + split)
    w = (torch.randn(M_, K, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
    x = torch.randn(rows, K, device="cuda", generator=g).to(torch.bfloat16)
    outs = []
    for _ in range(6):
        y = torch.full((rows, M_), float("nan"), device="cuda")
        lib.is_dbg_gemm(w, x, y, split=split)
        outs.append(y)
    torch.cuda.synchronize()
    for y in outs[1:]:
        assert torch.equal(y, outs[0])
    ref = (x.double() @ w.double().T).cpu().numpy()
    got = outs[0].cpu().numpy()
    for r in range(rows):
        assert _rel(got[r], ref[r]) < 1e-4, r


# ---------------------------------------------------------------------------- tiny end to end
TINY = SHAPES["tiny"]
SEED = 20261017


def _tiny_setup():
    w = gen_weights(TINY, seed=SEED)
    prompt = gen_prompt(TINY.vocab, 16, 0, seed=SEED)
    true = gen_trace("tiny", 8, 32, 1)
    pred = predict_lengths(true, "noisy", 0.3, seed=1)
    return w, prompt, true, pred


def _run(lib, w_dev, prompt, true, pred, mode, g, budget=0, prefix_k=0, pt=16, rc=16, logits=False,
         target=0, top_p=1.0, eos_id=None):
    cfg = lib.make_config(TINY, len(true), g, 32, 16, mode=mode, prefix_k=prefix_k, page_tokens=pt, row_capacity=rc,
                          kv_budget_bytes=budget, eps=0.1, temperature=0.8, seed=SEED,
                          dynamic_target=target, top_p=top_p, eos_id=eos_id)
    ctx = lib.Context(cfg, w_dev)
    ctx.is_prefill(torch.as_tensor(prompt, device="cuda"), 0)
    ctx.is_start_group(true, pred)
    dumps = []
    if logits:
        buf = torch.zeros(rc, TINY.vocab, device="cuda")
        ctx.is_set_logits_dump(buf)
        slots_seen = []
        while ctx.is_query()["completed"] < (target or len(true)):
            # rows of the step about to run
            ctx.is_decode_step()
            torch.cuda.synchronize()
            dumps.append(buf.cpu().numpy().copy())
        steps = ctx.is_query()["steps"]
    else:
        steps = ctx.is_run_group()
    st = ctx.is_query()
    slots, live = ctx.is_copy_schedule()
    toks = ctx.is_copy_tokens()
    lps = ctx.is_copy_logprobs()
    ctx.close()
    return dict(steps=steps, stats=st, slots=slots, live=live, tokens=toks, dumps=dumps, logprobs=lps)


@pytest.fixture(scope="module")
def tiny(lib):
    w, prompt, true, pred = _tiny_setup()
    w_dev = {k: v.cuda() for k, v in w.items()}
    budget = okv.prefix_bytes(TINY, 16) + 4 * 2 * okv.page_bytes(TINY, 16)  # config 1: "KV budget 4 slots"
    runs = {m: _run(lib, w_dev, prompt, true, pred, m, 2, budget=budget)
            for m in ("naive", "fifo", "infinite", "fptas_only", "sjf_only", "infinite_slots")}
    runs["full"] = _run(lib, w_dev, prompt, true, pred, "full", 8)
    return dict(w=w, w_dev=w_dev, prompt=prompt, true=true, pred=pred, runs=runs, budget=budget)


@pytest.mark.parametrize("mode", ["naive", "fifo", "infinite", "full", "fptas_only", "sjf_only", "infinite_slots"])
def test_tiny_schedule_bit_exact(tiny, mode):
    r = tiny["runs"][mode]
    ref = simulator.simulate(tiny["true"], mode, 2, pred=tiny["pred"], eps=0.1, page_tokens=16)
    assert r["stats"]["completed"] == 8 and r["stats"]["error"] == 0
    assert r["steps"] == ref.total_steps
    assert r["slots"].tolist() == ref.slot_table
    assert r["live"].tolist() == ref.live_pages
    assert r["stats"]["peak_pages"] == ref.peak_pages
    assert r["stats"]["tokens_decoded"] == int(np.sum(tiny["true"]))
    assert r["stats"]["peak_kv_bytes"] == okv.peak_kv_bytes(TINY, 16, ref.peak_pages)
    if mode != "full":
        assert r["stats"]["peak_kv_bytes"] <= tiny["budget"]


def test_tiny_token_streams_identical_across_modes(tiny):
    """Batch invariance (R12 iv): a uid's tokens do not depend on the schedule."""
    base = tiny["runs"]["infinite"]["tokens"]
    for mode in ("naive", "fifo", "full", "fptas_only", "sjf_only", "infinite_slots"):
        assert np.array_equal(tiny["runs"][mode]["tokens"], base), mode
    for i, L in enumerate(tiny["true"]):
        assert np.all(base[i, :L] >= 0) and np.all(base[i, :L] < TINY.vocab) and np.all(base[i, L:] == -1)


def _dump_index(slots):
    """(uid, t) -> (step, slot) of a logged schedule."""
    at, t_of = {}, {}
    for step, row in enumerate(slots):
        for s, uid in enumerate(row):
            if uid < 0:
                continue
            t = t_of.get(int(uid), 0)
            at[(int(uid), t)] = (step, s)
            t_of[int(uid)] = t + 1
    return at


@pytest.fixture(scope="module")
def tiny_dump(lib, tiny):
    return _run(lib, tiny["w_dev"], tiny["prompt"], tiny["true"], tiny["pred"], "infinite", 2,
                budget=tiny["budget"], logits=True)


def test_tiny_teacher_forced_tokens_and_logits(tiny, tiny_dump):
    """Every generated token of config 1 against the oracle's teacher-forced logits
    (SURVEY C12 ii/iii, C31): the GPU logits of that step within 2e-2 normwise and
    max-abs <= 2e-2 * max|z|; the token equal to the oracle's draw unless the oracle's
    top-2 score margin is below 2 * (1/T) * max|dz| (a near tie the bf16 logits may flip)."""
    r = tiny_dump
    toks = r["tokens"]
    at = _dump_index(r["slots"])
    mism, total = 0, 0
    for i, L in enumerate(tiny["true"]):
        gen = [int(x) for x in toks[i, :L]]
        z = M.teacher_forced_logits(tiny["w"], TINY, tiny["prompt"], gen, mirror=True)
        for t in range(L):
            step, s = at[(i, t)]
            d = r["dumps"][step][s].astype(np.float64)
            mabs = np.max(np.abs(d - z[t]))
            assert _rel(d, z[t]) < 2e-2, (i, t)
            assert mabs <= 2e-2 * np.max(np.abs(z[t])), (i, t, mabs)
            tok, margin = sampler.sample_margin(z[t].astype(np.float32), SEED, i, t)
            total += 1
            if tok != gen[t]:
                mism += 1
                assert margin < 2 * 1.25 * mabs, (i, t, margin, mabs)
    assert total == int(np.sum(tiny["true"]))
    assert mism <= max(1, total // 100)


def test_tiny_sampler_bit_exact_on_dumped_logits(tiny, tiny_dump):
    """The sampler on the kernel's own fp32 logits equals the oracle sampler bit for bit
    (SURVEY C12 i), every step and slot."""
    r = tiny_dump
    toks = r["tokens"]
    for (uid, t), (step, s) in _dump_index(r["slots"]).items():
        got = sampler.sample_token(r["dumps"][step][s], SEED, uid, t)
        assert got == toks[uid, t], (step, s, uid, t)


def test_tiny_budget_error_and_prefix_phase(lib, tiny):
    with pytest.raises(lib.InfsampError) as e:
        cfg = lib.make_config(TINY, 8, 2, 32, 16, mode="infinite", prefix_k=4, page_tokens=16,
                              kv_budget_bytes=tiny["budget"])
        lib.Context(cfg, tiny["w_dev"])
    assert e.value.status == lib.IS_ERR_BUDGET
    pred = predict_lengths(tiny["true"], "noisy", 0.3, seed=1, prefix_k=4)
    r = _run(lib, tiny["w_dev"], tiny["prompt"], tiny["true"], pred, "infinite", 2, budget=tiny["budget"],
             prefix_k=4, pt=4)
    ref = simulator.simulate(tiny["true"], "infinite", 2, pred=pred, eps=0.1, prefix_k=4, page_tokens=4)
    assert r["steps"] == ref.total_steps
    assert r["slots"].tolist() == ref.slot_table
    assert r["live"].tolist() == ref.live_pages
    assert r["stats"]["prefix_steps"] == ref.prefix_steps
    assert np.array_equal(r["tokens"], tiny["runs"]["infinite"]["tokens"])


def test_tiny_rewards_and_advantages(lib, tiny):
    from oracle import grpo
    cfg = lib.make_config(TINY, 8, 2, 32, 16, mode="infinite", kv_budget_bytes=tiny["budget"], seed=SEED)
    ctx = lib.Context(cfg, tiny["w_dev"])
    ctx.is_prefill(torch.as_tensor(tiny["prompt"], device="cuda"), 0)
    ctx.is_start_group(tiny["true"], tiny["pred"])
    ctx.is_run_group()
    rew = torch.zeros(8, device="cuda")
    ln = torch.zeros(8, dtype=torch.int32, device="cuda")
    ctx.is_group_results(rew, ln)
    toks = ctx.is_copy_tokens()
    ctx.close()
    ref = [grpo.bench_reward(toks[i, :L].tolist(), TINY.vocab) for i, L in enumerate(tiny["true"])]
    assert np.allclose(rew.cpu().numpy(), ref, atol=1e-7)
    assert ln.cpu().tolist() == [int(x) for x in tiny["true"]]
    adv = lib.is_group_advantages(rew.cpu().numpy())
    assert np.allclose(adv, grpo.advantages(ref), atol=1e-5)


def test_tiny_context_reused_across_prompts(lib, tiny):
    """The decode step is one CUDA graph per context, replayed for every prompt: prompt 1
    decoded after prompt 0 in the same context must equal prompt 1 in a fresh context
    (RNG uids prompt_id*G + i and the first input token come from device state)."""
    w_dev = tiny["w_dev"]
    p1 = gen_prompt(TINY.vocab, 16, 1, seed=SEED)
    true1 = gen_trace("tiny", 8, 32, 2)
    pred1 = predict_lengths(true1, "noisy", 0.3, seed=2)

    def mk():
        cfg = lib.make_config(TINY, 8, 2, 32, 16, mode="infinite", kv_budget_bytes=tiny["budget"], seed=SEED)
        return lib.Context(cfg, w_dev)

    a = mk()
    a.is_prefill(torch.as_tensor(tiny["prompt"], device="cuda"), 0)
    a.is_start_group(tiny["true"], tiny["pred"])
    a.is_run_group()
    a.is_prefill(torch.as_tensor(p1, device="cuda"), 1)
    a.is_start_group(true1, pred1)
    a.is_run_group()
    reused = a.is_copy_tokens()
    a.close()
    b = mk()
    b.is_prefill(torch.as_tensor(p1, device="cuda"), 1)
    b.is_start_group(true1, pred1)
    b.is_run_group()
    fresh = b.is_copy_tokens()
    b.close()
    assert np.array_equal(reused, fresh)
    # and prompt 1's stream is its own (uid base 1*G), not a replay of prompt 0's RNG
    z = M.teacher_forced_logits(tiny["w"], TINY, p1, [int(x) for x in fresh[0, :2]], mirror=True, rows=[0])[0]
    tok, margin = sampler.sample_margin(z.astype(np.float32), SEED, 1 * 8 + 0, 0)
    assert tok == fresh[0, 0] or margin < 0.05


def test_nccl_allgather_results_single_rank(lib, tiny):
    """The C-ABI NCCL exchange (a9) on a one-rank communicator: the gathered arrays
    are the rank's own (length, reward) per sample, in order."""
    try:
        uid = lib.nccl_unique_id()
    except lib.InfsampError as e:
        pytest.skip(f"no NCCL: {e}")
    comm = lib.nccl_comm_init(uid, 0, 1)
    cfg = lib.make_config(TINY, 8, 2, 32, 16, mode="infinite", kv_budget_bytes=tiny["budget"], seed=SEED)
    ctx = lib.Context(cfg, tiny["w_dev"])
    ctx.is_prefill(torch.as_tensor(tiny["prompt"], device="cuda"), 0)
    ctx.is_start_group(tiny["true"], tiny["pred"])
    ctx.is_run_group()
    rew = torch.zeros(8, device="cuda")
    ln = torch.zeros(8, dtype=torch.int32, device="cuda")
    ctx.is_group_results(rew, ln)
    all_rew = torch.full((8,), -1.0, device="cuda")
    all_len = torch.full((8,), -1, dtype=torch.int32, device="cuda")
    ctx.is_allgather_results(comm, ln, rew, all_len, all_rew)
    torch.cuda.synchronize()
    ctx.close()
    lib.nccl_comm_destroy(comm)
    assert all_len.cpu().tolist() == ln.cpu().tolist() == [int(x) for x in tiny["true"]]
    assert torch.equal(all_rew.cpu(), rew.cpu())


def _log_softmax64(z):
    z = np.asarray(z, np.float64)
    m = z.max()
    return z - (m + np.log(np.sum(np.exp(z - m))))


def test_tiny_logprobs(lib, tiny, tiny_dump):
    """NEXT-3: log pi(token) emitted by the lm_head/sampler path equals the exact fp64
    log-softmax of the kernel's own logits (1e-4, R31's fp32-accumulation class) and the
    oracle's teacher-forced one within 2 max|dz| (the logits tolerance propagated)."""
    r = tiny_dump
    toks, lps = r["tokens"], r["logprobs"]
    t_of, checked = {}, 0
    for step, row in enumerate(r["slots"]):
        for s, uid in enumerate(row):
            if uid < 0:
                continue
            t = t_of.get(uid, 0)
            tok = int(toks[uid, t])
            own = _log_softmax64(r["dump" + "s"][step][s])[tok]
            assert abs(lps[uid, t] - own) <= 1e-4, (step, uid, t, lps[uid, t], own)
            if t == 0 or step % 7 == 0:
                gen = [int(x) for x in toks[uid, :t + 1]]
                z = M.teacher_forced_logits(tiny["w"], TINY, tiny["prompt"], gen, mirror=True, rows=[t])[0]
                dz = np.max(np.abs(np.asarray(r["dumps"][step][s], np.float64) - z))
                assert abs(lps[uid, t] - _log_softmax64(z)[tok]) <= 2 * dz + 1e-5, (uid, t)
                checked += 1
            t_of[uid] = t + 1
    assert checked > 0
    for i, L in enumerate(tiny["true"]):
        assert np.all(lps[i, :L] < 0) and np.all(lps[i, L:] == 0)
    from oracle import grpo
    # P:311 reward and Eq. 3 value on the emitted log-probs (reference model = the tokens'
    # own log-probs shifted by a per-sample constant, so the KL sum has a closed form)
    G = len(tiny["true"])
    lens = np.asarray(tiny["true"], np.int32)
    rm = np.linspace(-1, 1, G).astype(np.float32)
    shift = np.float32(0.125)
    lref = (lps - shift).astype(np.float32)
    kr = lib.is_kl_rewards(rm, lps, lref, lens, 0.5)
    assert np.allclose(kr, rm - 0.5 * shift * lens, atol=1e-5)
    assert np.array_equal(kr, np.float32(grpo.kl_rewards(rm.astype(np.float64), lps.astype(np.float64),
                                                         lref.astype(np.float64), lens, 0.5)))
    adv = lib.is_group_advantages(kr, "mean_only")
    j = lib.is_grpo_objective(lps, lps, lps, adv, lens, 0.2, 0.04)
    assert abs(j - float(np.mean(adv.astype(np.float64)))) < 1e-9


def test_profile_hooks_then_decode_unchanged(lib, tiny):
    """bench.py's timing hooks (is_profile_kernel, is_profile_step[_graph]) run on a live
    context; a group started afterwards decodes the same tokens as an undisturbed run."""
    cfg = lib.make_config(TINY, 8, 2, 32, 16, mode="infinite", kv_budget_bytes=tiny["budget"], eps=0.1,
                          temperature=0.8, seed=SEED)
    ctx = lib.Context(cfg, tiny["w_dev"])
    ctx.is_prefill(torch.as_tensor(tiny["prompt"], device="cuda"), 0)
    ctx.is_start_group(tiny["true"], tiny["pred"])
    ctx.is_decode_step()
    for kind in (1, 3, 4, 5, 6):
        ms, n = ctx.is_profile_kernel(kind, reps=2)
        assert n == (2 if kind == 3 else 1) * 2 * TINY.layers and 0 < ms < 1.0, (kind, ms, n)
    with pytest.raises(lib.InfsampError) as e:
        ctx.is_profile_kernel(7)
    assert e.value.status == lib.IS_ERR_CONFIG
    for graph in (False, True):
        ms, kind = ctx.is_profile_step(graph=graph)
        assert len(ms) == len(kind) > 0 and np.all(ms >= 0) and 5 in set(kind.tolist())
    ctx.is_prefill(torch.as_tensor(tiny["prompt"], device="cuda"), 0)
    ctx.is_start_group(tiny["true"], tiny["pred"])
    ctx.is_run_group()
    toks = ctx.is_copy_tokens()
    ctx.close()
    assert np.array_equal(toks, tiny["runs"]["infinite"]["tokens"])


@pytest.mark.parametrize("target", [5, 8])
def test_tiny_dynamic_slot_mode(lib, tiny, target):
    """NEXT-2 dynamic-slot sampling (R35): the 8 samples are candidates in
    trace order; the run stops at the target-th completion and discards in-flight work.
    Slot table, page log, discards and counters equal the oracle's simulation; completed
    samples' tokens equal the same uids' tokens under every other schedule."""
    r = _run(lib, tiny["w_dev"], tiny["prompt"], tiny["true"], tiny["pred"], "dynamic", 2,
             budget=tiny["budget"], target=target)
    ref = simulator.simulate(tiny["true"], "dynamic", 2, page_tokens=16, target=target)
    st = r["stats"]
    assert st["completed"] == target and st["error"] == 0 and st["discarded"] == len(ref.discarded)
    assert r["steps"] == ref.total_steps
    assert r["slots"].tolist() == ref.slot_table
    assert r["live"].tolist() == ref.live_pages
    assert st["live_pages"] == 0 and st["peak_pages"] == ref.peak_pages
    assert st["tokens_decoded"] == ref.tokens_decoded
    base = tiny["runs"]["infinite"]["tokens"]
    for uid in ref.finish_step:
        assert np.array_equal(r["tokens"][uid], base[uid]), uid


@pytest.mark.parametrize("top_p", [0.9, 0.5, 0.05])
def test_tiny_topp_sampler_bit_exact(lib, tiny, top_p):
    """NEXT-4 top-p (R36): every token equals the oracle's nucleus Gumbel-max draw on the
    kernel's own dumped logits, bit-exactly; log pi(token) stays the full-softmax value
    (R33); the schedule is unchanged."""
    r = _run(lib, tiny["w_dev"], tiny["prompt"], tiny["true"], tiny["pred"], "infinite", 2,
             budget=tiny["budget"], logits=True, top_p=top_p)
    assert r["slots"].tolist() == tiny["runs"]["infinite"]["slots"].tolist()
    toks, lps = r["tokens"], r["logprobs"]
    t_of, n, in_nucleus_only = {}, 0, 0
    for step, row in enumerate(r["slots"]):
        for s, uid in enumerate(row):
            if uid < 0:
                continue
            t = t_of.get(uid, 0)
            z = r["dumps"][step][s]
            got = sampler.sample_token_topp(z, SEED, int(uid), t, 0.8, top_p)
            assert got == toks[uid, t], (step, s, uid, t)
            assert abs(lps[uid, t] - _log_softmax64(z)[got]) <= 1e-4
            in_nucleus_only += got != sampler.sample_token(z, SEED, int(uid), t, 0.8)
            t_of[uid] = t + 1
            n += 1
    assert n == int(np.sum(tiny["true"]))
    if top_p <= 0.5:
        assert in_nucleus_only > 0      # the nucleus actually changed some draws


@pytest.mark.parametrize("case", ["random", "all_equal", "quantised", "dominant", "vocab_151936"])
def test_topp_chain_edge_cases_bit_exact(lib, case):
    """The top-p kernels alone (is_dbg_topp) on synthetic logits with the edge cases of R36:
    every element tied, a few quantised levels (ties at the boundary), one dominant logit,
    and the full Qwen3 vocabulary; tokens equal the oracle's bit for bit."""
    rng = np.random.default_rng({"random": 1, "all_equal": 2, "quantised": 3, "dominant": 4,
                                 "vocab_151936": 5}[case])
    rows, V = (8, 151936) if case == "vocab_151936" else (16, 4096)
    z = rng.normal(size=(rows, V)).astype(np.float32) * np.float32(2.0)
    if case == "all_equal":
        z[:] = 0.0
    elif case == "quantised":
        z = (np.round(z * 2) / 2).astype(np.float32)
    elif case == "dominant":
        z[:, 7] = 20.0
    uid = np.arange(rows, dtype=np.int32) * 3 + 1
    t = np.arange(rows, dtype=np.int32) + 5
    for top_p in (0.05, 0.3, 0.9, 0.999):
        got = lib.is_dbg_topp(torch.as_tensor(z, device="cuda"), torch.as_tensor(uid, device="cuda"),
                              torch.as_tensor(t, device="cuda"), 0.8, top_p, SEED).cpu().numpy()
        for r in range(rows):
            ref = sampler.sample_token_topp(z[r], SEED, int(uid[r]), int(t[r]), 0.8, top_p)
            assert got[r] == ref, (case, top_p, r, got[r], ref)
        if case == "all_equal":   # nucleus = the first ceil(top_p * V) ids
            k = -(-int(np.ceil(float(np.float32(top_p)) * float(V * 2 ** 44))) // 2 ** 44)
            assert np.all(got < k)
        if case == "dominant" and top_p < 0.9:
            assert np.all(got == 7)


def test_tiny_eos_termination(lib, tiny):
    """R37 (SURVEY a8 "or token == eos if enabled"): with eos_id set, a sample stops at its first
    eos token.  Tokens are schedule-independent (batch invariance), so the effective lengths
    follow from the trace-driven run; the schedule then equals the oracle simulation on those
    lengths, tokens are the trace-driven ones truncated, and is_group_results reports them."""
    base = tiny["runs"]["infinite"]["tokens"]
    true = np.asarray(tiny["true"])
    eos = int(base[0, min(3, true[0] - 1)])
    eff = []
    for i, L in enumerate(true):
        hit = np.nonzero(base[i, :L] == eos)[0]
        eff.append(int(hit[0]) + 1 if len(hit) else int(L))
    assert eff[0] < true[0] or true[0] <= 4
    r = _run(lib, tiny["w_dev"], tiny["prompt"], tiny["true"], tiny["pred"], "infinite", 2,
             budget=tiny["budget"], eos_id=eos)
    ref = simulator.simulate(eff, "infinite", 2, pred=tiny["pred"], eps=0.1, page_tokens=16)
    assert r["stats"]["completed"] == 8 and r["stats"]["error"] == 0
    assert r["slots"].tolist() == ref.slot_table and r["live"].tolist() == ref.live_pages
    assert r["stats"]["tokens_decoded"] == sum(eff)
    for i, L in enumerate(eff):
        assert np.array_equal(r["tokens"][i, :L], base[i, :L]) and np.all(r["tokens"][i, L:] == -1)
    # is_group_results reports the emitted lengths and the reward over the truncated text
    from oracle import grpo
    cfg = lib.make_config(TINY, 8, 2, 32, 16, mode="infinite", kv_budget_bytes=tiny["budget"], seed=SEED,
                          eos_id=eos)
    ctx = lib.Context(cfg, tiny["w_dev"])
    ctx.is_prefill(torch.as_tensor(tiny["prompt"], device="cuda"), 0)
    ctx.is_start_group(tiny["true"], tiny["pred"])
    ctx.is_run_group()
    rew = torch.zeros(8, device="cuda")
    ln = torch.zeros(8, dtype=torch.int32, device="cuda")
    ctx.is_group_results(rew, ln)
    ctx.close()
    assert ln.cpu().tolist() == eff
    ref = [grpo.bench_reward(base[i, :L].tolist(), TINY.vocab) for i, L in enumerate(eff)]
    assert np.allclose(rew.cpu().numpy(), ref, atol=1e-7)
    with pytest.raises(lib.InfsampError) as e:
        lib.Context(lib.make_config(TINY, 8, 2, 32, 16, mode="infinite", prefix_k=4, page_tokens=4,
                                    eos_id=eos), tiny["w_dev"])
    assert e.value.status == lib.IS_ERR_CONFIG


def test_tiny_row_capacity_32_decode_path(lib, tiny):
    """row_capacity >= 32 (co-resident groups' row counts) selects the 64-token suffix units with
    the separate merge kernel: schedule, sampler on dumped logits (bit-exact) and
    teacher-forced logits (2e-2) against the oracle."""
    r = _run(lib, tiny["w_dev"], tiny["prompt"], tiny["true"], tiny["pred"], "infinite", 2,
             budget=tiny["budget"], logits=True, rc=32)
    ref = simulator.simulate(tiny["true"], "infinite", 2, pred=tiny["pred"], eps=0.1, page_tokens=16)
    assert r["slots"].tolist() == ref.slot_table and r["stats"]["completed"] == 8
    toks, t_of, checked = r["tokens"], {}, 0
    for step, row in enumerate(r["slots"]):
        for s, uid in enumerate(row):
            if uid < 0:
                continue
            t = t_of.get(uid, 0)
            assert sampler.sample_token(r["dumps"][step][s], SEED, int(uid), t) == toks[uid, t]
            if t == 0 or step % 6 == 0:
                gen = [int(x) for x in toks[uid, :t + 1]]
                z = M.teacher_forced_logits(tiny["w"], TINY, tiny["prompt"], gen, mirror=True, rows=[t])[0]
                assert _rel(r["dumps"][step][s], z) < 2e-2
                assert np.max(np.abs(r["dumps"][step][s] - z)) <= 2e-2 * np.max(np.abs(z))
                checked += 1
            t_of[uid] = t + 1
    assert checked > 0


def test_tiny_bin_slots_with_prefix_phase(lib, tiny):
    """bin_mode = slots after a k = 4 prefix phase (phase 1 runs Alg. 2 over g bins
    on the materialised predictions; heads skip samples finished in the prefix phase, R38):
    the schedule equals the oracle simulation and the tokens the trace-driven ones."""
    pred = predict_lengths(tiny["true"], "noisy", 0.3, seed=1, prefix_k=4)
    r = _run(lib, tiny["w_dev"], tiny["prompt"], tiny["true"], pred, "infinite_slots", 2, budget=tiny["budget"],
             prefix_k=4, pt=4)
    ref = simulator.simulate(tiny["true"], "infinite_slots", 2, pred=pred, eps=0.1, prefix_k=4, page_tokens=4)
    assert r["steps"] == ref.total_steps and r["stats"]["prefix_steps"] == ref.prefix_steps
    assert r["slots"].tolist() == ref.slot_table
    assert r["live"].tolist() == ref.live_pages
    assert np.array_equal(r["tokens"], tiny["runs"]["infinite"]["tokens"])


@pytest.mark.parametrize("extra_pages,S,pred_noise", [(3, 4, 0.3), (1, 3, 0.6), (0, 4, 0.3), (6, 6, 0.8)])
def test_tiny_memory_aware_admission(lib, tiny, extra_pages, S, pred_noise):
    """Memory-aware admission (NEXT-2, DESIGN R41): g = 2 guaranteed slots + S - 2 elastic ones
    sharing `extra_pages` pages beyond the R25 reservation.  The schedule (slot table with stalls
    logged as -2 - uid, pages held per step), the stall count and peak KV equal the oracle's
    simulate_admit; every sample's tokens equal the plain infinite run's (batch invariance)."""
    true = tiny["true"]
    pred = predict_lengths(true, "noisy", pred_noise, seed=3)
    pb = okv.page_bytes(TINY, 16)
    budget = tiny["budget"] + extra_pages * pb
    cfg = lib.make_config(TINY, 8, 2, 32, 16, mode="infinite", page_tokens=16, kv_budget_bytes=budget, eps=0.1,
                          temperature=0.8, seed=SEED, admit_slots=S)
    ctx = lib.Context(cfg, tiny["w_dev"])
    ctx.is_prefill(torch.as_tensor(tiny["prompt"], device="cuda"), 0)
    ctx.is_start_group(true, pred)
    steps = ctx.is_run_group()
    st = ctx.is_query()
    slots, live = ctx.is_copy_schedule()
    toks = ctx.is_copy_tokens()
    ctx.close()
    pool = st["num_pages"]
    ref = simulator.simulate_admit(true, 2, S, pred, max_new=32, pool_pages=pool, page_tokens=16)
    assert steps == ref.total_steps
    assert slots.tolist() == ref.slot_table
    assert live.tolist() == ref.live_pages
    assert st["stalls"] == ref.stalls and st["peak_pages"] == ref.peak_pages and st["error"] == 0
    assert st["peak_kv_bytes"] <= budget
    assert np.array_equal(toks, tiny["runs"]["infinite"]["tokens"])
