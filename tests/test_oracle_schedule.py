"""Pins for oracle/planner.py, oracle/simulator.py, oracle/grpo.py, oracle/kv.py."""
import math

import numpy as np
import pytest

from conftest import load_golden
from oracle import grpo, kv, planner, simulator
from synth import SHAPES, gen_trace, predict_lengths

SPEC = load_golden("spec_examples.json")
APPC = load_golden("schedules_appC.json")


@pytest.mark.parametrize("ex", SPEC["fptas"])
def test_fptas_spec_examples(ex):
    p = planner.fptas_plan(ex["pred"], ex["N"], ex["eps"])
    assert p["K"] == pytest.approx(ex["K"], rel=1e-12)
    assert p["scaled"] == ex["scaled"]
    assert p["capacity"] == ex["capacity"]
    assert p["overflow"] == ex["overflow"]
    if "mask" in ex:
        assert [list(m) for m in p["mask"]] == ex["mask"]
    if "loads" in ex:
        assert p["loads"] == ex["loads"]
    if "group_of" in ex:
        assert [m[0] for m in p["mask"]] == ex["group_of"]


def _random_instances(n, seed, gmax=10):
    rng = np.random.default_rng(seed)
    for _ in range(n):
        N = int(rng.integers(1, 5))
        G = int(rng.integers(N, gmax + 1))
        lens = [int(x) for x in np.clip(np.round(np.exp(rng.normal(3, 0.8, G))), 1, 200)]
        eps = float(rng.choice([0.05, 0.1, 0.2, 0.5, 1.0]))
        yield lens, N, eps


def test_fptas_invariants_and_derived_bound():
    """Bijection; SPEC l.157 load bounds; DESIGN R16 bound (S/N)(1 + eps(G/N + 1))."""
    ratios = []
    for lens, N, eps in _random_instances(600, 0):
        p = planner.fptas_plan(lens, N, eps)
        G = len(lens)
        # bijection onto {(n, 0..|G_n|-1)}
        seen = {}
        for i, (n, j) in enumerate(p["mask"]):
            seen.setdefault(n, []).append(j)
        for n, js in seen.items():
            assert sorted(js) == list(range(len(js)))
        assert sum(len(v) for v in seen.values()) == G
        # scaled-load bounds
        for n in range(N):
            load = sum(p["scaled"][i] for i in p["groups"][n])
            assert load == p["loads"][n]
            if not p["overflow"]:
                assert load <= p["capacity"]
            else:
                assert load <= p["capacity"] + max(p["scaled"])
        # provable true-length bound without overflow
        if not p["overflow"]:
            S = sum(lens)
            worst = max(sum(lens[i] for i in grp) for grp in p["groups"])
            assert worst <= (S / N) * (1 + eps * (G / N + 1)) + 1e-9
        if G <= 8:
            opt = planner.optimal_partition_bruteforce(lens, N)
            ratios.append(max(sum(lens[i] for i in grp) for grp in p["groups"]) / opt)
    # Reported, not asserted (R16: Alg. 2 has no (1+eps) guarantee); sanity only.
    assert min(ratios) >= 1.0


def test_fptas_counterexample_to_one_plus_eps():
    """DESIGN R16: Alg. 2 verbatim is NOT within (1+eps) of OPT on this instance."""
    p = planner.fptas_plan([3, 3, 2, 2, 2, 2], 2, 0.1)
    loads = sorted(sum([3, 3, 2, 2, 2, 2][i] for i in g) for g in p["groups"])
    assert loads == [6, 8]
    assert planner.optimal_partition_bruteforce([3, 3, 2, 2, 2, 2], 2) == 7


def test_fptas_config_errors():
    with pytest.raises(planner.PlanError):
        planner.fptas_plan([1, 2], 0, 0.1)
    with pytest.raises(planner.PlanError):
        planner.fptas_plan([1, 2], 2, 0.0)
    with pytest.raises(planner.PlanError):
        planner.fptas_plan([1, 0], 2, 0.1)


def test_sjf_examples_and_static_queue():
    assert planner.sjf_refill([50, 20, 90], set(), set()) == 1
    assert planner.sjf_refill([50, 20, 90], {1}, {0, 2}) is None
    assert planner.sjf_refill([30, 30], set(), set()) == 0
    rng = np.random.default_rng(3)
    for _ in range(50):
        G, g = 16, 4
        pred = [int(x) for x in rng.integers(1, 50, G)]
        fin = set(int(x) for x in rng.choice(G, 3, replace=False))
        plan = planner.build_plan("infinite", G, g, pred=pred, eps=0.1, finished=fin)
        # queue = remaining unfinished samples sorted by (pred, id)
        rest = [i for i in range(G) if i not in fin and i not in plan["init"]]
        assert plan["queue"] == sorted(rest, key=lambda i: (pred[i], i))
        assert not set(plan["queue"]) & fin


def test_lpt_and_optimal_makespan():
    for ex in SPEC["lpt"]:
        assert planner.lpt_plan(ex["lengths"], ex["g"])[1] == ex["makespan"]
    for ex in SPEC["opt"]:
        assert planner.optimal_makespan(ex["lengths"], ex["g"]) == ex["makespan"]
    rng = np.random.default_rng(4)
    for _ in range(200):
        n, g = int(rng.integers(1, 7)), int(rng.integers(1, 4))
        lens = [int(x) for x in rng.integers(1, 20, n)]
        opt = planner.optimal_makespan(lens, g)
        assert opt == planner.optimal_makespan_bruteforce(lens, g)
        assert opt <= planner.lpt_plan(lens, g)[1] <= sum(lens)
        assert opt >= max(max(lens), -(-sum(lens) // g))
    with pytest.raises(planner.PlanError):
        planner.optimal_makespan(list(range(1, 20)), 2)


def test_simulate_spec_examples():
    ex = SPEC["simulate_5342"]
    for mode in ("full", "naive", "fifo", "infinite"):
        r = simulator.simulate(ex["lengths"], mode, ex["g"], pred=ex["lengths"], eps=ex["eps"])
        assert r.total_steps == ex[mode], mode
    for lb in SPEC["lower_bound"]:
        assert simulator.step_lower_bound(lb["lengths"], lb["g"]) == lb["lb"]


@pytest.mark.parametrize("case", sorted(APPC["cases"]))
def test_golden_schedules_appendix_c(case):
    c = APPC["cases"][case]
    r = simulator.simulate(APPC["true_len"], c["mode"], APPC["g"], pred=c["pred"], eps=c["eps"],
                           prefix_k=c["prefix_k"], page_tokens=APPC["page_tokens"])
    assert r.total_steps == c["total_steps"]
    assert r.peak_pages == c["peak_pages"]
    assert r.slot_table == c["slot_table"]
    assert r.live_pages == c["live_pages"]
    assert r.init == c["init"] and r.queue == c["queue"]
    if "K" in c:
        assert r.plan["K"] == c["K"] and r.plan["scaled"] == c["scaled"]
        assert r.plan["capacity"] == c["capacity"] and r.plan["loads"] == c["loads"]
        assert [list(m) for m in r.plan["mask"]] == c["mask"]
    if "prefix_steps" in c:
        assert r.prefix_steps == c["prefix_steps"]
    assert simulator.simulate(APPC["true_len"], "naive", APPC["g"]).total_steps == APPC["naive_steps"]


def test_simulation_invariants_random():
    rng = np.random.default_rng(5)
    for _ in range(150):
        g = int(rng.integers(1, 4))
        G = g * int(rng.integers(1, 5))
        lens = [int(x) for x in rng.integers(1, 15, G)]
        pred = predict_lengths(lens, "noisy", 0.3, seed=int(rng.integers(1 << 30)))
        opt = planner.optimal_makespan(lens, g) if G <= 12 else None
        for mode in ("naive", "fifo", "infinite", "full", "fptas_only", "sjf_only"):
            r = simulator.simulate(lens, mode, g, pred=pred, eps=0.1, page_tokens=4)
            gg = G if mode == "full" else g
            assert r.total_steps >= simulator.step_lower_bound(lens, gg)
            if opt is not None and mode != "full":
                assert opt <= r.total_steps
            # token conservation
            assert r.tokens_decoded == sum(lens)
            assert sum(sum(1 for u in row if u >= 0) for row in r.slot_table) == sum(lens)
            # every sample runs contiguously for exactly its length
            for u in range(G):
                assert r.finish_step[u] - r.start_step[u] + 1 == lens[u]
        naive = simulator.simulate(lens, "naive", g)
        assert naive.total_steps == sum(max(lens[i:i + g]) for i in range(0, G, g))
        assert simulator.simulate(lens, "full", g).total_steps == max(lens)
        fifo = simulator.simulate(lens, "fifo", g)
        per_slot = [0] * g
        for (_, s, _, kind) in fifo.events:
            if kind == "finish":
                per_slot[s] += 1
        assert all(c <= G // g for c in per_slot) and sum(per_slot) == G


def test_constant_length_peaks_closed_form():
    """constant L: naive peak = g*ceil(L/pt) pages, full = G*ceil(L/pt)."""
    for G, g, L, pt in [(8, 2, 10, 4), (16, 4, 33, 16), (32, 8, 64, 16)]:
        lens = [L] * G
        assert simulator.simulate(lens, "naive", g, page_tokens=pt).peak_pages == g * math.ceil(L / pt)
        assert simulator.simulate(lens, "full", g, page_tokens=pt).peak_pages == G * math.ceil(L / pt)


def test_prefix_phase_accounting():
    rng = np.random.default_rng(6)
    for _ in range(50):
        g, G, k = 2, 8, int(rng.integers(1, 6))
        lens = [int(x) for x in rng.integers(1, 20, G)]
        pred = predict_lengths(lens, "noisy", 0.3, seed=1, prefix_k=k)
        r = simulator.simulate(lens, "infinite", g, pred=pred, eps=0.1, prefix_k=k, page_tokens=4)
        assert r.prefix_steps == sum(min(k, max(lens[i:i + g])) for i in range(0, G, g))
        assert r.tokens_decoded == sum(lens)


def test_budget_reservation_config1():
    """SURVEY §8(d) cfg 1: 4-slot budget = 292,864 B; k=4 with 16-token pages -> 358,400 B."""
    s = SHAPES["tiny"]
    pb, pre = kv.page_bytes(s, 16), kv.prefix_bytes(s, 16)
    budget = pre + 4 * 2 * pb
    assert budget == 292_864
    assert planner.reservation_bytes(8, 2, 32, 0, 16, pb, pre) <= budget
    assert planner.reservation_bytes(8, 2, 32, 4, 16, pb, pre) == 358_400
    assert planner.reservation_bytes(8, 2, 32, 4, 4, kv.page_bytes(s, 4), pre) == 210_944


def test_kv_bytes_spec_examples():
    for ex in SPEC["kv_bytes"]:
        assert kv.kv_bytes_per_token(ex["layers"], ex["kv_heads"], ex["head_dim"], ex["bytes"]) == ex["out"]


def test_advantages():
    for ex in SPEC["advantages"]:
        a = grpo.advantages(ex["r"], ex["mode"])
        assert np.allclose(a, ex["A"], atol=ex["tol"] + 1e-15)
    rng = np.random.default_rng(7)
    for _ in range(100):
        r = list(rng.normal(size=int(rng.integers(2, 64))))
        for mode in ("std_norm", "mean_only"):
            a = grpo.advantages(r, mode)
            assert abs(sum(a)) < 1e-9
            b = grpo.advantages([x + 3.5 for x in r], mode)
            assert np.allclose(a, b, atol=1e-9)
        s = grpo.advantages(r, "std_norm")
        assert abs(np.mean(np.square(s)) - 1.0) < 1e-9      # unit population variance


def test_kl_rewards_pins():
    """r = RM - beta * log(pi_theta(O|x) / pi_ref(O|x))."""
    rng = np.random.default_rng(11)
    G, T = 6, 9
    rm = list(rng.normal(size=G))
    lp = np.log(rng.uniform(0.05, 1.0, size=(G, T)))
    lr = np.log(rng.uniform(0.05, 1.0, size=(G, T)))
    lens = [int(x) for x in rng.integers(1, T + 1, size=G)]
    assert grpo.kl_rewards(rm, lp, lr, lens, 0.0) == rm                   # beta = 0 -> RM
    assert grpo.kl_rewards(rm, lp, lp, lens, 0.3) == rm                   # pi_theta = pi_ref -> RM
    # the sequence probability is the product of the token probabilities (chain rule)
    r = grpo.kl_rewards(rm, lp, lr, lens, 0.25)
    for i in range(G):
        p = np.prod(np.exp(lp[i, :lens[i]]))
        q = np.prod(np.exp(lr[i, :lens[i]]))
        assert abs(r[i] - (rm[i] - 0.25 * math.log(p / q))) < 1e-12
    assert grpo.kl_rewards([1.0], [[-1.0, -1.0, float("nan")]], [[-2.0, -2.0, 0.0]], [2], 0.1) == [1.0 - 0.1 * 2.0]
    a, b = grpo.kl_rewards(rm, lp, lr, lens, 0.1), grpo.kl_rewards(rm, lp, lr, lens, 0.3)
    assert np.allclose(np.subtract(b, rm), 3 * np.subtract(a, rm), atol=1e-12)   # linear in beta


def test_grpo_objective_pins():
    """Eq. 3 / Eq. 4 value; per-token KL estimator pi_ref/pi - log(pi_ref/pi) - 1 (R34)."""
    f = grpo.grpo_objective
    # lambda = 1, pi_ref = pi: the objective is the mean advantage
    assert abs(f([[-1.0, -2.0]] * 3, [[-1.0, -2.0]] * 3, [[-1.0, -2.0]] * 3, [0.5, -1.0, 2.0], [2, 1, 2], 0.2, 0.04)
               - 0.5) < 1e-15
    # clip (Eq. 3): A > 0, lambda = 2 -> 1.2 A; A < 0, lambda = 0.5 -> 0.8 A; A < 0, lambda = 2 -> 2 A
    ln2 = math.log(2.0)
    assert abs(f([[ln2]], [[0.0]], [[ln2]], [1.0], [1], 0.2, 0.0) - 1.2) < 1e-12
    assert abs(f([[-ln2]], [[0.0]], [[-ln2]], [-1.0], [1], 0.2, 0.0) - (-0.8)) < 1e-12
    assert abs(f([[ln2]], [[0.0]], [[ln2]], [-1.0], [1], 0.2, 0.0) - (-2.0)) < 1e-12
    # KL term alone: pi = 0.5, pi_ref = 0.25 -> 0.5 - ln 0.5 - 1
    kl = 0.5 - math.log(0.5) - 1.0
    assert abs(f([[math.log(0.5)]], [[math.log(0.5)]], [[math.log(0.25)]], [0.0], [1], 0.2, 0.1) + 0.1 * kl) < 1e-15
    # 1/|O_i| normalisation: repeating a token does not change a sample's term
    assert abs(f([[ln2, ln2]], [[0.0, 0.0]], [[0.0, 0.0]], [1.0], [2], 0.2, 0.04)
               - f([[ln2]], [[0.0]], [[0.0]], [1.0], [1], 0.2, 0.04)) < 1e-15
    # Eq. 4 = (1/N) sum_n J^(n) over equal micro groups = Eq. 3
    rng = np.random.default_rng(5)
    G, g, T = 8, 2, 7
    lp, lo, lr = (np.log(rng.uniform(0.05, 1.0, size=(G, T))) for _ in range(3))
    adv = list(rng.normal(size=G))
    lens = [int(x) for x in rng.integers(1, T + 1, size=G)]
    whole = f(lp, lo, lr, adv, lens, 0.2, 0.04)
    parts = [f(lp[n:n + g], lo[n:n + g], lr[n:n + g], adv[n:n + g], lens[n:n + g], 0.2, 0.04) for n in range(0, G, g)]
    assert abs(whole - sum(parts) / len(parts)) < 1e-12


def test_trace_generator_shape_and_determinism():
    a = gen_trace("math", 32, 1024, 1)
    assert a.dtype == np.int32 and len(a) == 32 and a.min() >= 1 and a.max() <= 1024
    assert np.array_equal(a, gen_trace("math", 32, 1024, 1))
    assert np.all(gen_trace((np.log(7.0), 0.0), 4, 100, 3) == 7)
    p = predict_lengths(a, "noisy", 0.0, seed=3)
    assert np.array_equal(p, a)


def test_table2_decomposition_definitions():
    """NEXT-2 (Table 2; SPEC's definitions, DESIGN R23): fptas_only = the Alg. 2
    plan in lexicographic (n, j) order with FIFO refill; sjf_only = trace-order start, SJF
    refill.  Pinned against their definitions written out independently of build_plan."""
    rng = np.random.default_rng(17)
    for _ in range(200):
        g = int(rng.integers(1, 5))
        G = g * int(rng.integers(1, 7))
        pred = [int(x) for x in rng.integers(1, 60, G)]
        plan = planner.fptas_plan(pred, G // g, 0.1)
        lex = sorted(range(G), key=lambda i: tuple(plan["mask"][i]))
        f = planner.build_plan("fptas_only", G, g, pred=pred, eps=0.1)
        assert f["init"] == lex[:g] and f["queue"] == lex[g:]
        inf = planner.build_plan("infinite", G, g, pred=pred, eps=0.1)
        assert f["init"] == inf["init"]  # same start, different refill order
        assert sorted(inf["queue"]) == sorted(f["queue"])
        s = planner.build_plan("sjf_only", G, g, pred=pred)
        assert s["init"] == list(range(g))
        assert s["queue"] == sorted(range(g, G), key=lambda i: (pred[i], i))
    # equal predictions: SJF keeps trace order, i.e. FIFO without a quota
    lens = [5, 3, 4, 2, 6, 1]
    r = simulator.simulate(lens, "sjf_only", 2, pred=[7] * 6)
    assert [e[2] for e in r.events if e[3] == "refill"] == [2, 3, 4, 5]


def _greedy_list_schedule(lengths, g):
    """Independent check: no-quota slot refill in trace order is greedy list scheduling;
    each sample goes to the slot that frees first (ties -> lower slot), makespan = steps."""
    free = [0] * g
    for L in lengths:
        s = min(range(g), key=lambda j: (free[j], j))
        free[s] += L
    return max(free)


def test_dynamic_slot_mode_pins():
    """R35: stop at the target-th completion."""
    # hand trace, g = 2, lengths [5,3,4,2,6,1,7,2], target 3:
    # steps 1-3 (0,1): uid 1 done at 3 -> slot 1 takes 2; steps 4-5 (0,2): uid 0 done at 5 ->
    # slot 0 takes 3; steps 6-7 (3,2): uid 3 done at 7 = 3rd completion (slot 0 first, R18),
    # uid 2 (also at its last token) is in flight on slot 1 -> discarded.
    r = simulator.simulate([5, 3, 4, 2, 6, 1, 7, 2], "dynamic", 2, target=3)
    assert r.total_steps == 7
    assert r.finish_step == {1: 3, 0: 5, 3: 7}
    assert r.discarded == [2]
    assert r.slot_table == [[0, 1]] * 3 + [[0, 2]] * 2 + [[3, 2]] * 2
    assert r.tokens_decoded == 3 + 5 + 2 + 4
    rng = np.random.default_rng(3)
    for _ in range(200):
        g = int(rng.integers(1, 5))
        G = g * int(rng.integers(1, 6))
        lens = [int(x) for x in rng.integers(1, 40, size=G)]
        full = simulator.simulate(lens, "dynamic", g)             # target = G: every candidate completes
        assert full.total_steps == _greedy_list_schedule(lens, g) and not full.discarded
        target = int(rng.integers(1, G + 1))
        d = simulator.simulate(lens, "dynamic", g, target=target, page_tokens=4)
        assert len(d.finish_step) == target and d.total_steps <= full.total_steps
        assert len(d.discarded) <= g - 1
        # token conservation: steps x active slots = completed + discarded partial work
        occ = sum(1 for row in d.slot_table for u in row if u >= 0)
        assert occ == d.tokens_decoded
        part = sum(sum(1 for row in d.slot_table for u in row if u == x) for x in d.discarded)
        assert d.tokens_decoded == sum(lens[u] for u in d.finish_step) + part
    with pytest.raises(ValueError):
        simulator.simulate([3, 4], "fifo", 1, target=1)


def test_bin_mode_slots_pins():
    """SPEC.md l.175 / l.204 / l.255 (bin_mode = slots; NEXT-2, DESIGN R38): Alg. 2 runs over g bins
    and slot j starts with bin j's head.  Hand-derived instance (G = 6, g = 2, eps = 1,
    pred = true = [5, 1, 1, 1, 1, 1]): S = 10, K = eps*S/2 = 5, l~ = [1]*6, C~ = 3, first fit in
    (l~ desc, id) order -> bins {0,1,2}, {3,4,5}; heads (0, 3); SJF queue over {1,2,4,5} by
    (pred, id) = [1, 2, 4, 5]; slot 0 runs 0 for 5 steps while slot 1 runs 3, 1, 2, 4, 5 one step
    each.  The groups reading (N = G/g = 3: K = 10/3, l~ = [2,1,1,1,1,1], C~ = 3 -> groups {0,1},
    {2,3,4}, {5}) starts (0, 1) instead -- the two readings differ."""
    pred = [5, 1, 1, 1, 1, 1]
    p = planner.build_plan("infinite_slots", 6, 2, pred=pred, eps=1.0)
    assert p["plan"]["groups"] == [[0, 1, 2], [3, 4, 5]] and p["plan"]["K"] == 5.0 and p["plan"]["capacity"] == 3
    assert p["init"] == [0, 3] and p["queue"] == [1, 2, 4, 5]
    q = planner.build_plan("infinite", 6, 2, pred=pred, eps=1.0)
    assert q["plan"]["groups"] == [[0, 1], [2, 3, 4], [5]] and q["init"] == [0, 1]
    r = simulator.simulate(pred, "infinite_slots", 2, pred=pred, eps=1.0)
    assert r.total_steps == 5
    assert r.slot_table == [[0, 3], [0, 1], [0, 2], [0, 4], [0, 5]]
    # an empty bin (every member finished in the prefix phase) takes the SJF queue head
    p2 = planner.build_plan("infinite_slots", 6, 2, pred=pred, eps=1.0, finished={3, 4, 5})
    assert p2["init"] == [0, 1] and p2["queue"] == [2]
    # with N = G/g == g the bins are Alg. 2's groups: same plan, heads = each group's first member
    rng = np.random.default_rng(7)
    for _ in range(50):
        g = int(rng.integers(1, 5))
        G = g * g
        pr = [int(x) for x in rng.integers(1, 50, G)]
        a = planner.build_plan("infinite_slots", G, g, pred=pr, eps=0.3)
        b = planner.build_plan("infinite", G, g, pred=pr, eps=0.3)
        assert a["plan"]["mask"] == b["plan"]["mask"]
        for j, grp in enumerate(a["plan"]["groups"]):
            if grp:
                assert a["init"][j] == grp[0]
    # schedule invariants on random traces: each sample runs exactly once, token conservation,
    # steps >= the lower bound, peak pages <= g full-length samples
    for trial in range(60):
        g = int(rng.choice([1, 2, 4, 8]))
        G = g * int(rng.integers(1, 6))
        true = [int(x) for x in rng.integers(1, 200, G)]
        pr = [max(1, int(t * (1 + 0.3 * rng.standard_normal()))) for t in true]
        r = simulator.simulate(true, "infinite_slots", g, pred=pr, eps=0.1, page_tokens=16)
        assert sorted(r.finish_step) == list(range(G))
        assert r.tokens_decoded == sum(true)
        assert r.total_steps >= simulator.step_lower_bound(true, g)
        assert r.peak_pages <= g * -(-max(true) // 16)


def test_memory_aware_admission_pins():
    """Memory-aware admission by predicted length (NEXT-2, DESIGN R41).
    Hand-traced instance: true = pred = [5,3,4,2,6,1,2,2], g = 2 guaranteed + 2 elastic slots,
    max_new = 8, 4-token pages -> W = 2 pages per worst-case sample, pool = 5 pages -> E = 1
    elastic page.  Alg. 2 (N = 4, K = 0.625, l~ = [8,5,7,4,10,2,4,4], C~ = 11) gives groups
    {4}, {0,7}, {2,3}, {1,6,5}: init (4, 0), SJF queue [5,3,6,7,1,2].  Slot 2 admits 5 (1 page
    <= E), slot 3 cannot admit 3 (1 + 1 > E).  5 ends at step 1 -> slot 2 admits 3 (steps 2-3),
    then 6 (steps 4-5); at step 5 sample 0 ends: slot 1 pops 7, slot 2 admits 1; 4 ends at
    step 6 -> slot 0 pops 2; 7 ends at 7, 1 at 8, 2 at 10: 10 steps against 14 for plain Alg. 1-3."""
    t = [5, 3, 4, 2, 6, 1, 2, 2]
    r = simulator.simulate_admit(t, 2, 4, t, max_new=8, pool_pages=5, page_tokens=4)
    assert r.slot_table == [[4, 0, 5, -1], [4, 0, 3, -1], [4, 0, 3, -1], [4, 0, 6, -1], [4, 0, 6, -1],
                            [4, 7, 1, -1], [2, 7, 1, -1], [2, -1, 1, -1], [2, -1, -1, -1], [2, -1, -1, -1]]
    assert r.total_steps == 10 and r.stalls == 0
    assert simulator.simulate(t, "infinite", 2, pred=t, page_tokens=4).total_steps == 14
    # a mispredicted elastic sample outgrows the elastic pool: it stalls, then a guaranteed slot
    # adopts it with its pages (true 8 but predicted 1: admitted on a 1-page reservation)
    t2, p2 = [8, 8, 8, 1], [8, 8, 1, 1]
    r2 = simulator.simulate_admit(t2, 1, 2, p2, max_new=8, pool_pages=3, page_tokens=4)
    assert r2.stalls > 0 and any(k == "adopt" for *_, k in r2.events)
    assert any(u <= -2 for row in r2.slot_table for u in row[1:])          # logged stalls
    assert all(u >= -1 for row in r2.slot_table for u in row[:1])           # never in a guaranteed slot
    assert r2.peak_pages <= 3 and r2.tokens_decoded == sum(t2)
    # E = 0 (a pool of exactly g worst-case samples): nothing is admitted, Alg. 1-3 exactly
    rng = np.random.default_rng(11)
    for _ in range(40):
        g = int(rng.choice([1, 2, 4]))
        G = g * int(rng.integers(1, 6))
        mx = int(rng.integers(4, 64))
        true = [int(x) for x in rng.integers(1, mx + 1, G)]
        pr = [max(1, int(x * (1 + 0.3 * rng.standard_normal()))) for x in true]
        a = simulator.simulate_admit(true, g, g + 2, pr, max_new=mx, pool_pages=g * -(-mx // 8), page_tokens=8)
        b = simulator.simulate(true, "infinite", g, pred=pr, page_tokens=8)
        assert [row[:g] for row in a.slot_table] == b.slot_table
        assert all(row[g:] == [-1, -1] for row in a.slot_table) and a.live_pages == b.live_pages
    # random instances: the budget is a hard invariant, every sample runs once, no dead step
    for _ in range(300):
        g = int(rng.choice([1, 2, 4]))
        S = g + int(rng.integers(1, 5))
        G = g * int(rng.integers(1, 6))
        mx = int(rng.integers(4, 64))
        pt = int(rng.choice([4, 8, 16]))
        true = [int(x) for x in rng.integers(1, mx + 1, G)]
        pr = [max(1, int(x * (1 + 0.4 * rng.standard_normal()))) for x in true]
        W = -(-mx // pt)
        pool = g * W + int(rng.integers(0, 3 * W))
        r = simulator.simulate_admit(true, g, S, pr, max_new=mx, pool_pages=pool, page_tokens=pt)
        assert r.peak_pages <= pool and max(r.live_pages) <= pool
        assert r.tokens_decoded == sum(true) and sorted(r.finish_step) == list(range(G))
        assert all(any(u >= 0 for u in row) for row in r.slot_table)
