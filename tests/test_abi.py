"""CPU-side checks of the C-ABI library: it builds/loads, exports every symbol
include/infsamp.h declares, and its host-only planner (is_plan,
is_group_advantages) is bit-exact against the oracle.  No device calls."""
import re

import numpy as np
import pytest

from conftest import ROOT, load_golden
from oracle import grpo, planner
from synth import SHAPES, gen_trace, predict_lengths


@pytest.fixture(scope="module")
def lib():
    from paper_2506_22950_b200 import _lib
    return _lib


def test_library_exports_every_declared_symbol(lib):
    import ctypes
    hdr = open(f"{ROOT}/include/infsamp.h").read()
    declared = set(re.findall(r"\b(is_[a-z_]+)\s*\(", hdr))
    declared -= {"is_status"}
    L = lib.load()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert set(lib.EXPORTS) == declared
    assert b"sm_100a" in L.is_version()
    with open(lib.lib_path(), "rb") as f:
        assert f.read(4) == b"\x7fELF"
    assert isinstance(L, ctypes.CDLL)


def _cfg(lib, G, g, mode="infinite", eps=0.1, prefix_k=0, budget=0, max_new=1024, shape="qwen3-1.7b", pt=16, P=256):
    return lib.make_config(SHAPES[shape], G, g, max_new, P, mode=mode, prefix_k=prefix_k, page_tokens=pt,
                           kv_budget_bytes=budget, eps=eps)


def test_is_plan_matches_oracle_spec_examples(lib):
    for ex in load_golden("spec_examples.json")["fptas"]:
        G, N = len(ex["pred"]), ex["N"]
        p = lib.is_plan(_cfg(lib, G, G // N, eps=ex["eps"]), ex["pred"])
        assert p["K"] == pytest.approx(ex["K"], rel=1e-15)
        assert p["scaled"] == ex["scaled"] and p["capacity"] == ex["capacity"]
        assert p["overflow"] == ex["overflow"]


def test_is_plan_bit_exact_vs_oracle_random(lib):
    rng = np.random.default_rng(11)
    for trial in range(300):
        g = int(rng.choice([1, 2, 4, 8]))
        G = g * int(rng.integers(1, 9))
        eps = float(rng.choice([0.05, 0.1, 0.3, 0.5, 1.0]))
        true = gen_trace("math", G, 1024, int(rng.integers(1 << 30)))
        pred = predict_lengths(true, "noisy", 0.3, seed=trial)
        fin = None
        if trial % 3 == 0:
            fin = (rng.random(G) < 0.2).astype(np.uint8)
        got = lib.is_plan(_cfg(lib, G, g, eps=eps), pred, fin)
        ref = planner.build_plan("infinite", G, g, pred=[int(x) for x in pred], eps=eps,
                                 finished=set(np.nonzero(fin)[0].tolist()) if fin is not None else ())
        P = ref["plan"]
        assert got["K"] == P["K"]
        assert got["scaled"] == P["scaled"] and got["capacity"] == P["capacity"]
        assert got["loads"] == P["loads"] and got["overflow"] == P["overflow"]
        assert got["mask"] == [tuple(m) for m in P["mask"]]
        init = [x for x in got["init"] if x >= 0]
        assert init == ref["init"] and got["queue"] == ref["queue"]


def test_is_plan_table2_modes_bit_exact_vs_oracle(lib):
    rng = np.random.default_rng(23)
    for trial in range(150):
        g = int(rng.choice([1, 2, 4, 8]))
        G = g * int(rng.integers(1, 9))
        true = gen_trace("math", G, 1024, int(rng.integers(1 << 30)))
        pred = [int(x) for x in predict_lengths(true, "noisy", 0.3, seed=trial)]
        for mode in ("fptas_only", "sjf_only"):
            got = lib.is_plan(_cfg(lib, G, g, mode=mode), pred)
            ref = planner.build_plan(mode, G, g, pred=pred, eps=0.1)
            assert [x for x in got["init"] if x >= 0] == ref["init"], (mode, trial)
            assert got["queue"] == ref["queue"], (mode, trial)


def test_is_plan_trace_order_modes(lib):
    for mode in ("naive", "fifo"):
        p = lib.is_plan(_cfg(lib, 8, 2, mode=mode), None)
        r = planner.build_plan(mode, 8, 2)
        assert p["init"] == r["init"] and p["queue"] == r["queue"]


def test_is_plan_budget_and_config_errors(lib):
    from oracle import kv
    s = SHAPES["tiny"]
    budget = kv.prefix_bytes(s, 16) + 4 * 2 * kv.page_bytes(s, 16)   # config 1 "4 slots"
    ok = lib.is_plan(_cfg(lib, 8, 2, budget=budget, max_new=32, shape="tiny", P=16), [3] * 8)
    assert ok["reserved_bytes"] == planner.reservation_bytes(8, 2, 32, 0, 16, kv.page_bytes(s, 16),
                                                             kv.prefix_bytes(s, 16))
    with pytest.raises(lib.InfsampError) as e:   # k = 4 with 16-token pages: 358,400 B > budget
        lib.is_plan(_cfg(lib, 8, 2, budget=budget, max_new=32, shape="tiny", P=16, prefix_k=4), [3] * 8)
    assert e.value.status == lib.IS_ERR_BUDGET
    lib.is_plan(_cfg(lib, 8, 2, budget=budget, max_new=32, shape="tiny", P=16, prefix_k=4, pt=4), [3] * 8)
    for bad in (dict(G=8, g=3), dict(G=8, g=2, eps=0.0)):
        with pytest.raises(lib.InfsampError) as e:
            lib.is_plan(_cfg(lib, bad["G"], bad["g"], eps=bad.get("eps", 0.1)), [3] * bad["G"])
        assert e.value.status == lib.IS_ERR_CONFIG
    with pytest.raises(lib.InfsampError) as e:
        lib.is_plan(_cfg(lib, 4, 2), [3, 0, 1, 2])
    assert e.value.status == lib.IS_ERR_DATA


def test_group_advantages_match_oracle(lib):
    rng = np.random.default_rng(12)
    for _ in range(50):
        r = rng.normal(size=int(rng.integers(1, 65))).astype(np.float32)
        for mode in ("std_norm", "mean_only"):
            a = lib.is_group_advantages(r, mode)
            ref = np.float32(grpo.advantages([float(x) for x in r], mode))
            assert np.array_equal(a, ref)
    assert np.all(lib.is_group_advantages(np.full(5, 2.0, np.float32)) == 0)


def test_kl_rewards_and_objective_match_oracle(lib):
    rng = np.random.default_rng(21)
    for _ in range(20):
        G, T = int(rng.integers(1, 17)), int(rng.integers(1, 40))
        rm = rng.normal(size=G).astype(np.float32)
        lp, lo, lr = (np.log(rng.uniform(0.01, 1.0, size=(G, T))).astype(np.float32) for _ in range(3))
        lens = rng.integers(1, T + 1, size=G).astype(np.int32)
        beta = float(np.float32(rng.uniform(0, 0.2)))
        got = lib.is_kl_rewards(rm, lp, lr, lens, beta)
        ref = np.float32(grpo.kl_rewards(rm.astype(np.float64), lp.astype(np.float64), lr.astype(np.float64),
                                         lens, beta))
        assert np.array_equal(got, ref)
        adv = rng.normal(size=G).astype(np.float32)
        j = lib.is_grpo_objective(lp, lo, lr, adv, lens, float(np.float32(0.2)), beta)
        jr = grpo.grpo_objective(lp.astype(np.float64), lo.astype(np.float64), lr.astype(np.float64),
                                 adv.astype(np.float64), lens, float(np.float32(0.2)), beta)
        assert abs(j - jr) <= 1e-12 * max(1.0, abs(jr))
    with pytest.raises(lib.InfsampError) as e:
        lib.is_kl_rewards(np.zeros(2, np.float32), np.zeros((2, 4), np.float32), np.zeros((2, 4), np.float32),
                          np.array([1, 5], np.int32), 0.1)
    assert e.value.status == lib.IS_ERR_DATA


def test_dynamic_mode_plan_and_config_errors(lib):
    cfg = _cfg(lib, 8, 2)
    cfg.mode = lib.MODES["dynamic"]
    out = lib.is_plan(cfg, [3] * 8)
    ref = planner.build_plan("dynamic", 8, 2)
    assert out["init"] == ref["init"] and out["queue"] == ref["queue"]
    for mode, target in (("dynamic", 9), ("dynamic", -1), ("infinite", 3)):
        bad = _cfg(lib, 8, 2)
        bad.mode = lib.MODES[mode]
        bad.dynamic_target = target
        with pytest.raises(lib.InfsampError) as e:
            lib.is_plan(bad, [3] * 8)
        assert e.value.status == lib.IS_ERR_CONFIG


def test_is_plan_bin_slots_bit_exact_vs_oracle(lib):
    """bin_mode = slots (DESIGN R38): init heads, SJF queue and the g-bin loads
    bit-exact against the oracle, incl. samples finished in a prefix phase."""
    rng = np.random.default_rng(29)
    for trial in range(200):
        g = int(rng.choice([1, 2, 4, 8]))
        G = g * int(rng.integers(1, 9))
        true = gen_trace("math", G, 1024, int(rng.integers(1 << 30)))
        pred = [int(x) for x in predict_lengths(true, "noisy", 0.3, seed=trial)]
        fin = set(int(i) for i in np.nonzero(rng.random(G) < 0.2)[0]) if trial % 2 else set()
        cfg = _cfg(lib, G, g, mode="infinite_slots")
        got = lib.is_plan(cfg, pred, finished=[1 if i in fin else 0 for i in range(G)] if fin else None)
        ref = planner.build_plan("infinite_slots", G, g, pred=pred, eps=0.1, finished=fin)
        assert got["init"] == ref["init"], trial
        assert got["queue"] == ref["queue"], trial
        assert got["loads"] == ref["plan"]["loads"], trial
        assert got["capacity"] == ref["plan"]["capacity"]
