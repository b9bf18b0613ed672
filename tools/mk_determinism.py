"""Determinism / batch-invariance probe of the decode implementations (tiny config)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from paper_2506_22950_b200 import _lib
from oracle import kv as okv
from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths

TINY = SHAPES["tiny"]
SEED = 20261017
w = gen_weights(TINY, seed=SEED)
wd = {k: v.cuda() for k, v in w.items()}
prompt = gen_prompt(TINY.vocab, 16, 0, seed=SEED)
true = gen_trace("tiny", 8, 32, 1)
pred = predict_lengths(true, "noisy", 0.3, seed=1)
budget = okv.prefix_bytes(TINY, 16) + 4 * 2 * okv.page_bytes(TINY, 16)


def run(mode, g, impl, dump_steps=4):
    cfg = _lib.make_config(TINY, 8, g, 32, 16, mode=mode, kv_budget_bytes=budget if mode != "full" else 0,
                           seed=SEED, decode_impl=impl)
    ctx = _lib.Context(cfg, wd)
    ctx.is_prefill(torch.as_tensor(prompt, device="cuda"), 0)
    ctx.is_start_group(true, pred)
    buf = torch.zeros(16, TINY.vocab, device="cuda")
    ctx.is_set_logits_dump(buf)
    dumps = []
    for _ in range(dump_steps):
        if ctx.is_query()["completed"] >= 8:
            break
        ctx.is_decode_step()
        torch.cuda.synchronize()
        dumps.append(buf.cpu().numpy().copy())
    ctx.is_set_logits_dump(None)
    ctx.is_run_group()
    sl, _ = ctx.is_copy_schedule()
    toks = ctx.is_copy_tokens()
    ctx.close()
    return toks, dumps, sl


for impl in ():
    a = run("naive", 2, impl)
    b = run("naive", 2, impl)
    c = run("infinite", 2, impl)
    d = run("full", 8, impl)
    print(f"impl {impl}: naive==naive {np.array_equal(a[0], b[0])}  naive==infinite {np.array_equal(a[0], c[0])}  "
          f"naive==full {np.array_equal(a[0], d[0])}")
    # logits of uid 0 at t = 0..3 (naive: slot 0; full: slot 0) -- both start at step 0
    for t in range(4):
        za, zb, zd = a[1][t][0], b[1][t][0], d[1][t][0]
        print(f"  t={t} |naive-naive| {np.abs(za - zb).max():.3e}  |naive-full| {np.abs(za - zd).max():.3e}  "
              f"rows naive {a[2][t][:2]} full {d[2][t][:2]}")


def per_uid(mode, g, impl):
    toks, dumps, sl = run(mode, g, impl, dump_steps=200)
    out = {}
    tcount = {}
    for step in range(min(len(dumps), len(sl))):
        for s, uid in enumerate(sl[step]):
            if uid < 0:
                continue
            t = tcount.get(int(uid), 0)
            out[(int(uid), t)] = dumps[step][s]
            tcount[int(uid)] = t + 1
    return out, sl


for impl in (0,):
    A, sla = per_uid("naive", 2, impl)
    B, slb = per_uid("infinite", 2, impl)
    bad = []
    for k in sorted(A):
        if k in B:
            d = np.abs(A[k] - B[k]).max()
            if d > 0:
                bad.append((k, d))
    print("first differing (uid, t):", bad[:8])
    for uid in range(8):
        ds = [(t, float(np.abs(A[(uid, t)] - B[(uid, t)]).max())) for t in range(40) if (uid, t) in A and (uid, t) in B]
        print("uid", uid, "diffs", [(t, round(d, 3)) for t, d in ds[:6]])
    C, slc = per_uid("naive", 2, 1)
    for uid in range(8):
        ds = [(t, float(np.abs(A[(uid, t)] - C[(uid, t)]).max())) for t in range(40) if (uid, t) in A and (uid, t) in C]
        print("impl0 vs impl1 naive uid", uid, [(t, round(d, 3)) for t, d in ds[:6]])
    print("naive slots", sla[:40].tolist())
    print("infinite slots", slb[:40].tolist())
