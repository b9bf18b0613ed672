"""K5 microbenchmark: the decode split attention of one layer through
is_dbg_attn at a given (rows, groups, suffix lengths), each timed run after a 256 MiB
write that evicts L2.  Algorithmic bytes per launch = the shared prefix KV once per
group + every live row's suffix KV (K and V, bf16): one JSON line per case."""
import argparse
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_22950_b200 import _lib  # noqa: E402


def case(rows, groups, grp_rows, plen, lens, Hq=16, Hkv=8, pt=16, max_new=1024, impl=0, reps=20, seed=0):
    if os.environ.get("K5_SHAPE") == "4b":
        Hq, Hkv = 32, 8
    gen = torch.Generator(device="cuda").manual_seed(seed)
    maxp = math.ceil(max_new / pt)
    q = torch.randn(rows, Hq, 128, device="cuda", generator=gen).to(torch.bfloat16)
    prefix = torch.randn(groups, 2, Hkv, plen, 128, device="cuda", generator=gen).to(torch.bfloat16)
    need = [math.ceil(n / pt) for n in lens]
    num_pages = sum(need) + 1
    pool = torch.randn(num_pages, 2, Hkv, pt, 128, device="cuda", generator=gen).to(torch.bfloat16)
    perm = torch.randperm(num_pages, device="cpu").tolist()
    pagetab = torch.zeros(rows, maxp, dtype=torch.int32)
    k = 0
    for r, n in enumerate(need):
        for j in range(n):
            pagetab[r, j] = perm[k]
            k += 1
    row_len = torch.tensor(lens, dtype=torch.int32, device="cuda")
    _, ms = _lib.is_dbg_attn(q, prefix, pool, pagetab.cuda(), row_len, grp_rows, impl=impl, reps=reps)
    kv_tok = 2 * Hkv * 128 * 2
    nbytes = groups * plen * kv_tok + sum(lens) * kv_tok
    med = float(np.median(ms))
    return dict(rows=rows, groups=groups, grp_rows=grp_rows, plen=plen, impl=impl, live=sum(1 for n in lens if n),
                mean_len=float(np.mean([n for n in lens if n])), mbytes=round(nbytes / 1e6, 2),
                us_median=round(med * 1e3, 2), us_min=round(min(ms) * 1e3, 2),
                gbps=round(nbytes / (med * 1e-3) / 1e9, 1), gbps_best=round(nbytes / (min(ms) * 1e-3) / 1e9, 1))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--impls", default="0")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--case", default=None, help="run only this case")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    rng = np.random.default_rng(1)
    math_lens = lambda n: [int(min(1024, max(1, round(x)))) for x in rng.lognormal(6.337, 0.6, n)]
    cases = [
        ("config3_g8", 16, 1, 8, 255, math_lens(8) + [0] * 8),
        ("g8_t600", 16, 1, 8, 255, [600] * 8 + [0] * 8),
        ("rows32_t1024", 32, 4, 8, 255, [1024] * 32),
        ("groups8_math", 64, 8, 8, 255, math_lens(64)),
        ("groups8_t512", 64, 8, 8, 255, [512] * 64),
        ("groups8_t1024", 64, 8, 8, 255, [1024] * 64),
        ("full64_t512", 64, 1, 64, 255, [512] * 64),
    ]
    for impl in [int(x) for x in args.impls.split(",")]:
        for name, rows, groups, grp, plen, lens in cases:
            if args.case and name != args.case:
                continue
            r = case(rows, groups, grp, plen, lens, impl=impl, reps=args.reps)
            r["case"] = name
            print(json.dumps(r), flush=True)


if __name__ == "__main__":
    main()
