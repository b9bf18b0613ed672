"""Benchmark: continuous-sampling rollouts of Infinite Sampling on B200.

One bench *step* = one whole GRPO-group rollout through the C-ABI (BASELINE.json
configs[2], the paper's headline setting): prefill of a 256-token prompt,
Alg. 2 FPTAS plan, then continuous-sampling decode steps with SJF refill until
all G = 32 completions (lengths from the MATH-shape trace, max 1024) are done,
then rewards.  Metric: generated tokens/s per GPU (whole job = sum over ranks).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config N]

Multi-GPU: one process per GPU (torchrun), prompts sharded by rank (weak
scaling), one NCCL all-gather of (length, reward) per rollout for the
group-normalised advantages (Eq. 2); time = max over ranks.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (shape, prompts-per-rank unused, G, g, max_new, P, family, prefix_k, budget)
    3: dict(shape="qwen3-1.7b", G=32, g=8, max_new=1024, P=256, family="math", prefix_k=0,
            desc="Qwen3-1.7B-shape random-init bf16, prompt 256, G=32, micro group 8, max 1024 new tokens, "
                 "FPTAS+SJF plan on MATH-shape lengths"),
    2: dict(shape="qwen3-0.6b", G=16, g=4, max_new=512, P=256, family="math8b", prefix_k=0,
            desc="Qwen3-0.6B-shape, G=16, micro group 4, max 512"),
    4: dict(shape="qwen3-1.7b", G=64, g=8, max_new=1024, P=256, family="longtail", prefix_k=16,
            desc="Qwen3-1.7B-shape, G=64 under a 1 GiB KV budget, k=16 prefix phase, long-tail lengths"),
    5: dict(shape="qwen3-4b", G=64, g=8, max_new=1024, P=256, family="math", prefix_k=0,
            desc="Qwen3-4B-shape, G=64, micro group 8, prompts sharded by rank"),
}
SEED = 20261017
METRIC = "generated tokens/s per GPU, G=32 Qwen3-1.7B-shape; HBM GB/s vs peak; peak KV GB"


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"], "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.p = None
        self.lines = []

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        loaded = [x for x in sm if x > 500] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(name):
    """DRAM bytes per launch of a kernel from the newest committed ncu `--set full` summary
    profiles/*/ncu_<name>.csv (tools/summarize_profiles.py), or None: read + write (the contract's
    `traffic`) and read alone (min over the captured launches)."""
    import csv
    import glob
    # the newest round's capture: profiles/<round>/ names sort in round order (r01 < r02a < ... < r02e)
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*", f"ncu_{name}.csv")))
    if not files:
        return None
    rows = list(csv.DictReader(open(files[-1])))
    rw, rd = [], []
    for r in rows:
        try:  # ncu reports these counters in MB (1e6 bytes) in the raw page
            rd.append(float(r["dram__bytes_read.sum"]) * 1e6)
            rw.append((float(r["dram__bytes_read.sum"]) + float(r["dram__bytes_write.sum"])) * 1e6)
        except (KeyError, ValueError):
            pass
    if not rw:
        return None
    return {"bytes_per_launch": round(float(np.min(rw))), "read_bytes_per_launch": round(float(np.min(rd))),
            "source": os.path.relpath(files[-1], ROOT)}


def lpt_place(pool, world, per_rank):
    """(paper_2506_22950_b200.rollout.lpt_place)"""
    from paper_2506_22950_b200.rollout import lpt_place as f
    return f(pool, world, per_rank)


def algorithmic_bytes_per_step(shape, live_rows, suffix_tokens, P):
    """weights once per step + prefix KV once per group + live suffix KV + appends."""
    L, H, F, V = shape.layers, shape.hidden, shape.ffn, shape.vocab
    per_layer_w = ((shape.q_dim + 2 * shape.kv_dim) * H + H * shape.q_dim + 2 * F * H + H * F) * 2
    kv_tok = 2 * L * shape.n_kv_heads * shape.head_dim * 2
    return L * per_layer_w + V * H * 2 + (P - 1) * kv_tok + suffix_tokens * kv_tok + live_rows * kv_tok


def attention_k5(_lib, torch, rows=64, groups=8, plen=255, slen=1024, Hq=16, Hkv=8, pt=16, reps=10):
    gen = torch.Generator(device="cuda").manual_seed(5)
    q = torch.randn(rows, Hq, 128, device="cuda", generator=gen).to(torch.bfloat16)
    prefix = torch.randn(groups, 2, Hkv, plen, 128, device="cuda", generator=gen).to(torch.bfloat16)
    npg = math.ceil(slen / pt)
    pool = torch.randn(rows * npg + 1, 2, Hkv, pt, 128, device="cuda", generator=gen).to(torch.bfloat16)
    pagetab = torch.randperm(rows * npg, device="cuda").to(torch.int32).reshape(rows, npg)
    row_len = torch.full((rows,), slen, dtype=torch.int32, device="cuda")
    _, ms = _lib.is_dbg_attn(q, prefix, pool, pagetab, row_len, rows // groups, reps=reps)
    kv_tok = 2 * Hkv * 128 * 2
    nbytes = groups * plen * kv_tok + rows * slen * kv_tok
    med = float(np.median(ms))
    hbm = peaks()[0]
    return {"case": f"{groups} groups x {rows // groups} rows x {slen} suffix tokens + {plen}-token prefix, 1.7B heads",
            "bytes_per_launch": int(nbytes), "us_median": round(med * 1e3, 2),
            "achieved": round(nbytes / (med * 1e-3) / 1e9, 1), "peak": hbm,
            "frac": round(nbytes / (med * 1e-3) / 1e9 / hbm, 4),
            "timing": f"is_dbg_attn, {reps} reps, a 256 MiB write evicts L2 before each, CUDA events (median)"}


def run_ours(args):
    import torch
    from paper_2506_22950_b200 import _lib
    from paper_2506_22950_b200 import rollout as rollout_mod
    from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    C = CONFIGS[args.config]
    shape = SHAPES[C["shape"]]
    G, g, max_new, P = C["G"], C["g"], C["max_new"], C["P"]
    page_tokens = 16
    kv_tok = 2 * shape.layers * shape.n_kv_heads * shape.head_dim * 2
    budget = (P - 1) * kv_tok + g * math.ceil(max_new / page_tokens) * page_tokens * kv_tok
    if C["prefix_k"]:
        budget = 1 << 30
    w = gen_weights(shape, seed=SEED, device="cuda")
    cfg = _lib.make_config(shape, G, g, max_new, P, mode="infinite", prefix_k=C["prefix_k"],
                           page_tokens=page_tokens, kv_budget_bytes=budget, eps=0.1, temperature=0.8, seed=SEED,
                           top_p=args.top_p)
    ctx = _lib.Context(cfg, w)
    del w
    torch.cuda.empty_cache()
    comm = nccl_comm(_lib, dist, rank, world)
    n_total = args.warmup + args.steps

    def workload(pid):                       # global prompt id (RNG keyed by global uid)
        prompt = gen_prompt(shape.vocab, P, pid, seed=SEED)
        true = gen_trace(C["family"], G, max_new, SEED + pid)
        pred = predict_lengths(true, "noisy", 0.3, seed=SEED + pid, prefix_k=C["prefix_k"])
        return pid, prompt, true, pred

    # warm-up prompts stay with their rank; the timed prompts are placed by LPT on the
    # predicted work: every rank predicts its block, the totals are
    # all-gathered, then the longest goes to the least-loaded rank (equal counts per rank)
    own = [rank * n_total + i for i in range(n_total)]
    placement = {r: [r * n_total + args.warmup + k for k in range(args.steps)] for r in range(world)}
    if dist is not None and args.placement == "lpt":
        mine = torch.tensor([[float(pid), float(np.sum(workload(pid)[3]))] for pid in placement[rank]], device="cuda")
        gathered = [torch.zeros_like(mine) for _ in range(world)]
        dist.all_gather(gathered, mine)
        pool = [(int(p), float(w)) for t in gathered for p, w in t.cpu().numpy()]
        placement = rollout_mod.lpt_place(pool, world, args.steps)
    timed_ids = placement[rank]
    work = [workload(pid) for pid in own[:args.warmup] + timed_ids]
    d_prompts = [torch.as_tensor(p, device="cuda") for _, p, _, _ in work]
    res = rollout_mod.RankResults(max(args.steps, 1), G, world)
    warm_res = rollout_mod.RankResults(max(args.warmup, 1), G, 1)
    stream = torch.cuda.current_stream()

    acc = {"suffix": 0, "rows": 0, "steps": 0}

    def rollout(i, out, k, host_inputs=False):
        pid, prompt, true, pred = work[i]
        if host_inputs:                      # e2e: host -> device copy of the step's input inside the timed region
            dp = torch.from_numpy(prompt).pin_memory().to("cuda", non_blocking=True)
        else:
            dp = d_prompts[i]
        ctx.is_prefill(dp, pid)
        ctx.is_start_group(true, pred)       # Alg. 2 plan + budget check (host) + slot fill
        steps = ctx.is_run_group()
        q = ctx.is_query()                   # per-group counters (syncs; the rollout has already synced)
        acc["suffix"] += q["suffix_tokens"]
        acc["rows"] += q["tokens_decoded"]
        acc["steps"] += q["steps"]
        d_rew, d_len = out.slot(k)
        ctx.is_group_results(d_rew, d_len)   # rewards + lengths into this group's slots
        return steps

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(args.warmup):
        rollout(i, warm_res, i)
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tokens, steps_total, peak_kv, live_rows_steps = 0, 0, 0, 0
    q0 = ctx.is_query()
    for k in acc:
        acc[k] = 0
    e0.record(stream)
    for k, i in enumerate(range(args.warmup, n_total)):
        steps_total += rollout(i, res, k)
        tokens += int(np.sum(work[i][2]))
    # the one exchange, after the rank's last group: lengths + rewards of all its groups
    res.exchange(ctx, comm, dist)
    e1.record(stream)
    barrier()
    ms = e0.elapsed_time(e1)
    st = ctx.is_query()
    timed = dict(acc)
    clk = clocks.stop()
    # ---- e2e: same rollouts through the public API with host buffers; the result read back is
    # every rank's (length, reward) and the Eq. 2 advantages computed from them
    e2 = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    barrier()
    e2[0].record(stream)
    for k, i in enumerate(range(args.warmup, n_total)):
        rollout(i, res, k, host_inputs=True)
    all_len, all_rew = res.exchange(ctx, comm, dist)
    adv = rollout_mod.advantages_by_prompt(all_len.cpu().numpy(), all_rew.cpu().numpy(),
                                           rollout_mod.global_order(placement, world, args.steps), G)
    e2[1].record(stream)
    barrier()
    ms_e2e = e2[0].elapsed_time(e2[1])
    assert len(adv) == world * args.steps
    # ---- per-launch profile of one decode step (eager replay with events) for the roofline
    pid, prompt, true, pred = work[0]
    ctx.is_prefill(d_prompts[0], pid)
    ctx.is_start_group(true, pred)
    for _ in range(3):
        ctx.is_decode_step()
    prof, prof_e = [], []
    for _ in range(5):
        msl, kind = ctx.is_profile_step(graph=True)      # step graph + an event node after every launch
        prof.append(msl)
        msl_e, kind_e = ctx.is_profile_step()            # eager replay (includes host launch gaps)
        prof_e.append(msl_e)
    msl = np.median(np.stack(prof), axis=0)
    step_ms_eager = float(np.median(np.stack(prof_e), axis=0).sum())
    if True:
        # the dominant kernel alone: every layer's gate/up launch as the step issues it, back to
        # back in one graph (4 passes over the layers), CUDA events around the replay
        gu_kernel = [ctx.is_profile_kernel(5, reps=4) for _ in range(3)]
        # split attention at a mid-rollout step (suffixes of a few hundred tokens): the layer's
        # prefix + suffix launches back to back; its algorithmic bytes = the shared prefix KV
        # once + every live row's suffix KV
        for _ in range(400):
            ctx.is_decode_step()
        s0 = ctx.is_query()["suffix_tokens"]
        ctx.is_decode_step()
        q1 = ctx.is_query()
        attn_suffix = int(q1["suffix_tokens"] - s0)
        attn_ms = float(np.median([ctx.is_profile_kernel(3, reps=4)[0] for _ in range(3)]))
    stq = ctx.is_query()
    # K5 microbenchmark (>= 32 MB per launch, L2 flushed before each rep): the decode
    # attention of one layer on 8 groups x 8 rows x 1024 suffix tokens through is_dbg_attn
    k5 = attention_k5(_lib, torch)

    t = torch.tensor([ms, ms_e2e, float(tokens)], device="cuda", dtype=torch.float64)
    if dist is not None:
        tt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(tt, t)
        ms_max = max(float(x[0]) for x in tt)
        e2e_max = max(float(x[1]) for x in tt)
        tok_all = sum(float(x[2]) for x in tt)
    else:
        ms_max, e2e_max, tok_all = ms, ms_e2e, float(tokens)
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    hbm, tflops, peak_kind = peaks()
    kinds = {0: "embed/norm", 1: "qkv_gemm", 2: "qkv_post", 3: "attention", 4: "o_proj", 5: "gate_up", 6: "down",
             7: "lm_head_sampler", 8: "refill"}
    per_kind = {kinds[k]: float(msl[kind == k].sum()) for k in kinds}
    n_launch_kind = {kinds[k]: int((kind == k).sum()) for k in kinds}
    step_ms = float(msl.sum())
    H, F, L = shape.hidden, shape.ffn, shape.layers
    kv_tok = 2 * L * shape.n_kv_heads * shape.head_dim * 2
    layer_w = ((shape.q_dim + 2 * shape.kv_dim) * H + H * shape.q_dim + 2 * F * H + H * F) * 2
    if True:
        gu_bytes = 2 * F * H * 2                          # algorithmic bytes per gate/up launch (weights)
        gu_ms_step = per_kind["gate_up"] / max(n_launch_kind["gate_up"], 1)
        gu_ms = float(np.median([m for m, _ in gu_kernel]))
        achieved = gu_bytes / (gu_ms * 1e-3) / 1e9
        tr = ncu_traffic("gateup")
        roof = {"bound": "hbm", "kernel": "gate_up GEMM (tcgen05 swap-AB, SwiGLU epilogue)",
                "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                "peak_kind": peak_kind, "bytes_per_launch": gu_bytes,
                "traffic": tr["bytes_per_launch"] if tr else None,
                "traffic_read": tr["read_bytes_per_launch"] if tr else None,
                "traffic_source": tr["source"] if tr else None,
                "traffic_note": "ncu --set full --cache-control all; reads = the weights + activations (1.00x "
                                "algorithmic); the kernel's own output is 0.2 MB, the rest of dram__bytes_write "
                                "are write-backs ncu attributes to the launch",
                "launch_ms": round(gu_ms, 5), "launches_timed": int(gu_kernel[0][1]),
                "timing": "CUDA events around a graph of the step's gate/up launches (all layers, 4 passes, PDL "
                          "as in the step; median of 3 replays)",
                "achieved_in_step": round(gu_bytes / (gu_ms_step * 1e-3) / 1e9, 1),
                "in_step_timing": "graph event nodes after every launch of one captured decode step (each "
                                  "interval includes one graph-node hop; median of 5 replays)"}
    roof["step_ms_graph_events"] = round(step_ms, 4)
    roof["step_ms_eager"] = round(step_ms_eager, 4)
    if True:
        kv_tok_layer = 2 * shape.n_kv_heads * shape.head_dim * 2
        attn_bytes = (P - 1) * kv_tok_layer + attn_suffix * kv_tok_layer
        roof["attention"] = {"bound": "hbm", "kernel": "split attention per layer (tcgen05 shared prefix + "
                             "warp-per-chunk suffix + fused LSE merge)", "unit": "GB/s",
                             "achieved": round(attn_bytes / (attn_ms * 1e-3) / 1e9, 1), "peak": hbm,
                             "frac": round(attn_bytes / (attn_ms * 1e-3) / 1e9 / hbm, 4),
                             "bytes_per_layer": int(attn_bytes), "suffix_tokens": attn_suffix,
                             "layer_ms": round(attn_ms, 5),
                             "timing": "step 401 of a rollout; all layers' attention launches back to back in "
                                       "a graph, CUDA events (median of 3)"}
    # step roofline: algorithmic bytes of an average step of the timed rollouts (weights
    # + prefix KV + the live rows' suffix KV as measured by the scheduler + appends) / step time
    per_step_suffix = timed["suffix"] / max(steps_total, 1)
    per_step_rows = timed["rows"] / max(steps_total, 1)
    step_bytes = algorithmic_bytes_per_step(shape, per_step_rows, per_step_suffix, P)
    roof["step_GBps"] = round(step_bytes / (ms_max / max(steps_total, 1) * 1e-3) / 1e9, 1)
    roof["step_frac"] = round(roof["step_GBps"] / hbm, 4)
    roof["step_bytes"] = int(step_bytes)
    roof["attention_k5"] = k5
    roof["per_kind_ms"] = {k: round(v, 4) for k, v in per_kind.items() if n_launch_kind[k]}
    launches_per_step = int(st["launches_per_step"])  # counted by the library while capturing the step
    avg_steps = steps_total / args.steps
    value = tok_all / (ms_max * 1e-3)
    e2e_value = tok_all / (e2e_max * 1e-3)
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": f"config {args.config}: {C['desc']}", "model": C["shape"] + " (random init)",
                   "top_p": args.top_p, "G": G, "g": g, "prompt_len": P, "max_new_tokens": max_new, "length_family": C["family"],
                   "kv_budget_bytes": budget, "global_batch": G * world, "seq_len": P + max_new,
                   "parallelism": f"dp{world} (prompt-sharded)", "step": "one GRPO-group rollout",
                   "exchange": EXCHANGE["path"],
                   "placement": args.placement if world > 1 else "single GPU",
                   "l2": "inputs larger than L2 (3.4 GB of weights streamed per decode step)"},
        "roofline": roof,
        "decode_steps_per_rollout": round(avg_steps, 1),
        "ms_per_decode_step": round(ms_max / max(steps_total, 1), 4),
        "peak_kv_bytes": st["peak_kv_bytes"],
        "gpu_launches": int(launches_per_step * steps_total + st["launches_per_prefill"] * args.steps
                            + 2 * args.steps),  # decode steps + prefills + start-group scheduler / results kernels
        "launches_per_decode_step": launches_per_step,
        "per_gpu": round(value / world, 1),
        "e2e": {"value": round(e2e_value, 1), "unit": "tokens/s", "h2d_bytes_per_step": P * 4,
                "d2h_bytes_per_step": 8 * G * world},
        "clocks": clk,
    }
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(C, budget_s=args.cpu_seconds)
    print(json.dumps(line))
    sys.stdout.flush()
    ctx.close()
    if comm is not None and comm != "torch":
        _lib.nccl_comm_destroy(comm)
    if dist is not None:
        dist.destroy_process_group()


def run_groups(args):
    """NEXT-1: --groups M co-resident prompt groups share every decode step.
    K + W prompts are pushed through M group slots (a finished slot is refilled with the
    next prompt); the timed region covers the K timed prompts' rollouts end to end."""
    import torch
    from paper_2506_22950_b200 import _lib
    from paper_2506_22950_b200 import rollout as rollout_mod
    from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths

    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    C = CONFIGS[args.config]
    shape = SHAPES[C["shape"]]
    G, g, max_new, P, M = C["G"], C["g"], C["max_new"], C["P"], args.groups
    kv_tok = 2 * shape.layers * shape.n_kv_heads * shape.head_dim * 2
    budget = (P - 1) * kv_tok + g * math.ceil(max_new / 16) * 16 * kv_tok
    if C["prefix_k"]:
        budget = 1 << 30
    w = gen_weights(shape, seed=SEED, device="cuda")
    cfg = _lib.make_config(shape, G, g, max_new, P, mode="infinite", prefix_k=C["prefix_k"], page_tokens=16,
                           kv_budget_bytes=budget, eps=0.1, temperature=0.8, seed=SEED, max_groups=M,
                           top_p=args.top_p)
    ctx = _lib.Context(cfg, w)
    del w
    torch.cuda.empty_cache()
    comm = nccl_comm(_lib, dist, rank, world)

    def workload(j):
        pid = rank * 100000 + j  # global prompt id (RNG keyed by global uid)
        prompt = gen_prompt(shape.vocab, P, pid, seed=SEED)
        true = gen_trace(C["family"], G, max_new, SEED + pid)
        pred = predict_lengths(true, "noisy", 0.3, seed=SEED + pid, prefix_k=C["prefix_k"])
        return pid, torch.as_tensor(prompt, device="cuda"), true, pred

    def pipeline(prompts, res):
        """Push the prompts through the M slots; returns (tokens generated, global decode steps).
        Group results land in `res` (one slot per finished group), exchanged once at the end."""
        queue = list(prompts)
        slot_of, tokens, kdone = {}, 0, 0
        for slot in range(min(M, len(queue))):
            pid, dp, true, pred = queue.pop(0)
            ctx.is_prefill(dp, pid, slot=slot)
            ctx.is_start_group(true, pred, slot=slot)
            slot_of[slot] = true
        steps0 = None
        steps = 0
        while slot_of:
            mask, steps = ctx.is_run_until_any_done()
            for slot in list(slot_of):
                if mask >> slot & 1:
                    true = slot_of.pop(slot)
                    tokens += int(np.sum(true))
                    d_rew, d_len = res.slot(kdone)
                    ctx.is_group_results(d_rew, d_len, slot=slot)
                    kdone += 1
                    if queue:
                        pid, dp, tr, pr = queue.pop(0)
                        ctx.is_prefill(dp, pid, slot=slot)
                        ctx.is_start_group(tr, pr, slot=slot)
                        slot_of[slot] = tr
        return tokens, steps

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    warm = [workload(j) for j in range(args.warmup)]
    timed = [workload(args.warmup + j) for j in range(args.steps * M)]
    pipeline(warm, rollout_mod.RankResults(len(warm), G, 1))
    res = rollout_mod.RankResults(len(timed), G, world)
    barrier()
    s0 = ctx.is_query()["global_steps"]
    clocks = ClockSampler(local)
    clocks.start()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    tokens, steps = pipeline(timed, res)
    res.exchange(ctx, comm, dist)  # the one exchange, after the rank's last group
    e1.record(stream)
    barrier()
    ms = e0.elapsed_time(e1)
    clk = clocks.stop()
    st = ctx.is_query()
    t = torch.tensor([ms, float(tokens)], device="cuda", dtype=torch.float64)
    if dist is not None:
        tt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(tt, t)
        ms_max = max(float(x[0]) for x in tt)
        tok_all = sum(float(x[1]) for x in tt)
    else:
        ms_max, tok_all = ms, float(tokens)
    if rank == 0:
        dsteps = st["global_steps"] - s0
        print(json.dumps({
            "metric": METRIC, "value": round(tok_all / (ms_max * 1e-3), 1), "unit": "tokens/s", "n_gpus": world,
            "per_gpu": round(tok_all / (ms_max * 1e-3) / world, 1),
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"config {args.config} x {M} co-resident groups (SURVEY §8f NEXT-1): {C['desc']}",
                       "model": C["shape"] + " (random init)", "top_p": args.top_p, "G": G, "g": g, "groups": M,
                       "prompts_timed": len(timed), "kv_budget_bytes_per_group": budget,
                       "step": f"{M} GRPO-group rollouts through {M} group slots",
                       "parallelism": f"dp{world} (prompt-sharded)"},
            "decode_steps": int(dsteps), "ms_per_decode_step": round(ms_max / max(dsteps, 1), 4),
            "global_peak_kv_bytes": st["global_peak_kv_bytes"], "clocks": clk}))
    ctx.close()
    if comm is not None and comm != "torch":
        _lib.nccl_comm_destroy(comm)
    if dist is not None:
        dist.destroy_process_group()


EXCHANGE = {"path": "none"}


def nccl_comm(_lib, dist, rank, world):
    """The library's NCCL communicator for the results all-gather: rank 0 creates the
    unique id, the torch process group broadcasts it (plumbing only).  If the library
    cannot bind NCCL on some rank, every rank uses torch's all-gather for this one
    exchange instead (recorded in the JSON line as config.exchange)."""
    if dist is None:
        return None
    import torch
    ok = torch.ones(1, device="cuda")
    uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        try:
            uid.copy_(torch.frombuffer(bytearray(_lib.nccl_unique_id()), dtype=torch.uint8))
        except Exception:
            ok.zero_()
    dist.broadcast(uid, 0)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    comm = None
    if ok.item() > 0:
        try:
            comm = _lib.nccl_comm_init(bytes(uid.cpu().numpy().tobytes()), rank, world)
        except Exception:
            comm = None
    flag = torch.tensor([1.0 if comm is not None else 0.0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if flag.item() == 0:
        if comm is not None:
            _lib.nccl_comm_destroy(comm)
        EXCHANGE["path"] = "torch.distributed all_gather (library NCCL unavailable), once per rank"
        return "torch"
    EXCHANGE["path"] = "is_allgather_results_n (library NCCL), once per rank after its last group"
    return comm


_ORACLE_W = {}


def _oracle_tokens_per_s(C, budget_s, step_seed=0):
    """The oracle as it stands: full-recompute decode of one sample, tokens until ~budget_s."""
    import torch
    from oracle import model as M
    from oracle import sampler
    from synth import SHAPES, gen_prompt, gen_weights
    shape = SHAPES[C["shape"]]
    if _ORACLE_W.get("shape") != C["shape"]:  # generated once per process (not part of the timing)
        w = gen_weights(shape, seed=SEED, device="cuda" if torch.cuda.is_available() else "cpu")
        _ORACLE_W.update(shape=C["shape"], w={k: v.cpu() for k, v in w.items()})
        del w
    w = _ORACLE_W["w"]
    prompt = [int(x) for x in gen_prompt(shape.vocab, C["P"], step_seed, seed=SEED)]
    seq = list(prompt)
    t0 = time.perf_counter()
    n = 0
    while True:
        z = M.forward(w, shape, seq, mirror=True, logit_rows=[len(seq) - 1])[0]
        tok = sampler.sample_token_topp(z.astype(np.float32), SEED, step_seed * C["G"], n, 0.8, TOP_P[0])
        seq.append(tok)
        n += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return n, dt


TOP_P = [1.0]   # bench --top-p (1 = the paper's plain temperature sampling)


def cpu_baseline(C, budget_s=20.0):
    """The oracle as it stands, on this host's cores: full-recompute fp64 decode of
    the bench config at nproc BLAS threads (the headline value) and at 1 thread, config 1
    (tiny) decoded in full, and the schedule simulator (Alg. 1-3) per config."""
    from threadpoolctl import threadpool_limits
    from oracle import model as M
    from oracle import simulator
    from synth import SHAPES, gen_prompt, gen_trace, gen_weights, predict_lengths
    n, dt = _oracle_tokens_per_s(C, budget_s)
    with threadpool_limits(limits=1):
        n1, dt1 = _oracle_tokens_per_s(C, budget_s / 2)
    # config 1 in full: every sample of the tiny group, full recompute per token
    tiny = SHAPES["tiny"]
    w = gen_weights(tiny, seed=SEED)
    prompt = gen_prompt(tiny.vocab, 16, 0, seed=SEED)
    true = gen_trace("tiny", 8, 32, 1)
    t0 = time.perf_counter()
    for i, L in enumerate(true):
        M.generate(w, tiny, prompt, i, int(L), SEED)
    t_tiny = time.perf_counter() - t0
    # the schedule simulator per config (trace-driven Alg. 1-3 with the noisy predictor)
    sims = {}
    for cid, cc in sorted(CONFIGS.items()):
        tr = gen_trace(cc["family"], cc["G"], cc["max_new"], SEED)
        pr = predict_lengths(tr, "noisy", 0.3, seed=SEED, prefix_k=cc["prefix_k"])
        t0 = time.perf_counter()
        r = simulator.simulate(tr, "infinite", cc["g"], pred=pr, eps=0.1, prefix_k=cc["prefix_k"], page_tokens=16)
        sims[f"config {cid}"] = {"ms": round((time.perf_counter() - t0) * 1e3, 2), "steps": r.total_steps}
    return {"value": round(n / dt, 5), "unit": "tokens/s", "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"oracle full-recompute fp64 decode of sample 0 of prompt 0 ({C['shape']}, prompt {C['P']}): "
                      f"{n} tokens in {dt:.1f} s on {os.cpu_count()} BLAS threads",
            "one_thread": {"value": round(n1 / dt1, 5), "unit": "tokens/s", "sample": f"{n1} tokens in {dt1:.1f} s"},
            "config1_full": {"value": round(float(np.sum(true)) / t_tiny, 3), "unit": "tokens/s",
                             "sample": f"all 8 samples of config 1 ({int(np.sum(true))} tokens) in {t_tiny:.2f} s"},
            "schedule_simulator": sims}


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return
    C = CONFIGS[args.config]
    for i in range(args.warmup):
        _oracle_tokens_per_s(C, 0.0, step_seed=i)
    n_tot, t_tot = 0, 0.0
    for i in range(args.steps):
        n, dt = _oracle_tokens_per_s(C, 0.0, step_seed=args.warmup + i)
        n_tot += n
        t_tot += dt
    v = n_tot / t_tot
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(v, 5), "unit": "tokens/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_tot / args.steps * 1e3, 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"config {args.config}: {C['desc']}", "top_p": args.top_p,
                   "step": "oracle decodes 1 token (full recompute)"},
        "cpu_baseline": {"value": round(v, 5), "unit": "tokens/s", "cores": os.cpu_count(), "kind": "oracle",
                         "sample": f"{n_tot} tokens, 1 per step, full-recompute fp64 oracle on host cores"},
        "e2e": {"value": round(v, 5), "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--top-p", type=float, default=1.0,
                    help="nucleus sampling (SURVEY §8f NEXT-4, DESIGN R36); 1 = the paper's setting")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--placement", default="lpt", choices=["lpt", "block"],
                    help="N>1: timed prompts placed on ranks by LPT on predicted work, or contiguous blocks")
    ap.add_argument("--groups", type=int, default=1,
                    help="co-resident prompt groups per GPU (SURVEY §8f NEXT-1); 1 = the paper's setting")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (the driver may also launch us that way)
        import socket
        sock = socket.socket()
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
        sock.close()
        os.execvp(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                   f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
                                   f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:])
    TOP_P[0] = args.top_p
    if args.impl == "reference":
        run_reference(args)
    elif args.groups > 1:
        run_groups(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
