"""Thin ctypes binding of libinfsamp (include/infsamp.h).

Argument marshalling only: every step of the decode path runs in the CUDA
kernels of libinfsamp.so.  There is no Python or CPU fallback; if the shared
library is missing or the device is not sm_100 the calls raise.
"""
import ctypes
import os

import numpy as np

from . import build as _build

IS_OK, IS_ERR_CONFIG, IS_ERR_BUDGET, IS_ERR_CAPACITY, IS_ERR_DATA, IS_ERR_STATE, IS_ERR_CUDA = range(7)
MODES = {"full": 0, "naive": 1, "fifo": 2, "infinite": 3, "fptas_only": 4, "sjf_only": 5, "dynamic": 6}
ADV_MODES = {"std_norm": 0, "mean_only": 1}

EXPORTS = ["is_plan", "is_create", "is_destroy", "is_prefill", "is_start_group", "is_decode_step",
           "is_refill", "is_run_group", "is_query", "is_copy_tokens", "is_copy_schedule",
           "is_group_results", "is_group_advantages", "is_set_logits_dump", "is_profile_step",
           "is_profile_step_graph", "is_profile_kernel", "is_dbg_topp", "is_dbg_attn",
           "is_dbg_gemm", "is_dbg_copy", "is_prefill_slot", "is_start_group_slot",
           "is_run_until_any_done", "is_query_slot", "is_copy_tokens_slot", "is_copy_schedule_slot",
           "is_group_results_slot", "is_nccl_unique_id", "is_nccl_comm_init", "is_allgather_results", "is_allgather_results_n",
           "is_nccl_comm_destroy", "is_copy_logprobs", "is_copy_logprobs_slot", "is_kl_rewards", "is_grpo_objective", "is_last_error",
           "is_version"]


class InfsampError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


class Shape(ctypes.Structure):
    _fields_ = [("layers", ctypes.c_int32), ("hidden", ctypes.c_int32), ("n_q_heads", ctypes.c_int32),
                ("n_kv_heads", ctypes.c_int32), ("head_dim", ctypes.c_int32), ("ffn", ctypes.c_int32),
                ("vocab", ctypes.c_int32), ("rms_eps", ctypes.c_float), ("rope_theta", ctypes.c_float)]


class Config(ctypes.Structure):
    _fields_ = [("shape", Shape), ("G", ctypes.c_int32), ("g", ctypes.c_int32),
                ("max_new_tokens", ctypes.c_int32), ("prompt_len", ctypes.c_int32),
                ("prefix_k", ctypes.c_int32), ("page_tokens", ctypes.c_int32),
                ("row_capacity", ctypes.c_int32), ("kv_budget_bytes", ctypes.c_int64),
                ("eps", ctypes.c_double), ("temperature", ctypes.c_float), ("seed", ctypes.c_uint64),
                ("mode", ctypes.c_int32), ("decode_impl", ctypes.c_int32), ("max_groups", ctypes.c_int32),
                ("dynamic_target", ctypes.c_int32), ("eos_enabled", ctypes.c_int32), ("eos_id", ctypes.c_int32),
                ("bin_slots", ctypes.c_int32), ("admit_slots", ctypes.c_int32), ("top_p", ctypes.c_float)]


class PlanOut(ctypes.Structure):
    _fields_ = [("mask", ctypes.POINTER(ctypes.c_int32)), ("scaled_len", ctypes.POINTER(ctypes.c_int64)),
                ("loads", ctypes.POINTER(ctypes.c_int64)), ("overflow_ids", ctypes.POINTER(ctypes.c_int32)),
                ("init_slots", ctypes.POINTER(ctypes.c_int32)),
                ("refill_queue", ctypes.POINTER(ctypes.c_int32)), ("K", ctypes.c_double),
                ("capacity", ctypes.c_int64), ("n_overflow", ctypes.c_int32), ("queue_len", ctypes.c_int32),
                ("reserved_bytes", ctypes.c_int64)]


class Stats(ctypes.Structure):
    _fields_ = [("steps", ctypes.c_int32), ("prefix_steps", ctypes.c_int32), ("completed", ctypes.c_int32),
                ("live_pages", ctypes.c_int32), ("peak_pages", ctypes.c_int32), ("error", ctypes.c_int32),
                ("tokens_decoded", ctypes.c_int64), ("peak_kv_bytes", ctypes.c_int64),
                ("page_bytes", ctypes.c_int64), ("prefix_bytes", ctypes.c_int64),
                ("num_pages", ctypes.c_int32), ("row_capacity", ctypes.c_int32),
                ("suffix_tokens", ctypes.c_int64),
                ("groups", ctypes.c_int32), ("global_steps", ctypes.c_int64), ("global_peak_kv_bytes", ctypes.c_int64),
                ("launches_per_step", ctypes.c_int32), ("launches_per_prefill", ctypes.c_int32),
                ("discarded", ctypes.c_int32), ("stalls", ctypes.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_LIB = None


def lib_path():
    return _build.OUT


def load(build_if_missing=True):
    """Load libinfsamp.so (building it in-tree first if it is missing or stale)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if build_if_missing:
        try:
            _build.build()
        except Exception:
            if not os.path.exists(_build.OUT):
                raise
    if not os.path.exists(_build.OUT):
        raise InfsampError(IS_ERR_STATE, f"libinfsamp.so not found at {_build.OUT}; run paper_2506_22950_b200.build")
    L = ctypes.CDLL(_build.OUT)
    vp, i32, i64p = ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_int64)
    L.is_plan.argtypes = [ctypes.POINTER(Config), vp, vp, ctypes.POINTER(PlanOut)]
    L.is_create.argtypes = [ctypes.POINTER(Config), ctypes.POINTER(ctypes.c_void_p), i32, vp, ctypes.POINTER(vp)]
    L.is_destroy.argtypes = [vp]
    L.is_destroy.restype = None
    L.is_prefill.argtypes = [vp, vp, i32]
    L.is_start_group.argtypes = [vp, vp, vp]
    L.is_decode_step.argtypes = [vp, vp, vp]
    L.is_refill.argtypes = [vp, vp, vp]
    L.is_run_group.argtypes = [vp, i32, ctypes.POINTER(i32)]
    L.is_query.argtypes = [vp, ctypes.POINTER(Stats)]
    L.is_copy_tokens.argtypes = [vp, vp, i32]
    L.is_copy_schedule.argtypes = [vp, vp, vp, i32, ctypes.POINTER(i32)]
    L.is_group_results.argtypes = [vp, vp, vp]
    L.is_group_advantages.argtypes = [vp, i32, i32, vp]
    L.is_set_logits_dump.argtypes = [vp, vp]
    L.is_profile_step.argtypes = [vp, vp, vp, i32, ctypes.POINTER(i32)]
    L.is_profile_step_graph.argtypes = [vp, vp, vp, i32, ctypes.POINTER(i32)]
    L.is_profile_kernel.argtypes = [vp, i32, i32, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(i32)]
    L.is_dbg_gemm.argtypes = [vp, vp, vp, i32, i32, i32, i32, vp]
    L.is_dbg_topp.argtypes = [vp, i32, i32, ctypes.c_float, ctypes.c_float, ctypes.c_uint64, vp, vp, vp, vp]
    L.is_dbg_copy.argtypes = [vp, i32, vp, ctypes.c_int64]
    L.is_dbg_attn.argtypes = [vp, vp, i32, i32, i32, vp, i32, i32, vp, i32, vp, i32, i32, i32, i32, vp, vp, i32,
                              ctypes.POINTER(ctypes.c_float), vp]
    L.is_prefill_slot.argtypes = [vp, i32, vp, i32]
    L.is_start_group_slot.argtypes = [vp, i32, vp, vp]
    L.is_run_until_any_done.argtypes = [vp, i32, ctypes.POINTER(i32), i64p]
    L.is_query_slot.argtypes = [vp, i32, ctypes.POINTER(Stats)]
    L.is_copy_tokens_slot.argtypes = [vp, i32, vp, i32]
    L.is_copy_schedule_slot.argtypes = [vp, i32, vp, vp, i32, ctypes.POINTER(i32)]
    L.is_group_results_slot.argtypes = [vp, i32, vp, vp]
    L.is_nccl_unique_id.argtypes = [vp]
    L.is_nccl_comm_init.argtypes = [vp, i32, i32, ctypes.POINTER(vp)]
    L.is_allgather_results.argtypes = [vp, vp, vp, vp, vp, vp]
    L.is_allgather_results_n.argtypes = [vp, vp, i32, vp, vp, vp, vp]
    L.is_nccl_comm_destroy.argtypes = [vp]
    L.is_copy_logprobs.argtypes = [vp, vp]
    L.is_kl_rewards.argtypes = [vp, vp, vp, vp, i32, i32, ctypes.c_float, vp]
    L.is_grpo_objective.argtypes = [vp, vp, vp, vp, vp, i32, i32, ctypes.c_float, ctypes.c_float,
                                    ctypes.POINTER(ctypes.c_double)]
    L.is_copy_logprobs_slot.argtypes = [vp, i32, vp]
    L.is_last_error.restype = ctypes.c_char_p
    L.is_last_error.argtypes = []
    L.is_version.restype = ctypes.c_char_p
    for name in EXPORTS:
        if name not in ("is_destroy", "is_last_error", "is_version"):
            getattr(L, name).restype = ctypes.c_int
    _LIB = L
    return L


def _check(status):
    if status != IS_OK:
        raise InfsampError(status, _LIB.is_last_error().decode())


def _np_ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def make_config(shape, G, g, max_new_tokens, prompt_len, mode="infinite", prefix_k=0, page_tokens=16,
                row_capacity=0, kv_budget_bytes=0, eps=0.1, temperature=0.8, seed=20261017,
                max_groups=1, dynamic_target=0, top_p=1.0, eos_id=None, admit_slots=0):
    c = Config()
    c.shape = Shape(shape.layers, shape.hidden, shape.n_q_heads, shape.n_kv_heads, shape.head_dim, shape.ffn,
                    shape.vocab, shape.rms_eps, shape.rope_theta)
    c.G, c.g, c.max_new_tokens, c.prompt_len = G, g, max_new_tokens, prompt_len
    c.prefix_k, c.page_tokens, c.row_capacity = prefix_k, page_tokens, row_capacity
    c.kv_budget_bytes, c.eps, c.temperature, c.seed = kv_budget_bytes, eps, temperature, seed
    c.bin_slots = 0
    c.admit_slots = admit_slots  # memory-aware admission by predicted length (DESIGN R41): 0 = off
    if mode == "infinite_slots":  # Alg. 2 over g slot bins (SPEC bin_mode = slots, DESIGN R38)
        mode, c.bin_slots = "infinite", 1
    c.mode = MODES[mode] if isinstance(mode, str) else int(mode)
    c.decode_impl = 0  # reserved (include/infsamp.h)
    c.max_groups = max_groups
    c.dynamic_target = dynamic_target
    c.top_p = top_p
    c.eos_enabled, c.eos_id = (0, 0) if eos_id is None else (1, int(eos_id))
    return c


def is_plan(cfg, pred_len, finished=None):
    """Alg. 2 + initial fill + SJF queue + budget check (host)."""
    L = load()
    G = cfg.G
    g = G if cfg.mode == MODES["full"] else cfg.g
    N = max(G // g if g else 1, g)  # loads has G/g entries, or g with bin_slots
    mask = np.zeros(2 * G, np.int32)
    sl = np.zeros(G, np.int64)
    loads = np.zeros(max(N, 1), np.int64)
    ovf = np.zeros(G, np.int32)
    init = np.zeros(max(g, 1), np.int32)
    queue = np.zeros(G, np.int32)
    out = PlanOut(mask.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), sl.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                  loads.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ovf.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                  init.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), queue.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                  0.0, 0, 0, 0, 0)
    pred = None if pred_len is None else np.ascontiguousarray(pred_len, np.int32)
    fin = None if finished is None else np.ascontiguousarray(finished, np.uint8)
    _check(L.is_plan(ctypes.byref(cfg), None if pred is None else _np_ptr(pred),
                     None if fin is None else _np_ptr(fin), ctypes.byref(out)))
    nb = g if cfg.bin_slots else (G // g if g else 1)
    return dict(mask=[(int(mask[2 * i]), int(mask[2 * i + 1])) for i in range(G)], scaled=[int(x) for x in sl],
                loads=[int(x) for x in loads[:nb]], overflow=[int(x) for x in ovf[:out.n_overflow]],
                init=[int(x) for x in init[:g]], queue=[int(x) for x in queue[:out.queue_len]], K=out.K,
                capacity=out.capacity, reserved_bytes=out.reserved_bytes)


def is_group_advantages(rewards, mode="std_norm"):
    L = load()
    r = np.ascontiguousarray(rewards, np.float32)
    a = np.zeros_like(r)
    _check(L.is_group_advantages(_np_ptr(r), len(r), ADV_MODES[mode], _np_ptr(a)))
    return a


def is_dbg_topp(logits, uid, t, temperature, top_p, seed, stream=0):
    """Top-p chain on device logits [rows][V] fp32 with int32 uid / t per row; returns tokens."""
    import torch
    rows, V = logits.shape
    tok = torch.empty(rows, dtype=torch.int32, device=logits.device)
    _check(load().is_dbg_topp(logits.data_ptr(), rows, V, float(temperature), float(top_p), int(seed),
                              uid.data_ptr(), t.data_ptr(), tok.data_ptr(), stream))
    return tok


def is_dbg_gemm(w, x, y, split=1, stream=0):
    """Y[rows][M] (fp32) = X[rows][K] . W[M][K]^T on the tcgen05 kernel (device tensors)."""
    L = load()
    M, K = w.shape
    _check(L.is_dbg_gemm(w.data_ptr(), x.data_ptr(), y.data_ptr(), M, K, x.shape[0], split, stream))


def is_dbg_attn(q, prefix, pool, pagetab, row_len, grp_rows, impl=0, out_f32=None, reps=0, stream=0):
    """Decode split attention of one layer on caller device tensors (include/infsamp.h):
    q [rows][Hq][128] bf16, prefix [groups][2][Hkv][plen][128] bf16, pool [pages][2][Hkv][pt][128]
    bf16, pagetab [rows][maxp] int32, row_len [rows] int32.  Returns (out bf16 [rows][Hq][128],
    per-rep milliseconds)."""
    import torch
    rows, Hq, _ = q.shape
    groups, _, Hkv, plen, _ = prefix.shape
    num_pages, _, _, pt, _ = pool.shape
    out = torch.zeros(rows, Hq, 128, dtype=torch.bfloat16, device=q.device)
    ms = (ctypes.c_float * max(reps, 1))()
    _check(load().is_dbg_attn(q.data_ptr(), prefix.data_ptr(), plen, groups, grp_rows, pool.data_ptr(), num_pages,
                              pt, pagetab.data_ptr(), pagetab.shape[1], row_len.data_ptr(), rows, Hq, Hkv, impl,
                              out.data_ptr(), None if out_f32 is None else out_f32.data_ptr(), reps, ms, stream))
    return out, [float(ms[i]) for i in range(reps)]


def weight_pointer_list(weights, layers):
    from synth import GLOBAL_WEIGHT_NAMES, layer_weight_names
    names = list(GLOBAL_WEIGHT_NAMES)
    for l in range(layers):
        names += layer_weight_names(l)
    ptrs = []
    for n in names:
        t = weights[n]
        if not t.is_cuda or not t.is_contiguous():
            raise InfsampError(IS_ERR_DATA, f"weight {n} must be a contiguous CUDA tensor")
        ptrs.append(t.data_ptr())
    return ptrs


def is_kl_rewards(rm, logp, logp_ref, lengths, beta):
    """P:311 KL-penalised reward (host): rm[G], logp / logp_ref [G][T], lengths[G]."""
    rm = np.ascontiguousarray(rm, np.float32)
    lp = np.ascontiguousarray(logp, np.float32)
    lr = np.ascontiguousarray(logp_ref, np.float32)
    ln = np.ascontiguousarray(lengths, np.int32)
    out = np.zeros(len(rm), np.float32)
    _check(load().is_kl_rewards(_np_ptr(rm), _np_ptr(lp), _np_ptr(lr), _np_ptr(ln), len(rm), lp.shape[1],
                                float(beta), _np_ptr(out)))
    return out


def is_grpo_objective(logp, logp_old, logp_ref, adv, lengths, clip_eps=0.2, beta=0.04):
    """Eq. 3 / Eq. 4 objective value (host, fp64)."""
    a = [np.ascontiguousarray(x, np.float32) for x in (logp, logp_old, logp_ref, adv)]
    ln = np.ascontiguousarray(lengths, np.int32)
    out = ctypes.c_double()
    _check(load().is_grpo_objective(_np_ptr(a[0]), _np_ptr(a[1]), _np_ptr(a[2]), _np_ptr(a[3]), _np_ptr(ln),
                                    len(ln), a[0].shape[1], float(clip_eps), float(beta), ctypes.byref(out)))
    return out.value


def nccl_unique_id():
    """128-byte ncclUniqueId (rank 0); broadcast it to the other ranks."""
    buf = (ctypes.c_char * 128)()
    _check(load().is_nccl_unique_id(buf))
    return bytes(buf)


def nccl_comm_init(uid, rank, world):
    """Join the communicator; returns an opaque handle (pass to is_allgather_results / nccl_comm_destroy)."""
    buf = (ctypes.c_char * 128).from_buffer_copy(uid)
    comm = ctypes.c_void_p()
    _check(load().is_nccl_comm_init(buf, int(rank), int(world), ctypes.byref(comm)))
    return comm


def nccl_comm_destroy(comm):
    _check(load().is_nccl_comm_destroy(comm))


class Context:
    """Owning handle of an is_ctx (library-owned device state for one GPU)."""

    def __init__(self, cfg, weights, stream=None):
        import torch
        L = load()
        self.cfg = cfg
        self.G = cfg.G
        self.g = cfg.G if cfg.mode == MODES["full"] else (cfg.admit_slots or cfg.g)  # slots per group
        ptrs = weight_pointer_list(weights, cfg.shape.layers)
        arr = (ctypes.c_void_p * len(ptrs))(*ptrs)
        h = ctypes.c_void_p()
        st = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        self._stream = st
        _check(L.is_create(ctypes.byref(cfg), arr, len(ptrs), ctypes.c_void_p(st), ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            load().is_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def is_prefill(self, d_prompt, prompt_id, slot=0):
        _check(load().is_prefill_slot(self._h, int(slot), d_prompt.data_ptr(), int(prompt_id)))

    def is_start_group(self, true_len, pred_len=None, slot=0):
        t = np.ascontiguousarray(true_len, np.int32)
        p = None if pred_len is None else np.ascontiguousarray(pred_len, np.int32)
        _check(load().is_start_group_slot(self._h, int(slot), _np_ptr(t), None if p is None else _np_ptr(p)))

    def is_run_until_any_done(self, max_steps=1 << 30):
        """Decode until a started group completes: (done-slot mask, global decode steps so far)."""
        mask = ctypes.c_int32()
        steps = ctypes.c_int64()
        _check(load().is_run_until_any_done(self._h, int(min(max_steps, 2 ** 31 - 1)), ctypes.byref(mask),
                                            ctypes.byref(steps)))
        return mask.value, steps.value

    def is_decode_step(self, d_next=None, d_fin=None):
        _check(load().is_decode_step(self._h, None if d_next is None else d_next.data_ptr(),
                                     None if d_fin is None else d_fin.data_ptr()))

    def is_refill(self, d_fin=None, d_new_uid=None):
        _check(load().is_refill(self._h, None if d_fin is None else d_fin.data_ptr(),
                                None if d_new_uid is None else d_new_uid.data_ptr()))

    def is_run_group(self, max_steps=1 << 30):
        n = ctypes.c_int32()
        _check(load().is_run_group(self._h, int(min(max_steps, 2 ** 31 - 1)), ctypes.byref(n)))
        return n.value

    def is_query(self, slot=0):
        s = Stats()
        _check(load().is_query_slot(self._h, int(slot), ctypes.byref(s)))
        return s.as_dict()

    def is_copy_tokens(self, slot=0):
        out = np.zeros((self.G, self.cfg.max_new_tokens), np.int32)
        _check(load().is_copy_tokens_slot(self._h, int(slot), _np_ptr(out), 0))
        return out

    def is_copy_logprobs(self, slot=0):
        out = np.zeros((self.G, self.cfg.max_new_tokens), np.float32)
        _check(load().is_copy_logprobs_slot(self._h, int(slot), _np_ptr(out)))
        return out

    def is_copy_schedule(self, max_steps=None, slot=0):
        if max_steps is None:
            max_steps = self.is_query(slot)["steps"]
        slots = np.zeros((max(max_steps, 1), self.g), np.int32)
        live = np.zeros(max(max_steps, 1), np.int32)
        n = ctypes.c_int32()
        _check(load().is_copy_schedule_slot(self._h, int(slot), _np_ptr(slots), _np_ptr(live), max_steps,
                                            ctypes.byref(n)))
        return slots[:n.value], live[:n.value]

    def is_group_results(self, d_reward, d_len, slot=0):
        _check(load().is_group_results_slot(self._h, int(slot), d_reward.data_ptr(), d_len.data_ptr()))

    def is_allgather_results(self, comm, d_len, d_reward, d_all_len, d_all_reward):
        _check(load().is_allgather_results(self._h, comm, d_len.data_ptr(), d_reward.data_ptr(),
                                           d_all_len.data_ptr(), d_all_reward.data_ptr()))

    def is_allgather_results_n(self, comm, d_len, d_reward, d_all_len, d_all_reward):
        """One all-gather of this rank's n = d_len.numel() (length, reward) pairs."""
        _check(load().is_allgather_results_n(self._h, comm, int(d_len.numel()), d_len.data_ptr(), d_reward.data_ptr(),
                                             d_all_len.data_ptr(), d_all_reward.data_ptr()))

    def is_set_logits_dump(self, d_logits):
        _check(load().is_set_logits_dump(self._h, None if d_logits is None else d_logits.data_ptr()))

    def is_dbg_copy(self, which, nbytes):
        out = np.zeros(nbytes, np.uint8)
        _check(load().is_dbg_copy(self._h, int(which), _np_ptr(out), nbytes))
        return out

    def is_profile_kernel(self, kind, reps=4):
        ms = ctypes.c_float()
        n = ctypes.c_int32()
        _check(load().is_profile_kernel(self._h, int(kind), int(reps), ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def is_profile_step(self, cap=4096, graph=False):
        ms = np.zeros(cap, np.float32)
        kind = np.zeros(cap, np.int32)
        n = ctypes.c_int32()
        fn = load().is_profile_step_graph if graph else load().is_profile_step
        _check(fn(self._h, _np_ptr(ms), _np_ptr(kind), cap, ctypes.byref(n)))
        return ms[:n.value], kind[:n.value]
