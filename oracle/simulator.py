"""Oracle: discrete-step simulation of one group's sampling loop.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows PAPER.md Alg. 1 (l.218-241) step by step, with the modes of §3.1-3.2:
  full      all G samples decode in parallel (g = G)
  naive     N = G/g micro groups in trace order with a barrier  §3.1 l.164-170
  fifo      fixed-slot continuous sampling, quota N per slot,   §3.2 l.196-198
            trace-order refill                                  (reading R19)
  infinite  Alg. 1: [optional prefix phase of k tokens in ceil(G/g) barriered
            rounds, l.215-216, l.371] -> Alg. 2 plan -> first g samples from the
            mask -> SJF refill (Alg. 3) with no quota           (R17-R22)
  infinite_slots  the same with Alg. 2 over g bins (SPEC bin_mode = slots, l.175,
            l.204, l.255): slot j starts with bin j's head      (R38)
  dynamic   dynamic-slot sampling, §3.2 l.199-200 ("slot is immediately
            reassigned"): g slots, no quota, candidates drawn in trace order from
            the len(true_len) >= target candidates; the run stops at the step of
            the target-th completion and every in-flight sample is discarded
            (R35)

One step = one token for every occupied slot (R20: a step
happens while >= 1 slot is active).  Termination is trace-driven (R5): sample
uid finishes after exactly true_len[uid] tokens.  Several slots finishing in
one step are handled in ascending slot index; a refilled sample decodes its
first token in the next step (R18).

KV accounting ("fixed-size memory pool", l.205 "recycled
upon completion"; R26): each sample owns pages of `page_tokens` tokens,
allocated when it writes token t with t % page_tokens == 0 and released when
it finishes; parked prefix-phase samples keep theirs (l.371).  live_pages[step]
is counted after the step's allocations.
"""
from dataclasses import dataclass, field

from .planner import build_plan


@dataclass
class SimResult:
    total_steps: int = 0
    slot_table: list = field(default_factory=list)   # [step][slot] -> uid or -1
    live_pages: list = field(default_factory=list)   # [step] -> pages allocated
    peak_pages: int = 0
    start_step: dict = field(default_factory=dict)   # uid -> first step decoded (1-based)
    finish_step: dict = field(default_factory=dict)  # uid -> step its last token was decoded
    events: list = field(default_factory=list)       # (step, slot, uid, kind)
    tokens_decoded: int = 0
    prefix_steps: int = 0
    init: list = field(default_factory=list)
    queue: list = field(default_factory=list)
    plan: dict = None
    discarded: list = field(default_factory=list)    # dynamic: in-flight uids at the stop, ascending slot


def simulate(true_len, mode, g, pred=None, eps=0.1, prefix_k=0, page_tokens=16, target=0):
    true_len = [int(x) for x in true_len]
    G = len(true_len)
    if target and (mode != "dynamic" or not 1 <= target <= G):
        raise ValueError("IS_ERR_CONFIG: target needs dynamic mode and 1 <= target <= G")
    if mode == "full":
        g = G
    if g < 1 or G % g != 0:
        raise ValueError("IS_ERR_CONFIG: G mod g != 0")
    N = G // g
    res = SimResult()
    t = [0] * G
    pages = [0] * G
    finished = set()
    slot = [-1] * g
    count = [0] * g              # samples ever run by slot (fifo quota)
    step = 0

    def run_phase(queue, stop_at, barrier, quota, init):
        nonlocal step
        for s, uid in enumerate(init):
            slot[s] = uid if uid is not None else -1
        q = list(queue)
        while any(u >= 0 for u in slot):
            step += 1
            for s in range(g):
                uid = slot[s]
                if uid >= 0:
                    if t[uid] == 0 and uid not in res.start_step:
                        res.start_step[uid] = step
                    if t[uid] % page_tokens == 0:
                        pages[uid] += 1
            live = sum(pages)
            res.live_pages.append(live)
            res.peak_pages = max(res.peak_pages, live)
            res.slot_table.append(list(slot))
            for s in range(g):
                if slot[s] >= 0:
                    t[slot[s]] += 1
                    res.tokens_decoded += 1
            for s in range(g):                     # ascending slot index (R18)
                uid = slot[s]
                if uid < 0:
                    continue
                if t[uid] == true_len[uid]:
                    finished.add(uid)
                    res.finish_step[uid] = step
                    pages[uid] = 0
                    res.events.append((step, s, uid, "finish"))
                    if target and len(finished) == target:   # dynamic: stop, discard in-flight work
                        slot[s] = -1
                        for s2 in range(g):
                            if slot[s2] >= 0:
                                res.discarded.append(slot[s2])
                                res.events.append((step, s2, slot[s2], "discard"))
                                pages[slot[s2]] = 0
                                slot[s2] = -1
                        q.clear()
                        return
                elif t[uid] == stop_at(uid):
                    res.events.append((step, s, uid, "park"))
                else:
                    continue
                slot[s] = -1
                count[s] += 1
                if not barrier and q and (quota == 0 or count[s] < quota):
                    slot[s] = q.pop(0)
                    res.events.append((step, s, slot[s], "refill"))
            if barrier and all(u < 0 for u in slot) and q:
                for s in range(g):
                    if q:
                        slot[s] = q.pop(0)
                        res.events.append((step, s, slot[s], "refill"))

    big = 1 << 30
    if mode in ("full", "naive"):
        p = build_plan(mode, G, g)
        res.init, res.queue = p["init"], p["queue"]
        run_phase(p["queue"], lambda u: big, True, 0, p["init"])
    elif mode == "fifo":
        p = build_plan(mode, G, g)
        res.init, res.queue = p["init"], p["queue"]
        run_phase(p["queue"], lambda u: big, False, N, p["init"])
    elif mode == "dynamic":
        p = build_plan(mode, G, g)
        res.init, res.queue = p["init"], p["queue"]
        target = target or G
        run_phase(p["queue"], lambda u: big, False, 0, p["init"])
    elif mode in ("fptas_only", "sjf_only"):
        if pred is None:
            raise ValueError(f"{mode} mode needs predicted lengths")
        p = build_plan(mode, G, g, pred=pred, eps=eps)
        res.init, res.queue, res.plan = p["init"], p["queue"], p["plan"]
        run_phase(p["queue"], lambda u: big, False, 0, p["init"])
    elif mode in ("infinite", "infinite_slots"):
        if pred is None:
            raise ValueError("infinite mode needs predicted lengths")
        if prefix_k > 0:
            order = list(range(G))
            run_phase(order[g:], lambda u: min(prefix_k, true_len[u]), True, 0, order[:g])
            res.prefix_steps = step
            # R22 / SPEC l.59: samples that finished in the prefix phase have pred = true
            pred = [true_len[i] if true_len[i] <= prefix_k else int(pred[i]) for i in range(G)]
        p = build_plan(mode, G, g, pred=pred, eps=eps, finished=finished)
        res.init, res.queue, res.plan = p["init"], p["queue"], p["plan"]
        count[:] = [0] * g
        run_phase(p["queue"], lambda u: big, False, 0, p["init"])
    else:
        raise ValueError(f"IS_ERR_CONFIG: unknown mode {mode}")
    res.total_steps = step
    assert len(finished) == (target or G)
    return res


def simulate_admit(true_len, g, S, pred, max_new, pool_pages, eps=0.1, page_tokens=16):
    """Memory-aware admission by predicted length ("samples from future micro
    groups may be promoted early if they fit the current memory profile"; NEXT-2, reading R41).

    Alg. 1-3 as in `infinite` on slots 0..g-1 (guaranteed slots: each owns the worst-case
    reservation W = ceil(max_new / page_tokens) pages of R25) plus S - g elastic slots that share
    the rest of the page pool, E = pool_pages - g W pages.  Per step:
      1. pages for the step's token, ascending slot: a guaranteed slot always gets its page; an
         elastic one while the elastic slots hold < E pages; else the lowest idle guaranteed
         slot adopts it now (its pages leave the elastic count) and it gets a guaranteed page;
         else it STALLS (no token this step, keeps its pages; logged as -2 - uid);
      2. every occupied, unstalled slot decodes one token;
      3. finishes in ascending slot order (pages freed);
      4. refill in ascending slot order: an idle guaranteed slot first adopts the stalled elastic
         sample admitted earliest (it moves with its pages, which leave the elastic count), else pops
         the SJF queue head; an idle elastic slot admits the queue head iff the elastic slots'
         reservations sum(max(held, ceil(pred / pt))) plus ceil(pred_head / pt) fit E (SJF order
         kept: a head that does not fit stops admission).
    At the start the g slots take the plan's initial fill and the elastic slots are admitted as
    in 4.  Live pages never exceed pool_pages; a stalled elastic sample is always adopted by the
    next guaranteed slot that frees, so the run terminates.
    """
    true_len = [int(x) for x in true_len]
    pred = [int(p) for p in pred]
    G = len(true_len)
    pt = page_tokens
    W = -(-max_new // pt)
    E = pool_pages - g * W
    if not (g < S and G % g == 0 and E >= 0):
        raise ValueError("IS_ERR_CONFIG: need g < S, G mod g == 0 and a pool of at least g worst-case slots")
    res = SimResult()
    p = build_plan("infinite", G, g, pred=pred, eps=eps)
    res.init, res.queue, res.plan = p["init"], p["queue"], p["plan"]
    q = list(p["queue"])
    slot = [-1] * S
    t = [0] * G
    pages = [0] * G
    seq = {}                      # uid -> admission order
    nseq = [0]
    finished = set()
    step = 0

    def place(s, uid, kind):
        slot[s] = uid
        seq[uid] = nseq[0]
        nseq[0] += 1
        res.events.append((step, s, uid, kind))

    def elastic_reserved():
        return sum(max(pages[u], -(-pred[u] // pt)) for u in slot[g:] if u >= 0)

    def refill(stalled):
        for s in range(S):
            if slot[s] >= 0:
                continue
            if s < g:
                cand = [e for e in range(g, S) if stalled[e] and slot[e] >= 0]
                if cand:
                    e = min(cand, key=lambda e: seq[slot[e]])
                    slot[s], slot[e] = slot[e], -1
                    stalled[e] = False
                    res.events.append((step, s, slot[s], "adopt"))
                elif q:
                    place(s, q.pop(0), "refill")
            elif q and elastic_reserved() + -(-pred[q[0]] // pt) <= E:
                place(s, q.pop(0), "admit")

    for s, uid in enumerate(p["init"]):
        place(s, uid, "init")
    refill([False] * S)
    res.stalls = 0
    while any(u >= 0 for u in slot):
        step += 1
        stalled = [False] * S
        held_e = sum(pages[u] for u in slot[g:] if u >= 0)
        for s in range(S):
            uid = slot[s]
            if uid < 0:
                continue
            if t[uid] % pt == 0:
                if s < g:
                    pages[uid] += 1
                elif held_e < E:
                    pages[uid] += 1
                    held_e += 1
                else:
                    idle = [q for q in range(g) if slot[q] < 0]
                    if idle:
                        slot[idle[0]], slot[s] = uid, -1
                        held_e -= pages[uid]
                        pages[uid] += 1
                        res.events.append((step, idle[0], uid, "adopt"))
                    else:
                        stalled[s] = True
                        res.stalls += 1
        for s in range(S):
            uid = slot[s]
            if uid >= 0 and not stalled[s] and t[uid] == 0 and uid not in res.start_step:
                res.start_step[uid] = step
        live = sum(pages)
        res.live_pages.append(live)
        res.peak_pages = max(res.peak_pages, live)
        res.slot_table.append([(-2 - u if stalled[s] else u) if u >= 0 else -1 for s, u in enumerate(slot)])
        for s in range(S):
            if slot[s] >= 0 and not stalled[s]:
                t[slot[s]] += 1
                res.tokens_decoded += 1
        for s in range(S):
            uid = slot[s]
            if uid >= 0 and not stalled[s] and t[uid] == true_len[uid]:
                finished.add(uid)
                res.finish_step[uid] = step
                pages[uid] = 0
                slot[s] = -1
                res.events.append((step, s, uid, "finish"))
        refill(stalled)
    res.total_steps = step
    assert len(finished) == G
    return res


def step_lower_bound(true_len, g):
    """max(max len, ceil(sum / g))."""
    return max(max(true_len), -(-sum(true_len) // g))
