"""Oracle: Alg. 2 (FPTAS micro-group assignment), Alg. 3 (SJF refill), plan
construction, KV budget check, and the brute-force / LPT references.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

fptas_plan follows PAPER.md Alg. 2 (l.243-271) line by line:
    S <- sum l^_i,  K <- eps*S/N                         (l.254)
    l~_i <- ceil(l^_i / K)                                (l.255-257)
    C~ <- ceil(sum l~_i / N)                              (l.258)
    for i sorted by descending l~_i:                      (l.260)
        for n = 1..N: if L_n + l~_i <= C~: assign, break  (l.261-267)
with the DESIGN.md readings: K in IEEE double evaluated as (eps*S)/N (R14);
ties in the sort -> ascending id; an item that fits no group goes to the
least-loaded group (ties -> lowest index) and is recorded as overflow (R15,
SPEC.md l.121).

sjf_refill follows Alg. 3 (l.280-295) with "i not in mask" read as "not yet
started" (R17); ties -> ascending id.

build_plan adds Alg. 1's "first g samples from mask" (l.230, reading R13:
lexicographic (n, j) order, skipping samples finished in the prefix phase) and
the refill queue.  Because Alg. 3's candidate set and key are static (R17),
repeated SJF refills pop the unstarted samples in ascending (l^, id) order;
`refill_queue` is that sequence, and tests check it against repeated
sjf_refill calls.
"""
import math
from itertools import product


class PlanError(ValueError):
    pass


def fptas_plan(pred, N, eps):
    """Alg. 2.  Returns dict(mask, scaled, K, capacity, loads, groups, overflow)."""
    if N <= 0 or not eps > 0:
        raise PlanError("IS_ERR_CONFIG: N must be >= 1 and eps > 0")
    pred = [int(p) for p in pred]
    if any(p < 1 for p in pred):
        raise PlanError("IS_ERR_DATA: predicted lengths must be >= 1")
    G = len(pred)
    S = sum(pred)
    K = (eps * S) / N
    lt = [math.ceil(p / K) for p in pred]
    Ct = -(-sum(lt) // N)
    loads = [0] * N
    groups = [[] for _ in range(N)]
    mask = [None] * G
    overflow = []
    for i in sorted(range(G), key=lambda i: (-lt[i], i)):
        target = None
        for n in range(N):
            if loads[n] + lt[i] <= Ct:
                target = n
                break
        if target is None:
            target = min(range(N), key=lambda n: (loads[n], n))
            overflow.append(i)
        mask[i] = (target + 1, len(groups[target]))
        groups[target].append(i)
        loads[target] += lt[i]
    return dict(mask=mask, scaled=lt, K=K, capacity=Ct, loads=loads,
                groups=groups, overflow=overflow)


def sjf_refill(pred, finished, started):
    """Alg. 3: argmin over C = {i not finished, not started} of pred, ties -> lowest id."""
    cand = [i for i in range(len(pred)) if i not in finished and i not in started]
    if not cand:
        return None
    return min(cand, key=lambda i: (pred[i], i))


def build_plan(mode, G, g, pred=None, eps=0.1, finished=()):
    """Initial slot fill + static refill queue for one group.

    mode: 'full' | 'naive' | 'fifo' | 'infinite' | 'infinite_slots' | 'fptas_only' | 'sjf_only' | 'dynamic'.
    dynamic (R35): the G candidates in trace order, no quota.
    `finished` = samples that completed in the prefix phase (infinite only).
    Table 2's decomposition is undefined in the paper; SPEC.md's
    definitions (R23): fptas_only = the Alg. 2 plan executed in its
    lexicographic (n, j) order with FIFO refill; sjf_only = trace-order start
    (samples 0..g-1) with the Alg. 3 SJF refill of the rest.
    """
    if g < 1 or g > G or G % g != 0:
        raise PlanError("IS_ERR_CONFIG: need 1 <= g <= G and G mod g == 0")
    if mode == "full":
        return dict(init=list(range(G)), queue=[], plan=None)
    if mode in ("naive", "fifo", "dynamic"):
        return dict(init=list(range(g)), queue=list(range(g, G)), plan=None)
    if mode == "sjf_only":
        init = list(range(g))
        started = set(init)
        queue = []
        while True:
            j = sjf_refill(pred, set(), started)
            if j is None:
                break
            queue.append(j)
            started.add(j)
        return dict(init=init, queue=queue, plan=None)
    if mode == "fptas_only":
        plan = fptas_plan(pred, G // g, eps)
        lex = sorted(range(G), key=lambda i: plan["mask"][i])
        return dict(init=lex[:g], queue=lex[g:], plan=plan)
    if mode == "infinite_slots":
        # SPEC.md l.175 / l.204 / l.255 (bin_mode = slots): Alg. 2 with g bins instead of N
        # groups; slot j starts with the head of bin j (its first member in Alg. 2's placement
        # order that did not finish in the prefix phase); an empty bin's slot takes the SJF
        # queue head, in ascending slot order (DESIGN R38); the rest is the Alg. 3 SJF queue.
        plan = fptas_plan(pred, g, eps)
        fin = set(finished)
        heads = []
        for j in range(g):
            members = [i for i in plan["groups"][j] if i not in fin]
            heads.append(members[0] if members else None)
        started = set(i for i in heads if i is not None)
        queue = []
        while True:
            j = sjf_refill(pred, fin, started)
            if j is None:
                break
            queue.append(j)
            started.add(j)
        init = []
        for h in heads:
            if h is None:
                h = queue.pop(0) if queue else -1
            init.append(h)
        return dict(init=init, queue=queue, plan=plan)
    if mode != "infinite":
        raise PlanError(f"IS_ERR_CONFIG: unknown mode {mode}")
    N = G // g
    plan = fptas_plan(pred, N, eps)
    fin = set(finished)
    lex = sorted(range(G), key=lambda i: plan["mask"][i])
    lex = [i for i in lex if i not in fin]
    init = lex[:g]
    started = set(init)
    queue = []
    while True:
        j = sjf_refill(pred, fin, started)
        if j is None:
            break
        queue.append(j)
        started.add(j)
    return dict(init=init, queue=queue, plan=plan)


def reservation_bytes(G, g, max_new, prefix_k, page_tokens, page_bytes, prefix_bytes):
    """Worst-case live KV (R25): prefix + g full-length samples +
    (G-g) parked prefix-phase samples."""
    per_full = -(-max_new // page_tokens)
    per_park = -(-prefix_k // page_tokens) if prefix_k > 0 else 0
    return prefix_bytes + g * per_full * page_bytes + (G - g) * per_park * page_bytes


def lpt_plan(lengths, g):
    """longest-processing-time; ties -> lowest-index slot."""
    loads = [0] * g
    queues = [[] for _ in range(g)]
    for i in sorted(range(len(lengths)), key=lambda i: (-lengths[i], i)):
        s = min(range(g), key=lambda s: (loads[s], s))
        queues[s].append(i)
        loads[s] += lengths[i]
    return queues, max(loads)


def optimal_makespan(lengths, g, max_jobs=16):
    """exact min makespan by exhaustive search with pruning."""
    n = len(lengths)
    if n > max_jobs:
        raise PlanError("IS_ERR_CAPACITY: instance too large for exact search")
    if n == 0:
        return 0
    jobs = sorted(lengths, reverse=True)
    best = [lpt_plan(lengths, g)[1]]
    lb = max(max(jobs), -(-sum(jobs) // g))
    loads = [0] * g

    def rec(k):
        if best[0] == lb:
            return
        if k == n:
            best[0] = min(best[0], max(loads))
            return
        seen = set()
        for s in range(g):
            if loads[s] in seen:
                continue
            seen.add(loads[s])
            if loads[s] + jobs[k] >= best[0]:
                continue
            loads[s] += jobs[k]
            rec(k + 1)
            loads[s] -= jobs[k]

    rec(0)
    return best[0]


def optimal_makespan_bruteforce(lengths, g):
    """Plain enumeration of every assignment (g^n); tiny n only (test pin)."""
    best = None
    for assign in product(range(g), repeat=len(lengths)):
        loads = [0] * g
        for i, s in enumerate(assign):
            loads[s] += lengths[i]
        m = max(loads)
        best = m if best is None else min(best, m)
    return best


def optimal_partition_bruteforce(lengths, N):
    """min over partitions into N groups of the max group sum (Alg. 2's objective, l.247)."""
    return optimal_makespan_bruteforce(lengths, N)
