"""Per-kind latency breakdown of GEMM units from a persistent-kernel trace."""
import sys
import numpy as np
KIND = {1: "QKV", 3: "O", 4: "GU", 5: "DN"}
d = np.load(sys.argv[1])
tasks, off, tr = d["tasks"], d["off"], d["trace"].astype(np.int64)
grid = len(off) - 1
per = {}
merged = {}
kinds_of = {}
for b in range(grid):
    for role in range(4):
        recs = {}
        prev_t = 0
        for n in range(tr.shape[2]):
            t, c = tr[b, role, n]
            if t == 0 or t < prev_t:  # stale tail from an older step
                break
            prev_t = t
            ty, i = c >> 32, c & 0xFFFFFFFF
            if ty in (5, 6):
                continue
            recs.setdefault(int(i), {})[int(ty)] = t
        for i, r in recs.items():
            kind = tasks[off[b] + i][0] & 0xFF
            if kind not in KIND:
                continue
            key = (b, i)
            merged.setdefault(key, {}).update(r)
            kinds_of[key] = kind
for key, r in merged.items():
    per.setdefault(kinds_of[key], []).append(r)
pairs = [(1, 2, "wait deps"), (2, 16, "fill loads"), (16, 17, "fill write"), (7, 18, "A first stage(prod->mma)"), (2, 18, "deps->A ready"), (17, 19, "fill->mma sees B"), (19, 20, "mma kb loop"), (20, 3, "last kb->acc"), (2, 3, "B load+MMA"), (3, 11, "partial st+fence"), (11, 12, "atomic"),
         (12, 13, "reduce ld"), (3, 13, "acc->reduced"), (13, 14, "rowscale"), (14, 15, "epilogue"), (15, 10, "fence+signal"),
         (1, 10, "total(last)"), (1, 4, "total(non-last)")]
for kind, lst in per.items():
    out = []
    for a, b_, name in pairs:
        v = [r[b_] - r[a] for r in lst if a in r and b_ in r]
        if v:
            out.append(f"{name} {np.median(v)/1e3:.2f}/{np.max(v)/1e3:.2f}")
    print(KIND[kind], len(lst), " | ".join(out))
