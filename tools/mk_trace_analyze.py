"""Summarise a persistent-kernel timeline saved by tools/mk_trace.py."""
import sys
import numpy as np

KIND = {0: "EMBED", 1: "QKV", 2: "ATT", 3: "O", 4: "GU", 5: "DN", 6: "FINAL"}
d = np.load(sys.argv[1])
tasks, off, tr = d["tasks"], d["off"], d["trace"].astype(np.int64)
grid = len(off) - 1
t = tr[..., 0]
code = tr[..., 1]
valid = t > 0
t0 = t[valid].min()
typ = (code >> 32)
idx = code & 0xFFFFFFFF
print("kernel span us", (t[valid].max() - t0) / 1e3)
# per (layer, kind): first start / last end of GEMM units
rows = []
ev = {}
for b in range(grid):
    for role in range(4):
        for n in range(t.shape[2]):
            if t[b, role, n] == 0:
                break
            i = int(idx[b, role, n]); ty = int(typ[b, role, n])
            if ty in (5, 6):
                continue
            tk = tasks[off[b] + i]
            kind = tk[0] & 0xFF; layer = (tk[0] >> 8) & 0xFF
            ev.setdefault((layer, kind, ty), []).append((t[b, role, n] - t0) / 1e3)
names = {1: "start", 2: "deps_ok", 3: "acc_ready", 4: "partial_done", 10: "tile_done", 7: "prod_issue", 8: "mma_start", 9: "mma_done"}
for layer in sorted(set(k[0] for k in ev))[:4] + [27]:
    for kind in (1, 3, 4, 5):
        parts = []
        for ty in (7, 8, 1, 2, 3, 9, 10):
            v = ev.get((layer, kind, ty))
            if v:
                parts.append(f"{names[ty]} {min(v):7.1f}-{max(v):7.1f}")
        print(f"L{layer:2d} {KIND[kind]:3s} " + " | ".join(parts))
# attention units per layer
att = {}
for b in range(grid):
    for role in range(2):
        for n in range(t.shape[2]):
            if t[b, role, n] == 0:
                break
            if typ[b, role, n] == 5:
                s = t[b, role, n]
                e = t[b, role, n + 1] if n + 1 < t.shape[2] else s
                att.setdefault(b, []).append(((s - t0) / 1e3, (e - s) / 1e3))
allu = sorted(x for v in att.values() for x in v)
print("attention units", len(allu), "mean dur us", np.mean([x[1] for x in allu]) if allu else 0,
      "max", max(x[1] for x in allu) if allu else 0)
