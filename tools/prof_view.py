"""Summarise a TQ_PROFILE dump: per role, mean cycles in each timed slot."""
import sys
import numpy as np
a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 32, 8).astype(np.int64)
NAMES = {0: ("code", ["c_empty", "e_empty", "bulk_issue", "-"]), 3: ("mma2/xprod", ["full/x_empty", "d_empty", "chunks(n)", "x_full"]),
         1: ("mma", ["full", "d_empty", "chunks(n)", "x_full"]), 2: ("mma1", ["full", "d_empty", "chunks(n)", "x_full"])}
rows = {}
for cta in range(a.shape[0]):
    for w in range(32):
        r = a[cta, w]
        if r[0] <= 0:
            continue
        role = int(r[1])
        rows.setdefault(role, []).append(r)
for role in sorted(rows):
    r = np.array(rows[role])
    if role in NAMES:
        name, slots = NAMES[role]
    elif role >= 4 and role < 4 + 4 * 4 and any(k in rows for k in ()):
        name, slots = "dq", []
    else:
        name, slots = f"role{role}", ["s0", "s1", "s2", "s3"]
    if role >= 4 and name.startswith("role"):
        name = "dequant" if role < max(rows) - 3 else "epilogue"
        slots = ["wait_st+arrive", "c_full+lds", "dq+st", "empty"] if name == "dequant" else ["d_full", "-", "-", "-"]
    tot = r[:, 0].mean()
    parts = " ".join(f"{s}={r[:, 2 + k].mean():9.0f} ({r[:, 2 + k].mean() / tot * 100:4.1f}%)" for k, s in enumerate(slots) if s != "-")
    print(f"{name:9s} role={role:2d} n={len(r):4d} total={tot:9.0f}  {parts}")
# prologue cycles and the spread of CTA start times (globaltimer, ns)
pro = [int(a[c, w, 6]) for c in range(a.shape[0]) for w in range(32) if a[c, w, 0] > 0]
ent = np.array([int(a[c, 0, 7]) for c in range(a.shape[0]) if a[c, 0, 0] > 0])
if len(pro):
    print(f"prologue cycles: mean {np.mean(pro):.0f} max {np.max(pro):.0f}; CTA entry spread {(ent.max() - ent.min()) / 1e3:.2f} us")

# per-CTA spans (row 31: units, exit globaltimer)
ex = np.array([int(a[c, 31, 7]) for c in range(a.shape[0]) if a[c, 31, 7] > 0])
if len(ex) and len(ent):
    units = np.array([int(a[c, 31, 1]) for c in range(a.shape[0]) if a[c, 31, 7] > 0])
    dur = (ex - ent[:len(ex)]) / 1e3
    print(f"CTA span us: min {dur.min():.2f} median {np.median(dur):.2f} max {dur.max():.2f}; kernel span {(ex.max() - ent.min()) / 1e3:.2f} us; "
          f"units/CTA min {units.min()} max {units.max()}; slowest CTAs {np.argsort(-dur)[:5].tolist()} units {units[np.argsort(-dur)[:5]].tolist()}")
