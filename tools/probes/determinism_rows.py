import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np
os.environ["HSVD_TWO_STAGE_MIN_N"] = "1"
os.environ["HSVD_BACK_SKIP"] = "1"
import paper_1710_02812_b200 as H
count, n, kk = 64, 256, 200
rng = np.random.default_rng(5)
a = np.empty((count, n, n))
for g in range(count):
    u = np.linalg.qr(rng.standard_normal((n, n)))[0]
    s = np.concatenate([100 * np.exp(-0.05 * np.arange(1, 41)), 1e-3 * (1 + 0.05 * rng.standard_normal(n - 40))])
    a[g] = (u * s ** 2) @ u.T
    a[g] = 0.5 * (a[g] + a[g].T)
ctx = H.Context(0)
outs = []
for i in range(30):
    lam, z = H.syevx_topk_batch(a, kk, ctx=ctx)
    outs.append(z.copy())
# majority reference: the most common output
import collections
keys = [hash(o.tobytes()) for o in outs]
ref = outs[keys.index(collections.Counter(keys).most_common(1)[0][0])]
for i, o in enumerate(outs):
    if not np.array_equal(o, ref):
        d = np.abs(o - ref)
        g = int(d.reshape(count, -1).max(axis=1).argmax())
        rows = np.nonzero(d[g].max(axis=1) > 0)[0]
        cols = np.nonzero(d[g].max(axis=0) > 0)[0]
        print(f"call {i}: matrix {g} rows {rows.min()}..{rows.max()} ({len(rows)}) cols {cols.min()}..{cols.max()} ({len(cols)}) max {d[g].max():.2e}")
        # per 8-row tile max
        print("   tile maxima:", " ".join(f"{d[g][t*8:(t+1)*8, cols].max():.0e}" for t in range(n // 8)))
print("distinct outputs:", len(set(keys)))
