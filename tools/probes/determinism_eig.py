#!/usr/bin/env python
"""Bitwise repeatability of the batched two-stage eigensolver on small
matrices: python tools/probes/determinism_eig.py COUNT N KK [REPS]"""
import os
import sys

ROOT = os.environ.get("PROBE_ROOT", os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

os.environ.setdefault("HSVD_TWO_STAGE_MIN_N", "1")
import paper_1710_02812_b200 as H  # noqa: E402

count, n, kk = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rng = np.random.default_rng(5)
a = np.empty((count, n, n))
for g in range(count):
    # leaf-like spectrum: decaying signal + a flat noise tail (one big cluster)
    u = np.linalg.qr(rng.standard_normal((n, n)))[0]
    s = np.concatenate([100 * np.exp(-0.05 * np.arange(1, 41)), 1e-3 * (1 + 0.05 * rng.standard_normal(n - 40))])
    a[g] = (u * s ** 2) @ u.T
    a[g] = 0.5 * (a[g] + a[g].T)
ctx = H.Context(0)
ref = None
bad = badl = 0
hashes = []
zs = []
for i in range(reps):
    lam, z = H.syevx_topk_batch(a, kk, ctx=ctx)
    hashes.append(hash(z.tobytes()))
    zs.append(z.copy())
    if ref is None:
        ref = (lam.copy(), z.copy())
        w = np.linalg.eigvalsh(a[0])[::-1][:kk]
        print("lam err vs LAPACK", np.abs(lam[0] - w).max() / w[0],
              "resid", np.abs(a[0] @ z[0] - z[0] * lam[0]).max() / w[0],
              "orth", np.abs(z[0].T @ z[0] - np.eye(kk)).max())
        continue
    if not np.array_equal(lam, ref[0]):
        badl += 1
    if not np.array_equal(z, ref[1]):
        bad += 1
        if bad <= 3:
            d = np.abs(z - ref[1]).max(axis=(1,))
            g = int(np.abs(z - ref[1]).reshape(count, -1).max(axis=1).argmax())
            cols = np.nonzero(np.abs(z[g] - ref[1][g]).max(axis=0) > 0)[0]
            print(f"call {i}: Z differs, matrix {g}, columns {cols[:8]}..{cols[-1]} ({len(cols)}), max {np.abs(z - ref[1]).max():.2e}")
            for nm, zz in (("this", z[g]), ("first", ref[1][g])):
                print("   ", nm, "resid", np.abs(a[g] @ zz - zz * lam[g]).max() / lam[g][0],
                      "orth", np.abs(zz.T @ zz - np.eye(kk)).max(),
                      "resid cols", np.abs(a[g] @ zz[:, cols] - zz[:, cols] * lam[g][cols]).max() / lam[g][0])
import collections
cnt = collections.Counter(hashes)
zmaj = zs[hashes.index(cnt.most_common(1)[0][0])]
print("MAXDEV from majority:", max(float(np.abs(zz - zmaj).max()) for zz in zs))
print(f"MAJORITY: {len(cnt)} distinct outputs, {reps - cnt.most_common(1)[0][1]} of {reps} calls off the majority")
print(f"count={count} n={n} kk={kk}: lam differs in {badl}, Z differs in {bad} of {reps - 1} calls;"
      f" env { {k: v for k, v in os.environ.items() if k.startswith('HSVD_')} }")
