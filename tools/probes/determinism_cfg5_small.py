#!/usr/bin/env python
"""Run-to-run repeatability of the reduced config-5 stand-in with the
two-stage eigensolver forced (the case tests/test_gpu_parity.py compares with
the oracle): N calls in one process, every sigma / V compared bitwise with the
first call's.  Usage: python tools/probes/determinism_cfg5_small.py [N]"""
import os
import sys

ROOT = os.environ.get("PROBE_ROOT", os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

os.environ.setdefault("HSVD_TWO_STAGE_MIN_N", "256")
import paper_1710_02812_b200 as H  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 30
m = n = 2048
r, k = 200, 200
rng = np.random.default_rng(171002812 + len("cfg5_small"))
u = np.linalg.qr(rng.standard_normal((m, r)))[0]
v = np.linalg.qr(rng.standard_normal((n, r)))[0]
s = 100 * np.exp(-0.05 * np.arange(1, r + 1, dtype=np.float64))
x = ((u * s) @ v.T + 1e-4 * rng.standard_normal((m, n))).astype(np.float32)
cfg = H.MatConfig(gamma=1e-12, row_block_rows=m // 8, col_block_cols=n // 8, max_rank=k)
ctx = H.Context(0)
ref = None
bad = 0
worst = 0.0
for i in range(N):
    got = H.rank_k_svd(x, cfg, ctx=ctx)
    if ref is None:
        ref = got
        continue
    same = np.array_equal(got.sigma, ref.sigma) and np.array_equal(got.v, ref.v)
    if not same:
        bad += 1
        worst = max(worst, float(np.abs(got.sigma - ref.sigma).max() / ref.sigma[0]),
                    )
        rel = np.abs(got.sigma - ref.sigma) / ref.sigma
        print(f"call {i}: differs, max rel sigma diff {rel.max():.3e} at index {int(rel.argmax())}")
print(f"{bad} of {N - 1} calls differ from the first; env BIG={os.environ.get('HSVD_BIG_CLUSTER')} "
      f"NO_SIDE={os.environ.get('HSVD_NO_SIDE')}")
