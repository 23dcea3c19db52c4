"""Wall time of one device eigensolve (hsvd_cu_syevx_topk, one matrix)
for both reductions, to place the one-stage / two-stage crossover."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1710_02812_b200 as H  # noqa: E402

rng = np.random.default_rng(0)
ctx = H.Context(0)
for n, kk in ((1024, 100), (2048, 100), (4096, 200)):
    x = rng.standard_normal((n + 7, n)) * np.exp(-np.linspace(0, 8, n))[None, :]
    a = x.T @ x
    for path, thr in (("one", 1 << 30), ("two", 1)):
        os.environ["HSVD_TWO_STAGE_MIN_N"] = str(thr)
        H.syevx_topk(a, kk, ctx)
        t0 = time.perf_counter()
        for _ in range(3):
            H.syevx_topk(a, kk, ctx)
        print(f"n={n} kk={kk} {path}: {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms", flush=True)
