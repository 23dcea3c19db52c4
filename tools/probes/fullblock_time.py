"""Probe: default MatConfig (one block, kk = min(m, n)) on a rank-48 matrix;
per-kernel device times."""
import sys
import os
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import paper_1710_02812_b200 as H  # noqa: E402

for spec in sys.argv[1].split(","):
    m, n = (int(v) for v in spec.split("x")) if "x" in spec else (int(spec), int(spec))
    rng = np.random.default_rng(n)
    r = 48
    s = 10.0 * np.exp(-0.12 * np.arange(r))
    x = (np.linalg.qr(rng.standard_normal((m, r)))[0] * s) @ np.linalg.qr(rng.standard_normal((n, r)))[0].T
    ctx = H.Context(0)
    ctx.profile(True)
    ctx.profile_report()
    t0 = time.time()
    f = H.rank_k_svd(x, H.MatConfig(gamma=1e-6), ctx=ctx)
    dt = time.time() - t0
    rep = ctx.profile_report()
    top = sorted(rep.items(), key=lambda kv: -kv[1][1])[:8]
    print(spec, f"{dt:.2f}s rank", f.rank(), [(k, v[0], round(v[1], 1)) for k, v in top], flush=True)
