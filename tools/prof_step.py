"""One rank-k HSVD step of a BASELINE workload with the per-kernel event
profile printed (for ncu / quick timing runs on the GPU box)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1710_02812_b200 as H  # noqa: E402
from paper_1710_02812_b200 import configs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--rows", type=int, default=0, help="use only the first ROWS rows (P scaled)")
ap.add_argument("--top", type=int, default=8, help="kernels listed")
a = ap.parse_args()
w = configs.WORKLOADS[a.config]
if a.rows:
    P = max(1, a.rows // w.d)
    w = w.scaled(P * w.d, w.n, P=P)
x = configs.generate_torch(w, device="cuda")
ctx = H.Context(0)
cfg = H.MatConfig(gamma=1e-12, row_block_rows=w.d, col_block_cols=w.c, max_rank=w.k)
ctx.profile(True)
for _ in range(a.steps):
    H.rank_k_svd_device(x, cfg, ctx)
ctx.synchronize()
prof = ctx.profile_report()
tot = sum(v[1] for v in prof.values())
print(json.dumps({"workload": w.name, "total_ms": tot / a.steps,
                  "top": sorted(((k, v[0], round(v[1] / a.steps, 3)) for k, v in prof.items()),
                                key=lambda t: -t[2])[:a.top]}))
