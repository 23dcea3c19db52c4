#!/usr/bin/env python
"""A/B a library knob in one process: the same rank-k HSVD step of a
BASELINE workload, re-run for each value of one HSVD_* environment variable
(the library reads its knobs at every launch), with the per-kernel event
profile of each run.

  python tools/env_sweep.py --config 5 --var HSVD_CHASE_L2PF --values 0,2,4 [--kernels k_chase]
"""
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
ap.add_argument("--var", required=True)
ap.add_argument("--values", required=True, help="comma-separated; 'unset' removes the variable")
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--rounds", type=int, default=2, help="passes over the value list")
ap.add_argument("--kernels", default="", help="comma-separated kernel-name substrings to report")
a = ap.parse_args()
w = configs.WORKLOADS[a.config]
x = configs.generate_torch(w, device="cuda")
ctx = H.Context(0)
cfg = H.MatConfig(gamma=1e-12, row_block_rows=w.d, col_block_cols=w.c, max_rank=w.k)
H.rank_k_svd_device(x, cfg, ctx)  # warm-up
ctx.synchronize()
want = [k for k in a.kernels.split(",") if k]
for rnd in range(a.rounds):
    for val in a.values.split(","):
        if val == "unset":
            os.environ.pop(a.var, None)
        else:
            os.environ[a.var] = val
        ctx.profile(True)
        ctx.profile_report()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(a.steps):
            res = H.rank_k_svd_device(x, cfg, ctx)
        ctx.synchronize()
        prof = ctx.profile_report()
        ctx.profile(False)
        # an un-profiled pass for the wall time of the step
        torch.cuda.synchronize()
        st.record(torch.cuda.ExternalStream(ctx.stream))
        for _ in range(a.steps):
            res = H.rank_k_svd_device(x, cfg, ctx)
        en.record(torch.cuda.ExternalStream(ctx.stream))
        ctx.synchronize()
        torch.cuda.synchronize()
        sel = {k: round(v[1] / a.steps, 3) for k, v in prof.items()
               if not want or any(s in k for s in want)}
        print(json.dumps({"round": rnd, a.var: val, "ms_per_step": st.elapsed_time(en) / a.steps,
                          "kernel_ms": sel, "rank": res}), flush=True)
