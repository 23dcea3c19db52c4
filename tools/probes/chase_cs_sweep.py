#!/usr/bin/env python
"""k_chase time against the cluster size (HSVD_CHASE_CS = 1, 2, 4, 8) on the
small leaf batches a rank of a multi-GPU run sees (config 5 on 8 GPUs: 32
Grams of order 4096 per rank; configs 2-4: 8).  Device time of k_chase from
the per-launch events, best of 3; eigenvalues checked against the CS = 1 run.

  python tools/probes/chase_cs_sweep.py [--out profiles/r02_chase_cs.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import numpy as np  # noqa: E402
from eig_batch_time import grams  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import paper_1710_02812_b200 as H
    ctx = H.Context(0)
    os.environ["HSVD_TWO_STAGE_MIN_N"] = "1"
    rows = []
    for count, n, kk in [(8, 2500, 100), (8, 2048, 64), (16, 2048, 128), (16, 4096, 200),
                         (32, 4096, 200), (37, 2500, 100), (4, 4096, 200)]:
        a = grams(count, n, count * n + 1)
        ref = None
        row = {"count": count, "n": n, "kk": kk}
        for cs in (1, 2, 4, 8):
            os.environ["HSVD_CHASE_CS"] = str(cs)
            best = None
            for _ in range(3):
                ctx.profile(True)
                ctx.profile_report()
                lam, _ = H.syevx_topk_batch(a, kk, ctx=ctx)
                rep = ctx.profile_report()
                ctx.profile(False)
                ms = sum(v[1] for k, v in rep.items() if k.endswith("k_chase"))
                best = ms if best is None else min(best, ms)
            if ref is None:
                ref = lam
            row[f"cs{cs}_ms"] = round(best, 3)
            row[f"cs{cs}_lam_maxdiff"] = float(np.abs(lam - ref).max() / np.abs(ref).max())
        rows.append(row)
        print(json.dumps(row), flush=True)
    del os.environ["HSVD_CHASE_CS"]
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"what": "k_chase device ms against the cluster size, best of 3", "rows": rows},
                      f, indent=1)


if __name__ == "__main__":
    main()
