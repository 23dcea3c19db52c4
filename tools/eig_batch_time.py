#!/usr/bin/env python
"""One-stage vs two-stage eigensolver on small leaf batches (the per-rank
leaf stage of a multi-GPU run: configs 2-4 give each of 8 ranks 8 leaves).
Device time = the sum of the library's kernel times (per-launch CUDA events),
best of 3, for top-kk of `count` Grams of order n.

  python tools/eig_batch_time.py [--out profiles/r02_eig_batch.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def grams(count, n, seed):
    import torch
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    x = torch.randn((count, n + 64, n), dtype=torch.float64, device="cuda", generator=g)
    x *= torch.exp(-torch.linspace(0, 8, n, dtype=torch.float64, device="cuda"))[None, None, :]
    a = torch.matmul(x.transpose(1, 2), x)
    return a.cpu().numpy()


def time_eig(H, ctx, a, kk, mode):
    os.environ["HSVD_TWO_STAGE_MIN_N"] = "1" if mode == "two" else str(1 << 30)
    best = None
    for _ in range(3):
        ctx.profile(True)
        ctx.profile_report()
        H.syevx_topk_batch(a, kk, ctx=ctx)
        rep = ctx.profile_report()
        ctx.profile(False)
        ms = sum(v[1] for k, v in rep.items())
        best = ms if best is None else min(best, ms)
    del os.environ["HSVD_TWO_STAGE_MIN_N"]
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--cases", default="", help="comma-separated case indices")
    args = ap.parse_args()
    import paper_1710_02812_b200 as H
    ctx = H.Context(0)
    rows = []
    ap_cases = [(8, 2500, 100), (8, 2048, 64), (8, 2048, 128), (16, 2048, 128),
                (2, 4096, 200), (4, 4096, 200), (32, 2500, 100), (1, 2048, 128), (1, 1024, 64),
                (2, 1024, 64), (4, 1024, 64), (8, 1024, 64), (1, 1536, 64), (2, 1536, 64)]
    sel = [int(i) for i in args.cases.split(",")] if args.cases else range(len(ap_cases))
    for count, n, kk in [ap_cases[i] for i in sel]:
        a = grams(count, n, count * n)
        one = time_eig(H, ctx, a, kk, "one")
        two = time_eig(H, ctx, a, kk, "two")
        rows.append({"count": count, "n": n, "kk": kk, "one_stage_ms": one, "two_stage_ms": two,
                     "faster": "two" if two < one else "one"})
        print(json.dumps(rows[-1]), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"what": "top-kk eigensolver, device ms (sum of kernel events), best of 3",
                       "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
