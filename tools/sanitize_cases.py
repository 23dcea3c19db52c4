#!/usr/bin/env python
"""Small invocations of the concurrency-heavy kernels for compute-sanitizer
(racecheck / synccheck): the two-stage eigensolver with the 2-CTA cluster
bulge chase (progress flags over DSMEM) and the cluster panel QR (DSMEM
exchange), the one-stage k_latrd on a CTA cluster, the tcgen05/TMA Ozaki
Gram (mbarrier pipeline) and the Jacobi / QR kernels.  No torch import (the
library is driven through ctypes only), sizes kept small for the tools'
slowdown.

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def gram(n, seed):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n + 5, n)) * np.exp(-np.linspace(0, 6, n))[None, :]
    return x.T @ x


def main():
    import paper_1710_02812_b200 as H
    ctx = H.Context(0)
    # two-stage (forced), batch of 4 -> 2-CTA cluster chase, cluster panel QR
    os.environ["HSVD_TWO_STAGE_MIN_N"] = "1"
    a = np.stack([gram(320, s) for s in range(4)])
    lam, z = H.syevx_topk_batch(a, 24, ctx=ctx)
    assert np.isfinite(lam).all()
    # one-stage blocked (k_latrd on a cluster for a single matrix)
    os.environ["HSVD_TWO_STAGE_MIN_N"] = str(1 << 30)
    lam1, _ = H.syevx_topk(gram(640, 9), 16, ctx=ctx)
    assert np.allclose(lam1[:4], np.linalg.eigvalsh(gram(640, 9))[::-1][:4], rtol=1e-10)
    del os.environ["HSVD_TWO_STAGE_MIN_N"]
    # tcgen05 Ozaki Gram (TMA + mbarriers + TMEM), Jacobi, Householder QR
    rng = np.random.default_rng(1)
    x = rng.standard_normal((600, 300)).astype(np.float32)
    g = H.block_gram(x, ctx=ctx)
    assert np.allclose(g, x.astype(np.float64).T @ x.astype(np.float64), rtol=1e-12, atol=1e-9)
    f = H.full_svd(rng.standard_normal((60, 20)), ctx=ctx)
    assert f.rank() == 20
    q, r = H.qr_thin(rng.standard_normal((50, 12)), ctx=ctx)
    assert q.shape == (50, 12)
    # a small whole pipeline (leaves, merges, recoveries)
    y = rng.standard_normal((512, 256)).astype(np.float32)
    res = H.rank_k_svd(y, H.MatConfig(gamma=1e-12, row_block_rows=256, col_block_cols=128,
                                      max_rank=24), ctx=ctx)
    assert res.rank() == 24
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
