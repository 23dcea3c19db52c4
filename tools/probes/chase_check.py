"""Probe: two-stage eigenvalues vs LAPACK for a few n and chase cluster sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

import paper_1710_02812_b200 as H  # noqa: E402

os.environ["HSVD_TWO_STAGE_MIN_N"] = "1"
for n in [int(a) for a in sys.argv[1].split(",")]:
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n + 7, n)) * np.exp(-np.linspace(0, 6, n))[None, :]
    a = x.T @ x
    w = np.linalg.eigvalsh(a)[::-1][:64]
    for cs in sys.argv[2].split(","):
        os.environ["HSVD_CHASE_CS"] = cs
        errs = []
        for rep in range(3):
            lam, z = H.syevx_topk(a, 64)
            errs.append(np.abs(lam - w).max() / w[0])
        print(f"n={n} cs={cs} rel err per rep: " + " ".join(f"{e:.1e}" for e in errs), flush=True)
