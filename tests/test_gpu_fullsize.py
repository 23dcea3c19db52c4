"""Full-size parity on the exact bytes bench.py times (BASELINE configs 2-4).

X comes from ``configs.generate_torch`` (the bench's generator and seed) on
cuda:0; the B200 path runs through the C ABI call the bench times
(``hsvd_cu_rank_k_svd``); the CPU oracle (hierarchy.cpp:65-112 restated, one
LAPACK thread per task over all host cores) runs on a host copy of the same
bytes.  Tolerances are the north-star's: sigma within 1e-4 relative (fp32
input), largest principal angle of U and of V <= 1e-3 rad, relative Frobenius
reconstruction error within 1% of the oracle's.  Config 5 (16 GiB, ~15 CPU
minutes for the oracle) is run by ``tools/parity_full.py --config 5`` and its
record is committed as ``profiles/parity_cfg5.json``.
"""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_full_size_parity_with_oracle(cfg):
    import parity_full
    res = parity_full.run(cfg)
    m = res["gpu_vs_oracle"]
    assert m["rank_a"] == m["rank_b"], m
    assert all(m["pass"].values()), m
    assert m["orth_u_b"] < 1e-8 and m["orth_v_b"] < 1e-8, m
