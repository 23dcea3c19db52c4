"""Pin the CPU oracle (oracle/hsvd_oracle.py) against the reference's own
known-answer tests and golden values.  CPU only."""
import numpy as np
import pytest

import hsvd_oracle as O
import ref_cases as R


@pytest.mark.parametrize("case", R.ALL_CASES, ids=lambda c: c.__name__)
def test_oracle_reference_case(case, golden):
    case(O, golden)


def test_oracle_rank_k_error_pin_is_tight(golden):
    # test_factor.cpp:176-198 -- the oracle reproduces the pinned value far
    # inside the reference's own 1e-6 relative tolerance.
    x, _ = R.lowrank(golden, 64, 32, 2024, "exp", 8, ratio=0.5, floor=1e-4)
    right = O.hierarchical_svd(x, O.MatConfig(gamma=1e-3, row_block_rows=16,
                                              col_block_cols=8))
    approx = O.recover_left_vectors(x, right.v)
    err = O.rank_k_error(x, approx, 8)
    assert abs(err - 8.1960876183812958e-09) / 8.1960876183812958e-09 < 1e-7


def test_oracle_truncation_properties():
    # test_factor.cpp:69-100 -- 500 random spectra: prefix, threshold, idempotence.
    rng = np.random.default_rng(321)
    for trial in range(500):
        n = 1 + int(rng.integers(0, 12))
        sigma = np.empty(n)
        v = 1.0 + 9.0 * rng.random()
        for i in range(n):
            sigma[i] = v
            v *= rng.random()
        gamma = 0.0 if trial % 5 == 0 else rng.random()
        t = O.truncate_factor(O.SvdFactor(None, sigma, None), gamma)
        assert 1 <= t.rank() <= n
        assert np.array_equal(t.sigma, sigma[:t.rank()])
        cutoff = gamma * sigma[0]
        assert t.sigma[-1] >= cutoff
        if t.rank() < n:
            assert sigma[t.rank()] < cutoff
        tt = O.truncate_factor(t, gamma)
        assert tt.rank() == t.rank()


def test_oracle_config_validation():
    # test_factor.cpp:212-226
    O.validate(O.MatConfig())
    for bad in (dict(gamma=-0.1), dict(epsilon=0.0), dict(max_iters=0), dict(max_rank=0)):
        with pytest.raises(ValueError):
            O.validate(O.MatConfig(**bad))


def test_golden_gaussians_match_libstdcxx(golden, tmp_path):
    # The committed fixture must equal what the reference's generator
    # stream produces with this toolchain (rebuilt here when g++ exists).
    import shutil
    import subprocess
    import os
    if shutil.which("g++") is None:
        pytest.skip("g++ not available")
    src = os.path.join(os.path.dirname(O.__file__), "gen_ref_gaussians.cpp")
    exe = str(tmp_path / "gen")
    subprocess.check_call(["g++", "-O2", "-std=c++17", src, "-o", exe])
    raw = subprocess.run([exe], input=b"matrix 5 3 7\nlowrank 16 8 77\n",
                         stdout=subprocess.PIPE, check=True).stdout
    buf = np.frombuffer(raw, dtype="<f8")
    assert np.array_equal(buf[:15].reshape(5, 3), golden["m_5x3_s7"])
    assert np.array_equal(buf[15:15 + 128].reshape(16, 8), golden["lr_16x8_s77_gu"])
