"""Parity of the B200 path (through the C ABI) with the CPU oracle and the
reference's own known-answer tests.  Needs a B200: marked ``gpu``.

Stated tolerances (BASELINE.json north_star): sigma within 1e-4 relative for
fp32 inputs and 1e-10 for fp64, largest principal angle of each retained
subspace <= 1e-3 rad, relative Frobenius reconstruction error within 1% of the
reference's own.  The reference's own unit-test pins are held at the
reference's tolerances (no overrides).
"""
import numpy as np
import pytest

import hsvd_oracle as O
import ref_cases as R

pytestmark = pytest.mark.gpu

# No overrides: every reference pin is held at the reference's own tolerance,
# including rank_k_error = 8.1960876183812958e-09 to 1e-6 relative
# (test_factor.cpp:176-198).  That pin needs the reference's small-SVD route:
# every SVD whose smaller side is <= 32 runs one-sided Jacobi on the matrix
# itself (csrc/jacobi.cu, kernels.cpp:28) instead of the Gram route, whose
# eps * kappa^2 error it could not meet.
PRODUCT_TOL = None


@pytest.fixture(scope="module")
def H():
    import paper_1710_02812_b200 as H
    H.load_library()
    return H


@pytest.mark.parametrize("case", R.ALL_CASES, ids=lambda c: c.__name__)
def test_reference_case_on_gpu(case, H, golden):
    case(H, golden, PRODUCT_TOL)


def _synthetic(m, n, r, spectrum, noise, dtype, seed):
    """Seeded stand-in for a BASELINE config at reduced size (same recipe:
    X = U diag(s) V^T + noise*N, U,V orthonormal from QR of Gaussians)."""
    rng = np.random.default_rng(seed)
    u = np.linalg.qr(rng.standard_normal((m, r)))[0]
    v = np.linalg.qr(rng.standard_normal((n, r)))[0]
    s = spectrum(np.arange(1, r + 1, dtype=np.float64))
    x = (u * s) @ v.T + noise * rng.standard_normal((m, n))
    return x.astype(dtype)


CONFIG_CASES = {
    # name: (m, n, r, spectrum, noise, dtype, P, Q, k)
    "cfg1_fp64": (2000, 2000, 50, lambda i: 10 * np.exp(-0.15 * i), 1e-4, np.float64, 4, 4, 50),
    "cfg2_small": (2000, 2000, 100, lambda i: i ** -1.5, 1e-3, np.float32, 8, 8, 100),
    "cfg3_small": (16384, 256, 64, lambda i: np.exp(-0.1 * i), 1e-4, np.float32, 64, 1, 64),
    "cfg5_small": (2048, 2048, 200, lambda i: 100 * np.exp(-0.05 * i), 1e-4, np.float32, 8, 8, 200),
}


CONFIG_CASES["cfg4_small"] = (8192, 1024, 128, lambda i: i ** -2.0, 1e-3, np.float32, 4, 1, 128)
CONFIG_CASES["cfg2_leaf1250"] = (5000, 5000, 100, lambda i: i ** -1.5, 1e-3, np.float32, 4, 4, 100)


@pytest.mark.parametrize("shape", [(700, 600), (600, 700), (1100, 1030)])
def test_full_svd_blocked_eigensolver(shape, H):
    """full_svd through the blocked (n >= 512) tridiagonalisation: every
    singular value and both bases against LAPACK."""
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    a = rng.standard_normal(shape) * np.exp(-np.linspace(0, 8, shape[1]))[None, :]
    got = H.full_svd(a)
    ref = O.full_svd(a)
    p = min(shape)
    assert got.rank() == p
    assert np.abs(got.sigma - ref.sigma).max() <= 1e-10 * ref.sigma[0]
    # The eigenvector side of the Gram is orthonormal to eps*n; the projected
    # side A z / sigma to ~eps*kappa^2 (kappa ~ e^8 here): the reference bar 1e-8.
    assert O.orthonormality_defect(got.v) < 1e-8
    assert O.orthonormality_defect(got.u) < 1e-8
    rec = (got.u * got.sigma) @ got.v.T
    assert np.linalg.norm(rec - a) <= 1e-11 * np.linalg.norm(a)


@pytest.mark.parametrize("eig", ["auto", "two_stage"])
@pytest.mark.parametrize("name", sorted(CONFIG_CASES))
def test_config_parity_with_oracle(name, eig, H, monkeypatch):
    """Whole pipeline against the oracle; eig="two_stage" forces the
    dense -> band -> tridiagonal eigensolver for every matrix of n >= 256
    (the default picks it only for large batched leaves)."""
    if eig == "two_stage":
        monkeypatch.setenv("HSVD_TWO_STAGE_MIN_N", "256")
    m, n, r, spec, noise, dt, P, Q, k = CONFIG_CASES[name]
    x = _synthetic(m, n, r, spec, noise, dt, seed=171002812 + len(name))
    cfg = dict(gamma=1e-12, row_block_rows=m // P, col_block_cols=n // Q, max_rank=k)
    got = H.rank_k_svd(x, H.MatConfig(**cfg))
    ref_r = O.hierarchical_svd(x, O.MatConfig(**cfg), workers=8)
    ref = O.recover_left_vectors(x, ref_r.v)
    assert got.rank() == ref.rank() == k
    tol = 1e-10 if dt == np.float64 else 1e-4
    rel = np.abs(got.sigma - ref.sigma) / ref.sigma
    assert rel.max() <= tol, rel.max()
    assert O.largest_principal_angle(ref.v, got.v) <= 1e-3
    assert O.largest_principal_angle(ref.u, got.u) <= 1e-3
    x64 = x.astype(np.float64)
    err_ref = np.linalg.norm(x64 - O.reconstruct(ref)) / np.linalg.norm(x64)
    err_got = np.linalg.norm(x64 - (got.u * got.sigma) @ got.v.T) / np.linalg.norm(x64)
    assert abs(err_got - err_ref) <= 1e-2 * err_ref
    assert O.orthonormality_defect(got.u) < 1e-8 and O.orthonormality_defect(got.v) < 1e-8


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_refine_parity_with_oracle(dt, H):
    """refine_factors (Alg. 2, refine.cpp:26-72) on hierarchical output at a
    few-thousand scale: same iteration count and convergence, sigma and both
    subspaces against the oracle (north-star tolerances)."""
    m, n, r = 3000, 1200, 40
    x = _synthetic(m, n, r, lambda i: np.exp(-0.08 * i), 1e-4, dt, seed=17102)
    cfg = dict(gamma=1e-3, row_block_rows=750, col_block_cols=300, max_rank=30)
    # both start from the same (oracle) hierarchical output
    ref_right = O.hierarchical_svd(x, O.MatConfig(**cfg), workers=8)
    got = H.refine_factors(x, ref_right.v, ref_right.sigma, 1e-9, 6)
    ref = O.refine_factors(x.astype(np.float64), ref_right.v, ref_right.sigma, 1e-9, 6)
    assert got.iterations == ref.iterations and got.converged == ref.converged
    assert got.factor.rank() == ref.factor.rank()
    rel = np.abs(got.factor.sigma - ref.factor.sigma) / ref.factor.sigma
    assert rel.max() <= 1e-8, rel.max()
    assert O.largest_principal_angle(ref.factor.v, got.factor.v) <= 1e-6
    assert O.largest_principal_angle(ref.factor.u, got.factor.u) <= 1e-6
    assert O.orthonormality_defect(got.factor.u) < 1e-8
    assert O.orthonormality_defect(got.factor.v) < 1e-8


def test_host_input_and_large_result_copies(H):
    """Host input crosses PCIe in row-slice chunks while the leaf Grams of the
    chunks already landed run (GEMM descriptors staged through mapped memory
    meanwhile), and a result above 8 MB comes back through the pinned double
    buffer with a multi-threaded copy-out: both must agree with the
    device-resident call and stay orthonormal."""
    import torch
    m, n, k = 120000, 256, 48
    x = _synthetic(m, n, 64, lambda i: np.exp(-0.05 * i), 1e-4, np.float32, seed=99)
    cfg = H.MatConfig(gamma=1e-12, row_block_rows=30000, col_block_cols=128, max_rank=k)
    host = H.rank_k_svd(x, cfg)
    dev = H.rank_k_svd(torch.from_numpy(x).cuda(), cfg)
    assert host.u.nbytes > 8 << 20  # the chunked device->host path
    assert host.rank() == dev.rank() == k
    np.testing.assert_allclose(host.sigma, dev.sigma, rtol=1e-9)
    assert O.largest_principal_angle(dev.u, host.u) <= 1e-9
    assert O.largest_principal_angle(dev.v, host.v) <= 1e-9
    assert O.orthonormality_defect(host.u) < 1e-8 and O.orthonormality_defect(host.v) < 1e-8
