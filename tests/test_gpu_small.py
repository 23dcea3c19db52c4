"""Small dense kernels of the reference API on the device: the one-sided
Jacobi route for SVDs whose smaller side is <= 32 (kernels.cpp:28), the
Householder thin QR (kernels.cpp:50-61), and run-to-run bitwise determinism
of the whole pipeline (tests/test_cli.cpp:91-105)."""
import numpy as np
import pytest

import hsvd_oracle as O

pytestmark = pytest.mark.gpu


def _graded(m, n, kappa_log10, seed):
    rng = np.random.default_rng(seed)
    u = np.linalg.qr(rng.standard_normal((m, min(m, n))))[0]
    v = np.linalg.qr(rng.standard_normal((n, min(m, n))))[0]
    s = np.logspace(0, -kappa_log10, min(m, n))
    return (u * s) @ v.T, s


@pytest.mark.parametrize("shape", [(40, 16), (16, 40), (300, 32), (32, 300), (1000, 7), (5, 5)])
def test_full_svd_jacobi_route(shape):
    """min(m, n) <= 32 runs one-sided Jacobi: normwise backward stable
    (|sigma_i - sigma_i^ref| ~ eps sigma_1, not eps kappa sigma_1 as the Gram
    route), orthonormal bases, exact reconstruction."""
    import paper_1710_02812_b200 as H
    a, _ = _graded(*shape, 10, shape[0] * 100 + shape[1])
    got = H.full_svd(a)
    ref = O.full_svd(a)  # dgejsv, the oracle's JacobiSVD
    assert got.rank() == min(shape)
    assert np.abs(got.sigma - ref.sigma).max() <= 1e-14 * ref.sigma[0]
    assert O.orthonormality_defect(got.u) < 1e-12 and O.orthonormality_defect(got.v) < 1e-12
    rec = (got.u * got.sigma) @ got.v.T
    assert np.linalg.norm(rec - a) <= 1e-13 * np.linalg.norm(a)


@pytest.mark.parametrize("shape", [(200, 24), (24, 200)])
def test_full_svd_jacobi_column_graded_relative_accuracy(shape):
    """A = B D with B well conditioned and D spanning twelve decades: one-sided
    Jacobi resolves every singular value to high relative accuracy (the
    property the reference's JacobiSVD route exists for)."""
    import paper_1710_02812_b200 as H
    rng = np.random.default_rng(sum(shape))
    m, n = shape
    p = min(m, n)
    b = rng.standard_normal((max(m, n), p))
    b = b @ np.diag(np.logspace(0, -12, p))
    a = b if m >= n else b.T
    got = H.full_svd(a)
    ref = O.full_svd(a)
    rel = np.abs(got.sigma - ref.sigma) / ref.sigma
    assert rel.max() < 1e-10, rel.max()


def test_small_svd_gram_route_is_the_loser(monkeypatch):
    """The same matrix through the forced Gram route misses the small
    singular values by orders of magnitude: the reason for the Jacobi route."""
    import paper_1710_02812_b200 as H
    a, _ = _graded(40, 16, 10, 4016)
    ref = O.full_svd(a)
    monkeypatch.setenv("HSVD_SMALL_SVD", "gram")
    gram = H.full_svd(a)
    monkeypatch.delenv("HSVD_SMALL_SVD")
    jac = H.full_svd(a)
    err_gram = np.abs(gram.sigma - ref.sigma).max() / ref.sigma[0]
    err_jac = np.abs(jac.sigma - ref.sigma).max() / ref.sigma[0]
    assert err_jac < 1e-14 and err_gram > 1e2 * err_jac


@pytest.mark.parametrize("shape", [(50, 20), (20, 50), (64, 64), (3000, 40)])
def test_qr_thin_matches_lapack(shape):
    import paper_1710_02812_b200 as H
    rng = np.random.default_rng(shape[0] + 7 * shape[1])
    a = rng.standard_normal(shape)
    a[:, 3] = 0.0  # a zero column: tau = 0 at that step
    q, r = H.qr_thin(a)
    q_ref, r_ref = O.qr_thin(a)  # dgeqrf + dorgqr: the same sign convention
    assert q.shape == q_ref.shape and r.shape == r_ref.shape
    assert np.allclose(q, q_ref, atol=1e-12) and np.allclose(r, r_ref, atol=1e-12)
    assert np.abs(np.tril(r, -1)).max() == 0.0
    assert np.linalg.norm(q @ r - a) <= 1e-13 * np.linalg.norm(a)


def test_qr_thin_rejects_empty():
    import paper_1710_02812_b200 as H
    with pytest.raises(ValueError, match="qr_thin: matrix is empty"):
        H.qr_thin(np.zeros((0, 3)))


def test_rerun_bitwise_deterministic():
    """Fixed input -> bitwise identical factors on rerun and on a fresh
    context: fixed tree pairing, fixed-order reductions everywhere (split-K,
    DSMEM sums, Jacobi and chase schedules, Ozaki level sums)."""
    import paper_1710_02812_b200 as H
    rng = np.random.default_rng(271)
    m, n, r = 4096, 2048, 80
    u = np.linalg.qr(rng.standard_normal((m, r)))[0]
    v = np.linalg.qr(rng.standard_normal((n, r)))[0]
    x = ((u * np.exp(-0.05 * np.arange(r))) @ v.T + 1e-4 * rng.standard_normal((m, n))).astype(
        np.float32)
    cfg = H.MatConfig(gamma=1e-12, row_block_rows=1024, col_block_cols=1024, max_rank=64)
    a = H.rank_k_svd(x, cfg)
    b = H.rank_k_svd(x, cfg)
    c = H.rank_k_svd(x, cfg, ctx=H.Context(0))
    for f in (b, c):
        assert np.array_equal(a.sigma, f.sigma)
        assert np.array_equal(a.u, f.u) and np.array_equal(a.v, f.v)
