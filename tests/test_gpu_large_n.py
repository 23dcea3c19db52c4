"""Blocks with a smaller side above 6144 (the reference's full_svd has no
size limit, kernels.cpp:21-48): the two-stage eigensolver keeps the panel of
k_panel_qr and the tridiagonal of k_steig in global memory once they no
longer fit shared memory.  Known-answer checks (LAPACK on these sizes would
take minutes on the host)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _orth(rng, n, r):
    return np.linalg.qr(rng.standard_normal((n, r)))[0]


def test_syevx_topk_n9500_global_panel_and_tridiagonal():
    """n = 9500: the panel (8-CTA cluster) and k_steig's d, e, e^2 exceed
    shared memory."""
    import paper_1710_02812_b200 as H
    n, kk, r = 9500, 40, 80
    rng = np.random.default_rng(9500)
    q = _orth(rng, n, r)
    lam_true = 50.0 * np.exp(-0.08 * np.arange(r))
    a = (q * lam_true) @ q.T + 1e-5 * np.eye(n)
    lam, z = H.syevx_topk(a, kk)
    assert np.abs(lam - (lam_true[:kk] + 1e-5)).max() <= 1e-11 * lam_true[0]
    assert np.abs(a @ z - z * lam).max() <= 1e-10 * lam_true[0]
    assert np.abs(z.T @ z - np.eye(kk)).max() < 1e-10


def test_hierarchical_svd_default_config_one_large_block():
    """MatConfig() defaults (d = c = 0: the whole matrix is one block,
    svd_factor.hpp:31-32) on a 9400 x 9600 matrix of known spectrum."""
    import paper_1710_02812_b200 as H
    m, n, r = 9400, 9600, 48
    rng = np.random.default_rng(9400)
    s = 10.0 * np.exp(-0.12 * np.arange(r))
    x = (_orth(rng, m, r) * s) @ _orth(rng, n, r).T
    f = H.rank_k_svd(x, H.MatConfig(gamma=1e-6))
    k = f.rank()
    kept = s[s >= 1e-6 * s[0]]
    assert k == len(kept)
    assert np.abs(f.sigma[:k] - kept).max() <= 1e-10 * s[0]
    assert np.abs(f.u.T @ f.u - np.eye(k)).max() < 1e-10
    assert np.abs(f.v.T @ f.v - np.eye(k)).max() < 1e-10
