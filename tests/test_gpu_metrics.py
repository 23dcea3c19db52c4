"""Device evaluation of reconstruction errors:
factor_diff_norm (bench.cpp:30-42), rank_k_error (svd_factor.cpp:66-83) and
the residual ||X - U S V^T||_F, against explicit numpy evaluation and the
oracle, with the reference's argument checks."""
import numpy as np
import pytest

import hsvd_oracle as O

pytestmark = pytest.mark.gpu


def _factor(rng, m, n, k, top=3.0):
    u = np.linalg.qr(rng.standard_normal((m, k)))[0]
    v = np.linalg.qr(rng.standard_normal((n, k)))[0]
    s = top * 0.8 ** np.arange(k)
    return u, s, v


@pytest.mark.parametrize("m,n,ka,kb", [(70, 40, 5, 3), (300, 129, 17, 30), (1000, 700, 64, 64)])
def test_factor_diff_norm(m, n, ka, kb):
    import paper_1710_02812_b200 as H
    rng = np.random.default_rng(m + n)
    ua, sa, va = _factor(rng, m, n, ka)
    ub, sb, vb = _factor(rng, m, n, kb, top=2.5)
    got = H.factor_diff_norm(H.SvdFactor(ua, sa, va), H.SvdFactor(ub, sb, vb))
    ref = np.linalg.norm((ua * sa) @ va.T - (ub * sb) @ vb.T)
    assert abs(got - ref) <= 1e-12 * ref
    # nearly coincident factors: no cancellation (bench.cpp:27-29)
    eps = 1e-9
    got2 = H.factor_diff_norm(H.SvdFactor(ua, sa, va), H.SvdFactor(ua, sa * (1 + eps), va))
    ref2 = eps * np.linalg.norm(sa)
    assert abs(got2 - ref2) <= 1e-6 * ref2


def test_rank_k_error_matches_oracle():
    import paper_1710_02812_b200 as H
    rng = np.random.default_rng(3)
    m, n = 120, 60
    x = rng.standard_normal((m, n)) * np.exp(-0.1 * np.arange(n))[None, :]
    full = O.full_svd(x)
    approx = O.SvdFactor(full.u[:, :10] + 1e-7 * rng.standard_normal((m, 10)), full.sigma[:10],
                         full.v[:, :10])
    for k in (1, 5, 10):
        ref = O.rank_k_error(full, approx, k)
        got = H.rank_k_error(H.SvdFactor(full.u, full.sigma, full.v),
                             H.SvdFactor(approx.u, approx.sigma, approx.v), k)
        assert abs(got - ref) <= 1e-9 * ref + 1e-15, (k, got, ref)
    # X overload: full SVD taken on the device first (svd_factor.cpp:82-84)
    got_x = H.rank_k_error(x, H.SvdFactor(approx.u, approx.sigma, approx.v), 10)
    assert abs(got_x - O.rank_k_error(x, approx, 10)) <= 1e-6 * O.rank_k_error(x, approx, 10)


def test_rank_k_error_argument_checks():
    import paper_1710_02812_b200 as H
    rng = np.random.default_rng(4)
    u, s, v = _factor(rng, 20, 10, 4)
    full = H.SvdFactor(u, s, v)
    with pytest.raises(ValueError, match="approx must carry both u and v"):
        H.rank_k_error(full, H.SvdFactor(None, s, v), 2)
    with pytest.raises(ValueError, match=r"k must be in \[1, approx.rank\(\)\]"):
        H.rank_k_error(full, full, 5)
    with pytest.raises(ValueError, match=r"k must be in \[1, approx.rank\(\)\]"):
        H.rank_k_error(full, full, 0)
    zero = H.SvdFactor(u, np.zeros(4), v)
    with pytest.raises(ValueError, match="reference rank-k approximation is zero"):
        H.rank_k_error(zero, full, 2)


@pytest.mark.parametrize("dt", [np.float64, np.float32])
def test_residual_norm(dt):
    import paper_1710_02812_b200 as H
    rng = np.random.default_rng(5)
    m, n, k = 2000, 900, 40
    u, s, v = _factor(rng, m, n, k)
    x = ((u * s) @ v.T + 1e-3 * rng.standard_normal((m, n))).astype(dt)
    f = H.rank_k_svd(x, H.MatConfig(gamma=1e-12, row_block_rows=500, col_block_cols=300,
                                    max_rank=k))
    got = H.residual_norm(x, f)
    ref = np.linalg.norm(x.astype(np.float64) - (f.u * f.sigma) @ f.v.T)
    assert abs(got - ref) <= 1e-10 * np.linalg.norm(x.astype(np.float64))
