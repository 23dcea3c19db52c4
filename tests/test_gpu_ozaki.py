"""The leaf Gram on the tcgen05 int8 tensor cores (Ozaki slices, fp64-grade;
csrc/ozaki_gram.cu) against the fp64 Gram of the same fp32 bytes, and the
leaf SVD built on it against the oracle (kernels.cpp:21-48 on
hierarchy.cpp:57's blocks)."""
import numpy as np
import pytest

import hsvd_oracle as O

pytestmark = pytest.mark.gpu


def _block(d, c, seed, decay=6.0, dtype=np.float32):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((d, c)) * np.exp(-np.linspace(0, decay, c))[None, :]
    return x.astype(dtype)


@pytest.mark.parametrize("d,c", [(128, 256), (300, 200), (2500, 640), (4096, 513), (1000, 1000),
                                 (16384, 96)])
def test_block_gram_fp64_grade(d, c):
    import paper_1710_02812_b200 as H
    x = _block(d, c, d * 31 + c)
    g = H.block_gram(x)
    x64 = x.astype(np.float64)
    ref = x64.T @ x64
    assert np.array_equal(g, g.T)  # full symmetric storage, mirrored exactly
    err = np.abs(g - ref).max() / np.abs(ref).max()
    assert err < 1e-14, err
    # per element relative to the column norms (the diagonal dominates)
    dn = np.sqrt(np.outer(np.diag(ref), np.diag(ref)))
    assert (np.abs(g - ref) / dn).max() < 1e-13


def test_block_gram_strided_and_wide_range():
    """A strided view (ld > c) and columns spanning 2^-40..2^40 in scale:
    per-column power-of-two scaling keeps every column exact to fp64 grade."""
    import torch
    import paper_1710_02812_b200 as H
    rng = np.random.default_rng(5)
    big = rng.standard_normal((700, 400)).astype(np.float32)
    big *= np.exp2(np.linspace(-40, 40, 400)).astype(np.float32)[None, :]
    big[:, 17] = 0.0  # an all-zero column
    xt = torch.from_numpy(big).cuda()[:, 10:310]  # ld = 400, c = 300
    g = H.block_gram(xt)
    x64 = big[:, 10:310].astype(np.float64)
    ref = x64.T @ x64
    dn = np.sqrt(np.outer(np.diag(ref), np.diag(ref)))
    dn[dn == 0] = 1.0
    assert (np.abs(g - ref) / dn).max() < 1e-13


def test_block_gram_matches_dmma(monkeypatch):
    import paper_1710_02812_b200 as H
    x = _block(3000, 700, 11)
    g_oz = H.block_gram(x)
    monkeypatch.setenv("HSVD_GRAM", "dmma")
    g_dm = H.block_gram(x)
    assert np.abs(g_oz - g_dm).max() <= 1e-14 * np.abs(g_dm).max()


@pytest.mark.parametrize("gram", ["ozaki", "dmma"])
def test_leaves_on_int8_gram_vs_oracle(gram, monkeypatch):
    """svd_of_col_slices of an fp32 row slice: 6 leaves whose Grams run on the
    int8 tensor cores (or the DMMA SYRK), merged; sigma and U against the
    oracle at the fp64 bar the reference's own tests use (1e-9)."""
    import paper_1710_02812_b200 as H
    if gram == "dmma":
        monkeypatch.setenv("HSVD_GRAM", "dmma")
    rng = np.random.default_rng(3)
    m, n, r = 1500, 1800, 40
    u = np.linalg.qr(rng.standard_normal((m, r)))[0]
    v = np.linalg.qr(rng.standard_normal((n, r)))[0]
    x = ((u * np.exp(-0.1 * np.arange(r))) @ v.T + 1e-5 * rng.standard_normal((m, n))).astype(
        np.float32)
    got = H.svd_of_col_slices(x, 300, 1e-12, 30)
    ref = O.svd_of_col_slices(x, 300, 1e-12, 30)
    assert got.rank() == ref.rank() == 30
    assert np.abs(got.sigma - ref.sigma).max() <= 1e-9 * ref.sigma[0]
    assert O.largest_principal_angle(ref.u, got.u) < 1e-7


@pytest.mark.parametrize("shape,grid,k", [((3000, 2400), (3, 4), 200), ((8000, 1024), (4, 1), 180),
                                          ((1500, 3000), (2, 3), 200)])
def test_projections_on_int8_match_dmma(shape, grid, k, monkeypatch):
    """The projection GEMMs (leaf X_b Z, V-recovery X_j^T U_j, U-recovery
    X V_r; routed to the tcgen05 Ozaki planes for N > 160 columns) against the
    same pipeline with them on the fp64 DMMA GEMM: fp64-grade agreement."""
    import paper_1710_02812_b200 as H
    rng = np.random.default_rng(shape[0] + shape[1])
    m, n = shape
    r = min(m, n, 2 * k)
    u = np.linalg.qr(rng.standard_normal((m, r)))[0]
    v = np.linalg.qr(rng.standard_normal((n, r)))[0]
    x = ((u * np.exp(-0.04 * np.arange(r))) @ v.T + 1e-5 * rng.standard_normal((m, n))).astype(
        np.float32)
    cfg = H.MatConfig(gamma=1e-12, row_block_rows=m // grid[0], col_block_cols=n // grid[1],
                      max_rank=k)
    oz = H.rank_k_svd(x, cfg)
    monkeypatch.setenv("HSVD_PROJ", "dmma")
    dm = H.rank_k_svd(x, cfg)
    assert oz.rank() == dm.rank() == k
    assert np.abs(oz.sigma - dm.sigma).max() <= 1e-12 * dm.sigma[0]
    # 1e-8 rad: the two pipelines differ by rounding (~1e-15) amplified by the
    # gap of the last retained direction to the noise tail (observed <= 1.2e-9)
    assert O.largest_principal_angle(dm.u, oz.u) < 1e-8
    assert O.largest_principal_angle(dm.v, oz.v) < 1e-8
