"""The reference's own known-answer / property tests, restated once and run
against any implementation module ``impl`` that exposes the reference API
(``oracle/hsvd_oracle.py`` for the CPU oracle, ``paper_1710_02812_b200`` for
the B200 product).  Each case cites the reference test it restates and uses
the reference's tolerance unless the caller passes an override in ``tol``
(the product states its own bounds in tests/test_gpu_parity.py).
"""
from __future__ import annotations

import math

import numpy as np

import hsvd_oracle as O


# --------------------------------------------------------------------------
# fixture helpers (tests/test_support.hpp)
# --------------------------------------------------------------------------

def rm(golden, r, c, s):
    """random_matrix(r, c, s) -- test_support.hpp:11-18."""
    return golden[f"m_{r}x{c}_s{s}"].copy()


def ro(golden, r, c, s):
    """random_orthonormal(r, c, s) -- test_support.hpp:20-22."""
    return O.qr_thin(rm(golden, r, c, s))[0]


def geometric_sigma(k, top=1.0, ratio=0.8):
    """test_support.hpp:25-30."""
    out = np.empty(k)
    s = top
    for i in range(k):
        out[i] = s
        s *= ratio
    return out


def random_factor(impl, golden, m, n, k, seed, ratio=0.8, keep="u"):
    """random_factor(m, n, k, seed) -- test_support.hpp:34-41 (one side kept)."""
    sigma = geometric_sigma(k, 1.0 + 0.1 * (seed % 7), ratio)
    if keep == "u":
        return impl.SvdFactor(u=ro(golden, m, k, seed), sigma=sigma, v=None)
    return impl.SvdFactor(u=None, sigma=sigma, v=ro(golden, n, k, seed + 1))


def lowrank(golden, m, n, seed, kind, rank, ratio=0.5, values=None, floor=0.0):
    """gen_low_rank -- generate.cpp:75-94."""
    p = min(m, n)
    sig = O.build_spectrum(p, kind, rank, ratio=ratio, values=values,
                           noise_floor=floor)
    x = O.gen_low_rank_from_gaussians(golden[f"lr_{m}x{n}_s{seed}_gu"],
                                      golden[f"lr_{m}x{n}_s{seed}_gv"], sig)
    return x, sig


def _t(tol, key, default):
    return (tol or {}).get(key, default)


def raises(exc, fn, *a, **kw):
    try:
        fn(*a, **kw)
    except exc:
        return True
    return False


# --------------------------------------------------------------------------
# test_merge.cpp
# --------------------------------------------------------------------------

def case_merge_self_sqrt2(impl, golden, tol=None):
    """test_merge.cpp:31-42."""
    e1 = np.zeros((4, 1))
    e1[0, 0] = 1.0
    f = impl.SvdFactor(u=e1, sigma=np.ones(1), v=None)
    m = impl.merge_pair_qr(f, f, impl.COLUMN_CONCAT, 0.0)
    assert m.rank() >= 1
    assert abs(m.sigma[0] - math.sqrt(2.0)) <= 1e-12 * math.sqrt(2.0)
    assert abs(abs(m.u[0, 0]) - 1.0) <= 1e-12
    for i in range(1, m.rank()):
        assert m.sigma[i] < _t(tol, "null", 1e-12)


def case_merge_orthogonal_units(impl, golden, tol=None):
    """test_merge.cpp:44-59."""
    e1 = np.zeros((4, 1))
    e2 = np.zeros((4, 1))
    e1[0, 0] = 1.0
    e2[1, 0] = 1.0
    f1 = impl.SvdFactor(u=e1, sigma=np.ones(1), v=None)
    f2 = impl.SvdFactor(u=e2, sigma=np.ones(1), v=None)
    for merge in (impl.merge_pair_naive, impl.merge_pair_qr):
        m = merge(f1, f2, impl.COLUMN_CONCAT, 0.0)
        assert m.rank() == 2
        assert abs(m.sigma[0] - 1.0) <= 1e-12
        assert abs(m.sigma[1] - 1.0) <= 1e-12


def case_naive_concat_oracle(impl, golden, tol=None):
    """test_merge.cpp:61-75 (ColumnConcat) and :77-89 (RowConcat)."""
    x1, x2 = rm(golden, 20, 6, 51), rm(golden, 20, 6, 52)
    oracle = O.full_svd(np.hstack([x1, x2])).sigma
    f1 = impl.full_svd(x1)
    f2 = impl.full_svd(x2)
    f1.v = None
    f2.v = None
    m = impl.merge_pair_naive(f1, f2, impl.COLUMN_CONCAT, 0.0)
    assert m.rank() == oracle.shape[0]
    assert np.abs(m.sigma - oracle).max() < 1e-10 * oracle[0]
    assert m.v is None and m.u is not None

    x1, x2 = rm(golden, 5, 14, 53), rm(golden, 7, 14, 54)
    oracle = O.full_svd(np.vstack([x1, x2])).sigma
    f1 = impl.full_svd(x1)
    f2 = impl.full_svd(x2)
    f1.u = None
    f2.u = None
    m = impl.merge_pair_naive(f1, f2, impl.ROW_CONCAT, 0.0)
    assert m.rank() == oracle.shape[0]
    assert np.abs(m.sigma - oracle).max() < 1e-10 * oracle[0]
    assert m.u is None and m.v is not None


def case_identical_basis(impl, golden, tol=None):
    """test_merge.cpp:91-106."""
    u = ro(golden, 10, 3, 55)
    f1 = impl.SvdFactor(u=u, sigma=geometric_sigma(3, 2.0, 0.5), v=None)
    f2 = impl.SvdFactor(u=u.copy(), sigma=geometric_sigma(3, 1.0, 0.25), v=None)
    naive = O.merge_pair_naive(O.SvdFactor(u, f1.sigma, None),
                               O.SvdFactor(u, f2.sigma, None), O.COLUMN_CONCAT, 0.0)
    fast = impl.merge_pair_qr(f1, f2, impl.COLUMN_CONCAT, 0.0)
    assert O.orthonormality_defect(fast.u) < 1e-8
    eff = fast.rank()
    while eff > 0 and fast.sigma[eff - 1] < 1e-12:
        eff -= 1
    assert eff <= 3
    assert np.abs(fast.sigma[:3] - naive.sigma[:3]).max() < 1e-10 * naive.sigma[0]


def case_orthogonal_union(impl, golden, tol=None):
    """test_merge.cpp:108-124."""
    u1 = np.zeros((8, 2))
    u2 = np.zeros((8, 2))
    u1[0, 0] = u1[1, 1] = 1.0
    u2[2, 0] = u2[3, 1] = 1.0
    f1 = impl.SvdFactor(u=u1, sigma=np.array([5.0, 2.0]), v=None)
    f2 = impl.SvdFactor(u=u2, sigma=np.array([4.0, 3.0]), v=None)
    m = impl.merge_pair_qr(f1, f2, impl.COLUMN_CONCAT, 0.0)
    assert m.rank() == 4
    assert np.abs(m.sigma - np.array([5.0, 4.0, 3.0, 2.0])).max() < 1e-12


def case_qr_equals_naive_100(impl, golden, tol=None):
    """test_merge.cpp:126-155 -- the product's merge against the oracle's naive
    merge (SVD of the concatenation) over 100 random pairs."""
    worst = 0.0
    for t in range(100):
        m = 8 + t % 23
        k = 1 + t % 5
        l = 1 + (t * 3) % 5
        column = t % 2 == 0
        orient = impl.COLUMN_CONCAT if column else impl.ROW_CONCAT
        o_orient = O.COLUMN_CONCAT if column else O.ROW_CONCAT
        keep = "u" if column else "v"
        if column:
            f1 = random_factor(impl, golden, m, 6, k, 1000 + 7 * t, keep=keep)
            f2 = random_factor(impl, golden, m, 9, l, 2000 + 7 * t, keep=keep)
        else:
            f1 = random_factor(impl, golden, 6, m, k, 1000 + 7 * t, keep=keep)
            f2 = random_factor(impl, golden, 9, m, l, 2000 + 7 * t, keep=keep)
        o1 = O.SvdFactor(f1.u, f1.sigma, f1.v)
        o2 = O.SvdFactor(f2.u, f2.sigma, f2.v)
        naive = O.merge_pair_naive(o1, o2, o_orient, 0.0)
        fast = impl.merge_pair_qr(f1, f2, orient, 0.0)
        assert fast.rank() == naive.rank(), t
        worst = max(worst, O.max_sigma_rel_diff(fast.sigma, naive.sigma, 1e-6))
        bn = naive.u if column else naive.v
        bf = fast.u if column else fast.v
        assert O.orthonormality_defect(bf) < 1e-8, t
        assert O.subspace_angle_sin(bn, bf) < _t(tol, "sin", 1e-7), t
        assert O.subspace_angle_sin(bf, bn) < _t(tol, "sin", 1e-7), t
    assert worst < 1e-9, worst


def case_merge_properties(impl, golden, tol=None):
    """test_merge.cpp:157-166 (top sigma never shrinks), :168-178 (energy
    additivity), :180-191 (commutativity)."""
    for t in range(20):
        f1 = random_factor(impl, golden, 15, 4, 3, 3000 + t)
        f2 = random_factor(impl, golden, 15, 4, 4, 4000 + t)
        m = impl.merge_pair_qr(f1, f2, impl.COLUMN_CONCAT, 0.0)
        assert m.sigma[0] >= max(f1.sigma[0], f2.sigma[0]) - 1e-10
    for t in range(20):
        f1 = random_factor(impl, golden, 18, 5, 4, 5000 + t)
        f2 = random_factor(impl, golden, 18, 6, 5, 6000 + t)
        m = impl.merge_pair_qr(f1, f2, impl.COLUMN_CONCAT, 0.0)
        exp = float(np.sum(f1.sigma ** 2) + np.sum(f2.sigma ** 2))
        assert abs(float(np.sum(m.sigma ** 2)) - exp) <= 1e-8 * exp
    for t in range(20):
        f1 = random_factor(impl, golden, 16, 5, 3, 7000 + t)
        f2 = random_factor(impl, golden, 16, 4, 5, 8000 + t)
        a = impl.merge_pair_qr(f1, f2, impl.COLUMN_CONCAT, 0.0)
        b = impl.merge_pair_qr(f2, f1, impl.COLUMN_CONCAT, 0.0)
        assert a.rank() == b.rank()
        assert np.abs(a.sigma - b.sigma).max() < 1e-10 * a.sigma[0]


def case_merge_gamma_and_cap(impl, golden, tol=None):
    """test_merge.cpp:193-205 (gamma) and :207-218 (max_rank cap)."""
    f1 = random_factor(impl, golden, 12, 5, 3, 9100)
    f2 = random_factor(impl, golden, 12, 5, 3, 9200)
    unt = impl.merge_pair_qr(f1, f2, impl.COLUMN_CONCAT, 0.0)
    merged = impl.merge_pair_qr(f1, f2, impl.COLUMN_CONCAT, 0.3)
    exp = impl.truncate_factor(unt, 0.3)
    assert merged.rank() == exp.rank()
    assert np.abs(merged.sigma - exp.sigma).max() < 1e-12
    f1 = random_factor(impl, golden, 12, 5, 4, 9300)
    f2 = random_factor(impl, golden, 12, 5, 4, 9400)
    for merge in (impl.merge_pair_naive, impl.merge_pair_qr):
        assert merge(f1, f2, impl.COLUMN_CONCAT, 0.0, 3).rank() == 3


def case_merge_fallback(impl, golden, tol=None):
    """test_merge.cpp:220-234 -- k+l > shared dimension."""
    f1 = random_factor(impl, golden, 5, 4, 4, 9500)
    f2 = random_factor(impl, golden, 5, 4, 4, 9600)
    naive = O.merge_pair_naive(O.SvdFactor(f1.u, f1.sigma, None),
                               O.SvdFactor(f2.u, f2.sigma, None), O.COLUMN_CONCAT, 0.0)
    fast = impl.merge_pair_qr(f1, f2, impl.COLUMN_CONCAT, 0.0)
    assert fast.rank() == naive.rank()
    assert fast.rank() <= 5
    assert np.abs(fast.sigma - naive.sigma).max() < 1e-10 * naive.sigma[0]
    assert O.orthonormality_defect(fast.u) < 1e-8


def case_merge_degenerate(impl, golden, tol=None):
    """test_merge.cpp:236-250."""
    zero = impl.SvdFactor(u=ro(golden, 10, 1, 9700), sigma=np.zeros(1), v=None,
                          degenerate=True)
    f = random_factor(impl, golden, 10, 4, 3, 9800)
    m = impl.merge_pair_qr(zero, f, impl.COLUMN_CONCAT, 1e-3)
    assert m.rank() == 3
    assert np.abs(m.sigma - f.sigma).max() < 1e-10
    both = impl.merge_pair_qr(zero, zero, impl.COLUMN_CONCAT, 1e-3)
    assert both.rank() == 1
    assert both.sigma[0] < 1e-14


def case_merge_rejects(impl, golden, tol=None):
    """test_merge.cpp:252-265."""
    f1 = impl.SvdFactor(u=np.linalg.qr(np.ones((10, 2)) + np.eye(10, 2))[0],
                        sigma=np.array([1.0, 0.5]), v=None)
    f2 = impl.SvdFactor(u=np.linalg.qr(np.ones((11, 2)) + np.eye(11, 2))[0],
                        sigma=np.array([1.0, 0.5]), v=None)
    assert raises(ValueError, impl.merge_pair_naive, f1, f2, impl.COLUMN_CONCAT, 0.0)
    assert raises(ValueError, impl.merge_pair_qr, f1, f2, impl.COLUMN_CONCAT, 0.0)
    f3 = impl.SvdFactor(u=None, sigma=np.array([1.0, 0.5]),
                        v=np.linalg.qr(np.ones((4, 2)) + np.eye(4, 2))[0])
    assert raises(ValueError, impl.merge_pair_qr, f3, f1, impl.COLUMN_CONCAT, 0.0)


# --------------------------------------------------------------------------
# test_hierarchy.cpp
# --------------------------------------------------------------------------

def case_block_plan(impl, golden, tol=None):
    """test_hierarchy.cpp:14-34."""
    plan = impl.BlockPlan.make(10, 7, 4, 3)
    assert len(plan.row_slices) == 3 and len(plan.col_slices) == 3
    assert plan.row_slices[2][1] == 2 and plan.col_slices[2][1] == 1
    nxt = 0
    for s, c in plan.row_slices:
        assert s == nxt
        nxt += c
    assert nxt == 10
    plan = impl.BlockPlan.make(10, 7, 0, 99)
    assert len(plan.row_slices) == 1 and len(plan.col_slices) == 1
    assert plan.row_slices[0][1] == 10 and plan.col_slices[0][1] == 7


def case_tree_merge_counts(impl, golden, tol=None):
    """test_hierarchy.cpp:36-70 (single factor unchanged, len-1 merges)."""
    f = random_factor(impl, golden, 15, 4, 3, 3000)
    st = impl.MergeStats()
    out = impl.tree_merge([f], impl.COLUMN_CONCAT, 0.0, None, st)
    assert st.pair_merges == 0
    assert np.abs(out.sigma - f.sigma).max() == 0.0
    for length in (2, 3, 4, 5, 7, 8, 11):
        fs = [random_factor(impl, golden, 15, 4, 3, 3000 + (i % 20)) for i in range(length)]
        st = impl.MergeStats()
        impl.tree_merge(fs, impl.COLUMN_CONCAT, 0.0, None, st)
        assert st.pair_merges == length - 1


def case_tree_merge_eight_blocks(impl, golden, tol=None):
    """test_hierarchy.cpp:72-84."""
    x = rm(golden, 40, 64, 456)
    fs = []
    for j in range(8):
        f = impl.full_svd(x[:, 8 * j:8 * j + 8])
        f.v = None
        fs.append(f)
    merged = impl.tree_merge(fs, impl.COLUMN_CONCAT, 0.0)
    oracle = O.full_svd(x).sigma
    assert merged.rank() == oracle.shape[0]
    assert np.abs(merged.sigma - oracle).max() < 1e-9 * oracle[0]
    assert raises(ValueError, impl.tree_merge, [], impl.COLUMN_CONCAT, 0.0)


def case_col_slices(impl, golden, tol=None):
    """test_hierarchy.cpp:91-126."""
    x = rm(golden, 16, 8, 510)
    whole = impl.svd_of_col_slices(x, 8, 0.1)
    exp = O.truncate_factor(O.full_svd(x), 0.1)
    assert whole.rank() == exp.rank()
    assert np.abs(whole.sigma - exp.sigma).max() < _t(tol, "abs12", 1e-12)
    assert whole.v is None
    xg, _ = lowrank(golden, 16, 8, 77, "explicit", 2, values=[1.0, 0.4])
    f = impl.svd_of_col_slices(xg, 2, 1e-6)
    oracle = O.full_svd(xg).sigma
    assert f.rank() == 2
    assert abs(f.sigma[0] - oracle[0]) < 1e-8 and abs(f.sigma[1] - oracle[1]) < 1e-8
    z = impl.svd_of_col_slices(np.zeros((12, 6)), 2, 1e-2)
    assert z.rank() == 1 and z.sigma[0] == 0.0 and z.degenerate


def case_hsvd_single_block(impl, golden, tol=None):
    """test_hierarchy.cpp:128-141."""
    x = rm(golden, 24, 10, 610)
    cfg = impl.MatConfig(gamma=0.05, row_block_rows=0, col_block_cols=0)
    f = impl.hierarchical_svd(x, cfg)
    exp = O.truncate_factor(O.full_svd(x), 0.05)
    assert f.rank() == exp.rank()
    assert np.abs(f.sigma - exp.sigma).max() < 1e-10 * exp.sigma[0]
    assert f.u is None and f.v is not None
    assert O.orthonormality_defect(f.v) < 1e-8


def case_hsvd_rank10(impl, golden, tol=None):
    """test_hierarchy.cpp:143-157."""
    x, true_sigma = lowrank(golden, 256, 64, 620, "exp", 10, ratio=0.6)
    cfg = impl.MatConfig(gamma=1e-8, row_block_rows=64, col_block_cols=16)
    f = impl.hierarchical_svd(x, cfg)
    assert f.rank() == 10
    assert O.max_sigma_rel_diff(f.sigma, true_sigma[:10]) < 1e-7


def case_hsvd_exact_plans(impl, golden, tol=None):
    """test_hierarchy.cpp:159-175 -- gamma 0 is exact for every block plan."""
    x = rm(golden, 48, 32, 630)
    oracle = O.full_svd(x).sigma
    for d in (48, 24, 12):
        for c in (32, 16, 4):
            cfg = impl.MatConfig(gamma=0.0, row_block_rows=d, col_block_cols=c)
            f = impl.hierarchical_svd(x, cfg)
            assert f.rank() == oracle.shape[0], (d, c)
            assert np.abs(f.sigma - oracle).max() < 1e-8 * oracle[0], (d, c)


def case_hsvd_no_inflation(impl, golden, tol=None):
    """test_hierarchy.cpp:177-187."""
    x = rm(golden, 60, 30, 640)
    oracle = O.full_svd(x).sigma
    f = impl.hierarchical_svd(x, impl.MatConfig(gamma=5e-2, row_block_rows=20,
                                                col_block_cols=6))
    for i in range(f.rank()):
        assert f.sigma[i] <= oracle[i] + 1e-8 * oracle[0]


def case_recover_left(impl, golden, tol=None):
    """test_hierarchy.cpp:189-231."""
    x = rm(golden, 30, 14, 650)
    full = O.full_svd(x)
    r = 5
    rec = impl.recover_left_vectors(x, full.v[:, :r].copy())
    assert rec.rank() == r
    assert np.abs(rec.sigma - full.sigma[:r]).max() < 1e-9 * full.sigma[0]
    trunc = O.SvdFactor(full.u[:, :r], full.sigma[:r], full.v[:, :r])
    assert (np.linalg.norm(O.reconstruct(O.SvdFactor(rec.u, rec.sigma, rec.v))
                           - O.reconstruct(trunc)) < 1e-9 * np.linalg.norm(x))

    x = rm(golden, 12, 12, 660)
    rec = impl.recover_left_vectors(x, np.eye(12))
    full = O.full_svd(x)
    assert np.abs(rec.sigma - full.sigma).max() < 1e-10 * full.sigma[0]
    rx = O.reconstruct(O.SvdFactor(rec.u, rec.sigma, rec.v))
    assert np.linalg.norm(rx - x) < 1e-10 * np.linalg.norm(x)

    x = rm(golden, 50, 20, 670)
    right = impl.hierarchical_svd(x, impl.MatConfig(gamma=1e-2, row_block_rows=25,
                                                    col_block_cols=5))
    rec = impl.recover_left_vectors(x, right.v)
    proj = x @ right.v @ right.v.T
    rx = O.reconstruct(O.SvdFactor(rec.u, rec.sigma, rec.v))
    assert np.linalg.norm(rx - proj) < 1e-10 * np.linalg.norm(x)
    assert O.orthonormality_defect(rec.u) < 1e-8
    assert O.orthonormality_defect(rec.v) < 1e-8

    bad = rm(golden, 10, 6, 680)[:6, :3].copy()
    assert raises(ValueError, impl.recover_left_vectors, rm(golden, 10, 6, 680), bad)


def case_full_width_row_slices(impl, golden, tol=None):
    """test_hierarchy.cpp:233-249 (BDCSVD misfactor regression)."""
    x = rm(golden, 40, 16, 10000)
    oracle = O.full_svd(x).sigma
    f = impl.hierarchical_svd(x, impl.MatConfig(gamma=1e-12, row_block_rows=20,
                                                col_block_cols=8))
    assert f.rank() == oracle.shape[0]
    eps = _t(tol, "approx10", 1e-10)
    for i in range(f.rank()):
        # doctest::Approx(b).epsilon(e): |a-b| < e*(1 + max(|a|,|b|))
        assert abs(f.sigma[i] - oracle[i]) < eps * (1.0 + max(abs(f.sigma[i]), abs(oracle[i])))


# --------------------------------------------------------------------------
# test_factor.cpp
# --------------------------------------------------------------------------

def case_rank_k_error_regression(impl, golden, tol=None):
    """test_factor.cpp:176-198: pinned rank_k_error = 8.1960876183812958e-09."""
    x, _ = lowrank(golden, 64, 32, 2024, "exp", 8, ratio=0.5, floor=1e-4)
    cfg = impl.MatConfig(gamma=1e-3, row_block_rows=16, col_block_cols=8)
    right = impl.hierarchical_svd(x, cfg)
    approx = impl.recover_left_vectors(x, right.v)
    assert approx.rank() == 8
    if impl is O:
        err = O.rank_k_error(x, O.SvdFactor(approx.u, approx.sigma, approx.v), 8)
    else:  # the product evaluates the metric on the device too
        err = impl.rank_k_error(x, approx, 8)
    rel = _t(tol, "rank_k_error_rel", 1e-6)
    assert abs(err - 8.1960876183812958e-09) <= rel * 8.1960876183812958e-09, err


def case_cli_gen_svd(impl, golden, tol=None):
    """test_cli.cpp:56-66 / acceptance.cpp:365-403: gen 64x32 rank 4 exp:0.5
    seed 7, svd --gamma 1e-6 -> rank 4, sigma 1 0.5 0.25 0.125."""
    x, _ = lowrank(golden, 64, 32, 7, "exp", 4, ratio=0.5)
    right = impl.hierarchical_svd(x, impl.MatConfig(gamma=1e-6))
    f = impl.recover_left_vectors(x, right.v)
    assert f.rank() == 4
    assert np.abs(f.sigma - np.array([1.0, 0.5, 0.25, 0.125])).max() < 1e-7


# --------------------------------------------------------------------------
# test_kernels.cpp
# --------------------------------------------------------------------------

def case_full_svd_kernels(impl, golden, tol=None):
    """test_kernels.cpp:10-57 and :108-122 (Gram-spectrum oracle across the
    Jacobi/BDCSVD crossover)."""
    f = impl.full_svd(np.eye(2))
    assert np.abs(f.sigma - 1.0).max() < 1e-12
    a = np.zeros((2, 2))
    a[0, 0], a[1, 1] = 3.0, -2.0
    f = impl.full_svd(a)
    assert abs(f.sigma[0] - 3.0) < 1e-12 and abs(f.sigma[1] - 2.0) < 1e-12
    a = rm(golden, 5, 3, 7)
    f = impl.full_svd(a)
    assert f.u.shape == (5, 3) and f.v.shape == (3, 3)
    assert O.orthonormality_defect(f.u) < 1e-10 and O.orthonormality_defect(f.v) < 1e-10
    assert np.linalg.norm(O.reconstruct(O.SvdFactor(f.u, f.sigma, f.v)) - a) < 1e-12 * np.linalg.norm(a)
    for n in (8, 16, 31, 32, 33, 48):
        a = rm(golden, 2 * n, n, 5000 + n)
        f = impl.full_svd(a)
        ev = np.linalg.eigvalsh(a.T @ a)[::-1]
        oracle = np.sqrt(np.maximum(ev, 0.0))
        for i in range(n):
            assert abs(f.sigma[i] - oracle[i]) < 1e-10 * (1.0 + max(f.sigma[i], oracle[i]))
        assert abs(np.sum(f.sigma ** 2) - np.sum(a * a)) < 1e-12 * (1.0 + np.sum(a * a))


# --------------------------------------------------------------------------
# acceptance.cpp
# --------------------------------------------------------------------------

def case_acceptance_exactness(impl, golden, tol=None, trials=20):
    """acceptance.cpp:77-112: 20 matrices x 4 plans, sigma 1e-8, recon 1e-8."""
    for t in range(trials):
        m = 40 + 8 * (t % 21)
        n = 16 + 8 * (t % 7)
        x = rm(golden, m, n, 10000 + t)
        oracle = O.full_svd(x).sigma
        xnorm = np.linalg.norm(x)
        for d, c in ((m, n), (m // 2, n // 2), (m // 4, n // 8), (64, 8)):
            cfg = impl.MatConfig(gamma=1e-12, row_block_rows=d, col_block_cols=c)
            f = impl.hierarchical_svd(x, cfg)
            assert f.rank() == oracle.shape[0], (t, d, c)
            denom = np.maximum(np.abs(oracle), 1e-6 * abs(oracle[0]))
            assert (np.abs(f.sigma - oracle) / denom).max() <= 1e-8, (t, d, c)
            ap = impl.recover_left_vectors(x, f.v)
            rx = O.reconstruct(O.SvdFactor(ap.u, ap.sigma, ap.v))
            assert np.linalg.norm(rx - x) <= 1e-8 * xnorm, (t, d, c)


def case_acceptance_merge_oracle(impl, golden, tol=None):
    """acceptance.cpp:115-149: both orientations, worst deviation 1e-9."""
    worst = 0.0
    for t in range(100):
        shared = 10 + t % 41
        k = 1 + t % 6
        l = 1 + (t * 5) % 6
        s1 = np.array([0.75 ** i for i in range(k)])
        s2 = np.array([1.3 * 0.6 ** i for i in range(l)])
        for column in (True, False):
            if column:
                b1, b2 = ro(golden, shared, k, 20000 + 4 * t), ro(golden, shared, l, 20001 + 4 * t)
                f1 = impl.SvdFactor(u=b1, sigma=s1, v=None)
                f2 = impl.SvdFactor(u=b2, sigma=s2, v=None)
                o1, o2 = O.SvdFactor(b1, s1, None), O.SvdFactor(b2, s2, None)
            else:
                b1, b2 = ro(golden, shared, k, 20002 + 4 * t), ro(golden, shared, l, 20003 + 4 * t)
                f1 = impl.SvdFactor(u=None, sigma=s1, v=b1)
                f2 = impl.SvdFactor(u=None, sigma=s2, v=b2)
                o1, o2 = O.SvdFactor(None, s1, b1), O.SvdFactor(None, s2, b2)
            orient = impl.COLUMN_CONCAT if column else impl.ROW_CONCAT
            naive = O.merge_pair_naive(o1, o2, O.COLUMN_CONCAT if column else O.ROW_CONCAT, 0.0)
            fast = impl.merge_pair_qr(f1, f2, orient, 0.0)
            assert fast.rank() == naive.rank(), t
            denom = np.maximum(np.abs(naive.sigma), 1e-6 * abs(naive.sigma[0]))
            worst = max(worst, float((np.abs(fast.sigma - naive.sigma) / denom).max()))
    assert worst <= 1e-9, worst


# --------------------------------------------------------------------------
# test_refine.cpp (refine_factors, Alg. 2 -- SURVEY 8(f) next #1)
# --------------------------------------------------------------------------

def case_refine_fixed_point(impl, golden, tol=None):
    """test_refine.cpp:13-23."""
    x = rm(golden, 24, 12, 800)
    full = O.full_svd(x)
    r = 4
    res = impl.refine_factors(x, full.v[:, :r].copy(), full.sigma[:r].copy(), 1e-3, 10)
    assert res.iterations == 1
    assert res.converged
    assert res.final_error <= 1e-12
    assert np.abs(res.factor.sigma - full.sigma[:r]).max() < 1e-10 * full.sigma[0]


def case_refine_rotated_subspace(impl, golden, tol=None):
    """test_refine.cpp:25-36: the fixed point depends only on the span."""
    x = rm(golden, 30, 15, 810)
    full = O.full_svd(x)
    r = 5
    rotated = full.v[:, :r] @ ro(golden, r, r, 811)
    res = impl.refine_factors(x, rotated, full.sigma[:r].copy(), 1e-10, 20)
    assert res.converged
    assert np.abs(res.factor.sigma - full.sigma[:r]).max() < 1e-10


def case_refine_hierarchical_output(impl, golden, tol=None):
    """test_refine.cpp:38-54."""
    x, _ = lowrank(golden, 512, 128, 820, "exp", 25, ratio=0.7, floor=1e-6)
    cfg = impl.MatConfig(gamma=1e-2, row_block_rows=128, col_block_cols=16)
    right = impl.hierarchical_svd(x, cfg)
    res = impl.refine_factors(x, right.v, right.sigma, 1e-3, 10)
    assert res.converged
    assert res.iterations <= 3


def case_refine_sigma_bounded(impl, golden, tol=None):
    """test_refine.cpp:56-67: refined sigma never exceeds the true ones."""
    x = rm(golden, 40, 18, 830)
    true_sigma = O.full_svd(x).sigma
    right = impl.hierarchical_svd(x, impl.MatConfig(gamma=0.1, row_block_rows=10,
                                                    col_block_cols=6))
    res = impl.refine_factors(x, right.v, right.sigma, 1e-6, 10)
    for i in range(res.factor.rank()):
        assert res.factor.sigma[i] <= true_sigma[i] + 1e-10 * true_sigma[0]


def case_refine_top_monotone(impl, golden, tol=None):
    """test_refine.cpp:69-89: chained single iterations, sigma_1 grows."""
    x = rm(golden, 50, 25, 840)
    right = impl.hierarchical_svd(x, impl.MatConfig(gamma=0.2, row_block_rows=25,
                                                    col_block_cols=5))
    v, sigma = right.v, right.sigma
    prev_top = sigma[0]
    for _ in range(4):
        res = impl.refine_factors(x, v, sigma, 1e-15, 1)
        assert res.factor.sigma[0] >= prev_top - 1e-10 * prev_top
        prev_top = res.factor.sigma[0]
        v, sigma = res.factor.v, res.factor.sigma


def case_refine_never_hurts(impl, golden, tol=None):
    """test_refine.cpp:91-110 (50 trials)."""
    checked = 0
    for trial in range(50):
        m, n = 24 + 4 * (trial % 5), 12 + 2 * (trial % 4)
        x = rm(golden, m, n, 850 + trial)
        cfg = impl.MatConfig(gamma=0.05 + 0.05 * (trial % 3), row_block_rows=m // 2,
                             col_block_cols=n // 3)
        right = impl.hierarchical_svd(x, cfg)
        before = impl.recover_left_vectors(x, right.v)
        res = impl.refine_factors(x, right.v, right.sigma, 1e-6, 10)
        k = min(before.rank(), res.factor.rank())
        full = O.full_svd(x)
        err_before = O.rank_k_error(full, O.SvdFactor(before.u, before.sigma, before.v), k)
        err_after = O.rank_k_error(full, O.SvdFactor(res.factor.u, res.factor.sigma,
                                                     res.factor.v), k)
        assert err_after <= err_before + _t(tol, "refine_never_hurts", 1e-12), trial
        checked += 1
    assert checked == 50


def case_refine_orthonormal(impl, golden, tol=None):
    """test_refine.cpp:112-122."""
    x = rm(golden, 30, 20, 860)
    right = impl.hierarchical_svd(x, impl.MatConfig(gamma=0.1, row_block_rows=15,
                                                    col_block_cols=5))
    res = impl.refine_factors(x, right.v, right.sigma, 1e-4, 10)
    assert O.orthonormality_defect(res.factor.u) < 1e-8
    assert O.orthonormality_defect(res.factor.v) < 1e-8


def case_refine_nonconvergence(impl, golden, tol=None):
    """test_refine.cpp:124-136: reported, not thrown."""
    x = rm(golden, 20, 10, 870)
    right = impl.hierarchical_svd(x, impl.MatConfig(gamma=0.5, row_block_rows=5,
                                                    col_block_cols=2))
    res = impl.refine_factors(x, right.v, right.sigma, 1e-300, 1)
    assert res.iterations == 1
    assert not res.converged
    assert res.final_error > 0.0


def case_refine_validation(impl, golden, tol=None):
    """test_refine.cpp:138-150."""
    x = rm(golden, 10, 6, 880)
    full = O.full_svd(x)
    v2 = full.v[:, :2].copy()
    assert raises(ValueError, impl.refine_factors, x, v2, full.sigma[:3].copy(), 1e-3, 10)
    assert raises(ValueError, impl.refine_factors, x, v2, full.sigma[:2].copy(), 0.0, 10)
    assert raises(ValueError, impl.refine_factors, x, v2, full.sigma[:2].copy(), 1e-3, 0)
    assert raises(ValueError, impl.refine_factors, x, rm(golden, 6, 2, 881),
                  full.sigma[:2].copy(), 1e-3, 10)


ALL_CASES = [
    case_merge_self_sqrt2, case_merge_orthogonal_units, case_naive_concat_oracle,
    case_identical_basis, case_orthogonal_union, case_qr_equals_naive_100,
    case_merge_properties, case_merge_gamma_and_cap, case_merge_fallback,
    case_merge_degenerate, case_merge_rejects, case_block_plan,
    case_tree_merge_counts, case_tree_merge_eight_blocks, case_col_slices,
    case_hsvd_single_block, case_hsvd_rank10, case_hsvd_exact_plans,
    case_hsvd_no_inflation, case_recover_left, case_full_width_row_slices,
    case_rank_k_error_regression, case_cli_gen_svd, case_full_svd_kernels,
    case_acceptance_exactness, case_acceptance_merge_oracle,
    case_refine_fixed_point, case_refine_rotated_subspace, case_refine_hierarchical_output,
    case_refine_sigma_bounded, case_refine_top_monotone, case_refine_never_hurts,
    case_refine_orthonormal, case_refine_nonconvergence, case_refine_validation,
]
