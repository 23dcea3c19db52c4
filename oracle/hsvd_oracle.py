"""CPU oracle: a numpy/LAPACK restatement of the reference hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product (``paper_1710_02812_b200``)
imports this module.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and its ``--impl reference`` arm) may
import it, and only as the checker / the timed CPU baseline.

It restates, in fp64, the algorithm of the reference C++ library
(``/root/reference/proj/core``; Eigen 3.4 is not installed here, so the dense
kernels are LAPACK through numpy/scipy):

* ``full_svd``           kernels.cpp:21-48   (Jacobi for min<=32 -> ``dgejsv``;
                                              else BDCSVD -> ``dgesdd``; energy
                                              check -> Jacobi fallback)
* ``qr_thin``            kernels.cpp:50-61   (HouseholderQR -> ``dgeqrf+dorgqr``)
* ``retained_count``     svd_factor.cpp:23-30
* ``truncate_factor``    svd_factor.cpp:32-46
* ``reconstruct``/``rank_k_error``/``normalize_signs``  svd_factor.cpp:48-104
* ``merge_pair_naive``   merge.cpp:42-69
* ``merge_pair_qr``      merge.cpp:71-117
* ``partition``/``BlockPlan``  hierarchy.cpp:11-29
* ``tree_merge``         hierarchy.cpp:31-48
* ``svd_of_col_slices``  hierarchy.cpp:50-63
* ``hierarchical_svd``   hierarchy.cpp:65-94
* ``recover_left_vectors`` hierarchy.cpp:96-112
* ``build_spectrum``/``gen_low_rank`` generate.cpp:46-94 (from caller-supplied
  Gaussians: the reference's mt19937_64 + std::normal_distribution stream is
  reproduced by ``oracle/gen_ref_gaussians.cpp`` into ``tests/golden``)

Parity of this restatement is pinned against the reference's own known-answer
tests (see ``tests/test_oracle_golden.py``), e.g. the ``rank_k_error``
regression value 8.1960876183812958e-09 of ``tests/test_factor.cpp:176-198``.

fp32 inputs are promoted to fp64 per block, which is exactly what the
reference's fp64 ``DenseMatrix`` computes on the same bytes.
"""
from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

try:  # scipy is in the image; it supplies dgejsv (Jacobi SVD)
    from scipy.linalg import lapack as _lapack
except Exception:  # pragma: no cover
    _lapack = None


class DecompositionError(RuntimeError):
    """kernels.hpp:12-17 -- a dense kernel failed to converge."""

    def __init__(self, what: str, rows: int, cols: int):
        super().__init__(what)
        self.rows = rows
        self.cols = cols


COLUMN_CONCAT = "ColumnConcat"
ROW_CONCAT = "RowConcat"


@dataclass
class SvdFactor:
    """svd_factor.hpp:14-25."""

    u: Optional[np.ndarray]
    sigma: np.ndarray
    v: Optional[np.ndarray]
    degenerate: bool = False

    def rank(self) -> int:
        return int(self.sigma.shape[0])

    def has_u(self) -> bool:
        return self.u is not None

    def has_v(self) -> bool:
        return self.v is not None


@dataclass
class MatConfig:
    """svd_factor.hpp:28-35."""

    gamma: float = 1e-2
    row_block_rows: int = 0
    col_block_cols: int = 0
    epsilon: float = 1e-3
    max_iters: int = 10
    max_rank: Optional[int] = None


def validate(cfg: MatConfig) -> None:
    """svd_factor.cpp:10-21."""
    if cfg.gamma < 0.0 or not math.isfinite(cfg.gamma):
        raise ValueError("MatConfig: gamma must be finite and >= 0")
    if not (cfg.epsilon > 0.0):
        raise ValueError("MatConfig: epsilon must be > 0")
    if cfg.max_iters < 1:
        raise ValueError("MatConfig: max_iters must be >= 1")
    if cfg.row_block_rows < 0 or cfg.col_block_cols < 0:
        raise ValueError("MatConfig: block sizes must be >= 0")
    if cfg.max_rank is not None and cfg.max_rank < 1:
        raise ValueError("MatConfig: max_rank must be >= 1")


# --------------------------------------------------------------------------
# L1 dense kernels (kernels.cpp)
# --------------------------------------------------------------------------

def _jacobi_svd(a: np.ndarray) -> SvdFactor:
    """kernels.cpp:10-18: two-sided Jacobi (Eigen JacobiSVD) -> LAPACK dgejsv."""
    m, n = a.shape
    wide = m < n
    t = a.T if wide else a
    if _lapack is not None:
        sva, u, v, work, _iw, info = _lapack.dgejsv(
            np.asfortranarray(t), joba=4, jobu=0, jobv=0, jobr=1, jobt=0, jobp=0)
        if info != 0:
            raise DecompositionError(
                f"SVD did not converge for a {m}x{n} matrix", m, n)
        s = sva * (work[0] / work[1])
        order = np.argsort(-s, kind="stable")
        s, u, v = s[order], u[:, order], v[:, order]
    else:  # pragma: no cover
        u, s, vt = np.linalg.svd(t, full_matrices=False)
        v = vt.T
    if wide:
        u, v = v, u
    return SvdFactor(u=np.ascontiguousarray(u), sigma=np.ascontiguousarray(s),
                     v=np.ascontiguousarray(v))


def full_svd(a: np.ndarray) -> SvdFactor:
    """kernels.cpp:21-48 -- thin SVD, U rows x p, sigma p, V cols x p."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] == 0 or a.shape[1] == 0:
        raise ValueError("full_svd: matrix is empty")
    if min(a.shape) <= 32:
        return _jacobi_svd(a)
    try:
        u, s, vt = np.linalg.svd(a, full_matrices=False)  # dgesdd ~ BDCSVD
    except np.linalg.LinAlgError as exc:  # pragma: no cover
        raise DecompositionError(
            f"SVD did not converge for a {a.shape[0]}x{a.shape[1]} matrix",
            a.shape[0], a.shape[1]) from exc
    energy = float(np.sum(a * a))
    sigma_energy = float(np.sum(s * s))
    if abs(sigma_energy - energy) > 1e-10 * energy:  # kernels.cpp:36-41
        return _jacobi_svd(a)
    return SvdFactor(u=u, sigma=s, v=np.ascontiguousarray(vt.T))


def qr_thin(a: np.ndarray):
    """kernels.cpp:50-61 -- Householder thin QR (q rows x p, r p x cols)."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] == 0 or a.shape[1] == 0:
        raise ValueError("qr_thin: matrix is empty")
    q, r = np.linalg.qr(a, mode="reduced")
    return q, r


# --------------------------------------------------------------------------
# L2 factor algebra (svd_factor.cpp)
# --------------------------------------------------------------------------

def retained_count(sigma: np.ndarray, gamma: float) -> int:
    """svd_factor.cpp:23-30: sigma_i >= gamma*sigma_1 (ties kept), min 1."""
    sigma = np.asarray(sigma)
    if sigma.shape[0] == 0:
        return 0
    if sigma[0] == 0.0:
        return 1
    cutoff = gamma * sigma[0]
    kept = 0
    while kept < sigma.shape[0] and sigma[kept] >= cutoff:
        kept += 1
    return max(kept, 1)


def truncate_factor(f: SvdFactor, gamma: float,
                    max_rank: Optional[int] = None) -> SvdFactor:
    """svd_factor.cpp:32-46."""
    if f.sigma.shape[0] == 0:
        raise ValueError("truncate_factor: factor has an empty spectrum")
    keep = retained_count(f.sigma, gamma)
    if max_rank is not None:
        keep = min(keep, max(int(max_rank), 1))
    return SvdFactor(
        u=None if f.u is None else f.u[:, :keep].copy(),
        sigma=f.sigma[:keep].copy(),
        v=None if f.v is None else f.v[:, :keep].copy(),
        degenerate=bool(f.degenerate or f.sigma[0] == 0.0))


def reconstruct(f: SvdFactor) -> np.ndarray:
    """svd_factor.cpp:48-52."""
    if f.u is None or f.v is None:
        raise ValueError("reconstruct: factor must carry both u and v")
    return (f.u * f.sigma) @ f.v.T


def _head(f: SvdFactor, k: int) -> SvdFactor:
    return SvdFactor(u=None if f.u is None else f.u[:, :k],
                     sigma=f.sigma[:k],
                     v=None if f.v is None else f.v[:, :k])


def rank_k_error(full_of_x_or_x, approx: SvdFactor, k: int) -> float:
    """svd_factor.cpp:65-85 (both overloads)."""
    if approx.u is None or approx.v is None:
        raise ValueError("rank_k_error: approx must carry both u and v")
    if k < 1 or k > approx.rank():
        raise ValueError("rank_k_error: k must be in [1, approx.rank()]")
    full = (full_of_x_or_x if isinstance(full_of_x_or_x, SvdFactor)
            else full_svd(full_of_x_or_x))
    k_ref = min(k, full.rank())
    x_k = reconstruct(_head(full, k_ref))
    denom = float(np.linalg.norm(x_k))
    if denom == 0.0:
        raise ValueError("rank_k_error: reference rank-k approximation is zero")
    xhat_k = reconstruct(_head(approx, k))
    return float(np.linalg.norm(x_k - xhat_k)) / denom


def normalize_signs(f: SvdFactor) -> None:
    """svd_factor.cpp:87-104."""
    for j in range(f.rank()):
        flip = 1.0
        if f.u is not None:
            imax = int(np.argmax(np.abs(f.u[:, j])))
            if f.u[imax, j] < 0.0:
                flip = -1.0
        elif f.v is not None:
            imax = int(np.argmax(np.abs(f.v[:, j])))
            if f.v[imax, j] < 0.0:
                flip = -1.0
        if flip < 0.0:
            if f.u is not None:
                f.u[:, j] = -f.u[:, j]
            if f.v is not None:
                f.v[:, j] = -f.v[:, j]


# --------------------------------------------------------------------------
# L3 merge (merge.cpp)
# --------------------------------------------------------------------------

def _carried_basis(f: SvdFactor, orient: str) -> np.ndarray:
    """merge.cpp:11-19."""
    if orient == COLUMN_CONCAT:
        if f.u is None:
            raise ValueError("merge: ColumnConcat requires both factors to carry u")
        return f.u
    if f.v is None:
        raise ValueError("merge: RowConcat requires both factors to carry v")
    return f.v


def _check_dims(b1, b2, orient):
    """merge.cpp:21-26."""
    if b1.shape[0] != b2.shape[0]:
        raise ValueError(
            "merge: ColumnConcat factors must have equal row counts"
            if orient == COLUMN_CONCAT else
            "merge: RowConcat factors must have equal column counts")


def _make_result(basis, sigma, orient, degenerate) -> SvdFactor:
    if orient == COLUMN_CONCAT:
        return SvdFactor(u=basis, sigma=sigma, v=None, degenerate=degenerate)
    return SvdFactor(u=None, sigma=sigma, v=basis, degenerate=degenerate)


def merge_pair_naive(f1: SvdFactor, f2: SvdFactor, orient: str, gamma: float,
                     max_rank: Optional[int] = None) -> SvdFactor:
    """merge.cpp:42-69: one SVD of the stacked weighted vectors."""
    b1 = _carried_basis(f1, orient)
    b2 = _carried_basis(f2, orient)
    _check_dims(b1, b2, orient)
    if orient == COLUMN_CONCAT:
        stacked = np.hstack([b1 * f1.sigma, b2 * f2.sigma])
        s = full_svd(stacked)
        s.v = None
    else:
        stacked = np.vstack([(b1 * f1.sigma).T, (b2 * f2.sigma).T])
        s = full_svd(stacked)
        s.u = None
    return truncate_factor(s, gamma, max_rank)


def merge_pair_qr(f1: SvdFactor, f2: SvdFactor, orient: str, gamma: float,
                  max_rank: Optional[int] = None) -> SvdFactor:
    """merge.cpp:71-117: merge through the orthogonal complement."""
    b1 = _carried_basis(f1, orient)
    b2 = _carried_basis(f2, orient)
    _check_dims(b1, b2, orient)
    k, l = f1.rank(), f2.rank()
    shared = b1.shape[0]
    if k + l > shared:  # merge.cpp:84
        return merge_pair_naive(f1, f2, orient, gamma, max_rank)
    w = b1.T @ b2                                   # merge.cpp:86
    q = b2 - b1 @ w
    b_o, r = qr_thin(q)                             # merge.cpp:88-90
    if np.abs(b_o.T @ b1).max() > 1e-8:             # merge.cpp:94-99
        q = b_o - b1 @ (b1.T @ b_o)
        b_o2, r2 = qr_thin(q)
        b_o = b_o2
        r = r2 @ r
    e = np.zeros((k + l, k + l))                    # merge.cpp:101-104
    e[:k, :k] = np.diag(f1.sigma)
    e[:k, k:] = w * f2.sigma
    e[k:, k:] = r * f2.sigma
    se = full_svd(e)
    cap = max(int(max_rank), 1) if max_rank is not None else k + l
    keep = min(retained_count(se.sigma, gamma), cap)  # merge.cpp:107-109
    ue = se.u
    basis = b1 @ ue[:k, :keep] + b_o @ ue[k:, :keep]  # merge.cpp:113
    return _make_result(basis, se.sigma[:keep].copy(), orient,
                        bool(se.sigma[0] == 0.0))


# --------------------------------------------------------------------------
# L4 hierarchy (hierarchy.cpp)
# --------------------------------------------------------------------------

def partition(extent: int, block: int):
    """hierarchy.cpp:11-18: contiguous ceil-division slices (start, count)."""
    if block < 1 or block > extent:
        block = extent
    return [(s, min(block, extent - s)) for s in range(0, extent, block)]


@dataclass
class BlockPlan:
    """hierarchy.hpp:18-23 / hierarchy.cpp:22-29."""

    row_slices: list = field(default_factory=list)
    col_slices: list = field(default_factory=list)

    @staticmethod
    def make(rows: int, cols: int, d: int, c: int) -> "BlockPlan":
        if rows < 1 or cols < 1:
            raise ValueError("BlockPlan: matrix must be nonempty")
        return BlockPlan(partition(rows, d), partition(cols, c))


@dataclass
class MergeStats:
    pair_merges: int = 0


def tree_merge(factors: Sequence[SvdFactor], orient: str, gamma: float,
               max_rank: Optional[int] = None,
               stats: Optional[MergeStats] = None,
               workers: int = 1) -> SvdFactor:
    """hierarchy.cpp:31-48: (0,1),(2,3),... per level, odd factor carried."""
    factors = list(factors)
    if not factors:
        raise ValueError("tree_merge: factor list is empty")
    while len(factors) > 1:
        pairs = [(factors[i], factors[i + 1]) for i in range(0, len(factors) - 1, 2)]
        if workers > 1 and len(pairs) > 1:
            with ThreadPoolExecutor(workers) as ex:
                nxt = list(ex.map(
                    lambda p: merge_pair_qr(p[0], p[1], orient, gamma, max_rank), pairs))
        else:
            nxt = [merge_pair_qr(a, b, orient, gamma, max_rank) for a, b in pairs]
        if stats is not None:
            stats.pair_merges += len(pairs)
        if len(factors) % 2 == 1:
            nxt.append(factors[-1])
        factors = nxt
    return factors[0]


def _leaf(x_slice: np.ndarray, s0: int, cnt: int, gamma, max_rank) -> SvdFactor:
    block = np.asarray(x_slice[:, s0:s0 + cnt], dtype=np.float64)
    f = truncate_factor(full_svd(block), gamma, max_rank)
    f.v = None  # hierarchy.cpp:59
    return f


def svd_of_col_slices(x_slice: np.ndarray, c: int, gamma: float,
                      max_rank: Optional[int] = None, workers: int = 1) -> SvdFactor:
    """hierarchy.cpp:50-63."""
    slices = partition(x_slice.shape[1], c)
    if workers > 1 and len(slices) > 1:
        with ThreadPoolExecutor(workers) as ex:
            leaves = list(ex.map(lambda s: _leaf(x_slice, s[0], s[1], gamma, max_rank),
                                 slices))
    else:
        leaves = [_leaf(x_slice, s0, cnt, gamma, max_rank) for s0, cnt in slices]
    return tree_merge(leaves, COLUMN_CONCAT, gamma, max_rank, workers=workers)


def _row_slice_factor(x: np.ndarray, j: int, s0: int, cnt: int, cfg: MatConfig,
                      workers: int) -> SvdFactor:
    try:
        x_j = x[s0:s0 + cnt]
        col_merged = svd_of_col_slices(x_j, cfg.col_block_cols, cfg.gamma,
                                       cfg.max_rank, workers)
        b = _ut_x(col_merged.u, x_j)  # hierarchy.cpp:83
        recovered = full_svd(b)
        recovered.u = None
        return truncate_factor(recovered, cfg.gamma, cfg.max_rank)
    except DecompositionError as err:  # hierarchy.cpp:86-89
        raise DecompositionError(f"row slice {j}: {err}", err.rows, err.cols) from err


_CHUNK_ELEMS = 1 << 25  # fp64 promotion done in pieces of <= 256 MB


def _ut_x(u: np.ndarray, x_j: np.ndarray) -> np.ndarray:
    """B = U^T X_j with X_j promoted to fp64 a column chunk at a time (the
    same column-by-column product; bounds host memory at full BASELINE
    sizes, where one promoted row slice would be GBs per thread)."""
    rows, cols = x_j.shape
    step = max(1, _CHUNK_ELEMS // max(1, rows))
    if step >= cols:
        return u.T @ np.asarray(x_j, dtype=np.float64)
    b = np.empty((u.shape[1], cols))
    for c0 in range(0, cols, step):
        b[:, c0:c0 + step] = u.T @ np.asarray(x_j[:, c0:c0 + step], dtype=np.float64)
    return b


def _x_v(x: np.ndarray, v: np.ndarray) -> np.ndarray:
    """Y = X V with X promoted to fp64 a row chunk at a time (row by row the
    same product)."""
    rows, cols = x.shape
    step = max(1, _CHUNK_ELEMS // max(1, cols))
    if step >= rows:
        return np.asarray(x, dtype=np.float64) @ v
    y = np.empty((rows, v.shape[1]))
    for r0 in range(0, rows, step):
        y[r0:r0 + step] = np.asarray(x[r0:r0 + step], dtype=np.float64) @ v
    return y


def hierarchical_svd(x: np.ndarray, cfg: MatConfig, workers: int = 1) -> SvdFactor:
    """hierarchy.cpp:65-94 -> (Sigma, V) with u absent."""
    x = np.asarray(x)
    if x.ndim != 2 or x.shape[0] == 0 or x.shape[1] == 0:
        raise ValueError("hierarchical_svd: matrix is empty")
    validate(cfg)
    row_slices = partition(x.shape[0], cfg.row_block_rows)
    if workers > 1 and len(row_slices) > 1:
        inner = max(1, workers // len(row_slices))
        with ThreadPoolExecutor(workers) as ex:
            slice_factors = list(ex.map(
                lambda js: _row_slice_factor(x, js[0], js[1][0], js[1][1], cfg, inner),
                enumerate(row_slices)))
    else:
        slice_factors = [_row_slice_factor(x, j, s0, cnt, cfg, workers)
                         for j, (s0, cnt) in enumerate(row_slices)]
    return tree_merge(slice_factors, ROW_CONCAT, cfg.gamma, cfg.max_rank,
                      workers=workers)


def recover_left_vectors(x: np.ndarray, v_r: np.ndarray) -> SvdFactor:
    """hierarchy.cpp:96-112 -> full (U, Sigma, V)."""
    v_r = np.asarray(v_r, dtype=np.float64)
    if v_r.shape[0] != x.shape[1]:
        raise ValueError("recover_left_vectors: v_r must have x.cols() rows")
    r = v_r.shape[1]
    defect = np.abs(v_r.T @ v_r - np.eye(r)).max()
    if defect > 1e-6:
        raise ValueError("recover_left_vectors: v_r columns are not orthonormal")
    y = full_svd(_x_v(x, v_r))
    return SvdFactor(u=y.u, sigma=y.sigma, v=v_r @ y.v)


# --------------------------------------------------------------------------
# Refinement (refine.cpp, Alg. 2 of the paper) -- SURVEY 8(f) next #1
# --------------------------------------------------------------------------

@dataclass
class RefineResult:
    """refine.hpp:9-14."""
    factor: SvdFactor
    iterations: int = 0
    final_error: float = 0.0
    converged: bool = False


def _padded_diff_norm(a: np.ndarray, b: np.ndarray) -> float:
    """refine.cpp:13-22: ||a - b||_2 with the shorter vector zero-padded."""
    n = max(a.shape[0], b.shape[0])
    aa = np.zeros(n)
    bb = np.zeros(n)
    aa[:a.shape[0]] = a
    bb[:b.shape[0]] = b
    return float(math.sqrt(float(((aa - bb) ** 2).sum())))


def refine_factors(x: np.ndarray, v_hat: np.ndarray, sigma_hat: np.ndarray,
                   epsilon: float, max_iters: int) -> RefineResult:
    """refine.cpp:26-72: alternate thin SVDs of X V and U_outer^T X until the
    relative change of the singular-value vector is <= epsilon or max_iters
    is reached (non-convergence is reported, not raised)."""
    x = np.asarray(x, dtype=np.float64)
    v_hat = np.asarray(v_hat, dtype=np.float64)
    sigma_hat = np.asarray(sigma_hat, dtype=np.float64)
    if not epsilon > 0.0:
        raise ValueError("refine_factors: epsilon must be > 0")
    if max_iters < 1:
        raise ValueError("refine_factors: max_iters must be >= 1")
    if sigma_hat.shape[0] != v_hat.shape[1]:
        raise ValueError("refine_factors: sigma_hat length must match v_hat columns")
    if v_hat.shape[0] != x.shape[1]:
        raise ValueError("refine_factors: v_hat must have x.cols() rows")
    defect = np.abs(v_hat.T @ v_hat - np.eye(v_hat.shape[1])).max()
    if defect > 1e-6:
        raise ValueError("refine_factors: v_hat columns are not orthonormal")
    sigma = sigma_hat.copy()
    v = v_hat
    res = RefineResult(factor=SvdFactor(None, sigma, None))
    error = 0.0
    while True:
        res.iterations += 1
        u_outer = full_svd(x @ v).u                   # refine.cpp:50-51
        step = full_svd(u_outer.T @ x)                 # refine.cpp:53
        denom = float(np.linalg.norm(sigma))
        diff = _padded_diff_norm(sigma, step.sigma)
        error = diff / denom if denom > 0.0 else (math.inf if diff > 0.0 else 0.0)
        sigma, v, u_inner = step.sigma, step.v, step.u
        if not (error > epsilon and res.iterations < max_iters):
            break
    res.factor = SvdFactor(u=u_outer @ u_inner, sigma=sigma, v=v)
    res.final_error = error
    res.converged = error <= epsilon
    return res


# --------------------------------------------------------------------------
# Generator (generate.cpp) -- spectrum + assembly from supplied Gaussians
# --------------------------------------------------------------------------

def build_spectrum(p: int, kind: str, rank: int, ratio: float = 0.5,
                   exponent: float = 1.0, values=None,
                   noise_floor: float = 0.0) -> np.ndarray:
    """generate.cpp:46-73 (sigma_1 = 1, decay to rank, constant floor)."""
    if kind == "explicit":
        rank = min(len(values), p)
    else:
        rank = min(rank, p)
    sigma = np.empty(p)
    if kind == "exp":
        for i in range(rank):
            sigma[i] = math.pow(ratio, float(i))
    elif kind == "pow":
        for i in range(rank):
            sigma[i] = math.pow(float(i + 1), -exponent)
    elif kind == "explicit":
        top = max(values)
        scale = 1.0 / top if top > 0.0 else 1.0
        for i in range(rank):
            sigma[i] = values[i] * scale
    else:
        raise ValueError(kind)
    sigma[rank:] = noise_floor
    return np.sort(sigma)[::-1].copy()


def gen_low_rank_from_gaussians(g_u: np.ndarray, g_v: np.ndarray,
                                sigma: np.ndarray) -> np.ndarray:
    """generate.cpp:75-94: X = qr(Gu).Q diag(sigma) qr(Gv).Q^T."""
    u = qr_thin(g_u)[0]
    v = qr_thin(g_v)[0]
    return (u * sigma) @ v.T


# --------------------------------------------------------------------------
# Parity metrics (tests/test_support.hpp)
# --------------------------------------------------------------------------

def orthonormality_defect(m: np.ndarray) -> float:
    """test_support.hpp:43-46."""
    g = m.T @ m
    return float(np.abs(g - np.eye(m.shape[1])).max())


def max_sigma_rel_diff(a, b, floor_frac: float = 0.0) -> float:
    """test_support.hpp:50-62."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape:
        return float("inf")
    floor = floor_frac * (abs(b[0]) if b.shape[0] > 0 else 0.0)
    scale = np.maximum(np.abs(b), floor)
    diff = np.abs(a - b)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(scale > 0, diff / np.where(scale > 0, scale, 1.0),
                     np.where(diff > 0, np.inf, 0.0))
    return float(r.max()) if r.size else 0.0


def subspace_angle_sin(u1: np.ndarray, u2: np.ndarray) -> float:
    """test_support.hpp:67-70: ||U2 - U1 U1^T U2||_F."""
    return float(np.linalg.norm(u2 - u1 @ (u1.T @ u2)))


def largest_principal_angle(u1: np.ndarray, u2: np.ndarray) -> float:
    """arcsin of the largest sine between span(u1) and span(u2) (radians)."""
    resid = u2 - u1 @ (u1.T @ u2)
    s = np.linalg.svd(resid, compute_uv=False)
    return float(np.arcsin(min(1.0, s[0]))) if s.size else 0.0
