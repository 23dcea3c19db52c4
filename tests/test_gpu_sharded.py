"""The sharded (multi-GPU) device pipeline, driven on one B200 by an
in-process thread group: every rank is a host thread with its own context
and stream; ranks exchange through host-synchronised device copies (no
device-side waits between ranks).  The result must equal the single-context
rank_k_svd: the row-phase tree keeps the reference pairing, so sigma and V
agree to roundoff of the all-reduced Gram."""
import threading

import numpy as np
import pytest

import hsvd_oracle as O

pytestmark = pytest.mark.gpu


def _run_group(H, x, cfg, world):
    grp = H.ThreadGroup(world)
    out = [None] * world
    err = []

    def body(rank):
        try:
            ctx = H.Context(0)
            ctx.join_group(grp, rank)
            r0, ml = H.shard_rows(x.shape[0], cfg.row_block_rows, rank, world)
            out[rank] = (r0, ml, H.rank_k_svd_sharded(x[r0:r0 + ml], x.shape[0], r0, cfg, ctx))
        except Exception as e:  # pragma: no cover
            err.append(repr(e))

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not err, err
    return out


@pytest.mark.parametrize("world,P,Q", [(1, 4, 2), (2, 4, 2), (3, 8, 2), (4, 6, 1)])
def test_sharded_equals_single(world, P, Q):
    import paper_1710_02812_b200 as H
    rng = np.random.default_rng(11 + world)
    m, n, k = 1536, 768, 40
    x = ((np.linalg.qr(rng.standard_normal((m, 60)))[0] * (1.0 / np.arange(1, 61))) @
         np.linalg.qr(rng.standard_normal((n, 60)))[0].T +
         1e-3 * rng.standard_normal((m, n))).astype(np.float32)
    cfg = H.MatConfig(gamma=1e-12, row_block_rows=m // P, col_block_cols=n // Q, max_rank=k)
    single = H.rank_k_svd(x, cfg)
    res = _run_group(H, x, cfg, world)
    u = np.vstack([r[2].u for r in res if r[1] > 0])
    assert sum(r[1] for r in res) == m
    for r0, ml, f in res:
        assert f.rank() == single.rank() == k
        assert np.abs(f.sigma - single.sigma).max() <= 1e-11 * single.sigma[0]
        assert O.largest_principal_angle(single.v, f.v) < 1e-9
    assert O.largest_principal_angle(single.u, u) < 1e-9
    assert O.orthonormality_defect(u) < 1e-8


def test_nccl_world1_path():
    """The NCCL communicator (dlopen'd libnccl) at world size 1 runs the same
    sharded code path as the multi-GPU bench."""
    import paper_1710_02812_b200 as H
    rng = np.random.default_rng(3)
    m, n, k = 1024, 512, 24
    x = (rng.standard_normal((m, 30)) @ rng.standard_normal((30, n)) +
         1e-3 * rng.standard_normal((m, n))).astype(np.float32)
    cfg = H.MatConfig(gamma=1e-12, row_block_rows=m // 4, col_block_cols=n // 2, max_rank=k)
    single = H.rank_k_svd(x, cfg)
    ctx = H.Context(0)
    ctx.init_nccl(0, 1, H.nccl_unique_id())
    f = H.rank_k_svd_sharded(x, m, 0, cfg, ctx)
    assert np.abs(f.sigma - single.sigma).max() <= 1e-11 * single.sigma[0]
    assert O.largest_principal_angle(single.u, f.u) < 1e-9


def test_failing_rank_releases_peers():
    """A rank that fails inside the sharded pipeline aborts the group: its
    peers return an error instead of blocking on it forever."""
    import paper_1710_02812_b200 as H
    rng = np.random.default_rng(5)
    m, n = 512, 256
    x = rng.standard_normal((m, n)).astype(np.float32)
    cfg = H.MatConfig(gamma=1e-12, row_block_rows=128, col_block_cols=128, max_rank=16)
    grp = H.ThreadGroup(2)
    errs = [None, None]

    def body(rank):
        try:
            ctx = H.Context(0)
            ctx.join_group(grp, rank)
            r0, ml = H.shard_rows(m, cfg.row_block_rows, rank, 2)
            if rank == 1:
                ml -= 1  # rows no longer match the shard plan -> this rank fails
            H.rank_k_svd_sharded(x[r0:r0 + ml], m, r0, cfg, ctx)
        except Exception as e:
            errs[rank] = str(e)

    th = [threading.Thread(target=body, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in th), "a rank is still blocked"
    assert errs[1] is not None and "must hold rows" in errs[1]
    assert errs[0] is not None and "peer rank failed" in errs[0]


def test_world8_cfg2_like_equals_single():
    """Eight ranks at a config-2-like shape (8x8 grid, k = 100, fp32, the
    noise-bulk spectrum of config 2): every rank owns one row slice, the row
    tree crosses ranks at all three levels (pairs (0,1),(2,3).. then
    (01,23).. then (0123,4567): SPEC.md:271), V_r is broadcast and the U
    Gram all-reduced.  Equal to the single-context result."""
    import paper_1710_02812_b200 as H
    rng = np.random.default_rng(2)
    m = n = 10000
    r = 100
    u = np.linalg.qr(rng.standard_normal((m, r)))[0]
    v = np.linalg.qr(rng.standard_normal((n, r)))[0]
    x = ((u * np.arange(1, r + 1) ** -1.5) @ v.T + 1e-3 * rng.standard_normal((m, n))).astype(
        np.float32)
    cfg = H.MatConfig(gamma=1e-12, row_block_rows=m // 8, col_block_cols=n // 8, max_rank=100)
    single = H.rank_k_svd(x, cfg)
    res = _run_group(H, x, cfg, 8)
    assert [r[1] for r in res] == [m // 8] * 8
    u_all = np.vstack([r[2].u for r in res])
    for _, _, f in res:
        assert f.rank() == single.rank() == 100
        assert np.abs(f.sigma - single.sigma).max() <= 1e-11 * single.sigma[0]
        assert O.largest_principal_angle(single.v, f.v) < 1e-8
    assert O.largest_principal_angle(single.u, u_all) < 1e-8
    assert O.orthonormality_defect(u_all) < 1e-8
