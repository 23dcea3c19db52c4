"""The multi-GPU (row-sharded) algorithm of engine_shard.cu, restated on the
CPU oracle and run with world_size 2 and 3 over torch.distributed gloo.

It checks the host-side logic the GPU path shares: the row-shard plan
(``hsvd_cu_shard_rows`` from the C ABI), the ownership of slices, the
cross-rank pairing of the row-phase tree (the reference's (0,1),(2,3),...
order with an odd factor carried, hierarchy.cpp:37-46), the V_r broadcast
and the all-reduced U-recovery -- against the single-process oracle.
"""
import os
import socket

import numpy as np
import pytest

import hsvd_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _owner(s, P, world):
    for g in range(world):
        if (g + 1) * P // world > s:
            return g
    return world - 1


def _send_arr(dist, torch, a, dst):
    hdr = torch.tensor(list(a.shape) + [0] * (2 - a.ndim), dtype=torch.int64)
    dist.send(hdr, dst)
    dist.send(torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)), dst)


def _recv_arr(dist, torch, src, ndim):
    hdr = torch.zeros(2, dtype=torch.int64)
    dist.recv(hdr, src)
    shape = tuple(int(v) for v in hdr[:ndim])
    buf = torch.zeros(shape, dtype=torch.float64)
    dist.recv(buf, src)
    return buf.numpy()


def sharded_oracle(x_local, m_total, cfg, rank, world):
    """engine_shard.cu's schedule with oracle arithmetic."""
    import torch
    import torch.distributed as dist
    import paper_1710_02812_b200 as H
    P = len(O.partition(m_total, cfg.row_block_rows))
    first, last = rank * P // world, (rank + 1) * P // world
    local_rows = O.partition(x_local.shape[0], cfg.row_block_rows) if x_local.shape[0] else []
    assert len(local_rows) == last - first
    items = [[_owner(s, P, world), None] for s in range(P)]
    for j, (s0, cnt) in enumerate(local_rows):
        xj = x_local[s0:s0 + cnt]
        um = O.svd_of_col_slices(xj, cfg.col_block_cols, cfg.gamma, cfg.max_rank)
        rec = O.full_svd(um.u.T @ xj)
        rec.u = None
        items[first + j][1] = O.truncate_factor(rec, cfg.gamma, cfg.max_rank)
    while len(items) > 1:
        nxt = []
        for i in range(0, len(items) - 1, 2):
            (oa, fa), (ob, fb) = items[i], items[i + 1]
            res = None
            if oa == rank and ob == rank:
                res = O.merge_pair_qr(fa, fb, O.ROW_CONCAT, cfg.gamma, cfg.max_rank)
            elif oa == rank:
                sig = _recv_arr(dist, torch, ob, 1)
                v = _recv_arr(dist, torch, ob, 2)
                res = O.merge_pair_qr(fa, O.SvdFactor(None, sig, v), O.ROW_CONCAT, cfg.gamma,
                                      cfg.max_rank)
            elif ob == rank:
                _send_arr(dist, torch, fb.sigma, oa)
                _send_arr(dist, torch, fb.v, oa)
            nxt.append([oa, res])
        if len(items) % 2:
            nxt.append(items[-1])
        items = nxt
    root, fin = items[0]
    shp = torch.tensor(list(fin.v.shape) if rank == root else [0, 0], dtype=torch.int64)
    dist.broadcast(shp, root)
    vr = torch.from_numpy(fin.v.copy()) if rank == root else torch.zeros(tuple(shp.tolist()),
                                                                          dtype=torch.float64)
    dist.broadcast(vr, root)
    vr = vr.numpy()
    y = x_local.astype(np.float64) @ vr
    g = torch.from_numpy(y.T @ y)
    dist.all_reduce(g)
    lam, z = np.linalg.eigh(g.numpy())
    z = z[:, ::-1]
    yh = y @ z
    nrm = torch.from_numpy((yh * yh).sum(axis=0))
    dist.all_reduce(nrm)
    sig = np.sqrt(nrm.numpy())
    order = np.argsort(-sig, kind="stable")
    sig = sig[order]
    return O.SvdFactor(yh[:, order] / sig, sig, vr @ z[:, order])


def _worker(rank, world, port, m, n, P, Q, k, out_q):
    import torch.distributed as dist
    import paper_1710_02812_b200 as H
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    rng = np.random.default_rng(7)
    x = (np.linalg.qr(rng.standard_normal((m, 12)))[0] * np.exp(-0.3 * np.arange(12))) @ \
        np.linalg.qr(rng.standard_normal((n, 12)))[0].T + 1e-3 * rng.standard_normal((m, n))
    cfg = O.MatConfig(gamma=1e-12, row_block_rows=m // P, col_block_cols=n // Q, max_rank=k)
    row0, ml = H.shard_rows(m, cfg.row_block_rows, rank, world)
    got = sharded_oracle(x[row0:row0 + ml], m, cfg, rank, world)
    out_q.put((rank, row0, ml, got.sigma, got.v, got.u))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,P", [(2, 4), (3, 8), (2, 3)])
def test_sharded_schedule_matches_single_process(world, P):
    import torch.multiprocessing as mp
    m, n, Q, k = 240, 48, 2, 10
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, n, P, Q, k, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(7)
    x = (np.linalg.qr(rng.standard_normal((m, 12)))[0] * np.exp(-0.3 * np.arange(12))) @ \
        np.linalg.qr(rng.standard_normal((n, 12)))[0].T + 1e-3 * rng.standard_normal((m, n))
    cfg = O.MatConfig(gamma=1e-12, row_block_rows=m // P, col_block_cols=n // Q, max_rank=k)
    ref_r = O.hierarchical_svd(x, cfg)
    ref = O.recover_left_vectors(x, ref_r.v)
    u = np.vstack([r[5] for r in res])
    assert sum(r[2] for r in res) == m
    for _rank, _r0, _ml, sig, v, _u in res:
        assert np.abs(sig - ref.sigma).max() <= 1e-12 * ref.sigma[0]
        assert O.largest_principal_angle(ref.v, v) < 1e-10
    assert O.largest_principal_angle(ref.u, u) < 1e-10
    assert O.orthonormality_defect(u) < 1e-10
