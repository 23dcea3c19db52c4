// Multi-GPU rank-k HSVD: contiguous row slices per rank, no
// data-path collective until the row-phase tree.  Only rank-k factors move:
//   * leaves, column merges and V-recovery are rank-local;
//   * the row-phase tree keeps the reference pairing (0,1),(2,3),... with an
//     odd factor carried (hierarchy.cpp:37-46): a cross-rank pair ships the
//     right factor (sigma, V: n x r) to the left factor's owner;
//   * V_r is broadcast from rank 0; U-recovery all-reduces the r x r Gram of
//     Y = X V_r and the squared column norms of Y Z, so U stays row-sharded.
#include <algorithm>
#include <cstring>
#include <string>

#include "comm.h"
#include "engine.h"
#include "factor_ops.h"
#include "syev.h"

namespace hsvdcu {

void shard_rows(long long m_total, long long d, int rank, int world, long long* row0,
                long long* m_local, int* first_slice, int* last_slice) {
  auto rows = partition(m_total, d);
  const int P = static_cast<int>(rows.size());
  const int first = static_cast<int>((long long)rank * P / world);
  const int last = static_cast<int>((long long)(rank + 1) * P / world);
  long long r0 = first < P ? rows[first].start : m_total, cnt = 0;
  for (int s = first; s < last; ++s) cnt += rows[s].count;
  if (row0) *row0 = r0;
  if (m_local) *m_local = cnt;
  if (first_slice) *first_slice = first;
  if (last_slice) *last_slice = last;
}

namespace {

int owner_of(int slice, int P, int world) {
  // inverse of shard_rows' floor(rank*P/world) split
  for (int g = 0; g < world; ++g)
    if ((long long)(g + 1) * P / world > slice) return g;
  return world - 1;
}

struct Item {
  int owner;
  DFac f;  // valid when owner == me
};

}  // namespace

DFac rank_k_svd_sharded(Ctx& ctx, Comm& comm, const XView& xl, long long m_total, long long row0,
                        const HsvdConfig& cfg) {
  const int me = comm.rank(), world = comm.size();
  const int n = static_cast<int>(xl.n);
  long long exp_row0 = 0, exp_m = 0;
  int first = 0, last = 0;
  shard_rows(m_total, cfg.d, me, world, &exp_row0, &exp_m, &first, &last);
  if (xl.m != exp_m || (exp_m > 0 && row0 != exp_row0))
    throw Error(kInvalid, "sharded: rank " + std::to_string(me) + " must hold rows [" +
                              std::to_string(exp_row0) + ", " + std::to_string(exp_row0 + exp_m) +
                              ")");
  const int P = static_cast<int>(partition(m_total, cfg.d).size());
  const long long d_eff = (cfg.d < 1 || cfg.d > m_total) ? m_total : cfg.d;

  // 1. rank-local: leaves, column merges, V-recovery of the owned slices
  std::vector<Item> items(P);
  for (int s = 0; s < P; ++s) items[s].owner = owner_of(s, P, world);
  if (exp_m > 0) {
    auto rows = partition(xl.m, d_eff);
    auto cols = partition(xl.n, cfg.c);
    const int Pl = static_cast<int>(rows.size()), Q = static_cast<int>(cols.size());
    if (Pl != last - first) throw Error(kInvalid, "sharded: local slices do not match the plan");
    std::vector<Block> blocks;
    for (int j = 0; j < Pl; ++j)
      for (int i = 0; i < Q; ++i)
        blocks.push_back({rows[j].start, (int)rows[j].count, cols[i].start, (int)cols[i].count});
    std::vector<DFac> leaves = block_svd_batch(ctx, xl, blocks, cfg.gamma, cfg.cap, false, false);
    std::vector<std::vector<DFac>> trees(Pl);
    for (int j = 0; j < Pl; ++j)
      trees[j].assign(leaves.begin() + j * Q, leaves.begin() + (j + 1) * Q);
    std::vector<DFac> us = tree_merge_many(ctx, trees, cfg.gamma, cfg.cap, nullptr);
    // V-recovery: reuse the single-GPU path on the local rows
    std::vector<DFac> vs = vrecover_batch(ctx, xl, rows, us, cfg.gamma, cfg.cap);
    for (int j = 0; j < Pl; ++j) items[first + j].f = vs[j];
  }

  // 2. row-phase tree across ranks, reference pairing
  double* hdr_send = ctx.arena.alloc_n<double>(std::max(P, 1));
  double* hdr_recv = ctx.arena.alloc_n<double>(std::max(P, 1));
  std::vector<Item> cur = items;
  while (cur.size() > 1) {
    std::vector<Item> nxt;
    std::vector<std::pair<DFac, DFac>> local_pairs;
    std::vector<size_t> local_pos;
    struct X {
      size_t pos;
      int peer;
      DFac f;
    };
    std::vector<X> sends, recvs;
    for (size_t i = 0; i + 1 < cur.size(); i += 2) {
      const Item& a = cur[i];
      const Item& b = cur[i + 1];
      Item r;
      r.owner = a.owner;
      const size_t pos = nxt.size();
      nxt.push_back(r);
      if (a.owner == me && b.owner == me) {
        local_pairs.push_back({a.f, b.f});
        local_pos.push_back(pos);
      } else if (a.owner == me) {
        recvs.push_back({pos, b.owner, a.f});
      } else if (b.owner == me) {
        sends.push_back({pos, a.owner, b.f});
      }
    }
    if (cur.size() % 2 == 1) nxt.push_back(cur.back());
    // headers (rank of the shipped factor), then payloads (sigma, V)
    if (!sends.empty() || !recvs.empty()) {
      std::vector<double> hv(sends.size());
      for (size_t i = 0; i < sends.size(); ++i) hv[i] = sends[i].f.rank;
      if (!hv.empty())
        HSVD_CUDA(cudaMemcpyAsync(hdr_send, hv.data(), hv.size() * sizeof(double),
                                  cudaMemcpyHostToDevice, ctx.stream));
    }
    comm.group_start();
    for (size_t i = 0; i < sends.size(); ++i) comm.send(ctx, hdr_send + i, sizeof(double), sends[i].peer);
    for (size_t i = 0; i < recvs.size(); ++i) comm.recv(ctx, hdr_recv + i, sizeof(double), recvs[i].peer);
    comm.group_end();
    std::vector<double> rh(recvs.size());
    if (!recvs.empty()) {
      HSVD_CUDA(cudaMemcpyAsync(rh.data(), hdr_recv, rh.size() * sizeof(double),
                                cudaMemcpyDeviceToHost, ctx.stream));
    }
    HSVD_CUDA(cudaStreamSynchronize(ctx.stream));
    std::vector<DFac> incoming(recvs.size());
    for (size_t i = 0; i < recvs.size(); ++i) {
      DFac& f = incoming[i];
      f.rank = static_cast<int>(rh[i]);
      f.dim = n;
      f.ld = n;
      f.sigma = ctx.arena.alloc_n<double>(f.rank);
      f.B = ctx.arena.alloc_n<double>((size_t)n * f.rank);
    }
    comm.group_start();
    for (auto& s : sends) {
      if (s.f.ld != n) throw Error(kInvalid, "sharded: V factor must be contiguous");
      comm.send(ctx, s.f.sigma, s.f.rank * sizeof(double), s.peer);
      comm.send(ctx, s.f.B, (size_t)n * s.f.rank * sizeof(double), s.peer);
    }
    for (size_t i = 0; i < recvs.size(); ++i) {
      comm.recv(ctx, incoming[i].sigma, incoming[i].rank * sizeof(double), recvs[i].peer);
      comm.recv(ctx, incoming[i].B, (size_t)n * incoming[i].rank * sizeof(double), recvs[i].peer);
    }
    comm.group_end();
    for (size_t i = 0; i < recvs.size(); ++i) {
      local_pairs.push_back({recvs[i].f, incoming[i]});
      local_pos.push_back(recvs[i].pos);
    }
    if (!local_pairs.empty()) {
      ctx.phase = "merge.row";
      std::vector<DFac> merged = merge_batch(ctx, local_pairs, cfg.gamma, cfg.cap);
      for (size_t i = 0; i < merged.size(); ++i) nxt[local_pos[i]].f = merged[i];
    }
    cur.swap(nxt);
  }

  // 3. broadcast V_r from its owner (the owner of slice 0 is rank 0)
  const int root = cur[0].owner;
  double* hb = ctx.arena.alloc_n<double>(1);
  if (me == root) {
    const double rr = cur[0].f.rank;
    HSVD_CUDA(cudaMemcpyAsync(hb, &rr, sizeof(double), cudaMemcpyHostToDevice, ctx.stream));
  }
  comm.bcast(ctx, hb, sizeof(double), root);
  double hr = 0.0;
  HSVD_CUDA(cudaMemcpyAsync(&hr, hb, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
  HSVD_CUDA(cudaStreamSynchronize(ctx.stream));
  const int r = static_cast<int>(hr);
  double* vr = (me == root) ? reorthonormalize(ctx, cur[0].f.B, cur[0].f.ld, n, r)
                            : ctx.arena.alloc_n<double>((size_t)n * r);
  comm.bcast(ctx, vr, (size_t)n * r * sizeof(double), root);

  // 4. U-recovery with all-reduced Gram and column norms (hierarchy.cpp:96-112)
  const int ml = static_cast<int>(exp_m);
  const int kk = static_cast<int>(std::min<long long>(r, m_total));
  double* H = ctx.arena.alloc_n<double>((size_t)r * r);
  double* dd = ctx.arena.alloc_n<double>(1);
  ctx.phase = "urec.check";
  gemm_grouped(ctx, DType::F64, DType::F64, true, false, true, {{vr, vr, H, n, n, r, r, r, n, 1.0, 0.0}});
  ortho_defect(ctx, H, r, r, dd);
  double hdv = 0.0;
  HSVD_CUDA(cudaMemcpyAsync(&hdv, dd, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
  HSVD_CUDA(cudaStreamSynchronize(ctx.stream));
  if (!(hdv <= 1e-6)) throw Error(kInvalid, "recover_left_vectors: v_r columns are not orthonormal");
  double* Y = ctx.arena.alloc_n<double>((size_t)std::max(ml, 1) * r);
  double* lam = ctx.arena.alloc_n<double>(kk);
  double* Z = ctx.arena.alloc_n<double>((size_t)r * kk);
  double* Yh = ctx.arena.alloc_n<double>((size_t)std::max(ml, 1) * kk);
  double* U = ctx.arena.alloc_n<double>((size_t)std::max(ml, 1) * kk);
  double* nrm = ctx.arena.alloc_n<double>(kk);
  double* sig = ctx.arena.alloc_n<double>(kk);
  int* perm = ctx.arena.alloc_n<int>(kk);
  double* Zp = ctx.arena.alloc_n<double>((size_t)r * kk);
  double* V = ctx.arena.alloc_n<double>((size_t)n * kk);
  int* d_rd = ctx.arena.alloc_n<int>(2);
  ctx.phase = "urec.proj";
  if (ml > 0) {
    project_x(ctx, xl.dt, true, {{xl.X, vr, Y, xl.ld, n, ml, ml, r, n, 1.0, 0.0}});
    ctx.phase = "urec.gram";
    gemm_grouped(ctx, DType::F64, DType::F64, true, false, true, {{Y, Y, H, ml, ml, r, r, r, ml, 1.0, 0.0}});
  } else {
    HSVD_CUDA(cudaMemsetAsync(H, 0, (size_t)r * r * sizeof(double), ctx.stream));
  }
  comm.allreduce_sum(ctx, H, (size_t)r * r);
  ctx.phase = "urec.eig";
  eig_topk(ctx, {{H, r, r, kk, lam, Z, r}});
  ctx.phase = "urec.back";
  if (ml > 0) {
    gemm_grouped(ctx, DType::F64, DType::F64, false, false, false, {{Y, Z, Yh, ml, r, ml, ml, kk, r, 1.0, 0.0}});
    colnorms2(ctx, Yh, ml, ml, kk, nrm);
  } else {
    HSVD_CUDA(cudaMemsetAsync(nrm, 0, kk * sizeof(double), ctx.stream));
  }
  comm.allreduce_sum(ctx, nrm, kk);
  ctx.phase = "urec.fin";
  FinJob fj{Yh, std::max(ml, 1), ml, kk, 0.0, 0, U, std::max(ml, 1), sig, perm, d_rd, d_rd + 1, 1};
  fj.norms2 = nrm;
  finalize(ctx, {fj});
  gather_cols(ctx, {{Zp, r, Z, r, r, kk, perm}});
  gemm_grouped(ctx, DType::F64, DType::F64, false, false, false, {{vr, Zp, V, n, r, n, n, kk, r, 1.0, 0.0}});
  std::vector<int> rd;
  fetch_ranks(ctx, d_rd, 2, rd);
  if (rd[1] == 2)
    throw Error(kDecomposition, "SVD did not converge for a " + std::to_string(m_total) + "x" +
                                    std::to_string(r) + " matrix", m_total, r);
  // U orthonormal to eps: C = sum over ranks of U_g^T U_g = R^T R, U_g <- U_g R^{-1}
  double* C = ctx.arena.alloc_n<double>((size_t)kk * kk);
  double* Ri = ctx.arena.alloc_n<double>((size_t)kk * kk);
  double* U2 = ctx.arena.alloc_n<double>((size_t)std::max(ml, 1) * kk);
  ctx.phase = "reorth";
  if (ml > 0)
    gemm_grouped(ctx, DType::F64, DType::F64, true, false, true, {{U, U, C, ml, ml, kk, kk, kk, ml, 1.0, 0.0}});
  else
    HSVD_CUDA(cudaMemsetAsync(C, 0, (size_t)kk * kk * sizeof(double), ctx.stream));
  comm.allreduce_sum(ctx, C, (size_t)kk * kk);
  chol_inverse(ctx, C, kk, Ri);
  if (ml > 0)
    gemm_grouped(ctx, DType::F64, DType::F64, false, false, false, {{U, Ri, U2, ml, kk, ml, ml, kk, kk, 1.0, 0.0}});
  DFac f;
  f.B = U2;
  f.ld = std::max(ml, 1);
  f.dim = ml;
  f.rank = kk;
  f.sigma = sig;
  f.degenerate = rd[1] == 1;
  f.B2 = V;
  f.ld2 = n;
  f.dim2 = n;
  return f;
}

}  // namespace hsvdcu
