// Host orchestration of Algorithm 1 (hierarchical merge-and-truncate SVD) on
// device-resident data.  Mirrors /root/reference/proj/core/src/hierarchy.cpp
// and merge.cpp; every dense step is one batched launch across all blocks /
// pairs / row slices of a tree level.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <string>

#include "engine.h"
#include "jacobi.h"
#include "ozaki.h"
#include "factor_ops.h"
#include "syev.h"

namespace hsvdcu {

namespace {

size_t esize(DType t) { return t == DType::F32 ? 4 : 8; }

const void* xptr(const XView& x, long long r0, long long c0) {
  return static_cast<const char*>(x.X) + (r0 * x.ld + c0) * (long long)esize(x.dt);
}

void check_decomp(const std::vector<int>& deg, const std::vector<std::pair<long long, long long>>& dims,
                  const std::string& prefix) {
  for (size_t i = 0; i < deg.size(); ++i)
    if (deg[i] == 2)
      throw Error(kDecomposition,
                  prefix + "SVD did not converge for a " + std::to_string(dims[i].first) + "x" +
                      std::to_string(dims[i].second) + " matrix",
                  dims[i].first, dims[i].second);
}

}  // namespace

// B (rows x k) nearly orthonormal -> B R^{-1} with B^T B = R^T R.
double* reorthonormalize(Ctx& ctx, const double* B, long long ld, int rows, int k) {
  const char* ph = ctx.phase;
  ctx.phase = "reorth";
  double* C = ctx.arena.alloc_n<double>((size_t)k * k);
  double* Ri = ctx.arena.alloc_n<double>((size_t)k * k);
  double* out = ctx.arena.alloc_n<double>((size_t)rows * k);
  gemm_grouped(ctx, DType::F64, DType::F64, true, false, true, {{B, B, C, ld, ld, k, k, k, rows, 1.0, 0.0}});
  chol_inverse(ctx, C, k, Ri);
  gemm_grouped(ctx, DType::F64, DType::F64, false, false, false,
               {{B, Ri, out, ld, k, rows, rows, k, k, 1.0, 0.0}});
  ctx.phase = ph;
  return out;
}

std::vector<Slice> partition(long long extent, long long block) {
  if (block < 1 || block > extent) block = extent;
  std::vector<Slice> out;
  for (long long s = 0; s < extent; s += block) out.push_back({s, std::min(block, extent - s)});
  return out;
}

void fetch_ranks(Ctx& ctx, const int* d_ranks, int count, std::vector<int>& out) {
  out.assign(count, 0);
  if (count == 0) return;
  int* h = ctx.pinned_ints(count);
  HSVD_CUDA(cudaMemcpyAsync(h, d_ranks, count * sizeof(int), cudaMemcpyDeviceToHost, ctx.stream));
  if (Ctx::trace()) std::fprintf(stderr, "[r%d] fetch_ranks sync\n", ctx.rank);
  HSVD_CUDA(cudaStreamSynchronize(ctx.stream));
  if (Ctx::trace()) std::fprintf(stderr, "[r%d] fetch_ranks done\n", ctx.rank);
  std::memcpy(out.data(), h, count * sizeof(int));
}

void x_wait_chunk(Ctx& ctx, const XView& x, size_t i) {
  if (x.stager) x.stager->wait_issued(i);
  HSVD_CUDA(cudaStreamWaitEvent(ctx.stream, x.ready[i].ev, 0));
}

void x_wait_rows(Ctx& ctx, const XView& x, long long row_end) {
  long long prev = 0;
  for (size_t i = 0; i < x.ready.size(); ++i) {
    if (row_end >= 0 && prev >= row_end) break;
    x_wait_chunk(ctx, x, i);
    prev = x.ready[i].row_end;
  }
}

// Leaf Grams G = Xt Xt^T of tall blocks: fp32 blocks on the tcgen05 int8
// tensor cores (Ozaki slices, fp64-grade; ozaki_gram.cu), fp64 blocks (and
// HSVD_GRAM=dmma) on the fp64 DMMA SYRK.
void leaf_gram_tall(Ctx& ctx, DType dt, const std::vector<GemmDesc>& descs) {
  std::vector<GemmDesc> oz, dm;
  for (const GemmDesc& g : descs) (ozaki_gram_applicable(dt, g) ? oz : dm).push_back(g);
  ozaki_gram_batch(ctx, oz);
  gemm_grouped(ctx, dt, dt, false, true, true, dm);
}

// Projections of the fp32 input onto fp64 factors (leaf P = X_b Z, V-recovery
// X_j^T U_j, U-recovery X V_r, refinement X^T U): on the tcgen05 int8 tensor
// cores through the Ozaki planes (fp64-grade; ozaki_gram.cu) when they fit
// (N <= 256, K <= 65536), else -- and for fp64 inputs, or HSVD_PROJ=dmma --
// the DMMA GEMM.
void project_x(Ctx& ctx, DType xt, bool trans_a, const std::vector<GemmDesc>& descs) {
  std::vector<GemmDesc> oz, dm;
  for (const GemmDesc& d : descs) (ozaki_gemm_applicable(xt, trans_a, d) ? oz : dm).push_back(d);
  ozaki_gemm_batch(ctx, trans_a, oz);
  gemm_grouped(ctx, xt, DType::F64, trans_a, false, false, dm);
}

// ---------------------------------------------------------------------------
// block SVD (leaves): Gram of the smaller side + top-k eigenpairs + projection
// ---------------------------------------------------------------------------
std::vector<DFac> block_svd_batch(Ctx& ctx, const XView& x, const std::vector<Block>& blocks,
                                  double gamma, int cap, bool keep_both, bool write_all) {
  const int nb = static_cast<int>(blocks.size());
  std::vector<DFac> out(nb);
  if (nb == 0) return out;
  struct Tmp {
    bool tall, jac;
    int q, kk, s;
    double *G, *lam, *Z, *P, *Bp, *sig;
    int* perm;
  };
  std::vector<Tmp> t(nb);
  std::vector<GemmDesc> gram_t, gram_w, proj_t, proj_w;
  std::vector<EigJob> ej;
  std::vector<JacJob> jj;
  int* d_rd = ctx.arena.alloc_n<int>(2 * (size_t)nb);
  for (int b = 0; b < nb; ++b) {
    const Block& bl = blocks[b];
    Tmp& m = t[b];
    m.tall = bl.d >= bl.c;
    m.q = m.tall ? bl.c : bl.d;
    const int p = std::min(bl.d, bl.c);
    m.kk = cap > 0 ? std::min(cap, p) : p;
    m.s = m.tall ? bl.d : bl.c;
    // kernels.cpp:28: the smaller side <= 32 -> one-sided Jacobi on the block
    // itself (all q columns, ordered by norm; the cap is finalize's)
    m.jac = small_svd_jacobi(m.s, m.q);
    m.Bp = ctx.arena.alloc_n<double>((size_t)m.s * m.kk);
    m.sig = ctx.arena.alloc_n<double>(m.kk);
    m.perm = ctx.arena.alloc_n<int>(m.kk);
    const void* base = xptr(x, bl.r0, bl.c0);
    if (m.jac) {
      m.G = m.lam = nullptr;
      m.Z = ctx.arena.alloc_n<double>((size_t)m.q * m.q);
      m.P = ctx.arena.alloc_n<double>((size_t)m.s * m.q);
      const int f64 = x.dt == DType::F64 ? 1 : 0;
      if (m.tall)  // columns of the block: (i, j) at base + i*ld + j
        jj.push_back({base, f64, x.ld, 1, m.q, nullptr, nullptr, 0, 0, nullptr, m.s, nullptr,
                      m.P, m.s, m.Z, m.q});
      else  // columns of the block's transpose: (i, j) at base + j*ld + i
        jj.push_back({base, f64, 1, x.ld, m.q, nullptr, nullptr, 0, 0, nullptr, m.s, nullptr,
                      m.P, m.s, m.Z, m.q});
      continue;
    }
    m.G = ctx.arena.alloc_n<double>((size_t)m.q * m.q);
    m.lam = ctx.arena.alloc_n<double>(m.kk);
    m.Z = ctx.arena.alloc_n<double>((size_t)m.q * m.kk);
    m.P = ctx.arena.alloc_n<double>((size_t)m.s * m.kk);
    // column-major view of the row-major block: Xt (c x d, ld = x.ld)
    if (m.tall)  // G = X_b^T X_b = Xt Xt^T
      gram_t.push_back({base, base, m.G, x.ld, x.ld, m.q, m.q, m.q, bl.d, 1.0, 0.0});
    else  // G = X_b X_b^T = Xt^T Xt
      gram_w.push_back({base, base, m.G, x.ld, x.ld, m.q, m.q, m.q, bl.c, 1.0, 0.0});
    ej.push_back({m.G, m.q, m.q, m.kk, m.lam, m.Z, m.q});
    if (m.tall)  // P = X_b Z = Xt^T Z  (d x kk)
      proj_t.push_back({base, m.Z, m.P, x.ld, m.q, m.s, bl.d, m.kk, bl.c, 1.0, 0.0});
    else  // P = X_b^T Z = Xt Z  (c x kk)
      proj_w.push_back({base, m.Z, m.P, x.ld, m.q, m.s, bl.c, m.kk, bl.d, 1.0, 0.0});
  }
  ctx.phase = "leaf.gram";
  if (x.ready.empty()) {
    leaf_gram_tall(ctx, x.dt, gram_t);
    gemm_grouped(ctx, x.dt, x.dt, true, false, true, gram_w);
  } else {
    // input still arriving: one Gram launch per row-chunk group of blocks,
    // each after its rows' copy (the copies overlap the earlier Grams)
    // (the copy stream is in order: chunk c done implies every earlier one)
    std::vector<GemmDesc> gt, gw;
    long long prev = 0;
    for (size_t ci = 0; ci < x.ready.size(); ++ci) {
      const RowChunk& c = x.ready[ci];
      gt.clear();
      gw.clear();
      size_t it = 0, iw = 0;
      for (int b = 0; b < nb; ++b) {
        if (t[b].jac) continue;
        const bool tall = t[b].tall;
        const GemmDesc& gd = tall ? gram_t[it++] : gram_w[iw++];
        const Block& bl = blocks[b];
        if (bl.r0 + bl.d <= prev || bl.r0 + bl.d > c.row_end) continue;
        (tall ? gt : gw).push_back(gd);
      }
      if (gt.empty() && gw.empty()) continue;  // no block ends in this chunk
      x_wait_chunk(ctx, x, ci);
      leaf_gram_tall(ctx, x.dt, gt);
      gemm_grouped(ctx, x.dt, x.dt, true, false, true, gw);
      prev = c.row_end;
    }
    long long row_end = 0;  // everything after reads any row of these blocks
    for (const Block& bl : blocks) row_end = std::max<long long>(row_end, bl.r0 + bl.d);
    x_wait_rows(ctx, x, row_end);
  }
  ctx.phase = "leaf.eig";
  eig_topk(ctx, ej);
  ctx.phase = "leaf.proj";
  project_x(ctx, x.dt, true, proj_t);
  project_x(ctx, x.dt, false, proj_w);
  ctx.phase = "leaf.jacobi";
  jacobi_svd_batch(ctx, jj);
  ctx.phase = "leaf.fin";
  // the projected side is written (and its null directions completed) for
  // the retained columns only, unless the caller keeps it whole (full_svd:
  // write_all / keep_both); a wide block's factor basis is the gathered
  // eigenvector side, whose permutation covers all kk columns
  std::vector<FinJob> fj;
  for (int b = 0; b < nb; ++b) {
    Tmp& m = t[b];
    fj.push_back({m.P, m.s, m.s, m.kk, gamma, cap, m.Bp, m.s, m.sig, m.perm, d_rd + b,
                  d_rd + nb + b, (write_all || keep_both) ? 1 : 0});
  }
  finalize(ctx, fj);
  // the eigenvector side, permuted to the sigma order
  std::vector<GatherJob> gj;
  std::vector<double*> zside(nb, nullptr);
  for (int b = 0; b < nb; ++b) {
    Tmp& m = t[b];
    if (!m.tall || keep_both) {
      zside[b] = ctx.arena.alloc_n<double>((size_t)m.q * m.kk);
      gj.push_back({zside[b], m.q, m.Z, m.q, m.q, m.kk, m.perm});
    }
  }
  gather_cols(ctx, gj);
  std::vector<int> rd;
  fetch_ranks(ctx, d_rd, 2 * nb, rd);
  std::vector<int> deg(rd.begin() + nb, rd.end());
  std::vector<std::pair<long long, long long>> dims;
  for (auto& bl : blocks) dims.push_back({bl.d, bl.c});
  check_decomp(deg, dims, "");
  for (int b = 0; b < nb; ++b) {
    Tmp& m = t[b];
    DFac& f = out[b];
    f.rank = rd[b];
    f.degenerate = deg[b] == 1;
    f.sigma = m.sig;
    if (m.tall) {
      f.B = m.Bp;
      f.ld = m.s;
      f.dim = blocks[b].d;
      if (keep_both) {
        f.B2 = zside[b];
        f.ld2 = m.q;
        f.dim2 = blocks[b].c;
      }
    } else {
      f.B = zside[b];
      f.ld = m.q;
      f.dim = blocks[b].d;
      if (keep_both) {
        f.B2 = m.Bp;
        f.ld2 = m.s;
        f.dim2 = blocks[b].c;
      }
    }
  }
  return out;
}

// ---------------------------------------------------------------------------
// merge (Gram form of merge_pair_qr / merge_pair_naive)
// ---------------------------------------------------------------------------
std::vector<DFac> merge_batch(Ctx& ctx, const std::vector<std::pair<DFac, DFac>>& pairs,
                              double gamma, int cap) {
  const int np = static_cast<int>(pairs.size());
  std::vector<DFac> out(np);
  if (np == 0) return out;
  struct Tmp {
    int s, k1, k2, q, kk;
    double *G, *w, *lam, *Z, *Zh, *P, *Bn, *sig;
  };
  std::vector<Tmp> t(np);
  std::vector<GemmDesc> gsy, gx, p1, p2;
  std::vector<EigJob> ej;
  std::vector<JacJob> jj;
  std::vector<ScaleSymJob> ss;
  std::vector<ScaleRowsJob> sr;
  int* d_rd = ctx.arena.alloc_n<int>(2 * (size_t)np);
  for (int i = 0; i < np; ++i) {
    const DFac& a = pairs[i].first;
    const DFac& b = pairs[i].second;
    if (a.dim != b.dim) throw Error(kInvalid, "merge: factors must share the basis dimension");
    Tmp& m = t[i];
    m.s = a.dim;
    m.k1 = a.rank;
    m.k2 = b.rank;
    m.q = m.k1 + m.k2;
    m.kk = std::min(m.q, m.s);
    if (cap > 0) m.kk = std::min(m.kk, cap);
    m.Bn = ctx.arena.alloc_n<double>((size_t)m.s * m.kk);
    m.sig = ctx.arena.alloc_n<double>(m.kk);
    if (small_svd_jacobi(m.s, m.q)) {
      // SVD of [B1 S1 | B2 S2] by one-sided Jacobi (k + l <= 32: the
      // reference's full_svd of E / of the concatenation goes to JacobiSVD)
      m.G = m.w = m.lam = m.Zh = nullptr;
      m.Z = ctx.arena.alloc_n<double>((size_t)m.q * m.q);
      m.P = ctx.arena.alloc_n<double>((size_t)m.s * m.q);
      jj.push_back({a.B, 1, 1, a.ld, m.k1, a.sigma, b.B, b.ld, m.k2, b.sigma, m.s, nullptr, m.P,
                    m.s, m.Z, m.q});
      continue;
    }
    m.G = ctx.arena.alloc_n<double>((size_t)m.q * m.q);
    m.w = ctx.arena.alloc_n<double>(m.q);
    m.lam = ctx.arena.alloc_n<double>(m.kk);
    m.Z = ctx.arena.alloc_n<double>((size_t)m.q * m.kk);
    m.Zh = ctx.arena.alloc_n<double>((size_t)m.q * m.kk);
    m.P = ctx.arena.alloc_n<double>((size_t)m.s * m.kk);
    HSVD_CUDA(cudaMemcpyAsync(m.w, a.sigma, m.k1 * sizeof(double), cudaMemcpyDeviceToDevice,
                              ctx.stream));
    HSVD_CUDA(cudaMemcpyAsync(m.w + m.k1, b.sigma, m.k2 * sizeof(double),
                              cudaMemcpyDeviceToDevice, ctx.stream));
    // Gram of [B1 | B2]
    gsy.push_back({a.B, a.B, m.G, a.ld, a.ld, m.q, m.k1, m.k1, m.s, 1.0, 0.0});
    gsy.push_back({b.B, b.B, m.G + m.k1 + (long long)m.k1 * m.q, b.ld, b.ld, m.q, m.k2, m.k2,
                   m.s, 1.0, 0.0});
    gx.push_back({a.B, b.B, m.G + (long long)m.k1 * m.q, a.ld, b.ld, m.q, m.k1, m.k2, m.s, 1.0,
                  0.0});
    gx.push_back({b.B, a.B, m.G + m.k1, b.ld, a.ld, m.q, m.k2, m.k1, m.s, 1.0, 0.0});
    ss.push_back({m.G, m.q, m.q, m.w});
    ej.push_back({m.G, m.q, m.q, m.kk, m.lam, m.Z, m.q});
    sr.push_back({m.Zh, m.q, m.Z, m.q, m.q, m.kk, m.w});
    // P = B1 (S1 Z1) + B2 (S2 Z2)
    p1.push_back({a.B, m.Zh, m.P, a.ld, m.q, m.s, m.s, m.kk, m.k1, 1.0, 0.0});
    p2.push_back({b.B, m.Zh + m.k1, m.P, b.ld, m.q, m.s, m.s, m.kk, m.k2, 1.0, 1.0});
  }
  ctx.phase = "merge.gram";
  gemm_grouped(ctx, DType::F64, DType::F64, true, false, true, gsy);
  gemm_grouped(ctx, DType::F64, DType::F64, true, false, false, gx);
  scale_sym(ctx, ss);
  ctx.phase = "merge.eig";
  eig_topk(ctx, ej);
  ctx.phase = "merge.proj";
  scale_rows(ctx, sr);
  gemm_grouped(ctx, DType::F64, DType::F64, false, false, false, p1);
  gemm_grouped(ctx, DType::F64, DType::F64, false, false, false, p2);
  ctx.phase = "merge.jacobi";
  jacobi_svd_batch(ctx, jj);
  ctx.phase = "merge.fin";
  std::vector<FinJob> fj;
  for (int i = 0; i < np; ++i) {
    Tmp& m = t[i];
    fj.push_back({m.P, m.s, m.s, m.kk, gamma, cap, m.Bn, m.s, m.sig, nullptr, d_rd + i,
                  d_rd + np + i, 0});
  }
  finalize(ctx, fj);
  std::vector<int> rd;
  fetch_ranks(ctx, d_rd, 2 * np, rd);
  std::vector<int> deg(rd.begin() + np, rd.end());
  std::vector<std::pair<long long, long long>> dims;
  for (auto& m : t) dims.push_back({m.q, m.q});
  check_decomp(deg, dims, "");
  for (int i = 0; i < np; ++i) {
    DFac& f = out[i];
    f.B = t[i].Bn;
    f.ld = t[i].s;
    f.dim = t[i].s;
    f.rank = rd[i];
    f.sigma = t[i].sig;
    f.degenerate = deg[i] == 1;
  }
  return out;
}

std::vector<DFac> tree_merge_many(Ctx& ctx, std::vector<std::vector<DFac>> trees, double gamma,
                                  int cap, long long* pair_merges) {
  for (auto& tr : trees)
    if (tr.empty()) throw Error(kInvalid, "tree_merge: factor list is empty");
  while (true) {
    std::vector<std::pair<DFac, DFac>> pairs;
    for (auto& tr : trees)
      for (size_t i = 0; i + 1 < tr.size(); i += 2) pairs.push_back({tr[i], tr[i + 1]});
    if (pairs.empty()) break;
    std::vector<DFac> merged = merge_batch(ctx, pairs, gamma, cap);
    if (pair_merges) *pair_merges += (long long)pairs.size();
    size_t k = 0;
    for (auto& tr : trees) {
      std::vector<DFac> nxt;
      for (size_t i = 0; i + 1 < tr.size(); i += 2) nxt.push_back(merged[k++]);
      if (tr.size() % 2 == 1) nxt.push_back(tr.back());
      tr.swap(nxt);
    }
  }
  std::vector<DFac> out;
  for (auto& tr : trees) out.push_back(tr.front());
  return out;
}

// ---------------------------------------------------------------------------
// V-recovery of each row slice: SVD of U_j^T X_j through its k x k Gram
// ---------------------------------------------------------------------------
std::vector<DFac> vrecover_batch(Ctx& ctx, const XView& x, const std::vector<Slice>& rows,
                                        const std::vector<DFac>& us, double gamma, int cap) {
  const int ns = static_cast<int>(rows.size());
  std::vector<DFac> out(ns);
  struct Tmp {
    int r, kk;
    double *Bt, *H, *lam, *Z, *V, *Vn, *sig;
  };
  std::vector<Tmp> t(ns);
  const int n = static_cast<int>(x.n);
  std::vector<GemmDesc> g1, g2, g3;
  std::vector<EigJob> ej;
  std::vector<JacJob> jj;
  int* d_rd = ctx.arena.alloc_n<int>(2 * (size_t)ns);
  for (int j = 0; j < ns; ++j) {
    Tmp& m = t[j];
    const DFac& u = us[j];
    m.r = u.rank;
    m.kk = std::min(m.r, n);
    if (cap > 0) m.kk = std::min(m.kk, cap);
    m.Bt = ctx.arena.alloc_n<double>((size_t)n * m.r);
    m.Vn = ctx.arena.alloc_n<double>((size_t)n * m.kk);
    m.sig = ctx.arena.alloc_n<double>(m.kk);
    const void* base = xptr(x, rows[j].start, 0);
    // B^T = X_j^T U_j (n x r): Xt (n x d_j) * U_j
    g1.push_back({base, u.B, m.Bt, x.ld, u.ld, n, n, m.r, (int)rows[j].count, 1.0, 0.0});
    if (m.r <= n && small_svd_jacobi(n, m.r)) {  // kernels.cpp:28 on B (r x n, r <= 32)
      m.H = m.lam = nullptr;
      m.Z = ctx.arena.alloc_n<double>((size_t)m.r * m.r);
      m.V = ctx.arena.alloc_n<double>((size_t)n * m.r);
      jj.push_back({m.Bt, 1, 1, n, m.r, nullptr, nullptr, 0, 0, nullptr, n, nullptr, m.V, n, m.Z,
                    m.r});
      continue;
    }
    m.H = ctx.arena.alloc_n<double>((size_t)m.r * m.r);
    m.lam = ctx.arena.alloc_n<double>(m.kk);
    m.Z = ctx.arena.alloc_n<double>((size_t)m.r * m.kk);
    m.V = ctx.arena.alloc_n<double>((size_t)n * m.kk);
    g2.push_back({m.Bt, m.Bt, m.H, n, n, m.r, m.r, m.r, n, 1.0, 0.0});
    ej.push_back({m.H, m.r, m.r, m.kk, m.lam, m.Z, m.r});
    g3.push_back({m.Bt, m.Z, m.V, n, m.r, n, n, m.kk, m.r, 1.0, 0.0});
  }
  ctx.phase = "vrec.proj";
  project_x(ctx, x.dt, false, g1);
  ctx.phase = "vrec.gram";
  gemm_grouped(ctx, DType::F64, DType::F64, true, false, true, g2);
  ctx.phase = "vrec.eig";
  eig_topk(ctx, ej);
  ctx.phase = "vrec.back";
  gemm_grouped(ctx, DType::F64, DType::F64, false, false, false, g3);
  ctx.phase = "vrec.jacobi";
  jacobi_svd_batch(ctx, jj);
  ctx.phase = "vrec.fin";
  std::vector<FinJob> fj;
  for (int j = 0; j < ns; ++j) {
    Tmp& m = t[j];
    fj.push_back({m.V, n, n, m.kk, gamma, cap, m.Vn, n, m.sig, nullptr, d_rd + j, d_rd + ns + j, 0});
  }
  finalize(ctx, fj);
  std::vector<int> rd;
  fetch_ranks(ctx, d_rd, 2 * ns, rd);
  for (int j = 0; j < ns; ++j)
    if (rd[ns + j] == 2)
      throw Error(kDecomposition,
                  "row slice " + std::to_string(j) + ": SVD did not converge for a " +
                      std::to_string(t[j].r) + "x" + std::to_string(n) + " matrix",
                  t[j].r, n);
  for (int j = 0; j < ns; ++j) {
    DFac& f = out[j];
    f.B = t[j].Vn;
    f.ld = n;
    f.dim = n;
    f.rank = rd[j];
    f.sigma = t[j].sig;
    f.degenerate = rd[ns + j] == 1;
  }
  return out;
}

DFac svd_of_col_slices(Ctx& ctx, const XView& x, long long c, double gamma, int cap) {
  auto cols = partition(x.n, c);
  std::vector<Block> blocks;
  for (auto& cs : cols) blocks.push_back({0, (int)x.m, cs.start, (int)cs.count});
  std::vector<DFac> leaves = block_svd_batch(ctx, x, blocks, gamma, cap, false, false);
  return tree_merge_many(ctx, {leaves}, gamma, cap, nullptr).front();
}

// (Measured, round 2: running the leaves in two halves by row slices when
// the input arrives from the host, so the first half's eigensolver overlaps
// the second half's transfer, did not pay at config 5 -- e2e 2414 -> 2442 ms
// pinned: the second half's Grams, which overlapped the transfer before,
// then run alone.)

DFac hierarchical_svd(Ctx& ctx, const XView& x, const HsvdConfig& cfg) {
  auto rows = partition(x.m, cfg.d);
  auto cols = partition(x.n, cfg.c);
  const int P = static_cast<int>(rows.size()), Q = static_cast<int>(cols.size());
  std::vector<Block> blocks;
  for (int j = 0; j < P; ++j)
    for (int i = 0; i < Q; ++i)
      blocks.push_back({rows[j].start, (int)rows[j].count, cols[i].start, (int)cols[i].count});
  std::vector<DFac> leaves;
  try {
    leaves = block_svd_batch(ctx, x, blocks, cfg.gamma, cfg.cap, false, false);
  } catch (const Error& e) {
    if (e.code != kDecomposition) throw;
    for (int j = 0; j < P; ++j)  // attribute to the first failing slice
      if (e.rows <= rows[j].count)
        throw Error(kDecomposition, "row slice " + std::to_string(j) + ": " + e.what(), e.rows,
                    e.cols);
    throw;
  }
  std::vector<std::vector<DFac>> trees(P);
  for (int j = 0; j < P; ++j) trees[j].assign(leaves.begin() + j * Q, leaves.begin() + (j + 1) * Q);
  std::vector<DFac> us = tree_merge_many(ctx, trees, cfg.gamma, cfg.cap, nullptr);
  std::vector<DFac> vs = vrecover_batch(ctx, x, rows, us, cfg.gamma, cfg.cap);
  DFac root = tree_merge_many(ctx, {vs}, cfg.gamma, cfg.cap, nullptr).front();
  root.B = reorthonormalize(ctx, root.B, root.ld, root.dim, root.rank);
  root.ld = root.dim;
  return root;
}

DFac recover_left_vectors(Ctx& ctx, const XView& x, const double* v_r, long long ldv, int r) {
  const int m = static_cast<int>(x.m), n = static_cast<int>(x.n);
  if (r < 1) throw Error(kInvalid, "recover_left_vectors: v_r has no columns");
  double* H = ctx.arena.alloc_n<double>((size_t)r * r);
  double* dd = ctx.arena.alloc_n<double>(1);
  ctx.phase = "urec.check";
  gemm_grouped(ctx, DType::F64, DType::F64, true, false, true,
               {{v_r, v_r, H, ldv, ldv, r, r, r, n, 1.0, 0.0}});
  ortho_defect(ctx, H, r, r, dd);
  double* hd = ctx.pinned_dbl(1);
  HSVD_CUDA(cudaMemcpyAsync(hd, dd, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
  HSVD_CUDA(cudaStreamSynchronize(ctx.stream));
  if (!(hd[0] <= 1e-6))
    throw Error(kInvalid, "recover_left_vectors: v_r columns are not orthonormal");
  const int kk = std::min(r, m);
  double* Y = ctx.arena.alloc_n<double>((size_t)m * r);
  double* lam = ctx.arena.alloc_n<double>(kk);
  double* Z = ctx.arena.alloc_n<double>((size_t)r * kk);
  double* Yh = ctx.arena.alloc_n<double>((size_t)m * kk);
  double* U = ctx.arena.alloc_n<double>((size_t)m * kk);
  double* sig = ctx.arena.alloc_n<double>(kk);
  int* perm = ctx.arena.alloc_n<int>(kk);
  double* Zp = ctx.arena.alloc_n<double>((size_t)r * kk);
  double* V = ctx.arena.alloc_n<double>((size_t)n * kk);
  int* d_rd = ctx.arena.alloc_n<int>(2);
  // Y = X V_r : Xt (n x m) transposed
  ctx.phase = "urec.proj";
  project_x(ctx, x.dt, true, {{x.X, v_r, Y, x.ld, ldv, m, m, r, n, 1.0, 0.0}});
  if (kk == r && small_svd_jacobi(m, r)) {  // kernels.cpp:28: full_svd(Y), r <= 32
    ctx.phase = "urec.jacobi";
    std::vector<JacJob> jj{{Y, 1, 1, m, r, nullptr, nullptr, 0, 0, nullptr, m, nullptr, Yh, m, Z,
                            r}};
    jacobi_svd_batch(ctx, jj);
  } else {
    ctx.phase = "urec.gram";
    gemm_grouped(ctx, DType::F64, DType::F64, true, false, true,
                 {{Y, Y, H, m, m, r, r, r, m, 1.0, 0.0}});
    ctx.phase = "urec.eig";
    eig_topk(ctx, {{H, r, r, kk, lam, Z, r}});
    ctx.phase = "urec.back";
    gemm_grouped(ctx, DType::F64, DType::F64, false, false, false,
                 {{Y, Z, Yh, m, r, m, m, kk, r, 1.0, 0.0}});
  }
  ctx.phase = "urec.fin";
  finalize(ctx, {{Yh, m, m, kk, 0.0, 0, U, m, sig, perm, d_rd, d_rd + 1, 1}});
  gather_cols(ctx, {{Zp, r, Z, r, r, kk, perm}});
  gemm_grouped(ctx, DType::F64, DType::F64, false, false, false,
               {{v_r, Zp, V, ldv, r, n, n, kk, r, 1.0, 0.0}});
  std::vector<int> rd;
  fetch_ranks(ctx, d_rd, 2, rd);
  if (rd[1] == 2)
    throw Error(kDecomposition,
                "SVD did not converge for a " + std::to_string(m) + "x" + std::to_string(r) + " matrix",
                m, r);
  DFac f;
  f.B = reorthonormalize(ctx, U, m, m, kk);
  f.ld = m;
  f.dim = m;
  f.rank = kk;
  f.sigma = sig;
  f.degenerate = rd[1] == 1;
  f.B2 = V;
  f.ld2 = n;
  f.dim2 = n;
  return f;
}

// refine.cpp:26-72 (Alg. 2): alternate thin SVDs of X V (left basis kept,
// via recover_left_vectors) and of U_outer^T X (Gram of the r-side, eigen-
// pairs, V = (X^T U_outer) Z / sigma, U_inner = Z), tracking the relative
// change of sigma; the sigma vectors are read back each iteration (a few
// hundred bytes) for the convergence test.
DFac refine_factors(Ctx& ctx, const XView& x, const double* v_hat, long long ldv, int r,
                    const std::vector<double>& sigma_hat, double epsilon, int max_iters,
                    RefineStats* stats) {
  const int m = static_cast<int>(x.m), n = static_cast<int>(x.n);
  if (!(epsilon > 0.0)) throw Error(kInvalid, "refine_factors: epsilon must be > 0");
  if (max_iters < 1) throw Error(kInvalid, "refine_factors: max_iters must be >= 1");
  if ((int)sigma_hat.size() != r)
    throw Error(kInvalid, "refine_factors: sigma_hat length must match v_hat columns");
  {  // refine.cpp:37-42
    double* H = ctx.arena.alloc_n<double>((size_t)r * r);
    double* dd = ctx.arena.alloc_n<double>(1);
    ctx.phase = "refine.check";
    gemm_grouped(ctx, DType::F64, DType::F64, true, false, true,
                 {{v_hat, v_hat, H, ldv, ldv, r, r, r, n, 1.0, 0.0}});
    ortho_defect(ctx, H, r, r, dd);
    double* hd = ctx.pinned_dbl(1);
    HSVD_CUDA(cudaMemcpyAsync(hd, dd, sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    HSVD_CUDA(cudaStreamSynchronize(ctx.stream));
    if (!(hd[0] <= 1e-6)) throw Error(kInvalid, "refine_factors: v_hat columns are not orthonormal");
  }
  std::vector<double> sigma = sigma_hat;
  const double* V = v_hat;
  long long ldV = ldv;
  int rV = r;
  DFac out;
  double* Uo = nullptr;
  double* Uin = nullptr;
  int p = 0, kk = 0;
  double error = 0.0;
  int it = 0;
  do {
    ++it;
    DFac L = recover_left_vectors(ctx, x, V, ldV, rV);  // left basis of X V
    Uo = L.B;
    p = L.rank;
    kk = std::min(p, n);
    double* Bt = ctx.arena.alloc_n<double>((size_t)n * p);
    double* H = ctx.arena.alloc_n<double>((size_t)p * p);
    double* lam = ctx.arena.alloc_n<double>(kk);
    double* Z = ctx.arena.alloc_n<double>((size_t)p * kk);
    double* P = ctx.arena.alloc_n<double>((size_t)n * kk);
    double* Vn = ctx.arena.alloc_n<double>((size_t)n * kk);
    double* sig = ctx.arena.alloc_n<double>(kk);
    int* perm = ctx.arena.alloc_n<int>(kk);
    double* Zp = ctx.arena.alloc_n<double>((size_t)p * kk);
    int* d_rd = ctx.arena.alloc_n<int>(2);
    ctx.phase = "refine.proj";  // B^T = X^T U_outer (n x p): Xt is n x m, ld x.ld
    project_x(ctx, x.dt, false, {{x.X, Uo, Bt, x.ld, L.ld, n, n, p, m, 1.0, 0.0}});
    if (kk == p && small_svd_jacobi(n, p)) {  // kernels.cpp:28: full_svd(U^T X), p <= 32
      ctx.phase = "refine.jacobi";
      std::vector<JacJob> jj{{Bt, 1, 1, n, p, nullptr, nullptr, 0, 0, nullptr, n, nullptr, P, n,
                              Z, p}};
      jacobi_svd_batch(ctx, jj);
    } else {
      ctx.phase = "refine.gram";
      gemm_grouped(ctx, DType::F64, DType::F64, true, false, true,
                   {{Bt, Bt, H, n, n, p, p, p, n, 1.0, 0.0}});
      ctx.phase = "refine.eig";
      eig_topk(ctx, {{H, p, p, kk, lam, Z, p}});
      ctx.phase = "refine.back";
      gemm_grouped(ctx, DType::F64, DType::F64, false, false, false,
                   {{Bt, Z, P, n, p, n, n, kk, p, 1.0, 0.0}});
    }
    ctx.phase = "refine.fin";
    finalize(ctx, {{P, n, n, kk, 0.0, 0, Vn, n, sig, perm, d_rd, d_rd + 1, 1}});
    gather_cols(ctx, {{Zp, p, Z, p, p, kk, perm}});
    std::vector<int> rd;
    fetch_ranks(ctx, d_rd, 2, rd);
    const int rk = std::max(1, std::min(kk, rd[0]));
    std::vector<double> sn(rk);
    double* hs = ctx.pinned_dbl(rk);
    HSVD_CUDA(cudaMemcpyAsync(hs, sig, rk * sizeof(double), cudaMemcpyDeviceToHost, ctx.stream));
    HSVD_CUDA(cudaStreamSynchronize(ctx.stream));
    std::memcpy(sn.data(), hs, rk * sizeof(double));
    // refine.cpp:13-22, 55-57: padded difference relative to the old sigma
    const size_t len = std::max(sigma.size(), sn.size());
    double diff2 = 0.0, den2 = 0.0;
    for (size_t i = 0; i < len; ++i) {
      const double a = i < sigma.size() ? sigma[i] : 0.0, b = i < sn.size() ? sn[i] : 0.0;
      diff2 += (a - b) * (a - b);
    }
    for (double a : sigma) den2 += a * a;
    const double diff = std::sqrt(diff2), denom = std::sqrt(den2);
    error = denom > 0.0 ? diff / denom
                        : (diff > 0.0 ? std::numeric_limits<double>::infinity() : 0.0);
    sigma = sn;
    kk = rk;
    V = reorthonormalize(ctx, Vn, n, n, kk);
    ldV = n;
    rV = kk;
    Uin = Zp;
    out.sigma = sig;
    out.degenerate = rd[1] == 1;
  } while (error > epsilon && it < max_iters);
  // U = U_outer U_inner (m x kk)
  double* U = ctx.arena.alloc_n<double>((size_t)m * kk);
  ctx.phase = "refine.u";
  gemm_grouped(ctx, DType::F64, DType::F64, false, false, false,
               {{Uo, Uin, U, m, p, m, m, kk, p, 1.0, 0.0}});
  out.B = U;
  out.ld = m;
  out.dim = m;
  out.rank = kk;
  out.B2 = const_cast<double*>(V);
  out.ld2 = n;
  out.dim2 = n;
  if (stats) {
    stats->iterations = it;
    stats->final_error = error;
    stats->converged = error <= epsilon;
  }
  return out;
}

}  // namespace hsvdcu
