// Drop-in check of include/hsvd/hsvd_b200.hpp: reference-style calls of the
// hsvd:: API (hierarchy.hpp, merge.hpp, kernels.hpp, svd_factor.hpp) compiled
// unchanged against the B200 library.  Exit code = number of failures.
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "hsvd/hsvd_b200.hpp"

using namespace hsvd;

static int failures = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);      \
      ++failures;                                                  \
    }                                                              \
  } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

// Orthonormal cosine basis column j of length n.
static double basis(Index i, Index j, Index n) {
  const double pi = std::acos(-1.0);
  const double s = j == 0 ? std::sqrt(1.0 / n) : std::sqrt(2.0 / n);
  return s * std::cos(pi * (i + 0.5) * j / n);
}

int main() {
  // X = U diag(5,4,3,2,1) V^T, exact rank 5 (generate.cpp recipe, fixed bases)
  const Index m = 96, n = 40, r = 5;
  DenseMatrix x(m, n);
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < n; ++j) {
      double s = 0.0;
      for (Index t = 0; t < r; ++t) s += basis(i, t + 1, m) * (5.0 - t) * basis(j, t + 2, n);
      x(i, j) = s;
    }
  MatConfig cfg;
  cfg.gamma = 1e-8;
  cfg.row_block_rows = 24;
  cfg.col_block_cols = 10;
  const SvdFactor right = hierarchical_svd(x, cfg);
  CHECK(right.rank() == r);
  CHECK(!right.has_u() && right.has_v());
  const SvdFactor full = recover_left_vectors(x, *right.v);
  CHECK(full.rank() == r);
  for (Index t = 0; t < r; ++t) CHECK(std::abs(full.sigma[(size_t)t] - (5.0 - t)) < 1e-10);
  const DenseMatrix rec = reconstruct(full);
  double diff = 0.0;
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < n; ++j) diff += (rec(i, j) - x(i, j)) * (rec(i, j) - x(i, j));
  CHECK(std::sqrt(diff) < 1e-10 * frobenius_norm(x));

  // refinement (refine.hpp): exact subspace is a fixed point after one pass
  const RefineResult rr = refine_factors(x, *right.v, right.sigma, 1e-6, 5);
  CHECK(rr.converged && rr.iterations <= 2 && rr.factor.rank() == r);
  for (Index t = 0; t < r; ++t) CHECK(std::abs(rr.factor.sigma[(size_t)t] - (5.0 - t)) < 1e-10);
  CHECK(throws<std::invalid_argument>([&] { refine_factors(x, *right.v, right.sigma, 0.0, 5); }));
  CHECK(throws<std::invalid_argument>([&] { refine_factors(x, *right.v, right.sigma, 1e-6, 0); }));

  // merges and the tree (merge.hpp / hierarchy.hpp)
  SvdFactor f1, f2;
  f1.u = DenseMatrix(4, 1);
  (*f1.u)(0, 0) = 1.0;
  f1.sigma = {1.0};
  f2.u = DenseMatrix(4, 1);
  (*f2.u)(1, 0) = 1.0;
  f2.sigma = {1.0};
  const SvdFactor mg = merge_pair_qr(f1, f2, MergeOrientation::ColumnConcat, 0.0);
  CHECK(mg.rank() == 2 && std::abs(mg.sigma[0] - 1.0) < 1e-12);
  MergeStats st;
  tree_merge({f1, f2, f1}, MergeOrientation::ColumnConcat, 0.0, std::nullopt, &st);
  CHECK(st.pair_merges == 2);

  // error behaviour of the reference
  CHECK(throws<std::invalid_argument>([] { hierarchical_svd(DenseMatrix(), MatConfig()); }));
  MatConfig bad;
  bad.gamma = -1.0;
  CHECK(throws<std::invalid_argument>([&] { hierarchical_svd(x, bad); }));
  CHECK(throws<std::invalid_argument>([&] { recover_left_vectors(x, DenseMatrix(n, 2)); }));
  CHECK(throws<std::invalid_argument>([] { tree_merge({}, MergeOrientation::RowConcat, 0.0); }));
  SvdFactor g;
  g.u = DenseMatrix(5, 1);
  (*g.u)(0, 0) = 1.0;
  g.sigma = {1.0};
  CHECK(throws<std::invalid_argument>([&] { merge_pair_qr(f1, g, MergeOrientation::ColumnConcat, 0.0); }));
  CHECK(throws<std::invalid_argument>([&] { merge_pair_qr(f1, f2, MergeOrientation::RowConcat, 0.0); }));
  const BlockPlan plan = BlockPlan::make(10, 7, 4, 3);
  CHECK(plan.row_slices.size() == 3 && plan.col_slices[2].count == 1);

  // Eigen-style sigma(i) access (hsvd_main.cpp:100 prints sigma(i))
  CHECK(std::abs(full.sigma(0) - 5.0) < 1e-10 && full.sigma.size() == r);

  // fp32 overloads (the BASELINE dtype) agree with the fp64 path
  DenseMatrixF32 xf(m, n);
  for (Index i = 0; i < m; ++i)
    for (Index j = 0; j < n; ++j) xf(i, j) = (float)x(i, j);
  const SvdFactor rf = hierarchical_svd(xf, cfg);
  const SvdFactor ff = recover_left_vectors(xf, *rf.v);
  CHECK(ff.rank() == r);
  for (Index t = 0; t < r; ++t) CHECK(std::abs(ff.sigma(t) - (5.0 - t)) < 1e-5);

  // kernels.hpp:29 qr_thin: Q R = A, Q orthonormal, R upper triangular
  DenseMatrix a(7, 4);
  for (Index i = 0; i < 7; ++i)
    for (Index j = 0; j < 4; ++j) a(i, j) = std::sin(1.0 + i * 0.7 + j * 1.3);
  const auto qr = qr_thin(a);
  double qerr = 0.0, oerr = 0.0;
  for (Index i = 0; i < 7; ++i)
    for (Index j = 0; j < 4; ++j) {
      double s = 0.0;
      for (Index t = 0; t < 4; ++t) s += qr.first(i, t) * qr.second(t, j);
      qerr = std::max(qerr, std::abs(s - a(i, j)));
    }
  for (Index i = 0; i < 4; ++i)
    for (Index j = 0; j < 4; ++j) {
      double s = 0.0;
      for (Index t = 0; t < 7; ++t) s += qr.first(t, i) * qr.first(t, j);
      oerr = std::max(oerr, std::abs(s - (i == j ? 1.0 : 0.0)));
      if (i > j) CHECK(qr.second(i, j) == 0.0);
    }
  CHECK(qerr < 1e-13 && oerr < 1e-13);
  CHECK(throws<std::invalid_argument>([] { qr_thin(DenseMatrix()); }));

  // device selection (one context per thread and device)
  set_device(0);
  CHECK(current_device() == 0);
  CHECK(hierarchical_svd(x, cfg).rank() == r);

  std::printf("cpp api: %d failure(s)\n", failures);
  return failures;
}
