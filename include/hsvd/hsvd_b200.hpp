// hsvd_b200.hpp -- header-only C++ drop-in for the hot path of the reference
// library hsvd::core (/root/reference/proj/core/include/hsvd/*.hpp), running
// on a B200 through the C ABI in hsvd_cu.h.
//
// Same names, signatures and error behaviour as the reference:
//   hierarchy.hpp:18-50   BlockPlan, MergeStats, tree_merge, svd_of_col_slices,
//                         hierarchical_svd, recover_left_vectors
//   merge.hpp:12-30       MergeOrientation, merge_pair_naive, merge_pair_qr
//   kernels.hpp:12-29     DecompositionError, full_svd, qr_thin
//   svd_factor.hpp:14-49  SvdFactor, MatConfig, validate, retained_count,
//                         truncate_factor, reconstruct
//   refine.hpp:9-21       RefineResult, refine_factors
// DenseMatrix is an Eigen-free row-major real64 matrix with the accessors the
// callers of the path use (rows(), cols(), data(), operator()); Eigen is not
// available to this build.  std::invalid_argument and
// DecompositionError are thrown exactly where the reference throws them.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../hsvd_cu.h"

namespace hsvd {

using Index = std::int64_t;

class DenseMatrix {
 public:
  DenseMatrix() = default;
  DenseMatrix(Index rows, Index cols) : r_(rows), c_(cols), d_((size_t)(rows * cols), 0.0) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double& operator()(Index i, Index j) { return d_[(size_t)(i * c_ + j)]; }
  double operator()(Index i, Index j) const { return d_[(size_t)(i * c_ + j)]; }
  static DenseMatrix Identity(Index n, Index m) {
    DenseMatrix a(n, m);
    for (Index i = 0; i < std::min(n, m); ++i) a(i, i) = 1.0;
    return a;
  }
  DenseMatrix leftCols(Index k) const {
    DenseMatrix o(r_, k);
    for (Index i = 0; i < r_; ++i)
      for (Index j = 0; j < k; ++j) o(i, j) = (*this)(i, j);
    return o;
  }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> d_;
};

// Eigen::VectorXd stand-in: a std::vector<double> with Eigen-style element
// access (sigma(i), size()), so call sites like hsvd_main.cpp:100 compile.
class Vector : public std::vector<double> {
 public:
  using std::vector<double>::vector;
  Vector() = default;
  Vector(const std::vector<double>& v) : std::vector<double>(v) {}  // NOLINT
  double& operator()(Index i) { return (*this)[(size_t)i]; }
  double operator()(Index i) const { return (*this)[(size_t)i]; }
  Index size() const { return (Index)std::vector<double>::size(); }
};

// fp32 input matrix (the BASELINE configs' dtype): row-major float, the same
// accessors as DenseMatrix.  The reference promotes to its fp64 DenseMatrix;
// here fp32 crosses the C ABI as is (HSVD_CU_F32) and is computed on in fp64
// grade on the device.
class DenseMatrixF32 {
 public:
  DenseMatrixF32() = default;
  DenseMatrixF32(Index rows, Index cols) : r_(rows), c_(cols), d_((size_t)(rows * cols), 0.0f) {}
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  float* data() { return d_.data(); }
  const float* data() const { return d_.data(); }
  float& operator()(Index i, Index j) { return d_[(size_t)(i * c_ + j)]; }
  float operator()(Index i, Index j) const { return d_[(size_t)(i * c_ + j)]; }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<float> d_;
};

// A matrix already resident on the device (row-major, leading dimension ld,
// HSVD_CU_F32 or HSVD_CU_F64), e.g. produced by a CUDA kernel of the caller;
// it must be ready on the context's stream (see hsvd_cu.h).
struct DeviceMatrixView {
  const void* data = nullptr;
  int dtype = HSVD_CU_F32;
  Index rows = 0, cols = 0, ld = 0;
};

inline double frobenius_norm(const DenseMatrix& a) {
  double s = 0.0;
  for (Index i = 0; i < a.rows() * a.cols(); ++i) s += a.data()[i] * a.data()[i];
  return std::sqrt(s);
}

struct DecompositionError : std::runtime_error {
  DecompositionError(const std::string& what, Index rows, Index cols)
      : std::runtime_error(what), rows(rows), cols(cols) {}
  Index rows;
  Index cols;
};

struct SvdFactor {
  std::optional<DenseMatrix> u;
  Vector sigma;
  std::optional<DenseMatrix> v;
  bool degenerate = false;
  Index rank() const { return (Index)sigma.size(); }
  bool has_u() const { return u.has_value(); }
  bool has_v() const { return v.has_value(); }
};

struct MatConfig {
  double gamma = 1e-2;
  Index row_block_rows = 0;
  Index col_block_cols = 0;
  double epsilon = 1e-3;
  int max_iters = 10;
  std::optional<Index> max_rank;
};

enum class MergeOrientation { ColumnConcat, RowConcat };

struct Slice {
  Index start = 0;
  Index count = 0;
};

struct BlockPlan {
  std::vector<Slice> row_slices;
  std::vector<Slice> col_slices;
  static BlockPlan make(Index rows, Index cols, Index d, Index c) {
    if (rows < 1 || cols < 1) throw std::invalid_argument("BlockPlan: matrix must be nonempty");
    auto part = [](Index extent, Index block) {
      if (block < 1 || block > extent) block = extent;
      std::vector<Slice> s;
      for (Index st = 0; st < extent; st += block) s.push_back({st, std::min(block, extent - st)});
      return s;
    };
    return {part(rows, d), part(cols, c)};
  }
};

struct MergeStats {
  int pair_merges = 0;
};

namespace detail {

// One B200 context per thread (the C ABI context is not shared across
// threads), on the device chosen by hsvd::set_device (default 0).
struct Holder {
  hsvd_cu_ctx* c = nullptr;
  int device = 0;
  ~Holder() {
    if (c) hsvd_cu_ctx_destroy(c);
  }
};
inline Holder& holder() {
  thread_local Holder h;
  return h;
}
inline hsvd_cu_ctx* ctx() {
  Holder& h = holder();
  if (!h.c && hsvd_cu_ctx_create(h.device, &h.c) != HSVD_CU_OK)
    throw std::runtime_error(std::string("hsvd_b200: ") + hsvd_cu_last_error());
  return h.c;
}

inline void check(int code) {
  if (code == HSVD_CU_OK) return;
  const std::string msg = hsvd_cu_last_error();
  if (code == HSVD_CU_EINVAL) throw std::invalid_argument(msg);
  if (code == HSVD_CU_EDECOMP) {
    int64_t r = 0, c = 0;
    hsvd_cu_last_error_dims(&r, &c);
    throw DecompositionError(msg, r, c);
  }
  throw std::runtime_error("hsvd_b200: " + msg);
}

inline hsvd_cu_config to_c(const MatConfig& cfg) {
  hsvd_cu_config c;
  c.gamma = cfg.gamma;
  c.row_block_rows = cfg.row_block_rows;
  c.col_block_cols = cfg.col_block_cols;
  c.epsilon = cfg.epsilon;
  c.max_iters = cfg.max_iters;
  c.max_rank = cfg.max_rank ? *cfg.max_rank : 0;
  return c;
}

inline SvdFactor take(hsvd_cu_result* r) {
  std::unique_ptr<hsvd_cu_result, void (*)(hsvd_cu_result*)> guard(r, hsvd_cu_result_free);
  int64_t rank = 0, ur = 0, vr = 0;
  int32_t hu = 0, hv = 0, deg = 0;
  check(hsvd_cu_result_info(r, &rank, &hu, &hv, &ur, &vr, &deg));
  SvdFactor f;
  f.sigma.resize((size_t)rank);
  check(hsvd_cu_result_sigma(r, f.sigma.data()));
  if (hu) {
    f.u = DenseMatrix(ur, rank);
    check(hsvd_cu_result_u(r, f.u->data()));
  }
  if (hv) {
    f.v = DenseMatrix(vr, rank);
    check(hsvd_cu_result_v(r, f.v->data()));
  }
  f.degenerate = deg != 0;
  return f;
}

inline hsvd_cu_factor_in side(const SvdFactor& f, MergeOrientation o) {
  const std::optional<DenseMatrix>& b = o == MergeOrientation::ColumnConcat ? f.u : f.v;
  if (!b)
    throw std::invalid_argument(o == MergeOrientation::ColumnConcat
                                    ? "merge: ColumnConcat requires both factors to carry u"
                                    : "merge: RowConcat requires both factors to carry v");
  return {b->data(), b->rows(), b->cols(), b->cols(), f.sigma.data(), f.degenerate ? 1 : 0};
}

}  // namespace detail

// Selects the CUDA device of this thread's calls (one context per thread and
// device; the previous context is released).
inline void set_device(int device) {
  detail::Holder& h = detail::holder();
  if (h.c && h.device == device) return;
  if (h.c) {
    hsvd_cu_ctx_destroy(h.c);
    h.c = nullptr;
  }
  h.device = device;
}
inline int current_device() { return detail::holder().device; }

inline void validate(const MatConfig& cfg) {
  if (cfg.gamma < 0.0 || !std::isfinite(cfg.gamma))
    throw std::invalid_argument("MatConfig: gamma must be finite and >= 0");
  if (!(cfg.epsilon > 0.0)) throw std::invalid_argument("MatConfig: epsilon must be > 0");
  if (cfg.max_iters < 1) throw std::invalid_argument("MatConfig: max_iters must be >= 1");
  if (cfg.row_block_rows < 0 || cfg.col_block_cols < 0)
    throw std::invalid_argument("MatConfig: block sizes must be >= 0");
  if (cfg.max_rank && *cfg.max_rank < 1)
    throw std::invalid_argument("MatConfig: max_rank must be >= 1");
}

inline Index retained_count(const Vector& sigma, double gamma) {
  if (sigma.empty()) return 0;
  if (sigma[0] == 0.0) return 1;
  const double cutoff = gamma * sigma[0];
  Index kept = 0;
  while (kept < (Index)sigma.size() && sigma[(size_t)kept] >= cutoff) ++kept;
  return std::max<Index>(kept, 1);
}

inline SvdFactor truncate_factor(const SvdFactor& f, double gamma,
                                 std::optional<Index> max_rank = std::nullopt) {
  if (f.sigma.empty()) throw std::invalid_argument("truncate_factor: factor has an empty spectrum");
  Index keep = retained_count(f.sigma, gamma);
  if (max_rank) keep = std::min(keep, std::max<Index>(*max_rank, 1));
  SvdFactor out;
  out.sigma.assign(f.sigma.begin(), f.sigma.begin() + keep);
  if (f.u) out.u = f.u->leftCols(keep);
  if (f.v) out.v = f.v->leftCols(keep);
  out.degenerate = f.degenerate || f.sigma[0] == 0.0;
  return out;
}

inline DenseMatrix reconstruct(const SvdFactor& f) {
  if (!f.u || !f.v) throw std::invalid_argument("reconstruct: factor must carry both u and v");
  DenseMatrix x(f.u->rows(), f.v->rows());
  for (Index i = 0; i < x.rows(); ++i)
    for (Index j = 0; j < x.cols(); ++j) {
      double s = 0.0;
      for (Index t = 0; t < f.rank(); ++t) s += (*f.u)(i, t) * f.sigma[(size_t)t] * (*f.v)(j, t);
      x(i, j) = s;
    }
  return x;
}

inline SvdFactor full_svd(const DenseMatrix& a) {
  if (a.rows() == 0 || a.cols() == 0) throw std::invalid_argument("full_svd: matrix is empty");
  hsvd_cu_result* r = nullptr;
  detail::check(hsvd_cu_full_svd(detail::ctx(), a.data(), a.rows(), a.cols(), a.cols(), &r));
  return detail::take(r);
}

// kernels.hpp:29 qr_thin -> (Q rows x p, R p x cols), Householder on the device.
inline std::pair<DenseMatrix, DenseMatrix> qr_thin(const DenseMatrix& a) {
  if (a.rows() == 0 || a.cols() == 0) throw std::invalid_argument("qr_thin: matrix is empty");
  const Index p = std::min(a.rows(), a.cols());
  std::pair<DenseMatrix, DenseMatrix> qr{DenseMatrix(a.rows(), p), DenseMatrix(p, a.cols())};
  detail::check(hsvd_cu_qr_thin(detail::ctx(), a.data(), a.rows(), a.cols(), a.cols(),
                                qr.first.data(), qr.second.data()));
  return qr;
}

inline SvdFactor merge_pair_qr(const SvdFactor& f1, const SvdFactor& f2, MergeOrientation o,
                               double gamma, std::optional<Index> max_rank = std::nullopt) {
  hsvd_cu_factor_in a = detail::side(f1, o), b = detail::side(f2, o);
  hsvd_cu_result* r = nullptr;
  detail::check(hsvd_cu_merge_pair(detail::ctx(),
                                   o == MergeOrientation::ColumnConcat ? HSVD_CU_COLUMN_CONCAT
                                                                       : HSVD_CU_ROW_CONCAT,
                                   &a, &b, gamma, max_rank ? *max_rank : 0, &r));
  return detail::take(r);
}

inline SvdFactor merge_pair_naive(const SvdFactor& f1, const SvdFactor& f2, MergeOrientation o,
                                  double gamma, std::optional<Index> max_rank = std::nullopt) {
  return merge_pair_qr(f1, f2, o, gamma, max_rank);
}

inline SvdFactor tree_merge(std::vector<SvdFactor> factors, MergeOrientation o, double gamma,
                            std::optional<Index> max_rank = std::nullopt,
                            MergeStats* stats = nullptr) {
  if (factors.empty()) throw std::invalid_argument("tree_merge: factor list is empty");
  if (factors.size() == 1) return std::move(factors.front());
  std::vector<hsvd_cu_factor_in> in;
  for (const auto& f : factors) in.push_back(detail::side(f, o));
  int64_t pm = 0;
  hsvd_cu_result* r = nullptr;
  detail::check(hsvd_cu_tree_merge(detail::ctx(),
                                   o == MergeOrientation::ColumnConcat ? HSVD_CU_COLUMN_CONCAT
                                                                       : HSVD_CU_ROW_CONCAT,
                                   in.data(), (int64_t)in.size(), gamma,
                                   max_rank ? *max_rank : 0, &pm, &r));
  if (stats) stats->pair_merges += (int)pm;
  return detail::take(r);
}

inline SvdFactor svd_of_col_slices(const DenseMatrix& x_slice, Index c, double gamma,
                                   std::optional<Index> max_rank = std::nullopt) {
  hsvd_cu_result* r = nullptr;
  detail::check(hsvd_cu_svd_of_col_slices(detail::ctx(), x_slice.data(), HSVD_CU_F64,
                                          x_slice.rows(), x_slice.cols(), x_slice.cols(),
                                          HSVD_CU_HOST, c, gamma, max_rank ? *max_rank : 0, &r));
  return detail::take(r);
}

inline SvdFactor hierarchical_svd(const DenseMatrix& x, const MatConfig& cfg) {
  if (x.rows() == 0 || x.cols() == 0)
    throw std::invalid_argument("hierarchical_svd: matrix is empty");
  validate(cfg);
  const hsvd_cu_config c = detail::to_c(cfg);
  hsvd_cu_result* r = nullptr;
  detail::check(hsvd_cu_hierarchical_svd(detail::ctx(), x.data(), HSVD_CU_F64, x.rows(), x.cols(),
                                         x.cols(), HSVD_CU_HOST, &c, &r));
  return detail::take(r);
}

inline SvdFactor recover_left_vectors(const DenseMatrix& x, const DenseMatrix& v_r) {
  if (v_r.rows() != x.cols())
    throw std::invalid_argument("recover_left_vectors: v_r must have x.cols() rows");
  hsvd_cu_result* r = nullptr;
  detail::check(hsvd_cu_recover_left_vectors(detail::ctx(), x.data(), HSVD_CU_F64, x.rows(),
                                             x.cols(), x.cols(), HSVD_CU_HOST, v_r.data(),
                                             v_r.cols(), v_r.cols(), HSVD_CU_HOST, &r));
  return detail::take(r);
}

namespace detail {
inline SvdFactor hsvd_raw(const void* x, int dtype, Index m, Index n, Index ld, int where,
                          const MatConfig& cfg) {
  if (m == 0 || n == 0) throw std::invalid_argument("hierarchical_svd: matrix is empty");
  validate(cfg);
  const hsvd_cu_config c = to_c(cfg);
  hsvd_cu_result* r = nullptr;
  check(hsvd_cu_hierarchical_svd(ctx(), x, dtype, m, n, ld, where, &c, &r));
  return take(r);
}
inline SvdFactor recover_raw(const void* x, int dtype, Index m, Index n, Index ld, int where,
                             const DenseMatrix& v_r) {
  if (v_r.rows() != n)
    throw std::invalid_argument("recover_left_vectors: v_r must have x.cols() rows");
  hsvd_cu_result* r = nullptr;
  check(hsvd_cu_recover_left_vectors(ctx(), x, dtype, m, n, ld, where, v_r.data(), v_r.cols(),
                                     v_r.cols(), HSVD_CU_HOST, &r));
  return take(r);
}
}  // namespace detail

// fp32 and device-resident overloads of the drop-in (same contracts).
inline SvdFactor hierarchical_svd(const DenseMatrixF32& x, const MatConfig& cfg) {
  return detail::hsvd_raw(x.data(), HSVD_CU_F32, x.rows(), x.cols(), x.cols(), HSVD_CU_HOST, cfg);
}
inline SvdFactor hierarchical_svd(const DeviceMatrixView& x, const MatConfig& cfg) {
  return detail::hsvd_raw(x.data, x.dtype, x.rows, x.cols, x.ld, HSVD_CU_DEVICE, cfg);
}
inline SvdFactor recover_left_vectors(const DenseMatrixF32& x, const DenseMatrix& v_r) {
  return detail::recover_raw(x.data(), HSVD_CU_F32, x.rows(), x.cols(), x.cols(), HSVD_CU_HOST,
                             v_r);
}
inline SvdFactor recover_left_vectors(const DeviceMatrixView& x, const DenseMatrix& v_r) {
  return detail::recover_raw(x.data, x.dtype, x.rows, x.cols, x.ld, HSVD_CU_DEVICE, v_r);
}
inline SvdFactor svd_of_col_slices(const DenseMatrixF32& x_slice, Index c, double gamma,
                                   std::optional<Index> max_rank = std::nullopt) {
  hsvd_cu_result* r = nullptr;
  detail::check(hsvd_cu_svd_of_col_slices(detail::ctx(), x_slice.data(), HSVD_CU_F32,
                                          x_slice.rows(), x_slice.cols(), x_slice.cols(),
                                          HSVD_CU_HOST, c, gamma, max_rank ? *max_rank : 0, &r));
  return detail::take(r);
}

// refine.hpp:9-21 (Alg. 2).
struct RefineResult {
  SvdFactor factor;  // full (U, Sigma, V)
  int iterations = 0;
  double final_error = 0.0;  // last inter-iteration Sigma change
  bool converged = false;
};

inline RefineResult refine_factors(const DenseMatrix& x, const DenseMatrix& v_hat,
                                   const Vector& sigma_hat, double epsilon, int max_iters) {
  hsvd_cu_result* r = nullptr;
  std::int32_t it = 0, conv = 0;
  double err = 0.0;
  detail::check(hsvd_cu_refine_factors(
      detail::ctx(), x.data(), HSVD_CU_F64, x.rows(), x.cols(), x.cols(), HSVD_CU_HOST,
      v_hat.data(), v_hat.rows(), v_hat.cols(), v_hat.cols(), HSVD_CU_HOST, sigma_hat.data(),
      static_cast<std::int64_t>(sigma_hat.size()), epsilon, max_iters, &it, &err, &conv, &r));
  RefineResult out;
  out.factor = detail::take(r);
  out.iterations = it;
  out.final_error = err;
  out.converged = conv != 0;
  return out;
}

}  // namespace hsvd
