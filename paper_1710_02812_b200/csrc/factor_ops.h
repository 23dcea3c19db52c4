// Small per-factor kernels: finalisation (sigma, sort, truncation count,
// normalisation, null-direction completion), Gram scaling, gathers.
#pragma once

#include <vector>

#include "ctx.h"
#include "gemm.h"

namespace hsvdcu {

// P (s x p, col-major) holds the projected, unnormalised singular directions
// (columns = A z_i).  finalize writes, for the first `write` (= keep, or p
// when write_all) sorted columns, U[:, i] = P[:, perm[i]] / sigma_i, with
// sigma sorted non-increasing; columns whose sigma is below 1e-6*sigma_1
// (or zero) are completed to an orthonormal set.  rank = keep =
// min(retained_count(sigma, gamma), cap) (svd_factor.cpp:23-46).
struct FinJob {
  const double* P;
  long long ldp;
  int s;
  int p;
  double gamma;
  int cap;
  double* U;
  long long ldu;
  double* sigma;  // p
  int* perm;      // p (may be null)
  int* rank;      // 1
  int* degenerate;  // 1
  int write_all;
  // Sharded mode: squared column norms summed over all ranks (P holds this
  // rank's rows only).  Null directions are then not completed.
  const double* norms2 = nullptr;
};
void finalize(Ctx& ctx, const std::vector<FinJob>& jobs);

// G[i,j] *= w_i * w_j  (q x q)
struct ScaleSymJob {
  double* G;
  long long ld;
  int q;
  const double* w;
};
void scale_sym(Ctx& ctx, const std::vector<ScaleSymJob>& jobs);

// dst[i, j] = src[i, j] * w_i   (rows x cols)
struct ScaleRowsJob {
  double* dst;
  long long ldd;
  const double* src;
  long long lds;
  int rows, cols;
  const double* w;
};
void scale_rows(Ctx& ctx, const std::vector<ScaleRowsJob>& jobs);

// dst[:, i] = src[:, perm[i]]   (rows x cols); perm null -> identity copy
struct GatherJob {
  double* dst;
  long long ldd;
  const double* src;
  long long lds;
  int rows, cols;
  const int* perm;
};
void gather_cols(Ctx& ctx, const std::vector<GatherJob>& jobs);

// "Twice is enough" pass for a nearly orthonormal basis (defect ~eps*kappa^2
// from the Gram-form SVD): C = U^T U = R^T R (Cholesky, columns in sigma
// order), U <- U R^{-1}.  Removes the error components of small-sigma
// columns along larger ones; span and order are kept.  C is supplied by the
// caller (computed locally, or all-reduced in the sharded path).
void chol_inverse(Ctx& ctx, const double* C, int k, double* Rinv);

// out[c] = sum_r P[r, c]^2   (rows x cols)
void colnorms2(Ctx& ctx, const double* P, long long ld, int rows, int cols, double* out);

// out[0] = max |G - I| over the q x q matrix
void ortho_defect(Ctx& ctx, const double* G, long long ld, int q, double* out);

// Row-major (rows x cols, ld) fp64 host layout -> column-major device.
void rowmajor_to_colmajor(Ctx& ctx, const double* src, long long lds, int rows, int cols,
                          double* dst, long long ldd);
void colmajor_to_rowmajor(Ctx& ctx, const double* src, long long lds, int rows, int cols,
                          double* dst, long long ldd);

}  // namespace hsvdcu
