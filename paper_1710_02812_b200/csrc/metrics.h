// Device evaluation of reconstruction errors: the
// chunked analog of the reference's factor_diff_norm (bench.cpp:30-42) and
// rank_k_error (svd_factor.cpp:66-80), without materialising the m x n
// difference.
#pragma once

#include "ctx.h"
#include "gemm.h"

namespace hsvdcu {

// sum_{i<m, j<n} ( (A B^T)[i,j] + X[i,j] )^2 with A (m x k, column-major,
// lda), B (n x k, column-major, ldb) and an optional X (row-major m x n,
// ldx; dt its element type; null = 0).  Fused DMMA tiles with a
// sum-of-squares epilogue and a fixed-order final reduction (deterministic).
double product_plus_sumsq(Ctx& ctx, const double* A, long long lda, const double* B,
                          long long ldb, int m, int n, int k, const void* X, DType dt,
                          long long ldx);

// dst[:, c] = sign * w[c] * src[:, c] (w null: 1), column-major.
void scale_cols_copy(Ctx& ctx, double* dst, long long ldd, const double* src, long long lds,
                     int rows, int cols, const double* w, double sign);

}  // namespace hsvdcu
