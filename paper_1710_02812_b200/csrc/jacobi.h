// Batched one-sided Jacobi SVD for narrow matrices (width <= 32): jacobi.cu.
#pragma once

#include <vector>

#include "ctx.h"

namespace hsvdcu {

constexpr int kJacMaxW = 32;

// A = [part 1 | part 2], s rows, w = w1 + w2 <= 32 columns.
//   part 1: element (i, j) = A[i*rs + j*cs] (fp32 or fp64), optionally times s1[j]
//   part 2: column-major fp64 (ld2), optionally times s2[j]
// Outputs: P = A V (s x w, column-major ldp, columns by decreasing norm) and
// V (w x w, column-major ldz, same order).
struct JacJob {
  const void* A;
  int f64;
  long long rs, cs;
  int w1;
  const double* s1;
  const double* A2;
  long long ld2;
  int w2;
  const double* s2;
  int s;
  double* W;  // scratch s x w (allocated by jacobi_svd_batch when null)
  double* P;
  long long ldp;
  double* Z;
  long long ldz;
};

// The reference's routing (kernels.cpp:28): the smaller side <= 32 goes to
// Jacobi.  (Bounded to s <= 2^20 rows: one CTA rotates the whole column set;
// HSVD_SMALL_SVD=gram forces the Gram route.)
bool small_svd_jacobi(long long s, int w);

void jacobi_svd_batch(Ctx& ctx, std::vector<JacJob>& jobs);

// Householder thin QR of the column-major m x n fp64 matrix A (overwritten:
// R on and above the diagonal, reflectors below); Q (m x min(m, n),
// column-major, ld m) written.  kernels.cpp:50-61.
void householder_qr(Ctx& ctx, double* A, int m, int n, double* Q);

}  // namespace hsvdcu
