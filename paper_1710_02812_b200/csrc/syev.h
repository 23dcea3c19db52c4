// Batched fp64 symmetric eigensolver for the top-kk eigenpairs.
#pragma once

#include <vector>

#include "ctx.h"

namespace hsvdcu {

// A is n x n symmetric, column-major (full storage), overwritten.
// Outputs: lam[0..kk) descending, Z (n x kk, column-major, ldz) orthonormal.
struct EigJob {
  double* A;
  long long lda;
  int n;
  int kk;
  double* lam;
  double* Z;
  long long ldz;
};

void eig_topk(Ctx& ctx, const std::vector<EigJob>& jobs);

}  // namespace hsvdcu
