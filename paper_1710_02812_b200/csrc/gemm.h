// Grouped fp64-accumulating GEMM on the sm_100a fp64 tensor path (DMMA).
#pragma once

#include <vector>

#include "ctx.h"

namespace hsvdcu {

enum class DType : int { F32 = 0, F64 = 1 };

// Column-major (BLAS) convention: C (MxN) = alpha * op(A) (MxK) * op(B) (KxN)
// + beta * C.  op(A) = A (col-major, lda) or A^T; A and B may be fp32 or fp64
// (promoted to fp64 on load); C is fp64.  A row-major matrix with leading
// dimension ld is the transposed column-major view with the same ld.
struct GemmDesc {
  const void* A;
  const void* B;
  double* C;
  long long lda, ldb, ldc;
  int M, N, K;
  double alpha, beta;
};

// flags for gemm_grouped
enum : int {
  kGemmLowerOnly = 1,  // with syrk: write the lower tile triangle only (no mirror)
};

// syrk=true: op(A) op(B) is known symmetric (op(B) == op(A)^T); only the
// lower tile triangle is computed (and mirrored unless kGemmLowerOnly).
void gemm_grouped(Ctx& ctx, DType ta, DType tb, bool trans_a, bool trans_b, bool syrk,
                  const std::vector<GemmDesc>& descs, int flags = 0);

// Skinny fp64 GEMM (N <= 32, no transposes) fed by cp.async.bulk (gemm_sk.cu);
// gemm_grouped routes to it when the operands allow 16-byte bulk copies and
// the grid is large enough without split-K (HSVD_GEMM_SK=0 disables).
bool gemm_sk_applicable(const std::vector<GemmDesc>& descs, int num_sms);
void gemm_sk(Ctx& ctx, const std::vector<GemmDesc>& descs);

}  // namespace hsvdcu
