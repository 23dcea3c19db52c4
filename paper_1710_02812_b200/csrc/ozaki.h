// Leaf block Gram on tcgen05 kind::i8 (Ozaki slicing, fp64-grade): ozaki_gram.cu
#pragma once

#include <vector>

#include "ctx.h"
#include "gemm.h"

namespace hsvdcu {

// True when the SYRK descriptor (G = Xt Xt^T of a row-major fp32 block, as
// block_svd_batch builds it) runs on the int8 tensor-core Gram.  Disabled by
// HSVD_GRAM=dmma (then the fp64 DMMA SYRK runs).
bool ozaki_gram_applicable(DType dt, const GemmDesc& d);

// G (full symmetric storage, column-major ldc) = A A^T for every descriptor
// (A = the row-major d x c fp32 block viewed column-major c x d, lda; M = N =
// c, K = d).
void ozaki_gram_batch(Ctx& ctx, const std::vector<GemmDesc>& descs);

// The projection GEMMs of the path on the same int8 tensor-core machinery:
// C (M x N, column-major ldc) = op(A) B with A fp32 (op(A) = A^T of the
// column-major lda view when trans_a, i.e. rows of a row-major matrix; else
// the columns of a row-major K x M block), B fp64 column-major K x N
// (N <= 256), alpha = 1, beta = 0 -- gemm_grouped(ctx, F32, F64, trans_a,
// false, false, descs) semantics, fp64-grade.
bool ozaki_gemm_applicable(DType ta, bool trans_a, const GemmDesc& d);
void ozaki_gemm_batch(Ctx& ctx, bool trans_a, const std::vector<GemmDesc>& descs);

// Stage-1 trailing update of the two-stage eigensolver (ozaki_syr2k.cu):
// C (M x M, column-major ldc, full symmetric storage) -= VW WV^T for
// descriptors {VW + r0, WV + r0, A22, ld, ld, lda, m, m, K, -1, 1} of
// syev_band.cu, VW = [V_1 W_1 ...] (K = 64 x panels <= 256) and WV its
// panel-swapped copy (only VW is read).  Opt-in: HSVD_SYR2K=ozaki (measured
// slower than the DMMA SYR2K; see ozaki_syr2k.cu).
bool ozaki_syr2k_applicable(const GemmDesc& d);
void ozaki_syr2k_batch(Ctx& ctx, const std::vector<GemmDesc>& descs);

}  // namespace hsvdcu
