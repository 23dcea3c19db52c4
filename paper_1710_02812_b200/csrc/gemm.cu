// Grouped fp64 GEMM for the HSVD path on sm_100a.
//
// Every contraction of the hot path (block Grams X_b^T X_b, projections
// X_b Z, V-recovery X_j^T U_j, U-recovery X V_r, merge Grams/projections,
// the two-stage band reduction and the blocked Householder back-transforms)
// runs through this kernel.  The reference computes all of them in IEEE
// binary64 (Eigen, dense_matrix.hpp:9); tcgen05.mma has no f64 kind, so the
// fp64-exact tensor path on B200 is DMMA (mma.sync.m8n8k4.f64 -> SASS
// DMMA.8x8x4).  fp32 inputs (the BASELINE matrices) are promoted to fp64 on
// the way into shared memory, which is exactly what the reference's fp64
// DenseMatrix computes on the same bytes.
//
// Tiles: 64x64 (2x2 warps) or, for skinny outputs (N <= 32), 128x32 (4x1
// warps); each warp owns 32x32 = 4x4 DMMA tiles; BK = 16 with register-
// prefetch double buffering; C (when beta != 0) is fetched before the main
// loop so its latency overlaps the products.  Optional split-K with a
// deterministic fixed-order reduction (run-to-run bitwise stable).
// Options: SYRK (lower tile triangle, mirrored unless kGemmLowerOnly) and
// kGemmSymA (A symmetric, only its lower triangle is read).
#include <algorithm>

#include "gemm.h"

namespace hsvdcu {

namespace {

constexpr int BK = 16, PAD = 4, NT = 128;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <typename T>
__device__ __forceinline__ double ldg(const T* p) { return static_cast<double>(__ldg(p)); }

// mode bits
constexpr int kModeSyrk = 1, kModeLower = 2, kModeSymA = 4;

// EXT: C prefetched into registers before the main loop and the SymA
// loader (fp64 operands only; costs registers, so the plain variant serves
// every other call)
template <typename TA, typename TB, bool TRA, bool TRB, int BM, int BN, bool EXT>
__global__ void __launch_bounds__(NT) k_gemm(const GemmDesc* __restrict__ descs, int mode,
                                             int splits, double* __restrict__ ws,
                                             long long ws_slot) {
  constexpr int WN = BN / 32;  // warps along N
  constexpr int LA = BM * BK / NT, LB = BN * BK / NT;
  const int g = blockIdx.z / splits;
  const int split = blockIdx.z - g * splits;
  const GemmDesc d = descs[g];
  const int tm = blockIdx.x, tn = blockIdx.y;
  if (tm * BM >= d.M || tn * BN >= d.N) return;
  const bool syrk = (mode & kModeSyrk) != 0;
  if (syrk && tn * BN >= (tm + 1) * BM) return;  // strictly upper tile
  const bool symA = EXT && !TRA && (mode & kModeSymA) != 0;

  int kchunk = (d.K + splits - 1) / splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  const int kb = split * kchunk;
  const int ke = min(d.K, kb + kchunk);

  constexpr int A_ELEMS = 2 * BK * (BM + PAD), B_ELEMS = 2 * BK * (BN + PAD);
  constexpr int T_LD = BN + 1;
  static_assert(A_ELEMS + B_ELEMS >= BM * T_LD, "epilogue tile must fit");
  __shared__ __align__(16) double smem_raw[A_ELEMS + B_ELEMS];
  double (*As)[BK][BM + PAD] = reinterpret_cast<double (*)[BK][BM + PAD]>(smem_raw);
  double (*Bs)[BK][BN + PAD] = reinterpret_cast<double (*)[BK][BN + PAD]>(smem_raw + A_ELEMS);

  const TA* A = static_cast<const TA*>(d.A);
  const TB* B = static_cast<const TB*>(d.B);
  const int tid = threadIdx.x;
  const int m0 = tm * BM, n0 = tn * BN;
  const int lane = tid & 31, warp = tid >> 5;
  const int grp = lane >> 2, tig = lane & 3;
  const int wm = (warp / WN) * 32, wn = (warp % WN) * 32;

  // C prefetch (epilogue operand), issued before the main loop
  const bool to_ws = ws != nullptr;
  const bool pre_c = EXT && !to_ws && d.beta != 0.0;
  double cpre[EXT ? 4 : 1][4][2];
  if (EXT) {
#pragma unroll
    for (int i = 0; i < (EXT ? 4 : 1); ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int m = m0 + wm + i * 8 + grp, n = n0 + wn + j * 8 + 2 * tig + r;
          cpre[i][j][r] = (pre_c && m < d.M && n < d.N) ? d.C[m + (long long)n * d.ldc] : 0.0;
        }
  }

  // A-tile layout of a k-tile: 0 = m fastest (A column-major), 1 = k fastest
  // (A^T, or the mirrored upper part of a symmetric A), 2 = diagonal-crossing
  // tile of a symmetric A (m fastest, per-element mirror)
  auto a_layout = [&](int k0) -> int {
    if (TRA) return 1;
    if (!EXT || !symA) return 0;
    if (k0 >= m0 + BM) return 1;
    if (k0 + BK <= m0 + 1) return 0;
    return 2;
  };
  double ra[LA], rb[LB];
  int lay_ld = 0;
  auto load = [&](int k0) {
    const int lay = a_layout(k0);
    lay_ld = lay;
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      const int idx = tid + i * NT;
      int m, k;
      if (lay == 1) { k = idx % BK; m = idx / BK; }
      else          { m = idx % BM; k = idx / BM; }
      const int gm = m0 + m, gk = k0 + k;
      double v = 0.0;
      if (gm < d.M && gk < ke) {
        const bool tr = lay == 1 || (lay == 2 && gk > gm);
        v = tr ? ldg(A + (long long)gk + (long long)gm * d.lda)
               : ldg(A + (long long)gm + (long long)gk * d.lda);
      }
      ra[i] = v;
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const int idx = tid + i * NT;
      int n, k;
      if (!TRB) { k = idx % BK; n = idx / BK; }
      else      { n = idx % BN; k = idx / BN; }
      const int gn = n0 + n, gk = k0 + k;
      double v = 0.0;
      if (gn < d.N && gk < ke)
        v = TRB ? ldg(B + (long long)gn + (long long)gk * d.ldb)
                : ldg(B + (long long)gk + (long long)gn * d.ldb);
      rb[i] = v;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      const int idx = tid + i * NT;
      int m, k;
      if (lay_ld == 1) { k = idx % BK; m = idx / BK; }
      else             { m = idx % BM; k = idx / BM; }
      As[buf][k][m] = ra[i];
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const int idx = tid + i * NT;
      int n, k;
      if (!TRB) { k = idx % BK; n = idx / BK; }
      else      { n = idx % BN; k = idx / BN; }
      Bs[buf][k][n] = rb[i];
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  int buf = 0;
  if (kb < ke) {
    load(kb);
    store(0);
  }
  __syncthreads();
  for (int k0 = kb; k0 < ke; k0 += BK) {
    const bool more = k0 + BK < ke;
    if (more) load(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[buf][kk + tig][wm + i * 8 + grp];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[buf][kk + tig][wn + j * 8 + grp];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
    }
    if (more) {
      store(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }

  // epilogue: direct store (each warp instruction writes 4 columns x 8
  // consecutive rows); the SYRK mirror of an off-diagonal tile reuses the
  // final values staged in shared memory so the transposed store is coalesced
  double* out = to_ws ? ws + (long long)blockIdx.z * ws_slot : d.C;
  const long long ldo = to_ws ? (long long)d.M : d.ldc;
  const double alpha = d.alpha, beta = d.beta;
  const bool diag_tile = n0 < m0 + BM && m0 < n0 + BN;
  const bool mirror = syrk && !(mode & kModeLower) && !to_ws && !diag_tile;
  double* tile = smem_raw;  // [BM][T_LD], tile[ml * T_LD + nl]
  if (mirror) __syncthreads();  // operand tiles no longer read
  // C reads batched before any store (see k_gemm64)
  if (!to_ws) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int m = m0 + wm + i * 8 + grp, n = n0 + wn + j * 8 + 2 * tig + r;
          double c = 0.0;
          if (pre_c) c = cpre[EXT ? i : 0][j][r];
          else if (beta != 0.0 && m < d.M && n < d.N) c = out[m + (long long)n * ldo];
          acc[i][j][r] = alpha * acc[i][j][r] + beta * c;
        }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int ml = wm + i * 8 + grp;
    const int m = m0 + ml;
    if (m >= d.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int nl = wn + j * 8 + 2 * tig + r;
        const int n = n0 + nl;
        if (n >= d.N) continue;
        const double v = acc[i][j][r];
        out[m + (long long)n * ldo] = v;
        if (mirror) tile[ml * T_LD + nl] = v;
      }
    }
  }
  if (mirror) {
    __syncthreads();
    for (int idx = tid; idx < BM * BN; idx += NT) {
      const int nl = idx % BN, ml = idx / BN;
      const int m = m0 + ml, n = n0 + nl;
      if (m >= d.M || n >= d.N) continue;
      out[n + (long long)m * ldo] = tile[ml * T_LD + nl];
    }
  }
}

// ---------------------------------------------------------------------------
// fp64 x fp64: cp.async multi-stage pipeline.  Operands go global -> shared
// memory without register staging (LDGSTS, zero-filled out of bounds), four
// k-stages in flight; each operand tile keeps the memory-contiguous
// dimension contiguous in shared memory, so the copies are coalesced and
// conflict-free and the address arithmetic is one increment per element.
// ---------------------------------------------------------------------------
constexpr int STAGES = 3;

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool ok) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src),
               "r"(ok ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Shared layout of one operand tile (R rows of the output dimension, BK of
// k): KF (k contiguous in memory) -> [R][BK + 4]; else [BK][R + 4].
template <int R, bool KF>
struct OpTile {
  static constexpr int LD = KF ? BK + 4 : R + 4;
  static constexpr int ELEMS = KF ? R * (BK + 4) : BK * (R + 4);
  __device__ static int at(int r, int k) { return KF ? r * LD + k : k * LD + r; }
};

template <bool TRA, bool TRB, int BM, int BN>
__global__ void __launch_bounds__(NT) k_gemm64(const GemmDesc* __restrict__ descs, int mode,
                                               int splits, double* __restrict__ ws,
                                               long long ws_slot) {
  // A element (m, k): !TRA -> A[m + k lda] (m contiguous), TRA -> A[k + m lda]
  // B element (k, n): !TRB -> B[k + n ldb] (k contiguous), TRB -> B[n + k ldb]
  using TA_ = OpTile<BM, TRA>;
  using TB_ = OpTile<BN, !TRB>;
  constexpr int WN = BN / 32;
  constexpr int LA = BM * BK / NT, LB = BN * BK / NT;
  constexpr int STAGE = TA_::ELEMS + TB_::ELEMS;
  extern __shared__ __align__(16) double dsm[];

  const int g = blockIdx.z / splits;
  const int split = blockIdx.z - g * splits;
  const GemmDesc d = descs[g];
  const int tm = blockIdx.x, tn = blockIdx.y;
  if (tm * BM >= d.M || tn * BN >= d.N) return;
  const bool syrk = (mode & kModeSyrk) != 0;
  if (syrk && tn * BN >= (tm + 1) * BM) return;
  int kchunk = (d.K + splits - 1) / splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  const int kb = split * kchunk;
  const int ke = min(d.K, kb + kchunk);
  const int nkt = ke > kb ? (ke - kb + BK - 1) / BK : 0;

  const double* A = static_cast<const double*>(d.A);
  const double* B = static_cast<const double*>(d.B);
  const int tid = threadIdx.x;
  const int m0 = tm * BM, n0 = tn * BN;

  // per-thread copy assignments: element e = tid + i*NT of the tile, the
  // contiguous dimension fastest
  auto a_rc = [&](int i, int& r, int& k) {
    const int e = tid + i * NT;
    if (TRA) { k = e % BK; r = e / BK; } else { r = e % BM; k = e / BM; }
  };
  auto b_rc = [&](int i, int& r, int& k) {
    const int e = tid + i * NT;
    if (!TRB) { k = e % BK; r = e / BK; } else { r = e % BN; k = e / BN; }
  };
  auto issue = [&](int kt) {
    double* As = dsm + (kt % STAGES) * STAGE;
    double* Bs = As + TA_::ELEMS;
    const int k0 = kb + kt * BK;
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      int r, k;
      a_rc(i, r, k);
      const int gm = m0 + r, gk = k0 + k;
      const bool ok = gm < d.M && gk < ke;
      const double* src = ok ? (TRA ? A + (long long)gk + (long long)gm * d.lda
                                    : A + (long long)gm + (long long)gk * d.lda)
                             : A;
      cp_async8(As + TA_::at(r, k), src, ok);
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      int r, k;
      b_rc(i, r, k);
      const int gn = n0 + r, gk = k0 + k;
      const bool ok = gn < d.N && gk < ke;
      const double* src = ok ? (TRB ? B + (long long)gn + (long long)gk * d.ldb
                                    : B + (long long)gk + (long long)gn * d.ldb)
                             : B;
      cp_async8(Bs + TB_::at(r, k), src, ok);
    }
  };

  const int lane = tid & 31, warp = tid >> 5;
  const int grp = lane >> 2, tig = lane & 3;
  const int wm = (warp / WN) * 32, wn = (warp % WN) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nkt) issue(s);
    cp_async_commit();
  }
  for (int kt = 0; kt < nkt; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (kt + STAGES - 1 < nkt) issue(kt + STAGES - 1);
    cp_async_commit();
    const double* As = dsm + (kt % STAGES) * STAGE;
    const double* Bs = As + TA_::ELEMS;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[TA_::at(wm + i * 8 + grp, kk + tig)];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[TB_::at(wn + j * 8 + grp, kk + tig)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
    }
  }
  cp_async_wait<0>();

  const bool to_ws = ws != nullptr;
  double* out = to_ws ? ws + (long long)blockIdx.z * ws_slot : d.C;
  const long long ldo = to_ws ? (long long)d.M : d.ldc;
  const double alpha = d.alpha, beta = d.beta;
  const bool diag_tile = n0 < m0 + BM && m0 < n0 + BN;
  const bool mirror = syrk && !(mode & kModeLower) && !to_ws && !diag_tile;
  constexpr int T_LD = BN + 1;
  static_assert(STAGES * STAGE >= BM * T_LD, "epilogue tile must fit");
  double* tile = dsm;
  if (mirror) __syncthreads();
  // all C reads issued before any store (the stores could alias them, so the
  // compiler would otherwise serialise load -> store pairs)
  if (!to_ws && beta != 0.0) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int m = m0 + wm + i * 8 + grp, n = n0 + wn + j * 8 + 2 * tig + r;
          const double c = (m < d.M && n < d.N) ? out[m + (long long)n * ldo] : 0.0;
          acc[i][j][r] = alpha * acc[i][j][r] + beta * c;
        }
  } else if (!to_ws) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc[i][j][0] *= alpha;
        acc[i][j][1] *= alpha;
      }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int ml = wm + i * 8 + grp;
    const int m = m0 + ml;
    if (m >= d.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int nl = wn + j * 8 + 2 * tig + r;
        const int n = n0 + nl;
        if (n >= d.N) continue;
        const double v = acc[i][j][r];
        out[m + (long long)n * ldo] = v;
        if (mirror) tile[ml * T_LD + nl] = v;
      }
    }
  }
  if (mirror) {
    __syncthreads();
    for (int idx = tid; idx < BM * BN; idx += NT) {
      const int nl = idx % BN, ml = idx / BN;
      const int m = m0 + ml, n = n0 + nl;
      if (m >= d.M || n >= d.N) continue;
      out[n + (long long)m * ldo] = tile[ml * T_LD + nl];
    }
  }
}

template <bool TRA, bool TRB, int BM, int BN>
void launch64_t(Ctx& ctx, dim3 grid, const GemmDesc* dd, int mode, int splits, double* ws,
                long long slot) {
  constexpr size_t smem = (size_t)STAGES *
                          (OpTile<BM, TRA>::ELEMS + OpTile<BN, !TRB>::ELEMS) * sizeof(double);
  auto* k = k_gemm64<TRA, TRB, BM, BN>;
  smem_optin(k, smem);
  k<<<grid, NT, smem, ctx.stream>>>(dd, mode, splits, ws, slot);
}

template <int BM, int BN>
void launch64(Ctx& ctx, bool ta, bool tb, dim3 grid, const GemmDesc* dd, int mode, int splits,
              double* ws, long long slot) {
  ctx.launch_begin();
  if (!ta && !tb) launch64_t<false, false, BM, BN>(ctx, grid, dd, mode, splits, ws, slot);
  else if (!ta && tb) launch64_t<false, true, BM, BN>(ctx, grid, dd, mode, splits, ws, slot);
  else if (ta && !tb) launch64_t<true, false, BM, BN>(ctx, grid, dd, mode, splits, ws, slot);
  else launch64_t<true, true, BM, BN>(ctx, grid, dd, mode, splits, ws, slot);
  ctx.check_launch("k_gemm");
}

__global__ void k_splitk_reduce(const GemmDesc* __restrict__ descs, int splits, int mode,
                                const double* __restrict__ ws, long long ws_slot) {
  const int g = blockIdx.y;
  const GemmDesc d = descs[g];
  const bool syrk = (mode & kModeSyrk) != 0, mirror = syrk && !(mode & kModeLower);
  const long long total = (long long)d.M * d.N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(e % d.M), n = (int)(e / d.M);
    if (syrk && m < n) continue;
    double s = 0.0;
    const double* base = ws + (long long)g * splits * ws_slot + m + (long long)n * d.M;
    for (int t = 0; t < splits; ++t) s += base[t * ws_slot];
    s *= d.alpha;
    double* c = d.C + m + (long long)n * d.ldc;
    if (d.beta != 0.0) s += d.beta * *c;
    *c = s;
    if (mirror && m != n) d.C[n + (long long)m * d.ldc] = s;
  }
}

template <typename TA, typename TB, int BM, int BN, bool EXT>
void launch_tile(Ctx& ctx, bool ta, bool tb, dim3 grid, const GemmDesc* dd, int mode, int splits,
                 double* ws, long long slot) {
  cudaStream_t s = ctx.stream;
  ctx.launch_begin();
  if (!ta && !tb)
    k_gemm<TA, TB, false, false, BM, BN, EXT><<<grid, NT, 0, s>>>(dd, mode, splits, ws, slot);
  else if (!ta && tb)
    k_gemm<TA, TB, false, true, BM, BN, EXT><<<grid, NT, 0, s>>>(dd, mode, splits, ws, slot);
  else if (ta && !tb)
    k_gemm<TA, TB, true, false, BM, BN, EXT><<<grid, NT, 0, s>>>(dd, mode, splits, ws, slot);
  else
    k_gemm<TA, TB, true, true, BM, BN, EXT><<<grid, NT, 0, s>>>(dd, mode, splits, ws, slot);
  ctx.check_launch("k_gemm");
}

template <typename TA, typename TB, bool EXT>
void launch_typed(Ctx& ctx, bool ta, bool tb, bool skinny, int maxM, int maxN, int count,
                  const GemmDesc* dd, int mode, int splits, double* ws, long long slot) {
  if (skinny) {
    dim3 grid(ceil_div(maxM, 128), ceil_div(maxN, 32), count * splits);
    launch_tile<TA, TB, 128, 32, EXT>(ctx, ta, tb, grid, dd, mode, splits, ws, slot);
  } else {
    dim3 grid(ceil_div(maxM, 64), ceil_div(maxN, 64), count * splits);
    launch_tile<TA, TB, 64, 64, EXT>(ctx, ta, tb, grid, dd, mode, splits, ws, slot);
  }
}

}  // namespace

void gemm_grouped(Ctx& ctx, DType ta, DType tb, bool trans_a, bool trans_b, bool syrk,
                  const std::vector<GemmDesc>& descs, int flags) {
  std::vector<GemmDesc> live;
  live.reserve(descs.size());
  int maxM = 0, maxN = 0, maxK = 0;
  for (const auto& d : descs) {
    if (d.M <= 0 || d.N <= 0) continue;
    live.push_back(d);
    maxM = std::max(maxM, d.M);
    maxN = std::max(maxN, d.N);
    maxK = std::max(maxK, d.K);
  }
  if (live.empty()) return;
  const int count = static_cast<int>(live.size());
  if (count > 65535) throw Error(kInvalid, "gemm_grouped: too many groups");
  if ((flags & kGemmSymA) && (trans_a || ta != DType::F64 || tb != DType::F64))
    throw Error(kInvalid, "gemm_grouped: SymA needs op(A) = A and fp64 operands");
  const bool skinny = !syrk && maxN <= 32;
  const int BMt = skinny ? 128 : 64, BNt = skinny ? 32 : 64;
  long long tiles = 0;
  double flops = 0.0;  // algorithmic (SYRK: the lower triangle)
  for (const auto& d : live) {
    long long t = (long long)ceil_div(d.M, BMt) * ceil_div(d.N, BNt);
    if (syrk) t = (t + ceil_div(d.M, BMt)) / 2;
    tiles += t;
    flops += syrk ? (double)d.M * (d.M + 1) * d.K : 2.0 * d.M * d.N * d.K;
  }

  int splits = 1;
  const long long target = 4LL * ctx.num_sms;
  if (tiles < target && maxK >= 2 * 256) {
    splits = static_cast<int>(std::min<long long>((target + tiles - 1) / tiles, maxK / 256));
    splits = std::max(1, std::min(splits, 128));
    while (splits > 1 && (long long)count * splits > 65535) --splits;
  }
  const GemmDesc* dd =
      static_cast<const GemmDesc*>(ctx.staging.put(live.data(), live.size() * sizeof(GemmDesc),
                                                   ctx.stream));
  double* ws = nullptr;
  long long slot = 0;
  Arena::Mark mk = ctx.arena.mark();
  if (splits > 1) {
    slot = (long long)maxM * maxN;
    ws = ctx.arena.alloc_n<double>((size_t)slot * count * splits);
  }
  const int mode = (syrk ? kModeSyrk : 0) | ((flags & kGemmLowerOnly) ? kModeLower : 0) |
                   ((flags & kGemmSymA) ? kModeSymA : 0);
  ctx.pending_flops = flops;
  const bool ext = (flags & kGemmSymA) != 0;
  if (ta == DType::F64 && tb == DType::F64 && ext)
    launch_typed<double, double, true>(ctx, trans_a, trans_b, skinny, maxM, maxN, count, dd, mode,
                                       splits, ws, slot);
  else if (ta == DType::F64 && tb == DType::F64) {
    if (skinny)
      launch64<128, 32>(ctx, trans_a, trans_b, dim3(ceil_div(maxM, 128), ceil_div(maxN, 32),
                                                    count * splits),
                        dd, mode, splits, ws, slot);
    else
      launch64<64, 64>(ctx, trans_a, trans_b, dim3(ceil_div(maxM, 64), ceil_div(maxN, 64),
                                                   count * splits),
                       dd, mode, splits, ws, slot);
  }
  else if (ta == DType::F32 && tb == DType::F64)
    launch_typed<float, double, false>(ctx, trans_a, trans_b, skinny, maxM, maxN, count, dd, mode,
                                splits, ws, slot);
  else if (ta == DType::F64 && tb == DType::F32)
    launch_typed<double, float, false>(ctx, trans_a, trans_b, skinny, maxM, maxN, count, dd, mode,
                                splits, ws, slot);
  else
    launch_typed<float, float, false>(ctx, trans_a, trans_b, skinny, maxM, maxN, count, dd, mode, splits,
                               ws, slot);
  if (splits > 1) {
    const long long elems = (long long)maxM * maxN;
    int bx = static_cast<int>(std::min<long long>((elems + 255) / 256, 4096));
    ctx.launch_begin();
    k_splitk_reduce<<<dim3(bx, count), 256, 0, ctx.stream>>>(dd, splits, mode, ws, slot);
    ctx.check_launch("k_splitk_reduce");
  }
  ctx.arena.release(mk);
}

}  // namespace hsvdcu
