// Grouped fp64 GEMM for the HSVD path on sm_100a.
//
// Every contraction of the hot path (block Grams X_b^T X_b, projections
// X_b Z, V-recovery X_j^T U_j, U-recovery X V_r, merge Grams/projections,
// the two-stage band reduction and the blocked Householder back-transforms)
// runs through this kernel.  The reference computes all of them in IEEE
// binary64 (Eigen, dense_matrix.hpp:9); tcgen05.mma has no f64 kind, so the
// fp64-exact tensor path on B200 is DMMA (mma.sync.m8n8k4.f64 -> SASS
// DMMA.8x8x4).  fp32 operands (the BASELINE matrices) are copied as fp32 and
// promoted to fp64 when the DMMA fragments are read from shared memory,
// which is exactly what the reference's fp64 DenseMatrix computes on the
// same bytes (and halves their shared-memory and copy footprint).
//
// Operands go global -> shared memory by cp.async (LDGSTS, zero-filled out
// of bounds) in a 3-stage pipeline, no register staging; each operand tile
// keeps the memory-contiguous dimension contiguous in shared memory, so the
// copies are coalesced and the fragment reads conflict-free.  Tiles: 64x64
// (2x2 warps) or, for skinny outputs (N <= 32), 128x32 (4x1 warps); each
// warp owns 32x32 = 4x4 DMMA tiles; BK = 16, 3 stages (skinny: 2).  C reads are batched before the
// stores.  Split-K (chosen against the wave count of the resident CTA slots)
// with a deterministic fixed-order reduction
// (run-to-run bitwise stable).  SYRK mode computes the lower tile
// triangle and mirrors it through a shared-memory transpose (or not, with
// kGemmLowerOnly).
#include <algorithm>
#include <atomic>

#include "gemm.h"

namespace hsvdcu {

namespace {

constexpr int NT = 128;

// k depth and pipeline stages per tile shape.  The skinny 128x32 tile
// streams a large A against a small B and is bound by resident warps (4 CTAs
// per SM at 128 registers): double buffering keeps its shared memory small
// (measured on the config-2 Y = A22 V launches: BK/stages 16/3 -> 37.4 ms,
// 8/4 -> 33.5, 16/2 -> 32.2; forcing 5-6 CTAs per SM spills and loses).
template <int BM, int BN>
struct TileCfg {
  static constexpr int BK = 16, STAGES = 3;
};
template <>
struct TileCfg<128, 32> {
  static constexpr int BK = 16, STAGES = 2;
};
constexpr int kModeSyrk = 1, kModeLower = 2;  // mode bits

// Up to kPackMax descriptors travel in the launch parameters (read from the
// constant bank); larger groups go through the staging ring.
constexpr int kPackMax = 64;
struct DescPack {
  GemmDesc d[kPackMax];
};

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <typename T>
__device__ __forceinline__ void cp_async(T* dst, const T* src, bool ok) {
  static_assert(sizeof(T) == 4 || sizeof(T) == 8, "cp.async element");
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(d), "l"(src),
               "n"(sizeof(T)), "r"(ok ? (int)sizeof(T) : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// Shared layout of one operand tile (R rows of the output dimension, BK of
// k): KF (k contiguous in memory) -> [R][BK + 4]; else [BK][R + pad] with
// the pad chosen so a warp's 8x4 fragment reads hit distinct banks.
template <typename T, int R, bool KF, int BK>
struct OpTile {
  static constexpr int PAD = sizeof(T) == 4 ? 8 : 4;
  static constexpr int LD = KF ? BK + 4 : R + PAD;
  static constexpr int ELEMS = KF ? R * (BK + 4) : BK * (R + PAD);
  static constexpr size_t BYTES = ((size_t)ELEMS * sizeof(T) + 15) / 16 * 16;
  __device__ static int at(int r, int k) { return KF ? r * LD + k : k * LD + r; }
};

template <typename TA, typename TB, bool TRA, bool TRB, int BM, int BN>
struct GemmShape {
  static constexpr int BK = TileCfg<BM, BN>::BK, STAGES = TileCfg<BM, BN>::STAGES;
  using TAt = OpTile<TA, BM, TRA, BK>;
  using TBt = OpTile<TB, BN, !TRB, BK>;
  static constexpr size_t STAGE_BYTES = TAt::BYTES + TBt::BYTES;
  static constexpr size_t TILE_BYTES = (size_t)BM * (BN + 1) * sizeof(double);  // mirror staging
  static constexpr size_t SMEM =
      STAGES * STAGE_BYTES > TILE_BYTES ? STAGES * STAGE_BYTES : TILE_BYTES;
};

template <typename TA, typename TB, bool TRA, bool TRB, int BM, int BN>
__global__ void __launch_bounds__(NT) k_gemm(const GemmDesc* __restrict__ descs, int mode,
                                             int splits, double* __restrict__ ws,
                                             long long ws_slot, const __grid_constant__ DescPack pack) {
  // A element (m, k): !TRA -> A[m + k lda] (m contiguous), TRA -> A[k + m lda]
  // B element (k, n): !TRB -> B[k + n ldb] (k contiguous), TRB -> B[n + k ldb]
  using Sh = GemmShape<TA, TB, TRA, TRB, BM, BN>;
  using TAt = typename Sh::TAt;
  using TBt = typename Sh::TBt;
  constexpr int BK = Sh::BK, STAGES = Sh::STAGES;
  constexpr int WN = BN / 32;
  constexpr int LA = BM * BK / NT, LB = BN * BK / NT;
  extern __shared__ __align__(16) unsigned char smem[];

  const int g = blockIdx.z / splits;
  const int split = blockIdx.z - g * splits;
  const GemmDesc d = descs ? descs[g] : pack.d[g];
  const int tm = blockIdx.x, tn = blockIdx.y;
  if (tm * BM >= d.M || tn * BN >= d.N) return;
  const bool syrk = (mode & kModeSyrk) != 0;
  if (syrk && tn * BN >= (tm + 1) * BM) return;  // strictly upper tile
  int kchunk = (d.K + splits - 1) / splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  const int kb = split * kchunk;
  const int ke = min(d.K, kb + kchunk);
  const int nkt = ke > kb ? (ke - kb + BK - 1) / BK : 0;

  const TA* A = static_cast<const TA*>(d.A);
  const TB* B = static_cast<const TB*>(d.B);
  const int tid = threadIdx.x;
  const int m0 = tm * BM, n0 = tn * BN;
  auto a_tile = [&](int s) {
    return reinterpret_cast<TA*>(smem + (size_t)s * Sh::STAGE_BYTES);
  };
  auto b_tile = [&](int s) {
    return reinterpret_cast<TB*>(smem + (size_t)s * Sh::STAGE_BYTES + TAt::BYTES);
  };

  // element e = tid + i*NT of a tile, the memory-contiguous dimension fastest
  auto issue = [&](int kt) {
    TA* As = a_tile(kt % STAGES);
    TB* Bs = b_tile(kt % STAGES);
    const int k0 = kb + kt * BK;
#pragma unroll
    for (int i = 0; i < LA; ++i) {
      const int e = tid + i * NT;
      const int r = TRA ? e / BK : e % BM, k = TRA ? e % BK : e / BM;
      const int gm = m0 + r, gk = k0 + k;
      const bool ok = gm < d.M && gk < ke;
      const TA* src = ok ? (TRA ? A + (long long)gk + (long long)gm * d.lda
                                : A + (long long)gm + (long long)gk * d.lda)
                         : A;
      cp_async(As + TAt::at(r, k), src, ok);
    }
#pragma unroll
    for (int i = 0; i < LB; ++i) {
      const int e = tid + i * NT;
      const int r = TRB ? e % BN : e / BK, k = TRB ? e / BN : e % BK;
      const int gn = n0 + r, gk = k0 + k;
      const bool ok = gn < d.N && gk < ke;
      const TB* src = ok ? (TRB ? B + (long long)gn + (long long)gk * d.ldb
                                : B + (long long)gk + (long long)gn * d.ldb)
                         : B;
      cp_async(Bs + TBt::at(r, k), src, ok);
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
    const TA* As = a_tile(kt % STAGES);
    const TB* Bs = b_tile(kt % STAGES);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = static_cast<double>(As[TAt::at(wm + i * 8 + grp, kk + tig)]);
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = static_cast<double>(Bs[TBt::at(wn + j * 8 + grp, kk + tig)]);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
    }
  }
  cp_async_wait<0>();

  // epilogue: direct store (each warp instruction writes 4 columns x 8
  // consecutive rows); the SYRK mirror of an off-diagonal tile reuses the
  // final values staged in shared memory so the transposed store is coalesced
  const bool to_ws = ws != nullptr;
  double* out = to_ws ? ws + (long long)blockIdx.z * ws_slot : d.C;
  const long long ldo = to_ws ? (long long)d.M : d.ldc;
  const double alpha = d.alpha, beta = d.beta;
  const bool diag_tile = n0 < m0 + BM && m0 < n0 + BN;
  const bool mirror = syrk && !(mode & kModeLower) && !to_ws && !diag_tile;
  constexpr int T_LD = BN + 1;
  double* tile = reinterpret_cast<double*>(smem);
  if (mirror) __syncthreads();  // operand tiles no longer read
  // all C reads issued before any store (the stores could alias them, so the
  // compiler would otherwise serialise load -> store pairs)
  if (!to_ws) {
    const bool rd = beta != 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int m = m0 + wm + i * 8 + grp, n = n0 + wn + j * 8 + 2 * tig + r;
          const double c = (rd && m < d.M && n < d.N) ? out[m + (long long)n * ldo] : 0.0;
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

__global__ void k_splitk_reduce(const GemmDesc* __restrict__ descs, int splits, int mode,
                                const double* __restrict__ ws, long long ws_slot,
                                const __grid_constant__ DescPack pack) {
  const int g = blockIdx.y;
  const GemmDesc d = descs ? descs[g] : pack.d[g];
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

template <typename TA, typename TB, bool TRA, bool TRB, int BM, int BN>
void launch_t(Ctx& ctx, dim3 grid, const GemmDesc* dd, int mode, int splits, double* ws,
              long long slot, const DescPack& pack) {
  constexpr size_t smem = GemmShape<TA, TB, TRA, TRB, BM, BN>::SMEM;
  auto* k = k_gemm<TA, TB, TRA, TRB, BM, BN>;
  smem_optin(k, smem);
  k<<<grid, NT, smem, ctx.stream>>>(dd, mode, splits, ws, slot, pack);
}

template <typename TA, typename TB, int BM, int BN>
void launch_tile(Ctx& ctx, bool ta, bool tb, dim3 grid, const GemmDesc* dd, int mode, int splits,
                 double* ws, long long slot, const DescPack& pack) {
  ctx.launch_begin();
  if (!ta && !tb) launch_t<TA, TB, false, false, BM, BN>(ctx, grid, dd, mode, splits, ws, slot, pack);
  else if (!ta && tb) launch_t<TA, TB, false, true, BM, BN>(ctx, grid, dd, mode, splits, ws, slot, pack);
  else if (ta && !tb) launch_t<TA, TB, true, false, BM, BN>(ctx, grid, dd, mode, splits, ws, slot, pack);
  else launch_t<TA, TB, true, true, BM, BN>(ctx, grid, dd, mode, splits, ws, slot, pack);
  ctx.check_launch("k_gemm");
}

// Resident CTAs per SM of one instantiation (cached: every device of a run
// is the same B200 part).
template <typename TA, typename TB, bool TRA, bool TRB, int BM, int BN>
int occupancy_t() {
  static std::atomic<int> cached{0};
  int occ = cached.load(std::memory_order_relaxed);
  if (occ > 0) return occ;
  constexpr size_t smem = GemmShape<TA, TB, TRA, TRB, BM, BN>::SMEM;
  auto* k = k_gemm<TA, TB, TRA, TRB, BM, BN>;
  smem_optin(k, smem);
  HSVD_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NT, smem));
  occ = std::max(1, occ);
  cached.store(occ, std::memory_order_relaxed);
  return occ;
}

template <typename TA, typename TB, int BM, int BN>
int occupancy_tile(bool ta, bool tb) {
  if (!ta && !tb) return occupancy_t<TA, TB, false, false, BM, BN>();
  if (!ta && tb) return occupancy_t<TA, TB, false, true, BM, BN>();
  if (ta && !tb) return occupancy_t<TA, TB, true, false, BM, BN>();
  return occupancy_t<TA, TB, true, true, BM, BN>();
}

template <typename TA, typename TB>
int occupancy_typed(bool ta, bool tb, bool skinny) {
  return skinny ? occupancy_tile<TA, TB, 128, 32>(ta, tb) : occupancy_tile<TA, TB, 64, 64>(ta, tb);
}

int occupancy(DType a, DType b, bool ta, bool tb, bool skinny) {
  if (a == DType::F64 && b == DType::F64) return occupancy_typed<double, double>(ta, tb, skinny);
  if (a == DType::F32 && b == DType::F64) return occupancy_typed<float, double>(ta, tb, skinny);
  if (a == DType::F64 && b == DType::F32) return occupancy_typed<double, float>(ta, tb, skinny);
  return occupancy_typed<float, float>(ta, tb, skinny);
}

// Split-K factor: minimises (waves of CTAs) x (K per CTA + a fixed
// prologue/epilogue cost), so a grid that would leave most of its last wave
// empty is split instead (K per split >= 128; one extra cost unit for the
// reduction launch).
int choose_splits(long long tiles, int maxK, long long slots, int count) {
  constexpr double kFixed = 64.0;
  const int smax = std::min(128, maxK / 128);
  int best = 1;
  double best_cost = (double)((tiles + slots - 1) / slots) * (maxK + kFixed);
  for (int s = 2; s <= smax; ++s) {
    if ((long long)count * s > 65535) break;
    const double waves = (double)((tiles * s + slots - 1) / slots);
    const double cost = waves * ((double)maxK / s + kFixed) + kFixed;
    if (cost < best_cost * 0.97) {
      best_cost = cost;
      best = s;
    }
  }
  return best;
}

template <typename TA, typename TB>
void launch_typed(Ctx& ctx, bool ta, bool tb, bool skinny, int maxM, int maxN, int count,
                  const GemmDesc* dd, int mode, int splits, double* ws, long long slot,
                  const DescPack& pack) {
  if (skinny) {
    dim3 grid(ceil_div(maxM, 128), ceil_div(maxN, 32), count * splits);
    launch_tile<TA, TB, 128, 32>(ctx, ta, tb, grid, dd, mode, splits, ws, slot, pack);
  } else {
    dim3 grid(ceil_div(maxM, 64), ceil_div(maxN, 64), count * splits);
    launch_tile<TA, TB, 64, 64>(ctx, ta, tb, grid, dd, mode, splits, ws, slot, pack);
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
  if (ta == DType::F64 && tb == DType::F64 && !trans_a && !trans_b && !syrk &&
      gemm_sk_applicable(live, ctx.num_sms)) {
    gemm_sk(ctx, live);
    return;
  }
  const int count = static_cast<int>(live.size());
  if (count > 65535) throw Error(kInvalid, "gemm_grouped: too many groups");
  const bool skinny = !syrk && maxN <= 32;
  const int BMt = skinny ? 128 : 64, BNt = skinny ? 32 : 64;
  long long tiles = 0;
  double flops = 0.0;  // algorithmic (SYRK: the lower triangle)
  double bytes = 0.0;
  for (const auto& d : live) {
    long long t = (long long)ceil_div(d.M, BMt) * ceil_div(d.N, BNt);
    if (syrk) t = (t + ceil_div(d.M, BMt)) / 2;
    tiles += t;
    flops += syrk ? (double)d.M * (d.M + 1) * d.K : 2.0 * d.M * d.N * d.K;
    // algorithmic HBM bytes: each operand once (SYRK: op(A) only), C written
    // (and read when beta != 0)
    const double sa = ta == DType::F64 ? 8.0 : 4.0, sb = tb == DType::F64 ? 8.0 : 4.0;
    bytes += sa * d.M * d.K + (syrk ? 0.0 : sb * d.K * d.N) +
             8.0 * d.M * d.N * (d.beta != 0.0 ? 2.0 : 1.0);
  }

  const long long slots = (long long)ctx.num_sms * occupancy(ta, tb, trans_a, trans_b, skinny);
  const int splits = choose_splits(tiles, maxK, slots, count);
  // descriptors: in the launch parameters when they fit, else staged
  static thread_local DescPack pack;
  const GemmDesc* dd = nullptr;
  if (count <= kPackMax)
    std::copy(live.begin(), live.end(), pack.d);
  else
    dd = static_cast<const GemmDesc*>(ctx.staging.put(live.data(), live.size() * sizeof(GemmDesc),
                                                      ctx.stream));
  double* ws = nullptr;
  long long slot = 0;
  Arena::Mark mk = ctx.arena.mark();
  if (splits > 1) {
    slot = (long long)maxM * maxN;
    ws = ctx.arena.alloc_n<double>((size_t)slot * count * splits);
  }
  const int mode = (syrk ? kModeSyrk : 0) | ((flags & kGemmLowerOnly) ? kModeLower : 0);
  ctx.pending_flops = flops;
  ctx.pending_bytes = bytes;
  if (ta == DType::F64 && tb == DType::F64)
    launch_typed<double, double>(ctx, trans_a, trans_b, skinny, maxM, maxN, count, dd, mode,
                                 splits, ws, slot, pack);
  else if (ta == DType::F32 && tb == DType::F64)
    launch_typed<float, double>(ctx, trans_a, trans_b, skinny, maxM, maxN, count, dd, mode,
                                splits, ws, slot, pack);
  else if (ta == DType::F64 && tb == DType::F32)
    launch_typed<double, float>(ctx, trans_a, trans_b, skinny, maxM, maxN, count, dd, mode,
                                splits, ws, slot, pack);
  else
    launch_typed<float, float>(ctx, trans_a, trans_b, skinny, maxM, maxN, count, dd, mode, splits,
                               ws, slot, pack);
  if (splits > 1) {
    const long long elems = (long long)maxM * maxN;
    int bx = static_cast<int>(std::min<long long>((elems + 255) / 256, 4096));
    ctx.launch_begin();
    k_splitk_reduce<<<dim3(bx, count), 256, 0, ctx.stream>>>(dd, splits, mode, ws, slot, pack);
    ctx.check_launch("k_splitk_reduce");
  }
  ctx.arena.release(mk);
}

}  // namespace hsvdcu
