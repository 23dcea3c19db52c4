// Skinny fp64 GEMM fed by bulk copies: C (M x N<=32) = alpha A B + beta C,
// A (M x K) and B (K x N) column-major -- the stage-1 Y = A22 V of the
// two-stage eigensolver (syev_band.cu) and its pending-pair corrections.
//
// The grouped k_gemm (gemm.cu) loads its tiles with per-thread cp.async of
// one element each (LDGSTS.E.64): 20 copy instructions per thread per k-step
// next to 64 DMMAs per warp.  Here one producer warp moves the A tile with
// cp.async.bulk (the 1-D TMA): every column of the 128 x 16 A tile is one
// contiguous 1 KB copy completing on an mbarrier with a transaction count;
// four consumer warps (32 x 32 each, 4 x 4 DMMA.8x8x4 per k4) read the A
// fragments from shared memory (column stride padded by 4 doubles:
// conflict-free) and the small, L2-resident B fragments straight from
// global memory, and release a stage with one arrive per warp.  4 stages,
// 68 KB, two CTAs per SM.  Measured on B200 (round 2): config 2's Y = A22 V
// 33.3 -> 31.6 ms, config 5's 459 -> 463 ms (parity).  Also measured and
// rejected: copying the 16 x 32 B tile too (32 more 128-byte copies per
// stage made the single producer thread the bottleneck: 459 -> 588 ms at
// config 5), and 256-row tiles with 8 consumer warps (register-capped at
// two CTAs per SM, spills: 726 ms).
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "gemm.h"
#include "ozaki_tc.cuh"

namespace hsvdcu {

namespace {

using namespace oztc;

constexpr int SK_BM = 128, SK_BN = 32, SK_BK = 16, SK_ST = 4;
constexpr int SK_CW = SK_BM / 32;                 // consumer warps
constexpr int SK_LDA = SK_BM + 4;                 // A tile column stride (doubles)
constexpr int SK_LDB = SK_BK + 4;                 // B tile column stride (doubles)
constexpr int SK_ABYTES = SK_BK * SK_LDA * 8;     // 16896
constexpr int SK_STAGE = SK_ABYTES;              // B fragments come straight from L2
constexpr int SK_THREADS = (SK_CW + 1) * 32;      // consumer warps + 1 producer
constexpr size_t SK_SMEM = (size_t)SK_ST * SK_STAGE + 128;
static_assert(SK_STAGE % 16 == 0, "bulk copy destinations");

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void dmma_sk(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(SK_THREADS, 2) k_gemm_sk(const GemmDesc* __restrict__ descs) {
  const GemmDesc d = descs[blockIdx.y];
  const int m0 = blockIdx.x * SK_BM;
  if (m0 >= d.M) return;
  extern __shared__ __align__(128) unsigned char sk_smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sk_smem + SK_ST * SK_STAGE);
  uint64_t* empty = full + SK_ST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < SK_ST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], SK_CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const double* A = static_cast<const double*>(d.A);
  const double* B = static_cast<const double*>(d.B);
  const int nkt = (d.K + SK_BK - 1) / SK_BK;
  const int rows = min(SK_BM, d.M - m0);
  const int ncols = min(SK_BN, d.N);
  if (warp == SK_CW) {
    // ---------------- producer ----------------
    if (lane == 0) {
      for (int kt = 0; kt < nkt; ++kt) {
        const int s = kt % SK_ST;
        if (kt >= SK_ST) mbar_wait(&empty[s], ((kt / SK_ST) & 1) ^ 1);
        const int k0 = kt * SK_BK, kc = min(SK_BK, d.K - k0);
        unsigned char* st = sk_smem + (size_t)s * SK_STAGE;
        double* As = reinterpret_cast<double*>(st);
        mbar_expect_tx(&full[s], (uint32_t)(kc * rows) * 8u);
        for (int k = 0; k < kc; ++k)
          bulk_g2s(As + k * SK_LDA, A + m0 + (long long)(k0 + k) * d.lda, (uint32_t)rows * 8u, &full[s]);
      }
    }
    return;
  }
  // ---------------- consumers: warp w owns rows 32w .. 32w+31 ----------------
  const int g = lane >> 2, t = lane & 3;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int kt = 0; kt < nkt; ++kt) {
    const int s = kt % SK_ST;
    mbar_wait(&full[s], (kt / SK_ST) & 1);
    const int kc = min(SK_BK, d.K - kt * SK_BK);
    const double* As = reinterpret_cast<const double*>(sk_smem + (size_t)s * SK_STAGE);
#pragma unroll
    for (int kk = 0; kk < SK_BK; kk += 4) {
      const int k = kk + t;
      const bool ok = k < kc;  // past K: stale shared memory, both factors zeroed
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = ok ? As[k * SK_LDA + warp * 32 + i * 8 + g] : 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        b[j] = (ok && j * 8 + g < ncols) ? __ldg(B + kt * SK_BK + k + (long long)(j * 8 + g) * d.ldb) : 0.0;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_sk(acc[i][j], a[i], b[j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  // epilogue (rows past M and columns past N hold stale-operand values: dropped)
  double cold[4][4][2];
  const bool rd = d.beta != 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = m0 + warp * 32 + i * 8 + g, c = j * 8 + 2 * t + h;
        cold[i][j][h] = (rd && r < d.M && c < d.N) ? d.C[r + (long long)c * d.ldc] : 0.0;
      }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = m0 + warp * 32 + i * 8 + g, c = j * 8 + 2 * t + h;
        if (r < d.M && c < d.N)
          d.C[r + (long long)c * d.ldc] = d.alpha * acc[i][j][h] + (rd ? d.beta * cold[i][j][h] : 0.0);
      }
}

}  // namespace

bool gemm_sk_applicable(const std::vector<GemmDesc>& descs, int num_sms) {
  const char* e = std::getenv("HSVD_GEMM_SK");
  if (e && std::atoi(e) == 0) return false;
  long long ctas = 0;
  for (const GemmDesc& d : descs) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(d.A), b = reinterpret_cast<uintptr_t>(d.B);
    // bulk copies: 16-byte aligned sources and sizes (even M, K, lda, ldb)
    if (d.N > SK_BN || d.M % 2 || d.K % 2 || d.lda % 2 || d.ldb % 2 || (a & 15) || (b & 15) ||
        d.K < 4 * SK_BK)
      return false;
    ctas += (d.M + SK_BM - 1) / SK_BM;
  }
  return ctas >= 2LL * num_sms;  // enough CTAs without split-K
}

void gemm_sk(Ctx& ctx, const std::vector<GemmDesc>& descs) {
  int maxM = 0;
  double flops = 0.0, bytes = 0.0;  // algorithmic flops and HBM bytes (profile)
  for (const GemmDesc& d : descs) {
    maxM = std::max(maxM, d.M);
    flops += 2.0 * d.M * d.N * d.K;
    bytes += 8.0 * ((double)d.M * d.K + (double)d.K * d.N + (double)d.M * d.N * (d.beta != 0.0 ? 2.0 : 1.0));
  }
  const GemmDesc* dd = static_cast<const GemmDesc*>(
      ctx.staging.put(descs.data(), descs.size() * sizeof(GemmDesc), ctx.stream));
  smem_optin(k_gemm_sk, SK_SMEM);
  ctx.pending_flops = flops;
  ctx.pending_bytes = bytes;
  ctx.launch_begin();
  k_gemm_sk<<<dim3(ceil_div(maxM, SK_BM), (unsigned)descs.size()), SK_THREADS, SK_SMEM, ctx.stream>>>(dd);
  ctx.check_launch("k_gemm_sk");
}

}  // namespace hsvdcu
