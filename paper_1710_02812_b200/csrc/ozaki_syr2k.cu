// Stage-1 trailing update of the two-stage eigensolver on the 5th-generation
// tensor cores: A22 -= V W^T + W V^T (the delayed SYR2K of syev_band.cu,
// K = 32 reflectors x up to 4 panels) in fp64-grade arithmetic from int8
// Ozaki slices -- the same scheme as the leaf Gram (ozaki_gram.cu).
//
// The pending pairs arrive as VW = [V_1 W_1 V_2 W_2 ...] (column-major,
// 64 columns per panel); WV is its panel-swapped copy, so
// VW WV^T = V W^T + W V^T with V, W the stacked m x 32p blocks.  V (entries
// O(1)) and W (entries O(|A|)) get separate per-row power-of-two scales, so
// the update is two products with their own scales ("segments"):
//   C_ij -= sV_i sW_j (V^_i . W^_j) + sW_i sV_j (W^_i . V^_j),
// each digit-sliced into 7 int8 planes (x / s = sum_a D_a 2^-(6+7(a-1)),
// D_a in [-64, 64]) and accumulated exactly per level t = a + b in int32
// (|sum| <= 7 * 128 * 64^2 < 2^31); products with a + b > 8 (weight
// <= 2^-54) are dropped, as in the Gram.  The error per element is then
// ~K 2^-49 max|V_i| max|W_j|: normwise within a small factor of an fp64
// GEMM's, which is what the backward stability of the reduction needs.
//
// Status: correct (tests/test_gpu_eig.py with HSVD_SYR2K=ozaki) but slower
// than the DMMA SYR2K it would replace, so opt-in only (see
// ozaki_syr2k_applicable).
//
// k_oz_split_vw  VW rows -> per-row scales and 2 x 7 digit planes (K-major,
//                128 bytes per row = 4 panels x 32 reflectors, zero padded)
// k_oz_syr2k     one CTA per 128 x 32 tile of the lower triangle of one
//                matrix's A22 (2 CTAs per SM: 104 KB of shared memory and
//                256 TMEM columns each): warp 0 loads the 7 B planes of the
//                tile's 32 columns once per segment and streams the 7 A
//                planes of its 128 rows through a 3-stage ring (TMA, 128B
//                swizzle); warp 1 issues the 28 products per segment
//                (tcgen05.mma kind::i8, M = 128, N = 32, K = 32) into 7
//                level accumulators (7 x 32 TMEM columns); warps 2-5 drain
//                the levels (tcgen05.ld), recombine them in fp64 with the
//                segment's scales, and after both segments update C (read,
//                subtract, store) and its mirror image in the upper triangle.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ozaki.h"
#include "ozaki_tc.cuh"

namespace hsvdcu {

namespace {

using namespace oztc;

constexpr int kS = 7;
constexpr int TM = 128;                 // tile rows (TMEM lanes)
constexpr int TN = 32;                  // tile columns
constexpr int KB = 128;                 // K bytes per plane row (4 panels x 32)
constexpr int kABytes = TM * KB;        // 16 KB
constexpr int kBBytes = TN * KB;        // 4 KB
constexpr int kAStages = 3;
constexpr int kThreads = 192;
constexpr int kTmemCols = 256;          // 7 levels x 32 columns used
constexpr size_t kSmem = (size_t)2 * kS * kBBytes + (size_t)kAStages * kABytes + 1024 + 256;

struct SyRows {  // slicing source
  const double* vw;
  long long ldv;
  int m, K;
  long long prow;  // first plane row of the job ([seg][plane][mpad] rows)
  int mpad;
  double* sc;      // [2][mpad] row scales
};

struct SyJob {
  double* C;
  long long ldc;
  int m, mpad;
  long long prow;
  const double* sc;
  int mt, nt;
};

// Thread (r, g): row blockIdx.x*32 + r, VW columns 32g .. 32g+31 (g even: V
// of panel g/2, odd: W).  Loads are coalesced over r.
__global__ void __launch_bounds__(256) k_oz_split_vw(const SyRows* __restrict__ srcs,
                                                     signed char* __restrict__ planes) {
  __shared__ double red[2][4][32];
  const SyRows S = srcs[blockIdx.y];
  const int r = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int row = blockIdx.x * 32 + r;
  if (blockIdx.x * 32 >= S.mpad) return;
  const int seg = g & 1, p = g >> 1;
  const bool present = row < S.m && 64 * p < S.K;
  const double* src = S.vw + row + (long long)(64 * p + 32 * seg) * S.ldv;
  double x[32];
  double mx = 0.0;
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    x[q] = present ? src[(long long)q * S.ldv] : 0.0;
    mx = fmax(mx, fabs(x[q]));
  }
  red[seg][p][r] = mx;
  __syncthreads();
  mx = fmax(fmax(red[seg][0][r], red[seg][1][r]), fmax(red[seg][2][r], red[seg][3][r]));
  int e = 0;
  if (mx > 0.0) frexp(mx, &e);  // mx < 2^e
  const double scale = mx > 0.0 ? ldexp(1.0, e) : 1.0;
  if (p == 0 && row < S.mpad) S.sc[(long long)seg * S.mpad + row] = scale;
  const double inv = 1.0 / scale;  // exact
  uint32_t packed[kS][8];
#pragma unroll
  for (int a = 0; a < kS; ++a)
#pragma unroll
    for (int w = 0; w < 8; ++w) packed[a][w] = 0u;
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    double v = x[q] * inv * 64.0;
#pragma unroll
    for (int a = 0; a < kS; ++a) {
      const double d = rint(v);
      v = (v - d) * 128.0;
      packed[a][q >> 2] |= (uint32_t)(uint8_t)(signed char)(int)d << (8 * (q & 3));
    }
  }
#pragma unroll
  for (int a = 0; a < kS; ++a) {
    uint4* dst = reinterpret_cast<uint4*>(
        planes + (S.prow + (long long)(seg * kS + a) * S.mpad + row) * KB + 32 * p);
    dst[0] = make_uint4(packed[a][0], packed[a][1], packed[a][2], packed[a][3]);
    dst[1] = make_uint4(packed[a][4], packed[a][5], packed[a][6], packed[a][7]);
  }
}

__global__ void __launch_bounds__(kThreads, 2)
    k_oz_syr2k(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const SyJob* __restrict__ jobs) {
  const SyJob J = jobs[blockIdx.y];
  // tile (mb, nb) of the lower triangle: nb*TN <= mb*TM + TM - 1
  int idx = blockIdx.x, mb = 0;
  for (; mb < J.mt; ++mb) {
    const int cnt = min(J.nt, (mb * TM + TM - 1) / TN + 1);
    if (idx < cnt) break;
    idx -= cnt;
  }
  if (mb >= J.mt) return;
  const int nb = idx;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* bbuf = smem;                                  // [2 seg][kS][4 KB]
  uint8_t* aring = smem + 2 * kS * kBBytes;              // [kAStages][16 KB]
  uint64_t* afull = reinterpret_cast<uint64_t*>(aring + kAStages * kABytes);
  uint64_t* aempty = afull + kAStages;
  uint64_t* bfull = aempty + kAStages;  // [2]
  uint64_t* tfull = bfull + 2;
  uint64_t* tempty = tfull + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kAStages; ++s) {
      mbar_init(&afull[s], 1);
      mbar_init(&aempty[s], 1);
    }
    mbar_init(&bfull[0], 1);
    mbar_init(&bfull[1], 1);
    mbar_init(tfull, 1);
    mbar_init(tempty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int seg = 0; seg < 2; ++seg) {
        const int segB = 1 - seg;  // seg 0: V rows x W columns; seg 1: W rows x V columns
        mbar_expect_tx(&bfull[seg], kS * kBBytes);
        for (int b = 0; b < kS; ++b)
          tma_load_2d(bbuf + (seg * kS + b) * kBBytes, &tmB, 0,
                      (int)(J.prow + (long long)(segB * kS + b) * J.mpad + nb * TN), &bfull[seg]);
        for (int a = 0; a < kS; ++a) {
          mbar_wait(&aempty[stage], phase ^ 1);
          mbar_expect_tx(&afull[stage], kABytes);
          tma_load_2d(aring + stage * kABytes, &tmA, 0,
                      (int)(J.prow + (long long)(seg * kS + a) * J.mpad + mb * TM), &afull[stage]);
          if (++stage == kAStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int seg = 0; seg < 2; ++seg) {
        if (seg == 1) mbar_wait(tempty, 0);  // segment 0's levels drained
        mbar_wait(&bfull[seg], 0);
        tc_fence_after();
        uint32_t init = 0;
        for (int a = 1; a <= kS; ++a) {
          mbar_wait(&afull[stage], phase);
          tc_fence_after();
          const uint64_t ad = umma_desc(smem_u32(aring + stage * kABytes));
          for (int b = 1; a + b <= kS + 1; ++b) {
            const int lvl = a + b - 2;
            const uint64_t bd = umma_desc(smem_u32(bbuf + (seg * kS + b - 1) * kBBytes));
            const uint32_t d = tmem + lvl * TN;
#pragma unroll
            for (int k = 0; k < KB / 32; ++k)
              mma_i8<idesc_i8(TM, TN)>(d, ad + 2 * k, bd + 2 * k,
                                       (k > 0 || ((init >> lvl) & 1u)) ? 1u : 0u);
            init |= 1u << lvl;
          }
          mma_commit(&aempty[stage]);
          if (++stage == kAStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(tfull);
      }
    }
  } else {
    // ---------------- epilogue ----------------
    const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31 (warp % 4 rule)
    const int r = quarter * 32 + lane;
    const int i = mb * TM + r;  // row of C
    double tot[TN];
#pragma unroll
    for (int c = 0; c < TN; ++c) tot[c] = 0.0;
    for (int seg = 0; seg < 2; ++seg) {
      const int segB = 1 - seg;
      mbar_wait(tfull, seg);
      tc_fence_after();
      double acc[TN];
#pragma unroll
      for (int c = 0; c < TN; ++c) acc[c] = 0.0;
#pragma unroll 1
      for (int t = 0; t < kS; ++t) {  // most significant level first (fixed order)
        int v[32];
        tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + t * TN, v);
        const double w = ldexp(1.0, -(12 + 7 * t));
#pragma unroll
        for (int c = 0; c < TN; ++c) acc[c] += (double)v[c] * w;
      }
      tc_fence_before();
      __syncwarp();
      if (seg == 0 && lane == 0) mbar_arrive(tempty);
      const double sa = J.sc[(long long)seg * J.mpad + i];
      const double* sb = J.sc + (long long)segB * J.mpad + nb * TN;
#pragma unroll
      for (int c = 0; c < TN; ++c) tot[c] += sa * sb[c] * acc[c];
    }
    if (i < J.m) {
      // every C read issued before any store (the mirror stores could alias
      // them, so the compiler would otherwise serialise load -> store pairs)
      double* Crow = J.C + i;
      const int jn = min(TN, min(i + 1, J.m) - nb * TN);  // columns j <= i, j < m
      double cv[TN];
#pragma unroll
      for (int c = 0; c < TN; ++c) cv[c] = c < jn ? __ldcg(Crow + (long long)(nb * TN + c) * J.ldc) : 0.0;
#pragma unroll
      for (int c = 0; c < TN; ++c) {
        const int j = nb * TN + c;
        if (c < jn) {
          const double cij = cv[c] - tot[c];
          Crow[(long long)j * J.ldc] = cij;
          if (j < i) J.C[j + (long long)i * J.ldc] = cij;  // mirror (full symmetric storage)
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

CUtensorMap plane_map(signed char* planes, long long rows, int box_rows) {
  CUtensorMap tmap;
  const cuuint64_t gdim[2] = {(cuuint64_t)KB, (cuuint64_t)rows};
  const cuuint64_t gstride[1] = {(cuuint64_t)KB};
  const cuuint32_t box[2] = {(cuuint32_t)KB, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult cr = encode_fn()(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, planes, gdim, gstride, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) throw Error(kCuda, "cuTensorMapEncodeTiled failed");
  return tmap;
}

template <typename T>
T* stage_table(Ctx& ctx, const std::vector<T>& v) {
  return static_cast<T*>(ctx.staging.put_to(ctx.arena.alloc(v.size() * sizeof(T)), v.data(),
                                            v.size() * sizeof(T), ctx.stream));
}

constexpr size_t kPlaneBudget = size_t(4) << 30;

}  // namespace

// Opt-in (HSVD_SYR2K=ozaki).  Measured on B200 (round 2): slower than the
// DMMA SYR2K -- config 5: 571 ms against 412, config 2: 34.4 against 25.5 ms.
// ncu (profiles/r02j_syr2k.md): tensor pipe ~10% active.  Per output element
// the 128 x 32 tile reads 56 B of TMEM (2 segments x 7 int32 levels; TMEM
// reads run at 64 B/cycle/SM) and ~70 B of digit planes from L2, against
// ~4 DMMA cycles per element for the fp64 update -- a persistent,
// A-stationary kernel with double-buffered TMEM would be needed to pay off.
bool ozaki_syr2k_applicable(const GemmDesc& d) {
  const char* e = std::getenv("HSVD_SYR2K");
  if (!(e && std::strcmp(e, "ozaki") == 0)) return false;
  return d.M >= 1 && d.M == d.N && d.K >= 64 && d.K <= 256 && d.K % 64 == 0 && d.alpha == -1.0 &&
         d.beta == 1.0;
}

void ozaki_syr2k_batch(Ctx& ctx, const std::vector<GemmDesc>& descs) {
  size_t i0 = 0;
  while (i0 < descs.size()) {
    size_t i1 = i0;
    size_t used = 0;
    while (i1 < descs.size()) {
      const size_t need = (size_t)2 * kS * ceil_div(descs[i1].M, TM) * TM * KB;
      if (i1 > i0 && used + need > kPlaneBudget) break;
      used += need;
      ++i1;
    }
    Arena::Mark mk = ctx.arena.mark();
    std::vector<SyRows> src;
    std::vector<SyJob> jobs;
    long long rows = 0;
    int mpad_max = 0, tiles_max = 0;
    double tiles_total = 0.0;
    for (size_t i = i0; i < i1; ++i) {
      const GemmDesc& d = descs[i];
      const int mpad = ceil_div(d.M, TM) * TM;
      SyRows s{static_cast<const double*>(d.A), d.lda, d.M, d.K, rows, mpad,
               ctx.arena.alloc_n<double>((size_t)2 * mpad)};
      SyJob j{d.C, d.ldc, d.M, mpad, rows, s.sc, mpad / TM, ceil_div(d.M, TN)};
      int tiles = 0;
      for (int mb = 0; mb < j.mt; ++mb) tiles += std::min(j.nt, (mb * TM + TM - 1) / TN + 1);
      tiles_max = std::max(tiles_max, tiles);
      tiles_total += tiles;
      src.push_back(s);
      jobs.push_back(j);
      rows += (long long)2 * kS * mpad;
      mpad_max = std::max(mpad_max, mpad);
    }
    signed char* planes = ctx.arena.alloc_n<signed char>((size_t)rows * KB);
    const SyRows* ds = stage_table(ctx, src);
    const unsigned nj = (unsigned)(i1 - i0);
    ctx.launch_begin();
    k_oz_split_vw<<<dim3(mpad_max / 32, nj), 256, 0, ctx.stream>>>(ds, planes);
    ctx.check_launch("k_oz_split_vw");
    const CUtensorMap mapA = plane_map(planes, rows, TM);
    const CUtensorMap mapB = plane_map(planes, rows, TN);
    const SyJob* dj = stage_table(ctx, jobs);
    smem_optin(k_oz_syr2k, kSmem);
    // int8 multiply-adds x 2 of the 2 x 28 products per tile (profiler's "flops")
    ctx.pending_flops = tiles_total * 2.0 * (kS * (kS + 1) / 2) * 2.0 * TM * TN * KB;
    ctx.launch_begin();
    k_oz_syr2k<<<dim3(tiles_max, nj), kThreads, kSmem, ctx.stream>>>(mapA, mapB, dj);
    ctx.check_launch("k_oz_syr2k");
    ctx.arena.release(mk);
    i0 = i1;
  }
}

}  // namespace hsvdcu
