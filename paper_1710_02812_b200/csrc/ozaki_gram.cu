// Leaf block Gram G = X_b^T X_b on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, operands staged by TMA, int32 accumulators in TMEM)
// with fp64-grade accuracy for fp32 inputs: Ozaki-style splitting.
//
// The reference computes the leaf SVD in IEEE binary64 on the fp32-promoted
// values (kernels.cpp:21-48 on hierarchy.cpp:57's block).  tcgen05 has no f64
// kind, so the Gram is computed exactly in integer arithmetic on slices:
//
//   every column j of the block gets a power-of-two scale 2^e_j > max_i |x_ij|
//   and x_ij / 2^e_j = sum_{a=1..S} D_a[i][j] * 2^-(6 + 7(a-1)),
//   D_1 = rint(64 r), D_{a+1} = rint(128 * residual_a), all in [-64, 64]
//   (exact in fp32 arithmetic: power-of-two scalings and Sterbenz
//   subtractions).  Then
//   G_jl = 2^(e_j+e_l) * sum_{t=2..S+1} 2^-(12 + 7(t-2)) * sum_{a+b=t} (D_a^T D_b)_jl
//
// Each "level" t is one int32 accumulation on the tensor cores (|sum| <=
// (t-1) * K * 64^2 < 2^31 for K <= 65536): products with a + b > S + 1 are
// dropped.  S = 7 keeps every fp32 mantissa bit of elements down to 2^-24 of
// their column maximum and the dropped levels weigh ~2^-54: the measured
// |G - G_fp64| / |G| is 1.7e-15..2.7e-15 at the config-4 and config-5 leaf
// shapes (tools/study/ozaki_gram.py; the same 28 products emulated exactly on
// the CPU), i.e. the Gram is fp64-grade.
//
// Kernels:
//   k_oz_colmax   max |x_ij| per column (HBM-bound read of X)
//   k_oz_split    X (fp32, row-major) -> S int8 digit planes, transposed to
//                 K-major (the leaf's rows contiguous per column), zero padded
//   k_oz_gram     one CTA per 128x256 tile of the lower triangle of one leaf's
//                 Gram: warp 0 issues TMA loads (128B swizzle) into a 4-stage
//                 ring, warp 1 issues tcgen05.mma (M=128, N=256, K=32 per
//                 instruction) into one of two TMEM accumulators (levels
//                 alternate, 2 x 256 columns), warps 2-5 drain a finished level
//                 (tcgen05.ld) to an int32 level tile in global memory while
//                 the next level is being multiplied (store-only: an epilogue
//                 that read-modify-wrote fp64 G per level held the MMA warp on
//                 the TMEM-empty barrier; ncu, profiles/r02_oz_gram_cfg5.md)
//   k_oz_combine  G = scales * sum_t 2^-w(t) P_t in fp64 for j >= l, mirrored
//                 to the strict upper triangle (full storage for the
//                 eigensolver)
#include <cuda.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "engine.h"
#include "gemm.h"
#include "ozaki.h"

namespace hsvdcu {

namespace {

constexpr int kS = 7;            // digit planes
constexpr int kBM = 128;         // tile rows (TMEM lanes)
constexpr int kBN = 256;         // tile columns (TMEM columns per accumulator)
constexpr int kBK = 128;         // bytes of K per stage (one 128B swizzle row)
constexpr int kStages = 4;
constexpr int kABytes = kBM * kBK;                 // 16 KB
constexpr int kBBytes = kBN * kBK;                 // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;     // 48 KB
constexpr int kGramThreads = 192;                  // 6 warps
constexpr size_t kGramSmem = (size_t)kStages * kStageBytes + 1024 + 256;

struct OzLeaf {
  const float* x;      // block base (row-major, ld)
  long long ld;
  int K;               // rows of the block (Gram contraction length)
  int q;               // columns of the block (Gram order)
  long long row_base;  // first row of this leaf's digit planes in the slice tensor
  double* G;           // q x q column-major output
  long long ldg;
  double* scale;       // per column 2^e_j (q_pad entries)
  unsigned* colmax;    // per column max |x| bits (q_pad entries)
};

struct OzTile {
  int leaf, jb, lb;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---------------------------------------------------------------------------
// slicing
// ---------------------------------------------------------------------------

__global__ void k_oz_colmax(const OzLeaf* __restrict__ leaves, int rows_per_block) {
  const OzLeaf L = leaves[blockIdx.z];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i0 = blockIdx.y * rows_per_block;
  if (j >= L.q || i0 >= L.K) return;
  const int i1 = min(L.K, i0 + rows_per_block);
  const float* p = L.x + (long long)i0 * L.ld + j;
  float m = 0.0f;
#pragma unroll 4
  for (int i = i0; i < i1; ++i, p += L.ld) m = fmaxf(m, fabsf(__ldg(p)));
  if (m > 0.0f) atomicMax(L.colmax + j, __float_as_uint(m));
}

// One CTA: 128 rows (K) x 32 columns of one leaf -> S planes of 32 rows x 128
// bytes (K-major).  Thread (tx, ty): column tx, rows 4*ty + 32*rep + 0..3.
__global__ void __launch_bounds__(256) k_oz_split(const OzLeaf* __restrict__ leaves,
                                                  signed char* __restrict__ planes,
                                                  long long kpad, long long plane_rows) {
  __shared__ uint32_t sw[kS][32][33];
  const OzLeaf L = leaves[blockIdx.z];
  const int j0 = blockIdx.y * 32, i0 = blockIdx.x * 128;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int q_pad = (L.q + kBN - 1) / kBN * kBN;
  if (j0 >= q_pad) return;
  const int j = j0 + tx;
  float inv = 0.0f;
  if (j < L.q) {
    const float m = __uint_as_float(L.colmax[j]);
    int e = 0;
    if (m > 0.0f) {
      frexpf(m, &e);  // m = f 2^e, f in [0.5, 1): m < 2^e
      inv = ldexpf(1.0f, -e);
    }
    if (blockIdx.x == 0 && ty == 0) L.scale[j] = m > 0.0f ? ldexp(1.0, e) : 1.0;
  } else if (blockIdx.x == 0 && ty == 0 && j < q_pad) {
    L.scale[j] = 1.0;
  }
#pragma unroll
  for (int rep = 0; rep < 4; ++rep) {
    const int r4 = ty * 4 + rep * 32;
    uint32_t packed[kS];
#pragma unroll
    for (int a = 0; a < kS; ++a) packed[a] = 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + r4 + u;
      float r = 0.0f;
      if (j < L.q && i < L.K) r = __ldg(L.x + (long long)i * L.ld + j) * inv;
      float v = r * 64.0f;
#pragma unroll
      for (int a = 0; a < kS; ++a) {
        const float d = rintf(v);
        v = (v - d) * 128.0f;
        packed[a] |= (uint32_t)(uint8_t)(signed char)(int)d << (8 * u);
      }
    }
#pragma unroll
    for (int a = 0; a < kS; ++a) sw[a][tx][r4 >> 2] = packed[a];
  }
  __syncthreads();
  // write out: per plane 32 rows x 128 bytes; thread -> (row jr, 16-byte part p)
  const int jr = threadIdx.x >> 3, p = threadIdx.x & 7;
#pragma unroll
  for (int a = 0; a < kS; ++a) {
    uint4 w;
    w.x = sw[a][jr][p * 4 + 0];
    w.y = sw[a][jr][p * 4 + 1];
    w.z = sw[a][jr][p * 4 + 2];
    w.w = sw[a][jr][p * 4 + 3];
    const long long row = L.row_base + (long long)a * plane_rows + j0 + jr;
    *reinterpret_cast<uint4*>(planes + row * kpad + i0 + p * 16) = w;
  }
}

// ---------------------------------------------------------------------------
// tcgen05 / TMA / mbarrier primitives
// ---------------------------------------------------------------------------

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// K-major operand, 128B swizzle: rows of 128 bytes, 8-row atoms of 1024 bytes
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;              // leading byte offset (unused for swizzled K-major)
  d |= (uint64_t)(1024 >> 4) << 32;    // stride byte offset: next 8-row atom
  d |= (uint64_t)1 << 46;              // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;              // SWIZZLE_128B
  return d;
}
// kind::i8: D s32, A s8, B s8, both K-major, M = 128, N = 256
constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kBN >> 3) << 17) |
                            ((uint32_t)(kBM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---------------------------------------------------------------------------
// the Gram kernel
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kGramThreads, 1)
    k_oz_gram(const __grid_constant__ CUtensorMap tmap, const OzLeaf* __restrict__ leaves,
              const OzTile* __restrict__ tiles, long long plane_rows, int nk,
              int* __restrict__ part) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  uint64_t* empty = full + kStages;
  uint64_t* tfull = empty + kStages;   // [2]
  uint64_t* tempty = tfull + 2;        // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const OzTile T = tiles[blockIdx.x];
  const OzLeaf L = leaves[T.leaf];

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const long long rowA0 = L.row_base + (long long)T.jb * kBM;
  const long long rowB0 = L.row_base + (long long)T.lb * kBN;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 2; t <= kS + 1; ++t) {
        for (int a = max(1, t - kS); a <= min(kS, t - 1); ++a) {
          const int b = t - a;
          const int ra = static_cast<int>(rowA0 + (long long)(a - 1) * plane_rows);
          const int rb = static_cast<int>(rowB0 + (long long)(b - 1) * plane_rows);
          for (int kc = 0; kc < nk; ++kc) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + stage * kStageBytes;
            mbar_expect_tx(&full[stage], kStageBytes);
            tma_load_2d(sa, &tmap, kc * kBK, ra, &full[stage]);
            tma_load_2d(sa + kABytes, &tmap, kc * kBK, rb, &full[stage]);
            tma_load_2d(sa + kABytes + kABytes, &tmap, kc * kBK, rb + kBM, &full[stage]);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 2; t <= kS + 1; ++t) {
        const int buf = t & 1;
        if (t >= 4) mbar_wait(&tempty[buf], ((t - 4) >> 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * kBN;
        bool first = true;
        for (int a = max(1, t - kS); a <= min(kS, t - 1); ++a) {
          for (int kc = 0; kc < nk; ++kc) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + stage * kStageBytes);
            const uint64_t ad = umma_desc(sa), bd = umma_desc(sa + kABytes);
#pragma unroll
            for (int k = 0; k < kBK / 32; ++k) {
              mma_i8(d, ad + 2 * k, bd + 2 * k, first ? 0u : 1u);
              first = false;
            }
            mma_commit(&empty[stage]);
            if (++stage == kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
        mma_commit(&tfull[buf]);
      }
    }
  } else {
    // ---------------- epilogue: TMEM -> int32 level tiles (store only) ----------------
    // level t of this tile -> P[tile][t-2][col][row] (a warp stores 32
    // consecutive rows of one column: 128 contiguous bytes); no global reads,
    // so a drained accumulator is released as fast as TMEM can be read
    const int quarter = warp & 3;  // TMEM lanes 32*quarter .. +31 (warp % 4 rule)
    const int r = quarter * 32 + lane;
    int* P = part + (long long)blockIdx.x * (kS * kBN * kBM) + r;
    for (int t = 2; t <= kS + 1; ++t) {
      const int buf = t & 1;
      mbar_wait(&tfull[buf], ((t - 2) >> 1) & 1);
      tc_fence_after();
      int* Pt = P + (t - 2) * (kBN * kBM);
#pragma unroll 1
      for (int c0 = 0; c0 < kBN; c0 += 32) {
        int v[32];
        tmem_ld32(tmem + ((uint32_t)(quarter * 32) << 16) + buf * kBN + c0, v);
#pragma unroll
        for (int i = 0; i < 32; ++i) Pt[(c0 + i) * kBM] = v[i];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// G from the int32 level tiles: G_jl = 2^(e_j+e_l) sum_t 2^-(12+7(t-2)) P_t
// (most significant level first, fp64), written for j >= l and mirrored to
// (l, j) through a shared-memory transpose (full symmetric storage for the
// eigensolver).  One CTA per Gram tile, 32x32 sub-blocks.
__global__ void __launch_bounds__(256) k_oz_combine(const OzLeaf* __restrict__ leaves,
                                                    const OzTile* __restrict__ tiles,
                                                    const int* __restrict__ part) {
  __shared__ double sub[32][33];
  const OzTile T = tiles[blockIdx.x];
  const OzLeaf L = leaves[T.leaf];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int* P = part + (long long)blockIdx.x * (kS * kBN * kBM);
  for (int rb = 0; rb < kBM; rb += 32) {
    const int row0 = T.jb * kBM + rb;
    for (int cb = 0; cb < kBN; cb += 32) {
      const int col0 = T.lb * kBN + cb;
      if (row0 + 31 < col0 || row0 >= L.q || col0 >= L.q) continue;  // no j >= l element
      const int row = row0 + tx;
      const double sr = row < L.q ? L.scale[row] : 0.0;
      for (int y = ty; y < 32; y += 8) {
        const int col = col0 + y;
        const int* p = P + (cb + y) * kBM + rb + tx;
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t < kS; ++t) acc += ldexp((double)__ldcs(p + t * kBN * kBM), -(12 + 7 * t));
        acc *= sr * (col < L.q ? L.scale[col] : 0.0);
        sub[y][tx] = acc;
        if (row < L.q && col < L.q && row >= col) L.G[row + (long long)col * L.ldg] = acc;
      }
      __syncthreads();
      for (int y = ty; y < 32; y += 8) {
        // mirror: (row0 + y, col0 + tx) <- sub[tx][y] when row0 + y > col0 + tx
        const int mrow = col0 + tx, mcol = row0 + y;
        if (mcol < L.q && mrow < L.q && mcol > mrow) L.G[mrow + (long long)mcol * L.ldg] = sub[tx][y];
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      throw Error(kCuda, "cuTensorMapEncodeTiled entry point not available");
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

int slices_env() {
  const char* e = std::getenv("HSVD_GRAM");
  return (e && std::strcmp(e, "dmma") == 0) ? 0 : kS;
}

}  // namespace

bool ozaki_gram_applicable(DType dt, const GemmDesc& d) {
  // tall fp32 blocks (G = X_b^T X_b, K = rows): every BASELINE fp32 leaf
  return slices_env() > 0 && dt == DType::F32 && d.K >= 1 && d.K <= 65536 && d.M >= 1 &&
         d.M == d.N && d.A == d.B;
}

void ozaki_gram_batch(Ctx& ctx, const std::vector<GemmDesc>& descs) {
  if (descs.empty()) return;
  int Kmax = 0;
  for (const auto& d : descs) Kmax = std::max(Kmax, d.K);
  const long long kpad = (long long)ceil_div(Kmax, kBK) * kBK;
  smem_optin(k_oz_gram, kGramSmem);
  // batches of leaves bounded by the digit-plane memory (~2 GB)
  const size_t kPlaneBudget = size_t(2) << 30;
  size_t i0 = 0;
  while (i0 < descs.size()) {
    size_t i1 = i0;
    long long rows = 0;
    while (i1 < descs.size()) {
      const long long qp = (long long)ceil_div(descs[i1].M, kBN) * kBN;
      // planes (S q_pad K_pad bytes) + level tiles (~ S q_pad^2 / 2 int32)
      const long long need = kS * qp * kpad + 2LL * kS * qp * (qp + kBN);
      if (i1 > i0 && (size_t)(rows + need) > kPlaneBudget) break;
      rows += need;
      ++i1;
    }
    Arena::Mark mk = ctx.arena.mark();
    const int nl = static_cast<int>(i1 - i0);
    std::vector<OzLeaf> hl(nl);
    std::vector<OzTile> ht;
    long long base = 0, plane_rows = 0;
    int max_qp = 0;
    for (int l = 0; l < nl; ++l) max_qp = std::max(max_qp, ceil_div(descs[i0 + l].M, kBN) * kBN);
    // plane layout: rows = a * plane_rows + leaf_base + j, plane_rows = sum_l q_pad(l)
    for (int l = 0; l < nl; ++l) plane_rows += (long long)ceil_div(descs[i0 + l].M, kBN) * kBN;
    double* scales = ctx.arena.alloc_n<double>((size_t)plane_rows);
    unsigned* cmax = ctx.arena.alloc_n<unsigned>((size_t)plane_rows);
    signed char* planes = ctx.arena.alloc_n<signed char>((size_t)(kS * plane_rows * kpad));
    for (int l = 0; l < nl; ++l) {
      const GemmDesc& d = descs[i0 + l];
      const int qp = ceil_div(d.M, kBN) * kBN;
      hl[l] = {static_cast<const float*>(d.A), d.lda, d.K, d.M, base, d.C, d.ldc, scales + base,
               cmax + base};
      for (int jb = 0; jb * kBM < qp; ++jb)
        for (int lb = 0; lb * kBN <= jb * kBM + kBM - 1 && lb * kBN < qp; ++lb)
          ht.push_back({l, jb, lb});
      base += qp;
    }
    // job tables read by several launches: staged into arena memory
    OzLeaf* dl = static_cast<OzLeaf*>(ctx.staging.put_to(
        ctx.arena.alloc(hl.size() * sizeof(OzLeaf)), hl.data(), hl.size() * sizeof(OzLeaf),
        ctx.stream));
    OzTile* dt = static_cast<OzTile*>(ctx.staging.put_to(
        ctx.arena.alloc(ht.size() * sizeof(OzTile)), ht.data(), ht.size() * sizeof(OzTile),
        ctx.stream));
    HSVD_CUDA(cudaMemsetAsync(cmax, 0, (size_t)plane_rows * sizeof(unsigned), ctx.stream));

    const int rpb = 256;
    ctx.launch_begin();
    k_oz_colmax<<<dim3(ceil_div(max_qp, 256), ceil_div(Kmax, rpb), nl), 256, 0, ctx.stream>>>(dl,
                                                                                              rpb);
    ctx.check_launch("k_oz_colmax");
    ctx.launch_begin();
    k_oz_split<<<dim3((unsigned)(kpad / 128), max_qp / 32, nl), 256, 0, ctx.stream>>>(
        dl, planes, kpad, plane_rows);
    ctx.check_launch("k_oz_split");

    CUtensorMap tmap;
    const cuuint64_t gdim[2] = {(cuuint64_t)kpad, (cuuint64_t)(kS * plane_rows)};
    const cuuint64_t gstride[1] = {(cuuint64_t)kpad};
    const cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)kBM};
    const cuuint32_t estr[2] = {1, 1};
    CUresult cr = encode_fn()(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, planes, gdim, gstride, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) throw Error(kCuda, "cuTensorMapEncodeTiled failed");
    // tensor-pipe work of the launch: int8 multiply-adds x 2 over every
    // tile, product and padded K (the profiler's "flops" for this kernel)
    ctx.pending_flops = (double)ht.size() * (kS * (kS + 1) / 2) * 2.0 * kBM * kBN * (double)kpad;
    int* part = ctx.arena.alloc_n<int>(ht.size() * (size_t)kS * kBN * kBM);
    ctx.launch_begin();
    k_oz_gram<<<(unsigned)ht.size(), kGramThreads, kGramSmem, ctx.stream>>>(
        tmap, dl, dt, plane_rows, static_cast<int>(kpad / kBK), part);
    ctx.check_launch("k_oz_gram");
    ctx.launch_begin();
    k_oz_combine<<<(unsigned)ht.size(), 256, 0, ctx.stream>>>(dl, dt, part);
    ctx.check_launch("k_oz_combine");
    ctx.arena.release(mk);
    i0 = i1;
  }
}

}  // namespace hsvdcu
