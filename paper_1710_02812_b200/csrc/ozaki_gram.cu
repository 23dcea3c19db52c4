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
#include "ozaki_tc.cuh"

namespace hsvdcu {

namespace {

using namespace oztc;

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
constexpr int kMaxK = 65536;  // |level sum| <= 7 * K * 64^2 < 2^31

// Column-scaled source (k_oz_split): the columns of a row-major fp32 block
// become digit-plane rows (transposed, K = the block's rows).
struct OzLeaf {
  const float* x;      // block base (row-major, ld)
  long long ld;
  int K;               // rows of the block (contraction length)
  int q;               // columns of the block (operand rows)
  long long row_base;  // first row of this block's digit planes in the slice tensor
  double* G;           // unused by the slicer
  long long ldg;
  double* scale;       // per column 2^e_j (q_pad entries)
  unsigned* colmax;    // per column max |x| bits (q_pad entries)
};

// Row-scaled source (k_oz_split_rows): rows with K contiguous (a row-major
// fp32 block, or the columns of a column-major fp64 factor).
struct OzRows {
  const void* x;
  int f64;
  long long ld;        // row stride (elements)
  int rows, K;
  long long row_base;  // first digit-plane row
  double* scale;       // per row 2^e (rows entries)
};

// One product C (M x N, column-major ldc) = A_op B_op^T over digit planes.
struct OzJob {
  long long a_row, b_row;  // plane-1 rows of A_op row 0 / B_op row 0
  double* C;
  long long ldc;
  const double* sa;        // scale of each C row (A_op row)
  const double* sb;        // scale of each C column (B_op row)
  int M, N;
  int sym;                 // Gram: write j >= l and mirror to the upper triangle
};

// One CTA: rows mb*128.., columns nb*256.. of job, K chunks [k0, k0 + nk).
struct OzTile {
  int job, mb, nb, k0, nk;
};


// ---------------------------------------------------------------------------
// slicing
// ---------------------------------------------------------------------------

// Digit extraction without the conversion unit: rintf / (int) go through
// FRND / F2I (16 lanes per clock per SM), which bound the split kernels at
// ~0.47 of the HBM peak (14 conversions per element).  Adding 1.5 * 2^23
// rounds v to the nearest-even integer in the mantissa's low bits (|v| < 2^22):
// d = t - M is rintf(v) exactly, and the low byte of t's bit pattern is d as
// an int8 -- full-rate FADD + one PRMT per digit, bit-identical digits.
template <int U>
__device__ __forceinline__ uint32_t put_byte(uint32_t packed, uint32_t src) {
  constexpr uint32_t sel = U == 0 ? 0x3214u : U == 1 ? 0x3240u : U == 2 ? 0x3410u : 0x4210u;
  return __byte_perm(packed, src, sel);
}
template <int U>
__device__ __forceinline__ void oz_digits(float v, uint32_t (&packed)[kS]) {
  const float M = 12582912.0f;  // 1.5 * 2^23
#pragma unroll
  for (int a = 0; a < kS; ++a) {
    const float t = v + M;
    const float d = t - M;
    v = (v - d) * 128.0f;
    packed[a] = put_byte<U>(packed[a], __float_as_uint(t));
  }
}
template <int U>
__device__ __forceinline__ void oz_digits(double v, uint32_t (&packed)[kS]) {
  const double M = 6755399441055744.0;  // 1.5 * 2^52
#pragma unroll
  for (int a = 0; a < kS; ++a) {
    const double t = v + M;
    const double d = t - M;
    v = (v - d) * 128.0;
    packed[a] = put_byte<U>(packed[a], (uint32_t)__double2loint(t));
  }
}
template <typename T>
__device__ __forceinline__ void oz_digits4(const T (&v)[4], uint32_t (&packed)[kS]) {
  oz_digits<0>(v[0], packed);
  oz_digits<1>(v[1], packed);
  oz_digits<2>(v[2], packed);
  oz_digits<3>(v[3], packed);
}

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
// blockIdx.x walks super-tiles of 8 column tiles x 32 K chunks (column tile
// fastest): CTAs resident together read 1 KB runs of the same rows and write
// 4 KB runs of the same plane rows (DRAM page locality on both sides).
__global__ void __launch_bounds__(256) k_oz_split(const OzLeaf* __restrict__ leaves,
                                                  signed char* __restrict__ planes,
                                                  long long kpad, long long plane_rows, int ntj) {
  __shared__ uint32_t sw[kS][32][33];
  const OzLeaf L = leaves[blockIdx.z];
  int j0, i0;
  {
    const unsigned per_super = 32u * (unsigned)ntj;  // CTAs per band of 32 K chunks
    const unsigned sup = blockIdx.x / per_super, r = blockIdx.x % per_super;
    const unsigned cs = r / 256u, r2 = r % 256u;     // 8 x 32 tiles per super-tile
    j0 = (int)(cs * 8u + (r2 & 7u)) * 32;
    i0 = (int)(sup * 32u + (r2 >> 3)) * 128;
    if (i0 >= kpad) return;
  }
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
    if (i0 == 0 && ty == 0) L.scale[j] = m > 0.0f ? ldexp(1.0, e) : 1.0;
  } else if (i0 == 0 && ty == 0 && j < q_pad) {
    L.scale[j] = 1.0;
  }
  // all 16 loads of the thread first, then the digit arithmetic
  float x[4][4];
#pragma unroll
  for (int rep = 0; rep < 4; ++rep)
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + ty * 4 + rep * 32 + u;
      x[rep][u] = (j < L.q && i < L.K) ? __ldg(L.x + (long long)i * L.ld + j) : 0.0f;
    }
#pragma unroll
  for (int rep = 0; rep < 4; ++rep) {
    const int r4 = ty * 4 + rep * 32;
    uint32_t packed[kS];
#pragma unroll
    for (int a = 0; a < kS; ++a) packed[a] = 0u;
    const float v[4] = {x[rep][0] * inv * 64.0f, x[rep][1] * inv * 64.0f, x[rep][2] * inv * 64.0f,
                        x[rep][3] * inv * 64.0f};
    oz_digits4(v, packed);
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

// per-row scale of a row-scaled source: max |x| over K.  One CTA per 8 rows,
// the whole CTA walking along one row at a time (4 KB per load instruction):
// with a warp per row, ~9000 rows were streamed at once across the GPU, each
// from its own DRAM page (0.55 of the HBM peak).
__global__ void __launch_bounds__(256) k_oz_rowmax(const OzRows* __restrict__ srcs) {
  const OzRows S = srcs[blockIdx.y];
  const int row0 = blockIdx.x * 8, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (row0 >= S.rows) return;
  __shared__ double red[8][8];
  double m[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) m[r] = 0.0;
  if (S.f64) {
    // fp64 factors are short (kk rows): a warp per row, four loads in flight
    if (row0 + warp < S.rows) {
      const double* p = static_cast<const double*>(S.x) + (long long)(row0 + warp) * S.ld;
      double a = 0.0, b = 0.0, c = 0.0, d = 0.0;
      int k = lane;
      for (; k + 96 < S.K; k += 128) {
        a = fmax(a, fabs(p[k]));
        b = fmax(b, fabs(p[k + 32]));
        c = fmax(c, fabs(p[k + 64]));
        d = fmax(d, fabs(p[k + 96]));
      }
      for (; k < S.K; k += 32) a = fmax(a, fabs(p[k]));
      double v = fmax(fmax(a, b), fmax(c, d));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (lane == 0) {
        int e = 0;
        if (v > 0.0) frexp(v, &e);  // v < 2^e
        S.scale[row0 + warp] = v > 0.0 ? ldexp(1.0, e) : 1.0;
      }
    }
    return;  // uniform per CTA
  } else {
    for (int r = 0; r < 8 && row0 + r < S.rows; ++r) {
      const float* p = static_cast<const float*>(S.x) + (long long)(row0 + r) * S.ld;
      float f0 = 0.0f, f1 = 0.0f;
      int k = tid;
      if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {  // 16-byte loads, four in flight
        const float4* p4 = reinterpret_cast<const float4*>(p);
        const int K4 = S.K >> 2;
        int q = tid;
        for (; q + 768 < K4; q += 1024) {
          const float4 a = __ldg(p4 + q), b = __ldg(p4 + q + 256), c = __ldg(p4 + q + 512),
                       d = __ldg(p4 + q + 768);
          f0 = fmaxf(f0, fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))));
          f1 = fmaxf(f1, fmaxf(fmaxf(fabsf(b.x), fabsf(b.y)), fmaxf(fabsf(b.z), fabsf(b.w))));
          f0 = fmaxf(f0, fmaxf(fmaxf(fabsf(c.x), fabsf(c.y)), fmaxf(fabsf(c.z), fabsf(c.w))));
          f1 = fmaxf(f1, fmaxf(fmaxf(fabsf(d.x), fabsf(d.y)), fmaxf(fabsf(d.z), fabsf(d.w))));
        }
        for (; q < K4; q += 256) {
          const float4 a = __ldg(p4 + q);
          f0 = fmaxf(f0, fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))));
        }
        k = (K4 << 2) + tid;  // tail elements
      }
      for (; k < S.K; k += 256) f0 = fmaxf(f0, fabsf(__ldg(p + k)));
      m[r] = (double)fmaxf(f0, f1);
    }
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m[r] = fmax(m[r], __shfl_xor_sync(0xffffffffu, m[r], o));
    if (lane == 0) red[warp][r] = m[r];
  }
  __syncthreads();
  if (tid < 8 && row0 + tid < S.rows) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) v = fmax(v, red[w][tid]);
    int e = 0;
    if (v > 0.0) frexp(v, &e);  // v < 2^e
    S.scale[row0 + tid] = v > 0.0 ? ldexp(1.0, e) : 1.0;
  }
}

// rows x K -> S digit planes (K-major, rows padded by the caller's zeroed
// tail, K padded to kpad with zeros).  Thread: 4 consecutive K of one row.
__global__ void __launch_bounds__(256) k_oz_split_rows(const OzRows* __restrict__ srcs,
                                                       signed char* __restrict__ planes,
                                                       long long kpad, long long plane_rows) {
  const OzRows S = srcs[blockIdx.z];
  const int row = blockIdx.y * 8 + (threadIdx.x >> 5);
  const int k4 = blockIdx.x * 128 + (threadIdx.x & 31) * 4;
  if (row >= S.rows) return;
  const double inv = 1.0 / S.scale[row];  // exact: a power of two
  uint32_t packed[kS];
#pragma unroll
  for (int a = 0; a < kS; ++a) packed[a] = 0u;
  if (S.f64) {
    const double* p = static_cast<const double*>(S.x) + (long long)row * S.ld + k4;
    double v[4];
    if (k4 + 3 < S.K && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
      const double2 a = *reinterpret_cast<const double2*>(p);
      const double2 b = *reinterpret_cast<const double2*>(p + 2);
      v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = k4 + u < S.K ? p[u] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = v[u] * inv * 64.0;
    oz_digits4(v, packed);
  } else {
    const float* p = static_cast<const float*>(S.x) + (long long)row * S.ld + k4;
    float v[4];
    if (k4 + 3 < S.K && (reinterpret_cast<uintptr_t>(p) & 15) == 0) {
      const float4 a = __ldg(reinterpret_cast<const float4*>(p));
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = k4 + u < S.K ? __ldg(p + u) : 0.0f;
    }
    const float finv = (float)inv;
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = v[u] * finv * 64.0f;
    oz_digits4(v, packed);
  }
#pragma unroll
  for (int a = 0; a < kS; ++a)
    *reinterpret_cast<uint32_t*>(planes + (S.row_base + (long long)a * plane_rows + row) * kpad +
                                 k4) = packed[a];
}

// ---------------------------------------------------------------------------
// the Gram kernel
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kGramThreads, 1)
    k_oz_gram(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const OzJob* __restrict__ jobs, const OzTile* __restrict__ tiles,
              long long planeA, long long planeB, int* __restrict__ part) {
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
  const OzJob J = jobs[T.job];

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
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
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

  const long long rowA0 = J.a_row + (long long)T.mb * kBM;
  const long long rowB0 = J.b_row + (long long)T.nb * kBN;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 2; t <= kS + 1; ++t) {
        for (int a = max(1, t - kS); a <= min(kS, t - 1); ++a) {
          const int b = t - a;
          const int ra = static_cast<int>(rowA0 + (long long)(a - 1) * planeA);
          const int rb = static_cast<int>(rowB0 + (long long)(b - 1) * planeB);
          for (int kc = T.k0; kc < T.k0 + T.nk; ++kc) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + stage * kStageBytes;
            mbar_expect_tx(&full[stage], kStageBytes);
            tma_load_2d(sa, &tmA, kc * kBK, ra, &full[stage]);
            tma_load_2d(sa + kABytes, &tmB, kc * kBK, rb, &full[stage]);
            tma_load_2d(sa + kABytes + kABytes, &tmB, kc * kBK, rb + kBM, &full[stage]);
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
          for (int kc = 0; kc < T.nk; ++kc) {
            mbar_wait(&full[stage], phase);
            tc_fence_after();
            const uint32_t sa = smem_u32(smem + stage * kStageBytes);
            const uint64_t ad = umma_desc(sa), bd = umma_desc(sa + kABytes);
#pragma unroll
            for (int k = 0; k < kBK / 32; ++k) {
              mma_i8<idesc_i8(kBM, kBN)>(d, ad + 2 * k, bd + 2 * k, first ? 0u : 1u);
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

// C from the int32 level tiles of the K splits of one output tile:
// C_jl = sa_j sb_l sum_t 2^-(12+7(t-2)) sum_split P_t (most significant level
// first, fixed order: deterministic), fp64.  Gram jobs (sym) write j >= l
// and mirror to (l, j) through a shared-memory transpose (full symmetric
// storage for the eigensolver).  One CTA (512 threads) per output tile in
// 32-column x 128-row slabs: every thread keeps its 7 x NSPLIT level loads
// of two elements in flight (the pass is HBM-bound: 28 B read per element).
template <int NSPLIT>
__global__ void __launch_bounds__(512) k_oz_combine(const OzJob* __restrict__ jobs,
                                                    const OzTile* __restrict__ tiles,
                                                    const int* __restrict__ part, int nsplit_rt) {
  __shared__ double sub[32][kBM + 1];  // [col in slab][row]
  const int nsplit = NSPLIT > 0 ? NSPLIT : nsplit_rt;
  const OzTile T = tiles[(long long)blockIdx.x * nsplit];
  const OzJob J = jobs[T.job];
  const int tid = threadIdx.x;
  const int row = T.mb * kBM + (tid & (kBM - 1));  // 128 rows
  const int cq = tid >> 7;                          // 4 column groups
  const double sr = row < J.M ? J.sa[row] : 0.0;
  const int* P = part + (long long)blockIdx.x * nsplit * (kS * kBN * kBM) + (tid & (kBM - 1));
  for (int cb = 0; cb < kBN; cb += 32) {
    const int col0 = T.nb * kBN + cb;
    if (col0 >= J.N) break;
    if (J.sym && T.mb * kBM + kBM - 1 < col0) break;  // the rest of the tile is j < l
#pragma unroll
    for (int h = 0; h < 8; h += 2) {
      // two columns per thread per pass: cb + cq*8 + h, +1
      const int c0 = cb + cq * 8 + h;
      double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
      for (int t = 0; t < kS; ++t) {
        long long l0 = 0, l1 = 0;
        if (NSPLIT > 0) {
#pragma unroll
          for (int sp = 0; sp < (NSPLIT > 0 ? NSPLIT : 1); ++sp) {
            const int* q = P + ((long long)sp * kS + t) * (kBN * kBM);
            l0 += __ldcs(q + c0 * kBM);
            l1 += __ldcs(q + (c0 + 1) * kBM);
          }
        } else {
          for (int sp = 0; sp < nsplit; ++sp) {
            const int* q = P + ((long long)sp * kS + t) * (kBN * kBM);
            l0 += __ldcs(q + c0 * kBM);
            l1 += __ldcs(q + (c0 + 1) * kBM);
          }
        }
        acc0 += ldexp((double)l0, -(12 + 7 * t));
        acc1 += ldexp((double)l1, -(12 + 7 * t));
      }
      const int col = T.nb * kBN + c0;
      acc0 *= sr * (col < J.N ? J.sb[col] : 0.0);
      acc1 *= sr * (col + 1 < J.N ? J.sb[col + 1] : 0.0);
      sub[c0 - cb][tid & (kBM - 1)] = acc0;
      sub[c0 - cb + 1][tid & (kBM - 1)] = acc1;
      if (row < J.M) {
        if (col < J.N && (!J.sym || row >= col)) J.C[row + (long long)col * J.ldc] = acc0;
        if (col + 1 < J.N && (!J.sym || row >= col + 1))
          J.C[row + (long long)(col + 1) * J.ldc] = acc1;
      }
    }
    if (J.sym) {
      __syncthreads();
      // mirror: C[col][row] <- C[row][col] for row > col; 32 columns of the
      // slab become 32 rows; a warp writes 32 consecutive destination rows
      for (int e = tid; e < 32 * kBM; e += 512) {
        const int rr = e >> 5, cc = e & 31;  // source row rr (0..127), slab column cc
        const int srow = T.mb * kBM + rr, scol = col0 + cc;
        if (srow < J.M && scol < J.N && srow > scol) J.C[scol + (long long)srow * J.ldc] = sub[cc][rr];
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

int slices_env() {
  const char* e = std::getenv("HSVD_GRAM");
  return (e && std::strcmp(e, "dmma") == 0) ? 0 : kS;
}

}  // namespace

bool ozaki_gram_applicable(DType dt, const GemmDesc& d) {
  // tall fp32 blocks (G = X_b^T X_b, K = rows): every BASELINE fp32 leaf
  return slices_env() > 0 && dt == DType::F32 && d.K >= 1 && d.K <= kMaxK && d.M >= 1 &&
         d.M == d.N && d.A == d.B;
}

bool ozaki_gemm_applicable(DType ta, bool trans_a, const GemmDesc& d) {
  (void)trans_a;
  const char* e = std::getenv("HSVD_PROJ");
  if (e && std::strcmp(e, "dmma") == 0) return false;
  // N > 160: the 256-wide MMA tile wastes < 40% and the 28 products beat
  // the fp64 DMMA GEMM (measured, round 2: config 5's N = 200 projections
  // 70 -> ~40 ms; config 3/4's N = 64/128 were slower than DMMA, bound by
  // the padded tile and the A-plane traffic of 28 products)
  return ta == DType::F32 && d.K >= 1 && d.K <= kMaxK && d.M >= 1 && d.N > 160 && d.N <= kBN &&
         d.alpha == 1.0 && d.beta == 0.0;
}

namespace {

struct PlaneSet {
  signed char* planes = nullptr;
  long long plane_rows = 0;  // rows of one digit plane (all sources)
  long long kpad = 0;
  CUtensorMap map;
};

CUtensorMap make_map(signed char* planes, long long kpad, long long rows) {
  CUtensorMap tmap;
  const cuuint64_t gdim[2] = {(cuuint64_t)kpad, (cuuint64_t)rows};
  const cuuint64_t gstride[1] = {(cuuint64_t)kpad};
  const cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)kBM};
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

// Column-scaled, transposed planes of fp32 blocks (sources' rows_base and
// scale pointers are filled in here; each source takes q_pad = ceil(q/256)
// plane rows).
PlaneSet slice_cols(Ctx& ctx, std::vector<OzLeaf>& src, long long kpad) {
  PlaneSet ps;
  ps.kpad = kpad;
  int max_qp = 0, Kmax = 0;
  for (auto& l : src) {
    const int qp = ceil_div(l.q, kBN) * kBN;
    l.row_base = ps.plane_rows;
    ps.plane_rows += qp;
    max_qp = std::max(max_qp, qp);
    Kmax = std::max(Kmax, l.K);
  }
  double* scales = ctx.arena.alloc_n<double>((size_t)ps.plane_rows);
  unsigned* cmax = ctx.arena.alloc_n<unsigned>((size_t)ps.plane_rows);
  for (auto& l : src) {
    l.scale = scales + l.row_base;
    l.colmax = cmax + l.row_base;
  }
  ps.planes = ctx.arena.alloc_n<signed char>((size_t)(kS * ps.plane_rows * kpad));
  const int nl = static_cast<int>(src.size());
  OzLeaf* dl = stage_table(ctx, src);
  HSVD_CUDA(cudaMemsetAsync(cmax, 0, (size_t)ps.plane_rows * sizeof(unsigned), ctx.stream));
  const int rpb = 256;
  // algorithmic HBM bytes (profile): the max pass reads the fp32 block once;
  // the split reads it again and writes kS int8 digit planes
  double elems = 0.0;
  for (const auto& l : src) elems += (double)l.K * l.q;
  ctx.launch_begin();
  ctx.pending_bytes = 4.0 * elems;
  k_oz_colmax<<<dim3(ceil_div(max_qp, 256), ceil_div(Kmax, rpb), nl), 256, 0, ctx.stream>>>(dl, rpb);
  ctx.check_launch("k_oz_colmax");
  ctx.launch_begin();
  ctx.pending_bytes = (4.0 + kS) * elems;
  k_oz_split<<<dim3((unsigned)(ceil_div((int)(kpad / 128), 32) * 32 * (max_qp / 32)), 1, nl), 256, 0,
               ctx.stream>>>(
      dl, ps.planes, kpad, ps.plane_rows, max_qp / 32);
  ctx.check_launch("k_oz_split");
  ps.map = make_map(ps.planes, kpad, kS * ps.plane_rows);
  return ps;
}

// Row-scaled planes (rows with K contiguous): fp32 blocks or the columns of
// column-major fp64 factors.  Each source takes ceil(rows/256)*256 plane
// rows (the padding rows stay unwritten: they only reach C rows / columns
// that are never stored).
PlaneSet slice_rows(Ctx& ctx, std::vector<OzRows>& src, long long kpad) {
  PlaneSet ps;
  ps.kpad = kpad;
  int max_rows = 0;
  for (auto& r : src) {
    r.row_base = ps.plane_rows;
    ps.plane_rows += (long long)ceil_div(r.rows, kBN) * kBN;
    max_rows = std::max(max_rows, r.rows);
  }
  double* scales = ctx.arena.alloc_n<double>((size_t)ps.plane_rows);
  for (auto& r : src) r.scale = scales + r.row_base;
  ps.planes = ctx.arena.alloc_n<signed char>((size_t)(kS * ps.plane_rows * kpad));
  const int ns = static_cast<int>(src.size());
  OzRows* ds = stage_table(ctx, src);
  double in_bytes = 0.0, elems = 0.0;  // algorithmic HBM bytes, as in slice_cols
  for (const auto& r : src) {
    in_bytes += (r.f64 ? 8.0 : 4.0) * r.rows * r.K;
    elems += (double)r.rows * r.K;
  }
  ctx.launch_begin();
  ctx.pending_bytes = in_bytes;
  k_oz_rowmax<<<dim3(ceil_div(max_rows, 8), ns), 256, 0, ctx.stream>>>(ds);
  ctx.check_launch("k_oz_rowmax");
  ctx.launch_begin();
  ctx.pending_bytes = in_bytes + kS * elems;
  k_oz_split_rows<<<dim3((unsigned)(kpad / 128), ceil_div(max_rows, 8), ns), 256, 0, ctx.stream>>>(
      ds, ps.planes, kpad, ps.plane_rows);
  ctx.check_launch("k_oz_split_rows");
  ps.map = make_map(ps.planes, kpad, kS * ps.plane_rows);
  return ps;
}

// Tiles of every job (Gram jobs: the lower triangle only), each output tile
// split over nsplit K ranges (consecutive tile entries), then the
// tensor-core launch and the combine.
void run_products(Ctx& ctx, const PlaneSet& A, const PlaneSet& B, const std::vector<OzJob>& jobs) {
  const int nk = static_cast<int>(A.kpad / kBK);
  long long outs = 0;
  for (const auto& j : jobs) {
    const int mt = ceil_div(j.M, kBM), nt = ceil_div(j.N, kBN);
    for (int mb = 0; mb < mt; ++mb)
      for (int nb = 0; nb < nt; ++nb)
        if (!j.sym || nb * kBN <= mb * kBM + kBM - 1) ++outs;
  }
  // enough CTAs for two per SM slot, each split keeping >= 8 K chunks
  int nsplit = (int)std::max<long long>(1, (2LL * ctx.num_sms + outs - 1) / std::max(1LL, outs));
  nsplit = std::max(1, std::min({nsplit, nk / 8, 16}));
  const int per = ceil_div(nk, nsplit);
  nsplit = ceil_div(nk, per);
  std::vector<OzTile> ht;
  ht.reserve((size_t)outs * nsplit);
  for (int ji = 0; ji < (int)jobs.size(); ++ji) {
    const OzJob& j = jobs[ji];
    const int mt = ceil_div(j.M, kBM), nt = ceil_div(j.N, kBN);
    for (int mb = 0; mb < mt; ++mb)
      for (int nb = 0; nb < nt; ++nb) {
        if (j.sym && nb * kBN > mb * kBM + kBM - 1) continue;
        for (int sp = 0; sp < nsplit; ++sp)
          ht.push_back({ji, mb, nb, sp * per, std::min(per, nk - sp * per)});
      }
  }
  OzJob* dj = stage_table(ctx, jobs);
  OzTile* dt = stage_table(ctx, ht);
  int* part = ctx.arena.alloc_n<int>(ht.size() * (size_t)kS * kBN * kBM);
  smem_optin(k_oz_gram, kGramSmem);
  // tensor-pipe work of the launch: int8 multiply-adds x 2 over every tile,
  // product and K chunk (the profiler's "flops" for this kernel)
  ctx.pending_flops = (double)ht.size() * (kS * (kS + 1) / 2) * 2.0 * kBM * kBN * (double)per * kBK;
  ctx.launch_begin();
  k_oz_gram<<<(unsigned)ht.size(), kGramThreads, kGramSmem, ctx.stream>>>(
      A.map, B.map, dj, dt, A.plane_rows, B.plane_rows, part);
  ctx.check_launch("k_oz_gram");
  ctx.launch_begin();
  if (nsplit == 1)
    k_oz_combine<1><<<(unsigned)outs, 512, 0, ctx.stream>>>(dj, dt, part, 1);
  else
    k_oz_combine<0><<<(unsigned)outs, 512, 0, ctx.stream>>>(dj, dt, part, nsplit);
  ctx.check_launch("k_oz_combine");
}

constexpr size_t kPlaneBudget = size_t(4) << 30;  // digit planes + level tiles per launch

}  // namespace

void ozaki_gram_batch(Ctx& ctx, const std::vector<GemmDesc>& descs) {
  if (descs.empty()) return;
  int Kmax = 0;
  for (const auto& d : descs) Kmax = std::max(Kmax, d.K);
  const long long kpad = (long long)ceil_div(Kmax, kBK) * kBK;
  size_t i0 = 0;
  while (i0 < descs.size()) {
    size_t i1 = i0;
    long long used = 0;
    while (i1 < descs.size()) {
      const long long qp = (long long)ceil_div(descs[i1].M, kBN) * kBN;
      // planes (S q_pad K_pad bytes) + level tiles (~ S q_pad^2 / 2 int32)
      const long long need = kS * qp * kpad + 2LL * kS * qp * (qp + kBN);
      if (i1 > i0 && (size_t)(used + need) > kPlaneBudget) break;
      used += need;
      ++i1;
    }
    Arena::Mark mk = ctx.arena.mark();
    std::vector<OzLeaf> src;
    for (size_t i = i0; i < i1; ++i) {
      const GemmDesc& d = descs[i];
      src.push_back({static_cast<const float*>(d.A), d.lda, d.K, d.M, 0, d.C, d.ldc, nullptr,
                     nullptr});
    }
    PlaneSet ps = slice_cols(ctx, src, kpad);
    std::vector<OzJob> jobs;
    for (size_t i = i0; i < i1; ++i) {
      const OzLeaf& l = src[i - i0];
      jobs.push_back({l.row_base, l.row_base, descs[i].C, descs[i].ldc, l.scale, l.scale,
                      descs[i].M, descs[i].M, 1});
    }
    run_products(ctx, ps, ps, jobs);
    ctx.arena.release(mk);
    i0 = i1;
  }
}

void ozaki_gemm_batch(Ctx& ctx, bool trans_a, const std::vector<GemmDesc>& descs) {
  if (descs.empty()) return;
  int Kmax = 0;
  for (const auto& d : descs) Kmax = std::max(Kmax, d.K);
  const long long kpad = (long long)ceil_div(Kmax, kBK) * kBK;
  // split every product into row chunks whose A planes fit half the budget
  struct Piece {
    const GemmDesc* d;
    int m0, mc;
  };
  const long long chunk_rows =
      std::max<long long>(kBN, (long long)(kPlaneBudget / 2 / (kS * kpad)) / kBN * kBN);
  std::vector<Piece> pieces;
  for (const auto& d : descs)
    for (int m0 = 0; m0 < d.M; m0 += (int)chunk_rows)
      pieces.push_back({&d, m0, (int)std::min<long long>(chunk_rows, d.M - m0)});
  size_t i0 = 0;
  while (i0 < pieces.size()) {
    size_t i1 = i0;
    long long used = 0;
    while (i1 < pieces.size()) {
      const long long mp = (long long)ceil_div(pieces[i1].mc, kBN) * kBN;
      const long long need = kS * (mp + kBN) * kpad + 16LL * kS * kBM * kBN * (mp / kBM);
      if (i1 > i0 && (size_t)(used + need) > kPlaneBudget) break;
      used += need;
      ++i1;
    }
    Arena::Mark mk = ctx.arena.mark();
    std::vector<OzLeaf> acol;
    std::vector<OzRows> arow, brow;
    for (size_t i = i0; i < i1; ++i) {
      const Piece& pc = pieces[i];
      const GemmDesc& d = *pc.d;
      const float* A = static_cast<const float*>(d.A);
      if (trans_a)  // op(A) rows = rows of a row-major fp32 matrix (ld = lda), K contiguous
        arow.push_back({A + (long long)pc.m0 * d.lda, 0, d.lda, pc.mc, d.K, 0, nullptr});
      else  // op(A) rows = columns of a row-major fp32 K x M block: transposed planes
        acol.push_back({A + pc.m0, d.lda, d.K, pc.mc, 0, nullptr, 0, nullptr, nullptr});
      // B: column-major K x N fp64; its columns are the operand rows
      brow.push_back({d.B, 1, d.ldb, d.N, d.K, 0, nullptr});
    }
    PlaneSet pa = trans_a ? slice_rows(ctx, arow, kpad) : slice_cols(ctx, acol, kpad);
    PlaneSet pb = slice_rows(ctx, brow, kpad);
    std::vector<OzJob> jobs;
    for (size_t i = i0; i < i1; ++i) {
      const Piece& pc = pieces[i];
      const GemmDesc& d = *pc.d;
      const long long ar = trans_a ? arow[i - i0].row_base : acol[i - i0].row_base;
      const double* sa = trans_a ? arow[i - i0].scale : acol[i - i0].scale;
      jobs.push_back({ar, brow[i - i0].row_base, d.C + pc.m0, d.ldc, sa, brow[i - i0].scale,
                      pc.mc, d.N, 0});
    }
    run_products(ctx, pa, pb, jobs);
    ctx.arena.release(mk);
    i0 = i1;
  }
}

}  // namespace hsvdcu
