// Internals shared by the two translation units of the batched fp64
// symmetric eigensolver (see syev.cu for the algorithm overview):
//   syev.cu       one-stage reduction, tridiagonal eigenpairs, cluster
//                 Gram-Schmidt, compact-WY back-transform, eig_topk driver;
//   syev_band.cu  two-stage reduction (dense -> band -> tridiagonal) and the
//                 band-side eigenvector steps.
#pragma once

#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "gemm.h"
#include "syev.h"

namespace hsvdcu {
namespace syev_impl {

namespace cg = cooperative_groups;


constexpr int TRD_THREADS = 1024;
constexpr int TRD_QMAX = 8;  // rows per thread when n > 1024 (n <= 8192)
constexpr int EIG_THREADS = 512;
constexpr int NB = 32;       // reflectors per compact-WY block
constexpr int B2 = 32;       // bandwidth of the two-stage reduction
constexpr int LDBB = 2 * B2 + 2;  // band storage: diagonals 0..2*B2 (chase fill) + pad (16-byte columns)
constexpr int kBandInvitMinN = 1 << 30;  // band inverse iteration: only when forced
constexpr int kBandGroupDefault = 4;  // panels per delayed trailing update (two-stage stage 1)
constexpr int INV_WARPS = 4;      // warps (= LU workspace slots) per band inverse iteration CTA
constexpr int NBT = 128;     // reflectors per back-transform block (k_build_t)


struct EigDev {
  double* A;
  long long lda;
  int n;
  int kk;
  double* d;
  double* e;
  double* tau;
  double* lam;
  double* Z;
  long long ldz;
  double* piv;   // 2 * n * kk scratch (k_steig: LDL^T pivots + iterates, [n][kk])
  double* T;     // (nblocks * NBT * NBT) compact-WY T factors
  double* S;     // (nblocks * NBT * NBT) V^T V of each reflector block
  double* VW;    // n x 2*NB panel [V | W] (blocked tridiagonalisation)
  double* WV;    // n x 2*NB panel [W | V]
  // two-stage path
  int vals_only;     // k_steig: 1 eigenvalues (+ shifts, clusters) only; 2 vectors
                     // without the in-iteration Gram-Schmidt (k_band_mgs follows)
  double* shifts;    // kk perturbed inverse-iteration shifts
  int* cstarts;      // kk cluster starts
  double* band;      // (2*B2+1) x n lower band, chased to tridiagonal
  double* band0;     // copy of the band after stage 1 (inverse iteration)
  double* Tp;        // npanels x B2 x B2 panel T factors
  double* psum;      // 8 x B2 x B2 per-CTA partials of V^T V (k_panel_qr)
  double* Y;         // n x B2
  double* P1;        // B2 x B2
  double* Mb;        // B2 x B2
  double* Z1;        // (2*B2*group) x B2: pending-update products
  double* lu;        // per-warp band LU workspace (cpm * INV_WARPS slots per matrix)
  double* trig;      // k_steig's d, e, e^2 in global memory (n too large for shared memory), or null
  double* pscr;      // k_panel_qr's panel in global memory (n too large for shared memory), or null
  double* refl;      // chase reflectors, step-major: (refl_off(n, k) + s) * RS (v[0..31], tau, pad)
  double* q2T;       // WY T factors of the Q2 blocks, step-major: (tblk_off(n, k) + a) * 64
  long long lu_slot;  // doubles per slot
};

__device__ __forceinline__ double guard_pivot(double D, double tiny) {
  if (fabs(D) < tiny) return D < 0.0 ? -tiny : tiny;
  return D;
}

__device__ __forceinline__ unsigned hash32(unsigned x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

// Chase reflector storage (two-stage path).  Sweep s, step k acts on rows
// s+1+B2*k .. s+B2+B2*k; step k exists for sweeps 0 .. n-3-B2*k, so the
// reflectors are stored step-major (the WY blocks of k_q2_wy are runs of
// consecutive sweeps at one step: one contiguous bulk copy each).
constexpr int RS = 34;  // doubles per stored reflector: v[0..31], tau, pad (272 B, 16-byte multiple)
constexpr int QG = 8;   // sweeps per WY block of the Q2 back-transform (group a: sweeps QG*a-1 ..)
__host__ __device__ __forceinline__ int chase_steps(int n) { return n < 3 ? 0 : (n - 3) / B2 + 1; }
__host__ __device__ __forceinline__ long long refl_off(int n, int k) {  // first entry of step k
  return (long long)k * (n - 2) - (long long)(B2 / 2) * k * (k - 1);
}
// groups with a sweep at step k: A_k = A_0 - (B2/QG) k
__host__ __device__ __forceinline__ int tgroups0(int n) { return (n - 2) / QG + 1; }
__host__ __device__ __forceinline__ long long tblk_off(int n, int k) {
  return (long long)k * tgroups0(n) - (long long)(B2 / QG / 2) * k * (k - 1);
}

// element (i, j), i >= j, of the lower band storage (two-stage path)
__device__ __forceinline__ double& band_at(double* bb, int i, int j) {
  return bb[(i - j) + (long long)j * LDBB];
}

// Host steps shared between the translation units (all on ctx.stream; dd is
// the device copy of dev made by upload_jobs).
const EigDev* upload_jobs(Ctx& ctx, const std::vector<EigDev>& dev);
// k_steig: top-kk eigenvalues of the tridiagonal (d, e) + vectors or shifts
void launch_steig(Ctx& ctx, const EigDev* dd, int count, int nmax, int kkmax);
// k_band_mgs: orthonormalise the vectors of every eigenvalue cluster in Z
void launch_band_mgs(Ctx& ctx, const EigDev* dd, const std::vector<EigDev>& dev);
// Z <- Q Z through the reflectors stored in A (unit at row j + off)
void back_prepare(Ctx& ctx, const std::vector<EigDev>& dev, const EigDev* dd, int nmax, int off);
void back_apply(Ctx& ctx, const std::vector<EigJob>& jobs, const std::vector<EigDev>& dev, int nmax,
                int off);
void back_transform(Ctx& ctx, const std::vector<EigJob>& jobs, const std::vector<EigDev>& dev,
                    const EigDev* dd, int nmax, int off);
// two-stage path of eig_topk (syev_band.cu)
void two_stage(Ctx& ctx, const std::vector<EigJob>& jobs, std::vector<EigDev>& dev, int nmax,
               int kkmax);

}  // namespace syev_impl
}  // namespace hsvdcu
