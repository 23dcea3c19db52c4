// Host orchestrator of the hierarchical merge-and-truncate SVD on one B200
// (and, with a communicator, on the row shards of several).
#pragma once

#include <memory>
#include <vector>

#include "ctx.h"
#include "gemm.h"

namespace hsvdcu {

// Device factor: one (or two) column-major bases + sigma, all in ctx.arena.
struct DFac {
  double* B = nullptr;  // carried basis, dim x rank (col-major, ld)
  long long ld = 0;
  int dim = 0;
  int rank = 0;
  double* sigma = nullptr;
  bool degenerate = false;
  double* B2 = nullptr;  // optional other side (dim2 x rank)
  long long ld2 = 0;
  int dim2 = 0;
};

// Row-major m x n matrix on the device (reference DenseMatrix layout).
// Row chunk [.., row_end) of a staged input is resident once `ev` completes.
struct RowChunk {
  long long row_end;
  cudaEvent_t ev;
};

// Host thread that copies a pageable host input through pinned buffers
// (capi.cu): chunk i's DMA and event are issued once wait_issued(i) returns.
class HostStager {
 public:
  virtual ~HostStager() = default;
  virtual void wait_issued(size_t i) = 0;
};

struct XView {
  const void* X;
  DType dt;
  long long ld;
  long long m, n;
  // non-empty when X is still being copied in on the context's copy stream:
  // work on rows < row_end must wait for the chunk's event first
  std::vector<RowChunk> ready = {};
  // set when the chunks are issued by a host staging thread (pageable input)
  std::shared_ptr<HostStager> stager = {};
};

// Orders ctx.stream after chunk i of a staged input (waits on the host for
// a staging thread to have issued it first).
void x_wait_chunk(Ctx& ctx, const XView& x, size_t i);

// Orders ctx.stream after the copies of rows [0, row_end) (all rows: -1).
void x_wait_rows(Ctx& ctx, const XView& x, long long row_end = -1);

struct Block {
  long long r0;
  int d;
  long long c0;
  int c;
};

struct Slice {
  long long start;
  long long count;
};
std::vector<Slice> partition(long long extent, long long block);  // hierarchy.cpp:11-18

struct HsvdConfig {
  double gamma = 1e-2;
  long long d = 0, c = 0;
  int cap = 0;  // max_rank, 0 = none
};

// Leaf Grams G = Xt Xt^T (tall blocks, SYRK descriptors): fp32 on the
// tcgen05 int8 Ozaki path, fp64 on the DMMA SYRK (engine.cu).
void leaf_gram_tall(Ctx& ctx, DType dt, const std::vector<GemmDesc>& descs);

// op(A) B projections of the fp32/fp64 input onto fp64 factors (tcgen05
// Ozaki GEMM when applicable, else DMMA): engine.cu.
void project_x(Ctx& ctx, DType xt, bool trans_a, const std::vector<GemmDesc>& descs);

// Exact thin SVD of each block, truncated (hierarchy.cpp:57: truncate_factor
// (full_svd(block))).  keep_both: also return the other side in B2.
std::vector<DFac> block_svd_batch(Ctx& ctx, const XView& x, const std::vector<Block>& blocks,
                                  double gamma, int cap, bool keep_both, bool write_all);

// merge_pair_qr semantics (merge.cpp:71-117) for a batch of pairs sharing
// the basis dimension per pair.
std::vector<DFac> merge_batch(Ctx& ctx, const std::vector<std::pair<DFac, DFac>>& pairs,
                              double gamma, int cap);

// Several independent trees advanced level by level (hierarchy.cpp:31-48).
std::vector<DFac> tree_merge_many(Ctx& ctx, std::vector<std::vector<DFac>> trees, double gamma,
                                  int cap, long long* pair_merges);

// hierarchy.cpp:83-85 for every row slice: SVD of U_j^T X_j -> (sigma, V_j).
std::vector<DFac> vrecover_batch(Ctx& ctx, const XView& x, const std::vector<Slice>& rows,
                                 const std::vector<DFac>& us, double gamma, int cap);

// Nearly orthonormal B (rows x k) -> B R^{-1}, B^T B = R^T R (new buffer).
double* reorthonormalize(Ctx& ctx, const double* B, long long ld, int rows, int k);

// hierarchy.cpp:65-94 -> (sigma, V).
DFac hierarchical_svd(Ctx& ctx, const XView& x, const HsvdConfig& cfg);

// Row-slice ownership of rank `rank` in a world of `world` ranks.
void shard_rows(long long m_total, long long d, int rank, int world, long long* row0,
                long long* m_local, int* first_slice, int* last_slice);

class Comm;
// hierarchical_svd + recover_left_vectors over row shards (one rank per GPU):
// returns U (this rank's rows) in B, V (replicated) in B2.
DFac rank_k_svd_sharded(Ctx& ctx, Comm& comm, const XView& x_local, long long m_total,
                        long long row0, const HsvdConfig& cfg);

// hierarchy.cpp:50-63
DFac svd_of_col_slices(Ctx& ctx, const XView& x, long long c, double gamma, int cap);

// hierarchy.cpp:96-112 -> U (m x r) in B, V (n x r) in B2.
DFac recover_left_vectors(Ctx& ctx, const XView& x, const double* v_r, long long ldv, int r);

// refine.hpp:9-21 / refine.cpp:26-72 -> U in B (m x r), V in B2 (n x r).
struct RefineStats {
  int iterations = 0;
  double final_error = 0.0;
  bool converged = false;
};
DFac refine_factors(Ctx& ctx, const XView& x, const double* v_hat, long long ldv, int r,
                    const std::vector<double>& sigma_hat, double epsilon, int max_iters,
                    RefineStats* stats);

// Reads back ranks / degenerate flags written by finalize (synchronises).
void fetch_ranks(Ctx& ctx, const int* d_ranks, int count, std::vector<int>& out);

}  // namespace hsvdcu
