// C ABI (include/hsvd_cu.h) over the device engine.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hsvd_cu.h"
#include "comm.h"
#include "engine.h"
#include "factor_ops.h"
#include "jacobi.h"
#include "metrics.h"
#include "ozaki.h"
#include "syev.h"

using namespace hsvdcu;

struct hsvd_cu_ctx {
  Ctx c;
  long long generation = 0;
  std::unique_ptr<Comm> comm;
  // matrix loaded by hsvd_cu_load_hsvd1 (outside the per-call arena)
  double* loaded = nullptr;
  size_t loaded_cap = 0;
  ~hsvd_cu_ctx() {
    if (loaded) cudaFree(loaded);
  }
};

struct hsvd_cu_group {
  std::shared_ptr<ThreadGroup> g;
};

struct hsvd_cu_result {
  hsvd_cu_ctx* ctx = nullptr;
  long long gen = 0;
  int rank = 0;
  bool degenerate = false;
  const double* sigma = nullptr;
  const double* u = nullptr;
  long long ldu = 0, u_rows = 0;
  const double* v = nullptr;
  long long ldv = 0, v_rows = 0;
};

namespace {

thread_local std::string g_err;
thread_local long long g_err_rows = 0, g_err_cols = 0;

int fail(int code, const std::string& msg, long long rows = 0, long long cols = 0) {
  g_err = msg;
  g_err_rows = rows;
  g_err_cols = cols;
  return code;
}

template <typename F>
int guarded(F&& f) {
  try {
    g_err.clear();
    return f();
  } catch (const Error& e) {
    return fail(e.code, e.what(), e.rows, e.cols);
  } catch (const std::bad_alloc&) {
    return fail(HSVD_CU_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(HSVD_CU_EINVAL, e.what());
  }
}

void begin(hsvd_cu_ctx* ctx) {
  if (!ctx) throw Error(kInvalid, "null context");
  HSVD_CUDA(cudaSetDevice(ctx->c.device));
  ctx->c.nvtx_close();
  ctx->c.arena.reset();
  // a call that failed between a side-stream fork and its join may have left
  // side work queued: the new call's stream waits for it before reusing memory
  ctx->c.side_join();
  ctx->c.side_arena.reset();
  ++ctx->generation;
}

DType dtype_of(int dt) {
  if (dt == HSVD_CU_F32) return DType::F32;
  if (dt == HSVD_CU_F64) return DType::F64;
  throw Error(kInvalid, "dtype must be HSVD_CU_F32 or HSVD_CU_F64");
}

// Pageable host input (the C++ drop-in's std::vector storage): a copy
// straight from it is staged by the driver and serialises with the caller.
// Instead a host thread copies row chunks into a ring of pinned buffers
// (the memcpy split over several threads) and issues each chunk's DMA on the
// copy stream, while the calling thread launches the Grams of the chunks
// already issued (x_wait_chunk blocks only until a chunk is issued).
class PageableStager final : public HostStager {
 public:
  // Pageable host input: every 64 MB chunk is copied into one of the
  // context's pinned slots by a persistent pool of host threads (created once
  // per call: spawning threads per chunk cost ~10% of the copy), then DMAed
  // on the copy stream while the pool fills the next slot.
  PageableStager(Ctx& c, char* dst, const char* src, int64_t row_bytes, int64_t src_pitch,
                 std::vector<int64_t> ends, std::vector<cudaEvent_t> evs)
      : c_(c), dst_(dst), src_(src), row_bytes_(row_bytes), pitch_(src_pitch),
        ends_(std::move(ends)), evs_(std::move(evs)) {
    const unsigned hw = std::thread::hardware_concurrency();
    // leave a core to the caller's thread (it keeps launching the compute)
    nt_ = std::max<size_t>(1, std::min<size_t>(16, hw > 2 ? hw - 2 : 1));
    for (size_t w = 1; w < nt_; ++w) {
      try {
        pool_.emplace_back([this, w] { worker(w); });
      } catch (...) {
        nt_ = w;  // fewer workers
        break;
      }
    }
    th_ = std::thread([this] { run(); });
  }
  ~PageableStager() override {
    if (th_.joinable()) th_.join();
    {
      std::lock_guard<std::mutex> lk(pm_);
      quit_ = true;
    }
    pcv_.notify_all();
    for (auto& t : pool_) t.join();
  }
  void wait_issued(size_t i) override {
    std::unique_lock<std::mutex> lk(mu_);
    cv_.wait(lk, [&] { return issued_ > i || failed_; });
    if (failed_) throw Error(kCuda, "host staging of the input failed: " + why_);
  }

 private:
  // rows [a, b) of the current chunk (pinned slot pin_, first row r0_)
  void piece(size_t w) {
    const int64_t per = (rows_ + (int64_t)nt_ - 1) / (int64_t)nt_;
    const int64_t a = std::min(rows_, (int64_t)w * per), b = std::min(rows_, a + per);
    if (pitch_ == row_bytes_) {
      if (b > a)
        std::memcpy(pin_ + a * row_bytes_, src_ + (r0_ + a) * pitch_, (size_t)((b - a) * row_bytes_));
    } else {
      for (int64_t r = a; r < b; ++r)
        std::memcpy(pin_ + r * row_bytes_, src_ + (r0_ + r) * pitch_, (size_t)row_bytes_);
    }
  }
  void worker(size_t w) {
    uint64_t seen = 0;
    while (true) {
      {
        std::unique_lock<std::mutex> lk(pm_);
        pcv_.wait(lk, [&] { return quit_ || gen_ != seen; });
        if (quit_) return;
        seen = gen_;
      }
      piece(w);
      {
        std::lock_guard<std::mutex> lk(pm_);
        ++done_;
      }
      pcv_.notify_all();
    }
  }
  void run() {
    try {
      HSVD_CUDA(cudaSetDevice(c_.device));
      cudaStream_t cs = c_.get_copy_stream();
      int64_t r0 = 0;
      for (size_t i = 0; i < ends_.size(); ++i) {
        const int slot = static_cast<int>(i % Ctx::kH2dSlots);
        HSVD_CUDA(cudaEventSynchronize(c_.h2d_ev[slot]));  // slot's previous DMA done
        const int64_t rows = ends_[i] - r0;
        {
          std::lock_guard<std::mutex> lk(pm_);
          pin_ = static_cast<char*>(c_.h2d_pin[slot]);
          r0_ = r0;
          rows_ = rows;
          done_ = 0;
          ++gen_;
        }
        pcv_.notify_all();
        piece(0);
        {
          std::unique_lock<std::mutex> lk(pm_);
          pcv_.wait(lk, [&] { return done_ + 1 >= nt_; });
        }
        HSVD_CUDA(cudaMemcpyAsync(dst_ + r0 * row_bytes_, c_.h2d_pin[slot], (size_t)(rows * row_bytes_),
                                  cudaMemcpyHostToDevice, cs));
        HSVD_CUDA(cudaEventRecord(c_.h2d_ev[slot], cs));
        HSVD_CUDA(cudaEventRecord(evs_[i], cs));
        {
          std::lock_guard<std::mutex> lk(mu_);
          issued_ = i + 1;
        }
        cv_.notify_all();
        r0 = ends_[i];
      }
    } catch (const std::exception& e) {
      std::lock_guard<std::mutex> lk(mu_);
      failed_ = true;
      why_ = e.what();
      cv_.notify_all();
    }
  }
  Ctx& c_;
  char* dst_;
  const char* src_;
  int64_t row_bytes_, pitch_;
  std::vector<int64_t> ends_;
  std::vector<cudaEvent_t> evs_;
  std::thread th_;
  std::mutex mu_;
  std::condition_variable cv_;
  size_t issued_ = 0;
  bool failed_ = false;
  std::string why_;
  // copy pool
  std::vector<std::thread> pool_;
  size_t nt_ = 1;
  std::mutex pm_;
  std::condition_variable pcv_;
  uint64_t gen_ = 0;
  size_t done_ = 0;
  bool quit_ = false;
  char* pin_ = nullptr;
  int64_t r0_ = 0, rows_ = 0;
};

bool is_pageable(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

// Brings x to the device (contiguous, ld = n) unless it already is there.
// Host input: copied into the arena.  With chunk_rows > 0 the copy runs on
// the context's copy stream in row chunks of that height (one per row slice
// of the plan), each marked by an event, so the leaf Grams of the first
// slices overlap the transfer of the later ones (XView::ready).
constexpr size_t kPageableMin = size_t(64) << 20;  // smaller inputs: one driver-staged copy

XView stage_x(Ctx& c, const void* x, int dtype, int64_t m, int64_t n, int64_t ldx, int where,
              int64_t chunk_rows = 0) {
  if (!x) throw Error(kInvalid, "x is null");
  if (m <= 0 || n <= 0) throw Error(kInvalid, "matrix is empty");
  if (ldx < n) throw Error(kInvalid, "ldx < n");
  if (m > 0x7fffffffLL || n > 0x7fffffffLL) throw Error(kInvalid, "dimension exceeds 2^31-1");
  XView v{x, dtype_of(dtype), ldx, m, n};
  if (where == HSVD_CU_DEVICE) return v;
  const size_t es = v.dt == DType::F32 ? 4 : 8;
  void* d = c.arena.alloc((size_t)m * n * es);
  v.X = d;
  v.ld = n;
  const int64_t row_bytes = n * (int64_t)es;
  if ((size_t)(m * row_bytes) >= kPageableMin && row_bytes <= (int64_t)Ctx::kH2dChunk &&
      is_pageable(x)) {
    c.ensure_h2d_stage();
    // chunk ends: pinned-buffer sized, and cut at the row-slice boundaries
    const int64_t per = std::max<int64_t>(1, (int64_t)Ctx::kH2dChunk / row_bytes);
    std::vector<int64_t> ends;
    for (int64_t r = 0; r < m;) {
      int64_t e = std::min(m, r + per);
      if (chunk_rows > 0) e = std::min(e, (r / chunk_rows + 1) * chunk_rows);
      ends.push_back(e);
      r = e;
    }
    std::vector<cudaEvent_t> evs;
    for (size_t i = 0; i < ends.size(); ++i) {
      evs.push_back(c.get_chunk_event(i + 1));
      v.ready.push_back({ends[i], evs.back()});
    }
    // the arena block may still be in use by earlier work on the compute stream
    cudaStream_t cs = c.get_copy_stream();
    cudaEvent_t start = c.get_chunk_event(0);
    HSVD_CUDA(cudaEventRecord(start, c.stream));
    HSVD_CUDA(cudaStreamWaitEvent(cs, start, 0));
    v.stager = std::make_shared<PageableStager>(c, static_cast<char*>(d),
                                                static_cast<const char*>(x), row_bytes,
                                                ldx * (int64_t)es, std::move(ends), std::move(evs));
    if (chunk_rows <= 0 || chunk_rows >= m) {
      // the caller reads any row: order the compute stream after every chunk
      x_wait_rows(c, v);
      v.ready.clear();
    }
    return v;
  }
  if (chunk_rows <= 0 || chunk_rows >= m) {
    HSVD_CUDA(cudaMemcpy2DAsync(d, n * es, x, ldx * es, n * es, m, cudaMemcpyHostToDevice, c.stream));
    return v;
  }
  // the arena block may still be in use by earlier work on the compute stream
  cudaStream_t cs = c.get_copy_stream();
  cudaEvent_t start = c.get_chunk_event(0);
  HSVD_CUDA(cudaEventRecord(start, c.stream));
  HSVD_CUDA(cudaStreamWaitEvent(cs, start, 0));
  size_t k = 1;
  for (int64_t r = 0; r < m; r += chunk_rows, ++k) {
    const int64_t rows = std::min<int64_t>(chunk_rows, m - r);
    HSVD_CUDA(cudaMemcpy2DAsync(static_cast<char*>(d) + (size_t)r * n * es, n * es,
                                static_cast<const char*>(x) + (size_t)r * ldx * es, ldx * es,
                                n * es, rows, cudaMemcpyHostToDevice, cs));
    cudaEvent_t ev = c.get_chunk_event(k);
    HSVD_CUDA(cudaEventRecord(ev, cs));
    v.ready.push_back({r + rows, ev});
  }
  return v;
}

// Copy-chunk height for the overlapped input transfer: the plan's row slice
// (hierarchy.cpp:11-18 partition), when there are several.
int64_t overlap_rows(const HsvdConfig& hc, int64_t m) {
  const int64_t d = (hc.d < 1 || hc.d > m) ? m : hc.d;
  return d < m ? d : 0;
}

// Row-major host/device fp64 (rows x cols, ld) -> column-major device.
double* stage_rowmajor(Ctx& c, const double* a, int64_t rows, int64_t cols, int64_t ld, int where) {
  double* raw;
  if (where == HSVD_CU_DEVICE) {
    raw = const_cast<double*>(a);
  } else {
    raw = c.arena.alloc_n<double>((size_t)rows * cols);
    HSVD_CUDA(cudaMemcpy2DAsync(raw, cols * 8, a, ld * 8, cols * 8, rows, cudaMemcpyHostToDevice,
                                c.stream));
    ld = cols;
  }
  double* colm = c.arena.alloc_n<double>((size_t)rows * cols);
  rowmajor_to_colmajor(c, raw, ld, (int)rows, (int)cols, colm, rows);
  return colm;
}

hsvd_cu_result* make_result(hsvd_cu_ctx* ctx, const DFac& f, bool b_is_u, bool with_b2) {
  auto* r = new hsvd_cu_result();
  r->ctx = ctx;
  r->gen = ctx->generation;
  r->rank = f.rank;
  r->degenerate = f.degenerate;
  r->sigma = f.sigma;
  if (b_is_u) {
    r->u = f.B;
    r->ldu = f.ld;
    r->u_rows = f.dim;
    if (with_b2) {
      r->v = f.B2;
      r->ldv = f.ld2;
      r->v_rows = f.dim2;
    }
  } else {
    r->v = f.B;
    r->ldv = f.ld;
    r->v_rows = f.dim;
    if (with_b2) {
      r->u = f.B2;
      r->ldu = f.ld2;
      r->u_rows = f.dim2;
    }
  }
  return r;
}

void check_cfg(const hsvd_cu_config* cfg) {
  if (!cfg) throw Error(kInvalid, "MatConfig is null");
  if (cfg->gamma < 0.0 || !std::isfinite(cfg->gamma))
    throw Error(kInvalid, "MatConfig: gamma must be finite and >= 0");
  if (!(cfg->epsilon > 0.0)) throw Error(kInvalid, "MatConfig: epsilon must be > 0");
  if (cfg->max_iters < 1) throw Error(kInvalid, "MatConfig: max_iters must be >= 1");
  if (cfg->row_block_rows < 0 || cfg->col_block_cols < 0)
    throw Error(kInvalid, "MatConfig: block sizes must be >= 0");
  if (cfg->max_rank < 0) throw Error(kInvalid, "MatConfig: max_rank must be >= 1");
}

HsvdConfig to_cfg(const hsvd_cu_config* cfg) {
  HsvdConfig h;
  h.gamma = cfg->gamma;
  h.d = cfg->row_block_rows;
  h.c = cfg->col_block_cols;
  h.cap = cfg->max_rank > 0 ? (int)std::min<int64_t>(cfg->max_rank, 0x7fffffff) : 0;
  return h;
}

int cap_of(int64_t max_rank) { return max_rank > 0 ? (int)std::min<int64_t>(max_rank, 0x7fffffff) : 0; }

DFac stage_factor(Ctx& c, const hsvd_cu_factor_in& f) {
  if (!f.basis || !f.sigma) throw Error(kInvalid, "merge: factor requires a carried basis");
  if (f.rank < 1 || f.dim < 1) throw Error(kInvalid, "merge: factor is empty");
  DFac d;
  d.dim = (int)f.dim;
  d.rank = (int)f.rank;
  d.ld = f.dim;
  d.B = stage_rowmajor(c, f.basis, f.dim, f.rank, f.ld > 0 ? f.ld : f.rank, HSVD_CU_HOST);
  d.sigma = c.arena.alloc_n<double>(f.rank);
  HSVD_CUDA(cudaMemcpyAsync(d.sigma, f.sigma, f.rank * sizeof(double), cudaMemcpyHostToDevice,
                            c.stream));
  d.degenerate = f.degenerate != 0;
  return d;
}

int check_result(const hsvd_cu_result* r) {
  if (!r) return fail(HSVD_CU_EINVAL, "null result");
  if (!r->ctx || r->ctx->generation != r->gen)
    return fail(HSVD_CU_EINVAL, "stale result: the context has run another call since");
  return HSVD_CU_OK;
}

// Device -> caller host memory.  Large results go through two pinned chunks
// alternately: the DMA of one chunk overlaps the host copy of the previous
// one, and that host copy (which also faults in the caller's fresh pages,
// the slow part for pageable memory) is split over several threads.
void copy_to_host(Ctx& c, void* dst, const void* src, size_t bytes) {
  constexpr size_t kSmall = size_t(8) << 20;
  if (bytes < kSmall) {
    HSVD_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c.stream));
    HSVD_CUDA(cudaStreamSynchronize(c.stream));
    return;
  }
  c.ensure_d2h_stage();
  constexpr size_t kChunk = Ctx::kD2hChunk;
  char* d = static_cast<char*>(dst);
  const char* s = static_cast<const char*>(src);
  const size_t nch = (bytes + kChunk - 1) / kChunk;
  auto len_of = [&](size_t i) { return std::min(kChunk, bytes - i * kChunk); };
  auto issue = [&](size_t i) {
    HSVD_CUDA(cudaMemcpyAsync(c.d2h_pin[i & 1], s + i * kChunk, len_of(i), cudaMemcpyDeviceToHost,
                              c.stream));
    HSVD_CUDA(cudaEventRecord(c.d2h_ev[i & 1], c.stream));
  };
  const unsigned hw = std::thread::hardware_concurrency();
  const size_t nt = std::max(1u, std::min(8u, hw == 0 ? 1u : hw));
  issue(0);
  if (nch > 1) issue(1);
  for (size_t i = 0; i < nch; ++i) {
    HSVD_CUDA(cudaEventSynchronize(c.d2h_ev[i & 1]));
    const size_t len = len_of(i), part = (len + nt - 1) / nt;
    const char* from = static_cast<const char*>(c.d2h_pin[i & 1]);
    char* to = d + i * kChunk;
    std::vector<std::thread> th;
    for (size_t t = 1; t < nt && t * part < len; ++t) {
      auto piece = [=] { std::memcpy(to + t * part, from + t * part, std::min(part, len - t * part)); };
      try {
        th.emplace_back(piece);
      } catch (...) {  // no thread available: copy this piece here
        piece();
      }
    }
    std::memcpy(to, from, std::min(part, len));
    for (auto& x : th) x.join();
    if (i + 2 < nch) issue(i + 2);
  }
}

int copy_side(const hsvd_cu_result* r, const double* src, long long ld, long long rows, double* out) {
  if (int s = check_result(r)) return s;
  if (!src) return fail(HSVD_CU_EINVAL, "result has no such factor");
  return guarded([&] {
    Ctx& c = r->ctx->c;
    HSVD_CUDA(cudaSetDevice(c.device));
    Arena::Mark mk = c.arena.mark();
    double* tmp = c.arena.alloc_n<double>((size_t)rows * r->rank);
    colmajor_to_rowmajor(c, src, ld, (int)rows, r->rank, tmp, r->rank);
    copy_to_host(c, out, tmp, (size_t)rows * r->rank * 8);
    c.arena.release(mk);
    return HSVD_CU_OK;
  });
}

}  // namespace

extern "C" {

int hsvd_cu_version(void) { return 100; }
const char* hsvd_cu_last_error(void) { return g_err.c_str(); }
void hsvd_cu_last_error_dims(int64_t* rows, int64_t* cols) {
  if (rows) *rows = g_err_rows;
  if (cols) *cols = g_err_cols;
}

int hsvd_cu_ctx_create(int device, hsvd_cu_ctx** out) {
  if (!out) return fail(HSVD_CU_EINVAL, "out is null");
  *out = nullptr;
  return guarded([&] {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
      (void)cudaGetLastError();
      throw Error(kCuda, "no CUDA device available (this library has no CPU fallback)");
    }
    if (device < 0 || device >= n) throw Error(kInvalid, "device index out of range");
    auto* c = new hsvd_cu_ctx();
    try {
      c->c.device = device;
      HSVD_CUDA(cudaSetDevice(device));
      cudaDeviceProp prop;
      HSVD_CUDA(cudaGetDeviceProperties(&prop, device));
      if (prop.major < 10)
        throw Error(kCuda, std::string("device ") + prop.name + " is not sm_100 (Blackwell)");
      c->c.num_sms = prop.multiProcessorCount;
      HSVD_CUDA(cudaStreamCreateWithFlags(&c->c.stream, cudaStreamNonBlocking));
      c->c.own_stream = true;
      c->c.staging.init(size_t(8) << 20);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
    return HSVD_CU_OK;
  });
}

int hsvd_cu_ctx_destroy(hsvd_cu_ctx* ctx) {
  if (!ctx) return HSVD_CU_OK;
  cudaSetDevice(ctx->c.device);
  cudaStreamSynchronize(ctx->c.stream);
  if (ctx->c.own_stream) cudaStreamDestroy(ctx->c.stream);
  delete ctx;
  return HSVD_CU_OK;
}

int hsvd_cu_ctx_stream(hsvd_cu_ctx* ctx, void** stream) {
  if (!ctx || !stream) return fail(HSVD_CU_EINVAL, "null argument");
  *stream = ctx->c.stream;
  return HSVD_CU_OK;
}

int64_t hsvd_cu_launch_count(const hsvd_cu_ctx* ctx) { return ctx ? ctx->c.launches : 0; }
int64_t hsvd_cu_arena_bytes(const hsvd_cu_ctx* ctx) {
  return ctx ? (int64_t)(ctx->c.arena.capacity() + ctx->c.side_arena.capacity()) : 0;
}

int hsvd_cu_profile(hsvd_cu_ctx* ctx, int enable) {
  if (!ctx) return fail(HSVD_CU_EINVAL, "null context");
  ctx->c.profiling = enable != 0;
  return HSVD_CU_OK;
}

int64_t hsvd_cu_profile_report(hsvd_cu_ctx* ctx, char* buf, int64_t len) {
  if (!ctx) return -1;
  std::string out;
  int64_t rc = guarded([&] {
    Ctx& c = ctx->c;
    HSVD_CUDA(cudaSetDevice(c.device));
    HSVD_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<std::string> order;
    std::vector<std::pair<long long, double>> agg;
    std::vector<double> fl, by;
    for (auto& r : c.prof) {
      float ms = 0.f;
      HSVD_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
      size_t i = 0;
      while (i < order.size() && order[i] != r.name) ++i;
      if (i == order.size()) {
        order.push_back(r.name);
        agg.push_back({0, 0.0});
        fl.push_back(0.0);
        by.push_back(0.0);
      }
      agg[i].first += 1;
      agg[i].second += ms;
      fl[i] += r.flops;
      by[i] += r.bytes;
    }
    if (buf && len > 0) {  // a sizing query (buf == NULL) keeps the records
      for (auto& r : c.prof) {
        c.ev_free.push_back(r.a);
        c.ev_free.push_back(r.b);
      }
      c.prof.clear();
    }
    for (size_t i = 0; i < order.size(); ++i)
      out += order[i] + "\t" + std::to_string(agg[i].first) + "\t" + std::to_string(agg[i].second) +
             "\t" + std::to_string(fl[i]) + "\t" + std::to_string(by[i]) + "\n";
    return HSVD_CU_OK;
  });
  if (rc != HSVD_CU_OK) return -1;
  if (buf && len > 0) {
    const size_t n = std::min<size_t>(out.size(), (size_t)len - 1);
    std::memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return (int64_t)out.size() + 1;
}

int hsvd_cu_synchronize(hsvd_cu_ctx* ctx) {
  return guarded([&] {
    if (!ctx) throw Error(kInvalid, "null context");
    HSVD_CUDA(cudaStreamSynchronize(ctx->c.stream));
    return HSVD_CU_OK;
  });
}

int hsvd_cu_validate(const hsvd_cu_config* cfg) {
  return guarded([&] {
    check_cfg(cfg);
    return HSVD_CU_OK;
  });
}

int hsvd_cu_hierarchical_svd(hsvd_cu_ctx* ctx, const void* x, int dtype, int64_t m, int64_t n,
                             int64_t ldx, int where, const hsvd_cu_config* cfg,
                             hsvd_cu_result** out) {
  return guarded([&] {
    if (!out) throw Error(kInvalid, "out is null");
    *out = nullptr;
    if (!x || m <= 0 || n <= 0) throw Error(kInvalid, "hierarchical_svd: matrix is empty");
    check_cfg(cfg);
    begin(ctx);
    XView xv = stage_x(ctx->c, x, dtype, m, n, ldx, where);
    DFac f = hierarchical_svd(ctx->c, xv, to_cfg(cfg));
    *out = make_result(ctx, f, false, false);
    return HSVD_CU_OK;
  });
}

int hsvd_cu_recover_left_vectors(hsvd_cu_ctx* ctx, const void* x, int dtype, int64_t m, int64_t n,
                                 int64_t ldx, int where, const double* v_r, int64_t r,
                                 int64_t ldv, int v_where, hsvd_cu_result** out) {
  return guarded([&] {
    if (!out) throw Error(kInvalid, "out is null");
    *out = nullptr;
    if (!v_r || r < 1) throw Error(kInvalid, "recover_left_vectors: v_r must have x.cols() rows");
    begin(ctx);
    XView xv = stage_x(ctx->c, x, dtype, m, n, ldx, where);
    double* vd = stage_rowmajor(ctx->c, v_r, n, r, ldv > 0 ? ldv : r, v_where);
    DFac f = recover_left_vectors(ctx->c, xv, vd, n, (int)r);
    *out = make_result(ctx, f, true, true);
    return HSVD_CU_OK;
  });
}

int hsvd_cu_refine_factors(hsvd_cu_ctx* ctx, const void* x, int dtype, int64_t m, int64_t n,
                           int64_t ldx, int where, const double* v_hat, int64_t v_rows,
                           int64_t r, int64_t ldv, int v_where, const double* sigma_hat,
                           int64_t sigma_len, double epsilon, int32_t max_iters,
                           int32_t* iterations, double* final_error, int32_t* converged,
                           hsvd_cu_result** out) {
  return guarded([&] {
    if (!out) throw Error(kInvalid, "out is null");
    *out = nullptr;
    // refine.cpp:29-36 (argument checks in the reference's order)
    if (!(epsilon > 0.0)) throw Error(kInvalid, "refine_factors: epsilon must be > 0");
    if (max_iters < 1) throw Error(kInvalid, "refine_factors: max_iters must be >= 1");
    if (sigma_len != r || (r > 0 && !sigma_hat))
      throw Error(kInvalid, "refine_factors: sigma_hat length must match v_hat columns");
    if (v_rows != n || !v_hat || r < 1)
      throw Error(kInvalid, "refine_factors: v_hat must have x.cols() rows");
    begin(ctx);
    XView xv = stage_x(ctx->c, x, dtype, m, n, ldx, where);
    double* vd = stage_rowmajor(ctx->c, v_hat, n, r, ldv > 0 ? ldv : r, v_where);
    std::vector<double> sh(sigma_hat, sigma_hat + r);
    RefineStats st;
    DFac f = refine_factors(ctx->c, xv, vd, n, (int)r, sh, epsilon, max_iters, &st);
    if (iterations) *iterations = st.iterations;
    if (final_error) *final_error = st.final_error;
    if (converged) *converged = st.converged ? 1 : 0;
    *out = make_result(ctx, f, true, true);
    return HSVD_CU_OK;
  });
}

// ---- reconstruction-error evaluation ---------------
namespace {

struct UVDev {  // column-major device copy of (U S, V) heads, or views
  const double* u;
  long long ldu;
  const double* v;
  long long ldv;
  const double* sigma;
};

void check_uv(const hsvd_cu_factor_uv* f, const char* who) {
  if (!f || !f->u || !f->v || !f->sigma)
    throw Error(kInvalid, std::string(who) + ": factor must carry both u and v");
  if (f->m < 1 || f->n < 1 || f->rank < 1) throw Error(kInvalid, std::string(who) + ": empty factor");
}

UVDev stage_uv(Ctx& c, const hsvd_cu_factor_uv* f, long long k) {
  UVDev d;
  if (f->where == HSVD_CU_DEVICE) {
    d.u = f->u;
    d.ldu = f->ldu > 0 ? f->ldu : f->m;
    d.v = f->v;
    d.ldv = f->ldv > 0 ? f->ldv : f->n;
    d.sigma = f->sigma;
    return d;
  }
  // host row-major -> device column-major (the first k columns)
  d.u = stage_rowmajor(c, f->u, f->m, k, f->ldu > 0 ? f->ldu : f->rank, HSVD_CU_HOST);
  d.ldu = f->m;
  d.v = stage_rowmajor(c, f->v, f->n, k, f->ldv > 0 ? f->ldv : f->rank, HSVD_CU_HOST);
  d.ldv = f->n;
  double* s = c.arena.alloc_n<double>(k);
  HSVD_CUDA(cudaMemcpyAsync(s, f->sigma, k * sizeof(double), cudaMemcpyHostToDevice, c.stream));
  d.sigma = s;
  return d;
}

// ||sum_i s_i * U_i S_i V_i^T (+ X)||_F^2 for up to two factor heads
double heads_sumsq(Ctx& c, int m, int n, const UVDev& a, int ka, double sa, const UVDev* b, int kb,
                   double sb, const void* X, DType dt, long long ldx) {
  const int K = ka + (b ? kb : 0);
  double* A = c.arena.alloc_n<double>((size_t)m * K);
  double* B = c.arena.alloc_n<double>((size_t)n * K);
  scale_cols_copy(c, A, m, a.u, a.ldu, m, ka, a.sigma, sa);
  scale_cols_copy(c, B, n, a.v, a.ldv, n, ka, nullptr, 1.0);
  if (b) {
    scale_cols_copy(c, A + (size_t)m * ka, m, b->u, b->ldu, m, kb, b->sigma, sb);
    scale_cols_copy(c, B + (size_t)n * ka, n, b->v, b->ldv, n, kb, nullptr, 1.0);
  }
  return product_plus_sumsq(c, A, m, B, n, m, n, K, X, dt, ldx);
}

}  // namespace

int hsvd_cu_factor_diff_norm(hsvd_cu_ctx* ctx, const hsvd_cu_factor_uv* a,
                             const hsvd_cu_factor_uv* b, double* out) {
  return guarded([&] {
    if (!out) throw Error(kInvalid, "out is null");
    check_uv(a, "factor_diff_norm");
    check_uv(b, "factor_diff_norm");
    if (a->m != b->m || a->n != b->n)
      throw Error(kInvalid, "factor_diff_norm: factors must describe matrices of the same shape");
    begin(ctx);
    Ctx& c = ctx->c;
    c.phase = "metric";
    const UVDev da = stage_uv(c, a, a->rank), db = stage_uv(c, b, b->rank);
    *out = std::sqrt(heads_sumsq(c, (int)a->m, (int)a->n, da, (int)a->rank, 1.0, &db,
                                 (int)b->rank, -1.0, nullptr, DType::F64, 0));
    return HSVD_CU_OK;
  });
}

int hsvd_cu_rank_k_error(hsvd_cu_ctx* ctx, const hsvd_cu_factor_uv* full_of_x,
                         const hsvd_cu_factor_uv* approx, int64_t k, double* out) {
  return guarded([&] {
    if (!out) throw Error(kInvalid, "out is null");
    if (!approx || !approx->u || !approx->v)
      throw Error(kInvalid, "rank_k_error: approx must carry both u and v");
    if (k < 1 || k > approx->rank)
      throw Error(kInvalid, "rank_k_error: k must be in [1, approx.rank()]");
    check_uv(full_of_x, "rank_k_error");
    if (full_of_x->m != approx->m || full_of_x->n != approx->n)
      throw Error(kInvalid, "rank_k_error: factors must describe matrices of the same shape");
    begin(ctx);
    Ctx& c = ctx->c;
    c.phase = "metric";
    const long long kref = std::min<long long>(k, full_of_x->rank);  // svd_factor.cpp:72
    const UVDev df = stage_uv(c, full_of_x, kref), da = stage_uv(c, approx, k);
    const int m = (int)approx->m, n = (int)approx->n;
    // ||X_k||_F of the reconstructed reference head (svd_factor.cpp:73-74)
    const double denom =
        std::sqrt(heads_sumsq(c, m, n, df, (int)kref, 1.0, nullptr, 0, 0.0, nullptr, DType::F64, 0));
    if (denom == 0.0)
      throw Error(kInvalid, "rank_k_error: reference rank-k approximation is zero");
    const double num = std::sqrt(heads_sumsq(c, m, n, df, (int)kref, 1.0, &da, (int)k, -1.0,
                                             nullptr, DType::F64, 0));
    *out = num / denom;
    return HSVD_CU_OK;
  });
}

int hsvd_cu_residual_norm(hsvd_cu_ctx* ctx, const void* x, int dtype, int64_t m, int64_t n,
                          int64_t ldx, int where, const hsvd_cu_factor_uv* f, double* out) {
  return guarded([&] {
    if (!out) throw Error(kInvalid, "out is null");
    check_uv(f, "residual_norm");
    if (f->m != m || f->n != n)
      throw Error(kInvalid, "residual_norm: factor shape does not match x");
    begin(ctx);
    Ctx& c = ctx->c;
    c.phase = "metric";
    XView xv = stage_x(c, x, dtype, m, n, ldx, where);
    const UVDev d = stage_uv(c, f, f->rank);
    *out = std::sqrt(heads_sumsq(c, (int)m, (int)n, d, (int)f->rank, -1.0, nullptr, 0, 0.0, xv.X,
                                 xv.dt, xv.ld));
    return HSVD_CU_OK;
  });
}

// ---- HSVD1 loader (matrix_io.cpp:91-113), streamed to the device ---------
extern "C++" {
namespace {

template <typename T>
__global__ void k_all_finite(const T* __restrict__ x, long long count, int* __restrict__ bad) {
  int b = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    b |= !isfinite(x[i]);
  if (__syncthreads_or(b) && threadIdx.x == 0) atomicOr(bad, 1);
}

// HSVD1 (fp64 payload, matrix_io.cpp:91-113) and, when allow_f32, its fp32
// payload variant "HSVF1\0" (same 22-byte header layout, 4-byte elements).
int load_matrix(hsvd_cu_ctx* ctx, const char* path, bool allow_f32, int64_t* rows, int64_t* cols,
                int* dtype, const void** dev_x) {
  return guarded([&] {
    if (!ctx || !path || !rows || !cols || !dev_x) throw Error(kInvalid, "null argument");
    const std::string p(path);
    std::FILE* f = std::fopen(path, "rb");
    if (!f) throw Error(kIo, p + ": cannot open for reading");
    std::unique_ptr<std::FILE, int (*)(std::FILE*)> guard(f, &std::fclose);
    unsigned char header[22];
    if (std::fread(header, 1, sizeof(header), f) != sizeof(header))
      throw Error(kFormat, p + ": truncated header");
    static const char kMagic[6] = {'H', 'S', 'V', 'D', '1', '\0'};
    static const char kMagicF32[6] = {'H', 'S', 'V', 'F', '1', '\0'};
    bool f32 = false;
    if (std::memcmp(header, kMagic, sizeof(kMagic)) != 0) {
      if (allow_f32 && std::memcmp(header, kMagicF32, sizeof(kMagicF32)) == 0)
        f32 = true;
      else
        throw Error(kFormat, p + ": bad magic, not an HSVD1 file");
    }
    const size_t esize = f32 ? sizeof(float) : sizeof(double);
    auto u64 = [&](int off) {
      std::uint64_t v = 0;
      for (int i = 0; i < 8; ++i) v |= static_cast<std::uint64_t>(header[off + i]) << (8 * i);
      return v;
    };
    const std::uint64_t r = u64(6), c = u64(14);
    if (r == 0 || c == 0) throw Error(kFormat, p + ": empty matrix");
    constexpr std::uint64_t kMaxElems = std::uint64_t(1) << 34;
    if (r > kMaxElems || c > kMaxElems || r * c > kMaxElems)
      throw Error(kFormat, p + ": implausible dimensions");
    Ctx& cx = ctx->c;
    HSVD_CUDA(cudaSetDevice(cx.device));
    const size_t count = (size_t)(r * c), bytes = count * esize;
    if (ctx->loaded_cap < bytes) {
      if (ctx->loaded) HSVD_CUDA(cudaFree(ctx->loaded));
      ctx->loaded = nullptr;
      ctx->loaded_cap = 0;
      if (cudaMalloc(&ctx->loaded, bytes) != cudaSuccess) {
        (void)cudaGetLastError();
        throw Error(kNoMemory, p + ": device allocation for the matrix failed");
      }
      ctx->loaded_cap = bytes;
    }
    // two pinned chunks: the file read of one overlaps the copy of the other
    constexpr size_t kChunk = size_t(64) << 20;
    void* pin[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    auto cleanup = [&] {
      for (int i = 0; i < 2; ++i) {
        if (ev[i]) cudaEventDestroy(ev[i]);
        if (pin[i]) cudaFreeHost(pin[i]);
      }
    };
    try {
      for (int i = 0; i < 2; ++i) {
        HSVD_CUDA(cudaMallocHost(&pin[i], kChunk));
        HSVD_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
      }
      char* dst = reinterpret_cast<char*>(ctx->loaded);
      size_t done = 0;
      int b = 0;
      while (done < bytes) {
        const size_t len = std::min(kChunk, bytes - done);
        HSVD_CUDA(cudaEventSynchronize(ev[b]));  // this buffer's previous copy is done
        if (std::fread(pin[b], 1, len, f) != len) throw Error(kFormat, p + ": truncated payload");
        HSVD_CUDA(cudaMemcpyAsync(dst + done, pin[b], len, cudaMemcpyHostToDevice, cx.stream));
        HSVD_CUDA(cudaEventRecord(ev[b], cx.stream));
        done += len;
        b ^= 1;
      }
      int* bad = nullptr;
      HSVD_CUDA(cudaMalloc(&bad, sizeof(int)));
      HSVD_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), cx.stream));
      if (f32)
        k_all_finite<float><<<4 * cx.num_sms, 256, 0, cx.stream>>>(
            reinterpret_cast<const float*>(ctx->loaded), (long long)count, bad);
      else
        k_all_finite<double><<<4 * cx.num_sms, 256, 0, cx.stream>>>(ctx->loaded, (long long)count,
                                                                    bad);
      int hb = 0;
      HSVD_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, cx.stream));
      HSVD_CUDA(cudaStreamSynchronize(cx.stream));
      cudaFree(bad);
      if (hb) throw Error(kFormat, p + ": matrix contains NaN or Inf");
    } catch (...) {
      cudaStreamSynchronize(cx.stream);
      cleanup();
      throw;
    }
    cleanup();
    *rows = (int64_t)r;
    *cols = (int64_t)c;
    if (dtype) *dtype = f32 ? HSVD_CU_F32 : HSVD_CU_F64;
    *dev_x = ctx->loaded;
    return HSVD_CU_OK;
  });
}

}  // namespace
}  // extern "C++"

int hsvd_cu_load_hsvd1(hsvd_cu_ctx* ctx, const char* path, int64_t* rows, int64_t* cols,
                       const double** dev_x) {
  const void* p = nullptr;
  const int rc = load_matrix(ctx, path, false, rows, cols, nullptr, &p);
  if (rc == HSVD_CU_OK) *dev_x = static_cast<const double*>(p);
  return rc;
}

int hsvd_cu_load_matrix(hsvd_cu_ctx* ctx, const char* path, int64_t* rows, int64_t* cols,
                        int* dtype, const void** dev_x) {
  if (!dtype) return fail(HSVD_CU_EINVAL, "null argument");
  return load_matrix(ctx, path, true, rows, cols, dtype, dev_x);
}

int hsvd_cu_rank_k_svd(hsvd_cu_ctx* ctx, const void* x, int dtype, int64_t m, int64_t n,
                       int64_t ldx, int where, const hsvd_cu_config* cfg, hsvd_cu_result** out) {
  return guarded([&] {
    if (!out) throw Error(kInvalid, "out is null");
    *out = nullptr;
    if (!x || m <= 0 || n <= 0) throw Error(kInvalid, "hierarchical_svd: matrix is empty");
    check_cfg(cfg);
    begin(ctx);
    const HsvdConfig hc = to_cfg(cfg);
    XView xv = stage_x(ctx->c, x, dtype, m, n, ldx, where, overlap_rows(hc, m));
    DFac right = hierarchical_svd(ctx->c, xv, hc);
    DFac f = recover_left_vectors(ctx->c, xv, right.B, right.ld, right.rank);
    *out = make_result(ctx, f, true, true);
    return HSVD_CU_OK;
  });
}

int hsvd_cu_svd_of_col_slices(hsvd_cu_ctx* ctx, const void* x, int dtype, int64_t m, int64_t n,
                              int64_t ldx, int where, int64_t c, double gamma, int64_t max_rank,
                              hsvd_cu_result** out) {
  return guarded([&] {
    if (!out) throw Error(kInvalid, "out is null");
    *out = nullptr;
    begin(ctx);
    XView xv = stage_x(ctx->c, x, dtype, m, n, ldx, where);
    DFac f = svd_of_col_slices(ctx->c, xv, c, gamma, cap_of(max_rank));
    *out = make_result(ctx, f, true, false);
    return HSVD_CU_OK;
  });
}

int hsvd_cu_full_svd(hsvd_cu_ctx* ctx, const double* a, int64_t rows, int64_t cols, int64_t lda,
                     hsvd_cu_result** out) {
  return guarded([&] {
    if (!out) throw Error(kInvalid, "out is null");
    *out = nullptr;
    if (!a || rows <= 0 || cols <= 0) throw Error(kInvalid, "full_svd: matrix is empty");
    begin(ctx);
    XView xv = stage_x(ctx->c, a, HSVD_CU_F64, rows, cols, lda > 0 ? lda : cols, HSVD_CU_HOST);
    std::vector<DFac> f =
        block_svd_batch(ctx->c, xv, {{0, (int)rows, 0, (int)cols}}, 0.0, 0, true, true);
    // full_svd keeps every singular value (no truncation)
    int p = (int)std::min(rows, cols);
    f[0].rank = p;
    *out = make_result(ctx, f[0], true, true);
    return HSVD_CU_OK;
  });
}

int hsvd_cu_merge_pair(hsvd_cu_ctx* ctx, int orient, const hsvd_cu_factor_in* f1,
                       const hsvd_cu_factor_in* f2, double gamma, int64_t max_rank,
                       hsvd_cu_result** out) {
  return guarded([&] {
    if (!out) throw Error(kInvalid, "out is null");
    *out = nullptr;
    if (!f1 || !f2) throw Error(kInvalid, "merge: null factor");
    if (f1->dim != f2->dim)
      throw Error(kInvalid, orient == HSVD_CU_COLUMN_CONCAT
                                ? "merge: ColumnConcat factors must have equal row counts"
                                : "merge: RowConcat factors must have equal column counts");
    begin(ctx);
    DFac a = stage_factor(ctx->c, *f1), b = stage_factor(ctx->c, *f2);
    std::vector<DFac> r = merge_batch(ctx->c, {{a, b}}, gamma, cap_of(max_rank));
    *out = make_result(ctx, r[0], orient == HSVD_CU_COLUMN_CONCAT, false);
    return HSVD_CU_OK;
  });
}

int hsvd_cu_tree_merge(hsvd_cu_ctx* ctx, int orient, const hsvd_cu_factor_in* factors,
                       int64_t count, double gamma, int64_t max_rank, int64_t* pair_merges,
                       hsvd_cu_result** out) {
  return guarded([&] {
    if (!out) throw Error(kInvalid, "out is null");
    *out = nullptr;
    if (!factors || count < 1) throw Error(kInvalid, "tree_merge: factor list is empty");
    for (int64_t i = 1; i < count; ++i)
      if (factors[i].dim != factors[0].dim)
        throw Error(kInvalid, orient == HSVD_CU_COLUMN_CONCAT
                                  ? "merge: ColumnConcat factors must have equal row counts"
                                  : "merge: RowConcat factors must have equal column counts");
    begin(ctx);
    std::vector<DFac> fs;
    for (int64_t i = 0; i < count; ++i) fs.push_back(stage_factor(ctx->c, factors[i]));
    long long pm = 0;
    DFac f = tree_merge_many(ctx->c, {fs}, gamma, cap_of(max_rank), &pm).front();
    if (pair_merges) *pair_merges = pm;
    *out = make_result(ctx, f, orient == HSVD_CU_COLUMN_CONCAT, false);
    return HSVD_CU_OK;
  });
}

int hsvd_cu_syevx_topk(hsvd_cu_ctx* ctx, const double* a, int64_t n, int64_t kk, double* lam,
                       double* z) {
  return guarded([&] {
    if (!a || !lam || !z || n < 1 || kk < 1 || kk > n)
      throw Error(kInvalid, "syevx_topk: bad arguments");
    begin(ctx);
    Ctx& c = ctx->c;
    double* A = c.arena.alloc_n<double>((size_t)n * n);
    double* L = c.arena.alloc_n<double>(kk);
    double* Z = c.arena.alloc_n<double>((size_t)n * kk);
    HSVD_CUDA(cudaMemcpyAsync(A, a, (size_t)n * n * 8, cudaMemcpyHostToDevice, c.stream));
    eig_topk(c, {{A, n, (int)n, (int)kk, L, Z, n}});
    HSVD_CUDA(cudaMemcpyAsync(lam, L, kk * 8, cudaMemcpyDeviceToHost, c.stream));
    HSVD_CUDA(cudaMemcpyAsync(z, Z, (size_t)n * kk * 8, cudaMemcpyDeviceToHost, c.stream));
    HSVD_CUDA(cudaStreamSynchronize(c.stream));
    return HSVD_CU_OK;
  });
}

int hsvd_cu_syevx_topk_batch(hsvd_cu_ctx* ctx, const double* a, int64_t count, int64_t n,
                             int64_t kk, double* lam, double* z) {
  return guarded([&] {
    if (!a || !lam || !z || count < 1 || n < 1 || kk < 1 || kk > n)
      throw Error(kInvalid, "syevx_topk_batch: bad arguments");
    begin(ctx);
    Ctx& c = ctx->c;
    double* A = c.arena.alloc_n<double>((size_t)count * n * n);
    double* L = c.arena.alloc_n<double>((size_t)count * kk);
    double* Z = c.arena.alloc_n<double>((size_t)count * n * kk);
    HSVD_CUDA(cudaMemcpyAsync(A, a, (size_t)count * n * n * 8, cudaMemcpyHostToDevice, c.stream));
    std::vector<EigJob> jobs;
    for (int64_t g = 0; g < count; ++g)
      jobs.push_back({A + g * n * n, n, (int)n, (int)kk, L + g * kk, Z + g * n * kk, n});
    eig_topk(c, jobs);
    HSVD_CUDA(cudaMemcpyAsync(lam, L, (size_t)count * kk * 8, cudaMemcpyDeviceToHost, c.stream));
    HSVD_CUDA(cudaMemcpyAsync(z, Z, (size_t)count * n * kk * 8, cudaMemcpyDeviceToHost, c.stream));
    HSVD_CUDA(cudaStreamSynchronize(c.stream));
    return HSVD_CU_OK;
  });
}

int hsvd_cu_qr_thin(hsvd_cu_ctx* ctx, const double* a, int64_t m, int64_t n, int64_t lda,
                    double* q, double* r) {
  return guarded([&] {
    if (!a || m <= 0 || n <= 0) throw Error(kInvalid, "qr_thin: matrix is empty");
    if (!q || !r || lda < n) throw Error(kInvalid, "qr_thin: bad arguments");
    if (m > 0x7fffffffLL || n > 0x7fffffffLL) throw Error(kInvalid, "qr_thin: dimension too large");
    begin(ctx);
    Ctx& c = ctx->c;
    const int64_t p = std::min(m, n);
    double* A = stage_rowmajor(c, a, m, n, lda, HSVD_CU_HOST);  // column-major m x n
    double* Q = c.arena.alloc_n<double>((size_t)m * p);
    householder_qr(c, A, (int)m, (int)n, Q);
    std::vector<double> ha((size_t)m * n), hq((size_t)m * p);
    HSVD_CUDA(cudaMemcpyAsync(ha.data(), A, ha.size() * 8, cudaMemcpyDeviceToHost, c.stream));
    HSVD_CUDA(cudaMemcpyAsync(hq.data(), Q, hq.size() * 8, cudaMemcpyDeviceToHost, c.stream));
    HSVD_CUDA(cudaStreamSynchronize(c.stream));
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < p; ++j) q[i * p + j] = hq[i + j * m];
    for (int64_t i = 0; i < p; ++i)
      for (int64_t j = 0; j < n; ++j) r[i * n + j] = j >= i ? ha[i + j * m] : 0.0;
    return HSVD_CU_OK;
  });
}

int hsvd_cu_block_gram(hsvd_cu_ctx* ctx, const void* x, int dtype, int64_t d, int64_t c,
                       int64_t ldx, int where, double* g) {
  return guarded([&] {
    if (!g) throw Error(kInvalid, "block_gram: g is null");
    begin(ctx);
    Ctx& cc = ctx->c;
    XView xv = stage_x(cc, x, dtype, d, c, ldx, where);
    if (c > 65536 || d > 65536) throw Error(kInvalid, "block_gram: block too large");
    double* G = cc.arena.alloc_n<double>((size_t)c * c);
    std::vector<GemmDesc> one{{xv.X, xv.X, G, xv.ld, xv.ld, c, (int)c, (int)c, (int)d, 1.0, 0.0}};
    leaf_gram_tall(cc, xv.dt, one);
    HSVD_CUDA(cudaMemcpyAsync(g, G, (size_t)c * c * 8, cudaMemcpyDeviceToHost, cc.stream));
    HSVD_CUDA(cudaStreamSynchronize(cc.stream));
    return HSVD_CU_OK;
  });
}

int hsvd_cu_nccl_unique_id(void* out128) {
  return guarded([&] {
    if (!out128) throw Error(kInvalid, "out is null");
    nccl_unique_id(out128);
    return HSVD_CU_OK;
  });
}

int hsvd_cu_ctx_init_nccl(hsvd_cu_ctx* ctx, int rank, int world, const void* id128) {
  return guarded([&] {
    if (!ctx || !id128 || world < 1 || rank < 0 || rank >= world)
      throw Error(kInvalid, "init_nccl: bad arguments");
    ctx->comm = make_nccl_comm(rank, world, id128, ctx->c.device);
    ctx->c.rank = rank;
    ctx->c.world = world;
    return HSVD_CU_OK;
  });
}

int hsvd_cu_thread_group_create(int world, hsvd_cu_group** out) {
  return guarded([&] {
    if (!out) throw Error(kInvalid, "out is null");
    auto* g = new hsvd_cu_group();
    g->g = make_thread_group(world);
    *out = g;
    return HSVD_CU_OK;
  });
}

void hsvd_cu_thread_group_free(hsvd_cu_group* g) { delete g; }

int hsvd_cu_ctx_join_group(hsvd_cu_ctx* ctx, hsvd_cu_group* g, int rank) {
  return guarded([&] {
    if (!ctx || !g) throw Error(kInvalid, "join_group: null argument");
    ctx->comm = make_thread_comm(g->g, rank);
    ctx->c.rank = rank;
    ctx->c.world = ctx->comm->size();
    return HSVD_CU_OK;
  });
}

int hsvd_cu_shard_rows(int64_t m_total, int64_t d, int rank, int world, int64_t* row0,
                       int64_t* m_local) {
  return guarded([&] {
    if (m_total < 1 || world < 1 || rank < 0 || rank >= world)
      throw Error(kInvalid, "shard_rows: bad arguments");
    long long r0 = 0, ml = 0;
    shard_rows(m_total, d, rank, world, &r0, &ml, nullptr, nullptr);
    if (row0) *row0 = r0;
    if (m_local) *m_local = ml;
    return HSVD_CU_OK;
  });
}

int hsvd_cu_rank_k_svd_sharded(hsvd_cu_ctx* ctx, const void* x, int dtype, int64_t m_local,
                               int64_t n, int64_t ldx, int where, int64_t m_total, int64_t row0,
                               const hsvd_cu_config* cfg, hsvd_cu_result** out) {
  return guarded([&] {
    if (!out) throw Error(kInvalid, "out is null");
    *out = nullptr;
    if (!ctx || !ctx->comm) throw Error(kInvalid, "sharded: context has no communicator");
    if (n <= 0 || m_total <= 0) throw Error(kInvalid, "hierarchical_svd: matrix is empty");
    check_cfg(cfg);
    begin(ctx);
    XView xv{x, dtype_of(dtype), ldx > 0 ? ldx : n, m_local, n};
    if (m_local > 0) xv = stage_x(ctx->c, x, dtype, m_local, n, ldx, where);
    DFac f;
    try {
      f = rank_k_svd_sharded(ctx->c, *ctx->comm, xv, m_total, row0, to_cfg(cfg));
    } catch (...) {
      ctx->comm->abort();  // release the peers blocked on this rank
      throw;
    }
    *out = make_result(ctx, f, true, true);
    return HSVD_CU_OK;
  });
}

int hsvd_cu_result_info(const hsvd_cu_result* r, int64_t* rank, int32_t* has_u, int32_t* has_v,
                        int64_t* u_rows, int64_t* v_rows, int32_t* degenerate) {
  if (int s = check_result(r)) return s;
  if (rank) *rank = r->rank;
  if (has_u) *has_u = r->u != nullptr;
  if (has_v) *has_v = r->v != nullptr;
  if (u_rows) *u_rows = r->u_rows;
  if (v_rows) *v_rows = r->v_rows;
  if (degenerate) *degenerate = r->degenerate;
  return HSVD_CU_OK;
}

int hsvd_cu_result_sigma(const hsvd_cu_result* r, double* out) {
  if (int s = check_result(r)) return s;
  return guarded([&] {
    Ctx& c = r->ctx->c;
    HSVD_CUDA(cudaSetDevice(c.device));
    HSVD_CUDA(cudaMemcpyAsync(out, r->sigma, r->rank * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    HSVD_CUDA(cudaStreamSynchronize(c.stream));
    return HSVD_CU_OK;
  });
}

int hsvd_cu_result_u(const hsvd_cu_result* r, double* out) {
  if (!r) return fail(HSVD_CU_EINVAL, "null result");
  return copy_side(r, r->u, r->ldu, r->u_rows, out);
}

int hsvd_cu_result_v(const hsvd_cu_result* r, double* out) {
  if (!r) return fail(HSVD_CU_EINVAL, "null result");
  return copy_side(r, r->v, r->ldv, r->v_rows, out);
}

int hsvd_cu_result_device(const hsvd_cu_result* r, const double** sigma, const double** u,
                          int64_t* ldu, const double** v, int64_t* ldv) {
  if (int s = check_result(r)) return s;
  if (sigma) *sigma = r->sigma;
  if (u) *u = r->u;
  if (ldu) *ldu = r->ldu;
  if (v) *v = r->v;
  if (ldv) *ldv = r->ldv;
  return HSVD_CU_OK;
}

void hsvd_cu_result_free(hsvd_cu_result* r) { delete r; }

}  // extern "C"
