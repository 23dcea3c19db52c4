// Per-device execution context: stream, device arena, pinned staging ring,
// launch accounting.  Host-side only.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "common.cuh"

namespace hsvdcu {

// Stream-ordered bump allocator over cudaMalloc'd chunks.  Everything on the
// context's single stream, so memory released with release(mark) may be
// reused by later launches without a sync.
class Arena {
 public:
  struct Mark {
    size_t chunk;
    size_t off;
  };
  ~Arena() { free_all(); }
  void* alloc(size_t bytes) {
    bytes = (bytes + 255) & ~size_t(255);
    if (bytes == 0) bytes = 256;
    while (cur_ < chunks_.size()) {
      Chunk& c = chunks_[cur_];
      if (off_ + bytes <= c.size) {
        void* p = static_cast<char*>(c.ptr) + off_;
        off_ += bytes;
        peak_ = peak_ > used() ? peak_ : used();
        return p;
      }
      ++cur_;
      off_ = 0;
    }
    size_t want = chunks_.empty() ? (size_t(256) << 20) : chunks_.back().size * 2;
    if (want < bytes) want = bytes;
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, want);
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      want = bytes;
      e = cudaMalloc(&p, want);
      if (e != cudaSuccess) {
        (void)cudaGetLastError();
        throw Error(kNoMemory, "device arena: cudaMalloc of " + std::to_string(want) +
                                   " bytes failed: " + cudaGetErrorString(e));
      }
    }
    chunks_.push_back({p, want});
    cur_ = chunks_.size() - 1;
    off_ = bytes;
    peak_ = peak_ > used() ? peak_ : used();
    return p;
  }
  template <typename T>
  T* alloc_n(size_t n) { return static_cast<T*>(alloc(n * sizeof(T))); }
  Mark mark() const { return {cur_, off_}; }
  void release(Mark m) {
    cur_ = m.chunk;
    off_ = m.off;
  }
  void reset() {
    cur_ = 0;
    off_ = 0;
  }
  size_t used() const {
    size_t u = off_;
    for (size_t i = 0; i < cur_ && i < chunks_.size(); ++i) u += chunks_[i].size;
    return u;
  }
  size_t capacity() const {
    size_t u = 0;
    for (auto& c : chunks_) u += c.size;
    return u;
  }
  void swap(Arena& o) {
    chunks_.swap(o.chunks_);
    std::swap(cur_, o.cur_);
    std::swap(off_, o.off_);
    std::swap(peak_, o.peak_);
  }
  void free_all() {
    for (auto& c : chunks_) cudaFree(c.ptr);
    chunks_.clear();
    cur_ = off_ = 0;
  }

 private:
  struct Chunk {
    void* ptr;
    size_t size;
  };
  std::vector<Chunk> chunks_;
  size_t cur_ = 0, off_ = 0, peak_ = 0;
};

// Device copy of `bytes` from pinned (mapped) host memory by a one-CTA
// kernel on stream s: no copy engine involved (staging.cu).
void copy_mapped_to_device(void* dst, const void* host_src, size_t bytes, cudaStream_t s);

// Pinned host ring mirrored on the device: small descriptor arrays are
// written on the host and copied to the device by a one-CTA kernel reading
// the mapped ring (cudaMemcpyAsync when the ring cannot be mapped).  The
// kernel copy keeps these per-launch transfers off the copy engines: a
// host->device cudaMemcpyAsync per GEMM queued behind the chunked input
// transfer (the compute stream then waited for the whole input), and even
// on an idle engine it cost ~3 ms per config-2 step against the kernel.
class Staging {
 public:
  void init(size_t bytes) {
    size_ = bytes;
    HSVD_CUDA(cudaMallocHost(&host_, bytes));
    HSVD_CUDA(cudaMalloc(&dev_, bytes));
    // the device's address of the (mapped) pinned ring, for zero-copy reads
    if (cudaHostGetDevicePointer(&host_dev_, host_, 0) != cudaSuccess) {
      (void)cudaGetLastError();
      host_dev_ = nullptr;  // copy-engine path only
    }
  }
  ~Staging() {
    if (host_) cudaFreeHost(host_);
    if (dev_) cudaFree(dev_);
  }
  // Copies `bytes` from src into the ring and returns the device address.
  // The device copy is only valid until the ring wraps (one launch): arrays
  // read by several launches go through put_to() into arena memory.
  void* put(const void* src, size_t bytes, cudaStream_t s) { return put_to(nullptr, src, bytes, s); }
  // Same, with the device destination `dst` (nullptr = the ring's own copy).
  void* put_to(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    size_t b = (bytes + 255) & ~size_t(255);
    if (b > size_) throw Error(kInvalid, "staging ring too small");
    if (off_ + b > size_) {
      HSVD_CUDA(cudaStreamSynchronize(s));  // all earlier copies consumed
      for (cudaStream_t o : other_)
        if (o && o != s) HSVD_CUDA(cudaStreamSynchronize(o));
      off_ = 0;
    }
    char* h = static_cast<char*>(host_) + off_;
    char* d = dst ? static_cast<char*>(dst) : static_cast<char*>(dev_) + off_;
    std::memcpy(h, src, bytes);
    if (host_dev_)
      copy_mapped_to_device(d, static_cast<char*>(host_dev_) + off_, bytes, s);
    else
      HSVD_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
    off_ += b;
    return d;
  }

  // the two streams whose launches read the ring once a side stream exists
  // (Ctx::side_begin): a wrap waits for both
  void also_sync(cudaStream_t a, cudaStream_t b) {
    other_[0] = a;
    other_[1] = b;
  }

 private:
  cudaStream_t other_[2] = {nullptr, nullptr};
  void* host_ = nullptr;
  void* host_dev_ = nullptr;  // device address of host_
  void* dev_ = nullptr;
  size_t size_ = 0, off_ = 0;
};

// Opt a kernel in to the device's full dynamic shared memory, once per
// (device, kernel).  The attribute is process-global state shared by every
// context; setting it to each launch's own size would race between host
// threads driving different contexts (a smaller size set by one thread makes
// another thread's larger launch fail).
inline void smem_optin_impl(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  HSVD_CUDA(cudaGetDevice(&dev));
  int optin = 0;
  HSVD_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  cudaFuncAttributes fa;
  HSVD_CUDA(cudaFuncGetAttributes(&fa, func));
  const int dyn_max = optin - static_cast<int>(fa.sharedSizeBytes);
  if (bytes > (size_t)dyn_max)
    throw Error(kInvalid, "kernel needs more shared memory than a CTA may use");
  std::lock_guard<std::mutex> lk(mu);
  if (!done.insert({dev, func}).second) return;
  HSVD_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_max));
}
template <typename K>
void smem_optin(K* kernel, size_t bytes) {
  smem_optin_impl(reinterpret_cast<const void*>(kernel), bytes);
}

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  Arena arena;
  Staging staging;
  long long launches = 0;  // kernels launched by this library on this context
  int* d_flags = nullptr;  // device status word (bit0: non-finite seen)
  int num_sms = 148;
  // multi-GPU (optional)
  void* nccl_comm = nullptr;
  int rank = 0, world = 1;

  int* h_ints = nullptr;  // pinned readback buffer
  size_t h_ints_cap = 0;
  double* h_dbl = nullptr;
  size_t h_dbl_cap = 0;

  int* pinned_ints(size_t n) {
    if (n > h_ints_cap) {
      if (h_ints) cudaFreeHost(h_ints);
      h_ints_cap = n < 1024 ? 1024 : n;
      HSVD_CUDA(cudaMallocHost(&h_ints, h_ints_cap * sizeof(int)));
    }
    return h_ints;
  }
  double* pinned_dbl(size_t n) {
    if (n > h_dbl_cap) {
      if (h_dbl) cudaFreeHost(h_dbl);
      h_dbl_cap = n < 1024 ? 1024 : n;
      HSVD_CUDA(cudaMallocHost(&h_dbl, h_dbl_cap * sizeof(double)));
    }
    return h_dbl;
  }
  // two pinned chunks for large device->host result copies (copy_to_host)
  static constexpr size_t kD2hChunk = size_t(32) << 20;
  void* d2h_pin[2] = {nullptr, nullptr};
  cudaEvent_t d2h_ev[2] = {nullptr, nullptr};
  void ensure_d2h_stage() {
    for (int i = 0; i < 2; ++i) {
      if (!d2h_pin[i]) HSVD_CUDA(cudaMallocHost(&d2h_pin[i], kD2hChunk));
      if (!d2h_ev[i]) HSVD_CUDA(cudaEventCreateWithFlags(&d2h_ev[i], cudaEventDisableTiming));
    }
  }
  // pinned ring for pageable host inputs (PageableStager, capi.cu)
  static constexpr size_t kH2dChunk = size_t(64) << 20;
  static constexpr int kH2dSlots = 3;
  void* h2d_pin[kH2dSlots] = {nullptr, nullptr, nullptr};
  cudaEvent_t h2d_ev[kH2dSlots] = {nullptr, nullptr, nullptr};
  void ensure_h2d_stage() {
    for (int i = 0; i < kH2dSlots; ++i) {
      if (!h2d_pin[i]) HSVD_CUDA(cudaMallocHost(&h2d_pin[i], kH2dChunk));
      if (!h2d_ev[i]) HSVD_CUDA(cudaEventCreateWithFlags(&h2d_ev[i], cudaEventDisableTiming));
    }
  }
  // side stream for host->device input copies that overlap the compute
  // stream, and the events marking the copied row chunks
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> chunk_ev;
  cudaStream_t get_copy_stream() {
    if (!copy_stream) HSVD_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    return copy_stream;
  }
  cudaEvent_t get_chunk_event(size_t i) {
    while (chunk_ev.size() <= i) {
      cudaEvent_t e;
      HSVD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      chunk_ev.push_back(e);
    }
    return chunk_ev[i];
  }
  // Side compute stream: independent launches of one call (the back-
  // transform's T factors, the chase's WY blocks) run there while the
  // latency-bound kernels of the main stream leave SMs idle.  side_begin()
  // makes the side stream wait for everything queued on the main stream so
  // far and routes the following launches to it; side_end() routes back;
  // side_join() makes the main stream wait for the side stream.  The arena's
  // mark/release reuse is ordered by ONE stream, so the side launches take
  // their workspaces from an arena of their own (stack discipline per scope;
  // the side stream is in-order, so reuse across scopes is safe too).
  // Results the main stream reads after the join must be allocated outside.
  Arena side_arena;
  Arena::Mark side_mark{};
  cudaStream_t side_stream = nullptr, main_saved = nullptr;
  cudaEvent_t side_ev[2] = {nullptr, nullptr};
  void side_begin() {
    if (!side_stream) {
      HSVD_CUDA(cudaStreamCreateWithFlags(&side_stream, cudaStreamNonBlocking));
      for (auto& e : side_ev) HSVD_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    staging.also_sync(stream, side_stream);
    HSVD_CUDA(cudaEventRecord(side_ev[0], stream));
    HSVD_CUDA(cudaStreamWaitEvent(side_stream, side_ev[0], 0));
    main_saved = stream;
    stream = side_stream;
    arena.swap(side_arena);
    side_mark = arena.mark();
  }
  void side_end() {
    arena.release(side_mark);
    arena.swap(side_arena);
    stream = main_saved;
    main_saved = nullptr;
  }
  void side_join() {
    if (!side_stream) return;
    HSVD_CUDA(cudaEventRecord(side_ev[1], side_stream));
    HSVD_CUDA(cudaStreamWaitEvent(stream, side_ev[1], 0));
  }
  ~Ctx() {
    if (side_stream) {
      cudaStreamSynchronize(side_stream);
      cudaStreamDestroy(side_stream);
      for (auto e : side_ev) cudaEventDestroy(e);
    }
    for (auto e : chunk_ev) cudaEventDestroy(e);
    if (copy_stream) {
      cudaStreamSynchronize(copy_stream);
      cudaStreamDestroy(copy_stream);
    }
    if (h_ints) cudaFreeHost(h_ints);
    if (h_dbl) cudaFreeHost(h_dbl);
    for (int i = 0; i < kH2dSlots; ++i) {
      if (h2d_ev[i]) cudaEventDestroy(h2d_ev[i]);
      if (h2d_pin[i]) cudaFreeHost(h2d_pin[i]);
    }
    for (int i = 0; i < 2; ++i) {
      if (d2h_ev[i]) cudaEventDestroy(d2h_ev[i]);
      if (d2h_pin[i]) cudaFreeHost(d2h_pin[i]);
    }
    for (auto& r : prof) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    for (auto e : ev_free) cudaEventDestroy(e);
  }

  // --- per-launch CUDA-event profiler (off unless enabled) ---
  struct ProfRec {
    std::string name;
    cudaEvent_t a, b;
    double flops;  // algorithmic flops of the launch (GEMMs), else 0
    double bytes;  // algorithmic HBM bytes of the launch (factor streaming kernels), else 0
  };
  double pending_flops = 0.0;
  double pending_bytes = 0.0;
  bool profiling = false;
  const char* phase = "";
  const char* sub = nullptr;  // optional sub-phase inside a phase (profile key phase/sub)
  std::vector<ProfRec> prof;
  std::vector<cudaEvent_t> ev_free;
  cudaEvent_t pending = nullptr;

  cudaEvent_t get_event() {
    if (!ev_free.empty()) {
      cudaEvent_t e = ev_free.back();
      ev_free.pop_back();
      return e;
    }
    cudaEvent_t e;
    HSVD_CUDA(cudaEventCreate(&e));
    return e;
  }
  // NVTX: one range per phase ("leaf.gram", "leaf.eig", "merge.eig", ...),
  // opened lazily at the phase's first launch and closed at the next phase
  // or the next API call (header-only NVTX3: a no-op without a tool)
  const char* nvtx_open = nullptr;
  void nvtx_phase() {
    if (phase == nvtx_open) return;
    if (nvtx_open) nvtxRangePop();
    nvtxRangePushA(phase && *phase ? phase : "hsvd");
    nvtx_open = phase;
  }
  void nvtx_close() {
    if (nvtx_open) nvtxRangePop();
    nvtx_open = nullptr;
  }
  void launch_begin() {
    nvtx_phase();
    if (!profiling) return;
    pending = get_event();
    HSVD_CUDA(cudaEventRecord(pending, stream));
  }

  void count(int n = 1) { launches += n; }
  static bool trace() {
    static const bool on = std::getenv("HSVD_TRACE") != nullptr;
    return on;
  }
  void check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw Error(kCuda, std::string(what) + ": " + cudaGetErrorString(e));
    if (trace()) {
      std::fprintf(stderr, "[r%d] launch %s:%s\n", rank, phase, what);
      std::fflush(stderr);
    }
    count();
    if (profiling && pending) {
      cudaEvent_t b = get_event();
      HSVD_CUDA(cudaEventRecord(b, stream));
      prof.push_back({std::string(phase) + (sub ? std::string("/") + sub : std::string()) + ":" + what,
                      pending, b, pending_flops, pending_bytes});
      pending = nullptr;
    }
    pending_flops = 0.0;
    pending_bytes = 0.0;
  }
};

struct PhaseScope {
  Ctx& c;
  const char* prev;
  PhaseScope(Ctx& ctx, const char* p) : c(ctx), prev(ctx.phase) { c.phase = p; }
  ~PhaseScope() { c.phase = prev; }
};

// Routes the launches of a scope to the side stream (exception-safe).
struct SideScope {
  Ctx& c;
  explicit SideScope(Ctx& ctx) : c(ctx) { c.side_begin(); }
  ~SideScope() { c.side_end(); }
};

struct SubPhase {
  Ctx& c;
  const char* prev;
  SubPhase(Ctx& ctx, const char* s) : c(ctx), prev(ctx.sub) { c.sub = s; }
  ~SubPhase() { c.sub = prev; }
};

}  // namespace hsvdcu
