// NCCL (dlopen'd) and in-process thread-group communicators.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "comm.h"

namespace hsvdcu {

// ---------------------------------------------------------------------------
// NCCL
// ---------------------------------------------------------------------------
namespace {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // 1. HSVD_NCCL_LIB; 2. an NCCL the process already has (torch's); 3. the
    // default search.  Whatever is loaded first owns the soname libnccl.so.2
    // for the process, so the Python layer points HSVD_NCCL_LIB at the NCCL
    // torch is built against (an older system NCCL would break torch's import).
    if (const char* env = std::getenv("HSVD_NCCL_LIB")) api.h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
    if (!api.h) api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      if (api.h) break;
      api.h = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
    }
    if (!api.h) return;
#define LOAD(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(api.h, "nccl" #f))
    LOAD(GetUniqueId);
    LOAD(CommInitRank);
    LOAD(CommDestroy);
    LOAD(CommAbort);
    LOAD(Send);
    LOAD(Recv);
    LOAD(Broadcast);
    LOAD(AllReduce);
    LOAD(GroupStart);
    LOAD(GroupEnd);
    LOAD(GetErrorString);
#undef LOAD
  });
  if (!api.h || !api.CommInitRank)
    throw Error(kNccl, "libnccl.so.2 could not be loaded (set HSVD_NCCL_LIB)");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(kNccl, std::string(what) + ": " + nccl().GetErrorString(r));
}

class NcclComm : public Comm {
 public:
  NcclComm(int rank, int world, const void* id, int device) : rank_(rank), world_(world) {
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    HSVD_CUDA(cudaSetDevice(device));
    nccl_check(nccl().CommInitRank(&comm_, world, uid, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) nccl().CommDestroy(comm_);
  }
  void abort() override {
    if (comm_ && nccl().CommAbort) {
      nccl().CommAbort(comm_);
      comm_ = nullptr;
    }
  }
  int rank() const override { return rank_; }
  int size() const override { return world_; }
  void send(Ctx& c, const void* buf, size_t bytes, int peer) override {
    nccl_check(nccl().Send(buf, bytes, ncclUint8, peer, comm_, c.stream), "ncclSend");
  }
  void recv(Ctx& c, void* buf, size_t bytes, int peer) override {
    nccl_check(nccl().Recv(buf, bytes, ncclUint8, peer, comm_, c.stream), "ncclRecv");
  }
  void bcast(Ctx& c, void* buf, size_t bytes, int root) override {
    nccl_check(nccl().Broadcast(buf, buf, bytes, ncclUint8, root, comm_, c.stream), "ncclBroadcast");
  }
  void allreduce_sum(Ctx& c, double* buf, size_t count) override {
    nccl_check(nccl().AllReduce(buf, buf, count, ncclFloat64, ncclSum, comm_, c.stream),
               "ncclAllReduce");
  }
  void barrier(Ctx& c) override {
    double* d = c.arena.alloc_n<double>(1);
    HSVD_CUDA(cudaMemsetAsync(d, 0, sizeof(double), c.stream));
    allreduce_sum(c, d, 1);
    HSVD_CUDA(cudaStreamSynchronize(c.stream));
  }
  void group_start() override { nccl_check(nccl().GroupStart(), "ncclGroupStart"); }
  void group_end() override { nccl_check(nccl().GroupEnd(), "ncclGroupEnd"); }

 private:
  int rank_, world_;
  ncclComm_t comm_ = nullptr;
};

}  // namespace

void nccl_unique_id(void* out128) {
  ncclUniqueId uid;
  nccl_check(nccl().GetUniqueId(&uid), "ncclGetUniqueId");
  std::memcpy(out128, &uid, sizeof(uid));
}

std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const void* id, int device) {
  return std::unique_ptr<Comm>(new NcclComm(rank, world, id, device));
}

// ---------------------------------------------------------------------------
// in-process thread group
// ---------------------------------------------------------------------------
struct ThreadGroup {
  explicit ThreadGroup(int w) : world(w), slots(w * w), coll(w, nullptr), hostbuf(w) {}
  struct Slot {
    const void* ptr = nullptr;
    size_t bytes = 0;
    bool posted = false, consumed = false;
  };
  int world;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<Slot> slots;  // [src * world + dst]
  std::vector<const void*> coll;
  std::vector<std::vector<double>> hostbuf;
  int bar_count = 0;
  long long bar_gen = 0;
  bool aborted = false;  // a rank failed: every wait returns with an error

  void check_abort() const {
    if (aborted) throw Error(kNccl, "thread group: a peer rank failed");
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    check_abort();
    const long long gen = bar_gen;
    if (++bar_count == world) {
      bar_count = 0;
      ++bar_gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return bar_gen != gen || aborted; });
      check_abort();
    }
  }
  void abort() {
    {
      std::lock_guard<std::mutex> lk(mu);
      aborted = true;
    }
    cv.notify_all();
  }
};

namespace {

bool trace_on() {
  static const bool on = std::getenv("HSVD_TRACE") != nullptr;
  return on;
}
#define TRACE(...)                                  \
  do {                                              \
    if (trace_on()) {                               \
      std::fprintf(stderr, __VA_ARGS__);            \
      std::fflush(stderr);                          \
    }                                               \
  } while (0)

class ThreadComm : public Comm {
 public:
  ThreadComm(std::shared_ptr<ThreadGroup> g, int rank) : g_(std::move(g)), rank_(rank) {}
  int rank() const override { return rank_; }
  int size() const override { return g_->world; }
  void send(Ctx& c, const void* buf, size_t bytes, int peer) override {
    TRACE("[r%d] send %zu -> %d: sync\n", rank_, bytes, peer);
    HSVD_CUDA(cudaStreamSynchronize(c.stream));
    std::unique_lock<std::mutex> lk(g_->mu);
    auto& s = g_->slots[rank_ * g_->world + peer];
    g_->cv.wait(lk, [&] { return !s.posted || g_->aborted; });
    g_->check_abort();
    s.ptr = buf;
    s.bytes = bytes;
    s.posted = true;
    s.consumed = false;
    g_->cv.notify_all();
    g_->cv.wait(lk, [&] { return s.consumed || g_->aborted; });
    s.posted = false;
    g_->check_abort();
    g_->cv.notify_all();
    TRACE("[r%d] send -> %d done\n", rank_, peer);
  }
  void recv(Ctx& c, void* buf, size_t bytes, int peer) override {
    TRACE("[r%d] recv %zu <- %d: sync\n", rank_, bytes, peer);
    HSVD_CUDA(cudaStreamSynchronize(c.stream));
    const void* src = nullptr;
    {
      std::unique_lock<std::mutex> lk(g_->mu);
      auto& s = g_->slots[peer * g_->world + rank_];
      g_->cv.wait(lk, [&] { return (s.posted && !s.consumed) || g_->aborted; });
      g_->check_abort();
      if (s.bytes != bytes) throw Error(kNccl, "thread comm: size mismatch");
      src = s.ptr;
    }
    // copy outside the lock (the sender is parked until `consumed`)
    HSVD_CUDA(cudaMemcpyAsync(buf, src, bytes, cudaMemcpyDeviceToDevice, c.stream));
    HSVD_CUDA(cudaStreamSynchronize(c.stream));
    {
      std::lock_guard<std::mutex> lk(g_->mu);
      g_->slots[peer * g_->world + rank_].consumed = true;
    }
    g_->cv.notify_all();
    TRACE("[r%d] recv <- %d done\n", rank_, peer);
  }
  void bcast(Ctx& c, void* buf, size_t bytes, int root) override {
    TRACE("[r%d] bcast root %d\n", rank_, root);
    HSVD_CUDA(cudaStreamSynchronize(c.stream));
    if (rank_ == root) {
      std::lock_guard<std::mutex> lk(g_->mu);
      g_->coll[root] = buf;
    }
    g_->barrier();
    if (rank_ != root) {
      HSVD_CUDA(cudaMemcpyAsync(buf, g_->coll[root], bytes, cudaMemcpyDeviceToDevice, c.stream));
      HSVD_CUDA(cudaStreamSynchronize(c.stream));
    }
    g_->barrier();
    TRACE("[r%d] bcast done\n", rank_);
  }
  void allreduce_sum(Ctx& c, double* buf, size_t count) override {
    TRACE("[r%d] allreduce %zu\n", rank_, count);
    HSVD_CUDA(cudaStreamSynchronize(c.stream));
    auto& mine = g_->hostbuf[rank_];
    mine.resize(count);
    HSVD_CUDA(cudaMemcpyAsync(mine.data(), buf, count * sizeof(double), cudaMemcpyDeviceToHost,
                              c.stream));
    HSVD_CUDA(cudaStreamSynchronize(c.stream));
    g_->barrier();
    std::vector<double> sum(count, 0.0);
    for (int r = 0; r < g_->world; ++r)  // fixed rank order: deterministic
      for (size_t i = 0; i < count; ++i) sum[i] += g_->hostbuf[r][i];
    g_->barrier();
    HSVD_CUDA(cudaMemcpyAsync(buf, sum.data(), count * sizeof(double), cudaMemcpyHostToDevice,
                              c.stream));
    HSVD_CUDA(cudaStreamSynchronize(c.stream));
    TRACE("[r%d] allreduce done\n", rank_);
  }
  void barrier(Ctx& c) override {
    HSVD_CUDA(cudaStreamSynchronize(c.stream));
    g_->barrier();
  }
  void abort() override { g_->abort(); }

 private:
  std::shared_ptr<ThreadGroup> g_;
  int rank_;
};

}  // namespace

std::shared_ptr<ThreadGroup> make_thread_group(int world) {
  if (world < 1) throw Error(kInvalid, "thread group: world must be >= 1");
  return std::make_shared<ThreadGroup>(world);
}

std::unique_ptr<Comm> make_thread_comm(std::shared_ptr<ThreadGroup> g, int rank) {
  if (!g || rank < 0 || rank >= g->world) throw Error(kInvalid, "thread comm: bad rank");
  return std::unique_ptr<Comm>(new ThreadComm(std::move(g), rank));
}

}  // namespace hsvdcu
