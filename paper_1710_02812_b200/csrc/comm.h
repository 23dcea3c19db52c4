// Communicator used by the sharded (multi-GPU) pipeline.  Only rank-k
// factors, k x k Grams and column norms ever cross it.
#pragma once

#include <cstddef>
#include <memory>

#include "ctx.h"

namespace hsvdcu {

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  // Blocking from the host's point of view once the call returns the data is
  // usable on ctx.stream (device pointers).
  virtual void send(Ctx& ctx, const void* buf, size_t bytes, int peer) = 0;
  virtual void recv(Ctx& ctx, void* buf, size_t bytes, int peer) = 0;
  virtual void bcast(Ctx& ctx, void* buf, size_t bytes, int root) = 0;
  virtual void allreduce_sum(Ctx& ctx, double* buf, size_t count) = 0;
  virtual void barrier(Ctx& ctx) = 0;
  // Brackets the point-to-point calls of one tree level (ncclGroupStart/End).
  virtual void group_start() {}
  virtual void group_end() {}
  // Called by a rank that failed mid-collective: peers blocked on it return
  // an error instead of waiting forever (ncclCommAbort / group abort).
  virtual void abort() {}
};

// NCCL over NVLink/NVSwitch (libnccl.so.2 loaded at runtime).
std::unique_ptr<Comm> make_nccl_comm(int rank, int world, const void* unique_id128, int device);
// Fills a 128-byte ncclUniqueId (rank 0 calls this and shares the bytes).
void nccl_unique_id(void* out128);

// In-process group: several host threads, each with its own Ctx, exchange
// through host-synchronised device copies (used to test the sharded path
// on a single GPU; no device-side waits between ranks).
struct ThreadGroup;
std::shared_ptr<ThreadGroup> make_thread_group(int world);
std::unique_ptr<Comm> make_thread_comm(std::shared_ptr<ThreadGroup> g, int rank);

}  // namespace hsvdcu
