// Transport of the z-slab layer (slab.cu, slab_solver.cu): the two
// collectives a partitioned apply / hierarchy / PCG needs, behind one
// communicator handle (emfgpu_comm):
//   exchange()         ghost data with the z neighbours (each rank sends
//                      one buffer down and one up, receives the mirror);
//   allgather_ranges() every rank's owned index range of a global buffer
//                      copied into every other rank's copy of it (no
//                      arithmetic, so the result is bitwise the same as if
//                      one GPU had produced the whole buffer).
// Two implementations:
//   * NCCL (one process per GPU): send/recv in one group, and one in-place
//     broadcast per rank; NCCL is loaded at run time (dlopen libnccl.so.2,
//     preferring the copy already in the process).
//   * thread group (one process, one host thread per rank, any devices):
//     pointers and CUDA events published through a shared rendezvous, host
//     barriers, peer copies.  The ranks' kernels never wait on one another
//     (only stream-event waits on work already enqueued), which is what lets
//     several ranks share one GPU in the tests.
// All calls are SPMD: every rank makes the same sequence of calls.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "capi_util.h"

namespace emfgpu {
namespace capi {

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

inline const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.h = h;
    auto sym = [h](const char* n) { return dlsym(h, n); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.Broadcast = reinterpret_cast<decltype(api.Broadcast)>(sym("ncclBroadcast"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!api.h || !api.Send || !api.Recv || !api.GroupStart || !api.GroupEnd || !api.Broadcast)
    throw ApiError(EMFGPU_ERR_CONFIG, "slab: libnccl.so.2 could not be loaded");
  return api;
}

#define NCK(call)                                                                                 \
  do {                                                                                            \
    ncclResult_t r_ = (call);                                                                     \
    if (r_ != ncclSuccess)                                                                        \
      throw ApiError(EMFGPU_ERR_CUDA, std::string(#call) + ": " + nccl().GetErrorString(r_));     \
  } while (0)

// Rendezvous of a thread group: a reusable barrier plus per-rank published
// pointers and events.
struct GroupState {
  explicit GroupState(int w) : world(w), p0(w), p1(w), dev(w, 0), ev_ready(w, nullptr), ev_read(w, nullptr) {}
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  std::vector<const void*> p0, p1;
  std::vector<int> dev;
  std::vector<cudaEvent_t> ev_ready, ev_read;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const unsigned long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

}  // namespace capi
}  // namespace emfgpu

struct emfgpu_comm {
  ncclComm_t comm = nullptr;  // NCCL transport
  bool owned = false;
  int world = 1, rank = 0;
  std::shared_ptr<emfgpu::capi::GroupState> group;  // thread-group transport
  int device = 0;

  ~emfgpu_comm() {
    if (group) {
      if (group->ev_ready[rank]) cudaEventDestroy(group->ev_ready[rank]);
      if (group->ev_read[rank]) cudaEventDestroy(group->ev_read[rank]);
    }
  }

  // ghost data with the z neighbours: send_lo goes to rank-1 (which receives
  // it in its recv_hi), send_hi to rank+1; absent neighbours are skipped
  void exchange(const void* send_lo, void* recv_lo, const void* send_hi, void* recv_hi, size_t bytes,
                cudaStream_t s) {
    using namespace emfgpu::capi;
    const bool lo = rank > 0, hi = rank < world - 1;
    if (world == 1 || bytes == 0) return;
    if (!group) {
      const NcclApi& N = nccl();
      NCK(N.GroupStart());
      if (lo) {
        NCK(N.Send(send_lo, bytes, ncclInt8, rank - 1, comm, s));
        NCK(N.Recv(recv_lo, bytes, ncclInt8, rank - 1, comm, s));
      }
      if (hi) {
        NCK(N.Send(send_hi, bytes, ncclInt8, rank + 1, comm, s));
        NCK(N.Recv(recv_hi, bytes, ncclInt8, rank + 1, comm, s));
      }
      NCK(N.GroupEnd());
      return;
    }
    GroupState& g = *group;
    g.p0[rank] = send_lo;
    g.p1[rank] = send_hi;
    CK(cudaEventRecord(g.ev_ready[rank], s));
    g.barrier();
    if (lo) {
      CK(cudaStreamWaitEvent(s, g.ev_ready[rank - 1], 0));
      CK(cudaMemcpyPeerAsync(recv_lo, device, g.p1[rank - 1], g.dev[rank - 1], bytes, s));
    }
    if (hi) {
      CK(cudaStreamWaitEvent(s, g.ev_ready[rank + 1], 0));
      CK(cudaMemcpyPeerAsync(recv_hi, device, g.p0[rank + 1], g.dev[rank + 1], bytes, s));
    }
    CK(cudaEventRecord(g.ev_read[rank], s));
    g.barrier();
    // the neighbours copied out of this rank's send buffers: later writes
    // to them (on this stream) come after those copies
    if (lo) CK(cudaStreamWaitEvent(s, g.ev_read[rank - 1], 0));
    if (hi) CK(cudaStreamWaitEvent(s, g.ev_read[rank + 1], 0));
  }

  // buf (elem bytes per element) is a global buffer; rank q owns elements
  // [off[q], off[q] + len[q]) of it; afterwards every rank's buf holds every
  // rank's owned range
  void allgather_ranges(void* buf, size_t elem, const std::vector<long long>& off, const std::vector<long long>& len,
                        cudaStream_t s) {
    using namespace emfgpu::capi;
    if (world == 1) return;
    char* b = static_cast<char*>(buf);
    if (!group) {
      const NcclApi& N = nccl();
      NCK(N.GroupStart());
      for (int q = 0; q < world; ++q)
        if (len[q] > 0)
          NCK(N.Broadcast(b + off[q] * elem, b + off[q] * elem, (size_t)len[q] * elem, ncclInt8, q, comm, s));
      NCK(N.GroupEnd());
      return;
    }
    GroupState& g = *group;
    g.p0[rank] = buf;
    CK(cudaEventRecord(g.ev_ready[rank], s));
    g.barrier();
    for (int q = 0; q < world; ++q) {
      if (q == rank || len[q] <= 0) continue;
      CK(cudaStreamWaitEvent(s, g.ev_ready[q], 0));
      CK(cudaMemcpyPeerAsync(b + off[q] * elem, device, static_cast<const char*>(g.p0[q]) + off[q] * elem, g.dev[q],
                             (size_t)len[q] * elem, s));
    }
    CK(cudaEventRecord(g.ev_read[rank], s));
    g.barrier();
    for (int q = 0; q < world; ++q)
      if (q != rank) CK(cudaStreamWaitEvent(s, g.ev_read[q], 0));
  }
};
