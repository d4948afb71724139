// Host-side helpers shared by the C-ABI translation units (capi.cu, slab.cu):
// the error model (ApiError -> status code + per-handle message, following
// proj/src/capi.cpp:26-41), CUDA-call checking, stream arguments and the
// per-handle entry ordering (UseGuard).
#pragma once
#include <cuda_runtime.h>

#include <mutex>
#include <stdexcept>
#include <string>

#include "../../include/emfgpu.h"

namespace emfgpu {
namespace capi {

// message of the last failed call on this thread (emfgpu_global_last_error)
inline thread_local std::string g_error;

struct ApiError : std::runtime_error {
  emfgpu_status code;
  ApiError(emfgpu_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(call)                                                                                     \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess)                                                                           \
      throw ApiError(EMFGPU_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));           \
  } while (0)

template <typename Fn>
inline emfgpu_status guarded(std::string* slot, Fn&& fn) {
  try {
    fn();
    if (slot) slot->clear();
    return EMFGPU_OK;
  } catch (const ApiError& e) {
    if (slot) *slot = e.what();
    g_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    if (slot) *slot = e.what();
    g_error = e.what();
    return EMFGPU_ERR_CUDA;
  }
}

// Stream arguments are taken literally (NULL = the legacy default stream, as in
// cuBLAS); the handle's private stream is used only by the *_host entry points.
inline cudaStream_t S(void* s, cudaStream_t /*def*/) { return static_cast<cudaStream_t>(s); }

// Calls on one handle are ordered among themselves on the device, whatever
// streams and host threads they come from (the reference's apply is const and
// may be called concurrently; here the handle's work buffers --
// element-local results, ticket counters, staging vectors -- are shared, so
// concurrent calls are serialised, not overlapped): an entry takes the
// handle's lock for its enqueue, makes its stream wait for the event the
// previous entry recorded, and records the event on its stream when it
// leaves.  Inside a stream capture the caller owns the ordering (no event).
struct UseGuard {
  std::unique_lock<std::recursive_mutex> lk;
  cudaEvent_t* ev;
  cudaStream_t s;
  bool active = false;
  UseGuard(std::recursive_mutex& mu, cudaEvent_t& e, cudaStream_t st, int device) : lk(mu), ev(&e), s(st) {
    CK(cudaSetDevice(device));
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CK(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone) return;
    if (!*ev) CK(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
    CK(cudaStreamWaitEvent(s, *ev, 0));
    active = true;
  }
  ~UseGuard() {
    if (active) cudaEventRecord(*ev, s);
  }
  UseGuard(const UseGuard&) = delete;
  UseGuard& operator=(const UseGuard&) = delete;
};
#define OP_USE(op, st) UseGuard use_guard_((op)->use_mu, (op)->ev_use, (st), (op)->L->device)

// split-apply phases (capi.cu) for the slab layer (slab.cu)
void op_elements(emfgpu_op* op, const void* x, int k0, int k1, cudaStream_t s);
void op_nodes(emfgpu_op* op, const void* x, void* y, const void* ghost_lo, const void* ghost_hi, cudaStream_t s);
void op_pack_face(emfgpu_op* op, int k, int side, void* face, cudaStream_t s);
// element-local diagonal contributions into the operator's local buffer (capi.cu)
void op_diag_elements(emfgpu_op* op, cudaStream_t s);
// TransferOp kinds 0 prolongate, 1 restrict, 2 interpolate down (capi.cu)
template <typename T>
void transfer_apply_T(emfgpu_transfer* t, int kind, const T* in, T* out, cudaStream_t s);
// the single-GPU hierarchy from its level 0 (capi.cu)
void mg_linearize_any(emfgpu_mg* m, const double* d_u, cudaStream_t s);
void mg_vcycle0(emfgpu_mg* m, cudaStream_t s);  // x0 = V-cycle(b0)
void* mg_b0(emfgpu_mg* m);
void* mg_x0(emfgpu_mg* m);

}  // namespace capi
}  // namespace emfgpu
