// z-slab multi-GPU tangent apply behind the C ABI (include/emfgpu.h,
// DESIGN.md §6).  The reference has no distributed path; this
// is the B200 design of SURVEY §8(e):
//  * rank r owns element layers [k0, k1) of the global box (its level was
//    created with z_offset = k0 and the slab's own Dirichlet faces) and node
//    planes [k0 p, k1 p]; the interface plane is duplicated on both ranks;
//  * one apply: the two boundary element layers, their interface faces packed
//    from the element-local results; the faces go to the z neighbours on the
//    slab's communication stream (NCCL send/recv between processes, or
//    peer copies over NVLink inside one process) while the interior layers
//    run on the compute stream; the node phase then sums every node's <= 8
//    contributions, own and ghost, in the reference's global colour order
//    (operator.hpp:145-153, 439), so each rank's slab of y is bitwise the
//    single-GPU result;
//  * everything is stream-ordered (events between the compute and the
//    communication stream), so a slab apply can sit inside a CUDA graph;
//  * dot products count every interface plane once (owned by the upper rank)
//    and sum the per-rank partials in rank order on the device.
// NCCL is loaded at run time (dlopen of libnccl.so.2: the copy the process
// already has, e.g. torch's, else the system one), so the library has no
// link-time NCCL dependency and single-GPU users never touch it.
#include <cstring>
#include <memory>
#include <vector>

#include "capi_util.h"
#include "internal.h"
#include "slab_transport.h"

using namespace emfgpu;
using namespace emfgpu::capi;

namespace {

// out = sum_{r < world} part[r], in rank order (bit-identical on every rank)
__global__ void rank_sum_kernel(const double* part, int world, double* out) {
  double s = 0.0;
  for (int r = 0; r < world; ++r) s += part[r];
  *out = s;
}

}  // namespace

struct emfgpu_slab {
  emfgpu_op* op = nullptr;
  emfgpu_comm* comm = nullptr;
  int rank = 0, world = 1, lo = -1, hi = -1;
  int64_t face_values = 0;
  size_t esize = 8;
  void *send_lo = nullptr, *send_hi = nullptr, *recv_lo = nullptr, *recv_hi = nullptr;
  double* dot_buf = nullptr;  // dot partial work space + world partials
  cudaStream_t cs = nullptr;  // communication stream
  cudaEvent_t ev_packed = nullptr, ev_comm = nullptr;
  std::string last_error;
};

namespace {

void slab_enqueue_boundary(emfgpu_slab* s, const void* x, cudaStream_t st) {
  const int nzl = s->op->L->nz;
  op_elements(s->op, x, 0, 1, st);
  if (nzl > 1) op_elements(s->op, x, nzl - 1, nzl, st);
  if (s->lo >= 0) op_pack_face(s->op, 0, 0, s->send_lo, st);
  if (s->hi >= 0) op_pack_face(s->op, nzl - 1, 1, s->send_hi, st);
  CK(cudaEventRecord(s->ev_packed, st));
}

void slab_enqueue_interior_and_nodes(emfgpu_slab* s, const void* x, void* y, cudaStream_t st) {
  const int nzl = s->op->L->nz;
  if (nzl > 2) op_elements(s->op, x, 1, nzl - 1, st);
  CK(cudaStreamWaitEvent(st, s->ev_comm, 0));
  op_nodes(s->op, x, y, s->lo >= 0 ? s->recv_lo : nullptr, s->hi >= 0 ? s->recv_hi : nullptr, st);
}

// dot partial over the owned node planes (the interface plane belongs to the upper rank)
void slab_dot_partial(emfgpu_slab* s, const void* a, const void* b, double* out, cudaStream_t st) {
  const emfgpu_level* L = s->op->L;
  const int64_t plane = 3 * (int64_t)L->mx * L->my;
  const int64_t first = s->lo >= 0 ? 1 : 0;
  const int64_t n = (L->mz - first) * plane;
  if (s->op->precision == 64)
    launch_dot<double>(static_cast<const double*>(a) + first * plane, static_cast<const double*>(b) + first * plane, n,
                       s->dot_buf + 1 + s->world, out, st);
  else
    launch_dot<float>(static_cast<const float*>(a) + first * plane, static_cast<const float*>(b) + first * plane, n,
                      s->dot_buf + 1 + s->world, out, st);
}

}  // namespace

// ---- communicator ------------------------------------------------------------
emfgpu_status emfgpu_comm_unique_id(unsigned char* id) {
  if (!id) return EMFGPU_ERR_INVALID;
  return guarded(nullptr, [&] {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId u;
    NCK(nccl().GetUniqueId(&u));
    std::memcpy(id, &u, sizeof(u));
  });
}

emfgpu_status emfgpu_comm_create(const unsigned char* id, int world, int rank, int device, emfgpu_comm** out) {
  if (!id || !out || world < 1 || rank < 0 || rank >= world) return EMFGPU_ERR_INVALID;
  *out = nullptr;
  return guarded(nullptr, [&] {
    CK(cudaSetDevice(device));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    auto c = std::make_unique<emfgpu_comm>();
    NCK(nccl().CommInitRank(&c->comm, world, u, rank));
    c->owned = true;
    c->device = device;
    c->world = world;
    c->rank = rank;
    *out = c.release();
  });
}

emfgpu_status emfgpu_comm_create_group(int world, const int* devices, emfgpu_comm** out) {
  if (world < 1 || !out) return EMFGPU_ERR_INVALID;
  return guarded(nullptr, [&] {
    auto g = std::make_shared<GroupState>(world);
    std::vector<std::unique_ptr<emfgpu_comm>> cs;
    for (int r = 0; r < world; ++r) {
      auto c = std::make_unique<emfgpu_comm>();
      c->world = world;
      c->rank = r;
      c->group = g;
      c->device = devices ? devices[r] : 0;
      g->dev[r] = c->device;
      CK(cudaSetDevice(c->device));
      CK(cudaEventCreateWithFlags(&g->ev_ready[r], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&g->ev_read[r], cudaEventDisableTiming));
      cs.push_back(std::move(c));
    }
    for (int r = 0; r < world; ++r) out[r] = cs[r].release();
  });
}

emfgpu_status emfgpu_comm_wrap(void* nccl_comm, int world, int rank, emfgpu_comm** out) {
  if (!nccl_comm || !out || world < 1 || rank < 0 || rank >= world) return EMFGPU_ERR_INVALID;
  auto c = new emfgpu_comm();
  c->comm = static_cast<ncclComm_t>(nccl_comm);
  c->world = world;
  c->rank = rank;
  *out = c;
  return EMFGPU_OK;
}

void emfgpu_comm_destroy(emfgpu_comm* c) {
  if (!c) return;
  if (c->owned && c->comm) {
    try {
      nccl().CommDestroy(c->comm);
    } catch (...) {
    }
  }
  delete c;
}

// ---- slab ----------------------------------------------------------------------
emfgpu_status emfgpu_slab_create(emfgpu_op* op, int rank, int world, emfgpu_comm* comm, emfgpu_slab** out) {
  if (!op || !out || world < 1 || rank < 0 || rank >= world) return EMFGPU_ERR_INVALID;
  *out = nullptr;
  auto sl = std::make_unique<emfgpu_slab>();
  emfgpu_status st = guarded(&op->last_error, [&] {
    if (comm && (comm->world != world || comm->rank != rank))
      throw ApiError(EMFGPU_ERR_CONFIG, "slab: communicator rank/world differ from the slab's");
    CK(cudaSetDevice(op->L->device));
    sl->op = op;
    sl->comm = comm;
    sl->rank = rank;
    sl->world = world;
    sl->lo = rank > 0 ? rank - 1 : -1;
    sl->hi = rank < world - 1 ? rank + 1 : -1;
    sl->esize = op->precision == 64 ? 8 : 4;
    sl->face_values = emfgpu_op_face_values(op);
    const size_t fb = sl->esize * sl->face_values;
    if (sl->lo >= 0) {
      CK(cudaMalloc(&sl->send_lo, fb));
      CK(cudaMalloc(&sl->recv_lo, fb));
    }
    if (sl->hi >= 0) {
      CK(cudaMalloc(&sl->send_hi, fb));
      CK(cudaMalloc(&sl->recv_hi, fb));
    }
    CK(cudaMalloc(&sl->dot_buf, sizeof(double) * (1 + world + dot_partial_count())));
    CK(cudaStreamCreateWithFlags(&sl->cs, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&sl->ev_packed, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&sl->ev_comm, cudaEventDisableTiming));
  });
  if (st != EMFGPU_OK) {
    emfgpu_slab_destroy(sl.release());
    return st;
  }
  *out = sl.release();
  return EMFGPU_OK;
}

void emfgpu_slab_destroy(emfgpu_slab* s) {
  if (!s) return;
  cudaFree(s->send_lo);
  cudaFree(s->send_hi);
  cudaFree(s->recv_lo);
  cudaFree(s->recv_hi);
  cudaFree(s->dot_buf);
  if (s->ev_packed) cudaEventDestroy(s->ev_packed);
  if (s->ev_comm) cudaEventDestroy(s->ev_comm);
  if (s->cs) cudaStreamDestroy(s->cs);
  delete s;
}

const char* emfgpu_slab_last_error(const emfgpu_slab* s) { return s ? s->last_error.c_str() : ""; }

emfgpu_status emfgpu_slab_apply(emfgpu_slab* s, const void* d_x, void* d_y, void* stream) {
  if (!s || !d_x || !d_y) return EMFGPU_ERR_INVALID;
  return guarded(&s->last_error, [&] {
    emfgpu_op* op = s->op;
    if (!op->linearized) throw ApiError(EMFGPU_ERR_STALE, "slab apply: update_linearization has not run");
    if ((s->lo >= 0 || s->hi >= 0) && !s->comm)
      throw ApiError(EMFGPU_ERR_CONFIG, "slab apply: no communicator (single-process groups use slab_group_apply)");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    OP_USE(op, st);
    slab_enqueue_boundary(s, d_x, st);
    // face exchange on the communication stream, overlapped with the interior layers
    CK(cudaStreamWaitEvent(s->cs, s->ev_packed, 0));
    if (s->comm)  // world 1 needs none (no neighbours)
      s->comm->exchange(s->send_lo, s->recv_lo, s->send_hi, s->recv_hi, s->esize * (size_t)s->face_values, s->cs);
    CK(cudaEventRecord(s->ev_comm, s->cs));
    slab_enqueue_interior_and_nodes(s, d_x, d_y, st);
  });
}

emfgpu_status emfgpu_slab_group_apply(emfgpu_slab* const* slabs, int n, const void* const* d_x, void* const* d_y,
                                      void* const* streams) {
  if (!slabs || n < 1 || !d_x || !d_y || !streams) return EMFGPU_ERR_INVALID;
  for (int i = 0; i < n; ++i)
    if (!slabs[i] || !d_x[i] || !d_y[i] || slabs[i]->rank != i || slabs[i]->world != n) return EMFGPU_ERR_INVALID;
  return guarded(&slabs[0]->last_error, [&] {
    std::vector<std::unique_ptr<UseGuard>> use;
    for (int i = 0; i < n; ++i) {
      emfgpu_op* op = slabs[i]->op;
      if (!op->linearized) throw ApiError(EMFGPU_ERR_STALE, "slab apply: update_linearization has not run");
      use.push_back(std::make_unique<UseGuard>(op->use_mu, op->ev_use, static_cast<cudaStream_t>(streams[i]),
                                               op->L->device));
    }
    auto st = [&](int i) { return static_cast<cudaStream_t>(streams[i]); };
    // 1) every slab's boundary layers and face packs
    for (int i = 0; i < n; ++i) {
      CK(cudaSetDevice(slabs[i]->op->L->device));
      slab_enqueue_boundary(slabs[i], d_x[i], st(i));
    }
    // 2) ghost faces: peer copies on each slab's communication stream, after
    //    its own and its neighbours' packs (all recorded in step 1)
    for (int i = 0; i < n; ++i) {
      emfgpu_slab* s = slabs[i];
      const int dev = s->op->L->device;
      CK(cudaSetDevice(dev));
      CK(cudaStreamWaitEvent(s->cs, s->ev_packed, 0));
      const size_t fb = s->esize * s->face_values;
      if (s->lo >= 0) {
        emfgpu_slab* o = slabs[i - 1];
        CK(cudaStreamWaitEvent(s->cs, o->ev_packed, 0));
        CK(cudaMemcpyPeerAsync(s->recv_lo, dev, o->send_hi, o->op->L->device, fb, s->cs));
      }
      if (s->hi >= 0) {
        emfgpu_slab* o = slabs[i + 1];
        CK(cudaStreamWaitEvent(s->cs, o->ev_packed, 0));
        CK(cudaMemcpyPeerAsync(s->recv_hi, dev, o->send_lo, o->op->L->device, fb, s->cs));
      }
      CK(cudaEventRecord(s->ev_comm, s->cs));
    }
    // 3) interior layers, then the node phase with ghosts
    for (int i = 0; i < n; ++i) {
      CK(cudaSetDevice(slabs[i]->op->L->device));
      slab_enqueue_interior_and_nodes(slabs[i], d_x[i], d_y[i], st(i));
    }
    // the neighbours read this slab's send buffers in 2): the next apply's
    // packs (on this slab's stream) must come after those copies
    for (int i = 0; i < n; ++i) {
      CK(cudaSetDevice(slabs[i]->op->L->device));
      if (i > 0) CK(cudaStreamWaitEvent(st(i), slabs[i - 1]->ev_comm, 0));
      if (i < n - 1) CK(cudaStreamWaitEvent(st(i), slabs[i + 1]->ev_comm, 0));
    }
  });
}

emfgpu_status emfgpu_slab_dot(emfgpu_slab* s, const void* a, const void* b, double* d_out, void* stream) {
  if (!s || !a || !b || !d_out) return EMFGPU_ERR_INVALID;
  return guarded(&s->last_error, [&] {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CK(cudaSetDevice(s->op->L->device));
    double* part = s->dot_buf + 1;  // world partials
    slab_dot_partial(s, a, b, part + s->rank, st);
    if (s->world > 1) {
      if (!s->comm) throw ApiError(EMFGPU_ERR_CONFIG, "slab dot: no communicator (use slab_group_dot)");
      std::vector<long long> off(s->world), len(s->world, 1);
      for (int q = 0; q < s->world; ++q) off[q] = q;
      s->comm->allgather_ranges(part, sizeof(double), off, len, st);
    }
    rank_sum_kernel<<<1, 1, 0, st>>>(part, s->world, d_out);
    CK(cudaGetLastError());
  });
}

emfgpu_status emfgpu_slab_group_dot(emfgpu_slab* const* slabs, int n, const void* const* a, const void* const* b,
                                    double* const* d_out, void* const* streams) {
  if (!slabs || n < 1 || !a || !b || !d_out || !streams) return EMFGPU_ERR_INVALID;
  return guarded(&slabs[0]->last_error, [&] {
    auto st = [&](int i) { return static_cast<cudaStream_t>(streams[i]); };
    for (int i = 0; i < n; ++i) {
      CK(cudaSetDevice(slabs[i]->op->L->device));
      slab_dot_partial(slabs[i], a[i], b[i], slabs[i]->dot_buf + 1 + i, st(i));
      CK(cudaEventRecord(slabs[i]->ev_packed, st(i)));
    }
    // every slab gathers the others' partials (peer copies), then sums in rank order
    for (int i = 0; i < n; ++i) {
      const int dev = slabs[i]->op->L->device;
      CK(cudaSetDevice(dev));
      for (int j = 0; j < n; ++j) {
        if (j == i) continue;
        CK(cudaStreamWaitEvent(st(i), slabs[j]->ev_packed, 0));
        CK(cudaMemcpyPeerAsync(slabs[i]->dot_buf + 1 + j, dev, slabs[j]->dot_buf + 1 + j, slabs[j]->op->L->device,
                               sizeof(double), st(i)));
      }
      rank_sum_kernel<<<1, 1, 0, st(i)>>>(slabs[i]->dot_buf + 1, n, d_out[i]);
      CK(cudaGetLastError());
      CK(cudaEventRecord(slabs[i]->ev_comm, st(i)));
    }
    // the next partial written into a slab's buffer comes after the others read it
    for (int i = 0; i < n; ++i) {
      CK(cudaSetDevice(slabs[i]->op->L->device));
      for (int j = 0; j < n; ++j)
        if (j != i) CK(cudaStreamWaitEvent(st(i), slabs[j]->ev_comm, 0));
    }
  });
}
