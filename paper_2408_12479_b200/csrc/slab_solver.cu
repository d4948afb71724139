// The cfg4 solve partitioned in z slabs (SURVEY §8(e) ¶3): fp64 PCG
// preconditioned by the fp32 hp-multigrid V-cycle, one rank per GPU, every
// rank's iterates bitwise the single-GPU solve's on its node planes.
//
// Partition (the reference has no distributed path):
//   * the fine level (the outer operator and the multigrid's finest level)
//     keeps the slab partition: rank r owns element layers [k0, k1) and node
//     planes [k0 p, k1 p], the interface plane duplicated and consistent;
//     applies exchange the packed interface faces of the element-local
//     results (as emfgpu_slab_apply), the diagonal the same way;
//   * the next level down (p/2 on the same mesh) and everything below it are
//     small (cfg4: 2.7M DoFs of 21.6M) and agglomerated: every rank holds the
//     whole coarse level and runs the coarse part of the V-cycle redundantly
//     (the single-GPU hierarchy itself, built on that level);
//   * restriction to that level needs the fine planes of one element layer
//     beyond each interface: they are exchanged, the transfer runs on the
//     slab extended by those ghost layers, and every rank's own coarse planes
//     are all-gathered into the replicated coarse vector;
//   * prolongation reads the replicated coarse vector, interpolation of u_k
//     goes like restriction;
//   * dots sum whole node planes (the single-GPU PCG and Lanczos use the same
//     plane-chunked dot): each rank computes the partials of the planes it
//     owns (an interface plane belongs to the lower rank), the partials are
//     all-gathered and summed in plane order on every rank;
//   * the Lanczos start vector is element (global index) of the reference's
//     seeded stream.
// Every operation therefore produces, on each rank, bitwise the values the
// single-GPU solve produces on that rank's planes.  The PCG runs the same
// kernels as emfgpu_pcg_solve's host-driven loop (no graph: the thread-group
// transport synchronises host threads between the phases).
#include <algorithm>
#include <memory>
#include <vector>

#include "capi_util.h"
#include "internal.h"
#include "krylov_core.h"
#include "slab_transport.h"

using namespace emfgpu;
using namespace emfgpu::capi;

struct emfgpu_slab_solver {
  emfgpu_comm* comm = nullptr;
  int rank = 0, world = 1;
  const emfgpu_level* Lf = nullptr;  // the rank's fine slab level
  emfgpu_level_desc gdesc{};         // the global fine level
  int nzg = 0, k0 = 0, k1 = 0, lo = 0, hi = 0, pf = 0, pc = 0;
  int64_t plane_f = 0, plane_c = 0;  // DoFs per node plane
  int nplanes_g = 0;                 // global fine node planes
  emfgpu_mg_config cfg{};
  emfgpu_op* op64 = nullptr;  // outer operator
  emfgpu_op* opm = nullptr;   // finest multigrid level (cfg.precision)
  emfgpu_level* Lc = nullptr;  // replicated coarse level
  emfgpu_mg* mgc = nullptr;    // the hierarchy below, replicated
  emfgpu_level fext{}, cext{};  // dimension-only shadows of the extended slab
  emfgpu_transfer* tr = nullptr;
  // device buffers
  void *face_lo = nullptr, *face_hi = nullptr, *ghost_lo = nullptr, *ghost_hi = nullptr;
  size_t face_bytes = 0;
  void* fine_ext = nullptr;   // extended fine vector (max precision)
  void* coarse_ext = nullptr;
  void *x0 = nullptr, *b0 = nullptr, *t0 = nullptr, *dg = nullptr, *inv = nullptr, *cr = nullptr, *cd = nullptr,
       *cad = nullptr;
  double* uf = nullptr;  // u_k on the slab
  double* uc = nullptr;  // u_k on the replicated coarse level
  double* part = nullptr;  // dot partials (global plane slots) + result
  double* lz = nullptr;
  size_t lz_bytes = 0;
  double* pcg = nullptr;
  size_t pcg_bytes = 0;
  unsigned long long* nbad = nullptr;
  double lmax = 0, lmin = 0;
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_packed = nullptr, ev_comm = nullptr;
  bool linearized = false;
  std::string last_error;
};

namespace {

// element layers [k0, k1) of rank q (SlabPartition, slab.py)
void slab_range(int nzg, int world, int q, int& k0, int& k1) {
  const int base = nzg / world, rem = nzg % world;
  k0 = q * base + std::min(q, rem);
  k1 = k0 + base + (q < rem ? 1 : 0);
}

size_t esize(const emfgpu_slab_solver* S) { return S->cfg.precision == 64 ? 8 : 4; }

// y = K x on the slab (boundary layers, face exchange on the communication
// stream overlapped with the interior layers, node phase with the ghosts)
template <typename T>
void slab_apply(emfgpu_slab_solver* S, emfgpu_op* op, const T* x, T* y, cudaStream_t st) {
  const int nzl = op->L->nz;
  op_elements(op, x, 0, 1, st);
  if (nzl > 1) op_elements(op, x, nzl - 1, nzl, st);
  if (S->lo) op_pack_face(op, 0, 0, S->face_lo, st);
  if (S->hi) op_pack_face(op, nzl - 1, 1, S->face_hi, st);
  CK(cudaEventRecord(S->ev_packed, st));
  CK(cudaStreamWaitEvent(S->cs, S->ev_packed, 0));
  if (S->comm)
    S->comm->exchange(S->face_lo, S->ghost_lo, S->face_hi, S->ghost_hi,
                      sizeof(T) * (size_t)emfgpu_op_face_values(op), S->cs);
  CK(cudaEventRecord(S->ev_comm, S->cs));
  if (nzl > 2) op_elements(op, x, 1, nzl - 1, st);
  CK(cudaStreamWaitEvent(st, S->ev_comm, 0));
  op_nodes(op, x, y, S->lo ? S->ghost_lo : nullptr, S->hi ? S->ghost_hi : nullptr, st);
}

// compute_diagonal on the slab: element-local diagonal, faces exchanged, node
// gather with the ghosts, constrained rows 1
template <typename T>
void slab_diagonal(emfgpu_slab_solver* S, emfgpu_op* op, T* d, cudaStream_t st) {
  const emfgpu_level* L = op->L;
  op_diag_elements(op, st);
  if (S->lo) op_pack_face(op, 0, 0, S->face_lo, st);
  if (S->hi) op_pack_face(op, L->nz - 1, 1, S->face_hi, st);
  if (S->comm)
    S->comm->exchange(S->face_lo, S->ghost_lo, S->face_hi, S->ghost_hi,
                      sizeof(T) * (size_t)emfgpu_op_face_values(op), st);
  op_nodes(op, d, d, S->lo ? S->ghost_lo : nullptr, S->hi ? S->ghost_hi : nullptr, st);
  launch_diag_finish<T>(d, L->nnodes, L->mx, L->my, L->mz, L->faces, S->nbad, nullptr, 0, st);
  CK(cudaGetLastError());
}

// global dot of two slab vectors over whole node planes: bitwise the
// single-GPU launch_dot_planes of the global vectors
template <typename T>
void slab_dot(emfgpu_slab_solver* S, const T* a, const T* b, double* part, double* out, cudaStream_t st) {
  const int split = dot_plane_split();
  std::vector<long long> off(S->world), len(S->world);
  for (int q = 0; q < S->world; ++q) {
    int a0, a1;
    slab_range(S->nzg, S->world, q, a0, a1);
    const int first = a0 * S->pf, last = q < S->world - 1 ? a1 * S->pf - 1 : a1 * S->pf;  // owned global planes
    off[q] = (long long)first * split;
    len[q] = (long long)(last - first + 1) * split;
  }
  const int own = (int)(len[S->rank] / split);
  launch_dot_plane_partials<T>(a, b, S->plane_f, own, S->k0 * S->pf, part, st);
  if (S->comm) S->comm->allgather_ranges(part, sizeof(double), off, len, st);
  launch_sum_ordered(part, (int64_t)S->nplanes_g * split, out, st);
}

// Chebyshev-Jacobi smoother on the slab (cheb_run, capi.cu; solver.hpp:330-362)
template <typename T>
void slab_cheb(emfgpu_slab_solver* S, T* x, const T* b, int zero_start, cudaStream_t st) {
  const int64_t n = S->Lf->ndofs;
  const double lam_max = S->cfg.safety * S->lmax, lam_min = lam_max / S->cfg.range_factor;
  const double theta = 0.5 * (lam_max + lam_min), delta = 0.5 * (lam_max - lam_min);
  const double sigma1 = theta / delta;
  double rho_old = 1.0 / sigma1;
  T* r = static_cast<T*>(S->cr);
  T* d = static_cast<T*>(S->cd);
  T* ad = static_cast<T*>(S->cad);
  const T* inv = static_cast<const T*>(S->inv);
  if (!zero_start) slab_apply<T>(S, S->opm, x, r, st);
  launch_cheb_first<T>(x, r, d, b, inv, 1.0 / theta, zero_start, n, st);
  for (int k = 1; k < S->cfg.degree; ++k) {
    slab_apply<T>(S, S->opm, d, ad, st);
    const double rho_new = 1.0 / (2.0 * sigma1 - rho_old);
    launch_cheb_step<T>(x, r, d, ad, inv, rho_new * rho_old, 2.0 * rho_new / delta, n, st);
    rho_old = rho_new;
  }
}

// fine slab vector -> coarse: restriction (kind 1) or interpolation of u_k
// (kind 2) on the slab extended by one ghost element layer per interface;
// the rank's own coarse planes are written into the replicated coarse vector
// `cg`, then all-gathered
template <typename T>
void slab_to_coarse(emfgpu_slab_solver* S, int kind, const T* f, T* cg, cudaStream_t st) {
  const emfgpu_level* L = S->Lf;
  const int64_t pf_n = S->plane_f, pc_n = S->plane_c;
  T* ext = static_cast<T*>(S->fine_ext);
  const int64_t own_off = (int64_t)(S->lo ? S->pf : 0) * pf_n;
  CK(cudaMemcpyAsync(ext + own_off, f, sizeof(T) * L->ndofs, cudaMemcpyDeviceToDevice, st));
  // ghost planes: the pf fine planes beyond each interface (from the neighbours)
  const size_t gbytes = sizeof(T) * (size_t)S->pf * pf_n;
  T* recv_lo = ext;
  T* recv_hi = ext + own_off + (int64_t)L->mz * pf_n;
  const T* send_lo = f + pf_n;                               // local planes 1..pf
  const T* send_hi = f + (int64_t)(L->mz - 1 - S->pf) * pf_n;  // local planes mz-1-pf .. mz-2
  if (S->comm) S->comm->exchange(send_lo, recv_lo, send_hi, recv_hi, gbytes, st);
  T* cext = static_cast<T*>(S->coarse_ext);
  transfer_apply_T<T>(S->tr, kind, ext, cext, st);
  // own coarse planes [k0 pc, k1 pc] sit at extended plane lo*pc
  CK(cudaMemcpyAsync(cg + (int64_t)S->k0 * S->pc * pc_n, cext + (int64_t)(S->lo ? S->pc : 0) * pc_n,
                     sizeof(T) * (size_t)((S->k1 - S->k0) * S->pc + 1) * pc_n, cudaMemcpyDeviceToDevice, st));
  std::vector<long long> off(S->world), len(S->world);
  for (int q = 0; q < S->world; ++q) {
    int a0, a1;
    slab_range(S->nzg, S->world, q, a0, a1);
    const int first = a0 * S->pc + (q > 0 ? 1 : 0), last = a1 * S->pc;
    off[q] = (long long)first * pc_n;
    len[q] = (long long)(last - first + 1) * pc_n;
  }
  if (S->comm) S->comm->allgather_ranges(cg, sizeof(T), off, len, st);
}

// replicated coarse vector -> fine slab (prolongation), result in the own
// planes of the extended fine buffer; returns their address
template <typename T>
T* coarse_to_slab(emfgpu_slab_solver* S, const T* cg, cudaStream_t st) {
  const T* slice = cg + (int64_t)(S->k0 - (S->lo ? 1 : 0)) * S->pc * S->plane_c;
  T* ext = static_cast<T*>(S->fine_ext);
  transfer_apply_T<T>(S->tr, 0, slice, ext, st);
  return ext + (int64_t)(S->lo ? S->pf : 0) * S->plane_f;
}

// the V-cycle (v_cycle, capi.cu; solver.hpp:544-569) with its finest level on the slab
template <typename T>
void slab_vcycle(emfgpu_slab_solver* S, cudaStream_t st) {
  const emfgpu_level* L = S->Lf;
  const int64_t n = L->ndofs;
  T* x = static_cast<T*>(S->x0);
  T* b = static_cast<T*>(S->b0);
  T* t = static_cast<T*>(S->t0);
  CK(cudaMemsetAsync(x, 0, sizeof(T) * n, st));
  slab_cheb<T>(S, x, b, 1, st);
  slab_apply<T>(S, S->opm, x, t, st);
  launch_bminus<T>(b, t, n, st);
  launch_mask_zero<T>(t, L->nnodes, L->mx, L->my, L->mz, L->faces, st);
  T* bc = static_cast<T*>(mg_b0(S->mgc));
  slab_to_coarse<T>(S, 1, t, bc, st);
  launch_mask_zero<T>(bc, S->Lc->nnodes, S->Lc->mx, S->Lc->my, S->Lc->mz, S->Lc->faces, st);
  mg_vcycle0(S->mgc, st);
  T* tp = coarse_to_slab<T>(S, static_cast<const T*>(mg_x0(S->mgc)), st);
  launch_mask_zero<T>(tp, L->nnodes, L->mx, L->my, L->mz, L->faces, st);
  launch_add<T>(tp, x, n, st);
  slab_cheb<T>(S, x, b, 0, st);
}

template <typename T>
void slab_precondition(emfgpu_slab_solver* S, const double* r, double* z, cudaStream_t st) {
  const emfgpu_level* L = S->Lf;
  T* b = static_cast<T*>(S->b0);
  launch_cast<double, T>(r, b, L->ndofs, st);
  launch_mask_zero<T>(b, L->nnodes, L->mx, L->my, L->mz, L->faces, st);
  slab_vcycle<T>(S, st);
  launch_cast<T, double>(static_cast<const T*>(S->x0), z, L->ndofs, st);
}

// MgHierarchy::update_linearization (mg_linearize, capi.cu) with the finest
// level on the slab and the rest replicated
template <typename T>
void slab_linearize(emfgpu_slab_solver* S, const double* d_u, cudaStream_t st) {
  const emfgpu_level* L = S->Lf;
  CK(cudaMemcpyAsync(S->uf, d_u, sizeof(double) * L->ndofs, cudaMemcpyDeviceToDevice, st));
  int64_t be = -1;
  int bq = -1;
  for (emfgpu_op* op : {S->op64, S->opm}) {
    const emfgpu_status s1 = emfgpu_op_update_linearization(op, S->uf, &be, &bq, st);
    if (s1 != EMFGPU_OK) throw ApiError(s1, emfgpu_op_last_error(op));
  }
  T* d = static_cast<T*>(S->dg);
  CK(cudaMemsetAsync(S->nbad, 0, sizeof(unsigned long long), st));
  slab_diagonal<T>(S, S->opm, d, st);
  // Lanczos on the slab: the generic core with the slab apply and the plane dot
  const size_t need = lanczos_work_bytes<T>(L->ndofs, S->cfg.eig_iterations, S->nplanes_g);
  if (S->lz_bytes < need) {
    cudaFree(S->lz);
    S->lz = nullptr;
    S->lz_bytes = 0;
    CK(cudaMalloc(&S->lz, need));
    S->lz_bytes = need;
  }
  auto apply = [&](const T* x, T* y) { slab_apply<T>(S, S->opm, x, y, st); };
  auto dot = [&](const double* a, const double* b, double* part, double* out) {
    slab_dot<double>(S, a, b, part, out, st);
  };
  lanczos_core<T>(L->ndofs, (int64_t)S->k0 * S->pf * S->plane_f, S->nplanes_g, S->lz, d, S->cfg.eig_iterations,
                  S->cfg.seed, apply, dot, &S->lmin, &S->lmax, st);
  launch_inv<T>(d, static_cast<T*>(S->inv), L->ndofs, st);
  // u_k on the coarse level: interpolated down, Dirichlet values zeroed
  slab_to_coarse<double>(S, 2, S->uf, S->uc, st);
  launch_mask_zero<double>(S->uc, S->Lc->nnodes, S->Lc->mx, S->Lc->my, S->Lc->mz, S->Lc->faces, st);
  mg_linearize_any(S->mgc, S->uc, st);
  CK(cudaStreamSynchronize(st));
  S->linearized = true;
}

void solver_free(emfgpu_slab_solver* S) {
  if (!S) return;
  emfgpu_mg_destroy(S->mgc);
  emfgpu_level_destroy(S->Lc);
  emfgpu_transfer_destroy(S->tr);
  emfgpu_op_destroy(S->op64);
  emfgpu_op_destroy(S->opm);
  for (void* p : {S->face_lo, S->face_hi, S->ghost_lo, S->ghost_hi, S->fine_ext, S->coarse_ext, S->x0, S->b0, S->t0,
                  S->dg, S->inv, S->cr, S->cd, S->cad})
    cudaFree(p);
  cudaFree(S->uf);
  cudaFree(S->uc);
  cudaFree(S->part);
  cudaFree(S->lz);
  cudaFree(S->pcg);
  cudaFree(S->nbad);
  if (S->cs) cudaStreamDestroy(S->cs);
  if (S->ev_packed) cudaEventDestroy(S->ev_packed);
  if (S->ev_comm) cudaEventDestroy(S->ev_comm);
  delete S;
}

}  // namespace

emfgpu_status emfgpu_slab_solver_create(const emfgpu_level* slab, const emfgpu_level_desc* global, int rank,
                                        int world, emfgpu_comm* comm, int model, const emfgpu_material* params,
                                        int strategy, const emfgpu_mg_config* cfg, emfgpu_slab_solver** out) {
  if (!slab || !global || !params || !out || world < 1 || rank < 0 || rank >= world) return EMFGPU_ERR_INVALID;
  *out = nullptr;
  auto* S = new emfgpu_slab_solver;
  const emfgpu_status st = guarded(nullptr, [&] {
    if (world > 1 && (!comm || comm->world != world || comm->rank != rank))
      throw ApiError(EMFGPU_ERR_CONFIG, "slab solver: communicator rank/world differ");
    if (cfg)
      S->cfg = *cfg;
    else
      emfgpu_mg_default_config(&S->cfg);
    if (S->cfg.precision != 32 && S->cfg.precision != 64) throw ApiError(EMFGPU_ERR_CONFIG, "slab solver: precision");
    S->comm = comm;
    S->rank = rank;
    S->world = world;
    S->Lf = slab;
    S->gdesc = *global;
    S->gdesc.coords = nullptr;
    S->nzg = global->nz;
    slab_range(S->nzg, world, rank, S->k0, S->k1);
    if (slab->nz != S->k1 - S->k0 || slab->z_offset != S->k0 || slab->nx != global->nx || slab->ny != global->ny ||
        slab->p != global->p)
      throw ApiError(EMFGPU_ERR_CONFIG, "slab solver: the slab level is not rank's z-slab of the global level "
                                        "(SlabPartition: the first nz % world ranks take one more layer)");
    if (global->map == EMFGPU_MAP_COORDS)
      throw ApiError(EMFGPU_ERR_CONFIG, "slab solver: the global level needs a generated map (reference / shear_x)");
    if (slab->p < 2) throw ApiError(EMFGPU_ERR_CONFIG, "slab solver: the fine degree must be >= 2 (p-coarsened)");
    if (slab->periodic_y) throw ApiError(EMFGPU_ERR_CONFIG, "slab solver: periodic lattices are not supported");
    if (world > 1 && S->k1 - S->k0 < 2)
      throw ApiError(EMFGPU_ERR_CONFIG, "slab solver: every rank needs at least 2 element layers");
    S->lo = rank > 0;
    S->hi = rank < world - 1;
    S->pf = slab->p;
    S->pc = slab->p / 2;
    S->plane_f = 3 * (int64_t)slab->mx * slab->my;
    S->nplanes_g = S->nzg * S->pf + 1;
    const int dev = slab->device;
    CK(cudaSetDevice(dev));
    // operators on the slab
    emfgpu_status s1 = emfgpu_op_create(slab, model, params, 0, strategy, 64, &S->op64);
    if (s1 != EMFGPU_OK) throw ApiError(s1, std::string("slab solver: ") + emfgpu_global_last_error());
    s1 = emfgpu_op_create(slab, model, params, 0, strategy, S->cfg.precision, &S->opm);
    if (s1 != EMFGPU_OK) throw ApiError(s1, std::string("slab solver: ") + emfgpu_global_last_error());
    // the replicated coarse level and its hierarchy (the single-GPU MgHierarchy below level 0)
    emfgpu_level_desc dc = S->gdesc;
    dc.p = S->pc;
    dc.device = dev;
    s1 = emfgpu_level_create(&dc, &S->Lc);
    if (s1 != EMFGPU_OK) throw ApiError(s1, std::string("slab solver: coarse level: ") + emfgpu_global_last_error());
    s1 = emfgpu_mg_create(S->Lc, model, params, strategy, &S->cfg, &S->mgc);
    if (s1 != EMFGPU_OK) throw ApiError(s1, std::string("slab solver: coarse hierarchy: ") + emfgpu_global_last_error());
    S->plane_c = 3 * (int64_t)S->Lc->mx * S->Lc->my;
    // the slab extended by one ghost element layer per interface (dimensions only)
    const int nze = slab->nz + S->lo + S->hi;
    for (emfgpu_level* e : {&S->fext, &S->cext}) {
      e->nx = slab->nx;
      e->ny = slab->ny;
      e->nz = nze;
      e->device = dev;
    }
    S->fext.p = S->pf;
    S->cext.p = S->pc;
    for (emfgpu_level* e : {&S->fext, &S->cext}) {
      e->mx = e->nx * e->p + 1;
      e->my = e->ny * e->p + 1;
      e->mz = e->nz * e->p + 1;
      e->nnodes = (int64_t)e->mx * e->my * e->mz;
      e->ndofs = 3 * e->nnodes;
    }
    s1 = emfgpu_transfer_create(&S->fext, &S->cext, &S->tr);
    if (s1 != EMFGPU_OK) throw ApiError(s1, "slab solver: transfer");
    // buffers
    const size_t es = esize(S), n = (size_t)slab->ndofs;
    S->face_bytes = 8 * (size_t)emfgpu_op_face_values(S->op64);
    for (void** p : {&S->face_lo, &S->face_hi, &S->ghost_lo, &S->ghost_hi}) CK(cudaMalloc(p, S->face_bytes));
    CK(cudaMalloc(&S->fine_ext, 8 * (size_t)S->fext.ndofs));
    CK(cudaMalloc(&S->coarse_ext, 8 * (size_t)S->cext.ndofs));
    for (void** p : {&S->x0, &S->b0, &S->t0, &S->dg, &S->inv, &S->cr, &S->cd, &S->cad}) CK(cudaMalloc(p, es * n));
    CK(cudaMalloc(&S->uf, sizeof(double) * n));
    CK(cudaMalloc(&S->uc, sizeof(double) * (size_t)S->Lc->ndofs));
    CK(cudaMalloc(&S->part, sizeof(double) * ((size_t)S->nplanes_g * dot_plane_split() + 8)));
    CK(cudaMalloc(&S->nbad, sizeof(unsigned long long)));
    CK(cudaStreamCreateWithFlags(&S->cs, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&S->ev_packed, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&S->ev_comm, cudaEventDisableTiming));
  });
  if (st != EMFGPU_OK) {
    solver_free(S);
    return st;
  }
  *out = S;
  return EMFGPU_OK;
}

void emfgpu_slab_solver_destroy(emfgpu_slab_solver* s) { solver_free(s); }

const char* emfgpu_slab_solver_last_error(const emfgpu_slab_solver* s) { return s ? s->last_error.c_str() : ""; }

emfgpu_status emfgpu_slab_solver_update_linearization(emfgpu_slab_solver* S, const double* d_u, void* stream) {
  if (!S || !d_u) return EMFGPU_ERR_INVALID;
  return guarded(&S->last_error, [&] {
    CK(cudaSetDevice(S->Lf->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (S->cfg.precision == 64)
      slab_linearize<double>(S, d_u, st);
    else
      slab_linearize<float>(S, d_u, st);
  });
}

emfgpu_status emfgpu_slab_solver_apply(emfgpu_slab_solver* S, const double* d_x, double* d_y, void* stream) {
  if (!S || !d_x || !d_y) return EMFGPU_ERR_INVALID;
  return guarded(&S->last_error, [&] {
    if (!S->linearized) throw ApiError(EMFGPU_ERR_STALE, "slab solver: update_linearization has not run");
    CK(cudaSetDevice(S->Lf->device));
    slab_apply<double>(S, S->op64, d_x, d_y, static_cast<cudaStream_t>(stream));
  });
}

emfgpu_status emfgpu_slab_solver_precondition(emfgpu_slab_solver* S, const double* d_r, double* d_z, void* stream) {
  if (!S || !d_r || !d_z) return EMFGPU_ERR_INVALID;
  return guarded(&S->last_error, [&] {
    if (!S->linearized) throw ApiError(EMFGPU_ERR_STALE, "slab solver: update_linearization has not run");
    CK(cudaSetDevice(S->Lf->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (S->cfg.precision == 64)
      slab_precondition<double>(S, d_r, d_z, st);
    else
      slab_precondition<float>(S, d_r, d_z, st);
  });
}

// emfgpu_pcg_solve's host-driven loop (same kernels, same order) with the
// slab apply, the plane dot and the slab V-cycle
emfgpu_status emfgpu_slab_pcg_solve(emfgpu_slab_solver* S, const double* d_b, double* d_x, double rtol, int maxit,
                                    int* iterations, double* history, void* stream) {
  if (!S || !d_b || !d_x) return EMFGPU_ERR_INVALID;
  return guarded(&S->last_error, [&] {
    if (!S->linearized) throw ApiError(EMFGPU_ERR_STALE, "slab solver: update_linearization has not run");
    CK(cudaSetDevice(S->Lf->device));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t n = S->Lf->ndofs;
    const size_t need = sizeof(double) * (4 * (size_t)n + 8 + (size_t)maxit + 1) + 16;
    if (S->pcg_bytes < need) {
      cudaFree(S->pcg);
      S->pcg = nullptr;
      S->pcg_bytes = 0;
      CK(cudaMalloc(&S->pcg, need));
      S->pcg_bytes = need;
    }
    double* const r = S->pcg;
    double* const z = r + n;
    double* const p = z + n;
    double* const ap = p + n;
    double* const sc = ap + n;
    double* const dhist = sc + 8;
    int* const ic = reinterpret_cast<int*>(dhist + maxit + 1);
    auto dot_to = [&](const double* a, const double* b, double* out) { slab_dot<double>(S, a, b, S->part, out, s); };
    auto prec = [&](const double* rr, double* zz) {
      if (S->cfg.precision == 64)
        slab_precondition<double>(S, rr, zz, s);
      else
        slab_precondition<float>(S, rr, zz, s);
    };
    auto tail = [&]() {
      slab_apply<double>(S, S->op64, p, ap, s);
      dot_to(p, ap, sc + 1);
      launch_pcg_xr(d_x, r, p, ap, sc, n, s);
      dot_to(r, r, sc + 2);
      launch_pcg_check(sc, ic, dhist, rtol, maxit, cudaGraphConditionalHandle{}, 0, s);
    };
    CK(cudaMemsetAsync(d_x, 0, sizeof(double) * n, s));
    CK(cudaMemsetAsync(ic, 0, sizeof(int) * 3, s));
    CK(cudaMemcpyAsync(r, d_b, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
    dot_to(d_b, d_b, sc + 4);
    launch_pcg_sqrt(sc + 4, s);
    double bnorm = 0;
    CK(cudaMemcpyAsync(&bnorm, sc + 4, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    int it = 0;
    bool breakdown = false;
    double last_rel = 0.0;
    if (history) history[0] = 1.0;
    if (bnorm != 0 && maxit > 0) {
      prec(r, z);
      CK(cudaMemcpyAsync(p, z, sizeof(double) * n, cudaMemcpyDeviceToDevice, s));
      dot_to(r, z, sc + 0);
      tail();
      int hic[3] = {0, 0, 0};
      CK(cudaMemcpyAsync(hic, ic, sizeof(hic), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      while (!hic[1]) {
        prec(r, z);
        dot_to(r, z, sc + 3);
        launch_pcg_p(p, z, sc, n, s);
        launch_pcg_shift(sc, s);
        tail();
        CK(cudaMemcpyAsync(hic, ic, sizeof(hic), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
      }
      it = hic[0];
      breakdown = hic[2] != 0;
      if (it > 0) CK(cudaMemcpy(&last_rel, dhist + it, sizeof(double), cudaMemcpyDeviceToHost));
      if (history && it > 0) CK(cudaMemcpy(history + 1, dhist + 1, sizeof(double) * it, cudaMemcpyDeviceToHost));
    }
    if (iterations) *iterations = it;
    CK(cudaStreamSynchronize(s));
    if (breakdown)
      throw ApiError(EMFGPU_ERR_NUMERICAL, "slab pcg: breakdown (p^T A p <= 0) at iteration " + std::to_string(it));
    if (it > 0 && !(last_rel <= rtol))
      throw ApiError(EMFGPU_ERR_NUMERICAL, "slab pcg: no convergence in " + std::to_string(it) + " iterations");
  });
}
