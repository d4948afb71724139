/* emfgpu — B200 (sm_100a) matrix-free finite-strain tangent operator.
 *
 * C ABI of libemfgpu.so.  Plain pointers and sizes only.  Every entry point
 * replaces one method of the reference's operator-level C++ interface
 * (proj/include/elastmf/operator.hpp, solver.hpp, mesh.hpp — header-only
 * templates, no C ABI of their own; the reference's only C ABI,
 * proj/include/elastmf.h, is session-level).  Status codes and the per-handle
 * last-error string follow that C ABI's convention (elastmf.h:19-38,
 * capi.cpp:26-41).  A C++ adapter with the reference's exact method
 * signatures is in include/emfgpu/operator.hpp; INTEGRATION.md shows the
 * bindings a maintainer would add.
 *
 * Conventions (binding for parity):
 *   DoF = 3*node + comp; node = (c*my + b)*mx + a (a fastest); element
 *   e = (k*ny + j)*nx + i; Dirichlet faces bit f = -x,+x,-y,+y,-z,+z.
 *   Device-pointer entry points are stream-ordered (stream = cudaStream_t,
 *   taken literally: NULL = the legacy default stream) and do not
 *   synchronise; *_host entry points take host vectors, run on the handle's
 *   private stream, synchronise and report numerical errors.
 *   Calls on one handle (operator, hierarchy, transfer) may come from any
 *   streams and host threads at once: the handle orders them on the device
 *   (each call's work starts after the previous call's work on that handle,
 *   whichever stream it ran on), so they are serialised, never interleaved.
 *   Inside a CUDA stream capture the capturing caller owns that ordering.
 */
#ifndef EMFGPU_H
#define EMFGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum emfgpu_status {
  EMFGPU_OK = 0,
  EMFGPU_ERR_CONFIG = 1,    /* bad arguments / unsupported configuration (ConfigError) */
  EMFGPU_ERR_NUMERICAL = 2, /* det F <= 0, singular mapping (NonPositiveJacobian, ...) */
  EMFGPU_ERR_IO = 3,        /* reserved (EMF_ERR_IO) */
  EMFGPU_ERR_INVALID = 4,   /* null handle / out pointer */
  EMFGPU_ERR_STALE = 5,     /* apply/diagonal before update_linearization (StaleCache) */
  EMFGPU_ERR_CUDA = 6       /* CUDA runtime failure or no device */
} emfgpu_status;

typedef enum emfgpu_model { EMFGPU_CNH = 0, EMFGPU_INH = 1, EMFGPU_FIBER = 2 } emfgpu_model;
/* Strategy: the reference's none/scalar/tensor (material.hpp:25) plus the
 * cached displacement gradient (north star "cached F").  TENSOR caches
 * everything the apply needs of the linearization point: in the material
 * domain as the push-forward state K = J0^-1 F^-1, b and the coefficients with
 * det J0 w folded in (19 values per point, 35 for the fibre model, no geometry
 * read in the apply) instead of the reference's F, F^-1, S, C^-1 cell -- the
 * same operator to round-off, 152 B per point in fp64. */
typedef enum emfgpu_strategy {
  EMFGPU_NONE = 0,
  EMFGPU_SCALAR = 1,
  EMFGPU_TENSOR = 2,
  EMFGPU_CACHED_F = 3
} emfgpu_strategy;
typedef enum emfgpu_map {
  EMFGPU_MAP_REFERENCE = 0, /* DeformMap, mesh.cpp:128-136: param[0] = amplitude */
  EMFGPU_MAP_SHEAR_X = 1,   /* x' = x + param[0] sin(2 pi y) e_x (BASELINE cfg2) */
  EMFGPU_MAP_COORDS = 2,    /* node coordinates given in emfgpu_level_desc.coords */
  EMFGPU_MAP_TUBE = 3       /* BASELINE cfg3: x = radial, y = theta (use EMFGPU_LEVEL_PERIODIC_Y),
                               z = axial; param = {r_inner, r_outer, length} */
} emfgpu_map;

/* FeLevel(HexMesh, degree, DeformMap) + set_dirichlet, mesh.hpp:71-138.
 * EXT: boxes with nx,ny,nz elements and per-axis extents (the reference has a
 * single n, mesh.hpp:48-58). */
typedef struct emfgpu_level_desc {
  int nx, ny, nz;        /* elements per axis */
  int p;                 /* polynomial degree, 1..4 */
  double extent[3];      /* box lengths */
  int map;               /* emfgpu_map */
  double map_param[4];
  const double* coords;  /* host, 3 per node, when map == EMFGPU_MAP_COORDS */
  int dirichlet_faces;   /* bit mask, clamped to zero */
  int device;            /* CUDA device ordinal */
  int z_offset;          /* global index of element layer 0 (z slabs; colour parity) */
  int flags;             /* EMFGPU_LEVEL_* bits: disable geometry fast paths (testing) */
} emfgpu_level_desc;
#define EMFGPU_LEVEL_NO_CARTESIAN 1 /* use the general J0^-1 products even if J0 is diagonal */
#define EMFGPU_LEVEL_NO_AFFINE 2    /* store geometry per quadrature point even if affine */
#define EMFGPU_LEVEL_PERIODIC_Y 4   /* periodic lattice in y (my = ny*p; ny even) */

/* MaterialParams, material.hpp:36-50 (phi in radians; e1,e2,e3 frame). */
typedef struct emfgpu_material {
  double mu, lambda, kappa_b, k1, k2, a, b, phi;
  double e1[3], e2[3], e3[3];
} emfgpu_material;

typedef struct emfgpu_level emfgpu_level;
typedef struct emfgpu_op emfgpu_op;
typedef struct emfgpu_transfer emfgpu_transfer;
typedef struct emfgpu_cheb emfgpu_cheb;

const char* emfgpu_version(void);
/* Message of the last failure of a create call (thread-local). */
const char* emfgpu_global_last_error(void);

/* ---- FE level (FeLevel, mesh.hpp:71-138) -------------------------------- */
emfgpu_status emfgpu_level_create(const emfgpu_level_desc* desc, emfgpu_level** out);
void emfgpu_level_destroy(emfgpu_level* l);
int64_t emfgpu_level_n_dofs(const emfgpu_level* l);          /* FeLevel::dof_count */
int64_t emfgpu_level_n_elements(const emfgpu_level* l);
int emfgpu_level_affine(const emfgpu_level* l);              /* 1: geometry stored per element */
int emfgpu_level_cartesian(const emfgpu_level* l);           /* 1: affine, J0 diagonal (axis-aligned) fast path */
/* Reference->material Jacobians J0 (9 per qp, element-major, row = comp),
 * FeLevel::jacobians (mesh.hpp:97-99). host_out holds nel*(p+1)^3*9. */
emfgpu_status emfgpu_level_jacobians(const emfgpu_level* l, double* host_out);
emfgpu_status emfgpu_level_coords(const emfgpu_level* l, double* host_out); /* node_coords */
const char* emfgpu_level_last_error(const emfgpu_level* l);

/* ---- operator (ElasticOperator<Number>, operator.hpp:49-204) ---------------
 * domain: 0 material, 1 spatial (Formulation::domain, material.hpp:18-23; the
 * spatial form integrates on Omega_t with per-qp J_t and 1/J, operator.hpp:506-519;
 * cachedF is material-only -> EMFGPU_ERR_CONFIG).
 * precision: 64 (double) or 32 (float): the Number template argument. */
emfgpu_status emfgpu_op_create(const emfgpu_level* l, int model, const emfgpu_material* params, int domain,
                               int strategy, int precision, emfgpu_op** out);
/* The reference constructor's remaining arguments (operator.hpp:55-70):
 * Formulation (material.hpp:20-23; stability 1 = stable, the default, 0 =
 * standard) and KernelConfig (fastscalar.hpp:29-39).  The device kernels
 * implement the stable formulation with the default KernelConfig (16 ln
 * terms, 3 J^-2/3 Newton steps, exact exp, Newton J^-2/3); any other value
 * returns EMFGPU_ERR_CONFIG naming the field.  NULL = the defaults. */
typedef struct emfgpu_formulation {
  int stability; /* 0 standard, 1 stable */
  int domain;    /* 0 material, 1 spatial */
} emfgpu_formulation;
typedef struct emfgpu_kernel_config {
  int ln_series_terms;   /* 16 */
  int jpow_newton_steps; /* 3 */
  int exp_mode;          /* 0 exact, 1 fast */
  int jpow_mode;         /* 0 newton, 1 exact */
} emfgpu_kernel_config;
emfgpu_status emfgpu_op_create_ex(const emfgpu_level* l, int model, const emfgpu_material* params,
                                  const emfgpu_formulation* form, int strategy, int precision,
                                  const emfgpu_kernel_config* kernel_config, emfgpu_op** out);
void emfgpu_op_destroy(emfgpu_op* op);
int64_t emfgpu_op_n_dofs(const emfgpu_op* op);               /* n_dofs, operator.hpp:82 */
int emfgpu_op_precision(const emfgpu_op* op);
const char* emfgpu_op_last_error(const emfgpu_op* op);

/* update_linearization(u_k), operator.hpp:87/643-770: u_k in double, caches
 * computed in double and stored in Number.  NonPositiveJacobian ->
 * EMFGPU_ERR_NUMERICAL with the first (element, qpoint) in bad_element /
 * bad_qpoint (either may be NULL). */
emfgpu_status emfgpu_op_update_linearization_host(emfgpu_op* op, const double* u_k, int64_t* bad_element,
                                                  int* bad_qpoint);
emfgpu_status emfgpu_op_update_linearization(emfgpu_op* op, const double* d_u_k, int64_t* bad_element,
                                             int* bad_qpoint, void* stream);
int emfgpu_op_linearized(const emfgpu_op* op);               /* linearized(), :89 */
uint64_t emfgpu_op_checksum(const emfgpu_op* op);            /* checksum(), FNV-1a of u_k, :90 (computed on demand; synchronises) */

/* apply_tangent(du, y), operator.hpp:99-100/597-621: y = K(u_k) du with the
 * Dirichlet identity.  x, y: device arrays of n_dofs Number values. */
emfgpu_status emfgpu_op_apply(emfgpu_op* op, const void* d_x, void* d_y, void* stream);
/* Same through host vectors (H2D, apply, D2H, synchronise, error check).
 * With page-locked x and y (cudaHostAlloc / cudaHostRegister) and nz >= 8 the
 * copies are pipelined with the compute in z-chunks on the copy engines and
 * the whole sequence is replayed as a CUDA graph from the second call with
 * the same buffers; pageable buffers take the plain copy-apply-copy path. */
emfgpu_status emfgpu_op_apply_host(emfgpu_op* op, const void* x, void* y);
/* Numerical-error word of the stream-ordered calls (synchronises op's work). */
emfgpu_status emfgpu_op_check(emfgpu_op* op, int64_t* bad_element, int* bad_qpoint);

/* compute_diagonal(), operator.hpp:106-107/772-878: exact diag(K), 1 on
 * constrained rows; *n_nonpositive = number of free rows with diag <= 0. */
emfgpu_status emfgpu_op_compute_diagonal(emfgpu_op* op, void* d_diag, int64_t* n_nonpositive, void* stream);
/* Same, also returning compute_diagonal's second member: the DoF indices of
 * the free rows with diag <= 0, ascending (operator.hpp:869-877), the first
 * min(*n_nonpositive, capacity) of them in nonpositive_idx (host).
 * Synchronises the stream. */
emfgpu_status emfgpu_op_compute_diagonal_indices(emfgpu_op* op, void* d_diag, int64_t* nonpositive_idx,
                                                 int64_t capacity, int64_t* n_nonpositive, void* stream);
emfgpu_status emfgpu_op_compute_diagonal_host(emfgpu_op* op, void* diag, int64_t* n_nonpositive);

/* Byte ledger (operator.hpp:109-116, ledger.cpp:22-76): analytic per-qp
 * storage/traffic bytes of this operator's cell as stored on the device. */
emfgpu_status emfgpu_op_ledger(const emfgpu_op* op, int* storage_bytes_per_qp, int* traffic_bytes_per_qp,
                               double* traffic_bytes_per_dof);

/* Split apply for z-slab multi-GPU: element-phase on the
 * element layers [k0, k1) only, writing element-local results; then the node
 * phase for node planes [c0, c1].  apply == elements(0,nz) + nodes(0, mz-1). */
emfgpu_status emfgpu_op_apply_elements(emfgpu_op* op, const void* d_x, int k0, int k1, void* stream);
emfgpu_status emfgpu_op_apply_nodes(emfgpu_op* op, const void* d_x, void* d_y, int c0, int c1,
                                    const void* d_ghost_lo, const void* d_ghost_hi, void* stream);
/* Element-local result buffer of the last element phase (device, Number,
 * (e*(p+1)^3 + m)*3 + c) and its ghost-face layout size in values. */
void* emfgpu_op_local_buffer(emfgpu_op* op);
int64_t emfgpu_op_face_values(const emfgpu_op* op);
/* Pack the element-local results of element layer k restricted to its lower
 * (side 0) or upper (side 1) local node face into d_face (face_values). */
emfgpu_status emfgpu_op_pack_face(emfgpu_op* op, int k, int side, void* d_face, void* stream);

/* ---- hp-multigrid ingredients (solver.hpp, mesh.hpp) ------------------------ */
/* TransferOp(fine, coarse), mesh.hpp:157-182: p-coarsening (same mesh) or one
 * uniform h-step (n_fine = 2 n_coarse per axis). */
emfgpu_status emfgpu_transfer_create(const emfgpu_level* fine, const emfgpu_level* coarse, emfgpu_transfer** out);
void emfgpu_transfer_destroy(emfgpu_transfer* t);
/* kind 0 prolongate (coarse->fine), 1 restrict_ (fine->coarse, transpose),
 * 2 interpolate_down (fine->coarse nodal evaluation); precision 64|32. */
emfgpu_status emfgpu_transfer_apply(emfgpu_transfer* t, int kind, int precision, const void* d_in, void* d_out,
                                    void* stream);

/* ChebyshevSmoother<Number>::setup/smooth, solver.hpp:312-362. */
emfgpu_status emfgpu_cheb_create(emfgpu_op* op, const void* d_diag, double lmax_est, int degree,
                                 double range_factor, double safety, emfgpu_cheb** out);
void emfgpu_cheb_destroy(emfgpu_cheb* c);
emfgpu_status emfgpu_cheb_smooth(emfgpu_cheb* c, void* d_x, const void* d_b, int zero_start, void* stream);

/* estimate_eigenvalues(op, diag, iterations, seed), solver.hpp:262-308. */
emfgpu_status emfgpu_op_estimate_eigenvalues(emfgpu_op* op, const void* d_diag, int iterations, uint64_t seed,
                                             double* lambda_min, double* lambda_max);

/* Deterministic (fixed-order) double-accumulated dot product of two device
 * vectors of Number (dot_d, solver.hpp:95-100). */
emfgpu_status emfgpu_dot(int precision, const void* d_a, const void* d_b, int64_t n, double* out, void* stream);

/* ---- hp-multigrid preconditioner (MgHierarchy<Prec>, solver.hpp:437-581) ---
 * Ladder p -> p/2 -> ... -> 1 on the fine mesh, then uniform h-coarsening
 * (all of nx, ny, nz halved) while every count stays >= coarse_n (the
 * reference's n0, build_cube(n0, l)).  Coarse levels regenerate the fine
 * level's map.  Smoother: Chebyshev-Jacobi on every level; coarsest level:
 * Jacobi-PCG to coarse_rtol (the reference's CoarseSolver CG path). */
typedef struct emfgpu_mg emfgpu_mg;
typedef struct emfgpu_mg_config {
  int degree;            /* operator applications per smoothing pass (default 6) */
  double range_factor;   /* lambda_min = lambda_max / range_factor (15) */
  double safety;         /* lambda_max = safety * Lanczos estimate (1.2) */
  int eig_iterations;    /* Lanczos steps (20) */
  uint64_t seed;         /* Lanczos start vector seed (0x9e3779b97f4a7c15) */
  double coarse_rtol;    /* coarse CG relative tolerance (1e-4) */
  int coarse_maxit;      /* coarse CG iteration cap (500) */
  int coarse_n;          /* smallest element count per axis of the h-ladder (1) */
  int precision;         /* level precision: 32 (MgHierarchy<float>, default) or 64 */
  int64_t coarse_direct_limit; /* dense coarse solve below this many DoFs (2000, solver.hpp:444;
                                  0 = always the Jacobi-PCG path) */
} emfgpu_mg_config;
void emfgpu_mg_default_config(emfgpu_mg_config* cfg);
emfgpu_status emfgpu_mg_create(const emfgpu_level* fine, int model, const emfgpu_material* params, int strategy,
                               const emfgpu_mg_config* cfg, emfgpu_mg** out);
void emfgpu_mg_destroy(emfgpu_mg* mg);
int emfgpu_mg_n_levels(const emfgpu_mg* mg);
emfgpu_status emfgpu_mg_level_info(const emfgpu_mg* mg, int level, int* nx, int* ny, int* nz, int* p,
                                   int64_t* n_dofs);
const char* emfgpu_mg_last_error(const emfgpu_mg* mg);
/* MgHierarchy::update_linearization (solver.hpp:490-509): interpolate u_k down
 * the ladder, relinearize, diagonal, Lanczos, smoother setup. d_u: device fp64. */
emfgpu_status emfgpu_mg_update_linearization(emfgpu_mg* mg, const double* d_u_fine, void* stream);
/* MgHierarchy::precondition (solver.hpp:512-520): z = V-cycle(r), fp64 in/out. */
emfgpu_status emfgpu_mg_precondition(emfgpu_mg* mg, const double* d_r, double* d_z, void* stream);
/* Preconditioned CG in fp64 (BASELINE cfg4 outer solve; the reference's outer
 * solver is FGMRES, solver.hpp:120-203): x0 = 0, stop at ||r|| <= rtol ||b||.
 * mg may be NULL (unpreconditioned).  history (host, maxit+1) optional.
 * Returns EMFGPU_ERR_NUMERICAL (iterations, history and x still written) when
 * maxit is reached without ||r|| <= rtol ||b||, or on breakdown (p^T A p <= 0),
 * like the reference's CgNoConvergence / LinearSolveFailure (solver.hpp:202, 423). */
emfgpu_status emfgpu_pcg_solve(emfgpu_op* op, emfgpu_mg* mg, const double* d_b, double* d_x, double rtol,
                               int maxit, int* iterations, double* history, void* stream);

/* Fibre model with a per-quadrature-point frame field (SURVEY §8(c) gap 2):
 * kind 0 = the global frame of the material (default), 1 = cylindrical frame
 * about the z axis at each qp (e1 circumferential, e2 axial, e3 radial; the
 * families at +-phi from e1), 2 = the material's frame replicated per qp.
 * Call before update_linearization. */
emfgpu_status emfgpu_op_set_fibre_frame(emfgpu_op* op, int kind);
/* Per-qp H4,H6 (12 per qp, SoA field-major) and M1_4,M1_6 (6 per qp). */
emfgpu_status emfgpu_op_fibre_field(const emfgpu_op* op, double* h_out, double* m1_out);

/* ---- z-slab multi-GPU apply ------------------------
 * One slab per GPU: rank r of `world` owns element layers [k0, k1) of the
 * global box; its level is created with z_offset = k0, the slab's node
 * planes [k0 p, k1 p] (interface planes duplicated) and the slab's own
 * Dirichlet faces.  The reference has no distributed path; these calls replace
 * ElasticOperator::apply_tangent for a partitioned operator.
 * Communicator: NCCL, loaded at run time (libnccl.so.2 already in the process,
 * e.g. torch's, else the system one).  emfgpu_comm_unique_id on one rank, the
 * 128 bytes shipped to the others by the caller, emfgpu_comm_create on every
 * rank (ncclGetUniqueId / ncclCommInitRank); or emfgpu_comm_wrap of an
 * existing ncclComm_t (not destroyed by emfgpu_comm_destroy). */
typedef struct emfgpu_comm emfgpu_comm;
typedef struct emfgpu_slab emfgpu_slab;
emfgpu_status emfgpu_comm_unique_id(unsigned char id[128]);
emfgpu_status emfgpu_comm_create(const unsigned char id[128], int world, int rank, int device, emfgpu_comm** out);
emfgpu_status emfgpu_comm_wrap(void* nccl_comm, int world, int rank, emfgpu_comm** out);
/* One process, one host thread per rank: `world` communicators (out[r] for
 * rank r, devices[r] its GPU, NULL = all on device 0) joined by a host
 * rendezvous; the collectives become peer copies.  Rank r's calls must come
 * from its own thread (every rank makes the same sequence of calls). */
emfgpu_status emfgpu_comm_create_group(int world, const int* devices, emfgpu_comm** out);
void emfgpu_comm_destroy(emfgpu_comm* c);
/* comm may be NULL for world == 1 and for single-process groups. */
emfgpu_status emfgpu_slab_create(emfgpu_op* op, int rank, int world, emfgpu_comm* comm, emfgpu_slab** out);
void emfgpu_slab_destroy(emfgpu_slab* s);
const char* emfgpu_slab_last_error(const emfgpu_slab* s);
/* y = K x on this rank's slab vectors: boundary element layers, interface
 * faces packed, NCCL send/recv with the z neighbours on the slab's own
 * communication stream overlapped with the interior layers, node phase with
 * the ghost faces in the global colour order.  Each rank's y is bitwise the
 * single-GPU result on its node planes.  Stream-ordered, graph-capturable. */
emfgpu_status emfgpu_slab_apply(emfgpu_slab* s, const void* d_x, void* d_y, void* stream);
/* One process driving all n slabs (slabs[r] = rank r of world n; one per
 * device, or several on one device): the same apply with the ghost faces
 * copied peer-to-peer (NVLink) instead of NCCL, phases enqueued in order
 * across the group so no kernel ever waits on another. */
emfgpu_status emfgpu_slab_group_apply(emfgpu_slab* const* slabs, int n, const void* const* d_x, void* const* d_y,
                                      void* const* streams);
/* Global dot of two slab vectors into a device double: each interface plane
 * counted once (owned by the upper rank); the per-rank fixed-order partials
 * are all-gathered (NCCL) and summed in rank order on the device --
 * identical on every rank, no host synchronisation. */
emfgpu_status emfgpu_slab_dot(emfgpu_slab* s, const void* d_a, const void* d_b, double* d_out, void* stream);
emfgpu_status emfgpu_slab_group_dot(emfgpu_slab* const* slabs, int n, const void* const* d_a, const void* const* d_b,
                                    double* const* d_out, void* const* streams);

/* ---- the cfg4 solve in z slabs (SURVEY §8(e) ¶3) -------------------------------
 * fp64 PCG preconditioned by the hp-multigrid V-cycle with the finest level
 * partitioned like the apply (faces exchanged, node-plane dots all-gathered)
 * and the next level (p/2, same mesh) and everything below agglomerated:
 * every rank holds them whole and runs that part of the V-cycle redundantly.
 * Every rank's iterates are bitwise the single-GPU emfgpu_pcg_solve's with
 * emfgpu_mg_create(global level, ..., cfg) on its node planes.
 * slab: the rank's z-slab level of `global` (the SlabPartition split: the
 * first nz % world ranks take one more element layer; z_offset = first
 * layer); global: the whole fine level's description (generated map);
 * fine degree >= 2, >= 2 element layers per rank.  All calls are collective
 * (SPMD) over the communicator. */
typedef struct emfgpu_slab_solver emfgpu_slab_solver;
emfgpu_status emfgpu_slab_solver_create(const emfgpu_level* slab, const emfgpu_level_desc* global, int rank,
                                        int world, emfgpu_comm* comm, int model, const emfgpu_material* params,
                                        int strategy, const emfgpu_mg_config* cfg, emfgpu_slab_solver** out);
void emfgpu_slab_solver_destroy(emfgpu_slab_solver* s);
const char* emfgpu_slab_solver_last_error(const emfgpu_slab_solver* s);
/* update_linearization of the outer operator and the whole hierarchy; d_u: the slab's u_k (fp64). */
emfgpu_status emfgpu_slab_solver_update_linearization(emfgpu_slab_solver* s, const double* d_u, void* stream);
emfgpu_status emfgpu_slab_solver_apply(emfgpu_slab_solver* s, const double* d_x, double* d_y, void* stream);
emfgpu_status emfgpu_slab_solver_precondition(emfgpu_slab_solver* s, const double* d_r, double* d_z, void* stream);
/* emfgpu_pcg_solve on the slab vectors (same status conventions). */
emfgpu_status emfgpu_slab_pcg_solve(emfgpu_slab_solver* s, const double* d_b, double* d_x, double rtol, int maxit,
                                    int* iterations, double* history, void* stream);

/* ---- residual and loads ----------------------------------
 * evaluate_residual(u, r), operator.hpp:94-95/623-641 (both domains):
 * r_i = (Grad v_i, F S) - load_scale * load_i, Dirichlet rows zeroed. */
emfgpu_status emfgpu_op_residual(emfgpu_op* op, const void* d_u, void* d_r, void* stream);
emfgpu_status emfgpu_op_residual_host(emfgpu_op* op, const void* u, void* r);
/* Loads::pressure on face (operator.hpp:23-32, 995-1001): traction -p N on the
 * reference geometry of face `face` (-x,+x,-y,+y,-z,+z = 0..5). */
emfgpu_status emfgpu_op_set_pressure(emfgpu_op* op, double pressure, int face);
emfgpu_status emfgpu_op_set_load_scale(emfgpu_op* op, double scale); /* set_load_scale, :80 */
/* The full Loads struct (operator.hpp:23-32): pressure on one face, a body
 * force B(X) integrated over Omega_0 at the Gauss points, and general
 * tractions h(X, N) on the faces flagged in traction_faces (bit f = face f);
 * build_load_vector, operator.hpp:880-1008.  The reference's std::function
 * members become C callbacks evaluated on the host while the load vector is
 * built (once, here; the vector is then kept on the device).  NULL callbacks
 * = absent.  Replaces any earlier loads of the operator. */
typedef void (*emfgpu_body_force_fn)(const double X[3], double out[3], void* user);
typedef void (*emfgpu_traction_fn)(const double X[3], const double N[3], double out[3], void* user);
typedef struct emfgpu_loads {
  double pressure;
  int pressure_face;
  emfgpu_body_force_fn body_force;
  void* body_force_user;
  emfgpu_traction_fn traction;
  void* traction_user;
  int traction_faces;
} emfgpu_loads;
emfgpu_status emfgpu_op_set_loads(emfgpu_op* op, const emfgpu_loads* loads);

/* ---- Newton-Krylov on the device ------------------------
 * fgmres_solve (solver.hpp:120-203): right-preconditioned FGMRES(restart) with
 * modified Gram-Schmidt; x in/out; mg may be NULL. */
emfgpu_status emfgpu_fgmres_solve(emfgpu_op* op, emfgpu_mg* mg, const double* d_b, double* d_x, double abs_tol,
                                  double rel_tol, int restart, int max_restarts, int* iterations,
                                  double* final_residual, void* stream);
typedef struct emfgpu_newton_config {
  double eps_abs, eps_rel; /* NewtonConfig (solver.hpp:26-30): 1e-8, 1e-3 */
  int max_iter;            /* 25 */
  double lin_abs_tol, lin_rel_tol; /* FgmresConfig (solver.hpp:32-37): 1e-12, 1e-3 */
  int restart, max_restarts;        /* 30, 40 */
} emfgpu_newton_config;
void emfgpu_newton_default_config(emfgpu_newton_config* cfg);
/* newton_solve (solver.hpp:603-656) with the op's loads: d_u (fp64) in/out. */
emfgpu_status emfgpu_newton_solve(emfgpu_op* op, emfgpu_mg* mg, double* d_u, const emfgpu_newton_config* cfg,
                                  int* newton_iterations, int* linear_iterations, double* final_residual,
                                  void* stream);

/* ---- forward-stability lab ------------------------------
 * run_sweep (stability.hpp, stability.cpp:163-251) on the device: per scale,
 * samples_per_scale seeded gradient/direction pairs (SweepRng streams), every
 * cell evaluated in fp64 and fp32 with the reference formulas (no FMA
 * contraction).  Outputs n_scales * 32 cells, scale-major, then model (cNH,
 * iNH, fibre, SVK), formulation (standard-material, stable-material,
 * standard-spatial, stable-spatial), quantity (stress, tangent) — the
 * reference's write_csv order.  Scales must be positive and increasing. */
#define EMFGPU_SWEEP_CELLS 32
emfgpu_status emfgpu_stability_sweep(const double* scales, int n_scales, int samples_per_scale, uint64_t seed,
                                     const emfgpu_material* params, double* max_rel_error, int64_t* count_invalid);

/* Host-vector Newton solve (u in/out on the host, one upload and one download):
 * the signature of newton_solve(op, &mg, u, ...) for reference-style drivers
 * (runner.cpp:166-204). */
emfgpu_status emfgpu_newton_solve_host(emfgpu_op* op, emfgpu_mg* mg, double* u, const emfgpu_newton_config* cfg,
                                       int* newton_iterations, int* linear_iterations, double* final_residual);

/* FMA-pipe peak (TFLOP/s, 2 flops per FMA) measured by a register-resident
 * FMA loop over one wave of CTAs for `seconds`: the FP64/FP32 roofline
 * denominator (bench.py). */
emfgpu_status emfgpu_bench_fma_peak(int precision, double seconds, double* tflops);

#ifdef __cplusplus
}
#endif

#endif /* EMFGPU_H */
