// Internal declarations shared by the CUDA translation units of libemfgpu.
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/emfgpu.h"
#include "kernels.cuh"

namespace emfgpu {

constexpr int kMaxP = 4;


// Per-(T,P) launchers, defined in inst_<t><p>.cu.
template <typename T, int P>
void launch_apply(int model, int strategy, const KArgs<T>& a, int64_t e0, int64_t e1, cudaStream_t s);
template <typename T, int P>
void launch_linearize(int model, const KArgs<T>& a, cudaStream_t s);
template <typename T, int P>
void launch_diagonal(int model, const KArgs<T>& a, cudaStream_t s);
template <typename T, int P>
void launch_residual(int model, const KArgs<T>& a, cudaStream_t s);
// solver.cu: r = r - scale * load, then Dirichlet rows zeroed
template <typename T>
void launch_sub_load_mask(T* r, const T* load, double scale, int64_t nnodes, int mx, int my, int mz, int faces,
                          cudaStream_t s);

// gather.cu
template <typename T>
void launch_node_gather(const T* loc, const T* ghost_lo, const T* ghost_hi, const T* x, T* y, int nx, int ny,
                        int nz, int p, int faces, int kpar, int c0, int c1, int periodic_y, cudaStream_t s,
                        bool pdl = true);
template <typename T>
void launch_pack_face(const T* loc, T* face, int nx, int ny, int p, int k, int side, cudaStream_t s);
template <typename T>
void launch_diag_finish(T* d, int64_t nnodes, int mx, int my, int mz, int faces, unsigned long long* nbad,
                        long long* bad_idx, long long cap, cudaStream_t s);

// coarse.cu: dense coarse solve (probing assembly, Gauss-Jordan inverse, GEMV)
template <typename T>
void launch_probe_fill(T* x, int mx, int my, int mz, int s, int ca, int cb, int cc, int comp, cudaStream_t st);
template <typename T>
void launch_probe_extract(const T* y, double* A, int64_t n, int mx, int my, int mz, int p, int s, int ca, int cb,
                          int cc, int comp, cudaStream_t st);
void launch_dense_invert(const double* A, double* M, int n, int* d_singular, cudaStream_t st);
template <typename T>
void launch_coarse_gemv(const double* M, const T* b, T* x, int n, cudaStream_t st);

// stability.cu
void run_stability_sweep(const double* scales, int n_scales, int samples, uint64_t seed, const emfgpu_material& p,
                         const double h[2][6], const double m1[2][3], double* max_rel_error, int64_t* count_invalid);

// geometry.cu
void launch_geometry(const double* coords, double* geo_q, double* j0_out, int nx, int ny, int nz, int p,
                     const double* B, const double* D, const double* qw, int* nonaffine, int* degenerate,
                     int periodic_y, cudaStream_t s);
void launch_fibre_frame(const double* coords, double* hq, double* m1q, int nx, int ny, int nz, int p, int periodic_y,
                        const double* B, double h11, double h22, double h33, double phi, int kind,
                        const double* frame, cudaStream_t s);
void launch_geo_compact(const double* geo_q, double* geo_e, int64_t nel, int nq3, cudaStream_t s);
void launch_cast_d2f(const double* in, float* out, int64_t n, cudaStream_t s);

// solver.cu
template <typename T>
void launch_transfer_axis(const T* in, T* out, const int* src_elem, const double* w, const int* t_ptr, const int* t_d,
                          const int* t_s, int stencil, int p_src, int transpose, int axis, int in0, int in1, int in2,
                          int out_na, cudaStream_t s);
template <typename T>
void launch_cheb_first(T* x, T* r, T* d, const T* b, const T* inv_diag, double inv_theta, int zero_start, int64_t n,
                       cudaStream_t s);
template <typename T>
void launch_cheb_step(T* x, T* r, T* d, const T* ad, const T* inv_diag, double f1, double f2, int64_t n,
                      cudaStream_t s);
template <typename T>
void launch_inv(const T* d, T* inv, int64_t n, cudaStream_t s);
template <typename T>
void launch_dot(const T* a, const T* b, int64_t n, double* partial, double* out, cudaStream_t s);
int dot_partial_count();
// node-plane-chunked deterministic dot (solver.cu): partial slots = nplanes * dot_plane_split()
template <typename T>
void launch_dot_plane_partials(const T* a, const T* b, int64_t plane_len, int nplanes, int first_plane,
                               double* partial, cudaStream_t s);
void launch_sum_ordered(const double* partial, int64_t m, double* out, cudaStream_t s);
int dot_plane_split();
template <typename T>
void launch_dot_planes(const T* a, const T* b, int64_t plane_len, int nplanes, double* partial, double* out,
                       cudaStream_t s);

template <typename T>
void launch_scale_to_T(const double* s, const double* v, T* t, int64_t n, cudaStream_t st);
template <typename T>
void launch_scale_from_T(const double* s, const T* at, double* w, int64_t n, cudaStream_t st);
template <typename T>
void launch_dinv_sqrt(const T* d, double* s, int64_t n, cudaStream_t st);
void launch_axpy_minus(double a, const double* x, double* y, int64_t n, cudaStream_t st);
void launch_lanczos_start(double* v, int64_t n, unsigned long long seed, cudaStream_t st, int64_t offset = 0);
void launch_axpy_dev(const double* c, const double* x, double* y, int64_t n, cudaStream_t st);
// k plane-chunked dots of a against basis + v * stride in one pass (out[v], bitwise
// launch_dot_planes per vector; partial: k rows of pstride doubles), and
// y -= sum_v c[v] basis_v in order
void launch_multi_dot_planes(const double* a, const double* basis, int64_t stride, int k, int64_t plane_len,
                             int nplanes, double* partial, int64_t pstride, double* out, cudaStream_t s);
void launch_multi_axpy_dev(const double* c, const double* basis, int64_t stride, int k, double* y, int64_t n,
                           cudaStream_t s);
void launch_div_sqrt_dev(const double* d, const double* x, double* y, int64_t n, cudaStream_t st);
void launch_div(const double* x, double b, double* y, int64_t n, cudaStream_t st);
template <typename T>
void launch_mask_zero(T* v, int64_t nnodes, int mx, int my, int mz, int faces, cudaStream_t s);
template <typename Ti, typename To>
void launch_cast(const Ti* in, To* out, int64_t n, cudaStream_t s);
template <typename T>
void launch_bminus(const T* b, T* t, int64_t n, cudaStream_t s);
template <typename T>
void launch_add(const T* x, T* y, int64_t n, cudaStream_t s);
template <typename T>
void launch_cg_xr(T* x, T* r, const T* p, const T* ap, double alpha, int64_t n, cudaStream_t s);
template <typename T>
void launch_cg_p(T* p, const T* z, double beta, int64_t n, cudaStream_t s);
// geometry.cu: u_k in the Q3 staging layout per element (size = Lay<4>::SIZE)
template <typename T>
void launch_uk_elem(const T* uk, T* out, int64_t nel, int nx, int ny, int mx, int my, int size, cudaStream_t s);
// device-resident PCG (solver.cu)
void launch_pcg_xr(double* x, double* r, const double* p, const double* ap, const double* sc, int64_t n,
                   cudaStream_t s);
void launch_pcg_p(double* p, const double* z, const double* sc, int64_t n, cudaStream_t s);
void launch_pcg_shift(double* sc, cudaStream_t s);
void launch_pcg_sqrt(double* v, cudaStream_t s);
void launch_pcg_check(const double* sc, int* ic, double* hist, double rtol, int maxit, cudaGraphConditionalHandle h,
                      int use_h, cudaStream_t s);
template <typename T>
void launch_jacobi(const T* inv, const T* r, T* z, int64_t n, cudaStream_t s);

}  // namespace emfgpu

struct emfgpu_level {
  int nx = 0, ny = 0, nz = 0, p = 0, mx = 0, my = 0, mz = 0;
  int64_t nnodes = 0, ndofs = 0, nel = 0, nq3 = 0;
  int faces = 0, device = 0, affine = 0, z_offset = 0, cartesian = 0, periodic_y = 0;
  double extent[3] = {1, 1, 1};
  // basis tables (host): GLL nodes, Gauss points/weights, B/D (row = qp)
  std::vector<double> nodes, qpts, qwts, B, D;
  std::vector<double> Dc;  // collocated derivative on the Gauss points: Dc[q][r] = l_r'(g_q), D = Dc B
  double* d_coords = nullptr;  // 3 per node
  double* d_geo = nullptr;     // SoA, 10 fields: J0^-1 (9), det J0 * w_q (or det J0 if affine)
  float* d_geo_f = nullptr;
  int64_t geo_stride = 0;
  emfgpu_level_desc desc{};  // creation parameters (coords pointer cleared), for hierarchies
  std::string last_error;
};

struct emfgpu_op {
  const emfgpu_level* L = nullptr;
  int model = 0, strategy = 0, precision = 64;
  int domain = 0;  // 0 material, 1 spatial (Formulation::domain, material.hpp:18-23)
  emfgpu_material params{};
  emfgpu::MatConst<double> matd{};
  emfgpu::MatConst<float> matf{};
  void* d_cache = nullptr;
  int64_t cache_stride = 0;
  int n_cache_fields = 0;
  void* d_uk = nullptr;        // u_k in Number (none/scalar)
  double* d_ukd = nullptr;     // u_k in double (transfers / host checks)
  void* d_loc = nullptr;       // element-local results, nel*nn3*3 Number
  void* d_x = nullptr;         // staging for host entry points
  void* d_y = nullptr;
  unsigned long long* d_err = nullptr;
  unsigned long long* d_nbad = nullptr;  // compute_diagonal: count of nonpositive free rows
  unsigned long long* h_err = nullptr;  // pinned
  // Lanczos work space (estimate_eigenvalues), kept across relinearizations
  double* lz_buf = nullptr;
  size_t lz_bytes = 0;
  // PCG / FGMRES work spaces, kept across solves
  void* pcg_buf = nullptr;
  size_t pcg_bytes = 0;
  void* fgmres_buf = nullptr;
  size_t fgmres_bytes = 0;
  // per-qp fibre frame field (fibre model): H4/H6 in double and Number, M1s
  int frame_kind = 0;
  double* d_hqd = nullptr;
  double* d_m1qd = nullptr;
  void* d_hq = nullptr;
  cudaStream_t stream = nullptr;
  // pipelined host-vector apply: copy streams + per-chunk events
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  static constexpr int kMaxChunks = 32;
  cudaEvent_t ev_h2d[kMaxChunks] = {}, ev_comp[kMaxChunks] = {}, ev_start = nullptr, ev_done = nullptr;
  cudaGraphExec_t gexec = nullptr;  // captured pipeline for (g_x, g_y, g_nch)
  // Loads (operator.hpp:23-32, 880-1008): pressure on one face, scaled
  void* d_load = nullptr;  // Number, n_dofs (null: no load)
  double load_scale = 1.0;
  const void* g_x = nullptr;
  void* g_y = nullptr;
  int g_nch = 0;
  // apply_v2 ticket counters: a ring of slots, one per launch, so launches
  // of this operator on different streams never share a counter
  static constexpr int kTicketSlots = 256;
  unsigned* d_ctr = nullptr;
  void* d_uk_el = nullptr;  // Q3 none/scalar: u_k per element in the staging layout (KArgs::uk_el)
  mutable std::atomic<unsigned> ticket_seq{0};  // host threads may launch concurrently
  // entry-point ordering across streams and host threads (capi.cu, UseGuard)
  std::recursive_mutex use_mu;
  cudaEvent_t ev_use = nullptr;
  bool linearized = false;
  // checksum() (operator.hpp:90): FNV-1a of u_k.  The hash is byte-serial
  // (0.19 s on the host for cfg4's 172 MB), so it is computed on demand from
  // the device copy of u_k instead of in every update_linearization.
  mutable uint64_t checksum = 0;
  mutable bool checksum_valid = true;
  std::string last_error;
};
