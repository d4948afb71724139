// Explicit instantiation of the element kernels for one (Number, degree).
// Included by inst_<t><p>.cu with EMF_T and EMF_P defined, so the 8 units
// compile in parallel.
#include <algorithm>

#include "apply_v2.cuh"
#include "apply_v3.cuh"
#include "internal.h"

// fp32 Q3 none / scalar on axis-aligned meshes ran on the warp-per-element v3
// until the dense v2 got the collocated sweeps (cNH none 0.1096 -> 0.0953 ms,
// profiles/r02_q3_collocated_ab.txt); v3 now serves Q2 only.
#ifndef EMF_F32_V3CART
#define EMF_F32_V3CART 0
#endif
#ifndef EMF_V3_ENABLE
#define EMF_V3_ENABLE 1
#endif

namespace emfgpu {


template <int MODEL, int STRAT, bool CART>
static void apply_one(const KArgs<EMF_T>& a, int64_t e0, int64_t e1, cudaStream_t s) {
  constexpr int N = EMF_P + 1, EPB = TileV2<EMF_P, sizeof(EMF_T)>::EPB, THREADS = EPB * N * N * N;
  const int64_t cnt = e1 - e0;
  if (cnt <= 0) return;
  // Kernel choice measured on B200 (tools/apply_ab.py; profiles/r01_e2e_findings.md):
  // the warp-per-element v3 for Q2 (fp32, and fp64 tensor / cachedF); the
  // dense v2 everywhere else (after the ticket loop and the dense Q3 mapping it
  // beat v3 for Q3 tensor / cachedF in both precisions: fp32 curved iNH tensor
  // 0.169 -> 0.114 ms, fibre 0.169 -> 0.120; fp64 iNH tensor 0.214 -> 0.163,
  // cNH tensor 0.1445 -> 0.1384, cachedF 0.159 -> 0.151).
  constexpr bool kTC = STRAT == S_CACHEDF || STRAT == S_TENSOR;
  constexpr bool kF32V3 = EMF_F32_V3CART && sizeof(EMF_T) == 4 && CART && !is_spatial(STRAT) &&
                          (STRAT == S_NONE || STRAT == S_SCALAR);
  // (v3 reads the material tensor bundle; the cNH / iNH tensor cache holds the
  // push-forward state, which only v2 consumes -- v2 and v3 measured equal at Q2)
  constexpr bool kV3 = EMF_V3_ENABLE && !is_resid(STRAT) && !(STRAT == S_TENSOR && tensor_compact(MODEL, 0)) &&
                       (EMF_P == 2 ? (sizeof(EMF_T) == 4 || kTC) : (EMF_P == 3 && kF32V3));
  if constexpr (kV3) {
    // warp-per-element kernel (apply_v3.cuh)
    constexpr size_t smem = sizeof(ApplyV3Warp<EMF_T, EMF_P, MODEL, STRAT>) * kV3Warps;
    static std::atomic<int> shape3[64];
    int per_sm3 = 0, sms3 = 0;
    per_device_shape(shape3, sms3, per_sm3, [&](int& p) {
      cudaFuncSetAttribute(apply_v3_kernel<EMF_T, EMF_P, MODEL, STRAT, CART>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p, apply_v3_kernel<EMF_T, EMF_P, MODEL, STRAT, CART>,
                                                    32 * kV3Warps, smem);
    });
    KArgs<EMF_T> b = a;
    b.e_begin = e0;
    b.nel = e1;
    const int64_t blocks = (cnt + kV3Warps - 1) / kV3Warps;
    const int64_t grid = std::min<int64_t>(blocks, (int64_t)sms3 * per_sm3);
    apply_v3_kernel<EMF_T, EMF_P, MODEL, STRAT, CART><<<(unsigned)grid, 32 * kV3Warps, smem, s>>>(b);
    return;
  }
  // persistent grid: one wave at the kernel's occupancy
  static std::atomic<int> shape[64];
  int per_sm = 0, sms = 0;
  per_device_shape(shape, sms, per_sm, [&](int& p) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p, apply_v2_kernel<EMF_T, EMF_P, MODEL, STRAT, CART>, THREADS, 0);
  });
  KArgs<EMF_T> b = a;
  b.e_begin = e0;
  b.nel = e1;
  const int64_t groups = (cnt + EPB - 1) / EPB;
  const int64_t grid = std::min<int64_t>(groups, (int64_t)sms * per_sm);
  apply_v2_kernel<EMF_T, EMF_P, MODEL, STRAT, CART><<<(unsigned)grid, THREADS, 0, s>>>(b, groups);
}

template <>
void launch_apply<EMF_T, EMF_P>(int model, int strategy, const KArgs<EMF_T>& a, int64_t e0, int64_t e1,
                               cudaStream_t s) {
#define EMF_CASE(M, S)                                                  \
  if (model == M && strategy == S) {                                    \
    if (a.cartesian) return apply_one<M, S, true>(a, e0, e1, s);        \
    return apply_one<M, S, false>(a, e0, e1, s);                        \
  }
  EMF_CASE(CNH, S_NONE) EMF_CASE(CNH, S_SCALAR) EMF_CASE(CNH, S_TENSOR) EMF_CASE(CNH, S_CACHEDF)
  EMF_CASE(INH, S_NONE) EMF_CASE(INH, S_SCALAR) EMF_CASE(INH, S_TENSOR) EMF_CASE(INH, S_CACHEDF)
  EMF_CASE(FIBER, S_NONE) EMF_CASE(FIBER, S_SCALAR) EMF_CASE(FIBER, S_TENSOR) EMF_CASE(FIBER, S_CACHEDF)
#undef EMF_CASE
#define EMF_SP(M, S) \
  if (model == M && strategy == S) return apply_one<M, S, false>(a, e0, e1, s);
  EMF_SP(CNH, S_SP_NONE) EMF_SP(CNH, S_SP_SCALAR) EMF_SP(CNH, S_SP_TENSOR)
  EMF_SP(INH, S_SP_NONE) EMF_SP(INH, S_SP_SCALAR) EMF_SP(INH, S_SP_TENSOR)
  EMF_SP(FIBER, S_SP_NONE) EMF_SP(FIBER, S_SP_SCALAR) EMF_SP(FIBER, S_SP_TENSOR)
#undef EMF_SP
}

template <>
void launch_linearize<EMF_T, EMF_P>(int model, const KArgs<EMF_T>& a, cudaStream_t s) {
  constexpr int N = EMF_P + 1, EPB = Tile<EMF_P>::EPB;
  KArgs<EMF_T> b = a;
  b.e_begin = 0;
  const unsigned blocks = (unsigned)((a.nel + EPB - 1) / EPB);
  if (model == CNH) linearize_kernel<EMF_T, EMF_P, CNH><<<blocks, EPB * N * N * N, 0, s>>>(b);
  if (model == INH) linearize_kernel<EMF_T, EMF_P, INH><<<blocks, EPB * N * N * N, 0, s>>>(b);
  if (model == FIBER) linearize_kernel<EMF_T, EMF_P, FIBER><<<blocks, EPB * N * N * N, 0, s>>>(b);
}

template <>
void launch_diagonal<EMF_T, EMF_P>(int model, const KArgs<EMF_T>& a, cudaStream_t s) {
  constexpr int N = EMF_P + 1, EPB = Tile<EMF_P>::EPB;
  KArgs<EMF_T> b = a;
  b.e_begin = 0;
  const unsigned blocks = (unsigned)((a.nel + EPB - 1) / EPB);
  if (model == CNH) diagonal_kernel<EMF_T, EMF_P, CNH><<<blocks, EPB * N * N * N, 0, s>>>(b);
  if (model == INH) diagonal_kernel<EMF_T, EMF_P, INH><<<blocks, EPB * N * N * N, 0, s>>>(b);
  if (model == FIBER) diagonal_kernel<EMF_T, EMF_P, FIBER><<<blocks, EPB * N * N * N, 0, s>>>(b);
}

// evaluate_residual's element phase: the persistent v2 element kernel with the
// stress integrand (EMF_RESID_V2 = 0: the round-1 thread-per-point kernel)
#ifndef EMF_RESID_V2
#define EMF_RESID_V2 1
#endif
template <>
void launch_residual<EMF_T, EMF_P>(int model, const KArgs<EMF_T>& a, cudaStream_t s) {
  if (EMF_RESID_V2) {
#define EMF_RCASE(M)                                                                       \
  if (model == M) {                                                                        \
    if (a.spatial) return apply_one<M, S_RESID_SP, false>(a, 0, a.nel, s);                 \
    if (a.cartesian) return apply_one<M, S_RESID, true>(a, 0, a.nel, s);                   \
    return apply_one<M, S_RESID, false>(a, 0, a.nel, s);                                   \
  }
    EMF_RCASE(CNH) EMF_RCASE(INH) EMF_RCASE(FIBER)
#undef EMF_RCASE
    return;
  }
  constexpr int N = EMF_P + 1, EPB = Tile<EMF_P>::EPB;
  KArgs<EMF_T> b = a;
  b.e_begin = 0;
  const unsigned blocks = (unsigned)((a.nel + EPB - 1) / EPB);
  if (model == CNH) residual_kernel<EMF_T, EMF_P, CNH><<<blocks, EPB * N * N * N, 0, s>>>(b);
  if (model == INH) residual_kernel<EMF_T, EMF_P, INH><<<blocks, EPB * N * N * N, 0, s>>>(b);
  if (model == FIBER) residual_kernel<EMF_T, EMF_P, FIBER><<<blocks, EPB * N * N * N, 0, s>>>(b);
}

}  // namespace emfgpu
