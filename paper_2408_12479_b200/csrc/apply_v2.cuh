// Tangent-apply element phase, v2: persistent CTAs, EPB elements per CTA.
//
// Design (each point driven by an ncu profile, see DESIGN.md §3 and
// profiles/r01_*):
//  * persistent CTAs (one wave, occupancy-sized) take element groups from a
//    ticket counter and prefetch the NEXT group's x / u_k / affine geometry
//    into a second shared staging buffer with cp.async while the current
//    group computes; 10 barriers per group (the u_k forward pass runs through
//    swapped buffers, and a group has no closing barrier);
//  * sum factorization by pencil workers: a worker owns one (component, line)
//    pencil and performs the full 1D contraction in registers, so every
//    shared load feeds n FMAs and the 1D tables are compile-time-indexed
//    kernel parameters (constant-bank operands, no shared loads);
//  * padded element arrays (Lay below) chosen by measurement so the pencil
//    orientations and the per-point accesses avoid bank conflicts;
//  * Q3: the two elements of a CTA share one pencil index space (dense
//    mapping, CTA-wide barriers); EMF_V2_DENSE=0 builds the older variant
//    where each element synchronises on its own named barrier;
//  * element-local results are stored component-major, loc[(e*3 + c)*n^3 + m],
//    as contiguous vector stores, for the node phase (gather.cu).
// The quadrature-point algebra is in qp.cuh.
#pragma once
#include "eo_sweeps.cuh"
#include "kernels.cuh"

#ifndef EMF_TEN_EARLY
#define EMF_TEN_EARLY 1  // tensor: cached bundle loaded before the sweeps
#endif
#ifndef EMF_SPT_EARLY
#define EMF_SPT_EARLY 1
#endif
#ifndef EMF_SC_EARLY
#define EMF_SC_EARLY 1
#endif
#ifndef EMF_TEN_EARLY_F32
#define EMF_TEN_EARLY_F32 1
#endif
#ifndef EMF_CF_EARLY
#define EMF_CF_EARLY 1  // cachedF: G loaded before the sweeps
#endif
#ifndef EMF_MINB_F32Q3
#define EMF_MINB_F32Q3 0  // fp32 Q3 CTAs/SM override (experiments)
#endif
// fp64 Q4 tensor on the cached push-forward state (cfg2 element phase,
// profiles/r02_tensor_push_state.txt): 1.492 ms at 4 CTAs/SM with the late
// load, 1.353 with the 19 fields loaded before the sweeps, 1.305 with that at
// 5 CTAs/SM; fp32 keeps the late load (0.853 vs 0.865 ms)
#ifndef EMF_MINB_F32_FIBER_TENP
#define EMF_MINB_F32_FIBER_TENP 6
#endif
#ifndef EMF_MINB_FIBER_TENP
#define EMF_MINB_FIBER_TENP 4
#endif
#ifndef EMF_TENP_EARLY_Q4
#define EMF_TENP_EARLY_Q4 1
#endif
#ifndef EMF_MINB_Q4_TENP
#define EMF_MINB_Q4_TENP 5
#endif
#ifndef EMF_F32Q4_OCC
#define EMF_F32Q4_OCC 1  // the per-strategy fp32 Q4 CTAs/SM below
#endif
#ifndef EMF_MINB_F32Q12
#define EMF_MINB_F32Q12 0  // fp32 Q1 / Q2 CTAs/SM override (experiments)
#endif
#ifndef EMF_MINB_F32Q4
#define EMF_MINB_F32Q4 0  // fp32 Q4 CTAs/SM override (experiments)
#endif

// Q4: collocated even-odd sweeps (eo_sweeps.cuh) instead of the B/D sweeps
#ifndef EMF_COLL
#define EMF_COLL 1
#endif

namespace emfgpu {

// Per-element array layout: a + SY*b + SZ*c with padded strides chosen (by
// exhaustive search over small paddings) so that the three pencil
// orientations and the per-point accesses of a half-warp hit at most 2 banks
// per 8-byte word, while every pencil access stays base + compile-time offset.
// Q3: SZ = 20, SIZE = 80 (was 18 / 72), picked by a measured sweep over
// (SZ, SIZE) (tools/layout_sweep.sh): SZ = 4 mod 16 makes the y-pencils'
// 64-bit half-warp accesses conflict-free; cfg1 element phase fp64 none
// 0.1648 -> 0.1625 ms, fp64 scalar -3%, fp32 none 0.104 -> 0.096 ms.
template <int N, int ES = 8>  // ES: element size in bytes (array stride may differ)
struct Lay;
template <int ES>
struct Lay<2, ES> { static constexpr int N = 2, N2 = 4, N3 = 8, SY = 2, SZ = 4, SIZE = 8; };
template <int ES>
struct Lay<3, ES> { static constexpr int N = 3, N2 = 9, N3 = 27, SY = 3, SZ = 12, SIZE = 36; };
// fp64: SIZE = 82 (41 16-byte units, odd) with the j-c-k pencil order of the
// x-sweeps puts the two components of a quarter-warp's LDS.128 on disjoint
// bank groups; fp32 keeps 80 (float4 alignment of every pencil).
template <int ES>
struct Lay<4, ES> { static constexpr int N = 4, N2 = 16, N3 = 64, SY = 4, SZ = 20, SIZE = ES == 8 ? 82 : 80; };
template <int ES>
struct Lay<5, ES> { static constexpr int N = 5, N2 = 25, N3 = 125, SY = 5, SZ = 25, SIZE = 125; };
template <int N>
__device__ __forceinline__ constexpr int lat(int a, int b, int c) {
  return a + Lay<N>::SY * b + Lay<N>::SZ * c;
}

// Element coordinates and this thread's node for element e (< 2^31) with
// precomputed-multiplier divisions (no 64-bit division in the hot loop).
template <int P, typename A>
__device__ __forceinline__ ElemPos elem_pos_fast(int64_t e64, const A& a, int i, int j, int k) {
  const uint32_t e = (uint32_t)e64;
  const uint32_t ek = a.fd_nxy.div(e);
  const uint32_t r = e - ek * a.fd_nxy.d;
  const uint32_t ej = a.fd_nx.div(r);
  ElemPos p;
  p.e = e64;
  p.ei = (int)(r - ej * a.fd_nx.d);
  p.ej = (int)ej;
  p.ek = (int)ek;
  p.ga = p.ei * P + i;
  p.gb = p.ej * P + j;
  if (p.gb >= a.my) p.gb -= a.my;  // periodic y lattice
  p.gc = p.ek * P + k;
  p.node = ((int64_t)p.gc * a.my + p.gb) * a.mx + p.ga;
  return p;
}

// Elements per CTA and CTAs per SM (fp32; fp64 see minb_v2) by degree and
// element size in bytes.  EMF_Q4F_EPB=2 runs fp32 Q4 with 2 elements per CTA
// on the dense pencil mapping (measured 1-4% slower than 1 element per CTA).
#ifndef EMF_Q4F_EPB
#define EMF_Q4F_EPB 1
#endif
template <int P, int ES = 8>
struct TileV2;
template <int ES>
struct TileV2<1, ES> { static constexpr int EPB = 16, MINB = 4; };
template <int ES>
struct TileV2<2, ES> { static constexpr int EPB = 4, MINB = 4; };
template <int ES>
struct TileV2<3, ES> { static constexpr int EPB = 2, MINB = 4; };
template <>
struct TileV2<4, 8> { static constexpr int EPB = 1, MINB = 4; };
template <>
struct TileV2<4, 4> { static constexpr int EPB = EMF_Q4F_EPB, MINB = 4 / EMF_Q4F_EPB; };

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
template <typename T>
__device__ __forceinline__ void cp_async_T(T* smem, const T* gmem) {
  if constexpr (sizeof(T) == 8)
    cp_async8(smem, gmem);
  else
    cp_async4(smem, gmem);
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int K>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(K));
}

// ---- 1D tables ------------------------------------------------------------------
// B[q][a] (basis a at Gauss point q) and D[q][a] on the symmetric GLL nodes /
// Gauss points: B[n-1-q][n-1-a] = B[q][a] and D[n-1-q][n-1-a] = -D[q][a]
// (exact in exact arithmetic; the stored rows q > (n-1)/2 differ from their
// mirror by rounding only).  With EMF_SYMTAB the sweeps read only the
// unique half, so a sweep's distinct table operands drop from 2n^2 to
// ~n^2 (Q4: 50 -> 25 doubles); they then fit the uniform register file as
// DFMA operands instead of pinning ~50 general registers for the kernel's
// lifetime (Q4 fp64: 210+ registers -> see DESIGN).  D[c][c] of the centre
// point (odd n) is an exact zero and its FMAs are dropped.
#ifndef EMF_SYMTAB
#define EMF_SYMTAB 1
#endif
#ifndef EMF_SYMTAB_ALL
#define EMF_SYMTAB_ALL 0  // also Q1-Q3 (experiments)
#endif
template <int N>
__host__ __device__ constexpr bool symtab_on() { return EMF_SYMTAB && (N == 5 || EMF_SYMTAB_ALL); }
template <typename T, int N>
__device__ __forceinline__ T tB(const T* M, int q, int a) {
  if (symtab_on<N>()) {
    if (2 * q > N - 1) { q = N - 1 - q; a = N - 1 - a; }
    if (2 * q == N - 1 && 2 * a > N - 1) a = N - 1 - a;
  }
  return M[q * N + a];
}
template <typename T, int N>
__device__ __forceinline__ T tD(const T* M, int q, int a) {
  if (symtab_on<N>()) {
    bool neg = false;
    if (2 * q > N - 1) { q = N - 1 - q; a = N - 1 - a; neg = true; }
    if (2 * q == N - 1 && 2 * a > N - 1) { a = N - 1 - a; neg = !neg; }
    return neg ? -M[q * N + a] : M[q * N + a];
  }
  return M[q * N + a];
}
// s + D[q][a] u, skipping the structural zero D[c][c]
template <typename T, int N>
__device__ __forceinline__ T dacc(T s, const T* M, int q, int a, T u) {
  if (symtab_on<N>() && 2 * q == N - 1 && 2 * a == N - 1) return s;
  return s + tD<T, N>(M, q, a) * u;
}

// Array of gradient entry (component c, direction t) in a 9-array buffer:
// component-major 3c + t, or with TA direction-major 3t + c, which makes every
// sweep access's array index "c + constant", so one thread -> pencil map can
// be bank-conflict-free for all of a sweep's accesses (Q4 fp64, see q4_pen).
template <bool TA>
__host__ __device__ constexpr int garr(int c, int t) { return TA ? 3 * t + c : 3 * c + t; }
// array of gradient entry m = 3c + t (the per-point 3x3 index)
template <bool TA>
__host__ __device__ constexpr int garr_m(int m) { return garr<TA>(m / 3, m % 3); }

// Thread -> pencil maps of the Q4 fp64 single-element sweeps (125 threads,
// 75 pencils per orientation), found by tools/pencil_milp.py (solve_min,
// layout SY 5, SZ 25, SIZE 125): every half-warp's pencils hit distinct bank
// pairs for all accesses of the x and y sweeps, and 4 of the 5 half-warps of
// the z sweeps (the fifth is 2-way); the natural order had 2-way conflicts
// on most half-warps (profiles/r02_ncu_cfg2_*).  Entry = pencil index in the
// sweep's own decoding, packed x | y << 8 | z << 16; 255 = no pencil.
#ifndef EMF_Q4MAP
#define EMF_Q4MAP 1
#endif
#ifndef EMF_Q4MAP32
#define EMF_Q4MAP32 1
#endif
#ifndef EMF_Q4MAP_TENSOR
#define EMF_Q4MAP_TENSOR 0  // tensor measured slower with the maps (2.63 -> 2.85 ms, profiles/r02_cfg2_tenmap.txt)
#endif
struct Q4PenMap {
  unsigned char x[75], y[75], z[75];
};
static constexpr Q4PenMap kQ4Pen = {
    {7, 9, 15, 16, 17, 24, 42, 43, 46, 47, 49, 51, 52, 54, 60, 72, 11, 12, 19, 20, 21, 30, 32, 33, 39,
     44, 50, 53, 55, 56, 59, 70, 5, 6, 8, 13, 22, 25, 26, 29, 35, 38, 48, 58, 65, 66, 67, 69, 1, 4,
     10, 14, 18, 28, 31, 34, 37, 40, 41, 45, 57, 63, 68, 73, 0, 2, 3, 23, 27, 36, 61, 62, 64, 71, 74},
    {5, 7, 20, 31, 35, 37, 38, 42, 44, 47, 53, 58, 65, 68, 70, 72, 1, 6, 8, 15, 21, 27, 28, 30, 32,
     33, 39, 46, 56, 59, 61, 62, 11, 12, 13, 19, 22, 24, 25, 26, 29, 50, 51, 52, 64, 67, 69, 74, 0, 4,
     9, 10, 14, 16, 18, 23, 34, 40, 41, 43, 55, 57, 63, 73, 2, 3, 17, 36, 45, 48, 49, 54, 60, 66, 71},
    {0, 1, 7, 11, 13, 15, 16, 17, 38, 42, 46, 47, 48, 49, 52, 74, 6, 8, 9, 12, 14, 19, 20, 21, 23,
     27, 30, 39, 50, 53, 56, 73, 18, 24, 26, 29, 32, 33, 35, 41, 44, 55, 59, 62, 65, 66, 67, 68, 4, 5,
     10, 28, 31, 34, 36, 37, 40, 43, 51, 54, 57, 58, 63, 69, 2, 3, 22, 25, 45, 60, 61, 64, 70, 71, 72}};
struct Q4PenPacked {
  unsigned v[128];
};
constexpr Q4PenPacked q4pen_pack() {
  Q4PenPacked r{};
  for (int t = 0; t < 128; ++t)
    r.v[t] = t < 75 ? (unsigned)kQ4Pen.x[t] | (unsigned)kQ4Pen.y[t] << 8 | (unsigned)kQ4Pen.z[t] << 16 : 0xffffffu;
  return r;
}
static __constant__ Q4PenPacked c_q4pen = q4pen_pack();

// fp32 Q4 maps (4-byte words, 32 banks, whole-warp groups; tools/pencil_milp.py
// f32_q4_maps): the fused x / u_k forward sweeps (150 pencils, rounds over
// threads 0-124 then 0-24) and the transposed sweeps (75 pencils), arrays
// direction-major.  Costs: wavefronts per element-sweep access, ideal 5 / 3.
struct Q4PenMap32 {
  unsigned char fx[150], fy[150], fz[150], tx[75], ty[75], tz[75];
};
static constexpr Q4PenMap32 kQ4Pen32 = {
    // fwc_x (MILP cost 5)
    {8, 9, 16, 20, 37, 39, 45, 47, 54, 55, 56, 57, 58, 59, 62, 81, 83, 92, 95, 97, 98, 100, 106, 107, 110,
     114, 125, 128, 131, 134, 140, 149, 0, 1, 11, 13, 18, 19, 22, 27, 28, 29, 31, 38, 48, 67, 73, 76, 84, 85,
     87, 90, 94, 103, 113, 120, 121, 130, 132, 133, 136, 138, 142, 143, 6, 10, 17, 23, 32, 35, 36, 40, 41,
     43, 60, 65, 66, 69, 71, 78, 79, 80, 82, 88, 89, 91, 93, 108, 109, 116, 117, 118, 122, 126, 127, 147, 2,
     4, 14, 15, 21, 24, 26, 33, 42, 44, 49, 51, 52, 63, 75, 77, 86, 96, 99, 101, 102, 104, 105, 119, 123,
     124, 135, 144, 146, 3, 5, 7, 12, 25, 30, 34, 46, 50, 53, 61, 64, 68, 70, 72, 74, 111, 112, 115, 129,
     137, 139, 141, 145, 148},
    // fwc_y (MILP cost 5)
    {7, 8, 9, 16, 17, 23, 36, 42, 45, 47, 48, 55, 58, 68, 69, 71, 72, 74, 76, 78, 82, 87, 98, 101, 103, 107,
     109, 110, 128, 134, 137, 149, 0, 13, 18, 19, 31, 33, 39, 43, 51, 64, 65, 67, 73, 81, 85, 90, 91, 97, 99,
     100, 105, 112, 120, 122, 126, 130, 132, 136, 138, 140, 142, 146, 3, 4, 10, 14, 25, 26, 32, 34, 37, 40,
     41, 49, 52, 56, 57, 60, 61, 63, 66, 79, 106, 108, 111, 114, 116, 117, 118, 121, 127, 131, 143, 147, 2,
     5, 6, 15, 24, 29, 35, 38, 44, 53, 54, 75, 80, 83, 84, 86, 89, 92, 93, 94, 95, 102, 104, 115, 124, 125,
     135, 144, 145, 1, 11, 12, 20, 21, 22, 27, 28, 30, 46, 50, 59, 62, 70, 77, 88, 96, 113, 119, 123, 129,
     133, 139, 141, 148},
    // fwc_z (MILP cost 6)
    {0, 1, 4, 5, 7, 8, 33, 37, 39, 45, 47, 53, 54, 55, 57, 58, 59, 68, 71, 78, 87, 88, 90, 97, 109, 114, 118,
     119, 120, 122, 140, 149, 6, 14, 17, 18, 19, 21, 22, 31, 38, 41, 43, 44, 50, 51, 56, 64, 65, 67, 75, 76,
     80, 81, 91, 96, 100, 105, 113, 116, 117, 138, 139, 142, 26, 28, 30, 32, 34, 36, 40, 42, 61, 66, 69, 72,
     73, 74, 83, 85, 99, 106, 108, 121, 123, 127, 128, 129, 130, 131, 132, 133, 135, 137, 143, 147, 3, 11,
     13, 15, 16, 24, 27, 29, 35, 48, 52, 60, 77, 79, 82, 86, 89, 92, 93, 94, 98, 101, 102, 103, 112, 124,
     125, 126, 146, 2, 9, 10, 12, 20, 23, 25, 46, 49, 62, 63, 70, 84, 95, 104, 107, 110, 111, 115, 134, 136,
     141, 144, 145, 148},
    // tr_x (MILP cost 3)
    {1, 3, 4, 5, 12, 13, 14, 15, 22, 24, 26, 27, 28, 30, 32, 34, 38, 39, 40, 41, 42, 43, 48, 49, 50, 51, 52,
     53, 55, 57, 61, 63, 2, 6, 7, 11, 16, 17, 18, 19, 20, 21, 23, 25, 29, 31, 37, 44, 45, 46, 47, 54, 56, 58,
     59, 60, 62, 64, 65, 67, 68, 72, 73, 74, 0, 8, 9, 10, 33, 35, 36, 66, 69, 70, 71},
    // tr_y (MILP cost 4)
    {0, 4, 5, 8, 9, 10, 13, 14, 15, 17, 18, 19, 21, 28, 30, 39, 41, 44, 45, 46, 50, 51, 53, 55, 56, 59, 60,
     63, 64, 68, 70, 73, 1, 3, 6, 7, 11, 12, 16, 20, 22, 23, 25, 31, 32, 33, 35, 36, 37, 38, 40, 42, 43, 52,
     54, 57, 58, 61, 62, 65, 69, 71, 72, 74, 2, 24, 26, 27, 29, 34, 47, 48, 49, 66, 67},
    // tr_z (MILP cost 5)
    {5, 7, 13, 21, 22, 23, 24, 27, 28, 33, 36, 40, 42, 43, 44, 45, 46, 47, 51, 53, 54, 57, 58, 59, 60, 62,
     63, 65, 66, 67, 70, 73, 0, 2, 3, 4, 8, 9, 10, 12, 14, 15, 16, 17, 18, 19, 20, 25, 26, 29, 31, 34, 35,
     37, 38, 39, 41, 49, 50, 52, 55, 61, 68, 71, 1, 6, 11, 30, 32, 48, 56, 64, 69, 72, 74}};
struct Q4PenPacked32 {
  unsigned v[128][3];
};
// per thread: [0] = fwc x round 1 | x round 2 << 8 | y r1 << 16 | y r2 << 24,
// [1] = z r1 | z r2 << 8 | tr x << 16 | tr y << 24, [2] = tr z; 255 = none
constexpr Q4PenPacked32 q4pen32_pack() {
  Q4PenPacked32 r{};
  for (int t = 0; t < 128; ++t) {
    auto f = [&](const unsigned char* m, int round) -> unsigned {
      const int i = round == 0 ? t : 125 + t;
      return (round == 0 ? t < 125 : t < 25) ? (unsigned)m[i] : 255u;
    };
    auto g = [&](const unsigned char* m) -> unsigned { return t < 75 ? (unsigned)m[t] : 255u; };
    r.v[t][0] = f(kQ4Pen32.fx, 0) | f(kQ4Pen32.fx, 1) << 8 | f(kQ4Pen32.fy, 0) << 16 | f(kQ4Pen32.fy, 1) << 24;
    r.v[t][1] = f(kQ4Pen32.fz, 0) | f(kQ4Pen32.fz, 1) << 8 | g(kQ4Pen32.tx) << 16 | g(kQ4Pen32.ty) << 24;
    r.v[t][2] = g(kQ4Pen32.tz);
  }
  return r;
}
static __constant__ Q4PenPacked32 c_q4pen32 = q4pen32_pack();

// fp64 Q4 with the x and u_k forward sweeps fused (fwc_*: 150 pencils over
// the 6 staged arrays, round 1 on threads 0-124, round 2 on threads 0-24;
// tools/pencil_milp.py f64_q4_fused_maps): every half-warp conflict-free.
struct Q4PenMapF64 {
  unsigned char fx[150], fy[150], fz[150];
};
static constexpr Q4PenMapF64 kQ4PenF64 = {
    // fwc_x (MILP cost 10, ideal 10)
    {16, 31, 33, 37, 51, 58, 59, 70, 76, 77, 78, 84, 87, 89, 98, 120, 0, 7, 15, 68, 73, 75, 83, 88, 90, 101,
     109, 114, 118, 124, 126, 129, 8, 11, 26, 39, 49, 57, 60, 67, 69, 102, 116, 125, 128, 130, 142, 143, 9, 13,
     17, 23, 40, 42, 62, 66, 79, 80, 117, 123, 134, 140, 147, 148, 18, 29, 32, 38, 44, 46, 63, 71, 91, 97, 99,
     100, 106, 136, 137, 149, 12, 20, 35, 43, 47, 61, 86, 94, 103, 104, 113, 121, 122, 133, 144, 146, 5, 10,
     19, 22, 27, 30, 34, 48, 72, 92, 95, 105, 119, 132, 141, 145, 2, 25, 28, 52, 54, 65, 74, 85, 107, 110, 112,
     115, 127, 3, 6, 14, 21, 24, 36, 41, 50, 55, 64, 81, 93, 108, 111, 138, 139, 1, 4, 45, 53, 56, 82, 96, 131,
     135},
    // fwc_y (MILP cost 10, ideal 10)
    {0, 10, 16, 21, 26, 31, 43, 56, 63, 66, 76, 77, 83, 109, 130, 141, 11, 27, 37, 41, 50, 51, 52, 53, 68, 90,
     103, 108, 129, 134, 136, 138, 2, 5, 14, 15, 18, 28, 49, 61, 67, 71, 84, 91, 96, 114, 117, 120, 8, 9, 13,
     20, 22, 42, 45, 62, 79, 82, 113, 119, 143, 144, 147, 148, 7, 29, 32, 36, 38, 39, 44, 48, 58, 86, 105, 106,
     107, 111, 137, 149, 12, 54, 57, 72, 73, 85, 87, 88, 94, 97, 99, 104, 122, 126, 135, 139, 19, 23, 30, 33,
     34, 40, 47, 60, 70, 74, 81, 89, 92, 95, 116, 145, 65, 69, 75, 80, 98, 110, 112, 115, 123, 127, 128, 133,
     140, 3, 4, 17, 24, 35, 59, 64, 78, 93, 118, 121, 124, 125, 131, 142, 146, 1, 6, 25, 46, 55, 100, 101, 102,
     132},
    // fwc_z (MILP cost 10, ideal 10)
    {52, 60, 63, 67, 70, 74, 76, 77, 78, 83, 84, 85, 87, 101, 109, 130, 0, 4, 15, 31, 36, 50, 51, 65, 75, 90,
     97, 114, 117, 125, 136, 138, 8, 18, 21, 39, 42, 57, 71, 96, 102, 105, 119, 122, 128, 137, 140, 143, 11,
     13, 37, 40, 45, 46, 47, 49, 62, 82, 99, 100, 112, 134, 147, 148, 25, 29, 32, 35, 44, 95, 98, 106, 108,
     111, 115, 120, 126, 129, 146, 149, 3, 7, 12, 26, 28, 34, 43, 53, 61, 86, 94, 104, 113, 133, 135, 144, 10,
     19, 20, 23, 27, 30, 54, 68, 72, 79, 81, 89, 92, 93, 118, 141, 2, 6, 24, 55, 66, 73, 80, 88, 91, 110, 123,
     127, 145, 5, 14, 16, 17, 22, 38, 41, 48, 59, 107, 121, 124, 131, 132, 139, 142, 1, 9, 33, 56, 58, 64, 69,
     103, 116}};
struct Q4PenPackedF64 {
  unsigned v[128][2];
};
// [0] = x round 1 | x round 2 << 8 | y r1 << 16 | y r2 << 24, [1] = z r1 | z r2 << 8; 255 = none
constexpr Q4PenPackedF64 q4penf64_pack() {
  Q4PenPackedF64 r{};
  for (int t = 0; t < 128; ++t) {
    auto f = [&](const unsigned char* m, int round) -> unsigned {
      return (round == 0 ? t < 125 : t < 25) ? (unsigned)m[round == 0 ? t : 125 + t] : 255u;
    };
    r.v[t][0] = f(kQ4PenF64.fx, 0) | f(kQ4PenF64.fx, 1) << 8 | f(kQ4PenF64.fy, 0) << 16 | f(kQ4PenF64.fy, 1) << 24;
    r.v[t][1] = f(kQ4PenF64.fz, 0) | f(kQ4PenF64.fz, 1) << 8;
  }
  return r;
}
static __constant__ Q4PenPackedF64 c_q4penf64 = q4penf64_pack();

// The same maps with the pencil decoded at compile time: entry = array *
// SIZE + offset of the pencil's first point (pencil_decode, eo_sweeps.cuh),
// so the collocated Q4 sweeps take their addresses from one 16-bit table
// read instead of ~8 integer instructions per pencil task (the fp32 kernel
// is issue-bound at 6-7 CTAs/SM).  Columns: 0-5 the 150-pencil forward maps
// over x and u_k (x round 1, round 2, y, y, z, z), 6-8 the 75-pencil maps
// (x, y, z), 9 the x pencil's offset in the element-local results
// (c N^3 + (k N + j) N); kPenNone = no pencil.
constexpr unsigned short kPenNone = 0xffffu;
constexpr int q4_pen_off(int wk, int dir, bool jck, int na) {
  constexpr int N = 5, N2 = 25, SY = 5, SZ = 25, SIZE = 125;
  int vc = 0, off = 0;
  if (dir == 0) {
    int j = 0, k = 0;
    if (jck) {
      j = wk % N;
      vc = (wk / N) % na;
      k = wk / (na * N);
    } else {
      vc = wk / N2;
      const int r = wk % N2;
      j = r % N;
      k = r / N;
    }
    off = SY * j + SZ * k;
  } else {
    vc = wk / N2;
    const int r = wk % N2, i = r % N, t = r / N;
    off = dir == 1 ? i + SZ * t : i + SY * t;
  }
  return vc * SIZE + off;
}
struct Q4OffTab {
  unsigned short v[128][10];
};
template <typename FX, typename FY, typename FZ, typename TX, typename TY, typename TZ>
constexpr Q4OffTab q4off_build(const FX& fx, const FY& fy, const FZ& fz, const TX& tx, const TY& ty, const TZ& tz,
                               bool jck) {
  Q4OffTab r{};
  for (int t = 0; t < 128; ++t) {
    for (int c = 0; c < 10; ++c) r.v[t][c] = kPenNone;
    for (int round = 0; round < 2; ++round) {
      if (round == 0 ? t < 125 : t < 25) {
        const int i = round == 0 ? t : 125 + t;
        r.v[t][0 + round] = (unsigned short)q4_pen_off(fx[i], 0, false, 6);
        r.v[t][2 + round] = (unsigned short)q4_pen_off(fy[i], 1, false, 6);
        r.v[t][4 + round] = (unsigned short)q4_pen_off(fz[i], 2, false, 6);
      }
    }
    if (t < 75) {
      const int ox = q4_pen_off(tx[t], 0, jck, 3);
      r.v[t][6] = (unsigned short)ox;
      r.v[t][7] = (unsigned short)q4_pen_off(ty[t], 1, false, 3);
      r.v[t][8] = (unsigned short)q4_pen_off(tz[t], 2, false, 3);
      const int c = ox / 125, rem = ox % 125, k = rem / 25, j = (rem % 25) / 5;
      r.v[t][9] = (unsigned short)(c * 125 + (k * 5 + j) * 5);
    }
  }
  return r;
}
static __constant__ Q4OffTab c_q4off64 =
    q4off_build(kQ4PenF64.fx, kQ4PenF64.fy, kQ4PenF64.fz, kQ4Pen.x, kQ4Pen.y, kQ4Pen.z, true);
static __constant__ Q4OffTab c_q4off32 =
    q4off_build(kQ4Pen32.fx, kQ4Pen32.fy, kQ4Pen32.fz, kQ4Pen32.tx, kQ4Pen32.ty, kQ4Pen32.tz, false);
// Measured (cfg2 element phase, profiles/r02_q4_decoded_offsets.txt): with the
// rows in shared memory fp64 none 1.912 -> 1.903 ms, scalar 2.070 -> 1.996,
// but cachedF 1.590 -> 1.658 and fp32 none 1.215 -> 1.278 (shared memory is
// already at 65% of its wavefront peak); read straight from the constant
// bank the thread-indexed loads serialise (fp64 none 3.24 ms); packed into 5
// registers per thread (fp32 only, which has them to spare) fp32 none 1.213 ->
// 1.304 ms.  Off.
#ifndef EMF_Q4_PRE
#define EMF_Q4_PRE 0
#endif
#ifndef EMF_FUSED64
#define EMF_FUSED64 1  // fp64 Q4 on axis-aligned meshes: x and u_k forward sweeps fused on kQ4PenF64
#endif

// ---- pencil sweeps ------------------------------------------------------------
// Arguments are base pointers of consecutive per-element arrays of N3 values
// (array t at base + t*N3) with Lay<N>::at addressing.  `w` is the worker
// index inside the element (0 .. N3-1); a worker with w < 3*N2 owns
// (component c, line l).  M[row*N + col] are compile-time-indexed tables.

// Forward x-sweep: in[c] -> tB[c] = Bx in, tD[c] = Dx in.
// Dense pencil mapping (NE > 1): the NE elements of a CTA share one pencil
// index space, pencil wk of element wk / (3 N^2); SI / SO are the element
// strides of the input / output arrays.  The CTA's threads then run the
// NE * 3N^2 pencils back to back, so only the warps that own pencils issue
// sweep instructions (Q3: 3 of 4 warps instead of 4 half-used ones).
template <typename T, int N, int STRIDE = (3 * Lay<N>::N2 <= Lay<N>::N3 ? 3 * Lay<N>::N2 : Lay<N>::N3), int NE = 1,
          int SI = 0, int SO = 0>
__device__ __forceinline__ void fw_x(const T* in0, T* tb0, T* td0, const T* Bm, const T* Dm, int w) {
  using L = Lay<N, sizeof(T)>;
  for (int wp = w; wp < NE * 3 * L::N2; wp += STRIDE) {
    const int e_l = NE > 1 ? wp / (3 * L::N2) : 0;
    const int wk = wp - e_l * 3 * L::N2;
    const T* const in = in0 + e_l * SI;
    T* const tb = tb0 + e_l * SO;
    T* const td = td0 + e_l * SO;
    // fp64: pencil order j, c, k (j fastest) so a quarter-warp spans two
    // components (SIZE 82); fp32: component-major (measured better)
    const int j = sizeof(T) == 8 ? wk % N : (wk % L::N2) % N;
    const int c = sizeof(T) == 8 ? (wk / N) % 3 : wk / L::N2;
    const int k = sizeof(T) == 8 ? wk / (3 * N) : (wk % L::N2) / N;
    T u[N];
#pragma unroll
    for (int a = 0; a < N; ++a) u[a] = in[c * L::SIZE + lat<N>(a, j, k)];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      T sb = tB<T, N>(Bm, q, 0) * u[0], sd = tD<T, N>(Dm, q, 0) * u[0];
#pragma unroll
      for (int a = 1; a < N; ++a) {
        sb += tB<T, N>(Bm, q, a) * u[a];
        sd = dacc<T, N>(sd, Dm, q, a, u[a]);
      }
      tb[c * L::SIZE + lat<N>(q, j, k)] = sb;
      td[c * L::SIZE + lat<N>(q, j, k)] = sd;
    }
  }
}

// Forward y-sweep: sBB = By tB, sBD = Dy tB, sDB = By tD.
template <typename T, int N, int STRIDE = (3 * Lay<N>::N2 <= Lay<N>::N3 ? 3 * Lay<N>::N2 : Lay<N>::N3), int NE = 1,
          int SR = 0>
__device__ __forceinline__ void fw_y(const T* tb0, const T* td0, T* sbb0, T* sbd0, T* sdb0,
                                     const T* Bm, const T* Dm, int w) {
  using L = Lay<N, sizeof(T)>;
  for (int wp = w; wp < NE * 3 * L::N2; wp += STRIDE) {
    const int e_l = NE > 1 ? wp / (3 * L::N2) : 0;
    const int wk = wp - e_l * 3 * L::N2;
    const T* const tb = tb0 + e_l * SR;
    const T* const td = td0 + e_l * SR;
    T* const sbb = sbb0 + e_l * SR;
    T* const sbd = sbd0 + e_l * SR;
    T* const sdb = sdb0 + e_l * SR;
    const int c = wk / L::N2, r = wk % L::N2, i = r % N, k = r / N;
    T ub[N], ud[N];
#pragma unroll
    for (int b = 0; b < N; ++b) {
      ub[b] = tb[c * L::SIZE + lat<N>(i, b, k)];
      ud[b] = td[c * L::SIZE + lat<N>(i, b, k)];
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
      T s1 = tB<T, N>(Bm, q, 0) * ub[0], s2 = tD<T, N>(Dm, q, 0) * ub[0], s3 = tB<T, N>(Bm, q, 0) * ud[0];
#pragma unroll
      for (int b = 1; b < N; ++b) {
        s1 += tB<T, N>(Bm, q, b) * ub[b];
        s2 = dacc<T, N>(s2, Dm, q, b, ub[b]);
        s3 += tB<T, N>(Bm, q, b) * ud[b];
      }
      sbb[c * L::SIZE + lat<N>(i, q, k)] = s1;
      sbd[c * L::SIZE + lat<N>(i, q, k)] = s2;
      sdb[c * L::SIZE + lat<N>(i, q, k)] = s3;
    }
  }
}

// Forward z-sweep: g[c][0] = Bz sDB, g[c][1] = Bz sBD, g[c][2] = Dz sBB.
template <typename T, int N, int STRIDE = (3 * Lay<N>::N2 <= Lay<N>::N3 ? 3 * Lay<N>::N2 : Lay<N>::N3), int NE = 1,
          int SR = 0, bool TA = false>
__device__ __forceinline__ void fw_z(const T* sbb0, const T* sbd0, const T* sdb0, T* g0, const T* Bm,
                                     const T* Dm, int w) {
  using L = Lay<N, sizeof(T)>;
  for (int wp = w; wp < NE * 3 * L::N2; wp += STRIDE) {
    const int e_l = NE > 1 ? wp / (3 * L::N2) : 0;
    const int wk = wp - e_l * 3 * L::N2;
    const T* const sbb = sbb0 + e_l * SR;
    const T* const sbd = sbd0 + e_l * SR;
    const T* const sdb = sdb0 + e_l * SR;
    T* const g = g0 + e_l * SR;
    const int c = wk / L::N2, r = wk % L::N2, i = r % N, j = r / N;
    T u0[N], u1[N], u2[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      u0[k] = sdb[c * L::SIZE + lat<N>(i, j, k)];
      u1[k] = sbd[c * L::SIZE + lat<N>(i, j, k)];
      u2[k] = sbb[c * L::SIZE + lat<N>(i, j, k)];
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
      T g0 = tB<T, N>(Bm, q, 0) * u0[0], g1 = tB<T, N>(Bm, q, 0) * u1[0], g2 = tD<T, N>(Dm, q, 0) * u2[0];
#pragma unroll
      for (int k = 1; k < N; ++k) {
        g0 += tB<T, N>(Bm, q, k) * u0[k];
        g1 += tB<T, N>(Bm, q, k) * u1[k];
        g2 = dacc<T, N>(g2, Dm, q, k, u2[k]);
      }
      g[garr<TA>(c, 0) * L::SIZE + lat<N>(i, j, q)] = g0;
      g[garr<TA>(c, 1) * L::SIZE + lat<N>(i, j, q)] = g1;
      g[garr<TA>(c, 2) * L::SIZE + lat<N>(i, j, q)] = g2;
    }
  }
}

// Forward sweeps of NV staged vectors at once, in place.  Array (v, c) of a
// stage lives at base + (v*3 + c)*SIZE.  A pencil's positions belong to one
// worker in every stage, so outputs overwrite consumed inputs:
//   x: S -> S (B-sweep), T (D-sweep)
//   y: S, T -> S (BB), T (BD), U (DB)
//   z: U, T, S -> U (d/dx), T (d/dy), S (d/dz)
// With NV = 2 (x and u_k) 2*3N^2 pencils keep every lane busy for N = 4
// (96 pencils = 3 warp-rounds of 32, vs 4 half-empty rounds one vector at a time).
template <typename T, int N, int NV, int STRIDE, bool PAIR = false>
__device__ __forceinline__ void fwc_x(T* S, T* Tt, const T* Bm, const T* Dm, int w, int w1 = 0) {
  using L = Lay<N, sizeof(T)>;
  // PAIR: the thread's pencils are w and w1 (a thread -> pencil map) instead of w, w + STRIDE, ...
  for (int it = 0, wk = w; PAIR ? it < 2 : wk < NV * 3 * L::N2; ++it, wk = PAIR ? w1 : wk + STRIDE) {
    if (PAIR && wk >= NV * 3 * L::N2) continue;
    const int vc = wk / L::N2, r = wk % L::N2, j = r % N, k = r / N;
    T* const s = S + vc * L::SIZE;
    T* const t = Tt + vc * L::SIZE;
    T u[N];
#pragma unroll
    for (int a = 0; a < N; ++a) u[a] = s[lat<N>(a, j, k)];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      T sb = tB<T, N>(Bm, q, 0) * u[0], sd = tD<T, N>(Dm, q, 0) * u[0];
#pragma unroll
      for (int a = 1; a < N; ++a) {
        sb += tB<T, N>(Bm, q, a) * u[a];
        sd = dacc<T, N>(sd, Dm, q, a, u[a]);
      }
      s[lat<N>(q, j, k)] = sb;
      t[lat<N>(q, j, k)] = sd;
    }
  }
}
template <typename T, int N, int NV, int STRIDE, bool PAIR = false>
__device__ __forceinline__ void fwc_y(T* S, T* Tt, T* U, const T* Bm, const T* Dm, int w, int w1 = 0) {
  using L = Lay<N, sizeof(T)>;
  for (int it = 0, wk = w; PAIR ? it < 2 : wk < NV * 3 * L::N2; ++it, wk = PAIR ? w1 : wk + STRIDE) {
    if (PAIR && wk >= NV * 3 * L::N2) continue;
    const int vc = wk / L::N2, r = wk % L::N2, i = r % N, k = r / N;
    T* const s = S + vc * L::SIZE;
    T* const t = Tt + vc * L::SIZE;
    T* const u = U + vc * L::SIZE;
    T ub[N], ud[N];
#pragma unroll
    for (int b = 0; b < N; ++b) {
      ub[b] = s[lat<N>(i, b, k)];
      ud[b] = t[lat<N>(i, b, k)];
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
      T s1 = tB<T, N>(Bm, q, 0) * ub[0], s2 = tD<T, N>(Dm, q, 0) * ub[0], s3 = tB<T, N>(Bm, q, 0) * ud[0];
#pragma unroll
      for (int b = 1; b < N; ++b) {
        s1 += tB<T, N>(Bm, q, b) * ub[b];
        s2 = dacc<T, N>(s2, Dm, q, b, ub[b]);
        s3 += tB<T, N>(Bm, q, b) * ud[b];
      }
      s[lat<N>(i, q, k)] = s1;
      t[lat<N>(i, q, k)] = s2;
      u[lat<N>(i, q, k)] = s3;
    }
  }
}
template <typename T, int N, int NV, int STRIDE, bool PAIR = false>
__device__ __forceinline__ void fwc_z(T* S, T* Tt, T* U, const T* Bm, const T* Dm, int w, int w1 = 0) {
  using L = Lay<N, sizeof(T)>;
  for (int it = 0, wk = w; PAIR ? it < 2 : wk < NV * 3 * L::N2; ++it, wk = PAIR ? w1 : wk + STRIDE) {
    if (PAIR && wk >= NV * 3 * L::N2) continue;
    const int vc = wk / L::N2, r = wk % L::N2, i = r % N, j = r / N;
    T* const s = S + vc * L::SIZE;
    T* const t = Tt + vc * L::SIZE;
    T* const u = U + vc * L::SIZE;
    T u0[N], u1[N], u2[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      u0[k] = u[lat<N>(i, j, k)];
      u1[k] = t[lat<N>(i, j, k)];
      u2[k] = s[lat<N>(i, j, k)];
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
      T g0 = tB<T, N>(Bm, q, 0) * u0[0], g1 = tB<T, N>(Bm, q, 0) * u1[0], g2 = tD<T, N>(Dm, q, 0) * u2[0];
#pragma unroll
      for (int k = 1; k < N; ++k) {
        g0 += tB<T, N>(Bm, q, k) * u0[k];
        g1 += tB<T, N>(Bm, q, k) * u1[k];
        g2 = dacc<T, N>(g2, Dm, q, k, u2[k]);
      }
      u[lat<N>(i, j, q)] = g0;
      t[lat<N>(i, j, q)] = g1;
      s[lat<N>(i, j, q)] = g2;
    }
  }
}

// Transposed z-sweep (node index along z): A0 = Bz^T w0, A1 = Bz^T w1, A2 = Dz^T w2.
template <typename T, int N, int STRIDE = (3 * Lay<N>::N2 <= Lay<N>::N3 ? 3 * Lay<N>::N2 : Lay<N>::N3), int NE = 1,
          int SR = 0, bool TA = false>
__device__ __forceinline__ void tr_z(const T* wv0, T* av0, const T* Bm, const T* Dm, int w) {
  using L = Lay<N, sizeof(T)>;
  for (int wp = w; wp < NE * 3 * L::N2; wp += STRIDE) {
    const int e_l = NE > 1 ? wp / (3 * L::N2) : 0;
    const int wk = wp - e_l * 3 * L::N2;
    const T* const wv = wv0 + e_l * SR;
    T* const av = av0 + e_l * SR;
    const int c = wk / L::N2, r = wk % L::N2, i = r % N, j = r / N;
    T u0[N], u1[N], u2[N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      u0[q] = wv[garr<TA>(c, 0) * L::SIZE + lat<N>(i, j, q)];
      u1[q] = wv[garr<TA>(c, 1) * L::SIZE + lat<N>(i, j, q)];
      u2[q] = wv[garr<TA>(c, 2) * L::SIZE + lat<N>(i, j, q)];
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
      T a0 = tB<T, N>(Bm, 0, k) * u0[0], a1 = tB<T, N>(Bm, 0, k) * u1[0], a2 = tD<T, N>(Dm, 0, k) * u2[0];
#pragma unroll
      for (int q = 1; q < N; ++q) {
        a0 += tB<T, N>(Bm, q, k) * u0[q];
        a1 += tB<T, N>(Bm, q, k) * u1[q];
        a2 = dacc<T, N>(a2, Dm, q, k, u2[q]);
      }
      av[garr<TA>(c, 0) * L::SIZE + lat<N>(i, j, k)] = a0;
      av[garr<TA>(c, 1) * L::SIZE + lat<N>(i, j, k)] = a1;
      av[garr<TA>(c, 2) * L::SIZE + lat<N>(i, j, k)] = a2;
    }
  }
}

// Array of (Q0 | Q12, component c) in the transposed-sweep buffer.  fp64:
// the three components of one kind are adjacent arrays (stride SIZE = 41
// 16-byte units, odd), so the j-c-k x-pencils of a quarter-warp's LDS.128 in
// tr_x fall on distinct bank groups (measured 2-way conflicts with the
// (Q0, Q12) pair adjacent: component stride 82 units); fp32 keeps the pairs.
#ifndef EMF_QV_SPLIT
#define EMF_QV_SPLIT 1
#endif
template <typename T, bool TA = false>
__device__ __forceinline__ constexpr int qv_arr(int t, int c) {
  return ((sizeof(T) == 8 && EMF_QV_SPLIT) || TA) ? t * 3 + c : 2 * c + t;
}

// Transposed y-sweep: Q0 = By^T A0, Q12 = Dy^T A1 + By^T A2.
template <typename T, int N, int STRIDE = (3 * Lay<N>::N2 <= Lay<N>::N3 ? 3 * Lay<N>::N2 : Lay<N>::N3), int NE = 1,
          int SR = 0, bool TA = false>
__device__ __forceinline__ void tr_y(const T* av0, T* qv0, const T* Bm, const T* Dm, int w) {
  using L = Lay<N, sizeof(T)>;
  for (int wp = w; wp < NE * 3 * L::N2; wp += STRIDE) {
    const int e_l = NE > 1 ? wp / (3 * L::N2) : 0;
    const int wk = wp - e_l * 3 * L::N2;
    const T* const av = av0 + e_l * SR;
    T* const qv = qv0 + e_l * SR;
    const int c = wk / L::N2, r = wk % L::N2, i = r % N, k = r / N;
    T u0[N], u1[N], u2[N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      u0[q] = av[garr<TA>(c, 0) * L::SIZE + lat<N>(i, q, k)];
      u1[q] = av[garr<TA>(c, 1) * L::SIZE + lat<N>(i, q, k)];
      u2[q] = av[garr<TA>(c, 2) * L::SIZE + lat<N>(i, q, k)];
    }
#pragma unroll
    for (int b = 0; b < N; ++b) {
      T q0 = tB<T, N>(Bm, 0, b) * u0[0], q12 = tD<T, N>(Dm, 0, b) * u1[0] + tB<T, N>(Bm, 0, b) * u2[0];
#pragma unroll
      for (int q = 1; q < N; ++q) {
        q0 += tB<T, N>(Bm, q, b) * u0[q];
        q12 = dacc<T, N>(q12 + tB<T, N>(Bm, q, b) * u2[q], Dm, q, b, u1[q]);
      }
      qv[qv_arr<T, TA>(0, c) * L::SIZE + lat<N>(i, b, k)] = q0;
      qv[qv_arr<T, TA>(1, c) * L::SIZE + lat<N>(i, b, k)] = q12;
    }
  }
}

// Transposed x-sweep: out = Dx^T Q0 + Bx^T Q12, written as N contiguous
// values (one element row of one component) of the element-local results
// (loc_index, kernels.cuh); elements e0 + e_l.
template <typename T, int N, int STRIDE = (3 * Lay<N>::N2 <= Lay<N>::N3 ? 3 * Lay<N>::N2 : Lay<N>::N3), int NE = 1,
          int SR = 0, bool TA = false>
__device__ __forceinline__ void tr_x(const T* qv0, T* loc, int64_t e0, int nx, FastDiv fd_nx, const T* Bm,
                                     const T* Dm, int w, int nvalid = 1) {
  using L = Lay<N, sizeof(T)>;
  for (int wp = w; wp < NE * 3 * L::N2; wp += STRIDE) {
    const int e_l = NE > 1 ? wp / (3 * L::N2) : 0;
    const int wk = wp - e_l * 3 * L::N2;
    if (NE > 1 && e_l >= nvalid) break;
    const T* const qv = qv0 + e_l * SR;
    const int64_t e = e0 + e_l;
    const int j = sizeof(T) == 8 ? wk % N : (wk % L::N2) % N;  // pencil order as fw_x
    const int c = sizeof(T) == 8 ? (wk / N) % 3 : wk / L::N2;
    const int k = sizeof(T) == 8 ? wk / (3 * N) : (wk % L::N2) / N;
    T u0[N], u1[N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      u0[q] = qv[qv_arr<T, TA>(0, c) * L::SIZE + lat<N>(q, j, k)];
      u1[q] = qv[qv_arr<T, TA>(1, c) * L::SIZE + lat<N>(q, j, k)];
    }
    T o[N];
#pragma unroll
    for (int a = 0; a < N; ++a) {
      T s = tD<T, N>(Dm, 0, a) * u0[0] + tB<T, N>(Bm, 0, a) * u1[0];
#pragma unroll
      for (int q = 1; q < N; ++q) s = dacc<T, N>(s + tB<T, N>(Bm, q, a) * u1[q], Dm, q, a, u0[q]);
      o[a] = s;
    }
    T* dst;
    if constexpr (EMF_LOC_ROWS) {
      const int64_t row = fd_nx.div((uint32_t)e);
      dst = loc + loc_index<N>(row, (int)(e - row * nx), nx, k, j, 0, c);
    } else {
      dst = loc + (e * 3 + c) * L::N3 + (k * N + j) * N;
    }
#pragma unroll
    for (int a = 0; a < N; ++a) dst[a] = o[a];
  }
}

// ---- collocated even-odd sweeps (eo_sweeps.cuh) ---------------------------------
// Arrays: S = the staged vectors (NV*3 arrays: x [, u_k]), interpolated in
// place to the Gauss points; G = the gradients at the Gauss points, array
// (3 NV) t + vc for direction t and staged array vc, so every access of a
// sweep is "vc + constant" (the thread -> pencil maps stay conflict-free).
template <int NV>
__host__ __device__ constexpr int coll_gi(int t, int vc) { return 3 * NV * t + vc; }

// Interpolation along DIR, in place; WITHD (the last direction): also the
// collocated derivative along DIR of the interpolated pencil, into G.
template <typename T, int N, int NV, int DIR, bool JCK, bool WITHD, bool PRE = false>
__device__ __forceinline__ void coll_interp(T* S, T* G, const EoT<T>& t, int wk) {
  using L = Lay<N, sizeof(T)>;
  using E = EO<T, N>;
  if (PRE ? wk == (int)kPenNone : wk >= NV * 3 * L::N2) return;
  int po;  // array * SIZE + offset of the pencil's first point
  if (PRE) po = wk;
  else {
    int vc, off;
    pencil_decode<N, L::SY, L::SZ, DIR, JCK, 3 * NV>(wk, vc, off);
    po = vc * L::SIZE + off;
  }
  constexpr int ST = pencil_step<L::SY, L::SZ, DIR>();
  T* const p = S + po;
  T u[N], o[N], e[E::CH], d[E::H];
  pencil_load<T, N, ST>(p, u);
  E::split(u, e, d);
  E::B_split(t, e, d, o);
  pencil_store<T, N, ST>(p, o);
  if (WITHD) {
    E::split(o, e, d);
    E::D_split(t, e, d, u);
    pencil_store<T, N, ST>(G + coll_gi<NV>(DIR, 0) * L::SIZE + po, u);
  }
}
// Collocated derivative along DIR of the interpolated arrays: S -> G.
template <typename T, int N, int NV, int DIR, bool JCK, bool PRE = false>
__device__ __forceinline__ void coll_deriv(const T* S, T* G, const EoT<T>& t, int wk) {
  using L = Lay<N, sizeof(T)>;
  using E = EO<T, N>;
  if (PRE ? wk == (int)kPenNone : wk >= NV * 3 * L::N2) return;
  int po;
  if (PRE) po = wk;
  else {
    int vc, off;
    pencil_decode<N, L::SY, L::SZ, DIR, JCK, 3 * NV>(wk, vc, off);
    po = vc * L::SIZE + off;
  }
  constexpr int ST = pencil_step<L::SY, L::SZ, DIR>();
  T u[N], o[N], e[E::CH], d[E::H];
  pencil_load<T, N, ST>(S + po, u);
  E::split(u, e, d);
  E::D_split(t, e, d, o);
  pencil_store<T, N, ST>(G + coll_gi<NV>(DIR, 0) * L::SIZE + po, o);
}
// Transposed derivative along DIR of the integrand's column DIR (W = its
// three component arrays): A[c] = Dc^T W[c].
template <typename T, int N, int DIR, bool JCK, bool PRE = false>
__device__ __forceinline__ void coll_dT(const T* W, T* A, const EoT<T>& t, int wk) {
  using L = Lay<N, sizeof(T)>;
  using E = EO<T, N>;
  if (PRE ? wk == (int)kPenNone : wk >= 3 * L::N2) return;
  int po;
  if (PRE) po = wk;
  else {
    int c, off;
    pencil_decode<N, L::SY, L::SZ, DIR, JCK>(wk, c, off);
    po = c * L::SIZE + off;
  }
  constexpr int ST = pencil_step<L::SY, L::SZ, DIR>();
  T u[N], o[N], e[E::CH], d[E::H];
  pencil_load<T, N, ST>(W + po, u);
  E::split(u, e, d);
  E::Dt_split(t, e, d, o);
  pencil_store<T, N, ST>(A + po, o);
}
// z: Z[c] = Bz^T (A0[c] + A1[c] + Dc_z^T W2[c])
template <typename T, int N, bool PRE = false>
__device__ __forceinline__ void coll_trz(const T* W2, const T* A0, const T* A1, T* Z, const EoT<T>& t, int wk) {
  using L = Lay<N, sizeof(T)>;
  using E = EO<T, N>;
  if (PRE ? wk == (int)kPenNone : wk >= 3 * L::N2) return;
  int po;
  if (PRE) po = wk;
  else {
    int c, off;
    pencil_decode<N, L::SY, L::SZ, 2, false>(wk, c, off);
    po = c * L::SIZE + off;
  }
  constexpr int ST = L::SZ;
  T u[N], o[N], e[E::CH], d[E::H];
  pencil_load<T, N, ST>(W2 + po, u);
  E::split(u, e, d);
  E::Dt_split(t, e, d, o);
  T a0[N], a1[N];
  pencil_load<T, N, ST>(A0 + po, a0);
  pencil_load<T, N, ST>(A1 + po, a1);
#pragma unroll
  for (int t = 0; t < N; ++t) o[t] += a0[t] + a1[t];
  E::split(o, e, d);
  E::Bt_split(t, e, d, u);
  pencil_store<T, N, ST>(Z + po, u);
}
// y: in place
template <typename T, int N, bool PRE = false>
__device__ __forceinline__ void coll_try(T* Z, const EoT<T>& t, int wk) {
  using L = Lay<N, sizeof(T)>;
  using E = EO<T, N>;
  if (PRE ? wk == (int)kPenNone : wk >= 3 * L::N2) return;
  int po;
  if (PRE) po = wk;
  else {
    int c, off;
    pencil_decode<N, L::SY, L::SZ, 1, false>(wk, c, off);
    po = c * L::SIZE + off;
  }
  T* const p = Z + po;
  T u[N], o[N], e[E::CH], d[E::H];
  pencil_load<T, N, L::SY>(p, u);
  E::split(u, e, d);
  E::Bt_split(t, e, d, o);
  pencil_store<T, N, L::SY>(p, o);
}
// x: one element row of one component of the element-local results
// PRE: wk = the pencil's array * SIZE + offset, goff = its offset in the
// element's 3 N^3 block of the element-local results
template <typename T, int N, bool JCK, bool PRE = false>
__device__ __forceinline__ void coll_trx(const T* Z, T* loc, int64_t e_, int nx, FastDiv fd_nx, const EoT<T>& t, int wk,
                                         int goff = 0) {
  using L = Lay<N, sizeof(T)>;
  using E = EO<T, N>;
  if (PRE ? wk == (int)kPenNone : wk >= 3 * L::N2) return;
  if constexpr (PRE && !EMF_LOC_ROWS) {
    T u[N], o[N], e[E::CH], d[E::H];
    pencil_load<T, N, 1>(Z + wk, u);
    E::split(u, e, d);
    E::Bt_split(t, e, d, o);
    pencil_store<T, N, 1>(loc + e_ * 3 * L::N3 + goff, o);
    return;
  }
  int c, off;
  pencil_decode<N, L::SY, L::SZ, 0, JCK>(wk, c, off);
  T u[N], o[N], e[E::CH], d[E::H];
  pencil_load<T, N, 1>(Z + c * L::SIZE + off, u);
  E::split(u, e, d);
  E::Bt_split(t, e, d, o);
  const int k = off / L::SZ, j = (off - k * L::SZ) / L::SY;
  T* dst;
  if constexpr (EMF_LOC_ROWS) {
    const int64_t row = fd_nx.div((uint32_t)e_);
    dst = loc + loc_index<N>(row, (int)(e_ - row * nx), nx, k, j, 0, c);
  } else {
    dst = loc + (e_ * 3 + c) * L::N3 + (k * N + j) * N;
  }
  if constexpr (EMF_LOC_ROWS) {
#pragma unroll
    for (int a = 0; a < N; ++a) dst[a] = o[a];
  } else {
    pencil_store<T, N, 1>(dst, o);
  }
}
// Q4 (one element per CTA, mapped pencils) and Q3 (two elements per CTA on
// the dense pencil index space)
#ifndef EMF_COLL_Q3
#define EMF_COLL_Q3 1
#endif
#ifndef EMF_V2_DENSE
#define EMF_V2_DENSE 1
#endif
template <typename T, int P>
constexpr bool coll_v2() {
  return EMF_COLL && ((P == 4 && TileV2<P, sizeof(T)>::EPB == 1) ||
                      (EMF_COLL_Q3 && EMF_V2_DENSE && P == 3 && TileV2<P, sizeof(T)>::EPB == 2));
}

// ---- the kernel -------------------------------------------------------------------
#ifndef EMF_GX_SMEM
#define EMF_GX_SMEM 1
#endif
template <typename T, int P, int MODEL, int STRAT, bool CART>
struct ApplyV2Smem {
  static constexpr int N = P + 1, N3 = N * N * N, EPB = TileV2<P, sizeof(T)>::EPB;
  static constexpr bool kUk = (STRAT == S_NONE || STRAT == S_SCALAR || STRAT == S_SP_NONE || STRAT == S_SP_SCALAR);
  static constexpr int NST = kUk ? 6 : 3;  // staged fields: x (3) [+ u_k (3)]
  static constexpr int SZ = Lay<N, sizeof(T)>::SIZE;
  static constexpr bool kColl = coll_v2<T, P>();
  T stage[2][EPB][NST][SZ];
  T geo[2][EPB][10];
  T r1[kColl ? 1 : EPB][kColl ? 1 : 9][kColl ? 1 : SZ];
  T r2[kColl ? 1 : EPB][kColl ? 1 : 9][kColl ? 1 : SZ];
  // fp64 Q4 with u_k swept: the x gradient parks in its own arrays until the
  // integrand needs it, instead of 9 registers held across the u_k sweeps
  static constexpr bool kGx3 = !kColl && EMF_GX_SMEM && P == 4 && sizeof(T) == 8 && kUk && !(EMF_FUSED64 && CART);
  T r3[kGx3 ? EPB : 1][kGx3 ? 9 : 1][kGx3 ? SZ : 1];
  // collocated sweeps: gradients at the Gauss points, array coll_gi(t, vc);
  // without u_k three more arrays for the transposed y-derivative
  alignas(16) T g[kColl ? EPB : 1][kColl ? 3 * NST : 1][kColl ? SZ : 1];
  alignas(16) T xa[kColl && !kUk ? EPB : 1][kColl && !kUk ? 3 : 1][kColl && !kUk ? SZ : 1];
};

// CTAs per SM for the launch bounds.  fp64 keeps 3 CTAs/SM (<= 168 registers)
// except for the variants that ptxas fits into 128 registers without spills,
// which measured faster at 4 CTAs/SM (cfg1: headline fp64 none 0.1676 ->
// 0.1654 ms, spatial tensor 0.1205 -> 0.1148 ms); fp32 always 4.
#ifndef EMF_V2_PAIRSTAGE
#define EMF_V2_PAIRSTAGE 1
#endif
#ifndef EMF_V2_DENSE
#define EMF_V2_DENSE 1
#endif
#ifndef EMF_MINB_V2D_FORCE
#define EMF_MINB_V2D_FORCE 0
#endif
#ifndef EMF_MINB_Q4C
#define EMF_MINB_Q4C 4
#endif
#ifndef EMF_MINB_Q4_CART
#define EMF_MINB_Q4_CART 3
#endif
#ifndef EMF_MINB_Q4_FIBER
#define EMF_MINB_Q4_FIBER 2
#endif
#ifndef EMF_MINB_FIBER_V2D
#define EMF_MINB_FIBER_V2D 2
#endif
template <typename T, int P, int MODEL, int STRAT, bool CART>
constexpr int minb_v2() {
  if (sizeof(T) == 4) {
    if (P == 4 && EMF_MINB_F32Q4) return EMF_MINB_F32Q4;
    // fp32 Q4 on the collocated sweeps is bound by latency and barriers at 4
    // CTAs/SM (16 warps); more resident CTAs pay even with some spilling
    // (cfg2 element phase, profiles/r02_fp32_q4_occupancy.txt: none 1.363 ->
    // 1.211 ms at 6, cachedF 1.278 -> 1.033 at 6, tensor 1.402 -> 1.154 at 7,
    // scalar 1.364 -> 1.276 at 5)
    if (P == 4 && EMF_F32Q4_OCC && coll_v2<T, P>() && MODEL != FIBER) {
      if (STRAT == S_NONE || STRAT == S_CACHEDF || is_resid(STRAT)) return 6;
      if (STRAT == S_TENSOR) return 7;
      if (STRAT == S_SCALAR) return 5;
    }
    if (P == 3 && EMF_MINB_F32Q3) return EMF_MINB_F32Q3;
    if (P <= 2 && EMF_MINB_F32Q12) return EMF_MINB_F32Q12;
    // fibre tensor on the cached push-forward state (cfg3 fp32 element phase
    // 1.111 ms at 4 CTAs/SM, 1.083 at 5, 1.027 at 6)
    if (P == 3 && MODEL == FIBER && STRAT == S_TENSOR && tensor_compact(MODEL, 0)) return EMF_MINB_F32_FIBER_TENP;
    // 5 CTAs/SM measured faster for these cNH fp32 Q3 variants (tensor
    // 0.0912 -> 0.0871 ms, spatial none 0.1137 -> 0.1076), slower for fibre
    // tensor (0.1178 -> 0.1280) and no better elsewhere
    // collocated Q3 sweeps, cNH (profiles/r02_fp32_q3_occupancy.txt): cachedF
    // 0.0891 -> 0.0830 ms and tensor 0.0850 -> 0.0810 at 7 CTAs/SM, none /
    // scalar 0.0953 -> 0.0932 at 6; curved iNH loses beyond 5
    if (P == 3 && MODEL == CNH && coll_v2<T, P>()) {
      if (STRAT == S_TENSOR || STRAT == S_CACHEDF) return 7;
      if (STRAT == S_NONE || STRAT == S_SCALAR) return 6;
    }
    if (P == 3 && MODEL == CNH && (STRAT == S_TENSOR || STRAT == S_SP_NONE)) return 5;
    // collocated Q3 sweeps (fewer live values): none / scalar at 5 CTAs/SM
    // too (cNH axis-aligned none 0.0993 -> 0.0953 ms, scalar 0.0973 -> 0.0952,
    // curved iNH none 0.1035 -> 0.1014; cachedF slower, 0.0891 -> 0.0911)
    if (P == 3 && MODEL != FIBER && coll_v2<T, P>() && (STRAT == S_NONE || STRAT == S_SCALAR)) return 5;
    return TileV2<P, 4>::MINB;
  }
  if (EMF_MINB_V2D_FORCE) return EMF_MINB_V2D_FORCE;  // experiments (tools/build_variant.sh)
  if (P == 3 && MODEL == CNH && ((STRAT == S_NONE && CART) || STRAT == S_SP_NONE || STRAT == S_SP_TENSOR)) return 4;
  // re-measured after the ticket / dense-mapping / barrier work: cNH on
  // axis-aligned meshes fits 128 registers for these too (scalar 0.1649 ->
  // 0.1588 ms, tensor 0.1383 -> 0.1281, cachedF 0.1486 -> 0.1444)
  // tensor on the cached push-forward state: 0.1076 -> 0.1036 ms at 5
  if (P == 3 && MODEL == CNH && CART && STRAT == S_TENSOR && tensor_compact(MODEL, 0)) return 5;
  if (P == 3 && MODEL == CNH && CART && (STRAT == S_SCALAR || STRAT == S_TENSOR || STRAT == S_CACHEDF)) return 4;
  if (P == 3 && MODEL == INH && STRAT == S_SP_TENSOR) return 4;
  // collocated Q3 sweeps: curved iNH none 0.1506 -> 0.1465 ms, cachedF 0.1301 -> 0.1260
  // (tensor 0.1547 -> 0.2018 and the fibre model stay at 3 / 2)
  if (P == 3 && MODEL == INH && coll_v2<T, P>() && (STRAT == S_NONE || STRAT == S_CACHEDF)) return 4;
  // Q4 fp64: with the half 1D tables (symtab_on) the cNH / iNH variants fit
  // 128 registers (was 210-250: the 50 table doubles had been pinned in
  // general registers), so 4 CTAs/SM; the fibre model keeps 2 (spill-free at
  // up to 255 registers; 3 spilled 100-190 B)
  // fibre tensor on the cached push-forward state is as light as the iNH one
  // (curved Q3 0.1588 ms at 2 CTAs/SM, 0.1424 at 3, 0.1383 at 4; Q4 0.1628 -> 0.1301)
  if (P >= 3 && MODEL == FIBER && STRAT == S_TENSOR && tensor_compact(MODEL, 0)) return EMF_MINB_FIBER_TENP;
  if (P == 4 && MODEL == FIBER) return EMF_MINB_Q4_FIBER;
  if (P == 4 && STRAT == S_TENSOR && tensor_compact(MODEL, 0)) return EMF_MINB_Q4_TENP;
  if (P == 4 && !CART) return EMF_MINB_Q4C;
  if (P == 4 && CART) return EMF_MINB_Q4_CART;
  // fibre fp64 at Q3: 2 CTAs/SM, spill-free (32^3 curved none 0.278 -> 0.249 ms,
  // scalar 0.261 -> 0.232 ms); Q2 stays at 3 (0.128 vs 0.136 ms)
  if (MODEL == FIBER && P >= 3) return EMF_MINB_FIBER_V2D;
  return TileV2<P>::MINB > 3 ? 3 : TileV2<P>::MINB;
}

// Push-forward integrand (qp.cuh: push_state / push_integrand) for cNH / iNH
// with the linearization state computed or half-cached (none, scalar,
// cachedF); EMF_PUSH=0 builds the material-form algebra everywhere.
#ifndef EMF_PUSH
#define EMF_PUSH 1
#endif
template <typename T, int P, int MODEL, int STRAT>
constexpr bool push_form() {
  return EMF_PUSH && MODEL != FIBER && (STRAT == S_NONE || STRAT == S_SCALAR || STRAT == S_CACHEDF);
}

#ifndef EMF_V2_FRESH
#define EMF_V2_FRESH -1
#endif
// Re-derive the thread's point inside the loop bodies (EMF_V2_FRESH_POS)?
template <typename T, int P, int MODEL, int STRAT, bool CART>
constexpr bool fresh_pos_v2() {
  if (EMF_V2_FRESH >= 0) return EMF_V2_FRESH != 0;  // experiments (tools/build_variant.sh)
  // measured with tools/v2_sweep.sh (profiles/r01_e2e_findings.md): a win only
  // for these fp64 iNH variants (32^3 Q3 curved none 0.1956 -> 0.1854 ms,
  // scalar 0.2202 -> 0.1997; 24^3 Q4 curved tensor 0.1875 -> 0.1813), a loss
  // of 1-25% elsewhere (more recomputation, different load scheduling)
  // (re-measured at the end of the round: iNH none no longer gains, 0.1793 vs
  // 0.1772 ms without; scalar 0.1916 vs 0.1936 and Q4 tensor 0.1772 vs 0.1853 do)
  if (sizeof(T) == 8 && MODEL == INH && P == 3 && STRAT == S_SCALAR) return true;
  if (sizeof(T) == 8 && MODEL == INH && P == 4 && STRAT == S_TENSOR) return true;
  // collocated Q4 kernel, cfg2 fp64 scalar: 2.070 -> 2.016 ms (every other variant 1-9% slower)
  if (sizeof(T) == 8 && MODEL == INH && P == 4 && STRAT == S_SCALAR) return true;
  return false;
}

template <typename T, int P, int MODEL, int STRAT, bool CART>
__global__ void __launch_bounds__(TileV2<P, sizeof(T)>::EPB*(P + 1) * (P + 1) * (P + 1), (minb_v2<T, P, MODEL, STRAT, CART>()))
    apply_v2_kernel(const KArgs<T> a, int64_t ngroups) {
  using SM = ApplyV2Smem<T, P, MODEL, STRAT, CART>;
  // CART: affine elements with a diagonal J0^-1 (axis-aligned boxes): the
  // geometry factors reduce to 3 scalings per direction.
  const T* const Dfx = a.Dm;
  const T* const Dfy = a.Dm;
  const T* const Dfz = a.Dm;
  const T* const Btx = a.Bm;
  const T* const Dtx = a.Dm;
  const T* const Bty = a.Bm;
  const T* const Dty = a.Dm;
  const T* const Btz = a.Bm;
  const T* const Dtz = a.Dm;
  constexpr int N = P + 1, N3 = N * N * N, EPB = TileV2<P, sizeof(T)>::EPB;
  constexpr bool kUk = SM::kUk;
  constexpr int SZ = Lay<N, sizeof(T)>::SIZE;
  __shared__ __align__(16) SM sm;
  const EoT<T> eot{a.eoB, a.eoD, a.eoP};
  const int tid = threadIdx.x;
  const int el = tid / N3, q = tid % N3;
  constexpr bool kColl = SM::kColl;  // collocated even-odd sweeps (Q4)
  constexpr bool kMap = EMF_Q4MAP && P == 4 && sizeof(T) == 8 && !(EMF_V2_DENSE && EPB == 2) &&
                        !(SM::kUk && sizeof(T) == 4) && (EMF_Q4MAP_TENSOR || STRAT != S_TENSOR || kColl);
  constexpr int kStr = 3 * Lay<N>::N2 <= Lay<N>::N3 ? 3 * Lay<N>::N2 : Lay<N>::N3;
  const unsigned pen = kMap ? c_q4pen.v[tid] : 0u;
  // fp32 Q4 with u_k swept (fused forward sweeps): kQ4Pen32
  constexpr bool kMap32 = EMF_Q4MAP32 && P == 4 && sizeof(T) == 4 && SM::kUk && !(EMF_V2_DENSE && EPB == 2);
  constexpr bool kTA = kMap || kMap32;  // direction-major gradient arrays
  // collocated Q4 sweeps on mapped pencils: addresses from the decoded tables
  // (each thread keeps its own row in shared memory: a constant-bank read
  // indexed by the thread serialises 32 ways, and 5 more live registers spill)
  constexpr bool kPre = EMF_Q4_PRE && !EMF_LOC_ROWS && SM::kColl && P == 4 && (kMap || kMap32);
  __shared__ unsigned short s_pot[kPre ? 128 : 1][10];
  if constexpr (kPre) {
#pragma unroll
    for (int c = 0; c < 10; ++c) s_pot[tid][c] = sizeof(T) == 8 ? c_q4off64.v[tid][c] : c_q4off32.v[tid][c];
  }
  // fp64 Q4 fused forward sweeps: kQ4PenF64
  // measured: axis-aligned Q4 cNH none 0.132 -> 0.128 ms (24^3), curved cfg2
  // iNH none 2.21 -> 2.55 ms (both gradients and the early J0^-1 loads live
  // through the longer fused sweeps), so axis-aligned meshes only
  constexpr bool kFused64 = EMF_FUSED64 && kMap && SM::kUk && CART && !kColl;
  // the 150-pencil maps also serve the collocated sweeps over x and u_k
  constexpr bool kMapF64 = kFused64 || (kColl && kMap && SM::kUk);
  unsigned pen32[3] = {0u, 0u, 0u};
  if constexpr (kMapF64) {
    pen32[0] = c_q4penf64.v[tid][0];
    pen32[1] = c_q4penf64.v[tid][1];
  }
  if constexpr (kMap32) {
    pen32[0] = c_q4pen32.v[tid][0];
    pen32[1] = c_q4pen32.v[tid][1];
    pen32[2] = c_q4pen32.v[tid][2];
  }
  // Elements of a CTA only share data through their own slices, so when an
  // element spans whole warps it synchronises on its own named barrier.
  // Q3 (two 64-thread elements per CTA): dense pencil mapping over the CTA
  // (see fw_x) with CTA-wide barriers; measured against per-element named
  // barriers with 48 of 64 threads per element sweeping
  constexpr bool kDense = EMF_V2_DENSE && (N3 == 64 || N3 == 125) && EPB == 2;
  auto esync = [&]() {
    if constexpr (N3 % 32 == 0 && EPB > 1 && !kDense)
      asm volatile("bar.sync %0, %1;\n" ::"r"(el + 1), "n"(N3) : "memory");
    else
      __syncthreads();
  };

  // Work units handed out by a ticket counter (dynamic load balance; the
  // unit index is opaque to the compiler, which keeps it from building
  // strength-reduced address induction variables that spilled on Q4).  When
  // every element of the CTA synchronises on its own named barrier, each
  // element is its own worker with its own ticket stream; otherwise a unit is
  // a group of EPB elements.
  constexpr bool kPerElem = N3 % 32 == 0 && EPB > 1 && !kDense;
  constexpr bool kFreshPos = fresh_pos_v2<T, P, MODEL, STRAT, CART>();
  const int64_t nunits = kPerElem ? a.nel - a.e_begin : ngroups;
  // The thread's point (el, q, qi, qj, qk, qs) is re-derived from a fresh
  // %tid.x read inside the loop bodies instead of being kept live across the
  // loop: at 128 registers ptxas spilled these loop invariants and reloaded
  // them every iteration (long-scoreboard stalls on the reloads).
#define EMF_V2_FRESH_POS                                                       \
  int tid_f = tid;                                                            \
  if constexpr (kFreshPos) asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid_f)); \
  const int el = tid_f / N3, q = tid_f % N3;                                  \
  const int qi = q % N, qj = (q / N) % N, qk = q / (N * N);                   \
  const int qs = lat<N>(qi, qj, qk);                                          \
  (void)qs;
  auto elem_of = [&](int64_t u, int el_) -> int64_t { return (kPerElem ? u : u * EPB + el_) + a.e_begin; };
  // issue the cp.async copies of unit u into staging buffer b; returns true
  // when this thread's staged x value must be zeroed (Dirichlet node or
  // padding element), decided here where the lattice position is at hand
  // The node a thread stages (sel, si, sj, sk): its own point, or with the
  // dense Q3 mapping a row-paired one -- lanes 4m..4m+3 take a row of element
  // 0 and the next 4 lanes the same row of element 1 (its x neighbour when
  // nx is even), so a warp's 8-byte copies cover 4 lattice rows instead of 8
  // (the copies' shared-memory wavefronts follow the global lines touched).
  auto stage_pos = [&](int tid_, int& sel, int& si, int& sj, int& sk) {
    if constexpr (kDense && N3 == 64 && EMF_V2_PAIRSTAGE) {
      const int lane = tid_ & 31, row = (lane >> 3) + 4 * (tid_ >> 5);
      sel = (lane >> 2) & 1;
      si = lane & 3;
      sj = row & 3;
      sk = row >> 2;
    } else {
      sel = tid_ / N3;
      const int q_ = tid_ % N3;
      si = q_ % N;
      sj = (q_ / N) % N;
      sk = q_ / (N * N);
    }
  };
  auto prefetch = [&](int64_t u, int b) -> bool {
    EMF_V2_FRESH_POS
    int sel, si, sj, sk;
    stage_pos(tid_f, sel, si, sj, sk);
    const int sqs = lat<N>(si, sj, sk);
    const int64_t es = elem_of(u, sel);
    bool zero = true;
    // Q3: u_k comes from its per-element copy in the staging layout, as
    // contiguous 16-byte copies (a warp moves 512 contiguous bytes) instead
    // of 3 scattered 8-byte words per thread
    constexpr bool kUkEl = kUk && P == 3;
    const bool uk_el = kUkEl && a.uk_el != nullptr;
    if (es < a.nel) {
      const ElemPos ep = elem_pos_fast<P>(es, a, si, sj, sk);
      // the residual takes u with its Dirichlet values (no column masking)
      zero = !is_resid(STRAT) && node_constrained(ep.ga, ep.gb, ep.gc, a.mx, a.my, a.mz, a.faces);
#pragma unroll
      for (int c = 0; c < 3; ++c) cp_async_T(&sm.stage[b][sel][c][sqs], a.x + 3 * ep.node + c);
      if constexpr (kUk) {
        if (!uk_el) {
#pragma unroll
          for (int c = 0; c < 3; ++c) cp_async_T(&sm.stage[b][sel][3 + c][sqs], a.uk + 3 * ep.node + c);
        }
      }
    }
    if constexpr (kUkEl) {
      if (uk_el) {
        constexpr int CH = 3 * SZ * (int)sizeof(T) / 16;  // 16-byte chunks per element
        constexpr int NE = kPerElem ? 1 : EPB, NT = kPerElem ? N3 : EPB * N3;
        const int t0 = kPerElem ? q : tid_f;
        for (int ch = t0; ch < NE * CH; ch += NT) {
          const int ee = kPerElem ? el : ch / CH, cc = ch - (kPerElem ? 0 : ee) * CH;
          const int64_t e2 = elem_of(u, ee);
          if (e2 < a.nel)
            cp_async16(reinterpret_cast<char*>(&sm.stage[b][ee][3][0]) + 16 * cc,
                       reinterpret_cast<const char*>(a.uk_el + e2 * 3 * SZ) + 16 * cc);
        }
      }
    }
    const int64_t e = elem_of(u, el);
    if (e < a.nel) {
      if (a.affine && (!is_spatial(STRAT) || kUk))
        for (int f = q; f < 10; f += N3) cp_async_T(&sm.geo[b][el][f], a.geo + f * a.geo_stride + e);
    }
    cp_async_commit();
    return zero;
  };

  // unit u, staged in buffer buf (its cp.async group complete)
  auto compute = [&](int64_t u, int buf, bool zero_me) {
    EMF_V2_FRESH_POS
    // this thread's pencil per sweep orientation (kQ4Pen) or its point index
    // (kPre: the pencils' decoded offsets from c_q4off64 / c_q4off32 instead)
    const unsigned short* const pot = &s_pot[kPre ? tid_f : 0][0];
    const int wx = kPre ? (int)pot[6] : kMap ? (int)(pen & 255u) : kMap32 ? (int)((pen32[1] >> 16) & 255u) : q;
    const int wy = kPre ? (int)pot[7] : kMap ? (int)((pen >> 8) & 255u) : kMap32 ? (int)(pen32[1] >> 24) : q;
    const int wz = kPre ? (int)pot[8] : kMap ? (int)(pen >> 16) : kMap32 ? (int)pen32[2] : q;
    // tensor-product weight of this thread's point (operator.hpp:492)
    const T wq3 = T(a.qwd[qi] * a.qwd[qj] * a.qwd[qk]);
    const int64_t e = elem_of(u, el);
    const bool valid = e < a.nel;
    // Dirichlet columns are masked (operator.hpp:604-605); zero the stale
    // staging values of padding elements.
    if (zero_me) {
      int sel, si, sj, sk;
      stage_pos(tid_f, sel, si, sj, sk);
#pragma unroll
      for (int c = 0; c < 3; ++c) sm.stage[buf][sel][c][lat<N>(si, sj, sk)] = T(0);
    }
    // per-qp geometry / cache loads are issued before the sweeps
    const int64_t qidx = (valid ? e : a.e_begin) * N3 + q;
    const MatConst<T> mq = mat_at<T, MODEL>(a.mat, a.hq, a.hq_stride, qidx);
    // tensor with the cached push-forward state: K and the coefficients carry
    // the geometry, nothing else is read per point
    constexpr bool kTenPush = STRAT == S_TENSOR && tensor_compact(MODEL, 0);
    T j0inv[9], detw;
    if ((!is_spatial(STRAT) || kUk) && !CART && !a.affine && !kTenPush) {
#pragma unroll
      for (int m = 0; m < 9; ++m) j0inv[m] = a.geo[m * a.geo_stride + qidx];
      detw = a.geo[9 * a.geo_stride + qidx];
    }
    const T* cs = a.cache;
    const int64_t st = a.cache_stride;
    T sj[10];  // spatial: J_t (9) and 1/J, loaded before the sweeps
    if constexpr (is_spatial(STRAT)) {
#pragma unroll
      for (int m = 0; m < 9; ++m) sj[m] = cs[(C_JT + m) * st + qidx];
      sj[9] = cs[C_INVJ * st + qidx];
    }
    // cachedF fp64: G = F - I loaded before the sweeps, its latency hidden
    // behind them (cNH 0.1444 -> 0.1403 ms, curved iNH 0.2059 -> 0.1977;
    // fp32 measured 2% slower, keeps the late load)
    constexpr bool kCfEarly = STRAT == S_CACHEDF && EMF_CF_EARLY && sizeof(T) == 8;
    // tensor Q3: the cached bundle loaded before the sweeps, its latency
    // hidden behind them (fp64 cNH 0.1281 -> 0.1219 ms, curved iNH 0.1628 ->
    // 0.1567, fibre 0.2018 -> 0.1854; fp32 2-4%; Q4 iNH slower, 0.1772 -> 0.1874)
    constexpr bool kTenEarly = STRAT == S_TENSOR && EMF_TEN_EARLY &&
                               (P == 3 || (EMF_TENP_EARLY_Q4 && P == 4 && kTenPush && sizeof(T) == 8)) &&
                               (sizeof(T) == 8 || EMF_TEN_EARLY_F32);
    auto load_tensor_bundle = [&](Bundle<T>& b) {
      if (MODEL == CNH) b.lnj = cs[C_LNJ * st + qidx];
      else {
        b.jp = cs[C_JP * st + qidx];
        b.c1 = cs[C_C1 * st + qidx];
        b.c2 = cs[C_C2 * st + qidx];
      }
      if (MODEL == FIBER) {
        b.c3[0] = cs[(C_C3 + 0) * st + qidx];
        b.c3[1] = cs[(C_C3 + 1) * st + qidx];
        b.efib[0] = cs[(C_EF + 0) * st + qidx];
        b.efib[1] = cs[(C_EF + 1) * st + qidx];
      }
#pragma unroll
      for (int m = 0; m < 9; ++m) {
        b.F[m] = cs[(C_F + m) * st + qidx];
        b.Finv[m] = cs[(C_FINV + m) * st + qidx];
      }
#pragma unroll
      for (int m = 0; m < 6; ++m) {
        b.S[m] = cs[(C_S + m) * st + qidx];
        b.Cinv[m] = cs[(C_CINV + m) * st + qidx];
      }
    };
    Bundle<T> cbe;
    PushState<T> pse;
    if constexpr (kTenEarly && kTenPush) {
      load_push_state<T>(cs, st, qidx, pse);
      if constexpr (MODEL == FIBER) load_push_state_fibre<T>(cs, st, qidx, pse);
    }
    else if constexpr (kTenEarly) load_tensor_bundle(cbe);
    // spatial tensor: the cached spatial bundle loaded before the sweeps
    constexpr bool kSpTenEarly = STRAT == S_SP_TENSOR && EMF_SPT_EARLY;
    Bundle<T> cbst;
    SpCell<T> spst;
    if constexpr (kSpTenEarly) spatial_bundle<T, MODEL>(S_TENSOR, mq, nullptr, cs, st, qidx, cbst, spst);
    // scalar strategy: its 1-4 cached scalars loaded before the sweeps too
    // (fp64 Q4: the late load is faster, cfg2 scalar element phase 2.118 -> 2.073 ms)
    constexpr bool kScEarly = STRAT == S_SCALAR && EMF_SC_EARLY && !(P == 4 && sizeof(T) == 8);
    Bundle<T> cbs;
    if constexpr (kScEarly) load_scalars<T, MODEL>(cs, st, qidx, cbs);
    T gcf[9];
    if constexpr (kCfEarly) {
#pragma unroll
      for (int m = 0; m < 9; ++m) gcf[m] = cs[(C_G + m) * st + qidx];
    }
    esync();

    T* const R1 = &sm.r1[el][0][0];  // 9 arrays of SZ, contiguous
    T* const R2 = &sm.r2[el][0][0];
    T gx[9];
    T* const S = &sm.stage[buf][el][0][0];  // kUk: x (arrays 0-2), u_k (3-5)
    // forward sweeps of staged vector arrays [f0, f0+3): gradients into R2
    // swap: the u_k pass runs R1 -> R2 -> R1 so that its first stage can
    // start while the threads still read the x gradient from R2 (no barrier
    // between the two passes); its gradient then ends in R1
    auto fwd_sweeps = [&](int f0, bool swap) {
      if constexpr (kDense) {
        constexpr int SI = SM::NST * SZ, SR = 9 * SZ, TH = EPB * N3;
        T* const P1 = swap ? &sm.r2[0][0][0] : &sm.r1[0][0][0];
        T* const P2 = swap ? &sm.r1[0][0][0] : &sm.r2[0][0][0];
        fw_x<T, N, TH, EPB, SI, SR>(&sm.stage[buf][0][f0][0], P2, P2 + 3 * SZ, a.Bm, Dfx, tid);
        esync();
        fw_y<T, N, TH, EPB, SR>(P2, P2 + 3 * SZ, P1, P1 + 3 * SZ, P1 + 6 * SZ, a.Bm, Dfy, tid);
        esync();
        fw_z<T, N, TH, EPB, SR>(P1, P1 + 3 * SZ, P1 + 6 * SZ, P2, a.Bm, Dfz, tid);
        esync();
      } else {
        T* const P1 = swap ? R2 : R1;
        T* const P2 = swap ? R1 : R2;
        fw_x<T, N>(&sm.stage[buf][el][f0][0], P2, P2 + 3 * SZ, a.Bm, Dfx, wx);
        esync();
        fw_y<T, N>(P2, P2 + 3 * SZ, P1, P1 + 3 * SZ, P1 + 6 * SZ, a.Bm, Dfy, wy);
        esync();
        fw_z<T, N, kStr, 1, 0, kMap>(P1, P1 + 3 * SZ, P1 + 6 * SZ, P2, a.Bm, Dfz, wz);
        esync();
      }
    };
    // gradient of staged vector v at this thread's point after the in-place
    // sweeps: d/dx in R1, d/dy in R2, d/dz in the stage (read late: registers)
    auto grad_at = [&](int v, T* g) {
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        g[3 * c + 0] = R1[(3 * v + c) * SZ + qs];
        g[3 * c + 1] = R2[(3 * v + c) * SZ + qs];
        g[3 * c + 2] = S[(3 * v + c) * SZ + qs];
      }
    };
    // fp32: x and u_k swept together (full lanes); fp64 keeps one vector per
    // sweep, whose shorter live ranges fit its 128/168-register budget
    // (measured: fused sweeps cost fp64 none 0.165 -> 0.175 ms, gave fp32 -3%)
    constexpr bool kFused = kUk && (sizeof(T) == 4 || kFused64) && !kDense && !kColl;
    constexpr bool kJck = sizeof(T) == 8;  // pencil order of the 75-pencil x-sweeps (fw_x / tr_x)
    constexpr int NVc = kUk ? 2 : 1;
    T* const G = &sm.g[el][0][0];
    // dense pencil index space of the CTA's EPB elements (Q3): task wp of
    // NT per element belongs to element wp / NT
    constexpr int kGS = 3 * SM::NST * SZ, kSS = SM::NST * SZ;
    T* const S0 = &sm.stage[buf][0][0][0];
    T* const G0 = &sm.g[0][0][0];
    auto dense = [&](auto nt, auto&& f) {
      constexpr int NT = decltype(nt)::value;
#pragma unroll
      for (int w0 = 0; w0 < EPB * NT; w0 += EPB * N3) {
        const int wp = w0 + tid_f;
        if (wp < EPB * NT) {
          const int e_l = wp / NT;
          f(e_l, wp - e_l * NT);
        }
      }
    };
    constexpr bool kJckD = sizeof(T) == 8;
    if constexpr (kColl && kDense) {
      using NTf = std::integral_constant<int, NVc * 3 * N * N>;
      dense(NTf{}, [&](int e_l, int wk) {
        coll_interp<T, N, NVc, 0, kJckD, false>(S0 + e_l * kSS, G0 + e_l * kGS, eot, wk);
      });
      esync();
      dense(NTf{}, [&](int e_l, int wk) {
        coll_interp<T, N, NVc, 1, false, false>(S0 + e_l * kSS, G0 + e_l * kGS, eot, wk);
      });
      esync();
      dense(NTf{}, [&](int e_l, int wk) {
        coll_interp<T, N, NVc, 2, false, true>(S0 + e_l * kSS, G0 + e_l * kGS, eot, wk);
      });
      esync();
      dense(NTf{}, [&](int e_l, int wk) {
        coll_deriv<T, N, NVc, 0, kJckD>(S0 + e_l * kSS, G0 + e_l * kGS, eot, wk);
      });
      dense(NTf{}, [&](int e_l, int wk) {
        coll_deriv<T, N, NVc, 1, false>(S0 + e_l * kSS, G0 + e_l * kGS, eot, wk);
      });
      esync();
    } else if constexpr (kColl) {
      // ---- interpolate x [and u_k] to the Gauss points in place, then the
      // collocated derivatives (d/dz from the z pencils' registers)
      if constexpr (kUk) {
        constexpr bool kM = kMapF64 || kMap32;
        static_assert(!kPre || kM, "decoded offsets belong to the mapped pencils");
        const int fx0 = kPre ? (int)pot[0] : kM ? (int)(pen32[0] & 255u) : q;
        const int fx1 = kPre ? (int)pot[1] : kM ? (int)((pen32[0] >> 8) & 255u) : q + N3;
        const int fy0 = kPre ? (int)pot[2] : kM ? (int)((pen32[0] >> 16) & 255u) : q;
        const int fy1 = kPre ? (int)pot[3] : kM ? (int)(pen32[0] >> 24) : q + N3;
        const int fz0 = kPre ? (int)pot[4] : kM ? (int)(pen32[1] & 255u) : q;
        const int fz1 = kPre ? (int)pot[5] : kM ? (int)((pen32[1] >> 8) & 255u) : q + N3;
        coll_interp<T, N, 2, 0, false, false, kPre>(S, G, eot, fx0);
        coll_interp<T, N, 2, 0, false, false, kPre>(S, G, eot, fx1);
        esync();
        coll_interp<T, N, 2, 1, false, false, kPre>(S, G, eot, fy0);
        coll_interp<T, N, 2, 1, false, false, kPre>(S, G, eot, fy1);
        esync();
        coll_interp<T, N, 2, 2, false, true, kPre>(S, G, eot, fz0);
        coll_interp<T, N, 2, 2, false, true, kPre>(S, G, eot, fz1);
        esync();
        coll_deriv<T, N, 2, 0, false, kPre>(S, G, eot, fx0);
        coll_deriv<T, N, 2, 1, false, kPre>(S, G, eot, fy0);
        coll_deriv<T, N, 2, 0, false, kPre>(S, G, eot, fx1);
        // (running the 25 second-round y pencils on warp 1 beside warp 0's
        // second-round x pencils measured slower: 1.913 -> 1.947 ms)
        coll_deriv<T, N, 2, 1, false, kPre>(S, G, eot, fy1);
        esync();
      } else {
        coll_interp<T, N, 1, 0, kJck, false, kPre>(S, G, eot, wx);
        esync();
        coll_interp<T, N, 1, 1, false, false, kPre>(S, G, eot, wy);
        esync();
        coll_interp<T, N, 1, 2, false, true, kPre>(S, G, eot, wz);
        esync();
        coll_deriv<T, N, 1, 0, kJck, kPre>(S, G, eot, wx);
        coll_deriv<T, N, 1, 1, false, kPre>(S, G, eot, wy);
        esync();
      }
    } else if constexpr (kFused && (kMap32 || kFused64)) {
      // ---- both vectors per sweep, in place, on the thread's mapped pencil pair
      fwc_x<T, N, 2, N3, true>(S, R2, a.Bm, Dfx, (int)(pen32[0] & 255u), (int)((pen32[0] >> 8) & 255u));
      esync();
      fwc_y<T, N, 2, N3, true>(S, R2, R1, a.Bm, Dfy, (int)((pen32[0] >> 16) & 255u), (int)(pen32[0] >> 24));
      esync();
      fwc_z<T, N, 2, N3, true>(S, R2, R1, a.Bm, Dfz, (int)(pen32[1] & 255u), (int)((pen32[1] >> 8) & 255u));
      esync();
    } else if constexpr (kFused) {
      // ---- gradients of x and u_k at the qps, both vectors per sweep, in place
      fwc_x<T, N, 2, N3>(S, R2, a.Bm, Dfx, q);
      esync();
      fwc_y<T, N, 2, N3>(S, R2, R1, a.Bm, Dfy, q);
      esync();
      fwc_z<T, N, 2, N3>(S, R2, R1, a.Bm, Dfz, q);
      esync();
    } else {
      // ---- gradient of x at the qps
      if constexpr (SM::kGx3) {
        T* const R3 = &sm.r3[el][0][0];
        fw_x<T, N>(&sm.stage[buf][el][0][0], R2, R2 + 3 * SZ, a.Bm, Dfx, wx);
        esync();
        fw_y<T, N>(R2, R2 + 3 * SZ, R1, R1 + 3 * SZ, R1 + 6 * SZ, a.Bm, Dfy, wy);
        esync();
        fw_z<T, N, kStr, 1, 0, kMap>(R1, R1 + 3 * SZ, R1 + 6 * SZ, R3, a.Bm, Dfz, wz);
        esync();
      } else {
        fwd_sweeps(0, false);
#pragma unroll
        for (int m = 0; m < 9; ++m) gx[m] = R2[garr_m<kMap>(m) * SZ + qs];
      }
    }
    if (CART) {  // diagonal J0^-1 (entries 0, 4, 8)
      j0inv[0] = sm.geo[buf][el][0];
      j0inv[4] = sm.geo[buf][el][4];
      j0inv[8] = sm.geo[buf][el][8];
      detw = sm.geo[buf][el][9] * wq3;
    } else if (a.affine) {
#pragma unroll
      for (int m = 0; m < 9; ++m) j0inv[m] = sm.geo[buf][el][m];
      detw = sm.geo[buf][el][9] * wq3;
    }
    // push-forward form of the cNH / iNH integrand (qp.cuh, push_state)
    constexpr bool kPush = push_form<T, P, MODEL, STRAT>();
    PushState<T> ps;
    Bundle<T> cb;
    SpCell<T> sp;
    if constexpr (kSpTenEarly) {
      cb = cbst;
      sp = spst;
    }
    if constexpr (kUk) {
      T gk[9], gg[9];
      if constexpr (kColl) {
#pragma unroll
        for (int m = 0; m < 9; ++m) gk[m] = G[coll_gi<2>(m % 3, 3 + m / 3) * SZ + qs];
      } else if constexpr (kFused) {
        grad_at(1, gk);
      } else {
        if constexpr (SM::kGx3) {
          // R2 / R1 were last read before the barriers of the x pass
          fw_x<T, N>(&sm.stage[buf][el][3][0], R2, R2 + 3 * SZ, a.Bm, Dfx, wx);
          esync();
          fw_y<T, N>(R2, R2 + 3 * SZ, R1, R1 + 3 * SZ, R1 + 6 * SZ, a.Bm, Dfy, wy);
          esync();
          fw_z<T, N, kStr, 1, 0, kMap>(R1, R1 + 3 * SZ, R1 + 6 * SZ, R2, a.Bm, Dfz, wz);
          esync();
#pragma unroll
          for (int m = 0; m < 9; ++m) gk[m] = R2[garr_m<kMap>(m) * SZ + qs];
        } else {
          fwd_sweeps(3, true);
#pragma unroll
          for (int m = 0; m < 9; ++m) gk[m] = R1[garr_m<kMap>(m) * SZ + qs];
        }
      }
      if constexpr (CART) {
#pragma unroll
        for (int m = 0; m < 9; ++m) gg[m] = gk[m] * j0inv[4 * (m % 3)];
      } else {
        mm(gk, j0inv, gg);
      }
      if constexpr (kPush) {
        if constexpr (kScEarly) {
          if (!push_state<T, MODEL, STRAT == S_SCALAR, CART>(mq, gg, j0inv, detw, cbs, ps) && valid)
            atomicMin(a.err, (unsigned long long)qidx);
        } else {
          if (STRAT == S_SCALAR) load_scalars<T, MODEL>(cs, st, qidx, cb);
          if (!push_state<T, MODEL, STRAT == S_SCALAR, CART>(mq, gg, j0inv, detw, cb, ps) && valid)
            atomicMin(a.err, (unsigned long long)qidx);
        }
      } else if constexpr (is_spatial(STRAT)) {
        if (!spatial_bundle<T, MODEL>(STRAT - S_SP_NONE, mq, gg, cs, st, qidx, cb, sp) && valid)
          atomicMin(a.err, (unsigned long long)qidx);
      } else {
        if (!make_strain(gg, cb) && valid) atomicMin(a.err, (unsigned long long)qidx);
        if constexpr (STRAT == S_NONE) cache_scalars<T, MODEL>(mq, cb);
        else if constexpr (kScEarly) {
          cb.lnj = cbs.lnj;
          cb.jp = cbs.jp;
          cb.c1 = cbs.c1;
          cb.c2 = cbs.c2;
          cb.c3[0] = cbs.c3[0];
          cb.c3[1] = cbs.c3[1];
          cb.efib[0] = cbs.efib[0];
          cb.efib[1] = cbs.efib[1];
        } else
          load_scalars<T, MODEL>(cs, st, qidx, cb);
        second_pk<T, MODEL>(mq, cb);
      }
    } else if constexpr (STRAT == S_SP_TENSOR) {
      if constexpr (!kSpTenEarly) spatial_bundle<T, MODEL>(S_TENSOR, mq, nullptr, cs, st, qidx, cb, sp);
    } else if constexpr (STRAT == S_CACHEDF) {
      T gg[9];
#pragma unroll
      for (int m = 0; m < 9; ++m) gg[m] = kCfEarly ? gcf[m] : cs[(C_G + m) * st + qidx];
      if constexpr (kPush) {
        if (!push_state<T, MODEL, false, CART>(mq, gg, j0inv, detw, cb, ps) && valid)
          atomicMin(a.err, (unsigned long long)qidx);
      } else {
      if (!make_strain(gg, cb) && valid) atomicMin(a.err, (unsigned long long)qidx);
      cache_scalars<T, MODEL>(mq, cb);
      second_pk<T, MODEL>(mq, cb);
      }
    } else if constexpr (kTenPush) {
      if constexpr (kTenEarly) ps = pse;
      else {
        load_push_state<T>(cs, st, qidx, ps);
        if constexpr (MODEL == FIBER) load_push_state_fibre<T>(cs, st, qidx, ps);
      }
    } else if constexpr (STRAT == S_TENSOR) {
      if constexpr (kTenEarly) cb = cbe;
      else load_tensor_bundle(cb);
    }
    if constexpr (kFused) grad_at(0, gx);
    if constexpr (kColl) {
#pragma unroll
      for (int m = 0; m < 9; ++m) gx[m] = G[coll_gi<NVc>(m % 3, m / 3) * SZ + qs];
    }
    if constexpr (SM::kGx3) {
#pragma unroll
      for (int m = 0; m < 9; ++m) gx[m] = sm.r3[el][garr_m<kMap>(m)][qs];
    }
    T wv[9];
    if constexpr (is_resid(STRAT)) {
      if constexpr (CART) {  // the full J0^-1 from its diagonal
        j0inv[1] = j0inv[2] = j0inv[3] = j0inv[5] = j0inv[6] = j0inv[7] = T(0);
      }
      if (!resid_integrand<T, MODEL, STRAT == S_RESID_SP>(mq, gx, j0inv, detw, wq3, wv) && valid)
        atomicMin(a.err, (unsigned long long)qidx);
    } else if constexpr (kPush || kTenPush) {
      push_integrand<T, MODEL>(ps, gx, wv);
    } else if constexpr (is_spatial(STRAT)) {
      T jtinv[9];
      inverse3(sj, jtinv);
      const T ssc = (sj[9] * det3(sj)) * wq3;
      spatial_integrand<T, MODEL>(mq, cb, sp, gx, jtinv, ssc, wv);
    } else if constexpr (CART) {
      T dg[9], wm[9];
#pragma unroll
      for (int m = 0; m < 9; ++m) dg[m] = gx[m] * j0inv[4 * (m % 3)];
      tangent_wm<T, MODEL>(mq, cb, dg, wm);
      const T s0 = detw * j0inv[0], s1 = detw * j0inv[4], s2 = detw * j0inv[8];
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        wv[3 * c + 0] = wm[3 * c + 0] * s0;
        wv[3 * c + 1] = wm[3 * c + 1] * s1;
        wv[3 * c + 2] = wm[3 * c + 2] * s2;
      }
    } else
      tangent_integrand<T, MODEL>(mq, cb, gx, j0inv, detw, wv);
    // ---- test with the gradients of the basis functions
    if constexpr (kColl) {
      // the integrand takes the slots of the last staged vector's gradient
      // (each thread has read its own point's values)
      constexpr int v3 = 3 * (NVc - 1);
#pragma unroll
      for (int m = 0; m < 9; ++m) G[coll_gi<NVc>(m % 3, v3 + m / 3) * SZ + qs] = wv[m];
      esync();
      // A0 = Dc_x^T W0 and A1 = Dc_y^T W1 go to dead arrays: the interpolated
      // x (and u_k) in the stage; Z takes the slots of the x gradient's d/dx
      // (with u_k) or of W0 (without), both dead by the z-sweep.  The stage is
      // last read two barriers before the unit ends (the prefetch of the unit
      // after next refills it).
      if constexpr (kDense) {
        using NTb = std::integral_constant<int, 3 * N * N>;
        T* const X0 = &sm.xa[0][0][0];
        auto a1_of = [&](int e_l) { return kUk ? S0 + e_l * kSS + 3 * SZ : X0 + e_l * 3 * SZ; };
        dense(NTb{}, [&](int e_l, int wk) {
          coll_dT<T, N, 0, kJckD>(G0 + e_l * kGS + coll_gi<NVc>(0, v3) * SZ, S0 + e_l * kSS, eot, wk);
        });
        dense(NTb{}, [&](int e_l, int wk) {
          coll_dT<T, N, 1, false>(G0 + e_l * kGS + coll_gi<NVc>(1, v3) * SZ, a1_of(e_l), eot, wk);
        });
        esync();
        dense(NTb{}, [&](int e_l, int wk) {
          coll_trz<T, N>(G0 + e_l * kGS + coll_gi<NVc>(2, v3) * SZ, S0 + e_l * kSS, a1_of(e_l), G0 + e_l * kGS, eot,
                         wk);
        });
        esync();
        dense(NTb{}, [&](int e_l, int wk) { coll_try<T, N>(G0 + e_l * kGS, eot, wk); });
        esync();
        const int64_t e0 = e - el;
        dense(NTb{}, [&](int e_l, int wk) {
          if (e0 + e_l < a.nel) coll_trx<T, N, kJckD>(G0 + e_l * kGS, a.loc, e0 + e_l, a.nx, a.fd_nx, eot, wk);
        });
        return;
      }
      T* const A0 = S;
      T* const A1 = kUk ? S + 3 * SZ : &sm.xa[el][0][0];
      T* const Z = G;
      coll_dT<T, N, 0, kJck, kPre>(G + coll_gi<NVc>(0, v3) * SZ, A0, eot, wx);
      coll_dT<T, N, 1, false, kPre>(G + coll_gi<NVc>(1, v3) * SZ, A1, eot, wy);
      esync();
      coll_trz<T, N, kPre>(G + coll_gi<NVc>(2, v3) * SZ, A0, A1, Z, eot, wz);
      esync();
      coll_try<T, N, kPre>(Z, eot, wy);
      esync();
      if (valid) coll_trx<T, N, kJck, kPre>(Z, a.loc, e, a.nx, a.fd_nx, eot, wx, kPre ? (int)pot[9] : 0);
      return;
    }
#pragma unroll
    for (int m = 0; m < 9; ++m) R1[garr_m<kTA>(m) * SZ + qs] = wv[m];
    esync();
    if constexpr (kDense) {
      constexpr int SR = 9 * SZ, TH = EPB * N3;
      T* const R1a = &sm.r1[0][0][0];
      T* const R2a = &sm.r2[0][0][0];
      tr_z<T, N, TH, EPB, SR>(R1a, R2a, Btz, Dtz, tid);
      esync();
      tr_y<T, N, TH, EPB, SR>(R2a, R1a, Bty, Dty, tid);
      esync();
      const int64_t e0 = e - el;
      tr_x<T, N, TH, EPB, SR>(R1a, a.loc, e0, a.nx, a.fd_nx, Btx, Dtx, tid,
                              (int)(a.nel - e0 < EPB ? a.nel - e0 : EPB));
    } else {
      tr_z<T, N, kStr, 1, 0, kTA>(R1, R2, Btz, Dtz, wz);
      esync();
      tr_y<T, N, kStr, 1, 0, kTA>(R2, R1, Bty, Dty, wy);
      esync();
      if (valid) tr_x<T, N, kStr, 1, 0, kTA>(R1, a.loc, e, a.nx, a.fd_nx, Btx, Dtx, wx);
    }
    // No closing barrier: before the next unit's first barrier a thread only
    // zeroes its own staged words of the other buffer and issues the next
    // prefetch into this unit's buffer, whose last readers (the x-sweeps, or
    // the fp32 d/dz read) are behind several barriers already; r1/r2 are
    // first written after that barrier.
  };

  // The first two units of a worker are static (no atomic round trip before
  // the first element); later tickets come from a.tk[0], taken one unit ahead
  // of need by the worker's leader (its value used one unit later, so the
  // atomic's round trip is never waited on) and published through shared
  // memory, read after the barriers of the next compute.
  // Let a programmatically dependent node phase launch now: its CTAs take
  // the SM slots this persistent grid frees at its end and wait there
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  __shared__ int s_tk[EPB][2];
  const int nw = (int)gridDim.x * (kPerElem ? EPB : 1);
  const int wid = kPerElem ? (int)blockIdx.x * EPB + el : (int)blockIdx.x;
  const bool leader = kPerElem ? q == 0 : tid == 0;
  const int slot = kPerElem ? el : 0;
  const int nu = (int)nunits;
  int cur = wid, nxt = wid + nw;
  unsigned praw = 0;  // raw ticket of the unit after nxt, used one iteration later
  int buf = 0, par = 0;
  bool zero_cur = true, zero_next = true;
  if (cur < nu) zero_cur = prefetch(cur, 0);
  if (leader && nxt < nu) praw = atomicAdd(a.tk, 1u);
  while (cur < nu) {
    if (nxt < nu)
      zero_next = prefetch(nxt, buf ^ 1);
    else
      cp_async_commit();
    if (leader) {
      const int pt = nxt < nu ? 2 * nw + (int)praw : nu;
      s_tk[slot][par] = pt;
      if (pt < nu) praw = atomicAdd(a.tk, 1u);
    }
    cp_async_wait<1>();
    compute(cur, buf, zero_cur);  // the published ticket is read after its barriers
    const int nn = s_tk[slot][par];
    par ^= 1;
    cur = nxt;
    nxt = nn;
    buf ^= 1;
    zero_cur = zero_next;
  }
  cp_async_wait<0>();
  // the last worker out rewinds the counter for the next launch on this slot
  if (leader) {
    if (atomicAdd(a.tk + 1, 1u) == (unsigned)(nw - 1)) {
      a.tk[0] = 0;
      a.tk[1] = 0;
    }
  }
}

}  // namespace emfgpu
