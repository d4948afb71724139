// Collocated even-odd 1D contractions for the element kernels.
//
// The reference evaluates the reference-cell gradient at the Gauss points as
// (D (x) B (x) B, B (x) D (x) B, B (x) B (x) D) u (sumfact.hpp:67-85) and tests
// with the transposes (sumfact.hpp:90-110).  With n_q = p + 1 Gauss points the
// nodal derivative factors exactly through the interpolation: D = Dc B, where
// Dc[q][r] = l_r'(g_q) differentiates the Lagrange basis on the Gauss points
// themselves.  The gradient then is three interpolation sweeps (B along x, y,
// z) followed by three collocated derivative sweeps (Dc along x, y, z, all
// reading the same interpolated array), and the test is the transposed
// sequence: 6 one-array sweeps per vector instead of 3 sweeps over 2-3 arrays.
//
// On top of that the symmetric point sets give B[n-1-q][n-1-a] = B[q][a] and
// Dc[n-1-q][n-1-r] = -Dc[q][r], so each 1D contraction splits into an even
// and an odd half (sums and differences of mirrored entries): for n = 5,
// 21 (B) / 20 (Dc) instructions instead of 25.
//
// Tables (KArgs::eoB / eoD, filled by make_args in capi.cu), H = n/2,
// CH = (n+1)/2, c = H the centre index for odd n:
//   BE[q][a] = (B[q][a] + B[q][n-1-a]) / 2   q < CH, a < H;  BE[q][c] = B[q][c]
//   BO[q][a] = (B[q][a] - B[q][n-1-a]) / 2   q < H,  a < H
//   DE[q][a] = (Dc[q][a] + Dc[q][n-1-a]) / 2 q < H,  a < H;  DE[q][c] = Dc[q][c]
//   DO[q][a] = (Dc[q][a] - Dc[q][n-1-a]) / 2 q < CH, a < H
// All table indices are compile-time constants after unrolling, so the
// entries are constant-bank operands of the FMAs.
#pragma once

namespace emfgpu {

template <typename T, int N>
struct EO {
  static constexpr int H = N / 2, CH = (N + 1) / 2;
  static constexpr bool ODD = (N & 1) != 0;
  static constexpr int NB = CH * CH + H * H;  // entries of eoB
  static constexpr int ND = H * CH + CH * H;  // entries of eoD
  static __device__ __forceinline__ T be(const T* t, int q, int a) { return t[q * CH + a]; }
  static __device__ __forceinline__ T bo(const T* t, int q, int a) { return t[CH * CH + q * H + a]; }
  static __device__ __forceinline__ T de(const T* t, int q, int a) { return t[q * CH + a]; }
  static __device__ __forceinline__ T dd(const T* t, int q, int a) { return t[H * CH + q * H + a]; }

  // mirrored sums / differences of u; e[c] = u[c]
  static __device__ __forceinline__ void split(const T (&u)[N], T (&e)[CH], T (&d)[H ? H : 1]) {
#pragma unroll
    for (int a = 0; a < H; ++a) {
      e[a] = u[a] + u[N - 1 - a];
      d[a] = u[a] - u[N - 1 - a];
    }
    if (ODD) e[H] = u[H];
  }

  // o[q] = sum_a B[q][a] u[a] from the split halves
  static __device__ __forceinline__ void B_split(const T* tb, const T (&e)[CH], const T (&d)[H ? H : 1], T (&o)[N]) {
#pragma unroll
    for (int q = 0; q < H; ++q) {
      T se = be(tb, q, 0) * e[0], so = bo(tb, q, 0) * d[0];
#pragma unroll
      for (int a = 1; a < CH; ++a) se += be(tb, q, a) * e[a];
#pragma unroll
      for (int a = 1; a < H; ++a) so += bo(tb, q, a) * d[a];
      o[q] = se + so;
      o[N - 1 - q] = se - so;
    }
    if (ODD) {
      T s = be(tb, H, 0) * e[0];
#pragma unroll
      for (int a = 1; a < CH; ++a) s += be(tb, H, a) * e[a];
      o[H] = s;
    }
  }
  // o[q] = sum_r Dc[q][r] u[r] from the split halves
  static __device__ __forceinline__ void D_split(const T* td, const T (&e)[CH], const T (&d)[H ? H : 1], T (&o)[N]) {
#pragma unroll
    for (int q = 0; q < H; ++q) {
      T te = de(td, q, 0) * e[0], to = dd(td, q, 0) * d[0];
#pragma unroll
      for (int a = 1; a < CH; ++a) te += de(td, q, a) * e[a];
#pragma unroll
      for (int a = 1; a < H; ++a) to += dd(td, q, a) * d[a];
      o[q] = to + te;
      o[N - 1 - q] = to - te;
    }
    if (ODD) {
      T s = dd(td, H, 0) * d[0];
#pragma unroll
      for (int a = 1; a < H; ++a) s += dd(td, H, a) * d[a];
      o[H] = s;
    }
  }
  // o[a] = sum_q B[q][a] w[q] from the split halves of w
  static __device__ __forceinline__ void Bt_split(const T* tb, const T (&e)[CH], const T (&d)[H ? H : 1], T (&o)[N]) {
#pragma unroll
    for (int a = 0; a < H; ++a) {
      T se = be(tb, 0, a) * e[0], so = bo(tb, 0, a) * d[0];
#pragma unroll
      for (int q = 1; q < CH; ++q) se += be(tb, q, a) * e[q];
#pragma unroll
      for (int q = 1; q < H; ++q) so += bo(tb, q, a) * d[q];
      o[a] = se + so;
      o[N - 1 - a] = se - so;
    }
    if (ODD) {
      T s = be(tb, 0, H) * e[0];
#pragma unroll
      for (int q = 1; q < CH; ++q) s += be(tb, q, H) * e[q];
      o[H] = s;
    }
  }
  // o[r] = sum_q Dc[q][r] w[q] from the split halves of w
  static __device__ __forceinline__ void Dt_split(const T* td, const T (&e)[CH], const T (&d)[H ? H : 1], T (&o)[N]) {
#pragma unroll
    for (int r = 0; r < H; ++r) {
      T s1 = dd(td, 0, r) * e[0], s2 = de(td, 0, r) * d[0];
#pragma unroll
      for (int q = 1; q < CH; ++q) s1 += dd(td, q, r) * e[q];
#pragma unroll
      for (int q = 1; q < H; ++q) s2 += de(td, q, r) * d[q];
      o[r] = s2 + s1;
      o[N - 1 - r] = s2 - s1;
    }
    if (ODD) {
      T s = de(td, 0, H) * d[0];
#pragma unroll
      for (int q = 1; q < H; ++q) s += de(td, q, H) * d[q];
      o[H] = s;
    }
  }
};

// Pencil wk of a sweep along DIR: array index vc (component, or vector * 3 +
// component) and the offset of the pencil's first point inside the array.
// The decodings are those of fw_x / fw_y / fw_z (apply_v2.cuh), which the
// thread -> pencil maps (kQ4Pen*, tools/pencil_milp.py) were built for; JCK
// is the j-c-k order of the fp64 x-sweeps (j fastest, then the NA arrays).
template <int N, int SY, int SZ, int DIR, bool JCK, int NA = 3>
__device__ __forceinline__ void pencil_decode(int wk, int& vc, int& off) {
  constexpr int N2 = N * N;
  if (DIR == 0) {
    int j, k;
    if (JCK) {
      j = wk % N;
      vc = (wk / N) % NA;
      k = wk / (NA * N);
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
    off = DIR == 1 ? i + SZ * t : i + SY * t;
  }
}
template <int SY, int SZ, int DIR>
__host__ __device__ constexpr int pencil_step() { return DIR == 0 ? 1 : DIR == 1 ? SY : SZ; }

// Q3 x-pencils (4 contiguous values, 16-byte aligned in Lay<4>) move as
// 16-byte words: the j-c-k order then keeps a quarter-warp conflict-free.
template <typename T, int N, int ST>
__device__ __forceinline__ void pencil_load(const T* p, T (&u)[N]) {
  if constexpr (N == 4 && ST == 1 && sizeof(T) == 8) {
    const double2 a = *reinterpret_cast<const double2*>(p), b = *reinterpret_cast<const double2*>(p + 2);
    u[0] = a.x, u[1] = a.y, u[2] = b.x, u[3] = b.y;
  } else if constexpr (N == 4 && ST == 1 && sizeof(T) == 4) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    u[0] = a.x, u[1] = a.y, u[2] = a.z, u[3] = a.w;
  } else {
#pragma unroll
    for (int t = 0; t < N; ++t) u[t] = p[t * ST];
  }
}
template <typename T, int N, int ST>
__device__ __forceinline__ void pencil_store(T* p, const T (&o)[N]) {
  if constexpr (N == 4 && ST == 1 && sizeof(T) == 8) {
    *reinterpret_cast<double2*>(p) = make_double2(o[0], o[1]);
    *reinterpret_cast<double2*>(p + 2) = make_double2(o[2], o[3]);
  } else if constexpr (N == 4 && ST == 1 && sizeof(T) == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
  } else {
#pragma unroll
    for (int t = 0; t < N; ++t) p[t * ST] = o[t];
  }
}

}  // namespace emfgpu
