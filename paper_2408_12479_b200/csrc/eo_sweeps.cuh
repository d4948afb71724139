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

// The tables of one kernel launch: scalar halves (B, D) and, for fp32, the
// same entries as pairs for the packed f32x2 instructions of sm_100 (P):
//   P[0..2]   (BE[0][a], BE[1][a])   P[3..4]   (BO[0][a], BO[1][a])
//   P[5..7]   (DE[0][a], DE[1][a])   P[8..9]   (DO[0][a], DO[1][a])
//   P[10..12] (BE[q][0], BE[q][1])   P[13..14] (BO[q][0], BO[q][1])
//   P[15..17] (DO[q][0], DO[q][1])   P[18..19] (DE[q][0], DE[q][1])
template <typename T>
struct EoT {
  const T* B;
  const T* D;
  const float2* P;
};
#ifndef EMF_F32X2
#define EMF_F32X2 0
#endif
// Packed pairs: the two mirrored output pairs of a contraction share every
// multiplier, so one FFMA2 / FADD2 (operands: a pair of table entries, a
// broadcast scalar) does the work of two FFMA / FADD in the same order and
// rounding -- the results are bit-identical to the scalar form, the fp32
// kernels issue ~45% fewer sweep instructions.
__device__ __forceinline__ float2 pk(float x, float y) { return make_float2(x, y); }
__device__ __forceinline__ float2 pk1(float x) { return make_float2(x, x); }
__device__ __forceinline__ float2 pneg(float2 a) { return make_float2(-a.x, -a.y); }

template <typename T, int N>
struct EO {
  static constexpr int H = N / 2, CH = (N + 1) / 2;
  static constexpr bool ODD = (N & 1) != 0;
  static constexpr int NB = CH * CH + H * H;  // entries of eoB
  static constexpr int ND = H * CH + CH * H;  // entries of eoD
  static constexpr bool kPack = EMF_F32X2 && sizeof(T) == 4 && H == 2;
  static __device__ __forceinline__ T be(const T* t, int q, int a) { return t[q * CH + a]; }
  static __device__ __forceinline__ T bo(const T* t, int q, int a) { return t[CH * CH + q * H + a]; }
  static __device__ __forceinline__ T de(const T* t, int q, int a) { return t[q * CH + a]; }
  static __device__ __forceinline__ T dd(const T* t, int q, int a) { return t[H * CH + q * H + a]; }
  // acc = sum_a tab[a] * (m[a], m[a]): NA terms, the first one a product
  template <int NA, int NM>
  static __device__ __forceinline__ float2 pdot(const float2* tab, const T (&m)[NM]) {
    float2 acc = __fmul2_rn(tab[0], pk1((float)m[0]));
#pragma unroll
    for (int a = 1; a < NA; ++a) acc = __ffma2_rn(tab[a], pk1((float)m[a]), acc);
    return acc;
  }
  // o[0], o[1] = x + y and o[N-1], o[N-2] = x - y
  static __device__ __forceinline__ void psum(float2 x, float2 y, T (&o)[N]) {
    const float2 lo = __fadd2_rn(x, y), hi = __fadd2_rn(x, pneg(y));
    o[0] = lo.x, o[1] = lo.y, o[N - 1] = hi.x, o[N - 2] = hi.y;
  }

  // mirrored sums / differences of u; e[c] = u[c]
  static __device__ __forceinline__ void split(const T (&u)[N], T (&e)[CH], T (&d)[H ? H : 1]) {
    if constexpr (kPack) {
      const float2 lo = pk((float)u[0], (float)u[1]), hi = pk((float)u[N - 1], (float)u[N - 2]);
      const float2 e2 = __fadd2_rn(lo, hi), d2 = __fadd2_rn(lo, pneg(hi));
      e[0] = e2.x, e[1] = e2.y, d[0] = d2.x, d[1] = d2.y;
    } else {
#pragma unroll
      for (int a = 0; a < H; ++a) {
        e[a] = u[a] + u[N - 1 - a];
        d[a] = u[a] - u[N - 1 - a];
      }
    }
    if (ODD) e[H] = u[H];
  }

  // o[q] = sum_a B[q][a] u[a] from the split halves
  static __device__ __forceinline__ void B_split(const EoT<T>& t, const T (&e)[CH], const T (&d)[H ? H : 1],
                                                 T (&o)[N]) {
    const T* const tb = t.B;
    if constexpr (kPack) {
      psum(pdot<CH>(t.P, e), pdot<H>(t.P + 3, d), o);  // se + so, se - so
    } else {
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
    }
    if (ODD) {
      T s = be(tb, H, 0) * e[0];
#pragma unroll
      for (int a = 1; a < CH; ++a) s += be(tb, H, a) * e[a];
      o[H] = s;
    }
  }
  // o[q] = sum_r Dc[q][r] u[r] from the split halves
  static __device__ __forceinline__ void D_split(const EoT<T>& t, const T (&e)[CH], const T (&d)[H ? H : 1],
                                                 T (&o)[N]) {
    const T* const td = t.D;
    if constexpr (kPack) {
      psum(pdot<H>(t.P + 8, d), pdot<CH>(t.P + 5, e), o);  // to + te, to - te
    } else {
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
    }
    if (ODD) {
      T s = dd(td, H, 0) * d[0];
#pragma unroll
      for (int a = 1; a < H; ++a) s += dd(td, H, a) * d[a];
      o[H] = s;
    }
  }
  // o[a] = sum_q B[q][a] w[q] from the split halves of w
  static __device__ __forceinline__ void Bt_split(const EoT<T>& t, const T (&e)[CH], const T (&d)[H ? H : 1],
                                                  T (&o)[N]) {
    const T* const tb = t.B;
    if constexpr (kPack) {
      psum(pdot<CH>(t.P + 10, e), pdot<H>(t.P + 13, d), o);  // se + so, se - so
    } else {
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
    }
    if (ODD) {
      T s = be(tb, 0, H) * e[0];
#pragma unroll
      for (int q = 1; q < CH; ++q) s += be(tb, q, H) * e[q];
      o[H] = s;
    }
  }
  // o[r] = sum_q Dc[q][r] w[q] from the split halves of w
  static __device__ __forceinline__ void Dt_split(const EoT<T>& t, const T (&e)[CH], const T (&d)[H ? H : 1],
                                                  T (&o)[N]) {
    const T* const td = t.D;
    if constexpr (kPack) {
      psum(pdot<H>(t.P + 18, d), pdot<CH>(t.P + 15, e), o);  // s2 + s1, s2 - s1
    } else {
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
