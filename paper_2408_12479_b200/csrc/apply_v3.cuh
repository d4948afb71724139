// Tangent-apply element phase, v3: one warp per element (Q2, Q3).
//
// Each warp streams its own sequence of elements (persistent), so there is no
// CTA-wide barrier anywhere: phases are separated by __syncwarp() and warps of
// the same SM sit in different phases (sweeps vs quadrature-point algebra),
// which keeps the FP64 pipe and the shared-memory pipe busy at the same time.
// The next element's x / u_k / affine geometry are prefetched with cp.async
// into the warp's single staging buffer as soon as the current element has
// consumed it (after the first x-sweep of u_k).  A lane owns N3/32 quadrature
// points (2 for Q3, 1 for Q2) and up to 2 sweep pencils.
// Sweeps, layout, geometry paths and qp algebra are those of apply_v2.cuh.
#pragma once
#include "apply_v2.cuh"

namespace emfgpu {

template <typename T, int P, int MODEL, int STRAT>
struct ApplyV3Warp {
  static constexpr int N = P + 1, SZ = Lay<N, sizeof(T)>::SIZE;
  static constexpr bool kUk = (STRAT == S_NONE || STRAT == S_SCALAR || STRAT == S_SP_NONE || STRAT == S_SP_SCALAR);
  static constexpr int NST = kUk ? 6 : 3;
  T stage[NST][SZ];
  T geo[10];
  T r1[9][SZ];
  T r2[9][SZ];
};

constexpr int kV3Warps = 4;

// CTAs per SM for the launch bounds: fp32 4, fp64 3 (4 measured slower even
// where it fits without spills: cfg1 fp64 tensor 0.1251 -> 0.1382 ms).
#ifndef EMF_MINB_V3F
#define EMF_MINB_V3F 0  // fp32 v3 CTAs/SM override (experiments)
#endif
#ifndef EMF_MINB_FIBER_V3F
#define EMF_MINB_FIBER_V3F 4
#endif
#ifndef EMF_MINB_FIBER_V3D
#define EMF_MINB_FIBER_V3D 2
#endif
template <typename T, int MODEL, int STRAT>
constexpr int minb_v3() {
  // fibre: fp64 2 CTAs/SM, spill-free (32^3 Q3 tensor 0.226 -> 0.208 ms);
  // fp32 keeps 4 (3 measured slower: 0.167 -> 0.187 ms)
  if (MODEL == FIBER) return sizeof(T) == 4 ? EMF_MINB_FIBER_V3F : EMF_MINB_FIBER_V3D;
  return sizeof(T) == 4 ? (EMF_MINB_V3F ? EMF_MINB_V3F : 4) : 3;
}

template <typename T, int P, int MODEL, int STRAT, bool CART>
__global__ void __launch_bounds__(32 * kV3Warps, (minb_v3<T, MODEL, STRAT>())) apply_v3_kernel(const KArgs<T> a) {
  using WS = ApplyV3Warp<T, P, MODEL, STRAT>;
  constexpr int N = P + 1, N3 = N * N * N, SZ = Lay<N, sizeof(T)>::SIZE;
  constexpr int QPL = (N3 + 31) / 32;  // quadrature points per lane
  constexpr bool kUk = WS::kUk;
  extern __shared__ __align__(16) unsigned char v3_smem[];  // kV3Warps * sizeof(WS), dynamic
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WS& sm = reinterpret_cast<WS*>(v3_smem)[warp];
  T* const R1 = &sm.r1[0][0];
  T* const R2 = &sm.r2[0][0];
  const T* Bm = a.Bm;
  const T* Dm = a.Dm;

  // cp.async of element e's inputs into the staging buffer; `which` selects
  // x (1), u_k (2) or both (3)
  // returns, per point r of this lane (bit r), whether its staged x value
  // must be zeroed (Dirichlet node); only meaningful when x is fetched
  auto prefetch = [&](int64_t e, int which) -> unsigned {
    unsigned zero = 0;
    if (e < a.nel) {
#pragma unroll
      for (int r = 0; r < QPL; ++r) {
        const int q = lane + 32 * r;
        if (q < N3) {
          const int qi = q % N, qj = (q / N) % N, qk = q / (N * N);
          const ElemPos ep = elem_pos_fast<P>(e, a, qi, qj, qk);
          if (node_constrained(ep.ga, ep.gb, ep.gc, a.mx, a.my, a.mz, a.faces)) zero |= 1u << r;
          const int qs = lat<N>(qi, qj, qk);
          if (which & 1)
#pragma unroll
            for (int c = 0; c < 3; ++c) cp_async_T(&sm.stage[c][qs], a.x + 3 * ep.node + c);
          if constexpr (kUk)
            if (which & 2)
#pragma unroll
              for (int c = 0; c < 3; ++c) cp_async_T(&sm.stage[3 + c][qs], a.uk + 3 * ep.node + c);
        }
      }
      if ((which & 1) && a.affine && (!is_spatial(STRAT) || kUk) && lane < 10)
        cp_async_T(&sm.geo[lane], a.geo + lane * a.geo_stride + e);
    }
    cp_async_commit();
    return zero;
  };

  T wq3[QPL];  // tensor-product weights of this lane's points (operator.hpp:492), fp32 path
#pragma unroll
  for (int r = 0; r < QPL; ++r) {
    const int q = lane + 32 * r < N3 ? lane + 32 * r : 0;
    wq3[r] = T(a.qwd[q % N] * a.qwd[(q / N) % N] * a.qwd[q / (N * N)]);
  }
  // Elements handed out by a ticket counter, one warp = one worker (as
  // apply_v2): the first two elements of a warp are static, later tickets
  // are taken by lane 0 one element ahead and their values used an element
  // later, so the atomic's round trip is never waited on.
  // The fibre tensor variants keep the static stride (measured: tickets
  // 0.218 / 0.177 ms vs static 0.206 / 0.165 ms fp64 / fp32 at 32^3 Q3;
  // cNH fp32 and fp64 cachedF gain 2-2.5% from tickets).
  constexpr bool kTk = MODEL != FIBER;
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");  // see apply_v2_kernel
  const int nw = (int)gridDim.x * kV3Warps;
  const int nu = (int)(a.nel - a.e_begin);
  int cur = (int)blockIdx.x * kV3Warps + warp, nxt = cur + nw;
  unsigned praw = 0;
  if (kTk && lane == 0 && nxt < nu) praw = atomicAdd(a.tk, 1u);
  unsigned zero_cur = prefetch(cur + a.e_begin, 3);
  while (cur < nu) {
    const int64_t e = cur + a.e_begin;
    const int64_t e_next = nxt + a.e_begin;
    cp_async_wait<0>();
    __syncwarp();
    // Dirichlet columns of x are masked (operator.hpp:604-605)
#pragma unroll
    for (int r = 0; r < QPL; ++r) {
      const int q = lane + 32 * r;
      if (q < N3 && ((zero_cur >> r) & 1u)) {
        const int qs = lat<N>(q % N, (q / N) % N, q / (N * N));
#pragma unroll
        for (int c = 0; c < 3; ++c) sm.stage[c][qs] = T(0);
      }
    }
    // affine geometry to registers now: the staging buffer is refilled with
    // the next element's data before the quadrature-point phase
    T j0d[3], g9[9], det0 = T(0);
    if (CART || a.affine) {
#pragma unroll
      for (int m = 0; m < 9; ++m) g9[m] = sm.geo[m];
      j0d[0] = g9[0];
      j0d[1] = g9[4];
      j0d[2] = g9[8];
      det0 = sm.geo[9];
    }
    __syncwarp();
    // fp32 with u_k: x and u_k swept together in place (apply_v2.cuh fwc_*),
    // 3 full 32-lane rounds per stage instead of 4 half-empty ones; the
    // staging buffer then holds d/dz until the points have read it
    // scalar strategy: this lane's cached scalars loaded before the sweeps
    // (their latency hidden behind them, as in apply_v2)
    constexpr bool kScEarly3 = STRAT == S_SCALAR && EMF_SC_EARLY;
    Bundle<T> scb[QPL];
    if constexpr (kScEarly3) {
#pragma unroll
      for (int r = 0; r < QPL; ++r) {
        const int q = lane + 32 * r;
        if (q < N3) load_scalars<T, MODEL>(a.cache, a.cache_stride, e * N3 + q, scb[r]);
      }
    }
    constexpr bool kFused = kUk && sizeof(T) == 4;
    T* const S = &sm.stage[0][0];
    T gx[QPL][9];
    if constexpr (kFused) {
      fwc_x<T, N, 2, 32>(S, R2, Bm, Dm, lane);
      __syncwarp();
      fwc_y<T, N, 2, 32>(S, R2, R1, Bm, Dm, lane);
      __syncwarp();
      fwc_z<T, N, 2, 32>(S, R2, R1, Bm, Dm, lane);
      __syncwarp();
#pragma unroll
      for (int r = 0; r < QPL; ++r) {
        const int q = lane + 32 * r;
        const int qs = q < N3 ? lat<N>(q % N, (q / N) % N, q / (N * N)) : 0;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          gx[r][3 * c + 0] = R1[c * SZ + qs];
          gx[r][3 * c + 1] = R2[c * SZ + qs];
          gx[r][3 * c + 2] = S[c * SZ + qs];
        }
      }
    } else {
    // ---- gradient of x
    fw_x<T, N, 32>(&sm.stage[0][0], R2, R2 + 3 * SZ, Bm, Dm, lane);
    __syncwarp();
    if constexpr (!kUk) zero_cur = prefetch(e_next, 1);
    fw_y<T, N, 32>(R2, R2 + 3 * SZ, R1, R1 + 3 * SZ, R1 + 6 * SZ, Bm, Dm, lane);
    __syncwarp();
    fw_z<T, N, 32>(R1, R1 + 3 * SZ, R1 + 6 * SZ, R2, Bm, Dm, lane);
    __syncwarp();
#pragma unroll
    for (int r = 0; r < QPL; ++r) {
      const int q = lane + 32 * r;
      const int qs = q < N3 ? lat<N>(q % N, (q / N) % N, q / (N * N)) : 0;
#pragma unroll
      for (int m = 0; m < 9; ++m) gx[r][m] = R2[m * SZ + qs];
    }
    }
    if constexpr (kUk && !kFused) {
      __syncwarp();
      fw_x<T, N, 32>(&sm.stage[3][0], R2, R2 + 3 * SZ, Bm, Dm, lane);
      __syncwarp();
      zero_cur = prefetch(e_next, 3);  // the staging buffer is free from here on
      fw_y<T, N, 32>(R2, R2 + 3 * SZ, R1, R1 + 3 * SZ, R1 + 6 * SZ, Bm, Dm, lane);
      __syncwarp();
      fw_z<T, N, 32>(R1, R1 + 3 * SZ, R1 + 6 * SZ, R2, Bm, Dm, lane);
      __syncwarp();
    }
    // ---- quadrature-point phase.  fp64: the points of a lane one after the
    // other (interleaving them exceeds the register budget); fp32: unrolled so
    // the two points' instruction streams interleave.
    const T* cs = a.cache;
    const int64_t st = a.cache_stride;
    auto qp_point = [&](int r) {
      const int q = lane + 32 * r;
      if (q >= N3) return;
      T gxr[9];
#pragma unroll
      for (int m = 0; m < 9; ++m) gxr[m] = gx[0][m];
      if constexpr (QPL > 1)
        if (r == 1)
#pragma unroll
          for (int m = 0; m < 9; ++m) gxr[m] = gx[QPL > 1 ? 1 : 0][m];
      const int qi = q % N, qj = (q / N) % N, qk = q / (N * N);
      const int qs = lat<N>(qi, qj, qk);
      const int64_t qidx = e * N3 + q;
      // fp32: hoisted per-lane weights; fp64 (sequential points, register-bound): recomputed
      const T wqr = sizeof(T) == 8 ? T(a.qwd[qi] * a.qwd[qj] * a.qwd[qk])
                                   : ((QPL > 1 && r == 1) ? wq3[QPL > 1 ? 1 : 0] : wq3[0]);
      const MatConst<T> mq = mat_at<T, MODEL>(a.mat, a.hq, a.hq_stride, qidx);
      T j0inv[9], detw;
      if (CART) {
        detw = det0 * wqr;
      } else if (a.affine) {
#pragma unroll
        for (int m = 0; m < 9; ++m) j0inv[m] = g9[m];
        detw = det0 * wqr;
      } else if (!is_spatial(STRAT) || kUk) {
#pragma unroll
        for (int m = 0; m < 9; ++m) j0inv[m] = a.geo[m * a.geo_stride + qidx];
        detw = a.geo[9 * a.geo_stride + qidx];
      }
      Bundle<T> cb;
      SpCell<T> sp;
      if constexpr (is_spatial(STRAT)) {
        // spatial formulation (operator.hpp:506-519): bundle from G_k (none,
        // scalar) or the stored spatial cell (tensor), test with J_t^-1
        T gg[9];
        if constexpr (kUk) {
          T gk[9];
          if constexpr (kFused) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              gk[3 * c + 0] = R1[(3 + c) * SZ + qs];
              gk[3 * c + 1] = R2[(3 + c) * SZ + qs];
              gk[3 * c + 2] = S[(3 + c) * SZ + qs];
            }
          } else {
#pragma unroll
            for (int m = 0; m < 9; ++m) gk[m] = R2[m * SZ + qs];
          }
          mm(gk, j0inv, gg);
        }
        if (!spatial_bundle<T, MODEL>(STRAT - S_SP_NONE, mq, gg, cs, st, qidx, cb, sp))
          atomicMin(a.err, (unsigned long long)qidx);
      } else if constexpr (kUk) {
        T gk[9], gg[9];
        if constexpr (kFused) {
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            gk[3 * c + 0] = R1[(3 + c) * SZ + qs];
            gk[3 * c + 1] = R2[(3 + c) * SZ + qs];
            gk[3 * c + 2] = S[(3 + c) * SZ + qs];
          }
        } else {
#pragma unroll
          for (int m = 0; m < 9; ++m) gk[m] = R2[m * SZ + qs];
        }
        if constexpr (CART) {
#pragma unroll
          for (int m = 0; m < 9; ++m) gg[m] = gk[m] * j0d[m % 3];
        } else {
          mm(gk, j0inv, gg);
        }
        if (!make_strain(gg, cb)) atomicMin(a.err, (unsigned long long)qidx);
        if constexpr (STRAT == S_NONE) {
          cache_scalars<T, MODEL>(mq, cb);
        } else if constexpr (kScEarly3) {
          const Bundle<T>& sb = (QPL > 1 && r == 1) ? scb[QPL > 1 ? 1 : 0] : scb[0];
          cb.lnj = sb.lnj;
          cb.jp = sb.jp;
          cb.c1 = sb.c1;
          cb.c2 = sb.c2;
          cb.c3[0] = sb.c3[0];
          cb.c3[1] = sb.c3[1];
          cb.efib[0] = sb.efib[0];
          cb.efib[1] = sb.efib[1];
        } else {
          if (MODEL == CNH) cb.lnj = cs[C_LNJ * st + qidx];
          else {
            cb.jp = cs[C_JP * st + qidx];
            cb.c1 = cs[C_C1 * st + qidx];
            cb.c2 = cs[C_C2 * st + qidx];
          }
          if (MODEL == FIBER) {
            cb.c3[0] = cs[(C_C3 + 0) * st + qidx];
            cb.c3[1] = cs[(C_C3 + 1) * st + qidx];
            cb.efib[0] = cs[(C_EF + 0) * st + qidx];
            cb.efib[1] = cs[(C_EF + 1) * st + qidx];
          }
        }
        second_pk<T, MODEL>(mq, cb);
      } else if constexpr (STRAT == S_CACHEDF) {
        T gg[9];
#pragma unroll
        for (int m = 0; m < 9; ++m) gg[m] = cs[(C_G + m) * st + qidx];
        if (!make_strain(gg, cb)) atomicMin(a.err, (unsigned long long)qidx);
        cache_scalars<T, MODEL>(mq, cb);
        second_pk<T, MODEL>(mq, cb);
      } else {  // S_TENSOR
        if (MODEL == CNH) cb.lnj = cs[C_LNJ * st + qidx];
        else {
          cb.jp = cs[C_JP * st + qidx];
          cb.c1 = cs[C_C1 * st + qidx];
          cb.c2 = cs[C_C2 * st + qidx];
        }
        if (MODEL == FIBER) {
          cb.c3[0] = cs[(C_C3 + 0) * st + qidx];
          cb.c3[1] = cs[(C_C3 + 1) * st + qidx];
          cb.efib[0] = cs[(C_EF + 0) * st + qidx];
          cb.efib[1] = cs[(C_EF + 1) * st + qidx];
        }
#pragma unroll
        for (int m = 0; m < 9; ++m) {
          cb.F[m] = cs[(C_F + m) * st + qidx];
          cb.Finv[m] = cs[(C_FINV + m) * st + qidx];
        }
#pragma unroll
        for (int m = 0; m < 6; ++m) {
          cb.S[m] = cs[(C_S + m) * st + qidx];
          cb.Cinv[m] = cs[(C_CINV + m) * st + qidx];
        }
      }
      T wv[9];
      if constexpr (is_spatial(STRAT)) {
        T jt[9], jtinv[9];
#pragma unroll
        for (int m = 0; m < 9; ++m) jt[m] = cs[(C_JT + m) * st + qidx];
        inverse3(jt, jtinv);
        const T ssc = (cs[C_INVJ * st + qidx] * det3(jt)) * wqr;
        spatial_integrand<T, MODEL>(mq, cb, sp, gxr, jtinv, ssc, wv);
      } else if constexpr (CART) {
        T dg[9], wm[9];
#pragma unroll
        for (int m = 0; m < 9; ++m) dg[m] = gxr[m] * j0d[m % 3];
        tangent_wm<T, MODEL>(mq, cb, dg, wm);
#pragma unroll
        for (int m = 0; m < 9; ++m) wv[m] = wm[m] * (detw * j0d[m % 3]);
      } else {
        tangent_integrand<T, MODEL>(mq, cb, gxr, j0inv, detw, wv);
      }
#pragma unroll
      for (int m = 0; m < 9; ++m) R1[m * SZ + qs] = wv[m];
    };
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int r = 0; r < QPL; ++r) qp_point(r);
    } else {
#pragma unroll 1
      for (int r = 0; r < QPL; ++r) qp_point(r);
    }
    __syncwarp();
    if constexpr (kFused) zero_cur = prefetch(e_next, 3);  // the staging buffer is free from here on
    // ---- test with the gradients of the basis functions
    tr_z<T, N, 32>(R1, R2, Bm, Dm, lane);
    __syncwarp();
    tr_y<T, N, 32>(R2, R1, Bm, Dm, lane);
    __syncwarp();
    tr_x<T, N, 32>(R1, a.loc, e, a.nx, a.fd_nx, Bm, Dm, lane);
    __syncwarp();
    if constexpr (kTk) {
      int pt = nu;
      if (lane == 0) {
        pt = nxt < nu ? 2 * nw + (int)praw : nu;
        if (pt < nu) praw = atomicAdd(a.tk, 1u);
      }
      cur = nxt;
      nxt = __shfl_sync(0xffffffffu, pt, 0);
    } else {
      cur = nxt;
      nxt = cur + nw;
    }
  }
  cp_async_wait<0>();
  // the last worker out rewinds the counter for the next launch on this slot
  if (kTk && lane == 0) {
    if (atomicAdd(a.tk + 1, 1u) == (unsigned)(nw - 1)) {
      a.tk[0] = 0;
      a.tk[1] = 0;
    }
  }
}

}  // namespace emfgpu
