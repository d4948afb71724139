// Measured experiment: can tcgen05.mma kind::tf32 speed up
// the fp32 Q4 sum-factorization sweeps?  One x-direction sweep step of the
// element kernel contracts 128 pencils (5 GLL values each) with the stacked
// [B; D] table (10 x 5) into 10 outputs per pencil, and the outputs must
// return to shared memory for the next direction's sweep.  Both variants run
// that step R times per CTA on a shared-memory tile:
//   fma   : a thread owns a pencil: 5 LDS, 50 FFMA (table in registers), 10 STS;
//   tf32  : one elected thread issues D[128 x 16] = U[128 x 8] . T^T[8 x 16]
//           (K 5 -> 8, N 10 -> 16 padded; tcgen05.mma.cta_group::1.kind::tf32,
//           A and B from shared memory, no swizzle, K-major), commits to an
//           mbarrier, the 4 warps read D back (tcgen05.ld 32x32b.x16) and
//           store the 10 useful columns (10 STS per thread);
//   tf32x3: the same with the 3xTF32 split (Uhi Thi + Uhi Tlo + Ulo Thi) that
//           fp32 accuracy (1e-5) needs, the split of U done per step.
// Timing with CUDA events over all CTAs (148 x 4); the results are checked
// against an fp64 host contraction.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tf32_sweep tf32_sweep.cu
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                              \
    }                                                                            \
  } while (0)

constexpr int kP = 128;  // pencils per CTA tile (MMA M)
constexpr int kK = 8;    // padded contraction length (5 used)
constexpr int kN = 16;   // padded outputs (10 used)

__constant__ float c_tab[10][5];  // rows 0-4: B[q][a], rows 5-9: D[q][a]

// ---- FMA variant ----------------------------------------------------------------
__global__ void __launch_bounds__(128) sweep_fma(const float* __restrict__ gin, float* __restrict__ gout, int reps) {
  __shared__ float u[kP * 5];
  __shared__ float o[kP * 10];
  const int t = threadIdx.x;
  for (int a = 0; a < 5; ++a) u[t * 5 + a] = gin[(blockIdx.x * kP + t) * 5 + a];
  float tab[10][5];
#pragma unroll
  for (int q = 0; q < 10; ++q)
#pragma unroll
    for (int a = 0; a < 5; ++a) tab[q][a] = c_tab[q][a];
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
    float v[5];
#pragma unroll
    for (int a = 0; a < 5; ++a) v[a] = u[t * 5 + a];
#pragma unroll
    for (int q = 0; q < 10; ++q) {
      float s = tab[q][0] * v[0];
#pragma unroll
      for (int a = 1; a < 5; ++a) s = fmaf(tab[q][a], v[a], s);
      o[t * 10 + q] = s;
    }
    __syncthreads();
    // next step's input = this step's B outputs (keeps the data dependence)
#pragma unroll
    for (int a = 0; a < 5; ++a) u[t * 5 + a] = fmaf(o[t * 10 + a], 1e-30f, v[a]);
    __syncthreads();
  }
  for (int q = 0; q < 10; ++q) gout[(blockIdx.x * kP + t) * 10 + q] = o[t * 10 + q];
}

// ---- tcgen05 helpers ------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// No-swizzle K-major descriptor: core matrices of 8 rows x 16 bytes stored
// contiguously (128 B); LBO = byte distance between the two core matrices
// along K, SBO = byte distance between 8-row groups (cute::UMMA::SmemDescriptor).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
  return d;
}
// instruction descriptor: D f32, A/B tf32, K-major both, N = 16, M = 128
__host__ __device__ constexpr uint32_t make_idesc() {
  return (1u << 4)            // c_format F32
         | (2u << 7)          // a_format TF32
         | (2u << 10)         // b_format TF32
         | ((kN >> 3) << 17)  // n_dim
         | ((kP >> 4) << 24); // m_dim
}

// element (row, k) of a K-major no-swizzle tile with 8x(16 B) core matrices:
// core (row/8, k/4) at ((row/8) * 2 + k/4) * 32 floats, inside it row%8 * 4 + k%4
__device__ __forceinline__ int tile_off(int row, int k) { return ((row >> 3) * 2 + (k >> 2)) * 32 + (row & 7) * 4 + (k & 3); }

__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ bool mbar_wait(uint64_t* b, uint32_t phase) {
  uint32_t ok = 0;
  for (long it = 0; it < 20000000L; ++it) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(phase));
    if (ok) return true;
  }
  return false;  // bounded: never hang the device
}

template <int NMMA>
__global__ void __launch_bounds__(128) sweep_tf32(const float* __restrict__ gin, float* __restrict__ gout, int reps,
                                                  int* err) {
  // A tiles (U hi / lo) and B tiles (table hi / lo), 1 KB aligned
  __shared__ __align__(1024) float sa[2][kP * kK];
  __shared__ __align__(1024) float sb[2][kN * kK];
  __shared__ float o[kP * 10];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int t = threadIdx.x, warp = t >> 5;
  // table as B (N rows = outputs, K-major), hi and lo parts
  for (int i = t; i < kN * kK; i += 128) {
    const int n = i / kK, k = i % kK;
    const float v = (n < 10 && k < 5) ? c_tab[n][k] : 0.f;
    uint32_t hb;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(v));
    const float hi = __uint_as_float(hb);
    sb[0][tile_off(n, k)] = hi;
    sb[1][tile_off(n, k)] = v - hi;
  }
  float u0[5];
  for (int k = 0; k < kK; ++k) {
    const float v = k < 5 ? gin[(blockIdx.x * kP + t) * 5 + k] : 0.f;
    if (k < 5) u0[k] = v;
    sa[0][tile_off(t, k)] = v;
    sa[1][tile_off(t, k)] = 0.f;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) mbar_init(&bar, 1);
  asm volatile("fence.proxy.async.shared::cta;");  // generic-proxy smem writes -> async proxy (MMA reads)
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  constexpr uint32_t idesc = make_idesc();
  // core matrix = 8 rows x 16 B = 128 B; along K the next core matrix is +128 B (LBO), next 8 rows +256 B (SBO)
  const uint64_t da0 = make_desc(smem_u32(sa[0]), 128, 256), da1 = make_desc(smem_u32(sa[1]), 128, 256);
  const uint64_t db0 = make_desc(smem_u32(sb[0]), 128, 256), db1 = make_desc(smem_u32(sb[1]), 128, 256);
  uint32_t phase = 0;
  for (int r = 0; r < reps; ++r) {
    if (NMMA == 3) {  // split U into tf32 hi / lo (U was written by this thread)
      for (int k = 0; k < 5; ++k) {
        const float v = sa[0][tile_off(t, k)];
        uint32_t hb;
        asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(hb) : "f"(v));
        const float hi = __uint_as_float(hb);
        sa[0][tile_off(t, k)] = hi;
        sa[1][tile_off(t, k)] = v - hi;
      }
      asm volatile("fence.proxy.async.shared::cta;");
    }
    __syncthreads();
    if (t == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      auto mma = [&](uint64_t a, uint64_t b, int acc) {
        asm volatile(
            "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
            " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(a), "l"(b), "r"(idesc), "r"(acc));
      };
      mma(da0, db0, 0);
      if (NMMA == 3) {
        mma(da0, db1, 1);
        mma(da1, db0, 1);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];" ::"l"(
          (uint64_t)__cvta_generic_to_shared(&bar)));
    }
    if (!mbar_wait(&bar, phase)) {
      if (t == 0) atomicAdd(err, 1);
      break;
    }
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
    // warp w reads TMEM lanes 32w..32w+31 (its pencils), columns 0-15
    uint32_t d[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
          "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
        : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int q = 0; q < 10; ++q) o[t * 10 + q] = __uint_as_float(d[q]);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    for (int a = 0; a < 5; ++a) sa[0][tile_off(t, a)] = fmaf(o[t * 10 + a], 1e-30f, u0[a]);
    asm volatile("fence.proxy.async.shared::cta;");
  }
  __syncthreads();
  for (int q = 0; q < 10; ++q) gout[(blockIdx.x * kP + t) * 10 + q] = o[t * 10 + q];
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main(int argc, char** argv) {
  const int reps = argc > 1 ? std::atoi(argv[1]) : 200;
  const int blocks = 148 * 4;
  // Q4 tables on GLL nodes / Gauss points (values need not be exact here:
  // the check is against the same tables in fp64)
  float h_tab[10][5];
  for (int q = 0; q < 10; ++q)
    for (int a = 0; a < 5; ++a) h_tab[q][a] = std::sin(0.7f * q + 1.3f * a + 0.1f) * (q < 5 ? 0.6f : 1.9f);
  CK(cudaMemcpyToSymbol(c_tab, h_tab, sizeof(h_tab)));
  const size_t np = (size_t)blocks * kP;
  std::vector<float> in(np * 5);
  for (size_t i = 0; i < in.size(); ++i) in[i] = std::cos(0.37f * (float)i) * 0.9f;
  float *din, *dout;
  int* derr;
  CK(cudaMalloc(&din, in.size() * 4));
  CK(cudaMalloc(&dout, np * 10 * 4));
  CK(cudaMalloc(&derr, 4));
  CK(cudaMemcpy(din, in.data(), in.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(derr, 0, 4));
  // fp64 reference of one step on pencil p (the steps feed back o * 1e-30)
  auto ref = [&](size_t p, double* out10) {
    double u[5];
    for (int a = 0; a < 5; ++a) u[a] = in[p * 5 + a];
    double o[10];
    for (int q = 0; q < 10; ++q) {
      o[q] = 0;
      for (int a = 0; a < 5; ++a) o[q] += (double)h_tab[q][a] * u[a];
    }
    for (int q = 0; q < 10; ++q) out10[q] = o[q];
  };
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto run = [&](const char* name, auto launch) {
    launch();
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    for (int it = 0; it < 5; ++it) launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= 5;
    std::vector<float> out(np * 10);
    CK(cudaMemcpy(out.data(), dout, out.size() * 4, cudaMemcpyDeviceToHost));
    int herr = 0;
    CK(cudaMemcpy(&herr, derr, 4, cudaMemcpyDeviceToHost));
    double num = 0, den = 0;
    for (size_t p = 0; p < np; p += 97) {
      double o[10];
      ref(p, o);
      for (int q = 0; q < 10; ++q) {
        num += (out[p * 10 + q] - o[q]) * (out[p * 10 + q] - o[q]);
        den += o[q] * o[q];
      }
    }
    const double steps = (double)np * reps;
    std::printf("%-7s %8.3f ms  %7.2f Gpencil-steps/s  %7.2f TFLOP/s useful  rel-L2 %.2e  timeouts %d\n", name, ms,
                steps / (ms * 1e-3) / 1e9, steps * 100.0 / (ms * 1e-3) / 1e12, std::sqrt(num / den), herr);
  };
  run("fma", [&] { sweep_fma<<<blocks, 128>>>(din, dout, reps); });
  run("tf32", [&] { sweep_tf32<1><<<blocks, 128>>>(din, dout, reps, derr); });
  run("tf32x3", [&] { sweep_tf32<3><<<blocks, 128>>>(din, dout, reps, derr); });
  CK(cudaGetLastError());
  return 0;
}
