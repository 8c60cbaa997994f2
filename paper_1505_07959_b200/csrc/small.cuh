// K6: small-n persistent slice kernels (n <= 64): a whole propagation inside one CTA's shared memory.
//
// At n = 32 (BASELINE cfg[0]) one GEMM is 65 kflop, so a launch per GEMM is pure latency (the fine
// propagator of one sweep would be 8 x 64 x (dependent) launches).  Here
//   * fine_smem_kernel: one CTA per slice runs all m_F RK4 steps of F(U^k_n) (R1) with every
//     operand resident in shared memory; one launch per sweep;
//   * coarse_smem_kernel: one CTA runs the rank's whole sequential coarse sweep -- Step 0
//     (eq. eqStep0) or the correction sweep (eq. eqStepk+1, R3) -- keeping the
//     running state in shared memory; one launch per sweep per rank.
// The DMMA issue order, the lane -> k mapping (k = 8kb + 2c + s) and the epilogue arithmetic are the
// same as in gemm.cuh, so results are bitwise identical to the launch-per-GEMM path (tested).
#pragma once
#include <cuda_runtime.h>

#include "gemm.cuh"
#include "ptx.cuh"

namespace mfode {

constexpr int kSmallThreads = 256;   // 8 warps

template <int NP>
struct SmallCfg {
  static constexpr int LDS = NP + 4;                 // smem row stride (doubles): conflict-free LDS.64
  static constexpr int MAT = NP * LDS;               // doubles per smem matrix
  static constexpr int TILES = (NP / 8) * (NP / 8);  // m8n8 output tiles
  static constexpr int TPW = TILES / 8;              // tiles per warp
  static_assert(TILES % 8 == 0, "NP must be a multiple of 16 (8 warps)");
};

// acc[t][0..1] (+)= P * Q for this warp's TPW tiles; P, Q: NP x NP in smem with stride LDS.
template <int NP>
__device__ __forceinline__ void smem_gemm(const double* __restrict__ P, const double* __restrict__ Q,
                                          double (&acc)[SmallCfg<NP>::TPW][2]) {
  using C = SmallCfg<NP>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
#pragma unroll
  for (int t = 0; t < C::TPW; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll 2
  for (int kb = 0; kb < NP / 8; ++kb) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int k = kb * 8 + 2 * c + s;
#pragma unroll
      for (int t = 0; t < C::TPW; ++t) {
        const int tile = warp * C::TPW + t;
        const int mt = tile / (NP / 8), nt = tile % (NP / 8);
        const double a = P[(mt * 8 + g) * C::LDS + k];
        const double b = Q[k * C::LDS + nt * 8 + g];
        dmma(acc[t][0], acc[t][1], a, b);
      }
    }
  }
}

// element (row, col) of accumulator entry (t, e) of this thread
template <int NP>
__device__ __forceinline__ void acc_pos(int t, int e, int& row, int& col) {
  using C = SmallCfg<NP>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = warp * C::TPW + t;
  row = (tile / (NP / 8)) * 8 + (lane >> 2);
  col = (tile % (NP / 8)) * 8 + 2 * (lane & 3) + e;
}

template <int NP>
__device__ __forceinline__ void load_mat(double* dst, const double* __restrict__ src, int n, int ld) {
  using C = SmallCfg<NP>;
  for (int i = threadIdx.x; i < NP * NP; i += blockDim.x) {
    const int r = i / NP, cc = i % NP;
    dst[r * C::LDS + cc] = (r < n && cc < n) ? src[(long long)r * ld + cc] : 0.0;
  }
}

template <int NP>
__device__ __forceinline__ void store_mat(double* __restrict__ dst, const double* src, int n, int ld) {
  using C = SmallCfg<NP>;
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
    const int r = i / n, cc = i % n;
    dst[(long long)r * ld + cc] = src[r * C::LDS + cc];
  }
}

// K = F(Y) in registers.  inverse: W = B Y (to smem W), K = Y W;  sqrt: K = -(Y Y) + A (A in `M`);
// exp: K = A Y.
template <int NP>
__device__ __forceinline__ void rhs_regs(int flow, const double* M, const double* Y, double* W,
                                         double (&K)[SmallCfg<NP>::TPW][2]) {
  using C = SmallCfg<NP>;
  if (flow == 0) {
    double w[C::TPW][2];
    smem_gemm<NP>(M, Y, w);
#pragma unroll
    for (int t = 0; t < C::TPW; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int r, cc;
        acc_pos<NP>(t, e, r, cc);
        W[r * C::LDS + cc] = w[t][e];
      }
    __syncthreads();
    smem_gemm<NP>(Y, W, K);
  } else if (flow == 2) {   // exp: K = A Y
    smem_gemm<NP>(M, Y, K);
  } else {
    smem_gemm<NP>(Y, Y, K);
#pragma unroll
    for (int t = 0; t < C::TPW; ++t)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int r, cc;
        acc_pos<NP>(t, e, r, cc);
        K[t][e] = fma(-1.0, K[t][e], 1.0 * M[r * C::LDS + cc]);
      }
  }
}

// ------------------------------------------------------------------------------------------------
// fine propagator: blockIdx.x = batch index z; slice input X0 = Uin + z*mstride, output Fout + z*mstride
// ------------------------------------------------------------------------------------------------
template <int NP>
__global__ void __launch_bounds__(kSmallThreads, 1)
    fine_smem_kernel(int flow, int n, int ld, const double* __restrict__ M, const double* __restrict__ Uin,
                     double* __restrict__ Fout, long long mstride, int mF, double h, const int* stop_flag) {
  using C = SmallCfg<NP>;
  if (cta_stop(stop_flag)) return;
  extern __shared__ double sm[];
  double* sM = sm;
  double* sX = sM + C::MAT;
  double* sY = sX + C::MAT;
  double* sW = sY + C::MAT;
  double* sS = sW + C::MAT;
  const int z = blockIdx.x;
  load_mat<NP>(sM, M, n, ld);
  load_mat<NP>(sX, Uin + z * mstride, n, ld);
  for (int i = threadIdx.x; i < C::MAT; i += blockDim.x) sY[i] = 0.0;
  __syncthreads();
  const double h6 = h / 6.0;
  for (int step = 0; step < mF; ++step) {
    for (int s = 1; s <= 4; ++s) {
      const double* Yin = (s == 1) ? sX : sY;
      double K[C::TPW][2];
      rhs_regs<NP>(flow, sM, Yin, sW, K);
      __syncthreads();   // every read of Yin / W done before the epilogue overwrites Y
      const double cy = (s == 3) ? h : 0.5 * h;
#pragma unroll
      for (int t = 0; t < C::TPW; ++t)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int r, cc;
          acc_pos<NP>(t, e, r, cc);
          const int o = r * C::LDS + cc;
          const double k = K[t][e];
          if (s == 4) {
            sX[o] = fma(h6, sS[o] + k, sX[o]);
          } else {
            sS[o] = (s == 1) ? k : fma(2.0, k, sS[o]);
            sY[o] = fma(cy, k, sX[o]);
          }
        }
      __syncthreads();
    }
  }
  store_mat<NP>(Fout + z * mstride, sX, n, ld);
}

// ------------------------------------------------------------------------------------------------
// coarse sweep over local slices j = j0 .. nloc-1 (single CTA).
//   V_{j0} = Vin;  for each j: g = G(V_j) (mG Euler steps);
//   correct == 0 (Step 0): U[j+1] = g, Gold[j] = g
//   correct == 1:          U[j+1] = Fk[j] + (g - Gold[j]), Gold[j] = g
//   V_{j+1} = U[j+1]
// ------------------------------------------------------------------------------------------------
template <int NP>
__global__ void __launch_bounds__(kSmallThreads, 1)
    coarse_smem_kernel(int flow, int n, int ld, const double* __restrict__ M, const double* __restrict__ Vin,
                       double* __restrict__ U, double* __restrict__ Gold, const double* __restrict__ Fk,
                       long long mstride, int j0, int nloc, int mG, double h, int correct) {
  using C = SmallCfg<NP>;
  extern __shared__ double sm[];
  double* sM = sm;
  double* sV = sM + C::MAT;   // running state
  double* sT = sV + C::MAT;   // Euler temp
  double* sW = sT + C::MAT;
  load_mat<NP>(sM, M, n, ld);
  load_mat<NP>(sV, Vin, n, ld);
  for (int i = threadIdx.x; i < C::MAT; i += blockDim.x) sT[i] = 0.0;
  __syncthreads();
  for (int j = j0; j < nloc; ++j) {
    double* X = sV;
    for (int i = 0; i < mG; ++i) {
      double K[C::TPW][2];
      rhs_regs<NP>(flow, sM, X, sW, K);
      __syncthreads();
      const bool last = (i == mG - 1);
      // Euler: g = X + h K; intermediate steps go to sT/sV alternately (X is read before overwritten)
      double* dst = (X == sV) ? sT : sV;
#pragma unroll
      for (int t = 0; t < C::TPW; ++t)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int r, cc;
          acc_pos<NP>(t, e, r, cc);
          const int o = r * C::LDS + cc;
          const double g = fma(h, K[t][e], X[o]);
          if (!last) {
            dst[o] = g;
          } else if (r < n && cc < n) {
            const long long go = (long long)j * mstride + (long long)r * ld + cc;
            double u;
            if (correct) {
              u = Fk[go] + (g - Gold[go]);
            } else {
              u = g;
            }
            Gold[go] = g;
            U[(long long)(j + 1) * mstride + (long long)r * ld + cc] = u;
            dst[o] = u;
          } else {
            dst[o] = 0.0;
          }
        }
      __syncthreads();
      X = dst;
    }
    if (X != sV) {   // keep the running state in sV
      for (int i = threadIdx.x; i < C::MAT; i += blockDim.x) sV[i] = X[i];
      __syncthreads();
    }
  }
}

}  // namespace mfode
