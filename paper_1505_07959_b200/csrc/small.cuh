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
//
// Shared-memory layout (round 2): every matrix is NP x NP doubles, rows of NP (128-byte aligned),
// with the 16-byte column pairs of each 128-byte line XOR-swizzled by the row,
//   pair p of row r lives at pair (p & ~7) | ((p ^ h(r)) & 7),  h(r) = 2 ((r >> 1) & 3) ^ 4 (r & 1),
// so that BOTH fragment reads of gemm.cuh's DMMA mapping are 128-bit and conflict-free:
//   A role (row r = 8 mt + g, k pair 4 kb + c): the two rows of a quarter-warp differ in bit 2 of h;
//   B role (row k = 8 kb + 2 c + s, column pair 8 grp + g): the four rows of a quarter-warp have
//   h = 2c ^ 4s, distinct even values, and g fills the odd bit.
// (Round 1 used padded rows and scalar 64-bit loads: 2-way bank conflicts, two loads per DMMA.)
// Each warp owns WT_M x WT_G units of 8 rows x 16 columns (two n-tiles: the even and the odd columns
// of the group, as gemm.cuh); Y is double-buffered, so a stage needs two CTA barriers, not three;
// X and S, touched element-wise by their owning thread only, are kept in registers.
#pragma once
#include <cuda_runtime.h>

#include "gemm.cuh"
#include "ptx.cuh"

namespace mfode {

constexpr int kSmallThreads = 256;   // 8 warps

template <int NP>
struct SmallCfg {
  static constexpr int MAT = NP * NP;                        // doubles per smem matrix
  static constexpr int UNITS = (NP / 8) * (NP / 16);         // 8 x 16 units
  static constexpr int WT_G = (NP >= 64) ? 2 : 1;            // column groups per warp
  static constexpr int WT_M = UNITS / 8 / WT_G;              // m-tiles per warp
  static constexpr int WARPS_G = (NP / 16) / WT_G;           // warps along the columns
  static_assert(UNITS % 8 == 0 && WT_M >= 1, "NP must be 32 or 64");
};

__device__ __forceinline__ int swz_h(int r) { return (((r >> 1) & 3) << 1) ^ ((r & 1) << 2); }
// element (r, c) of a swizzled NP x NP matrix
template <int NP>
__device__ __forceinline__ int sidx(int r, int c) {
  const int p = c >> 1;
  return r * NP + (((p & ~7) | ((p ^ swz_h(r)) & 7)) << 1) + (c & 1);
}

template <int NP>
struct SmallAcc {
  double v[SmallCfg<NP>::WT_M][SmallCfg<NP>::WT_G][2][2];   // [m-tile][group][even/odd n-tile][e]
};

// position of accumulator entry (mi, gi, par, e) of this thread
template <int NP>
__device__ __forceinline__ void acc_pos(int mi, int gi, int par, int e, int& row, int& col) {
  using C = SmallCfg<NP>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp / C::WARPS_G, wg = warp % C::WARPS_G;
  row = (wm * C::WT_M + mi) * 8 + (lane >> 2);
  col = (wg * C::WT_G + gi) * 16 + 4 * (lane & 3) + 2 * e + par;
}

// acc = P * Q (P, Q: swizzled NP x NP in smem).  Per output element the DMMAs accumulate k in the
// order kb = 0.., s = 0, 1 over k = 8 kb + 2 c + s, exactly as gemm.cuh.
// A-role fragments of a constant matrix, kept in registers for a whole propagation
template <int NP>
struct SmallAFrag {
  double2 f[SmallCfg<NP>::WT_M][NP / 8];
};

template <int NP>
__device__ __forceinline__ void load_afrag(const double* P, SmallAFrag<NP>& fr) {
  using C = SmallCfg<NP>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  const int wm = warp / C::WARPS_G;
#pragma unroll
  for (int mi = 0; mi < C::WT_M; ++mi)
#pragma unroll
    for (int kb = 0; kb < NP / 8; ++kb)
      fr.f[mi][kb] = *reinterpret_cast<const double2*>(P + sidx<NP>((wm * C::WT_M + mi) * 8 + g, 8 * kb + 2 * c));
}

// REGA: the A-role operand comes from `fr` (registers) instead of P
template <int NP, bool REGA = false>
__device__ __forceinline__ void smem_gemm(const double* __restrict__ P, const double* __restrict__ Q, SmallAcc<NP>& acc,
                                          const SmallAFrag<NP>* fr = nullptr) {
  using C = SmallCfg<NP>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, c = lane & 3;
  const int wm = warp / C::WARPS_G, wg = warp % C::WARPS_G;
  const uint32_t sP = smem_u32(P), sQ = smem_u32(Q);
#pragma unroll
  for (int mi = 0; mi < C::WT_M; ++mi)
#pragma unroll
    for (int gi = 0; gi < C::WT_G; ++gi) acc.v[mi][gi][0][0] = acc.v[mi][gi][0][1] = acc.v[mi][gi][1][0] = acc.v[mi][gi][1][1] = 0.0;
#pragma unroll
  for (int kb = 0; kb < NP / 8; ++kb) {
    double2 af[C::WT_M];
#pragma unroll
    for (int mi = 0; mi < C::WT_M; ++mi) {
      if constexpr (REGA) {
        af[mi] = fr->f[mi][kb];
      } else {
        const int r = (wm * C::WT_M + mi) * 8 + g;
        af[mi] = lds128(sP + 8u * (uint32_t)sidx<NP>(r, 8 * kb + 2 * c));
      }
    }
    double2 bf[C::WT_G][2];
#pragma unroll
    for (int gi = 0; gi < C::WT_G; ++gi)
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const int k = 8 * kb + 2 * c + s;
        bf[gi][s] = lds128(sQ + 8u * (uint32_t)sidx<NP>(k, (wg * C::WT_G + gi) * 16 + 2 * g));
      }
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int mi = 0; mi < C::WT_M; ++mi) {
        const double a = s ? af[mi].y : af[mi].x;
#pragma unroll
        for (int gi = 0; gi < C::WT_G; ++gi) {
          dmma(acc.v[mi][gi][0][0], acc.v[mi][gi][0][1], a, bf[gi][s].x);
          dmma(acc.v[mi][gi][1][0], acc.v[mi][gi][1][1], a, bf[gi][s].y);
        }
      }
  }
}

template <int NP>
__device__ __forceinline__ void load_mat(double* dst, const double* __restrict__ src, int n, int ld) {
  for (int i = threadIdx.x; i < NP * NP; i += blockDim.x) {
    const int r = i / NP, cc = i % NP;
    dst[sidx<NP>(r, cc)] = (r < n && cc < n) ? src[(long long)r * ld + cc] : 0.0;
  }
}

template <int NP>
__device__ __forceinline__ void store_mat(double* __restrict__ dst, const double* src, int n, int ld) {
  for (int i = threadIdx.x; i < n * n; i += blockDim.x) {
    const int r = i / n, cc = i % n;
    dst[(long long)r * ld + cc] = src[sidx<NP>(r, cc)];
  }
}

// K = F(Y) in registers.  inverse: W = B Y (to smem W, then one barrier), K = Y W;
// sqrt: K = -(Y Y) + A (A in `M`); exp: K = A Y.
template <int NP, bool REGA = false>
__device__ __forceinline__ void rhs_regs(int flow, const double* M, const double* Y, double* W, SmallAcc<NP>& K,
                                         const SmallAFrag<NP>* mfr = nullptr) {
  using C = SmallCfg<NP>;
  if (flow == 0) {
    SmallAcc<NP> w;
    smem_gemm<NP, REGA>(M, Y, w, mfr);
#pragma unroll
    for (int mi = 0; mi < C::WT_M; ++mi)
#pragma unroll
      for (int gi = 0; gi < C::WT_G; ++gi)
#pragma unroll
        for (int e = 0; e < 2; ++e) {   // columns 4c+2e (even n-tile) and 4c+2e+1 (odd): one 16-byte pair
          int r, cc;
          acc_pos<NP>(mi, gi, 0, e, r, cc);
          *reinterpret_cast<double2*>(W + sidx<NP>(r, cc)) = make_double2(w.v[mi][gi][0][e], w.v[mi][gi][1][e]);
        }
    __syncthreads();
    smem_gemm<NP>(Y, W, K);
  } else if (flow == 2) {   // exp: K = A Y
    smem_gemm<NP, REGA>(M, Y, K, mfr);
  } else {
    smem_gemm<NP>(Y, Y, K);
#pragma unroll
    for (int mi = 0; mi < C::WT_M; ++mi)
#pragma unroll
      for (int gi = 0; gi < C::WT_G; ++gi)
#pragma unroll
        for (int par = 0; par < 2; ++par)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            int r, cc;
            acc_pos<NP>(mi, gi, par, e, r, cc);
            K.v[mi][gi][par][e] = fma(-1.0, K.v[mi][gi][par][e], 1.0 * M[sidx<NP>(r, cc)]);
          }
  }
}

// ------------------------------------------------------------------------------------------------
// fine propagator: blockIdx.x = batch index z; slice input X0 = Uin + z*mstride, output Fout + z*mstride
// ------------------------------------------------------------------------------------------------
// m_F RK4 steps on the shared-memory state (sX) with X and S in registers; REGA: the constant left
// operand's fragments (mfr) come from registers
template <int NP, bool REGA>
__device__ __forceinline__ void fine_steps(int flow, const double* sM, double* sX, double* sYa, double* sYb, double* sW,
                                           int mF, double h, const SmallAFrag<NP>* mfr) {
  using C = SmallCfg<NP>;
  // X and S are touched element-wise only by the thread owning the element: they live in registers
  // (X is also the stage-1 GEMM operand, so its shared copy is refreshed at stage 4)
  SmallAcc<NP> xr, sr;
#pragma unroll
  for (int mi = 0; mi < C::WT_M; ++mi)
#pragma unroll
    for (int gi = 0; gi < C::WT_G; ++gi)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int r, cc;
        acc_pos<NP>(mi, gi, 0, e, r, cc);
        const double2 x = *reinterpret_cast<const double2*>(sX + sidx<NP>(r, cc));
        xr.v[mi][gi][0][e] = x.x;
        xr.v[mi][gi][1][e] = x.y;
        sr.v[mi][gi][0][e] = sr.v[mi][gi][1][e] = 0.0;
      }
  const double h6 = h / 6.0;
  for (int step = 0; step < mF; ++step) {
    for (int s = 1; s <= 4; ++s) {
      // Y_1 = X, Y_2 -> Ya, Y_3 -> Yb, Y_4 -> Ya (double-buffered: the epilogue never overwrites the
      // stage's own GEMM operand, so one barrier per stage suffices after it)
      const double* Yin = (s == 1) ? sX : (s == 3 ? sYb : sYa);
      double* Yout = (s == 4) ? sX : ((s == 2) ? sYb : sYa);
      SmallAcc<NP> K;
      rhs_regs<NP, REGA>(flow, sM, Yin, sW, K, mfr);
      const double cy = (s == 3) ? h : 0.5 * h;
#pragma unroll
      for (int mi = 0; mi < C::WT_M; ++mi)
#pragma unroll
        for (int gi = 0; gi < C::WT_G; ++gi)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            double out[2];
#pragma unroll
            for (int par = 0; par < 2; ++par) {
              const double k = K.v[mi][gi][par][e];
              double& x = xr.v[mi][gi][par][e];
              double& sv = sr.v[mi][gi][par][e];
              if (s == 4) {
                x = fma(h6, sv + k, x);
                out[par] = x;
              } else {
                sv = (s == 1) ? k : fma(2.0, k, sv);
                out[par] = fma(cy, k, x);
              }
            }
            int r, cc;
            acc_pos<NP>(mi, gi, 0, e, r, cc);
            *reinterpret_cast<double2*>(Yout + sidx<NP>(r, cc)) = make_double2(out[0], out[1]);
          }
      __syncthreads();
    }
  }
}

template <int NP>
__global__ void __launch_bounds__(kSmallThreads, 1)
    fine_smem_kernel(int flow, int n, int ld, const double* __restrict__ M, const double* __restrict__ Uin,
                     double* __restrict__ Fout, long long mstride, int mF, double h, const int* stop_flag) {
  using C = SmallCfg<NP>;
  if (cta_stop(stop_flag)) return;
  extern __shared__ double sm[];
  double* sM = sm;
  double* sX = sM + C::MAT;
  double* sYa = sX + C::MAT;
  double* sYb = sYa + C::MAT;
  double* sW = sYb + C::MAT;
  const int z = blockIdx.x;
  load_mat<NP>(sM, M, n, ld);
  load_mat<NP>(sX, Uin + z * mstride, n, ld);
  for (int i = threadIdx.x; i < C::MAT; i += blockDim.x) sYa[i] = sYb[i] = 0.0;
  __syncthreads();
  if (flow == 0 || flow == 2) {   // the constant left operand (B = I - A, or A) stays in registers
    SmallAFrag<NP> mfr;
    load_afrag<NP>(sM, mfr);
    fine_steps<NP, true>(flow, sM, sX, sYa, sYb, sW, mF, h, &mfr);
  } else {
    fine_steps<NP, false>(flow, sM, sX, sYa, sYb, sW, mF, h, nullptr);
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
      SmallAcc<NP> K;
      rhs_regs<NP>(flow, sM, X, sW, K);
      const bool last = (i == mG - 1);
      // Euler: g = X + h K into the OTHER buffer (sT/sV alternately): this step's GEMMs only read X,
      // and the previous step's reads of dst ended at its closing barrier
      double* dst = (X == sV) ? sT : sV;
#pragma unroll
      for (int mi = 0; mi < C::WT_M; ++mi)
#pragma unroll
        for (int gi = 0; gi < C::WT_G; ++gi)
#pragma unroll
          for (int par = 0; par < 2; ++par)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              int r, cc;
              acc_pos<NP>(mi, gi, par, e, r, cc);
              const int o = sidx<NP>(r, cc);
              const double g = fma(h, K.v[mi][gi][par][e], X[o]);
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
