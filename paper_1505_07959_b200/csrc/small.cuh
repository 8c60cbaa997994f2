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
// K6c: one slice's fine propagation spread over a cluster of CS CTAs (one per SM), column-split.
//
// CTA q of the cluster owns a set of output columns (NP/CS of them) of every GEMM and of the RK state.
// A column split keeps most of each stage local: W[:, own] = B Y[:, own] needs only the own columns
// of Y, the stage combination and the RK state (X, S) are element-wise, and only the A-role operand of
// K = Y W (inverse flow) or Y Y (sqrt flow) needs every column of Y.  So each stage exchanges its new
// Y once: every thread pushes its own elements of Y_out into the other CTAs' copies with
// st.async ... mbarrier::complete_tx (DSMEM stores that count bytes on the receiver's mbarrier), and
// the receiver waits for (CS-1) x NP x NP/CS x 8 bytes just before the GEMM that needs them -- for the
// inverse flow after W = B Y[:, own], so the exchange latency hides under that GEMM.  The exp flow
// (K = A Y[:, own]) is column-local and exchanges nothing.
//
// Per output element the DMMA sequence (k = 8 kb + 2 c + s, kb-major) is the one of smem_gemm and
// gemm.cuh, so results are bitwise identical to fine_smem_kernel and to the launch-per-GEMM path.
//
// Exchange t (the Y_out of global stage t = 4 step + s - 1) lands on xbar[t & 1].  A CTA can run at
// most one exchange ahead of any other (its stage t+1 GEMM waits for exchange t from everyone), so two
// alternating barriers keep every phase unambiguous; every write into a peer's buffer Y_out(t) happens
// after the peer's threads all finished reading it as Y_in(t-1) (the peer's exchange t-1 bytes, sent by
// each thread after its own stage t-1 GEMMs, had to arrive first).
// ------------------------------------------------------------------------------------------------
template <int NP, int CS>
struct ClusterCfg {
  static constexpr int MAT = NP * NP;
  static constexpr int NPC = NP / CS;                   // columns owned by one CTA
  static constexpr bool PSPLIT = (NPC == 8);            // a CTA owns one parity n-tile of a 16-column group
  static constexpr int GC = PSPLIT ? 1 : NPC / 16;      // 16-column groups per CTA
  static constexpr int NPAR = PSPLIT ? 1 : 2;           // n-tiles per group held by a thread
  static constexpr int MT = NP / 8;                     // m-tiles
  static constexpr int UNITS = MT * GC;
  static constexpr int WARPS = UNITS < 8 ? UNITS : 8;
  static constexpr int WARPS_G = GC;
  static constexpr int WARPS_M = WARPS / WARPS_G;
  static constexpr int WT_M = MT / WARPS_M;
  static constexpr int THREADS = 32 * WARPS;
  static constexpr uint32_t XBYTES = (uint32_t)(CS - 1) * NP * NPC * 8;   // received per exchange
  static_assert(NPC >= 8 && NP % CS == 0 && WARPS % WARPS_G == 0 && MT % WARPS_M == 0, "cluster split");
};

template <int NP, int CS>
struct ClAcc {
  double v[ClusterCfg<NP, CS>::WT_M][ClusterCfg<NP, CS>::NPAR][2];   // [m-tile][n-tile][e]
};

template <int NP, int CS>
struct ClAFrag {
  double2 f[ClusterCfg<NP, CS>::WT_M][NP / 8];
};

// owner coordinates of this thread: first row of m-tile mi is 8 (wm WT_M + mi); the thread's columns
// are 16 grp + 4 c + 2 e + par(p)
template <int NP, int CS>
struct ClPos {
  int wm, grp, par0, g, c;
  __device__ __forceinline__ ClPos(uint32_t q) {
    using C = ClusterCfg<NP, CS>;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    wm = warp / C::WARPS_G;
    const int wg = warp % C::WARPS_G;
    grp = C::PSPLIT ? (int)(q >> 1) : (int)q * C::GC + wg;
    par0 = C::PSPLIT ? (int)(q & 1) : 0;
    g = lane >> 2;
    c = lane & 3;
  }
  __device__ __forceinline__ int row(int mi) const { return (wm * ClusterCfg<NP, CS>::WT_M + mi) * 8 + g; }
  __device__ __forceinline__ int col(int p, int e) const { return 16 * grp + 4 * c + 2 * e + par0 + p; }
};

__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(cta));
  return r;
}
// DSMEM store into a peer CTA counted as transaction bytes on the peer's mbarrier (both addresses
// already mapped to the peer)
__device__ __forceinline__ void st_async_v2(uint32_t raddr, double a, double b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(raddr),
               "d"(a), "d"(b), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_1(uint32_t raddr, double a, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(raddr), "d"(a),
               "r"(rbar)
               : "memory");
}
__device__ __forceinline__ int ld_cluster_s32(uint32_t raddr) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];\n" : "=r"(v) : "r"(raddr) : "memory");
  return v;
}

// acc = P[own rows, :] * Q[:, own columns]; P from smem or (REGA) register fragments
template <int NP, int CS, bool REGA>
__device__ __forceinline__ void cl_gemm(const ClPos<NP, CS>& o, const double* __restrict__ P,
                                        const double* __restrict__ Q, ClAcc<NP, CS>& acc,
                                        const ClAFrag<NP, CS>* fr) {
  using C = ClusterCfg<NP, CS>;
  const uint32_t sP = smem_u32(P), sQ = smem_u32(Q);
#pragma unroll
  for (int mi = 0; mi < C::WT_M; ++mi)
#pragma unroll
    for (int p = 0; p < C::NPAR; ++p) acc.v[mi][p][0] = acc.v[mi][p][1] = 0.0;
#pragma unroll
  for (int kb = 0; kb < NP / 8; ++kb) {
    double2 af[C::WT_M];
#pragma unroll
    for (int mi = 0; mi < C::WT_M; ++mi) {
      if constexpr (REGA) {
        af[mi] = fr->f[mi][kb];
      } else {
        af[mi] = lds128(sP + 8u * (uint32_t)sidx<NP>(o.row(mi), 8 * kb + 2 * o.c));
      }
    }
    double bf[2][C::NPAR];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const int k = 8 * kb + 2 * o.c + s;
      if constexpr (C::PSPLIT) {
        bf[s][0] = lds64(sQ + 8u * (uint32_t)sidx<NP>(k, 16 * o.grp + 2 * o.g + o.par0));
      } else {
        const double2 b = lds128(sQ + 8u * (uint32_t)sidx<NP>(k, 16 * o.grp + 2 * o.g));
        bf[s][0] = b.x;
        bf[s][1] = b.y;
      }
    }
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
      for (int mi = 0; mi < C::WT_M; ++mi) {
        const double a = s ? af[mi].y : af[mi].x;
#pragma unroll
        for (int p = 0; p < C::NPAR; ++p) dmma(acc.v[mi][p][0], acc.v[mi][p][1], a, bf[s][p]);
      }
  }
}

// tools/k6c_probe.cu defines K6C_PROF to timestamp the phases of a few stages (not in the library)
#ifdef K6C_PROF
__device__ long long g_k6c_prof[2][16][8];
#define K6C_MARK(i)                                                                              \
  if (blockIdx.x < 2 && threadIdx.x == 0 && t >= 200 && t < 216) g_k6c_prof[blockIdx.x][t - 200][i] = clock64();
#else
#define K6C_MARK(i)
#endif

template <int NP, int CS>
__global__ void __launch_bounds__(ClusterCfg<NP, CS>::THREADS, 1)
    fine_cluster_kernel(int flow, int n, int ld, const double* __restrict__ M, const double* __restrict__ Uin,
                        double* __restrict__ Fout, long long mstride, int mF, double h, const int* stop_flag) {
  using C = ClusterCfg<NP, CS>;
  extern __shared__ double sm[];
  __shared__ __align__(8) uint64_t xbar[2];
  __shared__ int s_stop;
  double* sM = sm;
  double* sX = sM + C::MAT;
  double* sYa = sX + C::MAT;
  double* sYb = sYa + C::MAT;
  double* sW = sYb + C::MAT;
  const uint32_t q = cluster_ctarank();
  const int z = blockIdx.x / CS;
  if (threadIdx.x == 0) {
    s_stop = (stop_flag != nullptr && *(volatile const int*)stop_flag != 0) ? 1 : 0;
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    fence_barrier_init();
  }
  cluster_sync_all();
  // the cluster follows rank 0's reading of the (concurrently written) stop flag
  const bool stop = ld_cluster_s32(mapa_u32(smem_u32(&s_stop), 0)) != 0;
  if (!stop) {
    load_mat<NP>(sM, M, n, ld);
    load_mat<NP>(sX, Uin + z * mstride, n, ld);
    for (int i = threadIdx.x; i < C::MAT; i += blockDim.x) sYa[i] = sYb[i] = sW[i] = 0.0;
    __syncthreads();
    const ClPos<NP, CS> o(q);
    const bool xchg = (flow != 2);   // exp: K = A Y[:, own] is column-local
    ClAFrag<NP, CS> mfr;             // the constant left operand (B or A) as register fragments
    if (flow == 0 || flow == 2) {
#pragma unroll
      for (int mi = 0; mi < C::WT_M; ++mi)
#pragma unroll
        for (int kb = 0; kb < NP / 8; ++kb)
          mfr.f[mi][kb] = *reinterpret_cast<const double2*>(sM + sidx<NP>(o.row(mi), 8 * kb + 2 * o.c));
    }
    ClAcc<NP, CS> xr, sr;
#pragma unroll
    for (int mi = 0; mi < C::WT_M; ++mi)
#pragma unroll
      for (int p = 0; p < C::NPAR; ++p)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          xr.v[mi][p][e] = sX[sidx<NP>(o.row(mi), o.col(p, e))];
          sr.v[mi][p][e] = 0.0;
        }
    // peer CTAs' shared-memory windows (same dynamic-smem offsets in every CTA of the cluster)
    uint32_t rsm[CS > 1 ? CS - 1 : 1], rbar[CS > 1 ? CS - 1 : 1];
#pragma unroll
    for (int r = 1; r < CS; ++r) {
      rsm[r - 1] = mapa_u32(smem_u32(sm), (q + r) % CS);
      rbar[r - 1] = mapa_u32(smem_u32(&xbar[0]), (q + r) % CS);
    }
    const double h6 = h / 6.0;
    const int nT = 4 * mF;
    for (int t = 0; t < nT; ++t) {
      const int s = (t & 3) + 1;
      const double* Yin = (s == 1) ? sX : (s == 3 ? sYb : sYa);
      double* Yout = (s == 4) ? sX : ((s == 2) ? sYb : sYa);
      const bool send = xchg && (t + 1 < nT);
      K6C_MARK(0);
      if (send && threadIdx.x == 0) mbar_arrive_expect_tx(&xbar[t & 1], C::XBYTES);
      ClAcc<NP, CS> K;
      if (flow == 0) {   // W[:, own] = B Y[:, own] (local), then K = Y W[:, own] (needs all of Y)
        ClAcc<NP, CS> w;
        cl_gemm<NP, CS, true>(o, sM, Yin, w, &mfr);
        K6C_MARK(1);
#pragma unroll
        for (int mi = 0; mi < C::WT_M; ++mi)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            if constexpr (C::NPAR == 2) {   // columns (par 0, par 1) are one 16-byte pair
              *reinterpret_cast<double2*>(sW + sidx<NP>(o.row(mi), o.col(0, e))) =
                  make_double2(w.v[mi][0][e], w.v[mi][1][e]);
            } else {
              sW[sidx<NP>(o.row(mi), o.col(0, e))] = w.v[mi][0][e];
            }
          }
        __syncthreads();
        K6C_MARK(2);
        if (t > 0) mbar_wait(&xbar[(t - 1) & 1], ((t - 1) >> 1) & 1);
        K6C_MARK(3);
        cl_gemm<NP, CS, false>(o, Yin, sW, K, nullptr);
        K6C_MARK(4);
      } else if (flow == 2) {   // exp: K = A Y[:, own]
        cl_gemm<NP, CS, true>(o, sM, Yin, K, &mfr);
      } else {                  // sqrt: K = -(Y Y[:, own]) + A[:, own]
        if (t > 0) mbar_wait(&xbar[(t - 1) & 1], ((t - 1) >> 1) & 1);
        cl_gemm<NP, CS, false>(o, Yin, Yin, K, nullptr);
#pragma unroll
        for (int mi = 0; mi < C::WT_M; ++mi)
#pragma unroll
          for (int p = 0; p < C::NPAR; ++p)
#pragma unroll
            for (int e = 0; e < 2; ++e)
              K.v[mi][p][e] = fma(-1.0, K.v[mi][p][e], 1.0 * sM[sidx<NP>(o.row(mi), o.col(p, e))]);
      }
      // RK stage combination on the owned elements (epilogue.cuh EPI_RK arithmetic), new Y to the
      // local copy and to every peer
      const double cy = (s == 3) ? h : 0.5 * h;
      const uint32_t yoff = 8u * (uint32_t)(Yout - sm), boff = 8u * (uint32_t)(t & 1);
#pragma unroll
      for (int mi = 0; mi < C::WT_M; ++mi)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double out[C::NPAR];
#pragma unroll
          for (int p = 0; p < C::NPAR; ++p) {
            const double k = K.v[mi][p][e];
            double& x = xr.v[mi][p][e];
            double& sv = sr.v[mi][p][e];
            if (s == 4) {
              x = fma(h6, sv + k, x);
              out[p] = x;
            } else {
              sv = (s == 1) ? k : fma(2.0, k, sv);
              out[p] = fma(cy, k, x);
            }
          }
          const uint32_t off = 8u * (uint32_t)sidx<NP>(o.row(mi), o.col(0, e));
          if constexpr (C::NPAR == 2) {
            *reinterpret_cast<double2*>(Yout + off / 8) = make_double2(out[0], out[1]);
          } else {
            Yout[off / 8] = out[0];
          }
          if (send) {
#pragma unroll
            for (int r = 0; r < CS - 1; ++r) {
              if constexpr (C::NPAR == 2) {
                st_async_v2(rsm[r] + yoff + off, out[0], out[1], rbar[r] + boff);
              } else {
                st_async_1(rsm[r] + yoff + off, out[0], rbar[r] + boff);
              }
            }
          }
        }
      K6C_MARK(5);
      __syncthreads();
      K6C_MARK(6);
    }
    // result: the owned columns straight from the registers
#pragma unroll
    for (int mi = 0; mi < C::WT_M; ++mi)
#pragma unroll
      for (int p = 0; p < C::NPAR; ++p)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int r = o.row(mi), cc = o.col(p, e);
          if (r < n && cc < n) Fout[z * mstride + (long long)r * ld + cc] = xr.v[mi][p][e];
        }
  }
  cluster_sync_all();   // no CTA leaves while a peer may still touch its shared memory
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
    // the correction's F(U^k_j) and G(U^k_j) terms do not depend on this slice's GEMMs: load them first
    // so their global latency hides under the coarse step
    SmallAcc<NP> fk, gold;
    if (correct) {
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
              const bool in = r < n && cc < n;
              const long long go = (long long)j * mstride + (long long)r * ld + cc;
              fk.v[mi][gi][par][e] = in ? Fk[go] : 0.0;
              gold.v[mi][gi][par][e] = in ? Gold[go] : 0.0;
            }
    }
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
                  u = fk.v[mi][gi][par][e] + (g - gold.v[mi][gi][par][e]);
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
