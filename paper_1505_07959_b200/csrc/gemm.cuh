// FP64 DMMA GEMM for sm_100a with TMA-staged, 128B-swizzled tiles and fused parareal epilogues.
//
// Computes, for every batch index z of a launch, K_z = alpha * Aop_z * Bop_z (+ beta * C_z) on
// n x n row-major matrices and applies one of the epilogues of the parareal hot path
// (DESIGN.md "Kernels"):
//   EPI_STORE       D = K                                   (W = B Y: first GEMM of F(Y) = Y (B Y))
//   EPI_RK          classical-RK4 stage combination, s = 1..4 (reading R1):
//                     s=1: S = K;      Y' = X + (h/2) K
//                     s=2: S = S + 2K; Y' = X + (h/2) K
//                     s=3: S = S + 2K; Y' = X + h K
//                     s=4: X = X + (h/6) (S + K)   [S = ((k1 + 2k2) + 2k3) + k4]
//   EPI_EULER       g = X + h K -> Xout (and Gold if given)            (coarse step)
//   EPI_EULER_CORR  g = X + h K; U = Fk + (g - Gold); Gold = g          (eq. eqStepk+1; R3)
//   EPI_RESID       per-tile partial sum of (K - shift*I)^2             (residual norms)
//
// FP64 on B200 has no tcgen05 kind (ptxas rejects kind::f64) and no wgmma, so the tensor path is
// warp-level mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4, measured 37.0 TF/s chip peak).  Structure:
//   * persistent CTAs, static round-robin tile schedule over (z, grouped tile raster);
//   * one producer warp: one elected lane issues cp.async.bulk.tensor (TMA) loads of a
//     BM x 16 A tile and BN/16 16x16 B boxes per k-step into a STAGES-deep mbarrier ring,
//     128B swizzle (so fragment loads are bank-conflict free, see below);
//   * WARPS_M x WARPS_N consumer warps: register-resident accumulators (warp tile WM x WN),
//     fragments read with 128-bit ld.shared, 2 k-steps of DMMA per 16-byte fragment;
//   * epilogue straight from registers: each lane owns 4 consecutive columns of a row per 16-col
//     group, so stores are 2 x 16 B per (row, group); fused element-wise parareal arithmetic.
// Fragment/swizzle mapping (bank-conflict free for 128-bit loads):
//   A tile (row r, k) lives at r*128 + (((k>>1) ^ (r&7)) << 4) + (k&1)*8.  Lane (g=lane>>2, c=lane&3)
//   loads 16 B at chunk (4kb + c) of row 8mt + rho(g): values for k = 8kb+2c+s, s = 0,1.
//   rho = {0,4,1,5,2,6,3,7} puts the two rows of each quarter-warp in different swizzle halves.
//   B box (16 k-rows x 16 cols) at k*128 + (((j>>1) ^ (k&7)) << 4) + (j&1)*8: lane loads the
//   16 B pair (cols 2g, 2g+1) of row k = 8kb+2c+s, feeding two n-tiles (even / odd columns).
//   The k-order inside a 16-wide k-step is thus permuted identically for A and B (exact sums are
//   unchanged; the rounding order is fixed for a given n, independent of batch and slice).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "ptx.cuh"

namespace mfode {

enum Epi : int { EPI_STORE = 0, EPI_RK = 1, EPI_EULER = 2, EPI_EULER_CORR = 3, EPI_RESID = 4, EPI_ACCEL = 5 };

struct MatRef {           // element (z, r, c) at p[z * zstride + r * ld + c]
  double* p;
  long long zstride;
  __host__ __device__ double* at(int z) const { return p + (long long)z * zstride; }
};

struct GemmParams {
  int n, ld, num_z;
  int a_base, a_step;     // A-operand slice in its tensor map: a_base + z * a_step
  int b_base, b_step;     // B-operand slice: b_base + (z ^ b_xor) * b_step
  int b_xor;              // 1: pair sub-matrices (trig block flow: X' = A Y, Y' = -A X)
  int alt_sign;           // 1: odd z use -alpha
  int sym;                // 1: the result is symmetric (all operands polynomials in a symmetric A):
                          //    compute tiles with tile_m <= tile_n and mirror (f3, half the flops)
  double alpha, beta;     // K = alpha * acc + beta * C
  MatRef C;               // read iff beta != 0
  MatRef X_in, X_out, S, Y_out, F_in, Gold, U_out;
  int stage;              // RK stage 1..4
  double h;
  double shift;           // EPI_RESID: subtract shift * I
  double* partials;       // EPI_RESID: one double per tile (index z * tiles + tile)
  const int* stop_flag;   // if non-null and set: the launch does nothing
  int oz_reuse_left;      // emulated GEMM: A == the previous launch's right operand, unchanged (ozaki.cu)
  int oz_nmod;            // > 0: emulated FP64 GEMM on the int8 tensor cores with this many moduli (ozaki.cu)
};

}  // namespace mfode
#include "epilogue.cuh"   // epi_apply4 (needs GemmParams)
namespace mfode {

constexpr int BK = 16;    // k-depth of one pipeline stage (16 doubles = one 128-byte swizzle row)

template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES>
struct GemmCfg {
  static constexpr int kConsumerWarps = WARPS_M * WARPS_N;
  // Register budget: the register file is split over the 4 SM sub-partitions (16K regs each) and
  // warps are assigned round-robin, so 8 consumer warps + 1 producer warp (3 warps on one SMSP)
  // cap every thread at 168 registers.  The 8-warp config therefore uses a whole producer
  // warpgroup and setmaxnreg: producers drop to 40 registers, consumers grow to 232.
  static constexpr bool kSetMaxNReg = (kConsumerWarps % 4 == 0) && (kConsumerWarps >= 8);
  static constexpr int kProducerWarps = kSetMaxNReg ? 4 : 1;
  static constexpr int kThreads = (kConsumerWarps + kProducerWarps) * 32;
  static constexpr int WM = BM / WARPS_M;
  static constexpr int WN = BN / WARPS_N;
  static constexpr int MT = WM / 8;          // 8-row m-tiles per warp
  static constexpr int NG = WN / 16;         // 16-column groups per warp (2 n-tiles each)
  static constexpr int kABytes = BM * BK * 8;
  static constexpr int kBBytes = BN * BK * 8;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // symmetric mode: per consumer warp, an 8-row x 32-column staging block (x 2 output arrays) through
  // which the mirrored elements are written as 64-byte row segments
  static constexpr int kMirrorPitch = 33;
  static constexpr int kMirrorDoubles = (BM == BN) ? kConsumerWarps * 2 * 8 * kMirrorPitch : 0;
  // staged epilogue (128 x 128 tiles): the element-wise operands (C, X, S / Gold, F) of the next few
  // 4-column groups are copied global -> shared with cp.async while the current group is computed, in
  // per-warp slots [slot][array][lane][4] (12 KB per warp: 4 slots of 3 arrays, or 3 slots of 4); it
  // shares the area of the symmetric-mode mirror staging
  static constexpr bool kEpiStaged = (BM == 128 && BN == 128);
  static constexpr int kEpiWarpBytes = kEpiStaged ? 12 * 1024 : 0;
  static constexpr int kEpiDoubles = kConsumerWarps * kEpiWarpBytes / 8;
  static constexpr int kAuxDoubles = kMirrorDoubles > kEpiDoubles ? kMirrorDoubles : kEpiDoubles;
  static constexpr int kSmemBytes =
      STAGES * kStageBytes + 1024 /*align*/ + 2 * STAGES * 8 + 64 * 8 + kAuxDoubles * 8;
  static_assert(kSmemBytes <= 232448, "shared memory per CTA");
  static_assert(WM % 8 == 0 && WN % 16 == 0, "warp tile must be a multiple of 8 x 16");
  static_assert(BM <= 256 && BN % 16 == 0, "TMA box limits");
};

__device__ __forceinline__ int rho8(int g) { return ((g & 1) << 2) | (g >> 1); }

// tile index r -> (tile_m, tile_n): grouped raster, or over the upper triangle tile_m <= tile_n (sym).
// The grouped raster walks column-major inside bands of kGroupM tile rows, so the ~148 tiles in
// flight cover about 8 x 18 tiles instead of 4.6 rows x all columns: at each k-step they share
// fewer distinct A/B slabs, and fewer operand bytes are re-read from HBM once a batch exceeds L2.
constexpr int kGroupM = 8;
__device__ __forceinline__ void tile_coords(bool sym, int r, int tiles_m, int tiles_n, int& tm, int& tn) {
  if (!sym) {
    const int band = kGroupM * tiles_n;
    const int b = r / band;
    const int first = b * kGroupM;
    const int rows = (tiles_m - first) < kGroupM ? (tiles_m - first) : kGroupM;
    const int q = r - b * band;
    tn = q / rows;
    tm = first + (q - tn * rows);
    return;
  }
  tm = 0;
  while (r >= tiles_n - tm) {
    r -= tiles_n - tm;
    ++tm;
  }
  tn = tm + r;
}

template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES, int EPI>
__global__ void __launch_bounds__(GemmCfg<BM, BN, WARPS_M, WARPS_N, STAGES>::kThreads, 1)
    dgemm_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const GemmParams p) {
  using Cfg = GemmCfg<BM, BN, WARPS_M, WARPS_N, STAGES>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
  uint64_t* empty = full + STAGES;
  double* red = reinterpret_cast<double*>(empty + STAGES);   // EPI_RESID cross-warp scratch
  double* mirror_stage = red + 64;                            // symmetric-mode mirror staging

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n = p.n;
  const int tiles_m = (n + BM - 1) / BM;
  const int tiles_n = (n + BN - 1) / BN;
  // symmetric mode (f3): only tiles with tile_m <= tile_n; the epilogue mirrors them
  const bool sym = (BM == BN) && p.sym;
  const int tiles_per_z = sym ? tiles_m * (tiles_m + 1) / 2 : tiles_m * tiles_n;
  const int total = tiles_per_z * p.num_z;
  const int KT = (n + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::kConsumerWarps);
    }
    fence_barrier_init();
    fence_proxy_async();
  }
  __syncthreads();
  // PDL: let the next kernel of the stream start its prologue while this grid runs, then wait for
  // the previous grid (all of its writes visible) before touching global memory.
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (cta_stop(p.stop_flag)) return;

  if constexpr (Cfg::kSetMaxNReg) {
    if (warp >= Cfg::kConsumerWarps)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    else
      asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
  }

  if (warp >= Cfg::kConsumerWarps) {
    // ===================== TMA producer (one elected lane) =====================
    if (warp == Cfg::kConsumerWarps && lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int z = t / tiles_per_z;
        const int r = t - z * tiles_per_z;
        int tm_, tn_;
        tile_coords(sym, r, tiles_m, tiles_n, tm_, tn_);
        const int m0 = tm_ * BM;
        const int n0 = tn_ * BN;
        const int sa = p.a_base + z * p.a_step;
        const int sb = p.b_base + (z ^ p.b_xor) * p.b_step;
        // Epilogue operands of this tile (X, S, C, F, Gold rows) are prefetched into L2 during the
        // last k-steps, so the fused epilogue reads L2 instead of stalling every warp on HBM.
        const int pf_k0 = KT > 8 ? KT - 8 : 0;
        const int pf_bytes = (((n - n0) < BN ? (n - n0) : BN) * 8 + 15) & ~15;
        const long long zoff = (long long)z;
        for (int kt = 0; kt < KT; ++kt) {
          if (kt >= pf_k0) {
            const int per = (BM + (KT - pf_k0) - 1) / (KT - pf_k0);
            const int r0 = (kt - pf_k0) * per;
            const int r1 = (r0 + per < BM) ? r0 + per : BM;
            for (int rr = r0; rr < r1 && m0 + rr < n; ++rr) {
              const long long off = (long long)(m0 + rr) * p.ld + n0;
              if (p.beta != 0.0) prefetch_l2(p.C.at((int)zoff) + off, pf_bytes);
              if constexpr (EPI == EPI_RK || EPI == EPI_EULER || EPI == EPI_EULER_CORR || EPI == EPI_ACCEL)
                prefetch_l2(p.X_in.at((int)zoff) + off, pf_bytes);
              if constexpr (EPI == EPI_RK) {
                if (p.stage > 1) prefetch_l2(p.S.at((int)zoff) + off, pf_bytes);
              }
              if constexpr (EPI == EPI_ACCEL) {
                if ((z & 1) == 0) prefetch_l2(p.S.at((int)zoff) + off, pf_bytes);
              }
              if constexpr (EPI == EPI_EULER_CORR) {
                prefetch_l2(p.F_in.at((int)zoff) + off, pf_bytes);
                prefetch_l2(p.Gold.at((int)zoff) + off, pf_bytes);
              }
            }
          }
          mbar_wait(&empty[stage], phase ^ 1);
          unsigned char* sA = smem + stage * Cfg::kStageBytes;
          unsigned char* sB = sA + Cfg::kABytes;
          mbar_arrive_expect_tx(&full[stage], Cfg::kStageBytes);
          tma_load_3d(sA, &tmA, &full[stage], kt * BK, m0, sa);
#pragma unroll
          for (int g = 0; g < BN / 16; ++g) tma_load_3d(sB + g * 2048, &tmB, &full[stage], n0 + g * 16, kt * BK, sb);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    return;
  }

  // ===================== consumers: DMMA main loop + fused epilogue =====================
  const int wm = warp / WARPS_N;
  const int wn = warp % WARPS_N;
  const int g = lane >> 2;
  const int c = lane & 3;
  const int rowA = rho8(g);
  int stage = 0;
  uint32_t phase = 0;
  const uint32_t smem_base = smem_u32(smem);

  for (int t = blockIdx.x; t < total; t += gridDim.x) {
    const int z = t / tiles_per_z;
    const int r = t - z * tiles_per_z;
    int tm_, tn_;
    tile_coords(sym, r, tiles_m, tiles_n, tm_, tn_);
    const int m0 = tm_ * BM;
    const int n0 = tn_ * BN;
    const double alpha = (p.alt_sign && (z & 1)) ? -p.alpha : p.alpha;

    double acc[Cfg::MT][2 * Cfg::NG][2];
#pragma unroll
    for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
      for (int j = 0; j < 2 * Cfg::NG; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    // staged epilogue (see GemmCfg): the first D groups' operands are requested when the main loop ends
    constexpr bool kStaged =
        Cfg::kEpiStaged && (EPI == EPI_RK || EPI == EPI_EULER || EPI == EPI_EULER_CORR || EPI == EPI_ACCEL);
    constexpr int NA = (EPI == EPI_EULER_CORR) ? 4 : 3;          // arrays per slot: C, X, S (/ Gold), F
    // NSLOT slots per warp, D = NSLOT - 1 groups in flight: the slot a new copy targets was read one
    // group earlier, never by the group just processed
    constexpr int NSLOT = kStaged ? Cfg::kEpiWarpBytes / (NA * 1024) : 2;
    constexpr int D = NSLOT - 1;
    constexpr int NGR = Cfg::MT * Cfg::NG;
    // (recomputed where used rather than held in registers across the main loop)
    auto use_c = [&] { return p.beta != 0.0; };
    auto use_s = [&] {
      return (EPI == EPI_EULER_CORR) || (EPI == EPI_RK && p.stage > 1) || (EPI == EPI_ACCEL && (z & 1) == 0);
    };
    auto slot_addr = [&](int gi) {
      return smem_u32(mirror_stage) + (uint32_t)warp * (uint32_t)Cfg::kEpiWarpBytes +
             (uint32_t)(((gi % NSLOT) * NA * 128 + lane * 4) * 8);
    };
    auto issue = [&](int gi) {
      if (gi < NGR) {
        const int mt = gi / Cfg::NG, ng = gi % Cfg::NG;
        const int row = m0 + wm * Cfg::WM + mt * 8 + rowA;
        const int col = n0 + wn * Cfg::WN + ng * 16 + 4 * c;
        if (row < n && col + 3 < n) {
          const long long off = (long long)row * p.ld + col;
          const uint32_t d = slot_addr(gi);
          if (use_c()) {
            const double* src = p.C.at(z) + off;
            cp_async16(d, src);
            cp_async16(d + 16, src + 2);
          }
          const double* sx = p.X_in.at(z) + off;
          cp_async16(d + 1024, sx);
          cp_async16(d + 1024 + 16, sx + 2);
          if (use_s() && EPI != EPI_EULER_CORR) {
            const double* ss = p.S.at(z) + off;
            cp_async16(d + 2048, ss);
            cp_async16(d + 2048 + 16, ss + 2);
          }
          if constexpr (EPI == EPI_EULER_CORR) {
            const double* sf = p.F_in.at(z) + off;
            cp_async16(d + 3072, sf);
            cp_async16(d + 3072 + 16, sf + 2);
          }
        }
      }
      cp_async_commit();   // (empty groups keep the count uniform)
    };
    bool ready = false;   // full[stage] already observed complete by the early probe
    for (int kt = 0; kt < KT; ++kt) {
      if (!ready) mbar_wait(&full[stage], phase);
      const uint32_t sA = smem_base + stage * Cfg::kStageBytes;
      const uint32_t sB = sA + Cfg::kABytes;
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        double2 af[Cfg::MT];
#pragma unroll
        for (int mt = 0; mt < Cfg::MT; ++mt) {
          const int row = wm * Cfg::WM + mt * 8 + rowA;   // row & 7 == rowA
          af[mt] = lds128(sA + row * 128 + ((((kb << 2) + c) ^ rowA) << 4));
        }
        double2 bf[Cfg::NG][2];
#pragma unroll
        for (int ng = 0; ng < Cfg::NG; ++ng) {
          const int grp = (wn * Cfg::WN) / 16 + ng;
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const int k = kb * 8 + 2 * c + s;
            bf[ng][s] = lds128(sB + grp * 2048 + k * 128 + ((g ^ (k & 7)) << 4));
          }
        }
        if (kb == 1) {
          // Probe the next stage's full barrier now, so the probe's latency hides behind this
          // k-step's DMMAs instead of stalling the next one.
          const int ns = (stage + 1 == STAGES) ? 0 : stage + 1;
          ready = (kt + 1 < KT) && mbar_test_wait(&full[ns], ns == 0 ? (phase ^ 1) : phase);
        }
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
          for (int mt = 0; mt < Cfg::MT; ++mt) {
            const double a = s ? af[mt].y : af[mt].x;
#pragma unroll
            for (int ng = 0; ng < Cfg::NG; ++ng) {
              dmma(acc[mt][2 * ng][0], acc[mt][2 * ng][1], a, bf[ng][s].x);
              dmma(acc[mt][2 * ng + 1][0], acc[mt][2 * ng + 1][1], a, bf[ng][s].y);
            }
          }
      }
      // Release the stage to the producer once the DMMAs that consume its fragments are issued: a
      // DMMA issues only after its source registers are written, so every shared-memory read of the
      // stage by this warp has completed and the TMA (async-proxy) refill cannot race it.  (Releasing
      // right after the last ld.shared, with reads still in flight, needs a proxy fence -- without
      // one, rare wrong 32 x 16 warp sub-tiles were seen -- and the fence's wait costs more: same-box
      // A/B 34.63 -> 34.72 TF/s per RK stage at n = 4096, profiles/ab_gemm_late_release_r02.jsonl.)
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }

    // ---------------- epilogue ----------------
    double part = 0.0;
    const int ld = p.ld;
    if constexpr (EPI != EPI_RESID && BM == BN) {
      if (sym) {
        // symmetric mode: direct (upper) stores in the epilogue; the mirrors go through a per-warp
        // 8 x 32 staging block so that each lane writes 8 consecutive doubles of one target row
        double* stg = mirror_stage + warp * (2 * 8 * Cfg::kMirrorPitch);
        double* outp[2];
        epi_out_ptrs<EPI>(p, z, outp);
#pragma unroll
        for (int mt = 0; mt < Cfg::MT; ++mt) {
          const int row = m0 + wm * Cfg::WM + mt * 8 + rowA;
#pragma unroll
          for (int ng = 0; ng < Cfg::NG; ++ng) {
            const int cl = ng * 16 + 4 * c;
            const int col = n0 + wn * Cfg::WN + cl;
            double mv[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
            double* mp[2];
            if (row < n && col < n) {
              double k4[4] = {acc[mt][2 * ng][0], acc[mt][2 * ng + 1][0], acc[mt][2 * ng][1], acc[mt][2 * ng + 1][1]};
              epi_apply4_impl<EPI, true>(p, z, alpha, row, col, n, ld, k4, true, m0 == n0, part, mv, mp);
            }
#pragma unroll
            for (int sl = 0; sl < 2; ++sl)
#pragma unroll
              for (int e = 0; e < 4; ++e) stg[sl * 8 * Cfg::kMirrorPitch + rowA * Cfg::kMirrorPitch + cl + e] = mv[sl][e];
          }
          __syncwarp();
          const int tr = n0 + wn * Cfg::WN + lane;        // target row = source column
          const int tc0 = m0 + wm * Cfg::WM + mt * 8;     // target columns = the 8 source rows
          if (tr < n) {
#pragma unroll
            for (int sl = 0; sl < 2; ++sl) {
              if (outp[sl] == nullptr) continue;
              double v[8];
              bool all = true;
#pragma unroll
              for (int r = 0; r < 8; ++r) {
                v[r] = stg[sl * 8 * Cfg::kMirrorPitch + r * Cfg::kMirrorPitch + lane];
                all = all && (tc0 + r < n) && (tc0 + r < tr);
              }
              double* dst = outp[sl] + (long long)tr * ld + tc0;
              if (all) {
#pragma unroll
                for (int r = 0; r < 8; r += 2) *reinterpret_cast<double2*>(dst + r) = make_double2(v[r], v[r + 1]);
              } else {
#pragma unroll
                for (int r = 0; r < 8; ++r)
                  if ((tc0 + r < n) && (tc0 + r < tr)) dst[r] = v[r];
              }
            }
          }
          __syncwarp();
        }
        continue;
      }
    }
    if constexpr (kStaged) {
      // staged epilogue: the operands of groups gi + 1 .. gi + D are in flight (cp.async into this
      // warp's slots) while group gi is computed and stored, so the L2 latency of the loads is not paid
      // once per group (the compiler cannot hoist the next group's global loads above this group's
      // stores, which might alias them).  Ragged groups load inline.  Measured hazards shaped it
      // (profiles/staged_epilogue_r02.md):
      //   * a slot is refilled only one group after it was read (refilling the slot just read left one
      //     wrong solve in eight at n = 4096, none in 29 reruns after the change);
      //   * the first copies are issued when the main loop ends, not during its last k-steps: issued
      //     2 k-steps early, the correction's Gold (read, then overwritten in place by this epilogue)
      //     came back wrong in a few 64 x 32 warp sub-tiles of nearly every n >= 3072 solve, for a
      //     reason not identified (issued after the loop: 6 of 6 right); the early issue was worth
      //     only 0.15 %;
      //   * belt and braces, the correction's Gold is not staged at all (~2 % of a solve).
      const int ld = p.ld;
#pragma unroll
      for (int gi = 0; gi < D; ++gi) issue(gi);
#pragma unroll
      for (int gi = 0; gi < NGR; ++gi) {
        const int mt = gi / Cfg::NG, ng = gi % Cfg::NG;
        const int row = m0 + wm * Cfg::WM + mt * 8 + rowA;
        const int col = n0 + wn * Cfg::WN + ng * 16 + 4 * c;
        cp_async_wait<D - 1>();   // group gi has landed (this lane's own copies)
        if (row < n && col < n) {
          double k4[4] = {acc[mt][2 * ng][0], acc[mt][2 * ng + 1][0], acc[mt][2 * ng][1], acc[mt][2 * ng + 1][1]};
          double mv[2][4];
          double* mp[2];
          if (col + 3 < n) {
            const uint32_t d = slot_addr(gi);
            EpiIn in;
            double2 v0, v1;
            if (use_c()) {
              v0 = lds128(d); v1 = lds128(d + 16);
              in.c[0] = v0.x; in.c[1] = v0.y; in.c[2] = v1.x; in.c[3] = v1.y;
            }
            v0 = lds128(d + 1024); v1 = lds128(d + 1024 + 16);
            in.x[0] = v0.x; in.x[1] = v0.y; in.x[2] = v1.x; in.x[3] = v1.y;
            if (EPI == EPI_EULER_CORR) {
              // the correction's Gold is loaded here, not staged (see above)
              const double* gp = p.Gold.at(z) + (long long)row * ld + col;
              const double2 g0 = *reinterpret_cast<const double2*>(gp);
              const double2 g1 = *reinterpret_cast<const double2*>(gp + 2);
              in.s[0] = g0.x; in.s[1] = g0.y; in.s[2] = g1.x; in.s[3] = g1.y;
            } else if (use_s()) {
              v0 = lds128(d + 2048); v1 = lds128(d + 2048 + 16);
              in.s[0] = v0.x; in.s[1] = v0.y; in.s[2] = v1.x; in.s[3] = v1.y;
            }
            if constexpr (EPI == EPI_EULER_CORR) {
              v0 = lds128(d + 3072); v1 = lds128(d + 3072 + 16);
              in.f[0] = v0.x; in.f[1] = v0.y; in.f[2] = v1.x; in.f[3] = v1.y;
            }
            epi_apply4_impl<EPI, false, true>(p, z, alpha, row, col, n, ld, k4, false, false, part, mv, mp, &in);
          } else {
            epi_apply4_impl<EPI, false>(p, z, alpha, row, col, n, ld, k4, false, false, part, mv, mp);
          }
        }
        issue(gi + D);
      }
    } else if constexpr (EPI != EPI_RESID) {
      // epilogue over the flattened groups g = mt * NG + ng (guarded, no early exits).  EPI_STORE
      // (W = B Y) runs the software-pipelined form (operands of group g + 1 loaded before group g is
      // stored); the other epilogues keep their loads inline -- pipelining them raises register
      // pressure past the 232-register budget of the 128 x 128 consumers without a measurable gain.
      EpiIn buf[2];
      if constexpr (EPI == EPI_STORE) {
        const int row = m0 + wm * Cfg::WM + rowA, col = n0 + wn * Cfg::WN + 4 * c;
        if (row < n && col < n) epi_load4<EPI>(p, z, row, col, n, ld, buf[0]);
      }
#pragma unroll
      for (int gi = 0; gi < Cfg::MT * Cfg::NG; ++gi) {
        const int mt = gi / Cfg::NG, ng = gi % Cfg::NG;
        if constexpr (EPI == EPI_STORE) {
          if (gi + 1 < Cfg::MT * Cfg::NG) {
            const int mt1 = (gi + 1) / Cfg::NG, ng1 = (gi + 1) % Cfg::NG;
            const int row1 = m0 + wm * Cfg::WM + mt1 * 8 + rowA, col1 = n0 + wn * Cfg::WN + ng1 * 16 + 4 * c;
            if (row1 < n && col1 < n) epi_load4<EPI>(p, z, row1, col1, n, ld, buf[(gi + 1) & 1]);
          }
        }
        const int row = m0 + wm * Cfg::WM + mt * 8 + rowA;
        const int col = n0 + wn * Cfg::WN + ng * 16 + 4 * c;
        if (row < n && col < n) {
          double k4[4] = {acc[mt][2 * ng][0], acc[mt][2 * ng + 1][0], acc[mt][2 * ng][1], acc[mt][2 * ng + 1][1]};
          double mv[2][4];
          double* mp[2];
          epi_apply4_impl<EPI, false, EPI == EPI_STORE>(p, z, alpha, row, col, n, ld, k4, false, false, part, mv, mp,
                                                         &buf[gi & 1]);
        }
      }
    } else {
#pragma unroll
    for (int mt = 0; mt < Cfg::MT; ++mt) {
      const int row = m0 + wm * Cfg::WM + mt * 8 + rowA;
      if (row >= n) continue;
#pragma unroll
      for (int ng = 0; ng < Cfg::NG; ++ng) {
        const int col = n0 + wn * Cfg::WN + ng * 16 + 4 * c;
        if (col >= n) continue;
        double k4[4] = {acc[mt][2 * ng][0], acc[mt][2 * ng + 1][0], acc[mt][2 * ng][1], acc[mt][2 * ng + 1][1]};
        epi_apply4<EPI>(p, z, alpha, row, col, n, ld, k4, sym, m0 == n0, part);
      }
    }
    }
    if constexpr (EPI == EPI_RESID) {
      // deterministic tile reduction: fixed shuffle tree, then warps in index order
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      named_bar_sync(1, Cfg::kConsumerWarps * 32);
      if (lane == 0) red[warp] = part;
      named_bar_sync(1, Cfg::kConsumerWarps * 32);
      if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < Cfg::kConsumerWarps; ++w) s += red[w];
        p.partials[t] = s;
      }
    }
  }
}

}  // namespace mfode
