// EXPERIMENT (round 2, not built into libmfode.so): measured slower than gemm.cuh, see DESIGN.md §14.
// K1p: "ping-pong" variant of the FP64 DMMA GEMM (gemm.cuh) for large n, non-symmetric launches.
//
// gemm.cuh's 128 x 128 CTA keeps the DMMA pipe ~95 % busy; the rest is its fused epilogue (X, S loads,
// S, Y stores of the finished tile), during which all eight consumer warps stop issuing DMMAs.  Here
// the CTA holds TWO consumer groups of four warps, each with its own 64 x 128 tile, its own TMA
// producer thread and its own 4-stage ring, and the groups take turns on the tensor pipe: an order
// barrier lets only one group run its main loop at a time, so group A's epilogue runs while group B's
// main loop owns the DMMA pipe (one warp per SM sub-partition issues one DMMA per 16 cycles with 32
// independent accumulators, enough to keep the pipe full).
// Per warp the tile is the same 64 x 32 as gemm.cuh's (same registers, fragment mapping, k order and
// epilogue code), so every output element is bitwise identical to the 128 x 128 kernel's.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "gemm.cuh"
#include "ptx.cuh"

namespace mfode {

struct PPCfg {
  static constexpr int BM = 64, BN = 128, STAGES = 4, GROUPS = 2;
  static constexpr int kGroupWarps = 4;                        // consumer warps per group (1 x 4)
  static constexpr int kConsumerWarps = GROUPS * kGroupWarps;  // 8
  static constexpr int kThreads = (kConsumerWarps + 4) * 32;   // + producer warpgroup = 384
  static constexpr int WM = 64, WN = 32, MT = WM / 8, NG = WN / 16;
  static constexpr int kABytes = BM * BK * 8, kBBytes = BN * BK * 8;
  static constexpr int kStageBytes = kABytes + kBBytes;         // 24 KB
  static constexpr int kGroupBytes = STAGES * kStageBytes;
  static constexpr int kSmemBytes = GROUPS * kGroupBytes + 1024 + (GROUPS * 2 * STAGES + 2) * 8 + 64 * 8;
};

template <int EPI, bool TURN>
__global__ void __launch_bounds__(PPCfg::kThreads, 1)
    dgemm_pp_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const GemmParams p) {
  using C = PPCfg;
  constexpr int STAGES = C::STAGES;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::GROUPS * C::kGroupBytes);
  // full[g][s] = bars[g * 2 * STAGES + s], empty[g][s] = bars[g * 2 * STAGES + STAGES + s], turn[g]
  uint64_t* turn = bars + C::GROUPS * 2 * STAGES;
  double* red = reinterpret_cast<double*>(turn + 2);   // EPI_RESID cross-warp scratch (8 warps)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n = p.n;
  const int tiles_m = (n + C::BM - 1) / C::BM;
  const int tiles_n = (n + C::BN - 1) / C::BN;
  const int tiles_per_z = tiles_m * tiles_n;
  const int total = tiles_per_z * p.num_z;
  const int KT = (n + BK - 1) / BK;
  const int vgrid = 2 * (int)gridDim.x;   // virtual CTAs: group g of CTA b is 2b + g

  if (threadIdx.x == 0) {
    for (int g = 0; g < C::GROUPS; ++g)
      for (int s = 0; s < STAGES; ++s) {
        mbar_init(&bars[g * 2 * STAGES + s], 1);
        mbar_init(&bars[g * 2 * STAGES + STAGES + s], C::kGroupWarps);
      }
    mbar_init(&turn[0], C::kGroupWarps);
    mbar_init(&turn[1], C::kGroupWarps);
    fence_barrier_init();
    fence_proxy_async();
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  if (cta_stop(p.stop_flag)) return;

  if (warp >= C::kConsumerWarps)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
  else
    asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");

  if (warp >= C::kConsumerWarps) {
    // ===================== TMA producers: warp 8 + g, lane 0, serves group g =====================
    const int g = warp - C::kConsumerWarps;
    if (g < C::GROUPS && lane == 0) {
      if (g == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
      }
      uint64_t* full = bars + g * 2 * STAGES;
      uint64_t* empty = full + STAGES;
      unsigned char* ring = smem + g * C::kGroupBytes;
      int stage = 0;
      uint32_t phase = 0;
      for (int t = 2 * (int)blockIdx.x + g; t < total; t += vgrid) {
        const int z = t / tiles_per_z;
        const int r = t - z * tiles_per_z;
        int tm_, tn_;
        tile_coords(false, r, tiles_m, tiles_n, tm_, tn_);
        const int m0 = tm_ * C::BM;
        const int n0 = tn_ * C::BN;
        const int sa = p.a_base + z * p.a_step;
        const int sb = p.b_base + (z ^ p.b_xor) * p.b_step;
        const int pf_k0 = KT > 8 ? KT - 8 : 0;
        const int pf_bytes = (((n - n0) < C::BN ? (n - n0) : C::BN) * 8 + 15) & ~15;
        for (int kt = 0; kt < KT; ++kt) {
          if (kt >= pf_k0) {   // the epilogue's operand rows into L2 during the last k-steps
            const int per = (C::BM + (KT - pf_k0) - 1) / (KT - pf_k0);
            const int r0 = (kt - pf_k0) * per;
            const int r1 = (r0 + per < C::BM) ? r0 + per : C::BM;
            for (int rr = r0; rr < r1 && m0 + rr < n; ++rr) {
              const long long off = (long long)(m0 + rr) * p.ld + n0;
              if (p.beta != 0.0) prefetch_l2(p.C.at(z) + off, pf_bytes);
              if constexpr (EPI == EPI_RK || EPI == EPI_EULER || EPI == EPI_EULER_CORR)
                prefetch_l2(p.X_in.at(z) + off, pf_bytes);
              if constexpr (EPI == EPI_RK) {
                if (p.stage > 1) prefetch_l2(p.S.at(z) + off, pf_bytes);
              }
              if constexpr (EPI == EPI_EULER_CORR) {
                prefetch_l2(p.F_in.at(z) + off, pf_bytes);
                prefetch_l2(p.Gold.at(z) + off, pf_bytes);
              }
            }
          }
          mbar_wait(&empty[stage], phase ^ 1);
          unsigned char* sA = ring + stage * C::kStageBytes;
          unsigned char* sB = sA + C::kABytes;
          mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
          tma_load_3d(sA, &tmA, &full[stage], kt * BK, m0, sa);
#pragma unroll
          for (int gg = 0; gg < C::BN / 16; ++gg)
            tma_load_3d(sB + gg * 2048, &tmB, &full[stage], n0 + gg * 16, kt * BK, sb);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    return;
  }

  // ===================== consumers: group g = warp / 4 =====================
  const int g = warp / C::kGroupWarps;
  const int wn = warp % C::kGroupWarps;
  const int g8 = lane >> 2;
  const int c = lane & 3;
  const int rowA = rho8(g8);
  uint64_t* full = bars + g * 2 * STAGES;
  uint64_t* empty = full + STAGES;
  const uint32_t ring = smem_u32(smem + g * C::kGroupBytes);
  int stage = 0;
  uint32_t phase = 0;
  uint32_t turn_phase = 0;
  // group 0 owns the tensor pipe first: complete turn[0]'s phase 0 with the other group's arrivals
  if (TURN && g == 1 && lane == 0) mbar_arrive(&turn[0]);

  for (int t = 2 * (int)blockIdx.x + g; t < total; t += vgrid) {
    const int z = t / tiles_per_z;
    const int r = t - z * tiles_per_z;
    int tm_, tn_;
    tile_coords(false, r, tiles_m, tiles_n, tm_, tn_);
    const int m0 = tm_ * C::BM;
    const int n0 = tn_ * C::BN;
    const double alpha = (p.alt_sign && (z & 1)) ? -p.alpha : p.alpha;

    double acc[C::MT][2 * C::NG][2];
#pragma unroll
    for (int i = 0; i < C::MT; ++i)
#pragma unroll
      for (int j = 0; j < 2 * C::NG; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    if (TURN) {
      mbar_wait(&turn[g], turn_phase);   // this group's turn on the tensor pipe
      turn_phase ^= 1;
    }
    bool ready = false;
    for (int kt = 0; kt < KT; ++kt) {
      if (!ready) mbar_wait(&full[stage], phase);
      const uint32_t sA = ring + stage * C::kStageBytes;
      const uint32_t sB = sA + C::kABytes;
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        double2 af[C::MT];
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt) {
          const int row = mt * 8 + rowA;
          af[mt] = lds128(sA + row * 128 + ((((kb << 2) + c) ^ rowA) << 4));
        }
        double2 bf[C::NG][2];
#pragma unroll
        for (int ng = 0; ng < C::NG; ++ng) {
          const int grp = (wn * C::WN) / 16 + ng;
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const int k = kb * 8 + 2 * c + s;
            bf[ng][s] = lds128(sB + grp * 2048 + k * 128 + ((g8 ^ (k & 7)) << 4));
          }
        }
        if (kb == 1) {
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[stage]);
          const int ns = (stage + 1 == STAGES) ? 0 : stage + 1;
          ready = (kt + 1 < KT) && mbar_test_wait(&full[ns], ns == 0 ? (phase ^ 1) : phase);
        }
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
          for (int mt = 0; mt < C::MT; ++mt) {
            const double a = s ? af[mt].y : af[mt].x;
#pragma unroll
            for (int ng = 0; ng < C::NG; ++ng) {
              dmma(acc[mt][2 * ng][0], acc[mt][2 * ng][1], a, bf[ng][s].x);
              dmma(acc[mt][2 * ng + 1][0], acc[mt][2 * ng + 1][1], a, bf[ng][s].y);
            }
          }
      }
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    // hand the tensor pipe to the other group (its main loop overlaps this group's epilogue)
    if (TURN) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&turn[g ^ 1]);
    }

    // ---------------- epilogue (gemm.cuh's) ----------------
    double part = 0.0;
    const int ld = p.ld;
    if constexpr (EPI != EPI_RESID) {
      EpiIn buf[2];
      if constexpr (EPI == EPI_STORE) {
        const int row = m0 + rowA, col = n0 + wn * C::WN + 4 * c;
        if (row < n && col < n) epi_load4<EPI>(p, z, row, col, n, ld, buf[0]);
      }
#pragma unroll
      for (int gi = 0; gi < C::MT * C::NG; ++gi) {
        const int mt = gi / C::NG, ng = gi % C::NG;
        if constexpr (EPI == EPI_STORE) {
          if (gi + 1 < C::MT * C::NG) {
            const int mt1 = (gi + 1) / C::NG, ng1 = (gi + 1) % C::NG;
            const int row1 = m0 + mt1 * 8 + rowA, col1 = n0 + wn * C::WN + ng1 * 16 + 4 * c;
            if (row1 < n && col1 < n) epi_load4<EPI>(p, z, row1, col1, n, ld, buf[(gi + 1) & 1]);
          }
        }
        const int row = m0 + mt * 8 + rowA;
        const int col = n0 + wn * C::WN + ng * 16 + 4 * c;
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
      for (int mt = 0; mt < C::MT; ++mt) {
        const int row = m0 + mt * 8 + rowA;
        if (row >= n) continue;
#pragma unroll
        for (int ng = 0; ng < C::NG; ++ng) {
          const int col = n0 + wn * C::WN + ng * 16 + 4 * c;
          if (col >= n) continue;
          double k4[4] = {acc[mt][2 * ng][0], acc[mt][2 * ng + 1][0], acc[mt][2 * ng][1], acc[mt][2 * ng + 1][1]};
          epi_apply4<EPI>(p, z, alpha, row, col, n, ld, k4, false, false, part);
        }
      }
      // deterministic per-tile reduction inside the group: fixed shuffle tree, warps in order
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      named_bar_sync(1 + g, C::kGroupWarps * 32);
      if (lane == 0) red[warp] = part;
      named_bar_sync(1 + g, C::kGroupWarps * 32);
      if (wn == 0 && lane == 0) {
        double s = 0.0;
        for (int w = 0; w < C::kGroupWarps; ++w) s += red[g * C::kGroupWarps + w];
        p.partials[t] = s;
      }
    }
  }
}

}  // namespace mfode
