// K10: the whole fine propagator of a batch of slices in ONE persistent launch (moderate n).
//
// F(U^k_n) = m_F classical RK4 steps ("compute in parallel"; reading R1) is a chain of
// 4 * gps GEMM phases per step (gps = 2 for the inverse flow, W = B Y then K = Y W; 1 otherwise).
// At n ~ 256 one phase of one slice is only 16 tiles of 64 x 64 with a 16-step k-loop, so the
// launch-per-GEMM path (gemm.cuh, 8 m_F launches per chunk) spends much of each launch in launch
// latency, pipeline fill, the last partial wave and the epilogue tail.  Here one launch runs every
// phase of every slice of the batch:
//   * work items (phase g, slice z, tile) are handed out in that order by a global ticket counter
//     (one atomicAdd per tile by the producer warp) to persistent CTAs;
//   * tile-level dependencies through per-slice row / column completion counters (release by the
//     CTA that finished a tile, polled by the producer before its TMA loads): with K-phase q the
//     q-th K = ... GEMM of the slice (Y_{q+1} = X + c K_q, or X at stage 4),
//       inverse W-phase q, tile (i, j):  K-phase q-1 column j          (W = B Y_q reads Y_q col j)
//       inverse K-phase q, tile (i, j):  K-phase q-1 row i, W-phase q column j
//       sqrt    K-phase q, tile (i, j):  K-phase q-1 row i and column j (K = A - Y Y)
//       exp/affine K-phase q:            K-phase q-1 column j            (K = A Y (+ G))
//     Items are taken in order and a taken item depends only on earlier (taken) items whose
//     loads are all issued, so the schedule cannot deadlock whatever the residency;
//   * the WAR hazards on the ping-pong buffers (Y_a/Y_b, W, S, X) are implied by these read-after-
//     write dependencies (DESIGN.md §7 "K10" walks through each buffer);
//   * main loop, fragment mapping, k order and epilogue arithmetic are those of gemm.cuh
//     (epi_apply4_impl), so results are bitwise identical to the launch-per-GEMM path (tested).
// Generic-proxy epilogue stores are read by the TMA (async proxy) of other CTAs: writers fence
// (fence.proxy.async.global) before the release, the producer fences after its acquire.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include "gemm.cuh"
#include "ptx.cuh"

namespace mfode {

// tensor maps of the operand slabs (3-D: n, n, count); A-role maps have BM-row boxes, B-role 16
struct FusedMaps {
  CUtensorMap mA_M;                    // constant M (B = I - A for inverse, A for exp / affine), A-role
  CUtensorMap mA_in, mA_out, mA_ya, mA_yb;
  CUtensorMap mB_in, mB_out, mB_ya, mB_yb, mB_w;
};

struct FusedParams {
  int n, ld, Z, mF, flow, gps, T_tiles, tiles_n;
  int in_base, out_base;   // first slice of the batch in the IN / OUT slabs
  double h;
  MatRef Xin, Xout, Ya, Yb, W, S;   // z-indexed (Xin / Xout already offset to the batch)
  const double* Cterm;              // beta = 1 term: A (sqrt) or the source G (affine); null otherwise
  const int* stop_flag;
  unsigned int* sched;              // [0] ticket, then per slice: rowK[tiles_m], colK[tiles_n], colW[tiles_n]
  int tiles_m;
  long long total;                  // number of work items
};

__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acquire_gpu() { asm volatile("fence.acq_rel.gpu;\n" ::: "memory"); }
__device__ __forceinline__ void red_release_add_u32(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

// phase g of a step-major schedule: step = g / (4 gps), stage s = (g / gps) % 4 + 1, sub = g % gps
struct PhaseInfo {
  int step, stage, sub;
};
__device__ __forceinline__ PhaseInfo phase_info(int g, int gps) {
  PhaseInfo r;
  r.sub = g % gps;
  const int sg = g / gps;
  r.stage = (sg & 3) + 1;
  r.step = sg >> 2;
  return r;
}

template <int BM, int BN, int WARPS_M, int WARPS_N, int STAGES>
// 168 registers per thread at launch: three warps share one SM sub-partition (16K registers) in both
// configurations -- 12 warps of the 8-consumer-warp CTA, 2 x 5 warps of two resident 4-warp CTAs --
// so a 169th register halves the 4-warp configuration's occupancy (seen at 173 registers: 2 -> 1
// CTA per SM, 29.2 -> 20.7 TF/s at n = 256 with 32 slices).
__global__ void __maxnreg__(168)
    fine_fused_kernel(const __grid_constant__ FusedMaps maps, const FusedParams p) {
  using Cfg = GemmCfg<BM, BN, WARPS_M, WARPS_N, STAGES>;
  constexpr int kQ = 8;   // tile-info ring (the producer runs at most STAGES tiles ahead)
  static_assert(STAGES < kQ, "tile ring too small");
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
  uint64_t* empty = full + STAGES;
  long long* tinfo = reinterpret_cast<long long*>(empty + STAGES);   // kQ work-item tickets (-1: done)

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n = p.n;
  const int T = p.T_tiles;
  const int KT = (n + BK - 1) / BK;
  const int phases_per_launch = p.mF * 4 * p.gps;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], Cfg::kConsumerWarps);
    }
    fence_barrier_init();
    fence_proxy_async();
  }
  __syncthreads();
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
    // ===================== producer: tickets, dependencies, TMA =====================
    if (warp == Cfg::kConsumerWarps && lane == 0) {
      tma_prefetch_desc(&maps.mA_M);
      tma_prefetch_desc(&maps.mA_in);
      tma_prefetch_desc(&maps.mA_out);
      tma_prefetch_desc(&maps.mA_ya);
      tma_prefetch_desc(&maps.mA_yb);
      tma_prefetch_desc(&maps.mB_in);
      tma_prefetch_desc(&maps.mB_out);
      tma_prefetch_desc(&maps.mB_ya);
      tma_prefetch_desc(&maps.mB_yb);
      tma_prefetch_desc(&maps.mB_w);
      // Y-operand maps by source (0 in, 1 out, 2 Y_a, 3 Y_b), selected without a local array
      auto mapA = [&](int src) {
        return src == 0 ? &maps.mA_in : (src == 1 ? &maps.mA_out : (src == 2 ? &maps.mA_ya : &maps.mA_yb));
      };
      auto mapB = [&](int src) {
        return src == 0 ? &maps.mB_in : (src == 1 ? &maps.mB_out : (src == 2 ? &maps.mB_ya : &maps.mB_yb));
      };
      int stage = 0;
      uint32_t phase = 0;
      int seq = 0;
      while (true) {
        long long t = (long long)atomicAdd(p.sched, 1u);
        // a speculative launch whose sweep was cancelled stops taking work (every taken item's
        // dependencies are earlier, already taken items, so the holders still finish)
        if (t < p.total && p.stop_flag && *(volatile const int*)p.stop_flag != 0) t = p.total;
        if (t >= p.total) {
          // sentinel: wake the consumers on the next stage without data
          mbar_wait(&empty[stage], phase ^ 1);
          tinfo[seq % kQ] = -1;
          mbar_arrive(&full[stage]);
          break;
        }
        const int per_phase = p.Z * T;
        const int g = (int)(t / per_phase);
        const int r = (int)(t - (long long)g * per_phase);
        const int z = r / T;
        const int tile = r - z * T;
        const PhaseInfo ph = phase_info(g, p.gps);
        // tile-level dependencies (see the header): relaxed polling (an acquire per poll would
        // invalidate the SM's L1 every time), then one acquire fence once the counts are reached
        {
          const int ti = tile / p.tiles_n, tj = tile % p.tiles_n;
          const unsigned* base = p.sched + 1 + (size_t)z * (p.tiles_m + 2 * p.tiles_n);
          const unsigned* rowK = base + ti;
          const unsigned* colK = base + p.tiles_m + tj;
          const unsigned* colW = base + p.tiles_m + p.tiles_n + tj;
          const int q = g / p.gps;   // K-phase index (the W-phase of the inverse flow shares it)
          const unsigned needRow = (unsigned)q * (unsigned)p.tiles_n;
          const unsigned needCol = (unsigned)q * (unsigned)p.tiles_m;
          bool waited = false;
          if (p.flow == 0 && ph.sub == 0) {
            if (q > 0) { while (ld_relaxed_u32(colK) < needCol) __nanosleep(20); waited = true; }
          } else if (p.flow == 0) {
            if (q > 0) { while (ld_relaxed_u32(rowK) < needRow) __nanosleep(20); }
            while (ld_relaxed_u32(colW) < needCol + (unsigned)p.tiles_m) __nanosleep(20);
            waited = true;
          } else if (p.flow == 1) {
            if (q > 0) {
              while (ld_relaxed_u32(rowK) < needRow) __nanosleep(20);
              while (ld_relaxed_u32(colK) < needCol) __nanosleep(20);
              waited = true;
            }
          } else if (q > 0) {
            while (ld_relaxed_u32(colK) < needCol) __nanosleep(20);
            waited = true;
          }
          if (waited) {
            fence_acquire_gpu();
            fence_proxy_async_global();
          }
        }
        // operand selection (the same operands as driver.cu fine_prop / flow_gemms)
        const int ysrc = (ph.stage == 1) ? (ph.step == 0 ? 0 : 1) : (ph.stage == 3 ? 3 : 2);   // in, out, ya, yb
        const int ybase = (ysrc == 0) ? p.in_base : (ysrc == 1 ? p.out_base : 0);
        const CUtensorMap* ma;
        const CUtensorMap* mb;
        int sa, sb;
        const bool left_const = (p.flow == 0 && ph.sub == 0) || p.flow == 2 || p.flow == 4;
        if (left_const) {   // W = B Y (inverse), K = A Y (exp, affine)
          ma = &maps.mA_M;
          sa = 0;
          mb = mapB(ysrc);
          sb = ybase + z;
        } else if (p.flow == 0) {   // K = Y W
          ma = mapA(ysrc);
          sa = ybase + z;
          mb = &maps.mB_w;
          sb = z;
        } else {   // sqrt: K = A - Y Y
          ma = mapA(ysrc);
          sa = ybase + z;
          mb = mapB(ysrc);
          sb = ybase + z;
        }
        const int m0 = (tile / p.tiles_n) * BM;
        const int n0 = (tile % p.tiles_n) * BN;
        for (int kt = 0; kt < KT; ++kt) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (kt == 0) tinfo[seq % kQ] = t;   // published by the arrive below (release.cta)
          unsigned char* sA = smem + stage * Cfg::kStageBytes;
          unsigned char* sB = sA + Cfg::kABytes;
          mbar_arrive_expect_tx(&full[stage], Cfg::kStageBytes);
          tma_load_3d(sA, ma, &full[stage], kt * BK, m0, sa);
#pragma unroll
          for (int gg = 0; gg < BN / 16; ++gg) tma_load_3d(sB + gg * 2048, mb, &full[stage], n0 + gg * 16, kt * BK, sb);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        ++seq;
      }
    }
    return;
  }

  // ===================== consumers: DMMA main loop + fused epilogue =====================
  const int wm = warp / WARPS_N;
  const int wn = warp % WARPS_N;
  const int g8 = lane >> 2;
  const int c = lane & 3;
  const int rowA = rho8(g8);
  int stage = 0;
  uint32_t phase = 0;
  int seq = 0;
  const uint32_t smem_base = smem_u32(smem);
  const int per_phase = p.Z * T;

  while (true) {
    mbar_wait(&full[stage], phase);
    const long long t = tinfo[seq % kQ];
    if (t < 0) break;   // sentinel (no data, no release)
    const int g = (int)(t / per_phase);
    const int r = (int)(t - (long long)g * per_phase);
    const int z = r / T;
    const int tile = r - z * T;
    const PhaseInfo ph = phase_info(g, p.gps);
    const int m0 = (tile / p.tiles_n) * BM;
    const int n0 = (tile % p.tiles_n) * BN;

    double acc[Cfg::MT][2 * Cfg::NG][2];
#pragma unroll
    for (int i = 0; i < Cfg::MT; ++i)
#pragma unroll
      for (int j = 0; j < 2 * Cfg::NG; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    bool ready = true;   // full[stage] of kt = 0 observed above
    for (int kt = 0; kt < KT; ++kt) {
      if (!ready) mbar_wait(&full[stage], phase);
      const uint32_t sA = smem_base + stage * Cfg::kStageBytes;
      const uint32_t sB = sA + Cfg::kABytes;
#pragma unroll
      for (int kb = 0; kb < 2; ++kb) {
        double2 af[Cfg::MT];
#pragma unroll
        for (int mt = 0; mt < Cfg::MT; ++mt) {
          const int row = wm * Cfg::WM + mt * 8 + rowA;
          af[mt] = lds128(sA + row * 128 + ((((kb << 2) + c) ^ rowA) << 4));
        }
        double2 bf[Cfg::NG][2];
#pragma unroll
        for (int ng = 0; ng < Cfg::NG; ++ng) {
          const int grp = (wn * Cfg::WN) / 16 + ng;
#pragma unroll
          for (int s = 0; s < 2; ++s) {
            const int k = kb * 8 + 2 * c + s;
            bf[ng][s] = lds128(sB + grp * 2048 + k * 128 + ((g8 ^ (k & 7)) << 4));
          }
        }
        if (kb == 1) {
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
      // stage release after the consuming DMMAs are issued (no proxy fence), as in gemm.cuh (same-box
      // A/B here: n = 256 / 16 slices 27.07 -> 27.60 TF/s, 4-warp configuration +4-5 %,
      // profiles/ab_k10_r02.jsonl)
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    ++seq;

    // ---------------- epilogue (the launch-per-GEMM path's arithmetic) ----------------
    GemmParams q = {};
    q.n = n;
    q.ld = p.ld;
    q.sym = 0;
    q.alt_sign = 0;
    q.alpha = 1.0;
    q.beta = 0.0;
    q.C = MatRef{const_cast<double*>(p.Cterm), 0};
    q.h = p.h;
    q.stage = ph.stage;
    const bool store_w = (p.flow == 0 && ph.sub == 0);
    if (!store_w) {
      if (p.flow == 1) {   // sqrt: K = -(Y Y) + A
        q.alpha = -1.0;
        q.beta = 1.0;
      } else if (p.flow == 4) {   // affine: K = A Y + G
        q.beta = 1.0;
      }
      q.X_in = (ph.step == 0) ? p.Xin : p.Xout;
      q.S = p.S;
      if (ph.stage == 4) {
        q.X_out = p.Xout;
        q.Y_out = MatRef{nullptr, 0};
      } else {
        q.Y_out = (ph.stage == 2) ? p.Yb : p.Ya;
      }
    } else {
      q.Y_out = p.W;
    }
    const int ld = p.ld;
    double part = 0.0;
#pragma unroll
    for (int gi = 0; gi < Cfg::MT * Cfg::NG; ++gi) {
      const int mt = gi / Cfg::NG, ng = gi % Cfg::NG;
      const int row = m0 + wm * Cfg::WM + mt * 8 + rowA;
      const int col = n0 + wn * Cfg::WN + ng * 16 + 4 * c;
      if (row < n && col < n) {
        double k4[4] = {acc[mt][2 * ng][0], acc[mt][2 * ng + 1][0], acc[mt][2 * ng][1], acc[mt][2 * ng + 1][1]};
        double mv[2][4];
        double* mp[2];
        if (store_w)
          epi_apply4_impl<EPI_STORE, false>(q, z, 1.0, row, col, n, ld, k4, false, false, part, mv, mp);
        else
          epi_apply4_impl<EPI_RK, false>(q, z, q.alpha, row, col, n, ld, k4, false, false, part, mv, mp);
      }
    }
    // publish the tile: every consumer's stores, then one release of the slice's counter
    fence_proxy_async_global();
    named_bar_sync(1, Cfg::kConsumerWarps * 32);
    if (threadIdx.x == 0) {   // releases are cumulative over the CTA barrier
      unsigned* base = p.sched + 1 + (size_t)z * (p.tiles_m + 2 * p.tiles_n);
      const int ti = tile / p.tiles_n, tj = tile % p.tiles_n;
      if (store_w) {
        red_release_add_u32(base + p.tiles_m + p.tiles_n + tj, 1u);   // colW
      } else {
        red_release_add_u32(base + ti, 1u);                           // rowK
        red_release_add_u32(base + p.tiles_m + tj, 1u);               // colK
      }
    }
  }
  (void)phases_per_launch;
}

}  // namespace mfode
