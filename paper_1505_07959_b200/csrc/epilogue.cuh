// Fused element-wise epilogues of the parareal hot path, shared by the FP64
// DMMA GEMM (gemm.cuh) and the decode step of the emulated GEMM (ozaki.cu).  See gemm.cuh for the
// list of epilogues and the paper passages they implement.
#pragma once
#include <cuda_runtime.h>
// Included by gemm.cuh after GemmParams is declared.

namespace mfode {

// Fused parareal epilogue on 4 consecutive columns (col .. col+3, cnt valid) of one row, shared by
// the DMMA GEMM (gemm.cuh) and the emulated-GEMM decode (ozaki.cu).  k4 = the raw product A*B;
// applies K = alpha*k4 + beta*C and the EPI element-wise arithmetic, then stores.  `sym`: symmetric
// mode (write element and mirror); `diag`: strictly-lower elements are skipped (their mirror writes
// them).  EPI_RESID accumulates into `part` instead of storing.
// Epilogue operands of one 4-column group, loaded ahead of the arithmetic (software pipelining of
// the DMMA epilogue: the loads of group g+1 are in flight while group g is computed and stored).
struct EpiIn {
  double c[4], x[4], s[4], f[4];
};

__device__ __forceinline__ void epi_ld4(const double* src, bool full4, int cnt, double (&v)[4]) {
  if (full4) {
    const double2 a0 = *reinterpret_cast<const double2*>(src);
    const double2 a1 = *reinterpret_cast<const double2*>(src + 2);
    v[0] = a0.x; v[1] = a0.y; v[2] = a1.x; v[3] = a1.y;
  } else {
#pragma unroll
    for (int e = 0; e < 4; ++e) v[e] = (e < cnt) ? src[e] : 0.0;
  }
}

// Loads exactly the operands epi_apply4_impl<EPI> reads for (row, col .. col+3).
template <int EPI>
__device__ __forceinline__ void epi_load4(const GemmParams& p, int z, int row, int col, int n, int ld, EpiIn& in) {
  const long long off = (long long)row * ld + col;
  const bool full4 = (col + 3 < n);
  const int cnt = full4 ? 4 : (n - col);
  if (p.beta != 0.0) epi_ld4(p.C.at(z) + off, full4, cnt, in.c);
  if constexpr (EPI != EPI_STORE && EPI != EPI_RESID) {
    epi_ld4(p.X_in.at(z) + off, full4, cnt, in.x);
    if constexpr (EPI == EPI_RK) {
      if (p.stage > 1) epi_ld4(p.S.at(z) + off, full4, cnt, in.s);
    }
    if constexpr (EPI == EPI_ACCEL) {
      if ((z & 1) == 0) epi_ld4(p.S.at(z) + off, full4, cnt, in.s);
    }
    if constexpr (EPI == EPI_EULER_CORR) {
      epi_ld4(p.Gold.at(z) + off, full4, cnt, in.s);
      epi_ld4(p.F_in.at(z) + off, full4, cnt, in.f);
    }
  }
}

// DEFER (symmetric mode only): the mirrored stores are not issued; the values of the (up to two)
// output arrays land in mv[slot][0..3] and the arrays' base pointers in mp[slot] (null = unused),
// so the caller can write the mirrors coalesced through a shared-memory transpose.
template <int EPI, bool DEFER, bool PRE = false>
__device__ __forceinline__ void epi_apply4_impl(const GemmParams& p, int z, double alpha, int row, int col, int n,
                                                int ld, double (&k4)[4], bool sym, bool diag, double& part,
                                                double (&mv)[2][4], double* (&mp)[2], const EpiIn* pre = nullptr) {
  const long long off = (long long)row * ld + col;
  const bool full4 = (col + 3 < n);
  const int cnt = full4 ? 4 : (n - col);
  // K = alpha*acc + beta*C
  if (PRE && p.beta != 0.0) {
#pragma unroll
    for (int e = 0; e < 4; ++e) k4[e] = fma(alpha, k4[e], p.beta * pre->c[e]);
  } else if (p.beta != 0.0) {
    const double* Cp = p.C.at(z) + off;
    if (full4) {
      const double2 c0 = *reinterpret_cast<const double2*>(Cp);
      const double2 c1 = *reinterpret_cast<const double2*>(Cp + 2);
      k4[0] = fma(alpha, k4[0], p.beta * c0.x);
      k4[1] = fma(alpha, k4[1], p.beta * c0.y);
      k4[2] = fma(alpha, k4[2], p.beta * c1.x);
      k4[3] = fma(alpha, k4[3], p.beta * c1.y);
    } else {
      #pragma unroll
      for (int e = 0; e < 4; ++e)
        if (e < cnt) k4[e] = fma(alpha, k4[e], p.beta * Cp[e]);
    }
  } else if (alpha != 1.0) {
#pragma unroll
    for (int e = 0; e < 4; ++e) k4[e] *= alpha;
  }
  double in0[4] = {0, 0, 0, 0}, in1[4] = {0, 0, 0, 0}, o0[4] = {0, 0, 0, 0}, o1[4] = {0, 0, 0, 0};
  if constexpr (EPI == EPI_STORE) {
#pragma unroll
    for (int e = 0; e < 4; ++e) o0[e] = k4[e];
  } else if constexpr (EPI == EPI_RESID) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      // symmetric mode: off-diagonal entries stand for themselves and their mirror
      const double w = !sym ? 1.0 : ((diag && row > col + e) ? 0.0 : (row == col + e ? 1.0 : 2.0));
      if (e < cnt) {
        const double v = k4[e] - ((row == col + e) ? p.shift : 0.0);
        part = fma(w * v, v, part);
      }
    }
  } else {
    // load X (and S / Fk / Gold as needed)
    const double* Xp = p.X_in.at(z) + off;
    if (PRE) {
#pragma unroll
      for (int e = 0; e < 4; ++e) in0[e] = pre->x[e];
    } else if (full4) {
      const double2 a0 = *reinterpret_cast<const double2*>(Xp);
      const double2 a1 = *reinterpret_cast<const double2*>(Xp + 2);
      in0[0] = a0.x; in0[1] = a0.y; in0[2] = a1.x; in0[3] = a1.y;
    } else {
      #pragma unroll
      for (int e = 0; e < 4; ++e) in0[e] = (e < cnt) ? Xp[e] : 0.0;
    }
    const double* Sp = nullptr;
    if constexpr (EPI == EPI_RK || EPI == EPI_ACCEL) Sp = p.S.at(z) + off;
    if constexpr (EPI == EPI_EULER_CORR) Sp = p.Gold.at(z) + off;
    if constexpr (EPI == EPI_RK || EPI == EPI_EULER_CORR || EPI == EPI_ACCEL) {
      if (EPI == EPI_EULER_CORR || (EPI == EPI_RK && p.stage > 1) || (EPI == EPI_ACCEL && (z & 1) == 0)) {
        if (PRE) {
#pragma unroll
          for (int e = 0; e < 4; ++e) in1[e] = pre->s[e];
        } else if (full4) {
          const double2 a0 = *reinterpret_cast<const double2*>(Sp);
          const double2 a1 = *reinterpret_cast<const double2*>(Sp + 2);
          in1[0] = a0.x; in1[1] = a0.y; in1[2] = a1.x; in1[3] = a1.y;
        } else {
          #pragma unroll
          for (int e = 0; e < 4; ++e) in1[e] = (e < cnt) ? Sp[e] : 0.0;
        }
      }
    }
    if constexpr (EPI == EPI_RK) {
      const double h = p.h;
      const int st = p.stage;
      if (st == 4) {
        const double h6 = h / 6.0;
#pragma unroll
        for (int e = 0; e < 4; ++e) o0[e] = fma(h6, in1[e] + k4[e], in0[e]);   // X
      } else {
        const double cy = (st == 3) ? h : 0.5 * h;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          o1[e] = (st == 1) ? k4[e] : fma(2.0, k4[e], in1[e]);                // S
          o0[e] = fma(cy, k4[e], in0[e]);                                      // Y'
        }
      }
    } else if constexpr (EPI == EPI_EULER) {
#pragma unroll
      for (int e = 0; e < 4; ++e) o0[e] = fma(p.h, k4[e], in0[e]);
    } else if constexpr (EPI == EPI_ACCEL) {
      // Algorithm 8: even z: X' = X + dt ((I - A X) + u); odd z: u' = u - dt A u
      if ((z & 1) == 0) {
#pragma unroll
        for (int e = 0; e < 4; ++e) o0[e] = fma(p.h, (((row == col + e) ? 1.0 : 0.0) - k4[e]) + in1[e], in0[e]);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) o0[e] = fma(-p.h, k4[e], in0[e]);
      }
    } else if constexpr (EPI == EPI_EULER_CORR) {
      const double* Fp = p.F_in.at(z) + off;
      double fk[4];
      if (PRE) {
#pragma unroll
        for (int e = 0; e < 4; ++e) fk[e] = pre->f[e];
      } else if (full4) {
        const double2 a0 = *reinterpret_cast<const double2*>(Fp);
        const double2 a1 = *reinterpret_cast<const double2*>(Fp + 2);
        fk[0] = a0.x; fk[1] = a0.y; fk[2] = a1.x; fk[3] = a1.y;
      } else {
        #pragma unroll
        for (int e = 0; e < 4; ++e) fk[e] = (e < cnt) ? Fp[e] : 0.0;
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const double gnew = fma(p.h, k4[e], in0[e]);
        o1[e] = gnew;                         // Gold <- G(U^{k+1}_n)
        o0[e] = fk[e] + (gnew - in1[e]);      // U^{k+1}_{n+1} = F + (Gnew - Gold)   (R3)
      }
    }
  }
  // ---- stores ----
  int slot = 0;
  auto store4 = [&](double* dst, const double* v) {
    if (DEFER) {
      double* base = dst - off;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int cc = col + e;
        if (e < cnt && row <= cc) base[(long long)row * ld + cc] = v[e];
        mv[slot][e] = v[e];
      }
      mp[slot] = base;
      ++slot;
    } else if (sym) {
      // upper-triangle tile: write (row, col+e) and its mirror (col+e, row); in a diagonal
      // tile the strictly-lower elements are written by the mirror of their partner
      double* base = dst - off;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int cc = col + e;
        if (e < cnt && !(diag && row > cc)) {
          base[(long long)row * ld + cc] = v[e];
          if (row != cc) base[(long long)cc * ld + row] = v[e];
        }
      }
    } else if (full4) {
      *reinterpret_cast<double2*>(dst) = make_double2(v[0], v[1]);
      *reinterpret_cast<double2*>(dst + 2) = make_double2(v[2], v[3]);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (e < cnt) dst[e] = v[e];
    }
  };
  if constexpr (EPI == EPI_STORE) {
    store4(p.Y_out.at(z) + off, o0);
  } else if constexpr (EPI == EPI_RK) {
    if (p.stage == 4) {
      store4(p.X_out.at(z) + off, o0);
      if (p.Y_out.p) store4(p.Y_out.at(z) + off, o0);
    } else {
      store4(p.S.at(z) + off, o1);
      store4(p.Y_out.at(z) + off, o0);
    }
  } else if constexpr (EPI == EPI_EULER || EPI == EPI_ACCEL) {
    store4(p.X_out.at(z) + off, o0);
    if (p.Gold.p) store4(p.Gold.at(z) + off, o0);
  } else if constexpr (EPI == EPI_EULER_CORR) {
    store4(p.U_out.at(z) + off, o0);
    store4(p.Gold.at(z) + off, o1);
  }
}

// The output arrays epi_apply4_impl<EPI, true> reports in mv / mp, in the same slot order.
template <int EPI>
__device__ __forceinline__ void epi_out_ptrs(const GemmParams& p, int z, double* (&mp)[2]) {
  mp[0] = mp[1] = nullptr;
  if constexpr (EPI == EPI_STORE) {
    mp[0] = p.Y_out.at(z);
  } else if constexpr (EPI == EPI_RK) {
    if (p.stage == 4) {
      mp[0] = p.X_out.at(z);
      if (p.Y_out.p) mp[1] = p.Y_out.at(z);
    } else {
      mp[0] = p.S.at(z);
      mp[1] = p.Y_out.at(z);
    }
  } else if constexpr (EPI == EPI_EULER || EPI == EPI_ACCEL) {
    mp[0] = p.X_out.at(z);
    if (p.Gold.p) mp[1] = p.Gold.at(z);
  } else if constexpr (EPI == EPI_EULER_CORR) {
    mp[0] = p.U_out.at(z);
    mp[1] = p.Gold.at(z);
  }
}

template <int EPI>
__device__ __forceinline__ void epi_apply4(const GemmParams& p, int z, double alpha, int row, int col, int n,
                                           int ld, double (&k4)[4], bool sym, bool diag, double& part) {
  double mv[2][4];
  double* mp[2];
  epi_apply4_impl<EPI, false>(p, z, alpha, row, col, n, ld, k4, sym, diag, part, mv, mp);
}

}  // namespace mfode
