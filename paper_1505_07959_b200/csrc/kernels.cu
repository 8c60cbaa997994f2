// Device kernels of the parareal hot path other than the GEMM main loop, and the GEMM launcher.
//   K3 setup:        X = I, B = I - A                      (X0 = I; R2)
//   K5 reductions:   ||X - Y||_F, ||X||_F, residual partial sums -> one scalar, deterministic
//                    (fixed grid, fixed shuffle tree, fixed-order final pass; no FP atomics)
//   stop flag:       flag = (metric <= tol) for speculative-work cancellation
//   GEMM launcher:   TMA tensor-map cache + tile-config dispatch of gemm.cuh
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <algorithm>

#include "fused.cuh"
#include "gemm.cuh"
#include "internal.h"
#include "small.cuh"

namespace mfode {

std::atomic<long long> g_launches{0};
bool g_pdl = true;
double g_cta_share_s = 2e-3;

// --------------------------------------------------------------------------------------------
// Element-wise kernels (HBM-bound; 16-byte vector accesses; padding columns kept at zero)
// --------------------------------------------------------------------------------------------
__global__ void k_identity(double* X, int n, int ld, int count, long long zstride) {
  const long long per = (long long)n * ld;
  const long long total = per * count;
  for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; i < total;
       i += (long long)gridDim.x * blockDim.x * 2) {
    const long long z = i / per;
    const long long e = i - z * per;
    const int r = (int)(e / ld), c = (int)(e - (long long)r * ld);
    double2 v;
    v.x = (r == c && c < n) ? 1.0 : 0.0;
    v.y = (r == c + 1 && c + 1 < n) ? 1.0 : 0.0;
    *reinterpret_cast<double2*>(X + z * zstride + e) = v;
  }
}

__global__ void k_i_minus(double* B, const double* A, int n, int ld) {
  const long long total = (long long)n * ld;
  for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; i < total;
       i += (long long)gridDim.x * blockDim.x * 2) {
    const int r = (int)(i / ld), c = (int)(i - (long long)r * ld);
    const double2 a = *reinterpret_cast<const double2*>(A + i);
    double2 v;
    v.x = (c < n) ? ((r == c ? 1.0 : 0.0) - a.x) : 0.0;
    v.y = (c + 1 < n) ? ((r == c + 1 ? 1.0 : 0.0) - a.y) : 0.0;
    *reinterpret_cast<double2*>(B + i) = v;
  }
}

// partials[b] = (sum (X-Y)^2, sum X^2) over block b's fixed share; Y may be null.
constexpr int kRedBlocks = 296;
constexpr int kRedThreads = 256;

__global__ void __launch_bounds__(kRedThreads) k_frob_partial(const double* X, const double* Y,
                                                              long long total, double* partials) {
  double d = 0.0, x = 0.0;
  for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; i < total;
       i += (long long)gridDim.x * blockDim.x * 2) {
    const double2 a = *reinterpret_cast<const double2*>(X + i);
    double2 b = make_double2(0.0, 0.0);
    if (Y) b = *reinterpret_cast<const double2*>(Y + i);
    const double e0 = a.x - b.x, e1 = a.y - b.y;
    d = fma(e0, e0, d);
    d = fma(e1, e1, d);
    x = fma(a.x, a.x, x);
    x = fma(a.y, a.y, x);
  }
  __shared__ double sd[kRedThreads / 32], sx[kRedThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    d += __shfl_xor_sync(0xffffffffu, d, o);
    x += __shfl_xor_sync(0xffffffffu, x, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sd[threadIdx.x >> 5] = d;
    sx[threadIdx.x >> 5] = x;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) {
      a += sd[w];
      b += sx[w];
    }
    partials[2 * blockIdx.x] = a;
    partials[2 * blockIdx.x + 1] = b;
  }
}

// Fixed-order final reduction of `count` interleaved pairs (stride 2) or singles (stride 1).
// mode 0 (delta): out = sqrt(sum0)/sqrt(sum1) ; mode 1 (norms): out[0] = sqrt(sum0), out[1] = sqrt(sum1)
// mode 2 (residual): out = sqrt(sum)/denom
__global__ void k_reduce_final(const double* partials, int count, int stride, int mode, double denom,
                               double* out, double tol, int* stop_flag) {
  __shared__ double s0[32], s1[32];
  // fixed order: thread t sums indices t, t+blockDim, ... ; then a fixed warp tree; then warps in order
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < count; i += blockDim.x) {
    a += partials[(long long)i * stride];
    if (stride == 2) b += partials[(long long)i * stride + 1];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) {
    s0[threadIdx.x >> 5] = a;
    s1[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
      x += s0[w];
      y += s1[w];
    }
    double metric;
    if (mode == 0) {
      metric = sqrt(x) / sqrt(y);
      out[0] = metric;
    } else if (mode == 1) {
      out[0] = sqrt(x);
      out[1] = sqrt(y);
      metric = out[0];
    } else {
      metric = sqrt(x) / denom;
      out[0] = metric;
    }
    if (stop_flag) *stop_flag = (metric <= tol) ? 1 : 0;
  }
}

__global__ void k_copy_flag(const double* metric, double tol, int* stop_flag) {
  *stop_flag = (*metric <= tol) ? 1 : 0;
}

// ---- Frobenius subspace algebra of the modified parareal (§3) -------------------------
// multi-dot: partials[i * gridDim.x + b] = sum over block b's fixed share of Q_i . V, i < count.
// V is read once per block share and pass, every Q_i once (HBM traffic (count + passes) * elems).
// kMaxDots coefficients per pass keep the accumulators in registers at full occupancy (a 64-wide
// pass needed 255 registers and spilled: one CTA per SM on a bandwidth-bound kernel).  Each
// coefficient's summation order (thread share, warp shuffle, block sum) does not depend on the pass
// width, so results are bitwise those of any other width.
constexpr int kMaxDots = 16;   // coefficients per multi-dot pass (the driver loops over passes)

__global__ void __launch_bounds__(kRedThreads) k_multidot(const double* Q, long long qstride, int count,
                                                          const double* V, long long total, double* partials) {
  double acc[kMaxDots];
#pragma unroll
  for (int i = 0; i < kMaxDots; ++i) acc[i] = 0.0;
  for (long long e = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; e < total;
       e += (long long)gridDim.x * blockDim.x * 2) {
    const double2 v = *reinterpret_cast<const double2*>(V + e);
#pragma unroll
    for (int i = 0; i < kMaxDots; ++i) {
      if (i < count) {
        const double2 q = *reinterpret_cast<const double2*>(Q + i * qstride + e);
        acc[i] = fma(q.x, v.x, acc[i]);
        acc[i] = fma(q.y, v.y, acc[i]);
      }
    }
  }
  __shared__ double red[kMaxDots][kRedThreads / 32];
#pragma unroll
  for (int i = 0; i < kMaxDots; ++i) {
    if (i < count) {
      double a = acc[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if ((threadIdx.x & 31) == 0) red[i][threadIdx.x >> 5] = a;
    }
  }
  __syncthreads();
  if (threadIdx.x < count) {
    double s = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) s += red[threadIdx.x][w];
    partials[(long long)threadIdx.x * gridDim.x + blockIdx.x] = s;
  }
}

// out[i] = sum_b partials[i * blocks + b] (fixed order), one block per i
__global__ void k_reduce_rows(const double* partials, int blocks, double* out) {
  __shared__ double s0[32];
  double a = 0.0;
  for (int b = threadIdx.x; b < blocks; b += blockDim.x) a += partials[(long long)blockIdx.x * blocks + b];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if ((threadIdx.x & 31) == 0) s0[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) x += s0[w];
    out[blockIdx.x] = x;
  }
}

// out = add + sign * sum_{i < count} coef[i] * Q_i   (ascending i; add may be null)
__global__ void k_lincomb(double* out, const double* Q, long long qstride, const double* coef, int count,
                          long long total, const double* add, double sign) {
  for (long long e = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; e < total;
       e += (long long)gridDim.x * blockDim.x * 2) {
    double2 s = make_double2(0.0, 0.0);
    for (int i = 0; i < count; ++i) {
      const double c = coef[i];
      const double2 q = *reinterpret_cast<const double2*>(Q + i * qstride + e);
      s.x = fma(c, q.x, s.x);
      s.y = fma(c, q.y, s.y);
    }
    double2 r;
    if (add) {
      const double2 a = *reinterpret_cast<const double2*>(add + e);
      r.x = fma(sign, s.x, a.x);
      r.y = fma(sign, s.y, a.y);
    } else {
      r.x = sign * s.x;
      r.y = sign * s.y;
    }
    *reinterpret_cast<double2*>(out + e) = r;
  }
}

// Y = (Y - coef[0] * X) (axpy with a device scalar) or, with scale != 0, Y = Y / coef[0]
__global__ void k_axpy_dev(double* Y, const double* X, const double* coef, long long total, int divide) {
  const double c = *coef;
  for (long long e = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; e < total;
       e += (long long)gridDim.x * blockDim.x * 2) {
    double2 y = *reinterpret_cast<double2*>(Y + e);
    if (divide) {
      y.x = y.x / c;
      y.y = y.y / c;
    } else {
      const double2 x = *reinterpret_cast<const double2*>(X + e);
      y.x = fma(-c, x.x, y.x);
      y.y = fma(-c, x.y, y.y);
    }
    *reinterpret_cast<double2*>(Y + e) = y;
  }
}

// ---- device-side Gram-Schmidt decision of Algorithm 2 (modified parareal) ----------
// stats = [., ||Z_i||_F, ., r_ii] (two launch_frob mode-1 outputs).  Keep the block (reading R16)
// iff r_ii > tol * max(1, ||Z_i||_F): Q_i = Q / r_ii; otherwise zero it, so later projections onto
// this slot add exact zeros (the host compacts the basis once per sweep).  keep = 1 / 0, or -1 if
// the candidate is not finite.
__global__ void k_gs_keep(double* Q, long long total, const double* stats, double tol, int* keep) {
  const double zn = stats[1], rii = stats[3];
  const bool k = rii > tol * fmax(1.0, zn);
  // -1: a non-finite candidate (reported as MFODE_ENONFINITE with its slice)
  if (blockIdx.x == 0 && threadIdx.x == 0) *keep = (isfinite(zn) && isfinite(rii)) ? (k ? 1 : 0) : -1;
  for (long long e = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; e < total;
       e += (long long)gridDim.x * blockDim.x * 2) {
    double2 q = *reinterpret_cast<double2*>(Q + e);
    if (k) {
      q.x = q.x / rii;
      q.y = q.y / rii;
    } else {
      q.x = 0.0;
      q.y = 0.0;
    }
    *reinterpret_cast<double2*>(Q + e) = q;
  }
}

// D_i = F(Q_i) - F(0) for `count` consecutive states (Algorithm 4, Remark P:424-428)
__global__ void k_sub_bcast(double* D, long long stride, int count, const double* F0, long long total) {
  for (int i = blockIdx.y; i < count; i += gridDim.y) {
    double* d = D + (long long)i * stride;
    for (long long e = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; e < total;
         e += (long long)gridDim.x * blockDim.x * 2) {
      double2 v = *reinterpret_cast<double2*>(d + e);
      const double2 f = *reinterpret_cast<const double2*>(F0 + e);
      v.x = v.x - f.x;
      v.y = v.y - f.y;
      *reinterpret_cast<double2*>(d + e) = v;
    }
  }
}

// eq. (update2): out = ((sum_i coef[i] D_i + F0) + Gv) - G0  (ascending i)
__global__ void k_lincomb_affine(double* out, const double* D, long long qstride, const double* coef, int count,
                                 long long total, const double* F0, const double* Gv, const double* G0) {
  for (long long e = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; e < total;
       e += (long long)gridDim.x * blockDim.x * 2) {
    double2 s = make_double2(0.0, 0.0);
    for (int i = 0; i < count; ++i) {
      const double c = coef[i];
      const double2 q = *reinterpret_cast<const double2*>(D + i * qstride + e);
      s.x = fma(c, q.x, s.x);
      s.y = fma(c, q.y, s.y);
    }
    const double2 f = *reinterpret_cast<const double2*>(F0 + e);
    const double2 g = *reinterpret_cast<const double2*>(Gv + e);
    const double2 g0 = *reinterpret_cast<const double2*>(G0 + e);
    double2 r;
    r.x = ((s.x + f.x) + g.x) - g0.x;
    r.y = ((s.y + f.y) + g.y) - g0.y;
    *reinterpret_cast<double2*>(out + e) = r;
  }
}

// ---- SPEC stop rule: max_n ||X_n - Y_n||_F over `count` consecutive states -----------------
constexpr int kSliceBlocks = 64;
__global__ void __launch_bounds__(kRedThreads) k_frob_slices(const double* X, const double* Y, long long stride,
                                                             long long total, double* partials) {
  const double* x = X + (long long)blockIdx.y * stride;
  const double* y = Y + (long long)blockIdx.y * stride;
  double d = 0.0;
  for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * 2; i < total;
       i += (long long)gridDim.x * blockDim.x * 2) {
    const double2 a = *reinterpret_cast<const double2*>(x + i);
    const double2 b = *reinterpret_cast<const double2*>(y + i);
    const double e0 = a.x - b.x, e1 = a.y - b.y;
    d = fma(e0, e0, d);
    d = fma(e1, e1, d);
  }
  __shared__ double sd[kRedThreads / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
  if ((threadIdx.x & 31) == 0) sd[threadIdx.x >> 5] = d;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) a += sd[w];
    partials[(long long)blockIdx.y * gridDim.x + blockIdx.x] = a;
  }
}

// out = max over slices of sqrt(fixed-order sum of that slice's partials); count == 0 -> 0
__global__ void k_reduce_slices_max(const double* partials, int count, int blocks, double* out) {
  double best = 0.0;
  for (int sl = 0; sl < count; ++sl) {
    double a = (threadIdx.x < blocks) ? partials[(long long)sl * blocks + threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    __shared__ double s0[2];
    if ((threadIdx.x & 31) == 0) s0[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x == 0) best = fmax(best, sqrt(s0[0] + s0[1]));
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = best;
}

// out = max_i vals[i][0] / denom; stop flag = (out <= tol)
struct PtrList {
  const double* p[64];
  int count;
};
__global__ void k_max_ptrs(PtrList l, double denom, double* out, double tol, int* stop_flag) {
  double m = 0.0;
  for (int i = 0; i < l.count; ++i) m = fmax(m, *l.p[i]);
  const double v = m / denom;
  *out = v;
  if (stop_flag) *stop_flag = (v <= tol) ? 1 : 0;
}

// flag = 1 if A != A^T anywhere (exact comparison, NaN counts as a mismatch); the caller zeroes flag.
// One 32 x 32 tile pair (i <= j) per block, both tiles staged through shared memory (coalesced reads).
__global__ void k_check_symmetric(const double* A, int n, int ld, int* flag) {
  const int ti = blockIdx.y, tj = blockIdx.x;
  if (ti > tj) return;
  __shared__ double a[32][33], b[32][33];
  const int r = threadIdx.y, cc = threadIdx.x;   // 32 x 8 threads
  for (int rr = r; rr < 32; rr += 8) {
    const int i1 = ti * 32 + rr, j1 = tj * 32 + cc;
    a[rr][cc] = (i1 < n && j1 < n) ? A[(long long)i1 * ld + j1] : 0.0;
    const int i2 = tj * 32 + rr, j2 = ti * 32 + cc;
    b[rr][cc] = (i2 < n && j2 < n) ? A[(long long)i2 * ld + j2] : 0.0;
  }
  __syncthreads();
  bool bad = false;
  for (int rr = r; rr < 32; rr += 8) bad |= (a[rr][cc] != b[cc][rr]);
  if (__any_sync(0xffffffffu, bad) && cc == 0) *flag = 1;
}

// --------------------------------------------------------------------------------------------
// host wrappers
// --------------------------------------------------------------------------------------------
static int ew_grid(long long elems) {
  long long g = (elems / 2 + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

cudaError_t launch_check_symmetric(const double* A, int n, int ld, int* flag, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(flag, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  const int t = (n + 31) / 32;
  k_check_symmetric<<<dim3(t, t), dim3(32, 8), 0, st>>>(A, n, ld, flag);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_identity(double* X, int n, int ld, int count, long long zstride, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  k_identity<<<ew_grid((long long)n * ld * count), 256, 0, st>>>(X, n, ld, count, zstride);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_i_minus(double* B, const double* A, int n, int ld, cudaStream_t st) {
  k_i_minus<<<ew_grid((long long)n * ld), 256, 0, st>>>(B, A, n, ld);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_frob(const double* X, const double* Y, int n, int ld, double* partials, double* out,
                        int mode, double tol, int* stop_flag, cudaStream_t st) {
  const long long total = (long long)n * ld;
  k_frob_partial<<<kRedBlocks, kRedThreads, 0, st>>>(X, Y, total, partials);
  k_reduce_final<<<1, 1024, 0, st>>>(partials, kRedBlocks, 2, mode, 1.0, out, tol, stop_flag);
  g_launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_reduce_partials(const double* partials, int count, double denom, double* out,
                                   double tol, int* stop_flag, cudaStream_t st) {
  k_reduce_final<<<1, 1024, 0, st>>>(partials, count, 1, 2, denom, out, tol, stop_flag);
  ++g_launches;
  return cudaGetLastError();
}

constexpr int kDotBlocks = 296;

// out[i] = <Q_i, V>_F for i < count (device), fixed reduction order; partials: count * kDotBlocks
cudaError_t launch_multidot(const double* Q, long long qstride, int count, const double* V, long long total,
                            double* partials, double* out, cudaStream_t st) {
  for (int i0 = 0; i0 < count; i0 += kMaxDots) {
    const int c = std::min(kMaxDots, count - i0);
    k_multidot<<<kDotBlocks, kRedThreads, 0, st>>>(Q + i0 * qstride, qstride, c, V, total, partials);
    k_reduce_rows<<<c, 256, 0, st>>>(partials, kDotBlocks, out + i0);
    g_launches += 2;
  }
  return cudaGetLastError();
}

cudaError_t launch_lincomb(double* out, const double* Q, long long qstride, const double* coef, int count,
                           long long total, const double* add, double sign, cudaStream_t st) {
  k_lincomb<<<ew_grid(total), 256, 0, st>>>(out, Q, qstride, coef, count, total, add, sign);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_axpy_dev(double* Y, const double* X, const double* coef, long long total, int divide,
                            cudaStream_t st) {
  k_axpy_dev<<<ew_grid(total), 256, 0, st>>>(Y, X, coef, total, divide);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_gs_keep(double* Q, long long total, const double* stats, double tol, int* keep, cudaStream_t st) {
  k_gs_keep<<<ew_grid(total), 256, 0, st>>>(Q, total, stats, tol, keep);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_sub_bcast(double* D, long long stride, int count, const double* F0, long long total,
                             cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const int gx = std::max(1, ew_grid(total) / std::max(1, count));
  k_sub_bcast<<<dim3(gx, std::min(count, 65535)), 256, 0, st>>>(D, stride, count, F0, total);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_lincomb_affine(double* out, const double* D, long long qstride, const double* coef, int count,
                                  long long total, const double* F0, const double* Gv, const double* G0,
                                  cudaStream_t st) {
  k_lincomb_affine<<<ew_grid(total), 256, 0, st>>>(out, D, qstride, coef, count, total, F0, Gv, G0);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_frob_slices_max(const double* X, const double* Y, long long stride, int count, long long total,
                                   double* partials, double* out, cudaStream_t st) {
  if (count > 0) {
    k_frob_slices<<<dim3(kSliceBlocks, count), kRedThreads, 0, st>>>(X, Y, stride, total, partials);
    ++g_launches;
  }
  k_reduce_slices_max<<<1, kSliceBlocks, 0, st>>>(partials, count, kSliceBlocks, out);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_max_ptrs(const double* const* ptrs, int count, double denom, double* out, double tol,
                            int* stop_flag, cudaStream_t st) {
  PtrList l;
  if (count < 1 || count > 64) return cudaErrorInvalidValue;
  for (int i = 0; i < count; ++i) l.p[i] = ptrs[i];
  l.count = count;
  k_max_ptrs<<<1, 1, 0, st>>>(l, denom, out, tol, stop_flag);
  ++g_launches;
  return cudaGetLastError();
}

cudaError_t launch_copy_flag(const double* metric, double tol, int* stop_flag, cudaStream_t st) {
  k_copy_flag<<<1, 1, 0, st>>>(metric, tol, stop_flag);
  ++g_launches;
  return cudaGetLastError();
}

// --------------------------------------------------------------------------------------------
// TMA tensor maps
// --------------------------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encoder() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  return fn;
}

// slab = `count` n x n matrices of leading dimension ld, matrix s at base + s * n * ld.
bool encode_slab_map(CUtensorMap* m, const double* base, int n, int ld, int count, int box_rows) {
  PFN_encodeTiled enc = get_encoder();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)count};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 8, (cuuint64_t)n * ld * 8};
  cuuint32_t box[3] = {16, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

struct MapCache {
  std::mutex mu;
  std::map<std::tuple<const double*, int, int, int, int>, CUtensorMap> maps;
};
static MapCache& map_cache() {
  static MapCache c;
  return c;
}

static bool get_map(CUtensorMap* out, const double* base, int n, int ld, int count, int box_rows) {
  auto& c = map_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  auto key = std::make_tuple(base, n, ld, count, box_rows);
  auto it = c.maps.find(key);
  if (it != c.maps.end()) {
    *out = it->second;
    return true;
  }
  if (!encode_slab_map(out, base, n, ld, count, box_rows)) return false;
  if (c.maps.size() > 4096) c.maps.clear();
  c.maps[key] = *out;
  return true;
}

void forget_maps(const double* lo, const double* hi) {
  auto& c = map_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  for (auto it = c.maps.begin(); it != c.maps.end();) {
    const double* b = std::get<0>(it->first);
    if (b >= lo && b < hi)
      it = c.maps.erase(it);
    else
      ++it;
  }
}

// --------------------------------------------------------------------------------------------
// GEMM dispatch
// --------------------------------------------------------------------------------------------
static int num_sms() {
  static int sms[kMaxDevices];
  const int dev = cur_device();
  if (!sms[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    sms[dev] = v > 0 ? v : 148;
  }
  return sms[dev];
}

template <int BM, int BN, int WM_, int WN_, int ST, int EPI>
static cudaError_t launch_cfg(const CUtensorMap& ma, const CUtensorMap& mb, const GemmParams& p, cudaStream_t st) {
  using Cfg = GemmCfg<BM, BN, WM_, WN_, ST>;
  auto kern = dgemm_tma_kernel<BM, BN, WM_, WN_, ST, EPI>;
  static int occ_dev[kMaxDevices];
  static std::once_flag once[kMaxDevices];
  const int dev = cur_device();
  std::call_once(once[dev], [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, Cfg::kThreads, Cfg::kSmemBytes);
    occ_dev[dev] = o > 0 ? o : 1;
  });
  const int occ = occ_dev[dev];
  const long long tm = (p.n + BM - 1) / BM;
  const long long tiles = ((BM == BN && p.sym) ? tm * (tm + 1) / 2 : tm * ((p.n + BN - 1) / BN)) * p.num_z;
  // Bounded persistence: a CTA owns at most ~2 ms of tiles.  Kernels are never preempted, so a grid
  // that pinned every SM for a whole (batched, ~100 ms) launch would starve the high-priority coarse
  // stream (the sequential critical path); retiring CTAs every ~2 ms lets its CTAs in.
  const double tile_s = 2.0 * BM * BN * (double)p.n / (37e12 / (num_sms() * occ));
  const long long max_tiles_per_cta = std::max<long long>(1, (long long)(g_cta_share_s / tile_s));
  // The grid is a whole number of waves (a multiple of the resident-CTA slots), so the static
  // round-robin gives every CTA floor/ceil(tiles / grid) tiles and no wave is left half empty.
  // (A per-stream atomic tile ticket was built in round 2 and measured 1.3 % slower on this kernel,
  // in its static form too -- profiles/ab_dyn_sched_regression_r02_*.jsonl -- so it was removed.)
  const long long slots = (long long)num_sms() * occ;
  const long long waves = std::max<long long>(1, (tiles + slots * max_tiles_per_cta - 1) / (slots * max_tiles_per_cta));
  long long grid = slots * waves;
  if (grid > tiles) grid = tiles;
  // Programmatic dependent launch: this grid may be scheduled while the previous kernel of the
  // stream drains; the kernel's griddepcontrol.wait orders every global access after it.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = Cfg::kSmemBytes;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ma, mb, p);
  ++g_launches;
  return e;
}

int tile_box_rows(int tile) { return tile == TILE_128 ? 128 : (tile == TILE_64 ? 64 : 32); }

int choose_tile(int n, int num_z, bool sym) {
  auto tiles = [&](int bm, int bn) {
    const long long tm = (n + bm - 1) / bm;
    return ((sym && bm == bn) ? tm * (tm + 1) / 2 : tm * ((n + bn - 1) / bn)) * num_z;
  };
  const int sms = num_sms();
  if (tiles(128, 128) >= 2LL * sms) return TILE_128;
  if (sym || tiles(64, 64) >= (long long)sms) return TILE_64;   // symmetric mode needs square tiles
  return TILE_32;
}

long long gemm_tiles(int tile, int n, int num_z, bool sym) {
  const int bm = tile_box_rows(tile), bn = (tile == TILE_128) ? 128 : 64;
  const long long tm = (n + bm - 1) / bm;
  return ((sym && bm == bn) ? tm * (tm + 1) / 2 : tm * ((n + bn - 1) / bn)) * num_z;
}

template <int EPI>
static cudaError_t dispatch_tile(int tile, const CUtensorMap& ma, const CUtensorMap& mb, const GemmParams& p,
                                 cudaStream_t st) {
  switch (tile) {
    case TILE_128: return launch_cfg<128, 128, 2, 4, 4, EPI>(ma, mb, p, st);
    case TILE_64: return launch_cfg<64, 64, 2, 2, 4, EPI>(ma, mb, p, st);
    default: return launch_cfg<32, 64, 1, 2, 4, EPI>(ma, mb, p, st);
  }
}

cudaError_t launch_gemm(int epi, int tile, const Operand& A, const Operand& B, GemmParams p, cudaStream_t st) {
  if (p.oz_nmod > 0 && epi != EPI_RESID) return launch_gemm_oz(epi, A, B, p, st);
  if (tile == TILE_AUTO) tile = choose_tile(p.n, p.num_z, p.sym != 0);
  CUtensorMap ma, mb;
  if (!get_map(&ma, A.slab, p.n, p.ld, A.count, tile_box_rows(tile))) return cudaErrorInvalidValue;
  if (!get_map(&mb, B.slab, p.n, p.ld, B.count, 16)) return cudaErrorInvalidValue;
  p.a_base = A.base;
  p.a_step = A.step;
  p.b_base = B.base;
  p.b_step = B.step;
  p.b_xor = B.xr;
  switch (epi) {
    case EPI_STORE: return dispatch_tile<EPI_STORE>(tile, ma, mb, p, st);
    case EPI_RK: return dispatch_tile<EPI_RK>(tile, ma, mb, p, st);
    case EPI_EULER: return dispatch_tile<EPI_EULER>(tile, ma, mb, p, st);
    case EPI_EULER_CORR: return dispatch_tile<EPI_EULER_CORR>(tile, ma, mb, p, st);
    case EPI_RESID: return dispatch_tile<EPI_RESID>(tile, ma, mb, p, st);
    case EPI_ACCEL: return dispatch_tile<EPI_ACCEL>(tile, ma, mb, p, st);
  }
  return cudaErrorInvalidValue;
}

// --------------------------------------------------------------------------------------------
// K10 fused fine propagator (fused.cuh)
// --------------------------------------------------------------------------------------------
template <int BM, int BN, int WM_, int WN_, int ST>
static cudaError_t launch_fused_cfg(const FusedMaps& maps, const FusedParams& p, cudaStream_t st) {
  using Cfg = GemmCfg<BM, BN, WM_, WN_, ST>;
  auto kern = fine_fused_kernel<BM, BN, WM_, WN_, ST>;
  constexpr int kSmem = Cfg::kSmemBytes + 8 * 8;   // + the tile-info ring
  static int occ_dev[kMaxDevices];
  static std::once_flag once[kMaxDevices];
  const int dev = cur_device();
  std::call_once(once[dev], [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, Cfg::kThreads, kSmem);
    occ_dev[dev] = o > 0 ? o : 1;
  });
  long long grid = (long long)num_sms() * occ_dev[dev];
  if (grid > p.total) grid = p.total;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)std::max<long long>(1, grid));
  cfg.blockDim = dim3(Cfg::kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = g_pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, maps, p);
  ++g_launches;
  return e;
}

template <int BM, int BN, int WM_, int WN_, int ST>
static cudaError_t launch_fine_fused_tiles(const FusedLaunch& L, cudaStream_t st) {
  const int n = L.n, ld = L.ld;
  FusedMaps maps;
  const int rows_a = BM;
  if (!get_map(&maps.mA_M, L.M, n, ld, 1, rows_a) || !get_map(&maps.mA_in, L.in, n, ld, L.in_count, rows_a) ||
      !get_map(&maps.mA_out, L.out, n, ld, L.out_count, rows_a) ||
      !get_map(&maps.mA_ya, L.Ya, n, ld, L.cap, rows_a) || !get_map(&maps.mA_yb, L.Yb, n, ld, L.cap, rows_a) ||
      !get_map(&maps.mB_in, L.in, n, ld, L.in_count, 16) || !get_map(&maps.mB_out, L.out, n, ld, L.out_count, 16) ||
      !get_map(&maps.mB_ya, L.Ya, n, ld, L.cap, 16) || !get_map(&maps.mB_yb, L.Yb, n, ld, L.cap, 16))
    return cudaErrorInvalidValue;
  if (L.W) {
    if (!get_map(&maps.mB_w, L.W, n, ld, L.cap, 16)) return cudaErrorInvalidValue;
  } else {
    maps.mB_w = maps.mB_ya;   // unused (only the inverse flow has a W phase)
  }
  const long long me = (long long)n * ld;
  FusedParams p;
  memset(&p, 0, sizeof(p));
  p.n = n;
  p.ld = ld;
  p.Z = L.Z;
  p.mF = L.mF;
  p.flow = L.flow;
  p.gps = (L.flow == 0) ? 2 : 1;
  p.tiles_n = (n + BN - 1) / BN;
  p.tiles_m = (n + BM - 1) / BM;
  p.T_tiles = p.tiles_m * p.tiles_n;
  p.in_base = L.ja;
  p.out_base = L.ja;
  p.h = L.h;
  p.Xin = MatRef{const_cast<double*>(L.in) + (size_t)L.ja * me, me};
  p.Xout = MatRef{L.out + (size_t)L.ja * me, me};
  p.Ya = MatRef{L.Ya, me};
  p.Yb = MatRef{L.Yb, me};
  p.W = MatRef{L.W, me};
  p.S = MatRef{L.S, me};
  p.Cterm = L.Cterm;
  p.stop_flag = L.stop_flag;
  p.sched = L.sched;
  p.total = (long long)L.mF * 4 * p.gps * L.Z * p.T_tiles;
  cudaError_t e = cudaMemsetAsync(L.sched, 0, sizeof(unsigned) * fused_sched_words(L.Z, n), st);
  if (e != cudaSuccess) return e;
  return launch_fused_cfg<BM, BN, WM_, WN_, ST>(maps, p, st);
}

// Tile configuration by parallelism, always two 4-consumer-warp CTAs per SM (one CTA's dependency
// waits and epilogue overlap the other's main loop).  Few tiles per phase (Z * T64 <= 2 per SM):
// 64 x 32 tiles, so each tile takes half as long and every slice's phase chain -- the critical path
// -- is shorter; more tiles: 64 x 64 (twice the operand reuse).  Same-box A/B (profiles/
// ab_k10_r02.jsonl): n = 256 with 16 slices 27.1 (one 8-warp CTA per SM, 64 x 64) -> 28.2 TF/s,
// cfg[1] 108.1 -> 103.1 ms; 64 x 32 everywhere loses 7-10 % at 32+ slices.  Serves n <= 512.
cudaError_t launch_fine_fused(const FusedLaunch& L, cudaStream_t st) {
  const long long tiles64 = (long long)L.Z * ((L.n + 63) / 64) * ((L.n + 63) / 64);
  if (tiles64 <= 2LL * num_sms()) return launch_fine_fused_tiles<64, 32, 2, 2, 4>(L, st);
  return launch_fine_fused_tiles<64, 64, 2, 2, 4>(L, st);
}

// --------------------------------------------------------------------------------------------
// K6 small-n launchers
// --------------------------------------------------------------------------------------------
template <int NP>
static cudaError_t fine_small_np(int flow, int n, int ld, const double* M, const double* Uin, double* Fout,
                                 long long mstride, int Z, int mF, double h, const int* flag, cudaStream_t st) {
  const size_t smem = 5 * SmallCfg<NP>::MAT * sizeof(double);   // M, X, Y_a, Y_b, W (S in registers)
  static std::once_flag once[kMaxDevices];
  std::call_once(once[cur_device()], [&] {
    cudaFuncSetAttribute(fine_smem_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  fine_smem_kernel<NP><<<Z, kSmallThreads, smem, st>>>(flow, n, ld, M, Uin, Fout, mstride, mF, h, flag);
  ++g_launches;
  return cudaGetLastError();
}

template <int NP>
static cudaError_t coarse_small_np(int flow, int n, int ld, const double* M, const double* Vin, double* U,
                                   double* Gold, const double* Fk, long long mstride, int j0, int nloc, int mG,
                                   double h, int correct, cudaStream_t st) {
  const size_t smem = 4 * SmallCfg<NP>::MAT * sizeof(double);
  static std::once_flag once[kMaxDevices];
  std::call_once(once[cur_device()], [&] {
    cudaFuncSetAttribute(coarse_smem_kernel<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  coarse_smem_kernel<NP><<<1, kSmallThreads, smem, st>>>(flow, n, ld, M, Vin, U, Gold, Fk, mstride, j0, nloc, mG, h,
                                                          correct);
  ++g_launches;
  return cudaGetLastError();
}

// K6c: Z clusters of CS CTAs, one slice per cluster (small.cuh fine_cluster_kernel)
template <int NP, int CS>
static cudaError_t fine_cluster_np(int flow, int n, int ld, const double* M, const double* Uin, double* Fout,
                                   long long mstride, int Z, int mF, double h, const int* flag, cudaStream_t st) {
  using C = ClusterCfg<NP, CS>;
  const size_t smem = 5 * C::MAT * sizeof(double);   // M, X, Y_a, Y_b, W (S in registers)
  auto kern = fine_cluster_kernel<NP, CS>;
  static std::once_flag once[kMaxDevices];
  std::call_once(once[cur_device()], [&] {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(Z * CS));
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, flow, n, ld, M, Uin, Fout, mstride, mF, h, flag);
  ++g_launches;
  return e;
}

cudaError_t launch_fine_small(int flow, int n, int ld, const double* M, const double* Uin, double* Fout,
                              long long mstride, int Z, int mF, double h, const int* flag, int cs, cudaStream_t st) {
  if (n <= 32) {
    if (cs == 2) return fine_cluster_np<32, 2>(flow, n, ld, M, Uin, Fout, mstride, Z, mF, h, flag, st);
    if (cs == 4) return fine_cluster_np<32, 4>(flow, n, ld, M, Uin, Fout, mstride, Z, mF, h, flag, st);
    return fine_small_np<32>(flow, n, ld, M, Uin, Fout, mstride, Z, mF, h, flag, st);
  }
  if (cs == 2) return fine_cluster_np<64, 2>(flow, n, ld, M, Uin, Fout, mstride, Z, mF, h, flag, st);
  if (cs == 4) return fine_cluster_np<64, 4>(flow, n, ld, M, Uin, Fout, mstride, Z, mF, h, flag, st);
  if (cs == 8) return fine_cluster_np<64, 8>(flow, n, ld, M, Uin, Fout, mstride, Z, mF, h, flag, st);
  return fine_small_np<64>(flow, n, ld, M, Uin, Fout, mstride, Z, mF, h, flag, st);
}

cudaError_t launch_coarse_small(int flow, int n, int ld, const double* M, const double* Vin, double* U, double* Gold,
                                const double* Fk, long long mstride, int j0, int nloc, int mG, double h, int correct,
                                cudaStream_t st) {
  if (n <= 32) return coarse_small_np<32>(flow, n, ld, M, Vin, U, Gold, Fk, mstride, j0, nloc, mG, h, correct, st);
  return coarse_small_np<64>(flow, n, ld, M, Vin, U, Gold, Fk, mstride, j0, nloc, mG, h, correct, st);
}

}  // namespace mfode
