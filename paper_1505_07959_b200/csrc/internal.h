// Internal declarations shared by kernels.cu and driver.cu (not part of the C ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>

#include "gemm.cuh"

namespace mfode {

enum Tile : int { TILE_AUTO = 0, TILE_128 = 1, TILE_64 = 2, TILE_32 = 3 };

// A GEMM operand: matrix `base + z * step` of a slab of `count` n x n matrices at `slab`.
struct Operand {
  const double* slab;
  int count;
  int base;
  int step;
  int xr = 0;   // B operand only: batch z reads matrix base + (z ^ xr) * step (trig block pairs)
  unsigned long long cache_key = 0;   // != 0: a constant matrix (step 0) whose emulated-GEMM encoding may be
                                      // cached per stream; the key changes whenever its content does
};

extern std::atomic<long long> g_launches;

// Kernel attributes (max dynamic shared memory, occupancy) are per device: one-time set-up is
// keyed by the current device ordinal (a process may drive several GPUs).
constexpr int kMaxDevices = 64;
inline int cur_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) dev = 0;
  return dev;
}
extern bool g_pdl;   // programmatic dependent launch for the GEMM kernels (option "pdl")
// Bounded persistence of the DMMA GEMM: seconds of tiles per CTA (option "cta_share_us"; 2 ms, or 0.5 ms
// once a multi-rank NCCL communicator exists, whose parked kernels may hold SMs: with static tile
// ownership every SM held by another kernel delays one CTA share to the end of each launch).
extern double g_cta_share_s;

cudaError_t launch_identity(double* X, int n, int ld, int count, long long zstride, cudaStream_t st);
cudaError_t launch_i_minus(double* B, const double* A, int n, int ld, cudaStream_t st);
// *flag = 1 iff A != A^T somewhere (exact, NaN counts as a mismatch); zeroes flag first
cudaError_t launch_check_symmetric(const double* A, int n, int ld, int* flag, cudaStream_t st);
// mode 0: out[0] = ||X-Y||/||X||; mode 1: out[0] = ||X-Y||, out[1] = ||X||.  partials: 2*296 doubles.
cudaError_t launch_frob(const double* X, const double* Y, int n, int ld, double* partials, double* out, int mode,
                        double tol, int* stop_flag, cudaStream_t st);
cudaError_t launch_reduce_partials(const double* partials, int count, double denom, double* out, double tol,
                                   int* stop_flag, cudaStream_t st);
cudaError_t launch_copy_flag(const double* metric, double tol, int* stop_flag, cudaStream_t st);
// Frobenius subspace algebra (modified parareal, §3): out[i] = <Q_i, V>_F (device); partials >= count*296
cudaError_t launch_multidot(const double* Q, long long qstride, int count, const double* V, long long total,
                            double* partials, double* out, cudaStream_t st);
// out = add + sign * sum_i coef[i] Q_i (coef on the device, ascending i)
cudaError_t launch_lincomb(double* out, const double* Q, long long qstride, const double* coef, int count,
                           long long total, const double* add, double sign, cudaStream_t st);
// Y -= coef[0] X, or (divide) Y /= coef[0]
cudaError_t launch_axpy_dev(double* Y, const double* X, const double* coef, long long total, int divide,
                            cudaStream_t st);
cudaError_t launch_gemm(int epi, int tile, const Operand& A, const Operand& B, GemmParams p, cudaStream_t st);
// Gram-Schmidt keep decision on the device (stats: two launch_frob mode-1 outputs, ||Z|| and r_ii)
cudaError_t launch_gs_keep(double* Q, long long total, const double* stats, double tol, int* keep, cudaStream_t st);
// D_i -= F0 for count states of stride `stride`
cudaError_t launch_sub_bcast(double* D, long long stride, int count, const double* F0, long long total,
                             cudaStream_t st);
// out = ((sum_i coef[i] D_i + F0) + Gv) - G0   (Algorithm 4, eq. update2)
cudaError_t launch_lincomb_affine(double* out, const double* D, long long qstride, const double* coef, int count,
                                  long long total, const double* F0, const double* Gv, const double* G0,
                                  cudaStream_t st);
// out[0] = max over count states of ||X_i - Y_i||_F (0 if count == 0); partials >= 64 * count
cudaError_t launch_frob_slices_max(const double* X, const double* Y, long long stride, int count, long long total,
                                   double* partials, double* out, cudaStream_t st);
// out = max_i *ptrs[i] / denom; stop flag = out <= tol (count <= 64)
cudaError_t launch_max_ptrs(const double* const* ptrs, int count, double denom, double* out, double tol,
                            int* stop_flag, cudaStream_t st);

// f3(ii): FP64 GEMM emulated on the int8 tensor cores (ozaki.cu).  launch_gemm routes here when
// p.oz_nmod > 0 (every epilogue except EPI_RESID).  Workspaces are per stream.
constexpr int kOzMaxModuli = 16;
struct OzConst {
  int nmod;
  int abits;                           // operands are scaled to integers of magnitude <= 2^abits
  uint32_t m[kOzMaxModuli];            // moduli
  unsigned long long Mlo, Mhi;         // M = prod m_t (128-bit)
  uint32_t pw[kOzMaxModuli / 2][4];    // CRT weights of the pair groups (m_2i m_2i+1), 32-bit limbs
  uint32_t pwq[kOzMaxModuli / 2];      // pair weight / M in 0.32 fixed point (decode quotient)
  uint32_t pinv[kOzMaxModuli / 2];     // m_2i^-1 mod m_2i+1 (epilogue pair CRT)
};
bool oz_make_const(int nmod, int k, OzConst* c);
cudaError_t launch_gemm_oz(int epi, const Operand& A, const Operand& B, GemmParams p, cudaStream_t st);
cudaError_t oz_reserve(cudaStream_t st, int n, int max_z, int nmod);
void oz_release(cudaStream_t st);
void oz_forget(const double* ptr);   // drop cached encodings of a matrix about to be freed
extern bool g_oz_pair;   // option "oz_pair" (process-wide)
int choose_tile(int n, int num_z, bool sym = false);
long long gemm_tiles(int tile, int n, int num_z, bool sym = false);
void forget_maps(const double* lo, const double* hi);

constexpr int kFrobPartials = 2 * 296;
constexpr int kSmallMaxN = 64;   // K6 small-n persistent kernels handle n <= 64

// K10: the whole fine propagator (m_F RK4 steps) of Z slices in one persistent launch (fused.cuh).
// in/out: slabs of in_count/out_count states (the batch is states ja .. ja+Z-1 of both); Ya, Yb, S,
// W (inverse flow only): scratch of `cap` states; M = B (inverse) or A; Cterm = A (sqrt), G (affine)
// or null; sched: fused_sched_words(Z, n) unsigned counters (zeroed by the launcher).  flow: 0 inverse, 1 sqrt, 2 exp,
// 4 affine (one-matrix states).
constexpr int kFusedMaxN = 512;
struct FusedLaunch {
  int flow, n, ld, Z, mF, ja, in_count, out_count, cap;
  double h;
  const double* M;
  const double* Cterm;
  const double* in;
  double *out, *Ya, *Yb, *W, *S;
  const int* stop_flag;
  unsigned* sched;
};
cudaError_t launch_fine_fused(const FusedLaunch& L, cudaStream_t st);
// scheduler words of a fused launch: the ticket + per slice rowK[tm], colK[tn], colW[tn] (tiles of at
// least 32 columns / 64 rows; sized for 32 x 32 so every tile configuration fits)
inline size_t fused_sched_words(int Z, int n) {
  const size_t t = (size_t)(n + 31) / 32;
  return 1 + (size_t)Z * 3 * t;
}

// K6: all m_F RK4 steps of Z slices in shared memory; M = B (inverse) or A (sqrt).  cs = 1: one CTA
// per slice; cs = 2, 4 (n <= 32) or 2, 4, 8 (n <= 64): one cluster of cs CTAs per slice (K6c)
cudaError_t launch_fine_small(int flow, int n, int ld, const double* M, const double* Uin, double* Fout,
                              long long mstride, int Z, int mF, double h, const int* flag, int cs, cudaStream_t st);
// K6: the rank's sequential coarse sweep (Step 0 if correct == 0, else the correction) in one CTA
cudaError_t launch_coarse_small(int flow, int n, int ld, const double* M, const double* Vin, double* U, double* Gold,
                                const double* Fk, long long mstride, int j0, int nloc, int mG, double h, int correct,
                                cudaStream_t st);

}  // namespace mfode
