/*
 * mfode.h -- C ABI of the B200 (sm_100a) parareal matrix-function solver.
 *
 * What it computes (Chehab & Petcu, arXiv 1505.07959; P:n = PAPER.md line n):
 *   f(A) as the state of the matrix ODE dX/dt = F(X), X(0) = X0 = I, solved on [0, T] with the
 *   classical parareal algorithm (Algorithm 1):
 *     Step 0     U^0_{n+1} = G(U^0_n), U^0_0 = X0                                  eq. (eqStep0)
 *     Step k+1   F(U^k_n) for all n in parallel, then sequentially
 *                U^{k+1}_{n+1} = G(U^{k+1}_n) + F(U^k_n) - G(U^k_n)               eq. (eqStepk+1) P:145-147
 *   G = m_G forward-Euler steps per slice, F = m_F classical RK4 steps per slice (P:44
 *   "Runge Kutta"; reading R1).  Flows:
 *     MFODE_FLOW_INVERSE  F(X) = X (I - A) X, T = 1  =>  X(1) = A^{-1}             P:44; eq. (eqQ)
 *     MFODE_FLOW_SQRT     F(X) = A - X^2, steady state X* = A^{1/2} for SPD A      P:46-51 eq. (stat); north star
 *   The correction is evaluated as F(U^k_n) + (G(U^{k+1}_n) - G(U^k_n)) (reading R3), which makes
 *   the prefix U^k_n, n <= k, bitwise equal to the sequential fine solution.
 *
 * Layout: every matrix crossing this ABI is n x n FP64, ROW-MAJOR, leading dimension n (host or
 * device as stated per argument).  Internally the library keeps matrices with a padded leading
 * dimension ld = round_up(n, 16) whose padding columns are zero.
 *
 * Errors: every call returns an mfode_status; nothing throws or aborts across the ABI.  On error
 * the message is available from mfode_last_error(handle) (or mfode_last_global_error() for
 * calls without a valid handle).  MFODE_NOT_CONVERGED is a warning: the result is valid.
 *
 * Ownership: input buffers are copied before the call returns (host) or before the library's
 * streams read them (device, ordered after the caller's stream); output buffers are caller-owned.
 * A handle owns all device memory, CUDA streams/events and the NCCL communicator it created and
 * is not thread-safe (one handle per host thread / rank).
 *
 * Multi-GPU: the N slices are split in contiguous blocks over the ranks (mfode_partition); slice
 * boundary states travel rank g -> g+1 over NCCL (one process per GPU, dist->nccl_uid from
 * ncclGetUniqueId broadcast by the caller) or, with dist->nccl_uid == NULL and dist->world > 1,
 * between LOGICAL ranks inside one process on one device (same partition, same kernels, boundary
 * copies by cudaMemcpyAsync; used to check P-invariance on one GPU).  In NCCL mode every rank
 * calls every function collectively.  A non-NULL nccl_uid with world == 1 creates a one-rank
 * communicator (the NCCL code path -- metric and result broadcasts -- on a single GPU).
 */
#ifndef MFODE_H
#define MFODE_H

#include <stdint.h>

#if defined(__GNUC__)
#define MFODE_API __attribute__((visibility("default")))
#else
#define MFODE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mfode_ctx mfode_ctx; /* opaque */

typedef enum {
  MFODE_OK = 0,
  MFODE_NOT_CONVERGED = 1, /* warning: K_max reached with metric > tol; result valid   */
  MFODE_EINVAL = -1,       /* bad argument (n<1, N<1, steps<1, K_max<0, tol<0, NULL, rank...)  */
  MFODE_ENOMEM = -2,       /* device allocation failed                                         */
  MFODE_ECUDA = -3,        /* CUDA runtime / driver error (message in mfode_last_error)        */
  MFODE_ENCCL = -4,        /* NCCL error or NCCL unavailable                                   */
  MFODE_ENONFINITE = -5    /* NaN/Inf met; info->bad_slice names the first bad slice   */
} mfode_status;

typedef enum {
  MFODE_FLOW_INVERSE = 0, /* F(X) = X (I - A) X, X0 = I  => X(1) = A^{-1} */
  MFODE_FLOW_SQRT = 1,    /* F(X) = A - X^2,     X0 = I  => X(inf) = A^{1/2}         */
  MFODE_FLOW_EXP = 2,     /* F(X) = A X,         X0 = I  => X(1) = exp(A)       (Ex. 2) */
  MFODE_FLOW_TRIG = 3,    /* U = (X, Y), X' = A Y, Y' = -A X, U(0) = (0, I) => U(1) = (sin A, cos A)
                             (Ex. 3, eq. eqB P:441-456 with X0 = 0).  The state is the 2n x n stack
                             [X; Y]: results and slices are 2n x n (row-major, sin block first). */
  MFODE_FLOW_AFFINE = 4   /* F(U) = A U + G, U(0) = U0: the linear inhomogeneous problem du/dt = Au + g
                             of eq. (eq1) P:72-76 with a matrix state; G = 0 and U0 = I unless set by
                             mfode_set_affine.  Example 5's dX/dt = I - A X (X -> A^{-1})
                             is the instance (A, G) -> (-A, I).  Modified parareal: Algorithm 4. */
} mfode_flow;

/* Stop rules.  The paper gives none (it plots errors); DELTA is reading R6 (endpoint delta,
 * BASELINE cfg[1]).  SPEC's CPU program uses max_n ||U^{k+1}_n - U^k_n||_F <= tol max(1,
 * ||U_0||_F) instead: that is MFODE_STOP_MAX_SLICE.  All rules stop at k = N (R15). */
typedef enum {
  MFODE_STOP_FIXED_K = 0,  /* exactly K_max correction sweeps (capped at N, reading R15)            */
  MFODE_STOP_DELTA = 1,    /* stop at the first k with ||U_N^k - U_N^{k-1}||_F/||U_N^k||_F <= tol  */
  MFODE_STOP_RESIDUAL = 2, /* stop at the first k >= 1 with the flow residual <= tol (R10)         */
  MFODE_STOP_MAX_SLICE = 3 /* stop at the first k with max_n ||U^k_n - U^{k-1}_n||_F
                              <= tol * max(1, ||U_0||_F)  (SPEC classical_parareal)        */
} mfode_stop;

typedef struct {
  int rank;                        /* this process' rank (NCCL mode); ignored in logical mode      */
  int world;                       /* number of ranks (>= 1)                                       */
  int device;                      /* CUDA device ordinal of this rank                             */
  const unsigned char *nccl_uid;   /* 128-byte ncclUniqueId (NCCL mode) or NULL (logical ranks)    */
} mfode_dist;

typedef struct {
  int k_done;          /* correction sweeps performed (0 = coarse only)                          */
  int bad_slice;       /* first slice with a non-finite state (MFODE_ENONFINITE), else -1        */
  int converged;       /* 1 if the stop criterion was met (always 1 for FIXED_K)                 */
  int world;           /* ranks used                                                             */
  double last_delta;   /* delta of the last sweep (NaN if k_done == 0)                           */
  double residual;     /* flow residual at U_N after the last sweep (see mfode_residual)         */
  double residual0;    /* flow residual after Step 0 (coarse sweep only)                         */
  double ms_total;     /* device time of the solve, max over ranks (CUDA events)                 */
  double ms_fine;      /* device time of the last rank's fine stream busy period (informational);
                          modified parareal: sum of its fine-image spans (needs phase_timing) */
  double fine_flops;   /* algorithmic flops of the fine propagations performed (all ranks)       */
  double coarse_flops; /* algorithmic flops of coarse propagations + residual GEMMs (all ranks)  */
  int gpu_launches;    /* kernels launched by the solve (all logical ranks of this process)      */
  int fine_kernel_launches;  /* fine-propagator GEMM launches of the used sweeps (this process)  */
  double fine_kernel_ms;     /* summed CUDA-event duration of those launches (fine stream)       */
  double fine_kernel_flops;  /* flops those launches executed (algorithmic; in the symmetric
                                mode only the upper-triangle tiles, i.e. ~half)                  */
  double deltas[64];   /* delta of sweep k+1 in deltas[k] (first 64 sweeps); MAX_SLICE: that metric */
  int basis_size;      /* modified parareal: F-orthonormal basis blocks of S^k at return; else 0  */
  /* Per-phase device time (CUDA events on the stream each phase runs on; summed over this
   * process' ranks).  ms_coarse: Step 0; ms_correct: correction sweeps, coarse-stream busy time
   * EXCLUDING the waits for fine results; ms_comm: boundary send/recv and metric broadcasts
   * (stream time inside the transfers, including the wait for the peer); ms_metric: stop tests. */
  double ms_coarse, ms_correct, ms_comm, ms_metric;
} mfode_solve_info;

/* ---- solver handle ------------------------------------------------------------------------ */

/* Create a solver for A (HOST, row-major n*n, caller-owned, copied before return).
 * flow: mfode_flow; T > 0: final time; N_slices >= 1; coarse_steps (m_G) >= 1; fine_steps
 * (m_F) >= 1.  dist == NULL means one rank on the current device.  Allocates every device
 * buffer the solve needs (about (3N + 3) n^2 doubles + RK scratch).  Errors: EINVAL, ENOMEM,
 * ECUDA, ENCCL.  Defined by Algorithm 1 P:133-150 with the flows of P:44 / P:46-51. */
MFODE_API int mfode_create(mfode_ctx **out, const double *A, int64_t n, int flow, double T, int N_slices,
                 int coarse_steps, int fine_steps, const mfode_dist *dist);

/* As mfode_create but A is a DEVICE pointer (row-major, leading dimension n) read on the
 * library's streams after all work already enqueued on `cuda_stream` (a cudaStream_t, or NULL
 * for the legacy default stream). */
MFODE_API int mfode_create_device(mfode_ctx **out, const double *dA, int64_t n, int flow, double T,
                        int N_slices, int coarse_steps, int fine_steps, const mfode_dist *dist,
                        void *cuda_stream);

/* Replace A by a new HOST matrix of the same n (H2D copy, then I - A is re-formed).  Lets a
 * caller solve for many matrices with one allocation.  Errors: EINVAL, ECUDA. */
MFODE_API int mfode_set_matrix(mfode_ctx *h, const double *A);

/* MFODE_FLOW_AFFINE only: set the source G (HOST row-major n*n, copied; NULL = 0) and the initial
 * state U0 (HOST row-major n*n, copied; NULL = I) of dU/dt = A U + G (eq. eq1).  Collective
 * in NCCL mode (rank 0 keeps U0).  Errors: EINVAL (other flows, NULL handle), ECUDA. */
MFODE_API int mfode_set_affine(mfode_ctx *h, const double *G, const double *U0);

/* Run Algorithm 1 from Step 0.  K_max >= 0 sweeps at most (0 = coarse sweep only); tol >= 0;
 * stop: mfode_stop.  Idempotent: each call restarts from Step 0.  info may be NULL.
 * Returns OK, NOT_CONVERGED (result valid), ENONFINITE, ECUDA, ENCCL, EINVAL. */
MFODE_API int mfode_parareal_solve(mfode_ctx *h, int K_max, double tol, int stop, mfode_solve_info *info);

/* Modified parareal for the linear flows.  Homogeneous (MFODE_FLOW_EXP, MFODE_FLOW_TRIG):
 * Algorithm 3.  Each sweep enlarges S^k = span(S^{k-1} u {U^k_n}) with the global QR
 * of Algorithm 2 (Gram-Schmidt in the Frobenius inner product, applied twice -- reading
 * R17; blocks with r_ii <= 1e-12 max(1, ||Z_i||_F) are eliminated, R16), propagates only the NEW
 * basis blocks with the fine propagator (batched, one image per block since the flows are
 * autonomous on a uniform grid), then updates U^{k+1}_{n+1} = F(P U^{k+1}_n) + G((I - P) U^{k+1}_n)
 * (eq. eq_update).  Inhomogeneous (MFODE_FLOW_AFFINE): Algorithm 4 -- Step -1 computes
 * F(0) and G(0) once, and eq. (update2) U^{k+1}_{n+1} = F(P U) + G((I - P) U) - G(0) uses
 * F(P U) = sum_i alpha_i (F(Q_i) - F(0)) + F(0) (Remark P:424-428).  The Gram-Schmidt runs on the
 * device (one host synchronisation per sweep); info->basis_size reports dim S^k.
 * max_basis (0 = (N+1)(min(K_max, N)+1)) caps the basis.  stop: FIXED_K or DELTA.  One rank.
 * Returns as mfode_parareal_solve; EINVAL for nonlinear flows or world > 1. */
MFODE_API int mfode_modified_parareal_solve(mfode_ctx *h, int K_max, double tol, int stop, int max_basis,
                                            mfode_solve_info *info);

/* The reference of P:180/P:189: S_0 = X0, S_{n+1} = F(S_n), n = 0..N-1 (sequential fine; equals
 * parareal at K = N bitwise).  Leaves the result where mfode_get_result reads it. */
MFODE_API int mfode_sequential_fine(mfode_ctx *h, mfode_solve_info *info);

/* Residual of the current result X = U_N: inverse flow ||A X - I||_F / sqrt(n);
 * sqrt flow ||A - X^2||_F / ||A||_F.  One GEMM with a fused deterministic reduction.
 * The exp flow has no residual of this kind: EINVAL (and MFODE_STOP_RESIDUAL is rejected for it). */
MFODE_API int mfode_residual(mfode_ctx *h, double *rel_residual);

/* Copy the current result X = U_N to HOST memory (row-major n*n, caller-owned).  In NCCL mode the
 * last rank broadcasts it, so every rank receives it (collective). */
MFODE_API int mfode_get_result(mfode_ctx *h, double *X);

/* Same, to a DEVICE buffer (leading dimension n), ordered before further work on cuda_stream. */
MFODE_API int mfode_get_result_device(mfode_ctx *h, double *dX, void *cuda_stream);

/* Copy U_n (0 <= n_index <= N) of the last solve to HOST memory.  The slice must be owned by this
 * process (always true in logical mode).  Errors: EINVAL. */
MFODE_API int mfode_get_slice(mfode_ctx *h, int n_index, double *U);

/* Tuning knobs (all optional).  key: "fine_batch" (max slices per batched fine launch; 0 = auto),
 * "overlap" (1 = speculative next-iteration fine work overlapped with the correction sweep,
 * 0 = strictly phased), "tile" (0 = auto, 1 = 128x128, 2 = 64x64, 3 = 32x64 GEMM tiles), "small" (1 = K6
 * shared-memory persistent kernels, default for n <= 64; 0 = one launch per GEMM), "small_cluster" (K6 CTAs
 * per slice: 1 = one CTA, 2 / 4 (/ 8 for 32 < n <= 64) = a thread-block cluster splitting the columns,
 * new stage values exchanged through distributed shared memory; -1 = auto by n and flow; bitwise identical),
 * "symmetric" (1 = f3(i)
 * half-flop symmetric GEMMs, needs A == A^T bitwise), "emulation" (f3(ii): 0 = FP64 DMMA GEMMs;
 * 8..16 = every GEMM except the residual's emulated on the int8 tensor cores with that many CRT
 * moduli, see mfode_dgemm_emulated; EINVAL if n leaves fewer than 8 bits per operand).  Process-wide
 * keys (they affect every handle of the process): "pdl" (1 = programmatic dependent launch of
 * consecutive GEMMs, default; 0 = plain stream order), "oz_pair" (1 = CTA-pair int8 GEMM kernel,
 * default; 0 = single-CTA kernel; results are bitwise identical), "cta_share_us" (bounded persistence of the
 * DMMA GEMM's CTAs, microseconds of tiles each; default 2000, 500 once a multi-rank NCCL communicator is
 * created; results are bitwise identical).  Per handle also: "fused" (-1 = auto: the one-launch fine propagator K10 for 64 < n <= 512, 0 = off,
 * 1 = on where eligible; bitwise identical), "phase_timing" (1 = per-phase CUDA-event spans in
 * mfode_solve_info, default; 0 = off) and the failure-detection test hook "inject_nan_slice" (j in 1..N-1:
 * mfode_parareal_solve overwrites U^0_j with NaN after Step 0, so the solve must end in MFODE_ENONFINITE
 * naming the first non-finite slice; 0 = off). */
MFODE_API int mfode_set_option(mfode_ctx *h, const char *key, int64_t value);

MFODE_API const char *mfode_last_error(const mfode_ctx *h);
MFODE_API void mfode_destroy(mfode_ctx *h);

/* Algorithm 5: cos(A) for a HOST matrix A (row-major n*n, copied).  m = the smallest
 * m >= 0 with 2^-m ||A||_inf <= 1, A0 = 2^-m A; C0 = cos(A0) by classical parareal on the trig
 * block flow (MFODE_FLOW_TRIG, T = 1, N_slices / coarse / fine steps as in mfode_create, K_max /
 * tol / stop as in mfode_parareal_solve); then C_{i+1} = 2 C_i^2 - I, m times, on the GPU.
 * C: HOST n*n output (caller-owned); *m_out (nullable) receives m; info (nullable) the solve's
 * info.  dist as in mfode_create (collective in NCCL mode).  Returns as mfode_parareal_solve. */
MFODE_API int mfode_cosine(const double *A, int64_t n, int N_slices, int coarse_steps, int fine_steps, int K_max,
                           double tol, int stop, const mfode_dist *dist, double *C, int *m_out,
                           mfode_solve_info *info);

/* Algorithm 8 (Example 5): accelerated steady-state inverse, dX/dt = I - A X,
 *   X^{k+1} = X^k + dt (I - A X^k + u^k),  u^{k+1} = (I - dt A) u^k,  u^0 = E0 (~ A^{-1} - X^0).
 * A, X0 (NULL -> 0), E0 (NULL -> 0: the unaccelerated flow) are HOST row-major n*n (copied).
 * Runs at most max_steps steps; with tol > 0 stops at the first checked step (every check_every
 * steps) with ||A X - I||_F / sqrt(n) <= tol.  X: HOST n*n output; *steps_done and *residual
 * (nullable) receive the step count and the final residual.  Sequential in k, one GPU.
 * Returns OK, NOT_CONVERGED (tol > 0 not met), ENONFINITE, EINVAL, ECUDA. */
MFODE_API int mfode_accel_inverse(const double *A, const double *X0, const double *E0, int64_t n, double dt,
                                  int max_steps, double tol, int check_every, double *X, int *steps_done,
                                  double *residual);

/* ---- kernel-level entry points (parity tests, roofline measurement) ---------------------- */

/* D = alpha * A_op * B_op + beta * C on DEVICE row-major n x n matrices with leading dimension
 * ld (ld >= n, ld*8 a multiple of 16 bytes; ld = n is allowed when n is even).  C may be NULL
 * when beta == 0; D must not alias A_op or B_op.  The FP64 DMMA GEMM of the fine propagator
 * (SASS DMMA.8x8x4, TMA-staged tiles).  stream: cudaStream_t or NULL.  `tile` as in
 * mfode_set_option.  Errors: EINVAL, ECUDA. */
MFODE_API int mfode_dgemm(const double *dA, const double *dB, const double *dC, double *dD, int64_t n,
                int64_t ld, double alpha, double beta, int tile, void *cuda_stream);

/* f3(ii): the same product D = alpha * A_op * B_op + beta * C computed on the int8
 * tensor cores (tcgen05.mma kind::i8, TMEM accumulators) by CRT ("Ozaki scheme II") emulation:
 * row i of A_op and column j of B_op are scaled by powers of two and rounded to integers of
 * a + 1 bits (a = floor((log2 M - 2 - ceil(log2 n)) / 2), M = product of the first n_moduli of
 * {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193}: a = 55 for 16
 * moduli at n = 4096); the integer product is formed EXACTLY from n_moduli int8 GEMMs (one per
 * modulus) and the Chinese remainder theorem, then scaled back with one correctly rounded
 * conversion.  Error per element <= 2^-(a+1) (2^e_i sum_k |B_kj| + 2^f_j sum_k |A_ik|) + rounding,
 * where 2^e_i > max_k |A_ik|, 2^f_j > max_k |B_kj|.  Deterministic (bitwise reproducible).
 * n_moduli in 2..16, n <= 32768 (int32 accumulation of uint8 residue products).  Same buffers / layout / stream semantics as mfode_dgemm.  Scratch
 * (3 n_moduli n^2 bytes + O(n)) is cached per stream until mfode_release_workspace(stream).
 * Errors: EINVAL, ECUDA, ENOMEM. */
MFODE_API int mfode_dgemm_emulated(const double *dA, const double *dB, const double *dC, double *dD, int64_t n,
                                   int64_t ld, double alpha, double beta, int n_moduli, void *cuda_stream);

/* Free the emulation scratch cached for cuda_stream (synchronises the stream). */
MFODE_API int mfode_release_workspace(void *cuda_stream);

/* One fused RK4 stage on device buffers (the fine propagator's second GEMM with its stage
 * epilogue): K = alpha*Yop*Bop + beta*C, then for stage s (1..4) with step h:
 *   s=1: S = K;           Ynext = X + (h/2) K
 *   s=2: S = S + 2K;      Ynext = X + (h/2) K
 *   s=3: S = S + 2K;      Ynext = X + h K
 *   s=4: X = X + (h/6)(S + K)           (Ynext ignored)
 * All buffers n x n, leading dimension ld, device.  Errors: EINVAL, ECUDA. */
MFODE_API int mfode_rk_stage(const double *dYop, const double *dBop, const double *dC, double alpha,
                   double beta, double *dX, double *dS, double *dYnext, int stage, double h,
                   int64_t n, int64_t ld, int tile, void *cuda_stream);

/* Deterministic Frobenius norms on device buffers: out[0] = ||X - Y||_F (Y may be NULL -> 0),
 * out[1] = ||X||_F; out is HOST memory (2 doubles).  Synchronises the stream. */
MFODE_API int mfode_frobenius(const double *dX, const double *dY, int64_t n, int64_t ld, double *out,
                    void *cuda_stream);

/* Host-only: contiguous slice partition used by the multi-rank driver: rank r of `world` owns
 * global slices [*first, *first + *count).  Blocks differ in size by at most one, larger blocks
 * first.  Errors: EINVAL. */
MFODE_API int mfode_partition(int N, int world, int rank, int *first, int *count);

/* Number of kernels this process launched through the library so far (all handles). */
MFODE_API int64_t mfode_kernel_launches(void);

MFODE_API const char *mfode_last_global_error(void);
MFODE_API const char *mfode_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MFODE_H */
