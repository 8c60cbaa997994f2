// Parareal driver and C ABI (include/mfode.h).
//
// Algorithm 1 of Chehab & Petcu on dense n x n FP64 matrices, B200-first:
//   * every propagation is a chain of TMA/DMMA GEMM launches with fused epilogues (gemm.cuh);
//   * the fine propagations F(U^k_n) of one sweep are batched over slices (blockIdx -> slice) on a
//     "fine" stream; Step 0 and the sequential correction run on a high-priority "coarse" stream;
//   * per-slice events let the fine work of slice chunk [ja, jb) start as soon as the coarse
//     phase has produced its inputs, and let correction step n start as soon as F(U^k_n) exists;
//     with overlap on, sweep k+1's fine work is enqueued speculatively before the host reads the
//     stop metric of sweep k, and a device flag set by the metric kernel cancels it if converged;
//   * U is ping-pong buffered by sweep parity (the correction of sweep k writes U^{k+1} while the
//     fine work of sweep k may still read U^k); Fk / Gold are single (WAR ordered by events);
//   * slices n < k are skipped in sweep k (bitwise identical, reading R14);
//   * ranks own contiguous slice blocks; boundary states move rank g -> g+1 by NCCL send/recv
//     (one process per GPU) or by cudaMemcpyAsync between logical ranks in one process.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/mfode.h"
#include "internal.h"
#include "nccl_min.h"

namespace mfode {

static thread_local std::string g_err;

static int set_global_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

// ---------------------------------------------------------------------------------------------
// NCCL, loaded at run time from the library torch already loaded (never both 2.27 and 2.28)
// ---------------------------------------------------------------------------------------------
struct NcclApi {
  bool ok = false;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commInitRankConfig)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*) = nullptr;
  ncclResult_t (*getVersion)(int*) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*bcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allreduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*errstr)(ncclResult_t) = nullptr;
};

static NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  const char* env = getenv("MFODE_NCCL_LIB");
  void* h = nullptr;
  if (env) h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
  api.commInitRankConfig = (decltype(api.commInitRankConfig))dlsym(h, "ncclCommInitRankConfig");
  api.getVersion = (decltype(api.getVersion))dlsym(h, "ncclGetVersion");
  api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
  api.send = (decltype(api.send))dlsym(h, "ncclSend");
  api.recv = (decltype(api.recv))dlsym(h, "ncclRecv");
  api.bcast = (decltype(api.bcast))dlsym(h, "ncclBroadcast");
  api.allreduce = (decltype(api.allreduce))dlsym(h, "ncclAllReduce");
  api.errstr = (decltype(api.errstr))dlsym(h, "ncclGetErrorString");
  api.ok = api.commInitRank && api.commDestroy && api.send && api.recv && api.bcast && api.allreduce;
  return api;
}

// NVTX ranges around the host-side enqueue of each phase (visible to ncu --nvtx / nsys)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// per-phase device timing (mfode_solve_info ms_coarse / ms_correct / ms_comm / ms_metric)
enum Phase : int { PH_COARSE = 0, PH_CORRECT = 1, PH_COMM = 2, PH_METRIC = 3, PH_FINE = 4, PH_COUNT = 5 };
// PH_FINE spans are recorded by the modified parareal only (its fine images are separate busy periods of
// the fine stream; the classical solve times one ev_f0..ev_f1 period instead).

// ---------------------------------------------------------------------------------------------
// context
// ---------------------------------------------------------------------------------------------
struct Rank {
  int id = 0, s0 = 0, s1 = 0, nloc = 0;
  double* U[2] = {nullptr, nullptr};  // nloc+1 matrices each; local j <-> global slice s0 + j
  double* Fk = nullptr;               // nloc: F(U^k_n), also the RK state X in place
  double* Gold = nullptr;             // nloc: G(U^k_n)
  double *Ya = nullptr, *Yb = nullptr, *W = nullptr, *S = nullptr;  // RK scratch, `cap` each
  double *Xa = nullptr, *Xb = nullptr, *Wc = nullptr;              // coarse scratch
  double* partials = nullptr;  // reductions
  double* metric = nullptr;    // device scalars [4]
  double* host_metric = nullptr;  // pinned [4]
  cudaStream_t fine = nullptr, coarse = nullptr;
  std::vector<cudaEvent_t> evC;   // nloc: coarse-phase step j done
  std::vector<cudaEvent_t> evF;   // per fine chunk
  std::vector<int> chunk_of;      // nloc: fine chunk index of slice j (current sweep)
  cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr, ev_fine_end = nullptr, ev_metric = nullptr, ev_aux = nullptr;
  cudaEvent_t ev_f0 = nullptr, ev_f1 = nullptr;
  bool fine_started = false;
  // per-chunk timing of the fine GEMM launches (roofline of the dominant kernel)
  struct ChunkTiming {
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    int iter = 0, launches = 0;
    double flops = 0.0;
  };
  std::vector<ChunkTiming> tpool;
  int tused = 0;
  // phase spans: pairs of timing events recorded on the stream the phase runs on
  std::vector<cudaEvent_t> pev;
  int pev_used = 0;
  struct Span {
    int phase, e0, e1;
  };
  std::vector<Span> spans;
  double* spart = nullptr;   // per-slice partial sums (MAX_SLICE stop test)
  unsigned* sched = nullptr; // K10 fused fine kernel: ticket + per-slice counters (1 + cap)
};

}  // namespace mfode

struct mfode_ctx {
  int n = 0, ld = 0, flow = 0, N = 0, mG = 1, mF = 1;
  int ms = 1;                // matrices per state (2 for the trig block flow)
  double T = 1.0;
  int world = 1, device = 0;
  bool nccl_mode = false;
  int my_rank = 0;           // NCCL mode: this process' rank
  ncclComm_t comm = nullptr;
  double* A = nullptr;       // n x ld
  double* B = nullptr;       // I - A (inverse flow)
  int* stop_flag = nullptr;  // device
  int cap = 1;               // fine batch capacity (slices per launch)
  int tile = 0;              // 0 auto
  bool small = false;        // K6 shared-memory kernels (n <= kSmallMaxN)
  bool sym = false;          // f3: symmetric GEMMs (upper tiles + mirror), needs A == A^T exactly
  int oz_nmod = 0;           // f3(ii): > 0 = GEMMs emulated on the int8 tensor cores with this many moduli
  bool a_symmetric = false;  // A == A^T bitwise (checked at load)
  bool overlap = true;
  int fine_batch_opt = 0;
  double normA = 0.0;        // ||A||_F
  double normU0 = 0.0;       // ||U_0||_F (host; MAX_SLICE stop test)
  double* Gsrc = nullptr;    // MFODE_FLOW_AFFINE: source G (device, zero by default)
  double* X0dev = nullptr;   // MFODE_FLOW_AFFINE: U_0 (device copy; identity by default)
  bool phase_timing = true;  // option "phase_timing"
  int fused = -1;            // option "fused": K10 one-launch fine propagator (-1 auto, 0 off, 1 on)
  int small_cs = -1;         // option "small_cluster": K6 CTAs per slice (-1 auto, 1, 2, 4, 8)
  int inject_nan = -1;       // option "inject_nan_slice": fault injection -- U^0_j := NaN after Step 0
  unsigned long long mat_gen = 0;   // content generation of A / B (emulated-GEMM encoding cache key)
  std::vector<mfode::Rank> ranks;
  // modified parareal (Algorithm 3): F-orthonormal basis Q of S^k, fine images F(Q), scratch
  double* Qb = nullptr;
  double* FQ = nullptr;
  double* mtmp = nullptr;    // 3 states: P V, (I - P) V, G((I - P) V)
  double* coef = nullptr;    // device coefficients (bcap + 8)
  double* mpart = nullptr;   // multi-dot partials
  double* gstat = nullptr;   // device Gram-Schmidt statistics (4 per candidate block)
  int* keep_dev = nullptr;   // device keep flags of the candidate blocks of a sweep
  int* keep_host = nullptr;  // pinned copy
  double* F0 = nullptr;      // Algorithm 4 Step -1: F(0), G(0) and a zero state
  double* G0 = nullptr;
  double* Z0 = nullptr;
  int bcap = 0, kcap = 0;
  // result
  int result_rank = -1;
  const double* result_ptr = nullptr;
  bool has_result = false;
  int last_k = 0;
  bool seq_mode = false;
  std::string err;
  long long launches_at_start = 0;
};

namespace mfode {

static int fail(mfode_ctx* h, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (h) h->err = buf;
  g_err = buf;
  return code;
}

#define CUDA_TRY(h, x)                                                                         \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess)                                                                     \
      return fail(h, e_ == cudaErrorMemoryAllocation ? MFODE_ENOMEM : MFODE_ECUDA, "%s: %s (%s:%d)", #x, \
                  cudaGetErrorString(e_), __FILE__, __LINE__);                                 \
  } while (0)

#define NCCL_TRY(h, x)                                                                       \
  do {                                                                                       \
    ncclResult_t r_ = (x);                                                                   \
    if (r_ != ncclSuccess)                                                                   \
      return fail(h, MFODE_ENCCL, "%s: nccl error %d (%s)", #x, (int)r_,                     \
                  nccl().errstr ? nccl().errstr(r_) : "?");                                  \
  } while (0)

#define TRY(x)              \
  do {                      \
    int s_ = (x);           \
    if (s_ < 0) return s_;  \
  } while (0)

// A state is `ms` consecutive n x ld matrices (ms = 2 for the trig block flow U = (X, Y), else 1).
static inline size_t mat_elems(const mfode_ctx* h) { return (size_t)h->n * h->ld; }
static inline size_t state_elems(const mfode_ctx* h) { return (size_t)h->ms * h->n * h->ld; }
static inline double* slot(const mfode_ctx* h, double* slab, int j) { return slab + (size_t)j * state_elems(h); }

// GEMMs per rhs evaluation: inverse X (B X) = 2; trig (A Y, -A X) = 2; sqrt, exp = 1
static int rhs_gemms(const mfode_ctx* h) {
  return (h->flow == MFODE_FLOW_INVERSE || h->flow == MFODE_FLOW_TRIG) ? 2 : 1;
}
static double rk4_flops(const mfode_ctx* h) {
  const double n3 = (double)h->n * h->n * h->n;
  return 4.0 * rhs_gemms(h) * 2.0 * n3;
}
static double euler_flops(const mfode_ctx* h) {
  const double n3 = (double)h->n * h->n * h->n;
  return rhs_gemms(h) * 2.0 * n3;
}

int partition(int N, int world, int rank, int* first, int* count) {
  if (N < 1 || world < 1 || rank < 0 || rank >= world || !first || !count) return MFODE_EINVAL;
  const int base = N / world, rem = N % world;
  *count = base + (rank < rem ? 1 : 0);
  *first = rank * base + std::min(rank, rem);
  return MFODE_OK;
}

// ---------------------------------------------------------------------------------------------
// phase spans: a span is a pair of timing events on one stream; its duration counts towards one
// phase of mfode_solve_info.  span_open returns -1 (and span_close does nothing) when disabled.
// ---------------------------------------------------------------------------------------------
static int span_event(mfode_ctx* h, Rank& R, cudaStream_t st, int* idx) {
  if (R.pev_used == (int)R.pev.size()) {
    cudaEvent_t e;
    CUDA_TRY(h, cudaEventCreate(&e));
    R.pev.push_back(e);
  }
  *idx = R.pev_used++;
  CUDA_TRY(h, cudaEventRecord(R.pev[*idx], st));
  return MFODE_OK;
}

static int span_open(mfode_ctx* h, Rank& R, cudaStream_t st, int* open) {
  *open = -1;
  if (!h->phase_timing) return MFODE_OK;
  return span_event(h, R, st, open);
}

static int span_close(mfode_ctx* h, Rank& R, cudaStream_t st, int phase, int* open) {
  if (*open < 0) return MFODE_OK;
  int e1;
  TRY(span_event(h, R, st, &e1));
  R.spans.push_back(Rank::Span{phase, *open, e1});
  *open = -1;
  return MFODE_OK;
}

// A span that is suspended around a cross-stream wait (the correction's wait for F(U^k_n)), so
// that only the stream's busy time is counted.
struct SpanCtx {
  Rank* R;
  cudaStream_t st;
  int phase;
  int open;
};

static int wait_in_span(mfode_ctx* h, SpanCtx* sc, cudaStream_t st, cudaEvent_t ev) {
  const bool was_open = sc && sc->open >= 0;
  if (was_open) TRY(span_close(h, *sc->R, sc->st, sc->phase, &sc->open));
  CUDA_TRY(h, cudaStreamWaitEvent(st, ev, 0));
  if (was_open) TRY(span_open(h, *sc->R, sc->st, &sc->open));
  return MFODE_OK;
}

// ---------------------------------------------------------------------------------------------
// one GEMM-based step: K = F-operands ... with epilogue
// ---------------------------------------------------------------------------------------------
static GemmParams base_params(const mfode_ctx* h, int num_z) {
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.n = h->n;
  p.ld = h->ld;
  p.num_z = num_z;
  p.alpha = 1.0;
  p.beta = 0.0;
  p.sym = h->sym ? 1 : 0;
  p.oz_nmod = h->oz_nmod;
  return p;
}

// rhs GEMM(s) of the flow for batch z: returns via epilogue params; Y operand given as Operand.
// inverse: W = B Y (EPI_STORE into Wbuf), then K = Y W with epilogue `epi`
// sqrt:    K = -(Y Y) + A with epilogue `epi`
// exp:     K = A Y with epilogue `epi`
static int flow_gemms(mfode_ctx* h, const Operand& Y, double* Wbuf, int Wcount, int num_z, GemmParams p, int epi,
                      cudaStream_t st, cudaEvent_t wait_before_second, SpanCtx* sc = nullptr) {
  const long long me = (long long)mat_elems(h);
  if (h->flow == MFODE_FLOW_INVERSE) {
    GemmParams q = base_params(h, num_z);
    q.Y_out = MatRef{Wbuf, me};
    q.stop_flag = p.stop_flag;
    Operand Bop{h->B, 1, 0, 0, 0, h->mat_gen};
    CUDA_TRY(h, launch_gemm(EPI_STORE, h->tile, Bop, Y, q, st));
    if (wait_before_second) TRY(wait_in_span(h, sc, st, wait_before_second));
    Operand Wop{Wbuf, Wcount, 0, 1};
    p.alpha = 1.0;
    p.beta = 0.0;
    p.oz_reuse_left = 1;   // Y was the right operand of the launch just above and is unchanged
    CUDA_TRY(h, launch_gemm(epi, h->tile, Y, Wop, p, st));
  } else if (h->flow == MFODE_FLOW_SQRT) {
    if (wait_before_second) TRY(wait_in_span(h, sc, st, wait_before_second));
    p.alpha = -1.0;
    p.beta = 1.0;
    p.C = MatRef{h->A, 0};
    CUDA_TRY(h, launch_gemm(epi, h->tile, Y, Y, p, st));
  } else if (h->flow == MFODE_FLOW_EXP || h->flow == MFODE_FLOW_AFFINE) {
    // exp: K = A Y;  affine: K = A Y + G (eq. eq1, the source as the GEMM's beta term)
    if (wait_before_second) TRY(wait_in_span(h, sc, st, wait_before_second));
    p.alpha = 1.0;
    p.beta = 0.0;
    if (h->flow == MFODE_FLOW_AFFINE) {
      p.beta = 1.0;
      p.C = MatRef{h->Gsrc, 0};
    }
    Operand Aop{h->A, 1, 0, 0, 0, h->mat_gen};
    CUDA_TRY(h, launch_gemm(epi, h->tile, Aop, Y, p, st));
  } else {   // MFODE_FLOW_TRIG: the batch runs over sub-matrices (X, Y) of each state:
             // K_X = A Y (even z), K_Y = -A X (odd z)  -- eq. (eqB) P:448-456 with X0 = 0
    if (wait_before_second) TRY(wait_in_span(h, sc, st, wait_before_second));
    p.alpha = 1.0;
    p.beta = 0.0;
    p.alt_sign = 1;
    Operand Aop{h->A, 1, 0, 0, 0, h->mat_gen};
    Operand Ysw = Y;
    Ysw.xr = 1;
    CUDA_TRY(h, launch_gemm(epi, h->tile, Aop, Ysw, p, st));
  }
  return MFODE_OK;
}

// Coarse propagator G on one slice (m_G Euler steps) on the rank's coarse stream.
// Input matrix `in` (an operand), last step writes according to `last_epi`:
//   EPI_EULER: Xout = g, and Gold (if non-null) = g
//   EPI_EULER_CORR: Uout = Fk + (g - Gold); Gold = g  (waits `fk_ready` first)
static int coarse_G(mfode_ctx* h, Rank& R, const double* in_slab, int in_count, int in_idx, int last_epi,
                    double* Xout, double* Gold, double* Fk, cudaEvent_t fk_ready, SpanCtx* sc = nullptr) {
  const double hG = h->T / ((double)h->N * h->mG);
  const long long me = (long long)mat_elems(h);
  const int ms = h->ms;
  const double* cur_slab = in_slab;
  int cur_count = in_count, cur_idx = in_idx;
  for (int i = 0; i < h->mG; ++i) {
    const bool last = (i == h->mG - 1);
    GemmParams p = base_params(h, ms);   // one state = ms sub-matrices
    p.h = hG;
    p.X_in = MatRef{const_cast<double*>(cur_slab) + (size_t)cur_idx * ms * me, me};
    double* tmp = (i % 2 == 0) ? R.Xa : R.Xb;
    int epi;
    if (!last) {
      epi = EPI_EULER;
      p.X_out = MatRef{tmp, me};
    } else if (last_epi == EPI_EULER) {
      epi = EPI_EULER;
      p.X_out = MatRef{Xout, me};
      p.Gold = MatRef{Gold, me};
    } else {
      epi = EPI_EULER_CORR;
      p.U_out = MatRef{Xout, me};
      p.Gold = MatRef{Gold, me};
      p.F_in = MatRef{Fk, me};
    }
    Operand Y{cur_slab, cur_count * ms, cur_idx * ms, 1};
    TRY(flow_gemms(h, Y, R.Wc, 1, ms, p, epi, R.coarse, (last && last_epi == EPI_EULER_CORR) ? fk_ready : nullptr,
                   sc));
    cur_slab = tmp;
    cur_count = 1;
    cur_idx = 0;
  }
  return MFODE_OK;
}

// Fine propagator F (m_F RK4 steps) on Z = jb - ja states, batched: input states ja.. of the slab
// `in` (in_count states), output states ja.. of the slab `out` (out_count states), in place.
// K10 (fused.cuh) serves moderate n with one-matrix states and plain FP64 GEMMs
static bool use_fused(const mfode_ctx* h) {
  const bool eligible = !h->small && !h->sym && h->oz_nmod == 0 && h->ms == 1 && h->flow != MFODE_FLOW_TRIG &&
                        h->n <= kFusedMaxN;
  if (h->fused == 0) return false;
  if (h->fused == 1) return eligible;
  return eligible && h->n > kSmallMaxN;
}

// K6 CTAs per slice unless the option fixes it (bitwise identical).  Measured on B200 (tools/k6c_probe.cu,
// profiles/k6c_probe_sizes_r02.log, us per RK4 step for 8 slices, CTAs per slice 1 / 2 / 4 / 8):
//   n <= 32: inverse 3.00 / 2.37 / 3.58, sqrt 1.95 / 2.24 / 3.62, exp 1.57 / 1.31 / 1.19
//   n <= 64: inverse 18.9 / 11.7 / 9.0 / 14.2, sqrt 10.3 / 8.3 / 7.8 / 13.9, exp 9.8 / 5.3 / 3.0 / 1.95
// (the sqrt flow's exchange sits on its critical path: no column-local GEMM hides it)
static int small_cluster(const mfode_ctx* h) {
  if (h->small_cs > 0) return h->small_cs;
  if (h->n <= 32) return h->flow == MFODE_FLOW_INVERSE ? 2 : (h->flow == MFODE_FLOW_EXP ? 4 : 1);
  return h->flow == MFODE_FLOW_EXP ? 8 : 4;
}

static int fine_prop(mfode_ctx* h, Rank& R, const double* in, int in_count, double* out, int out_count, int ja,
                     int jb, const int* stop_flag) {
  const int Z = jb - ja;
  const double hF = h->T / ((double)h->N * h->mF);
  const long long me = (long long)mat_elems(h);
  if (use_fused(h)) {
    if (Z > h->cap) return fail(h, MFODE_EINVAL, "fused fine batch %d exceeds capacity %d", Z, h->cap);
    FusedLaunch L;
    L.flow = h->flow;
    L.n = h->n;
    L.ld = h->ld;
    L.Z = Z;
    L.mF = h->mF;
    L.ja = ja;
    L.in_count = in_count;
    L.out_count = out_count;
    L.cap = h->cap;
    L.h = hF;
    L.M = (h->flow == MFODE_FLOW_INVERSE) ? h->B : h->A;
    L.Cterm = (h->flow == MFODE_FLOW_SQRT) ? h->A : (h->flow == MFODE_FLOW_AFFINE ? h->Gsrc : nullptr);
    L.in = in;
    L.out = out;
    L.Ya = R.Ya;
    L.Yb = R.Yb;
    L.W = R.W;
    L.S = R.S;
    L.stop_flag = stop_flag;
    L.sched = R.sched;
    CUDA_TRY(h, launch_fine_fused(L, R.fine));
    return MFODE_OK;
  }
  if (h->small) {
    const double* M = (h->flow == MFODE_FLOW_INVERSE) ? h->B : h->A;
    CUDA_TRY(h, launch_fine_small(h->flow, h->n, h->ld, M, in + (size_t)ja * state_elems(h),
                                  slot(h, out, ja), me, Z, h->mF, hF, stop_flag, small_cluster(h), R.fine));
    return MFODE_OK;
  }
  // batch index = sub-matrix index (ms per state)
  const int ms = h->ms;
  Operand Xu{in, in_count * ms, ja * ms, 1};
  Operand Xf{out, out_count * ms, ja * ms, 1};
  Operand Ya{R.Ya, h->cap * ms, 0, 1}, Yb{R.Yb, h->cap * ms, 0, 1};
  for (int i = 0; i < h->mF; ++i) {
    const Operand& X = (i == 0) ? Xu : Xf;
    double* Xin = (i == 0) ? const_cast<double*>(in) + (size_t)ja * state_elems(h) : slot(h, out, ja);
    for (int s = 1; s <= 4; ++s) {
      GemmParams p = base_params(h, Z * ms);
      p.stop_flag = stop_flag;
      p.stage = s;
      p.h = hF;
      p.X_in = MatRef{Xin, me};
      p.S = MatRef{R.S, me};
      const Operand* Yin;
      if (s == 1) {
        Yin = &X;
        p.Y_out = MatRef{R.Ya, me};
      } else if (s == 2) {
        Yin = &Ya;
        p.Y_out = MatRef{R.Yb, me};
      } else if (s == 3) {
        Yin = &Yb;
        p.Y_out = MatRef{R.Ya, me};
      } else {
        Yin = &Ya;
        p.X_out = MatRef{slot(h, out, ja), me};
        p.Y_out = MatRef{nullptr, 0};
      }
      TRY(flow_gemms(h, *Yin, R.W, h->cap, Z * ms, p, EPI_RK, R.fine, nullptr));
    }
  }
  return MFODE_OK;
}

// Fine propagator on local slices [ja, jb) of rank R: input U[par][j], output Fk[j].
static int fine_chunk(mfode_ctx* h, Rank& R, int par, int ja, int jb, const int* stop_flag) {
  return fine_prop(h, R, R.U[par], R.nloc + 1, R.Fk, R.nloc, ja, jb, stop_flag);
}

// Slices per batched fine launch: balanced chunks whose total number of persistent-CTA tile
// rounds (tiles / concurrently resident CTAs, rounded up per launch) is minimal -- the last,
// partial round of every launch is idle tensor time.  Ties go to larger chunks (fewer launches).
static int fine_chunk_size(const mfode_ctx* h, int active) {
  if (h->small || use_fused(h) || active <= 1) return std::max(1, std::min(active, h->cap));
  const int tile = (h->tile != TILE_AUTO) ? h->tile : choose_tile(h->n, std::min(active, h->cap), h->sym);
  const long long t1 = gemm_tiles(tile, h->n, 1, h->sym) * h->ms;   // tiles of one slice's GEMM launch
  const long long slots = 148LL * (tile == TILE_128 ? 1 : (tile == TILE_64 ? 2 : 4));
  const long long launches = (long long)h->mF * 4 * (h->flow == MFODE_FLOW_INVERSE ? 2 : 1);
  const long long euler_gemms = (long long)h->mG * (h->flow == MFODE_FLOW_INVERSE ? 2 : 1);
  const long long coarse_rounds = (t1 + slots - 1) / slots;
  int best = 1;
  long long best_cost = -1;
  for (int s = std::min(active, h->cap); s >= 1; --s) {
    const int nch = (active + s - 1) / s;
    const int q = active / nch, r = active % nch;   // r chunks of q+1, nch-r of q
    // fine tile rounds (every launch's last round is partly idle) + the correction steps of the
    // last chunk, which can only run after the whole fine sweep (the sweep's tail)
    const long long cost =
        launches * (r * ((t1 * (q + 1) + slots - 1) / slots) + (nch - r) * ((t1 * q + slots - 1) / slots)) +
        (long long)(r == nch ? q + 1 : q) * euler_gemms * coarse_rounds;
    if (best_cost < 0 || cost < best_cost) {
      best_cost = cost;
      best = (active + nch - 1) / nch;
    }
  }
  return best;
}

static int enqueue_fine(mfode_ctx* h, Rank& R, int k, bool speculative) {
  if (k >= R.s1) return MFODE_OK;
  NvtxRange nv(speculative ? "mfode:fine(speculative)" : "mfode:fine");
  const int ja0 = std::max(0, k - R.s0);
  const int active = R.nloc - ja0;
  if (active <= 0) return MFODE_OK;
  const int size = fine_chunk_size(h, active);
  const int nchunks = (active + size - 1) / size;
  if ((int)R.evF.size() < nchunks) {
    int old = (int)R.evF.size();
    R.evF.resize(nchunks);
    for (int c = old; c < nchunks; ++c) CUDA_TRY(h, cudaEventCreateWithFlags(&R.evF[c], cudaEventDisableTiming));
  }
  const int par = k % 2;
  const int* flag = speculative ? h->stop_flag : nullptr;
  for (int c = 0; c < nchunks; ++c) {
    const int ja = ja0 + c * size;
    const int jb = std::min(R.nloc, ja + size);
    if (ja >= jb) break;
    CUDA_TRY(h, cudaStreamWaitEvent(R.fine, R.evC[jb - 1], 0));
    if (!R.fine_started) {
      CUDA_TRY(h, cudaEventRecord(R.ev_f0, R.fine));
      R.fine_started = true;
    }
    if (R.tused == (int)R.tpool.size()) {
      R.tpool.emplace_back();
      CUDA_TRY(h, cudaEventCreate(&R.tpool.back().t0));
      CUDA_TRY(h, cudaEventCreate(&R.tpool.back().t1));
    }
    Rank::ChunkTiming& ct = R.tpool[R.tused++];
    ct.iter = k;
    ct.launches = (h->small || use_fused(h)) ? 1 : h->mF * 4 * (h->flow == MFODE_FLOW_INVERSE ? 2 : 1);
    ct.flops = (double)(jb - ja) * h->mF * rk4_flops(h);
    if (h->sym && !h->small) {   // executed (not algorithmic) flops: only upper-triangle tiles run
      const int tl = (h->tile != TILE_AUTO) ? h->tile : choose_tile(h->n, (jb - ja) * h->ms, true);
      ct.flops *= (double)gemm_tiles(tl, h->n, 1, true) / (double)gemm_tiles(tl, h->n, 1, false);
    }
    CUDA_TRY(h, cudaEventRecord(ct.t0, R.fine));
    TRY(fine_chunk(h, R, par, ja, jb, flag));
    CUDA_TRY(h, cudaEventRecord(ct.t1, R.fine));
    CUDA_TRY(h, cudaEventRecord(R.evF[c], R.fine));
    for (int j = ja; j < jb; ++j) R.chunk_of[j] = c;
  }
  CUDA_TRY(h, cudaEventRecord(R.ev_f1, R.fine));
  return MFODE_OK;
}

// boundary: rank g's U[par][nloc] -> rank g+1's U[par][0]
static int send_boundary(mfode_ctx* h, Rank& R, int par) {
  if (R.id >= h->world - 1) return MFODE_OK;
  if (h->nccl_mode) {
    NvtxRange nv("mfode:send_boundary");
    int sp;
    TRY(span_open(h, R, R.coarse, &sp));
    NCCL_TRY(h, nccl().send(slot(h, R.U[par], R.nloc), state_elems(h), ncclFloat64, R.id + 1, h->comm, R.coarse));
    TRY(span_close(h, R, R.coarse, PH_COMM, &sp));
  } else {
    // logical ranks: the receiver copies after the sender's event (recorded in evC[nloc-1])
  }
  return MFODE_OK;
}

static int recv_boundary(mfode_ctx* h, Rank& R, int par) {
  if (R.id == 0) return MFODE_OK;
  NvtxRange nv("mfode:recv_boundary");
  int sp;
  if (h->nccl_mode) {
    TRY(span_open(h, R, R.coarse, &sp));
    NCCL_TRY(h, nccl().recv(R.U[par], state_elems(h), ncclFloat64, R.id - 1, h->comm, R.coarse));
  } else {
    Rank& P = h->ranks[R.id - 1];
    CUDA_TRY(h, cudaStreamWaitEvent(R.coarse, P.evC[P.nloc - 1], 0));
    TRY(span_open(h, R, R.coarse, &sp));
    CUDA_TRY(h, cudaMemcpyAsync(R.U[par], slot(h, P.U[par], P.nloc), state_elems(h) * sizeof(double),
                                cudaMemcpyDeviceToDevice, R.coarse));
  }
  TRY(span_close(h, R, R.coarse, PH_COMM, &sp));
  return MFODE_OK;
}

static int coarse_small_sweep(mfode_ctx* h, Rank& R, const double* Vin, double* Uslab, int j0, int correct) {
  const double hG = h->T / ((double)h->N * h->mG);
  const double* M = (h->flow == MFODE_FLOW_INVERSE) ? h->B : h->A;
  int sp;
  TRY(span_open(h, R, R.coarse, &sp));
  CUDA_TRY(h, launch_coarse_small(h->flow, h->n, h->ld, M, Vin, Uslab, R.Gold, R.Fk, (long long)mat_elems(h), j0,
                                  R.nloc, h->mG, hG, correct, R.coarse));
  TRY(span_close(h, R, R.coarse, correct ? PH_CORRECT : PH_COARSE, &sp));
  for (int j = j0; j < R.nloc; ++j) CUDA_TRY(h, cudaEventRecord(R.evC[j], R.coarse));
  return MFODE_OK;
}

static int enqueue_step0(mfode_ctx* h, Rank& R) {
  NvtxRange nv("mfode:step0");
  TRY(recv_boundary(h, R, 0));
  if (h->small) {
    TRY(coarse_small_sweep(h, R, R.U[0], R.U[0], 0, 0));
    TRY(send_boundary(h, R, 0));
    return MFODE_OK;
  }
  int sp;
  TRY(span_open(h, R, R.coarse, &sp));
  for (int j = 0; j < R.nloc; ++j) {
    TRY(coarse_G(h, R, R.U[0], R.nloc + 1, j, EPI_EULER, slot(h, R.U[0], j + 1), slot(h, R.Gold, j), nullptr,
                 nullptr));
    CUDA_TRY(h, cudaEventRecord(R.evC[j], R.coarse));
  }
  TRY(span_close(h, R, R.coarse, PH_COARSE, &sp));
  TRY(send_boundary(h, R, 0));
  return MFODE_OK;
}

static int enqueue_correction(mfode_ctx* h, Rank& R, int k) {
  if (k >= R.s1) return MFODE_OK;
  NvtxRange nv("mfode:correction");
  const int cur = k % 2, nxt = (k + 1) % 2;
  const int j0 = std::max(0, k - R.s0);
  if (k < R.s0) {
    // NCCL: the upstream rank sends its boundary only after ITS correction sweep, i.e. about when this
    // rank's fine sweep ends; posting the receive earlier would park NCCL's kernel on SMs for the whole
    // fine sweep (every persistent fine launch would then run with a tail).  Waiting for this rank's
    // last fine chunk first costs nothing on the critical path.
    if (h->nccl_mode && R.nloc > 0) CUDA_TRY(h, cudaStreamWaitEvent(R.coarse, R.evF[R.chunk_of[R.nloc - 1]], 0));
    TRY(recv_boundary(h, R, nxt));
  }
  if (h->small) {
    // the single-CTA sweep needs every F(U^k_n), n >= j0, before it starts
    for (int j = j0; j < R.nloc; ++j)
      if (j == j0 || R.chunk_of[j] != R.chunk_of[j - 1]) CUDA_TRY(h, cudaStreamWaitEvent(R.coarse, R.evF[R.chunk_of[j]], 0));
    const double* Vin = (k >= R.s0) ? slot(h, R.U[cur], j0) : R.U[nxt];
    TRY(coarse_small_sweep(h, R, Vin, R.U[nxt], j0, 1));
    TRY(send_boundary(h, R, nxt));
    return MFODE_OK;
  }
  // K10: the fused fine sweep is one launch holding every SM, so no coarse GEMM can run beside it;
  // wait for it here (outside the span) so that ms_correct stays the correction's own time
  if (use_fused(h) && R.nloc > 0) CUDA_TRY(h, cudaStreamWaitEvent(R.coarse, R.evF[R.chunk_of[R.nloc - 1]], 0));
  SpanCtx sc{&R, R.coarse, PH_CORRECT, -1};
  TRY(span_open(h, R, R.coarse, &sc.open));
  for (int j = j0; j < R.nloc; ++j) {
    const double* in_slab;
    int in_idx;
    if (j == j0 && k >= R.s0) {
      in_slab = R.U[cur];
      in_idx = j0;
    } else {
      in_slab = R.U[nxt];
      in_idx = j;
    }
    TRY(coarse_G(h, R, in_slab, R.nloc + 1, in_idx, EPI_EULER_CORR, slot(h, R.U[nxt], j + 1), slot(h, R.Gold, j),
                 slot(h, R.Fk, j), R.evF[R.chunk_of[j]], &sc));
    CUDA_TRY(h, cudaEventRecord(R.evC[j], R.coarse));
  }
  TRY(span_close(h, R, R.coarse, PH_CORRECT, &sc.open));
  TRY(send_boundary(h, R, nxt));
  return MFODE_OK;
}

// flow residual of X (device, on rank R's coarse stream) into R.metric[idx]
static int enqueue_residual(mfode_ctx* h, Rank& R, const double* slab, int count, int idx, int out_idx, double tol,
                            int* flag) {
  const int tile = (h->tile != TILE_AUTO) ? h->tile : choose_tile(h->n, 1, h->sym);
  GemmParams p = base_params(h, 1);
  p.partials = R.partials;
  const long long ntiles = gemm_tiles(tile, h->n, 1, h->sym);
  double denom;
  if (h->flow == MFODE_FLOW_INVERSE) {
    p.shift = 1.0;
    Operand Aop{h->A, 1, 0, 0, 0, h->mat_gen};
    Operand Xop{slab, count, idx, 0};
    CUDA_TRY(h, launch_gemm(EPI_RESID, tile, Aop, Xop, p, R.coarse));
    denom = sqrt((double)h->n);
  } else {
    p.alpha = -1.0;
    p.beta = 1.0;
    p.C = MatRef{h->A, 0};
    Operand Xop{slab, count, idx, 0};
    CUDA_TRY(h, launch_gemm(EPI_RESID, tile, Xop, Xop, p, R.coarse));
    denom = h->normA;
  }
  CUDA_TRY(h, launch_reduce_partials(R.partials, (int)ntiles, denom, R.metric + out_idx, tol, flag, R.coarse));
  return MFODE_OK;
}

static int alloc_rank(mfode_ctx* h, Rank& R) {
  const size_t me = state_elems(h) * sizeof(double);   // bytes of one state (ms matrices)
  CUDA_TRY(h, cudaMalloc(&R.U[0], me * (R.nloc + 1)));
  CUDA_TRY(h, cudaMalloc(&R.U[1], me * (R.nloc + 1)));
  CUDA_TRY(h, cudaMalloc(&R.Fk, me * std::max(1, R.nloc)));
  CUDA_TRY(h, cudaMalloc(&R.Gold, me * std::max(1, R.nloc)));
  CUDA_TRY(h, cudaMalloc(&R.Ya, me * h->cap));
  CUDA_TRY(h, cudaMalloc(&R.Yb, me * h->cap));
  CUDA_TRY(h, cudaMalloc(&R.S, me * h->cap));
  if (h->flow == MFODE_FLOW_INVERSE) CUDA_TRY(h, cudaMalloc(&R.W, me * h->cap));
  CUDA_TRY(h, cudaMalloc(&R.Xa, me));
  CUDA_TRY(h, cudaMalloc(&R.Xb, me));
  CUDA_TRY(h, cudaMalloc(&R.Wc, me));
  const long long maxtiles = std::max<long long>(gemm_tiles(TILE_32, h->n, 1), kFrobPartials);
  CUDA_TRY(h, cudaMalloc(&R.partials, sizeof(double) * (maxtiles + 16)));
  CUDA_TRY(h, cudaMalloc(&R.metric, sizeof(double) * 8));
  CUDA_TRY(h, cudaMalloc(&R.spart, sizeof(double) * 64 * (size_t)(R.nloc + 1)));
  CUDA_TRY(h, cudaMalloc(&R.sched, sizeof(unsigned) * fused_sched_words(h->cap, std::min(h->n, kFusedMaxN))));
  CUDA_TRY(h, cudaMallocHost(&R.host_metric, sizeof(double) * 8));
  // zero everything once: padding columns stay zero forever (kernels never write them)
  CUDA_TRY(h, cudaMemset(R.U[0], 0, me * (R.nloc + 1)));
  CUDA_TRY(h, cudaMemset(R.U[1], 0, me * (R.nloc + 1)));
  CUDA_TRY(h, cudaMemset(R.Fk, 0, me * std::max(1, R.nloc)));
  CUDA_TRY(h, cudaMemset(R.Gold, 0, me * std::max(1, R.nloc)));
  CUDA_TRY(h, cudaMemset(R.Ya, 0, me * h->cap));
  CUDA_TRY(h, cudaMemset(R.Yb, 0, me * h->cap));
  CUDA_TRY(h, cudaMemset(R.S, 0, me * h->cap));
  if (R.W) CUDA_TRY(h, cudaMemset(R.W, 0, me * h->cap));
  CUDA_TRY(h, cudaMemset(R.Xa, 0, me));
  CUDA_TRY(h, cudaMemset(R.Xb, 0, me));
  CUDA_TRY(h, cudaMemset(R.Wc, 0, me));
  int lo, hi;
  CUDA_TRY(h, cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CUDA_TRY(h, cudaStreamCreateWithPriority(&R.fine, cudaStreamNonBlocking, lo));
  CUDA_TRY(h, cudaStreamCreateWithPriority(&R.coarse, cudaStreamNonBlocking, hi));
  R.evC.resize(std::max(1, R.nloc));
  for (auto& e : R.evC) CUDA_TRY(h, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  R.chunk_of.assign(std::max(1, R.nloc), 0);
  CUDA_TRY(h, cudaEventCreate(&R.ev_t0));
  CUDA_TRY(h, cudaEventCreate(&R.ev_t1));
  CUDA_TRY(h, cudaEventCreate(&R.ev_f0));
  CUDA_TRY(h, cudaEventCreate(&R.ev_f1));
  CUDA_TRY(h, cudaEventCreateWithFlags(&R.ev_fine_end, cudaEventDisableTiming));
  CUDA_TRY(h, cudaEventCreateWithFlags(&R.ev_metric, cudaEventDisableTiming));
  CUDA_TRY(h, cudaEventCreateWithFlags(&R.ev_aux, cudaEventDisableTiming));
  return MFODE_OK;
}

static void free_rank(mfode_ctx* h, Rank& R) {
  double* bufs[] = {R.U[0], R.U[1], R.Fk, R.Gold, R.Ya, R.Yb, R.W, R.S, R.Xa, R.Xb, R.Wc, R.partials, R.metric, R.spart};
  const size_t me = state_elems(h);
  for (double* b : bufs)
    if (b) {
      forget_maps(b, b + me * (size_t)(std::max(R.nloc, h->cap) + 2));
      cudaFree(b);
    }
  if (R.host_metric) cudaFreeHost(R.host_metric);
  if (R.sched) cudaFree(R.sched);
  if (R.fine) {
    cudaStreamSynchronize(R.fine);
    oz_release(R.fine);
    cudaStreamDestroy(R.fine);
  }
  if (R.coarse) {
    cudaStreamSynchronize(R.coarse);
    oz_release(R.coarse);
    cudaStreamDestroy(R.coarse);
  }
  for (auto e : R.evC) cudaEventDestroy(e);
  for (auto e : R.evF) cudaEventDestroy(e);
  for (auto& ct : R.tpool) {
    cudaEventDestroy(ct.t0);
    cudaEventDestroy(ct.t1);
  }
  for (auto e : R.pev) cudaEventDestroy(e);
  cudaEvent_t evs[] = {R.ev_t0, R.ev_t1, R.ev_f0, R.ev_f1, R.ev_fine_end, R.ev_metric, R.ev_aux};
  for (auto e : evs)
    if (e) cudaEventDestroy(e);
}

// A (device, leading dim ld_src) -> h->A (ld), B = I - A, ||A||_F
static int load_matrix(mfode_ctx* h, const double* src, bool host, size_t ld_src, cudaStream_t st) {
  static std::atomic<unsigned long long> gen{0};
  h->mat_gen = ++gen;   // A and B change: cached encodings keyed by the old generation are never hit again
  CUDA_TRY(h, cudaMemcpy2DAsync(h->A, h->ld * sizeof(double), src, ld_src * sizeof(double), h->n * sizeof(double),
                                h->n, host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
  if (h->B) CUDA_TRY(h, launch_i_minus(h->B, h->A, h->n, h->ld, st));
  Rank& R = h->ranks[0];
  CUDA_TRY(h, launch_frob(h->A, nullptr, h->n, h->ld, R.partials, R.metric, 1, 0.0, nullptr, st));
  // exact symmetry of A (the symmetric GEMM mode f3 relies on every iterate being a symmetric
  // polynomial in A), checked on the device copy: A == A^T element by element (`!=`, so NaN fails)
  int* asym_flag = reinterpret_cast<int*>(R.metric + 7);
  CUDA_TRY(h, launch_check_symmetric(h->A, h->n, h->ld, asym_flag, st));
  CUDA_TRY(h, cudaMemcpyAsync(R.host_metric, R.metric, 8 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  h->normA = R.host_metric[1];
  h->has_result = false;
  {
    int asym = 0;
    memcpy(&asym, R.host_metric + 7, sizeof(int));
    const bool s = (asym == 0);
    h->a_symmetric = s;
    if (!s) h->sym = false;
  }
  return MFODE_OK;
}

static int create_impl(mfode_ctx** out, const double* A, bool host, int64_t n, int flow, double T, int N, int mG,
                       int mF, const mfode_dist* dist, cudaStream_t user_stream) {
  if (!out) return set_global_err(MFODE_EINVAL, "out is NULL");
  *out = nullptr;
  if (!A) return set_global_err(MFODE_EINVAL, "A is NULL");
  if (n < 1 || n > 65536) return set_global_err(MFODE_EINVAL, "n=%lld out of range [1, 65536]", (long long)n);
  if (flow != MFODE_FLOW_INVERSE && flow != MFODE_FLOW_SQRT && flow != MFODE_FLOW_EXP && flow != MFODE_FLOW_TRIG &&
      flow != MFODE_FLOW_AFFINE)
    return set_global_err(MFODE_EINVAL, "unknown flow %d", flow);
  if (!(T > 0.0) || !std::isfinite(T)) return set_global_err(MFODE_EINVAL, "T must be finite and > 0");
  if (N < 1 || mG < 1 || mF < 1) return set_global_err(MFODE_EINVAL, "N, coarse_steps, fine_steps must be >= 1");
  int world = dist ? dist->world : 1;
  if (world < 1 || world > N) return set_global_err(MFODE_EINVAL, "world=%d must be in [1, N=%d]", world, N);
  std::unique_ptr<mfode_ctx> h(new mfode_ctx());
  h->n = (int)n;
  h->ld = (int)((n + 15) / 16 * 16);
  h->flow = flow;
  h->T = T;
  h->N = N;
  h->mG = mG;
  h->mF = mF;
  h->world = world;
  h->ms = (flow == MFODE_FLOW_TRIG) ? 2 : 1;
  // K6 small-n kernels: the flows whose right-hand side they implement (not the affine source)
  h->small = (h->n <= kSmallMaxN) && h->ms == 1 && flow != MFODE_FLOW_AFFINE;
  h->normU0 = std::sqrt((double)n);   // ||I||_F (and ||(0; I)||_F for the trig flow)
  int dev = 0;
  if (dist) dev = dist->device;
  else cudaGetDevice(&dev);
  h->device = dev;
  if (cudaSetDevice(dev) != cudaSuccess) return set_global_err(MFODE_ECUDA, "cudaSetDevice(%d) failed", dev);
  h->nccl_mode = dist && dist->nccl_uid;   // world == 1 is a one-rank communicator (same code path)
  if (h->nccl_mode) {
    if (dist->rank < 0 || dist->rank >= world) return set_global_err(MFODE_EINVAL, "rank out of range");
    h->my_rank = dist->rank;
    if (!nccl().ok) return set_global_err(MFODE_ENCCL, "NCCL library not available (set MFODE_NCCL_LIB)");
    ncclUniqueId uid;
    memcpy(&uid, dist->nccl_uid, sizeof(uid));
    // Cap NCCL's CTAs (config.maxCTAs, default 8; env MFODE_NCCL_MAX_CTAS): a downstream rank posts
    // its boundary receive while the upstream rank's fine sweep runs, and those NCCL kernels stay
    // resident on SMs that the fine DMMA grid would otherwise use.
    int ver = 0;
    ncclResult_t r;
    if (nccl().commInitRankConfig && nccl().getVersion && nccl().getVersion(&ver) == ncclSuccess && ver >= 22800) {
      ncclConfig_t cfg = nccl_config_init(22809);
      const char* mc = getenv("MFODE_NCCL_MAX_CTAS");
      cfg.minCTAs = 1;
      cfg.maxCTAs = mc ? std::max(1, atoi(mc)) : 8;
      r = nccl().commInitRankConfig(&h->comm, world, uid, dist->rank, &cfg);
    } else {
      r = nccl().commInitRank(&h->comm, world, uid, dist->rank);
    }
    if (r != ncclSuccess) return set_global_err(MFODE_ENCCL, "ncclCommInitRank failed: %d", (int)r);
    if (world > 1 && g_cta_share_s > 0.5e-3) g_cta_share_s = 0.5e-3;   // see internal.h
  }
  // fine batch capacity: enough batched tiles to fill the chip, bounded by the slice count
  {
    // Scratch for up to `cap` in-flight slices (3-4 matrices each) within a 16 GiB budget; the
    // chunk size actually used per sweep is chosen by fine_chunk_size() to minimise tile rounds.
    const int nloc_max = (N + world - 1) / world;
    const double per_slice = 4.0 * 8.0 * h->ms * (double)h->n * (double)h->ld;
    const int budget = (int)std::max(1.0, std::floor(16.0 * (1LL << 30) / per_slice));
    h->cap = std::max(1, std::min(nloc_max, budget));
  }
  // ranks
  const int nranks_here = h->nccl_mode ? 1 : world;
  h->ranks.resize(nranks_here);
  for (int i = 0; i < nranks_here; ++i) {
    Rank& R = h->ranks[i];
    R.id = h->nccl_mode ? h->my_rank : i;
    int first, count;
    partition(N, world, R.id, &first, &count);
    R.s0 = first;
    R.s1 = first + count;
    R.nloc = count;
  }
  mfode_ctx* hp = h.get();
  const size_t me = mat_elems(hp) * sizeof(double);
  if (cudaMalloc(&hp->A, me) != cudaSuccess) return set_global_err(MFODE_ENOMEM, "alloc A failed");
  cudaMemset(hp->A, 0, me);
  if (flow == MFODE_FLOW_INVERSE) {
    if (cudaMalloc(&hp->B, me) != cudaSuccess) return set_global_err(MFODE_ENOMEM, "alloc B failed");
    cudaMemset(hp->B, 0, me);
  }
  if (flow == MFODE_FLOW_AFFINE) {   // source G = 0 and U_0 = I until mfode_set_affine
    if (cudaMalloc(&hp->Gsrc, me) != cudaSuccess || cudaMalloc(&hp->X0dev, me) != cudaSuccess) {
      mfode_destroy(h.release());
      return set_global_err(MFODE_ENOMEM, "alloc source failed");
    }
    cudaMemset(hp->Gsrc, 0, me);
    launch_identity(hp->X0dev, hp->n, hp->ld, 1, 0, nullptr);
  }
  if (cudaMalloc(&hp->stop_flag, sizeof(int)) != cudaSuccess) return set_global_err(MFODE_ENOMEM, "alloc flag failed");
  cudaMemset(hp->stop_flag, 0, sizeof(int));
  for (auto& R : hp->ranks) {
    int s = alloc_rank(hp, R);
    if (s < 0) {
      std::string e = hp->err;
      mfode_destroy(h.release());
      return set_global_err(s, "%s", e.c_str());
    }
  }
  // X0 = I in slot 0 of both U buffers of rank 0 (logical or NCCL), once.  Trig block flow:
  // U(0) = (sin 0, cos 0) = (0, I) (eq. eqB with X0 = 0): the identity is sub-matrix 1.
  for (auto& R : hp->ranks)
    if (R.id == 0) {
      const size_t off = (hp->flow == MFODE_FLOW_TRIG) ? mat_elems(hp) : 0;
      launch_identity(R.U[0] + off, hp->n, hp->ld, 1, 0, R.coarse);
      launch_identity(R.U[1] + off, hp->n, hp->ld, 1, 0, R.coarse);
    }
  cudaStream_t st = hp->ranks[0].coarse;
  if (!host && user_stream != (cudaStream_t)-1) {
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    cudaEventRecord(ev, user_stream);
    cudaStreamWaitEvent(st, ev, 0);
    cudaEventDestroy(ev);
  }
  int s = load_matrix(hp, A, host, (size_t)n, st);
  if (s < 0) {
    std::string e = hp->err;
    mfode_destroy(h.release());
    return set_global_err(s, "%s", e.c_str());
  }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    mfode_destroy(h.release());
    return set_global_err(MFODE_ECUDA, "create: device error");
  }
  *out = h.release();
  return MFODE_OK;
}

static Rank& last_rank(mfode_ctx* h) { return h->ranks.back(); }
static bool owns_last(mfode_ctx* h) { return last_rank(h).id == h->world - 1; }

// host-visible broadcast of metric[idx] from the last rank (NCCL) -> every rank's host_metric[idx]
static int fetch_metric(mfode_ctx* h, int idx, int count) {
  Rank& L = last_rank(h);
  if (h->nccl_mode) {
    int sp;
    TRY(span_open(h, L, L.coarse, &sp));
    NCCL_TRY(h, nccl().bcast(L.metric + idx, L.metric + idx, count, ncclFloat64, h->world - 1, h->comm, L.coarse));
    TRY(span_close(h, L, L.coarse, PH_COMM, &sp));
  }
  CUDA_TRY(h, cudaMemcpyAsync(L.host_metric + idx, L.metric + idx, count * sizeof(double), cudaMemcpyDeviceToHost,
                              L.coarse));
  CUDA_TRY(h, cudaEventRecord(L.ev_metric, L.coarse));
  return MFODE_OK;
}

static int first_bad_slice(mfode_ctx* h) {
  // scan U (latest buffers) of every local rank for non-finite entries; -1 if none
  for (auto& R : h->ranks) {
    for (int j = 0; j <= R.nloc; ++j) {
      const int gidx = R.s0 + j;
      const int par = (gidx <= h->last_k ? gidx : h->last_k) % 2;
      launch_frob(slot(h, R.U[par], j), nullptr, h->ms * h->n, h->ld, R.partials, R.metric + 6, 1, 0.0, nullptr,
                  R.coarse);
      cudaMemcpyAsync(R.host_metric + 6, R.metric + 6, 2 * sizeof(double), cudaMemcpyDeviceToHost, R.coarse);
      cudaStreamSynchronize(R.coarse);
      if (!std::isfinite(R.host_metric[7])) return gidx;
    }
  }
  return -1;
}

// Sum the recorded phase spans of every local rank into info (events already complete).
static int collect_phases(mfode_ctx* h, mfode_solve_info* info) {
  double ph[PH_COUNT] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (auto& R : h->ranks)
    for (const auto& sp : R.spans) {
      float ms = 0.f;
      CUDA_TRY(h, cudaEventSynchronize(R.pev[sp.e1]));
      CUDA_TRY(h, cudaEventElapsedTime(&ms, R.pev[sp.e0], R.pev[sp.e1]));
      ph[sp.phase] += ms;
    }
  info->ms_coarse = ph[PH_COARSE];
  info->ms_correct = ph[PH_CORRECT];
  info->ms_comm = ph[PH_COMM];
  info->ms_metric = ph[PH_METRIC];
  if (ph[PH_FINE] > 0.0) info->ms_fine = ph[PH_FINE];
  return MFODE_OK;
}

// SPEC's stop metric: max_n ||U^{k+1}_n - U^k_n||_F / max(1, ||U_0||_F) over every slice of
// every rank -> last rank's metric[0] (and `flag`).  Slices n <= k are unchanged by sweep k (R14).
static int enqueue_max_slice(mfode_ctx* h, int k, double tol, int* flag) {
  const int nxt = (k + 1) % 2, cur = k % 2;
  const double denom = std::max(1.0, h->normU0);
  Rank& L = last_rank(h);
  std::vector<const double*> parts;
  for (auto& R : h->ranks) {
    const int jf = std::max(1, k + 1 - R.s0);   // local slot j <-> global slice s0 + j
    const int count = (k < R.s1) ? std::max(0, R.nloc - jf + 1) : 0;
    int sp;
    TRY(span_open(h, R, R.coarse, &sp));
    CUDA_TRY(h, launch_frob_slices_max(slot(h, R.U[nxt], jf), slot(h, R.U[cur], jf), (long long)state_elems(h), count,
                                       (long long)state_elems(h), R.spart, R.metric + 3, R.coarse));
    TRY(span_close(h, R, R.coarse, PH_METRIC, &sp));
    if (h->nccl_mode) {
      int sc;
      TRY(span_open(h, R, R.coarse, &sc));
      NCCL_TRY(h, nccl().allreduce(R.metric + 3, R.metric + 3, 1, ncclFloat64, ncclMax, h->comm, R.coarse));
      TRY(span_close(h, R, R.coarse, PH_COMM, &sc));
      const double* one = R.metric + 3;
      CUDA_TRY(h, launch_max_ptrs(&one, 1, denom, R.metric + 0, tol, nullptr, R.coarse));
    } else {
      parts.push_back(R.metric + 3);
      if (&R != &L) {
        CUDA_TRY(h, cudaEventRecord(R.ev_aux, R.coarse));
        CUDA_TRY(h, cudaStreamWaitEvent(L.coarse, R.ev_aux, 0));
      }
    }
  }
  if (!h->nccl_mode) CUDA_TRY(h, launch_max_ptrs(parts.data(), (int)parts.size(), denom, L.metric + 0, tol, flag, L.coarse));
  return MFODE_OK;
}

static int solve_impl(mfode_ctx* h, int K_max, double tol, int stop, mfode_solve_info* info) {
  if (K_max < 0 || !(tol >= 0.0) || stop < 0 || stop > 3) return fail(h, MFODE_EINVAL, "bad K_max/tol/stop");
  if (stop == MFODE_STOP_MAX_SLICE && h->world > 64) return fail(h, MFODE_EINVAL, "MAX_SLICE needs world <= 64");
  if (stop == MFODE_STOP_RESIDUAL && (h->flow == MFODE_FLOW_EXP || h->flow == MFODE_FLOW_TRIG ||
                                      h->flow == MFODE_FLOW_AFFINE))
    return fail(h, MFODE_EINVAL, "the exp/trig/affine flows have no residual stop test");
  CUDA_TRY(h, cudaSetDevice(h->device));
  const long long L0 = g_launches.load();
  const int K_eff = std::min(K_max, h->N);
  mfode_solve_info loc;
  memset(&loc, 0, sizeof(loc));
  loc.bad_slice = -1;
  loc.last_delta = NAN;
  loc.world = h->world;
  for (int i = 0; i < 64; ++i) loc.deltas[i] = NAN;
  h->seq_mode = false;
  h->has_result = false;
  // start: every stream waits for the previous work of this handle (serialised solves)
  for (auto& R : h->ranks) {
    CUDA_TRY(h, cudaStreamSynchronize(R.fine));
    CUDA_TRY(h, cudaStreamSynchronize(R.coarse));
  }
  Rank& L = last_rank(h);
  CUDA_TRY(h, cudaMemsetAsync(h->stop_flag, 0, sizeof(int), h->ranks[0].coarse));
  CUDA_TRY(h, cudaStreamSynchronize(h->ranks[0].coarse));
  for (auto& R : h->ranks) {
    R.fine_started = false;
    R.tused = 0;
    R.pev_used = 0;
    R.spans.clear();
    CUDA_TRY(h, cudaEventRecord(R.ev_t0, R.coarse));
    CUDA_TRY(h, cudaStreamWaitEvent(R.fine, R.ev_t0, 0));
  }
  // ---- Step 0 ----
  for (auto& R : h->ranks) TRY(enqueue_step0(h, R));
  // Fault injection (failure-detection test hook): overwrite U^0_j with NaNs once Step 0 has
  // produced it (and G(U^0_j)), in the rank that propagates slice j; its fine work then waits for it.
  if (h->inject_nan >= 1 && h->inject_nan < h->N)
    for (auto& R : h->ranks)
      if (h->inject_nan >= R.s0 && h->inject_nan < R.s1) {
        CUDA_TRY(h, cudaMemsetAsync(slot(h, R.U[0], h->inject_nan - R.s0), 0xFF, state_elems(h) * sizeof(double),
                                    R.coarse));
        for (int j = 0; j < R.nloc; ++j) CUDA_TRY(h, cudaEventRecord(R.evC[j], R.coarse));
      }
  double res0 = NAN;
  if (stop == MFODE_STOP_RESIDUAL && owns_last(h)) {
    int sp;
    TRY(span_open(h, L, L.coarse, &sp));
    TRY(enqueue_residual(h, L, L.U[0], L.nloc + 1, L.nloc, 1, 0.0, nullptr));
    TRY(span_close(h, L, L.coarse, PH_METRIC, &sp));
  }
  if (stop == MFODE_STOP_RESIDUAL) {
    TRY(fetch_metric(h, 1, 1));
    CUDA_TRY(h, cudaEventSynchronize(L.ev_metric));
    res0 = L.host_metric[1];
  }
  loc.residual0 = res0;
  int k_done = 0;
  bool converged = (stop == MFODE_STOP_FIXED_K);
  int status = MFODE_OK;
  // Speculation (sweep k+1's fine work enqueued before the host reads sweep k's metric) pays when the
  // fine sweep is chunked, so that chunk c can start as soon as the correction produced its inputs.
  // The fused fine kernel (K10) is one persistent launch holding every SM: it cannot overlap the
  // correction, and the metric kernel that would cancel it could not get an SM until it ends (a
  // converged solve would pay one whole wasted sweep), so it runs strictly phased.
  const bool spec = h->overlap && stop != MFODE_STOP_FIXED_K && !use_fused(h);
  if (K_eff > 0)
    for (auto& R : h->ranks) TRY(enqueue_fine(h, R, 0, false));
  for (int k = 0; k < K_eff; ++k) {
    for (auto& R : h->ranks) TRY(enqueue_correction(h, R, k));
    // stop metric on the last rank: delta of U_N (always), residual (STOP_RESIDUAL)
    const int nxt = (k + 1) % 2, cur = k % 2;
    int* flag = nullptr;
    {
      NvtxRange nv("mfode:metric");
      if (stop == MFODE_STOP_MAX_SLICE) {
        TRY(enqueue_max_slice(h, k, tol, (spec && !h->nccl_mode) ? h->stop_flag : nullptr));
      } else if (owns_last(h)) {
        int sp;
        TRY(span_open(h, L, L.coarse, &sp));
        flag = (stop == MFODE_STOP_DELTA && spec && !h->nccl_mode) ? h->stop_flag : nullptr;
        CUDA_TRY(h, launch_frob(slot(h, L.U[nxt], L.nloc), slot(h, L.U[cur], L.nloc), h->ms * h->n, h->ld,
                                L.partials, L.metric + 0, 0, tol, flag, L.coarse));
        if (stop == MFODE_STOP_RESIDUAL) {
          int* rflag = (spec && !h->nccl_mode) ? h->stop_flag : nullptr;
          TRY(enqueue_residual(h, L, L.U[nxt], L.nloc + 1, L.nloc, 1, tol, rflag));
        }
        TRY(span_close(h, L, L.coarse, PH_METRIC, &sp));
      }
      TRY(fetch_metric(h, 0, 2));
    }
    if (spec && h->nccl_mode) {
      // every rank sets its own flag from the broadcast metric
      for (auto& R : h->ranks)
        CUDA_TRY(h, launch_copy_flag(R.metric + (stop == MFODE_STOP_RESIDUAL ? 1 : 0), tol, h->stop_flag, R.coarse));
    }
    const bool more = (k + 1 < K_eff);
    if (more && (spec || stop == MFODE_STOP_FIXED_K))
      for (auto& R : h->ranks) TRY(enqueue_fine(h, R, k + 1, spec));
    CUDA_TRY(h, cudaEventSynchronize(L.ev_metric));
    const double delta = L.host_metric[0];
    const double resid = L.host_metric[1];
    k_done = k + 1;
    h->last_k = k_done;
    loc.last_delta = delta;
    if (k < 64) loc.deltas[k] = delta;
    if (!std::isfinite(delta) || (stop == MFODE_STOP_RESIDUAL && !std::isfinite(resid))) {
      status = MFODE_ENONFINITE;
      break;
    }
    if ((stop == MFODE_STOP_DELTA || stop == MFODE_STOP_MAX_SLICE) && delta <= tol) {
      converged = true;
      break;
    }
    if (stop == MFODE_STOP_RESIDUAL && resid <= tol) {
      converged = true;
      break;
    }
    if (k_done == h->N) {  // R15: U^N = sequential fine, exact
      converged = true;
      break;
    }
    if (more && !(spec || stop == MFODE_STOP_FIXED_K))
      for (auto& R : h->ranks) TRY(enqueue_fine(h, R, k + 1, false));
  }
  if (K_eff == 0) h->last_k = 0;
  if (k_done == h->N) converged = true;
  // join: the coarse stream waits for (possibly cancelled) speculative fine work
  for (auto& R : h->ranks) {
    CUDA_TRY(h, cudaEventRecord(R.ev_fine_end, R.fine));
    CUDA_TRY(h, cudaStreamWaitEvent(R.coarse, R.ev_fine_end, 0));
    CUDA_TRY(h, cudaEventRecord(R.ev_t1, R.coarse));
  }
  double ms_max = 0.0;
  for (auto& R : h->ranks) {
    CUDA_TRY(h, cudaEventSynchronize(R.ev_t1));
    float ms = 0.f;
    CUDA_TRY(h, cudaEventElapsedTime(&ms, R.ev_t0, R.ev_t1));
    ms_max = std::max(ms_max, (double)ms);
  }
  if (h->nccl_mode) {
    // max over ranks of the device time
    L.host_metric[5] = ms_max;
    CUDA_TRY(h, cudaMemcpyAsync(L.metric + 5, L.host_metric + 5, sizeof(double), cudaMemcpyHostToDevice, L.coarse));
    NCCL_TRY(h, nccl().allreduce(L.metric + 5, L.metric + 5, 1, ncclFloat64, ncclMax, h->comm, L.coarse));
    CUDA_TRY(h, cudaMemcpyAsync(L.host_metric + 5, L.metric + 5, sizeof(double), cudaMemcpyDeviceToHost, L.coarse));
    CUDA_TRY(h, cudaStreamSynchronize(L.coarse));
    ms_max = L.host_metric[5];
  }
  if (L.fine_started) {
    float fms = 0.f;
    if (cudaEventElapsedTime(&fms, L.ev_f0, L.ev_f1) == cudaSuccess) loc.ms_fine = fms;
  }
  loc.ms_total = ms_max;
  loc.k_done = k_done;
  TRY(collect_phases(h, &loc));
  for (auto& R : h->ranks)
    for (int i = 0; i < R.tused; ++i) {
      const Rank::ChunkTiming& ct = R.tpool[i];
      if (ct.iter >= k_done) continue;   // cancelled speculative sweep
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, ct.t0, ct.t1) == cudaSuccess) {
        loc.fine_kernel_ms += ms;
        loc.fine_kernel_launches += ct.launches;
        loc.fine_kernel_flops += ct.flops;
      }
    }
  loc.converged = converged ? 1 : 0;
  // flops: slice-solves of the sweeps actually used (all ranks)
  double slice_solves = 0.0;
  for (int k = 0; k < k_done; ++k) slice_solves += (double)(h->N - k);
  double corr_slices = 0.0;
  for (int k = 0; k < k_done; ++k) corr_slices += (double)(h->N - k);
  loc.fine_flops = slice_solves * h->mF * rk4_flops(h);
  loc.coarse_flops = (h->N + corr_slices) * h->mG * euler_flops(h);
  loc.gpu_launches = (int)(g_launches.load() - L0);
  // result
  h->result_rank = h->world - 1;
  h->result_ptr = owns_last(h) ? slot(h, L.U[k_done % 2], L.nloc) : nullptr;
  h->has_result = true;
  if (status == MFODE_ENONFINITE) {
    loc.bad_slice = first_bad_slice(h);
  } else if (owns_last(h) || h->nccl_mode) {
    double r = NAN;
    if (stop == MFODE_STOP_RESIDUAL && k_done > 0) {
      r = L.host_metric[1];
    } else if (stop == MFODE_STOP_RESIDUAL && k_done == 0) {
      r = res0;
    }
    loc.residual = r;
  }
  if (info) *info = loc;
  if (status < 0) return fail(h, status, "non-finite state (first bad slice %d)", loc.bad_slice);
  if (!converged) {
    h->err = "not converged within K_max sweeps";
    return MFODE_NOT_CONVERGED;
  }
  return MFODE_OK;
}

// ---------------------------------------------------------------------------------------------
// Modified parareal for linear flows: Algorithm 3 (homogeneous) and Algorithm 4
// (inhomogeneous)
//   Step -1 (Algorithm 4 only): F(0) and G(0) -- one of each, the flow being autonomous on a
//   uniform grid (reading R18).  Step 0 as Algorithm 1.  Step k+1: S^k = span(S^{k-1} u {U^k_n})
//   with an F-orthonormal basis extended by the global QR of Algorithm 2 (Frobenius inner product,
//   P:250-304; Gram-Schmidt applied twice, reading R17; a block with r_ii <= 1e-12 max(1, ||Z_i||_F)
//   is eliminated, R16); the fine images F(Q_i) of the NEW basis blocks only are propagated in
//   parallel (batched); the update is sequential:
//     Alg. 3, eq. (eq_update):  U^{k+1}_{n+1} = sum_i a_i F(Q_i) + G(U - sum_i a_i Q_i)
//     Alg. 4, eq. (update2):    U^{k+1}_{n+1} = (sum_i a_i (F(Q_i) - F(0)) + F(0)) + G(U - P U) - G(0)
//   with a = Q^T <> U^{k+1}_n.  One image per basis block serves every n (reading R18).
// Device-side Gram-Schmidt: the N + 1 candidate blocks of a sweep are orthogonalised in turn, each
// against every earlier slot with a batched multi-dot and one linear combination per pass
// (classical Gram-Schmidt applied twice, CGS2 -- the same projection as Algorithm 2's modified
// Gram-Schmidt in exact arithmetic; DESIGN reading R17), and the keep decision stays on the
// device: an eliminated block is zeroed in place (later projections onto it add exact zeros).
// The host reads the keep flags once per sweep and compacts the basis.
// ---------------------------------------------------------------------------------------------
static double host_frob(mfode_ctx* h, Rank& R, const double* X, const double* Y, cudaStream_t st, int* err) {
  if (launch_frob(X, Y, h->ms * h->n, h->ld, R.partials, R.metric + 6, 1, 0.0, nullptr, st) != cudaSuccess ||
      cudaMemcpyAsync(R.host_metric + 6, R.metric + 6, 2 * sizeof(double), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    *err = fail(h, MFODE_ECUDA, "frobenius failed");
    return NAN;
  }
  return Y ? R.host_metric[6] : R.host_metric[7];
}

static void free_modified(mfode_ctx* h) {
  const size_t se = state_elems(h);
  double* bufs[] = {h->Qb, h->FQ, h->mtmp};
  for (double* b : bufs)
    if (b) {
      forget_maps(b, b + se * (size_t)(h->bcap + 3));
      cudaFree(b);
    }
  double* small[] = {h->F0, h->G0, h->Z0};
  for (double* b : small)
    if (b) {
      forget_maps(b, b + se);
      cudaFree(b);
    }
  if (h->coef) cudaFree(h->coef);
  if (h->mpart) cudaFree(h->mpart);
  if (h->gstat) cudaFree(h->gstat);
  if (h->keep_dev) cudaFree(h->keep_dev);
  if (h->keep_host) cudaFreeHost(h->keep_host);
  h->Qb = h->FQ = h->mtmp = h->coef = h->mpart = h->gstat = h->F0 = h->G0 = h->Z0 = nullptr;
  h->keep_dev = h->keep_host = nullptr;
  h->bcap = h->kcap = 0;
}

static int modified_impl(mfode_ctx* h, int K_max, double tol, int stop, int max_basis, mfode_solve_info* info) {
  if (K_max < 0 || !(tol >= 0.0) || (stop != MFODE_STOP_FIXED_K && stop != MFODE_STOP_DELTA))
    return fail(h, MFODE_EINVAL, "bad K_max/tol/stop (modified parareal supports FIXED_K and DELTA)");
  if (h->flow != MFODE_FLOW_EXP && h->flow != MFODE_FLOW_TRIG && h->flow != MFODE_FLOW_AFFINE)
    return fail(h, MFODE_EINVAL, "modified parareal needs a linear flow (exp, trig: Algorithm 3; affine: Algorithm 4)");
  if (h->world != 1) return fail(h, MFODE_EINVAL, "modified parareal runs on one rank");
  CUDA_TRY(h, cudaSetDevice(h->device));
  const long long L0 = g_launches.load();
  Rank& R = h->ranks[0];
  const int N = h->N;
  const bool inhom = (h->flow == MFODE_FLOW_AFFINE);
  const size_t se = state_elems(h);
  const long long tot = (long long)se;
  const int bcap = (max_basis > 0) ? max_basis : (N + 1) * (std::min(K_max, N) + 1);
  if (bcap > h->bcap || N + 1 > h->kcap) {   // (re)allocate the basis storage
    free_modified(h);
    CUDA_TRY(h, cudaMalloc(&h->Qb, se * bcap * sizeof(double)));
    CUDA_TRY(h, cudaMalloc(&h->FQ, se * bcap * sizeof(double)));
    CUDA_TRY(h, cudaMalloc(&h->mtmp, se * 3 * sizeof(double)));
    CUDA_TRY(h, cudaMalloc(&h->F0, se * sizeof(double)));
    CUDA_TRY(h, cudaMalloc(&h->G0, se * sizeof(double)));
    CUDA_TRY(h, cudaMalloc(&h->Z0, se * sizeof(double)));
    CUDA_TRY(h, cudaMalloc(&h->coef, (bcap + 8) * sizeof(double)));
    CUDA_TRY(h, cudaMalloc(&h->mpart, (size_t)std::min(bcap, 64) * 296 * sizeof(double)));
    CUDA_TRY(h, cudaMalloc(&h->gstat, (size_t)4 * (N + 1) * sizeof(double)));
    CUDA_TRY(h, cudaMalloc(&h->keep_dev, (size_t)(N + 1) * sizeof(int)));
    CUDA_TRY(h, cudaMallocHost(&h->keep_host, (size_t)(N + 1) * sizeof(int)));
    CUDA_TRY(h, cudaMemset(h->Qb, 0, se * bcap * sizeof(double)));
    CUDA_TRY(h, cudaMemset(h->FQ, 0, se * bcap * sizeof(double)));
    CUDA_TRY(h, cudaMemset(h->mtmp, 0, se * 3 * sizeof(double)));
    CUDA_TRY(h, cudaMemset(h->F0, 0, se * sizeof(double)));
    CUDA_TRY(h, cudaMemset(h->G0, 0, se * sizeof(double)));
    CUDA_TRY(h, cudaMemset(h->Z0, 0, se * sizeof(double)));
    h->bcap = bcap;
    h->kcap = N + 1;
  }
  cudaStream_t st = R.coarse;
  CUDA_TRY(h, cudaStreamSynchronize(R.fine));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  R.pev_used = 0;
  R.spans.clear();
  mfode_solve_info loc;
  memset(&loc, 0, sizeof(loc));
  loc.bad_slice = -1;
  loc.last_delta = NAN;
  loc.residual = loc.residual0 = NAN;
  loc.world = 1;
  for (int i = 0; i < 64; ++i) loc.deltas[i] = NAN;
  h->seq_mode = false;
  h->has_result = false;
  CUDA_TRY(h, cudaEventRecord(R.ev_t0, st));
  CUDA_TRY(h, cudaStreamWaitEvent(R.fine, R.ev_t0, 0));
  double fine_solves = 0.0;
  if (inhom) {
    // Step -1: F(0) on the fine stream, G(0) on the coarse stream
    NvtxRange nv("mfode:step-1");
    TRY(fine_prop(h, R, h->Z0, 1, h->F0, 1, 0, 1, nullptr));
    TRY(coarse_G(h, R, h->Z0, 1, 0, EPI_EULER, h->G0, nullptr, nullptr, nullptr));
    CUDA_TRY(h, cudaEventRecord(R.ev_fine_end, R.fine));
    CUDA_TRY(h, cudaStreamWaitEvent(st, R.ev_fine_end, 0));
    fine_solves += 1.0;
  }
  TRY(enqueue_step0(h, R));   // U^0 in U[0]; slot 0 = X0 in both buffers
  int nb = 0, err = MFODE_OK, k_done = 0, status = MFODE_OK;
  bool converged = (stop == MFODE_STOP_FIXED_K);
  double* Wv = h->mtmp + se;
  double* Gv = h->mtmp + 2 * se;
  const int K_eff = std::min(K_max, N);
  for (int k = 0; k < K_eff; ++k) {
    const int cur = k % 2, nxt = (k + 1) % 2;
    // (a) enhance the subspace with U^k_0..U^k_N (Algorithm 2, device-side): candidate i goes to the
    //     tentative slot nb + i; an eliminated candidate is zeroed there.
    const int nb_old = nb;
    const int ncand = std::min(N + 1, h->bcap - nb);
    {
      NvtxRange nv("mfode:global_qr");
      for (int i = 0; i < ncand; ++i) {
        const double* Z = slot(h, R.U[cur], i);
        double* q = slot(h, h->Qb, nb + i);
        double* gs = h->gstat + 4 * i;
        CUDA_TRY(h, cudaMemcpyAsync(q, Z, se * sizeof(double), cudaMemcpyDeviceToDevice, st));
        CUDA_TRY(h, launch_frob(Z, nullptr, h->ms * h->n, h->ld, R.partials, gs, 1, 0.0, nullptr, st));   // ||Z_i||
        const int cnt = nb + i;
        if (cnt > 0)
          for (int pass = 0; pass < 2; ++pass) {   // reading R17: the projection applied twice
            CUDA_TRY(h, launch_multidot(h->Qb, tot, cnt, q, tot, h->mpart, h->coef, st));    // r_j = <q, Q_j>_F
            CUDA_TRY(h, launch_lincomb(q, h->Qb, tot, h->coef, cnt, tot, q, -1.0, st));       // q -= sum r_j Q_j
          }
        CUDA_TRY(h, launch_frob(q, nullptr, h->ms * h->n, h->ld, R.partials, gs + 2, 1, 0.0, nullptr, st));  // r_ii
        CUDA_TRY(h, launch_gs_keep(q, tot, gs, 1e-12, h->keep_dev + i, st));
      }
      CUDA_TRY(h, cudaMemcpyAsync(h->keep_host, h->keep_dev, ncand * sizeof(int), cudaMemcpyDeviceToHost, st));
      CUDA_TRY(h, cudaStreamSynchronize(st));
      for (int i = 0; i < ncand; ++i)
        if (h->keep_host[i] == -1) {   // a non-finite iterate
          status = MFODE_ENONFINITE;
          loc.bad_slice = i;
          break;
        }
      if (status < 0) break;
      // compact the kept blocks (ascending; destination never after its source)
      for (int i = 0; i < ncand; ++i) {
        if (!h->keep_host[i]) continue;
        if (nb != nb_old + i)
          CUDA_TRY(h, cudaMemcpyAsync(slot(h, h->Qb, nb), slot(h, h->Qb, nb_old + i), se * sizeof(double),
                                      cudaMemcpyDeviceToDevice, st));
        ++nb;
      }
    }
    // (b) fine images of the new blocks, in parallel (batched over the blocks, chunks of `cap`)
    if (nb > nb_old) {
      NvtxRange nv("mfode:fine_images");
      CUDA_TRY(h, cudaEventRecord(R.ev_metric, st));
      CUDA_TRY(h, cudaStreamWaitEvent(R.fine, R.ev_metric, 0));
      int fsp = -1;
      TRY(span_open(h, R, R.fine, &fsp));
      for (int ja = nb_old; ja < nb; ja += h->cap) {
        const int jb = std::min(nb, ja + h->cap);
        TRY(fine_prop(h, R, h->Qb, h->bcap, h->FQ, h->bcap, ja, jb, nullptr));
      }
      // Algorithm 4: keep D_i = F(Q_i) - F(0) (Remark P:424-428)
      if (inhom) CUDA_TRY(h, launch_sub_bcast(slot(h, h->FQ, nb_old), tot, nb - nb_old, h->F0, tot, R.fine));
      fine_solves += nb - nb_old;
      TRY(span_close(h, R, R.fine, PH_FINE, &fsp));
      CUDA_TRY(h, cudaEventRecord(R.ev_fine_end, R.fine));
      CUDA_TRY(h, cudaStreamWaitEvent(st, R.ev_fine_end, 0));
    }
    // (c) sequential update, V_0 = X0
    {
      NvtxRange nv("mfode:update");
      SpanCtx sc{&R, st, PH_CORRECT, -1};
      TRY(span_open(h, R, st, &sc.open));
      for (int n = 0; n < N; ++n) {
        const double* V = slot(h, R.U[nxt], n);
        CUDA_TRY(h, launch_multidot(h->Qb, tot, nb, V, tot, h->mpart, h->coef, st));               // a = Q^T <> V
        CUDA_TRY(h, launch_lincomb(Wv, h->Qb, tot, h->coef, nb, tot, V, -1.0, st));                 // (I - P) V
        TRY(coarse_G(h, R, Wv, 1, 0, EPI_EULER, Gv, nullptr, nullptr, nullptr));                   // G((I - P) V)
        if (inhom)
          CUDA_TRY(h, launch_lincomb_affine(slot(h, R.U[nxt], n + 1), h->FQ, tot, h->coef, nb, tot, h->F0, Gv, h->G0,
                                            st));                                                   // eq. (update2)
        else
          CUDA_TRY(h, launch_lincomb(slot(h, R.U[nxt], n + 1), h->FQ, tot, h->coef, nb, tot, Gv, 1.0, st));  // eq_update
      }
      TRY(span_close(h, R, st, PH_CORRECT, &sc.open));
    }
    const double num = host_frob(h, R, slot(h, R.U[nxt], N), slot(h, R.U[cur], N), st, &err);
    TRY(err);
    const double den = R.host_metric[7];
    const double delta = num / den;
    k_done = k + 1;
    h->last_k = k_done;
    loc.last_delta = delta;
    if (k < 64) loc.deltas[k] = delta;
    if (!std::isfinite(delta)) {
      status = MFODE_ENONFINITE;
      for (int n = 0; n <= N; ++n) {   // first non-finite slice of the new iterate
        const double v = host_frob(h, R, slot(h, R.U[nxt], n), nullptr, st, &err);
        TRY(err);
        if (!std::isfinite(v)) {
          loc.bad_slice = n;
          break;
        }
      }
      break;
    }
    if (stop == MFODE_STOP_DELTA && delta <= tol) {
      converged = true;
      break;
    }
    if (k_done == N) {
      converged = true;
      break;
    }
  }
  if (K_eff == 0) h->last_k = 0;
  CUDA_TRY(h, cudaEventRecord(R.ev_t1, st));
  CUDA_TRY(h, cudaEventSynchronize(R.ev_t1));
  float ms = 0.f;
  CUDA_TRY(h, cudaEventElapsedTime(&ms, R.ev_t0, R.ev_t1));
  loc.ms_total = ms;
  loc.k_done = k_done;
  loc.converged = converged ? 1 : 0;
  loc.basis_size = nb;
  loc.fine_flops = fine_solves * h->mF * rk4_flops(h);
  loc.coarse_flops = (double)N * (k_done + 1) * h->mG * euler_flops(h);
  loc.gpu_launches = (int)(g_launches.load() - L0);
  TRY(collect_phases(h, &loc));
  h->result_rank = 0;
  h->result_ptr = slot(h, R.U[k_done % 2], R.nloc);
  h->has_result = true;
  if (info) *info = loc;
  if (status < 0) return fail(h, status, "non-finite state in the modified parareal (first bad slice %d)", loc.bad_slice);
  if (!converged) {
    h->err = "not converged within K_max sweeps";
    return MFODE_NOT_CONVERGED;
  }
  return MFODE_OK;
}

static int sequential_impl(mfode_ctx* h, mfode_solve_info* info) {
  CUDA_TRY(h, cudaSetDevice(h->device));
  NvtxRange nv("mfode:sequential_fine");
  const long long L0 = g_launches.load();
  for (auto& R : h->ranks) {
    CUDA_TRY(h, cudaStreamSynchronize(R.fine));
    CUDA_TRY(h, cudaStreamSynchronize(R.coarse));
    R.pev_used = 0;
    R.spans.clear();
    CUDA_TRY(h, cudaEventRecord(R.ev_t0, R.coarse));
  }
  const int saved_cap = h->cap;
  for (auto& R : h->ranks) {
    // S_{s0} arrives from the previous rank; each slice: Fk_j = F(S_j) on the coarse stream, S_{j+1} = Fk_j
    TRY(recv_boundary(h, R, 0));
    std::swap(R.fine, R.coarse);  // run the fine chunks on the coarse stream (strictly sequential)
    h->cap = 1;
    int s = MFODE_OK;
    for (int j = 0; j < R.nloc && s == MFODE_OK; ++j) {
      s = fine_chunk(h, R, 0, j, j + 1, nullptr);
      if (s == MFODE_OK) {
        cudaError_t e = cudaMemcpyAsync(slot(h, R.U[0], j + 1), slot(h, R.Fk, j), state_elems(h) * sizeof(double),
                                        cudaMemcpyDeviceToDevice, R.fine);
        if (e != cudaSuccess) s = fail(h, MFODE_ECUDA, "copy: %s", cudaGetErrorString(e));
      }
    }
    std::swap(R.fine, R.coarse);
    h->cap = saved_cap;
    TRY(s);
    if (R.nloc > 0) CUDA_TRY(h, cudaEventRecord(R.evC[R.nloc - 1], R.coarse));
    TRY(send_boundary(h, R, 0));
    CUDA_TRY(h, cudaEventRecord(R.ev_t1, R.coarse));
  }
  double ms_max = 0.0;
  for (auto& R : h->ranks) {
    CUDA_TRY(h, cudaEventSynchronize(R.ev_t1));
    float ms = 0.f;
    CUDA_TRY(h, cudaEventElapsedTime(&ms, R.ev_t0, R.ev_t1));
    ms_max = std::max(ms_max, (double)ms);
  }
  h->seq_mode = true;
  h->last_k = 0;
  Rank& L = last_rank(h);
  h->result_rank = h->world - 1;
  h->result_ptr = owns_last(h) ? slot(h, L.U[0], L.nloc) : nullptr;
  h->has_result = true;
  if (info) {
    memset(info, 0, sizeof(*info));
    info->k_done = 0;
    info->bad_slice = -1;
    info->converged = 1;
    info->world = h->world;
    info->last_delta = NAN;
    info->residual = NAN;
    info->residual0 = NAN;
    info->ms_total = ms_max;
    info->fine_flops = (double)h->N * h->mF * rk4_flops(h);
    info->gpu_launches = (int)(g_launches.load() - L0);
    for (int i = 0; i < 64; ++i) info->deltas[i] = NAN;
  }
  return MFODE_OK;
}

}  // namespace mfode

using namespace mfode;

// =============================================================================================
// C ABI
// =============================================================================================
extern "C" {

int mfode_create(mfode_ctx** out, const double* A, int64_t n, int flow, double T, int N_slices, int coarse_steps,
                 int fine_steps, const mfode_dist* dist) {
  return create_impl(out, A, true, n, flow, T, N_slices, coarse_steps, fine_steps, dist, (cudaStream_t)-1);
}

int mfode_create_device(mfode_ctx** out, const double* dA, int64_t n, int flow, double T, int N_slices,
                        int coarse_steps, int fine_steps, const mfode_dist* dist, void* cuda_stream) {
  return create_impl(out, dA, false, n, flow, T, N_slices, coarse_steps, fine_steps, dist, (cudaStream_t)cuda_stream);
}

int mfode_set_matrix(mfode_ctx* h, const double* A) {
  if (!h || !A) return set_global_err(MFODE_EINVAL, "NULL argument");
  if (cudaSetDevice(h->device) != cudaSuccess) return fail(h, MFODE_ECUDA, "cudaSetDevice");
  for (auto& R : h->ranks) {
    cudaStreamSynchronize(R.fine);
    cudaStreamSynchronize(R.coarse);
  }
  return load_matrix(h, A, true, (size_t)h->n, h->ranks[0].coarse);
}

int mfode_set_affine(mfode_ctx* h, const double* G, const double* U0) {
  if (!h) return set_global_err(MFODE_EINVAL, "NULL handle");
  if (h->flow != MFODE_FLOW_AFFINE) return fail(h, MFODE_EINVAL, "mfode_set_affine needs MFODE_FLOW_AFFINE");
  CUDA_TRY(h, cudaSetDevice(h->device));
  for (auto& R : h->ranks) {
    CUDA_TRY(h, cudaStreamSynchronize(R.fine));
    CUDA_TRY(h, cudaStreamSynchronize(R.coarse));
  }
  cudaStream_t st = h->ranks[0].coarse;
  const size_t rowb = (size_t)h->n * sizeof(double), ldb = (size_t)h->ld * sizeof(double);
  oz_forget(h->Gsrc);
  if (G)
    CUDA_TRY(h, cudaMemcpy2DAsync(h->Gsrc, ldb, G, rowb, rowb, h->n, cudaMemcpyHostToDevice, st));
  else
    CUDA_TRY(h, cudaMemsetAsync(h->Gsrc, 0, mat_elems(h) * sizeof(double), st));
  if (U0) {
    CUDA_TRY(h, cudaMemcpy2DAsync(h->X0dev, ldb, U0, rowb, rowb, h->n, cudaMemcpyHostToDevice, st));
    double ss = 0.0;
    for (size_t i = 0; i < (size_t)h->n * h->n; ++i) ss += U0[i] * U0[i];
    h->normU0 = std::sqrt(ss);
  } else {
    CUDA_TRY(h, launch_identity(h->X0dev, h->n, h->ld, 1, 0, st));
    h->normU0 = std::sqrt((double)h->n);
  }
  // U_0 lives in slot 0 of both U buffers of rank 0
  for (auto& R : h->ranks)
    if (R.id == 0)
      for (int b = 0; b < 2; ++b)
        CUDA_TRY(h, cudaMemcpyAsync(R.U[b], h->X0dev, mat_elems(h) * sizeof(double), cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  h->has_result = false;
  return MFODE_OK;
}

int mfode_parareal_solve(mfode_ctx* h, int K_max, double tol, int stop, mfode_solve_info* info) {
  if (!h) return set_global_err(MFODE_EINVAL, "NULL handle");
  return solve_impl(h, K_max, tol, stop, info);
}

int mfode_modified_parareal_solve(mfode_ctx* h, int K_max, double tol, int stop, int max_basis,
                                  mfode_solve_info* info) {
  if (!h) return set_global_err(MFODE_EINVAL, "NULL handle");
  return modified_impl(h, K_max, tol, stop, max_basis, info);
}

int mfode_sequential_fine(mfode_ctx* h, mfode_solve_info* info) {
  if (!h) return set_global_err(MFODE_EINVAL, "NULL handle");
  return sequential_impl(h, info);
}

int mfode_residual(mfode_ctx* h, double* rel) {
  if (!h || !rel) return set_global_err(MFODE_EINVAL, "NULL argument");
  if (!h->has_result) return fail(h, MFODE_EINVAL, "no result yet (call a solve first)");
  if (h->flow == MFODE_FLOW_EXP || h->flow == MFODE_FLOW_TRIG || h->flow == MFODE_FLOW_AFFINE)
    return fail(h, MFODE_EINVAL, "the exp/trig/affine flows have no residual");
  CUDA_TRY(h, cudaSetDevice(h->device));
  Rank& L = last_rank(h);
  if (owns_last(h)) {
    TRY(enqueue_residual(h, L, h->result_ptr, 1, 0, 2, 0.0, nullptr));
  }
  TRY(fetch_metric(h, 2, 1));
  CUDA_TRY(h, cudaEventSynchronize(L.ev_metric));
  *rel = L.host_metric[2];
  return MFODE_OK;
}

static int get_result_impl(mfode_ctx* h, double* dst, bool host, cudaStream_t user) {
  if (!h || !dst) return set_global_err(MFODE_EINVAL, "NULL argument");
  if (!h->has_result) return fail(h, MFODE_EINVAL, "no result yet (call a solve first)");
  CUDA_TRY(h, cudaSetDevice(h->device));
  Rank& L = last_rank(h);
  const double* src = h->result_ptr;
  if (h->nccl_mode) {
    // broadcast the result from the last rank into this rank's Xa scratch
    double* buf = L.Xa;
    if (owns_last(h))
      CUDA_TRY(h, cudaMemcpyAsync(buf, src, state_elems(h) * sizeof(double), cudaMemcpyDeviceToDevice, L.coarse));
    NCCL_TRY(h, nccl().bcast(buf, buf, state_elems(h), ncclFloat64, h->world - 1, h->comm, L.coarse));
    src = buf;
  }
  // the state's ms matrices are consecutive with equal stride, so one 2-D copy of ms*n rows
  CUDA_TRY(h, cudaMemcpy2DAsync(dst, h->n * sizeof(double), src, h->ld * sizeof(double), h->n * sizeof(double),
                                (size_t)h->ms * h->n, host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                                L.coarse));
  if (host) {
    CUDA_TRY(h, cudaStreamSynchronize(L.coarse));
  } else {
    cudaEvent_t ev;
    CUDA_TRY(h, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    cudaEventRecord(ev, L.coarse);
    cudaStreamWaitEvent(user, ev, 0);
    cudaEventDestroy(ev);
  }
  return MFODE_OK;
}

int mfode_get_result(mfode_ctx* h, double* X) { return get_result_impl(h, X, true, nullptr); }

int mfode_get_result_device(mfode_ctx* h, double* dX, void* stream) {
  return get_result_impl(h, dX, false, (cudaStream_t)stream);
}

int mfode_get_slice(mfode_ctx* h, int n_index, double* U) {
  if (!h || !U) return set_global_err(MFODE_EINVAL, "NULL argument");
  if (n_index < 0 || n_index > h->N) return fail(h, MFODE_EINVAL, "slice %d out of range", n_index);
  if (!h->has_result) return fail(h, MFODE_EINVAL, "no solve yet");
  CUDA_TRY(h, cudaSetDevice(h->device));
  for (auto& R : h->ranks) {
    // U_n is stored by the rank with s0 <= n <= s1 (n == s1 also as the next rank's boundary)
    if (n_index < R.s0 || n_index > R.s1) continue;
    const int j = n_index - R.s0;
    const int par = h->seq_mode ? 0 : ((n_index <= h->last_k ? n_index : h->last_k) % 2);
    CUDA_TRY(h, cudaMemcpy2DAsync(U, h->n * sizeof(double), slot(h, R.U[par], j), h->ld * sizeof(double),
                                  h->n * sizeof(double), (size_t)h->ms * h->n, cudaMemcpyDeviceToHost, R.coarse));
    CUDA_TRY(h, cudaStreamSynchronize(R.coarse));
    return MFODE_OK;
  }
  return fail(h, MFODE_EINVAL, "slice %d not owned by this rank", n_index);
}

int mfode_set_option(mfode_ctx* h, const char* key, int64_t value) {
  if (!h || !key) return set_global_err(MFODE_EINVAL, "NULL argument");
  if (!strcmp(key, "overlap")) {
    h->overlap = value != 0;
    return MFODE_OK;
  }
  if (!strcmp(key, "fused")) {   // K10 one-launch fine propagator: -1 auto (64 < n <= 512), 0 off, 1 on
    if (value < -1 || value > 1) return fail(h, MFODE_EINVAL, "fused must be -1, 0 or 1");
    h->fused = (int)value;
    return MFODE_OK;
  }
  if (!strcmp(key, "inject_nan_slice")) {   // test hook: 1..N-1 poisons U^0_j after Step 0; <= 0 disables
    if (value >= h->N) return fail(h, MFODE_EINVAL, "inject_nan_slice must be < N");
    h->inject_nan = value >= 1 ? (int)value : -1;
    return MFODE_OK;
  }
  if (!strcmp(key, "phase_timing")) {   // per-phase CUDA-event spans (mfode_solve_info ms_coarse ...)
    h->phase_timing = value != 0;
    return MFODE_OK;
  }
  if (!strcmp(key, "symmetric")) {
    if (value && !h->a_symmetric) return fail(h, MFODE_EINVAL, "symmetric mode needs A == A^T exactly");
    if (value && h->flow == MFODE_FLOW_AFFINE)
      return fail(h, MFODE_EINVAL, "symmetric mode needs every iterate to be a polynomial in A (not the affine flow)");
    if (value && h->small) h->small = false;   // K6 kernels compute full products
    h->sym = value != 0;
    return MFODE_OK;
  }
  if (!strcmp(key, "emulation")) {
    // f3(ii): FP64 GEMMs emulated on the int8 tensor cores (ozaki.cu) with `value` moduli; 0 = DMMA
    if (value != 0 && (value < 8 || value > kOzMaxModuli))
      return fail(h, MFODE_EINVAL, "emulation needs 0 (off) or 8..%d moduli", kOzMaxModuli);
    OzConst c;
    if (value != 0 && (h->n > 32768 || !oz_make_const((int)value, h->n, &c)))
      return fail(h, MFODE_EINVAL, "n = %d too large for %lld moduli", h->n, (long long)value);
    if (value && h->small) h->small = false;   // K6 kernels do not go through the GEMM dispatch
    h->oz_nmod = (int)value;
    if (value) {
      CUDA_TRY(h, cudaSetDevice(h->device));
      for (auto& R : h->ranks) {
        CUDA_TRY(h, oz_reserve(R.fine, h->n, h->cap * h->ms, (int)value));
        CUDA_TRY(h, oz_reserve(R.coarse, h->n, h->ms, (int)value));
      }
    }
    return MFODE_OK;
  }
  if (!strcmp(key, "oz_pair")) {   // process-wide: CTA-pair (1, default) or single-CTA (0) int8 GEMM kernel
    g_oz_pair = value != 0;
    return MFODE_OK;
  }
  if (!strcmp(key, "pdl")) {   // process-wide: programmatic dependent launch of the GEMMs
    g_pdl = value != 0;
    return MFODE_OK;
  }
  if (!strcmp(key, "cta_share_us")) {   // process-wide: DMMA GEMM bounded persistence (us of tiles per CTA)
    if (value < 10 || value > 1000000) return fail(h, MFODE_EINVAL, "cta_share_us must be in [10, 1e6]");
    g_cta_share_s = value * 1e-6;
    return MFODE_OK;
  }
  if (!strcmp(key, "small")) {
    if (value && (h->n > kSmallMaxN || h->ms != 1 || h->flow == MFODE_FLOW_AFFINE))
      return fail(h, MFODE_EINVAL, "small kernels need n <= %d, a one-matrix state and no source", kSmallMaxN);
    h->small = value != 0;
    return MFODE_OK;
  }
  if (!strcmp(key, "small_cluster")) {
    if (value != -1 && value != 1 && value != 2 && value != 4 && !(value == 8 && h->n > 32))
      return fail(h, MFODE_EINVAL, "small_cluster must be -1 (auto), 1, 2, 4 (or 8 for 32 < n <= 64)");
    h->small_cs = (int)value;
    return MFODE_OK;
  }
  if (!strcmp(key, "tile")) {
    if (value < 0 || value > 3) return fail(h, MFODE_EINVAL, "tile must be 0..3");
    h->tile = (int)value;
    return MFODE_OK;
  }
  if (!strcmp(key, "fine_batch")) {
    // shrinking only (scratch is allocated at create for the automatic capacity)
    int nloc_max = 0;
    for (auto& R : h->ranks) nloc_max = std::max(nloc_max, R.nloc);
    if (value < 0) return fail(h, MFODE_EINVAL, "fine_batch must be >= 0");
    if (value == 0) return MFODE_OK;
    if (value > h->cap) return fail(h, MFODE_EINVAL, "fine_batch %lld exceeds allocated capacity %d", (long long)value, h->cap);
    h->cap = (int)value;
    return MFODE_OK;
  }
  return fail(h, MFODE_EINVAL, "unknown option '%s'", key);
}

const char* mfode_last_error(const mfode_ctx* h) { return h ? h->err.c_str() : g_err.c_str(); }

void mfode_destroy(mfode_ctx* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  cudaDeviceSynchronize();
  for (auto& R : h->ranks) free_rank(h, R);
  const size_t me = mat_elems(h);
  if (h->A) {
    oz_forget(h->A);
    forget_maps(h->A, h->A + me);
    cudaFree(h->A);
  }
  if (h->B) {
    oz_forget(h->B);
    forget_maps(h->B, h->B + me);
    cudaFree(h->B);
  }
  if (h->stop_flag) cudaFree(h->stop_flag);
  free_modified(h);
  double* abufs[] = {h->Gsrc, h->X0dev};
  for (double* b : abufs)
    if (b) {
      oz_forget(b);
      forget_maps(b, b + me);
      cudaFree(b);
    }
  if (h->comm && nccl().ok) nccl().commDestroy(h->comm);
  delete h;
}

// ---- kernel-level ----------------------------------------------------------------------------
int mfode_dgemm(const double* dA, const double* dB, const double* dC, double* dD, int64_t n, int64_t ld, double alpha,
                double beta, int tile, void* stream) {
  if (!dA || !dB || !dD || (beta != 0.0 && !dC)) return set_global_err(MFODE_EINVAL, "NULL argument");
  if (n < 1 || ld < n || (ld * 8) % 16 != 0 || tile < 0 || tile > 3)
    return set_global_err(MFODE_EINVAL, "bad n/ld/tile");
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.n = (int)n;
  p.ld = (int)ld;
  p.num_z = 1;
  p.alpha = alpha;
  p.beta = beta;
  p.C = MatRef{const_cast<double*>(dC), 0};
  p.Y_out = MatRef{dD, 0};
  Operand A{dA, 1, 0, 0}, B{dB, 1, 0, 0};
  cudaError_t e = launch_gemm(EPI_STORE, tile, A, B, p, (cudaStream_t)stream);
  if (e != cudaSuccess) return set_global_err(MFODE_ECUDA, "dgemm: %s", cudaGetErrorString(e));
  return MFODE_OK;
}

int mfode_dgemm_emulated(const double* dA, const double* dB, const double* dC, double* dD, int64_t n, int64_t ld,
                         double alpha, double beta, int n_moduli, void* stream) {
  if (!dA || !dB || !dD || (beta != 0.0 && !dC)) return set_global_err(MFODE_EINVAL, "NULL argument");
  if (n < 1 || ld < n || (ld * 8) % 16 != 0) return set_global_err(MFODE_EINVAL, "bad n/ld");
  OzConst c;
  if (n > 32768 || n_moduli < 2 || n_moduli > kOzMaxModuli || !oz_make_const(n_moduli, (int)n, &c))
    return set_global_err(MFODE_EINVAL, "n_moduli must be 2..%d and leave >= 8 bits per operand", kOzMaxModuli);
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.n = (int)n;
  p.ld = (int)ld;
  p.num_z = 1;
  p.alpha = alpha;
  p.beta = beta;
  p.C = MatRef{const_cast<double*>(dC), 0};
  p.Y_out = MatRef{dD, 0};
  p.oz_nmod = n_moduli;
  Operand A{dA, 1, 0, 0}, B{dB, 1, 0, 0};
  cudaError_t e = launch_gemm(EPI_STORE, TILE_AUTO, A, B, p, (cudaStream_t)stream);
  if (e != cudaSuccess) return set_global_err(MFODE_ECUDA, "dgemm_emulated: %s", cudaGetErrorString(e));
  return MFODE_OK;
}

int mfode_release_workspace(void* stream) {
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  oz_release((cudaStream_t)stream);
  if (e != cudaSuccess) return set_global_err(MFODE_ECUDA, "release_workspace: %s", cudaGetErrorString(e));
  return MFODE_OK;
}

int mfode_rk_stage(const double* dYop, const double* dBop, const double* dC, double alpha, double beta, double* dX,
                   double* dS, double* dYnext, int stage, double h, int64_t n, int64_t ld, int tile, void* stream) {
  if (!dYop || !dBop || !dX || !dS || (stage < 4 && !dYnext) || (beta != 0.0 && !dC))
    return set_global_err(MFODE_EINVAL, "NULL argument");
  if (stage < 1 || stage > 4 || n < 1 || ld < n || (ld * 8) % 16 != 0 || tile < 0 || tile > 3)
    return set_global_err(MFODE_EINVAL, "bad stage/n/ld/tile");
  GemmParams p;
  memset(&p, 0, sizeof(p));
  p.n = (int)n;
  p.ld = (int)ld;
  p.num_z = 1;
  p.alpha = alpha;
  p.beta = beta;
  p.C = MatRef{const_cast<double*>(dC), 0};
  p.X_in = MatRef{dX, 0};
  p.X_out = MatRef{dX, 0};
  p.S = MatRef{dS, 0};
  p.Y_out = MatRef{stage < 4 ? dYnext : nullptr, 0};
  p.stage = stage;
  p.h = h;
  Operand A{dYop, 1, 0, 0}, B{dBop, 1, 0, 0};
  cudaError_t e = launch_gemm(EPI_RK, tile, A, B, p, (cudaStream_t)stream);
  if (e != cudaSuccess) return set_global_err(MFODE_ECUDA, "rk_stage: %s", cudaGetErrorString(e));
  return MFODE_OK;
}

// Algorithm 5: m = min{m >= 0 : 2^-m ||A||_inf <= 1}; A0 = 2^-m A (exact in FP64);
// C0 = cos(A0) = second block of the trig flow's state at T = 1 (classical parareal here; the paper
// uses its modified variant); C_{i+1} = 2 C_i^2 - I, m times (one DMMA GEMM each: alpha = 2,
// beta = -1, C = I).  Collective in NCCL mode; every rank receives C.
int mfode_cosine(const double* A, int64_t n, int N_slices, int coarse_steps, int fine_steps, int K_max, double tol,
                 int stop, const mfode_dist* dist, double* C, int* m_out, mfode_solve_info* info) {
  if (!A || !C) return set_global_err(MFODE_EINVAL, "NULL argument");
  if (n < 1 || n > 65536) return set_global_err(MFODE_EINVAL, "bad n");
  double ninf = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t j = 0; j < n; ++j) s += fabs(A[i * n + j]);
    ninf = std::max(ninf, s);
  }
  if (!std::isfinite(ninf)) return set_global_err(MFODE_EINVAL, "A is not finite");
  int m = 0;
  while (ldexp(ninf, -m) > 1.0) ++m;
  std::vector<double> A0((size_t)n * n);
  for (size_t i = 0; i < A0.size(); ++i) A0[i] = ldexp(A[i], -m);
  mfode_ctx* h = nullptr;
  int s = mfode_create(&h, A0.data(), n, MFODE_FLOW_TRIG, 1.0, N_slices, coarse_steps, fine_steps, dist);
  if (s < 0) return s;
  std::unique_ptr<mfode_ctx, void (*)(mfode_ctx*)> guard(h, mfode_destroy);
  int st = mfode_parareal_solve(h, K_max, tol, stop, info);
  if (st < 0) return set_global_err(st, "%s", h->err.c_str());
  Rank& L = last_rank(h);
  const size_t me = mat_elems(h);
  double* cur = L.Xa;            // trig scratch holds 2 matrices: ping-pong Xa[0], Xa[1]
  double* nxt = L.Xa + me;
  double* I = L.Xb;              // identity
  if (owns_last(h)) {
    CUDA_TRY(h, cudaMemcpyAsync(cur, h->result_ptr + me, me * sizeof(double), cudaMemcpyDeviceToDevice, L.coarse));
    CUDA_TRY(h, launch_identity(I, h->n, h->ld, 1, 0, L.coarse));
    for (int i = 0; i < m; ++i) {
      GemmParams p = base_params(h, 1);
      p.alpha = 2.0;
      p.beta = -1.0;
      p.C = MatRef{I, 0};
      p.Y_out = MatRef{nxt, 0};
      Operand Cop{cur, 1, 0, 0};
      CUDA_TRY(h, launch_gemm(EPI_STORE, h->tile, Cop, Cop, p, L.coarse));
      std::swap(cur, nxt);
    }
  }
  if (h->nccl_mode) NCCL_TRY(h, nccl().bcast(cur, cur, me, ncclFloat64, h->world - 1, h->comm, L.coarse));
  CUDA_TRY(h, cudaMemcpy2DAsync(C, h->n * sizeof(double), cur, h->ld * sizeof(double), h->n * sizeof(double), h->n,
                                cudaMemcpyDeviceToHost, L.coarse));
  CUDA_TRY(h, cudaStreamSynchronize(L.coarse));
  if (m_out) *m_out = m;
  return st;
}

// Algorithm 8 (Example 5): dX/dt = I - A X with the accelerator u,
//   X^{k+1} = X^k + dt (I - A X^k + u^k),  u^{k+1} = (I - dt A) u^k,  u^0 = e ~ A^{-1} - X^0.
// The state (X, u) is two sub-matrices; one batched DMMA GEMM per step computes (A X, A u) and
// the EPI_ACCEL epilogue applies both updates (out of place, ping-pong).  Sequential in k.
int mfode_accel_inverse(const double* A, const double* X0, const double* E0, int64_t n, double dt, int max_steps,
                        double tol, int check_every, double* X, int* steps_done, double* residual) {
  if (!A || !X || max_steps < 0 || !(dt > 0.0) || !(tol >= 0.0) || check_every < 0)
    return set_global_err(MFODE_EINVAL, "bad argument");
  mfode_ctx* h = nullptr;
  // one "slice" context (inverse-flow residual machinery; N = 1) owns A, the streams and scratch
  int s = mfode_create(&h, A, n, MFODE_FLOW_INVERSE, 1.0, 1, 1, 1, nullptr);
  if (s < 0) return s;
  std::unique_ptr<mfode_ctx, void (*)(mfode_ctx*)> guard(h, mfode_destroy);
  Rank& R = h->ranks[0];
  const size_t me = mat_elems(h);
  cudaStream_t st = R.coarse;
  // state buffers: U[0] holds slots (X, u) -> use U[0] and U[1] (each >= 2 matrices: nloc+1 = 2)
  double* cur = R.U[0];
  double* nxt = R.U[1];
  CUDA_TRY(h, cudaMemsetAsync(cur, 0, 2 * me * sizeof(double), st));
  if (X0)
    CUDA_TRY(h, cudaMemcpy2DAsync(cur, h->ld * sizeof(double), X0, n * sizeof(double), n * sizeof(double), n,
                                  cudaMemcpyHostToDevice, st));
  if (E0)
    CUDA_TRY(h, cudaMemcpy2DAsync(cur + me, h->ld * sizeof(double), E0, n * sizeof(double), n * sizeof(double), n,
                                  cudaMemcpyHostToDevice, st));
  int k = 0;
  double r = NAN;
  while (k < max_steps) {
    GemmParams p = base_params(h, 2);
    p.h = dt;
    p.X_in = MatRef{cur, (long long)me};
    p.S = MatRef{cur + me, 0};          // even z reads u at the same position
    p.X_out = MatRef{nxt, (long long)me};
    Operand Aop{h->A, 1, 0, 0, 0, h->mat_gen};
    Operand Sop{cur, 2, 0, 1};
    CUDA_TRY(h, launch_gemm(EPI_ACCEL, h->tile, Aop, Sop, p, st));
    std::swap(cur, nxt);
    ++k;
    if (tol > 0.0 && check_every > 0 && (k % check_every == 0 || k == max_steps)) {
      h->result_ptr = cur;
      h->has_result = true;
      TRY(enqueue_residual(h, R, cur, 1, 0, 2, 0.0, nullptr));
      CUDA_TRY(h, cudaMemcpyAsync(R.host_metric + 2, R.metric + 2, sizeof(double), cudaMemcpyDeviceToHost, st));
      CUDA_TRY(h, cudaStreamSynchronize(st));
      r = R.host_metric[2];
      if (!std::isfinite(r)) return fail(h, MFODE_ENONFINITE, "non-finite iterate at step %d", k);
      if (r <= tol) break;
    }
  }
  TRY(enqueue_residual(h, R, cur, 1, 0, 2, 0.0, nullptr));
  CUDA_TRY(h, cudaMemcpyAsync(R.host_metric + 2, R.metric + 2, sizeof(double), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaMemcpy2DAsync(X, n * sizeof(double), cur, h->ld * sizeof(double), n * sizeof(double), n,
                                cudaMemcpyDeviceToHost, st));
  CUDA_TRY(h, cudaStreamSynchronize(st));
  r = R.host_metric[2];
  if (steps_done) *steps_done = k;
  if (residual) *residual = r;
  if (tol > 0.0 && !(r <= tol)) return MFODE_NOT_CONVERGED;
  return MFODE_OK;
}

int mfode_frobenius(const double* dX, const double* dY, int64_t n, int64_t ld, double* out, void* stream) {
  if (!dX || !out) return set_global_err(MFODE_EINVAL, "NULL argument");
  if (n < 1 || ld < n || ld % 2 != 0) return set_global_err(MFODE_EINVAL, "bad n/ld");
  cudaStream_t st = (cudaStream_t)stream;
  double *part = nullptr, *res = nullptr;
  if (cudaMallocAsync(&part, sizeof(double) * kFrobPartials, st) != cudaSuccess ||
      cudaMallocAsync(&res, sizeof(double) * 2, st) != cudaSuccess)
    return set_global_err(MFODE_ENOMEM, "frobenius scratch");
  // Note: padding columns (ld > n) are included; callers keep them zero or pass ld == n.
  cudaError_t e = launch_frob(dX, dY, (int)n, (int)ld, part, res, 1, 0.0, nullptr, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, res, 2 * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(part, st);
  cudaFreeAsync(res, st);
  if (e != cudaSuccess) return set_global_err(MFODE_ECUDA, "frobenius: %s", cudaGetErrorString(e));
  return MFODE_OK;
}

int mfode_partition(int N, int world, int rank, int* first, int* count) {
  int s = partition(N, world, rank, first, count);
  if (s != MFODE_OK) return set_global_err(s, "bad partition arguments");
  return MFODE_OK;
}

int64_t mfode_kernel_launches(void) { return (int64_t)g_launches.load(); }

const char* mfode_last_global_error(void) { return g_err.c_str(); }

const char* mfode_version(void) { return "mfode 0.1 (sm_100a, FP64 DMMA + TMA)"; }

}  // extern "C"
