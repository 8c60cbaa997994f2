// Do DMMA (FP64 tensor, mma.sync m8n8k4) and DFMA (FP64 FMA) share one execution pipe on B200?
// The two measure the same chip peak alone (tools/fp64_peaks.cu: 37.05 / 36.7 TF/s); if they
// are separate pipes, a GEMM that feeds part of its tile to DFMA could exceed the DMMA roofline.
// Probes (register-resident loops, grid = 2 x SMs):
//   split  : warp w runs DFMA if (w % R) < D, else DMMA  (D of R warps on DFMA)
//   inter  : every warp issues ND DMMAs and NF DFMAs per iteration, interleaved
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// D of every R warps run DFMA (ILP 8), the rest DMMA (ILP 8); iters per warp fixed
__global__ void split_kernel(double* out, int iters, int D, int R, int fma_per_dmma) {
  const int w = threadIdx.x >> 5;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double s = 0.0;
  if ((w % R) < D) {
    double c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = i * 1e-3;
    const int it2 = iters * fma_per_dmma;   // same wall-work scale as the DMMA warps
    for (int it = 0; it < it2; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) c[i] = fma(c[i], b, a);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i];
  } else {
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) dmma(c[i][0], c[i][1], a, b);
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  }
  if (s == 12345.678) out[0] = s;
}

template <int ND, int NF>
__global__ void inter_kernel(double* out, int iters) {
  const double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999;
  double c[ND > 0 ? ND : 1][2];
  double f[NF > 0 ? NF : 1];
#pragma unroll
  for (int i = 0; i < (ND > 0 ? ND : 1); ++i) c[i][0] = c[i][1] = 0.0;
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) f[i] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < (ND > NF ? ND : NF); ++i) {
      if (i < ND) dmma(c[i][0], c[i][1], a, b);
      if (i < NF) f[i] = fma(f[i], b, a);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < (ND > 0 ? ND : 1); ++i) s += c[i][0] + c[i][1];
#pragma unroll
  for (int i = 0; i < (NF > 0 ? NF : 1); ++i) s += f[i];
  if (s == 12345.678) out[0] = s;
}

static cudaEvent_t e0, e1;
template <typename F>
static double time_ms(F launch, int reps = 5) {
  launch();
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  return best;
}

template <int ND, int NF>
static void run_inter(double* d, int grid, int block, int iters) {
  const double ms = time_ms([&] { inter_kernel<ND, NF><<<grid, block>>>(d, iters); });
  const double warps = double(grid) * (block / 32);
  const double fl_mma = warps * iters * ND * 512.0, fl_fma = warps * iters * NF * 64.0;
  printf("{\"probe\": \"inter\", \"nd\": %d, \"nf\": %d, \"block\": %d, \"ms\": %.3f, \"tflops_dmma\": %.3f, "
         "\"tflops_dfma\": %.3f, \"tflops_total\": %.3f}\n",
         ND, NF, block, ms, fl_mma / ms / 1e9, fl_fma / ms / 1e9, (fl_mma + fl_fma) / ms / 1e9);
}

int main() {
  double* d; CK(cudaMalloc(&d, 64));
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int grid = 2 * sms, block = 512, iters = 4000;
  // split: warp-level mix (D of R warps on DFMA); a DFMA warp runs fpd x more iterations of 8 FMAs
  // so its 64-flop instructions take comparable pipe time to 8 DMMAs of 512 flops
  for (int fpd : {4, 8}) {
    for (int D = 0; D <= 4; ++D) {
      const int R = 4;
      const double ms = time_ms([&] { split_kernel<<<grid, block>>>(d, iters, D, R, fpd); });
      const double warps = double(grid) * (block / 32);
      const double wf = warps * D / R, wm = warps - wf;
      const double fl_mma = wm * iters * 8 * 512.0, fl_fma = wf * iters * fpd * 8 * 64.0;
      printf("{\"probe\": \"split\", \"dfma_warps_of_4\": %d, \"fma_iter_scale\": %d, \"ms\": %.3f, "
             "\"tflops_dmma\": %.3f, \"tflops_dfma\": %.3f, \"tflops_total\": %.3f}\n",
             D, fpd, ms, fl_mma / ms / 1e9, fl_fma / ms / 1e9, (fl_mma + fl_fma) / ms / 1e9);
    }
  }
  run_inter<8, 0>(d, grid, block, iters);
  run_inter<0, 8>(d, grid, block, iters * 8);
  run_inter<8, 8>(d, grid, block, iters);
  run_inter<4, 8>(d, grid, block, iters);
  run_inter<8, 16>(d, grid, block, iters);
  run_inter<4, 16>(d, grid, block, iters);
  run_inter<2, 16>(d, grid, block, iters);
  CK(cudaFree(d));
  return 0;
}
