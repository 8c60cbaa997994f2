// FP64 roofline probes for B200 (sm_100a): DMMA (mma.sync f64 -> SASS DMMA.8x8x4) and DFMA
// register-resident throughput, plus single-warp DMMA latency. MEASURED_PEAKS.json has no FP64
// entry, so the FP64 roofline denominator is measured here.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peaks fp64_peaks.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int ILP>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = seed * 0.5;
  double c[ILP][2];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;  // keep live
}

template <int ILP>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-9, b = 0.999999;
  double c[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) c[i] = i * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

template <typename K>
static double time_kernel(K kern, int grid, int block, double* d, int iters, int reps = 5) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  kern<<<grid, block>>>(d, iters, 1.0);  // warm
  CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    kern<<<grid, block>>>(d, iters, 1.0);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  double* d; CK(cudaMalloc(&d, 64));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  int clk; CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
  printf("{\"sms\": %d, \"clock_khz_attr\": %d}\n", sms, clk);
  const int iters = 20000;
  // DMMA throughput: grid = k*SMs, 256 threads (8 warps/CTA)
  for (int cpb : {1, 2, 4}) {
    for (int block : {128, 256, 512}) {
      int grid = sms * cpb;
      double ms = time_kernel(dmma_loop<8>, grid, block, d, iters);
      double flops = double(grid) * (block / 32) * iters * 8 * 512.0;
      printf("{\"probe\": \"dmma_m8n8k4\", \"ilp\": 8, \"grid\": %d, \"block\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n",
             grid, block, ms, flops / ms / 1e9);
    }
  }
  for (int block : {256, 512}) {
    int grid = sms * 2;
    double ms = time_kernel(dmma_loop<4>, grid, block, d, iters);
    double flops = double(grid) * (block / 32) * iters * 4 * 512.0;
    printf("{\"probe\": \"dmma_m8n8k4\", \"ilp\": 4, \"grid\": %d, \"block\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n",
           grid, block, ms, flops / ms / 1e9);
  }
  // DMMA latency: one warp, ILP 1
  {
    double ms = time_kernel(dmma_loop<1>, 1, 32, d, iters);
    printf("{\"probe\": \"dmma_latency\", \"ns_per_dmma\": %.3f}\n", ms * 1e6 / iters);
    double ms4 = time_kernel(dmma_loop<4>, 1, 32, d, iters);
    printf("{\"probe\": \"dmma_1warp_ilp4\", \"ns_per_dmma\": %.3f}\n", ms4 * 1e6 / (iters * 4.0));
    double ms8 = time_kernel(dmma_loop<8>, 1, 128, d, iters);
    printf("{\"probe\": \"dmma_1cta4w_ilp8\", \"ns_per_dmma_per_sm\": %.3f}\n", ms8 * 1e6 / (iters * 32.0));
  }
  // DFMA throughput
  for (int block : {256, 512, 1024}) {
    int grid = sms * 2;
    double ms = time_kernel(dfma_loop<8>, grid, block, d, iters);
    double flops = double(grid) * block * iters * 8 * 2.0;
    printf("{\"probe\": \"dfma\", \"ilp\": 8, \"grid\": %d, \"block\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n",
           grid, block, ms, flops / ms / 1e9);
  }
  CK(cudaFree(d));
  return 0;
}
