// K6 / K6c probe (not part of the library): times the one-CTA fine kernel against the cluster
// variants on a cfg[0]-shaped batch (n = 32, 8 slices, 64 RK4 steps, inverse flow) and, built with
// -DK6C_PROF, prints per-phase cycle stamps of 16 stages of CTA 0 and 1.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DK6C_PROF -I paper_1505_07959_b200/csrc \
//        tools/k6c_probe.cu -o /tmp/k6c_probe -lcuda
#include <cstdio>
#include <vector>

#include "small.cuh"

using namespace mfode;

template <typename F>
static float time_it(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

template <int NP, int CS>
static void run_cluster(int flow, int n, const double* M, const double* U, double* F, int Z, int mF, double h) {
  using C = ClusterCfg<NP, CS>;
  const size_t smem = 5 * C::MAT * sizeof(double);
  cudaFuncSetAttribute(fine_cluster_kernel<NP, CS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(Z * CS);
  cfg.blockDim = dim3(C::THREADS);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const long long ms = (long long)n * n;
  cudaLaunchKernelEx(&cfg, fine_cluster_kernel<NP, CS>, flow, n, n, M, U, F, ms, mF, h, (const int*)nullptr);
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 32, Z = 8, mF = 64, flow = argc > 2 ? atoi(argv[2]) : 0;
  const double h = 1.0 / 8 / mF;
  std::vector<double> hM(n * n), hU((size_t)Z * n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) hM[i * n + j] = (i == j ? 0.3 : 0.0) + 0.01 * ((i * 7 + j * 3) % 11 - 5);
  for (int z = 0; z < Z; ++z)
    for (int i = 0; i < n; ++i) hU[(size_t)z * n * n + i * n + i] = 1.0;
  double *M, *U, *F;
  cudaMalloc(&M, n * n * 8);
  cudaMalloc(&U, Z * n * n * 8);
  cudaMalloc(&F, Z * n * n * 8);
  cudaMemcpy(M, hM.data(), n * n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(U, hU.data(), Z * n * n * 8, cudaMemcpyHostToDevice);
  const long long ms = (long long)n * n;
  if (n > 32) {   // NP = 64 variants: timing only
    cudaFuncSetAttribute(fine_smem_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 5 * 64 * 64 * 8);
    auto one = [&] { fine_smem_kernel<64><<<Z, kSmallThreads, 5 * 64 * 64 * 8>>>(flow, n, n, M, U, F, ms, mF, h, nullptr); };
    const float t1 = time_it(one, 20);
    const float t2 = time_it([&] { run_cluster<64, 2>(flow, n, M, U, F, Z, mF, h); }, 20);
    const float t4 = time_it([&] { run_cluster<64, 4>(flow, n, M, U, F, Z, mF, h); }, 20);
    const float t8 = time_it([&] { run_cluster<64, 8>(flow, n, M, U, F, Z, mF, h); }, 20);
    printf("{\"n\": %d, \"flow\": %d, \"us_per_step\": {\"cs1\": %.3f, \"cs2\": %.3f, \"cs4\": %.3f, \"cs8\": %.3f}}\n",
           n, flow, t1 * 1e3 / mF, t2 * 1e3 / mF, t4 * 1e3 / mF, t8 * 1e3 / mF);
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
  }
  cudaFuncSetAttribute(fine_smem_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 5 * 32 * 32 * 8);
  auto one = [&] { fine_smem_kernel<32><<<Z, kSmallThreads, 5 * 32 * 32 * 8>>>(flow, n, n, M, U, F, ms, mF, h, nullptr); };
  auto c2 = [&] { run_cluster<32, 2>(flow, n, M, U, F, Z, mF, h); };
  auto c4 = [&] { run_cluster<32, 4>(flow, n, M, U, F, Z, mF, h); };
  const float t1 = time_it(one, 50), t2 = time_it(c2, 50), t4 = time_it(c4, 50);
  printf("{\"n\": %d, \"flow\": %d, \"us_per_step\": {\"cs1\": %.3f, \"cs2\": %.3f, \"cs4\": %.3f}}\n", n, flow,
         t1 * 1e3 / mF, t2 * 1e3 / mF, t4 * 1e3 / mF);
#ifdef K6C_PROF
  for (int cs : {2, 4}) {
    if (cs == 2) c2(); else c4();
    cudaDeviceSynchronize();
    long long p[2][16][8];
    cudaMemcpyFromSymbol(p, g_k6c_prof, sizeof(p));
    for (int b = 0; b < 2; ++b)
      for (int t = 0; t < 16; t += 1) {
        printf("cs%d cta%d stage%3d:", cs, b, 200 + t);
        for (int i = 1; i < 7; ++i) printf(" %6lld", p[b][t][i] - p[b][t][0]);
        if (t + 1 < 16) printf("  next %6lld", p[b][t + 1][0] - p[b][t][0]);
        printf("\n");
      }
  }
#endif
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
