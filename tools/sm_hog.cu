// Test tool: occupy `nsm` SMs with one spinning CTA each (large shared-memory request, so no other CTA
// of a big kernel fits beside it) for `seconds` -- a stand-in for NCCL kernels parked on SMs while the
// fine sweep runs (tools/ab_sm_hog.py).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -shared
// -Xcompiler -fPIC tools/sm_hog.cu -o tools/libsmhog.so
#include <cuda_runtime.h>

__global__ void k_hog(long long cycles) {
  extern __shared__ char pad[];
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) __nanosleep(1000);
  if (threadIdx.x == 0) pad[0] = 0;
}

extern "C" int hog_launch(int nsm, double seconds, void* stream) {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_hog, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int clk_khz = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  const long long cycles = (long long)(seconds * clk_khz * 1e3);
  k_hog<<<nsm, 32, smem, (cudaStream_t)stream>>>(cycles);
  return (int)cudaGetLastError();
}
