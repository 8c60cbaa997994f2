// Microbenchmark: peak tcgen05.mma issue rate per SM for kind::i8 (int8 -> int32) and kind::f16
// (bf16 -> fp32), M = 128 (cta_group::1), N = 256, operands resident in shared memory (no loads),
// one CTA per SM, accumulating into TMEM.  Reports dense TOPS/TFLOPS for the whole chip.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1505_07959_b200/csrc umma_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace mfode;

template <int KIND>   // 0: i8, 1: bf16
__global__ void __launch_bounds__(128, 1) peak_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem =
      reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 48 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  fence_proxy_async();
  if (threadIdx.x < 32) tmem_alloc(&slot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a0 = smem_u32(smem), b0 = a0 + 16384;
    uint32_t idesc;
    if (KIND == 0)
      idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    else   // bf16 x bf16 -> f32: c_format 1, a/b format 1 (BF16)
      idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t ad = umma_desc_k_sw128(a0 + 32 * k), bd = umma_desc_k_sw128(b0 + 32 * k);
        if (KIND == 0) {
          umma_i8(tmem, ad, bd, idesc, 1);
        } else {
          asm volatile(
              "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
              " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
              "l"(ad), "l"(bd), "r"(idesc), "r"(1u)
              : "memory");
        }
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) cycles[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc(tmem, 256);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* dcyc;
  cudaMalloc(&dcyc, 8);
  const int smem = 48 * 1024 + 1024;
  cudaFuncSetAttribute(peak_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(peak_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int kind = 0; kind < 2; ++kind) {
    const int iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (kind == 0)
        peak_kernel<0><<<sms, 128, smem>>>(iters, dcyc);
      else
        peak_kernel<1><<<sms, 128, smem>>>(iters, dcyc);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
    }
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
    // per MMA: M=128, N=256, K = 32 (i8) or 16 (bf16) -> MACs
    const double macs_per = 128.0 * 256.0 * (kind == 0 ? 32 : 16);
    const double total = 2.0 * macs_per * 4.0 * iters * sms;
    printf("%s: %.3f ms, %.1f T(FL)OPS dense, %.1f MAC/clk/SM (clock64 %.0f cyc/MMA) err=%s\n",
           kind == 0 ? "kind::i8  " : "kind::f16 ", ms, total / (ms * 1e-3) / 1e12,
           macs_per * 4.0 * iters / (double)cyc, (double)cyc / (4.0 * iters), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
