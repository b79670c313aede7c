// peak.cu -- FP64 roofline denominator: a DFMA-dense kernel timed with CUDA events.
// MEASURED_PEAKS.json holds HBM and bf16 peaks only; the pair passes of this
// path are FP64-pipe bound, so bench.py measures the FP64 peak live with this.
#include <cuda_runtime.h>

#include "../../include/sph.h"

namespace {
constexpr int kChains = 8;
constexpr int kIters = 4096;

__global__ void __launch_bounds__(256) k_dfma_peak(double* out, double seed) {
  double a[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) a[k] = seed + threadIdx.x * 1e-9 + k * 1e-7;
  const double b = 0.999999999, c = 1e-12;
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int k = 0; k < kChains; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += a[k];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}
}  // namespace

extern "C" sph_status sph_measure_fp64_peak(void* stream, double* tflops) {
  if (!tflops) return SPH_ERR_CONFIG;
  cudaStream_t st = (cudaStream_t)stream;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* out = nullptr;
  if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return SPH_ERR_CUDA;
  const int blocks = sms * 8, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k_dfma_peak<<<blocks, threads, 0, st>>>(out, 1.0);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0, st);
    k_dfma_peak<<<blocks, threads, 0, st>>>(out, 1.0 + r);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (cudaGetLastError() != cudaSuccess) return SPH_ERR_CUDA;
  double flops = 2.0 * kChains * (double)kIters * blocks * threads;
  *tflops = flops / (best * 1e-3) / 1e12;
  return SPH_OK;
}
