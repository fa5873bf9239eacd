// FP32-pipe and MUFU throughput microbenchmarks: the denominators of the
// FP32-bound kernels' roofline fractions (K3 composite, K4a backward raster).
// MEASURED_PEAKS.json carries HBM and bf16 tensor numbers only, so the bench
// measures these on the box it runs on, at the clock the box runs at.
//
// FFMA: every thread runs 8 independent FMA chains (enough ILP to cover the
// 4-cycle FMA latency at full occupancy), 2 FLOP per FFMA. MUFU: ex2.approx
// on 8 independent chains (the exp2 of K3/K4a's alpha = o * 2^(-g/2 log2 e)).
// Grids are 148 SMs x 8 CTAs x 256 threads, launched back to back.
#include <cuda_runtime.h>

#include <cstdint>

#include "gsb_internal.cuh"

namespace gsb {

template <int ITERS>
__global__ void __launch_bounds__(256) peak_ffma_kernel(float* out, float a, float b) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = (float)(threadIdx.x + k) * 1e-3f;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1234.5678f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;  // keep the chains live
}

template <int ITERS>
__global__ void __launch_bounds__(256) peak_mufu_kernel(float* out, float a) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = (float)(threadIdx.x & 7) * -1e-3f - 0.01f * k;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[k]));
      x[k] = y * a;  // one FMUL per MUFU keeps the chain dependent; MUFU is the bound (16/clk/SM vs 128)
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1234.5678f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

}  // namespace gsb

extern "C" int gsb_measure_fp32_peaks(int32_t device, double* ffma_tflops, double* mufu_tops) {
  using namespace gsb;
  if (cudaSetDevice(device) != cudaSuccess) return GSB_ERR_NO_DEVICE;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int blocks = sms * 8, threads = 256;
  constexpr int kIters = 4096;
  float* out = nullptr;
  if (cudaMalloc(&out, sizeof(float) * blocks * threads) != cudaSuccess) return GSB_ERR_OUT_OF_MEMORY;
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double threads_total = (double)blocks * threads;
  auto timed = [&](auto launch, int reps) {
    launch();  // warm-up (clocks ramp)
    launch();
    cudaEventRecord(e0, st);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    return (double)ms / reps;
  };
  const double ms_f = timed([&] { peak_ffma_kernel<kIters><<<blocks, threads, 0, st>>>(out, 0.9999f, 1e-4f); }, 20);
  const double ms_m = timed([&] { peak_mufu_kernel<kIters / 4><<<blocks, threads, 0, st>>>(out, 0.999f); }, 20);
  const cudaError_t err = cudaGetLastError();
  if (ffma_tflops) *ffma_tflops = threads_total * kIters * 8 * 2 / (ms_f * 1e-3) / 1e12;
  if (mufu_tops) *mufu_tops = threads_total * (kIters / 4) * 8 / (ms_m * 1e-3) / 1e12;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamDestroy(st);
  cudaFree(out);
  return err == cudaSuccess ? GSB_OK : GSB_ERR_CUDA;
}
