// Measured FP64 / FP32 FMA and MUFU throughput of the B200 this runs on — the
// roofline denominators for the Tersoff kernels (MEASURED_PEAKS.json has only
// HBM and bf16 tensor peaks).  Prints one JSON object.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp_peak tools/fp_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

template <typename T>
__global__ void fma_kernel(T* out, T a, T b) {
  T acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = T(threadIdx.x + c);
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], a, b);
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == T(-1.2345)) out[0] = s;
}

// packed FP32 (sm_100: FFMA2, one instruction for two lanes' worth of FMAs)
__global__ void fma2_kernel(float* out, float a, float b) {
  float2 acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = make_float2(threadIdx.x + c, threadIdx.x - c);
  const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = __ffma2_rn(acc[c], a2, b2);
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c].x + acc[c].y;
  if (s == -1.2345f) out[0] = s;
}

__global__ void mufu_kernel(float* out, float a) {
  float acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = 0.001f * (threadIdx.x + c);
  for (int it = 0; it < kIters; ++it) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = exp2f(acc[c]) * a;  // MUFU.EX2 + FMUL
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == -1.2345f) out[0] = s;
}

template <typename K>
double time_ms(K launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  const int blocks = sms * 8, threads = 256;
  const double lanes = double(blocks) * threads * kChains * kIters;
  double* d64;
  float* d32;
  cudaMalloc(&d64, 8);
  cudaMalloc(&d32, 8);
  const double t64 = time_ms([&] { fma_kernel<double><<<blocks, threads>>>(d64, 0.999, 1e-3); });
  const double t32 = time_ms([&] { fma_kernel<float><<<blocks, threads>>>(d32, 0.999f, 1e-3f); });
  const double tmu = time_ms([&] { mufu_kernel<<<blocks, threads>>>(d32, 0.5f); });
  const double tf2 = time_ms([&] { fma2_kernel<<<blocks, threads>>>(d32, 0.999f, 1e-3f); });
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  std::printf(
      "{\"gpu\": \"%s\", \"sms\": %d, \"clock_mhz_attr\": %.0f, "
      "\"fp64_tflops\": %.3f, \"fp32_tflops\": %.3f, \"fp32x2_tflops\": %.3f, "
      "\"mufu_ex2_gops\": %.1f, "
      "\"fp64_fma_per_clk_sm\": %.1f, \"fp32_fma_per_clk_sm\": %.1f, "
      "\"how\": \"8 independent FMA chains x 4096 iters, %d blocks x %d threads, best of 5; "
      "TFLOP/s counts an FMA as 2 flops\"}\n",
      prop.name, sms, clk / 1e3, 2.0 * lanes / (t64 * 1e-3) / 1e12,
      2.0 * lanes / (t32 * 1e-3) / 1e12, 4.0 * lanes / (tf2 * 1e-3) / 1e12,
      lanes / (tmu * 1e-3) / 1e9,
      lanes / (t64 * 1e-3) / sms / (clk * 1e3), lanes / (t32 * 1e-3) / sms / (clk * 1e3), blocks,
      threads);
  return 0;
}
