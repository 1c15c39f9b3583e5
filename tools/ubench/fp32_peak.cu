// Measured FP32 CUDA-core peak of this B200 for the GNN kernel's roofline: packed
// FFMA2 (fma.rn.f32x2) on 16 independent register pairs per thread, every SM
// fully occupied, ~0.2 s per run; prints one JSON line (best of 5 runs, FLOP = 2 per
// lane-FMA).  Run beside `nvidia-smi --query-gpu=clocks.sm --format=csv -lms 100`.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}

__global__ void __launch_bounds__(512) ffma2_peak(float* out, int iters) {
  unsigned long long a[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) a[j] = pk(threadIdx.x * 1e-3f + j, j * 0.5f);
  const unsigned long long x = pk(0.999f, 0.998f), w = pk(1e-7f, 2e-7f);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j) asm volatile("fma.rn.f32x2 %0, %1, %0, %2;" : "+l"(a[j]) : "l"(x), "l"(w));
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    float lo, hi;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[j]));
    s += lo + hi;
  }
  if (s == 1234.5f) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 4, threads = 512, iters = 1 << 16;
  ffma2_peak<<<blocks, threads>>>(out, 256);
  double best = 0.0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    ffma2_peak<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flop = 4.0 * blocks * threads * static_cast<double>(iters) * 16;
    const double tf = flop / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  printf("{\"fp32_ffma2_tflops\": %.2f, \"sms\": %d, \"blocks\": %d, \"threads\": %d, "
         "\"nominal_at_max_clock_tflops\": %.2f, \"err\": \"%s\"}\n",
         best, sms, blocks, threads, sms * 128.0 * 2.0 * clk_khz * 1e3 / 1e12,
         cudaGetErrorString(cudaGetLastError()));
  return 0;
}
