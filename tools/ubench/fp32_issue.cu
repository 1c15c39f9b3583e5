// Microbenchmark: FP32 issue rates on sm_100a (FFMA with a uniform/constant
// operand vs packed FFMA2, and legacy HMMA tf32) — informs the GNN kernel design.
#include <cstdio>
#include <cuda_runtime.h>

__constant__ float cw[64];

__global__ void ffma_k(float* out, int iters) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3f + j;
  float x = threadIdx.x * 1e-4f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int m = 0; m < 16; ++m)
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = fmaf(x, cw[m * 4 + (j & 3)], a[j]);
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 1234.5f) out[0] = s;
}

__device__ __forceinline__ unsigned long long pk(float lo, float hi) {
  unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(lo), "f"(hi)); return r;
}
__global__ void ffma2_k(float* out, int iters) {
  unsigned long long a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = pk(threadIdx.x * 1e-3f + j, j * 0.5f);
  float x = threadIdx.x * 1e-4f;
  unsigned long long xx = pk(x, x);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int m = 0; m < 16; ++m) {
      unsigned long long w = pk(cw[m * 4], cw[m * 4 + 1]);
#pragma unroll
      for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a[j]) : "l"(xx), "l"(w));
    }
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) { float lo, hi; asm("mov.b64 {%0,%1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a[j])); s += lo + hi; }
  if (s == 1234.5f) out[0] = s;
}

__global__ void hmma_k(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, b0 = a0 * 3, b1 = a0 * 5;
  float c[4][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[q][0]), "+f"(c[q][1]), "+f"(c[q][2]), "+f"(c[q][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  float s = 0; for (int q = 0; q < 4; ++q) for (int j = 0; j < 4; ++j) s += c[q][j];
  if (s == 1234.5f) out[0] = s;
}

int main() {
  float* out; cudaMalloc(&out, 4);
  float h[64]; for (int i = 0; i < 64; ++i) h[i] = 1e-3f * i; cudaMemcpyToSymbol(cw, h, sizeof h);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = 148 * 4, threads = 256, iters = 4096;
  for (int warps : {4, 8, 16}) {
    threads = 32 * warps; blocks = 148;
    float ms;
    ffma_k<<<blocks, threads>>>(out, 16); cudaEventRecord(e0); ffma_k<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * blocks * threads * iters * 16 * 8;
    printf("warps/SM %2d FFMA(UR)  : %.1f TFLOP/s\n", warps, fl / ms / 1e9);
    ffma2_k<<<blocks, threads>>>(out, 16); cudaEventRecord(e0); ffma2_k<<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 4.0 * blocks * threads * iters * 16 * 8;
    printf("warps/SM %2d FFMA2     : %.1f TFLOP/s\n", warps, fl / ms / 1e9);
    hmma_k<<<blocks, threads>>>(out, 16); cudaEventRecord(e0); hmma_k<<<blocks, threads>>>(out, iters / 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 16 * 8 * 8 * (blocks * threads / 32.0) * (iters / 4) * 16;
    printf("warps/SM %2d HMMA tf32  : %.1f TFLOP/s\n", warps, fl / ms / 1e9);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
