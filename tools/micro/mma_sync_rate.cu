#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_tf32(float* out, int iters) {
  float c[8][4] = {};
  unsigned a0 = threadIdx.x, a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3, b0 = a0 ^ 5, b1 = a0 ^ 7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_f16(float* out, int iters) {
  float c[8][4] = {};
  unsigned a0 = threadIdx.x, a1 = a0 ^ 1, a2 = a0 ^ 2, a3 = a0 ^ 3, b0 = a0 ^ 5, b1 = a0 ^ 7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma(float* out, int iters) {
  float c[32];
  for (int j = 0; j < 32; ++j) c[j] = threadIdx.x * j;
  float a = out[0], b = out[1];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 32; ++j) c[j] = fmaf(c[j], a, b);
  }
  float s = 0; for (int j = 0; j < 32; ++j) s += c[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* d; cudaMalloc(&d, 148 * 32 * 1024 * 4); cudaMemset(d, 0, 16);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    int iters = 4096;
    for (int kind = 0; kind < 3; ++kind) {
      auto run = [&]() {
        if (kind == 0) k_tf32<<<148 * 4, warps * 8>>>(d, iters);
        else if (kind == 1) k_f16<<<148 * 4, warps * 8>>>(d, iters);
        else k_ffma<<<148 * 4, warps * 8>>>(d, iters);
      };
      run(); cudaDeviceSynchronize();
      cudaEventRecord(e0); run(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flop = kind == 0 ? 2.0 * 16 * 8 * 8 * 8 : kind == 1 ? 2.0 * 16 * 8 * 16 * 8 : 2.0 * 32 * 32;
      double total = flop * iters * (148.0 * 4 * warps * 8 / 32);
      printf("warps/SM %d kind %s: %.1f TFLOP/s\n", warps, kind == 0 ? "tf32" : kind == 1 ? "f16" : "ffma", total / ms / 1e9);
    }
  }
  return 0;
}
