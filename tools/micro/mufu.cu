// MUFU ex2 throughput: f32 vs f16x2 vs bf16x2 (elements per clock per SM)
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
__global__ void k32(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k16(float* out, int iters) {
  unsigned a[8];
  for (int i = 0; i < 8; ++i) { __half2 h = __floats2half2_rn(-0.001f * threadIdx.x, -0.002f * i); a[i] = *(unsigned*)&h; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i]));
  float s = 0; for (int i = 0; i < 8; ++i) { __half2 h = *(__half2*)&a[i]; s += __low2float(h) + __high2float(h); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void kb16(float* out, int iters) {
  unsigned a[8];
  for (int i = 0; i < 8; ++i) { __nv_bfloat162 h = __floats2bfloat162_rn(-0.001f * threadIdx.x, -0.002f * i); a[i] = *(unsigned*)&h; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i]));
  float s = 0; for (int i = 0; i < 8; ++i) { __nv_bfloat162 h = *(__nv_bfloat162*)&a[i]; s += __low2float(h) + __high2float(h); }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  int iters = 4096; cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int r = 0; r < 2; ++r) {
    float ms;
    cudaEventRecord(a); k32<<<148 * 8, 1024>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    double n32 = 148.0 * 8 * 1024 * 8 * iters;
    printf("f32   ex2: %.3f ms  %.1f elem/clk/SM (at %d MHz)\n", ms, n32 / (ms * 1e-3) / 148 / (clk * 1e3), clk / 1000);
    cudaEventRecord(a); k16<<<148 * 8, 1024>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("f16x2 ex2: %.3f ms  %.1f elem/clk/SM\n", ms, 2 * n32 / (ms * 1e-3) / 148 / (clk * 1e3));
    cudaEventRecord(a); kb16<<<148 * 8, 1024>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("bf16x2 ex2: %.3f ms  %.1f elem/clk/SM\n", ms, 2 * n32 / (ms * 1e-3) / 148 / (clk * 1e3));
  }
}
