// FP64 add / f32->f64 convert throughput and latency on this GPU
#include <cstdio>
__global__ void kadd(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __dadd_rn(a[i], 1.0000001);
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void klat(double* out, int iters) {
  double a = threadIdx.x;
  for (int it = 0; it < iters; ++it) a = __dadd_rn(a, 1.0000001);
  out[blockIdx.x * blockDim.x + threadIdx.x] = a;
}
__global__ void kcvt(double* out, int iters) {
  float f[8]; double a[8];
  for (int i = 0; i < 8; ++i) { f[i] = threadIdx.x * 1e-3f + i; a[i] = 0; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) { double d = (double)f[i]; f[i] = __int_as_float(__float_as_int(f[i]) ^ (int)it); a[i] = d; }
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* o; cudaMalloc(&o, 148 * 8 * 1024 * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float ms; int iters = 2048;
  for (int r = 0; r < 2; ++r) {
    cudaEventRecord(a); kadd<<<148 * 8, 1024>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    double n = 148.0 * 8 * 1024 * 8 * iters;
    printf("DADD throughput: %.1f /clk/SM\n", n / (ms * 1e-3) / 148 / (clk * 1e3));
    cudaEventRecord(a); klat<<<148, 32>>>(o, iters * 8); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("DADD latency: %.1f clk\n", (ms * 1e-3) * (clk * 1e3) / (iters * 8));
    cudaEventRecord(a); kcvt<<<148 * 8, 1024>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("F2F.F64.F32 (+1 LOP) throughput: %.1f /clk/SM\n", n / (ms * 1e-3) / 148 / (clk * 1e3));
  }
}
