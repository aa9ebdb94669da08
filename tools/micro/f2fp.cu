// F2FP (cvt.rn.bf16x2.f32) throughput alone and interleaved with MUFU ex2:
// do they share the XU pipe?  (conversions per clock per SM)
#include <cstdio>
__global__ void kcvt(float* out, int iters) {
  float a[8]; unsigned w[8];
  for (int i = 0; i < 8; ++i) { a[i] = 0.001f * (threadIdx.x + i); w[i] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      unsigned r;
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[(i + 1) & 7]));
      w[i] ^= r;
      a[i] = __uint_as_float(__float_as_uint(a[i]) ^ (r & 1));
    }
  }
  unsigned s = 0; for (int i = 0; i < 8; ++i) s ^= w[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
}
__global__ void kex2(float* out, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void kmix(float* out, int iters) {
  float a[8], b[8]; unsigned w[8];
  for (int i = 0; i < 8; ++i) { a[i] = -0.001f * (threadIdx.x + i); b[i] = 0.002f * i; w[i] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      unsigned r;
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b[i]), "f"(b[(i + 1) & 7]));
      w[i] ^= r;
      b[i] = __uint_as_float(__float_as_uint(b[i]) ^ (r & 1));
    }
  }
  float s = 0; unsigned t = 0; for (int i = 0; i < 8; ++i) { s += a[i]; t ^= w[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (float)t;
}
int main() {
  float* o; cudaMalloc(&o, 148 * 8 * 1024 * 4);
  int iters = 4096; cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double n = 148.0 * 8 * 1024 * 8 * iters;
  for (int r = 0; r < 2; ++r) {
    float ms;
    cudaEventRecord(a); kcvt<<<148 * 8, 1024>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("cvt bf16x2 alone: %.3f ms  %.1f instr/clk/SM\n", ms, n / (ms * 1e-3) / 148 / (clk * 1e3));
    cudaEventRecord(a); kex2<<<148 * 8, 1024>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("ex2 alone:        %.3f ms  %.1f instr/clk/SM\n", ms, n / (ms * 1e-3) / 148 / (clk * 1e3));
    cudaEventRecord(a); kmix<<<148 * 8, 1024>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("ex2+cvt mixed:    %.3f ms  %.1f pairs/clk/SM\n", ms, n / (ms * 1e-3) / 148 / (clk * 1e3));
  }
}
