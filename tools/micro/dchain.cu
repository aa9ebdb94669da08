// Latency of the centroid update's serial f64 chain: one warp, 2 dims per
// lane, N rows from shared memory (acc += (double)x), cycles per row.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const float* g, double* out, int n, long long* cyc) {
  __shared__ float2 s[128 * 32];
  for (int i = threadIdx.x; i < 128 * 32; i += 32) s[i] = make_float2(g[i], g[i + 1]);
  __syncwarp();
  double a0 = 0, a1 = 0;
  long long t0 = clock64();
  for (int r = 0; r < n; ++r) {
    const float2 v = s[(r & 127) * 32 + threadIdx.x];
    a0 = __dadd_rn(a0, (double)v.x);
    a1 = __dadd_rn(a1, (double)v.y);
  }
  long long t1 = clock64();
  out[threadIdx.x] = a0 + a1;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  float* g; double* o; long long* c;
  cudaMalloc(&g, 2048 * 32 * 2 * 4 + 16); cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 8);
  cudaMemset(g, 0, 2048 * 32 * 2 * 4 + 16);
  for (int n : {256, 1024, 2048}) {
    k<<<1, 32>>>(g, o, n, c);
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("rows %d: %lld cycles, %.1f cycles/row\n", n, h, (double)h / n);
  }
}
