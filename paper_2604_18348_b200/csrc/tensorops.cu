// Dense f32 tensor ops of the reference's substrate and the scalar Quest form:
//   ac_matmul       tensorops.py:29-37  `a @ b` (f32, OpenBLAS accumulation order)
//   ac_row_softmax  tensorops.py:40-51  softmax over the last axis of scale * s
//   ac_quest_pairs  quest.py:74-91      quest_scalar / quest_scores_loop: per
//                   (query rep, cluster) sum_t max(q_t*max_ct, q_t*min_ct)
// None of these is on the per-step hot path (the pipeline uses the fused
// selection and attention kernels); they complete the drop-in surface of the
// reference's __init__.py:37-41.  Compiled with --fmad=false: every product
// and sum is the unfused f32 operation numpy performs, FMAs are explicit.
#include <cfloat>

#include "common.cuh"

namespace ac {

// a [m, kd] row-major, b [kd, n] row-major -> out [m, n].  One thread per
// output element; consecutive threads own consecutive columns j, so the b
// reads of one k-step are coalesced.
__global__ void k_matmul_nn(const float* __restrict__ a, const float* __restrict__ b,
                            float* __restrict__ out, int64_t m, int64_t n, int kd, int order) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = blockIdx.y;
  if (j >= n || i >= m) return;
  const float* ar = a + i * kd;
  auto ga = [&](int t) { return ar[t]; };
  auto gb = [&](int t) { return b[(int64_t)t * n + j]; };
  float acc;
  if (order == AC_ORDER_LANES16) {
    // small-matrix kernel: 16 lane chains, adjacent-pair tree (the corner
    // (m%4) x (n%4) elements use the halves tree, as in the selection kernel)
    const bool hv = (i >= m - m % 4) && (j >= n - n % 4);
    float r[16];
#pragma unroll
    for (int l = 0; l < 16; ++l) r[l] = 0.f;
    for (int t = 0; t < kd; ++t) r[t & 15] = __fmaf_rn(ga(t), gb(t), r[t & 15]);
    float s[8], u[4];
    if (hv) {
#pragma unroll
      for (int l = 0; l < 8; ++l) s[l] = __fadd_rn(r[l], r[l + 8]);
#pragma unroll
      for (int l = 0; l < 4; ++l) u[l] = __fadd_rn(s[l], s[l + 4]);
      acc = __fadd_rn(__fadd_rn(u[0], u[2]), __fadd_rn(u[1], u[3]));
    } else {
#pragma unroll
      for (int l = 0; l < 8; ++l) s[l] = __fadd_rn(r[2 * l], r[2 * l + 1]);
#pragma unroll
      for (int l = 0; l < 4; ++l) u[l] = __fadd_rn(s[2 * l], s[2 * l + 1]);
      acc = __fadd_rn(__fadd_rn(u[0], u[1]), __fadd_rn(u[2], u[3]));
    }
  } else if (order == AC_ORDER_GEMV8) {
    float r[8];
#pragma unroll
    for (int l = 0; l < 8; ++l) r[l] = 0.f;
    for (int t = 0; t < kd; ++t) r[t & 7] = __fmaf_rn(ga(t), gb(t), r[t & 7]);
    const float s0 = __fadd_rn(r[0], r[4]), s1 = __fadd_rn(r[1], r[5]);
    const float s2 = __fadd_rn(r[2], r[6]), s3 = __fadd_rn(r[3], r[7]);
    acc = __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
  } else {
    acc = 0.f;
    for (int t = 0; t < kd; ++t) acc = __fmaf_rn(ga(t), gb(t), acc);
  }
  out[i * n + j] = acc;
}

// One CTA per row: z = scale * s; z -= max(z); z = exp(z); z /= sum(z).
__global__ void __launch_bounds__(256)
k_row_softmax(const float* __restrict__ s, float* __restrict__ out, int64_t cols, float scale) {
  const int64_t row = blockIdx.x;
  const float* sr = s + row * cols;
  float* orow = out + row * cols;
  __shared__ float red[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float mx = -INFINITY;
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
    const float z = __fmul_rn(scale, sr[c]);
    orow[c] = z;
    mx = np_maximum(mx, z);
  }
  for (int o = 16; o; o >>= 1) mx = np_maximum(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  if (warp == 0) {
    float v = lane < nw ? red[lane] : -INFINITY;
    for (int o = 16; o; o >>= 1) v = np_maximum(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  mx = red[0];
  __syncthreads();
  float sum = 0.f;
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
    const float e = expf(__fsub_rn(orow[c], mx));
    orow[c] = e;
    sum = __fadd_rn(sum, e);
  }
  for (int o = 16; o; o >>= 1) sum = __fadd_rn(sum, __shfl_xor_sync(0xffffffffu, sum, o));
  if (lane == 0) red[warp] = sum;
  __syncthreads();
  if (warp == 0) {
    float v = lane < nw ? red[lane] : 0.f;
    for (int o = 16; o; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[0] = v;
  }
  __syncthreads();
  sum = red[0];
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) orow[c] = __fdiv_rn(orow[c], sum);
}

AC_DEV void quest_pair(const float* __restrict__ q, int d, const float* __restrict__ emax,
                       const float* __restrict__ emin, int g, int cl, float* out) {
  const float* qr = q + (int64_t)g * d;
  const float* mx = emax + (int64_t)cl * d;
  const float* mn = emin + (int64_t)cl * d;
  auto get = [&](int t) {
    return np_maximum(__fmul_rn(qr[t], mx[t]), __fmul_rn(qr[t], mn[t]));
  };
  *out = pw_sum<float>(get, d);
}

// quest_scalar (quest.py:74-77): float(np.maximum(q*max_c, q*min_c).sum()),
// the products in f32 and the length-d sum in numpy's pairwise order.
// quest_scores_loop (quest.py:80-91) is the reference's deliberately
// pair-at-a-time timing baseline for tensor_quest, so this kernel runs as ONE
// thread walking the pairs in (g, c) order -- the scalar form, not a second
// parallel scorer (the parallel scorer is k_select's matmul form).
__global__ void k_quest_pairs(const float* __restrict__ q, int gq, int d,
                              const float* __restrict__ emax, const float* __restrict__ emin,
                              int c, float* __restrict__ out) {
  for (int64_t e = 0; e < (int64_t)gq * c; ++e) {
    const int g = (int)(e / c), cl = (int)(e - (int64_t)g * c);
    quest_pair(q, d, emax, emin, g, cl, out + e);
  }
}

}  // namespace ac

using namespace ac;

extern "C" int ac_matmul(const float* a, int64_t m, int kd, const float* b, int64_t n,
                         float* out, int order, void* stream) {
  if (m < 0 || n < 0 || kd < 0) {
    ac_host::set_error("ac_matmul: negative size m=%lld n=%lld k=%d", (long long)m, (long long)n, kd);
    return AC_ERR_DIM;
  }
  if (m == 0 || n == 0) return AC_OK;
  if (m > 65535) {
    ac_host::set_error("ac_matmul: m=%lld > 65535 rows per call", (long long)m);
    return AC_ERR_DIM;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_matmul_nn<<<dim3((unsigned)((n + 127) / 128), (unsigned)m), 128, 0, st>>>(a, b, out, m, n, kd,
                                                                               order);
  AC_CHECK_LAUNCH("ac_matmul");
  return AC_OK;
}

extern "C" int ac_row_softmax(const float* s, int64_t rows, int64_t cols, float scale, float* out,
                              void* stream) {
  if (rows < 0 || cols < 0) {
    ac_host::set_error("ac_row_softmax: negative size");
    return AC_ERR_DIM;
  }
  if (rows == 0 || cols == 0) return AC_OK;
  if (rows > INT32_MAX) {
    ac_host::set_error("ac_row_softmax: too many rows");
    return AC_ERR_DIM;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_row_softmax<<<(unsigned)rows, 256, 0, st>>>(s, out, cols, scale);
  AC_CHECK_LAUNCH("ac_row_softmax");
  return AC_OK;
}

extern "C" int ac_quest_pairs(const float* q, int gq, int d, const float* emax, const float* emin,
                              int c, float* out, void* stream) {
  if (gq < 0 || c < 0 || d < 0) {
    ac_host::set_error("ac_quest_pairs: negative size");
    return AC_ERR_DIM;
  }
  const int64_t total = (int64_t)gq * c;
  if (total == 0) return AC_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  k_quest_pairs<<<1, 1, 0, st>>>(q, gq, d, emax, emin, c, out);
  AC_CHECK_LAUNCH("ac_quest_pairs");
  return AC_OK;
}
