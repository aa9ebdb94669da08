// Clustering kernels: row norms, l2 normalisation, k-means++ seeding,
// the Lloyd iteration (assign -> empty repair -> inertia -> stable segment
// sort -> f64 centroid update -> movement), and the multi-stage helpers.
//
// Reference: /root/reference/pkg/src/adacluster/clustering.py and
// tensorops.py.  Every arithmetic step reproduces numpy's f32/f64 semantics
// (pairwise sums, non-fused products, first-index argmin/argmax, f64 centre
// sums in member order), so labels and centres are bit-identical to the
// reference.  Compiled with --fmad=false.
#include <cfloat>
#include <climits>
#include <cstdlib>

#include "common.cuh"
#include "pairwise.cuh"

namespace ac {


// f32 NT dot product in the accumulation order of the reference's sgemm.
template <typename GetX, typename GetC>
AC_DEV float ordered_dot(const GetX& gx, const GetC& gc, int d, int order, bool halves = false) {
  if (order == AC_ORDER_LANES16) {
    float r[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) r[j] = 0.f;
    for (int t = 0; t < d; ++t) r[t & 15] = __fmaf_rn(gx(t), gc(t), r[t & 15]);
    float s[8], u[4];
    if (halves) {  // corner tile of the small kernel: _mm512_reduce_add_ps order
#pragma unroll
      for (int l = 0; l < 8; ++l) s[l] = __fadd_rn(r[l], r[l + 8]);
#pragma unroll
      for (int l = 0; l < 4; ++l) u[l] = __fadd_rn(s[l], s[l + 4]);
      return __fadd_rn(__fadd_rn(u[0], u[2]), __fadd_rn(u[1], u[3]));
    }
#pragma unroll
    for (int l = 0; l < 8; ++l) s[l] = __fadd_rn(r[2 * l], r[2 * l + 1]);
#pragma unroll
    for (int l = 0; l < 4; ++l) u[l] = __fadd_rn(s[2 * l], s[2 * l + 1]);
    return __fadd_rn(__fadd_rn(u[0], u[1]), __fadd_rn(u[2], u[3]));
  }
  if (order == AC_ORDER_GEMV8) {
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = 0.f;
    for (int t = 0; t < d; ++t) a[t & 7] = __fmaf_rn(gx(t), gc(t), a[t & 7]);
    float s0 = __fadd_rn(a[0], a[4]), s1 = __fadd_rn(a[1], a[5]);
    float s2 = __fadd_rn(a[2], a[6]), s3 = __fadd_rn(a[3], a[7]);
    return __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
  }
  float acc = 0.f;
  for (int t = 0; t < d; ++t) acc = __fmaf_rn(gx(t), gc(t), acc);
  return acc;
}


// ---------------------------------------------------------------------------
// K1: row squared norms and l2 normalisation (tensorops.py:59-76)
// ---------------------------------------------------------------------------
// Rows are staged through shared memory (coalesced global access, padded
// row stride d+1 so the thread-per-row pairwise sums are bank-conflict
// free); every row's arithmetic is the reference's numpy order.
constexpr int kNormRows = 128;

AC_DEV void stage_rows_f32(const void* __restrict__ x, int dtype, int64_t row0, int rows, int d,
                           float* s) {
  const int ld = d + 1;
  const int64_t base = row0 * d;
  for (int e = threadIdx.x; e < rows * d; e += blockDim.x) {
    const int r = e / d, t = e - r * d;
    s[r * ld + t] = ld_elem(x, dtype, base + e);
  }
}

AC_DEV float row_sq_pw(const float* s, int d) {
  return pw_sum<float>([&](int i) { return __fmul_rn(s[i], s[i]); }, d);
}

__global__ void __launch_bounds__(kNormRows)
k_row_sqnorm(const void* __restrict__ x, int dtype, int64_t rows, int d, float* __restrict__ out) {
  extern __shared__ float nsm[];
  const int64_t row0 = (int64_t)blockIdx.x * kNormRows;
  const int nr = (int)min((int64_t)kNormRows, rows - row0);
  stage_rows_f32(x, dtype, row0, nr, d, nsm);
  __syncthreads();
  if ((int)threadIdx.x < nr) out[row0 + threadIdx.x] = row_sq_pw(nsm + threadIdx.x * (d + 1), d);
}

__global__ void __launch_bounds__(kNormRows)
k_l2norm(const void* __restrict__ x, int dtype, int64_t rows, int d, float* __restrict__ out,
         float* __restrict__ out_sq, uint8_t* __restrict__ degenerate) {
  extern __shared__ float nsm[];
  const int ld = d + 1;
  const int64_t row0 = (int64_t)blockIdx.x * kNormRows;
  const int nr = (int)min((int64_t)kNormRows, rows - row0);
  stage_rows_f32(x, dtype, row0, nr, d, nsm);
  __syncthreads();
  const int r = threadIdx.x;
  if (r < nr) {
    float* s = nsm + r * ld;
    const float norm = __fsqrt_rn(row_sq_pw(s, d));
    const bool degen = norm < 1e-12f;                         // DEGENERATE_NORM
    const bool unit = fabsf(__fsub_rn(norm, 1.0f)) <= 2e-6f;  // already unit
    const float safe = (degen || unit) ? 1.0f : norm;
    for (int i = 0; i < d; ++i) s[i] = degen ? 0.f : __fdiv_rn(s[i], safe);
    if (degenerate) degenerate[row0 + r] = degen ? 1 : 0;
    if (out_sq) out_sq[row0 + r] = row_sq_pw(s, d);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nr * d; e += blockDim.x) {
    const int rr = e / d, t = e - rr * d;
    out[row0 * d + e] = nsm[rr * ld + t];
  }
}

// ---- fast path for D = 64 / 128 (16-byte aligned rows) --------------------
// 64 rows per 256-thread block staged as f32 [64][D+8] with 16-byte loads;
// 8 lanes per row each run one of numpy's 8 pairwise accumulators
// (pw_leaf: r_j = sum_m a[j+8m] in order) and the shuffle tree combines them
// as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) -- same operations, same bits.
// The stride D+8 puts the 4 rows x 8 lanes of one access on 32 banks.
constexpr int kRowsV = 64;

template <int D>
AC_DEV void stage_rows_v(const void* __restrict__ x, int dtype, int64_t row0, int nr, float* s) {
  constexpr int LD = D + 8;
  if (reinterpret_cast<uintptr_t>(x) & 15) {  // unaligned rows: element loads
    for (int e = threadIdx.x; e < nr * D; e += blockDim.x)
      s[(e / D) * LD + e % D] = ld_elem(x, dtype, row0 * D + e);
    return;
  }
  if (dtype == AC_DTYPE_BF16) {
    const uint4* src = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(x) + row0 * D);
    for (int c = threadIdx.x; c < nr * (D / 8); c += blockDim.x) {
      const int r = c / (D / 8), j = c % (D / 8);
      const uint4 w = __ldg(src + c);
      const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
      float4* dst = reinterpret_cast<float4*>(s + r * LD + 8 * j);
      dst[0] = make_float4(__uint_as_float(ww[0] << 16), __uint_as_float(ww[0] & 0xffff0000u),
                           __uint_as_float(ww[1] << 16), __uint_as_float(ww[1] & 0xffff0000u));
      dst[1] = make_float4(__uint_as_float(ww[2] << 16), __uint_as_float(ww[2] & 0xffff0000u),
                           __uint_as_float(ww[3] << 16), __uint_as_float(ww[3] & 0xffff0000u));
    }
  } else {
    const float4* src = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(x) + row0 * D);
    for (int c = threadIdx.x; c < nr * (D / 4); c += blockDim.x) {
      const int r = c / (D / 4), j = c % (D / 4);
      *reinterpret_cast<float4*>(s + r * LD + 4 * j) = __ldg(src + c);
    }
  }
}

// combine the 8 accumulators of a lane group (lanes 8g..8g+7) in numpy's order
AC_DEV float pw8_combine(float r) {
  r = __fadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
  r = __fadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
  return __fadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
}

template <int D>
AC_DEV float row_sq_pw8(const float* srow, int j) {
  float r = __fmul_rn(srow[j], srow[j]);
#pragma unroll
  for (int m = 1; m < D / 8; ++m) r = __fadd_rn(r, __fmul_rn(srow[j + 8 * m], srow[j + 8 * m]));
  return pw8_combine(r);
}

// exact bf16 hi/mid/lo split of 8 staged values -> planes[q][row][8j..8j+7]
AC_DEV void write_planes8(const float* v, __nv_bfloat16* pl, int64_t plane, int64_t o) {
  uint32_t h[4], m[4], l[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    uint32_t hh[2], mm[2], ll[2];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const float a = v[2 * e + u];
      const __nv_bfloat16 b0 = __float2bfloat16_rn(a);
      const float r1 = __fsub_rn(a, __bfloat162float(b0));
      const __nv_bfloat16 b1 = __float2bfloat16_rn(r1);
      const __nv_bfloat16 b2 = __float2bfloat16_rn(__fsub_rn(r1, __bfloat162float(b1)));
      hh[u] = __bfloat16_as_ushort(b0);
      mm[u] = __bfloat16_as_ushort(b1);
      ll[u] = __bfloat16_as_ushort(b2);
    }
    h[e] = hh[0] | (hh[1] << 16);
    m[e] = mm[0] | (mm[1] << 16);
    l[e] = ll[0] | (ll[1] << 16);
  }
  *reinterpret_cast<uint4*>(pl + o) = make_uint4(h[0], h[1], h[2], h[3]);
  *reinterpret_cast<uint4*>(pl + plane + o) = make_uint4(m[0], m[1], m[2], m[3]);
  *reinterpret_cast<uint4*>(pl + 2 * plane + o) = make_uint4(l[0], l[1], l[2], l[3]);
}

// One block of rows [row0, row0+nr): optional l2 normalisation (K1
// semantics of k_l2norm), ||row||^2 of the (normalised) rows, the f32 rows
// (when normalising) and their bf16 planes.  Plane rows are addressed per
// problem: global row g -> problem g / prob_rows, [3][prob_rows][D] each.
template <int D>
AC_DEV void rows_block_v(const void* __restrict__ x, int dtype, int64_t row0, int nr, bool normalise,
                         float* __restrict__ out, float* __restrict__ out_sq,
                         uint8_t* __restrict__ degenerate, __nv_bfloat16* __restrict__ planes,
                         int64_t prob_rows, float* s) {
  constexpr int LD = D + 8;
  stage_rows_v<D>(x, dtype, row0, nr, s);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, j = lane & 7;
  const int nwarps = blockDim.x >> 5;
  for (int rb = warp * 4; rb < nr; rb += nwarps * 4) {
    const int r = rb + (lane >> 3);
    const bool ok = r < nr;
    float* srow = s + (ok ? r : 0) * LD;
    float sq = row_sq_pw8<D>(srow, j);
    if (normalise) {
      const float norm = __fsqrt_rn(sq);
      const bool degen = norm < 1e-12f;                         // DEGENERATE_NORM
      const bool unit = fabsf(__fsub_rn(norm, 1.0f)) <= 2e-6f;  // already unit
      const float safe = (degen || unit) ? 1.0f : norm;
      float acc = 0.f;
#pragma unroll
      for (int m = 0; m < D / 8; ++m) {
        const float v = degen ? 0.f : __fdiv_rn(srow[j + 8 * m], safe);
        if (ok) srow[j + 8 * m] = v;
        acc = m == 0 ? __fmul_rn(v, v) : __fadd_rn(acc, __fmul_rn(v, v));
      }
      sq = pw8_combine(acc);
      if (ok && j == 0 && degenerate) degenerate[row0 + r] = degen ? 1 : 0;
    }
    if (ok && j == 0 && out_sq) out_sq[row0 + r] = sq;
  }
  __syncthreads();
  if (normalise && out) {
    float4* dst = reinterpret_cast<float4*>(out + row0 * D);
    for (int c = threadIdx.x; c < nr * (D / 4); c += blockDim.x) {
      const int r = c / (D / 4), jj = c % (D / 4);
      dst[c] = *reinterpret_cast<const float4*>(s + r * LD + 4 * jj);
    }
  }
  if (planes && !(reinterpret_cast<uintptr_t>(planes) & 15)) {
    for (int c = threadIdx.x; c < nr * (D / 8); c += blockDim.x) {
      const int r = c / (D / 8), jj = c % (D / 8);
      const int64_t g = row0 + r, p = g / prob_rows, i = g - p * prob_rows;
      const int64_t plane = prob_rows * D;
      write_planes8(s + r * LD + 8 * jj, planes + 3 * p * plane, plane, i * D + 8 * jj);
    }
  }
}

template <int D>
__global__ void __launch_bounds__(256)
k_l2norm_v(const void* __restrict__ x, int dtype, int64_t rows, float* __restrict__ out,
           float* __restrict__ out_sq, uint8_t* __restrict__ degenerate,
           __nv_bfloat16* __restrict__ planes, int64_t prob_rows) {
  extern __shared__ float nsm[];
  const int64_t row0 = (int64_t)blockIdx.x * kRowsV;
  const int nr = (int)min((int64_t)kRowsV, rows - row0);
  rows_block_v<D>(x, dtype, row0, nr, true, out, out_sq, degenerate, planes, prob_rows, nsm);
}

template <int D>
__global__ void __launch_bounds__(256)
k_problem_xx_v(const ac_cluster_problem* __restrict__ probs, int dtype) {
  extern __shared__ float nsm[];
  const ac_cluster_problem& P = probs[blockIdx.y];
  const int64_t row0 = (int64_t)blockIdx.x * kRowsV;
  if (row0 >= P.n) return;
  const int nr = (int)min((int64_t)kRowsV, P.n - row0);
  __nv_bfloat16* pl = (P.planes && dtype == AC_DTYPE_F32) ? reinterpret_cast<__nv_bfloat16*>(P.planes) : nullptr;
  rows_block_v<D>(P.x, dtype, row0, nr, false, nullptr, P.xx, nullptr, pl, P.n, nsm);
}

// center squared norms cc[c] for problem blockIdx.y
__global__ void k_center_sqnorm(const ac_cluster_problem* __restrict__ probs, int d,
                                int c_lo) {
  pdl_wait();
  pdl_trigger();
  const ac_cluster_problem& P = probs[blockIdx.y];
  const int c = c_lo + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= P.k) return;
  const float* row = P.centers + (int64_t)c * d;
  auto get = [&](int i) { return __fmul_rn(row[i], row[i]); };
  P.cc[c] = pw_sum<float>(get, d);
}

__global__ void __launch_bounds__(kNormRows)
k_problem_xx(const ac_cluster_problem* __restrict__ probs, int dtype, int d) {
  extern __shared__ float nsm[];
  const ac_cluster_problem& P = probs[blockIdx.y];
  const int64_t row0 = (int64_t)blockIdx.x * kNormRows;
  if (row0 >= P.n) return;
  const int nr = (int)min((int64_t)kNormRows, P.n - row0);
  stage_rows_f32(P.x, dtype, row0, nr, d, nsm);
  __syncthreads();
  if ((int)threadIdx.x < nr) P.xx[row0 + threadIdx.x] = row_sq_pw(nsm + threadIdx.x * (d + 1), d);
  if (P.planes && dtype == AC_DTYPE_F32) {
    // exact split x = hi + mid + lo into bf16 planes [3][n][d] (coalesced)
    __nv_bfloat16* pl = reinterpret_cast<__nv_bfloat16*>(P.planes);
    const int64_t plane = P.n * d;
    for (int e = threadIdx.x; e < nr * d; e += blockDim.x) {
      const int r = e / d, t = e - r * d;
      const float v = nsm[r * (d + 1) + t];
      const __nv_bfloat16 hi = __float2bfloat16_rn(v);
      const float r1 = __fsub_rn(v, __bfloat162float(hi));
      const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
      const __nv_bfloat16 lo = __float2bfloat16_rn(__fsub_rn(r1, __bfloat162float(mid)));
      const int64_t o = row0 * d + e;
      pl[o] = hi;
      pl[plane + o] = mid;
      pl[2 * plane + o] = lo;
    }
  }
}

__global__ void k_status_init(const ac_cluster_problem* __restrict__ probs, int nprob) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nprob) return;
  int32_t* st = probs[p].status;
  st[AC_ST_ACTIVE] = 1;
  st[AC_ST_NITER] = 0;
  st[AC_ST_DONE] = 0;
  st[AC_ST_FLAGS] = 0;
  st[AC_ST_KPP_STOP] = -1;
  st[AC_ST_REPAIRS] = 0;
  st[AC_ST_FIXUPS] = 0;
  st[AC_ST_WIDE] = 0;
}

// ---------------------------------------------------------------------------
// K3: assignment.  x @ centers.T as per-thread sequential fmaf chains
// (the reference's OpenBLAS general-path order), 128 rows x 64 centres per
// CTA pass, 8x4 register tile per thread; fused distance + first-index argmin
// + per-tile label histogram.
// ---------------------------------------------------------------------------
constexpr int kAsgBM = 128;
constexpr int kAsgBN = 64;
constexpr int kAsgPadM = kAsgBM + 4;
constexpr int kAsgPadN = kAsgBN + 4;

__host__ __device__ inline size_t assign_smem_bytes(int d, int kcap) {
  return sizeof(float) * ((size_t)d * kAsgPadM + (size_t)d * kAsgPadN + kAsgBM + kAsgBN +
                          8 * kAsgBM) +
         sizeof(int) * (8 * kAsgBM + (size_t)kcap + 4);
}

__global__ void __launch_bounds__(256)
k_assign_seq(const ac_cluster_problem* __restrict__ probs, int dtype, int d, int c_lo,
             int flags, int kcap) {
  extern __shared__ __align__(16) float smem[];
  const ac_cluster_problem& P = probs[blockIdx.y];
  if (!(flags & AC_ASSIGN_ALL) && P.status[AC_ST_ACTIVE] == 0) return;
  const int64_t n = P.n;
  const int64_t row0 = (int64_t)blockIdx.x * kAsgBM;
  if (row0 >= n) return;
  const int rows = (int)min((int64_t)kAsgBM, n - row0);
  const int k = P.k;

  float* xs = smem;                       // [d][kAsgPadM]
  float* cs = xs + (size_t)d * kAsgPadM;  // [d][kAsgPadN]
  float* s_xx = cs + (size_t)d * kAsgPadN;
  float* s_cc = s_xx + kAsgBM;
  float* s_bd = s_cc + kAsgBN;            // [8][kAsgBM]
  int* s_bi = reinterpret_cast<int*>(s_bd + 8 * kAsgBM);
  int* s_hist = s_bi + 8 * kAsgBM;        // [kcap]

  const int tid = threadIdx.x;
  // x tile, transposed: consecutive threads take consecutive rows so the
  // shared-memory stores are conflict-free
  for (int e = tid; e < kAsgBM * d; e += blockDim.x) {
    const int t = e / kAsgBM, r = e - t * kAsgBM;
    xs[t * kAsgPadM + r] = (r < rows) ? ld_elem(P.x, dtype, (row0 + r) * d + t) : 0.f;
  }
  for (int r = tid; r < kAsgBM; r += blockDim.x) s_xx[r] = (r < rows) ? P.xx[row0 + r] : 0.f;

  // thread (tm, tn): rows tm*4+i and 64+tm*4+i (i < 4) — two 16-lane-contiguous
  // float4 reads per k step, conflict-free — and centres tn*4 .. tn*4+3
  const int tm = tid & 15;
  const int tn = tid >> 4;
  float bd[8];
  int bi[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { bd[i] = INFINITY; bi[i] = INT_MAX; }

  for (int cb = c_lo; cb < k; cb += kAsgBN) {
    __syncthreads();
    const int nc = min(kAsgBN, k - cb);
    for (int e = tid; e < kAsgBN * d; e += blockDim.x) {
      const int t = e / kAsgBN, j = e - t * kAsgBN;
      cs[t * kAsgPadN + j] = (j < nc) ? P.centers[(int64_t)(cb + j) * d + t] : 0.f;
    }
    for (int j = tid; j < kAsgBN; j += blockDim.x) s_cc[j] = (j < nc) ? P.cc[cb + j] : 0.f;
    __syncthreads();
    if (tn * 4 < nc) {
      float acc[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
      const float* xp = xs + tm * 4;
      const float* cp = cs + tn * 4;
#pragma unroll 4
      for (int t = 0; t < d; ++t) {
        const float4 a0 = *reinterpret_cast<const float4*>(xp + t * kAsgPadM);
        const float4 a1 = *reinterpret_cast<const float4*>(xp + t * kAsgPadM + 64);
        const float4 b = *reinterpret_cast<const float4*>(cp + t * kAsgPadN);
        const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float bb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(a[i], bb[j], acc[i][j]);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int rr = (i < 4) ? tm * 4 + i : 64 + tm * 4 + (i - 4);
        const float xx = s_xx[rr];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int jj = tn * 4 + j;
          if (jj < nc) {
            const float dd = sq_dist(xx, acc[i][j], s_cc[jj]);
            if (dd < bd[i]) { bd[i] = dd; bi[i] = cb + jj; }
          }
        }
      }
    }
  }
  // merge the 16 centre groups of each row: lanes l and l^16 share tm
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float od = __shfl_xor_sync(0xffffffffu, bd[i], 16);
    const int oi = __shfl_xor_sync(0xffffffffu, bi[i], 16);
    argmin_merge(bd[i], bi[i], od, oi);
  }
  __syncthreads();
  const int warp = tid >> 5, lane = tid & 31;
  if (lane < 16) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int rr = (i < 4) ? tm * 4 + i : 64 + tm * 4 + (i - 4);
      s_bd[warp * kAsgBM + rr] = bd[i];
      s_bi[warp * kAsgBM + rr] = bi[i];
    }
  }
  const bool count = !(flags & AC_ASSIGN_MERGE);
  if (count)
    for (int c = tid; c < k; c += blockDim.x) s_hist[c] = 0;
  __syncthreads();
  if (tid < rows) {
    float b = s_bd[tid];
    int l = s_bi[tid];
    for (int w = 1; w < 8; ++w) argmin_merge(b, l, s_bd[w * kAsgBM + tid], s_bi[w * kAsgBM + tid]);
    const int64_t r = row0 + tid;
    if (flags & AC_ASSIGN_MERGE) {
      const float eb = P.best[r];
      if (!(b < eb)) { b = eb; l = P.labels[r]; }
    }
    if (l == INT_MAX) l = c_lo;  // all-NaN row: numpy argmin returns the first index
    P.labels[r] = l;
    P.best[r] = b;
    if (count) atomicAdd(&s_hist[l], 1);
  }
  if (count) {
    __syncthreads();
    const int64_t ntiles = (n + kAsgBM - 1) / kAsgBM;
    int32_t* th = P.tile_hist + blockIdx.x;
    for (int c = tid; c < k; c += blockDim.x) th[(int64_t)c * ntiles] = s_hist[c];
  }
}

// Generic-order assignment for the small shapes the reference sends through
// OpenBLAS's small-matrix / GEMV kernels (M*N <= ~1.2K or a unit dimension).
// One thread per row; centres staged in shared memory.
__global__ void k_assign_generic(const ac_cluster_problem* __restrict__ probs, int dtype,
                                 int d, int c_lo, int flags, int kcap) {
  extern __shared__ __align__(16) float smem[];
  const ac_cluster_problem& P = probs[blockIdx.y];
  if (!(flags & AC_ASSIGN_ALL) && P.status[AC_ST_ACTIVE] == 0) return;
  const int64_t n = P.n;
  const int64_t row0 = (int64_t)blockIdx.x * kAsgBM;
  if (row0 >= n) return;
  const int k = P.k;
  int* s_hist = reinterpret_cast<int*>(smem);
  const bool count = !(flags & AC_ASSIGN_MERGE);
  if (count)
    for (int c = threadIdx.x; c < k; c += blockDim.x) s_hist[c] = 0;
  __syncthreads();
  const int64_t r = row0 + threadIdx.x;
  if (threadIdx.x < kAsgBM && r < n) {
    const int64_t base = r * d;
    const float xx = P.xx[r];
    float b = INFINITY;
    int l = INT_MAX;
    for (int c = c_lo; c < k; ++c) {
      const float* crow = P.centers + (int64_t)c * d;
      const bool halves = (r >= n - n % 4) && (c >= k - k % 4);
      const float xc = ordered_dot([&](int t) { return ld_elem(P.x, dtype, base + t); },
                                   [&](int t) { return crow[t]; }, d, P.order, halves);
      const float dd = sq_dist(xx, xc, P.cc[c]);
      if (dd < b) { b = dd; l = c; }
    }
    if (flags & AC_ASSIGN_MERGE) {
      const float eb = P.best[r];
      if (!(b < eb)) { b = eb; l = P.labels[r]; }
    }
    if (l == INT_MAX) l = c_lo;
    P.labels[r] = l;
    P.best[r] = b;
    if (count) atomicAdd(&s_hist[l], 1);
  }
  if (count) {
    __syncthreads();
    const int64_t ntiles = (n + kAsgBM - 1) / kAsgBM;
    int32_t* th = P.tile_hist + blockIdx.x;
    for (int c = threadIdx.x; c < k; c += blockDim.x) th[(int64_t)c * ntiles] = s_hist[c];
  }
}

// per-tile label histogram from existing labels (sort without re-assigning)
__global__ void k_tile_hist(const ac_cluster_problem* __restrict__ probs, int kcap) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) int thsm[];
  const ac_cluster_problem& P = probs[blockIdx.y];
  const int64_t row0 = (int64_t)blockIdx.x * kAsgBM;
  if (row0 >= P.n) return;
  const int rows = (int)min((int64_t)kAsgBM, P.n - row0);
  const int k = P.k;
  for (int c = threadIdx.x; c < k; c += blockDim.x) thsm[c] = 0;
  __syncthreads();
  if ((int)threadIdx.x < rows) atomicAdd(&thsm[P.labels[row0 + threadIdx.x]], 1);
  __syncthreads();
  const int64_t ntiles = (P.n + kAsgBM - 1) / kAsgBM;
  int32_t* th = P.tile_hist + blockIdx.x;
  for (int c = threadIdx.x; c < k; c += blockDim.x) th[(int64_t)c * ntiles] = thsm[c];
}

// ---------------------------------------------------------------------------
// Stable counting sort by label (np.argsort(labels, kind="stable")):
//   scan:    per label, exclusive prefix of the per-tile histograms (relative
//            tile bases) and the label's total count
//   post:    (one CTA per problem) empty-cluster repair, inertia, starts
//   scatter: perm[starts[c] + base[tile][c] + rank-in-tile] = row
// ---------------------------------------------------------------------------
__global__ void k_hist_scan(const ac_cluster_problem* __restrict__ probs, int flags) {
  pdl_wait();
  pdl_trigger();
  const ac_cluster_problem& P = probs[blockIdx.y];
  if (!(flags & AC_ASSIGN_ALL) && P.status[AC_ST_ACTIVE] == 0) return;
  const int k = P.k;
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= k) return;
  const int tiles = (int)((P.n + kAsgBM - 1) / kAsgBM);
  int32_t* h = P.tile_hist + (int64_t)c * tiles;  // this label's row, contiguous over tiles
  int run = 0;
  for (int t0 = 0; t0 < tiles; t0 += 32) {
    const int t = t0 + lane;
    const int v = (t < tiles) ? h[t] : 0;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (t < tiles) h[t] = run + inc - v;
    run += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) P.counts[c] = run;
}

// _repair_empty (clustering.py:100-116) + inertia (:132) + segment starts.
// One CTA (1024 threads) per problem.  `iter` < 0 skips the inertia entry.
__global__ void __launch_bounds__(1024)
k_post(const ac_cluster_problem* __restrict__ probs, int dtype, int d, int iter, int flags) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char psm[];
  const ac_cluster_problem& P = probs[blockIdx.x];
  if (!(flags & AC_ASSIGN_ALL) && P.status[AC_ST_ACTIVE] == 0) return;
  const int k = P.k;
  const int64_t n = P.n;
  const int tid = threadIdx.x;
  __shared__ int s_empty;
  __shared__ float s_far_d[32];
  __shared__ long long s_far_i[32];
  __shared__ int s_scan[1024];

  // labels-only assignment left approximate distances in `best`: the repair
  // below needs the reference's exact ones, so recompute them (rare: only
  // when some cluster is empty)
  if (flags & AC_ASSIGN_LABELS_ONLY) {
    if (tid == 0) s_empty = INT_MAX;
    __syncthreads();
    for (int c = tid; c < k; c += blockDim.x)
      if (P.counts[c] == 0) atomicMin(&s_empty, c);
    __syncthreads();
    if (s_empty != INT_MAX) {
      for (int64_t i = tid; i < n; i += blockDim.x) {
        const int l = P.labels[i];
        const float* crow = P.centers + (int64_t)l * d;
        const int64_t base = i * d;
        const bool halves = (i >= n - n % 4) && (l >= k - k % 4);
        const float xc = ordered_dot([&](int t) { return ld_elem(P.x, dtype, base + t); },
                                     [&](int t) { return crow[t]; }, d, P.order, halves);
        P.best[i] = sq_dist(P.xx[i], xc, P.cc[l]);
      }
      __threadfence_block();
    }
    __syncthreads();
  }

  // ---- empty-cluster repair: loop to a fixed point, at most k times ----
  for (int guard = 0; guard < k; ++guard) {
    if (tid == 0) s_empty = INT_MAX;
    __syncthreads();
    for (int c = tid; c < k; c += blockDim.x)
      if (P.counts[c] == 0) atomicMin(&s_empty, c);
    __syncthreads();
    const int c = s_empty;
    if (c == INT_MAX) break;
    // far = argmax of the assigned distances (first maximum)
    float bdv = -INFINITY;
    long long bix = LLONG_MAX;
    for (int64_t i = tid; i < n; i += blockDim.x) {
      const float v = P.best[i];
      if (v > bdv) { bdv = v; bix = i; }
    }
    for (int o = 16; o; o >>= 1) {
      const float od = __shfl_xor_sync(0xffffffffu, bdv, o);
      const long long oi = __shfl_xor_sync(0xffffffffu, bix, o);
      if (od > bdv || (od == bdv && oi < bix)) { bdv = od; bix = oi; }
    }
    if ((tid & 31) == 0) { s_far_d[tid >> 5] = bdv; s_far_i[tid >> 5] = bix; }
    __syncthreads();
    if (tid == 0) {
      float fd = s_far_d[0];
      long long fi = s_far_i[0];
      for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
        if (s_far_d[w] > fd || (s_far_d[w] == fd && s_far_i[w] < fi)) { fd = s_far_d[w]; fi = s_far_i[w]; }
      s_far_i[0] = fi;
    }
    __syncthreads();
    const int64_t far = s_far_i[0];
    const int old = P.labels[far];
    for (int t = tid; t < d; t += blockDim.x)
      P.centers[(int64_t)c * d + t] = ld_elem(P.x, dtype, far * d + t);
    __syncthreads();
    if (tid == 0) {
      P.labels[far] = c;
      P.best[far] = 0.f;  // ((x[far] - x[far])**2).sum() == 0
      P.counts[c] += 1;
      P.counts[old] -= 1;
      P.status[AC_ST_REPAIRS] += 1;
    }
    // relative tile bases: tiles after far's tile see one fewer `old`, one more `c`
    const int tiles = (int)((n + kAsgBM - 1) / kAsgBM);
    const int ft = (int)(far / kAsgBM);
    for (int t = ft + 1 + tid; t < tiles; t += blockDim.x) {
      P.tile_hist[(int64_t)old * tiles + t] -= 1;
      P.tile_hist[(int64_t)c * tiles + t] += 1;
    }
    __syncthreads();
  }

  // ---- inertia_history entry: float(d[arange(n), labels].sum()) ----
  if (iter >= 0) {
    PwPlan plan{P.plan_n};
    float* vals = reinterpret_cast<float*>(psm);
    const float* best = P.best;
    const float s = pw_eval_block_g8<float>(plan, [&](int i) { return best[i]; }, vals);
    if (tid == 0) P.inertia[iter] = s;
  }

  // ---- starts = exclusive scan of counts (k <= 1024 * chunk) ----
  const int per = (k + blockDim.x - 1) / blockDim.x;
  int local = 0;
  for (int j = 0; j < per; ++j) {
    const int c = tid * per + j;
    if (c < k) local += P.counts[c];
  }
  s_scan[tid] = local;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {
    const int v = (tid >= off) ? s_scan[tid - off] : 0;
    __syncthreads();
    s_scan[tid] += v;
    __syncthreads();
  }
  int run = s_scan[tid] - local;
  for (int j = 0; j < per; ++j) {
    const int c = tid * per + j;
    if (c < k) { P.starts[c] = run; run += P.counts[c]; }
  }
  if (tid == blockDim.x - 1) P.starts[k] = s_scan[tid];
}

__global__ void k_scatter(const ac_cluster_problem* __restrict__ probs, int flags) {
  pdl_wait();
  pdl_trigger();
  const ac_cluster_problem& P = probs[blockIdx.y];
  if (!(flags & AC_ASSIGN_ALL) && P.status[AC_ST_ACTIVE] == 0) return;
  const int64_t row0 = (int64_t)blockIdx.x * kAsgBM;
  if (row0 >= P.n) return;
  const int rows = (int)min((int64_t)kAsgBM, P.n - row0);
  __shared__ int s_lab[kAsgBM];
  const int tid = threadIdx.x;
  if (tid < rows) s_lab[tid] = P.labels[row0 + tid];
  __syncthreads();
  if (tid < rows) {
    const int l = s_lab[tid];
    int rank = 0;
    for (int j = 0; j < tid; ++j) rank += (s_lab[j] == l);
    const int64_t ntiles = (P.n + kAsgBM - 1) / kAsgBM;
    const int pos = P.starts[l] + P.tile_hist[(int64_t)l * ntiles + blockIdx.x] + rank;
    P.perm[pos] = (int32_t)(row0 + tid);
  }
}

// ---------------------------------------------------------------------------
// K4: centroid update (clustering.py:133-143).  One CTA per centre: member
// rows (in stable label order) are staged through shared memory with
// cp.async double buffering so ~64 rows are in flight; thread t < D owns the
// f64 chain of dimension t and adds the members in order, exactly like
// np.add.reduceat(x[order].astype(f64), starts) (first row initialises).
// Then / count -> f32, the f32 movement norm and the new ||c||^2; the last
// CTA of a problem reduces the movement mean and clears `active` when
// movement < tol.  mode 1 = segment mean into outs[p] (query reps).
// ---------------------------------------------------------------------------
constexpr int kUpdRows = 32;    // rows per pipeline stage
constexpr int kUpdStages = 4;   // row stages in flight
constexpr int kUpdIdx = kUpdStages + 2;  // member-index slots (fetched two chunks ahead)

AC_DEV void cp_async16(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
AC_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
AC_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__host__ __device__ inline size_t update_smem_bytes(int d, int dtype) {
  const size_t rb = (size_t)d * (dtype == AC_DTYPE_BF16 ? 2 : 4);
  return kUpdStages * kUpdRows * ((rb + 15) / 16 * 16) + sizeof(int) * kUpdIdx * kUpdRows +
         sizeof(float) * 2 * (size_t)d + 16;
}

// One CTA per centre.  Member rows (stable label order) are gathered into a
// 4-stage shared-memory ring with cp.async.  The member indices are
// register-prefetched two chunks ahead, so neither the index load nor the
// row load sits on the critical path.  Thread t < D owns the f64 chain of
// dimension t and adds the members strictly in order (first row
// initialises), exactly like np.add.reduceat(x[order].astype(f64), starts).
__global__ void __launch_bounds__(256)
k_update(const ac_cluster_problem* __restrict__ probs, int dtype, int d, double tol,
         int mode /*0 = lloyd update, 1 = segment mean into out*/, float* const* outs) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char usm[];
  const ac_cluster_problem& P = probs[blockIdx.y];
  if (mode == 0 && P.status[AC_ST_ACTIVE] == 0) return;
  const int c = blockIdx.x;
  const int k = P.k;
  if (c >= k) return;
  const int tid = threadIdx.x;
  const int esz = dtype == AC_DTYPE_BF16 ? 2 : 4;
  const int row_bytes = d * esz;
  const int rbp = (row_bytes + 15) / 16 * 16;
  unsigned char* ring = usm;
  int* pidx = reinterpret_cast<int*>(usm + (size_t)kUpdStages * kUpdRows * rbp);
  float* sq = reinterpret_cast<float*>(pidx + kUpdIdx * kUpdRows);
  const int cnt = P.counts[c], s0 = P.starts[c];
  const char* xb = reinterpret_cast<const char*>(P.x);
  const bool vec = (row_bytes % 16 == 0) && ((reinterpret_cast<uintptr_t>(P.x) & 15) == 0) &&
                   (row_bytes / 16 <= (int)blockDim.x);
  const int nchunks = (cnt + kUpdRows - 1) / kUpdRows;
  // gather layout: `tpr` threads per row, each one 16-byte piece
  const int tpr = vec ? row_bytes / 16 : 1;
  const int rpp = blockDim.x / tpr;  // rows per pass
  const int my_r = tid / tpr, my_part = tid - my_r * tpr;

  auto fetch_idx = [&](int chunk) -> int {  // issue (do not wait for) one member index
    const int m = chunk * kUpdRows + tid;
    return (chunk < nchunks && tid < kUpdRows && m < cnt) ? P.perm[s0 + m] : 0;
  };
  auto put_idx = [&](int chunk, int v) {
    if (tid < kUpdRows) pidx[(chunk % kUpdIdx) * kUpdRows + tid] = v;
  };
  auto issue_rows = [&](int chunk) {  // rows of `chunk` (indices already in smem)
    if (chunk < nchunks) {
      const int rows = min(kUpdRows, cnt - chunk * kUpdRows);
      unsigned char* dst = ring + (size_t)(chunk % kUpdStages) * kUpdRows * rbp;
      const int* idx = pidx + (chunk % kUpdIdx) * kUpdRows;
      if (vec) {
        for (int r = my_r; r < rows; r += rpp)
          cp_async16(dst + (size_t)r * rbp + my_part * 16,
                     xb + (int64_t)idx[r] * row_bytes + my_part * 16);
      } else {
        for (int e = tid; e < rows * d; e += blockDim.x) {
          const int r = e / d, t = e - r * d;
          const int64_t row = idx[r];
          if (esz == 2)
            reinterpret_cast<__nv_bfloat16*>(dst + (size_t)r * rbp)[t] =
                reinterpret_cast<const __nv_bfloat16*>(P.x)[row * d + t];
          else
            reinterpret_cast<float*>(dst + (size_t)r * rbp)[t] =
                reinterpret_cast<const float*>(P.x)[row * d + t];
        }
      }
    }
    cp_async_commit();  // (possibly empty group: keeps the group count uniform)
  };

  for (int ch = 0; ch < kUpdStages; ++ch) put_idx(ch, fetch_idx(ch));
  int pf0 = fetch_idx(kUpdStages);      // in flight: consumed at iteration 0
  int pf1 = fetch_idx(kUpdStages + 1);  // ... at iteration 1
  __syncthreads();
  for (int ch = 0; ch < kUpdStages - 1; ++ch) issue_rows(ch);

  double acc = 0.0;
  for (int j = 0; j < nchunks; ++j) {
    put_idx(j + kUpdStages, pf0);
    pf0 = pf1;
    pf1 = fetch_idx(j + kUpdStages + 2);
    issue_rows(j + kUpdStages - 1);
    cp_async_wait<kUpdStages - 1>();
    __syncthreads();
    if (tid < d) {
      // all loads of the chunk first, then the dependent f64 chain
      const int rows = min(kUpdRows, cnt - j * kUpdRows);
      const unsigned char* cur = ring + (size_t)(j % kUpdStages) * kUpdRows * rbp + (size_t)tid * esz;
      float v[kUpdRows];
#pragma unroll
      for (int r = 0; r < kUpdRows; ++r) {
        float f = 0.f;
        if (r < rows)
          f = (esz == 2) ? __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(cur + (size_t)r * rbp))
                         : *reinterpret_cast<const float*>(cur + (size_t)r * rbp);
        v[r] = f;
      }
      if (j == 0) acc = (double)v[0];  // np.add.reduceat: the first member initialises
#pragma unroll
      for (int r = 0; r < kUpdRows; ++r)
        if (r < rows && (j > 0 || r > 0)) acc = __dadd_rn(acc, (double)v[r]);
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  float* dst = (mode == 0) ? P.centers + (int64_t)c * d : outs[blockIdx.y] + (int64_t)c * d;
  if (tid < d) {
    const float nv = __double2float_rn(__ddiv_rn(acc, (double)cnt));
    if (mode == 0) {
      const float df = __fsub_rn(nv, dst[tid]);
      sq[tid] = __fmul_rn(df, df);
      sq[d + tid] = __fmul_rn(nv, nv);
    }
    dst[tid] = nv;
  }
  if (mode != 0) return;
  __syncthreads();
  if (tid == 0) {
    const float* a = sq;
    const float* b = sq + d;
    P.movement[c] = __fsqrt_rn(pw_sum<float>([&](int i) { return a[i]; }, d));
    P.cc[c] = pw_sum<float>([&](int i) { return b[i]; }, d);
    __threadfence();
    const int prev = atomicAdd(&P.status[AC_ST_DONE], 1);
    if (prev == k - 1) {
      __threadfence();
      const volatile float* mv = P.movement;
      const float s = pw_sum<float>([&](int i) { return mv[i]; }, k);
      const float mean = __double2float_rn(__ddiv_rn((double)s, (double)k));
      P.status[AC_ST_DONE] = 0;
      P.status[AC_ST_NITER] += 1;
      if ((double)mean < tol) P.status[AC_ST_ACTIVE] = 0;
    }
  }
}

// Warp-per-centre variant for d a multiple of 32 (the hot path: D = 64/128).
// Lane l owns dimensions [l*DPL, l*DPL + DPL) — DPL independent f64 chains —
// and walks the members in order.  Member rows are gathered by the warp
// itself into a private 3-stage shared-memory ring (cp.async, 32 rows per
// stage), so ~3 x 32 rows per centre are in flight while the current stage
// is added; hundreds of centres run concurrently and the kernel is bound by
// the gather bandwidth, not by the f64 add latency.
#ifndef AC_UPD_ROWS
#define AC_UPD_ROWS 16  // rows per ring stage (C4: 76.3 vs 77.9 ms with 32; C2/C3 neutral)
#endif
#ifndef AC_UPD_STAGES
#define AC_UPD_STAGES 3
#endif
constexpr int kUpdWRows = AC_UPD_ROWS;
constexpr int kUpdWStages = AC_UPD_STAGES;
#ifndef AC_UPD_WARPS
#define AC_UPD_WARPS 4
#endif
constexpr int kUpdWarps = AC_UPD_WARPS;  // centres per CTA

inline size_t update_w_smem(int d, int dtype) {
  const int esz = dtype == AC_DTYPE_BF16 ? 2 : 4;
  return (size_t)kUpdWarps * kUpdWStages * kUpdWRows * d * esz + (size_t)kUpdWarps * 2 * d * 4;
}

template <int DPL, bool BF16>
__global__ void __launch_bounds__(32 * kUpdWarps)
k_update_w(const ac_cluster_problem* __restrict__ probs, int d, double tol, int mode,
           float* const* outs) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char wsm[];
  const ac_cluster_problem& P = probs[blockIdx.y];
  if (mode == 0 && P.status[AC_ST_ACTIVE] == 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * kUpdWarps + warp;
  const int k = P.k;
  if (c >= k) return;
  constexpr int ESZ = BF16 ? 2 : 4;
  constexpr int row_bytes = 32 * DPL * ESZ;  // d == 32 * DPL (host dispatch)
  constexpr int stage_bytes = kUpdWRows * row_bytes;
  unsigned char* ring = wsm + (size_t)warp * kUpdWStages * stage_bytes;
  float* s_sq = reinterpret_cast<float*>(wsm + (size_t)kUpdWarps * kUpdWStages * stage_bytes) +
                warp * 2 * d;
  const int cnt = P.counts[c], s0 = P.starts[c];
  const int32_t* perm = P.perm + s0;
  const char* xb = reinterpret_cast<const char*>(P.x);
  constexpr int cpr = row_bytes / 16;    // 16-byte pieces per row
  const int nb = (cnt + kUpdWRows - 1) / kUpdWRows;

  // member indices are register-prefetched one stage ahead of their rows
  auto fetch = [&](int b) -> int {
    const int m = b * kUpdWRows + lane;
    return (b < nb && m < cnt) ? perm[m] : 0;
  };
  int nxt = fetch(0);
  auto issue = [&](int b) {
    const int myidx = nxt;
    nxt = fetch(b + 1);
    if (b < nb) {
      const int base = b * kUpdWRows;
      const int rows = min(kUpdWRows, cnt - base);
      // lane = (row `sub` of RPI rows, 16-byte piece `part`) per iteration
      constexpr int RPI = 32 / cpr;
      const int sub = lane / cpr, part = lane % cpr;
      unsigned char* dst = ring + (size_t)(b % kUpdWStages) * stage_bytes + sub * row_bytes + part * 16;
      const char* src = xb + part * 16;
#pragma unroll 4
      for (int it = 0; it < kUpdWRows / RPI; ++it) {
        const int r = it * RPI + sub;
        const int row = __shfl_sync(0xffffffffu, myidx, r);
        if (r < rows) cp_async16(dst + it * RPI * row_bytes, src + (int64_t)row * row_bytes);
      }
    }
    cp_async_commit();
  };

  double acc[DPL];
#pragma unroll
  for (int i = 0; i < DPL; ++i) acc[i] = 0.0;
  for (int b = 0; b < kUpdWStages - 1; ++b) issue(b);
  for (int b = 0; b < nb; ++b) {
    issue(b + kUpdWStages - 1);
    cp_async_wait<kUpdWStages - 1>();
    __syncwarp();
    const unsigned char* cur = ring + (size_t)(b % kUpdWStages) * stage_bytes + lane * DPL * ESZ;
    const int rows = min(kUpdWRows, cnt - b * kUpdWRows);
    // 8 rows at a time: loads of the next group overlap the f64 chain of this one
    auto load8 = [&](int r0, float (&v)[8][DPL]) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const unsigned char* rp = cur + (r0 + r) * row_bytes;
        if constexpr (BF16) {
          if constexpr (DPL == 2) {
            const uint32_t w = *reinterpret_cast<const uint32_t*>(rp);
            v[r][0] = __uint_as_float(w << 16); v[r][1] = __uint_as_float(w & 0xffff0000u);
          } else {
            const uint2 w = *reinterpret_cast<const uint2*>(rp);
            v[r][0] = __uint_as_float(w.x << 16); v[r][1] = __uint_as_float(w.x & 0xffff0000u);
            v[r][2] = __uint_as_float(w.y << 16); v[r][3] = __uint_as_float(w.y & 0xffff0000u);
          }
        } else {
          if constexpr (DPL == 2) {
            const float2 f = *reinterpret_cast<const float2*>(rp);
            v[r][0] = f.x; v[r][1] = f.y;
          } else {
            const float4 f = *reinterpret_cast<const float4*>(rp);
            v[r][0] = f.x; v[r][1] = f.y; v[r][2] = f.z; v[r][3] = f.w;
          }
        }
      }
    };
    if (rows == kUpdWRows && b > 0) {  // full stage: no per-row guards
#pragma unroll
      for (int r0 = 0; r0 < kUpdWRows; r0 += 8) {
        float v[8][DPL];
        load8(r0, v);
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int i = 0; i < DPL; ++i) acc[i] = __dadd_rn(acc[i], (double)v[r][i]);
      }
    } else {
      for (int r0 = 0; r0 < rows; r0 += 8) {
        float v[8][DPL];
        load8(r0, v);  // (rows past `rows` read stale ring bytes and are skipped)
#pragma unroll
        for (int r = 0; r < 8; ++r) {
          if (r0 + r >= rows) break;
          if (b == 0 && r0 + r == 0) {
#pragma unroll
            for (int i = 0; i < DPL; ++i) acc[i] = (double)v[r][i];  // first member initialises
            continue;
          }
#pragma unroll
          for (int i = 0; i < DPL; ++i) acc[i] = __dadd_rn(acc[i], (double)v[r][i]);
        }
      }
    }
    __syncwarp();  // the stage is refilled by the next issue
  }
  cp_async_wait<0>();
  float* dst = (mode == 0) ? P.centers + (int64_t)c * d : outs[blockIdx.y] + (int64_t)c * d;
#pragma unroll
  for (int i = 0; i < DPL; ++i) {
    const int t = lane * DPL + i;
    const float nv = __double2float_rn(__ddiv_rn(acc[i], (double)cnt));
    if (mode == 0) {
      const float df = __fsub_rn(nv, dst[t]);
      s_sq[t] = __fmul_rn(df, df);
      s_sq[d + t] = __fmul_rn(nv, nv);
    }
    dst[t] = nv;
  }
  if (mode != 0) return;
  __syncwarp();
  if (lane == 0) {
    const float* a = s_sq;
    const float* bq = s_sq + d;
    P.movement[c] = __fsqrt_rn(pw_sum<float>([&](int i) { return a[i]; }, d));
    P.cc[c] = pw_sum<float>([&](int i) { return bq[i]; }, d);
    __threadfence();
    const int prev = atomicAdd(&P.status[AC_ST_DONE], 1);
    if (prev == k - 1) {
      __threadfence();
      const volatile float* mv = P.movement;
      const float sm = pw_sum<float>([&](int i) { return mv[i]; }, k);
      const float mean = __double2float_rn(__ddiv_rn((double)sm, (double)k));
      P.status[AC_ST_DONE] = 0;
      P.status[AC_ST_NITER] += 1;
      if ((double)mean < tol) P.status[AC_ST_ACTIVE] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// K4, split-chain form (d = 64/128).  The reference sums each cluster's
// members in f64, in member order (np.add.reduceat), divides by the count
// and rounds to f32.  Any summation order of n values has error
// <= (n-1)·u·Σ|x| (u = 2^-53), so the reference's f64 sum s_ref and a sum Σ
// formed in ANY order satisfy |s_ref - Σ| <= 2n·u·Σ|x|; f32(fl64(s/n)) is
// monotone in s, so when both ends of that enclosure round to the same f32
// value it IS the reference's value, bit for bit.
//
//   k_usum   one warp per 128-member chunk of the member order (chunks may
//            straddle clusters): f64 Σx and f32 Σ|x| per (cluster, dim) in
//            registers, flushed with global reductions at cluster ends —
//            the long per-cluster chains are split over many warps;
//   k_ufin   one warp per centre: the enclosure test per dimension (and
//            re-zeroing of the workspaces); the rare dimension whose
//            enclosure straddles an f32 rounding boundary is recomputed with
//            the reference's own sequential chain; then movement / ||c||^2 /
//            convergence exactly as k_update.
// ---------------------------------------------------------------------------
constexpr int kUsChunk = 128;  // members per warp task
constexpr int kUsWarps = 8;
constexpr int kUsGroup = 8;    // member rows in flight per warp (16 measured slower)

// lane's DPL consecutive dimensions of row `row` (one vector load)
template <int DPL, bool BF16>
AC_DEV void load_row_part(const void* x, int64_t row, int d, int lane, float (&v)[DPL]) {
  if constexpr (BF16) {
    const __nv_bfloat16* p = reinterpret_cast<const __nv_bfloat16*>(x) + row * d + lane * DPL;
    if constexpr (DPL == 2) {
      const uint32_t w = *reinterpret_cast<const uint32_t*>(p);
      v[0] = __uint_as_float(w << 16); v[1] = __uint_as_float(w & 0xffff0000u);
    } else {
      const uint2 w = *reinterpret_cast<const uint2*>(p);
      v[0] = __uint_as_float(w.x << 16); v[1] = __uint_as_float(w.x & 0xffff0000u);
      v[2] = __uint_as_float(w.y << 16); v[3] = __uint_as_float(w.y & 0xffff0000u);
    }
  } else {
    const float* p = reinterpret_cast<const float*>(x) + row * d + lane * DPL;
    if constexpr (DPL == 2) {
      const float2 f = *reinterpret_cast<const float2*>(p);
      v[0] = f.x; v[1] = f.y;
    } else {
      const float4 f = *reinterpret_cast<const float4*>(p);
      v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
    }
  }
}

template <int DPL, bool BF16>
__global__ void __launch_bounds__(32 * kUsWarps)
k_usum(const ac_cluster_problem* __restrict__ probs, int d) {
  pdl_wait();
  pdl_trigger();
  const ac_cluster_problem& P = probs[blockIdx.y];
  if (P.status[AC_ST_ACTIVE] == 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = ((int64_t)blockIdx.x * kUsWarps + warp) * kUsChunk;
  const int64_t n = P.n;
  if (m0 >= n) return;
  const int m1 = (int)min((int64_t)kUsChunk, n - m0);  // members in this chunk
  const int k = P.k;
  // cluster of member m0: the last c with starts[c] <= m0
  int lo = 0, hi = k - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (P.starts[mid] <= m0) lo = mid; else hi = mid - 1;
  }
  int c = lo;
  int64_t c_end = P.starts[c + 1];
  double acc[DPL];
  float ab[DPL];
  float amin[DPL];  // smallest |x| (its exponent bounds every member's last bit)
#pragma unroll
  for (int i = 0; i < DPL; ++i) { acc[i] = 0.0; ab[i] = 0.f; amin[i] = INFINITY; }
  auto flush = [&]() {
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
      const int64_t e = (int64_t)c * d + lane * DPL + i;
      atomicAdd(P.csum + e, acc[i]);
      atomicAdd(P.cabs + e, ab[i]);
      atomicMin(P.clsb + e, __float_as_int(amin[i]));  // >= 0: int order == float order
      acc[i] = 0.0;
      ab[i] = 0.f;
      amin[i] = INFINITY;
    }
  };
  int pj_next = (lane < m1) ? P.perm[m0 + lane] : 0;
  for (int j = 0; j < m1; j += 32) {
    const int pj = pj_next;  // member indices of this 32-member group (prefetched)
    pj_next = (j + 32 + lane < m1) ? P.perm[m0 + j + 32 + lane] : 0;
    for (int g = 0; g < 32; g += kUsGroup) {
      if (j + g >= m1) break;
      float v[kUsGroup][DPL];
#pragma unroll
      for (int r = 0; r < kUsGroup; ++r) {
        const int row = __shfl_sync(0xffffffffu, pj, g + r);
        if (j + g + r < m1) load_row_part<DPL, BF16>(P.x, row, d, lane, v[r]);
      }
#pragma unroll
      for (int r = 0; r < kUsGroup; ++r) {
        const int64_t m = m0 + j + g + r;
        if (j + g + r >= m1) break;
        while (m >= c_end) {  // cluster boundary (warp-uniform)
          flush();
          ++c;
          c_end = P.starts[c + 1];
        }
#pragma unroll
        for (int i = 0; i < DPL; ++i) {
          acc[i] = __dadd_rn(acc[i], (double)v[r][i]);
          ab[i] = __fadd_rn(ab[i], fabsf(v[r][i]));
          amin[i] = fminf(amin[i], fabsf(v[r][i]));
        }
      }
    }
  }
  flush();
}

template <int DPL, bool BF16>
__global__ void __launch_bounds__(128)
k_ufin(const ac_cluster_problem* __restrict__ probs, int d, double tol) {
  pdl_wait();
  pdl_trigger();
  __shared__ float s_sq[4][2][256];
  const ac_cluster_problem& P = probs[blockIdx.y];
  if (P.status[AC_ST_ACTIVE] == 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * 4 + warp;
  const int k = P.k;
  if (c >= k) return;
  const int cnt = P.counts[c], s0 = P.starts[c];
  const double dn = (double)cnt;
  float nvs[DPL];
  uint32_t fail = 0;
#pragma unroll
  for (int i = 0; i < DPL; ++i) {
    const int64_t e = (int64_t)c * d + lane * DPL + i;
    const double sum = P.csum[e];
    const double sab = (double)P.cabs[e] * (1.0 + dn * 0x1p-23);
    const float amin = __int_as_float(P.clsb[e]);
    P.csum[e] = 0.0;
    P.cabs[e] = 0.f;
    P.clsb[e] = 0x7f800000;  // +inf
    // (a) every member is a multiple of 2^q (q = exponent of the smallest
    //     |x| minus 23: an f32 has 24 significant bits) and Σ|x| < 2^(53+q):
    //     no partial sum of ANY order rounds, so Σ is exactly the
    //     reference's sum;
    // (b) otherwise the order-free enclosure must land on one f32 value
    if (amin > 0.f && sab < ldexp(1.0, 53 + ilogbf(amin) - 23)) {
      nvs[i] = __double2float_rn(__ddiv_rn(sum, dn));
    } else {
      const double err = 2.02 * dn * 0x1p-53 * sab + 1e-300;
      const float lo = __double2float_rn(__ddiv_rn(__dsub_rd(sum, err), dn));
      const float hi = __double2float_rn(__ddiv_rn(__dadd_ru(sum, err), dn));
      nvs[i] = lo;
      if (!(lo == hi)) fail |= 1u << i;
    }
  }
  // rare: the enclosure straddles an f32 rounding boundary -> the reference's
  // own sequential f64 chain over the members (first member initialises)
  unsigned lanes = __ballot_sync(0xffffffffu, fail != 0);
  {  // statistic: fallback chains, counted in status[AC_ST_FLAGS] bits 8..
    const int nf = __reduce_add_sync(0xffffffffu, __popc(fail));
    if (lane == 0 && nf) atomicAdd(&P.status[AC_ST_FLAGS], nf << 8);
  }
  while (lanes) {
    const int src = __ffs(lanes) - 1;
    lanes &= lanes - 1;
    const uint32_t f = __shfl_sync(0xffffffffu, fail, src);
    for (int i = 0; i < DPL; ++i) {
      if (!(f & (1u << i))) continue;
      const int t = src * DPL + i;
      // 128 members per round in flight, then the ordered chain
      double acc = 0.0;
      for (int base = 0; base < cnt; base += 128) {
        float v[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int m = base + 32 * q + lane;
          v[q] = (m < cnt) ? ld_elem(P.x, BF16 ? AC_DTYPE_BF16 : AC_DTYPE_F32,
                                     (int64_t)P.perm[s0 + m] * d + t)
                           : 0.f;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int nr = min(32, cnt - base - 32 * q);
          for (int r = 0; r < nr; ++r) {
            const double vv = (double)__shfl_sync(0xffffffffu, v[q], r);
            acc = (base == 0 && q == 0 && r == 0) ? vv : __dadd_rn(acc, vv);
          }
        }
      }
      const float nv = __double2float_rn(__ddiv_rn(acc, dn));
      if (lane == src) nvs[i] = nv;
    }
  }
  float* dst = P.centers + (int64_t)c * d;
#pragma unroll
  for (int i = 0; i < DPL; ++i) {
    const int t = lane * DPL + i;
    const float nv = nvs[i];
    const float df = __fsub_rn(nv, dst[t]);
    s_sq[warp][0][t] = __fmul_rn(df, df);
    s_sq[warp][1][t] = __fmul_rn(nv, nv);
    dst[t] = nv;
  }
  __syncwarp();
  if (lane == 0) {
    const float* a = s_sq[warp][0];
    const float* bq = s_sq[warp][1];
    P.movement[c] = __fsqrt_rn(pw_sum<float>([&](int i) { return a[i]; }, d));
    P.cc[c] = pw_sum<float>([&](int i) { return bq[i]; }, d);
    __threadfence();
    const int prev = atomicAdd(&P.status[AC_ST_DONE], 1);
    if (prev == k - 1) {
      __threadfence();
      const volatile float* mv = P.movement;
      const float sm = pw_sum<float>([&](int i) { return mv[i]; }, k);
      const float mean = __double2float_rn(__ddiv_rn((double)sm, (double)k));
      P.status[AC_ST_DONE] = 0;
      P.status[AC_ST_NITER] += 1;
      if ((double)mean < tol) P.status[AC_ST_ACTIVE] = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// K4, streaming form of the split-chain sums (d = 64/128).  The enclosure
// test in k_ufin holds for ANY summation order, so the global member order
// (a gather through perm whose longest cluster walk bounds the member-order
// kernel) is not needed to form Σx and the bounds.  Each CTA owns a
// contiguous range of at most kUsmChunk rows, counting-sorts the range by
// label in shared memory (order inside a label is irrelevant), and its warps
// take equal contiguous slices of that local order: f64 sums in registers
// (lane = DPL consecutive dimensions), two batches of kUsmBatch rows in
// flight (each row one coalesced 256/512-byte read from the CTA's range),
// flushed into csum/cabs/clsb with global reductions at label boundaries.
// The bounds are per lane rather than per dimension: Σ_rows max_i|x_i| over
// the lane's DPL dimensions bounds Σ|x_t| of each of them and
// min_rows min_i|x_i| bounds min|x_t| from below, so k_ufin's enclosure
// stays valid (a few times wider; it still decides virtually every
// dimension) and k_ufin finishes exactly as after k_usum.
// ---------------------------------------------------------------------------
constexpr int kUsmWarps = 8;
constexpr int kUsmBatch = 8;     // rows per batch (two batches in flight per warp)
constexpr int kUsmMaxK = 1024;   // labels a CTA can sort in shared memory
constexpr int kUsmChunk = 4096;  // rows per CTA at most (12-bit row, 10-bit label packing)
static int kUsmCtasPerSm = getenv("AC_USM_CTAS") ? atoi(getenv("AC_USM_CTAS")) : 4;

template <int DPL, bool BF16>
__global__ void __launch_bounds__(32 * kUsmWarps)
k_ustream(const ac_cluster_problem* __restrict__ probs, int d, int64_t chunk) {
  pdl_wait();
  pdl_trigger();
  __shared__ int s_pos[kUsmMaxK];
  __shared__ int s_sorted[kUsmChunk];  // label << 12 | row
  const ac_cluster_problem& P = probs[blockIdx.y];
  if (P.status[AC_ST_ACTIVE] == 0) return;
  const int64_t n = P.n;
  const int64_t r0 = (int64_t)blockIdx.x * chunk;
  if (r0 >= n) return;
  const int r1 = (int)min(n - r0, chunk);  // rows of this CTA: [r0, r0 + r1)
  const int k = P.k;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int32_t* labels = P.labels + r0;
  // counting sort of the range by label
  for (int c = tid; c < k; c += blockDim.x) s_pos[c] = 0;
  __syncthreads();
  for (int r = tid; r < r1; r += blockDim.x) atomicAdd(&s_pos[labels[r]], 1);
  __syncthreads();
  if (warp == 0) {  // exclusive scan of the counts
    int run = 0;
    for (int c0 = 0; c0 < k; c0 += 32) {
      const int c = c0 + lane;
      const int v = c < k ? s_pos[c] : 0;
      int inc = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      if (c < k) s_pos[c] = run + inc - v;
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
  __syncthreads();
  for (int r = tid; r < r1; r += blockDim.x) {
    const int l = labels[r];
    s_sorted[atomicAdd(&s_pos[l], 1)] = (l << 12) | r;
  }
  __syncthreads();
  // this warp's slice of the local order
  const int per = (r1 + kUsmWarps - 1) / kUsmWarps;
  const int p0 = warp * per, p1 = min(r1, p0 + per);
  if (p0 >= p1) return;
  const char* xb = reinterpret_cast<const char*>(P.x) + r0 * (int64_t)d * (BF16 ? 2 : 4);
  double acc[DPL];
#pragma unroll
  for (int i = 0; i < DPL; ++i) acc[i] = 0.0;
  float ab = 0.f, mn = INFINITY;
  int cur = s_sorted[p0] >> 12;
  auto flush = [&]() {
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
      const int64_t g = (int64_t)cur * d + lane * DPL + i;
      atomicAdd(P.csum + g, acc[i]);
      atomicAdd(P.cabs + g, ab);
      atomicMin(P.clsb + g, __float_as_int(mn));  // >= 0: int order == float order
      acc[i] = 0.0;
    }
    ab = 0.f;
    mn = INFINITY;
  };
  float va[kUsmBatch][DPL], vb[kUsmBatch][DPL];
  auto load = [&](int q0, float (&v)[kUsmBatch][DPL]) {
#pragma unroll
    for (int r = 0; r < kUsmBatch; ++r)
      if (q0 + r < p1) load_row_part<DPL, BF16>(xb, s_sorted[q0 + r] & 0xfff, d, lane, v[r]);
  };
  auto consume = [&](int q0, float (&v)[kUsmBatch][DPL]) {
#pragma unroll
    for (int r = 0; r < kUsmBatch; ++r) {
      if (q0 + r >= p1) break;
      const int l = s_sorted[q0 + r] >> 12;
      if (l != cur) { flush(); cur = l; }
      float mx = 0.f, mi = INFINITY;
#pragma unroll
      for (int i = 0; i < DPL; ++i) {
        acc[i] = __dadd_rn(acc[i], (double)v[r][i]);
        mx = fmaxf(mx, fabsf(v[r][i]));
        mi = fminf(mi, fabsf(v[r][i]));
      }
      ab = __fadd_rn(ab, mx);
      mn = fminf(mn, mi);
    }
  };
  load(p0, va);
  for (int q = p0; q < p1; q += 2 * kUsmBatch) {
    load(q + kUsmBatch, vb);
    consume(q, va);
    load(q + 2 * kUsmBatch, va);
    consume(q + kUsmBatch, vb);
  }
  flush();
}

// ---------------------------------------------------------------------------
// K2: k-means++ seeding (clustering.py:78-91)
// ---------------------------------------------------------------------------
__global__ void k_kpp_init(const ac_cluster_problem* __restrict__ probs, int dtype, int d,
                           const double* __restrict__ draws, int max_k) {
  const ac_cluster_problem& P = probs[blockIdx.x];
  const int64_t first = (int64_t)draws[(int64_t)blockIdx.x * max_k];
  for (int t = threadIdx.x; t < d; t += blockDim.x)
    P.centers[t] = ld_elem(P.x, dtype, first * d + t);
}

// closest = min(closest, ((x - centers[s]) ** 2).sum(axis=1))  (s == 0: assign)
__global__ void k_kpp_dist(const ac_cluster_problem* __restrict__ probs, int dtype, int d,
                           int s) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) float ksm[];
  const ac_cluster_problem& P = probs[blockIdx.y];
  if (s + 1 >= P.k || P.status[AC_ST_KPP_STOP] >= 0) return;
  for (int t = threadIdx.x; t < d; t += blockDim.x) ksm[t] = P.centers[(int64_t)s * d + t];
  __syncthreads();
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= P.n) return;
  const int64_t base = r * d;
  auto get = [&](int i) {
    const float df = __fsub_rn(ld_elem(P.x, dtype, base + i), ksm[i]);
    return __fmul_rn(df, df);
  };
  const float dist = pw_sum<float>(get, d);
  P.best[r] = (s == 0) ? dist : np_minimum(P.best[r], dist);
}

// D = 64 / 128 form of k_kpp_dist: 8 lanes per row, lane j runs numpy's
// pairwise accumulator r_j = sum_m (x[j+8m] - c[j+8m])^2 in order and
// pw8_combine folds the 8 (same operations as pw_sum, same bits); each load
// instruction of a warp touches 4 rows x 8 consecutive elements.
//
// Rows whose minimum cannot change are not read: labels[r] holds the centre
// a whose distance is best[r] (scratch during seeding) and movement[a] =
// ||c_s - c_a|| rounded down (written by k_kpp_pick).  By the triangle
// inequality ||x - c_s|| >= ||c_s - c_a|| - ||x - c_a||, so when
// ||c_s - c_a|| >= 2(1 + 1e-3) sqrt(best) the new distance exceeds best by a
// factor ~1.004 -- far beyond the ~1e-5 relative rounding of either f32
// distance -- and np.minimum keeps best, bit for bit.  ~80 % of the rows
// of a C2/C3 head are skipped this way (keys and queries alike).  A warp
// tests 32 consecutive rows (coalesced best/labels, the distance table in
// shared memory), then computes the surviving rows four at a time.
constexpr int kKppTab = 4096;
template <int D>
__global__ void __launch_bounds__(256)
k_kpp_dist_v(const ac_cluster_problem* __restrict__ probs, int dtype, int s) {
  pdl_wait();
  pdl_trigger();
  __shared__ float s_tab[kKppTab];
  const ac_cluster_problem& P = probs[blockIdx.y];
  if (s + 1 >= P.k || P.status[AC_ST_KPP_STOP] >= 0) return;
  const bool prune = s > 0 && P.labels && P.movement;
  const bool tab_smem = prune && s <= kKppTab;
  if (tab_smem)
    for (int t = threadIdx.x; t < s; t += blockDim.x) s_tab[t] = P.movement[t];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t r0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32;
  if (r0 >= P.n) return;
  const int64_t r = r0 + lane;
  const bool ok = r < P.n;
  float b = 0.f;
  bool need = ok;
  if (ok && s > 0) {
    b = P.best[r];
    if (prune) {
      const int a = P.labels[r];
      const float dc = tab_smem ? s_tab[a] : P.movement[a];
      if ((b == 0.f && !isnan(dc)) || (b >= 1e-30f && dc >= 2.002f * __fsqrt_rn(b))) need = false;
    }
  }
  unsigned mask = __ballot_sync(0xffffffffu, need);
  const int j = lane & 7, g = lane >> 3;
  const float* c = P.centers + (int64_t)s * D;
  float cv[D / 8];
#pragma unroll
  for (int m = 0; m < D / 8; ++m) cv[m] = c[j + 8 * m];
  while (mask) {
    // rows of this round: the first four surviving rows, one per 8-lane group
    const unsigned pos = __fns(mask, 0, g + 1);
    const bool have = pos < 32u;
    const int sel = have ? (int)pos : 0;
    for (int q = 0; q < 4 && mask; ++q) mask &= mask - 1;
    const float bs = __shfl_sync(0xffffffffu, b, sel);
    const int64_t rs = r0 + sel;
    float xv[D / 8];
    if (!have) {
#pragma unroll
      for (int m = 0; m < D / 8; ++m) xv[m] = 0.f;
    } else if (dtype == AC_DTYPE_BF16) {
      const __nv_bfloat16* x = reinterpret_cast<const __nv_bfloat16*>(P.x) + rs * D;
#pragma unroll
      for (int m = 0; m < D / 8; ++m) xv[m] = __bfloat162float(x[j + 8 * m]);
    } else {
      const float* x = reinterpret_cast<const float*>(P.x) + rs * D;
#pragma unroll
      for (int m = 0; m < D / 8; ++m) xv[m] = __ldg(x + j + 8 * m);
    }
    float acc = 0.f;
#pragma unroll
    for (int m = 0; m < D / 8; ++m) {
      const float df = __fsub_rn(xv[m], cv[m]);
      acc = m == 0 ? __fmul_rn(df, df) : __fadd_rn(acc, __fmul_rn(df, df));
    }
    const float dist = pw8_combine(acc);
    if (have && j == 0) {
      if (s == 0) {
        P.best[rs] = dist;
        if (P.labels) P.labels[rs] = 0;
      } else {
        P.best[rs] = np_minimum(bs, dist);
        if (prune && dist < bs) P.labels[rs] = s;
      }
    }
  }
}

// total = closest.sum(); p = closest / total; choice(n, p): f64 cumsum,
// /= cdf[-1], searchsorted(u, 'right').  One CTA of 1024 threads per problem.
//
// When every non-zero p >= 2^-29 (the normal case), every p is a multiple of
// 2^-52 below 1 and every partial sum a multiple of 2^-52 below 2: numpy's
// sequential f64 cumsum is then exact, and equals p * 2^52 summed as int64 in
// any order.  The search runs in two passes over coalesced 32-element rows:
//   1. warp w owns a contiguous chunk of rows; each lane sums its column of
//      the chunk (int64 adds, loads batched 8 rows deep), one warp reduction
//      per chunk; warp 0 scans the 32 chunk sums and picks the first chunk
//      whose cdf passes u;
//   2. that chunk's row sums (all warps), a warp scan over them picks the
//      row, and one warp scan of the row picks the element.
// Otherwise (tiny non-zero p) thread 0 replays the sequential f64 cumsum.
AC_DEV long long warp_incl_scan_i64(long long v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long w = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += w;
  }
  return v;
}
AC_DEV long long warp_sum_i64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
AC_DEV long long p_fixed52(float p) {
  return __double2ll_rn(__dmul_rn((double)p, 4503599627370496.0));  // p * 2^52 (exact)
}
constexpr double kTwoM52 = 2.220446049250313e-16;  // 2^-52

__global__ void __launch_bounds__(1024)
k_kpp_pick(const ac_cluster_problem* __restrict__ probs, int dtype, int d, int s,
           const double* __restrict__ draws, int max_k, int64_t rows_off) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ __align__(16) unsigned char kpsm[];
  const ac_cluster_problem& P = probs[blockIdx.x];
  if (s + 1 >= P.k || P.status[AC_ST_KPP_STOP] >= 0) return;
  const int64_t n = P.n;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nw = (int)(blockDim.x >> 5);
  const float* closest = P.best;
  PwPlan plan{P.plan_n};
  const float total =
      pw_eval_block_g8<float>(plan, [&](int i) { return closest[i]; }, reinterpret_cast<float*>(kpsm));
  const double draw = draws[(int64_t)blockIdx.x * max_k + s + 1];
  __shared__ long long s_idx;
  __shared__ int s_inexact, s_chunk;
  __shared__ long long s_csum[32];  // chunk sums -> inclusive chunk prefixes
  long long* rsum = reinterpret_cast<long long*>(kpsm + rows_off);  // rows of the chosen chunk
  if (!(total > 0.f)) {
    // `if total <= 0: idx = int(rng.integers(n))` — forced draw or stop
    if (tid == 0) {
      if (draw < 0) s_idx = (long long)(-draw) - 1;
      else { s_idx = -1; P.status[AC_ST_KPP_STOP] = s + 1; }
    }
    __syncthreads();
  } else {
    const int64_t R = (n + 31) / 32;
    const int64_t C = (R + nw - 1) / nw;  // rows per chunk
    auto pval = [&](float c, int& inexact) -> long long {
      const float p = __fdiv_rn(c, total);
      if (p != 0.f && p < 1.8626451e-09f) inexact = 1;  // 2^-29
      return p_fixed52(p);
    };
    if (tid == 0) { s_inexact = 0; s_chunk = -1; }
    __syncthreads();
    // pass 1: chunk sums
    int inexact = 0;
    {
      const int64_t r0 = (int64_t)warp * C, r1 = min(R, r0 + C);
      long long acc = 0;
      for (int64_t rb = r0; rb < r1; rb += 8) {
        float cl[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int64_t jj = (rb + q) * 32 + lane;
          cl[q] = (rb + q < r1 && jj < n) ? closest[jj] : 0.f;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) acc += pval(cl[q], inexact);
      }
      acc = warp_sum_i64(acc);
      if (lane == 0) s_csum[warp] = acc;
    }
    if (__any_sync(0xffffffffu, inexact) && lane == 0) s_inexact = 1;
    __syncthreads();
    if (!s_inexact) {
      if (warp == 0) {
        const long long inc = warp_incl_scan_i64(lane < nw ? s_csum[lane] : 0);
        const double last = (double)__shfl_sync(0xffffffffu, inc, nw - 1) * kTwoM52;  // cdf[-1]
        const unsigned hit = __ballot_sync(0xffffffffu, lane < nw && __ddiv_rn((double)inc * kTwoM52, last) > draw);
        if (lane == 0) s_chunk = hit ? __ffs(hit) - 1 : -1;
        s_csum[lane] = inc;
      }
      __syncthreads();
      const int f = s_chunk;
      const double last = (double)s_csum[nw - 1] * kTwoM52;
      if (f >= 0) {
        // pass 2: row sums of chunk f
        const int64_t r0 = (int64_t)f * C, r1 = min(R, r0 + C);
        for (int64_t r = r0 + warp; r < r1; r += nw) {
          const int64_t jj = r * 32 + lane;
          long long v = jj < n ? pval(closest[jj], inexact) : 0;
          v = warp_sum_i64(v);
          if (lane == 0) rsum[r - r0] = v;
        }
        __syncthreads();
        if (warp == 0) {
          long long carry = f > 0 ? s_csum[f - 1] : 0;
          long long idx = -1, base = 0;
          for (int64_t b = r0; b < r1 && idx < 0; b += 32) {
            const long long v = (b + lane < r1) ? rsum[b + lane - r0] : 0;
            const long long inc = warp_incl_scan_i64(v);
            const unsigned hit = __ballot_sync(
                0xffffffffu, b + lane < r1 && __ddiv_rn((double)(carry + inc) * kTwoM52, last) > draw);
            if (hit) {
              const int l = __ffs(hit) - 1;
              idx = b + l;  // the row
              base = carry + __shfl_sync(0xffffffffu, inc - v, l);  // exclusive prefix of the row
            }
            carry += __shfl_sync(0xffffffffu, inc, 31);
          }
          if (idx >= 0) {
            const int64_t jj = idx * 32 + lane;
            const long long v = jj < n ? pval(closest[jj], inexact) : 0;
            const long long runj = base + warp_incl_scan_i64(v);
            const unsigned hit =
                __ballot_sync(0xffffffffu, jj < n && __ddiv_rn((double)runj * kTwoM52, last) > draw);
            if (lane == 0) s_idx = hit ? idx * 32 + __ffs(hit) - 1 : n;
          } else if (lane == 0) {
            s_idx = n;
          }
        }
      } else if (tid == 0) {
        s_idx = n;  // u beyond the cdf (cannot happen)
      }
      __syncthreads();
    } else {
      if (tid == 0) {  // sequential replay of numpy's cumsum
        double run = 0.0;
        for (int64_t j2 = 0; j2 < n; ++j2) run = __dadd_rn(run, (double)__fdiv_rn(closest[j2], total));
        const double lastv = run;
        run = 0.0;
        long long idx = n;
        for (int64_t j2 = 0; j2 < n; ++j2) {
          run = __dadd_rn(run, (double)__fdiv_rn(closest[j2], total));
          if (__ddiv_rn(run, lastv) > draw) { idx = j2; break; }
        }
        s_idx = idx;
        P.status[AC_ST_FLAGS] |= 1;  // sequential cumsum fallback used
      }
      __syncthreads();
    }
  }
  const long long idx = s_idx;
  if (idx < 0) return;
  const int64_t ci = min((long long)n - 1, idx);
  for (int t = tid; t < d; t += blockDim.x)
    P.centers[(int64_t)(s + 1) * d + t] = ld_elem(P.x, dtype, ci * d + t);
  // ||c_{s+1} - c_j|| for j <= s, f64, rounded down to f32: the skip test of
  // k_kpp_dist_v at step s + 1 (one warp per centre)
  if (P.movement && P.labels) {
    for (int jc = warp; jc <= s; jc += nw) {
      double acc = 0.0;
      for (int t = lane; t < d; t += 32) {
        const double df = (double)ld_elem(P.x, dtype, ci * d + t) - (double)P.centers[(int64_t)jc * d + t];
        acc = fma(df, df, acc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) P.movement[jc] = __double2float_rd(sqrt(acc));
    }
  }
}

// ---------------------------------------------------------------------------
// multi-stage helpers
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024)
k_reduce_best(const ac_cluster_problem* __restrict__ probs, float* sum_out, float* mean_out) {
  extern __shared__ __align__(16) unsigned char rsm[];
  const ac_cluster_problem& P = probs[blockIdx.x];
  const float* best = P.best;
  PwPlan plan{P.plan_n};
  const float s = pw_eval_block_g8<float>(plan, [&](int i) { return best[i]; },
                                       reinterpret_cast<float*>(rsm));
  if (threadIdx.x == 0) {
    if (sum_out) sum_out[blockIdx.x] = s;
    if (mean_out) mean_out[blockIdx.x] = __double2float_rn(__ddiv_rn((double)s, (double)P.n));
  }
}

// per-row f64 distance to the assigned centre; sqrt_it: norm (tau) or squared (mse)
__global__ void k_row_dist_f64(const ac_cluster_problem* __restrict__ probs, int dtype, int d,
                               int sqrt_it) {
  const ac_cluster_problem& P = probs[blockIdx.y];
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= P.n) return;
  const int64_t base = r * d;
  const float* crow = P.centers + (int64_t)P.labels[r] * d;
  auto get = [&](int i) {
    const double df = __dsub_rn((double)ld_elem(P.x, dtype, base + i), (double)crow[i]);
    return __dmul_rn(df, df);
  };
  const double s = pw_sum<double>(get, d);
  P.dscratch[r] = sqrt_it ? __dsqrt_rn(s) : s;
}

__global__ void __launch_bounds__(1024)
k_reduce_dscratch(const ac_cluster_problem* __restrict__ probs, double factor, double* out) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const ac_cluster_problem& P = probs[blockIdx.x];
  const double* v = P.dscratch;
  PwPlan plan{P.plan_n};
  const double s = pw_eval_block_g8<double>(plan, [&](int i) { return v[i]; },
                                         reinterpret_cast<double*>(dsm));
  if (threadIdx.x == 0) out[blockIdx.x] = __dmul_rn(factor, __ddiv_rn(s, (double)P.n));
}

// retire distances: keep[i] = ||x_i - c[label_i]|| (f32) >= tau32
__global__ void k_retire_flags(const ac_cluster_problem* __restrict__ probs, int dtype, int d,
                               const float* __restrict__ tau32) {
  const ac_cluster_problem& P = probs[blockIdx.y];
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= P.n) return;
  const int64_t base = r * d;
  const float* crow = P.centers + (int64_t)P.labels[r] * d;
  auto get = [&](int i) {
    const float df = __fsub_rn(ld_elem(P.x, dtype, base + i), crow[i]);
    return __fmul_rn(df, df);
  };
  const float dist = __fsqrt_rn(pw_sum<float>(get, d));
  reinterpret_cast<uint8_t*>(P.dscratch)[r] = (dist >= tau32[blockIdx.y]) ? 1 : 0;
}

// order-preserving compaction of idx_in by the keep flags; one CTA per problem
__global__ void __launch_bounds__(1024)
k_retire_compact(const ac_cluster_problem* __restrict__ probs, const int64_t* const* idx_in,
                 int64_t* const* idx_out, int64_t* out_count) {
  const ac_cluster_problem& P = probs[blockIdx.x];
  const int64_t n = P.n;
  const uint8_t* keep = reinterpret_cast<const uint8_t*>(P.dscratch);
  const int tid = threadIdx.x;
  const int64_t seg = (n + blockDim.x - 1) / blockDim.x;
  const int64_t lo = min(n, (int64_t)tid * seg), hi = min(n, lo + seg);
  __shared__ long long s_sc[1024];
  long long local = 0;
  for (int64_t i = lo; i < hi; ++i) local += keep[i];
  s_sc[tid] = local;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {
    const long long v = (tid >= off) ? s_sc[tid - off] : 0;
    __syncthreads();
    s_sc[tid] += v;
    __syncthreads();
  }
  long long pos = s_sc[tid] - local;
  const int64_t* in = idx_in[blockIdx.x];
  int64_t* out = idx_out[blockIdx.x];
  for (int64_t i = lo; i < hi; ++i)
    if (keep[i]) out[pos++] = in[i];
  if (tid == blockDim.x - 1) out_count[blockIdx.x] = s_sc[tid];
}

__global__ void k_gather_rows(const void* __restrict__ src, int dtype, int d,
                              const int64_t* __restrict__ idx, int64_t rows,
                              void* __restrict__ dst) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= rows * d) return;
  const int64_t r = e / d, t = e - r * d;
  const int64_t s = idx[r] * d + t;
  if (dtype == AC_DTYPE_BF16)
    reinterpret_cast<__nv_bfloat16*>(dst)[e] = reinterpret_cast<const __nv_bfloat16*>(src)[s];
  else
    reinterpret_cast<float*>(dst)[e] = reinterpret_cast<const float*>(src)[s];
}

// drop centres without members (clustering.py:303-310).  One CTA per problem.
__global__ void __launch_bounds__(1024)
k_drop_empty(const ac_cluster_problem* __restrict__ probs, int d, int32_t* new_k) {
  const ac_cluster_problem& P = probs[blockIdx.x];
  const int k = P.k;
  const int64_t n = P.n;
  const int tid = threadIdx.x;
  for (int c = tid; c < k; c += blockDim.x) P.counts[c] = 0;
  __syncthreads();
  for (int64_t i = tid; i < n; i += blockDim.x) atomicAdd(&P.counts[P.labels[i]], 1);
  __syncthreads();
  // remap: serial prefix over k (k <= a few thousand) by thread 0 into starts[]
  int32_t* remap = P.starts;
  if (tid == 0) {
    int j = 0;
    for (int c = 0; c < k; ++c) remap[c] = (P.counts[c] > 0) ? j++ : -1;
    new_k[blockIdx.x] = j;
  }
  __syncthreads();
  // compact centres and counts in increasing order (remap[c] <= c, so row c is
  // read before any later write can touch it)
  for (int c = 0; c < k; ++c) {
    const int j = remap[c];
    if (j >= 0 && j != c) {
      for (int t = tid; t < d; t += blockDim.x)
        P.centers[(int64_t)j * d + t] = P.centers[(int64_t)c * d + t];
    }
    __syncthreads();
  }
  if (tid == 0) {
    for (int c = 0; c < k; ++c) {
      const int j = remap[c];
      if (j >= 0) P.counts[j] = P.counts[c];
    }
  }
  __syncthreads();
  for (int64_t i = tid; i < n; i += blockDim.x) P.labels[i] = remap[P.labels[i]];
}

// ---------------------------------------------------------------------------
// K9: envelopes (quest.py:61-71) — sequential np.maximum/np.minimum over the
// members in label order, one warp per cluster.
// ---------------------------------------------------------------------------
__global__ void k_envelopes(const ac_cluster_problem* __restrict__ probs, int dtype, int d,
                            float* const* env_max, float* const* env_min) {
  const ac_cluster_problem& P = probs[blockIdx.y];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = blockIdx.x * (blockDim.x >> 5) + warp;
  if (c >= P.k) return;
  const int cnt = P.counts[c], s0 = P.starts[c];
  float* mx = env_max[blockIdx.y] + (int64_t)c * d;
  float* mn = env_min[blockIdx.y] + (int64_t)c * d;
  for (int t0 = 0; t0 < d; t0 += 32) {
    const int t = t0 + lane;
    if (t >= d) break;
    float a = 0.f, b = 0.f;
    for (int m = 0; m < cnt; ++m) {
      const float v = ld_elem(P.x, dtype, (int64_t)P.perm[s0 + m] * d + t);
      if (m == 0) { a = v; b = v; }
      else { a = np_maximum(a, v); b = np_minimum(b, v); }
    }
    mx[t] = a;
    mn[t] = b;
  }
}

// D = 32*DPL fast path: one CTA per cluster, its 8 warps scanning 8
// contiguous chunks of the member list (lane = DPL dimensions, 8 member rows
// in flight), then the chunk results combined in chunk order.  The sequential
// fold keeps the first maximal element (ties such as +0/-0 keep the earlier
// one, the first NaN wins); folding chunk results in order with the same
// np.maximum / np.minimum gives exactly the same element.
constexpr int kEnvWarps = 8;

template <int DPL, bool BF16>
__global__ void __launch_bounds__(32 * kEnvWarps)
k_envelopes_w(const ac_cluster_problem* __restrict__ probs, float* const* env_max,
              float* const* env_min) {
  constexpr int D = 32 * DPL;
  __shared__ float s_mx[kEnvWarps][D], s_mn[kEnvWarps][D];
  __shared__ int s_has[kEnvWarps];
  const ac_cluster_problem& P = probs[blockIdx.y];
  const int c = blockIdx.x;
  if (c >= P.k) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cnt = P.counts[c], s0 = P.starts[c];
  const int per = (cnt + kEnvWarps - 1) / kEnvWarps;
  const int m0 = min(cnt, warp * per), m1 = min(cnt, m0 + per);
  const int32_t* perm = P.perm + s0;
  float a[DPL], b[DPL];
  auto load_row = [&](int32_t row, float (&v)[DPL]) {
    if constexpr (BF16) {
      const __nv_bfloat16* xr = reinterpret_cast<const __nv_bfloat16*>(P.x) + (int64_t)row * D + lane * DPL;
      if constexpr (DPL == 2) {
        const uint32_t w = __ldg(reinterpret_cast<const uint32_t*>(xr));
        v[0] = __uint_as_float(w << 16); v[1] = __uint_as_float(w & 0xffff0000u);
      } else {
        const uint2 w = __ldg(reinterpret_cast<const uint2*>(xr));
        v[0] = __uint_as_float(w.x << 16); v[1] = __uint_as_float(w.x & 0xffff0000u);
        v[2] = __uint_as_float(w.y << 16); v[3] = __uint_as_float(w.y & 0xffff0000u);
      }
    } else {
      const float* xr = reinterpret_cast<const float*>(P.x) + (int64_t)row * D + lane * DPL;
      if constexpr (DPL == 2) {
        const float2 f = __ldg(reinterpret_cast<const float2*>(xr));
        v[0] = f.x; v[1] = f.y;
      } else {
        const float4 f = __ldg(reinterpret_cast<const float4*>(xr));
        v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
      }
    }
  };
  if (m0 < m1) {
    float v[DPL];
    load_row(perm[m0], v);
#pragma unroll
    for (int i = 0; i < DPL; ++i) { a[i] = v[i]; b[i] = v[i]; }
    int m = m0 + 1;
    for (; m + 8 <= m1; m += 8) {
      int32_t rows[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) rows[u] = perm[m + u];
      float w[8][DPL];
#pragma unroll
      for (int u = 0; u < 8; ++u) load_row(rows[u], w[u]);
#pragma unroll
      for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int i = 0; i < DPL; ++i) { a[i] = np_maximum(a[i], w[u][i]); b[i] = np_minimum(b[i], w[u][i]); }
    }
    for (; m < m1; ++m) {
      load_row(perm[m], v);
#pragma unroll
      for (int i = 0; i < DPL; ++i) { a[i] = np_maximum(a[i], v[i]); b[i] = np_minimum(b[i], v[i]); }
    }
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
      s_mx[warp][lane * DPL + i] = a[i];
      s_mn[warp][lane * DPL + i] = b[i];
    }
  }
  if (lane == 0) s_has[warp] = m0 < m1;
  __syncthreads();
  float* mx = env_max[blockIdx.y] + (int64_t)c * D;
  float* mn = env_min[blockIdx.y] + (int64_t)c * D;
  for (int t = threadIdx.x; t < D; t += blockDim.x) {
    float x = 0.f, y = 0.f;  // empty cluster: zeros, as the sequential kernel
    bool any = false;
    for (int w = 0; w < kEnvWarps; ++w) {
      if (!s_has[w]) continue;
      if (!any) { x = s_mx[w][t]; y = s_mn[w][t]; any = true; }
      else { x = np_maximum(x, s_mx[w][t]); y = np_minimum(y, s_mn[w][t]); }
    }
    mx[t] = x;
    mn[t] = y;
  }
}

}  // namespace ac

// ===========================================================================
// host side
// ===========================================================================
using namespace ac;

namespace ac_host {
bool assign_tc_eligible(const ac_cluster_problem* host_probs, int nprob, int dtype, int d,
                        int c_lo, int order, int c_hi = INT_MAX);
int assign_tc_launch(const ac_cluster_problem* probs, const ac_cluster_problem* host_probs,
                     int nprob, int dtype, int d, int c_lo, int flags, cudaStream_t st,
                     int c_hi = INT_MAX);
}  // namespace ac_host

namespace {
// kernel-selection modes are per calling thread (a process may drive several
// GPUs or serve concurrent callers from several threads)
thread_local int g_assign_mode = AC_ASSIGN_MODE_AUTO;
// 0: split-chain update when eligible, 1: member-order chains (default)
thread_local int g_update_mode =
    getenv("AC_UPDATE_MODE") ? atoi(getenv("AC_UPDATE_MODE")) : AC_UPDATE_MODE_AUTO;
inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int set_smem(const void* fn, size_t bytes) {
  if (bytes > 48 * 1024) return ac_host::func_smem(fn, (int)bytes, "cudaFuncSetAttribute");
  return AC_OK;
}
size_t plan_vals_bytes(int64_t n, size_t elem) {
  // for n > 128 every leaf holds >= 57 elements (n2 >= n/2 - 7 >= 57), so
  // leaves <= n/56 + 1; internal nodes = leaves - 1
  const int64_t L = n <= 128 ? 1 : n / 56 + 2;
  return (size_t)(2 * L + 2) * elem;
}
}  // namespace

extern "C" int ac_row_sqnorm(const void* x, int dtype, int64_t rows, int d, float* out,
                             void* stream) {
  if (rows < 0 || d < 1) { ac_host::set_error("ac_row_sqnorm: bad shape"); return AC_ERR_DIM; }
  if (rows == 0) return AC_OK;
  const size_t smem = sizeof(float) * kNormRows * (d + 1);
  int rc = set_smem((const void*)k_row_sqnorm, smem);
  if (rc) return rc;
  k_row_sqnorm<<<(unsigned)((rows + kNormRows - 1) / kNormRows), kNormRows, smem, S(stream)>>>(
      x, dtype, rows, d, out);
  AC_CHECK_LAUNCH("k_row_sqnorm");
  return AC_OK;
}

static bool rows_v_ok(const void* x, int dtype, int d) {
  return (d == 64 || d == 128) && (dtype == AC_DTYPE_F32 || dtype == AC_DTYPE_BF16) &&
         !(reinterpret_cast<uintptr_t>(x) & 15);
}

static size_t rows_v_smem(int d) { return sizeof(float) * kRowsV * (d + 8); }

extern "C" int ac_l2norm_ex(const void* x, int dtype, int64_t rows, int d, float* out,
                            float* out_sq, uint8_t* degenerate, void* planes, int64_t prob_rows,
                            void* stream) {
  if (rows < 0 || d < 1) { ac_host::set_error("ac_l2norm: bad shape"); return AC_ERR_DIM; }
  if (rows == 0) return AC_OK;
  const bool fast = rows_v_ok(x, dtype, d) && !(reinterpret_cast<uintptr_t>(out) & 15) &&
                    !(reinterpret_cast<uintptr_t>(planes) & 15);
  if (planes && (!fast || prob_rows <= 0 || rows % prob_rows)) {
    ac_host::set_error("ac_l2norm_ex: planes need d=64/128, aligned rows and rows %% prob_rows == 0");
    return AC_ERR_PARAM;
  }
  if (fast) {
    const size_t smem = rows_v_smem(d);
    const void* fn = d == 64 ? (const void*)k_l2norm_v<64> : (const void*)k_l2norm_v<128>;
    int rc = set_smem(fn, smem);
    if (rc) return rc;
    const unsigned grid = (unsigned)((rows + kRowsV - 1) / kRowsV);
    __nv_bfloat16* pl = reinterpret_cast<__nv_bfloat16*>(planes);
    if (d == 64)
      k_l2norm_v<64><<<grid, 256, smem, S(stream)>>>(x, dtype, rows, out, out_sq, degenerate, pl, prob_rows);
    else
      k_l2norm_v<128><<<grid, 256, smem, S(stream)>>>(x, dtype, rows, out, out_sq, degenerate, pl, prob_rows);
    AC_CHECK_LAUNCH("k_l2norm_v");
    return AC_OK;
  }
  const size_t smem = sizeof(float) * kNormRows * (d + 1);
  int rc = set_smem((const void*)k_l2norm, smem);
  if (rc) return rc;
  k_l2norm<<<(unsigned)((rows + kNormRows - 1) / kNormRows), kNormRows, smem, S(stream)>>>(
      x, dtype, rows, d, out, out_sq, degenerate);
  AC_CHECK_LAUNCH("k_l2norm");
  return AC_OK;
}

extern "C" int ac_l2norm(const void* x, int dtype, int64_t rows, int d, float* out,
                         float* out_sq, uint8_t* degenerate, void* stream) {
  return ac_l2norm_ex(x, dtype, rows, d, out, out_sq, degenerate, nullptr, 0, stream);
}

static int prepare_impl(const ac_cluster_problem* probs, int nprob, int dtype, int d, int64_t max_n,
                        int max_k, bool rows_done, void* stream) {
  if (nprob <= 0) return AC_OK;
  const bool rows_fast = (d == 64 || d == 128) && (dtype == AC_DTYPE_F32 || dtype == AC_DTYPE_BF16);
  k_status_init<<<(nprob + 127) / 128, 128, 0, S(stream)>>>(probs, nprob);
  if (rows_done) {
    // ||x||^2 (and the f32 planes) are current: written by ac_l2norm_ex
  } else if (rows_fast) {
    const size_t xsm = rows_v_smem(d);
    const void* fn = d == 64 ? (const void*)k_problem_xx_v<64> : (const void*)k_problem_xx_v<128>;
    int rc = set_smem(fn, xsm);
    if (rc) return rc;
    const dim3 grid((unsigned)((max_n + kRowsV - 1) / kRowsV), nprob);
    if (d == 64) k_problem_xx_v<64><<<grid, 256, xsm, S(stream)>>>(probs, dtype);
    else k_problem_xx_v<128><<<grid, 256, xsm, S(stream)>>>(probs, dtype);
  } else {
    const size_t xsm = sizeof(float) * kNormRows * (d + 1);
    int rc = set_smem((const void*)k_problem_xx, xsm);
    if (rc) return rc;
    k_problem_xx<<<dim3((unsigned)((max_n + kNormRows - 1) / kNormRows), nprob), kNormRows, xsm,
                   S(stream)>>>(probs, dtype, d);
  }
  k_center_sqnorm<<<dim3((max_k + 127) / 128, nprob), 128, 0, S(stream)>>>(probs, d, 0);
  AC_CHECK_LAUNCH("ac_lloyd_prepare");
  return AC_OK;
}

extern "C" int ac_lloyd_prepare(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                                int64_t max_n, int max_k, void* stream) {
  return prepare_impl(probs, nprob, dtype, d, max_n, max_k, false, stream);
}

// `generic` is decided per batch by the host (every problem of a batch shares
// one accumulation order; the host splits batches otherwise).
// internal assign flag: ||c||^2 is already current (inside a Lloyd run the
// centroid update writes it), skip k_center_sqnorm
constexpr int kAssignCcValid = 1 << 8;

static int assign_impl(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                       int64_t max_n, int max_k, int c_lo, int flags, int order,
                       const ac_cluster_problem* host_probs, cudaStream_t st) {
  const bool cc_valid = flags & kAssignCcValid;
  flags &= ~kAssignCcValid;
  const unsigned tiles = (unsigned)((max_n + kAsgBM - 1) / kAsgBM);
  const int mode = g_assign_mode;
  const bool tc_ok = ac_host::assign_tc_eligible(host_probs, nprob, dtype, d, c_lo, order);
  // more than 128 centres: tensor-core passes over 128-centre chunks
  bool chunk_ok = !tc_ok && mode != AC_ASSIGN_MODE_EXACT && c_lo == 0 &&
                  !(flags & AC_ASSIGN_MERGE) && max_k <= 4096 &&
                  ac_host::assign_tc_eligible(host_probs, nprob, dtype, d, 0, order, ac::kAsgTcChunk);
  for (int c0 = ac::kAsgTcChunk; c0 < max_k && chunk_ok; c0 += ac::kAsgTcChunk) {
    bool reached = false;  // a chunk no problem reaches is fine
    for (int p = 0; p < nprob; ++p) reached |= host_probs[p].k > c0;
    chunk_ok = !reached ||
               ac_host::assign_tc_eligible(host_probs, nprob, dtype, d, c0, order, c0 + ac::kAsgTcChunk);
  }
  if (mode == AC_ASSIGN_MODE_TC && !tc_ok && !chunk_ok) {
    ac_host::set_error("assign: tensor-core path forced but the batch is not eligible "
                       "(needs D=64/128, general order, k-c_lo<=128, host descriptors)");
    return AC_ERR_PARAM;
  }
  if (tc_ok && mode != AC_ASSIGN_MODE_EXACT) {
    if (!cc_valid) ac_host::launch_pdl(k_center_sqnorm, dim3(dim3((max_k + 127) / 128, nprob)), dim3(128), 0, st, probs, d, c_lo);
    AC_CHECK_LAUNCH("k_center_sqnorm");
    return ac_host::assign_tc_launch(probs, host_probs, nprob, dtype, d, c_lo, flags, st);
  }
  // the first chunk with exact distances, the rest merged with strict '<'
  // (earlier chunks win ties: the first-index argmin over the whole set),
  // then the tile histograms of the final labels
  {
    const bool ok = chunk_ok;
    if (ok) {
      if (!cc_valid) ac_host::launch_pdl(k_center_sqnorm, dim3(dim3((max_k + 127) / 128, nprob)), dim3(128), 0, st, probs, d, 0);
      AC_CHECK_LAUNCH("k_center_sqnorm");
      const int base = (flags & ~AC_ASSIGN_LABELS_ONLY) | ac::kAsgNoHist;
      for (int c0 = 0; c0 < max_k; c0 += ac::kAsgTcChunk) {
        bool any = false;
        for (int p = 0; p < nprob; ++p) any |= host_probs[p].k > c0;
        if (!any) break;
        const int rc = ac_host::assign_tc_launch(probs, host_probs, nprob, dtype, d, c0,
                                                 base | (c0 ? AC_ASSIGN_MERGE : 0), st,
                                                 c0 + ac::kAsgTcChunk);
        if (rc) return rc;
      }
      const size_t hsm = sizeof(int) * (size_t)(max_k + 4);
      int rc = set_smem((const void*)k_tile_hist, hsm);
      if (rc) return rc;
      ac_host::launch_pdl(k_tile_hist, dim3(dim3(tiles, nprob)), dim3(kAsgBM), hsm, st, probs, max_k);
      AC_CHECK_LAUNCH("k_tile_hist");
      return AC_OK;
    }
  }
  if (order == AC_ORDER_SEQ) {
    const size_t smem = assign_smem_bytes(d, max_k);
    int rc = set_smem((const void*)k_assign_seq, smem);
    if (rc) return rc;
    if (!cc_valid) ac_host::launch_pdl(k_center_sqnorm, dim3(dim3((max_k + 127) / 128, nprob)), dim3(128), 0, st, probs, d, c_lo);
    k_assign_seq<<<dim3(tiles, nprob), 256, smem, st>>>(probs, dtype, d, c_lo, flags, max_k);
  } else {
    const size_t smem = sizeof(int) * (size_t)(max_k + 4);
    int rc = set_smem((const void*)k_assign_generic, smem);
    if (rc) return rc;
    if (!cc_valid) ac_host::launch_pdl(k_center_sqnorm, dim3(dim3((max_k + 127) / 128, nprob)), dim3(128), 0, st, probs, d, c_lo);
    k_assign_generic<<<dim3(tiles, nprob), kAsgBM, smem, st>>>(probs, dtype, d, c_lo, flags, max_k);
  }
  AC_CHECK_LAUNCH("ac_assign");
  return AC_OK;
}

extern "C" int ac_assign_ordered(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                                 int64_t max_n, int max_k, int c_lo, int flags, int order,
                                 const ac_cluster_problem* host_probs, void* stream) {
  if (nprob <= 0 || max_n <= 0) return AC_OK;
  if (d < 1 || d > 256) { ac_host::set_error("assign: d=%d unsupported (1..256)", d); return AC_ERR_DIM; }
  return assign_impl(probs, nprob, dtype, d, max_n, max_k, c_lo, flags, order, host_probs,
                     S(stream));
}

extern "C" int ac_assign(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                         int64_t max_n, int max_k, int c_lo, int flags, void* stream) {
  return ac_assign_ordered(probs, nprob, dtype, d, max_n, max_k, c_lo, flags, AC_ORDER_SEQ,
                           nullptr, stream);
}

extern "C" int ac_set_assign_mode(int mode) {
  if (mode < AC_ASSIGN_MODE_AUTO || mode > AC_ASSIGN_MODE_TC) {
    ac_host::set_error("ac_set_assign_mode: bad mode %d", mode);
    return AC_ERR_PARAM;
  }
  g_assign_mode = mode;
  return AC_OK;
}
extern "C" int ac_get_assign_mode(void) { return g_assign_mode; }
extern "C" int ac_set_update_mode(int mode) {
  if (mode < AC_UPDATE_MODE_SPLIT || mode > AC_UPDATE_MODE_AUTO) {
    ac_host::set_error("ac_set_update_mode: bad mode %d", mode);
    return AC_ERR_PARAM;
  }
  g_update_mode = mode;
  return AC_OK;
}

extern "C" int ac_get_update_mode(void) { return g_update_mode; }

static int repair_sort_impl(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                            int64_t max_n, int max_k, int iter, int flags, cudaStream_t st) {
  const unsigned tiles = (unsigned)((max_n + kAsgBM - 1) / kAsgBM);
  ac_host::launch_pdl(k_hist_scan, dim3(dim3((max_k + 7) / 8, nprob)), dim3(256), 0, st, probs, flags);
  const size_t psm = plan_vals_bytes(max_n, sizeof(float));
  int rc = set_smem((const void*)k_post, psm);
  if (rc) return rc;
  ac_host::launch_pdl(k_post, dim3(nprob), dim3(1024), psm, st, probs, dtype, d, iter, flags);
  ac_host::launch_pdl(k_scatter, dim3(dim3(tiles, nprob)), dim3(kAsgBM), 0, st, probs, flags);
  AC_CHECK_LAUNCH("ac_repair_sort");
  return AC_OK;
}

extern "C" int ac_repair_sort(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                              int64_t max_n, int max_k, int iter, int flags, void* stream) {
  if (nprob <= 0 || max_n <= 0) return AC_OK;
  return repair_sort_impl(probs, nprob, dtype, d, max_n, max_k, iter, flags, S(stream));
}

// split-chain update (k_usum + k_ufin) for a Lloyd iteration
static int usum_update_impl(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                            int64_t max_n, int max_k, double tol, int mode, cudaStream_t st) {
  const bool bf = dtype == AC_DTYPE_BF16;
  const dim3 g2((unsigned)((max_k + 3) / 4), nprob);
  if (mode == AC_UPDATE_MODE_STREAM && max_k <= kUsmMaxK) {
    // one wave of kUsmCtasPerSm CTAs per SM over all problems, each a
    // contiguous multiple of 256 rows
    const int64_t ctas = (int64_t)ac_host::sm_count() * kUsmCtasPerSm;
    int64_t chunk = (max_n * nprob + ctas - 1) / ctas;
    chunk = min((int64_t)kUsmChunk, (chunk + 255) / 256 * 256);
    const dim3 g1((unsigned)((max_n + chunk - 1) / chunk), nprob);
    const size_t ssm = 0;
    const int nt = 32 * kUsmWarps;
    if (d == 64) {
      if (bf) { ac_host::launch_pdl(k_ustream<2, true>, dim3(g1), dim3(nt), ssm, st, probs, d, chunk); ac_host::launch_pdl(k_ufin<2, true>, dim3(g2), dim3(128), 0, st, probs, d, tol); }
      else { ac_host::launch_pdl(k_ustream<2, false>, dim3(g1), dim3(nt), ssm, st, probs, d, chunk); ac_host::launch_pdl(k_ufin<2, false>, dim3(g2), dim3(128), 0, st, probs, d, tol); }
    } else {
      if (bf) { ac_host::launch_pdl(k_ustream<4, true>, dim3(g1), dim3(nt), ssm, st, probs, d, chunk); ac_host::launch_pdl(k_ufin<4, true>, dim3(g2), dim3(128), 0, st, probs, d, tol); }
      else { ac_host::launch_pdl(k_ustream<4, false>, dim3(g1), dim3(nt), ssm, st, probs, d, chunk); ac_host::launch_pdl(k_ufin<4, false>, dim3(g2), dim3(128), 0, st, probs, d, tol); }
    }
    AC_CHECK_LAUNCH("k_ustream/k_ufin");
    return AC_OK;
  }
  const dim3 g1((unsigned)((max_n + kUsChunk * kUsWarps - 1) / (kUsChunk * kUsWarps)), nprob);
  if (d == 64) {
    if (bf) { ac_host::launch_pdl(k_usum<2, true>, dim3(g1), dim3(32 * kUsWarps), 0, st, probs, d); ac_host::launch_pdl(k_ufin<2, true>, dim3(g2), dim3(128), 0, st, probs, d, tol); }
    else { ac_host::launch_pdl(k_usum<2, false>, dim3(g1), dim3(32 * kUsWarps), 0, st, probs, d); ac_host::launch_pdl(k_ufin<2, false>, dim3(g2), dim3(128), 0, st, probs, d, tol); }
  } else {
    if (bf) { ac_host::launch_pdl(k_usum<4, true>, dim3(g1), dim3(32 * kUsWarps), 0, st, probs, d); ac_host::launch_pdl(k_ufin<4, true>, dim3(g2), dim3(128), 0, st, probs, d, tol); }
    else { ac_host::launch_pdl(k_usum<4, false>, dim3(g1), dim3(32 * kUsWarps), 0, st, probs, d); ac_host::launch_pdl(k_ufin<4, false>, dim3(g2), dim3(128), 0, st, probs, d, tol); }
  }
  AC_CHECK_LAUNCH("k_usum/k_ufin");
  return AC_OK;
}

static bool usum_ws(const ac_cluster_problem* host_probs, int nprob, int d) {
  if (!host_probs || !(d == 64 || d == 128)) return false;
  for (int p = 0; p < nprob; ++p)
    if (!host_probs[p].csum || !host_probs[p].cabs || !host_probs[p].clsb) return false;
  return true;
}

// Mode 0 (split chains): used for f32 points, whose 256/512-byte rows make
// the gather efficient and the member-order chains the longest; bf16 points
// (128-byte rows) measured faster with the member-order kernel.
static bool usum_ok(const ac_cluster_problem* host_probs, int nprob, int dtype, int d) {
  if (g_update_mode != AC_UPDATE_MODE_SPLIT || !host_probs || !(d == 64 || d == 128)) return false;
  static const int bf_ok = getenv("AC_USUM_BF16") ? atoi(getenv("AC_USUM_BF16")) : 0;
  if (dtype != AC_DTYPE_F32 && !(dtype == AC_DTYPE_BF16 && bf_ok)) return false;
  for (int p = 0; p < nprob; ++p)
    if (!host_probs[p].csum || !host_probs[p].cabs || !host_probs[p].clsb) return false;
  return true;
}

// Update kernel of a Lloyd run.  The member-order kernel runs one warp per
// centre on ceil(k / kUpdWarps) CTAs per problem: in a batch with few centres
// in total and long clusters (the multi-stage planner's rounds: one to a few
// heads, m_t = 8..100 centres over thousands of rows) most SMs idle while
// single warps walk clusters of thousands of members, so such batches take
// the streamed sums, which spread the rows over every SM (one "mixed" C3
// head's planner: 133 ms of member-order updates over 925 launches).  Short
// clusters (C1: 4,096 rows over 65 centres, warm step 1.07 vs 1.15 ms) and
// larger batches keep the member-order kernel.
static int update_mode_for(const ac_cluster_problem* host_probs, int nprob, int dtype, int d,
                           int64_t max_n, int max_k) {
  static const int small = getenv("AC_USM_SMALL") ? atoi(getenv("AC_USM_SMALL")) : 512;
  static const int per_centre = getenv("AC_USM_ROWS") ? atoi(getenv("AC_USM_ROWS")) : 128;
  const int mode = g_update_mode;
  if (mode == AC_UPDATE_MODE_MEMBER) return mode;
  if (mode == AC_UPDATE_MODE_AUTO) {
    if ((int64_t)nprob * max_k < small && max_n >= (int64_t)per_centre * max_k &&
        max_k <= kUsmMaxK && usum_ws(host_probs, nprob, d))
      return AC_UPDATE_MODE_STREAM;
    return AC_UPDATE_MODE_MEMBER;
  }
  if (mode == AC_UPDATE_MODE_STREAM && max_k <= kUsmMaxK && usum_ws(host_probs, nprob, d))
    return mode;
  return usum_ok(host_probs, nprob, dtype, d) ? AC_UPDATE_MODE_SPLIT : AC_UPDATE_MODE_MEMBER;
}


static int update_impl(const ac_cluster_problem* probs, int nprob, int dtype, int d, int max_k,
                       double tol, int mode, float* const* outs, cudaStream_t st) {
  if (d > 256) { ac_host::set_error("update: d=%d > 256", d); return AC_ERR_DIM; }
  if (d % 32 == 0 && (d == 64 || d == 128)) {
    const dim3 grid((unsigned)((max_k + kUpdWarps - 1) / kUpdWarps), nprob);
    const bool bf = dtype == AC_DTYPE_BF16;
    const size_t wsmem = update_w_smem(d, dtype);
    const void* fn = d == 64 ? (bf ? (const void*)k_update_w<2, true> : (const void*)k_update_w<2, false>)
                             : (bf ? (const void*)k_update_w<4, true> : (const void*)k_update_w<4, false>);
    int rc = set_smem(fn, wsmem);
    if (rc) return rc;
    if (d == 64) {
      if (bf) ac_host::launch_pdl(k_update_w<2, true>, dim3(grid), dim3(32 * kUpdWarps), wsmem, st, probs, d, tol, mode, outs);
      else ac_host::launch_pdl(k_update_w<2, false>, dim3(grid), dim3(32 * kUpdWarps), wsmem, st, probs, d, tol, mode, outs);
    } else {
      if (bf) ac_host::launch_pdl(k_update_w<4, true>, dim3(grid), dim3(32 * kUpdWarps), wsmem, st, probs, d, tol, mode, outs);
      else ac_host::launch_pdl(k_update_w<4, false>, dim3(grid), dim3(32 * kUpdWarps), wsmem, st, probs, d, tol, mode, outs);
    }
    AC_CHECK_LAUNCH("k_update_w");
    return AC_OK;
  }
  const size_t smem = update_smem_bytes(d, dtype);
  int rc = set_smem((const void*)k_update, smem);
  if (rc) return rc;
  ac_host::launch_pdl(k_update, dim3(dim3(max_k, nprob)), dim3(d <= 128 ? 128 : 256), smem, st, probs, dtype, d, tol, mode, outs);
  AC_CHECK_LAUNCH("k_update");
  return AC_OK;
}

extern "C" int ac_segment_mean(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                               int max_k, float* const* out, void* stream) {
  if (nprob <= 0) return AC_OK;
  return update_impl(probs, nprob, dtype, d, max_k, 0.0, 1, out, S(stream));
}

static int lloyd_impl(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                      int64_t max_n, int max_k, int max_iter, double tol, int poll_every,
                      int lflags, const ac_cluster_problem* host_probs, void* stream) {
  if (nprob <= 0) return AC_OK;
  if (d < 1 || d > 256) { ac_host::set_error("lloyd: d=%d unsupported (1..256)", d); return AC_ERR_DIM; }
  if (max_k > 16384) { ac_host::set_error("lloyd: k=%d too large", max_k); return AC_ERR_PARAM; }
  cudaStream_t st = S(stream);
  // every problem of a batch must share the accumulation order
  int order = AC_ORDER_SEQ;
  if (host_probs) order = host_probs[0].order;
  const bool inertia = !(lflags & AC_LLOYD_NO_INERTIA);
  // without inertia_history nothing but the (rare) empty-cluster repair reads
  // `best`: the tensor-core assign may then skip the exact chain of rows with
  // a single candidate, and the repair recomputes exact distances if needed
  const int lo_flag = (!inertia && g_assign_mode != AC_ASSIGN_MODE_EXACT &&
                       ac_host::assign_tc_eligible(host_probs, nprob, dtype, d, 0, order))
                          ? AC_ASSIGN_LABELS_ONLY : 0;
  const int umode = update_mode_for(host_probs, nprob, dtype, d, max_n, max_k);
  int rc = prepare_impl(probs, nprob, dtype, d, max_n, max_k, (lflags & AC_LLOYD_PREPARED) != 0,
                        stream);
  if (rc) return rc;
  // host copy of the active flags for polling (kept across calls: a
  // cudaMallocHost per call costs more than the iterations it saves)
  thread_local int32_t* t_pinned = nullptr;
  thread_local int t_pinned_n = 0;
  int32_t* pinned = nullptr;
  if (poll_every > 0 && host_probs) {
    if (t_pinned_n < nprob) {
      if (t_pinned) cudaFreeHost(t_pinned);
      t_pinned = nullptr;
      t_pinned_n = 0;
      if (cudaMallocHost(&t_pinned, sizeof(int32_t) * nprob) == cudaSuccess) t_pinned_n = nprob;
    }
    pinned = t_pinned;
  }
  for (int it = 0; it < max_iter; ++it) {
    // ||c||^2 is current: prepare wrote it, then every centroid update does
    if ((rc = assign_impl(probs, nprob, dtype, d, max_n, max_k, 0, kAssignCcValid | lo_flag, order,
                          host_probs, st)))
      break;
    if ((rc = repair_sort_impl(probs, nprob, dtype, d, max_n, max_k, inertia ? it : -1, lo_flag, st)))
      break;
    if (umode != AC_UPDATE_MODE_MEMBER)
      rc = usum_update_impl(probs, nprob, dtype, d, max_n, max_k, tol, umode, st);
    else rc = update_impl(probs, nprob, dtype, d, max_k, tol, 0, nullptr, st);
    if (rc) break;
    if (pinned && (it + 1) % poll_every == 0 && it + 1 < max_iter) {
      for (int p = 0; p < nprob; ++p)
        cudaMemcpyAsync(pinned + p, host_probs[p].status + AC_ST_ACTIVE, sizeof(int32_t),
                        cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      int any = 0;
      for (int p = 0; p < nprob; ++p) any |= pinned[p];
      if (!any) break;
    }
  }
  if (rc) return rc;
  if ((rc = assign_impl(probs, nprob, dtype, d, max_n, max_k, 0,
                        AC_ASSIGN_ALL | kAssignCcValid | lo_flag, order, host_probs, st)))
    return rc;
  return repair_sort_impl(probs, nprob, dtype, d, max_n, max_k, -1, AC_ASSIGN_ALL | lo_flag, st);
}

extern "C" int ac_lloyd(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                        int64_t max_n, int max_k, int max_iter, double tol, int poll_every,
                        const ac_cluster_problem* host_probs, void* stream) {
  return lloyd_impl(probs, nprob, dtype, d, max_n, max_k, max_iter, tol, poll_every, 0, host_probs,
                    stream);
}

extern "C" int ac_lloyd_ex(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                           int64_t max_n, int max_k, int max_iter, double tol, int flags,
                           const ac_cluster_problem* host_probs, void* stream) {
  return lloyd_impl(probs, nprob, dtype, d, max_n, max_k, max_iter, tol, 0, flags, host_probs,
                    stream);
}

extern "C" int ac_kmeanspp(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                           int64_t max_n, int max_k, const double* draws, void* stream) {
  if (nprob <= 0) return AC_OK;
  cudaStream_t st = S(stream);
  k_status_init<<<(nprob + 127) / 128, 128, 0, st>>>(probs, nprob);
  k_kpp_init<<<nprob, 128, 0, st>>>(probs, dtype, d, draws, max_k);
  // pairwise-tree values, then one int64 per 32-element row of one chunk
  // (a 32nd of the rows)
  const int64_t rows_off = (int64_t)((plan_vals_bytes(max_n, sizeof(float)) + 15) & ~size_t(15));
  const int64_t chunk_rows = ((max_n + 31) / 32 + 31) / 32;
  const size_t psm = (size_t)(rows_off + chunk_rows * 8);
  if (psm > 200 * 1024) {
    ac_host::set_error("ac_kmeanspp: n=%lld too large", (long long)max_n);
    return AC_ERR_PARAM;
  }
  // (static shared memory included: the attribute is needed below 48 KB too)
  int rc = ac_host::func_smem((const void*)k_kpp_pick, (int)psm, "k_kpp_pick smem");
  if (rc) return rc;
  const bool rows_fast = (d == 64 || d == 128) && (dtype == AC_DTYPE_F32 || dtype == AC_DTYPE_BF16);
  for (int s = 0; s + 1 < max_k; ++s) {
    if (rows_fast) {
      const dim3 grid((unsigned)((max_n + 255) / 256), nprob);
      if (d == 64) ac_host::launch_pdl(k_kpp_dist_v<64>, grid, dim3(256), 0, st, probs, dtype, s);
      else ac_host::launch_pdl(k_kpp_dist_v<128>, grid, dim3(256), 0, st, probs, dtype, s);
    } else {
      ac_host::launch_pdl(k_kpp_dist, dim3((unsigned)((max_n + 255) / 256), nprob), dim3(256),
                          sizeof(float) * d, st, probs, dtype, d, s);
    }
    ac_host::launch_pdl(k_kpp_pick, dim3(nprob), dim3(1024), psm, st, probs, dtype, d, s, draws,
                        max_k, rows_off);
  }
  AC_CHECK_LAUNCH("ac_kmeanspp");
  return AC_OK;
}

extern "C" int ac_reduce_best(const ac_cluster_problem* probs, int nprob, int64_t max_n,
                              float* sum_out, float* mean_out, void* stream) {
  if (nprob <= 0) return AC_OK;
  const size_t psm = plan_vals_bytes(max_n, sizeof(float));
  int rc = set_smem((const void*)k_reduce_best, psm);
  if (rc) return rc;
  k_reduce_best<<<nprob, 1024, psm, S(stream)>>>(probs, sum_out, mean_out);
  AC_CHECK_LAUNCH("k_reduce_best");
  return AC_OK;
}

extern "C" int ac_tau(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                      int64_t max_n, double factor, double* tau_out, void* stream) {
  if (nprob <= 0) return AC_OK;
  cudaStream_t st = S(stream);
  k_row_dist_f64<<<dim3((unsigned)((max_n + 255) / 256), nprob), 256, 0, st>>>(probs, dtype, d, 1);
  const size_t psm = plan_vals_bytes(max_n, sizeof(double));
  int rc = set_smem((const void*)k_reduce_dscratch, psm);
  if (rc) return rc;
  k_reduce_dscratch<<<nprob, 1024, psm, st>>>(probs, factor, tau_out);
  AC_CHECK_LAUNCH("ac_tau");
  return AC_OK;
}

extern "C" int ac_mse_f64(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                          int64_t max_n, double* out, void* stream) {
  if (nprob <= 0) return AC_OK;
  cudaStream_t st = S(stream);
  k_row_dist_f64<<<dim3((unsigned)((max_n + 255) / 256), nprob), 256, 0, st>>>(probs, dtype, d, 0);
  const size_t psm = plan_vals_bytes(max_n, sizeof(double));
  int rc = set_smem((const void*)k_reduce_dscratch, psm);
  if (rc) return rc;
  k_reduce_dscratch<<<nprob, 1024, psm, st>>>(probs, 1.0, out);
  AC_CHECK_LAUNCH("ac_mse_f64");
  return AC_OK;
}

extern "C" int ac_retire(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                         int64_t max_n, const float* tau32, const int64_t* const* idx_in,
                         int64_t* const* idx_out, int64_t* out_count, void* stream) {
  if (nprob <= 0) return AC_OK;
  cudaStream_t st = S(stream);
  k_retire_flags<<<dim3((unsigned)((max_n + 255) / 256), nprob), 256, 0, st>>>(probs, dtype, d, tau32);
  k_retire_compact<<<nprob, 1024, 0, st>>>(probs, idx_in, idx_out, out_count);
  AC_CHECK_LAUNCH("ac_retire");
  return AC_OK;
}

extern "C" int ac_gather_rows(const void* src, int dtype, int d, const int64_t* idx,
                              int64_t rows, void* dst, void* stream) {
  if (rows <= 0) return AC_OK;
  const int64_t total = rows * d;
  k_gather_rows<<<(unsigned)((total + 255) / 256), 256, 0, S(stream)>>>(src, dtype, d, idx, rows, dst);
  AC_CHECK_LAUNCH("k_gather_rows");
  return AC_OK;
}

extern "C" int ac_drop_empty(const ac_cluster_problem* probs, int nprob, int d, int64_t max_n,
                             int max_k, int32_t* new_k, void* stream) {
  if (nprob <= 0) return AC_OK;
  k_drop_empty<<<nprob, 1024, 0, S(stream)>>>(probs, d, new_k);
  AC_CHECK_LAUNCH("k_drop_empty");
  return AC_OK;
}

extern "C" int ac_envelopes(const ac_cluster_problem* probs, int nprob, int dtype, int d,
                            int max_k, float* const* env_max, float* const* env_min,
                            void* stream) {
  if (nprob <= 0) return AC_OK;
  if ((d == 64 || d == 128) && (dtype == AC_DTYPE_BF16 || dtype == AC_DTYPE_F32)) {
    const dim3 grid((unsigned)max_k, nprob);
    const bool bf = dtype == AC_DTYPE_BF16;
    if (d == 64) {
      if (bf) k_envelopes_w<2, true><<<grid, 32 * kEnvWarps, 0, S(stream)>>>(probs, env_max, env_min);
      else k_envelopes_w<2, false><<<grid, 32 * kEnvWarps, 0, S(stream)>>>(probs, env_max, env_min);
    } else {
      if (bf) k_envelopes_w<4, true><<<grid, 32 * kEnvWarps, 0, S(stream)>>>(probs, env_max, env_min);
      else k_envelopes_w<4, false><<<grid, 32 * kEnvWarps, 0, S(stream)>>>(probs, env_max, env_min);
    }
  } else {
    k_envelopes<<<dim3((max_k + 7) / 8, nprob), 256, 0, S(stream)>>>(probs, dtype, d, env_max, env_min);
  }
  AC_CHECK_LAUNCH("k_envelopes");
  return AC_OK;
}

extern "C" int ac_sort_by_label(const ac_cluster_problem* probs, int nprob, int64_t max_n,
                                int max_k, void* stream) {
  if (nprob <= 0 || max_n <= 0) return AC_OK;
  cudaStream_t st = S(stream);
  const unsigned tiles = (unsigned)((max_n + kAsgBM - 1) / kAsgBM);
  const size_t smem = sizeof(int) * (size_t)(max_k + 4);
  int rc = set_smem((const void*)k_tile_hist, smem);
  if (rc) return rc;
  k_tile_hist<<<dim3(tiles, nprob), kAsgBM, smem, st>>>(probs, max_k);
  AC_CHECK_LAUNCH("k_tile_hist");
  // dtype/d are only used by the (inactive) repair path: counts are all >= 1
  return repair_sort_impl(probs, nprob, AC_DTYPE_F32, 1, max_n, max_k, -1, AC_ASSIGN_ALL, st);
}
