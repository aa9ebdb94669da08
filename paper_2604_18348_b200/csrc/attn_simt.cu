// Token permutation into cluster-contiguous order, the per-head query layout
// (query clusters padded to 128-row tiles + work items), and the CUDA-core
// block-sparse attention used for f32 inputs (the reference's f32 numerics,
// reference.py:25-45, within 1e-4 rel-L2) and as the cross-check of the
// tcgen05 kernel.
//
// Work item = (head, query cluster g, 128-row tile).  The item attends over
// the union of the selected key clusters of g, given as [start, end) runs of
// the cluster-contiguous Kp/Vp (adjacent selected clusters are merged).
#include <cfloat>
#include <climits>

#include "common.cuh"

namespace ac {

// dst[j] = src[perm[j]] — 16-byte vectors when the row size allows it
__global__ void k_permute_rows16(const uint4* __restrict__ src, const int32_t* __restrict__ perm,
                                 int64_t n, int vec_per_row, uint4* __restrict__ dst) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * vec_per_row) return;
  const int64_t j = e / vec_per_row;
  const int part = (int)(e - j * vec_per_row);
  dst[e] = src[(int64_t)perm[j] * vec_per_row + part];
}

// per-head gather: dst[h, j] = src[h, perm[h, j]]
__global__ void k_permute_rows16_heads(const uint4* __restrict__ src, const int32_t* __restrict__ perm,
                                       int64_t L, int heads, int vec_per_row, uint4* __restrict__ dst) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)heads * L * vec_per_row) return;
  const int64_t j = e / vec_per_row;  // global row h*L + jj
  const int part = (int)(e - j * vec_per_row);
  const int64_t h = j / L;
  dst[e] = src[(h * L + perm[j]) * vec_per_row + part];
}

__global__ void k_permute_rows_b(const uint8_t* __restrict__ src, const int32_t* __restrict__ perm,
                                 int64_t n, int row_bytes, uint8_t* __restrict__ dst) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n * row_bytes) return;
  const int64_t j = e / row_bytes;
  const int part = (int)(e - j * row_bytes);
  dst[e] = src[(int64_t)perm[j] * row_bytes + part];
}

// per head: padded block starts of every query cluster and the work items
__global__ void k_q_layout_items(int64_t L, const int32_t* __restrict__ qcounts,
                                 const int32_t* __restrict__ gq, int gq_max,
                                 const int32_t* __restrict__ nruns, int topk_max,
                                 int64_t qp_cap, int32_t* __restrict__ padstart,
                                 ac_attn_item* __restrict__ items, int item_cap, int item_rows) {
  const int h = blockIdx.x;
  const int G = gq[h];
  if (threadIdx.x != 0) return;
  int64_t rowpos = 0;
  int it = 0;
  ac_attn_item* out = items + (int64_t)h * item_cap;
  for (int g = 0; g < G; ++g) {
    const int cnt = qcounts[(int64_t)h * gq_max + g];
    padstart[(int64_t)h * gq_max + g] = (int32_t)rowpos;
    for (int r0 = 0; r0 < cnt; r0 += item_rows) {
      if (it < item_cap) {
        ac_attn_item m;
        m.q_row0 = (int64_t)h * qp_cap + rowpos + r0;
        m.q_rows = min(item_rows, cnt - r0);
        m.head = h;
        m.run0 = (h * gq_max + g) * topk_max;
        m.nruns = nruns[(int64_t)h * gq_max + g];
        out[it] = m;
      }
      ++it;
    }
    rowpos += ((cnt + 127) / 128) * 128;
  }
  for (; it < item_cap; ++it) {
    ac_attn_item m;
    m.q_row0 = 0; m.q_rows = 0; m.head = h; m.run0 = 0; m.nruns = 0;
    out[it] = m;
  }
}

// scatter queries into the padded per-cluster layout
__global__ void k_q_layout_rows(const void* __restrict__ q, int dtype, int d, int64_t L,
                                const int32_t* __restrict__ qperm, const int32_t* __restrict__ qstarts,
                                const int32_t* __restrict__ qlabels, int gq_max,
                                const int32_t* __restrict__ padstart, void* __restrict__ qp,
                                int32_t* __restrict__ qidx, int64_t qp_cap) {
  const int h = blockIdx.y;
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= L) return;
  const int32_t tok = qperm[(int64_t)h * L + j];
  const int g = qlabels[(int64_t)h * L + tok];
  const int64_t local = j - qstarts[(int64_t)h * (gq_max + 1) + g];
  const int64_t row = (int64_t)h * qp_cap + padstart[(int64_t)h * gq_max + g] + local;
  qidx[row] = tok;
  const int64_t src = ((int64_t)h * L + tok) * d, dst = row * d;
  const int esz = dtype == AC_DTYPE_BF16 ? 2 : 4;
  const char* sp = reinterpret_cast<const char*>(q) + src * esz;
  char* op = reinterpret_cast<char*>(qp) + dst * esz;
  const int bytes = d * esz;
  if ((bytes & 15) == 0 && ((reinterpret_cast<uintptr_t>(sp) | reinterpret_cast<uintptr_t>(op)) & 15) == 0) {
    for (int o = 0; o < bytes; o += 16)
      *reinterpret_cast<uint4*>(op + o) = *reinterpret_cast<const uint4*>(sp + o);
  } else {
    for (int o = 0; o < bytes; ++o) op[o] = sp[o];
  }
}

// the same scatter with one thread per 16-byte piece (rows of 16-byte
// multiples, 16-byte aligned bases): a warp moves whole contiguous rows
__global__ void k_q_layout_rows16(const uint4* __restrict__ q, int pieces, int64_t L,
                                  const int32_t* __restrict__ qperm, const int32_t* __restrict__ qstarts,
                                  const int32_t* __restrict__ qlabels, int gq_max,
                                  const int32_t* __restrict__ padstart, uint4* __restrict__ qp,
                                  int32_t* __restrict__ qidx, int64_t qp_cap) {
  const int h = blockIdx.y;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;  // L * pieces < 2^31 (host check)
  const int j = e / pieces;
  const int part = e - j * pieces;
  if (j >= L) return;
  const int32_t tok = qperm[(int64_t)h * L + j];
  const int g = qlabels[(int64_t)h * L + tok];
  const int64_t local = j - qstarts[(int64_t)h * (gq_max + 1) + g];
  const int64_t row = (int64_t)h * qp_cap + padstart[(int64_t)h * gq_max + g] + local;
  if (part == 0) qidx[row] = tok;
  qp[row * pieces + part] = __ldg(q + ((int64_t)h * L + tok) * pieces + part);
}

// ---------------------------------------------------------------------------
// CUDA-core flash attention over runs.  128 query rows x 64-key tiles,
// 256 threads: thread (rg = tid/16, kg = tid%16) owns rows rg*8..rg*8+7,
// keys kg*4..kg*4+3 of the S tile and dims kg*(D/16).. of O.
// ---------------------------------------------------------------------------
constexpr int kSimtBQ = 128;
constexpr int kSimtBK = 64;

template <int D>
__global__ void __launch_bounds__(256)
k_attn_simt(const void* __restrict__ q, const int32_t* __restrict__ qidx,
            const void* __restrict__ kp, const void* __restrict__ vp, int dtype, int64_t L,
            const ac_attn_item* __restrict__ items, const int32_t* __restrict__ runs, float scale,
            void* __restrict__ out, int out_dtype) {
  constexpr int DPT = D / 16;  // O dims per thread
  extern __shared__ __align__(16) float asm_[];
  float* Qs = asm_;                          // [D][BQ]
  float* Ks = Qs + D * kSimtBQ;              // [D][BK]
  float* Vs = Ks + D * kSimtBK;              // [BK][D]
  float* Pt = Vs + kSimtBK * D;              // [BK][BQ + 4]
  const ac_attn_item it = items[blockIdx.x];
  if (it.q_rows <= 0) return;
  const int tid = threadIdx.x, rg = tid >> 4, kg = tid & 15;
  const int64_t hoff = (int64_t)it.head * L * D;
  auto ld = [&](const void* base, int64_t i) -> float { return ld_elem(base, dtype, i); };

  for (int e = tid; e < kSimtBQ * D; e += 256) {
    const int r = e / D, t = e % D;
    Qs[t * kSimtBQ + r] = (r < it.q_rows) ? ld(q, (it.q_row0 + r) * D + t) : 0.f;
  }
  float m[8], l[8], o[8][DPT];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    m[i] = -INFINITY; l[i] = 0.f;
#pragma unroll
    for (int j = 0; j < DPT; ++j) o[i][j] = 0.f;
  }
  for (int ri = 0; ri < it.nruns; ++ri) {
    const int rs = runs[2 * (it.run0 + ri)], re = runs[2 * (it.run0 + ri) + 1];
    for (int k0 = rs; k0 < re; k0 += kSimtBK) {
      const int nk = min(kSimtBK, re - k0);
      __syncthreads();
      for (int e = tid; e < kSimtBK * D; e += 256) {
        const int r = e / D, t = e % D;
        const bool ok = r < nk;
        Ks[t * kSimtBK + r] = ok ? ld(kp, hoff + (int64_t)(k0 + r) * D + t) : 0.f;
        Vs[r * D + t] = ok ? ld(vp, hoff + (int64_t)(k0 + r) * D + t) : 0.f;
      }
      __syncthreads();
      float s[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) s[i][j] = 0.f;
#pragma unroll 8
      for (int t = 0; t < D; ++t) {
        const float4 a0 = *reinterpret_cast<const float4*>(Qs + t * kSimtBQ + rg * 8);
        const float4 a1 = *reinterpret_cast<const float4*>(Qs + t * kSimtBQ + rg * 8 + 4);
        const float4 b = *reinterpret_cast<const float4*>(Ks + t * kSimtBK + kg * 4);
        const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        const float bb[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) s[i][j] = fmaf(a[i], bb[j], s[i][j]);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float tmax = -INFINITY;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          s[i][j] = (kg * 4 + j < nk) ? s[i][j] * scale : -INFINITY;
          tmax = fmaxf(tmax, s[i][j]);
        }
#pragma unroll
        for (int off = 8; off; off >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, off));
        const float mnew = fmaxf(m[i], tmax);
        const float alpha = (mnew == -INFINITY) ? 1.f : expf(m[i] - mnew);
        float psum = 0.f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float p = (mnew == -INFINITY) ? 0.f : expf(s[i][j] - mnew);
          psum += p;
          Pt[(kg * 4 + j) * (kSimtBQ + 4) + rg * 8 + i] = p;
        }
#pragma unroll
        for (int off = 8; off; off >>= 1) psum += __shfl_xor_sync(0xffffffffu, psum, off);
        l[i] = l[i] * alpha + psum;
        m[i] = mnew;
#pragma unroll
        for (int j = 0; j < DPT; ++j) o[i][j] *= alpha;
      }
      __syncthreads();
      for (int j = 0; j < nk; ++j) {
        const float4 p0 = *reinterpret_cast<const float4*>(Pt + j * (kSimtBQ + 4) + rg * 8);
        const float4 p1 = *reinterpret_cast<const float4*>(Pt + j * (kSimtBQ + 4) + rg * 8 + 4);
        const float p[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
        float vv[DPT];
#pragma unroll
        for (int u = 0; u < DPT; ++u) vv[u] = Vs[j * D + kg * DPT + u];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int u = 0; u < DPT; ++u) o[i][u] = fmaf(p[i], vv[u], o[i][u]);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = rg * 8 + i;
    if (r >= it.q_rows) continue;
    const int tok = qidx[it.q_row0 + r];
    if (tok < 0) continue;
    const float inv = 1.f / l[i];
    const int64_t ob = hoff + (int64_t)tok * D + kg * DPT;
#pragma unroll
    for (int u = 0; u < DPT; ++u) {
      const float val = o[i][u] * inv;
      if (out_dtype == AC_DTYPE_BF16)
        reinterpret_cast<__nv_bfloat16*>(out)[ob + u] = __float2bfloat16_rn(val);
      else
        reinterpret_cast<float*>(out)[ob + u] = val;
    }
  }
}

template <int D>
size_t simt_smem() {
  return sizeof(float) * ((size_t)D * kSimtBQ + (size_t)D * kSimtBK + (size_t)kSimtBK * D +
                          (size_t)kSimtBK * (kSimtBQ + 4));
}

template <int D>
int launch_simt(const void* q, const int32_t* qidx, const void* k, const void* v, int dtype,
                int64_t L, const ac_attn_item* items, int nitems, const int32_t* runs, float scale,
                void* out, int out_dtype, cudaStream_t st) {
  const size_t smem = simt_smem<D>();
  const int rc = ac_host::func_smem((const void*)k_attn_simt<D>, (int)smem, "k_attn_simt smem");
  if (rc) return rc;
  k_attn_simt<D><<<nitems, 256, smem, st>>>(q, qidx, k, v, dtype, L, items, runs, scale, out, out_dtype);
  AC_CHECK_LAUNCH("k_attn_simt");
  return AC_OK;
}


// ---------------------------------------------------------------------------
// Work-item order for the attention launch: longest first.  The attention
// kernels take one item per CTA in blockIdx order, which the hardware
// dispatches roughly in order as SMs free up, so issuing the items by
// descending cost (Q tiles x K/V tiles of its runs) is greedy LPT list
// scheduling: the last CTAs to start are the shortest, which shortens the
// tail of the launch.  Items write disjoint output rows, so the order does
// not change any result.  One CTA: cost buckets (descending), counting-sort
// scatter into `scratch`, copy back.
// ---------------------------------------------------------------------------
constexpr int kOrdBuckets = 4096;

AC_DEV int item_cost(const ac_attn_item& m, const int32_t* runs) {
  if (m.q_rows <= 0) return 0;
  const int32_t* r = runs + 2 * (int64_t)m.run0;
  int tiles = 0;
  for (int i = 0; i < m.nruns; ++i) tiles += (r[2 * i + 1] - r[2 * i] + 127) / 128;
  return ((m.q_rows + 127) / 128) * (tiles + 2);  // +2: per-item prologue / epilogue
}

__global__ void __launch_bounds__(1024)
k_order_items(ac_attn_item* __restrict__ items, int nitems, const int32_t* __restrict__ runs,
              ac_attn_item* __restrict__ scratch) {
  __shared__ int hist[kOrdBuckets];
  __shared__ int wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int b = tid; b < kOrdBuckets; b += blockDim.x) hist[b] = 0;
  __syncthreads();
  auto key = [&](int i) {  // descending cost
    return kOrdBuckets - 1 - min(item_cost(items[i], runs), kOrdBuckets - 1);
  };
  for (int i = tid; i < nitems; i += blockDim.x) atomicAdd(&hist[key(i)], 1);
  __syncthreads();
  // exclusive scan: 4 buckets per thread, then a block scan of the thread sums
  constexpr int kPer = kOrdBuckets / 1024;
  int loc[kPer], tot = 0;
#pragma unroll
  for (int j = 0; j < kPer; ++j) { loc[j] = hist[tid * kPer + j]; tot += loc[j]; }
  int inc = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) wsum[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    int w = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    wsum[lane] = w;
  }
  __syncthreads();
  int run = (warp ? wsum[warp - 1] : 0) + inc - tot;
#pragma unroll
  for (int j = 0; j < kPer; ++j) { hist[tid * kPer + j] = run; run += loc[j]; }
  __syncthreads();
  for (int i = tid; i < nitems; i += blockDim.x) scratch[atomicAdd(&hist[key(i)], 1)] = items[i];
  __syncthreads();
  for (int i = tid; i < nitems; i += blockDim.x) items[i] = scratch[i];
}

}  // namespace ac

using namespace ac;

extern "C" int ac_permute_rows(const void* src, int dtype, int d, const int32_t* perm, int64_t n,
                               void* dst, void* stream) {
  if (n <= 0) return AC_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int esz = dtype == AC_DTYPE_BF16 ? 2 : 4;
  const int row_bytes = d * esz;
  if (row_bytes % 16 == 0 && ((uintptr_t)src % 16 == 0) && ((uintptr_t)dst % 16 == 0)) {
    const int vpr = row_bytes / 16;
    const int64_t total = n * vpr;
    k_permute_rows16<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<const uint4*>(src), perm, n, vpr, reinterpret_cast<uint4*>(dst));
  } else {
    const int64_t total = n * row_bytes;
    k_permute_rows_b<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<const uint8_t*>(src), perm, n, row_bytes, reinterpret_cast<uint8_t*>(dst));
  }
  AC_CHECK_LAUNCH("ac_permute_rows");
  return AC_OK;
}

extern "C" int ac_permute_rows_heads(const void* src, int dtype, int d, const int32_t* perm,
                                     int64_t L, int heads, void* dst, void* stream) {
  if (L <= 0 || heads <= 0) return AC_OK;
  const int esz = dtype == AC_DTYPE_BF16 ? 2 : 4;
  const int row_bytes = d * esz;
  if (row_bytes % 16 != 0 || ((uintptr_t)src % 16) || ((uintptr_t)dst % 16)) {
    ac_host::set_error("ac_permute_rows_heads: rows must be 16-byte multiples (d=%d)", d);
    return AC_ERR_DIM;
  }
  const int vpr = row_bytes / 16;
  const int64_t total = (int64_t)heads * L * vpr;
  k_permute_rows16_heads<<<(unsigned)((total + 255) / 256), 256, 0,
                           reinterpret_cast<cudaStream_t>(stream)>>>(
      reinterpret_cast<const uint4*>(src), perm, L, heads, vpr, reinterpret_cast<uint4*>(dst));
  AC_CHECK_LAUNCH("ac_permute_rows_heads");
  return AC_OK;
}

extern "C" int ac_build_q_layout(const void* q, int dtype, int d, int64_t L, int heads,
                                 const int32_t* qperm, const int32_t* qstarts,
                                 const int32_t* qcounts, const int32_t* qlabels, const int32_t* gq,
                                 int gq_max, const int32_t* nruns, int topk_max, void* qp,
                                 int32_t* qidx, int64_t qp_cap, ac_attn_item* items, int item_cap,
                                 int item_rows, void* stream) {
  if (heads <= 0 || L <= 0) return AC_OK;
  if (item_rows != 128 && item_rows != 256) {
    ac_host::set_error("ac_build_q_layout: item_rows must be 128 or 256");
    return AC_ERR_PARAM;
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int32_t* padstart = nullptr;
  // padstart lives right after qidx's used range: callers size qidx as
  // heads * qp_cap + heads * gq_max
  padstart = qidx + (int64_t)heads * qp_cap;
  cudaMemsetAsync(qidx, 0xff, sizeof(int32_t) * (size_t)heads * qp_cap, st);
  k_q_layout_items<<<heads, 32, 0, st>>>(L, qcounts, gq, gq_max, nruns, topk_max, qp_cap, padstart,
                                         items, item_cap, item_rows);
  const int bytes = d * (dtype == AC_DTYPE_BF16 ? 2 : 4);
  if ((bytes & 15) == 0 && L * (bytes / 16) < (int64_t)INT_MAX - 256 &&
      ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(qp)) & 15) == 0) {
    const int pieces = bytes / 16;
    k_q_layout_rows16<<<dim3((unsigned)((L * pieces + 255) / 256), heads), 256, 0, st>>>(
        reinterpret_cast<const uint4*>(q), pieces, L, qperm, qstarts, qlabels, gq_max, padstart,
        reinterpret_cast<uint4*>(qp), qidx, qp_cap);
  } else {
    k_q_layout_rows<<<dim3((unsigned)((L + 255) / 256), heads), 256, 0, st>>>(
        q, dtype, d, L, qperm, qstarts, qlabels, gq_max, padstart, qp, qidx, qp_cap);
  }
  AC_CHECK_LAUNCH("ac_build_q_layout");
  return AC_OK;
}

extern "C" int ac_sparse_attention_simt(const void* q, const int32_t* qidx, const void* k,
                                        const void* v, int dtype, int d, int64_t L,
                                        const ac_attn_item* items, int nitems, const int32_t* runs,
                                        float scale, void* out, int out_dtype, void* stream) {
  if (nitems <= 0) return AC_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  switch (d) {
    case 16: return launch_simt<16>(q, qidx, k, v, dtype, L, items, nitems, runs, scale, out, out_dtype, st);
    case 32: return launch_simt<32>(q, qidx, k, v, dtype, L, items, nitems, runs, scale, out, out_dtype, st);
    case 64: return launch_simt<64>(q, qidx, k, v, dtype, L, items, nitems, runs, scale, out, out_dtype, st);
    case 128: return launch_simt<128>(q, qidx, k, v, dtype, L, items, nitems, runs, scale, out, out_dtype, st);
    default:
      ac_host::set_error("attention: head_dim %d unsupported (16/32/64/128; pad smaller dims)", d);
      return AC_ERR_DIM;
  }
}

extern "C" int ac_order_items(ac_attn_item* items, int nitems, const int32_t* runs,
                              ac_attn_item* scratch, void* stream) {
  if (nitems <= 0) return AC_OK;
  if (!items || !runs || !scratch) {
    ac_host::set_error("ac_order_items: null pointer");
    return AC_ERR_PARAM;
  }
  k_order_items<<<1, 1024, 0, reinterpret_cast<cudaStream_t>(stream)>>>(items, nitems, runs, scratch);
  AC_CHECK_LAUNCH("k_order_items");
  return AC_OK;
}
