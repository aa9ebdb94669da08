// Critical-cluster selection: TensorQuest scores, stable top-k, run
// coalescing of the selected key clusters, and density.
//
// Reference: /root/reference/pkg/src/adacluster/quest.py:94-143 and
// pipeline.py:144-151, :188-195.  Scores are the reference's two f32 GEMMs in
// OpenBLAS accumulation order followed by an f32 add, so rankings (and hence
// the selected sets) are bit-identical.  Compiled with --fmad=false.
#include <climits>

#include "common.cuh"

namespace ac {

AC_DEV float np_max0(float a) { return (a >= 0.f || isnan(a)) ? a : 0.f; }  // np.maximum(a, 0.0)
AC_DEV float np_min0(float a) { return (a <= 0.f || isnan(a)) ? a : 0.f; }  // np.minimum(a, 0.0)

template <typename GetX, typename GetC>
AC_DEV float sel_dot(const GetX& gx, const GetC& gc, int d, int order, bool halves = false) {
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
    const float s0 = __fadd_rn(a[0], a[4]), s1 = __fadd_rn(a[1], a[5]);
    const float s2 = __fadd_rn(a[2], a[6]), s3 = __fadd_rn(a[3], a[7]);
    return __fadd_rn(__fadd_rn(s0, s1), __fadd_rn(s2, s3));
  }
  float acc = 0.f;
  for (int t = 0; t < d; ++t) acc = __fmaf_rn(gx(t), gc(t), acc);
  return acc;
}

// One CTA per (query cluster g, problem).  Threads own key clusters.
__global__ void __launch_bounds__(256)
k_select(const ac_select_problem* __restrict__ probs, int d, int scorer, float top_p,
         float mass_scale_log2) {
  extern __shared__ __align__(16) float ssm[];
  const ac_select_problem& P = probs[blockIdx.y];
  const int g = blockIdx.x;
  if (g >= P.gq) return;
  const int C = P.c, topk = P.topk, tid = threadIdx.x;
  float* s_q = ssm;                 // [d] representative row
  float* s_sc = s_q + d;            // [C] scores
  int* s_rank = reinterpret_cast<int*>(s_sc + C);  // [C] rank (or INT_MAX)
  int* s_start = s_rank + C;        // [C] run-start flags -> run ids
  __shared__ unsigned long long s_cov;
  __shared__ int s_nr;
  __shared__ int s_nsel;
  for (int t = tid; t < d; t += blockDim.x) s_q[t] = P.reps[(int64_t)g * d + t];
  if (tid == 0) { s_cov = 0ull; s_nr = 0; }
  __syncthreads();
  const int gq = P.gq;
  for (int c = tid; c < C; c += blockDim.x) {
    const bool hv = (g >= gq - gq % 4) && (c >= C - C % 4);
    const float* ma = P.emax + (int64_t)c * d;
    const float* mi = P.emin + (int64_t)c * d;
    float s;
    if (scorer == AC_SCORER_GIVEN) {
      s = P.scores[(int64_t)g * C + c];
    } else if (scorer == AC_SCORER_MEAN) {
      s = sel_dot([&](int t) { return s_q[t]; }, [&](int t) { return ma[t]; }, d, P.order, hv);
    } else if (scorer == AC_SCORER_CLAMPED) {
      const float a = sel_dot([&](int t) { return np_max0(s_q[t]); },
                              [&](int t) { return np_max0(ma[t]); }, d, P.order, hv);
      const float b = sel_dot([&](int t) { return np_min0(s_q[t]); },
                              [&](int t) { return np_min0(ma[t]); }, d, P.order, hv);
      s = __fadd_rn(a, b);
    } else {
      const float a = sel_dot([&](int t) { return np_max0(s_q[t]); },
                              [&](int t) { return ma[t]; }, d, P.order, hv);
      const float b = sel_dot([&](int t) { return np_min0(s_q[t]); },
                              [&](int t) { return mi[t]; }, d, P.order, hv);
      s = __fadd_rn(a, b);
    }
    s_sc[c] = s;
    if (scorer != AC_SCORER_GIVEN) P.scores[(int64_t)g * C + c] = s;
  }
  __syncthreads();
  // np.argsort(-scores, kind="stable")[:topk]: rank = #greater + #equal-before
  for (int c = tid; c < C; c += blockDim.x) {
    const float v = s_sc[c];
    int r = 0;
    for (int i = 0; i < C; ++i) {
      const float o = s_sc[i];
      r += (o > v) || (o == v && i < c);
    }
    s_rank[c] = r;
    s_start[r] = c;  // rank -> cluster (reused below as run flags)
  }
  if (tid == 0) s_nsel = topk;
  __syncthreads();
  if (top_p > 0.f && tid < 32) {
    // top-p: the smallest score-ordered prefix whose estimated attention mass
    // counts_c * 2^((s_c - s_max) * scale) reaches top_p of the total (at
    // least one cluster, at most topk); warp-level prefix sums in rank order
    const float smax = s_sc[s_start[0]];
    float tot = 0.f;
    for (int r = tid; r < C; r += 32) {
      const int c = s_start[r];
      tot += (float)P.counts[c] * exp2f((s_sc[c] - smax) * mass_scale_log2);
    }
    for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    const float goal = top_p * tot;
    float run = 0.f;
    int nsel = min(C, topk);
    for (int r0 = 0; r0 < C; r0 += 32) {
      const int r = r0 + tid;
      float m = 0.f;
      if (r < C) {
        const int c = s_start[r];
        m = (float)P.counts[c] * exp2f((s_sc[c] - smax) * mass_scale_log2);
      }
      float inc = m;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const float y = __shfl_up_sync(0xffffffffu, inc, o);
        if (tid >= o) inc += y;
      }
      const unsigned hit = __ballot_sync(0xffffffffu, r < C && run + inc >= goal);
      if (hit) {
        nsel = min(nsel, r0 + __ffs(hit));
        break;
      }
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (tid == 0) s_nsel = max(1, nsel);
  }
  __syncthreads();
  const int nsel = s_nsel;
  for (int r = tid; r < topk; r += blockDim.x)
    if (r >= nsel) P.selected[(int64_t)g * topk + r] = -1;
  for (int c = tid; c < C; c += blockDim.x) {
    const int r = s_rank[c];
    if (r < nsel) {
      P.selected[(int64_t)g * topk + r] = c;
      atomicAdd(&s_cov, (unsigned long long)P.counts[c]);
    }
  }
  __syncthreads();
  // maximal runs of consecutive selected clusters -> contiguous Kp ranges
  for (int c = tid; c < C; c += blockDim.x) {
    const bool in = s_rank[c] < nsel;
    const bool prev = (c > 0) && (s_rank[c - 1] < nsel);
    s_start[c] = (in && !prev) ? 1 : 0;
  }
  __syncthreads();
  if (tid == 0) {
    int nr = 0;
    for (int c = 0; c < C; ++c) {
      const int f = s_start[c];
      s_start[c] = f ? nr : -1;
      nr += f;
    }
    s_nr = nr;
    P.nruns[g] = nr;
    P.covered[g] = (long long)s_cov;
  }
  __syncthreads();
  for (int c = tid; c < C; c += blockDim.x) {
    const int rid = s_start[c];
    if (rid < 0) continue;
    int e = c;
    while (e + 1 < C && s_rank[e + 1] < nsel) ++e;
    int32_t* run = P.runs + ((int64_t)g * P.run_stride + rid) * 2;
    run[0] = P.kstarts[c];
    run[1] = P.kstarts[e] + P.counts[e];
  }
}

// density = mean_g(covered_g) / sum(counts)   (quest.py:141-142, all exact)
__global__ void k_density(const ac_select_problem* __restrict__ probs) {
  const ac_select_problem& P = probs[blockIdx.x];
  __shared__ unsigned long long s_cov, s_tot;
  if (threadIdx.x == 0) { s_cov = 0; s_tot = 0; }
  __syncthreads();
  for (int g = threadIdx.x; g < P.gq; g += blockDim.x) atomicAdd(&s_cov, (unsigned long long)P.covered[g]);
  for (int c = threadIdx.x; c < P.c; c += blockDim.x) atomicAdd(&s_tot, (unsigned long long)P.counts[c]);
  __syncthreads();
  if (threadIdx.x == 0)
    P.density[0] = __ddiv_rn(__ddiv_rn((double)s_cov, (double)P.gq), (double)s_tot);
}

}  // namespace ac

using namespace ac;

static int select_impl(const ac_select_problem* probs, int nprob, int d, int scorer, int max_gq,
                       int max_c, float top_p, float mass_scale_log2, void* stream) {
  if (nprob <= 0) return AC_OK;
  if (scorer < 0 || scorer > AC_SCORER_GIVEN) { ac_host::set_error("ac_select: bad scorer %d", scorer); return AC_ERR_PARAM; }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const size_t smem = sizeof(float) * ((size_t)d + max_c) + sizeof(int) * 2 * (size_t)max_c;
  if (smem > 48 * 1024) {
    const int rc = ac_host::func_smem((const void*)k_select, (int)smem, "k_select smem");
    if (rc) return rc;
  }
  k_select<<<dim3(max_gq, nprob), 256, smem, st>>>(probs, d, scorer, top_p, mass_scale_log2);
  k_density<<<nprob, 256, 0, st>>>(probs);
  AC_CHECK_LAUNCH("ac_select");
  return AC_OK;
}

extern "C" int ac_select(const ac_select_problem* probs, int nprob, int d, int scorer,
                         int max_gq, int max_c, int max_topk, void* stream) {
  (void)max_topk;
  return select_impl(probs, nprob, d, scorer, max_gq, max_c, 0.f, 0.f, stream);
}

extern "C" int ac_select_topp(const ac_select_problem* probs, int nprob, int d, int scorer,
                              int max_gq, int max_c, int max_topk, float top_p,
                              float mass_scale, void* stream) {
  (void)max_topk;
  if (!(top_p > 0.f && top_p <= 1.f)) {
    ac_host::set_error("ac_select_topp: top_p=%g not in (0, 1]", (double)top_p);
    return AC_ERR_PARAM;
  }
  return select_impl(probs, nprob, d, scorer, max_gq, max_c, top_p,
                     mass_scale * 1.4426950408889634f, stream);
}
