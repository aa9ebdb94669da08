// K3 on the 5th-generation tensor cores: the Lloyd assignment step
// (clustering.py:68-97, `_pairwise_sq_dists` + `_assign`) as a tcgen05 GEMM
// with an exact fix-up epilogue.
//
// The reference computes d = (||x||^2 - 2 x·c) + ||c||^2 in f32 with
// OpenBLAS's sequential FMA chain for x·c, and takes the first-index argmin.
// Labels must be bit-identical (Lloyd is not converged at max_iter, so one
// flipped near-tie cascades — SURVEY.md §7 hard part 1).  Design:
//
//   1. x·c on tcgen05 (kind::f16, f32 accumulation in TMEM).  Centres are
//      split into three bf16 planes c = hi + mid + lo (exact for f32);
//      bf16 points are one exact plane (3 MMAs per K step), f32 points are
//      split the same way in shared memory (6 MMAs: every plane product
//      down to 2^-16 relative).
//   2. Epilogue, one thread per row (= TMEM lane): approximate d~_c, its
//      minimum, and every centre with d~_c <= min + 2T is a candidate, where
//      T bounds |d~ - d_ref| rigorously (split + accumulation error and the
//      reference chain's own rounding, both <= c·u·||x||·||c||).
//   3. Candidates are recomputed with the reference's exact sequential
//      fmaf chain (x and c reconstructed exactly from the bf16 planes in
//      shared memory) and the first-index minimum of the exact values wins.
//      Almost every row has one candidate — its exact d is what `best`
//      (inertia, repair, stage MSE) needs anyway.
//
// So labels and distances equal k_assign_seq's (the all-FFMA kernel) bit
// for bit; tests/test_gpu_parity.py checks exactly that.
//
// Warp roles (448 threads, one CTA per SM, persistent over the tiles of a
// batch of problems):
//   warp 0      TMA producer: 128-row x tiles (f32: two 32-column SW128
//               boxes; bf16: one 64-column box) into a ring
//   warp 1      MMA issuer (single thread), TMEM owner (2 x 128 columns)
//   warps 2-5   f32 input only: split x into hi/mid/lo bf16 planes (SW128
//               K-major, the canonical UMMA layout)
//   warps 6-13  two epilogue warpgroups, alternating tiles (one TMEM
//               accumulator each): argmin, exact fix-up, labels / best /
//               per-tile label histogram (the tiling matches k_scatter).
// Compiled with --fmad=false: the fix-up reproduces numpy's unfused ops.
#include <cfloat>
#include <climits>

#include <algorithm>
#include <cstring>

#include "tc_common.cuh"

namespace ac {
namespace asg {
using namespace ac::tc;

constexpr int BM = 128;     // rows per tile (== kAsgBM: shared tiling with the sort kernels)
constexpr int DIM = 64;     // head_dim handled by this kernel
constexpr int NBMAX = 128;  // centres per problem per launch (k - c_lo)
constexpr int MAXP = 32;    // problems per launch (tensor maps travel as kernel params)
constexpr int XS_F32 = 2;   // f32 x stages
constexpr int XS_BF16 = 4;  // bf16 x stages (the f32 plane region is free in bf16 mode)
constexpr int THREADS = 448;
constexpr int W_TMA = 0, W_MMA = 1, W_CONV0 = 2, W_EPI0 = 6;

constexpr int XF_BYTES = BM * DIM * 4;  // f32 tile: two 16 KB SW128 boxes of 32 columns
constexpr int PL_BYTES = BM * DIM * 2;  // one bf16 plane of a tile (16 KB)
constexpr int CP_BYTES = NBMAX * DIM * 2;
constexpr int OFF_X = 0;                              // f32: [2] x 32 KB | bf16: [4] x 16 KB
constexpr int OFF_XP = OFF_X + XS_F32 * XF_BYTES;     // f32: [2][3] planes
constexpr int OFF_CP = OFF_XP + XS_F32 * 3 * PL_BYTES;  // [3] centre planes
constexpr int OFF_CC = OFF_CP + 3 * CP_BYTES;           // [NBMAX] ||c||^2
constexpr int OFF_HIST = OFF_CC + NBMAX * 4;            // [2][NBMAX] label histograms
constexpr int OFF_BAR = OFF_HIST + 2 * NBMAX * 4;
constexpr int NBAR = 2 * XS_BF16 + 2 * 2 + 2 * 2;
constexpr int OFF_MISC = OFF_BAR + NBAR * 8;
constexpr int SMEM = OFF_MISC + 64 + 1024;  // + 1 KB alignment slack
static_assert(XS_BF16 * PL_BYTES <= OFF_CP - OFF_X, "bf16 ring must fit the x region");
static_assert(SMEM <= 227 * 1024, "shared memory budget");

struct Params {
  CUtensorMap x[MAXP];
  int tile0[MAXP + 1];  // first tile of each problem (prefix of ceil(n/128))
  int nprob;
  int dtype;
  int c_lo;
  int flags;
};

AC_DEV unsigned char* align1024(unsigned char* p) {
  return reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}
// byte offset of 16-byte chunk j of row r in a 128-byte-row SW128 tile
AC_DEV int sw128(int r, int j) { return r * 128 + ((j ^ (r & 7)) << 4); }

// exact 3-way bf16 split of f32 values (hi + mid + lo == v)
AC_DEV void split8(const float (&v)[8], uint4& h, uint4& m, uint4& l) {
  uint32_t hw[4], mw[4], lw[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    float r0 = v[2 * e], r1 = v[2 * e + 1];
    __nv_bfloat162 a = __floats2bfloat162_rn(r0, r1);
    r0 = __fsub_rn(r0, __low2float(a));
    r1 = __fsub_rn(r1, __high2float(a));
    __nv_bfloat162 b = __floats2bfloat162_rn(r0, r1);
    r0 = __fsub_rn(r0, __low2float(b));
    r1 = __fsub_rn(r1, __high2float(b));
    __nv_bfloat162 c = __floats2bfloat162_rn(r0, r1);
    hw[e] = *reinterpret_cast<uint32_t*>(&a);
    mw[e] = *reinterpret_cast<uint32_t*>(&b);
    lw[e] = *reinterpret_cast<uint32_t*>(&c);
  }
  h = make_uint4(hw[0], hw[1], hw[2], hw[3]);
  m = make_uint4(mw[0], mw[1], mw[2], mw[3]);
  l = make_uint4(lw[0], lw[1], lw[2], lw[3]);
}
AC_DEV float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
AC_DEV float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
// the 8 f32 values of a chunk: (hi + mid) + lo, exact
AC_DEV void join8(const uint4& h, const uint4& m, const uint4& l, float (&v)[8]) {
  const uint32_t hw[4] = {h.x, h.y, h.z, h.w}, mw[4] = {m.x, m.y, m.z, m.w},
                 lw[4] = {l.x, l.y, l.z, l.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    v[2 * e] = __fadd_rn(__fadd_rn(bf_lo(hw[e]), bf_lo(mw[e])), bf_lo(lw[e]));
    v[2 * e + 1] = __fadd_rn(__fadd_rn(bf_hi(hw[e]), bf_hi(mw[e])), bf_hi(lw[e]));
  }
}

// exact reference distance of this thread's row (xr) to smem centre c
AC_DEV float exact_dist(const unsigned char* cp, int c, const float (&xr)[DIM], float xx, float cc) {
  const unsigned char* cb = cp + c * 128;
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int off = (j ^ (c & 7)) << 4;
    const uint4 h = *reinterpret_cast<const uint4*>(cb + off);
    const uint4 m = *reinterpret_cast<const uint4*>(cb + CP_BYTES + off);
    const uint4 l = *reinterpret_cast<const uint4*>(cb + 2 * CP_BYTES + off);
    float cv[8];
    join8(h, m, l, cv);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc = __fmaf_rn(xr[8 * j + e], cv[e], acc);
  }
  return sq_dist(xx, acc, cc);
}

__global__ void __launch_bounds__(THREADS, 1)
k_assign_tc(const __grid_constant__ Params prm, const ac_cluster_problem* __restrict__ probs) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = align1024(smraw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool f32in = prm.dtype == AC_DTYPE_F32;
  const int XS = f32in ? XS_F32 : XS_BF16;
  const int XSTRIDE = f32in ? XF_BYTES : PL_BYTES;

  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + OFF_BAR);
  uint64_t* xfull = bars;
  uint64_t* xempty = bars + XS_BF16;
  uint64_t* pfull = bars + 2 * XS_BF16;
  uint64_t* pempty = pfull + 2;
  uint64_t* afull = pfull + 4;
  uint64_t* aempty = pfull + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + OFF_MISC);
  int* s_ccmax = reinterpret_cast<int*>(sm + OFF_MISC + 16);
  float* s_cc = reinterpret_cast<float*>(sm + OFF_CC);
  int* s_hist = reinterpret_cast<int*>(sm + OFF_HIST);
  unsigned char* cplanes = sm + OFF_CP;

  if (tid == 0) {
    for (int s = 0; s < XS_BF16; ++s) {
      mbar_init(xfull + s, 1);
      mbar_init(xempty + s, 128);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(pfull + b, 128);
      mbar_init(pempty + b, 128);
      mbar_init(afull + b, 1);
      mbar_init(aempty + b, 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == W_MMA) tmem_alloc(tmem_slot, 256);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  const int total = prm.tile0[prm.nprob];
  const int t_begin = (int)((int64_t)blockIdx.x * total / gridDim.x);
  const int t_end = (int)((int64_t)(blockIdx.x + 1) * total / gridDim.x);
  int g0 = 0;  // CTA-local sequence number of the segment's first tile
  int p = 0;
  for (int t = t_begin; t < t_end;) {
    while (prm.tile0[p + 1] <= t) ++p;
    const int seg_end = min(t_end, prm.tile0[p + 1]);
    const ac_cluster_problem& P = probs[p];
    const bool active = (prm.flags & AC_ASSIGN_ALL) || P.status[AC_ST_ACTIVE] != 0;
    if (!active) {
      t = seg_end;
      continue;
    }
    const int k = P.k, c_lo = prm.c_lo, nb = k - c_lo;
    const int nbp = max(16, (nb + 15) & ~15);
    const int64_t n = P.n;
    const int ptile0 = prm.tile0[p];
    const int ntiles_p = prm.tile0[p + 1] - ptile0;
    const int T = seg_end - t;

    // ---- centre planes, ||c||^2 and max ||c||^2 of this problem (all threads) ----
    if (tid == 0) *s_ccmax = 0;
    __syncthreads();
    for (int e = tid; e < nbp * 8; e += THREADS) {
      const int c = e >> 3, j = e & 7;
      float v[8];
      if (c < nb) {
        const float4* src = reinterpret_cast<const float4*>(P.centers + (int64_t)(c_lo + c) * DIM + 8 * j);
        const float4 a = src[0], b = src[1];
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = 0.f;
      }
      uint4 h, m, l;
      split8(v, h, m, l);
      const int off = sw128(c, j);
      *reinterpret_cast<uint4*>(cplanes + off) = h;
      *reinterpret_cast<uint4*>(cplanes + CP_BYTES + off) = m;
      *reinterpret_cast<uint4*>(cplanes + 2 * CP_BYTES + off) = l;
    }
    for (int c = tid; c < nbp; c += THREADS) {
      const float cc = (c < nb) ? P.cc[c_lo + c] : 0.f;
      s_cc[c] = cc;
      if (c < nb && cc > 0.f) atomicMax(s_ccmax, __float_as_int(cc));
    }
    fence_proxy_async();  // generic-proxy smem writes -> tensor-core (async proxy) reads
    __syncthreads();
    const float ccmax = __int_as_float(*s_ccmax);
    const float cmax = sqrtf(ccmax);

    if (warp == W_TMA) {
      // ------------------------------ TMA producer ------------------------------
      if (lane == 0) {
        for (int i = 0; i < T; ++i) {
          const int g = g0 + i, s = g % XS;
          if (g >= XS) mbar_wait(xempty + s, ((g / XS) - 1) & 1, 20);
          const int row = (t + i - ptile0) * BM;
          unsigned char* dst = sm + OFF_X + s * XSTRIDE;
          if (f32in) {
            mbar_expect_tx(xfull + s, XF_BYTES);
            tma_load_2d(dst, &prm.x[p], 0, row, xfull + s);
            tma_load_2d(dst + XF_BYTES / 2, &prm.x[p], 32, row, xfull + s);
          } else {
            mbar_expect_tx(xfull + s, PL_BYTES);
            tma_load_2d(dst, &prm.x[p], 0, row, xfull + s);
          }
        }
      }
      __syncwarp();
    } else if (warp == W_MMA) {
      // ------------------------------ MMA issuer --------------------------------
      if (lane == 0) {
        const uint32_t idesc = idesc_bf16(BM, nbp, false);
        const uint32_t ca = smem_u32(cplanes);
        // plane products kept: (x plane, c plane); dropped terms are < 2^-23 relative
        const int xi[6] = {0, 0, 1, 0, 1, 2};
        const int ci[6] = {0, 1, 0, 2, 1, 0};
        const int nterm = f32in ? 6 : 3;
        for (int i = 0; i < T; ++i) {
          const int g = g0 + i, s = g % XS, b = g & 1;
          if (f32in) mbar_wait(pfull + b, (g >> 1) & 1, 21);
          else mbar_wait(xfull + s, (g / XS) & 1, 22);
          if (g >= 2) mbar_wait(aempty + b, ((g >> 1) - 1) & 1, 23);
          fence_after();
          const uint32_t xa = f32in ? smem_u32(sm + OFF_XP + b * 3 * PL_BYTES)
                                    : smem_u32(sm + OFF_X + s * PL_BYTES);
          const uint32_t d = tmem + (uint32_t)(b * 128);
          for (int term = 0; term < nterm; ++term) {
#pragma unroll
            for (int kk = 0; kk < DIM / 16; ++kk) {
              const uint64_t ad = sdesc(xa + xi[term] * PL_BYTES + kk * 32, 16, 1024);
              const uint64_t bd = sdesc(ca + ci[term] * CP_BYTES + kk * 32, 16, 1024);
              umma_f16(d, ad, bd, idesc, (term > 0 || kk > 0) ? 1u : 0u);
            }
          }
          umma_commit(afull + b);
        }
      }
      __syncwarp();
    } else if (warp < W_EPI0) {
      // -------------------- f32 points: split into bf16 planes --------------------
      if (f32in) {
        const int r = tid - W_CONV0 * 32;  // 0..127
        for (int i = 0; i < T; ++i) {
          const int g = g0 + i, s = g % XS, b = g & 1;
          mbar_wait(xfull + s, (g / XS) & 1, 24);
          if (g >= 2) mbar_wait(pempty + b, ((g >> 1) - 1) & 1, 25);
          const unsigned char* xs = sm + OFF_X + s * XF_BYTES;
          unsigned char* xp = sm + OFF_XP + b * 3 * PL_BYTES;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const unsigned char* box = xs + (j >> 2) * (XF_BYTES / 2);
            const int q0 = (2 * j) & 7;
            const float4 a = *reinterpret_cast<const float4*>(box + sw128(r, q0));
            const float4 c = *reinterpret_cast<const float4*>(box + sw128(r, q0 + 1));
            const float v[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
            uint4 h, m, l;
            split8(v, h, m, l);
            const int off = sw128(r, j);
            *reinterpret_cast<uint4*>(xp + off) = h;
            *reinterpret_cast<uint4*>(xp + PL_BYTES + off) = m;
            *reinterpret_cast<uint4*>(xp + 2 * PL_BYTES + off) = l;
          }
          mbar_arrive(xempty + s);
          fence_proxy_async();
          mbar_arrive(pfull + b);
        }
      }
    } else {
      // ------------------------------ epilogue ------------------------------
      const int wg = (warp - W_EPI0) >> 2;
      const int q = warp & 3;  // TMEM lane quarter this warp may access
      const int r = q * 32 + lane;
      const uint32_t lane_base = (uint32_t)(q * 32) << 16;
      int* hist = s_hist + wg * NBMAX;
      int fixups = 0;
      for (int i = 0; i < T; ++i) {
        const int g = g0 + i;
        if ((g & 1) != wg) continue;
        const int b = wg, s = g % XS;
        const int tile = t + i - ptile0;
        const int64_t row = (int64_t)tile * BM + r;
        const bool valid = row < n;
        const float xx = valid ? P.xx[row] : 0.f;
        // rigorous bound on |d~ - d_ref|
        const float tb = 0x1p-13f * sqrtf(xx) * cmax + 0x1p-20f * (xx + ccmax) + 1e-30f;
        mbar_wait(afull + b, (g >> 1) & 1, 26);
        fence_after();
        const uint32_t acc_col = tmem + lane_base + (uint32_t)(b * 128);
        float dmin = INFINITY;
        for (int c0 = 0; c0 < nbp; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(acc_col + c0, v);
          tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const int c = c0 + u;
            if (c < nb) {
              const float d = sq_dist(xx, __uint_as_float(v[u]), s_cc[c]);
              if (d < dmin) dmin = d;
            }
          }
        }
        const float thr = dmin + 2.f * tb;
        int c1 = -1, c2 = -1, ncand = 0;
        for (int c0 = 0; c0 < nbp; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(acc_col + c0, v);
          tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < 32; ++u) {
            const int c = c0 + u;
            if (c < nb) {
              const float d = sq_dist(xx, __uint_as_float(v[u]), s_cc[c]);
              if (d <= thr) {
                c1 = (ncand == 0) ? c : c1;
                c2 = (ncand == 1) ? c : c2;
                ++ncand;
              }
            }
          }
        }
        fence_before();
        mbar_arrive(aempty + b);

        // this row's exact f32 values
        float xr[DIM];
        if (f32in) {
          const unsigned char* xp = sm + OFF_XP + b * 3 * PL_BYTES;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int off = sw128(r, j);
            float v8[8];
            join8(*reinterpret_cast<const uint4*>(xp + off),
                  *reinterpret_cast<const uint4*>(xp + PL_BYTES + off),
                  *reinterpret_cast<const uint4*>(xp + 2 * PL_BYTES + off), v8);
#pragma unroll
            for (int e = 0; e < 8; ++e) xr[8 * j + e] = v8[e];
          }
        } else {
          const unsigned char* xb = sm + OFF_X + s * PL_BYTES;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const uint4 w = *reinterpret_cast<const uint4*>(xb + sw128(r, j));
            const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              xr[8 * j + 2 * e] = bf_lo(ww[e]);
              xr[8 * j + 2 * e + 1] = bf_hi(ww[e]);
            }
          }
        }
        float best = INFINITY;
        int lbl = INT_MAX;
        if (valid) {
          if (ncand <= 2) {
            if (ncand >= 1) {
              const float d = exact_dist(cplanes, c1, xr, xx, s_cc[c1]);
              if (d < best) { best = d; lbl = c1; }
            }
            if (ncand == 2) {
              const float d = exact_dist(cplanes, c2, xr, xx, s_cc[c2]);
              if (d < best) { best = d; lbl = c2; }
            }
          } else {  // many near-ties (degenerate rows): exact over every centre
            for (int c = 0; c < nb; ++c) {
              const float d = exact_dist(cplanes, c, xr, xx, s_cc[c]);
              if (d < best) { best = d; lbl = c; }
            }
          }
          fixups += (ncand >= 2);
        }
        // x values are no longer needed: release the stage / planes
        if (f32in) mbar_arrive(pempty + b);
        else mbar_arrive(xempty + s);

        int label = (lbl == INT_MAX) ? c_lo : c_lo + lbl;
        if (valid) {
          if (prm.flags & AC_ASSIGN_MERGE) {
            const float eb = P.best[row];
            if (!(best < eb)) { best = eb; label = P.labels[row]; }
          }
          P.labels[row] = label;
          P.best[row] = best;
        }
        if (!(prm.flags & AC_ASSIGN_MERGE)) {
          named_sync(1 + wg, 128);
          for (int c = r; c < k; c += 128) hist[c] = 0;
          named_sync(1 + wg, 128);
          if (valid) atomicAdd(&hist[label], 1);
          named_sync(1 + wg, 128);
          int32_t* th = P.tile_hist + tile;
          for (int c = r; c < k; c += 128) th[(int64_t)c * ntiles_p] = hist[c];
        }
      }
      // per-problem statistics: rows that needed more than one exact chain
      fixups = __reduce_add_sync(0xffffffffu, fixups);
      if (lane == 0 && fixups) atomicAdd(&P.status[AC_ST_FIXUPS], fixups);
    }
    g0 += T;
    t = seg_end;
    __syncthreads();  // every role done with this problem before the centre planes change
  }

  fence_before();
  __syncthreads();
  if (warp == W_MMA) {
    fence_after();
    tmem_dealloc(tmem, 256);
  }
}

}  // namespace asg
}  // namespace ac

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
namespace ac_host {

// Can the tensor-core kernel take this batch?  (D = 64, general-path
// accumulation order, <= 128 centres past c_lo, 16-byte aligned rows.)
bool assign_tc_eligible(const ac_cluster_problem* host_probs, int nprob, int dtype, int d,
                        int c_lo, int order) {
  if (!host_probs || order != AC_ORDER_SEQ || d != ac::asg::DIM) return false;
  if (dtype != AC_DTYPE_F32 && dtype != AC_DTYPE_BF16) return false;
  for (int p = 0; p < nprob; ++p) {
    const ac_cluster_problem& P = host_probs[p];
    if (P.k - c_lo < 1 || P.k - c_lo > ac::asg::NBMAX) return false;
    if ((reinterpret_cast<uintptr_t>(P.x) & 15) || (reinterpret_cast<uintptr_t>(P.centers) & 15))
      return false;
  }
  return true;
}

int assign_tc_launch(const ac_cluster_problem* probs, const ac_cluster_problem* host_probs,
                     int nprob, int dtype, int c_lo, int flags, cudaStream_t st) {
  using namespace ac::asg;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaFuncSetAttribute((const void*)k_assign_tc,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return check_cuda(e, "k_assign_tc smem");
  }
  for (int p0 = 0; p0 < nprob; p0 += MAXP) {
    const int np = std::min(MAXP, nprob - p0);
    Params prm;
    memset(&prm, 0, sizeof(prm));
    prm.nprob = np;
    prm.dtype = dtype;
    prm.c_lo = c_lo;
    prm.flags = flags;
    prm.tile0[0] = 0;
    for (int j = 0; j < np; ++j) {
      const ac_cluster_problem& P = host_probs[p0 + j];
      const int64_t tiles = (P.n + BM - 1) / BM;
      prm.tile0[j + 1] = prm.tile0[j] + (int)tiles;
      int rc;
      if (dtype == AC_DTYPE_F32)
        rc = make_map_2d(&prm.x[j], P.x, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, std::max<int64_t>(P.n, 1),
                         DIM, 32, BM);
      else
        rc = make_map_2d(&prm.x[j], P.x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                         std::max<int64_t>(P.n, 1), DIM, 64, BM);
      if (rc) return rc;
    }
    const int total = prm.tile0[np];
    if (total == 0) continue;
    const int grid = std::min(total, sms);
    k_assign_tc<<<grid, THREADS, SMEM, st>>>(prm, probs + p0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return check_cuda(e, "k_assign_tc");
  }
  return AC_OK;
}

}  // namespace ac_host
