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
constexpr int THREADS = 448;
constexpr int W_TMA = 0, W_MMA = 1, W_CONV0 = 2, W_EPI0 = 6;
constexpr int XF_BYTES = BM * DIM * 4;  // f32 tile: two 16 KB SW128 boxes of 32 columns
constexpr int PL_BYTES = BM * DIM * 2;  // one bf16 plane of a tile (16 KB)
constexpr int CF_STRIDE = DIM + 4;      // f32 centre rows, padded against bank conflicts
constexpr int NBAR = 16;
constexpr int QCAP = 64;  // per-warp queue of extra (row, centre) fix-up candidates
constexpr int SMEM_MAX = 227 * 1024;

// Shared-memory layout, sized per launch from the largest centre count
// (cap = max round16(k - c_lo)).  f32 points: x stages (1 or 2) of 32 KB +
// 2 x 3 split planes; bf16 points: 4 x 16 KB x stages (the MMA operand).
// Then the centre planes [3][cap][64] bf16 (SW128), the exact f32 centres
// [cap][68], ||c||^2 [128], two label histograms [2][128], the epilogue
// warps' fix-up queues [8][64] x (entry, result), barriers.
struct Layout {
  int xs, xstride, off_xp, off_cp, cp_bytes, off_cf, off_cc, off_hist, off_q, off_bar, off_misc,
      smem;
};

struct Params {
  CUtensorMap x[MAXP];
  int tile0[MAXP + 1];  // first tile of each problem (prefix of ceil(n/128))
  int nprob;
  int dtype;
  int c_lo;
  int flags;
  Layout lay;
};

__host__ __device__ inline Layout make_layout(int dtype, int cap) {
  Layout l;
  const bool f32 = dtype == AC_DTYPE_F32;
  l.xs = f32 ? (cap <= 80 ? 2 : 1) : 4;
  l.xstride = f32 ? XF_BYTES : PL_BYTES;
  l.off_xp = l.xs * l.xstride;
  l.off_cp = l.off_xp + (f32 ? 2 * 3 * PL_BYTES : 0);
  l.cp_bytes = cap * 128;
  l.off_cf = l.off_cp + 3 * l.cp_bytes;
  l.off_cc = l.off_cf + cap * CF_STRIDE * 4;
  l.off_hist = l.off_cc + NBMAX * 4;
  l.off_q = l.off_hist + 2 * NBMAX * 4;
  l.off_bar = l.off_q + 8 * QCAP * 8;
  l.off_misc = l.off_bar + NBAR * 8;
  l.smem = l.off_misc + 64 + 1024;  // + alignment slack
  return l;
}

// 1 KB-aligned view of dynamic shared memory (offset arithmetic on the
// shared pointer itself, so the compiler keeps shared-space accesses)
AC_DEV unsigned char* align1024(unsigned char* p) {
  return p + ((1024u - (smem_u32(p) & 1023u)) & 1023u);
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

// the reference's d for row r of the x tile and f32 centre row cf:
// sequential fmaf chain from 0 (OpenBLAS general path), then sq_dist.
// x comes from shared memory: the three split planes (f32 points, joined
// exactly) or the bf16 tile itself.
AC_DEV float exact_dist(const unsigned char* xsm, bool f32in, int r, const float* cf, float xx,
                        float cc) {
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int off = sw128(r, j);
    float xv[8];
    if (f32in) {
      join8(*reinterpret_cast<const uint4*>(xsm + off),
            *reinterpret_cast<const uint4*>(xsm + PL_BYTES + off),
            *reinterpret_cast<const uint4*>(xsm + 2 * PL_BYTES + off), xv);
    } else {
      const uint4 w = *reinterpret_cast<const uint4*>(xsm + off);
      const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        xv[2 * e] = bf_lo(ww[e]);
        xv[2 * e + 1] = bf_hi(ww[e]);
      }
    }
    const float4 c0 = *reinterpret_cast<const float4*>(cf + 8 * j);
    const float4 c1 = *reinterpret_cast<const float4*>(cf + 8 * j + 4);
    const float cv[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
    for (int e = 0; e < 8; ++e) acc = __fmaf_rn(xv[e], cv[e], acc);
  }
  return sq_dist(xx, acc, cc);
}

__global__ void __launch_bounds__(THREADS, 1)
k_assign_tc(const __grid_constant__ Params prm, const ac_cluster_problem* __restrict__ probs) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = align1024(smraw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool f32in = prm.dtype == AC_DTYPE_F32;
  const Layout& lay = prm.lay;
  const int XS = lay.xs;

  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + lay.off_bar);
  uint64_t* xfull = bars;       // [4] TMA -> converter (f32) / MMA (bf16)
  uint64_t* xempty = bars + 4;  // [4] converter (f32) / epilogue (bf16) -> TMA
  uint64_t* pfull = bars + 8;   // [2] converter -> MMA
  uint64_t* pempty = bars + 10; // [2] epilogue -> converter
  uint64_t* afull = bars + 12;  // [2] MMA commit -> epilogue
  uint64_t* aempty = bars + 14; // [2] epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + lay.off_misc);
  int* s_ccmax = reinterpret_cast<int*>(sm + lay.off_misc + 16);
  float* s_cc = reinterpret_cast<float*>(sm + lay.off_cc);
  int* s_hist = reinterpret_cast<int*>(sm + lay.off_hist);
  unsigned char* cplanes = sm + lay.off_cp;
  float* cf32 = reinterpret_cast<float*>(sm + lay.off_cf);
  const int CPB = lay.cp_bytes;

  if (tid == 0) {
    for (int s = 0; s < 4; ++s) {
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

    // ---- centres of this problem: bf16 planes (MMA), exact f32 rows
    //      (fix-up), ||c||^2 (+inf past nb, masking the pad columns) ----
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
        float4* dst = reinterpret_cast<float4*>(cf32 + c * CF_STRIDE + 8 * j);
        dst[0] = a;
        dst[1] = b;
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = 0.f;
      }
      uint4 h, m, l;
      split8(v, h, m, l);
      const int off = sw128(c, j);
      *reinterpret_cast<uint4*>(cplanes + off) = h;
      *reinterpret_cast<uint4*>(cplanes + CPB + off) = m;
      *reinterpret_cast<uint4*>(cplanes + 2 * CPB + off) = l;
    }
    for (int c = tid; c < NBMAX; c += THREADS) {
      const float cc = (c < nb) ? P.cc[c_lo + c] : INFINITY;
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
          if (g >= XS) mbar_wait_sleep(xempty + s, ((g / XS) - 1) & 1, 20);
          const int row = (t + i - ptile0) * BM;
          unsigned char* dst = sm + s * lay.xstride;
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
        // plane products kept: (x plane, c plane), the x-hi terms first (bf16
        // points are exact in plane 0, so they use only those three); the
        // dropped terms are < 2^-23 relative
        const int xi[6] = {0, 0, 0, 1, 1, 2};
        const int ci[6] = {0, 1, 2, 0, 1, 0};
        const int nterm = f32in ? 6 : 3;
        for (int i = 0; i < T; ++i) {
          const int g = g0 + i, s = g % XS, b = g & 1;
          if (f32in) mbar_wait_sleep(pfull + b, (g >> 1) & 1, 21);
          else mbar_wait_sleep(xfull + s, (g / XS) & 1, 22);
          if (g >= 2) mbar_wait_sleep(aempty + b, ((g >> 1) - 1) & 1, 23);
          fence_after();
          const uint32_t xa = f32in ? smem_u32(sm + lay.off_xp + b * 3 * PL_BYTES)
                                    : smem_u32(sm + s * PL_BYTES);
          const uint32_t d = tmem + (uint32_t)(b * 128);
#pragma unroll
          for (int term = 0; term < 6; ++term) {
            if (term >= nterm) break;
#pragma unroll
            for (int kk = 0; kk < DIM / 16; ++kk) {
              const uint64_t ad = sdesc(xa + xi[term] * PL_BYTES + kk * 32, 16, 1024);
              const uint64_t bd = sdesc(ca + ci[term] * CPB + kk * 32, 16, 1024);
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
          mbar_wait_sleep(xfull + s, (g / XS) & 1, 24);
          if (g >= 2) mbar_wait_sleep(pempty + b, ((g >> 1) - 1) & 1, 25);
          const unsigned char* xs = sm + s * XF_BYTES;
          unsigned char* xp = sm + lay.off_xp + b * 3 * PL_BYTES;
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
      // e_c = cc - 2 acc ~ d~_c - ||x||^2; candidates: max(xx + e_c, 0) <=
      // d~_min + 2T  <=>  e_c <= d~_min + 2T - xx (slack 0.5T for roundings)
      const int wg = (warp - W_EPI0) >> 2;
      const int q = warp & 3;  // TMEM lane quarter this warp may access
      const int r = q * 32 + lane;
      const uint32_t lane_base = (uint32_t)(q * 32) << 16;
      int* hist = s_hist + wg * NBMAX;
      int fixups = 0, wide = 0;
      for (int i = 0; i < T; ++i) {
        const int g = g0 + i;
        if ((g & 1) != wg) continue;
        const int b = wg, s = g % XS;
        const int tile = t + i - ptile0;
        const int64_t row = (int64_t)tile * BM + r;
        const bool valid = row < n;
        const float xx = valid ? P.xx[row] : 0.f;
        const float tb = 0x1p-15f * sqrtf(xx) * cmax + 0x1p-20f * (xx + ccmax) + 1e-30f;
        mbar_wait_sleep(afull + b, (g >> 1) & 1, 26);
        fence_after();
        const uint32_t acc_col = tmem + lane_base + (uint32_t)(b * 128);
        float emin = INFINITY;
        for (int c0 = 0; c0 < nbp; c0 += 32) {
          uint32_t v[32];
          tmem_ld32(acc_col + c0, v);
          tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < 32; ++u)
            emin = fminf(emin, __fmaf_rn(-2.f, __uint_as_float(v[u]), s_cc[c0 + u]));
        }
        const float dmin = fmaxf(xx + emin, 0.f);
        const float ethr = (dmin + 2.5f * tb) - xx;
        int c1 = INT_MAX, ncand = 0;
        uint32_t mk[NBMAX / 32];
#pragma unroll
        for (int ch = 0; ch < NBMAX / 32; ++ch) {
          mk[ch] = 0u;
          const int c0 = ch * 32;
          if (c0 >= nbp) continue;
          uint32_t v[32];
          tmem_ld32(acc_col + c0, v);
          tmem_wait_ld();
          uint32_t m = 0;
#pragma unroll
          for (int u = 0; u < 32; ++u)
            m |= (__fmaf_rn(-2.f, __uint_as_float(v[u]), s_cc[c0 + u]) <= ethr) ? (1u << u) : 0u;
          mk[ch] = m;
          if (m) {
            c1 = min(c1, c0 + __ffs(m) - 1);
            ncand += __popc(m);
          }
        }
        fence_before();
        mbar_arrive(aempty + b);

        // exact chains: every row's first candidate on its own lane, then the
        // warp's extra candidates (near-ties) spread over all 32 lanes
        const unsigned char* xsm = f32in ? sm + lay.off_xp + b * 3 * PL_BYTES : sm + s * PL_BYTES;
        float best = INFINITY;
        int lbl = INT_MAX;
        if (valid && ncand >= 1) {
          best = exact_dist(xsm, f32in, r, cf32 + c1 * CF_STRIDE, xx, s_cc[c1]);
          lbl = c1;
          if (!(best < INFINITY)) { best = INFINITY; lbl = INT_MAX; }  // as `d < best` from +inf
        }
        const int extra = (valid && ncand > 1) ? ncand - 1 : 0;
        int incl = extra;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        if (total > 0) {
          uint32_t* qe = reinterpret_cast<uint32_t*>(sm + lay.off_q) + (warp - W_EPI0) * 2 * QCAP;
          float* qr = reinterpret_cast<float*>(qe + QCAP);
          const int off = incl - extra;
          if (total <= QCAP) {
            int e = off;
#pragma unroll
            for (int ch = 0; ch < NBMAX / 32; ++ch) {
              uint32_t m = mk[ch];
              while (m) {
                const int c = ch * 32 + __ffs(m) - 1;
                m &= m - 1;
                if (c != c1) qe[e++] = ((uint32_t)lane << 8) | (uint32_t)c;
              }
            }
            __syncwarp();
            for (int e2 = lane; e2 < total; e2 += 32) {
              const int src = (int)(qe[e2] >> 8), c = (int)(qe[e2] & 255u);
              const int64_t srow = (int64_t)tile * BM + q * 32 + src;
              qr[e2] = exact_dist(xsm, f32in, q * 32 + src, cf32 + c * CF_STRIDE, P.xx[srow], s_cc[c]);
            }
            __syncwarp();
            for (int e2 = off; e2 < off + extra; ++e2) {  // ascending centre order
              const float d = qr[e2];
              if (d < best) { best = d; lbl = (int)(qe[e2] & 255u); }
            }
            __syncwarp();
          } else {  // very many near-ties in this warp: each lane walks its own
#pragma unroll
            for (int ch = 0; ch < NBMAX / 32; ++ch) {
              uint32_t m = mk[ch];
              while (m) {
                const int c = ch * 32 + __ffs(m) - 1;
                m &= m - 1;
                if (c == c1) continue;
                const float d = exact_dist(xsm, f32in, r, cf32 + c * CF_STRIDE, xx, s_cc[c]);
                if (d < best) { best = d; lbl = c; }
              }
            }
          }
        }
        if (valid) {
          fixups += (ncand >= 2);
          wide += (ncand > 2);
        }
        // x is no longer needed: release the planes / stage
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
      wide = __reduce_add_sync(0xffffffffu, wide);
      if (lane == 0 && fixups) atomicAdd(&P.status[AC_ST_FIXUPS], fixups);
      if (lane == 0 && wide) atomicAdd(&P.status[AC_ST_WIDE], wide);
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
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_MAX);
    if (e != cudaSuccess) return check_cuda(e, "k_assign_tc smem");
  }
  for (int p0 = 0; p0 < nprob; p0 += MAXP) {
    const int np = std::min(MAXP, nprob - p0);
    Params prm;
    memset(&prm, 0, sizeof(prm));
    int cap = 16;
    for (int j = 0; j < np; ++j)
      cap = std::max(cap, (host_probs[p0 + j].k - c_lo + 15) & ~15);
    prm.lay = make_layout(dtype, cap);
    if (prm.lay.smem > SMEM_MAX) {
      set_error("k_assign_tc: shared-memory layout %d B exceeds the budget", prm.lay.smem);
      return AC_ERR_PARAM;
    }
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
    k_assign_tc<<<grid, THREADS, prm.lay.smem, st>>>(prm, probs + p0);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return check_cuda(e, "k_assign_tc");
  }
  return AC_OK;
}

}  // namespace ac_host
