// K3 on the 5th-generation tensor cores: the Lloyd assignment step
// (clustering.py:68-97, `_pairwise_sq_dists` + `_assign`) as a tcgen05 GEMM
// with an exact fix-up epilogue.
//
// The reference computes d = (||x||^2 - 2 x·c) + ||c||^2 in f32 with
// OpenBLAS's sequential FMA chain for x·c, and takes the first-index argmin.
// Labels must be bit-identical (Lloyd is not converged at max_iter, so one
// flipped near-tie cascades — SURVEY.md §7 hard part 1).  Design:
//
//   1. e_c = ||c||^2 - 2 x·c on tcgen05 (kind::f16, f32 accumulation in
//      TMEM), D = 64 or 128 (D/64 SWIZZLE_128B K-atoms per row).  Centres
//      enter as three bf16 planes of -2c (exact split of f32), ||c||^2 as a
//      3-way split picked up by one extra K=16 MMA against a constant ones
//      block (SWIZZLE_32B operands); bf16 points are one exact plane (x times
//      the three centre planes), f32 points arrive as their exact hi/mid/lo
//      bf16 planes (written by the fused normalisation pass or
//      ac_lloyd_prepare) and the MMA runs the three largest products
//      hi·hi, hi·mid, mid·hi (all six with AC_ASG_F32_TERMS=6).
//   2. Epilogue, one thread per row (= TMEM lane): e_min and the candidate
//      mask e_c <= d~_min + 2.5T - ||x||^2 straight from TMEM, where T bounds
//      |d~ - d_ref| for every column (dropped split products, tensor-core
//      accumulation and the reference chain's own rounding).
//   3. Candidates of rows with more than one (every row's, when the caller
//      needs exact `best`) are recomputed with the reference's exact
//      sequential fmaf chain (x and c reconstructed exactly from shared
//      memory), one (row, candidate) per lane in a warp-wide pass, and the
//      first-index minimum of the exact values wins.
//
// So labels and distances equal k_assign_seq's (the all-FFMA kernel) bit
// for bit; tests/test_assign_tc.py checks exactly that, on adversarial ties.
//
// Warp roles (448 threads = NWG 3, or 320 = NWG 2; one CTA per SM, persistent
// over the tiles of a batch of problems):
//   warp 0      TMA producer: 128-row x tiles (1 or 3 planes) into a ring
//   warp 1      MMA issuer (single thread), TMEM owner (NWG x 128 columns)
//   warps 2..   NWG epilogue warpgroups, taking tiles round-robin (one TMEM
//               accumulator each): argmin, exact fix-up, labels / best /
//               per-tile label histogram (the tiling matches k_scatter).
// Compiled with --fmad=false: the fix-up reproduces numpy's unfused ops.
#include <cfloat>
#include <climits>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "tc_common.cuh"

namespace ac {
namespace asg {
using namespace ac::tc;

constexpr int BM = 128;     // rows per tile (== kAsgBM: shared tiling with the sort kernels)
constexpr int NBMAX = kAsgTcChunk;  // centres per problem per launch (k - c_lo)
constexpr int ATOM = BM * 128;  // one SW128 K-atom (64 bf16 columns) of a 128-row tile
constexpr int MAXP = 32;    // problems per launch (tensor maps travel as kernel params)
constexpr int W_TMA = 0, W_MMA = 1, W_EPI0 = 2;
constexpr int NWG_MAX = 4;  // epilogue warpgroups (one tile / TMEM accumulator each)
constexpr int threads_for(int nwg) { return 64 + 128 * nwg; }
constexpr int CF_STRIDE = 64 + 4;       // f32 centre rows (D = 64), padded against bank conflicts
constexpr int QCAP = 64;                // per-warp queue of extra (row, centre) fix-up candidates
constexpr int SMEM_MAX = 227 * 1024;
constexpr float kPadE = 3.0e38f;        // e of the padding columns (never a candidate)
constexpr int kNoHist = kAsgNoHist;     // internal flag: skip the per-tile label histogram

// Shared-memory layout, sized per launch from the largest centre count
// (cap = max round16(k - c_lo)):
//   x stages   XS x NP planes x [128 rows][64] bf16 (SW128, TMA-written);
//              NP = 1 for bf16 points (exact), 2 for f32 points (hi/mid: the
//              planes the three-product MMA reads; exact chains read the f32
//              row from global memory), 3 (hi/mid/lo) in the six-product form
//   centres    3 planes of -2c [cap][64] bf16 (SW128)
//   aug        A: [128][64] bf16 with columns 0..2 = 1;  B: [cap][64] with
//              columns 0..2 = the exact 3-way split of ||c||^2  -> one extra
//              K=16 MMA adds ||c||^2, so TMEM holds e_c = ||c||^2 - 2 x.c
//   exact      f32 centres [cap][68], ||c||^2 [128]
//   epilogue   two label histograms [2][128], fix-up queues [8][64] x 2 words
struct Layout {
  int np, xs, stage_bytes, off_cp, cp_bytes, off_aa, off_ab, off_cf, off_cc, off_hist, off_q,
      off_bar, off_misc, smem;
};

struct Params {
  CUtensorMap x[MAXP];
  int tile0[MAXP + 1];  // first tile of each problem (prefix of ceil(n/128))
  int nprob;
  int dtype;
  int c_lo;
  int c_hi;   // centres [c_lo, min(k, c_hi)) of each problem (chunked assignment)
  int flags;
  int f32_terms;  // split products for f32 points: 3 (default) or 6
  Layout lay;
};

// D = 64: exact f32 centres in shared memory; D = 128: the exact centres
// are re-joined from the -2c planes (no room for both)
#ifndef AC_ASG_X_GLOBAL
#define AC_ASG_X_GLOBAL 1  // 3-product f32 form: stage hi/mid only, exact chains read the f32 row
#endif
inline int f32_terms_env() {
  static const int t = getenv("AC_ASG_F32_TERMS") ? atoi(getenv("AC_ASG_F32_TERMS")) : 3;
  return t == 6 ? 6 : 3;
}
// bf16 planes of x staged per tile: bf16 points 1; f32 points hi/mid (the
// planes the three-product MMA reads; the exact chains then read the f32
// row from global memory) or hi/mid/lo (six products, or AC_ASG_X_GLOBAL=0)
__host__ __device__ inline int x_planes(int dtype, int terms) {
  if (dtype != AC_DTYPE_F32) return 1;
  return (AC_ASG_X_GLOBAL && terms != 6) ? 2 : 3;
}
__host__ __device__ inline Layout make_layout(int dtype, int dim, int cap, int xs, int terms) {
  Layout l;
  const int kb = dim / 64;
  l.np = x_planes(dtype, terms);
  l.xs = xs;
  l.stage_bytes = l.np * kb * ATOM;
  l.off_cp = l.xs * l.stage_bytes;
  l.cp_bytes = kb * cap * 128;
  l.off_aa = l.off_cp + 3 * l.cp_bytes;
  l.off_ab = l.off_aa + BM * 32;   // aug operands: one K=16 step, SWIZZLE_32B
  l.off_cf = l.off_ab + cap * 32;
  l.off_cc = l.off_cf + (dim == 64 ? cap * CF_STRIDE * 4 : 0);
  l.off_hist = l.off_cc + NBMAX * 4;
  l.off_q = l.off_hist + NWG_MAX * NBMAX * 4;
  l.off_bar = l.off_q + 4 * NWG_MAX * QCAP * 8;
  l.off_misc = l.off_bar + 16 * 8;
  l.smem = l.off_misc + 32 + 4 * (MAXP + 1) + 1024;  // + alignment slack
  return l;
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

// the reference's d for row r of the x tile and centre c: sequential fmaf
// chain from 0 (OpenBLAS general path), then sq_dist.  x comes from the
// tile's planes in shared memory (exactly joined); c from the f32 rows
// (D = 64) or re-joined from the -2c planes (exact, times -1/2).
template <int DIM>
AC_DEV float exact_dist(const unsigned char* xsm, bool f32in, int r, const float* cf,
                        const unsigned char* cp, int cpb, int cap, int c, float xx, float cc,
                        const float* __restrict__ xg = nullptr) {
  constexpr int PLB = BM * DIM * 2;
  constexpr int UNR = DIM == 64 ? 8 : 2;  // bounded register footprint at D = 128
  float acc = 0.f;
#pragma unroll UNR
  for (int j = 0; j < DIM / 8; ++j) {
    const int off = (j >> 3) * ATOM + sw128(r, j & 7);
    float xv[8];
    if (xg) {  // the f32 row itself (global memory / L2)
      const float4 a = __ldg(reinterpret_cast<const float4*>(xg + 8 * j));
      const float4 b = __ldg(reinterpret_cast<const float4*>(xg + 8 * j + 4));
      xv[0] = a.x; xv[1] = a.y; xv[2] = a.z; xv[3] = a.w;
      xv[4] = b.x; xv[5] = b.y; xv[6] = b.z; xv[7] = b.w;
    } else if (f32in) {
      join8(*reinterpret_cast<const uint4*>(xsm + off),
            *reinterpret_cast<const uint4*>(xsm + PLB + off),
            *reinterpret_cast<const uint4*>(xsm + 2 * PLB + off), xv);
    } else {
      const uint4 w = *reinterpret_cast<const uint4*>(xsm + off);
      const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        xv[2 * e] = bf_lo(ww[e]);
        xv[2 * e + 1] = bf_hi(ww[e]);
      }
    }
    float cv[8];
    if constexpr (DIM == 64) {
      const float4 c0 = *reinterpret_cast<const float4*>(cf + 8 * j);
      const float4 c1 = *reinterpret_cast<const float4*>(cf + 8 * j + 4);
      cv[0] = c0.x; cv[1] = c0.y; cv[2] = c0.z; cv[3] = c0.w;
      cv[4] = c1.x; cv[5] = c1.y; cv[6] = c1.z; cv[7] = c1.w;
    } else {
      const int coff = (j >> 3) * cap * 128 + sw128(c, j & 7);
      join8(*reinterpret_cast<const uint4*>(cp + coff), *reinterpret_cast<const uint4*>(cp + cpb + coff),
            *reinterpret_cast<const uint4*>(cp + 2 * cpb + coff), cv);
#pragma unroll
      for (int e = 0; e < 8; ++e) cv[e] = __fmul_rn(-0.5f, cv[e]);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) acc = __fmaf_rn(xv[e], cv[e], acc);
  }
  return sq_dist(xx, acc, cc);
}

AC_DEV void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// NWG = 2: 320 threads (<= 168 registers); NWG = 3: 448 threads, compiled
// for 512 (<= 128 registers: 4 warps share an SM sub-partition's 64 KB file)
template <int DIM, int NWG>
__global__ void __launch_bounds__(NWG == 2 ? 320 : (NWG == 3 ? 512 : 576), 1)
k_assign_tc(const __grid_constant__ Params prm, const ac_cluster_problem* __restrict__ probs) {
  pdl_wait();
  pdl_trigger();
  constexpr int THREADS = threads_for(NWG);
  constexpr int KB = DIM / 64;           // SW128 K-atoms per row
  constexpr int PL_BYTES = KB * ATOM;    // one bf16 plane of a tile
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool f32in = prm.dtype == AC_DTYPE_F32;
  const Layout& lay = prm.lay;
  const int XS = lay.xs, NP = lay.np, SB = lay.stage_bytes, CPB = lay.cp_bytes;

  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + lay.off_bar);
  uint64_t* xfull = bars;        // [4] TMA -> MMA
  uint64_t* xempty = bars + 4;   // [4] epilogue -> TMA
  uint64_t* afull = bars + 8;          // [NWG] MMA commit -> epilogue
  uint64_t* aempty = bars + 8 + NWG;   // [NWG] epilogue -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + lay.off_misc);
  int* s_ccmax = reinterpret_cast<int*>(sm + lay.off_misc + 16);
  float* s_cc = reinterpret_cast<float*>(sm + lay.off_cc);
  int* s_hist = reinterpret_cast<int*>(sm + lay.off_hist);
  unsigned char* cplanes = sm + lay.off_cp;
  unsigned char* aug_a = sm + lay.off_aa;
  unsigned char* aug_b = sm + lay.off_ab;
  float* cf32 = reinterpret_cast<float*>(sm + lay.off_cf);

  if (tid == 0) {
    for (int s = 0; s < 4; ++s) {
      mbar_init(xfull + s, 1);
      mbar_init(xempty + s, 128);
    }
    for (int b = 0; b < NWG; ++b) {
      mbar_init(afull + b, 1);
      mbar_init(aempty + b, 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  // aug A: rows of (1, 1, 1, 0, ...): picks up the 3-way split of ||c||^2
  for (int e = tid; e < BM * 2; e += THREADS) {
    const int r = e >> 1, j = e & 1;
    uint4 w = make_uint4(0u, 0u, 0u, 0u);
    if (j == 0) w = make_uint4(0x3f803f80u, 0x00003f80u, 0u, 0u);  // bf16 1.0 = 0x3f80
    *reinterpret_cast<uint4*>(aug_a + sw32(r, j)) = w;
  }
  if (warp == W_MMA) tmem_alloc(tmem_slot, NWG == 2 ? 256 : 512);
  fence_proxy_async();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  // The tiles are split evenly over the CTAs counting only problems with
  // work in this launch (Lloyd-converged problems and problems without a
  // centre in this chunk contribute none), so converged heads shorten the
  // launch instead of idling the CTAs they were statically assigned to.
  // Every CTA derives the same prefix from the device-side status words.
  int* s_act0 = reinterpret_cast<int*>(sm + lay.off_misc + 32);  // [MAXP + 1]
  if (tid < prm.nprob) {  // one thread per problem: the loads run in parallel
    const ac_cluster_problem& Q = probs[tid];
    const bool act = ((prm.flags & AC_ASSIGN_ALL) || Q.status[AC_ST_ACTIVE] != 0) &&
                     min(Q.k, prm.c_hi) - prm.c_lo >= 1;
    s_act0[tid + 1] = act ? prm.tile0[tid + 1] - prm.tile0[tid] : 0;
  }
  __syncthreads();
  if (tid == 0) {
    s_act0[0] = 0;
    for (int q = 0; q < prm.nprob; ++q) s_act0[q + 1] += s_act0[q];
  }
  __syncthreads();
  const int total = s_act0[prm.nprob];
  const int t_begin = (int)((int64_t)blockIdx.x * total / gridDim.x);
  const int t_end = (int)((int64_t)(blockIdx.x + 1) * total / gridDim.x);
  int g0 = 0;  // CTA-local sequence number of the segment's first tile
  int p = 0;
  for (int t = t_begin; t < t_end;) {
    while (s_act0[p + 1] <= t) ++p;
    const int seg_end = min(t_end, s_act0[p + 1]);
    const ac_cluster_problem& P = probs[p];
    const int k = P.k, c_lo = prm.c_lo, nb = min(k, prm.c_hi) - c_lo;
    const int nbp = max(16, (nb + 15) & ~15);
    const int64_t n = P.n;
    const int ptile0 = s_act0[p];                            // virtual (active-only) numbering
    const int ntiles_p = prm.tile0[p + 1] - prm.tile0[p];    // the problem's real tile count
    const int T = seg_end - t;

    // ---- centres of this problem: -2c planes and ||c||^2 split (MMA),
    //      exact f32 rows and ||c||^2 (fix-up) ----
    if (tid == 0) *s_ccmax = 0;
    __syncthreads();
    const int cap = CPB / (KB * 128);  // centre rows per plane atom
    for (int e = tid; e < nbp * (DIM / 8); e += THREADS) {
      const int c = e / (DIM / 8), j = e % (DIM / 8);
      float v[8];
      if (c < nb) {
        const float4* src = reinterpret_cast<const float4*>(P.centers + (int64_t)(c_lo + c) * DIM + 8 * j);
        const float4 a = src[0], b = src[1];
        if constexpr (DIM == 64) {
          float4* dst = reinterpret_cast<float4*>(cf32 + c * CF_STRIDE + 8 * j);
          dst[0] = a;
          dst[1] = b;
        }
        v[0] = -2.f * a.x; v[1] = -2.f * a.y; v[2] = -2.f * a.z; v[3] = -2.f * a.w;
        v[4] = -2.f * b.x; v[5] = -2.f * b.y; v[6] = -2.f * b.z; v[7] = -2.f * b.w;
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = 0.f;
      }
      uint4 h, m, l;
      split8(v, h, m, l);
      const int off = (j >> 3) * cap * 128 + sw128(c, j & 7);
      *reinterpret_cast<uint4*>(cplanes + off) = h;
      *reinterpret_cast<uint4*>(cplanes + CPB + off) = m;
      *reinterpret_cast<uint4*>(cplanes + 2 * CPB + off) = l;
    }
    for (int c = tid; c < NBMAX; c += THREADS) {
      const float cc = (c < nb) ? P.cc[c_lo + c] : INFINITY;
      s_cc[c] = cc;
      if (c < nb && cc > 0.f) atomicMax(s_ccmax, __float_as_int(cc));
      if (c < nbp) {
        // ||c||^2 split into columns 0..2 of the aug B row; padding rows get
        // a huge e so that they are never a minimum or a candidate
        const float v0 = (c < nb) ? cc : kPadE;
        const __nv_bfloat16 h0 = __float2bfloat16_rn(v0);
        const float r1 = __fsub_rn(v0, __bfloat162float(h0));
        const __nv_bfloat16 h1 = __float2bfloat16_rn(r1);
        const __nv_bfloat16 h2 = __float2bfloat16_rn(__fsub_rn(r1, __bfloat162float(h1)));
        const uint32_t w0 = (uint32_t)__bfloat16_as_ushort(h0) | ((uint32_t)__bfloat16_as_ushort(h1) << 16);
        const uint32_t w1 = (uint32_t)__bfloat16_as_ushort(h2);
        *reinterpret_cast<uint4*>(aug_b + sw32(c, 0)) = make_uint4(w0, w1, 0u, 0u);
        *reinterpret_cast<uint4*>(aug_b + sw32(c, 1)) = make_uint4(0u, 0u, 0u, 0u);
      }
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
          unsigned char* dst = sm + s * SB;
          mbar_expect_tx(xfull + s, SB);
          for (int q = 0; q < NP; ++q)
#pragma unroll
            for (int kb = 0; kb < KB; ++kb)
              tma_load_2d(dst + q * PL_BYTES + kb * ATOM, &prm.x[p], kb * 64, (int)(q * n) + row,
                          xfull + s);
        }
      }
      __syncwarp();
    } else if (warp == W_MMA) {
      // ------------------------------ MMA issuer --------------------------------
      if (lane == 0) {
        const uint32_t idesc = idesc_bf16(BM, nbp, false);
        const uint32_t ca = smem_u32(cplanes);
        const uint32_t aa = smem_u32(aug_a), ab = smem_u32(aug_b);
        // plane products kept, (x plane, c plane): bf16 points are exact in
        // plane 0 -> x.c_hi, x.c_mid, x.c_lo (the exact product); f32 points
        // -> the three largest, hi.hi, hi.mid, mid.hi (the dropped ones are
        // < 3.02*2^-18 sum|x_i c'_i|, covered by the widened epilogue bound),
        // or all six with AC_ASG_F32_TERMS=6 (dropped < 2^-26)
        const bool six = f32in && prm.f32_terms == 6;
        const int xi[6] = {0, 0, f32in ? 1 : 0, 0, 1, 2};
        const int ci[6] = {0, 1, f32in ? 0 : 2, 2, 1, 0};
        const int nterm = six ? 6 : 3;
        for (int i = 0; i < T; ++i) {
          const int g = g0 + i, s = g % XS, b = g % NWG;
          mbar_wait_sleep(xfull + s, (g / XS) & 1, 22);
          if (g >= NWG) mbar_wait_sleep(aempty + b, ((g / NWG) - 1) & 1, 23);
          fence_after();
          const uint32_t xa = smem_u32(sm + s * SB);
          const uint32_t d = tmem + (uint32_t)(b * 128);
          // ||c||^2 first (one K=16 step of the aug operands), then -2 x.c
          umma_f16(d, sdesc_sw32(aa), sdesc_sw32(ab), idesc, 0u);
#pragma unroll
          for (int term = 0; term < 6; ++term) {
            if (term >= nterm) break;
#pragma unroll
            for (int kk = 0; kk < DIM / 16; ++kk) {
              const uint32_t kx = (kk >> 2) * ATOM + (kk & 3) * 32;
              const uint32_t kc = (kk >> 2) * (CPB / KB) + (kk & 3) * 32;
              const uint64_t ad = sdesc(xa + xi[term] * PL_BYTES + kx, 16, 1024);
              const uint64_t bd = sdesc(ca + ci[term] * CPB + kc, 16, 1024);
              umma_f16(d, ad, bd, idesc, 1u);
            }
          }
          umma_commit(afull + b);
        }
      }
      __syncwarp();
    } else {
      // ------------------------------ epilogue ------------------------------
      // TMEM holds e_c ~ ||c||^2 - 2 x.c = d~_c - ||x||^2.  Candidates:
      // max(xx + e_c, 0) <= d~_min + 2T  <=>  e_c <= d~_min + 2T - xx
      // (slack 0.5T for the roundings of the comparison itself)
      const int wg = (warp - W_EPI0) >> 2;
      const int q = warp & 3;  // TMEM lane quarter this warp may access
      const int r = q * 32 + lane;
      const uint32_t lane_base = (uint32_t)(q * 32) << 16;
      int* hist = s_hist + wg * NBMAX;
      uint32_t* qe = reinterpret_cast<uint32_t*>(sm + lay.off_q) + (warp - W_EPI0) * 2 * QCAP;
      float* qr = reinterpret_cast<float*>(qe + QCAP);
      const int nch = nbp >> 4;  // 16-column chunks
      int fixups = 0, wide = 0;
      // ||x||^2 of this warpgroup's next tile, prefetched one tile ahead
      auto load_xx = [&](int i) -> float {
        const int64_t rw = (int64_t)(t + i - ptile0) * BM + r;
        return (i < T && rw < n) ? P.xx[rw] : 0.f;
      };
      const int i_first = (wg - g0 % NWG + NWG) % NWG;
      float xx_next = load_xx(i_first);
      for (int i = i_first; i < T; i += NWG) {
        const int g = g0 + i;
        const int b = wg, s = g % XS;
        const int tile = t + i - ptile0;
        const int64_t row = (int64_t)tile * BM + r;
        const bool valid = row < n;
        const float xx = xx_next;
        xx_next = load_xx(i + NWG);
        // |e~ - e_ref| <= tb for every column (assignment); with
        // only three split products for f32 points, + 0x1.9p-16 ||x|| cmax
        const float tb = (0x1p-15f + (f32in && prm.f32_terms != 6 ? 0x1.9p-16f : 0.f)) * sqrtf(xx) * cmax +
                         0x1p-17f * (xx + ccmax) + 1e-30f;
        mbar_wait_sleep(afull + b, (g / NWG) & 1, 26);
        fence_after();
        const uint32_t acc_col = tmem + lane_base + (uint32_t)(b * 128);
        float m4[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
        for (int ch = 0; ch < nch; ++ch) {
          uint32_t v[16];
          tmem_ld16(acc_col + ch * 16, v);
          tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < 16; u += 4)
#pragma unroll
            for (int a = 0; a < 2; ++a)
              m4[a + 2 * (u >> 3)] = fminf(m4[a + 2 * (u >> 3)],
                                           fminf(__uint_as_float(v[u + 2 * a]), __uint_as_float(v[u + 2 * a + 1])));
        }
        const float emin = fminf(fminf(m4[0], m4[1]), fminf(m4[2], m4[3]));
        const float dmin = fmaxf(xx + emin, 0.f);
        const float ethr = (dmin + 2.5f * tb) - xx;
        int c1 = INT_MAX, ncand = 0;
        uint32_t mk[NBMAX / 32] = {0u, 0u, 0u, 0u};
#pragma unroll
        for (int ch = 0; ch < NBMAX / 16; ++ch) {
          if (ch >= nch) break;
          uint32_t v[16];
          tmem_ld16(acc_col + ch * 16, v);
          tmem_wait_ld();
          // four independent partial masks (short dependency chains)
          uint32_t mq[4] = {0u, 0u, 0u, 0u};
#pragma unroll
          for (int u = 0; u < 16; ++u) mq[u & 3] |= (__uint_as_float(v[u]) <= ethr) ? (1u << u) : 0u;
          mk[ch >> 1] |= ((mq[0] | mq[1]) | (mq[2] | mq[3])) << ((ch & 1) * 16);
        }
#pragma unroll
        for (int w = NBMAX / 32 - 1; w >= 0; --w) {
          if (mk[w]) c1 = w * 32 + __ffs(mk[w]) - 1;  // lowest set bit overall
          ncand += __popc(mk[w]);
        }
        fence_before();
        mbar_arrive(aempty + b);

        // exact chains, one per (row, candidate) that needs one, spread over
        // all 32 lanes of the warp (a row whose single candidate is already
        // decided needs none when only labels are asked for)
        const unsigned char* xsm = sm + s * SB;
        const float* xglob = (f32in && NP == 2) ? reinterpret_cast<const float*>(P.x) : nullptr;
        const bool lonly = (prm.flags & AC_ASSIGN_LABELS_ONLY) != 0;
        float best = INFINITY;
        int lbl = INT_MAX;
        if (valid && ncand == 1 && lonly) {
          best = dmin;  // the label is decided; `best` approximate (see AC_ASSIGN_LABELS_ONLY)
          lbl = c1;
        }
        const int cnt = (valid && (ncand >= 2 || (ncand == 1 && !lonly))) ? ncand : 0;
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        const int total = __shfl_sync(0xffffffffu, incl, 31);
        if (total > 0) {
          const int off = incl - cnt;
          if (total <= QCAP) {
            if (cnt) {
              int e = off;
#pragma unroll
              for (int ch = 0; ch < NBMAX / 32; ++ch) {
                uint32_t m = mk[ch];
                while (m) {
                  qe[e++] = ((uint32_t)lane << 8) | (uint32_t)(ch * 32 + __ffs(m) - 1);
                  m &= m - 1;
                }
              }
            }
            __syncwarp();
            for (int base = 0; base < total; base += 32) {
              const int e2 = base + lane;
              const uint32_t ent = e2 < total ? qe[e2] : 0u;
              const int src = (int)(ent >> 8), c = (int)(ent & 255u);
              const float xs = __shfl_sync(0xffffffffu, xx, src);
              if (e2 < total)
                qr[e2] = exact_dist<DIM>(xsm, f32in, q * 32 + src, cf32 + c * CF_STRIDE, cplanes, CPB,
                                         CPB / (KB * 128), c, xs, s_cc[c],
                                         xglob ? xglob + ((int64_t)tile * BM + q * 32 + src) * DIM : nullptr);
            }
            __syncwarp();
            for (int e2 = off; e2 < off + cnt; ++e2) {  // ascending centre order, first wins
              const float d = qr[e2];
              if (d < best) { best = d; lbl = (int)(qe[e2] & 255u); }
            }
            __syncwarp();
          } else if (cnt) {  // very many near-ties in this warp: each lane walks its own
#pragma unroll
            for (int ch = 0; ch < NBMAX / 32; ++ch) {
              uint32_t m = mk[ch];
              while (m) {
                const int c = ch * 32 + __ffs(m) - 1;
                m &= m - 1;
                const float d = exact_dist<DIM>(xsm, f32in, r, cf32 + c * CF_STRIDE, cplanes, CPB,
                                                CPB / (KB * 128), c, xx, s_cc[c],
                                                xglob ? xglob + row * DIM : nullptr);
                if (d < best) { best = d; lbl = c; }
              }
            }
          }
        }
        if (valid) {
          fixups += (ncand >= 2);
          wide += (ncand > 2);
        }
        // x is no longer needed: release the stage
        mbar_arrive(xempty + s);

        int label = (lbl == INT_MAX) ? c_lo : c_lo + lbl;
        if (valid) {
          if (prm.flags & AC_ASSIGN_MERGE) {
            const float eb = P.best[row];
            if (!(best < eb)) { best = eb; label = P.labels[row]; }
          }
          P.labels[row] = label;
          P.best[row] = best;
        }
        if (!(prm.flags & (AC_ASSIGN_MERGE | kNoHist))) {
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
    tmem_dealloc(tmem, NWG == 2 ? 256 : 512);
  }
}

}  // namespace asg
}  // namespace ac

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
namespace ac_host {

static int tc_cap(const ac_cluster_problem* host_probs, int nprob, int c_lo, int c_hi) {
  int cap = 16;
  for (int j = 0; j < nprob; ++j)
    cap = std::max(cap, (std::min(host_probs[j].k, c_hi) - c_lo + 15) & ~15);
  return cap;
}

// Can the tensor-core kernel take this batch?  (D = 64 or 128, general-path
// accumulation order, <= 128 centres in [c_lo, c_hi), 16-byte aligned rows,
// and a shared-memory layout with at least one x stage.)
bool assign_tc_eligible(const ac_cluster_problem* host_probs, int nprob, int dtype, int d,
                        int c_lo, int order, int c_hi) {
  if (!host_probs || order != AC_ORDER_SEQ || (d != 64 && d != 128)) return false;
  if (dtype != AC_DTYPE_F32 && dtype != AC_DTYPE_BF16) return false;
  bool any = false;
  for (int p = 0; p < nprob; ++p) {
    const ac_cluster_problem& P = host_probs[p];
    const int nb = std::min(P.k, c_hi) - c_lo;
    if (nb > ac::asg::NBMAX) return false;
    any |= nb >= 1;
    if ((reinterpret_cast<uintptr_t>(P.x) & 15) || (reinterpret_cast<uintptr_t>(P.centers) & 15))
      return false;
    // f32 points are read as their exact bf16 planes (written by ac_lloyd_prepare)
    if (dtype == AC_DTYPE_F32 && (!P.planes || (reinterpret_cast<uintptr_t>(P.planes) & 15)))
      return false;
  }
  if (!any) return false;
  for (int p0 = 0; p0 < nprob; p0 += ac::asg::MAXP) {
    const int cap = tc_cap(host_probs + p0, std::min(ac::asg::MAXP, nprob - p0), c_lo, c_hi);
    if (ac::asg::make_layout(dtype, d, cap, 1, ac::asg::f32_terms_env()).smem > ac::asg::SMEM_MAX)
      return false;
  }
  return true;
}

int assign_tc_launch(const ac_cluster_problem* probs, const ac_cluster_problem* host_probs,
                     int nprob, int dtype, int d, int c_lo, int flags, cudaStream_t st, int c_hi) {
  using namespace ac::asg;
  const int sms = ac_host::sm_count();
  for (const void* f : {(const void*)k_assign_tc<64, 2>, (const void*)k_assign_tc<128, 2>,
                        (const void*)k_assign_tc<64, 3>, (const void*)k_assign_tc<128, 3>,
                        (const void*)k_assign_tc<64, 4>, (const void*)k_assign_tc<128, 4>}) {
    const int rc = ac_host::func_smem(f, SMEM_MAX, "k_assign_tc smem");
    if (rc) return rc;
  }
  for (int p0 = 0; p0 < nprob; p0 += MAXP) {
    const int np = std::min(MAXP, nprob - p0);
    Params prm;
    memset(&prm, 0, sizeof(prm));
    const int cap = tc_cap(host_probs + p0, np, c_lo, c_hi);
    int xs = 4;
    prm.f32_terms = f32_terms_env();
    while (xs > 1 && make_layout(dtype, d, cap, xs, prm.f32_terms).smem > SMEM_MAX) --xs;
    prm.lay = make_layout(dtype, d, cap, xs, prm.f32_terms);
    if (prm.lay.smem > SMEM_MAX) {
      set_error("k_assign_tc: shared-memory layout %d B exceeds the budget", prm.lay.smem);
      return AC_ERR_PARAM;
    }
    prm.nprob = np;
    prm.dtype = dtype;
    prm.c_lo = c_lo;
    prm.c_hi = c_hi;
    prm.flags = flags;
    prm.tile0[0] = 0;
    for (int j = 0; j < np; ++j) {
      const ac_cluster_problem& P = host_probs[p0 + j];
      const int64_t tiles = (P.n + BM - 1) / BM;
      prm.tile0[j + 1] = prm.tile0[j] + (int)tiles;
      // bf16 points: the tile itself; f32 points: the [3][n][d] planes.
      // Box = one 64-column SW128 atom; the kernel issues d/64 boxes per plane.
      const void* base = dtype == AC_DTYPE_F32 ? P.planes : P.x;
      const int64_t rows = (dtype == AC_DTYPE_F32 ? 3 : 1) * std::max<int64_t>(P.n, 1);  // map spans all planes
      int rc = make_map_2d(&prm.x[j], base, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, rows, d, 64, BM);
      if (rc) return rc;
    }
    const int total = prm.tile0[np];
    if (total == 0) continue;
    const int grid = std::min(total, sms);
    // 3 epilogue warpgroups (measured faster than 2 for both dtypes once the
    // f32 MMA runs three split products); AC_ASG_WG=2 selects the 320-thread form
    // epilogue warpgroups: 4 at D = 64 (measured -0.27 ms per C2 step: more
    // warps hide the epilogue's latency chains), 3 at D = 128 (4 spill there);
    // AC_ASG_WG overrides
    static const int env_wg = getenv("AC_ASG_WG") ? atoi(getenv("AC_ASG_WG")) : 0;
    const int nwg = (env_wg >= 2 && env_wg <= 4) ? env_wg : (d == 64 ? 4 : 3);
    if (nwg == 4) {
      if (d == 64) ac_host::launch_pdl(k_assign_tc<64, 4>, dim3(grid), dim3(threads_for(4)), prm.lay.smem, st, prm, probs + p0);
      else ac_host::launch_pdl(k_assign_tc<128, 4>, dim3(grid), dim3(threads_for(4)), prm.lay.smem, st, prm, probs + p0);
    } else if (nwg == 2) {
      if (d == 64) ac_host::launch_pdl(k_assign_tc<64, 2>, dim3(grid), dim3(threads_for(2)), prm.lay.smem, st, prm, probs + p0);
      else ac_host::launch_pdl(k_assign_tc<128, 2>, dim3(grid), dim3(threads_for(2)), prm.lay.smem, st, prm, probs + p0);
    } else {
      if (d == 64) ac_host::launch_pdl(k_assign_tc<64, 3>, dim3(grid), dim3(threads_for(3)), prm.lay.smem, st, prm, probs + p0);
      else ac_host::launch_pdl(k_assign_tc<128, 3>, dim3(grid), dim3(threads_for(3)), prm.lay.smem, st, prm, probs + p0);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return check_cuda(e, "k_assign_tc");
  }
  return AC_OK;
}

}  // namespace ac_host
