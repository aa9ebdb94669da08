// Block-sparse flash attention for head_dim 128 on the 5th-generation tensor
// cores: two query tiles per CTA, P aliased into S, anti-phase MMA schedule.
//
// Reference semantics: pipeline.py:154-165 (_gathered_attention) and
// reference.py:25-45 (full_attention) -- every query cluster attends, with a
// plain max-subtracted softmax (scale 1/sqrt(D)), over the union of its
// selected key clusters, stored cluster-contiguous as [start, end) runs of
// Kp/Vp and walked in 128-key tiles (keys past a run's end are masked).
//
// One CTA = one work item = up to 256 query rows (two 128-row Q tiles) of
// one query cluster, sharing every K/V tile:
//   warps 0-3 / 4-7   softmax of Q tile 0 / 1 (thread = query row = TMEM lane)
//   warp 8            TMA: Q0/Q1 once, K/V tiles through a 2-stage ring
//                     (each 128-column row = two SWIZZLE_128B atoms)
//   warp 9            MMA issuer
// TMEM (512 columns): S0 | S1 | O0 | O1, 128 columns each; the softmax writes
// P_t (bf16, 64 packed columns) over the consumed S_t, so S_t(j+1) waits for
// PV_t(j) to complete.  The MMA issue order is anti-phase
//     S0(0) | PV1(j-1) S1(j) | PV0(j) S0(j+1) | ...
// so that while one tile's softmax runs, the tensor core drains the other
// tile's PV and computes its next S.  At D = 128 the exponentials (1024
// clk/tile on the MUFU) and the MMAs (~1080 clk/tile) are balanced.
#include <cfloat>

#include "attn_common.cuh"

namespace ac {
namespace f128 {
using namespace ac::tc;
using namespace ac::attn;

constexpr int D = 128;
constexpr int KB = D / 64;  // SW128 atoms per row
constexpr int BM = 128;
constexpr int BN = 128;
constexpr int STAGES = 2;
constexpr int THREADS = 320;
constexpr int W_TMA = 8, W_MMA = 9;
constexpr int ATOM_Q = BM * 128;   // one 64-column atom of a Q tile
constexpr int ATOM_KV = BN * 128;  // one 64-column atom of a K/V tile
constexpr int Q_BYTES = KB * ATOM_Q;
constexpr int KV_BYTES = KB * ATOM_KV;
constexpr int OFF_Q = 0;
constexpr int OFF_K = OFF_Q + 2 * Q_BYTES;
constexpr int OFF_V = OFF_K + STAGES * KV_BYTES;
constexpr int OFF_BAR = OFF_V + STAGES * KV_BYTES;
constexpr int NBAR = 1 + 2 * STAGES + 2 + 2 + 2;
constexpr int OFF_MISC = OFF_BAR + NBAR * 8;
constexpr int SMEM = OFF_MISC + 16 + 1024;
constexpr uint32_t COL_S = 0, COL_O = 256;
#ifndef AC_F128_POLY
#define AC_F128_POLY 1  // of every 8 exp2 pairs, this many on the FMA pipe (polynomial)
#endif
#ifndef AC_F128_INORDER
// 1: S_t(j+1) is issued right behind PV_t(j) without waiting for its
// completion -- tcgen05.mma ops of one thread execute in issue order, so the
// S write lands after PV's read of the aliased P columns; the softmax's
// s_full commit still covers PV_t(j) (a commit tracks all prior MMAs)
#define AC_F128_INORDER 1
#endif

__global__ void __launch_bounds__(THREADS, 1)
k_attn_fa4_d128(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmk,
                const __grid_constant__ CUtensorMap tmv, const int32_t* __restrict__ qidx, int64_t L,
                const ac_attn_item* __restrict__ items, const int32_t* __restrict__ runs,
                float scale_log2, void* __restrict__ out, int out_dtype) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  const ac_attn_item it = items[blockIdx.x];
  if (it.q_rows <= 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool two = it.q_rows > BM;
  const int ntile = two ? 2 : 1;

  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = bars + 1 + STAGES;
  uint64_t* s_full = bars + 1 + 2 * STAGES;  // [2] S_t in TMEM
  uint64_t* p_full = s_full + 2;             // [2] P_t in TMEM (128 arrivals)
  uint64_t* o_done = s_full + 4;             // [2] PV_t complete (S_t/P_t columns free)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + OFF_MISC);

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(kv_full + s, 1);
      mbar_init(kv_empty + s, 1);
    }
    for (int t = 0; t < 2; ++t) {
      // only warps holding at least one real query row take part
      const int live = 32 * max(1, min(4, (min(BM, it.q_rows - t * BM) + 31) / 32));
      mbar_init(s_full + t, 1);
      mbar_init(p_full + t, live);
      mbar_init(o_done + t, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == W_MMA) tmem_alloc(tmem_slot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const int32_t* iruns = runs + 2 * it.run0;
  const int64_t krow0 = (int64_t)it.head * L;

  if (warp == W_TMA) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      mbar_expect_tx(q_full, ntile * Q_BYTES);
      for (int t = 0; t < ntile; ++t)
#pragma unroll
        for (int kb = 0; kb < KB; ++kb)
          tma_load_2d(sm + OFF_Q + t * Q_BYTES + kb * ATOM_Q, &tmq, kb * 64, (int)it.q_row0 + t * BM,
                      q_full);
      TileIter ti(iruns, it.nruns);
      int start, nk;
      for (int j = 0; ti.next(start, nk); ++j) {
        const int st = j % STAGES;
        if (j >= STAGES) mbar_wait_sleep(kv_empty + st, ((j / STAGES) - 1) & 1, 70);
        mbar_expect_tx(kv_full + st, 2 * KV_BYTES);
        const int row = (int)(krow0 + start);
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
          tma_load_2d(sm + OFF_K + st * KV_BYTES + kb * ATOM_KV, &tmk, kb * 64, row, kv_full + st);
          tma_load_2d(sm + OFF_V + st * KV_BYTES + kb * ATOM_KV, &tmv, kb * 64, row, kv_full + st);
        }
      }
    }
    __syncwarp();
  } else if (warp == W_MMA) {
    // ------------------------------ MMA issuer --------------------------------
    if (lane == 0) {
      constexpr uint32_t IS = idesc_bf16(BM, BN, false);
      constexpr uint32_t IO = idesc_bf16(BM, D, true);
      const uint32_t sq = smem_u32(sm + OFF_Q);
      auto issue_s = [&](int t, int st) {
        const uint32_t sk = smem_u32(sm + OFF_K + st * KV_BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t ko = (kk >> 2) * ATOM_Q + (kk & 3) * 32;
          const uint64_t ad = sdesc(sq + t * Q_BYTES + ko, 16, 1024);
          const uint64_t bd = sdesc(sk + (kk >> 2) * ATOM_KV + (kk & 3) * 32, 16, 1024);
          umma_f16(tmem + COL_S + t * BN, ad, bd, IS, kk > 0 ? 1u : 0u);
        }
        umma_commit(s_full + t);
      };
      auto issue_pv = [&](int t, int j, int st) {
        mbar_wait_sleep(p_full + t, j & 1, 71);
        fence_after();
        const uint32_t sv = smem_u32(sm + OFF_V + st * KV_BYTES);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          // V tile: [64-dim atom][key][64 dims]; N = D spans the two atoms (LBO)
          const uint64_t bd = sdesc(sv + kk * 2048, ATOM_KV, 1024);
          umma_ts(tmem + COL_O + t * D, tmem + COL_S + t * BN + kk * 8, bd, IO,
                  (j > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(o_done + t);
      };
      mbar_wait_sleep(q_full, 0, 72);
      int n = 0, start, nk;
      {
        TileIter cnt(iruns, it.nruns);
        while (cnt.next(start, nk)) ++n;
      }
      if (n > 0) {
        mbar_wait_sleep(kv_full, 0, 73);
        fence_after();
        issue_s(0, 0);
      }
      for (int j = 0; j < n; ++j) {
        const int st = j % STAGES;
        if (two) {
          if (j > 0) {
            issue_pv(1, j - 1, (j - 1) % STAGES);
            umma_commit(kv_empty + (j - 1) % STAGES);  // last reader of stage j-1
#if !AC_F128_INORDER
            mbar_wait_sleep(o_done + 1, (j - 1) & 1, 74);
            fence_after();
#endif
          }
          issue_s(1, st);
        } else if (j > 0) {
          umma_commit(kv_empty + (j - 1) % STAGES);
        }
        issue_pv(0, j, st);
        if (j + 1 < n) {
          const int st1 = (j + 1) % STAGES;
          mbar_wait_sleep(kv_full + st1, ((j + 1) / STAGES) & 1, 75);
#if !AC_F128_INORDER
          mbar_wait_sleep(o_done + 0, j & 1, 76);
#endif
          fence_after();
          issue_s(0, st1);
        }
      }
      if (n > 0) {
        if (two) issue_pv(1, n - 1, (n - 1) % STAGES);
        umma_commit(kv_empty + (n - 1) % STAGES);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------ softmax ------------------------------
    const int t = warp >> 2;
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    const uint32_t tS = tmem + lane_base + COL_S + t * BN;
    const uint32_t tO = tmem + lane_base + COL_O + t * D;
    float m_run = -INFINITY, l_run = 0.f;
    int j = 0;
    const bool live = q4 * 32 < it.q_rows - t * BM;  // this warp holds real rows
    if (t < ntile && live) {
      TileIter ti(iruns, it.nruns);
      int start, nk;
      while (ti.next(start, nk)) {
        mbar_wait_sleep(s_full + t, j & 1, 77);
        fence_after();
        uint32_t sr[BN / 32][32];
#pragma unroll
        for (int ch = 0; ch < BN / 32; ++ch) tmem_ld32(tS + ch * 32, sr[ch]);
        tmem_wait_ld();
        if (nk < BN) {
#pragma unroll
          for (int ch = 0; ch < BN / 32; ++ch)
#pragma unroll
            for (int u = 0; u < 32; ++u)
              if (ch * 32 + u >= nk) sr[ch][u] = __float_as_uint(-INFINITY);
        }
        float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int ch = 0; ch < BN / 32; ++ch)
#pragma unroll
          for (int u = 0; u < 32; u += 8)
#pragma unroll
            for (int a = 0; a < 4; ++a)
              mx[a] = fmax3(mx[a], __uint_as_float(sr[ch][u + 2 * a]),
                                         __uint_as_float(sr[ch][u + 2 * a + 1]));
        const float ms = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])) * scale_log2;
        // PV_t(j-1) has completed (S_t(j) was issued after it): O_t may be
        // rescaled below, before P_t(j) is published.  Lazy: the running max
        // only moves when a row max grows by more than 2^8.
        const bool need = ms > m_run + 8.f;
        const bool warp_need = __any_sync(0xffffffffu, need);
        float alpha = 1.f;
        if (need) {
          alpha = (m_run == -INFINITY) ? 0.f : exp2f(m_run - ms);
          l_run *= alpha;
          m_run = ms;
        }
        const uint64_t sc = pk2(scale_log2, scale_log2);
        const uint64_t nm = pk2(-m_run, -m_run);
        uint64_t acc0 = pk2(0.f, 0.f), acc1 = pk2(0.f, 0.f);
#pragma unroll
        for (int ch = 0; ch < BN / 32; ++ch) {
          if (ch * 32 >= nk) {  // whole chunk past the run's end: P = 0, no exponentials
#pragma unroll
            for (int i = 0; i < 16; ++i) sr[ch][i] = 0u;
            tmem_st16(tS + ch * 16, sr[ch]);
            continue;
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const uint64_t x =
                fma2(pk2(__uint_as_float(sr[ch][2 * i]), __uint_as_float(sr[ch][2 * i + 1])), sc, nm);
            float x0, x1, p0, p1;
            up2(x, x0, x1);
            if ((i & 7) < AC_F128_POLY) {
              exp2_poly2(x0, x1, p0, p1);
            } else {
              p0 = ex2(x0);
              p1 = ex2(x1);
            }
            if (i & 1) acc1 = add2(acc1, pk2(p0, p1));
            else acc0 = add2(acc0, pk2(p0, p1));
            sr[ch][i] = pack_bf16(p0, p1);
          }
          tmem_st16(tS + ch * 16, sr[ch]);  // P over the consumed S columns
        }
        float a0, a1, b0, b1;
        up2(acc0, a0, a1);
        up2(acc1, b0, b1);
        l_run += (a0 + a1) + (b0 + b1);
        if (warp_need && j > 0) {  // O_t *= alpha before PV_t(j) accumulates into it
#pragma unroll 1
          for (int c0 = 0; c0 < D; c0 += 32) {
            uint32_t r[32];
            tmem_ld32(tO + c0, r);
            tmem_wait_ld();
#pragma unroll
            for (int u = 0; u < 32; ++u) r[u] = __float_as_uint(__uint_as_float(r[u]) * alpha);
            tmem_st32(tO + c0, r);
          }
        }
        tmem_wait_st();
        fence_before();
        mbar_arrive(p_full + t);
        ++j;
      }
      // ------------------------------ epilogue ------------------------------
      if (j > 0) {
        mbar_wait_sleep(o_done + t, (j - 1) & 1, 78);
        fence_after();
      }
      const int rows_t = min(BM, it.q_rows - t * BM);
      const int tok = (row < rows_t) ? qidx[it.q_row0 + t * BM + row] : -1;
      const float inv = (l_run > 0.f) ? 1.f / l_run : 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t r[32];
        if (j > 0) {
          tmem_ld32(tO + c0, r);
          tmem_wait_ld();
        } else {
#pragma unroll
          for (int u = 0; u < 32; ++u) r[u] = 0u;
        }
        if (tok >= 0) {
          const int64_t ob = ((int64_t)it.head * L + tok) * D + c0;
          if (out_dtype == AC_DTYPE_BF16) {
            uint32_t w[16];
#pragma unroll
            for (int u = 0; u < 16; ++u)
              w[u] = pack_bf16(__uint_as_float(r[2 * u]) * inv, __uint_as_float(r[2 * u + 1]) * inv);
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out) + ob);
#pragma unroll
            for (int u = 0; u < 4; ++u) dst[u] = make_uint4(w[4 * u], w[4 * u + 1], w[4 * u + 2], w[4 * u + 3]);
          } else {
            float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + ob);
#pragma unroll
            for (int u = 0; u < 8; ++u)
              dst[u] = make_float4(__uint_as_float(r[4 * u]) * inv, __uint_as_float(r[4 * u + 1]) * inv,
                                   __uint_as_float(r[4 * u + 2]) * inv, __uint_as_float(r[4 * u + 3]) * inv);
          }
        }
      }
    }
  }
  fence_before();
  __syncthreads();
  if (warp == W_MMA) {
    fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace f128
}  // namespace ac

extern "C" int ac_sparse_attention_fa4_d128(const void* q, int64_t q_rows_total, const int32_t* qidx,
                                            const void* k, const void* v, int d, int64_t L, int heads,
                                            const ac_attn_item* items, int nitems, const int32_t* runs,
                                            float scale, void* out, int out_dtype, void* stream) {
  using namespace ac::f128;
  if (nitems <= 0) return AC_OK;
  if (d != D) {
    ac_host::set_error("fa4 d128 attention: head_dim %d unsupported (128)", d);
    return AC_ERR_DIM;
  }
  CUtensorMap mq, mk, mv;
  int rc;
  if ((rc = ac_host::make_map_2d(&mq, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, q_rows_total, D, 64, BM)))
    return rc;
  if ((rc = ac_host::make_map_2d(&mk, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (int64_t)heads * L, D, 64, BN)))
    return rc;
  if ((rc = ac_host::make_map_2d(&mv, v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (int64_t)heads * L, D, 64, BN)))
    return rc;
  if ((rc = ac_host::func_smem((const void*)k_attn_fa4_d128, SMEM, "k_attn_fa4_d128 smem"))) return rc;
  const float scale_log2 = scale * 1.4426950408889634f;
  k_attn_fa4_d128<<<nitems, THREADS, SMEM, reinterpret_cast<cudaStream_t>(stream)>>>(
      mq, mk, mv, qidx, L, items, runs, scale_log2, out, out_dtype);
  AC_CHECK_LAUNCH("k_attn_fa4_d128");
  return AC_OK;
}
