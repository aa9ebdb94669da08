// Block-sparse flash attention for head_dim 64 on the 5th-generation tensor
// cores, two query tiles per CTA (FA4-style ping-pong).
//
// Reference semantics: pipeline.py:154-165 (_gathered_attention) and
// reference.py:25-45 (full_attention): every query cluster attends, with a
// plain softmax (scale 1/sqrt(D), max-subtracted), over the union of its
// selected key clusters.  Keys/values are stored cluster-contiguous (Kp/Vp),
// so a query cluster's keys are a handful of [start, end) runs, walked in
// 128-key tiles; keys past a run's end are masked.
//
// One CTA = one work item = up to 256 query rows (two 128-row tiles) of one
// query cluster, which share every K/V tile:
//   warps 0-3   softmax of Q tile 0 (thread = query row = TMEM lane)
//   warps 4-7   softmax of Q tile 1
//   warp 8      TMA producer: Q0/Q1 once, K/V tiles through a 4-stage ring
//   warps 9/10  MMA issuers, one per Q tile: S_t = Q_t·Kᵀ into TMEM
//               (kind::f16, f32 accum), O_t += P_t·V with P_t read from TMEM
//               (the A-from-TMEM form); a K/V stage is released when both
//               tiles' PV on it have completed
// TMEM (512 columns): S0 | S1 (128 each) | O0 | O1 (64 each) | P0 | P1
// (64 x 32-bit columns = 128 bf16 each).  While one tile's softmax runs the
// tensor core works on the other tile's S or PV.
// Softmax in the exp2 domain with lazy rescaling (the running max only
// moves when a row max grows by more than 2^8); 1/8 of the exponentials
// are evaluated with a cubic polynomial on the FMA pipe (packed f32x2) to
// offload the MUFU unit, which otherwise bounds D = 64 attention on B200
// (2/8 measured slower: the softmax warps are then issue-limited).
// Epilogue: O / l, bf16 or f32, stored at the query's original token row
// (the inverse permutation is fused into the store).
#include <cfloat>

#include "attn_common.cuh"

namespace ac {
namespace fa {
using namespace ac::tc;
using namespace ac::attn;

constexpr int D = 64;
constexpr int BM = 128;
constexpr int BN = 128;
#ifndef AC_FA4_STAGES
#define AC_FA4_STAGES 4
#endif
constexpr int STAGES = AC_FA4_STAGES;
#ifndef AC_FA4_SPLIT_MMA
#define AC_FA4_SPLIT_MMA 1  // one MMA-issuing warp per Q tile (no head-of-line blocking)
#endif
#if AC_FA4_SPLIT_MMA
constexpr int THREADS = 352;
#else
constexpr int THREADS = 320;
#endif
constexpr int W_TMA = 8, W_MMA = 9, W_MMA1 = 10;
constexpr int Q_BYTES = BM * D * 2;
constexpr int KV_BYTES = BN * D * 2;
constexpr int OFF_Q = 0;
constexpr int OFF_K = OFF_Q + 2 * Q_BYTES;
constexpr int OFF_V = OFF_K + STAGES * KV_BYTES;
constexpr int OFF_BAR = OFF_V + STAGES * KV_BYTES;
constexpr int NBAR = 1 + 2 * STAGES + 2 + 2 + 2 + 2;
constexpr int OFF_MISC = OFF_BAR + NBAR * 8;
constexpr int OFF_RUNS = OFF_MISC + 16;  // the item's key runs (<= kRunsSmem), read by every role
constexpr int kRunsSmem = 128;
constexpr int SMEM = OFF_RUNS + 8 * kRunsSmem + 1024;
constexpr uint32_t COL_S = 0, COL_O = 256, COL_P = 384;
#ifndef AC_FA4_ORDER
#define AC_FA4_ORDER 1  // MMA issue order per K tile (0: S0 S1 PV0 PV1, 1: S0 PV0 S1 PV1)
#endif
#ifndef AC_FA4_LATE_WAIT
#define AC_FA4_LATE_WAIT 1  // wait for PV_t(j-1) after the exponentials (P kept in registers)
#endif
#ifndef AC_FA4_SPIN
#define AC_FA4_SPIN 0  // softmax warps spin on their barriers instead of sleeping
#endif
#if AC_FA4_SPIN
#define SM_WAIT(b, p, tag) mbar_wait(b, p, tag)
#else
#define SM_WAIT(b, p, tag) mbar_wait_sleep(b, p, tag)
#endif
#ifndef AC_FA4_POLY
#define AC_FA4_POLY 1  // of every 8 exp2 pairs, this many on the FMA pipe (polynomial)
#endif

__global__ void __launch_bounds__(THREADS, 1)
k_attn_fa4(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmk,
           const __grid_constant__ CUtensorMap tmv, const int32_t* __restrict__ qidx, int64_t L,
           const ac_attn_item* __restrict__ items, const int32_t* __restrict__ runs,
           float scale_log2, void* __restrict__ out, int out_dtype) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = smraw + ((1024u - (smem_u32(smraw) & 1023u)) & 1023u);
  const ac_attn_item it = items[blockIdx.x];
  if (it.q_rows <= 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool two = it.q_rows > BM;

  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = bars + 1 + STAGES;
  uint64_t* s_full = bars + 1 + 2 * STAGES;
  uint64_t* p_full = s_full + 2;
  uint64_t* o_done = s_full + 4;
  uint64_t* s_free = s_full + 6;  // softmax has S_t in registers: the MMA may overwrite it
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + OFF_MISC);

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(kv_full + s, 1);
      mbar_init(kv_empty + s, (AC_FA4_SPLIT_MMA && two) ? 2 : 1);
    }
    for (int t = 0; t < 2; ++t) {
      // only warps holding at least one real query row take part (the rest
      // of a partial tile's rows are padding and skip the softmax entirely)
      const int live = 32 * max(1, min(4, (min(BM, it.q_rows - t * BM) + 31) / 32));
      mbar_init(s_full + t, 1);
      mbar_init(p_full + t, live);
      mbar_init(o_done + t, 1);
      mbar_init(s_free + t, live);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  int32_t* s_runs = reinterpret_cast<int32_t*>(sm + OFF_RUNS);
  const bool runs_smem = it.nruns <= kRunsSmem;
  if (runs_smem)
    for (int i = threadIdx.x; i < 2 * it.nruns; i += blockDim.x) s_runs[i] = runs[2 * it.run0 + i];
  if (warp == W_MMA) tmem_alloc(tmem_slot, 512);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  // (the tile walk reads the runs at every run change: from shared memory,
  // not a dependent global load on the softmax warps' critical path)
  const int32_t* iruns = runs_smem ? s_runs : runs + 2 * it.run0;
  const int64_t krow0 = (int64_t)it.head * L;

  if (warp == W_TMA) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      mbar_expect_tx(q_full, (two ? 2 : 1) * Q_BYTES);
      tma_load_2d(sm + OFF_Q, &tmq, 0, (int)it.q_row0, q_full);
      if (two) tma_load_2d(sm + OFF_Q + Q_BYTES, &tmq, 0, (int)it.q_row0 + BM, q_full);
      TileIter ti(iruns, it.nruns);
      int start, nk;
      for (int j = 0; ti.next(start, nk); ++j) {
        const int st = j % STAGES;
        if (j >= STAGES) mbar_wait_sleep(kv_empty + st, ((j / STAGES) - 1) & 1, 40);
        mbar_expect_tx(kv_full + st, 2 * KV_BYTES);
        const int row = (int)(krow0 + start);
        tma_load_2d(sm + OFF_K + st * KV_BYTES, &tmk, 0, row, kv_full + st);
        tma_load_2d(sm + OFF_V + st * KV_BYTES, &tmv, 0, row, kv_full + st);
      }
    }
    __syncwarp();
#if AC_FA4_SPLIT_MMA
  } else if (warp == W_MMA || warp == W_MMA1) {
    // ------------------- MMA issuers: one warp per Q tile -----------------------
    // Each tile's S/PV chain only waits for its own softmax; a K/V stage is
    // released once every tile's PV on it has completed (kv_empty count).
    const int t = warp - W_MMA;
    if (lane == 0 && (t == 0 || two)) {
      constexpr uint32_t IS = idesc_bf16(BM, BN, false);
      constexpr uint32_t IO = idesc_bf16(BM, D, true);
      const uint32_t sq = smem_u32(sm + OFF_Q) + t * Q_BYTES;
      auto issue_pv = [&](int jj, int st, bool release) {
        mbar_wait_sleep(p_full + t, jj & 1, 41);
        fence_after();
        const uint32_t sv = smem_u32(sm + OFF_V + st * KV_BYTES);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          const uint64_t bd = sdesc(sv + kk * 2048, BN * 128, 1024);
          umma_ts(tmem + COL_O + t * D, tmem + COL_P + t * 64 + kk * 8, bd, IO,
                  (jj > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(o_done + t);
        if (release) umma_commit(kv_empty + st);
      };
      mbar_wait_sleep(q_full, 0, 42);
      TileIter ti(iruns, it.nruns);
      int start, nk, j = 0;
      while (ti.next(start, nk)) {
        const int st = j % STAGES;
        mbar_wait_sleep(kv_full + st, (j / STAGES) & 1, 43);
        fence_after();
        if (j > 0) mbar_wait_sleep(s_free + t, (j - 1) & 1, 47);
        const uint32_t sk = smem_u32(sm + OFF_K + st * KV_BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t ad = sdesc(sq + kk * 32, 16, 1024);
          const uint64_t bd = sdesc(sk + kk * 32, 16, 1024);
          umma_f16(tmem + COL_S + t * BN, ad, bd, IS, kk > 0 ? 1u : 0u);
        }
        umma_commit(s_full + t);
        if (j > 0) issue_pv(j - 1, (j - 1) % STAGES, true);
        ++j;
      }
      if (j > 0) issue_pv(j - 1, (j - 1) % STAGES, false);
    }
    __syncwarp();
#else
  } else if (warp == W_MMA) {
    // ------------------------------ MMA issuer --------------------------------
    if (lane == 0) {
      constexpr uint32_t IS = idesc_bf16(BM, BN, false);
      constexpr uint32_t IO = idesc_bf16(BM, D, true);
      const uint32_t sq = smem_u32(sm + OFF_Q);
      auto issue_s = [&](int t, int j, int st) {
        if (j > 0) mbar_wait_sleep(s_free + t, (j - 1) & 1, 47);
        const uint32_t sk = smem_u32(sm + OFF_K + st * KV_BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t ad = sdesc(sq + t * Q_BYTES + kk * 32, 16, 1024);
          const uint64_t bd = sdesc(sk + kk * 32, 16, 1024);
          umma_f16(tmem + COL_S + t * BN, ad, bd, IS, kk > 0 ? 1u : 0u);
        }
        umma_commit(s_full + t);
      };
      auto issue_pv = [&](int t, int j, int st) {
        mbar_wait_sleep(p_full + t, j & 1, 41);
        fence_after();
        const uint32_t sv = smem_u32(sm + OFF_V + st * KV_BYTES);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk) {
          const uint64_t bd = sdesc(sv + kk * 2048, BN * 128, 1024);
          umma_ts(tmem + COL_O + t * D, tmem + COL_P + t * 64 + kk * 8, bd, IO,
                  (j > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(o_done + t);
      };
      mbar_wait_sleep(q_full, 0, 42);
      TileIter ti(iruns, it.nruns);
      int start, nk, j = 0;
      while (ti.next(start, nk)) {
        const int st = j % STAGES;
        mbar_wait_sleep(kv_full + st, (j / STAGES) & 1, 43);
        fence_after();
        // S for tile j as soon as each softmax has pulled S_{j-1} into
        // registers, then the PV products of tile j-1 once P_{j-1} is in TMEM
#if AC_FA4_ORDER == 0
        issue_s(0, j, st);
        if (two) issue_s(1, j, st);
        if (j > 0) {
          issue_pv(0, j - 1, (j - 1) % STAGES);
          if (two) issue_pv(1, j - 1, (j - 1) % STAGES);
        }
#else
        issue_s(0, j, st);
        if (j > 0) issue_pv(0, j - 1, (j - 1) % STAGES);
        if (two) {
          issue_s(1, j, st);
          if (j > 0) issue_pv(1, j - 1, (j - 1) % STAGES);
        }
#endif
        if (j > 0) umma_commit(kv_empty + (j - 1) % STAGES);
        ++j;
      }
      if (j > 0) {
        issue_pv(0, j - 1, (j - 1) % STAGES);
        if (two) issue_pv(1, j - 1, (j - 1) % STAGES);
      }
    }
    __syncwarp();
#endif
  } else {
    // ------------------------------ softmax ------------------------------
    const int t = warp >> 2;  // Q tile of this warpgroup
    const int q4 = warp & 3;
    const int row = q4 * 32 + lane;  // TMEM lane / row in the tile
    const uint32_t lane_base = (uint32_t)(q4 * 32) << 16;
    const uint32_t tS = tmem + lane_base + COL_S + t * BN;
    const uint32_t tO = tmem + lane_base + COL_O + t * D;
    const uint32_t tP = tmem + lane_base + COL_P + t * 64;
    float m_run = -INFINITY, l_run = 0.f;
    int j = 0;
    const bool live = q4 * 32 < it.q_rows - t * BM;  // this warp holds real rows
    if ((t == 0 || two) && live) {
      TileIter ti(iruns, it.nruns);
      int start, nk;
      while (ti.next(start, nk)) {
        SM_WAIT(s_full + t, j & 1, 44);
        fence_after();
        uint32_t sr[BN / 32][32];
#pragma unroll
        for (int ch = 0; ch < BN / 32; ++ch) tmem_ld32(tS + ch * 32, sr[ch]);
        tmem_wait_ld();
        fence_before();
        mbar_arrive(s_free + t);
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
#if !AC_FA4_LATE_WAIT
        // P_t / O_t are free once the previous tile's PV has completed
        if (j > 0) {
          SM_WAIT(o_done + t, (j - 1) & 1, 45);
          fence_after();
        }
#endif
        // lazy rescale: a row's running max only moves when it grows by > 2^8
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
        auto exp_chunk = [&](int ch) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const uint64_t x =
                fma2(pk2(__uint_as_float(sr[ch][2 * i]), __uint_as_float(sr[ch][2 * i + 1])), sc, nm);
            float x0, x1, p0, p1;
            up2(x, x0, x1);
            if ((i & 7) < AC_FA4_POLY) {
              exp2_poly2(x0, x1, p0, p1);
            } else {
              p0 = ex2(x0);
              p1 = ex2(x1);
            }
            if (i & 1) acc1 = add2(acc1, pk2(p0, p1));
            else acc0 = add2(acc0, pk2(p0, p1));
            sr[ch][i] = pack_bf16(p0, p1);  // packed P overwrites consumed S slots
          }
#if !AC_FA4_LATE_WAIT
          tmem_st16(tP + ch * 16, sr[ch]);
#endif
        };
        if (nk == BN) {
#pragma unroll
          for (int ch = 0; ch < BN / 32; ++ch) exp_chunk(ch);
        } else {  // the run's last tile: 32-key chunks past its end get P = 0, no exponentials
#pragma unroll
          for (int ch = 0; ch < BN / 32; ++ch) {
            if (ch * 32 < nk) {
              exp_chunk(ch);
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) sr[ch][i] = 0u;
#if !AC_FA4_LATE_WAIT
              tmem_st16(tP + ch * 16, sr[ch]);
#endif
            }
          }
        }
#if AC_FA4_LATE_WAIT
        // P_t / O_t are free once the previous tile's PV has completed: the
        // exponentials above ran while PV_t(j-1) was still on the tensor core
        if (j > 0) {
          SM_WAIT(o_done + t, (j - 1) & 1, 45);
          fence_after();
        }
#pragma unroll
        for (int ch = 0; ch < BN / 32; ++ch) tmem_st16(tP + ch * 16, sr[ch]);
#endif
        float a0, a1, b0, b1;
        up2(acc0, a0, a1);
        up2(acc1, b0, b1);
        l_run += (a0 + a1) + (b0 + b1);
        tmem_wait_st();
        if (warp_need && j > 0) {  // O_t *= alpha before PV_j accumulates into it
#pragma unroll
          for (int c0 = 0; c0 < D; c0 += 32) {
            uint32_t r[32];
            tmem_ld32(tO + c0, r);
            tmem_wait_ld();
#pragma unroll
            for (int u = 0; u < 32; ++u) r[u] = __float_as_uint(__uint_as_float(r[u]) * alpha);
            tmem_st32(tO + c0, r);
          }
          tmem_wait_st();
        }
        fence_before();
        mbar_arrive(p_full + t);
        ++j;
      }
      // ------------------------------ epilogue ------------------------------
      if (j > 0) {
        mbar_wait_sleep(o_done + t, (j - 1) & 1, 46);
        fence_after();
      }
      const int rows_t = min(BM, it.q_rows - t * BM);
      const int tok = (row < rows_t) ? qidx[it.q_row0 + t * BM + row] : -1;
      const float inv = (l_run > 0.f) ? 1.f / l_run : 0.f;
#pragma unroll
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

}  // namespace fa
}  // namespace ac

extern "C" int ac_sparse_attention_fa4(const void* q, int64_t q_rows_total, const int32_t* qidx,
                                       const void* k, const void* v, int d, int64_t L, int heads,
                                       const ac_attn_item* items, int nitems, const int32_t* runs,
                                       float scale, void* out, int out_dtype, void* stream) {
  using namespace ac::fa;
  if (nitems <= 0) return AC_OK;
  if (d != D) {
    ac_host::set_error("fa4 attention: head_dim %d unsupported (64)", d);
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
  if ((rc = ac_host::func_smem((const void*)k_attn_fa4, SMEM, "k_attn_fa4 smem"))) return rc;
  const float scale_log2 = scale * 1.4426950408889634f;
  k_attn_fa4<<<nitems, THREADS, SMEM, reinterpret_cast<cudaStream_t>(stream)>>>(
      mq, mk, mv, qidx, L, items, runs, scale_log2, out, out_dtype);
  AC_CHECK_LAUNCH("k_attn_fa4");
  return AC_OK;
}
