// Block-sparse flash attention on the 5th-generation tensor cores (sm_100a).
//
// Reference semantics: pipeline.py:154-165 (_gathered_attention) and
// reference.py:25-45 (full_attention): for every query cluster g, softmax
// attention over the union of the selected key clusters' tokens.  Keys and
// values are stored cluster-contiguous (Kp/Vp), so a query cluster attends
// over a handful of contiguous [start, end) runs; every run is walked in
// BN-row tiles fetched by TMA, and rows past the run end are masked.
//
// One CTA = one work item (<= 128 query rows of one query cluster):
//   warp 4      TMA producer (Q once, then K/V tiles through a 2-stage ring)
//   warp 5      MMA issuer: S = Q·Kᵀ (tcgen05.mma kind::f16, f32 in TMEM,
//               double-buffered S), then O += P·V (P from smem, V MN-major)
//   warps 0..3  softmax: thread i owns TMEM lane i = query row i; online
//               softmax in the exp2 domain with lazy O rescaling (the running
//               max only moves when it grows by > 2^8), P written as bf16 into
//               a 128B-swizzled K-major smem tile; epilogue O / l -> scattered
//               to the original token rows (inverse permutation fused).
// Compiled for sm_100a only; SASS shows UTCHMMA / UTMALDG / LDTM / STTM.
#include <cfloat>

#include "tc_common.cuh"

namespace ac {
namespace tc {
template <int D>
struct Cfg {
  static constexpr int BM = 128;
  static constexpr int BN = (D == 64) ? 128 : 64;
  static constexpr int KB = D / 64;  // 64-wide (128 B) K blocks of Q/K, N blocks of V
  static constexpr int STAGES = 2;
  static constexpr int Q_BYTES = BM * D * 2;
  static constexpr int K_BYTES = BN * D * 2;
  static constexpr int V_BYTES = BN * D * 2;
  static constexpr int P_BYTES = BM * BN * 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + Q_BYTES;
  static constexpr int OFF_V = OFF_K + STAGES * K_BYTES;
  static constexpr int OFF_P = OFF_V + STAGES * V_BYTES;
  static constexpr int OFF_BAR = OFF_P + 2 * P_BYTES;
  static constexpr int NBAR = 1 + 2 * STAGES + 8;
  static constexpr int OFF_TILES = OFF_BAR + NBAR * 8 + 16;
  static constexpr int MAX_TILES = 4096;
  static constexpr int SMEM = OFF_TILES + MAX_TILES * 8 + 1024;  // + alignment slack
  static constexpr int TMEM_COLS = 512;
  static constexpr int S_COL0 = 0;          // two S buffers of BN columns
  static constexpr int O_COL = 2 * BN;      // O accumulator (D columns)
};

template <int D>
__global__ void __launch_bounds__(192, 1)
k_attn_tc(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tmk,
          const __grid_constant__ CUtensorMap tmv, const int32_t* __restrict__ qidx, int64_t L,
          const ac_attn_item* __restrict__ items, const int32_t* __restrict__ runs,
          float scale_log2, void* __restrict__ out, int out_dtype) {
  using C = Cfg<D>;
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  const ac_attn_item it = items[blockIdx.x];
  if (it.q_rows <= 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + C::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = bars + 1 + C::STAGES;
  uint64_t* s_full = bars + 1 + 2 * C::STAGES;
  uint64_t* s_free = s_full + 2;
  uint64_t* p_full = s_full + 4;
  uint64_t* o_done = s_full + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);
  int2* tiles = reinterpret_cast<int2*>(sm + C::OFF_TILES);
  __shared__ int s_ntiles;

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(kv_full + s, 1);
      mbar_init(kv_empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(s_full + b, 1);
      mbar_init(s_free + b, 128);
      mbar_init(p_full + b, 128);
      mbar_init(o_done + b, 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    // tile list: (Kp row of the tile start within the head, valid rows)
    int nt = 0;
    for (int r = 0; r < it.nruns; ++r) {
      const int rs = runs[2 * (it.run0 + r)], re = runs[2 * (it.run0 + r) + 1];
      for (int s = rs; s < re && nt < C::MAX_TILES; s += C::BN) tiles[nt++] = make_int2(s, min(C::BN, re - s));
    }
    s_ntiles = nt;
  }
  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const int T = s_ntiles;
  const int64_t krow0 = (int64_t)it.head * L;

  if (warp == 4) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0 && T > 0) {
      mbar_expect_tx(q_full, C::Q_BYTES);
      for (int kb = 0; kb < C::KB; ++kb)
        tma_load_2d(sm + C::OFF_Q + kb * (C::BM * 128), &tmq, kb * 64, (int)it.q_row0, q_full);
      for (int j = 0; j < T; ++j) {
        const int st = j % C::STAGES;
        if (j >= C::STAGES) mbar_wait(kv_empty + st, ((j / C::STAGES) - 1) & 1, 1);
        mbar_expect_tx(kv_full + st, C::K_BYTES + C::V_BYTES);
        const int row = (int)(krow0 + tiles[j].x);
        for (int kb = 0; kb < C::KB; ++kb) {
          tma_load_2d(sm + C::OFF_K + st * C::K_BYTES + kb * (C::BN * 128), &tmk, kb * 64, row,
                      kv_full + st);
          tma_load_2d(sm + C::OFF_V + st * C::V_BYTES + kb * (C::BN * 128), &tmv, kb * 64, row,
                      kv_full + st);
        }
      }
    }
    __syncwarp();
  } else if (warp == 5) {
    // ------------------------------ MMA issuer --------------------------------
    if (lane == 0 && T > 0) {
      constexpr uint32_t IS = idesc_bf16(C::BM, C::BN, false);
      constexpr uint32_t IO = idesc_bf16(C::BM, D, true);
      const uint32_t sq = smem_u32(sm + C::OFF_Q);
      auto issue_pv = [&](int i) {
        const int b = i & 1, st = i % C::STAGES;
        mbar_wait(p_full + b, (i >> 1) & 1, 2);
        fence_after();
        const uint32_t sp = smem_u32(sm + C::OFF_P + b * C::P_BYTES);
        const uint32_t sv = smem_u32(sm + C::OFF_V + st * C::V_BYTES);
#pragma unroll
        for (int kk = 0; kk < C::BN / 16; ++kk) {
          const uint64_t ad = sdesc(sp + (kk >> 2) * (C::BM * 128) + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = sdesc(sv + kk * 2048, C::BN * 128, 1024);
          umma_f16(tmem + C::O_COL, ad, bd, IO, (i > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(kv_empty + st);
        umma_commit(o_done + b);
      };
      mbar_wait(q_full, 0, 3);
      for (int j = 0; j < T; ++j) {
        const int b = j & 1, st = j % C::STAGES;
        mbar_wait(kv_full + st, (j / C::STAGES) & 1, 4);
        if (j >= 2) mbar_wait(s_free + b, ((j - 2) >> 1) & 1, 5);
        fence_after();
        const uint32_t sk = smem_u32(sm + C::OFF_K + st * C::K_BYTES);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint64_t ad = sdesc(sq + (kk >> 2) * (C::BM * 128) + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = sdesc(sk + (kk >> 2) * (C::BN * 128) + (kk & 3) * 32, 16, 1024);
          umma_f16(tmem + C::S_COL0 + b * C::BN, ad, bd, IS, kk > 0 ? 1u : 0u);
        }
        umma_commit(s_full + b);
        if (j >= 1) issue_pv(j - 1);
      }
      issue_pv(T - 1);
    }
    __syncwarp();
  } else {
    // ------------------------------ softmax warps ------------------------------
    const int row = threadIdx.x;  // 0..127 == TMEM lane
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    float m_run = -INFINITY, l_run = 0.f;
    unsigned char* pbase = sm + C::OFF_P;
    for (int j = 0; j < T; ++j) {
      const int b = j & 1;
      mbar_wait(s_full + b, (j >> 1) & 1, 6);
      fence_after();
      float s[C::BN];
#pragma unroll
      for (int c0 = 0; c0 < C::BN; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_base + C::S_COL0 + b * C::BN + c0, r);
        tmem_wait_ld();
#pragma unroll
        for (int u = 0; u < 32; ++u) s[c0 + u] = __uint_as_float(r[u]);
      }
      fence_before();
      mbar_arrive(s_free + b);
      const int nk = tiles[j].y;
      float mt = -INFINITY;
#pragma unroll
      for (int c = 0; c < C::BN; ++c) {
        s[c] = (c < nk) ? s[c] * scale_log2 : -INFINITY;
        mt = fmaxf(mt, s[c]);
      }
      // P buffer b is free once PV(j-2) has completed
      if (j >= 2) mbar_wait(o_done + b, ((j - 2) >> 1) & 1, 7);
      // lazy rescale: a row's max only moves when it grows by > 2^8.  The
      // TMEM load/store of O is warp-collective (.sync.aligned), so the
      // decision is made per warp; rows that do not move scale by 1.
      const bool need = mt > m_run + 8.f;
      if (__any_sync(0xffffffffu, need)) {
        float alpha = 1.f;
        if (need) {
          if (m_run != -INFINITY) alpha = ex2(m_run - mt);
          l_run *= alpha;
          m_run = mt;
        }
        if (j >= 1) {
          // O must include PV(j-1) before it is rescaled
          mbar_wait(o_done + ((j - 1) & 1), ((j - 1) >> 1) & 1, 8);
          fence_after();
#pragma unroll
          for (int c0 = 0; c0 < D; c0 += 32) {
            uint32_t r[32];
            tmem_ld32(tmem + lane_base + C::O_COL + c0, r);
            tmem_wait_ld();
#pragma unroll
            for (int u = 0; u < 32; ++u) r[u] = __float_as_uint(__uint_as_float(r[u]) * alpha);
            tmem_st32(tmem + lane_base + C::O_COL + c0, r);
          }
          tmem_wait_st();
        }
      }
      float psum = 0.f;
      unsigned char* prow = pbase + b * C::P_BYTES + row * 128;
#pragma unroll
      for (int kb = 0; kb < C::BN / 64; ++kb) {
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
          uint32_t w[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = kb * 64 + ch * 8 + 2 * u;
            const float p0 = ex2(s[c] - m_run);
            const float p1 = ex2(s[c + 1] - m_run);
            psum += p0 + p1;
            __nv_bfloat162 h2 = __floats2bfloat162_rn(p0, p1);
            w[u] = *reinterpret_cast<uint32_t*>(&h2);
          }
          const int sw = ch ^ (row & 7);
          *reinterpret_cast<uint4*>(prow + kb * (C::BM * 128) + sw * 16) = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
      l_run += psum;
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      fence_before();
      mbar_arrive(p_full + b);
    }
    // ------------------------------ epilogue ------------------------------
    if (T > 0) {
      mbar_wait(o_done + ((T - 1) & 1), ((T - 1) >> 1) & 1, 9);
      fence_after();
    }
    const int tok = (row < it.q_rows) ? qidx[it.q_row0 + row] : -1;
    const float inv = (l_run > 0.f) ? 1.f / l_run : 0.f;
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 32) {
      uint32_t r[32];
      if (T > 0) {
        tmem_ld32(tmem + lane_base + C::O_COL + c0, r);
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
          for (int u = 0; u < 16; ++u) {
            __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(r[2 * u]) * inv,
                                                      __uint_as_float(r[2 * u + 1]) * inv);
            w[u] = *reinterpret_cast<uint32_t*>(&h2);
          }
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
  fence_before();
  __syncthreads();
  if (warp == 5) {
    __syncwarp();
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(C::TMEM_COLS));
  }
}

// --------------------------------------------------------------------------
// host: tensor maps through the driver entry point (tc_common.cu)
// --------------------------------------------------------------------------
int make_map(CUtensorMap* m, const void* base, int64_t rows, int d, int box_rows) {
  return ac_host::make_map_2d(m, base, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, rows, d, 64, box_rows);
}

template <int D>
int launch_tc(const void* q, int64_t q_rows_total, const int32_t* qidx, const void* k,
              const void* v, int64_t L, int heads, const ac_attn_item* items, int nitems,
              const int32_t* runs, float scale, void* out, int out_dtype, cudaStream_t st) {
  using C = Cfg<D>;
  CUtensorMap mq, mk, mv;
  int rc;
  if ((rc = make_map(&mq, q, q_rows_total, D, C::BM))) return rc;
  if ((rc = make_map(&mk, k, (int64_t)heads * L, D, C::BN))) return rc;
  if ((rc = make_map(&mv, v, (int64_t)heads * L, D, C::BN))) return rc;
  cudaError_t e = cudaFuncSetAttribute((const void*)k_attn_tc<D>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
  if (e != cudaSuccess) return ac_host::check_cuda(e, "k_attn_tc smem");
  const float scale_log2 = scale * 1.4426950408889634f;
  k_attn_tc<D><<<nitems, 192, C::SMEM, st>>>(mq, mk, mv, qidx, L, items, runs, scale_log2, out,
                                             out_dtype);
  AC_CHECK_LAUNCH("k_attn_tc");
  return AC_OK;
}

}  // namespace tc
}  // namespace ac

extern "C" int ac_sparse_attention_tc(const void* q, int64_t q_rows_total, const int32_t* qidx,
                                      const void* k, const void* v, int d, int64_t L, int heads,
                                      const ac_attn_item* items, int nitems, const int32_t* runs,
                                      float scale, void* out, int out_dtype, void* stream) {
  if (nitems <= 0) return AC_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (d == 64)
    return ac::tc::launch_tc<64>(q, q_rows_total, qidx, k, v, L, heads, items, nitems, runs, scale,
                                 out, out_dtype, st);
  if (d == 128)
    return ac::tc::launch_tc<128>(q, q_rows_total, qidx, k, v, L, heads, items, nitems, runs, scale,
                                  out, out_dtype, st);
  ac_host::set_error("tcgen05 attention: head_dim %d unsupported (64, 128)", d);
  return AC_ERR_DIM;
}
