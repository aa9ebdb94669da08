// Device evaluation of numpy's pairwise-summation tree over long vectors
// (length n up to a few million), driven by a host-built plan.
//
// numpy reduces a contiguous 1-D float array with pairwise_sum(): blocks of
// <= 128 elements are summed with 8 strided accumulators, larger ranges are
// split at n2 = n/2 - (n/2 % 8) and the halves added.  The tree shape depends
// only on n, so the host flattens it once (ac_pw_plan_build) into:
//
//   plan[0] = L (leaves)   plan[1] = I (internal nodes)   plan[2] = H (levels)
//   plan[3 .. 3+L]        leaf start offsets, plus sentinel n  (L+1 words)
//   plan[4+L .. 4+L+H]    level boundaries into the node table (H+1 words)
//   then I triples (dst, a, b): vals[dst] = vals[a] + vals[b]
//
// Leaves are numbered 0..L-1 in DFS order, internal nodes L..L+I-1; levels
// are grouped by height so every child is final before its parent is read.
#pragma once
#include "common.cuh"

namespace ac {

struct PwPlan {
  const int32_t* p;
  AC_DEV int leaves() const { return p[0]; }
  AC_DEV int internal() const { return p[1]; }
  AC_DEV int levels() const { return p[2]; }
  AC_DEV int leaf_lo(int i) const { return p[3 + i]; }
  AC_DEV int level_begin(int h) const { return p[4 + p[0] + h]; }
  AC_DEV const int32_t* nodes() const { return p + 5 + p[0] + p[2]; }
  AC_DEV int nvals() const { return p[0] + p[1]; }
  AC_DEV int root() const { return p[1] ? p[0] + p[1] - 1 : 0; }
};

// Whole-CTA evaluation.  `vals` has plan.nvals() slots (shared or global).
// Returns the sum in every thread.  Must be called by all threads of the CTA.
template <typename T, typename Get>
__device__ T pw_eval_block(const PwPlan plan, const Get& get, T* vals) {
  const int L = plan.leaves();
  for (int leaf = threadIdx.x; leaf < L; leaf += blockDim.x) {
    const int lo = plan.leaf_lo(leaf);
    const int hi = plan.leaf_lo(leaf + 1);
    vals[leaf] = pw_leaf<T>(get, lo, hi - lo);
  }
  __syncthreads();
  const int H = plan.levels();
  const int32_t* nd = plan.nodes();
  for (int h = 0; h < H; ++h) {
    const int b = plan.level_begin(h), e = plan.level_begin(h + 1);
    for (int j = b + threadIdx.x; j < e; j += blockDim.x) {
      const int dst = nd[3 * j], a = nd[3 * j + 1], c = nd[3 * j + 2];
      vals[dst] = vals[a] + vals[c];
    }
    __syncthreads();
  }
  T r = vals[plan.root()];
  __syncthreads();
  return r;
}


// Same tree, leaves evaluated by 8-lane groups (four leaves per warp): lane
// j of a group runs numpy's accumulator r_j = a[j] + a[j+8] + ... in order,
// the three xor-shuffles fold ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and lane 0
// adds the n % 8 tail in order -- pw_leaf's operations, so the same bits,
// with each load instruction touching 4 x 32 contiguous bytes instead of 32
// scattered words (the one-thread-per-leaf form is bound by L1 wavefronts).
template <typename T, typename Get>
__device__ T pw_eval_block_g8(const PwPlan plan, const Get& get, T* vals) {
  const int L = plan.leaves();
  const int lane = threadIdx.x & 31, j = lane & 7;
  for (int base = (threadIdx.x >> 5) * 4; base < L; base += (blockDim.x >> 5) * 4) {
    const int leaf = base + (lane >> 3);
    int lo = 0, m = 0;
    if (leaf < L) {
      lo = plan.leaf_lo(leaf);
      m = plan.leaf_lo(leaf + 1) - lo;
    }
    const int full = m >= 8 ? m - (m % 8) : 0;
    T r = T(0);
    if (full > 0) {
      // leaves hold <= 128 elements: all 16 loads of a lane are issued first
      T v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = (8 * q < full) ? get(lo + 8 * q + j) : T(0);
      r = v[0];
#pragma unroll
      for (int q = 1; q < 16; ++q)
        if (8 * q < full) r = r + v[q];
    }
    r = r + __shfl_xor_sync(0xffffffffu, r, 1);
    r = r + __shfl_xor_sync(0xffffffffu, r, 2);
    r = r + __shfl_xor_sync(0xffffffffu, r, 4);
    if (leaf < L && j == 0) {
      T res = full > 0 ? r : T(0);
      for (int i = full; i < m; ++i) res = res + get(lo + i);
      vals[leaf] = res;
    }
  }
  __syncthreads();
  const int H = plan.levels();
  const int32_t* nd = plan.nodes();
  for (int h = 0; h < H; ++h) {
    const int b = plan.level_begin(h), e = plan.level_begin(h + 1);
    for (int jn = b + threadIdx.x; jn < e; jn += blockDim.x) {
      const int dst = nd[3 * jn], a = nd[3 * jn + 1], c = nd[3 * jn + 2];
      vals[dst] = vals[a] + vals[c];
    }
    __syncthreads();
  }
  T res = vals[plan.root()];
  __syncthreads();
  return res;
}

}  // namespace ac
