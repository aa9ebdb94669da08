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

}  // namespace ac
