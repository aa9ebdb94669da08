// Shared device helpers for the AdaCluster sm_100a kernels.
//
// Everything on the clustering / selection path must reproduce the reference's
// numpy + OpenBLAS arithmetic bit-for-bit, so these
// files are compiled with --fmad=false and every fused multiply-add that the
// reference performs is written explicitly with __fmaf_rn.  The attention
// kernels live in separate translation units that allow contraction.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/adacluster_sm100.h"

#define AC_DEV __device__ __forceinline__

namespace ac {

constexpr int kWarp = 32;
// tensor-core assignment (assign_tc.cu): centres per pass, and the internal
// flag that skips its per-tile label histogram (chunked passes rebuild it)
constexpr int kAsgTcChunk = 128;
constexpr int kAsgNoHist = 1 << 8;

// ---------------------------------------------------------------------------
// element loads: the clustering path reads keys either as f32 or as bf16
// (bf16 -> f32 is exact, so the arithmetic on the upcast values is identical
// to the oracle's arithmetic on the f32 copy).
// ---------------------------------------------------------------------------
AC_DEV float ld_elem(const void* base, int dtype, int64_t i) {
  if (dtype == AC_DTYPE_BF16) {
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(base)[i]);
  }
  return reinterpret_cast<const float*>(base)[i];
}

// ---------------------------------------------------------------------------
// numpy pairwise summation (numpy/_core/src/umath/loops_utils.h.src,
// pairwise_sum): n < 8 -> sequential from 0; n <= 128 -> 8 strided
// accumulators combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then the tail;
// otherwise split at n2 = n/2 - (n/2 % 8) and recurse.
// Used for every `.sum(axis=1)` and `np.linalg.norm(axis=1)` over D.
// ---------------------------------------------------------------------------
template <typename T, typename Get>
AC_DEV T pw_leaf(const Get& get, int lo, int n) {
  if (n < 8) {
    T res = T(0);
    for (int i = 0; i < n; ++i) res = res + get(lo + i);
    return res;
  }
  T r0 = get(lo + 0), r1 = get(lo + 1), r2 = get(lo + 2), r3 = get(lo + 3);
  T r4 = get(lo + 4), r5 = get(lo + 5), r6 = get(lo + 6), r7 = get(lo + 7);
  int i = 8;
  const int full = n - (n % 8);
  for (; i < full; i += 8) {
    r0 = r0 + get(lo + i + 0); r1 = r1 + get(lo + i + 1);
    r2 = r2 + get(lo + i + 2); r3 = r3 + get(lo + i + 3);
    r4 = r4 + get(lo + i + 4); r5 = r5 + get(lo + i + 5);
    r6 = r6 + get(lo + i + 6); r7 = r7 + get(lo + i + 7);
  }
  T res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
  for (; i < n; ++i) res = res + get(lo + i);
  return res;
}

// Arbitrary n (short vectors: D, or k <= a few thousand): the recursion
// depth is log2(n/128)+1, so plain device recursion is fine.
template <typename T, typename Get>
__device__ T pw_sum_rec(const Get& get, int lo, int n) {
  if (n <= 128) return pw_leaf<T>(get, lo, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  T a = pw_sum_rec<T>(get, lo, n2);
  T b = pw_sum_rec<T>(get, lo + n2, n - n2);
  return a + b;
}
template <typename T, typename Get>
AC_DEV T pw_sum(const Get& get, int n) {
  if (n <= 128) return pw_leaf<T>(get, 0, n);
  return pw_sum_rec<T>(get, 0, n);
}

// numpy elementwise semantics that differ from the CUDA intrinsics on
// signed zeros: np.maximum(a, b) = (a >= b || isnan(a)) ? a : b
AC_DEV float np_maximum(float a, float b) { return (a >= b || isnan(a)) ? a : b; }
AC_DEV float np_minimum(float a, float b) { return (a <= b || isnan(a)) ? a : b; }

// d = (xx - 2 xc) + cc, clipped at 0 exactly as np.maximum(d, 0.0)
// (clustering.py:70-75); explicit intrinsics, never contracted
AC_DEV float sq_dist(float xx, float xc, float cc) {
  float d = __fadd_rn(__fsub_rn(xx, __fmul_rn(2.f, xc)), cc);
  return np_maximum(d, 0.f);
}

AC_DEV float warp_min_f(float v) {
  for (int o = 16; o; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// (value, index) lexicographic argmin helper: smaller value wins, ties -> smaller index
AC_DEV void argmin_merge(float& bd, int& bi, float od, int oi) {
  if (od < bd || (od == bd && oi < bi)) { bd = od; bi = oi; }
}
// argmax with ties -> smaller index (numpy argmax returns the first maximum)
AC_DEV void argmax_merge(float& bd, int64_t& bi, float od, int64_t oi) {
  if (od > bd || (od == bd && oi < bi)) { bd = od; bi = oi; }
}

// Programmatic dependent launch.  A kernel of a Lloyd chain that may be
// launched with the programmatic-serialisation attribute starts with
// pdl_wait() (griddepcontrol.wait: returns once the previous kernel of the
// stream has completed and its memory is visible; a no-op for a normal
// launch), so nothing it reads can be stale.  The next kernel of the stream
// is then set up while this one drains, which hides part of the launch
// latency of the ~125 dependent launches of a 25-iteration chain.
AC_DEV void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
#ifndef AC_PDL_EARLY
// 1: trigger at kernel start (the next grid's CTAs wait on SM slots while
// this one runs -- faster for a lone chain, C1 1.135 vs 1.152 ms, but it
// starves concurrent chains, C2 29.3 vs 25.6 ms); 0: no explicit trigger,
// the next grid launches as this one's CTAs exit (the default)
#define AC_PDL_EARLY 0
#endif
AC_DEV void pdl_trigger() {
#if AC_PDL_EARLY
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
#endif
}

}  // namespace ac

// host-side error reporting shared by every translation unit
namespace ac_host {
void set_error(const char* fmt, ...);
int check_cuda(cudaError_t e, const char* what);
// cudaFuncAttributeMaxDynamicSharedMemorySize for `fn` on the CURRENT device,
// raised only when a call needs more than already set for (kernel, device) --
// thread-safe, so one process may drive
// several GPUs from several threads.
int func_smem(const void* fn, int bytes, const char* what);
// multiprocessor count of the current device (cached per device)
int sm_count();
// programmatic dependent launches of the Lloyd-chain kernels (env AC_PDL, default on)
bool pdl_on();

// kern<<<grid, block, smem, st>>>(args...) with the programmatic stream
// serialisation attribute when pdl_on(): the kernel must begin with
// ac::pdl_wait()
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_on() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}
}  // namespace ac_host

#define AC_CHECK_LAUNCH(what)                                                   \
  do {                                                                          \
    cudaError_t _e = cudaGetLastError();                                        \
    if (_e != cudaSuccess) return ac_host::check_cuda(_e, what);                \
  } while (0)
