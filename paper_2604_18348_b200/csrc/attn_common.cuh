// Helpers shared by the tcgen05 attention kernels (attn_fa4.cu, D = 64;
// attn_fa4_d128.cu, D = 128): the A-from-TMEM MMA, TMEM stores, packed
// f32x2 arithmetic (FFMA2 / FADD2), the FMA-pipe exp2 and the K/V tile walk.
#pragma once
#include "tc_common.cuh"

namespace ac {
namespace attn {
using namespace ac::tc;

constexpr int kBN = 128;  // keys per K/V tile

AC_DEV void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                    uint32_t accum) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
// the first 16 words of r
AC_DEV void tmem_st16(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16};\n" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

// packed f32x2 helpers (FFMA2 / FADD2 on sm_100)
AC_DEV uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
AC_DEV void up2(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
AC_DEV uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
AC_DEV uint64_t add2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
AC_DEV uint64_t add2_rm(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// 2^x for a pair on the FMA pipe: x = n + f, f in [0,1), 2^f by a cubic
// (max rel. error 7.5e-5, below the bf16 rounding of P), n into the exponent
AC_DEV void exp2_poly2(float x0, float x1, float& p0, float& p1) {
  const float kMagic = 12582912.f;  // 1.5 * 2^23
  // clamp so that the result exponent stays >= 1 (poly(f) >= 0.9999, n >= -125)
  x0 = fmaxf(x0, -125.f);
  x1 = fmaxf(x1, -125.f);
  const uint64_t x = pk2(x0, x1);
  const uint64_t xr = add2_rm(x, pk2(kMagic, kMagic));          // floor(x) in the low bits
  const uint64_t nf = add2(xr, pk2(-kMagic, -kMagic));          // floor(x) as float
  float n0, n1;
  up2(nf, n0, n1);
  const uint64_t f = add2(x, pk2(-n0, -n1));
  uint64_t p = fma2(pk2(0.07802446f, 0.07802446f), f, pk2(0.22606731f, 0.22606731f));
  p = fma2(p, f, pk2(0.69583344f, 0.69583344f));
  p = fma2(p, f, pk2(0.99992523f, 0.99992523f));
  float q0, q1, r0, r1;
  up2(p, q0, q1);
  up2(xr, r0, r1);
  p0 = __uint_as_float(__float_as_uint(q0) + (__float_as_uint(r0) << 23));
  p1 = __uint_as_float(__float_as_uint(q1) + (__float_as_uint(r1) << 23));
}

AC_DEV uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// the K/V tiles of one work item: its runs walked in BN-key steps
struct TileIter {
  const int32_t* runs;
  int nruns, r, s, e;
  AC_DEV TileIter(const int32_t* runs_, int nruns_) : runs(runs_), nruns(nruns_), r(-1), s(0), e(0) {}
  AC_DEV bool next(int& start, int& nk) {
    while (s >= e) {
      if (++r >= nruns) return false;
      s = runs[2 * r];
      e = runs[2 * r + 1];
    }
    start = s;
    nk = min(kBN, e - s);
    s += kBN;
    return true;
  }
};

}  // namespace attn
}  // namespace ac
