// theta.cuh -- on-the-fly sketching operator Theta (device side), generated in registers and
// never stored in HBM ("seeded random number generator, implying negligible memory
// consumption of Theta"; "Theta ... possibly provided as a function handle").
//
// Normative definition: DESIGN.md "Theta specification" (readings A1-A4).  This file is an
// independent implementation of that text; it shares no code with oracle/.  Every fp32 step is a
// single correctly-rounded IEEE operation written with __f*_rn intrinsics so nvcc cannot contract
// or reassociate it -- that is what makes the exported Theta bit-identical to the CPU oracle.
#pragma once
#include <cstdint>

namespace rcq {

// Philox4x32-10 bijection (Salmon et al. SC'11): ctr (4 words), key (2 words).
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    if (round > 0) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
  }
  return c;
}

// Counter layout (A2): ctr = (lo32(i), hi32(i), q, domain), key = (lo32(seed), hi32(seed)).
enum : uint32_t { kDomainGauss = 1u, kDomainSparse = 2u };

__device__ __forceinline__ uint4 philox_at(uint64_t seed, uint64_t i, uint32_t q, uint32_t domain) {
  return philox4x32_10(make_uint4((uint32_t)i, (uint32_t)(i >> 32), q, domain), (uint32_t)seed,
                       (uint32_t)(seed >> 32));
}

// ln(a), a in [2^-24, 1]: a = 2^e f, f in [sqrt(1/2), sqrt(2)); t = (f-1)/(f+1);
// ln f = 2t + t^3 (2/3 + t^2 (2/5 + t^2 (2/7 + t^2 * 2/9))); ln a = e ln2_hi + (e ln2_lo + ln f).
__device__ __forceinline__ float ln_unit(float a) {
  const uint32_t bits = __float_as_uint(a);
  int e = (int)(bits >> 23) - 127;
  float f = __uint_as_float((bits & 0x007FFFFFu) | 0x3F800000u);
  if (f > 0x1.6a09e6p+0f) { f = __fmul_rn(f, 0.5f); e += 1; }
  const float t = __fdiv_rn(__fsub_rn(f, 1.0f), __fadd_rn(f, 1.0f));
  const float t2 = __fmul_rn(t, t);
  float p = 0x1.c71c72p-3f;
  p = __fmaf_rn(p, t2, 0x1.24924ap-2f);
  p = __fmaf_rn(p, t2, 0x1.99999ap-2f);
  p = __fmaf_rn(p, t2, 0x1.555556p-1f);
  const float lnf = __fmaf_rn(__fmul_rn(t, t2), p, __fmul_rn(2.0f, t));
  const float ef = (float)e;  // exact: |e| <= 24
  return __fmaf_rn(ef, 0x1.62e4p-1f, __fmaf_rn(ef, 0x1.7f7d1cp-20f, lnf));
}

// sin/cos(2 pi b), b in [0,1): x = 4b, n = floor(x + 1/2), r = x - n; angle = n pi/2 + (pi/2) r.
__device__ __forceinline__ void sincos_2pi(float b, float& so, float& co) {
  const float x = __fmul_rn(4.0f, b);
  const float nf = floorf(__fadd_rn(x, 0.5f));
  const float r = __fsub_rn(x, nf);
  const int n = ((int)nf) & 3;
  const float r2 = __fmul_rn(r, r);
  float ps = 0x1.507834p-13f;
  ps = __fmaf_rn(ps, r2, -0x1.32d2ccp-8f);
  ps = __fmaf_rn(ps, r2, 0x1.466bc6p-4f);
  ps = __fmaf_rn(ps, r2, -0x1.4abbcep-1f);
  ps = __fmaf_rn(ps, r2, 0x1.921fb6p+0f);
  const float s = __fmul_rn(ps, r);
  float pc = -0x1.a6d1f2p-16f;
  pc = __fmaf_rn(pc, r2, 0x1.e1f506p-11f);
  pc = __fmaf_rn(pc, r2, -0x1.55d3c8p-6f);
  pc = __fmaf_rn(pc, r2, 0x1.03c1f0p-2f);
  pc = __fmaf_rn(pc, r2, -0x1.3bd3ccp+0f);
  const float c = __fmaf_rn(pc, r2, 1.0f);
  so = (n == 0) ? s : (n == 1) ? c : (n == 2) ? -s : -c;
  co = (n == 0) ? c : (n == 1) ? -s : (n == 2) ? -c : s;
}

// Box-Muller on one Philox word pair: z_a = rho cos, z_b = rho sin.
__device__ __forceinline__ void box_muller(uint32_t wa, uint32_t wb, float& za, float& zb) {
  const float ua = __fmul_rn(__uint2float_rn((wa >> 8) + 1u), 0x1p-24f);  // (0, 1]
  const float ub = __fmul_rn(__uint2float_rn(wb >> 8), 0x1p-24f);         // [0, 1)
  const float rho = __fsqrt_rn(__fmul_rn(-2.0f, ln_unit(ua)));
  float s, c;
  sincos_2pi(ub, s, c);
  za = __fmul_rn(rho, c);
  zb = __fmul_rn(rho, s);
}

// Four unscaled N(0,1) draws for Theta rows 4q..4q+3 at global X-row i (Gaussian domain).
__device__ __forceinline__ float4 gauss4(uint64_t seed, uint64_t i, uint32_t q) {
  const uint4 w = philox_at(seed, i, q, kDomainGauss);
  float4 z;
  box_muller(w.x, w.y, z.x, z.y);
  box_muller(w.z, w.w, z.z, z.w);
  return z;
}

// Sparse-sign column (A3): half-word t of Philox(i, t/8, domain 2) selects row t*beta +
// ((h & 0x7FFF) * beta >> 15) inside block t and sign (h >> 15 ? -1 : +1).
__device__ __forceinline__ uint32_t sparse_halfword(const uint4& w, int t) {
  const int u = (t & 7) >> 1;
  const uint32_t word = (u == 0) ? w.x : (u == 1) ? w.y : (u == 2) ? w.z : w.w;
  return (t & 1) ? (word >> 16) : (word & 0xFFFFu);
}
__device__ __forceinline__ int sparse_row(uint32_t h, int t, int beta) {
  return t * beta + (int)(((h & 0x7FFFu) * (uint32_t)beta) >> 15);
}

}  // namespace rcq
