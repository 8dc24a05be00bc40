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
enum : uint32_t { kDomainGauss = 1u, kDomainSparse = 2u, kDomainRademacher = 5u, kDomainSrhtD = 6u,
                  kDomainSrhtRows = 7u };

__device__ __forceinline__ uint4 philox_at(uint64_t seed, uint64_t i, uint32_t q, uint32_t domain) {
  return philox4x32_10(make_uint4((uint32_t)i, (uint32_t)(i >> 32), q, domain), (uint32_t)seed,
                       (uint32_t)(seed >> 32));
}

// Exact small-integer -> fp32 without an I2F: 0x4B400000 is 1.5 * 2^23.
__device__ __forceinline__ float small_int_f32(int e) {
  return __fsub_rn(__int_as_float(0x4B400000 + e), 12582912.0f);
}

// ln(a), a in [2^-23, 1]: a = 2^e f, f in [sqrt(1/2), sqrt(2)), s = f - 1;
// ln f = s P(s), P degree 9 (A1 coefficients); ln a = e ln2_hi + (e ln2_lo + ln f).
__device__ __forceinline__ float ln_unit(float a) {
  const uint32_t bits = __float_as_uint(a);
  int e = (int)(bits >> 23) - 127;
  float f = __uint_as_float((bits & 0x007FFFFFu) | 0x3F800000u);
  if (f > 0x1.6a09e6p+0f) { f = __fmul_rn(f, 0.5f); e += 1; }
  const float s = __fsub_rn(f, 1.0f);
  float p = -0x1.31335cp-4f;
  p = __fmaf_rn(p, s, 0x1.064786p-3f);
  p = __fmaf_rn(p, s, -0x1.0fb036p-3f);
  p = __fmaf_rn(p, s, 0x1.22cf10p-3f);
  p = __fmaf_rn(p, s, -0x1.5423b0p-3f);
  p = __fmaf_rn(p, s, 0x1.999e86p-3f);
  p = __fmaf_rn(p, s, -0x1.000424p-2f);
  p = __fmaf_rn(p, s, 0x1.55555ep-2f);
  p = __fmaf_rn(p, s, -0x1.fffff8p-2f);
  p = __fmaf_rn(p, s, 1.0f);
  const float lnf = __fmul_rn(s, p);
  const float ef = small_int_f32(e);
  return __fmaf_rn(ef, 0x1.62e4p-1f, __fmaf_rn(ef, 0x1.7f7d1cp-20f, lnf));
}

// sin/cos(2 pi j 2^-23): n = (j + 2^20) >> 21, ri = j - n 2^21, r = ri 2^-21; angle = n pi/2 + (pi/2) r.
__device__ __forceinline__ void sincos_2pi_j(uint32_t j, float& so, float& co) {
  const uint32_t n = (j + (1u << 20)) >> 21;
  const int ri = (int)j - (int)(n << 21);
  const float r = __fmul_rn(small_int_f32(ri), 0x1p-21f);
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
  const uint32_t q = n & 3u;
  const float sa = (q & 1u) ? c : s;      // |sin| source
  const float ca = (q & 1u) ? s : c;      // |cos| source
  so = (q >= 2u) ? -sa : sa;
  co = (q == 1u || q == 2u) ? -ca : ca;
}

// Box-Muller on one Philox word pair: ua = 2 - (1 + ja 2^-23) in (0, 1], angle index jb.
__device__ __forceinline__ void box_muller(uint32_t wa, uint32_t wb, float& za, float& zb) {
  const float ua = __fsub_rn(2.0f, __uint_as_float(0x3F800000u | (wa >> 9)));
  const float rho = __fsqrt_rn(__fmul_rn(-2.0f, ln_unit(ua)));
  float s, c;
  sincos_2pi_j(wb >> 9, s, c);
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

// The same four draws with the two Box-Muller pairs evaluated in packed FP32x2 arithmetic (sm_100
// FADD2/FMUL2/FFMA2): every lane of a packed op is one correctly rounded IEEE op, applied in the
// same order as above, so the result is bit-identical to gauss4 (the exported-Theta tests check it)
// while the polynomial work costs half the instructions.  Lane 0 = pair (w.x, w.y), lane 1 =
// pair (w.z, w.w); subtraction a - b is written a + (-b) (identical rounding).
__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

__device__ __forceinline__ float2 ln_unit_x2(float2 a) {
  const uint32_t b0 = __float_as_uint(a.x), b1 = __float_as_uint(a.y);
  int e0 = (int)(b0 >> 23) - 127, e1 = (int)(b1 >> 23) - 127;
  float f0 = __uint_as_float((b0 & 0x007FFFFFu) | 0x3F800000u);
  float f1 = __uint_as_float((b1 & 0x007FFFFFu) | 0x3F800000u);
  if (f0 > 0x1.6a09e6p+0f) { f0 = __fmul_rn(f0, 0.5f); e0 += 1; }
  if (f1 > 0x1.6a09e6p+0f) { f1 = __fmul_rn(f1, 0.5f); e1 += 1; }
  const float2 s = __fadd2_rn(make_float2(f0, f1), f2(-1.0f));
  float2 p = f2(-0x1.31335cp-4f);
  p = __ffma2_rn(p, s, f2(0x1.064786p-3f));
  p = __ffma2_rn(p, s, f2(-0x1.0fb036p-3f));
  p = __ffma2_rn(p, s, f2(0x1.22cf10p-3f));
  p = __ffma2_rn(p, s, f2(-0x1.5423b0p-3f));
  p = __ffma2_rn(p, s, f2(0x1.999e86p-3f));
  p = __ffma2_rn(p, s, f2(-0x1.000424p-2f));
  p = __ffma2_rn(p, s, f2(0x1.55555ep-2f));
  p = __ffma2_rn(p, s, f2(-0x1.fffff8p-2f));
  p = __ffma2_rn(p, s, f2(1.0f));
  const float2 lnf = __fmul2_rn(s, p);
  const float2 ef = __fadd2_rn(make_float2(__int_as_float(0x4B400000 + e0), __int_as_float(0x4B400000 + e1)),
                               f2(-12582912.0f));
  return __ffma2_rn(ef, f2(0x1.62e4p-1f), __ffma2_rn(ef, f2(0x1.7f7d1cp-20f), lnf));
}

__device__ __forceinline__ void sincos_2pi_j_x2(uint32_t j0, uint32_t j1, float2& so, float2& co) {
  const uint32_t n0 = (j0 + (1u << 20)) >> 21, n1 = (j1 + (1u << 20)) >> 21;
  const int r0 = (int)j0 - (int)(n0 << 21), r1 = (int)j1 - (int)(n1 << 21);
  const float2 ri = __fadd2_rn(make_float2(__int_as_float(0x4B400000 + r0), __int_as_float(0x4B400000 + r1)),
                               f2(-12582912.0f));
  const float2 r = __fmul2_rn(ri, f2(0x1p-21f));
  const float2 r2 = __fmul2_rn(r, r);
  float2 ps = f2(0x1.507834p-13f);
  ps = __ffma2_rn(ps, r2, f2(-0x1.32d2ccp-8f));
  ps = __ffma2_rn(ps, r2, f2(0x1.466bc6p-4f));
  ps = __ffma2_rn(ps, r2, f2(-0x1.4abbcep-1f));
  ps = __ffma2_rn(ps, r2, f2(0x1.921fb6p+0f));
  const float2 s = __fmul2_rn(ps, r);
  float2 pc = f2(-0x1.a6d1f2p-16f);
  pc = __ffma2_rn(pc, r2, f2(0x1.e1f506p-11f));
  pc = __ffma2_rn(pc, r2, f2(-0x1.55d3c8p-6f));
  pc = __ffma2_rn(pc, r2, f2(0x1.03c1f0p-2f));
  pc = __ffma2_rn(pc, r2, f2(-0x1.3bd3ccp+0f));
  const float2 c = __ffma2_rn(pc, r2, f2(1.0f));
  const uint32_t q0 = n0 & 3u, q1 = n1 & 3u;
  const float sa0 = (q0 & 1u) ? c.x : s.x, ca0 = (q0 & 1u) ? s.x : c.x;
  const float sa1 = (q1 & 1u) ? c.y : s.y, ca1 = (q1 & 1u) ? s.y : c.y;
  so = make_float2((q0 >= 2u) ? -sa0 : sa0, (q1 >= 2u) ? -sa1 : sa1);
  co = make_float2((q0 == 1u || q0 == 2u) ? -ca0 : ca0, (q1 == 1u || q1 == 2u) ? -ca1 : ca1);
}

__device__ __forceinline__ float4 gauss4_x2(uint64_t seed, uint64_t i, uint32_t q) {
  const uint4 w = philox_at(seed, i, q, kDomainGauss);
  const float2 ua = __fadd2_rn(f2(2.0f), make_float2(-__uint_as_float(0x3F800000u | (w.x >> 9)),
                                                      -__uint_as_float(0x3F800000u | (w.z >> 9))));
  const float2 m2 = __fmul2_rn(f2(-2.0f), ln_unit_x2(ua));
  const float2 rho = make_float2(__fsqrt_rn(m2.x), __fsqrt_rn(m2.y));
  float2 sn, cs;
  sincos_2pi_j_x2(w.y >> 9, w.w >> 9, sn, cs);
  const float2 zc = __fmul2_rn(rho, cs), zs = __fmul2_rn(rho, sn);
  return make_float4(zc.x, zs.x, zc.y, zs.y);
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

// Rademacher signs (reading A22) of sketch rows rb..rb+3 (rb % 4 == 0) at global X-row i:
// bit (r mod 32) of word ((r mod 128) / 32) of Philox(i, r / 128, domain 5); 0 -> +1, 1 -> -1.
__device__ __forceinline__ float4 rademacher4(uint64_t seed, uint64_t i, uint32_t rb) {
  const uint4 w = philox_at(seed, i, rb >> 7, kDomainRademacher);
  const uint32_t q = (rb >> 5) & 3u;
  const uint32_t word = q == 0 ? w.x : (q == 1 ? w.y : (q == 2 ? w.z : w.w));
  const uint32_t b = word >> (rb & 31u);
  return make_float4((b & 1u) ? -1.f : 1.f, (b & 2u) ? -1.f : 1.f, (b & 4u) ? -1.f : 1.f, (b & 8u) ? -1.f : 1.f);
}

// SRHT (reading A23): Theta_ri = (-1)^popcount(s_r & i) d_i / sqrt(k); the sign of rows
// rb..rb+3 at global X-row i given the sampled Hadamard rows s (k of them, device array).
__device__ __forceinline__ float srht_d(uint64_t seed, uint64_t i) {
  return (philox_at(seed, i, 0u, kDomainSrhtD).x & 1u) ? -1.f : 1.f;
}
__device__ __forceinline__ float4 srht4(const uint64_t* __restrict__ s, int k, uint64_t seed, uint64_t i, uint32_t rb) {
  const float d = srht_d(seed, i);
  float v[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const uint64_t sr = (int)rb + t < k ? s[rb + t] : 0ull;
    v[t] = (__popcll(sr & i) & 1) ? -d : d;
  }
  return make_float4(v[0], v[1], v[2], v[3]);
}

}  // namespace rcq
