/*
 * oracle.c -- plain, slow, obviously-correct CPU fp64 oracle for the direct randomized
 * Cholesky QR (RCholeskyQR, Algorithm 2 of Balabanov, arXiv 2210.09953).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2210_09953_b200/) never imports, links or executes anything under oracle/, and
 * this file shares no code, header, table or constant generator with it.
 *
 * What it computes (alg:RCQR; alg:RCQR2, and alg:oneRCQR,
 * PAPER.md:263-276, below):
 *     1. P <- Theta X   oracle_sketch
 *     2. [R, S] <- QR(P)   oracle_householder  (Householder)
 *     3. Q <- X R^{-1}   oracle_forward_subst (forward substitution,
 *                                                 PAPER.md:178, row-wise)
 * Theta is defined normatively in DESIGN.md section "Theta specification" (readings A1-A4):
 * Philox4x32-10 keyed by (seed, global row i, block q, domain), Box-Muller in fp32 with
 * fixed polynomials, scaled by fl64(1/sqrt(k)) (Gaussian, "scaled by a factor
 * sqrt(1/k)"), or an OSNAP-style sparse-sign map (BASELINE.json C4; reading A3).
 *
 * Precision: every step of the method is fp64 (PAPER.md:83, 406 -- minor operations in
 * higher precision; reading A7: step 3 in fp64 rounded once to Q's dtype).  The only fp32
 * arithmetic is inside the normative definition of Theta (the normal transform), which is
 * written with explicit fmaf and compiled with -ffp-contract=off.
 *
 * Layouts: X (m x n, leading dim ldx), Q (m x n, ldq), P (k x n), R (n x n), S (k x n) are
 * all ROW-MAJOR.  dtype 0 = fp64, 1 = fp32 for X and Q.
 *
 * Sketch accuracy (reading A15): the paper performs "random projections and low-dimensional
 * operations" with a unit roundoff u_f lower than u (u_f = O(u/(mn)) for the
 * sketch).  The oracle therefore evaluates every sketch sum with the compensated
 * dot product Dot2 (Ogita, Rump, Oishi, SIAM J. Sci. Comput. 26(6), 2005: TwoProduct by fma +
 * TwoSum), i.e. as if in twice the working precision, so that it is a reference for P rather
 * than one more fp64 summation order.
 *
 * Determinism: the sketch sums fixed 65536-row blocks (independent of thread count) and adds
 * the block partials in block order; Householder is serial; substitution is per row.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { OR_OK = 0, OR_E_INVALID = 1, OR_E_SHAPE = 2, OR_E_NONFINITE = 3, OR_E_SINGULAR = 4,
       OR_E_NOMEM = 7 };
enum { OR_GAUSSIAN = 0, OR_SPARSE_SIGN = 1, OR_RADEMACHER = 2, OR_SRHT = 3 };
#define OR_SRHT_LOG2M 48   /* the SRHT's Hadamard order m' = 2^48 (reading A23) */
#define OR_SKETCH_BLOCK 65536

/* ------------------------------------------------------------------------------------------
 * Philox4x32-10 (Salmon et al., SC'11; the generator BASELINE.json's north star names).
 * One round: (hi0,lo0) = M0*c0, (hi1,lo1) = M1*c2;
 *            c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0);   key bumped by (W0, W1) between
 * rounds.  10 rounds.
 * ---------------------------------------------------------------------------------------- */
void oracle_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    uint32_t c[4] = {ctr_in[0], ctr_in[1], ctr_in[2], ctr_in[3]};
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        if (round > 0) { k0 += W0; k1 += W1; }
        uint64_t p0 = (uint64_t)M0 * c[0];
        uint64_t p1 = (uint64_t)M1 * c[2];
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c[1] ^ k0, n1 = lo1, n2 = hi0 ^ c[3] ^ k1, n3 = lo0;
        c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* Counter layout (reading A2): ctr = (lo32(i), hi32(i), q, domain), key = (lo32(seed), hi32(seed)). */
static void philox_for(uint64_t seed, uint64_t i, uint32_t q, uint32_t domain, uint32_t out[4]) {
    uint32_t ctr[4] = {(uint32_t)i, (uint32_t)(i >> 32), q, domain};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    oracle_philox4x32_10(ctr, key, out);
}

/* ------------------------------------------------------------------------------------------
 * Normative fp32 normal transform (reading A1).  All operations are single correctly-rounded
 * IEEE fp32 operations in the order written.
 * ---------------------------------------------------------------------------------------- */
static float u32_as_f32(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t f32_as_u32(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/* float(e) for a small integer e without a conversion instruction: 0x4B400000 is 1.5 * 2^23. */
static float small_int_to_f32(int e) { return u32_as_f32((uint32_t)(0x4B400000 + e)) - 12582912.0f; }

/* natural log for a in [2^-23, 1] (reading A1): a = 2^e f with f in [sqrt(1/2), sqrt(2)),
 * s = f - 1 (exact), ln f = s P(s) with P the degree-9 polynomial below (Chebyshev fit of
 * ln(1+s)/s on [sqrt(1/2)-1, sqrt(2)-1], coefficients rounded to fp32), Horner with fmaf;
 * ln a = e*ln2_hi + (e*ln2_lo + ln f).  No division. */
float oracle_ln32(float a) {
    uint32_t bits = f32_as_u32(a);
    int e = (int)(bits >> 23) - 127;
    float f = u32_as_f32((bits & 0x007FFFFFu) | 0x3F800000u);
    if (f > 0x1.6a09e6p+0f) { f = f * 0.5f; e = e + 1; }
    float s = f - 1.0f;
    float p = -0x1.31335cp-4f;
    p = fmaf(p, s, 0x1.064786p-3f);
    p = fmaf(p, s, -0x1.0fb036p-3f);
    p = fmaf(p, s, 0x1.22cf10p-3f);
    p = fmaf(p, s, -0x1.5423b0p-3f);
    p = fmaf(p, s, 0x1.999e86p-3f);
    p = fmaf(p, s, -0x1.000424p-2f);
    p = fmaf(p, s, 0x1.55555ep-2f);
    p = fmaf(p, s, -0x1.fffff8p-2f);
    p = fmaf(p, s, 1.0f);
    float lnf = s * p;
    float ef = small_int_to_f32(e);
    float r = fmaf(ef, 0x1.7f7d1cp-20f, lnf); /* ln2_lo */
    r = fmaf(ef, 0x1.62e4p-1f, r);            /* ln2_hi (16 significant bits: e*ln2_hi exact) */
    return r;
}

/* sin(2 pi b), cos(2 pi b) for b = j 2^-23, j in [0, 2^23) (reading A1): quadrant
 * n = (j + 2^20) >> 21, remainder ri = j - n 2^21 in [-2^20, 2^20), r = ri 2^-21 in [-1/2, 1/2)
 * (exact); angle = n pi/2 + (pi/2) r; Taylor polynomials of sin/cos((pi/2) r) with fmaf. */
void oracle_sincos2pi_j(uint32_t j, float* s_out, float* c_out) {
    uint32_t n = (j + (1u << 20)) >> 21;
    int ri = (int)j - (int)(n << 21);
    float r = small_int_to_f32(ri) * 0x1p-21f;
    float r2 = r * r;
    float ps = 0x1.507834p-13f;
    ps = fmaf(ps, r2, -0x1.32d2ccp-8f);
    ps = fmaf(ps, r2, 0x1.466bc6p-4f);
    ps = fmaf(ps, r2, -0x1.4abbcep-1f);
    ps = fmaf(ps, r2, 0x1.921fb6p+0f);
    float s = ps * r;
    float pc = -0x1.a6d1f2p-16f;
    pc = fmaf(pc, r2, 0x1.e1f506p-11f);
    pc = fmaf(pc, r2, -0x1.55d3c8p-6f);
    pc = fmaf(pc, r2, 0x1.03c1f0p-2f);
    pc = fmaf(pc, r2, -0x1.3bd3ccp+0f);
    float c = fmaf(pc, r2, 1.0f);
    float so, co;
    switch (n & 3u) {
        case 0: so = s; co = c; break;
        case 1: so = c; co = -s; break;
        case 2: so = -s; co = -c; break;
        default: so = -c; co = s; break;
    }
    *s_out = so; *c_out = co;
}

/* Four N(0,1) draws z[0..3] for Theta rows 4q..4q+3 at global X-row i (domain 1): Box-Muller on
 * the word pairs (w0, w1) and (w2, w3) with 23-bit uniforms ua = 2 - (1 + ja 2^-23) in (0, 1]
 * (ja = wa >> 9) and angle index jb = wb >> 9. */
void oracle_gauss4(uint64_t seed, uint64_t i, uint32_t q, float z[4]) {
    uint32_t w[4];
    philox_for(seed, i, q, 1u, w);
    for (int p = 0; p < 2; ++p) {
        uint32_t ja = w[2 * p] >> 9, jb = w[2 * p + 1] >> 9;
        float ua = 2.0f - u32_as_f32(0x3F800000u | ja);   /* exact: 1 - ja 2^-23 */
        float rho = sqrtf(-2.0f * oracle_ln32(ua));
        float s, c;
        oracle_sincos2pi_j(jb, &s, &c);
        z[2 * p] = rho * c;
        z[2 * p + 1] = rho * s;
    }
}

/* Gaussian Theta entry (fp64): Theta_ri = (double) z_ri * fl64(1/sqrt(k)). */
double oracle_theta_gauss(uint64_t seed, int k, uint64_t i, int r) {
    float z[4];
    oracle_gauss4(seed, i, (uint32_t)(r / 4), z);
    double sk = 1.0 / sqrt((double)k);
    return (double)z[r % 4] * sk;
}

/* Sparse-sign column i of Theta (reading A3): zeta blocks of beta = k/zeta rows; half-word t of
 * Philox call (i, q = t/8, domain 2) picks row t*beta + ((h & 0x7FFF) * beta >> 15) and sign
 * (h >> 15) ? -1 : +1.  Value +-1/sqrt(zeta). */
void oracle_sparse_col(uint64_t seed, int k, int zeta, uint64_t i, int32_t* rows, int8_t* signs) {
    int beta = k / zeta;
    uint32_t w[4];
    for (int t = 0; t < zeta; ++t) {
        if (t % 8 == 0) philox_for(seed, i, (uint32_t)(t / 8), 2u, w);
        uint32_t word = w[(t % 8) / 2];
        uint32_t h = (t % 2 == 0) ? (word & 0xFFFFu) : (word >> 16);
        rows[t] = t * beta + (int32_t)(((h & 0x7FFFu) * (uint32_t)beta) >> 15);
        signs[t] = (h >> 15) ? (int8_t)-1 : (int8_t)1;
    }
}

/* Rademacher Theta (reading A22): Theta_ri = s_ri fl64(1/sqrt(k)) with
 * s_ri = +1 if bit (r mod 32) of word ((r mod 128) / 32) of Philox(ctr = (i, q = r / 128, domain 5))
 * is 0, else -1 -- one Philox call gives the signs of 128 consecutive sketch rows. */
int oracle_rademacher_sign(uint64_t seed, uint64_t i, int r) {
    uint32_t w[4];
    philox_for(seed, i, (uint32_t)(r / 128), 5u, w);
    uint32_t word = w[(r % 128) / 32];
    return ((word >> (r % 32)) & 1u) ? -1 : 1;
}

/* SRHT (reading A23; "SRHT", used in all of the paper's experiments):
 * Theta = sqrt(m'/k) R H D with m' = 2^48 (X zero-padded), D = diag(d_i) random signs, H the
 * normalised Walsh-Hadamard matrix, H_si = (-1)^popcount(s & i) / sqrt(m'), R the k sampled rows
 * s_0..s_{k-1}.  Hence Theta_ri = (-1)^popcount(s_r & i) d_i / sqrt(k) -- a dense +-1/sqrt(k) matrix
 * evaluated entry by entry (no transform over m rows, so any row partition just sums).
 *   d_i = +1 if bit 0 of word 0 of Philox(ctr = (i, 0, 6)) is 0, else -1;
 *   s_r = 48-bit value (w1 << 32 | w0) & (2^48 - 1) of Philox(ctr = (r, a, 7)), the attempt a = 0, 1, ...
 *         advancing until s_r differs from s_0..s_{r-1} (sampling without replacement). */
void oracle_srht_rows(uint64_t seed, int k, uint64_t* s) {
    for (int r = 0; r < k; ++r) {
        for (uint32_t a = 0;; ++a) {
            uint32_t w[4];
            philox_for(seed, (uint64_t)r, a, 7u, w);
            uint64_t v = (((uint64_t)w[1] << 32) | w[0]) & ((1ull << OR_SRHT_LOG2M) - 1);
            int dup = 0;
            for (int q = 0; q < r && !dup; ++q) dup = s[q] == v;
            if (!dup) { s[r] = v; break; }
        }
    }
}
int oracle_srht_sign(uint64_t seed, uint64_t s_r, uint64_t i) {
    uint32_t w[4];
    philox_for(seed, i, 0u, 6u, w);
    int d = (w[0] & 1u) ? -1 : 1;
    int h = (__builtin_popcountll(s_r & i) & 1) ? -1 : 1;
    return h * d;
}

/* ---------------- batch helpers for the tests ---------------- */
void oracle_ln32_batch(const float* a, float* out, int64_t n) {
    for (int64_t t = 0; t < n; ++t) out[t] = oracle_ln32(a[t]);
}
void oracle_sincos2pi_j_batch(const uint32_t* j, float* s, float* c, int64_t n) {
    for (int64_t t = 0; t < n; ++t) oracle_sincos2pi_j(j[t], &s[t], &c[t]);
}
/* Z: k x m row-major, Z[r*m + (i-row_offset)] = z_ri (unscaled N(0,1) draw, fp32). */
void oracle_theta_gauss_z(uint64_t seed, int k, int64_t row_offset, int64_t m, float* Z) {
    #pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < m; ++ii) {
        float z[4];
        for (int q = 0; q < (k + 3) / 4; ++q) {
            oracle_gauss4(seed, (uint64_t)(row_offset + ii), (uint32_t)q, z);
            for (int t = 0; t < 4 && 4 * q + t < k; ++t) Z[(int64_t)(4 * q + t) * m + ii] = z[t];
        }
    }
}
/* S: k x m row-major int8 signs of the Rademacher Theta (unscaled). */
void oracle_theta_rademacher(uint64_t seed, int k, int64_t row_offset, int64_t m, int8_t* S) {
    #pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < m; ++ii)
        for (int r = 0; r < k; ++r)
            S[(int64_t)r * m + ii] = (int8_t)oracle_rademacher_sign(seed, (uint64_t)(row_offset + ii), r);
}
/* S: k x m row-major int8 signs of the SRHT Theta (unscaled). */
void oracle_theta_srht(uint64_t seed, int k, int64_t row_offset, int64_t m, int8_t* S) {
    uint64_t* sr = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(k > 0 ? k : 1));
    oracle_srht_rows(seed, k, sr);
    #pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < m; ++ii)
        for (int r = 0; r < k; ++r)
            S[(int64_t)r * m + ii] = (int8_t)oracle_srht_sign(seed, sr[r], (uint64_t)(row_offset + ii));
    free(sr);
}
/* rows/signs: m x zeta row-major. */
void oracle_theta_sparse(uint64_t seed, int k, int zeta, int64_t row_offset, int64_t m,
                         int32_t* rows, int8_t* signs) {
    #pragma omp parallel for schedule(static)
    for (int64_t ii = 0; ii < m; ++ii)
        oracle_sparse_col(seed, k, zeta, (uint64_t)(row_offset + ii), rows + ii * zeta,
                          signs + ii * zeta);
}

static double load_x(const void* X, int dtype, int64_t idx) {
    return dtype == 0 ? ((const double*)X)[idx] : (double)((const float*)X)[idx];
}

/* Dot2 accumulator (Ogita-Rump-Oishi 2005, Alg. 5.3): s + c carries the sum of a*b terms.
 * TwoProduct: p = fl(a b), e = fma(a, b, -p) exact.  TwoSum: t = s + p, z = t - s,
 * err = (s - (t - z)) + (p - z) exact. */
static void dot2_add(double* s, double* c, double a, double b) {
    double p = a * b;
    double e = fma(a, b, -p);
    double t = *s + p;
    double z = t - *s;
    double err = (*s - (t - z)) + (p - z);
    *s = t;
    *c += err + e;
}
static void sum2_add(double* s, double* c, double v) {
    double t = *s + v;
    double z = t - *s;
    double err = (*s - (t - z)) + (v - z);
    *s = t;
    *c += err;
}

/* ------------------------------------------------------------------------------------------
 * Step 1: P = Theta X.  P_rj = sum_i Theta_ri x_ij, fp64, i ascending inside
 * fixed 65536-row blocks, block partials added in block order.  Theta is keyed by the GLOBAL
 * row index row_offset + i (so a row-partitioned X gives the same Theta for any partition).
 * ---------------------------------------------------------------------------------------- */
int oracle_sketch(const void* X, int dtype, int64_t m, int n, int64_t ldx, int64_t row_offset,
                  int k, int sketch, int zeta, uint64_t seed, double* P) {
    if (!P || (m > 0 && !X) || n < 1 || k < 1 || ldx < n || m < 0) return OR_E_INVALID;
    if (sketch == OR_SPARSE_SIGN && (zeta < 1 || zeta > k || k % zeta != 0)) return OR_E_SHAPE;
    int64_t nb = (m + OR_SKETCH_BLOCK - 1) / OR_SKETCH_BLOCK;
    size_t kn = (size_t)k * n;
    double* part = (double*)calloc((size_t)(nb > 0 ? nb : 1) * kn, sizeof(double));
    double* comp = (double*)calloc((size_t)(nb > 0 ? nb : 1) * kn, sizeof(double));
    uint64_t* srows = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)k);
    if (!part || !comp || !srows) { free(part); free(comp); free(srows); return OR_E_NOMEM; }
    if (sketch == OR_SRHT) oracle_srht_rows(seed, k, srows);
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nb; ++b) {
        double* Pb = part + (size_t)b * kn;
        double* Cb = comp + (size_t)b * kn;
        double* th = (double*)malloc(sizeof(double) * (size_t)k);
        int32_t* rows = (int32_t*)malloc(sizeof(int32_t) * (size_t)(zeta > 0 ? zeta : 1));
        int8_t* sg = (int8_t*)malloc((size_t)(zeta > 0 ? zeta : 1));
        double sk = 1.0 / sqrt((double)k);
        double sz = zeta > 0 ? 1.0 / sqrt((double)zeta) : 0.0;
        int64_t i0 = b * OR_SKETCH_BLOCK, i1 = i0 + OR_SKETCH_BLOCK < m ? i0 + OR_SKETCH_BLOCK : m;
        for (int64_t i = i0; i < i1; ++i) {
            uint64_t gi = (uint64_t)(row_offset + i);
            if (sketch == OR_GAUSSIAN || sketch == OR_RADEMACHER || sketch == OR_SRHT) {
                if (sketch == OR_SRHT) {
                    for (int r = 0; r < k; ++r) th[r] = oracle_srht_sign(seed, srows[r], gi) > 0 ? sk : -sk;
                } else if (sketch == OR_GAUSSIAN) {
                    float z[4];
                    for (int q = 0; q < (k + 3) / 4; ++q) {
                        oracle_gauss4(seed, gi, (uint32_t)q, z);
                        for (int t = 0; t < 4 && 4 * q + t < k; ++t) th[4 * q + t] = (double)z[t] * sk;
                    }
                } else {
                    for (int r = 0; r < k; ++r) th[r] = oracle_rademacher_sign(seed, gi, r) > 0 ? sk : -sk;
                }
                for (int r = 0; r < k; ++r) {
                    double* prow = Pb + (size_t)r * n;
                    double* crow = Cb + (size_t)r * n;
                    for (int j = 0; j < n; ++j) dot2_add(&prow[j], &crow[j], th[r], load_x(X, dtype, i * ldx + j));
                }
            } else {
                oracle_sparse_col(seed, k, zeta, gi, rows, sg);
                for (int t = 0; t < zeta; ++t) {
                    double theta = sg[t] > 0 ? sz : -sz;
                    double* prow = Pb + (size_t)rows[t] * n;
                    double* crow = Cb + (size_t)rows[t] * n;
                    for (int j = 0; j < n; ++j) dot2_add(&prow[j], &crow[j], theta, load_x(X, dtype, i * ldx + j));
                }
            }
        }
        free(th); free(rows); free(sg);
    }
    for (size_t t = 0; t < kn; ++t) {
        double s = 0.0, c = 0.0;
        for (int64_t b = 0; b < nb; ++b) {
            sum2_add(&s, &c, part[(size_t)b * kn + t]);
            c += comp[(size_t)b * kn + t];
        }
        P[t] = s + c;
    }
    free(part);
    free(comp);
    free(srows);
    for (size_t t = 0; t < kn; ++t)
        if (!isfinite(P[t])) return OR_E_NONFINITE;
    return OR_OK;
}

/* ------------------------------------------------------------------------------------------
 * Step 2: [R, S] = QR(P), unblocked textbook Householder.
 * For j = 0..n-1 on the working copy A (= P):
 *   alpha = ||A[j:,j]||_2; v = A[j:,j]; v_0 += sign(v_0) alpha  (sign(0) = +1);
 *   H_j = I - v v^T / (alpha |v_0|);  A[j:, l] -= v (v^T A[j:, l]) / (alpha |v_0|), l > j;
 *   R_jj = -sign(x_0) alpha, R_jl = A[j, l].
 * Sign convention (reading A5): rows of R with R_jj < 0 are negated (and the matching columns
 * of S), so diag(R) >= 0.  S = H_0 ... H_{n-1} [I_n; 0] (Alg. 2's S).
 * Returns OR_E_SINGULAR if some R_jj == 0 or is non-finite (reading A6).
 * ---------------------------------------------------------------------------------------- */
int oracle_householder(const double* P, int k, int n, double* R, double* S) {
    if (!P || !R || n < 1 || k < n) return k < n ? OR_E_SHAPE : OR_E_INVALID;
    double* A = (double*)malloc(sizeof(double) * (size_t)k * n);      /* column-major copy */
    double* V = (double*)calloc((size_t)k * n, sizeof(double));       /* reflectors, col-major */
    double* tau = (double*)calloc((size_t)n, sizeof(double));         /* 1/(alpha |v0|) or 0 */
    if (!A || !V || !tau) { free(A); free(V); free(tau); return OR_E_NOMEM; }
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < n; ++j) A[(size_t)j * k + i] = P[(size_t)i * n + j];
    memset(R, 0, sizeof(double) * (size_t)n * n);
    int status = OR_OK;
    for (int j = 0; j < n; ++j) {
        double* a = A + (size_t)j * k;
        double ss = 0.0;
        for (int i = j; i < k; ++i) ss += a[i] * a[i];
        double alpha = sqrt(ss);
        double* v = V + (size_t)j * k;
        if (alpha == 0.0) {               /* zero column: no reflector, R_jj = 0 */
            tau[j] = 0.0;
            R[(size_t)j * n + j] = 0.0;
            for (int l = j + 1; l < n; ++l) R[(size_t)j * n + l] = A[(size_t)l * k + j];
            status = OR_E_SINGULAR;
            continue;
        }
        double sgn = a[j] >= 0.0 ? 1.0 : -1.0;
        for (int i = j; i < k; ++i) v[i] = a[i];
        v[j] = a[j] + sgn * alpha;
        double beta = 1.0 / (alpha * fabs(v[j]));
        tau[j] = beta;
        for (int l = j + 1; l < n; ++l) {
            double* c = A + (size_t)l * k;
            double w = 0.0;
            for (int i = j; i < k; ++i) w += v[i] * c[i];
            w *= beta;
            for (int i = j; i < k; ++i) c[i] -= v[i] * w;
        }
        R[(size_t)j * n + j] = -sgn * alpha;
        for (int l = j + 1; l < n; ++l) R[(size_t)j * n + l] = A[(size_t)l * k + j];
    }
    /* S = H_0 H_1 ... H_{n-1} E, E = [I_n; 0], applied right-to-left. */
    if (S) {
        double* E = (double*)calloc((size_t)k * n, sizeof(double));   /* column-major k x n */
        if (!E) { free(A); free(V); free(tau); return OR_E_NOMEM; }
        for (int j = 0; j < n; ++j) E[(size_t)j * k + j] = 1.0;
        for (int j = n - 1; j >= 0; --j) {
            if (tau[j] == 0.0) continue;
            const double* v = V + (size_t)j * k;
            for (int l = 0; l < n; ++l) {
                double* c = E + (size_t)l * k;
                double w = 0.0;
                for (int i = j; i < k; ++i) w += v[i] * c[i];
                w *= tau[j];
                for (int i = j; i < k; ++i) c[i] -= v[i] * w;
            }
        }
        for (int i = 0; i < k; ++i)
            for (int j = 0; j < n; ++j) S[(size_t)i * n + j] = E[(size_t)j * k + i];
        free(E);
    }
    for (int j = 0; j < n; ++j) {
        double d = R[(size_t)j * n + j];
        if (d < 0.0) {
            for (int l = j; l < n; ++l) R[(size_t)j * n + l] = -R[(size_t)j * n + l];
            if (S) for (int i = 0; i < k; ++i) S[(size_t)i * n + j] = -S[(size_t)i * n + j];
        }
        d = R[(size_t)j * n + j];
        if (d == 0.0 || !isfinite(d)) status = OR_E_SINGULAR;
    }
    free(A); free(V); free(tau);
    return status;
}

/* ------------------------------------------------------------------------------------------
 * Step 3: Q = X R^{-1} by forward substitution, row by row:
 *   q_ij = (x_ij - sum_{l<j, ascending} q_il R_lj) / R_jj  in fp64, rounded once to Q's dtype.
 * ---------------------------------------------------------------------------------------- */
int oracle_forward_subst(const void* X, int dtype, int64_t m, int n, int64_t ldx,
                         const double* R, void* Q, int64_t ldq) {
    if (!R || (m > 0 && (!X || !Q)) || n < 1 || ldx < n || ldq < n || m < 0) return OR_E_INVALID;
    for (int j = 0; j < n; ++j) {
        double d = R[(size_t)j * n + j];
        if (d == 0.0 || !isfinite(d)) return OR_E_SINGULAR;
    }
    #pragma omp parallel
    {
        double* q = (double*)malloc(sizeof(double) * (size_t)n);
        #pragma omp for schedule(static)
        for (int64_t i = 0; i < m; ++i) {
            for (int j = 0; j < n; ++j) {
                double s = load_x(X, dtype, i * ldx + j);
                for (int l = 0; l < j; ++l) s -= q[l] * R[(size_t)l * n + j];
                q[j] = s / R[(size_t)j * n + j];
            }
            if (dtype == 0) {
                for (int j = 0; j < n; ++j) ((double*)Q)[i * ldq + j] = q[j];
            } else {
                for (int j = 0; j < n; ++j) ((float*)Q)[i * ldq + j] = (float)q[j];
            }
        }
        free(q);
    }
    return OR_OK;
}

/* Whole Algorithm 2 on one row block (single process).  P (k x n) and S (k x n) optional. */
int oracle_factor(const void* X, int dtype, int64_t m, int n, int64_t ldx, int64_t row_offset,
                  int k, int sketch, int zeta, uint64_t seed, void* Q, int64_t ldq, double* R,
                  double* P_out, double* S_out) {
    if (k < n) return OR_E_SHAPE;
    double* P = P_out ? P_out : (double*)malloc(sizeof(double) * (size_t)k * n);
    if (!P) return OR_E_NOMEM;
    int st = oracle_sketch(X, dtype, m, n, ldx, row_offset, k, sketch, zeta, seed, P);
    if (st == OR_OK) st = oracle_householder(P, k, n, R, S_out);
    if (st == OR_OK) st = oracle_forward_subst(X, dtype, m, n, ldx, R, Q, ldq);
    if (!P_out) free(P);
    return st;
}

/* ------------------------------------------------------------------------------------------
 * Algorithm 3, RCholeskyQR2 (alg:RCQR2):
 *   1. [Q, S, R] <- RCholeskyQR(X, Theta)          (oracle_factor)
 *   2. A <- Q^T Q                                   (oracle_gram)
 *   3. R' <- chol(A), R <- R' R                     (oracle_cholesky, oracle_trmm_upper)
 *   4. Q <- Q R'^{-1}                               (oracle_forward_subst with R')
 * Implicit form: return Q (step 1) and R' instead of step 4's product.
 * ---------------------------------------------------------------------------------------- */

/* A = Q^T Q (n x n, both triangles), each entry a compensated Dot2 sum over the rows in fixed
 * 65536-row blocks whose partials are added in block order (same accuracy policy as the sketch,
 * reading A15: "low-dimensional operations" in higher precision). */
int oracle_gram(const void* Q, int dtype, int64_t m, int n, int64_t ldq, double* A) {
    if (!A || n < 1 || ldq < n || m < 0 || (m > 0 && !Q)) return OR_E_INVALID;
    int64_t nb = (m + OR_SKETCH_BLOCK - 1) / OR_SKETCH_BLOCK;
    if (nb == 0) nb = 1;
    size_t nn = (size_t)n * n;
    double* part = (double*)calloc((size_t)nb * nn * 2, sizeof(double));
    if (!part) return OR_E_NOMEM;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nb; ++b) {
        double* ps = part + (size_t)b * nn * 2;
        double* pc = ps + nn;
        int64_t i0 = b * OR_SKETCH_BLOCK, i1 = i0 + OR_SKETCH_BLOCK < m ? i0 + OR_SKETCH_BLOCK : m;
        for (int64_t r = i0; r < i1; ++r)
            for (int i = 0; i < n; ++i) {
                double qi = load_x(Q, dtype, r * ldq + i);
                for (int j = i; j < n; ++j)
                    dot2_add(&ps[(size_t)i * n + j], &pc[(size_t)i * n + j], qi, load_x(Q, dtype, r * ldq + j));
            }
    }
    for (int i = 0; i < n; ++i)
        for (int j = i; j < n; ++j) {
            double s = 0.0, c = 0.0;
            for (int64_t b = 0; b < nb; ++b) {
                sum2_add(&s, &c, part[(size_t)b * nn * 2 + (size_t)i * n + j]);
                c += part[(size_t)b * nn * 2 + nn + (size_t)i * n + j];
            }
            A[(size_t)i * n + j] = A[(size_t)j * n + i] = s + c;
        }
    free(part);
    return OR_OK;
}

/* R' upper triangular with A = R'^T R' (textbook Cholesky, row by row, "chol"):
 *   r_ii = sqrt(a_ii - sum_{l<i} r_li^2),  r_ij = (a_ij - sum_{l<i} r_li r_lj) / r_ii  (j > i).
 * A non-positive or non-finite pivot returns OR_E_SINGULAR (A not numerically positive definite). */
int oracle_cholesky(const double* A, int n, double* Rp) {
    if (!A || !Rp || n < 1) return OR_E_INVALID;
    for (size_t c = 0; c < (size_t)n * n; ++c) Rp[c] = 0.0;
    for (int i = 0; i < n; ++i) {
        double d = A[(size_t)i * n + i];
        for (int l = 0; l < i; ++l) d -= Rp[(size_t)l * n + i] * Rp[(size_t)l * n + i];
        if (!(d > 0.0) || !isfinite(d)) return OR_E_SINGULAR;
        double rii = sqrt(d);
        Rp[(size_t)i * n + i] = rii;
        for (int j = i + 1; j < n; ++j) {
            double s = A[(size_t)i * n + j];
            for (int l = 0; l < i; ++l) s -= Rp[(size_t)l * n + i] * Rp[(size_t)l * n + j];
            Rp[(size_t)i * n + j] = s / rii;
        }
    }
    return OR_OK;
}

/* out = U V for upper triangular U, V (n x n): out_ij = sum_{l=i..j} u_il v_lj. */
void oracle_trmm_upper(const double* U, const double* V, int n, double* out) {
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double s = 0.0;
            for (int l = i; l <= j; ++l) s += U[(size_t)i * n + l] * V[(size_t)l * n + j];
            out[(size_t)i * n + j] = j >= i ? s : 0.0;
        }
}

/* Whole Algorithm 3.  Q1 (RCholeskyQR's Q, same dtype as X) and R' (n x n) are outputs too
 * (the implicit-Q form of PAPER.md:206); Q = Q1 R'^{-1} (explicit form), R = R' R1. */
int oracle_factor2(const void* X, int dtype, int64_t m, int n, int64_t ldx, int64_t row_offset,
                   int k, int sketch, int zeta, uint64_t seed, void* Q, int64_t ldq, double* R,
                   void* Q1, double* Rp) {
    if (!Q1 || !Rp || !R || !Q) return OR_E_INVALID;
    double* R1 = (double*)malloc(sizeof(double) * (size_t)n * n);
    double* A = (double*)malloc(sizeof(double) * (size_t)n * n);
    if (!R1 || !A) { free(R1); free(A); return OR_E_NOMEM; }
    int st = oracle_factor(X, dtype, m, n, ldx, row_offset, k, sketch, zeta, seed, Q1, n, R1, NULL, NULL);
    if (st == OR_OK) st = oracle_gram(Q1, dtype, m, n, n, A);
    if (st == OR_OK) st = oracle_cholesky(A, n, Rp);
    if (st == OR_OK) oracle_trmm_upper(Rp, R1, n, R);
    if (st == OR_OK) st = oracle_forward_subst(Q1, dtype, m, n, n, Rp, Q, ldq);
    free(R1);
    free(A);
    return st;
}

/* ------------------------------------------------------------------------------------------
 * Algorithm 5, reduced RCholeskyQR (alg:oneRCQR):
 *   1. P <- Theta X,  Y <- L X          (oracle_sketch, oracle_extract; one pass over X on the GPU)
 *   2. [S, R] <- QR(P)                   (oracle_householder)
 *   3. Z <- Y R^{-1}                     (oracle_forward_subst on the l x n matrix Y, fp64)
 * The extractor L (l x m, "possibly randomized ... possibly provided as a function handle",
 * PAPER.md:266-270) is a Gaussian OSE drawn from the SAME normative Gaussian stream as Theta
 * (reading A20): L_ji = z(seed, i, row l0 + j) * fl64(1/sqrt(l)), with l0 = k when Theta is
 * Gaussian (L continues Theta's rows, so [Theta; L] is one (k + l)-row draw) and l0 = 0 when
 * Theta is sparse-sign (domain 2; the Gaussian stream is then unused by Theta).
 * ---------------------------------------------------------------------------------------- */

/* Y = L X (l x n): Y_jc = sum_i L_ji x_ic with the Dot2 fixed-block policy of oracle_sketch. */
int oracle_extract(const void* X, int dtype, int64_t m, int n, int64_t ldx, int64_t row_offset,
                   int l0, int l, uint64_t seed, double* Y) {
    if (!Y || (m > 0 && !X) || n < 1 || l < 1 || l0 < 0 || ldx < n || m < 0) return OR_E_INVALID;
    int64_t nb = (m + OR_SKETCH_BLOCK - 1) / OR_SKETCH_BLOCK;
    size_t ln = (size_t)l * n;
    double* part = (double*)calloc((size_t)(nb > 0 ? nb : 1) * ln * 2, sizeof(double));
    if (!part) return OR_E_NOMEM;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nb; ++b) {
        double* Yb = part + (size_t)b * ln * 2;
        double* Cb = Yb + ln;
        double* lr = (double*)malloc(sizeof(double) * (size_t)l);
        double sl = 1.0 / sqrt((double)l);
        int64_t i0 = b * OR_SKETCH_BLOCK, i1 = i0 + OR_SKETCH_BLOCK < m ? i0 + OR_SKETCH_BLOCK : m;
        for (int64_t i = i0; i < i1; ++i) {
            uint64_t gi = (uint64_t)(row_offset + i);
            for (int j = 0; j < l; ++j) {
                float z[4];
                int r = l0 + j;
                oracle_gauss4(seed, gi, (uint32_t)(r / 4), z);
                lr[j] = (double)z[r % 4] * sl;
            }
            for (int j = 0; j < l; ++j)
                for (int c = 0; c < n; ++c)
                    dot2_add(&Yb[(size_t)j * n + c], &Cb[(size_t)j * n + c], lr[j], load_x(X, dtype, i * ldx + c));
        }
        free(lr);
    }
    for (size_t t = 0; t < ln; ++t) {
        double s = 0.0, c = 0.0;
        for (int64_t b = 0; b < nb; ++b) {
            sum2_add(&s, &c, part[(size_t)b * ln * 2 + t]);
            c += part[(size_t)b * ln * 2 + ln + t];
        }
        Y[t] = s + c;
    }
    free(part);
    for (size_t t = 0; t < ln; ++t)
        if (!isfinite(Y[t])) return OR_E_NONFINITE;
    return OR_OK;
}

/* Whole Algorithm 5.  Z (l x n fp64) and R (n x n) are outputs; Y (l x n) and S (k x n) optional. */
int oracle_factor_reduced(const void* X, int dtype, int64_t m, int n, int64_t ldx, int64_t row_offset,
                          int k, int sketch, int zeta, uint64_t seed, int l, double* Z, double* R,
                          double* Y_out, double* S_out) {
    if (!Z || !R || l < 1) return OR_E_INVALID;
    if (k < n) return OR_E_SHAPE;
    double* P = (double*)malloc(sizeof(double) * (size_t)k * n);
    double* Y = Y_out ? Y_out : (double*)malloc(sizeof(double) * (size_t)l * n);
    if (!P || !Y) { free(P); if (!Y_out) free(Y); return OR_E_NOMEM; }
    int l0 = sketch == OR_GAUSSIAN ? k : 0;
    int st = oracle_sketch(X, dtype, m, n, ldx, row_offset, k, sketch, zeta, seed, P);
    if (st == OR_OK) st = oracle_extract(X, dtype, m, n, ldx, row_offset, l0, l, seed, Y);
    if (st == OR_OK) st = oracle_householder(P, k, n, R, S_out);
    if (st == OR_OK) st = oracle_forward_subst(Y, 0, l, n, n, R, Z, n);
    free(P);
    if (!Y_out) free(Y);
    return st;
}

/* ------------------------------------------------------------------------------------------
 * Algorithm 7, rank-revealing RCholeskyQR (alg:RRRCholeskyQR), with the column
 * normalisation of PAPER.md:350:
 *   1. P <- Theta X, D = diag(||X(:,j)||_2) in the same pass; P <- P D^{-1}
 *   2. [S, R, Pi] <- RRQR(P): strong rank-revealing QR (Gu & Eisenstat 1996, f = 1.5; PAPER.md:652,
 *      778), reading A21: Businger-Golub column pivoting picks Pi, then -- for the rank r of step 3 --
 *      Gu-Eisenstat swaps of a leading column i and a trailing column r + j while
 *      rho_ij = sqrt((R11^{-1} R12)_ij^2 + (gamma_j(R22) / omega_i(R11))^2) > f.
 *   3. r = min r such that ||R(r+1:n, r+1:n)||_F <= tau ||R||_2
 *   4. Q <- (X Pi(:, 1:r)) R(1:r, 1:r)^{-1}  (with R already post-processed R <- R Pi^T D Pi)
 *   5. R <- R(1:r, :)
 * ---------------------------------------------------------------------------------------- */

/* d_j = ||X(:, j)||_2: compensated sums of squares (Dot2) in the fixed 65536-row blocks. */
int oracle_colnorms(const void* X, int dtype, int64_t m, int n, int64_t ldx, double* d) {
    if (!d || n < 1 || ldx < n || m < 0 || (m > 0 && !X)) return OR_E_INVALID;
    int64_t nb = (m + OR_SKETCH_BLOCK - 1) / OR_SKETCH_BLOCK;
    if (nb == 0) nb = 1;
    double* part = (double*)calloc((size_t)nb * n * 2, sizeof(double));
    if (!part) return OR_E_NOMEM;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nb; ++b) {
        double* ps = part + (size_t)b * n * 2;
        double* pc = ps + n;
        int64_t i0 = b * OR_SKETCH_BLOCK, i1 = i0 + OR_SKETCH_BLOCK < m ? i0 + OR_SKETCH_BLOCK : m;
        for (int64_t i = i0; i < i1; ++i)
            for (int j = 0; j < n; ++j) {
                double x = load_x(X, dtype, i * ldx + j);
                dot2_add(&ps[j], &pc[j], x, x);
            }
    }
    for (int j = 0; j < n; ++j) {
        double s = 0.0, c = 0.0;
        for (int64_t b = 0; b < nb; ++b) {
            sum2_add(&s, &c, part[(size_t)b * n * 2 + j]);
            c += part[(size_t)b * n * 2 + n + j];
        }
        d[j] = sqrt(s + c);
    }
    free(part);
    for (int j = 0; j < n; ++j)
        if (!isfinite(d[j])) return OR_E_NONFINITE;
    return OR_OK;
}

/* Businger-Golub QR with column pivoting of the k x n matrix P (k >= n): at step j the pivot is the
 * first trailing column of largest 2-norm over rows j..k-1 (norms recomputed, not downdated); the
 * reflectors are those of oracle_householder.  Only the permutation is returned (perm[j] = original
 * column in position j); R is recomputed by oracle_householder on P(:, perm), which performs the
 * same operations. */
static int qrcp_perm(const double* P, int k, int n, int* perm) {
    double* A = (double*)malloc(sizeof(double) * (size_t)k * n);   /* column-major working copy */
    if (!A) return OR_E_NOMEM;
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < n; ++j) A[(size_t)j * k + i] = P[(size_t)i * n + j];
    for (int j = 0; j < n; ++j) perm[j] = j;
    for (int j = 0; j < n; ++j) {
        int best = j;
        double bn = -1.0;
        for (int l = j; l < n; ++l) {
            double ss = 0.0;
            for (int i = j; i < k; ++i) ss += A[(size_t)l * k + i] * A[(size_t)l * k + i];
            if (ss > bn) { bn = ss; best = l; }
        }
        if (best != j) {
            for (int i = 0; i < k; ++i) {
                double t = A[(size_t)j * k + i];
                A[(size_t)j * k + i] = A[(size_t)best * k + i];
                A[(size_t)best * k + i] = t;
            }
            int t = perm[j]; perm[j] = perm[best]; perm[best] = t;
        }
        double* a = A + (size_t)j * k;
        double alpha = sqrt(bn);
        if (alpha == 0.0) break;                       /* the trailing columns are all zero */
        double v0 = a[j] + (a[j] >= 0.0 ? alpha : -alpha);
        double scale = 1.0 / (alpha * fabs(v0));
        for (int l = j + 1; l < n; ++l) {
            double* c = A + (size_t)l * k;
            double dot = v0 * c[j];
            for (int i = j + 1; i < k; ++i) dot += a[i] * c[i];
            double t = dot * scale;
            c[j] -= t * v0;
            for (int i = j + 1; i < k; ++i) c[i] -= t * a[i];
        }
        a[j] = a[j] >= 0.0 ? -alpha : alpha;
        for (int i = j + 1; i < k; ++i) a[i] = 0.0;
    }
    free(A);
    return OR_OK;
}

/* ||R||_2 of the n x n upper triangular R (reading A21): 64 power iterations on R^T R from the
 * all-ones vector, sigma = ||R x|| for the final unit x. */
static double norm2_upper(const double* R, int n) {
    double* x = (double*)malloc(sizeof(double) * (size_t)n);
    double* y = (double*)malloc(sizeof(double) * (size_t)n);
    for (int j = 0; j < n; ++j) x[j] = 1.0 / sqrt((double)n);
    double sigma = 0.0;
    for (int it = 0; it <= 64; ++it) {
        for (int i = 0; i < n; ++i) {                  /* y = R x */
            double s = 0.0;
            for (int j = i; j < n; ++j) s += R[(size_t)i * n + j] * x[j];
            y[i] = s;
        }
        double ny = 0.0;
        for (int i = 0; i < n; ++i) ny += y[i] * y[i];
        sigma = sqrt(ny);
        if (it == 64 || sigma == 0.0) break;
        for (int j = 0; j < n; ++j) {                  /* x = R^T y / ||R^T y|| */
            double s = 0.0;
            for (int i = 0; i <= j; ++i) s += R[(size_t)i * n + j] * y[i];
            x[j] = s;
        }
        double nx = 0.0;
        for (int j = 0; j < n; ++j) nx += x[j] * x[j];
        nx = sqrt(nx);
        if (nx == 0.0) break;
        for (int j = 0; j < n; ++j) x[j] /= nx;
    }
    free(x); free(y);
    return sigma;
}

/* Step 3: min r with ||R(r:n, r:n)||_F <= tau ||R||_2 (0-based r = number of kept columns). */
static int rank_rule(const double* R, int n, double tau) {
    double thr = tau * norm2_upper(R, n);
    /* t_r^2 = sum_{i >= r, j >= i} R_ij^2, accumulated from the bottom-right corner */
    double t2 = 0.0;
    int r = n;
    for (int j = n - 1; j >= 0; --j) {               /* t_j^2 = t_{j+1}^2 + row j of the trailing block */
        double row = 0.0;
        for (int l = j; l < n; ++l) row += R[(size_t)j * n + l] * R[(size_t)j * n + l];
        t2 += row;
        if (sqrt(t2) <= thr) r = j;
        else break;
    }
    return r;
}

/* Strong-RRQR check at rank r for the upper triangular R (n x n): returns max rho_ij^2 and its (i, j)
 * (j counted from r), rho_ij^2 = (R11^{-1} R12)_ij^2 + (gamma_j(R22) / omega_i(R11))^2 with
 * omega_i = 1 / ||row i of R11^{-1}||, gamma_j = ||column j of R22||. */
static double strong_rho(const double* R, int n, int r, int* bi, int* bj) {
    double* W = (double*)calloc((size_t)r * r, sizeof(double));   /* R11^{-1}, upper */
    for (int j = 0; j < r; ++j) {                                  /* column j: R11 w = e_j */
        for (int i = j; i >= 0; --i) {
            double s = i == j ? 1.0 : 0.0;
            for (int l = i + 1; l <= j; ++l) s -= R[(size_t)i * n + l] * W[(size_t)l * r + j];
            W[(size_t)i * r + j] = s / R[(size_t)i * n + i];
        }
    }
    double best = -1.0;
    *bi = 0; *bj = 0;
    for (int i = 0; i < r; ++i) {
        double wi2 = 0.0;                                          /* 1 / omega_i^2 */
        for (int l = i; l < r; ++l) wi2 += W[(size_t)i * r + l] * W[(size_t)i * r + l];
        for (int j = 0; j < n - r; ++j) {
            double a = 0.0;                                        /* (R11^{-1} R12)_ij */
            for (int l = i; l < r; ++l) a += W[(size_t)i * r + l] * R[(size_t)l * n + r + j];
            double g2 = 0.0;                                       /* gamma_j^2 */
            for (int l = r; l <= r + j; ++l) g2 += R[(size_t)l * n + r + j] * R[(size_t)l * n + r + j];
            double rho2 = a * a + g2 * wi2;
            if (rho2 > best) { best = rho2; *bi = i; *bj = j; }
        }
    }
    free(W);
    return best;
}

/* RRQR of the k x n matrix P (step 2 + step 3).  Outputs perm (n), R (n x n, of P(:, perm), diag >= 0),
 * S (k x n, optional), *rank, *swaps.  rank_fixed > 0 replaces the tau rule (fixed-rank strong RRQR). */
int oracle_rrqr(const double* P, int k, int n, double tau, double f, int rank_fixed, int* perm, double* R,
                double* S, int* rank, int* swaps) {
    if (!P || !perm || !R || !rank || n < 1) return OR_E_INVALID;
    if (k < n) return OR_E_SHAPE;
    double* Pp = (double*)malloc(sizeof(double) * (size_t)k * n);
    if (!Pp) return OR_E_NOMEM;
    int st = qrcp_perm(P, k, n, perm);
    int nsw = 0, r = 0;
    for (int pass = 0; st == OR_OK; ++pass) {
        for (int i = 0; i < k; ++i)
            for (int j = 0; j < n; ++j) Pp[(size_t)i * n + j] = P[(size_t)i * n + perm[j]];
        st = oracle_householder(Pp, k, n, R, S);
        if (st == OR_E_SINGULAR) st = OR_OK;          /* zero pivots are expected beyond the rank */
        if (st != OR_OK) break;
        if (pass == 0) r = rank_fixed > 0 ? (rank_fixed < n ? rank_fixed : n) : rank_rule(R, n, tau);
        if (r == 0 || r == n || pass >= 64) break;
        int bi, bj;
        if (strong_rho(R, n, r, &bi, &bj) <= f * f) break;
        int t = perm[bi]; perm[bi] = perm[r + bj]; perm[r + bj] = t;
        ++nsw;
    }
    free(Pp);
    *rank = r;
    if (swaps) *swaps = nsw;
    if (st == OR_OK && r == 0) st = OR_E_SINGULAR;
    return st;
}

/* Whole Algorithm 7.  Outputs: Q (m x r, ldq >= n columns available), R (n x n buffer: rows 0..r-1 hold
 * R(1:r, :) Pi^T D Pi, the rest zero), perm (n), *rank, D (n, optional), S (k x n buffer, optional: the
 * first r columns are Alg. 7's S), *swaps. */
int oracle_factor_rr(const void* X, int dtype, int64_t m, int n, int64_t ldx, int64_t row_offset, int k,
                     int sketch, int zeta, uint64_t seed, double tau, double f, int rank_fixed, void* Q,
                     int64_t ldq, double* R, int* perm, int* rank, double* D_out, double* S, int* swaps) {
    if (!R || !perm || !rank || !Q) return OR_E_INVALID;
    if (k < n) return OR_E_SHAPE;
    double* P = (double*)malloc(sizeof(double) * (size_t)k * n);
    double* D = D_out ? D_out : (double*)malloc(sizeof(double) * (size_t)n);
    if (!P || !D) { free(P); if (!D_out) free(D); return OR_E_NOMEM; }
    int st = oracle_sketch(X, dtype, m, n, ldx, row_offset, k, sketch, zeta, seed, P);
    if (st == OR_OK) st = oracle_colnorms(X, dtype, m, n, ldx, D);
    if (st == OR_OK)                                   /* P <- P D^{-1} (zero columns stay zero) */
        for (int i = 0; i < k; ++i)
            for (int j = 0; j < n; ++j) P[(size_t)i * n + j] = D[j] > 0.0 ? P[(size_t)i * n + j] / D[j] : 0.0;
    int r = 0;
    if (st == OR_OK) st = oracle_rrqr(P, k, n, tau, f, rank_fixed, perm, R, S, &r, swaps);
    *rank = r;
    if (st == OR_OK) {
        /* R <- R(1:r, :) Pi^T D Pi: column l of the permuted R is scaled by d_{perm[l]} */
        for (int i = 0; i < n; ++i)
            for (int l = 0; l < n; ++l) R[(size_t)i * n + l] = i < r ? R[(size_t)i * n + l] * D[perm[l]] : 0.0;
        /* Q <- (X Pi(:, 1:r)) R(1:r, 1:r)^{-1} by forward substitution */
        size_t es = dtype == 0 ? 8 : 4;
        void* Xr = malloc(es * (size_t)(m > 0 ? m : 1) * r);
        double* R11 = (double*)malloc(sizeof(double) * (size_t)r * r);
        if (!Xr || !R11) st = OR_E_NOMEM;
        else {
            for (int64_t i = 0; i < m; ++i)
                for (int j = 0; j < r; ++j) {
                    if (dtype == 0) ((double*)Xr)[i * r + j] = ((const double*)X)[i * ldx + perm[j]];
                    else ((float*)Xr)[i * r + j] = ((const float*)X)[i * ldx + perm[j]];
                }
            for (int i = 0; i < r; ++i)
                for (int j = 0; j < r; ++j) R11[(size_t)i * r + j] = R[(size_t)i * n + j];
            void* Qr = malloc(es * (size_t)(m > 0 ? m : 1) * r);
            if (!Qr) st = OR_E_NOMEM;
            else {
                st = oracle_forward_subst(Xr, dtype, m, r, r, R11, Qr, r);
                for (int64_t i = 0; st == OR_OK && i < m; ++i)
                    memcpy((char*)Q + (size_t)i * ldq * es, (char*)Qr + (size_t)i * r * es, es * (size_t)r);
                free(Qr);
            }
        }
        free(Xr); free(R11);
    }
    free(P);
    if (!D_out) free(D);
    return st;
}

/* One sketch entry P_rj = sum_i Theta_ri x_i for a single column x (m fp64 values), in the same
 * fixed-block order as oracle_sketch -- used to check sampled entries of full-size sketches. */
double oracle_sketch_entry(const double* x, int64_t m, int64_t row_offset, int k, int sketch, int zeta,
                           uint64_t seed, int r) {
    /* invalid arguments give NaN (the same rules as oracle_sketch: 0 <= r < k, sparse 1 <= zeta <= k, k % zeta == 0) */
    if (k < 1 || r < 0 || r >= k || m < 0 || (m > 0 && !x)) return NAN;
    if (sketch < OR_GAUSSIAN || sketch > OR_SRHT) return NAN;
    if (sketch == OR_SPARSE_SIGN && (zeta < 1 || zeta > k || k % zeta != 0)) return NAN;
    int64_t nb = (m + OR_SKETCH_BLOCK - 1) / OR_SKETCH_BLOCK;
    uint64_t sr_r = 0;
    if (sketch == OR_SRHT) {
        uint64_t* sr = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)k);
        if (!sr) return NAN;
        oracle_srht_rows(seed, k, sr);
        sr_r = sr[r];
        free(sr);
    }
    double* part = (double*)calloc((size_t)(nb > 0 ? 2 * nb : 2), sizeof(double));
    if (!part) return NAN;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t b = 0; b < nb; ++b) {
        int zc = sketch == OR_SPARSE_SIGN ? zeta : 1;
        int32_t* rows = (int32_t*)malloc(sizeof(int32_t) * (size_t)zc);
        int8_t* sg = (int8_t*)malloc((size_t)zc);
        double acc = (rows && sg) ? 0.0 : NAN, cmp = 0.0;
        double sk = 1.0 / sqrt((double)k), sz = zeta > 0 ? 1.0 / sqrt((double)zeta) : 0.0;
        int64_t i0 = b * OR_SKETCH_BLOCK, i1 = i0 + OR_SKETCH_BLOCK < m ? i0 + OR_SKETCH_BLOCK : m;
        for (int64_t i = i0; i < i1; ++i) {
            uint64_t gi = (uint64_t)(row_offset + i);
            if (sketch == OR_GAUSSIAN) {
                float z[4];
                oracle_gauss4(seed, gi, (uint32_t)(r / 4), z);
                dot2_add(&acc, &cmp, (double)z[r % 4] * sk, x[i]);
            } else if (sketch == OR_RADEMACHER) {
                dot2_add(&acc, &cmp, oracle_rademacher_sign(seed, gi, r) > 0 ? sk : -sk, x[i]);
            } else if (sketch == OR_SRHT) {
                dot2_add(&acc, &cmp, oracle_srht_sign(seed, sr_r, gi) > 0 ? sk : -sk, x[i]);
            } else {
                oracle_sparse_col(seed, k, zeta, gi, rows, sg);
                for (int t = 0; t < zeta; ++t)
                    if (rows[t] == r) dot2_add(&acc, &cmp, sg[t] > 0 ? sz : -sz, x[i]);
            }
        }
        free(rows);
        free(sg);
        part[2 * b] = acc;
        part[2 * b + 1] = cmp;
    }
    double s = 0.0, c = 0.0;
    for (int64_t b = 0; b < nb; ++b) {
        sum2_add(&s, &c, part[2 * b]);
        c += part[2 * b + 1];
    }
    free(part);
    return s + c;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
