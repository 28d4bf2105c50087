// fastmath.cuh -- fp64 elementary functions for the performance walk mode
// (analytic drift, SDDG_GRAD_ANALYTIC).
//
// Why: the CUDA library's fp64 exp/log/sincos carry their polynomial
// coefficients as 64-bit immediates, which ptxas materialises with two UMOVs
// per coefficient inside the step loop (18% of all issued instructions in the
// first profile, profiles/r01_walk_kernel_ncu_v0_first.txt), and handle
// inf/nan/denormal arguments the walk never produces.  Here:
//   frcp(d), fsqrt_pos(v)          MUFU seed + Newton, d, v > 0 normal
//   fexp_tab(x)                    x <= 0 (drift densities)
//   fm2log_tab(u), flog_tab(u)     u in (2^-54, 1] (Box-Muller radius)
//   fsincos_2pi_tab(u)             u in [0, 1)
//   u01_open_bits, fsincos_2pi_bits  Box-Muller inputs from the raw draws
// use shared-memory tables (glibc-style reductions) and constant-bank or
// immediate coefficients.  Accuracy ~1 ulp (sddg_selftest_fastmath).  The
// reference-parity kernels keep the CUDA library (walk_ref.cu).
#pragma once
#include <cstddef>
#include <cstdint>

namespace sddg {
namespace fm {

constexpr double kLn2Hi = 0.6931471805599453;
constexpr double kLn2Lo = 2.3190468138462996e-17;
constexpr double kRound = 6755399441055744.0;  // 1.5 * 2^52

__device__ __forceinline__ double frcp(double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    // 1/d = r / (1 - e) = r (1 + e + e^2 + ...): one cubic step (error e^3)
    const double e = fma(-d, r, 1.0);
    return fma(r, fma(e, e, e), r);
}

// sqrt(v) for v > 0 normal: rsqrt seed + Newton, no special-case branch
__device__ __forceinline__ double fsqrt_pos(double v) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(v));
    const double h = 0.5 * y;
    double g = v * y;                 // ~sqrt(v)
    const double r = fma(-g, h, 0.5);
    g = fma(g, r, g);
    // one coupled step leaves g with error ~e0^2; the residual correction
    // squares it again (h's own error only enters at second order)
    const double d = fma(-g, g, v);
    return fma(d, h, g);
}

}  // namespace fm
}  // namespace sddg

// ---------------------------------------------------------------------------
// Table-driven variants (glibc-style reductions) used by the walk kernel:
// tables in shared memory replace most polynomial terms.  Tables are built on
// the host in 80-bit long double and rounded once (runtime.cu make_fm_tables);
// each CTA copies them to shared memory at start.
//
// Table sizes: 2^kExBits entries of 2^(j/N) for exp, 2^kLgBits of (1/c, log c)
// for log, 2^kScBits of (sin, cos)(2 pi j/N).  The default (large) tables fill
// 96 KB and leave polynomials of degree 3 (exp), 4 (log1p) and 5/4 (sin/cos);
// they need one 1024-thread CTA per SM (walk_kernel.cuh).  Bigger tables buy
// no further degree (the next terms stay above 2^-53).  SDDG_FM_SMALL selects
// the 7.9 KB set that fits 8 x 128-thread CTAs per SM.
namespace sddg {
namespace fm {

#if defined(SDDG_FM_SMALL)
constexpr int kExBits = 6, kLgBits = 7, kScBits = 8;      // 7.9 KB
#elif defined(SDDG_FM_MEDIUM)
constexpr int kExBits = 10, kLgBits = 10, kScBits = 11;   // 56 KB (A/B: 2.9% slower)
#else
constexpr int kExBits = 12, kLgBits = 11, kScBits = 11;   // 96 KB
#endif
constexpr int kExN = 1 << kExBits, kLgN = 1 << kLgBits, kScN = 1 << kScBits;
// first j with c_j = 1 + (j + 1/2)/kLgN >= sqrt 2 (log(c_j / 2) branch)
constexpr int kLgSplit = kLgBits == 7 ? 53 : (kLgBits == 10 ? 424 : 848);
static_assert(kLgBits == 7 || kLgBits == 10 || kLgBits == 11, "log split index");

struct FmTables {
    double k[32];          // polynomial / reduction constants (FmK), read with LDS so the
                           // step loop does not rematerialise 64-bit immediates (2 UMOV each)
    double e2[kExN];       // 2^(j/kExN)
    double lg[kLgN][2];    // -2 rc_j, 2 log(rc_j) [+2 ln2 for j >= kLgSplit]: rc_j ~ 1/c_j chosen
                           // so that log(rc_j) is within 2^-8 ulp of a double (no lo part)
    double sc[kScN][2];    // sin, cos of 2 pi j / kScN
};

// Table reads.  SDDG_SMEM_ABS=<byte offset of the tables in the CTA's shared
// window>: plain ld.shared at [index + constant], so ptxas does not rebuild
// the dynamic-shared-memory symbol address (S2UR CgaCtaId + 3 uniform ops)
// inside the step loop.  The kernel checks the offset at entry.
#ifdef SDDG_SMEM_ABS
#define SDDG_STR2(x) #x
#define SDDG_STR(x) SDDG_STR2(x)
__device__ __forceinline__ double tab_ld1(uint32_t off) {
    double r;
    asm("ld.shared.f64 %0, [%1+" SDDG_STR(SDDG_SMEM_ABS) "];" : "=d"(r) : "r"(off));
    return r;
}
__device__ __forceinline__ void tab_ld2(uint32_t off, double& a, double& b) {
    asm("ld.shared.v2.f64 {%0, %1}, [%2+" SDDG_STR(SDDG_SMEM_ABS) "];"
        : "=d"(a), "=d"(b)
        : "r"(off));
}
#endif

// indices into FmTables::k (pairs adjacent in use order -> LDS.128)
enum FmK {
    K_E6 = 0, K_E5, K_E4, K_E3,            // 1/720, 1/120, 1/24, 1/6
    K_EXS, K_EXHI, K_EXLO, K_PAD0,         // kExN/ln2, ln2/kExN hi, lo
    K_L7, K_L6, K_L5, K_L3,                // 1/448, 1/192, 1/80, 1/12 (log1p in R = -2r)
    K_LN2HI, K_LN2LO, K_I2D, K_TWOPI,      // 2 ln2 hi, lo, (unused), 2 pi
    K_S7, K_S5, K_S3, K_C6,                // -1/5040, 1/120, -1/6, -1/720
    K_C4, K_OPEN, K_SCB, K_TWOPI53         // 1/24, 1 - 2^-53, 2^52 + 2^52/kScN, 2 pi 2^-53
};
// Constants: SDDG_FM_IMMEDIATES -> 64-bit immediates (ptxas rematerialises
// them with UMOV pairs in the loop); SDDG_FM_LDS_HOISTED -> plain smem reads
// (ptxas hoists and spills them); SDDG_FM_LDS -> one ld.shared per use (adds
// a third of the step's shared-memory wavefronts); default -> __constant__
// bank (LDC or direct operands; no shared-memory traffic).
__device__ __forceinline__ double lds_f64(const double* p) {
    double r;
    asm volatile("ld.shared.f64 %0, [%1];"
                 : "=d"(r)
                 : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
    return r;
}
#if defined(SDDG_FM_IMMEDIATES)
#define FMK(i, v) (v)
#elif defined(SDDG_FM_LDS)
#define FMK(i, v) (lds_f64(&T.k[i]))  // +3.6% vs immediates; keeps the LSU busier than CBANK
#elif defined(SDDG_FM_LDS_HOISTED)
#define FMK(i, v) (T.k[i])
#else
#define SDDG_FM_CBANK
#define FMK(i, v) (kFmC[i])  // default: constant-bank operands (A/B best, +1% vs LDS)
#endif

// host-side values of the reduction constants (runtime.cu fills FmTables::k)
constexpr double kExScale = kExN / 0.69314718055994530941723212145818;
// Low-order coefficients rounded to 21 significant bits (low word zero), so
// each is a 32-bit immediate of its DFMA instead of a constant load: their
// terms are <= 2^-36 of the result, so the 2^-22 coefficient error stays
// below 0.02 ulp.  The reduction scale only picks n (r is exact from n).
constexpr double kE4i = 0x1.55555p-5;    // ~1/24
constexpr double kE3i = 0x1.55555p-3;    // ~1/6
constexpr double kS5i = 0x1.11111p-7;    // ~1/120
constexpr double kC4i = 0x1.55555p-5;    // ~1/24
constexpr double kExScaleI = kExBits == 10 ? 0x1.71547p+10 : 0x1.71547p+6;  // ~N/ln2
constexpr double kExHi = kLn2Hi / kExN;  // exact power-of-two scalings of ln2 hi/lo
constexpr double kExLo = kLn2Lo / kExN;
#ifdef SDDG_FM_CBANK
// the FmTables::k values in FmK order, as a constant bank
static __constant__ double kFmC[32] = {
    1.0 / 720.0, 1.0 / 120.0, 1.0 / 24.0, 1.0 / 6.0,
    kExScale, kExHi, kExLo, 0.0,
    1.0 / 448.0, 1.0 / 192.0, 1.0 / 80.0, 1.0 / 12.0,
    2.0 * kLn2Hi, 2.0 * kLn2Lo, 4503601774854144.0, 6.283185307179586,
    -1.0 / 5040.0, 1.0 / 120.0, -1.0 / 6.0, -1.0 / 720.0,
    1.0 / 24.0, 1.0 - 0x1.0p-53, 4503599627370496.0 + 4503599627370496.0 / kScN,
    6.283185307179586 * 0x1.0p-53};
#endif

// exp(x), x <= 0 (POS: x >= 0): x = (N e + j) ln2/N + r, |r| <= ln2/(2N),
// N = kExN.  The scale exponent is clamped with integer min/max (instead of a
// double fmax): below x = -707.7 the result stays a tiny positive normal, and
// (POS) above 709 a huge finite one, instead of wrapping.
template <bool POS = false>
__device__ __forceinline__ double fexp_tab(const FmTables& T, double x) {
    const double t = kExBits >= 12 ? fma(x, FMK(K_EXS, kExScale), kRound) : fma(x, kExScaleI, kRound);
    const double n = t - kRound;
    double r = fma(n, -FMK(K_EXHI, kExHi), x);
    r = fma(n, -FMK(K_EXLO, kExLo), r);
    double p;
    if constexpr (kExBits >= 12) {
        // e^r - 1 = r + r^2/2 + r^3/6  (|r| <= 8.5e-5: next term ~2e-18)
        p = kE3i;
    } else if constexpr (kExBits >= 10) {
        // e^r - 1 = r + r^2/2 + r^3/6 + r^4/24  (|r| <= 3.4e-4: next term ~4e-20)
        p = fma(r, kE4i, kE3i);
    } else {
        // e^r - 1 = r + r^2/2 + ... + r^6/720  (next term ~3e-20)
        p = fma(r, FMK(K_E6, 0.001388888888888889), FMK(K_E5, 0.008333333333333333));
        p = fma(p, r, FMK(K_E4, 0.041666666666666664));
        p = fma(p, r, FMK(K_E3, 0.16666666666666666));
    }
    p = fma(p, r, 0.5);
    p = fma(p, r, 1.0);
    p = p * r;
    const int ni = POS ? min(__double2loint(t), kExN * 1022) : max(__double2loint(t), -kExN * 1021);
#ifdef SDDG_SMEM_ABS
    const double s = tab_ld1(offsetof(FmTables, e2) + 8u * static_cast<uint32_t>(ni & (kExN - 1)));
#else
    const double s = T.e2[ni & (kExN - 1)];
#endif
    const double v = fma(s, p, s);  // 2^(j/N) e^r
    return __hiloint2double(__double2hiint(v) + ((ni >> kExBits) << 20), __double2loint(v));
}

// -2 log(u), u in (2^-54, 1] (the Box-Muller radius squared): u = 2^k m,
// m in [1,2); c_j = 1 + (j+1/2)/N of m's top kLgBits mantissa bits; rc_j a
// double within a few hundred ulp of 1/c_j whose log is almost exactly a
// double (Gal's accurate-table trick, so one table word suffices);
// r = m rc_j - 1 (|r| <= 1/(2N) + 2^-44); log u = (k + a) ln2 - log(rc_j 2^a)
// + log1p(r), a = [c_j >= sqrt 2] (no cancellation near u = 1).  Everything
// is carried pre-scaled by -2 -- R = -2 r = m (-2 rc_j) + 2, the table's
// 2 log rc_j, the polynomial coefficients scaled by powers of two -- so each
// rounding is the exact -2 multiple of the unscaled one: the result equals
// -2 * log(u) computed the plain way, minus the multiply.
__device__ __forceinline__ double fm2log_tab(const FmTables& T, double u) {
    const int hi = __double2hiint(u);
    const int lo = __double2loint(u);
    const int j = (hi >> (20 - kLgBits)) & (kLgN - 1);
    const int nk = (1023 - (hi >> 20)) - (j >= kLgSplit ? 1 : 0);  // -k >= 0
    const double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);
#ifdef SDDG_SMEM_ABS
    double e0, e1;
    tab_ld2(offsetof(FmTables, lg) + 16u * static_cast<uint32_t>(j), e0, e1);
#else
    const double* e = T.lg[j];
    const double e0 = e[0], e1 = e[1];
#endif
    const double R = fma(m, e0, 2.0);
    double p;
    if constexpr (kLgBits >= 11) {
        // log1p(r) = r - r^2/2 + r^3/3 - r^4/4 (|r| <= 2^-12: next term
        // < 2e-19, 0.02 ulp of any |log u| >= 0.1), Horner in R = -2r
        p = 0.03125;
    } else if constexpr (kLgBits >= 10) {
        // log1p(r) = r - r^2/2 + r^3/3 - r^4/4 + r^5/5 (|r| <= 2^-11: next
        // term ~5e-18 relative), Horner in R = -2r
        p = fma(R, FMK(K_L5, 1.0 / 80.0), 0.03125);
    } else {
        // log1p(r) = r - r^2/2 + ... + r^7/7 (next term ~3e-20), Horner in R
        p = fma(R, FMK(K_L7, 1.0 / 448.0), FMK(K_L6, 1.0 / 192.0));
        p = fma(p, R, FMK(K_L5, 1.0 / 80.0));
        p = fma(p, R, 0.03125);
    }
    p = fma(p, R, FMK(K_L3, 1.0 / 12.0));
    p = fma(p, R, 0.25);
    p = p * R;
    // -k as a double without the conversion pipe: (2^52 + nk) - 2^52
    const double dnk = __hiloint2double(0x43300000, nk) - 4503599627370496.0;
    const double h = fma(dnk, FMK(K_LN2HI, 2.0 * kLn2Hi), e1);
    return h + fma(dnk, FMK(K_LN2LO, 2.0 * kLn2Lo), fma(p, R, R));
}

// log(u), u in (2^-54, 1]: exactly -1/2 of fm2log_tab
__device__ __forceinline__ double flog_tab(const FmTables& T, double u) {
    return -0.5 * fm2log_tab(T, u);
}

// sin d, cos d - 1 for |d| <= pi/kScN, then the table rotation
__device__ __forceinline__ void sincos_rotate(const FmTables& T, int j, double d, double& sn,
                                              double& cs) {
    const double d2 = d * d;
    double ps, pc;
    if constexpr (kScBits >= 11) {
        // sin d = d (1 - d^2/6 + d^4/120), cos d - 1 = d^2 (-1/2 + d^2/24)
        // (|d| <= 1.5e-3: next terms ~3e-21 and ~2e-20)
        ps = fma(d2, kS5i, FMK(K_S3, -0.16666666666666666));
        pc = fma(d2, kC4i, -0.5);
    } else {
        // sin d = d (1 - d^2/6 + d^4/120 - d^6/5040), cos d - 1 = d^2 (-1/2 + d^2/24 - d^4/720)
        ps = fma(d2, FMK(K_S7, -0.0001984126984126984), FMK(K_S5, 0.008333333333333333));
        ps = fma(ps, d2, FMK(K_S3, -0.16666666666666666));
        pc = fma(d2, FMK(K_C6, -0.001388888888888889), FMK(K_C4, 0.041666666666666664));
        pc = fma(pc, d2, -0.5);
    }
    const double sd = fma(ps * d2, d, d);
    const double cm1 = pc * d2;
#ifdef SDDG_SMEM_ABS
    double s0, c0;
    tab_ld2(offsetof(FmTables, sc) + 16u * static_cast<uint32_t>(j), s0, c0);
#else
    const double* e = T.sc[j];
    const double s0 = e[0], c0 = e[1];
#endif
    // big terms first: two roundings of size <= ulp/2 each (selftest <= 3 ulp)
    sn = fma(s0, cm1, fma(c0, sd, s0));
    cs = fma(c0, cm1, fma(-s0, sd, c0));
}

// sin, cos of 2 pi u, u in [0, 1): 2 pi u = 2 pi j/N + d, |d| <= pi/N
__device__ __forceinline__ void fsincos_2pi_tab(const FmTables& T, double u, double& sn,
                                                double& cs) {
    const double t = fma(static_cast<double>(kScN), u, kRound);
    const double q = t - kRound;                       // rint(N u)
    const double d = FMK(K_TWOPI, 6.283185307179586) * fma(-1.0 / kScN, q, u);  // exact f
    sincos_rotate(T, __double2loint(t) & (kScN - 1), d, sn, cs);
}

// Box-Muller inputs straight from the raw 64-bit draws (performance mode):
// the same values as u01_open_d / u01_d without the I2F conversion pipe.
//
// u1 = (2k + 1) 2^-53, k = a >> 12 (rng.hpp:61-63): M = 1 + k 2^-52 is built
// from the bits and M - (1 - 2^-53) is exact (Sterbenz).
__device__ __forceinline__ double u01_open_bits(const FmTables& T, uint64_t a) {
    const uint32_t hi = static_cast<uint32_t>(a >> 44) | 0x3ff00000u;
    const uint32_t lo = static_cast<uint32_t>(a >> 12);
    return __hiloint2double(static_cast<int>(hi), static_cast<int>(lo)) -
           FMK(K_OPEN, 1.0 - 0x1.0p-53);
}

// sin, cos of 2 pi u2 with u2 = k 2^-53, k = b >> 11 (rng.hpp:58): the
// reduction N u2 = j + f (N = 2^B = kScN) is done on the integer k.  With
// s = b + 2^(63-B) (mod 2^64), j = s >> (64-B) (mod N) and
// k - 2^(53-B) j + 2^(52-B) = bits 11..(63-B) of s, so f 2^53 is an exact
// double after one subtraction and d = 2 pi f = (f 2^53)(2 pi 2^-53) rounds
// exactly like 2 pi * f.  Ties (f = +-1/(2N)) round up instead of to even:
// both are correct.
__device__ __forceinline__ void fsincos_2pi_bits(const FmTables& T, uint64_t b, double& sn,
                                                 double& cs) {
    constexpr int B = kScBits;
    const uint32_t sh = static_cast<uint32_t>(b >> 32) + (1u << (31 - B));  // high word of s
    const uint32_t sl = static_cast<uint32_t>(b);
    const uint32_t j = sh >> (32 - B);
    const uint32_t vlo = __funnelshift_r(sl, sh, 11);                          // bits 11..42
    const uint32_t vhi = ((sh >> 11) & ((1u << (21 - B)) - 1u)) | 0x43300000u;  // bits 43..63-B
    const double fi = __hiloint2double(static_cast<int>(vhi), static_cast<int>(vlo)) -
                      (4503599627370496.0 + 4503599627370496.0 / kScN);  // f 2^53 (immediate)
    const double d = fi * FMK(K_TWOPI53, 6.283185307179586 * 0x1.0p-53);
    sincos_rotate(T, static_cast<int>(j), d, sn, cs);
}

}  // namespace fm
}  // namespace sddg
