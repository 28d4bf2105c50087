// walk_kernel.cuh -- K1: persistent first-exit walk kernel.
//
// One walk per lane at a time; a lane whose walk exits writes the walk's
// record and immediately takes the next walk index from a global counter, so
// the heavy-tailed walk lengths (SURVEY.md 7 "Divergence") never idle a lane
// until the batch tail.  Walk g of the batch is walk (walk_lo + g % walks) of
// node perm[g / walks]; the host orders nodes longest-expected-walk first so
// the batch tail is made of short walks.  Records go to HBM by walk index; K2
// (reduce.cu) sums them in the reference's fixed 256-walk chunk order, so
// results do not depend on which lane ran which walk.
//
// Per step (reference: run_walk, proj/src/sde.cpp:151-183; SURVEY.md
// Appendix A): drift -> one Philox block -> Box-Muller -> Euler-Maruyama
// update -> explicit exit (segment_exit, sde.cpp:31-65) -> bridge test
// (edge_crossing_test, sde.cpp:72-121).  The bridge test draws only for
// edges with d0 d1/dt <= 40 (sde.cpp:92); a step whose old and new positions
// both lie in the inner box (every edge distance > sqrt(40 dt)) cannot have
// such an edge, so the exact sorted test runs only near the boundary.
//
// Template parameters: DV drift variant (density.cuh), Real (double/float),
// SCHEME (0 linear, 1 exponential), BRIDGE (linear bridge test on/off).
#pragma once
#include <atomic>
#include <cstdint>

#include "density.cuh"
#include "fastmath.cuh"
#include "philox.cuh"
#include "sddg_internal.h"

// fp64 walks hand their batch tail to the tail kernel; fp32 walks (config 3's
// huge batches, whose tail is a small share) keep the 72-register loop
template <typename Real>
constexpr bool kTailHandoff = sizeof(Real) == 8;

#ifndef SDDG_FP32_LN_V1
#define SDDG_FP32_LN_V1 0  // A/B: round 1's six-term log1p series for d <= 1/16
#endif
#ifndef SDDG_FP32_BOX_V1
#define SDDG_FP32_BOX_V1 0  // A/B: round 1's floating-point box compares in the fp32 walks
#endif
#ifndef SDDG_SHOCK64_HEAVY
#define SDDG_SHOCK64_HEAVY 0
#endif
#ifndef SDDG_BRIDGE_SINGLE
#define SDDG_BRIDGE_SINGLE 1  // 0: round 1's band path of the fp64 performance mode (A/B: -4.5%)
#endif
#ifndef SDDG_BRIDGE_SINGLE_REF
#define SDDG_BRIDGE_SINGLE_REF 1  // the same band path in the reference-mode (parity) kernels (0: A/B, -10%)
#endif
#ifndef SDDG_BRIDGE_SINGLE_F32
#define SDDG_BRIDGE_SINGLE_F32 1  // the same band path in the fp32 shock kernel, whose bridge test is inline (0: A/B, -7%)
#endif
#ifndef SDDG_FP32_BAND_INLINE_ALL
#define SDDG_FP32_BAND_INLINE_ALL 1  // band_exit inline in every fp32 kernel (0: bridge_rare out of line for ring/two-bump, A/B -5%)
#endif
#ifndef SDDG_EXP_MASK_REF
#define SDDG_EXP_MASK_REF 1  // exponential scheme, reference mode: the qualifying-edge mask (sort only for two or more); A/B:
                             // running example +18%, FD shock +21%, FD ring +1%; the register-bound five-ring kernel loses 10% and keeps edge_crossing
#endif
#ifndef SDDG_EXP_MASK_F32
#define SDDG_EXP_MASK_F32 0  // A/B: the same in the fp32 walks (-8% to -19%: kept off)
#endif
#ifndef SDDG_BRIDGE_DIV_BY
#define SDDG_BRIDGE_DIV_BY 0
#endif
#ifndef SDDG_BRIDGE_EXP_BOUND
#define SDDG_BRIDGE_EXP_BOUND 1  // fp64 performance mode: skip the bridge test's exponential when a polynomial bound decides (0: A/B)
#endif
#ifndef SDDG_WALK_UNROLL
#define SDDG_WALK_UNROLL 2  // step-loop copies (A/B: tools/ab.sh with -DSDDG_WALK_UNROLL=n)
#endif
#define SDDG_PRAGMA_STR(x) _Pragma(#x)
#define SDDG_UNROLL(n) SDDG_PRAGMA_STR(unroll n)

namespace sddg {

// Elementary functions per mode: FAST (analytic fp64) uses fastmath.cuh;
// the reference-parity mode uses the CUDA library (closest to glibc).
template <typename Real, bool FAST>
struct RealOps;

template <bool FAST>
struct RealOps<double, FAST> {
    __device__ static __forceinline__ double u(uint64_t u) { return u01_d(u); }
    __device__ static __forceinline__ double u_open(uint64_t u) { return u01_open_d(u); }
    // rng.hpp:66-73: r = sqrt(-2 ln u1), a = 2 pi u2, z = (r cos a, r sin a)
    __device__ static __forceinline__ void box_muller(const fm::FmTables& T, uint64_t a,
                                                      uint64_t b, double& z0, double& z1) {
        const double u1 = u01_open_d(a);
        const double u2 = u01_d(b);
        double s, c;
        const double r = sqrt(-2.0 * log_cuda_cb(u1));
        sincos_cuda_cb(6.283185307179586476925286766559 * u2, &s, &c);
        z0 = r * c;
        z1 = r * s;
    }
    // performance mode: scale * radius and the angle's sin/cos, with u1, u2
    // built from the raw bits (fastmath.cuh); z = (R cs, R sn) / scale
    __device__ static __forceinline__ void bm_polar(const fm::FmTables& T, uint64_t a, uint64_t b,
                                                    double scale, double& R, double& sn,
                                                    double& cs) {
        R = scale * fm::fsqrt_pos(fm::fm2log_tab(T, fm::u01_open_bits(T, a)));
        fm::fsincos_2pi_bits(T, b, sn, cs);
    }
    // the same with the squared scale inside the root: R = sqrt(-2 ln u1 * scale2)
    __device__ static __forceinline__ void bm_polar_sq(const fm::FmTables& T, uint64_t a, uint64_t b,
                                                       double scale2, double& R, double& sn,
                                                       double& cs) {
        R = fm::fsqrt_pos(fm::fm2log_tab(T, fm::u01_open_bits(T, a)) * scale2);
        fm::fsincos_2pi_bits(T, b, sn, cs);
    }
    // -2 ln u_open(a) (rng.hpp:61-63) from the raw bits: Exp(lambda) = that * 1/(2 lambda)
    __device__ static __forceinline__ double m2ln_open(const fm::FmTables& T, uint64_t a) {
        return fm::fm2log_tab(T, fm::u01_open_bits(T, a));
    }
    __device__ static __forceinline__ double ex(const fm::FmTables& T, double v) {
        if constexpr (FAST) return fm::fexp_tab(T, v);
        else return exp_cuda_cb(v);
    }
    __device__ static __forceinline__ double lg(const fm::FmTables& T, double v) {
        if constexpr (FAST) return fm::flog_tab(T, v);
        else return log_cuda_cb(v);
    }
    __device__ static __forceinline__ double sq(double v) { return sqrt(v); }
};

// fp32 walks (config 3): SFU intrinsics.  ln u1 near 1 goes through a short
// log1p series in d = 1 - u1 (exact on the 24-bit grid of u01_open_f), so the
// radius keeps its relative accuracy where MUFU.LG2 is only absolutely accurate.
template <bool FAST>
struct RealOps<float, FAST> {
    __device__ static __forceinline__ float u(uint64_t u) { return u01_f(u); }
    __device__ static __forceinline__ float u_open(uint64_t u) { return u01_open_f(u); }
    // -2 ln u1, u1 = u01_open_f(a) = (k + 1/2) 2^-24.  MUFU.LG2 is absolutely
    // accurate (~2^-22), so near u1 = 1 the radius would lose its relative
    // accuracy: for d = 1 - u1 <= 2^-8 the log1p series -ln(1-d) = d + d^2/2 +
    // d^3/3 (next term < 2e-8 relative) takes over; above, the SFU's error is
    // < 3e-5 of -2 ln u1, i.e. < 6e-9 on sqrt(2 dt) z next to x (ulp 3e-8).
    // d comes from the complement of k (1 - u1 in floating point would round
    // away the low bits of a small u1, down to u1 = 0).
    __device__ static __forceinline__ float m2ln_open(uint64_t a) {
        const uint32_t kc = 0xFFFFFFu ^ static_cast<uint32_t>(a >> 40);
        const float d = __fmaf_rn(static_cast<float>(kc), 0x1.0p-24f, 0x1.0p-25f);  // 1 - u1
        const float u1 = __fmaf_rn(static_cast<float>(static_cast<uint32_t>(a >> 40)), 0x1.0p-24f, 0x1.0p-25f);
#if SDDG_FP32_LN_V1
        // round-1 form: six-term series for d <= 1/16
        float p = __fmaf_rn(d, 0.16666667f, 0.2f);
        p = __fmaf_rn(p, d, 0.25f);
        p = __fmaf_rn(p, d, 0.33333334f);
        p = __fmaf_rn(p, d, 0.5f);
        p = __fmaf_rn(p, d, 1.0f);
        const float series = -(p * d);
        return -2.0f * (d <= 0.0625f ? series : __logf(u1));
#else
        float p = __fmaf_rn(d, 0.66666669f, 1.0f);
        p = __fmaf_rn(p, d, 2.0f);
        return d <= 0x1.0p-8f ? p * d : __log2f(u1) * -1.3862944f;
#endif
    }
    __device__ static __forceinline__ void bm_polar(const fm::FmTables&, uint64_t a, uint64_t b,
                                                    float scale, float& R, float& sn, float& cs) {
        const float v = m2ln_open(a);
#if SDDG_FP32_LN_V1
        R = scale * (v * rsqrtf(v));
#else
        R = scale * sqrt_approx(v);  // one MUFU.SQRT (v >= 2^-24 > 0)
#endif
        // 2 pi u2 with u2 = top 24 bits 2^-24 (u01_f), one multiply
        __sincosf(static_cast<float>(static_cast<uint32_t>(b >> 40)) * (6.2831853f * 0x1.0p-24f),
                  &sn, &cs);
    }
    __device__ static __forceinline__ float ex(const fm::FmTables&, float v) { return __expf(v); }
    __device__ static __forceinline__ float lg(const fm::FmTables&, float v) { return __logf(v); }
    __device__ static __forceinline__ float sq(float v) { return sqrtf(v); }
};

template <int DV, typename Real>
__device__ __forceinline__ bool drift(const DensityParams& P, const fm::FmTables& T, Real x, Real y,
                                      Real& bx, Real& by) {
    if constexpr (DV >= DV_RING_AN) {
        return drift_an<DV>(T, P, x, y, bx, by);
    } else {
        static_assert(sizeof(Real) == 8, "reference drifts are fp64 only");
        return drift_ref<DV>(P, x, y, bx, by);
    }
}

template <typename Real>
__device__ __forceinline__ Real clampr(Real v, Real lo, Real hi) {
    return v < lo ? lo : (hi < v ? hi : v);  // std::clamp
}

template <typename Real>
struct Dom {
    Real xmin, xmax, ymin, ymax;
    Real bx0, bx1, by0, by1;  // inner box: every edge distance > sqrt(40 dt)
    int hx0, hx1, hy0, hy1;   // high words of the box edges (integer test)
    __device__ __forceinline__ bool inside(Real x, Real y) const {
        return x > xmin && x < xmax && y > ymin && y < ymax;  // geometry.hpp:38-40
    }
    __device__ __forceinline__ bool in_box(Real x, Real y) const {
        return x > bx0 && x < bx1 && y > by0 && y < by1;
    }
    // Conservative box test on the high words (fp64 performance mode): four
    // integer compares instead of four FP64-pipe DSETPs.  A strictly larger
    // high word of a positive double means a strictly larger value, and a
    // negative x has a negative high word, so a true result implies in_box.
    __device__ __forceinline__ bool in_box_hi(double x, double y) const {
        const int xi = __double2hiint(x), yi = __double2hiint(y);
        return xi > hx0 && xi < hx1 && yi > hy0 && yi < hy1;
    }
    // fp32 walks: the whole bit pattern, so the test is in_box exactly (a
    // negative x has a negative pattern and fails x > bx0 > 0 either way)
    __device__ __forceinline__ bool in_box_hi(float x, float y) const {
        const int xi = __float_as_int(x), yi = __float_as_int(y);
        return xi > hx0 && xi < hx1 && yi > hy0 && yi < hy1;
    }
    // geometry.cpp:24-32
    __device__ __forceinline__ Real dist(Real x, Real y, int e) const {
        return e == 0 ? y - ymin : (e == 1 ? ymax - y : (e == 2 ? x - xmin : xmax - x));
    }
    __device__ __forceinline__ void project(int e, Real& hx, Real& hy) const {
        if (e == 0) hy = ymin;
        else if (e == 1) hy = ymax;
        else if (e == 2) hx = xmin;
        else hx = xmax;
        hx = clampr(hx, xmin, xmax);
        hy = clampr(hy, ymin, ymax);
    }
};

// Walk parameters in the walk's precision: fp32 walks take the host-rounded
// float copies (constant-bank operands, no conversion in the step loop)
template <typename Real>
__device__ __forceinline__ Real walk_prm(double d, float f) {
    if constexpr (sizeof(Real) == 4) return f;
    else return d;
}
template <typename Real>
__device__ __forceinline__ Dom<Real> walk_dom(const WalkArgs& a) {
    return Dom<Real>{walk_prm<Real>(a.xmin, a.f_dom[0]), walk_prm<Real>(a.xmax, a.f_dom[1]),
                     walk_prm<Real>(a.ymin, a.f_dom[2]), walk_prm<Real>(a.ymax, a.f_dom[3]),
                     walk_prm<Real>(a.box[0], a.f_dom[4]), walk_prm<Real>(a.box[1], a.f_dom[5]),
                     walk_prm<Real>(a.box[2], a.f_dom[6]), walk_prm<Real>(a.box[3], a.f_dom[7]),
                     sizeof(Real) == 4 ? a.box_fi[0] : a.box_hi[0], sizeof(Real) == 4 ? a.box_fi[1] : a.box_hi[1],
                     sizeof(Real) == 4 ? a.box_fi[2] : a.box_hi[2], sizeof(Real) == 4 ? a.box_fi[3] : a.box_hi[3]};
}

// segment_exit (proj/src/sde.cpp:31-65)
template <typename Real>
__device__ __forceinline__ void segment_exit(const Dom<Real>& d, Real x0, Real y0, Real x1,
                                             Real y1, Real& hx, Real& hy, int& edge) {
    Real best_t = Real(2);
    int best = 0;
    auto consider = [&](int e, Real c0, Real c1, Real target) {
        if (c1 == c0) return;
        const Real t = (target - c0) / (c1 - c0);
        if (t >= Real(0) && t <= Real(1) && t < best_t) {
            best_t = t;
            best = e;
        }
    };
    if (y1 <= d.ymin) consider(0, y0, y1, d.ymin);
    if (y1 >= d.ymax) consider(1, y0, y1, d.ymax);
    if (x1 <= d.xmin) consider(2, x0, x1, d.xmin);
    if (x1 >= d.xmax) consider(3, x0, x1, d.xmax);
    if (best_t > Real(1)) {
        best_t = Real(1);
        if (y1 <= d.ymin) best = 0;
        else if (y1 >= d.ymax) best = 1;
        else if (x1 <= d.xmin) best = 2;
        else best = 3;
    }
    hx = x0 + best_t * (x1 - x0);
    hy = y0 + best_t * (y1 - y0);
    d.project(best, hx, hy);
    edge = best;
}

// edge_crossing_test (proj/src/sde.cpp:72-109): edges sorted by
// (min(d0,d1), id); exponent > 40 skips without a draw; else fire if
// u01 < exp(-ex).  SCHEME 0: ex = d0 d1 / dt (bridge_exit_test); 1: nu2 min(d0,d1).
template <typename Real, bool FAST, int SCHEME, typename Stream>
__device__ __forceinline__ bool edge_crossing(const Dom<Real>& d, Real x0, Real y0, Real x1,
                                              Real y1, Real par, const RoundKeys& rk,
                                              const fm::FmTables& T, Stream& rng, Real& hx,
                                              Real& hy, int& edge) {
    const Real k0 = d.dist(x0, y0, 0), k1 = d.dist(x0, y0, 1), k2 = d.dist(x0, y0, 2),
               k3 = d.dist(x0, y0, 3);
    const Real m0 = d.dist(x1, y1, 0), m1 = d.dist(x1, y1, 1), m2 = d.dist(x1, y1, 2),
               m3 = d.dist(x1, y1, 3);
    // std::min(a, b) = b < a ? b : a
    Real s0 = m0 < k0 ? m0 : k0, s1 = m1 < k1 ? m1 : k1, s2 = m2 < k2 ? m2 : k2,
         s3 = m3 < k3 ? m3 : k3;
    int e0 = 0, e1 = 1, e2 = 2, e3 = 3;
    auto cswap = [](Real& da, int& ea, Real& db, int& eb) {
        const bool less = db != da ? db < da : eb < ea;
        if (less) {
            const Real t = da; da = db; db = t;
            const int u = ea; ea = eb; eb = u;
        }
    };
    cswap(s0, e0, s1, e1);
    cswap(s2, e2, s3, e3);
    cswap(s0, e0, s2, e2);
    cswap(s1, e1, s3, e3);
    cswap(s1, e1, s2, e2);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int e = i == 0 ? e0 : (i == 1 ? e1 : (i == 2 ? e2 : e3));
        const Real d0 = e == 0 ? k0 : (e == 1 ? k1 : (e == 2 ? k2 : k3));
        const Real d1 = e == 0 ? m0 : (e == 1 ? m1 : (e == 2 ? m2 : m3));
        const Real ex = SCHEME == 0 ? d0 * d1 / par : par * (d1 < d0 ? d1 : d0);
        if (ex > Real(40)) continue;
        const Real u = RealOps<Real, FAST>::u(rng.next_one(rk));
#if SDDG_BRIDGE_EXP_BOUND
        // exp(-ex) <= 1 / (1 + ex + ex^2/2): a draw above that bound cannot
        // fire, and most do not come near it -- the exponential is evaluated
        // only for the few that do (same decisions: the margin covers the
        // rounding of the bound by many orders)
        if constexpr (FAST && sizeof(Real) == 8) {
            if (u * fma(ex, fma(ex, Real(0.5), Real(1)), Real(1)) >= Real(1.000001)) continue;
        }
#endif
        if (u < RealOps<Real, FAST>::ex(T, -ex)) {
            const Real sum = d0 + d1;
            const Real s = sum > Real(0) ? d0 / sum : Real(0);
            hx = x0 + s * (x1 - x0);
            hy = y0 + s * (y1 - y0);
            d.project(e, hx, hy);
            edge = e;
            return true;
        }
    }
    return false;
}

// Performance-mode bridge test (SCHEME 0, fp32 walks).  pe = d0 d1 of edge
// e, exactly the products the reference forms (sde.cpp:83-92).  Only edges
// with ex = pe / dt <= 40 draw (here pe * (1/dt)), and the sort order matters
// only among those: with one such edge (all but corner steps) the sort is
// skipped.  Skipped edges draw nothing, so the stream is consumed exactly as
// in edge_crossing.
#ifndef SDDG_FP32_BRIDGE_OOL_SHOCK
#define SDDG_FP32_BRIDGE_OOL_SHOCK 0  // A/B: out of line the shock kernel needs 96 registers (-3.5%)
#endif

template <typename Real>
__device__ __forceinline__ uint32_t sorted_edge_order(const Dom<Real>& d, Real x0, Real y0,
                                                      Real x1, Real y1) {
    Real s[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const Real k = d.dist(x0, y0, e), m = d.dist(x1, y1, e);
        s[e] = m < k ? m : k;  // std::min
    }
    // rank of edge e in the (min(d0,d1), id) order
    uint32_t order = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        int r = 0;
#pragma unroll
        for (int f = 0; f < 4; ++f)
            if (f != e) r += (s[f] < s[e] || (s[f] == s[e] && f < e)) ? 1 : 0;
        order |= static_cast<uint32_t>(e) << (4 * r);
    }
    return order;
}

// The rare path as a real subroutine: ptxas allocates the step loop's
// registers without it (inlined, its temporaries cost the step loop
// constant-bank operand forms or spills).  State in and out by value.
struct BridgeRes {
    double hx, hy;
    uint32_t n, cw2, cw3;
    int edge;  // -1: no exit
};

template <typename Real>
__device__ __noinline__ BridgeRes bridge_rare(Real x0, Real y0, Real x1, Real y1, int mask,
                                              LaneStream rng, const WalkArgs* a,
                                              const fm::FmTables* T) {
    const Dom<Real> d{Real(a->xmin), Real(a->xmax), Real(a->ymin), Real(a->ymax)};
    const Real idt = Real(a->inv_dt);
    uint32_t order = 0x3210u;
    if (mask & (mask - 1)) order = sorted_edge_order(d, x0, y0, x1, y1);
    BridgeRes r;
    r.edge = -1;
#pragma unroll 1
    for (int i = 0; i < 4; ++i, order >>= 4) {
        const int e = static_cast<int>(order & 15u);
        if (!((mask >> e) & 1)) continue;
        const Real d0 = d.dist(x0, y0, e), d1 = d.dist(x1, y1, e);
        const Real ex = d0 * d1 * idt;
        const Real u = RealOps<Real, true>::u(rng.next_one(a->rk));
        if (u < RealOps<Real, true>::ex(*T, -ex)) {
            const Real sum = d0 + d1;
            const Real sc = sum > Real(0) ? d0 / sum : Real(0);
            Real hx = x0 + sc * (x1 - x0), hy = y0 + sc * (y1 - y0);
            d.project(e, hx, hy);
            r.hx = hx;
            r.hy = hy;
            r.edge = e;
            break;
        }
    }
    r.n = rng.n;
    r.cw2 = rng.cw2;
    r.cw3 = rng.cw3;
    return r;
}

// Performance-mode exit test of the exponential scheme (edge_crossing_test
// with exponent nu2 min(d0, d1), sde.cpp:72-109,131-140).  With large
// exponential steps most edges qualify (ex <= 40 within 40/nu2 of an edge),
// so this runs on nearly every step: the qualifying set is a bitmask, the
// edge sort runs only when two or more edges qualify, and the draws share one
// rolled loop.  Skipped edges draw nothing, as in edge_crossing.
template <typename Real, bool FAST, typename Stream>
__device__ __forceinline__ bool bridge_exp_fast(const Dom<Real>& d, Real x0, Real y0, Real x1, Real y1,
                                                Real nu2, const RoundKeys& rk, const fm::FmTables& T,
                                                Stream& rng, Real& hx, Real& hy, int& edge) {
    int mask = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        const Real k = d.dist(x0, y0, e), m = d.dist(x1, y1, e);
        mask |= int(!(nu2 * (m < k ? m : k) > Real(40))) << e;
    }
    if (mask == 0) return false;
    uint32_t order = 0x3210u;
    if (mask & (mask - 1)) order = sorted_edge_order(d, x0, y0, x1, y1);
#pragma unroll 1
    for (int i = 0; i < 4; ++i, order >>= 4) {
        const int e = static_cast<int>(order & 15u);
        if (!((mask >> e) & 1)) continue;
        const Real d0 = d.dist(x0, y0, e), d1 = d.dist(x1, y1, e);
        const Real ex = nu2 * (d1 < d0 ? d1 : d0);
        const Real u = RealOps<Real, FAST>::u(rng.next_one(rk));
        if (u < RealOps<Real, FAST>::ex(T, -ex)) {
            const Real sum = d0 + d1;
            const Real sc = sum > Real(0) ? d0 / sum : Real(0);
            hx = x0 + sc * (x1 - x0);
            hy = y0 + sc * (y1 - y0);
            d.project(e, hx, hy);
            edge = e;
            return true;
        }
    }
    return false;
}

// table_at / f_at / g_at (proj/src/boundary.cpp:10-42)
__device__ __forceinline__ double table_at(const double* __restrict__ t, int n, double s) {
    int k = static_cast<int>(floor(s));
    k = k < 0 ? 0 : (k > n - 2 ? n - 2 : k);
    double u = s - k;
    u = u < 0.0 ? 0.0 : (1.0 < u ? 1.0 : u);
    return (1.0 - u) * __ldg(t + k) + u * __ldg(t + k + 1);
}

// ---------------------------------------------------------------- one step
// The arithmetic of one step, shared by the walk kernel K1 and the tail
// kernel (walk_tail.cuh), so that both compute every step bit for bit alike.

// u64 draws of a step's own randoms (the exit test may draw more)
template <int SCHEME>
constexpr uint32_t kStepDraws = SCHEME == 0 ? 2u : 3u;

// Random-derived values of one step: a pure function of the stream words it
// consumes (SCHEME 0: the normal pair's two u64s; SCHEME 1: the Exp(lambda)
// step's u64, then the pair's two).  FAST: (R, sn, cs) of the polar form;
// reference: (z0, z1) and, for SCHEME 1, s = sqrt(2 edt).
template <typename Real>
struct StepRand {
    Real edt, r0, r1, r2;
};

template <int DV, typename Real, int SCHEME>
__device__ __forceinline__ StepRand<Real> step_rand(const fm::FmTables& T, const WalkArgs& a, Real sq2dt,
                                                    uint64_t w0, uint64_t w1, uint64_t w2) {
    constexpr bool FAST = DV >= DV_RING_AN;
    using Ops = RealOps<Real, FAST>;
    StepRand<Real> r;
    r.edt = Real(0);
    r.r2 = Real(0);
    if constexpr (SCHEME == 0 && FAST) {
        // sqrt(2 dt) z = R (cs, sn)
        Ops::bm_polar(T, w0, w1, sq2dt, r.r0, r.r1, r.r2);
    } else if constexpr (SCHEME == 0) {
        Ops::box_muller(T, w0, w1, r.r0, r.r1);
    } else if constexpr (FAST && sizeof(Real) == 8) {
        // step_exponential (sde.cpp:123-140), fp64 performance mode: edt =
        // -ln u / lambda from the raw bits, one root for the radius
        // sqrt(-2 ln u1) * sqrt(2 edt) = sqrt(-2 ln u1 * 2 edt)
        r.edt = Ops::m2ln_open(T, w0) * Real(a.half_inv_lambda);
        Ops::bm_polar_sq(T, w1, w2, Real(2) * r.edt, r.r0, r.r1, r.r2);
    } else {
        // step_exponential (sde.cpp:123-140): dt ~ Exp(lambda) first
        r.edt = -Ops::lg(T, Ops::u_open(w0)) / Real(a.lambda);
        const Real sv = Ops::sq(Real(2) * r.edt);
        if constexpr (FAST) {  // fp32 (A/B: the fp64 form above is 10-18% slower here)
            Ops::bm_polar(T, w1, w2, sv, r.r0, r.r1, r.r2);
        } else {
            Ops::box_muller(T, w1, w2, r.r0, r.r1);
            r.r2 = sv;
        }
    }
    return r;
}

// The drift of one step at (x, y): linear performance mode the scaled form
// dt grad(w)/w = c (vx, vy) (drift_cv), otherwise (bx, by) = grad(w)/w;
// ok false where the reference throws EvaluationError (non-finite drift).
template <typename Real>
struct StepDrift {
    Real c, vx, vy;  // bx, by in vx, vy for the unscaled forms
    Real s, w;       // literal SDE: noise scale sqrt(w) and w (the bridge's time scale); else 1
    bool ok;
};

template <int DV, typename Real, int SCHEME>
__device__ __forceinline__ StepDrift<Real> step_drift(const fm::FmTables& T, const DensityParams& P, Real dt,
                                                      Real x, Real y) {
    StepDrift<Real> d;
    d.s = Real(1);
    d.w = Real(1);
    if constexpr (kLiteral<DV>) {
        // BASELINE's literal SDE (linear scheme only, validated on the host)
        drift_lit(DV, T, x, y, dt, d.c, d.vx, d.vy, d.w);
        if constexpr (sizeof(Real) == 8) d.s = fm::fsqrt_pos(d.w);
        else d.s = sqrtf(d.w);
        d.ok = true;
    } else if constexpr (SCHEME == 0 && DV >= DV_RING_AN) {
        if constexpr (sizeof(Real) == 4 && (DV == DV_RING_AN || DV == DV_SHOCK_AN || DV == DV_TWOBUMP_AN))
            drift_cv<DV, true>(T, P, x, y, dt, d.c, d.vx, d.vy);
        else
            drift_cv<DV>(T, P, x, y, dt, d.c, d.vx, d.vy);
        d.ok = true;  // closed forms: finite everywhere
    } else {
        d.c = Real(0);
        d.ok = drift<DV, Real>(P, T, x, y, d.vx, d.vy);
    }
    return d;
}

// Euler-Maruyama update (step_linear, sde.cpp:21-29; step_exponential,
// :123-140) from the step's drift and randoms.
template <int DV, typename Real, int SCHEME>
__device__ __forceinline__ void step_update(const StepDrift<Real>& d, const StepRand<Real>& r, Real dt,
                                            Real sq2dt, Real x, Real y, Real& nxp, Real& nyp) {
    constexpr bool FAST = DV >= DV_RING_AN;
    if constexpr (SCHEME == 0 && kLiteral<DV>) {
        // x + grad(w) dt + sqrt(2 w dt) z = x + c v + sqrt(w) R (cs, sn)
        const Real Rs = r.r0 * d.s;
        nxp = fma(Rs, r.r2, fma(d.c, d.vx, x));
        nyp = fma(Rs, r.r1, fma(d.c, d.vy, y));
    } else if constexpr (SCHEME == 0 && FAST) {
        // x + b dt + sqrt(2 dt) z with b dt = c v and sqrt(2 dt) z = R (cs, sn)
        nxp = fma(r.r0, r.r2, fma(d.c, d.vx, x));
        nyp = fma(r.r0, r.r1, fma(d.c, d.vy, y));
    } else if constexpr (SCHEME == 0) {
        nxp = x + d.vx * dt + sq2dt * r.r0;
        nyp = y + d.vy * dt + sq2dt * r.r1;
    } else if constexpr (FAST && sizeof(Real) == 8) {
        nxp = fma(r.r0, r.r2, fma(d.vx, r.edt, x));
        nyp = fma(r.r0, r.r1, fma(d.vy, r.edt, y));
    } else if constexpr (FAST) {
        nxp = x + d.vx * r.edt + r.r0 * r.r2;
        nyp = y + d.vy * r.edt + r.r0 * r.r1;
    } else {
        nxp = x + d.vx * r.edt + r.r2 * r.r0;
        nyp = y + d.vy * r.edt + r.r2 * r.r1;
    }
}

// The inner-box test of the step loop: the integer high-word form in the
// fp64 table kernels (performance mode), the exact one otherwise.
template <int DV, typename Real>
__device__ __forceinline__ bool box_test(const Dom<Real>& d, Real px, Real py) {
    if constexpr (DV >= DV_RING_AN && (sizeof(Real) == 8 || !SDDG_FP32_BOX_V1)) return d.in_box_hi(px, py);
    else return d.in_box(px, py);
}

// The band path (a step with an end outside the inner box) of the fp64 walks
// and of the fp32 kernels with an inline bridge test, same decisions as
// segment_exit + edge_crossing:
//  * the four products p_e = d0 d1 decide everything first: an end outside
//    the domain makes one of them <= 0 (the start is strictly inside), an
//    edge can draw only if p_e <= 40 dt;
//  * all but corner steps have ONE edge that can draw.  Its exponent is p_e /
//    dt -- the quotient edge_crossing forms from the same two distances -- and
//    with one candidate the edge order cannot matter: no sort, one division
//    instead of four;
//  * exp(-ex) <= 1 / (1 + ex + ex^2/2): most draws lie above that bound and
//    cannot fire; the exponential decides the few that do not (the margin
//    covers the bound's rounding by many orders).
// Reference mode (FAST false) takes the same shortcuts where they cannot
// change a decision: one candidate edge needs no sort, and the bound only
// skips exponentials whose comparison is already decided; it keeps the
// reference's own inside test.
template <typename Real, bool FAST, typename Stream>
__device__ __forceinline__ bool band_exit(const Dom<Real>& dom, const WalkArgs& a, const fm::FmTables& T, Real thr,
                                          Real dt, Real x, Real y, Real nxp, Real nyp, Stream& rng, Real& hx,
                                          Real& hy, int& edge) {
    if constexpr (!FAST) {
        if (!dom.inside(nxp, nyp)) {
            segment_exit(dom, x, y, nxp, nyp, hx, hy, edge);
            return true;
        }
    }
    const Real pB = (y - dom.ymin) * (nyp - dom.ymin);
    const Real pT = (dom.ymax - y) * (dom.ymax - nyp);
    const Real pL = (x - dom.xmin) * (nxp - dom.xmin);
    const Real pR = (dom.xmax - x) * (dom.xmax - nxp);
    const bool qB = pB <= thr, qT = pT <= thr, qL = pL <= thr, qR = pR <= thr;
    if (!(qB || qT || qL || qR)) return false;
    if constexpr (FAST) {
        if (!(pB > Real(0) && pT > Real(0) && pL > Real(0) && pR > Real(0))) {  // !inside(nxp, nyp)
            segment_exit(dom, x, y, nxp, nyp, hx, hy, edge);
            return true;
        }
    }
    if (int(qB) + int(qT) + int(qL) + int(qR) != 1)
        return edge_crossing<Real, FAST, 0>(dom, x, y, nxp, nyp, dt, a.rk, T, rng, hx, hy, edge);
    const int e = qB ? 0 : (qT ? 1 : (qL ? 2 : 3));
    const Real pe = qB ? pB : (qT ? pT : (qL ? pL : pR));
#if SDDG_BRIDGE_DIV_BY  // A/B (-0.5%): the same correctly rounded quotient from the host's RN(1/dt)
    Real ex;
    if constexpr (sizeof(Real) == 8) ex = pe > 0x1p-500 ? div_rn_by(pe, dt, a.inv_dt) : pe / dt;
    else ex = pe / dt;
#else
    const Real ex = pe / dt;
#endif
    if (ex > Real(40)) return false;
    const Real u = RealOps<Real, FAST>::u(rng.next_one(a.rk));
    // the margin covers the rounding of the bound and of the exponential it stands in for
    if (u * fma(ex, fma(ex, Real(0.5), Real(1)), Real(1)) >= (sizeof(Real) == 8 ? Real(1.000001) : Real(1.0001)))
        return false;
    if (!(u < RealOps<Real, FAST>::ex(T, -ex))) return false;
    const Real d0 = dom.dist(x, y, e), d1 = dom.dist(nxp, nyp, e);
    const Real sum = d0 + d1;
    const Real sc = sum > Real(0) ? d0 / sum : Real(0);
    hx = x + sc * (nxp - x);
    hy = y + sc * (nyp - y);
    dom.project(e, hx, hy);
    edge = e;
    return true;
}

// Exit test of the step (x, y) -> (nxp, nyp): explicit exit (segment_exit,
// sde.cpp:31-65) or the scheme's edge-crossing draws (sde.cpp:72-121), from
// the stream `rng` (the lane's own Philox stream in K1, the warp's window in
// the tail kernel).  nb: whether (nxp, nyp) lies in the inner box.
template <int DV, typename Real, int SCHEME, bool BRIDGE, typename Stream>
__device__ __forceinline__ bool exit_test(const Dom<Real>& dom, const WalkArgs& a, const fm::FmTables& T,
                                          Real thr, Real dt, Real x, Real y, Real nxp, Real nyp,
                                          bool in_box, Stream& rng, Real& hx, Real& hy, int& edge,
                                          bool& nb) {
    constexpr bool FAST = DV >= DV_RING_AN;
    bool exited = false;
    nb = true;
    if constexpr (SCHEME == 0 && BRIDGE) {
        // inner box first: box inside the domain, so both ends in the
        // box means no exit and no bridge draw (the common step)
        nb = box_test<DV, Real>(dom, nxp, nyp);
        if (!(nb && in_box)) {
            // fp32: the kernels whose bridge test is inline (the shock drift; the
            // others call bridge_rare out of line, below)
            constexpr bool kInline32 = sizeof(Real) == 4 && FAST && SDDG_BRIDGE_SINGLE_F32 &&
                                       (SDDG_FP32_BAND_INLINE_ALL || !(SDDG_FP32_BRIDGE_OOL_SHOCK || DV != DV_SHOCK_AN));
            // (the literal SDE passes its own threshold and time scale, w dt: same path)
            if constexpr (SDDG_BRIDGE_SINGLE &&
                          ((sizeof(Real) == 8 && (FAST || SDDG_BRIDGE_SINGLE_REF)) || kInline32)) {
                exited = band_exit<Real, FAST>(dom, a, T, thr, dt, x, y, nxp, nyp, rng, hx, hy, edge);
            } else if (!dom.inside(nxp, nyp)) {
                segment_exit(dom, x, y, nxp, nyp, hx, hy, edge);
                exited = true;
            } else {
                // exact pre-filter: an edge draws only if d0*d1 <= 40 dt
                const Real pB = (y - dom.ymin) * (nyp - dom.ymin);
                const Real pT = (dom.ymax - y) * (dom.ymax - nyp);
                const Real pL = (x - dom.xmin) * (nxp - dom.xmin);
                const Real pR = (dom.xmax - x) * (dom.xmax - nxp);
                if constexpr (FAST && sizeof(Real) == 4 && !kLiteral<DV> &&
                              (SDDG_FP32_BRIDGE_OOL_SHOCK || DV != DV_SHOCK_AN)) {
                    // fp32: out of line (A/B +2.4%); fp64 keeps the inline test below
                    // (out of line it costs the step loop a local-memory round trip: -0.5%)
                    static_assert(sizeof(Stream) == sizeof(LaneStream), "fp32 runs in K1 only");
                    const Real idt = Real(a.inv_dt);
                    const int mask = int(!(pB * idt > Real(40))) | (int(!(pT * idt > Real(40))) << 1) |
                                     (int(!(pL * idt > Real(40))) << 2) | (int(!(pR * idt > Real(40))) << 3);
                    if (mask) {
                        const BridgeRes r = bridge_rare<Real>(x, y, nxp, nyp, mask, rng, &a, &T);
                        rng.n = r.n;
                        rng.cw2 = r.cw2;
                        rng.cw3 = r.cw3;
                        if (r.edge >= 0) {
                            hx = Real(r.hx);
                            hy = Real(r.hy);
                            edge = r.edge;
                            exited = true;
                        }
                    }
                } else if (pB <= thr || pT <= thr || pL <= thr || pR <= thr) {
                    exited = edge_crossing<Real, FAST, 0>(dom, x, y, nxp, nyp, dt, a.rk, T, rng, hx, hy, edge);
                }
            }
        }
    } else if (!dom.inside(nxp, nyp)) {
        segment_exit(dom, x, y, nxp, nyp, hx, hy, edge);
        exited = true;
    } else if constexpr (SCHEME == 1 && ((sizeof(Real) == 8 && (FAST || (SDDG_EXP_MASK_REF && DV != DV_FIVE_RING))) ||
                                         (sizeof(Real) == 4 && FAST && SDDG_EXP_MASK_F32))) {
        // (reference mode too: the same edges draw in the same order, so every decision is the same)
        exited = bridge_exp_fast<Real, FAST, Stream>(dom, x, y, nxp, nyp, Real(a.nu2), a.rk, T, rng, hx, hy, edge);
    } else if constexpr (SCHEME == 1) {
        exited = edge_crossing<Real, FAST, 1>(dom, x, y, nxp, nyp, Real(a.nu2), a.rk, T, rng, hx, hy, edge);
    }
    return exited;
}

// A walk's exit (run_walk, sde.cpp:170-177): boundary values at the exit
// point (table_at, boundary.cpp:10-42), the walk record (or per-path dump)
// at slot g, and its path-steps over all epochs into the node's counter.
template <typename Real>
__device__ __forceinline__ void record_exit(const WalkArgs& a, uint64_t g, uint32_t node, uint32_t epoch,
                                            uint32_t step, int edge, Real hx, Real hy, uint32_t max_steps) {
    const double dhx = static_cast<double>(hx), dhy = static_cast<double>(hy);
    const bool horiz = edge < 2;
    const double par = horiz ? (dhx - a.txmin) / a.thx : (dhy - a.tymin) / a.thy;
    const int tn = horiz ? a.tnx : a.tny;
    const double fv = table_at(a.tf[edge], tn, par);
    const double gv = table_at(a.tg[edge], tn, par);
    SDDG_CHECK(g < a.total && node < static_cast<uint64_t>(a.n_nodes) && edge >= 0 && edge < 4);
    // restarts happen at exactly max_steps: one atomic per finished walk
    if (a.node_steps)
        atomicAdd(a.node_steps + node, static_cast<unsigned long long>(epoch) * max_steps + step);
    if (a.dump) {
        sddg_path& r = a.dump[g];
        r.f = fv;
        r.g = gv;
        r.ex = dhx;
        r.ey = dhy;
        r.steps = step;
        r.epoch = static_cast<int32_t>(epoch);
        r.edge = edge;
    } else {
        a.rec_f[g] = fv;
        a.rec_g[g] = gv;
        a.rec_meta[g] = static_cast<uint32_t>(edge) | (epoch << 2);
    }
}

// Launch shape per variant.  Performance-mode fp64 reads the fastmath tables
// from shared memory; with the large tables (64 KB) one CTA fills an SM:
// 1024 threads at 64 registers, or 640 at 96 for the register-hungrier
// shock drift.  Everything else: 128-thread CTAs, several per SM.
template <int DV, typename Real>
__host__ __device__ constexpr bool walk_uses_tables() {
    return DV >= DV_RING_AN && sizeof(Real) == 8;
}
constexpr bool kBigTables = sizeof(fm::FmTables) > 24 * 1024;
// drifts that need more than 64 registers in the fp64 table kernel
template <int DV>
__host__ __device__ constexpr bool walk_heavy_drift() {
#if SDDG_SHOCK64_HEAVY  // A/B: round 1's 640-thread, 96-register shape for the shock and five-ring drifts
    return DV == DV_SHOCK_AN || DV == DV_FIVE_RING_AN || DV == DV_TABLE_AN;
#else
    // The one-reciprocal shock drift and the five-ring fit the 1024-thread,
    // 64-register shape without spills (shock +4%; five-ring +4.6% with the
    // exponential scheme, the paper's workload, -1% with the linear one); the
    // table interpolant's exponential-scheme kernel would spill.
    return DV == DV_TABLE_AN;
#endif
}
template <int DV, typename Real>
__host__ __device__ constexpr int walk_block() {
#ifdef SDDG_WALK_TABLE_BLOCK
    if constexpr (walk_uses_tables<DV, Real>() && kBigTables && !walk_heavy_drift<DV>())
        return SDDG_WALK_TABLE_BLOCK;
#endif
    if constexpr (walk_uses_tables<DV, Real>() && kBigTables) return walk_heavy_drift<DV>() ? 640 : 1024;
    return kWalkBlock;
}
template <int DV, typename Real>
__host__ __device__ constexpr int walk_min_blocks() {
#ifdef SDDG_WALK_TABLE_BLOCKS_PER_SM
    if constexpr (walk_uses_tables<DV, Real>() && kBigTables && !walk_heavy_drift<DV>())
        return SDDG_WALK_TABLE_BLOCKS_PER_SM;
#endif
    if constexpr (walk_uses_tables<DV, Real>() && kBigTables) return 1;
#ifndef SDDG_SHOCK32_MIN_BLOCKS
#define SDDG_SHOCK32_MIN_BLOCKS 7  // 7 x 128 threads per SM: ptxas keeps the shock fp32 loop <= 72 registers
#endif
    if constexpr (DV == DV_SHOCK_AN && sizeof(Real) == 4) return SDDG_SHOCK32_MIN_BLOCKS;
#ifndef SDDG_REF_MIN_BLOCKS
// reference-mode (parity) kernels: 128-thread CTAs per SM.  A/B (tools/ab_walk.sh, profiles/r02_ref_blocks_ab.log):
// 3/4/5/6/7/8/10 CTAs -> FD ring 2.43/2.55/2.68/2.70/2.74/2.77/2.75e10 at 2,000 paths (8: +8% at 1e4 paths);
// the 64-register cap spills 40-130 B, and the warps to hide the FP64 chains are worth more
#define SDDG_REF_MIN_BLOCKS 8
#endif
    if constexpr (DV < DV_RING_AN) return SDDG_REF_MIN_BLOCKS;
    return walk_heavy_drift<DV>() ? 5 : kWalkMinBlocks;
}

template <int DV, typename Real>
__host__ __device__ constexpr size_t walk_table_bytes() {
    return walk_uses_tables<DV, Real>() ? sizeof(fm::FmTables) : 0;
}
static_assert(sizeof(fm::FmTables) % 16 == 0, "LaneState alignment after the tables");

// TAIL: the batch hands its last walks to the tail kernel (walk_tail.cuh):
// the step loop counts chunks of a.chunk32 steps with check points between
// them.  Without TAIL the loop is the plain one (1.5 instructions per step
// fewer: the large batches, where the tail is a negligible share).
// DRAIN: a drain round (a.src set): the same loop on a few walks per SM, where
// a step's latency, not issue, bounds it -- so compiled for kDrainBlock-thread
// CTAs, with the registers to overlap the step's random-number and drift chains.
template <int DV, typename Real, int SCHEME, bool BRIDGE, bool TAIL = false, bool DRAIN = false>
__global__ void __launch_bounds__(DRAIN ? kDrainBlock : walk_block<DV, Real>(), DRAIN ? 1 : walk_min_blocks<DV, Real>())
    walk_kernel(const __grid_constant__ WalkArgs a) {
    static_assert(!TAIL || kTailHandoff<Real>, "tail handoff is fp64 only");
    static_assert(!DRAIN || TAIL, "drain rounds hand over to the tail kernel");
    constexpr bool FAST = DV >= DV_RING_AN;
    using Ops = RealOps<Real, FAST>;
    const Dom<Real> dom = walk_dom<Real>(a);
    const DensityParams P{a.R, a.alpha, a.fd_h, 1.0 / (2.0 * a.fd_h), a.tab, a.f_kd};
    const Real dt = walk_prm<Real>(a.dt, a.f_dt);
    const Real sq2dt = walk_prm<Real>(a.sqrt2dt, a.f_sqrt2dt);
    const Real thr = walk_prm<Real>(a.bridge_thr, a.f_thr);
    const uint32_t max_steps = a.max_steps32;
    // Dynamic shared memory: the fastmath tables (performance-mode fp64) then
    // the per-lane bookkeeping.  No static shared memory, so the tables sit at
    // a fixed offset of the CTA's shared window (SDDG_SMEM_ABS, fastmath.cuh).
    extern __shared__ double dyn_smem[];
    fm::FmTables& T = *reinterpret_cast<fm::FmTables*>(dyn_smem);
#ifdef SDDG_SMEM_ABS
    if constexpr (walk_uses_tables<DV, Real>()) {
        const uint32_t at = static_cast<uint32_t>(__cvta_generic_to_shared(dyn_smem));
        if (at != static_cast<uint32_t>(SDDG_SMEM_ABS)) {
            if (threadIdx.x == 0) {
                atomicCAS(a.err_flag, 0, 5);
                atomicExch(a.err_info, static_cast<unsigned long long>(at));
            }
            return;
        }
    }
#endif
    if constexpr (walk_uses_tables<DV, Real>()) {
        const double2* src = reinterpret_cast<const double2*>(a.fm_tables);
        double2* dst = reinterpret_cast<double2*>(dyn_smem);
        for (int k = threadIdx.x; k < static_cast<int>(sizeof(fm::FmTables) / 16); k += blockDim.x)
            dst[k] = src[k];
        __syncthreads();
    }

    // Per-walk bookkeeping that only the rare exit / restart paths touch
    // (record slot, node, walk, epoch, step total) lives in shared memory, so
    // the step loop keeps its 64 registers for the step itself.
    LaneState* lane_state = reinterpret_cast<LaneState*>(
        reinterpret_cast<char*>(dyn_smem) + walk_table_bytes<DV, Real>());
    LaneState& L = lane_state[threadIdx.x];
    L.g = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    L.steps = 0;
    // drain round: walk ci of the previous round's handoffs, 32 per warp, the
    // warps dealt round-robin over the CTAs (one CTA per SM)
    uint32_t ci = 0;
    bool have = L.g < a.total;
    if constexpr (DRAIN) {
        {
            ci = (((threadIdx.x >> 5) * gridDim.x + blockIdx.x) << 5) + (threadIdx.x & 31);
            have = ci < min(*a.n_src, a.src_cap);
        }
    }
    if (have) {
        Real x, y;
        LaneStream rng;
        // ---- walk setup (re-entered for every new walk)
        auto start_walk = [&](uint64_t g) {
            const uint64_t slot = g / static_cast<uint64_t>(a.walks);
            const uint32_t node = a.perm ? a.perm[slot] : static_cast<uint32_t>(slot);
            SDDG_CHECK(g < a.total && node < static_cast<uint64_t>(a.n_nodes));
            L.node = node;
            L.walk = static_cast<uint32_t>(a.walk_lo + (g - slot * a.walks));
            L.epoch = 0;
            if constexpr (TAIL) L.base = 0;
            x = Real(a.px[node]);
            y = Real(a.py[node]);
            rng.init(a.rk, a.pid[node], L.walk, 0);
        };
        bool resumed = false;
        if constexpr (DRAIN) {
            {
                // the walk as handed over at a check point: position, stream
                // position (and the cached half block of an odd one), chunks done
                const WalkCont c = a.src[ci];
                SDDG_CHECK(c.g < a.total && c.node < static_cast<uint64_t>(a.n_nodes) && c.epoch < 1024u &&
                           c.step < max_steps && c.step % a.chunk32 == 0);
                L.g = c.g;
                L.node = c.node;
                L.walk = c.walk;
                L.epoch = c.epoch;
                L.base = c.step;
                x = Real(c.x);
                y = Real(c.y);
                rng.init(a.rk, a.pid[c.node], c.walk, c.epoch);
                rng.n = c.n;
                if (c.n & 1u) {
                    const PhiloxWords w = rng.block(a.rk, c.n >> 1);
                    rng.cw2 = w.w2;
                    rng.cw3 = w.w3;
                }
                resumed = true;
            }
        }
        if (!resumed) start_walk(L.g);
        bool in_box = box_test<DV, Real>(dom, x, y);
        uint32_t step = 0;
        // `step` counts the steps of the current chunk of a.chunk32 steps;
        // L.base the chunks completed in this epoch.  The loop's only compare
        // is the one it always had (a.chunk32 = max_steps without the tail
        // kernel); with it, a.chunk32 divides max_steps and each chunk end is
        // a handoff check point.
        const uint32_t chunk = a.chunk32;
        SDDG_UNROLL(SDDG_WALK_UNROLL)  // 2: step copies alternate x, y registers (no loop-carried moves)
        for (;;) {
            // ---- one step (step_drift, step_rand, step_update: shared with the
            // tail kernel so both compute every step bit for bit alike)
            Real nxp, nyp;
            bool ok;
            Real wl = Real(1);  // literal SDE: w at the step's start (the bridge's time scale)
            {
                uint64_t w0, w1, w2 = 0;
                if constexpr (SCHEME == 0) {
                    rng.next_pair(a.rk, w0, w1);
                } else {
                    w0 = rng.next_one(a.rk);
                    rng.next_pair(a.rk, w1, w2);
                }
                const StepRand<Real> r = step_rand<DV, Real, SCHEME>(T, a, sq2dt, w0, w1, w2);
                const StepDrift<Real> sd = step_drift<DV, Real, SCHEME>(T, P, dt, x, y);
                ok = sd.ok;
                if constexpr (kLiteral<DV>) wl = sd.w;
                step_update<DV, Real, SCHEME>(sd, r, dt, sq2dt, x, y, nxp, nyp);
            }
            ++step;
            if (!ok) {
                atomicCAS(a.err_flag, 0, 3);  // EvaluationError
                atomicExch(a.err_info, static_cast<unsigned long long>(a.pid[L.node]));
                break;
            }
            Real hx = Real(0), hy = Real(0);
            int edge = 0;
            bool nb;
            const bool exited = exit_test<DV, Real, SCHEME, BRIDGE>(
                dom, a, T, kLiteral<DV> ? thr * wl : thr, kLiteral<DV> ? dt * wl : dt, x, y, nxp, nyp, in_box, rng,
                hx, hy, edge, nb);
            if (!exited) {
                x = nxp;
                y = nyp;
                in_box = nb;
                if (step < (TAIL ? chunk : max_steps)) continue;
                const uint32_t done = TAIL ? L.base + step : step;  // steps of this epoch
                if (TAIL && done < max_steps) {
                    // handoff check point: once the batch counter has run out
                    // and few walks remain, the walk moves to the tail kernel,
                    // which runs it on a whole warp at a fraction of a lane's
                    // step latency (walk_tail.cuh)
                    L.base = done;
                    step = 0;
                    if (*reinterpret_cast<volatile unsigned long long*>(a.next) >= a.total &&
                        *reinterpret_cast<volatile unsigned long long*>(a.live) <= a.cont_cap) {
                        const uint32_t k = atomicAdd(a.n_cont, 1u);
                        SDDG_CHECK(done < max_steps);
                        if (k < a.cont_cap) {
                            WalkCont& c = a.cont[k];
                            c.x = static_cast<double>(x);
                            c.y = static_cast<double>(y);
                            c.g = L.g;
                            c.node = L.node;
                            c.walk = L.walk;
                            c.epoch = L.epoch;
                            c.step = done;
                            c.n = rng.n;
                            break;
                        }
                    }
                    continue;
                }
                // max_steps reached: restart on the next epoch's stream
                L.steps += done;
                const uint32_t epoch = ++L.epoch;
                const uint32_t node = L.node;
                if (epoch >= 1024u) {
                    atomicCAS(a.err_flag, 0, 4);  // NumericalError
                    atomicExch(a.err_info, static_cast<unsigned long long>(a.pid[node]));
                    break;
                }
                rng.init(a.rk, a.pid[node], L.walk, epoch);
                x = Real(a.px[node]);
                y = Real(a.py[node]);
                in_box = box_test<DV, Real>(dom, x, y);
                if constexpr (TAIL) L.base = 0;
                step = 0;
                continue;
            }
            // ---- exit: boundary values, record, next walk
            const uint32_t walk_steps = TAIL ? L.base + step : step;
            L.steps += walk_steps;
            record_exit<Real>(a, L.g, L.node, L.epoch, walk_steps, edge, hx, hy, max_steps);
            const uint64_t gn = atomicAdd(a.next, 1ull);
            if (gn >= a.total) {
                if constexpr (TAIL) atomicAdd(a.live, ~0ull);  // one walk fewer in flight (-1)
                break;
            }
            L.g = gn;
            start_walk(gn);
            in_box = box_test<DV, Real>(dom, x, y);
            step = 0;
        }
    }
    uint64_t my_steps = L.steps;
    // path-step count: warp sum, one atomic per warp
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) my_steps += __shfl_xor_sync(0xffffffffu, my_steps, o);
    if ((threadIdx.x & 31) == 0 && my_steps)
        atomicAdd(a.steps, static_cast<unsigned long long>(my_steps));
}

// All (SCHEME, BRIDGE) instantiations of one drift variant: dynamic shared
// memory = tables + one LaneState per thread.
template <int DV, typename Real>
constexpr size_t walk_smem() {
    return walk_table_bytes<DV, Real>() + sizeof(LaneState) * walk_block<DV, Real>();
}

template <int DV, typename Real, int SCHEME, bool BRIDGE, bool TAIL = false, bool DRAIN = false>
cudaError_t launch_one(const WalkArgs& a, int grid, cudaStream_t s, int block = 0) {
    constexpr size_t sm = walk_smem<DV, Real>();
    if constexpr (sm > 48 * 1024) {
        // once per device and variant (a process may drive several devices
        // from several host threads: setting it twice is harmless)
        static std::atomic<bool> attr[64];
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 64 || !attr[dev].load(std::memory_order_relaxed)) {
            const cudaError_t e = cudaFuncSetAttribute(walk_kernel<DV, Real, SCHEME, BRIDGE, TAIL, DRAIN>,
                                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                       static_cast<int>(sm));
            if (e != cudaSuccess) return e;
            if (dev >= 0 && dev < 64) attr[dev].store(true, std::memory_order_relaxed);
        }
    }
    // a drain round: CTAs of `block` threads, smem for their lanes only
    const int blk = DRAIN ? std::min(block, kDrainBlock) : walk_block<DV, Real>();
    walk_kernel<DV, Real, SCHEME, BRIDGE, TAIL, DRAIN>
        <<<grid, blk, walk_table_bytes<DV, Real>() + sizeof(LaneState) * blk, s>>>(a);
    return cudaGetLastError();
}

}  // namespace sddg

#include "walk_tail.cuh"

namespace sddg {

template <int DV, typename Real>
cudaError_t launch_variant(const WalkArgs& a, int grid, cudaStream_t s, int block = 0) {
    if constexpr (kTailHandoff<Real>) {
        if (a.src) {
            if (a.scheme == SDDG_SCHEME_EXPONENTIAL) return launch_one<DV, Real, 1, false, true, true>(a, grid, s, block);
            if (a.bridge) return launch_one<DV, Real, 0, true, true, true>(a, grid, s, block);
            return launch_one<DV, Real, 0, false, true, true>(a, grid, s, block);
        }
        if (a.cont) {
            if (a.scheme == SDDG_SCHEME_EXPONENTIAL) return launch_one<DV, Real, 1, false, true>(a, grid, s);
            if (a.bridge) return launch_one<DV, Real, 0, true, true>(a, grid, s);
            return launch_one<DV, Real, 0, false, true>(a, grid, s);
        }
    }
    if (a.scheme == SDDG_SCHEME_EXPONENTIAL) return launch_one<DV, Real, 1, false>(a, grid, s);
    if (a.bridge) return launch_one<DV, Real, 0, true>(a, grid, s);
    return launch_one<DV, Real, 0, false>(a, grid, s);
}

// The tail kernel after K1 on the same stream (fp64, a.cont set)
template <int DV, typename Real>
cudaError_t launch_tail_variant(const WalkArgs& a, cudaStream_t s) {
    if constexpr (kTailHandoff<Real>) {
        if (a.scheme == SDDG_SCHEME_EXPONENTIAL) return launch_tail_one<DV, Real, 1, false>(a, s);
        if (a.bridge) return launch_tail_one<DV, Real, 0, true>(a, s);
        return launch_tail_one<DV, Real, 0, false>(a, s);
    }
    return cudaErrorInvalidValue;
}

// CTAs per SM and threads per CTA of the variant's bridge-test kernel
template <int DV, typename Real>
cudaError_t occupancy_variant(int* b, int* block) {
    constexpr size_t sm = walk_smem<DV, Real>();
    *block = walk_block<DV, Real>();
    if constexpr (sm > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(walk_kernel<DV, Real, 0, true>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(sm));
        if (e != cudaSuccess) return e;
    }
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(b, walk_kernel<DV, Real, 0, true>,
                                                         walk_block<DV, Real>(), sm);
}

}  // namespace sddg
