// physics.cuh — device physics shared by the transport and primary kernels:
// vector algebra, the interaction cross sections and samplers' helpers
// (REF cross_sections.cpp, samplers.cpp, material.cpp:253-271) and the
// Siddon ray set-up (REF trace.cpp:29-103).  Expression order follows the
// reference (the library is compiled with -fmad=false).
#pragma once

#include <math_constants.h>

#include "xs_device.cuh"

namespace xsd {

// Out-of-line fp64 libm calls: each inlined copy is 50-150 SASS instructions,
// and the persistent transport kernel is instruction-cache bound when they
// are replicated at every call site (profiles/README.md).
static __device__ __noinline__ double nl_log(double x) { return log(x); }
static __device__ __noinline__ double nl_exp(double x) { return exp(x); }
static __device__ __noinline__ double nl_sin(double x) { return sin(x); }
static __device__ __noinline__ double nl_cos(double x) { return cos(x); }
static __device__ __noinline__ double nl_acos(double x) { return acos(x); }

struct V3 {
    double x, y, z;
};

__device__ __forceinline__ V3 v3(double x, double y, double z) { return V3{x, y, z}; }
__device__ __forceinline__ V3 operator+(V3 a, V3 b) { return v3(a.x + b.x, a.y + b.y, a.z + b.z); }
__device__ __forceinline__ V3 operator-(V3 a, V3 b) { return v3(a.x - b.x, a.y - b.y, a.z - b.z); }
__device__ __forceinline__ V3 operator*(V3 a, double s) { return v3(a.x * s, a.y * s, a.z * s); }
__device__ __forceinline__ V3 operator/(V3 a, double s) { return v3(a.x / s, a.y / s, a.z / s); }
__device__ __forceinline__ double dot(V3 a, V3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
__device__ __forceinline__ V3 cross(V3 a, V3 b)
{
    return v3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ V3 normalized(V3 v) { return v / sqrt(dot(v, v)); }

// REF samplers.cpp:127-134
__device__ __forceinline__ V3 rotate_direction(V3 dir, double theta, double phi)
{
    const V3 pick = fabs(dir.x) < 0.5 ? v3(1.0, 0.0, 0.0) : v3(0.0, 1.0, 0.0);
    const V3 e1 = normalized(cross(dir, pick));
    const V3 e2 = cross(dir, e1);
    const double st = nl_sin(theta), ct = nl_cos(theta);
    return normalized(dir * ct + (e1 * nl_cos(phi) + e2 * nl_sin(phi)) * st);
}

// ------------------------------------------------------------ physics helpers
__device__ __forceinline__ double momentum_transfer(double e, double theta)
{
    return nl_sin(0.5 * theta) * e / kHc; // cross_sections.cpp:19-22
}

__device__ __forceinline__ double compton_ratio(double e, double theta)
{
    const double alpha = e / kMec2; // cross_sections.cpp:24-28
    return 1.0 / (1.0 + alpha * (1.0 - nl_cos(theta)));
}

__device__ __forceinline__ double kn_core(double e, double theta)
{
    const double ratio = compton_ratio(e, theta);
    const double s = nl_sin(theta);
    return ratio * ratio * (ratio + 1.0 / ratio - s * s);
}

__device__ __forceinline__ Tab mtab(const TransportParams& P, TabDesc d) { return tab_at(P.tabs, d); }

// material.cpp:253-261
__device__ __forceinline__ double form_S(const TransportParams& P, const MatDesc& m, double q)
{
    const Tab t = mtab(P, m.s);
    if (q >= __ldg(t.x + t.n - 1))
        return m.z_eff;
    double y = 0.0;
    tab_linear(t, q, y);
    return y;
}

__device__ __forceinline__ double form_F(const TransportParams& P, const MatDesc& m, double q)
{
    return tab_linear_clamped(mtab(P, m.f), q);
}

static __device__ __noinline__ double loglog_or_fail(const TransportParams& P, TabDesc d, double e,
                                                 DevStatus* st, int bin)
{
    double y = 0.0;
    if (!tab_loglog(mtab(P, d), e, y))
        raise(st, XS_E_OUT_OF_RANGE, kErrTableRange, bin, e, 0.0);
    return y;
}

// samplers.cpp:56-88
__device__ __forceinline__ double segment_mass(double q0, double a, double b, double u)
{
    const double c0 = a * a, c1 = 2.0 * a * b, c2 = b * b;
    return 2.0 * (c0 * q0 * u + (c0 + c1 * q0) * u * u / 2.0 + (c1 + c2 * q0) * u * u * u / 3.0 +
                  c2 * u * u * u * u / 4.0);
}

static __device__ double cumulative_mass(const TransportParams& P, const MatDesc& m, double q)
{
    const double* knots = P.tabs + m.f.off;
    const double* fv = knots + m.f.n;
    const double* cdf = P.tabs + m.cdf_off;
    const int n = m.f.n;
    const double k_last = __ldg(knots + n - 1);
    if (q >= k_last) {
        const double f_last = __ldg(fv + n - 1);
        return __ldg(cdf + n - 1) + f_last * f_last * (q * q - k_last * k_last);
    }
    int lo = 0, hi = n - 1;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(knots + mid) <= q)
            lo = mid;
        else
            hi = mid;
    }
    const double k0 = __ldg(knots + lo), k1 = __ldg(knots + lo + 1);
    const double a = __ldg(fv + lo);
    const double b = (__ldg(fv + lo + 1) - a) / (k1 - k0);
    return __ldg(cdf + lo) + segment_mass(k0, a, b, q - k0);
}

// REF's 64-step bisection, bit for bit: every probe evaluates exactly
// cumulative_mass(mid).  The knot segment of mid lies between those of the
// bracket ends, so the segment search is confined to that range (empty once
// the bracket sits in one segment) and a segment's coefficients are loaded
// (and its slope divided) only when the probe moves to another segment.
static __device__ double invert_mass(const TransportParams& P, const MatDesc& m, double target, double q_hi)
{
    const double* knots = P.tabs + m.f.off;
    const double* fv = knots + m.f.n;
    const double* cdf = P.tabs + m.cdf_off;
    const int n = m.f.n;
    const double k_last = __ldg(knots + n - 1);
    const double f_last = __ldg(fv + n - 1);
    const double c_last = __ldg(cdf + n - 1);
    int s_lo = 0, s_hi = n - 1; // segments of the bracket ends (n - 1: at/after the last knot)
    int seg = -1;               // segment whose coefficients are loaded
    double k0 = 0.0, a = 0.0, b = 0.0, c0 = 0.0;
    double lo = 0.0, hi = q_hi;
#pragma unroll 1
    for (int it = 0; it < 64; ++it) {
        const double mid = 0.5 * (lo + hi);
        double cm;
        int s_mid;
        if (mid >= k_last) {
            s_mid = n - 1;
            cm = c_last + f_last * f_last * (mid * mid - k_last * k_last);
        } else {
            int l = s_lo, h = s_hi < n - 1 ? s_hi + 1 : n - 1; // knots[l] <= mid < knots[h]
            while (h - l > 1) {
                const int md = (l + h) >> 1;
                if (__ldg(knots + md) <= mid)
                    l = md;
                else
                    h = md;
            }
            s_mid = l;
            if (l != seg) {
                seg = l;
                k0 = __ldg(knots + l);
                const double k1 = __ldg(knots + l + 1);
                a = __ldg(fv + l);
                b = (__ldg(fv + l + 1) - a) / (k1 - k0);
                c0 = __ldg(cdf + l);
            }
            cm = c0 + segment_mass(k0, a, b, mid - k0);
        }
        if (cm < target) {
            lo = mid;
            s_lo = s_mid;
        } else {
            hi = mid;
            s_hi = s_mid;
        }
    }
    return 0.5 * (lo + hi);
}

// REF clip_to_grid (trace.cpp:29-56); returns false for a miss.
// FAST: multiply by the reciprocal direction instead of dividing (the
// macro-cell mode, which already differs from REF at rounding level);
// otherwise REF's exact divisions.
template <bool FAST = false>
__device__ __forceinline__ bool clip_to_grid(const Grid& G, V3 o, V3 d, double& t0, double& t1,
                                             bool& bad)
{
    bad = !(isfinite(o.x) && isfinite(o.y) && isfinite(o.z) && isfinite(d.x) && isfinite(d.y) &&
            isfinite(d.z));
    if (bad)
        return false;
    t0 = 0.0;
    t1 = CUDART_INF;
    const double oo[3] = {o.x, o.y, o.z};
    const double dd[3] = {d.x, d.y, d.z};
    const double l[3] = {G.ox, G.oy, G.oz};
    const double h[3] = {G.ux, G.uy, G.uz};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        if (dd[a] == 0.0) {
            if (oo[a] < l[a] || oo[a] >= h[a])
                return false;
            continue;
        }
        double ta, tb;
        if (FAST) {
            const double r = 1.0 / dd[a];
            ta = (l[a] - oo[a]) * r;
            tb = (h[a] - oo[a]) * r;
        } else {
            ta = (l[a] - oo[a]) / dd[a];
            tb = (h[a] - oo[a]) / dd[a];
        }
        if (ta > tb) {
            const double s = ta;
            ta = tb;
            tb = s;
        }
        t0 = t0 < ta ? ta : t0; // std::max(t0, ta)
        t1 = tb < t1 ? tb : t1;
    }
    return t0 < t1;
}

template <bool FAST = false>
__device__ __forceinline__ void start_axis(double p, double o, double d, double org, double hs,
                                           double inv_h, int n, double t0, int& idx, int& step,
                                           double& tn, double& dt)
{
    idx = voxel_of(p, org, inv_h, n);
    const double r = FAST && d != 0.0 ? 1.0 / d : 0.0;
    if (d > 0.0) {
        step = 1;
        dt = FAST ? hs * r : hs / d;
        tn = FAST ? (org + (idx + 1) * hs - o) * r : (org + (idx + 1) * hs - o) / d;
    } else if (d < 0.0) {
        step = -1;
        dt = FAST ? -hs * r : -hs / d;
        tn = FAST ? (org + idx * hs - o) * r : (org + idx * hs - o) / d;
    } else { // (FAST, the block walk: finite sentinels, see cross_n)
        step = 0;
        dt = FAST ? 1e300 : CUDART_INF;
        tn = FAST ? 1e300 : CUDART_INF;
    }
    while (tn <= t0 && step != 0) {
        idx += step;
        tn += dt;
    }
    // REF leaves an out-of-grid index here only in degenerate tangent cases
    // (it would then read outside the grid); keep the device read in bounds.
    idx = idx < 0 ? 0 : (idx > n - 1 ? n - 1 : idx);
}


} // namespace xsd
